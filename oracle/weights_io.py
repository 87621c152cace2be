"""Oracle's own reader of the weight file (test infrastructure only).

File layout: see synth/weights.py (the file is the contract, SURVEY.md §8(c)
reading row 9).  This reader shares no code with the writer or with the CUDA
library's C++ reader.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

from . import irreps


@dataclass
class Model:
    n_layers: int
    lmax: int
    C: int
    D: int
    n_basis: int
    n_species: int
    p: int
    two_body: tuple
    edge_hidden: int
    r_max: float
    nbar: float
    sigma: np.ndarray
    mu: np.ndarray
    t: dict = field(default_factory=dict)  # name -> float64 array
    specs: list = field(default_factory=list)


def read(path: str) -> Model:
    with open(path, "rb") as f:
        buf = f.read()
    if buf[:4] != b"ALGW":
        raise ValueError("bad magic")
    (version,) = struct.unpack_from("<i", buf, 4)
    if version != 1:
        raise ValueError("bad version")
    ints = struct.unpack_from("<12i", buf, 8)
    L, lmax, C, D, nb, ns, p, t0, t1, t2, eh, nt = ints
    off = 8 + 48
    r_max, nbar, s0, s1, m0, m1 = struct.unpack_from("<6d", buf, off)
    off += 48
    tensors = {}
    for _ in range(nt):
        name = buf[off : off + 32].split(b"\0")[0].decode()
        off += 32
        (ndim,) = struct.unpack_from("<i", buf, off)
        off += 4
        shape = struct.unpack_from(f"<{ndim}i", buf, off)
        off += 4 * ndim
        count = int(np.prod(shape))
        tensors[name] = np.frombuffer(buf, dtype="<f8", count=count, offset=off).reshape(shape).copy()
        off += 8 * count
    m = Model(L, lmax, C, D, nb, ns, p, (t0, t1, t2), eh, r_max, nbar, np.array([s0, s1]), np.array([m0, m1]), tensors)
    m.specs = irreps.layer_specs(L, lmax)
    # independent check of the file's tensor shapes against this side's derivation
    n_env = lmax + 1
    for spec in m.specs:
        k = spec.k
        if tensors[f"env_{k}"].shape != (D, C * n_env * (2 if k == 0 else 1)):
            raise ValueError(f"env_{k} shape mismatch")
        n_paths = sum(1 for nm in tensors if nm.startswith(f"tplin_{k}_"))
        if n_paths != len(spec.paths):
            raise ValueError(f"layer {k}: {n_paths} TP-linear tensors, expected {len(spec.paths)}")
        if tensors[f"lat_{k}"].shape != (D + C * spec.n_scalar, D):
            raise ValueError(f"lat_{k} shape mismatch")
    total = sum(v.size for v in tensors.values())
    if total != irreps.param_count(L, lmax, C, D, nb, (t0, t1, t2), eh, ns):
        raise ValueError("parameter count mismatch")
    return m
