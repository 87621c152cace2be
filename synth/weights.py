"""Random-init Allegro weight files (the binary file is the contract).

The paper ships no weights (§2.4 -- a TorchScript file); the
build uses seeded U(-sqrt3, sqrt3) weights of the architecture recovered from
Table 2's parameter counts.

This module only draws numbers and writes them in a fixed order.  The tensor
*shapes* come from the hard-coded table ``ARCH`` below, copied from SURVEY.md
App. A/B (number of tensor-product paths and of scalar paths per layer).  Both
the oracle and the CUDA library re-derive these counts independently from the
irreps rules and reject a file that disagrees.

File layout (little endian):

    char[4]  magic "ALGW";  int32 version = 1
    int32    n_layers, lmax, C, D, n_basis, n_species, p_envelope,
             tb0, tb1, tb2 (two-body widths), edge_hidden, n_tensors
    float64  r_max, nbar, sigma[2], mu[2]
    n_tensors x { char[32] name; int32 ndim; int32 shape[ndim]; float64 data[] }

Tensor order (SURVEY.md App. A "Weight-file tensor order"):
    bessel_freq[8] (n*pi), tb_w0[12,32], tb_w1[32,64], tb_w2[64,128],
    for k in 0..L-1: env_k[128, n_w(k)], tplin_k_p[32,32] for each path p,
                     lat_k[128 + 32*n_s(k), 128],
    out_w1[128,32], out_w2[32,1]
"""
from __future__ import annotations

import json
import math
import os
import struct

import numpy as np

MAGIC = b"ALGW"
VERSION = 1
C_CHANNELS = 32
D_LATENT = 128
N_BASIS = 8
N_SPECIES = 2
P_ENVELOPE = 6
TWO_BODY = (32, 64, 128)
EDGE_HIDDEN = 32

# (n_layers, lmax) -> per-layer (#TP paths, #scalar paths).  Copied from
# SURVEY.md App. B (o3_full with backward pruning); verified independently by
# oracle.irreps and by the CUDA library's own derivation.
ARCH = {
    (2, 1): ((4, 2), (2, 2)),  # C1: 94,632 params
    (2, 2): ((11, 3), (3, 3)),  # C2: 123,304
    (3, 2): ((15, 3), (15, 3), (3, 3)),  # C3: 183,720 (paper's l=2 model)
    (3, 1): ((5, 2), (5, 2), (2, 2)),  # paper's l=1 production model: 133,544
    (3, 0): ((1, 1), (1, 1), (1, 1)),  # paper's l=0 model: 95,656
}

_CAL_PATH = os.path.join(os.path.dirname(__file__), "calibration.json")


def nbar_for(r_cut: float) -> float:
    """Mean directed neighbours per atom at liquid-NH3 density:
    n_bar = rho_atoms * (4/3) pi r_c^3 (reading D6 in
    DESIGN.md).  A constant of the input recipe, not of the method."""
    rho_atoms = 4.0 * 0.025813
    return rho_atoms * 4.0 / 3.0 * math.pi * r_cut**3


def tensor_list(n_layers: int, lmax: int):
    """[(name, shape)] in file order for the ARCH entry."""
    paths = ARCH[(n_layers, lmax)]
    n_env = lmax + 1
    out = [("bessel_freq", (N_BASIS,))]
    dims = (2 * N_SPECIES + N_BASIS,) + TWO_BODY
    for i in range(3):
        out.append((f"tb_w{i}", (dims[i], dims[i + 1])))
    for k in range(n_layers):
        n_paths, n_s = paths[k]
        n_w = C_CHANNELS * n_env * (2 if k == 0 else 1)
        out.append((f"env_{k}", (D_LATENT, n_w)))
        for p in range(n_paths):
            out.append((f"tplin_{k}_{p}", (C_CHANNELS, C_CHANNELS)))
        out.append((f"lat_{k}", (D_LATENT + C_CHANNELS * n_s, D_LATENT)))
    out.append(("out_w1", (D_LATENT, EDGE_HIDDEN)))
    out.append(("out_w2", (EDGE_HIDDEN, 1)))
    return out


def generate(n_layers: int, lmax: int, seed: int = 0):
    """Seeded tensors: Bessel frequencies n*pi, every weight U(-sqrt3, sqrt3)
    drawn from ``default_rng(seed)`` in file order."""
    rng = np.random.default_rng(seed)
    s3 = math.sqrt(3.0)
    tensors = []
    for name, shape in tensor_list(n_layers, lmax):
        if name == "bessel_freq":
            t = math.pi * np.arange(1, N_BASIS + 1, dtype=np.float64)
        else:
            t = rng.uniform(-s3, s3, size=shape)
        tensors.append((name, np.ascontiguousarray(t, dtype=np.float64)))
    return tensors


def load_calibration():
    if not os.path.exists(_CAL_PATH):
        return {}
    with open(_CAL_PATH) as f:
        return json.load(f)


def model_key(n_layers: int, lmax: int, r_cut: float, seed: int) -> str:
    return f"L{n_layers}_l{lmax}_rc{r_cut:g}_s{seed}"


def write(path, n_layers, lmax, r_cut, tensors, nbar, sigma=(1.0, 1.0), mu=(0.0, 0.0)):
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<i", VERSION))
        f.write(
            struct.pack(
                "<12i",
                n_layers,
                lmax,
                C_CHANNELS,
                D_LATENT,
                N_BASIS,
                N_SPECIES,
                P_ENVELOPE,
                TWO_BODY[0],
                TWO_BODY[1],
                TWO_BODY[2],
                EDGE_HIDDEN,
                len(tensors),
            )
        )
        f.write(struct.pack("<6d", r_cut, nbar, sigma[0], sigma[1], mu[0], mu[1]))
        for name, t in tensors:
            nb = name.encode()
            f.write(nb + b"\0" * (32 - len(nb)))
            f.write(struct.pack("<i", t.ndim))
            f.write(struct.pack(f"<{t.ndim}i", *t.shape))
            f.write(np.ascontiguousarray(t, dtype="<f8").tobytes())


def make_weight_file(path, n_layers, lmax, r_cut, seed=0, sigma=None):
    """Write the weight file of model (n_layers, lmax) at cutoff r_cut.

    sigma: None -> the calibrated value from calibration.json (written by
    scripts/calibrate_sigma.py, which calls only oracle/), else 1.0 when
    uncalibrated."""
    if sigma is None:
        sigma = load_calibration().get(model_key(n_layers, lmax, r_cut, seed), 1.0)
    tensors = generate(n_layers, lmax, seed)
    write(path, n_layers, lmax, r_cut, tensors, nbar_for(r_cut), (sigma, sigma), (0.0, 0.0))
    return path
