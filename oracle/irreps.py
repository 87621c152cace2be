"""Irreps, tensor-product paths and parameter counts (oracle; test infrastructure only).

PAPER.md:130 (§2.1) -- "tensors up to rank l and tensor products using their
irreducible representations" -- and Table 2 (§4.1), whose
parameter counts 95,656 / 133,544 / 183,720 for l = 0 / 1 / 2 pin the
architecture (reading rows 2 and 7):

* irreps are (l, p), p = +1 (even, 'e') or -1 (odd, 'o'); ordered by l
  ascending, even before odd.
* SH irreps: (l, (-1)^l) for l <= lmax.
* layer k's TP couples V^k (irreps in_k) with the environment Gamma (SH irreps);
  a path (ir1, ir2 -> ir_o) exists iff p1*p2 = p_o and |l1-l2| <= l_o <= l1+l2.
* ``o3_full``: out_k = every irrep with l <= lmax reachable from in_k x SH; the
  last layer outputs 0e only; then backward pruning keeps, in out_k = in_{k+1},
  only irreps used by some path of layer k+1.
* path order: for ir_o in out_k: for ir1 in in_k: for ir2 in SH.
"""
from __future__ import annotations

from dataclasses import dataclass

C_DEFAULT = 32
D_DEFAULT = 128


def irrep_key(ir):
    l, p = ir
    return (l, 0 if p == 1 else 1)


def irrep_name(ir) -> str:
    return f"{ir[0]}{'e' if ir[1] == 1 else 'o'}"


def irrep_dim(ir) -> int:
    return 2 * ir[0] + 1


def sh_irreps(lmax: int):
    return [(l, (-1) ** l) for l in range(lmax + 1)]


def _allowed(ir1, ir2, iro) -> bool:
    return ir1[1] * ir2[1] == iro[1] and abs(ir1[0] - ir2[0]) <= iro[0] <= ir1[0] + ir2[0]


def _paths(in_irreps, out_irreps, sh):
    out = []
    for iro in out_irreps:
        for ir1 in in_irreps:
            for ir2 in sh:
                if _allowed(ir1, ir2, iro):
                    out.append((ir1, ir2, iro))
    return out


@dataclass
class LayerSpec:
    k: int
    in_irreps: list  # irreps of V^k
    out_irreps: list  # irreps of the TP output of layer k (= V^{k+1} irreps)
    paths: list  # [(ir1, ir2, ir_o)]

    @property
    def n_scalar(self) -> int:
        return sum(1 for p in self.paths if p[2] == (0, 1))


def layer_specs(n_layers: int, lmax: int):
    sh = sh_irreps(lmax)
    all_ir = sorted([(l, p) for l in range(lmax + 1) for p in (1, -1)], key=irrep_key)
    # forward reachability
    ins = [list(sh)]
    outs = []
    for k in range(n_layers):
        if k == n_layers - 1:
            o = [(0, 1)]
        else:
            o = [iro for iro in all_ir if any(_allowed(a, b, iro) for a in ins[k] for b in sh)]
        outs.append(o)
        ins.append(o)
    # backward pruning: keep in out_k only irreps used by a path of layer k+1
    for k in range(n_layers - 2, -1, -1):
        used = {p[0] for p in _paths(outs[k], outs[k + 1], sh)}
        outs[k] = [ir for ir in outs[k] if ir in used]
        ins[k + 1] = outs[k]
    return [LayerSpec(k, ins[k], outs[k], _paths(ins[k], outs[k], sh)) for k in range(n_layers)]


def param_count(n_layers: int, lmax: int, C: int = C_DEFAULT, D: int = D_DEFAULT, n_basis: int = 8,
                two_body=(32, 64, 128), edge_hidden: int = 32, n_species: int = 2) -> int:
    """Trainable parameters (SURVEY.md App. A counting model, no biases)."""
    n_env = lmax + 1
    total = n_basis
    dims = (2 * n_species + n_basis,) + tuple(two_body)
    total += sum(dims[i] * dims[i + 1] for i in range(len(dims) - 1))
    for spec in layer_specs(n_layers, lmax):
        total += D * C * n_env * (2 if spec.k == 0 else 1)
        total += len(spec.paths) * C * C
        total += (D + C * spec.n_scalar) * D
    total += D * edge_hidden + edge_hidden
    return total
