"""Independent float64 torch-autograd implementation of the Allegro energy
(TEST-ONLY second witness for the oracle's hand-written reverse mode).

Written from SURVEY.md §8(c) E1-E8 without calling any oracle function except
the pinned W3j table and the layer/path enumeration.  Forces come from
torch.autograd, not from a hand derivation.
"""
import math

import numpy as np
import torch

from oracle import so3


def _sh(r, lmax):
    d = torch.linalg.norm(r, dim=1, keepdim=True)
    n = r / d
    x, y, z = n[:, 0], n[:, 1], n[:, 2]
    out = [torch.ones_like(x)[:, None]]
    if lmax >= 1:
        out.append(math.sqrt(3) * torch.stack([y, z, x], 1))
    if lmax >= 2:
        s15, s5 = math.sqrt(15), math.sqrt(5)
        out.append(torch.stack([s15 * x * y, s15 * y * z, s5 / 2 * (3 * z * z - 1), s15 * x * z, s15 / 2 * (x * x - y * y)], 1))
    return torch.cat(out, 1)


def energy(model, pos, species, box, edges):
    """E(pos) as a differentiable torch function; pos is a float64 tensor [N,3]."""
    t = {k: torch.as_tensor(v) for k, v in model.t.items()}
    ei, ej, en = (torch.as_tensor(a) for a in edges)
    box_t = torch.as_tensor(box)
    spc = torch.as_tensor(np.asarray(species, dtype=np.int64))
    rc = model.r_max
    C, D = model.C, model.D
    rv = pos[ej] + en.double() * box_t - pos[ei]
    d = torch.linalg.norm(rv, dim=1)
    x = d / rc
    u = torch.where(x < 1, 1 - 28 * x**6 + 48 * x**7 - 21 * x**8, torch.zeros_like(x))
    B = (2 / rc) * torch.sin(t["bessel_freq"][None, :] * d[:, None] / rc) / d[:, None]
    z = torch.cat([torch.nn.functional.one_hot(spc[ei], 2).double(), torch.nn.functional.one_hot(spc[ej], 2).double(), u[:, None] * B], 1)
    c = 1.6765324703
    h = torch.nn.functional.silu(z @ t["tb_w0"] / math.sqrt(12))
    h = torch.nn.functional.silu(h @ t["tb_w1"] * c / math.sqrt(32))
    lat = u[:, None] * (h @ t["tb_w2"] * c / math.sqrt(64))
    Y = _sh(rv, model.lmax)
    n_env = model.lmax + 1
    lm_l = torch.as_tensor(np.concatenate([[l] * (2 * l + 1) for l in range(n_env)]))
    n_atoms = pos.shape[0]
    E = rv.shape[0]
    V = None
    for spec in model.specs:
        k = spec.k
        w = lat @ t[f"env_{k}"] / math.sqrt(D)
        if k == 0:
            w_edge = w[:, : C * n_env].reshape(E, C, n_env)
            w_env = w[:, C * n_env :].reshape(E, C, n_env)
            V = w_edge[:, :, lm_l] * Y[:, None, :]
        else:
            w_env = w.reshape(E, C, n_env)
        G = torch.zeros(n_atoms, C, Y.shape[1], dtype=torch.float64).index_add(0, ei, w_env[:, :, lm_l] * Y[:, None, :])
        G = G / math.sqrt(model.nbar)
        Ge = G[ei]
        # slices
        in_off, off = {}, 0
        for ir in spec.in_irreps:
            in_off[ir] = off
            off += 2 * ir[0] + 1
        sh_off = {(l, (-1) ** l): l * l for l in range(n_env)}
        Ts, s_list = [], []
        for ir1, ir2, iro in spec.paths:
            W = torch.as_tensor(so3.w3j(ir1[0], ir2[0], iro[0]))
            a = V[:, :, in_off[ir1] : in_off[ir1] + 2 * ir1[0] + 1]
            b = Ge[:, :, sh_off[ir2] : sh_off[ir2] + 2 * ir2[0] + 1]
            Tp = math.sqrt(2 * iro[0] + 1) * torch.einsum("abk,eca,ecb->eck", W, a, b)
            Ts.append((iro, Tp))
        s = torch.cat([Tp for iro, Tp in Ts if iro == (0, 1)], 2)  # [E, C, n_s]
        s = s.reshape(E, -1)
        if k < model.n_layers - 1:
            parts = []
            for iro in spec.out_irreps:
                idx = [q for q, (o, _) in enumerate(Ts) if o == iro]
                acc = sum(torch.einsum("ecm,cv->evm", Ts[q][1], t[f"tplin_{k}_{q}"]) for q in idx)
                parts.append(acc / math.sqrt(C * len(idx)))
            V_next = torch.cat(parts, 2)
        hl = torch.cat([lat, s], 1) @ t[f"lat_{k}"] / math.sqrt(D + s.shape[1])
        lat = (2 * lat + u[:, None] * hl) / math.sqrt(5)
        if k < model.n_layers - 1:
            V = V_next
    Ee = (lat @ t["out_w1"] / math.sqrt(D) @ t["out_w2"] / math.sqrt(model.edge_hidden))[:, 0]
    sig = torch.as_tensor(model.sigma)[spc]
    mu = torch.as_tensor(model.mu)[spc]
    Ei = torch.zeros(n_atoms, dtype=torch.float64).index_add(0, ei, Ee) * sig / math.sqrt(model.nbar) + mu
    return Ei.sum()


def energy_forces(model, pos, species, box, edges):
    p = torch.tensor(pos, dtype=torch.float64, requires_grad=True)
    E = energy(model, p, species, box, edges)
    (g,) = torch.autograd.grad(E, p)
    return float(E.detach()), (-g).numpy()
