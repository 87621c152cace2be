"""Allegro energy and analytic forces in fp64 (oracle; test infrastructure only).

The paper states the model only as (§2.1): E is a sum of
pairwise embedding energies E_ij within a finite cutoff, E(3)-equivariant, built
from tensors up to rank l and tensor products of irreps; forces are
f_i = -dE/dr_i (Eq. 1).  Every concrete equation below is the
reading written out in SURVEY.md §8(c) E1-E9 (rows 1-8, 10, 20, 22 of its
readings table; DESIGN.md §3 lists them).  Steps are evaluated in the order of
that definition; the reverse mode is the one spelled out in E9.

  E1  u(d) = 1 - 28x^6 + 48x^7 - 21x^8, x = d/r_c (0 for x >= 1)
  E2  B_n(d) = (2/r_c) sin(b_n d / r_c) / d,  n = 1..8
  E3  Y^l(r_hat), component normalised (oracle.so3)
  E4  MLP: h_{k+1} = phi(h_k W_k gamma_k / sqrt(d_k)); gamma = c_SiLU after a SiLU
  E5  x0 = u * MLP_2b([onehot(Z_i), onehot(Z_j), u B])       (12 -> 32 -> 64 -> 128)
  E6  per layer k: w = x^k W_env / sqrt(D);  V^0 = w_edge (x) Y;
      Gamma_i = nbar^-1/2 sum_{e in row i} w_env (x) Y;
      T = sqrt(2 l_o + 1) W3j . V (x) Gamma_i (per channel, "uuu");
      s = scalar outputs;  V^{k+1} = per-irrep channel mix of T / sqrt(C n_->o);
      x^{k+1} = (2 x^k + u [x^k, s] W_lat / sqrt(D + C n_s)) / sqrt5
  E7  E_e = x^L W_o1 / sqrt(D) W_o2 / sqrt(32)
  E8  E_i = sigma_Z nbar^-1/2 sum_{row i} E_e + mu_Z;  E = sum_i E_i
  E9  g_e = dE/dr_e by reverse mode;  F_a = sum_{center a} g_e - sum_{nbr a} g_e

Centre atoms are processed in batches only to bound memory: each E_i depends on
its own row of edges alone.
"""
from __future__ import annotations

import math

import numpy as np

from . import neighbors, so3
from .irreps import irrep_dim

# c_SiLU = E[SiLU(z)^2]^(-1/2), z ~ N(0, 1)  (SURVEY.md §8(c) reading row 5;
# pinned by tests/test_oracle_model.py against numerical quadrature)
C_SILU = 1.6765324703
RES_A = 2.0 / math.sqrt(5.0)  # resnet ratio sigmoid(0) = 1/2: a = 1/sqrt(1+c^2), c = 1/2
RES_B = 1.0 / math.sqrt(5.0)  # b = c * a


# ---------------------------------------------------------------- E1, E2
def envelope(d, r_c):
    x = d / r_c
    u = 1.0 - 28.0 * x**6 + 48.0 * x**7 - 21.0 * x**8
    return np.where(x < 1.0, u, 0.0)


def envelope_deriv(d, r_c):
    x = d / r_c
    du = -(168.0 / r_c) * x**5 * (1.0 - x) ** 2
    return np.where(x < 1.0, du, 0.0)


def bessel(d, r_c, freq):
    arg = freq[None, :] * d[:, None] / r_c
    return (2.0 / r_c) * np.sin(arg) / d[:, None]


def bessel_deriv(d, r_c, freq):
    arg = freq[None, :] * d[:, None] / r_c
    dd = d[:, None]
    return (2.0 / r_c) * ((freq[None, :] / r_c) * np.cos(arg) / dd - np.sin(arg) / dd**2)


def silu(t):
    return t / (1.0 + np.exp(-t))


def silu_deriv(t):
    s = 1.0 / (1.0 + np.exp(-t))
    return s * (1.0 + t * (1.0 - s))


# ---------------------------------------------------------------- helpers
def _seg_sum(vals, seg, n):
    out = np.zeros((n,) + vals.shape[1:])
    np.add.at(out, seg, vals)
    return out


def _lm_to_l(lmax):
    return np.concatenate([np.full(2 * l + 1, l) for l in range(lmax + 1)])


def _slices(irreps_list):
    out, off = [], 0
    for ir in irreps_list:
        out.append(slice(off, off + irrep_dim(ir)))
        off += irrep_dim(ir)
    return out, off


def _path_tables(model, spec):
    """Slices and W3j for each path of a layer: (s1 in V, s2 in Y/Gamma, so in T, W, alpha)."""
    sh_ir = [(l, (-1) ** l) for l in range(model.lmax + 1)]
    in_sl, _ = _slices(spec.in_irreps)
    sh_sl, _ = _slices(sh_ir)
    out = []
    off = 0
    for ir1, ir2, iro in spec.paths:
        s1 = in_sl[spec.in_irreps.index(ir1)]
        s2 = sh_sl[sh_ir.index(ir2)]
        so = slice(off, off + irrep_dim(iro))
        off += irrep_dim(iro)
        out.append((s1, s2, so, so3.w3j(ir1[0], ir2[0], iro[0]), math.sqrt(2 * iro[0] + 1), iro))
    return out, off


# ---------------------------------------------------------------- batch
def _rows(model, rvec, zi, zj, seg, n_c, zc):
    """Forward E1-E8 and reverse E9 for a batch of complete rows.

    rvec [E,3] fp64, zi/zj species of centre/neighbour per edge, seg = local
    centre index per edge (0..n_c-1), zc = species of the n_c centres.
    Returns (E_atom_local [n_c] without mu, E_e [E], g [E,3])."""
    M = model
    t = M.t
    r_c = M.r_max
    C, D = M.C, M.D
    n_env = M.lmax + 1
    E = rvec.shape[0]
    inv_sqrt_nbar = 1.0 / math.sqrt(M.nbar)
    lm_l = _lm_to_l(M.lmax)

    # E1-E3 geometry
    d = np.linalg.norm(rvec, axis=1)
    u = envelope(d, r_c)
    B = bessel(d, r_c, t["bessel_freq"])
    Y = so3.sh(rvec, M.lmax)

    # E5 two-body
    onehot_i = np.eye(M.n_species)[zi]
    onehot_j = np.eye(M.n_species)[zj]
    z = np.concatenate([onehot_i, onehot_j, u[:, None] * B], axis=1)
    a1 = z @ t["tb_w0"] / math.sqrt(z.shape[1])
    h1 = silu(a1)
    a2 = h1 @ t["tb_w1"] * (C_SILU / math.sqrt(h1.shape[1]))
    h2 = silu(a2)
    mlp = h2 @ t["tb_w2"] * (C_SILU / math.sqrt(h2.shape[1]))
    x = u[:, None] * mlp

    # E6 layers (forward, caching what the reverse mode needs)
    cache = []
    V = None
    for spec in M.specs:
        k = spec.k
        w = x @ t[f"env_{k}"] / math.sqrt(D)
        if k == 0:
            w_edge = w[:, : C * n_env].reshape(E, C, n_env)
            w_env = w[:, C * n_env :].reshape(E, C, n_env)
            V = w_edge[:, :, lm_l] * Y[:, None, :]
        else:
            w_edge = None
            w_env = w.reshape(E, C, n_env)
        G = inv_sqrt_nbar * _seg_sum(w_env[:, :, lm_l] * Y[:, None, :], seg, n_c)  # [n_c, C, sh]
        Ge = G[seg]
        paths, t_dim = _path_tables(M, spec)
        T = np.zeros((E, C, t_dim))
        for s1, s2, so, W, alpha, _ in paths:
            T[:, :, so] = alpha * np.einsum("abk,eca,ecb->eck", W, V[:, :, s1], Ge[:, :, s2], optimize=True)
        n_s = spec.n_scalar
        s = T[:, :, :n_s].reshape(E, C * n_s)
        V_next = None
        if k < M.n_layers - 1:
            out_sl, v_dim = _slices(spec.out_irreps)
            V_next = np.zeros((E, C, v_dim))
            for o, iro in enumerate(spec.out_irreps):
                idx = [q for q, p in enumerate(paths) if p[5] == iro]
                norm = 1.0 / math.sqrt(C * len(idx))
                for q in idx:
                    so = paths[q][2]
                    V_next[:, :, out_sl[o]] += np.einsum("ecm,cv->evm", T[:, :, so], t[f"tplin_{k}_{q}"]) * norm
        xs = np.concatenate([x, s], axis=1)
        fan = math.sqrt(xs.shape[1])
        h = xs @ t[f"lat_{k}"] / fan
        x_next = RES_A * x + RES_B * u[:, None] * h
        cache.append(dict(spec=spec, w_edge=w_edge, w_env=w_env, V=V, G=G, paths=paths, h=h, fan=fan, n_s=n_s))
        x = x_next
        V = V_next

    # E7, E8
    wo = t["out_w1"] / math.sqrt(D)
    wo2 = t["out_w2"] / math.sqrt(M.edge_hidden)
    E_e = (x @ wo @ wo2)[:, 0]
    E_loc = M.sigma[zc] * inv_sqrt_nbar * _seg_sum(E_e, seg, n_c)

    # E9 reverse mode
    Ebar = M.sigma[zi] * inv_sqrt_nbar  # dE/dE_e
    xbar = Ebar[:, None] * (wo @ wo2)[:, 0][None, :]
    ubar = np.zeros(E)
    Ybar = np.zeros_like(Y)
    Vbar_next = None
    for k in range(M.n_layers - 1, -1, -1):
        c = cache[k]
        spec = c["spec"]
        # latent update x^{k+1} = a x^k + b u h
        ubar += RES_B * np.sum(c["h"] * xbar, axis=1)
        hbar = RES_B * u[:, None] * xbar
        xsbar = hbar @ t[f"lat_{k}"].T / c["fan"]
        xbar_k = RES_A * xbar + xsbar[:, :D]
        sbar = xsbar[:, D:]
        # TP-linear and scalars
        paths = c["paths"]
        t_dim = paths[-1][2].stop
        Tbar = np.zeros((E, C, t_dim))
        if k < M.n_layers - 1:
            out_sl, _ = _slices(spec.out_irreps)
            for o, iro in enumerate(spec.out_irreps):
                idx = [q for q, p in enumerate(paths) if p[5] == iro]
                norm = 1.0 / math.sqrt(C * len(idx))
                for q in idx:
                    so = paths[q][2]
                    Tbar[:, :, so] += np.einsum("evm,cv->ecm", Vbar_next[:, :, out_sl[o]], t[f"tplin_{k}_{q}"]) * norm
        Tbar[:, :, : c["n_s"]] += sbar.reshape(E, C, c["n_s"])
        # TP adjoints
        V = c["V"]
        Ge = c["G"][seg]
        Vbar = np.zeros_like(V)
        Gbar_e = np.zeros_like(Ge)
        for s1, s2, so, W, alpha, _ in paths:
            Vbar[:, :, s1] += alpha * np.einsum("abk,eck,ecb->eca", W, Tbar[:, :, so], Ge[:, :, s2], optimize=True)
            Gbar_e[:, :, s2] += alpha * np.einsum("abk,eck,eca->ecb", W, Tbar[:, :, so], V[:, :, s1], optimize=True)
        Gbar = _seg_sum(Gbar_e, seg, n_c)  # [n_c, C, sh]
        Gb = Gbar[seg]
        # environment adjoint
        w_env = c["w_env"]
        prod = Gb * Y[:, None, :]  # [E, C, sh]
        wbar_env = np.zeros((E, C, n_env))
        for l in range(n_env):
            wbar_env[:, :, l] = inv_sqrt_nbar * prod[:, :, lm_l == l].sum(axis=2)
        Ybar += inv_sqrt_nbar * np.sum(Gb * w_env[:, :, lm_l], axis=1)
        if k == 0:
            w_edge = c["w_edge"]
            prod = Vbar * Y[:, None, :]
            wbar_edge = np.zeros((E, C, n_env))
            for l in range(n_env):
                wbar_edge[:, :, l] = prod[:, :, lm_l == l].sum(axis=2)
            Ybar += np.sum(Vbar * w_edge[:, :, lm_l], axis=1)
            wbar = np.concatenate([wbar_edge.reshape(E, -1), wbar_env.reshape(E, -1)], axis=1)
        else:
            wbar = wbar_env.reshape(E, -1)
            Vbar_next = Vbar
        xbar = xbar_k + wbar @ t[f"env_{k}"].T / math.sqrt(D)

    # two-body reverse
    ubar += np.sum(mlp * xbar, axis=1)
    mbar = u[:, None] * xbar
    h2bar = mbar @ t["tb_w2"].T * (C_SILU / math.sqrt(h2.shape[1]))
    a2bar = h2bar * silu_deriv(a2)
    h1bar = a2bar @ t["tb_w1"].T * (C_SILU / math.sqrt(h1.shape[1]))
    a1bar = h1bar * silu_deriv(a1)
    zbar = a1bar @ t["tb_w0"].T / math.sqrt(z.shape[1])
    zb = zbar[:, 2 * M.n_species :]
    Bbar = u[:, None] * zb
    ubar += np.sum(zb * B, axis=1)

    # geometry reverse
    dbar = ubar * envelope_deriv(d, r_c) + np.sum(Bbar * bessel_deriv(d, r_c, t["bessel_freq"]), axis=1)
    g = dbar[:, None] * rvec / d[:, None] + np.einsum("el,elx->ex", Ybar, so3.sh_grad(rvec, M.lmax))
    return E_loc, E_e, g


def energy_forces(model, pos, species, box, centers=None, batch_edges: int = 60000, edges=None):
    """E, E_i and F for a periodic box (oracle definition E1-E9).

    centers: optional subset of centre atoms; then e_atom is NaN elsewhere and
    ``forces`` holds only the contributions of the computed rows (use
    ``sampled_forces`` for exact forces on a sample).
    Returns dict(energy, e_atom [N], forces [N,3], edges (i, j, n), g [E,3])."""
    box = np.asarray(box, dtype=np.float64)
    pos = neighbors.wrap(np.asarray(pos, dtype=np.float64), box)
    species = np.asarray(species, dtype=np.int64)
    n_atoms = pos.shape[0]
    if edges is None:
        ei, ej, en = neighbors.cell_list(pos, box, model.r_max, centers)
    else:
        ei, ej, en = edges
    rvec = neighbors.edge_vectors(pos, box, ei, ej, en)
    cs = np.arange(n_atoms) if centers is None else np.unique(np.asarray(centers))
    e_atom = np.full(n_atoms, np.nan)
    forces = np.zeros((n_atoms, 3))
    g_all = np.zeros((ei.shape[0], 3))
    # row boundaries (edges sorted by centre)
    starts = np.searchsorted(ei, cs, side="left")
    ends = np.searchsorted(ei, cs, side="right")
    b0 = 0
    while b0 < cs.size:
        b1 = b0
        n_e = 0
        while b1 < cs.size and (b1 == b0 or n_e + (ends[b1] - starts[b1]) <= batch_edges):
            n_e += ends[b1] - starts[b1]
            b1 += 1
        sl = slice(starts[b0], ends[b1 - 1])
        ci = cs[b0:b1]
        if sl.stop > sl.start:
            loc = np.searchsorted(ci, ei[sl])
            E_loc, _, g = _rows(model, rvec[sl], species[ei[sl]], species[ej[sl]], loc, ci.size, species[ci])
            g_all[sl] = g
        else:
            E_loc = np.zeros(ci.size)
        e_atom[ci] = E_loc + model.mu[species[ci]]
        b0 = b1
    np.add.at(forces, ei, g_all)
    np.add.at(forces, ej, -g_all)
    energy = float(np.sum(e_atom[cs]))
    return dict(energy=energy, e_atom=e_atom, forces=forces, edges=(ei, ej, en), g=g_all)


def sampled_forces(model, pos, species, box, atoms):
    """Exact F on ``atoms`` of a large box: evaluates the rows of the atoms and
    of all their neighbours (F_a needs g of every edge touching a)."""
    box = np.asarray(box, dtype=np.float64)
    pos = neighbors.wrap(np.asarray(pos, dtype=np.float64), box)
    atoms = np.unique(np.asarray(atoms))
    ei, ej, _ = neighbors.cell_list(pos, box, model.r_max, atoms)
    closure = np.unique(np.concatenate([atoms, ej]))
    res = energy_forces(model, pos, species, box, centers=closure)
    return res["forces"][atoms], res["e_atom"][atoms], res
