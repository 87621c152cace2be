"""World-size-2 CPU test of the N > 1 path (gloo): two processes each own one domain
of a (2,1,1) grid, build the halo with the staged exchange (real send/recv between the
processes; self-messages along axes with p = 1), evaluate their owned rows and return
ghost forces in reverse stage order (z, y, x) -- the message pattern of
paper_2303_08169_b200/csrc/domain.cu -- and must reproduce the single-domain oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import allegro, domains, neighbors, weights_io
from synth import nh3, weights as sw


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _send_arr(a, peer):
    a = np.ascontiguousarray(a, dtype=np.float64)
    dist.send(torch.tensor([a.size], dtype=torch.int64), peer)
    if a.size:
        dist.send(torch.from_numpy(a.reshape(-1)), peer)


def _recv_arr(peer, cols):
    n = torch.zeros(1, dtype=torch.int64)
    dist.recv(n, peer)
    buf = torch.zeros(int(n.item()), dtype=torch.float64)
    if buf.numel():
        dist.recv(buf, peer)
    return buf.numpy().reshape(-1, cols) if cols else buf.numpy()


def _pack(msg):
    return np.concatenate([msg["gid"][:, None], msg["species"][:, None], msg["pos"], msg["shift"]], axis=1)


def _unpack(a):
    return dict(gid=a[:, 0].astype(np.int64), species=a[:, 1].astype(np.int64), pos=a[:, 2:5].copy(),
                shift=a[:, 5:8].astype(np.int64))


def _exchange(rank, peer_m, peer_p, send_m, send_p):
    """send_m -> -neighbour, send_p -> +neighbour; returns (from -, from +).  Pairwise
    ordering: lower rank sends first (gloo send/recv are blocking)."""
    if peer_m == rank and peer_p == rank:
        return send_p, send_m
    peer = peer_m  # p = 2 along this axis: both neighbours are the same process
    assert peer_p == peer
    if rank < peer:
        _send_arr(send_p, peer), _send_arr(send_m, peer)
        from_m, from_p = _recv_arr(peer, send_p.shape[1]), _recv_arr(peer, send_m.shape[1])
    else:
        from_m, from_p = _recv_arr(peer, send_p.shape[1]), _recv_arr(peer, send_m.shape[1])
        _send_arr(send_p, peer), _send_arr(send_m, peer)
    return from_m, from_p


def _worker(rank, port, wpath, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    model = weights_io.read(wpath)
    s = nh3.nh3_box("fcc", (2, 2, 2))
    grid = (2, 1, 1)
    box = s.box
    pos = neighbors.wrap(s.pos, box)
    coord = domains.grid_coords(rank, grid)
    own = domains.owner_coords(pos, box, grid)
    idx = np.nonzero(np.all(own == coord, axis=1))[0]
    loc = dict(gid=idx.astype(np.int64), species=s.species[idx].astype(np.int64), pos=pos[idx].copy(),
               shift=np.zeros((idx.size, 3), np.int64))
    n_own = idx.size
    stages = []
    for axis in range(3):
        m_, p_ = domains.stage_messages(loc, axis, coord, box, grid, model.r_max)
        pm, pp = domains.neighbour_ranks(coord, axis, grid)
        from_m, from_p = _exchange(rank, pm, pp, _pack(m_), _pack(p_))
        base = loc["gid"].size
        loc = domains.append(loc, _unpack(from_m))
        loc = domains.append(loc, _unpack(from_p))
        stages.append(dict(src_m=m_["src"], src_p=p_["src"], rm=(base, base + len(from_m)),
                           rp=(base + len(from_m), base + len(from_m) + len(from_p)), pm=pm, pp=pp))
    e_loc, (ei, ej), g = domains.domain_rows(model, loc, n_own, model.r_max)
    f = np.zeros((loc["gid"].size, 3))
    np.add.at(f, ei, g)
    np.add.at(f, ej, -g)
    for axis in (2, 1, 0):  # reverse halo: ghost forces back to their senders
        st = stages[axis]
        ret_m = f[st["rm"][0]:st["rm"][1]]  # ghosts that came from -, back to -
        ret_p = f[st["rp"][0]:st["rp"][1]]
        back_for_m, back_for_p = _exchange(rank, st["pm"], st["pp"], ret_m, ret_p)
        np.add.at(f, st["src_m"], back_for_m)
        np.add.at(f, st["src_p"], back_for_p)
    res = np.concatenate([idx[:, None].astype(np.float64), e_loc[:, None], f[:n_own]], axis=1)
    np.save(f"{out_path}.{rank}.npy", res)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_decomposition(tmp_path):
    wpath = str(tmp_path / "m.algw")
    sw.write(wpath, 2, 1, 5.0, sw.generate(2, 1, 0), sw.nbar_for(5.0), (1.5, 1.5), (0.0, 0.0))
    out = str(tmp_path / "res")
    mp.spawn(_worker, args=(_free_port(), wpath, out), nprocs=2, join=True)
    model = weights_io.read(wpath)
    s = nh3.nh3_box("fcc", (2, 2, 2))
    ref = allegro.energy_forces(model, s.pos, s.species, s.box)
    parts = [np.load(f"{out}.{r}.npy") for r in range(2)]
    gids = np.concatenate([p[:, 0] for p in parts]).astype(int)
    assert sorted(gids.tolist()) == list(range(s.n))  # every atom owned exactly once
    for p in parts:
        g = p[:, 0].astype(int)
        assert np.array_equal(p[:, 1], ref["e_atom"][g])
        np.testing.assert_allclose(p[:, 2:5], ref["forces"][g], atol=1e-12)
