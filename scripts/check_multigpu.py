"""Multi-GPU equivalence check (torchrun --nproc-per-node N): the spatially decomposed
force evaluation and MD steps equal one GPU on the same box."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import paper_2303_08169_b200 as pb
from synth import configs, nh3

rank, ws, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl")
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
prec = pb.PREC_3XTF32
grids = {2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}
if os.environ.get("ALG_GRID"):  # e.g. ALG_GRID=1,1,2 exercises the z-axis halo on 2 GPUs
    grids[int(os.environ["WORLD_SIZE"])] = tuple(int(v) for v in os.environ["ALG_GRID"].split(","))
s = configs.system(cfg)
if cfg == "C2":
    s = nh3.replicate(s, (2, 1, 1)) if ws >= 2 else s
wf = configs.weight_file(cfg)
obj = [pb.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
m = pb.Allegro(wf, s.box, device=local, precision=prec, rank=rank, world_size=ws, nccl_id=obj[0], grid=grids[ws])
out = {}
# 1) force evaluation: each rank passes its owned atoms (ownership = lower domain on ties)
P = np.array(grids[ws]); w = s.box / P
coord = np.array([rank % P[0], (rank // P[0]) % P[1], rank // (P[0] * P[1])])
pos = nh3.wrap_positions(s.pos, s.box)
own = np.clip(np.ceil(pos / w) - 1, 0, P - 1).astype(int)
mine = np.nonzero(np.all(own == coord, axis=1))[0]
e, ea, F = m.compute_energy_forces(pos[mine], s.species[mine], gid=mine.astype(np.int32))
allF = [None] * ws
dist.all_gather_object(allF, (mine, F, ea))
if rank == 0:
    ref0 = pb.Allegro(wf, s.box, device=local, precision=prec)
    e1, ea1, F1 = ref0.compute_energy_forces(pos, s.species)
    Fm = np.zeros_like(F1); Em = np.zeros_like(ea1)
    for idx, Fr, er in allF:
        Fm[idx] = Fr; Em[idx] = er
    print("FORCE-EVAL", json.dumps({"dE": abs(e - e1), "E": e1, "max_dE_atom": float(np.abs(Em - ea1).max()),
                                    "max_dF": float(np.abs(Fm - F1).max())}), flush=True)
    ref0.close()
# 2) MD: 5 steps
m.md_set_state(s.species, s.pos, s.vel)
rep = m.md_step(5, 2.0)
pos5, vel5, f5 = m.md_get_state()
if rank == 0:
    ref = pb.Allegro(wf, s.box, device=local, precision=prec)
    e1, ea1, F1 = ref.compute_energy_forces(pos, s.species)
    Fm = np.zeros_like(F1); Em = np.zeros_like(ea1)
    for idx, Fr, er in allF:
        Fm[idx] = Fr; Em[idx] = er
    out["n_atoms"] = int(s.n)
    out["dE_total"] = abs(e - e1)
    out["E_total"] = e1
    out["max_dE_atom"] = float(np.abs(Em - ea1).max())
    out["max_dF"] = float(np.abs(Fm - F1).max())
    ref.md_set_state(s.species, s.pos, s.vel)
    rep1 = ref.md_step(5, 2.0)
    p1, v1, f1 = ref.md_get_state()
    dp = pos5 - p1; dp -= s.box * np.round(dp / s.box)
    out["md_max_dpos"] = float(np.abs(dp).max())
    out["md_max_dvel"] = float(np.abs(vel5 - v1).max())
    out["md_max_dF"] = float(np.abs(f5 - f1).max())
    out["md_dEpot"] = abs(rep.e_pot - rep1.e_pot)
    out["md_edges"] = [int(rep.n_edges), int(rep1.n_edges)]
    out["ok"] = bool(out["max_dF"] < 1e-6 and out["max_dE_atom"] == 0.0 and out["md_max_dF"] < 1e-5 and rep.n_edges == rep1.n_edges)
    print(json.dumps(out), flush=True)
m.close()
dist.destroy_process_group()
