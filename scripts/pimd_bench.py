"""NEXT-3: ring-polymer PIMD throughput on one B200 (32 replicas per atom).

32 beads x N atoms of liquid NH3 (the paper's Fig. 4 sizes 1,728 / 6,912 / 13,824 atoms), the
(3,1) model at r_c = 6 A, all beads evaluated in one batched pass per step.
usage: python scripts/pimd_bench.py [--beads 32] [--steps 5] [--warmup 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2303_08169_b200 as pb  # noqa: E402
from synth import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--beads", type=int, default=32)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--dt", type=float, default=0.5)
args = ap.parse_args()
for lat, cells in (("bcc", (6, 6, 6)), ("bcc", (12, 12, 6)), ("bcc", (12, 12, 12))):
    cfg = configs.Config(f"PIMD-{cells}", lat, cells, 6.0, 3, 1, "PIMD bench")
    s = configs.system(cfg)
    rng = np.random.default_rng(0)
    P = args.beads
    q = s.pos[None] + rng.normal(size=(P, s.n, 3)) * 0.05
    v = np.repeat(s.vel[None], P, axis=0)
    m = pb.Allegro(configs.weight_file(cfg), s.box, n_atoms=P * s.n, precision=pb.PREC_3XTF32,
                   stream=torch.cuda.current_stream().cuda_stream)
    m.pimd_set_state(s.species, q, v, 200.0)
    m.pimd_step(args.warmup, args.dt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = m.pimd_step(args.steps, args.dt)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    print(json.dumps({"atoms": s.n, "beads": P, "bead_atoms": P * s.n, "edges": r.n_edges, "ms_per_step": round(ms, 3),
                      "bead_atom_steps_per_s": round(P * s.n / (ms / 1e3), 1), "h_conserved": r.h_conserved,
                      "temperature_beads": r.temperature_beads}), flush=True)
    m.close()
