"""NEXT-4: Table 2's tensor-rank sweep on B200 (§4.1 Table 2).

The paper's three models -- 3 layers, C = 32, D = 128, lmax = 0 / 1 / 2 with 95,656 / 133,544 /
183,720 parameters -- timed per MD step on one GPU.  Table 2 does not state the system it was
timed on, so the C3 box (110,592 atoms, liquid NH3, r_c = 6 A) is used for all three, plus the
C5 box (500,000 atoms) for the production lmax = 1 model; ratios between the ranks are the
comparable quantity (paper: 395 : 916 : 2,580 ms = 0.43 : 1 : 2.82).

usage: python scripts/table2_sweep.py [--steps K] [--warmup W] > table2.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2303_08169_b200 as pb  # noqa: E402
from synth import configs  # noqa: E402

PAPER_MS = {0: 395.0, 1: 916.0, 2: 2580.0}  # Table 2, other hardware, system size unstated
PAPER_PARAMS = {0: 95656, 1: 133544, 2: 183720}


def run(cfg, steps, warmup, prec, dt=2.0):
    s = configs.system(cfg)
    stream = torch.cuda.current_stream()
    m = pb.Allegro(configs.weight_file(cfg), s.box, n_atoms=s.n, stream=stream.cuda_stream, precision=prec)
    m.md_set_state(s.species, s.pos, s.vel)
    m.md_step(warmup, dt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    rep = m.md_step(steps, dt)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    m.close()
    return ms, rep, s.n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--precision", default="3xtf32", choices=["3xtf32", "fp32"])
    args = ap.parse_args()
    prec = pb.PREC_3XTF32 if args.precision == "3xtf32" else pb.PREC_FP32
    rows = []
    for lmax in (0, 1, 2):
        cfg = configs.Config(f"T2-l{lmax}", "bcc", (24, 24, 24), 6.0, 3, lmax, f"C3 box, 3-layer lmax={lmax}")
        ms, rep, n = run(cfg, args.steps, args.warmup, prec)
        rows.append({"model": f"Allegro (l={lmax})", "params": pb.param_count(3, lmax),
                     "params_paper": PAPER_PARAMS[lmax], "atoms": n, "edges": int(rep.n_edges),
                     "ms_per_step": round(ms, 3), "atom_steps_per_s": round(n / (ms / 1e3), 1),
                     "paper_ms_per_step": PAPER_MS[lmax], "precision": args.precision})
    base = next(r for r in rows if r["model"].endswith("l=1)"))
    for r in rows:
        r["ratio_to_l1"] = round(r["ms_per_step"] / base["ms_per_step"], 3)
        r["paper_ratio_to_l1"] = round(r["paper_ms_per_step"] / PAPER_MS[1], 3)
        print(json.dumps(r), flush=True)
    ms, rep, n = run(configs.CONFIGS["C5"], args.steps, args.warmup, prec)
    print(json.dumps({"model": "Allegro (l=1), C5 box", "params": pb.param_count(3, 1), "atoms": n,
                      "edges": int(rep.n_edges), "ms_per_step": round(ms, 3),
                      "atom_steps_per_s": round(n / (ms / 1e3), 1)}), flush=True)


if __name__ == "__main__":
    main()
