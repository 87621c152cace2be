"""NEXT-2: the paper's time-to-failure experiment shape on the GPU (§3.2, Eq. 4).

For each system size N (liquid NH3, fcc cells^3; 432 atoms = the paper's smallest size) and
>= 10 seeds: NVT at 200 K for 1,000 steps, then NVE at dt = 2 fs until failure (md_run_ttf;
criteria in DESIGN.md D24), then the Eq. 4 fit t = alpha N^-beta (paper_2303_08169_b200.ttf).

CAVEAT: the weights are random (no trained Allegro / Allegro-Legato model exists here), so
t_failure measures the harness on an arbitrary smooth landscape, not the paper's models.

usage: python scripts/ttf_run.py --cells 2 3 4 5 --seeds 10 --max-nve 5000 --out profiles/r01_ttf
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2303_08169_b200 as pb  # noqa: E402
from paper_2303_08169_b200 import ttf  # noqa: E402
from synth import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, nargs="+", default=[2, 3, 4, 5])
    ap.add_argument("--seeds", type=int, default=10)
    ap.add_argument("--nvt", type=int, default=1000)
    ap.add_argument("--max-nve", type=int, default=5000)
    ap.add_argument("--out", default="gpurun_out/ttf")
    args = ap.parse_args()
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    rows, series_out = [], []
    t0 = time.time()
    for n_c in args.cells:
        cfg = configs.Config(f"TTF-{n_c}", "fcc", (n_c, n_c, n_c), 6.0, 3, 1, f"fcc {n_c}^3, (3,1) model")
        wf = configs.weight_file(cfg)
        for seed in range(args.seeds):
            s = configs.system(cfg, seed=seed)
            m = pb.Allegro(wf, s.box, n_atoms=s.n, precision=pb.PREC_3XTF32)
            m.md_set_state(s.species, s.pos, s.vel)
            r, series = m.md_run_ttf(dt_fs=2.0, nvt_steps=args.nvt, T_K=200.0, tau_fs=100.0,
                                     max_nve_steps=args.max_nve, check_interval=100, drift_tol=0.1, disp_max=0.5,
                                     outlier_k=5.0, outlier_interval=10)
            m.close()
            rows.append({"n_atoms": s.n, "seed": seed, "steps_survived": r["steps_survived"],
                         "fail_step": r["fail_step"],
                         "failure_reason": r["reason_name"], "e0": r["e0"], "e_last": r["e_last"]})
            series_out.append({"n_atoms": s.n, "seed": seed, "interval": 10, "outliers": series.tolist()})
            print(json.dumps(rows[-1]), flush=True)
    with open(args.out + "_records.csv", "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(rows[0]))
        w.writeheader()
        w.writerows(rows)
    with open(args.out + "_series.jsonl", "w") as f:
        for r in series_out:
            f.write(json.dumps(r) + "\n")
    codes = {v: k for k, v in pb.TTF_REASONS.items()}
    try:
        fit = ttf.fit_power_law([(r["n_atoms"], r["fail_step"], codes[r["failure_reason"]]) for r in rows])
    except ttf.FitError as e:
        fit = {"error": str(e)}
    fit["wall_s"] = round(time.time() - t0, 1)
    fit["note"] = "random-weight model: harness demonstration, not the paper's beta"
    with open(args.out + "_fit.json", "w") as f:
        json.dump(fit, f, indent=1)
    print(json.dumps(fit), flush=True)


if __name__ == "__main__":
    main()
