"""Summarise an ncu launch list per kernel class (the classes of prof.cuh / bench.py).

Input: the CSV of
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file X.csv python bench.py ...
Output (JSON): per class the launches, the mean serialised (cold-cache) duration, the mean
DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) and the class's
share of the summed duration.  bench.py reports the traffic of its dominant class from
this file as ``roofline.traffic`` (it is an ncu measurement, never taken inside a bench).

usage: python scripts/ncu_traffic.py launches.csv out.json
"""
from __future__ import annotations

import csv
import json
import re
import sys
from collections import defaultdict

# kernel-name substring -> class (prof.cuh prof_name); first match wins
CLASSES = [
    ("k_tb_fwd", "twobody"), ("k_tb_bwd", "twobody_bwd"), ("k_tpl_fwd", "tp_lin_fwd"), ("k_tpl_bwd", "tp_lin_bwd"), ("k_env_adj", "env_adj"), ("k_last", "last_layer"),
    ("true>", "gamma"), ("k_tc_gemm", "gemm"), ("k_gemm", "gemm"), ("k_tp_fwd", "tp_fwd"), ("k_tp_bwd", "tp_bwd"),
    ("k_energy", "energy"), ("k_rowdot", "rowdot"), ("k_geom_bwd", "geom_bwd"), ("k_geom", "geom"),
    ("k_force", "force_gather"), ("k_edge", "edge_build"), ("k_cell", "cell"), ("scan_", "scan"),
    ("k_ghost", "ghost"), ("k_wrap", "wrap"), ("k_kick", "verlet"), ("k_scale", "verlet"), ("k_ke", "reduce"),
    ("k_sum", "reduce"), ("k_fnorm", "reduce"), ("k_outliers", "reduce"), ("k_finite", "reduce"),
    ("k_halo", "halo"), ("k_mig", "halo"), ("k_ret_add", "halo"), ("k_owned", "halo"),
]


def classify(name: str) -> str:
    if re.search(r"k_tp_fwd<\d+, \d+, \d+, (1|true)>", name):  # the Gamma-only instantiation
        return "gamma"
    for sub, cls in CLASSES:
        if sub in name:
            return cls
    return "other:" + name.split("(")[0].split("::")[-1]


def main(src: str, dst: str) -> None:
    rows = [ln for ln in open(src) if not ln.startswith("==")]
    launches: dict[str, dict[str, float]] = defaultdict(dict)
    names: dict[str, str] = {}
    for r in csv.DictReader(rows):
        launches[r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        names[r["ID"]] = r["Kernel Name"]
    acc: dict[str, list[float]] = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    TP = "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
    per_kernel: dict[str, list[float]] = defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in launches.items():
        a = acc[classify(names[i])]
        t = m.get("gpu__time_duration.sum", 0.0)
        a[0] += 1
        a[1] += t
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a[3] += t * m.get(TP, 0.0)
        if TP in m:  # tensor-pipe activity per kernel instance (the contraction's epilogue template)
            k = per_kernel[names[i].split("(")[0]]
            k[0] += 1
            k[1] += t
            k[2] += t * m[TP]
    total = sum(a[1] for a in acc.values())
    out = {"source": src, "classes": {}}
    for cls, (n, ns, by, tpw) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
        out["classes"][cls] = {"launches": int(n), "ms_per_launch": ns / n / 1e6, "dram_bytes_per_launch": by / n,
                               "share": ns / total, "dram_gbs": by / max(ns, 1e-9),
                               "tensor_pipe_pct": tpw / max(ns, 1e-9)}
    out["tensor_pipe_per_kernel"] = {k: {"launches": int(n), "ms_total": ns / 1e6, "tensor_pipe_pct": w / max(ns, 1e-9)}
                                     for k, (n, ns, w) in sorted(per_kernel.items(), key=lambda kv: -kv[1][1])}
    json.dump(out, open(dst, "w"), indent=1)
    for cls, v in out["classes"].items():
        print(f"{cls:14s} n={v['launches']:6d} share={v['share']:.3f} ms/launch={v['ms_per_launch']:.4f} "
              f"dram/launch={v['dram_bytes_per_launch']:.4g} B ({v['dram_gbs']:.0f} GB/s) tensor {v['tensor_pipe_pct']:.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
