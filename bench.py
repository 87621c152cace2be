"""Benchmark of the Allegro-Legato NNQMD hot path: one MD step = neighbour build +
Allegro energy/forces + velocity Verlet (BASELINE.json metric: atom-steps/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5|C4|C3|C2|C1]
                    [--impl ours|reference] [--no-cpu-baseline]

N > 1 is launched by torchrun (one process per GPU).  The default workload is C5
(BASELINE.json configs[4], the metric's weak-scaling configuration): 500,000 atoms of
liquid NH3 per GPU with the paper's l=1 3-layer model.  Prints ONE JSON line on rank 0.
``--impl reference`` times the fp64 CPU oracle (the reference arm of this tier) on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "atom-steps/s (Allegro force+Verlet) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "atom-steps/s"
DT_FS = 2.0


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def _fp32_alu_peak_tflops(sm_mhz):
    # 148 SMs x 128 FP32 lanes x 2 flop/FMA x clock (B200_PROFILING.md unit counts)
    return 148 * 128 * 2 * sm_mhz * 1e6 / 1e12


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int, interval_ms: int = 200):
        self.path = tempfile.mktemp(suffix=".csv")
        self.p = None
        if interval_ms <= 0:
            return
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-i", str(gpu), "-lms", str(interval_ms)], stdout=open(self.path, "w"),
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    """The reference arm: the fp64 oracle as it stands, on host cores, rank 0 only."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    from oracle import irreps
    from synth import configs

    cfg = configs.CONFIGS[args.config]
    sample = args.ref_sample
    rec = _oracle_rate(cfg, sample, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": rec["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": rec["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config_dict(cfg, args.gpus, None, "oracle", irreps.param_count(cfg.n_layers, cfg.lmax)),
        "cpu_baseline": {"value": rec["value"], "unit": UNIT, "cores": rec["cores"], "kind": "oracle",
                         "sample": rec["sample"]},
        "e2e": {"value": rec["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _oracle_rate(cfg, sample, steps, warmup):
    """Oracle force evaluation of ``sample`` centre rows of the cfg box per step."""
    from threadpoolctl import threadpool_info

    from oracle import allegro as oa, neighbors as onb, weights_io
    from synth import configs

    s = configs.system(cfg)
    model = weights_io.read(configs.weight_file(cfg))
    pos = onb.wrap(s.pos, s.box)
    rng = np.random.default_rng(0)
    times = []
    for it in range(warmup + steps):
        centers = np.sort(rng.choice(s.n, sample, replace=False))
        t0 = time.perf_counter()
        oa.energy_forces(model, pos, s.species, s.box, centers=centers)
        dt = time.perf_counter() - t0
        if it >= warmup:
            times.append(dt)
    t = float(np.mean(times))
    cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    return {
        "value": sample / t,
        "ms_per_step": 1e3 * t,
        "cores": cores,
        "sample": (f"{sample} random centre rows of the {cfg.name} box per step (neighbour search + Allegro "
                   f"energy/forces of those rows, fp64 numpy; Verlet O(N) excluded), mean of {steps} steps; "
                   f"value = rows / s"),
    }


GRIDS = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}

PREC_TEXT = {
    "oracle": "fp64 numpy oracle (oracle/allegro.py) on host cores",
    "3xtf32": "3xTF32 tcgen05 GEMMs (fp32-level accuracy) + fp32 TP (fp64 positions, Verlet, energy sums)",
    "fp32": "fp32 CUDA-core GEMMs + fp32 TP (fp64 positions, Verlet, energy sums)",
    "tf32": "single-pass TF32 tcgen05 GEMMs (outside the force bound; reported, not gated) + fp32 TP",
}


def _ncu_traffic(cfg_name, cls, alg_bytes_per_launch):
    """roofline.traffic: DRAM bytes per launch of kernel class ``cls`` from the newest
    committed ncu launch list (profiles/rNN_traffic_<config>.json, scripts/ncu_traffic.py)."""
    import glob

    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                          f"r*_traffic_{cfg_name.lower()}.json")))
    if not files:
        return {"traffic": None}
    rec = json.load(open(files[-1]))["classes"].get(cls)
    if not rec:
        return {"traffic": None}
    return {"traffic": round(rec["dram_bytes_per_launch"]),
            "traffic_source": (f"{os.path.basename(files[-1])}: ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                               f"mean over {rec['launches']} launches of class {cls}"),
            "traffic_over_algorithmic": round(rec["dram_bytes_per_launch"] / max(alg_bytes_per_launch, 1e-9), 3)}


def _config_dict(cfg, n_gpus, edges, precision, params, strong=False):
    return {
        "workload": f"{cfg.name}: {cfg.description}, r_c={cfg.r_cut} A, NVE dt={DT_FS} fs, rebuild every step",
        "atoms_per_gpu": cfg.n_atoms // n_gpus if strong else cfg.n_atoms,
        "atoms_total": cfg.n_atoms if strong else cfg.n_atoms * n_gpus,
        "edges_per_gpu": None if edges is None else edges // n_gpus,
        "edges_total": edges,
        "layers": cfg.n_layers,
        "lmax": cfg.lmax,
        "params": params,
        "precision": PREC_TEXT[precision],
        "parallelism": ("single domain" if n_gpus == 1 else
                        f"spatial decomposition {GRIDS.get(n_gpus, (n_gpus, 1, 1))} domains, NCCL halo + ghost-force return"),
        "l2": "inputs larger than L2 (per-edge activations are GBs per step)",
    }


def _spawn(args_list, n):
    """`bench.py --gpus N` outside torchrun: re-launch itself with one process per GPU."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + args_list
    return subprocess.call(cmd)


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _cpu_baseline(cfg, sample_all, sample_1t):
    """The oracle as it stands on this host: all BLAS threads, and one thread."""
    from threadpoolctl import threadpool_limits

    rec = _oracle_rate(cfg, sample_all, 1, 0)
    out = {"value": round(rec["value"], 2), "unit": UNIT, "cores": rec["cores"], "kind": "oracle",
           "sample": rec["sample"], "cpu_model": _cpu_model(), "logical_cpus": os.cpu_count()}
    if sample_1t > 0:
        with threadpool_limits(limits=1):
            r1 = _oracle_rate(cfg, sample_1t, 1, 0)
        out["one_thread"] = {"value": round(r1["value"], 2), "unit": UNIT, "cores": 1, "sample": r1["sample"]}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=512)
    ap.add_argument("--cpu-sample-1t", type=int, default=96)
    ap.add_argument("--ref-sample", type=int, default=96)
    ap.add_argument("--profile-steps", type=int, default=1)
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: split the config's box over the GPUs (default: replicate it per GPU)")
    ap.add_argument("--precision", default="3xtf32", choices=["3xtf32", "fp32", "tf32"])
    ap.add_argument("--skin", type=float, default=0.0,
                    help="neighbour-list skin (A); the list is still rebuilt every step (NEXT-4 A/B of its cost)")
    ap.add_argument("--clock-interval-ms", type=int, default=200,
                    help="nvidia-smi sampling period during the timed region (0: off)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _spawn(sys.argv[1:], args.gpus)

    import torch

    import paper_2303_08169_b200 as pb
    from synth import configs

    ws, rank, local = _dist()
    if ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
    nccl_id = None
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
        obj = [pb.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    torch.cuda.set_device(local)
    cfg = configs.CONFIGS[args.config]
    grid = GRIDS.get(ws, (ws, 1, 1))
    # weak scaling: the N-GPU box is the per-GPU box replicated over the domain grid;
    # strong scaling (--strong, e.g. C4): the same box split over the grid
    s = configs.system(cfg) if args.strong else configs.system(cfg, reps=grid)
    wf = configs.weight_file(cfg)
    stream = torch.cuda.current_stream()
    prec = {"3xtf32": pb.PREC_3XTF32, "fp32": pb.PREC_FP32, "tf32": pb.PREC_TF32}[args.precision]
    m = pb.Allegro(wf, s.box, device=local, n_atoms=s.n, stream=stream.cuda_stream, precision=prec, rank=rank,
                   world_size=ws, nccl_id=nccl_id, grid=grid, skin=args.skin)
    m.md_set_state(s.species, s.pos, s.vel)
    r_w = m.md_step(args.warmup, DT_FS)
    edges_first = int(r_w.n_edges)

    # the start state of the timed window, kept so that the e2e leg runs the SAME MD steps
    pos_w, vel_w, _ = m.md_get_state()  # world_size > 1: gathered on rank 0
    if ws > 1:
        tp = torch.from_numpy(pos_w).cuda()
        tv = torch.from_numpy(vel_w).cuda()
        torch.distributed.broadcast(tp, 0)
        torch.distributed.broadcast(tv, 0)
        pos_w, vel_w = tp.cpu().numpy(), tv.cpu().numpy()

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    # The random-weight liquid heats and its neighbour counts drift, so the K steps visit buffer sizes
    # the warm-up did not: run them once untimed (every device buffer reaches its size for this
    # trajectory), then restart from the same state and time them (deterministic: the same steps).
    m.md_step(args.steps, DT_FS)
    m.md_set_state(s.species, pos_w, vel_w)

    # ---- timed region: K steps with inputs resident in HBM ----
    clocks = ClockSampler(local, args.clock_interval_ms)
    time.sleep(0.3)
    # The first P timed steps carry per-launch CUDA events (the kernel breakdown and the
    # roofline); the remaining K - P run without them (each event record costs a few us).
    n_prof = max(1, min(args.profile_steps, args.steps))
    m.profile(True)  # resets the totals and the launch counter (synchronises the stream)
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    rep = m.md_step(n_prof, DT_FS)
    edges_prof = int(rep.n_edges)
    evp = torch.cuda.Event(enable_timing=True)  # the profiled steps' own span (kernel sum + gaps)
    evp.record(stream)
    m.profile(False)
    if args.steps > n_prof:
        rep = m.md_step(args.steps - n_prof, DT_FS)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = ev0.elapsed_time(ev1)
    ms_prof_span = ev0.elapsed_time(evp) / n_prof
    launches = m.launch_count()
    prof = m.profile_read()
    detail = sorted(m.profile_detail(), key=lambda x: -x[1])
    clk = clocks.stop()
    edges_last = int(rep.n_edges)
    e_pot_dev = rep.e_pot
    t = torch.tensor([ms], device="cuda")
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms_max = float(t.item())
    value = s.n * args.steps / (ms_max / 1e3)  # s.n = atoms of the whole (replicated) box
    ranks = None
    if ws > 1:  # per-rank view of the same timed region: the max above is set by the slowest device
        ksum = sum(v[0] for v in prof.values()) / n_prof  # this rank's own kernel time per profiled step
        mine = torch.tensor([ms / args.steps, ms_prof_span, float((clk or {}).get("sm_mhz") or 0.0), ksum],
                            device="cuda", dtype=torch.float64)
        allr = [torch.zeros_like(mine) for _ in range(ws)]
        torch.distributed.all_gather(allr, mine)
        ranks = {"ms_per_step": [round(float(x[0]), 3) for x in allr],
                 "profiled_step_span_ms": [round(float(x[1]), 3) for x in allr],
                 "sm_mhz": [round(float(x[2]), 1) for x in allr],
                 "kernel_ms_per_step": [round(float(x[3]), 3) for x in allr]}

    # ---- e2e: the SAME K steps (same start state) through md_step_host, state in pinned host memory ----
    m.md_set_state(s.species, pos_w, vel_w)
    n_loc = m.local_count()
    cap = 2 * n_loc + 1024  # migration may change the local count
    _, spc, _, pos, vel, frc = m.md_get_local_state(cap)
    h_spc = torch.from_numpy(spc).pin_memory()
    h_pos = torch.from_numpy(pos).pin_memory()
    h_vel = torch.from_numpy(vel).pin_memory()
    h_frc = torch.from_numpy(frc).pin_memory()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h2d = d2h = 0
    for _ in range(args.steps):
        h2d += n_loc * (4 + 3 * 24)
        r = m.md_step_host(h_spc, h_pos, h_vel, h_frc, 1, DT_FS, n_local=n_loc)
        n_loc = r.n_local
        d2h += n_loc * (3 * 24 + (4 if ws > 1 else 0))
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    te = torch.tensor([e0.elapsed_time(e1), h2d, d2h], device="cuda", dtype=torch.float64)
    if ws > 1:
        tm = te[:1].clone()
        torch.distributed.all_reduce(tm, op=torch.distributed.ReduceOp.MAX)
        tb = te[1:].clone()
        torch.distributed.all_reduce(tb, op=torch.distributed.ReduceOp.SUM)
        te = torch.cat([tm, tb])
    e2e_value = s.n * args.steps / (float(te[0].item()) / 1e3)
    h2d = int(te[1].item()) // args.steps
    d2h = int(te[2].item()) // args.steps
    e2e_same = bool(r.e_pot == e_pot_dev and int(r.n_edges) == edges_last)

    # ---- roofline: dominant kernel class + the step bound ----
    peaks, peak_src = _peaks()
    total_ms = sum(v[0] for v in prof.values())
    dom = max(prof, key=lambda k: prof[k][0])
    d_ms, d_fl, d_by, d_n = prof[dom]
    kernels = {}
    for k, (kms, kfl, kby, kn) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
        if kn == 0:
            continue
        kernels[k] = {"ms_per_step": round(kms / n_prof, 4), "share": round(kms / max(total_ms, 1e-9), 4),
                      "launches_per_step": kn / n_prof,
                      "gflops": round(kfl / max(kms, 1e-9) / 1e6, 1), "gbs": round(kby / max(kms, 1e-9) / 1e6, 1)}
    alu_peak = _fp32_alu_peak_tflops(peaks.get("sm_max_mhz", 1965.0))
    # tensor peak for the contraction dtype: measured bf16 x 0.5 (TF32 : BF16 nominal) / passes
    # (3 for 3xTF32); the contractions run inside a long, power-capped step, so the sustained
    # bf16 figure applies (B200_PROFILING.md)
    tc_key = "bf16_tflops_sustained" if "bf16_tflops_sustained" in peaks else "bf16_tflops"
    passes = {"3xtf32": 3.0, "tf32": 1.0, "fp32": None}[args.precision]
    tc_peak = peaks.get(tc_key, 1400.0) * 0.5 / passes if passes else None
    gbs = d_by / (d_ms / 1e3) / 1e9
    tfs = d_fl / (d_ms / 1e3) / 1e12
    hbm_frac = gbs / peaks["hbm_gbs"]
    if d_fl > 0 and dom in ("gemm", "tp_lin_fwd", "tp_lin_bwd") and tc_peak:
        roof = {"kernel": dom, "bound": "tensor", "achieved": round(tfs, 2), "peak": round(tc_peak, 1),
                "unit": "TFLOP/s", "frac": round(tfs / tc_peak, 4), "traffic": None,
                "peak_source": (f"{peak_src} {tc_key} {peaks.get(tc_key)} x 0.5 (TF32/BF16 nominal) / {passes:g} "
                                f"({args.precision} passes)"),
                "per_launch": f"{d_fl / d_n:.4g} algorithmic flop / {d_ms / d_n:.4g} ms",
                "hbm_secondary": {"achieved_gbs": round(gbs, 1), "frac": round(hbm_frac, 4),
                                  "note": "bytes this design materialises per contraction, not the method's minimum"}}
    elif d_fl > 0 and hbm_frac < tfs / alu_peak:
        roof = {"kernel": dom, "bound": "alu", "achieved": round(tfs, 2), "peak": round(alu_peak, 1),
                "unit": "TFLOP/s", "frac": round(tfs / alu_peak, 4), "traffic": None,
                "peak_source": "derived: 148 SMs x 128 fp32 lanes x 2 x sm_max_mhz",
                "per_launch": f"{d_fl / d_n:.4g} flop / {d_ms / d_n:.4g} ms"}
    else:
        roof = {"kernel": dom, "bound": "hbm", "achieved": round(gbs, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(hbm_frac, 4), "traffic": None, "peak_source": f"{peak_src} hbm_gbs",
                "per_launch": f"{d_by / d_n:.4g} B / {d_ms / d_n:.4g} ms"}
    roof.update(_ncu_traffic(cfg.name, dom, d_by / d_n))
    # step-level bound: T_roof = max(bytes_alg / BW, GEMM_flop_alg / P_tensor, TP_flop_alg / P_fp32)
    mac_e, tpf_e = pb.work_per_edge(cfg.n_layers, cfg.lmax)
    e_step = edges_prof / ws  # edges per GPU of the profiled step
    a_step = s.n / ws
    gemm_flop = 4.0 * mac_e * e_step      # forward + input-gradient reverse (no dW), 2 flop per MAC
    tp_flop = 6.0 * tpf_e * e_step        # forward + 2x in the reverse, 2 flop per FMA
    bytes_alg = 190.0 * a_step + 32.0 * e_step  # §8(d): state + cells ~190 B/atom; CSR + g ~32 B/edge
    t_gemm = gemm_flop / ((tc_peak or alu_peak) * 1e12) * 1e3
    t_tp = tp_flop / (alu_peak * 1e12) * 1e3
    t_hbm = bytes_alg / (peaks["hbm_gbs"] * 1e9) * 1e3
    t_roof = max(t_gemm, t_tp, t_hbm)
    t_meas = ms_max / args.steps
    roof["step"] = {"t_roof_ms": round(t_roof, 3), "t_meas_ms": round(t_meas, 3), "frac": round(t_roof / t_meas, 4),
                    "t_gemm_ms": round(t_gemm, 3), "t_tp_ms": round(t_tp, 3), "t_hbm_ms": round(t_hbm, 3),
                    "gemm_mflop_per_atom_step": round(gemm_flop / a_step / 1e6, 2),
                    "tp_mflop_per_atom_step": round(tp_flop / a_step / 1e6, 3),
                    "note": "SURVEY.md §8(d): T_roof = max(bytes_alg/BW, GEMM_FLOP/P_tensor(mode), TP_FLOP/P_fp32)"}
    # HBM roofline of the streaming edge kernel (north_star: >= 60% on the edge kernels)
    fg = prof.get("force_gather")
    if fg and fg[3]:
        roof["force_gather_hbm_frac"] = round(fg[2] / (fg[0] / 1e3) / 1e9 / peaks["hbm_gbs"], 4)

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3), "higher_is_better": True,
        "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": _config_dict(cfg, ws, int(rep.n_edges), args.precision, pb.param_count(cfg.n_layers, cfg.lmax),
                               args.strong),
        "roofline": roof,
        "kernels": kernels,
        "gpu_launches": launches,
        "shapes": [{"tag": t, "ms_per_step": round(ms_ / n_prof, 3), "gbs": round(by / max(ms_, 1e-9) / 1e6, 1),
                    "launches_per_step": n_ / n_prof} for t, ms_, by, n_ in detail[:40]],
        "profiled_steps": n_prof,
        "profiled_step_span_ms": round(ms_prof_span, 3),  # device span of a profiled step (kernels + gaps)
        "edges": {"first": edges_first, "profiled": edges_prof, "last": edges_last,
                  "edges_per_s": round(0.5 * (edges_first + edges_last) * args.steps / (ms_max / 1e3), 1)},
        "e2e": {"value": round(e2e_value, 1), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "same_steps_as_value": e2e_same},
        "clocks": clk,
        "ranks": ranks,
        "md": {"e_pot": rep.e_pot, "e_kin": rep.e_kin, "temperature": rep.temperature,
               "n_outliers_last": rep.n_outliers_last},
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = _cpu_baseline(cfg, args.cpu_sample, args.cpu_sample_1t)
    if rank == 0:
        print(json.dumps(line), flush=True)
    m.close()
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main() or 0)
