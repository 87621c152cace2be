"""C2 (BASELINE configs[1]): liquid NH3, 1,024 atoms, 2-layer lmax=2 Allegro, 1,000 NVE steps at
dt = 2 fs on one B200 from the 200 K Maxwell-Boltzmann start (SURVEY.md §8(d):
"1,000 NVE steps ... snapshot parity at steps 0, 100, ..., 1,000; drift, T(t) and n_out(t)
reported").  Every 100 steps the GPU state is re-evaluated by the fp64 oracle (per evaluation:
trajectories are chaotic, reading D21) against the bars of DESIGN.md D20 (energy) and D26
(forces: 1e-4 eV/A x max(1, RMS|F|_oracle)).  Optional first argument: NVT steps at 200 K before
the NVE run (the paper's protocol; default 0)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2303_08169_b200 as pb
from oracle import allegro as oa, weights_io
from synth import configs

n_nvt = int(sys.argv[1]) if len(sys.argv) > 1 else 0
n_nve = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
tau = float(sys.argv[3]) if len(sys.argv) > 3 else 100.0
out_dir = sys.argv[4] if len(sys.argv) > 4 else "gpurun_out"
E_TOL, F_TOL = 1e-5, 1e-4
s = configs.system("C2")
wf = configs.weight_file("C2")
model = weights_io.read(wf)
m = pb.Allegro(wf, s.box, precision=pb.PREC_3XTF32)
m.md_set_state(s.species, s.pos, s.vel)
log = []
snaps = {}
t0 = time.time()
if n_nvt:
    m.md_set_thermostat(200.0, tau)
    m.md_set_state(s.species, s.pos, s.vel)
    for step in range(0, n_nvt, 10):
        r = m.md_step(10, 2.0)
        log.append(dict(phase="nvt", step=step + 10, e_pot=r.e_pot, e_kin=r.e_kin, T=r.temperature,
                        e_conserved=r.e_conserved, edges=r.n_edges))
    m.md_set_thermostat(200.0, 0.0)
mean0, sig0 = m.md_force_baseline()
r = m.md_step(0, 2.0)
for step in range(0, n_nve + 1, 10):
    if step % 100 == 0:
        snaps[step] = (m.md_get_state(), r.e_pot)
    log.append(dict(phase="nve", step=step, e_pot=r.e_pot, e_kin=r.e_kin, T=r.temperature,
                    n_out=m.md_count_outliers(mean0, sig0, 5.0), edges=r.n_edges))
    if step == n_nve:
        break
    r = m.md_step(10, 2.0)
wall = time.time() - t0
parity = {}
for step, ((p, v, f), e_pot) in snaps.items():
    ref = oa.energy_forces(model, p, s.species, s.box)
    rms = float(np.sqrt((ref["forces"] ** 2).sum(1).mean()))
    dF = float(np.abs(f - ref["forces"]).max())
    dE = abs(e_pot - ref["energy"]) / float(np.abs(ref["e_atom"]).sum())
    parity[step] = dict(max_dF=dF, rms_F=rms, bar_F=F_TOL * max(1.0, rms), rel_dE=dE,
                        ok=bool(dF <= F_TOL * max(1.0, rms) and dE <= E_TOL))
os.makedirs(out_dir, exist_ok=True)
with open(os.path.join(out_dir, "c2_md_log.json"), "w") as fh:
    json.dump(log, fh)
nve = [x for x in log if x["phase"] == "nve"]
summary = dict(
    steps=dict(nvt=n_nvt, nve=n_nve), dt_fs=2.0, wall_s=round(wall, 2),
    ms_per_step=round(1e3 * wall / max(1, n_nvt + n_nve), 3),
    T_nve_first=nve[0]["T"], T_nve_last=nve[-1]["T"],
    nve_drift_per_atom_eV=(nve[-1]["e_pot"] + nve[-1]["e_kin"] - nve[0]["e_pot"] - nve[0]["e_kin"]) / s.n,
    n_out_max=max(x["n_out"] for x in nve), edges_first=nve[0]["edges"], edges_last=nve[-1]["edges"],
    bars="D20 energy |dE| / sum|E_a| <= 1e-5; D26 forces max|dF| <= 1e-4 eV/A x max(1, RMS|F|_oracle)",
    snapshot_parity=parity,
    parity_ok=all(v["ok"] for v in parity.values()))
print(json.dumps(summary), flush=True)
