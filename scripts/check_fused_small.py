"""Fused TP + TP-linear forward / backward vs the unfused path (debugging aid): C1 replicated
rep^3 times with the given models; prints whether E and F agree bit for bit and max|dF|."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2303_08169_b200 as pb
from synth import configs, nh3, weights as sw

rep = int(sys.argv[1]) if len(sys.argv) > 1 else 4
arch = [tuple(int(x) for x in a.split(",")) for a in (sys.argv[2:] or ["2,1", "3,1"])]
s = nh3.replicate(configs.system("C1"), (rep, rep, rep))
for L, lmax in arch:
    wf = f"/tmp/m{L}{lmax}.algw"
    sw.write(wf, L, lmax, 5.0, sw.generate(L, lmax, 0), sw.nbar_for(5.0), (1.0, 1.0), (0.0, 0.0))
    m = pb.Allegro(wf, s.box, precision=pb.PREC_3XTF32, n_atoms=s.n)
    os.environ["ALLEGRO_FUSED_TP"] = "0"
    os.environ["ALLEGRO_FUSED_TP_BWD"] = "0"
    e0, ea0, f0 = m.compute_energy_forces(s.pos, s.species)
    for fwd, bwd in (("-1", "0"), ("-1", "-1")):
        os.environ["ALLEGRO_FUSED_TP"] = fwd
        os.environ["ALLEGRO_FUSED_TP_BWD"] = bwd
        e1, ea1, f1 = m.compute_energy_forces(s.pos, s.species)
        print(f"({L},{lmax}) n={s.n} fused fwd {fwd} bwd {bwd}: bitwise E {e1 == e0} F {np.array_equal(f1, f0)} "
              f"max|dF| {np.abs(f1 - f0).max():.3g} max|F| {np.abs(f0).max():.3g}", flush=True)
