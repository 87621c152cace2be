"""Quick A/B of the fused TP + TP-linear forward (tp_fused.cu) against the unfused path and the
oracle on C1 and C2 (3xTF32)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2303_08169_b200 as pb
from oracle import allegro as oa, weights_io
from synth import configs

for cfg in sys.argv[1:] or ["C1", "C2"]:
    s = configs.system(cfg)
    wf = configs.weight_file(cfg)
    m = pb.Allegro(wf, s.box, precision=pb.PREC_3XTF32, n_atoms=s.n)
    os.environ["ALLEGRO_FUSED_TP"] = "0"
    os.environ["ALLEGRO_FUSED_TP_BWD"] = "0"
    e0, ea0, f0 = m.compute_energy_forces(s.pos, s.species)
    os.environ["ALLEGRO_FUSED_TP"] = "-1"
    os.environ["ALLEGRO_FUSED_TP_BWD"] = "-1"
    e1, ea1, f1 = m.compute_energy_forces(s.pos, s.species)
    line = f"{cfg}: E fused {e1:.9f} unfused {e0:.9f} bitwise {e1 == e0} {np.array_equal(f1, f0)} max|dF| {np.abs(f1 - f0).max():.3g}"
    if s.n < 2000:
        ref = oa.energy_forces(weights_io.read(wf), s.pos, s.species, s.box)
        line += f" | vs oracle max|dF| {np.abs(f1 - ref['forces']).max():.3g}"
    print(line, flush=True)
