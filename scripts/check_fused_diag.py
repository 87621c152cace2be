"""Debugging aid: the (3,1) model on C1, fused layer-1 kernel under ALLEGRO_TPL_DIAG masks."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2303_08169_b200 as pb
from synth import configs, weights as sw

s = configs.system("C1")
wf = "/tmp/m31.algw"
sw.write(wf, 3, 1, 5.0, sw.generate(3, 1, 0), sw.nbar_for(5.0), (1.0, 1.0), (0.0, 0.0))
m = pb.Allegro(wf, s.box, n_atoms=s.n)
os.environ["ALLEGRO_FUSED_TP"] = os.environ.get("MASK", "2")
try:
    e1, a1, f1 = m.compute_energy_forces(s.pos, s.species)
    print("diag", os.environ.get("ALLEGRO_TPL_DIAG"), "ok", e1)
except Exception as ex:
    print("diag", os.environ.get("ALLEGRO_TPL_DIAG"), ex)
