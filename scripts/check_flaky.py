"""Repeat the C2 3xTF32 force evaluation to expose nondeterminism (diagnostics)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("ALG_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2303_08169_b200 as pb  # noqa: E402
from oracle import allegro as oa, weights_io  # noqa: E402
from synth import configs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
s = configs.system("C2")
wf = configs.weight_file("C2")
ref = oa.energy_forces(weights_io.read(wf), s.pos, s.species, s.box)
errs = []
m = pb.Allegro(wf, s.box, precision=pb.PREC_3XTF32)
for it in range(n):
    e, ea, F = m.compute_energy_forces(s.pos, s.species)
    errs.append(float(np.abs(F - ref["forces"]).max()))
m.close()
bad = sum(x > 1e-4 for x in errs)
print(os.environ.get("TAG", ""), "bad", bad, "of", n, "max", "%.2e" % max(errs), flush=True)
