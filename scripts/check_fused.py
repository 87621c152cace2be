"""A/B of the fused kernels against the unfused path (3xTF32) on the given configs:
(a) the fused last layer (k_last) alone and the fused two-body kernels alone -- expected
bit-identical; (b) everything fused vs nothing
fused -- equal up to the re-associated Gamma-bar sum of k_tpl_bwd; and, for small boxes, the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2303_08169_b200 as pb
from oracle import allegro as oa, weights_io
from synth import configs


def run(m, s, fwd, bwd, last, merge="1", tb="0"):
    os.environ["ALLEGRO_FUSED_2B"] = tb
    os.environ["ALLEGRO_FUSED_TP"] = fwd
    os.environ["ALLEGRO_FUSED_TP_BWD"] = bwd
    os.environ["ALLEGRO_FUSED_LAST"] = last
    os.environ["ALLEGRO_MERGE_XBAR"] = merge
    return m.compute_energy_forces(s.pos, s.species)


for cfg in sys.argv[1:] or ["C1", "C2"]:
    s = configs.system(cfg)
    wf = configs.weight_file(cfg)
    m = pb.Allegro(wf, s.box, precision=pb.PREC_3XTF32, n_atoms=s.n)
    e0, ea0, f0 = run(m, s, "0", "0", "0", "0")
    eL, eaL, fL = run(m, s, "0", "0", "1", "0")
    eT, eaT, fT = run(m, s, "0", "0", "0", "0", "3")
    e1, ea1, f1 = run(m, s, "-1", "-1", "1", "1", "3")
    line = (f"{cfg}: last layer fused vs not: bitwise E {eL == e0} E_i {np.array_equal(eaL, ea0)} F {np.array_equal(fL, f0)}"
            f" | two-body fused vs not: bitwise E {eT == e0} E_i {np.array_equal(eaT, ea0)} F {np.array_equal(fT, f0)}"
            f" | all fused vs none: bitwise E {e1 == e0} F {np.array_equal(f1, f0)} max|dF| {np.abs(f1 - f0).max():.3g}")
    if s.n < 2000:
        ref = oa.energy_forces(weights_io.read(wf), s.pos, s.species, s.box)
        line += f" | vs oracle max|dF| {np.abs(f1 - ref['forces']).max():.3g}"
    print(line, flush=True)
