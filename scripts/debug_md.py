"""Step-by-step GPU vs oracle trajectory comparison (debug aid; test infrastructure)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2303_08169_b200 as pb
from oracle import allegro as oa, md, weights_io
from synth import configs, nh3

wf = configs.weight_file('C2')
model = weights_io.read(wf)
s = nh3.maxwell_boltzmann(nh3.nh3_box('fcc', (2, 2, 2)), 200.0)
fn = lambda p: (lambda r: (r['energy'], r['forces']))(oa.energy_forces(model, p, s.species, s.box))
m = pb.Allegro(wf, s.box)
m.md_set_state(s.species, s.pos, s.vel)
p, v, f = m.md_get_state()
po, vo, fo = nh3.wrap_positions(s.pos, s.box), s.vel.copy(), fn(s.pos)[1]
print('step0 |dF|', np.abs(f - fo).max(), '|dp|', np.abs(p - po).max())
for step in range(1, 11):
    r = m.md_step(1, 0.5)
    p, v, f = m.md_get_state()
    po, vo, fo, lg = md.verlet(fn, po, vo, s.species, s.box, 0.5, 1, forces=fo)
    dp = p - po; dp -= s.box * np.round(dp / s.box)
    print(step, 'gpu E', r.e_pot, r.e_kin, r.e_total, '| oracle', lg[-1][0], lg[-1][1], sum(lg[-1]),
          '| dp', np.abs(dp).max(), 'dv', np.abs(v - vo).max(), 'dF', np.abs(f - fo).max(), flush=True)
