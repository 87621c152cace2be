"""The measured A/B switches of the contraction path stay correct: every variant
of the C2 evaluation agrees with the oracle within D20 and with the default build's result.

Each variant runs in its own process because the library reads the switches once:
ALLEGRO_TC_TMASTORE=0 (STG-scatter epilogue instead of TMA stores), ALLEGRO_FUSE_R2=0 and
ALLEGRO_FUSE_ROWDOT=0 (standalone row-dot passes), ALLEGRO_TC_STOREHINT=1 (L2 policy on the
stores), ALLEGRO_TC_PAIR_MULTI=0 / ALLEGRO_TC_PAIR_STORE=0 (single-CTA N-tiles instead of CTA pairs),
ALLEGRO_TC_STORE4=0 (two output slots per epilogue warp).  Switches that change only where bytes go are bit-identical to the default; the row-dot
switches change a summation order (tolerance)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import allegro as oa, weights_io
from synth import configs

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
E_TOL, F_TOL = 1e-5, 1e-4

_CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2303_08169_b200 as pb
from synth import configs
s = configs.system("C2")
m = pb.Allegro(configs.weight_file("C2"), s.box, precision=pb.PREC_3XTF32)
e, ea, f = m.compute_energy_forces(s.pos, s.species)
np.save(sys.argv[2], np.concatenate([[e], ea, f.ravel()]))
"""


def _run(tmp_path, name, env_extra):
    out = str(tmp_path / f"{name}.npy")
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", _CHILD, ROOT, out], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


@pytest.fixture(scope="module")
def reference():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    s = configs.system("C2")
    return s, oa.energy_forces(weights_io.read(configs.weight_file("C2")), s.pos, s.species, s.box)


@pytest.mark.parametrize("name,env,bitwise", [
    ("tmastore0", {"ALLEGRO_TC_TMASTORE": "0"}, True),
    ("storehint1", {"ALLEGRO_TC_STOREHINT": "1"}, True),
    ("fuse_r2_0", {"ALLEGRO_FUSE_R2": "0"}, False),
    ("fuse_rowdot0", {"ALLEGRO_FUSE_ROWDOT": "0"}, False),
    # l = 2 contractions over four N-tiles as two CTA pairs vs four sibling CTAs (the row-dot
    # partials are summed in a different grouping: tolerance), and the paired plain store
    ("pair_multi0", {"ALLEGRO_TC_PAIR_MULTI": "0"}, False),
    ("pair_store0", {"ALLEGRO_TC_PAIR_STORE": "0"}, True),
    ("store4_0", {"ALLEGRO_TC_STORE4": "0"}, True),
])
def test_switch_variants(reference, tmp_path, name, env, bitwise):
    s, ref = reference
    base = _run(tmp_path, "default", {})
    var = _run(tmp_path, name, env)
    n = s.n
    for v in (base, var):
        assert abs(v[0] - ref["energy"]) <= E_TOL * np.abs(ref["e_atom"]).sum()
        assert np.abs(v[1 + n:].reshape(n, 3) - ref["forces"]).max() <= F_TOL
    if bitwise:
        assert np.array_equal(base, var)
    else:
        assert np.abs(var - base).max() <= 1e-5 * max(1.0, np.abs(base).max())
