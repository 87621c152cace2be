"""CTA-pair contractions (cta_group::2, M = 256; csrc/tc_gemm.cu PAIR mode) against
the sibling-CTA path on the two-N-tile shapes: bit-identical outputs (same MMAs, same accumulation
order per element), including odd M-tile counts (the pair's second CTA without rows) and the
two-operand (A2) form.  Each mode runs in its own process (the switch is read once per process)."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_pair_matches_sibling_bitwise(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = {}
    for mode in ("0", "1"):
        f = str(tmp_path / f"pair{mode}.npz")
        r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "check_pair.py"), f], cwd=ROOT,
                           env={**os.environ, "ALLEGRO_TC_PAIR": mode}, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
        out[mode] = np.load(f)
    a, b = out["0"], out["1"]
    assert set(a.files) == set(b.files) and a.files
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
