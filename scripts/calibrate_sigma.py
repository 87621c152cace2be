"""Write synth/calibration.json: the energy scale sigma of each model.

Reading row 10 of SURVEY.md §8(c): mu_Z = 0, sigma_H = sigma_N = sigma chosen so
that RMS |F| = 1 eV/A on the calibration box (C2 geometry: fcc 4^3 liquid NH3,
1,024 atoms, step 0) at the model's r_c.  Forces are linear in sigma (mu = 0),
so sigma = 1 / RMS|F|(sigma = 1).  Calls only oracle/ (and synth/ for inputs).
"""
import json
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import allegro, weights_io  # noqa: E402
from synth import nh3, weights as sw  # noqa: E402

MODELS = [(2, 1, 5.0), (2, 2, 6.0), (3, 2, 6.0), (3, 1, 6.0), (3, 0, 6.0)]


def main():
    box = nh3.nh3_box("fcc", (4, 4, 4))
    out = sw.load_calibration()
    for L, lmax, rc in MODELS:
        key = sw.model_key(L, lmax, rc, 0)
        path = os.path.join(tempfile.gettempdir(), f"cal_{key}.algw")
        sw.make_weight_file(path, L, lmax, rc, seed=0, sigma=1.0)
        m = weights_io.read(path)
        t0 = time.time()
        r = allegro.energy_forces(m, box.pos, box.species, box.box)
        rms = float(np.sqrt(np.mean(np.sum(r["forces"] ** 2, axis=1))))
        out[key] = 1.0 / rms
        print(key, "rms|F|(sigma=1) =", rms, "sigma =", out[key], f"({time.time() - t0:.1f} s)", flush=True)
        with open(sw._CAL_PATH, "w") as f:
            json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
