"""Step time of small boxes (launch / synchronisation bound regime) on one GPU."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2303_08169_b200 as pb  # noqa: E402
from synth import configs  # noqa: E402

for name, lat, cells in (("C1", "fcc", (1, 1, 1)), ("C2", "fcc", (4, 4, 4)), ("1728", "bcc", (6, 6, 6)),
                         ("6912", "bcc", (12, 12, 6)), ("13824", "bcc", (12, 12, 12))):
    cfg = configs.Config(name, lat, cells, 6.0 if name != "C1" else 5.0, 3 if name != "C1" else 2, 1, name)
    s = configs.system(cfg)
    m = pb.Allegro(configs.weight_file(cfg), s.box, n_atoms=s.n, precision=pb.PREC_3XTF32,
                   stream=torch.cuda.current_stream().cuda_stream)
    m.md_set_state(s.species, s.pos, s.vel)
    m.md_step(5, 0.5)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 50
    m.md_step(n, 0.5)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(json.dumps({"system": name, "atoms": s.n, "ms_per_step": round(ms, 3),
                      "atom_steps_per_s": round(s.n / ms * 1e3, 1), "launches_per_step": None}), flush=True)
    m.close()
