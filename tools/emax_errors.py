"""E_max record differences vs the reference's 200-step runs (tests/golden/run_cfg*.npz)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2603_19959_b200 as sv  # noqa: E402

CFGS = {
    "cfg1": dict(dim=3, n_base=16, levels=0, degree=1, n_x=16),
    "cfg2": dict(dim=3, n_base=32, levels=0, degree=2, n_x=64),
    "cfg3": dict(dim=3, n_base=4, levels=1, degree=2, n_x=64),
    "cfg4": dict(dim=3, n_base=4, levels=2, degree=3, n_x=128),
}
for name, kw in CFGS.items():
    g = np.load(os.path.join(ROOT, "tests", "golden", f"run_{name}.npz"))
    res = sv.run(sv.SimConfig(**kw, n_steps=200))
    rec = np.array([[r.t, r.e_max, r.m0, r.m1, r.m2, r.e_field, r.e_total] for r in res.records])
    ref = g["records"]
    d = np.abs(rec[:, 1] - ref[:, 1])
    print(name, "E_max normwise", d.max() / ref[0, 1], "relative max", (d / ref[:, 1]).max(),
          "e_field rel", (np.abs(rec[:, 5] - ref[:, 5]) / ref[:, 5]).max(),
          "m0 rel", (np.abs(rec[:, 2] - ref[:, 2]) / ref[:, 2]).max(),
          "rate", res.fit.rate, float(g["rate"]))
