"""Coefficient errors vs the reference's multi-step runs (tests/golden/coeffs_*.npz)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2603_19959_b200 as sv  # noqa: E402
COEF_CFGS = {
    "cfg1": dict(dim=3, n_base=16, levels=0, degree=1, n_x=16),
    "cfg2": dict(dim=3, n_base=32, levels=0, degree=2, n_x=64),
    "cfg3": dict(dim=3, n_base=4, levels=1, degree=2, n_x=64),
    "cfg4": dict(dim=3, n_base=4, levels=2, degree=3, n_x=128),
}

for name in sys.argv[1:] or list(COEF_CFGS):
    g = np.load(os.path.join(ROOT, "tests", "golden", f"coeffs_{name}.npz"))
    sim = sv.Simulation(sv.SimConfig(**COEF_CFGS[name], n_steps=200))
    done = 0
    for n in [int(v) for v in g["save_at"]]:
        sim.advance(n - done)
        done = n
        f = sim.f.cpu().numpy().ravel()[g["sample_idx"]]
        ref = g[f"s{n}_val"]
        fmax = float(g[f"s{n}_fmax"])
        err = np.abs(f - ref)
        out = {"cfg": name, "step": n, "normwise": err.max() / fmax}
        for thr in (1e-3, 1e-2, 1e-1):
            big = np.abs(ref) >= thr * fmax
            out[f"rel@{thr:g}"] = float((err[big] / np.abs(ref[big])).max())
        print(json.dumps(out), flush=True)
