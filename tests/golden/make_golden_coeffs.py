"""Multi-step COEFFICIENT goldens from the reference (build container only).

Run:  python tests/golden/make_golden_coeffs.py cfg1 cfg3 cfg4 cfg2

For each config, runs the REFERENCE package's own Simulation (sldg_vlasov.driver,
driver.py:194-253: t=0 record, then step() n_steps times) and, after the steps listed in
SAVE_AT, stores a seeded sample of DG coefficients of f, max|f| and the column sums of f.
Writes tests/golden/coeffs_<cfg>.npz.

These pin SURVEY.md §8(c) parity protocol (2): the GPU state after 5 and 200 steps must
match the reference per coefficient (<= 1e-12 max|f|).  /root/reference does not exist on
the GPU box; only the .npz files travel.
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True
from sldg_vlasov import driver as drv  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CFGS = {
    "cfg1": dict(dim=3, n_base=16, levels=0, degree=1, n_x=16),
    "cfg2": dict(dim=3, n_base=32, levels=0, degree=2, n_x=64, workers=8),
    "cfg3": dict(dim=3, n_base=4, levels=1, degree=2, n_x=64),
    "cfg4": dict(dim=3, n_base=4, levels=2, degree=3, n_x=128),
}
SAVE_AT = (1, 5, 50, 200)
N_SAMPLE = 8192


def main(names):
    for name in names:
        t0 = time.perf_counter()
        cfg = drv.SimConfig(**CFGS[name], n_steps=max(SAVE_AT))
        sim = drv.Simulation(cfg)
        rng = np.random.default_rng(4242)
        idx = np.sort(rng.choice(sim.f.size, size=min(N_SAMPLE, sim.f.size), replace=False))
        # add the largest coefficients so the per-coefficient relative check sees the bulk
        big = np.argsort(np.abs(sim.f).ravel())[-512:]
        idx = np.unique(np.concatenate([idx, big]))
        out = {"sample_idx": idx, "save_at": np.array(SAVE_AT)}
        recs = [sim.diagnostics(sim.field_solve())]
        for n in range(1, cfg.n_steps + 1):
            recs.append(sim.step())
            if n in SAVE_AT:
                out[f"s{n}_val"] = sim.f.ravel()[idx]
                out[f"s{n}_fmax"] = np.array(np.abs(sim.f).max())
                out[f"s{n}_colsum"] = sim.f.sum(axis=0)
                print(name, n, f"{time.perf_counter() - t0:.1f}s", flush=True)
        out["records"] = np.array([[r.t, r.e_max, r.m0, r.m1, r.m2, r.e_field, r.e_total]
                                   for r in recs])
        path = os.path.join(HERE, f"coeffs_{name}.npz")
        np.savez_compressed(path, **out)
        print("wrote", path, os.path.getsize(path) // 1024, "KiB",
              f"{time.perf_counter() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg1", "cfg3", "cfg4", "cfg2"])
