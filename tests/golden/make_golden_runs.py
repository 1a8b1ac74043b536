"""Full 200-step reference runs (build container only): E_max series, fit, invariants.

Run:  python tests/golden/make_golden_runs.py cfg1 cfg3 cfg4 [cfg2]
Writes tests/golden/run_<cfg>.npz from the REFERENCE package's run(SimConfig)
(sldg_vlasov.driver.run, driver.py:275-276), workers=8 for cfg2.
"""
import os
import sys

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

for name in sys.argv[1:]:
    res = drv.run(drv.SimConfig(**CFGS[name], n_steps=200))
    rec = np.array([[r.t, r.e_max, r.m0, r.m1, r.m2, r.e_field, r.e_total] for r in res.records])
    np.savez_compressed(os.path.join(HERE, f"run_{name}.npz"), records=rec,
                        rate=np.array(np.nan if res.fit.rate is None else res.fit.rate),
                        n_peaks=np.array(res.fit.n_peaks), mass_error=np.array(res.mass_error),
                        energy_drift=np.array(res.energy_drift), wall=np.array(res.wall_time))
    print(name, res.fit.rate, res.fit.n_peaks, res.mass_error, res.energy_drift, res.wall_time)
