"""SM clock and throttle reasons (NVML) while advance(n) runs on a config: is a long
AMR step power-capped?   python tools/amr_clocks.py [--config cfg5] [--steps 10]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_19959_b200 as sv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--steps", type=int, default=10)
args = ap.parse_args()
sim = sv.Simulation(sv.SimConfig(**bench.CONFIGS[args.config], n_steps=args.steps))
sim.advance(2)
torch.cuda.synchronize()
cs = bench.ClockSampler(0).start()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
a.record()
sim.advance(args.steps)
b.record()
torch.cuda.synchronize()
t1 = time.perf_counter()
cs.stop()
mhz = sorted(m for t, m, r in cs.samples if t0 <= t <= t1)
reasons = sorted({k for t, m, r in cs.samples if t0 <= t <= t1
                  for k, v in bench.ClockSampler.REASONS.items() if r & k})
print(json.dumps({"config": args.config, "ms_per_step": a.elapsed_time(b) / args.steps,
                  "sm_mhz_min": mhz[0] if mhz else None, "sm_mhz_median": mhz[len(mhz) // 2] if mhz else None,
                  "sm_mhz_max": mhz[-1] if mhz else None, "samples": len(mhz),
                  "reasons": [bench.ClockSampler.REASONS[k] for k in reasons]}))
