"""Time k_step_fused at config 2 (or --config) with CUDA events, steady-state launches.

  python tools/fused_probe.py [--config cfg2] [--steps 20]
Prints ms per fused launch, GB/s at 16 B/DOF and the fraction of MEASURED_PEAKS hbm_gbs.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_19959_b200 as sv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--steps", type=int, default=20)
args = ap.parse_args()
sim = sv.Simulation(sv.SimConfig(**bench.CONFIGS[args.config], n_steps=args.steps))
assert sim.fused_step_supported()
sim.advance(5)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
      for _ in range(args.steps)]
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
sim.advance(args.steps)
b.record()
torch.cuda.synchronize()
step_ms = a.elapsed_time(b) / args.steps
sim.advance(args.steps, v_events=ev)
torch.cuda.synchronize()
ms = float(np.mean([x.elapsed_time(y) for x, y in ev[:-1]]))
gbs = 16 * sim.f.numel() / (ms * 1e-3) / 1e9
peak, _ = bench.measured_peaks()
print(json.dumps({"config": args.config, "fused_ms": ms, "step_ms": step_ms, "gbs": gbs,
                  "frac": gbs / peak, "variant": os.environ.get("SLDG_FUSED_VARIANT", "")}))
