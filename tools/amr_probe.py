"""Time advance() of an AMR config (default cfg5) with CUDA events; for ncu launch lists.

  python tools/amr_probe.py [--config cfg5] [--steps 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_19959_b200 as sv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--steps", type=int, default=3)
args = ap.parse_args()
sim = sv.Simulation(sv.SimConfig(**bench.CONFIGS[args.config], n_steps=args.steps))
sim.advance(1)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
sim.advance(args.steps)
b.record()
torch.cuda.synchronize()
print(json.dumps({"config": args.config, "ms_per_step": a.elapsed_time(b) / args.steps,
                  "plan": sim.sweep_plan.info()}))
