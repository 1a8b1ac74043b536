"""advance(n) on a config once (for ncu captures of single launches).
  python tools/cfg_advance.py [--config cfg5] [--steps 3]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_19959_b200 as sv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--steps", type=int, default=3)
args = ap.parse_args()
sim = sv.Simulation(sv.SimConfig(**bench.CONFIGS[args.config], n_steps=args.steps))
sim.advance(args.steps)
torch.cuda.synchronize()
print("ok")
