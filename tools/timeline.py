"""Device timeline of advance(n) (torch.profiler / CUPTI; nsys is not in the image):
per-kernel busy time and the idle gaps between consecutive kernels on the stream.

  python tools/timeline.py [--config cfg5] [--steps 5]
"""
import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2603_19959_b200 as sv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--steps", type=int, default=5)
args = ap.parse_args()
sim = sv.Simulation(sv.SimConfig(**bench.CONFIGS[args.config], n_steps=args.steps))
sim.advance(2)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    sim.advance(args.steps)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev = sorted(ev, key=lambda e: e.time_range.start)
busy = collections.defaultdict(float)
gaps = []
for a, b in zip(ev, ev[1:]):
    gaps.append((b.time_range.start - a.time_range.end, a.name[:40], b.name[:40]))
for e in ev:
    busy[e.name.split("(")[0][:60]] += e.time_range.end - e.time_range.start
span = ev[-1].time_range.end - ev[0].time_range.start
out = {"config": args.config, "steps": args.steps, "span_ms": span / 1e3,
       "busy_ms": sum(busy.values()) / 1e3,
       "gap_ms": sum(max(g[0], 0) for g in gaps) / 1e3,
       "top_kernels_ms": {k: round(v / 1e3, 3) for k, v in
                          sorted(busy.items(), key=lambda kv: -kv[1])[:10]},
       "largest_gaps_us": [(round(g[0], 1), g[1], g[2]) for g in sorted(gaps)[::-1][:8]]}
print(json.dumps(out, indent=1))
