"""Per-rank device work of an N-rank x-slab run, emulated on ONE GPU.

The ranks' own advance() generators (shard.ShardedSimulation.advance_steps) are driven in
lockstep exactly like shard.Collectives.lockstep -- no kernel waits on another rank's
kernel, the exchanges are serviced on the host between the ranks' segments -- with CUDA
events around every rank segment and every exchange.  A rank's segments are its own
kernels (V, the row-chunked slab X.X with its halo pack / unpack, field chain), so their
sum is what that rank's GPU would execute per step at N GPUs; the exchange segments are
device copies here (over NVLink/NCCL on a real node: their bytes are reported).  This is a
PROJECTION of the compute part of an N-GPU step, not a scaling measurement.

  python tools/rank_projection.py --config cfg5 --world 4 [--steps 3]
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
from paper_2603_19959_b200 import shard  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--world", type=int, default=4)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--kernels", action="store_true", help="also list kernel time per rank-step")
ap.add_argument("--pencils", action="store_true",
                help="pencil sharding (PencilShardedSimulation, uniform meshes) instead of x-slabs")
args = ap.parse_args()
W, K = args.world, args.steps
cfg = sv.SimConfig(**bench.CONFIGS[args.config], n_steps=K)
cls = shard.PencilShardedSimulation if args.pencils else shard.ShardedSimulation
sims = [cls(cfg, r, W) for r in range(W)]


def timed_lockstep(gens):
    """Collectives.lockstep with events: (kind, rank, start, end) per segment."""
    segs = []
    world = len(gens)

    def resume(r, g, first):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        try:
            q = next(g) if first else g.send(None)
        except StopIteration:
            q = None
        b.record()
        segs.append(("rank", r, a, b))
        return q

    reqs = [resume(r, g, True) for r, g in enumerate(gens)]
    xbytes = 0
    while any(q is not None for q in reqs):
        kind = reqs[0][0]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if kind == "sum":
            parts = torch.stack([q[1].reshape(-1) for q in reqs])
            tot = torch.empty_like(parts[0])
            shard.ordered_sum(parts, tot)
            for q in reqs:
                q[1].view(-1).copy_(tot)
            xbytes += parts.numel() * 8
        elif kind == "allgather":
            cat = torch.cat([q[1] for q in reqs])
            for q in reqs:
                shard.gather_index(cat, q[3].index, q[2])
            xbytes += cat.numel() * 8
        elif kind == "halo":
            for r, q in enumerate(reqs):
                fr_l, fr_r = q[1][2], q[1][3]
                left, right = reqs[(r - 1) % world], reqs[(r + 1) % world]
                if fr_l.numel():
                    fr_l.copy_(left[1][0])
                    xbytes += fr_l.numel() * 8
                if fr_r.numel():
                    fr_r.copy_(right[1][1])
                    xbytes += fr_r.numel() * 8
            for q in reqs:
                q[2]()
        b.record()
        segs.append(("exchange", -1, a, b))
        reqs = [resume(r, g, False) for r, g in enumerate(gens)]
    return segs, xbytes


tabs = [torch.empty((K, 5), dtype=torch.float64, device="cuda") for _ in sims]
timed_lockstep([s.advance_steps(K, t) for s, t in zip(sims, tabs)])   # warm-up
torch.cuda.synchronize()
if args.kernels:
    import collections

    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        segs, xbytes = timed_lockstep([s.advance_steps(K, t) for s, t in zip(sims, tabs)])
        torch.cuda.synchronize()
    agg = collections.defaultdict(lambda: [0.0, 0])
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            k = e.name.split("(")[0][:50]
            agg[k][0] += (e.time_range.end - e.time_range.start) / 1e3
            agg[k][1] += 1
    print(json.dumps({k: [round(v[0] / (W * K), 4), v[1] / (W * K)] for k, v in
                      sorted(agg.items(), key=lambda kv: -kv[1][0])[:14]}, indent=0))
else:
    segs, xbytes = timed_lockstep([s.advance_steps(K, t) for s, t in zip(sims, tabs)])
torch.cuda.synchronize()
per_rank = [0.0] * W
exch = 0.0
for kind, r, a, b in segs:
    t = a.elapsed_time(b)
    if kind == "rank":
        per_rank[r] += t
    else:
        exch += t
n_v = len(sims[0].vweights)
dofs = n_v * sims[0].xgrid.n_dofs
print(json.dumps({
    "config": args.config, "world": W, "steps": K, "phase_dofs": dofs,
    "sharding": "pencils" if args.pencils else "x-slabs",
    "rank_ms_per_step": [round(t / K, 4) for t in per_rank],
    "max_rank_ms_per_step": round(max(per_rank) / K, 4),
    "exchange_copy_ms_per_step_here": round(exch / K, 4),
    "exchange_bytes_per_step_all_ranks": xbytes // K,
    "note": "projection: per-rank device work of a W-rank x-slab step emulated in lockstep "
            "on one GPU (exchanges are device copies here)"}))
