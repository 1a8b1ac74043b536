"""Time the x-slab sharded step (world 1, self halo) against Simulation on one config."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402

import paper_2603_19959_b200 as sv  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_2603_19959_b200.shard import ShardedSimulation  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = sv.SimConfig(**CONFIGS[cfg], n_steps=K)
for name, mk in (("sharded-x1", lambda: ShardedSimulation(c, 0, 1)), ("simulation", lambda: sv.Simulation(c))):
    s = mk()
    s.advance(2)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    s.advance(K)
    b.record()
    torch.cuda.synchronize()
    print(name, cfg, a.elapsed_time(b) / K, "ms/step")
    del s
    torch.cuda.empty_cache()
