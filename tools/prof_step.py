"""Small driver for ncu: build a config's Simulation and run a few pipelined steps."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402

import paper_2603_19959_b200 as sv  # noqa: E402
from bench import CONFIGS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sim = sv.Simulation(sv.SimConfig(**CONFIGS[cfg], n_steps=n))
sim.advance(n)
torch.cuda.synchronize()
print("ok", cfg, n)
