"""Time k_field_chain alone on the GPU (events around single launches) on the cfg2 plans."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402

import paper_2603_19959_b200 as sv  # noqa: E402
from bench import CONFIGS  # noqa: E402

sim = sv.Simulation(sv.SimConfig(**CONFIGS["cfg2"], n_steps=4))
sim.advance(2)
tab = torch.empty(4, 5, dtype=torch.float64, device="cuda")
for _ in range(5):
    sim._field_chain(sim._e, tab[0, 0:2], tab[1, 2:5])
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
for a, b in ev:   # one launch between its own events, the GPU idle before it
    torch.cuda._sleep(2_000_000)
    a.record()
    sim._field_chain(sim._e, tab[0, 0:2], tab[1, 2:5])
    b.record()
torch.cuda.synchronize()
t = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
print("field chain us (median of 50, GPU)", t[len(t) // 2])
