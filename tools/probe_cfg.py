"""ms/step of advance() for an ad-hoc config, fused vs forced-unfused."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402

import paper_2603_19959_b200 as sv  # noqa: E402

kw = eval("dict(" + sys.argv[1] + ")")
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
for fused in (True, False):
    s = sv.Simulation(sv.SimConfig(**kw, n_steps=K))
    if not fused:
        s._fused_ok = False
    s.advance(3)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    s.advance(K)
    b.record()
    torch.cuda.synchronize()
    print(kw, "fused" if fused else "unfused", s.fused_step_supported(), a.elapsed_time(b) / K)
    del s
