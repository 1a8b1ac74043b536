"""Wall time per step of advance() eager vs replayed from a CUDA graph (per config)."""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402

import paper_2603_19959_b200 as sv  # noqa: E402
from bench import CONFIGS  # noqa: E402

K = 20
for name in sys.argv[1:] or ["cfg1", "cfg3", "cfg4", "cfg2"]:
    sim = sv.Simulation(sv.SimConfig(**CONFIGS[name], n_steps=K))
    res = {}
    for mode in ("eager", "graph", "eager", "graph"):
        fn = sim.advance if mode == "eager" else sim.advance_graph
        for _ in range(3):
            fn(K)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            fn(K)
        torch.cuda.synchronize()
        res[mode] = (time.perf_counter() - t) / (5 * K) * 1e3
    print(f"{name}: ms/step eager {res['eager']:.4f} graph {res['graph']:.4f}")
