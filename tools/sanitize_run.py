"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

  compute-sanitizer --tool racecheck python tools/sanitize_run.py [which]

Covers k_step_fused (lead / steady / last-step modes) + k_field_chain on a uniform Q2 mesh
(N_x = 64, the headline row length), k_sweep_stream, k_vclassify/k_vitems + k_writeback on
AMR L1/L2 plans (hybrid and forced slow), and k_xx_tiles (X, X.X, rho/moments epilogues).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("SLDG_FUSED", "force")

import torch  # noqa: E402

import paper_2603_19959_b200 as sv  # noqa: E402


def fused():
    sim = sv.Simulation(sv.SimConfig(dim=3, n_base=4, levels=0, degree=2, n_x=64, n_steps=3))
    assert sim.fused_step_supported()
    sim.advance(3)


def sweep_uniform():
    sim = sv.Simulation(sv.SimConfig(dim=3, n_base=4, levels=0, degree=2, n_x=64))
    sim.fused_policy = "off"
    sim._fused_ok = None
    sim.step()


def amr():
    for lv, p, bc in ((1, 2, "absorbing"), (2, 3, "periodic")):
        for fs in (False, True):
            sim = sv.Simulation(sv.SimConfig(dim=3, n_base=4, levels=lv, degree=p, n_x=16,
                                             bc=bc, force_slow=fs))
            sim.step()
            sim.advance(2)


WHICH = {"fused": fused, "sweep": sweep_uniform, "amr": amr}

if __name__ == "__main__":
    for name in (sys.argv[1:] or list(WHICH)):
        WHICH[name]()
        torch.cuda.synchronize()
        print("ok", name, flush=True)
