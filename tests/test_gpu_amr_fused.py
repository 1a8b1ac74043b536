"""The one-pass AMR step (csrc/amr_fused.cuh, sldg_amr_step) against the separate passes
(k_sweep_stream + worklist + write-back, then k_xx_tiles X.X) on the same states.

With SLDG_AMR_FUSED=on, Simulation.advance() takes the one-pass step for every step but the
last when the library supports the plans (the default, off, keeps the separate passes: they
measure faster).  Both compute the same
operators; the one-pass step re-associates X(X(u)) as one composed stencil and sums the
moments of the intermediate through (A^T + B^T) xw, so states agree to ~1e-16 relative per
step and the records to ~1e-14 (the separate passes are the ones pinned to the oracle:
test_gpu_multistep, test_gpu_damping, test_gpu_reference_suite).  Cluster shapes covered:
one CTA per row (n_x 64, 32, 24, 40, 30) and four-CTA clusters exchanging slices through
DSMEM (n_x 512); races: tests/test_gpu_schedule_fuzz.py ("amr_onepass").
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_19959_b200 as sv  # noqa: E402

CASES = [
    dict(dim=3, n_base=4, levels=1, degree=2, n_x=64),                    # cfg3 shape
    dict(dim=3, n_base=4, levels=2, degree=3, n_x=32),                    # cfg4 shape (Q3)
    dict(dim=3, n_base=6, levels=1, degree=2, n_x=24, bc="periodic"),
    dict(dim=3, n_base=4, levels=1, degree=2, n_x=512),                   # 4-CTA clusters
    dict(dim=3, n_base=4, levels=1, degree=2, n_x=40, degree_x=3),
    dict(dim=3, n_base=4, levels=1, degree=2, n_x=30, degree_x=1),
    dict(dim=3, n_base=8, levels=1, degree=1, n_x=32),
]


def _run(kw, mode, n_steps, monkeypatch):
    monkeypatch.setenv("SLDG_AMR_FUSED", mode)
    sim = sv.Simulation(sv.SimConfig(**kw, n_steps=n_steps))
    table = sim.advance(n_steps).cpu().numpy()
    return sim, sim.f.cpu().numpy(), table


@pytest.mark.parametrize("kw", CASES, ids=lambda k: "-".join(f"{a}{b}" for a, b in k.items()))
def test_one_pass_amr_step_matches_separate_passes(kw, monkeypatch):
    n_steps = 4
    ref, fr, tr = _run(kw, "off", n_steps, monkeypatch)
    assert not ref.amr_step_supported()
    sim, f, t = _run(kw, "on", n_steps, monkeypatch)
    assert sim.amr_step_supported(), "one-pass AMR step not taken"
    assert np.abs(f - fr).max() <= 1e-13 * np.abs(fr).max()
    np.testing.assert_allclose(t[:, 2:], tr[:, 2:], rtol=1e-13, atol=1e-14 * abs(tr[0, 2]))
    assert np.abs(t[:, 0] - tr[:, 0]).max() <= 1e-11 * tr[0, 0]
    np.testing.assert_allclose(t[:, 1], tr[:, 1], rtol=1e-10)


def test_one_pass_amr_step_is_deterministic(monkeypatch):
    kw = CASES[3]
    _, f1, t1 = _run(kw, "on", 3, monkeypatch)
    _, f2, t2 = _run(kw, "on", 3, monkeypatch)
    np.testing.assert_array_equal(f1, f2)
    np.testing.assert_array_equal(t1, t2)


def test_uniform_mesh_keeps_the_uniform_fused_step(monkeypatch):
    monkeypatch.setenv("SLDG_FUSED", "force")
    monkeypatch.setenv("SLDG_AMR_FUSED", "on")
    sim = sv.Simulation(sv.SimConfig(dim=3, n_base=8, levels=0, degree=2, n_x=64, n_steps=2))
    assert sim.fused_step_supported() and not sim.amr_step_supported()
