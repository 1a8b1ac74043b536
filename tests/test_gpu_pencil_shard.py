"""Pencil sharding of the fused step (shard.PencilShardedSimulation), needs a B200.

Only one GPU is available here, so the multi-rank case runs its ranks in
lockstep on one device with the rank-order sum done by the test (exactly what
sum_in_rank_order does across processes): every rank advances only its tiles,
the union of the ranks' rows must equal the single-device run.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_19959_b200 as sv  # noqa: E402
from paper_2603_19959_b200.shard import PencilShardedSimulation  # noqa: E402

CASES = [dict(dim=3, n_base=6, levels=0, degree=2, n_x=32),
         dict(dim=3, n_base=5, levels=0, degree=1, n_x=16, bc="periodic")]


def _close(a, b, tol=1e-13):
    return np.abs(a - b).max() <= tol * np.abs(b).max()


@pytest.mark.parametrize("kw", CASES)
def test_world1_matches_simulation(kw):
    ref = sv.Simulation(sv.SimConfig(**kw, n_steps=3))
    tr = ref.advance(3).cpu().numpy()
    s = PencilShardedSimulation(sv.SimConfig(**kw, n_steps=3), 0, 1)
    ts = s.advance(3).cpu().numpy()
    assert len(s.owned_rows()) == s.f.shape[0]
    assert _close(s.f.cpu().numpy(), ref.f.cpu().numpy())
    np.testing.assert_allclose(ts[:, 2:], tr[:, 2:], rtol=1e-13, atol=1e-13 * abs(tr[0, 2]))
    np.testing.assert_allclose(ts[:, :2], tr[:, :2], rtol=1e-10)


@pytest.mark.parametrize("kw", CASES)
@pytest.mark.parametrize("world", [2, 3])
def test_ranks_in_lockstep_match_simulation(kw, world):
    n_steps = 3
    ref = sv.Simulation(sv.SimConfig(**kw, n_steps=n_steps))
    tr = ref.advance(n_steps).cpu().numpy()
    sims = [PencilShardedSimulation(sv.SimConfig(**kw, n_steps=n_steps), r, world)
            for r in range(world)]
    n = sims[0].f.shape[1]
    tabs = [torch.empty((n_steps, 5), dtype=torch.float64, device="cuda") for _ in sims]

    def rank_sum(parts):   # sum_in_rank_order
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p
        return acc

    for s in sims:
        s._fused_step_deferred(s._e, mode=2)
    tot = rank_sum([s._fold_partials(False).clone() for s in sims])
    for s in sims:
        s._take_sums(tot)
    for k in range(n_steps):
        for s, t in zip(sims, tabs):
            s._field_chain(s._e, t[k, 0:2], None)
        last = k + 1 == n_steps
        parts = []
        for s in sims:
            if last:
                s._fused_step_deferred(s._e, final=True, mom_out3=s._part[n:])
                s._part[:n].zero_()
                parts.append(s._part.clone())
            else:
                s._fused_step_deferred(s._e)
                parts.append(s._fold_partials(True).clone())
        tot = rank_sum(parts)
        for s, t in zip(sims, tabs):
            if last:
                t[k, 2:5].copy_(tot[n:])
            else:
                s._take_sums(tot, t[k, 2:5])
    rows = [s.owned_rows() for s in sims]
    allr = np.concatenate(rows)
    assert len(np.unique(allr)) == len(allr) == sims[0].f.shape[0]   # disjoint cover
    fref = ref.f.cpu().numpy()
    for s, r in zip(sims, rows):
        assert _close(s.f.cpu().numpy()[r], fref[r])
    for t in tabs:
        tt = t.cpu().numpy()
        np.testing.assert_allclose(tt[:, 2:], tr[:, 2:], rtol=1e-13, atol=1e-13 * abs(tr[0, 2]))
        np.testing.assert_allclose(tt[:, :2], tr[:, :2], rtol=1e-10)
