"""Race check by schedule fuzzing (needs a B200 and _lib/libsldg_fuzz.so).

compute-sanitizer (racecheck / synccheck / memcheck) is closed on this GPU pool
(profiles/r02_compute_sanitizer_refused.txt), so races are hunted the other way round:
libsldg_fuzz.so (tools/fuzz_build.sh, -DSLDG_FUZZ) sleeps a pseudo-random 0-2 us before
~1 in 4 bulk-copy issues, cp.async issues, mbarrier waits, pipeline barriers, cluster
barriers and worklist fetches, which scrambles the relative order of every producer and
consumer of the shared-memory rings, tile buffers, tables and worklists.  Each pipeline
below runs once with the normal library in this process and twice with the fuzzing
library in child processes; the results must be bit-identical.  Covered: the fused step
(lead / steady / last-step modes, field chain cluster) on the headline 64-cell rows,
the AMR path (stream sweep, per-cell worklist, write-back, X.X tiles), and the x-slab
pipeline with two ranks in lockstep (halo pack / unpack, slab X.X in chunks), and the
opt-in one-pass AMR step (one-CTA and four-CTA clusters).
"""
import hashlib
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FUZZ_LIB = os.path.join(ROOT, "paper_2603_19959_b200", "_lib", "libsldg_fuzz.so")

CASES = {
    "fused": dict(dim=3, n_base=8, levels=0, degree=2, n_x=64),
    "amr": dict(dim=3, n_base=4, levels=2, degree=3, n_x=32),
    "amr_periodic": dict(dim=3, n_base=6, levels=1, degree=2, n_x=24, bc="periodic"),
}


def digests():
    """Digest of the state and record table of every pipeline (run in this process)."""
    import paper_2603_19959_b200 as sv
    from paper_2603_19959_b200 import shard
    out = {}
    for name, kw in CASES.items():
        sim = sv.Simulation(sv.SimConfig(**kw, n_steps=4))
        table = sim.advance(4).cpu().numpy()
        f = sim.f.cpu().numpy()
        out[name] = hashlib.sha256(f.tobytes() + table.tobytes()).hexdigest()
    # the one-pass AMR step (opt-in): bulk-copy ring, per-cell cluster barrier, DSMEM
    # reads of the peers' slices, bulk stores
    os.environ["SLDG_AMR_FUSED"] = "on"
    try:
        for name, kw in (("amr_onepass", CASES["amr"]),
                         ("amr_onepass_cluster", dict(dim=3, n_base=4, levels=1, degree=2,
                                                      n_x=512))):
            sim = sv.Simulation(sv.SimConfig(**kw, n_steps=4))
            assert sim.amr_step_supported()
            table = sim.advance(4).cpu().numpy()
            out[name] = hashlib.sha256(sim.f.cpu().numpy().tobytes() + table.tobytes()).hexdigest()
    finally:
        os.environ.pop("SLDG_AMR_FUSED", None)
    kw = CASES["amr"]
    sims = [shard.ShardedSimulation(sv.SimConfig(**kw, n_steps=3), r, 2, n_chunks=3)
            for r in range(2)]
    tabs = [torch.empty((3, 5), dtype=torch.float64, device="cuda") for _ in sims]
    shard.Collectives.lockstep([s.advance_steps(3, t) for s, t in zip(sims, tabs)])
    h = hashlib.sha256()
    for s, t in zip(sims, tabs):
        h.update(s.f.cpu().numpy().tobytes())
        h.update(t.cpu().numpy().tobytes())
    out["slab2"] = h.hexdigest()
    return out


@pytest.mark.skipif(not os.path.exists(FUZZ_LIB), reason="libsldg_fuzz.so not built")
def test_results_survive_schedule_fuzzing():
    os.environ.setdefault("SLDG_FUSED", "force")
    ref = digests()
    env = dict(os.environ, SLDG_LIB_VARIANT="fuzz", SLDG_FUSED="force")
    code = ("import json, sys; sys.path.insert(0, %r); sys.path.insert(0, %r); "
            "import test_gpu_schedule_fuzz as t; "
            "from paper_2603_19959_b200 import _capi; "
            "assert _capi.LIB_PATH.endswith('libsldg_fuzz.so'); "
            "assert _capi.lib().sldg_build_flags() & 1; "
            "print(json.dumps(t.digests()))") % (ROOT, os.path.join(ROOT, "tests"))
    for _ in range(2):
        res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                             text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-2000:]
        got = json.loads(res.stdout.strip().splitlines()[-1])
        assert got == ref, {k: (got[k] == ref[k]) for k in ref}


def test_digests_are_deterministic():
    os.environ.setdefault("SLDG_FUSED", "force")
    from paper_2603_19959_b200 import _capi
    assert _capi.lib().sldg_build_flags() == 0   # the product library never fuzzes
    assert digests() == digests()
