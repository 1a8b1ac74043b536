"""The ctypes stub of INTEGRATION.md (section 2) executed as written: a reference-side
GPU backend for advect_velocity through the C ABI only (no torch), against the
package's own advect_velocity (needs a B200)."""
import ctypes
import os
import re

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_19959_b200 as sv  # noqa: E402

DOC = os.path.join(os.path.dirname(os.path.dirname(__file__)), "INTEGRATION.md")


def _stub_namespace():
    text = open(DOC).read()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    code = next(b for b in blocks if "advect_velocity_gpu" in b)
    try:
        ctypes.CDLL("libcudart.so.12")
    except OSError:
        pytest.skip("libcudart.so.12 not on the loader path")
    ns = {}
    exec(compile(code, "INTEGRATION.md:stub", "exec"), ns)
    return ns


@pytest.mark.parametrize("nb,lv,p,bc", [(6, 0, 2, "absorbing"), (4, 1, 2, "periodic")])
def test_integration_stub_matches_package(nb, lv, p, bc):
    ns = _stub_namespace()
    m = sv.build_mesh(3, nb, lv, 6.0)
    b = sv.DGBasis(p)
    ps = sv.classify_conforming(sv.extract_pencils(m, 0), m, bc)
    plan = sv.build_sweep_plan(m, ps, sv.build_permutation(b, 3), b)
    h = ns["make_device_plan"](plan, plan._arrays, dim=3)
    rng = np.random.default_rng(nb + lv)
    f = rng.standard_normal((plan.n_dofs, 24))
    speeds = rng.uniform(-3, 3, 24)
    speeds[5] = 0.0
    got = ns["advect_velocity_gpu"](f.copy(), speeds, 0.1, h, bc)
    ref = sv.advect_velocity(f.copy(), speeds, 0.1, plan, bc)
    assert np.array_equal(got, ref)
    ns["_lib"].sldg_vplan_destroy(h)
