"""CPU-only checks: host plan builders vs the reference's golden arrays, and the C ABI
(library loads, exports every symbol include/sldg_capi.h declares)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2603_19959_b200 as sv
from paper_2603_19959_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MESHES = [(3, 4, 0), (3, 4, 1), (3, 4, 2), (3, 3, 1), (3, 3, 2), (1, 16, 0), (3, 6, 1),
          (3, 5, 2)]


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "sldg_capi.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|int64_t)\s+(sldg_\w+)\s*\(", txt,
                                 flags=re.M)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(_capi.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    # and the Python binding declares every one of them
    assert set(syms) == set(_capi.EXPORTED)


def test_library_reports_errors_without_gpu():
    lib = _capi.lib()
    assert lib.sldg_version() >= 10000
    assert lib.sldg_advect_v(None, None, None, 0, 1, None, 0.1, 1, 0, None, None) == \
        _capi.SLDG_ERR_ARG
    assert b"null plan" in lib.sldg_last_error()


@pytest.mark.parametrize("dim,nb,lv", MESHES)
def test_host_builders_bit_identical(golden, dim, nb, lv):
    g = golden("meshes_plans.npz")
    tag = f"d{dim}_b{nb}_l{lv}"
    m = sv.build_mesh(dim, nb, lv, 6.0)
    np.testing.assert_array_equal(m.levels, g[f"{tag}_levels"])
    np.testing.assert_array_equal(m.lo, g[f"{tag}_lo"])
    np.testing.assert_array_equal(m.width, g[f"{tag}_width"])
    for bc in ("absorbing", "periodic"):
        for d in range(dim):
            k = f"{tag}_{bc}_dir{d}"
            ps = sv.classify_conforming(sv.extract_pencils(m, d), m, bc)
            for name in ("offsets", "cell_ids", "weights", "conforming"):
                np.testing.assert_array_equal(getattr(ps, name), g[f"{k}_{name}"])
            if d:
                continue
            for p in (1, 2, 3):
                b = sv.DGBasis(p)
                plan = sv.build_sweep_plan(m, ps, sv.build_permutation(b, dim), b)
                kk = f"{k}_p{p}"
                lay = np.array([(gr.n_lines, gr.n_cells) for gr in plan.groups])
                np.testing.assert_array_equal(lay, g[f"{kk}_layout"])
                np.testing.assert_array_equal(
                    np.concatenate([gr.gather.ravel() for gr in plan.groups]), g[f"{kk}_gather"])
                np.testing.assert_array_equal([gr.simple for gr in plan.groups], g[f"{kk}_simple"])


def test_basis_constants_golden(golden):
    g = golden("basis_1d.npz")
    for p in range(1, 6):
        b = sv.DGBasis(p)
        np.testing.assert_allclose(b.nodes, g[f"p{p}_nodes"], atol=1e-15, rtol=0)
        np.testing.assert_allclose(b.weights, g[f"p{p}_weights"], atol=1e-15, rtol=0)
        np.testing.assert_allclose(b.mass_inv, g[f"p{p}_mass_inv"], rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(b.diff, g[f"p{p}_diff"], rtol=1e-13, atol=1e-13)


def test_decompose_shift_golden(golden):
    g = golden("basis_1d.npz")
    for s, d, w, n, fr in zip(g["shift_speed"], g["shift_dt"], g["shift_width"], g["shift_n"],
                              g["shift_frac"]):
        dd = sv.decompose_shift(float(s), float(d), float(w))
        assert dd.n_shift == n and dd.frac == fr


def test_mesh_counts_and_config5_builder():
    counts = {(4, 0): 64, (4, 1): 120, (4, 2): 176, (3, 1): 34, (3, 0): 27, (8, 0): 512}
    for (nb, lv), n in counts.items():
        assert sv.build_mesh(3, nb, lv, 6.0).n_cells == n
    assert sv.ip_count(sv.build_mesh(3, 4, 1, 6.0), 3) == 7680
    # BASELINE config 5 (48^3, two levels): unbuildable by the reference's O(n^2) balance
    m = sv.build_mesh(3, 48, 2, 6.0)
    assert m.n_cells == 110704
    ps = sv.extract_pencils(m, 0)
    assert ps.n_pencils == 2704 and len(ps.cell_ids) == 129896


def test_config_validation():
    with pytest.raises(ValueError):
        sv.SimConfig(dim=2).validate()
    with pytest.raises(ValueError):
        sv.SimConfig(bc="reflecting").validate()
    assert sv.SimConfig().validate().length == pytest.approx(4 * np.pi)


def test_fit_damping_rate():
    t = np.arange(0.0, 20.0 + 1e-12, 0.1)
    fit = sv.fit_damping_rate(t, np.exp(-0.1533 * t) * np.abs(np.cos(1.4156 * t)))
    assert fit.ok and abs(fit.rate + 0.1533) <= 1e-3
    mono = sv.fit_damping_rate(t, np.exp(-0.2 * t))
    assert not mono.ok and mono.rate is None
    y = np.array([0.0, 1.0, 1.0, 0.5, 0.8, 0.2, 0.1, 0.0])
    np.testing.assert_array_equal(sv.fit_damping_rate(np.arange(8.0), y).peak_times[:1], [1.0])


@pytest.mark.parametrize("p", [1, 2, 3])
def test_pack_and_scatter_lines(p):
    """pack_line / scatter_line follow tensor.py:108-122: the line along direction d at
    transverse pair (t1, t2) of the first and second remaining directions."""
    o = p + 1
    perm = sv.build_permutation(sv.DGBasis(p), 3)
    vals = np.arange(o ** 3, dtype=float) * 1.5
    for d in range(3):
        rest = [t for t in range(3) if t != d]
        for t2 in range(o):
            for t1 in range(o):
                trip = [None, None, None]
                trip[d], trip[rest[0]], trip[rest[1]] = np.arange(o), t1, t2
                idx = trip[0] + o * trip[1] + o * o * trip[2]
                assert np.array_equal(sv.pack_line(vals, perm, d, t1, t2), vals[idx])
                out = np.zeros_like(vals)
                sv.scatter_line(vals[idx], out, perm, d, t1, t2)
                assert np.array_equal(out[idx], vals[idx])


def test_dump_mesh_csv(tmp_path):
    m = sv.build_mesh(3, 3, 1, 6.0)
    path = tmp_path / "mesh.csv"
    sv.dump_mesh(m, path)
    lines = path.read_text().splitlines()
    assert lines[0] == "cell,level,lo_0,lo_1,lo_2,h_0,h_1,h_2"
    assert len(lines) == m.n_cells + 1
    for i in (0, m.n_cells // 2, m.n_cells - 1):
        f = lines[i + 1].split(",")
        assert int(f[0]) == i and int(f[1]) == int(m.levels[i])
        assert [float(x) for x in f[2:5]] == list(m.lo[i])
        assert [float(x) for x in f[5:8]] == list(m.width[i])


def test_dump_pencils_and_shifted_source(tmp_path):
    m = sv.build_mesh(3, 3, 1, 6.0)
    ps = sv.classify_conforming(sv.extract_pencils(m, 0), m, "absorbing")
    from paper_2603_19959_b200.pencil import dump_pencils
    from paper_2603_19959_b200.sldg1d import shifted_source
    path = tmp_path / "pencils.csv"
    dump_pencils(ps, path)
    lines = path.read_text().splitlines()
    assert lines[0] == "pencil,cell,lower,width,weight,conforming"
    assert len(lines) == len(ps.cell_ids) + 1
    v = np.arange(2 * 5 * 3, dtype=float).reshape(2, 5, 3)
    for k in (-6, -2, 0, 3, 5):
        per = shifted_source(v, k, "periodic")
        ab = shifted_source(v, k, "absorbing")
        for i in range(5):
            assert np.array_equal(per[:, i], v[:, (i - k) % 5])
            assert np.array_equal(ab[:, i], v[:, i - k] if 0 <= i - k < 5 else 0 * v[:, i])


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not present")
@pytest.mark.parametrize("nb,lv,p", [(4, 2, 3), (3, 1, 2), (4, 1, 2)])
def test_pencil_group_partitions_match_reference(nb, lv, p):
    """_PencilGroup copy_pos / copy_targets / acc_pos / acc_targets / acc_weights equal the
    reference's (vsweep.py:285-291, 366-383), in both bcs."""
    import sys
    if REF_SRC not in sys.path:
        sys.path.append(REF_SRC)
    import sldg_vlasov as ref
    for bc in ("absorbing", "periodic"):
        m = ref.build_mesh(3, nb, lv, 6.0)
        b = ref.DGBasis(p)
        rp = ref.build_sweep_plan(m, ref.classify_conforming(ref.extract_pencils(m, 0), m, bc),
                                  ref.build_permutation(b, 3), b)
        m2 = sv.build_mesh(3, nb, lv, 6.0)
        b2 = sv.DGBasis(p)
        op = sv.build_sweep_plan(m2, sv.classify_conforming(sv.extract_pencils(m2, 0), m2, bc),
                                 sv.build_permutation(b2, 3), b2)
        assert len(rp.groups) == len(op.groups)
        for g, h in zip(rp.groups, op.groups):
            for k in ("copy_pos", "copy_targets", "acc_pos", "acc_targets", "acc_weights"):
                np.testing.assert_array_equal(getattr(g, k), getattr(h, k))
