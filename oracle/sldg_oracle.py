"""CPU ORACLE for the SLDG transport step -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference algorithm
(`/root/reference/pkg/src/sldg_vlasov`, pure Python) for the hot path named
in BASELINE.json: the Strang step's hybrid fast/slow v-sweep with weighted
write-back, the x-advection shift, the charge-density reduction and the 1D
Poisson solve, plus the setup they need (basis, mesh, pencils, sweep plan).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it, and only as the checker or as the
timed CPU baseline. The product package `paper_2603_19959_b200` never imports
it; the product path has no CPU fallback.

Parity pinning: every function here is checked against golden vectors
produced by the reference itself (`tests/golden/make_golden.py`, which
imports `/root/reference/pkg/src` in the build container and writes
`tests/golden/*.npz`).  See tests/test_oracle_golden.py.

Each function cites the reference file:line it restates.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

PERIODIC = "periodic"
ABSORBING = "absorbing"
ONE_MINUS_ULP = float(np.nextafter(1.0, 0.0))


# --------------------------------------------------------------------------
# Reference element  (basis.py:19-148)
# --------------------------------------------------------------------------
def legendre_with_derivs(p, x):
    """P_p, P_p', P_p'' by the three-term recurrence (basis.py:19-40)."""
    x = np.asarray(x, dtype=float)
    p0, d0, s0 = np.zeros_like(x), np.zeros_like(x), np.zeros_like(x)
    p1, d1, s1 = np.ones_like(x), np.zeros_like(x), np.zeros_like(x)
    for k in range(1, p + 1):
        a = (2.0 * k - 1.0) / k
        b = (k - 1.0) / k
        pn = a * x * p1 - b * p0
        dn = a * (p1 + x * d1) - b * d0
        sn = a * (2.0 * d1 + x * s1) - b * s0
        p0, d0, s0, p1, d1, s1 = p1, d1, s1, pn, dn, sn
    return p1, d1, s1


def gll(p):
    """GLL nodes/weights via Newton on (1-x^2)P_p' (basis.py:43-74)."""
    if p == 1:
        return np.array([-1.0, 1.0]), np.array([1.0, 1.0])
    x = np.cos(np.pi * np.arange(1, p) / p)
    for _ in range(100):
        _, d1, d2 = legendre_with_derivs(p, x)
        step = -((1.0 - x * x) * d1) / (-2.0 * x * d1 + (1.0 - x * x) * d2)
        x = x + step
        if np.max(np.abs(step)) < 1e-15:
            break
    nodes = np.concatenate(([-1.0], np.sort(x), [1.0]))
    nodes = 0.5 * (nodes - nodes[::-1])
    nodes[0], nodes[-1] = -1.0, 1.0
    pv, _, _ = legendre_with_derivs(p, nodes)
    w = 2.0 / (p * (p + 1) * pv * pv)
    return nodes, 0.5 * (w + w[::-1])


class Basis:
    """Nodal GLL basis with 2p+2 Gauss rule and exact mass (basis.py:84-148)."""

    def __init__(self, p):
        self.p = int(p)
        self.o = self.p + 1
        self.nodes, self.weights = gll(self.p)
        self.gq, self.gw = np.polynomial.legendre.leggauss(2 * self.p + 2)
        o = self.o
        self.others = np.array([[m for m in range(o) if m != j] for j in range(o)])
        self.inv_denoms = 1.0 / np.array(
            [np.prod(self.nodes[j] - self.nodes[self.others[j]]) for j in range(o)])
        v = self.lagrange(self.gq)
        mass = v.T @ (self.gw[:, None] * v)
        self.mass = 0.5 * (mass + mass.T)
        self.mass_inv = np.linalg.inv(self.mass)
        d = np.zeros((o, o))
        for i in range(o):
            for j in range(o):
                if i != j:
                    d[i, j] = (self.inv_denoms[j] / self.inv_denoms[i]) / (
                        self.nodes[i] - self.nodes[j])
        np.fill_diagonal(d, -d.sum(axis=1))
        self.diff = d

    def lagrange(self, x):
        """All Lagrange polynomials at x, shape x.shape + (o,) (basis.py:119-128)."""
        x = np.asarray(x, dtype=float)
        dx = x[..., None] - self.nodes
        return dx[..., self.others].prod(axis=-1) * self.inv_denoms


# --------------------------------------------------------------------------
# 1D SLDG  (sldg1d.py:39-136)
# --------------------------------------------------------------------------
def split_shift(speed, dt, width):
    """(n, alpha) with speed*dt/width = n + alpha, 1-ulp fold (sldg1d.py:39-55)."""
    r = speed * dt / width
    n = math.floor(r)
    a = r - n
    if a >= ONE_MINUS_ULP:
        return n + 1, 0.0
    return n, a


def _interval_integral(b: Basis, lo, hi, shift):
    """int_lo^hi l_i(xi) l_j(xi+shift) by the 2p+2 Gauss rule (sldg1d.py:72-79)."""
    h = 0.5 * (hi - lo)
    xs = lo + h * (b.gq + 1.0)
    return b.lagrange(xs).T @ ((h * b.gw)[:, None] * b.lagrange(xs + shift))


def overlap_mats(b: Basis, alpha):
    """(A, B) = same/neighbour projection blocks incl. M^-1 (sldg1d.py:82-100)."""
    if alpha == 0.0:
        return np.eye(b.o), np.zeros((b.o, b.o))
    c = 2.0 * alpha - 1.0
    A = b.mass_inv @ _interval_integral(b, c, 1.0, -2.0 * alpha)
    B = b.mass_inv @ _interval_integral(b, -1.0, c, 2.0 * (1.0 - alpha))
    return A, B


def _shift_cells(u, k, bc):
    """out[..., i, :] = u[..., i-k, :], wrap or zero-fill (sldg1d.py:103-121)."""
    if bc == PERIODIC:
        return np.roll(u, k, axis=-2)
    if k == 0:
        return u
    n = u.shape[-2]
    out = np.zeros_like(u)
    if 0 < k < n:
        out[..., k:, :] = u[..., :n - k, :]
    elif 0 < -k < n:
        out[..., :n + k, :] = u[..., -k:, :]
    return out


def uniform_update(u, n, A, B, bc):
    """out_i = A u_{i-n} + B u_{i-n-1} on a uniform pencil (sldg1d.py:124-136)."""
    u = np.asarray(u, dtype=float)
    return _shift_cells(u, n, bc) @ A.T + _shift_cells(u, n + 1, bc) @ B.T


def brute_projection(u, disp, width, b: Basis, bc):
    """50-point-Gauss translate-and-project oracle (sldg1d.py:139-175)."""
    u = np.asarray(u, dtype=float)
    n, o = u.shape
    gq, gw = np.polynomial.legendre.leggauss(50)
    length = n * width
    imgs = range(-(int(abs(disp) / length) + 2), int(abs(disp) / length) + 3) \
        if bc == PERIODIC else (0,)
    out = np.zeros_like(u)
    for i in range(n):
        flo = i * width - disp
        acc = np.zeros(o)
        for c in range(n):
            for k in imgs:
                slo = c * width + k * length
                a, z = max(flo, slo), min(flo + width, slo + width)
                if z <= a:
                    continue
                xs = 0.5 * (a + z) + 0.5 * (z - a) * gq
                ws = 0.5 * (z - a) * gw
                sv = b.lagrange(2.0 * (xs - slo) / width - 1.0) @ u[c]
                dv = b.lagrange(2.0 * (xs + disp - i * width) / width - 1.0)
                acc += (2.0 / width) * ((ws * sv) @ dv)
        out[i] = b.mass_inv @ acc
    return out


# --------------------------------------------------------------------------
# AMR velocity mesh  (vmesh.py:65-168)
# --------------------------------------------------------------------------
@dataclass
class Mesh:
    dim: int
    radius: float
    n_base: int
    levels: np.ndarray
    lo: np.ndarray
    width: np.ndarray

    @property
    def n_cells(self):
        return len(self.levels)

    @property
    def base_width(self):
        return 2.0 * self.radius / self.n_base


def _split_cells(levels, lo, width, mark):
    """Marked cells -> 2^dim children appended after survivors (vmesh.py:72-94)."""
    dim = lo.shape[1]
    corners = np.array(np.meshgrid(*([[0.0, 0.5]] * dim), indexing="ij")).reshape(dim, -1).T
    plo, pw = lo[mark], width[mark]
    clo = (plo[:, None, :] + corners[None] * pw[:, None, :]).reshape(-1, dim)
    cw = np.repeat(0.5 * pw, 2 ** dim, axis=0)
    cl = np.repeat(levels[mark] + 1, 2 ** dim)
    keep = ~mark
    return (np.concatenate([levels[keep], cl]), np.concatenate([lo[keep], clo]),
            np.concatenate([width[keep], cw]))


def _unbalanced(levels, lo, width, tol):
    """Cells face-touching a cell >= 2 levels finer (vmesh.py:97-116), dense O(n^2)."""
    hi = lo + width
    dim = lo.shape[1]
    bad = np.zeros(len(levels), dtype=bool)
    finer2 = (levels[None, :] - levels[:, None]) >= 2
    for d in range(dim):
        touching = (np.abs(hi[:, None, d] - lo[None, :, d]) < tol) | (
            np.abs(hi[None, :, d] - lo[:, None, d]) < tol)
        for t in range(dim):
            if t != d:
                touching &= (np.minimum(hi[:, None, t], hi[None, :, t])
                             - np.maximum(lo[:, None, t], lo[None, :, t])) > tol
        bad |= (touching & finer2).any(axis=1)
    return bad


def make_mesh(dim, n_base, max_level, radius):
    """Uniform grid + origin-nearest refinement + 2:1 balance + lexsort (vmesh.py:119-168)."""
    h0 = 2.0 * radius / n_base
    tol = 1e-9 * h0
    ijk = np.array(np.meshgrid(*([np.arange(n_base)] * dim), indexing="ij")).reshape(dim, -1).T
    lo = -radius + ijk * h0
    width = np.full_like(lo, h0)
    levels = np.zeros(len(lo), dtype=np.int64)
    for _ in range(max_level):
        ctr = lo + 0.5 * width
        dist = np.sqrt((ctr * ctr).sum(axis=1))
        mark = dist <= dist.min() + tol
        if not mark.any():
            break
        levels, lo, width = _split_cells(levels, lo, width, mark)
        for _ in range(max_level + 2):
            bad = _unbalanced(levels, lo, width, tol)
            if not bad.any():
                break
            levels, lo, width = _split_cells(levels, lo, width, bad)
        else:
            raise RuntimeError("2:1 balance not restored")
    order = np.lexsort(tuple(lo[:, d] for d in reversed(range(dim))))
    return Mesh(dim, float(radius), int(n_base), levels[order], lo[order], width[order])


# --------------------------------------------------------------------------
# Pencils  (pencil.py:54-168)
# --------------------------------------------------------------------------
@dataclass
class Pencils:
    direction: int
    offsets: np.ndarray
    cell_ids: np.ndarray
    lowers: np.ndarray
    widths: np.ndarray
    levels: np.ndarray
    weights: np.ndarray
    conforming: np.ndarray = None

    @property
    def n_pencils(self):
        return len(self.offsets) - 1

    def span(self, q):
        return slice(int(self.offsets[q]), int(self.offsets[q + 1]))


def _dedup_sorted(v, tol):
    v = np.sort(v)
    return v[np.concatenate(([True], np.diff(v) > tol))]


def make_pencils(mesh: Mesh, direction, weights="count"):
    """CSR pencils along `direction`, weights 1/n_c (pencil.py:60-138).

    weights="area" (not in the reference): each entry weighs the fraction
    of the cell's transverse area its pencil covers, normalised per cell; 1.0 for cells in
    a single pencil."""
    tol = 1e-9 * mesh.base_width
    tdims = [t for t in range(mesh.dim) if t != direction]
    areas = []
    if tdims:
        ivs = []
        for t in tdims:
            e = _dedup_sorted(np.concatenate([mesh.lo[:, t], mesh.lo[:, t] + mesh.width[:, t]]), tol)
            ivs.append(np.stack([e[:-1], e[1:]], axis=1))
        members = []
        for b2 in ivs[1]:          # first transverse dim fastest (pencil.py:85-86)
            for b1 in ivs[0]:
                t0, t1 = tdims
                hit = ((mesh.lo[:, t0] <= b1[0] + tol)
                       & (mesh.lo[:, t0] + mesh.width[:, t0] >= b1[1] - tol)
                       & (mesh.lo[:, t1] <= b2[0] + tol)
                       & (mesh.lo[:, t1] + mesh.width[:, t1] >= b2[1] - tol))
                members.append(np.nonzero(hit)[0])
                areas.append((b1[1] - b1[0]) * (b2[1] - b2[0]))
    else:
        members = [np.arange(mesh.n_cells)]
        areas = [1.0]
    order = [np.argsort(mesh.lo[m, direction], kind="stable") for m in members]
    ids = [m[o] for m, o in zip(members, order)]
    offsets = np.concatenate(([0], np.cumsum([len(m) for m in ids]))).astype(np.int64)
    cid = np.concatenate(ids)
    counts = np.bincount(cid, minlength=mesh.n_cells)
    if weights == "area":
        pa = np.repeat(np.array(areas), [len(m) for m in ids])
        ca = (np.prod(mesh.width[cid][:, tdims], axis=1) if tdims else np.ones(len(cid)))
        frac = pa / ca
        tot = np.bincount(cid, weights=frac, minlength=mesh.n_cells)
        w = np.where(counts[cid] == 1, 1.0, frac / tot[cid])
    else:
        w = 1.0 / counts[cid]
    return Pencils(direction, offsets, cid, mesh.lo[cid, direction].copy(),
                   mesh.width[cid, direction].copy(), mesh.levels[cid].copy(), w)


def mark_conforming(ps: Pencils, bc):
    """+-2 same-level neighbourhood flags, single-cell pencils slow (pencil.py:141-168)."""
    conf = np.zeros(len(ps.cell_ids), dtype=bool)
    for q in range(ps.n_pencils):
        sl = ps.span(q)
        lev = ps.levels[sl]
        n = len(lev)
        if n == 1:
            continue
        ok = np.ones(n, dtype=bool)
        for off in (-2, -1, 1, 2):
            j = np.arange(n) + off
            if bc == PERIODIC:
                ok &= lev[j % n] == lev
            else:
                inside = (j >= 0) & (j < n)
                ok[inside] &= lev[j[inside]] == lev[inside]
        conf[sl] = ok
    ps.conforming = conf
    return ps


def line_lists(p, dim):
    """Per-direction cell-local line index lists (tensor.py:56-106)."""
    o = p + 1
    if dim == 1:
        return (np.arange(o)[None, :],)
    out = []
    for d in range(3):
        rows = np.empty((o * o, o), dtype=np.int64)
        td = [t for t in range(3) if t != d]
        for t2 in range(o):
            for t1 in range(o):
                idx = [None] * 3
                idx[d] = np.arange(o)
                idx[td[0]] = t1
                idx[td[1]] = t2
                rows[t1 + o * t2] = idx[0] + o * idx[1] + o * o * idx[2]
        out.append(rows)
    return tuple(out)


# --------------------------------------------------------------------------
# Sweep plan  (vsweep.py:275-387)
# --------------------------------------------------------------------------
@dataclass
class Group:
    lowers: np.ndarray
    widths: np.ndarray
    levels: np.ndarray
    conforming: np.ndarray
    gather: np.ndarray          # (n_lines, n_cells*o) int64
    weights: np.ndarray         # (n_lines, n_cells*o)
    pencils: list = field(default_factory=list)

    @property
    def n_lines(self):
        return self.gather.shape[0]

    @property
    def n_cells(self):
        return len(self.lowers)


@dataclass
class Plan:
    basis: Basis
    radius: float
    base_width: float
    n_levels: int
    n_dofs: int
    groups: list


def make_plan(mesh: Mesh, ps: Pencils, p):
    """Group congruent pencils; DOF gather = cell*o^dim + line (vsweep.py:307-387)."""
    b = Basis(p)
    o = b.o
    n_local = o ** mesh.dim
    lines = line_lists(p, mesh.dim)[ps.direction]
    keyed = {}
    for q in range(ps.n_pencils):
        sl = ps.span(q)
        k = (ps.levels[sl].tobytes(), ps.lowers[sl].tobytes(),
             ps.widths[sl].tobytes(), ps.conforming[sl].tobytes())
        keyed.setdefault(k, []).append(q)
    groups = []
    for qs in keyed.values():       # dict preserves first-seen order
        sl0 = ps.span(qs[0])
        g_rows, w_rows = [], []
        for q in qs:
            sl = ps.span(q)
            base = ps.cell_ids[sl] * n_local
            wq = np.repeat(ps.weights[sl], o)
            for ln in lines:
                g_rows.append((base[:, None] + ln[None, :]).ravel())
                w_rows.append(wq)
        groups.append(Group(ps.lowers[sl0].copy(), ps.widths[sl0].copy(),
                            ps.levels[sl0].copy(), ps.conforming[sl0].copy(),
                            np.asarray(g_rows, dtype=np.int64), np.asarray(w_rows), list(qs)))
    return Plan(b, mesh.radius, mesh.base_width, int(mesh.levels.max()) + 1,
                mesh.n_cells * n_local, groups)


# --------------------------------------------------------------------------
# Hybrid sweep  (vsweep.py:47-246, 390-441)
# --------------------------------------------------------------------------
def level_shifts(b: Basis, speed, dt, base_width, n_levels):
    """Per-level (n, alpha, A, B) (vsweep.py:47-61)."""
    out = []
    for lev in range(n_levels):
        n, a = split_shift(speed, dt, base_width / 2 ** lev)
        A, B = overlap_mats(b, a)
        out.append((n, a, A, B))
    return out


def general_blocks(b: Basis, vl, vr, dlo, dw, slo, sw, disp):
    """Raw cross-size overlap blocks, (2/h_dest) scaled (vsweep.py:77-95)."""
    h = 0.5 * (vr - vl)
    xs = vl[:, None] + h[:, None] * (b.gq[None, :] + 1.0)
    ws = h[:, None] * b.gw[None, :]
    dv = b.lagrange(2.0 * (xs + disp[:, None] - dlo[:, None]) / dw[:, None] - 1.0)
    sv = b.lagrange(2.0 * (xs - slo[:, None]) / sw[:, None] - 1.0)
    raw = np.einsum("nq,nqi,nqj->nij", ws, dv, sv)
    return raw * (2.0 / dw)[:, None, None]


def general_overlap(b: Basis, dlo, dw, slo, sw, disp):
    """M^-1 * general block for one pair, plus [vl, vr] (vsweep.py:98-122)."""
    flo = dlo - disp
    vl, vr = max(flo, slo), min(flo + dw, slo + sw)
    if vr <= vl:
        return np.zeros((b.o, b.o)), vl, vl
    raw = general_blocks(b, np.array([vl]), np.array([vr]), np.array([dlo]),
                         np.array([dw]), np.array([slo]), np.array([sw]), np.array([disp]))[0]
    return b.mass_inv @ raw, vl, vr


def same_level_ok(s, n_shift, levels, bc):
    """Cells between dest and its sources share dest's level (vsweep.py:125-146)."""
    n = len(levels)
    a, z = min(s, s - n_shift - 1), max(s, s - n_shift)
    if bc == PERIODIC:
        if z - a + 1 >= n:
            return bool((levels == levels[s]).all())
        return bool((levels[np.arange(a, z + 1) % n] == levels[s]).all())
    return bool((levels[max(a, 0):min(z, n - 1) + 1] == levels[s]).all())


def foot_pieces(flo, width, disp, bc, radius):
    """Foot interval clipped (absorbing) or wrapped/split (periodic) (vsweep.py:149-170)."""
    fhi = flo + width
    if bc == ABSORBING:
        a, z = max(flo, -radius), min(fhi, radius)
        return [(a, z, disp)] if z > a else []
    period = 2.0 * radius
    k = np.floor((flo + radius) / period)
    a, z = flo - k * period, fhi - k * period
    if z <= radius:
        return [(a, z, disp + k * period)]
    return [(a, radius, disp + k * period), (-radius, z - period, disp + (k + 1.0) * period)]


def pencil_update(vals, lowers, widths, levels, conforming, speed, dt, lsh, bc, radius,
                  b: Basis, force_slow=False):
    """Hybrid update of one pencil batch (..., n_cells, o) (vsweep.py:173-246)."""
    vals = np.asarray(vals, dtype=float)
    n = len(lowers)
    disp = speed * dt
    if not force_slow and conforming.all() and (levels == levels[0]).all():
        ns, _, A, B = lsh[int(levels[0])]
        return uniform_update(vals, ns, A, B, bc)
    out = np.zeros(vals.shape)
    uppers = lowers + widths
    slow = []
    for s in range(n):
        ns, _, A, B = lsh[int(levels[s])]
        if not force_slow and conforming[s] and same_level_ok(s, ns, levels, bc):
            acc = 0.0
            for q, M in ((s - ns, A), (s - ns - 1, B)):
                if bc == PERIODIC:
                    acc = acc + vals[..., q % n, :] @ M.T
                elif 0 <= q < n:
                    acc = acc + vals[..., q, :] @ M.T
            out[..., s, :] = acc
        else:
            slow.append(s)
    recs = []
    for s in slow:
        for a, z, de in foot_pieces(lowers[s] - disp, widths[s], disp, bc, radius):
            c0 = int(np.searchsorted(uppers, a, side="right"))
            c1 = int(np.searchsorted(lowers, z, side="left")) - 1
            for c in range(max(c0, 0), min(c1, n - 1) + 1):
                vl, vr = max(a, lowers[c]), min(z, uppers[c])
                if vr - vl > 1e-14 * widths[s]:
                    recs.append((s, c, vl, vr, de))
    if recs:
        r = np.array(recs)
        si, ci = r[:, 0].astype(int), r[:, 1].astype(int)
        raw = general_blocks(b, r[:, 2], r[:, 3], lowers[si], widths[si],
                             lowers[ci], widths[ci], r[:, 4])
        mats = np.matmul(b.mass_inv, raw)
        for m in range(len(recs)):
            out[..., si[m], :] += vals[..., ci[m], :] @ mats[m].T
    return out


def writeback(f_in, gather, weights, values):
    """f_in + sum w (value - f_in), copy when w == 1 (vsweep.py:249-272)."""
    f_in = np.asarray(f_in, dtype=float)
    cnt = np.bincount(gather, minlength=f_in.size)
    if (cnt == 0).any():
        raise RuntimeError(f"element {int(np.nonzero(cnt == 0)[0][0])} uncovered")
    out = f_in.copy()
    cp = weights == 1.0
    out[gather[cp]] = values[cp]
    if (~cp).any():
        out += np.bincount(gather[~cp], weights=weights[~cp] * (values[~cp] - f_in[gather[~cp]]),
                           minlength=f_in.size)
    return out


def sweep_column(fv, speed, dt, plan: Plan, bc, force_slow=False):
    """One x column through every group + weighted write-back (vsweep.py:390-410)."""
    b = plan.basis
    o = b.o
    lsh = level_shifts(b, speed, dt, plan.base_width, plan.n_levels)
    out = fv.copy()
    for g in plan.groups:
        res = pencil_update(fv[g.gather].reshape(g.n_lines, g.n_cells, o), g.lowers,
                            g.widths, g.levels, g.conforming, speed, dt, lsh, bc,
                            plan.radius, b, force_slow).reshape(-1)
        flat_t = g.gather.ravel()
        flat_w = g.weights.ravel()
        cp = flat_w == 1.0
        if cp.all():
            out[flat_t] = res
            continue
        out[flat_t[cp]] = res[cp]
        out += np.bincount(flat_t[~cp], weights=flat_w[~cp] * (res[~cp] - fv[flat_t[~cp]]),
                           minlength=out.size)
    return out


def advect_v(f, speeds, dt, plan: Plan, bc=ABSORBING, force_slow=False, workers=1):
    """Column loop; exact-zero speeds skipped; optional thread pool over columns like the
    reference's `workers` (vsweep.py:413-441). In place."""
    speeds = np.asarray(speeds, dtype=float)
    assert f.shape == (plan.n_dofs, speeds.size)

    def one(ix):
        f[:, ix] = sweep_column(np.ascontiguousarray(f[:, ix]), speeds[ix], dt, plan, bc,
                                force_slow)

    cols = np.nonzero(speeds != 0.0)[0]
    if workers <= 1:
        for ix in cols:
            one(ix)
    else:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=workers) as pool:
            list(pool.map(one, cols))
    return f


# --------------------------------------------------------------------------
# x side  (xfield.py:22-195)
# --------------------------------------------------------------------------
class XGrid:
    """Periodic DG x grid (xfield.py:22-45)."""

    def __init__(self, n_cells, p, length):
        self.n_cells = int(n_cells)
        self.length = float(length)
        self.basis = Basis(p)
        self.p = p
        self.h = self.length / self.n_cells
        lows = np.arange(self.n_cells) * self.h
        self.dof_coords = (lows[:, None] + 0.5 * (self.basis.nodes + 1.0) * self.h).ravel()
        self.dof_weights = np.tile(0.5 * self.h * self.basis.weights, self.n_cells)

    @property
    def n_dofs(self):
        return self.n_cells * (self.p + 1)


def x_plan(xg: XGrid, speeds, dt):
    """Rows grouped by unique speed with (n, alpha, A, B) (xfield.py:63-79)."""
    speeds = np.asarray(speeds, dtype=float)
    uniq, inv = np.unique(speeds, return_inverse=True)
    groups = []
    for u in range(len(uniq)):
        n, a = split_shift(uniq[u], dt, xg.h)
        A, B = overlap_mats(xg.basis, a)
        groups.append((np.nonzero(inv == u)[0], n, a, A, B))
    return groups


def advect_x(f, groups, n_cells, workers=1):
    """Periodic x shift per row group; identity rows untouched; optional thread pool over
    speed groups like the reference (xfield.py:82-104)."""
    def one(grp):
        rows, n, a, A, B = grp
        if n == 0 and a == 0.0:
            return
        blk = f[rows].reshape(len(rows), n_cells, -1)
        f[rows] = uniform_update(blk, n, A, B, PERIODIC).reshape(len(rows), -1)

    if workers <= 1:
        for grp in groups:
            one(grp)
    else:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=workers) as pool:
            list(pool.map(one, groups))
    return f


def rho(f, vweights):
    """rho = w_v . f (xfield.py:107-109)."""
    return np.asarray(vweights) @ f


class Poisson:
    """CG-FE periodic Poisson with zero-mean augmented LU (xfield.py:112-179)."""

    def __init__(self, xg: XGrid):
        from scipy.linalg import lu_factor
        self.xg = xg
        b = xg.basis
        p = xg.p
        nn = xg.n_cells * p
        self.nn = nn
        self.conn = (np.arange(xg.n_cells)[:, None] * p + np.arange(p + 1)[None, :]) % nn
        kloc = (2.0 / xg.h) * b.diff.T @ (b.weights[:, None] * b.diff)
        K = np.zeros((nn, nn))
        for c in range(xg.n_cells):
            K[np.ix_(self.conn[c], self.conn[c])] += kloc
        lump = np.zeros(nn)
        np.add.at(lump, self.conn.ravel(), np.tile(0.5 * xg.h * b.weights, xg.n_cells))
        aug = np.zeros((nn + 1, nn + 1))
        aug[:nn, :nn] = K
        aug[:nn, nn] = lump
        aug[nn, :nn] = lump
        self.K, self.lump, self.aug = K, lump, aug
        self.lu = lu_factor(aug)

    def rhs(self, r):
        r = np.asarray(r, dtype=float)
        rbar = (self.xg.dof_weights @ r) / self.xg.length
        bvec = np.zeros(self.nn)
        np.add.at(bvec, self.conn.ravel(), self.xg.dof_weights * (r - rbar))
        return bvec

    def solve(self, r):
        from scipy.linalg import lu_solve
        bb = np.zeros(self.nn + 1)
        bb[:self.nn] = self.rhs(r)
        return lu_solve(self.lu, bb, check_finite=False)[:self.nn]

    def efield(self, phi):
        return (-(2.0 / self.xg.h) * phi[self.conn] @ self.xg.basis.diff.T).ravel()


def field_energy(e, xg: XGrid):
    """0.5 * GLL quadrature of E^2 (xfield.py:192-195)."""
    e = np.asarray(e, dtype=float)
    return 0.5 * float(xg.dof_weights @ (e * e))


# --------------------------------------------------------------------------
# Driver pieces  (driver.py:112-272)
# --------------------------------------------------------------------------
def forward_map(p, dim):
    o = p + 1
    ids = np.arange(o ** dim)
    if dim == 1:
        return ids[:, None]
    return np.stack([ids % o, (ids // o) % o, ids // (o * o)], axis=1)


def vcoords(mesh: Mesh, b: Basis):
    """Velocity DOF coordinates (driver.py:112-116)."""
    ref = 0.5 * (b.nodes[forward_map(b.p, mesh.dim)] + 1.0)
    return (mesh.lo[:, None, :] + ref[None] * mesh.width[:, None, :]).reshape(-1, mesh.dim)


def vweights(mesh: Mesh, b: Basis):
    """Tensor GLL weights x Jacobian (driver.py:119-123)."""
    wp = b.weights[forward_map(b.p, mesh.dim)].prod(axis=1)
    return ((0.5 * mesh.width).prod(axis=1)[:, None] * wp[None, :]).ravel()


def landau_initial(vc, xc, dim, k=0.5, eps=0.01):
    """Perturbed Maxwellian at all DOF pairs (driver.py:126-136)."""
    g = (2.0 * np.pi) ** (-dim / 2.0) * np.exp(-0.5 * (np.asarray(vc) ** 2).sum(axis=-1))
    return g[:, None] * (1.0 + eps * np.cos(k * np.asarray(xc)))[None, :]


def moments(f, vw, vc, xw):
    """(m0, m1, m2) (driver.py:139-146)."""
    col = f @ xw
    return (float(vw @ col), float((vw * vc[:, 0]) @ col),
            float((vw * (vc ** 2).sum(axis=1)) @ col))


class Sim:
    """Strang-split Landau simulation mirroring driver.Simulation (driver.py:194-272)."""

    def __init__(self, dim=3, n_base=4, levels=0, radius=6.0, degree=3, n_x=64, degree_x=2,
                 wave_number=0.5, perturbation=0.01, dt=0.1, bc=ABSORBING, force_slow=False,
                 mesh=None, pencil_weights="count", workers=1):
        self.dt, self.bc, self.force_slow, self.workers = dt, bc, force_slow, workers
        self.basis = Basis(degree)
        self.mesh = mesh if mesh is not None else make_mesh(dim, n_base, levels, radius)
        ps = mark_conforming(make_pencils(self.mesh, 0, pencil_weights), bc)
        self.plan = make_plan(self.mesh, ps, degree)
        self.xg = XGrid(n_x, degree_x, 2.0 * np.pi / wave_number)
        self.vc = vcoords(self.mesh, self.basis)
        self.vw = vweights(self.mesh, self.basis)
        self.xplan = x_plan(self.xg, self.vc[:, 0], 0.5 * dt)
        self.poisson = Poisson(self.xg)
        self.f = landau_initial(self.vc, self.xg.dof_coords, self.mesh.dim, wave_number,
                                perturbation)
        self.t = 0.0

    def field_solve(self):
        return self.poisson.efield(self.poisson.solve(rho(self.f, self.vw)))

    def diagnostics(self, e):
        m0, m1, m2 = moments(self.f, self.vw, self.vc, self.xg.dof_weights)
        ee = field_energy(e, self.xg)
        return dict(t=self.t, e_max=float(np.max(np.abs(e))), m0=m0, m1=m1, m2=m2,
                    e_field=ee, e_total=0.5 * m2 + ee)

    def step(self):
        w = self.workers
        advect_x(self.f, self.xplan, self.xg.n_cells, workers=w)
        e = self.field_solve()
        advect_v(self.f, e, self.dt, self.plan, self.bc, self.force_slow, workers=w)
        advect_x(self.f, self.xplan, self.xg.n_cells, workers=w)
        self.t += self.dt
        return self.diagnostics(e)


def peak_run_fit(times, values):
    """Envelope-peak damping fit (driver.py:149-191). Returns (rate, n_peaks)."""
    times = np.asarray(times, dtype=float)
    values = np.asarray(values, dtype=float)
    n = len(values)
    if n < 3:
        return None, 0
    peaks, i = [], 1
    while i < n - 1:
        if values[i] > values[i - 1]:
            j = i
            while j < n - 1 and values[j + 1] == values[i]:
                j += 1
            if j < n - 1 and values[j + 1] < values[i]:
                peaks.append(i)
            i = j + 1
        else:
            i += 1
    run = peaks[:1]
    for k in peaks[1:]:
        if values[k] < values[run[-1]]:
            run.append(k)
        else:
            break
    if len(run) < 2:
        return None, len(run)
    slope, _ = np.polyfit(times[run], np.log(values[run]), 1)
    return float(slope), len(run)
