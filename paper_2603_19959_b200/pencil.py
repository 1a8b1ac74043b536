"""Per-direction CSR pencils (host setup, uploaded once per mesh).

Same arrays as `sldg_vlasov.pencil.extract_pencils` / `classify_conforming`
(pencil.py:60-168): pencils in lexicographic transverse order (first
transverse dimension fastest), entries sorted along the sweep axis, weights
1/n_c, +-2 same-level conforming flags.  Membership is found by interval
search over the unique transverse edges (O(n log n)) instead of the
reference's per-pencil scan over all cells.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .sldg1d import PERIODIC, check_bc
from .vmesh import VelocityMesh


class PencilError(ValueError):
    pass


@dataclass
class PencilSet:
    """CSR pencil arrays for one sweep direction (pencil.py:25-50)."""

    direction: int
    n_pencils: int
    offsets: np.ndarray
    cell_ids: np.ndarray
    lowers: np.ndarray
    widths: np.ndarray
    levels: np.ndarray
    weights: np.ndarray
    conforming: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.conforming is None:
            self.conforming = np.zeros(len(self.cell_ids), dtype=bool)

    def pencil_slice(self, q: int) -> slice:
        return slice(int(self.offsets[q]), int(self.offsets[q + 1]))


def _edges(vals, tol):
    vals = np.sort(vals)
    return vals[np.concatenate(([True], np.diff(vals) > tol))]


WEIGHT_MODES = ("count", "area")


def extract_pencils(mesh: VelocityMesh, direction: int, weights: str = "count") -> PencilSet:
    """Pencil decomposition along `direction` (pencil.py:60-138).

    weights="count" (default) gives the reference's entry weights 1/n_c, n_c the number of
    pencils cell c lies in (pencil.py:124,137).  weights="area" gives each entry the
    fraction of the cell's transverse area that the pencil covers, normalised per cell:
    with two AMR levels a coarse cell can be cut into transverse intervals of unequal
    width, where 1/n_c is not mass conservative and the area fractions are (SURVEY.md
    §8 N1).  Cells in one pencil have weight 1.0 in both modes.
    """
    if weights not in WEIGHT_MODES:
        raise PencilError(f"weights must be one of {WEIGHT_MODES}, got {weights!r}")
    if not 0 <= direction < mesh.dim:
        raise PencilError(f"direction must be in [0, {mesh.dim}), got {direction}")
    tol = 1e-9 * mesh.base_width
    n = mesh.n_cells
    tdims = [t for t in range(mesh.dim) if t != direction]
    if tdims:
        ranges = []
        n_iv = []
        edges = []
        for t in tdims:
            e = _edges(np.concatenate([mesh.lo[:, t], mesh.lo[:, t] + mesh.width[:, t]]), tol)
            lo_t, hi_t = mesh.lo[:, t], mesh.lo[:, t] + mesh.width[:, t]
            # interval k = [e_k, e_{k+1}] is covered iff lo <= e_k + tol and hi >= e_{k+1} - tol
            k0 = np.searchsorted(e, lo_t - tol, side="left")
            k1 = np.searchsorted(e, hi_t + tol, side="right") - 1   # exclusive interval bound
            ranges.append((k0, k1))
            n_iv.append(len(e) - 1)
            edges.append(e)
        (a0, b0), (a1, b1) = ranges
        c0, c1 = np.maximum(b0 - a0, 0), np.maximum(b1 - a1, 0)
        cnt = c0 * c1
        cell = np.repeat(np.arange(n), cnt)
        local = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        i0 = a0[cell] + local % c0[cell]
        i1 = a1[cell] + local // c0[cell]
        pencil = i1 * n_iv[0] + i0
        n_pencils = n_iv[0] * n_iv[1]
        # transverse area of the pencil / transverse area of the cell
        frac = ((edges[0][i0 + 1] - edges[0][i0]) * (edges[1][i1 + 1] - edges[1][i1])
                / (mesh.width[cell, tdims[0]] * mesh.width[cell, tdims[1]]))
    else:
        cell = np.arange(n)
        pencil = np.zeros(n, dtype=np.int64)
        n_pencils = 1
        frac = np.ones(n)
    order = np.lexsort((cell, mesh.lo[cell, direction], pencil))
    cell, pencil, frac = cell[order], pencil[order], frac[order]
    counts_p = np.bincount(pencil, minlength=n_pencils)
    if (counts_p == 0).any():
        q = int(np.nonzero(counts_p == 0)[0][0])
        raise PencilError(f"pencil {q} in direction {direction} covers no cells")
    offsets = np.concatenate(([0], np.cumsum(counts_p))).astype(np.int64)
    lo = mesh.lo[cell, direction]
    w = mesh.width[cell, direction]
    first, last = offsets[:-1], offsets[1:] - 1
    bad_span = (np.abs(lo[first] + mesh.radius) > tol) | (
        np.abs(lo[last] + w[last] - mesh.radius) > tol)
    if bad_span.any():
        q = int(np.nonzero(bad_span)[0][0])
        raise PencilError(f"pencil {q} in direction {direction} does not span the domain: "
                          f"[{lo[first[q]]}, {lo[last[q]] + w[last[q]]}]")
    if len(cell) > 1:
        gap = np.abs(lo[1:] - (lo[:-1] + w[:-1]))
        same = pencil[1:] == pencil[:-1]
        badg = same & (gap > tol)
        if badg.any():
            k = int(np.nonzero(badg)[0][0])
            raise PencilError(f"pencil {int(pencil[k])} in direction {direction}: gap or "
                              f"overlap at coordinate {lo[k] + w[k]}")
    counts = np.bincount(cell, minlength=n)
    if (counts == 0).any():
        missing = int(np.nonzero(counts == 0)[0][0])
        raise PencilError(f"cell {missing} appears in no pencil of direction {direction}")
    if weights == "area":
        total = np.bincount(cell, weights=frac, minlength=n)
        wts = np.where(counts[cell] == 1, 1.0, frac / total[cell])
    else:
        wts = 1.0 / counts[cell]
    return PencilSet(direction=direction, n_pencils=int(n_pencils), offsets=offsets,
                     cell_ids=cell.astype(np.int64), lowers=lo.copy(), widths=w.copy(),
                     levels=mesh.levels[cell].copy(), weights=wts)


def classify_conforming(pset: PencilSet, mesh: VelocityMesh, bc: str = "absorbing") -> PencilSet:
    """+-2 same-level flags; single-cell pencils slow (pencil.py:141-168). Vectorised."""
    check_bc(bc)
    off = pset.offsets
    n_e = len(pset.cell_ids)
    q = np.repeat(np.arange(pset.n_pencils), np.diff(off))
    pos = np.arange(n_e) - off[q]
    ln = np.diff(off)[q]
    conf = np.ones(n_e, dtype=bool)
    for d in (-2, -1, 1, 2):
        j = pos + d
        if bc == PERIODIC:
            j = np.mod(j, ln)
            conf &= pset.levels[off[q] + j] == pset.levels
        else:
            inside = (j >= 0) & (j < ln)
            nb = pset.levels[np.where(inside, off[q] + j, np.arange(n_e))]
            conf &= ~inside | (nb == pset.levels)
    conf[ln == 1] = False
    pset.conforming = conf
    return pset


def dump_pencils(pset: PencilSet, path) -> None:
    """Pencil entries as CSV (pencil, cell, lower, width, weight, conforming), %.17e
    floats (pencil.py:171-182)."""
    with open(path, "w", newline="\n") as fh:
        fh.write("pencil,cell,lower,width,weight,conforming\n")
        for q in range(pset.n_pencils):
            sl = pset.pencil_slice(q)
            for k in range(sl.start, sl.stop):
                fh.write(f"{q},{int(pset.cell_ids[k])},{pset.lowers[k]:.17e},"
                         f"{pset.widths[k]:.17e},{pset.weights[k]:.17e},"
                         f"{int(pset.conforming[k])}\n")
