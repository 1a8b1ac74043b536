"""AMR velocity mesh (host setup).

Same cells, same floating-point coordinates and the same final order as
`sldg_vlasov.vmesh.build_mesh` (vmesh.py:119-168), but the 2:1 face-balance
test runs on an integer occupancy grid at the finest level instead of the
reference's dense n x n comparison (vmesh.py:97-116, O(n^2) memory, which
cannot build BASELINE config 5: 48^3 base, 110,704 cells).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class MeshError(ValueError):
    pass


@dataclass(frozen=True)
class VelocityCell:
    level: int
    lo: np.ndarray
    width: np.ndarray


class VelocityMesh:
    """Flat leaf-cell list (vmesh.py:27-62)."""

    def __init__(self, dim, radius, n_base, max_level, levels, lo, width):
        self.dim = dim
        self.radius = radius
        self.n_base = n_base
        self.max_level = max_level
        self.levels = levels
        self.lo = lo
        self.width = width

    @property
    def n_cells(self) -> int:
        return len(self.levels)

    @property
    def base_width(self) -> float:
        return 2.0 * self.radius / self.n_base

    def cell(self, i: int) -> VelocityCell:
        return VelocityCell(int(self.levels[i]), self.lo[i], self.width[i])

    @property
    def cells(self):
        return [self.cell(i) for i in range(self.n_cells)]


def _children(levels, lo, width, mark):
    """Survivors then 2^dim children per marked cell (vmesh.py:72-94 arithmetic)."""
    dim = lo.shape[1]
    corner = np.stack(np.meshgrid(*([np.array([0.0, 0.5])] * dim), indexing="ij"),
                      axis=-1).reshape(-1, dim)
    plo, pw = lo[mark], width[mark]
    clo = (plo[:, None, :] + corner[None, :, :] * pw[:, None, :]).reshape(-1, dim)
    return (np.concatenate([levels[~mark], np.repeat(levels[mark] + 1, 2 ** dim)]),
            np.concatenate([lo[~mark], clo]),
            np.concatenate([width[~mark], np.repeat(0.5 * pw, 2 ** dim, axis=0)]))


def _violators(levels, lo, width, radius, h_fine, n_fine):
    """Cells face-adjacent to a cell >= 2 levels finer, via an occupancy grid.

    Every cell boundary lies on the finest grid (spacing h_fine); cell boxes
    are rasterised into an int8 level map and each cell inspects the voxel
    layer just outside each of its faces (restricted to its own transverse
    extent -- exactly the reference's touch & positive-overlap test).
    """
    dim = lo.shape[1]
    ilo = np.rint((lo + radius) / h_fine).astype(np.int64)
    iw = np.rint(width / h_fine).astype(np.int64)
    grid = np.full((n_fine,) * dim, -1, dtype=np.int16)
    for size in np.unique(iw[:, 0]):
        sel = np.nonzero(iw[:, 0] == size)[0]
        offs = np.stack(np.meshgrid(*([np.arange(size)] * dim), indexing="ij"),
                        axis=-1).reshape(-1, dim)
        pts = ilo[sel][:, None, :] + offs[None, :, :]
        grid[tuple(pts.reshape(-1, dim).T)] = np.repeat(levels[sel], len(offs))
    bad = np.zeros(len(levels), dtype=bool)
    for size in np.unique(iw[:, 0]):
        sel = np.nonzero(iw[:, 0] == size)[0]
        if size < 4:       # a violator is >= 2 levels coarser than a neighbour: width >= 4 voxels
            continue
        face = np.stack(np.meshgrid(*([np.arange(size)] * (dim - 1)), indexing="ij"),
                        axis=-1).reshape(-1, dim - 1) if dim > 1 else np.zeros((1, 0), np.int64)
        for d in range(dim):
            t = [k for k in range(dim) if k != d]
            for side in (-1, size):
                pos = ilo[sel, d] + side
                ok = (pos >= 0) & (pos < n_fine)
                if not ok.any():
                    continue
                s2 = sel[ok]
                idx = np.empty((len(s2), len(face), dim), dtype=np.int64)
                idx[:, :, d] = (ilo[s2, d] + side)[:, None]
                for j, k in enumerate(t):
                    idx[:, :, k] = ilo[s2, k][:, None] + face[None, :, j]
                nb = grid[tuple(idx.reshape(-1, dim).T)].reshape(len(s2), len(face))
                bad[s2] |= (nb.max(axis=1) - levels[s2]) >= 2
    return bad


def build_mesh(dim: int, n_base: int, max_level: int, radius: float, marker=None) -> VelocityMesh:
    """AMR mesh with origin-nearest refinement and 2:1 balance (vmesh.py:119-168)."""
    if dim not in (1, 3):
        raise MeshError(f"velocity dimension must be 1 or 3, got {dim}")
    if not isinstance(n_base, (int, np.integer)) or n_base < 2:
        raise MeshError(f"base cell count must be an integer >= 2, got {n_base!r}")
    if not isinstance(max_level, (int, np.integer)) or not 0 <= max_level <= 3:
        raise MeshError(f"refinement level must be an integer in [0, 3], got {max_level!r}")
    if radius <= 0:
        raise MeshError(f"domain radius must be positive, got {radius}")
    h0 = 2.0 * radius / n_base
    tol = 1e-9 * h0
    ijk = np.stack(np.meshgrid(*([np.arange(n_base)] * dim), indexing="ij"),
                   axis=-1).reshape(-1, dim)
    lo = -radius + ijk * h0
    width = np.full_like(lo, h0)
    levels = np.zeros(len(lo), dtype=np.int64)
    n_fine = n_base * 2 ** max_level
    h_fine = h0 / 2 ** max_level
    for _ in range(max_level):
        if marker is None:
            ctr = lo + 0.5 * width
            dist = np.sqrt((ctr * ctr).sum(axis=1))
            mark = dist <= dist.min() + tol
        else:
            mark = np.array([bool(marker(VelocityCell(int(levels[i]), lo[i], width[i])))
                             for i in range(len(levels))])
        if not mark.any():
            break
        levels, lo, width = _children(levels, lo, width, mark)
        for _ in range(max_level + 2):
            bad = _violators(levels, lo, width, radius, h_fine, n_fine)
            if not bad.any():
                break
            levels, lo, width = _children(levels, lo, width, bad)
        else:
            raise MeshError("2:1 balance could not be restored")
    order = np.lexsort(tuple(lo[:, d] for d in reversed(range(dim))))
    return VelocityMesh(dim, float(radius), int(n_base), int(max_level),
                        levels[order], lo[order], width[order])


def ip_count(mesh: VelocityMesh, degree: int) -> int:
    """Total integration points (vmesh.py:171-173)."""
    return mesh.n_cells * (degree + 1) ** mesh.dim


def dump_mesh(mesh: VelocityMesh, path) -> None:
    """Cell list as CSV: id, level, lower corner, widths, %.17e (vmesh.py:176-187)."""
    names = ["cell", "level"] + [f"lo_{d}" for d in range(mesh.dim)] + \
        [f"h_{d}" for d in range(mesh.dim)]
    with open(path, "w", newline="\n") as fh:
        fh.write(",".join(names) + "\n")
        for i in range(mesh.n_cells):
            vals = [f"{v:.17e}" for v in (*mesh.lo[i], *mesh.width[i])]
            fh.write(",".join([str(i), str(int(mesh.levels[i]))] + vals) + "\n")
