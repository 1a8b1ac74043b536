"""1D SLDG pieces of the public API (sldg_vlasov.sldg1d, sldg1d.py:18-100).

`decompose_shift` is the scalar split every kernel restates on the device
(bit-identical, csrc/sldg_common.cuh split_shift); `overlap_pair` evaluates
the A/B projection blocks ON THE DEVICE through sldg_overlap_pairs -- the same
code the sweep kernels run per column and level.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

PERIODIC = "periodic"
ABSORBING = "absorbing"

_ONE_MINUS_ULP = float(np.nextafter(1.0, 0.0))


def check_bc(bc: str) -> str:
    if bc not in (PERIODIC, ABSORBING):
        raise ValueError(f"boundary mode must be {PERIODIC!r} or {ABSORBING!r}, got {bc!r}")
    return bc


@dataclass(frozen=True)
class ShiftDecomposition:
    n_shift: int
    frac: float


def decompose_shift(speed: float, dt: float, width: float) -> ShiftDecomposition:
    """speed*dt/width = n + frac, frac in [0, 1), 1-ulp fold (sldg1d.py:39-55)."""
    if width <= 0.0:
        raise ValueError(f"cell width must be positive, got {width}")
    if dt <= 0.0:
        raise ValueError(f"time step must be positive, got {dt}")
    r = speed * dt / width
    n = math.floor(r)
    frac = r - n
    if frac >= _ONE_MINUS_ULP:
        return ShiftDecomposition(n + 1, 0.0)
    return ShiftDecomposition(n, frac)


@dataclass(frozen=True)
class OverlapPair:
    same: np.ndarray
    neighbor: np.ndarray
    frac: float


def overlap_pairs_device(basis, fracs):
    """A/B blocks for many fractional shifts, computed by the CUDA kernel."""
    import torch

    from . import _capi
    from ._device import current_stream, device

    fr = np.ascontiguousarray(np.asarray(fracs, dtype=np.float64).ravel())
    if fr.size and (fr.min() < 0.0 or fr.max() >= 1.0):
        raise ValueError("fractional shift must lie in [0, 1)")
    o = basis.degree + 1
    dev = device()
    f_d = torch.from_numpy(fr).to(dev)
    A = torch.empty((fr.size, o, o), dtype=torch.float64, device=dev)
    B = torch.empty_like(A)
    ba = _capi.BasisArrays(basis)
    _capi.check(_capi.lib().sldg_overlap_pairs(ba.struct, f_d.data_ptr(), fr.size, A.data_ptr(),
                                               B.data_ptr(), current_stream()), ValueError)
    return A.cpu().numpy(), B.cpu().numpy()


def overlap_pair(basis, frac: float) -> OverlapPair:
    """Same/neighbour blocks for one fractional shift (sldg1d.py:82-100), on device."""
    if not 0.0 <= frac < 1.0:
        raise ValueError(f"fractional shift must lie in [0, 1), got {frac}")
    A, B = overlap_pairs_device(basis, [frac])
    return OverlapPair(A[0], B[0], float(frac))
