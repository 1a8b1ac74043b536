"""Reference-element constants (host setup, uploaded once to the device).

Mirror of `sldg_vlasov.basis` (basis.py:19-148): GLL nodes/weights, the
2p+2-point Gauss rule, the exact Lagrange mass matrix and its inverse, the
differentiation matrix.  These are per-degree constants computed once on the
host; every per-step evaluation (Lagrange products for overlap matrices) runs
on the GPU (csrc/sldg_common.cuh).
"""
from __future__ import annotations

import numpy as np

MAX_DEGREE = 8
MAX_GAUSS_POINTS = 20


def _legendre3(p, x):
    """P_p and its first two derivatives by recurrence (basis.py:19-40)."""
    x = np.asarray(x, dtype=float)
    prev = [np.zeros_like(x)] * 3
    cur = [np.ones_like(x), np.zeros_like(x), np.zeros_like(x)]
    for k in range(1, p + 1):
        a, b = (2.0 * k - 1.0) / k, (k - 1.0) / k
        nxt = [a * x * cur[0] - b * prev[0],
               a * (cur[0] + x * cur[1]) - b * prev[1],
               a * (2.0 * cur[1] + x * cur[2]) - b * prev[2]]
        prev, cur = cur, nxt
    return cur


def gll_rule(p: int):
    """GLL nodes and weights, p+1 points (basis.py:43-74)."""
    if not isinstance(p, (int, np.integer)) or not 1 <= p <= MAX_DEGREE:
        raise ValueError(f"degree must be an integer in [1, {MAX_DEGREE}], got {p!r}")
    if p == 1:
        return np.array([-1.0, 1.0]), np.array([1.0, 1.0])
    x = np.cos(np.pi * np.arange(1, p) / p)
    for _ in range(100):
        _, d1, d2 = _legendre3(p, x)
        dx = -((1.0 - x * x) * d1) / (-2.0 * x * d1 + (1.0 - x * x) * d2)
        x = x + dx
        if np.max(np.abs(dx)) < 1e-15:
            break
    nodes = np.concatenate(([-1.0], np.sort(x), [1.0]))
    nodes = 0.5 * (nodes - nodes[::-1])
    nodes[0], nodes[-1] = -1.0, 1.0
    val = _legendre3(p, nodes)[0]
    w = 2.0 / (p * (p + 1) * val * val)
    return nodes, 0.5 * (w + w[::-1])


def gauss_rule(n: int):
    """n-point Gauss-Legendre rule (basis.py:77-81)."""
    if not isinstance(n, (int, np.integer)) or not 1 <= n <= MAX_GAUSS_POINTS:
        raise ValueError(f"point count must be an integer in [1, {MAX_GAUSS_POINTS}], got {n!r}")
    return np.polynomial.legendre.leggauss(int(n))


class DGBasis:
    """Degree-p nodal GLL basis (basis.DGBasis, basis.py:84-148)."""

    def __init__(self, degree: int):
        self.degree = int(degree)
        self.nodes, self.weights = gll_rule(degree)
        self.gauss_nodes, self.gauss_weights = gauss_rule(2 * self.degree + 2)
        o = self.degree + 1
        self._others = np.array([[m for m in range(o) if m != j] for j in range(o)],
                                dtype=np.intp)
        self._inv_denoms = 1.0 / np.array(
            [np.prod(self.nodes[j] - self.nodes[self._others[j]]) for j in range(o)])
        v = self.eval_all(self.gauss_nodes)
        m = v.T @ (self.gauss_weights[:, None] * v)
        self.mass = 0.5 * (m + m.T)
        self.mass_inv = np.linalg.inv(self.mass)
        bw = self._inv_denoms
        d = np.where(np.eye(o, dtype=bool), 0.0,
                     (bw[None, :] / bw[:, None])
                     / np.where(np.eye(o, dtype=bool), 1.0,
                                self.nodes[:, None] - self.nodes[None, :]))
        np.fill_diagonal(d, -d.sum(axis=1))
        self.diff = d

    @property
    def n_nodes(self) -> int:
        return self.degree + 1

    def eval_all(self, x) -> np.ndarray:
        """Every Lagrange polynomial at x (host; basis.py:119-128)."""
        x = np.asarray(x, dtype=float)
        return (x[..., None] - self.nodes)[..., self._others].prod(axis=-1) * self._inv_denoms

    def eval_lagrange(self, j: int, x):
        return self.eval_all(x)[..., j]
