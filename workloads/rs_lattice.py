"""Seeded inputs of the RS long-range front-end: the geometry
and amplitudes of the multi-Slater lattices of PAPER.md section 4.5 (Tables 2-3,
Fig. 5).  INPUTS ONLY - no quadrature, split or any other step of the method (those
live in oracle/rs_oracle.py and in the CUDA library, independently).

Readings:
  * grid: n = 384 cell-centred points on [-b, b], b = 12 (reading A5; the paper gives
    n = 384 but not the box);
  * lattice: L1 x L2 x L3 nodes ON grid points, spacing 16 cells (= 1.0), centred at
    grid index n / 2 (the paper does not give the spacing);
  * amplitudes c_j ~ U[-5, 5] ("randomly chosen weights c_j in the interval [-5, 5]",
    PAPER.md:1474-1476), or the functional amplitudes of Eq. (func2)
    F(x, y, z) = 6 cos(x + 2y + 4z) exp(-0.1 sqrt(x^2 + 2y^2 + 4z^2));
  * Slater exponent lambda = 0.5 (PAPER.md:1488 / 1536 figure captions).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .generators import grid

__all__ = ["RSLattice", "make_rs_lattice", "TABLE2_LATTICES", "TABLE3_LATTICES"]

# PAPER.md:1447-1469 (Table 2) and PAPER.md:1541-1563 (Table 3)
TABLE2_LATTICES = [(4, 4, 4), (6, 6, 6), (8, 8, 8), (16, 16, 8), (16, 16, 16)]
TABLE3_LATTICES = TABLE2_LATTICES


@dataclass
class RSLattice:
    name: str
    n: int
    b: float
    lam: float
    L: tuple
    node_idx: np.ndarray   # (N, 3) int32 grid indices of the nodes
    nodes: np.ndarray      # (N, 3) node coordinates x[node_idx]
    c: np.ndarray          # (N,) amplitudes

    @property
    def N(self) -> int:
        return int(self.node_idx.shape[0])

    @property
    def h(self) -> float:
        return 2.0 * self.b / self.n

    @property
    def x(self) -> np.ndarray:
        return grid(self.n, self.b)


def make_rs_lattice(L, n=384, b=12.0, spacing=16, lam=0.5, amplitudes="random", seed=2022, first=None) -> RSLattice:
    """L1 x L2 x L3 lattice of Slater centres on the n-grid (node-major order: the
    last lattice index fastest); centred at grid index n / 2, or starting at grid index
    `first` in every mode."""
    L = tuple(int(v) for v in L)
    x = grid(n, b)
    if first is None:
        axes = [n // 2 + spacing * (np.arange(Lk) - (Lk - 1) // 2) for Lk in L]
    else:
        axes = [first + spacing * np.arange(Lk) for Lk in L]
    for a in axes:
        if a.min() < 0 or a.max() >= n:
            raise ValueError("lattice does not fit the grid")
    idx = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1).reshape(-1, 3).astype(np.int32)
    nodes = x[idx]
    if amplitudes == "random":
        c = np.random.default_rng(seed + 7 * L[0] + 131 * L[2]).uniform(-5.0, 5.0, idx.shape[0])
    elif amplitudes == "func":
        X, Y, Zc = nodes[:, 0], nodes[:, 1], nodes[:, 2]
        c = 6.0 * np.cos(X + 2 * Y + 4 * Zc) * np.exp(-0.1 * np.sqrt(X * X + 2 * Y * Y + 4 * Zc * Zc))
    else:
        raise ValueError(amplitudes)
    return RSLattice(name=f"slater-lattice-{L[0]}x{L[1]}x{L[2]}-{amplitudes}", n=n, b=b, lam=lam, L=L,
                     node_idx=np.ascontiguousarray(idx), nodes=np.ascontiguousarray(nodes), c=c)
