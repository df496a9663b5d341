"""Seeded synthetic workloads for the RHOSVD canonical-to-Tucker hot path.

This module holds INPUTS ONLY: it draws the parameters of the five
BASELINE.json configurations (and small random cases for parity tests) and
samples the canonical vectors u_k^(l)(x_i) on the grid.  It contains none of
the method's arithmetic (no normalisation, no SVD, no projection, no core), so
it may serve both the CPU oracle (oracle/) and the CUDA path
(paper_2201_12663_b200/) without the two sharing any code of the method.

Input contract (Eq. (can_A3), Eq.
(can_A_Tuck)): A = sum_k xi_k u_k^(1) (x) u_k^(2) (x) u_k^(3), side matrices
U^(l) = [u_1 ... u_R] in R^{n x R}.  Layout used everywhere in this repo:
U^(l) is stored COLUMN-MAJOR n x R, i.e. as a C-contiguous array of shape
(R, n) whose row k is the canonical vector u_k^(l).

Readings:
  * A5 grid: cell-centred x_i = -b + (i + 1/2) * 2b/n, i = 0..n-1, the same in
    all three modes; collocation (point sampling).
  * A6 Gaussians u(x) = exp(-a (x - c)^2) with `a` the exponent.
  * A7 Newton kernel 1/|x| by the BASELINE.json sinc rule p_t = e^{t h},
    h = 0.3, t = -12..11, exponent p_t^2, weight h p_t 2/sqrt(pi)
    (trapezoid rule of 1/z = 2/sqrt(pi) int_0^inf e^{-z^2 s^2} ds in
    w = ln s).
  * A8 Hartree-like density: one orbital with N(0,1) coefficients, pair
    products of Gaussians in analytic (Gaussian product theorem) form,
    pairs i <= j in numpy.triu_indices order (Eq. rho_ten).

Every config uses numpy.random.default_rng(1000 + k) and draws in the order
listed in SURVEY.md 8(d).  Sharded generation: every rank draws the full
parameter arrays and evaluates only its own contiguous column block, so the
p-way sharded input is bit-identical to the 1-way input.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Params", "CONFIGS", "make_params", "grid", "eval_columns",
    "make_config", "make_random_params", "shard_bounds",
]


@dataclass
class Params:
    """Per-term parameters of a Gaussian-sum canonical tensor.

    a[k]   : exponent of term k (same in all modes)
    c[k,l] : centre of term k in mode l
    xi[k]  : weight of term k (before normalisation)
    """
    name: str
    n: int
    b: float                  # box half-width: grid covers [-b, b]
    a: np.ndarray             # (R,)
    c: np.ndarray             # (R, 3)
    xi: np.ndarray            # (R,)
    eps: float | None = None  # epsilon-mode truncation
    ranks: tuple | None = None  # fixed-rank mode
    meta: dict = field(default_factory=dict)

    @property
    def R(self) -> int:
        return int(self.a.shape[0])


# BASELINE.json "configs", indexed 1..5 as in SURVEY.md.
CONFIGS = {
    1: dict(name="cfg1-gauss-sum", n=64, b=5.0, R=200, ranks=(10, 10, 10), eps=None),
    2: dict(name="cfg2-newton-100", n=512, b=8.0, R=2400, ranks=None, eps=1e-5),
    3: dict(name="cfg3-hartree-120", n=2048, b=10.0, R=7260, ranks=None, eps=1e-6),
    4: dict(name="cfg4-biomol-2000", n=2048, b=12.0, R=48000, ranks=None, eps=1e-5),
    5: dict(name="cfg5-scattered-1e5", n=4096, b=1.2, R=100000, ranks=None, eps=1e-6),
}


def grid(n: int, b: float) -> np.ndarray:
    """Cell-centred grid on [-b, b] (reading A5)."""
    h = 2.0 * b / n
    return -b + (np.arange(n, dtype=np.float64) + 0.5) * h


def _newton_sinc_rule():
    """BASELINE.json sinc rule for 1/|x| (reading A7)."""
    hq = 0.3
    t = np.arange(-12, 12, dtype=np.float64)
    p = np.exp(t * hq)
    w = hq * p * 2.0 / math.sqrt(math.pi)
    return p * p, w  # exponents p_t^2 and weights


def make_params(k: int) -> Params:
    """Draw the parameters of BASELINE.json config k (1..5), SURVEY.md 8(d)."""
    cfg = CONFIGS[k]
    rng = np.random.default_rng(1000 + k)
    n, b, R = cfg["n"], cfg["b"], cfg["R"]
    if k == 1:
        a = np.exp(rng.uniform(math.log(0.5), math.log(20.0), R))
        c = rng.uniform(-3.0, 3.0, (R, 3))
        xi = rng.uniform(0.5, 1.5, R)
    elif k in (2, 4):
        nq = 100 if k == 2 else 2000
        lo = 4.0 if k == 2 else 6.0
        X = rng.uniform(-lo, lo, (nq, 3))
        if k == 2:
            q = rng.choice(np.array([-1.0, 1.0]), nq)
        else:
            q = rng.uniform(-1.0, 1.0, nq)
        ex, w = _newton_sinc_rule()
        # term index k = 24 j + (t + 12)
        a = np.tile(ex, nq)
        c = np.repeat(X, 24, axis=0)
        xi = (q[:, None] * w[None, :]).reshape(-1)
    elif k == 3:
        nb = 120
        al = np.exp(rng.uniform(math.log(0.1), math.log(50.0), nb))
        Cb = rng.uniform(-3.0, 3.0, (nb, 3))
        cc = rng.normal(size=nb)
        ii, jj = np.triu_indices(nb)
        a = al[ii] + al[jj]
        c = (al[ii, None] * Cb[ii] + al[jj, None] * Cb[jj]) / a[:, None]
        d2 = np.sum((Cb[ii] - Cb[jj]) ** 2, axis=1)
        xi = np.where(ii == jj, 1.0, 2.0) * cc[ii] * cc[jj] * np.exp(-al[ii] * al[jj] / a * d2)
    elif k == 5:
        c = rng.uniform(-1.0, 1.0, (R, 3))
        a = np.exp(rng.uniform(math.log(5.0), math.log(500.0), R))
        xi = rng.normal(size=R)
    else:
        raise ValueError(f"unknown config {k}")
    assert a.shape[0] == R, (k, a.shape, R)
    return Params(name=cfg["name"], n=n, b=b, a=np.ascontiguousarray(a, np.float64),
                  c=np.ascontiguousarray(c, np.float64), xi=np.ascontiguousarray(xi, np.float64),
                  eps=cfg["eps"], ranks=cfg["ranks"], meta={"config": k})


def make_random_params(n: int, R: int, seed: int, eps: float | None = None,
                       ranks: tuple | None = None, b: float = 5.0,
                       a_range=(0.5, 20.0), signed: bool = True) -> Params:
    """Small random Gaussian-sum case shaped like cfg 1 (for parity tests at
    sizes the oracle finishes in seconds, spanning several tiles and a ragged
    tail).  Same value distribution as cfg 1, signed weights optional."""
    rng = np.random.default_rng(seed)
    a = np.exp(rng.uniform(math.log(a_range[0]), math.log(a_range[1]), R))
    c = rng.uniform(-0.6 * b, 0.6 * b, (R, 3))
    xi = rng.normal(size=R) if signed else rng.uniform(0.5, 1.5, R)
    return Params(name=f"random-n{n}-R{R}-s{seed}", n=n, b=b, a=a, c=c, xi=xi,
                  eps=eps, ranks=ranks, meta={"seed": seed})


def shard_bounds(R: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous column block of rank `rank`: ceil(R/p) terms, last gets fewer."""
    per = -(-R // world) if world > 0 else R
    lo = min(R, rank * per)
    hi = min(R, lo + per)
    return lo, hi


def eval_columns(p: Params, mode: int, k0: int = 0, k1: int | None = None,
                 backend: str = "numpy", device=None):
    """Sample u_k^(mode)(x_i) = exp(-a_k (x_i - c_k,mode)^2) for k in [k0, k1).

    Returns an array of shape (k1-k0, n), C-contiguous (column-major n x R).
    backend="numpy" (host) or "torch" (torch.float64 on `device`).
    """
    k1 = p.R if k1 is None else k1
    x = grid(p.n, p.b)
    a = p.a[k0:k1]
    c = p.c[k0:k1, mode]
    if backend == "numpy":
        out = np.empty((k1 - k0, p.n), dtype=np.float64)
        step = max(1, (1 << 24) // max(1, p.n))
        for s in range(0, k1 - k0, step):
            e = min(k1 - k0, s + step)
            d = x[None, :] - c[s:e, None]
            np.exp(-a[s:e, None] * (d * d), out=out[s:e])
        return out
    if backend == "torch":
        import torch
        xt = torch.as_tensor(x, dtype=torch.float64, device=device)
        at = torch.as_tensor(a, dtype=torch.float64, device=device)
        ct = torch.as_tensor(c, dtype=torch.float64, device=device)
        d = xt[None, :] - ct[:, None]
        return torch.exp(-at[:, None] * (d * d)).contiguous()
    raise ValueError(backend)


def make_config(p: Params | int, k0: int = 0, k1: int | None = None,
                backend: str = "numpy", device=None):
    """Return (U1, U2, U3, xi) for terms [k0, k1) of a workload.

    U_l: (k1-k0, n) C-contiguous = column-major n x (k1-k0); xi: (k1-k0,).
    """
    if isinstance(p, int):
        p = make_params(p)
    k1 = p.R if k1 is None else k1
    Us = [eval_columns(p, m, k0, k1, backend, device) for m in range(3)]
    xi = p.xi[k0:k1].copy()
    if backend == "torch":
        import torch
        xi = torch.as_tensor(xi, dtype=torch.float64, device=device)
    return Us[0], Us[1], Us[2], xi
