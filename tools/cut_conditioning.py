"""How well is the rank-r Tucker tensor of a sweep case determined in fp64 at all?

Runs the CPU oracle (QR-first gesdd, oracle/rhosvd_oracle.py) and a second fp64 route
(scipy gesvd on the n x R side matrix directly, no QR) on the same input and prints the
Tucker-tensor distance between the two, next to the per-mode cut gaps
sigma_r^2 - sigma_{r+1}^2 (relative to sigma_1^2).  If two textbook fp64 SVDs disagree
by ~1e-9 on a case, the 1e-9 bound is not attainable there by any fp64 method and a
GPU-vs-oracle distance of the same size is the cut's conditioning, not an error.

Usage: python tools/cut_conditioning.py SWEEP_SEED CASE [CASE ...]
(the case parameters are drawn exactly as tools/parity_sweep.py draws them)."""
import sys

import numpy as np
import scipy.linalg as sla

sys.path.insert(0, "/root/repo")
from workloads import make_config, make_random_params
from oracle import rhosvd as orh, tucker_diff
from oracle.rhosvd_oracle import normalize, select_rank, project, core_kr


def sweep_params(seed, upto):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(upto + 1):
        n = int(rng.integers(100, 1100)); R = int(rng.integers(200, 6000))
        if rng.random() < 0.7:
            eps, ranks = float(rng.choice([1e-3, 1e-4, 1e-5, 1e-6, 1e-7])), None
        else:
            eps, ranks = None, tuple(int(x) for x in rng.integers(1, min(n, R, 200), size=3))
        wide = bool(rng.random() < 0.5)
        out.append((n, R, eps, ranks, wide, i))
    return out


def second_route(Us, xi, ranks):
    """Tucker tensor of the same ranks from gesvd on the n x R matrix (no QR first)."""
    Uh, xip = normalize(Us, xi)[:2]
    Zs, Ws = [], []
    for l in range(3):
        Z, s, _ = sla.svd(Uh[l].T, full_matrices=False, lapack_driver="gesvd")
        Zs.append(Z[:, :ranks[l]])
        Ws.append(project(Zs[-1], Uh[l]))
    return core_kr(Ws[0], Ws[1], Ws[2], xip), Zs


def main():
    seed = int(sys.argv[1])
    cases = [int(c) for c in sys.argv[2:]]
    table = sweep_params(seed, max(cases))
    for c in cases:
        n, R, eps, ranks, wide, i = table[c]
        p = make_random_params(n, R, seed=50000 + i, eps=eps, ranks=ranks,
                               a_range=(0.05, 400.0) if wide else (0.5, 20.0), signed=bool(i % 2))
        U1, U2, U3, xi = make_config(p)
        o = orh([U1, U2, U3], xi, eps=eps, ranks=ranks)
        beta2, Z2 = second_route([U1, U2, U3], xi, o.ranks)
        d, nrm = tucker_diff(beta2, Z2, o.beta, o.Z)
        gaps = []
        for l in range(3):
            s = o.sigma[l]; r = o.ranks[l]
            g = (s[r - 1] ** 2 - s[r] ** 2) / s[0] ** 2 if r < len(s) else float("inf")
            gaps.append(g)
        print(f"case {c}: n {n} R {R} eps {eps} ranks {tuple(o.ranks)}  gesdd(QR) vs gesvd Tucker "
              f"{d / nrm:.2e}  cut gaps (sigma_r^2 - sigma_r+1^2)/sigma_1^2 "
              + " ".join(f"{g:.2e}" for g in gaps), flush=True)


if __name__ == "__main__":
    main()
