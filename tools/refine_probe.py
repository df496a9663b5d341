"""Accuracy of the retained sigma and of the Tucker tensor against the CPU oracle as a
function of the refinement step count (RHOSVD_REFINE_MAX caps the model's count).

    RHOSVD_REFINE_MAX=1 python tools/refine_probe.py 1 2 3 5
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main(ks):
    import torch
    from oracle import rhosvd as oracle_rhosvd, sigma_rel_err, tucker_diff
    from paper_2201_12663_b200 import rhosvd
    from workloads import make_config, make_params
    dev = torch.device("cuda:0")
    for k in ks:
        p = make_params(k)
        U1, U2, U3, xi = make_config(p)
        Ud = [torch.as_tensor(u, device=dev) for u in (U1, U2, U3)]
        xd = torch.as_tensor(xi, device=dev)
        g = rhosvd.c2t(Ud, xd, eps=p.eps, ranks=p.ranks)
        out = {"config": k, "refine_max": os.environ.get("RHOSVD_REFINE_MAX"), "ranks": list(g.ranks),
               "refines": g.report["refines"], "iters": g.report["iters"], "block": g.report["block"],
               "ms": g.report["ms"]["total"]}
        if k <= 3:
            o = oracle_rhosvd([U1, U2, U3], xi, eps=p.eps, ranks=p.ranks)
            out["ranks_ok"] = tuple(g.ranks) == tuple(o.ranks)
            out["sigma_err"] = [sigma_rel_err(g.sigma[l].cpu().numpy(), o.sigma[l][:o.ranks[l]]) for l in range(3)]
            d, nrm = tucker_diff(g.beta.cpu().numpy(), [z.cpu().numpy() for z in g.Z], o.beta, o.Z)
            out["tucker_rel"] = d / nrm
        else:
            fx = np.load(os.path.join(ROOT, "tests", "golden", "large", f"oracle_cfg{k}_frames.npz"))
            out["ranks_ok"] = tuple(g.ranks) == tuple(int(x) for x in fx["ranks"])
            out["sigma_err"] = [sigma_rel_err(g.sigma[l].cpu().numpy(), fx[f"sigma{l + 1}"]) for l in range(3)]
            Zo = [fx["Z1"], fx["Z2"], fx["Z3"]]
            if k == 5:
                d, nrm = tucker_diff(g.beta.cpu().numpy(), [z.cpu().numpy() for z in g.Z], fx["beta"], Zo)
            else:
                from fullsize_compare import tucker_diff_cp
                from oracle import normalize, project
                Uh, xip, _, _ = normalize([U1, U2, U3], xi)
                Wo = [project(Zo[l], Uh[l]) for l in range(3)]
                del Uh
                d, nrm = tucker_diff_cp(g.beta, g.Z, Zo, Wo, xip, device=dev)
            out["tucker_rel"] = d / nrm
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 3, 5, 4])
