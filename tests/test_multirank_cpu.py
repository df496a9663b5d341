"""World-size-2 gloo tests of the R-sharded host logic (CPU, no GPU).

The CUDA path shards the R canonical terms over ranks and combines every
R-dependent quantity with an fp64 SUM all-reduce:
T_l, G_l = Uhat_l Uhat_l^T, the b x b Gram W W^T, Uhat X, rho and the core beta.
These tests run the same decomposition with the ORACLE's arithmetic on two gloo
ranks and check that (i) sharded generation is bit-identical to the unsharded
input, (ii) the all-reduced partial sums equal the unsharded quantities, and
(iii) the bench's max-over-ranks timing reduction picks the slowest rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import rhosvd as oracle_rhosvd
from oracle import normalize, project, core_kr
from workloads import make_config, make_random_params, shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = make_random_params(40, 257, seed=7, eps=1e-6)  # ragged: 257 terms over 2 ranks
        full = make_config(p)
        k0, k1 = shard_bounds(p.R, world, rank)
        loc = make_config(p, k0, k1)
        # (i) sharded generation == slice of the full input, bitwise
        same = all(np.array_equal(loc[i], full[i][k0:k1]) for i in range(3)) and \
            np.array_equal(loc[3], full[3][k0:k1])
        # the frames come from the full problem (in the library they are replicated
        # after the all-reduced Gram; here the oracle provides them)
        o = oracle_rhosvd(list(full[:3]), full[3], eps=p.eps)
        Uh, xip, _, T = normalize(list(loc[:3]), loc[3])
        # (ii) partial sums -> all-reduce
        Tt = torch.tensor(T, dtype=torch.float64)
        G = torch.tensor(np.stack([u.T @ u for u in Uh]), dtype=torch.float64)
        Ws = [project(o.Z[l], Uh[l]) for l in range(3)]
        S = torch.tensor(np.concatenate([(w @ w.T).ravel() for w in Ws]), dtype=torch.float64)
        beta = torch.tensor(core_kr(Ws[0], Ws[1], Ws[2], xip), dtype=torch.float64)
        xi2 = torch.tensor([float(xip @ xip)], dtype=torch.float64)
        for t in (Tt, G, S, beta, xi2):
            dist.all_reduce(t)
        # (iii) max-over-ranks timing (bench.py)
        from bench import max_over_ranks
        ms = max_over_ranks(10.0 + rank, None)
        if rank == 0:
            Uf, xipf, _, Tf = normalize(list(full[:3]), full[3])
            Gf = np.stack([u.T @ u for u in Uf])
            Wf = [project(o.Z[l], Uf[l]) for l in range(3)]
            Sf = np.concatenate([(w @ w.T).ravel() for w in Wf])
            q.put(dict(
                same=same, R=(k0, k1),
                dT=float(np.max(np.abs(Tt.numpy() - Tf))),
                dG=float(np.max(np.abs(G.numpy() - Gf)) / np.max(np.abs(Gf))),
                dS=float(np.max(np.abs(S.numpy() - Sf)) / np.max(np.abs(Sf))),
                dbeta=float(np.linalg.norm(beta.numpy() - o.beta) / np.linalg.norm(o.beta)),
                dxi=abs(float(np.sqrt(xi2.item())) - float(np.linalg.norm(xipf))),
                ms=ms))
        else:
            q.put(dict(same=same, R=(k0, k1), ms=ms))
    finally:
        dist.destroy_process_group()


def test_r_sharded_sums_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0 = [r for r in res if "dG" in r][0]
    assert all(r["same"] for r in res)
    assert sorted(r["R"] for r in res) == [(0, 129), (129, 257)]
    assert r0["dT"] < 1e-12
    assert r0["dG"] < 1e-14
    assert r0["dS"] < 1e-13
    assert r0["dbeta"] < 1e-13
    assert r0["dxi"] < 1e-12
    assert all(r["ms"] == 11.0 for r in res)


@pytest.mark.parametrize("R,world", [(0, 2), (1, 2), (7, 4), (48000, 8), (100000, 8), (10, 3)])
def test_shard_bounds_partition(R, world):
    b = [shard_bounds(R, world, r) for r in range(world)]
    assert b[0][0] == 0 and b[-1][1] == R
    for (lo, hi), (lo2, _) in zip(b, b[1:]):
        assert hi == lo2 and lo <= hi
    assert max(hi - lo for lo, hi in b) == (-(-R // world) if R else 0)
