"""The collective path of rhosvd_c2t on ONE GPU: a world-1 communicator with
RHOSVD_COMM_FORCE=1 runs every all-reduce anyway (NCCL: a real ncclAllReduce over one
rank; callback: the gloo round trip), through the same comm thread / CommSched that the
R-sharded multi-GPU path uses with concurrent per-mode solves.  An all-reduce over one rank
is an identity, so the outputs must be BITWISE those of the communicator-free call; the
host-buffer entry point takes its after-all-reduce beta D2H branch here."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

SCRIPT = r'''
import os, socket, sys
sys.path.insert(0, {root!r})
import torch, torch.distributed as dist
s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
dist.init_process_group("gloo", rank=0, world_size=1)
from paper_2201_12663_b200 import rhosvd
from workloads import make_config, make_params, make_random_params
kind = sys.argv[1]
for p in (make_random_params(70, 517, seed=23, eps=1e-7), make_params(2)):
    U1, U2, U3, xi = make_config(p, backend="torch", device=torch.device("cuda:0"))
    ref = rhosvd.c2t([U1, U2, U3], xi, eps=p.eps, ranks=p.ranks, keep_w=False)
    comm = rhosvd.Comm.nccl() if kind == "nccl" else rhosvd.Comm.callback()
    got = rhosvd.c2t([U1, U2, U3], xi, eps=p.eps, ranks=p.ranks, comm=comm, keep_w=False)
    assert tuple(got.ranks) == tuple(ref.ranks), (got.ranks, ref.ranks)
    assert torch.equal(got.beta, ref.beta)
    for a, b in zip(got.Z, ref.Z):
        assert torch.equal(a, b)
    # RHOSVD_F_ROOT_ONLY_CORE: ncclReduce to rank 0 (a world-1 reduce is an identity)
    ro = rhosvd.c2t([U1, U2, U3], xi, eps=p.eps, ranks=p.ranks, comm=comm, keep_w=False, root_only_core=True)
    assert torch.equal(ro.beta, ref.beta)
    hU = [u.cpu().pin_memory() for u in (U1, U2, U3)]
    h = rhosvd.c2t_host(hU, xi.cpu().pin_memory(), eps=p.eps, ranks=p.ranks, comm=comm)
    assert torch.equal(h.beta, ref.beta.cpu())
    h.close()
    comm.close()
dist.destroy_process_group()
print("ok")
'''


@pytest.mark.parametrize("kind", ["nccl", "callback"])
def test_forced_collectives_world1(kind):
    env = dict(os.environ, RHOSVD_COMM_FORCE="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT), kind], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout[-2000:], r.stderr[-3000:])
