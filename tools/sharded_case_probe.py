"""World-2 (one GPU, host-callback all-reduce) probe of one fixed-rank case under a set of
environment variants, each with a wall-clock limit: prints which variants finish and the
library's RHOSVD_DEBUG trace of those that do not.  Usage: sharded_case_probe.py [limit_s]"""
import os
import socket
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = r'''
import os, sys
sys.path.insert(0, {root!r})
import torch, torch.distributed as dist
rank, n, R, seed = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
ranks = tuple(int(x) for x in sys.argv[5].split(","))
dist.init_process_group("gloo", rank=rank, world_size=2)
from paper_2201_12663_b200 import rhosvd
from workloads import make_config, make_random_params, shard_bounds
p = make_random_params(n, R, seed=seed, ranks=ranks, signed=(sys.argv[6] == "1"))
k0, k1 = shard_bounds(p.R, 2, rank)
U1, U2, U3, xi = make_config(p, k0, k1, backend="torch", device=torch.device("cuda:0"))
comm = rhosvd.Comm.callback()
res = rhosvd.c2t([U1, U2, U3], xi, ranks=p.ranks, comm=comm, keep_w=False)
torch.cuda.synchronize()
print("rank", rank, "done", res.ranks, flush=True)
comm.close()
dist.destroy_process_group()
'''

CASES = {"rltn": (589, 221, 50010, "133,31,107", "0"), "meqn": (644, 1571, 50019, "198,101,144", "1")}
VARIANTS = [("rltn", {}), ("rltn", {"RHOSVD_FULL_EYE": "2"}), ("rltn", {"RHOSVD_MODE_PARALLEL": "0"}),
            ("rltn", {"RHOSVD_SERIAL_MODES": "1"}), ("meqn", {}), ("meqn", {"RHOSVD_MODE_PARALLEL": "0"})]


def main():
    limit = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
    for case, env in VARIANTS:
        s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
        e = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RHOSVD_DEBUG="1", **env)
        procs = [subprocess.Popen([sys.executable, "-c", WORKER.format(root=ROOT), str(r), *map(str, CASES[case])],
                                  env=e, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(2)]
        t0 = time.time()
        while time.time() - t0 < limit and any(p.poll() is None for p in procs):
            time.sleep(0.5)
        hung = [p.poll() is None for p in procs]
        for p in procs:
            if p.poll() is None:
                p.kill()
        outs = [p.communicate()[0] for p in procs]
        print(f"=== {case} {env}: {'HUNG' if any(hung) else 'ok'} rc {[p.returncode for p in procs]} in {time.time() - t0:.1f} s", flush=True)
        for r, o in enumerate(outs):
            lines = o.strip().splitlines()
            print(f"--- rank {r} ({len(lines)} lines), tail:")
            print("\n".join(lines[-14:] if any(hung) or procs[r].returncode else lines[-2:]), flush=True)


if __name__ == "__main__":
    main()
