"""SASS guard for the TMA ring's release invariant ("Pipeline
invariant"; profiles/README.md r1z).

A consumer warp of tma_gemm_kernel / core_kr_tma_kernel releases a ring stage
(SYNCS.ARRIVE.TRANS64.A1T0 on the stage's empty mbarrier) through
mbar_arrive_after(): the arrive is predicated on a DSETP of one accumulator of the
stage's last k-step.  That orders the release after every fragment load of the stage
only if the DMMA producing that accumulator is the LAST DMMA issued before the
arrive (in-order issue: a DMMA issues once its shared-memory operands have
returned, so every earlier DMMA of the stage, and the loads feeding it, are done).
A compiler or flag change that schedules another DMMA after it would bring back
the transiently wrong GEMMs (~2 % of cfg 4 calls before the fix).  This test reads
the built library's SASS (cuobjdump, no GPU needed) and checks, for every release
arrive, that the DSETP operand comes from the last DMMA before it.
"""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2201_12663_b200", "librhosvd.so")

INS = re.compile(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Za-z0-9_.]*)\s*([^;]*);")


def _functions(sass):
    cur, body = None, []
    for ln in sass.splitlines():
        if "Function :" in ln:
            if cur:
                yield cur, body
            cur, body = ln.split("Function :")[1].strip(), []
            continue
        m = INS.search(ln)
        if m and cur:
            body.append((m.group(2), m.group(3)))
    if cur:
        yield cur, body


def _reg(tok):
    m = re.match(r"-?\|?R(\d+)", tok.strip())
    return int(m.group(1)) if m else None


def check_ring_release(body):
    """Return (n_arrives_checked, [problems]) for one kernel's instruction list."""
    probs, n = [], 0
    for i, (op, args) in enumerate(body):
        if not (op.startswith("SYNCS.ARRIVE.TRANS64") and ".A1T0" in op):
            continue
        # the predicate's DSETP, then the last DMMA before it
        j = next((k for k in range(i - 1, max(-1, i - 40), -1) if body[k][0].startswith("DSETP")), None)
        if j is None:
            continue  # unpredicated arrive (producer side / not a consumer release)
        n += 1
        src = [_reg(t) for t in body[j][1].split(",")[2:4]]
        src = [s for s in src if s is not None]
        m = next((k for k in range(j - 1, -1, -1) if body[k][0].startswith("DMMA")), None)
        if m is None or not src:
            probs.append(f"arrive @{i}: no DMMA / register before its DSETP")
            continue
        dst = _reg(body[m][1].split(",")[0])
        if dst is None or not (dst <= src[0] <= dst + 3):
            probs.append(f"arrive @{i}: DSETP reads R{src[0]}, last DMMA writes R{dst}..R{dst + 3 if dst else '?'}")
    return n, probs


@pytest.mark.skipif(not os.path.exists(SO) or not shutil.which("cuobjdump"), reason="librhosvd.so / cuobjdump missing")
def test_ring_release_depends_on_last_dmma():
    sass = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True, check=True).stdout
    checked, kernels, problems = 0, 0, []
    for name, body in _functions(sass):
        if "tma_gemm_kernel" not in name and "core_kr_tma_kernel" not in name:
            continue
        n, p = check_ring_release(body)
        assert n > 0, f"{name}: no predicated release arrive found (mbar_arrive_after missing?)"
        kernels += 1
        checked += n
        problems += [f"{name}: {x}" for x in p]
    assert kernels >= 20, kernels
    assert not problems, "\n".join(problems[:20])


def test_checker_flags_a_reordered_dmma():
    """The checker itself: a DMMA scheduled between the dependency DMMA and the DSETP fails."""
    good = [("DMMA.8x8x4", "R12, R68, R58, R12"), ("DMMA.8x8x4", "R36, R62, R58, R36"),
            ("DSETP.NEU.AND", "P0, PT, R38, R38, PT"), ("SYNCS.ARRIVE.TRANS64.A1T0", "RZ, [R5+URZ], RZ")]
    assert check_ring_release(good) == (1, [])
    bad = [good[1], good[0], good[2], good[3]]
    n, p = check_ring_release(bad)
    assert n == 1 and len(p) == 1
