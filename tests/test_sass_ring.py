"""SASS guard for the TMA ring's release invariant ("Pipeline
invariant"; profiles/README.md r1z).

A consumer warp of tma_gemm_kernel / core_kr_tma_kernel releases a ring stage
(SYNCS.ARRIVE.TRANS64.A1T0 on the stage's empty mbarrier) through
mbar_arrive_after(): the arrive is predicated on a DSETP of one accumulator of the
stage's last k-step.  The stage may be refilled as soon as the arrive lands, so every
shared-memory fragment load (LDS) of the stage must have RETURNED by then.  Issue is
in order and a DMMA issues only once its register operands are written, so the
invariant holds when every LDS result loaded since the stage's full-barrier wait
(SYNCS.PHASECHK) is read by an instruction placed before the arrive (a DMMA, or
the DMUL forming the core kernel's Khatri-Rao fragment); the DSETP dependency
keeps the arrive below the DMMAs it is predicated on.  Round 1's race was an arrive
hoisted above the stage's last DMMAs (loads still in flight: ~2 % of cfg 4 calls
transiently wrong).  This test reads the built library's SASS (cuobjdump, no GPU
needed) and checks that dataflow for every release arrive (ptxas may order the last
DMMAs either way; what matters is that none of them - and so none of the loads -
falls after the arrive).
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


def _dst_regs(args):
    r = _reg(args.split(",")[0])
    return [] if r is None else [r, r + 1]  # 64-bit loads write a register pair


def check_ring_release(body):
    """Return (n_arrives_checked, [problems]) for one kernel's instruction list."""
    probs, n = [], 0
    for i, (op, args) in enumerate(body):
        if not (op.startswith("SYNCS.ARRIVE.TRANS64") and ".A1T0" in op):
            continue
        # the predicate's DSETP (unpredicated arrives are the producer's / end marker)
        j = next((k for k in range(i - 1, max(-1, i - 40), -1) if body[k][0].startswith("DSETP")), None)
        if j is None:
            continue
        n += 1
        src = [_reg(t) for t in body[j][1].split(",")[2:4]]
        src = [s for s in src if s is not None]
        w = next((k for k in range(j - 1, -1, -1) if body[k][0].startswith("SYNCS.PHASECHK")), -1)
        pending, dmma_dst, saw_lds = {}, set(), False
        for k in range(w + 1, i):
            o, a = body[k]
            if o.startswith("LDS"):
                saw_lds = True
                for r in _dst_regs(a):
                    pending[r] = k
            else:
                # any reader of the loaded register (DMMA, or the core kernel's DMUL that
                # forms the Khatri-Rao fragment) issues only after the load returned
                ops = a.split(",")
                if o.startswith("DMMA"):
                    d = _reg(ops[0])
                    if d is not None:
                        dmma_dst.update(range(d, d + 4))
                for t in ops[1:]:
                    for r in map(int, re.findall(r"\bR(\d+)", t)):
                        pending.pop(r, None)  # fp64 operands name the pair's low register
                        pending.pop(r + 1, None)
        if not saw_lds:
            probs.append(f"arrive @{i}: no fragment load between the stage wait and the arrive")
        if not src or src[0] not in dmma_dst:
            probs.append(f"arrive @{i}: DSETP reads R{src[0] if src else '?'}, not a DMMA result of the stage")
        if pending:
            probs.append(f"arrive @{i}: LDS results {sorted(set(pending.values()))} not consumed by a DMMA before it")
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


def test_checker_flags_a_late_consumer():
    """The checker itself: an LDS whose DMMA falls after the arrive fails; either order
    of the stage's last two DMMAs passes."""
    wait = ("SYNCS.PHASECHK.TRANS64.TRYWAIT", "P0, [R5+URZ], R4")
    lds = [("LDS.64", "R68, [R2]"), ("LDS.64", "R58, [R3]"), ("LDS.64", "R62, [R4]")]
    d1, d2 = ("DMMA.8x8x4", "R12, R68, R58, R12"), ("DMMA.8x8x4", "R36, R62, R58, R36")
    tail = [("DSETP.NEU.AND", "P0, PT, R38, R38, PT"), ("SYNCS.ARRIVE.TRANS64.A1T0", "RZ, [R5+URZ], RZ")]
    assert check_ring_release([wait] + lds + [d1, d2] + tail) == (1, [])
    assert check_ring_release([wait] + lds + [d2, d1] + tail) == (1, [])
    n, p = check_ring_release([wait] + lds + [d2] + tail + [d1])
    assert n == 1 and len(p) == 1 and "not consumed" in p[0]
