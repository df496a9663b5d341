"""Thin ctypes binding of librhosvd.so (include/rhosvd.h).

Argument marshalling only: every step of the RHOSVD path runs in the CUDA
kernels of librhosvd.so.  PyTorch provides device memory, streams and
torch.distributed process groups.  There is no CPU fallback: if the library
or a CUDA device is missing, every call raises.

Layout: U_l are torch.float64 CUDA tensors of shape (R_local, n), contiguous,
i.e. the column-major n x R_local side matrices (ldu = n).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librhosvd.so")

RHOSVD_OK = 0
RHOSVD_FIXED_RANK, RHOSVD_EPS = 0, 1
RHOSVD_F_SIGN_FIX, RHOSVD_F_KEEP_W, RHOSVD_F_ROOT_ONLY_CORE = 1, 2, 4
STATUS = {0: "OK", -1: "EINVAL", -2: "ENONFINITE", -3: "ENOCONV", -4: "ENOMEM",
          -5: "ECUDA", -6: "ENCCL", -7: "EMISMATCH"}
PHASES = ["normalize", "gram", "eigensolve", "rr_refine", "residual_rank", "projection",
          "core", "collectives", "total"]


class Opts(C.Structure):
    _fields_ = [("rank_mode", C.c_int32), ("r", C.c_int32 * 3), ("eps", C.c_double),
                ("oversample", C.c_int32), ("block0", C.c_int32), ("max_iters", C.c_int32),
                ("refine_steps", C.c_int32), ("seed", C.c_uint64), ("flags", C.c_uint32)]


class Report(C.Structure):
    _fields_ = [("trace", C.c_double * 3), ("tail", C.c_double * 3), ("xi_norm", C.c_double),
                ("bound_paper", C.c_double), ("bound_ns", C.c_double), ("beta_norm", C.c_double),
                ("rho", C.c_double * 3), ("ranks", C.c_int32 * 3), ("block", C.c_int32 * 3),
                ("iters", C.c_int32 * 3), ("grow_events", C.c_int32 * 3), ("R_global", C.c_int64),
                ("ms", C.c_double * 16), ("gemm_flops", C.c_double), ("core_ms", C.c_double),
                ("gram_ms", C.c_double), ("launches", C.c_int32), ("refines", C.c_int32 * 3)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_int64, C.c_void_p, C.c_void_p)

_lib = None


class RhosvdError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"rhosvd {STATUS.get(status, status)}: {msg}")
        self.status = status


def lib():
    """Load librhosvd.so (fails loudly: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing - run __graft_entry__.build() "
                           "(python -m paper_2201_12663_b200.build)")
    L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    P, I64, I32, D = C.c_void_p, C.c_int64, C.c_int32, C.c_double
    sig = {
        "rhosvd_opts_default": (None, [C.POINTER(Opts)]),
        "rhosvd_c2t": (C.c_int, [P, P, P, I64, P, I64, I64, C.POINTER(Opts), P, P, C.POINTER(P)]),
        "rhosvd_c2t_host": (C.c_int, [P, P, P, I64, P, I64, I64, C.POINTER(Opts), P, P, C.POINTER(P)]),
        "rhosvd_c2t_als": (C.c_int, [P, P, P, I64, P, I64, I64, C.POINTER(Opts), I32, P, P, C.POINTER(P)]),
        "rhosvd_conv3d": (C.c_int, [C.POINTER(P), I64, P, I64, C.POINTER(P), I64, P, I64, I64, D,
                                    C.POINTER(P), P, P]),
        "rhosvd_result_host_frame": (C.c_int, [P, C.c_int, C.POINTER(P), C.POINTER(I64)]),
        "rhosvd_result_host_sigma": (C.c_int, [P, C.c_int, C.POINTER(P), C.POINTER(I64)]),
        "rhosvd_result_host_core": (C.c_int, [P, C.POINTER(P)]),
        "rhosvd_result_ranks": (C.c_int, [P, C.POINTER(I32)]),
        "rhosvd_result_frame": (C.c_int, [P, C.c_int, C.POINTER(P), C.POINTER(I64)]),
        "rhosvd_result_sigma": (C.c_int, [P, C.c_int, C.POINTER(P), C.POINTER(I64)]),
        "rhosvd_result_core": (C.c_int, [P, C.POINTER(P)]),
        "rhosvd_result_cpfactor": (C.c_int, [P, C.c_int, C.POINTER(P), C.POINTER(I64)]),
        "rhosvd_result_report": (C.c_int, [P, C.POINTER(Report)]),
        "rhosvd_result_free": (None, [P]),
        "rhosvd_last_error": (C.c_char_p, []),
        "rhosvd_version": (C.c_char_p, []),
        "rhosvd_nccl_get_unique_id": (C.c_int, [C.c_char_p]),
        "rhosvd_comm_init_nccl": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.POINTER(P)]),
        "rhosvd_comm_init_callback": (C.c_int, [ALLREDUCE_FN, P, C.c_int, C.c_int, C.POINTER(P)]),
        "rhosvd_comm_destroy": (None, [P]),
        "rhosvd_gram": (C.c_int, [P, I64, I64, I64, P, I64, P]),
        "rhosvd_dgemm": (C.c_int, [C.c_char, C.c_char, I64, I64, I64, D, P, I64, P, I64, D, P, I64, P]),
        "rhosvd_syevj": (C.c_int, [I64, P, I64, P, P, I64, D, C.POINTER(I32), P]),
        "rhosvd_core": (C.c_int, [P, P, P, I64, P, I64, I64, I64, I64, P, P]),
        "rhosvd_chol_inv": (C.c_int, [I64, P, I64, D, P, I64, P]),
        "rhosvd_t2c": (C.c_int, [P, D, P, C.POINTER(P)]),
        "rhosvd_cp_rank": (C.c_int, [P, C.POINTER(I64)]),
        "rhosvd_cp_factor": (C.c_int, [P, C.c_int, C.POINTER(P), C.POINTER(I64)]),
        "rhosvd_cp_core_factor": (C.c_int, [P, C.c_int, C.POINTER(P), C.POINTER(I64)]),
        "rhosvd_cp_weights": (C.c_int, [P, C.POINTER(P), C.POINTER(P)]),
        "rhosvd_cp_info": (C.c_int, [P, C.POINTER(D), C.POINTER(D), C.POINTER(D), C.POINTER(I32)]),
        "rhosvd_cp_free": (None, [P]),
        "rhosvd_sinc_slater": (C.c_int, [D, D, I32, D, P, P, I64, C.POINTER(I64)]),
        "rhosvd_rs_split": (C.c_int, [P, P, I64, P, P, C.POINTER(I64), P, P, C.POINTER(I64)]),
        "rhosvd_rs_lattice": (C.c_int, [P, P, I64, D, I64, P, P, I64, P, P, P, I64, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


EXPORTED = ["rhosvd_opts_default", "rhosvd_c2t", "rhosvd_result_ranks", "rhosvd_result_frame",
            "rhosvd_result_sigma", "rhosvd_result_core", "rhosvd_result_cpfactor",
            "rhosvd_result_report", "rhosvd_result_free", "rhosvd_last_error", "rhosvd_version",
            "rhosvd_nccl_get_unique_id", "rhosvd_comm_init_nccl", "rhosvd_comm_init_callback",
            "rhosvd_comm_destroy", "rhosvd_gram", "rhosvd_dgemm", "rhosvd_syevj", "rhosvd_core",
            "rhosvd_chol_inv", "rhosvd_t2c", "rhosvd_cp_rank", "rhosvd_cp_factor", "rhosvd_cp_core_factor",
            "rhosvd_cp_weights", "rhosvd_cp_info", "rhosvd_cp_free", "rhosvd_c2t_host",
            "rhosvd_result_host_frame", "rhosvd_result_host_sigma", "rhosvd_result_host_core",
            "rhosvd_c2t_als", "rhosvd_conv3d", "rhosvd_sinc_slater", "rhosvd_rs_split", "rhosvd_rs_lattice"]


def _check(status):
    if status != RHOSVD_OK:
        raise RhosvdError(status, lib().rhosvd_last_error().decode())


def _stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None and t.numel() > 0 else C.c_void_p(0)


def _need_cuda_f64(t, name):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64:
        raise TypeError(f"{name} must be a torch.float64 CUDA tensor")


def make_opts(eps=None, ranks=None, oversample=16, block0=0, max_iters=30, refine_steps=1,
              seed=12345, sign_fix=True, root_only_core=False):
    o = Opts()
    lib().rhosvd_opts_default(C.byref(o))
    if (eps is None) == (ranks is None):
        raise ValueError("give exactly one of eps or ranks")
    if eps is not None:
        o.rank_mode = RHOSVD_EPS
        o.eps = float(eps)
    else:
        o.rank_mode = RHOSVD_FIXED_RANK
        for i in range(3):
            o.r[i] = int(ranks[i])
    o.oversample = int(oversample)
    o.block0 = int(block0)
    o.max_iters = int(max_iters)
    o.refine_steps = int(refine_steps)
    o.seed = int(seed)
    o.flags = (RHOSVD_F_SIGN_FIX if sign_fix else 0) | (RHOSVD_F_ROOT_ONLY_CORE if root_only_core else 0)
    return o


# ---------------------------------------------------------------- communicators
class Comm:
    """Wraps rhosvd_comm (NCCL or host-callback all-reduce)."""

    def __init__(self, handle, keep=None, rank=0, world=1):
        self.handle = handle
        self._keep = keep  # keep ctypes callback alive
        self.rank, self.world = rank, world

    def close(self):
        if self.handle:
            lib().rhosvd_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def nccl(group=None):
        """NCCL communicator over the ranks of a torch.distributed group."""
        import torch
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        idbuf = C.create_string_buffer(128)
        if rank == 0:
            _check(lib().rhosvd_nccl_get_unique_id(idbuf))
        t = torch.tensor(list(idbuf.raw), dtype=torch.uint8,
                         device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
        dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        raw = bytes(t.cpu().tolist())
        h = C.c_void_p()
        _check(lib().rhosvd_comm_init_nccl(raw, world, rank, C.byref(h)))
        return Comm(h, rank=rank, world=world)

    @staticmethod
    def callback(group=None):
        """Host-callback communicator: device -> host -> torch.distributed
        all_reduce (gloo) -> device.  For tests of the sharded path."""
        import torch
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)

        def _ar(dptr, count, stream, user):
            try:
                n = int(count)
                nbytes = n * 8
                host = torch.empty(n, dtype=torch.float64)
                cudart = torch.cuda.cudart()
                # synchronous copies on the library's stream (already synchronised)
                _memcpy(host.data_ptr(), C.cast(dptr, C.c_void_p).value, nbytes, 2)
                dist.all_reduce(host, group=group)
                _memcpy(C.cast(dptr, C.c_void_p).value, host.data_ptr(), nbytes, 1)
                del cudart
                return 0
            except Exception:  # pragma: no cover
                import traceback
                traceback.print_exc()
                return 1

        cb = ALLREDUCE_FN(_ar)
        h = C.c_void_p()
        _check(lib().rhosvd_comm_init_callback(cb, None, world, rank, C.byref(h)))
        return Comm(h, keep=cb, rank=rank, world=world)


_cudart = None


def _memcpy(dst, src, nbytes, kind):
    """cudaMemcpy via the CUDA runtime (kind 1 = H2D, 2 = D2H)."""
    global _cudart
    if _cudart is None:
        import ctypes.util
        for nm in ("libcudart.so.12", "libcudart.so"):
            try:
                _cudart = C.CDLL(nm)
                break
            except OSError:
                continue
        if _cudart is None:
            import torch  # noqa: F401  (torch loads its cudart)
            _cudart = C.CDLL("libcudart.so.12")
        _cudart.cudaMemcpy.restype = C.c_int
        _cudart.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
    r = _cudart.cudaMemcpy(C.c_void_p(dst), C.c_void_p(src), C.c_size_t(nbytes), C.c_int(kind))
    if r != 0:
        raise RuntimeError(f"cudaMemcpy failed: {r}")


# ---------------------------------------------------------------- result
@dataclass
class Result:
    ranks: tuple
    Z: list            # torch (n, r_l) float64 CUDA (copies; library memory freed)
    sigma: list        # torch (r_l,)
    beta: object       # torch (r1, r2, r3)
    W: list            # torch (r_l, R_local) CP factors of the core (Prop. 2.1)
    report: dict = field(default_factory=dict)


def _report_dict(rep: Report):
    return dict(
        trace=list(rep.trace), tail=list(rep.tail), xi_norm=rep.xi_norm,
        bound_paper=rep.bound_paper, bound_ns=rep.bound_ns, beta_norm=rep.beta_norm,
        rho=list(rep.rho), ranks=list(rep.ranks), block=list(rep.block), iters=list(rep.iters),
        grow_events=list(rep.grow_events), R_global=rep.R_global,
        ms={PHASES[i]: rep.ms[i] for i in range(len(PHASES))},
        ms_modes_summed={nm: rep.ms[9 + i] for i, nm in
                         enumerate(["eigensolve", "rr_refine", "residual_rank", "projection", "collectives"])},
        gemm_flops=rep.gemm_flops,
        core_ms=rep.core_ms, gram_ms=rep.gram_ms, launches=rep.launches, refines=list(rep.refines))


def c2t_raw(U, xi, opts: Opts, comm: Comm | None = None, stream=None, als_sweeps=None):
    """Call rhosvd_c2t (or rhosvd_c2t_als when als_sweeps is given); returns the raw
    result handle (caller frees)."""
    import torch
    U1, U2, U3 = U
    for i, u in enumerate((U1, U2, U3)):
        _need_cuda_f64(u, f"U{i+1}")
        if not u.is_contiguous():
            raise ValueError("U must be contiguous (R_local, n)")
    _need_cuda_f64(xi, "xi")
    R, n = U1.shape
    if U2.shape != (R, n) or U3.shape != (R, n) or xi.shape != (R,):
        raise ValueError("shape mismatch: U_l (R_local, n), xi (R_local,)")
    h = C.c_void_p()
    st = _stream_ptr(stream)
    with torch.cuda.device(U1.device):
        if als_sweeps is None:
            _check(lib().rhosvd_c2t(_ptr(U1), _ptr(U2), _ptr(U3), n, _ptr(xi), n, R, C.byref(opts),
                                    comm.handle if comm is not None else None, st, C.byref(h)))
        else:
            _check(lib().rhosvd_c2t_als(_ptr(U1), _ptr(U2), _ptr(U3), n, _ptr(xi), n, R, C.byref(opts),
                                        int(als_sweeps), comm.handle if comm is not None else None, st,
                                        C.byref(h)))
    return h


class HostResult:
    """Result of rhosvd_c2t_host: host (pinned, library-owned) outputs viewed as torch CPU
    tensors WITHOUT a copy.  The views are valid until close() (or garbage collection of
    this object); copy what must outlive it."""

    def __init__(self, h, n, ranks, report):
        import numpy as np
        import torch
        self._h = h
        self.ranks = ranks
        self.report = report
        L = lib()

        def view(ptr, count):
            if count == 0 or not ptr:
                return torch.empty(0, dtype=torch.float64)
            arr = np.ctypeslib.as_array((C.c_double * count).from_address(ptr))
            return torch.from_numpy(arr)

        self.Z, self.sigma = [], []
        for l in range(3):
            p, ld = C.c_void_p(), C.c_int64()
            _check(L.rhosvd_result_host_frame(h, l, C.byref(p), C.byref(ld)))
            rl = ranks[l]
            self.Z.append(view(p.value, rl * int(ld.value)).view(rl, int(ld.value))[:, :n].t() if rl
                          else torch.empty(n, 0, dtype=torch.float64))
            sp, cnt = C.c_void_p(), C.c_int64()
            _check(L.rhosvd_result_host_sigma(h, l, C.byref(sp), C.byref(cnt)))
            self.sigma.append(view(sp.value, int(cnt.value)))
        bp = C.c_void_p()
        _check(L.rhosvd_result_host_core(h, C.byref(bp)))
        tot = ranks[0] * ranks[1] * ranks[2]
        self.beta = view(bp.value, tot).view(*ranks) if tot else torch.zeros(*ranks, dtype=torch.float64)

    def close(self):
        if self._h is not None:
            self.Z = self.sigma = self.beta = None
            lib().rhosvd_result_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def c2t_host(U, xi, eps=None, ranks=None, comm: Comm | None = None, stream=None, device=None, **kw):
    """rhosvd_c2t_host: host inputs (torch CPU float64 (R_local, n) contiguous, ideally
    pinned) -> HostResult with host outputs.  H2D / D2H happen inside the call."""
    import torch
    U1, U2, U3 = U
    for i, u in enumerate((U1, U2, U3)):
        if u.device.type != "cpu" or u.dtype != torch.float64 or not u.is_contiguous():
            raise ValueError(f"U{i+1} must be a contiguous float64 CPU tensor (R_local, n)")
    if xi.device.type != "cpu" or xi.dtype != torch.float64 or not xi.is_contiguous():
        raise ValueError("xi must be a contiguous float64 CPU tensor")
    R, n = U1.shape
    if U2.shape != (R, n) or U3.shape != (R, n) or xi.shape != (R,):
        raise ValueError("shape mismatch: U_l (R_local, n), xi (R_local,)")
    opts = make_opts(eps=eps, ranks=ranks, **kw)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    h = C.c_void_p()
    with torch.cuda.device(dev):
        st = _stream_ptr(stream)
        _check(lib().rhosvd_c2t_host(_ptr(U1), _ptr(U2), _ptr(U3), n, _ptr(xi), n, R, C.byref(opts),
                                     comm.handle if comm is not None else None, st, C.byref(h)))
    L = lib()
    r = (C.c_int32 * 3)()
    _check(L.rhosvd_result_ranks(h, r))
    rep = Report()
    _check(L.rhosvd_result_report(h, C.byref(rep)))
    return HostResult(h, n, tuple(int(x) for x in r), _report_dict(rep))


def _wrap_dev(ptr, nelem, device):
    """Copy nelem doubles at a device pointer into a new torch tensor."""
    import torch
    out = torch.empty(nelem, dtype=torch.float64, device=device)
    if nelem > 0:
        # device-to-device copy through the runtime (kind 3)
        _memcpy(out.data_ptr(), ptr, nelem * 8, 3)
    return out


def c2t(U, xi, eps=None, ranks=None, comm: Comm | None = None, stream=None, keep_w=True, als_sweeps=None, **kw):
    """RHOSVD canonical-to-Tucker transform on the GPU (rhosvd_c2t).

    U: (U1, U2, U3) torch.float64 CUDA tensors of shape (R_local, n); xi: (R_local,).
    Returns Result(ranks, Z=[n x r_l], sigma=[r_l], beta=r1 x r2 x r3, W=[r_l x R_local], report).
    """
    import torch
    opts = make_opts(eps=eps, ranks=ranks, **kw)
    h = c2t_raw(U, xi, opts, comm, stream, als_sweeps=als_sweeps)
    L = lib()
    dev = U[0].device
    try:
        torch.cuda.synchronize(dev)
        r = (C.c_int32 * 3)()
        _check(L.rhosvd_result_ranks(h, r))
        ranks_ = tuple(int(x) for x in r)
        n = U[0].shape[1]
        Rl = U[0].shape[0]
        Zs, sig, Ws = [], [], []
        for l in range(3):
            p, ld = C.c_void_p(), C.c_int64()
            _check(L.rhosvd_result_frame(h, l, C.byref(p), C.byref(ld)))
            rl = ranks_[l]
            flat = _wrap_dev(p.value, int(ld.value) * rl, dev) if rl else torch.empty(0, dtype=torch.float64, device=dev)
            Zs.append(flat.view(rl, int(ld.value))[:, :n].t() if rl else torch.empty(n, 0, dtype=torch.float64, device=dev))
            sp, cnt = C.c_void_p(), C.c_int64()
            _check(L.rhosvd_result_sigma(h, l, C.byref(sp), C.byref(cnt)))
            sig.append(_wrap_dev(sp.value, int(cnt.value), dev))
            if keep_w:
                wp, ldw = C.c_void_p(), C.c_int64()
                _check(L.rhosvd_result_cpfactor(h, l, C.byref(wp), C.byref(ldw)))
                wf = _wrap_dev(wp.value, rl * int(ldw.value), dev) if rl else torch.empty(0, dtype=torch.float64, device=dev)
                Ws.append(wf.view(rl, int(ldw.value))[:, :Rl] if rl else torch.empty(0, Rl, dtype=torch.float64, device=dev))
        bp = C.c_void_p()
        tot = ranks_[0] * ranks_[1] * ranks_[2]
        if opts.flags & RHOSVD_F_ROOT_ONLY_CORE and comm is not None and comm.rank != 0:
            beta = None  # reduced to rank 0 only
        else:
            _check(L.rhosvd_result_core(h, C.byref(bp)))
            beta = _wrap_dev(bp.value, tot, dev).view(*ranks_) if tot else torch.zeros(*ranks_, dtype=torch.float64, device=dev)
        rep = Report()
        _check(L.rhosvd_result_report(h, C.byref(rep)))
        return Result(ranks=ranks_, Z=Zs, sigma=sig, beta=beta, W=Ws if keep_w else None,
                      report=_report_dict(rep))
    finally:
        L.rhosvd_result_free(h)


@dataclass
class CPResult:
    """C2C output: A ~ sum_j w_j F1[:, j] (x) F2[:, j] (x) F3[:, j] (unit factor columns)."""
    R: int
    F: list            # torch (n, R) x 3
    w: object          # torch (R,)
    slice_of: object   # torch (R,) int32: mode-3 slice of each term
    U: object          # torch (r1, R) core-space left factors u_j
    V: object          # torch (r2, R) core-space right factors v_j
    eps: float         # absolute eps = eps_rel ||beta||
    thr: float         # singular-value threshold eps / (r3 sqrt(min(r1, r2)))
    err2: float        # ||beta - beta_(R)||^2 (discarded energy)
    sweeps: int        # largest one-sided Jacobi sweep count over the slices
    c2t: Result = None


def c2c(U, xi, t2c_eps, eps=None, ranks=None, comm: Comm | None = None, stream=None, **kw):
    """Canonical-to-canonical rank reduction C2C = T2C o C2T (PAPER.md 2.3, Remark 2.1):
    rhosvd_c2t, then rhosvd_t2c of its core within t2c_eps * ||beta||_F, lifted through
    the frames."""
    import torch
    opts = make_opts(eps=eps, ranks=ranks, **kw)
    L = lib()
    h = c2t_raw(U, xi, opts, comm, stream)
    cp = C.c_void_p()
    dev = U[0].device
    try:
        with torch.cuda.device(dev):
            _check(L.rhosvd_t2c(h, float(t2c_eps), _stream_ptr(stream), C.byref(cp)))
        torch.cuda.synchronize(dev)
        R = C.c_int64()
        _check(L.rhosvd_cp_rank(cp, C.byref(R)))
        R = int(R.value)
        n = U[0].shape[1]
        F = []
        for l in range(3):
            fp, ld = C.c_void_p(), C.c_int64()
            _check(L.rhosvd_cp_factor(cp, l, C.byref(fp), C.byref(ld)))
            F.append(_wrap_dev(fp.value, int(ld.value) * R, dev).view(R, int(ld.value))[:, :n].t() if R
                     else torch.empty(n, 0, dtype=torch.float64, device=dev))
        core = []
        r = (C.c_int32 * 3)()
        _check(L.rhosvd_result_ranks(h, r))
        for l in range(2):
            fp, ld = C.c_void_p(), C.c_int64()
            _check(L.rhosvd_cp_core_factor(cp, l, C.byref(fp), C.byref(ld)))
            rl = int(r[l])
            core.append(_wrap_dev(fp.value, int(ld.value) * R, dev).view(R, int(ld.value))[:, :rl].t() if R
                        else torch.empty(rl, 0, dtype=torch.float64, device=dev))
        wp, sp = C.c_void_p(), C.c_void_p()
        _check(L.rhosvd_cp_weights(cp, C.byref(wp), C.byref(sp)))
        w = _wrap_dev(wp.value, R, dev)
        sl = torch.empty(R, dtype=torch.int32, device=dev)
        if R:
            _memcpy(sl.data_ptr(), sp.value, R * 4, 3)
        e, t, e2, sw = C.c_double(), C.c_double(), C.c_double(), C.c_int32()
        _check(L.rhosvd_cp_info(cp, C.byref(e), C.byref(t), C.byref(e2), C.byref(sw)))
        return CPResult(R=R, F=F, w=w, slice_of=sl, U=core[0], V=core[1], eps=e.value, thr=t.value,
                        err2=e2.value, sweeps=int(sw.value))
    finally:
        if cp.value:
            L.rhosvd_cp_free(cp)
        L.rhosvd_result_free(h)


# ---------------------------------------------------------------- kernel-level calls
def gram(U, stream=None):
    """G = U U^T for a (R, n) contiguous float64 CUDA tensor (column-major n x R)."""
    import torch
    _need_cuda_f64(U, "U")
    R, n = U.shape
    ld = n + (n & 1)
    if ld != n:
        Up = torch.zeros(R, ld, dtype=torch.float64, device=U.device)
        Up[:, :n] = U
        U = Up
    G = torch.empty(n, n, dtype=torch.float64, device=U.device)
    _check(lib().rhosvd_gram(_ptr(U), ld, n, R, _ptr(G), n, _stream_ptr(stream)))
    return G  # symmetric; column-major == row-major


def _even_ld(X):
    """Row-major 2-D tensor with an even, 16-byte aligned leading dimension (zero padded)."""
    import torch
    X = X.contiguous()
    r, c = X.shape
    if c % 2 == 0 and X.data_ptr() % 16 == 0:
        return X, c
    P = torch.zeros(r, c + (c % 2), dtype=X.dtype, device=X.device)
    P[:, :c] = X
    return P, P.shape[1]


def dgemm(A, B, transa=False, transb=False, stream=None):
    """C = op(A) op(B) for torch row-major tensors (mapped onto the col-major ABI:
    row-major C (M x N) is col-major C^T = op(B)^T op(A)^T)."""
    import torch
    _need_cuda_f64(A, "A")
    _need_cuda_f64(B, "B")
    M, K = (A.shape[1], A.shape[0]) if transa else (A.shape[0], A.shape[1])
    K2, N = (B.shape[1], B.shape[0]) if transb else (B.shape[0], B.shape[1])
    assert K == K2
    Ab, lda = _even_ld(A)
    Bb, ldb = _even_ld(B)
    Ct = torch.empty(M, N, dtype=torch.float64, device=A.device)
    # col-major view of a row-major buffer X is X^T: op(B)^T is 'N' on B's buffer unless transb
    ta = b"T" if transb else b"N"
    tb = b"T" if transa else b"N"
    _check(lib().rhosvd_dgemm(ta, tb, N, M, K, 1.0, _ptr(Bb), ldb, _ptr(Ab), lda, 0.0,
                              _ptr(Ct), N, _stream_ptr(stream)))
    return Ct


def syevj(S, tol=1e-15, stream=None):
    """Symmetric Jacobi eigensolver: returns (lambda desc, V, sweeps)."""
    import torch
    _need_cuda_f64(S, "S")
    b = S.shape[0]
    A = S.t().contiguous().clone()  # col-major copy
    lam = torch.empty(b, dtype=torch.float64, device=S.device)
    V = torch.empty(b, b, dtype=torch.float64, device=S.device)
    sw = C.c_int32()
    _check(lib().rhosvd_syevj(b, _ptr(A), b, _ptr(lam), _ptr(V), b, tol, C.byref(sw), _stream_ptr(stream)))
    return lam, V.t(), int(sw.value)  # V col-major -> columns are eigenvectors


def chol_inv(S, shift=0.0, stream=None):
    """Bp = D L^{-T}, D = diag(S)^{-1/2}, L = chol(D S D + shift I) (S symmetric, CUDA f64)."""
    import torch
    _need_cuda_f64(S, "S")
    b = S.shape[0]
    Sc = S.t().contiguous()
    Bp = torch.empty(b, b, dtype=torch.float64, device=S.device)
    _check(lib().rhosvd_chol_inv(b, _ptr(Sc), b, float(shift), _ptr(Bp), b, _stream_ptr(stream)))
    return Bp.t()  # col-major buffer -> row-major view


def core(W1, W2, W3, xi, stream=None):
    """beta[a,b,c] = sum_k xi_k W1[a,k] W2[b,k] W3[c,k] (W_l row-major r_l x R)."""
    import torch
    for t, nm in ((W1, "W1"), (W2, "W2"), (W3, "W3"), (xi, "xi")):
        _need_cuda_f64(t, nm)
    R = W1.shape[1]
    ld = R + (R & 1)

    def pad(W):
        if ld == R and W.is_contiguous():
            return W
        P = torch.zeros(W.shape[0], ld, dtype=torch.float64, device=W.device)
        P[:, :R] = W
        return P
    W1p, W2p, W3p = pad(W1), pad(W2), pad(W3)
    r1, r2, r3 = W1.shape[0], W2.shape[0], W3.shape[0]
    beta = torch.empty(r1, r2, r3, dtype=torch.float64, device=W1.device)
    _check(lib().rhosvd_core(_ptr(W1p), _ptr(W2p), _ptr(W3p), ld, _ptr(xi.contiguous()), r1, r2, r3, R,
                             _ptr(beta), _stream_ptr(stream)))
    return beta


def conv3d(Fa, ca, Fp, cp, h, stream=None):
    """rhosvd_conv3d: tensor-product convolution of two canonical tensors on one n^3 grid.
    Fa: 3 CUDA float64 tensors (Ra, n) (row k = u_k^(l)), ca (Ra,); Fp: 3 tensors (Rp, n),
    cp (Rp,).  Returns (F = 3 tensors (Ra*Rp, n), w (Ra*Rp,)); row m*Rp + q = u_m * p_q."""
    import torch
    Ra, n = Fa[0].shape
    Rp = Fp[0].shape[0]
    for t in list(Fa) + list(Fp) + [ca, cp]:
        _need_cuda_f64(t, "conv3d operand")
    dev = Fa[0].device
    lda = n + (n & 1)
    if lda != n:  # 16-B aligned rows for TMA: pad each density vector with one zero
        Fa = [torch.nn.functional.pad(f, (0, 1)).contiguous() for f in Fa]
    else:
        Fa = [f.contiguous() for f in Fa]
    Fp = [f.contiguous() for f in Fp]
    F = [torch.empty(Ra * Rp, n, dtype=torch.float64, device=dev) for _ in range(3)]
    w = torch.empty(Ra * Rp, dtype=torch.float64, device=dev)
    pa = (C.c_void_p * 3)(*[f.data_ptr() for f in Fa])
    pp = (C.c_void_p * 3)(*[f.data_ptr() for f in Fp])
    po = (C.c_void_p * 3)(*[f.data_ptr() for f in F])
    with torch.cuda.device(dev):
        _check(lib().rhosvd_conv3d(pa, lda, _ptr(ca.contiguous()), Ra, pp, n, _ptr(cp.contiguous()), Rp, n,
                                   float(h), po, _ptr(w), _stream_ptr(stream)))
    return F, w


# ---------------------------------------------------------------- RS long-range front-end (f3)
def sinc_slater(lam, h, M, w_min=0.0):
    """rhosvd_sinc_slater: (tau, w) numpy arrays of the Slater kernel's sinc rule."""
    import numpy as np
    cap = 2 * int(M) + 1
    tau = np.zeros(cap)
    w = np.zeros(cap)
    R = C.c_int64()
    _check(lib().rhosvd_sinc_slater(float(lam), float(h), int(M), float(w_min), tau.ctypes.data_as(C.c_void_p),
                                    w.ctypes.data_as(C.c_void_p), cap, C.byref(R)))
    return tau[:R.value].copy(), w[:R.value].copy()


def rs_split(tau, w):
    """rhosvd_rs_split: ((tau_l, w_l), (tau_s, w_s))."""
    import numpy as np
    tau = np.ascontiguousarray(tau, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    R = tau.shape[0]
    tl, wl, ts, ws = (np.zeros(max(R, 1)) for _ in range(4))
    Rl, Rs = C.c_int64(), C.c_int64()
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    _check(lib().rhosvd_rs_split(P(tau), P(w), R, P(tl), P(wl), C.byref(Rl), P(ts), P(ws), C.byref(Rs)))
    return (tl[:Rl.value].copy(), wl[:Rl.value].copy()), (ts[:Rs.value].copy(), ws[:Rs.value].copy())


def rs_lattice(tau_l, w_l, h, n, node_idx, c, stream=None):
    """rhosvd_rs_lattice: the long-range lattice tensor on the device.

    node_idx: torch.int32 CUDA (N, 3); c: torch.float64 CUDA (N,).  Returns (U1, U2, U3, xi)
    as torch.float64 CUDA tensors, U_l of shape (N R_l, n) (column-major n x R)."""
    import numpy as np
    import torch
    tau_l = np.ascontiguousarray(tau_l, dtype=np.float64)
    w_l = np.ascontiguousarray(w_l, dtype=np.float64)
    if not (node_idx.is_cuda and node_idx.dtype == torch.int32 and node_idx.is_contiguous()):
        raise TypeError("node_idx must be a contiguous torch.int32 CUDA tensor (N, 3)")
    _need_cuda_f64(c, "c")
    N, Rl = int(node_idx.shape[0]), int(tau_l.shape[0])
    dev = c.device
    U = [torch.empty(N * Rl, n, dtype=torch.float64, device=dev) for _ in range(3)]
    xi = torch.empty(N * Rl, dtype=torch.float64, device=dev)
    _check(lib().rhosvd_rs_lattice(tau_l.ctypes.data_as(C.c_void_p), w_l.ctypes.data_as(C.c_void_p), Rl, float(h),
                                   int(n), _ptr(node_idx), _ptr(c), N, _ptr(U[0]), _ptr(U[1]), _ptr(U[2]), int(n),
                                   _ptr(xi), _stream_ptr(stream)))
    return U[0], U[1], U[2], xi
