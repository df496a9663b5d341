/*
 * rhosvd.h - C ABI of the B200-native RHOSVD canonical-to-Tucker (C2T) library
 *            (librhosvd.so, built from paper_2201_12663_b200/csrc for sm_100a).
 *
 * What it computes (arXiv 2201.12663, section 2.1):
 *   Input  : a rank-R canonical tensor (Eq. can_A3)
 *              A = sum_k xi_k u_k^(1) (x) u_k^(2) (x) u_k^(3),
 *            given as three side matrices U_l = [u_1 ... u_R] in R^{n x R}
 *            (Eq. can_A_Tuck) and the weights xi.
 *   Output : the RHOSVD Tucker approximation (Def. 2.1)
 *              A_(r)^0 = beta x_1 Z_1 x_2 Z_2 x_3 Z_3,
 *            Z_l = the r_l dominant left singular vectors of the normalized
 *            side matrix Uhat_l (Eq. svdr), sigma_l the
 *            retained singular values, and the core
 *              beta = xi' x_l (Z_l^T Uhat_l)   (Prop. 2.1),
 *            i.e. beta[a,b,c] = sum_k xi'_k W1[a,k] W2[b,k] W3[c,k].
 *
 * Conventions:
 *   - A2: columns are normalized internally (2-norm per column per mode);
 *     xi'_k = xi_k * prod_l ||u_k^(l)||.  Inputs are never modified.
 *   - A3: a zero column stays zero and gets xi'_k = 0.
 *   - A1: eps mode selects r_l = min{ r >= 1 : sum_{k>r} sigma_{l,k}^2
 *     <= eps^2 * T_l }, T_l = ||Uhat_l||_F^2.  The GPU evaluates the tail as
 *     sum_{r<k<=b} sigma_k^2 + ||Uhat_l - Z_b W_b||_F^2 (direct residual).
 *   - A17: fixed mode clamps r_l to min(n, R_global).
 *   - A9: frame columns are sign-fixed (largest-|.| entry positive, lowest
 *     row index on ties) when RHOSVD_F_SIGN_FIX is set (default).
 *   - FP64 (IEEE binary64) throughout.
 *
 * Memory: every array pointer is a CUDA DEVICE pointer unless the comment
 * says "host".  All matrices are column-major:
 *   U_l : n x R_local, leading dimension ldu >= n (column k = u_k^(l)
 *         contiguous) == a C-contiguous (R_local, n) row-major array.
 *   xi  : R_local doubles.
 *
 * Errors: every entry point returns an rhosvd_status (0 = OK).  On error the
 * *out handle is set to NULL and rhosvd_last_error() (thread-local) holds a
 * message.  In multi-rank mode every rank returns the same status.
 *
 * Thread safety: calls on different streams/handles may be made concurrently
 * from several threads; the library serialises them (host side by a mutex,
 * device side by making each call's stream wait for the previous call's work,
 * since workspaces are process-wide).  One rhosvd_comm must not be used by two
 * calls at once.
 *
 * Devices: one CUDA device per process.  The first call pins the current device
 * (workspaces, output caches and kernel attributes are process-wide); a call made
 * while another device is current returns RHOSVD_EINVAL.
 */
#ifndef RHOSVD_H_
#define RHOSVD_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RHOSVD_OK = 0,
  RHOSVD_EINVAL = -1,      /* bad argument (null pointer, n < 1, R_local < 0, ldu < n, eps not in (0,1), r < 1) */
  RHOSVD_ENONFINITE = -2,  /* NaN/Inf in U or xi (detected by the normalisation kernel) */
  RHOSVD_ENOCONV = -3,     /* no convergence: the subspace iteration stopped at max_iters
                              short of its modelled count (sin theta_r ~ rho^(iters + refine)
                              > 1e-7, rho = block-edge Rayleigh quotient / r-th), the eps rank
                              rule was not met inside the final block (A1),
                              or a small dense Jacobi solve did not converge.  Never a silently
                              truncated rank. */
  RHOSVD_ENOMEM = -4,      /* device allocation failed */
  RHOSVD_ECUDA = -5,       /* CUDA runtime error */
  RHOSVD_ENCCL = -6,       /* collective failed */
  RHOSVD_EMISMATCH = -7    /* ranks disagree on n / options */
} rhosvd_status;

enum { RHOSVD_FIXED_RANK = 0, RHOSVD_EPS = 1 };
/* Flags.  SIGN_FIX: canonical frame signs (A9).  KEEP_W: the CP factors W_l of the core
 * are kept in the result (always the case in this build; the flag is accepted for ABI
 * compatibility).  ROOT_ONLY_CORE (multi-rank only): the core's sum over the R shards is
 * reduced to rank 0 (ncclReduce) instead of all-reduced; on the other ranks
 * rhosvd_result_core / rhosvd_result_host_core / rhosvd_t2c return EINVAL and
 * report.beta_norm is NaN.  Frames, sigma and ranks stay replicated. */
enum { RHOSVD_F_SIGN_FIX = 1u, RHOSVD_F_KEEP_W = 2u, RHOSVD_F_ROOT_ONLY_CORE = 4u };

/* Options.  Initialise with rhosvd_opts_default(). */
typedef struct {
  int32_t  rank_mode;    /* RHOSVD_FIXED_RANK or RHOSVD_EPS                                  */
  int32_t  r[3];         /* fixed mode: requested r_l >= 1 (clamped to min(n, R_global))      */
  double   eps;          /* eps mode: 0 < eps < 1, relative Frobenius tail per mode (A1)     */
  int32_t  oversample;   /* p: block size b = r + p (default 16)                             */
  int32_t  block0;       /* eps mode: first block size (0 = default 128); grows adaptively    */
  int32_t  max_iters;    /* subspace-iteration cap per block size (default 30)               */
  int32_t  refine_steps; /* non-squared refinement steps (default 1)                         */
  uint64_t seed;         /* start-block seed                                                 */
  uint32_t flags;        /* default RHOSVD_F_SIGN_FIX                                        */
} rhosvd_opts;

/* Per-call report (host struct).  ms[] holds per-phase device times:
 *   0 normalize, 1 gram, 2 eigensolve (subspace iteration), 3 one-sided RR +
 *   refinement, 4 residual + rank, 5 projection W_r, 6 core, 7 collectives,
 *   8 total (all in milliseconds, CUDA events on the call's stream).  When the three
 *   per-mode eigensolves run concurrently (one GPU), ms[2] is the wall time of that
 *   region and ms[9..13] hold the per-mode device times summed over the modes
 *   (eigensolve, RR + refinement, residual + rank, projection, collectives). */
typedef struct {
  double  trace[3];      /* T_l = ||Uhat_l||_F^2                                   */
  double  tail[3];       /* (sum_{k>r_l} sigma_{l,k}^2)^{1/2} (direct residual form) */
  double  xi_norm;       /* ||xi'||                                                */
  double  bound_paper;   /* ||xi'|| sum_l tail_l           (Thm. 2.2) */
  double  bound_ns;      /* ||xi'|| (sum_l tail_l^2)^{1/2} (reading A12)           */
  double  beta_norm;     /* ||beta||_F                                             */
  double  rho[3];        /* ||Uhat_l - Z_b W_b||_F^2 (out-of-block energy)         */
  int32_t ranks[3];
  int32_t block[3];      /* final block size b_l                                   */
  int32_t iters[3];      /* subspace iterations                                    */
  int32_t grow_events[3];
  int64_t R_global;
  double  ms[16];
  double  gemm_flops;    /* executed DMMA flops (all GEMM-type kernels)            */
  double  core_ms;       /* device time of the core kernel(s) alone                */
  double  gram_ms;       /* device time of the Gram kernel(s) alone                */
  int32_t launches;      /* kernels launched by this call                          */
  int32_t refines[3];    /* non-squared refinement steps per mode                  */
} rhosvd_report;

typedef struct rhosvd_comm rhosvd_comm;       /* NULL => single GPU                */
typedef struct rhosvd_result rhosvd_result;   /* opaque; owns all device outputs   */
typedef void* rhosvd_stream;                  /* a cudaStream_t (NULL = legacy)    */

/* Host-side all-reduce callback (sum, fp64) for rhosvd_comm_init_callback:
 * must leave the element-wise sum over all ranks in `dptr` (device pointer,
 * `count` doubles) when it returns; work queued on `stream` before the call
 * is complete when the library invokes it.  Returns 0 on success. */
typedef int (*rhosvd_allreduce_fn)(double* dptr, int64_t count, rhosvd_stream stream, void* user);

void rhosvd_opts_default(rhosvd_opts* o);                                   /* host */

/* Multi-GPU (R-sharded).  NCCL communicator from a unique id
 * (128 host bytes) created on rank 0 and broadcast by the caller. */
int  rhosvd_nccl_get_unique_id(uint8_t id[128]);                            /* host */
int  rhosvd_comm_init_nccl(const uint8_t id[128], int world, int rank, rhosvd_comm** out);
/* Host-callback communicator (e.g. torch.distributed gloo); used by tests. */
int  rhosvd_comm_init_callback(rhosvd_allreduce_fn fn, void* user, int world, int rank,
                               rhosvd_comm** out);
void rhosvd_comm_destroy(rhosvd_comm* c);

/* The product entry point: RHOSVD C2T of the local column block.
 *   U1,U2,U3 : device, n x R_local column-major, leading dimension ldu >= n
 *   xi       : device, R_local weights
 *   comm     : NULL for one GPU; otherwise every rank calls collectively with
 *              the same n and opts and its own contiguous column block
 *   stream   : cudaStream_t the work is ordered on
 *   out      : receives a result handle (free with rhosvd_result_free)
 * Blocks the host until the result is complete (ranks size the outputs). */
int  rhosvd_c2t(const double* U1, const double* U2, const double* U3, int64_t ldu,
                const double* xi, int64_t n, int64_t R_local, const rhosvd_opts* opts,
                rhosvd_comm* comm, rhosvd_stream stream, rhosvd_result** out);

/* The same with HOST buffers (the end-to-end entry point bench.py's "e2e" times).
 *   U1,U2,U3 : host, n x R_local column-major (ld ldu; elements (R_local-1) ldu + n are
 *              read); xi : host, R_local.  Pinned memory (cudaHostAlloc / torch
 *              pin_memory) gives full PCIe bandwidth; pageable memory works, slower.
 *              The buffers must stay valid until the call returns (it never writes them).
 *   Inputs go H2D on a library copy stream, one side matrix at a time, and mode l's
 *   normalize + Gram start as soon as U_l has arrived.  Outputs (frames, sigma, core)
 *   are copied back into library-owned pinned host buffers while the core contraction
 *   still runs (single GPU: beta row chunk by row chunk), read with the
 *   rhosvd_result_host_* accessors below; the device accessors stay valid too.
 *   Errors, collectives, blocking and ownership as rhosvd_c2t. */
int  rhosvd_c2t_host(const double* U1, const double* U2, const double* U3, int64_t ldu,
                     const double* xi, int64_t n, int64_t R_local, const rhosvd_opts* opts,
                     rhosvd_comm* comm, rhosvd_stream stream, rhosvd_result** out);
/* Host copies (owned by the handle; EINVAL for a result of rhosvd_c2t). */
int  rhosvd_result_host_frame(const rhosvd_result* res, int mode, const double** Z, int64_t* ldz);
int  rhosvd_result_host_sigma(const rhosvd_result* res, int mode, const double** s, int64_t* count);
int  rhosvd_result_host_core (const rhosvd_result* res, const double** beta);

/* C2T followed by `sweeps` ALS sweeps on the frames (PAPER.md:336-366,
 * Eq. can_A_Tuck_als, Fig. 2: "only one or two ALS iterations are required").  Per sweep,
 * for l = 1, 2, 3: Z_l <- the r_l dominant left singular vectors of the mode-l unfolding
 * of A x_b Z_b^T x_c Z_c^T (the other modes' current frames), computed from its Gram
 * Uhat_l D [(W_b^T W_b) o (W_c^T W_c)] D Uhat_l^T (D = diag(xi'), W_m = Z_m^T Uhat_m; the
 * R x R middle factor in column blocks, never stored whole).  The ranks are those of the
 * RHOSVD start; the result's frames, CP factors and core are the ALS ones, sigma_l the
 * singular values of the last mode-l unfolding.  sweeps = 0 is rhosvd_c2t.  Cost per
 * mode ~ 2 n R^2 + 4 R^2 r FLOP (cfg 4: ~1.6e13).  Single GPU: comm must be NULL (EINVAL
 * otherwise); sweeps < 0: EINVAL.  Other arguments, errors and ownership as rhosvd_c2t. */
int  rhosvd_c2t_als(const double* U1, const double* U2, const double* U3, int64_t ldu,
                    const double* xi, int64_t n, int64_t R_local, const rhosvd_opts* opts,
                    int32_t sweeps, rhosvd_comm* comm, rhosvd_stream stream, rhosvd_result** out);

/* Result accessors (device pointers stay owned by the handle). */
int  rhosvd_result_ranks   (const rhosvd_result* res, int32_t r[3]);               /* host out */
int  rhosvd_result_frame   (const rhosvd_result* res, int mode, const double** Z, int64_t* ldz); /* n x r_l col-major */
int  rhosvd_result_sigma   (const rhosvd_result* res, int mode, const double** s, int64_t* count); /* r_l values, descending */
int  rhosvd_result_core    (const rhosvd_result* res, const double** beta);        /* r1 x r2 x r3, C order */
int  rhosvd_result_cpfactor(const rhosvd_result* res, int mode, const double** W, int64_t* ldw); /* r_l x R_local row-major (KEEP_W) */
int  rhosvd_result_report  (const rhosvd_result* res, rhosvd_report* host_out);
void rhosvd_result_free    (rhosvd_result* res);
const char* rhosvd_last_error(void);
const char* rhosvd_version(void);

/* ---- Tucker-to-canonical (T2C) and canonical-to-canonical (C2C) rank reduction ----
 * (Remark 2.1.)  The core beta of `res` is split
 * into its r3 mode-3 slices B_m (r1 x r2); each is replaced by its truncated SVD keeping
 * the singular values > thr = eps / (r3 sqrt(min(r1, r2)))  (eps / r^{3/2} for a cubic
 * core), eps = eps_rel ||beta||_F, so that ||beta - beta_(R)||_F <= eps with
 * R = p_1 + ... + p_r3 <= r3 min(r1, r2).  The result is lifted through the frames:
 *   A ~ sum_j w_j F1[:, j] (x) F2[:, j] (x) F3[:, j],
 *   F1 = Z1 u_j, F2 = Z2 v_j, F3 = Z3 e_{slice_j}   (unit columns, w_j = sigma_j).
 * Signs: the largest-|.| entry of u_j is positive.  The slices are processed in shared
 * memory (one CTA each): r1 (r2 + 1) must stay below ~27 000 doubles, else EINVAL.
 * All output pointers are device pointers owned by the rhosvd_cp handle. */
typedef struct rhosvd_cp rhosvd_cp;
int  rhosvd_t2c(const rhosvd_result* res, double eps_rel, rhosvd_stream stream, rhosvd_cp** out);
int  rhosvd_cp_rank(const rhosvd_cp* cp, int64_t* R);                                /* host out */
int  rhosvd_cp_factor(const rhosvd_cp* cp, int mode, const double** F, int64_t* ld);  /* n x R col-major */
int  rhosvd_cp_core_factor(const rhosvd_cp* cp, int mode, const double** F, int64_t* ld); /* mode 0: u (r1 x R), 1: v (r2 x R) */
int  rhosvd_cp_weights(const rhosvd_cp* cp, const double** w, const int32_t** slice);   /* R each */
int  rhosvd_cp_info(const rhosvd_cp* cp, double* eps_abs, double* thr, double* err2,
                    int32_t* max_sweeps);                                          /* host out */
void rhosvd_cp_free(rhosvd_cp* cp);

/* ---- 3-D tensor-product convolution of canonical tensors ----
 * Theta' * P = sum_m sum_q c_m w_q (u_m^(1) * p_q^(1)) (x) (u_m^(2) * p_q^(2))
 * (x) (u_m^(3) * p_q^(3)), "a sum of tensor products of 1D convolutions".  1-D convolution
 * (reading C1): (u * p)_i = h sum_j u_j p_{i + floor(n/2) - j}, p_k = 0 outside
 * [0, n) - the Riemann sum of the continuous convolution on the common grid, central n
 * samples.  All pointers device, column-major factors:
 *   Fa[l] : n x Ra (ld lda, even), ca : Ra   - the density (e.g. the C2C output)
 *   Fp[l] : n x Rp (ld ldp),       cp : Rp   - the kernel
 *   Fout[l] : n x Ra*Rp (ld n), column m*Rp + q = u_m^(l) * p_q^(l); wout : Ra*Rp = c_m w_q
 * (caller-allocated).  Runs as one DMMA GEMM per mode against the stacked Toeplitz
 * matrices of the kernel vectors (2 n^2 Ra Rp FLOP per mode).  EINVAL on null pointers,
 * n < 1, ld < n, odd lda. */
int  rhosvd_conv3d(const double* const Fa[3], int64_t lda, const double* ca, int64_t Ra,
                   const double* const Fp[3], int64_t ldp, const double* cp, int64_t Rp, int64_t n,
                   double h, double* const Fout[3], double* wout, rhosvd_stream stream);

/* ---- range-separated (RS) long-range front-end (section 4) ----
 * The long-range part of a lattice sum of Slater kernels G_{N,l} = sum_j c_j W_j G_l
 * (Eq. Slater_interp_multi) as a canonical tensor for rhosvd_c2t; its
 * Tucker rank grows only as log^{3/2} log(N / eps) (Prop. 4.2).
 *
 * rhosvd_sinc_slater (host arrays): the sinc rule of the Slater kernel's Laplace transform
 *   e^{-lambda sqrt(rho)} = sqrt(alpha/pi) int_0^inf tau^{-3/2} e^{-alpha/tau - rho tau} dtau,
 *   alpha = lambda^2 / 4, trapezoid in s = ln tau with nodes s_k = k h,
 *   |k| <= M:  w_k = h sqrt(alpha/pi) e^{-s_k/2} e^{-alpha e^{-s_k}},  tau_k = e^{s_k}; terms
 *   with w_k < w_min are dropped (reading RS1).  Writes R <= 2M + 1 terms (increasing tau)
 *   into tau[], w[] (capacity cap, else EINVAL).  G(x) ~ sum_k w_k prod_l e^{-tau_k x_l^2}.
 * rhosvd_rs_split (host arrays): K_l = {k : t_k <= 1}, K_s = {k : t_k > 1}, t_k = sqrt(tau_k)
 *   (Eq. RS_repres); copies the long / short terms in order.  Any of
 *   tau_l, w_l, tau_s, w_s may be NULL (counts only).
 * rhosvd_rs_lattice (device outputs): the long-range lattice tensor by shift-and-windowing
 *   (reading RS3): the reference vectors g_k[o] = e^{-tau_k (o h)^2}, o = -(n-1)..(n-1) (the
 *   doubled grid), are windowed at each node's grid index m_{j,l} (node_idx: device int32,
 *   N x 3 row-major; indices in [0, n) - others read zeros outside the table):
 *     column j R_l + k of U_l (n rows, ld ldu >= n):  U_l[i] = g_k[i - m_{j,l}],
 *     xi[j R_l + k] = c_j w_k   (c: device, N amplitudes).
 *   tau_l, w_l: host, R_l <= 128 terms.  U1..U3 / xi: caller-allocated device buffers of
 *   N R_l columns.  Runs on `stream` (two kernels).  EINVAL on bad sizes / null pointers. */
int rhosvd_sinc_slater(double lambda, double h, int32_t M, double w_min, double* tau, double* w,
                       int64_t cap, int64_t* R);
int rhosvd_rs_split(const double* tau, const double* w, int64_t R, double* tau_l, double* w_l,
                    int64_t* R_l, double* tau_s, double* w_s, int64_t* R_s);
int rhosvd_rs_lattice(const double* tau_l, const double* w_l, int64_t R_l, double h, int64_t n,
                      const int32_t* node_idx, const double* c, int64_t N, double* U1, double* U2,
                      double* U3, int64_t ldu, double* xi, rhosvd_stream stream);

/* ---- kernel-level entry points (used by the parity unit tests and bench) ----
 * Each runs ONE device kernel family on `stream`, all pointers device.     */

/* K1 Gram: G = Uhat Uhat^T (n x n, col-major, ldg) for Uhat n x R (ld ldu).
 * Full symmetric output. (SVD of the side matrices.) */
int rhosvd_gram(const double* U, int64_t ldu, int64_t n, int64_t R,
                double* G, int64_t ldg, rhosvd_stream stream);

/* Generic DMMA GEMM (col-major): C = alpha * op(A) op(B) + beta * C,
 * op(X) = X or X^T selected by transa/transb ('N'/'T'). M x N x K. */
int rhosvd_dgemm(char transa, char transb, int64_t M, int64_t N, int64_t K, double alpha,
                 const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                 double* C, int64_t ldc, rhosvd_stream stream);

/* Symmetric Jacobi eigensolver (b x b, col-major lda): on return A's diagonal
 * is overwritten, lambda (b) holds the eigenvalues in descending order and V
 * (b x b, ldv) the eigenvectors.  High relative accuracy for scaled-diagonally
 * dominant positive definite input (stopping rule |a_pq| <= tol sqrt(a_pp a_qq)). */
int rhosvd_syevj(int64_t b, double* A, int64_t lda, double* lambda, double* V, int64_t ldv,
                 double tol, int32_t* sweeps_out, rhosvd_stream stream);

/* Scaled Cholesky inverse (the CholeskyQR building block):
 * Bp (b x b, ldb) = D L^{-T} with D = diag(S)^{-1/2}, L = chol(D S D + shift I),
 * S (b x b, lds) symmetric positive semi-definite.  Q = M Bp then has orthonormal
 * columns for M^T M = S.  Numerically dependent columns (pivot < 1e-13) get a unit
 * pivot and a zero sub-column.  All pointers device. */
int rhosvd_chol_inv(int64_t b, const double* S, int64_t lds, double shift, double* Bp, int64_t ldb,
                    rhosvd_stream stream);

/* Core: beta[a,b,c] = sum_k xi[k] W1[a,k] W2[b,k] W3[c,k]; W_l row-major
 * r_l x R with leading dimension ldw; beta C order.  (Prop. 2.1.) */
int rhosvd_core(const double* W1, const double* W2, const double* W3, int64_t ldw,
                const double* xi, int64_t r1, int64_t r2, int64_t r3, int64_t R,
                double* beta, rhosvd_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* RHOSVD_H_ */
