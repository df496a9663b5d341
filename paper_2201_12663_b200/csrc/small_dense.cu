// small_dense.cu - the b x b kernels of the RHOSVD eigensolver on sm_100a.
//
//  * syevj: two-sided Jacobi - a single-CTA shared-memory kernel for small b and a
//    cooperative block Jacobi (see below) otherwise.  Stopping rule
//    |a_pq| <= tol sqrt(|a_pp a_qq|) (Demmel-Veselic relative criterion) gives
//    eigenvalues of scaled-diagonally-dominant positive definite matrices to high
//    relative accuracy - which is what the one-sided Rayleigh-Ritz on W W^T needs
//    (DESIGN.md).
//  * chol_inv_scaled: column-scaled (optionally shifted) Cholesky of a b x b Gram and
//    the inverse of its factor as one cooperative blocked kernel (see below); the
//    output D L^{-T} turns M into Q = M D L^{-T} (CholeskyQR).
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

#include "small_dense.cuh"

namespace rhosvd {

// ------------------------------------------------------------------ grid barrier
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  // cooperative-groups grid sync (the kernels are launched cooperatively); `bar` is kept in
  // the signature for the callers and is unused
  (void)bar;
  cooperative_groups::this_grid().sync();
}

// round-robin tournament position pos at step (0 <= step < m - 1, 0 <= pos < m): position 0
// fixed, the others rotate.  pos - 1 + step < 2 (m - 1), so one conditional subtraction
// replaces the modulo (an integer division).
__device__ __forceinline__ int rr_index(int pos, int step, int m) {
  if (pos == 0) return 0;
  int x = pos - 1 + step;
  if (x >= m - 1) x -= m - 1;
  return 1 + x;
}

// ------------------------------------------------------------------ Jacobi
struct JacParams {
  int b, m, h;
  const double* Ain;
  int64_t lda;
  double* A0;
  double* A1;
  int64_t ld;
  double* V;
  double* lam;  // unsorted eigenvalues out
  double tol, abstol;  // abstol relative to max |a_ii| of the input
  int max_sweeps;
  unsigned* bar;
  int* info;
};

// Single-CTA variant for b <= 160: A lives in shared memory and is updated in
// place (each 2x2 block (P,Q), P <= Q, is read and written by one thread, its
// mirror (Q,P) by the same thread), so a step costs two __syncthreads.
constexpr int JAC_SMEM_MAXB = 160;
__device__ __forceinline__ int64_t cdiv_d(int64_t a, int64_t b) { return (a + b - 1) / b; }
__global__ void __launch_bounds__(1024) jacobi_smem_kernel(JacParams p) {
  extern __shared__ double sh[];
  const int h = p.h, b = p.b, m = p.m;
  const int lds = b | 1;  // odd pitch
  double* A = sh;
  double* c_ = A + (size_t)b * lds;
  double* s_ = c_ + h;
  double* t_ = s_ + h;
  int* act_ = reinterpret_cast<int*>(t_ + h);
  int* pp_ = act_ + h;
  int* qq_ = pp_ + h;
  __shared__ int red[32];
  __shared__ double sdmax[32];
  const int tid = threadIdx.x, nth = blockDim.x;
  const int64_t ld = p.ld;
  for (int e = tid; e < b * b; e += nth) {
    int i = e % b, j = e / b;
    A[j * lds + i] = p.Ain[(int64_t)j * p.lda + i];
    p.V[j * ld + i] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  {
    double dm = 0.0;
    for (int i = tid; i < b; i += nth) dm = fmax(dm, fabs(A[i * lds + i]));
    for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    if ((tid & 31) == 0) sdmax[tid >> 5] = dm;
    __syncthreads();
    dm = 0.0;
    for (int w = 0; w < (nth >> 5); ++w) dm = fmax(dm, sdmax[w]);
    __syncthreads();
    if (tid == 0) sdmax[0] = dm;
    __syncthreads();
  }
  const double abstol = p.abstol * sdmax[0];
  const int nblk = h * (h + 1) / 2;
  const int items = nblk + b * h;
  int sweeps = 0;
  bool converged = false;
  for (int sw = 0; sw < p.max_sweeps; ++sw) {
    int mycount = 0;
    for (int step = 0; step < m - 1; ++step) {
      for (int k = tid; k < h; k += nth) {
        int i1 = rr_index(k, step, m), i2 = rr_index(m - 1 - k, step, m);
        int pq = min(i1, i2), qq = max(i1, i2);
        pp_[k] = pq;
        qq_[k] = qq;
        double c = 1.0, s = 0.0, t = 0.0;
        int act = 0;
        if (qq < b) {
          double app = A[pq * lds + pq], aqq = A[qq * lds + qq], apq = A[qq * lds + pq];
          double thr = fmax(abstol, p.tol * sqrt(fabs(app * aqq)));
          if (fabs(apq) > thr) {
            act = 1;
            double theta = (aqq - app) / (2.0 * apq);
            if (fabs(theta) > 1e150)
              t = 0.5 / theta;
            else
              t = copysign(1.0 / (fabs(theta) + sqrt(1.0 + theta * theta)), theta);
            if (theta == 0.0) t = 1.0;
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
          }
        }
        c_[k] = c; s_[k] = s; t_[k] = t; act_[k] = act;
        mycount += act;
      }
      __syncthreads();
      for (int it = tid; it < items; it += nth) {
        if (it < nblk) {
          int Q = (int)((sqrtf(8.0f * (float)it + 1.0f) - 1.0f) * 0.5f);
          while ((Q + 1) * (Q + 2) / 2 <= it) ++Q;
          while (Q * (Q + 1) / 2 > it) --Q;
          int P = it - Q * (Q + 1) / 2;
          int p1 = pp_[P], q1 = qq_[P];
          if (!act_[P] && !act_[Q]) continue;  // identity rotation on both sides
          if (P == Q) {
            double app = A[p1 * lds + p1], aqq = A[q1 * lds + q1], apq = A[q1 * lds + p1];
            double t = t_[P];
            A[p1 * lds + p1] = app - t * apq;
            A[q1 * lds + q1] = aqq + t * apq;
            A[q1 * lds + p1] = 0.0;
            A[p1 * lds + q1] = 0.0;
          } else {
            int p2 = pp_[Q], q2 = qq_[Q];
            bool vq1 = q1 < b, vq2 = q2 < b;
            double a11 = A[p2 * lds + p1];
            double a12 = vq2 ? A[q2 * lds + p1] : 0.0;
            double a21 = vq1 ? A[p2 * lds + q1] : 0.0;
            double a22 = (vq1 && vq2) ? A[q2 * lds + q1] : 0.0;
            double c1 = c_[P], s1 = s_[P], c2 = c_[Q], s2 = s_[Q];
            double b11 = c2 * a11 - s2 * a12, b12 = s2 * a11 + c2 * a12;
            double b21 = c2 * a21 - s2 * a22, b22 = s2 * a21 + c2 * a22;
            double n11 = c1 * b11 - s1 * b21, n21 = s1 * b11 + c1 * b21;
            double n12 = c1 * b12 - s1 * b22, n22 = s1 * b12 + c1 * b22;
            A[p2 * lds + p1] = n11; A[p1 * lds + p2] = n11;
            if (vq2) { A[q2 * lds + p1] = n12; A[p1 * lds + q2] = n12; }
            if (vq1) { A[p2 * lds + q1] = n21; A[q1 * lds + p2] = n21; }
            if (vq1 && vq2) { A[q2 * lds + q1] = n22; A[q1 * lds + q2] = n22; }
          }
        } else {
          int j = it - nblk;
          int i = j % b, P = j / b;
          if (act_[P]) {
            int pc = pp_[P], qc = qq_[P];
            double vp = p.V[pc * ld + i], vq = p.V[qc * ld + i];
            double c = c_[P], s = s_[P];
            p.V[pc * ld + i] = c * vp - s * vq;
            p.V[qc * ld + i] = s * vp + c * vq;
          }
        }
      }
      __syncthreads();
    }
    ++sweeps;
    int v = mycount;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    int tot = 0;
    for (int w = 0; w < (nth >> 5); ++w) tot += red[w];
    __syncthreads();
    if (tot == 0) {
      converged = true;
      break;
    }
  }
  for (int i = tid; i < b; i += nth) p.lam[i] = A[i * lds + i];
  if (tid == 0) {
    p.info[0] = sweeps;
    p.info[2] = converged ? 0 : 1;
  }
}

// ------------------------------------------------------------------ block Jacobi
// Two-sided block Jacobi for b > JAC_SMEM_MAXB.  The b x b matrix is padded to
// bp = m * BJ_W (m even; padded rows/columns are zero and never rotate) and split
// into m blocks of BJ_W = 16.  A sweep is m-1 rounds of the round-robin tournament
// over blocks; in a round the m/2 disjoint block pairs are processed in parallel:
//   phase 1  one CTA per pair diagonalises the 32 x 32 sub-matrix A[I u J, I u J] in
//            shared memory with cyclic two-sided Jacobi (relative stopping rule),
//            accumulating Q_k; it writes Q_k and the rotated diagonal block;
//   phase 2  every off-diagonal pair block A'[k, l] = Q_k^T A[k, l] Q_l (in place; the
//            blocks of two unrotated pairs are skipped) and V[:, l] <- V[:, l] Q_l,
//            spread over the whole grid.
// Two grid barriers per round instead of one per rotation step.  Plane rotations
// inside the pairs keep the relative accuracy of graded (scaled diagonally dominant)
// matrices; the off-pair blocks see only orthogonal transformations.
constexpr int BJ_W = 16, BJ_P = 32, BJ_LD = 33, BJ_VT = 64, BJ_THREADS = 288;
struct BJParams {
  int b, bp, m, h;
  const double* Ain;
  int64_t lda;
  double* A0;
  double* A1;
  int64_t ld;
  double* V;
  double* Qb;   // h x 32 x 32, Q_k[p][l] at Qb[k*1024 + p*32 + l]
  int* rotf;    // h flags: pair k rotated this round
  double* lam;
  double tol, abstol;
  int max_sweeps, inner_sweeps;
  int band_d, band_max;
  int select;  // mark-driven selective sweeps (RHOSVD_JAC_SELECT=0: every step of every sweep)  // banded pre-phase: block distance D (0: off), at most band_max band sweeps
  unsigned* bar;
  int* cnt;     // [0, 120) rotations per sweep, [120, 128) per band sweep, [128, 256) tests
  int* info;
  unsigned long long* ts;  // optional: [0] phase 1, [1] barrier 1, [2] phase 2, [3] barrier 2 (ns, CTA 0)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int bj_g(int l, int I, int J) { return l < BJ_W ? I * BJ_W + l : J * BJ_W + (l - BJ_W); }
// Band round (d, par) of the banded pre-phase: block i with (i / d) % 2 == par and
// i + d < m pairs with i + d (these pairs are disjoint: i + d has the other parity); the
// blocks left over pair with each other in increasing order.  Pair k of the round.
__device__ __forceinline__ void bj_band_pair(int k, int d, int par, int m, int& I, int& J) {
  int cnt = 0;
  for (int i = 0; i + d < m; ++i)
    if (((i / d) & 1) == par) {
      if (cnt == k) {
        I = i;
        J = i + d;
        return;
      }
      ++cnt;
    }
  int first = -1;
  for (int i = 0; i < m; ++i) {
    const bool left = ((i / d) & 1) == par && i + d < m, right = i >= d && (((i - d) / d) & 1) == par;
    if (left || right) continue;
    if (first < 0) {
      first = i;
    } else {
      if (cnt == k) {
        I = first;
        J = i;
        return;
      }
      ++cnt;
      first = -1;
    }
  }
  I = 0;
  J = 1;  // not reached: k < m / 2
}
// pairing of schedule step stp: stp >= 0 the round-robin step, stp < 0 band round
// (d, par) with -1 - stp = 2 (d - 1) + par
__device__ __forceinline__ void bj_pair(int k, int stp, int m, int& I, int& J) {
  if (stp < 0) {
    const int code = -1 - stp;
    bj_band_pair(k, code / 2 + 1, code & 1, m, I, J);
    return;
  }
  int i1 = rr_index(k, stp, m), i2 = rr_index(m - 1 - k, stp, m);
  I = min(i1, i2);
  J = max(i1, i2);
}

// ---- inner (pair-block) Jacobi helpers
// S swizzle: column c of a 32-wide row at c ^ 15 (c >= 16) - for every step of the xor
// ordering the 16 lower (or upper) indices of the pairs land in 16 distinct double banks
__device__ __forceinline__ int jb_swz(int c) { return c ^ ((c >> 4) * 15); }
__device__ __forceinline__ int jb_hbit(int m) { return 1 << (31 - __clz(m)); }
// the k-th (0..15) index with bit hb clear = the lower element of pair k at a step with
// highest bit hb; jb_pairof inverts it for either element of the pair
__device__ __forceinline__ int jb_lower(int k, int hb) { return ((k & ~(hb - 1)) << 1) | (k & (hb - 1)); }
__device__ __forceinline__ int jb_pairof(int r, int hb) { return ((r >> 1) & ~(hb - 1)) | (r & (hb - 1)); }
// MUFU seed + two Newton steps: full double precision up to an ulp or two
__device__ __forceinline__ double jb_rsqrt(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double h = 0.5 * x;
  r = r * fma(-h * r, r, 1.5);
  r = r * fma(-h * r, r, 1.5);
  return r;
}
// Rotation annihilating a_pq of [[app, apq], [apq, aqq]] (p < q): with rho =
// 1/sqrt(zeta^2 + 4 apq^2), zeta = aqq - app, cos 2th = |zeta| rho, u = 1 + cos 2th >= 1
// (no cancellation), w = 1/sqrt(2u):  c = u w, s = sgn(zeta) 2 apq rho w,
// t = s / c = 2 sin2th w^2 (the tangent of the standard formula); the new diagonal
// app - t apq, aqq + t apq keeps high relative accuracy.  Applied only if
// apq^2 > max(abs^2, tol^2 |app aqq|) (Demmel-Veselic), else the identity.
__device__ __forceinline__ void jac_rot(double app, double aqq, double apq, double tol2, double abs2, double& c,
                                        double& s, double& dA, double& dB, int& act) {
  const double zeta = aqq - app, two = 2.0 * apq;
  const double rho = jb_rsqrt(fma(zeta, zeta, two * two));
  const double u = fma(fabs(zeta), rho, 1.0);
  const double w = jb_rsqrt(2.0 * u);
  const double sg = (zeta >= 0.0 ? two : -two) * rho;
  act = apq * apq > fmax(abs2, tol2 * fabs(app * aqq));
  c = u * w;
  s = sg * w;
  const double t = 2.0 * sg * (w * w);
  dA = app - t * apq;
  dB = aqq + t * apq;
  if (!act) { c = 1.0; s = 0.0; dA = app; dB = aqq; }
}

__global__ void __launch_bounds__(BJ_THREADS, 3) jacobi_block_kernel(BJParams p) {
  extern __shared__ double sh[];
  double* S = sh;                     // 32 x 33
  double* Q = S + BJ_P * BJ_LD;       // 32 x 33
  double* X = Q + BJ_P * BJ_LD;       // BJ_VT x 33 (phase 2)
  double* Y = X + BJ_VT * BJ_LD;      // BJ_VT x 33 (phase 2)
  __shared__ double c_[2][BJ_W], s_[2][BJ_W], dA_[2][BJ_W], dB_[2][BJ_W];
  __shared__ int act_[2][BJ_W];
  __shared__ int srot, srot2;
  __shared__ double sdmax[16];
  const int tid = threadIdx.x, nth = blockDim.x;
  const int64_t ld = p.ld;
  const int bp = p.bp, b = p.b;
  const int64_t gtid = (int64_t)blockIdx.x * nth + tid, gthreads = (int64_t)gridDim.x * nth;

  {  // absolute floor relative to max |a_ii| (same in every CTA)
    double dm = 0.0;
    for (int i = tid; i < b; i += nth) dm = fmax(dm, fabs(p.Ain[(int64_t)i * p.lda + i]));
    for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    if ((tid & 31) == 0) sdmax[tid >> 5] = dm;
    __syncthreads();
    dm = 0.0;
    for (int w = 0; w < (nth >> 5); ++w) dm = fmax(dm, sdmax[w]);
    __syncthreads();
    if (tid == 0) sdmax[0] = dm;
    __syncthreads();
  }
  const double abstol = p.abstol * sdmax[0];
  const double abs2 = abstol * abstol, tol2 = p.tol * p.tol;
  for (int64_t e = gtid; e < (int64_t)bp * bp; e += gthreads) {
    int i = (int)(e % bp), j = (int)(e / bp);
    p.A0[j * ld + i] = (i < b && j < b) ? p.Ain[(int64_t)j * p.lda + i] : 0.0;
    p.V[j * ld + i] = (i == j) ? 1.0 : 0.0;
  }
  for (int64_t e = gtid; e < 256; e += gthreads) p.cnt[e] = 0;  // rotation counts [0, 128), tests [128, 256)
  // block-pair marks of the convergence pass (A1 is not used by this kernel): marks[I m + J]
  // = g when block pair (I, J) held an entry above the threshold after sweep g - 1
  int* const marks = (int*)p.A1;
  for (int64_t e = gtid; e < (int64_t)p.m * p.m; e += gthreads) marks[e] = 0;
  grid_barrier(p.bar);

  double* cur = p.A0;  // updated in place: blocks of unrotated pairs are never touched
  const int m = p.m, h = p.h;
  const int vt = (int)cdiv_d(bp, BJ_VT);
  const int nkl = h * (h - 1) / 2;
  // phase-2 thread tile: rows ty (+32), cols tx + 8c (threads 0-255; warp 8 idles there)
  const int ty = tid < 256 ? tid >> 3 : 1 << 20, tx = tid & 7;
  // one update item: the off-diagonal pair block (k, l) (t < 0: both sides rotate) or the
  // 64-row V tile t of pair l (k == l: V <- V Q_l), with the pairing of step stp and the
  // rotations of buffer par (rotations are double-buffered so the V tiles of step s can be
  // updated during phase 1 of step s + 1 by the CTAs that have no pair block there)
  auto item = [&](int k, int l, int t, int stp, int par) {
        int Ik, Jk, Il, Jl;
        bj_pair(k, stp, m, Ik, Jk);
        bj_pair(l, stp, m, Il, Jl);
        const int* rf = p.rotf + par * h;
        const bool rk = t < 0 && rf[k], rl = rf[l];
        const int rows = t < 0 ? BJ_P : min(BJ_VT, bp - t * BJ_VT);
        if (!rk && !rl) return;  // identity on both sides: the block (or V tile) is unchanged
        const double* Qk = p.Qb + ((int64_t)par * h + k) * BJ_P * BJ_P;
        const double* Ql = p.Qb + ((int64_t)par * h + l) * BJ_P * BJ_P;
        if (tid < 256) {  // all loads of a thread in flight before its stores
          // X: rows x 32 (column c of the l pair, rows of the k pair or of V tile t);
          // thread: row r = tid % 64 (< rows), columns tid / 64 + 4 j
          double xv[8], qkv[4], qlv[4];
          const int r = tid & 63, c0 = tid >> 6;
          const bool rv = r < rows;
          const int64_t roff = (t < 0) ? (r < BJ_P ? bj_g(r, Ik, Jk) : 0) : (int64_t)t * BJ_VT + r;
          const double* base = (t < 0) ? cur : p.V;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int c = c0 + 4 * j;
            xv[j] = rv ? base[(int64_t)bj_g(c, Il, Jl) * ld + roff] : 0.0;
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            qkv[j] = rk ? Qk[tid + 256 * j] : 0.0;
            qlv[j] = rl ? Ql[tid + 256 * j] : 0.0;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (rv) X[r * BJ_LD + c0 + 4 * j] = xv[j];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int e = tid + 256 * j, qr = e >> 5, qc = e & 31;
            if (rk) S[qr * BJ_LD + qc] = qkv[j];
            if (rl) Q[qr * BJ_LD + qc] = qlv[j];
          }
        }
        __syncthreads();
        if (rk) {  // Y = Qk^T X (32 x 32)
          double a4[4];
          if (tid < 256) {
#pragma unroll
          for (int c = 0; c < 4; ++c) a4[c] = 0.0;
          for (int q = 0; q < BJ_P; ++q) {
            const double qa = S[q * BJ_LD + ty];
#pragma unroll
            for (int c = 0; c < 4; ++c) a4[c] = fma(qa, X[q * BJ_LD + tx + 8 * c], a4[c]);
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) Y[ty * BJ_LD + tx + 8 * c] = a4[c];
          }
          __syncthreads();
          double* tmp = X; X = Y; Y = tmp;
        }
        // out = X Ql (or X), rows <= 64: thread rows ty, ty + 32
        for (int r = ty; r < rows; r += 32) {
          double a4[4];
          if (rl) {
#pragma unroll
            for (int c = 0; c < 4; ++c) a4[c] = 0.0;
            for (int q = 0; q < BJ_P; ++q) {
              const double xa = X[r * BJ_LD + q];
#pragma unroll
              for (int c = 0; c < 4; ++c) a4[c] = fma(xa, Q[q * BJ_LD + tx + 8 * c], a4[c]);
            }
          } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) a4[c] = X[r * BJ_LD + tx + 8 * c];
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int cc = tx + 8 * c;
            const int gc = bj_g(cc, Il, Jl);
            if (t < 0) {
              const int gr = bj_g(r, Ik, Jk);
              cur[(int64_t)gc * ld + gr] = a4[c];  // in place: block (k, l) and its mirror
              cur[(int64_t)gr * ld + gc] = a4[c];  // belong to this item alone
            } else {
              p.V[(int64_t)gc * ld + t * BJ_VT + r] = a4[c];
            }
          }
        }
        if (rk) {  // restore buffer roles
          double* tmp = X; X = Y; Y = tmp;
        }
        __syncthreads();
  };
  // the V tiles of one step, over the CTAs [c0, gridDim.x)
  auto v_items = [&](int stp, int par, int c0) {
    if ((int)blockIdx.x < c0) return;
    for (int j = blockIdx.x - c0; j < vt * h; j += gridDim.x - c0) item(j / vt, j / vt, j % vt, stp, par);
  };
  int sweeps = 0, band_sweeps = 0;
  bool converged = false;
  int gs = 0, prev_stp = 0;  // global round counter (rotation buffer parity), previous round's pairing
  unsigned long long tacc[4] = {0, 0, 0, 0}, tq = gtimer();
  // one round: the m/2 disjoint block pairs of schedule step stp (rotation count -> cnt[cslot])
  auto do_round = [&](const int stp, const int cslot) __attribute__((always_inline)) {
      // ---------------- phase 1: diagonalise each pair block
      for (int k = blockIdx.x; k < h; k += gridDim.x) {
        int I, J;
        bj_pair(k, stp, m, I, J);
        double* const S0 = S;  // phase 1: S ping-pong between S and X (phase-2 scratch)
        double* const S1 = X;
        // S: the pair block, swizzled (jb_swz) so every half-warp access below is bank-
        // conflict free; Q: accumulated rotations (pitch BJ_LD)
        if (tid < 256) {  // 4 loads each, all in flight before the stores
          double v4[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int e = tid + 256 * q, r = e & 31, c = e >> 5;
            v4[q] = cur[(int64_t)bj_g(c, I, J) * ld + bj_g(r, I, J)];
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int e = tid + 256 * q, r = e & 31, c = e >> 5;
            S0[r * BJ_P + jb_swz(c)] = v4[q];
            Q[r * BJ_LD + c] = (r == c) ? 1.0 : 0.0;
          }
        }
        __syncthreads();
        // early exit: no off-diagonal entry of the pair block above its threshold means
        // the inner sweep would rotate nothing (converged sweeps, nearly diagonal input)
        bool any = false;
        if (tid < 256) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int e = tid + 256 * q, r = e & 31, c = e >> 5;
            if (r < c) {
              const double apq = S0[r * BJ_P + jb_swz(c)];
              const double app = S0[r * BJ_P + jb_swz(r)], aqq = S0[c * BJ_P + jb_swz(c)];
              any |= apq * apq > fmax(abs2, tol2 * fabs(app * aqq));
            }
          }
        }
        int rot_total = 0, sbuf = 0;
        if (__syncthreads_or(any)) {
          // inner cyclic sweeps in the xor ordering: step m (1..31) pairs r with r ^ m.
          // Rotations of step 1 first; then per step ONE __syncthreads: warps 0-7 apply
          // the step's 16 rotations (thread (k, l) owns the 2 x 2 block rows {p_k, q_k} x
          // cols {p_l, q_l}, and Q's columns p_k, q_k), while warp 8 computes the NEXT
          // step's rotations from the step-start data (it re-forms the one rotated entry
          // it needs).  Rotation counts: warp 8, lane 0.
          if (tid < 16) {
            const int pp = 2 * tid, qq = pp + 1;
            double c, s, dA, dB;
            int act;
            jac_rot(S0[pp * BJ_P + jb_swz(pp)], S0[qq * BJ_P + jb_swz(qq)], S0[pp * BJ_P + jb_swz(qq)], tol2, abs2, c,
                    s, dA, dB, act);
            c_[0][tid] = c; s_[0][tid] = s; dA_[0][tid] = dA; dB_[0][tid] = dB; act_[0][tid] = act;
            const unsigned bal = __ballot_sync(0xffffu, act);
            if (tid == 0) srot = __popc(bal);
          }
          __syncthreads();
          int nrot = srot;  // rotations of the current sweep (warp 8 keeps counting)
          const int k2 = (tid >> 4) & 15, l2 = tid & 15;
          int buf = 0;
          for (int isw = 0; isw < p.inner_sweeps; ++isw) {
            for (int mm = 1; mm < BJ_P; ++mm) {
              const int hb = jb_hbit(mm);
              // S ping-pong: the step reads Sc and writes every entry to Sn (warp 8 reads
              // step-start entries of Sc while warps 0-7 update)
              const double* Sc = sbuf ? S1 : S0;
              double* Sn = sbuf ? S0 : S1;
              if (tid < 256) {
                const int pk = jb_lower(k2, hb), qk = pk ^ mm, pl = jb_lower(l2, hb), ql = pl ^ mm;
                const bool ak = act_[buf][k2], al = act_[buf][l2];
                double x00 = Sc[pk * BJ_P + jb_swz(pl)], x01 = Sc[pk * BJ_P + jb_swz(ql)];
                double x10 = Sc[qk * BJ_P + jb_swz(pl)], x11 = Sc[qk * BJ_P + jb_swz(ql)];
                if (ak || al) {
                  if (k2 == l2) {  // exact diagonal / annihilated entries
                    x00 = dA_[buf][k2]; x01 = 0.0; x10 = 0.0; x11 = dB_[buf][k2];
                  } else {
                    const double ck = c_[buf][k2], sk = s_[buf][k2], cl = c_[buf][l2], sl = s_[buf][l2];
                    const double y00 = ck * x00 - sk * x10, y01 = ck * x01 - sk * x11;
                    const double y10 = sk * x00 + ck * x10, y11 = sk * x01 + ck * x11;
                    x00 = cl * y00 - sl * y01; x01 = sl * y00 + cl * y01;
                    x10 = cl * y10 - sl * y11; x11 = sl * y10 + cl * y11;
                  }
                }
                Sn[pk * BJ_P + jb_swz(pl)] = x00; Sn[pk * BJ_P + jb_swz(ql)] = x01;
                Sn[qk * BJ_P + jb_swz(pl)] = x10; Sn[qk * BJ_P + jb_swz(ql)] = x11;
                if (ak) {
                  const double c = c_[buf][k2], s = s_[buf][k2];
#pragma unroll
                  for (int h2 = 0; h2 < 2; ++h2) {
                    const int j = l2 + 16 * h2;
                    const double vp = Q[j * BJ_LD + pk], vq = Q[j * BJ_LD + qk];
                    Q[j * BJ_LD + pk] = c * vp - s * vq;
                    Q[j * BJ_LD + qk] = s * vp + c * vq;
                  }
                }
              } else if (tid < 256 + 32) {
                // next step's pair j = lane: (pn, qn = pn ^ mn), pn < qn
                const int j = tid & 15;
                const int mn = (mm == BJ_P - 1) ? 1 : mm + 1, hn = jb_hbit(mn);
                const int pn = jb_lower(j, hn), qn = pn ^ mn;
                // this step's pairs of pn and qn (an upper element r is r0 ^ mm, r0 its lower)
                const int kp = jb_pairof((pn & hb) ? pn ^ mm : pn, hb), kq = jb_pairof((qn & hb) ? qn ^ mm : qn, hb);
                const int r0 = jb_lower(kp, hb), r1 = r0 ^ mm, c0 = jb_lower(kq, hb), c1 = c0 ^ mm;
                const double x00 = Sc[r0 * BJ_P + jb_swz(c0)], x01 = Sc[r0 * BJ_P + jb_swz(c1)];
                const double x10 = Sc[r1 * BJ_P + jb_swz(c0)], x11 = Sc[r1 * BJ_P + jb_swz(c1)];
                const double ck = c_[buf][kp], sk = s_[buf][kp], cl = c_[buf][kq], sl = s_[buf][kq];
                // entry (pn, qn) after this step (pn, qn lie in different pairs kp != kq)
                const bool rlo = (pn & hb) == 0, clo = (qn & hb) == 0;
                const double ya = rlo ? ck * x00 - sk * x10 : sk * x00 + ck * x10;
                const double yb = rlo ? ck * x01 - sk * x11 : sk * x01 + ck * x11;
                const double apq = clo ? cl * ya - sl * yb : sl * ya + cl * yb;
                const double app = rlo ? dA_[buf][kp] : dB_[buf][kp];
                const double aqq = clo ? dA_[buf][kq] : dB_[buf][kq];
                double c, s, dA, dB;
                int act;
                jac_rot(app, aqq, apq, tol2, abs2, c, s, dA, dB, act);
                if (tid < 256 + 16) {
                  c_[buf ^ 1][j] = c; s_[buf ^ 1][j] = s; dA_[buf ^ 1][j] = dA; dB_[buf ^ 1][j] = dB;
                  act_[buf ^ 1][j] = act;
                }
                const unsigned bal = __ballot_sync(0xffffffffu, act && tid < 256 + 16);
                if (mm < BJ_P - 1) nrot += __popc(bal);  // mm = 31 produced the next sweep's step 1
                if (mm == BJ_P - 1 && tid == 256) srot = __popc(bal);
              }
              __syncthreads();
              buf ^= 1;
              sbuf ^= 1;
            }
            // the sweep's count lives in warp 8; publish it (and the next sweep's step-1 count)
            if (tid == 256) srot2 = nrot;
            __syncthreads();
            const int rot_sw = srot2;
            nrot = srot;
            __syncthreads();
            rot_total += rot_sw;
            if (rot_sw == 0) break;
          }
        }
        // write Q_k, the flag and the rotated diagonal block
        double* Qk = p.Qb + ((int64_t)(gs & 1) * h + k) * BJ_P * BJ_P;
        if (rot_total && tid < 256) {  // in place: the pair's diagonal block belongs to this CTA alone
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int e = tid + 256 * q;
            const int r = e >> 5, c = e & 31;  // Q_k row-major: consecutive threads, consecutive c
            Qk[r * BJ_P + c] = Q[r * BJ_LD + c];
            const int r2 = e & 31, c2 = e >> 5;  // cur col-major: consecutive threads, consecutive rows
            cur[(int64_t)bj_g(c2, I, J) * ld + bj_g(r2, I, J)] = (sbuf ? S1 : S0)[r2 * BJ_P + jb_swz(c2)];
          }
        }
        if (tid == 0) {
          p.rotf[(gs & 1) * h + k] = rot_total > 0;
          if (rot_total) atomicAdd(&p.cnt[cslot], rot_total);
        }
        __syncthreads();
      }
      // the previous step's V tiles, by the CTAs without a pair block (all CTAs after their
      // pair blocks when the grid is not larger than h)
      if (gs > 0) v_items(prev_stp, (gs - 1) & 1, (int)gridDim.x > h ? h : 0);
      { unsigned long long t = gtimer(); tacc[0] += t - tq; tq = t; }
      grid_barrier(p.bar);
      { unsigned long long t = gtimer(); tacc[1] += t - tq; tq = t; }
      // ---------------- phase 2: off-diagonal pair blocks (32 x 32); the V tiles of this step
      // are deferred into the next step's phase 1
      for (int it = blockIdx.x; it < nkl; it += gridDim.x) {
        int l = (int)((sqrtf(8.0f * (float)it + 1.0f) + 1.0f) * 0.5f);
        while (l * (l - 1) / 2 > it) --l;
        while ((l + 1) * l / 2 <= it) ++l;
        const int k = it - l * (l - 1) / 2;  // k < l
        item(k, l, -1, stp, gs & 1);
      }
      { unsigned long long t = gtimer(); tacc[2] += t - tq; tq = t; }
      grid_barrier(p.bar);
      { unsigned long long t = gtimer(); tacc[3] += t - tq; tq = t; }
      prev_stp = stp;
      ++gs;
  };
  // Banded pre-phase.  The Rayleigh-Ritz matrices this solver gets (W W^T of a block from
  // simultaneous iteration, columns aligned with the eigenvectors except inside clusters)
  // couple only nearby indices: on cfg 2 / 4 the relative couplings |a_ij| / sqrt(a_ii a_jj)
  // fall below 1e-8 beyond |i - j| ~ 64 / ~128.  Sweeps over the block pairs at distance
  // <= D (2 D rounds each, against m - 1 for a round-robin sweep) annihilate the band
  // first; the round-robin sweeps then start from ~1e-7 instead of ~1e-1 and need 1-2
  // instead of 4-5 (CPU simulation of this kernel's rotation sequence on emulated cfg 2 / 3 /
  // 4 matrices: 95 -> 43, 36 -> 21, 235 -> 111 rounds).  Skipped when some coupling beyond
  // the band exceeds 1e-3 (no band structure: e.g. random eigenvectors).  Band sweeps stop
  // once one rotates < 30 % of the first one's count, at most band_max.
  if (p.band_d > 0) {
    const int D = p.band_d;
    int far = 0;
    for (int64_t e = gtid; e < (int64_t)b * b; e += gthreads) {
      const int i = (int)(e % b), j = (int)(e / b);
      if (i < j && j / BJ_W - i / BJ_W > D) {
        const double apq = cur[(int64_t)j * ld + i];
        const double app = cur[(int64_t)i * ld + i], aqq = cur[(int64_t)j * ld + j];
        far |= apq * apq > 1e-6 * fabs(app * aqq);
      }
    }
    if (__syncthreads_or(far) && tid == 0) atomicAdd(p.cnt + 250, 1);
    grid_barrier(p.bar);
    if (*(volatile int*)(p.cnt + 250) == 0) {
      int c0 = 0;
      for (int bs = 0; bs < p.band_max && bs < 8; ++bs) {
        for (int d = 1; d <= D; ++d)
          for (int par = 0; par < 2; ++par) do_round(-1 - (2 * (d - 1) + par), 120 + bs);
        ++band_sweeps;
        const int c = *(volatile int*)(p.cnt + 120 + bs);  // after the round's last barrier
        if (bs == 0) c0 = c;
        if (c == 0 || (bs > 0 && 10LL * c < 3LL * c0)) break;
      }
    }
  }
  // Round-robin sweeps.  After every sweep one pass over the strict upper triangle applies
  // the rotation test to the current matrix and marks the block pairs holding an entry that
  // would rotate: none means converged (the next sweep would change nothing, bitwise); else
  // the next sweep runs only the steps that contain a marked pair (the other steps' pair
  // solves would all exit early).  Pairs that a later round of the same sweep pushes above
  // the threshold are caught by the next pass.  cfg 4 after the band phase: the second
  // sweep rotates 37-271 entries, in a handful of the 47 steps.
  for (int sw = 0; sw < p.max_sweeps; ++sw) {
    for (int step = 0; step < m - 1; ++step) {
      if (sw > 0 && p.select) {  // marks are written only between sweeps: every CTA decides alike
        bool need = false;
        for (int k = 0; k < h && !need; ++k) {
          int I, J;
          bj_pair(k, step, m, I, J);
          need = marks[I * m + J] == sw;
        }
        if (!need) continue;
      }
      do_round(step, sw);
    }
    ++sweeps;
    const int rot_sw = *(volatile int*)(p.cnt + sw);  // read after the barrier: identical in every CTA
    if (rot_sw == 0) {
      converged = true;
      break;
    }
    {
      int* flag = p.cnt + 128 + sw;
      int any = 0;
      for (int64_t e = gtid; e < (int64_t)b * b; e += gthreads) {
        const int i = (int)(e % b), j = (int)(e / b);
        if (i < j) {
          const double apq = cur[(int64_t)j * ld + i];
          const double app = cur[(int64_t)i * ld + i], aqq = cur[(int64_t)j * ld + j];
          if (apq * apq > fmax(abs2, tol2 * fabs(app * aqq))) {
            any = 1;
            marks[(i / BJ_W) * m + j / BJ_W] = sw + 1;
          }
        }
      }
      if (__syncthreads_or(any) && tid == 0) atomicAdd(flag, 1);
      grid_barrier(p.bar);
      if (*(volatile int*)flag == 0) {
        converged = true;
        break;
      }
    }
  }
  // the last step's V tiles (its rotations are complete: phase 2 ended with a barrier)
  if (gs > 0) v_items(prev_stp, (gs - 1) & 1, 0);
  for (int64_t i = gtid; i < b; i += gthreads) p.lam[i] = cur[i * ld + i];
  if (gtid == 0) {
    p.info[0] = sweeps;
    p.info[2] = converged ? 0 : 1;
    p.info[3] = band_sweeps;
    if (p.ts)
      for (int i = 0; i < 4; ++i) p.ts[i] = tacc[i];
  }
}

// sort eigenpairs descending (ties: lower index first); one CTA computes ranks
__global__ void rank_sort_kernel(int b, const double* lam_u, double* lam, int* perm) {
  for (int i = threadIdx.x; i < b; i += blockDim.x) {
    double li = lam_u[i];
    int r = 0;
    for (int j = 0; j < b; ++j) {
      double lj = lam_u[j];
      r += (lj > li) || (lj == li && j < i);
    }
    perm[r] = i;
    lam[r] = li;
  }
}

__global__ void permute_cols_kernel(int b, const double* V, int64_t ldv_in, const int* perm, double* Vout,
                                    int64_t ldv) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)b * b) return;
  int i = (int)(e % b), j = (int)(e / b);
  Vout[j * ldv + i] = V[(int64_t)perm[j] * ldv_in + i];
}

// ------------------------------------------------------------------ workspace
int DenseWs::ensure(int64_t b, cudaStream_t st) {
  if (b <= cap_b && bar) return RHOSVD_OK;
  release(st);
  int64_t bb = std::max<int64_t>(b, 32);
  ld = round_up(bb, 2);
  size_t mat = (size_t)ld * bb;
  RH_CUDA(cudaMallocAsync((void**)&bar, 64, st));
  RH_CUDA(cudaMemsetAsync(bar, 0, 64, st));
  RH_CUDA(cudaMallocAsync((void**)&A0, mat * sizeof(double), st));
  RH_CUDA(cudaMallocAsync((void**)&A1, mat * sizeof(double), st));
  RH_CUDA(cudaMallocAsync((void**)&V, mat * sizeof(double), st));
  RH_CUDA(cudaMallocAsync((void**)&cs, (size_t)(2 * bb + 64) * sizeof(double), st));
  RH_CUDA(cudaMallocAsync((void**)&perm, (size_t)(bb + 64) * sizeof(int), st));
  RH_CUDA(cudaMallocAsync((void**)&info, 64, st));
  RH_CUDA(cudaMemsetAsync(info, 0, 64, st));
  const int64_t hmax = cdiv(bb, 64) + 1;
  RH_CUDA(cudaMallocAsync((void**)&Qb, (size_t)hmax * 4096 * sizeof(double), st));
  RH_CUDA(cudaMallocAsync((void**)&rotf, (size_t)(2 * hmax + 64) * sizeof(int), st));
  RH_CUDA(cudaMallocAsync((void**)&cnt, 256 * sizeof(int), st));
  cap_b = bb;
  return RHOSVD_OK;
}
void DenseWs::release(cudaStream_t st) {
  if (bar) cudaFreeAsync(bar, st);
  if (A0) cudaFreeAsync(A0, st);
  if (A1) cudaFreeAsync(A1, st);
  if (V) cudaFreeAsync(V, st);
  if (cs) cudaFreeAsync(cs, st);
  if (perm) cudaFreeAsync(perm, st);
  if (info) cudaFreeAsync(info, st);
  if (Qb) cudaFreeAsync(Qb, st);
  if (rotf) cudaFreeAsync(rotf, st);
  if (cnt) cudaFreeAsync(cnt, st);
  bar = nullptr; A0 = A1 = V = cs = Qb = nullptr; perm = info = rotf = cnt = nullptr;
  cap_b = 0;
}

// Cooperative grid size: at most the co-resident CTAs, further capped by
// RHOSVD_COOP_MAX (the three per-mode solves run concurrently, and a cooperative kernel
// that asks for every SM waits for all of them to be free).
static int coop_grid(const void* kern, int threads, size_t smem, int64_t want_blocks) {
  static const int cap = [] {
    const char* e = getenv("RHOSVD_COOP_MAX");
    return e ? std::max(1, atoi(e)) : 1 << 30;
  }();
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
  if (occ < 1) occ = 1;
  int64_t maxb = std::min<int64_t>((int64_t)occ * num_sms(), cap);
  if (g_coop_cap > 0) maxb = std::min<int64_t>(maxb, g_coop_cap);
  int64_t g = std::min<int64_t>(maxb, std::max<int64_t>(1, want_blocks));
  return (int)g;
}

int syevj(int64_t b, const double* A, int64_t lda, double* lambda, double* Vout, int64_t ldv, double tol,
          double abstol, int max_sweeps, DenseWs& ws, cudaStream_t st, int* sweeps_host) {
  if (b <= 0) return RHOSVD_OK;
  if (b > 4096) return fail(RHOSVD_EINVAL, "syevj: b > 4096");
  RH_CHECK(ws.ensure(b, st));
  JacParams jp{};
  jp.b = (int)b;
  jp.m = (int)(b + (b & 1));
  jp.h = jp.m / 2;
  if (jp.m < 2) jp.m = 2, jp.h = 1;
  jp.Ain = A; jp.lda = lda; jp.A0 = ws.A0; jp.A1 = ws.A1; jp.ld = ws.ld; jp.V = ws.V;
  jp.lam = ws.cs;  // unsorted eigenvalues staged in cs
  jp.tol = tol; jp.abstol = abstol; jp.max_sweeps = max_sweeps; jp.bar = ws.bar; jp.info = ws.info;
  static const int smem_maxb = [] {
    const char* e = getenv("RHOSVD_JAC_SMEM_MAXB");
    return e ? std::max(0, std::min(atoi(e), JAC_SMEM_MAXB)) : 32;
  }();
  if (b <= smem_maxb) {
    const int threads = 1024;
    size_t smem = (size_t)b * (b | 1) * sizeof(double) + (size_t)jp.h * (3 * sizeof(double) + 3 * sizeof(int)) + 64;
    static const cudaError_t attr_s =
        cudaFuncSetAttribute(jacobi_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    RH_CUDA(attr_s);
    jacobi_smem_kernel<<<1, threads, smem, st>>>(jp);
    count_launch();
    RH_LAUNCH_CHECK();
  } else {
    const int nb = (int)cdiv(b, BJ_W);
    BJParams bj{};
    bj.b = (int)b;
    bj.m = nb + (nb & 1);
    bj.h = bj.m / 2;
    bj.bp = bj.m * BJ_W;
    RH_CHECK(ws.ensure(bj.bp, st));
    bj.Ain = A; bj.lda = lda; bj.A0 = ws.A0; bj.A1 = ws.A1; bj.ld = ws.ld; bj.V = ws.V; bj.Qb = ws.Qb;
    bj.rotf = ws.rotf; bj.lam = ws.cs; bj.tol = tol; bj.abstol = abstol;
    bj.max_sweeps = std::min(max_sweeps, 120);  // cnt[0, 128): per-sweep rotations, [128, 256): tests
    {
      static const int inner = [] {
        const char* e = getenv("RHOSVD_JAC_INNER");
        return e ? std::max(1, atoi(e)) : 1;
      }();
      bj.inner_sweeps = inner;
    }
    bj.bar = ws.bar; bj.cnt = ws.cnt; bj.info = ws.info;
    // banded pre-phase (see the kernel): block distance D ~ b / 96 (the coupling band of the
    // Rayleigh-Ritz matrices grows with the block: ~48 indices at b ~ 300, ~128 at b ~ 760),
    // at least 2, at most m/2 - 1; off for m < 8.  RHOSVD_JAC_BAND=0 disables it,
    // RHOSVD_JAC_BAND_D forces D.
    {
      static const int band_env = [] {
        const char* e = getenv("RHOSVD_JAC_BAND");
        return e ? atoi(e) : 1;
      }();
      static const int band_d_env = [] {
        const char* e = getenv("RHOSVD_JAC_BAND_D");
        return e ? atoi(e) : 0;
      }();
      int D = band_d_env > 0 ? band_d_env : (int)std::lround((double)b / 96.0);
      D = std::max(2, std::min(D, bj.m / 2 - 1));
      bj.band_d = (band_env && bj.m >= 8) ? D : 0;
      bj.band_max = 6;
      static const int sel_env = [] {
        const char* e = getenv("RHOSVD_JAC_SELECT");
        return e ? atoi(e) : 1;
      }();
      bj.select = sel_env;
    }
    const int threads = BJ_THREADS;
    const size_t smem = (size_t)(2 * BJ_P + 2 * BJ_VT) * BJ_LD * sizeof(double);
    static const cudaError_t attr_b =
        cudaFuncSetAttribute(jacobi_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    RH_CUDA(attr_b);
    int64_t want = (int64_t)bj.h * (bj.h - 1) / 2 + cdiv(bj.bp, BJ_VT) * bj.h;
    // one CTA per SM: the grid barriers (two per round) cost more with 3 CTAs per SM than
    // the extra phase-2 items per CTA (b = 732: 444 CTAs 51.5 ms, 296: 38.5, 148: 36.3, 74: 51.3)
    // the Jacobi's cooperative grid takes twice the per-mode cap (RHOSVD_JAC_CAP_MULT): it is
    // throughput-bound (2.5x slower at 49 CTAs than at 148), unlike the latency-bound
    // Cholesky, so under the concurrent modes it should not be held to a third of the SMs
    // (r2r, cfg 4 eigensolve 98.8 -> 90.0 ms, cfg 2 8.2 -> 7.6; x3 = the whole GPU: 93.3)
    static const int jac_mult = [] {
      const char* e = getenv("RHOSVD_JAC_CAP_MULT");
      return e ? std::max(1, atoi(e)) : 2;
    }();
    const int cap_saved = g_coop_cap;
    if (g_coop_cap > 0) g_coop_cap = std::min(num_sms(), g_coop_cap * jac_mult);
    int grid = coop_grid((const void*)jacobi_block_kernel, threads, smem, std::min<int64_t>(want, num_sms()));
    g_coop_cap = cap_saved;
    static const int tsm = [] {
      const char* e = getenv("RHOSVD_TS");
      return (e && e[0] == '1') ? 1 : 0;
    }();
    unsigned long long* tsb = nullptr;
    if (tsm) cudaMallocAsync((void**)&tsb, 64 * sizeof(unsigned long long), st);
    bj.ts = tsb;
    void* args[] = {&bj};
    RH_CUDA(cudaLaunchCooperativeKernel((const void*)jacobi_block_kernel, dim3(grid), dim3(threads), args, smem, st));
    count_launch();
    if (tsm) {
      unsigned long long h[4];
      int inf[4];
      cudaStreamSynchronize(st);
      cudaMemcpy(h, tsb, sizeof(h), cudaMemcpyDeviceToHost);
      cudaMemcpy(inf, ws.info, sizeof(inf), cudaMemcpyDeviceToHost);
      fprintf(stderr,
              "[jacobi ts] b=%d m=%d grid=%d band D=%d sweeps=%d+%d: phase1 %.1f bar1 %.1f phase2 %.1f bar2 %.1f us\n",
              (int)b, bj.m, grid, bj.band_d, inf[3], inf[0], h[0] * 1e-3, h[1] * 1e-3, h[2] * 1e-3, h[3] * 1e-3);
      if (inf[3] > 0) {
        int bc[8] = {0};
        cudaMemcpy(bc, ws.cnt + 120, sizeof(bc), cudaMemcpyDeviceToHost);
        fprintf(stderr, "[jacobi ts] rotations per band sweep:");
        for (int i = 0; i < std::min(inf[3], 8); ++i) fprintf(stderr, " %d", bc[i]);
        fprintf(stderr, "\n");
      }
      {
        int cnt[16] = {0};
        cudaMemcpy(cnt, ws.cnt, sizeof(int) * std::min(16, bj.max_sweeps), cudaMemcpyDeviceToHost);
        fprintf(stderr, "[jacobi ts] rotations per sweep:");
        for (int i = 0; i < std::min(inf[0], 16); ++i) fprintf(stderr, " %d", cnt[i]);
        fprintf(stderr, "\n");
      }
      cudaFreeAsync(tsb, st);
    }
  }
  rank_sort_kernel<<<1, 1024, 0, st>>>((int)b, ws.cs, lambda, ws.perm);
  permute_cols_kernel<<<(unsigned)cdiv(b * b, 256), 256, 0, st>>>((int)b, ws.V, ws.ld, ws.perm, Vout, ldv);
  count_launch(2);
  RH_LAUNCH_CHECK();
  if (sweeps_host) {
    int info[4];
    RH_CHECK(d2h_wait(info, ws.info, sizeof(info), st));
    *sweeps_host = info[0];
    if (info[2]) *sweeps_host = -info[0];  // negative: not converged
  }
  return RHOSVD_OK;
}

// ------------------------------------------------------------------ Cholesky
// chol_inv_scaled: Bp = D L^{-T}, D = diag(S)^{-1/2}, L = chol(D S D + shift I), as ONE
// cooperative kernel over 64 x 64 blocks (P = ceil(b/64) block rows):
//   panel j : every trailing block (i, k), j < k <= i, is owned by one CTA, which forms
//             L_ij = A_ij Linv_jj^T and L_kj (64 x 64 GEMMs from shared memory) and
//             applies A_ik -= L_ij L_kj^T; the owner of (j+1, j+1) then factors that
//             diagonal block in shared memory and inverts it, so ONE grid barrier per
//             panel suffices;
//   inverse : X = L^{-1} by block diagonals d = 1..P-1 (one barrier each):
//             X_{j+d, j} = -Linv_{j+d} sum_{k=j}^{j+d-1} L_{j+d, k} X_{k, j}.
// A pivot below delta marks a numerically dependent column: it gets a unit pivot and
// a zero sub-column (its tiny residual is kept; the next column-scaled pass
// normalises it) - stable, unlike flooring the pivot.
constexpr int CB = 64, CLD = 65;
struct CholParams {
  int b, P;
  const double* S;
  int64_t lds;
  double shift, delta;
  double* A;     // scaled matrix, bp x bp (ld)
  double* L;     // lower blocks of L (ld)
  double* X;     // L^{-1} (ld)
  double* Linv;  // P diagonal inverses, 64 x 64 row-major each
  unsigned* dep; // P x 2 words: dependent-column mask per panel
  double* d;
  double* Bp;
  int64_t ldb;
  int64_t ld;
  unsigned* bar;
  int* info;
  unsigned long long* ts;  // optional phase timestamps (RHOSVD_TS=1), CTA 0
};

__device__ __forceinline__ void stamp(unsigned long long* ts, int i) {
  if (ts && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    ts[i] = t;
  }
}

// acc[a][c] (+)= sum_q A(r, q) B(q, cc), r = ty + 16 a, cc = tx + 16 c, 64 x 64 x 64 in smem
template <bool AT, bool BT>
__device__ __forceinline__ void mm64(const double* A, const double* B, double acc[4][4], int ty, int tx) {
#pragma unroll 4
  for (int q = 0; q < CB; ++q) {
    double av[4], bv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int r = ty + 16 * a;
      av[a] = AT ? A[q * CLD + r] : A[r * CLD + q];
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int cc = tx + 16 * c;
      bv[c] = BT ? B[cc * CLD + q] : B[q * CLD + cc];
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][c] = fma(av[a], bv[c], acc[a][c]);
  }
}
__device__ __forceinline__ void zero44(double acc[4][4]) {
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
}
// global col-major block (I, J) of M (ld) <-> smem [r][c] (pitch CLD)
// (blockDim.x == 256: all 16 loads of a thread are issued before the first store)
__device__ __forceinline__ void ld_blk(double* sm, const double* M, int64_t ld, int I, int J) {
  const int r = threadIdx.x & 63, c0 = threadIdx.x >> 6;
  const double* src = M + (int64_t)(J * CB + c0) * ld + I * CB + r;
  double v[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = src[(int64_t)(4 * q) * ld];
#pragma unroll
  for (int q = 0; q < 16; ++q) sm[r * CLD + c0 + 4 * q] = v[q];
}
// row-major 64 x 64 (pitch 64) -> smem [r][c] (pitch CLD)
__device__ __forceinline__ void ld_rm(double* sm, const double* G) {
  const int c = threadIdx.x & 63, r0 = threadIdx.x >> 6;
  double v[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = G[(r0 + 4 * q) * CB + c];
#pragma unroll
  for (int q = 0; q < 16; ++q) sm[(r0 + 4 * q) * CLD + c] = v[q];
}

// ---- warp-level 32 x 32 building blocks (lane i holds row i in registers; all loops
// fully unrolled so every register index is static)
// Cholesky of the lower triangle of T (pitch CLD) in place; returns the dependent-
// column mask (pivot <= delta, or c >= wvalid: unit pivot, zero sub-column).
__device__ __forceinline__ unsigned warp_chol32(double* T, double delta, int wvalid) {
  const int lane = threadIdx.x & 31;
  double a[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) a[k] = (k <= lane) ? T[lane * CLD + k] : 0.0;
  unsigned dep = 0u;
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const double d = __shfl_sync(0xffffffffu, a[c], c);
    if (c >= wvalid || !(d > delta)) {  // warp-uniform
      dep |= 1u << c;
      if (lane > c) a[c] = 0.0;
      if (lane == c) a[c] = 1.0;
      continue;
    }
    const double rp = rsqrt(d);  // one MUFU + Newton: shorter chain than sqrt + divide
    if (lane > c) a[c] *= rp;
    if (lane == c) a[c] = d * rp;
#pragma unroll
    for (int k = c + 1; k < 32; ++k) {
      const double lkc = __shfl_sync(0xffffffffu, a[c], k);
      if (lane >= k) a[k] = fma(-a[c], lkc, a[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < 32; ++k) T[lane * CLD + k] = (k <= lane) ? a[k] : 0.0;
  __syncwarp();
  return dep;
}
// X = L^{-1} (both 32 x 32 lower, pitch CLD); lane j computes column j
__device__ __forceinline__ void warp_inv32(const double* L, double* X) {
  const int lane = threadIdx.x & 31;
  const double rdl = 1.0 / L[lane * CLD + lane];
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    double s = (i == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) s = fma(-L[i * CLD + k], x[k], s);
    const double rd = __shfl_sync(0xffffffffu, rdl, i);
    x[i] = (i >= lane) ? s * rd : 0.0;
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) X[i * CLD + lane] = x[i];
  __syncwarp();
}
// C(32 x 32, 4 outputs per thread: row tid/8, cols tid%8 + 8q) = sum_k A(r, k) B'(c, k)
// with B' = B (BT) or B^T
template <bool BT>
__device__ __forceinline__ void mm32(const double* A, const double* B, double acc[4]) {
  const int r = threadIdx.x >> 3, c0 = threadIdx.x & 7;
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] = 0.0;
#pragma unroll 8
  for (int k = 0; k < 32; ++k) {
    const double av = A[r * CLD + k];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = c0 + 8 * q;
      acc[q] = fma(av, BT ? B[c * CLD + k] : B[k * CLD + c], acc[q]);
    }
  }
}

// Factor the (already updated) diagonal block in sm (64 x 64, lower used) in place into
// L_jj, write it to L, its inverse to Linv[j] and X, and the dependent-column mask.
// Register-resident right-looking Cholesky: thread t owns row i = t / 4, columns
// k = t % 4 + 4 s (s = 0..15); at step c the owners of column c publish it to a
// double-buffered shared vector, ONE __syncthreads, and every thread applies
// a_ik -= a_ic a_kc / d_c to its elements (unscaled; columns scaled at the end).  The
// inverse is row-sequential forward substitution, 4 threads per column j (all inside
// one warp: __syncwarp only).  Dependent columns (pivot <= delta, or padding): unit
// pivot, zero sub-column.
#ifndef RHOSVD_PROBE_STAMP
#define RHOSVD_PROBE_STAMP(i)
#endif
__device__ void chol_diag_block(double* sm, double* inv, const CholParams& p, int j) {
  const int tid = threadIdx.x;
  const int w = min(CB, p.b - j * CB);
  RHOSVD_PROBE_STAMP(0);
  const int i = tid >> 2, kq = tid & 3;
  __shared__ double colbuf[2][CB];
  __shared__ double dd[CB];
  __shared__ unsigned long long depm;
  double a[16];
#pragma unroll
  for (int s = 0; s < 16; ++s) {
    const int k = kq + 4 * s;
    a[s] = (k <= i) ? sm[i * CLD + k] : 0.0;
  }
  unsigned long long dep = 0ull;
#pragma unroll
  for (int s = 0; s < 16; ++s) {
    for (int q = 0; q < 4; ++q) {
      const int c = 4 * s + q;
      double* cb = colbuf[c & 1];
      if (kq == q && i >= c) cb[i] = a[s];  // publish column c (final from now on)
      __syncthreads();
      const double d = cb[c];
      const bool skip = (c >= w) || !(d > p.delta);
      dep |= (skip ? 1ull : 0ull) << c;
      if (tid == 0) dd[c] = d;
      if (!skip && i > c) {
        const double rs = rsqrt(d);
        const double f = cb[i] * (rs * rs);
#pragma unroll
        for (int s2 = 0; s2 < 16; ++s2) {
          const int k = kq + 4 * s2;
          if (k > c && k <= i) a[s2] = fma(-f, cb[k], a[s2]);
        }
      }
    }
  }
  __syncthreads();
  RHOSVD_PROBE_STAMP(1);
  // scale: L(i, k) = a_ik / sqrt(d_k) (k < i), L(i, i) = sqrt(d_i); dependent: 1 / 0
#pragma unroll
  for (int s = 0; s < 16; ++s) {
    const int k = kq + 4 * s;
    double v = 0.0;
    if (k <= i) {
      const bool dk = (dep >> k) & 1ull;
      if (k == i) v = dk ? 1.0 : sqrt(dd[k]);
      else v = dk ? 0.0 : a[s] * rsqrt(dd[k]);
    }
    sm[i * CLD + k] = v;  // upper part (k > i) zeroed
  }
  if (tid == 0) depm = dep;
  __syncthreads();
  // inverse by 2 x 2 blocks of 32: warps 0 and 1 invert the diagonal halves at the same
  // time (warp-level, registers), then Linv21 = -Linv22 L21 Linv11 (two 32^3 products)
  {
    const int warp = tid >> 5;
    if (warp == 0) warp_inv32(sm, inv);
    if (warp == 1) warp_inv32(sm + 32 * CLD + 32, inv + 32 * CLD + 32);
    __syncthreads();
    const int r = tid >> 3, c0 = tid & 7;
    double acc[4];
    mm32<false>(sm + 32 * CLD, inv, acc);  // T = L21 Linv11 -> scratch in inv's upper right
#pragma unroll
    for (int q = 0; q < 4; ++q) inv[r * CLD + 32 + c0 + 8 * q] = acc[q];
    __syncthreads();
    mm32<false>(inv + 32 * CLD + 32, inv + 32, acc);
#pragma unroll
    for (int q = 0; q < 4; ++q) inv[(32 + r) * CLD + c0 + 8 * q] = -acc[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) inv[r * CLD + 32 + c0 + 8 * q] = 0.0;
  }
  __syncthreads();
  RHOSVD_PROBE_STAMP(2);
  const unsigned long long valid = (w >= 64) ? ~0ull : ((1ull << w) - 1ull);
  if (tid == 0 && (depm & valid)) atomicOr(p.info + 1, 1);
  double* Lg = p.Linv + (int64_t)j * CB * CB;
  for (int e = tid; e < CB * CB; e += blockDim.x) {
    const int rr = e >> 6, c = e & 63;  // row-major Linv: consecutive threads, consecutive c
    Lg[rr * CB + c] = inv[rr * CLD + c];
    const int r2 = e & 63, c2 = e >> 6;  // column-major L, X: consecutive threads, consecutive rows
    p.L[(int64_t)(j * CB + c2) * p.ld + j * CB + r2] = sm[r2 * CLD + c2];
    p.X[(int64_t)(j * CB + c2) * p.ld + j * CB + r2] = inv[r2 * CLD + c2];
  }
  if (tid == 0) {
    p.dep[2 * j] = (unsigned)(depm & 0xffffffffu);
    p.dep[2 * j + 1] = (unsigned)(depm >> 32);
  }
  __syncthreads();
  RHOSVD_PROBE_STAMP(3);
}

__global__ void __launch_bounds__(256) chol_blk_kernel(CholParams p) {
  extern __shared__ double sh[];
  double* s0 = sh;
  double* s1 = s0 + CB * CLD;
  double* s2 = s1 + CB * CLD;
  const int tid = threadIdx.x;
  const int ty = tid >> 4, tx = tid & 15;
  const int b = p.b, P = p.P, bp = P * CB;
  const int64_t ld = p.ld;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + tid, gthreads = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = gtid; i < bp; i += gthreads) {
    double sii = i < b ? p.S[i * p.lds + i] : 1.0;
    p.d[i] = sii > 0.0 ? 1.0 / sqrt(sii) : 1.0;
  }
  grid_barrier(p.bar);
  for (int64_t e = gtid; e < (int64_t)bp * bp; e += gthreads) {
    int i = (int)(e % bp), j = (int)(e / bp);
    double v = 0.0;
    if (i < b && j < b) v = p.S[(int64_t)j * p.lds + i] * p.d[i] * p.d[j];
    if (i == j) v += (i < b) ? p.shift : 1.0;
    p.A[(int64_t)j * ld + i] = v;  // (L and X: only their lower blocks are ever read,
  }                                 //  and every one of those is written below)
  grid_barrier(p.bar);
  stamp(p.ts, 0);
  if (blockIdx.x == 0) {
    ld_blk(s0, p.A, ld, 0, 0);
    __syncthreads();
    chol_diag_block(s0, s1, p, 0);
  }
  stamp(p.ts, 1);
  grid_barrier(p.bar);
  stamp(p.ts, 2);
  double acc[4][4];
  for (int j = 0; j + 1 < P; ++j) {
    const int t = P - j - 1;
    const int nitems = t * (t + 1) / 2;
    const unsigned long long dm = ((unsigned long long)p.dep[2 * j + 1] << 32) | p.dep[2 * j];
    for (int q = blockIdx.x; q < nitems; q += gridDim.x) {
      int I = (int)((sqrtf(8.0f * (float)q + 1.0f) - 1.0f) * 0.5f);
      while ((I + 1) * (I + 2) / 2 <= q) ++I;
      while (I * (I + 1) / 2 > q) --I;
      int K = q - I * (I + 1) / 2;
      I += j + 1;
      K += j + 1;
      // s2 = Linv_jj ; s0 = L_Ij = A_Ij Linv^T ; s1 = L_Kj
      ld_rm(s2, p.Linv + (int64_t)j * CB * CB);
      ld_blk(s0, p.A, ld, I, j);
      if (K != I) ld_blk(s1, p.A, ld, K, j);
      __syncthreads();
      zero44(acc);
      mm64<false, true>(s0, s2, acc, ty, tx);
      double acc2[4][4];
      if (K != I) {
        zero44(acc2);
        mm64<false, true>(s1, s2, acc2, ty, tx);
      }
      __syncthreads();
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int cc = tx + 16 * c;
          const bool z = (dm >> cc) & 1ull;
          s0[(ty + 16 * a) * CLD + cc] = z ? 0.0 : acc[a][c];
          if (K != I) s1[(ty + 16 * a) * CLD + cc] = z ? 0.0 : acc2[a][c];
        }
      __syncthreads();
      const double* LK = (K != I) ? s1 : s0;
      if (K == j + 1) {  // the owner of (I, j+1) publishes L_Ij
        for (int e = tid; e < CB * CB; e += blockDim.x) {
          int r = e & 63, c = e >> 6;
          p.L[(int64_t)(j * CB + c) * ld + I * CB + r] = s0[r * CLD + c];
        }
      }
      // A_IK -= L_Ij L_Kj^T
      zero44(acc);
      mm64<false, true>(s0, LK, acc, ty, tx);
      if (I == j + 1 && K == j + 1) {
        // next diagonal block: update in smem, then factor it right here
        __syncthreads();
        ld_blk(s2, p.A, ld, I, K);
        __syncthreads();
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) s2[(ty + 16 * a) * CLD + tx + 16 * c] -= acc[a][c];
        __syncthreads();
        chol_diag_block(s2, s1, p, j + 1);
      } else {  // stage through smem so the global read-modify-write is coalesced
        __syncthreads();
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) s2[(ty + 16 * a) * CLD + tx + 16 * c] = acc[a][c];
        __syncthreads();
        {
          const int r = tid & 63, c0 = tid >> 6;
          double* dst = p.A + (int64_t)(K * CB + c0) * ld + I * CB + r;
#pragma unroll
          for (int q = 0; q < 16; ++q) dst[(int64_t)(4 * q) * ld] -= s2[r * CLD + c0 + 4 * q];
        }
      }
      __syncthreads();
    }
    grid_barrier(p.bar);
    stamp(p.ts, 3 + j);
  }
  // ---------------- X = L^{-1}, right-looking over block rows k (one barrier each):
  // T_ij = sum_{k<i} L_ik X_kj accumulates in A's lower blocks (free after the panels);
  // at step k, item (i, j) (i > k >= j) forms X_kj = -Linv_kk T_kj (X_kk = Linv_kk) and
  // adds L_ik X_kj to T_ij (the first term, k = j, is stored); the items with i = k + 1
  // publish X_kj.  The last step finalises row P - 1.  (Round 1 walked the block diagonals:
  // block (j + d, j) summed its d products alone, a critical path of ~P^2 / 2 products -
  // 420 us of the 985 us at b = 873.)
  for (int k = 0; k < P; ++k) {
    const int rows = P - 1 - k;  // i = k + 1 .. P - 1
    const int nit = rows > 0 ? (k + 1) * rows : k;
    for (int q = blockIdx.x; q < nit; q += gridDim.x) {
      const int jj = rows > 0 ? q / rows : q, i = rows > 0 ? k + 1 + q % rows : -1;
      __syncthreads();
      if (jj < k) {  // s1 = X_kj = -Linv_kk T_kj
        ld_rm(s2, p.Linv + (int64_t)k * CB * CB);
        ld_blk(s0, p.A, ld, k, jj);
        __syncthreads();
        zero44(acc);
        mm64<false, false>(s2, s0, acc, ty, tx);
        __syncthreads();
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) s1[(ty + 16 * a) * CLD + tx + 16 * c] = -acc[a][c];
      } else {  // X_kk = Linv_kk
        ld_rm(s1, p.Linv + (int64_t)k * CB * CB);
      }
      __syncthreads();
      if (jj < k && (i == k + 1 || rows == 0)) {  // publish X_kj
        const int r = tid & 63, c0 = tid >> 6;
        double* dst = p.X + (int64_t)(jj * CB + c0) * ld + k * CB + r;
#pragma unroll
        for (int t = 0; t < 16; ++t) dst[(int64_t)(4 * t) * ld] = s1[r * CLD + c0 + 4 * t];
      }
      if (rows == 0) continue;
      // T_ij (+)= L_ik X_kj
      ld_blk(s0, p.L, ld, i, k);
      __syncthreads();
      zero44(acc);
      mm64<false, false>(s0, s1, acc, ty, tx);
      __syncthreads();
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) s2[(ty + 16 * a) * CLD + tx + 16 * c] = acc[a][c];
      __syncthreads();
      {
        const int r = tid & 63, c0 = tid >> 6;
        double* dst = p.A + (int64_t)(jj * CB + c0) * ld + i * CB + r;
        if (jj == k) {
#pragma unroll
          for (int t = 0; t < 16; ++t) dst[(int64_t)(4 * t) * ld] = s2[r * CLD + c0 + 4 * t];
        } else {
#pragma unroll
          for (int t = 0; t < 16; ++t) dst[(int64_t)(4 * t) * ld] += s2[r * CLD + c0 + 4 * t];
        }
      }
    }
    grid_barrier(p.bar);
    stamp(p.ts, 3 + P + k);
  }
  // ---------------- Bp(c, i) = d_c X(i, c) (i >= c), 0 above: 64 x 64 tiles transposed
  // through smem (coalesced on both sides)
  for (int t = blockIdx.x; t < P * P; t += gridDim.x) {
    const int I = t % P, J = t / P;  // X block (I, J) -> Bp block (J, I)
    const int c = tid & 63, r0 = tid >> 6;
    __syncthreads();
    if (I >= J) ld_blk(s0, p.X, ld, I, J);  // s0[r][c] = X(I*64 + r, J*64 + c)
    __syncthreads();
    const int gc = J * CB + c;
    if (gc < b) {
      const double dc = p.d[gc];
#pragma unroll 4
      for (int q = 0; q < 16; ++q) {
        const int r = r0 + 4 * q, gi = I * CB + r;
        if (gi < b) p.Bp[(int64_t)gi * p.ldb + gc] = (I >= J) ? dc * s0[r * CLD + c] : 0.0;
      }
    }
  }
}

// ---------------------------------------------------------------- one-CTA Cholesky inverse
// The same Bp = D L^{-T} as chol_blk_kernel for b <= 32 E <= 160, in ONE CTA of 32 x 32
// threads with the lower triangle in registers: thread (ty, tx) owns the elements
// (i, k) = (ty + 32 a, tx + 32 c), c <= a < E (the lower 32 x 32 blocks, 2D block-cyclic).
// No grid barrier and no cooperative launch: the kernel occupies one SM, so the three
// concurrent per-mode eigensolves keep the rest of the GPU for their GEMMs (the blocked
// cooperative kernel takes every SM for ~0.1-0.2 ms at b ~ 150).
//   Cholesky (right-looking, unscaled updates): at step c the owners of column c publish
//     it to a double-buffered shared vector, ONE __syncthreads, every thread applies
//     a_ik -= a_ic a_kc / d_c (c < k <= i); pivot d_c <= delta: dependent column (unit
//     pivot, zero sub-column, as the blocked kernel).  L is then written to shared memory.
//   Inverse X = L^{-1} (right-looking forward substitution; row r is final at step r):
//     the owners of row r scale it by 1 / L_rr and publish it, ONE __syncthreads, rows
//     i > r apply x_ic -= L_ir x_rc (c <= r), L_ir read from shared memory (broadcast).
//   Output Bp(c, i) = d_c X(i, c) (c <= i), 0 above.
template <int E>
__global__ void __launch_bounds__(1024, 1) chol_small_kernel(int b, const double* __restrict__ S, int64_t lds,
                                                              double shift, double delta, double* __restrict__ Bp,
                                                              int64_t ldb, int* info) {
  extern __shared__ double Ls[];  // b x (b | 1) lower triangle of L
  __shared__ double cbuf[2][32 * E];
  __shared__ double dsc[32 * E];
  __shared__ double piv[32 * E];
  __shared__ int depf[32 * E];
  const int P = b | 1;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  for (int k = tid; k < b; k += 1024) {
    const double sk = S[(int64_t)k * lds + k];
    dsc[k] = sk > 0.0 ? 1.0 / sqrt(sk) : 1.0;
  }
  __syncthreads();
  double a[E][E];  // a[A][C]: element (ty + 32 A, tx + 32 C), C <= A
#pragma unroll
  for (int A = 0; A < E; ++A)
#pragma unroll
    for (int C = 0; C < E; ++C) {
      const int i = ty + 32 * A, k = tx + 32 * C;
      double v = 0.0;
      if (C <= A && i < b && k <= i) {
        v = S[(int64_t)i * lds + k] * dsc[i] * dsc[k];  // upper-part entry (k, i)
        if (k == i) v += shift;
      }
      a[A][C] = v;
    }
  // ---- Cholesky
#pragma unroll
  for (int Cb = 0; Cb < E; ++Cb) {
    for (int cc = 0; cc < 32; ++cc) {
      const int c = 32 * Cb + cc;
      if (c >= b) break;  // uniform
      double* col = cbuf[c & 1];
      if (tx == cc) {
#pragma unroll
        for (int A = Cb; A < E; ++A) {
          const int i = ty + 32 * A;
          if (i >= c && i < b) col[i] = a[A][Cb];
        }
      }
      __syncthreads();
      const double d = col[c];
      const bool dep = !(d > delta);
      if (tid == 0) {
        piv[c] = d;
        depf[c] = dep ? 1 : 0;
      }
      if (!dep) {
        // blocks left of column block Cb are final (k < 32 Cb <= c): only A, C >= Cb update
        const double rd = 1.0 / d;
        double ci[E], ck[E];
#pragma unroll
        for (int A = Cb; A < E; ++A) {
          const int i = ty + 32 * A, k = tx + 32 * A;
          ci[A] = (i > c && i < b) ? col[i] * rd : 0.0;
          ck[A] = (k > c && k < b) ? col[k] : 0.0;
        }
#pragma unroll
        for (int A = Cb; A < E; ++A)
#pragma unroll
          for (int C = Cb; C <= A; ++C) a[A][C] = fma(-ci[A], ck[C], a[A][C]);
      }
    }
  }
  __syncthreads();
  // scale into L: L(i, k) = a_ik / sqrt(d_k) (k < i), L(i, i) = sqrt(d_i); dependent: 1 / 0
#pragma unroll
  for (int A = 0; A < E; ++A)
#pragma unroll
    for (int C = 0; C <= A; ++C) {
      const int i = ty + 32 * A, k = tx + 32 * C;
      if (i < b && k <= i) {
        const bool dk = depf[k] != 0;
        Ls[i * P + k] = (k == i) ? (dk ? 1.0 : sqrt(piv[k])) : (dk ? 0.0 : a[A][C] / sqrt(piv[k]));
      }
    }
  if (tid == 0) {
    int any = 0;
    for (int c = 0; c < b; ++c) any |= depf[c];
    if (any) atomicOr(info + 1, 1);
  }
  __syncthreads();
  // ---- X = L^{-1}, reusing a[][] for X (Y = I initially)
#pragma unroll
  for (int A = 0; A < E; ++A)
#pragma unroll
    for (int C = 0; C <= A; ++C) a[A][C] = (ty + 32 * A == tx + 32 * C) ? 1.0 : 0.0;
#pragma unroll
  for (int Rb = 0; Rb < E; ++Rb) {
    for (int rr = 0; rr < 32; ++rr) {
      const int r = 32 * Rb + rr;
      if (r >= b) break;
      double* xrow = cbuf[r & 1];
      if (ty == rr) {  // the owners of row r: x_r <- x_r / L_rr, publish
        const double rl = 1.0 / Ls[r * P + r];
#pragma unroll
        for (int C = 0; C <= Rb; ++C) {
          const int c = tx + 32 * C;
          if (c <= r) {
            a[Rb][C] *= rl;
            xrow[c] = a[Rb][C];
          }
        }
      }
      __syncthreads();
      double xv[E];  // x_rc for this thread's columns c = tx + 32 C <= r (0 beyond r)
#pragma unroll
      for (int C = 0; C <= Rb; ++C) {
        const int c = tx + 32 * C;
        xv[C] = (c <= r) ? xrow[c] : 0.0;
      }
#pragma unroll
      for (int A = Rb; A < E; ++A) {
        const int i = ty + 32 * A;
        if (i > r && i < b) {
          const double l = Ls[i * P + r];
#pragma unroll
          for (int C = 0; C <= Rb; ++C) a[A][C] = fma(-l, xv[C], a[A][C]);
        }
      }
    }
  }
  // ---- Bp(c, i) = d_c X(i, c) for c <= i, 0 for c > i
#pragma unroll
  for (int A = 0; A < E; ++A)
#pragma unroll
    for (int C = 0; C < E; ++C) {
      const int i = ty + 32 * A, c = tx + 32 * C;
      if (i < b && c < b) Bp[(int64_t)i * ldb + c] = (C <= A && c <= i) ? dsc[c] * a[A][C] : 0.0;
    }
}

template <int E>
static int chol_small_launch(int64_t b, const double* S, int64_t lds, double shift, double* Bp, int64_t ldb,
                             int* info, cudaStream_t st) {
  const size_t smem = (size_t)b * (b | 1) * sizeof(double);
  static const cudaError_t attr =
      cudaFuncSetAttribute(chol_small_kernel<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * E * (32 * E + 1) * 8);
  RH_CUDA(attr);
  chol_small_kernel<E><<<1, 1024, smem, st>>>((int)b, S, lds, shift, 1e-13, Bp, ldb, info);
  count_launch();
  RH_LAUNCH_CHECK();
  return RHOSVD_OK;
}

// one-CTA path for b <= RHOSVD_CHOL_SMALL_MAXB (default 160; 0 disables)
static int chol_small(int64_t b, const double* S, int64_t lds, double shift, double* Bp, int64_t ldb, int* info,
                      cudaStream_t st) {
  switch ((int)cdiv(b, 32)) {
    case 1: return chol_small_launch<1>(b, S, lds, shift, Bp, ldb, info, st);
    case 2: return chol_small_launch<2>(b, S, lds, shift, Bp, ldb, info, st);
    case 3: return chol_small_launch<3>(b, S, lds, shift, Bp, ldb, info, st);
    case 4: return chol_small_launch<4>(b, S, lds, shift, Bp, ldb, info, st);
    default: return chol_small_launch<5>(b, S, lds, shift, Bp, ldb, info, st);
  }
}

int chol_inv_scaled(int64_t b, const double* S, int64_t lds, double shift_rel, double* Bp, int64_t ldb,
                    DenseWs& ws, cudaStream_t st) {
  if (b <= 0) return RHOSVD_OK;
  static const int small_maxb = [] {
    const char* e = getenv("RHOSVD_CHOL_SMALL_MAXB");
    return e ? std::max(0, std::min(atoi(e), 160)) : 160;
  }();
  if (b <= small_maxb) {
    RH_CHECK(ws.ensure(b, st));
    return chol_small(b, S, lds, shift_rel, Bp, ldb, ws.info, st);
  }
  const int P = (int)cdiv(b, CB);
  RH_CHECK(ws.ensure((int64_t)P * CB, st));
  CholParams cp{};
  cp.b = (int)b; cp.P = P; cp.S = S; cp.lds = lds; cp.shift = shift_rel; cp.delta = 1e-13;
  cp.A = ws.A0; cp.L = ws.A1; cp.X = ws.V; cp.Linv = ws.Qb; cp.dep = (unsigned*)ws.rotf; cp.d = ws.cs;
  cp.Bp = Bp; cp.ldb = ldb; cp.ld = ws.ld; cp.bar = ws.bar; cp.info = ws.info;
  const int threads = 256;
  const size_t smem = (size_t)3 * CB * CLD * sizeof(double);
  static const cudaError_t attr =
      cudaFuncSetAttribute(chol_blk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  RH_CUDA(attr);
  int64_t want = std::max<int64_t>(1, (int64_t)(P - 1) * P / 2);
  int grid = coop_grid((const void*)chol_blk_kernel, threads, smem, want);
  static const int tsmode = [] {
    const char* e = getenv("RHOSVD_TS");
    return (e && e[0] == '1') ? 1 : 0;
  }();
  unsigned long long* tsbuf = nullptr;
  if (tsmode) cudaMallocAsync((void**)&tsbuf, 1024 * sizeof(unsigned long long), st);
  cp.ts = tsbuf;
  void* args[] = {&cp};
  RH_CUDA(cudaLaunchCooperativeKernel((const void*)chol_blk_kernel, dim3(grid), dim3(threads), args, smem, st));
  count_launch();
  RH_LAUNCH_CHECK();
  if (tsmode) {
    unsigned long long h[256];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, tsbuf, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(stderr, "[chol ts] b=%d P=%d grid=%d:", (int)b, P, grid);
    for (int i = 1; i < 3 + 2 * P; ++i)
      if (i != P + 2) fprintf(stderr, " %.1f", (h[i] - h[0]) * 1e-3);
    fprintf(stderr, " us\n");
    cudaFreeAsync(tsbuf, st);
  }
  return RHOSVD_OK;
}

}  // namespace rhosvd
