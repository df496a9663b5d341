// t2c.cu - Tucker-to-canonical (T2C) of the RHOSVD core and its lift through the frames:
// the canonical-to-canonical (C2C) rank reduction C2C = T2C o C2T.
//
// Remark 2.1: beta = sum_m B_m (x) z_m over the mode-3 slices B_m
// (r1 x r2); each slice is replaced by its truncated SVD B_{p_m} keeping the singular values
// above thr = eps / (r3 sqrt(min(r1, r2))) (eps / r^{3/2} for a cubic core; reading T2),
// so that ||beta - beta_(R)|| <= eps with R = p_1 + ... + p_r3.  Lifting the core's CP
// factors through the orthonormal frames (Lemma 2.1) gives
//     A ~ sum_m sum_{k <= p_m} sigma_k^(m) (Z1 u_k) (x) (Z2 v_k) (x) (Z3 e_m).
//
// GPU design: one CTA per slice keeps the whole slice in shared memory and runs a
// one-sided (Hestenes) Jacobi SVD on its columns - warp-parallel over the r2/2 disjoint
// column pairs of a round-robin step, column dot products by warp reductions (fixed
// order), one __syncthreads per step.  sigma_k = ||b_k||, u_k = b_k / sigma_k and
// v_k = B^T u_k / sigma_k from the original slice (no V accumulation, so the slice alone
// must fit in shared memory: r1 x r2 <= ~27 000 doubles).  The kept triplets are
// compacted after a host prefix sum over the r3 counts; the lift is two DMMA GEMMs
// (Z1 U, Z2 V) and a column gather of Z3.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gemm.cuh"
#include "result.h"

namespace rhosvd {

constexpr int T2C_THREADS = 256;
constexpr int T2C_MAX_SWEEPS = 40;

// round-robin tournament position pos at step (0 <= step < m - 1, 0 <= pos < m): position 0
// fixed, the others rotate.  pos - 1 + step < 2 (m - 1), so one conditional subtraction
// replaces the modulo (an integer division; measured no faster on the T2C block kernel,
// whose stall samples put 9 % on it - r2z ncu - but cheaper to issue).
__device__ __forceinline__ int t2c_rr(int pos, int step, int m) {
  if (pos == 0) return 0;
  int x = pos - 1 + step;
  if (x >= m - 1) x -= m - 1;
  return 1 + x;
}

struct T2CParams {
  const double* Bt;    // slice-major copy of beta: Bt[(m r1 + a) r2 + b] = beta[a][b][m]
  int r1, r2, r3, ldb;  // ldb: smem column pitch (odd)
  double thr, tol;
  double* Us;     // per slice: r2 columns of length r1 (u_k, descending sigma)
  double* Vs;     // per slice: r2 columns of length r2 (v_k)
  double* sg;     // per slice: r2 sigma (descending)
  int* cnt;       // per slice: kept count p_m
  int* sweeps;    // per slice: sweeps used (-1: not converged)
  double* drop;   // per slice: discarded energy sum_{k > p_m} sigma_k^2 (smallest first)
};

__global__ void __launch_bounds__(T2C_THREADS) t2c_slice_kernel(T2CParams p) {
  extern __shared__ double sb[];  // B (col-major, pitch ldb) | sigma | order
  const int r1 = p.r1, r2 = p.r2, ld = p.ldb;
  const int m2 = r2 + (r2 & 1);  // even number of columns for the tournament
  double* B = sb;
  double* sig = B + (size_t)ld * m2;
  int* ord = reinterpret_cast<int*>(sig + m2);
  __shared__ int srot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = T2C_THREADS / 32;
  for (int m = blockIdx.x; m < p.r3; m += gridDim.x) {
    // B_m[a][b] = beta[a][b][m], stored column b contiguous; padded column zero
    const double* Bm = p.Bt + (size_t)m * r1 * r2;
    for (int e = tid; e < ld * m2; e += T2C_THREADS) {
      const int a = e % ld, b = e / ld;
      B[e] = (a < r1 && b < r2) ? Bm[(size_t)a * r2 + b] : 0.0;
    }
    __syncthreads();
    // ||B||_F^2 (fixed order): columns with ||b||^2 <= (16 u ||B||_F)^2 are numerically zero
    // and never rotate (their pair cosines are rounding noise)
    __shared__ double sfro;
    if (warp == 0) {
      double s = 0.0;
      for (int e = lane; e < ld * m2; e += 32) s = fma(B[e], B[e], s);
      s = warp_sum(s);
      if (lane == 0) sfro = s;
    }
    __syncthreads();
    const double tiny2 = 256.0 * 1.2325951644078309e-32 * sfro;
    int sw = 0;
    bool conv = false;
    for (; sw < T2C_MAX_SWEEPS && !conv; ++sw) {
      // de Rijk pivoting: visit the columns in decreasing-norm order this sweep (the
      // position -> column map lives in ord; any visiting order is a valid cyclic sweep)
      for (int k = warp; k < r2; k += nw) {
        double s = 0.0;
        for (int i = lane; i < r1; i += 32) s = fma(B[(size_t)k * ld + i], B[(size_t)k * ld + i], s);
        s = warp_sum(s);
        if (lane == 0) sig[k] = s;
      }
      if (tid == 0) srot = 0;
      __syncthreads();
      for (int k = tid; k < r2; k += T2C_THREADS) {
        const double v = sig[k];
        int r = 0;
        for (int j = 0; j < r2; ++j) r += (sig[j] > v) || (sig[j] == v && j < k);
        ord[r] = k;
      }
      if (tid == 0 && m2 > r2) ord[r2] = r2;  // the zero padding column
      __syncthreads();
      for (int st = 0; st < m2 - 1; ++st) {
        for (int k = warp; k < m2 / 2; k += nw) {
          const int pc = ord[t2c_rr(k, st, m2)], qc = ord[t2c_rr(m2 - 1 - k, st, m2)];
          double* bp = B + (size_t)pc * ld;
          double* bq = B + (size_t)qc * ld;
          double al = 0.0, be = 0.0, ga = 0.0;
          for (int i = lane; i < r1; i += 32) {
            const double x = bp[i], y = bq[i];
            al = fma(x, x, al);
            be = fma(y, y, be);
            ga = fma(x, y, ga);
          }
          al = warp_sum(al);
          be = warp_sum(be);
          ga = warp_sum(ga);
          if (al > tiny2 && be > tiny2 && fabs(ga) > p.tol * sqrt(al * be)) {
            // Hestenes rotation annihilating b_p^T b_q
            const double zeta = (be - al) / (2.0 * ga);
            const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double c = rsqrt(1.0 + t * t), s = c * t;
            for (int i = lane; i < r1; i += 32) {
              const double x = bp[i], y = bq[i];
              bp[i] = c * x - s * y;
              bq[i] = s * x + c * y;
            }
            if (lane == 0) atomicAdd(&srot, 1);
          }
        }
        __syncthreads();
      }
      conv = (srot == 0);
      __syncthreads();
    }
    // sigma_k = ||b_k|| (fixed-order warp reductions)
    for (int k = warp; k < r2; k += nw) {
      double s = 0.0;
      for (int i = lane; i < r1; i += 32) s = fma(B[(size_t)k * ld + i], B[(size_t)k * ld + i], s);
      s = warp_sum(s);
      if (lane == 0) sig[k] = sqrt(s);
    }
    __syncthreads();
    // descending order (ties: lower column first)
    for (int k = tid; k < r2; k += T2C_THREADS) {
      const double v = sig[k];
      int r = 0;
      for (int j = 0; j < r2; ++j) r += (sig[j] > v) || (sig[j] == v && j < k);
      ord[r] = k;
    }
    __syncthreads();
    double* Us = p.Us + (size_t)m * r2 * r1;
    double* Vs = p.Vs + (size_t)m * r2 * r2;
    double* sg = p.sg + (size_t)m * r2;
    int keep = 0;
    for (int j = 0; j < r2; ++j) keep += sig[ord[j]] > p.thr;  // same value in every thread
    // kept triplets, one warp each: u = b / sigma with the sign rule (largest-|.| entry of u
    // positive, lowest index on ties); v = B_orig^T u / sigma from the original slice
    // (coalesced rows of Bt), renormalised (its direction error is ~u sigma_1 / sigma)
    for (int j = warp; j < keep; j += nw) {
      const int k = ord[j];
      const double s = sig[k], inv = 1.0 / s;
      const double* bk = B + (size_t)k * ld;
      double best = -1.0;
      int bi = 0x7fffffff;
      for (int i = lane; i < r1; i += 32) {
        const double a = fabs(bk[i]);
        if (a > best || (a == best && i < bi)) {
          best = a;
          bi = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      const double sgn = (bk[bi] < 0.0) ? -inv : inv;
      double* uo = Us + (size_t)j * r1;
      for (int i = lane; i < r1; i += 32) uo[i] = sgn * bk[i];
      double* vo = Vs + (size_t)j * r2;
      double vn = 0.0;
      for (int b = lane; b < r2; b += 32) {
        double acc = 0.0;
        for (int a = 0; a < r1; ++a) acc = fma(Bm[(size_t)a * r2 + b], bk[a], acc);
        acc *= sgn * inv;  // B^T u / sigma with u = sgn * b_k
        vo[b] = acc;
        vn = fma(acc, acc, vn);
      }
      vn = warp_sum(vn);
      const double rv = vn > 0.0 ? 1.0 / sqrt(vn) : 0.0;
      __syncwarp();
      for (int b = lane; b < r2; b += 32) vo[b] *= rv;
      if (lane == 0) sg[j] = s;
    }
    __syncthreads();
    if (tid == 0) {
      p.cnt[m] = keep;
      p.sweeps[m] = conv ? sw : -1;
      double d = 0.0;
      for (int j = r2 - 1; j >= keep; --j) d = fma(sig[ord[j]], sig[ord[j]], d);
      p.drop[m] = d;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- QR-preconditioned slices
// Drmac-Veselic preconditioning: the one-sided Jacobi above needs ~30 sweeps on Tucker-core
// slices (sigma over ~20 decades: the parallel ordering converges slowly among the many
// graded columns).  A Householder QR with column pivoting first, B P = Q R, then the
// one-sided Jacobi on the ROWS of R (= columns of R^T, whose singular values are those of B)
// converges in ~8 (CPU experiment on cfg 3 slices, same tolerance).  With the rotated rows
// w_k: sigma_k = ||w_k||, v_k = P w_k / sigma_k (right singular vectors, in the original
// column order) and u_k = B v_k / sigma_k from the original slice (renormalised).  Q is
// never formed.  Same outputs and conventions as t2c_slice_kernel.
template <int NT>
__global__ void __launch_bounds__(NT) t2c_slice_qr_kernel(T2CParams p) {
  extern __shared__ double sb[];  // B (col-major, pitch ldb) | norms | Householder vector | order | perm
  const int r1 = p.r1, r2 = p.r2, ld = p.ldb;
  const int m2 = r2 + (r2 & 1);
  const int rr = min(r1, r2);
  const int mr = rr + (rr & 1);   // even row count for the tournament (row rr: virtual zero)
  double* B = sb;
  double* sig = B + (size_t)ld * m2;       // m2
  double* hv = sig + m2;                   // ld
  int* ord = reinterpret_cast<int*>(hv + ld);  // m2
  int* perm = ord + m2;                    // m2
  __shared__ int srot, spiv;
  __shared__ double salpha, svn2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = NT / 32;
  for (int m = blockIdx.x; m < p.r3; m += gridDim.x) {
    const double* Bm = p.Bt + (size_t)m * r1 * r2;
    for (int e = tid; e < ld * m2; e += NT) {
      const int a = e % ld, b = e / ld;
      B[e] = (a < r1 && b < r2) ? Bm[(size_t)a * r2 + b] : 0.0;
    }
    for (int j = tid; j < m2; j += NT) perm[j] = j;
    __shared__ double sfro;
    __syncthreads();
    if (warp == 0) {
      double s = 0.0;
      for (int e = lane; e < ld * m2; e += 32) s = fma(B[e], B[e], s);
      s = warp_sum(s);
      if (lane == 0) sfro = s;
    }
    // ---- Householder QR with column pivoting (largest remaining column norm, lowest index on ties)
    for (int k = 0; k < rr; ++k) {
      for (int j = k + warp; j < r2; j += nw) {
        double s = 0.0;
        for (int i = k + lane; i < r1; i += 32) s = fma(B[(size_t)j * ld + i], B[(size_t)j * ld + i], s);
        s = warp_sum(s);
        if (lane == 0) sig[j] = s;
      }
      __syncthreads();
      if (warp == 0) {
        double best = -1.0;
        int bi = 0x7fffffff;
        for (int j = k + lane; j < r2; j += 32)
          if (sig[j] > best) { best = sig[j]; bi = j; }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (lane == 0) spiv = bi;
      }
      __syncthreads();
      const int pv = spiv;
      if (pv != k) {
        for (int i = tid; i < r1; i += NT) {
          const double t = B[(size_t)k * ld + i];
          B[(size_t)k * ld + i] = B[(size_t)pv * ld + i];
          B[(size_t)pv * ld + i] = t;
        }
        if (tid == 0) {
          const int t = perm[k];
          perm[k] = perm[pv];
          perm[pv] = t;
        }
      }
      __syncthreads();
      if (warp == 0) {  // reflector for column k, rows k..r1-1: H x = alpha e_1
        double s = 0.0;
        for (int i = k + lane; i < r1; i += 32) s = fma(B[(size_t)k * ld + i], B[(size_t)k * ld + i], s);
        s = warp_sum(s);
        const double x0 = B[(size_t)k * ld + k];
        const double nrm = sqrt(s);
        const double alpha = (x0 >= 0.0) ? -nrm : nrm;
        for (int i = k + lane; i < r1; i += 32) hv[i] = (i == k) ? x0 - alpha : B[(size_t)k * ld + i];
        if (lane == 0) {
          salpha = alpha;
          svn2 = s - x0 * x0 + (x0 - alpha) * (x0 - alpha);
        }
      }
      __syncthreads();
      const double vn2 = svn2;
      if (vn2 > 0.0) {
        for (int j = k + 1 + warp; j < r2; j += nw) {
          double w = 0.0;
          for (int i = k + lane; i < r1; i += 32) w = fma(hv[i], B[(size_t)j * ld + i], w);
          w = warp_sum(w);
          const double f = 2.0 * w / vn2;
          for (int i = k + lane; i < r1; i += 32) B[(size_t)j * ld + i] = fma(-f, hv[i], B[(size_t)j * ld + i]);
        }
        for (int i = k + tid; i < r1; i += NT) B[(size_t)k * ld + i] = (i == k) ? salpha : 0.0;
      }
      __syncthreads();
    }
    // ---- one-sided Jacobi on the rows of R (row r: B[c ld + r], c < r2)
    const double tiny2 = 256.0 * 1.2325951644078309e-32 * sfro;
    int sw = 0;
    bool conv = false;
    for (; sw < T2C_MAX_SWEEPS && !conv; ++sw) {
      for (int r = warp; r < rr; r += nw) {
        double s = 0.0;
        for (int c = lane; c < r2; c += 32) s = fma(B[(size_t)c * ld + r], B[(size_t)c * ld + r], s);
        s = warp_sum(s);
        if (lane == 0) sig[r] = s;
      }
      if (tid == 0) srot = 0;
      __syncthreads();
      for (int k = tid; k < rr; k += NT) {  // de Rijk: decreasing-norm visiting order
        const double v = sig[k];
        int q = 0;
        for (int j = 0; j < rr; ++j) q += (sig[j] > v) || (sig[j] == v && j < k);
        ord[q] = k;
      }
      if (tid == 0 && mr > rr) ord[rr] = rr;  // the virtual zero row
      __syncthreads();
      for (int st = 0; st < mr - 1; ++st) {
        for (int k = warp; k < mr / 2; k += nw) {
          const int pr = ord[t2c_rr(k, st, mr)], qr = ord[t2c_rr(mr - 1 - k, st, mr)];
          if (pr >= rr || qr >= rr) continue;
          double al = 0.0, be = 0.0, ga = 0.0;
          for (int c = lane; c < r2; c += 32) {
            const double x = B[(size_t)c * ld + pr], y = B[(size_t)c * ld + qr];
            al = fma(x, x, al);
            be = fma(y, y, be);
            ga = fma(x, y, ga);
          }
          al = warp_sum(al);
          be = warp_sum(be);
          ga = warp_sum(ga);
          if (al > tiny2 && be > tiny2 && fabs(ga) > p.tol * sqrt(al * be)) {
            const double zeta = (be - al) / (2.0 * ga);
            const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double c = rsqrt(1.0 + t * t), s = c * t;
            for (int cc = lane; cc < r2; cc += 32) {
              const double x = B[(size_t)cc * ld + pr], y = B[(size_t)cc * ld + qr];
              B[(size_t)cc * ld + pr] = c * x - s * y;
              B[(size_t)cc * ld + qr] = s * x + c * y;
            }
            if (lane == 0) atomicAdd(&srot, 1);
          }
        }
        __syncthreads();
      }
      conv = (srot == 0);
      __syncthreads();
    }
    // sigma_r = ||row r||, descending order (ties: lower row first)
    for (int r = warp; r < rr; r += nw) {
      double s = 0.0;
      for (int c = lane; c < r2; c += 32) s = fma(B[(size_t)c * ld + r], B[(size_t)c * ld + r], s);
      s = warp_sum(s);
      if (lane == 0) sig[r] = sqrt(s);
    }
    __syncthreads();
    for (int k = tid; k < rr; k += NT) {
      const double v = sig[k];
      int q = 0;
      for (int j = 0; j < rr; ++j) q += (sig[j] > v) || (sig[j] == v && j < k);
      ord[q] = k;
    }
    __syncthreads();
    double* Us = p.Us + (size_t)m * r2 * r1;
    double* Vs = p.Vs + (size_t)m * r2 * r2;
    double* sg = p.sg + (size_t)m * r2;
    int keep = 0;
    for (int j = 0; j < rr; ++j) keep += sig[ord[j]] > p.thr;
    // kept triplets, one warp each: v = P w / sigma; u = B v / sigma from the original slice
    // (rows of Bt, gathered through P), renormalised; sign rule on u (largest |.| positive)
    for (int j = warp; j < keep; j += nw) {
      const int r = ord[j];
      const double s = sig[r], inv = 1.0 / s;
      double* uo = Us + (size_t)j * r1;
      double un = 0.0;
      double best = -1.0;
      double bval = 0.0;
      for (int a = 0; a < r1; ++a) {
        const double* brow = Bm + (size_t)a * r2;
        double acc = 0.0;
        for (int c = lane; c < r2; c += 32) acc = fma(brow[perm[c]], B[(size_t)c * ld + r], acc);
        acc = warp_sum(acc) * inv * inv;  // (B P w)_a / sigma^2 = (B v)_a / sigma
        if (lane == 0) uo[a] = acc;
        un = fma(acc, acc, un);
        const double aa = fabs(acc);
        if (aa > best) { best = aa; bval = acc; }  // first maximum: lowest index on ties
      }
      const double sgn = ((bval < 0.0) ? -1.0 : 1.0) * (un > 0.0 ? 1.0 / sqrt(un) : 0.0);
      __syncwarp();
      __threadfence_block();
      for (int a = lane; a < r1; a += 32) uo[a] *= sgn;
      const double vs = (bval < 0.0 ? -inv : inv);
      double* vo = Vs + (size_t)j * r2;
      for (int c = lane; c < r2; c += 32) vo[perm[c]] = vs * B[(size_t)c * ld + r];
      if (lane == 0) sg[j] = s;
    }
    __syncthreads();
    if (tid == 0) {
      p.cnt[m] = keep;
      p.sweeps[m] = conv ? sw : -1;
      double d = 0.0;
      for (int j = rr - 1; j >= keep; --j) d = fma(sig[ord[j]], sig[ord[j]], d);
      p.drop[m] = d;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- large slices
// Slices too large for shared memory: block one-sided Jacobi with the slice in global
// memory (column-major per slice, L2-resident working set).  One-sided rotations only
// mix the two columns involved, so a block pair (I, J) of CB columns each is loaded
// into shared memory, swept once with the in-CTA one-sided Jacobi, and written back;
// the blocks meet in round-robin order, an outer sweep covers every column pair.
struct T2CBlockParams {
  const double* Bo;  // original slices, column-major: Bo[(m r2 + b) r1 + a] = beta[a][b][m]
  double* Bw;        // working copy (rotated in place), same layout
  int r1, r2, r3, ldp, CB, nb;  // ldp: smem column pitch (odd); nb: even block count
  double thr, tol;
  double* Us;
  double* Vs;
  double* sg;
  int* cnt;
  int* sweeps;
  double* drop;
};

template <int NT>
__global__ void __launch_bounds__(NT) t2c_slice_block_kernel(T2CBlockParams p) {
  extern __shared__ double sbk[];
  const int r1 = p.r1, r2 = p.r2, ld = p.ldp, CB = p.CB, nb = p.nb;
  double* P = sbk;                              // 2 CB columns, pitch ld
  double* sig = P + (size_t)2 * CB * ld;        // r2
  int* ord = reinterpret_cast<int*>(sig + r2);  // r2
  __shared__ int srot;
  __shared__ double sfro;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = NT / 32;
  for (int m = blockIdx.x; m < p.r3; m += gridDim.x) {
    const double* Bo = p.Bo + (size_t)m * r2 * r1;
    double* Bw = p.Bw + (size_t)m * r2 * r1;
    for (int e = tid; e < r1 * r2; e += NT) Bw[e] = Bo[e];
    if (warp == 0) {  // ||B||_F^2 (fixed order)
      double s = 0.0;
      for (int e = lane; e < r1 * r2; e += 32) s = fma(Bo[e], Bo[e], s);
      s = warp_sum(s);
      if (lane == 0) sfro = s;
    }
    __syncthreads();
    const double tiny2 = 256.0 * 1.2325951644078309e-32 * sfro;
    int sw = 0;
    bool conv = false;
    for (; sw < T2C_MAX_SWEEPS && !conv; ++sw) {
      // de Rijk pivoting: blocks are formed over the columns in decreasing-norm order
      for (int k = warp; k < r2; k += nw) {
        double s = 0.0;
        for (int i = lane; i < r1; i += 32) s = fma(Bw[(size_t)k * r1 + i], Bw[(size_t)k * r1 + i], s);
        s = warp_sum(s);
        if (lane == 0) sig[k] = s;
      }
      if (tid == 0) srot = 0;
      __syncthreads();
      for (int k = tid; k < r2; k += NT) {
        const double v = sig[k];
        int r = 0;
        for (int j = 0; j < r2; ++j) r += (sig[j] > v) || (sig[j] == v && j < k);
        ord[r] = k;
      }
      __syncthreads();
      for (int rd = 0; rd < nb - 1; ++rd) {
        for (int k = 0; k < nb / 2; ++k) {
          const int b1 = t2c_rr(k, rd, nb), b2 = t2c_rr(nb - 1 - k, rd, nb);
          const int I = min(b1, b2), J = max(b1, b2);
          // local column l < CB -> global I CB + l, else J CB + (l - CB); beyond r2 -> zero
          for (int e = tid; e < 2 * CB * ld; e += NT) {
            const int l = e / ld, a = e % ld;
            const int pos = l < CB ? I * CB + l : J * CB + (l - CB);
            P[e] = (a < r1 && pos < r2) ? Bw[(size_t)ord[pos] * r1 + a] : 0.0;
          }
          __syncthreads();
          const int m2 = 2 * CB;
          for (int st = 0; st < m2 - 1; ++st) {
            for (int q = warp; q < CB; q += nw) {
              const int c1 = t2c_rr(q, st, m2), c2 = t2c_rr(m2 - 1 - q, st, m2);
              double* bp = P + (size_t)min(c1, c2) * ld;
              double* bq = P + (size_t)max(c1, c2) * ld;
              double al = 0.0, be = 0.0, ga = 0.0;
              for (int i = lane; i < r1; i += 32) {
                const double x = bp[i], y = bq[i];
                al = fma(x, x, al);
                be = fma(y, y, be);
                ga = fma(x, y, ga);
              }
              al = warp_sum(al);
              be = warp_sum(be);
              ga = warp_sum(ga);
              if (al > tiny2 && be > tiny2 && fabs(ga) > p.tol * sqrt(al * be)) {
                const double zeta = (be - al) / (2.0 * ga);
                const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = rsqrt(1.0 + t * t), s = c * t;
                for (int i = lane; i < r1; i += 32) {
                  const double x = bp[i], y = bq[i];
                  bp[i] = c * x - s * y;
                  bq[i] = s * x + c * y;
                }
                if (lane == 0) atomicAdd(&srot, 1);
              }
            }
            __syncthreads();
          }
          for (int e = tid; e < 2 * CB * ld; e += NT) {
            const int l = e / ld, a = e % ld;
            const int pos = l < CB ? I * CB + l : J * CB + (l - CB);
            if (a < r1 && pos < r2) Bw[(size_t)ord[pos] * r1 + a] = P[e];
          }
          __syncthreads();
        }
      }
      conv = (srot == 0);
      __syncthreads();
    }
    // sigma_k = ||b_k||, descending order, kept count (as in the shared-memory kernel)
    for (int k = warp; k < r2; k += nw) {
      double s = 0.0;
      for (int i = lane; i < r1; i += 32) s = fma(Bw[(size_t)k * r1 + i], Bw[(size_t)k * r1 + i], s);
      s = warp_sum(s);
      if (lane == 0) sig[k] = sqrt(s);
    }
    __syncthreads();
    for (int k = tid; k < r2; k += NT) {
      const double v = sig[k];
      int r = 0;
      for (int j = 0; j < r2; ++j) r += (sig[j] > v) || (sig[j] == v && j < k);
      ord[r] = k;
    }
    __syncthreads();
    int keep = 0;
    for (int j = 0; j < r2; ++j) keep += sig[ord[j]] > p.thr;
    double* Us = p.Us + (size_t)m * r2 * r1;
    double* Vs = p.Vs + (size_t)m * r2 * r2;
    double* sg = p.sg + (size_t)m * r2;
    // u_j = sgn b_k / sigma (largest-|.| entry positive, lowest index on ties)
    for (int j = warp; j < keep; j += nw) {
      const int k = ord[j];
      const double* bk = Bw + (size_t)k * r1;
      double best = -1.0;
      int bi = 0x7fffffff;
      for (int i = lane; i < r1; i += 32) {
        const double a = fabs(bk[i]);
        if (a > best || (a == best && i < bi)) {
          best = a;
          bi = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      const double sc = ((bk[bi] < 0.0) ? -1.0 : 1.0) / sig[k];
      for (int i = lane; i < r1; i += 32) Us[(size_t)j * r1 + i] = sc * bk[i];
      if (lane == 0) sg[j] = sig[k];
    }
    __syncthreads();
    // v_j = B_orig^T u_j / sigma_j, 8 u's per pass staged in shared memory (the pair buffer),
    // one warp per column b of the original slice (coalesced), renormalised at the end
    const int JT = min(8, 2 * CB * ld / max(r1, 1));
    for (int j0 = 0; j0 < keep; j0 += JT) {
      const int jn = min(JT, keep - j0);
      for (int e = tid; e < jn * r1; e += NT) P[e] = Us[(size_t)j0 * r1 + e];
      __syncthreads();
      for (int b = warp; b < r2; b += nw) {
        const double* ob = Bo + (size_t)b * r1;
        double acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.0;
        for (int i = lane; i < r1; i += 32) {
          const double x = ob[i];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j < jn) acc[j] = fma(x, P[(size_t)j * r1 + i], acc[j]);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const double v = warp_sum(acc[j]);
          if (lane == 0 && j < jn) Vs[(size_t)(j0 + j) * r2 + b] = v / sg[j0 + j];
        }
      }
      __syncthreads();
    }
    for (int j = warp; j < keep; j += nw) {
      double* vo = Vs + (size_t)j * r2;
      double vn = 0.0;
      for (int b = lane; b < r2; b += 32) vn = fma(vo[b], vo[b], vn);
      vn = warp_sum(vn);
      const double rv = vn > 0.0 ? 1.0 / sqrt(vn) : 0.0;
      __syncwarp();
      for (int b = lane; b < r2; b += 32) vo[b] *= rv;
    }
    if (tid == 0) {
      p.cnt[m] = keep;
      p.sweeps[m] = conv ? sw : -1;
      double d = 0.0;
      for (int j = r2 - 1; j >= keep; --j) d = fma(sig[ord[j]], sig[ord[j]], d);
      p.drop[m] = d;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- large slices, QR-preconditioned
// The Drmac-Veselic preconditioning of t2c_slice_qr_kernel for slices beyond shared memory:
// the block one-sided Jacobi above needs ~25 sweeps on cfg 2 / cfg 4 core slices.
//   1. Householder QR with column pivoting B P = Q R on the global working copy (one CTA
//      per slice; warp per column for the norms and the reflector, Q never formed);
//   2. R^T (columns = the rows of R, length r2) into a second buffer, and the block
//      one-sided Jacobi of t2c_slice_block_kernel on its columns (same pair-buffer rounds,
//      de Rijk order, tolerance on rows of length r2);
//   3. sigma_k = ||w_k||, v_k = P w_k / sigma_k, u_k = B v_k / sigma_k from the original
//      slice (eight u's per pass over B, columns gathered through P), renormalised, sign
//      rule on u - the shared-memory QR kernel's outputs and conventions.
struct T2CBlockQRParams {
  const double* Bo;  // original slices, column-major: Bo[(m r2 + b) r1 + a] = beta[a][b][m]
  double* Bw;        // QR working copy, same layout
  double* Rt;        // per slice: R^T, r2 rows x rr columns (column-major, ld r2)
  int r1, r2, r3, ldp, CB, nb;  // ldp: smem pitch >= r2 (odd); nb: even block count over rr
  double thr, tol;
  double* Us;
  double* Vs;
  double* sg;
  int* cnt;
  int* sweeps;
  double* drop;
};

template <int NT>
__global__ void __launch_bounds__(NT) t2c_slice_blockqr_kernel(T2CBlockQRParams p) {
  extern __shared__ double sbq[];
  const int r1 = p.r1, r2 = p.r2, ld = p.ldp, CB = p.CB, nb = p.nb;
  const int rr = min(r1, r2);
  double* P = sbq;                              // 2 CB columns, pitch ld (QR: Householder vector)
  double* sig = P + (size_t)2 * CB * ld;        // r2
  int* ord = reinterpret_cast<int*>(sig + r2);  // r2
  int* perm = ord + r2;                         // r2
  __shared__ int srot, spiv;
  __shared__ double sfro, salpha, svn2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = NT / 32;
  for (int m = blockIdx.x; m < p.r3; m += gridDim.x) {
    const double* Bo = p.Bo + (size_t)m * r2 * r1;
    double* B = p.Bw + (size_t)m * r2 * r1;
    double* W = p.Rt + (size_t)m * r2 * rr;
    for (int e = tid; e < r1 * r2; e += NT) B[e] = Bo[e];
    for (int j = tid; j < r2; j += NT) perm[j] = j;
    if (warp == 0) {
      double s = 0.0;
      for (int e = lane; e < r1 * r2; e += 32) s = fma(Bo[e], Bo[e], s);
      s = warp_sum(s);
      if (lane == 0) sfro = s;
    }
    __syncthreads();
    // ---- 1. Householder QR with column pivoting (largest remaining norm, lowest index on ties)
    double* hv = P;
    for (int k = 0; k < rr; ++k) {
      for (int j = k + warp; j < r2; j += nw) {
        double s = 0.0;
        for (int i = k + lane; i < r1; i += 32) s = fma(B[(size_t)j * r1 + i], B[(size_t)j * r1 + i], s);
        s = warp_sum(s);
        if (lane == 0) sig[j] = s;
      }
      __syncthreads();
      if (warp == 0) {
        double best = -1.0;
        int bi = 0x7fffffff;
        for (int j = k + lane; j < r2; j += 32)
          if (sig[j] > best) { best = sig[j]; bi = j; }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (lane == 0) spiv = bi;
      }
      __syncthreads();
      const int pv = spiv;
      if (pv != k) {
        for (int i = tid; i < r1; i += NT) {
          const double t = B[(size_t)k * r1 + i];
          B[(size_t)k * r1 + i] = B[(size_t)pv * r1 + i];
          B[(size_t)pv * r1 + i] = t;
        }
        if (tid == 0) {
          const int t = perm[k];
          perm[k] = perm[pv];
          perm[pv] = t;
        }
      }
      __syncthreads();
      if (warp == 0) {  // reflector for column k, rows k..r1-1: H x = alpha e_1
        double s = 0.0;
        for (int i = k + lane; i < r1; i += 32) s = fma(B[(size_t)k * r1 + i], B[(size_t)k * r1 + i], s);
        s = warp_sum(s);
        const double x0 = B[(size_t)k * r1 + k];
        const double nrm = sqrt(s);
        const double alpha = (x0 >= 0.0) ? -nrm : nrm;
        for (int i = k + lane; i < r1; i += 32) hv[i] = (i == k) ? x0 - alpha : B[(size_t)k * r1 + i];
        if (lane == 0) {
          salpha = alpha;
          svn2 = s - x0 * x0 + (x0 - alpha) * (x0 - alpha);
        }
      }
      __syncthreads();
      const double vn2 = svn2;
      if (vn2 > 0.0) {
        for (int j = k + 1 + warp; j < r2; j += nw) {
          double w = 0.0;
          for (int i = k + lane; i < r1; i += 32) w = fma(hv[i], B[(size_t)j * r1 + i], w);
          w = warp_sum(w);
          const double f = 2.0 * w / vn2;
          for (int i = k + lane; i < r1; i += 32) B[(size_t)j * r1 + i] = fma(-f, hv[i], B[(size_t)j * r1 + i]);
        }
        for (int i = k + tid; i < r1; i += NT) B[(size_t)k * r1 + i] = (i == k) ? salpha : 0.0;
      }
      __syncthreads();
    }
    // ---- 2. W = R^T (column r = row r of R: W[r r2 + c] = R[r][c], zero left of the diagonal)
    for (int e = tid; e < r2 * rr; e += NT) {
      const int r = e / r2, c = e % r2;
      W[e] = (c >= r) ? B[(size_t)c * r1 + r] : 0.0;
    }
    __syncthreads();
    // block one-sided Jacobi on the rr columns of W (length r2)
    const int rows = r2, cols = rr;
    const double tiny2 = 256.0 * 1.2325951644078309e-32 * sfro;
    int sw = 0;
    bool conv = false;
    for (; sw < T2C_MAX_SWEEPS && !conv; ++sw) {
      for (int k = warp; k < cols; k += nw) {
        double s = 0.0;
        for (int i = lane; i < rows; i += 32) s = fma(W[(size_t)k * rows + i], W[(size_t)k * rows + i], s);
        s = warp_sum(s);
        if (lane == 0) sig[k] = s;
      }
      if (tid == 0) srot = 0;
      __syncthreads();
      for (int k = tid; k < cols; k += NT) {  // de Rijk: decreasing-norm order
        const double v = sig[k];
        int r = 0;
        for (int j = 0; j < cols; ++j) r += (sig[j] > v) || (sig[j] == v && j < k);
        ord[r] = k;
      }
      __syncthreads();
      for (int rd = 0; rd < nb - 1; ++rd) {
        for (int k = 0; k < nb / 2; ++k) {
          const int b1 = t2c_rr(k, rd, nb), b2 = t2c_rr(nb - 1 - k, rd, nb);
          const int I = min(b1, b2), J = max(b1, b2);
          for (int e = tid; e < 2 * CB * ld; e += NT) {
            const int l = e / ld, a = e % ld;
            const int pos = l < CB ? I * CB + l : J * CB + (l - CB);
            P[e] = (a < rows && pos < cols) ? W[(size_t)ord[pos] * rows + a] : 0.0;
          }
          __syncthreads();
          const int m2 = 2 * CB;
          for (int st = 0; st < m2 - 1; ++st) {
            for (int q = warp; q < CB; q += nw) {
              const int c1 = t2c_rr(q, st, m2), c2 = t2c_rr(m2 - 1 - q, st, m2);
              double* bp = P + (size_t)min(c1, c2) * ld;
              double* bq = P + (size_t)max(c1, c2) * ld;
              double al = 0.0, be = 0.0, ga = 0.0;
              for (int i = lane; i < rows; i += 32) {
                const double x = bp[i], y = bq[i];
                al = fma(x, x, al);
                be = fma(y, y, be);
                ga = fma(x, y, ga);
              }
              al = warp_sum(al);
              be = warp_sum(be);
              ga = warp_sum(ga);
              if (al > tiny2 && be > tiny2 && fabs(ga) > p.tol * sqrt(al * be)) {
                const double zeta = (be - al) / (2.0 * ga);
                const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = rsqrt(1.0 + t * t), s = c * t;
                for (int i = lane; i < rows; i += 32) {
                  const double x = bp[i], y = bq[i];
                  bp[i] = c * x - s * y;
                  bq[i] = s * x + c * y;
                }
                if (lane == 0) atomicAdd(&srot, 1);
              }
            }
            __syncthreads();
          }
          for (int e = tid; e < 2 * CB * ld; e += NT) {
            const int l = e / ld, a = e % ld;
            const int pos = l < CB ? I * CB + l : J * CB + (l - CB);
            if (a < rows && pos < cols) W[(size_t)ord[pos] * rows + a] = P[e];
          }
          __syncthreads();
        }
      }
      conv = (srot == 0);
      __syncthreads();
    }
    // ---- 3. sigma_k = ||w_k||, descending order (ties: lower index), kept count
    for (int k = warp; k < cols; k += nw) {
      double s = 0.0;
      for (int i = lane; i < rows; i += 32) s = fma(W[(size_t)k * rows + i], W[(size_t)k * rows + i], s);
      s = warp_sum(s);
      if (lane == 0) sig[k] = sqrt(s);
    }
    __syncthreads();
    for (int k = tid; k < cols; k += NT) {
      const double v = sig[k];
      int r = 0;
      for (int j = 0; j < cols; ++j) r += (sig[j] > v) || (sig[j] == v && j < k);
      ord[r] = k;
    }
    __syncthreads();
    int keep = 0;
    for (int j = 0; j < cols; ++j) keep += sig[ord[j]] > p.thr;
    double* Us = p.Us + (size_t)m * r2 * r1;
    double* Vs = p.Vs + (size_t)m * r2 * r2;
    double* sg = p.sg + (size_t)m * r2;
    // u_j = B v_j / sigma_j = (B P) w_j / sigma_j^2, eight at a time: w's staged in the pair
    // buffer (original column order: Pw[perm[c]] = w[c]), one thread per row a of B
    const int JT = min(8, 2 * CB * ld / max(r2, 1));
    for (int j0 = 0; j0 < keep; j0 += JT) {
      const int jn = min(JT, keep - j0);
      for (int e = tid; e < jn * r2; e += NT) {
        const int jj = e / r2, c = e % r2;
        P[(size_t)jj * r2 + perm[c]] = W[(size_t)ord[j0 + jj] * rows + c];
      }
      __syncthreads();
      for (int a = tid; a < r1; a += NT) {
        double acc[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) acc[jj] = 0.0;
        for (int b = 0; b < r2; ++b) {
          const double x = Bo[(size_t)b * r1 + a];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj)
            if (jj < jn) acc[jj] = fma(x, P[(size_t)jj * r2 + b], acc[jj]);
        }
#pragma unroll
        for (int jj = 0; jj < 8; ++jj)
          if (jj < jn) {
            const double s = sig[ord[j0 + jj]];
            Us[(size_t)(j0 + jj) * r1 + a] = acc[jj] / (s * s);
          }
      }
      __syncthreads();
    }
    // renormalise u, sign rule (largest |u_a| positive, lowest index on ties), v = +-P w / sigma
    for (int j = warp; j < keep; j += nw) {
      double* uo = Us + (size_t)j * r1;
      double un = 0.0, best = -1.0;
      int bi = 0x7fffffff;
      for (int a = lane; a < r1; a += 32) {
        const double x = uo[a];
        un = fma(x, x, un);
        const double ax = fabs(x);
        if (ax > best || (ax == best && a < bi)) { best = ax; bi = a; }
      }
      un = warp_sum(un);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      const double bval = uo[bi];
      const double sgn = ((bval < 0.0) ? -1.0 : 1.0) * (un > 0.0 ? 1.0 / sqrt(un) : 0.0);
      __syncwarp();
      for (int a = lane; a < r1; a += 32) uo[a] *= sgn;
      const int r = ord[j];
      const double s = sig[r];
      const double vs = (bval < 0.0 ? -1.0 : 1.0) / s;
      double* vo = Vs + (size_t)j * r2;
      for (int c = lane; c < r2; c += 32) vo[perm[c]] = vs * W[(size_t)r * rows + c];
      if (lane == 0) sg[j] = s;
    }
    __syncthreads();
    if (tid == 0) {
      p.cnt[m] = keep;
      p.sweeps[m] = conv ? sw : -1;
      double d = 0.0;
      for (int j = cols - 1; j >= keep; --j) d = fma(sig[ord[j]], sig[ord[j]], d);
      p.drop[m] = d;
    }
    __syncthreads();
  }
}

// Bc[(m r2 + b) r1 + a] = beta[(a r2 + b) r3 + m]  (slice-major, column-major copy)
__global__ void t2c_transpose_cm_kernel(const double* beta, int r1, int r2, int r3, double* Bc) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tot = (int64_t)r1 * r2 * r3;
  if (e >= tot) return;
  const int m = (int)(e % r3);
  const int64_t ab = e / r3;
  const int a = (int)(ab / r2), b = (int)(ab % r2);
  Bc[((int64_t)m * r2 + b) * r1 + a] = beta[e];
}

// Bt[(m r1 + a) r2 + b] = beta[(a r2 + b) r3 + m]  (slice-major copy)
__global__ void t2c_transpose_kernel(const double* beta, int r1, int r2, int r3, double* Bt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tot = (int64_t)r1 * r2 * r3;
  if (e >= tot) return;
  const int64_t ab = e / r3;
  const int m = (int)(e % r3);
  Bt[(int64_t)m * r1 * r2 + ab] = beta[e];
}

// compaction: term t of slice m -> column off[m] + t
__global__ void t2c_compact_kernel(const double* Us, const double* Vs, const double* sg, const int* cnt,
                                   const int64_t* off, int r1, int r2, int r3, double* Uc, int64_t ldu,
                                   double* Vc, int64_t ldv, double* w, int* slice) {
  const int m = blockIdx.x;
  if (m >= r3) return;
  const int keep = cnt[m];
  const int64_t o = off[m];
  for (int e = threadIdx.x; e < keep * (r1 + r2 + 1); e += blockDim.x) {
    const int j = e / (r1 + r2 + 1), i = e % (r1 + r2 + 1);
    if (i < r1) Uc[(o + j) * ldu + i] = Us[((size_t)m * r2 + j) * r1 + i];
    else if (i < r1 + r2) Vc[(o + j) * ldv + (i - r1)] = Vs[((size_t)m * r2 + j) * r2 + (i - r1)];
    else {
      w[o + j] = sg[(size_t)m * r2 + j];
      slice[o + j] = m;
    }
  }
}

// F3[:, j] = Z3[:, slice[j]]
__global__ void t2c_gather_kernel(const double* Z3, int64_t ldz, int n, const int* slice, int64_t R, double* F3,
                                  int64_t ldf) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * R) return;
  const int64_t j = e / n;
  const int i = (int)(e % n);
  F3[j * ldf + i] = Z3[(int64_t)slice[j] * ldz + i];
}

}  // namespace rhosvd

using namespace rhosvd;

struct rhosvd_cp {
  int64_t R = 0, n = 0, ldf = 0;
  int32_t r[3] = {0, 0, 0};
  double* F[3] = {nullptr, nullptr, nullptr};   // n x R, col-major, ld ldf
  double* Ucore = nullptr;                      // r1 x R (ld ldu)
  double* Vcore = nullptr;                      // r2 x R (ld ldv)
  int64_t ldu = 0, ldv = 0;
  double* w = nullptr;
  int* slice = nullptr;
  double eps = 0, thr = 0, err2 = 0;
  int max_sweeps = 0;
};

static void cp_release(rhosvd_cp* c) {
  if (!c) return;
  for (int l = 0; l < 3; ++l) cudaFree(c->F[l]);
  cudaFree(c->Ucore);
  cudaFree(c->Vcore);
  cudaFree(c->w);
  cudaFree(c->slice);
  delete c;
}

extern "C" {

int rhosvd_t2c(const rhosvd_result* res, double eps_rel, rhosvd_stream stream, rhosvd_cp** out) {
  if (!out) return fail(RHOSVD_EINVAL, "out is null");
  *out = nullptr;
  if (!res || !(eps_rel >= 0.0 && eps_rel < 1.0)) return fail(RHOSVD_EINVAL, "t2c: need a result and 0 <= eps < 1");
  RH_CHECK(device_guard());
  if (!res->beta_valid) return fail(RHOSVD_EINVAL, "t2c: RHOSVD_F_ROOT_ONLY_CORE result on a rank != 0 holds no core");
  cudaStream_t st = (cudaStream_t)stream;
  const int r1 = res->ranks[0], r2 = res->ranks[1], r3 = res->ranks[2];
  auto* cp = new rhosvd_cp();
  cp->n = res->n;
  cp->r[0] = r1; cp->r[1] = r2; cp->r[2] = r3;
  cp->eps = eps_rel * res->rep.beta_norm;
  const int q = std::min(r1, r2);
  cp->thr = (r3 > 0 && q > 0) ? cp->eps / (r3 * std::sqrt((double)q)) : 0.0;
  const int64_t ldf = round_up(std::max<int64_t>(res->n, 1), 16);
  cp->ldf = ldf;
  if ((int64_t)r1 * r2 * r3 == 0) {
    *out = cp;
    return RHOSVD_OK;
  }
  const int ldb = r1 | 1;
  const int m2 = r2 + (r2 & 1);
  const size_t smem = ((size_t)ldb * m2 + m2) * sizeof(double) + (size_t)m2 * sizeof(int) + 64;
  const bool small = smem <= 220 * 1024;
  // large slices: block width CB with a 2 CB-column pair buffer in shared memory
  int CB = 32;
  while (CB > 4 && (size_t)2 * CB * ldb * sizeof(double) + (size_t)r2 * 12 + 64 > 200 * 1024) CB /= 2;
  const size_t smem_blk = (size_t)2 * CB * ldb * sizeof(double) + (size_t)r2 * (sizeof(double) + sizeof(int)) + 64;
  if (!small && (smem_blk > 220 * 1024 || r1 * 8 > 2 * CB * ldb)) {
    cp_release(cp);
    return fail(RHOSVD_EINVAL, "t2c: core slices of " + std::to_string(r1) + " x " + std::to_string(r2) +
                                   " are too large (r1 > ~3000)");
  }
  // per-slice scratch
  double *Us = nullptr, *Vs = nullptr, *sg = nullptr, *drop = nullptr, *Bt = nullptr;
  int *cnt = nullptr, *sweeps = nullptr;
  int64_t* off = nullptr;
  auto cleanup = [&]() {
    cudaFree(Us); cudaFree(Vs); cudaFree(sg); cudaFree(cnt); cudaFree(sweeps); cudaFree(off); cudaFree(drop); cudaFree(Bt);
  };
  if (cudaMalloc(&Us, (size_t)r3 * r2 * r1 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&Vs, (size_t)r3 * r2 * r2 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&sg, (size_t)r3 * r2 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&cnt, (size_t)r3 * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&sweeps, (size_t)r3 * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&off, (size_t)r3 * sizeof(int64_t)) != cudaSuccess ||
      cudaMalloc(&drop, (size_t)r3 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&Bt, (size_t)r1 * r2 * r3 * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    cleanup();
    cp_release(cp);
    return fail(RHOSVD_ENOMEM, "t2c scratch");
  }
  // one-sided Jacobi stopping rule |b_p^T b_q| <= tol ||b_p|| ||b_q||, tol = 4 sqrt(r1) u
  static const double tol_mult = [] {
    const char* e = getenv("RHOSVD_T2C_TOL");
    return e ? atof(e) : 4.0;
  }();
  const double tol = tol_mult * std::sqrt((double)std::max(r1, 1)) * 1.1102230246251565e-16;
  if (small) {
    const int64_t tot = (int64_t)r1 * r2 * r3;
    t2c_transpose_kernel<<<(unsigned)cdiv(tot, 256), 256, 0, st>>>(res->beta, r1, r2, r3, Bt);
  }
  cudaError_t e = cudaSuccess;
  if (small) {
    // QR-preconditioned kernel when its extra shared memory fits (RHOSVD_T2C_QR=0: plain);
    // its row Jacobi works on rows of length r2, so the tolerance uses max(r1, r2)
    static const bool qr_on = [] {
      const char* e2 = getenv("RHOSVD_T2C_QR");
      return !(e2 && e2[0] == '0');
    }();
    const size_t smem_qr = smem + (size_t)ldb * sizeof(double) + (size_t)m2 * sizeof(int);
    const bool use_qr = qr_on && smem_qr <= 220 * 1024;
    const double tol_qr = tol_mult * std::sqrt((double)std::max(std::max(r1, r2), 1)) * 1.1102230246251565e-16;
    T2CParams tp{Bt, r1, r2, r3, ldb, cp->thr, use_qr ? tol_qr : tol, Us, Vs, sg, cnt, sweeps, drop};
    static const cudaError_t attr =
        cudaFuncSetAttribute(t2c_slice_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    // QR kernel block size (RHOSVD_T2C_QR_THREADS): more warps = fewer column pairs per warp
    // per Jacobi step (the per-pair dot-product latency is the cost)
    static const int qr_nt = [] {
      const char* e2 = getenv("RHOSVD_T2C_QR_THREADS");
      const int v = e2 ? atoi(e2) : 1024;  // cfg 3: 256 17.6 ms, 512 12.6, 1024 11.2
      return (v == 256 || v == 512) ? v : 1024;
    }();
    static const cudaError_t attr_q1 =
        cudaFuncSetAttribute(t2c_slice_qr_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    static const cudaError_t attr_q2 =
        cudaFuncSetAttribute(t2c_slice_qr_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    static const cudaError_t attr_q4 =
        cudaFuncSetAttribute(t2c_slice_qr_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    (void)attr;
    (void)attr_q1;
    (void)attr_q2;
    (void)attr_q4;
    const int qgrid = std::min(r3, 4 * num_sms());
    if (use_qr && qr_nt == 256)
      t2c_slice_qr_kernel<256><<<qgrid, 256, smem_qr, st>>>(tp);
    else if (use_qr && qr_nt == 1024)
      t2c_slice_qr_kernel<1024><<<qgrid, 1024, smem_qr, st>>>(tp);
    else if (use_qr)
      t2c_slice_qr_kernel<512><<<qgrid, 512, smem_qr, st>>>(tp);
    else
      t2c_slice_kernel<<<std::min(r3, 4 * num_sms()), T2C_THREADS, smem, st>>>(tp);
    e = cudaGetLastError();
  } else {
    // column-major slice copies: the original (for v = B^T u / sigma) and the working copy
    static const bool qr_big = [] {
      const char* e2 = getenv("RHOSVD_T2C_QR");
      return !(e2 && e2[0] == '0');
    }();
    const int rrq = std::min(r1, r2);
    const int ldq = r2 | 1;  // pair-buffer pitch of the R^T columns (length r2)
    int CBq = 32;
    while (CBq > 4 && (size_t)2 * CBq * ldq * sizeof(double) + (size_t)r2 * 16 + 64 > 200 * 1024) CBq /= 2;
    const size_t smem_q = (size_t)2 * CBq * ldq * sizeof(double) + (size_t)r2 * (sizeof(double) + 2 * sizeof(int)) + 64;
    const bool use_bqr = qr_big && smem_q <= 220 * 1024 && (size_t)2 * CBq * ldq >= (size_t)r1;
    double* Bw = nullptr;
    double* Rtq = nullptr;
    e = cudaMalloc(&Bw, (size_t)r1 * r2 * r3 * sizeof(double));
    if (e == cudaSuccess && use_bqr) e = cudaMalloc(&Rtq, (size_t)r2 * rrq * r3 * sizeof(double));
    if (e == cudaSuccess && use_bqr) {
      const int64_t tot = (int64_t)r1 * r2 * r3;
      t2c_transpose_cm_kernel<<<(unsigned)cdiv(tot, 256), 256, 0, st>>>(res->beta, r1, r2, r3, Bt);
      const int nbk = (int)cdiv(rrq, CBq);
      const double tol_qr = tol_mult * std::sqrt((double)std::max(std::max(r1, r2), 1)) * 1.1102230246251565e-16;
      T2CBlockQRParams bq{Bt, Bw, Rtq, r1, r2, r3, ldq, CBq, nbk + (nbk & 1), cp->thr, tol_qr, Us, Vs, sg, cnt, sweeps,
                          drop};
      static const cudaError_t attr3 =
          cudaFuncSetAttribute(t2c_slice_blockqr_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      (void)attr3;
      t2c_slice_blockqr_kernel<1024><<<std::min(r3, num_sms()), 1024, smem_q, st>>>(bq);
      e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      cudaFree(Rtq);
      cudaFree(Bw);
    } else if (e == cudaSuccess) {
      const int64_t tot = (int64_t)r1 * r2 * r3;
      t2c_transpose_cm_kernel<<<(unsigned)cdiv(tot, 256), 256, 0, st>>>(res->beta, r1, r2, r3, Bt);
      const int nbk = (int)cdiv(r2, CB);
      T2CBlockParams bp{Bt, Bw, r1, r2, r3, ldb, CB, nbk + (nbk & 1), cp->thr, tol, Us, Vs, sg, cnt, sweeps, drop};
      // block size (RHOSVD_T2C_BLK_THREADS, default 1024): one warp per column pair of a step
      static const int blk_nt = [] {
        const char* e2 = getenv("RHOSVD_T2C_BLK_THREADS");
        const int v = e2 ? atoi(e2) : 1024;
        return (v == 256 || v == 512) ? v : 1024;
      }();
      static const cudaError_t attr2a =
          cudaFuncSetAttribute(t2c_slice_block_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      static const cudaError_t attr2b =
          cudaFuncSetAttribute(t2c_slice_block_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      static const cudaError_t attr2c =
          cudaFuncSetAttribute(t2c_slice_block_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      (void)attr2a;
      (void)attr2b;
      (void)attr2c;
      const int bgrid = std::min(r3, num_sms());
      if (blk_nt == 256)
        t2c_slice_block_kernel<256><<<bgrid, 256, smem_blk, st>>>(bp);
      else if (blk_nt == 512)
        t2c_slice_block_kernel<512><<<bgrid, 512, smem_blk, st>>>(bp);
      else
        t2c_slice_block_kernel<1024><<<bgrid, 1024, smem_blk, st>>>(bp);
      e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      cudaFree(Bw);
    } else {
      cudaGetLastError();
      cudaFree(Rtq);
      cudaFree(Bw);
    }
  }
  std::vector<int> hc(r3), hs(r3);
  std::vector<double> hd(r3);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hc.data(), cnt, r3 * sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hd.data(), drop, r3 * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hs.data(), sweeps, r3 * sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    cleanup();
    cp_release(cp);
    return fail(RHOSVD_ECUDA, std::string("t2c slice kernel: ") + cudaGetErrorString(e));
  }
  std::vector<int64_t> ho(r3);
  int64_t R = 0;
  for (int m = 0; m < r3; ++m) {
    ho[m] = R;
    R += hc[m];
    if (hs[m] < 0) {
      cleanup();
      cp_release(cp);
      return fail(RHOSVD_ENOCONV, "t2c: one-sided Jacobi did not converge on slice " + std::to_string(m));
    }
    cp->max_sweeps = std::max(cp->max_sweeps, hs[m]);
  }
  cp->R = R;
  if (getenv("RHOSVD_DEBUG") && getenv("RHOSVD_DEBUG")[0] == '1') {  // sweep-count histogram
    std::vector<int> hist(T2C_MAX_SWEEPS + 1, 0);
    for (int m = 0; m < r3; ++m) hist[std::max(0, std::min(hs[m], T2C_MAX_SWEEPS))]++;
    fprintf(stderr, "[rhosvd dbg] t2c %s path, sweeps histogram:", small ? "smem" : "block");
    for (int k = 0; k <= T2C_MAX_SWEEPS; ++k)
      if (hist[k]) fprintf(stderr, " %d:%d", k, hist[k]);
    fprintf(stderr, "\n");
  }
  // exact error^2 (the slices are orthogonal in mode 3): the discarded energy, summed in slice order
  cp->err2 = 0.0;
  for (int m = 0; m < r3; ++m) cp->err2 += hd[m];
  cp->ldu = round_up(std::max(r1, 2), 2);
  cp->ldv = round_up(std::max(r2, 2), 2);
  const int64_t Rm = std::max<int64_t>(R, 1);
  bool ok = cudaMalloc(&cp->Ucore, (size_t)cp->ldu * Rm * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&cp->Vcore, (size_t)cp->ldv * Rm * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&cp->w, (size_t)Rm * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&cp->slice, (size_t)Rm * sizeof(int)) == cudaSuccess;
  for (int l = 0; l < 3 && ok; ++l) ok = cudaMalloc(&cp->F[l], (size_t)ldf * Rm * sizeof(double)) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    cleanup();
    cp_release(cp);
    return fail(RHOSVD_ENOMEM, "t2c outputs");
  }
  e = cudaMemsetAsync(cp->Ucore, 0, (size_t)cp->ldu * Rm * sizeof(double), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(cp->Vcore, 0, (size_t)cp->ldv * Rm * sizeof(double), st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(off, ho.data(), r3 * sizeof(int64_t), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) {
    cleanup();
    cp_release(cp);
    return fail(RHOSVD_ECUDA, cudaGetErrorString(e));
  }
  if (R > 0) {
    t2c_compact_kernel<<<r3, 256, 0, st>>>(Us, Vs, sg, cnt, off, r1, r2, r3, cp->Ucore, cp->ldu, cp->Vcore,
                                           cp->ldv, cp->w, cp->slice);
    // lift: F1 = Z1 U, F2 = Z2 V (DMMA GEMMs), F3 = Z3[:, slice]
    Scratch scr;
    const int rr[2] = {r1, r2};
    double* core_f[2] = {cp->Ucore, cp->Vcore};
    const int64_t ldc[2] = {cp->ldu, cp->ldv};
    for (int l = 0; l < 2; ++l) {
      GemmArgs g;
      g.M = res->n; g.N = R; g.K = rr[l];
      g.A = res->Z[l]; g.lda = res->ldz; g.a_k = false;
      g.B = core_f[l]; g.ldb = ldc[l]; g.b_k = true;
      g.C = cp->F[l]; g.ldc = ldf;
      int s = gemm(g, scr, st);
      if (s != RHOSVD_OK) {
        std::string msg = rhosvd_last_error();
        scr.release(st);
        cleanup();
        cp_release(cp);
        return fail(s, msg);
      }
    }
    t2c_gather_kernel<<<(unsigned)cdiv(res->n * R, 256), 256, 0, st>>>(res->Z[2], res->ldz, (int)res->n, cp->slice,
                                                                      R, cp->F[2], ldf);
    e = cudaStreamSynchronize(st);
    scr.release(st);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
      cleanup();
      cp_release(cp);
      return fail(RHOSVD_ECUDA, std::string("t2c lift: ") + cudaGetErrorString(e));
    }
  }
  cudaStreamSynchronize(st);
  cleanup();
  *out = cp;
  return RHOSVD_OK;
}

int rhosvd_cp_rank(const rhosvd_cp* cp, int64_t* R) {
  if (!cp || !R) return fail(RHOSVD_EINVAL, "null");
  *R = cp->R;
  return RHOSVD_OK;
}
int rhosvd_cp_factor(const rhosvd_cp* cp, int mode, const double** F, int64_t* ld) {
  if (!cp || !F || !ld || mode < 0 || mode > 2) return fail(RHOSVD_EINVAL, "bad args");
  *F = cp->F[mode];
  *ld = cp->ldf;
  return RHOSVD_OK;
}
int rhosvd_cp_core_factor(const rhosvd_cp* cp, int mode, const double** F, int64_t* ld) {
  if (!cp || !F || !ld || mode < 0 || mode > 1) return fail(RHOSVD_EINVAL, "bad args");
  *F = mode == 0 ? cp->Ucore : cp->Vcore;
  *ld = mode == 0 ? cp->ldu : cp->ldv;
  return RHOSVD_OK;
}
int rhosvd_cp_weights(const rhosvd_cp* cp, const double** w, const int32_t** slice) {
  if (!cp || !w || !slice) return fail(RHOSVD_EINVAL, "bad args");
  *w = cp->w;
  *slice = cp->slice;
  return RHOSVD_OK;
}
int rhosvd_cp_info(const rhosvd_cp* cp, double* eps_abs, double* thr, double* err2, int32_t* max_sweeps) {
  if (!cp || !eps_abs || !thr || !err2 || !max_sweeps) return fail(RHOSVD_EINVAL, "bad args");
  *eps_abs = cp->eps;
  *thr = cp->thr;
  *err2 = cp->err2;
  *max_sweeps = cp->max_sweeps;
  return RHOSVD_OK;
}
void rhosvd_cp_free(rhosvd_cp* cp) {
  cudaDeviceSynchronize();
  cp_release(cp);
}

}  // extern "C"
