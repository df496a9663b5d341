// misc_kernels.cu - HBM-bound and scalar kernels of the RHOSVD path (sm_100a).
//
//  K0 normalize   : s_{l,k} = ||u_k^(l)||_2 (overflow/underflow-safe), Uhat = U diag(s)^-1
//                   written once to a padded workspace (ld multiple of 16 doubles,
//                   zero rows/columns), xi'_k = xi_k prod_l s_{l,k}, T_l, non-finite
//                   flag.  PAPER.md:252 "normalized canonical vectors"; readings A2/A3.
//  start block    : counter-based Gaussian random n x b block (seeded, deterministic).
//  ritz floor     : 1 / max(theta_k, tau theta_1).
//  select_rank    : eps rule A1 with the direct-residual tail:
//                   tail(r) = sum_{r<k<=b} lambda_k + rho, summed smallest-first.
//  sign fix       : reading A9 (largest-|.| entry positive, lowest row on ties).
#include "common.cuh"

namespace rhosvd {

// ---------------------------------------------------------------- K0 normalize
// One warp per column k of one mode.  HBM-bound: the column is read from DRAM once (the
// scaling pass re-reads it from L2) and Uhat written once.  16-B aligned columns (U 16-B
// aligned, ldu even - the torch layout) take double2 loads, four in flight per lane, so
// an SM keeps ~128 KB of reads outstanding (one-double loads: 4.3 TB/s on cfg 5).
__global__ void normalize_kernel(const double* __restrict__ U, int64_t ldu, int n, int R, int Rp,
                                 double* __restrict__ Uh, int64_t ldn, double* __restrict__ s_out,
                                 double* __restrict__ tcol, int* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= Rp) return;
  double* dst = Uh + (int64_t)k * ldn;
  if (k >= R) {
    for (int64_t i = lane; i < ldn; i += 32) dst[i] = 0.0;
    if (lane == 0) {
      s_out[k] = 0.0;
      tcol[k] = 0.0;
    }
    return;
  }
  const double* src = U + (int64_t)k * ldu;
  const bool vec = (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  double ss = 0.0, mx = 0.0;
  bool bad = false;
  if (vec) {
    const double2* s2 = reinterpret_cast<const double2*>(src);
    const int n2 = n >> 1;
    int i = lane;
    for (; i + 96 < n2; i += 128) {
      const double2 v0 = __ldg(s2 + i), v1 = __ldg(s2 + i + 32), v2 = __ldg(s2 + i + 64), v3 = __ldg(s2 + i + 96);
      const double w[8] = {v0.x, v0.y, v1.x, v1.y, v2.x, v2.y, v3.x, v3.y};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        bad |= !isfinite(w[q]);
        ss = fma(w[q], w[q], ss);
        mx = fmax(mx, fabs(w[q]));
      }
    }
    for (; i < n2; i += 32) {
      const double2 v = __ldg(s2 + i);
      bad |= !isfinite(v.x) || !isfinite(v.y);
      ss = fma(v.x, v.x, ss);
      ss = fma(v.y, v.y, ss);
      mx = fmax(mx, fmax(fabs(v.x), fabs(v.y)));
    }
    if ((n & 1) && lane == 0) {
      const double v = src[n - 1];
      bad |= !isfinite(v);
      ss = fma(v, v, ss);
      mx = fmax(mx, fabs(v));
    }
  } else {
    for (int i = lane; i < n; i += 32) {
      double v = src[i];
      bad |= !isfinite(v);
      ss = fma(v, v, ss);
      mx = fmax(mx, fabs(v));
    }
  }
  ss = warp_sum(ss);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  bad = __any_sync(0xffffffffu, bad);
  if (bad) {
    if (lane == 0) atomicOr(flag, 1);
    ss = 0.0;
    mx = 0.0;
  }
  double s;
  if (mx == 0.0) {
    s = 0.0;
  } else if (ss > 1e-280 && ss < 1e280) {
    s = sqrt(ss);
  } else {  // rescaled second pass (underflow / overflow safe)
    double inv = 1.0 / mx, t = 0.0;
    for (int i = lane; i < n; i += 32) {
      double v = src[i] * inv;
      t = fma(v, v, t);
    }
    t = warp_sum(t);
    s = mx * sqrt(t);
  }
  const double inv = s > 0.0 ? 1.0 / s : 0.0;
  double tt = 0.0;
  if (vec && (ldn & 1) == 0) {  // dst is 16-B aligned (ldn is a multiple of 16 doubles)
    const double2* s2 = reinterpret_cast<const double2*>(src);
    double2* d2 = reinterpret_cast<double2*>(dst);
    for (int64_t i = lane; i < (ldn >> 1); i += 32) {
      const int64_t e = 2 * i;
      double2 v;
      if (e + 1 < n) {
        const double2 x = s2[i];
        v = make_double2(x.x * inv, x.y * inv);
      } else {
        v = make_double2(e < n ? src[e] * inv : 0.0, 0.0);
      }
      d2[i] = v;
      tt = fma(v.x, v.x, tt);
      tt = fma(v.y, v.y, tt);
    }
  } else {
    for (int64_t i = lane; i < ldn; i += 32) {
      double v = (i < n) ? src[i] * inv : 0.0;
      dst[i] = v;
      tt = fma(v, v, tt);
    }
  }
  tt = warp_sum(tt);
  if (lane == 0) {
    s_out[k] = s;
    tcol[k] = tt;
  }
}

// K0 for 512 <= n <= 4096 (every BASELINE config but cfg 1): one CTA of T = 32 ceil(n / 512)
// threads per column holds the column in registers (16 doubles per thread, eight double2
// loads issued back to back), so the column is read from DRAM once and never re-read: norm by
// a block reduction, then the scaled column written from registers.  The one-warp kernel
// above re-reads each column from L2 for the scaling pass and keeps fewer loads in flight.
// Same outputs as normalize_kernel up to the summation order of the norms.
constexpr int NRM_PER = 16;
__global__ void __launch_bounds__(256) normalize_col_kernel(const double* __restrict__ U, int64_t ldu, int n, int R,
                                                            double* __restrict__ Uh, int64_t ldn,
                                                            double* __restrict__ s_out, double* __restrict__ tcol,
                                                            int* __restrict__ flag) {
  __shared__ double red[3][8];
  const int k = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const double* src = U + (int64_t)k * ldu;
  double* dst = Uh + (int64_t)k * ldn;
  // thread t owns elements 2 (t + T j) and 2 (t + T j) + 1, j < 8 (coalesced double2 accesses)
  const int T = blockDim.x;
  double2 v[NRM_PER / 2];
#pragma unroll
  for (int j = 0; j < NRM_PER / 2; ++j) {
    const int e = 2 * (tid + T * j);
    if (e + 1 < n) v[j] = __ldg(reinterpret_cast<const double2*>(src + e));
    else v[j] = make_double2(e < n ? src[e] : 0.0, 0.0);
  }
  double ss = 0.0, mx = 0.0;
  bool bad = false;
#pragma unroll
  for (int j = 0; j < NRM_PER / 2; ++j) {
    bad |= !isfinite(v[j].x) || !isfinite(v[j].y);
    ss = fma(v[j].x, v[j].x, ss);
    ss = fma(v[j].y, v[j].y, ss);
    mx = fmax(mx, fmax(fabs(v[j].x), fabs(v[j].y)));
  }
  ss = warp_sum(ss);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  bad = __syncthreads_or(bad);
  if (lane == 0) {
    red[0][warp] = ss;
    red[1][warp] = mx;
  }
  __syncthreads();
  ss = 0.0;
  mx = 0.0;
  for (int w = 0; w < nw; ++w) {  // fixed order
    ss += red[0][w];
    mx = fmax(mx, red[1][w]);
  }
  if (bad) {
    if (tid == 0) atomicOr(flag, 1);
    ss = 0.0;
    mx = 0.0;
  }
  double s;
  if (mx == 0.0) {
    s = 0.0;
  } else if (ss > 1e-280 && ss < 1e280) {
    s = sqrt(ss);
  } else {  // rescaled sum (underflow / overflow safe), from the registers
    const double inv = 1.0 / mx;
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < NRM_PER / 2; ++j) {
      t = fma(v[j].x * inv, v[j].x * inv, t);
      t = fma(v[j].y * inv, v[j].y * inv, t);
    }
    t = warp_sum(t);
    __syncthreads();
    if (lane == 0) red[2][warp] = t;
    __syncthreads();
    t = 0.0;
    for (int w = 0; w < nw; ++w) t += red[2][w];
    s = mx * sqrt(t);
  }
  const double inv = s > 0.0 ? 1.0 / s : 0.0;
  double tt = 0.0;
#pragma unroll
  for (int j = 0; j < NRM_PER / 2; ++j) {
    const int e = 2 * (tid + T * j);
    if (e < ldn) {  // ldn even: the pair (e, e + 1) lies inside the padded column
      const double2 x = make_double2(v[j].x * inv, v[j].y * inv);
      *reinterpret_cast<double2*>(dst + e) = x;
      tt = fma(x.x, x.x, tt);
      tt = fma(x.y, x.y, tt);
    }
  }
  // padding rows beyond the registers' reach (ldn > 2 T NRM_PER / 2 cannot happen: T >= n / 16
  // and ldn - n < 16) are zero-filled by the loop above only up to 2 T NRM_PER / 2
  for (int64_t e = (int64_t)T * NRM_PER + tid; e < ldn; e += T) dst[e] = 0.0;
  tt = warp_sum(tt);
  __syncthreads();
  if (lane == 0) red[2][warp] = tt;
  __syncthreads();
  if (tid == 0) {
    double t2 = 0.0;
    for (int w = 0; w < nw; ++w) t2 += red[2][w];
    s_out[k] = s;
    tcol[k] = t2;
  }
}

// xi'_k = xi_k s1 s2 s3 ; non-finite check on xi ; xi'^2 per term
__global__ void xiprime_kernel(const double* xi, const double* s1, const double* s2, const double* s3, int R,
                               int Rp, double* xip, double* xip2, int* flag) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= Rp) return;
  if (k >= R) {
    xip[k] = 0.0;
    xip2[k] = 0.0;
    return;
  }
  double x = xi[k];
  if (!isfinite(x)) atomicOr(flag, 1);
  double v = x * s1[k] * s2[k] * s3[k];
  if (!isfinite(v)) v = 0.0;
  xip[k] = v;
  xip2[k] = v * v;
}

// fixed-order sum of n doubles (one block of 1024): deterministic
__global__ void fixed_sum_kernel(const double* x, int64_t n, double* out) {
  __shared__ double sh[1024];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// sum of squares per block -> partials, then fixed_sum
__global__ void sumsq_partial_kernel(const double* x, int64_t n, double* part) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s = fma(x[i], x[i], s);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// ---------------------------------------------------------------- random start block
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__global__ void random_block_kernel(double* M, int64_t ldm, int n, int c0, int c1, uint64_t seed) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t rows = ldm, cols = c1 - c0;
  if (e >= rows * cols) return;
  int i = (int)(e % rows), j = c0 + (int)(e / rows);
  double v = 0.0;
  if (i < n) {
    uint64_t h = splitmix64(seed ^ splitmix64(((uint64_t)j << 32) | (uint64_t)i));
    uint64_t h2 = splitmix64(h);
    double u1 = ((h >> 11) + 1) * (1.0 / 9007199254740993.0);  // (0,1]
    double u2 = (h2 >> 11) * (1.0 / 9007199254740992.0);
    v = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
  M[(int64_t)j * ldm + i] = v;
}

// ---------------------------------------------------------------- Ritz floor
__global__ void ritz_floor_kernel(const double* th, int b, double tau, double* inv) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= b) return;
  double t0 = th[0];
  double f = fmax(th[k], tau * fabs(t0));
  inv[k] = f > 0.0 ? 1.0 / f : 1.0;
}

// ---------------------------------------------------------------- rank selection
// out[0] = r (as double; -1 if no r <= b satisfies the rule), out[1] = tail^2(r),
// out[2] = tail^2(b - guard) (for block-growth decisions), sigma[k] = sqrt(lambda_k), k < b
__global__ void select_rank_kernel(const double* lam, int b, const double* rho, double T, double eps,
                                   int r_fixed, int guard, double* tail2, double* out, double* sigma) {
  for (int k = threadIdx.x; k < b; k += blockDim.x) sigma[k] = sqrt(fmax(lam[k], 0.0));
  if (threadIdx.x != 0) return;
  double acc = *rho;
  tail2[b] = acc;
  for (int k = b - 1; k >= 0; --k) {  // smallest-first
    acc += fmax(lam[k], 0.0);
    tail2[k] = acc;
  }
  int r;
  if (r_fixed > 0) {
    r = min(r_fixed, b);
  } else {
    double thr = eps * eps * T;
    r = -1;
    for (int c = 1; c <= b; ++c)
      if (tail2[c] <= thr) {
        r = c;
        break;
      }
  }
  out[0] = (double)r;
  out[1] = r >= 0 ? tail2[r] : tail2[b];
  out[2] = tail2[max(0, b - guard)];
}

// ---------------------------------------------------------------- sign fix
__global__ void sign_col_kernel(const double* Z, int64_t ldz, int n, double* sgn) {
  __shared__ double bv[1024];
  __shared__ int bi[1024];
  const int j = blockIdx.x;
  const double* z = Z + (int64_t)j * ldz;
  double best = -1.0;
  int bidx = 0x7fffffff;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double a = fabs(z[i]);
    if (a > best || (a == best && i < bidx)) {
      best = a;
      bidx = i;
    }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = bidx;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      double a = bv[threadIdx.x + w];
      int ia = bi[threadIdx.x + w];
      if (a > bv[threadIdx.x] || (a == bv[threadIdx.x] && ia < bi[threadIdx.x])) {
        bv[threadIdx.x] = a;
        bi[threadIdx.x] = ia;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) sgn[j] = (bi[0] < n && z[bi[0]] < 0.0) ? -1.0 : 1.0;
}

__global__ void apply_sign_kernel(double* Z, int64_t ldz, int n, int r, double* W, int64_t ldw, int64_t Rl,
                                  const double* sgn) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t nz = (int64_t)n * r;
  if (e < nz) {
    int i = (int)(e % n), j = (int)(e / n);
    Z[(int64_t)j * ldz + i] *= sgn[j];
    return;
  }
  e -= nz;
  if (W && e < (int64_t)r * Rl) {
    int j = (int)(e / Rl);
    int64_t k = e % Rl;
    W[(int64_t)j * ldw + k] *= sgn[j];
  }
}

// d_j = sum_i Z(i,j) Y(i,j)  (diagonal of Z^T Y; one warp per column, fixed order)
__global__ void coldot_kernel(const double* Z, const double* Y, int64_t ld, int n, int b, double* d) {
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= b) return;
  const double* z = Z + (int64_t)j * ld;
  const double* y = Y + (int64_t)j * ld;
  double s = 0.0;
  for (int i = lane; i < n; i += 32) s = fma(z[i], y[i], s);
  s = warp_sum(s);
  if (lane == 0) d[j] = s;
}

// ---------------------------------------------------------------- host wrappers
#define LAUNCH_OK() \
  do {              \
    count_launch(); \
    RH_LAUNCH_CHECK(); \
  } while (0)

int k_normalize(const double* U, int64_t ldu, int64_t n, int64_t R, int64_t Rp, double* Uh, int64_t ldn,
                double* s, double* tcol, int* flag, cudaStream_t st) {
  if (Rp <= 0) return RHOSVD_OK;
  const int wpb = 8;
  // register-resident column kernel for 512 <= n <= 4096 with 16-B aligned columns; the
  // padding columns R..Rp-1 (zero) and every other shape take the one-warp kernel
  const bool col = n >= 512 && n <= 4096 && (ldn & 1) == 0 && (ldu & 1) == 0 &&
                   (reinterpret_cast<uintptr_t>(U) & 15) == 0 && (reinterpret_cast<uintptr_t>(Uh) & 15) == 0;
  if (col && R > 0) {
    const int T = (int)(32 * cdiv(n, 32 * NRM_PER));
    normalize_col_kernel<<<(unsigned)R, T, 0, st>>>(U, ldu, (int)n, (int)R, Uh, ldn, s, tcol, flag);
    LAUNCH_OK();
    if (Rp > R) {  // zero padding columns
      normalize_kernel<<<(unsigned)cdiv(Rp - R, wpb), 32 * wpb, 0, st>>>(U, ldu, (int)n, 0, (int)(Rp - R),
                                                                        Uh + R * ldn, ldn, s + R, tcol + R, flag);
      LAUNCH_OK();
    }
    return RHOSVD_OK;
  }
  normalize_kernel<<<(unsigned)cdiv(Rp, wpb), 32 * wpb, 0, st>>>(U, ldu, (int)n, (int)R, (int)Rp, Uh, ldn, s,
                                                                  tcol, flag);
  LAUNCH_OK();
  return RHOSVD_OK;
}
int k_xiprime(const double* xi, const double* s1, const double* s2, const double* s3, int64_t R, int64_t Rp,
              double* xip, double* xip2, int* flag, cudaStream_t st) {
  if (Rp <= 0) return RHOSVD_OK;
  xiprime_kernel<<<(unsigned)cdiv(Rp, 256), 256, 0, st>>>(xi, s1, s2, s3, (int)R, (int)Rp, xip, xip2, flag);
  LAUNCH_OK();
  return RHOSVD_OK;
}
int k_coldot(const double* Z, const double* Y, int64_t ld, int64_t n, int64_t b, double* d, cudaStream_t st) {
  if (b <= 0) return RHOSVD_OK;
  coldot_kernel<<<(unsigned)cdiv(b, 8), 256, 0, st>>>(Z, Y, ld, (int)n, (int)b, d);
  LAUNCH_OK();
  return RHOSVD_OK;
}
int k_fixed_sum(const double* x, int64_t n, double* out, cudaStream_t st) {
  fixed_sum_kernel<<<1, 1024, 0, st>>>(x, n, out);
  LAUNCH_OK();
  return RHOSVD_OK;
}
int k_sumsq(const double* x, int64_t n, double* part /* >= 256 */, double* out, cudaStream_t st) {
  int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(256, cdiv(n, 256)));
  sumsq_partial_kernel<<<blocks, 256, 0, st>>>(x, n, part);
  LAUNCH_OK();
  return k_fixed_sum(part, blocks, out, st);
}
int k_random(double* M, int64_t ldm, int64_t n, int64_t c0, int64_t c1, uint64_t seed, cudaStream_t st) {
  if (c1 <= c0) return RHOSVD_OK;
  int64_t tot = ldm * (c1 - c0);
  random_block_kernel<<<(unsigned)cdiv(tot, 256), 256, 0, st>>>(M, ldm, (int)n, (int)c0, (int)c1, seed);
  LAUNCH_OK();
  return RHOSVD_OK;
}
int k_ritz_floor(const double* th, int64_t b, double tau, double* inv, cudaStream_t st) {
  ritz_floor_kernel<<<(unsigned)cdiv(b, 256), 256, 0, st>>>(th, (int)b, tau, inv);
  LAUNCH_OK();
  return RHOSVD_OK;
}
int k_select_rank(const double* lam, int64_t b, const double* rho, double T, double eps, int r_fixed, int guard,
                  double* tail2, double* out, double* sigma, cudaStream_t st) {
  select_rank_kernel<<<1, 256, 0, st>>>(lam, (int)b, rho, T, eps, r_fixed, guard, tail2, out, sigma);
  LAUNCH_OK();
  return RHOSVD_OK;
}
// ALS: C <- A o C elementwise on an M x N column-major block (ld)
__global__ void hadamard_kernel(const double* A, double* C, int64_t ld, int64_t M, int64_t N) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M * N) return;
  const int64_t i = e % M, j = e / M;
  C[j * ld + i] *= A[j * ld + i];
}
int k_hadamard(const double* A, double* C, int64_t ld, int64_t M, int64_t N, cudaStream_t st) {
  if (M <= 0 || N <= 0) return RHOSVD_OK;
  hadamard_kernel<<<(unsigned)cdiv(M * N, 256), 256, 0, st>>>(A, C, ld, M, N);
  LAUNCH_OK();
  return RHOSVD_OK;
}
// B[i * ldb + k] = A[k * lda + i]  (i < rows, k < cols): 32 x 32 tiles through shared
// memory, coalesced on both sides
__global__ void transpose_kernel(const double* A, int64_t lda, int64_t rows, int64_t cols, double* B, int64_t ldb) {
  __shared__ double t[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32, k0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int q = ty; q < 32; q += 8) {
    const int64_t i = i0 + tx, k = k0 + q;
    t[q][tx] = (i < rows && k < cols) ? A[k * lda + i] : 0.0;
  }
  __syncthreads();
  for (int q = ty; q < 32; q += 8) {
    const int64_t k = k0 + tx, i = i0 + q;
    if (i < rows && k < cols) B[i * ldb + k] = t[tx][q];
  }
}
int k_transpose(const double* A, int64_t lda, int64_t rows, int64_t cols, double* B, int64_t ldb, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return RHOSVD_OK;
  if (cdiv(cols, 32) > 65535) return fail(RHOSVD_EINVAL, "transpose: too many columns");
  transpose_kernel<<<dim3((unsigned)cdiv(rows, 32), (unsigned)cdiv(cols, 32)), dim3(32, 8), 0, st>>>(A, lda, rows,
                                                                                                    cols, B, ldb);
  LAUNCH_OK();
  return RHOSVD_OK;
}

// out[k] = sqrt(max(lam[k], 0)), k < r  (singular values from Gram eigenvalues)
__global__ void sqrt_clamp_kernel(const double* lam, int r, double* out) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < r) out[k] = sqrt(fmax(lam[k], 0.0));
}
int k_sqrt_clamp(const double* lam, int64_t r, double* out, cudaStream_t st) {
  if (r <= 0) return RHOSVD_OK;
  sqrt_clamp_kernel<<<(unsigned)cdiv(r, 256), 256, 0, st>>>(lam, (int)r, out);
  LAUNCH_OK();
  return RHOSVD_OK;
}

int k_sign_fix(double* Z, int64_t ldz, int64_t n, int64_t r, double* W, int64_t ldw, int64_t Rl, double* sgn,
               cudaStream_t st) {
  if (r <= 0) return RHOSVD_OK;
  sign_col_kernel<<<(unsigned)r, 1024, 0, st>>>(Z, ldz, (int)n, sgn);
  LAUNCH_OK();
  int64_t tot = n * r + (W ? r * Rl : 0);
  apply_sign_kernel<<<(unsigned)cdiv(tot, 256), 256, 0, st>>>(Z, ldz, (int)n, (int)r, W, ldw, Rl, sgn);
  LAUNCH_OK();
  return RHOSVD_OK;
}

}  // namespace rhosvd
