// gemm.cu - FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) GEMM engine for sm_100a.
//
// sm_100a has no FP64 tcgen05 kind (ptxas rejects kind::f64), so
// the FP64 tensor path is the warp-synchronous mma.sync.m8n8k4 (SASS
// DMMA.8x8x4) with register accumulators.  Operand tiles are staged in shared
// memory by a STAGES-deep cp.async pipeline; smem row pitches are padded so
// every fragment load is two 128-byte wavefronts (conflict-free):
//   m/n-contiguous tile  T[k][m], pitch BM+8 (== 8 mod 16 doubles)
//   k-contiguous  tile   T[m][k], pitch BK+4 (== 4 mod 16 doubles)
// Split-K writes fixed-order partials that a reduce kernel sums in order, so
// results are bitwise reproducible (no FP64 atomics).
#include "gemm.cuh"

namespace rhosvd {

struct KParams {
  int M, N, K;
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  double alpha, beta;
  const double* cs;
  const double* rs;
  int upper;      // compute only tiles tm <= tn
  int epi;
  const double* D;
  int64_t ldd;
  double* part;   // split-K partials [split][N][M] (col-major, ld M) or residual per-CTA sums
  int splits;
  int kchunk;     // K per split (multiple of BK)
  int tiles_m, tiles_n;
};

template <int BM, int BN, int BK, int WM, int WN, bool AK, bool BKM, int STAGES>
struct GemmCfg {
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
  static constexpr int FM = WM / 8, FN = WN / 8;
  // A tile: AK ? [BM][BK+4] : [BK][BM+8]
  static constexpr int A_ROWS = AK ? BM : BK, A_PITCH = AK ? BK + 4 : BM + 8;
  static constexpr int B_ROWS = BKM ? BN : BK, B_PITCH = BKM ? BK + 4 : BN + 8;
  static constexpr int A_STAGE = A_ROWS * A_PITCH, B_STAGE = B_ROWS * B_PITCH;
  static constexpr size_t SMEM = size_t(STAGES) * (A_STAGE + B_STAGE) * sizeof(double);
};

template <int BM, int BN, int BK, int WM, int WN, bool AK, bool BKM, int STAGES>
__global__ void __launch_bounds__(GemmCfg<BM, BN, BK, WM, WN, AK, BKM, STAGES>::THREADS)
    dmma_gemm_kernel(KParams p) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, AK, BKM, STAGES>;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * Cfg::A_STAGE;

  // ---- tile coordinates
  int tile = blockIdx.x, tm, tn;
  if (p.upper) {
    // enumerate upper-triangular tiles (tm <= tn) column by column
    tn = (int)((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
    while ((tn + 1) * (tn + 2) / 2 <= tile) ++tn;
    while (tn * (tn + 1) / 2 > tile) --tn;
    tm = tile - tn * (tn + 1) / 2;
  } else {
    tm = tile % p.tiles_m;
    tn = tile / p.tiles_m;
  }
  const int m0 = tm * BM, n0 = tn * BN;
  const int split = blockIdx.y;
  const int kbeg = split * p.kchunk;
  const int kend = min(p.K, kbeg + p.kchunk);
  const int nk = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp % Cfg::WARPS_M) * WM, wn0 = (warp / Cfg::WARPS_M) * WN;

  auto load_tile = [&](int stage, int kt) {
    const int k0 = kbeg + kt * BK;
    double* as = As + stage * Cfg::A_STAGE;
    double* bs = Bs + stage * Cfg::B_STAGE;
    // A
    if (AK) {
      constexpr int CPR = BK / 2, TOT = BM * CPR;
      for (int c = tid; c < TOT; c += Cfg::THREADS) {
        int r = c / CPR, cc = (c % CPR) * 2;
        int gm = m0 + r, gk = k0 + cc;
        int nb = (gm < p.M) ? max(0, min(2, kend - gk)) : 0;
        const double* src = nb ? p.A + (int64_t)gm * p.lda + gk : p.A;
        cp_async16(as + r * Cfg::A_PITCH + cc, src, nb * 8);
      }
    } else {
      constexpr int CPR = BM / 2, TOT = BK * CPR;
      for (int c = tid; c < TOT; c += Cfg::THREADS) {
        int r = c / CPR, cc = (c % CPR) * 2;
        int gk = k0 + r, gm = m0 + cc;
        int nb = (gk < kend) ? max(0, min(2, p.M - gm)) : 0;
        const double* src = nb ? p.A + (int64_t)gk * p.lda + gm : p.A;
        cp_async16(as + r * Cfg::A_PITCH + cc, src, nb * 8);
      }
    }
    // B
    if (BKM) {
      constexpr int CPR = BK / 2, TOT = BN * CPR;
      for (int c = tid; c < TOT; c += Cfg::THREADS) {
        int r = c / CPR, cc = (c % CPR) * 2;
        int gn = n0 + r, gk = k0 + cc;
        int nb = (gn < p.N) ? max(0, min(2, kend - gk)) : 0;
        const double* src = nb ? p.B + (int64_t)gn * p.ldb + gk : p.B;
        cp_async16(bs + r * Cfg::B_PITCH + cc, src, nb * 8);
      }
    } else {
      constexpr int CPR = BN / 2, TOT = BK * CPR;
      for (int c = tid; c < TOT; c += Cfg::THREADS) {
        int r = c / CPR, cc = (c % CPR) * 2;
        int gk = k0 + r, gn = n0 + cc;
        int nb = (gk < kend) ? max(0, min(2, p.N - gn)) : 0;
        const double* src = nb ? p.B + (int64_t)gk * p.ldb + gn : p.B;
        cp_async16(bs + r * Cfg::B_PITCH + cc, src, nb * 8);
      }
    }
  };

  double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_tile(s, s);
    cp_async_commit();
  }

  const int fr = lane >> 2, fc = lane & 3;
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int nx = kt + STAGES - 1;
      if (nx < nk) load_tile(nx % STAGES, nx);
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * Cfg::A_STAGE;
    const double* bs = Bs + (kt % STAGES) * Cfg::B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[Cfg::FM], bf[Cfg::FN];
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i) {
        int m = wm0 + i * 8 + fr, k = kk + fc;
        af[i] = AK ? as[m * Cfg::A_PITCH + k] : as[k * Cfg::A_PITCH + m];
      }
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) {
        int n = wn0 + j * 8 + fr, k = kk + fc;
        bf[j] = BKM ? bs[n * Cfg::B_PITCH + k] : bs[k * Cfg::B_PITCH + n];
      }
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // ---- epilogue
  if (p.epi == EPI_RESID) {
    double ss = 0.0;
#pragma unroll
    for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int m = m0 + wm0 + i * 8 + fr, n = n0 + wn0 + j * 8 + 2 * fc + h;
          if (m < p.M && n < p.N) {
            double e = p.D[(int64_t)n * p.ldd + m] - acc[i][j][h];
            ss = fma(e, e, ss);
          }
        }
    ss = warp_sum(ss);
    __syncthreads();
    double* red = smem;
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < Cfg::THREADS / 32; ++w) t += red[w];
      p.part[blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
    return;
  }
  if (p.splits > 1) {
    double* out = p.part + (int64_t)split * p.M * p.N;
#pragma unroll
    for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int m = m0 + wm0 + i * 8 + fr, n = n0 + wn0 + j * 8 + 2 * fc + h;
          if (m < p.M && n < p.N) out[(int64_t)n * p.M + m] = acc[i][j][h];
        }
    return;
  }
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int m = m0 + wm0 + i * 8 + fr, n = n0 + wn0 + j * 8 + 2 * fc + h;
        if (m < p.M && n < p.N && (!p.upper || m <= n)) {
          double v = p.alpha * acc[i][j][h];
          if (p.cs) v *= p.cs[n];
          if (p.rs) v *= p.rs[m];
          double* c = p.C + (int64_t)n * p.ldc + m;
          if (p.beta != 0.0) v = fma(p.beta, *c, v);
          *c = v;
          if (p.upper && m < n) p.C[(int64_t)m * p.ldc + n] = v;  // mirror (M == N)
        }
      }
}

// Fixed-order split-K reduction + epilogue (and symmetric mirror).
__global__ void splitk_reduce_kernel(KParams p) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = (int64_t)p.M * p.N;
  if (idx >= total) return;
  int m = (int)(idx % p.M), n = (int)(idx / p.M);
  int sm = m, sn = n;
  if (p.upper && m > n) { sm = n; sn = m; }  // read the computed upper entry
  int64_t src = (int64_t)sn * p.M + sm;
  double s = 0.0;
  for (int k = 0; k < p.splits; ++k) s += p.part[(int64_t)k * total + src];
  double v = p.alpha * s;
  if (p.cs) v *= p.cs[n];
  if (p.rs) v *= p.rs[m];
  double* c = p.C + (int64_t)n * p.ldc + m;
  if (p.beta != 0.0) v = fma(p.beta, *c, v);
  *c = v;
}

__global__ void sum_fixed_order_kernel(const double* x, int n, double* out) {
  // one block, fixed order: strided partial sums then a fixed tree
  __shared__ double sh[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// ------------------------------------------------------------------ host side
int Scratch::ensure(size_t doubles, cudaStream_t st) {
  if (doubles <= cap) return RHOSVD_OK;
  if (ptr) cudaFreeAsync(ptr, st);
  ptr = nullptr;
  cap = 0;
  size_t want = doubles + doubles / 4 + 1024;
  cudaError_t e = cudaMallocAsync((void**)&ptr, want * sizeof(double), st);
  if (e != cudaSuccess) {
    ptr = nullptr;
    return fail(RHOSVD_ENOMEM, std::string("scratch alloc: ") + cudaGetErrorString(e));
  }
  cap = want;
  return RHOSVD_OK;
}
void Scratch::release(cudaStream_t st) {
  if (ptr) cudaFreeAsync(ptr, st);
  ptr = nullptr;
  cap = 0;
}

template <int BM, int BN, int BK, int WM, int WN, bool AK, bool BKM, int STAGES>
static int launch_cfg(KParams kp, int ntiles, cudaStream_t st) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, AK, BKM, STAGES>;
  auto kern = dmma_gemm_kernel<BM, BN, BK, WM, WN, AK, BKM, STAGES>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    RH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
    attr_set = true;
  }
  dim3 grid(ntiles, kp.splits);
  kern<<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(kp);
  count_launch();
  RH_LAUNCH_CHECK();
  return RHOSVD_OK;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
static int launch_layout(bool ak, bool bk, KParams kp, int ntiles, cudaStream_t st) {
  if (ak && bk) return launch_cfg<BM, BN, BK, WM, WN, true, true, STAGES>(kp, ntiles, st);
  if (ak && !bk) return launch_cfg<BM, BN, BK, WM, WN, true, false, STAGES>(kp, ntiles, st);
  if (!ak && bk) return launch_cfg<BM, BN, BK, WM, WN, false, true, STAGES>(kp, ntiles, st);
  return launch_cfg<BM, BN, BK, WM, WN, false, false, STAGES>(kp, ntiles, st);
}

int gemm(const GemmArgs& g, Scratch& scr, cudaStream_t st, double* flops_acc) {
  if (g.M <= 0 || g.N <= 0) return RHOSVD_OK;
  if (g.M > INT32_MAX || g.N > INT32_MAX || g.K > INT32_MAX)
    return fail(RHOSVD_EINVAL, "gemm: dimension exceeds int32");
  if (g.upper_sym && g.M != g.N) return fail(RHOSVD_EINVAL, "gemm: upper_sym needs M == N");
  KParams kp{};
  kp.M = (int)g.M; kp.N = (int)g.N; kp.K = (int)g.K;
  kp.A = g.A; kp.lda = g.lda; kp.B = g.B; kp.ldb = g.ldb; kp.C = g.C; kp.ldc = g.ldc;
  kp.alpha = g.alpha; kp.beta = g.beta; kp.cs = g.col_scale; kp.rs = g.row_scale;
  kp.upper = g.upper_sym ? 1 : 0; kp.epi = g.epi; kp.D = g.D; kp.ldd = g.ldd;

  // tile choice: big tiles when there is enough output to fill the GPU
  const int sms = num_sms();
  const bool big = (cdiv(g.M, 128) * cdiv(g.N, 128) >= sms) ||
                   (g.M >= 128 && g.N >= 128 && g.K >= 2048);
  const int BT = big ? 128 : 64, BK = 16;
  int tm = (int)cdiv(g.M, BT), tn = (int)cdiv(g.N, BT);
  int ntiles = g.upper_sym ? tn * (tn + 1) / 2 : tm * tn;
  kp.tiles_m = tm; kp.tiles_n = tn;

  int splits = g.splits;
  if (g.epi == EPI_RESID) splits = 1;
  if (splits <= 0) {
    // enough CTAs for ~2 waves, each split >= 512 of K
    int64_t want = cdiv(2LL * sms, ntiles);
    int64_t maxs = std::max<int64_t>(1, g.K / 512);
    splits = (int)std::max<int64_t>(1, std::min<int64_t>(want, maxs));
    if (splits > 64) splits = 64;
  }
  int kchunk = (int)round_up(cdiv(std::max<int64_t>(g.K, 1), splits), BK);
  splits = (int)std::max<int64_t>(1, cdiv(std::max<int64_t>(g.K, 1), kchunk));
  kp.splits = splits;
  kp.kchunk = kchunk;

  if (g.epi == EPI_RESID) {
    RH_CHECK(scr.ensure((size_t)ntiles, st));
    kp.part = scr.ptr;
  } else if (splits > 1) {
    RH_CHECK(scr.ensure((size_t)splits * g.M * g.N, st));
    kp.part = scr.ptr;
  }
  if (big)
    RH_CHECK((launch_layout<128, 128, 16, 64, 32, 3>(g.a_k, g.b_k, kp, ntiles, st)));
  else
    RH_CHECK((launch_layout<64, 64, 16, 32, 32, 3>(g.a_k, g.b_k, kp, ntiles, st)));

  if (g.epi == EPI_RESID) {
    sum_fixed_order_kernel<<<1, 256, 0, st>>>(kp.part, ntiles, g.resid_out);
    count_launch();
    RH_LAUNCH_CHECK();
  } else if (splits > 1) {
    int64_t total = g.M * g.N;
    splitk_reduce_kernel<<<(unsigned)cdiv(total, 256), 256, 0, st>>>(kp);
    count_launch();
    RH_LAUNCH_CHECK();
  }
  if (flops_acc) *flops_acc += 2.0 * (double)g.M * (double)g.N * (double)g.K * (g.upper_sym ? 0.5 : 1.0);
  return RHOSVD_OK;
}

}  // namespace rhosvd
