// core_kr.cu - K7: the RHOSVD core as a Khatri-Rao DMMA contraction (sm_100a, FP64).
//
// Prop. 2.1: the core beta_0 = xi x_1 U_0^(1)T x_2 U_0^(2)T x_3 U_0^(3)T
// of the RHOSVD Tucker tensor is the rank-R CP tensor with factors W_l = Z_l^T Uhat_l,
// "calculated entry-wise in O(R r1 ... rd) operations".  We compute it densely as
//     beta_(12)(3) = (W1 (.) W2) (xi' o W3)^T      M = r1 r2, N = r3, K = R
// where the Khatri-Rao row (a,b) of a k-tile is never materialised: the CTA
// stages W1 (TA rows), W2 (TB rows) and W3 (BN rows) k-tiles in shared memory by
// cp.async and each DMMA A-fragment is formed in registers as W1[a,k] * W2[b,k]
// (one DMUL per fragment element; xi' is pre-folded into W1).  The materialised
// Khatri-Rao operand would be 152 GiB on cfg 4.
// Output beta[a,b,c] in C order (c fastest).  Split-K (for small r, large R)
// writes fixed-order partials reduced by a second kernel (deterministic).
#include "common.cuh"

namespace rhosvd {

struct CoreParams {
  int r1, r2, r3, R;
  const double* W1;  // xi' o W1, row-major r1 x R (ld ldw1)
  int64_t ldw1;
  const double* W2;
  const double* W3;
  int64_t ldw;
  double* out;       // beta or partials [split][r1 r2 r3]
  int splits, kchunk;
  int tiles_a, tiles_b, tiles_n;
};

template <int TA, int TB, int BN, int BK, int WM, int WN, int STAGES>
struct CoreCfg {
  static constexpr int BM = TA * TB;
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
  static constexpr int FM = WM / 8, FN = WN / 8;
  static constexpr int P = BK + 4;  // k-contiguous pitch (== 4 mod 16)
  static constexpr int S1 = TA * P, S2 = TB * P, S3 = BN * P;
  static constexpr int STAGE = S1 + S2 + S3;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE * sizeof(double);
};

template <int TA, int TB, int BN, int BK, int WM, int WN, int STAGES>
__global__ void __launch_bounds__(CoreCfg<TA, TB, BN, BK, WM, WN, STAGES>::THREADS)
    core_kr_kernel(CoreParams p) {
  using Cfg = CoreCfg<TA, TB, BN, BK, WM, WN, STAGES>;
  static_assert(TB % 8 == 0, "TB multiple of 8");
  extern __shared__ __align__(16) double smem[];
  int t = blockIdx.x;
  const int tn = t % p.tiles_n;
  t /= p.tiles_n;
  const int tb = t % p.tiles_b;
  const int ta = t / p.tiles_b;
  const int a0 = ta * TA, b0 = tb * TB, n0 = tn * BN;
  const int split = blockIdx.y;
  const int kbeg = split * p.kchunk, kend = min(p.R, kbeg + p.kchunk);
  const int nk = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp % Cfg::WARPS_M) * WM, wn0 = (warp / Cfg::WARPS_M) * WN;

  auto load_rows = [&](double* dst, const double* src, int64_t ld, int row0, int nrows_tile, int nrows_tot,
                       int k0) {
    constexpr int CPR = BK / 2;
    const int TOT = nrows_tile * CPR;
    for (int c = tid; c < TOT; c += Cfg::THREADS) {
      int r = c / CPR, cc = (c % CPR) * 2;
      int gr = row0 + r, gk = k0 + cc;
      int nb = (gr < nrows_tot) ? max(0, min(2, kend - gk)) : 0;
      const double* s = nb ? src + (int64_t)gr * ld + gk : src;
      cp_async16(dst + r * Cfg::P + cc, s, nb * 8);
    }
  };
  auto load_stage = [&](int stage, int kt) {
    const int k0 = kbeg + kt * BK;
    double* base = smem + stage * Cfg::STAGE;
    load_rows(base, p.W1, p.ldw1, a0, TA, p.r1, k0);
    load_rows(base + Cfg::S1, p.W2, p.ldw, b0, TB, p.r2, k0);
    load_rows(base + Cfg::S1 + Cfg::S2, p.W3, p.ldw, n0, BN, p.r3, k0);
  };

  double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }
  const int fr = lane >> 2, fc = lane & 3;
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int nx = kt + STAGES - 1;
      if (nx < nk) load_stage(nx % STAGES, nx);
      cp_async_commit();
    }
    const double* w1 = smem + (kt % STAGES) * Cfg::STAGE;
    const double* w2 = w1 + Cfg::S1;
    const double* w3 = w2 + Cfg::S2;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[Cfg::FM], bf[Cfg::FN];
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i) {
        const int mi = wm0 + i * 8;        // fragment rows mi .. mi+7 share a_loc
        const int al = mi / TB, bl = mi % TB + fr;
        af[i] = w1[al * Cfg::P + kk + fc] * w2[bl * Cfg::P + kk + fc];
      }
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) bf[j] = w3[(wn0 + j * 8 + fr) * Cfg::P + kk + fc];
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  double* out = p.out + (p.splits > 1 ? (int64_t)split * p.r1 * p.r2 * p.r3 : 0);
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i) {
    const int mi = wm0 + i * 8 + fr;
    const int a = a0 + mi / TB, bb = b0 + mi % TB;
    if (a >= p.r1 || bb >= p.r2) continue;
    double* row = out + ((int64_t)a * p.r2 + bb) * p.r3;
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int n = n0 + wn0 + j * 8 + 2 * fc + h;
        if (n < p.r3) row[n] = acc[i][j][h];
      }
  }
}

__global__ void core_splitk_reduce(const double* part, int splits, int64_t total, double* beta) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  double s = 0.0;
  for (int k = 0; k < splits; ++k) s += part[(int64_t)k * total + i];
  beta[i] = s;
}

// xi' o W1 (row-major r1 x R, ld ldw) -> out (ld ldo)
__global__ void scale_cols_kernel(const double* W, int64_t ldw, const double* xi, int r, int R, double* out,
                                  int64_t ldo) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)r * R) return;
  int a = (int)(e / R), k = (int)(e % R);
  out[a * ldo + k] = W[a * ldw + k] * xi[k];
}

// host entry: beta (r1 x r2 x r3, C order) = sum_k xi_k W1[:,k] (x) W2[:,k] (x) W3[:,k]
// W1x must already hold xi' o W1.  part: scratch for split-K (may be null when splits == 1)
int core_kr(const double* W1x, int64_t ldw1, const double* W2, const double* W3, int64_t ldw, int64_t r1,
            int64_t r2, int64_t r3, int64_t R, double* beta, double* part, size_t part_cap, cudaStream_t st,
            double* flops_acc) {
  if (r1 <= 0 || r2 <= 0 || r3 <= 0) return RHOSVD_OK;
  constexpr int TA = 2, TB = 64, BN = 128, BK = 16, WM = 64, WN = 32, ST = 3;
  using Cfg = CoreCfg<TA, TB, BN, BK, WM, WN, ST>;
  auto kern = core_kr_kernel<TA, TB, BN, BK, WM, WN, ST>;
  static bool attr = false;
  if (!attr) {
    RH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
    attr = true;
  }
  CoreParams cp{};
  cp.r1 = (int)r1; cp.r2 = (int)r2; cp.r3 = (int)r3; cp.R = (int)R;
  cp.W1 = W1x; cp.ldw1 = ldw1; cp.W2 = W2; cp.W3 = W3; cp.ldw = ldw;
  cp.tiles_a = (int)cdiv(r1, TA); cp.tiles_b = (int)cdiv(r2, TB); cp.tiles_n = (int)cdiv(r3, BN);
  int64_t tiles = (int64_t)cp.tiles_a * cp.tiles_b * cp.tiles_n;
  int64_t total = r1 * r2 * r3;
  int splits = 1;
  const int sms = num_sms();
  if (tiles < 2 * sms && R >= 1024) {
    splits = (int)std::min<int64_t>(cdiv(2 * sms, tiles), R / 512);
    splits = std::max(1, std::min(splits, 32));
    while (splits > 1 && (size_t)splits * total > part_cap) --splits;
  }
  cp.kchunk = (int)round_up(cdiv(std::max<int64_t>(R, 1), splits), BK);
  splits = (int)std::max<int64_t>(1, cdiv(std::max<int64_t>(R, 1), cp.kchunk));
  cp.splits = splits;
  cp.out = splits > 1 ? part : beta;
  if (tiles > INT32_MAX) return fail(RHOSVD_EINVAL, "core: too many tiles");
  kern<<<dim3((unsigned)tiles, splits), Cfg::THREADS, Cfg::SMEM, st>>>(cp);
  count_launch();
  RH_LAUNCH_CHECK();
  if (splits > 1) {
    core_splitk_reduce<<<(unsigned)cdiv(total, 256), 256, 0, st>>>(part, splits, total, beta);
    count_launch();
    RH_LAUNCH_CHECK();
  }
  if (flops_acc) *flops_acc += 2.0 * (double)r1 * r2 * r3 * R;
  return RHOSVD_OK;
}

int scale_cols(const double* W, int64_t ldw, const double* xi, int64_t r, int64_t R, double* out, int64_t ldo,
               cudaStream_t st) {
  if (r <= 0 || R <= 0) return RHOSVD_OK;
  scale_cols_kernel<<<(unsigned)cdiv(r * R, 256), 256, 0, st>>>(W, ldw, xi, (int)r, (int)R, out, ldo);
  count_launch();
  RH_LAUNCH_CHECK();
  return RHOSVD_OK;
}

}  // namespace rhosvd
