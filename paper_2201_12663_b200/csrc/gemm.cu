// gemm.cu - FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) GEMM engine for sm_100a, TMA-fed.
//
// sm_100a has no FP64 tcgen05 kind (ptxas rejects kind::f64), so the FP64
// tensor path is the warp-synchronous mma.sync.m8n8k4 (SASS DMMA.8x8x4) with register
// accumulators.  Operand tiles move global -> shared by TMA (cp.async.bulk.tensor.2d)
// into a STAGES-deep ring guarded by full/empty mbarriers; thread 0 issues the copies
// (refilling the stage the 8 warps released one step earlier), so the ring stays
// STAGES-1 k-slabs ahead.  Two operand layouts, both conflict-free for the 8x4 / 4x8
// fragment loads:
//   k-contiguous  (X[row * ld + k]) : box {16, rows}, 128-B swizzle -> [rows][16]
//   m-contiguous  (X[k * ld + row]) : box {rows + 8, 16}, no swizzle -> [16][rows + 8]
//                 (pitch == 8 mod 16 doubles; the 8 extra rows are the next tile's)
// The grid is persistent (one CTA per SM, static stride over work items = tiles x
// K-splits).  Split-K writes fixed-order partials that a second kernel sums in order:
// results are bitwise reproducible (no FP64 atomics).
#include <algorithm>
#include <type_traits>

#include "gemm.cuh"
#include "tma.cuh"

namespace rhosvd {

constexpr int GBK = 16, GTHREADS = 256;

struct GParams {
  int M, N, K;
  double* C;
  int64_t ldc;
  double alpha, beta;
  const double* cs;
  const double* rs;
  int upper;      // compute only tiles tm <= tn, mirror
  int epi;
  const double* D;
  int64_t ldd;
  double* part;   // split-K partials [split][N][M] (col-major, ld M) or residual per-item sums
  int splits, kchunk;
  int tiles_m, tiles_n, tiles, items;
  int n_off;      // first output column of this launch (column segments)
  int nbatch, per_batch;  // batched form: items = nbatch * per_batch, per_batch = splits * tiles
  int a_koff, b_koff;     // k-coordinate shift of batch b's operands (b * koff)
  int64_t c_bstride;      // C offset of batch b (doubles)
  int stages;
  uint32_t a_bytes, stage_bytes, tx_bytes;
  uint32_t b_bytes;  // one k-slab of B (the stage holds KS slabs of A, then KS of B)
};

template <int BM, int BN, bool AK, bool BKM, int KS>
__global__ void __launch_bounds__(GTHREADS, 1)
    tma_gemm_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB, const GParams p) {
  constexpr int WM = BM / 2, WN = BN / 4, FM = WM / 8, FN = WN / 8;
  constexpr int APITCH = BM + 8, BPITCH = BN + 8;  // doubles, m/n-contiguous layouts
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = (uint64_t*)(ring + (size_t)p.stages * p.stage_bytes);
  uint64_t* empty = full + p.stages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool producer = (tid == 0);

  auto tile_of = [&](int tile, int& tm, int& tn) {
    if (p.upper) {
      tn = (int)((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
      while ((tn + 1) * (tn + 2) / 2 <= tile) ++tn;
      while (tn * (tn + 1) / 2 > tile) --tn;
      tm = tile - tn * (tn + 1) / 2;
    } else {
      tm = tile % p.tiles_m;
      tn = tile / p.tiles_m;
    }
  };
  // Item order.  Plain GEMMs: static stride, item = (batch, split, tile) with the tile
  // fastest.  Symmetric (upper) 128 x 128 form: the off-diagonal items of every batch
  // first, the diagonal ones (cheaper: 36 of 64 DMMAs per sub-partition, see below) last,
  // dealt to the CTAs in a snake (odd rounds in reverse CTA order), so the CTAs that take
  // one item more than the others take diagonal ones.  cfg 4 (3 x 136 tiles x 5 splits on
  // 148 SMs): the busiest CTA runs 12 off-diagonal + 2 diagonal items instead of 14.  The
  // split-K partials and their fixed-order sum are independent of the item order, so G is
  // bitwise unchanged.
  constexpr bool kDiag = (BM == 128 && BN == 128);
  const bool snake = kDiag && p.upper;
  auto item_at = [&](int round) {
    const int G = (int)gridDim.x, b = (int)blockIdx.x;
    return round * G + ((snake && (round & 1)) ? G - 1 - b : b);
  };
  auto decode = [&](int it, int& bt, int& split, int& tm, int& tn) {
    if (snake) {
      const int nd = p.tiles_n, nf = p.tiles - nd, full = p.nbatch * p.splits * nf;
      if (it < full) {
        bt = it / (p.splits * nf);
        const int r = it - bt * p.splits * nf;
        split = r / nf;
        const int f = r - split * nf;  // off-diagonal tile f: tm < tn, tn (tn - 1) / 2 <= f
        tn = (int)((1.0f + sqrtf(8.0f * f + 1.0f)) * 0.5f);
        while (tn * (tn - 1) / 2 > f) --tn;
        while ((tn + 1) * tn / 2 <= f) ++tn;
        tm = f - tn * (tn - 1) / 2;
      } else {
        const int j = it - full;
        bt = j / (p.splits * nd);
        const int r = j - bt * p.splits * nd;
        split = r / nd;
        tm = tn = r - split * nd;
      }
      return;
    }
    bt = it / p.per_batch;
    const int rit = it - bt * p.per_batch;
    split = rit / p.tiles;
    tile_of(rit % p.tiles, tm, tn);
  };
  // producer cursor over this CTA's k-slab stream (a work-fetching schedule was tried in
  // r2p - bitwise the same results, but the concurrent per-mode eigensolves ran 0-1 %
  // slower and their step times spread 886-899 ms instead of 889-891, so the static
  // schedule stays)
  int pround = 0, pit = item_at(0), pk = 0, pkend = 0, pm = 0, pn = 0, pka = 0, pkb = 0;
  auto set_item = [&]() {
    if (pit >= p.items) return;
    int bt, split, tm, tn;
    decode(pit, bt, split, tm, tn);
    pm = tm * BM;
    pn = p.n_off + tn * BN;
    pk = split * p.kchunk;
    pkend = min(p.K, pk + p.kchunk);
    pka = bt * p.a_koff;
    pkb = bt * p.b_koff;
  };
  auto issue_next = [&](int stage) {
    if (pit >= p.items) return;
    unsigned char* st = ring + (size_t)stage * p.stage_bytes;
    mbar_arrive_expect_tx(&full[stage], p.tx_bytes);
#pragma unroll
    for (int j = 0; j < KS; ++j) {
      unsigned char* sa_ = st + j * p.a_bytes;
      unsigned char* sb_ = st + KS * p.a_bytes + j * p.b_bytes;
      const int kk = pk + GBK * j;
      if (AK) tma_load_2d(sa_, &tA, kk + pka, pm, &full[stage]);
      else tma_load_2d(sa_, &tA, pm, kk + pka, &full[stage]);
      if (BKM) tma_load_2d(sb_, &tB, kk + pkb, pn, &full[stage]);
      else tma_load_2d(sb_, &tB, pn, kk + pkb, &full[stage]);
    }
    pk += GBK * KS;
    if (pk >= pkend) {
      pit = item_at(++pround);
      set_item();
    }
  };
  if (producer) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], GTHREADS / 32);
    }
    fence_mbar_init();
    tma_prefetch_desc(&tA);
    tma_prefetch_desc(&tB);
  }
  __syncthreads();
  if (producer) {
    set_item();
    for (int s = 0; s < p.stages; ++s) issue_next(s);
  }

  const int fr = lane >> 2, fc = lane & 3;
  const int wm0 = (warp & 1) * WM, wn0 = (warp >> 1) * WN;
  // per-lane byte offsets of the fragment element (row % 8 == fr, k = 4 q + fc)
  uint32_t aoff[GBK / 4], boff[GBK / 4];
#pragma unroll
  for (int q = 0; q < GBK / 4; ++q) {
    const int k = 4 * q + fc;
    aoff[q] = AK ? (uint32_t)((wm0 + fr) * 128) + sw128_off(fr, k) - fr * 128
                 : (uint32_t)((k * APITCH + wm0 + fr) * 8);
    boff[q] = BKM ? (uint32_t)((wn0 + fr) * 128) + sw128_off(fr, k) - fr * 128
                  : (uint32_t)((k * BPITCH + wn0 + fr) * 8);
  }
  constexpr uint32_t ASTEP = AK ? 1024u : 64u, BSTEP = BKM ? 1024u : 64u;  // next 8 rows
  // Diagonal tiles of the symmetric (upper) form, 128 x 128 only: the strictly lower half
  // is not needed, so the warps take 16-row strips of the tile instead of 64 x 32 blocks
  // (the same 64 accumulators: fragment (i', j') of the strip, i' < 2, j' < 16, lives in
  // acc[e >> 2][e & 3], e = 16 i' + j') and skip the fragment columns left of the strip
  // (8 j' + 7 < 16 s: every entry below the diagonal).  Strip s = warp for warps 0-3 and
  // 11 - warp for warps 4-7, so the two warps of each SM sub-partition (warp w and w + 4)
  // hold strips s and 7 - s: 36 of 64 DMMAs per k-step on every sub-partition, where the
  // 64 x 32 blocks left a full 64 on two of them (the tile's DMMA time is set by the
  // busiest sub-partition's tensor pipe).  Diagonal tiles are 12 % of cfg 4's upper tiles.
  const int dstrip = warp < 4 ? warp : 11 - warp;
  uint32_t daoff[GBK / 4], dboff[GBK / 4];
#pragma unroll
  for (int q = 0; q < GBK / 4; ++q) {
    const int k = 4 * q + fc, wmd = 16 * dstrip;
    daoff[q] = AK ? (uint32_t)((wmd + fr) * 128) + sw128_off(fr, k) - fr * 128 : (uint32_t)((k * APITCH + wmd + fr) * 8);
    dboff[q] = BKM ? (uint32_t)(fr * 128) + sw128_off(fr, k) - fr * 128 : (uint32_t)((k * BPITCH + fr) * 8);
  }
  const uint32_t ring_s = smem_u32(ring);
  uint32_t g = 0;
  // ring position of k-tile g (stage g % stages, parity (g / stages) & 1), advanced
  // incrementally: no integer division on the per-stage path
  uint32_t cs = 0, cph = 0;
  const uint32_t nst = (uint32_t)p.stages;
  for (int round = 0;; ++round) {
    const int it = item_at(round);
    if (it >= p.items) break;
    int bt, split, tm, tn;
    decode(it, bt, split, tm, tn);
    double* const Cb = p.C + bt * p.c_bstride;
    const int m0 = tm * BM, n0 = p.n_off + tn * BN;
    const int kbeg = split * p.kchunk, kend = min(p.K, kbeg + p.kchunk);
    const bool diag = kDiag && p.upper && tm == tn;
    // output coordinates of accumulator fragment (i, j): the 64 x 32 warp block, or on a
    // diagonal tile fragment (e >> 4, e & 15) of the warp's 16-row strip, e = FN i + j
    auto frag_m = [&](int i, int j) {
      return diag ? m0 + 16 * dstrip + 8 * ((FN * i + j) >> 4) + fr : m0 + wm0 + i * 8 + fr;
    };
    auto frag_n = [&](int i, int j) { return diag ? n0 + 8 * ((FN * i + j) & 15) + 2 * fc : n0 + wn0 + j * 8 + 2 * fc; };
    double acc[FM][FN][2];
    if (p.epi == EPI_RESID) {
      // residual form: the accumulators start at -D, so after the k-loop they hold
      // op(A)op(B) - D and the epilogue is a sum of squares with no global loads (the
      // short-K residual GEMM used to stall on its D loads after the last DMMA).  Every
      // thread with a column of the NEXT item's D tile prefetches it to L2 now (one bulk
      // prefetch per column, spread over the CTA: a 128-prefetch loop in the producer
      // thread delayed warp 0 and with it the ring, cfg 5 residual 4.6 -> 5.4 ms).
      {
        const int nit = it + (int)gridDim.x;
        if (nit < p.items && tid < BN) {
          const int nm0 = (nit % p.tiles_m) * BM, nn0 = p.n_off + (nit / p.tiles_m) * BN;
          const int rows = min(BM, p.M - nm0) & ~1;
          if (rows > 0 && nn0 + tid < p.N)
            l2_prefetch_bulk(p.D + (int64_t)(nn0 + tid) * p.ldd + nm0, (uint32_t)rows * 8u);
        }
      }
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int m = m0 + wm0 + i * 8 + fr, n = n0 + wn0 + j * 8 + 2 * fc + h;
            acc[i][j][h] = (m < p.M && n < p.N) ? -p.D[(int64_t)n * p.ldd + m] : 0.0;
          }
    } else {
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    }
    for (int k0 = kbeg; k0 < kend; k0 += GBK * KS, ++g) {
      if (producer && g >= 1) {
        const uint32_t sp = cs == 0 ? nst - 1 : cs - 1, php = cs == 0 ? cph ^ 1u : cph;
        mbar_wait(&empty[sp], php);
        issue_next((int)sp);
      }
      const uint32_t s = cs;
      mbar_wait(&full[s], cph);
      if (kDiag && diag) {
        // one unrolled body per strip (a warp-uniform switch): predicated-off DMMAs still
        // occupied the tensor pipe (measured: no gain with a predicate per fragment pair)
        auto body = [&](auto S) {
          constexpr int ST = decltype(S)::value;
#pragma unroll
          for (int js = 0; js < KS; ++js) {
            const uint32_t sa = ring_s + s * p.stage_bytes + js * p.a_bytes;
            const uint32_t sb = ring_s + s * p.stage_bytes + KS * p.a_bytes + js * p.b_bytes;
#pragma unroll
            for (int q = 0; q < GBK / 4; ++q) {
              double af[2], bf[16 - 2 * ST];
#pragma unroll
              for (int i = 0; i < 2; ++i) af[i] = lds_f64(sa + daoff[q] + i * ASTEP);
#pragma unroll
              for (int j = 2 * ST; j < 16; ++j) bf[j - 2 * ST] = lds_f64(sb + dboff[q] + j * BSTEP);
#pragma unroll
              for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 2 * ST; j < 16; ++j) {
                  const int e = 16 * i + j;
                  dmma_8x8x4(acc[e >> 2][e & 3][0], acc[e >> 2][e & 3][1], af[i], bf[j - 2 * ST]);
                }
            }
          }
        };
        switch (dstrip) {
          case 0: body(std::integral_constant<int, 0>{}); break;
          case 1: body(std::integral_constant<int, 1>{}); break;
          case 2: body(std::integral_constant<int, 2>{}); break;
          case 3: body(std::integral_constant<int, 3>{}); break;
          case 4: body(std::integral_constant<int, 4>{}); break;
          case 5: body(std::integral_constant<int, 5>{}); break;
          case 6: body(std::integral_constant<int, 6>{}); break;
          default: body(std::integral_constant<int, 7>{}); break;
        }
      } else {
#pragma unroll
      for (int js = 0; js < KS; ++js) {
      const uint32_t sa = ring_s + s * p.stage_bytes + js * p.a_bytes;
      const uint32_t sb = ring_s + s * p.stage_bytes + KS * p.a_bytes + js * p.b_bytes;
#pragma unroll
      for (int q = 0; q < GBK / 4; ++q) {
        double af[FM], bf[FN];
#pragma unroll
        for (int i = 0; i < FM; ++i) af[i] = lds_f64(sa + aoff[q] + i * ASTEP);
#pragma unroll
        for (int j = 0; j < FN; ++j) bf[j] = lds_f64(sb + boff[q] + j * BSTEP);
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
      }
      }
      __syncwarp();
      // release the stage only once its last fragment loads have been consumed: the
      // compiler hoisted a plain arrive above the stage's last DMMAs, and the producer's
      // next TMA into the stage could then overwrite fragments still being read (a
      // transiently wrong GEMM, seen as a wrong rank residual in ~2 % of cfg 4 calls)
      if (lane == 0) mbar_arrive_after(&empty[s], acc[FM - 1][FN - 1][1]);
      if (++cs == nst) {
        cs = 0;
        cph ^= 1u;
      }
    }

    // ---- epilogue
    if (p.epi == EPI_RESID) {
      // acc = op(A)op(B) - D (zero outside the matrix: zero-filled operands, zero start)
      double ss = 0.0;
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) ss = fma(acc[i][j][h], acc[i][j][h], ss);
      ss = warp_sum(ss);
      // per-warp partials in fixed slots; summed in fixed order by sum_fixed_order_kernel
      if (lane == 0) p.part[(int64_t)it * (GTHREADS / 32) + warp] = ss;
      continue;
    }
    if (p.splits > 1) {
      double* out = p.part + ((int64_t)bt * p.splits + split) * p.M * p.N;
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            int m = frag_m(i, j), n = frag_n(i, j) + h;
            if (m < p.M && n < p.N) out[(int64_t)n * p.M + m] = acc[i][j][h];
          }
      continue;
    }
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int m = frag_m(i, j), n = frag_n(i, j) + h;
          if (m < p.M && n < p.N && (!p.upper || m <= n)) {
            double v = p.alpha * acc[i][j][h];
            if (p.cs) v *= p.cs[n];
            if (p.rs) v *= p.rs[m];
            double* c = Cb + (int64_t)n * p.ldc + m;
            if (p.beta != 0.0) v = fma(p.beta, *c, v);
            *c = v;
            if (p.upper && m < n) Cb[(int64_t)m * p.ldc + n] = v;  // mirror (M == N)
          }
        }
  }
}

// Fixed-order split-K reduction + epilogue (and symmetric mirror).
__global__ void splitk_reduce_kernel(GParams p) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = (int64_t)p.M * p.N;
  if (idx >= total * p.nbatch) return;
  const int bt = (int)(idx / total);
  idx -= bt * total;
  int m = (int)(idx % p.M), n = (int)(idx / p.M);
  int sm = m, sn = n;
  if (p.upper && m > n) { sm = n; sn = m; }  // read the computed upper entry
  int64_t src = (int64_t)sn * p.M + sm;
  const double* part = p.part + (int64_t)bt * p.splits * total;
  double s = 0.0;
  for (int k = 0; k < p.splits; ++k) s += part[(int64_t)k * total + src];
  double v = p.alpha * s;
  if (p.cs) v *= p.cs[n];
  if (p.rs) v *= p.rs[m];
  double* c = p.C + bt * p.c_bstride + (int64_t)n * p.ldc + m;
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

// k-slabs per pipeline stage (one mbarrier round trip each): 2, RHOSVD_GEMM_KS=1 for 1
static int gemm_ks() {
  static const int ks = [] {
    const char* e = getenv("RHOSVD_GEMM_KS");
    return (e && atoi(e) == 1) ? 1 : 2;
  }();
  return ks;
}

template <int BM, int BN, bool AK, bool BKM, int KS>
static int launch_cfg(const GemmArgs& g, GParams gp, cudaStream_t st) {
  auto kern = tma_gemm_kernel<BM, BN, AK, BKM, KS>;
  CUtensorMap tA, tB;
  // batched: the k-extent of the maps spans every batch (batch b at k + b * koff)
  const int64_t KA = g.K + (int64_t)(gp.nbatch - 1) * gp.a_koff, KB = g.K + (int64_t)(gp.nbatch - 1) * gp.b_koff;
  if (AK) RH_CHECK(make_tmap_2d(&tA, g.A, g.M, KA, g.lda, GBK, BM, true));
  else RH_CHECK(make_tmap_2d(&tA, g.A, KA, g.M, g.lda, BM + 8, GBK, false));
  if (BKM) RH_CHECK(make_tmap_2d(&tB, g.B, g.N, KB, g.ldb, GBK, BN, true));
  else RH_CHECK(make_tmap_2d(&tB, g.B, KB, g.N, g.ldb, BN + 8, GBK, false));
  const uint32_t a_box = AK ? BM * 128u : (BM + 8) * GBK * 8u;
  const uint32_t b_box = BKM ? BN * 128u : (BN + 8) * GBK * 8u;
  gp.a_bytes = (uint32_t)round_up(a_box, 1024);
  gp.b_bytes = (uint32_t)round_up(b_box, 1024);
  gp.stage_bytes = KS * (gp.a_bytes + gp.b_bytes);
  gp.tx_bytes = KS * (a_box + b_box);
  const size_t budget = 227 * 1024 - 1024 - 256;
  gp.stages = (int)std::min<size_t>(8, budget / gp.stage_bytes);
  const size_t smem = 1024 + (size_t)gp.stages * gp.stage_bytes + 2 * gp.stages * sizeof(uint64_t);
  static const cudaError_t attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                        227 * 1024);  // per instantiation, thread-safe
  RH_CUDA(attr);
  const int grid = (int)std::min<int64_t>(gp.items, num_sms());
  kern<<<grid, GTHREADS, smem, st>>>(tA, tB, gp);
  count_launch();
  RH_LAUNCH_CHECK();
  return RHOSVD_OK;
}

template <int BM, int BN, int KS>
static int launch_layout_ks(const GemmArgs& g, const GParams& gp, cudaStream_t st) {
  if (g.a_k && g.b_k) return launch_cfg<BM, BN, true, true, KS>(g, gp, st);
  if (g.a_k && !g.b_k) return launch_cfg<BM, BN, true, false, KS>(g, gp, st);
  if (!g.a_k && g.b_k) return launch_cfg<BM, BN, false, true, KS>(g, gp, st);
  return launch_cfg<BM, BN, false, false, KS>(g, gp, st);
}
template <int BM, int BN>
static int launch_layout(const GemmArgs& g, const GParams& gp, cudaStream_t st) {
  return gemm_ks() == 2 ? launch_layout_ks<BM, BN, 2>(g, gp, st) : launch_layout_ks<BM, BN, 1>(g, gp, st);
}
// the narrow last column segment of a 128 x 128 GEMM (KS 2 only)
static int launch_edge(int bn, const GemmArgs& g, const GParams& gp, cudaStream_t st) {
  switch (bn) {
    case 32: return launch_layout_ks<128, 32, 2>(g, gp, st);
    case 64: return launch_layout_ks<128, 64, 2>(g, gp, st);
    case 96: return launch_layout_ks<128, 96, 2>(g, gp, st);
    default: return fail(RHOSVD_EINVAL, "gemm: unsupported edge width");
  }
}

static bool gemm_big(int64_t M, int64_t N, int64_t K) {
  // (long-K products with N a little under 128, e.g. cfg 5's M = Uhat W^T with b = 124:
  // the 128 x 128 engine with 4 padded columns beats 64 x 64 tiles, DMMA pipe 84 -> 9x %)
  return (cdiv(M, 128) * cdiv(N, 128) >= num_sms() / 2) || (M >= 128 && N >= 128 && K >= 2048) ||
         (M >= 128 && N >= 96 && K >= 16384);
}

int gemm_batch_splits(int64_t M, int64_t N, int64_t K, bool upper, int nb) {
  // the cheapest wave schedule over the K-split count (a split costs one more M x N partial
  // per batch, ~0.3 % here, and a fixed per-item cost).  cfg 4's three 2048^2 Grams: 408
  // upper tiles -> 5 splits = 2040 items on 148 SMs, 98.4 % of the last wave busy (one
  // 136-tile Gram per launch: 92 %)
  const int sms = num_sms();
  const int BT = gemm_big(M, N, K) ? 128 : 64;
  const int64_t tn = cdiv(N, BT), tiles = upper ? tn * (tn + 1) / 2 : cdiv(M, BT) * tn;
  const int64_t tot = (int64_t)nb * tiles;
  // few tiles (cfg 2: 3 x 10 upper tiles of a 512^2 Gram) need deep splits: chunks down to
  // 256 of K, up to 64 splits; otherwise chunks >= 2048, up to 8 splits
  const bool few = tot < sms;
  const int smax = few ? 64 : 8;
  const int64_t kmin = few ? 256 : 2048;
  double best = 1e30;
  int splits = 1;
  for (int s2 = 1; s2 <= smax; ++s2) {
    if (s2 > 1 && K / s2 < kmin) break;
    // waves x (k per item + ~256 k of fixed cost per item: pipeline fill, epilogue)
    const double cost = (double)cdiv(tot * s2, sms) * ((double)cdiv(K, s2) + 256.0) * (1.0 + 0.003 * (s2 - 1));
    if (cost < best * 0.999) {
      best = cost;
      splits = s2;
    }
  }
  return splits;
}

// K-split count of a single GEMM: the cheapest wave schedule, in units of one tile's
// k-step time per SM: waves x (k per item + ~256 k of fixed per-item cost: pipeline fill,
// epilogue) + the split-K partials' HBM round trip ((s + 1) M N doubles at ~6.5 TB/s).
// Chunks stay >= 256 of K, at most 64 splits.  (The former rule - ~2 items per SM when
// the tiles do not fill the GPU - ran cfg 5's M = Uhat W^T (32 tiles, K = 100 000) as
// 10 splits = 3 waves where 9 splits fit in 2, and cfg 4's (96 tiles) as 4 splits = 3
// waves where 3 fit in 2.)
// Small GEMMs (< 30 GFLOP: the latency-bound Gram-domain and small-config products, which
// run three at a time under the concurrent modes) keep the older rule, ~2 items per SM
// when the tiles do not fill the GPU: the model's fixed cost made cfg 3's few-tile
// products use fewer splits, and its eigensolve got 0.4 ms slower (r2p).
static int gemm_plain_splits(int64_t tiles, int BT, int64_t M, int64_t N, int64_t K) {
  const int sms = num_sms();
  if (2.0 * (double)M * (double)N * (double)K < 3e10) {
    if (tiles >= sms) return 1;
    const int64_t want = cdiv(2LL * sms, tiles), maxs = std::max<int64_t>(1, K / 256);
    return (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(want, maxs), 64));
  }
  // seconds per k-unit of one BT x BT tile on one SM at the DMMA rate (37.2 TF / 148)
  const double t_k = 2.0 * BT * BT / (37.2e12 / 148.0);
  double best = 1e300;
  int splits = 1;
  for (int s2 = 1; s2 <= 64; ++s2) {
    if (s2 > 1 && K / s2 < 256) break;
    double cost = (double)cdiv(tiles * s2, sms) * ((double)cdiv(K, s2) + 256.0) * (1.0 + 0.003 * (s2 - 1));
    if (s2 > 1) cost += (double)(s2 + 1) * (double)M * (double)N * 8.0 / 6.5e12 / t_k;
    if (cost < best * 0.999) {
      best = cost;
      splits = s2;
    }
  }
  return splits;
}

int gemm(const GemmArgs& g, Scratch& scr, cudaStream_t st, double* flops_acc) {
  if (g.M <= 0 || g.N <= 0) return RHOSVD_OK;
  if (g.M > INT32_MAX || g.N > INT32_MAX || g.K > INT32_MAX)
    return fail(RHOSVD_EINVAL, "gemm: dimension exceeds int32");
  if (g.upper_sym && g.M != g.N) return fail(RHOSVD_EINVAL, "gemm: upper_sym needs M == N");
  if (g.epi == EPI_RESID && g.K <= 0) return fail(RHOSVD_EINVAL, "gemm: residual needs K > 0");
  const int nb = std::max(1, g.batch);
  if (nb > 1) {
    if (g.epi == EPI_RESID) return fail(RHOSVD_EINVAL, "gemm: batched form has no residual epilogue");
    if (g.K <= 0 || g.K % 32 || g.a_koff % 32 || g.b_koff % 32 || g.a_koff < g.K || g.b_koff < g.K)
      return fail(RHOSVD_EINVAL, "gemm: batched K / k offsets must be multiples of 32 with koff >= K");
  }
  GParams gp{};
  gp.M = (int)g.M; gp.N = (int)g.N; gp.K = (int)std::max<int64_t>(g.K, 0);
  gp.nbatch = nb;
  gp.a_koff = (int)g.a_koff;
  gp.b_koff = (int)g.b_koff;
  gp.c_bstride = g.c_bstride;
  gp.C = g.C; gp.ldc = g.ldc; gp.alpha = g.alpha; gp.beta = g.beta; gp.cs = g.col_scale; gp.rs = g.row_scale;
  gp.upper = g.upper_sym ? 1 : 0; gp.epi = g.epi; gp.D = g.D; gp.ldd = g.ldd;

  // tile choice: 128 x 128 when there is enough output to fill the GPU
  const int sms = num_sms();
  const bool big = gemm_big(g.M, g.N, g.K);
  const int BT = big ? 128 : 64;
  const int tm = (int)cdiv(g.M, BT), tn = (int)cdiv(g.N, BT);
  gp.tiles_m = tm;
  gp.tiles_n = tn;
  gp.tiles = g.upper_sym ? tn * (tn + 1) / 2 : tm * tn;

  int splits = g.splits;
  if (g.epi == EPI_RESID) splits = 1;
  if (splits <= 0 && nb > 1) splits = gemm_batch_splits(g.M, g.N, g.K, g.upper_sym, nb);
  if (splits <= 0) splits = gemm_plain_splits(gp.tiles, BT, g.M, g.N, g.K);
  int kchunk = (int)round_up(cdiv(std::max<int64_t>(g.K, 1), splits), GBK * gemm_ks());
  splits = (int)std::max<int64_t>(1, cdiv(std::max<int64_t>(g.K, 1), kchunk));
  gp.splits = splits;
  gp.kchunk = kchunk;
  gp.per_batch = gp.tiles * splits;
  gp.items = gp.per_batch * nb;

  if (g.epi == EPI_RESID) {
    RH_CHECK(scr.ensure((size_t)gp.items * (GTHREADS / 32), st));
    gp.part = scr.ptr;
  } else if (splits > 1) {
    RH_CHECK(scr.ensure((size_t)nb * splits * g.M * g.N, st));
    gp.part = scr.ptr;
  }
  if (g.K <= 0) {  // empty contraction: C = beta C
    GParams z = gp;
    z.splits = 1;
    RH_CHECK(scr.ensure((size_t)g.M * g.N, st));  // ENOMEM goes back to the caller
    RH_CUDA(cudaMemsetAsync(scr.ptr, 0, (size_t)g.M * g.N * sizeof(double), st));
    z.part = scr.ptr;
    splitk_reduce_kernel<<<(unsigned)cdiv(g.M * g.N, 256), 256, 0, st>>>(z);
    count_launch();
    RH_LAUNCH_CHECK();
    return RHOSVD_OK;
  }
  // column edge: N % 128 leftover columns as one narrower segment (BN 32 / 64 / 96) so
  // the last column tile does not run padded DMMAs (b = 730: 768 -> 736 columns; b = 147:
  // 256 -> 160).  Not for the symmetric (upper-tile) or residual-epilogue forms.
  // RHOSVD_GEMM_EDGE=0 disables it.  (Before the ring fix of r1z, profiles/README.md, the
  // extra launches made that race visible as run-to-run differences on cfg 3; after it,
  // 250 cfg 3 calls with the edge were bitwise identical.)
  static const bool edge_on = [] {
    const char* e = getenv("RHOSVD_GEMM_EDGE");
    return !(e && e[0] == '0');
  }();
  const int64_t rem = g.N % 128;
  const int ebn = (int)round_up(rem, 32);
  bool use_edge = big && edge_on && nb == 1 && !g.upper_sym && g.epi != EPI_RESID && gemm_ks() == 2 && g.N > 128 &&
                  rem > 0 && ebn < 128;
  if (use_edge) {
    // waves of 128-tile time: the two launches each end on their own partial wave, so the
    // edge only pays when it removes more padding than it adds tail (an edge tile costs
    // ~(ebn + 16) / 128 of a full one)
    const int64_t i1 = (int64_t)tm * (g.N / 128) * splits, i2 = (int64_t)tm * splits, ia = (int64_t)gp.tiles * splits;
    const double c_edge = (double)cdiv(i1, sms) + (double)cdiv(i2, sms) * (ebn + 16) / 128.0;
    const double c_pad = (double)cdiv(ia, sms);
    use_edge = c_edge < 0.95 * c_pad;
  }
  if (use_edge) {
    GParams g1 = gp;
    g1.tiles_n = (int)(g.N / 128);
    g1.tiles = tm * g1.tiles_n;
    g1.per_batch = g1.items = g1.tiles * splits;
    g1.n_off = 0;
    RH_CHECK((launch_layout<128, 128>(g, g1, st)));
    GParams g2 = gp;
    g2.tiles_n = 1;
    g2.tiles = tm;
    g2.per_batch = g2.items = g2.tiles * splits;
    g2.n_off = (int)(g.N - rem);
    RH_CHECK(launch_edge(ebn, g, g2, st));
  } else if (big) {
    RH_CHECK((launch_layout<128, 128>(g, gp, st)));
  } else {
    RH_CHECK((launch_layout<64, 64>(g, gp, st)));
  }

  if (g.epi == EPI_RESID) {
    sum_fixed_order_kernel<<<1, 256, 0, st>>>(gp.part, gp.items * (GTHREADS / 32), g.resid_out);
    count_launch();
    RH_LAUNCH_CHECK();
  } else if (splits > 1) {
    int64_t total = g.M * g.N * nb;
    splitk_reduce_kernel<<<(unsigned)cdiv(total, 256), 256, 0, st>>>(gp);
    count_launch();
    RH_LAUNCH_CHECK();
  }
  if (flops_acc) *flops_acc += 2.0 * nb * (double)g.M * (double)g.N * (double)g.K * (g.upper_sym ? 0.5 : 1.0);
  return RHOSVD_OK;
}

}  // namespace rhosvd
