// core_kr.cu - K7: the RHOSVD core as a Khatri-Rao DMMA contraction (sm_100a, FP64).
//
// Prop. 2.1: the core beta_0 = xi x_1 U_0^(1)T x_2 U_0^(2)T x_3 U_0^(3)T
// of the RHOSVD Tucker tensor is the rank-R CP tensor with factors W_l = Z_l^T Uhat_l,
// "calculated entry-wise in O(R r1 ... rd) operations".  We compute it densely as
//     beta_(12)(3) = (W1 (.) W2) (xi' o W3)^T      M = r1 r2, N = r3, K = R
// with the Khatri-Rao operand never materialised (152 GiB on cfg 4).
//
// Design (B200):
//  * M is the FLATTENED Khatri-Rao row index m = a r2 + b, tiled by BM = 128, so the
//    only padding is the ragged end of r1 r2 (no per-mode padding of r2).  N = r3 is
//    tiled by BN in {64, 96, 128}, chosen per call to minimise padding.
//  * Operands arrive by TMA (cp.async.bulk.tensor.2d, 128-B swizzle, 16-double k
//    slabs): per k-slab, one box of A1 = (BM-1)/r2 + 2 rows of xi' o W1 (every a the
//    tile touches), one box of 128 rows of W2ext (W2 with its first rows repeated
//    after the end, so the wrap b -> 0 inside a tile is a contiguous box), one box of
//    BN rows of W3.  Out-of-range rows/columns are zero-filled by TMA (ragged R, r1).
//  * Pipeline: thread 0 issues TMA into a STAGES-deep ring guarded by full/empty
//    mbarriers (it refills the stage the 8 warps released one step earlier, so the
//    ring stays STAGES-1 slabs ahead); 8 warps stacked along M (warp tile 16 x BN, so no
//    Khatri-Rao row is formed twice; 2 warps per SM sub-partition so each may hold 255
//    registers - a 9th producer warp would cap them at 168) form each A fragment in
//    registers as W1[a,k] * W2[b,k] (one DMUL) and
//    issue mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4 - the only FP64 tensor instruction on
//    sm_100a; tcgen05 has no f64 kind).
//  * Persistent grid (one CTA per SM, static stride over work items) so all CTAs
//    stream the same k-slabs at the same time and the W tiles are L2 hits.
//  * Small problems split K; partials go to scratch and a second kernel sums them in
//    fixed order (deterministic, no FP64 atomics; reading A18).
// Output beta[a,b,c] in C order (c fastest).
#include <algorithm>
#include <cstdlib>

#include "kernels.h"
#include "tma.cuh"

namespace rhosvd {

constexpr int CORE_BM = 128, CORE_BK = 16, CORE_WARPS = 8;
constexpr int CORE_THREADS = 32 * CORE_WARPS;

struct CoreArgs {
  int r1, r2, r3, R;
  int A1;            // W1 rows per box
  int A1pad;         // rounded to 8 (1024-B aligned sub-tiles)
  int mt, nt, tiles, splits, kchunk, items;
  int tm0;           // first row tile of this launch (row-chunked launches)
  int n_off, n_end;  // column segment [n_off, n_end) of this launch (edge segments)
  int stages;
  uint32_t stage_bytes, tx_bytes;
  double* out;       // beta (splits == 1) or partials [split][r1 r2 r3]
};

template <int BN, int KSUB>
__global__ void __launch_bounds__(CORE_THREADS, 1)
    core_kr_tma_kernel(const __grid_constant__ CUtensorMap tW1, const __grid_constant__ CUtensorMap tW2,
                       const __grid_constant__ CUtensorMap tW3, const CoreArgs p) {
  constexpr int WM = 16, FM = 2, FN = BN / 8;  // 8 warps stacked along M, each 16 x BN
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-B align the ring (128-B swizzle atoms); offsetting the __shared__ array keeps
  // the address space visible to the compiler (LDS, 32-bit addressing)
  unsigned char* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = (uint64_t*)(ring + (size_t)p.stages * p.stage_bytes);
  uint64_t* empty = full + p.stages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool producer = (tid == 0);
  const int M = p.r1 * p.r2;
  const uint32_t w2_off = (uint32_t)p.A1pad * 128, w3_off = w2_off + CORE_BM * 128;
  const uint32_t slab = p.stage_bytes / KSUB;  // one 16-wide k-slab of W1 | W2ext | W3

  // producer cursor over this CTA's k-tile stream (items strided by gridDim.x); the
  // item's box coordinates are recomputed only when the cursor moves to a new item
  int pit = blockIdx.x, pk = 0, pkend = 0, pa = 0, pb = 0, pn = 0;
  auto set_item = [&]() {
    if (pit >= p.items) return;
    const int split = pit / p.tiles, tile = pit % p.tiles;
    const int m0 = (p.tm0 + tile % p.mt) * CORE_BM;
    pk = split * p.kchunk;
    pkend = min(p.R, pk + p.kchunk);
    pa = m0 / p.r2;
    pb = m0 % p.r2;
    pn = p.n_off + (tile / p.mt) * BN;
  };
  auto issue_next = [&](int stage) {
    if (pit >= p.items) return;
    unsigned char* st = ring + (size_t)stage * p.stage_bytes;
    mbar_arrive_expect_tx(&full[stage], p.tx_bytes);
#pragma unroll
    for (int j = 0; j < KSUB; ++j) {
      tma_load_2d(st + j * slab, &tW1, pk + 16 * j, pa, &full[stage]);
      tma_load_2d(st + j * slab + w2_off, &tW2, pk + 16 * j, pb, &full[stage]);
      tma_load_2d(st + j * slab + w3_off, &tW3, pk + 16 * j, pn, &full[stage]);
    }
    pk += CORE_BK * KSUB;
    if (pk >= pkend) {
      pit += gridDim.x;
      set_item();
    }
  };

  if (producer) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CORE_WARPS);
    }
    fence_mbar_init();
    tma_prefetch_desc(&tW1);
    tma_prefetch_desc(&tW2);
    tma_prefetch_desc(&tW3);
  }
  __syncthreads();
  if (producer) {
    set_item();
    for (int s = 0; s < p.stages; ++s) issue_next(s);
  }

  const int fr = lane >> 2, fc = lane & 3;
  const int wm0 = warp * WM;
  // per-lane byte offsets of (row with row%8 == fr, k = kk + fc) inside a swizzled slab
  uint32_t koff[CORE_BK / 4];
#pragma unroll
  for (int q = 0; q < CORE_BK / 4; ++q) koff[q] = sw128_off(fr, 4 * q + fc) - fr * 128;
  const uint32_t ring_s = smem_u32(ring);
  uint32_t g = 0;  // k-tiles consumed by this CTA
  // ring position of k-tile g (stage g % stages, parity (g / stages) & 1), advanced
  // incrementally: no integer division on the per-stage path
  uint32_t cs = 0, cph = 0;
  const uint32_t nst = (uint32_t)p.stages;
  for (int it = blockIdx.x; it < p.items; it += gridDim.x) {
    const int split = it / p.tiles, tile = it % p.tiles;
    const int tm = p.tm0 + tile % p.mt, tn = tile / p.mt;
    const int m0 = tm * CORE_BM, n0 = p.n_off + tn * BN;
    const int a_lo = m0 / p.r2;
    const int kbeg = split * p.kchunk, kend = min(p.R, kbeg + p.kchunk);
    // W1 row (inside the box) of each fragment row this lane touches -> byte offsets
    uint32_t w1off[FM][CORE_BK / 4];
#pragma unroll
    for (int i = 0; i < FM; ++i) {
      const int m = min(m0 + wm0 + i * 8 + fr, M - 1);
      const int row = m / p.r2 - a_lo;
#pragma unroll
      for (int q = 0; q < CORE_BK / 4; ++q) w1off[i][q] = sw128_off(row, 4 * q + fc);
    }
    double acc[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int k0 = kbeg; k0 < kend; k0 += CORE_BK * KSUB, ++g) {
      // refill the stage released one step ago (its 8 warps are done with it)
      if (producer && g >= 1) {
        const uint32_t sp = cs == 0 ? nst - 1 : cs - 1, php = cs == 0 ? cph ^ 1u : cph;
        mbar_wait(&empty[sp], php);
        issue_next((int)sp);
      }
      const uint32_t s = cs;
      mbar_wait(&full[s], cph);
#pragma unroll
      for (int js = 0; js < KSUB; ++js) {
      const uint32_t w1 = ring_s + s * p.stage_bytes + js * slab;
      const uint32_t w2 = w1 + w2_off + (wm0 + fr) * 128;
      const uint32_t w3 = w1 + w3_off + fr * 128;
#pragma unroll
      for (int q = 0; q < CORE_BK / 4; ++q) {
        double af[FM], bf[FN];
#pragma unroll
        for (int i = 0; i < FM; ++i) af[i] = lds_f64(w1 + w1off[i][q]) * lds_f64(w2 + koff[q] + i * 1024);
#pragma unroll
        for (int j = 0; j < FN; ++j) bf[j] = lds_f64(w3 + koff[q] + j * 1024);
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int jn = 0; jn < FN; ++jn) dmma_8x8x4(acc[i][jn][0], acc[i][jn][1], af[i], bf[jn]);
      }
      }
      __syncwarp();
      // release the stage only once its last fragment loads have been consumed (an arrive
      // hoisted above them let the next TMA overwrite data still being read)
      if (lane == 0) mbar_arrive_after(&empty[s], acc[FM - 1][FN - 1][1]);
      if (++cs == nst) {
        cs = 0;
        cph ^= 1u;
      }
    }
    // epilogue: rows m (flattened a r2 + b), columns n of beta_(12)(3)
    double* out = p.out + (p.splits > 1 ? (int64_t)split * M * p.r3 : 0);
    const bool even = (p.r3 & 1) == 0;
#pragma unroll
    for (int i = 0; i < FM; ++i) {
      const int m = m0 + wm0 + i * 8 + fr;
      if (m >= M) continue;
      double* row = out + (int64_t)m * p.r3;
#pragma unroll
      for (int j = 0; j < FN; ++j) {
        const int n = n0 + j * 8 + 2 * fc;
        if (even && n + 1 < p.n_end) {
          *(double2*)(row + n) = make_double2(acc[i][j][0], acc[i][j][1]);
        } else {
          if (n < p.n_end) row[n] = acc[i][j][0];
          if (n + 1 < p.n_end) row[n + 1] = acc[i][j][1];
        }
      }
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

// W2ext[j] = W2[j mod r2] for j < r2 + ext (row-major, ld ldw -> ldo)
__global__ void wrap_rows_kernel(const double* W, int64_t ldw, int r2, int ext, int R, double* out, int64_t ldo) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)(r2 + ext) * R) return;
  int j = (int)(e / R), k = (int)(e % R);
  out[(int64_t)j * ldo + k] = W[(int64_t)(j % r2) * ldw + k];
}


static int pick_bn(int64_t r3) {
  // executed columns (the leftover r3 % BN as an edge segment padded to 16, or a padded
  // tile when that is no narrower) + ~8 column-equivalents of fixed cost per tile (A
  // fragment formation, pipeline fill, epilogue) - fitted on cfg 4 (r3 = 652): BN 128 +
  // edge 16: 789 ms, 96 + edge 80: 799 ms, 64 + edge 16: 834 ms, 96 padded: 809 ms
  const int cand[3] = {128, 96, 64};
  int best = 128;
  double bc = 1e300;
  for (int bn : cand) {
    const int64_t full = r3 / bn, rem = r3 - full * bn;
    double cols, tiles;
    if (rem == 0) {
      cols = (double)r3;
      tiles = (double)full;
    } else if (full > 0 && round_up(rem, 16) < bn) {
      // a narrow edge runs fewer DMMAs per fragment load: its columns cost 1 + (64 - w) / 128
      // of a wide tile's (cfg 2, r3 = 282: 2 x 128 + a 32-wide edge 3.57 ms, 3 x 96 padded
      // 3.37 ms - the unweighted count tied them and kept the edge)
      const double w = (double)round_up(rem, 16);
      cols = (double)(full * bn) + w * (w < 64.0 ? 1.0 + (64.0 - w) / 128.0 : 1.0);
      tiles = (double)full + 1.0;
    } else {
      cols = (double)(full + 1) * bn;
      tiles = (double)full + 1.0;
    }
    const double c = cols + 8.2 * tiles;
    if (c < bc) {
      bc = c;
      best = bn;
    }
  }
  return best;
}

// split-K factor for a problem (1 when the tiles alone fill the GPU)
static int core_splits(int64_t r1, int64_t r2, int64_t r3, int64_t R, int BN) {
  const int64_t tiles = cdiv(r1 * r2, CORE_BM) * cdiv(r3, BN);
  const int sms = num_sms();
  if (tiles >= sms || R < 2048) return 1;
  int s = (int)std::min<int64_t>(cdiv(sms, tiles), R / 1024);
  return std::max(1, std::min(s, 32));
}

// Tile plan of one core call.  The default (pick_bn + core_splits + an edge segment for the
// r3 % BN leftover) suits cores with many row tiles (cfg 4: 3317 x 5).  When the tiles do
// not fill a few waves (cfg 5: r1 r2 = 11 664 rows -> 92 row tiles; r3 = 108 -> a 96-wide
// and a 16-wide launch of 92 items each on 148 SMs, ~0.5 of the DMMA peak), a
// single-segment plan of width bn >= r3 / nt with a K-split that fills whole waves is
// cheaper; both are costed with the same model:
//   item time ~ (K / s) (bn + 8.2) (x 1/0.6 for the 16-wide edge), waves = ceil(items / SMs),
//   plus the split-K reduction ((s + 1) r1 r2 r3 doubles through HBM).
struct CorePlan {
  int bn = 128, splits = 1;
  bool single = false;  // one segment, no edge
};
static double core_seg_cost(int64_t tiles, int64_t K, int bn, int s, int sms) {
  const double per_item = (double)cdiv(K, s) * (bn + 8.2) * (bn <= 16 ? 1.0 / 0.6 : 1.0);
  return (double)cdiv(tiles * s, sms) * per_item;
}
static CorePlan core_plan(int64_t r1, int64_t r2, int64_t r3, int64_t R, int force_bn) {
  CorePlan d;
  d.bn = force_bn ? force_bn : pick_bn(r3);
  d.splits = core_splits(r1, r2, r3, R, d.bn);
  static const bool plan_on = [] {  // RHOSVD_CORE_PLAN=0: the default plan only
    const char* e = getenv("RHOSVD_CORE_PLAN");
    return !(e && e[0] == '0');
  }();
  const int sms = num_sms();
  const int64_t mt = cdiv(r1 * r2, CORE_BM);
  if (!plan_on || force_bn || mt * cdiv(r3, d.bn) >= 4 * sms || R < 4096) return d;
  // unit conversion: one (k, column) of a 128-row tile = 256 FLOP at the per-SM DMMA rate
  // (~2.5e11 FLOP/s); the reduction streams (s + 1) r1 r2 r3 doubles at ~6e12 B/s
  const double unit_s = 256.0 / 2.5e11, total = (double)r1 * r2 * r3;
  auto red = [&](int s) { return s > 1 ? (double)(s + 1) * total * 8.0 / 6e12 / unit_s : 0.0; };
  // the default plan, as core_kr would run it
  double best;
  {
    const int64_t full = (r3 / d.bn) * d.bn, rem = r3 - full;
    if (d.splits == 1 && rem > 0 && full > 0 && round_up(rem, 16) < d.bn)
      best = core_seg_cost(mt * (full / d.bn), R, d.bn, 1, sms) + core_seg_cost(mt, R, (int)round_up(rem, 16), 1, sms);
    else
      best = core_seg_cost(mt * cdiv(r3, d.bn), R, d.bn, d.splits, sms) + red(d.splits);
  }
  CorePlan out = d;
  const int cand[] = {64, 80, 96, 112, 128};
  for (int bn : cand) {
    const int64_t nt = cdiv(r3, bn);
    if (nt > 1 && bn < 128) continue;  // narrow single segments only when one column tile covers r3
    for (int sp = 1; sp <= 32 && R / sp >= 512; ++sp) {
      const double c = core_seg_cost(mt * nt, R, bn, sp, sms) + red(sp);
      if (c < best * 0.98) {
        best = c;
        out.bn = bn;
        out.splits = sp;
        out.single = true;
      }
    }
  }
  return out;
}

// split-K scratch (doubles) the call needs; 0 when no split is used
size_t core_part_doubles(int64_t r1, int64_t r2, int64_t r3, int64_t R) {
  static const int force_bn = [] {
    const char* e = getenv("RHOSVD_CORE_BN");
    const int v = e ? atoi(e) : 0;
    return (v == 64 || v == 80 || v == 96 || v == 112 || v == 128) ? v : 0;
  }();
  const int s = core_plan(r1, r2, r3, R, force_bn).splits;
  return s > 1 ? (size_t)s * r1 * r2 * r3 : 0;
}

size_t core_ws_doubles(int64_t r2, int64_t R, int64_t ldw) {
  return (size_t)(r2 + CORE_BM) * std::max<int64_t>(ldw, round_up(std::max<int64_t>(R, 2), 16));
}

template <int BN, int KSUB>
static int launch_core(const CUtensorMap& t1, const CUtensorMap& t2, const CUtensorMap& t3, const CoreArgs& a,
                       size_t smem, int grid, cudaStream_t st) {
  auto kern = core_kr_tma_kernel<BN, KSUB>;
  RH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<grid, CORE_THREADS, smem, st>>>(t1, t2, t3, a);
  count_launch();
  RH_LAUNCH_CHECK();
  return RHOSVD_OK;
}

// host entry: beta (r1 x r2 x r3, C order) = sum_k W1x[:,k] (x) W2[:,k] (x) W3[:,k]
// W1x must already hold xi' o W1.  All W row-major with k fastest, leading dims ldw1 / ldw
// (multiples of 2 doubles, 16-B aligned rows).  ws: >= core_ws_doubles(r2, R, ldw) doubles
// (W2ext); part: split-K scratch of part_cap doubles (may be 0).
int core_kr(const double* W1x, int64_t ldw1, const double* W2, const double* W3, int64_t ldw, int64_t r1,
            int64_t r2, int64_t r3, int64_t R, double* beta, double* ws, double* part, size_t part_cap,
            cudaStream_t st, double* flops_acc, const CoreChunks* chunks) {
  if (r1 <= 0 || r2 <= 0 || r3 <= 0) return RHOSVD_OK;
  const int64_t M = r1 * r2, total = M * r3;
  if (M > INT32_MAX || total > ((int64_t)1 << 40) || R > INT32_MAX)
    return fail(RHOSVD_EINVAL, "core: problem too large");
  if (R == 0) {
    RH_CUDA(cudaMemsetAsync(beta, 0, (size_t)total * sizeof(double), st));
    if (chunks && chunks->done) RH_CHECK(chunks->done(chunks->ctx, 0, 0, total, st));
    return RHOSVD_OK;
  }
  // 16-wide k-slabs per pipeline stage (one mbarrier round trip each); thread-safe init
  static const int ksub = [] {
    const char* e = getenv("RHOSVD_CORE_KSUB");
    return (e && atoi(e) == 1) ? 1 : 2;
  }();
  // column segments: full BN tiles, plus (no split-K, KSUB 2) an edge segment of the r3 %
  // BN leftover columns tiled at round_up(., 16) instead of BN, so the last column tile
  // does not run padded DMMAs (r3 = 652, BN = 96: 672 -> 656 columns).  RHOSVD_CORE_BN
  // forces the main BN, RHOSVD_CORE_EDGE=0 disables the edge segment.
  static const int force_bn = [] {
    const char* e = getenv("RHOSVD_CORE_BN");
    const int v = e ? atoi(e) : 0;
    return (v == 64 || v == 80 || v == 96 || v == 112 || v == 128) ? v : 0;
  }();
  static const bool edge_on = [] {
    const char* e = getenv("RHOSVD_CORE_EDGE");
    return !(e && e[0] == '0');
  }();
  static const bool wide_edge = [] {  // RHOSVD_CORE_WIDE_EDGE=0: keep the 16-wide edge
    const char* e = getenv("RHOSVD_CORE_WIDE_EDGE");
    return !(e && e[0] == '0');
  }();
  const CorePlan plan = core_plan(r1, r2, r3, R, force_bn);
  const int BN = plan.bn;
  CoreArgs a{};
  a.r1 = (int)r1; a.r2 = (int)r2; a.r3 = (int)r3; a.R = (int)R;
  a.A1 = (int)std::min<int64_t>((CORE_BM - 1) / r2 + 2, r1 + 1);
  a.A1 = std::max(1, std::min(a.A1, 256));
  a.A1pad = (int)round_up(a.A1, 8);
  a.mt = (int)cdiv(M, CORE_BM);
  const int sms = num_sms();
  int splits = plan.splits;
  while (splits > 1 && (size_t)splits * total > part_cap) --splits;
  a.kchunk = (int)round_up(cdiv(R, splits), CORE_BK * ksub);
  splits = (int)cdiv(R, a.kchunk);
  a.splits = splits;
  a.out = splits > 1 ? part : beta;
  struct Seg {
    int bn, n_off, n_end;
  };
  Seg segs[2];
  int nseg = 0;
  {
    const int64_t full = (r3 / BN) * BN, rem = r3 - full;
    if (plan.single) {
      segs[nseg++] = {BN, 0, (int)r3};
    } else if (splits == 1 && ksub == 2 && edge_on && rem > 0 && full > BN && BN == 128 && rem <= 16 && wide_edge) {
      // a thin leftover (<= 16 columns) joins the last full tile as one wide 144-column
      // edge tile (18 n-fragments, 239 registers): the 16-wide edge runs at ~60 % of the
      // main rate (2 n-fragments per A fragment), the wide one at the main rate
      segs[nseg++] = {BN, 0, (int)(full - BN)};
      segs[nseg++] = {144, (int)(full - BN), (int)r3};
    } else if (splits == 1 && ksub == 2 && edge_on && rem > 0 && full > 0 && round_up(rem, 16) < BN) {
      segs[nseg++] = {BN, 0, (int)full};
      segs[nseg++] = {(int)round_up(rem, 16), (int)full, (int)r3};
    } else {
      segs[nseg++] = {BN, 0, (int)r3};
    }
  }
  const size_t budget = 227 * 1024 - 1024 - 256;
  CoreArgs sa[2];
  size_t smem[2];
  CUtensorMap t3[2];
  for (int q = 0; q < nseg; ++q) {
    CoreArgs& x = sa[q];
    x = a;
    const int bn = segs[q].bn;
    x.n_off = segs[q].n_off;
    x.n_end = segs[q].n_end;
    x.nt = (int)cdiv(x.n_end - x.n_off, bn);
    x.tiles = x.mt * x.nt;
    x.items = x.tiles * splits;
    x.stage_bytes = (uint32_t)((a.A1pad + CORE_BM + bn) * 128 * ksub);
    x.tx_bytes = (uint32_t)((a.A1 + CORE_BM + bn) * 128 * ksub);
    x.stages = (int)std::min<size_t>(8, budget / x.stage_bytes);
    if (x.stages < 2) return fail(RHOSVD_EINVAL, "core: tile does not fit shared memory");
    smem[q] = 1024 + (size_t)x.stages * x.stage_bytes + 2 * x.stages * sizeof(uint64_t);
    RH_CHECK(make_tmap_2d(&t3[q], W3, r3, R, ldw, CORE_BK, bn, true));
  }

  // W2ext = W2 with rows [0, BM) repeated after row r2 - 1 (the wrap inside a tile)
  const int64_t ldx = round_up(std::max<int64_t>(R, 2), 16);
  {
    const int64_t n_el = (r2 + CORE_BM) * R;
    wrap_rows_kernel<<<(unsigned)cdiv(n_el, 256), 256, 0, st>>>(W2, ldw, (int)r2, CORE_BM, (int)R, ws, ldx);
    count_launch();
    RH_LAUNCH_CHECK();
  }
  CUtensorMap t1, t2;
  RH_CHECK(make_tmap_2d(&t1, W1x, r1, R, ldw1, CORE_BK, a.A1, true));
  RH_CHECK(make_tmap_2d(&t2, ws, r2 + CORE_BM, R, ldx, CORE_BK, CORE_BM, true));
  auto launch_seg = [&](int q, const CoreArgs& aa, cudaStream_t s) -> int {
    const int grid = (int)std::min<int64_t>(aa.items, sms);
    const int bn = segs[q].bn;
    const CUtensorMap& t = t3[q];
    const size_t sm = smem[q];
    if (ksub == 2) {
      switch (bn) {
        case 144: return launch_core<144, 2>(t1, t2, t, aa, sm, grid, s);
        case 128: return launch_core<128, 2>(t1, t2, t, aa, sm, grid, s);
        case 112: return launch_core<112, 2>(t1, t2, t, aa, sm, grid, s);
        case 96: return launch_core<96, 2>(t1, t2, t, aa, sm, grid, s);
        case 80: return launch_core<80, 2>(t1, t2, t, aa, sm, grid, s);
        case 64: return launch_core<64, 2>(t1, t2, t, aa, sm, grid, s);
        case 48: return launch_core<48, 2>(t1, t2, t, aa, sm, grid, s);
        case 32: return launch_core<32, 2>(t1, t2, t, aa, sm, grid, s);
        case 16: return launch_core<16, 2>(t1, t2, t, aa, sm, grid, s);
        default: return fail(RHOSVD_EINVAL, "core: unsupported tile width");
      }
    }
    if (bn == 128) return launch_core<128, 1>(t1, t2, t, aa, sm, grid, s);
    if (bn == 96) return launch_core<96, 1>(t1, t2, t, aa, sm, grid, s);
    if (bn == 64) return launch_core<64, 1>(t1, t2, t, aa, sm, grid, s);
    return fail(RHOSVD_EINVAL, "core: KSUB 1 supports BN 64 / 96 / 128 only");
  };
  // one row range [tm0, tm0 + mt) of every column segment, in order on stream s
  auto launch_rows = [&](int tm0, int mtc, cudaStream_t s) -> int {
    for (int q = 0; q < nseg; ++q) {
      CoreArgs ac = sa[q];
      ac.tm0 = tm0;
      ac.mt = mtc;
      ac.tiles = ac.mt * ac.nt;
      ac.items = ac.tiles * ac.splits;
      RH_CHECK(launch_seg(q, ac, s));
    }
    return RHOSVD_OK;
  };
  const int nch = (chunks && chunks->side && splits == 1) ? std::max(1, std::min(chunks->count, a.mt)) : 1;
  if (nch > 1) {
    // independent launches over disjoint row ranges, alternating between two streams
    cudaEvent_t e0, e1;
    RH_CUDA(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
    RH_CUDA(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
    RH_CUDA(cudaEventRecord(e0, st));
    RH_CUDA(cudaStreamWaitEvent(chunks->side, e0, 0));
    for (int c = 0; c < nch; ++c) {
      const int tm0 = (int)((int64_t)a.mt * c / nch);
      const int tm1 = (int)((int64_t)a.mt * (c + 1) / nch);
      cudaStream_t s = (c & 1) ? chunks->side : st;
      RH_CHECK(launch_rows(tm0, tm1 - tm0, s));
      const int64_t m_lo = (int64_t)tm0 * CORE_BM, m_hi = std::min<int64_t>(M, (int64_t)tm1 * CORE_BM);
      if (chunks->done) RH_CHECK(chunks->done(chunks->ctx, c, m_lo * r3, m_hi * r3, s));
    }
    RH_CUDA(cudaEventRecord(e1, chunks->side));
    RH_CUDA(cudaStreamWaitEvent(st, e1, 0));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  } else {
    RH_CHECK(launch_rows(0, a.mt, st));
    if (splits > 1) {
      core_splitk_reduce<<<(unsigned)cdiv(total, 256), 256, 0, st>>>(part, splits, total, beta);
      count_launch();
      RH_LAUNCH_CHECK();
    }
    if (chunks && chunks->done) RH_CHECK(chunks->done(chunks->ctx, 0, 0, total, st));
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

// ------------------------------------------------------------------ tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int make_tmap_2d(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld, int box_cols,
                 int box_rows, bool swizzle128) {
  static const EncodeTiledFn enc = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return (EncodeTiledFn)fn;
  }();
  if (!enc) return fail(RHOSVD_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if (((uintptr_t)base & 15) || ((ld * 8) & 15)) return fail(RHOSVD_EINVAL, "tensor map: 16-B alignment");
  cuuint64_t gdim[2] = {(cuuint64_t)std::max<int64_t>(cols, 1), (cuuint64_t)std::max<int64_t>(rows, 1)};
  cuuint64_t gstride[1] = {(cuuint64_t)(ld * 8)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(RHOSVD_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return RHOSVD_OK;
}

}  // namespace rhosvd
