// conv.cu - 3-D tensor-product convolution of canonical tensors.
//
// PAPER.md:853-871 (section 3): for a canonical density Theta' = sum_m c_m u_m^(1) (x)
// u_m^(2) (x) u_m^(3) and a canonical kernel P = sum_q w_q p_q^(1) (x) p_q^(2) (x) p_q^(3)
// on one n^3 grid,
//     Theta' * P = sum_m sum_q c_m w_q (u_m^(1) * p_q^(1)) (x) (u_m^(2) * p_q^(2))
//                                       (x) (u_m^(3) * p_q^(3)),
// "a sum of tensor products of 1D convolutions".  1-D convolution (reading C1): the
// Riemann sum on the grid, the central n samples of the full discrete convolution,
//     (u * p)_i = h sum_j u_j p_{i + s - j},   s = floor(n/2),  p_k = 0 outside [0, n).
//
// B200 design: for a fixed kernel vector p_q the map u -> u * p_q is the n x n Toeplitz
// matrix T_q[i][j] = p_q[i + s - j], so all R_a x R_p convolutions of one mode are ONE
// dense contraction
//     O = h [T_q0; T_q0+1; ...] U_a        (R_p n x n) (n x R_a),
// which runs on the FP64 DMMA GEMM engine (2 n^2 R_a R_p FLOP per mode).  The stacked
// Toeplitz block is materialised in chunks of kernel terms (HBM traffic n^2 per term,
// well under the GEMM time for R_a >= ~32), and O, column-major with ld = R_p n, IS the
// output factor matrix (n x R_a R_p, ld n): column m R_p + q = u_m * p_q (reading C2).
// That dense route is O(n^2) per 1-D convolution; for n <= 2730 (N = 2^k >= 1.5 n <=
// 4096) the FFT route below (O(n log n), the paper's complexity) is used instead.
#include <algorithm>

#include "gemm.cuh"

namespace rhosvd {

// T (rows = qc n, cols = n, col-major, ld ldt >= qc n): T[q n + i][j] = P[(q0 + q) ldp + i + s - j]
__global__ void toeplitz_stack_kernel(const double* P, int64_t ldp, int n, int q0, int qc, double* T, int64_t ldt) {
  const int64_t rows = (int64_t)qc * n;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * n) return;
  const int64_t r = e % rows;
  const int j = (int)(e / rows);
  const int q = (int)(r / n), i = (int)(r % n);
  const int k = i + n / 2 - j;
  T[(int64_t)j * ldt + r] = (k >= 0 && k < n) ? P[(int64_t)(q0 + q) * ldp + k] : 0.0;
}

// ---------------------------------------------------------------- FFT route (N <= 4096)
// The convolution theorem: with N = 2^k >= 1.5 n the circular convolution of the
// zero-padded vectors equals the linear one on the central window [s, s + n) (no wrap:
// the full convolution has length 2n - 1 and s + N > 2n - 2), so
//     (u * p)_i = h Re( IDFT_N( DFT_N(u) . DFT_N(p) ) )_{i + s}.
// One CTA per transform, the signal in shared memory (N complex doubles <= 64 KB),
// radix-2: forward transforms by decimation in frequency (spectra kept in bit-reversed
// order), the inverse by decimation in time (bit-reversed in, natural out),
// twiddles exp(-2 pi i k / N) from a table built with sincospi (accurate to an ulp).
// O(n log n) per 1-D convolution, as the paper's tensor-product convolution.
constexpr int FFT_THREADS = 256, FFT_MAXN = 4096;

__global__ void twiddle_kernel(int N, double2* tw) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N / 2) return;
  double sn, cs;
  sincospi(-2.0 * (double)k / (double)N, &sn, &cs);
  tw[k] = make_double2(cs, sn);
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// in-place forward DFT of A by decimation in time (bit-reversed input order -> natural
// output order)
__device__ void fft_radix2(double2* A, int N, const double2* __restrict__ tw) {
  for (int len = 2; len <= N; len <<= 1) {
    const int half = len >> 1, step = N / len;
    for (int b = threadIdx.x; b < N / 2; b += blockDim.x) {
      const int grp = b / half, pos = b - grp * half;
      const int i = grp * len + pos, j = i + half;
      const double2 t = cmul(__ldg(&tw[pos * step]), A[j]);
      const double2 a = A[i];
      A[i] = make_double2(a.x + t.x, a.y + t.y);
      A[j] = make_double2(a.x - t.x, a.y - t.y);
    }
    __syncthreads();
  }
}

// in-place forward DFT of A by decimation in frequency (natural input order -> bit-reversed
// output order), the mirror of fft_radix2: the spectra are kept in bit-reversed order, so
// every global access below is coalesced and no permutation is ever done
__device__ void fft_dif(double2* A, int N, const double2* __restrict__ tw) {
  for (int len = N; len >= 2; len >>= 1) {
    const int half = len >> 1, step = N / len;
    for (int b = threadIdx.x; b < N / 2; b += blockDim.x) {
      const int grp = b / half, pos = b - grp * half;
      const int i = grp * len + pos, j = i + half;
      const double2 a = A[i], c = A[j];
      A[i] = make_double2(a.x + c.x, a.y + c.y);
      A[j] = cmul(__ldg(&tw[pos * step]), make_double2(a.x - c.x, a.y - c.y));
    }
    __syncthreads();
  }
}

// spectra (bit-reversed order) of the real vectors X[v] (n values each, ld ldx),
// zero-padded to N: S[v N + j], one CTA per vector
__global__ void __launch_bounds__(FFT_THREADS) fft_forward_kernel(const double* X, int64_t ldx, int n, int N,
                                                                  int logN, const double2* tw, double2* S) {
  extern __shared__ double2 A[];
  const int v = blockIdx.x;
  const double* x = X + (int64_t)v * ldx;
  for (int j = threadIdx.x; j < N; j += blockDim.x) A[j] = make_double2(j < n ? x[j] : 0.0, 0.0);
  __syncthreads();
  fft_dif(A, N, tw);
  double2* out = S + (int64_t)v * N;
  for (int j = threadIdx.x; j < N; j += blockDim.x) out[j] = A[j];
}

// out column (m Rp + q) of the factor = h Re(IDFT(Su[m] . Sp[q]))[s .. s + n), one CTA per pair
__global__ void __launch_bounds__(FFT_THREADS) fft_pair_kernel(const double2* Su, const double2* Sp, int Rp, int n,
                                                               int N, int logN, const double2* tw, double h,
                                                               double* F) {
  extern __shared__ double2 A[];
  const int pr = blockIdx.x, m = pr / Rp, q = pr - m * Rp;
  const double2* su = Su + (int64_t)m * N;
  const double2* sp = Sp + (int64_t)q * N;
  // IDFT(Y) = conj(DFT(conj(Y))) / N; Y arrives in bit-reversed order, which is the input
  // order of the decimation-in-time transform (natural-order output)
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    const double2 y = cmul(__ldg(&su[j]), __ldg(&sp[j]));
    A[j] = make_double2(y.x, -y.y);
  }
  __syncthreads();
  fft_radix2(A, N, tw);
  const int s = n / 2;
  const double sc = h / (double)N;
  double* out = F + (int64_t)pr * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = sc * A[i + s].x;
}

// ---------------------------------------------------------------- four-step FFT (N > 4096)
// N = N1 N2 (both <= 4096), j = N2 j1 + j2, k = k1 + N1 k2:
//   X[k1 + N1 k2] = sum_j2 w_N2^(j2 k2) [ w_N^(j2 k1) sum_j1 w_N1^(j1 k1) x[N2 j1 + j2] ]
// step 1: N2 transforms of length N1 over strided columns (TB adjacent columns per CTA, so
// the loads are TB-wide contiguous), times the twiddle w_N^(j2 k1), stored row-major
// Y[k1 N2 + j2]; step 2: N1 transforms of length N2 over the rows (TB rows per CTA), written
// to X[k1 + N1 k2] (TB-wide contiguous).  Sub-transforms by decimation in time in shared
// memory, twiddles from the one N-point table (w_len^p = w_N^(p N / len)).  The inverse of a
// product of two spectra is the forward transform of its conjugate (real part / N).
__device__ __forceinline__ double2 tw_get(const double2* __restrict__ tw, int N, int64_t e) {
  // w_N^e for 0 <= e < N from the half table (w^(e + N/2) = -w^e)
  const int h = N >> 1;
  if (e < h) return __ldg(&tw[e]);
  const double2 v = __ldg(&tw[e - h]);
  return make_double2(-v.x, -v.y);
}

// cnt arrays of length L (array a at A + a * P; P = L + 1 keeps the column-wise accesses
// of the loads / stores bank-conflict free), bit-reversed in, natural out
__device__ void fft_dit_batch(double2* A, int L, int P, int cnt, const double2* __restrict__ tw, int Ntab) {
  const int hl = L >> 1;
  for (int len = 2; len <= L; len <<= 1) {
    const int half = len >> 1, step = Ntab / len;
    for (int b = threadIdx.x; b < cnt * hl; b += blockDim.x) {
      const int a = b / hl, bb = b - a * hl;
      const int grp = bb / half, pos = bb - grp * half;
      const int i = a * P + grp * len + pos, j = i + half;
      const double2 t = cmul(__ldg(&tw[pos * step]), A[j]);
      const double2 u = A[i];
      A[i] = make_double2(u.x + t.x, u.y + t.y);
      A[j] = make_double2(u.x - t.x, u.y - t.y);
    }
    __syncthreads();
  }
}

struct FS1 {  // step-1 input: a real vector (mode 0) or the conjugated product of two spectra
  int mode;
  const double* X;
  int64_t ldx;
  int n;
  const double2* Su;
  const double2* Sp;
  int Rp, pair0;
};
__global__ void __launch_bounds__(FFT_THREADS) fft4_step1_kernel(FS1 in, int N, int N1, int N2, int logN1, int TB,
                                                                  const double2* tw, double2* Y) {
  extern __shared__ double2 A[];
  const int tiles = N2 / TB;
  const int t = blockIdx.x / tiles, j20 = (blockIdx.x - t * tiles) * TB;
  const double* x = nullptr;
  const double2 *su = nullptr, *sp = nullptr;
  if (in.mode == 0) {
    x = in.X + (int64_t)t * in.ldx;
  } else {
    const int pr = in.pair0 + t, m = pr / in.Rp, q = pr - m * in.Rp;
    su = in.Su + (int64_t)m * N;
    sp = in.Sp + (int64_t)q * N;
  }
  for (int e = threadIdx.x; e < TB * N1; e += blockDim.x) {
    const int a = e % TB, j1 = e / TB;
    const int64_t j = (int64_t)N2 * j1 + j20 + a;
    double2 v;
    if (in.mode == 0) {
      v = make_double2(j < in.n ? x[j] : 0.0, 0.0);
    } else {
      const double2 y = cmul(__ldg(&su[j]), __ldg(&sp[j]));
      v = make_double2(y.x, -y.y);
    }
    A[a * (N1 + 1) + (int)(__brev((unsigned)j1) >> (32 - logN1))] = v;
  }
  __syncthreads();
  fft_dit_batch(A, N1, N1 + 1, TB, tw, N);
  double2* out = Y + (int64_t)t * N;
  for (int e = threadIdx.x; e < TB * N1; e += blockDim.x) {
    const int a = e % TB, k1 = e / TB;
    const int j2 = j20 + a;
    out[(int64_t)k1 * N2 + j2] = cmul(A[a * (N1 + 1) + k1], tw_get(tw, N, (int64_t)j2 * k1));
  }
}

struct FS2 {  // step-2 output: a spectrum (mode 0) or the central window of an inverse (mode 1)
  int mode;
  double2* S;
  double* F;
  int n;
  double scale;  // h / N (mode 1)
  int pair0;
};
__global__ void __launch_bounds__(FFT_THREADS) fft4_step2_kernel(const double2* Y, int N, int N1, int N2, int logN2,
                                                                  int TB, const double2* tw, FS2 o) {
  extern __shared__ double2 A[];
  const int tiles = N1 / TB;
  const int t = blockIdx.x / tiles, k10 = (blockIdx.x - t * tiles) * TB;
  const double2* y = Y + (int64_t)t * N;
  for (int e = threadIdx.x; e < TB * N2; e += blockDim.x) {
    const int a = e / N2, j2 = e - a * N2;  // row k10 + a, contiguous over j2
    A[a * (N2 + 1) + (int)(__brev((unsigned)j2) >> (32 - logN2))] = y[(int64_t)(k10 + a) * N2 + j2];
  }
  __syncthreads();
  fft_dit_batch(A, N2, N2 + 1, TB, tw, N);
  for (int e = threadIdx.x; e < TB * N2; e += blockDim.x) {
    const int a = e % TB, k2 = e / TB;
    const int64_t k = (int64_t)(k10 + a) + (int64_t)N1 * k2;
    const double2 v = A[a * (N2 + 1) + k2];
    if (o.mode == 0) {
      o.S[(int64_t)t * N + k] = v;
    } else {
      const int s = o.n / 2;
      if (k >= s && k < s + o.n) o.F[(int64_t)(o.pair0 + t) * o.n + (k - s)] = o.scale * v.x;
    }
  }
}

// stream-ordered device scratch released on every return path
struct AsyncBufs {
  cudaStream_t st;
  void* p[4] = {nullptr, nullptr, nullptr, nullptr};
  explicit AsyncBufs(cudaStream_t s) : st(s) {}
  template <class T>
  int get(int i, T** out, size_t bytes) {
    if (cudaMallocAsync(&p[i], bytes, st) != cudaSuccess) {
      cudaGetLastError();
      p[i] = nullptr;
      return fail(RHOSVD_ENOMEM, "conv3d: scratch allocation");
    }
    *out = (T*)p[i];
    return RHOSVD_OK;
  }
  ~AsyncBufs() {
    for (void* q : p)
      if (q) cudaFreeAsync(q, st);
  }
};

__global__ void outer_weights_kernel(const double* ca, int Ra, const double* cp, int Rp, double* w) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < (int64_t)Ra * Rp) w[e] = ca[e / Rp] * cp[e % Rp];
}

}  // namespace rhosvd

using namespace rhosvd;

extern "C" int rhosvd_conv3d(const double* const Fa[3], int64_t lda, const double* ca, int64_t Ra,
                             const double* const Fp[3], int64_t ldp, const double* cp, int64_t Rp, int64_t n,
                             double h, double* const Fout[3], double* wout, void* stream) {
  if (n < 1 || Ra < 0 || Rp < 0 || lda < n || ldp < n) return fail(RHOSVD_EINVAL, "conv3d: bad sizes");
  if (Ra == 0 || Rp == 0) return RHOSVD_OK;  // empty product: nothing to write
  if (!Fa || !Fp || !Fout || !ca || !cp || !wout) return fail(RHOSVD_EINVAL, "conv3d: null pointer");
  if (n > (1 << 24) || Ra * Rp > INT32_MAX) return fail(RHOSVD_EINVAL, "conv3d: too large");
  for (int l = 0; l < 3; ++l)
    if (!Fa[l] || !Fp[l] || !Fout[l]) return fail(RHOSVD_EINVAL, "conv3d: null factor");
  if (lda & 1) return fail(RHOSVD_EINVAL, "conv3d: lda must be even (16-B TMA rows)");
  RH_CHECK(device_guard());
  cudaStream_t st = (cudaStream_t)stream;
  g_launches = 0;
  outer_weights_kernel<<<(unsigned)cdiv(Ra * Rp, 256), 256, 0, st>>>(ca, (int)Ra, cp, (int)Rp, wout);
  count_launch();
  RH_LAUNCH_CHECK();
  int logN = 1;
  while ((1 << logN) < (3 * n + 1) / 2) ++logN;  // N = 2^logN >= 1.5 n
  const int N = 1 << logN;
  // RHOSVD_CONV_ROUTE=dense|fft forces a route (tests cover both)
  static const int route = [] {
    const char* e = getenv("RHOSVD_CONV_ROUTE");
    return !e ? 0 : (e[0] == 'd' ? 1 : (e[0] == 'f' ? 2 : 0));
  }();
  const bool use_fft = route == 2 ? N <= FFT_MAXN : (route == 0 && N <= FFT_MAXN);
  const bool use_fft4 = !use_fft && route != 1 && N > FFT_MAXN && logN <= 24;
  if (use_fft4) {
    const int logN1 = logN / 2, logN2 = logN - logN1;
    const int N1 = 1 << logN1, N2 = 1 << logN2;
    const int TB1 = std::min(N2, FFT_MAXN / N1), TB2 = std::min(N1, FFT_MAXN / N2);
    const size_t sm1 = (size_t)TB1 * (N1 + 1) * sizeof(double2), sm2 = (size_t)TB2 * (N2 + 1) * sizeof(double2);
    static const cudaError_t a3 =
        cudaFuncSetAttribute(fft4_step1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (FFT_MAXN + 64) * 16);
    static const cudaError_t a4 =
        cudaFuncSetAttribute(fft4_step2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (FFT_MAXN + 64) * 16);
    RH_CUDA(a3);
    RH_CUDA(a4);
    // pair batches: the step-1 buffer holds pb transforms of N complex (<= ~512 MiB)
    const int64_t pb = std::max<int64_t>(1, std::min<int64_t>(Ra * Rp, ((int64_t)1 << 25) / N));
    const int64_t vb = std::max<int64_t>(Ra, Rp);
    double2 *tw = nullptr, *Su = nullptr, *Sp = nullptr, *Y = nullptr;
    AsyncBufs bufs(st);
    RH_CHECK(bufs.get(0, &tw, (size_t)(N / 2 + 1) * sizeof(double2)));
    RH_CHECK(bufs.get(1, &Su, (size_t)Ra * N * sizeof(double2)));
    RH_CHECK(bufs.get(2, &Sp, (size_t)Rp * N * sizeof(double2)));
    RH_CHECK(bufs.get(3, &Y, (size_t)std::max(pb, vb) * N * sizeof(double2)));
    twiddle_kernel<<<(unsigned)cdiv(N / 2, 256), 256, 0, st>>>(N, tw);
    count_launch();
    int status = RHOSVD_OK;
    auto forward = [&](const double* X, int64_t ldx, int64_t cnt, double2* S) {
      FS1 in{0, X, ldx, (int)n, nullptr, nullptr, 0, 0};
      fft4_step1_kernel<<<(unsigned)(cnt * (N2 / TB1)), FFT_THREADS, sm1, st>>>(in, N, N1, N2, logN1, TB1, tw, Y);
      FS2 o{0, S, nullptr, (int)n, 0.0, 0};
      fft4_step2_kernel<<<(unsigned)(cnt * (N1 / TB2)), FFT_THREADS, sm2, st>>>(Y, N, N1, N2, logN2, TB2, tw, o);
      count_launch(2);
    };
    for (int l = 0; l < 3 && status == RHOSVD_OK; ++l) {
      forward(Fa[l], lda, Ra, Su);
      forward(Fp[l], ldp, Rp, Sp);
      for (int64_t p0 = 0; p0 < Ra * Rp; p0 += pb) {
        const int64_t cnt = std::min<int64_t>(pb, Ra * Rp - p0);
        FS1 in{1, nullptr, 0, (int)n, Su, Sp, (int)Rp, (int)p0};
        fft4_step1_kernel<<<(unsigned)(cnt * (N2 / TB1)), FFT_THREADS, sm1, st>>>(in, N, N1, N2, logN1, TB1, tw, Y);
        FS2 o{1, nullptr, Fout[l], (int)n, h / (double)N, (int)p0};
        fft4_step2_kernel<<<(unsigned)(cnt * (N1 / TB2)), FFT_THREADS, sm2, st>>>(Y, N, N1, N2, logN2, TB2, tw, o);
        count_launch(2);
      }
      if (cudaGetLastError() != cudaSuccess) status = fail(RHOSVD_ECUDA, "conv3d: four-step fft kernels");
    }
    return status;
  }
  if (use_fft) {
    if ((int64_t)(Ra + Rp) > INT32_MAX / 2) return fail(RHOSVD_EINVAL, "conv3d: too many terms");
    double2 *tw = nullptr, *Su = nullptr, *Sp = nullptr;
    AsyncBufs bufs(st);
    RH_CHECK(bufs.get(0, &tw, (size_t)(N / 2 + 1) * sizeof(double2)));
    RH_CHECK(bufs.get(1, &Su, (size_t)Ra * N * sizeof(double2)));
    RH_CHECK(bufs.get(2, &Sp, (size_t)Rp * N * sizeof(double2)));
    twiddle_kernel<<<(unsigned)cdiv(N / 2, 256), 256, 0, st>>>(N, tw);
    count_launch();
    const size_t smem = (size_t)N * sizeof(double2);
    static const cudaError_t a1 =
        cudaFuncSetAttribute(fft_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FFT_MAXN * 16);
    static const cudaError_t a2 =
        cudaFuncSetAttribute(fft_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FFT_MAXN * 16);
    RH_CUDA(a1);
    RH_CUDA(a2);
    int status = RHOSVD_OK;
    for (int l = 0; l < 3 && status == RHOSVD_OK; ++l) {
      fft_forward_kernel<<<(unsigned)Ra, FFT_THREADS, smem, st>>>(Fa[l], lda, (int)n, N, logN, tw, Su);
      fft_forward_kernel<<<(unsigned)Rp, FFT_THREADS, smem, st>>>(Fp[l], ldp, (int)n, N, logN, tw, Sp);
      fft_pair_kernel<<<(unsigned)(Ra * Rp), FFT_THREADS, smem, st>>>(Su, Sp, (int)Rp, (int)n, N, logN, tw, h,
                                                                       Fout[l]);
      count_launch(3);
      if (cudaGetLastError() != cudaSuccess) status = fail(RHOSVD_ECUDA, "conv3d: fft kernels");
    }
    return status;
  }
  // stacked Toeplitz chunk: qc kernel terms, qc n^2 doubles within ~1 GiB
  const int64_t qc = std::max<int64_t>(1, std::min<int64_t>(Rp, ((int64_t)1 << 27) / (n * n)));
  double* T = nullptr;
  AsyncBufs tbuf(st);
  RH_CHECK(tbuf.get(0, &T, (size_t)round_up(qc * n, 2) * n * sizeof(double)));
  Scratch scr;
  int status = RHOSVD_OK;
  for (int l = 0; l < 3 && status == RHOSVD_OK; ++l) {
    for (int64_t q0 = 0; q0 < Rp && status == RHOSVD_OK; q0 += qc) {
      const int64_t qn = std::min<int64_t>(qc, Rp - q0);
      const int64_t tot = qn * n * n;
      const int64_t ldt = round_up(qn * n, 2);  // even: 16-B aligned TMA rows
      toeplitz_stack_kernel<<<(unsigned)cdiv(tot, 256), 256, 0, st>>>(Fp[l], ldp, (int)n, (int)q0, (int)qn, T, ldt);
      count_launch();
      if (cudaGetLastError() != cudaSuccess) {
        status = fail(RHOSVD_ECUDA, "conv3d: toeplitz kernel");
        break;
      }
      // O[q n + i, m] (rows of terms q0..q0+qn) = h sum_j T[q n + i, j] U_a[j, m]
      GemmArgs g;
      g.M = qn * n; g.N = Ra; g.K = n;
      g.A = T; g.lda = ldt; g.a_k = false;            // T col-major: A[k * lda + m]
      g.B = Fa[l]; g.ldb = lda; g.b_k = true;         // U_a col-major: B[n * ldb + k]
      g.C = Fout[l] + q0 * n; g.ldc = Rp * n;         // column m of O = column block m of F
      g.alpha = h;
      status = gemm(g, scr, st, nullptr);
    }
  }
  scr.release(st);
  return status;
}
