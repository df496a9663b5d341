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
// O(n^2) per 1-D convolution against the paper's O(n log n) (FFT): on the tensor pipe
// the dense form is faster up to n ~ 16k at the ranks of the paper's applications
// (DESIGN.md section 11c).
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
  cudaStream_t st = (cudaStream_t)stream;
  g_launches = 0;
  outer_weights_kernel<<<(unsigned)cdiv(Ra * Rp, 256), 256, 0, st>>>(ca, (int)Ra, cp, (int)Rp, wout);
  count_launch();
  RH_LAUNCH_CHECK();
  // stacked Toeplitz chunk: qc kernel terms, qc n^2 doubles within ~1 GiB
  const int64_t qc = std::max<int64_t>(1, std::min<int64_t>(Rp, ((int64_t)1 << 27) / (n * n)));
  double* T = nullptr;
  RH_CUDA(cudaMallocAsync((void**)&T, (size_t)round_up(qc * n, 2) * n * sizeof(double), st));
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
  cudaFreeAsync(T, st);
  return status;
}
