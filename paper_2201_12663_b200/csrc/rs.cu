// rs.cu - range-separated (RS) long-range front-end of the RHOSVD path.
//
// PAPER.md section 4: a radial kernel is a sinc-quadrature sum of Gaussians
// G_R = sum_k w_k prod_l e^{-tau_k x_l^2} (Eq. sinc_general); the RS
// split keeps the terms with t_k = sqrt(tau_k) <= 1 as the long-range part
// (Eq. RS_repres); the long-range part of a lattice sum of kernels,
// G_{N,l} = sum_j c_j W_j G_l, is assembled by shift-and-windowing the reference long part
// (Eq. Slater_interp_multi) and handed to rhosvd_c2t, whose Tucker
// rank grows only as log^{3/2} log(N / eps) (Prop. 4.2).
//
//  * rhosvd_sinc_slater (host): the sinc rule of the Slater Laplace transform
//    e^{-lambda sqrt(rho)} = sqrt(alpha/pi) int tau^{-3/2} e^{-alpha/tau - rho tau} dtau,
//    alpha = lambda^2/4, trapezoid in s = ln tau.
//  * rhosvd_rs_split (host): K_l = {k : t_k <= 1}, K_s = {k : t_k > 1}.
//  * rhosvd_rs_lattice (device): reference table g_k[o] = e^{-tau_k (o h)^2} on the doubled
//    grid o = -(n-1)..(n-1) (one kernel), then every lattice column (node j, long term k)
//    of every mode is the window g_k[i - m_{j,l}], i = 0..n-1, of that table (one warp per
//    column, a coalesced gather: HBM-bound, 3 n 8 bytes written per output column; the
//    table, R_l (2n - 1) doubles, stays in L2), xi = c_j w_k.
#include <cmath>
#include <cstring>

#include "common.cuh"

namespace rhosvd {

constexpr int RS_MAX_TERMS = 128;

struct RsRef {
  int Rl, n;
  double h;
  double tau[RS_MAX_TERMS];
  double w[RS_MAX_TERMS];
};

// g[k * ldg + o] = exp(-tau_k ((o - (n-1)) h)^2),  o < 2n - 1
__global__ void rs_reference_kernel(const RsRef p, double* g, int64_t ldg) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t m = 2LL * p.n - 1;
  if (e >= (int64_t)p.Rl * m) return;
  const int k = (int)(e / m);
  const int64_t o = e - (int64_t)k * m;
  const double d = (double)(o - (p.n - 1)) * p.h;
  g[k * ldg + o] = exp(-p.tau[k] * (d * d));
}

// one warp per output column (j, k), all three modes (8 columns per 256-thread CTA); the
// lanes stream the n rows: every warp store is one coalesced 256-byte segment
__global__ void __launch_bounds__(256) rs_window_kernel(const RsRef p, const double* __restrict__ g, int64_t ldg,
                                                         const int32_t* __restrict__ node_idx,
                                                         const double* __restrict__ c, int64_t N,
                                                         double* __restrict__ U1, double* __restrict__ U2,
                                                         double* __restrict__ U3, int64_t ldu,
                                                         double* __restrict__ xi) {
  const int lane = threadIdx.x & 31;
  const int64_t col = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (col >= N * p.Rl) return;
  const int64_t j = col / p.Rl;
  const int k = (int)(col - j * p.Rl);
  const double* gk = g + k * ldg + (p.n - 1);
  double* const U[3] = {U1, U2, U3};
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    const int m = node_idx[3 * j + l];
    double* dst = U[l] + col * ldu;
    if (m >= 0 && m < p.n) {
      const double* src = gk - m;
      for (int i = lane; i < p.n; i += 32) dst[i] = src[i];
    } else {  // a node off the grid: its window is read only where it overlaps the table
      for (int i = lane; i < p.n; i += 32) {
        const int64_t o = (int64_t)i - m + (p.n - 1);
        dst[i] = (o >= 0 && o < 2LL * p.n - 1) ? gk[(int64_t)i - m] : 0.0;
      }
    }
  }
  if (lane == 0) xi[col] = c[j] * p.w[k];
}

}  // namespace rhosvd

using namespace rhosvd;

extern "C" {

int rhosvd_sinc_slater(double lambda, double h, int32_t M, double w_min, double* tau, double* w, int64_t cap,
                       int64_t* R) {
  if (!tau || !w || !R || !(lambda > 0.0) || !(h > 0.0) || M < 0) return fail(RHOSVD_EINVAL, "sinc_slater: bad args");
  const double alpha = 0.25 * lambda * lambda;
  const double c0 = h * std::sqrt(alpha / M_PI);
  int64_t cnt = 0;
  for (int32_t k = -M; k <= M; ++k) {
    const double s = (double)k * h;
    const double wk = c0 * std::exp(-0.5 * s) * std::exp(-alpha * std::exp(-s));
    if (!(wk >= w_min)) continue;
    if (cnt >= cap) return fail(RHOSVD_EINVAL, "sinc_slater: output capacity too small");
    tau[cnt] = std::exp(s);
    w[cnt] = wk;
    ++cnt;
  }
  *R = cnt;
  return RHOSVD_OK;
}

int rhosvd_rs_split(const double* tau, const double* w, int64_t R, double* tau_l, double* w_l, int64_t* R_l,
                    double* tau_s, double* w_s, int64_t* R_s) {
  if (R < 0 || (R > 0 && (!tau || !w)) || !R_l || !R_s) return fail(RHOSVD_EINVAL, "rs_split: bad args");
  int64_t nl = 0, ns = 0;
  for (int64_t k = 0; k < R; ++k) {
    if (std::sqrt(tau[k]) <= 1.0) {  // t_k <= 1: long range
      if (tau_l) tau_l[nl] = tau[k];
      if (w_l) w_l[nl] = w[k];
      ++nl;
    } else {
      if (tau_s) tau_s[ns] = tau[k];
      if (w_s) w_s[ns] = w[k];
      ++ns;
    }
  }
  *R_l = nl;
  *R_s = ns;
  return RHOSVD_OK;
}

int rhosvd_rs_lattice(const double* tau_l, const double* w_l, int64_t R_l, double h, int64_t n,
                      const int32_t* node_idx, const double* c, int64_t N, double* U1, double* U2, double* U3,
                      int64_t ldu, double* xi, rhosvd_stream stream) {
  if (R_l < 0 || R_l > RS_MAX_TERMS || n < 1 || N < 0 || ldu < n || !(h > 0.0))
    return fail(RHOSVD_EINVAL, "rs_lattice: need 0 <= R_l <= 128, n >= 1, N >= 0, ldu >= n, h > 0");
  if (N * R_l == 0) return RHOSVD_OK;
  if (!tau_l || !w_l || !node_idx || !c || !U1 || !U2 || !U3 || !xi) return fail(RHOSVD_EINVAL, "rs_lattice: null");
  if (N * R_l > INT32_MAX || n > (1 << 26)) return fail(RHOSVD_EINVAL, "rs_lattice: too large");
  RH_CHECK(device_guard());
  cudaStream_t st = (cudaStream_t)stream;
  RsRef p{};
  p.Rl = (int)R_l;
  p.n = (int)n;
  p.h = h;
  std::memcpy(p.tau, tau_l, R_l * sizeof(double));
  std::memcpy(p.w, w_l, R_l * sizeof(double));
  const int64_t ldg = round_up(2 * n - 1, 32);
  double* g = nullptr;
  RH_CUDA(cudaMallocAsync((void**)&g, (size_t)R_l * ldg * sizeof(double), st));
  g_launches = 0;
  rs_reference_kernel<<<(unsigned)cdiv(R_l * (2 * n - 1), 256), 256, 0, st>>>(p, g, ldg);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) {
    rs_window_kernel<<<(unsigned)cdiv(N * R_l, 8), 256, 0, st>>>(p, g, ldg, node_idx, c, N, U1, U2, U3, ldu, xi);
    count_launch();
    e = cudaGetLastError();
  }
  cudaFreeAsync(g, st);
  if (e != cudaSuccess) return fail(RHOSVD_ECUDA, std::string("rs_lattice: ") + cudaGetErrorString(e));
  return RHOSVD_OK;
}

}  // extern "C"
