// kernels.h - host wrappers of the device kernels (internal).
#pragma once
#include "common.cuh"

namespace rhosvd {
// Optional row-chunked core launch (overlaps the D2H of finished rows of beta with the
// rest of the contraction): the row tiles are split into `count` contiguous ranges,
// launched alternately on the call's stream and `side`; after chunk c, done(c, e0, e1, s)
// is called with the finished element range [e0, e1) of beta and the stream it was
// launched on.  Ignored (one launch, one done call) when the problem splits K.
struct CoreChunks {
  int count = 1;
  cudaStream_t side = nullptr;
  int (*done)(void* ctx, int c, int64_t e0, int64_t e1, cudaStream_t s) = nullptr;
  void* ctx = nullptr;
};
int k_normalize(const double* U, int64_t ldu, int64_t n, int64_t R, int64_t Rp, double* Uh, int64_t ldn,
                double* s, double* tcol, int* flag, cudaStream_t st);
int k_xiprime(const double* xi, const double* s1, const double* s2, const double* s3, int64_t R, int64_t Rp,
              double* xip, double* xip2, int* flag, cudaStream_t st);
int k_coldot(const double* Z, const double* Y, int64_t ld, int64_t n, int64_t b, double* d, cudaStream_t st);
int k_fixed_sum(const double* x, int64_t n, double* out, cudaStream_t st);
int k_sumsq(const double* x, int64_t n, double* part, double* out, cudaStream_t st);
int k_random(double* M, int64_t ldm, int64_t n, int64_t c0, int64_t c1, uint64_t seed, cudaStream_t st);
int k_ritz_floor(const double* th, int64_t b, double tau, double* inv, cudaStream_t st);
int k_select_rank(const double* lam, int64_t b, const double* rho, double T, double eps, int r_fixed, int guard,
                  double* tail2, double* out, double* sigma, cudaStream_t st);
int k_hadamard(const double* A, double* C, int64_t ld, int64_t M, int64_t N, cudaStream_t st);
int k_transpose(const double* A, int64_t lda, int64_t rows, int64_t cols, double* B, int64_t ldb, cudaStream_t st);
int k_sqrt_clamp(const double* lam, int64_t r, double* out, cudaStream_t st);
int k_sign_fix(double* Z, int64_t ldz, int64_t n, int64_t r, double* W, int64_t ldw, int64_t Rl, double* sgn,
               cudaStream_t st);
int core_kr(const double* W1x, int64_t ldw1, const double* W2, const double* W3, int64_t ldw, int64_t r1,
            int64_t r2, int64_t r3, int64_t R, double* beta, double* ws, double* part, size_t part_cap,
            cudaStream_t st, double* flops_acc, const CoreChunks* chunks = nullptr);
size_t core_ws_doubles(int64_t r2, int64_t R, int64_t ldw);
size_t core_part_doubles(int64_t r1, int64_t r2, int64_t r3, int64_t R);
int scale_cols(const double* W, int64_t ldw, const double* xi, int64_t r, int64_t R, double* out, int64_t ldo,
               cudaStream_t st);
}  // namespace rhosvd
