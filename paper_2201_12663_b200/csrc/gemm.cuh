// gemm.cuh - FP64 DMMA GEMM engine for sm_100a (host-side descriptor + launcher).
//
// Every dense contraction on the RHOSVD hot path is one of
//   C = alpha * op(A) op(B) * diag(col_scale) (row-scaled) + beta * C
// with op(A)(m,k) = a_k ? A[m*lda + k] : A[k*lda + m] and
//      op(B)(k,n) = b_k ? B[n*ldb + k] : B[k*ldb + n],   C(m,n) = C[n*ldc + m].
// K1 Gram, the subspace-iteration products, the one-sided
// Rayleigh-Ritz Grams, the projections W = Z^T Uhat and
// the refinement are all instances; the core (Prop. 2.1) has its own kernel.
#pragma once
#include "common.cuh"

namespace rhosvd {

enum GemmEpi { EPI_STORE = 0, EPI_RESID = 1 };

struct GemmArgs {
  int64_t M = 0, N = 0, K = 0;
  const double* A = nullptr;
  int64_t lda = 0;
  bool a_k = false;  // A stored k-contiguous (A[m*lda + k])
  const double* B = nullptr;
  int64_t ldb = 0;
  bool b_k = false;  // B stored k-contiguous (B[n*ldb + k])
  double* C = nullptr;
  int64_t ldc = 0;
  double alpha = 1.0, beta = 0.0;
  const double* col_scale = nullptr;  // per output column n
  const double* row_scale = nullptr;  // per output row m
  bool upper_sym = false;             // M == N symmetric: compute upper tiles, mirror
  int epi = EPI_STORE;
  const double* D = nullptr;          // EPI_RESID: sum_{m,n} (D(m,n) - acc)^2
  int64_t ldd = 0;
  double* resid_out = nullptr;        // EPI_RESID: one double (device), overwritten
  int splits = 0;                     // 0 = auto
  // Batched form (one persistent launch over `batch` independent GEMMs, e.g. the three
  // modes' Grams): batch b reads op(A) / op(B) at k-coordinates shifted by b * a_koff /
  // b * b_koff (the k-extents must lie back to back in one allocation; K and the k
  // offsets are multiples of 32 so no k-stage straddles two batches) and writes C +
  // b * c_bstride.  Not for EPI_RESID.
  int batch = 1;
  int64_t a_koff = 0, b_koff = 0, c_bstride = 0;
};

// Scratch for split-K partials (grown on demand, stream-ordered).
struct Scratch {
  double* ptr = nullptr;
  size_t cap = 0;  // doubles
  int ensure(size_t doubles, cudaStream_t st);
  void release(cudaStream_t st);
};

int gemm(const GemmArgs& g, Scratch& scr, cudaStream_t st, double* flops_acc = nullptr);
// K-split count the batched form picks for `nb` GEMMs of M x N x K (upper: symmetric
// upper tiles).  A single GEMM called with this `splits` and the same K sums every output
// element in the same order as its batch slot (bitwise identical results).
int gemm_batch_splits(int64_t M, int64_t N, int64_t K, bool upper, int nb);

}  // namespace rhosvd
