// small_dense.cuh - b x b dense kernels of the eigensolver (K3/K4 of SURVEY.md 2.2).
#pragma once
#include "common.cuh"

namespace rhosvd {

// Workspace for the cooperative small-dense kernels.
struct DenseWs {
  unsigned* bar = nullptr;  // grid barrier state (2 words), zeroed
  double* A0 = nullptr;     // b x b double buffers (Jacobi)
  double* A1 = nullptr;
  double* V = nullptr;      // b x b unsorted eigenvectors
  double* cs = nullptr;     // per-pair rotation params (unused: computed in smem)
  int* perm = nullptr;      // sort permutation
  int* info = nullptr;      // [0] sweeps, [1] not-PD flag, [2] spare
  double* Qb = nullptr;     // block Jacobi: per-pair 64 x 64 rotations
  int* rotf = nullptr;      // block Jacobi: per-pair rotated flags
  int* cnt = nullptr;       // block Jacobi: per-sweep rotation counters
  int64_t cap_b = 0, ld = 0;
  int ensure(int64_t b, cudaStream_t st);
  void release(cudaStream_t st);
};

// Symmetric Jacobi: lambda (desc), Vout (b x b, ld ldv) eigenvectors of A (b x b, lda).
// A is not modified.  tol: relative stopping rule |a_pq| <= tol sqrt(|a_pp a_qq|);
// abstol: absolute floor (entries below it are treated as zero).
int syevj(int64_t b, const double* A, int64_t lda, double* lambda, double* Vout, int64_t ldv,
          double tol, double abstol, int max_sweeps, DenseWs& ws, cudaStream_t st, int* sweeps_host);

// CholeskyQR building block: given S (b x b symmetric, ld lds, upper part valid or full),
// writes Bp (b x b, ld ldb) = D L^{-T}, D = diag(S)^{-1/2}, L = chol(D S D + shift I).
// Then Q = M Bp has orthonormal columns spanning M's leading columns.
int chol_inv_scaled(int64_t b, const double* S, int64_t lds, double shift_rel, double* Bp, int64_t ldb,
                    DenseWs& ws, cudaStream_t st);

}  // namespace rhosvd
