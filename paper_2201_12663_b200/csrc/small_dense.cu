// small_dense.cu - the b x b kernels of the RHOSVD eigensolver on sm_100a.
//
//  * syevj: parallel cyclic two-sided Jacobi (round-robin pair ordering,
//    b/2 disjoint rotations per step) as ONE cooperative persistent kernel:
//    every CTA recomputes all rotation parameters of a step from the current
//    matrix (so a step needs a single grid barrier), the 2x2 block updates of
//    A (double-buffered) and the column rotations of V are spread over the
//    whole GPU.  Stopping rule |a_pq| <= tol sqrt(|a_pp a_qq|) (Demmel-Veselic
//    relative criterion) gives eigenvalues of scaled-diagonally-dominant
//    positive definite matrices to high relative accuracy - which is what the
//    one-sided Rayleigh-Ritz on W W^T needs.
//  * chol_inv_scaled: column-scaled (optionally shifted) Cholesky of a b x b
//    Gram as a cooperative blocked right-looking kernel (32-wide panels, one
//    grid barrier per panel), then the inverse of L one warp per column; the
//    output D L^{-T} turns M into Q = M D L^{-T} (CholeskyQR).
#include <cooperative_groups.h>

#include "small_dense.cuh"

namespace rhosvd {

// ------------------------------------------------------------------ grid barrier
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  if (gridDim.x == 1) {
    __syncthreads();
    return;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = bar + 1;
    unsigned gen = *vgen;
    __threadfence();
    unsigned arrived = atomicAdd(bar, 1u);
    if (arrived == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*vgen == gen) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ int rr_index(int pos, int step, int m) {
  return pos == 0 ? 0 : 1 + (pos - 1 + step) % (m - 1);
}

// ------------------------------------------------------------------ Jacobi
struct JacParams {
  int b, m, h;
  const double* Ain;
  int64_t lda;
  double* A0;
  double* A1;
  int64_t ld;
  double* V;
  double* lam;  // unsorted eigenvalues out
  double tol, abstol;  // abstol relative to max |a_ii| of the input
  int max_sweeps;
  unsigned* bar;
  int* info;
};

__global__ void __launch_bounds__(512) jacobi_kernel(JacParams p) {
  extern __shared__ double sh[];
  const int h = p.h, b = p.b, m = p.m;
  double* c_ = sh;
  double* s_ = sh + h;
  double* t_ = sh + 2 * h;
  int* act_ = reinterpret_cast<int*>(sh + 3 * h);
  int* pp_ = act_ + h;
  int* qq_ = pp_ + h;
  __shared__ int red[32];

  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
  const int64_t ld = p.ld;

  // absolute floor relative to the largest diagonal entry (every CTA, same value)
  __shared__ double sdmax[32];
  {
    double dm = 0.0;
    for (int i = threadIdx.x; i < b; i += blockDim.x) dm = fmax(dm, fabs(p.Ain[i * p.lda + i]));
    for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    if ((threadIdx.x & 31) == 0) sdmax[threadIdx.x >> 5] = dm;
    __syncthreads();
    dm = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) dm = fmax(dm, sdmax[w]);
    __syncthreads();
    if (threadIdx.x == 0) sdmax[0] = dm;
    __syncthreads();
  }
  const double abstol = p.abstol * sdmax[0];
  // init: A0 = Ain, V = I
  for (int64_t e = gtid; e < (int64_t)b * b; e += gthreads) {
    int i = (int)(e % b), j = (int)(e / b);
    p.A0[j * ld + i] = p.Ain[j * p.lda + i];
    p.V[j * ld + i] = (i == j) ? 1.0 : 0.0;
  }
  grid_barrier(p.bar);

  double* cur = p.A0;
  double* nxt = p.A1;
  const int64_t nblk = (int64_t)h * (h + 1) / 2;
  const int64_t items = nblk + (int64_t)b * h;
  int sweeps = 0;
  bool converged = false;
  for (int sw = 0; sw < p.max_sweeps; ++sw) {
    int mycount = 0;
    for (int step = 0; step < m - 1; ++step) {
      // ---- phase 1: every CTA computes all rotations of this step
      for (int k = threadIdx.x; k < h; k += blockDim.x) {
        int i1 = rr_index(k, step, m), i2 = rr_index(m - 1 - k, step, m);
        int pq = min(i1, i2), qq = max(i1, i2);
        pp_[k] = pq;
        qq_[k] = qq;
        double c = 1.0, s = 0.0, t = 0.0;
        int act = 0;
        if (qq < b) {
          double app = cur[pq * ld + pq], aqq = cur[qq * ld + qq], apq = cur[qq * ld + pq];
          double thr = fmax(abstol, p.tol * sqrt(fabs(app * aqq)));
          if (fabs(apq) > thr) {
            act = 1;
            double theta = (aqq - app) / (2.0 * apq);
            if (fabs(theta) > 1e150)
              t = 0.5 / theta;
            else
              t = copysign(1.0 / (fabs(theta) + sqrt(1.0 + theta * theta)), theta);
            if (theta == 0.0) t = 1.0;
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
          }
        }
        c_[k] = c;
        s_[k] = s;
        t_[k] = t;
        act_[k] = act;
        mycount += act;
      }
      __syncthreads();
      // ---- phase 2: 2x2 block updates (upper blocks, mirrored) and V rotations
      for (int64_t it = gtid; it < items; it += gthreads) {
        if (it < nblk) {
          int Q = (int)((sqrt(8.0 * (double)it + 1.0) - 1.0) * 0.5);
          while ((int64_t)(Q + 1) * (Q + 2) / 2 <= it) ++Q;
          while ((int64_t)Q * (Q + 1) / 2 > it) --Q;
          int P = (int)(it - (int64_t)Q * (Q + 1) / 2);  // P <= Q
          int p1 = pp_[P], q1 = qq_[P];
          if (P == Q) {
            if (q1 >= b) {
              nxt[p1 * ld + p1] = cur[p1 * ld + p1];
            } else if (act_[P]) {
              double app = cur[p1 * ld + p1], aqq = cur[q1 * ld + q1], apq = cur[q1 * ld + p1];
              double t = t_[P];
              nxt[p1 * ld + p1] = app - t * apq;
              nxt[q1 * ld + q1] = aqq + t * apq;
              nxt[q1 * ld + p1] = 0.0;
              nxt[p1 * ld + q1] = 0.0;
            } else {
              nxt[p1 * ld + p1] = cur[p1 * ld + p1];
              nxt[q1 * ld + q1] = cur[q1 * ld + q1];
              double apq = cur[q1 * ld + p1];
              nxt[q1 * ld + p1] = apq;
              nxt[p1 * ld + q1] = apq;
            }
          } else {
            int p2 = pp_[Q], q2 = qq_[Q];
            bool vq1 = q1 < b, vq2 = q2 < b;
            double a11 = cur[p2 * ld + p1];
            double a12 = vq2 ? cur[q2 * ld + p1] : 0.0;
            double a21 = vq1 ? cur[p2 * ld + q1] : 0.0;
            double a22 = (vq1 && vq2) ? cur[q2 * ld + q1] : 0.0;
            double c1 = c_[P], s1 = s_[P], c2 = c_[Q], s2 = s_[Q];
            // columns (p2,q2) rotated by (c2,s2)
            double b11 = c2 * a11 - s2 * a12, b12 = s2 * a11 + c2 * a12;
            double b21 = c2 * a21 - s2 * a22, b22 = s2 * a21 + c2 * a22;
            // rows (p1,q1) rotated by (c1,s1)
            double n11 = c1 * b11 - s1 * b21, n21 = s1 * b11 + c1 * b21;
            double n12 = c1 * b12 - s1 * b22, n22 = s1 * b12 + c1 * b22;
            nxt[p2 * ld + p1] = n11;
            nxt[p1 * ld + p2] = n11;
            if (vq2) {
              nxt[q2 * ld + p1] = n12;
              nxt[p1 * ld + q2] = n12;
            }
            if (vq1) {
              nxt[p2 * ld + q1] = n21;
              nxt[q1 * ld + p2] = n21;
            }
            if (vq1 && vq2) {
              nxt[q2 * ld + q1] = n22;
              nxt[q1 * ld + q2] = n22;
            }
          }
        } else {
          int64_t j = it - nblk;
          int i = (int)(j % b), P = (int)(j / b);
          if (act_[P]) {
            int pc = pp_[P], qc = qq_[P];
            double vp = p.V[pc * ld + i], vq = p.V[qc * ld + i];
            double c = c_[P], s = s_[P];
            p.V[pc * ld + i] = c * vp - s * vq;
            p.V[qc * ld + i] = s * vp + c * vq;
          }
        }
      }
      grid_barrier(p.bar);
      double* tmp = cur;
      cur = nxt;
      nxt = tmp;
    }
    ++sweeps;
    // block-reduce the rotation count (identical in every CTA)
    int v = mycount;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    int tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    __syncthreads();
    if (tot == 0) {
      converged = true;
      break;
    }
  }
  for (int64_t i = gtid; i < b; i += gthreads) p.lam[i] = cur[i * ld + i];
  if (gtid == 0) {
    p.info[0] = sweeps;
    p.info[2] = converged ? 0 : 1;
  }
}

// Single-CTA variant for b <= 160: A lives in shared memory and is updated in
// place (each 2x2 block (P,Q), P <= Q, is read and written by one thread, its
// mirror (Q,P) by the same thread), so a step costs two __syncthreads.
constexpr int JAC_SMEM_MAXB = 160;
__global__ void __launch_bounds__(1024) jacobi_smem_kernel(JacParams p) {
  extern __shared__ double sh[];
  const int h = p.h, b = p.b, m = p.m;
  const int lds = b | 1;  // odd pitch
  double* A = sh;
  double* c_ = A + (size_t)b * lds;
  double* s_ = c_ + h;
  double* t_ = s_ + h;
  int* act_ = reinterpret_cast<int*>(t_ + h);
  int* pp_ = act_ + h;
  int* qq_ = pp_ + h;
  __shared__ int red[32];
  __shared__ double sdmax[32];
  const int tid = threadIdx.x, nth = blockDim.x;
  const int64_t ld = p.ld;
  for (int e = tid; e < b * b; e += nth) {
    int i = e % b, j = e / b;
    A[j * lds + i] = p.Ain[(int64_t)j * p.lda + i];
    p.V[j * ld + i] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  {
    double dm = 0.0;
    for (int i = tid; i < b; i += nth) dm = fmax(dm, fabs(A[i * lds + i]));
    for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    if ((tid & 31) == 0) sdmax[tid >> 5] = dm;
    __syncthreads();
    dm = 0.0;
    for (int w = 0; w < (nth >> 5); ++w) dm = fmax(dm, sdmax[w]);
    __syncthreads();
    if (tid == 0) sdmax[0] = dm;
    __syncthreads();
  }
  const double abstol = p.abstol * sdmax[0];
  const int nblk = h * (h + 1) / 2;
  const int items = nblk + b * h;
  int sweeps = 0;
  bool converged = false;
  for (int sw = 0; sw < p.max_sweeps; ++sw) {
    int mycount = 0;
    for (int step = 0; step < m - 1; ++step) {
      for (int k = tid; k < h; k += nth) {
        int i1 = rr_index(k, step, m), i2 = rr_index(m - 1 - k, step, m);
        int pq = min(i1, i2), qq = max(i1, i2);
        pp_[k] = pq;
        qq_[k] = qq;
        double c = 1.0, s = 0.0, t = 0.0;
        int act = 0;
        if (qq < b) {
          double app = A[pq * lds + pq], aqq = A[qq * lds + qq], apq = A[qq * lds + pq];
          double thr = fmax(abstol, p.tol * sqrt(fabs(app * aqq)));
          if (fabs(apq) > thr) {
            act = 1;
            double theta = (aqq - app) / (2.0 * apq);
            if (fabs(theta) > 1e150)
              t = 0.5 / theta;
            else
              t = copysign(1.0 / (fabs(theta) + sqrt(1.0 + theta * theta)), theta);
            if (theta == 0.0) t = 1.0;
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
          }
        }
        c_[k] = c; s_[k] = s; t_[k] = t; act_[k] = act;
        mycount += act;
      }
      __syncthreads();
      for (int it = tid; it < items; it += nth) {
        if (it < nblk) {
          int Q = (int)((sqrtf(8.0f * (float)it + 1.0f) - 1.0f) * 0.5f);
          while ((Q + 1) * (Q + 2) / 2 <= it) ++Q;
          while (Q * (Q + 1) / 2 > it) --Q;
          int P = it - Q * (Q + 1) / 2;
          int p1 = pp_[P], q1 = qq_[P];
          if (!act_[P] && !act_[Q]) continue;  // identity rotation on both sides
          if (P == Q) {
            double app = A[p1 * lds + p1], aqq = A[q1 * lds + q1], apq = A[q1 * lds + p1];
            double t = t_[P];
            A[p1 * lds + p1] = app - t * apq;
            A[q1 * lds + q1] = aqq + t * apq;
            A[q1 * lds + p1] = 0.0;
            A[p1 * lds + q1] = 0.0;
          } else {
            int p2 = pp_[Q], q2 = qq_[Q];
            bool vq1 = q1 < b, vq2 = q2 < b;
            double a11 = A[p2 * lds + p1];
            double a12 = vq2 ? A[q2 * lds + p1] : 0.0;
            double a21 = vq1 ? A[p2 * lds + q1] : 0.0;
            double a22 = (vq1 && vq2) ? A[q2 * lds + q1] : 0.0;
            double c1 = c_[P], s1 = s_[P], c2 = c_[Q], s2 = s_[Q];
            double b11 = c2 * a11 - s2 * a12, b12 = s2 * a11 + c2 * a12;
            double b21 = c2 * a21 - s2 * a22, b22 = s2 * a21 + c2 * a22;
            double n11 = c1 * b11 - s1 * b21, n21 = s1 * b11 + c1 * b21;
            double n12 = c1 * b12 - s1 * b22, n22 = s1 * b12 + c1 * b22;
            A[p2 * lds + p1] = n11; A[p1 * lds + p2] = n11;
            if (vq2) { A[q2 * lds + p1] = n12; A[p1 * lds + q2] = n12; }
            if (vq1) { A[p2 * lds + q1] = n21; A[q1 * lds + p2] = n21; }
            if (vq1 && vq2) { A[q2 * lds + q1] = n22; A[q1 * lds + q2] = n22; }
          }
        } else {
          int j = it - nblk;
          int i = j % b, P = j / b;
          if (act_[P]) {
            int pc = pp_[P], qc = qq_[P];
            double vp = p.V[pc * ld + i], vq = p.V[qc * ld + i];
            double c = c_[P], s = s_[P];
            p.V[pc * ld + i] = c * vp - s * vq;
            p.V[qc * ld + i] = s * vp + c * vq;
          }
        }
      }
      __syncthreads();
    }
    ++sweeps;
    int v = mycount;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    int tot = 0;
    for (int w = 0; w < (nth >> 5); ++w) tot += red[w];
    __syncthreads();
    if (tot == 0) {
      converged = true;
      break;
    }
  }
  for (int i = tid; i < b; i += nth) p.lam[i] = A[i * lds + i];
  if (tid == 0) {
    p.info[0] = sweeps;
    p.info[2] = converged ? 0 : 1;
  }
}

// sort eigenpairs descending (ties: lower index first); one CTA computes ranks
__global__ void rank_sort_kernel(int b, const double* lam_u, double* lam, int* perm) {
  for (int i = threadIdx.x; i < b; i += blockDim.x) {
    double li = lam_u[i];
    int r = 0;
    for (int j = 0; j < b; ++j) {
      double lj = lam_u[j];
      r += (lj > li) || (lj == li && j < i);
    }
    perm[r] = i;
    lam[r] = li;
  }
}

__global__ void permute_cols_kernel(int b, const double* V, int64_t ldv_in, const int* perm, double* Vout,
                                    int64_t ldv) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)b * b) return;
  int i = (int)(e % b), j = (int)(e / b);
  Vout[j * ldv + i] = V[(int64_t)perm[j] * ldv_in + i];
}

// ------------------------------------------------------------------ workspace
int DenseWs::ensure(int64_t b, cudaStream_t st) {
  if (b <= cap_b && bar) return RHOSVD_OK;
  release(st);
  int64_t bb = std::max<int64_t>(b, 32);
  ld = round_up(bb, 2);
  size_t mat = (size_t)ld * bb;
  RH_CUDA(cudaMallocAsync((void**)&bar, 64, st));
  RH_CUDA(cudaMemsetAsync(bar, 0, 64, st));
  RH_CUDA(cudaMallocAsync((void**)&A0, mat * sizeof(double), st));
  RH_CUDA(cudaMallocAsync((void**)&A1, mat * sizeof(double), st));
  RH_CUDA(cudaMallocAsync((void**)&V, mat * sizeof(double), st));
  RH_CUDA(cudaMallocAsync((void**)&cs, (size_t)(2 * bb + 64) * sizeof(double), st));
  RH_CUDA(cudaMallocAsync((void**)&perm, (size_t)(bb + 64) * sizeof(int), st));
  RH_CUDA(cudaMallocAsync((void**)&info, 64, st));
  RH_CUDA(cudaMemsetAsync(info, 0, 64, st));
  cap_b = bb;
  return RHOSVD_OK;
}
void DenseWs::release(cudaStream_t st) {
  if (bar) cudaFreeAsync(bar, st);
  if (A0) cudaFreeAsync(A0, st);
  if (A1) cudaFreeAsync(A1, st);
  if (V) cudaFreeAsync(V, st);
  if (cs) cudaFreeAsync(cs, st);
  if (perm) cudaFreeAsync(perm, st);
  if (info) cudaFreeAsync(info, st);
  bar = nullptr; A0 = A1 = V = cs = nullptr; perm = info = nullptr;
  cap_b = 0;
}

static int coop_grid(const void* kern, int threads, size_t smem, int64_t want_blocks) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
  if (occ < 1) occ = 1;
  int64_t maxb = (int64_t)occ * num_sms();
  int64_t g = std::min<int64_t>(maxb, std::max<int64_t>(1, want_blocks));
  return (int)g;
}

int syevj(int64_t b, const double* A, int64_t lda, double* lambda, double* Vout, int64_t ldv, double tol,
          double abstol, int max_sweeps, DenseWs& ws, cudaStream_t st, int* sweeps_host) {
  if (b <= 0) return RHOSVD_OK;
  if (b > 4096) return fail(RHOSVD_EINVAL, "syevj: b > 4096");
  RH_CHECK(ws.ensure(b, st));
  JacParams jp{};
  jp.b = (int)b;
  jp.m = (int)(b + (b & 1));
  jp.h = jp.m / 2;
  if (jp.m < 2) jp.m = 2, jp.h = 1;
  jp.Ain = A; jp.lda = lda; jp.A0 = ws.A0; jp.A1 = ws.A1; jp.ld = ws.ld; jp.V = ws.V;
  jp.lam = ws.cs;  // unsorted eigenvalues staged in cs
  jp.tol = tol; jp.abstol = abstol; jp.max_sweeps = max_sweeps; jp.bar = ws.bar; jp.info = ws.info;
  if (b <= JAC_SMEM_MAXB) {
    const int threads = 1024;
    size_t smem = (size_t)b * (b | 1) * sizeof(double) + (size_t)jp.h * (3 * sizeof(double) + 3 * sizeof(int)) + 64;
    static bool attr_s = false;
    if (!attr_s) {
      RH_CUDA(cudaFuncSetAttribute(jacobi_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
      attr_s = true;
    }
    jacobi_smem_kernel<<<1, threads, smem, st>>>(jp);
    count_launch();
    RH_LAUNCH_CHECK();
  } else {
    const int threads = 512;
    size_t smem = (size_t)jp.h * (3 * sizeof(double) + 3 * sizeof(int)) + 64;
    static bool attr = false;
    if (!attr) {
      RH_CUDA(cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
      attr = true;
    }
    int64_t items = (int64_t)jp.h * (jp.h + 1) / 2 + (int64_t)b * jp.h;
    int64_t want = cdiv(items, threads * 4);
    int grid = coop_grid((const void*)jacobi_kernel, threads, smem, want);
    void* args[] = {&jp};
    RH_CUDA(cudaLaunchCooperativeKernel((const void*)jacobi_kernel, dim3(grid), dim3(threads), args, smem, st));
    count_launch();
  }
  rank_sort_kernel<<<1, 1024, 0, st>>>((int)b, ws.cs, lambda, ws.perm);
  permute_cols_kernel<<<(unsigned)cdiv(b * b, 256), 256, 0, st>>>((int)b, ws.V, ws.ld, ws.perm, Vout, ldv);
  count_launch(2);
  RH_LAUNCH_CHECK();
  if (sweeps_host) {
    int info[4];
    RH_CUDA(cudaMemcpyAsync(info, ws.info, sizeof(info), cudaMemcpyDeviceToHost, st));
    RH_CUDA(cudaStreamSynchronize(st));
    *sweeps_host = info[0];
    if (info[2]) *sweeps_host = -info[0];  // negative: not converged
  }
  return RHOSVD_OK;
}

// ------------------------------------------------------------------ Cholesky
struct CholParams {
  int b;
  const double* S;
  int64_t lds;
  double shift;
  double delta;  // pivot floor (relative to the unit scaled diagonal)
  double* A;  // work copy, ld
  double* Lt; // L^T (upper), ld
  double* d;  // column scaling D
  int64_t ld;
  unsigned* bar;
  int* info;
};

constexpr int CW = 32;  // panel width

__global__ void __launch_bounds__(256) chol_kernel(CholParams p) {
  __shared__ double Ljj[CW][CW + 1];
  __shared__ double Xi[CW][CW + 1];
  __shared__ double Xk[CW][CW + 1];
  __shared__ unsigned depmask;
  const int b = p.b;
  const int64_t ld = p.ld;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
  // scaling D and A = D S D + shift I, Lt = 0
  for (int64_t i = gtid; i < b; i += gthreads) {
    double sii = p.S[i * p.lds + i];
    p.d[i] = sii > 0.0 ? 1.0 / sqrt(sii) : 1.0;
  }
  grid_barrier(p.bar);
  for (int64_t e = gtid; e < (int64_t)b * b; e += gthreads) {
    int i = (int)(e % b), j = (int)(e / b);
    double v = p.S[j * p.lds + i] * p.d[i] * p.d[j];
    if (i == j) v += p.shift;
    p.A[j * ld + i] = v;
    p.Lt[j * ld + i] = 0.0;
  }
  grid_barrier(p.bar);
  const int nb = (b + CW - 1) / CW;
  const int tid = threadIdx.x;
  for (int J = 0; J < nb; ++J) {
    const int j0 = J * CW, w = min(CW, b - j0);
    // every CTA: factor the diagonal block and invert it
    for (int e = tid; e < CW * CW; e += blockDim.x) {
      int r = e % CW, c = e / CW;
      Ljj[r][c] = (r < w && c < w && c <= r) ? p.A[(j0 + c) * ld + j0 + r] : 0.0;
    }
    __syncthreads();
    if (tid < 32) {
      const int lane = tid;
      unsigned dep = 0u;
      for (int c = 0; c < w; ++c) {
        double dcc = Ljj[c][c];
        // A pivot below delta means column c is numerically dependent on the
        // previous ones: give it a unit pivot and a zero sub-column, i.e. keep
        // the (tiny) residual of that column as is.  The next column-scaled
        // CholQR pass normalises it.  Stable, unlike flooring the pivot.
        const bool d = !(dcc > p.delta);
        __syncwarp();
        if (d) {
          if (lane == 0 && blockIdx.x == 0) atomicOr(p.info + 1, 1);
          dep |= 1u << c;
          if (lane == c) Ljj[c][c] = 1.0;
          if (lane > c && lane < w) Ljj[lane][c] = 0.0;
          __syncwarp();
          continue;
        }
        double piv = sqrt(dcc);
        if (lane == c) Ljj[c][c] = piv;
        if (lane > c && lane < w) Ljj[lane][c] /= piv;
        __syncwarp();
        if (lane > c && lane < w) {
          double lic = Ljj[lane][c];
          for (int k = c + 1; k <= lane; ++k) Ljj[lane][k] -= lic * Ljj[k][c];
        }
        __syncwarp();
      }
      if (lane == 0) depmask = dep;
    }
    __syncthreads();
    if (blockIdx.x == 0) {
      for (int e = tid; e < w * w; e += blockDim.x) {
        int r = e % w, c = e / w;  // L(j0+r, j0+c)
        if (c <= r) p.Lt[(int64_t)(j0 + r) * ld + j0 + c] = Ljj[r][c];
      }
    }
    // trailing blocks (I, K), J < K <= I < nb
    const int t = nb - J - 1;
    const int64_t nblocks = (int64_t)t * (t + 1) / 2;
    for (int64_t q = blockIdx.x; q < nblocks; q += gridDim.x) {
      int I = (int)((sqrt(8.0 * (double)q + 1.0) - 1.0) * 0.5);
      while ((int64_t)(I + 1) * (I + 2) / 2 <= q) ++I;
      while ((int64_t)I * (I + 1) / 2 > q) --I;
      int K = (int)(q - (int64_t)I * (I + 1) / 2);  // K <= I (relative)
      I += J + 1;
      K += J + 1;
      const int i0 = I * CW, wi = min(CW, b - i0), k0 = K * CW, wk = min(CW, b - k0);
      __syncthreads();
      // L_Ij = A_Ij Inv^T ; L_Kj = A_Kj Inv^T
      for (int e = tid; e < CW * CW; e += blockDim.x) {
        int r = e % CW, c = e / CW;
        double a = 0.0, ak = 0.0;
        if (r < wi && c < w) a = p.A[(int64_t)(j0 + c) * ld + i0 + r];
        if (r < wk && c < w) ak = p.A[(int64_t)(j0 + c) * ld + k0 + r];
        Xi[r][c] = a;
        Xk[r][c] = ak;
      }
      __syncthreads();
      // forward substitution L_Ij Ljj^T = A_Ij (and L_Kj), dependent columns zero
      if (tid < 2 * CW) {
        double(*X)[CW + 1] = tid < CW ? Xi : Xk;
        const int r = tid & (CW - 1);
        const int wr = tid < CW ? wi : wk;
        if (r < wr) {
          for (int cc = 0; cc < w; ++cc) {
            if (depmask & (1u << cc)) {
              X[r][cc] = 0.0;
              continue;
            }
            double v = X[r][cc];
            for (int k = 0; k < cc; ++k) v -= X[r][k] * Ljj[cc][k];
            X[r][cc] = v / Ljj[cc][cc];
          }
        }
      }
      __syncthreads();
      if (I == K) {  // owner writes the panel block of L (as L^T)
        for (int e = tid; e < wi * w; e += blockDim.x) {
          int r = e % wi, c = e / wi;
          p.Lt[(int64_t)(i0 + r) * ld + j0 + c] = Xi[r][c];
        }
      }
      // A_IK -= L_Ij L_Kj^T (lower part of diagonal blocks only is needed; do all)
      for (int e = tid; e < wi * wk; e += blockDim.x) {
        int r = e % wi, c = e / wi;
        double s = 0.0;
        for (int k = 0; k < w; ++k) s = fma(Xi[r][k], Xk[c][k], s);
        p.A[(int64_t)(k0 + c) * ld + i0 + r] -= s;
      }
    }
    grid_barrier(p.bar);
  }
}

// warp per column of L^{-1}; Bp(c, i) = d_c * Linv(i, c)
__global__ void trinv_kernel(int b, const double* Lt, int64_t ld, const double* d, double* Bp, int64_t ldb) {
  extern __shared__ double xs[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int c = blockIdx.x * (blockDim.x >> 5) + wib;
  if (c >= b) return;
  double* x = xs + (int64_t)wib * b;
  const double dc = d[c];
  for (int i = lane; i < c; i += 32) Bp[(int64_t)i * ldb + c] = 0.0;
  if (lane == 0) x[c] = 1.0 / Lt[(int64_t)c * ld + c];
  __syncwarp();
  for (int i = c + 1; i < b; ++i) {
    const double* Li = Lt + (int64_t)i * ld;  // row i of L
    double s = 0.0;
    for (int k = c + lane; k < i; k += 32) s = fma(Li[k], x[k], s);
    s = warp_sum(s);
    if (lane == 0) x[i] = -s / Li[i];
    __syncwarp();
  }
  for (int i = c + lane; i < b; i += 32) Bp[(int64_t)i * ldb + c] = dc * x[i];
}

int chol_inv_scaled(int64_t b, const double* S, int64_t lds, double shift_rel, double* Bp, int64_t ldb,
                    DenseWs& ws, cudaStream_t st) {
  if (b <= 0) return RHOSVD_OK;
  RH_CHECK(ws.ensure(b, st));
  CholParams cp{};
  cp.b = (int)b; cp.S = S; cp.lds = lds; cp.shift = shift_rel; cp.A = ws.A0; cp.Lt = ws.A1;
  cp.d = ws.cs; cp.ld = ws.ld; cp.bar = ws.bar; cp.info = ws.info;
  cp.delta = 1e-13;
  const int threads = 256;
  int nbk = (int)cdiv(b, CW);
  int64_t want = std::max<int64_t>(1, (int64_t)(nbk - 1) * nbk / 2);
  if (b <= 64) want = 1;
  int grid = coop_grid((const void*)chol_kernel, threads, 0, want);
  void* args[] = {&cp};
  RH_CUDA(cudaLaunchCooperativeKernel((const void*)chol_kernel, dim3(grid), dim3(threads), args, 0, st));
  const int wpb = 4;
  size_t smem = (size_t)wpb * b * sizeof(double);
  static int attr_b = 0;
  if ((int)smem > 48 * 1024 && attr_b < (int)smem) {
    RH_CUDA(cudaFuncSetAttribute(trinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_b = (int)smem;
  }
  trinv_kernel<<<(unsigned)cdiv(b, wpb), 32 * wpb, smem, st>>>((int)b, ws.A1, ws.ld, ws.cs, Bp, ldb);
  count_launch(2);
  RH_LAUNCH_CHECK();
  return RHOSVD_OK;
}

}  // namespace rhosvd
