// Micro-benchmark of the block-Jacobi phase-1 kernel body: one cyclic sweep over a
// 32 x 32 symmetric pair block.  A: the production layout (256 threads, shared memory,
// round-robin ordering, 2 __syncthreads per step).  B: one warp, the block in registers
// (lane l holds column l with row l^i in register i), xor ordering (step m pairs l with
// l^m), every register index static.  Prints cycles per step and off(S)/||S|| after
// each variant's sweeps.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o build/jac_inner_bench tools/jac_inner_bench.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int P = 32, LD = 33;

__device__ __forceinline__ int rr_index(int pos, int step, int m) {
  return pos == 0 ? 0 : 1 + (pos - 1 + step) % (m - 1);
}

__device__ __forceinline__ double rcp_nr(double x);
__device__ __forceinline__ double rsqrt_nr(double x);
template <int FAST>
__global__ void __launch_bounds__(256) kA(const double* Sin, double* Sout, long long* cyc, int sweeps, double tol) {
  __shared__ double S[P * LD], Q[P * LD];
  __shared__ double c_[16], s_[16], dA_[16], dB_[16];
  __shared__ int pp_[16], qq_[16], act_[16];
  __shared__ int srot;
  const int tid = threadIdx.x;
  for (int e = tid; e < P * P; e += 256) {
    int r = e & 31, c = e >> 5;
    S[r * LD + c] = Sin[e];
    Q[r * LD + c] = r == c;
  }
  __syncthreads();
  long long t0 = clock64();
  long long tp[4] = {0, 0, 0, 0}, tq = clock64();
  for (int sw = 0; sw < sweeps; ++sw)
    for (int st = 0; st < P - 1; ++st) {
      if (tid < 32) {
        int act = 0;
        if (tid < 16) {
          int a1 = rr_index(tid, st, P), a2 = rr_index(P - 1 - tid, st, P);
          int pq = min(a1, a2), qq = max(a1, a2);
          double app = S[pq * LD + pq], aqq = S[qq * LD + qq], apq = S[pq * LD + qq];
          const double zeta = aqq - app, two = 2.0 * apq;
          double t, c;
          if (FAST) {
            const double h2 = fma(zeta, zeta, two * two);
            t = (zeta >= 0.0 ? two : -two) * rcp_nr(fabs(zeta) + h2 * rsqrt_nr(h2));
            act = apq * apq > fmax(1e-300, tol * tol * fabs(app * aqq));
            if (!(fabs(t) <= 1.0)) t = copysign(1.0, two);
            c = rsqrt_nr(fma(t, t, 1.0));
          } else {
            t = (zeta >= 0.0 ? two : -two) / (fabs(zeta) + sqrt(fma(zeta, zeta, two * two)));
            const double thr = fmax(1e-300, tol * sqrt(fabs(app * aqq)));
            act = fabs(apq) > thr;
            if (!isfinite(t)) t = copysign(1.0, two);
            c = rsqrt(fma(t, t, 1.0));
          }
          double s = t * c;
          if (!act) { c = 1.0; s = 0.0; }
          c_[tid] = c; s_[tid] = s;
          dA_[tid] = act ? app - t * apq : app;
          dB_[tid] = act ? aqq + t * apq : aqq;
          pp_[tid] = pq; qq_[tid] = qq; act_[tid] = act;
        }
        unsigned bal = __ballot_sync(0xffffffffu, act);
        if (tid == 0) srot = __popc(bal);
      }
      { long long t = clock64(); tp[0] += t - tq; tq = t; }
      __syncthreads();
      { long long t = clock64(); tp[1] += t - tq; tq = t; }
      if (srot) {
        const int k = tid >> 4, l = tid & 15;
        const int pk = pp_[k], qk = qq_[k], pl = pp_[l], ql = qq_[l];
        const bool ak = act_[k], al = act_[l];
        if (ak || al) {
          double x00 = S[pk * LD + pl], x01 = S[pk * LD + ql];
          double x10 = S[qk * LD + pl], x11 = S[qk * LD + ql];
          if (k == l) {
            x00 = dA_[k]; x01 = 0.0; x10 = 0.0; x11 = dB_[k];
          } else {
            if (ak) {
              const double c = c_[k], s = s_[k];
              const double y00 = c * x00 - s * x10, y01 = c * x01 - s * x11;
              const double y10 = s * x00 + c * x10, y11 = s * x01 + c * x11;
              x00 = y00; x01 = y01; x10 = y10; x11 = y11;
            }
            if (al) {
              const double c = c_[l], s = s_[l];
              const double y00 = c * x00 - s * x01, y01 = s * x00 + c * x01;
              const double y10 = c * x10 - s * x11, y11 = s * x10 + c * x11;
              x00 = y00; x01 = y01; x10 = y10; x11 = y11;
            }
          }
          S[pk * LD + pl] = x00; S[pk * LD + ql] = x01;
          S[qk * LD + pl] = x10; S[qk * LD + ql] = x11;
        }
        if (ak) {
          const double c = c_[k], s = s_[k];
          for (int h2 = 0; h2 < 2; ++h2) {
            const int j = l + 16 * h2;
            double vp = Q[j * LD + pk], vq = Q[j * LD + qk];
            Q[j * LD + pk] = c * vp - s * vq;
            Q[j * LD + qk] = s * vp + c * vq;
          }
        }
      }
      { long long t = clock64(); tp[2] += t - tq; tq = t; }
      __syncthreads();
      { long long t = clock64(); tp[3] += t - tq; tq = t; }
    }
  long long t1 = clock64();
  if (tid == 0) cyc[FAST ? 2 : 0] = t1 - t0;
  if (tid == 0 && FAST) printf("A-fast thread0 per step: params %.0f sync1 %.0f update %.0f sync2 %.0f\n",
                               tp[0] / (31.0 * sweeps), tp[1] / (31.0 * sweeps), tp[2] / (31.0 * sweeps), tp[3] / (31.0 * sweeps));
  if (tid == 255 && FAST) printf("A-fast thread255 per step: params %.0f sync1 %.0f update %.0f sync2 %.0f\n",
                               tp[0] / (31.0 * sweeps), tp[1] / (31.0 * sweeps), tp[2] / (31.0 * sweeps), tp[3] / (31.0 * sweeps));
  for (int e = tid; e < P * P; e += 256) Sout[e] = S[(e & 31) * LD + (e >> 5)];
}

// fast reciprocal / rsqrt: MUFU seed + Newton (full double precision up to an ulp or two)
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  // two Newton steps: r <- r (3 - x r^2) / 2
  double h = 0.5 * x;
  r = r * fma(-h * r, r, 1.5);
  r = r * fma(-h * r, r, 1.5);
  return r;
}

template <int M>
__device__ __forceinline__ void xor_step(double (&a)[P], double (&q)[P], int lane, double tol2, double abs2, int& rot) {
  constexpr int HB = (M >= 16) ? 16 : (M >= 8) ? 8 : (M >= 4) ? 4 : (M >= 2) ? 2 : 1;  // highest bit of M
  const int partner = lane ^ M;
  const bool lo = (lane & HB) == 0;  // lane < partner
  const double dmine = a[0], doth = __shfl_xor_sync(0xffffffffu, dmine, M);
  const double apq = a[M];
  const double app = lo ? dmine : doth, aqq = lo ? doth : dmine;
  const double zeta = aqq - app, two = 2.0 * apq;
  const double h2 = fma(zeta, zeta, two * two);
  const double h = h2 * rsqrt_nr(h2);
  double t = (zeta >= 0.0 ? two : -two) * rcp_nr(fabs(zeta) + h);
  const bool act = apq * apq > fmax(abs2, tol2 * fabs(app * aqq));
  if (!(fabs(t) <= 1.0)) t = copysign(1.0, two);  // NaN / overflow guard (|t| <= 1 always)
  double c = rsqrt_nr(fma(t, t, 1.0));
  double s = t * c;
  if (!act) { c = 1.0; s = 0.0; }
  rot += act;
  // rows (J^T S): register pair (i, i^M) holds rows (lane^i, lane^i^M)
#pragma unroll
  for (int i = 0; i < P; ++i) {
    constexpr int dummy = 0;
    (void)dummy;
    const int j = i ^ M;
    if (i < j) {
      const double cr = __shfl_xor_sync(0xffffffffu, c, i), sr = __shfl_xor_sync(0xffffffffu, s, i);
      const bool ip = ((lane ^ i) & HB) == 0;  // register i holds the pair's lower row
      const double xp = ip ? a[i] : a[j], xq = ip ? a[j] : a[i];
      const double np = cr * xp - sr * xq, nq = sr * xp + cr * xq;
      a[i] = ip ? np : nq;
      a[j] = ip ? nq : np;
    }
  }
  // columns (S J): own pair; partner value at row lane^i is the partner's register i^M
  double y[P];
#pragma unroll
  for (int i = 0; i < P; ++i) y[i] = __shfl_xor_sync(0xffffffffu, a[i ^ M], M);
#pragma unroll
  for (int i = 0; i < P; ++i) a[i] = lo ? c * a[i] - s * y[i] : s * y[i] + c * a[i];
  if (act) {
    const double dA = app - t * apq, dB = aqq + t * apq;
    a[0] = lo ? dA : dB;
    a[M] = 0.0;
  }
#pragma unroll
  for (int i = 0; i < P; ++i) y[i] = __shfl_xor_sync(0xffffffffu, q[i ^ M], M);
#pragma unroll
  for (int i = 0; i < P; ++i) q[i] = lo ? c * q[i] - s * y[i] : s * y[i] + c * q[i];
}

template <int M>
__device__ __forceinline__ void xor_sweep(double (&a)[P], double (&q)[P], int lane, double tol2, double abs2, int& rot) {
  if constexpr (M < P) {
    xor_step<M>(a, q, lane, tol2, abs2, rot);
    xor_sweep<M + 1>(a, q, lane, tol2, abs2, rot);
  }
}

__global__ void __launch_bounds__(32) kB(const double* Sin, double* Sout, long long* cyc, int sweeps, double tol) {
  const int lane = threadIdx.x;
  double a[P], q[P];
#pragma unroll
  for (int i = 0; i < P; ++i) {
    a[i] = Sin[(lane ^ i) * P + lane];
    q[i] = (i == 0) ? 1.0 : 0.0;
  }
  int rot = 0;
  long long t0 = clock64();
  for (int sw = 0; sw < sweeps; ++sw) xor_sweep<1>(a, q, lane, tol * tol, 1e-300, rot);
  long long t1 = clock64();
  if (lane == 0) cyc[1] = t1 - t0;
#pragma unroll
  for (int i = 0; i < P; ++i) Sout[(lane ^ i) * P + lane] = a[i];
  if (rot == -1) Sout[0] = q[0];
}


// C: xor ordering (step m pairs r with r^m), S swizzled so every half-warp access is
// bank-conflict free, ONE __syncthreads per step: the thread that updates the entry
// (p', q') of the NEXT step's pair computes that pair's rotation right after its update
// (diagonals from the exact dA/dB of this step).
__device__ __forceinline__ int swz(int c) { return c ^ ((c >> 4) * 15); }
__device__ __forceinline__ int hbit(int m) { return 1 << (31 - __clz(m)); }
// k-th element (0..15) with bit hb clear
__device__ __forceinline__ int lower_of(int k, int hb) { return ((k & ~(hb - 1)) << 1) | (k & (hb - 1)); }
// pair index of row r at a step with highest bit hb
__device__ __forceinline__ int pair_of(int r, int hb) { return ((r >> 1) & ~(hb - 1)) | (r & (hb - 1)); }

__device__ __forceinline__ void rot_params(double app, double aqq, double apq, double tol2, double abs2,
                                           double& c, double& s, double& dA, double& dB, int& act) {
  const double zeta = aqq - app, two = 2.0 * apq;
  const double h2 = fma(zeta, zeta, two * two);
  double t = (zeta >= 0.0 ? two : -two) * rcp_nr(fabs(zeta) + h2 * rsqrt_nr(h2));
  act = apq * apq > fmax(abs2, tol2 * fabs(app * aqq));
  if (!(fabs(t) <= 1.0)) t = copysign(1.0, two);
  c = rsqrt_nr(fma(t, t, 1.0));
  s = t * c;
  dA = app - t * apq;
  dB = aqq + t * apq;
  if (!act) { c = 1.0; s = 0.0; dA = app; dB = aqq; }
}

template <int NOQ, int NOPAR, int NOS>
__global__ void __launch_bounds__(256) kC(const double* Sin, double* Sout, long long* cyc, int sweeps, double tol) {
  __shared__ double S[P * P], Q[P * LD];
  __shared__ double c_[2][16], s_[2][16], dA_[2][16], dB_[2][16];
  __shared__ int act_[2][16];
  const int tid = threadIdx.x;
  const double tol2 = tol * tol, abs2 = 1e-300;
  for (int e = tid; e < P * P; e += 256) {
    int r = e & 31, c = e >> 5;
    S[r * P + swz(c)] = Sin[e];
    Q[r * LD + c] = r == c;
  }
  __syncthreads();
  if (tid < 16) {  // parameters of step 1 (pairs (2k, 2k+1))
    const int p = 2 * tid, q = p + 1;
    double c, s, dA, dB;
    int act;
    rot_params(S[p * P + swz(p)], S[q * P + swz(q)], S[p * P + swz(q)], tol2, abs2, c, s, dA, dB, act);
    c_[0][tid] = c; s_[0][tid] = s; dA_[0][tid] = dA; dB_[0][tid] = dB; act_[0][tid] = act;
  }
  __syncthreads();
  long long t0 = clock64();
  const int k = tid >> 4, l = tid & 15;
  int buf = 0;
  long long tt[4] = {0, 0, 0, 0}, tq = clock64();
  for (int sw = 0; sw < sweeps; ++sw)
    for (int m = 1; m < P; ++m) {
      const int hb = hbit(m);
      const int pk = lower_of(k, hb), qk = pk ^ m, pl = lower_of(l, hb), ql = pl ^ m;
      const bool ak = act_[buf][k], al = act_[buf][l];
      double x00 = S[pk * P + swz(pl)], x01 = S[pk * P + swz(ql)];
      double x10 = S[qk * P + swz(pl)], x11 = S[qk * P + swz(ql)];
      if (k == l) {
        x00 = dA_[buf][k]; x01 = 0.0; x10 = 0.0; x11 = dB_[buf][k];
      } else {
        if (ak) {
          const double c = c_[buf][k], s = s_[buf][k];
          const double y00 = c * x00 - s * x10, y01 = c * x01 - s * x11;
          const double y10 = s * x00 + c * x10, y11 = s * x01 + c * x11;
          x00 = y00; x01 = y01; x10 = y10; x11 = y11;
        }
        if (al) {
          const double c = c_[buf][l], s = s_[buf][l];
          const double y00 = c * x00 - s * x01, y01 = s * x00 + c * x01;
          const double y10 = c * x10 - s * x11, y11 = s * x10 + c * x11;
          x00 = y00; x01 = y01; x10 = y10; x11 = y11;
        }
      }
      if ((ak || al || k == l) && !NOS) {
        S[pk * P + swz(pl)] = x00; S[pk * P + swz(ql)] = x01;
        S[qk * P + swz(pl)] = x10; S[qk * P + swz(ql)] = x11;
      }
      { long long t = clock64(); tt[0] += t - tq; tq = t; }
      if (ak && !NOQ) {
        const double c = c_[buf][k], s = s_[buf][k];
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int j = l + 16 * h2;
          const double vp = Q[j * LD + pk], vq = Q[j * LD + qk];
          Q[j * LD + pk] = c * vp - s * vq;
          Q[j * LD + qk] = s * vp + c * vq;
        }
      }
      // the next step's pair (p', q' = p' ^ m'), p' < q', whose entry (p', q') this thread
      // just produced computes that pair's rotation (its diagonals: this step's dA / dB)
      const int mn = (m == P - 1) ? 1 : m + 1, hn = hbit(mn);
      { long long t = clock64(); tt[1] += t - tq; tq = t; }
      if (!NOPAR) {
        // at most two of the four entries are next-step pair entries (r ^ c == m', r < c):
        // (pk, pl) / (qk, ql) share r ^ c, as do (pk, ql) / (qk, pl).  Both candidate
        // chains run unconditionally (straight-line code, no divergence); the owner stores.
        const bool d0 = ((pk ^ pl) == mn), d1 = ((pk ^ ql) == mn);
        // candidate A: (pk, pl) if d0 else (pk, ql); candidate B: (qk, ql) if d0 else (qk, pl)
        const int rA = pk, cA = d0 ? pl : ql, rB = qk, cB = d0 ? ql : pl;
        const double vA = d0 ? x00 : x01, vB = d0 ? x11 : x10;
        const bool okA = (k != l) && (d0 || d1) && rA < cA, okB = (k != l) && (d0 || d1) && rB < cB;
        const int krA = pair_of(rA, hb), kcA = pair_of(cA, hb), krB = pair_of(rB, hb), kcB = pair_of(cB, hb);
        const double appA = (rA & hb) ? dB_[buf][krA] : dA_[buf][krA];
        const double aqqA = (cA & hb) ? dB_[buf][kcA] : dA_[buf][kcA];
        const double appB = (rB & hb) ? dB_[buf][krB] : dA_[buf][krB];
        const double aqqB = (cB & hb) ? dB_[buf][kcB] : dA_[buf][kcB];
        double cA_, sA_, dAA, dBA, cB_, sB_, dAB, dBB;
        int actA, actB;
        if (okA || okB) {  // owners only (the two chains interleave)
        rot_params(appA, aqqA, vA, tol2, abs2, cA_, sA_, dAA, dBA, actA);
        rot_params(appB, aqqB, vB, tol2, abs2, cB_, sB_, dAB, dBB, actB);
        if (okA) {
          const int jn = pair_of(rA, hn);
          c_[buf ^ 1][jn] = cA_; s_[buf ^ 1][jn] = sA_; dA_[buf ^ 1][jn] = dAA; dB_[buf ^ 1][jn] = dBA;
          act_[buf ^ 1][jn] = actA;
        }
        if (okB) {
          const int jn = pair_of(rB, hn);
          c_[buf ^ 1][jn] = cB_; s_[buf ^ 1][jn] = sB_; dA_[buf ^ 1][jn] = dAB; dB_[buf ^ 1][jn] = dBB;
          act_[buf ^ 1][jn] = actB;
        }
        }
      }
      { long long t = clock64(); tt[2] += t - tq; tq = t; }
      __syncthreads();
      { long long t = clock64(); tt[3] += t - tq; tq = t; }
      buf ^= 1;
    }
  long long t1 = clock64();
  if (tid == 0) cyc[3] = t1 - t0;
  if (!NOQ && !NOPAR && sweeps == 4 && (tid == 0 || tid == 17 || tid == 100 || tid == 255))
    printf("kC tid %3d per step: S-update %.0f  Q %.0f  params %.0f  sync %.0f\n", tid, tt[0] / 124.0, tt[1] / 124.0,
           tt[2] / 124.0, tt[3] / 124.0);
  for (int e = tid; e < P * P; e += 256) Sout[e] = S[(e & 31) * P + swz(e >> 5)];
}


// D: as C, but the NEXT step's rotations are computed by a dedicated 9th warp from the
// step-start data (it re-forms the one rotated entry (p', q') it needs from the old 2x2
// block and this step's two rotations), in parallel with the 8 update warps.
// shorter chain: with rho = 1/sqrt(zeta^2 + 4 a^2), cos 2th = |zeta| rho, u = 1 + cos 2th,
// w = 1/sqrt(2u):  c = u w, s = sgn(zeta) 2 a rho w, t = s / c = 4 a sgn rho w^2
// (two rsqrt instead of rsqrt + reciprocal + rsqrt; no cancellation: u >= 1)
__device__ __forceinline__ void rot_params2(double app, double aqq, double apq, double tol2, double abs2,
                                            double& c, double& s, double& dA, double& dB, int& act) {
  const double zeta = aqq - app, two = 2.0 * apq;
  const double h2 = fma(zeta, zeta, two * two);
  const double rho = rsqrt_nr(h2);
  const double u = fma(fabs(zeta), rho, 1.0);
  const double w = rsqrt_nr(2.0 * u);
  const double sg = (zeta >= 0.0 ? two : -two) * rho;  // sin 2 theta
  act = apq * apq > fmax(abs2, tol2 * fabs(app * aqq));
  c = u * w;
  s = sg * w;
  const double t = 2.0 * sg * (w * w);
  dA = app - t * apq;
  dB = aqq + t * apq;
  if (!act) { c = 1.0; s = 0.0; dA = app; dB = aqq; }
}

template <int V2>
__global__ void __launch_bounds__(288) kD(const double* Sin, double* Sout, long long* cyc, int sweeps, double tol) {
  __shared__ double S[P * P], Q[P * LD];
  __shared__ double c_[2][16], s_[2][16], dA_[2][16], dB_[2][16];
  __shared__ int act_[2][16];
  const int tid = threadIdx.x;
  const double tol2 = tol * tol, abs2 = 1e-300;
  for (int e = tid; e < P * P; e += blockDim.x) {
    int r = e & 31, c = e >> 5;
    S[r * P + swz(c)] = Sin[e];
    Q[r * LD + c] = r == c;
  }
  __syncthreads();
  if (tid < 16) {  // parameters of step 1 (pairs (2k, 2k+1))
    const int p = 2 * tid, q = p + 1;
    double c, s, dA, dB;
    int act;
    rot_params(S[p * P + swz(p)], S[q * P + swz(q)], S[p * P + swz(q)], tol2, abs2, c, s, dA, dB, act);
    c_[0][tid] = c; s_[0][tid] = s; dA_[0][tid] = dA; dB_[0][tid] = dB; act_[0][tid] = act;
  }
  __syncthreads();
  long long t0 = clock64();
  const bool upd = tid < 256;
  const int k = (tid >> 4) & 15, l = tid & 15;
  int buf = 0;
  for (int sw = 0; sw < sweeps; ++sw)
    for (int m = 1; m < P; ++m) {
      const int hb = hbit(m);
      if (upd) {
        const int pk = lower_of(k, hb), qk = pk ^ m, pl = lower_of(l, hb), ql = pl ^ m;
        const bool ak = act_[buf][k], al = act_[buf][l];
        if (ak || al) {
          double x00 = S[pk * P + swz(pl)], x01 = S[pk * P + swz(ql)];
          double x10 = S[qk * P + swz(pl)], x11 = S[qk * P + swz(ql)];
          if (k == l) {
            x00 = dA_[buf][k]; x01 = 0.0; x10 = 0.0; x11 = dB_[buf][k];
          } else {
            const double ck = c_[buf][k], sk = s_[buf][k], cl = c_[buf][l], sl = s_[buf][l];
            const double y00 = ck * x00 - sk * x10, y01 = ck * x01 - sk * x11;
            const double y10 = sk * x00 + ck * x10, y11 = sk * x01 + ck * x11;
            x00 = cl * y00 - sl * y01; x01 = sl * y00 + cl * y01;
            x10 = cl * y10 - sl * y11; x11 = sl * y10 + cl * y11;
          }
          S[pk * P + swz(pl)] = x00; S[pk * P + swz(ql)] = x01;
          S[qk * P + swz(pl)] = x10; S[qk * P + swz(ql)] = x11;
        }
        if (ak) {
          const double c = c_[buf][k], s = s_[buf][k];
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int j = l + 16 * h2;
            const double vp = Q[j * LD + pk], vq = Q[j * LD + qk];
            Q[j * LD + pk] = c * vp - s * vq;
            Q[j * LD + qk] = s * vp + c * vq;
          }
        }
      } else if (tid < 256 + 16) {
        // next step's pair j: (p', q' = p' ^ m'), p' < q'
        const int j = tid - 256;
        const int mn = (m == P - 1) ? 1 : m + 1, hn = hbit(mn);
        const int pn = lower_of(j, hn), qn = pn ^ mn;
        const int kp = pair_of((pn & hb) ? pn ^ m : pn, hb), kq = pair_of((qn & hb) ? qn ^ m : qn, hb);
        const int r0 = lower_of(kp, hb), r1 = r0 ^ m, c0 = lower_of(kq, hb), c1 = c0 ^ m;
        const double x00 = S[r0 * P + swz(c0)], x01 = S[r0 * P + swz(c1)];
        const double x10 = S[r1 * P + swz(c0)], x11 = S[r1 * P + swz(c1)];
        const double ck = c_[buf][kp], sk = s_[buf][kp], cl = c_[buf][kq], sl = s_[buf][kq];
        // entry (pn, qn) after J_kp^T (.) J_kq (kp != kq: pn, qn lie in different pairs)
        const bool rlo = (pn & hb) == 0, clo = (qn & hb) == 0;
        const double ya = rlo ? ck * x00 - sk * x10 : sk * x00 + ck * x10;  // row pn, col c0
        const double yb = rlo ? ck * x01 - sk * x11 : sk * x01 + ck * x11;  // row pn, col c1
        const double apq = clo ? cl * ya - sl * yb : sl * ya + cl * yb;
        const double app = rlo ? dA_[buf][kp] : dB_[buf][kp];
        const double aqq = clo ? dA_[buf][kq] : dB_[buf][kq];
        double c, s, dA, dB;
        int act;
        if (V2) rot_params2(app, aqq, apq, tol2, abs2, c, s, dA, dB, act);
        else rot_params(app, aqq, apq, tol2, abs2, c, s, dA, dB, act);
        c_[buf ^ 1][j] = c; s_[buf ^ 1][j] = s; dA_[buf ^ 1][j] = dA; dB_[buf ^ 1][j] = dB;
        act_[buf ^ 1][j] = act;
      }
      __syncthreads();
      buf ^= 1;
    }
  long long t1 = clock64();
  if (tid == 0) cyc[3] = t1 - t0;
  for (int e = tid; e < P * P; e += blockDim.x) Sout[e] = S[(e & 31) * P + swz(e >> 5)];
}

static double offrel(const std::vector<double>& S) {
  double off = 0, tot = 0;
  for (int i = 0; i < P; ++i)
    for (int j = 0; j < P; ++j) {
      tot += S[i * P + j] * S[i * P + j];
      if (i != j) off += S[i * P + j] * S[i * P + j];
    }
  return std::sqrt(off / tot);
}

int main() {
  std::vector<double> S(P * P);
  srand(7);
  for (int i = 0; i < P; ++i)
    for (int j = 0; j <= i; ++j) {
      double v = (rand() / (double)RAND_MAX - 0.5) * std::exp(-0.2 * (i + j));
      S[i * P + j] = S[j * P + i] = v + (i == j ? 2.0 * std::exp(-0.4 * i) : 0.0);
    }
  double *dS, *dO;
  long long* dc;
  cudaMalloc(&dS, P * P * 8);
  cudaMalloc(&dO, P * P * 8);
  cudaMalloc(&dc, 32);
  cudaMemcpy(dS, S.data(), P * P * 8, cudaMemcpyHostToDevice);
  std::vector<double> O(P * P);
  long long c[4];
  for (int sweeps : {1, 4}) {
    kA<0><<<1, 256>>>(dS, dO, dc, sweeps, 1e-15);
    kA<1><<<1, 256>>>(dS, dO, dc, sweeps, 1e-15);
    kB<<<1, 32>>>(dS, dO, dc, sweeps, 1e-15);
    cudaDeviceSynchronize();
    kA<1><<<1, 256>>>(dS, dO, dc, sweeps, 1e-15);
    cudaMemcpy(O.data(), dO, P * P * 8, cudaMemcpyDeviceToHost);
    double oa1 = offrel(O);
    kA<0><<<1, 256>>>(dS, dO, dc, sweeps, 1e-15);
    cudaMemcpy(O.data(), dO, P * P * 8, cudaMemcpyDeviceToHost);
    double oa = offrel(O);
    kB<<<1, 32>>>(dS, dO, dc, sweeps, 1e-15);
    cudaMemcpy(O.data(), dO, P * P * 8, cudaMemcpyDeviceToHost);
    double ob = offrel(O);
    long long cc[8];
    kD<0><<<1, 288>>>(dS, dO, dc, sweeps, 1e-15);
    cudaMemcpy(O.data(), dO, P * P * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(cc, dc, 32, cudaMemcpyDeviceToHost);
    printf("D (param warp) %.0f cyc/step (off %.2e) %s\n", cc[3] / (31.0 * sweeps), offrel(O), cudaGetErrorString(cudaGetLastError()));
    kD<1><<<1, 288>>>(dS, dO, dc, sweeps, 1e-15);
    cudaMemcpy(O.data(), dO, P * P * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(cc, dc, 32, cudaMemcpyDeviceToHost);
    printf("D2 (param warp, 2-rsqrt chain) %.0f cyc/step (off %.2e) %s\n", cc[3] / (31.0 * sweeps), offrel(O), cudaGetErrorString(cudaGetLastError()));
    kC<0,0,0><<<1, 256>>>(dS, dO, dc, sweeps, 1e-15);
    cudaMemcpy(O.data(), dO, P * P * 8, cudaMemcpyDeviceToHost);
    double oc = offrel(O);
    cudaMemcpy(cc, dc, 32, cudaMemcpyDeviceToHost); cc[4] = cc[3];
    kC<1,0,0><<<1, 256>>>(dS, dO, dc, sweeps, 1e-15); cudaMemcpy(cc, dc, 32, cudaMemcpyDeviceToHost); cc[5] = cc[3];
    kC<0,1,0><<<1, 256>>>(dS, dO, dc, sweeps, 1e-15); cudaMemcpy(cc, dc, 32, cudaMemcpyDeviceToHost); cc[6] = cc[3];
    kC<1,1,1><<<1, 256>>>(dS, dO, dc, sweeps, 1e-15); cudaMemcpy(cc, dc, 32, cudaMemcpyDeviceToHost); cc[7] = cc[3];
    printf("C variants: full %.0f  noQ %.0f  noParams %.0f  nothing-stored %.0f\n", cc[4] / (31.0 * sweeps), cc[5] / (31.0 * sweeps), cc[6] / (31.0 * sweeps), cc[7] / (31.0 * sweeps));
    kC<0,0,0><<<1, 256>>>(dS, dO, dc, sweeps, 1e-15);
    cudaMemcpy(c, dc, 32, cudaMemcpyDeviceToHost);
    printf("C (xor, swizzled, 1 sync) %.0f cyc/step (off %.2e)\n", c[3] / (31.0 * sweeps), oc);
    printf("sweeps %d: A %.0f cyc/step (off %.2e)  A-fast %.0f (off %.2e)  B %.0f cyc/step (off %.2e)  err %s\n", sweeps,
           c[0] / (31.0 * sweeps), oa, c[2] / (31.0 * sweeps), oa1, c[1] / (31.0 * sweeps), ob,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
