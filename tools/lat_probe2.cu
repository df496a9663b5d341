#include <cstdio>
__device__ __forceinline__ double rcp_nr(double x) {
  double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0); r = fma(r, e, r); e = fma(-x, r, 1.0); return fma(r, e, r);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
  double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double h = 0.5 * x; r = r * fma(-h * r, r, 1.5); r = r * fma(-h * r, r, 1.5); return r;
}
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
__global__ void k(double* out, long long* cyc, double a, int n) {
  double x = a, y = 0.3, z = 0.1;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { double c, s, dA, dB; int act; rot_params(x, y, z, 1e-30, 1e-300, c, s, dA, dB, act); x = dA + c * 1e-3; y = dB; z = s * 0.5 + 0.01; }
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt_nr(x + 1.0);
  long long t2 = clock64();
  double r;
  for (int i = 0; i < n; ++i) { asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 1.0; }
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) { asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 1.0; }
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) { float f = (float)x; f = rsqrtf(f); x = (double)f + 1.0; }
  long long t5 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
  out[threadIdx.x] = x + y + z;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 256); cudaMalloc(&c, 64);
  for (int th : {1, 32}) {
    k<<<1, th>>>(o, c, 1.0, 1000); cudaDeviceSynchronize();
    k<<<1, th>>>(o, c, 1.0, 1000);
    long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
    printf("threads %d: rot_params %.1f  rsqrt_nr+add %.1f  MUFU.RSQ64H+add %.1f  MUFU.RCP64H+add %.1f  f32 rsqrt+cvt %.1f cycles\n", th, h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0, h[4] / 1000.0);
  }
}
