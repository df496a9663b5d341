#include <cstdio>
__device__ __forceinline__ double rcp_nr(double x) {
  double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0); r = fma(r, e, r); e = fma(-x, r, 1.0); return fma(r, e, r);
}
__global__ void k(double* out, long long* cyc, double a, int n) {
  __shared__ double sm[64];
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999, 1e-3);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = rcp_nr(x + 1.0);
  long long t2 = clock64();
  sm[threadIdx.x] = x; __syncthreads();
  int idx = threadIdx.x;
  for (int i = 0; i < n; ++i) { idx = (int)sm[idx & 63] & 63; }
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
  long long t5 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.0);
  long long t6 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5-t4; cyc[5]=t6-t5; }
  out[threadIdx.x] = x + idx;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 256); cudaMalloc(&c, 64);
  for (int th : {32, 256}) {
    k<<<1, th>>>(o, c, 1.0, 1000); cudaDeviceSynchronize();
    k<<<1, th>>>(o, c, 1.0, 1000);
    long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
    printf("threads %d: dfma %.1f  rcp_nr %.1f  lds-chain %.1f  syncthreads %.1f  sqrt %.1f  div %.1f cycles each\n", th, h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0, h[4]/1000.0, h[5]/1000.0);
  }
}
