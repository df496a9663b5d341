// dmma_sweep.cu - how many warps per SM and independent accumulator chains does
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4) need to saturate the B200 FP64 pipe?
// One CTA per SM; prints one JSON line per (warps, chains, smem-operand) point.
#include <cuda_runtime.h>
#include <cstdio>

template <int C, bool LDS>
__global__ void k(double* out, int iters) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
  __syncthreads();
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double d[C][2];
#pragma unroll
  for (int i = 0; i < C; ++i) d[i][0] = d[i][1] = 0.0;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    if (LDS) {
      a = sm[(lane + it * 32) & 1023];
      b = sm[(lane * 2 + it * 64 + 7) & 1023];
    }
#pragma unroll
    for (int i = 0; i < C; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) s += d[i][0] + d[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  int sms = prop.multiProcessorCount;
  double* out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, int C, bool lds, int warps) {
    int iters = 4096 * 32 / C;
    kern<<<sms, warps * 32>>>(out, iters / 8);
    cudaEventRecord(e0);
    kern<<<sms, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = (double)sms * warps * iters * C * 512.0;
    printf("{\"warps_per_sm\": %d, \"chains\": %d, \"lds_operands\": %d, \"tflops\": %.3f}\n", warps, C, (int)lds,
           fl / (ms * 1e-3) / 1e12);
  };
  int W[] = {4, 8, 12, 16, 24, 32};
  for (int w : W) {
    run(k<4, false>, 4, false, w);
    run(k<8, false>, 8, false, w);
    run(k<16, false>, 16, false, w);
    run(k<32, false>, 32, false, w);
    run(k<16, true>, 16, true, w);
    run(k<32, true>, 32, true, w);
  }
  return cudaGetLastError() != cudaSuccess;
}
