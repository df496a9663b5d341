// fp64_peak.cu - FP64 peak microbenchmarks on B200 (sm_100a): the roofline denominator
// for the DMMA kernels (MEASURED_PEAKS.json has no FP64 entry).
//   dmma : independent mma.sync.m8n8k4.f64 chains, register resident (SASS DMMA.8x8x4)
//   dfma : independent fma.rn.f64 chains
// Prints one JSON line.  Usage: fp64_peak [seconds_per_test]
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double d[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[i][0]), "+d"(d[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dfma_kernel(double* out, int iters) {
  double x[8];
  double a = 1.0 + threadIdx.x * 1e-12, b = 1e-9;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main(int argc, char** argv) {
  int dev = 0;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, dev);
  int sms = prop.multiProcessorCount;
  double* out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](bool mma, int blocks_per_sm, int threads, int iters) {
    dim3 g(sms * blocks_per_sm);
    for (int w = 0; w < 2; ++w) {
      if (mma) dmma_kernel<<<g, threads>>>(out, iters / 10);
      else dfma_kernel<<<g, threads>>>(out, iters / 10);
    }
    cudaEventRecord(e0);
    if (mma) dmma_kernel<<<g, threads>>>(out, iters);
    else dfma_kernel<<<g, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = mma ? (double)g.x * (threads / 32) * iters * 8 * 512.0
                       : (double)g.x * threads * iters * 8 * 2.0;
    return flops / (ms * 1e-3) / 1e12;
  };
  double best_mma = 0, best_fma = 0;
  int cfg_mma = 0, cfg_fma = 0;
  int tpb[] = {128, 256, 512, 1024};
  for (int t : tpb) {
    double v = run(true, 2, t, 20000);
    if (v > best_mma) best_mma = v, cfg_mma = t;
    double f = run(false, 2, t, 20000);
    if (f > best_fma) best_fma = f, cfg_fma = t;
  }
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d, \"dmma_tflops\": %.3f, \"dmma_threads\": %d, "
         "\"dfma_tflops\": %.3f, \"dfma_threads\": %d, \"nominal_fp64_tflops_at_max_clock\": %.2f}\n",
         prop.name, sms, clk, best_mma, cfg_mma, best_fma, cfg_fma, sms * 128.0 * clk * 1e3 / 1e12);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "CUDA error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
