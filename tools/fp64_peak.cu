// FP64 FMA throughput microbenchmark ("the FP64 figure is not measured: add an
// FP64-FMA microbenchmark").  Independent DFMA chains per thread, full-GPU grid, CUDA events.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_peak.cu -o /tmp/fp64_peak && /tmp/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;
constexpr int ITERS = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
  double v[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) v[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) v[c] = fma(v[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += v[c];
  if (s == 12345.678) out[0] = s;   // keep the chains alive
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, sizeof(double));
  const int threads = 256, blocks = sms * 8;
  dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(s);
    dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms;
    cudaEventElapsedTime(&ms, s, e);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * CHAINS * ITERS * (double)threads * blocks;
  const double tf = flops / (best * 1e-3) / 1e12;
  const double nominal = sms * 64.0 * 2.0 * clk * 1e3 / 1e12;   // 64 DFMA/clk/SM at the max clock
  printf("{\"fp64_tflops\": %.3f, \"nominal_tflops_at_max_clock\": %.3f, \"sms\": %d, \"max_clock_mhz\": %d, "
         "\"how\": \"%d independent DFMA chains x %d iterations per thread, %d x %d threads, best of 10, CUDA events\"}\n",
         tf, nominal, sms, clk / 1000, CHAINS, ITERS, blocks, threads);
  return 0;
}
