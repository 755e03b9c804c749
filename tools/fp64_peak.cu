// fp64_peak.cu — FP64 FMA-pipe throughput microbenchmark: the measured FP64
// roofline denominator (MEASURED_PEAKS.json has no FP64 entry).
//   burst:     best of 5 launches of ~50 ms each
//   sustained: back-to-back launches for ~4 s (power-capped steady state)
// Run under tools/gpu_fp64_peak.sh, which samples the SM clock with
// nvidia-smi during the run and writes profiles/round2_fp64_peak.json.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 16;   // independent FMA chains per thread (covers the DFMA latency)

__global__ void __launch_bounds__(256) dfma_loop(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 20000;
  dfma_loop<<<blocks, threads>>>(out, 100, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double flops = 2.0 * CH * (double)iters * blocks * threads;
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  // sustained: ~4 s of back-to-back launches
  int n = 0;
  const auto t0 = std::chrono::steady_clock::now();
  cudaEventRecord(e0);
  while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < 4.0) {
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    ++n;
    if (n % 8 == 0) cudaDeviceSynchronize();
  }
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float tot;
  cudaEventElapsedTime(&tot, e0, e1);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"fp64_fma_tflops_burst\": %.3f, \"fp64_fma_tflops_sustained\": %.3f, \"sms\": %d, \"burst_ms\": %.3f, "
         "\"sustained_launches\": %d, \"clock_attr_mhz\": %.0f}\n",
         flops / best / 1e9, flops * n / tot / 1e9, p.multiProcessorCount, best, n, clk / 1e3);
  return 0;
}
