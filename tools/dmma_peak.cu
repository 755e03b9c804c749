// dmma_peak.cu — FP64 tensor-core (mma.sync.m8n8k4.f64, DMMA) throughput on
// this B200, alone and interleaved with FP64 vector FMAs (do the two pipes run
// concurrently?).  Decides whether the predictor's 4x4 nodal contractions
// can move to the tensor cores.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_peak dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int MC = 8;    // independent DMMA accumulator chains per warp
constexpr int FC = 8;    // independent DFMA chains per thread

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <bool MMA, bool FMA>
__global__ void __launch_bounds__(256) loop(double* out, int iters, double a, double b) {
  double c[MC][2], x[FC];
#pragma unroll
  for (int i = 0; i < MC; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < FC; ++i) x[i] = threadIdx.x * 1e-3 + i;
  const double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
    if (MMA) {
#pragma unroll
      for (int i = 0; i < MC; ++i) dmma(c[i], av, bv);
    }
    if (FMA) {
#pragma unroll
      for (int i = 0; i < FC; ++i) x[i] = fma(x[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < MC; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < FC; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

template <bool MMA, bool FMA>
void run(const char* name, int blocks, double* out) {
  const int threads = 256, iters = 4000;
  loop<MMA, FMA><<<blocks, threads>>>(out, 100, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    loop<MMA, FMA><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double warps = (double)blocks * threads / 32;
  const double mma_fl = MMA ? 512.0 * MC * iters * warps : 0.0;   // 8x8x4 FMA per warp instruction
  const double fma_fl = FMA ? 2.0 * FC * iters * warps * 32 : 0.0;
  std::printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f, \"total_tflops\": %.2f}\n",
              name, best, mma_fl / best / 1e9, fma_fl / best / 1e9, (mma_fl + fma_fl) / best / 1e9);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int blocks = p.multiProcessorCount * 8;
  run<true, false>("dmma_m8n8k4", blocks, out);
  run<false, true>("dfma", blocks, out);
  run<true, true>("dmma+dfma", blocks, out);
  return 0;
}
