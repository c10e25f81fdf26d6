// FP64 peak microbenchmark ("FP64 peak is not measured ... measure
// it with a DFMA microbenchmark at sustained clocks").  Two kernels:
//   dfma: 8 independent DFMA chains per thread, grid = SMs x 8 CTAs x 256 threads;
//   dmma: mma.sync.aligned.m8n8k4 f64 (the only FP64 tensor-core form on sm_100a;
//         tcgen05 has no f64 kind), 4 independent accumulators per warp.
// Prints one JSON line: TFLOP/s of each (2 flops per FMA, 2*8*8*4 per MMA), best of
// `reps` timed runs of `iters` iterations, CUDA events around each launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1.2345) out[blockIdx.x] = s;  // keeps the chains alive
}

__global__ void dmma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
  double c[4][2];
#pragma unroll
  for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 1.2345) out[blockIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0, mhz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256, reps = 5;
  const int it_fma = 1 << 16, it_mma = 1 << 14;
  float best_fma = 1e30f, best_mma = 1e30f;
  dfma<<<blocks, threads>>>(out, 1024, 0.999999, 1e-7);  // warm-up (clocks up)
  dmma<<<blocks, threads>>>(out, 1024);
  for (int r = 0; r < reps; ++r) {
    float ms;
    cudaEventRecord(e0);
    dfma<<<blocks, threads>>>(out, it_fma, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best_fma = ms < best_fma ? ms : best_fma;
    cudaEventRecord(e0);
    dmma<<<blocks, threads>>>(out, it_mma);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best_mma = ms < best_mma ? ms : best_mma;
  }
  const double fma_flops = 2.0 * 8.0 * it_fma * double(blocks) * threads;
  const double mma_flops = 2.0 * 8 * 8 * 4 * 4.0 * it_mma * double(blocks) * (threads / 32);
  const cudaError_t err = cudaGetLastError();
  std::printf("{\"fp64_dfma_tflops\": %.3f, \"fp64_dmma_tflops\": %.3f, \"sms\": %d, \"clock_mhz_attr\": %d, "
              "\"dfma_ms\": %.3f, \"dmma_ms\": %.3f, \"how\": \"8 independent DFMA chains per thread / 4 "
              "independent m8n8k4 f64 mma.sync per warp, %d CTAs x %d threads, best of %d, CUDA events\", "
              "\"error\": \"%s\"}\n",
              fma_flops / best_fma / 1e9, mma_flops / best_mma / 1e9, sms, mhz / 1000, best_fma, best_mma, blocks,
              threads, reps, cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
