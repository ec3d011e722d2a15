// fp64_peak.cu -- measured FP64 (DFMA) peak of this B200, the FP64
// denominator of bench.py's roofline (profiles/fp64_peak.json).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_peak tools/fp64_peak.cu
//   tools/fp64_peak > profiles/fp64_peak.json
//
// Every thread runs NCHAIN independent DFMA chains (no memory traffic);
// timed with CUDA events over several launches; reports the best.  Also
// the rate at one 256-thread CTA per SM (the persistent kernels' shape).
#include <cuda_runtime.h>
#include <cstdio>

#define NCHAIN 16

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[NCHAIN];
#pragma unroll
  for (int i = 0; i < NCHAIN; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCHAIN; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NCHAIN; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

static double run(int blocks, int threads, int iters) {
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_loop<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaFree(d);
  const double flops = 2.0 * NCHAIN * (double)iters * blocks * threads;
  return flops / (best * 1e-3) / 1e12;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double full = run(sms * 8, 256, 4096);          // 64 warps / SM
  const double one = run(sms, 256, 4096 * 4);           // 8 warps / SM (persistent shape)
  std::printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_clock_khz\": %d, \"dfma_tflops\": %.3f, "
              "\"dfma_tflops_8warps_per_sm\": %.3f, \"how\": \"%d independent DFMA chains per "
              "thread, best of 5 launches, CUDA events; 2 flops per DFMA\"}\n",
              p.name, sms, clk, full, one, NCHAIN);
  return 0;
}
