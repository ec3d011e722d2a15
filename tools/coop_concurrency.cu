// Probe: do two cooperative launches on two streams of ONE device run
// concurrently?  (The single-GPU two-rank test of the sharded solver runs
// rank 0 and rank 1 as two half-grid persistent kernels that spin on each
// other's flags.)  Each kernel's block 0 raises its flag and waits up to
// 2 s for the other's; prints whether both saw each other.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/coop_concurrency tools/coop_concurrency.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_probe(volatile int* flags, int me, int* seen) {
  __shared__ double pad[6000];  // 48 KB
  pad[threadIdx.x] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    flags[me] = 1;
    __threadfence();
    const unsigned long long t0 = gt();
    int ok = 0;
    while (gt() - t0 < 2000000000ull) {
      if (flags[1 - me]) { ok = 1; break; }
    }
    seen[me] = ok;
  }
  __syncthreads();
  if (pad[threadIdx.x] != 0) seen[2] = 1;
}

int main() {
  int *flags, *seen;
  cudaMalloc(&flags, 16);
  cudaMalloc(&seen, 16);
  cudaMemset(flags, 0, 16);
  cudaMemset(seen, 0, 16);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 0);
  cudaStream_t s[2];
  for (int i = 0; i < 2; ++i) cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking);
  for (int coop = 1; coop >= 0; --coop) {
    cudaMemset(flags, 0, 16);
    cudaMemset(seen, 0, 16);
    cudaDeviceSynchronize();
    for (int me = 0; me < 2; ++me) {
      int mm = me;
      void* args[] = {&flags, &mm, &seen};
      cudaError_t e = coop ? cudaLaunchCooperativeKernel((void*)k_probe, dim3(74), dim3(256),
                                                         args, 0, s[me])
                           : cudaLaunchKernel((void*)k_probe, dim3(74), dim3(256), args, 0,
                                              s[me]);
      if (e != cudaSuccess) printf("launch %d: %s\n", me, cudaGetErrorString(e));
    }
    cudaError_t e = cudaDeviceSynchronize();
    int h[3];
    cudaMemcpy(h, seen, 12, cudaMemcpyDeviceToHost);
    printf("{\"cooperative\": %d, \"sync\": \"%s\", \"rank0_saw_rank1\": %d, "
           "\"rank1_saw_rank0\": %d}\n", coop, cudaGetErrorString(e), h[0], h[1]);
  }
  return 0;
}
