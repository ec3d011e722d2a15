// bw_probe.cu -- calibration of streaming bandwidth for the persistent-kernel
// geometry (development tool, not part of the product library).
// Pattern of the cone step: 5 float64 reads + 2 writes per element.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bw_probe tools/bw_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

template <int U>
__global__ void stream7(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                        const double* __restrict__ c, const double* __restrict__ d,
                        const double* __restrict__ e, double* __restrict__ o1,
                        double* __restrict__ o2, double tau) {
  const int64_t S = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < n; base += U * S) {
    double va[U], vb[U], vc[U], vd[U], ve[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t i = base + u * S;
      i = i < n ? i : n - 1;
      va[u] = a[i]; vb[u] = b[i]; vc[u] = c[i]; vd[u] = d[i]; ve[u] = e[i];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * S;
      if (i < n) {
        const double s = ((va[u] + vb[u]) - tau * vc[u]) - vd[u];
        const double u2 = fmax(s, 0.0);
        o1[i] = u2 - s;
        o2[i] = (u2 + (u2 - s)) * ve[u];
      }
    }
  }
}

// plain copy (1 read + 1 write) for the reference number
__global__ void copy1(int64_t n, const double* __restrict__ a, double* __restrict__ o) {
  const int64_t S = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += S) o[i] = a[i];
}

template <class K>
float timeit(K launch, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

// time one launch with a cold L2 (256 MiB scrub before it)
template <class K>
float timecold(K launch, double* scrub, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f, sum = 0;
  for (int r = 0; r < reps; ++r) {
    cudaMemsetAsync(scrub, r & 0xff, 256ull << 20);
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    sum += ms;
    best = ms < best ? ms : best;
  }
  return sum / reps;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int64_t n : {1000000LL, 2000000LL, 16000000LL}) {
    double* p[7];
    for (auto& q : p) {
      cudaMalloc(&q, n * 8);
      cudaMemset(q, 0, n * 8);
    }
    const double bytes7 = 7.0 * 8 * n;
    struct Cfg { int blocks_per_sm, threads, u; };
    Cfg cfgs[] = {{1, 512, 4}, {1, 512, 8}, {1, 1024, 4}, {2, 512, 4}, {4, 256, 4}, {8, 256, 2}};
    for (auto c : cfgs) {
      const int grid = sms * c.blocks_per_sm;
      float ms;
      if (c.u == 4)
        ms = timeit([&] { stream7<4><<<grid, c.threads>>>(n, p[0], p[1], p[2], p[3], p[4], p[5], p[6], 0.5); }, 20);
      else if (c.u == 8)
        ms = timeit([&] { stream7<8><<<grid, c.threads>>>(n, p[0], p[1], p[2], p[3], p[4], p[5], p[6], 0.5); }, 20);
      else
        ms = timeit([&] { stream7<2><<<grid, c.threads>>>(n, p[0], p[1], p[2], p[3], p[4], p[5], p[6], 0.5); }, 20);
      printf("n=%lld grid=%dx%d U=%d: %.2f us  %.0f GB/s\n", (long long)n, grid, c.threads, c.u,
             ms * 1e3, bytes7 / (ms * 1e-3) / 1e9);
    }
    double* scrub;
    cudaMalloc(&scrub, 256ull << 20);
    for (auto c : cfgs) {
      const int grid = sms * c.blocks_per_sm;
      float ms;
      if (c.u == 4)
        ms = timecold([&] { stream7<4><<<grid, c.threads>>>(n, p[0], p[1], p[2], p[3], p[4], p[5], p[6], 0.5); }, scrub, 10);
      else if (c.u == 8)
        ms = timecold([&] { stream7<8><<<grid, c.threads>>>(n, p[0], p[1], p[2], p[3], p[4], p[5], p[6], 0.5); }, scrub, 10);
      else
        ms = timecold([&] { stream7<2><<<grid, c.threads>>>(n, p[0], p[1], p[2], p[3], p[4], p[5], p[6], 0.5); }, scrub, 10);
      printf("COLD n=%lld grid=%dx%d U=%d: %.2f us  %.0f GB/s\n", (long long)n, grid, c.threads, c.u,
             ms * 1e3, bytes7 / (ms * 1e-3) / 1e9);
    }
    cudaFree(scrub);
    float ms = timeit([&] { copy1<<<sms * 8, 256>>>(n, p[0], p[5]); }, 20);
    printf("n=%lld copy: %.2f us %.0f GB/s\n", (long long)n, ms * 1e3, 16.0 * n / (ms * 1e-3) / 1e9);
    for (auto& q : p) cudaFree(q);
  }
  return 0;
}
