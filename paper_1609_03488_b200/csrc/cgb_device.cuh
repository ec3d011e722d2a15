// cgb_device.cuh -- device-side building blocks of the persistent solver
// kernels: grid barrier + deterministic grid reductions, the operator-plan
// executor (leaf tiles), cone projections.  Included by cgb200.cu only.
#pragma once

#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include "../../include/cgb200.h"

#ifndef CGB_BLOCK
#define CGB_BLOCK 256
#endif
#define CGB_WARPS (CGB_BLOCK / 32)
#ifndef CGB_MINB
#define CGB_MINB 1
#endif
#define CGB_MAXP 16          // reduction slots per grid reduction
#ifndef CGB_BAR_FENCE
#define CGB_BAR_FENCE 1      // grid-barrier fence flavour (see GridSync::sync)
#endif
#ifndef CGB_CTAS_PER_SM
#define CGB_CTAS_PER_SM CGB_MINB  // persistent CTAs per SM (grid = SMs x this)
#endif
#ifndef CGB_MAXG
#define CGB_MAXG (160 * CGB_CTAS_PER_SM)  // largest grid the reductions are unrolled for
#endif
#define CGB_MAX_LARGE_SOC 4  // SOC blocks reduced across the whole grid
#ifndef CGB_RC
#define CGB_RC 9             // rows per lane in convolution tiles (odd: no bank conflicts)
#endif
#ifndef CGB_DENSE_DR
#define CGB_DENSE_DR 8       // dense GEMV: rows per warp-group (loads in flight together)
#endif
#ifndef CGB_DENSE_UNROLL
#define CGB_DENSE_UNROLL 4   // dense GEMV: column chunks unrolled per row group
#endif
#define CGB_CONV_KMAX 240    // longest 1-d kernel of the register-blocked (TMA) tile path
#define CGB_SEP_KMAX 63      // widest rank-one 2-d kernel applied as column + row passes
#ifndef CGB_STRIP_RPW
#define CGB_STRIP_RPW 1      // output rows per warp per strip step
#endif
#define CGB_STRIP_RPS (CGB_WARPS * CGB_STRIP_RPW)  // output rows per strip step
#ifndef CGB_U
#define CGB_U 8              // elements per thread per batch in streaming loops
#endif

namespace cgb {

// ---------------------------------------------------------------------------
// device plan / cone descriptors (built by the host in cgb200.cu)
// ---------------------------------------------------------------------------
struct DevRowBlock {
  int64_t row_begin, row_end, tile_begin;
  int64_t period;     // > 0: the block is whole output rows of this width
                      // (a 2-d conv leaf); tiles never cross a row
  int32_t out_buf, term_begin, term_end;
  int32_t rfac;       // rows per lane in this block's tiles (1 or CGB_RC)
  int32_t conv_term;  // the block's only 1-d conv term (TMA-staged), or -1
  int32_t tpr;        // periodic blocks: tiles per row
  int32_t rpt;        // rows per tile (32 * rfac, or fewer for dense blocks)
  int32_t strip_term; // periodic blocks: the 2-d conv term run as CTA strips, or -1
};

// first row and row count of a tile of row block rb
template <bool PERIODIC>
__device__ __forceinline__ void tile_rows(const DevRowBlock& rb, int64_t tile, int64_t& row0,
                                          int& nvalid) {
  const int64_t rpt = rb.rpt;
  const int64_t t = tile - rb.tile_begin;
  if (PERIODIC && rb.period > 0) {
    const int64_t pr = t / rb.tpr, pc = t - pr * rb.tpr;
    row0 = rb.row_begin + pr * rb.period + pc * rpt;
    const int64_t rem = rb.period - pc * rpt;
    nvalid = (int)(rem < rpt ? rem : rpt);
  } else {
    row0 = rb.row_begin + t * rpt;
    const int64_t rem = rb.row_end - row0;
    nvalid = (int)(rem < rpt ? rem : rpt);
  }
}

// All metadata arrays of a plan live in one device blob [meta, meta +
// meta_bytes) so a kernel can copy the whole plan into shared memory once
// (cache_plan) and rebase the pointers.
struct DevPlan {
  const cgb_leaf* leaves;
  const cgb_term* terms;
  const DevRowBlock* rbs;
  const int32_t* level_rb;     // nlevels + 1, execution order (deepest first)
  const int64_t* level_tiles;  // nlevels
  const int64_t* temp_off;     // ntemps
  const int32_t* leaf_taps;    // per leaf: offset into taps, or -1
  const double* taps;          // correlation taps of the tiled 1-d conv leaves
                               // (reversed for conv), zero padded to RC
  const char* meta;            // blob holding every array above
  double* temp[2];             // two temporary sets (two applications per phase)
  int32_t meta_bytes;
  int32_t nlevels;
  int32_t smem_per_warp;  // doubles of dynamic shared memory per warp
  int32_t smem_cc;        // (unused, 0)
  int32_t smem_xs;        // one staged-input window; two windows, then the
                          // 32*RC+1 output transpose, then the 2-d ring
  int32_t smem_xs2;       // one 2-d conv row window (CGB_RING2 of them)
  int32_t strip_slot;     // 2-d strips: doubles per input-row slot of the CTA ring
  int32_t strip_nslot;    // slots in the ring (kh + 15)
  int32_t strip_rows;     // output rows per strip task (multiple of CGB_WARPS)
  int32_t smem_total;     // doubles of dynamic shared memory the plan needs per CTA
  int64_t in_len, out_len;
};

enum SegKind : int32_t { SEG_ZERO = 0, SEG_NONNEG = 1, SEG_SOC_LARGE = 2, SEG_SOC_TAIL = 3 };

struct DevSeg {
  int64_t begin, end;
  int32_t kind, slot;
};

struct DevCones {
  const DevSeg* seg;
  const int64_t* small_off;
  const int32_t* small_dim;
  const int64_t* exp_off;
  int64_t m;
  int32_t nseg, nsmall, nexp, nlarge;
};

// ---------------------------------------------------------------------------
// grid barrier and deterministic reductions
// ---------------------------------------------------------------------------
// Monotonic 64-bit arrival counter, zeroed by the host before every launch:
// barrier e completes when the counter reaches e * gridDim.x.  Arrival is a
// fire-and-forget release reduction; every block polls with acquire loads.
struct GridBar {
  unsigned long long count;
  unsigned int err;
  unsigned int pad;
};

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, sm_90+) with mbarrier completion
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// arrive (count 1) announcing `bytes` of transaction, then the bulk copy
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "{\n .reg .b64 st;\n"
      " mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "CGB_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra CGB_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// run_level timeline probe (profiling only): when cgb_tl_acc != null, warp 0
// of block 0 adds its per-tile phase times (ns) to cgb_tl_acc[0..7]
__shared__ double* cgb_tl_acc;

// lane 0 issues one bulk copy into `dst` once the warp's earlier reads of it
// are fenced off from the async proxy
__device__ __forceinline__ void issue_bulk(double* dst, const double* src, uint32_t bytes,
                                           uint64_t* bar, int lane) {
  __syncwarp();
  if (lane == 0) {
    fence_proxy_async();
    bulk_load(dst, src, bytes, bar);
  }
}

// per-warp pair of mbarriers for the double-buffered conv windows, and the
// parity each buffer's next completion will have (bit b for buffer b)
#define CGB_RING2 4  // row windows in flight per warp in a 2-d conv tile
__shared__ uint64_t cgb_mbar[CGB_WARPS][2 + CGB_RING2];
__shared__ uint32_t cgb_mbar_phase[CGB_WARPS];
// CTA-level mbarriers of the 2-d strip row ring (batch g uses g & 1) and the
// number of batches this CTA has issued
__shared__ uint64_t cgb_strip_mbar[2];
__shared__ uint32_t cgb_strip_seq;

// every persistent kernel calls this first (all threads)
__device__ __forceinline__ void tma_init() {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  if (lane == 0) {
    for (int i = 0; i < 2 + CGB_RING2; ++i) mbar_init(&cgb_mbar[wib][i], 1);
    cgb_mbar_phase[wib] = 0;
    fence_mbar_init();
  }
  if (threadIdx.x == 0) {
    cgb_tl_acc = nullptr;
    mbar_init(&cgb_strip_mbar[0], 1);
    mbar_init(&cgb_strip_mbar[1], 1);
    cgb_strip_seq = 0;
    fence_mbar_init();
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// plan cache: a kernel copies its (small) plans into shared memory once, so
// the per-tile metadata lookups of every later phase are shared loads
// ---------------------------------------------------------------------------
#define CGB_PLAN_SMEM 6144
__shared__ __align__(16) char cgb_plan_meta[2][CGB_PLAN_SMEM];
__shared__ DevPlan cgb_plan_view[2];

template <class T>
__device__ __forceinline__ const T* rebase(const T* p, const char* from, char* to) {
  return p ? reinterpret_cast<const T*>(to + (reinterpret_cast<const char*>(p) - from)) : p;
}

// all threads; returns the shared copy, or P itself if it does not fit
__device__ __forceinline__ const DevPlan* cache_plan(int slot, const DevPlan& P) {
  if (P.meta_bytes > CGB_PLAN_SMEM || P.meta == nullptr) return &P;
  const int4* src = reinterpret_cast<const int4*>(P.meta);
  int4* dst = reinterpret_cast<int4*>(cgb_plan_meta[slot]);
  for (int i = threadIdx.x; i < (P.meta_bytes + 15) / 16; i += blockDim.x) dst[i] = src[i];
  if (threadIdx.x == 0) {
    DevPlan v = P;
    char* to = cgb_plan_meta[slot];
    v.leaves = rebase(P.leaves, P.meta, to);
    v.terms = rebase(P.terms, P.meta, to);
    v.rbs = rebase(P.rbs, P.meta, to);
    v.level_rb = rebase(P.level_rb, P.meta, to);
    v.level_tiles = rebase(P.level_tiles, P.meta, to);
    v.temp_off = rebase(P.temp_off, P.meta, to);
    v.leaf_taps = rebase(P.leaf_taps, P.meta, to);
    v.taps = rebase(P.taps, P.meta, to);
    cgb_plan_view[slot] = v;
  }
  __syncthreads();
  return &cgb_plan_view[slot];
}

struct GridSync {
  GridBar* bar;
  double* partials;  // [2 banks][CGB_MAXP][grid]
  int bank;
  unsigned long long target;
  bool cluster;      // the grid is ONE thread-block cluster (small problems)

  __device__ GridSync(GridBar* b, double* p) : bar(b), partials(p), bank(0), target(0) {
    unsigned n;
    asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
    cluster = n > 1 && n == gridDim.x;
  }

  // All threads of all blocks must call this (uniform control flow).
  // FENCE selects the ordering around the arrival: 2 = fence.sc before and
  // after (cooperative-groups style), 1 = fence.acq_rel before the release
  // arrival, 0 = release / acquire only.  The CTA barrier on either side
  // carries the other threads' accesses (bar.sync is morally strong, and
  // release / acquire are cumulative over what thread 0 has observed).
  template <int FENCE = CGB_BAR_FENCE>
  __device__ void sync() {
    if (cluster) {
      // launched as one cluster: the hardware cluster barrier (release /
      // acquire at cluster scope orders the global-memory phases too)
      asm volatile("barrier.cluster.arrive.release.aligned;\n"
                   "barrier.cluster.wait.acquire.aligned;" ::: "memory");
      return;
    }
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
      if (FENCE == 2) __threadfence();
      if (FENCE == 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      red_release_add(&bar->count, 1ull);
      if (ld_acquire_u64(&bar->count) < target) {
        const uint64_t t0 = globaltimer();
        while (ld_acquire_u64(&bar->count) < target) {
          if (globaltimer() - t0 > 20000000000ull) {  // 20 s: never expected
            atomicExch(&bar->err, 1u);
            __trap();
          }
        }
      }
      if (FENCE == 2) __threadfence();
    }
    __syncthreads();
  }

  // Sum v[0..NP) over every thread of the grid.  The result is bitwise
  // identical in every thread of every block (fixed summation order), so
  // control decisions taken on it stay grid-uniform.  Warp p owns slot p:
  // it folds the block's warp sums into the block partial before the
  // barrier and, after it, reads all gridDim.x partials of its slot with
  // every load in flight at once (one L2 round trip for any NP <= 16).
  template <int NP>
  __device__ void reduce(double (&v)[NP]) {
    static_assert(NP <= CGB_MAXP && NP <= CGB_WARPS, "too many reduction slots");
    __shared__ double red_smem[CGB_WARPS][CGB_MAXP];
    __shared__ double red_out[CGB_MAXP];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      double s = v[p];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) red_smem[wid][p] = s;
    }
    __syncthreads();
    const int G = gridDim.x;
    double* bankp = partials + (size_t)bank * CGB_MAXP * G;
    if (wid < NP) {
      double s = lane < CGB_WARPS ? red_smem[lane][wid] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) bankp[(size_t)wid * G + blockIdx.x] = s;
    }
    sync();
    if (wid < NP) {
      constexpr int NI = (CGB_MAXG + 31) / 32;
      const double* src = bankp + (size_t)wid * G;
      double x[NI];
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int idx = lane + 32 * i;
        x[i] = idx < G ? __ldcg(src + idx) : 0.0;
      }
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < NI; ++i) s += x[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) red_out[wid] = s;
    }
    __syncthreads();
#pragma unroll
    for (int p = 0; p < NP; ++p) v[p] = red_out[p];
    bank ^= 1;
  }

  // Max of v[0..NP) over every thread of the grid (same structure as
  // reduce; max is order independent, so the result is exact).
  template <int NP>
  __device__ void reduce_max(double (&v)[NP]) {
    static_assert(NP <= CGB_MAXP && NP <= CGB_WARPS, "too many reduction slots");
    __shared__ double rmx_smem[CGB_WARPS][CGB_MAXP];
    __shared__ double rmx_out[CGB_MAXP];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      double s = v[p];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
      if (lane == 0) rmx_smem[wid][p] = s;
    }
    __syncthreads();
    const int G = gridDim.x;
    double* bankp = partials + (size_t)bank * CGB_MAXP * G;
    if (wid < NP) {
      double s = lane < CGB_WARPS ? rmx_smem[lane][wid] : -DBL_MAX;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
      if (lane == 0) bankp[(size_t)wid * G + blockIdx.x] = s;
    }
    sync();
    if (wid < NP) {
      const double* src = bankp + (size_t)wid * G;
      double s = -DBL_MAX;
      for (int i = lane; i < G; i += 32) s = fmax(s, __ldcg(src + i));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
      if (lane == 0) rmx_out[wid] = s;
    }
    __syncthreads();
#pragma unroll
    for (int p = 0; p < NP; ++p) v[p] = rmx_out[p];
    bank ^= 1;
  }
};

__device__ __forceinline__ int64_t gtid() {
  return (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
}
__device__ __forceinline__ int64_t gsize() { return (int64_t)gridDim.x * blockDim.x; }

// Batched grid-stride loop: each thread handles CGB_U elements per step
// (indices i, i+S, i+2S, ...), calling f.load(i, slot) for all of them
// before f.compute(i, slot), so the loads of a batch are in flight together.
// The ragged last batch loads from a clamped (valid) index instead of
// branching around the loads, which would serialise them; f.load must
// therefore be side-effect free.
template <class F>
__device__ __forceinline__ void stream_loop(int64_t n, F& f) {
  const int64_t S = gsize();
  for (int64_t base = gtid(); base < n; base += CGB_U * S) {
    if (base + (CGB_U - 1) * S < n) {
#pragma unroll
      for (int u = 0; u < CGB_U; ++u) f.load(base + u * S, u);
#pragma unroll
      for (int u = 0; u < CGB_U; ++u) f.compute(base + u * S, u);
    } else {
#pragma unroll
      for (int u = 0; u < CGB_U; ++u) {
        const int64_t i = base + u * S;
        f.load(i < n ? i : n - 1, u);
      }
#pragma unroll
      for (int u = 0; u < CGB_U; ++u) {
        const int64_t i = base + u * S;
        if (i < n) f.compute(i, u);
      }
    }
  }
}

// Stream pass over [0, n) of NIN input vectors: f.compute(i, v, j) with
// v[a] = src[a][i] and j a per-CTA slot index unique to (thread, visit)
// -- the same in every pass over the same n, so a pass can leave values in
// shared memory (stash) for a later one.  Grid-stride, CGB_U elements per
// thread per batch, every load of a batch in flight before the first use
// (the ragged batch loads clamped indices).  Contiguous per-CTA ranges fed
// by TMA bulk copies were measured slower on B200 for these 1e6-element
// passes (one block-wide sync per chunk), see DESIGN.md.
//
// CGB_STREAM_PF: the warp prefetches the next batch's lines of every input
// (lane l < 2 U takes line l & 1 of chunk u = l / 2) into L2 (1, default)
// or L1 (2) before waiting on this batch; 0 = off.  Measured per iteration
// (profiles/r02/ab_stream_prefetch.txt): deconv2d -1.1 %, deconv1d -1.7 %,
// sparse lasso -2.3 %, L1 and L2 alike; trajectories bitwise unchanged.
#ifndef CGB_STREAM_PF
#define CGB_STREAM_PF 1
#endif
template <int NIN, class F>
__device__ __forceinline__ void bulk_stream(int64_t n, const double* const (&src)[NIN], F& f) {
  const int64_t S = gsize();
  int b = 0;
  for (int64_t base = gtid(); base < n; base += CGB_U * S, ++b) {
    const bool full = base + (CGB_U - 1) * S < n;
    if (CGB_STREAM_PF) {
      const int lane = threadIdx.x & 31;
      const int64_t ip = base - lane + CGB_U * S + (lane >> 1) * S + 16 * (lane & 1);
      if (lane < 2 * CGB_U && ip < n) {
#pragma unroll
        for (int a = 0; a < NIN; ++a) {
          if (CGB_STREAM_PF == 1) asm volatile("prefetch.global.L2 [%0];" ::"l"(src[a] + ip));
          else asm volatile("prefetch.global.L1 [%0];" ::"l"(src[a] + ip));
        }
      }
    }
    double v[CGB_U][NIN];
#pragma unroll
    for (int u = 0; u < CGB_U; ++u) {
      const int64_t i = base + u * S;
      const int64_t ic = full || i < n ? i : n - 1;
#pragma unroll
      for (int a = 0; a < NIN; ++a) v[u][a] = src[a][ic];
    }
#pragma unroll
    for (int u = 0; u < CGB_U; ++u) {
      const int64_t i = base + u * S;
      if (full || i < n) f.compute(i, v[u], (int64_t)(b * CGB_U + u) * blockDim.x + threadIdx.x);
    }
  }
}

// doubles of per-CTA stash a bulk_stream pass over `len` elements can fill
__device__ __forceinline__ int64_t stream_span(int64_t len) {
  const int64_t S = gsize();
  return (len + CGB_U * S - 1) / (CGB_U * S) * CGB_U * blockDim.x;
}

// ---------------------------------------------------------------------------
// operator-plan executor
// ---------------------------------------------------------------------------
// Input accessor: a[i] or a[i] + beta * b[i] (the CG direction update
// p <- r + beta p fused into the operator read, cg.py:116).
struct InVec {
  const double* a;
  const double* b;
  double beta;
  __device__ __forceinline__ double operator()(int64_t i) const {
    double x = a[i];
    if (b) x = x + beta * b[i];
    return x;
  }
  __device__ __forceinline__ InVec shift(int64_t off) const {
    return InVec{a + off, b ? b + off : nullptr, beta};
  }
};

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// taps of a 1-d conv leaf as a correlation kernel (reversed for conv) are
// prepared by the host, zero padded to a multiple of CGB_RC
__device__ __forceinline__ int conv_ntaps(int64_t k) {
  return (int)((k + CGB_RC - 1) / CGB_RC) * CGB_RC;
}
// staged window length of an R == CGB_RC tile: 32*RC outputs + taps
__device__ __forceinline__ int conv_span(int64_t k) { return 32 * CGB_RC + conv_ntaps(k); }

// Register-blocked valid correlation over a staged window: lane l computes
// the CGB_RC consecutive outputs o0 = l*RC .. o0+RC-1,
//   y[r] = sum_j cc[j] xs[o0 + r + j],
// with a sliding register window -- one shared load of the window and one
// (broadcast) tap load per RC FMAs -- then transposes the results to the
// lane-strided tile layout through `os` and accumulates alpha * y.
__device__ __forceinline__ void conv_accum(int64_t k, const double* xs, const double* cc,
                                           double (&y)[CGB_RC], int lane) {
  const int ngroups = (int)((k + CGB_RC - 1) / CGB_RC);
  const int o0 = lane * CGB_RC;
  double w[CGB_RC];
#pragma unroll
  for (int r = 0; r < CGB_RC; ++r) w[r] = xs[o0 + r];
  for (int g = 0; g < ngroups; ++g) {
    const double* xg = xs + o0 + g * CGB_RC + CGB_RC;
    const double* cg = cc + g * CGB_RC;
#pragma unroll
    for (int jj = 0; jj < CGB_RC; ++jj) {
      const double cj = cg[jj];
#pragma unroll
      for (int r = 0; r < CGB_RC; ++r) y[r] = fma(cj, w[(jj + r) % CGB_RC], y[r]);
      w[jj] = xg[jj];  // slot jj slides from x[o0+gRC+jj] to x[o0+gRC+jj+RC]
    }
  }
}

// lane-consecutive results y (lane l holds outputs l*RC .. l*RC+RC-1) to the
// lane-strided tile layout, accumulated as acc += alpha * y
__device__ __forceinline__ void tile_transpose(const double (&y)[CGB_RC], double* os,
                                               double (&acc)[CGB_RC], double alpha, int nvalid,
                                               int lane) {
  const int o0 = lane * CGB_RC;
  __syncwarp();
#pragma unroll
  for (int r = 0; r < CGB_RC; ++r) os[o0 + r] = y[r];
  __syncwarp();
#pragma unroll
  for (int r = 0; r < CGB_RC; ++r)
    if (lane + 32 * r < nvalid) acc[r] += alpha * os[lane + 32 * r];
  __syncwarp();
}

__device__ __forceinline__ void conv_compute(int64_t k, const double* xs, const double* cc,
                                             double* os, double (&acc)[CGB_RC], double alpha,
                                             int nvalid, int lane) {
  double y[CGB_RC];
#pragma unroll
  for (int r = 0; r < CGB_RC; ++r) y[r] = 0.0;
  conv_accum(k, xs, cc, y, lane);
  tile_transpose(y, os, acc, alpha, nvalid, lane);
}

// Stage xs[0..span) = row[lo + i] (zero outside [0, len)) by hand.
__device__ __forceinline__ void stage_row(const double* row, int64_t lo, int64_t len, int span,
                                          double* xs, int lane) {
  for (int i0 = 0; i0 < span; i0 += 32 * CGB_U) {
    double xv[CGB_U];
#pragma unroll
    for (int u = 0; u < CGB_U; ++u) {
      const int i = i0 + lane + 32 * u;
      const int64_t xi = lo + i;
      const int64_t xc = xi < 0 ? 0 : (xi >= len ? len - 1 : xi);
      const double v = row[xc];
      xv[u] = (i < span && xi >= 0 && xi < len) ? v : 0.0;
    }
#pragma unroll
    for (int u = 0; u < CGB_U; ++u) {
      const int i = i0 + lane + 32 * u;
      if (i < span) xs[i] = xv[u];
    }
  }
}

// 2-d convolution (full, CONV2D) / correlation (valid, CORR2D) tile: the
// tile is a segment of one output row (periodic row block), lane l owns the
// RC consecutive outputs of the segment at l*RC.  Every kernel row a adds a
// 1-d correlation of one input row with that kernel row (reversed for conv,
// taps from the plan) -- conv_accum on a window of the input row.  The kh
// row windows stream through a per-warp ring of CGB_RING2 shared buffers,
// TMA bulk copies for interior windows, hand staging at the image edge.
static __device__ __noinline__ void conv2d_tile(const cgb_leaf& L, int64_t lrow0, int nvalid,
                                         const double* x, double alpha, const double* taps,
                                         double* ring, int xs2, double* os,
                                         double (&acc)[CGB_RC], int lane) {
  const bool conv = L.kind == CGB_LEAF_CONV2D;
  const int64_t H = L.n0, W = L.n1, kh = L.k0, kw = L.k1;
  const int64_t OW = conv ? W + kw - 1 : W;         // output row width
  const int64_t IW = conv ? W : W + kw - 1;         // input row width
  const int64_t IH = conv ? H : H + kh - 1;         // input rows
  const int64_t oi = lrow0 / OW, oj0 = lrow0 - oi * OW;
  const int ntaps = conv_ntaps(kw);
  const int span = 32 * CGB_RC + ntaps;
  const int64_t clo = conv ? oj0 - (kw - 1) : oj0;  // first input column of the window
  const int wib = threadIdx.x >> 5;
  uint64_t* bar = &cgb_mbar[wib][2];
  uint32_t ph = cgb_mbar_phase[wib] >> 2;
  // kernel rows that touch the image, as input rows xi(a) = oi - a / oi + a
  int64_t a_lo = 0, a_hi = kh - 1;
  if (conv) {
    a_lo = oi - (IH - 1) > 0 ? oi - (IH - 1) : 0;
    a_hi = oi < kh - 1 ? oi : kh - 1;
  }
  const int nrows = (int)(a_hi - a_lo + 1);
  const bool tma = clo >= 0 && clo + span <= IW;
  // rank-one kernel K = u v^T (CGB_LEAF_FLAG_SEPARABLE): each row window is
  // folded into column sums t = sum_a u[a] x_a (a lane per 32-strided window
  // position), then ONE row correlation y = v * t -- kh + kw multiply-adds
  // per output instead of kh * kw.  taps = [v row taps | u (kh)].
  const bool sep = (L.reserved & CGB_LEAF_FLAG_SEPARABLE) != 0;
  constexpr int kSepQ = (32 * CGB_RC + CGB_SEP_KMAX + 31) / 32;
  double tcol[kSepQ];
#pragma unroll
  for (int q = 0; q < kSepQ; ++q) tcol[q] = 0.0;
  const int nq = (span + 31) / 32;
  auto issue = [&](int idx) {
    const int64_t a = a_lo + idx;
    const int64_t xi = conv ? oi - a : oi + a;
    const double* src = x + xi * IW + clo;
    const int sh = (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
    const uint32_t bytes = (uint32_t)(((span + sh) * 8 + 15) & ~15);
    issue_bulk(ring + (idx % CGB_RING2) * xs2, src - sh, bytes, &bar[idx % CGB_RING2], lane);
  };
  if (tma)
    for (int i = 0; i < CGB_RING2 && i < nrows; ++i) issue(i);
  double y[CGB_RC];
#pragma unroll
  for (int r = 0; r < CGB_RC; ++r) y[r] = 0.0;
  for (int i = 0; i < nrows; ++i) {
    const int64_t a = a_lo + i;
    const int64_t xi = conv ? oi - a : oi + a;
    const double* rowp = x + xi * IW;
    double* xs = ring + (i % CGB_RING2) * xs2;
    int sh = 0;
    if (tma) {
      const int b = i % CGB_RING2;
      mbar_wait(&bar[b], (ph >> b) & 1u);
      ph ^= 1u << b;
      sh = (int)((reinterpret_cast<uintptr_t>(rowp + clo) >> 3) & 1);
    } else {
      __syncwarp();
      stage_row(rowp, clo, IW, span, xs, lane);
    }
    __syncwarp();
    if (sep) {
      const double ua = taps[ntaps + a];
#pragma unroll
      for (int q = 0; q < kSepQ; ++q) {
        const int ix = lane + 32 * q;
        if (q < nq && ix < span) tcol[q] = fma(ua, xs[sh + ix], tcol[q]);
      }
    } else {
      conv_accum(kw, xs + sh, taps + a * ntaps, y, lane);
    }
    if (tma && i + CGB_RING2 < nrows) issue(i + CGB_RING2);
  }
  if (lane == 0) cgb_mbar_phase[wib] = (cgb_mbar_phase[wib] & 3u) | (ph << 2);
  __syncwarp();
  if (sep) {
    // every ring copy of this tile has been waited for: slot 0 holds t
    double* ts = ring;
#pragma unroll
    for (int q = 0; q < kSepQ; ++q) {
      const int ix = lane + 32 * q;
      if (q < nq && ix < span) ts[ix] = tcol[q];
    }
    __syncwarp();
    conv_accum(kw, ts, taps, y, lane);
    __syncwarp();
  }
  tile_transpose(y, os, acc, alpha, nvalid, lane);
}

// Dense rows of a tile: a warp per row, CGB_DENSE_DR rows at a time so
// their loads are in flight together (one latency per row group instead of
// per row).  Two copies: dense_rows (inlined) and dense_tile (out of line,
// its own register allocation).  Inlined into the persistent solver kernel
// the loop ran at a third of its stand-alone bandwidth (2.0 vs 6.0 TB/s on
// configs[4]'s 2e5 x 2e3 operator); the host launches the MODE 2
// instantiation -- which calls dense_tile -- for plans with dense leaves,
// and the others keep the inline copy (the call site cost the convolution
// plans ~8 % when always present).
// Row-chunk prefetch of dense_tile.  ptxas schedules each load of the
// out-of-line callee next to its FMA (~5-8 loads in flight per lane: its
// register budget; loading a whole chunk first did not change that), so a
// GEMV streaming from HBM is latency-exposed.  The warp prefetches the row
// chunks CGB_DENSE_PF chunks ahead into L1 (no registers needed: lane l
// takes line l % 8 of rows l / 8 and l / 8 + 4 of the 8 x 1 KB chunk) and
// the loads hit L1: configs[4] 4-7 % faster per iteration at distance 2,
// slower at 4.  Same loads, same FMA order as dense_rows (bitwise identical
// trajectories).
#ifndef CGB_DENSE_PF
#define CGB_DENSE_PF 2
#endif
#ifndef CGB_DENSE_PF_MIN
#define CGB_DENSE_PF_MIN (int64_t(1) << 22)  // entries (32 MB of values)
#endif
__device__ __forceinline__ void dense_prefetch(const double* base, int64_t ld, int nrows,
                                               int64_t cchunk, int64_t cols, int lane) {
  const int64_t c = cchunk + 16 * (lane & 7);
  if (c >= cols) return;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int q = (lane >> 3) + 4 * h;
    if (q < nrows) asm volatile("prefetch.global.L1 [%0];" ::"l"(base + q * ld + c));
  }
}

static __device__ __noinline__ void dense_tile(const cgb_leaf& L, int64_t lrow0, int nvalid,
                                               InVec in, double alpha, double (&acc)[CGB_RC],
                                               int lane) {
  constexpr int CGB_DR = CGB_DENSE_DR;
  constexpr int CGB_DU = CGB_DENSE_UNROLL;
  constexpr int64_t CH = 32 * CGB_DU;  // columns per chunk
  double mine[CGB_RC];
#pragma unroll
  for (int r = 0; r < CGB_RC; ++r) mine[r] = 0.0;
  const int64_t cols = L.cols;
  // matrices far larger than L2 stream from HBM: prefetch; small ones are
  // L2-resident and the prefetch only adds issue slots (configs[0]: 25 %
  // slower with it)
  const bool stream = L.rows * cols >= CGB_DENSE_PF_MIN;
  for (int rr0 = 0; rr0 < nvalid; rr0 += CGB_DR) {
    double sacc[CGB_DR];
    const double* rowp[CGB_DR];
#pragma unroll
    for (int q = 0; q < CGB_DR; ++q) {
      sacc[q] = 0.0;
      const int rr = rr0 + q < nvalid ? rr0 + q : nvalid - 1;  // clamped
      rowp[q] = L.val + (lrow0 + rr) * L.ld;
    }
    if (stream) {
      const double* base = L.val + (lrow0 + rr0) * L.ld;
      const int nr = nvalid - rr0 < CGB_DR ? nvalid - rr0 : CGB_DR;
#pragma unroll
      for (int k = 0; k < CGB_DENSE_PF; ++k) dense_prefetch(base, L.ld, nr, k * CH, cols, lane);
      for (int64_t c0 = 0; c0 < cols; c0 += CH) {
        dense_prefetch(base, L.ld, nr, c0 + CGB_DENSE_PF * CH, cols, lane);
#pragma unroll
        for (int u = 0; u < CGB_DU; ++u) {
          const int64_t c = c0 + 32 * u + lane;
          if (c < cols) {
            const double xv = in(c);
#pragma unroll
            for (int q = 0; q < CGB_DR; ++q) sacc[q] += __ldg(rowp[q] + c) * xv;
          }
        }
      }
    } else {
#pragma unroll CGB_DU
      for (int64_t c = lane; c < cols; c += 32) {
        const double xv = in(c);
#pragma unroll
        for (int q = 0; q < CGB_DR; ++q) sacc[q] += __ldg(rowp[q] + c) * xv;
      }
    }
#pragma unroll
    for (int q = 0; q < CGB_DR; ++q) {
      const double sq = warp_sum(sacc[q]);
      const int rr = rr0 + q;
      if (rr < nvalid && lane == (rr & 31)) {
#pragma unroll
        for (int r = 0; r < CGB_RC; ++r)
          if (r == (rr >> 5)) mine[r] = sq;
      }
    }
  }
#pragma unroll
  for (int r = 0; r < CGB_RC; ++r) acc[r] += alpha * mine[r];
}

__device__ __forceinline__ void dense_rows(const cgb_leaf& L, int64_t lrow0, int nvalid,
                                               const InVec& in, double alpha, double (&acc)[CGB_RC],
                                               int lane) {
  constexpr int CGB_DR = CGB_DENSE_DR;
  constexpr int CGB_DU = CGB_DENSE_UNROLL;
  double mine[CGB_RC];
#pragma unroll
  for (int r = 0; r < CGB_RC; ++r) mine[r] = 0.0;
  const int64_t cols = L.cols;
  for (int rr0 = 0; rr0 < nvalid; rr0 += CGB_DR) {
    double sacc[CGB_DR];
    const double* rowp[CGB_DR];
#pragma unroll
    for (int q = 0; q < CGB_DR; ++q) {
      sacc[q] = 0.0;
      const int rr = rr0 + q < nvalid ? rr0 + q : nvalid - 1;  // clamped
      rowp[q] = L.val + (lrow0 + rr) * L.ld;
    }
#pragma unroll CGB_DU
    for (int64_t c = lane; c < cols; c += 32) {
      const double xv = in(c);
#pragma unroll
      for (int q = 0; q < CGB_DR; ++q) sacc[q] += __ldg(rowp[q] + c) * xv;
    }
#pragma unroll
    for (int q = 0; q < CGB_DR; ++q) {
      const double sq = warp_sum(sacc[q]);
      const int rr = rr0 + q;
      if (rr < nvalid && lane == (rr & 31)) {
#pragma unroll
        for (int r = 0; r < CGB_RC; ++r)
          if (r == (rr >> 5)) mine[r] = sq;
      }
    }
  }
#pragma unroll
  for (int r = 0; r < CGB_RC; ++r) acc[r] += alpha * mine[r];
}

// Contribution of one leaf to a warp tile.  The tile holds 32*R rows
// starting at leaf-local row lrow0; lane l owns rows lrow0 + l + 32 r
// (r < R), so epilogue stores are coalesced.  acc[r] accumulates.
// Warp-collective: every lane of the warp must call it.
//
// 1-d convolution / correlation leaves in R == CGB_RC tiles run the
// register-blocked path (conv_compute) on a window staged in shared memory:
// by TMA in run_level for interior tiles, by hand (zero-filled edges) here.
template <int MODE>
__device__ __forceinline__ void leaf_tile(const cgb_leaf& L, int64_t lrow0, int nvalid, int R,
                                          const InVec& in, double alpha,
                                          double (&acc)[CGB_RC], int lane, const double* cc,
                                          double* xs, double* os, double* ring, int xs2) {
  switch (L.kind) {
    case CGB_LEAF_IDENTITY: {
      double v[CGB_RC];
#pragma unroll
      for (int r = 0; r < CGB_RC; ++r) {  // clamped: every load in flight at once
        const int rr = lane + 32 * r;
        v[r] = in(lrow0 + (r < R && rr < nvalid ? rr : 0));
      }
#pragma unroll
      for (int r = 0; r < CGB_RC; ++r)
        if (r < R && lane + 32 * r < nvalid) acc[r] += alpha * v[r];
    } break;
    case CGB_LEAF_DENSE:
      if (MODE == 2) {
        dense_tile(L, lrow0, nvalid, in, alpha, acc, lane);
      } else {
        dense_rows(L, lrow0, nvalid, in, alpha, acc, lane);
      }
      break;
    case CGB_LEAF_CSR: {
#pragma unroll
      for (int r = 0; r < CGB_RC; ++r) {
        if (r < R && lane + 32 * r < nvalid) {
          const int64_t lrow = lrow0 + lane + 32 * r;
          double s = 0.0;
          const int64_t e0 = __ldg(L.rowptr + lrow), e1 = __ldg(L.rowptr + lrow + 1);
          int64_t e = e0;
          // batches of 8 nonzeros: all index / value loads, then all gathers
          for (; e + 8 <= e1; e += 8) {
            int32_t ci[8];
            double vv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              ci[q] = __ldg(L.colidx + e + q);
              vv[q] = __ldg(L.val + e + q);
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) s += vv[q] * in(ci[q]);
          }
          for (; e < e1; ++e) s += __ldg(L.val + e) * in(__ldg(L.colidx + e));
          acc[r] += alpha * s;
        }
      }
    } break;
    case CGB_LEAF_CONV1D:
    case CGB_LEAF_CORR1D: {
      const bool conv = L.kind == CGB_LEAF_CONV1D;
      const int64_t k = L.k0;
      if (R == CGB_RC && cc) {
        // edge tile (window leaves [0, cols)): stage by hand with zero fill
        const int64_t xlo = conv ? lrow0 - (k - 1) : lrow0;
        const int span = conv_span(k);
        __syncwarp();
        for (int i0 = 0; i0 < span; i0 += 32 * CGB_U) {
          double xv[CGB_U];
#pragma unroll
          for (int u = 0; u < CGB_U; ++u) {  // clamped loads: no branches
            const int i = i0 + lane + 32 * u;
            const int64_t xi = xlo + i;
            const int64_t xc = xi < 0 ? 0 : (xi >= L.cols ? L.cols - 1 : xi);
            const double v = in(xc);
            xv[u] = (i < span && xi >= 0 && xi < L.cols) ? v : 0.0;
          }
#pragma unroll
          for (int u = 0; u < CGB_U; ++u) {
            const int i = i0 + lane + 32 * u;
            if (i < span) xs[i] = xv[u];
          }
        }
        __syncwarp();
        conv_compute(k, xs, cc, os, acc, alpha, nvalid, lane);
      } else {
#pragma unroll
        for (int r = 0; r < CGB_RC; ++r) {
          if (r < R && lane + 32 * r < nvalid) {
            const int64_t lrow = lrow0 + lane + 32 * r;
            double s = 0.0;
            if (conv) {  // y[i] = sum_j c[j] x[i-j]  (np.convolve, linop.py:46)
              const int64_t n = L.n0;
              const int64_t jlo = lrow - (n - 1) > 0 ? lrow - (n - 1) : 0;
              const int64_t jhi = lrow < k - 1 ? lrow : k - 1;
              for (int64_t j = jlo; j <= jhi; ++j) s += __ldg(L.val + j) * in(lrow - j);
            } else {     // y[i] = sum_j c[j] x[i+j]  (np.correlate valid, linop.py:61)
              for (int64_t j = 0; j < k; ++j) s += __ldg(L.val + j) * in(lrow + j);
            }
            acc[r] += alpha * s;
          }
        }
      }
    } break;
    case CGB_LEAF_CONV2D:
    case CGB_LEAF_CORR2D: {
      // the tiled 2-d path (a call) exists only in the MODE 1 kernels, which
      // the host launches for plans with a 2-d leaf: it cost every other
      // plan ~10 % (register allocation around the call) when always present
      if (MODE == 1 && R == CGB_RC && cc && ring) {
        conv2d_tile(L, lrow0, nvalid, in.a, alpha, cc, ring, xs2, os, acc, lane);
        break;
      }
#pragma unroll
      for (int r = 0; r < CGB_RC; ++r) {
        if (r < R && lane + 32 * r < nvalid) {
          const int64_t lrow = lrow0 + lane + 32 * r;
          const int64_t H = L.n0, W = L.n1, kh = L.k0, kw = L.k1;
          const int64_t OW = W + kw - 1;
          double s = 0.0;
          if (L.kind == CGB_LEAF_CONV2D) {  // full 2-d convolution of an H x W image
            const int64_t oi = lrow / OW, oj = lrow - oi * OW;
            const int64_t alo = oi - (H - 1) > 0 ? oi - (H - 1) : 0;
            const int64_t ahi = oi < kh - 1 ? oi : kh - 1;
            const int64_t blo = oj - (W - 1) > 0 ? oj - (W - 1) : 0;
            const int64_t bhi = oj < kw - 1 ? oj : kw - 1;
            for (int64_t a = alo; a <= ahi; ++a) {
              const int64_t xrow = (oi - a) * W;
              for (int64_t bb = blo; bb <= bhi; ++bb)
                s += __ldg(L.val + a * kw + bb) * in(xrow + oj - bb);
            }
          } else {                           // valid 2-d correlation -> H x W image
            const int64_t i = lrow / W, j = lrow - i * W;
            for (int64_t a = 0; a < kh; ++a) {
              const int64_t yrow = (i + a) * OW + j;
              for (int64_t bb = 0; bb < kw; ++bb) s += __ldg(L.val + a * kw + bb) * in(yrow + bb);
            }
          }
          acc[r] += alpha * s;
        }
      }
    } break;
    default:
      break;
  }
}

// Window of a tile's TMA-staged conv term: the bulk copy reads `bytes` from
// the 16-byte aligned `src`; the window starts `shift` doubles into the
// shared buffer.  ok == false: no conv term, a fused (two-vector) input, or a
// window reaching outside the input (edge tile) -- staged by hand instead.
struct ConvWin {
  const double* src;
  uint32_t bytes;
  int shift;
  bool ok;
};

__device__ __forceinline__ ConvWin conv_window(const DevPlan& P, const DevRowBlock& rb,
                                               int64_t row0, const InVec& in,
                                               const double* temp) {
  ConvWin w{nullptr, 0u, 0, false};
  if (rb.conv_term < 0) return w;
  const cgb_term tm = P.terms[rb.conv_term];
  const cgb_leaf L = P.leaves[tm.leaf];
  const double* base;
  if (tm.in_buf == 0) {
    if (in.b) return w;
    base = in.a + tm.in_off;
  } else {
    base = temp + P.temp_off[tm.in_buf - 1] + tm.in_off;
  }
  const int64_t k = L.k0;
  const int64_t lrow0 = row0 - tm.row_origin;
  const int64_t xlo = L.kind == CGB_LEAF_CONV1D ? lrow0 - (k - 1) : lrow0;
  const int span = conv_span(k);
  if (xlo < 0 || xlo + span > L.cols) return w;
  const double* a = base + xlo;
  w.shift = (int)((reinterpret_cast<uintptr_t>(a) >> 3) & 1);
  w.src = a - w.shift;
  w.bytes = (uint32_t)(((span + w.shift) * 8 + 15) & ~15);
  w.ok = true;
  return w;
}

__device__ __forceinline__ int find_rowblock(const DevPlan& P, int lo, int hi, int64_t tile) {
  hi -= 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (P.rbs[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// lane 0 issues the bulk copy of a window into `dst` (after the warp's
// generic-proxy reads of that buffer are fenced off)
__device__ __forceinline__ void issue_window(const ConvWin& w, double* dst, uint64_t* bar,
                                             int lane) {
  __syncwarp();
  if (lane == 0) {
    fence_proxy_async();
    bulk_load(dst, w.src, w.bytes, bar);
  }
}

// bulk copy only (the caller has announced the bytes on the mbarrier)
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n .reg .b64 st;\n"
      " mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

template <int MODE>
__device__ __forceinline__ void leaf_tile(const cgb_leaf& L, int64_t lrow0, int nvalid, int R,
                                          const InVec& in, double alpha,
                                          double (&acc)[CGB_RC], int lane, const double* cc,
                                          double* xs, double* os, double* ring, int xs2);

// L2 prefetch of the 128-byte lines of p[j0, j0 + n) (one line per lane)
__device__ __forceinline__ void prefetch_range(const double* p, int64_t j0, int n, int lane) {
  if (!p || n <= 0) return;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(p + j0) & ~uintptr_t(127);
  const uintptr_t a1 = reinterpret_cast<uintptr_t>(p + j0 + n - 1);
  for (uintptr_t a = a0 + 128 * (uintptr_t)lane; a <= a1; a += 32 * 128)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
}
// epilogues may declare prefetch(j0, n, lane) for the operands they read
template <class E>
__device__ __forceinline__ auto epi_prefetch(const E& e, int64_t j0, int n, int lane, int)
    -> decltype(e.prefetch(j0, n, lane), void()) {
  e.prefetch(j0, n, lane);
}
template <class E>
__device__ __forceinline__ void epi_prefetch(const E&, int64_t, int, int, long) {}

// One output row segment of a strip: y = the conv of kernel rows
// [a_lo, a_hi] with the ring's input rows (slot = input row mod NS); xrow0
// != null: the rows came by TMA from x + row * IW (+ the copy's alignment
// shift), else they were staged at the slot start.  Out of line: it holds
// the column sums of the separable path in registers.
static __device__ __noinline__ void strip_row(const cgb_leaf& L, int64_t oi, int64_t a_lo,
                                              int64_t a_hi, const double* xrow0, int64_t IW,
                                              const double* ring, int SLOT, int NS,
                                              const double* taps, double* tb,
                                              double (&yout)[CGB_RC], int lane) {
  const bool conv = L.kind == CGB_LEAF_CONV2D;
  const bool sep = (L.reserved & CGB_LEAF_FLAG_SEPARABLE) != 0;
  const int64_t kw = L.k1;
  const int ntaps = conv_ntaps(kw);
  const int span = 32 * CGB_RC + ntaps;
  double y[CGB_RC];  // registers (yout, by reference across the call, lives in memory)
#pragma unroll
  for (int r = 0; r < CGB_RC; ++r) y[r] = 0.0;
  constexpr int kQ = (32 * CGB_RC + CGB_SEP_KMAX + 31) / 32;
  double tcol[kQ];
#pragma unroll
  for (int q = 0; q < kQ; ++q) tcol[q] = 0.0;
  const int nq = (span + 31) / 32;
  for (int64_t a = a_lo; a <= a_hi; ++a) {
    const int64_t xi = conv ? oi - a : oi + a;
    const int sh = xrow0 ? (int)((reinterpret_cast<uintptr_t>(xrow0 + xi * IW) >> 3) & 1) : 0;
    const double* xs = ring + (size_t)(xi % NS) * SLOT + sh;
    if (sep) {
      const double ua = taps[ntaps + a];
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        const int ix = lane + 32 * q;
        if (q < nq && ix < span) tcol[q] = fma(ua, xs[ix], tcol[q]);
      }
    } else {
      conv_accum(kw, xs, taps + a * ntaps, y, lane);
    }
  }
  if (sep) {
    __syncwarp();
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const int ix = lane + 32 * q;
      if (q < nq && ix < span) tb[ix] = tcol[q];
    }
    __syncwarp();
    conv_accum(kw, tb, taps, y, lane);
  }
#pragma unroll
  for (int r = 0; r < CGB_RC; ++r) yout[r] = y[r];
}

// Separable strips, column pass of one step: t_j[c] = sum_a w[a] X(base0 + j + a)
// for the CTA's CGB_WARPS output rows j, every thread a window column c,
// with a sliding register window over the rows (one shared load per kh
// multiply-adds per column and output row, conv_accum's scheme turned
// vertical).  X(i) = input row base0 + i of the ring (zero outside
// [0, IH)); w = u (corr) or u reversed (full conv); t_j goes to warp j's
// buffer tbase + j * tstride.
static __device__ __noinline__ void strip_colpass(const cgb_leaf& L, int64_t base0, int64_t IH,
                                                  int span, const double* ring, int SLOT, int NS,
                                                  int sh0, int shodd, const double* u,
                                                  double* tbase, int tstride) {
  const bool conv = L.kind == CGB_LEAF_CONV2D;
  const int kh = (int)L.k0;
  const int s0 = (int)(((base0 % NS) + NS) % NS);
  // shared-memory offset of every row the step reads (kh + 7 of them, at
  // most CGB_SEP_KMAX + 7), -1 for rows outside the image: computed once,
  // so the column loop's loads are one add + one shared load each
  constexpr int RPS = CGB_STRIP_RPS;
  constexpr int kMaxRows = 64 + RPS;
  __shared__ int32_t roff_s[kMaxRows];
  for (int i = threadIdx.x; i < kh + RPS; i += blockDim.x) {
    const int64_t r = base0 + i;
    const int slot = s0 + i >= NS ? s0 + i - NS : s0 + i;
    const int sh = (sh0 + (shodd & (int)(r & 1))) & 1;
    roff_s[i] = (r >= 0 && r < IH) ? slot * SLOT + sh : -1;
  }
  __syncthreads();
  const double* sring = ring;
  auto X = [&](int i, int c) -> double {
    const int o = roff_s[i];
    const double v = sring[(o < 0 ? 0 : o) + c];
    return o < 0 ? 0.0 : v;
  };
  // a thread owns column c and, when the window is wider than the CTA,
  // column c + blockDim.x too: both run interleaved in one loop (two
  // independent FMA chains per row hide the shared-load latency) instead of
  // one after the other, which doubled the step time of the first warps
  const int c0 = threadIdx.x, c1 = threadIdx.x + blockDim.x;
  const bool two = c1 < span;
  if (c0 >= span) return;
  const int c1s = two ? c1 : c0;
  double acc0[RPS], xw0[RPS], acc1[RPS], xw1[RPS];
#pragma unroll
  for (int j = 0; j < RPS; ++j) {
    acc0[j] = acc1[j] = 0.0;
    xw0[j] = X(j, c0);
    xw1[j] = X(j, c1s);
  }
  for (int g = 0; g < (kh + RPS - 1) / RPS; ++g) {
#pragma unroll
    for (int jj = 0; jj < RPS; ++jj) {
      const int a = RPS * g + jj;
      if (a < kh) {
        const double wa = u[conv ? kh - 1 - a : a];
#pragma unroll
        for (int j = 0; j < RPS; ++j) {
          acc0[j] = fma(wa, xw0[(jj + j) % RPS], acc0[j]);
          acc1[j] = fma(wa, xw1[(jj + j) % RPS], acc1[j]);
        }
        if (a + 1 < kh) {                       // slot jj: row a -> row a + RPS
          xw0[jj] = X(a + RPS, c0);
          xw1[jj] = X(a + RPS, c1s);
        }
      }
    }
  }
  // output row j of the step: warp j % 8's buffer j / 8
#pragma unroll
  for (int j = 0; j < RPS; ++j) {
    double* tj = tbase + (size_t)(j % CGB_WARPS) * tstride + (size_t)(j / CGB_WARPS) * SLOT;
    tj[c0] = acc0[j];
    if (two) tj[c1] = acc1[j];
  }
}

// the row pass of a separable strip row: y = v * t (register-blocked)
static __device__ __forceinline__ void strip_rowpass(int64_t kw, const double* t, const double* taps,
                                                  double (&yout)[CGB_RC], int lane) {
  double y[CGB_RC];
#pragma unroll
  for (int r = 0; r < CGB_RC; ++r) y[r] = 0.0;
  conv_accum(kw, t, taps, y, lane);
#pragma unroll
  for (int r = 0; r < CGB_RC; ++r) yout[r] = y[r];
}

// 2-d convolution row blocks as CTA strips.  A task is one 288-column
// segment of a run of P.strip_rows consecutive output rows; the CTA's 8
// warps compute 8 output rows per step (warp w: row 8 s + w) from a ring of
// input rows in shared memory that every warp reads, so each input row of
// the segment is brought in ONCE per task (the per-warp tile path re-reads
// it kh times).  Rows arrive by TMA bulk copies in batches, one batch per
// step, issued two steps ahead by thread 0 onto the two CTA mbarriers;
// segments reaching past the image edge are staged by hand with zero fill.
// Every other term of the block (identity, sparse, dense) and the epilogue
// run per warp on its output row segment, exactly as in run_level.
// Returns false (nothing done) when the apply input is a fused two-vector
// accessor, which the strips do not stage.
template <int MODE, class Epi>
__device__ bool run_strips(const DevPlan& P, int e, const InVec& in, int ts, Epi& epi,
                           double* part) {
  extern __shared__ __align__(16) double cgb_dyn_smem[];
  if (MODE != 1 || P.strip_rows == 0) return false;
  if (in.b) return false;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int rb_lo = P.level_rb[e], rb_hi = P.level_rb[e + 1];
  const double* temp = P.temp[ts];
  const int SLOT = P.strip_slot, NS = P.strip_nslot;
  double* ring = cgb_dyn_smem;
  // per warp: transpose buffer | two t buffers (separable strips alternate
  // them, so a step needs only the barrier after its column pass)
  // (one t buffer per row of the warp; a second one alternating by step
  // when a warp has one row -- not needed for correctness: the column
  // pass's own barrier orders the writes after every row pass)
  constexpr int TB = CGB_STRIP_RPW == 1 ? 2 : CGB_STRIP_RPW;
  const int WSTRIDE = TB * SLOT + 32 * CGB_RC + 2;
  double* os = ring + (size_t)NS * SLOT + (size_t)wib * WSTRIDE;
  const unsigned issuer = blockDim.x - 32;  // lane 0 of the last warp (one column)
  bool any = false;
  // timeline probe (profiling only): thread 0 of block 0 adds ns to
  // cgb_tl_acc[8..15]: 8 batch wait, 9 column pass, 10 its barrier, 11 row
  // pass + other terms + epilogue, 12 step barrier, 13 steps, 14 tasks
  double* tl = (blockIdx.x == 0 && threadIdx.x == 0) ? cgb_tl_acc : nullptr;
  uint64_t tl1 = tl ? globaltimer() : 0;
#define CGB_TL(slot)                                      \
  if (tl) {                                                \
    const uint64_t tl_x = globaltimer();                   \
    tl[slot] += (double)(tl_x - tl1);                      \
    tl1 = tl_x;                                            \
  }
  for (int rbi = rb_lo; rbi < rb_hi; ++rbi) {
    const DevRowBlock rb = P.rbs[rbi];
    if (rb.strip_term < 0) continue;
    any = true;
    const cgb_term tm = P.terms[rb.strip_term];
    const cgb_leaf L = P.leaves[tm.leaf];
    const bool conv = L.kind == CGB_LEAF_CONV2D;
    const bool sep = (L.reserved & CGB_LEAF_FLAG_SEPARABLE) != 0;
    const int64_t kh = L.k0, kw = L.k1;
    const int64_t OW = conv ? L.n1 + kw - 1 : L.n1;
    const int64_t IW = conv ? L.n1 : L.n1 + kw - 1;
    const int64_t IH = conv ? L.n0 : L.n0 + kh - 1;
    const int ntaps = conv_ntaps(kw);
    const int span = 32 * CGB_RC + ntaps;
    const double* taps = P.taps + P.leaf_taps[tm.leaf];
    const double* x = tm.in_buf == 0 ? in.a + tm.in_off
                                     : temp + P.temp_off[tm.in_buf - 1] + tm.in_off;
    const int64_t oi_first = (rb.row_begin - tm.row_origin) / OW;
    const int64_t prows = (rb.row_end - rb.row_begin) / OW;
    const int64_t chunk = P.strip_rows;
    const int64_t ntask = (prows + chunk - 1) / chunk * rb.tpr;
    for (int64_t task = blockIdx.x; task < ntask; task += gridDim.x) {
      const int64_t ch = task / rb.tpr, pc = task - ch * rb.tpr;
      const int64_t p0 = ch * chunk, p1 = p0 + chunk < prows ? p0 + chunk : prows;
      const int64_t oj0 = pc * (32 * CGB_RC);
      const int nvalid = (int)(OW - oj0 < 32 * CGB_RC ? OW - oj0 : 32 * CGB_RC);
      const int64_t clo = conv ? oj0 - (kw - 1) : oj0;
      const bool tma = clo >= 0 && clo + span <= IW;
      constexpr int RPS = CGB_STRIP_RPS, RPW = CGB_STRIP_RPW;
      const int nsteps = (int)((p1 - p0 + RPS - 1) / RPS);
      // input rows first needed at step s, clipped to the image and to the
      // rows this task's outputs reach
      const int64_t row_hi = oi_first + p1 - 1 + (conv ? 0 : kh - 1) + 1;
      auto batch = [&](int st, int64_t& r0, int64_t& r1) {
        const int64_t lo = oi_first + p0 + (int64_t)RPS * st - (conv ? kh - 1 : 0);
        r0 = st == 0 ? lo : lo + kh - 1;
        r1 = lo + kh - 1 + RPS;
        if (r0 < 0) r0 = 0;
        if (r1 > IH) r1 = IH;
        if (r1 > row_hi) r1 = row_hi;
      };
      auto row_src = [&](int64_t r, int& sh) {
        const double* a = x + r * IW + clo;
        sh = (int)((reinterpret_cast<uintptr_t>(a) >> 3) & 1);
        return a - sh;
      };
      __syncthreads();                 // the previous task's rows are consumed
      const uint32_t base = cgb_strip_seq;
      __syncthreads();
      auto issue = [&](int st) {       // thread 0: batch st onto mbarrier (base + st) & 1
        int64_t r0, r1;
        batch(st, r0, r1);
        uint32_t total = 0;
        for (int64_t r = r0; r < r1; ++r) {
          int sh;
          row_src(r, sh);
          total += (uint32_t)(((span + sh) * 8 + 15) & ~15);
        }
        uint64_t* bar = &cgb_strip_mbar[(base + st) & 1u];
        fence_proxy_async();
        mbar_arrive_tx(bar, total);
        for (int64_t r = r0; r < r1; ++r) {
          int sh;
          const double* src = row_src(r, sh);
          bulk_copy(ring + (size_t)(r % NS) * SLOT, src, (uint32_t)(((span + sh) * 8 + 15) & ~15),
                    bar);
        }
        cgb_strip_seq = base + st + 1;
      };
      if (tma && threadIdx.x == issuer) {
        issue(0);
        if (nsteps > 1) issue(1);
      }
      if (tl) tl[14] += 1.0;
      CGB_TL(12)
      for (int st = 0; st < nsteps; ++st) {
        if (tl) tl[13] += 1.0;
        for (int k = 0; k < RPW; ++k) {  // L2 prefetch: this warp's NEXT step rows
          const int64_t pn = p0 + (int64_t)RPS * (st + 1) + wib + CGB_WARPS * k;
          if (pn < p1) {
            const int64_t rn = rb.row_begin + pn * OW + oj0;
            epi_prefetch(epi, rn, nvalid, lane, 0);
            for (int t = rb.term_begin; t < rb.term_end; ++t) {
              const cgb_term tt = P.terms[t];
              if (t == rb.strip_term || P.leaves[tt.leaf].kind != CGB_LEAF_IDENTITY) continue;
              const double* src = tt.in_buf == 0 ? in.a + tt.in_off
                                                 : temp + P.temp_off[tt.in_buf - 1] + tt.in_off;
              prefetch_range(src, rn - tt.row_origin, nvalid, lane);
            }
          }
        }
        if (tma) {
          const uint32_t g = base + st;
          mbar_wait(&cgb_strip_mbar[g & 1u], (g >> 1) & 1u);
        } else {
          int64_t r0, r1;
          batch(st, r0, r1);
          for (int64_t r = r0 + wib; r < r1; r += CGB_WARPS)
            stage_row(x + r * IW, clo, IW, span, ring + (size_t)(r % NS) * SLOT, lane);
          __syncthreads();
        }
        CGB_TL(8)
        if (sep) {
          // all threads: column sums of the step's RPS output rows
          const int64_t o0 = oi_first + p0 + (int64_t)RPS * st;
          const int sh0 = tma ? (int)((reinterpret_cast<uintptr_t>(x + clo) >> 3) & 1) : 0;
          strip_colpass(L, conv ? o0 - (kh - 1) : o0, IH, span, ring, SLOT, NS, sh0,
                        tma ? (int)(IW & 1) : 0, taps + ntaps,
                        ring + (size_t)NS * SLOT + 32 * CGB_RC + 2 +
                            (RPW == 1 ? (st & 1) * SLOT : 0),
                        WSTRIDE);
          CGB_TL(9)
          __syncthreads();
          // the rows only this step read are free: batch st + 2 goes now,
          // under the row passes
          if (tma && threadIdx.x == issuer && st + 2 < nsteps) issue(st + 2);
          CGB_TL(10)
        }
        // this warp's rows of the step: p = p0 + RPS st + wib + 8 k.  The
        // terms ahead of the strip term are summed first for every row (their
        // loads overlap the row passes), then per row: the strip term from
        // its row pass, the remaining terms, the epilogue -- every tile's
        // terms in their order.
        double accs[RPW][CGB_RC];
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
#pragma unroll
          for (int r = 0; r < CGB_RC; ++r) accs[k][r] = 0.0;
          const int64_t p = p0 + (int64_t)RPS * st + wib + CGB_WARPS * k;
          if (p >= p1) continue;
          const int64_t row0 = rb.row_begin + p * OW + oj0;
          for (int t = rb.term_begin; t < rb.strip_term; ++t) {
            const cgb_term tt = P.terms[t];
            const cgb_leaf LL = P.leaves[tt.leaf];
            const InVec tin = tt.in_buf == 0
                                  ? in.shift(tt.in_off)
                                  : InVec{temp + P.temp_off[tt.in_buf - 1] + tt.in_off, nullptr,
                                          0.0};
            leaf_tile<0>(LL, row0 - tt.row_origin, nvalid, CGB_RC, tin, tt.alpha, accs[k], lane,
                         nullptr, nullptr, os, nullptr, 0);
          }
        }
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
          const int64_t p = p0 + (int64_t)RPS * st + wib + CGB_WARPS * k;
          if (p >= p1) continue;
          double* tb = os + 32 * CGB_RC + 2 + (RPW == 1 ? (st & 1) : k) * SLOT;
          const int64_t oi = oi_first + p;
          int64_t a_lo = 0, a_hi = kh - 1;
          if (conv) {
            a_lo = oi - (IH - 1) > 0 ? oi - (IH - 1) : 0;
            a_hi = oi < kh - 1 ? oi : kh - 1;
          }
          const int64_t row0 = rb.row_begin + p * OW + oj0;
          double y[CGB_RC];
          if (sep)
            strip_rowpass(kw, tb, taps, y, lane);
          else
            strip_row(L, oi, a_lo, a_hi, tma ? x + clo : nullptr, IW, ring, SLOT, NS, taps, tb,
                      y, lane);
          for (int t = rb.strip_term; t < rb.term_end; ++t) {
            const cgb_term tt = P.terms[t];
            if (t == rb.strip_term) {
              tile_transpose(y, os, accs[k], tt.alpha, nvalid, lane);
              continue;
            }
            const cgb_leaf LL = P.leaves[tt.leaf];
            const InVec tin = tt.in_buf == 0
                                  ? in.shift(tt.in_off)
                                  : InVec{temp + P.temp_off[tt.in_buf - 1] + tt.in_off, nullptr,
                                          0.0};
            leaf_tile<0>(LL, row0 - tt.row_origin, nvalid, CGB_RC, tin, tt.alpha, accs[k], lane,
                         nullptr, nullptr, os, nullptr, 0);
          }
          if (rb.out_buf == 0) {
            epi.tile(row0 + lane, row0, CGB_RC, nvalid - lane, accs[k], part);
          } else {
            double* dst = P.temp[ts] + P.temp_off[rb.out_buf - 1] + row0 + lane;
#pragma unroll
            for (int r = 0; r < CGB_RC; ++r)
              if (lane + 32 * r < nvalid) dst[32 * r] = accs[k][r];
          }
        }
        CGB_TL(11)
        if (!sep) {
          __syncthreads();             // every warp is done with step st's rows
          if (tma && threadIdx.x == issuer && st + 2 < nsteps) issue(st + 2);
        }
        CGB_TL(12)
      }
    }
  }
  if (any) __syncthreads();            // the ring overlays the per-warp buffers
#undef CGB_TL
  return any;
}

// Execute one level of a plan with temporary set `ts`.  Tiles are dealt
// round-robin across blocks first (tile t -> block t mod G) so every SM
// streams a similar share.  A warp's conv windows are double buffered: the
// TMA copy of its next tile's window is in flight while it computes the
// current one.  The epilogue gets a lane's whole tile at once:
// epi.tile(first_row, tile_row0, R, left, acc, part) with rows first_row + 32 r,
// valid while 32 r < left (see CGB_EPI_VALID) -- so it can issue all its
// loads before its stores.
template <int MODE, class Epi>
__device__ void run_level(const DevPlan& P, int e, const InVec& in, int ts, Epi& epi,
                          double* part) {
  extern __shared__ __align__(16) double cgb_dyn_smem[];
  const bool strips = run_strips<MODE>(P, e, in, ts, epi, part);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* xsb0 = cgb_dyn_smem + (size_t)wib * P.smem_per_warp;
  double* xsb1 = xsb0 + P.smem_xs;
  double* os = xsb1 + P.smem_xs;
  double* ring = P.smem_xs2 > 0 ? os + (32 * CGB_RC + 2) : nullptr;
  uint64_t* bar = cgb_mbar[wib];
  const int64_t G = gridDim.x;
  const int64_t stride = G * CGB_WARPS;
  const int64_t T = P.level_tiles[e];
  const int rb_lo = P.level_rb[e], rb_hi = P.level_rb[e + 1];
  const double* temp = P.temp[ts];
  __syncwarp();
  uint32_t ph = cgb_mbar_phase[wib];
  int cur = 0;
  int64_t tile = blockIdx.x + G * wib;
  int rbi = 0;
  int64_t row0 = 0;
  int nvalid = 0;
  ConvWin win{nullptr, 0u, 0, false};
  if (tile < T) {
    rbi = find_rowblock(P, rb_lo, rb_hi, tile);
    const DevRowBlock& rb = P.rbs[rbi];
    tile_rows<MODE == 1>(rb, tile, row0, nvalid);
    win = conv_window(P, rb, row0, in, temp);
    if (win.ok) issue_window(win, xsb0, &bar[0], lane);
  }
  double* tl = (blockIdx.x == 0 && wib == 0 && lane == 0) ? cgb_tl_acc : nullptr;
  uint64_t tl0 = tl ? globaltimer() : 0, tl1 = tl0;
  for (; tile < T; tile += stride) {
    const DevRowBlock rb = P.rbs[rbi];
    const int R = rb.rfac;
    double* xcur = cur ? xsb1 : xsb0;
    // prefetch the next tile's window into the other buffer
    const int64_t ntile = tile + stride;
    int nrbi = rbi;
    int64_t nrow0 = 0;
    int nnvalid = 0;
    ConvWin nwin{nullptr, 0u, 0, false};
    if (ntile < T) {
      nrbi = find_rowblock(P, rb_lo, rb_hi, ntile);
      const DevRowBlock& nrb = P.rbs[nrbi];
      tile_rows<MODE == 1>(nrb, ntile, nrow0, nnvalid);
      nwin = conv_window(P, nrb, nrow0, in, temp);
      if (nwin.ok) issue_window(nwin, cur ? xsb0 : xsb1, &bar[cur ^ 1], lane);
    }
    if (strips && rb.strip_term >= 0) {  // done by run_strips
      cur ^= 1;
      rbi = nrbi;
      row0 = nrow0;
      nvalid = nnvalid;
      win = nwin;
      continue;
    }
    double acc[CGB_RC];
#pragma unroll
    for (int r = 0; r < CGB_RC; ++r) acc[r] = 0.0;
    for (int t = rb.term_begin; t < rb.term_end; ++t) {
      const cgb_term tm = P.terms[t];
      const cgb_leaf L = P.leaves[tm.leaf];
      const int toff = P.leaf_taps[tm.leaf];
      const double* cc = toff >= 0 ? P.taps + toff : nullptr;
      if (t == rb.conv_term && win.ok) {
        // the window was issued one tile ago; wait for its bytes
        if (tl) { const uint64_t x = globaltimer(); tl[3] += (double)(x - tl1); tl1 = x; }
        mbar_wait(&bar[cur], (ph >> cur) & 1u);
        ph ^= 1u << cur;
        __syncwarp();
        if (tl) { const uint64_t x = globaltimer(); tl[1] += (double)(x - tl1); tl1 = x; }
        conv_compute(L.k0, xcur + win.shift, cc, os, acc, tm.alpha, nvalid, lane);
        if (tl) { const uint64_t x = globaltimer(); tl[2] += (double)(x - tl1); tl1 = x; }
        continue;
      }
      const InVec tin = tm.in_buf == 0
                            ? in.shift(tm.in_off)
                            : InVec{temp + P.temp_off[tm.in_buf - 1] + tm.in_off, nullptr, 0.0};
      leaf_tile<MODE>(L, row0 - tm.row_origin, nvalid, R, tin, tm.alpha, acc, lane, cc, xcur, os,
                tin.b ? nullptr : ring, P.smem_xs2);
    }
    if (tl) { const uint64_t x = globaltimer(); tl[3] += (double)(x - tl1); tl1 = x; }
    if (rb.out_buf == 0) {
      epi.tile(row0 + lane, row0, R, nvalid - lane, acc, part);
    } else {
      double* dst = P.temp[ts] + P.temp_off[rb.out_buf - 1] + row0 + lane;
#pragma unroll
      for (int r = 0; r < CGB_RC; ++r)
        if (r < R && lane + 32 * r < nvalid) dst[32 * r] = acc[r];
    }
    if (tl) {
      const uint64_t x = globaltimer();
      tl[4] += (double)(x - tl1);
      tl1 = x;
      tl[0] += 1.0;
    }
    cur ^= 1;
    rbi = nrbi;
    row0 = nrow0;
    nvalid = nnvalid;
    win = nwin;
  }
  if (tl) tl[5] += (double)(globaltimer() - tl0);
  __syncwarp();
  if (lane == 0) cgb_mbar_phase[wib] = (cgb_mbar_phase[wib] & ~3u) | (ph & 3u);
  __syncwarp();
}

// Full application; levels separated by grid barriers.  No barrier after the
// final level: the caller follows with a reduction or sync.
template <int MODE, class Epi>
__device__ void apply_plan(const DevPlan& P, const InVec& in, Epi& epi, double* part,
                           GridSync& gs, int ts = 0) {
  for (int e = 0; e < P.nlevels; ++e) {
    if (e) gs.sync();
    run_level<MODE>(P, e, in, ts, epi, part);
  }
}

// Two independent applications in one phase (levels aligned at the end);
// the second uses temporary set 1, so both may be the same plan.
template <int MODE, class E1, class E2>
__device__ void apply_two(const DevPlan& P1, const InVec& in1, E1& e1, const DevPlan& P2,
                          const InVec& in2, E2& e2, double* part, GridSync& gs) {
  const int L = P1.nlevels > P2.nlevels ? P1.nlevels : P2.nlevels;
  for (int s = 0; s < L; ++s) {
    if (s) gs.sync();
    const int a = s - (L - P1.nlevels);
    if (a >= 0) run_level<MODE>(P1, a, in1, 0, e1, part);
    const int b = s - (L - P2.nlevels);
    if (b >= 0) run_level<MODE>(P2, b, in2, 1, e2, part);
  }
}

// Epilogue helper: slot r of a lane tile is a valid row
#define CGB_EPI_VALID(r) ((r) < R && 32 * (r) < left)
// a row index that is always safe to LOAD from: the slot's row when valid,
// else the tile's first row -- loads are issued unconditionally (no branch
// per slot), only stores and sums are guarded
#define CGB_EPI_IDX(j, r) (CGB_EPI_VALID(r) ? (j) + 32 * (r) : jlo)

// ---------------------------------------------------------------------------
// cone projections
// ---------------------------------------------------------------------------
// SOC projection in the branch-free form the reference solver graph
// evaluates (scs.py:250-264): inside*z + p_else*cand.
struct SocCoef {
  double inside, p_else, coef, safe;
  __device__ __forceinline__ SocCoef() : inside(0), p_else(0), coef(0), safe(1) {}
  __device__ __forceinline__ SocCoef(double t, double nu) {
    inside = 1.0 - (nu > t ? 1.0 : 0.0);
    const double in_polar = 1.0 - (nu > -1.0 * t ? 1.0 : 0.0);
    p_else = (1.0 - inside) * (1.0 - in_polar);
    coef = 0.5 * (t + nu);
    safe = nu + (1.0 - (nu > 0.0 ? 1.0 : 0.0));
  }
  __device__ __forceinline__ double head(double t) const { return inside * t + p_else * coef; }
  __device__ __forceinline__ double tail(double z) const {
    return inside * z + p_else * (coef * (z / safe));
  }
};

// Exponential cone K_exp = cl{(x,y,z): y > 0, y e^{x/y} <= z}: projection of
// one 3-vector, the algorithm of oracle/expcone_ref.py (stationarity in
// rho = x/y, roots of the e^{-2rho}-scaled equation G bracketed on a unit
// grid over [-60, 40]; the root with s_p > 0, mu >= 0 or the face point
// y = 0, whichever is closer), with the roots polished by safeguarded Newton
// instead of bisection.  A thread per cone.
static __device__ void exp_project(double& r, double& s, double& t) {
  // 1. inside K_exp
  if (s > 0.0) {
    if (r / s < 700.0 && s * exp(r / s) <= t) return;
  } else if (r <= 0.0 && s == 0.0 && t >= 0.0) {
    return;
  }
  // 2. inside the polar cone -> 0
  if (r > 0.0) {
    if (s / r < 700.0 && r * exp(s / r) + 2.718281828459045 * t <= 0.0) {
      r = s = t = 0.0;
      return;
    }
  } else if (r == 0.0 && s <= 0.0 && t <= 0.0) {
    r = s = t = 0.0;
    return;
  }
  // 3. the face y = 0
  if (r < 0.0 && s < 0.0) {
    s = 0.0;
    t = fmax(t, 0.0);
    return;
  }
  // 4. curved boundary (or the face).  Brackets from a unit-step scan of G
  //    with e^{-rho} carried multiplicatively (no exp in the scan); then
  //    every lane polishes its k-th bracket by safeguarded Newton at the same
  //    time (polishing inside the scan serialised a warp's lanes).
  double br = fmin(r, 0.0), bs = 0.0, bt = fmax(t, 0.0);
  double bd = (r - br) * (r - br) + s * s + (t - bt) * (t - bt);
  const double kEm1 = 0.36787944117144233;  // e^{-1}
  constexpr int kMaxBr = 3;
  double blo[kMaxBr];
  bool bneg[kMaxBr];
  int nb = 0;
  double lo = -60.0;
  double e1 = exp(60.0);                     // e^{-lo}
  double glo = (r - s * lo) * e1 * e1 + (r - r * lo - s) + t * e1 * (lo * lo - lo + 1.0);
  for (int step = 0; step < 100; ++step) {
    const double hi = lo + 1.0;
    const double e1h = e1 * kEm1;
    const double ghi = (r - s * hi) * e1h * e1h + (r - r * hi - s) + t * e1h * (hi * hi - hi + 1.0);
    if (((glo < 0.0) != (ghi < 0.0) || ghi == 0.0) && nb < kMaxBr) {
      blo[nb] = lo;
      bneg[nb] = glo < 0.0;
      ++nb;
    }
    lo = hi;
    e1 = e1h;
    glo = ghi;
  }
#pragma unroll
  for (int j = 0; j < kMaxBr; ++j) {
    if (j < nb) {
      double a = blo[j], b = blo[j] + 1.0;
      const bool alo_neg = bneg[j];
      double x = 0.5 * (a + b);
      for (int it = 0; it < 40; ++it) {
        const double ex = exp(-x);
        const double g = (r - s * x) * ex * ex + (r - r * x - s) + t * ex * (x * x - x + 1.0);
        if (g == 0.0) break;
        if ((g < 0.0) == alo_neg) a = x; else b = x;
        const double dg = (-s - 2.0 * (r - s * x)) * ex * ex - r + t * ex * (-x * x + 3.0 * x - 2.0);
        double xn = x - g / dg;
        if (!(xn > a && xn < b)) xn = 0.5 * (a + b);   // safeguard: bisect
        const double stp = fabs(xn - x);
        x = xn;
        // quadratic convergence: a step of 1e-9 leaves ~1e-18 of error
        if (stp <= 1e-9 * (1.0 + fabs(x)) || b - a <= 4e-16 * (1.0 + fabs(x))) break;
      }
      const double rho = x;
      const double e = exp(rho);
      const double sp = (r * rho + s + t * e) / (rho * rho + 1.0 + e * e);
      const double mu = sp * e - t;
      if (sp > 0.0 && mu >= -1e-12 * (1.0 + fabs(t))) {
        const double px = sp * rho, py = sp, pz = sp * e;
        const double d = (r - px) * (r - px) + (s - py) * (s - py) + (t - pz) * (t - pz);
        if (d < bd) {
          br = px;
          bs = py;
          bt = pz;
          bd = d;
        }
      }
    }
  }
  r = br;
  s = bs;
  t = bt;
}

// Pi_{K_exp*}(v) = v + Pi_{K_exp}(-v)   (Moreau)
__device__ __forceinline__ void exp_project_dual(double& r, double& s, double& t) {
  double a = -r, b = -s, c = -t;
  exp_project(a, b, c);
  r += a;
  s += b;
  t += c;
}

template <class Src>
struct SqSum {
  const Src* src;
  int64_t b;
  double acc;
  double z[CGB_U];
  __device__ void load(int64_t i, int u) { z[u] = (*src)(b + i); }
  __device__ void compute(int64_t, int u) { acc += z[u] * z[u]; }
};

// Partial sums feeding the large-SOC norms: slot s gets sum of squares of the
// tail of large SOC s; slot nlarge+s gets its head element (block 0 only).
template <class Src>
__device__ void cone_large_partials(const DevCones& K, const Src& src, double* part) {
  for (int s = 0; s < K.nseg; ++s) {
    const DevSeg sg = K.seg[s];
    if (sg.kind != SEG_SOC_LARGE) continue;
    SqSum<Src> f{&src, sg.begin + 1, 0.0, {}};
    stream_loop(sg.end - sg.begin - 1, f);
    part[sg.slot] += f.acc;
    if (blockIdx.x == 0 && threadIdx.x == 0) part[K.nlarge + sg.slot] += src(sg.begin);
  }
}

template <class Src, class Dst>
struct SegProj {
  const Src* src;
  const Dst* dst;
  int64_t b;
  int kind, dual;
  SocCoef sc;
  double t;
  double z[CGB_U];
  __device__ void load(int64_t i, int u) { z[u] = (*src)(b + i); }
  __device__ void compute(int64_t i, int u) {
    double out;
    if (kind == SEG_ZERO) out = dual ? z[u] : 0.0;
    else if (kind == SEG_NONNEG) out = fmax(z[u], 0.0);
    else out = (i == 0) ? sc.head(t) : sc.tail(z[u]);
    (*dst)(b + i, out);
  }
};

// Projection pass: dst(i, Pi(src)(i)) for every i of the cone space.
// `red` holds the reduced large-SOC partials from cone_large_partials.
template <class Src, class Dst>
__device__ void cone_project(const DevCones& K, int dual, const Src& src, const Dst& dst,
                             const double* red) {
  for (int s = 0; s < K.nseg; ++s) {
    const DevSeg sg = K.seg[s];
    const bool large = sg.kind == SEG_SOC_LARGE;
    const double t = large ? red[K.nlarge + sg.slot] : 0.0;
    SegProj<Src, Dst> f{&src, &dst, sg.begin, sg.kind, dual,
                        large ? SocCoef(t, sqrt(red[sg.slot])) : SocCoef(), t, {}};
    stream_loop(sg.end - sg.begin, f);
  }
  // exponential cones: a thread per cone
  for (int64_t c = gtid(); c < K.nexp; c += gsize()) {
    const int64_t off = K.exp_off[c];
    double r = src(off), s = src(off + 1), t = src(off + 2);
    if (dual) exp_project_dual(r, s, t);
    else exp_project(r, s, t);
    dst(off, r);
    dst(off + 1, s);
    dst(off + 2, t);
  }
  // small SOC blocks: one warp per cone
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x + (int64_t)gridDim.x * (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * CGB_WARPS;
  for (int64_t c = gw; c < K.nsmall; c += nw) {
    const int64_t off = K.small_off[c];
    const int dim = K.small_dim[c];
    const double t = src(off);
    double nu2 = 0.0;
    for (int i = 1 + lane; i < dim; i += 32) {
      const double z = src(off + i);
      nu2 += z * z;
    }
    nu2 = warp_sum(nu2);
    const SocCoef sc(t, sqrt(nu2));
    __syncwarp();
    for (int i = lane; i < dim; i += 32) {
      const double z = src(off + i);
      dst(off + i, i == 0 ? sc.head(t) : sc.tail(z));
    }
  }
}

}  // namespace cgb
