// cgb_device.cuh -- device-side building blocks of the persistent solver
// kernels: grid barrier + deterministic grid reductions, the operator-plan
// executor (leaf tiles), cone projections.  Included by cgb200.cu only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/cgb200.h"

#ifndef CGB_BLOCK
#define CGB_BLOCK 512
#endif
#define CGB_WARPS (CGB_BLOCK / 32)
#ifndef CGB_MINB
#define CGB_MINB 1
#endif
#define CGB_MAXP 16          // reduction slots per grid reduction
#define CGB_MAXG 320         // largest grid the reductions are unrolled for
#define CGB_MAX_LARGE_SOC 4  // SOC blocks reduced across the whole grid
#ifndef CGB_RC
#define CGB_RC 9             // rows per lane in convolution tiles (odd: no bank conflicts)
#endif
#define CGB_CONV_KMAX 1024   // longest 1-d kernel staged in shared memory
#define CGB_U 4              // elements per thread per batch in streaming loops

namespace cgb {

// ---------------------------------------------------------------------------
// device plan / cone descriptors (built by the host in cgb200.cu)
// ---------------------------------------------------------------------------
struct DevRowBlock {
  int64_t row_begin, row_end, tile_begin;
  int32_t out_buf, term_begin, term_end;
  int32_t rfac;  // rows per lane in this block's tiles (1 or CGB_RC)
};

struct DevPlan {
  const cgb_leaf* leaves;
  const cgb_term* terms;
  const DevRowBlock* rbs;
  const int32_t* level_rb;     // nlevels + 1, execution order (deepest first)
  const int64_t* level_tiles;  // nlevels
  const int64_t* temp_off;     // ntemps
  double* temp[2];             // two temporary sets (two applications per phase)
  int32_t nlevels;
  int32_t smem_per_warp;  // doubles of dynamic shared memory per warp
  int32_t smem_cc;        // taps part (conv kernel, zero padded)
  int32_t smem_xs;        // staged-input part (output transpose follows)
  int64_t in_len, out_len;
};

enum SegKind : int32_t { SEG_ZERO = 0, SEG_NONNEG = 1, SEG_SOC_LARGE = 2 };

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

struct GridSync {
  GridBar* bar;
  double* partials;  // [2 banks][CGB_MAXP][grid]
  int bank;
  unsigned long long target;

  __device__ GridSync(GridBar* b, double* p) : bar(b), partials(p), bank(0), target(0) {}

  // All threads of all blocks must call this (uniform control flow).
  __device__ void sync() {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
      __threadfence();
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
      __threadfence();
    }
    __syncthreads();
  }

  // Sum v[0..NP) over every thread of the grid.  The result is bitwise
  // identical in every thread of every block (fixed summation order), so
  // control decisions taken on it stay grid-uniform.
  template <int NP>
  __device__ void reduce(double (&v)[NP]) {
    static_assert(NP <= CGB_MAXP, "too many reduction slots");
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
    if (wid == 0) {
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        double s = lane < CGB_WARPS ? red_smem[lane][p] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) bankp[(size_t)p * G + blockIdx.x] = s;
      }
    }
    sync();
    // warp 0 reads all partials (independent loads in flight) and broadcasts
    if (wid == 0) {
      constexpr int NI = (CGB_MAXG + 31) / 32;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        double x[NI];
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const int idx = lane + 32 * i;
          x[i] = idx < G ? __ldcg(bankp + (size_t)p * G + idx) : 0.0;
        }
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < NI; ++i) s += x[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) red_out[p] = s;
      }
    }
    __syncthreads();
#pragma unroll
    for (int p = 0; p < NP; ++p) v[p] = red_out[p];
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

// Contribution of one leaf to a warp tile.  The tile holds 32*R rows
// starting at leaf-local row lrow0; lane l owns rows lrow0 + l + 32 r
// (r < R), so epilogue stores are coalesced.  acc[r] accumulates.
// Warp-collective: every lane of the warp must call it.
//
// 1-d convolution / correlation leaves in R == CGB_RC tiles run the
// register-blocked path: the warp stages its taps and its input window
// (tile + halo, through the fused accessor) in shared memory once, each
// lane then computes CGB_RC *consecutive* outputs with a sliding register
// window (2*RC-1 + RC shared loads per RC*RC FMAs), and the results are
// transposed back to the lane-strided layout through shared memory.
__device__ __forceinline__ void leaf_tile(const cgb_leaf& L, int64_t lrow0, int nvalid, int R,
                                          const InVec& in, double alpha,
                                          double (&acc)[CGB_RC], int lane, double* cc,
                                          double* xs, double* os) {
  switch (L.kind) {
    case CGB_LEAF_IDENTITY: {
#pragma unroll
      for (int r = 0; r < CGB_RC; ++r)
        if (r < R && lane + 32 * r < nvalid) acc[r] += alpha * in(lrow0 + lane + 32 * r);
    } break;
    case CGB_LEAF_DENSE: {
      double mine[CGB_RC];
#pragma unroll
      for (int r = 0; r < CGB_RC; ++r) mine[r] = 0.0;
      const int64_t cols = L.cols;
      for (int rr = 0; rr < nvalid; ++rr) {
        const double* row = L.val + (lrow0 + rr) * L.ld;
        double s = 0.0;
#pragma unroll 4
        for (int64_t c = lane; c < cols; c += 32) s += __ldg(row + c) * in(c);
        s = warp_sum(s);
        if (lane == (rr & 31)) {
#pragma unroll
          for (int r = 0; r < CGB_RC; ++r)
            if (r == (rr >> 5)) mine[r] = s;
        }
      }
#pragma unroll
      for (int r = 0; r < CGB_RC; ++r) acc[r] += alpha * mine[r];
    } break;
    case CGB_LEAF_CSR: {
#pragma unroll
      for (int r = 0; r < CGB_RC; ++r) {
        if (r < R && lane + 32 * r < nvalid) {
          const int64_t lrow = lrow0 + lane + 32 * r;
          double s = 0.0;
          const int64_t e0 = __ldg(L.rowptr + lrow), e1 = __ldg(L.rowptr + lrow + 1);
          for (int64_t e = e0; e < e1; ++e) s += __ldg(L.val + e) * in(__ldg(L.colidx + e));
          acc[r] += alpha * s;
        }
      }
    } break;
    case CGB_LEAF_CONV1D:
    case CGB_LEAF_CORR1D: {
      const bool conv = L.kind == CGB_LEAF_CONV1D;
      const int64_t k = L.k0;
      if (R == CGB_RC) {
        // staged window: xs[i] = x[xlo + i]; every output is then the valid
        // correlation sum_j cc[j] xs[o + j] with cc = reversed kernel for conv
        const int64_t xlo = conv ? lrow0 - (k - 1) : lrow0;
        const int ngroups = (int)((k + CGB_RC - 1) / CGB_RC);
        const int ntaps = ngroups * CGB_RC;
        const int span = 32 * CGB_RC + ntaps + CGB_RC;
        const int o0 = lane * CGB_RC;
        __syncwarp();
        for (int i = lane; i < ntaps; i += 32)
          cc[i] = i < k ? __ldg(L.val + (conv ? k - 1 - i : i)) : 0.0;
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
        double y[CGB_RC];
#pragma unroll
        for (int r = 0; r < CGB_RC; ++r) y[r] = 0.0;
        for (int g = 0; g < ngroups; ++g) {
          const int j0 = g * CGB_RC;
          double w[2 * CGB_RC - 1];
#pragma unroll
          for (int i = 0; i < 2 * CGB_RC - 1; ++i) w[i] = xs[o0 + j0 + i];
#pragma unroll
          for (int jj = 0; jj < CGB_RC; ++jj) {
            const double cj = cc[j0 + jj];
#pragma unroll
            for (int r = 0; r < CGB_RC; ++r) y[r] += cj * w[r + jj];
          }
        }
#pragma unroll
        for (int r = 0; r < CGB_RC; ++r) os[o0 + r] = y[r];
        __syncwarp();
#pragma unroll
        for (int r = 0; r < CGB_RC; ++r)
          if (lane + 32 * r < nvalid) acc[r] += alpha * os[lane + 32 * r];
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

// Execute one level of a plan with temporary set `ts`.  Tiles are dealt
// round-robin across blocks first (tile t -> block t mod G) so every SM
// streams a similar share.  The epilogue gets a lane's whole tile at once:
// epi.tile(first_row, tile_row0, R, left, acc, part) with rows first_row + 32 r,
// valid while 32 r < left (see CGB_EPI_VALID) -- so it can issue all its
// loads before its stores.
template <class Epi>
__device__ void run_level(const DevPlan& P, int e, const InVec& in, int ts, Epi& epi,
                          double* part) {
  extern __shared__ double cgb_dyn_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* cc = cgb_dyn_smem + (size_t)wib * P.smem_per_warp;
  double* xs = cc + P.smem_cc;
  double* os = xs + P.smem_xs;
  const int64_t G = gridDim.x;
  const int64_t T = P.level_tiles[e];
  const int rb_lo = P.level_rb[e], rb_hi = P.level_rb[e + 1];
  double* temp = P.temp[ts];
  for (int64_t tile = blockIdx.x + G * wib; tile < T; tile += G * CGB_WARPS) {
    int lo = rb_lo, hi = rb_hi - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (P.rbs[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
    }
    const DevRowBlock rb = P.rbs[lo];
    const int R = rb.rfac;
    const int64_t row0 = rb.row_begin + (tile - rb.tile_begin) * (32 * R);
    const int64_t rem = rb.row_end - row0;
    const int nvalid = rem < 32 * R ? (int)rem : 32 * R;
    double acc[CGB_RC];
#pragma unroll
    for (int r = 0; r < CGB_RC; ++r) acc[r] = 0.0;
    for (int t = rb.term_begin; t < rb.term_end; ++t) {
      const cgb_term tm = P.terms[t];
      const cgb_leaf L = P.leaves[tm.leaf];
      const InVec tin = tm.in_buf == 0
                            ? in.shift(tm.in_off)
                            : InVec{temp + P.temp_off[tm.in_buf - 1] + tm.in_off, nullptr, 0.0};
      leaf_tile(L, row0 - tm.row_origin, nvalid, R, tin, tm.alpha, acc, lane, cc, xs, os);
    }
    if (rb.out_buf == 0) {
      epi.tile(row0 + lane, row0, R, nvalid - lane, acc, part);
    } else {
      double* dst = temp + P.temp_off[rb.out_buf - 1] + row0 + lane;
#pragma unroll
      for (int r = 0; r < CGB_RC; ++r)
        if (r < R && lane + 32 * r < nvalid) dst[32 * r] = acc[r];
    }
  }
}

// Full application; levels separated by grid barriers.  No barrier after the
// final level: the caller follows with a reduction or sync.
template <class Epi>
__device__ void apply_plan(const DevPlan& P, const InVec& in, Epi& epi, double* part,
                           GridSync& gs, int ts = 0) {
  for (int e = 0; e < P.nlevels; ++e) {
    if (e) gs.sync();
    run_level(P, e, in, ts, epi, part);
  }
}

// Two independent applications in one phase (levels aligned at the end);
// the second uses temporary set 1, so both may be the same plan.
template <class E1, class E2>
__device__ void apply_two(const DevPlan& P1, const InVec& in1, E1& e1, const DevPlan& P2,
                          const InVec& in2, E2& e2, double* part, GridSync& gs) {
  const int L = P1.nlevels > P2.nlevels ? P1.nlevels : P2.nlevels;
  for (int s = 0; s < L; ++s) {
    if (s) gs.sync();
    const int a = s - (L - P1.nlevels);
    if (a >= 0) run_level(P1, a, in1, 0, e1, part);
    const int b = s - (L - P2.nlevels);
    if (b >= 0) run_level(P2, b, in2, 1, e2, part);
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
