// cgb_shard.cuh -- the row-sharded splitting solver, one
// persistent kernel per rank.  Included by cgb200.cu only.
//
// Decomposition (oracle/shard_ref.py restates it on the host):
//   * rank q owns a contiguous range of the stuffed operator's rows (its
//     y-space: w_y, v_y, u_y, A x, b, g_y and the cone pieces there) and a
//     contiguous slice [x_begin[q], x_begin[q+1]) of the x-space vectors
//     (CG x, p, A^T A x, w_x, g_x);
//   * A x is local (the rank's rows of A times a full-length copy of x);
//   * A^T y = sum_q A_q^T y_q is a reduce-scatter fused into the adjoint's
//     epilogue: every output tile is stored straight into the inbox of the
//     rank owning those columns (NVLink peer stores), and the owner sums
//     the world's contributions in rank order;
//   * the CG residual r (the vector A is applied to next) is all-gathered
//     the same way: the slice update stores each new r_j into every rank's
//     full-length copy;
//   * every dot product is a grid reduction followed by an exchange of the
//     ranks' partials through per-rank mailboxes (one thread per peer
//     publishes, every CTA sums the R partials in rank order), so each
//     scalar -- and with it every loop decision -- is bitwise identical on
//     all ranks.
// Peer memory is the caller's: cgb_shard_comm carries every rank's inbox,
// full-length x buffer and mailbox as device pointers valid on this rank
// (cudaIpcOpenMemHandle'd across processes, or plain pointers when several
// ranks share one device).
#pragma once

#include "cgb_device.cuh"

namespace cgbs {

using namespace cgb;

__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// per-thread view of the world; `epoch` counts world synchronisations and
// is identical on every rank (they run the same sequence of them)
struct World {
  const cgb_shard_comm* c;
  unsigned long long epoch;
  __device__ __forceinline__ int owner(int64_t j) const {
    int o = 0;
    while (o + 1 < c->world && j >= c->x_begin[o + 1]) ++o;
    return o;
  }
};

// Grid reduction of v[0..NP) followed by the rank exchange: the result is
// sum_{q = 0..R-1} (rank q's grid sum), in rank order, in every thread of
// every rank.  pushed: this phase stored into peer memory (inbox / x
// copies); every thread fences those stores at system scope before the
// grid arrival, so they are visible to a peer that has seen this rank's
// mailbox entry (the same bar.sync + fence.sys pattern as a multi-grid
// sync).  NP == 0 is a world barrier.
template <int NP>
__device__ void world_reduce(GridSync& gs, World& W, double (&v)[NP > 0 ? NP : 1],
                             bool pushed) {
  if (pushed) __threadfence_system();
  if constexpr (NP > 0) {
    gs.reduce(v);
  } else {
    gs.sync();
  }
  W.epoch += 1;
  const int bank = (int)(W.epoch & 1ull);
  const int R = W.c->world, me = W.c->rank;
  if (blockIdx.x == 0 && threadIdx.x < (unsigned)R) {
    double* slot = W.c->mbox[threadIdx.x] +
                   ((size_t)bank * CGB_MAX_RANKS + (size_t)me) * CGB_MBOX_STRIDE;
#pragma unroll
    for (int p = 0; p < NP; ++p) slot[p] = v[p];
    st_release_sys_u64(reinterpret_cast<unsigned long long*>(slot + CGB_MAXP), W.epoch);
  }
  __shared__ double w_out[CGB_MAXP];
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double x[NP > 0 ? NP : 1];
#pragma unroll
    for (int p = 0; p < (NP > 0 ? NP : 1); ++p) x[p] = 0.0;
    if (lane < R) {
      const double* slot = W.c->mbox[me] +
                           ((size_t)bank * CGB_MAX_RANKS + (size_t)lane) * CGB_MBOX_STRIDE;
      const unsigned long long* seq = reinterpret_cast<const unsigned long long*>(slot + CGB_MAXP);
      if (ld_acquire_sys_u64(seq) < W.epoch) {
        const uint64_t t0 = globaltimer();
        while (ld_acquire_sys_u64(seq) < W.epoch) {
          if (globaltimer() - t0 > 20000000000ull) {  // 20 s: a peer is gone
            atomicExch(&gs.bar->err, 2u);
            __trap();
          }
        }
      }
#pragma unroll
      for (int p = 0; p < NP; ++p) x[p] = __ldcg(slot + p);
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      double s = 0.0;
      for (int q = 0; q < R; ++q) s += __shfl_sync(0xffffffffu, x[p], q);
      if (lane == 0) w_out[p] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int p = 0; p < NP; ++p) v[p] = w_out[p];
}

__device__ __forceinline__ void world_barrier(GridSync& gs, World& W, bool pushed) {
  double none[1] = {0.0};
  world_reduce<0>(gs, W, none, pushed);
}

// A^T tile -> the inbox of the rank owning its columns (reduce-scatter)
struct EpiPush {
  const cgb_shard_comm* c;
  __device__ void tile(int64_t j, int64_t jlo, int R, int left, const double (&y)[CGB_RC],
                       double*) const {
    World W{c, 0};
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q) {
      if (CGB_EPI_VALID(q)) {
        const int64_t jj = j + 32 * q;
        const int o = W.owner(jj);
        const int64_t len = c->x_begin[o + 1] - c->x_begin[o];
        c->inbox[o][(int64_t)c->rank * len + (jj - c->x_begin[o])] = y[q];
      }
    }
  }
};

// sum over the world of the contributions to local slice element i
__device__ __forceinline__ double inbox_sum(const cgb_shard_comm* c, const double* ib, int64_t nl,
                                            int64_t i) {
  double v[CGB_MAX_RANKS];
#pragma unroll
  for (int q = 0; q < CGB_MAX_RANKS; ++q) v[q] = q < c->world ? __ldcg(ib + q * nl + i) : 0.0;
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < CGB_MAX_RANKS; ++q)
    if (q < c->world) s += v[q];
  return s;
}

// store x-space value v of global index j into every rank's full-length copy
__device__ __forceinline__ void push_all(const cgb_shard_comm* c, int64_t j, double v) {
#pragma unroll
  for (int q = 0; q < CGB_MAX_RANKS; ++q)
    if (q < c->world) c->xfull[q][j] = v;
}

// grid-stride loop over the local slice, plain (the inbox sum is R loads)
template <class F>
__device__ __forceinline__ void slice_loop(int64_t nl, F& f) {
  const int64_t S = gsize();
  for (int64_t i = gtid(); i < nl; i += S) f(i);
}

}  // namespace cgbs
