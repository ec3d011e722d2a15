// cgb200.cu -- persistent sm_100a kernels for the conegraph solver path and
// the C ABI declared in include/cgb200.h.
//
// One cooperative kernel per call runs the whole algorithm on device:
//   k_apply   y = A x / A^T x                       (linop.py:299-307)
//   k_cones   Pi_K / Pi_K*                           (cones.py:93-115)
//   k_cg      conjugate gradient                     (cg.py:87-165)
//   k_inner   inner block solve                      (scs.py:170-187)
//   k_scs     splitting iterations to termination    (scs.py:314-469)
// Phases inside a kernel are separated by a grid barrier; dot products are
// deterministic grid reductions whose result is identical in every block,
// so data-dependent loop control (CG convergence, status latch) needs no
// host round trip.

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "cgb_device.cuh"
#include "cgb_shard.cuh"

// Translation units: by default this file defines everything.  The build
// (build.py) compiles it several times in parallel with -DCGB_SPLIT and one
// CGB_TU_* flag each -- the host C ABI, and groups of kernel instantiations
// -- and links the objects into one library.
#ifndef CGB_SPLIT
#define CGB_TU_HOST 1
#define CGB_TU_SCS0 1
#define CGB_TU_SCS1 1
#define CGB_TU_CG 1
#define CGB_TU_INNER 1
#define CGB_TU_MISC 1
#define CGB_TU_SHARD 1
#define CGB_TU_SCS2 1
#endif
#ifndef CGB_TU_HOST
#define CGB_TU_HOST 0
#endif
#ifndef CGB_TU_SCS0
#define CGB_TU_SCS0 0
#endif
#ifndef CGB_TU_SCS1
#define CGB_TU_SCS1 0
#endif
#ifndef CGB_TU_CG
#define CGB_TU_CG 0
#endif
#ifndef CGB_TU_INNER
#define CGB_TU_INNER 0
#endif
#ifndef CGB_TU_MISC
#define CGB_TU_MISC 0
#endif
#ifndef CGB_TU_SHARD
#define CGB_TU_SHARD 0
#endif
#ifndef CGB_TU_SCS2
#define CGB_TU_SCS2 0
#endif

using namespace cgb;

// ===========================================================================
// epilogues: called once per lane tile (rows first + 32 r, r < R, valid
// while 32 r < left); all loads are issued before any store.
// ===========================================================================
namespace cgbk {

struct EpiStore {  // y -> out
  double* out;
  __device__ void tile(int64_t row, int64_t jlo, int R, int left, const double (&y)[CGB_RC], double*) const {
#pragma unroll
    for (int r = 0; r < CGB_RC; ++r)
      if (CGB_EPI_VALID(r)) out[row + 32 * r] = y[r];
  }
};

// Splitting-step / inner-solve start: with y = A^T d2 and g = A^T A x0,
//   rhs = d1 - y ;  r = rhs - (x0 + g) ;  sums: rhs.rhs, r.r (+ c.x0)
// (scs.py:349 rhs = wz1 - A^T wz2 ; cg.py:129 r0 = b - (1*x + A^T A x))
//   dw != null: d1 is not in memory but d1 = x0 - tau_w dw (the splitting
//   solver's w_x = u~_x = p1 - tau~ g_x of the previous cone step, computed
//   with the same fused multiply-add as XStep, so bitwise identical)
struct EpiRhs {
  const double* d1;
  const double* x0;
  const double* g;
  const double* c;  // optional: slot 2 gets c.x0
  double* r;
  const double* dw;
  double tau_w;
  int64_t c_lo, c_hi;  // c is zero outside [c_lo, c_hi)
  __device__ void prefetch(int64_t j0, int n, int lane) const {
    prefetch_range(dw ? dw : d1, j0, n, lane);
    prefetch_range(x0, j0, n, lane);
    prefetch_range(g, j0, n, lane);
  }
  __device__ void tile(int64_t j, int64_t jlo, int R, int left, const double (&y)[CGB_RC],
                       double* part) const {
    const bool hc = c && jlo < c_hi && jlo + 32 * R > c_lo;  // warp-uniform
    double a[CGB_RC], x[CGB_RC], gg[CGB_RC], cc[CGB_RC];
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q) {
      const int64_t jq = CGB_EPI_IDX(j, q);
      a[q] = dw ? dw[jq] : d1[jq]; x[q] = x0[jq]; gg[q] = g[jq];
      if (hc) cc[q] = c[jq];
    }
    if (dw) {
#pragma unroll
      for (int q = 0; q < CGB_RC; ++q) a[q] = fma(-tau_w, a[q], x[q]);
    }
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q) {
      if (CGB_EPI_VALID(q)) {
        const double rhs = a[q] - y[q];
        const double rr = rhs - (x[q] + gg[q]);
        r[j + 32 * q] = rr;
        part[0] += rhs * rhs;
        part[1] += rr * rr;
        if (hc) part[2] += cc[q] * x[q];
      }
    }
  }
};

// standalone CG init: r = b - apply(x) ; sums r.r, b.b   (cg.py:129-132)
struct EpiR0 {
  const double* b;
  const double* x;
  double* r;
  double lam;
  int normal;
  __device__ void tile(int64_t j, int64_t jlo, int R, int left, const double (&y)[CGB_RC],
                       double* part) const {
    double bb[CGB_RC], xx[CGB_RC];
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q)
      { const int64_t jq = CGB_EPI_IDX(j, q); bb[q] = b[jq]; xx[q] = x[jq]; }
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q) {
      if (CGB_EPI_VALID(q)) {
        double ax = y[q];
        if (normal && lam != 0.0) ax = lam * xx[q] + y[q];
        const double rr = bb[q] - ax;
        r[j + 32 * q] = rr;
        part[0] += rr * rr;
        part[1] += bb[q] * bb[q];
      }
    }
  }
};

// CG phase F (direct recipe): q = A p = A r + beta q_old ; sum p.q with
// p = r + beta p_old read pointwise
struct EpiQDirect {
  InVec pin;
  double* qv;
  double beta;
  int first;
  __device__ void tile(int64_t j, int64_t jlo, int R, int left, const double (&y)[CGB_RC],
                       double* part) const {
    double pp[CGB_RC], qo[CGB_RC];
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q) {
      const int64_t jq = CGB_EPI_IDX(j, q);
      pp[q] = pin(jq);
      if (!first) qo[q] = qv[jq];
    }
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q) {
      if (CGB_EPI_VALID(q)) {
        const double qq = first ? y[q] : y[q] + beta * qo[q];
        qv[j + 32 * q] = qq;
        part[0] += pp[q] * qq;
      }
    }
  }
};

// z2 = d2 + A z1 ; sum b.z2   (scs.py:186, 355)
struct EpiZ2 {
  double* ax;
  double* z2;
  const double* d2;
  const double* b;
  __device__ void tile(int64_t i, int64_t jlo, int R, int left, const double (&y)[CGB_RC],
                       double* part) const {
    double dd[CGB_RC], bb[CGB_RC];
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q)
      { const int64_t iq = CGB_EPI_IDX(i, q); dd[q] = d2[iq]; bb[q] = b ? b[iq] : 0.0; }
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q) {
      if (CGB_EPI_VALID(q)) {
        if (ax) ax[i + 32 * q] = y[q];
        const double v = dd[q] + y[q];
        z2[i + 32 * q] = v;
        part[0] += bb[q] * v;
      }
    }
  }
};

// residual phase, primal side: raw_p = (A ux + s) - tau b   (scs.py:372,392)
struct EpiRawP {
  const double* s;
  const double* b;
  double utau;
  __device__ void tile(int64_t i, int64_t jlo, int R, int left, const double (&y)[CGB_RC],
                       double* part) const {
    double ss[CGB_RC], bb[CGB_RC];
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q)
      { const int64_t iq = CGB_EPI_IDX(i, q); ss[q] = s[iq]; bb[q] = b[iq]; }
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q) {
      if (CGB_EPI_VALID(q)) {
        const double raw = (y[q] + ss[q]) - utau * bb[q];
        part[0] += raw * raw;
        const double unb = raw + utau * bb[q];
        part[1] += unb * unb;
      }
    }
  }
};

// residual phase, dual side: raw_d = A^T uy + tau c   (scs.py:373,397)
struct EpiRawD {
  const double* c;
  double utau;
  __device__ void tile(int64_t j, int64_t jlo, int R, int left, const double (&y)[CGB_RC],
                       double* part) const {
    double cc[CGB_RC];
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q)
      cc[q] = c[CGB_EPI_IDX(j, q)];
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q) {
      if (CGB_EPI_VALID(q)) {
        const double raw = y[q] + utau * cc[q];
        part[2] += raw * raw;
        const double inf = raw - utau * cc[q];
        part[3] += inf * inf;
      }
    }
  }
};

// ===========================================================================
// phase profiler (optional): block 0 / thread 0 accumulates globaltimer
// deltas per phase; every mark sits right after a grid barrier, so the
// delta is the whole grid's time in that phase.
// ===========================================================================
enum ProfPhase : int {
  PROF_RHS = 0,     // subspace rhs: A^T w_y + r0 + reduce
  PROF_CG_F = 1,    // CG: t = A p + reduce
  PROF_CG_A = 2,    // CG: A^T t + fused updates + reduce
  PROF_CONE_X = 3,  // cone step: free x block   (profiling adds a barrier)
  PROF_CONE_E = 4,  // cone step: elementwise + small SOC segments (+ barrier)
  PROF_CONE_A = 5,  // cone step: large-SOC pass A + reduce
  PROF_CONE_B = 6,  // cone step: large-SOC pass B + barrier
  PROF_CHECK = 7,   // residual check
  PROF_INIT = 8,    // per-launch setup (b.Ax, b.w_y)
  PROF_CONE_AR = 9, // large-SOC pass A reduce alone (profiling only)
  PROF_N = 16
};

struct Prof {
  double* acc;  // PROF_N doubles (ns), or null
  uint64_t last;
  __device__ explicit Prof(double* p) : acc(p), last(0) {
    if (acc && blockIdx.x == 0 && threadIdx.x == 0) last = globaltimer();
  }
  __device__ __forceinline__ void mark(int phase) {
    if (acc && blockIdx.x == 0 && threadIdx.x == 0) {
      const uint64_t now = globaltimer();
      acc[phase] += (double)(now - last);
      last = now;
    }
  }
};

// ===========================================================================
// CG loop shared by k_cg, k_inner and k_scs  (cg.py:87-137)
// ===========================================================================
// Two grid reductions per iteration.
// Normal recipe, solve (lam I + A^T A) x = b:
//   phase F : t = A p by linearity: t <- A r + beta t_old (A applied to
//             the plain vector r, so its windows can be TMA-staged); a
//             stream pass sums p.p (+ c.p) with p = r + beta p_old, the
//             epilogue t.t (+ b.t), then
//             alpha = rns / (lam p.p + t.t)       [= rns / p.(lam p + A^T A p)]
//   phase A : y = A^T t; per element p = r + beta p_old (stored in place),
//             q = lam p + y, x += alpha p, r -= alpha q, gx += alpha y;
//             sum r.r ; ax += alpha t when tracking
// Direct recipe (A square SPD): phase F q = A r + beta q_old, sum p.q;
// phase U the stream update.  Same updates as the reference listing,
// reassociated only in how A p and p.Ap are summed.
struct CgBufs {
  double* x;
  double* r;
  double* p;   // direction, updated in place
  double* q;   // direct recipe only
  double* t;   // m scratch (normal recipe): A p
  double* ax;  // m, tracked A x (or null)
  double* gx;  // n, tracked A^T A x (or null)
  const double* b;  // m, tracking dots (or null)
  const double* c;  // n, tracking dots (or null)
  int64_t b_lo, b_hi;  // b is zero outside [b_lo, b_hi)
  int64_t c_lo, c_hi;  // c is zero outside [c_lo, c_hi)
};

// phase F (normal): t = A p by linearity, A p = A r + beta A p_old, i.e.
// t <- A r + beta t_old ; sums t.t (slot 0), b.t (slot 3)
struct EpiT {
  double* t;
  const double* b;
  double beta;
  int first;
  int64_t b_lo, b_hi;  // b is zero outside [b_lo, b_hi)
  __device__ void prefetch(int64_t j0, int n, int lane) const {
    if (!first) prefetch_range(t, j0, n, lane);
    if (b && j0 < b_hi && j0 + n > b_lo) prefetch_range(b, j0, n, lane);
  }
  __device__ void tile(int64_t i, int64_t jlo, int R, int left, const double (&y)[CGB_RC],
                       double* part) const {
    const bool hb = b && jlo < b_hi && jlo + 32 * R > b_lo;  // warp-uniform
    double bb[CGB_RC], to[CGB_RC];
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q) {
      const int64_t iq = CGB_EPI_IDX(i, q);
      if (hb) bb[q] = b[iq];
      if (!first) to[q] = t[iq];
    }
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q) {
      if (CGB_EPI_VALID(q)) {
        const double tv = first ? y[q] : y[q] + beta * to[q];
        t[i + 32 * q] = tv;
        part[0] += tv * tv;
        if (hb) part[3] += bb[q] * tv;
      }
    }
  }
};

// phase F stream: p = r + beta p_old ; sums p.p (slot 1), c.p (slot 2).
// Inputs (bulk_stream): r, [p_old unless first], [c when tracking].
template <bool P_OLD, bool C>
struct PDots {
  double beta;
  double pp, cp;
  template <int NIN>
  __device__ __forceinline__ void compute(int64_t, const double (&v)[NIN], int64_t) {
    const double p = P_OLD ? v[0] + beta * v[1] : v[0];
    pp += p * p;
    if (C) cp += v[NIN - 1] * p;
  }
};

template <bool P_OLD, bool C>
__device__ __forceinline__ void pdots(int64_t n, const double* r, const double* p,
                                      const double* c, double beta, double& pp, double& cp) {
  PDots<P_OLD, C> f{beta, 0.0, 0.0};
  if (P_OLD && C) {
    const double* src[3] = {r, p, c};
    bulk_stream<3>(n, src, f);
  } else if (P_OLD) {
    const double* src[2] = {r, p};
    bulk_stream<2>(n, src, f);
  } else if (C) {
    const double* src[2] = {r, c};
    bulk_stream<2>(n, src, f);
  } else {
    const double* src[1] = {r};
    bulk_stream<1>(n, src, f);
  }
  pp = f.pp;
  cp = f.cp;
}

// phase A (normal): the whole CG update in the A^T t epilogue ; sum r.r
struct EpiCgUpd {
  double* r; double* p; double* x; double* gx;
  double beta; int first; double lam, alpha;
  __device__ void prefetch(int64_t j0, int n, int lane) const {
    prefetch_range(r, j0, n, lane);
    if (!first) prefetch_range(p, j0, n, lane);
    prefetch_range(x, j0, n, lane);
    prefetch_range(gx, j0, n, lane);
  }
  __device__ void tile(int64_t j, int64_t jlo, int R, int left, const double (&y)[CGB_RC],
                       double* part) const {
    double rv[CGB_RC], pv[CGB_RC], xv[CGB_RC], gv[CGB_RC];
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q) {
      const int64_t jq = CGB_EPI_IDX(j, q);
      rv[q] = r[jq];
      if (!first) pv[q] = p[jq];
      xv[q] = x[jq];
      if (gx) gv[q] = gx[jq];
    }
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q) {
      if (CGB_EPI_VALID(q)) {
        const double pp = first ? rv[q] : rv[q] + beta * pv[q];
        const double qq = (lam != 0.0) ? lam * pp + y[q] : y[q];
        const double rn = rv[q] - alpha * qq;
        p[j + 32 * q] = pp;
        x[j + 32 * q] = xv[q] + alpha * pp;
        r[j + 32 * q] = rn;
        if (gx) gx[j + 32 * q] = gv[q] + alpha * y[q];
        part[0] += rn * rn;
      }
    }
  }
};

struct AxUpd {  // ax += alpha t   (inputs: ax, t)
  double* ax; double alpha;
  __device__ __forceinline__ void compute(int64_t i, const double (&v)[2], int64_t) {
    ax[i] = v[0] + alpha * v[1];
  }
};

// direct recipe phase U: p = r + beta p ; x += alpha p ; r -= alpha q ; sum r.r
// (inputs: x, r, q, [p_old unless first])
struct CgUpdDirect {
  double* x; double* r; double* p;
  double beta; double alpha;
  double rr;
  template <int NIN>
  __device__ __forceinline__ void compute(int64_t i, const double (&v)[NIN], int64_t) {
    const double pp = NIN == 4 ? v[1] + beta * v[NIN - 1] : v[1];
    p[i] = pp;
    x[i] = v[0] + alpha * pp;
    const double rn = v[1] - alpha * v[2];
    r[i] = rn;
    rr += rn * rn;
  }
};

// Runs CG from r = b - apply(x) (stored in B.r) with rns = r.r.  Returns the
// iteration count.  With tracking (B.c != null) *cx += alpha c.p and
// *bax += alpha b.t follow c.x and b.(A x) through the updates.
template <int TD>
__device__ int64_t cg_loop(const DevPlan& F, const DevPlan& Aj, int recipe, double lam,
                           const CgBufs& B, int64_t n, int64_t m, double& rns, double delta,
                           double floor_, int64_t max_iter, GridSync& gs, double* cx,
                           double* bax, Prof& prof) {
  int64_t k = 0;
  double beta = 0.0;
  const bool track = B.c != nullptr;
  while (sqrt(rns) > delta && rns > floor_ && (double)max_iter > (double)k) {
    const int first = k == 0;
    const InVec rin{B.r, nullptr, 0.0};
    const InVec pin = first ? rin : InVec{B.r, B.p, beta};
    if (recipe == CGB_RECIPE_NORMAL) {
      double s[4] = {0.0, 0.0, 0.0, 0.0};
      {
        EpiT et{B.t, track ? B.b : nullptr, beta, first, B.b_lo, B.b_hi};
        apply_plan<TD>(F, rin, et, s, gs);
        double pp = 0.0, cp = 0.0;
        // a c with few nonzeros (stuffed objectives) is dotted by one thread
        const bool c_short = track && B.c_hi - B.c_lo <= 64;
        const bool c_stream = track && !c_short;
        if (first) {
          if (c_stream) pdots<false, true>(n, B.r, B.p, B.c, beta, pp, cp);
          else pdots<false, false>(n, B.r, B.p, B.c, beta, pp, cp);
        } else {
          if (c_stream) pdots<true, true>(n, B.r, B.p, B.c, beta, pp, cp);
          else pdots<true, false>(n, B.r, B.p, B.c, beta, pp, cp);
        }
        if (c_short && blockIdx.x == 0 && threadIdx.x == 0) {
          for (int64_t i = B.c_lo; i < B.c_hi; ++i)
            cp += B.c[i] * (first ? B.r[i] : B.r[i] + beta * B.p[i]);
        }
        s[1] += pp;
        s[2] += cp;
      }
      gs.reduce(s);
      prof.mark(PROF_CG_F);
      const double alpha = rns / ((lam != 0.0 ? lam * s[1] : 0.0) + s[0]);
      if (track) {
        *cx += alpha * s[2];
        *bax += alpha * s[3];
      }
      double rr[1] = {0.0};
      {
        const InVec tin{B.t, nullptr, 0.0};
        EpiCgUpd eu{B.r, B.p, B.x, B.gx, beta, first, lam, alpha};
        apply_plan<TD>(Aj, tin, eu, rr, gs);
        if (B.ax) {
          AxUpd f{B.ax, alpha};
          const double* src[2] = {B.ax, B.t};
          bulk_stream<2>(m, src, f);
        }
      }
      gs.reduce(rr);
      prof.mark(PROF_CG_A);
      beta = rr[0] / rns;
      rns = rr[0];
    } else {
      double pq[1] = {0.0};
      EpiQDirect eq{pin, B.q, beta, first};
      apply_plan<TD>(F, rin, eq, pq, gs);
      gs.reduce(pq);
      prof.mark(PROF_CG_F);
      const double alpha = rns / pq[0];
      double rr[1] = {0.0};
      CgUpdDirect f{B.x, B.r, B.p, beta, alpha, 0.0};
      if (first) {
        const double* src[3] = {B.x, B.r, B.q};
        bulk_stream<3>(n, src, f);
      } else {
        const double* src[4] = {B.x, B.r, B.q, B.p};
        bulk_stream<4>(n, src, f);
      }
      rr[0] = f.rr;
      gs.reduce(rr);
      prof.mark(PROF_CG_A);
      beta = rr[0] / rns;
      rns = rr[0];
    }
    ++k;
  }
  return k;
}

// ===========================================================================
// kernels
// ===========================================================================
struct ApplyArgs {
  GridBar* bar; double* partials;
  DevPlan P;
  const double* x; double* y;
};

template <int TD>
__global__ void __launch_bounds__(CGB_BLOCK, CGB_MINB) k_apply(const __grid_constant__ ApplyArgs a) 
#if CGB_TU_MISC
{
  tma_init();
  const DevPlan& P = *cache_plan(0, a.P);
  GridSync gs(a.bar, a.partials);
  InVec in{a.x, nullptr, 0.0};
  EpiStore st{a.y};
  apply_plan<TD>(P, in, st, nullptr, gs);
}
#else
;
#endif

struct ConeArgs {
  GridBar* bar; double* partials;
  DevCones K;
  int dual;
  const double* v; double* out;
};

struct SrcVec {
  const double* v;
  __device__ double operator()(int64_t i) const { return v[i]; }
};
struct DstVec {
  double* out;
  __device__ void operator()(int64_t i, double x) const { out[i] = x; }
};

__global__ void __launch_bounds__(CGB_BLOCK, CGB_MINB) k_cones(const __grid_constant__ ConeArgs a) 
#if CGB_TU_MISC
{
  GridSync gs(a.bar, a.partials);
  SrcVec src{a.v};
  DstVec dst{a.out};
  double red[2 * CGB_MAX_LARGE_SOC];
#pragma unroll
  for (int i = 0; i < 2 * CGB_MAX_LARGE_SOC; ++i) red[i] = 0.0;
  if (a.K.nlarge > 0) {
    cone_large_partials(a.K, src, red);
    gs.reduce(red);
  }
  cone_project(a.K, a.dual, src, dst, red);
}
#else
;
#endif

struct CgArgs {
  GridBar* bar; double* partials;
  DevPlan F, Aj;
  int recipe; double lam;
  const double* b; double* x;
  double* r; double* p; double* q; double* t;
  int64_t n, m; double tol; int64_t max_iter; double eps_floor;
  double* result;  // [iterations, rns, bnorm2]
};

template <int TD>
__global__ void __launch_bounds__(CGB_BLOCK, CGB_MINB) k_cg(const __grid_constant__ CgArgs a) 
#if CGB_TU_CG
{
  tma_init();
  const DevPlan& F = *cache_plan(0, a.F);
  const DevPlan& Aj = *cache_plan(1, a.Aj);
  GridSync gs(a.bar, a.partials);
  Prof prof(nullptr);
  double s[2] = {0.0, 0.0};
  InVec xin{a.x, nullptr, 0.0};
  if (a.recipe == CGB_RECIPE_NORMAL) {
    EpiStore st{a.t};
    apply_plan<TD>(F, xin, st, nullptr, gs);
    gs.sync();
    InVec tin{a.t, nullptr, 0.0};
    EpiR0 e{a.b, a.x, a.r, a.lam, 1};
    apply_plan<TD>(Aj, tin, e, s, gs);
  } else {
    EpiR0 e{a.b, a.x, a.r, 0.0, 0};
    apply_plan<TD>(F, xin, e, s, gs);
  }
  gs.reduce(s);
  double rns = s[0];
  const double delta = a.tol * sqrt(s[1]);
  const double floor_ = a.eps_floor * s[1];
  CgBufs B{a.x, a.r, a.p, a.q, a.t, nullptr, nullptr, nullptr, nullptr, 0, 0, 0, 0};
  const int64_t k = cg_loop<TD>(F, Aj, a.recipe, a.lam, B, a.n, a.m, rns, delta, floor_,
                            a.max_iter, gs, nullptr, nullptr, prof);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.result[0] = (double)k;
    a.result[1] = rns;
    a.result[2] = s[1];
  }
}
#else
;
#endif

struct InnerArgs {
  GridBar* bar; double* partials;
  DevPlan F, Aj;
  const double* d1; const double* d2;
  double* z;  // n + m
  const double* c; const double* b;
  double* r; double* p; double* gx; double* t; double* tx;
  int64_t n, m; double tol; int64_t max_iter; double eps_floor;
  double* result;  // [iterations, rns, rhs2, hdot]
};

struct SideDot {  // acc += x[i] * y[i]   (inputs: x, y)
  double acc;
  __device__ __forceinline__ void compute(int64_t, const double (&v)[2], int64_t) {
    acc += v[0] * v[1];
  }
};

__device__ __forceinline__ double side_dot(int64_t n, const double* x, const double* y) {
  SideDot f{0.0};
  const double* src[2] = {x, y};
  bulk_stream<2>(n, src, f);
  return f.acc;
}

// Inner block solve, the reference's arithmetic (scs.py:170-187):
// rhs = d1 - A^T d2 ; r0 = rhs - (x0 + A^T A x0) ; CG ; z2 = d2 + A z1.
template <int TD>
__global__ void __launch_bounds__(CGB_BLOCK, CGB_MINB) k_inner(const __grid_constant__ InnerArgs a) 
#if CGB_TU_INNER
{
  tma_init();
  const DevPlan& F = *cache_plan(0, a.F);
  const DevPlan& Aj = *cache_plan(1, a.Aj);
  GridSync gs(a.bar, a.partials);
  Prof prof(nullptr);
  double* z1 = a.z;
  double* z2 = a.z + a.n;
  // tx = A x0 ; then gx = A^T tx
  {
    InVec xin{z1, nullptr, 0.0};
    EpiStore st{a.tx};
    apply_plan<TD>(F, xin, st, nullptr, gs);
    gs.sync();
    InVec tin{a.tx, nullptr, 0.0};
    EpiStore st2{a.gx};
    apply_plan<TD>(Aj, tin, st2, nullptr, gs);
    gs.sync();
  }
  double s[3] = {0.0, 0.0, 0.0};
  {
    InVec din{a.d2, nullptr, 0.0};
    EpiRhs e{a.d1, z1, a.gx, nullptr, a.r, nullptr, 0.0, 0, 0};
    apply_plan<TD>(Aj, din, e, s, gs);
    gs.reduce(s);
  }
  double rns = s[1];
  const double delta = a.tol * sqrt(s[0]);
  const double floor_ = a.eps_floor * s[0];
  CgBufs B{z1, a.r, a.p, nullptr, a.t, nullptr, nullptr, nullptr, nullptr, 0, 0, 0, 0};
  const int64_t k = cg_loop<TD>(F, Aj, CGB_RECIPE_NORMAL, 1.0, B, a.n, a.m, rns, delta, floor_,
                            a.max_iter, gs, nullptr, nullptr, prof);
  double h[2] = {0.0, 0.0};
  {
    InVec xin{z1, nullptr, 0.0};
    EpiZ2 e{nullptr, z2, a.d2, a.b};
    apply_plan<TD>(F, xin, e, h, gs);
    if (a.c) {
      h[1] = side_dot(a.n, a.c, z1);
    }
    gs.reduce(h);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.result[0] = (double)k;
    a.result[1] = rns;
    a.result[2] = s[0];
    a.result[3] = h[1] + h[0];
  }
}
#else
;
#endif

// ---------------------------------------------------------------------------
// the splitting solver
// ---------------------------------------------------------------------------
struct ScsArgs {
  GridBar* bar; double* partials;
  DevPlan F, Aj;
  DevCones K;
  cgb_scs_settings st;
  cgb_scs_work w;
  const double* b; const double* c; const double* g;
  int64_t n, m;
  double denom, pr_scale, dr_scale, eps_floor;
  int64_t max_steps;
  int resid_every;
  int stash_cap;   // doubles of shared memory per CTA for the SOC stash
  double* prof;    // PROF_N phase times (ns) or null
  int no_skip;     // 1: stream all of b and c (CGB_SCS_NO_ZERO_SKIP)
  double* park;    // m: large-SOC source between passes A and B (the CG scratch t), or null
  int refresh;     // > 0: recompute A cgx, A^T A cgx every `refresh` iterations
};

// [first, last + 1) of the nonzeros of b (slots 0, 1) and c (slots 2, 3),
// as maxima of (-first, last + 1) so one max-reduction gives both ends
struct NzRange {
  double r0, r1;
  __device__ __forceinline__ void compute(int64_t i, const double (&v)[1], int64_t) {
    if (v[0] != 0.0) {
      r0 = fmax(r0, -(double)i);
      r1 = fmax(r1, (double)(i + 1));
    }
  }
};

// CG tolerance exactly as the solver graph computes it (scs.py:290-311)
static __device__ double cg_tolerance_graph(double k, const cgb_scs_settings& s) {
  const double kp1 = k + 1.0;
  const double pw = s.cg_tol_power;
  double den;
  if (pw == 0.5) den = sqrt(kp1);
  else if (pw == 1.0) den = kp1;
  else if (pw == 1.25) den = kp1 * sqrt(sqrt(kp1));
  else if (pw == 1.5) den = kp1 * sqrt(kp1);
  else den = kp1 * kp1;
  const double tol_raw = 1.0 / den;
  const double sat = s.cg_eps_factor * s.eps;
  const double tol_sat = sat + fmax(tol_raw - sat, 0.0);
  const double tol_capped = s.cg_tol_cap - fmax(s.cg_tol_cap - tol_sat, 0.0);
  return s.cg_base_tol + fmax(tol_capped - s.cg_base_tol, 0.0);
}

// Cone step of one splitting iteration on the y block (scs.py:358-366):
//   src = u~_y - v_y with u~_y = (w_y + A p1) - tau~ g_y
//   u_y = Pi_{K*}(src) ;  v_y <- (v_y - u~_y) + u_y  ==  u_y - src  (bitwise:
//   fl(v - u~) = -fl(u~ - v)) ;  w_y = u_y + v_y
// and the running sum b.w_y for the next subspace step.
struct ConeStep {
  const double* wy; const double* ax; const double* gy; double* vy; double* uy; double* wyo;
  const double* b;
  double tau;
  int write_u;
  __device__ __forceinline__ double src(int64_t i) const {
    return ((wy[i] + ax[i]) - tau * gy[i]) - vy[i];
  }
  __device__ __forceinline__ double store(int64_t i, double s, double u2) const {
    const double v2 = u2 - s;
    const double w2 = u2 + v2;
    if (write_u) uy[i] = u2;
    vy[i] = v2;
    wyo[i] = w2;
    return w2;
  }
};

// elementwise segments (zero -> free in the dual, nonneg), one pass
// (inputs at the segment: w_y, A p1, g_y, v_y, b)
struct ConeElem {
  const ConeStep* cs;
  int64_t base;
  int kind;
  double bw;
  __device__ __forceinline__ void compute(int64_t i, const double (&v)[5], int64_t) {
    const double s = ((v[0] + v[1]) - cs->tau * v[2]) - v[3];
    const double u2 = kind == SEG_ZERO ? s : fmax(s, 0.0);
    bw += v[4] * cs->store(base + i, s, u2);
  }
};

// the same where b is zero on the segment (inputs: w_y, A p1, g_y, v_y)
struct ConeElemNoB {
  const ConeStep* cs;
  int64_t base;
  int kind;
  __device__ __forceinline__ void compute(int64_t i, const double (&v)[4], int64_t) {
    const double s = ((v[0] + v[1]) - cs->tau * v[2]) - v[3];
    const double u2 = kind == SEG_ZERO ? s : fmax(s, 0.0);
    cs->store(base + i, s, u2);
  }
};

// the free x block: v_x == 0 is an invariant of the embedding (v = (0, s,
// kappa)), so u_x = w_x = u~_x = p1 - tau~ g_x and v_x stays 0 bitwise.
// (inputs: p1, g_x)
struct XStep {
  double* u; double* w; double tau; int write_u;
  __device__ __forceinline__ void compute(int64_t i, const double (&v)[2], int64_t) {
    const double ut = fma(-tau, v[1], v[0]);
    w[i] = ut;
    if (write_u) u[i] = ut;
  }
};

// large SOC, pass A: tail sum of squares; the source kept in the CTA's
// shared-memory stash (slot = offset in the CTA's range) for pass B
// (inputs at the tail: w_y, A p1, g_y, v_y)
struct SocPassA {
  double tau;
  double* stash;  // or null
  double acc;
  __device__ __forceinline__ void compute(int64_t, const double (&v)[4], int64_t j) {
    const double z = ((v[0] + v[1]) - tau * v[2]) - v[3];
    acc += z * z;
    if (stash) stash[j] = z;
  }
};

// large SOC, pass B from the stash (input: b at the tail)
struct SocPassB {
  const ConeStep* cs;
  int64_t base;
  SocCoef sc;
  const double* stash;
  double bw;
  __device__ __forceinline__ void compute(int64_t i, const double (&v)[1], int64_t j) {
    const double z = stash[j];
    bw += v[0] * cs->store(base + i, z, sc.tail(z));
  }
};

// large SOC too big for the shared-memory stash: pass A parks its source in
// a global scratch vector (the CG scratch t, idle during the cone step) and
// pass B reads it back with b -- 2 reads instead of recomputing the source
// from 4 (bitwise the same source value).
struct SocPassAG {
  double tau;
  double* park;  // indexed like the tail
  double acc;
  __device__ __forceinline__ void compute(int64_t i, const double (&v)[4], int64_t) {
    const double z = ((v[0] + v[1]) - tau * v[2]) - v[3];
    acc += z * z;
    park[i] = z;
  }
};
struct SocPassBG {  // inputs: the parked source, b
  const ConeStep* cs;
  int64_t base;
  SocCoef sc;
  double bw;
  __device__ __forceinline__ void compute(int64_t i, const double (&v)[2], int64_t) {
    const double z = v[0];
    bw += v[1] * cs->store(base + i, z, sc.tail(z));
  }
};

// large SOC, pass B recomputing the source (inputs: w_y, A p1, g_y, v_y, b)
struct SocPassB2 {
  const ConeStep* cs;
  int64_t base;
  SocCoef sc;
  double bw;
  __device__ __forceinline__ void compute(int64_t i, const double (&v)[5], int64_t) {
    const double z = ((v[0] + v[1]) - cs->tau * v[2]) - v[3];
    bw += v[4] * cs->store(base + i, z, sc.tail(z));
  }
};

template <int TD>
__global__ void __launch_bounds__(CGB_BLOCK, CGB_MINB) k_scs(const __grid_constant__ ScsArgs a) 
#if CGB_TU_SCS0 || CGB_TU_SCS1 || CGB_TU_SCS2
{
  extern __shared__ __align__(16) double cgb_dyn_smem[];
  tma_init();
  GridSync gs(a.bar, a.partials);
  Prof prof(a.prof);
  const DevPlan& F = *cache_plan(0, a.F);
  const DevPlan& Aj = *cache_plan(1, a.Aj);
  const int64_t n = a.n, m = a.m, N = n + m + 1;
  const cgb_scs_settings& S = a.st;
  const cgb_scs_work& W = a.w;
  double* state = W.state;
  double k = state[CGB_ST_K], since = state[CGB_ST_SINCE], status = state[CGB_ST_STATUS];
  double cgt = state[CGB_ST_CGT];
  double pr = state[CGB_ST_PR], dr = state[CGB_ST_DR], gap = state[CGB_ST_GAP];
  double res_u_last = state[CGB_ST_RES_U], res_i_last = state[CGB_ST_RES_I];
  double lastcg = state[CGB_ST_LASTCG];
  const int64_t cg_max = S.cg_max_iter;
  int64_t steps = 0;
  const double* wy = W.w + n;
  const DevCones& K = a.K;

  // large-SOC stash: the pass-A source of every large SOC tail stays in the
  // CTA's shared memory (after the bulk-stream ring) until pass B
  int64_t stash_need = 0;
  for (int s = 0; s < K.nseg; ++s)
    if (K.seg[s].kind == SEG_SOC_LARGE) stash_need += stream_span(K.seg[s].end - K.seg[s].begin - 1);
  const bool use_stash = stash_need <= (int64_t)a.stash_cap;
  double* const stash_base = cgb_dyn_smem;

  // b and c are exactly zero outside [b_lo, b_hi) / [c_lo, c_hi) (stuffed
  // problems: deconv b = (0, 0, -b_signal), c = (0, 1)); the loop skips those
  // loads.  The ranges are measured here, once per launch (one pass over b
  // and c), so no caller-supplied hint can drop a nonzero.
  int64_t b_lo = 0, b_hi = m, c_lo = 0, c_hi = n;
  if (!a.no_skip) {
    double rr[4];
    {
      NzRange fb{-DBL_MAX, -DBL_MAX};
      const double* sb[1] = {a.b};
      bulk_stream<1>(m, sb, fb);
      NzRange fc{-DBL_MAX, -DBL_MAX};
      const double* sc[1] = {a.c};
      bulk_stream<1>(n, sc, fc);
      rr[0] = fb.r0; rr[1] = fb.r1; rr[2] = fc.r0; rr[3] = fc.r1;
    }
    gs.reduce_max(rr);
    b_lo = rr[1] > 0.0 ? (int64_t)(-rr[0]) : 0;
    b_hi = rr[1] > 0.0 ? (int64_t)rr[1] : 0;
    c_lo = rr[3] > 0.0 ? (int64_t)(-rr[2]) : 0;
    c_hi = rr[3] > 0.0 ? (int64_t)rr[3] : 0;
  }

  // running scalars: b.(A x) follows x through the CG updates; b.w_y is
  // summed by every cone step for the next subspace step.
  double bax = 0.0, bwy_part = 0.0;
  bool wx_stale = false;  // w_x not stored since the last cone step
  double tau_prev = 0.0;  // that cone step's tau~
  {
    double s[2] = {0.0, 0.0};
    s[0] = side_dot(m, a.b, W.tax);
    s[1] = side_dot(m, a.b, wy);
    gs.reduce(s);
    bax = s[0];
    bwy_part = (blockIdx.x == 0 && threadIdx.x == 0) ? s[1] : 0.0;
  }
  prof.mark(PROF_INIT);

  while (steps < a.max_steps && (double)S.max_iters > k && !(status > 0.5)) {
    const double wtau = W.w[N - 1];
    const double vtau = W.v[N - 1];
    const double since2 = since + 1.0;
    const bool is_check = since2 > (double)S.check_interval - 0.5;
    const bool last = steps + 1 >= a.max_steps || k + 1.0 >= (double)S.max_iters;
    const bool need_resid = is_check || a.resid_every;
    const int write_u = need_resid || last;

    // -- optional refresh of the tracked products from the warm start:
    //    tax = A cgx, gx = A^T tax, bax = b.tax (they are otherwise carried
    //    through the CG updates and accumulate rounding)
    if (a.refresh > 0 && k > 0.5 && fmod(k, (double)a.refresh) < 0.5) {
      {
        EpiStore st1{W.tax};
        apply_plan<TD>(F, InVec{W.cgx, nullptr, 0.0}, st1, nullptr, gs);
      }
      gs.sync();
      {
        EpiStore st2{W.gx};
        apply_plan<TD>(Aj, InVec{W.tax, nullptr, 0.0}, st2, nullptr, gs);
        double sb[1] = {side_dot(m, a.b, W.tax)};
        gs.reduce(sb);
        bax = sb[0];
      }
    }
    // -- subspace step: rhs = w_x - A^T w_y ; r0 = rhs - (x0 + A^T A x0)
    //    (scs.py:349-357); c.x0 and the b.w_y of the last cone step ride along
    double s[4] = {0.0, 0.0, 0.0, bwy_part};
    {
      InVec in{wy, nullptr, 0.0};
      EpiRhs e{W.w, W.cgx, W.gx, a.c, W.r, wx_stale ? a.g : nullptr, tau_prev, c_lo, c_hi};
      if (a.prof && threadIdx.x == 0) cgb_tl_acc = a.prof + 16;
      apply_plan<TD>(Aj, in, e, s, gs);
      if (a.prof && threadIdx.x == 0) cgb_tl_acc = nullptr;
      gs.reduce(s);
    }
    prof.mark(PROF_RHS);
    const double tol_k = cg_tolerance_graph(k, S);
    const double delta = tol_k * sqrt(s[0]);
    const double floor_ = a.eps_floor * s[0];
    double rns = s[1];
    double cx = s[2];
    const double bwy = s[3];
    CgBufs B{W.cgx, W.r, W.p0, nullptr, W.t, W.tax, W.gx, a.b, a.c, b_lo, b_hi, c_lo, c_hi};
    const int64_t cgk = cg_loop<TD>(F, Aj, CGB_RECIPE_NORMAL, 1.0, B, n, m, rns, delta, floor_,
                                cg_max, gs, &cx, &bax, prof);
    // tau~ = (w_tau + h.p) / (1 + h.g) with h.p = c.p1 + b.(w_y + A p1)
    const double tau_t = (wtau + (cx + (bwy + bax))) / a.denom;

    // -- cone step onto R^n x K* x R+   (scs.py:358-366)
    ConeStep cs{wy, W.tax, a.g + n, W.v + n, W.u + n, W.w + n, a.b, tau_t, write_u};
    double bw = 0.0;
    double red[2 * CGB_MAX_LARGE_SOC];
#pragma unroll
    for (int i = 0; i < 2 * CGB_MAX_LARGE_SOC; ++i) red[i] = 0.0;
    // w_x = u_x = p1 - tau~ g_x: stored only when u is (check / last
    // iteration / trace); otherwise the next rhs epilogue recomputes it
    if (write_u) {
      XStep fx{W.u, W.w, tau_t, write_u};
      const double* src[2] = {W.cgx, a.g};
      bulk_stream<2>(n, src, fx);
    }
    wx_stale = !write_u;
    tau_prev = tau_t;
    if (a.prof) {  // profiling only: separate the sub-phases
      gs.sync();
      prof.mark(PROF_CONE_X);
    }
    // elementwise segments (one pass each)
    for (int sg_i = 0; sg_i < K.nseg; ++sg_i) {
      const DevSeg sg = K.seg[sg_i];
      if (sg.kind == SEG_SOC_LARGE) continue;
      if (sg.end <= b_lo || sg.begin >= b_hi) {  // b == 0 here: no b.w_y term
        ConeElemNoB f{&cs, sg.begin, sg.kind};
        const double* src[4] = {wy + sg.begin, W.tax + sg.begin, a.g + n + sg.begin,
                                W.v + n + sg.begin};
        bulk_stream<4>(sg.end - sg.begin, src, f);
      } else {
        ConeElem f{&cs, sg.begin, sg.kind, 0.0};
        const double* src[5] = {wy + sg.begin, W.tax + sg.begin, a.g + n + sg.begin,
                                W.v + n + sg.begin, a.b + sg.begin};
        bulk_stream<5>(sg.end - sg.begin, src, f);
        bw += f.bw;
      }
    }
    // small SOC blocks: one warp per cone, norm then projection
    {
      const int lane = threadIdx.x & 31;
      const int64_t gw = (int64_t)blockIdx.x + (int64_t)gridDim.x * (threadIdx.x >> 5);
      const int64_t nw = (int64_t)gridDim.x * CGB_WARPS;
      for (int64_t cc = gw; cc < K.nsmall; cc += nw) {
        const int64_t off = K.small_off[cc];
        const int dim = K.small_dim[cc];
        const double t = cs.src(off);
        double nu2 = 0.0;
        for (int i = 1 + lane; i < dim; i += 32) {
          const double z = cs.src(off + i);
          nu2 += z * z;
        }
        nu2 = warp_sum(nu2);
        const SocCoef sc(t, sqrt(nu2));
        __syncwarp();
        for (int i = lane; i < dim; i += 32) {
          const double z = cs.src(off + i);
          bw += a.b[off + i] * cs.store(off + i, z, i == 0 ? sc.head(t) : sc.tail(z));
        }
      }
    }
    // exponential cones: a thread per cone, dual projection
    for (int64_t cc = gtid(); cc < K.nexp; cc += gsize()) {
      const int64_t off = K.exp_off[cc];
      const double z0 = cs.src(off), z1 = cs.src(off + 1), z2 = cs.src(off + 2);
      double p0 = z0, p1 = z1, p2 = z2;
      exp_project_dual(p0, p1, p2);
      bw += a.b[off] * cs.store(off, z0, p0);
      bw += a.b[off + 1] * cs.store(off + 1, z1, p1);
      bw += a.b[off + 2] * cs.store(off + 2, z2, p2);
    }
    if (a.prof) {
      gs.sync();
      prof.mark(PROF_CONE_E);
    }
    // large SOC blocks, pass A: tail sum of squares (+ stash), head from block 0
    {
      int64_t so = 0;
      for (int sg_i = 0; sg_i < K.nseg; ++sg_i) {
        const DevSeg sg = K.seg[sg_i];
        if (sg.kind != SEG_SOC_LARGE) continue;
        const int64_t b0 = sg.begin + 1, len = sg.end - sg.begin - 1;
        const double* src[4] = {wy + b0, W.tax + b0, a.g + n + b0, W.v + n + b0};
        if (use_stash || !a.park) {
          SocPassA f{tau_t, use_stash ? stash_base + so : nullptr, 0.0};
          bulk_stream<4>(len, src, f);
          red[sg.slot] += f.acc;
        } else {
          SocPassAG f{tau_t, a.park + b0, 0.0};
          bulk_stream<4>(len, src, f);
          red[sg.slot] += f.acc;
        }
        so += stream_span(len);
        if (blockIdx.x == 0 && threadIdx.x == 0) red[K.nlarge + sg.slot] += cs.src(sg.begin);
      }
    }
    if (K.nlarge > 0) {
      if (a.prof) {
        gs.sync();
        prof.mark(PROF_CONE_A);
      }
      if (K.nlarge == 1) {  // the common case: reduce just (tail^2, head)
        double r2[2] = {red[0], red[1]};
        gs.reduce(r2);
        red[0] = r2[0];
        red[1] = r2[1];
      } else {
        gs.reduce(red);
      }
      prof.mark(PROF_CONE_AR);
      // pass B: project the large SOC blocks
      int64_t so = 0;
      for (int sg_i = 0; sg_i < K.nseg; ++sg_i) {
        const DevSeg sg = K.seg[sg_i];
        if (sg.kind != SEG_SOC_LARGE) continue;
        const double t = red[K.nlarge + sg.slot];
        const SocCoef sc(t, sqrt(red[sg.slot]));
        const int64_t b0 = sg.begin + 1, len = sg.end - sg.begin - 1;
        if (use_stash) {
          SocPassB f{&cs, b0, sc, stash_base + so, 0.0};
          const double* src[1] = {a.b + b0};
          bulk_stream<1>(len, src, f);
          bw += f.bw;
        } else if (a.park) {
          SocPassBG f{&cs, b0, sc, 0.0};
          const double* src[2] = {a.park + b0, a.b + b0};
          bulk_stream<2>(len, src, f);
          bw += f.bw;
        } else {
          SocPassB2 f{&cs, b0, sc, 0.0};
          const double* src[5] = {wy + b0, W.tax + b0, a.g + n + b0, W.v + n + b0, a.b + b0};
          bulk_stream<5>(len, src, f);
          bw += f.bw;
        }
        so += stream_span(len);
        if (blockIdx.x == 0 && threadIdx.x == 0)
          bw += a.b[sg.begin] * cs.store(sg.begin, t, sc.head(t));
      }
    }
    const double utau = fmax(tau_t - vtau, 0.0);
    const double kappa = (vtau - tau_t) + utau;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      W.u[N - 1] = utau;
      W.v[N - 1] = kappa;
      W.w[N - 1] = utau + kappa;
    }
    bwy_part = bw;
    gs.sync();
    prof.mark(PROF_CONE_B);

    k += 1.0;
    cgt += (double)cgk;
    lastcg = (double)cgk;

    if (need_resid) {
      // -- termination measures (scs.py:369-402)
      double q[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      InVec uxin{W.u, nullptr, 0.0};
      InVec uyin{W.u + n, nullptr, 0.0};
      EpiRawP ep{W.v + n, a.b, utau};
      EpiRawD ed{a.c, utau};
      apply_two<TD>(F, uxin, ep, Aj, uyin, ed, q, gs);
      q[4] = side_dot(n, a.c, W.u);
      q[5] = side_dot(m, a.b, W.u + n);
      gs.reduce(q);
      prof.mark(PROF_CHECK);
      const double eps = S.eps;
      const double pos = utau > 0.0 ? 1.0 : 0.0;
      const double tinv = pos / (utau + (1.0 - pos));
      pr = a.pr_scale * (sqrt(q[0]) * tinv);
      dr = a.dr_scale * (sqrt(q[2]) * tinv);
      const double ctx = q[4], bty = q[5];
      const double sc = ctx * tinv, sb = bty * tinv;
      gap = sqrt((sc + sb) * (sc + sb)) / (1.0 + (sqrt(sc * sc) + sqrt(sb * sb)));
      const double solved = (eps > pr ? 1.0 : 0.0) * (eps > dr ? 1.0 : 0.0) *
                            ((eps > gap ? 1.0 : 0.0) * pos);
      const double max_k1 = fmax(kappa - 1.0, 0.0) + 1.0;
      const double tau_small = (S.cert_tau_ratio * max_k1 > utau) ? 1.0 : 0.0;
      const double den_u = fmax(-1.0 * ctx, 0.0);
      const double pos_u = den_u > 0.0 ? 1.0 : 0.0;
      const double res_u = sqrt(q[1]) / (den_u + (1.0 - pos_u));
      res_u_last = res_u;
      const double unb_ok = pos_u * (eps > res_u ? 1.0 : 0.0);
      const double den_i = fmax(-1.0 * bty, 0.0);
      const double pos_i = den_i > 0.0 ? 1.0 : 0.0;
      const double res_i = sqrt(q[3]) / (den_i + (1.0 - pos_i));
      res_i_last = res_i;
      const double inf_ok = pos_i * (eps > res_i ? 1.0 : 0.0);
      const double cert = tau_small * (2.0 * inf_ok + (1.0 - inf_ok) * (3.0 * unb_ok));
      const double cand = solved + (1.0 - solved) * cert;
      if (is_check) {
        const double not_set = 1.0 - (status > 0.5 ? 1.0 : 0.0);
        status = status + not_set * cand;
      }
    }
    since = is_check ? 0.0 : since2;
    ++steps;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    state[CGB_ST_K] = k;
    state[CGB_ST_SINCE] = since;
    state[CGB_ST_STATUS] = status;
    state[CGB_ST_CGT] = cgt;
    state[CGB_ST_PR] = pr;
    state[CGB_ST_DR] = dr;
    state[CGB_ST_GAP] = gap;
    state[CGB_ST_LASTCG] = lastcg;
    state[CGB_ST_RES_U] = res_u_last;
    state[CGB_ST_RES_I] = res_i_last;
  }
}
#else
;
#endif

struct BarArgs {
  GridBar* bar; double* partials;
  int64_t iters; int mode; double* out;
};

// diagnostics: cost of the grid barrier / grid reduction
__global__ void __launch_bounds__(CGB_BLOCK, CGB_MINB) k_barrier(const __grid_constant__ BarArgs a) 
#if CGB_TU_MISC
{
  GridSync gs(a.bar, a.partials);
  double acc = 0.0;
  for (int64_t i = 0; i < a.iters; ++i) {
    if (a.mode == 0) {
      gs.sync();
    } else if (a.mode == 1) {
      double v[1] = {1.0};
      gs.reduce(v);
      acc += v[0];
    } else if (a.mode == 2) {
      double v[4] = {1.0, 2.0, 3.0, 4.0};
      gs.reduce(v);
      acc += v[0] + v[3];
    } else if (a.mode == 3) {
      double v[8] = {1.0, 2.0, 3.0, 4.0, 5.0, 6.0, 7.0, 8.0};
      gs.reduce(v);
      acc += v[0] + v[7];
    } else if (a.mode == 4) {
      gs.sync<1>();
    } else {
      gs.sync<0>();
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) a.out[0] = acc;
}
#else
;
#endif


#include "cgb_shard_kernel.cuh"

// explicit instantiations, one group per translation unit
#if CGB_TU_SCS0
template __global__ void k_scs<0>(const __grid_constant__ ScsArgs);
#endif
#if CGB_TU_SCS1
template __global__ void k_scs<1>(const __grid_constant__ ScsArgs);
#endif
#if CGB_TU_SCS2
template __global__ void k_scs<2>(const __grid_constant__ ScsArgs);
#endif
#if CGB_TU_CG
template __global__ void k_cg<0>(const __grid_constant__ CgArgs);
template __global__ void k_cg<1>(const __grid_constant__ CgArgs);
#endif
#if CGB_TU_INNER
template __global__ void k_inner<0>(const __grid_constant__ InnerArgs);
template __global__ void k_inner<1>(const __grid_constant__ InnerArgs);
#endif
#if CGB_TU_SHARD
template __global__ void k_shard<0>(const __grid_constant__ ShardArgs);
#endif
#if CGB_TU_MISC
template __global__ void k_apply<0>(const __grid_constant__ ApplyArgs);
template __global__ void k_apply<1>(const __grid_constant__ ApplyArgs);
#endif

}  // namespace cgbk
using namespace cgbk;

#if CGB_TU_HOST

// ===========================================================================
// host side
// ===========================================================================
namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                              \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess)                                                          \
      return fail(CGB_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));   \
  } while (0)

}  // namespace

struct cgb_ctx {
  int device;
  int num_sms;
  int max_grid;
  GridBar* bar;
  double* partials;  // 2 banks * CGB_MAXP * max_grid
  double* result;    // small device result buffer
  double* host_result;
  double* prof;      // k_scs phase accumulator (device, PROF_N doubles) or null
  int grid_override; // CGB_GRID (experiments): fewer CTAs than SMs, 0 = off
  // launch ordering: every launch on this ctx follows the previous one
  std::mutex mu;            // host threads
  cudaStream_t last = nullptr;
  bool has_last = false;
  cudaEvent_t order_ev = nullptr;
};

struct PlanStore {
  DevPlan dp{};
  void* blob = nullptr;     // device allocation holding all arrays
  double* temps = nullptr;  // 2 * temp_total
  int64_t temp_total = 0;
  int64_t in_len = 0, out_len = 0;
  int64_t leaf_bytes = 0;   // operand bytes of one apply (cluster-mode choice)
  bool has_dense = false;   // a dense leaf: the solver runs its MODE 2 instantiation
};

struct cgb_op {
  PlanStore fwd, adj;
  const cgb_ctx* ctx = nullptr;
};

struct cgb_cones {
  const cgb_ctx* ctx = nullptr;
  bool sharded = false;      // pieces of a row-sharded problem (k_shard only)
  DevCones dc{};
  void* blob = nullptr;
  int64_t m = 0;
  std::vector<DevSeg> segs;  // host copy (stash sizing)
};

namespace {

size_t plan_smem(const DevPlan& P) { return sizeof(double) * (size_t)P.smem_total; }

// dynamic shared memory of a solver kernel: the plans' conv staging
size_t solver_smem(const DevPlan& F, const DevPlan& Aj) {
  return std::max(plan_smem(F), plan_smem(Aj));
}

template <class K>
int grid_for(const cgb_ctx* ctx, K kernel, size_t smem, int* grid) {
  CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)std::max<size_t>(smem, 1)));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, CGB_BLOCK, smem));
  if (per_sm < 1)
    return fail(CGB_ECOOP, "kernel cannot be resident (threads/registers/shared memory)");
  // one CTA per SM: the persistent kernels size every loop to the grid
  int g = std::min(ctx->num_sms * std::min(per_sm, CGB_CTAS_PER_SM), CGB_MAXG);
  if (ctx->grid_override > 0) g = std::min(g, ctx->grid_override);
  *grid = g;
  return CGB_OK;
}

// Order this launch after the ctx's previous one (the grid barrier, the
// reduction banks and the plan temporaries are per ctx).  Caller holds mu.
int order_after_last(cgb_ctx* ctx, cudaStream_t stream) {
  if (ctx->has_last && ctx->last != stream) {
    CUDA_TRY(cudaEventRecord(ctx->order_ev, ctx->last));
    CUDA_TRY(cudaStreamWaitEvent(stream, ctx->order_ev, 0));
  }
  ctx->last = stream;
  ctx->has_last = true;
  return CGB_OK;
}

// Cluster mode: the persistent kernel as ONE thread-block cluster of up to
// 16 CTAs, the grid barrier replaced by the hardware cluster barrier.
// Measured on configs[0] (dense lasso 1000 x 500): 264 us per iteration vs
// 260 us on the full cooperative grid -- the phases there are bound by
// their dependent-load latency, not by the barrier, and 16 SMs stretch
// each phase's work -- so it is opt-in: CGB_CLUSTER=N (N = 2..16) for
// problems with n + m <= 200000 and <= 64 MB of operator data.
int cluster_size_for(int64_t n, int64_t m, int64_t work_bytes) {
  const char* env = std::getenv("CGB_CLUSTER");
  if (!env) return 0;
  const int c = std::atoi(env);
  if (c <= 1 || n + m > 200000 || work_bytes > (64ll << 20)) return 0;
  return std::min(c, 16);
}

template <class K, class A>
int launch_cluster(cgb_ctx* ctx, K kernel, A& args, size_t smem, cudaStream_t stream, int csize) {
  CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)std::max<size_t>(smem, 1)));
  if (csize > 8)
    CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(csize);
  cfg.blockDim = dim3(CGB_BLOCK);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, (void*)kernel, &cfg) != cudaSuccess ||
      nclusters < 1) {
    cudaGetLastError();
    return -1;  // not placeable: the caller falls back to the cooperative grid
  }
  int rc = order_after_last(ctx, stream);
  if (rc) return rc;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, args);
  if (e != cudaSuccess)
    return fail(CGB_ECOOP, std::string("cluster launch failed: ") + cudaGetErrorString(e));
  return CGB_OK;
}

template <class K, class A>
int launch_coop(cgb_ctx* ctx, K kernel, A& args, size_t smem, cudaStream_t stream,
                int csize = 0) {
  for (; csize > 1; csize /= 2) {       // 16, then 8 if 16 SMs of one GPC are not free
    const int rc = launch_cluster(ctx, kernel, args, smem, stream, csize);
    if (rc != -1) return rc;
  }
  int grid = 0;
  int rc = grid_for(ctx, kernel, smem, &grid);
  if (rc) return rc;
  if (grid > CGB_MAXG) return fail(CGB_ECOOP, "grid larger than CGB_MAXG");
  rc = order_after_last(ctx, stream);
  if (rc) return rc;
  // the grid barrier counts arrivals from zero in every launch
  CUDA_TRY(cudaMemsetAsync(&ctx->bar->count, 0, sizeof(unsigned long long), stream));
  void* params[] = {&args};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)kernel, dim3(grid), dim3(CGB_BLOCK),
                                              params, smem, stream);
  if (e != cudaSuccess)
    return fail(CGB_ECOOP, std::string("cooperative launch failed: ") + cudaGetErrorString(e));
  return CGB_OK;
}

struct Blob {
  std::vector<char> host;
  // copy `bytes` from p (may be null when bytes == 0); reserve at least 16 bytes
  size_t add(const void* p, size_t bytes) {
    size_t off = (host.size() + 255) & ~size_t(255);
    host.resize(off + std::max<size_t>(bytes, 16));
    if (bytes && p) std::memcpy(host.data() + off, p, bytes);
    return off;
  }
};

// doubles of dynamic shared memory of the 2-d strips for a kh-row kernel:
// the row ring (kh + 2 RPS - 1 slots) and, per warp, the transpose buffer
// and its t buffers (two when a warp has one row per step)
int64_t strip_smem(int64_t kh, int64_t slot) {
  const int64_t tb = CGB_STRIP_RPW == 1 ? 2 : CGB_STRIP_RPW;
  return (kh + 2 * CGB_STRIP_RPS - 1) * slot + CGB_WARPS * (tb * slot + 32 * CGB_RC + 2);
}

int build_plan(const cgb_plan_desc* d, PlanStore* ps) {
  if (!d) return fail(CGB_EINVAL, "null plan descriptor");
  if (d->nleaves < 0 || d->nterms < 0 || d->nrowblocks < 1 || d->ntemps < 0)
    return fail(CGB_EINVAL, "plan: bad counts");
  std::vector<int64_t> buf_len(d->ntemps + 1);
  buf_len[0] = d->out_len;
  int64_t temp_total = 0;
  std::vector<int64_t> temp_off(d->ntemps);
  for (int t = 0; t < d->ntemps; ++t) {
    if (d->temp_len[t] < 0) return fail(CGB_EINVAL, "plan: negative temp length");
    buf_len[t + 1] = d->temp_len[t];
    temp_off[t] = temp_total;
    temp_total += d->temp_len[t];
  }
  std::vector<int64_t> in_len(d->ntemps + 1);
  in_len[0] = d->in_len;
  for (int t = 0; t < d->ntemps; ++t) in_len[t + 1] = d->temp_len[t];
  // leaves
  for (int i = 0; i < d->nleaves; ++i) {
    const cgb_leaf& L = d->leaves[i];
    switch (L.kind) {
      case CGB_LEAF_IDENTITY:
        if (L.rows != L.cols) return fail(CGB_EINVAL, "identity leaf not square");
        break;
      case CGB_LEAF_DENSE:
        if (!L.val || L.ld < L.cols) return fail(CGB_EINVAL, "dense leaf: bad data/ld");
        break;
      case CGB_LEAF_CSR:
        if (!L.val || !L.rowptr || !L.colidx) return fail(CGB_EINVAL, "csr leaf: null arrays");
        break;
      case CGB_LEAF_CONV1D:
        if (!L.val || L.k0 < 1 || L.n0 < 1 || L.rows != L.n0 + L.k0 - 1 || L.cols != L.n0)
          return fail(CGB_EINVAL, "conv1d leaf: inconsistent shape");
        break;
      case CGB_LEAF_CORR1D:
        if (!L.val || L.k0 < 1 || L.n0 < 1 || L.cols != L.n0 + L.k0 - 1 || L.rows != L.n0)
          return fail(CGB_EINVAL, "corr1d leaf: inconsistent shape");
        break;
      case CGB_LEAF_CONV2D:
        if (!L.val || L.rows != (L.n0 + L.k0 - 1) * (L.n1 + L.k1 - 1) || L.cols != L.n0 * L.n1)
          return fail(CGB_EINVAL, "conv2d leaf: inconsistent shape");
        break;
      case CGB_LEAF_CORR2D:
        if (!L.val || L.cols != (L.n0 + L.k0 - 1) * (L.n1 + L.k1 - 1) || L.rows != L.n0 * L.n1)
          return fail(CGB_EINVAL, "corr2d leaf: inconsistent shape");
        break;
      default:
        return fail(CGB_EINVAL, "unknown leaf kind " + std::to_string(L.kind));
    }
  }
  for (int i = 0; i < d->nterms; ++i) {
    const cgb_term& T = d->terms[i];
    if (T.leaf < 0 || T.leaf >= d->nleaves) return fail(CGB_EINVAL, "term: bad leaf index");
    if (T.in_buf < 0 || T.in_buf > d->ntemps) return fail(CGB_EINVAL, "term: bad input buffer");
    const cgb_leaf& L = d->leaves[T.leaf];
    if (T.in_off < 0 || T.in_off + L.cols > in_len[T.in_buf])
      return fail(CGB_EINVAL, "term: input range out of bounds");
  }
  // rowblocks: validate coverage, order by execution level
  int maxlevel = 0;
  for (int i = 0; i < d->nrowblocks; ++i) maxlevel = std::max(maxlevel, d->rowblocks[i].level);
  const int nlevels = maxlevel + 1;
  std::vector<std::vector<std::pair<int64_t, int64_t>>> cover(d->ntemps + 1);
  std::vector<int> buf_level(d->ntemps + 1, -1);
  for (int i = 0; i < d->nrowblocks; ++i) {
    const cgb_rowblock& R = d->rowblocks[i];
    if (R.out_buf < 0 || R.out_buf > d->ntemps) return fail(CGB_EINVAL, "rowblock: bad buffer");
    if (R.level < 0) return fail(CGB_EINVAL, "rowblock: negative level");
    if (R.out_buf == 0 && R.level != 0) return fail(CGB_EINVAL, "rowblock: output not at level 0");
    if (buf_level[R.out_buf] >= 0 && buf_level[R.out_buf] != R.level)
      return fail(CGB_EINVAL, "rowblock: buffer written at two levels");
    buf_level[R.out_buf] = R.level;
    if (R.row_begin < 0 || R.row_end <= R.row_begin || R.row_end > buf_len[R.out_buf])
      return fail(CGB_EINVAL, "rowblock: bad row range");
    if (R.term_begin < 0 || R.term_end < R.term_begin || R.term_end > d->nterms)
      return fail(CGB_EINVAL, "rowblock: bad term range");
    for (int t = R.term_begin; t < R.term_end; ++t) {
      const cgb_term& T = d->terms[t];
      const cgb_leaf& L = d->leaves[T.leaf];
      if (R.row_begin < T.row_origin || R.row_end > T.row_origin + L.rows)
        return fail(CGB_EINVAL, "rowblock: term does not cover its rows");
      if (T.in_buf > 0 && buf_level[T.in_buf] >= 0 && buf_level[T.in_buf] <= R.level)
        return fail(CGB_EINVAL, "rowblock: reads a temporary not produced earlier");
    }
    cover[R.out_buf].push_back({R.row_begin, R.row_end});
  }
  for (int b = 0; b <= d->ntemps; ++b) {
    auto& c = cover[b];
    std::sort(c.begin(), c.end());
    int64_t pos = 0;
    for (auto& iv : c) {
      if (iv.first != pos) return fail(CGB_EINVAL, "rowblocks do not tile buffer " + std::to_string(b));
      pos = iv.second;
    }
    if (pos != buf_len[b] && !(buf_len[b] == 0 && c.empty()))
      return fail(CGB_EINVAL, "rowblocks do not cover buffer " + std::to_string(b));
  }
  // temps read by a term must be produced at a deeper level (re-check now levels known)
  for (int i = 0; i < d->nrowblocks; ++i) {
    const cgb_rowblock& R = d->rowblocks[i];
    for (int t = R.term_begin; t < R.term_end; ++t) {
      const cgb_term& T = d->terms[t];
      if (T.in_buf > 0 && buf_len[T.in_buf] > 0 && buf_level[T.in_buf] <= R.level)
        return fail(CGB_EINVAL, "rowblock: temporary consumed before it is produced");
    }
  }
  std::vector<int> order(d->nrowblocks);
  for (int i = 0; i < d->nrowblocks; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
    return d->rowblocks[x].level > d->rowblocks[y].level;  // deepest first
  });
  std::vector<DevRowBlock> rbs(d->nrowblocks);
  const int64_t kLongBlock = 32 * CGB_RC * 256;
  int64_t kw2max = 0;  // widest 2-d kernel row of a periodic (tiled) block
  std::vector<int32_t> level_rb(nlevels + 1, 0);
  std::vector<int64_t> level_tiles(nlevels, 0);
  int64_t kmax = 0;
  int idx = 0;
  for (int e = 0; e < nlevels; ++e) {
    const int lvl = nlevels - 1 - e;
    level_rb[e] = idx;
    int64_t tiles = 0;
    while (idx < d->nrowblocks && d->rowblocks[order[idx]].level == lvl) {
      const cgb_rowblock& R = d->rowblocks[order[idx]];
      DevRowBlock& D = rbs[idx];
      D.row_begin = R.row_begin;
      D.row_end = R.row_end;
      D.tile_begin = tiles;
      D.out_buf = R.out_buf;
      D.term_begin = R.term_begin;
      D.term_end = R.term_end;
      D.rfac = 1;
      D.conv_term = -1;
      D.period = 0;
      D.tpr = 0;
      int nconv = 0;
      for (int t = R.term_begin; t < R.term_end; ++t) {
        const cgb_leaf& LF = d->leaves[d->terms[t].leaf];
        if ((LF.kind == CGB_LEAF_CONV1D || LF.kind == CGB_LEAF_CORR1D) &&
            LF.k0 <= CGB_CONV_KMAX) {
          D.rfac = CGB_RC;
          kmax = std::max<int64_t>(kmax, LF.k0);
          ++nconv;
          D.conv_term = t;
        }
      }
      if (nconv != 1) D.conv_term = -1;  // TMA staging for a single conv term only
      // long blocks of elementwise / sparse terms: RC rows per lane too, so a
      // tile carries enough work to amortise its setup (dense leaves keep a
      // warp per row and R = 1)
      if (D.rfac == 1 && R.row_end - R.row_begin >= kLongBlock) {
        bool dense = false;
        for (int t = R.term_begin; t < R.term_end; ++t)
          dense |= d->leaves[d->terms[t].leaf].kind == CGB_LEAF_DENSE;
        if (!dense) D.rfac = CGB_RC;
      }
      // 2-d conv terms: whole output rows of one width -> periodic tiles that
      // never cross a row (the tiled 2-d path needs a tile inside one row)
      int64_t period = 0;
      bool periodic_ok = true;
      for (int t = R.term_begin; t < R.term_end; ++t) {
        const cgb_term& T = d->terms[t];
        const cgb_leaf& LF = d->leaves[T.leaf];
        if (LF.kind != CGB_LEAF_CONV2D && LF.kind != CGB_LEAF_CORR2D) continue;
        const int64_t ow = LF.kind == CGB_LEAF_CONV2D ? LF.n1 + LF.k1 - 1 : LF.n1;
        if (LF.k1 > CGB_CONV_KMAX || (period && ow != period) ||
            (R.row_begin - T.row_origin) % ow != 0 || (R.row_end - R.row_begin) % ow != 0)
          periodic_ok = false;
        period = ow;
        kw2max = std::max<int64_t>(kw2max, LF.k1);
      }
      bool has_dense = false;
      for (int t = R.term_begin; t < R.term_end; ++t)
        has_dense |= d->leaves[d->terms[t].leaf].kind == CGB_LEAF_DENSE;
      D.rpt = 32 * D.rfac;
      D.strip_term = -1;
      if (period > 0 && periodic_ok) {
        D.rfac = CGB_RC;
        D.rpt = 32 * CGB_RC;
        D.period = period;
        D.tpr = (int32_t)((period + 32 * CGB_RC - 1) / (32 * CGB_RC));
        tiles += (R.row_end - R.row_begin) / period * D.tpr;
      } else {
        // dense (GEMV) blocks: a warp per 8 rows, so short-wide matrices
        // spread over many warps (the rows' loads of a tile are in flight
        // together; see leaf_tile)
        if (has_dense && D.rfac == 1) D.rpt = 8;
        tiles += (R.row_end - R.row_begin + D.rpt - 1) / D.rpt;
      }
      ++idx;
    }
    level_tiles[e] = tiles;
  }
  level_rb[nlevels] = idx;
  // correlation taps of the tiled 1-d conv leaves (reversed for conv)
  std::vector<int32_t> leaf_taps(std::max(1, d->nleaves), -1);
  std::vector<double> taps;
  std::vector<cgb_leaf> leaves(d->leaves, d->leaves + d->nleaves);
  for (int i = 0; i < d->nleaves; ++i) {
    cgb_leaf& L = leaves[i];
    const bool is2d = L.kind == CGB_LEAF_CONV2D || L.kind == CGB_LEAF_CORR2D;
    if (!is2d) L.reserved = 0;
    if (is2d && (L.reserved & CGB_LEAF_FLAG_SEPARABLE) && L.k1 <= CGB_SEP_KMAX &&
        L.k0 + (L.k1 + CGB_RC - 1) / CGB_RC * CGB_RC <= 4096) {
      // rank-one factorization through the largest entry (a*, b*):
      // u[a] = K[a, b*], v[b] = K[a*, b] / K[a*, b*]; kept only if it
      // reproduces every entry to a few ulp of max |K|
      std::vector<double> kv(L.k0 * L.k1);
      CUDA_TRY(cudaMemcpy(kv.data(), L.val, sizeof(double) * kv.size(), cudaMemcpyDeviceToHost));
      int64_t pa = 0, pb = 0;
      double pmax = 0.0;
      for (int64_t a = 0; a < L.k0; ++a)
        for (int64_t b = 0; b < L.k1; ++b)
          if (std::fabs(kv[a * L.k1 + b]) > pmax) { pmax = std::fabs(kv[a * L.k1 + b]); pa = a; pb = b; }
      std::vector<double> u(L.k0), v(L.k1);
      bool ok = pmax > 0.0;
      if (ok) {
        for (int64_t a = 0; a < L.k0; ++a) u[a] = kv[a * L.k1 + pb];
        for (int64_t b = 0; b < L.k1; ++b) v[b] = kv[pa * L.k1 + b] / kv[pa * L.k1 + pb];
        for (int64_t a = 0; a < L.k0 && ok; ++a)
          for (int64_t b = 0; b < L.k1 && ok; ++b)
            ok = std::fabs(kv[a * L.k1 + b] - u[a] * v[b]) <= 8.0 * DBL_EPSILON * pmax;
      }
      if (ok) {
        const int64_t nt = (L.k1 + CGB_RC - 1) / CGB_RC * CGB_RC;
        leaf_taps[i] = (int32_t)taps.size();
        for (int64_t j = 0; j < nt; ++j)
          taps.push_back(j < L.k1 ? v[L.kind == CGB_LEAF_CONV2D ? L.k1 - 1 - j : j] : 0.0);
        for (int64_t a = 0; a < L.k0; ++a) taps.push_back(u[a]);
        continue;
      }
    }
    L.reserved = 0;
    if ((L.kind == CGB_LEAF_CONV1D || L.kind == CGB_LEAF_CORR1D) && L.k0 <= CGB_CONV_KMAX) {
      std::vector<double> kv(L.k0);
      CUDA_TRY(cudaMemcpy(kv.data(), L.val, sizeof(double) * L.k0, cudaMemcpyDeviceToHost));
      const int64_t nt = (L.k0 + CGB_RC - 1) / CGB_RC * CGB_RC;
      leaf_taps[i] = (int32_t)taps.size();
      for (int64_t j = 0; j < nt; ++j)
        taps.push_back(j < L.k0 ? kv[L.kind == CGB_LEAF_CONV1D ? L.k0 - 1 - j : j] : 0.0);
    }
    if ((L.kind == CGB_LEAF_CONV2D || L.kind == CGB_LEAF_CORR2D) && L.k1 <= CGB_CONV_KMAX &&
        L.k0 * ((L.k1 + CGB_RC - 1) / CGB_RC * CGB_RC) <= 4096) {
      // one correlation row per kernel row a (reversed for the full conv)
      std::vector<double> kv(L.k0 * L.k1);
      CUDA_TRY(cudaMemcpy(kv.data(), L.val, sizeof(double) * kv.size(), cudaMemcpyDeviceToHost));
      const int64_t nt = (L.k1 + CGB_RC - 1) / CGB_RC * CGB_RC;
      leaf_taps[i] = (int32_t)taps.size();
      for (int64_t a = 0; a < L.k0; ++a)
        for (int64_t j = 0; j < nt; ++j)
          taps.push_back(j < L.k1 ? kv[a * L.k1 + (L.kind == CGB_LEAF_CONV2D ? L.k1 - 1 - j : j)]
                                  : 0.0);
    }
  }
  // 2-d conv row blocks as CTA strips (run_strips): a periodic block whose
  // only 2-d term has device taps and whose other terms are identity /
  // sparse / dense; the CTA ring of kh + 15 input-row slots overlays the
  // per-warp buffers.  CGB_STRIP=0 disables (A/B), CGB_STRIP_ROWS sets the
  // output rows per task.
  int32_t strip_slot = 0, strip_nslot = 0, strip_rows = 0;
  {
    const char* env = std::getenv("CGB_STRIP");
    const bool allow = !(env && env[0] == '0');
    int64_t khmax = 0, ntmax = 0;
    for (size_t i = 0; i < rbs.size() && allow; ++i) {
      DevRowBlock& D = rbs[i];
      if (D.period <= 0) continue;
      int n2 = 0, t2 = -1;
      bool others_ok = true;
      for (int t = D.term_begin; t < D.term_end; ++t) {
        const cgb_leaf& LF = leaves[d->terms[t].leaf];
        if (LF.kind == CGB_LEAF_CONV2D || LF.kind == CGB_LEAF_CORR2D) {
          ++n2;
          t2 = t;
        } else if (LF.kind != CGB_LEAF_IDENTITY && LF.kind != CGB_LEAF_CSR &&
                   LF.kind != CGB_LEAF_DENSE) {
          others_ok = false;
        }
      }
      if (n2 != 1 || !others_ok || leaf_taps[d->terms[t2].leaf] < 0) continue;
      const cgb_leaf& LF = leaves[d->terms[t2].leaf];
      const int64_t nt = (LF.k1 + CGB_RC - 1) / CGB_RC * CGB_RC;
      const int64_t slot = (32 * CGB_RC + nt + 2 + 1) & ~1;
      const int64_t need = strip_smem(LF.k0, slot);
      if (need > 24 * 1024) continue;  // 192 KB of shared memory at most
      D.strip_term = t2;
      khmax = std::max<int64_t>(khmax, LF.k0);
      ntmax = std::max<int64_t>(ntmax, nt);
    }
    const int64_t slot_all = (32 * CGB_RC + ntmax + 2 + 1) & ~1;
    if (khmax > 0 && strip_smem(khmax, slot_all) > 24 * 1024) {
      for (DevRowBlock& D : rbs) D.strip_term = -1;   // several kernels: over budget together
      khmax = 0;
    }
    if (khmax > 0) {
      strip_slot = (int32_t)((32 * CGB_RC + ntmax + 2 + 1) & ~1);
      strip_nslot = (int32_t)(khmax + 2 * CGB_STRIP_RPS - 1);
      int rows = 4 * CGB_STRIP_RPS;
      if (const char* er = std::getenv("CGB_STRIP_ROWS"))
        rows = std::max(CGB_STRIP_RPS, std::atoi(er) / CGB_STRIP_RPS * CGB_STRIP_RPS);
      strip_rows = rows;
    }
  }
  Blob blob;
  size_t o_leaves = blob.add(leaves.data(), sizeof(cgb_leaf) * d->nleaves);
  size_t o_terms = blob.add(d->terms, sizeof(cgb_term) * d->nterms);
  size_t o_rbs = blob.add(rbs.data(), sizeof(DevRowBlock) * rbs.size());
  size_t o_lrb = blob.add(level_rb.data(), sizeof(int32_t) * level_rb.size());
  size_t o_lt = blob.add(level_tiles.data(), sizeof(int64_t) * level_tiles.size());
  size_t o_to = blob.add(temp_off.data(), sizeof(int64_t) * temp_off.size());
  size_t o_lta = blob.add(leaf_taps.data(), sizeof(int32_t) * leaf_taps.size());
  size_t o_taps = blob.add(taps.data(), sizeof(double) * taps.size());
  char* dev = nullptr;
  CUDA_TRY(cudaMalloc(&dev, blob.host.size() + 256));
  CUDA_TRY(cudaMemcpy(dev, blob.host.data(), blob.host.size(), cudaMemcpyHostToDevice));
  ps->blob = dev;
  if (temp_total > 0) {
    CUDA_TRY(cudaMalloc(&ps->temps, sizeof(double) * 2 * temp_total));
  }
  ps->temp_total = temp_total;
  DevPlan& P = ps->dp;
  P.leaves = (const cgb_leaf*)(dev + o_leaves);
  P.terms = (const cgb_term*)(dev + o_terms);
  P.rbs = (const DevRowBlock*)(dev + o_rbs);
  P.level_rb = (const int32_t*)(dev + o_lrb);
  P.level_tiles = (const int64_t*)(dev + o_lt);
  P.temp_off = (const int64_t*)(dev + o_to);
  P.leaf_taps = (const int32_t*)(dev + o_lta);
  P.taps = (const double*)(dev + o_taps);
  P.meta = dev;
  P.meta_bytes = (int32_t)std::min<size_t>(blob.host.size(), INT32_MAX);
  P.temp[0] = ps->temps;
  P.temp[1] = ps->temps ? ps->temps + temp_total : nullptr;
  P.nlevels = nlevels;

  // per warp: 1-d window buffers 0 and 1 | output transpose | 2-d row ring
  P.smem_cc = 0;
  P.smem_xs = 0;
  P.smem_xs2 = 0;
  P.smem_per_warp = 0;
  if (kmax > 0) {
    const int64_t ntaps = (kmax + CGB_RC - 1) / CGB_RC * CGB_RC;
    P.smem_xs = (int32_t)((32 * CGB_RC + ntaps + 2 + 1) & ~1);
  }
  if (kw2max > 0) {
    const int64_t ntaps = (kw2max + CGB_RC - 1) / CGB_RC * CGB_RC;
    P.smem_xs2 = (int32_t)((32 * CGB_RC + ntaps + 2 + 1) & ~1);
  }
  if (kmax > 0 || kw2max > 0)
    P.smem_per_warp = 2 * P.smem_xs + (32 * CGB_RC + 2) + CGB_RING2 * P.smem_xs2;
  P.strip_slot = strip_slot;
  P.strip_nslot = strip_nslot;
  P.strip_rows = strip_rows;
  P.smem_total = CGB_WARPS * P.smem_per_warp;
  if (P.strip_rows > 0)
    P.smem_total = std::max<int32_t>(
        P.smem_total, (int32_t)strip_smem(P.strip_nslot - 2 * CGB_STRIP_RPS + 1, P.strip_slot));
  P.in_len = d->in_len;
  P.out_len = d->out_len;
  ps->in_len = d->in_len;
  ps->out_len = d->out_len;
  ps->leaf_bytes = 0;
  ps->has_dense = false;
  for (const cgb_leaf& L : leaves) {
    if (L.kind == CGB_LEAF_DENSE) ps->leaf_bytes += 8 * L.rows * L.cols;
    if (L.kind == CGB_LEAF_DENSE) ps->has_dense = true;
    if (L.kind == CGB_LEAF_CSR) {
      int64_t nnz = 0;
      CUDA_TRY(cudaMemcpy(&nnz, L.rowptr + L.rows, sizeof(int64_t), cudaMemcpyDeviceToHost));
      ps->leaf_bytes += 12 * nnz;
    }
  }
  return CGB_OK;
}

void free_plan(PlanStore* ps) {
  if (ps->blob) cudaFree(ps->blob);
  if (ps->temps) cudaFree(ps->temps);
  ps->blob = nullptr;
  ps->temps = nullptr;
}

double eps_floor_for(int64_t n) {
  return DBL_EPSILON * DBL_EPSILON * (double)std::max<int64_t>(n, 1);  // cg.py:100
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int cgb_abi_version(void) { return CGB_ABI_VERSION; }

const char* cgb_last_error(void) { return g_err.c_str(); }

int cgb_ctx_create(int device, cgb_ctx** out) {
  if (!out) return fail(CGB_EINVAL, "null out");
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count <= device || device < 0)
    return fail(CGB_ENODEV, "no CUDA device " + std::to_string(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(CGB_ENODEV, std::string("device is not sm_100 class: ") + prop.name);
  if (!prop.cooperativeLaunch) return fail(CGB_ECOOP, "device lacks cooperative launch");
  CUDA_TRY(cudaSetDevice(device));
  cgb_ctx* c = new cgb_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  if (const char* env = std::getenv("CGB_GRID")) c->grid_override = std::atoi(env);
  c->max_grid = prop.multiProcessorCount * 4;
  if (cudaMalloc(&c->bar, sizeof(GridBar)) != cudaSuccess ||
      cudaMalloc(&c->partials, sizeof(double) * 2 * CGB_MAXP * c->max_grid) != cudaSuccess ||
      cudaMalloc(&c->result, sizeof(double) * 16) != cudaSuccess) {
    delete c;
    return fail(CGB_ENOMEM, "ctx allocation failed");
  }
  cudaMemset(c->bar, 0, sizeof(GridBar));
  cudaMemset(c->partials, 0, sizeof(double) * 2 * CGB_MAXP * c->max_grid);
  cudaMallocHost(&c->host_result, sizeof(double) * 16);
  if (cudaEventCreateWithFlags(&c->order_ev, cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return fail(CGB_ECUDA, "ctx event creation failed");
  }
  CUDA_TRY(cudaDeviceSynchronize());
  *out = c;
  return CGB_OK;
}

int cgb_ctx_destroy(cgb_ctx* ctx) {
  if (!ctx) return CGB_OK;
  cudaFree(ctx->bar);
  cudaFree(ctx->partials);
  cudaFree(ctx->result);
  cudaFreeHost(ctx->host_result);
  if (ctx->order_ev) cudaEventDestroy(ctx->order_ev);
  delete ctx;
  return CGB_OK;
}

int cgb_ctx_geometry(const cgb_ctx* ctx, int32_t* out3) {
  if (!ctx || !out3) return fail(CGB_EINVAL, "null argument");
  int grid = 0;
  int rc = grid_for(ctx, k_scs<0>, 0, &grid);
  if (rc) return rc;
  out3[0] = ctx->num_sms;
  out3[1] = grid / ctx->num_sms;
  out3[2] = CGB_BLOCK;
  return CGB_OK;
}

int cgb_op_create(cgb_ctx* ctx, const cgb_plan_desc* fwd, const cgb_plan_desc* adj,
                  cgb_op** out) {
  if (!ctx || !out) return fail(CGB_EINVAL, "null argument");
  *out = nullptr;
  if (!fwd || !adj || fwd->in_len != adj->out_len || fwd->out_len != adj->in_len)
    return fail(CGB_EINVAL, "forward/adjoint plan shapes disagree");
  cgb_op* op = new cgb_op();
  op->ctx = ctx;
  int rc = build_plan(fwd, &op->fwd);
  if (rc == CGB_OK) rc = build_plan(adj, &op->adj);
  if (rc != CGB_OK) {
    free_plan(&op->fwd);
    free_plan(&op->adj);
    delete op;
    return rc;
  }
  *out = op;
  return CGB_OK;
}

int cgb_op_destroy(cgb_op* op) {
  if (!op) return CGB_OK;
  free_plan(&op->fwd);
  free_plan(&op->adj);
  delete op;
  return CGB_OK;
}

int cgb_op_apply(cgb_ctx* ctx, const cgb_op* op, int adjoint, const double* x, double* y,
                 void* stream) {
  if (!ctx || !op || !x || !y) return fail(CGB_EINVAL, "null argument");
  if (op->ctx != ctx) return fail(CGB_EINVAL, "operator belongs to another ctx");
  std::lock_guard<std::mutex> lk(ctx->mu);
  ApplyArgs a{ctx->bar, ctx->partials, adjoint ? op->adj.dp : op->fwd.dp, x, y};
  if (a.P.smem_xs2 > 0) return launch_coop(ctx, k_apply<1>, a, plan_smem(a.P), (cudaStream_t)stream);
  return launch_coop(ctx, k_apply<0>, a, plan_smem(a.P), (cudaStream_t)stream);
}

int cgb_cones_create(cgb_ctx* ctx, const int32_t* kinds, const int64_t* dims, int32_t ncones,
                     cgb_cones** out) {
  if (!ctx || !out || ncones < 1 || !kinds || !dims) return fail(CGB_EINVAL, "bad cone spec");
  *out = nullptr;
  std::vector<DevSeg> segs;
  std::vector<int64_t> small_off, exp_off;
  std::vector<int32_t> small_dim;
  int nlarge = 0;
  int64_t off = 0;
  const int64_t kSmallMax = 4096;
  for (int i = 0; i < ncones; ++i) {
    const int64_t d = dims[i];
    if (d < 1) return fail(CGB_EINVAL, "cone dimension must be >= 1");
    switch (kinds[i]) {
      case CGB_CONE_ZERO:
      case CGB_CONE_NONNEG: {
        const int32_t kind = kinds[i] == CGB_CONE_ZERO ? SEG_ZERO : SEG_NONNEG;
        if (!segs.empty() && segs.back().kind == kind && segs.back().end == off)
          segs.back().end = off + d;
        else
          segs.push_back(DevSeg{off, off + d, kind, 0});
      } break;
      case CGB_CONE_SOC:
        if (d > kSmallMax && nlarge < CGB_MAX_LARGE_SOC) {
          segs.push_back(DevSeg{off, off + d, SEG_SOC_LARGE, nlarge++});
        } else {
          if (d > INT32_MAX) return fail(CGB_EINVAL, "SOC too large");
          small_off.push_back(off);
          small_dim.push_back((int32_t)d);
        }
        break;
      case CGB_CONE_EXP:
        if (d != 3) return fail(CGB_EINVAL, "exponential cone has dimension 3");
        exp_off.push_back(off);
        break;
      default:
        return fail(CGB_EINVAL, "unknown cone kind");
    }
    off += d;
  }
  Blob blob;
  size_t o_seg = blob.add(segs.data(), sizeof(DevSeg) * segs.size());
  size_t o_so = blob.add(small_off.data(), sizeof(int64_t) * small_off.size());
  size_t o_sd = blob.add(small_dim.data(), sizeof(int32_t) * small_dim.size());
  size_t o_eo = blob.add(exp_off.data(), sizeof(int64_t) * exp_off.size());
  char* dev = nullptr;
  CUDA_TRY(cudaMalloc(&dev, blob.host.size() + 256));
  CUDA_TRY(cudaMemcpy(dev, blob.host.data(), blob.host.size(), cudaMemcpyHostToDevice));
  cgb_cones* K = new cgb_cones();
  K->ctx = ctx;
  K->blob = dev;
  K->m = off;
  K->segs = segs;
  DevCones& C = K->dc;
  C.seg = (const DevSeg*)(dev + o_seg);
  C.small_off = (const int64_t*)(dev + o_so);
  C.small_dim = (const int32_t*)(dev + o_sd);
  C.exp_off = (const int64_t*)(dev + o_eo);
  C.m = off;
  C.nseg = (int32_t)segs.size();
  C.nsmall = (int32_t)small_off.size();
  C.nexp = (int32_t)exp_off.size();
  C.nlarge = nlarge;
  *out = K;
  return CGB_OK;
}

int cgb_cones_destroy(cgb_cones* K) {
  if (!K) return CGB_OK;
  if (K->blob) cudaFree(K->blob);
  delete K;
  return CGB_OK;
}

int cgb_cones_project(cgb_ctx* ctx, const cgb_cones* K, int dual, const double* v, double* out,
                      void* stream) {
  if (!ctx || !K || !v || !out) return fail(CGB_EINVAL, "null argument");
  if (v == out) return fail(CGB_EINVAL, "cgb_cones_project: in-place projection not supported");
  if (K->sharded) return fail(CGB_EINVAL, "sharded cone pieces cannot be projected alone");
  if (K->ctx != ctx) return fail(CGB_EINVAL, "cones belong to another ctx");
  std::lock_guard<std::mutex> lk(ctx->mu);
  ConeArgs a{ctx->bar, ctx->partials, K->dc, dual, v, out};
  return launch_coop(ctx, k_cones, a, 0, (cudaStream_t)stream);
}

int cgb_cg_solve(cgb_ctx* ctx, const cgb_op* op, int recipe, double lam, const double* b,
                 double* x, double tol, int64_t max_iter, cgb_cg_result* res, void* stream) {
  if (!ctx || !op || !b || !x || !res) return fail(CGB_EINVAL, "null argument");
  if (op->ctx != ctx) return fail(CGB_EINVAL, "operator belongs to another ctx");
  if (recipe != CGB_RECIPE_DIRECT && recipe != CGB_RECIPE_NORMAL)
    return fail(CGB_EINVAL, "unknown CG recipe");
  const int64_t n = op->fwd.in_len, m = op->fwd.out_len;
  if (recipe == CGB_RECIPE_DIRECT && n != m) return fail(CGB_EINVAL, "direct CG needs square A");
  std::lock_guard<std::mutex> lk(ctx->mu);
  cudaStream_t s = (cudaStream_t)stream;
  double* scratch = nullptr;
  CUDA_TRY(cudaMallocAsync(&scratch, sizeof(double) * (3 * n + m + 1), s));
  CgArgs a{ctx->bar, ctx->partials, op->fwd.dp, op->adj.dp, recipe, lam, b, x,
           scratch, scratch + n, scratch + 2 * n, scratch + 3 * n,
           n, m, tol, max_iter, eps_floor_for(n), ctx->result};
  int rc = (a.F.smem_xs2 > 0 || a.Aj.smem_xs2 > 0)
               ? launch_coop(ctx, k_cg<1>, a, solver_smem(a.F, a.Aj), s)
               : launch_coop(ctx, k_cg<0>, a, solver_smem(a.F, a.Aj), s);
  cudaError_t ce = cudaSuccess;
  if (rc == CGB_OK)
    ce = cudaMemcpyAsync(ctx->host_result, ctx->result, 3 * sizeof(double),
                         cudaMemcpyDeviceToHost, s);
  // the scratch is released on every path, before any error return
  const cudaError_t fe = cudaFreeAsync(scratch, s);
  const cudaError_t se = cudaStreamSynchronize(s);
  if (rc) return rc;
  if (ce != cudaSuccess) return fail(CGB_ECUDA, std::string("result copy: ") + cudaGetErrorString(ce));
  if (fe != cudaSuccess) return fail(CGB_ECUDA, std::string("scratch free: ") + cudaGetErrorString(fe));
  if (se != cudaSuccess) return fail(CGB_ECUDA, std::string("k_cg: ") + cudaGetErrorString(se));
  res->iterations = (int64_t)ctx->host_result[0];
  res->final_residual_norm = std::sqrt(ctx->host_result[1]);
  res->b_norm = std::sqrt(ctx->host_result[2]);
  res->converged = res->final_residual_norm <= tol * res->b_norm;
  res->reserved = 0;
  return CGB_OK;
}

int cgb_inner_solve(cgb_ctx* ctx, const cgb_op* op, const double* d1, const double* d2,
                    double* z, double tol, int64_t max_iter, const double* c, const double* b,
                    double* scratch, cgb_cg_result* res, double* hdot, void* stream) {
  if (!ctx || !op || !d1 || !d2 || !z || !scratch) return fail(CGB_EINVAL, "null argument");
  if (op->ctx != ctx) return fail(CGB_EINVAL, "operator belongs to another ctx");
  std::lock_guard<std::mutex> lk(ctx->mu);
  const int64_t n = op->fwd.in_len, m = op->fwd.out_len;
  cudaStream_t s = (cudaStream_t)stream;
  InnerArgs a{ctx->bar, ctx->partials, op->fwd.dp, op->adj.dp, d1, d2, z, c, b,
              scratch, scratch + n, scratch + 2 * n, scratch + 3 * n, scratch + 3 * n + m,
              n, m, tol, max_iter, eps_floor_for(n), ctx->result};
  const int cs = cluster_size_for(n, m, op->fwd.leaf_bytes + op->adj.leaf_bytes);
  int rc = (a.F.smem_xs2 > 0 || a.Aj.smem_xs2 > 0)
               ? launch_coop(ctx, k_inner<1>, a, solver_smem(a.F, a.Aj), s, cs)
               : launch_coop(ctx, k_inner<0>, a, solver_smem(a.F, a.Aj), s, cs);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(ctx->host_result, ctx->result, 4 * sizeof(double),
                           cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (res) {
    res->iterations = (int64_t)ctx->host_result[0];
    res->final_residual_norm = std::sqrt(ctx->host_result[1]);
    res->b_norm = std::sqrt(ctx->host_result[2]);
    res->converged = res->final_residual_norm <= tol * res->b_norm;
    res->reserved = 0;
  }
  if (hdot) *hdot = ctx->host_result[3];
  return CGB_OK;
}

int cgb_debug_barrier(cgb_ctx* ctx, int64_t iters, int mode, void* stream) {
  if (!ctx || iters < 0) return fail(CGB_EINVAL, "bad argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  BarArgs a{ctx->bar, ctx->partials, iters, mode, ctx->result};
  return launch_coop(ctx, k_barrier, a, 0, (cudaStream_t)stream);
}

int cgb_scs_run(cgb_ctx* ctx, const cgb_scs_problem* prob, const cgb_scs_settings* st,
                cgb_scs_work* work, int64_t max_steps, int resid_every_iter, void* stream) {
  if (!ctx || !prob || !st || !work) return fail(CGB_EINVAL, "null argument");
  if (prob->struct_size != (int64_t)sizeof(cgb_scs_problem))
    return fail(CGB_EINVAL, "cgb_scs_problem.struct_size mismatch (ABI v" +
                                std::to_string(CGB_ABI_VERSION) + " layout expected)");
  if (!prob->A || !prob->K || !prob->b || !prob->c || !prob->g)
    return fail(CGB_EINVAL, "null problem member");
  const cgb_op* op = prob->A;
  if (op->ctx != ctx || prob->K->ctx != ctx)
    return fail(CGB_EINVAL, "operator / cones belong to another ctx");
  if (prob->K->sharded) return fail(CGB_EINVAL, "sharded cone pieces need cgb_shard_run");
  if (op->fwd.in_len != prob->n || op->fwd.out_len != prob->m || prob->K->m != prob->m)
    return fail(CGB_EINVAL, "problem dimensions disagree with operator / cones");
  if (st->check_interval < 1 || st->eps <= 0) return fail(CGB_EINVAL, "bad settings");
  std::lock_guard<std::mutex> lk(ctx->mu);
  ScsArgs a;
  a.bar = ctx->bar;
  a.partials = ctx->partials;
  a.F = op->fwd.dp;
  a.Aj = op->adj.dp;
  a.K = prob->K->dc;
  a.st = *st;
  a.w = *work;
  a.b = prob->b;
  a.c = prob->c;
  a.g = prob->g;
  a.n = prob->n;
  a.m = prob->m;
  a.denom = prob->denom;
  a.pr_scale = prob->pr_scale;
  a.dr_scale = prob->dr_scale;
  a.eps_floor = eps_floor_for(prob->n);
  a.max_steps = max_steps;
  a.resid_every = resid_every_iter;
  a.prof = ctx->prof;
  a.no_skip = (prob->flags & CGB_SCS_NO_ZERO_SKIP) ? 1 : 0;
  a.park = std::getenv("CGB_NO_SOC_PARK") ? nullptr : work->t;
  a.refresh = 0;
  if (const char* env = std::getenv("CGB_REFRESH")) a.refresh = std::max(0, std::atoi(env));
  // shared memory: conv staging of the plans, or the large-SOC stash of the
  // cone step, whichever is larger (never live together; one CTA per SM --
  // the kernel re-checks the stash need with the real grid)
  const size_t base = solver_smem(a.F, a.Aj);
  const int64_t S = (int64_t)std::min(ctx->num_sms * CGB_CTAS_PER_SM, CGB_MAXG) * CGB_BLOCK;
  int64_t need = 0;
  for (const DevSeg& sg : prob->K->segs)
    if (sg.kind == SEG_SOC_LARGE)
      need += (sg.end - sg.begin - 1 + CGB_U * S - 1) / (CGB_U * S) * CGB_U * CGB_BLOCK;
  const size_t kMaxSmem = 200 * 1024;
  size_t smem = base;
  if (sizeof(double) * (size_t)need <= kMaxSmem) smem = std::max(smem, sizeof(double) * (size_t)need);
  a.stash_cap = (int)(smem / sizeof(double));
  const int cs = cluster_size_for(prob->n, prob->m, op->fwd.leaf_bytes + op->adj.leaf_bytes);
  if (a.F.smem_xs2 > 0 || a.Aj.smem_xs2 > 0)
    return launch_coop(ctx, k_scs<1>, a, smem, (cudaStream_t)stream, cs);
  if (op->fwd.has_dense || op->adj.has_dense)
    return launch_coop(ctx, k_scs<2>, a, smem, (cudaStream_t)stream, cs);
  return launch_coop(ctx, k_scs<0>, a, smem, (cudaStream_t)stream, cs);
}

int cgb_ctx_set_grid(cgb_ctx* ctx, int32_t grid) {
  if (!ctx || grid < 0) return fail(CGB_EINVAL, "bad argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  ctx->grid_override = grid;
  return CGB_OK;
}

int cgb_shard_cones_create(cgb_ctx* ctx, const int32_t* kinds, const int64_t* begin,
                           const int64_t* end, const int32_t* soc_id, const int32_t* has_head,
                           int32_t npieces, int64_t m, int32_t nsoc, cgb_cones** out) {
  if (!ctx || !out || npieces < 0 || (npieces > 0 && (!kinds || !begin || !end || !soc_id ||
                                                      !has_head)))
    return fail(CGB_EINVAL, "bad cone piece spec");
  if (nsoc < 0 || nsoc > CGB_MAX_LARGE_SOC)
    return fail(CGB_EINVAL, "at most " + std::to_string(CGB_MAX_LARGE_SOC) +
                                " world-reduced second-order cones");
  *out = nullptr;
  std::vector<DevSeg> segs;
  std::vector<int64_t> small_off, exp_off;
  std::vector<int32_t> small_dim;
  int64_t prev = 0;
  for (int i = 0; i < npieces; ++i) {
    const int64_t b0 = begin[i], e0 = end[i];
    if (b0 != prev || e0 <= b0 || e0 > m)
      return fail(CGB_EINVAL, "cone pieces must tile [0, m) in order");
    prev = e0;
    switch (kinds[i]) {
      case CGB_CONE_ZERO:
      case CGB_CONE_NONNEG: {
        const int32_t kind = kinds[i] == CGB_CONE_ZERO ? SEG_ZERO : SEG_NONNEG;
        if (!segs.empty() && segs.back().kind == kind && segs.back().end == b0)
          segs.back().end = e0;
        else
          segs.push_back(DevSeg{b0, e0, kind, 0});
      } break;
      case CGB_CONE_SOC:
        if (soc_id[i] >= 0) {
          if (soc_id[i] >= nsoc) return fail(CGB_EINVAL, "soc_id out of range");
          segs.push_back(DevSeg{b0, e0, has_head[i] ? SEG_SOC_LARGE : SEG_SOC_TAIL, soc_id[i]});
        } else {
          if (e0 - b0 > INT32_MAX) return fail(CGB_EINVAL, "SOC too large");
          small_off.push_back(b0);
          small_dim.push_back((int32_t)(e0 - b0));
        }
        break;
      case CGB_CONE_EXP:
        if (e0 - b0 != 3) return fail(CGB_EINVAL, "exponential cone piece must be whole (3)");
        exp_off.push_back(b0);
        break;
      default:
        return fail(CGB_EINVAL, "unknown cone kind");
    }
  }
  if (prev != m) return fail(CGB_EINVAL, "cone pieces must tile [0, m)");
  Blob blob;
  size_t o_seg = blob.add(segs.data(), sizeof(DevSeg) * segs.size());
  size_t o_so = blob.add(small_off.data(), sizeof(int64_t) * small_off.size());
  size_t o_sd = blob.add(small_dim.data(), sizeof(int32_t) * small_dim.size());
  size_t o_eo = blob.add(exp_off.data(), sizeof(int64_t) * exp_off.size());
  char* dev = nullptr;
  CUDA_TRY(cudaMalloc(&dev, blob.host.size() + 256));
  CUDA_TRY(cudaMemcpy(dev, blob.host.data(), blob.host.size(), cudaMemcpyHostToDevice));
  cgb_cones* K = new cgb_cones();
  K->ctx = ctx;
  K->sharded = true;
  K->blob = dev;
  K->m = m;
  K->segs = segs;
  DevCones& C = K->dc;
  C.seg = (const DevSeg*)(dev + o_seg);
  C.small_off = (const int64_t*)(dev + o_so);
  C.small_dim = (const int32_t*)(dev + o_sd);
  C.exp_off = (const int64_t*)(dev + o_eo);
  C.m = m;
  C.nseg = (int32_t)segs.size();
  C.nsmall = (int32_t)small_off.size();
  C.nexp = (int32_t)exp_off.size();
  C.nlarge = nsoc;
  *out = K;
  return CGB_OK;
}

int cgb_shard_run(cgb_ctx* ctx, const cgb_shard_problem* prob, const cgb_scs_settings* st,
                  const cgb_shard_comm* comm, cgb_shard_work* work, int mode,
                  int64_t max_steps, void* stream) {
  if (!ctx || !prob || !st || !comm || !work) return fail(CGB_EINVAL, "null argument");
  if (prob->struct_size != (int64_t)sizeof(cgb_shard_problem))
    return fail(CGB_EINVAL, "cgb_shard_problem.struct_size mismatch");
  if (!prob->A || !prob->K || !prob->b || !prob->c) return fail(CGB_EINVAL, "null problem member");
  if (mode != 0 && mode != 1) return fail(CGB_EINVAL, "mode must be 0 (setup) or 1 (iterate)");
  const int R = comm->world, me = comm->rank;
  if (R < 1 || R > CGB_MAX_RANKS || me < 0 || me >= R)
    return fail(CGB_EINVAL, "world size must be 1.." + std::to_string(CGB_MAX_RANKS));
  if (comm->x_begin[0] != 0 || comm->x_begin[R] != prob->n)
    return fail(CGB_EINVAL, "x slices must tile [0, n)");
  for (int q = 0; q < R; ++q) {
    if (comm->x_begin[q + 1] < comm->x_begin[q]) return fail(CGB_EINVAL, "x slices out of order");
    if (!comm->inbox[q] || !comm->xfull[q] || !comm->mbox[q])
      return fail(CGB_EINVAL, "null peer buffer of rank " + std::to_string(q));
  }
  const cgb_op* op = prob->A;
  if (op->ctx != ctx || prob->K->ctx != ctx)
    return fail(CGB_EINVAL, "operator / cones belong to another ctx");
  if (op->fwd.in_len != prob->n || op->fwd.out_len != prob->m || prob->K->m != prob->m)
    return fail(CGB_EINVAL, "problem dimensions disagree with operator / cones");
  if (op->fwd.dp.smem_xs2 > 0 || op->adj.dp.smem_xs2 > 0)
    return fail(CGB_EINVAL, "2-d convolution leaves are not row-sharded (keep them on one GPU)");
  if (st->check_interval < 1 || st->eps <= 0) return fail(CGB_EINVAL, "bad settings");
  if (max_steps < 0) return CGB_OK;  // validation only (launch nothing)
  std::lock_guard<std::mutex> lk(ctx->mu);
  ShardArgs a;
  a.bar = ctx->bar;
  a.partials = ctx->partials;
  a.F = op->fwd.dp;
  a.Aj = op->adj.dp;
  a.K = prob->K->dc;
  a.st = *st;
  a.comm = *comm;
  a.w = *work;
  a.b = prob->b;
  a.c = prob->c;
  a.n = prob->n;
  a.m = prob->m;
  a.x0 = comm->x_begin[me];
  a.nl = comm->x_begin[me + 1] - comm->x_begin[me];
  a.pr_scale = prob->pr_scale;
  a.dr_scale = prob->dr_scale;
  a.eps_floor = eps_floor_for(prob->n);
  a.setup_tol = prob->setup_tol;
  a.max_steps = max_steps;
  a.mode = mode;
  return launch_coop(ctx, k_shard<0>, a, solver_smem(a.F, a.Aj), (cudaStream_t)stream);
}

int cgb_ipc_alloc(int device, int64_t bytes, void** ptr, void* handle64) {
  if (!ptr || !handle64 || bytes < 0) return fail(CGB_EINVAL, "bad argument");
  CUDA_TRY(cudaSetDevice(device));
  void* p = nullptr;
  CUDA_TRY(cudaMalloc(&p, (size_t)std::max<int64_t>(bytes, 256)));
  CUDA_TRY(cudaMemset(p, 0, (size_t)std::max<int64_t>(bytes, 256)));
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return fail(CGB_ECUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
  }
  std::memcpy(handle64, &h, sizeof(h));
  *ptr = p;
  return CGB_OK;
}

int cgb_ipc_open(int device, const void* handle64, void** ptr) {
  if (!ptr || !handle64) return fail(CGB_EINVAL, "bad argument");
  CUDA_TRY(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return CGB_OK;
}

int cgb_ipc_close(void* ptr) {
  if (ptr) CUDA_TRY(cudaIpcCloseMemHandle(ptr));
  return CGB_OK;
}

int cgb_ipc_free(void* ptr) {
  if (ptr) CUDA_TRY(cudaFree(ptr));
  return CGB_OK;
}

int cgb_scs_profile(cgb_ctx* ctx, double* dev_acc) {
  if (!ctx) return fail(CGB_EINVAL, "null argument");
  ctx->prof = dev_acc;
  return CGB_OK;
}

}  // extern "C"

#endif  // CGB_TU_HOST
