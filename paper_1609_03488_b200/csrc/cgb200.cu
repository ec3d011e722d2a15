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
#include <cstring>
#include <string>
#include <vector>

#include "cgb_device.cuh"

using namespace cgb;

// ===========================================================================
// epilogues: called once per lane tile (rows first + 32 r, r < R, valid
// while 32 r < left); all loads are issued before any store.
// ===========================================================================
namespace {

struct EpiStore {  // y -> out
  double* out;
  __device__ void tile(int64_t row, int R, int left, const double (&y)[CGB_RC], double*) const {
#pragma unroll
    for (int r = 0; r < CGB_RC; ++r)
      if (CGB_EPI_VALID(r)) out[row + 32 * r] = y[r];
  }
};

// Splitting-step / inner-solve start: with y = A^T d2 and g = A^T A x0,
//   rhs = d1 - y ;  r = rhs - (x0 + g) ;  p = r ;  sums: rhs.rhs, r.r
// (scs.py:349 rhs = wz1 - A^T wz2 ; cg.py:129 r0 = b - (1*x + A^T A x))
struct EpiRhs {
  const double* d1;
  const double* x0;
  const double* g;
  double* r;
  double* p;
  __device__ void tile(int64_t j, int R, int left, const double (&y)[CGB_RC],
                       double* part) const {
    double a[CGB_RC], x[CGB_RC], gg[CGB_RC];
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q)
      if (CGB_EPI_VALID(q)) { a[q] = d1[j + 32 * q]; x[q] = x0[j + 32 * q]; gg[q] = g[j + 32 * q]; }
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q) {
      if (CGB_EPI_VALID(q)) {
        const double rhs = a[q] - y[q];
        const double rr = rhs - (x[q] + gg[q]);
        r[j + 32 * q] = rr;
        p[j + 32 * q] = rr;
        part[0] += rhs * rhs;
        part[1] += rr * rr;
      }
    }
  }
};

// standalone CG init: r = b - apply(x), p = r ; sums r.r, b.b   (cg.py:129-132)
struct EpiR0 {
  const double* b;
  const double* x;
  double* r;
  double* p;
  double lam;
  int normal;
  __device__ void tile(int64_t j, int R, int left, const double (&y)[CGB_RC],
                       double* part) const {
    double bb[CGB_RC], xx[CGB_RC];
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q)
      if (CGB_EPI_VALID(q)) { bb[q] = b[j + 32 * q]; xx[q] = x[j + 32 * q]; }
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q) {
      if (CGB_EPI_VALID(q)) {
        double ax = y[q];
        if (normal && lam != 0.0) ax = lam * xx[q] + y[q];
        const double rr = bb[q] - ax;
        r[j + 32 * q] = rr;
        p[j + 32 * q] = rr;
        part[0] += rr * rr;
        part[1] += bb[q] * bb[q];
      }
    }
  }
};

// CG phase B (normal recipe): q = lam p + A^T t ; sum p.q   (cg.py:80-83,111)
struct EpiQ {
  const double* p;
  double* qv;
  double lam;
  __device__ void tile(int64_t j, int R, int left, const double (&y)[CGB_RC],
                       double* part) const {
    double pp[CGB_RC];
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q)
      if (CGB_EPI_VALID(q)) pp[q] = p[j + 32 * q];
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q) {
      if (CGB_EPI_VALID(q)) {
        const double qj = (lam != 0.0) ? lam * pp[q] + y[q] : y[q];
        qv[j + 32 * q] = qj;
        part[0] += pp[q] * qj;
      }
    }
  }
};

// CG phase A (direct recipe): q = A p ; sum p.q, p from the fused accessor
struct EpiQDirect {
  InVec pin;
  double* qv;
  __device__ void tile(int64_t j, int R, int left, const double (&y)[CGB_RC],
                       double* part) const {
    double pp[CGB_RC];
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q)
      if (CGB_EPI_VALID(q)) pp[q] = pin(j + 32 * q);
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q) {
      if (CGB_EPI_VALID(q)) {
        qv[j + 32 * q] = y[q];
        part[0] += pp[q] * y[q];
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
  __device__ void tile(int64_t i, int R, int left, const double (&y)[CGB_RC],
                       double* part) const {
    double dd[CGB_RC], bb[CGB_RC];
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q)
      if (CGB_EPI_VALID(q)) { dd[q] = d2[i + 32 * q]; bb[q] = b ? b[i + 32 * q] : 0.0; }
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
  __device__ void tile(int64_t i, int R, int left, const double (&y)[CGB_RC],
                       double* part) const {
    double ss[CGB_RC], bb[CGB_RC];
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q)
      if (CGB_EPI_VALID(q)) { ss[q] = s[i + 32 * q]; bb[q] = b[i + 32 * q]; }
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
  __device__ void tile(int64_t j, int R, int left, const double (&y)[CGB_RC],
                       double* part) const {
    double cc[CGB_RC];
#pragma unroll
    for (int q = 0; q < CGB_RC; ++q)
      if (CGB_EPI_VALID(q)) cc[q] = c[j + 32 * q];
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
// CG loop shared by k_cg, k_inner and k_scs  (cg.py:87-137)
// ===========================================================================
// Optional incremental tracking (splitting solver): ax = A x and gx = A^T A x
// follow x through the updates x += alpha p (ax += alpha A p, gx += alpha
// (q - p)), so the next splitting step needs neither A x nor A^T A x anew.
// With track, phase C also accumulates h.(x, wy + ax) for tau~ (scs.py:357).
struct CgBufs {
  double* x;
  double* r;
  double* pb[2];  // pb[0] holds r0 on entry
  double* q;
  double* t;      // m scratch (normal recipe): A p
  double* ax;     // m, tracked A x (or null)
  double* gx;     // n, tracked A^T A x (or null)
  const double* wy;  // m: wz2 for h.p (with tracking)
  const double* b;   // m
  const double* c;   // n
};

struct PNew {  // p_new = r + beta p_old
  const double* r; const double* po; double* pn; double beta;
  double rv[CGB_U], pv[CGB_U];
  __device__ void load(int64_t i, int u) { rv[u] = r[i]; pv[u] = po[i]; }
  __device__ void compute(int64_t i, int u) { pn[i] = rv[u] + beta * pv[u]; }
};

struct CgUpdateN {  // x += alpha p ; r -= alpha q ; gx += alpha (q - p)
  double* x; double* r; const double* p; const double* q; double* gx; const double* c;
  double alpha;
  double rr, hc;
  double xv[CGB_U], rv[CGB_U], pv[CGB_U], qv[CGB_U], gv[CGB_U], cv[CGB_U];
  __device__ void load(int64_t i, int u) {
    xv[u] = x[i]; rv[u] = r[i]; pv[u] = p[i]; qv[u] = q[i];
    if (gx) { gv[u] = gx[i]; cv[u] = c[i]; }
  }
  __device__ void compute(int64_t i, int u) {
    const double xn = xv[u] + alpha * pv[u];
    x[i] = xn;
    const double ri = rv[u] - alpha * qv[u];
    r[i] = ri;
    rr += ri * ri;
    if (gx) {
      gx[i] = gv[u] + alpha * (qv[u] - pv[u]);
      hc += cv[u] * xn;
    }
  }
};

struct CgUpdateM {  // ax += alpha t ; sum b.(wy + ax)
  double* ax; const double* t; const double* wy; const double* b; double alpha;
  double hb;
  double av[CGB_U], tv[CGB_U], wv[CGB_U], bv[CGB_U];
  __device__ void load(int64_t i, int u) { av[u] = ax[i]; tv[u] = t[i]; wv[u] = wy[i]; bv[u] = b[i]; }
  __device__ void compute(int64_t i, int u) {
    const double an = av[u] + alpha * tv[u];
    ax[i] = an;
    hb += bv[u] * (wv[u] + an);
  }
};

// Runs CG from the state prepared by the caller (r = b - apply(x),
// pb[0] = r, rns = r.r).  Returns the iteration count; `hp` receives the
// tracked h.p of the final iterate when tracking is on.
__device__ int64_t cg_loop(const DevPlan& F, const DevPlan& Aj, int recipe, double lam,
                           const CgBufs& B, int64_t n, int64_t m, double& rns, double delta,
                           double floor_, int64_t max_iter, GridSync& gs, double* hp) {
  int64_t k = 0;
  int cur = 0;
  double beta = 0.0;
  const bool track = B.ax != nullptr;
  while (sqrt(rns) > delta && rns > floor_ && (double)max_iter > (double)k) {
    InVec pin;
    if (k == 0) {
      pin = InVec{B.pb[cur], nullptr, 0.0};
    } else {
      pin = InVec{B.r, B.pb[cur], beta};
      PNew f{B.r, B.pb[cur], B.pb[cur ^ 1], beta, {}, {}};
      stream_loop(n, f);
      cur ^= 1;
    }
    const double* pc = B.pb[cur];
    double pq[1] = {0.0};
    if (recipe == CGB_RECIPE_NORMAL) {
      EpiStore st{B.t};
      apply_plan(F, pin, st, nullptr, gs);
      gs.sync();
      InVec tin{B.t, nullptr, 0.0};
      EpiQ eq{pc, B.q, lam};
      apply_plan(Aj, tin, eq, pq, gs);
    } else {
      EpiQDirect eq{pin, B.q};
      apply_plan(F, pin, eq, pq, gs);
    }
    gs.reduce(pq);
    const double alpha = rns / pq[0];
    double red[3] = {0.0, 0.0, 0.0};
    {
      CgUpdateN f{B.x, B.r, pc, B.q, track ? B.gx : nullptr, B.c, alpha, 0.0, 0.0,
                  {}, {}, {}, {}, {}, {}};
      stream_loop(n, f);
      red[0] = f.rr;
      red[2] = f.hc;
    }
    if (track) {
      CgUpdateM f{B.ax, B.t, B.wy, B.b, alpha, 0.0, {}, {}, {}, {}};
      stream_loop(m, f);
      red[1] = f.hb;
    }
    gs.reduce(red);
    beta = red[0] / rns;
    rns = red[0];
    if (hp) *hp = red[2] + red[1];
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

__global__ void __launch_bounds__(CGB_BLOCK, CGB_MINB) k_apply(ApplyArgs a) {
  GridSync gs(a.bar, a.partials);
  InVec in{a.x, nullptr, 0.0};
  EpiStore st{a.y};
  apply_plan(a.P, in, st, nullptr, gs);
}

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

__global__ void __launch_bounds__(CGB_BLOCK, CGB_MINB) k_cones(ConeArgs a) {
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

struct CgArgs {
  GridBar* bar; double* partials;
  DevPlan F, Aj;
  int recipe; double lam;
  const double* b; double* x;
  double* r; double* p0; double* p1; double* q; double* t;
  int64_t n, m; double tol; int64_t max_iter; double eps_floor;
  double* result;  // [iterations, rns, bnorm2]
};

__global__ void __launch_bounds__(CGB_BLOCK, CGB_MINB) k_cg(CgArgs a) {
  GridSync gs(a.bar, a.partials);
  double s[2] = {0.0, 0.0};
  InVec xin{a.x, nullptr, 0.0};
  if (a.recipe == CGB_RECIPE_NORMAL) {
    EpiStore st{a.t};
    apply_plan(a.F, xin, st, nullptr, gs);
    gs.sync();
    InVec tin{a.t, nullptr, 0.0};
    EpiR0 e{a.b, a.x, a.r, a.p0, a.lam, 1};
    apply_plan(a.Aj, tin, e, s, gs);
  } else {
    EpiR0 e{a.b, a.x, a.r, a.p0, 0.0, 0};
    apply_plan(a.F, xin, e, s, gs);
  }
  gs.reduce(s);
  double rns = s[0];
  const double delta = a.tol * sqrt(s[1]);
  const double floor_ = a.eps_floor * s[1];
  CgBufs B{a.x, a.r, {a.p0, a.p1}, a.q, a.t, nullptr, nullptr, nullptr, nullptr, nullptr};
  const int64_t k = cg_loop(a.F, a.Aj, a.recipe, a.lam, B, a.n, a.m, rns, delta, floor_,
                            a.max_iter, gs, nullptr);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.result[0] = (double)k;
    a.result[1] = rns;
    a.result[2] = s[1];
  }
}

struct InnerArgs {
  GridBar* bar; double* partials;
  DevPlan F, Aj;
  const double* d1; const double* d2;
  double* z;  // n + m
  const double* c; const double* b;
  double* r; double* p0; double* p1; double* q; double* t; double* tx;
  int64_t n, m; double tol; int64_t max_iter; double eps_floor;
  double* result;  // [iterations, rns, rhs2, hdot]
};

struct SideDot {  // acc += a[i] * b[i]
  const double* x; const double* y; double acc; double xv[CGB_U], yv[CGB_U];
  __device__ void load(int64_t i, int u) { xv[u] = x[i]; yv[u] = y[i]; }
  __device__ void compute(int64_t, int u) { acc += xv[u] * yv[u]; }
};

// Inner block solve, exactly the reference's arithmetic (scs.py:170-187):
// rhs = d1 - A^T d2 ; r0 = rhs - (x0 + A^T A x0) ; CG ; z2 = d2 + A z1.
__global__ void __launch_bounds__(CGB_BLOCK, CGB_MINB) k_inner(InnerArgs a) {
  GridSync gs(a.bar, a.partials);
  double* z1 = a.z;
  double* z2 = a.z + a.n;
  // tx = A x0 ; then p1 (scratch) = A^T tx
  {
    InVec xin{z1, nullptr, 0.0};
    EpiStore st{a.tx};
    apply_plan(a.F, xin, st, nullptr, gs);
    gs.sync();
    InVec tin{a.tx, nullptr, 0.0};
    EpiStore st2{a.p1};
    apply_plan(a.Aj, tin, st2, nullptr, gs);
    gs.sync();
  }
  double s[2] = {0.0, 0.0};
  {
    InVec din{a.d2, nullptr, 0.0};
    EpiRhs e{a.d1, z1, a.p1, a.r, a.p0};
    apply_plan(a.Aj, din, e, s, gs);
    gs.reduce(s);
  }
  double rns = s[1];
  const double delta = a.tol * sqrt(s[0]);
  const double floor_ = a.eps_floor * s[0];
  CgBufs B{z1, a.r, {a.p0, a.p1}, a.q, a.t, nullptr, nullptr, nullptr, nullptr, nullptr};
  const int64_t k = cg_loop(a.F, a.Aj, CGB_RECIPE_NORMAL, 1.0, B, a.n, a.m, rns, delta, floor_,
                            a.max_iter, gs, nullptr);
  double h[2] = {0.0, 0.0};
  {
    InVec xin{z1, nullptr, 0.0};
    EpiZ2 e{nullptr, z2, a.d2, a.b};
    apply_plan(a.F, xin, e, h, gs);
    if (a.c) {
      SideDot f{a.c, z1, 0.0, {}, {}};
      stream_loop(a.n, f);
      h[1] = f.acc;
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
};

// CG tolerance exactly as the solver graph computes it (scs.py:290-311)
__device__ double cg_tolerance_graph(double k, const cgb_scs_settings& s) {
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

// w2 = u~ - v on the cone block: u~_y = p2 - tau_t g_y, p2 = wz2 + A p1
// (scs.py:355, 358, 361)
struct ScsConeSrc {
  const double* wy; const double* ax; const double* gy; const double* vy; double tau_t;
  __device__ double operator()(int64_t i) const {
    return ((wy[i] + ax[i]) - tau_t * gy[i]) - vy[i];
  }
};
// u_y <- proj ; v_y <- (v - u~) + u ; w_y <- u + v   (scs.py:365-366)
struct ScsConeDst {
  const double* wy_in; const double* ax; const double* gy; double* uy; double* vy; double* wy;
  double tau_t;
  __device__ void operator()(int64_t i, double u2) const {
    const double ut = (wy_in[i] + ax[i]) - tau_t * gy[i];
    const double v2 = (vy[i] - ut) + u2;
    uy[i] = u2;
    vy[i] = v2;
    wy[i] = u2 + v2;
  }
};

// x block of the cone step (free): u = u~ - v, v <- (v - u~) + u, w = u + v
struct ScsXStep {
  const double* cgx; const double* g; double* u; double* v; double* w; double tau_t;
  double xv[CGB_U], gv[CGB_U], vv[CGB_U];
  __device__ void load(int64_t i, int k) { xv[k] = cgx[i]; gv[k] = g[i]; vv[k] = v[i]; }
  __device__ void compute(int64_t i, int k) {
    const double ut = xv[k] - tau_t * gv[k];
    const double u2 = ut - vv[k];
    const double v2 = (vv[k] - ut) + u2;
    u[i] = u2;
    v[i] = v2;
    w[i] = u2 + v2;
  }
};

struct HbSide {  // sum b.(wy + ax)
  const double* b; const double* wy; const double* ax; double acc;
  double bv[CGB_U], wv[CGB_U], av[CGB_U];
  __device__ void load(int64_t i, int u) { bv[u] = b[i]; wv[u] = wy[i]; av[u] = ax[i]; }
  __device__ void compute(int64_t, int u) { acc += bv[u] * (wv[u] + av[u]); }
};

__global__ void __launch_bounds__(CGB_BLOCK, CGB_MINB) k_scs(ScsArgs a) {
  GridSync gs(a.bar, a.partials);
  const int64_t n = a.n, m = a.m, N = n + m + 1;
  const cgb_scs_settings& S = a.st;
  const cgb_scs_work& W = a.w;
  double* state = W.state;
  double k = state[CGB_ST_K], since = state[CGB_ST_SINCE], status = state[CGB_ST_STATUS];
  double cgt = state[CGB_ST_CGT];
  double pr = state[CGB_ST_PR], dr = state[CGB_ST_DR], gap = state[CGB_ST_GAP];
  double lastcg = state[CGB_ST_LASTCG];
  const int64_t cg_max = S.cg_max_iter;
  int64_t steps = 0;
  const double* wy = W.w + n;

  while (steps < a.max_steps && (double)S.max_iters > k && !(status > 0.5)) {
    const double wtau = W.w[N - 1];
    const double vtau = W.v[N - 1];

    // -- subspace step: rhs = wz1 - A^T wz2 ; r0 = rhs - (x0 + A^T A x0)
    //    plus h.(x0, wz2 + A x0) in case CG takes no step (scs.py:349-357)
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    {
      InVec in{wy, nullptr, 0.0};
      EpiRhs e{W.w, W.cgx, W.gx, W.r, W.p0};
      apply_plan(a.Aj, in, e, s, gs);
      HbSide fb{a.b, wy, W.tax, 0.0, {}, {}, {}};
      stream_loop(m, fb);
      SideDot fc{a.c, W.cgx, 0.0, {}, {}};
      stream_loop(n, fc);
      s[2] = fb.acc;
      s[3] = fc.acc;
      gs.reduce(s);
    }
    const double tol_k = cg_tolerance_graph(k, S);
    const double delta = tol_k * sqrt(s[0]);
    const double floor_ = a.eps_floor * s[0];
    double rns = s[1];
    double hp = s[3] + s[2];
    CgBufs B{W.cgx, W.r, {W.p0, W.p1}, W.q, W.t, W.tax, W.gx, wy, a.b, a.c};
    const int64_t cgk = cg_loop(a.F, a.Aj, CGB_RECIPE_NORMAL, 1.0, B, n, m, rns, delta, floor_,
                                cg_max, gs, &hp);
    const double tau_t = (wtau + hp) / a.denom;

    // -- cone step onto R^n x K* x R+   (scs.py:360-366)
    ScsConeSrc src{wy, W.tax, a.g + n, W.v + n, tau_t};
    ScsConeDst dst{wy, W.tax, a.g + n, W.u + n, W.v + n, W.w + n, tau_t};
    double red[2 * CGB_MAX_LARGE_SOC];
#pragma unroll
    for (int i = 0; i < 2 * CGB_MAX_LARGE_SOC; ++i) red[i] = 0.0;
    if (a.K.nlarge > 0) {
      cone_large_partials(a.K, src, red);
      gs.reduce(red);
    }
    cone_project(a.K, 1, src, dst, red);
    {
      ScsXStep f{W.cgx, a.g, W.u, W.v, W.w, tau_t, {}, {}, {}};
      stream_loop(n, f);
    }
    const double utau = fmax(tau_t - vtau, 0.0);
    const double kappa = (vtau - tau_t) + utau;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      W.u[N - 1] = utau;
      W.v[N - 1] = kappa;
      W.w[N - 1] = utau + kappa;
    }
    gs.sync();

    k += 1.0;
    const double since2 = since + 1.0;
    const bool is_check = since2 > (double)S.check_interval - 0.5;
    cgt += (double)cgk;
    lastcg = (double)cgk;

    if (is_check || a.resid_every) {
      // -- termination measures (scs.py:369-402)
      double q[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      InVec uxin{W.u, nullptr, 0.0};
      InVec uyin{W.u + n, nullptr, 0.0};
      EpiRawP ep{W.v + n, a.b, utau};
      EpiRawD ed{a.c, utau};
      apply_two(a.F, uxin, ep, a.Aj, uyin, ed, q, gs);
      SideDot fc{a.c, W.u, 0.0, {}, {}};
      stream_loop(n, fc);
      SideDot fb{a.b, W.u + n, 0.0, {}, {}};
      stream_loop(m, fb);
      q[4] = fc.acc;
      q[5] = fb.acc;
      gs.reduce(q);
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
      const double unb_ok = pos_u * (eps > res_u ? 1.0 : 0.0);
      const double den_i = fmax(-1.0 * bty, 0.0);
      const double pos_i = den_i > 0.0 ? 1.0 : 0.0;
      const double res_i = sqrt(q[3]) / (den_i + (1.0 - pos_i));
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
  }
}

struct BarArgs {
  GridBar* bar; double* partials;
  int64_t iters; int mode; double* out;
};

// diagnostics: cost of the grid barrier / grid reduction
__global__ void __launch_bounds__(CGB_BLOCK, CGB_MINB) k_barrier(BarArgs a) {
  GridSync gs(a.bar, a.partials);
  double acc = 0.0;
  for (int64_t i = 0; i < a.iters; ++i) {
    if (a.mode == 0) {
      gs.sync();
    } else {
      double v[1] = {1.0};
      gs.reduce(v);
      acc += v[0];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) a.out[0] = acc;
}

}  // namespace

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
};

struct PlanStore {
  DevPlan dp{};
  void* blob = nullptr;     // device allocation holding all arrays
  double* temps = nullptr;  // 2 * temp_total
  int64_t temp_total = 0;
  int64_t in_len = 0, out_len = 0;
};

struct cgb_op {
  PlanStore fwd, adj;
};

struct cgb_cones {
  DevCones dc{};
  void* blob = nullptr;
  int64_t m = 0;
};

namespace {

size_t plan_smem(const DevPlan& P) { return sizeof(double) * CGB_WARPS * (size_t)P.smem_per_warp; }

template <class K>
int grid_for(const cgb_ctx* ctx, K kernel, size_t smem, int* grid) {
  CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)std::max<size_t>(smem, 1)));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, CGB_BLOCK, smem));
  if (per_sm < 1)
    return fail(CGB_ECOOP, "kernel cannot be resident (threads/registers/shared memory)");
  int g = ctx->num_sms * std::min(per_sm, 2);
  if (g > ctx->max_grid) g = ctx->max_grid;
  *grid = g;
  return CGB_OK;
}

template <class K, class A>
int launch_coop(const cgb_ctx* ctx, K kernel, A& args, size_t smem, cudaStream_t stream) {
  int grid = 0;
  int rc = grid_for(ctx, kernel, smem, &grid);
  if (rc) return rc;
  if (grid > CGB_MAXG) return fail(CGB_ECOOP, "grid larger than CGB_MAXG");
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
      for (int t = R.term_begin; t < R.term_end; ++t) {
        const cgb_leaf& LF = d->leaves[d->terms[t].leaf];
        if ((LF.kind == CGB_LEAF_CONV1D || LF.kind == CGB_LEAF_CORR1D) &&
            LF.k0 <= CGB_CONV_KMAX) {
          D.rfac = CGB_RC;
          kmax = std::max<int64_t>(kmax, LF.k0);
        }
      }
      const int64_t rows_per_tile = 32 * (int64_t)D.rfac;
      tiles += (R.row_end - R.row_begin + rows_per_tile - 1) / rows_per_tile;
      ++idx;
    }
    level_tiles[e] = tiles;
  }
  level_rb[nlevels] = idx;
  Blob blob;
  size_t o_leaves = blob.add(d->leaves, sizeof(cgb_leaf) * d->nleaves);
  size_t o_terms = blob.add(d->terms, sizeof(cgb_term) * d->nterms);
  size_t o_rbs = blob.add(rbs.data(), sizeof(DevRowBlock) * rbs.size());
  size_t o_lrb = blob.add(level_rb.data(), sizeof(int32_t) * level_rb.size());
  size_t o_lt = blob.add(level_tiles.data(), sizeof(int64_t) * level_tiles.size());
  size_t o_to = blob.add(temp_off.data(), sizeof(int64_t) * temp_off.size());
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
  P.temp[0] = ps->temps;
  P.temp[1] = ps->temps ? ps->temps + temp_total : nullptr;
  P.nlevels = nlevels;
  if (kmax > 0) {
    const int64_t groups = (kmax + CGB_RC - 1) / CGB_RC;
    P.smem_cc = (int32_t)(groups * CGB_RC + 1) & ~1;
    P.smem_xs = (int32_t)((32 * CGB_RC + (groups + 1) * CGB_RC + 1) & ~1);
    P.smem_per_warp = P.smem_cc + P.smem_xs + 32 * CGB_RC + 1;
  } else {
    P.smem_cc = 0;
    P.smem_xs = 0;
    P.smem_per_warp = 0;
  }
  P.in_len = d->in_len;
  P.out_len = d->out_len;
  ps->in_len = d->in_len;
  ps->out_len = d->out_len;
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
  delete ctx;
  return CGB_OK;
}

int cgb_ctx_geometry(const cgb_ctx* ctx, int32_t* out3) {
  if (!ctx || !out3) return fail(CGB_EINVAL, "null argument");
  int grid = 0;
  int rc = grid_for(ctx, k_scs, 0, &grid);
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
  ApplyArgs a{ctx->bar, ctx->partials, adjoint ? op->adj.dp : op->fwd.dp, x, y};
  return launch_coop(ctx, k_apply, a, plan_smem(a.P), (cudaStream_t)stream);
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
        return fail(CGB_EINVAL, "exponential cone not supported by this build");
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
  K->blob = dev;
  K->m = off;
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
  ConeArgs a{ctx->bar, ctx->partials, K->dc, dual, v, out};
  return launch_coop(ctx, k_cones, a, 0, (cudaStream_t)stream);
}

int cgb_cg_solve(cgb_ctx* ctx, const cgb_op* op, int recipe, double lam, const double* b,
                 double* x, double tol, int64_t max_iter, cgb_cg_result* res, void* stream) {
  if (!ctx || !op || !b || !x || !res) return fail(CGB_EINVAL, "null argument");
  if (recipe != CGB_RECIPE_DIRECT && recipe != CGB_RECIPE_NORMAL)
    return fail(CGB_EINVAL, "unknown CG recipe");
  const int64_t n = op->fwd.in_len, m = op->fwd.out_len;
  if (recipe == CGB_RECIPE_DIRECT && n != m) return fail(CGB_EINVAL, "direct CG needs square A");
  cudaStream_t s = (cudaStream_t)stream;
  double* scratch = nullptr;
  CUDA_TRY(cudaMallocAsync(&scratch, sizeof(double) * (4 * n + m + 1), s));
  CgArgs a{ctx->bar, ctx->partials, op->fwd.dp, op->adj.dp, recipe, lam, b, x,
           scratch, scratch + n, scratch + 2 * n, scratch + 3 * n, scratch + 4 * n,
           n, m, tol, max_iter, eps_floor_for(n), ctx->result};
  int rc = launch_coop(ctx, k_cg, a, std::max(plan_smem(a.F), plan_smem(a.Aj)), s);
  if (rc == CGB_OK) {
    CUDA_TRY(cudaMemcpyAsync(ctx->host_result, ctx->result, 3 * sizeof(double),
                             cudaMemcpyDeviceToHost, s));
  }
  cudaFreeAsync(scratch, s);
  CUDA_TRY(cudaStreamSynchronize(s));
  if (rc) return rc;
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
  const int64_t n = op->fwd.in_len, m = op->fwd.out_len;
  cudaStream_t s = (cudaStream_t)stream;
  InnerArgs a{ctx->bar, ctx->partials, op->fwd.dp, op->adj.dp, d1, d2, z, c, b,
              scratch, scratch + n, scratch + 2 * n, scratch + 3 * n, scratch + 4 * n,
              scratch + 4 * n + m, n, m, tol, max_iter, eps_floor_for(n), ctx->result};
  int rc = launch_coop(ctx, k_inner, a, std::max(plan_smem(a.F), plan_smem(a.Aj)), s);
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
  BarArgs a{ctx->bar, ctx->partials, iters, mode, ctx->result};
  return launch_coop(ctx, k_barrier, a, 0, (cudaStream_t)stream);
}

int cgb_scs_run(cgb_ctx* ctx, const cgb_scs_problem* prob, const cgb_scs_settings* st,
                cgb_scs_work* work, int64_t max_steps, int resid_every_iter, void* stream) {
  if (!ctx || !prob || !st || !work || !prob->A || !prob->K)
    return fail(CGB_EINVAL, "null argument");
  const cgb_op* op = prob->A;
  if (op->fwd.in_len != prob->n || op->fwd.out_len != prob->m || prob->K->m != prob->m)
    return fail(CGB_EINVAL, "problem dimensions disagree with operator / cones");
  if (st->check_interval < 1 || st->eps <= 0) return fail(CGB_EINVAL, "bad settings");
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
  return launch_coop(ctx, k_scs, a, std::max(plan_smem(a.F), plan_smem(a.Aj)),
                     (cudaStream_t)stream);
}

}  // extern "C"
