// cgb_shard_kernel.cuh -- k_shard, the per-rank persistent kernel of the
// row-sharded solver (see cgb_shard.cuh for the decomposition).  Included
// inside namespace cgbk of cgb200.cu, after k_scs, whose epilogues and
// cone-step functors it reuses.
//
// mode 0 (setup, scs.py:170-196): g = (I + Q_z)^{-1} h with h = (c, b):
//   rhs = c - A^T b ; CG on (I + A^T A) z1 = rhs ; z2 = b + A z1 ;
//   denom = 1 + c.z1 + b.z2   -> g_x slice, g_y rows, state[DENOM]
// mode 1 (iterate, scs.py:314-413): the splitting iteration, the same
//   arithmetic as k_scs with every A^T reduce-scattered, every dot product
//   reduced over the world, and the CG residual all-gathered.

struct ShardArgs {
  GridBar* bar; double* partials;
  DevPlan F, Aj;
  DevCones K;
  cgb_scs_settings st;
  cgb_shard_comm comm;
  cgb_shard_work w;
  const double* b;   // m: this rank's rows of b
  const double* c;   // nl: this rank's slice of c
  int64_t n, m, x0, nl;
  double pr_scale, dr_scale, eps_floor, setup_tol;
  int64_t max_steps;
  int mode;
};

// CG on (I + A^T A) x = rhs from r (= xfull[x0:x0+nl]) with rns = r.r;
// the k_scs cg_loop (normal recipe, lam = 1) with world reductions.
// track: cx += alpha c.p and bax += alpha b.t follow c.x and b.(A x).
template <int TD>
__device__ int64_t cg_shard(const DevPlan& F, const DevPlan& Aj, const ShardArgs& a,
                            double* x, double* gx, double* ax, bool track, double& rns,
                            double delta, double floor_, int64_t max_iter, GridSync& gs,
                            cgbs::World& W, double* cx, double* bax) {
  const cgb_shard_comm* cm = &a.comm;
  double* xfull = cm->xfull[cm->rank];
  const double* rs = xfull + a.x0;   // r, this rank's slice
  double* ib = cm->inbox[cm->rank];
  double* p = a.w.p;
  double* t = a.w.t;
  const int64_t nl = a.nl, m = a.m;
  int64_t k = 0;
  double beta = 0.0;
  while (sqrt(rns) > delta && rns > floor_ && (double)max_iter > (double)k) {
    const int first = k == 0;
    // phase F: t = A r + beta t_old (rows), p = r + beta p_old (slice)
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    {
      EpiT et{t, track ? a.b : nullptr, beta, first, 0, m};
      apply_plan<TD>(F, InVec{xfull, nullptr, 0.0}, et, s, gs);
      double pp = 0.0, cp = 0.0;
      if (first) {
        if (track) pdots<false, true>(nl, rs, p, a.c, beta, pp, cp);
        else pdots<false, false>(nl, rs, p, a.c, beta, pp, cp);
      } else {
        if (track) pdots<true, true>(nl, rs, p, a.c, beta, pp, cp);
        else pdots<true, false>(nl, rs, p, a.c, beta, pp, cp);
      }
      s[1] += pp;
      s[2] += cp;
    }
    cgbs::world_reduce<4>(gs, W, s, false);
    const double alpha = rns / (1.0 * s[1] + s[0]);
    if (track) {
      *cx += alpha * s[2];
      *bax += alpha * s[3];
    }
    // phase A1: A^T t reduce-scattered into the owners' inboxes; ax += alpha t
    {
      cgbs::EpiPush ep{cm};
      apply_plan<TD>(Aj, InVec{t, nullptr, 0.0}, ep, nullptr, gs);
      if (ax) {
        AxUpd f{ax, alpha};
        const double* src[2] = {ax, t};
        bulk_stream<2>(m, src, f);
      }
    }
    cgbs::world_barrier(gs, W, true);
    // phase A2: the CG update of the slice (EpiCgUpd's arithmetic), the new
    // r all-gathered into every rank's x copy
    double rr[1] = {0.0};
    {
      double acc = 0.0;
      auto upd = [&](int64_t i) {
        const double y = cgbs::inbox_sum(cm, ib, nl, i);
        const double rv = rs[i];
        const double pv = first ? 0.0 : p[i];
        const double xv = x[i];
        const double gv = gx ? gx[i] : 0.0;
        const double pp = first ? rv : rv + beta * pv;
        const double qq = 1.0 * pp + y;
        const double rn = rv - alpha * qq;
        p[i] = pp;
        x[i] = xv + alpha * pp;
        if (gx) gx[i] = gv + alpha * y;
        cgbs::push_all(cm, a.x0 + i, rn);
        acc += rn * rn;
      };
      cgbs::slice_loop(nl, upd);
      rr[0] = acc;
    }
    cgbs::world_reduce<1>(gs, W, rr, true);
    beta = rr[0] / rns;
    rns = rr[0];
    ++k;
  }
  return k;
}

template <int TD>
__global__ void __launch_bounds__(CGB_BLOCK, CGB_MINB) k_shard(const __grid_constant__ ShardArgs a)
#if CGB_TU_SHARD
{
  tma_init();
  GridSync gs(a.bar, a.partials);
  const DevPlan& F = *cache_plan(0, a.F);
  const DevPlan& Aj = *cache_plan(1, a.Aj);
  const cgb_shard_comm* cm = &a.comm;
  const cgb_shard_work& Wk = a.w;
  double* state = Wk.state;
  cgbs::World W{cm, (unsigned long long)state[CGB_ST_EPOCH]};
  const int me = cm->rank;
  double* xfull = cm->xfull[me];
  double* ib = cm->inbox[me];
  const int64_t m = a.m, x0 = a.x0, nl = a.nl;
  const cgb_scs_settings& S = a.st;

  if (a.mode == 0) {
    // ---- setup solve: g = (I + Q_z)^{-1} (c, b)   (scs.py:190-196)
    {
      cgbs::EpiPush ep{cm};
      apply_plan<TD>(Aj, InVec{a.b, nullptr, 0.0}, ep, nullptr, gs);
    }
    cgbs::world_barrier(gs, W, true);
    double s[2] = {0.0, 0.0};
    {
      double s0 = 0.0, s1 = 0.0;
      auto f = [&](int64_t i) {   // EpiRhs with x0 = 0, A^T A x0 = 0
        const double y = cgbs::inbox_sum(cm, ib, nl, i);
        const double rhs = a.c[i] - y;
        const double rr = rhs - (0.0 + 0.0);
        cgbs::push_all(cm, x0 + i, rr);
        Wk.gxs[i] = 0.0;
        s0 += rhs * rhs;
        s1 += rr * rr;
      };
      cgbs::slice_loop(nl, f);
      s[0] = s0;
      s[1] = s1;
    }
    cgbs::world_reduce<2>(gs, W, s, true);
    double rns = s[1];
    const double delta = a.setup_tol * sqrt(s[0]);
    const double floor_ = a.eps_floor * s[0];
    const int64_t k = cg_shard<TD>(F, Aj, a, Wk.gxs, nullptr, nullptr, false, rns, delta, floor_,
                                   S.cg_max_iter, gs, W, nullptr, nullptr);
    // z2 = b + A z1 on the rows, from the all-gathered z1
    {
      auto f = [&](int64_t i) { cgbs::push_all(cm, x0 + i, Wk.gxs[i]); };
      cgbs::slice_loop(nl, f);
    }
    cgbs::world_barrier(gs, W, true);
    double h[2] = {0.0, 0.0};
    {
      EpiZ2 e{nullptr, Wk.gy, a.b, a.b};
      apply_plan<TD>(F, InVec{xfull, nullptr, 0.0}, e, h, gs);
      h[1] = side_dot(nl, a.c, Wk.gxs);
    }
    cgbs::world_reduce<2>(gs, W, h, false);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      state[CGB_ST_DENOM] = 1.0 + (h[1] + h[0]);
      state[CGB_ST_SETUP_CG] = (double)k;
      state[CGB_ST_EPOCH] = (double)W.epoch;
    }
    return;
  }

  // ---- splitting iterations (scs.py:314-413)
  double k = state[CGB_ST_K], since = state[CGB_ST_SINCE], status = state[CGB_ST_STATUS];
  double cgt = state[CGB_ST_CGT];
  double pr = state[CGB_ST_PR], dr = state[CGB_ST_DR], gap = state[CGB_ST_GAP];
  double lastcg = state[CGB_ST_LASTCG];
  double utau = state[CGB_ST_TAU], kappa = state[CGB_ST_KAPPA];
  const double denom = state[CGB_ST_DENOM];
  const DevCones& K = a.K;
  double* wy = Wk.wy;
  // running scalars: b.(A x) follows x through the CG updates; b.w_y is
  // summed by every cone step for the next subspace step (enters that
  // reduction once: rank 0, thread 0)
  double bax = 0.0, bwy_part = 0.0;
  {
    double s[2] = {side_dot(m, a.b, Wk.tax), side_dot(m, a.b, wy)};
    cgbs::world_reduce<2>(gs, W, s, false);
    bax = s[0];
    bwy_part = (me == 0 && blockIdx.x == 0 && threadIdx.x == 0) ? s[1] : 0.0;
  }
  int64_t steps = 0;
  while (steps < a.max_steps && (double)S.max_iters > k && !(status > 0.5)) {
    const double wtau = utau + kappa;
    const double vtau = kappa;
    const double since2 = since + 1.0;
    const bool is_check = since2 > (double)S.check_interval - 0.5;
    const bool last = steps + 1 >= a.max_steps || k + 1.0 >= (double)S.max_iters;
    const bool need_resid = is_check;
    const int write_u = need_resid || last;

    // -- subspace step: rhs = w_x - A^T w_y ; r0 = rhs - (x0 + A^T A x0)
    {
      cgbs::EpiPush ep{cm};
      apply_plan<TD>(Aj, InVec{wy, nullptr, 0.0}, ep, nullptr, gs);
    }
    cgbs::world_barrier(gs, W, true);
    double s[4] = {0.0, 0.0, 0.0, bwy_part};
    {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      auto f = [&](int64_t i) {
        const double y = cgbs::inbox_sum(cm, ib, nl, i);
        const double xv = Wk.cgx[i];
        const double rhs = Wk.wx[i] - y;
        const double rr = rhs - (xv + Wk.gx[i]);
        cgbs::push_all(cm, x0 + i, rr);
        s0 += rhs * rhs;
        s1 += rr * rr;
        s2 += a.c[i] * xv;
      };
      cgbs::slice_loop(nl, f);
      s[0] += s0;
      s[1] += s1;
      s[2] += s2;
    }
    cgbs::world_reduce<4>(gs, W, s, true);
    const double tol_k = cg_tolerance_graph(k, S);
    const double delta = tol_k * sqrt(s[0]);
    const double floor_ = a.eps_floor * s[0];
    double rns = s[1];
    double cx = s[2];
    const double bwy = s[3];
    const int64_t cgk = cg_shard<TD>(F, Aj, a, Wk.cgx, Wk.gx, Wk.tax, true, rns, delta, floor_,
                                     S.cg_max_iter, gs, W, &cx, &bax);
    const double tau_t = (wtau + (cx + (bwy + bax))) / denom;

    // -- cone step onto R^n x K* x R+   (scs.py:358-366)
    ConeStep cs{wy, Wk.tax, Wk.gy, Wk.vy, Wk.uy, wy, a.b, tau_t, write_u};
    double bw = 0.0;
    {  // free x block: w_x = u_x = p1 - tau~ g_x ; all-gathered for the check
      auto f = [&](int64_t i) {
        const double ut = fma(-tau_t, Wk.gxs[i], Wk.cgx[i]);
        Wk.wx[i] = ut;
        if (need_resid) cgbs::push_all(cm, x0 + i, ut);
      };
      cgbs::slice_loop(nl, f);
    }
    for (int sg_i = 0; sg_i < K.nseg; ++sg_i) {
      const DevSeg sg = K.seg[sg_i];
      if (sg.kind != SEG_ZERO && sg.kind != SEG_NONNEG) continue;
      ConeElem f{&cs, sg.begin, sg.kind, 0.0};
      const double* src[5] = {wy + sg.begin, Wk.tax + sg.begin, Wk.gy + sg.begin,
                              Wk.vy + sg.begin, a.b + sg.begin};
      bulk_stream<5>(sg.end - sg.begin, src, f);
      bw += f.bw;
    }
    {  // small SOC blocks wholly on this rank: one warp per cone
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
    for (int64_t cc = gtid(); cc < K.nexp; cc += gsize()) {
      const int64_t off = K.exp_off[cc];
      const double z0 = cs.src(off), z1 = cs.src(off + 1), z2 = cs.src(off + 2);
      double p0 = z0, p1 = z1, p2 = z2;
      exp_project_dual(p0, p1, p2);
      bw += a.b[off] * cs.store(off, z0, p0);
      bw += a.b[off + 1] * cs.store(off + 1, z1, p1);
      bw += a.b[off + 2] * cs.store(off + 2, z2, p2);
    }
    if (K.nlarge > 0) {
      // world-reduced SOC blocks: this rank's pieces, pass A (tail^2, head)
      double red[2 * CGB_MAX_LARGE_SOC];
#pragma unroll
      for (int i = 0; i < 2 * CGB_MAX_LARGE_SOC; ++i) red[i] = 0.0;
      for (int sg_i = 0; sg_i < K.nseg; ++sg_i) {
        const DevSeg sg = K.seg[sg_i];
        if (sg.kind != SEG_SOC_LARGE && sg.kind != SEG_SOC_TAIL) continue;
        const bool head = sg.kind == SEG_SOC_LARGE;
        const int64_t b0 = sg.begin + (head ? 1 : 0), len = sg.end - b0;
        SocPassA f{tau_t, nullptr, 0.0};
        const double* src[4] = {wy + b0, Wk.tax + b0, Wk.gy + b0, Wk.vy + b0};
        bulk_stream<4>(len, src, f);
        red[sg.slot] += f.acc;
        if (head && blockIdx.x == 0 && threadIdx.x == 0) red[K.nlarge + sg.slot] += cs.src(sg.begin);
      }
      cgbs::world_reduce<2 * CGB_MAX_LARGE_SOC>(gs, W, red, false);
      for (int sg_i = 0; sg_i < K.nseg; ++sg_i) {
        const DevSeg sg = K.seg[sg_i];
        if (sg.kind != SEG_SOC_LARGE && sg.kind != SEG_SOC_TAIL) continue;
        const bool head = sg.kind == SEG_SOC_LARGE;
        const double t = red[K.nlarge + sg.slot];
        const SocCoef sc(t, sqrt(red[sg.slot]));
        const int64_t b0 = sg.begin + (head ? 1 : 0), len = sg.end - b0;
        SocPassB2 f{&cs, b0, sc, 0.0};
        const double* src[5] = {wy + b0, Wk.tax + b0, Wk.gy + b0, Wk.vy + b0, a.b + b0};
        bulk_stream<5>(len, src, f);
        bw += f.bw;
        if (head && blockIdx.x == 0 && threadIdx.x == 0)
          bw += a.b[sg.begin] * cs.store(sg.begin, t, sc.head(t));
      }
    }
    const double utau_n = fmax(tau_t - vtau, 0.0);
    kappa = (vtau - tau_t) + utau_n;
    utau = utau_n;
    bwy_part = bw;
    if (need_resid) cgbs::world_barrier(gs, W, true);
    else gs.sync();

    k += 1.0;
    cgt += (double)cgk;
    lastcg = (double)cgk;

    if (need_resid) {
      // -- termination measures (scs.py:369-402); xfull holds u_x
      double q[3] = {0.0, 0.0, 0.0};
      {
        EpiRawP ep{Wk.vy, a.b, utau};
        apply_plan<TD>(F, InVec{xfull, nullptr, 0.0}, ep, q, gs);
        q[2] = side_dot(m, a.b, Wk.uy);
        cgbs::EpiPush eq{cm};
        apply_plan<TD>(Aj, InVec{Wk.uy, nullptr, 0.0}, eq, nullptr, gs);
      }
      cgbs::world_reduce<3>(gs, W, q, true);
      double d[3] = {0.0, 0.0, 0.0};
      {
        double d0 = 0.0, d1 = 0.0, d2 = 0.0;
        auto f = [&](int64_t i) {
          const double y = cgbs::inbox_sum(cm, ib, nl, i);
          const double cc = a.c[i];
          const double raw = y + utau * cc;
          d0 += raw * raw;
          const double inf = raw - utau * cc;
          d1 += inf * inf;
          d2 += cc * Wk.wx[i];
        };
        cgbs::slice_loop(nl, f);
        d[0] = d0;
        d[1] = d1;
        d[2] = d2;
      }
      cgbs::world_reduce<3>(gs, W, d, false);
      const double eps = S.eps;
      const double pos = utau > 0.0 ? 1.0 : 0.0;
      const double tinv = pos / (utau + (1.0 - pos));
      pr = a.pr_scale * (sqrt(q[0]) * tinv);
      dr = a.dr_scale * (sqrt(d[0]) * tinv);
      const double ctx = d[2], bty = q[2];
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
      const double res_i = sqrt(d[1]) / (den_i + (1.0 - pos_i));
      const double inf_ok = pos_i * (eps > res_i ? 1.0 : 0.0);
      const double cert = tau_small * (2.0 * inf_ok + (1.0 - inf_ok) * (3.0 * unb_ok));
      const double cand = solved + (1.0 - solved) * cert;
      const double not_set = 1.0 - (status > 0.5 ? 1.0 : 0.0);
      status = status + not_set * cand;
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
    state[CGB_ST_TAU] = utau;
    state[CGB_ST_KAPPA] = kappa;
    state[CGB_ST_EPOCH] = (double)W.epoch;
  }
}
#else
;
#endif
