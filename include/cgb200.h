/*
 * cgb200.h -- C ABI of the B200-native conegraph solver path.
 *
 * The reference (conegraph, Python) exposes this path as Python calls on
 * operator / cone / solver objects.  Each entry point below replaces one
 * of those calls; the reference file:line it stands in for is cited.
 * Host code (paper_1609_03488_b200/*.py) binds this header with ctypes;
 * INTEGRATION.md shows the binding a conegraph maintainer would add.
 *
 * Conventions
 *   - All vectors are float64 DEVICE pointers (cudaMalloc / torch CUDA
 *     tensors) unless a parameter says "host".
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *   - Every function returns 0 on success or a negative CGB_E* code; the
 *     message of the last failure on the calling thread is available from
 *     cgb_last_error().  There is no CPU fallback: without a usable
 *     sm_100 device every compute call fails with CGB_ENODEV.
 *   - A cgb_ctx owns the persistent-kernel resources (grid barrier,
 *     reduction banks) and the plan temporaries of the operators created
 *     on it.  Every launching call on a ctx is ordered after the previous
 *     one: a call on a different stream first makes that stream wait for
 *     the ctx's last stream (event), and host threads are serialised by a
 *     ctx mutex.  Calls on one ctx therefore never overlap on the device;
 *     use one ctx per concurrent solver.  Operators and cones must be used
 *     with the ctx they were created on (CGB_EINVAL otherwise).
 */
#ifndef CGB200_H
#define CGB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CGB_ABI_VERSION 4

/* ---- error codes --------------------------------------------------------- */
#define CGB_OK 0
#define CGB_EINVAL (-1)   /* bad argument / inconsistent descriptor        */
#define CGB_ENODEV (-2)   /* no usable CUDA device                          */
#define CGB_ECUDA (-3)    /* CUDA runtime error (message has details)       */
#define CGB_ENOMEM (-4)   /* device allocation failed                       */
#define CGB_ECOOP (-5)    /* cooperative launch not possible                */

/* ---- operator plans (linop.py) ------------------------------------------- */
/* Leaf kinds: the primitive maps an operator expression lowers to.         */
#define CGB_LEAF_IDENTITY 0 /* rows = cols = n                                */
#define CGB_LEAF_DENSE 1    /* val row-major rows x cols, leading dim ld      */
#define CGB_LEAF_CSR 2      /* rowptr[rows+1] (int64), colidx (int32), val     */
#define CGB_LEAF_CONV1D 3   /* full conv, kernel val[k0]: rows n0+k0-1, cols n0 */
#define CGB_LEAF_CORR1D 4   /* valid corr (adjoint of CONV1D): rows n0, cols n0+k0-1 */
#define CGB_LEAF_CONV2D 5   /* full 2-d conv of n0 x n1 image, kernel k0 x k1 */
#define CGB_LEAF_CORR2D 6   /* valid 2-d corr (adjoint of CONV2D)             */
/* cgb_leaf.reserved flag for CONV2D / CORR2D: the kernel is rank one
 * (K = u v^T), apply it as a column pass and a row pass.  The library
 * re-verifies the factorization and applies K directly if it fails.       */
#define CGB_LEAF_FLAG_SEPARABLE 1

typedef struct cgb_leaf {
  int32_t kind;
  int32_t reserved;
  int64_t rows, cols;
  const double* val;      /* dense values / CSR values / conv kernel        */
  const int64_t* rowptr;  /* CSR only                                       */
  const int32_t* colidx;  /* CSR only                                       */
  int64_t ld;             /* dense leading dimension                        */
  int64_t k0, k1;         /* conv kernel extent(s)                          */
  int64_t n0, n1;         /* conv signal / image extent(s)                  */
} cgb_leaf;

/* One block term: out[row_origin + i] += alpha * leaf(in[in_off + .])[i]   */
typedef struct cgb_term {
  int32_t leaf;        /* index into leaves                                  */
  int32_t in_buf;      /* 0 = apply input, t+1 = plan temporary t            */
  int64_t row_origin;  /* output row of leaf row 0                           */
  int64_t in_off;      /* input index of leaf column 0                       */
  double alpha;
} cgb_term;

/* A row range of one output buffer, all of whose rows see the same terms.  */
typedef struct cgb_rowblock {
  int64_t row_begin, row_end;
  int32_t out_buf;     /* 0 = apply output, t+1 = plan temporary t           */
  int32_t level;       /* execution level; 0 = last (writes final output)    */
  int32_t term_begin, term_end; /* range into terms (empty => zero rows)     */
} cgb_rowblock;

/* Flattened lowering of one operator direction (forward or adjoint).        */
typedef struct cgb_plan_desc {
  int64_t in_len, out_len;
  int32_t nleaves, nterms, nrowblocks, ntemps;
  const cgb_leaf* leaves;         /* host arrays; copied by cgb_op_create    */
  const cgb_term* terms;
  const cgb_rowblock* rowblocks;  /* must tile every buffer it writes        */
  const int64_t* temp_len;        /* ntemps entries                          */
} cgb_plan_desc;

typedef struct cgb_ctx cgb_ctx;
typedef struct cgb_op cgb_op;
typedef struct cgb_cones cgb_cones;

/* Library / device */
int cgb_abi_version(void);
const char* cgb_last_error(void);
/* Create the persistent-kernel context on `device`; fails with CGB_ENODEV
 * unless the device is sm_100 (B200 class). */
int cgb_ctx_create(int device, cgb_ctx** out);
int cgb_ctx_destroy(cgb_ctx* ctx);
/* grid geometry of the persistent kernels: {num_sms, blocks_per_sm, threads} */
int cgb_ctx_geometry(const cgb_ctx* ctx, int32_t* out3);

/* Operator = forward + adjoint plan.  Replaces linop.Operator
 * (linop.py:266-321): adjoint derived structurally by the host lowering
 * (linop.py:187-207) and shipped as its own plan. */
int cgb_op_create(cgb_ctx* ctx, const cgb_plan_desc* fwd, const cgb_plan_desc* adj,
                  cgb_op** out);
int cgb_op_destroy(cgb_op* op);
/* y = A x (adjoint=0) or y = A^T x (adjoint=1).
 * Replaces Operator.forward / Operator.adjoint_apply (linop.py:299-307). */
int cgb_op_apply(cgb_ctx* ctx, const cgb_op* op, int adjoint, const double* x, double* y,
                 void* stream);

/* ---- cones (cones.py) ------------------------------------------------------ */
#define CGB_CONE_ZERO 0
#define CGB_CONE_NONNEG 1
#define CGB_CONE_SOC 2
#define CGB_CONE_EXP 3
int cgb_cones_create(cgb_ctx* ctx, const int32_t* kinds, const int64_t* dims, int32_t ncones,
                     cgb_cones** out);
int cgb_cones_destroy(cgb_cones* K);
/* out = Pi_K(v) (dual=0) or Pi_{K*}(v) (dual=1); v, out length = total dim.
 * Replaces cones.project_product / project_product_dual (cones.py:93-115)
 * and the solver's in-graph dual projection (scs.py:250-283). */
int cgb_cones_project(cgb_ctx* ctx, const cgb_cones* K, int dual, const double* v, double* out,
                      void* stream);

/* ---- conjugate gradient (cg.py) ------------------------------------------- */
#define CGB_RECIPE_DIRECT 0  /* solve A x = b, A square SPD  (cg.py:64-68)     */
#define CGB_RECIPE_NORMAL 1  /* solve (lam I + A^T A) x = b (cg.py:71-84)      */
typedef struct cgb_cg_result {
  int64_t iterations;
  double final_residual_norm;  /* sqrt(r_norm_sq)                             */
  double b_norm;
  int32_t converged;           /* frn <= tol * ||b||  (cg.py:152-161)         */
  int32_t reserved;
} cgb_cg_result;
/* x holds x_init on entry and the solution on exit.  Synchronises `stream`
 * to fill *res (host).  Replaces cg.cg_solve (cg.py:164-165). */
int cgb_cg_solve(cgb_ctx* ctx, const cgb_op* op, int recipe, double lam, const double* b,
                 double* x, double tol, int64_t max_iter, cgb_cg_result* res, void* stream);

/* ---- homogeneous self-dual embedding solver (scs.py) ---------------------- */
typedef struct cgb_scs_settings {       /* ScsSettings (scs.py:84-118)          */
  double eps;
  int64_t max_iters;
  int64_t check_interval;
  double cg_base_tol, cg_tol_cap, cg_tol_power, cg_eps_factor;
  int64_t cg_max_iter;                  /* resolved (None -> 10 n)              */
  double cert_tau_ratio;
} cgb_scs_settings;

typedef struct cgb_scs_problem {
  int64_t struct_size; /* sizeof(cgb_scs_problem): checked by cgb_scs_run    */
  int64_t n, m;
  const cgb_op* A;
  const cgb_cones* K;
  const double* b;     /* m */
  const double* c;     /* n */
  const double* g;     /* n+m : cached (I+Q_z)^{-1} h from cgb_inner_solve   */
  double denom;        /* 1 + h.g                                            */
  double pr_scale;     /* 1 / (1 + ||b||)                                    */
  double dr_scale;     /* 1 / (1 + ||c||)                                    */
  /* The loop measures the index ranges outside which b and c are exactly
   * zero once per call (one device pass) and skips those loads; the
   * trajectory is bitwise the same as with CGB_SCS_NO_ZERO_SKIP.          */
  int32_t flags;
  int32_t reserved;
} cgb_scs_problem;

/* Device buffers owned by the caller.  N = n + m + 1.
 * Invariant of the embedding: v = (0, s, kappa) -- the x block of v is zero
 * on entry (cgb_scs_run keeps it zero and never reads it).  u is written on
 * check iterations (and on the last iteration a call can run); between them
 * only u's tau entry is current.  p1 and q are reserved (unused). */
typedef struct cgb_scs_work {
  double* u; double* v; double* w;   /* N each; w = u + v maintained          */
  double* cgx;                        /* n : CG warm start (p1 of last iter)   */
  double* tax;                        /* m : A cgx, tracked through CG updates */
  double* gx;                         /* n : A^T A cgx, tracked likewise       */
  double* r; double* p0; double* p1; double* q;  /* n each : CG r, p (p0)      */
  double* t;                          /* m : A p scratch                       */
  double* state;                      /* CGB_STATE_LEN doubles, see below      */
} cgb_scs_work;

/* state[] layout (all float64; integers stored exactly) */
#define CGB_ST_K 0        /* iterations done                                  */
#define CGB_ST_SINCE 1    /* iterations since last check                      */
#define CGB_ST_STATUS 2   /* 0 running, 1 solved, 2 infeasible, 3 unbounded   */
#define CGB_ST_CGT 3      /* total inner CG iterations                        */
#define CGB_ST_PR 4       /* last computed primal residual                    */
#define CGB_ST_DR 5       /* last computed dual residual                      */
#define CGB_ST_GAP 6      /* last computed gap                                */
#define CGB_ST_LASTCG 7   /* CG iterations of the last splitting iteration    */
#define CGB_ST_TAU 8       /* shard solver: u_tau                               */
#define CGB_ST_KAPPA 9     /* shard solver: v_tau (kappa)                       */
#define CGB_ST_DENOM 10    /* shard solver: 1 + h.g of the setup solve          */
#define CGB_ST_EPOCH 11    /* shard solver: world synchronisations so far       */
#define CGB_ST_SETUP_CG 12 /* shard solver: CG iterations of the setup solve    */
#define CGB_ST_RES_U 13    /* last check: unboundedness certificate residual   */
#define CGB_ST_RES_I 14    /* last check: infeasibility certificate residual   */
#define CGB_STATE_LEN 16

#define CGB_SCS_NO_ZERO_SKIP 1  /* cgb_scs_problem.flags: stream all of b and c */

/* Run splitting iterations on device until the status latches, k reaches
 * settings->max_iters, or `max_steps` iterations have run in this call.
 * All loop state lives in `work`, so calls resume where they stopped.
 * resid_every_iter=1 evaluates the residual triple every iteration (trace
 * mode); otherwise only on check iterations, which is all the status latch
 * reads (scs.py:404-409).  Asynchronous on `stream`.
 * Replaces the while-loop of build_scs_graph / solve_built
 * (scs.py:314-469, 541-568). */
int cgb_scs_run(cgb_ctx* ctx, const cgb_scs_problem* prob, const cgb_scs_settings* st,
                cgb_scs_work* work, int64_t max_steps, int resid_every_iter, void* stream);

/* Inner block solve [[I, A^T], [-A, I]] z = (d1, d2) by CG on I + A^T A:
 * rhs = d1 - A^T d2, z1 = CG(rhs, x0 = z1 on entry), z2 = d2 + A z1.
 * z = (z1, z2) has length n + m; scratch needs 4n + 2m doubles.
 * If hdot != NULL, *hdot = c.z1 + b.z2 (host) is also returned.
 * Synchronises `stream`.  Replaces scs._solve_inner_block (scs.py:170-187),
 * the engine of prepare_subspace / subspace_project (scs.py:190-214). */
int cgb_inner_solve(cgb_ctx* ctx, const cgb_op* op, const double* d1, const double* d2,
                    double* z, double tol, int64_t max_iter, const double* c, const double* b,
                    double* scratch, cgb_cg_result* res, double* hdot, void* stream);

/* Phase profiler: when dev_acc != NULL, later cgb_scs_run calls on this ctx
 * add the nanoseconds spent in each phase to dev_acc[0..15] (device
 * memory): 0 subspace rhs, 1 CG t = A p, 2 CG A^T t + updates, 3 cone
 * step x block, 4 cone step elementwise / small SOC, 5 large-SOC pass A,
 * 6 large-SOC pass B, 7 residual check, 8 per-launch setup.  Profiling adds
 * two grid barriers per iteration to separate the cone sub-phases.  NULL
 * disables. */
int cgb_scs_profile(cgb_ctx* ctx, double* dev_acc);

/* ---- row-sharded solver (one rank per GPU) ------------------
 * The stuffed operator's rows are split into contiguous ranges, one per
 * rank; x-space vectors are split into contiguous slices.  Each rank runs
 * one persistent kernel; ranks exchange data only through peer memory:
 * A^T partial products are stored straight into the inbox of the rank
 * owning those columns (reduce-scatter in the adjoint's epilogue), the CG
 * residual is stored into every rank's full-length x copy (all-gather),
 * and dot products meet in per-rank mailboxes.  Replaces, for a problem
 * whose A is too large for one GPU, the same calls as cgb_inner_solve +
 * cgb_scs_run (scs.py:170-196, 314-413); the reference itself has no
 * sharding (the decomposition is restated in oracle/shard_ref.py). */
#define CGB_MAX_RANKS 8
#define CGB_MBOX_STRIDE 24  /* doubles per mailbox slot (16 values, sequence, pad) */

typedef struct cgb_shard_comm {
  int32_t world, rank;
  int64_t x_begin[CGB_MAX_RANKS + 1];  /* x slices: rank q owns [x_begin[q], x_begin[q+1]) */
  /* device pointers valid on THIS rank's device (peer-mapped):           */
  double* inbox[CGB_MAX_RANKS];  /* rank q's inbox: world x len_q doubles   */
  double* xfull[CGB_MAX_RANKS];  /* rank q's full-length x copy: n doubles  */
  double* mbox[CGB_MAX_RANKS];   /* rank q's mailbox: 2*CGB_MAX_RANKS*CGB_MBOX_STRIDE
                                    doubles, zeroed before the first call   */
} cgb_shard_comm;

typedef struct cgb_shard_problem {
  int64_t struct_size;  /* sizeof(cgb_shard_problem)                        */
  int64_t n;            /* global x-space length                            */
  int64_t m;            /* this rank's rows                                 */
  const cgb_op* A;      /* this rank's rows of A: forward n -> m            */
  const cgb_cones* K;   /* this rank's cone pieces (cgb_shard_cones_create) */
  const double* b;      /* m : this rank's rows of b                        */
  const double* c;      /* this rank's x slice of c                         */
  double pr_scale;      /* 1 / (1 + ||b||), global                          */
  double dr_scale;      /* 1 / (1 + ||c||), global                          */
  double setup_tol;     /* setup CG tolerance (ScsSettings.setup_cg_tol)    */
} cgb_shard_problem;

typedef struct cgb_shard_work {
  /* x slice (x_begin[rank+1] - x_begin[rank] doubles each) */
  double* cgx;   /* CG warm start p1                                        */
  double* gx;    /* A^T A cgx, tracked                                      */
  double* p;     /* CG direction                                            */
  double* wx;    /* w_x = u_x                                               */
  double* gxs;   /* g_x of the setup solve                                  */
  /* rows (m doubles each) */
  double* wy; double* vy; double* uy;
  double* tax;   /* A cgx, tracked                                          */
  double* t;     /* CG scratch                                              */
  double* gy;    /* g_y of the setup solve                                  */
  double* state; /* CGB_STATE_LEN; TAU = KAPPA = 1 and the rest 0 at start  */
} cgb_shard_work;

/* This rank's cone pieces.  Piece i covers local rows [begin[i], end[i])
 * of cone kind kinds[i]; a SOC cut by a rank boundary (or longer than the
 * single-GPU small-SOC limit) is world-reduced: soc_id[i] in [0, nsoc) is
 * its index in the global list of such cones (-1 otherwise) and
 * has_head[i] says whether its head entry is on this rank.  Exponential
 * cones and small SOCs must not be cut. */
int cgb_shard_cones_create(cgb_ctx* ctx, const int32_t* kinds, const int64_t* begin,
                           const int64_t* end, const int32_t* soc_id, const int32_t* has_head,
                           int32_t npieces, int64_t m, int32_t nsoc, cgb_cones** out);
/* mode 0: the setup solve (g, denom into work / state); mode 1: up to
 * max_steps splitting iterations.  Every rank must make the same sequence
 * of calls; each launch is asynchronous on `stream`.  max_steps < 0 only
 * validates the arguments (a caller launching several ranks checks them
 * all first: a rank that launched alone would wait for its peers). */
int cgb_shard_run(cgb_ctx* ctx, const cgb_shard_problem* prob, const cgb_scs_settings* st,
                  const cgb_shard_comm* comm, cgb_shard_work* work, int mode,
                  int64_t max_steps, void* stream);

/* Persistent-kernel grid of a ctx: 0 = one CTA per SM (default); g > 0
 * uses g CTAs, e.g. two ranks sharing one device in tests. */
int cgb_ctx_set_grid(cgb_ctx* ctx, int32_t grid);

/* Peer memory across processes: a cudaMalloc'd buffer and its 64-byte
 * CUDA IPC handle; open maps a peer's handle on the current device. */
int cgb_ipc_alloc(int device, int64_t bytes, void** ptr, void* handle64);
int cgb_ipc_open(int device, const void* handle64, void** ptr);
int cgb_ipc_close(void* ptr);
int cgb_ipc_free(void* ptr);

/* ---- diagnostics ------------------------------------------------------------ */
/* Run `iters` grid barriers (mode 0) or grid reductions (mode 1) in one
 * persistent launch; time it with events on `stream` to get the per-phase
 * synchronisation cost that bounds small problems. */
int cgb_debug_barrier(cgb_ctx* ctx, int64_t iters, int mode, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CGB200_H */
