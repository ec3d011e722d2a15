"""Generate golden vectors by running the REAL reference (conegraph) here.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Writes tests/golden/*.npz.  The fixtures are committed; nothing at test,
smoke or bench time reads /root/reference.  Every fixture stores its
inputs (raw arrays plus an operator-tree serialization) next to the
reference's outputs, so the oracle and the CUDA path can be replayed on
exactly the same data.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import scipy.sparse

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)

from conegraph import canon, linop  # noqa: E402
from conegraph.cg import CgSpec, cg_solve, make_normal_operator, operator_recipe  # noqa: E402
from conegraph.cones import (ConeProduct, NonNegCone, SecondOrderCone,  # noqa: E402
                             ZeroCone, project)
from conegraph.linop import (AdjointOf, Compose, Conv1D, DenseMatrix,  # noqa: E402
                             Identity, Scale, SparseMatrix, Sum, VStack, ZeroOp)
from conegraph.scs import (ConeProblem, ScsSettings, build_scs_graph,  # noqa: E402
                           iterate_states, prepare_subspace, solve,
                           subspace_project)
import oracles  # noqa: E402  (reference test helpers: random_operator)

OUT = os.path.dirname(os.path.abspath(__file__))


# -- operator tree serialization ------------------------------------------

def ser(expr, arrays: dict) -> dict:
    """Expression -> JSON-able dict; array payloads go into ``arrays``."""
    def put(a):
        key = f"arr{len(arrays)}"
        arrays[key] = np.asarray(a)
        return key
    k = type(expr).__name__
    if k == "DenseMatrix":
        return {"k": k, "values": put(expr.values)}
    if k == "SparseMatrix":
        mat = expr.matrix.tocsc()
        return {"k": k, "data": put(mat.data), "indices": put(mat.indices),
                "indptr": put(mat.indptr), "m": mat.shape[0], "n": mat.shape[1]}
    if k == "Conv1D":
        return {"k": k, "kernel": put(expr.kernel), "n": expr.n}
    if k == "Identity":
        return {"k": k, "n": expr.rows}
    if k == "ZeroOp":
        return {"k": k, "m": expr.rows, "n": expr.cols}
    if k == "Scale":
        return {"k": k, "alpha": expr.alpha, "child": ser(expr.child, arrays)}
    if k in ("Sum", "Compose"):
        return {"k": k, "left": ser(expr.left, arrays), "right": ser(expr.right, arrays)}
    if k == "VStack":
        return {"k": k, "children": [ser(c, arrays) for c in expr.children]}
    if k == "AdjointOf":
        return {"k": k, "child": ser(expr.child, arrays)}
    raise TypeError(k)


def cone_spec(K: ConeProduct) -> list:
    return [[type(f).__name__, f.dim] for f in K.factors]


def save(name: str, arrays: dict, meta: dict) -> None:
    arrays = dict(arrays)
    arrays["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrays)


# -- SCS end-to-end cases ----------------------------------------------------

def lp_geq_one():
    return ConeProblem(linop.dense([[-1.0]]), np.array([-1.0]), np.array([1.0]),
                       ConeProduct([NonNegCone(1)]))


def scs_cases():
    cases = []
    cases.append(("lp_geq_one", lp_geq_one(), ScsSettings(eps=1e-6, max_iters=2000), {}))
    cases.append(("lp_zero_obj", ConeProblem(linop.dense([[-1.0]]), np.array([0.0]),
                                             np.array([0.0]), ConeProduct([NonNegCone(1)])),
                  ScsSettings(eps=1e-6, max_iters=2000), {}))
    A_eq = np.array([[-1.0, -1.0], [-1.0, 0.0], [0.0, -1.0]])
    cases.append(("lp_equality", ConeProblem(linop.dense(A_eq), np.array([-1.0, 0.0, 0.0]),
                                             np.array([1.0, 1.0]),
                                             ConeProduct([ZeroCone(1), NonNegCone(2)])),
                  ScsSettings(eps=1e-6, max_iters=5000), {}))
    cases.append(("infeasible", ConeProblem(linop.dense([[-1.0], [1.0]]),
                                            np.array([-1.0, -1.0]), np.array([1.0]),
                                            ConeProduct([NonNegCone(2)])),
                  ScsSettings(eps=1e-6, max_iters=5000), {}))
    cases.append(("unbounded", ConeProblem(linop.dense([[-1.0]]), np.array([0.0]),
                                           np.array([-1.0]), ConeProduct([NonNegCone(1)])),
                  ScsSettings(eps=1e-6, max_iters=5000), {}))
    rows = linop.vstack([linop.zero(1, 2), linop.identity(2)])
    cases.append(("soc_ball", ConeProblem(linop.scale(-1.0, rows), np.array([1.0, 0.0, 0.0]),
                                          np.array([3.0, -4.0]),
                                          ConeProduct([SecondOrderCone(3)])),
                  ScsSettings(eps=1e-5, max_iters=10000), {}))
    rng = np.random.default_rng(17)
    Ad = rng.standard_normal((10, 6))
    cases.append(("max_iters", ConeProblem(linop.dense(Ad), rng.standard_normal(10),
                                           rng.standard_normal(6), ConeProduct([NonNegCone(10)])),
                  ScsSettings(eps=1e-12, max_iters=40), {}))
    # strictly feasible random LPs (test_scs._feasible_problem recipe)
    for seed, (n, m) in [(11, (4, 6)), (13, (5, 8)), (29, (12, 30))]:
        rng = np.random.default_rng(seed)
        Ad = rng.standard_normal((m, n))
        x0 = rng.standard_normal(n)
        s0 = np.abs(rng.standard_normal(m)) + 0.1
        y0 = np.abs(rng.standard_normal(m)) + 0.1
        cases.append((f"feasible_lp_{seed}", ConeProblem(linop.dense(Ad), Ad @ x0 + s0,
                                                         -Ad.T @ y0, ConeProduct([NonNegCone(m)])),
                      ScsSettings(eps=1e-5, max_iters=20000), {}))
    # paper families (canon builders)
    for fam, n, seed, eps in [("dense", 20, 21, 1e-4), ("dense", 50, 3, 1e-4),
                              ("sparse", 50, 3, 1e-4), ("conv", 50, 3, 1e-4),
                              ("conv", 20, 31, 1e-4), ("dense", 30, 7, 1e-3)]:
        A, b, _ = canon.gen_data(fam, n, seed)
        lam = 0.1 * canon.lasso_lambda_max(A, b)
        prob = canon.build_lasso(canon.LassoProblem(A, b, lam))
        cases.append((f"lasso_{fam}_{n}_{seed}", prob, ScsSettings(eps=eps, max_iters=20000),
                      {"family": fam, "n": n, "seed": seed, "lam": lam, "kind": "lasso"}))
    for n, seed, eps in [(100, 5, 1e-4), (20, 32, 1e-4), (100, 0, 1e-3)]:
        c, b, _ = canon.gen_spike_data(n, seed)
        prob = canon.build_deconv(canon.DeconvProblem(c, b))
        cases.append((f"deconv_{n}_{seed}", prob, ScsSettings(eps=eps, max_iters=20000),
                      {"n": n, "seed": seed, "kind": "deconv"}))
    # generalized deconvolution: signal n, short kernel k (north-star shape, tiny)
    for n, k, seed in [(300, 11, 1), (1000, 101, 2)]:
        rng = np.random.default_rng(seed)
        kern = canon.gaussian_kernel(k)
        x_hat = np.zeros(n)
        x_hat[rng.choice(n, 5, replace=False)] = rng.uniform(0.0, 10.0, 5)
        C = linop.conv1d(kern, n)
        b = C.forward(x_hat) + 0.01 * rng.standard_normal(n + k - 1)
        stuffed = linop.vstack([
            linop.hstack([linop.identity(n), linop.zero(n, 1)]),
            linop.hstack([linop.zero(1, n), linop.identity(1)]),
            linop.hstack([C, linop.zero(n + k - 1, 1)]),
        ])
        prob = ConeProblem(linop.scale(-1.0, stuffed),
                           np.concatenate([np.zeros(n), [0.0], -b]),
                           np.concatenate([np.zeros(n), [1.0]]),
                           ConeProduct([NonNegCone(n), SecondOrderCone(n + k)]))
        cases.append((f"deconv1d_n{n}_k{k}", prob, ScsSettings(eps=1e-3, max_iters=20000),
                      {"n": n, "k": k, "seed": seed, "kind": "deconv1d"}))
    return cases


def gen_scs():
    for name, prob, st, info in scs_cases():
        arrays: dict = {}
        tree = ser(prob.A.expr, arrays)
        sol = solve(prob, st)
        cached = prepare_subspace(prob, st.setup_cg_tol, st.cg_max_iter)
        meta = {"case": name, "tree": tree, "cones": cone_spec(prob.K),
                "settings": {k: getattr(st, k) for k in st.__dataclass_fields__},
                "status": sol.status, "iterations": sol.iterations,
                "avg_cg": sol.avg_cg_iterations, "pobj": sol.pobj, "dobj": sol.dobj,
                "pr": sol.primal_residual, "dr": sol.dual_residual, "gap": sol.gap,
                "denom": cached.denom, "info": info}
        arrays.update(b=prob.b, c=prob.c, x=sol.x, y=sol.y, s=sol.s, g=cached.g)
        # first iterates of the loop for per-iteration parity
        graph = build_scs_graph(prob, st)
        us, vs, cgts = [], [], []
        for k, state in iterate_states(graph, min(25, st.max_iters)):
            us.append(state[0].copy())
            vs.append(state[1].copy())
            cgts.append(float(state[6][0]))
        arrays.update(trace_u=np.array(us), trace_v=np.array(vs), trace_cgt=np.array(cgts))
        save("scs_" + name, arrays, meta)
        print(f"scs_{name}: {sol.status} iters={sol.iterations} avg_cg={sol.avg_cg_iterations:.3f}")


# -- CG cases -----------------------------------------------------------------

def gen_cg():
    arrays: dict = {}
    cases = []
    rng = np.random.default_rng(202)
    for i in range(6):
        n = int(rng.integers(10, 120))
        M = rng.standard_normal((n, n)) / np.sqrt(n)
        Ad = M.T @ M + np.eye(n)
        b = rng.standard_normal(n)
        res = cg_solve(CgSpec(operator_recipe(linop.dense(Ad)), b, np.zeros(n)))
        t = ser(DenseMatrix(Ad), arrays)
        ib = f"b{i}"
        ix = f"x{i}"
        arrays[ib], arrays[ix] = b, res.x
        cases.append({"recipe": "direct", "lam": None, "tree": t, "b": ib, "x": ix,
                      "iters": res.iterations, "frn": res.final_residual_norm,
                      "converged": res.converged, "tol": 1e-8})
    for i, (fam, n, seed) in enumerate([("dense", 30, 30), ("sparse", 60, 60),
                                        ("conv", 40, 40), ("conv", 200, 1)]):
        A, b, _ = canon.gen_data(fam, n, seed)
        spec = canon.build_regls(canon.RegLsProblem(A, b, 1.0))
        res = cg_solve(spec)
        t = ser(A.expr, arrays)
        ib, ix = f"nb{i}", f"nx{i}"
        arrays[ib], arrays[ix] = spec.b, res.x
        cases.append({"recipe": "normal", "lam": 1.0, "tree": t, "b": ib, "x": ix,
                      "iters": res.iterations, "frn": res.final_residual_norm,
                      "converged": res.converged, "tol": 1e-8})
    save("cg_cases", arrays, {"cases": cases})
    print(f"cg_cases: {len(cases)}")


# -- operator apply cases ------------------------------------------------------

def gen_linop():
    arrays: dict = {}
    cases = []
    rng = np.random.default_rng(7)
    for i in range(60):
        op = oracles.random_operator(rng, max_dim=40, depth=4)
        x = rng.standard_normal(op.cols)
        y = rng.standard_normal(op.rows)
        t = ser(op.expr, arrays)
        keys = {}
        for nm, val in (("x", x), ("y", y), ("ax", op.forward(x)), ("aty", op.adjoint_apply(y))):
            keys[nm] = f"{nm}{i}"
            arrays[keys[nm]] = val
        cases.append({"tree": t, "rows": op.rows, "cols": op.cols,
                      "nnz": int(linop.nnz_estimate(op)), **keys})
    # the stuffed paper operators
    for fam in ("dense", "sparse", "conv"):
        A, b, _ = canon.gen_data(fam, 30, 4)
        prob = canon.build_lasso(canon.LassoProblem(A, b, 0.3))
        op = prob.A
        x = rng.standard_normal(op.cols)
        y = rng.standard_normal(op.rows)
        i = len(cases)
        t = ser(op.expr, arrays)
        keys = {}
        for nm, val in (("x", x), ("y", y), ("ax", op.forward(x)), ("aty", op.adjoint_apply(y))):
            keys[nm] = f"{nm}{i}"
            arrays[keys[nm]] = val
        cases.append({"tree": t, "rows": op.rows, "cols": op.cols,
                      "nnz": int(linop.nnz_estimate(op)), **keys})
    save("linop_cases", arrays, {"cases": cases})
    print(f"linop_cases: {len(cases)}")


# -- cone projection + subspace cases -------------------------------------------

def gen_cones():
    rng = np.random.default_rng(303)
    arrays = {}
    meta = []
    for j, cone in enumerate([ZeroCone(5), NonNegCone(5), SecondOrderCone(5),
                              SecondOrderCone(1), SecondOrderCone(33)]):
        V = 3.0 * rng.standard_normal((200, cone.dim))
        V[0] = 0.0
        V[1, 0] = -1.0  # t<0, u=0
        P = np.stack([project(cone, v) for v in V])
        arrays[f"v{j}"], arrays[f"p{j}"] = V, P
        meta.append([type(cone).__name__, cone.dim])
    save("cone_cases", arrays, {"cones": meta})
    print("cone_cases")


def gen_subspace():
    rng = np.random.default_rng(404)
    arrays = {}
    cases = []
    for i in range(10):
        n = int(rng.integers(1, 11))
        m = int(rng.integers(1, 11))
        Ad = rng.standard_normal((m, n))
        prob = ConeProblem(linop.dense(Ad), rng.standard_normal(m), rng.standard_normal(n),
                           ConeProduct([NonNegCone(m)]))
        cached = prepare_subspace(prob)
        w = rng.standard_normal(n + m + 1)
        out = subspace_project(w, cached)
        for nm, val in (("A", Ad), ("b", prob.b), ("c", prob.c), ("w", w), ("out", out),
                        ("g", cached.g)):
            arrays[f"{nm}{i}"] = val
        cases.append({"n": n, "m": m, "denom": cached.denom})
    save("subspace_cases", arrays, {"cases": cases})
    print("subspace_cases")


if __name__ == "__main__":
    gen_linop()
    gen_cones()
    gen_cg()
    gen_subspace()
    gen_scs()
