"""Sharded solver vs the single-GPU solver vs the oracle on one lasso
instance: iterate distance at increasing k, and the full solves.
    python tools/shard_diag.py [m n seed]"""

import json
import os
import sys

import numpy as np
import scipy.sparse

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch
    from oracle import scs_ref
    from paper_1609_03488_b200 import canon, linop, scs, shard
    m, n, seed = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (2000, 300, 5)))
    rng = np.random.default_rng(seed)
    A = scipy.sparse.random(m, n, density=0.01, random_state=rng, format="csc")
    A.data = rng.standard_normal(A.nnz)
    x = rng.standard_normal(n) * (rng.uniform(size=n) < 0.1)
    b = A @ x + 0.01 * rng.standard_normal(m)
    lam = 0.1 * float(np.max(np.abs(A.T @ b)))
    prob = canon.build_lasso(canon.LassoProblem(linop.sparse_csc(A), b, lam))

    class P:
        pass
    op = P()
    op.A, op.b, op.c, op.K = prob.A.expr, prob.b, prob.c, prob.K
    s = scs_ref.ScsOracleSettings(eps=1e-3, max_iters=20000)
    cached = scs_ref.prepare_subspace(op, s.setup_cg_tol, s.cg_max_iter)
    ks = [1, 20, 40, 80, 160, 320]
    ref = {k: st for k, st in scs_ref.iterate(op, s, cached, max(ks)) if k in ks}
    st = scs.ScsSettings(eps=1e-3, max_iters=20000)
    out = {"instance": [m, n, seed]}
    single = scs.build_scs_graph(prob, st)
    for world in (1, 2):
        grp = shard.ShardGroup(prob, st, world=world)
        grp.reset()
        single.reset()
        done = 0
        rows = []
        for k in ks:
            if k not in ref:
                break
            grp.run(k - done)
            single.run(k - done)
            done = k
            torch.cuda.synchronize()
            ux, uy, vy, _, _ = grp.gather()
            sts = grp.states()
            u = np.concatenate([ux, uy, [sts[0][8]]])
            su = single.buf["u"].cpu().numpy()
            r = ref[k]
            sc = 1.0 + np.linalg.norm(r.u)
            rows.append({"k": k, "shard_vs_oracle": float(np.linalg.norm(u - r.u) / sc),
                         "single_vs_oracle": float(np.linalg.norm(su - r.u) / sc),
                         "shard_vs_single": float(np.linalg.norm(u - su) / sc),
                         "cgt": [sts[0][3], float(single.state()[3]), r.cgt]})
        sol = grp.solve()
        grp.close()
        out[f"world{world}"] = {"trace": rows, "status": sol.status, "iterations": sol.iterations,
                                "pobj": sol.pobj}
    ssol = scs.solve(prob, st)
    out["single"] = {"status": ssol.status, "iterations": ssol.iterations, "pobj": ssol.pobj}
    osol, _ = scs_ref.scs_solve(op, s)
    out["oracle"] = {"status": osol.status, "iterations": osol.iterations, "pobj": osol.pobj}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
