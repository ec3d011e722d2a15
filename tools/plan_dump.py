"""Print the lowered forward / adjoint plans of a bench workload's stuffed
operator (levels, row blocks, leaf kinds) -- development aid.

usage: python tools/plan_dump.py <workload>
"""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1609_03488_b200 import _lib, scs  # noqa: E402

KIND = {v: k for k, v in vars(_lib).items() if k.startswith("LEAF_") and not k.startswith("LEAF_FLAG")}


class A:
    workload = sys.argv[1]
    n = bench.N_SIGNAL


wl = bench.make_workload(A)
prob = wl.problem()
plan = scs.build_scs_graph(prob, scs.ScsSettings(eps=wl.eps, max_iters=10))
for name in ("fwd", "adj"):
    b = getattr(plan.dev, name)
    print(f"{name}: levels={b.nlevels} rowblocks={b.nrowblocks} terms={b.nterms} "
          f"temps={b.temp_len} temp_level={b.temp_level}")
    _, arr_terms, arr_rbs, _ = b.keep_c
    for i in range(b.nrowblocks):
        rb = arr_rbs[i]
        kinds = [KIND.get(b.leaves[arr_terms[t].leaf].kind, "?") + f"({b.leaves[arr_terms[t].leaf].rows}x{b.leaves[arr_terms[t].leaf].cols})"
                 for t in range(rb.term_begin, rb.term_end)]
        print(f"  rb[{rb.row_begin},{rb.row_end}) buf={rb.out_buf} level={rb.level}: {kinds}")
