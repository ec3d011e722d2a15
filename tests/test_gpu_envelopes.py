"""Parity at BASELINE-family sizes against committed rounding envelopes.

tests/golden/bench_envelopes.jsonl holds, for members of every BASELINE
config's family at CPU-feasible sizes (configs[0] at its full size), the
REAL reference's solve (or the pinned oracle's, for the north-star
extensions the reference lacks: 2-d convolution, exponential cones) of the
unperturbed instance and of copies with b, c multiplied by 1 + U(-d, d)
for d = 4 ulp, 1e-11 and (configs[0]) 1e-10 (tests/golden/
make_bench_envelopes.py).  Why the larger d: the device's summation order
moves the first iterate by ~6e-12 relative (tools/diverge_bench.py) and
the splitting map amplifies it; on configs[0] the device's own counts over
reduction orders (grid sizes 37..148, 1..4 sharded ranks:
tools/grid_spread.py) are {760, 780, 840, 920}, and the reference's counts
under d = 1e-10 are {740, 760, 780, 840, 920} -- the same distribution,
which a 4-ulp envelope ({840}) does not show.  The device solve of the same
instance (rebuilt from the same host-side generator, digest-checked) must
satisfy the north-star rule against that envelope:

  * zero-spread envelope -> the same status, the exact iteration count and
    the objective to 1e-6 relative;
  * otherwise            -> the same status, an iteration count inside
    [min - w, max + w] with w = max(check_interval, 2 % of the unperturbed
    count) -- a handful of samples underestimates a chaotic envelope's
    tails, and 2 % is the north star's own count tolerance -- and the
    objective inside the envelope's objective range widened by its spread.
"""

import importlib.util
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
_spec = importlib.util.spec_from_file_location(
    "make_bench_envelopes", os.path.join(HERE, "golden", "make_bench_envelopes.py"))
MBE = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(MBE)

ENV = MBE.load_envelopes()
# an instance is tested once its envelope has the unperturbed solve and at
# least 3 perturbed ones (the n = 1e6 bench instance's oracle solves take
# ~2.6 h of CPU each)
NAMES = sorted(n for n, e in ENV.items()
               if e["unperturbed"] is not None and len(e["perturbed"]) >= 3 and n in MBE.INSTANCES)


def _check(name, sol, settings):
    e = ENV[name]
    recs = [e["unperturbed"]] + e["perturbed"]
    its = [r["iterations"] for r in recs]
    pobjs = [r["pobj"] for r in recs if r["status"] == "solved"]
    ref = e["unperturbed"]
    assert sol.status == ref["status"], (sol.status, ref["status"])
    if min(its) == max(its):
        assert sol.iterations == ref["iterations"], (sol.iterations, its)
        if sol.status == "solved":
            assert abs(sol.pobj - ref["pobj"]) <= 1e-6 * max(1.0, abs(ref["pobj"])), \
                (sol.pobj, ref["pobj"])
    else:
        w = max(settings.check_interval, 0.02 * ref["iterations"])
        assert min(its) - w <= sol.iterations <= max(its) + w, (sol.iterations, its)
        if sol.status == "solved":
            lo, hi = min(pobjs), max(pobjs)
            spread = hi - lo
            assert lo - spread <= sol.pobj <= hi + spread, (sol.pobj, lo, hi)


@pytest.mark.parametrize("name", NAMES)
def test_device_solve_inside_reference_envelope(name):
    from paper_1609_03488_b200 import scs
    spec, _, _ = MBE.INSTANCES[name]
    prob = MBE.workload(spec).problem()
    # (the host generator's BLAS can differ in the last bit from the build
    # container's, b_digest; that is inside the envelope's 4-ulp family)
    st = scs.ScsSettings(eps=MBE.EPS, max_iters=MBE.MAX_ITERS)
    sol = scs.solve(prob, st)
    _check(name, sol, st)


@pytest.mark.parametrize("name", [n for n in NAMES if n.startswith("lasso_")])
def test_sharded_solve_inside_reference_envelope(name):
    """The row-sharded solver (2 ranks sharing the GPU) under the same rule:
    configs[0] / configs[3] family lasso instances."""
    from paper_1609_03488_b200 import scs, shard
    spec, _, _ = MBE.INSTANCES[name]
    prob = MBE.workload(spec).problem()
    st = scs.ScsSettings(eps=MBE.EPS, max_iters=MBE.MAX_ITERS)
    grp = shard.ShardGroup(prob, st, world=2)
    try:
        sol = grp.solve()
    finally:
        grp.close()
    _check(name, sol, st)


def test_envelopes_cover_every_baseline_config():
    """Every BASELINE config's family has a committed envelope."""
    fam = {n.split("_")[0] for n in NAMES}
    assert {"lasso", "deconv1d", "deconv2d", "soc", "logreg"} <= fam, fam
    assert np.all([len(ENV[n]["perturbed"]) >= 4 for n in NAMES])
