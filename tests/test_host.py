"""CPU-side checks of the product (no GPU): the C-ABI library loads and
exports every entry point include/cgb200.h declares, the host API mirrors
the reference's names and error behaviour, and the plan lowering / stuffing
logic (pure host code) is consistent.  Nothing here calls a compute entry
point: without a GPU those must fail loudly (also checked)."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "cgb200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(cgb_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1609_03488_b200 import _lib
    names = _header_functions()
    assert len(names) >= 15, names
    lib = _lib.load_library()          # loads and binds without a device
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for nm in names:
        assert hasattr(raw, nm), f"libcgb200.so does not export {nm}"
        assert nm in _lib.SIGNATURES, f"_lib.py does not bind {nm}"
    assert set(_lib.SIGNATURES) == set(names)
    assert lib.cgb_abi_version() == _lib.ABI_VERSION


def test_struct_layouts_match_header():
    """ctypes mirrors of the ABI structs: field order / sizes as declared."""
    from paper_1609_03488_b200 import _lib
    assert ctypes.sizeof(_lib.Leaf) == 4 + 4 + 8 * 2 + 8 * 3 + 8 * 5
    assert ctypes.sizeof(_lib.Term) == 4 + 4 + 8 + 8 + 8
    assert ctypes.sizeof(_lib.RowBlock) == 8 * 2 + 4 * 4
    assert ctypes.sizeof(_lib.ScsWorkC) == 8 * 12
    assert ctypes.sizeof(_lib.CgResult) == 8 + 8 + 8 + 4 + 4


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1609_03488_b200 import _lib, linop
    with pytest.raises((_lib.CgbError, RuntimeError)):
        linop.dense([[1.0, 2.0]]).forward(np.array([1.0, 1.0]))
    lib = _lib.load_library()
    h = ctypes.c_void_p()
    assert lib.cgb_ctx_create(0, ctypes.byref(h)) == _lib.CGB_ENODEV
    assert b"device" in lib.cgb_last_error().lower() or lib.cgb_last_error()


def test_reference_api_surface():
    """Every public name of the reference modules exists in the mirror."""
    import paper_1609_03488_b200 as pkg
    from paper_1609_03488_b200 import canon, cg, cones, linop, scs
    for mod, names in [
        (linop, ["Operator", "DenseMatrix", "SparseMatrix", "Conv1D", "Identity", "ZeroOp",
                 "Scale", "Sum", "Compose", "VStack", "AdjointOf", "derive_adjoint", "forward",
                 "adjoint_apply", "dense", "sparse_csc", "conv1d", "identity", "zero", "scale",
                 "vstack", "hstack", "materialize_dense", "nnz_estimate", "storage_nbytes",
                 "conv_full", "corr_valid", "LinOpError", "DimensionMismatch",
                 "MaterializeCapExceeded"]),
        (cones, ["ZeroCone", "NonNegCone", "SecondOrderCone", "ConeProduct", "project",
                 "project_dual", "project_product", "project_product_dual", "contains",
                 "contains_product", "ConeError"]),
        (cg, ["CgSpec", "CgResult", "operator_recipe", "make_normal_operator",
              "build_cg_graph", "solve_built", "cg_solve"]),
        (scs, ["ConeProblem", "ScsSettings", "ScsIterate", "ScsSolution", "TraceRecord",
               "PrecomputedSolve", "prepare_subspace", "subspace_project", "residuals",
               "build_scs_graph", "iterate_states", "solve_built", "solve"]),
        (canon, ["RegLsProblem", "LassoProblem", "DeconvProblem", "build_regls",
                 "lasso_dims", "deconv_dims", "build_lasso", "build_deconv", "gen_data",
                 "gen_spike_data", "regls_objective", "lasso_objective", "deconv_objective",
                 "save_instance", "load_instance"]),
    ]:
        for nm in names:
            assert hasattr(mod, nm), f"{mod.__name__}.{nm}"
    assert pkg.solve is scs.solve


def test_stuffed_dimensions_match_paper_tables():
    """Tables II-III stuffed sizes via the same builders the solver uses."""
    from paper_1609_03488_b200 import canon
    assert canon.lasso_dims(3000, 6000) == (6001, 12002)
    assert canon.lasso_dims(3000, 5999) == (6001, 12001)
    for n in (100, 1000, 10000):
        assert canon.deconv_dims(n) == (n + 1, 3 * n)
    assert canon.deconv_dims(10 ** 6, 101) == (10 ** 6 + 1, 2 * 10 ** 6 + 101)
    assert canon.logreg_dims(200_000, 2000) == (604_000, 1_404_000)


def test_settings_validation_mirrors_reference():
    from paper_1609_03488_b200 import scs
    with pytest.raises(ValueError):
        scs.ScsSettings(eps=0.0)
    with pytest.raises(ValueError):
        scs.ScsSettings(max_iters=0)
    with pytest.raises(ValueError):
        scs.ScsSettings(cg_tol_power=3.0)
    s = scs.ScsSettings()
    assert s.cg_tolerance(0) == 0.1 and s.cg_tolerance(10 ** 9) == 1e-4


def test_operator_algebra_shapes_and_errors():
    from paper_1609_03488_b200 import linop
    A = linop.dense(np.ones((3, 2)))
    B = linop.conv1d([1.0, 2.0, 3.0], 2)        # 4 x 2
    assert (A.T.shape, B.T.shape) == ((2, 3), (2, 4))
    assert A.T.T is A
    with pytest.raises(linop.DimensionMismatch):
        A + B
    with pytest.raises(linop.DimensionMismatch):
        A @ B
    assert linop.nnz_estimate(linop.dense(np.ones((6000, 3000)))) == 18_000_000
    H = linop.hstack([A, linop.identity(3)])
    assert H.shape == (3, 5)


def test_logreg_stuffing_permutation_is_a_bijection():
    """The exp-cone rows are interleaved into (x, y, z) triples by a sparse
    permutation composed on the left of the block operator."""
    from paper_1609_03488_b200 import canon, cones
    rng = np.random.default_rng(0)
    A = rng.standard_normal((7, 3))
    y = np.sign(rng.standard_normal(7))
    prob = canon.build_logreg(canon.LogRegProblem(A, y, 0.1))
    n_st, m_st = canon.logreg_dims(7, 3)
    assert prob.A.shape == (m_st, n_st)
    assert sum(isinstance(f, cones.ExpCone) for f in prob.K.factors) == 14
    perm = prob.A.expr.child.children[1].left.matrix   # Scale(-1, VStack([.., P @ B]))
    assert perm.nnz == 42 and (np.sort(perm.indices) == np.arange(42)).all()
    assert (perm.sum(axis=0) == 1).all() and (perm.sum(axis=1) == 1).all()


def test_nonzero_ranges_of_stuffed_vectors():
    """The b / c nonzero ranges of the stuffed vectors (the loop measures
    them on device and skips loads outside; the host copy feeds
    SolverPlan.bytes_model): exact first/last nonzero, (0, 0) when zero."""
    from paper_1609_03488_b200 import canon, scs
    assert scs._nonzero_range(np.zeros(5)) == (0, 0)
    assert scs._nonzero_range(np.array([0.0, 0.0, 3.0, 0.0, -1.0, 0.0])) == (2, 5)
    assert scs._nonzero_range(np.array([1.0])) == (0, 1)
    n, k = 50, 7
    rng = np.random.default_rng(0)
    sig = rng.standard_normal(n + k - 1)
    c = np.abs(rng.standard_normal(k)) + 0.1
    prob = canon.build_deconv(canon.DeconvProblem(c, sig, n=n))
    # stuffed deconv: b = (0_n, 0, -sig), c = (0_n, 1)
    assert scs._nonzero_range(prob.b) == (n + 1, 2 * n + k)
    assert scs._nonzero_range(prob.c) == (n, n + 1)


def test_abi_problem_struct_layout():
    """ABI v3: cgb_scs_problem starts with struct_size (checked by the
    library) and carries flags instead of caller-supplied b/c ranges."""
    from paper_1609_03488_b200 import _lib
    names = [f[0] for f in _lib.ScsProblemC._fields_]
    assert names[0] == "struct_size" and names[-2:] == ["flags", "reserved"]
    assert ctypes.sizeof(_lib.ScsProblemC) == 8 * 3 + 8 * 5 + 8 * 3 + 4 * 2
    assert _lib.ScsProblemC().struct_size == ctypes.sizeof(_lib.ScsProblemC)
    hdr = open(os.path.join(ROOT, "include", "cgb200.h")).read()
    for nm in names:
        assert nm in hdr
    assert "b_nz_begin" not in hdr
    assert f"#define CGB_ABI_VERSION {_lib.ABI_VERSION}" in hdr


def test_bench_generators_match_canon():
    """bench.py restates the data generators so the reference arm imports
    nothing of the product; they must equal canon's bit for bit."""
    import bench
    from paper_1609_03488_b200 import canon
    for n in (7, 101):
        assert np.array_equal(bench.gaussian_kernel(n), canon.gaussian_kernel(n))
    assert np.array_equal(bench.gaussian_kernel2d(15, 15), canon.gaussian_kernel2d(15, 15))
    a1, y1, w1 = bench.gen_logreg(50, 7, seed=3)
    a2, y2, w2 = canon.gen_logreg(50, 7, seed=3)
    assert np.array_equal(a1, a2) and np.array_equal(y1, y2) and np.array_equal(w1, w2)


@pytest.mark.parametrize("name,kw", [
    ("deconv2d", {"h": 16, "w": 21, "k": 3}),
    ("deconv1d", {"n": 40}),
    ("lasso_dense", {"m": 30, "n": 12}),
    ("lasso_sparse", {"m": 300, "n": 40, "density": 0.05}),
    ("logreg", {"m": 20, "n": 5}),
    ("soc_ls", {"m": 30, "n": 6}),
])
def test_oracle_stuffing_matches_product(name, kw):
    """oracle/canon_ref.py (reference arm) and the product's canon builders
    stuff the same problem: identical b, c, cone dims and operator applies."""
    import bench
    from oracle import linop_ref
    wl = bench.WORKLOADS[name](**kw) if name != "deconv1d" else bench.Deconv1D(kw["n"])
    if name == "deconv1d":
        c, _, _ = wl.data()
    pp, po = wl.problem(), wl.oracle_problem()
    assert np.array_equal(pp.b, po.b) and np.array_equal(pp.c, po.c)
    assert [(type(f).__name__, f.dim) for f in pp.K.factors] == \
        [(type(f).__name__, f.dim) for f in po.K.factors]
    rng = np.random.default_rng(0)
    x = rng.standard_normal(pp.A.cols)
    y = rng.standard_normal(pp.A.rows)
    np.testing.assert_array_equal(linop_ref.forward(pp.A.expr, x), linop_ref.forward(po.A, x))
    np.testing.assert_array_equal(linop_ref.adjoint(pp.A.expr, y), linop_ref.adjoint(po.A, y))


def test_long_conv_kernel_lowered_to_tap_blocks(monkeypatch):
    """A Conv1D longer than the tiled path's 240 taps is lowered to tap
    blocks of <= 240 (plan lowering only; leaf data kept on the host)."""
    import numpy as np
    import torch
    from paper_1609_03488_b200 import _plan
    from paper_1609_03488_b200 import linop as L
    monkeypatch.setattr(_plan, "_cuda", lambda a, dtype=None: torch.from_numpy(
        np.ascontiguousarray(a if dtype is None else a.astype(dtype))))
    e = L.Conv1D(np.ones(10001), 10001)
    for adj in (False, True):
        b = _plan._Builder()
        b.emit(e, adj, 0, 0, 0, 0, 1.0, 0)
        ks = [b.leaves[t[0]].k0 for t in b.terms]
        assert len(ks) == 42 and max(ks) <= _plan.CONV_KMAX and sum(ks) == 10001
        offs = sorted((t[3] if adj else t[2]) for t in b.terms)
        assert offs[0] == 0 and offs[-1] == 10001 - ks[-1]


def test_graph_engine_names_import_and_fail_clearly():
    """The reference's graph-engine exports (conegraph/__init__.py:3-4)
    import from the drop-in package and raise a clear error when used."""
    import pytest
    import paper_1609_03488_b200 as pkg
    from paper_1609_03488_b200.graph import GraphEngineUnavailable
    for name in ("Graph", "LoopSpec", "Node", "NodeId", "debug_dump", "evaluate",
                 "evaluate_args", "topological_order", "while_loop"):
        assert hasattr(pkg, name)
    with pytest.raises(GraphEngineUnavailable):
        pkg.Graph()
    with pytest.raises(GraphEngineUnavailable):
        pkg.evaluate(None)
