"""ctypes binding of the C ABI in include/cgb200.h.

The shared library ``lib/libcgb200.so`` is built in-tree (see build.py /
__graft_entry__.build()).  There is no CPU fallback: if the library or a
sm_100 device is missing, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
LIB_PATH = os.environ.get("CGB200_LIB") or os.path.join(LIB_DIR, "libcgb200.so")

ABI_VERSION = 4

# error codes
CGB_OK = 0
CGB_EINVAL = -1
CGB_ENODEV = -2

LEAF_IDENTITY, LEAF_DENSE, LEAF_CSR, LEAF_CONV1D, LEAF_CORR1D, LEAF_CONV2D, LEAF_CORR2D = range(7)
LEAF_FLAG_SEPARABLE = 1
CONE_ZERO, CONE_NONNEG, CONE_SOC, CONE_EXP = range(4)
RECIPE_DIRECT, RECIPE_NORMAL = 0, 1

ST_K, ST_SINCE, ST_STATUS, ST_CGT, ST_PR, ST_DR, ST_GAP, ST_LASTCG = range(8)
ST_TAU, ST_KAPPA, ST_DENOM, ST_EPOCH, ST_SETUP_CG, ST_RES_U, ST_RES_I = range(8, 15)
MAX_RANKS = 8
MBOX_STRIDE = 24
STATE_LEN = 16

_i32, _i64, _f64, _vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p


class Leaf(ctypes.Structure):
    _fields_ = [("kind", _i32), ("reserved", _i32), ("rows", _i64), ("cols", _i64),
                ("val", _vp), ("rowptr", _vp), ("colidx", _vp), ("ld", _i64),
                ("k0", _i64), ("k1", _i64), ("n0", _i64), ("n1", _i64)]


class Term(ctypes.Structure):
    _fields_ = [("leaf", _i32), ("in_buf", _i32), ("row_origin", _i64), ("in_off", _i64),
                ("alpha", _f64)]


class RowBlock(ctypes.Structure):
    _fields_ = [("row_begin", _i64), ("row_end", _i64), ("out_buf", _i32), ("level", _i32),
                ("term_begin", _i32), ("term_end", _i32)]


class PlanDesc(ctypes.Structure):
    _fields_ = [("in_len", _i64), ("out_len", _i64), ("nleaves", _i32), ("nterms", _i32),
                ("nrowblocks", _i32), ("ntemps", _i32), ("leaves", ctypes.POINTER(Leaf)),
                ("terms", ctypes.POINTER(Term)), ("rowblocks", ctypes.POINTER(RowBlock)),
                ("temp_len", ctypes.POINTER(_i64))]


class CgResult(ctypes.Structure):
    _fields_ = [("iterations", _i64), ("final_residual_norm", _f64), ("b_norm", _f64),
                ("converged", _i32), ("reserved", _i32)]


class ScsSettingsC(ctypes.Structure):
    _fields_ = [("eps", _f64), ("max_iters", _i64), ("check_interval", _i64),
                ("cg_base_tol", _f64), ("cg_tol_cap", _f64), ("cg_tol_power", _f64),
                ("cg_eps_factor", _f64), ("cg_max_iter", _i64), ("cert_tau_ratio", _f64)]


SCS_NO_ZERO_SKIP = 1


class ScsProblemC(ctypes.Structure):
    _fields_ = [("struct_size", _i64), ("n", _i64), ("m", _i64), ("A", _vp), ("K", _vp),
                ("b", _vp), ("c", _vp), ("g", _vp), ("denom", _f64), ("pr_scale", _f64),
                ("dr_scale", _f64), ("flags", _i32), ("reserved", _i32)]

    def __init__(self, **kw):
        super().__init__(struct_size=ctypes.sizeof(ScsProblemC), **kw)


class ScsWorkC(ctypes.Structure):
    _fields_ = [(nm, _vp) for nm in ("u", "v", "w", "cgx", "tax", "gx", "r", "p0", "p1",
                                     "q", "t", "state")]


class ShardCommC(ctypes.Structure):
    _fields_ = [("world", _i32), ("rank", _i32), ("x_begin", _i64 * (MAX_RANKS + 1)),
                ("inbox", _vp * MAX_RANKS), ("xfull", _vp * MAX_RANKS),
                ("mbox", _vp * MAX_RANKS)]


class ShardProblemC(ctypes.Structure):
    _fields_ = [("struct_size", _i64), ("n", _i64), ("m", _i64), ("A", _vp), ("K", _vp),
                ("b", _vp), ("c", _vp), ("pr_scale", _f64), ("dr_scale", _f64),
                ("setup_tol", _f64)]

    def __init__(self, **kw):
        super().__init__(struct_size=ctypes.sizeof(ShardProblemC), **kw)


class ShardWorkC(ctypes.Structure):
    _fields_ = [(nm, _vp) for nm in ("cgx", "gx", "p", "wx", "gxs", "wy", "vy", "uy", "tax",
                                     "t", "gy", "state")]


# every symbol include/cgb200.h declares, with its ctypes signature
SIGNATURES = {
    "cgb_abi_version": (ctypes.c_int, []),
    "cgb_last_error": (ctypes.c_char_p, []),
    "cgb_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_vp)]),
    "cgb_ctx_destroy": (ctypes.c_int, [_vp]),
    "cgb_ctx_geometry": (ctypes.c_int, [_vp, ctypes.POINTER(_i32)]),
    "cgb_op_create": (ctypes.c_int, [_vp, ctypes.POINTER(PlanDesc), ctypes.POINTER(PlanDesc),
                                     ctypes.POINTER(_vp)]),
    "cgb_op_destroy": (ctypes.c_int, [_vp]),
    "cgb_op_apply": (ctypes.c_int, [_vp, _vp, ctypes.c_int, _vp, _vp, _vp]),
    "cgb_cones_create": (ctypes.c_int, [_vp, ctypes.POINTER(_i32), ctypes.POINTER(_i64), _i32,
                                        ctypes.POINTER(_vp)]),
    "cgb_cones_destroy": (ctypes.c_int, [_vp]),
    "cgb_cones_project": (ctypes.c_int, [_vp, _vp, ctypes.c_int, _vp, _vp, _vp]),
    "cgb_cg_solve": (ctypes.c_int, [_vp, _vp, ctypes.c_int, _f64, _vp, _vp, _f64, _i64,
                                    ctypes.POINTER(CgResult), _vp]),
    "cgb_scs_run": (ctypes.c_int, [_vp, ctypes.POINTER(ScsProblemC),
                                   ctypes.POINTER(ScsSettingsC), ctypes.POINTER(ScsWorkC),
                                   _i64, ctypes.c_int, _vp]),
    "cgb_inner_solve": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _f64, _i64, _vp, _vp, _vp,
                                       ctypes.POINTER(CgResult), ctypes.POINTER(_f64), _vp]),
    "cgb_debug_barrier": (ctypes.c_int, [_vp, _i64, ctypes.c_int, _vp]),
    "cgb_scs_profile": (ctypes.c_int, [_vp, _vp]),
    "cgb_ctx_set_grid": (ctypes.c_int, [_vp, _i32]),
    "cgb_shard_cones_create": (ctypes.c_int, [_vp, ctypes.POINTER(_i32), ctypes.POINTER(_i64),
                                              ctypes.POINTER(_i64), ctypes.POINTER(_i32),
                                              ctypes.POINTER(_i32), _i32, _i64, _i32,
                                              ctypes.POINTER(_vp)]),
    "cgb_shard_run": (ctypes.c_int, [_vp, ctypes.POINTER(ShardProblemC),
                                     ctypes.POINTER(ScsSettingsC), ctypes.POINTER(ShardCommC),
                                     ctypes.POINTER(ShardWorkC), ctypes.c_int, _i64, _vp]),
    "cgb_ipc_alloc": (ctypes.c_int, [ctypes.c_int, _i64, ctypes.POINTER(_vp), ctypes.c_char_p]),
    "cgb_ipc_open": (ctypes.c_int, [ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(_vp)]),
    "cgb_ipc_close": (ctypes.c_int, [_vp]),
    "cgb_ipc_free": (ctypes.c_int, [_vp]),
}


class CgbError(RuntimeError):
    """A failure reported by the CUDA library (message from cgb_last_error)."""


_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load and bind libcgb200.so (no CUDA device needed to load)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise CgbError(
                f"CUDA extension not built: {path} is missing; run "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.cgb_abi_version() != ABI_VERSION:
            raise CgbError("libcgb200.so ABI version mismatch")
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc != CGB_OK:
        msg = load_library().cgb_last_error()
        raise CgbError(f"cgb error {rc}: {msg.decode() if msg else ''}")


class _Context:
    """Per-device persistent-kernel context (grid barrier + reduction banks)."""

    def __init__(self, device: int, grid: int = 0):
        lib = load_library()
        h = _vp()
        check(lib.cgb_ctx_create(device, ctypes.byref(h)))
        self.handle = h
        self.device = device
        if grid:
            check(lib.cgb_ctx_set_grid(h, int(grid)))

    def geometry(self):
        out = (_i32 * 3)()
        check(load_library().cgb_ctx_geometry(self.handle, out))
        return tuple(out)


_ctxs: dict[int, _Context] = {}


def new_context(device: int, grid: int = 0) -> _Context:
    """A private cgb_ctx (own grid barrier and reduction banks), e.g. one per
    rank when several ranks of a sharded solve share a device."""
    return _Context(device, grid)


def device_context():
    """The cgb_ctx for torch's current CUDA device; raises without CUDA."""
    import torch
    if not torch.cuda.is_available():
        raise CgbError("no CUDA device: the conegraph B200 path has no CPU fallback")
    dev = torch.cuda.current_device()
    ctx = _ctxs.get(dev)
    if ctx is None:
        ctx = _ctxs[dev] = _Context(dev)
    return ctx


def stream_handle():
    import torch
    return _vp(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> _vp:
    return _vp(t.data_ptr()) if t is not None else _vp(0)
