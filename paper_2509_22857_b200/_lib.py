"""ctypes binding of libpcnn.so (include/pcnn.h).

The structures below mirror the C declarations field for field (every field
is int64 or double, so there is no padding to disagree about).  The library
is built in-tree by ``__graft_entry__.build()`` / ``make``; importing the
package without it is fine on a CPU-only box, but every device entry point
raises ``PcnnError`` if the library or an sm_100 device is missing -- there
is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import pathlib
from typing import Optional

LIB_PATH = pathlib.Path(__file__).resolve().parent / "libpcnn.so"

c_i64 = ctypes.c_int64
c_f64 = ctypes.c_double

PCNN_OK = 0
PCNN_ERR_TRANSFORM = -4

# unit kinds
UNIT_INGEST, UNIT_CONV, UNIT_LINEAR, UNIT_POLY, UNIT_ADD, UNIT_POLYSKIP = 1, 2, 3, 4, 5, 6
UNIT_AFFINE, UNIT_LOCALPOOL, UNIT_BIPOOL, UNIT_GLOBALPOOL, UNIT_FLATTEN, UNIT_COPYOUT = 7, 8, 9, 10, 11, 12
# fused pool kinds
POOL_NONE, POOL_SUM2, POOL_BI2, POOL_GLOBAL, POOL_LOCAL = 0, 1, 2, 3, 4
# pack kinds
PACK_CAST, PACK_BN_AFFINE, PACK_TC_WEIGHTS, PACK_TC16_WEIGHTS, PACK_TCSS_WEIGHTS = 1, 2, 3, 4, 5
# conv implementations (pcnn_unit_desc.impl)
# unit flags
FLAG_S2D = 1
IMPL_AUTO, IMPL_SIMT, IMPL_TF32, IMPL_F16X2, IMPL_FP32_TENSORS, IMPL_F16X2_SS = 0, 1, 2, 3, 4, 5
# scale opcodes
(OP_FILL, OP_LOAD, OP_MUL, OP_DIV, OP_SUB, OP_POWI, OP_SROOT, OP_AROOT, OP_RECIP, OP_SOLVE,
 OP_CHECK_UNIFORM, OP_CHECK_NONZERO, OP_CHECK_NONNEG, OP_CHECK_CLOSE, OP_CHECK_ALLONE,
 OP_SQRT, OP_STORE, OP_ADD) = range(1, 19)

MAX_FACTORS = 6
ABI_VERSION = 3


class PcnnError(RuntimeError):
    """A libpcnn call failed (message from pcnn_last_error)."""


class TensorDesc(ctypes.Structure):
    _fields_ = [(n, c_i64) for n in ("c", "h", "w", "cb", "nblk", "is_vector", "offset", "scale_log2")]


_UNIT_FIELDS = ("kind", "in_", "in2", "out", "cin", "cout", "kh", "kw", "stride", "pad",
                "w_off", "b_off", "affine_off", "residual", "res_off", "poly_deg", "poly_off",
                "pool", "pool_off", "pool_deg", "pool_order", "in_mode", "in_div_off", "impl",
                "tc_off", "npad", "tc16_off", "tc16_scale_off", "tcss_off", "flags", "pool_geom")


class UnitDesc(ctypes.Structure):
    _fields_ = [(n, c_i64) for n in _UNIT_FIELDS]

    def __init__(self, **kw):
        defaults = {"in_": -1, "in2": -1, "out": -1, "w_off": -1, "b_off": -1, "affine_off": -1,
                    "res_off": -1, "poly_off": -1, "pool_off": -1, "in_div_off": -1, "tc_off": -1,
                    "tc16_off": -1, "tc16_scale_off": -1, "tcss_off": -1}
        defaults.update(kw)
        super().__init__(**defaults)


class PackDesc(ctypes.Structure):
    _fields_ = [(n, c_i64) for n in ("kind", "src", "dst", "n", "rows", "k", "aux", "reserved")]


class ScaleOp(ctypes.Structure):
    _fields_ = [(n, c_i64) for n in ("op", "n", "dst", "a", "b", "sa", "sb", "p", "err")] + \
               [(n, c_f64) for n in ("imm", "rtol", "atol")]


class Factor(ctypes.Structure):
    _fields_ = [(n, c_i64) for n in ("slot", "divide", "d1", "m1", "s1", "d2", "m2", "reserved")]


class RewriteDesc(ctypes.Structure):
    _fields_ = [(n, c_i64) for n in ("dst", "src", "n", "src_arena", "set_const", "n_factors")] + \
               [("value", c_f64), ("f", Factor * MAX_FACTORS)]


_OPT_INT_FIELDS_A = ("size", "split", "halo_tiles", "fuse_projection", "band_pool", "streamk")
_OPT_INT_FIELDS_B = ("flag_sync", "prezero", "linear_out", "pdl", "graph", "ss_mt", "ss_share", "ss_psub",
                     "ss_wres", "tc_stage", "timeline", "image_blocks", "debug", "fused_net", "ss_wide", "epi_pairs",
                     "ss_pair", "scratch_cb4")


class PlanOptions(ctypes.Structure):
    """pcnn_plan_options: every tuning / diagnostic switch of a plan (the
    library reads no environment variables)."""
    _fields_ = [(n, c_i64) for n in _OPT_INT_FIELDS_A] + [("streamk_fill", c_f64)] + \
               [(n, c_i64) for n in _OPT_INT_FIELDS_B] + [("reserved", c_i64 * 3)]

    @classmethod
    def default(cls, **overrides) -> "PlanOptions":
        o = cls()
        lib().pcnn_plan_options_default(ctypes.byref(o))
        for k, v in overrides.items():
            if k not in dict(cls._fields_):
                raise KeyError(f"unknown plan option {k!r}")
            setattr(o, k, v)
        return o

    def as_dict(self) -> dict:
        return {n: getattr(self, n) for n, _ in self._fields_ if n != "reserved"}


# Developer / tooling switches (tools/*.py): environment variable -> option.
# Only these helpers read the environment; Engine() uses explicit options.
ENV_OPTIONS = {
    "PCNN_NO_SPLIT": ("split", 0), "PCNN_NO_SS": ("halo_tiles", 0), "PCNN_NO_PROJ_FUSE": ("fuse_projection", 0),
    "PCNN_NO_BAND": ("band_pool", 0), "PCNN_BAND": ("band_pool", int), "PCNN_NO_STREAMK": ("streamk", 0), "PCNN_FLAGS": ("flag_sync", int),
    "PCNN_NO_PREZERO": ("prezero", 0), "PCNN_NO_LINEAR_OUT": ("linear_out", 0), "PCNN_NO_PDL": ("pdl", 0),
    "PCNN_NO_GRAPH": ("graph", 0), "PCNN_SS_MT": ("ss_mt", int), "PCNN_SS_SHARE": ("ss_share", int),
    "PCNN_SS_PSUB": ("ss_psub", int), "PCNN_SS_WRES": ("ss_wres", int), "PCNN_TC_NOSTAGE": ("tc_stage", 0),
    "PCNN_TC_DEBUG": ("debug", int), "PCNN_STREAMK_FILL": ("streamk_fill", float),
    "PCNN_NO_TIMELINE": ("timeline", 0), "PCNN_NO_NET": ("fused_net", 0), "PCNN_WIDE": ("ss_wide", int), "PCNN_PAIRS": ("epi_pairs", int), "PCNN_PAIR": ("ss_pair", int), "PCNN_SCRATCH_CB4": ("scratch_cb4", int), "PCNN_NO_BLOCKS": ("image_blocks", 0), "PCNN_BLOCKS": ("image_blocks", int),
}


def options_from_env(**overrides) -> "PlanOptions":
    """Defaults, then the PCNN_* developer variables of ENV_OPTIONS, then overrides."""
    kw = {}
    for var, (field, val) in ENV_OPTIONS.items():
        if var in os.environ:
            kw[field] = val(os.environ[var]) if callable(val) else val
    kw.update(overrides)
    return PlanOptions.default(**kw)


_lib: Optional[ctypes.CDLL] = None

SYMBOLS = {
    "pcnn_abi_version": ([], ctypes.c_int),
    "pcnn_last_error": ([], ctypes.c_char_p),
    "pcnn_device_ok": ([], ctypes.c_int),
    "pcnn_workspace_bytes": ([ctypes.POINTER(TensorDesc), ctypes.c_int, ctypes.c_int], ctypes.c_size_t),
    "pcnn_plan_create": ([ctypes.POINTER(UnitDesc), ctypes.c_int, ctypes.POINTER(TensorDesc), ctypes.c_int,
                          ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                          ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "pcnn_plan_create_ex": ([ctypes.POINTER(UnitDesc), ctypes.c_int, ctypes.POINTER(TensorDesc), ctypes.c_int,
                             ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                             ctypes.c_size_t, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "pcnn_plan_options_default": ([ctypes.c_void_p], None),
    "pcnn_plan_timeline": ([ctypes.c_void_p, ctypes.POINTER(c_i64), ctypes.c_int, ctypes.c_void_p], ctypes.c_int),
    "pcnn_plan_unit_launch": ([ctypes.c_void_p, ctypes.c_int], ctypes.c_int),
    "pcnn_plan_destroy": ([ctypes.c_void_p], ctypes.c_int),
    "pcnn_plan_num_launches": ([ctypes.c_void_p], ctypes.c_int),
    "pcnn_plan_unit_impl": ([ctypes.c_void_p, ctypes.c_int], ctypes.c_int),
    "pcnn_plan_tensor_split": ([ctypes.c_void_p, ctypes.c_int], ctypes.c_int),
    "pcnn_plan_status": ([ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "pcnn_plan_last_status": ([ctypes.c_void_p], ctypes.c_int),
    "pcnn_forward": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int],
                     ctypes.c_int),
    "pcnn_forward_host": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "pcnn_forward_host_many": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "pcnn_forward_unit": ([ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
                          ctypes.c_int),
    "pcnn_pack": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(PackDesc), ctypes.c_int, ctypes.c_void_p],
                  ctypes.c_int),
    "pcnn_redistribute": ([ctypes.c_void_p, ctypes.c_void_p, c_i64, ctypes.POINTER(ScaleOp), ctypes.c_int,
                           ctypes.POINTER(RewriteDesc), ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p], ctypes.c_int),
    "pcnn_program_create": ([ctypes.POINTER(ScaleOp), ctypes.c_int, ctypes.POINTER(RewriteDesc), ctypes.c_int, c_i64,
                             ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "pcnn_program_run": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
                         ctypes.c_int),
    "pcnn_program_destroy": ([ctypes.c_void_p], ctypes.c_int),
    "pcnn_packer_create": ([ctypes.POINTER(PackDesc), ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "pcnn_packer_run": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "pcnn_packer_destroy": ([ctypes.c_void_p], ctypes.c_int),
}


class DeviceProgram:
    """A redistribution program resident on the device (pcnn_program_*): its
    op and rewrite tables uploaded once, every run launches only."""

    def __init__(self, ops, n_ops: int, rws, n_rws: int, arena_len: int):
        h = ctypes.c_void_p()
        check(lib().pcnn_program_create(ops, n_ops, rws, n_rws, arena_len, ctypes.byref(h)), "pcnn_program_create")
        self.handle = h

    def run(self, master_ptr: int, status_ptr: int, flags_ptr: int, stream) -> None:
        check(lib().pcnn_program_run(self.handle, ctypes.c_void_p(master_ptr), ctypes.c_void_p(status_ptr),
                                     ctypes.c_void_p(flags_ptr), stream), "pcnn_program_run")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None:
            _lib.pcnn_program_destroy(h)
            self.handle = None


class DevicePacker:
    """The float64 master -> compute images step with its pack tables on the
    device (pcnn_packer_*)."""

    def __init__(self, packs, n: int):
        h = ctypes.c_void_p()
        check(lib().pcnn_packer_create(packs, n, ctypes.byref(h)), "pcnn_packer_create")
        self.handle = h

    def run(self, master_ptr: int, packed_ptr: int, stream) -> None:
        check(lib().pcnn_packer_run(self.handle, ctypes.c_void_p(master_ptr), ctypes.c_void_p(packed_ptr), stream),
              "pcnn_packer_run")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None:
            _lib.pcnn_packer_destroy(h)
            self.handle = None


def lib() -> ctypes.CDLL:
    """Load libpcnn.so (once); raise PcnnError if it was not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise PcnnError(f"{LIB_PATH} not built; run `make` or __graft_entry__.build()")
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (args, res) in SYMBOLS.items():
            fn = getattr(handle, name)
            fn.argtypes = args
            fn.restype = res
        if handle.pcnn_abi_version() != ABI_VERSION:
            raise PcnnError("libpcnn ABI version mismatch")
        _lib = handle
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc != PCNN_OK:
        msg = lib().pcnn_last_error().decode(errors="replace")
        raise PcnnError(f"{what or 'libpcnn'} failed ({rc}): {msg}")


def require_device() -> None:
    """Fail loudly unless the library is built and a B200-class GPU is visible."""
    if not lib().pcnn_device_ok():
        raise PcnnError("no compute-capability 10.x (B200) device visible; the B200 path has no CPU fallback")


def array(ctype, items):
    arr = (ctype * max(len(items), 1))()
    for i, it in enumerate(items):
        arr[i] = it
    return arr
