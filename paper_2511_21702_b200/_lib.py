"""ctypes binding of the C ABI in include/csvd_b200.h.

The shared library is built in-tree (`paper_2511_21702_b200/_build/
libcsvd_b200.so`, see build.py).  There is no fallback: if the library is
missing or fails to load, every entry point raises -- the product path never
silently runs on the CPU.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CSVD_LIB", os.path.join(_HERE, "_build", "libcsvd_b200.so"))

CSVD_MAX_LEVELS = 8

# mirrors of include/csvd_b200.h constants
E_CONFIG, E_DIM, E_VALUE, E_CUDA, E_STATE, E_NOMEM = -1, -2, -3, -4, -5, -6
W_F32, W_BF16 = 0, 1
MODE_CODES = {"euclidean": 0, "spherical": 1, "bias_augmented": 2}
KIND_NAMES = {0: "topk_exact", 1: "softmax_eps", 2: "topp_mass"}
TARGET_CODES = {"topk": 0, "softmax_eps": 1, "topp": 2}
FB_CODES = {"partial_expand": 0, "relax_eps": 1, "full_vocab": 2}
FB_NAMES = {-1: None, 0: "partial_expand", 1: "relax_eps", 2: "full_vocab"}
VARIANT_INCREMENTAL, VARIANT_BATCHSELECT = 0, 1


class TableDesc(ctypes.Structure):
    _fields_ = [
        ("vocab_size", ctypes.c_int64),
        ("hidden_dim", ctypes.c_int64),
        ("w_dtype", ctypes.c_int32),
        ("weights", ctypes.c_void_p),
        ("bias", ctypes.c_void_p),
    ]


class IndexDesc(ctypes.Structure):
    _fields_ = [
        ("n_clusters", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("perm", ctypes.c_void_p),
        ("starts", ctypes.c_void_p),
        ("sizes", ctypes.c_void_p),
        ("centroids", ctypes.c_void_p),
        ("radii", ctypes.c_void_p),
        ("max_biases", ctypes.c_void_p),
        ("log_sizes", ctypes.c_void_p),
        ("centroid_norms", ctypes.c_void_p),
        ("angulars", ctypes.c_void_p),
        ("max_norms", ctypes.c_void_p),
        ("min_norms", ctypes.c_void_p),
    ]


class Config(ctypes.Structure):
    _fields_ = [
        ("k", ctypes.c_int32),
        ("n_targets", ctypes.c_int32),
        ("targets", ctypes.c_int32 * 3),
        ("n_levels", ctypes.c_int32),
        ("level_kind", ctypes.c_int32 * CSVD_MAX_LEVELS),
        ("level_param", ctypes.c_double * CSVD_MAX_LEVELS),
        ("epsilon", ctypes.c_double),
        ("k_max", ctypes.c_int64),
        ("variant", ctypes.c_int32),
        ("slack_f32", ctypes.c_int32),
        ("first_wave_tokens", ctypes.c_int64),
        ("shard_lo", ctypes.c_int32),
        ("shard_hi", ctypes.c_int32),
    ]


class Result(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("fallback", ctypes.c_int32),
        ("sub_size", ctypes.c_int64),
        ("clusters_opened", ctypes.c_int32),
        ("heap_pops", ctypes.c_int32),
        ("epsilon_achieved", ctypes.c_double),
        ("u_max", ctypes.c_double),
        ("topk_min", ctypes.c_double),
        ("rho", ctypes.c_double),
        ("xi", ctypes.c_double),
        ("query_norm", ctypes.c_double),
        ("slack", ctypes.c_double),
        ("error", ctypes.c_int32),
        ("waves", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


FLAG_TIE_AMBIGUOUS = 1

# every symbol include/csvd_b200.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "csvd_create", "csvd_destroy", "csvd_strerror", "csvd_reserve_k", "csvd_step_host",
    "csvd_step_device", "csvd_outputs", "csvd_bounds_host", "csvd_dense_host",
    "csvd_dense_device", "csvd_info", "csvd_last_launches", "csvd_stream", "csvd_set_direct",
    "csvd_l2_flush", "csvd_create_shard", "csvd_shard_open", "csvd_shard_dense",
    "csvd_step_batch_host", "csvd_step_batch_device", "csvd_batch_lanes",
)

_lib = None
_load_error = None


class ExtensionMissing(RuntimeError):
    pass


def load():
    """Load the extension or raise (no CPU fallback exists)."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ExtensionMissing(
            f"CUDA extension not built: {LIB_PATH} missing (run __graft_entry__.build())")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as e:  # pragma: no cover
        _load_error = e
        raise ExtensionMissing(f"cannot load {LIB_PATH}: {e}") from e
    P = ctypes.c_void_p
    vp = ctypes.POINTER(ctypes.c_void_p)
    lib.csvd_create.argtypes = [vp, ctypes.c_int, ctypes.POINTER(TableDesc), ctypes.POINTER(IndexDesc)]
    lib.csvd_create_shard.argtypes = [vp, ctypes.c_int, ctypes.POINTER(TableDesc), ctypes.POINTER(IndexDesc), P]
    lib.csvd_shard_open.argtypes = [P, P, ctypes.POINTER(Config), P, P, P, P, ctypes.c_int64, P]
    lib.csvd_shard_dense.argtypes = [P, P, ctypes.c_int32, P, P, P, ctypes.c_int64, P]
    lib.csvd_step_batch_host.argtypes = [P, ctypes.c_int32, P, ctypes.POINTER(Config), P, P, P, ctypes.c_int64]
    lib.csvd_step_batch_device.argtypes = [P, ctypes.c_int32, P, ctypes.POINTER(Config), P]
    lib.csvd_batch_lanes.argtypes = [P, P, P]
    lib.csvd_destroy.argtypes = [P]
    lib.csvd_strerror.argtypes = [P]
    lib.csvd_strerror.restype = ctypes.c_char_p
    lib.csvd_reserve_k.argtypes = [P, ctypes.c_int32]
    lib.csvd_step_host.argtypes = [P, P, ctypes.POINTER(Config), ctypes.POINTER(Result), P, P,
                                   ctypes.c_int64]
    lib.csvd_step_device.argtypes = [P, P, ctypes.POINTER(Config), P]
    lib.csvd_outputs.argtypes = [P, vp, vp, vp]
    lib.csvd_bounds_host.argtypes = [P, P, ctypes.c_int32, P, P, P]
    lib.csvd_dense_host.argtypes = [P, P, P]
    lib.csvd_dense_device.argtypes = [P, P, P]
    lib.csvd_info.argtypes = [P, P, P, P, P, P, P, P]
    lib.csvd_last_launches.argtypes = [P, P]
    lib.csvd_stream.argtypes = [P, vp]
    lib.csvd_set_direct.argtypes = [P, ctypes.c_int32]
    lib.csvd_l2_flush.argtypes = [P, P]
    lib.csvd_test_sizes.argtypes = [P, P, P, P]
    lib.csvd_debug_timestamps.argtypes = [P, P]
    lib.csvd_test_scan_host.argtypes = [
        ctypes.POINTER(Config), ctypes.c_int, ctypes.c_longlong, ctypes.c_int, P, P, P, P, P, P, P,
        ctypes.c_int, P, ctypes.c_int, ctypes.POINTER(Result), P, P]
    for name in EXPORTS:
        getattr(lib, name).restype = getattr(lib, name).restype or ctypes.c_int
    lib.csvd_strerror.restype = ctypes.c_char_p
    _lib = lib
    return lib
