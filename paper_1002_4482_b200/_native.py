"""ctypes binding of libsg.so (include/sg.h).

The library is built in-tree by ``paper_1002_4482_b200.build`` (or
``__graft_entry__.build()``).  If it is missing, every compute entry point
raises -- there is no CPU fallback.
"""

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsg.so")

# status codes (sg.h)
SG_OK = 0
SG_ERR_INVALID_LIST = 1
SG_ERR_INVALID_GRAPH = 2
SG_ERR_CAPABILITY = 3
SG_ERR_VALUE = 4
SG_ERR_RUNTIME = 5
SG_ERR_CUDA = 6
SG_ERR_WORKSPACE = 7

SG_U32, SG_I32, SG_I64 = 0, 1, 2
SG_WY_MULTI_KERNEL, SG_WY_SINGLE_BLOCK = 0, 1
SG_CC_UF, SG_CC_SV = 0, 1

SG_MAX_LAUNCHES = 192
SG_MAX_ROUNDS = 96
SG_MAX_LEVELS = 8

# every symbol include/sg.h declares (tests check the export table)
EXPORTS = (
    "sg_strerror", "sg_kernel_name", "sg_version", "sg_tuning_reload", "sg_source_hash", "sg_last_cuda_error", "sg_stats_resolve",
    "sg_wyllie_workspace_bytes", "sg_rs_workspace_bytes", "sg_wyllie_rank", "sg_rs_rank",
    "sg_gather_i64", "sg_even_splitters", "sg_cc_multi_workspace_bytes", "sg_cc_multi", "sg_nccl_comms_init",
    "sg_nccl_comms_destroy", "sg_cc_workspace_bytes", "sg_cc", "sg_cc_init", "sg_cc_hook",
    "sg_cc_hook_workspace_bytes", "sg_cc_hook_part", "sg_splitter_meta_workspace_bytes", "sg_splitter_meta",
    "sg_rs_rank_meta", "sg_cc_changes", "sg_cc_apply_min",
    "sg_cc_compress", "sg_cc_labels", "sg_kiss_batch_host", "sg_kiss_device",
    "sg_list_from_order", "sg_edge_keys", "sg_edges_from_keys", "sg_list_violation_host",
    "sg_h2d_narrow_i64", "sg_d2h_widen_u32", "sg_xfer_threads",
)


class Launch(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int32), ("round", ctypes.c_int32), ("blocks", ctypes.c_uint32),
                ("threads", ctypes.c_uint32), ("items", ctypes.c_uint64), ("ms", ctypes.c_float),
                ("pad", ctypes.c_uint32)]


class Stats(ctypes.Structure):
    _fields_ = [("n_launches", ctypes.c_uint32), ("rounds", ctypes.c_uint32), ("levels", ctypes.c_uint32),
                ("fallback", ctypes.c_uint32), ("edge_sweeps", ctypes.c_uint64),
                ("vertex_sweeps", ctypes.c_uint64), ("level_size", ctypes.c_uint64 * SG_MAX_LEVELS),
                ("n_roots", ctypes.c_uint32), ("list_path", ctypes.c_uint32),
                ("roots_per_round", ctypes.c_uint64 * SG_MAX_ROUNDS), ("total_ms", ctypes.c_float),
                ("pad2", ctypes.c_uint32), ("launch", Launch * SG_MAX_LAUNCHES)]


class Violation(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("pad", ctypes.c_int32), ("index", ctypes.c_int64)]


_lib = None

_P = ctypes.c_void_p
_U64 = ctypes.c_uint64
_I = ctypes.c_int
_SZ = ctypes.c_size_t

_SIGS = {
    "sg_strerror": (ctypes.c_char_p, [_I]),
    "sg_kernel_name": (ctypes.c_char_p, [_I]),
    "sg_version": (_I, []),
    "sg_tuning_reload": (_I, []),
    "sg_h2d_narrow_i64": (_I, [ctypes.c_void_p, _U64, ctypes.c_void_p, _U64, ctypes.c_void_p,
                               ctypes.POINTER(ctypes.c_int)]),
    "sg_d2h_widen_u32": (_I, [ctypes.c_void_p, _U64, ctypes.c_void_p, ctypes.c_void_p]),
    "sg_xfer_threads": (_I, []),
    "sg_source_hash": (ctypes.c_char_p, []),
    "sg_last_cuda_error": (ctypes.c_char_p, []),
    "sg_stats_resolve": (_I, [ctypes.POINTER(Stats)]),
    "sg_wyllie_workspace_bytes": (_SZ, [_U64]),
    "sg_rs_workspace_bytes": (_SZ, [_U64]),
    "sg_wyllie_rank": (_I, [_P, _I, _P, _I, _U64, _I, _P, _SZ, _P, ctypes.POINTER(Stats),
                            ctypes.POINTER(Violation)]),
    "sg_rs_rank": (_I, [_P, _I, _P, _I, _U64, _U64, _P, _SZ, _P, ctypes.POINTER(Stats),
                        ctypes.POINTER(Violation)]),
    "sg_gather_i64": (_I, [_P, _P, _U64, _P, _P]),
    "sg_even_splitters": (_I, [_P, _I, _U64, _U64, _P, _P]),
    "sg_cc_multi_workspace_bytes": (_SZ, [_U64, _U64, _I]),
    "sg_cc_multi": (_I, [_I, _P, _P, _I, _P, _U64, _P, _I, _I, _I, _P, _P, _P, _P, _P, _P]),
    "sg_nccl_comms_init": (_I, [_I, _P, _P]),
    "sg_nccl_comms_destroy": (_I, [_I, _P]),
    "sg_splitter_meta_workspace_bytes": (_SZ, [ctypes.c_uint32]),
    "sg_splitter_meta": (_I, [_P, _I, _U64, _P, ctypes.c_uint32, _P, _P, _SZ, _P]),
    "sg_rs_rank_meta": (_I, [_P, _I, _P, _I, _U64, _U64, _P, _SZ, _P, ctypes.c_uint32, _P, _P, _P, _SZ, _P,
                             ctypes.POINTER(Stats), ctypes.POINTER(Violation)]),
    "sg_cc_workspace_bytes": (_SZ, [_U64, _U64]),
    "sg_cc": (_I, [_P, _I, _U64, _U64, _P, _I, _I, _I, _P, _SZ, _P, ctypes.POINTER(Stats),
                   ctypes.POINTER(Violation)]),
    "sg_cc_init": (_I, [_P, _U64, _P]),
    "sg_cc_hook": (_I, [_P, _I, _U64, _U64, _U64, _P, _I, _I, _P, _P]),
    "sg_cc_hook_workspace_bytes": (_SZ, [_U64, _U64]),
    "sg_cc_hook_part": (_I, [_P, _I, _U64, _U64, _U64, _P, _I, _I, _P, _P, _SZ, _I, _P]),
    "sg_cc_compress": (_I, [_P, _U64, _U64, _P, _P]),
    "sg_cc_changes": (_I, [_P, _P, _U64, _P, _P, _U64, _P, _P]),
    "sg_cc_apply_min": (_I, [_P, _P, _P, _U64, _P]),
    "sg_cc_labels": (_I, [_P, _U64, _P, _I, _P]),
    "sg_kiss_batch_host": (_I, [ctypes.POINTER(ctypes.c_uint64), _U64, _P]),
    "sg_kiss_device": (_I, [_P, _U64, _U64, _U64, _P, _P]),
    "sg_list_from_order": (_I, [_P, _U64, _P, _I, _P]),
    "sg_edge_keys": (_I, [_P, _U64, _U64, _P, _P]),
    "sg_edges_from_keys": (_I, [_P, _U64, _U64, _P, _P]),
    "sg_list_violation_host": (_I, [_P, _U64, ctypes.POINTER(Violation)]),
}


class NativeMissing(RuntimeError):
    pass


def lib():
    """Load libsg.so once; raise loudly if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeMissing(
                f"{LIB_PATH} is missing: build it with `python -m paper_1002_4482_b200.build` "
                "(or __graft_entry__.build()); the GPU path has no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def strerror(code):
    return lib().sg_strerror(code).decode()


def kernel_name(kid):
    return lib().sg_kernel_name(kid).decode()


def last_cuda_error():
    return lib().sg_last_cuda_error().decode()


def check(code, what):
    """Raise for library-level failures (not input errors, which callers map)."""
    if code == SG_OK:
        return
    if code == SG_ERR_CUDA:
        raise RuntimeError(f"{what}: CUDA error: {last_cuda_error()}")
    raise RuntimeError(f"{what}: {strerror(code)} ({code})")


# ---------------------------------------------------------------------------
# host helpers

def kiss_batch_host(state, n):
    """(uint64 draws, new state) -- KISS64 on the host (gen.py:51-64)."""
    st = (ctypes.c_uint64 * 4)(*[int(v) & 0xFFFFFFFFFFFFFFFF for v in state])
    out = np.empty(int(n), dtype=np.uint64)
    if n:
        lib().sg_kiss_batch_host(st, int(n), out.ctypes.data)
    return out, tuple(int(v) for v in st)


def list_violation_host(succ):
    succ = np.ascontiguousarray(succ, dtype=np.int64)
    v = Violation()
    lib().sg_list_violation_host(succ.ctypes.data, succ.shape[0], ctypes.byref(v))
    return v.kind, v.index
