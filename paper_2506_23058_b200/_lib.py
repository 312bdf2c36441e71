"""ctypes binding of libixgpu.so (the C ABI declared in include/ixgpu.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no fallback: if the
library or a B200 device is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IXGPU_LIB") or os.path.join(_HERE, "libixgpu.so")  # IXGPU_LIB: dev A/B builds

# status / return codes (include/ixgpu.h)
OK, OOB, CONFLICT, LENGTH, BADARG, NOMEM, OVERFLOW, NODEVICE = 0, 1, 2, 3, 4, 5, 6, 7
OVF_SITE = 254  # status site of an int64 overflow (IXG_OVF_SITE)
CUDA_ERR = 100
I32, I64, U8, F64 = 0, 1, 2, 3
V_BOUNDS, V_CONFLICT, V_INIT = 1, 2, 4
VARIANT_CHECKED = 0x77777777
VARIANT_ELIDED = 0
F_DUP, F_NARROW = 1, 2
HIST_MIN, HIST_MAX, HIST_ADD = 0, 1, 2
(OP_SCAN, OP_SEGSCAN, OP_SCATTER, OP_FILTER, OP_PARTITION2, OP_PARTITION3, OP_C2, OP_MKSGMDESCR, OP_MKFLAGS, OP_HIST,
 OP_SCATTER_BINNED) = range(1, 12)
SCATTER_DIRECT, SCATTER_BINNED = 0, 1


class ixg_pred(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("pad", ctypes.c_int32), ("thr", ctypes.c_int64), ("seed", ctypes.c_uint64)]


class ixg_vm_insn(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("dst", ctypes.c_int32), ("a", ctypes.c_int32), ("b", ctypes.c_int32),
                ("c", ctypes.c_int32), ("pad", ctypes.c_int32), ("imm", ctypes.c_int64)]


class ixg_array(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("len", ctypes.c_int64), ("dt", ctypes.c_int32), ("pad", ctypes.c_int32)]


VM_MAX_INSN, VM_MAX_IN, VM_MAX_OUT, VM_MAX_PRED, VM_REGS = 96, 8, 4, 4, 24
(VM_HALT, VM_IN, VM_CONST, VM_ADD, VM_SUB, VM_MUL, VM_EQ, VM_NE, VM_LT, VM_LE, VM_GT, VM_GE, VM_NOT, VM_MOV, VM_JZ,
 VM_JMP, VM_IDX, VM_PRED, VM_OUT, VM_LEN) = range(20)


class ixg_status(ctypes.Structure):
    _fields_ = [("first", ctypes.c_uint64), ("codes", ctypes.c_uint32), ("flags", ctypes.c_uint32)]


_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_U32 = ctypes.c_uint32
_U64 = ctypes.c_uint64
_SZ = ctypes.c_size_t
_PP = ctypes.POINTER(ixg_pred)

# name -> (restype, argtypes); every symbol include/ixgpu.h declares
SIGNATURES = {
    "ixg_version": (_I, []),
    "ixg_device_check": (_I, []),
    "ixg_ws_bytes": (_SZ, [_I, _I64, _I64]),
    "ixg_ws_init": (_I, [_P, _SZ, _P]),
    "ixg_status_init": (_I, [_P, _P]),
    "ixg_launch_count": (ctypes.c_ulonglong, []),
    "ixg_scan_add": (_I, [_I, _P, _I64, _I64, _I, _P, _P, _SZ, _P, _P]),
    "ixg_reduce_add": (_I, [_I, _P, _I64, _P, _P]),
    "ixg_jagged_dest": (_I, [_P, _I64, _P, _P, _P, _P]),
    "ixg_partition_counts": (_I, [_I, _P, _I64, _P, _P, _I, _P, _P, _SZ, _P]),
    "ixg_partition2_peer": (_I, [_I, _P, _I64, _P, _P, _I, _I64, _P, _I, _P, _SZ, _P]),
    "ixg_rank_offsets": (_I, [_P, _I, _I, _I, _P, _P]),
    "ixg_dev_alloc": (_I, [_SZ, _P]),
    "ixg_dev_free": (_I, [_P]),
    "ixg_ipc_handle": (_I, [_P, _P]),
    "ixg_ipc_open": (_I, [_P, _P]),
    "ixg_ipc_close": (_I, [_P]),
    "ixg_segscan_add": (_I, [_I, _P, _I, _P, _I64, _I, _I64, _P, _P, _P, _SZ, _P, _P]),
    "ixg_scatter": (_I, [_I, _P, _I64, _P, _I64, _P, _I64, _U32, _I, _I, _I, _P, _P, _SZ, _P]),
    "ixg_scatter_probe": (_I, [_P, _I64, _P, _P]),
    "ixg_gather": (_I, [_I, _P, _I64, _P, _I64, _P, _U32, _I, _I, _P, _P]),
    "ixg_hist": (_I, [_I, _I64, _I64, _P, _I64, _P, _I64, _P, _P, _SZ, _P, _P]),
    "ixg_fill": (_I, [_I, _P, _I64, _I64, _P]),
    "ixg_iota": (_I, [_P, _I64, _P]),
    "ixg_filter": (_I, [_I, _P, _I64, _PP, _P, _P, _U32, _P, _P, _SZ, _P]),
    "ixg_filter_by": (_I, [_I, _P, _P, _I64, _P, _P, _U32, _P, _P, _SZ, _P]),
    "ixg_partition2": (_I, [_I, _P, _I64, _PP, _P, _P, _U32, _P, _P, _SZ, _P]),
    "ixg_partition3": (_I, [_I, _P, _I64, _PP, _PP, _P, _P, _U32, _P, _P, _SZ, _P]),
    "ixg_c2": (_I, [_I, _P, _I64, _PP, _P, _I64, _P, _I, _P, _P, _U32, _P, _P, _SZ, _P]),
    "ixg_mksgmdescr": (_I, [_P, _P, _I64, _I64, _P, _I64, _P, _U32, _P, _P, _SZ, _P]),
    "ixg_csr_gather": (_I, [_I, _P, _I64, _P, _P, _I64, _P, _U32, _P, _P]),
    "ixg_kmeans_ker": (_I, [_P, _I64, _P, _I64, _P, _I64, _P, _P, _I64, _P, _U32, _P, _P]),
    "ixg_eq_gather": (_I, [_P, _I64, _P, _P, _I64, _P, _U32, _I, _P, _P]),
    "ixg_gen_uniform": (_I, [_I, _P, _I64, _I64, _I64, _U64, _I64, _P]),
    "ixg_minmax": (_I, [_I, _P, _I64, _P, _P]),
    "ixg_mono_check": (_I, [_I, _P, _I64, _I, _P, _P]),
    "ixg_inj_bitmap_bytes": (_I64, [_I64, _I64]),
    "ixg_inj_check": (_I, [_P, _I64, _I64, _I64, _I64, _I64, _P, _I64, _P, _P]),
    "ixg_mkflags": (_I, [_I64, _P, _I64, _P, _U32, _P, _P, _SZ, _P]),
    "ixg_map": (_I, [_P, _I, _P, _I, _P, _I, _P, _I, _I64, _I, _P, _P]),
    "ixg_bitmap_words": (_I64, [_I64]),
    "ixg_flag_bitmap": (_I, [_P, _I64, _P, _I64, _P, _P, _SZ, _P]),
    "ixg_flag_bitmap_window": (_I, [_P, _I64, _P, _I64, _P, _P, _P, _SZ, _P]),
    "ixg_segsum": (_I, [_I, _P, _I64, _P, _P, _I64, _P, _I, _P, _I64, _I, _P, _P, _P, _SZ, _P]),
    "ixg_seg_carry": (_I, [_P, _I64, _P, _I, _P, _I64, _P, _I64, _P, _I, _P, _P, _P]),
    "ixg_timer_start": (_I, [_I]),
    "ixg_trace_read": (_I, [_P, _SZ]),
    "ixg_timer_stop": (_I, [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]),
}
K_FILTER_FUSED, K_PLACE, K_CLASS_COUNT, K_SCAN, K_SCATTER, K_CSR_GATHER, K_SEGSUM, K_BIN = 1, 2, 3, 4, 5, 6, 7, 8

_lib = None
_lock = threading.Lock()


class NativeUnavailable(RuntimeError):
    """libixgpu.so is missing or no sm_100 device is visible (no fallback)."""


def load(require_device: bool = False):
    """Load libixgpu.so (raises NativeUnavailable when absent)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeUnavailable(
                    f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    if require_device and not _device_ok:
        rc = _lib.ixg_device_check()
        if rc != OK:
            raise NativeUnavailable("libixgpu.so needs an sm_100 (B200) CUDA device; none is current")
        _set_device_ok()
    return _lib


_device_ok = False  # an sm_100 device was found once (every op call used to re-query it)


def _set_device_ok():
    global _device_ok
    _device_ok = True


def check(rc: int, what: str) -> None:
    if rc == OK:
        return
    if rc >= CUDA_ERR:
        raise RuntimeError(f"{what}: CUDA error {rc - CUDA_ERR}")
    names = {BADARG: "bad argument", NOMEM: "out of memory", NODEVICE: "no sm_100 device"}
    raise RuntimeError(f"{what}: {names.get(rc, rc)}")
