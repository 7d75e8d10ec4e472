"""ctypes declarations of include/kvtc.h (argument marshalling only).

Loads the in-tree ``libkvtc.so`` built by ``__graft_entry__.build()``.  There is
no fallback: if the library is missing or the device is not sm_100, calls fail
loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkvtc.so")

KVTC_OK, KVTC_NOTHING_TO_COMPRESS = 0, 1
STATUS_NAMES = {0: "OK", 1: "NOTHING_TO_COMPRESS", -1: "E_INVALID", -2: "E_NUMERIC", -3: "E_CORRUPT",
                -4: "E_MISMATCH", -5: "E_CAPACITY", -6: "E_CUDA", -8: "E_NOMEM", -9: "E_UNSUPPORTED"}
KEYS, VALUES = 0, 1
T_NONE, T_INT2, T_INT4, T_FP8 = 0, 1, 2, 3
LAYOUT_CONTIGUOUS, LAYOUT_PAGED = 0, 1
HEADER_BYTES = 256
CODER_DEFLATE, CODER_RANS = 0, 1


class KvtcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"kvtc {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Shape(C.Structure):
    _fields_ = [("layers", C.c_int32), ("kv_heads", C.c_int32), ("head_dim", C.c_int32)]


class Rope(C.Structure):
    _fields_ = [("inv_freq_host", C.POINTER(C.c_float)), ("pairing", C.c_int32)]


class View(C.Structure):
    _fields_ = [("shape", Shape), ("tokens", C.c_int64), ("pos0", C.c_int64), ("layout", C.c_int32),
                ("page_tokens", C.c_int32), ("layer_base_host", C.POINTER(C.c_void_p)),
                ("block_table", C.c_void_p), ("keys_rotated", C.c_int32), ("reserved", C.c_int32)]


class Policy(C.Structure):
    _fields_ = [("sinks", C.c_int32), ("window", C.c_int32), ("chunk_bytes", C.c_int32), ("coder", C.c_int32)]


class DPConfig(C.Structure):
    _fields_ = [("target_cr", C.c_double), ("feature_bits", C.c_int32), ("nsizes", C.c_int32),
                ("sizes_host", C.POINTER(C.c_int32)), ("type_mask", C.c_uint32), ("dp_row_cap", C.c_int64)]


class ContainerInfo(C.Structure):
    _fields_ = [("magic", C.c_uint32), ("version", C.c_uint32), ("layers", C.c_int32), ("kv_heads", C.c_int32),
                ("head_dim", C.c_int32), ("sinks", C.c_int32), ("window", C.c_int32), ("chunk_bytes", C.c_int32),
                ("tokens", C.c_int64), ("pos0", C.c_int64), ("m", C.c_int64), ("total_bytes", C.c_uint64),
                ("raw_bytes", C.c_uint64), ("payload_bytes", C.c_uint64 * 2), ("entropy_bytes", C.c_uint64 * 2),
                ("basis_fp", C.c_uint64 * 2), ("plan_fp", C.c_uint64 * 2), ("flags", C.c_uint32),
                ("reserved", C.c_uint32), ("payload_hash", C.c_uint64 * 2), ("raw_hash", C.c_uint64)]


vp, i32, i64, u64, sz, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_size_t, C.c_double
P = C.POINTER
_SIGS = {
    "kvtc_abi_version": (i32, []),
    "kvtc_last_error": (C.c_char_p, []),
    "kvtc_device_check": (i32, []),
    "kvtc_basis_create": (i32, [P(Shape), i32, P(Rope), i32, P(C.c_float), P(C.c_float), P(C.c_float), P(vp)]),
    "kvtc_basis_destroy": (i32, [vp]),
    "kvtc_basis_get": (i32, [vp, P(i32), P(i32), P(C.c_float), P(C.c_float), P(C.c_float)]),
    "kvtc_calibrate_workspace_bytes": (sz, [P(Shape)]),
    "kvtc_calibrate_accumulate": (i32, [P(View), i32, P(i64), i64, i32, P(Rope), vp, vp, vp, sz, vp]),
    "kvtc_calibrate_finalize": (i32, [P(Shape), i32, P(Rope), vp, vp, i64, i32, vp, P(vp)]),
    "kvtc_calibrate": (i32, [P(View), i32, P(i64), i64, i32, P(Rope), i32, vp, P(vp)]),
    "kvtc_allocate_bits_from_coeffs": (i32, [vp, i64, i32, i32, P(DPConfig), vp, P(vp)]),
    "kvtc_allocate_bits": (i32, [vp, P(View), i32, P(i64), i64, P(DPConfig), vp, P(vp)]),
    "kvtc_allocate_bits_multi": (i32, [vp, P(View), i32, P(i64), i64, P(DPConfig), P(f64), i32, vp, P(vp)]),
    "kvtc_allocate_bits_from_coeffs_multi": (i32, [vp, i64, i32, i32, P(DPConfig), P(f64), i32, vp, P(vp)]),
    "kvtc_dp_best_table": (i32, [vp, i64, i32, i64, P(DPConfig), vp, vp]),
    "kvtc_plan_create": (i32, [i32, i32, P(i32), P(i32), P(i32), P(vp)]),
    "kvtc_plan_destroy": (i32, [vp]),
    "kvtc_plan_get": (i32, [vp, P(i32), P(i32), P(i32), P(i32), P(i32), P(i64), P(i32), P(f64), P(i64)]),
    "kvtc_compress_bound": (sz, [vp, vp, P(View), P(Policy)]),
    "kvtc_compress_workspace_bytes": (sz, [vp, vp, vp, vp, P(View), P(Policy)]),
    "kvtc_compress": (i32, [vp, vp, vp, vp, P(View), P(View), P(Policy), vp, sz, P(sz), vp, sz, vp]),
    "kvtc_decompress_workspace_bytes": (sz, [vp, vp, vp, vp, vp]),
    "kvtc_decompress": (i32, [vp, vp, vp, vp, vp, sz, i32, i32, P(View), P(View), vp, sz, vp]),
    "kvtc_decompress_async": (i32, [vp, vp, vp, vp, vp, sz, C.c_char_p, i32, i32, P(View), P(View), vp, vp, sz,
                                    vp]),
    "kvtc_decompress_begin": (i32, [vp, vp, vp, vp, vp, sz, vp, sz, vp]),
    "kvtc_decompress_layers": (i32, [vp, vp, vp, vp, vp, C.c_char_p, i32, i32, P(View), P(View), vp, sz, vp]),
    "kvtc_compress_batch_workspace_bytes": (sz, [vp, vp, vp, vp, P(View), i32, P(Policy)]),
    "kvtc_compress_batch": (i32, [vp, vp, vp, vp, P(View), P(View), i32, P(Policy), P(vp), P(sz), P(sz), vp, sz,
                                  vp]),
    "kvtc_decompress_batch_workspace_bytes": (sz, [vp, vp, vp, vp, P(vp), i32]),
    "kvtc_decompress_batch": (i32, [vp, vp, vp, vp, P(vp), P(sz), i32, P(View), P(View), vp, sz, vp]),
    "kvtc_decompress_batch_async": (i32, [vp, vp, vp, vp, P(vp), P(sz), P(vp), i32, P(View), P(View), vp, vp, sz,
                                          vp]),
    "kvtc_container_parse": (i32, [vp, P(ContainerInfo)]),
    "kvtc_stage_gather": (i32, [P(View), i64, i64, i32, P(Rope), vp, vp]),
    "kvtc_stage_project": (i32, [vp, vp, vp, i64, vp, vp]),
    "kvtc_payload_bytes": (sz, [vp, i64]),
    "kvtc_stage_quantize_pack": (i32, [vp, vp, i64, vp, vp]),
    "kvtc_stage_project_quantize": (i32, [vp, vp, vp, i64, vp, vp]),
    "kvtc_deflate_bound": (sz, [sz, i32]),
    "kvtc_deflate_workspace_bytes": (sz, [sz, i32]),
    "kvtc_stage_deflate": (i32, [vp, sz, i32, vp, sz, P(sz), vp, sz, vp]),
    "kvtc_stage_inflate": (i32, [vp, sz, vp, sz, vp]),
    "kvtc_stage_inflate_raw": (i32, [vp, vp, vp, i32, vp, vp, vp, vp, vp]),
    "kvtc_stage_dequantize": (i32, [vp, vp, i64, vp, i64, vp]),
    "kvtc_stage_reconstruct": (i32, [vp, vp, vp, i64, i64, i64, i32, i32, P(View), vp]),
    "kvtc_stage_reconstruct_payload": (i32, [vp, vp, vp, i64, i64, i32, i32, P(View), vp]),
    "kvtc_stage_project_partial": (i32, [vp, vp, vp, i64, i32, i32, i32, vp, vp]),
    "kvtc_rans_bound": (C.c_size_t, [C.c_size_t, i32, i64]),
    "kvtc_rans_workspace_bytes": (C.c_size_t, [C.c_size_t, i32, i64]),
    "kvtc_stage_rans_encode": (i32, [vp, C.c_size_t, i32, i64, vp, C.c_size_t, P(C.c_size_t), vp, C.c_size_t, vp]),
    "kvtc_stage_rans_decode": (i32, [vp, C.c_size_t, vp, C.c_size_t, vp]),
    "kvtc_profile_enable": (None, [i32]),
    "kvtc_profile_read": (i32, [C.c_char_p, sz, P(f64), P(i32), i32]),
    "kvtc_launch_count": (i64, []),
    "kvtc_launch_count_reset": (None, []),
}

_lib = None


def lib():
    """The loaded library (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(status: int, allow=(KVTC_OK,)) -> int:
    if status not in allow:
        raise KvtcError(status, lib().kvtc_last_error().decode(errors="replace"))
    return status
