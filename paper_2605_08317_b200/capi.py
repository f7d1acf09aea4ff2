"""ctypes bindings of the C-ABI in include/rdkv_cuda.h.

The native library is built in-tree (paper_2605_08317_b200/_lib/librdkv_b200.so)
by __graft_entry__.build(). There is no fallback: if the library is missing,
importing the device API raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "librdkv_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "rdkv_cuda.h")

RDKV_OK, RDKV_EINVAL, RDKV_ENUMERIC, RDKV_EFORMAT, RDKV_ECUDA = range(5)
RDKV_F32, RDKV_F16 = 0, 1
RDKV_DECODE_OUT_HOST, RDKV_DECODE_ZC_BOUND = 1, 2


class RdkvError(RuntimeError):
    """Raised for a non-zero rdkv_status; `.code` is the status."""

    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: {STATUS_NAMES.get(code, code)}")
        self.code = code


class InvalidArgument(RdkvError, ValueError):
    pass


class NumericError(RdkvError, ArithmeticError):
    pass


class FormatError(RdkvError):
    """rdkv::FormatError (errors.hpp:9-11): malformed containers."""


STATUS_NAMES = {0: "ok", 1: "invalid argument", 2: "numeric error", 3: "format error", 4: "CUDA error"}


def raise_for(code: int, what: str) -> None:
    if code == RDKV_OK:
        return
    if code == RDKV_EINVAL:
        raise InvalidArgument(code, what)
    if code == RDKV_ENUMERIC:
        raise NumericError(code, what)
    if code == RDKV_EFORMAT:
        raise FormatError(code, what)
    raise RdkvError(code, what)


class Shape(C.Structure):
    _fields_ = [("units", C.c_int32), ("seq_len", C.c_int32), ("head_dim", C.c_int32),
                ("group", C.c_int32), ("probe_rows", C.c_int32), ("kv_heads", C.c_int32)]


class Config(C.Structure):
    """rdkv_config: BudgetSpec + ProbeConfig + SolverConfig + PipelineConfig."""

    _fields_ = [
        ("n_tokens", C.c_int32), ("n_widths", C.c_int32), ("r_k", C.c_double),
        ("widths", C.c_int32 * 8), ("eps_v", C.c_double * 8), ("eps_k", C.c_double * 8),
        ("window", C.c_int32), ("pool_kernel", C.c_int32), ("tolerance", C.c_double),
        ("max_iterations", C.c_int32), ("strict_budget", C.c_int32),
        ("force_window_retain", C.c_int32), ("reserved", C.c_int32),
    ]


class HeadStats(C.Structure):
    _fields_ = [
        ("lambda_v", C.c_double), ("lambda_k", C.c_double), ("objective_v", C.c_double),
        ("objective_k", C.c_double), ("achieved_bits", C.c_double), ("avg_v", C.c_double),
        ("avg_k", C.c_double), ("v_converged", C.c_int32), ("k_converged", C.c_int32),
        ("n_kept", C.c_int32), ("n_v16", C.c_int32), ("k_bits_len", C.c_int32),
        ("status", C.c_int32),
    ]


HEAD_STATS_BYTES = C.sizeof(HeadStats)


class DecodePlan(C.Structure):
    _fields_ = [("max_decode_bytes", C.c_int32), ("max_slots", C.c_int32),
                ("max_zone_b_rows", C.c_int32), ("max_kq_slots", C.c_int32), ("uniform2", C.c_int32),
                ("n_uniform", C.c_int32), ("uniform2_split", C.c_int32), ("mix24", C.c_int32),
                ("min_chunks24", C.c_int32), ("max_krow_bytes24", C.c_int32)]


class DecodeArgs(C.Structure):
    _fields_ = [
        ("arena", C.c_void_p), ("tile_offsets", C.c_void_p), ("units", C.c_int32),
        ("group", C.c_int32), ("head_dim", C.c_int32), ("io_dtype", C.c_int32),
        ("q", C.c_void_p), ("out", C.c_void_p), ("zc_k", C.c_void_p), ("zc_v", C.c_void_p),
        ("zc_len", C.c_void_p), ("zc_cap", C.c_int32), ("split", C.c_int32),
        ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t), ("kernel", C.c_int32),
        ("flags", C.c_int32), ("tile_decode_bytes", C.c_void_p), ("plan", DecodePlan),
        ("zc_bound", C.c_int32), ("reserved2", C.c_int32), ("unit_ids", C.c_void_p),
    ]


class TileInfo(C.Structure):
    _fields_ = [("n_kept", C.c_int32), ("rows", C.c_int32 * 4), ("chans", C.c_int32 * 4),
                ("kslots", C.c_int32), ("krow_bytes", C.c_int32), ("nslot", C.c_int32),
                ("total_bytes", C.c_int64), ("decode_bytes", C.c_int64)]


class BisectResult(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("achieved_avg_bits", C.c_double), ("objective", C.c_double),
                ("converged", C.c_int32), ("status", C.c_int32)]


class CacheHeader(C.Structure):
    _fields_ = [("layers", C.c_int32), ("q_heads", C.c_int32), ("kv_heads", C.c_int32),
                ("head_dim", C.c_int32), ("seq_len", C.c_int32), ("probe_window", C.c_int32),
                ("payload_offset", C.c_int64), ("payload_bytes", C.c_int64)]


class DualBoundResult(C.Structure):
    _fields_ = [("g_lambda", C.c_double), ("primal", C.c_double), ("gap", C.c_double),
                ("feasible", C.c_int32), ("status", C.c_int32)]


_VP = C.c_void_p
_SIGS = {
    "rdkv_cuda_dual_bound": (C.c_int, [_VP, C.c_int32, C.c_int32, _VP, _VP, C.c_int32, _VP, C.c_double, _VP, _VP]),
    "rdkv_cuda_calibrate_workspace": (C.c_size_t, [C.c_int32] * 5),
    "rdkv_cuda_calibrate_partials": (C.c_int, [_VP, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                               _VP, C.c_int32, _VP, _VP, _VP, C.c_size_t, _VP]),
    "rdkv_calibrate_finalize": (C.c_int, [_VP, _VP, C.c_int32, _VP, C.c_int32, _VP, _VP]),
    "rdkv_cache_read_header": (C.c_int, [C.c_char_p, C.POINTER(CacheHeader)]),
    "rdkv_cuda_cache_load": (C.c_int, [C.c_char_p, C.POINTER(CacheHeader), _VP, _VP, _VP, C.c_int32, _VP]),
    "rdkv_cuda_weights_workspace": (C.c_size_t, [C.POINTER(Shape), C.c_int32]),
    "rdkv_cuda_weights": (C.c_int, [_VP, _VP, C.c_int32, C.POINTER(Shape), C.c_int32, C.c_int32,
                                    _VP, _VP, _VP, C.c_size_t, _VP]),
    "rdkv_cuda_allocate": (C.c_int, [_VP, _VP, C.POINTER(Shape), C.POINTER(Config), _VP, _VP,
                                     _VP, _VP]),
    "rdkv_cuda_pack_plan": (C.c_int, [_VP, _VP, C.POINTER(Shape), _VP, _VP]),
    "rdkv_cuda_pack": (C.c_int, [_VP, _VP, C.c_int32, _VP, _VP, C.POINTER(Shape), _VP, _VP, _VP,
                                 _VP]),
    "rdkv_cuda_decode_workspace": (C.c_size_t, [C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "rdkv_cuda_decode": (C.c_int, [C.POINTER(DecodeArgs), _VP]),
    "rdkv_cuda_decode_prepare": (C.c_int, [_VP, _VP, C.c_int32, _VP, C.POINTER(DecodePlan), _VP]),
    "rdkv_cuda_decode_prepare_split": (C.c_int, [_VP, _VP, C.c_int32, _VP, _VP, C.POINTER(DecodePlan), _VP]),
    "rdkv_cuda_decode_host": (C.c_int, [C.POINTER(DecodeArgs), _VP, _VP, _VP]),
    "rdkv_cuda_decode_partial": (C.c_int, [C.POINTER(DecodeArgs), C.c_int32, C.c_int32, _VP, _VP]),
    "rdkv_cuda_decode_merge": (C.c_int, [_VP, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _VP, C.c_int32, _VP]),
    "rdkv_cuda_decode_ctx_create": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p)]),
    "rdkv_cuda_decode_ctx_destroy": (C.c_int, [C.c_void_p]),
    "rdkv_cuda_decode_host_pipelined": (C.c_int, [C.c_void_p, C.POINTER(DecodeArgs), _VP, _VP, _VP]),
    "rdkv_cuda_append": (C.c_int, [_VP, _VP, _VP, C.c_int32, _VP, _VP, C.c_int32, C.c_int32,
                                   C.c_int32, _VP]),
    "rdkv_cuda_generate": (C.c_int, [_VP, C.c_int32, C.c_uint64, C.c_int32, C.c_uint64,
                                     C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_float,
                                     C.c_int32, C.c_float, _VP]),
    "rdkv_cuda_attention_probe_workspace": (C.c_size_t, [C.c_int32, C.c_int32]),
    "rdkv_cuda_attention_probe": (C.c_int, [_VP, C.c_int32, _VP, C.c_int32, C.c_int32, _VP, _VP, _VP,
                                            C.c_size_t, _VP]),
    "rdkv_cuda_token_weights": (C.c_int, [_VP, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _VP, _VP, _VP]),
    "rdkv_cuda_moving_average": (C.c_int, [_VP, C.c_int32, C.c_int32, _VP, _VP]),
    "rdkv_cuda_channel_weights": (C.c_int, [_VP, C.c_int32, _VP, C.c_int32, C.c_int32, _VP, _VP]),
    "rdkv_cuda_mckp_bisect": (C.c_int, [_VP, C.c_int32, C.c_int32, _VP, _VP, C.c_int32, C.c_double,
                                        C.c_double, C.c_int32, C.c_int32, _VP, _VP, _VP]),
    "rdkv_cuda_quantize_units": (C.c_int, [_VP, C.c_int32, C.c_int32, C.c_int32, _VP, _VP, _VP, _VP, _VP]),
    "rdkv_cuda_pack_bits": (C.c_int, [_VP, C.c_int64, C.c_int32, _VP, _VP, _VP]),
    "rdkv_cuda_unpack_bits": (C.c_int, [_VP, C.c_int64, C.c_int32, C.c_int64, _VP, _VP]),
    "rdkv_cuda_tile_logits": (C.c_int, [_VP, _VP, C.c_int32, C.c_int32, C.c_int32, _VP, C.c_int32,
                                        C.c_int32, _VP, _VP]),
    "rdkv_tile_import_bytes": (C.c_size_t, [C.c_int32, C.c_int32, _VP, _VP]),
    "rdkv_tile_import": (C.c_int, [C.c_int32, C.c_int32] + [_VP] * 12 + [C.c_size_t]),
    "rdkv_tile_info_get": (C.c_int, [_VP, C.POINTER(TileInfo)]),
    "rdkv_tile_export": (C.c_int, [_VP, C.c_int32] + [_VP] * 14),
    "rdkv_tile_export_payload_bytes": (C.c_size_t, [_VP, C.c_int32]),
    "rdkv_status_string": (C.c_char_p, [C.c_int]),
    "rdkv_version": (C.c_int, []),
}

_LIB = None


def declared_symbols() -> list[str]:
    """Every RDKV_API function declared in include/rdkv_cuda.h."""
    text = open(HEADER_PATH).read()
    return re.findall(r"RDKV_API\s+[\w\s\*]+?\b(rdkv_\w+)\s*\(", text)


def lib() -> C.CDLL:
    """Load the native library (raises if it was not built — no fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"native RDKV library missing at {LIB_PATH}; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def config_from(cfg) -> Config:
    """Copy any ctypes struct with the rdkv_config layout (e.g. oracle.Config)."""
    if isinstance(cfg, Config):
        return cfg
    out = Config()
    C.memmove(C.byref(out), C.byref(cfg), C.sizeof(Config))
    return out
