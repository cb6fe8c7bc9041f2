"""ctypes binding of the C-ABI in include/psp_gpu.h (libpsp_gpu.so, in-tree).

The library is the product: there is no Python or CPU fallback. Loading
fails loudly if the shared object is missing, and every compute call fails
with PSP_ECUDA when no CUDA device is usable.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpsp_gpu.so")

(PSP_OK, PSP_EINVAL, PSP_ENOMEM, PSP_ECUDA, PSP_ENCCL, PSP_EOVERFLOW, PSP_EGRAPH, PSP_EIO,
 PSP_EFORMAT, PSP_ECHECKSUM, PSP_EPARSE) = range(11)
FORMAT_EDGE_LIST, FORMAT_DIMACS = 0, 1
VALUE_AUTO, VALUE_U32, VALUE_F32 = 0, 1, 2
VALUE_NAMES = {VALUE_U32: "u32", VALUE_F32: "f32"}


class PspError(RuntimeError):
    """Non-invalid-argument failures (reference: std::runtime_error)."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class GraphInvariantError(PspError):
    """psp::GraphInvariantError (include/psp/errors.hpp:22-25)."""


class PspValueError(PspError, ValueError):
    """std::invalid_argument / PSP_EINVAL and PSP_EOVERFLOW."""


class OracleIoError(PspError, OSError):
    """psp::IoError (include/psp/errors.hpp:28-31): unreadable, truncated or
    inconsistent oracle file."""


class FormatVersionError(OracleIoError):
    """psp::FormatVersionError (include/psp/errors.hpp:34-37)."""


class ChecksumError(OracleIoError):
    """psp::ChecksumError (include/psp/errors.hpp:40-43)."""


class ParseError(PspError):
    """psp::ParseError (include/psp/errors.hpp:10-19): malformed graph text;
    the message is "<name>:<line>: <what>", `line` the 1-based line."""

    def __init__(self, status: int, msg: str, line: int):
        super().__init__(status, msg)
        self.line = line


class BuildStats(C.Structure):
    _fields_ = [
        ("partition_ms", C.c_double),
        ("component_apsp_ms", C.c_double),
        ("boundary_ms", C.c_double),
        ("boundary_total", C.c_uint64),
        ("bg_edges", C.c_uint64),
        ("stored_entries", C.c_uint64),
        ("peak_table_entries_per_worker", C.c_uint64),
        ("k1_device_ms", C.c_double),
        ("k2_device_ms", C.c_double),
        ("init_device_ms", C.c_double),
        ("k1_relaxations", C.c_uint64),
        ("k2_relaxations", C.c_uint64),
        ("value_kind", C.c_int32),
        ("fixed_point_shift", C.c_int32),
        ("device_bytes", C.c_uint64),
        ("k2_positions", C.c_uint64),
        ("k2_order", C.c_int32),
        ("k2_spilled", C.c_int32),
        ("split_ms", C.c_double),
        ("k1_order_ms", C.c_double),
        ("bg_order_ms", C.c_double),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class OracleInfo(C.Structure):
    _fields_ = [
        ("n", C.c_uint64),
        ("k", C.c_uint32),
        ("b", C.c_uint64),
        ("value_kind", C.c_int32),
        ("fixed_point_shift", C.c_int32),
        ("device", C.c_int32),
        ("tile", C.c_int32),
    ]


class RoutedStats(C.Structure):
    _fields_ = [
        ("queries", C.c_uint64),
        ("executed_here", C.c_uint64),
        ("sent_to_peers", C.c_uint64),
        ("transfer_queries", C.c_uint64),
        ("transfer_entries", C.c_uint64),
        ("transfer_bytes", C.c_uint64),
        ("route_ms", C.c_double),
        ("exec_ms", C.c_double),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


PLACE_ROUND_ROBIN, PLACE_PAIRS_PER_GPU = 0, 1

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_vp = C.c_void_p

# name -> (restype, argtypes); the exported surface of include/psp_gpu.h
SIGNATURES = {
    "psp_gpu_abi_version": (C.c_int, []),
    "psp_gpu_last_error": (C.c_char_p, []),
    "psp_gpu_device_count": (C.c_int, []),
    "psp_gpu_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, C.POINTER(_vp)]),
    "psp_gpu_ctx_destroy": (None, [_vp]),
    "psp_gpu_nccl_unique_id": (C.c_int, [_vp]),
    "psp_gpu_ctx_stream": (_vp, [_vp]),
    "psp_gpu_ctx_set_boundary_storage": (C.c_int, [_vp, C.c_int]),
    "psp_gpu_alloc_stats": (C.c_int, [_u64p]),
    "psp_gpu_build_oracle": (C.c_int, [_vp, C.c_uint64, C.c_uint64, _u32p, _u32p, _f64p,
                                       C.c_uint32, C.c_uint32, C.c_uint64, C.c_int,
                                       C.POINTER(_vp), C.POINTER(BuildStats)]),
    "psp_gpu_build_partitioned": (C.c_int, [_vp, C.c_uint64, C.c_uint64, _u32p, _u32p, _f64p,
                                            C.c_uint32, _u32p, C.c_int, C.POINTER(_vp),
                                            C.POINTER(BuildStats)]),
    "psp_gpu_oracle_import": (C.c_int, [_vp, C.c_uint64, C.c_uint32, _u32p, _u32p, _u64p, _u64p,
                                        _vp, _vp, C.c_int, C.POINTER(_vp)]),
    "psp_gpu_oracle_save": (C.c_int, [_vp, C.c_char_p]),
    "psp_gpu_oracle_load": (C.c_int, [_vp, C.c_char_p, C.c_int, C.POINTER(_vp)]),
    "psp_gpu_oracle_free": (None, [_vp]),
    "psp_gpu_oracle_info": (C.c_int, [_vp, C.POINTER(OracleInfo)]),
    "psp_gpu_oracle_ids": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "psp_gpu_export_component": (C.c_int, [_vp, C.c_uint32, _f64p]),
    "psp_gpu_export_boundary_rows": (C.c_int, [_vp, C.c_uint32, _f64p]),
    "psp_gpu_query_batch": (C.c_int, [_vp, C.c_uint64, _vp, _vp, _vp, _vp]),
    "psp_gpu_query_batch_device": (C.c_int, [_vp, C.c_uint64, _vp, _vp, _vp, _vp]),
    "psp_gpu_query_pipe_create": (C.c_int, [_vp, C.c_int, C.POINTER(_vp)]),
    "psp_gpu_query_pipe_submit": (C.c_int, [_vp, C.c_uint64, _vp, _vp, _vp]),
    "psp_gpu_query_pipe_wait": (C.c_int, [_vp]),
    "psp_gpu_query_pipe_destroy": (None, [_vp]),
    "psp_place_components": (C.c_int, [C.c_uint32, C.c_uint32, C.c_int, _u32p]),
    "psp_gpu_shard_create": (C.c_int, [_vp, _u32p, C.POINTER(_vp)]),
    "psp_gpu_shard_free": (C.c_int, [_vp]),
    "psp_gpu_shard_bytes": (C.c_int, [_vp, C.POINTER(C.c_uint64)]),
    "psp_gpu_routed_query_batch": (C.c_int, [_vp, C.c_uint64, _vp, _vp, _vp, _vp, _vp, _vp,
                                             C.POINTER(RoutedStats)]),
    "psp_gpu_load_graph": (C.c_int, [_vp, C.c_char_p, C.c_int, C.POINTER(_vp)]),
    "psp_gpu_read_graph": (C.c_int, [_vp, C.c_char_p, C.c_uint64, C.c_int, C.c_char_p,
                                     C.POINTER(_vp)]),
    "psp_graph_size": (C.c_int, [_vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "psp_graph_edges": (C.c_int, [_vp, _vp, _vp, _vp]),
    "psp_graph_free": (None, [_vp]),
    "psp_gpu_last_parse_line": (C.c_uint64, []),
    "psp_write_graph": (C.c_int, [C.c_uint64, C.c_uint64, _vp, _vp, _vp, C.c_int, _vp, C.c_uint64,
                                  C.POINTER(C.c_uint64)]),
    "psp_save_graph": (C.c_int, [C.c_uint64, C.c_uint64, _vp, _vp, _vp, C.c_char_p, C.c_int]),
    "psp_format_weight": (C.c_uint32, [C.c_double, C.c_char_p]),
    "psp_gpu_apsp_dense": (C.c_int, [_vp, C.c_uint64, C.c_uint64, _u32p, _u32p, _f64p,
                                     C.c_uint64, C.c_int, _f64p]),
    "psp_gpu_boundary_apsp": (C.c_int, [_vp, C.c_uint64, C.c_uint64, _u32p, _u32p, _f64p,
                                        C.c_int, _f64p]),
    "psp_gpu_minplus_peak": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double)]),
    "psp_partition_graph": (C.c_int, [C.c_uint64, C.c_uint64, _u32p, _u32p, _f64p, C.c_uint32,
                                      C.c_uint64, C.c_uint32, _u32p]),
    "psp_generate_grid": (C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_int, C.c_double,
                                    C.c_double, C.c_uint64, C.POINTER(C.c_uint64), _vp, _vp,
                                    _vp]),
    "psp_min_spanning_forest": (C.c_int, [C.c_uint64, C.c_uint64, _u32p, _u32p, _f64p, _u8p]),
    "psp_delaunay_edges": (C.c_int, [C.c_uint64, _f64p, C.c_uint64, _u32p, _u32p,
                                     C.POINTER(C.c_uint64)]),
    "psp_random_pairs": (None, [C.c_uint64, C.c_uint64, C.c_uint64, _u32p, _u32p]),
}

_lib = None


# include/psp_gpu.h PSP_GPU_ABI_VERSION (struct layouts above follow it)
ABI_VERSION = 5


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with "
                              f"`python -c 'import __graft_entry__ as g; g.build()'` "
                              f"(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.psp_gpu_abi_version() != ABI_VERSION:
            raise ImportError(f"{LIB_PATH} has ABI {L.psp_gpu_abi_version()}, this binding "
                              f"expects {ABI_VERSION}: rebuild it")
        _lib = L
    return _lib


def check(status: int) -> None:
    if status == PSP_OK:
        return
    msg = lib().psp_gpu_last_error().decode(errors="replace")
    if status in (PSP_EINVAL, PSP_EOVERFLOW):
        raise PspValueError(status, msg)
    if status == PSP_EGRAPH:
        raise GraphInvariantError(status, msg)
    if status == PSP_ECHECKSUM:
        raise ChecksumError(status, msg)
    if status == PSP_EFORMAT:
        raise FormatVersionError(status, msg)
    if status == PSP_EIO:
        raise OracleIoError(status, msg)
    if status == PSP_EPARSE:
        raise ParseError(status, msg, int(lib().psp_gpu_last_parse_line()))
    raise PspError(status, msg)
