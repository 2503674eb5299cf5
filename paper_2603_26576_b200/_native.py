"""ctypes binding of the C ABI in ``include/heteff_b200.h``.

The shared library ``libheteff_b200.so`` is built in-tree by
``__graft_entry__.build()`` (nvcc, ``-gencode arch=compute_100a,code=sm_100a``).
There is no fallback: if the library is missing or no CUDA device is
visible, every engine call raises -- the product path never computes on the
CPU.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

LIB_PATH = Path(os.environ.get("HETEFF_LIB", Path(__file__).resolve().parent / "libheteff_b200.so"))

# status codes (heteff_status)
OK, INVALID_TRACE, ANALYSIS_ERROR, VALUE_ERROR, CONTRACT, CUDA_ERROR, NOMEM, BAD_ARG, PARSE_FALLBACK = range(9)
# modes (heteff_mode)
MODE_REPORT, MODE_SUMMARIZE_DEVICE, MODE_VALIDATE, MODE_SUMMARIZE_HOST = range(4)
# list classes
HOST_MALFORMED, HOST_ZERO, HOST_UNDECLARED, HOST_OVERLAP = range(4)
DEV_MALFORMED, DEV_ZERO, DEV_UNDECLARED, DEV_LATE = range(4, 8)
NUM_LISTS = 8

_p = C.c_void_p


class Records(C.Structure):
    _fields_ = [("start", _p), ("end", _p), ("res", _p), ("kind", _p), ("count", C.c_int64)]


class TraceABI(C.Structure):
    _fields_ = [
        ("host", Records), ("dev", Records),
        ("host_ids", C.c_int32), ("dev_ids", C.c_int32),
        ("host_decl", _p), ("dev_decl", _p),
        ("n", C.c_int32), ("m", C.c_int32),
        ("host_elapsed_floor", C.c_uint64),
        ("host_seg", _p), ("dev_seg", _p),
    ]


class Options(C.Structure):
    _fields_ = [("mode", C.c_int32), ("flags", C.c_int32), ("elapsed", C.c_uint64),
                ("list_capacity", C.c_int64)]


class Result(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("contract_flags", C.c_int32), ("contract_index", C.c_int64),
        ("host_elapsed", C.c_uint64), ("elapsed", C.c_uint64), ("dev_max_end", C.c_uint64),
        ("host_present", C.c_int32), ("device_present", C.c_int32),
        ("host_metrics", C.c_double * 5), ("host_mask", C.c_uint32), ("device_mask", C.c_uint32),
        ("device_metrics", C.c_double * 4), ("counts", C.c_int64 * NUM_LISTS), ("kernel_ms", C.c_double),
    ]


class Outputs(C.Structure):
    _fields_ = [("host_summaries", _p), ("device_summaries", _p), ("lists", _p * NUM_LISTS)]


class Columns(C.Structure):
    _fields_ = [("start", _p), ("end", _p), ("res", _p), ("kind", _p)]


class SortInfo(C.Structure):
    _fields_ = [("key_bits", C.c_int32), ("passes", C.c_int32), ("wide", C.c_int32), ("start_sorted", C.c_int32),
                ("ms", C.c_double)]


class RegionsABI(C.Structure):
    _fields_ = [("start", _p), ("end", _p), ("count", C.c_int32), ("flags", C.c_int32), ("dev_owner", _p)]


REGIONS_PER_RANK = 1


class RegionResult(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("reserved", C.c_int32), ("elapsed", C.c_uint64),
        ("host_metrics", C.c_double * 5), ("host_mask", C.c_uint32), ("device_mask", C.c_uint32),
        ("device_metrics", C.c_double * 4), ("offload_busy_fraction", C.c_double),
        ("offload_busy_defined", C.c_uint32), ("reserved2", C.c_uint32),
    ]


class RegionOutputs(C.Structure):
    _fields_ = [("results", _p), ("host_summaries", _p), ("device_summaries", _p), ("offload_busy", _p),
                ("kernel_ms", C.c_double)]


FLAG_SORT_IF_NEEDED = 1
FLAG_ELAPSED_DEVICE_PTR = 2
CONTRACT_HOST_ORDER, CONTRACT_DEV_ORDER, CONTRACT_HOST_KIND, CONTRACT_DEV_KIND = 1, 2, 4, 8


class GenSide(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64), ("n_res", C.c_int32), ("res_base", C.c_int32),
        ("per_res", C.c_int64), ("extra_below", C.c_int32), ("serialized", C.c_int32),
        ("count", C.c_int64), ("gap_max", C.c_uint32), ("dur_max", C.c_uint32),
        ("dur_scale0", C.c_uint32), ("kernel_pct", C.c_uint32), ("is_host", C.c_int32),
        ("reserved", C.c_int32),
    ]


#: every symbol include/heteff_b200.h declares
EXPORTED = (
    "heteff_abi_version", "heteff_create", "heteff_destroy", "heteff_last_error",
    "heteff_analyze", "heteff_analyze_host", "heteff_analyze_host_csr", "heteff_overlap_covers",
    "heteff_host_metrics", "heteff_device_metrics", "heteff_generate", "heteff_prof_read",
    "heteff_sort_records", "heteff_analyze_regions",
    "heteff_flatten", "heteff_subtract", "heteff_intersect", "heteff_total_duration",
    "heteff_parse_trace", "heteff_parsed_info", "heteff_parsed_free",
    "heteff_import_events", "heteff_imported_info", "heteff_imported_free",
    "heteff_analyze_into", "heteff_merge_shards", "heteff_set_grid", "heteff_kernel_name",
)

_lib = None


def load() -> C.CDLL:
    """Load the engine library (no GPU needed to load; compute calls need one)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"native engine {LIB_PATH.name} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(str(LIB_PATH))
    lib.heteff_abi_version.restype = C.c_int
    lib.heteff_create.restype = _p
    lib.heteff_create.argtypes = [C.c_int]
    lib.heteff_destroy.argtypes = [_p]
    lib.heteff_last_error.restype = C.c_char_p
    lib.heteff_last_error.argtypes = [_p]
    for name in ("heteff_analyze", "heteff_analyze_host"):
        f = getattr(lib, name)
        f.restype = C.c_int
        f.argtypes = [_p, C.POINTER(TraceABI), C.POINTER(Options), C.POINTER(Result), C.POINTER(Outputs), _p]
    lib.heteff_analyze_host_csr.restype = C.c_int
    lib.heteff_analyze_host_csr.argtypes = [_p, C.POINTER(TraceABI), _p, _p, C.POINTER(Options), C.POINTER(Result),
                                            C.POINTER(Outputs), _p]
    lib.heteff_overlap_covers.restype = C.c_int
    lib.heteff_overlap_covers.argtypes = [_p, C.POINTER(TraceABI), C.c_int, _p, C.c_int64, _p, _p]
    for name in ("heteff_host_metrics", "heteff_device_metrics"):
        f = getattr(lib, name)
        f.restype = C.c_int
        f.argtypes = [_p, _p, C.c_int32, C.c_uint64, _p, C.POINTER(C.c_uint32), _p]
    lib.heteff_prof_read.restype = C.c_int
    lib.heteff_prof_read.argtypes = [_p, C.c_int]
    lib.heteff_sort_records.restype = C.c_int
    lib.heteff_sort_records.argtypes = [_p, C.POINTER(Records), C.POINTER(Columns), _p, C.POINTER(SortInfo), _p]
    lib.heteff_analyze_regions.restype = C.c_int
    lib.heteff_analyze_regions.argtypes = [_p, C.POINTER(TraceABI), C.POINTER(RegionsABI),
                                           C.POINTER(RegionOutputs), _p]
    lib.heteff_flatten.restype = C.c_int
    lib.heteff_flatten.argtypes = [_p, _p, _p, C.c_int64, _p, _p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), _p]
    lib.heteff_subtract.restype = C.c_int
    lib.heteff_subtract.argtypes = [_p, _p, _p, C.c_int64, _p, _p, C.c_int64, _p, _p, C.POINTER(C.c_int64), _p]
    lib.heteff_intersect.restype = C.c_int
    lib.heteff_intersect.argtypes = [_p, _p, _p, C.c_int64, C.c_uint64, C.c_uint64, _p, _p, C.POINTER(C.c_int64),
                                     _p]
    lib.heteff_total_duration.restype = C.c_int
    lib.heteff_total_duration.argtypes = [_p, _p, _p, C.c_int64, _p, _p]
    lib.heteff_parse_trace.restype = C.c_int
    lib.heteff_parse_trace.argtypes = [C.c_char_p, C.c_size_t, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]
    lib.heteff_parsed_info.restype = None
    lib.heteff_parsed_info.argtypes = [C.c_void_p, C.c_void_p]
    lib.heteff_parsed_free.restype = None
    lib.heteff_parsed_free.argtypes = [C.c_void_p]
    lib.heteff_import_events.restype = C.c_int
    lib.heteff_import_events.argtypes = [C.c_char_p, C.c_size_t, C.c_void_p, C.c_int, C.c_int,
                                         C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]
    lib.heteff_imported_info.restype = None
    lib.heteff_imported_info.argtypes = [C.c_void_p, C.c_void_p]
    lib.heteff_imported_free.restype = None
    lib.heteff_imported_free.argtypes = [C.c_void_p]
    lib.heteff_analyze_into.restype = C.c_int
    lib.heteff_analyze_into.argtypes = [_p, C.POINTER(TraceABI), C.POINTER(Options), _p, C.c_size_t, C.c_int32,
                                        C.c_int32, _p]
    lib.heteff_merge_shards.restype = C.c_int
    lib.heteff_merge_shards.argtypes = [_p, _p, C.c_int32, C.c_size_t, C.c_int32, C.c_int32, _p, _p, _p,
                                        C.POINTER(Result), C.POINTER(Outputs), _p]
    if hasattr(lib, "heteff_kernel_name"):
        lib.heteff_kernel_name.restype = C.c_char_p
        lib.heteff_kernel_name.argtypes = [_p]
    if hasattr(lib, "heteff_set_grid"):   # (older builds loaded through HETEFF_LIB for A/B runs)
        lib.heteff_set_grid.restype = C.c_int
        lib.heteff_set_grid.argtypes = [_p, C.c_int]
    lib.heteff_generate.restype = C.c_int
    lib.heteff_generate.argtypes = [_p, C.POINTER(GenSide), _p, _p, _p, _p, _p]
    _lib = lib
    return lib


class NativeError(RuntimeError):
    """The engine reported a CUDA / argument failure (not a trace property)."""


_tls = threading.local()


def context(device: int | None = None) -> int:
    """Engine context for ``device`` (default: $HETEFF_DEVICE or 0), one per THREAD.

    A context owns device workspace, pinned staging and the grid-wide counters of
    its launches, so it is not thread-safe (include/heteff_b200.h); ctypes drops
    the GIL during native calls, so threads sharing one would race.  Each thread
    gets its own, which keeps the drop-in API as safe to call from threads as
    the pure-Python reference (SPEC.md's "safe to share")."""
    if device is None:
        device = int(os.environ.get("HETEFF_DEVICE", "0"))
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = {}
    if device not in cache:
        lib = load()
        h = lib.heteff_create(device)
        if not h:
            raise NativeError(f"heteff_create({device}) failed: no usable CUDA device")
        cache[device] = h
    return cache[device]


def last_error(ctx: int) -> str:
    msg = load().heteff_last_error(ctx)
    return msg.decode() if msg else ""
