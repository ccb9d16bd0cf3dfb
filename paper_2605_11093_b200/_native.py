"""ctypes binding of ``include/ring2.h`` (the C-ABI drop-in boundary).

Every structure below mirrors the header field for field; ``check`` turns a
non-zero ``tf_status`` into the matching exception from ``errors``. There is
no CPU fallback: if the shared library is missing and cannot be built, the
first call raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from . import errors

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libring2.so"
_lock = threading.Lock()
_lib: C.CDLL | None = None

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)

# status codes (ring2.h tf_status)
TF_OK = 0
TF_ERR_CONFIG = 1
TF_ERR_ALLOCATION = 2
TF_ERR_PAYLOAD_RING_FULL = 3
TF_ERR_META_RING_FULL = 4
TF_ERR_OUT_OF_ORDER_RELEASE = 5
TF_ERR_PROTOCOL = 6
TF_ERR_META_MISMATCH = 7
TF_ERR_POLICY_UNDERESTIMATE = 8
TF_ERR_STAGING_EXHAUSTED = 9
TF_ERR_HOOK_DISABLED = 10
TF_ERR_VALUE = 11
TF_ERR_CUDA = 12
TF_ERR_TIMEOUT = 13
TF_ERR_EMPTY = 14

TF_DESC_DEAD_SKIP = 0x1
TF_DESC_EMPTY_RESET = 0x2
TF_DESC_HOST_RESERVED = 0x4

TF_DEVERR_UNDERESTIMATE = 0x1
TF_DEVERR_TIMEOUT = 0x2
TF_DEVERR_TOO_LARGE = 0x4
TF_DEVERR_PROTOCOL = 0x8

TF_FULL_RAISE = 0
TF_FULL_WAIT = 1
TF_FULL_DROP = 2
TF_CAP_DEFER_PUBLISH = 0x4
TF_CAP_SEALED = 0x10
TF_DESC_PENDING = 0x8000
TF_CAP_KEEP_PER_OUTER = 0x8

TF_OP_COPY, TF_OP_CAST, TF_OP_REDUCE = 0, 1, 2
TF_RED = {"mean": 0, "l2": 1, "absmax": 2, "rms": 3, "stats": 4}
TF_RED_K = {"mean": 1, "l2": 1, "absmax": 1, "rms": 1, "stats": 4}

TF_DTYPE = {"u8": 0, "i8": 1, "f16": 2, "bf16": 3, "f32": 4, "i32": 5,
            "f64": 6, "i64": 7, "f8e4m3": 8, "f8e5m2": 9}

TF_STAGE_COPY_ENGINE = 0
TF_STAGE_MAPPED = 1
TF_PAGE_OUT = {"copy": 0, "handoff": 1, "discard": 2}
REASONS = {0: "none", 1: "entries", 2: "bytes", 3: "timeout", 4: "flush"}


class CDescriptor(C.Structure):
    _fields_ = [("payload_offset", C.c_uint64), ("payload_len", C.c_uint64),
                ("hook_id", C.c_uint32), ("step_seq", C.c_uint32),
                ("ready_seq", C.c_uint64), ("skip_before", C.c_uint64),
                ("flags", C.c_uint32), ("n_rows", C.c_uint32),
                ("capture_seq", C.c_uint64), ("checksum", C.c_uint64)]


class CCaptureMeta(C.Structure):
    """tf_capture_meta (include/ring2.h): one matched capture for the sinks."""
    _fields_ = [("hook_name", C.c_char_p), ("layer", C.c_int64),
                ("step_seq", C.c_int64), ("tp_rank", C.c_int64),
                ("pp_stage", C.c_int64), ("dtype", C.c_char_p),
                ("n_req", C.c_uint32), ("ndim", C.c_uint32),
                ("request_ids", C.c_void_p), ("token_ranges", C.c_void_p),
                ("row_counts", C.c_void_p), ("shape", C.c_void_p),
                ("row_bytes", C.c_int64), ("payload", C.c_void_p),
                ("payload_len", C.c_uint64)]


class CRingConfig(C.Structure):
    _fields_ = [("payload_capacity", C.c_uint64), ("meta_slots", C.c_uint32),
                ("_pad", C.c_uint32), ("high_watermark", C.c_double),
                ("wait_timeout_ns", C.c_uint64)]


class CRingState(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "payload_head", "payload_tail", "occupancy", "payload_capacity",
        "meta_head", "meta_tail", "meta_slots")] + [
        ("high_watermark", C.c_double)] + [(n, C.c_uint64) for n in (
            "bytes_reserved", "bytes_released", "dead_created",
            "dead_reclaimed", "descriptors_published", "descriptors_consumed",
            "captures_launched", "drops", "drop_bytes", "stall_events",
            "stall_ns", "device_errors", "kernel_ns", "last_kernel_ns")]


class CCaptureArgs(C.Structure):
    _fields_ = [("src", C.c_void_p), ("outer", C.c_int64), ("mid", C.c_int64),
                ("row_bytes", C.c_int64), ("stride_outer", C.c_int64),
                ("stride_mid", C.c_int64), ("keep", C.c_void_p),
                ("step_seq_ptr", C.c_void_p), ("step_seq", C.c_uint32),
                ("hook_id", C.c_uint32), ("op", C.c_uint32),
                ("in_dtype", C.c_uint32), ("out_dtype", C.c_uint32),
                ("reduce_op", C.c_uint32), ("flags", C.c_uint32),
                ("max_ctas", C.c_uint32)]


class CCaptureResult(C.Structure):
    _fields_ = [("capture_seq", C.c_uint64), ("status", C.c_uint32),
                ("n_rows", C.c_uint32), ("payload_offset", C.c_uint64),
                ("payload_len", C.c_uint64), ("skip_before", C.c_uint64),
                ("ready_seq", C.c_uint64), ("desc", CDescriptor)]


class CDrainConfig(C.Structure):
    _fields_ = [("min_ready_entries", C.c_uint64),
                ("min_ready_bytes", C.c_uint64), ("max_wait", C.c_double),
                ("staging_buffer_size", C.c_uint64),
                ("staging_buffer_count", C.c_uint64), ("mode", C.c_uint32),
                ("mapped_ctas", C.c_uint32), ("numa_node", C.c_int32),
                ("stage_queue_slots", C.c_uint32),
                ("stage_threads", C.c_uint32), ("page_out", C.c_uint32),
                ("split_oversize", C.c_uint32)]


class CBatchInfo(C.Structure):
    _fields_ = [("batch_id", C.c_uint64), ("n_entries", C.c_uint32),
                ("buffer_index", C.c_uint32), ("bytes_total", C.c_uint64),
                ("reason", C.c_uint32), ("_pad", C.c_uint32)]


class CStagerStats(C.Structure):
    _fields_ = [("batches_drained", C.c_uint64), ("batches_staged", C.c_uint64),
                ("entries_drained", C.c_uint64), ("bytes_drained", C.c_uint64),
                ("transfer_seconds", C.c_double), ("pool_checkouts", C.c_uint64),
                ("pool_max_in_use", C.c_uint64),
                ("max_transient_bytes", C.c_uint64),
                ("pageable_bytes_in_flight", C.c_uint64),
                ("staging_exhausted_waits", C.c_uint64),
                ("first_drain_time", C.c_double),
                ("last_release_time", C.c_double),
                ("pool_total", C.c_uint64), ("pool_free", C.c_uint64),
                ("inflight_batches", C.c_uint64), ("to_stage_batches", C.c_uint64),
                ("out_q_batches", C.c_uint64), ("outstanding_paged", C.c_uint64),
                ("completion_phase", C.c_uint32), ("stage_phase", C.c_uint32)]


class CPagedBatch(C.Structure):
    _fields_ = [("batch_id", C.c_uint64), ("n_entries", C.c_uint32),
                ("reason", C.c_uint32), ("bytes_total", C.c_uint64),
                ("payload", C.c_void_p), ("descs", C.POINTER(CDescriptor)),
                ("starts", u64p), ("pinned_buffer", C.c_int32),
                ("oversize", C.c_uint32)]


assert C.sizeof(CDescriptor) == 64
assert C.sizeof(CCaptureArgs) == 96

# (name, restype, argtypes)
_SIGS = [
    ("tf_abi_version", C.c_int, []),
    ("tf_status_name", C.c_char_p, [C.c_int]),
    ("tf_last_error", C.c_char_p, []),
    ("tf_device_count", C.c_int, [C.POINTER(C.c_int)]),
    ("tf_plan_reservation", C.c_int, [C.c_uint64] * 5 + [u64p, u64p]),
    ("tf_ring_create", C.c_int, [C.POINTER(CRingConfig), C.c_int, C.POINTER(C.c_void_p)]),
    ("tf_ring_destroy", C.c_int, [C.c_void_p]),
    ("tf_ring_payload_ptr", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    ("tf_ring_meta_ptr", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    ("tf_capture", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(CCaptureArgs)]),
    ("tf_capture_out_row_bytes", C.c_int, [C.POINTER(CCaptureArgs), C.POINTER(C.c_int64)]),
    ("tf_ring_reserve", C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, u64p, u64p]),
    ("tf_ring_publish", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(CDescriptor), u64p]),
    ("tf_ring_last_result", C.c_int, [C.c_void_p, C.POINTER(CCaptureResult)]),
    ("tf_ring_ready_entries", C.c_int, [C.c_void_p, u64p]),
    ("tf_ring_ready_bytes", C.c_int, [C.c_void_p, u64p]),
    ("tf_ring_peek_ready", C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(CDescriptor), u32p]),
    ("tf_ring_poll_ready", C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(CDescriptor), u32p]),
    ("tf_ring_release_payload", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64]),
    ("tf_ring_sync_consumer", C.c_int, [C.c_void_p]),
    ("tf_ring_seal", C.c_int, [C.c_void_p, C.c_void_p]),
    ("tf_ring_get_state", C.c_int, [C.c_void_p, C.POINTER(CRingState)]),
    ("tf_ring_free_meta_slots", C.c_int, [C.c_void_p, u64p]),
    ("tf_ring_host_released", C.c_int, [C.c_void_p, u64p, u64p]),
    ("tf_ring_would_fit", C.c_int, [C.c_void_p, u64p, C.c_uint32, C.c_int64, C.POINTER(C.c_int)]),
    ("tf_stager_create", C.c_int, [C.c_void_p, C.POINTER(CDrainConfig), C.POINTER(C.c_void_p)]),
    ("tf_stager_destroy", C.c_int, [C.c_void_p]),
    ("tf_stager_thresholds_met", C.c_int, [C.c_void_p, C.c_double, u32p]),
    ("tf_stager_note_publish", C.c_int, [C.c_void_p, C.c_double]),
    ("tf_stager_drain_once", C.c_int, [C.c_void_p, C.c_double, C.c_int, C.POINTER(CBatchInfo)]),
    ("tf_stager_batch_entries", C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(CDescriptor), u64p, C.c_uint32]),
    ("tf_stager_batch_buffer", C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p)]),
    ("tf_stager_transfer_seconds", C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_double)]),
    ("tf_stager_complete_transfer", C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_double)]),
    ("tf_stager_stage_to_pageable", C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]),
    ("tf_stager_start", C.c_int, [C.c_void_p]),
    ("tf_stager_stop", C.c_int, [C.c_void_p]),
    ("tf_stager_flush", C.c_int, [C.c_void_p, C.c_double]),
    ("tf_stager_next", C.c_int, [C.c_void_p, C.c_double, C.POINTER(CPagedBatch)]),
    ("tf_stager_free_paged", C.c_int, [C.c_void_p, C.POINTER(CPagedBatch)]),
    ("tf_stager_note_sunk", C.c_int, [C.c_void_p, C.c_uint64]),
    ("tf_stager_stats_get", C.c_int, [C.c_void_p, C.POINTER(CStagerStats)]),
    ("tf_stager_error", C.c_int, [C.c_void_p]),
    ("tf_stager_stream", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    ("tf_stager_placement", C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_uint32,
                                      C.POINTER(C.c_uint32), C.POINTER(C.c_int32)]),
    ("tf_free_host", None, [C.c_void_p]),
    ("tf_measure_d2h", C.c_int, [C.c_int, C.c_uint64, C.c_int, C.POINTER(C.c_double)]),
    ("tf_monotonic", C.c_double, []),
    ("tf_sink_open_dataset", C.c_int, [C.c_char_p, C.c_uint32, C.POINTER(C.c_void_p)]),
    ("tf_sink_open_stream", C.c_int, [C.c_int, C.c_uint32, C.POINTER(C.c_void_p)]),
    ("tf_sink_open_dataset2", C.c_int, [C.c_char_p, C.c_uint32, C.c_uint32,
                                        C.POINTER(C.c_void_p)]),
    ("tf_sink_is_direct", C.c_int, [C.c_void_p]),
    ("tf_sink_write", C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32]),
    ("tf_sink_stats", C.c_int, [C.c_void_p, u64p, u64p]),
    ("tf_sink_flush", C.c_int, [C.c_void_p]),
    ("tf_sink_close", C.c_int, [C.c_void_p]),
    ("tf_sink_crc32", C.c_uint32, [C.c_uint32, C.c_void_p, C.c_uint64]),
]

EXPORTED = [name for name, _, _ in _SIGS]


def library_path() -> Path:
    return _LIB_PATH


def lib() -> C.CDLL:
    """Load (building first if absent) the C-ABI library."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        from . import build_ext
        build_ext.build()  # no-op unless sources are newer than the .so
        path = _LIB_PATH
        variant = os.environ.get("TF_LIB_VARIANT")
        if variant:  # experiment builds (build_ext --variant=trace)
            path = _LIB_PATH.with_name(f"libring2_{variant}.so")
        if not path.exists():  # pragma: no cover - build raises first
            raise RuntimeError(f"native library missing: {path}")
        handle = C.CDLL(str(path))
        for name, res, args in _SIGS:
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
        return handle


_STATUS_EXC = {
    TF_ERR_CONFIG: errors.ConfigError,
    TF_ERR_ALLOCATION: errors.AllocationError,
    TF_ERR_PAYLOAD_RING_FULL: errors.PayloadRingFull,
    TF_ERR_META_RING_FULL: errors.MetaRingFull,
    TF_ERR_OUT_OF_ORDER_RELEASE: errors.OutOfOrderRelease,
    TF_ERR_PROTOCOL: errors.ProtocolError,
    TF_ERR_META_MISMATCH: errors.MetaMismatch,
    TF_ERR_POLICY_UNDERESTIMATE: errors.PolicyUnderestimate,
    TF_ERR_STAGING_EXHAUSTED: errors.StagingExhausted,
    TF_ERR_HOOK_DISABLED: errors.HookDisabled,
    TF_ERR_VALUE: ValueError,
    TF_ERR_CUDA: errors.DeviceError,
    TF_ERR_TIMEOUT: errors.DeviceError,
}


def exception_for(rc: int, detail: str = "") -> BaseException:
    cls = _STATUS_EXC.get(rc, errors.TapflowError)
    name = lib().tf_status_name(rc).decode()
    return cls(detail or f"{name} (status {rc})")


def check(rc: int) -> None:
    if rc != TF_OK:
        detail = lib().tf_last_error().decode(errors="replace")
        raise exception_for(rc, detail)


def desc_to_tuple(d: CDescriptor) -> tuple:
    return (d.payload_offset, d.payload_len, d.hook_id, d.step_seq,
            d.ready_seq, d.skip_before, d.flags, d.n_rows, d.capture_seq)
