"""CPU oracle for the Ring^2 capture-and-stage path — TEST INFRASTRUCTURE.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline``
leg may import this package, and only as the checker / the timed CPU
baseline. The product path (``paper_2605_11093_b200``) never imports it.

Contents
  * ``liboracle.so`` (ring_oracle.c, cast_oracle.c): C restatement of the
    reference's allocator, descriptor ring, gather-compact (rings.py,
    hooks.py), plus the cast/reduce restatement for the north-star
    extensions;
  * ``workload``: restatement of the reference's synthetic content keying
    (workload.py:193-244) and synchronous reference records (oracle.py).

Parity pins: tests/test_oracle_golden.py checks this oracle against golden
vectors produced by importing the reference (tests/golden/make_golden.py)
and against the reference's own known-answer tests.
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

_DIR = Path(__file__).resolve().parent
_SO = _DIR / "_build" / "liboracle.so"
_lib = None

u64p = C.POINTER(C.c_uint64)


def build() -> Path:
    srcs = [_DIR / "ring_oracle.c", _DIR / "cast_oracle.c"]
    if not _SO.exists() or any(s.stat().st_mtime > _SO.stat().st_mtime for s in srcs):
        subprocess.run(["make", "-s", "-C", str(_DIR)], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        h = C.CDLL(str(_SO))
        sig = {
            "or_plan": (C.c_int, [C.c_uint64] * 5 + [u64p, u64p]),
            "or_ring_new": (C.c_void_p, [C.c_uint64, C.c_uint64]),
            "or_ring_free": (None, [C.c_void_p]),
            "or_reserve": (C.c_int, [C.c_void_p, C.c_uint64, u64p, u64p]),
            "or_publish": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64,
                                     C.c_uint32, C.c_uint32, u64p]),
            "or_poll": (C.c_int, [C.c_void_p, C.c_uint64, u64p, u64p]),
            "or_release": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64]),
            "or_would_fit": (C.c_int, [C.c_void_p, u64p, C.c_uint64, C.c_int64]),
            "or_state": (None, [C.c_void_p, u64p]),
            "or_desc_pack": (None, [C.c_uint64, C.c_uint64, C.c_uint32,
                                    C.c_uint32, C.c_uint64, C.c_char_p]),
            "or_gather": (C.c_uint64, [C.c_char_p, C.c_int64, C.c_int64,
                                       C.c_int64, C.c_int64, C.c_int64,
                                       C.c_char_p, C.c_int, C.c_char_p]),
            "or_cast": (C.c_long, [C.c_char_p, C.c_long, C.c_int, C.c_int,
                                   C.c_char_p]),
            "or_decode": (C.c_float, [C.c_char_p, C.c_int]),
            "or_reduce": (C.c_long, [C.c_char_p, C.c_long, C.c_long, C.c_long,
                                     C.c_int, C.c_int, C.POINTER(C.c_float)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(h, name)
            fn.restype, fn.argtypes = res, args
        _lib = h
    return _lib


OK, PAYLOAD_FULL, META_FULL, OUT_OF_ORDER, PROTOCOL, VALUE = 0, 3, 4, 5, 6, 11


def plan(head, tail, used, cap, length):
    o, d = C.c_uint64(), C.c_uint64()
    ok = lib().or_plan(head, tail, used, cap, length, C.byref(o), C.byref(d))
    return (o.value, d.value) if ok else None


class OracleRing:
    """The reference RingPair's rules restated in C (rings.py:196-431)."""

    def __init__(self, capacity: int, meta_slots: int) -> None:
        self.capacity, self.meta_slots = capacity, meta_slots
        self._h = lib().or_ring_new(capacity, meta_slots)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_ring_free(self._h)
            self._h = None

    def reserve(self, length: int):
        """(status, offset, dead)."""
        o, d = C.c_uint64(), C.c_uint64()
        rc = lib().or_reserve(self._h, length, C.byref(o), C.byref(d))
        return rc, o.value, d.value

    def publish(self, off, length, hook, step):
        s = C.c_uint64()
        rc = lib().or_publish(self._h, off, length, hook, step, C.byref(s))
        return rc, s.value

    def poll(self, max_entries: int):
        out = (C.c_uint64 * (5 * max(1, min(max_entries, self.meta_slots))))()
        n = C.c_uint64()
        rc = lib().or_poll(self._h, min(max_entries, self.meta_slots), out,
                           C.byref(n))
        return rc, [tuple(out[i * 5:(i + 1) * 5]) for i in range(n.value)]

    def release(self, off, length) -> int:
        return lib().or_release(self._h, off, length)

    def would_fit(self, lengths, meta_entries=None) -> bool:
        arr = (C.c_uint64 * max(1, len(lengths)))(*lengths)
        rc = lib().or_would_fit(self._h, arr, len(lengths),
                                -1 if meta_entries is None else meta_entries)
        if rc < 0:
            raise ValueError("lengths must be positive copy-unit multiples")
        return bool(rc)

    def state(self) -> dict:
        out = (C.c_uint64 * 14)()
        lib().or_state(self._h, out)
        keys = ("head", "tail", "used", "cap", "meta_head", "meta_tail",
                "slots", "bytes_reserved", "bytes_released", "dead_created",
                "dead_reclaimed", "published", "consumed", "ready")
        return dict(zip(keys, out))


def desc_pack(off, length, hook, step, ready) -> bytes:
    buf = C.create_string_buffer(64)
    lib().or_desc_pack(off, length, hook, step, ready, buf)
    return buf.raw


def gather(src: bytes, outer: int, mid: int, row_bytes: int, s_outer: int,
           s_mid: int, keep=None, per_outer: bool = False) -> bytes:
    """Kept rows packed in (o, m) order (hooks.py:266-278 generalised)."""
    n_units = outer if per_outer else outer * mid
    kb = None if keep is None else bytes(1 if k else 0 for k in keep)
    if kb is not None and len(kb) != n_units:
        raise ValueError("keep length mismatch")
    dst = C.create_string_buffer(max(1, outer * mid * row_bytes))
    n = lib().or_gather(bytes(src), outer, mid, row_bytes, s_outer, s_mid, kb,
                        1 if per_outer else 0, dst)
    return dst.raw[:n]


DT = {"f16": 2, "bf16": 3, "f32": 4, "f8e4m3": 8, "f8e5m2": 9}
WIDTH = {"f16": 2, "bf16": 2, "f32": 4, "f8e4m3": 1, "f8e5m2": 1}
RED = {"mean": 0, "l2": 1, "absmax": 2, "rms": 3, "stats": 4}


def cast(src: bytes, in_dt: str, out_dt: str) -> bytes:
    n = len(src) // WIDTH[in_dt]
    dst = C.create_string_buffer(max(1, n * WIDTH[out_dt]))
    w = lib().or_cast(bytes(src), n, DT[in_dt], DT[out_dt], dst)
    if w < 0:
        raise ValueError("unsupported cast")
    return dst.raw[:w]


def reduce(src: bytes, rows: int, h: int, in_dt: str, op: str):
    """Per-row reductions -> list of float tuples."""
    k = 4 if op == "stats" else 1
    out = (C.c_float * max(1, rows * k))()
    rc = lib().or_reduce(bytes(src), rows, h, h * WIDTH[in_dt], DT[in_dt],
                         RED[op], out)
    if rc < 0:
        raise ValueError("unsupported reduce")
    return [tuple(out[r * k:(r + 1) * k]) for r in range(rows)]


def decode(code: bytes, dt: str) -> float:
    return lib().or_decode(code, DT[dt])
