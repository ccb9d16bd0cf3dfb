"""Ring^2 on the device: payload ring in HBM, descriptor ring in mapped
pinned host memory, allocator state on the device.

Python face of the reference's ``rings.py`` (tapflow, rings.py:1-437): same
constants, ``RingConfig`` validation, 64-byte ``Descriptor`` wire layout,
``RingState`` snapshot, and a ``RingPair`` with the producer role
(reserve/publish) and the consumer role (poll/release). The difference is
where the work happens:

* reservations are made by the device allocator (``ring2_core.h``
  ``tf_reserve``), either inside a capture kernel or, for the protocol-level
  calls below, by a one-thread kernel;
* descriptors are written by the device into the mapped meta ring and
  polled by the host with acquire loads;
* payload bytes live in device memory; ``payload_view`` returns a window
  that reads/writes through CUDA.

Snapshots (``state``, ``would_fit``, ``occupancy``) read the producer's
mirrored cursors, so they wait for the last capture launch this object was
told about (``note_launch``) before reading.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field

from . import _native as N
from ._device import bytes_tensor, require_cuda, stream_handle, torch
from .errors import AllocationError, ConfigError

COPY_UNIT = 16
DESCRIPTOR_SIZE = 64
READY_SENTINEL = (1 << 64) - 1

_WIRE = struct.Struct("<QQIIQ")          # reference bytes 0..31
_WIRE_EXT = struct.Struct("<QIIQQ")      # our reserved bytes 32..63


def round_up_to_copy_unit(n: int) -> int:
    """Smallest multiple of the 16-byte copy unit >= n (rings.py:63-64)."""
    return -(-n // COPY_UNIT) * COPY_UNIT


@dataclass(frozen=True)
class RingConfig:
    """Capacity of one ring pair (rings.py:67-85)."""

    payload_capacity: int
    meta_slots: int
    high_watermark: float = 0.8

    def __post_init__(self) -> None:
        cap = self.payload_capacity
        if cap <= 0:
            raise ConfigError("payload_capacity must be positive")
        if cap % COPY_UNIT != 0:
            raise ConfigError(
                f"payload_capacity must be a multiple of {COPY_UNIT} bytes")
        if self.meta_slots <= 0:
            raise ConfigError("meta_slots must be positive")
        if not (0.0 < self.high_watermark <= 1.0):
            raise ConfigError("high_watermark must be in (0, 1]")


@dataclass(frozen=True)
class Descriptor:
    """One 64-byte meta slot (rings.py:88-118).

    The five reference fields take part in equality; the transport fields
    the device producer fills into the reserved bytes do not.
    """

    payload_offset: int
    payload_len: int
    hook_id: int
    step_seq: int
    ready_seq: int = 0
    skip_before: int = field(default=0, compare=False)
    flags: int = field(default=0, compare=False)
    n_rows: int = field(default=0, compare=False)
    capture_seq: int = field(default=0, compare=False)

    def pack(self) -> bytes:
        """Reference wire image: reserved bytes zero (rings.py:98-106)."""
        head = _WIRE.pack(self.payload_offset, self.payload_len,
                          self.hook_id, self.step_seq, self.ready_seq)
        return head + bytes(DESCRIPTOR_SIZE - len(head))

    def pack_device(self) -> bytes:
        """Image as the device writes it (transport facts in bytes 32..63)."""
        head = _WIRE.pack(self.payload_offset, self.payload_len,
                          self.hook_id, self.step_seq, self.ready_seq)
        return head + _WIRE_EXT.pack(self.skip_before, self.flags,
                                     self.n_rows, self.capture_seq, 0)

    @classmethod
    def unpack(cls, raw) -> "Descriptor":
        if len(raw) != DESCRIPTOR_SIZE:
            raise ValueError(f"descriptor must be {DESCRIPTOR_SIZE} bytes")
        off, length, hook, step, ready = _WIRE.unpack_from(raw, 0)
        skip, flags, rows, cseq, _ = _WIRE_EXT.unpack_from(raw, 32)
        return cls(off, length, hook, step, ready, skip, flags, rows, cseq)

    @classmethod
    def from_c(cls, d: N.CDescriptor) -> "Descriptor":
        return cls(d.payload_offset, d.payload_len, d.hook_id, d.step_seq,
                   d.ready_seq, d.skip_before, d.flags, d.n_rows,
                   d.capture_seq)

    def to_c(self) -> N.CDescriptor:
        return N.CDescriptor(self.payload_offset, self.payload_len,
                             self.hook_id, self.step_seq, self.ready_seq,
                             self.skip_before, self.flags, self.n_rows,
                             self.capture_seq, 0)

    @property
    def reserved_len(self) -> int:
        """Bytes the region holds in the payload ring (padded)."""
        return round_up_to_copy_unit(self.payload_len)


@dataclass(frozen=True)
class RingState:
    """Read-only snapshot (rings.py:121-144) plus device counters."""

    payload_head: int
    payload_tail: int
    occupancy: int
    payload_capacity: int
    meta_head: int
    meta_tail: int
    meta_slots: int
    high_watermark: float
    drops: int = 0
    drop_bytes: int = 0
    stall_events: int = 0
    stall_ns: int = 0
    device_errors: int = 0
    captures_launched: int = 0
    kernel_ns: int = 0

    @property
    def free_bytes(self) -> int:
        return self.payload_capacity - self.occupancy

    @property
    def free_meta_slots(self) -> int:
        return self.meta_slots - (self.meta_head - self.meta_tail)

    @property
    def pressure(self) -> float:
        return self.occupancy / self.payload_capacity


class Arena:
    """Capacity accounting for a memory arena (rings.py:147-163).

    Bounded arenas refuse an allocation before any device memory is taken;
    the real backing comes from cudaMalloc / cudaHostAlloc.
    """

    def __init__(self, capacity: int | None = None, name: str = "device") -> None:
        self.capacity = capacity
        self.name = name
        self.allocated = 0

    def allocate(self, nbytes: int) -> int:
        limit = self.capacity
        if limit is not None and self.allocated + nbytes > limit:
            raise AllocationError(
                f"{self.name} arena cannot satisfy {nbytes} bytes "
                f"({self.allocated}/{limit} in use)")
        base, self.allocated = self.allocated, self.allocated + nbytes
        return base


class PayloadWindow:
    """Borrowed window [offset, offset+length) of the device payload ring."""

    def __init__(self, ring: "RingPair", offset: int, length: int) -> None:
        self._ring, self.offset, self.length = ring, offset, length

    def __len__(self) -> int:
        return self.length

    @property
    def tensor(self):
        return bytes_tensor(self._ring.payload_ptr + self.offset, self.length,
                            self._ring.device)

    def __bytes__(self) -> bytes:
        self._ring.sync()
        return self.tensor.cpu().numpy().tobytes()

    def tobytes(self) -> bytes:
        return bytes(self)

    def __setitem__(self, index, value) -> None:
        if index != slice(None):
            raise TypeError("payload windows accept whole-window assignment")
        data = bytes(value)
        if len(data) != self.length:
            raise ValueError("assignment size differs from the window")
        t = torch()
        src = t.frombuffer(bytearray(data), dtype=t.uint8)
        self.tensor.copy_(src)
        t.cuda.synchronize(self._ring.device)


class RingPair:
    """One payload ring plus one meta ring, one producer, one consumer.

    ``device`` selects the GPU (default: torch's current device).
    ``wait_timeout`` bounds a device-side completeness stall (seconds).
    """

    def __init__(self, config: RingConfig, device_arena: Arena | None = None,
                 host_arena: Arena | None = None, *, device: int | None = None,
                 wait_timeout: float = 30.0) -> None:
        self.config = config
        self.device_base = (device_arena or Arena()).allocate(
            config.payload_capacity)
        self.host_base = (host_arena or Arena(name="host")).allocate(
            config.meta_slots * DESCRIPTOR_SIZE)
        require_cuda()
        t = torch()
        self.device = t.cuda.current_device() if device is None else int(device)
        cfg = N.CRingConfig(config.payload_capacity, config.meta_slots, 0,
                            config.high_watermark, int(wait_timeout * 1e9))
        handle = C.c_void_p()
        N.check(N.lib().tf_ring_create(C.byref(cfg), self.device,
                                       C.byref(handle)))
        self._h = handle
        ptr = C.c_void_p()
        N.check(N.lib().tf_ring_payload_ptr(handle, C.byref(ptr)))
        self.payload_ptr = int(ptr.value)
        self._pending = None  # torch event of the last producer launch

    # -- lifecycle ---------------------------------------------------------

    @property
    def handle(self) -> C.c_void_p:
        if self._h is None:
            raise ConfigError("ring pair is closed")
        return self._h

    def close(self) -> None:
        h, self._h = getattr(self, "_h", None), None
        if h is not None:
            N.lib().tf_ring_destroy(h)

    def __del__(self) -> None:  # pragma: no cover - GC timing
        try:
            self.close()
        except Exception:
            pass

    def note_launch(self, stream=None) -> None:
        """Remember the producer stream position for snapshot fencing (one
        event, re-recorded: a serving engine notes every step)."""
        t = torch()
        ev = getattr(self, "_note_ev", None)
        if ev is None:
            ev = self._note_ev = t.cuda.Event()
        ev.record(stream if stream is not None
                  else t.cuda.current_stream(self.device))
        self._pending = ev

    def sync(self) -> None:
        """Wait until every capture noted so far has finished on device."""
        ev, self._pending = self._pending, None
        if ev is not None:
            ev.synchronize()

    def seal(self, stream=None) -> None:
        """Stream-ordered: once the earlier work on `stream` (default: the
        current stream) has run, every descriptor posted so far is complete
        (captures launched with ``sealed=True``)."""
        N.check(N.lib().tf_ring_seal(self.handle, stream_handle(stream, self.device)))

    def sync_consumer(self) -> None:
        """Wait until the device sees every release/poll made so far."""
        N.check(N.lib().tf_ring_sync_consumer(self.handle))

    # -- shared --------------------------------------------------------------

    @property
    def capacity(self) -> int:
        return self.config.payload_capacity

    def _cstate(self) -> N.CRingState:
        self.sync()
        st = N.CRingState()
        N.check(N.lib().tf_ring_get_state(self.handle, C.byref(st)))
        return st

    @property
    def occupancy(self) -> int:
        return self._cstate().occupancy

    def state(self) -> RingState:
        s = self._cstate()
        return RingState(
            payload_head=s.payload_head, payload_tail=s.payload_tail,
            occupancy=s.occupancy, payload_capacity=s.payload_capacity,
            meta_head=s.meta_head, meta_tail=s.meta_tail,
            meta_slots=s.meta_slots, high_watermark=s.high_watermark,
            drops=s.drops, drop_bytes=s.drop_bytes,
            stall_events=s.stall_events, stall_ns=s.stall_ns,
            device_errors=s.device_errors,
            captures_launched=s.captures_launched, kernel_ns=s.kernel_ns)

    def counters(self) -> dict:
        s = self._cstate()
        return {name: getattr(s, name) for name, _ in N.CRingState._fields_}

    # conservation counters (rings.py:223-229)
    bytes_reserved = property(lambda self: self._cstate().bytes_reserved)
    bytes_released = property(lambda self: self._cstate().bytes_released)
    dead_created = property(lambda self: self._cstate().dead_created)
    dead_reclaimed = property(lambda self: self._cstate().dead_reclaimed)
    descriptors_published = property(
        lambda self: self._cstate().descriptors_published)
    descriptors_consumed = property(
        lambda self: self._cstate().descriptors_consumed)

    def free_meta_slots(self) -> int:
        self.sync()
        n = C.c_uint64()
        N.check(N.lib().tf_ring_free_meta_slots(self.handle, C.byref(n)))
        return n.value

    def would_fit(self, lengths, meta_entries: int | None = None) -> bool:
        """Replay the device allocator with a frozen consumer (rings.py:256-276)."""
        lengths = list(lengths)
        for n in lengths:
            if n <= 0 or n % COPY_UNIT:
                raise ValueError("lengths must be positive copy-unit multiples")
        self.sync()
        arr = (C.c_uint64 * max(1, len(lengths)))(*lengths)
        fits = C.c_int()
        N.check(N.lib().tf_ring_would_fit(
            self.handle, arr, len(lengths),
            -1 if meta_entries is None else int(meta_entries), C.byref(fits)))
        return bool(fits.value)

    def payload_view(self, offset: int, length: int) -> PayloadWindow:
        if offset < 0 or offset + length > self.config.payload_capacity:
            raise ValueError("payload window out of range")
        return PayloadWindow(self, offset, length)

    # -- producer role (protocol-level, synchronous) ------------------------

    def reserve_payload(self, length: int) -> int:
        """Reserve contiguous bytes via the device allocator (rings.py:286-319)."""
        if length <= 0:
            raise ValueError("reservation length must be positive")
        if length % COPY_UNIT:
            raise ValueError("reservation length must be a copy-unit multiple")
        if length > self.config.payload_capacity:
            raise ValueError("reservation exceeds payload capacity")
        self.sync()
        off = C.c_uint64()
        N.check(N.lib().tf_ring_reserve(self.handle, None, length,
                                        C.byref(off), None))
        return off.value

    def publish(self, desc: Descriptor) -> int:
        """Publish one descriptor from the device (rings.py:321-342)."""
        self.sync()
        seq = C.c_uint64()
        cd = desc.to_c()
        N.check(N.lib().tf_ring_publish(self.handle, None, C.byref(cd),
                                        C.byref(seq)))
        return seq.value

    # -- consumer role -------------------------------------------------------

    def ready_entries(self) -> int:
        n = C.c_uint64()
        N.check(N.lib().tf_ring_ready_entries(self.handle, C.byref(n)))
        return n.value

    def ready_bytes(self) -> int:
        n = C.c_uint64()
        N.check(N.lib().tf_ring_ready_bytes(self.handle, C.byref(n)))
        return n.value

    def _take(self, fn, max_entries: int) -> list[Descriptor]:
        if max_entries <= 0:
            return []
        cap = min(int(max_entries), self.config.meta_slots)
        buf = (N.CDescriptor * cap)()
        got = C.c_uint32()
        N.check(fn(self.handle, cap, buf, C.byref(got)))
        return [Descriptor.from_c(buf[i]) for i in range(got.value)]

    def peek_ready(self, max_entries: int) -> list[Descriptor]:
        return self._take(N.lib().tf_ring_peek_ready, max_entries)

    def poll_ready(self, max_entries: int) -> list[Descriptor]:
        """Consume published descriptors in order (rings.py:380-406)."""
        return self._take(N.lib().tf_ring_poll_ready, max_entries)

    def release_payload(self, through_offset: int, length: int) -> None:
        """Release the oldest region; must match reservation order."""
        N.check(N.lib().tf_ring_release_payload(self.handle, through_offset,
                                                length))


def allocate_rings(config: RingConfig, device_arena: Arena | None = None,
                   host_arena: Arena | None = None, **kw) -> RingPair:
    """One ring pair on the current CUDA device (rings.py:434-437)."""
    return RingPair(config, device_arena=device_arena, host_arena=host_arena,
                    **kw)
