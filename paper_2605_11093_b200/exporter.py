"""Export pipeline: drain ring regions to pinned host memory, page out,
reconstruct records, sink.

API and semantics of the reference ``ExportPipeline`` (exporter.py:1-327):
thresholds (ANY of entries / bytes / oldest age), ``drain_once`` taking the
ready descriptors that fit one staging buffer (oversize single capture ->
ConfigError, no free buffer -> StagingExhausted), ``complete_transfer``
releasing the regions once the copy has landed, ``stage_to_pageable``
returning the buffer to the pool before anything downstream, and
``sink_batch`` matching the FIFO (fatal on mismatch) and isolating sink
failures. The first two stages run in the native staging engine
(``csrc/stager.cu``): the D2H is a real ``cudaMemcpyAsync`` (or SM
mapped-store kernel) fenced by CUDA events, so ``transfer_time`` is a
measured duration rather than the reference's modelled one.

``start()`` runs the same stages continuously on native threads (drain +
page-out, no GIL) with a Python sink thread on the bounded hand-off queue,
the shape of the reference's ``run_threaded`` (wallclock.py:136-181).
"""

from __future__ import annotations

import ctypes as C
import threading
from collections import deque
import time
from dataclasses import dataclass, field

from . import _native as N
from .errors import ConfigError, MetaMismatch
from .hooks import DeviceCopyEngine
from .records import CaptureRecord, TensorMeta, TensorMetaFIFO
from .rings import Descriptor, RingPair

STAGE_QUEUE_SLOTS = 16
STAGING_MODES = {"copy-engine": N.TF_STAGE_COPY_ENGINE,
                 "mapped": N.TF_STAGE_MAPPED}


EVENT_LOG_MAX = 1 << 16


@dataclass(frozen=True)
class DrainConfig:
    """Drain thresholds and staging pool sizing (exporter.py:35-51)."""

    min_ready_entries: int = 8
    min_ready_bytes: int = 1 << 20
    max_wait: float = 2e-3
    staging_buffer_size: int = 8 << 20
    staging_buffer_count: int = 4
    mode: str = "copy-engine"
    mapped_ctas: int = 0
    numa_node: int = -1
    stage_threads: int = 0
    stage_queue_slots: int = STAGE_QUEUE_SLOTS
    # page-out stage: "copy" = pinned -> pageable then the buffer returns
    # (the reference's stage_to_pageable); "handoff" = zero-copy, the sink
    # reads the pinned buffer, which returns when the batch is sunk;
    # "discard" = D2H-only measurement
    page_out: str = "copy"
    discard_paged: bool = False   # alias for page_out="discard"
    # extension: a capture larger than one staging buffer is staged in
    # buffer-sized chunks through several pool buffers (default False keeps
    # the reference's ConfigError, exporter.py:197-202)
    split_oversize: bool = False

    @property
    def page_out_mode(self) -> str:
        return "discard" if self.discard_paged else self.page_out

    def __post_init__(self) -> None:
        if self.page_out not in N.TF_PAGE_OUT:
            raise ConfigError(f"unknown page-out mode {self.page_out!r}")
        if min(self.min_ready_entries, self.min_ready_bytes) <= 0:
            raise ConfigError("ready thresholds must be positive")
        if self.max_wait <= 0:
            raise ConfigError("max_wait must be positive")
        if self.staging_buffer_size <= 0 or self.staging_buffer_count <= 0:
            raise ConfigError("staging pool sizing must be positive")
        if self.mode not in STAGING_MODES:
            raise ConfigError(f"unknown staging mode {self.mode!r}")

    def to_c(self) -> N.CDrainConfig:
        return N.CDrainConfig(
            self.min_ready_entries, self.min_ready_bytes, self.max_wait,
            self.staging_buffer_size, self.staging_buffer_count,
            STAGING_MODES[self.mode], self.mapped_ctas, self.numa_node,
            self.stage_queue_slots, self.stage_threads,
            N.TF_PAGE_OUT[self.page_out_mode], int(self.split_oversize))


class StagingBuffer:
    """A checked-out pinned buffer and the descriptors batched into it."""

    def __init__(self, pipe: "ExportPipeline", index: int, batch_id: int,
                 used: int, entries: list) -> None:
        self._pipe, self.index, self._batch_id = pipe, index, batch_id
        self.used = used
        self.entries = entries

    @property
    def data(self) -> memoryview:
        """Pinned bytes of this batch (waits for the D2H to land)."""
        ptr = C.c_void_p()
        N.check(N.lib().tf_stager_batch_buffer(self._pipe._st, self._batch_id,
                                               C.byref(ptr)))
        size = self._pipe.config.staging_buffer_size
        return memoryview((C.c_char * size).from_address(ptr.value)).cast("B")


class StagingPool:
    """Read-only view of the native pinned pool."""

    def __init__(self, pipe: "ExportPipeline") -> None:
        self._pipe = pipe
        self.buffer_size = pipe.config.staging_buffer_size
        self.total = pipe.config.staging_buffer_count

    def _stats(self) -> N.CStagerStats:
        return self._pipe._stats()

    @property
    def available(self) -> int:
        return self._stats().pool_free

    @property
    def checkouts(self) -> int:
        return self._stats().pool_checkouts

    @property
    def max_in_use(self) -> int:
        return self._stats().pool_max_in_use


@dataclass(frozen=True)
class DrainBatch:
    """One staged batch (exporter.py:98-110)."""

    buffer: StagingBuffer | None
    entries: tuple
    bytes_total: int
    reason: str
    batch_id: int = 0
    _pipe: object = field(default=None, repr=False, compare=False)

    @property
    def empty(self) -> bool:
        return not self.entries

    @property
    def transfer_time(self) -> float:
        """Measured D2H duration in seconds (waits for the copy)."""
        if self.empty:
            return 0.0
        secs = C.c_double()
        N.check(N.lib().tf_stager_transfer_seconds(
            self._pipe._st, self.batch_id, C.byref(secs)))
        return secs.value


@dataclass(frozen=True)
class DrainEvent:
    time: float
    kind: str           # drained | staged | sunk | sink-error
    reason: str = ""
    entries: int = 0
    bytes: int = 0


@dataclass
class PageableBatch:
    items: list = field(default_factory=list)   # (Descriptor, payload)
    reason: str = ""
    _release: object = field(default=None, repr=False)


class ExportPipeline:
    """Consumer side of one ring: native drain/stage, Python reconstruct/sink."""

    def __init__(self, ring: RingPair, config: DrainConfig | None = None,
                 engine: DeviceCopyEngine | None = None,
                 fifo: TensorMetaFIFO | None = None,
                 hook_name_of=None, copy_payloads: bool = True) -> None:
        # copy_payloads=False hands sinks read-only views of the pageable
        # batch (valid only during sink.write): for sinks that consume the
        # bytes immediately (FileSink, NullSink, StreamSink).
        self.copy_payloads = copy_payloads
        self.ring = ring
        self.config = config or DrainConfig()
        self.engine = engine or DeviceCopyEngine()
        self.fifo = fifo if fifo is not None else TensorMetaFIFO()
        self._hook_name_of = hook_name_of or (lambda hook_id: str(hook_id))
        cfg = self.config.to_c()
        st = C.c_void_p()
        N.check(N.lib().tf_stager_create(ring.handle, C.byref(cfg), C.byref(st)))
        self._st = st
        self.pool = StagingPool(self)
        # the event log (exporter.py:98-121) is bounded: a serving process
        # sinks batches for hours
        self.events: deque = deque(maxlen=EVENT_LOG_MAX)
        self.pageable_bytes_in_flight = 0
        self.max_transient_bytes = 0
        self.batches_drained = 0
        self.batches_sunk = 0
        self.records_out = 0
        self.bytes_out = 0
        self.sink_failures = 0
        self._lock = threading.Lock()
        self._sink_thread: threading.Thread | None = None
        self._sink = None
        self._stop = threading.Event()
        self._bg_error: BaseException | None = None
        self._sunk_batches_bg = 0

    # -- lifecycle -----------------------------------------------------------

    def close(self) -> None:
        if getattr(self, "_st", None) is not None:
            if self.running:
                self.stop(flush=False)
            N.lib().tf_stager_destroy(self._st)
            self._st = None

    def __del__(self) -> None:  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def _stats(self) -> N.CStagerStats:
        s = N.CStagerStats()
        N.check(N.lib().tf_stager_stats_get(self._st, C.byref(s)))
        return s

    def stats(self) -> dict:
        s = self._stats()
        return {name: getattr(s, name) for name, _ in N.CStagerStats._fields_}

    # -- thresholds ------------------------------------------------------------

    def note_publish(self, now: float) -> None:
        N.check(N.lib().tf_stager_note_publish(self._st, now))

    def thresholds_met(self, now: float) -> str | None:
        r = C.c_uint32()
        N.check(N.lib().tf_stager_thresholds_met(self._st, now, C.byref(r)))
        return None if r.value == 0 else N.REASONS[r.value]

    # -- stage 1: drain ------------------------------------------------------

    def drain_once(self, now: float = 0.0, flush: bool = False) -> DrainBatch:
        info = N.CBatchInfo()
        N.check(N.lib().tf_stager_drain_once(self._st, now, 1 if flush else 0,
                                             C.byref(info)))
        if info.n_entries == 0:
            reason = "flush" if flush else (self.thresholds_met(now) or "none")
            return DrainBatch(None, (), 0, reason, 0, self)
        n = info.n_entries
        descs = (N.CDescriptor * n)()
        starts = (C.c_uint64 * n)()
        N.check(N.lib().tf_stager_batch_entries(self._st, info.batch_id, descs,
                                                starts, n))
        entries = tuple((Descriptor.from_c(descs[i]), starts[i])
                        for i in range(n))
        reason = N.REASONS[info.reason]
        buf = StagingBuffer(self, info.buffer_index, info.batch_id,
                            info.bytes_total, list(entries))
        self.batches_drained += 1
        self.events.append(DrainEvent(now, "drained", reason, n,
                                      info.bytes_total))
        return DrainBatch(buf, entries, info.bytes_total, reason,
                          info.batch_id, self)

    def complete_transfer(self, batch: DrainBatch) -> None:
        """Wait for the D2H, then release the payload regions in order."""
        if batch.empty:
            return
        N.check(N.lib().tf_stager_complete_transfer(self._st, batch.batch_id,
                                                    None))

    # -- stage 2: pinned -> pageable ----------------------------------------

    def stage_to_pageable(self, batch: DrainBatch, now: float = 0.0) -> PageableBatch:
        out = PageableBatch(reason=batch.reason)
        if batch.empty:
            return out
        dst = bytearray(batch.bytes_total)
        addr = C.addressof((C.c_char * max(1, len(dst))).from_buffer(dst)) \
            if dst else None
        N.check(N.lib().tf_stager_stage_to_pageable(
            self._st, batch.batch_id, addr, len(dst)))
        view = memoryview(dst)
        for desc, start in batch.entries:
            out.items.append((desc, view[start:start + desc.payload_len],
                              addr + start if addr else None))
        self.pageable_bytes_in_flight += batch.bytes_total
        self._note_transient()
        self.events.append(DrainEvent(now, "staged", batch.reason,
                                      len(batch.entries), batch.bytes_total))
        return out

    def _note_transient(self) -> None:
        pool = self.pool
        pinned = (pool.total - pool.available) * pool.buffer_size
        self.max_transient_bytes = max(self.max_transient_bytes,
                                       pinned + self.pageable_bytes_in_flight)

    # -- stage 3: reconstruct + sink -------------------------------------------

    def reconstruct(self, desc: Descriptor, payload) -> list[CaptureRecord]:
        meta = self.fifo.match(desc, self._hook_name_of(desc.hook_id))
        return split_payload(meta, payload, copy=self.copy_payloads)

    def _sink_captures(self, batch: PageableBatch, sink, now: float) -> int:
        """Fast path for sinks with ``write_captures``: match every payload
        to its FIFO entry (MetaMismatch stays fatal) and hand the whole
        batch over at once; no per-record Python objects. Returns bytes."""
        caps = []
        total = recs = 0
        for item in batch.items:
            desc, payload = item[0], item[1]
            addr = item[2] if len(item) > 2 else None
            meta = self.fifo.match(desc, self._hook_name_of(desc.hook_id))
            n = len(payload)
            if n != meta.expected_payload_len:  # split_payload's check
                raise MetaMismatch(
                    f"payload {n} bytes != expected {meta.expected_payload_len}")
            caps.append((meta, payload, addr))
            total += n
            recs += len(meta.request_ids)
        try:
            sink.write_captures(caps)
        except Exception as exc:  # sink faults are isolated (exporter.py:266-271)
            self.sink_failures += 1
            self.events.append(DrainEvent(now, "sink-error", str(exc), recs, total))
        else:
            self.records_out += recs
            self.bytes_out += total
        self.pageable_bytes_in_flight -= total
        return total

    @staticmethod
    def _wants_captures(sink) -> bool:
        """Whole-batch fast path only when the sink's ``write_captures`` is
        at least as specific as its ``write`` (a subclass that overrides
        ``write`` alone, e.g. a collecting NullSink, keeps the records
        path)."""
        wc = getattr(sink, "write_captures", None)
        if wc is None:
            return False
        mro = type(sink).__mro__
        def owner(name):
            return next((c for c in mro if name in c.__dict__), None)
        w_owner, c_owner = owner("write"), owner("write_captures")
        if c_owner is None:  # instance attribute
            return True
        return w_owner is None or issubclass(c_owner, w_owner)

    def sink_batch(self, batch: PageableBatch, sink, now: float = 0.0) -> None:
        total = 0
        if self._wants_captures(sink):
            total = self._sink_captures(batch, sink, now)
            self.batches_sunk += 1
            self.events.append(DrainEvent(now, "sunk", batch.reason,
                                          len(batch.items), total))
            if batch._release is not None:
                batch._release()
            return
        for desc, payload, *_ in batch.items:
            n = len(payload)
            total += n
            records = self.reconstruct(desc, payload)
            try:
                sink.write(records)
            except Exception as exc:  # sink faults are isolated (exporter.py:266-271)
                self.sink_failures += 1
                self.events.append(DrainEvent(now, "sink-error", str(exc),
                                              len(records), n))
            else:
                self.records_out += len(records)
                self.bytes_out += n
            self.pageable_bytes_in_flight -= n
        self.batches_sunk += 1
        self.events.append(DrainEvent(now, "sunk", batch.reason,
                                      len(batch.items), total))
        if batch._release is not None:
            batch._release()

    # -- synchronous flush -------------------------------------------------------

    def flush_sync(self, sink, now: float = 0.0) -> float:
        """Drain everything now; returns the summed measured D2H time."""
        total = 0.0
        while self.ring.ready_entries() > 0:
            batch = self.drain_once(now, flush=True)
            if batch.empty:
                break
            total += batch.transfer_time
            self.complete_transfer(batch)
            self.sink_batch(self.stage_to_pageable(batch, now), sink, now)
        self.ring.sync()
        if self.ring.occupancy != 0 and self.ring.ready_entries() == 0:
            from .errors import ProtocolError
            raise ProtocolError("flush with unpublished reservations in flight")
        return total

    # -- background engine -------------------------------------------------------

    @property
    def running(self) -> bool:
        return self._sink_thread is not None

    def start(self, sink) -> None:
        """Run drain + page-out natively and sink on a Python thread."""
        if self.running:
            return
        self._sink = sink
        self._stop.clear()
        self._bg_error = None
        N.check(N.lib().tf_stager_start(self._st))
        self._sink_thread = threading.Thread(target=self._sink_loop,
                                             name="ring2-sink", daemon=True)
        self._sink_thread.start()

    def _sink_loop(self) -> None:
        lib = N.lib()
        while True:
            pb = N.CPagedBatch()
            rc = lib.tf_stager_next(self._st, 0.05, C.byref(pb))
            if rc in (N.TF_ERR_EMPTY, N.TF_ERR_TIMEOUT):
                if self._stop.is_set():
                    return
                continue
            if rc != N.TF_OK:
                self._bg_error = N.exception_for(
                    rc, lib.tf_last_error().decode(errors="replace"))
                return
            try:
                self._sink_paged(pb)
            except BaseException as exc:  # MetaMismatch is fatal
                self._bg_error = exc
                lib.tf_stager_free_paged(self._st, C.byref(pb))
                return

    def _sink_paged(self, pb: N.CPagedBatch) -> None:
        lib = N.lib()
        n = pb.n_entries
        raw = (C.c_char * max(1, pb.bytes_total)).from_address(pb.payload)
        view = memoryview(raw).cast("B")
        if n and self._wants_captures(self._sink):
            # a raise (MetaMismatch) leaves the batch to _sink_loop to free
            self._sink_paged_captures(pb, n, view)
            del view
            lib.tf_stager_free_paged(self._st, C.byref(pb))
            return
        batch = PageableBatch(reason=N.REASONS.get(pb.reason, "none"))
        for i in range(n):
            d = Descriptor.from_c(pb.descs[i])
            s = pb.starts[i]
            batch.items.append((d, view[s:s + d.payload_len], pb.payload + s))
        with self._lock:
            self.pageable_bytes_in_flight += pb.bytes_total
            self.sink_batch(batch, self._sink, time.monotonic())
            self._sunk_batches_bg += 1
        del batch, view
        lib.tf_stager_free_paged(self._st, C.byref(pb))

    def _sink_paged_captures(self, pb, n: int, view) -> None:
        """Background fast path for batch sinks: the batch's descriptors are
        read as columns in one step and matched against the metadata FIFO
        without per-descriptor Python objects (the sink thread shares the
        GIL with the inference engine)."""
        import numpy as np
        cols = np.ctypeslib.as_array(pb.descs, shape=(n,))
        hooks = cols["hook_id"].tolist()
        steps = cols["step_seq"].tolist()
        lens = cols["payload_len"].tolist()
        starts = np.ctypeslib.as_array(pb.starts, shape=(n,)).tolist()
        base = pb.payload
        name_of = self._hook_name_of
        match = self.fifo.match_raw
        caps = []
        total = recs = 0
        for i in range(n):
            ln = lens[i]
            meta = match(steps[i], name_of(hooks[i]), ln)
            st = starts[i]
            caps.append((meta, view[st:st + ln], base + st))
            total += ln
            recs += len(meta.request_ids)
        now = time.monotonic()
        with self._lock:
            try:
                self._sink.write_captures(caps)
            except Exception as exc:  # sink faults are isolated (exporter.py:266-271)
                self.sink_failures += 1
                self.events.append(DrainEvent(now, "sink-error", str(exc), recs, total))
            else:
                self.records_out += recs
                self.bytes_out += total
            self.batches_sunk += 1
            self.events.append(DrainEvent(now, "sunk", N.REASONS.get(pb.reason, "none"),
                                          n, total))
            self._sunk_batches_bg += 1
        del caps

    def stream_handle(self) -> int:
        """cudaStream_t of the staging D2H work (for cross-stream events)."""
        p = C.c_void_p()
        N.check(N.lib().tf_stager_stream(self._st, C.byref(p)))
        return int(p.value or 0)

    def placement(self) -> dict:
        """CPUs the staging threads are bound to and the NUMA node of the
        pinned pool (replica placement)."""
        cpus = (C.c_int32 * 1024)()
        n, node = C.c_uint32(), C.c_int32()
        N.check(N.lib().tf_stager_placement(self._st, cpus, 1024, C.byref(n), C.byref(node)))
        return {"cpus": list(cpus[:min(n.value, 1024)]), "pool_numa_node": node.value}

    def _check_bg(self) -> None:
        if self._bg_error is not None:
            raise self._bg_error
        rc = N.lib().tf_stager_error(self._st)
        if rc:
            N.check(rc)

    def flush(self, timeout: float = 60.0) -> None:
        """Block until every published capture has been drained and sunk."""
        self._check_bg()
        N.check(N.lib().tf_stager_flush(self._st, timeout))
        if self.config.page_out_mode == "discard":
            return
        deadline = time.monotonic() + timeout
        while True:
            self._check_bg()
            staged = self._stats().batches_staged
            if self._sunk_batches_bg >= staged:
                return
            if time.monotonic() > deadline:
                raise N.exception_for(N.TF_ERR_TIMEOUT, "sink did not catch up")
            time.sleep(0.0005)

    def stop(self, flush: bool = True, timeout: float = 60.0) -> None:
        if not self.running:
            return
        try:
            if flush:
                self.flush(timeout)
        finally:
            rc = N.lib().tf_stager_stop(self._st)
            self._stop.set()
            self._sink_thread.join(timeout)
            self._sink_thread = None
        self._check_bg()
        if rc:
            N.check(rc)


def split_payload(meta: TensorMeta, payload, copy: bool = True) -> list[CaptureRecord]:
    """Per-request records of one capture payload, batch order kept."""
    if not copy:
        payload = memoryview(payload).toreadonly()
    if len(payload) != meta.expected_payload_len:
        raise MetaMismatch(
            f"payload {len(payload)} bytes != expected "
            f"{meta.expected_payload_len}")
    sizes = meta.request_bytes()
    out = []
    pos = 0
    for i, (rid, trange) in enumerate(zip(meta.request_ids, meta.token_ranges)):
        size = sizes[i]
        shape = meta.shape if meta.row_counts is None else \
            (meta.row_counts[i],) + tuple(meta.shape[1:])
        out.append(CaptureRecord(
            request_id=rid, hook_name=meta.hook_name,
            layer_index=meta.layer_index, step_seq=meta.step_seq,
            token_range=trange, shape=shape, dtype=meta.dtype,
            rank_coords=meta.rank_coords,
            payload=bytes(payload[pos:pos + size]) if copy
            else payload[pos:pos + size]))
        pos += size
    return out
