"""HookPoint and the per-device observation session (``Observer``).

``HookPoint`` is the paper's instrumentation primitive (§3.1): an
``nn.Module`` placed at an observation site whose forward is the identity
plus a capture launch — no host synchronisation, no Python callback on the
device timeline, legal inside CUDA-graph capture because the keep vector
and the step sequence live in fixed device buffers that are rewritten
between steps (§3.4 "index vector ... compatible with CUDA Graph
replay").

``Observer`` owns one ring pair, its export pipeline, the metadata FIFO and
those device buffers, and implements the reference's per-step protocol
(simulator.py:400-421 / wallclock.py:94-134):

    plan = obs.begin_step(batch, step_seq)   # prepare_step, flush gate,
                                             # FIFO entries, keep upload
    model(...)                               # HookPoints launch captures
    obs.end_step()                           # fence for the next snapshot

Capture behaviour on a full ring follows the policy: completeness waits on
the device for the consumer (the reference's in-step stall), best-effort
drops and flags ``PolicyUnderestimate`` (which the plan makes impossible).

Token-row sampling (north-star extension) keeps a per-token subset: a hook
with ``sample=True`` captures rows (request, token) selected by the
observer's ``TokenSampler``; its records carry ``row_counts`` and
``token_indices``.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

from . import _native as N
from ._device import torch
from .errors import ConfigError, PolicyUnderestimate
from .exporter import DrainConfig, ExportPipeline
from .hooks import HookRegistry, RowSource, capture_args, launch_capture
from .policy import COMPLETENESS, PolicyConfig, StepPlan, prepare_step
from .records import StepMetas, TensorMeta, TensorMetaFIFO
from .rings import RingConfig, RingPair

nn = torch().nn


@dataclass(frozen=True)
class TokenSampler:
    """Which tokens of a request to keep: every ``every``-th, or a seeded
    Bernoulli(``rate``) draw per (request, step)."""

    every: int | None = None
    rate: float | None = None
    seed: int = 0

    def __post_init__(self) -> None:
        if (self.every is None) == (self.rate is None):
            raise ConfigError("token sampler needs exactly one of every/rate")

    def select(self, request_id: int, step_seq: int, tokens: int) -> list[int]:
        if self.every is not None:
            return list(range(0, tokens, self.every))
        import random
        rng = random.Random((self.seed << 40) ^ (request_id << 20) ^ step_seq)
        return [t for t in range(tokens) if rng.random() < self.rate]


class Observer:
    """One device's capture session: ring, exporter, policy, keep buffers."""

    def __init__(self, registry: HookRegistry, *, ring: RingConfig,
                 drain: DrainConfig | None = None,
                 policy: PolicyConfig | None = None, sink=None,
                 device: int | None = None, max_batch: int = 1024,
                 max_tokens: int = 8192, max_rows_sampled: int = 1 << 22,
                 sampler: TokenSampler | None = None,
                 sampled_hooks: frozenset = frozenset(),
                 rank_coords: tuple = (0, 0), wait_timeout: float = 60.0,
                 flat_rows: int = 0, persistent: bool = False,
                 debug_row_bytes: dict | None = None, overlap: bool = False,
                 overlap_max_bytes: int | None = None,
                 sealed: bool = True):
        t = torch()
        self.registry = registry
        self.policy = policy or PolicyConfig()
        self.ring = RingPair(ring, device=device, wait_timeout=wait_timeout)
        self.device = self.ring.device
        self.fifo = TensorMetaFIFO()
        self.exporter = ExportPipeline(
            self.ring, drain or DrainConfig(), None, self.fifo,
            hook_name_of=lambda h: registry.hook(h).name)
        self.sink = sink
        self.sampler = sampler
        self.sampled_hooks = frozenset(sampled_hooks)
        self.rank_coords = rank_coords
        dev = f"cuda:{self.device}"
        # a persistent observer keeps nothing until its first begin_step
        self.keep_req = (t.zeros if persistent else t.ones)(max_batch, dtype=t.uint8,
                                                            device=dev)
        # per-token keep for sampled hooks, expanded over each hook's row
        # groups: a (heads, tokens, tokens) attention map has `heads` query
        # rows per token; fixed buffers so CUDA-graph replays see updates
        self._groups = {h: _row_groups(registry.hook(h), registry.hidden_extent)
                        for h in self.sampled_hooks}
        self._keep_m = {}
        for m in sorted(set(self._groups.values())):
            n = min(max_rows_sampled, max_batch * m * max_tokens)
            self._keep_m[m] = t.zeros(max(1, n), dtype=t.uint8, device=dev)
        self.keep_tok = self._keep_m.get(1)
        self._flat = {}
        self._flat_rows = max(flat_rows, max_batch * 64)
        # serving engines record HookPoints into their CUDA graphs once, so
        # captures stay armed between steps (persistent=True) and the keep
        # buffers are allocated up front at their final size (flat_rows):
        # a replay reads whatever keep vector the last begin_step uploaded
        self.persistent = persistent
        self._pinned = {}
        self._layout = "batch"
        if flat_rows:
            self._flat_buf("req", flat_rows)
            if self.sampled_hooks:
                self._flat_buf("tok", flat_rows)
            # engines that run (tokens, ...) activations: forwards before the
            # first begin_step (profiling, graph capture) see all-zero keeps
            self._layout = "flat"
        self.step_buf = t.zeros(1, dtype=t.int32, device=dev)
        # debug (parity checks of CUDA-graph engines): every capture also
        # copies the whole observed tensor into a fixed per-hook buffer, so
        # the copy is recorded into the same graphs as the capture kernel
        # and a replay leaves the rows the capture read for comparison
        self.debug_clone = {}
        for name, row_bytes in (debug_row_bytes or {}).items():
            hid = [h.name for h in registry.hooks].index(name)
            self.debug_clone[hid] = t.zeros(self._flat_rows * row_bytes, dtype=t.uint8,
                                            device=dev)
        self.token = t.zeros(1, dtype=t.uint8, device=dev)  # custom-op ordering token
        self.index = _register_observer(self)
        self._sc = (None, 0.0, 0, 0)  # policy snapshot, time, bytes planned since, max capture
        self.max_batch = max_batch
        self._names = {h.name: i for i, h in enumerate(registry.hooks)}
        self._plan: StepPlan | None = None
        self._batch = []
        self._tok_sel: dict[int, list[int]] = {}
        # persistent: armed from the start, so HookPoints are recorded into
        # CUDA graphs captured before the first step (keep vector all zero)
        self.active = persistent
        self.launches = 0
        self.steps = 0
        # Admission gate of eager captures under completeness (see _admit):
        # reserved bytes launched so far, released bytes last seen, the
        # largest reservation (dead-skip slack), this step's expected
        # reservation per hook, and whether a CUDA graph is being recorded
        self.wait_timeout = wait_timeout
        self._launched = 0
        self._released = 0
        self._max_need = 0
        self._need: dict[str, list[int]] = {}
        self._recording = False
        self.gate_waits = 0
        self.gate_wait_s = 0.0
        # overlap=True: capture kernels run on a side stream forked from the
        # producer stream at each HookPoint, so they overlap the model's next
        # kernels instead of sitting between them; join() (at end_step, or
        # an integration's join hook before an activation is mutated in
        # place) makes the producer stream wait for them. One side stream:
        # the captures stay serialised among themselves, as the producer
        # snapshot protocol requires.
        self.overlap = overlap
        # overlap_max_bytes: fork only captures whose source is at most this
        # large (decode-size captures overlap well; large ones compete with
        # the model for SMs); larger ones run inline after a join
        self.overlap_max_bytes = overlap_max_bytes
        self.side_stream = t.cuda.Stream(device=dev) if overlap else None
        self._forked = False
        # sealed=True: captures carry TF_CAP_SEALED (no per-CTA fence and
        # completion bytes; completion follows from stream order) and
        # end_step / flush / stop seal the ring on the producer stream
        self.sealed = sealed

    # -- session -----------------------------------------------------------

    def start(self) -> "Observer":
        if self.sink is not None and not self.exporter.running:
            self.exporter.start(self.sink)
        return self

    def stop(self, flush: bool = True) -> None:
        self.join()
        self._seal()
        if self.exporter.running:
            self.exporter.stop(flush=flush)

    def close(self) -> None:
        self.stop()
        self.exporter.close()
        self.ring.close()

    def flush(self, timeout: float = 120.0) -> None:
        self.join()
        self._seal()
        if self.side_stream is not None:
            self.side_stream.synchronize()  # every side-stream capture has published
        self.ring.sync()
        self.exporter.flush(timeout)

    def _seal(self, stream=None) -> None:
        if self.sealed and getattr(self.ring, "_h", None) is not None:
            self.ring.seal(stream)

    def join(self, stream=None) -> None:
        """Make the producer stream wait for the side-stream captures
        launched since the last join (overlap mode; a no-op otherwise).
        Must run before a captured activation is modified in place, and
        inside a CUDA-graph capture before the capture ends."""
        if not self._forked:
            return
        t = torch()
        cur = stream if stream is not None else t.cuda.current_stream(self.device)
        cur.wait_stream(self.side_stream)
        self._forked = False

    # -- per step --------------------------------------------------------------

    def begin_step(self, batch, step_seq: int, stream=None,
                   layout: str = "batch", rows_total: int | None = None) -> StepPlan:
        """Plan the step, honour the flush gate, queue metadata, upload keep.

        ``layout="batch"``: activations are (B, T, ...) with uniform T
        (the reference's model). ``layout="flat"``: continuous batching —
        activations are (sum of tokens, ...) in batch order and requests may
        carry different token counts (prefill chunks beside decodes);
        ``rows_total`` is the padded row count the engine runs (CUDA-graph
        batch sizes), whose padding rows are never kept.
        """
        t = torch()
        batch = list(batch)
        if len(batch) > self.max_batch:
            raise ConfigError("batch exceeds the observer's max_batch")
        if layout not in ("batch", "flat"):
            raise ConfigError(f"unknown activation layout {layout!r}")
        flat = layout == "flat"
        if flat and self.persistent:
            # fail before any state changes (FIFO, plan) if the recorded
            # graphs' keep buffers cannot hold this step's rows
            rows = max(sum(r.tokens for r in batch), rows_total or 0)
            for kind in ("req", "tok"):
                buf = self._flat.get(kind)
                if buf is not None and buf.numel() < rows:
                    self._flat_buf(kind, rows)   # raises ConfigError
        self.registry.commit_filter()
        if not batch:  # engine warm-up / dummy forwards: nothing to keep
            plan = StepPlan(keep=(), flush_before=False, fifo_entries=(), kept_ids=(),
                            dropped_ids=(), free_bytes_at_plan=0)
        else:
            plan = prepare_step(self.policy, batch, self._policy_ring(), self.registry,
                                step_seq=step_seq, rank_coords=self.rank_coords,
                                ragged=flat)
            if self.policy.mode == COMPLETENESS:
                st, t0, since, big = self._sc
                fe = plan.fifo_entries
                lens = fe.payload_lens() if isinstance(fe, StepMetas) else \
                    [m.expected_payload_len for m in fe]
                if lens:
                    since += sum(lens) + 16 * len(lens)
                    big = max(big, max(lens))
                self._sc = (st, t0, since, big)
        if plan.flush_before:
            self.flush()
        metas = plan.fifo_entries
        sel = {}
        kept_set = set(plan.kept_ids)
        if self.sampler is not None and plan.kept_ids and self.sampled_hooks:
            kept = [r for r in batch if r.request_id in kept_set]
            for r in kept:
                sel[r.request_id] = self.sampler.select(r.request_id, step_seq,
                                                        r.tokens)
            groups = {self.registry.hook(h).name: g
                      for h, g in self._groups.items()}
            metas = [self._sampled_meta(m, kept, sel, groups[m.hook_name])
                     if m.hook_name in groups else m
                     for m in metas]
        self.fifo.extend(metas)
        self._need = {}
        if self.policy.mode == COMPLETENESS and not self.persistent and metas:
            lens = metas.payload_lens() if isinstance(metas, StepMetas) else \
                [m.expected_payload_len for m in metas]
            names = [e[0] for e in metas.entries] if isinstance(metas, StepMetas) else \
                [m.hook_name for m in metas]
            for name, n in zip(names, lens):
                self._need.setdefault(name, []).append((n + 15) & ~15)
            for q in self._need.values():
                q.reverse()  # popped from the end, in firing order
        s = stream if stream is not None else t.cuda.current_stream(self.device)
        with t.cuda.stream(s):
            busy = self._pinned.get("_busy")
            if busy is not None:  # the previous step's uploads have left
                busy.synchronize()
            step = self._pinned.get("step")
            if step is None:
                step = t.zeros(1, dtype=t.int32).pin_memory()
                self._pinned["step"] = step
            step[0] = step_seq & 0x7FFFFFFF
            self.step_buf.copy_(step, non_blocking=True)
            if flat:
                # per-row keep over the flat token layout (padding rows 0)
                rows = max(sum(r.tokens for r in batch), rows_total or 0)
                flags = self._host_rows("req", max(1, rows))
                samp = self._host_rows("tok", max(1, rows)) if sel else None
                import numpy as np
                ntok = np.fromiter((r.tokens for r in batch), dtype=np.int64,
                                   count=len(batch))
                kmask = np.fromiter((r.request_id in kept_set for r in batch),
                                    dtype=np.uint8, count=len(batch))
                fl = np.repeat(kmask, ntok)
                flags.numpy()[:fl.size] = fl
                if sel:
                    pos = 0
                    for r in batch:
                        for tok in sel.get(r.request_id, ()):
                            samp[pos + tok] = 1
                        pos += r.tokens
                self._upload_pinned(self._flat_buf("req", rows), flags)
                if sel:
                    self._upload_pinned(self._flat_buf("tok", rows), samp)
            else:
                keep = t.tensor(list(plan.keep) or [0], dtype=t.uint8)
                self._upload(self.keep_req, keep)
                if sel:
                    tokens = batch[0].tokens
                    flags = t.zeros(len(batch), 1, tokens, dtype=t.uint8)
                    for i, r in enumerate(batch):
                        for tok in sel.get(r.request_id, ()):
                            flags[i, 0, tok] = 1
                    for m, buf in self._keep_m.items():
                        self._upload(buf, flags.expand(len(batch), m, tokens).reshape(-1))
            ev = self._pinned.get("_ev")
            if ev is None:
                ev = t.cuda.Event()
                self._pinned["_ev"] = ev
            ev.record(s)
            self._pinned["_busy"] = ev
        self._plan, self._batch, self._tok_sel = plan, batch, sel
        self._layout = layout
        self.active = bool(plan.kept_ids) or self.persistent
        self.steps += 1
        return plan

    def _host_rows(self, kind: str, rows: int):
        """Zeroed view of a reusable pinned host buffer (flat keep flags);
        begin_step waits for the previous upload from it before reuse."""
        t = torch()
        busy = self._pinned.get("_busy")
        if busy is not None:  # the previous step's upload has left the buffer
            busy.synchronize()
        buf = self._pinned.get(kind)
        if buf is None or buf.numel() < rows:
            buf = t.zeros(max(rows, self._flat_rows), dtype=t.uint8).pin_memory()
            self._pinned[kind] = buf
        v = buf[:rows]
        v.zero_()
        return v

    @staticmethod
    def _upload_pinned(dst, src) -> None:
        if src.numel() > dst.numel():
            raise ConfigError("keep vector exceeds its device buffer")
        dst[:src.numel()].copy_(src, non_blocking=True)

    def _policy_ring(self):
        """The ring as the planner sees it. Completeness only needs to know
        whether occupancy crossed the flush watermark, and occupancy cannot
        grow faster than the bytes this host has planned since the last
        device snapshot, so that snapshot is reused while snapshot +
        planned bytes + slack (dead-skip waste) stays under the watermark:
        the decision is the one a fresh snapshot would give, without a
        device round trip per step. Best-effort replays the allocator
        (would_fit) and always reads the device."""
        if self.policy.mode != COMPLETENESS:
            return self.ring
        return _CompletenessRingView(self)

    def _snapshot_for_policy(self):
        st, t0, since, big = self._sc
        now = time.monotonic()
        if st is not None and now - t0 < 0.5:
            bound = st.occupancy + since + 2 * big + (1 << 16)
            if bound < self.policy.pressure_watermark * st.payload_capacity:
                return st
        st = self.ring.state()
        self._sc = (st, now, 0, big)
        return st

    @staticmethod
    def _upload(dst, src) -> None:
        if src.numel() > dst.numel():
            raise ConfigError("keep vector exceeds its device buffer")
        dst[:src.numel()].copy_(src.pin_memory(), non_blocking=True)

    def _flat_buf(self, kind: str, rows: int):
        """Fixed per-row keep buffers for the flat layout. A persistent
        observer's buffers are referenced by recorded CUDA graphs, so they
        are never moved: a step with more rows than ``flat_rows`` raises
        instead of reallocating (a replay would read the stale buffer)."""
        t = torch()
        buf = self._flat.get(kind)
        if buf is not None and buf.numel() < rows and self.persistent:
            raise ConfigError(
                f"step has {rows} token rows but the persistent observer's keep "
                f"buffers hold {buf.numel()} (raise flat_rows to the engine's "
                "maximum batched tokens)")
        if buf is None or buf.numel() < rows:
            n = max(rows, self._flat_rows)
            buf = t.zeros(n, dtype=t.uint8, device=f"cuda:{self.device}")
            self._flat[kind] = buf
        return buf

    def step_token_start(self) -> int:
        """Position of this step's first token in each sequence (batch
        layout: uniform across the batch, the reference's model)."""
        return self._batch[0].token_start if self._batch else 0

    def end_step(self, stream=None) -> None:
        if stream is None:  # resolved once (a torch call costs microseconds)
            stream = torch().cuda.current_stream(self.device)
        self.join(stream)
        self._seal(stream)
        self.ring.note_launch(stream)
        self.active = self.persistent

    def graph_capture(self):
        """Context manager for recording a CUDA graph of one step: enabled
        HookPoints record their capture kernels into the graph. Replay it
        between begin_step()/end_step(); the keep vector and step sequence
        are read from the observer's fixed device buffers at replay time.
        Re-record after a hook-filter change (disabled hooks must vanish
        from the graph, §3.4)."""
        obs = self

        class _Rec:
            def __enter__(self_inner):
                obs.registry.commit_filter()
                obs._was_active = obs.active
                obs.active = True
                obs._recording = True

            def __exit__(self_inner, *exc):
                obs.active = obs._was_active
                obs._recording = False
        return _Rec()

    def check_device(self) -> None:
        """Raise if the device dropped a capture the plan admitted."""
        st = self.ring.state()
        if st.device_errors & N.TF_DEVERR_UNDERESTIMATE:
            raise PolicyUnderestimate(
                f"{st.drops} capture(s) dropped on a full ring")
        if st.device_errors & N.TF_DEVERR_TIMEOUT:
            from .errors import DeviceError
            raise DeviceError("device wait for ring space timed out")
        if st.device_errors & N.TF_DEVERR_TOO_LARGE:
            raise ValueError("a capture exceeded the payload ring capacity "
                             "(rings.py:297-298)")

    def _sampled_meta(self, meta: TensorMeta, kept, sel, groups: int) -> TensorMeta:
        # rows of request i: `groups` x its kept tokens, in memory order
        # (group-major, e.g. head-major for attention maps)
        counts = tuple(groups * len(sel[r.request_id]) for r in kept)
        per_row_shape = tuple(meta.shape[-1:])
        return TensorMeta(
            hook_name=meta.hook_name, layer_index=meta.layer_index,
            step_seq=meta.step_seq, request_ids=meta.request_ids,
            token_ranges=meta.token_ranges,
            shape=(max(1, max(counts, default=1)),) + per_row_shape,
            dtype=meta.dtype, rank_coords=meta.rank_coords,
            row_counts=counts,
            token_indices=tuple(tuple(sel[r.request_id]) for r in kept))

    # -- capture (called by HookPoint) -------------------------------------

    def hook_id(self, name: str) -> int | None:
        return self._names.get(name)

    def capture(self, hook_id: int, x, stream=None) -> None:
        """Launch the capture of ``x`` (batch-major (B, T, ...)) for this step."""
        if not self.active or not self.registry.is_enabled(hook_id):
            return
        hook = self.registry.hook(hook_id)
        sampled = hook_id in self.sampled_hooks and bool(self._tok_sel)
        if self._layout == "flat":
            # (sum of tokens, ...): one row per token, per-row keep
            src = _token_rows(x)
            keep = self._flat["tok" if sampled else "req"]
            per_outer = False
        else:
            src = _rows_of(x, hook)
            keep = self._keep_m[self._groups[hook_id]] if sampled else self.keep_req
            per_outer = not sampled
        args = capture_args(
            src, hook_id=hook_id, hook=hook, keep_ptr=keep.data_ptr(),
            keep_per_outer=per_outer, step_seq_ptr=self.step_buf.data_ptr(),
            full=self.policy.full_mode, sealed=self.sealed)
        if self._need and not self._recording:
            q = self._need.get(hook.name)
            if q:
                self._admit(q.pop())
        fork = self.overlap and (self.overlap_max_bytes is None or
                                 src.outer * src.mid * src.row_bytes <= self.overlap_max_bytes)
        if self.overlap and not fork:
            # inline after the forked ones: captures stay serialised on the
            # ring (one producer order for snapshots and sealed completion)
            self.join(stream)
        if fork:
            t = torch()
            cur = stream if stream is not None else t.cuda.current_stream(self.device)
            side = self.side_stream
            side.wait_stream(cur)         # the source rows and keep uploads first
            launch_capture(self.ring, args, side)
            if isinstance(x, t.Tensor):
                x.record_stream(side)     # no reuse of the rows before the copy
            self._forked = True
        else:
            launch_capture(self.ring, args, stream)
        self.launches += 1
        dbg = self.debug_clone.get(hook_id)
        if dbg is not None:
            flat_x = x.contiguous().reshape(-1).view(torch().uint8)
            if flat_x.numel() > dbg.numel():
                raise ConfigError("debug clone buffer too small")
            dbg[:flat_x.numel()].copy_(flat_x)


    def _admit(self, need: int) -> None:
        """Admission gate for eager captures under completeness.

        A capture that finds the ring full waits on the device
        (TF_FULL_WAIT) with its whole grid resident. That is right inside a
        CUDA graph, where the host cannot pause a replay, but in eager code it
        lets any host call that waits for the device (a synchronising copy,
        cudaFree under allocator pressure, a pinned allocation) block while
        the device waits for the staging engine. So before launching, the
        host waits until the bytes launched and not yet released, plus this
        reservation, leave room for one dead skip (the largest reservation):
        the device then always finds space. The estimate uses the planned
        payload lengths and the consumer's host-side release total; if it
        stays blocked (the estimate drifted), it is re-based once on an
        exact device snapshot."""
        if need > self._max_need:
            self._max_need = need
        cap = self.ring.capacity
        limit = cap - self._max_need - need  # in flight allowed before this one

        def admitted() -> bool:
            before = self._launched - self._released
            return before <= 0 or before <= limit   # an empty ring fits anything

        if admitted():
            self._launched += need
            return
        import ctypes as C
        lib = N.lib()
        rel = C.c_uint64()
        t0 = time.monotonic()
        rebased = False
        # the last sealed capture completes only with a later post or a seal,
        # and nothing is launched while the host waits here
        self.join()
        self._seal()
        while True:
            N.check(lib.tf_ring_host_released(self.ring.handle, C.byref(rel), None))
            self._released = rel.value
            if admitted():
                break
            self.exporter._check_bg()
            waited = time.monotonic() - t0
            if waited > 0.25 and not rebased:
                # every launched capture has reserved once the producer
                # stream is synchronised: occupancy is then exact (dead
                # bytes count as in flight: conservative by at most a skip)
                torch().cuda.current_stream(self.device).synchronize()
                if self.side_stream is not None:
                    self.side_stream.synchronize()
                occ = self.ring.state().occupancy
                N.check(lib.tf_ring_host_released(self.ring.handle, C.byref(rel), None))
                self._released = rel.value
                self._launched = self._released + occ
                rebased = True
                continue
            if waited > self.wait_timeout:
                from .errors import PayloadRingFull
                raise PayloadRingFull(
                    f"capture of {need} bytes: the consumer released nothing for "
                    f"{waited:.0f} s (ring {cap} bytes)")
            time.sleep(2e-5)
        self._launched += need
        self.gate_waits += 1
        self.gate_wait_s += time.monotonic() - t0


class _CompletenessRingView:
    """RingPair proxy whose state() may return a recent snapshot (see
    Observer._policy_ring); everything else goes to the ring."""

    def __init__(self, obs: "Observer") -> None:
        self._obs = obs

    def state(self):
        return self._obs._snapshot_for_policy()

    def __getattr__(self, name):
        return getattr(self._obs.ring, name)


def _row_groups(hook, hidden: int) -> int:
    """Row groups per token of a sampled hook: rows per request divided by
    the token count, e.g. `heads` for a (heads, tokens, tokens) map."""
    lead = hook.dims[:-1]
    if lead.count("tokens") != 1:
        raise ConfigError(
            f"sampled hook {hook.name!r} needs exactly one leading tokens axis")
    m = 1
    for d in lead:
        if d == "hidden":
            m *= hidden
        elif not isinstance(d, str):
            m *= d
    return m


def _token_rows(x) -> RowSource:
    """A flat (tokens, ...) activation as one row per token."""
    if x.dim() < 1:
        raise ConfigError("flat activations need a token axis")
    x2 = x.reshape(x.shape[0], -1)
    if x2.stride(-1) != 1:
        x2 = x2.contiguous()
    esz = x2.element_size()
    row = x2.shape[1] * esz
    return RowSource(x2.data_ptr(), x2.shape[0], 1, row, x2.stride(0) * esz,
                     row, x2)


def _rows_of(x, hook) -> RowSource:
    """Describe a (B, T, ..., H) activation as strided rows (b, t)."""
    if x.dim() < 2:
        raise ConfigError("captured activations are batch-major (B, ...)")
    esz = x.element_size()
    if x.dim() == 2:
        x2 = x if x.stride(-1) == 1 else x.contiguous()
        return RowSource(x2.data_ptr(), x2.shape[0], 1, x2.shape[1] * esz,
                         x2.stride(0) * esz, x2.shape[1] * esz, x2)
    b = x.shape[0]
    row_elems = x.shape[-1]
    if x.stride(-1) == 1:
        # the rows of one request as one uniformly strided run, without a
        # copy: contiguous per request, or e.g. a KV-cache slice
        # (B, kv_heads, new_tokens, head_dim) of a larger cache whose
        # new_tokens is 1 (decode) or the whole cache (prefill)
        try:
            xv = x.view(b, -1, row_elems)
        except RuntimeError:
            xv = None
        if xv is not None and xv.stride(2) == 1:
            mid = xv.shape[1]
            s_mid = xv.stride(1) * esz if mid > 1 else row_elems * esz
            return RowSource(xv.data_ptr(), b, mid, row_elems * esz,
                             xv.stride(0) * esz, s_mid, x)
    x = x.contiguous()  # any other layout: one torch copy, then rows
    mid = x[0].numel() // row_elems
    return RowSource(x.data_ptr(), b, mid, row_elems * esz, x.stride(0) * esz,
                     row_elems * esz, x)


class HookPoint(nn.Module):
    """Identity module that captures its input into the observer's ring."""

    def __init__(self, name: str, observer: Observer | None = None) -> None:
        super().__init__()
        self.name = name
        self.observer = observer
        self._hid = observer.hook_id(name) if observer is not None else None

    def bind(self, observer: Observer) -> None:
        self.observer = observer
        self._hid = observer.hook_id(self.name)

    def forward(self, x):
        obs = self.observer
        if obs is None or self._hid is None:
            return x
        t = torch()
        if t.compiler.is_compiling():
            # traced as an opaque custom op (§3.1): the compiled
            # graph keeps the capture launch and checks obs.active at run time
            t.ops.ring2.capture(x, obs.token, obs.index, self._hid)
        elif obs.active:
            obs.capture(self._hid, x)
        return x


# ---------------------------------------------------------------------------
# the custom operator behind HookPoint under torch.compile
# ---------------------------------------------------------------------------
_OBSERVERS: list = []


def _register_observer(obs: Observer) -> int:
    import weakref
    _OBSERVERS.append(weakref.ref(obs))
    return len(_OBSERVERS) - 1


@torch().library.custom_op(
    "ring2::capture", mutates_args=("token",),
    schema="(Tensor x, Tensor(a!) token, int observer, int hook_id) -> ()")
def _capture_op(x, token, observer, hook_id):
    ref = _OBSERVERS[observer] if 0 <= observer < len(_OBSERVERS) else None
    obs = ref() if ref is not None else None
    if obs is not None and obs.active:
        obs.capture(hook_id, x)


@_capture_op.register_fake
def _capture_fake(x, token, observer, hook_id) -> None:
    return None


@torch().library.custom_op(
    "ring2::join", mutates_args=("token",),
    schema="(Tensor(a!) token, int observer) -> ()")
def _join_op(token, observer):
    ref = _OBSERVERS[observer] if 0 <= observer < len(_OBSERVERS) else None
    obs = ref() if ref is not None else None
    if obs is not None:
        obs.join()


@_join_op.register_fake
def _join_fake(token, observer) -> None:
    return None


def join_point(observer: Observer) -> None:
    """Call from model code (or a hook) where the overlap-mode captures must
    be complete: traced as the ``ring2::join`` custom op under torch.compile,
    a direct ``Observer.join`` otherwise."""
    if observer is None or not observer.overlap:
        return
    t = torch()
    if t.compiler.is_compiling():
        t.ops.ring2.join(observer.token, observer.index)
    else:
        observer.join()


def total_step_bytes(registry: HookRegistry, batch) -> int:
    from .policy import estimate_step_bytes
    return sum(estimate_step_bytes(registry, batch))


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


__all__ = ["HookPoint", "Observer", "TokenSampler", "join_point", "total_step_bytes",
           "ceil_div"]
