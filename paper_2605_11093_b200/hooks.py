"""Observation points and the device capture call.

Same declaration API as the reference (hooks.py:24-195): ``DType``,
``ModelSpec``, ``HookSpec`` with the named axes ``tokens``/``hidden``,
``HookRegistry`` with step-boundary filtering, ``install_hooks`` (per-layer
expansion ``name[L]`` layer by layer, then globals). Two north-star
extensions ride on ``HookSpec``:

* ``cast_to``  — captured rows are converted element-wise (bf16 -> fp8/f16/
  f32 ...) inside the capture kernel;
* ``reduce``   — each captured row (token) is reduced to ``k`` f32 values
  (mean / l2 / absmax / rms / stats) inside the capture kernel.

``slice_bytes``/``resolve_shape`` describe what lands in the ring (the
record), ``source_shape`` what the model produced.

``capture`` (hooks.py:281-324) launches the sm_100a gather-compact kernel
through the C ABI. In this compat form it synchronises and raises the
reference's backpressure exceptions; the hot path (``launch_capture``,
``hookpoint.HookPoint``) never synchronises.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

from . import _native as N
from ._device import stream_handle, torch
from .errors import ConfigError, HookDisabled, MetaRingFull, PayloadRingFull
from .rings import Descriptor, RingPair

DTYPE_WIDTHS = {
    "u8": 1, "i8": 1, "f16": 2, "bf16": 2, "f32": 4, "i32": 4,
    "f64": 8, "i64": 8,
    # extension: cast targets
    "f8e4m3": 1, "f8e5m2": 1,
}

REDUCE_K = dict(N.TF_RED_K)

D2D_LAUNCH_OVERHEAD = 2e-6  # kept for DeviceCopyEngine's model (hooks.py:30)

TOKENS_AXIS = "tokens"
HIDDEN_AXIS = "hidden"


@dataclass(frozen=True)
class DType:
    name: str
    width: int

    @classmethod
    def of(cls, name: str) -> "DType":
        if name not in DTYPE_WIDTHS:
            raise ConfigError(f"unknown dtype {name!r}")
        return cls(name, DTYPE_WIDTHS[name])


@dataclass(frozen=True)
class ModelSpec:
    layers: int
    hidden: int

    def __post_init__(self) -> None:
        if min(self.layers, self.hidden) <= 0:
            raise ConfigError("layers and hidden must be positive")


@dataclass(frozen=True)
class HookSpec:
    """One capture point, or a per-layer template before installation."""

    name: str
    dims: tuple
    dtype: DType
    layer_index: int | None = None
    per_layer: bool = False
    cast_to: DType | None = None
    reduce: str | None = None

    def __post_init__(self) -> None:
        if not self.dims:
            raise ConfigError(f"hook {self.name!r} needs at least one dim")
        for d in self.dims:
            if isinstance(d, str):
                if d not in (TOKENS_AXIS, HIDDEN_AXIS):
                    raise ConfigError(
                        f"unknown axis {d!r} in hook {self.name!r}")
            elif d <= 0:
                raise ConfigError(f"non-positive dim in hook {self.name!r}")
        if self.per_layer and self.layer_index is not None:
            raise ConfigError("per_layer templates cannot carry a layer index")
        if self.cast_to is not None and self.reduce is not None:
            raise ConfigError("a hook either casts or reduces, not both")
        if self.reduce is not None and self.reduce not in REDUCE_K:
            raise ConfigError(f"unknown reduction {self.reduce!r}")
        if (self.cast_to is not None or self.reduce is not None) and \
                self.dtype.name not in ("f32", "f16", "bf16"):
            raise ConfigError("cast/reduce sources must be f32, f16 or bf16")
        if self.cast_to is not None and self.cast_to.name not in (
                "f32", "f16", "bf16", "f8e4m3", "f8e5m2"):
            raise ConfigError(f"cannot cast to {self.cast_to.name}")

    @property
    def sharded(self) -> bool:
        return HIDDEN_AXIS in self.dims

    @property
    def hidden_axis(self) -> int:
        return self.dims.index(HIDDEN_AXIS)

    @property
    def out_dtype(self) -> DType:
        if self.reduce is not None:
            return DType.of("f32")
        return self.cast_to if self.cast_to is not None else self.dtype

    @property
    def op(self) -> int:
        if self.reduce is not None:
            return N.TF_OP_REDUCE
        if self.cast_to is not None:
            return N.TF_OP_CAST
        return N.TF_OP_COPY

    def source_shape(self, tokens: int, hidden: int) -> tuple[int, ...]:
        table = {TOKENS_AXIS: tokens, HIDDEN_AXIS: hidden}
        return tuple(table.get(d, d) if isinstance(d, str) else d
                     for d in self.dims)

    def resolve_shape(self, tokens: int, hidden: int) -> tuple[int, ...]:
        """Per-request record shape (the source shape unless reduced)."""
        shape = self.source_shape(tokens, hidden)
        if self.reduce is not None:
            shape = shape[:-1] + (REDUCE_K[self.reduce],)
        return shape

    def slice_bytes(self, tokens: int, hidden: int) -> int:
        return math.prod(self.resolve_shape(tokens, hidden)) * \
            self.out_dtype.width


class HookRegistry:
    """Concrete hooks in firing order with a step-boundary enable filter."""

    def __init__(self, model: ModelSpec, hooks: list[HookSpec],
                 hidden_extent: int | None = None) -> None:
        self.model = model
        self.hooks = list(hooks)
        self.hidden_extent = hidden_extent if hidden_extent is not None \
            else model.hidden
        self._ids = {}
        for i, h in enumerate(self.hooks):
            if h.name in self._ids:
                raise ConfigError("duplicate concrete hook names")
            self._ids[h.name] = i
        self._enabled = frozenset(range(len(self.hooks)))
        self._staged: frozenset | None = None
        self._plan_cache: dict = {}

    def __len__(self) -> int:
        return len(self.hooks)

    def hook(self, hook_id: int) -> HookSpec:
        return self.hooks[hook_id]

    def id_of(self, name: str) -> int:
        if name not in self._ids:
            raise ConfigError(f"unknown hook {name!r}")
        return self._ids[name]

    def is_enabled(self, hook_id: int) -> bool:
        return hook_id in self._enabled

    def enabled_ids(self) -> list[int]:
        return sorted(self._enabled)

    def set_hook_filter(self, enabled_names) -> None:
        """Stage an enabled set (None = all); it applies at commit_filter."""
        if enabled_names is None:
            self._staged = frozenset(range(len(self.hooks)))
        else:
            self._staged = frozenset(self.id_of(n) for n in enabled_names)

    def commit_filter(self) -> None:
        if self._staged is not None:
            self._enabled, self._staged = self._staged, None

    def slice_bytes(self, hook_id: int, tokens: int) -> int:
        return self.hooks[hook_id].slice_bytes(tokens, self.hidden_extent)

    def plan_entries(self, tokens: int) -> tuple:
        """(hook_id, hook) and resolved per-request shape of every enabled
        hook in firing order for a step of ``tokens`` tokens; cached per
        enabled set and token count (the planner asks every step)."""
        c = self._plan_cache
        if c.get(None) is not self._enabled:
            c.clear()
            c[None] = self._enabled
        e = c.get(tokens)
        if e is None:
            e = tuple((hid, self.hooks[hid],
                       self.hooks[hid].resolve_shape(tokens, self.hidden_extent))
                      for hid in sorted(self._enabled))
            if len(c) > 512:
                c.clear()
                c[None] = self._enabled
            c[tokens] = e
        return e

    def step_entries(self, tokens: int, ragged: bool) -> tuple:
        """The planner's per-step view of plan_entries, cached the same way:
        (entries, per) with entries = [(name, layer, shape, out_dtype)] in
        firing order and per the record bytes of each per token row
        (ragged) or per request (uniform), so a step's payload lengths are
        rows x per, or requests x per.
        ragged=True validates once that every hook leads with tokens."""
        key = ("step", tokens, ragged)
        c = self._plan_cache
        e = c.get(key) if c.get(None) is self._enabled else None
        if e is None:
            entries = []
            per = []
            for hid, hook, shape in self.plan_entries(tokens):
                if ragged and (hook.dims[0] != "tokens" or "tokens" in hook.dims[1:]):
                    raise ConfigError(
                        f"ragged capture needs hook {hook.name!r} to lead with tokens")
                entries.append((hook.name, hook.layer_index, shape, hook.out_dtype))
                # ragged: bytes per token row; uniform: bytes per request
                per.append(math.prod(shape[1:] if ragged else shape) * hook.out_dtype.width)
            e = (tuple(entries), tuple(per))
            c[key] = e   # (plan_entries above has reset the cache if the set changed)
        return e


def install_hooks(model: ModelSpec, specs: list[HookSpec],
                  layers: list[int] | None = None,
                  hidden_extent: int | None = None,
                  include_globals: bool = True) -> HookRegistry:
    """Expand templates: ``name[L]`` layer-major, then globals (hooks.py:165-195)."""
    chosen = list(range(model.layers)) if layers is None else list(layers)
    per_layer = [s for s in specs if s.per_layer]
    concrete = [
        HookSpec(name=f"{s.name}[{layer}]", dims=s.dims, dtype=s.dtype,
                 layer_index=layer, cast_to=s.cast_to, reduce=s.reduce)
        for layer in chosen for s in per_layer
    ]
    for s in specs:
        if s.per_layer:
            continue
        if s.layer_index is None:
            if include_globals:
                concrete.append(s)
        elif s.layer_index in chosen:
            concrete.append(s)
    return HookRegistry(model, concrete, hidden_extent=hidden_extent)


@dataclass
class TensorView:
    """A batch-major tensor surface handed to a capture (hooks.py:198-229).

    ``data`` is a CUDA tensor (the normal case) or host bytes (uploaded on
    capture). ``shape`` is (batch, *per_request_dims).
    """

    data: object
    shape: tuple
    dtype: DType

    def __post_init__(self) -> None:
        if len(self.shape) < 1 or any(d <= 0 for d in self.shape):
            raise ConfigError("view shape must be non-empty and positive")
        need = math.prod(self.shape) * self.dtype.width
        have = _nbytes(self.data)
        if have != need:
            raise ConfigError(
                f"view of shape {self.shape} x {self.dtype.name} needs "
                f"{need} bytes, got {have}")

    @property
    def batch(self) -> int:
        return self.shape[0]

    @property
    def slice_size(self) -> int:
        return math.prod(self.shape[1:]) * self.dtype.width

    def slice(self, index: int) -> bytes:
        size = self.slice_size
        return _host_bytes(self.data)[index * size:(index + 1) * size]

    def device_tensor(self, device: int):
        """The view's bytes as a contiguous CUDA tensor (uploads host data)."""
        t = torch()
        d = self.data
        if isinstance(d, t.Tensor):
            if not d.is_cuda:
                d = d.to(f"cuda:{device}")
            return d.contiguous()
        buf = t.frombuffer(bytearray(bytes(d)), dtype=t.uint8)
        return buf.to(f"cuda:{device}")


def _nbytes(data) -> int:
    t = torch()
    if isinstance(data, t.Tensor):
        return data.numel() * data.element_size()
    return len(data)


def _host_bytes(data) -> bytes:
    t = torch()
    if isinstance(data, t.Tensor):
        return data.detach().contiguous().cpu().view(t.uint8).numpy().tobytes()
    return bytes(data)


@dataclass(frozen=True)
class DeviceCopyEngine:
    """Bandwidth/latency model kept for API parity (hooks.py:232-256).

    The device path does not consult it; measured times come from CUDA
    events. Exporter tests of the reference use it to predict durations.
    """

    d2d_bandwidth: float = math.inf
    d2h_bandwidth: float = 8e9
    d2h_latency: float = 10e-6
    d2d_launch_overhead: float = D2D_LAUNCH_OVERHEAD
    host_bandwidth: float = 64e9

    def __post_init__(self) -> None:
        if min(self.d2d_bandwidth, self.d2h_bandwidth, self.host_bandwidth) <= 0:
            raise ConfigError("bandwidths must be positive")
        if self.d2h_latency < 0 or self.d2d_launch_overhead < 0:
            raise ConfigError("latencies cannot be negative")

    def d2d_time(self, nbytes: int) -> float:
        return self.d2d_launch_overhead + nbytes / self.d2d_bandwidth

    def d2h_time(self, nbytes: int) -> float:
        return self.d2h_latency + nbytes / self.d2h_bandwidth

    def host_time(self, nbytes: int) -> float:
        return nbytes / self.host_bandwidth


@dataclass(frozen=True)
class CaptureOutcome:
    bytes_written: int
    copy_time: float
    stalled: float = 0.0


FULL_MODES = {"raise": N.TF_FULL_RAISE, "wait": N.TF_FULL_WAIT,
              "drop": N.TF_FULL_DROP}


@dataclass(frozen=True)
class RowSource:
    """Rows (o, m) of a strided device source: ptr + o*s_outer + m*s_mid."""

    ptr: int
    outer: int
    mid: int
    row_bytes: int
    stride_outer: int
    stride_mid: int
    keepalive: object = None

    @classmethod
    def batch_major(cls, tensor, batch: int) -> "RowSource":
        """Contiguous (batch, ...) tensor: one row per batch element."""
        nbytes = tensor.numel() * tensor.element_size()
        per = nbytes // batch
        return cls(tensor.data_ptr(), batch, 1, per, per, per, tensor)

    @classmethod
    def token_rows(cls, tensor) -> "RowSource":
        """(..., H) tensor with a contiguous last dim: one row per token."""
        t = tensor if tensor.stride(-1) == 1 else tensor.contiguous()
        h = t.shape[-1] * t.element_size()
        rows = t.numel() // t.shape[-1]
        if t.dim() >= 2 and not t.is_contiguous():
            t = t.reshape(-1, t.shape[-1])
            return cls(t.data_ptr(), rows, 1, h, t.stride(0) * t.element_size(),
                       h, t)
        return cls(t.data_ptr(), rows, 1, h, h, h, t)


def capture_args(src: RowSource, *, hook_id: int, hook: HookSpec | None = None,
                 op: int | None = None, in_dtype: str | None = None,
                 out_dtype: str | None = None, reduce: str | None = None,
                 keep_ptr: int = 0, keep_per_outer: bool = False,
                 step_seq: int = 0, step_seq_ptr: int = 0,
                 full: str = "wait", defer_publish: bool = False,
                 max_ctas: int = 0, sealed: bool = False) -> N.CCaptureArgs:
    """Fill the C argument block for one capture launch."""
    if hook is not None:
        op = hook.op
        in_dtype = hook.dtype.name
        out_dtype = hook.out_dtype.name
        reduce = hook.reduce
    op = N.TF_OP_COPY if op is None else op
    flags = FULL_MODES[full]
    if defer_publish:
        flags |= N.TF_CAP_DEFER_PUBLISH
    if sealed:  # completion by stream order; the caller seals (RingPair.seal)
        flags |= N.TF_CAP_SEALED
    if keep_per_outer:
        flags |= N.TF_CAP_KEEP_PER_OUTER
    return N.CCaptureArgs(
        src=src.ptr, outer=src.outer, mid=src.mid, row_bytes=src.row_bytes,
        stride_outer=src.stride_outer, stride_mid=src.stride_mid,
        keep=keep_ptr or None, step_seq_ptr=step_seq_ptr or None,
        step_seq=step_seq & 0xFFFFFFFF, hook_id=hook_id, op=op,
        in_dtype=N.TF_DTYPE.get(in_dtype or "u8", 0),
        out_dtype=N.TF_DTYPE.get(out_dtype or "u8", 0),
        reduce_op=N.TF_RED.get(reduce or "mean", 0), flags=flags,
        max_ctas=max_ctas)


def launch_capture(ring: RingPair, args: N.CCaptureArgs, stream=None) -> None:
    """Enqueue one capture kernel; never synchronises (graph-capturable)."""
    N.check(N.lib().tf_capture(ring.handle, stream_handle(stream, ring.device),
                               C.byref(args)))


def capture(
    registry: HookRegistry,
    ring: RingPair,
    hook_id: int,
    view: TensorView,
    keep,
    engine: DeviceCopyEngine | None = None,
    *,
    step_seq: int = 0,
    defer_publish: bool = False,
    stream=None,
):
    """Gather-compact the kept slices into the device ring and publish.

    Mirrors hooks.py:281-324: HookDisabled for filtered hooks, ConfigError
    for a keep vector of the wrong length, identity when nothing is kept,
    PayloadRingFull/MetaRingFull (meta checked first) with nothing mutated.
    This compat entry point synchronises to report those; ``copy_time`` is
    the measured kernel time.
    """
    hook = registry.hook(hook_id)
    if not registry.is_enabled(hook_id):
        raise HookDisabled(f"hook {hook.name!r} is disabled")
    t = torch()
    dev_keep = isinstance(keep, t.Tensor)
    if len(keep) != view.batch:
        raise ConfigError(
            f"keep vector length {len(keep)} != batch {view.batch}")
    if not dev_keep and not any(keep):
        out = CaptureOutcome(bytes_written=0, copy_time=0.0)
        return (out, None) if defer_publish else out
    data = view.device_tensor(ring.device)
    if dev_keep:
        keep_t = keep.to(device=f"cuda:{ring.device}", dtype=t.uint8)
    else:
        keep_t = t.tensor([1 if k else 0 for k in keep], dtype=t.uint8,
                          device=f"cuda:{ring.device}")
    per = view.slice_size
    if hook.reduce is not None:
        # reductions are per token: rows are the last axis
        row = view.shape[-1] * view.dtype.width
        src = RowSource(data.data_ptr(), view.batch, per // row, row, per,
                        row, data)
    else:
        src = RowSource(data.data_ptr(), view.batch, 1, per, per, per, data)
    args = capture_args(src, hook_id=hook_id, hook=hook,
                        keep_ptr=keep_t.data_ptr(), keep_per_outer=True,
                        step_seq=step_seq, full="raise",
                        defer_publish=defer_publish)
    s = stream if stream is not None else t.cuda.current_stream(ring.device)
    ring.sync()
    ring.sync_consumer()   # reserve against the consumer's latest releases
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    e0.record(s)
    launch_capture(ring, args, s)
    e1.record(s)
    e1.synchronize()
    res = N.CCaptureResult()
    N.check(N.lib().tf_ring_last_result(ring.handle, C.byref(res)))
    if res.status == N.TF_ERR_META_RING_FULL:
        raise MetaRingFull("no descriptor slot for this capture")
    if res.status == N.TF_ERR_PAYLOAD_RING_FULL:
        raise PayloadRingFull(
            f"need {res.desc.payload_len} bytes, ring {ring.capacity}")
    if res.status != N.TF_OK:
        raise N.exception_for(res.status, "capture rejected on device")
    out = CaptureOutcome(bytes_written=res.payload_len,
                         copy_time=e0.elapsed_time(e1) * 1e-3)
    if defer_publish:
        desc = Descriptor.from_c(res.desc) if res.payload_len else None
        return out, desc
    return out
