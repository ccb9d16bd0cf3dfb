"""Host-side logic of the package on CPU: policy decisions (against the
reference's recorded answers), hook expansion, FIFO/records, split_payload,
sink formats. The ring the policy consults is the oracle restatement wrapped
in the RingPair snapshot interface (no GPU needed)."""

import io
import json
import random
import socket

import pytest

import oracle
from paper_2605_11093_b200 import (BEST_EFFORT, COMPLETENESS, DROP_RECENT,
                                   KEEP_BY_PATTERN, CaptureRecord, ConfigError,
                                   DrainConfig, DType, FileSink, HookSpec,
                                   MetaMismatch, ModelSpec, NullSink,
                                   PolicyConfig, Predicate, RingConfig,
                                   RingState, StepRequest, StreamSink,
                                   TensorMeta, TensorMetaFIFO,
                                   estimate_step_bytes, install_hooks,
                                   prepare_step, read_dataset, read_stream,
                                   split_payload)
from paper_2605_11093_b200.hookpoint import TokenSampler
from paper_2605_11093_b200.rings import Descriptor


class OracleBackedRing:
    """RingPair's snapshot interface over the C oracle ring."""

    def __init__(self, capacity, slots, watermark=0.8):
        self.r = oracle.OracleRing(capacity, slots)
        self.cap, self.slots, self.wm = capacity, slots, watermark

    def state(self):
        s = self.r.state()
        return RingState(s["head"], s["tail"], s["used"], self.cap,
                         s["meta_head"], s["meta_tail"], self.slots, self.wm)

    def would_fit(self, lengths, meta_entries=None):
        return self.r.would_fit(list(lengths), meta_entries)


def _policy(desc):
    if desc["mode"] == "completeness":
        return PolicyConfig(mode=COMPLETENESS, pressure_watermark=desc["watermark"])
    if desc["strategy"] == "drop-recent":
        return PolicyConfig(mode=BEST_EFFORT, strategy=DROP_RECENT)
    pred = Predicate(request_ids=frozenset(desc["ids"])) if "ids" in desc \
        else Predicate(prompt_prefix=desc["prefix"])
    return PolicyConfig(mode=BEST_EFFORT, strategy=KEEP_BY_PATTERN, predicate=pred)


def test_prepare_step_matches_reference_decisions(golden):
    """300 recorded reference plans (keep, flush, kept/dropped, flagged,
    free bytes, FIFO entries) reproduced decision for decision."""
    for case in golden("policy_cases.json"):
        specs = [HookSpec(n, tuple(d), DType.of(dt), per_layer=pl)
                 for n, d, dt, pl in case["specs"]]
        reg = install_hooks(ModelSpec(case["layers"], case["hidden"]), specs)
        ring = OracleBackedRing(case["capacity"], case["slots"])
        for op in case["script"]:
            if op[0] == "R":
                rc, off, _ = ring.r.reserve(op[1])
                assert (None if rc else off) == op[2]
            else:
                assert ring.r.release(op[1], op[2]) == 0
        batch = [StepRequest(*r) for r in case["batch"]]
        plan = prepare_step(_policy(case["policy"]), batch, ring, reg,
                            step_seq=case["step"])
        e = case["expect"]
        assert list(plan.keep) == e["keep"]
        assert plan.flush_before == e["flush"]
        assert list(plan.kept_ids) == e["kept"]
        assert list(plan.dropped_ids) == e["dropped"]
        assert list(plan.flagged_ids) == e["flagged"]
        assert plan.free_bytes_at_plan == e["free"]
        assert [[m.hook_name, m.layer_index, list(m.shape), m.dtype.name,
                 list(m.request_ids), [list(t) for t in m.token_ranges],
                 m.expected_payload_len] for m in plan.fifo_entries] == e["fifo"]


def req(i, tokens=1, prompt=None, start=0):
    return StepRequest(i, i, prompt if prompt is not None else f"req {i}",
                       tokens, start)


def test_policy_known_answers():
    """PKG/tests/test_policy.py:74-136."""
    reg = install_hooks(ModelSpec(1, 8), [HookSpec(
        "resid", ("tokens", "hidden"), DType.of("u8"), per_layer=True)])
    ring = OracleBackedRing(160, 8)
    plan = prepare_step(PolicyConfig(), [req(0), req(1), req(2)], ring, reg,
                        step_seq=0)
    assert plan.keep == (1, 1, 1) and not plan.flush_before
    ring.r.reserve(128)
    assert prepare_step(PolicyConfig(), [req(0)], ring, reg, step_seq=1).flush_before
    reg16 = install_hooks(ModelSpec(1, 16), [HookSpec(
        "resid", ("tokens", "hidden"), DType.of("u8"), per_layer=True)])
    ring = OracleBackedRing(48, 8)
    best = PolicyConfig(mode=BEST_EFFORT, strategy=DROP_RECENT)
    batch = [req(2), req(0), req(1)]
    assert prepare_step(best, batch, ring, reg16, step_seq=0).keep == (1, 1, 1)
    ring.r.reserve(16)
    plan = prepare_step(best, batch, ring, reg16, step_seq=1)
    assert plan.keep == (0, 1, 1) and plan.dropped_ids == (2,)


def test_estimates_and_expansion():
    reg = install_hooks(ModelSpec(2, 64), [
        HookSpec("resid", ("tokens", "hidden"), DType.of("f16"), per_layer=True),
        HookSpec("logits", ("tokens", 32), DType.of("f32"))])
    assert [h.name for h in reg.hooks] == ["resid[0]", "resid[1]", "logits"]
    assert estimate_step_bytes(reg, [req(0, tokens=2)]) == [2 * (2 * 64 * 2) + 2 * 32 * 4]
    reg.set_hook_filter(["logits"])
    assert reg.enabled_ids() == [0, 1, 2]
    reg.commit_filter()
    assert estimate_step_bytes(reg, [req(0, tokens=2)]) == [2 * 32 * 4]
    with pytest.raises(ConfigError):
        reg.set_hook_filter(["nope"])


@pytest.mark.parametrize("layers,expected", [(36, 38), (32, 34), (40, 42)])
def test_hook_counts(layers, expected):
    specs = [HookSpec("resid", ("tokens", "hidden"), DType.of("bf16"), per_layer=True),
             HookSpec("final_ln", ("tokens", "hidden"), DType.of("bf16")),
             HookSpec("logits", ("tokens", 4096), DType.of("f32"))]
    assert len(install_hooks(ModelSpec(layers, 1024), specs)) == expected


def test_cast_and_reduce_hook_arithmetic():
    cast = HookSpec("resid", ("tokens", "hidden"), DType.of("bf16"),
                    cast_to=DType.of("f8e4m3"))
    assert cast.slice_bytes(tokens=4, hidden=4096) == 4 * 4096
    assert cast.out_dtype.name == "f8e4m3"
    red = HookSpec("resid", ("tokens", "hidden"), DType.of("bf16"), reduce="stats")
    assert red.resolve_shape(4, 4096) == (4, 4) and red.slice_bytes(4, 4096) == 64
    with pytest.raises(ConfigError):
        HookSpec("x", ("tokens",), DType.of("u8"), reduce="mean")
    with pytest.raises(ConfigError):
        HookSpec("x", ("tokens",), DType.of("bf16"), reduce="median")


def test_fifo_match_and_split():
    f16 = DType.of("f16")
    fifo = TensorMetaFIFO()
    meta = TensorMeta("resid[2]", 2, 7, (11, 13), ((4, 5), (4, 5)), (1, 64), f16)
    fifo.push(meta)
    with pytest.raises(MetaMismatch):
        fifo.match(Descriptor(0, 256, 5, 8), "resid[2]")   # wrong step
    assert len(fifo) == 1                                  # head survives
    got = fifo.match(Descriptor(0, 256, 5, 7), "resid[2]")
    payload = bytes(range(256))
    recs = split_payload(got, payload)
    assert [r.request_id for r in recs] == [11, 13]
    assert recs[0].payload == payload[:128] and recs[1].payload == payload[128:]
    views = split_payload(got, payload, copy=False)
    assert [bytes(r.payload) for r in views] == [r.payload for r in recs]
    with pytest.raises(MetaMismatch):
        split_payload(got, payload[:-2])


def test_ragged_token_rows_split():
    bf16 = DType.of("bf16")
    meta = TensorMeta("resid[0]", 0, 3, (1, 2), ((0, 8), (0, 8)), (8, 4), bf16,
                      row_counts=(2, 3), token_indices=((0, 4), (1, 2, 7)))
    assert meta.expected_payload_len == 5 * 8
    recs = split_payload(meta, bytes(40))
    assert [r.shape for r in recs] == [(2, 4), (3, 4)]


def test_token_sampler():
    assert TokenSampler(every=4).select(1, 0, 10) == [0, 4, 8]
    s = TokenSampler(rate=0.5, seed=3)
    assert s.select(7, 2, 64) == s.select(7, 2, 64)
    with pytest.raises(ConfigError):
        TokenSampler()


def test_sink_formats_match_reference(golden, tmp_path):
    g = golden("sinks.json")
    recs = [CaptureRecord(7, "resid[2]", 2, 5, (4, 8), (4, 2), DType.of("bf16"),
                          (0, 0), bytes(range(16))),
            CaptureRecord(9, "logits", None, 6, (8, 9), (1, 3), DType.of("f32"),
                          (1, 0), bytes(range(100, 112)))]
    with FileSink(tmp_path / "ds") as sink:
        sink.write(recs)
    lines = (tmp_path / "ds" / "records.ndjson").read_text().splitlines()
    assert lines == g["lines"]
    assert read_dataset(tmp_path / "ds") == recs
    buf = io.BytesIO()
    StreamSink(buf).write(recs)
    assert buf.getvalue().hex() == g["stream_hex"]
    assert [h for h, _ in read_stream(io.BytesIO(buf.getvalue()))] == \
        [json.loads(x) for x in g["lines"]]


def test_stream_sink_over_socket():
    a, b = socket.socketpair()
    rec = CaptureRecord(1, "h", 0, 0, (0, 1), (1, 2), DType.of("u8"), (0, 0), b"xy")
    sink = StreamSink(a)
    sink.write([rec])
    sink.flush()
    sink.close()
    a.close()
    with b.makefile("rb") as fh:
        ((header, payload),) = read_stream(fh)
    assert payload == b"xy" and header["hook"] == "h"


def test_null_sink_and_configs():
    s = NullSink()
    s.write([CaptureRecord(1, "h", 0, 0, (0, 1), (1, 2), DType.of("u8"),
                           (0, 0), b"ab")])
    assert (s.records_written, s.bytes_written) == (1, 2)
    with pytest.raises(ConfigError):
        RingConfig(payload_capacity=100, meta_slots=4)
    with pytest.raises(ConfigError):
        DrainConfig(max_wait=0)
    with pytest.raises(ConfigError):
        DrainConfig(mode="dma")
    with pytest.raises(ConfigError):
        PolicyConfig(mode=BEST_EFFORT, strategy=KEEP_BY_PATTERN)


def test_descriptor_wire_round_trip():
    d = Descriptor(4096, 48, 7, 3, 12, skip_before=32, flags=1, n_rows=4,
                   capture_seq=9)
    assert Descriptor.unpack(d.pack_device()) == d
    assert Descriptor.unpack(d.pack_device()).skip_before == 32
    assert d.pack() == oracle.desc_pack(4096, 48, 7, 3, 12)
    assert d.reserved_len == 48 and Descriptor(0, 17, 0, 0).reserved_len == 32


def test_hookpoint_custom_op_survives_tracing():
    """PAPER.md §3.1: HookPoint dispatches a custom operator, so compiler
    tracing keeps the capture as an opaque node instead of a Python hook."""
    import torch
    from torch.fx.experimental.proxy_tensor import make_fx

    from paper_2605_11093_b200.hookpoint import _capture_op  # noqa: F401

    def f(x, tok):
        torch.ops.ring2.capture(x, tok, 0, 3)
        return x + 1

    g = make_fx(f, tracing_mode="fake")(torch.randn(2, 4),
                                        torch.zeros(1, dtype=torch.uint8))
    assert "ring2.capture.default" in [str(n.target) for n in g.graph.nodes]


def test_ragged_continuous_batching_plan():
    """Extension: mixed prefill chunk + decodes in one step."""
    reg = install_hooks(ModelSpec(2, 16), [
        HookSpec("resid", ("tokens", "hidden"), DType.of("bf16"), per_layer=True),
        HookSpec("logits", ("tokens", 8), DType.of("f32"))])
    ring = OracleBackedRing(1 << 20, 64)
    batch = [StepRequest(1, 0, "a", 5, 0), StepRequest(2, 1, "b", 1, 40),
             StepRequest(3, 2, "c", 3, 7)]
    with pytest.raises(ConfigError):
        prepare_step(PolicyConfig(), batch, ring, reg, step_seq=0)
    plan = prepare_step(PolicyConfig(), batch, ring, reg, step_seq=0, ragged=True)
    assert [m.hook_name for m in plan.fifo_entries] == ["resid[0]", "resid[1]", "logits"]
    m = plan.fifo_entries[0]
    assert m.row_counts == (5, 1, 3) and m.shape == (5, 16)
    assert m.token_ranges == ((0, 5), (40, 41), (7, 10))
    assert m.expected_payload_len == 9 * 16 * 2
    recs = split_payload(m, bytes(range(256)) + bytes(32))
    assert [r.shape for r in recs] == [(5, 16), (1, 16), (3, 16)]
    best = PolicyConfig(mode=BEST_EFFORT, strategy=DROP_RECENT)
    small = OracleBackedRing(16 * 30, 64)     # 480 B: request 1 alone fits
    plan = prepare_step(best, batch, small, reg, step_seq=1, ragged=True)
    assert plan.kept_ids == (1,) and plan.dropped_ids == (2, 3)
    bad = install_hooks(ModelSpec(1, 16), [HookSpec(
        "attn", (4, "tokens", "tokens"), DType.of("bf16"), per_layer=True)])
    with pytest.raises(ConfigError):
        prepare_step(PolicyConfig(), batch, ring, bad, step_seq=0, ragged=True)


def test_binary_prefix_search_equals_linear_scan():
    """The policy's binary search over kept prefixes returns what the
    reference's linear scan (policy.py:135-145) returns."""
    rng = random.Random(17)
    for _ in range(200):
        reg = install_hooks(ModelSpec(rng.randint(1, 3), rng.choice([8, 17, 32])), [
            HookSpec("r", ("tokens", "hidden"), DType.of("u8"), per_layer=True)])
        ring = OracleBackedRing(16 * rng.randint(2, 40), rng.randint(1, 8))
        for _ in range(rng.randint(0, 6)):
            ring.r.reserve(16 * rng.randint(1, 6))
        batch = [req(i, tokens=2) for i in range(rng.randint(1, 9))]
        plan = prepare_step(PolicyConfig(mode=BEST_EFFORT, strategy=DROP_RECENT),
                            batch, ring, reg, step_seq=0)
        from paper_2605_11093_b200.policy import reservation_sizes
        linear = 0
        for m in range(len(batch), 0, -1):
            sizes = reservation_sizes(reg, batch[:m])
            if ring.would_fit(sizes, meta_entries=len(sizes)):
                linear = m
                break
        assert len(plan.kept_ids) == linear


def test_plan_entries_cache_follows_filter_and_tokens():
    reg = install_hooks(ModelSpec(2, 16), [
        HookSpec("resid", ("tokens", "hidden"), DType.of("bf16"), per_layer=True),
        HookSpec("logits", ("tokens", 8), DType.of("f32"))])
    e = reg.plan_entries(3)
    assert [(h, hk.name, sh) for h, hk, sh in e] == [
        (i, reg.hook(i).name, reg.hook(i).resolve_shape(3, 16)) for i in reg.enabled_ids()]
    assert reg.plan_entries(3) is e
    reg.set_hook_filter(["logits"])
    reg.commit_filter()
    assert [hk.name for _, hk, _ in reg.plan_entries(3)] == ["logits"]
    assert reg.plan_entries(5)[0][2] == (5, 8)


def test_with_hook_equals_full_construction():
    from paper_2605_11093_b200 import TensorMeta
    base = TensorMeta("a[0]", 0, 7, (3, 1), ((0, 2), (5, 9)), (4, 16), DType.of("bf16"),
                      (1, 0), row_counts=(2, 4))
    m = base.with_hook("b[1]", 1, (4, 32), DType.of("f32"))
    full = TensorMeta("b[1]", 1, 7, (3, 1), ((0, 2), (5, 9)), (4, 32), DType.of("f32"),
                      (1, 0), row_counts=(2, 4))
    assert m == full and m.expected_payload_len == full.expected_payload_len
    with pytest.raises(ConfigError):
        base.with_hook("c", 0, (0, 4), DType.of("u8"))


def test_step_metas_fifo_materialises_lazily_in_order():
    from paper_2605_11093_b200 import TensorMeta, TensorMetaFIFO
    from paper_2605_11093_b200.records import StepMetas
    bf = DType.of("bf16")
    base = TensorMeta("a[0]", 0, 3, (5, 2), ((0, 4), (1, 2)), (4, 8), bf, row_counts=(4, 1))
    sm = StepMetas(base, [("a[0]", 0, (4, 8), bf), ("b[0]", 0, (4, 16), bf),
                          ("c", None, (4, 2), DType.of("f32"))])
    assert sm._cache[1] is None and len(sm) == 3
    assert sm.payload_lens() == [m.expected_payload_len for m in sm]
    fifo = TensorMetaFIFO()
    fifo.push(TensorMeta("z", 0, 2, (9,), ((0, 1),), (1, 4), bf))
    fifo.extend(sm)
    assert len(fifo) == 4
    d = lambda name, n: Descriptor(0, n, 0, 3 if name != "z" else 2)  # noqa: E731
    assert fifo.match(d("z", 8), "z").hook_name == "z"
    assert fifo.peek().hook_name == "a[0]"
    for m in sm:
        assert fifo.match(d(m.hook_name, m.expected_payload_len), m.hook_name) == m
    assert len(fifo) == 0 and fifo.peek() is None


def test_step_entries_payload_lens_match_the_uncached_formula():
    """HookRegistry.step_entries caches per-entry byte factors; StepMetas
    payload lengths built from them equal the per-entry shape formula for
    uniform batches (per request) and ragged ones (per token row)."""
    from paper_2605_11093_b200.hooks import DType, HookSpec, ModelSpec, install_hooks
    from paper_2605_11093_b200.records import StepMetas, TensorMeta
    reg = install_hooks(ModelSpec(2, 64), [
        HookSpec("resid", ("tokens", "hidden"), DType.of("bf16"), per_layer=True),
        HookSpec("attn", (4, "tokens", "tokens"), DType.of("f32"), per_layer=True),
        HookSpec("red", ("tokens", "hidden"), DType.of("bf16"), per_layer=True,
                 reduce="stats")])
    entries, per = reg.step_entries(5, False)
    name, layer, shape, dt = entries[0]
    base = TensorMeta(name, layer, 3, (1, 2, 3), ((0, 5),) * 3, shape, dt)
    assert StepMetas(base, entries, per).payload_lens() == \
        StepMetas(base, list(entries)).payload_lens()
    reg2 = install_hooks(ModelSpec(2, 64), [
        HookSpec("resid", ("tokens", "hidden"), DType.of("bf16"), per_layer=True),
        HookSpec("mlp", ("tokens", 128), DType.of("bf16"), per_layer=True)])
    entries, per = reg2.step_entries(7, True)
    name, layer, shape, dt = entries[0]
    base = TensorMeta(name, layer, 3, (1, 2), ((0, 3), (0, 7)), shape, dt,
                      row_counts=(3, 7))
    assert StepMetas(base, entries, per).payload_lens() == \
        StepMetas(base, list(entries)).payload_lens()
    # the ragged view rejects a hook whose tokens axis is not first
    import pytest as _pt
    from paper_2605_11093_b200.errors import ConfigError
    with _pt.raises(ConfigError):
        reg.step_entries(5, True)
