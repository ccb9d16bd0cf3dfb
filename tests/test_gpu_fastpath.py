"""Capture-kernel reservation paths under a live consumer.

The capture kernel reserves ring space either on the fast path (every CTA
runs the allocator on the producer snapshot the previous producer
operation left, ring2_internal.h ProdSnap) or, when the snapshot says the
ring or the meta ring is full, on the leader path against the live
consumer cursors. Host protocol operations (reserve_payload / publish,
SRC/rings.py:286-353) rewrite the snapshot too. These tests stream
hundreds of captures of random shapes and keep vectors through a small
ring that the background staging engine drains concurrently (so the ring
wraps, dead-skips and empty-resets many times, and the snapshot is stale
most of the time), interleave host protocol captures, and check every
record byte-for-byte against the reference gather (SRC/hooks.py:266-278).
"""

import random

import pytest
import torch

from paper_2605_11093_b200 import (Descriptor, DrainConfig, DType,
                                   ExportPipeline, RingConfig, RingPair,
                                   TensorMeta, TensorMetaFIFO,
                                   round_up_to_copy_unit)
from paper_2605_11093_b200.hooks import RowSource, capture_args, launch_capture

pytestmark = pytest.mark.gpu
U8 = DType.of("u8")


class ListSink:
    def __init__(self):
        self.records = []

    def write(self, recs):
        self.records.extend(recs)


def _stream(seed, n_caps, payload_capacity, meta_slots, host_every=0,
            max_bytes=300_000, sealed=False):
    rng = random.Random(seed)
    torch.manual_seed(seed)
    ring = RingPair(RingConfig(payload_capacity=payload_capacity, meta_slots=meta_slots))
    names = {}
    fifo = TensorMetaFIFO()
    pipe = ExportPipeline(ring, DrainConfig(min_ready_entries=1, min_ready_bytes=1,
                                            max_wait=1e-4, staging_buffer_size=1 << 20,
                                            staging_buffer_count=4, page_out="handoff"),
                          None, fifo, hook_name_of=names.__getitem__)
    sink = ListSink()
    pipe.start(sink)
    s = torch.cuda.Stream()
    expected, keepalive = [], []
    launched = 0
    for i in range(n_caps):
        if host_every and i % host_every == host_every - 1:
            # host protocol capture: reserve + write + publish on the host
            if sealed:
                ring.seal(s)
            s.synchronize()
            total = rng.randrange(16, 4096)
            need = round_up_to_copy_unit(total)
            while ring.free_meta_slots() == 0 or not ring.would_fit([need]):
                pass
            payload = rng.randbytes(total)
            off = ring.reserve_payload(need)
            ring.payload_view(off, total)[:] = payload
            names[10_000 + i] = f"host{i}"
            fifo.push(TensorMeta(f"host{i}", 0, i, (0,), ((0, 1),), (1, total), U8))
            ring.publish(Descriptor(off, total, 10_000 + i, i))
            expected.append([payload])
            continue
        B = rng.randint(1, 12)
        T = rng.randint(1, 8)
        row = rng.choice([16, 48, 100, 1024, 4096, 7, 4000, 33]) * rng.randint(1, 8)
        while B * T * row > max_bytes:
            row = max(1, row // 2)
        x = torch.randint(0, 256, (B, T, row), dtype=torch.uint8, device="cuda")
        keep = [rng.random() < 0.7 for _ in range(B)]
        if rng.random() < 0.1:
            keep = [False] * B
        kt = torch.tensor(keep, dtype=torch.uint8, device="cuda")
        kept = [b for b in range(B) if keep[b]]
        src = RowSource(x.data_ptr(), B, T, row, T * row, row, x)
        if kept:
            names[i] = f"h{i}"
            fifo.push(TensorMeta(f"h{i}", 0, i, tuple(kept), tuple((0, T) for _ in kept),
                                 (T, row), U8))
            host = x.cpu()
            expected.append([host[b].numpy().tobytes() for b in kept])
        with torch.cuda.stream(s):
            launch_capture(ring, capture_args(src, hook_id=i, keep_ptr=kt.data_ptr(),
                                              keep_per_outer=True, step_seq=i,
                                              full="wait", sealed=sealed), s)
        launched += 1
        keepalive.append((x, kt))
        if len(keepalive) > 64:
            s.synchronize()
            keepalive.clear()
    if sealed:
        ring.seal(s)
    s.synchronize()
    pipe.stop(flush=True, timeout=120)
    got = [r.payload for r in sink.records]
    want = [p for group in expected for p in group]
    state = ring.state()
    counters = ring.counters()
    pipe.close()
    ring.close()
    return got, want, state, counters, launched


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_captures_stream_through_wrapping_ring_bit_exact(seed):
    got, want, state, counters, _ = _stream(seed, 300, 1 << 20, 16)
    assert len(got) == len(want)
    for i, (g, w) in enumerate(zip(got, want)):
        assert g == w, f"record {i} differs"
    assert state.occupancy == 0
    assert counters["drops"] == 0


def test_host_protocol_ops_interleaved_with_captures():
    """reserve_payload/publish between capture launches must refresh the
    kernel's producer snapshot (else the next capture reuses the region)."""
    got, want, state, counters, _ = _stream(11, 240, 1 << 20, 32, host_every=5)
    assert len(got) == len(want)
    for i, (g, w) in enumerate(zip(got, want)):
        assert g == w, f"record {i} differs"
    assert state.occupancy == 0


def test_tiny_meta_ring_forces_leader_path():
    """Two descriptor slots: the snapshot's meta tail is almost always stale,
    so most launches take the leader path and wait on the live cursor."""
    got, want, state, counters, _ = _stream(5, 120, 1 << 20, 2, max_bytes=20_000)
    assert got == want
    assert state.occupancy == 0


def test_huge_token_keep_uses_inline_publish_path():
    """> 512 copy CTAs (a 1.2 M-row token keep needs ~590 rank-table slices):
    the fast path falls back to the last-CTA publish; bytes must match the
    reference gather and the ring must drain empty."""
    torch.manual_seed(3)
    rows, row = 1_200_000, 16
    x = torch.randint(0, 256, (rows, row), dtype=torch.uint8, device="cuda")
    keep = (torch.rand(rows, device="cuda") < 0.5).to(torch.uint8)
    ring = RingPair(RingConfig(payload_capacity=64 << 20, meta_slots=16))
    src = RowSource(x.data_ptr(), rows, 1, row, row, row, x)
    launch_capture(ring, capture_args(src, hook_id=0, keep_ptr=keep.data_ptr(),
                                      step_seq=5, full="raise"), torch.cuda.current_stream())
    torch.cuda.synchronize()
    (d,) = ring.poll_ready(1)
    want = x[keep.bool()].cpu().numpy().tobytes()
    assert d.payload_len == len(want)
    assert bytes(ring.payload_view(d.payload_offset, d.payload_len)) == want
    assert (d.flags >> 16) == 0
    ring.release_payload(d.payload_offset, round_up_to_copy_unit(d.payload_len))
    ring.close()


@pytest.mark.parametrize("pattern", ["prefix", "all", "none_kept_tail", "holes"])
def test_token_row_keep_up_to_256_rows(pattern):
    """<= 256 keep units take the ballot path with speculative loads; a keep
    vector that is a prefix of ones (CUDA-graph padding rows at the end)
    keeps the speculation valid, any other pattern must fall back."""
    torch.manual_seed(17)
    rng = random.Random(17)
    for rows, row in ((256, 8192), (200, 28672), (40, 4096), (256, 48), (97, 4000)):
        x = torch.randint(0, 256, (rows, row), dtype=torch.uint8, device="cuda")
        if pattern == "prefix":
            n = rng.randint(1, rows)
            keep = [1] * n + [0] * (rows - n)
        elif pattern == "all":
            keep = [1] * rows
        elif pattern == "none_kept_tail":
            keep = [0] * (rows // 2) + [1] * (rows - rows // 2)
        else:
            keep = [int(rng.random() < 0.6) for _ in range(rows)]
            keep[0] = 1
        kt = torch.tensor(keep, dtype=torch.uint8, device="cuda")
        ring = RingPair(RingConfig(payload_capacity=64 << 20, meta_slots=16))
        src = RowSource(x.data_ptr(), rows, 1, row, row, row, x)
        launch_capture(ring, capture_args(src, hook_id=1, keep_ptr=kt.data_ptr(), step_seq=2,
                                          full="raise"), torch.cuda.current_stream())
        torch.cuda.synchronize()
        (d,) = ring.poll_ready(1)
        want = x[kt.bool()].cpu().numpy().tobytes()
        assert d.payload_len == len(want)
        assert bytes(ring.payload_view(d.payload_offset, d.payload_len)) == want, (rows, row)
        ring.close()


@pytest.mark.parametrize("seed", [21, 22])
def test_sealed_captures_complete_by_stream_order(seed):
    """TF_CAP_SEALED: no per-CTA completion bytes; each descriptor completes
    when the next capture on the stream posts, or at the seal. The ring
    (1 MiB) is small enough that captures wait on the device, where the
    waiting leader seals its predecessors."""
    got, want, state, counters, _ = _stream(seed, 300, 1 << 20, 16, sealed=True)
    assert len(got) == len(want)
    for i, (g, w) in enumerate(zip(got, want)):
        assert g == w, f"record {i} differs"
    assert state.occupancy == 0 and counters["drops"] == 0


def test_sealed_with_host_protocol_and_tiny_meta_ring():
    got, want, state, counters, _ = _stream(23, 200, 1 << 20, 2, host_every=7,
                                            max_bytes=20_000, sealed=True)
    assert got == want
    assert state.occupancy == 0 and counters["drops"] == 0


def test_sealed_last_capture_waits_for_the_seal():
    """The newest sealed descriptor is not handed out until a seal (or a
    later capture) completes it."""
    ring = RingPair(RingConfig(payload_capacity=1 << 20, meta_slots=16))
    s = torch.cuda.Stream()
    x = torch.randint(0, 256, (4, 1, 4096), dtype=torch.uint8, device="cuda")
    kt = torch.ones(4, dtype=torch.uint8, device="cuda")
    src = RowSource(x.data_ptr(), 4, 1, 4096, 4096, 4096, x)
    with torch.cuda.stream(s):
        for i in range(3):
            launch_capture(ring, capture_args(src, hook_id=i, keep_ptr=kt.data_ptr(),
                                              keep_per_outer=True, step_seq=i,
                                              full="wait", sealed=True), s)
    s.synchronize()
    assert ring.ready_entries() == 2      # the third waits for its seal
    ring.seal(s)
    s.synchronize()
    assert ring.ready_entries() == 3
    ring.close()
