"""Capture kernel parity: the reference's capture tests on the device, the
golden gather cases (criterion 3 recipe) and large-shape properties.

Reference: PKG/tests/test_hooks.py:101-203, test_acceptance.py:225-256.
"""

import hashlib
import random

import pytest

import oracle
from paper_2605_11093_b200 import (CaptureOutcome, ConfigError, DType,
                                   HookDisabled, HookSpec, ModelSpec,
                                   PayloadRingFull, RingConfig, TensorView,
                                   allocate_rings, capture, install_hooks,
                                   round_up_to_copy_unit)

pytestmark = pytest.mark.gpu


def make_view(rng, batch, slice_bytes, dtype):
    slices = [bytes(rng.randrange(256) for _ in range(slice_bytes))
              for _ in range(batch)]
    return TensorView(b"".join(slices), (batch, slice_bytes // dtype.width),
                      dtype), slices


def ref_gather(slices, keep):
    return b"".join(s for s, k in zip(slices, keep) if k)


def test_capture_gather_compact_basic():
    reg = install_hooks(ModelSpec(1, 8), [HookSpec("h", (4,), DType.of("u8"))])
    ring = allocate_rings(RingConfig(1024, 16))
    view, slices = make_view(random.Random(1), 4, 4, DType.of("u8"))
    out = capture(reg, ring, 0, view, (1, 0, 1, 1), step_seq=5)
    assert out.bytes_written == 12
    (d,) = ring.poll_ready(1)
    assert (d.payload_len, d.hook_id, d.step_seq) == (12, 0, 5)
    assert bytes(ring.payload_view(d.payload_offset, 12)) == \
        ref_gather(slices, [1, 0, 1, 1])


def test_capture_non_copy_unit_tail_path():
    reg = install_hooks(ModelSpec(1, 8), [HookSpec("h", (17,), DType.of("u8"))])
    ring = allocate_rings(RingConfig(1024, 16))
    view, slices = make_view(random.Random(2), 4, 17, DType.of("u8"))
    assert capture(reg, ring, 0, view, (1, 1, 1, 1)).bytes_written == 68
    (d,) = ring.poll_ready(1)
    assert d.reserved_len == 80
    assert bytes(ring.payload_view(d.payload_offset, d.payload_len)) == \
        ref_gather(slices, [1, 1, 1, 1])


def test_capture_all_dropped_is_identity():
    reg = install_hooks(ModelSpec(1, 8), [HookSpec("h", (16,), DType.of("u8"))])
    ring = allocate_rings(RingConfig(256, 4))
    view, _ = make_view(random.Random(3), 3, 16, DType.of("u8"))
    assert capture(reg, ring, 0, view, (0, 0, 0)) == CaptureOutcome(0, 0.0)
    assert ring.occupancy == 0 and ring.ready_entries() == 0


def test_capture_all_dropped_device_keep_is_identity():
    import torch
    reg = install_hooks(ModelSpec(1, 8), [HookSpec("h", (16,), DType.of("u8"))])
    ring = allocate_rings(RingConfig(256, 4))
    view, _ = make_view(random.Random(3), 3, 16, DType.of("u8"))
    keep = torch.zeros(3, dtype=torch.uint8, device="cuda")
    assert capture(reg, ring, 0, view, keep).bytes_written == 0
    assert ring.occupancy == 0 and ring.ready_entries() == 0


def test_capture_disabled_hook_rejected():
    reg = install_hooks(ModelSpec(1, 8), [HookSpec("h", (16,), DType.of("u8"))])
    reg.set_hook_filter([])
    reg.commit_filter()
    ring = allocate_rings(RingConfig(256, 4))
    view, _ = make_view(random.Random(4), 2, 16, DType.of("u8"))
    with pytest.raises(HookDisabled):
        capture(reg, ring, 0, view, (1, 1))
    enabled = install_hooks(ModelSpec(1, 8),
                            [HookSpec("h", (16,), DType.of("u8"))])
    with pytest.raises(ConfigError):      # keep length != batch
        capture(enabled, ring, 0, view, (1,))
    assert ring.occupancy == 0


def test_capture_backpressure_propagates_without_mutation():
    reg = install_hooks(ModelSpec(1, 8), [HookSpec("h", (64,), DType.of("u8"))])
    ring = allocate_rings(RingConfig(128, 4))
    view, _ = make_view(random.Random(5), 2, 64, DType.of("u8"))
    capture(reg, ring, 0, view, (1, 1))
    before = ring.state()
    with pytest.raises(PayloadRingFull):
        capture(reg, ring, 0, view, (1, 1))
    after = ring.state()
    assert (before.payload_head, before.occupancy, before.meta_head) == \
        (after.payload_head, after.occupancy, after.meta_head)


def test_randomized_gather_matches_reference():
    """test_hooks.py:181-203 recipe (random.Random(0xFEED))."""
    rng = random.Random(0xFEED)
    for _ in range(300):
        width = rng.choice([1, 2, 4])
        per_req = rng.randint(1, 97)
        slice_bytes = per_req * width
        batch = rng.randint(1, 8)
        dt = DType(f"w{width}", width)
        reg = install_hooks(ModelSpec(1, 8), [HookSpec("h", (per_req,), dt)])
        ring = allocate_rings(
            RingConfig(round_up_to_copy_unit(slice_bytes * batch) + 64, 4))
        view, slices = make_view(rng, batch, slice_bytes, dt)
        keep = tuple(rng.randint(0, 1) for _ in range(batch))
        out = capture(reg, ring, 0, view, keep)
        expected = ref_gather(slices, keep)
        assert out.bytes_written == len(expected)
        if expected:
            (d,) = ring.poll_ready(1)
            assert bytes(ring.payload_view(d.payload_offset, d.payload_len)) \
                == expected


def test_golden_gather_cases(golden):
    """Criterion-3 recipe (random.Random(7)); expected bytes hashed by the
    reference itself; also checked against the C oracle."""
    cases = golden("gather_cases.json")
    rng = random.Random(7)
    widths = {1: "u8", 2: "bf16", 4: "f32", 8: "f64"}
    ring = allocate_rings(RingConfig(32 << 10, 8))
    tails = 0
    for case, want in enumerate(cases):
        batch = rng.randint(1, 8)
        tokens = rng.randint(1, 9)
        feat = rng.randint(1, 33)
        dtype = DType.of(widths[rng.choice((1, 2, 4, 8))])
        slice_size = tokens * feat * dtype.width
        data = rng.randbytes(batch * slice_size)
        keep = [rng.randint(0, 1) for _ in range(batch)]
        assert (batch, tokens, feat, dtype.width, keep) == (
            want["batch"], want["tokens"], want["feat"], want["width"],
            want["keep"])
        tails += slice_size % 16 != 0
        reg = install_hooks(ModelSpec(1, 16),
                            [HookSpec(f"case{case}", (tokens, feat), dtype)])
        view = TensorView(data, (batch, tokens, feat), dtype)
        out = capture(reg, ring, 0, view, keep)
        got = b""
        if out.bytes_written:
            (d,) = ring.poll_ready(1)
            got = bytes(ring.payload_view(d.payload_offset, d.payload_len))
            ring.release_payload(d.payload_offset, d.reserved_len)
        assert len(got) == want["len"]
        assert hashlib.sha256(got).hexdigest()[:32] == want["sha"], case
        assert got == oracle.gather(data, batch, 1, slice_size, slice_size,
                                    slice_size, keep, per_outer=True)
    assert tails > 200
