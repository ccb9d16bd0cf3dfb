"""Device Ring^2 protocol parity: the reference's ring tests and golden
protocol scripts replayed through the device allocator and meta ring.

Reference: PKG/tests/test_rings.py, PKG/tests/test_acceptance.py:130-220.
"""

import pytest

from paper_2605_11093_b200 import (AllocationError, Arena, ConfigError,
                                   Descriptor, MetaRingFull, OutOfOrderRelease,
                                   PayloadRingFull, RingConfig, allocate_rings)
from paper_2605_11093_b200.rings import DESCRIPTOR_SIZE, READY_SENTINEL

pytestmark = pytest.mark.gpu


def test_fresh_ring_state():
    ring = allocate_rings(RingConfig(payload_capacity=1024, meta_slots=8))
    s = ring.state()
    assert s.occupancy == 0 and s.payload_head == s.payload_tail == 0
    assert s.free_meta_slots == 8
    assert ring.poll_ready(8) == []


def test_arena_accounting():
    arena = Arena(capacity=4096)
    a = allocate_rings(RingConfig(1024, 4), device_arena=arena)
    b = allocate_rings(RingConfig(1024, 4), device_arena=arena)
    assert a.device_base != b.device_base
    off = a.reserve_payload(32)
    a.payload_view(off, 32)[:] = b"x" * 32
    assert bytes(b.payload_view(0, 32)) == b"\x00" * 32
    assert bytes(a.payload_view(off, 32)) == b"x" * 32
    with pytest.raises(AllocationError):
        allocate_rings(RingConfig(1024, 4), device_arena=Arena(capacity=512))


def test_bad_lengths_and_config():
    ring = allocate_rings(RingConfig(256, 4))
    for bad in (0, 24, 512):
        with pytest.raises(ValueError):
            ring.reserve_payload(bad)
    with pytest.raises(ConfigError):
        RingConfig(payload_capacity=100, meta_slots=4)


def test_tail_end_skip_marks_dead_bytes():
    """test_rings.py:107-133 on the device allocator."""
    ring = allocate_rings(RingConfig(128, 8))
    first, second = ring.reserve_payload(48), ring.reserve_payload(48)
    assert (first, second) == (0, 48)
    with pytest.raises(PayloadRingFull):
        ring.reserve_payload(48)
    assert ring.occupancy == 96
    ring.release_payload(first, 48)
    third = ring.reserve_payload(48)
    assert third == 0
    assert ring.occupancy == 48 + 32 + 48
    assert ring.dead_created == 32
    ring.release_payload(second, 48)
    ring.release_payload(third, 48)
    assert ring.dead_reclaimed == 32
    assert ring.occupancy == 0


def test_empty_ring_resets_to_offset_zero():
    ring = allocate_rings(RingConfig(128, 8))
    first = ring.reserve_payload(96)
    ring.release_payload(first, 96)
    assert ring.would_fit([128])
    assert ring.reserve_payload(128) == 0
    assert ring.occupancy == 128 and ring.dead_created == 0
    ring.release_payload(0, 128)
    assert ring.occupancy == 0


def test_reset_then_wrapped_decisions():
    """After an empty reset the tail is 0 until the host releases past it."""
    ring = allocate_rings(RingConfig(128, 8))
    a = ring.reserve_payload(96)
    ring.release_payload(a, 96)
    b = ring.reserve_payload(48)          # reset: offset 0
    assert b == 0
    assert ring.state().payload_tail == 0
    assert ring.reserve_payload(64) == 48  # end space from head 48
    with pytest.raises(PayloadRingFull):
        ring.reserve_payload(32)


def test_out_of_order_release_detected():
    ring = allocate_rings(RingConfig(256, 8))
    a, b = ring.reserve_payload(32), ring.reserve_payload(32)
    with pytest.raises(OutOfOrderRelease):
        ring.release_payload(b, 32)
    ring.release_payload(a, 32)
    ring.release_payload(b, 32)
    with pytest.raises(OutOfOrderRelease):
        ring.release_payload(0, 32)


def test_publish_poll_round_trip_and_sentinel_reuse():
    ring = allocate_rings(RingConfig(1024, 2))
    off = ring.reserve_payload(48)
    assert ring.publish(Descriptor(off, 48, hook_id=3, step_seq=9)) == 0
    (d,) = ring.poll_ready(4)
    assert (d.payload_offset, d.payload_len, d.hook_id, d.step_seq,
            d.ready_seq) == (off, 48, 3, 9, 0)
    ring.release_payload(off, 48)
    for i in range(1, 5):
        o = ring.reserve_payload(16)
        assert ring.publish(Descriptor(o, 16, 0, i)) == i
        assert ring.poll_ready(1)[0].ready_seq == i
        ring.release_payload(o, 16)


def test_meta_ring_full_is_backpressure():
    ring = allocate_rings(RingConfig(1024, 2))
    for i in range(2):
        ring.publish(Descriptor(ring.reserve_payload(16), 16, 0, i))
    off = ring.reserve_payload(16)
    with pytest.raises(MetaRingFull):
        ring.publish(Descriptor(off, 16, 0, 2))
    ring.poll_ready(1)
    ring.publish(Descriptor(off, 16, 0, 2))


def test_meta_slots_hold_wire_layout():
    """Device-written slot bytes 0..31 equal the reference pack()."""
    import ctypes as C

    from paper_2605_11093_b200 import _native as N
    ring = allocate_rings(RingConfig(1024, 4))
    off = ring.reserve_payload(32)
    ring.publish(Descriptor(off, 32, 0x01020304, 0x05060708))
    p = C.c_void_p()
    N.check(N.lib().tf_ring_meta_ptr(ring.handle, C.byref(p)))
    raw = C.string_at(p.value, DESCRIPTOR_SIZE)
    assert raw[:32] == Descriptor(off, 32, 0x01020304, 0x05060708, 0).pack()[:32]
    ring.poll_ready(1)
    raw = C.string_at(p.value, DESCRIPTOR_SIZE)
    assert int.from_bytes(raw[24:32], "little") == READY_SENTINEL


def test_would_fit_matches_reality():
    ring = allocate_rings(RingConfig(128, 4))
    ring.reserve_payload(96)
    assert ring.would_fit([16])
    assert not ring.would_fit([48])
    assert not ring.would_fit([16, 32])
    assert ring.would_fit([16, 16])
    assert not ring.would_fit([16, 16], meta_entries=5)


def _replay(script):
    ring = allocate_rings(RingConfig(script["capacity"], script["meta_slots"]))
    for op in script["ops"]:
        kind = op[0]
        if kind == "R":
            _, length, want = op
            if want is None:
                with pytest.raises(PayloadRingFull):
                    ring.reserve_payload(length)
            else:
                assert ring.reserve_payload(length) == want, op
        elif kind == "P":
            _, off, length, hook, step, want = op
            if want is None:
                with pytest.raises(MetaRingFull):
                    ring.publish(Descriptor(off, length, hook, step))
            else:
                assert ring.publish(Descriptor(off, length, hook, step)) == want
        elif kind == "Q":
            got = ring.poll_ready(op[1])
            assert [[d.payload_offset, d.payload_len, d.hook_id, d.step_seq,
                     d.ready_seq] for d in got] == op[2]
        elif kind == "L":
            ring.release_payload(op[1], op[2])
        else:
            s = ring.state()
            assert [s.payload_head, s.payload_tail, s.occupancy, s.meta_head,
                    s.meta_tail, ring.dead_created,
                    ring.dead_reclaimed] == op[1:], op


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_golden_protocol_scripts(golden, idx):
    """1e4+ reference-recorded ops replayed on the device (criterion 2)."""
    _replay(golden("ring_script.json")[idx])


def test_golden_reserve_release_scripts(golden):
    for script in golden("reserve_release.json")[:60]:
        ring = allocate_rings(RingConfig(script["capacity"], 64))
        for kind, a, b, occ in script["ops"]:
            if kind == "R":
                if b is None:
                    with pytest.raises(PayloadRingFull):
                        ring.reserve_payload(a)
                else:
                    assert ring.reserve_payload(a) == b
            else:
                ring.release_payload(a, b)
            assert ring.occupancy == occ
