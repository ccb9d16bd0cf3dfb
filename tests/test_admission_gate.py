"""Host admission gate of eager captures under completeness
(hookpoint.Observer._admit), exercised without a GPU: the ring, the release
counter and the exporter are stand-ins. The gate must admit whenever the
ring is empty or the bytes in flight leave room for the capture plus one
dead skip, wait for releases otherwise, and raise PayloadRingFull when the
consumer stops releasing."""

import types

import pytest

from paper_2605_11093_b200 import hookpoint
from paper_2605_11093_b200.errors import PayloadRingFull


class FakeLib:
    """tf_ring_host_released returning a scripted sequence of totals."""

    def __init__(self, totals):
        self.totals = list(totals)
        self.calls = 0

    def tf_ring_host_released(self, handle, ref, _consumed):
        self.calls += 1
        ref._obj.value = self.totals.pop(0) if len(self.totals) > 1 else self.totals[0]
        return 0


def fake_observer(capacity, timeout=0.2):
    obs = types.SimpleNamespace(
        _max_need=0, _launched=0, _released=0, wait_timeout=timeout,
        gate_waits=0, gate_wait_s=0.0, side_stream=None,
        ring=types.SimpleNamespace(capacity=capacity, handle=1),
        exporter=types.SimpleNamespace(_check_bg=lambda: None),
        join=lambda stream=None: None, _seal=lambda stream=None: None)
    return obs


def admit(obs, need):
    return hookpoint.Observer._admit(obs, need)


def test_empty_ring_admits_without_polling(monkeypatch):
    lib = FakeLib([0])
    monkeypatch.setattr(hookpoint.N, "lib", lambda: lib)
    obs = fake_observer(1 << 20)
    admit(obs, 900 << 10)          # larger than half the ring: fine when empty
    assert obs._launched == 900 << 10 and lib.calls == 0 and obs.gate_waits == 0


def test_room_for_capture_plus_dead_skip(monkeypatch):
    lib = FakeLib([0])
    monkeypatch.setattr(hookpoint.N, "lib", lambda: lib)
    obs = fake_observer(1000)
    admit(obs, 200)                # in flight 0
    admit(obs, 200)                # 200 + 200 + max 200 <= 1000
    admit(obs, 200)                # 400 + 200 + 200 <= 1000
    assert obs._launched == 600 and lib.calls == 0


def test_waits_for_releases_then_admits(monkeypatch):
    # in flight 600 of a 1000-byte ring: a 300-byte capture needs
    # 600 - released + 300 + 300 <= 1000, i.e. 200 bytes released
    lib = FakeLib([0, 100, 150, 200])
    monkeypatch.setattr(hookpoint.N, "lib", lambda: lib)
    obs = fake_observer(1000, timeout=5.0)
    obs._launched = 600
    obs._max_need = 200
    admit(obs, 300)
    assert obs._released == 200 and obs._launched == 900
    assert obs.gate_waits == 1 and lib.calls == 4


def test_raises_when_nothing_is_released(monkeypatch):
    lib = FakeLib([0])
    monkeypatch.setattr(hookpoint.N, "lib", lambda: lib)
    obs = fake_observer(1000, timeout=0.05)
    obs._launched = 900
    obs._max_need = 100
    # the re-base after 0.25 s needs a device; keep the timeout below it
    with pytest.raises(PayloadRingFull):
        admit(obs, 100)
