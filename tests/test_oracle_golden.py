"""Pin the CPU oracle (oracle/) against golden vectors recorded from the
reference itself (tests/golden/make_golden.py) and against the reference's
own known-answer tests. CPU only."""

import hashlib
import random
import struct

import numpy as np
import pytest

import oracle
from oracle import workload as W


def h32(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()[:32]


def test_descriptor_pack_matches_reference(golden):
    for case in golden("descriptors.json"):
        assert oracle.desc_pack(*case["fields"]).hex() == case["hex"]


def test_descriptor_known_answers():
    """PKG/tests/test_rings.py:33-57."""
    raw = oracle.desc_pack(0x1122334455667788, 0xAABBCCDDEEFF0011, 0x01020304,
                           0x05060708, 0x1111222233334444)
    assert raw[0:8] == (0x1122334455667788).to_bytes(8, "little")
    assert raw[8:16] == (0xAABBCCDDEEFF0011).to_bytes(8, "little")
    assert raw[16:20] == (0x01020304).to_bytes(4, "little")
    assert raw[20:24] == (0x05060708).to_bytes(4, "little")
    assert raw[24:32] == (0x1111222233334444).to_bytes(8, "little")
    assert raw[32:64] == bytes(32) and len(raw) == 64


def test_allocator_known_answers():
    """PKG/tests/test_rings.py:107-164 on the oracle ring."""
    r = oracle.OracleRing(128, 8)
    assert r.reserve(48)[:2] == (0, 0) and r.reserve(48)[:2] == (0, 48)
    assert r.reserve(48)[0] == oracle.PAYLOAD_FULL
    assert r.state()["used"] == 96
    assert r.release(0, 48) == 0
    rc, off, dead = r.reserve(48)
    assert (rc, off, dead) == (0, 0, 32) and r.state()["used"] == 128
    assert r.release(48, 48) == 0 and r.release(0, 48) == 0
    assert r.state()["dead_reclaimed"] == 32 and r.state()["used"] == 0
    r = oracle.OracleRing(128, 8)
    r.reserve(96)
    r.release(0, 96)
    assert r.would_fit([128])
    assert r.reserve(128)[:2] == (0, 0)
    r = oracle.OracleRing(128, 4)
    r.reserve(96)
    assert r.would_fit([16]) and not r.would_fit([48])
    assert not r.would_fit([16, 32]) and r.would_fit([16, 16])
    assert not r.would_fit([16, 16], meta_entries=5)


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_protocol_scripts_replay_on_oracle(golden, idx):
    script = golden("ring_script.json")[idx]
    r = oracle.OracleRing(script["capacity"], script["meta_slots"])
    for op in script["ops"]:
        if op[0] == "R":
            rc, off, _ = r.reserve(op[1])
            assert (None if rc else off) == op[2], op
        elif op[0] == "P":
            rc, seq = r.publish(*op[1:5])
            assert (None if rc else seq) == op[5], op
        elif op[0] == "Q":
            rc, got = r.poll(op[1])
            assert rc == 0 and [list(g) for g in got] == op[2]
        elif op[0] == "L":
            assert r.release(op[1], op[2]) == 0
        else:
            s = r.state()
            assert [s["head"], s["tail"], s["used"], s["meta_head"],
                    s["meta_tail"], s["dead_created"],
                    s["dead_reclaimed"]] == op[1:], op


def test_reserve_release_scripts_on_oracle(golden):
    for script in golden("reserve_release.json"):
        r = oracle.OracleRing(script["capacity"], 64)
        for kind, a, b, occ in script["ops"]:
            if kind == "R":
                rc, off, _ = r.reserve(a)
                assert (None if rc else off) == b
            else:
                assert r.release(a, b) == 0
            assert r.state()["used"] == occ


def test_gather_cases_on_oracle(golden):
    """Criterion-3 recipe replayed; reference output hashes must match."""
    rng = random.Random(7)
    widths = (1, 2, 4, 8)
    for want in golden("gather_cases.json"):
        batch = rng.randint(1, 8)
        tokens = rng.randint(1, 9)
        feat = rng.randint(1, 33)
        width = rng.choice(widths)
        size = tokens * feat * width
        data = rng.randbytes(batch * size)
        keep = [rng.randint(0, 1) for _ in range(batch)]
        assert keep == want["keep"] and width == want["width"]
        got = oracle.gather(data, batch, 1, size, size, size, keep, True)
        assert len(got) == want["len"] and h32(got) == want["sha"]


def test_gather_generalised_rows():
    """Strided (outer, mid) rows and per-row keep equal numpy indexing."""
    rng = np.random.default_rng(3)
    outer, mid, row = 5, 7, 24
    buf = rng.integers(0, 256, size=(outer, 9, 40), dtype=np.uint8)
    keep = rng.integers(0, 2, size=outer * mid).astype(bool)
    got = oracle.gather(buf.tobytes(), outer, mid, row, 9 * 40, 40,
                        keep.tolist(), per_outer=False)
    want = buf[:, :mid, :row].reshape(outer * mid, row)[keep].tobytes()
    assert got == want


def test_workload_content_matches_reference(golden):
    for c in golden("workload.json")["payloads"]:
        data = W.request_payload(c["seed"], c["name"], c["layer"], c["rid"],
                                 c["step"], c["nbytes"])
        assert h32(data) == c["sha"]


def test_schedule_and_reference_records(golden):
    g = golden("workload.json")
    wl = g["workload"]
    sched = W.build_schedule(wl["batch"], wl["prefill_tokens"],
                             wl["decode_steps"], wl["seed"], wl["arrival"])
    assert [[s, k, [[r.request_id, r.arrival_index, r.prompt, r.tokens,
                     r.token_start] for r in b]] for s, k, b in sched] == \
        g["schedule"]
    import zlib
    hooks = [(f"resid[{L}]", L, (None, wl["hidden"]), 2)
             for L in range(wl["layers"])] + [("logits", None, (None, 8), 4)]
    want = g["records"]
    got = []
    for seq, _, batch in sched:
        for name, layer, (_, feat), width in hooks:
            for r in batch:
                n = r.tokens * feat * width
                data = W.request_payload(wl["seed"], name, layer, r.request_id,
                                         seq, n)
                got.append([r.request_id, name, layer, seq,
                            [r.token_start, r.token_start + r.tokens],
                            [r.tokens, feat], "bf16" if width == 2 else "f32",
                            zlib.crc32(data)])
    assert got == want


def test_cast_oracle_known_values():
    f32 = lambda xs: struct.pack(f"<{len(xs)}f", *xs)  # noqa: E731
    assert oracle.cast(f32([1.0, -2.0]), "f32", "bf16") == bytes.fromhex("803f00c0")
    assert oracle.cast(f32([1.0]), "f32", "f16") == bytes.fromhex("003c")
    assert oracle.cast(f32([448.0, 1000.0, -1e9]), "f32", "f8e4m3") == bytes([0x7E, 0x7E, 0xFE])
    assert oracle.cast(f32([57344.0, 1e9]), "f32", "f8e5m2") == bytes([0x7B, 0x7B])
    assert oracle.cast(f32([2.0 ** -9]), "f32", "f8e4m3") == bytes([0x01])   # min subnormal
    assert oracle.cast(f32([65520.0]), "f32", "f16") == bytes.fromhex("007c")  # -> inf


@pytest.mark.parametrize("dst", ["bf16", "f16", "f8e4m3", "f8e5m2"])
def test_cast_oracle_matches_torch_rne(dst):
    """Independent check: torch's CPU conversions (RNE) on in-range values."""
    import torch
    g = torch.Generator().manual_seed(11)
    x = torch.randn(4096, generator=g) * 8
    if dst.startswith("f8"):
        lim = 440.0 if dst == "f8e4m3" else 57000.0
        x = x.clamp(-lim, lim)
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16,
           "f8e4m3": torch.float8_e4m3fn, "f8e5m2": torch.float8_e5m2}[dst]
    want = x.to(tdt).view(torch.uint8).numpy().tobytes()
    got = oracle.cast(x.numpy().astype("<f4").tobytes(), "f32", dst)
    assert got == want


def test_reduce_oracle_against_numpy():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((6, 384)).astype(np.float32)
    out = oracle.reduce(x.tobytes(), 6, 384, "f32", "stats")
    for r in range(6):
        row = x[r].astype(np.float64)
        assert out[r][0] == pytest.approx(row.mean(), rel=1e-6, abs=1e-7)
        assert out[r][1] == pytest.approx(np.sqrt((row ** 2).sum()), rel=1e-6)
        assert out[r][2] == row.min() and out[r][3] == row.max()
