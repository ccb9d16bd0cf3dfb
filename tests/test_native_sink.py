"""Native record sinks (csrc/sink.cpp) against the reference formats
(SRC/sinks.py:35-136): golden bytes, byte equality with the Python sinks,
ragged captures split like split_payload (SRC/exporter.py:306-327), crc32
over multi-chunk payloads, JSON escaping, and the exporter's batch path.
Host-only code: runs without a GPU."""

import io
import json
import os
import random
import zlib

import pytest

from paper_2605_11093_b200 import CaptureRecord, DType, MetaMismatch, TensorMeta
from paper_2605_11093_b200.exporter import split_payload
from paper_2605_11093_b200.sinks import (FileSink, NativeFileSink, NativeStreamSink,
                                         StreamSink, read_dataset, read_stream,
                                         records_to_stream_bytes)

BF16, F32, U8 = DType.of("bf16"), DType.of("f32"), DType.of("u8")


def _golden_records():
    return [CaptureRecord(7, "resid[2]", 2, 5, (4, 8), (4, 2), BF16, (0, 0), bytes(range(16))),
            CaptureRecord(9, "logits", None, 6, (8, 9), (1, 3), F32, (1, 0),
                          bytes(range(100, 112)))]


def _random_records(rng, n):
    out = []
    for i in range(n):
        rows, width = rng.randint(1, 6), rng.choice([1, 3, 8, 100])
        dt = rng.choice([U8, BF16, F32])
        name = rng.choice(["resid_post[3]", "mlp_act[0]", "attn \"q\"\\k", "héad\n☃", "\x01x"])
        payload = rng.randbytes(rows * width * dt.width)
        out.append(CaptureRecord(rng.randint(0, 1 << 40), name, rng.choice([None, 0, 31]),
                                 rng.randint(0, 1 << 31), (i, i + rows), (rows, width), dt,
                                 (rng.randint(0, 3), rng.randint(0, 3)), payload))
    return out


def test_native_dataset_matches_golden(golden, tmp_path):
    g = golden("sinks.json")
    with NativeFileSink(tmp_path / "ds") as sink:
        sink.write(_golden_records())
    assert (tmp_path / "ds" / "records.ndjson").read_text().splitlines() == g["lines"]
    assert read_dataset(tmp_path / "ds") == _golden_records()


def test_native_stream_matches_golden(golden, tmp_path):
    g = golden("sinks.json")
    path = tmp_path / "stream.bin"
    with open(path, "wb") as fh:
        with NativeStreamSink(fh) as sink:
            sink.write(_golden_records())
    data = path.read_bytes()
    assert data.hex() == g["stream_hex"]
    assert [h for h, _ in read_stream(io.BytesIO(data))] == [json.loads(x) for x in g["lines"]]


def test_native_equals_python_sinks_byte_for_byte(tmp_path):
    rng = random.Random(11)
    recs = _random_records(rng, 200)
    with FileSink(tmp_path / "py") as a:
        a.write(recs[:70])
        a.write(recs[70:])
    with NativeFileSink(tmp_path / "nat", threads=3) as b:
        b.write(recs[:70])
        b.write(recs[70:])
    for name in ("records.ndjson", "records.bin"):
        assert (tmp_path / "py" / name).read_bytes() == (tmp_path / "nat" / name).read_bytes()
    path = tmp_path / "s.bin"
    with open(path, "wb") as fh:
        with NativeStreamSink(fh, threads=2) as s:
            s.write(recs)
    assert path.read_bytes() == records_to_stream_bytes(recs)


def test_captures_split_like_split_payload(tmp_path):
    rng = random.Random(5)
    caps, expected = [], []
    for step in range(6):
        ids = tuple(rng.sample(range(1000), rng.randint(1, 5)))
        rows = tuple(rng.randint(0, 7) for _ in ids)
        base = TensorMeta("resid_post[0]", 0, step, ids, tuple((3, 3 + max(1, r)) for r in rows),
                          (max(rows) or 1, 64), BF16, (0, 1), row_counts=rows)
        for hook in ("resid_post[0]", "mlp_act[0]"):
            meta = base if hook == "resid_post[0]" else base.with_hook(hook, 0, (max(rows) or 1, 64), BF16)
            payload = rng.randbytes(meta.expected_payload_len)
            caps.append((meta, payload, None))
            expected += split_payload(meta, payload)
    with NativeFileSink(tmp_path / "ds") as sink:
        sink.write_captures(caps)
        assert (sink.records_written, sink.bytes_written) == (
            len(expected), sum(len(r.payload) for r in expected))
    assert read_dataset(tmp_path / "ds") == expected
    with FileSink(tmp_path / "py") as py:
        py.write(expected)
    assert (tmp_path / "py" / "records.ndjson").read_bytes() == \
        (tmp_path / "ds" / "records.ndjson").read_bytes()


def test_multichunk_crc_and_append(tmp_path):
    half = (9 << 20) + 7                    # > 2 crc chunks per record
    payload = os.urandom(2 * half)
    meta = TensorMeta("big", 1, 0, (1, 2), ((0, 1), (0, 1)), (1, half), U8)
    caps = [(meta, payload, None)]
    with NativeFileSink(tmp_path / "ds", threads=4) as s:
        s.write_captures(caps)
    with NativeFileSink(tmp_path / "ds") as s:  # reopened: appends
        s.write_captures(caps)
    hdrs = [json.loads(x) for x in (tmp_path / "ds" / "records.ndjson").read_text().splitlines()]
    blob = (tmp_path / "ds" / "records.bin").read_bytes()
    assert blob == payload * 2 and len(hdrs) == 4
    assert [h["payload_offset"] for h in hdrs] == [0, half, 2 * half, 3 * half]
    for h in hdrs:
        a, b = h["payload_offset"], h["payload_offset"] + h["payload_len"]
        assert zlib.crc32(blob[a:b]) == h["checksum"]


def test_length_mismatch_is_meta_mismatch(tmp_path):
    meta = TensorMeta("h", 0, 0, (1,), ((0, 2),), (2, 4), U8)
    with NativeFileSink(tmp_path / "ds") as s:
        with pytest.raises(MetaMismatch):
            s.write_captures([(meta, b"x" * 7, None)])


def test_exporter_uses_batch_path_only_for_sinks_that_define_it(tmp_path):
    from paper_2605_11093_b200.exporter import ExportPipeline
    from paper_2605_11093_b200.sinks import NullSink

    class Collect(NullSink):          # overrides write only: records path
        def write(self, recs):
            pass

    class Both(NullSink):
        def write(self, recs):
            pass

        def write_captures(self, caps):
            pass

    want = ExportPipeline._wants_captures
    assert want(NullSink()) and not want(Collect()) and want(Both())
    assert not want(FileSink(tmp_path / "a"))
    with NativeFileSink(tmp_path / "b") as s:
        assert want(s)


def test_pclmul_crc32_equals_zlib():
    """The sinks' CRC-32 (PCLMULQDQ folding, csrc/crc32_fast.h) is zlib.crc32
    for every length, alignment and running seed."""
    import ctypes as C
    import random
    import zlib

    from paper_2605_11093_b200 import _native as N
    rng = random.Random(11)
    buf = rng.randbytes(1 << 20)
    cbuf = C.create_string_buffer(buf, len(buf))
    base = C.addressof(cbuf)
    for n in list(range(0, 300)) + [rng.randrange(0, 1 << 19) for _ in range(300)]:
        off = rng.randrange(0, 4096)
        seed = rng.randrange(0, 1 << 32)
        want = zlib.crc32(buf[off:off + n], seed)
        assert N.lib().tf_sink_crc32(seed, base + off, n) == want, (n, off)


@pytest.mark.parametrize("where", ["tmp", "repo"])
def test_direct_io_dataset_equals_buffered(tmp_path, where):
    """NativeFileSink(direct=True): O_DIRECT sidecar through aligned bounce
    buffers (partial last block carried between batches, preallocation
    trimmed on close, append to an existing dataset) writes the same bytes
    as the buffered native sink and the Python FileSink."""
    import shutil
    import tempfile
    base = tmp_path if where == "tmp" else \
        __import__("pathlib").Path(tempfile.mkdtemp(dir=os.path.dirname(__file__)))
    try:
        rng = random.Random(21)
        recs = _random_records(rng, 300)
        big = CaptureRecord(3, "mlp_act[1]", 1, 9, (0, 5), (5, (3 << 20) + 3), U8, (0, 0),
                            rng.randbytes(5 * ((3 << 20) + 3)))
        batches = [recs[:1], recs[1:90], [big], recs[90:200], recs[200:]]
        with FileSink(base / "py") as a:
            for b in batches:
                a.write(b)
        with NativeFileSink(base / "dio", threads=4, direct=True) as d:
            for b in batches[:3]:
                d.write(b)
        with NativeFileSink(base / "dio", threads=3, direct=True) as d:  # reopen: append
            for b in batches[3:]:
                d.write(b)
        for name in ("records.ndjson", "records.bin"):
            assert (base / "py" / name).read_bytes() == (base / "dio" / name).read_bytes()
    finally:
        if where == "repo":
            shutil.rmtree(base, ignore_errors=True)
