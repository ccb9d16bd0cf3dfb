"""Capture kernel modes beyond the raw copy, and large shapes.

* cast (north-star extension): bit-exact against oracle/cast_oracle.c;
* per-token reduction: fp64 restatement, 1e-3 relative (north star);
* token-row keep, strided (KV-slice) sources, deferred publish;
* full Llama-3-8B shapes: equal to torch's own gather of the kept rows
  (an independent implementation) and a checksum of checksums.
"""

import random
import zlib

import numpy as np
import pytest
import torch

import oracle
from paper_2605_11093_b200 import (DType, HookSpec, ModelSpec, RingConfig,
                                   TensorView, allocate_rings, capture,
                                   install_hooks)
from paper_2605_11093_b200.hooks import RowSource, capture_args, launch_capture
from paper_2605_11093_b200.rings import Descriptor

pytestmark = pytest.mark.gpu
TORCH = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}


def _drain_one(ring):
    (d,) = ring.poll_ready(1)
    data = bytes(ring.payload_view(d.payload_offset, d.payload_len))
    ring.release_payload(d.payload_offset, d.reserved_len)
    return d, data


@pytest.mark.parametrize("src", ["bf16", "f16", "f32"])
@pytest.mark.parametrize("dst", ["f32", "f16", "bf16", "f8e4m3", "f8e5m2"])
@pytest.mark.parametrize("hidden", [64, 72, 13])   # vector path, vector, scalar
def test_cast_bit_exact_vs_oracle(src, dst, hidden):
    if src == dst:
        pytest.skip("identity")
    g = torch.Generator().manual_seed(hash((src, dst, hidden)) & 0xFFFF)
    B, T = 5, 7
    x = (torch.randn(B, T, hidden, generator=g) * 30).to(TORCH[src])
    reg = install_hooks(ModelSpec(1, hidden), [HookSpec(
        "h", ("tokens", "hidden"), DType.of(src), cast_to=DType.of(dst))])
    ring = allocate_rings(RingConfig(1 << 20, 8))
    keep = [1, 0, 1, 1, 1]
    out = capture(reg, ring, 0, TensorView(x.cuda(), (B, T, hidden), DType.of(src)),
                  keep)
    _, got = _drain_one(ring)
    raw = x.view(torch.uint8).numpy().tobytes()
    per = T * hidden * DType.of(src).width
    kept = b"".join(raw[i * per:(i + 1) * per] for i in range(B) if keep[i])
    assert got == oracle.cast(kept, src, dst)
    assert out.bytes_written == len(got)


@pytest.mark.parametrize("src", ["bf16", "f16", "f32"])
@pytest.mark.parametrize("op", ["mean", "l2", "absmax", "rms", "stats"])
@pytest.mark.parametrize("hidden", [4096, 96, 37])
def test_per_token_reduce_vs_restatement(src, op, hidden):
    g = torch.Generator().manual_seed(hidden)
    B, T = 3, 9
    x = (torch.randn(B, T, hidden, generator=g) + 0.25).to(TORCH[src])
    reg = install_hooks(ModelSpec(1, hidden), [HookSpec(
        "h", ("tokens", "hidden"), DType.of(src), reduce=op)])
    ring = allocate_rings(RingConfig(1 << 20, 8))
    keep = [1, 0, 1]
    capture(reg, ring, 0, TensorView(x.cuda(), (B, T, hidden), DType.of(src)), keep)
    _, got = _drain_one(ring)
    k = 4 if op == "stats" else 1
    kept = x[[i for i in range(B) if keep[i]]].contiguous()
    want = np.array(oracle.reduce(kept.view(torch.uint8).numpy().tobytes(),
                                  kept.shape[0] * T, hidden, src, op),
                    dtype=np.float64).reshape(-1)
    have = np.frombuffer(got, dtype=np.float32).astype(np.float64)
    assert have.shape == want.shape == (kept.shape[0] * T * k,)
    # tolerance (north star): 1e-3 relative to the row's magnitude
    scale = np.maximum(np.abs(want), 1e-3 * np.abs(want).max())
    assert np.all(np.abs(have - want) <= 1e-3 * scale)


def test_token_row_keep_matches_index_select():
    """Token sampling: keep over (B*T) rows == torch mask gather."""
    B, T, H = 4, 64, 4096
    x = torch.randn(B, T, H, dtype=torch.bfloat16, device="cuda")
    mask = torch.zeros(B * T, dtype=torch.uint8)
    mask[::16] = 1
    mask[5] = 1
    ring = allocate_rings(RingConfig(64 << 20, 16))
    src = RowSource.token_rows(x)
    launch_capture(ring, capture_args(src, hook_id=3, keep_ptr=mask.cuda().data_ptr(),
                                      step_seq=7, full="raise"))
    torch.cuda.synchronize()
    ring.note_launch()
    d, got = _drain_one(ring)
    want = x.reshape(B * T, H)[mask.bool().cuda()].contiguous()
    assert got == want.view(torch.uint8).cpu().numpy().tobytes()
    assert d.n_rows == int(mask.sum()) and d.step_seq == 7 and d.hook_id == 3


def test_strided_kv_slice_source():
    """A step's tokens out of a (B, Hkv, S_max, D) cache: rows (b, h) of
    T*D contiguous elements at stride S_max*D, request-level keep."""
    B, Hkv, S, D, t0, T = 3, 8, 256, 128, 40, 17
    cache = torch.randn(B, Hkv, S, D, dtype=torch.bfloat16, device="cuda")
    view = cache[:, :, t0:t0 + T, :]
    keep = torch.tensor([1, 0, 1], dtype=torch.uint8, device="cuda")
    row = T * D * 2
    src = RowSource(view.data_ptr(), B, Hkv, row, view.stride(0) * 2,
                    view.stride(1) * 2, view)
    ring = allocate_rings(RingConfig(8 << 20, 8))
    launch_capture(ring, capture_args(src, hook_id=0, keep_ptr=keep.data_ptr(),
                                      keep_per_outer=True, full="raise"))
    torch.cuda.synchronize()
    ring.note_launch()
    _, got = _drain_one(ring)
    want = view[keep.bool()].contiguous().view(torch.uint8).cpu().numpy().tobytes()
    assert got == want


def test_deferred_publish_then_protocol_publish():
    reg = install_hooks(ModelSpec(1, 8), [HookSpec("h", (32,), DType.of("u8"))])
    ring = allocate_rings(RingConfig(1024, 4))
    data = bytes(range(64))
    out, desc = capture(reg, ring, 0, TensorView(data, (2, 32), DType.of("u8")),
                        (1, 1), step_seq=4, defer_publish=True)
    assert out.bytes_written == 64 and ring.ready_entries() == 0
    assert isinstance(desc, Descriptor) and desc.capture_seq > 0
    assert ring.publish(desc) == 0
    d, got = _drain_one(ring)
    assert got == data and d.step_seq == 4


@pytest.mark.parametrize("keep_mode", ["all", "drop_recent_half", "sparse_rows"])
def test_llama_shapes_equal_torch_gather(keep_mode):
    """Full configs[1] shapes (8x512x14336 bf16, 112 MiB): the captured bytes
    equal torch's gather of the kept rows; checksum of checksums per row."""
    B, T, F = 8, 512, 14336
    x = torch.randn(B, T, F, dtype=torch.bfloat16, device="cuda")
    ring = allocate_rings(RingConfig(256 << 20, 16))
    if keep_mode == "sparse_rows":
        mask = torch.zeros(B * T, dtype=torch.uint8, device="cuda")
        mask[torch.randperm(B * T, device="cuda")[:700]] = 1
        src = RowSource.token_rows(x)
        args = capture_args(src, hook_id=1, keep_ptr=mask.data_ptr(), full="raise")
        want = x.reshape(B * T, F)[mask.bool()]
    else:
        keep = torch.ones(B, dtype=torch.uint8, device="cuda")
        if keep_mode == "drop_recent_half":
            keep[B // 2:] = 0
        src = RowSource(x.data_ptr(), B, T, F * 2, x.stride(0) * 2, F * 2, x)
        args = capture_args(src, hook_id=1, keep_ptr=keep.data_ptr(),
                            keep_per_outer=True, full="raise")
        want = x[keep.bool()].reshape(-1, F)
    launch_capture(ring, args)
    torch.cuda.synchronize()
    ring.note_launch()
    (d,) = ring.poll_ready(1)
    got = ring.payload_view(d.payload_offset, d.payload_len).tensor
    want_b = want.contiguous().view(torch.uint8).reshape(-1)
    assert got.numel() == want_b.numel()
    assert torch.equal(got, want_b)
    rows = got.view(-1, F * 2).cpu().numpy()
    cks = [zlib.crc32(r.tobytes()) for r in rows[:: max(1, len(rows) // 64)]]
    ref = [zlib.crc32(r.tobytes()) for r in
           want_b.view(-1, F * 2).cpu().numpy()[:: max(1, len(rows) // 64)]]
    assert zlib.crc32(bytes(str(cks), "ascii")) == zlib.crc32(bytes(str(ref), "ascii"))


def test_random_shapes_vs_oracle():
    """Odd widths, strides and keep patterns (vector widths 16/8/4/2/1)."""
    rng = random.Random(4242)
    ring = allocate_rings(RingConfig(8 << 20, 64))
    for case in range(120):
        outer = rng.randint(1, 9)
        mid = rng.randint(1, 6)
        row = rng.choice([1, 2, 3, 4, 6, 8, 12, 16, 24, 48, 100, 160, 1000])
        pad_mid = rng.randint(0, 3) * rng.choice([1, 2, 16])
        s_mid = row + pad_mid
        s_outer = s_mid * mid + rng.randint(0, 2) * 16
        base_off = rng.choice([0, 1, 2, 4, 8, 16])
        n = base_off + s_outer * outer + 64
        buf = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
        per_outer = rng.random() < 0.5
        units = outer if per_outer else outer * mid
        keep = [rng.randint(0, 1) for _ in range(units)]
        kt = torch.tensor(keep, dtype=torch.uint8, device="cuda")
        src = RowSource(buf.data_ptr() + base_off, outer, mid, row, s_outer,
                        s_mid, buf)
        launch_capture(ring, capture_args(src, hook_id=case, keep_ptr=kt.data_ptr(),
                                          keep_per_outer=per_outer, full="raise"))
        torch.cuda.synchronize()
        ring.note_launch()
        want = oracle.gather(buf.cpu().numpy().tobytes()[base_off:], outer, mid,
                             row, s_outer, s_mid, keep, per_outer)
        if not want:
            assert ring.ready_entries() == 0
            continue
        d, got = _drain_one(ring)
        assert got == want, case
