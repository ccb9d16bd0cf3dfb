"""Cast and per-token reduction captures (north-star extensions): device
time per launch against their algorithmic bytes:

    cast    kept * H * (w_in + w_out)      bf16 -> fp8 e4m3 / e5m2, f16, f32
    reduce  kept * H * w_in + kept * k * 4 mean / l2 / absmax / rms (k=1), stats (k=4)

on the resid_post shape of the bench (8 x 512 x 4096 bf16, 32 MiB) and the
mlp_act shape (8 x 512 x 14336, 112 MiB). Each configuration: 16 launches
replayed as a CUDA graph into an empty ring, median of 5 replays; the copy
capture of the same tensor beside it. One JSON line per configuration.
With --ncu, launches each op once (for ncu --set full) and exits.

usage: python scripts/exp_ops.py [--ncu]
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11093_b200 import DrainConfig, ExportPipeline, RingConfig, RingPair  # noqa: E402
from paper_2605_11093_b200 import _native as N  # noqa: E402
from paper_2605_11093_b200.hooks import RowSource, capture_args, launch_capture  # noqa: E402

dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists(
    "MEASURED_PEAKS.json") else 6545.9
B, T, n = 8, 512, 16
ring = RingPair(RingConfig(payload_capacity=8 << 30, meta_slots=4096), device=0)
pipe = ExportPipeline(ring, DrainConfig(min_ready_entries=1, min_ready_bytes=1, max_wait=1e-4,
                                        staging_buffer_size=256 << 20, staging_buffer_count=4,
                                        discard_paged=True))
keep = torch.ones(B, dtype=torch.uint8, device=dev)
s = torch.cuda.Stream()
W = {"bf16": 2, "f16": 2, "f32": 4, "f8e4m3": 1, "f8e5m2": 1}
K = {"mean": 1, "l2": 1, "absmax": 1, "rms": 1, "stats": 4}


def drain():
    pipe.start(sink=None)
    pipe.flush(300)
    pipe.stop(flush=True)


def args_of(x, op, out=None, red=None):
    H = x.shape[-1]
    src = RowSource(x.data_ptr(), B, T, H * 2, x.stride(0) * 2, H * 2, x)
    return capture_args(src, hook_id=0, op=op, in_dtype="bf16", out_dtype=out, reduce=red,
                        keep_ptr=keep.data_ptr(), keep_per_outer=True, full="wait")


def timed(a):
    def step():
        for _ in range(n):
            launch_capture(ring, a, s)
    with torch.cuda.stream(s):
        step()
    s.synchronize()
    drain()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    out = []
    for _ in range(5):
        drain()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record()
            g.replay()
            e1.record()
        s.synchronize()
        out.append(e0.elapsed_time(e1) * 1e3 / n)
    del g
    drain()
    return statistics.median(out)


acts = {"resid_post": torch.randn(B, T, 4096, device=dev, dtype=torch.bfloat16),
        "mlp_act": torch.randn(B, T, 14336, device=dev, dtype=torch.bfloat16)}
cases = [("copy", N.TF_OP_COPY, None, None)]
cases += [(f"cast_{o}", N.TF_OP_CAST, o, None) for o in ("f8e4m3", "f8e5m2", "f16", "f32")]
cases += [(f"reduce_{r}", N.TF_OP_REDUCE, None, r) for r in ("mean", "rms", "stats")]
if "--ncu" in sys.argv:
    for name, x in acts.items():
        for label, op, out, red in cases:
            launch_capture(ring, args_of(x, op, out, red), s)
    s.synchronize()
    print("ok")
    sys.exit(0)
for name, x in acts.items():
    elems = x.numel()
    for label, op, out, red in cases:
        us = timed(args_of(x, op, out, red))
        if op == N.TF_OP_COPY:
            alg = 2 * elems * 2
        elif op == N.TF_OP_CAST:
            alg = elems * (2 + W[out])
        else:
            alg = elems * 2 + B * T * K[red] * 4
        gbs = alg / (us * 1e-6) / 1e9
        print(json.dumps({"tensor": name, "op": label, "us_per_launch": us,
                          "algorithmic_bytes": alg, "achieved_gbs": gbs, "peak_gbs": PEAK,
                          "frac": gbs / PEAK}), flush=True)
pipe.close()
ring.close()
