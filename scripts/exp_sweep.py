"""Capture-kernel size sweep: per-launch time of N back-to-back captures
replayed as a CUDA graph into an empty ring (staging idle), against a
plain D2D copy of the same bytes (torch copy_ and cudaMemcpyAsync) in the
same graph shape. Separates fixed per-launch cost from the bandwidth slope.

usage: python scripts/exp_sweep.py [--n 16] [--sizes-mib 1,4,16,32,64,112,224]
"""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11093_b200 import DrainConfig, ExportPipeline, RingConfig, RingPair  # noqa: E402
from paper_2605_11093_b200.hooks import RowSource, capture_args, launch_capture  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16)
ap.add_argument("--sizes-mib", default="1,4,16,32,64,112,224")
ap.add_argument("--sizes-kb", default="", help="overrides --sizes-mib (KiB)")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--row-bytes", type=int, default=0,
                help="source rows of this many bytes (e.g. 8192 = a Llama resid row); "
                     "0 = one row per batch element")
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--out", default="gpurun_out/sweep.json")
ap.add_argument("--busy-d2h", action="store_true",
                help="a 256 MiB pinned D2H loops on another stream during the timed "
                     "replays (PCIe saturated, as while the staging engine drains)")
ap.add_argument("--sealed", action="store_true",
                help="TF_CAP_SEALED captures (completion by stream order), one seal per replay")
args = ap.parse_args()

dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6545.9
B = args.batch
res = []
ring = RingPair(RingConfig(payload_capacity=24 << 30, meta_slots=4096), device=0)
pipe = ExportPipeline(ring, DrainConfig(min_ready_entries=1, min_ready_bytes=1, max_wait=1e-4,
                                        staging_buffer_size=256 << 20, staging_buffer_count=4,
                                        discard_paged=True))
keep = torch.ones(B, dtype=torch.uint8, device=dev)
s = torch.cuda.Stream()


def drain():
    pipe.start(sink=None)
    pipe.flush(300)
    pipe.stop(flush=True)


class BusyD2H:
    """Background thread looping a pinned 256 MiB D2H on its own stream."""

    def __init__(self):
        import threading
        self.src = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        self.dst = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
        self.st = torch.cuda.Stream()
        self.stop = threading.Event()
        self.th = threading.Thread(target=self.run, daemon=True)

    def run(self):
        torch.cuda.set_device(dev)
        while not self.stop.is_set():
            with torch.cuda.stream(self.st):
                self.dst.copy_(self.src, non_blocking=True)
            self.st.synchronize()

    def __enter__(self):
        self.th.start()
        import time
        time.sleep(0.05)
        return self

    def __exit__(self, *exc):
        self.stop.set()
        self.th.join()


def seal():
    if args.sealed:
        ring.seal(s)


def timed_graph(fn, reps):
    with torch.cuda.stream(s):
        fn()  # warm
    seal()
    s.synchronize()
    drain()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    out = []
    for _ in range(reps):
        drain()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        busy = BusyD2H() if args.busy_d2h else None
        if busy:
            busy.__enter__()
        with torch.cuda.stream(s):
            e0.record()
            g.replay()
            e1.record()
        seal()
        s.synchronize()
        if busy:
            busy.__exit__()
        out.append(e0.elapsed_time(e1) * 1e3 / args.n)
    del g
    drain()
    return statistics.median(out)


sizes = [int(x) << 10 for x in args.sizes_kb.split(",")] if args.sizes_kb else \
    [int(x) << 20 for x in args.sizes_mib.split(",")]
for nbytes in sizes:
    mib = nbytes / 1048576
    row = args.row_bytes or nbytes // B
    mid = nbytes // B // row
    xs = [torch.empty(nbytes, dtype=torch.uint8, device=dev).random_() for _ in range(min(args.n, 4))]
    assert nbytes % B == 0
    dsts = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(min(args.n, 4))]
    caps = []
    for i in range(args.n):
        x = xs[i % len(xs)]
        src = RowSource(x.data_ptr(), B, mid, row, mid * row, row, x)
        caps.append(capture_args(src, hook_id=i, keep_ptr=keep.data_ptr(), keep_per_outer=True,
                                 step_seq=0, full="wait", sealed=args.sealed))

    def cap_step():
        for a in caps:
            launch_capture(ring, a, s)

    def copy_step():
        for i in range(args.n):
            dsts[i % len(dsts)].copy_(xs[i % len(xs)])

    t_cap = timed_graph(cap_step, args.reps)
    t_copy = timed_graph(copy_step, args.reps)
    ideal = 2 * nbytes / (PEAK * 1e9) * 1e6
    r = {"mib": mib, "row_bytes": row, "busy_d2h": args.busy_d2h, "capture_us": t_cap, "torch_copy_us": t_copy, "ideal_us": ideal,
         "capture_frac": ideal / t_cap, "copy_frac": ideal / t_copy}
    print(json.dumps(r), flush=True)
    res.append(r)
    del xs, dsts, caps
os.makedirs(os.path.dirname(args.out), exist_ok=True)
json.dump(res, open(args.out, "w"), indent=1)
pipe.close()
ring.close()
