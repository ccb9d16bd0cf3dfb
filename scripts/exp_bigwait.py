"""Ring-full regime with oversize captures (the SURVEY C2 prefill shape):
alternating 896 MiB / 256 MiB captures into a 2 GiB ring under TF_FULL_WAIT,
drained concurrently through 128 MiB staging buffers (split_oversize).
Every capture after the first two waits on the device for space the stager
frees. Prints progress every second and exits 1 if the ring stops moving.

usage: python scripts/exp_bigwait.py [--n 24] [--timeout 60]
"""
import argparse
import json
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11093_b200 import DrainConfig, ExportPipeline, RingConfig, RingPair  # noqa: E402
from paper_2605_11093_b200.hooks import RowSource, capture_args, launch_capture  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=24)
ap.add_argument("--timeout", type=float, default=60.0)
ap.add_argument("--ring-mib", type=int, default=2048)
ap.add_argument("--sizes-mib", default="896,256")
ap.add_argument("--default-stream", action="store_true",
                help="launch on the legacy default stream (as HF eager code does)")
ap.add_argument("--host-op", default="none",
                choices=["none", "pin", "empty_cache", "malloc", "item", "sink"],
                help="what the main thread does while the captures wait on the device: "
                     "pin = pinned host allocations, empty_cache = cudaFree of cached "
                     "blocks, malloc = new device allocations, item = a blocking D2H "
                     "read on another stream, sink = a Python NullSink consumer thread")
args = ap.parse_args()

dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
B = 64
ring = RingPair(RingConfig(payload_capacity=args.ring_mib << 20, meta_slots=4096), device=0)
pipe = ExportPipeline(ring, DrainConfig(min_ready_entries=1, min_ready_bytes=1, max_wait=1e-4,
                                        staging_buffer_size=128 << 20, staging_buffer_count=12,
                                        split_oversize=True, discard_paged=True))
keep = torch.ones(B, dtype=torch.uint8, device=dev)
sizes = [int(x) << 20 for x in args.sizes_mib.split(",")]
xs = [torch.empty(n, dtype=torch.uint8, device=dev).random_() for n in sizes]
s = torch.cuda.default_stream(dev) if args.default_stream else torch.cuda.Stream()
if args.host_op == "sink":
    from paper_2605_11093_b200.sinks import NullSink
    pipe.start(sink=NullSink())
else:
    pipe.start(sink=None)
done = threading.Event()
t0 = time.perf_counter()


def meta_slots():
    """(ready_seq, CTA count, completion counter) of the first n slots of the
    host mirror (refreshed by tf_ring_meta_ptr; 128-B stride)."""
    import ctypes as C
    import struct
    from paper_2605_11093_b200 import _native as N
    p = C.c_void_p()
    N.check(N.lib().tf_ring_meta_ptr(ring.handle, C.byref(p)))
    raw = C.string_at(p.value, 128 * args.n)
    out = []
    for i in range(args.n):
        w = struct.unpack_from("<8Q", raw, 128 * i)
        done = struct.unpack_from("<I", raw, 128 * i + 64)[0]
        seq = w[3] if w[3] != 0xFFFFFFFFFFFFFFFF else -1
        out.append((seq, (w[5] & 0xFFFFFFFF) >> 16, done))
    return out


def watch():
    last = None
    still = 0
    while not done.wait(1.0):
        st = pipe.stats()
        key = (st.get("bytes_drained"), st.get("batches_staged"))
        print(json.dumps({"t": round(time.perf_counter() - t0, 1), "stager": st,
                          "slots": meta_slots()}), flush=True)
        still = still + 1 if key == last else 0
        last = key
        if still >= 10:
            print("STALL: stager made no progress for 10 s", flush=True)


th = threading.Thread(target=watch, daemon=True)
th.start()
with torch.cuda.stream(s):
    for i in range(args.n):
        x = xs[i % len(xs)]
        row = 8192 if x.numel() // B >= 8192 else x.numel() // B
        mid = x.numel() // B // row
        a = capture_args(RowSource(x.data_ptr(), B, mid, row, mid * row, row, x), hook_id=i % 2,
                         keep_ptr=keep.data_ptr(), keep_per_outer=True, step_seq=i, full="wait")
        launch_capture(ring, a, s)
ev = torch.cuda.Event()
ev.record(s)
deadline = time.perf_counter() + args.timeout
other = torch.cuda.Stream()
keepalive = []
k = 0
while not ev.query() and time.perf_counter() < deadline:
    k += 1
    if args.host_op == "pin":
        keepalive.append(torch.empty(64 << 20, dtype=torch.uint8).pin_memory())
        if len(keepalive) > 4:
            keepalive.pop(0)
    elif args.host_op == "empty_cache":
        keepalive.append(torch.empty(256 << 20, dtype=torch.uint8, device=dev))
        keepalive.clear()
        torch.cuda.empty_cache()
    elif args.host_op == "malloc":
        keepalive.append(torch.empty((256 + k) << 20, dtype=torch.uint8, device=dev))
        if len(keepalive) > 4:
            keepalive.pop(0)
    elif args.host_op == "item":
        with torch.cuda.stream(other):
            torch.ones(1, device=dev).sum().item()
    time.sleep(0.05)
print(json.dumps({"host_op": args.host_op, "host_op_iterations": k}), flush=True)
ok = ev.query()
print(json.dumps({"captures_done": ok, "elapsed_s": time.perf_counter() - t0}), flush=True)
if ok:
    pipe.flush(args.timeout)
    st = ring.state()
    print(json.dumps({"drops": st.drops, "stalls": st.stall_events, "errors": st.device_errors,
                      "bytes_released": ring.bytes_released,
                      "bytes_expected": sum(sizes[i % len(sizes)] for i in range(args.n)),
                      "stager": pipe.stats()}), flush=True)
done.set()
if not ok:
    os._exit(1)
pipe.close()
ring.close()
