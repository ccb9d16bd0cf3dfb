"""Capture-kernel phase breakdown with the trace build (TF_TRACE).

Per launch (averaged over a graph replay of N back-to-back captures):
entry spread (last CTA start - first), offset known (latest CTA), copy
done (latest CTA), publish done (last CTA), and the gap between the end
of one launch and the first CTA of the next.

usage: python -m paper_2605_11093_b200.build_ext --variant=trace
       python scripts/exp_trace.py [--sizes-mib 1,32,112]
"""
import argparse
import ctypes as C
import os
import sys

os.environ.setdefault("TF_LIB_VARIANT", "trace")
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11093_b200 import DrainConfig, ExportPipeline, RingConfig, RingPair  # noqa: E402
from paper_2605_11093_b200 import _native as N  # noqa: E402
from paper_2605_11093_b200.hooks import RowSource, capture_args, launch_capture  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32)
ap.add_argument("--sizes-mib", default="1,8,32,112")
ap.add_argument("--sizes-kb", default="", help="overrides --sizes-mib (KiB)")
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--rows", type=int, default=1, help="rows per batch element (T)")
args = ap.parse_args()

lib = N.lib()
import numpy as np  # noqa: E402

stamps = np.zeros((64, 1024, 6), dtype=np.uint64)
pub = np.zeros((64, 2), dtype=np.uint64)


def trace(n):
    """Phases of the n most recent launches (us, relative to first entry)."""
    assert lib.tf_debug_trace(stamps.ctypes.data_as(C.c_void_p), pub.ctypes.data_as(C.c_void_p)) == 0
    order = np.argsort(pub[:, 0])[-n:]
    rows = []
    for slot in order:
        g = int(pub[slot, 1])
        if g == 0:
            continue
        st = stamps[slot, 1:g].astype(np.int64)  # CTA 0 is the controller (no copy stamps)
        e0 = st[:, 0].min()
        rows.append(((st[:, 0].max() - e0), (st[:, 1].max() - e0), (st[:, 2].max() - e0),
                     (int(pub[slot, 0]) - e0), (st[:, 3].max() - e0), (st[:, 4].max() - e0),
                     (st[:, 5].max() - e0), e0, int(pub[slot, 0])))
    if not rows:
        return np.full(7, np.nan), float("nan")
    r = np.array(rows, dtype=np.float64)
    allst = np.unique(stamps[order, :, 0][stamps[order, :, 0] > 0])
    d = np.diff(allst)
    print("  timer granularity (min nonzero stamp delta, ns):", int(d[d > 0].min()) if d.size else None)
    gaps = r[1:, 7] - r[:-1, 8]
    return r[:, :7].mean(axis=0) / 1e3, gaps.mean() / 1e3


dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
ring = RingPair(RingConfig(payload_capacity=24 << 30, meta_slots=4096), device=0)
pipe = ExportPipeline(ring, DrainConfig(min_ready_entries=1, min_ready_bytes=1, max_wait=1e-4,
                                        staging_buffer_size=256 << 20, staging_buffer_count=4,
                                        discard_paged=True))
B = args.batch
keep = torch.ones(B, dtype=torch.uint8, device=dev)
s = torch.cuda.Stream()


def drain():
    pipe.start(sink=None)
    pipe.flush(300)
    pipe.stop(flush=True)


sizes = [int(x) << 10 for x in args.sizes_kb.split(",")] if args.sizes_kb else \
    [int(x) << 20 for x in args.sizes_mib.split(",")]
for nbytes in sizes:
    mib = nbytes / 1048576
    T = args.rows
    row = nbytes // (B * T)
    nsrc = max(1, min(args.n, (1 << 30) // nbytes))
    xs = [torch.empty(nbytes, dtype=torch.uint8, device=dev).random_() for _ in range(nsrc)]
    caps = [capture_args(RowSource(xs[i % nsrc].data_ptr(), B, T, row, row * T, row, xs[i % nsrc]),
                         hook_id=i, keep_ptr=keep.data_ptr(), keep_per_outer=True,
                         step_seq=0, full="wait") for i in range(args.n)]
    with torch.cuda.stream(s):
        for a in caps:
            launch_capture(ring, a, s)
    s.synchronize()
    drain()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for a in caps:
            launch_capture(ring, a, s)
    drain()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record()
        g.replay()
        e1.record()
    s.synchronize()
    ph, gap = trace(args.n)
    span = e0.elapsed_time(e1) * 1e3 / args.n
    print(f"{mib:8.3f} MiB  span/launch {span:7.2f} us | entry spread {ph[0]:6.2f} "
          f"| scan {ph[4]:5.2f} | fastplan {ph[5]:5.2f} | table {ph[6]:5.2f} | offset known {ph[1]:6.2f} | copy done {ph[2]:6.2f} | published {ph[3]:6.2f} "
          f"| gap to next {gap:6.2f} | ideal {2 * nbytes / 6545.9e3:6.2f}", flush=True)
    del g, xs, caps
    drain()
pipe.close()
ring.close()
