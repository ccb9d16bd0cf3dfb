import statistics, sys, time, torch, os
sys.path.insert(0, ".")
from paper_2605_11093_b200 import DrainConfig, ExportPipeline, RingConfig, RingPair
from paper_2605_11093_b200.hooks import RowSource, capture_args, launch_capture
dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
B, T = 8, 512
xs = [torch.randn(B, T, 4096, device=dev, dtype=torch.bfloat16) for _ in range(32)]
ys = [torch.randn(B, T, 14336, device=dev, dtype=torch.bfloat16) for _ in range(32)]
keep = torch.ones(B, dtype=torch.uint8, device=dev)
s = torch.cuda.current_stream()
def run(ring, flags=0, n=64, label=""):
    ev = []
    k0 = ring.state().kernel_ns
    for i in range(n):
        x = (ys if i % 2 == 0 else xs)[i // 2 % 32]
        src = RowSource(x.data_ptr(), B, T, x.shape[-1]*2, x.stride(0)*2, x.shape[-1]*2, x)
        a = capture_args(src, hook_id=i, keep_ptr=keep.data_ptr(), keep_per_outer=True, full="wait")
        a.flags |= flags
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); launch_capture(ring, a, s); e1.record(s); ev.append((e0, e1))
    torch.cuda.synchronize(); ring.note_launch(s)
    kdev = (ring.state().kernel_ns - k0) / n / 1e3
    m = [a.elapsed_time(b)*1e3 for a, b in ev[0::2]]; r = [a.elapsed_time(b)*1e3 for a, b in ev[1::2]]
    print(f"{label:44s} ev mlp {statistics.median(m):7.1f} resid {statistics.median(r):7.1f} | dev avg {kdev:7.1f}", flush=True)
    return ev
def torch_copy_kernel_timing(label):
    # plain torch kernels while our stager drains: are they delayed too?
    ev = []
    for i in range(32):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); y2 = ys[i].clone(); e1.record(s); ev.append((e0, e1))
    torch.cuda.synchronize()
    print(f"{label:44s} torch clone mlp {statistics.median([a.elapsed_time(b)*1e3 for a,b in ev]):7.1f}", flush=True)
ring = RingPair(RingConfig(10 << 30, 4096), device=0)
pipe = ExportPipeline(ring, DrainConfig(min_ready_entries=1, min_ready_bytes=1, max_wait=1e-4, staging_buffer_size=128<<20, staging_buffer_count=6, discard_paged=True))
pipe.start(None)
torch_copy_kernel_timing("idle")
run(ring, 0, label="stager busy, host writes"); torch_copy_kernel_timing("after (D2H still draining)")
pipe.flush()
run(ring, 0x100, label="no host writes (nothing to drain)")
# make D2H busy via our stager with real captures, then time no-host-write captures
run(ring, 0, n=16, label="prime (16 captures)")
run(ring, 0x100, label="stager busy (primed), no host writes")
pipe.flush(); pipe.stop(); pipe.close()
