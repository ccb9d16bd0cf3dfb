"""Does a busy D2H slow GPU work? GEMMs vs many small launches vs CUDA graph."""
import statistics, sys, time, torch
dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
s = torch.cuda.current_stream()
a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16); b = torch.randn_like(a)
x = torch.randn(1 << 18, device=dev)
def gemms():
    for _ in range(10): torch.mm(a, b)
def smalls():
    for _ in range(2000): x.add_(1.0)
g = torch.cuda.CUDAGraph()
smalls()
torch.cuda.synchronize()
with torch.cuda.graph(g): smalls()
def graph(): g.replay()
def timeit(fn, n=3):
    ts = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); fn(); e1.record(s); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)
big = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
host = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
side = torch.cuda.Stream()
def d2h(chunk_mb=None, reps=12):
    with torch.cuda.stream(side):
        for _ in range(reps):
            if chunk_mb is None: host.copy_(big, non_blocking=True)
            else:
                c = chunk_mb << 20
                for o in range(0, 1 << 30, c): host[o:o+c].copy_(big[o:o+c], non_blocking=True)
def h2d(reps=12):
    with torch.cuda.stream(side):
        for _ in range(reps): big.copy_(host, non_blocking=True)
for name, fn in (("gemm x10", gemms), ("2000 small launches", smalls), ("graph of 2000 small", graph)):
    fn(); torch.cuda.synchronize()
    base = timeit(fn)
    d2h(); busy = timeit(fn); torch.cuda.synchronize()
    d2h(8); busy8 = timeit(fn); torch.cuda.synchronize()
    h2d(); busyh = timeit(fn); torch.cuda.synchronize()
    print(f"{name:22s} idle {base:8.2f} ms | D2H 1GiB copies {busy:8.2f} ({(busy/base-1)*100:+5.1f}%) | D2H 8MiB chunks {busy8:8.2f} ({(busy8/base-1)*100:+5.1f}%) | H2D {busyh:8.2f} ({(busyh/base-1)*100:+5.1f}%)", flush=True)
