import ctypes as C, random, torch
from paper_2605_11093_b200 import *
from paper_2605_11093_b200 import _native as N
for per, keep in [(4, (1,0,1,1)), (17, (1,1,1,1)), (16, (1,1,1,1)), (17, (1,0,1,1)), (3,(1,1,1,1))]:
    reg = install_hooks(ModelSpec(1, 8), [HookSpec("h", (per,), DType.of("u8"))])
    ring = allocate_rings(RingConfig(1024, 16))
    data = bytes(random.Random(2).randrange(256) for _ in range(4*per))
    view = TensorView(data, (4, per), DType.of("u8"))
    try:
        out = capture(reg, ring, 0, view, keep)
    except Exception as e:
        print(per, keep, "EXC", repr(e)); continue
    res = N.CCaptureResult(); N.lib().tf_ring_last_result(ring.handle, C.byref(res))
    print(per, keep, out.bytes_written, "status", res.status, "rows", res.n_rows, "len", res.payload_len, "seq", res.capture_seq, "ready", res.ready_seq, ring.counters())
torch.cuda.synchronize()
