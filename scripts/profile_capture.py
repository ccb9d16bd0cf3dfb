"""Small driver for ncu: capture kernels of the bench workload shapes
(Llama-3-8B, 8x512 tokens: resid 32 MiB, mlp_act 112 MiB), no staging."""
import sys, torch
sys.path.insert(0, ".")
from paper_2605_11093_b200 import RingConfig, RingPair
from paper_2605_11093_b200.hooks import RowSource, capture_args, launch_capture
dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
B, T = 8, 512
r = torch.randn(B, T, 4096, device=dev, dtype=torch.bfloat16)
m = torch.randn(B, T, 14336, device=dev, dtype=torch.bfloat16)
keep = torch.ones(B, dtype=torch.uint8, device=dev)
ring = RingPair(RingConfig(4 << 30, 1024), device=0)
for i in range(8):
    x = m if i % 2 == 0 else r
    src = RowSource(x.data_ptr(), B, T, x.shape[-1] * 2, x.stride(0) * 2, x.shape[-1] * 2, x)
    launch_capture(ring, capture_args(src, hook_id=i, keep_ptr=keep.data_ptr(),
                                      keep_per_outer=True, full="raise"))
torch.cuda.synchronize()
print("ok", ring.state().captures_launched)
