"""Small driver for ncu: decode-size capture kernels (16 rows x 8 KiB =
128 KiB, one Llama-3-8B resid row per decoded token), back to back."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_11093_b200 import RingConfig, RingPair  # noqa: E402
from paper_2605_11093_b200.hooks import RowSource, capture_args, launch_capture  # noqa: E402
dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
B, H = 16, 4096
x = torch.randn(B, 1, H, device=dev, dtype=torch.bfloat16)
keep = torch.ones(B, dtype=torch.uint8, device=dev)
ring = RingPair(RingConfig(1 << 30, 4096), device=0)
for i in range(16):
    src = RowSource(x.data_ptr(), B, 1, H * 2, H * 2, H * 2, x)
    launch_capture(ring, capture_args(src, hook_id=i, keep_ptr=keep.data_ptr(),
                                      keep_per_outer=True, full="raise"))
torch.cuda.synchronize()
print("ok", ring.state().captures_launched)
