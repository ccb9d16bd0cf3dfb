"""Model step time under controlled interference (no per-step events)."""
import statistics, sys, time, torch
sys.path.insert(0, ".")
from paper_2605_11093_b200 import DrainConfig, ExportPipeline, RingConfig, RingPair, StepRequest
from paper_2605_11093_b200.hookpoint import Observer
from paper_2605_11093_b200.hooks import RowSource, capture_args, launch_capture
from paper_2605_11093_b200.integrations import attach_llama, detach, llama3_8b_config, llama_registry, random_llama
dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
B, T, N = 8, 512, 8
cfg = llama3_8b_config(); model = random_llama(cfg)
ids = torch.randint(0, cfg.vocab_size, (B, T), device=dev)
batch = [StepRequest(i, i, "p", T, 0) for i in range(B)]
s = torch.cuda.current_stream()
@torch.inference_mode()
def fwd(): model.model(input_ids=ids, use_cache=False)
def steps(obs=None, base=0):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for i in range(N):
        if obs: obs.begin_step(batch, base + i)
        fwd()
        if obs: obs.end_step(s)
    b.record(s); b.synchronize()
    return a.elapsed_time(b) / N
for _ in range(3): fwd()
base = steps(); print(f"V1 no capture                 {base:7.2f} ms", flush=True)
# background D2H traffic from our stager: pre-publish ~14 GiB, then drain during the steps
y = torch.randn(B, T, 14336, device=dev, dtype=torch.bfloat16)
keep = torch.ones(B, dtype=torch.uint8, device=dev)
def prefill_ring(n=120):
    ring = RingPair(RingConfig(16 << 30, 4096), device=0)
    src = RowSource(y.data_ptr(), B, T, 14336*2, y.stride(0)*2, 14336*2, y)
    for i in range(n):
        launch_capture(ring, capture_args(src, hook_id=i, keep_ptr=keep.data_ptr(), keep_per_outer=True, full="raise"), s)
    torch.cuda.synchronize()
    pipe = ExportPipeline(ring, DrainConfig(min_ready_entries=1, min_ready_bytes=1, max_wait=1e-4, staging_buffer_size=128<<20, staging_buffer_count=6, discard_paged=True))
    return ring, pipe
ring_bg, pipe_bg = prefill_ring()
pipe_bg.start(None); t = steps(); print(f"V4 D2H busy, no capture       {t:7.2f} ms  (+{(t/base-1)*100:5.1f}%)", flush=True)
pipe_bg.flush(); pipe_bg.stop(); pipe_bg.close(); ring_bg.close()
for sites in (("resid_post",), ("mlp_act", "resid_post")):
    reg = llama_registry(cfg, sites)
    # V2: capture kernels, no stager (ring holds everything)
    obs = Observer(reg, ring=RingConfig(60 << 30, 4096), drain=DrainConfig(discard_paged=True, staging_buffer_size=128<<20), device=0, max_batch=B)
    h = attach_llama(model, obs, sites)
    t = steps(obs, 0); print(f"V2 {str(sites):30s} kernels only   {t:7.2f} ms (+{(t/base-1)*100:5.1f}%)", flush=True)
    obs.exporter.start(None); obs.flush(300)
    t = steps(obs, 100); print(f"V3 {str(sites):30s} +stager D2H    {t:7.2f} ms (+{(t/base-1)*100:5.1f}%)", flush=True)
    obs.flush(300)
    detach(h); obs.close()
