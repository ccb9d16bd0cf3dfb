"""Where does model overhead come from? Variants of the resid capture run."""
import statistics, sys, time, torch
sys.path.insert(0, ".")
from paper_2605_11093_b200 import DrainConfig, NullSink, PolicyConfig, RingConfig, StepRequest
from paper_2605_11093_b200.hookpoint import Observer
from paper_2605_11093_b200.integrations import attach_llama, detach, llama3_8b_config, llama_registry, random_llama
dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
B, T = 8, 512
cfg = llama3_8b_config()
model = random_llama(cfg)
ids = torch.randint(0, cfg.vocab_size, (B, T), device=dev)
batch = [StepRequest(i, i, "p", T, 0) for i in range(B)]
s = torch.cuda.current_stream()
@torch.inference_mode()
def fwd(): model.model(input_ids=ids, use_cache=False)
def run(n, obs=None, sync=True):
    ts = []; t0 = time.perf_counter()
    a0 = torch.cuda.Event(enable_timing=True); a0.record(s)
    for i in range(n):
        if obs: obs.begin_step(batch, i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); fwd(); b.record(s)
        if obs: obs.end_step(s)
        if sync: b.synchronize(); ts.append(a.elapsed_time(b))
    b.synchronize()
    return statistics.median(ts) if ts else a0.elapsed_time(b)/n, (time.perf_counter()-t0)/n*1e3
for _ in range(3): fwd()
print("baseline sync", run(10)); print("baseline nosync", run(10, sync=False))
for sites in (("resid_post",), ("mlp_act", "resid_post")):
  reg = llama_registry(cfg, sites)
  for variant in ("inactive", "discard", "pysink"):
    obs = Observer(reg, ring=RingConfig(20 << 30, 1024), drain=DrainConfig(min_ready_entries=1, min_ready_bytes=1, max_wait=1e-4, staging_buffer_size=128<<20, staging_buffer_count=6, discard_paged=(variant!="pysink"), stage_threads=4),
                   sink=NullSink() if variant=="pysink" else None, device=0, max_batch=B)
    obs.exporter.copy_payloads = False
    if variant == "discard": obs.exporter.start(None)
    else: obs.start()
    h = attach_llama(model, obs, sites)
    if variant == "inactive":
        r = run(10)
    else:
        run(2, obs); obs.flush(); r = run(10, obs); obs.flush()
    print(sites, variant, r, obs.ring.state().stall_events, "launches", obs.launches)
    detach(h); obs.close()
# unstalled kernel timing: 32 resid captures into an empty ring
reg = llama_registry(cfg, ("resid_post","mlp_act"))
obs = Observer(reg, ring=RingConfig(20 << 30, 1024), drain=DrainConfig(discard_paged=True, staging_buffer_size=128<<20), device=0, max_batch=B)
x = torch.randn(B, T, 4096, device=dev, dtype=torch.bfloat16); y = torch.randn(B, T, 14336, device=dev, dtype=torch.bfloat16)
obs.exporter.start(None)
for rep in range(3):
    obs.begin_step(batch, rep)
    ev = []
    for L in range(32):
        for hid, t in ((2*L, y), (2*L+1, x)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s); obs.capture(hid, t); b.record(s); ev.append((a, b, t.numel()*2))
    obs.end_step(s); torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b, _ in ev]
    r_ms = ms[1::2]; m_ms = ms[0::2]
    print("rep", rep, "resid us med", statistics.median(r_ms)*1e3, "mlp us med", statistics.median(m_ms)*1e3,
          "resid GB/s", 2*B*T*4096*2/statistics.median(r_ms)/1e6, "mlp GB/s", 2*B*T*14336*2/statistics.median(m_ms)/1e6)
    obs.flush()
obs.close()
