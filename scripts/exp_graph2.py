"""Graph-mode resid+mlp: which export stage couples back into the step?"""
import statistics, sys, time, torch
sys.path.insert(0, ".")
from paper_2605_11093_b200 import DrainConfig, NullSink, RingConfig, StepRequest
from paper_2605_11093_b200.hookpoint import Observer
from paper_2605_11093_b200.integrations import attach_llama, detach, llama3_8b_config, llama_registry, random_llama
dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
B, T, N = 8, 512, 8
cfg = llama3_8b_config(); model = random_llama(cfg)
ids = torch.randint(0, cfg.vocab_size, (B, T), device=dev)
batch = [StepRequest(i, i, "p", T, 0) for i in range(B)]
s = torch.cuda.current_stream()
def fwd():
    with torch.inference_mode(): model.model(input_ids=ids, use_cache=False)
def make_graph(obs=None):
    cs = torch.cuda.Stream(); cs.wait_stream(s)
    with torch.cuda.stream(cs):
        for _ in range(2): fwd()
    s.wait_stream(cs)
    g = torch.cuda.CUDAGraph()
    if obs is None:
        with torch.inference_mode(), torch.cuda.graph(g): model.model(input_ids=ids, use_cache=False)
    else:
        with obs.graph_capture(), torch.inference_mode(), torch.cuda.graph(g): model.model(input_ids=ids, use_cache=False)
    return g
def run(g, obs=None, base=0):
    torch.cuda.synchronize(); hb = []
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for i in range(N):
        t0 = time.perf_counter()
        if obs: obs.begin_step(batch, base + i)
        hb.append((time.perf_counter() - t0) * 1e3)
        g.replay()
        if obs: obs.end_step(s)
    b.record(s); b.synchronize()
    return a.elapsed_time(b) / N, statistics.median(hb), max(hb)
g0 = make_graph(); run(g0)
base, _, _ = run(g0); print(f"graph no capture {base:7.2f} ms", flush=True)
sites = ("mlp_act", "resid_post")
reg = llama_registry(cfg, sites)
for variant in ("discard", "pageable-nosinkcopy", "pageable-sink"):
    sink = NullSink()
    obs = Observer(reg, ring=RingConfig(20 << 30, 1024), drain=DrainConfig(min_ready_entries=1, min_ready_bytes=1, max_wait=1e-4, staging_buffer_size=128<<20, staging_buffer_count=6, discard_paged=(variant=="discard"), stage_threads=4),
                   sink=None if variant == "discard" else sink, device=0, max_batch=B)
    obs.exporter.copy_payloads = False
    if variant == "discard": obs.exporter.start(None)
    else: obs.start()
    h = attach_llama(model, obs, sites)
    g = make_graph(obs)
    run(g, obs, 10); obs.flush(300)
    t, hmed, hmax = run(g, obs, 100)
    t_flush0 = time.perf_counter(); obs.flush(300); tf = time.perf_counter() - t_flush0
    st = obs.ring.state(); xs = obs.exporter.stats()
    print(f"{variant:22s} step {t:7.2f} ms (+{(t/base-1)*100:5.1f}%) begin_step med {hmed:6.2f} max {hmax:7.2f} ms | flush tail {tf*1e3:7.1f} ms | stalls {st.stall_events} exhausted_waits {xs['staging_exhausted_waits']} d2h {xs['bytes_drained']/max(xs['transfer_seconds'],1e-9)/1e9:5.1f} GB/s", flush=True)
    detach(h); obs.close(); del g
