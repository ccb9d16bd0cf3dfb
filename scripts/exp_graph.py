"""Llama-3-8B prefill as a CUDA graph, with and without in-graph captures."""
import statistics, sys, time, torch
sys.path.insert(0, ".")
from paper_2605_11093_b200 import DrainConfig, NullSink, RingConfig, StepRequest
from paper_2605_11093_b200.hookpoint import Observer
from paper_2605_11093_b200.integrations import attach_llama, detach, llama3_8b_config, llama_registry, random_llama
dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
B, T, N = 8, 512, 10
cfg = llama3_8b_config(); model = random_llama(cfg)
ids = torch.randint(0, cfg.vocab_size, (B, T), device=dev)
batch = [StepRequest(i, i, "p", T, 0) for i in range(B)]
def make_graph():
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs), torch.inference_mode():
        for _ in range(2): model.model(input_ids=ids, use_cache=False)
    torch.cuda.current_stream().wait_stream(cs)
    g = torch.cuda.CUDAGraph()
    with torch.inference_mode(), torch.cuda.graph(g):
        model.model(input_ids=ids, use_cache=False)
    return g
s = torch.cuda.current_stream()
def steps(g, obs=None, base=0, n=N):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for i in range(n):
        if obs: obs.begin_step(batch, base + i)
        g.replay()
        if obs: obs.end_step(s)
    b.record(s); b.synchronize()
    return a.elapsed_time(b) / n
g0 = make_graph(); steps(g0, n=3)
base = steps(g0); print(f"graph no capture {base:7.2f} ms", flush=True)
for sites in (("resid_post",), ("mlp_act", "resid_post")):
    reg = llama_registry(cfg, sites)
    obs = Observer(reg, ring=RingConfig(24 << 30, 4096), drain=DrainConfig(min_ready_entries=1, min_ready_bytes=1, max_wait=1e-4, staging_buffer_size=128<<20, staging_buffer_count=6, discard_paged=True), device=0, max_batch=B)
    h = attach_llama(model, obs, sites)
    obs.begin_step(batch, 0)            # active during capture -> captures recorded in the graph
    g = make_graph()
    obs.end_step(s)
    torch.cuda.synchronize()
    # graph capture launched captures during warmup iterations: drain them
    obs.exporter.start(None); obs.flush(300)
    t2 = steps(g, obs, 10); obs.flush(300)
    st = obs.ring.state()
    print(f"graph {sites} capture+stager {t2:7.2f} ms (+{(t2/base-1)*100:5.1f}%) stalls {st.stall_events} drops {st.drops} captures {st.captures_launched}", flush=True)
    detach(h); obs.close(); del g
