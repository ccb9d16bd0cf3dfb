"""Host cost of Observer.begin_step/end_step in the serving layout (flat,
64 hooks, 16 decode requests), with cProfile breakdown."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import torch
from paper_2605_11093_b200 import DrainConfig, RingConfig, StepRequest, PolicyConfig
from paper_2605_11093_b200.hookpoint import Observer
from paper_2605_11093_b200.vllm_worker import vllm_llama_specs
from paper_2605_11093_b200.hooks import ModelSpec, install_hooks
from paper_2605_11093_b200.sinks import NullSink
from paper_2605_11093_b200.integrations import llama3_8b_config
cfg = llama3_8b_config()
reg = install_hooks(ModelSpec(32, 4096), vllm_llama_specs(cfg, ("resid_post", "mlp_act")))
obs = Observer(reg, ring=RingConfig(1 << 30, 4096), drain=DrainConfig(min_ready_entries=1),
               policy=PolicyConfig(), sink=NullSink(), max_batch=256, flat_rows=9216, persistent=True)
obs.start()
batch = [StepRequest(i, i, "", 1, 100) for i in range(16)]
def run(n):
    t0 = time.perf_counter()
    for s in range(n):
        obs.begin_step(batch, s, layout="flat", rows_total=16)
        obs.end_step()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6
run(50)
print("begin+end us/step:", round(run(500), 1))
pr = cProfile.Profile(); pr.enable(); run(300); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
obs.close()
