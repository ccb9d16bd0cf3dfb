"""BASELINE configs[3]: Llama-3-8B online serving on vLLM 0.22 (CUDA graphs
on), Poisson arrivals, continuous probe capture; TPOT with capture off vs on.

Random-init ("dummy") weights from a local Llama-3-8B config (no network);
prompts are random token ids; every request generates exactly
--output-len tokens (ignore_eos). One process per setting (a fresh engine):

    python scripts/vllm_serving.py --capture off --rates 1,4,16
    python scripts/vllm_serving.py --capture on --rates 1,4,16 --sites resid_post,mlp_act

Timing is wall clock around the engine loop (the reference paper's TPOT,
REF/PAPER.md:394-396): per request, (finish - first token) / (tokens - 1).
Prints one JSON line per rate (observer counters are cumulative).
"""
import argparse
import json
import os
import random
import statistics
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("VLLM_ENABLE_V1_MULTIPROCESSING", "0")
# compiled-graph cache entries do not hash runtime-attached hooks
os.environ.setdefault("VLLM_DISABLE_COMPILE_CACHE", "1")

ap = argparse.ArgumentParser()
ap.add_argument("--capture", choices=["off", "on"], default="on")
ap.add_argument("--sites", default="resid_post")
ap.add_argument("--policy", default="completeness")
ap.add_argument("--rates", default="4", help="comma list of Poisson arrival rates, requests/s")
ap.add_argument("--num-requests", type=int, default=64)
ap.add_argument("--prompt-len", type=int, default=256)
ap.add_argument("--output-len", type=int, default=128)
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--gpu-mem", type=float, default=0.55)
ap.add_argument("--ring-gib", type=float, default=8.0)
ap.add_argument("--overlap", action="store_true",
                help="capture kernels on the observer's side stream (overlap mode)")
ap.add_argument("--overlap-max-kib", type=int, default=0,
                help="overlap mode: fork only captures up to this size (0 = all)")
args = ap.parse_args()

d = tempfile.mkdtemp(prefix="llama3_8b_")
json.dump({"architectures": ["LlamaForCausalLM"], "model_type": "llama",
           "hidden_size": 4096, "intermediate_size": 14336, "num_hidden_layers": 32,
           "num_attention_heads": 32, "num_key_value_heads": 8, "vocab_size": 128256,
           "max_position_embeddings": 8192, "rope_theta": 500000.0, "rms_norm_eps": 1e-5,
           "torch_dtype": "bfloat16", "hidden_act": "silu", "tie_word_embeddings": False,
           "bos_token_id": 128000, "eos_token_id": 128001},
          open(os.path.join(d, "config.json"), "w"))

kw = {}
if args.capture == "on":
    os.environ["TF_VLLM_OBSERVER"] = json.dumps({
        "sites": args.sites.split(","), "ring_bytes": int(args.ring_gib * (1 << 30)),
        "meta_slots": 8192, "policy": args.policy, "sink": "null",
        "overlap": args.overlap,
        "overlap_max_bytes": (args.overlap_max_kib << 10) or None})
    kw["worker_cls"] = "paper_2605_11093_b200.vllm_worker.ObservedWorker"

from vllm import LLM, SamplingParams  # noqa: E402
from vllm.inputs import TokensPrompt  # noqa: E402

t_start = time.time()
llm = LLM(model=d, load_format="dummy", skip_tokenizer_init=True,
          max_model_len=args.prompt_len + args.output_len + 64,
          gpu_memory_utilization=args.gpu_mem, seed=0, dtype="bfloat16", **kw)
startup = time.time() - t_start
eng = llm.llm_engine
rng = random.Random(args.seed)
sp = SamplingParams(max_tokens=args.output_len, ignore_eos=True, detokenize=False)

# warm-up: one short burst (JIT paths, allocator)
for i in range(4):
    eng.add_request(f"w{i}", TokensPrompt(prompt_token_ids=[rng.randrange(1000, 100000)
                                                             for _ in range(args.prompt_len)]), sp)
while eng.has_unfinished_requests():
    eng.step()

def serve(rate):
    arrivals, t = [], 0.0
    for i in range(args.num_requests):
        t += rng.expovariate(rate)
        arrivals.append(t)
    prompts = [[rng.randrange(1000, 100000) for _ in range(args.prompt_len)]
               for _ in range(args.num_requests)]
    tag = f"r{rate}-"
    first, done, ntok = {}, {}, {}
    t0 = time.perf_counter()
    nxt = 0
    steps = 0
    while nxt < args.num_requests or eng.has_unfinished_requests():
        now = time.perf_counter() - t0
        while nxt < args.num_requests and arrivals[nxt] <= now:
            eng.add_request(tag + str(nxt), TokensPrompt(prompt_token_ids=prompts[nxt]), sp)
            nxt += 1
        if not eng.has_unfinished_requests():
            time.sleep(max(0.0, min(arrivals[nxt] - now, 0.01)))
            continue
        outs = eng.step()
        steps += 1
        now = time.perf_counter() - t0
        for o in outs:
            r = int(o.request_id[len(tag):])
            n = len(o.outputs[0].token_ids)
            if n >= 1 and r not in first:
                first[r] = now
            ntok[r] = n
            if o.finished:
                done[r] = now
    wall = time.perf_counter() - t0
    tpot = [(done[r] - first[r]) / (ntok[r] - 1) * 1e3 for r in done if ntok[r] > 1]
    ttft = [(first[r] - arrivals[r]) * 1e3 for r in first]
    line = {"config": "llama3-8b-vllm-online", "capture": args.capture,
            "sites": args.sites if args.capture == "on" else None, "policy": args.policy,
            "overlap": args.overlap, "overlap_max_kib": args.overlap_max_kib,
            "rate_rps": rate, "requests": args.num_requests,
            "prompt_len": args.prompt_len, "output_len": args.output_len,
            "tpot_ms_mean": statistics.mean(tpot), "tpot_ms_median": statistics.median(tpot),
            "tpot_ms_p99": sorted(tpot)[int(0.99 * (len(tpot) - 1))],
            "ttft_ms_median": statistics.median(ttft), "wall_s": wall, "engine_steps": steps,
            "output_tok_s": sum(ntok.values()) / wall, "startup_s": startup,
            "data": "synthetic (random token ids, random-init weights)"}
    if args.capture == "on":
        llm.collective_rpc("observer_flush")
        line["observer"] = llm.collective_rpc("observer_stats")[0]
    print(json.dumps(line), flush=True)


for rate in [float(x) for x in args.rates.split(",")]:
    serve(rate)
