"""vLLM integration check on a tiny random-init Llama (one JSON line).

--mode eager: vLLM with enforce_eager; plain torch hooks at the same sites
  copy every observed tensor to the host (the reference); every record the
  observer exported must equal the reference rows of its request, byte for
  byte, and every (step, hook, scheduled request) must have exactly one
  record (completeness policy).
--mode graph: CUDA graphs and torch.compile on (the serving configuration):
  the capture kernels run from vLLM's recorded piecewise and full-decode
  graphs. The reference here is a debug copy of the whole observed tensor
  into a fixed per-hook buffer, recorded into the same graphs right beside
  each capture kernel (Observer.debug_clone) and read back after every
  forward: every record of every replay must equal its request's rows of
  that copy byte for byte, with requests of different output lengths so the
  decode batch shrinks through many padded CUDA-graph batch sizes (a stale
  keep vector or step number in a replay would show as a mismatch).
"""
import argparse
import json
import os
import random
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("VLLM_ENABLE_V1_MULTIPROCESSING", "0")
os.environ.setdefault("VLLM_DISABLE_COMPILE_CACHE", "1")

ap = argparse.ArgumentParser()
ap.add_argument("--mode", choices=["eager", "graph"], default="eager")
ap.add_argument("--requests", type=int, default=13)
ap.add_argument("--output-len", type=int, default=12)
ap.add_argument("--overlap", action="store_true",
                help="captures on the observer's side stream (Observer(overlap=True))")
args = ap.parse_args()

d = tempfile.mkdtemp(prefix="tiny_llama_")
json.dump({"architectures": ["LlamaForCausalLM"], "model_type": "llama",
           "hidden_size": 256, "intermediate_size": 512, "num_hidden_layers": 2,
           "num_attention_heads": 4, "num_key_value_heads": 2, "vocab_size": 2048,
           "max_position_embeddings": 1024, "rope_theta": 10000.0, "rms_norm_eps": 1e-5,
           "torch_dtype": "bfloat16", "hidden_act": "silu", "tie_word_embeddings": False,
           "bos_token_id": 1, "eos_token_id": 2, "head_dim": 64},
          open(os.path.join(d, "config.json"), "w"))
os.environ["TF_VLLM_OBSERVER"] = json.dumps({
    "sites": ["resid_post", "mlp_act"], "ring_bytes": 256 << 20, "meta_slots": 4096,
    "policy": "completeness", "sink": "list", "staging_buffer_mib": 16,
    "debug_clone": args.mode == "eager", "debug_graph_clone": args.mode == "graph",
    "overlap": args.overlap})

import torch  # noqa: E402
from vllm import LLM, SamplingParams  # noqa: E402
from vllm.inputs import TokensPrompt  # noqa: E402

llm = LLM(model=d, load_format="dummy", skip_tokenizer_init=True, max_model_len=512,
          gpu_memory_utilization=0.3, seed=0, dtype="bfloat16",
          enforce_eager=args.mode == "eager",
          worker_cls="paper_2605_11093_b200.vllm_worker.ObservedWorker")
rng = random.Random(7)
prompts = [TokensPrompt(prompt_token_ids=[rng.randrange(3, 2048)
                                          for _ in range(rng.randint(5, 90))])
           for _ in range(args.requests)]
# output lengths 2 .. output_len + 1: requests finish one after another, so
# the decode batch walks down through the padded graph batch sizes
sps = [SamplingParams(max_tokens=2 + (i * 7) % args.output_len, ignore_eos=True,
                      detokenize=False) for i in range(args.requests)]
llm.generate(prompts, sps)
llm.collective_rpc("observer_flush")
dbg = llm.collective_rpc("observer_debug")[0]
recs, layouts = dbg["records"], dbg["layouts"]
hooks = sorted({r[0] for r in recs})
expected = {(s, h, rid): n for s, lay in layouts.items() for rid, n in lay for h in hooks}
got = {}
dup = 0
for h, s, rid, shape, payload in recs:
    k = (s, h, rid)
    dup += k in got
    got[k] = (shape, payload)
missing = [k for k in expected if k not in got]
extra = [k for k in got if k not in expected]
rows_bad = [k for k, (shape, _) in got.items() if k in expected and shape[0] != expected[k]]
out = {"mode": args.mode, "overlap": args.overlap, "records": len(recs),
       "expected": len(expected),
       "hooks": len(hooks), "steps": len(layouts), "missing": len(missing),
       "extra": len(extra), "duplicates": dup, "row_count_mismatch": len(rows_bad)}
# every record against its request's rows of the reference copy
mism = checked = 0
padded = {}  # step -> (rows the forward ran, rows scheduled)
for s, name, t in dbg["clones"]:
    lay = layouts.get(s)
    if not lay:
        continue
    t2 = t.reshape(t.shape[0], -1).contiguous()
    padded[s] = (t2.shape[0], sum(n for _, n in lay))
    pos = 0
    for rid, n in lay:
        ref = t2[pos:pos + n].view(torch.uint8).numpy().tobytes()
        pos += n
        rec = got.get((s, name, rid))
        checked += 1
        if rec is None or rec[1] != ref:
            mism += 1
out.update({"bit_exact_checked": checked, "bit_exact_mismatch": mism,
            "padded_batch_sizes": sorted({r for r, n in padded.values() if r != n}),
            "steps_with_padding": sum(1 for r, n in padded.values() if r != n)})
out["ok"] = (not missing and not extra and not dup and not rows_bad and len(recs) > 0
             and out["bit_exact_mismatch"] == 0 and out["bit_exact_checked"] == len(expected)
             and (args.mode != "graph" or out["steps_with_padding"] > 0))
print(json.dumps(out), flush=True)
