"""Probe: vLLM 0.22 with a random-init (dummy) Llama-3-8B on one B200."""
import json, os, sys, time, tempfile
os.environ.setdefault("VLLM_ENABLE_V1_MULTIPROCESSING", "0")
t0 = time.time()
d = tempfile.mkdtemp(prefix="llama3_8b_")
cfg = {"architectures": ["LlamaForCausalLM"], "model_type": "llama", "hidden_size": 4096,
       "intermediate_size": 14336, "num_hidden_layers": 32, "num_attention_heads": 32,
       "num_key_value_heads": 8, "vocab_size": 128256, "max_position_embeddings": 8192,
       "rope_theta": 500000.0, "rms_norm_eps": 1e-5, "torch_dtype": "bfloat16",
       "hidden_act": "silu", "tie_word_embeddings": False, "bos_token_id": 128000, "eos_token_id": 128001}
json.dump(cfg, open(os.path.join(d, "config.json"), "w"))
from vllm import LLM, SamplingParams
llm = LLM(model=d, load_format="dummy", skip_tokenizer_init=True, max_model_len=2048,
          gpu_memory_utilization=0.6, seed=0, dtype="bfloat16")
print("startup_s", round(time.time() - t0, 1), flush=True)
from vllm.inputs import TokensPrompt
import random
rng = random.Random(0)
prompts = [TokensPrompt(prompt_token_ids=[rng.randrange(1000, 100000) for _ in range(128)]) for _ in range(16)]
sp = SamplingParams(max_tokens=64, ignore_eos=True, detokenize=False)
t1 = time.time()
outs = llm.generate(prompts, sp)
print("gen_s", round(time.time() - t1, 2), "tokens", sum(len(o.outputs[0].token_ids) for o in outs), flush=True)
eng = llm.llm_engine
print(type(eng), [a for a in dir(eng) if not a.startswith("_")][:60])
