"""BASELINE configs[2] at full scale: random-init Llama-3-8B (32 layers,
H 4096, 32 heads, 8 KV heads), eager attention, prefill T=512 then one
decode step. Captured per layer:

* ``attn_pattern[L]`` — attention probabilities (B, 32, T, T), token-sampled
  to every 16th query row (eager attention exposes them);
* ``k_cache[L]`` / ``v_cache[L]`` — the post-RoPE K and V rows the step
  appended to the layer's KV cache, read from the cache storage itself
  ("KV-cache slices"); at decode a strided (B, 8, 1, 128)
  view of the cache, no copy;
* ``resid_post[L]`` — the residual stream, token-sampled like the pattern.

Every record is compared byte for byte with what plain torch hooks see at
the same sites (raw captures are bit-exact)."""

import pytest
import torch

from paper_2605_11093_b200 import DrainConfig, RingConfig, StepRequest
from paper_2605_11093_b200.hookpoint import Observer, TokenSampler
from paper_2605_11093_b200.integrations import (attach_llama, llama3_8b_config,
                                                llama_registry, random_llama)

pytestmark = pytest.mark.gpu

EVERY = 16


class Collect:
    def __init__(self):
        self.records = []

    def write(self, recs):
        self.records.extend(recs)


def _b(t):
    return t.contiguous().view(torch.uint8).cpu().numpy().tobytes()


@pytest.fixture(scope="module")
def llama8b():
    cfg = llama3_8b_config(attn="eager")
    model = random_llama(cfg)
    yield cfg, model
    del model
    torch.cuda.empty_cache()


def test_config2_llama3_8b_attention_and_kv_cache(llama8b):
    from transformers import DynamicCache
    from transformers.models.llama.modeling_llama import apply_rotary_pos_emb
    cfg, model = llama8b
    B, T = 4, 512
    sites = ("k_cache", "v_cache", "attn_pattern", "resid_post")
    reg = llama_registry(cfg, sites)
    sampled = frozenset(i for i, h in enumerate(reg.hooks)
                        if h.name.startswith(("attn_pattern", "resid_post")))
    sink = Collect()
    obs = Observer(reg, ring=RingConfig(2 << 30, 1024), sink=sink, max_batch=B,
                   max_tokens=T, sampler=TokenSampler(every=EVERY),
                   sampled_hooks=sampled,
                   drain=DrainConfig(staging_buffer_size=64 << 20))
    obs.start()
    kept_tok = list(range(0, T, EVERY))
    ref = {}
    inner = model.model
    handles = []
    for L, layer in enumerate(inner.layers):
        def attn_ref(m, args, kwargs, out, L=L):
            if out[1] is not None and out[1].shape[-2] == T:
                ref[("attn_pattern", L)] = out[1][:, :, kept_tok, :].clone()
            ref[("pos", L, kwargs["hidden_states"].shape[1])] = kwargs["position_embeddings"]

        def kproj_ref(m, a, out, L=L):
            ref[("k_proj", L, out.shape[1])] = out.clone()

        def layer_ref(m, a, out, L=L):
            o = out[0] if isinstance(out, tuple) else out
            ref[("resid_post", L, o.shape[1])] = o.clone()
        handles.append(layer.self_attn.register_forward_hook(attn_ref, with_kwargs=True))
        handles.append(layer.self_attn.k_proj.register_forward_hook(kproj_ref))
        handles.append(layer.register_forward_hook(layer_ref))
    handles += attach_llama(model, obs, sites)

    g = torch.Generator().manual_seed(0)
    ids = torch.randint(0, cfg.vocab_size, (B, T), generator=g).cuda()
    reqs = [StepRequest(100 + i, i, "p", T, 0) for i in range(B)]
    cache = DynamicCache(config=cfg)
    obs.begin_step(reqs, 0)
    with torch.inference_mode():
        out = inner(input_ids=ids, past_key_values=cache, use_cache=True)
    obs.end_step()
    prefill_k = [cache.layers[L].keys.clone() for L in range(cfg.num_hidden_layers)]
    prefill_v = [cache.layers[L].values.clone() for L in range(cfg.num_hidden_layers)]

    # decode step: the attention map is (B, 32, 1, T+1), not a (tokens,
    # tokens) shape, so it is filtered out at the step boundary
    # (set_hook_filter, hooks.py) while the cache slices keep flowing
    reg.set_hook_filter([h.name for h in reg.hooks if not h.name.startswith("attn_pattern")])
    nxt = out.last_hidden_state[:, -1:, :].float().sum(-1).long().abs() % cfg.vocab_size
    obs.begin_step([StepRequest(100 + i, i, "p", 1, T) for i in range(B)], 1)
    with torch.inference_mode():
        inner(input_ids=nxt, past_key_values=cache, use_cache=True)
    obs.end_step()
    obs.flush(600)
    obs.close()
    for h in handles:
        h.remove()

    got = {(r.hook_name, r.request_id, r.step_seq): r for r in sink.records}
    n_layers = cfg.num_hidden_layers
    assert len(got) == B * n_layers * (4 + 3)
    d = cfg.hidden_size // cfg.num_attention_heads
    kvh = cfg.num_key_value_heads
    for L in range(n_layers):
        for i in range(B):
            rid = 100 + i
            # prefill
            a = got[(f"attn_pattern[{L}]", rid, 0)]
            assert a.shape == (cfg.num_attention_heads * len(kept_tok), T)
            assert bytes(a.payload) == _b(ref[("attn_pattern", L)][i])
            r = got[(f"resid_post[{L}]", rid, 0)]
            assert bytes(r.payload) == _b(ref[("resid_post", L, T)][i][kept_tok])
            k = got[(f"k_cache[{L}]", rid, 0)]
            v = got[(f"v_cache[{L}]", rid, 0)]
            assert k.shape == (kvh, T, d)
            assert bytes(k.payload) == _b(prefill_k[L][i])
            assert bytes(v.payload) == _b(prefill_v[L][i])
            # decode: the row the step appended, from the cache storage
            kd = got[(f"k_cache[{L}]", rid, 1)]
            vd = got[(f"v_cache[{L}]", rid, 1)]
            assert kd.shape == (kvh, 1, d)
            assert bytes(kd.payload) == _b(cache.layers[L].keys[i, :, T:T + 1, :])
            assert bytes(vd.payload) == _b(cache.layers[L].values[i, :, T:T + 1, :])
            rd = got[(f"resid_post[{L}]", rid, 1)]
            assert bytes(rd.payload) == _b(ref[("resid_post", L, 1)][i])
        # the cache rows are post-RoPE: equal to RoPE(k_proj) and, past
        # position 0, different from the k_proj output itself
        kp = ref[("k_proj", L, T)].view(B, T, kvh, d).transpose(1, 2)
        cos, sin = ref[("pos", L, T)]
        _, k_rope = apply_rotary_pos_emb(kp, kp, cos, sin)
        assert torch.equal(k_rope, prefill_k[L])
        assert not torch.equal(kp[:, :, 1:], prefill_k[L][:, :, 1:])
