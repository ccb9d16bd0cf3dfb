"""HookPoint placement for Hugging Face models (§4 "Framework
integration": observation sites declared once, HookPoints attached without
editing the backbone).

Sites (per decoder layer ``L``):

    resid_post[L]   decoder-layer output (B, T, H)            residual stream
    mlp_act[L]      input of down_proj: act(gate) * up (B, T, F)   MLP
    attn_out[L]     self-attention output before the residual add (B, T, H)
    attn_pattern[L] attention probabilities (B, heads, T, T)  (eager attention)
    k_slice[L]      k_proj output for this step's tokens (B, T, kv*d), pre-RoPE
    v_slice[L]      v_proj output (B, T, kv*d)  — the V rows the cache stores
    k_cache[L]      KV-cache slice: the post-RoPE K rows this step appended to
                    the layer's cache, read from the cache storage itself
                    (B, kv_heads, T, head_dim) — PAPER.md:26 "KV-cache slices"
    v_cache[L]      the V rows this step appended, from the cache storage

Each site becomes a ``HookPoint`` submodule registered on the model (so it
shows in ``named_modules``) and driven from a forward hook on the module
that produces the tensor. Declaration order inside a layer follows
execution order: attn sites, then mlp_act, then resid_post.
"""

from __future__ import annotations

from .hookpoint import HookPoint, Observer, join_point
from .hooks import DType, HookSpec, ModelSpec, install_hooks

SITE_ORDER = ("k_slice", "v_slice", "k_cache", "v_cache", "attn_pattern",
              "attn_out", "mlp_act", "resid_post")

_TORCH_TO_DTYPE = {"torch.bfloat16": "bf16", "torch.float16": "f16",
                   "torch.float32": "f32"}


def llama_specs(config, sites, dtype: str = "bf16", cast_to=None,
                reduce=None) -> list[HookSpec]:
    """Per-layer HookSpecs for a Llama-family config, in firing order."""
    dt = DType.of(dtype)
    head_dim = getattr(config, "head_dim", None) or \
        config.hidden_size // config.num_attention_heads
    kv = config.num_key_value_heads * head_dim
    dims = {
        "k_cache": (config.num_key_value_heads, "tokens", head_dim),
        "v_cache": (config.num_key_value_heads, "tokens", head_dim),
        "resid_post": ("tokens", "hidden"),
        "attn_out": ("tokens", "hidden"),
        "mlp_act": ("tokens", config.intermediate_size),
        "k_slice": ("tokens", kv),
        "v_slice": ("tokens", kv),
        "attn_pattern": (config.num_attention_heads, "tokens", "tokens"),
    }
    out = []
    for site in SITE_ORDER:
        if site in sites:
            out.append(HookSpec(site, dims[site], dt, per_layer=True,
                                cast_to=DType.of(cast_to) if cast_to else None,
                                reduce=reduce))
    return out


def gpt2_specs(config, dtype: str = "f32") -> list[HookSpec]:
    return [HookSpec("resid_post", ("tokens", "hidden"), DType.of(dtype),
                     per_layer=True)]


def llama_registry(config, sites, dtype: str = "bf16", **kw):
    model = ModelSpec(config.num_hidden_layers, config.hidden_size)
    return install_hooks(model, llama_specs(config, sites, dtype, **kw))


def _first(out):
    return out[0] if isinstance(out, (tuple, list)) else out


def _cache_rows(module, args, kwargs, observer):
    """The K and V rows this forward appended to the layer's KV cache, as
    views of the cache storage (no copy): (B, kv_heads, T, head_dim) each.

    ``DynamicLayer`` appends at the end, so the new rows are the last T; a
    ``StaticLayer`` (fixed buffers, CUDA-graph decoding) writes them at the
    step's token position, which the observer knows from the plan (reading
    the layer's device-side length would synchronise)."""
    cache = kwargs.get("past_key_values")
    if cache is None:
        return None
    hs = kwargs.get("hidden_states", args[0] if args else None)
    T = hs.shape[1]
    lay = cache.layers[module.layer_idx]
    k, v = lay.keys, lay.values
    if hasattr(lay, "max_cache_len"):      # static: written at the step position
        s0 = observer.step_token_start() if observer is not None else 0
        B = hs.shape[0]
        return (k[:B, :, s0:s0 + T, :], v[:B, :, s0:s0 + T, :])
    S = k.shape[-2]
    return k[:, :, S - T:, :], v[:, :, S - T:, :]


def attach_llama(model, observer: Observer | None, sites) -> list:
    """Insert HookPoints into a HF Llama model; returns the hook handles.

    Captures must fire in the registry's order (the metadata FIFO is
    matched strictly, records.py): k_proj / v_proj hooks run first, then
    one hook on the attention module fires k_cache, v_cache, attn_pattern
    and attn_out in ``SITE_ORDER``, then the MLP pre-hook, then the layer
    output."""
    inner = getattr(model, "model", model)
    handles = []
    for L, layer in enumerate(inner.layers):
        hps = {}
        for site in SITE_ORDER:
            if site in sites:
                hp = HookPoint(f"{site}[{L}]", observer)
                model.add_module(f"hookpoint_{site}_{L}", hp)
                hps[site] = hp
        attn = layer.self_attn
        if "k_slice" in hps:
            handles.append(attn.k_proj.register_forward_hook(
                lambda m, a, out, hp=hps["k_slice"]: (hp(out), None)[1]))
        if "v_slice" in hps:
            handles.append(attn.v_proj.register_forward_hook(
                lambda m, a, out, hp=hps["v_slice"]: (hp(out), None)[1]))
        attn_sites = [x for x in ("k_cache", "v_cache", "attn_pattern", "attn_out")
                      if x in hps]
        if attn_sites:
            def attn_hook(m, args, kwargs, out, hps=hps, attn_sites=attn_sites):
                rows = None
                if "k_cache" in hps or "v_cache" in hps:
                    rows = _cache_rows(m, args, kwargs, observer)
                for x in attn_sites:
                    if x == "k_cache" and rows is not None:
                        hps[x](rows[0])
                    elif x == "v_cache" and rows is not None:
                        hps[x](rows[1])
                    elif x == "attn_pattern" and out[1] is not None:
                        hps[x](out[1])
                    elif x == "attn_out":
                        hps[x](_first(out))
                return None
            handles.append(attn.register_forward_hook(attn_hook, with_kwargs=True))
        if "mlp_act" in hps:
            handles.append(layer.mlp.down_proj.register_forward_pre_hook(
                lambda m, args, hp=hps["mlp_act"]: (hp(args[0]), None)[1]))
        if "resid_post" in hps:
            handles.append(layer.register_forward_hook(
                lambda m, a, out, hp=hps["resid_post"]: (hp(_first(out)), None)[1]))
    if observer is not None and observer.overlap:
        # overlap mode: HF writes no captured activation in place, so one
        # join after the last layer suffices (inside a recorded graph too)
        handles.append(inner.norm.register_forward_hook(
            lambda m, a, out: (join_point(observer), None)[1]))
    return handles


def attach_gpt2(model, observer: Observer | None) -> list:
    """resid_post[L] on every GPT-2 block output."""
    inner = getattr(model, "transformer", model)
    handles = []
    for L, block in enumerate(inner.h):
        hp = HookPoint(f"resid_post[{L}]", observer)
        model.add_module(f"hookpoint_resid_post_{L}", hp)
        handles.append(block.register_forward_hook(
            lambda m, a, out, hp=hp: (hp(_first(out)), None)[1]))
    return handles


def detach(handles) -> None:
    for h in handles:
        h.remove()


def random_llama(config, device: str = "cuda", dtype=None, seed: int = 0):
    """Random-init Llama built directly on the device in bf16 (no weights)."""
    import torch
    from transformers import LlamaForCausalLM
    dtype = dtype or torch.bfloat16
    torch.manual_seed(seed)
    prev = torch.get_default_dtype()
    torch.set_default_dtype(dtype)
    try:
        with torch.device(device):
            model = LlamaForCausalLM(config)
    finally:
        torch.set_default_dtype(prev)
    return model.eval()


def llama3_8b_config(layers: int | None = None, attn: str = "sdpa"):
    from transformers import LlamaConfig
    cfg = LlamaConfig(hidden_size=4096, intermediate_size=14336,
                      num_hidden_layers=32 if layers is None else layers,
                      num_attention_heads=32, num_key_value_heads=8,
                      vocab_size=128256, max_position_embeddings=8192,
                      rope_theta=500000.0, rms_norm_eps=1e-5)
    cfg._attn_implementation = attn
    return cfg
