"""vLLM 0.22 integration: HookPoints inside a serving engine with CUDA graphs.

The paper integrates DMI-Lib with vLLM by subclassing the worker and
wrapping ``init_device`` / ``load_model`` / ``execute_model`` so the policy
runs once per step (§4, "vLLM Worker subclass").
This module does the same for vLLM 0.22's V1 GPU worker:

* ``load_model``: build one ``Observer`` for the device (ring pair, staging
  engine, exporter) and attach HookPoints to the loaded Llama model before
  vLLM compiles it and records its CUDA graphs. The observer is
  *persistent*: the capture kernels are recorded into vLLM's piecewise and
  full-decode CUDA graphs once, and every replay reads the keep vector and
  step number from the observer's fixed device buffers (§3.4).
* ``execute_model``: keep the scheduler output of the step.
* the runner's ``_model_forward`` (called for eager, piecewise and
  full-graph execution alike): lay out this step's requests in the runner's
  flat token order (``input_batch.req_ids`` × ``num_scheduled_tokens``),
  run the policy (``prepare_step`` with ragged rows), queue the metadata and
  upload the per-row keep vector padded to the CUDA-graph batch size, run
  the model, then close the step.

Observation sites on vLLM's Llama (``vllm/model_executor/models/llama.py``):

    resid_post[L]  the residual stream after layer L. vLLM fuses the
                   residual add into the next RMSNorm, so this is the
                   residual output of layer L+1's ``input_layernorm`` (and
                   of the final ``norm`` for the last layer): no extra add
    mlp_act[L]     the input of ``down_proj``: act(gate) * up, (tokens, F)

Configuration comes from the environment (the worker is constructed by
vLLM): ``TF_VLLM_OBSERVER`` holds a JSON object, e.g.
``{"sites": ["resid_post", "mlp_act"], "ring_bytes": 8589934592,
"meta_slots": 4096, "policy": "completeness", "sink": "null"}``.
Use it with ``LLM(..., worker_cls="paper_2605_11093_b200.vllm_worker.ObservedWorker")``
and ``VLLM_ENABLE_V1_MULTIPROCESSING=0`` to read ``stats()`` in-process,
or ``llm.collective_rpc("observer_stats")`` with multiprocessing.
"""

from __future__ import annotations

import json
import os
import time

from vllm.v1.worker.gpu_worker import Worker

from .exporter import DrainConfig
from .hookpoint import HookPoint, Observer, join_point
from .hooks import DType, HookSpec, ModelSpec, install_hooks
from .policy import BEST_EFFORT, COMPLETENESS, DROP_RECENT, PolicyConfig, StepRequest
from .rings import RingConfig
from .sinks import NullSink

ENV = "TF_VLLM_OBSERVER"


def vllm_llama_specs(hf_config, sites, dtype: str = "bf16") -> list[HookSpec]:
    """Per-layer HookSpecs in firing order within a decoder layer."""
    dt = DType.of(dtype)
    out = []
    if "mlp_act" in sites:
        out.append(HookSpec("mlp_act", ("tokens", hf_config.intermediate_size), dt,
                            per_layer=True))
    if "resid_post" in sites:
        out.append(HookSpec("resid_post", ("tokens", "hidden"), dt, per_layer=True))
    return out


def attach_vllm_llama(model, observer: Observer, sites) -> list:
    """HookPoints on a vLLM Llama model (LlamaForCausalLM or LlamaModel)."""
    inner = getattr(model, "model", model)
    layers = list(inner.layers)
    n = len(layers)
    handles = []

    def add(name):
        hp = HookPoint(name, observer)
        model.add_module("hookpoint_" + name.replace("[", "_").replace("]", ""), hp)
        return hp

    if observer.overlap:
        # overlap mode: side-stream captures must be complete before vLLM's
        # fused add+RMSNorm rewrites the residual in place (the layer's
        # post-attention norm) and before each CUDA-graph piece ends (vLLM
        # splits its graphs at the attention op): join right before every
        # attention call, and after the last capture at the final norm
        for layer in layers:
            handles.append(layer.self_attn.attn.register_forward_pre_hook(
                lambda m, args: (join_point(observer), None)[1]))
    for L, layer in enumerate(layers):
        if "mlp_act" in sites:
            hp = add(f"mlp_act[{L}]")
            handles.append(layer.mlp.down_proj.register_forward_pre_hook(
                lambda m, args, hp=hp: (hp(args[0]), None)[1]))
        if "resid_post" in sites and L >= 1:
            # the residual output of layer L's input norm is resid_post[L-1]
            hp = add(f"resid_post[{L - 1}]")
            handles.append(layer.input_layernorm.register_forward_hook(
                lambda m, a, out, hp=hp: (hp(out[1]) if isinstance(out, tuple)
                                          else None, None)[1]))
    if "resid_post" in sites:
        hp = add(f"resid_post[{n - 1}]")
        handles.append(inner.norm.register_forward_hook(
            lambda m, a, out, hp=hp: (hp(out[1]) if isinstance(out, tuple)
                                      else None, None)[1]))
    if observer.overlap:
        handles.append(inner.norm.register_forward_hook(
            lambda m, a, out: (join_point(observer), None)[1]))
    return handles


def observer_config() -> dict:
    cfg = {"sites": ["resid_post"], "ring_bytes": 4 << 30, "meta_slots": 4096,
           "policy": "completeness", "sink": "null", "staging_buffer_mib": 128,
           "staging_buffers": 8}
    raw = os.environ.get(ENV)
    if raw:
        cfg.update(json.loads(raw))
    return cfg


class CountingSink(NullSink):
    """NullSink that also keeps per-hook record counts (for checks)."""

    def __init__(self):
        super().__init__()
        self.by_hook = {}

    def write(self, records):
        super().write(records)
        for r in records:
            self.by_hook[r.hook_name] = self.by_hook.get(r.hook_name, 0) + 1

    def write_captures(self, caps):
        super().write_captures(caps)
        for meta, _, _ in caps:
            self.by_hook[meta.hook_name] = (self.by_hook.get(meta.hook_name, 0)
                                            + len(meta.request_ids))


class ListSink(CountingSink):
    """Keeps every record (tests: the debug-clone parity check)."""

    write_captures = None  # records path: keep the CaptureRecords

    def __init__(self):
        super().__init__()
        self.records = []

    def write(self, records):
        super().write(records)
        self.records.extend(records)


def _clone_hooks(model, store, step_of, sites) -> list:
    """Debug: plain torch hooks at the HookPoint sites that copy the tensor
    to the host on every eager forward (the parity reference)."""
    inner = getattr(model, "model", model)
    layers = list(inner.layers)
    hs = []

    def keep(name, x):
        store.append((step_of(), name, x.detach().to("cpu", copy=True)))
    for L, layer in enumerate(layers):
        if "mlp_act" in sites:
            hs.append(layer.mlp.down_proj.register_forward_pre_hook(
                lambda m, args, n=f"mlp_act[{L}]": keep(n, args[0])))
        if "resid_post" in sites and L >= 1:
            hs.append(layer.input_layernorm.register_forward_hook(
                lambda m, a, out, n=f"resid_post[{L - 1}]":
                keep(n, out[1]) if isinstance(out, tuple) else None))
    if "resid_post" in sites:
        hs.append(inner.norm.register_forward_hook(
            lambda m, a, out, n=f"resid_post[{len(layers) - 1}]":
            keep(n, out[1]) if isinstance(out, tuple) else None))
    return hs


class ObservedWorker(Worker):
    """vLLM GPU worker with a Ring² observer around every model forward."""

    def load_model(self, *args, **kwargs):
        super().load_model(*args, **kwargs)
        cfg = observer_config()
        self._tf_cfg = cfg
        self._tf_obs = None
        if not cfg.get("sites"):
            return
        runner = self.model_runner
        model = runner.model
        hf = self.vllm_config.model_config.hf_config
        sites = tuple(cfg["sites"])
        reg = install_hooks(ModelSpec(hf.num_hidden_layers, hf.hidden_size),
                            vllm_llama_specs(hf, sites))
        sched = self.vllm_config.scheduler_config
        max_tokens = int(sched.max_num_batched_tokens)
        max_seqs = int(sched.max_num_seqs)
        if cfg["policy"] == "best-effort":  # drop-recent unless configured
            policy = PolicyConfig(mode=BEST_EFFORT,
                                  strategy=cfg.get("strategy", DROP_RECENT))
        else:
            policy = PolicyConfig(mode=COMPLETENESS)
        self._tf_sink = ListSink() if cfg.get("sink") == "list" else CountingSink()
        # debug_graph_clone: every capture also copies its whole tensor into
        # a fixed buffer inside the recorded graphs (Observer.debug_clone);
        # the rows are read back after each forward as the parity reference
        dbg_rows = {}
        if cfg.get("debug_graph_clone"):
            for h in reg.hooks:
                width = (hf.intermediate_size if h.name.startswith("mlp_act")
                         else hf.hidden_size)
                dbg_rows[h.name] = width * h.dtype.width
        obs = Observer(
            reg, ring=RingConfig(int(cfg["ring_bytes"]), int(cfg["meta_slots"])),
            # reference-sized drain batches (exporter.py:35-51 defaults are
            # 8 entries / 1 MiB / 2 ms): one sink-thread pass per many
            # captures keeps the exporter's Python off the engine's GIL
            drain=DrainConfig(min_ready_entries=int(cfg.get("drain_entries", 32)),
                              min_ready_bytes=int(cfg.get("drain_bytes", 4 << 20)),
                              max_wait=float(cfg.get("drain_wait", 2e-3)),
                              staging_buffer_size=int(cfg["staging_buffer_mib"]) << 20,
                              staging_buffer_count=int(cfg["staging_buffers"]),
                              page_out="handoff",
                              # a prefill-heavy step (max_num_batched_tokens
                              # rows of mlp_act) can exceed one buffer
                              split_oversize=True),
            policy=policy, sink=self._tf_sink, device=self.local_rank,
            max_batch=max_seqs, flat_rows=max_tokens + 1024, persistent=True,
            debug_row_bytes=dbg_rows, overlap=bool(cfg.get("overlap", False)),
            overlap_max_bytes=cfg.get("overlap_max_bytes"))
        # records that outlive the batch (ListSink) must own their bytes
        obs.exporter.copy_payloads = cfg.get("sink") == "list"
        obs.start()
        self._tf_obs = obs
        self._tf_handles = attach_vllm_llama(model, obs, sites)
        self._tf_req = {}        # live vLLM request id -> int id (= arrival index)
        self._tf_next_id = 0
        self._tf_step = 0
        self._tf_layouts = {}    # debug: step -> [(request id, rows)]
        self._tf_clones = []
        if cfg.get("debug_clone"):
            # after the HookPoints, so both see the same tensors in order
            self._tf_handles += _clone_hooks(model, self._tf_clones,
                                             lambda: self._tf_step - 1, sites)
        self._tf_sched = None
        self._tf_host_s = 0.0
        self._tf_steps = 0
        inner_forward = runner._model_forward

        def observed_forward(*a, **kw):
            self._tf_begin(kw.get("input_ids"), kw.get("positions"))
            try:
                return inner_forward(*a, **kw)
            finally:
                obs.end_step()
                if dbg_rows:
                    self._tf_graph_clones()
        runner._model_forward = observed_forward
        self._tf_dbg_rows = {reg.hooks[h].name: dbg_rows[reg.hooks[h].name]
                             for h in obs.debug_clone}

    def _tf_graph_clones(self):
        """Debug: read back the per-hook clone buffers after a forward
        (eager, piecewise or full graph alike) as (step, hook, rows)."""
        import torch
        step = self._tf_step - 1
        if not self._tf_layouts.get(step):
            return
        torch.cuda.current_stream().synchronize()
        rows = self._tf_rows_total
        for hid, buf in self._tf_obs.debug_clone.items():
            name = self._tf_obs.registry.hook(hid).name
            rb = self._tf_dbg_rows[name]
            self._tf_clones.append((step, name, buf[:rows * rb].view(rows, rb).cpu()))

    def execute_model(self, scheduler_output):
        self._tf_sched = scheduler_output
        try:
            return super().execute_model(scheduler_output)
        finally:
            self._tf_sched = None

    def _tf_begin(self, input_ids, positions):
        obs = self._tf_obs
        t0 = time.perf_counter()
        so = self._tf_sched
        rows_total = (input_ids if input_ids is not None else positions).shape[0]
        batch = []
        if so is not None:
            for rid in getattr(so, "finished_req_ids", ()):  # ids of finished requests
                self._tf_req.pop(rid, None)
            ib = self.model_runner.input_batch
            sched = so.num_scheduled_tokens
            for rid in ib.req_ids:
                n = sched.get(rid, 0)
                if n <= 0:
                    continue
                ent = self._tf_req.get(rid)
                if ent is None:  # first sight: next arrival index
                    ent = self._tf_next_id
                    self._tf_next_id += 1
                    self._tf_req[rid] = ent
                start = int(ib.num_computed_tokens_cpu[ib.req_id_to_index[rid]])
                batch.append(StepRequest(ent, ent, "", int(n), start))
        self._tf_rows_total = int(rows_total)
        # dummy / warm-up forwards get an empty batch: every row dropped
        obs.begin_step(batch, self._tf_step, layout="flat", rows_total=rows_total)
        if (self._tf_cfg.get("debug_clone") or self._tf_cfg.get("debug_graph_clone")
                or self._tf_cfg.get("sink") == "list"):
            self._tf_layouts[self._tf_step] = [(r.request_id, r.tokens) for r in batch]
        self._tf_step += 1
        self._tf_steps += 1
        self._tf_host_s += time.perf_counter() - t0

    # -- introspection (collective_rpc("observer_stats")) -------------------

    def observer_stats(self) -> dict:
        obs = self._tf_obs
        if obs is None:
            return {}
        st = obs.ring.state()
        ex = obs.exporter.stats()
        return {"steps": self._tf_steps, "host_begin_step_s": self._tf_host_s,
                "launches": obs.launches, "records": self._tf_sink.records_written,
                "bytes": self._tf_sink.bytes_written, "by_hook": dict(self._tf_sink.by_hook),
                "drops": st.drops, "stall_events": st.stall_events,
                "captures": st.captures_launched, "exporter": ex}

    def observer_debug(self) -> dict:
        """Records, per-step layouts and reference clones (sink="list",
        debug_clone=true; in-process engines only)."""
        recs = [(r.hook_name, r.step_seq, r.request_id, r.shape, bytes(r.payload))
                for r in getattr(self._tf_sink, "records", [])]
        return {"records": recs, "layouts": dict(self._tf_layouts),
                "clones": list(self._tf_clones)}

    def observer_flush(self, timeout: float = 120.0) -> None:
        if self._tf_obs is not None:
            self._tf_obs.flush(timeout)


__all__ = ["ObservedWorker", "attach_vllm_llama", "vllm_llama_specs", "observer_config"]
