"""Device timeline of the Llama-3-8B prefill step with capture and staging
(the evidence nsys would give; nsys is not in this image, so CUPTI through
torch.profiler records every kernel and memcpy of the process, including the
staging engine's D2H on its own stream).

For each mode -- no capture, copy-engine staging, mapped-store staging --
runs a few 8x512 prefill steps of random-init Llama-3-8B as a CUDA graph with
resid_post + mlp_act captured at every layer (completeness, 2 GiB ring) and
reports per step: model-kernel time (sum of kernel durations that are not
ours), capture-kernel time, staging-kernel time (mapped mode), D2H bytes and
busy time, and how much of the D2H busy time overlaps kernel execution.
Writes one JSON line per mode and a gzipped Chrome trace per mode.

usage: python scripts/exp_timeline.py [--steps 4] [--out gpurun_out/timeline]
"""
import argparse
import faulthandler
import gzip
import json
import os
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11093_b200 import DrainConfig, NullSink, PolicyConfig, RingConfig, StepRequest  # noqa: E402
from paper_2605_11093_b200.hookpoint import Observer  # noqa: E402
from paper_2605_11093_b200.integrations import (attach_llama, detach, llama3_8b_config,  # noqa: E402
                                                llama_registry, random_llama)

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--out", default="gpurun_out/timeline")
ap.add_argument("--modes", default="off,copy-engine,mapped")
ap.add_argument("--unsealed", action="store_true", help="Observer(sealed=False)")
ap.add_argument("--no-flush", action="store_true",
                help="no observer flush between recording the graph and the first replay "
                     "(the first seal / snapshot launches then happen while captures wait)")
args = ap.parse_args()
os.makedirs(args.out, exist_ok=True)

dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
B, T = 8, 512
cfg = llama3_8b_config()
model = random_llama(cfg, device=str(dev))
ids = torch.randint(0, cfg.vocab_size, (B, T), device=dev,
                    generator=torch.Generator(device=dev).manual_seed(7))
stream = torch.cuda.current_stream(dev)
batch = [StepRequest(i, i, f"p{i}", T, 0) for i in range(B)]
OURS = ("capture_kernel", "mapped_copy_kernel", "seal_kernel", "snapshot_kernel",
        "reserve_kernel", "publish_kernel")


def make_graph(obs=None):
    cs = torch.cuda.Stream(device=dev)
    cs.wait_stream(stream)
    with torch.cuda.stream(cs), torch.inference_mode():
        for _ in range(2):
            model.model(input_ids=ids, use_cache=False)
    stream.wait_stream(cs)
    g = torch.cuda.CUDAGraph()
    if obs is None:
        with torch.inference_mode(), torch.cuda.graph(g):
            model.model(input_ids=ids, use_cache=False)
    else:
        with obs.graph_capture(), torch.inference_mode(), torch.cuda.graph(g):
            model.model(input_ids=ids, use_cache=False)
    return g


def union(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def overlap(a, b):
    """Total length of the intersection of two interval unions."""
    i = j = 0
    tot = 0.0
    while i < len(a) and j < len(b):
        lo, hi = max(a[i][0], b[j][0]), min(a[i][1], b[j][1])
        if hi > lo:
            tot += hi - lo
        if a[i][1] < b[j][1]:
            i += 1
        else:
            j += 1
    return tot


def summarise(trace, steps, wall_ms):
    ev = [e for e in trace.get("traceEvents", []) if e.get("ph") == "X"]
    kern = [e for e in ev if e.get("cat") == "kernel"]
    mem = [e for e in ev if e.get("cat") in ("gpu_memcpy", "gpu_memset")]
    ours = [e for e in kern if any(k in e.get("name", "") for k in OURS)]
    model = [e for e in kern if not any(k in e.get("name", "") for k in OURS)]
    cap = [e for e in ours if "capture_kernel" in e["name"]]
    mapped = [e for e in ours if "mapped_copy_kernel" in e["name"]]
    d2h = [e for e in mem if "DtoH" in e.get("name", "") or "Device -> Pinned" in e.get("name", "")
           or "D2H" in e.get("name", "")]
    d2h_bytes = sum(int((e.get("args") or {}).get("bytes", 0)) for e in d2h)
    k_iv = union([[e["ts"], e["ts"] + e["dur"]] for e in kern])
    d_iv = union([[e["ts"], e["ts"] + e["dur"]] for e in d2h])
    d_busy = sum(b - a for a, b in d_iv)
    return {"steps": steps, "wall_ms_per_step": wall_ms,
            "model_kernel_ms_per_step": sum(e["dur"] for e in model) / 1e3 / steps,
            "model_kernels_per_step": len(model) / steps,
            "capture_kernel_ms_per_step": sum(e["dur"] for e in cap) / 1e3 / steps,
            "mapped_staging_kernel_ms_per_step": sum(e["dur"] for e in mapped) / 1e3 / steps,
            "d2h_gb_per_step": d2h_bytes / 1e9 / steps,
            "d2h_busy_ms_per_step": d_busy / 1e3 / steps,
            "d2h_gbs_while_busy": d2h_bytes / (d_busy * 1e-6) / 1e9 if d_busy else None,
            "d2h_busy_overlapping_kernels": overlap(d_iv, k_iv) / d_busy if d_busy else None,
            "memcpy_names": sorted({e.get("name", "") for e in mem})[:6]}


def log(m):
    print(f"[timeline {time.perf_counter() - T0:7.1f}s] {m}", file=sys.stderr, flush=True)


T0 = time.perf_counter()
faulthandler.dump_traceback_later(240, repeat=True)  # where a hang sits
for mode in args.modes.split(","):
    log(f"mode {mode}")
    obs = handles = None
    if mode != "off":
        reg = llama_registry(cfg, ("mlp_act", "resid_post"))
        obs = Observer(reg, ring=RingConfig(2 << 30, 1024),
                       drain=DrainConfig(min_ready_entries=1, min_ready_bytes=1, max_wait=1e-4,
                                         staging_buffer_size=128 << 20, staging_buffer_count=12,
                                         mode=mode, stage_threads=4, page_out="handoff"),
                       policy=PolicyConfig(), sink=NullSink(), device=0, max_batch=B,
                       sealed=not args.unsealed)
        obs.exporter.copy_payloads = False
        obs.start()
        handles = attach_llama(model, obs, ("mlp_act", "resid_post"))
    g = make_graph(obs)

    def step(s):
        if obs is not None:
            obs.begin_step(batch, s)
        g.replay()
        if obs is not None:
            obs.end_step(stream)

    log("graph recorded")
    if obs is not None:
        if not args.no_flush:
            obs.flush(300)

        import threading

        def watch(o=obs):
            while o.exporter.running:
                time.sleep(20)
                try:
                    st = o.exporter.stats()
                    import ctypes
                    from paper_2605_11093_b200 import _native as N
                    rs = N.CRingState()
                    N.lib().tf_ring_get_state(o.ring.handle, ctypes.byref(rs))
                    log(f"watch: drained={st['bytes_drained']} batches={st['batches_drained']}/"
                        f"{st['batches_staged']} inflight={st['inflight_batches']} "
                        f"pool_free={st['pool_free']} occ={rs.occupancy} meta={rs.meta_head}/"
                        f"{rs.meta_tail} stalls={rs.stall_events} drops={rs.drops} "
                        f"err={rs.device_errors}")
                except Exception as exc:
                    log(f"watch: {exc!r}")
        threading.Thread(target=watch, daemon=True).start()
    for s in range(4):  # warm: the 2 GiB ring reaches its steady backlog
        step(s)
    torch.cuda.synchronize()
    log("warm")
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(args.steps):
            step(100 + s)
        e1.record(stream)
        e1.synchronize()
        log("steps done")
        if obs is not None:
            obs.flush(600)
        torch.cuda.synchronize()
    path = os.path.join(args.out, f"trace_{mode}.json")
    prof.export_chrome_trace(path)
    trace = json.load(open(path))
    with gzip.open(path + ".gz", "wt") as f:
        json.dump(trace, f)
    os.remove(path)
    line = {"mode": mode, **summarise(trace, args.steps, e0.elapsed_time(e1) / args.steps)}
    print(json.dumps(line), flush=True)
    if obs is not None:
        detach(handles)
        obs.close()
    del g
    torch.cuda.empty_cache()
