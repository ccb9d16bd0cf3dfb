"""Two replicas on one GPU, concurrently (the reference
analogue is run_multirank's independent per-rank instances,
SRC/simulator.py:158-192). Each process owns its Observer: ring pair,
staging engine, pinned pool and exporter, and captures content seeded by
its own rank. Records must stay isolated (every record equals its own
process's tensor, none of the other's), the byte accounting must add up,
and each staging engine must be bound to the GPU's PCIe-local CPUs."""

import os
import sys
import zlib
from pathlib import Path

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

LAYERS, B, T, H, STEPS = 4, 4, 64, 1024, 24


def _replica(rank, barrier, q):
    """Child entry: report a failure at once instead of leaving the parent
    waiting on the queue."""
    try:
        _replica_body(rank, barrier, q)
    except BaseException:
        import traceback
        q.put({"rank": rank, "error": traceback.format_exc()})
        raise


def _replica_body(rank, barrier, q):
    sys.path.insert(0, str(ROOT))
    import torch

    from paper_2605_11093_b200 import (DrainConfig, DType, HookSpec, ModelSpec,
                                       RingConfig, StepRequest, install_hooks)
    from paper_2605_11093_b200.hookpoint import HookPoint, Observer
    torch.cuda.set_device(0)
    reg = install_hooks(ModelSpec(LAYERS, H), [HookSpec("resid", ("tokens", "hidden"),
                                                        DType.of("bf16"), per_layer=True)])
    got = {}

    class Sink:
        def write(self, recs):
            for r in recs:
                got[(r.hook_name, r.request_id, r.step_seq)] = zlib.crc32(r.payload)

    # a small ring: both replicas wrap and wait for their own consumer
    obs = Observer(reg, ring=RingConfig(8 << 20, 64), sink=Sink(), max_batch=B,
                   drain=DrainConfig(min_ready_entries=2, staging_buffer_size=2 << 20,
                                     staging_buffer_count=3))
    obs.start()
    hps = [HookPoint(f"resid[{L}]", obs) for L in range(LAYERS)]
    want = {}
    g = torch.Generator().manual_seed(1000 + rank)
    reqs = [StepRequest(10 * rank + i, i, "p", T, 0) for i in range(B)]
    # content made on the host and uploaded without a device sync in the
    # loop (a blocking copy would hold the GIL while the device may wait for
    # the exporter thread)
    host = [torch.empty(B, T, H, dtype=torch.int16).random_(-32768, 32767, generator=g)
            .view(torch.bfloat16).pin_memory() for _ in range(LAYERS * STEPS)]
    dev = [torch.empty(B, T, H, dtype=torch.bfloat16, device="cuda") for _ in host]
    barrier.wait(120)  # both replicas capture at the same time
    for step in range(STEPS):
        obs.begin_step(reqs, step)
        for L, hp in enumerate(hps):
            k = step * LAYERS + L
            dev[k].copy_(host[k], non_blocking=True)
            hp(dev[k])
            for i, r in enumerate(reqs):
                want[(f"resid[{L}]", r.request_id, step)] = zlib.crc32(
                    host[k][i].contiguous().view(torch.uint8).numpy().tobytes())
        obs.end_step()
    obs.flush(120)
    place = obs.exporter.placement()
    st = obs.ring.state()
    released = obs.ring.bytes_released
    obs.close()
    bad = sum(1 for k, c in want.items() if got.get(k) != c)
    q.put({"rank": rank, "records": len(got), "expected": len(want), "mismatch": bad,
           "foreign": sum(1 for k in got if k not in want),
           "bytes": released, "stalls": st.stall_events, "placement": place,
           "pid": os.getpid()})


def _local_cpus():
    import torch
    pr = torch.cuda.get_device_properties(0)
    try:
        bus = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
    except AttributeError:
        return None
    p = Path(f"/sys/bus/pci/devices/{bus}/local_cpulist")
    if not p.exists():
        return None
    out = set()
    for part in p.read_text().strip().split(","):
        a, _, b = part.partition("-")
        out.update(range(int(a), int(b or a) + 1))
    return out & os.sched_getaffinity(0)


def test_two_replicas_on_one_gpu_are_isolated_and_numa_bound():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    barrier = ctx.Barrier(2)
    procs = [ctx.Process(target=_replica, args=(r, barrier, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in procs), key=lambda d: d["rank"])
    for r in res:
        assert "error" not in r, r["error"]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    per = LAYERS * B * STEPS
    slice_bytes = T * H * 2
    for r in res:
        assert r["expected"] == per and r["records"] == per, r
        assert r["mismatch"] == 0 and r["foreign"] == 0, r
        # every kept byte was released exactly once (16-B padded regions)
        assert r["bytes"] == per // B * ((B * slice_bytes + 15) // 16 * 16), r
    assert res[0]["pid"] != res[1]["pid"]
    local = _local_cpus()
    for r in res:
        cpus = set(r["placement"]["cpus"])
        if local:
            assert cpus == local, (cpus, local)
        assert r["placement"]["pool_numa_node"] == res[0]["placement"]["pool_numa_node"]
