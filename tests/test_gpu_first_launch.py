"""Regression test for a deadlock between CUDA's lazy kernel loading and a
capture that waits on the device: in a fresh process, a step recorded as a
CUDA graph whose captures overflow the ring is replayed without any other
launch of the library's kernels first (no flush, no snapshot), so the first
seal-kernel launch at end_step happens while captures wait for the staging
engine. Kernels are loaded at ring creation (ring2.cu preload_kernels);
before that this hung. Runs in a subprocess so no earlier test has loaded
the kernels already."""

import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent("""
    import sys, torch
    sys.path.insert(0, {root!r})
    from paper_2605_11093_b200 import (DrainConfig, DType, HookSpec, ModelSpec,
                                       RingConfig, StepRequest, install_hooks)
    from paper_2605_11093_b200.hookpoint import HookPoint, Observer
    from paper_2605_11093_b200.sinks import NullSink
    B, T, H, L = 8, 64, 2048, 8          # 2 MiB per capture, 16 MiB per step
    reg = install_hooks(ModelSpec(L, H), [HookSpec("resid", ("tokens", "hidden"),
                                                   DType.of("bf16"), per_layer=True)])
    obs = Observer(reg, ring=RingConfig(6 << 20, 64), sink=NullSink(), max_batch=B,
                   drain=DrainConfig(min_ready_entries=1, staging_buffer_size=4 << 20,
                                     staging_buffer_count=3))
    obs.start()
    hps = [HookPoint(f"resid[{{i}}]", obs) for i in range(L)]
    x = torch.randn(B, T, H, dtype=torch.bfloat16, device="cuda")
    ys = [torch.empty_like(x) for _ in range(L)]
    def body():
        for i in range(L):
            ys[i].copy_(x * (i + 1))
            hps[i](ys[i])
    g = torch.cuda.CUDAGraph()
    with obs.graph_capture(), torch.cuda.graph(g):
        body()
    for step in range(6):                 # no flush before the first replay
        obs.begin_step([StepRequest(i, i, "p", T, 0) for i in range(B)], step)
        g.replay()
        obs.end_step()
    obs.flush(60)
    st = obs.ring.state()
    obs.close()
    assert st.drops == 0, st
    print("FIRST_LAUNCH_OK", st.stall_events)
""")


def test_graph_replay_with_device_waits_before_any_other_launch():
    res = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)],
                         capture_output=True, text=True, timeout=180, cwd=ROOT)
    assert res.returncode == 0 and "FIRST_LAUNCH_OK" in res.stdout, \
        (res.stdout[-2000:], res.stderr[-3000:])
