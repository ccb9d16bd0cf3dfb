"""Multi-process plumbing on CPU (gloo, world_size 2): replicas only — no
data-path collective; ranks meet only for the barrier and the
max-over-ranks / sum-over-ranks reduction of the bench numbers."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _worker(rank, world, port, q, replicas=1):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, str(ROOT))
    import bench
    d = bench.Dist(replicas)
    d.barrier()
    s = d.reduce([10.0 * (rank + 1)], "sum")[0]
    m = d.reduce([float(rank + 3)], "max")[0]
    q.put((rank, s, m, d.local, d.backend))
    d.close()


def test_dist_reduce_sum_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 2000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    got = sorted(q.get(timeout=5) for _ in range(2))
    assert [g[:3] for g in got] == [(0, 30.0, 4.0), (1, 30.0, 4.0)]
    assert [g[3] for g in got] == [0, 1]


def test_two_replicas_per_gpu_share_the_device_over_gloo():
    # bench.py --replicas-per-gpu 2: ranks 0 and 1 both drive device 0 and
    # meet over gloo (NCCL rejects two ranks on one device)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 33500 + os.getpid() % 2000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, 2)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    got = sorted(q.get(timeout=5) for _ in range(2))
    assert [g[:3] for g in got] == [(0, 30.0, 4.0), (1, 30.0, 4.0)]
    assert [g[3] for g in got] == [0, 0]
    assert {g[4] for g in got} == {"gloo"}


def test_reference_arm_prints_once_under_torchrun():
    port = 31500 + os.getpid() % 2000
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(ROOT / "bench.py"), "--impl",
           "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
           "--batch", "1", "--seq", "4"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300,
                         cwd=ROOT, env={**os.environ, "OMP_NUM_THREADS": "1"})
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["value"] > 0
    assert rec["e2e"]["h2d_bytes_per_step"] == 0
    assert rec["cpu_baseline"]["kind"] in ("reference", "port")
