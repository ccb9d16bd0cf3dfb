"""vLLM 0.22 integration (BASELINE configs[3]) on a tiny
random-init Llama, each mode in its own process (scripts/vllm_check.py):
eager mode is bit-exact against torch hooks at the same sites; CUDA-graph
mode (the serving configuration) is bit-exact against a debug copy of each
observed tensor recorded into the same graphs beside the capture kernel,
for every record of every replay, across padded decode batch sizes; both
deliver exactly one record per step, hook and scheduled request."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(mode, *extra):
    pytest.importorskip("vllm")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "vllm_check.py"),
                          "--mode", mode, *extra], capture_output=True, text=True,
                         timeout=1200, cwd=ROOT)
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert res.returncode == 0 and lines, res.stderr[-3000:]
    return json.loads(lines[-1])


def test_vllm_eager_records_bit_exact():
    out = _run("eager")
    assert out["ok"], json.dumps(out)


def test_vllm_cuda_graph_records_bit_exact():
    out = _run("graph")
    assert out["ok"], json.dumps(out)
    assert out["bit_exact_checked"] == out["expected"] and out["steps_with_padding"] > 0


def test_vllm_cuda_graph_overlap_records_bit_exact():
    """Overlap mode inside vLLM's graphs: captures forked onto a side stream
    and joined before each attention op (before the residual is rewritten in
    place, and before each piecewise graph ends)."""
    out = _run("graph", "--overlap")
    assert out["ok"], json.dumps(out)
    assert out["bit_exact_checked"] == out["expected"]
