"""Synthetic workload source and the dataset verifier.

The package's workload keying (paper_2605_11093_b200/workload.py) is pinned
to the reference's golden hashes and schedule (tests/golden/workload.json,
made by importing the reference) and to the independent oracle
restatement; ``verify`` is checked on datasets written here (CPU) and, in
the GPU half, on datasets the capture path produced (lossless and
best-effort with a keep log)."""

import hashlib
import json
import zlib

import pytest

from oracle import workload as W
from paper_2605_11093_b200 import (BEST_EFFORT, COMPLETENESS, DROP_RECENT, DrainConfig, DType,
                                   HookSpec, ModelSpec, PolicyConfig, RingConfig,
                                   install_hooks)
from paper_2605_11093_b200.sinks import FileSink
from paper_2605_11093_b200.verify import (META_NAME, hook_to_dict, main,
                                          reference_records, run_synthetic,
                                          verify_dataset)
from paper_2605_11093_b200.workload import (WorkloadSpec, build_requests,
                                            build_schedule, request_payload)

BF16, F32 = DType.of("bf16"), DType.of("f32")
HOOKS = [HookSpec("resid", ("tokens", "hidden"), BF16, per_layer=True),
         HookSpec("logits", ("tokens", 8), F32)]


def _golden_setup(golden):
    wl = golden("workload.json")["workload"]
    spec = WorkloadSpec(wl["batch"], wl["prefill_tokens"], wl["decode_steps"],
                        tuple(wl["arrival"]))
    model = ModelSpec(wl["layers"], wl["hidden"])
    return wl, spec, model


def test_schedule_and_records_match_reference_golden(golden):
    g = golden("workload.json")
    wl, spec, model = _golden_setup(golden)
    sched = build_schedule(spec, build_requests(spec, wl["seed"]))
    assert [[s.step_seq, s.kind, [[r.request_id, r.arrival_index, r.prompt, r.tokens,
                                   r.token_start] for r in s.batch]] for s in sched] == \
        g["schedule"]
    reg = install_hooks(model, HOOKS)
    recs = reference_records(wl["seed"], sched, reg)
    assert [[r.request_id, r.hook_name, r.layer_index, r.step_seq, list(r.token_range),
             list(r.shape), r.dtype.name, zlib.crc32(r.payload)] for r in recs] == g["records"]


def test_content_keying_equals_oracle_restatement():
    reg = install_hooks(ModelSpec(3, 48), HOOKS)
    for seed in (0, 7, 94):
        for hid in reg.enabled_ids():
            h = reg.hook(hid)
            for rid, step, tokens in ((0, 0, 4), (5, 20, 1), (2, 3, 7)):
                n = tokens * (48 if h.dims[1] == "hidden" else 8) * h.dtype.width
                assert request_payload(seed, h, rid, step, tokens, 48) == \
                    W.request_payload(seed, h.name, h.layer_index, rid, step, n)


def _write_reference_dataset(path, golden, keep_log=None, drop_step=None):
    wl, spec, model = _golden_setup(golden)
    sched = build_schedule(spec, build_requests(spec, wl["seed"]))
    reg = install_hooks(model, HOOKS)
    log = keep_log or {s.step_seq: tuple(r.request_id for r in s.batch) for s in sched}
    recs = reference_records(wl["seed"], sched, reg, keep_log=log)
    with FileSink(path) as sink:
        sink.write(recs)
    meta = {"seed": wl["seed"], "hook_filter": None,
            "keep_log": {str(k): list(v) for k, v in log.items()},
            "workload": {"batch": spec.batch, "prefill_tokens": spec.prefill_tokens,
                         "decode_steps": spec.decode_steps, "arrival": list(spec.arrival)},
            "model": {"layers": model.layers, "hidden": model.hidden},
            "hooks": [hook_to_dict(h) for h in HOOKS]}
    (path / META_NAME).write_text(json.dumps(meta))
    return recs


def test_verify_accepts_exact_and_rejects_corruption(golden, tmp_path, capsys):
    ds = tmp_path / "ds"
    _write_reference_dataset(ds, golden)
    ok, rep = verify_dataset(ds)
    assert ok and rep["records"] == rep["expected"] > 0
    assert main([str(ds)]) == 0
    blob = bytearray((ds / "records.bin").read_bytes())
    blob[100] ^= 0xFF
    (ds / "records.bin").write_bytes(bytes(blob))
    ok, rep = verify_dataset(ds)
    assert not ok and rep["corrupt"] == 1 and rep["bad_checksums"] == 1
    assert main([str(ds)]) == 1


def test_verify_keep_log_narrows_and_flags_missing(golden, tmp_path):
    wl, spec, _ = _golden_setup(golden)
    sched = build_schedule(spec, build_requests(spec, wl["seed"]))
    keep = {s.step_seq: tuple(r.request_id for r in s.batch if r.request_id != 1)
            for s in sched}
    ds = tmp_path / "be"
    _write_reference_dataset(ds, golden, keep_log=keep)
    assert verify_dataset(ds)[0]
    lines = (ds / "records.ndjson").read_text().splitlines()
    (ds / "records.ndjson").write_text("\n".join(lines[1:]) + "\n")
    ok, rep = verify_dataset(ds)
    assert not ok and rep["missing"] == 1


def test_verify_without_meta_is_a_config_error(tmp_path):
    (tmp_path / "x").mkdir()
    assert main([str(tmp_path / "x")]) == 2


@pytest.mark.gpu
@pytest.mark.parametrize("policy,ring", [
    (COMPLETENESS, RingConfig(1 << 20, 64)),
    (BEST_EFFORT, RingConfig(96 << 10, 64)),   # too small for whole steps: drops
])
def test_gpu_run_verifies(tmp_path, policy, ring):
    spec = WorkloadSpec(5, 16, 6, (3, 0, 2))
    meta = run_synthetic(tmp_path / "run", spec=spec, model=ModelSpec(4, 256), hooks=HOOKS,
                         seed=2605, ring=ring,
                         policy=PolicyConfig(mode=policy, strategy=DROP_RECENT)
                         if policy == BEST_EFFORT else PolicyConfig(mode=policy),
                         drain=DrainConfig(min_ready_entries=1, staging_buffer_size=1 << 20))
    ok, rep = verify_dataset(tmp_path / "run")
    assert ok, rep
    kept = sum(len(v) for v in meta["keep_log"].values())
    full = sum(len(s.batch) for s in build_schedule(spec, build_requests(spec, 2605)))
    if policy == COMPLETENESS:
        assert kept == full
    assert rep["records"] == kept * 5          # 4 resid layers + logits
    digest = hashlib.sha1((tmp_path / "run" / "records.bin").read_bytes()).hexdigest()
    assert digest
