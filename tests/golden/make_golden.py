"""Generate golden vectors by importing the reference (tapflow) itself.

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

The outputs are small JSON fixtures committed next to this script; the GPU
box (no /root/reference) checks the oracle and the CUDA path against them.
Every generator below replays the reference's own seeded test recipes
(PKG/tests/test_acceptance.py, test_rings.py, test_hooks.py,
test_policy.py) and records the reference's answers.
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys
from pathlib import Path

sys.dont_write_bytecode = True
REF = Path(os.environ.get("TAPFLOW_SRC", "/root/reference/pkg/src"))
sys.path.insert(0, str(REF))

from tapflow.errors import MetaRingFull, PayloadRingFull  # noqa: E402
from tapflow.hooks import (DType, HookSpec, ModelSpec, TensorView,  # noqa: E402
                           capture, install_hooks)
from tapflow.oracle import reference_records  # noqa: E402
from tapflow.policy import (BEST_EFFORT, COMPLETENESS, DROP_RECENT,  # noqa: E402
                            KEEP_BY_PATTERN, PolicyConfig, Predicate,
                            StepRequest, prepare_step)
from tapflow.rings import (Descriptor, RingConfig, allocate_rings,  # noqa: E402
                           round_up_to_copy_unit)
from tapflow.sinks import record_header, records_to_stream_bytes  # noqa: E402
from tapflow.workload import (WorkloadSpec, build_requests,  # noqa: E402
                              build_schedule, request_payload)

OUT = Path(__file__).resolve().parent


def h16(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()[:32]


def descriptors():
    rng = random.Random(1234)
    cases = [(4096, 48, 7, 3, 12), (0, 0, 0, 0, 0),
             (2**64 - 16, 2**64 - 1, 2**32 - 1, 2**32 - 1, 2**64 - 1),
             (0x1122334455667788, 0xAABBCCDDEEFF0011, 0x01020304, 0x05060708,
              0x1111222233334444)]
    for _ in range(60):
        cases.append((rng.randrange(2**64), rng.randrange(2**64),
                      rng.randrange(2**32), rng.randrange(2**32),
                      rng.randrange(2**64)))
    return [{"fields": list(c), "hex": Descriptor(*c).pack().hex()} for c in cases]


def ring_script(seed, capacity, meta_slots, n_ops, max_units):
    """Mixed protocol script with the reference's answer for every op."""
    rng = random.Random(seed)
    ring = allocate_rings(RingConfig(capacity, meta_slots))
    unpublished, unreleased, ops = [], [], []
    step = 0
    while len(ops) < n_ops:
        op = rng.choice(("R", "R", "P", "Q", "L", "L"))
        if op == "R":
            length = 16 * rng.randint(1, max_units)
            try:
                off = ring.reserve_payload(length)
                unpublished.append((off, length))
                ops.append(["R", length, off])
            except PayloadRingFull:
                ops.append(["R", length, None])
        elif op == "P" and unpublished:
            off, length = unpublished[0]
            hook, stp = rng.randint(0, 2**31), step
            step += 1
            try:
                seq = ring.publish(Descriptor(off, length, hook, stp))
                unpublished.pop(0)
                ops.append(["P", off, length, hook, stp, seq])
            except MetaRingFull:
                ops.append(["P", off, length, hook, stp, None])
        elif op == "Q":
            k = rng.randint(1, 4)
            got = ring.poll_ready(k)
            ops.append(["Q", k, [[d.payload_offset, d.payload_len, d.hook_id,
                                  d.step_seq, d.ready_seq] for d in got]])
            unreleased.extend((d.payload_offset, d.reserved_len) for d in got)
        elif op == "L" and unreleased:
            off, length = unreleased.pop(0)
            ring.release_payload(off, length)
            ops.append(["L", off, length])
        else:
            continue
        if len(ops) % 50 == 0:
            s = ring.state()
            ops.append(["S", s.payload_head, s.payload_tail, s.occupancy,
                        s.meta_head, s.meta_tail, ring.dead_created,
                        ring.dead_reclaimed])
    return {"capacity": capacity, "meta_slots": meta_slots, "ops": ops}


def reserve_release_scripts():
    """Hypothesis-style reserve/release-only scripts (test_rings.py:245-271)."""
    rng = random.Random(99)
    out = []
    for _ in range(150):
        cap_units = rng.randint(2, 12)
        capacity = cap_units * 16
        ring = allocate_rings(RingConfig(capacity, 64))
        outstanding, ops = [], []
        for _ in range(rng.randint(0, 60)):
            is_reserve, units = rng.random() < 0.5, rng.randint(1, 8)
            length = units * 16
            if is_reserve and length <= capacity:
                try:
                    off = ring.reserve_payload(length)
                    outstanding.append((off, length))
                    ops.append(["R", length, off, ring.occupancy])
                except PayloadRingFull:
                    ops.append(["R", length, None, ring.occupancy])
            elif outstanding:
                off, length = outstanding.pop(0)
                ring.release_payload(off, length)
                ops.append(["L", off, length, ring.occupancy])
        out.append({"capacity": capacity, "ops": ops})
    return out


def gather_cases():
    """test_acceptance.py:225-256 recipe (random.Random(7)), 2000 cases."""
    rng = random.Random(7)
    widths = {1: "u8", 2: "bf16", 4: "f32", 8: "f64"}
    cases = []
    for case in range(2000):
        batch = rng.randint(1, 8)
        tokens = rng.randint(1, 9)
        feat = rng.randint(1, 33)
        dtype = DType.of(widths[rng.choice((1, 2, 4, 8))])
        slice_size = tokens * feat * dtype.width
        data = rng.randbytes(batch * slice_size)
        keep = [rng.randint(0, 1) for _ in range(batch)]
        view = TensorView(data, (batch, tokens, feat), dtype)
        reg = install_hooks(ModelSpec(1, 16),
                            [HookSpec(f"case{case}", (tokens, feat), dtype)])
        ring = allocate_rings(RingConfig(32 << 10, 8))
        out = capture(reg, ring, reg.enabled_ids()[0], view, keep)
        got = b""
        if out.bytes_written:
            (d,) = ring.poll_ready(1)
            got = bytes(ring.payload_view(d.payload_offset, d.payload_len))
        cases.append({"batch": batch, "tokens": tokens, "feat": feat,
                      "width": dtype.width, "keep": keep,
                      "len": len(got), "sha": h16(got)})
    return cases


def policy_cases():
    rng = random.Random(0xBEEF)
    cases = []
    for i in range(300):
        layers = rng.randint(1, 3)
        hidden = rng.choice([8, 16, 17, 32])
        specs = [HookSpec("resid", ("tokens", "hidden"), DType.of("u8"),
                          per_layer=True)]
        if rng.random() < 0.5:
            specs.append(HookSpec("logits", ("tokens", rng.choice([4, 12])),
                                  DType.of("f16")))
        reg = install_hooks(ModelSpec(layers, hidden), specs)
        cap = 16 * rng.randint(2, 64)
        slots = rng.randint(2, 16)
        ring = allocate_rings(RingConfig(cap, slots))
        script = []
        outstanding = []
        for _ in range(rng.randint(0, 8)):
            if outstanding and rng.random() < 0.4:
                off, ln = outstanding.pop(0)
                ring.release_payload(off, ln)
                script.append(["L", off, ln])
            else:
                ln = 16 * rng.randint(1, max(1, cap // 64))
                try:
                    off = ring.reserve_payload(ln)
                    outstanding.append((off, ln))
                    script.append(["R", ln, off])
                except PayloadRingFull:
                    script.append(["R", ln, None])
        n = rng.randint(1, 7)
        tokens = rng.randint(1, 3)
        arrivals = list(range(n))
        rng.shuffle(arrivals)
        batch = [StepRequest(100 + j, arrivals[j],
                             rng.choice(["hot x", "cold y"]) + str(j),
                             tokens, rng.randint(0, 5)) for j in range(n)]
        kind = rng.choice(["comp", "drop", "kbp_ids", "kbp_prefix"])
        if kind == "comp":
            pol = PolicyConfig(mode=COMPLETENESS,
                               pressure_watermark=rng.choice([0.5, 0.8, 1.0]))
            pdesc = {"mode": "completeness", "watermark": pol.pressure_watermark}
        elif kind == "drop":
            pol = PolicyConfig(mode=BEST_EFFORT, strategy=DROP_RECENT)
            pdesc = {"mode": "best-effort", "strategy": "drop-recent"}
        elif kind == "kbp_ids":
            ids = sorted(r.request_id for r in batch if rng.random() < 0.4)
            pol = PolicyConfig(mode=BEST_EFFORT, strategy=KEEP_BY_PATTERN,
                               predicate=Predicate(request_ids=frozenset(ids)))
            pdesc = {"mode": "best-effort", "strategy": "keep-by-pattern",
                     "ids": ids}
        else:
            pol = PolicyConfig(mode=BEST_EFFORT, strategy=KEEP_BY_PATTERN,
                               predicate=Predicate(prompt_prefix="hot"))
            pdesc = {"mode": "best-effort", "strategy": "keep-by-pattern",
                     "prefix": "hot"}
        plan = prepare_step(pol, batch, ring, reg, step_seq=i,
                            rank_coords=(0, 0))
        cases.append({
            "layers": layers, "hidden": hidden,
            "specs": [[s.name, list(s.dims), s.dtype.name, s.per_layer]
                      for s in specs],
            "capacity": cap, "slots": slots, "script": script,
            "batch": [[r.request_id, r.arrival_index, r.prompt, r.tokens,
                       r.token_start] for r in batch],
            "policy": pdesc, "step": i,
            "expect": {
                "keep": list(plan.keep), "flush": plan.flush_before,
                "kept": list(plan.kept_ids), "dropped": list(plan.dropped_ids),
                "flagged": list(plan.flagged_ids),
                "free": plan.free_bytes_at_plan,
                "fifo": [[m.hook_name, m.layer_index, list(m.shape),
                          m.dtype.name, list(m.request_ids),
                          [list(t) for t in m.token_ranges],
                          m.expected_payload_len] for m in plan.fifo_entries],
            }})
    return cases


def workload_vectors():
    out = {"payloads": [], "records": []}
    rng = random.Random(5)
    for _ in range(40):
        hook = HookSpec(rng.choice(["resid", "attn_out", "logits"]),
                        ("tokens", "hidden"), DType.of("bf16"),
                        layer_index=rng.choice([None, 0, 3]))
        seed, rid, step = rng.randint(0, 99), rng.randint(0, 9), rng.randint(0, 20)
        tokens, hidden = rng.randint(1, 8), rng.choice([16, 64])
        data = request_payload(seed, hook, rid, step, tokens, hidden)
        out["payloads"].append({"seed": seed, "name": hook.name,
                                "layer": hook.layer_index, "rid": rid,
                                "step": step, "nbytes": len(data),
                                "sha": h16(data)})
    # one small lossless run's full record set (oracle.py reference_records)
    wl = WorkloadSpec(layers=3, hidden=32, batch=3, prefill_tokens=4,
                      decode_steps=3, prefill_compute_time=2e-3,
                      decode_compute_time=1e-3, arrival=(2, 1))
    specs = [HookSpec("resid", ("tokens", "hidden"), DType.of("bf16"),
                      per_layer=True),
             HookSpec("logits", ("tokens", 8), DType.of("f32"))]
    reg = install_hooks(wl.model, specs)
    sched = build_schedule(wl, build_requests(wl, 11))
    recs = reference_records(11, sched, reg)
    out["workload"] = {"layers": 3, "hidden": 32, "batch": 3,
                       "prefill_tokens": 4, "decode_steps": 3, "seed": 11,
                       "arrival": [2, 1]}
    out["records"] = [[r.request_id, r.hook_name, r.layer_index, r.step_seq,
                       list(r.token_range), list(r.shape), r.dtype.name,
                       r.checksum] for r in recs]
    out["schedule"] = [[s.step_seq, s.kind,
                        [[q.request_id, q.arrival_index, q.prompt, q.tokens,
                          q.token_start] for q in s.batch]] for s in sched]
    return out


def sink_vectors():
    from tapflow.records import CaptureRecord
    recs = [CaptureRecord(7, "resid[2]", 2, 5, (4, 8), (4, 2), DType.of("bf16"),
                          (0, 0), bytes(range(16))),
            CaptureRecord(9, "logits", None, 6, (8, 9), (1, 3), DType.of("f32"),
                          (1, 0), bytes(range(100, 112)))]
    import json as _j
    lines = [_j.dumps(record_header(r, off), separators=(",", ":"))
             for r, off in zip(recs, (0, 16))]
    return {"lines": lines, "stream_hex": records_to_stream_bytes(recs).hex()}


def main() -> None:
    fixtures = {
        "descriptors.json": descriptors(),
        "ring_script.json": [ring_script(42, 1024, 32, 20000, 16),
                             ring_script(0xC0FFEE, 640, 8, 5000, 6),
                             ring_script(3, 4096, 3, 3000, 40)],
        "reserve_release.json": reserve_release_scripts(),
        "gather_cases.json": gather_cases(),
        "policy_cases.json": policy_cases(),
        "workload.json": workload_vectors(),
        "sinks.json": sink_vectors(),
    }
    for name, data in fixtures.items():
        (OUT / name).write_text(json.dumps(data, separators=(",", ":")))
        print(name, (OUT / name).stat().st_size)


if __name__ == "__main__":
    main()
