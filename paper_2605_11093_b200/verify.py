"""Verify a stored dataset against the deterministic reference, after the fact.

Mirrors ``tapflow --verify`` (SRC/cli.py:153-189, SRC/oracle.py:48-115): a
run on the GPU writes its dataset (records.ndjson + records.bin) and a
``run_meta.json`` next to it (seed, hook filter, the keep log of every
step, the workload and hooks); verification regenerates every record the
run owed from the synthetic workload's content keying, narrowed by the keep
log (so a best-effort run is checked to have dropped exactly what it said
it dropped and kept everything else intact), checks every stored crc32 and
compares the two as multisets, per hook.

    python -m paper_2605_11093_b200.verify DATASET     # 0 ok, 1 mismatch, 2 bad input

``run_synthetic`` is the matching producer: it drives the GPU capture path
(Observer + capture kernels + staging + sink) over the synthetic schedule.
"""

from __future__ import annotations

import json
import sys
import zlib
from collections import Counter
from dataclasses import dataclass
from pathlib import Path

from .errors import ConfigError, TapflowError
from .hooks import DType, HookSpec, ModelSpec, install_hooks
from .records import CaptureRecord
from .sinks import record_from_header, scan_dataset
from .workload import WorkloadSpec, build_requests, build_schedule, request_payload

META_NAME = "run_meta.json"          # SRC/cli.py:39


def hook_to_dict(h: HookSpec) -> dict:
    return {"name": h.name, "dims": list(h.dims), "dtype": h.dtype.name,
            "per_layer": h.per_layer, "layer_index": h.layer_index,
            "cast_to": h.cast_to.name if h.cast_to else None, "reduce": h.reduce}


def hook_from_dict(d: dict) -> HookSpec:
    return HookSpec(d["name"], tuple(d["dims"]), DType.of(d["dtype"]),
                    layer_index=d.get("layer_index"), per_layer=d.get("per_layer", False),
                    cast_to=DType.of(d["cast_to"]) if d.get("cast_to") else None,
                    reduce=d.get("reduce"))


def reference_records(seed: int, schedule, registry, keep_log=None) -> list:
    """Every record a lossless run owes (SRC/oracle.py:48-71), narrowed by
    ``keep_log`` (step -> kept request ids)."""
    out = []
    hidden = registry.hidden_extent
    for step in schedule:
        batch = step.batch
        if keep_log is not None:
            kept = set(keep_log.get(step.step_seq, ()))
            batch = tuple(r for r in batch if r.request_id in kept)
        if not batch:
            continue
        for hid in registry.enabled_ids():
            hook = registry.hook(hid)
            if hook.cast_to is not None or hook.reduce is not None:
                raise ConfigError(f"hook {hook.name!r} casts or reduces: its records "
                                  "are not reference bytes")
            shape = hook.resolve_shape(step.tokens, hidden)
            for r in batch:
                out.append(CaptureRecord(
                    r.request_id, hook.name, hook.layer_index, step.step_seq,
                    r.token_range, shape, hook.dtype, (0, 0),
                    request_payload(seed, hook, r.request_id, step.step_seq,
                                    step.tokens, hidden)))
    return out


@dataclass(frozen=True)
class DatasetDiff:
    """Multiset difference (SRC/oracle.py:74-115)."""

    missing: tuple
    unexpected: tuple
    corrupt: tuple

    @property
    def identical(self) -> bool:
        return not (self.missing or self.unexpected or self.corrupt)

    def per_hook_counts(self) -> dict:
        c = Counter()
        for k in self.missing + self.unexpected + self.corrupt:
            c[k[1]] += 1
        return dict(c)

    def summary(self) -> str:
        return (f"{len(self.missing)} missing, {len(self.unexpected)} unexpected, "
                f"{len(self.corrupt)} corrupt")


def _key(r) -> tuple:
    return (r.request_id, r.hook_name, r.layer_index, r.step_seq, tuple(r.rank_coords))


def compare_datasets(expected, actual) -> DatasetDiff:
    def sig(r):
        return (tuple(r.token_range), tuple(r.shape), r.dtype.name, bytes(r.payload))
    ek, ak = Counter(map(_key, expected)), Counter(map(_key, actual))
    missing = tuple((ek - ak).elements())
    unexpected = tuple((ak - ek).elements())
    esig = {}
    for r in expected:
        esig.setdefault(_key(r), Counter())[sig(r)] += 1
    asig = {}
    for r in actual:
        asig.setdefault(_key(r), Counter())[sig(r)] += 1
    corrupt = tuple(k for k in esig if k in asig and esig[k] != asig[k])
    return DatasetDiff(missing, unexpected, corrupt)


def verify_dataset(dataset) -> tuple:
    """(ok, report dict). Raises ConfigError on unusable input."""
    dataset = Path(dataset)
    meta_path = dataset / META_NAME
    if not meta_path.exists():
        raise ConfigError(f"no {META_NAME} next to the dataset at {dataset}")
    meta = json.loads(meta_path.read_text(encoding="utf-8"))
    seed = meta["seed"]
    keep_log = {int(s): tuple(ids) for s, ids in meta["keep_log"].items()}
    model = ModelSpec(**meta["model"])
    registry = install_hooks(model, [hook_from_dict(h) for h in meta["hooks"]])
    if meta.get("hook_filter") is not None:
        registry.set_hook_filter(list(meta["hook_filter"]))
    registry.commit_filter()
    w = meta["workload"]
    spec = WorkloadSpec(w["batch"], w["prefill_tokens"], w["decode_steps"],
                        tuple(w["arrival"]) if w.get("arrival") else None)
    schedule = build_schedule(spec, build_requests(spec, seed))
    expected = reference_records(seed, schedule, registry, keep_log=keep_log)
    actual, bad_crc = [], 0
    for header, payload in scan_dataset(dataset):
        if zlib.crc32(payload) != header["checksum"]:
            bad_crc += 1
        actual.append(record_from_header(header, payload))
    diff = compare_datasets(expected, actual)
    report = {"records": len(actual), "expected": len(expected),
              "missing": len(diff.missing), "unexpected": len(diff.unexpected),
              "corrupt": len(diff.corrupt), "bad_checksums": bad_crc,
              "per_hook": diff.per_hook_counts()}
    return diff.identical and not bad_crc, report


def run_synthetic(out_dir, *, spec: WorkloadSpec, model: ModelSpec, hooks, seed: int,
                  ring=None, drain=None, policy=None, hook_filter=None,
                  native_sink: bool = True, device: int | None = None) -> dict:
    """Drive the GPU path over the synthetic schedule into a dataset plus
    ``run_meta.json`` (SRC/cli.py:88-118 shape)."""
    from ._device import torch
    from .exporter import DrainConfig
    from .hookpoint import Observer
    from .rings import RingConfig
    from .sinks import FileSink, NativeFileSink
    from .workload import batch_payload
    t = torch()
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    registry = install_hooks(model, list(hooks))
    if hook_filter is not None:
        registry.set_hook_filter(list(hook_filter))
    registry.commit_filter()
    schedule = build_schedule(spec, build_requests(spec, seed))
    sink = NativeFileSink(out_dir) if native_sink else FileSink(out_dir)
    obs = Observer(registry, ring=ring or RingConfig(64 << 20, 1024),
                   drain=drain or DrainConfig(min_ready_entries=1), policy=policy,
                   sink=sink, device=device, max_batch=max(1, spec.batch))
    obs.start()
    keep_log = {}
    dev = f"cuda:{obs.device}"
    hidden = registry.hidden_extent
    for step in schedule:
        plan = obs.begin_step(step.batch, step.step_seq)
        keep_log[step.step_seq] = tuple(plan.kept_ids)
        for hid in registry.enabled_ids():
            hook = registry.hook(hid)
            data = batch_payload(seed, hook, step.batch, step.step_seq, step.tokens, hidden)
            x = t.frombuffer(bytearray(data), dtype=t.uint8).to(dev)
            obs.capture(hid, x.view(len(step.batch), -1))
        obs.end_step()
    obs.flush(300)
    obs.check_device()
    obs.close()
    n_records = sink.records_written
    sink.close()
    meta = {"seed": seed, "hook_filter": None if hook_filter is None else list(hook_filter),
            "keep_log": {str(s): list(ids) for s, ids in sorted(keep_log.items())},
            "record_count": n_records,
            "policy_mode": getattr(obs.policy, "mode", None),
            "workload": {"batch": spec.batch, "prefill_tokens": spec.prefill_tokens,
                         "decode_steps": spec.decode_steps,
                         "arrival": list(spec.arrival) if spec.arrival else None},
            "model": {"layers": model.layers, "hidden": model.hidden},
            "hooks": [hook_to_dict(h) for h in hooks]}
    (out_dir / META_NAME).write_text(json.dumps(meta, sort_keys=True, indent=2) + "\n",
                                     encoding="utf-8")
    return meta


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    if len(argv) != 1:
        print("usage: python -m paper_2605_11093_b200.verify DATASET", file=sys.stderr)
        return 2
    try:
        ok, rep = verify_dataset(argv[0])
    except ConfigError as exc:          # SRC/cli.py:293-298
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except TapflowError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    for hook, n in sorted(rep["per_hook"].items()):
        print(f"{hook}: {n} differing records")
    if rep["bad_checksums"]:
        print(f"stored checksums failing: {rep['bad_checksums']}")
    if ok:
        print(f"verified: {rep['records']} records match the reference exactly")
        return 0
    print(f"mismatch: {rep['missing']} missing, {rep['unexpected']} unexpected, "
          f"{rep['corrupt']} corrupt")
    return 1


if __name__ == "__main__":
    raise SystemExit(main())
