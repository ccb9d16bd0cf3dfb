"""Synthetic workload content + synchronous reference records — TEST
INFRASTRUCTURE (oracle).

Restates the reference's deterministic content keying so the GPU path can
be driven with the reference's own bytes on a box where the reference is
absent:

  * ``request_payload``   workload.py:193-233 — Philox(SeedSequence([seed,
    crc32(hook name) << 32 | layer+1, request, step])).bytes(n)
  * ``build_requests``    workload.py:79-88
  * ``build_schedule``    workload.py:103-143 (uniform prefill/decode steps)
  * ``reference_records`` oracle.py:22-71 (+ keep_log narrowing)
  * ``compare``           oracle.py:103-115 multiset diff

Pinned by tests/golden/workload.json (hashes produced by the reference).
"""

from __future__ import annotations

import math
import zlib
from collections import Counter
from dataclasses import dataclass

import numpy as np

PREFILL, DECODE = "prefill", "decode"
PROMPT_GROUPS = ("alpha", "beta")


def content_key(seed: int, hook_name: str, layer_index, request_id: int,
                step_seq: int) -> list[int]:
    layer = 0 if layer_index is None else layer_index + 1
    return [seed, (zlib.crc32(hook_name.encode()) << 32) | layer, request_id,
            step_seq]


def request_payload(seed, hook_name, layer_index, request_id, step_seq,
                    nbytes) -> bytes:
    gen = np.random.Generator(np.random.Philox(np.random.SeedSequence(
        content_key(seed, hook_name, layer_index, request_id, step_seq))))
    return gen.bytes(nbytes)


@dataclass(frozen=True)
class Req:
    request_id: int
    arrival_index: int
    prompt: str
    tokens: int = 0
    token_start: int = 0


def build_requests(batch: int, seed: int) -> list[Req]:
    rng = np.random.Generator(np.random.Philox(
        np.random.SeedSequence([seed, 0x70726F6D])))
    out = []
    for i in range(batch):
        group = PROMPT_GROUPS[int(rng.integers(len(PROMPT_GROUPS)))]
        out.append(Req(i, i, f"{group} prompt {i}"))
    return out


def build_schedule(batch: int, prefill_tokens: int, decode_steps: int,
                   seed: int, arrival=None):
    """[(step_seq, kind, [Req with tokens/token_start])]."""
    requests = build_requests(batch, seed)
    admissions = list(arrival) if arrival is not None else [batch]
    waiting = list(requests)
    active: list[tuple[Req, int]] = []
    steps = []
    seq = 0
    while waiting or active or admissions:
        admit = admissions.pop(0) if admissions else 0
        if admit > 0:
            cohort, waiting = waiting[:admit], waiting[admit:]
            steps.append((seq, PREFILL, [
                Req(r.request_id, r.arrival_index, r.prompt, prefill_tokens, 0)
                for r in cohort]))
            active.extend((r, 0) for r in cohort)
        elif active:
            steps.append((seq, DECODE, [
                Req(r.request_id, r.arrival_index, r.prompt, 1,
                    prefill_tokens + done) for r, done in active]))
            active = [(r, d + 1) for r, d in active if d + 1 < decode_steps]
        else:
            continue
        seq += 1
    return steps


def record_key(rec) -> tuple:
    return (rec.request_id, rec.hook_name, rec.layer_index, rec.step_seq,
            tuple(rec.rank_coords))


def compare(expected, actual) -> dict:
    """Multiset comparison of records by (key, payload)."""
    def sig(r):
        return (record_key(r), tuple(r.token_range), tuple(r.shape),
                r.dtype.name, bytes(r.payload))
    e, a = Counter(map(sig, expected)), Counter(map(sig, actual))
    missing = e - a
    unexpected = a - e
    return {"identical": not missing and not unexpected,
            "missing": sum(missing.values()),
            "unexpected": sum(unexpected.values())}


def slice_nbytes(shape, width) -> int:
    return math.prod(shape) * width
