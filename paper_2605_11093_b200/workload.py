"""Synthetic workload source: requests, schedule and content bytes.

The reference drives its capture path with a deterministic synthetic
workload (SRC/workload.py:79-143, 193-236): seeded requests with prompt-group
labels, a uniform prefill/decode schedule, and per (hook, request, step)
content bytes from Philox keyed by (seed, crc32(hook name) << 32 | layer+1,
request, step). Runs feed these bytes through the GPU path and
``verify.py`` regenerates them to check a stored dataset after the fact
(SRC/cli.py:153-189), so the keying here must be the reference's exactly;
``tests/test_workload_verify.py`` pins it against the independent oracle
restatement and the reference's golden hashes.
"""

from __future__ import annotations

import math
import zlib
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError
from .policy import StepRequest

PREFILL, DECODE = "prefill", "decode"
PROMPT_GROUPS = ("alpha", "beta")          # SRC/workload.py:20


@dataclass(frozen=True)
class WorkloadSpec:
    """SRC/workload.py:30-76 (the fields the capture path needs)."""

    batch: int
    prefill_tokens: int
    decode_steps: int
    arrival: tuple | None = None          # admissions per step; None = all at once

    def __post_init__(self) -> None:
        if self.batch <= 0 or self.prefill_tokens <= 0 or self.decode_steps < 0:
            raise ConfigError("batch, prefill_tokens must be positive")
        if self.arrival is not None and sum(self.arrival) != self.batch:
            raise ConfigError("arrival cohorts must sum to the batch")

    @property
    def cohorts(self) -> tuple:
        return tuple(self.arrival) if self.arrival is not None else (self.batch,)


@dataclass(frozen=True)
class ScheduledStep:
    step_seq: int
    kind: str
    batch: tuple

    @property
    def tokens(self) -> int:
        return self.batch[0].tokens


def build_requests(spec: WorkloadSpec, seed: int) -> tuple:
    """SRC/workload.py:79-88: prompt groups from Philox([seed, 'prom'])."""
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence([seed, 0x70726F6D])))
    out = []
    for i in range(spec.batch):
        group = PROMPT_GROUPS[int(rng.integers(len(PROMPT_GROUPS)))]
        out.append(StepRequest(i, i, f"{group} prompt {i}", 0, 0))
    return tuple(out)


def build_schedule(spec: WorkloadSpec, requests) -> tuple:
    """SRC/workload.py:103-143: admission k > 0 is a prefill step for that
    cohort; otherwise every active request decodes one token; requests
    retire after ``decode_steps`` decodes."""
    admissions = list(spec.cohorts)
    waiting = list(requests)
    active = []
    steps = []
    seq = 0
    while waiting or active or admissions:
        admit = admissions.pop(0) if admissions else 0
        if admit > 0:
            cohort, waiting = waiting[:admit], waiting[admit:]
            steps.append(ScheduledStep(seq, PREFILL, tuple(
                StepRequest(r.request_id, r.arrival_index, r.prompt, spec.prefill_tokens, 0)
                for r in cohort)))
            active.extend((r, 0) for r in cohort)
        elif active:
            steps.append(ScheduledStep(seq, DECODE, tuple(
                StepRequest(r.request_id, r.arrival_index, r.prompt, 1,
                            spec.prefill_tokens + done) for r, done in active)))
            active = [(r, d + 1) for r, d in active if d + 1 < spec.decode_steps]
        else:
            continue
        seq += 1
    return tuple(steps)


def content_key(seed: int, hook_name: str, layer_index, request_id: int,
                step_seq: int) -> list:
    """SRC/workload.py:193-197."""
    layer = 0 if layer_index is None else layer_index + 1
    return [seed, (zlib.crc32(hook_name.encode()) << 32) | layer, request_id, step_seq]


def request_payload(seed: int, hook, request_id: int, step_seq: int, tokens: int,
                    hidden: int) -> bytes:
    """One request's bytes for one hook firing (SRC/workload.py:200-233,
    unsharded)."""
    shape = hook.resolve_shape(tokens, hidden)
    nbytes = math.prod(shape) * hook.dtype.width
    gen = np.random.Generator(np.random.Philox(np.random.SeedSequence(
        content_key(seed, hook.name, hook.layer_index, request_id, step_seq))))
    return gen.bytes(nbytes)


def batch_payload(seed: int, hook, batch, step_seq: int, tokens: int, hidden: int) -> bytes:
    """The batch-major source buffer of one firing (SRC/workload.py:236-245)."""
    return b"".join(request_payload(seed, hook, r.request_id, step_seq, tokens, hidden)
                    for r in batch)


__all__ = ["WorkloadSpec", "ScheduledStep", "build_requests", "build_schedule",
           "content_key", "request_payload", "batch_payload", "PREFILL", "DECODE"]
