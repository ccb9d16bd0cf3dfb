"""The C-ABI boundary on CPU: the library loads, exports every entry point
include/ring2.h declares, the ctypes structs match the C layout, and the
allocator the device runs (ring2_core.h) makes the reference's decisions.
No CUDA calls are made (there is no GPU here)."""

import ctypes as C
import random
import re
import subprocess
import textwrap
from pathlib import Path

import pytest

import oracle
from paper_2605_11093_b200 import _native as N

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "ring2.h"


def header_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(
        r"^\s*(?:int|void|double|uint32_t|const char\*)\s+(tf_\w+)\s*\(", text, re.M)))


def test_library_loads_and_exports_every_symbol():
    lib = N.lib()
    assert lib.tf_abi_version() == 1
    declared = header_functions()
    assert len(declared) >= 40
    missing = [f for f in declared if not hasattr(lib, f)]
    assert missing == []
    assert sorted(set(N.EXPORTED)) == declared


def test_status_names_cover_error_taxonomy():
    lib = N.lib()
    names = [lib.tf_status_name(i).decode() for i in range(15)]
    assert names[:11] == ["ok", "ConfigError", "AllocationError",
                          "PayloadRingFull", "MetaRingFull",
                          "OutOfOrderRelease", "ProtocolError", "MetaMismatch",
                          "PolicyUnderestimate", "StagingExhausted",
                          "HookDisabled"]
    from paper_2605_11093_b200 import errors
    assert isinstance(N.exception_for(N.TF_ERR_PAYLOAD_RING_FULL), errors.RingFull)
    assert isinstance(N.exception_for(N.TF_ERR_META_RING_FULL), errors.MetaRingFull)
    assert isinstance(N.exception_for(N.TF_ERR_VALUE), ValueError)


def test_struct_layouts_match_header(tmp_path):
    """sizeof/offsetof from a C compile of ring2.h == the ctypes mirror."""
    fields = {
        "tf_descriptor": ("CDescriptor", ["payload_offset", "payload_len", "hook_id",
                                          "step_seq", "ready_seq", "skip_before",
                                          "flags", "n_rows", "capture_seq", "checksum"]),
        "tf_capture_args": ("CCaptureArgs", ["src", "keep", "step_seq_ptr", "flags",
                                             "max_ctas"]),
        "tf_ring_state": ("CRingState", ["occupancy", "high_watermark", "kernel_ns"]),
        "tf_drain_config": ("CDrainConfig", ["max_wait", "mode", "page_out", "split_oversize"]),
        "tf_stager_stats": ("CStagerStats", ["transfer_seconds", "pool_free"]),
        "tf_paged_batch": ("CPagedBatch", ["payload", "starts", "pinned_buffer", "oversize"]),
        "tf_capture_result": ("CCaptureResult", ["status", "desc"]),
        "tf_ring_config": ("CRingConfig", ["high_watermark", "wait_timeout_ns"]),
        "tf_batch_info": ("CBatchInfo", ["bytes_total", "reason"]),
    }
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"',
             "int main(void){"]
    for cname, (_, fl) in fields.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f in fl:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", str(src), "-o", str(exe)], check=True)
    out = dict(l.rsplit(" ", 1) for l in
               subprocess.run([str(exe)], capture_output=True, text=True,
                              check=True).stdout.split("\n") if l)
    for cname, (pyname, fl) in fields.items():
        cls = getattr(N, pyname)
        assert int(out[cname]) == C.sizeof(cls), cname
        for f in fl:
            assert int(out[f"{cname}.{f}"]) == getattr(cls, f).offset, (cname, f)


def test_plan_reservation_matches_oracle():
    lib = N.lib()
    rng = random.Random(99)
    o, d = C.c_uint64(), C.c_uint64()
    for _ in range(20000):
        cap = 16 * rng.randint(1, 64)
        used = 16 * rng.randint(0, cap // 16)
        head = 16 * rng.randint(0, cap // 16 - 1)
        tail = 16 * rng.randint(0, cap // 16 - 1)
        length = 16 * rng.randint(1, cap // 16)
        ok = lib.tf_plan_reservation(head, tail, used, cap, length,
                                     C.byref(o), C.byref(d))
        want = oracle.plan(head, tail, used, cap, length)
        assert (want is not None) == bool(ok)
        if ok:
            assert (o.value, d.value) == want


@pytest.fixture(scope="module")
def core(tmp_path_factory):
    out = tmp_path_factory.mktemp("core") / "libcore.so"
    subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-std=c11",
                    str(ROOT / "tests" / "native" / "core_harness.c"),
                    "-o", str(out)], check=True)
    lib = C.CDLL(str(out))
    u64 = C.c_uint64
    lib.core_reserve.argtypes = [C.c_void_p, u64, u64, u64, C.POINTER(u64),
                                 C.POINTER(u64), C.POINTER(C.c_uint32)]
    for n in ("core_used", "core_tail"):
        getattr(lib, n).restype = u64
    lib.core_used.argtypes = [C.c_void_p, u64]
    lib.core_tail.argtypes = [C.c_void_p, u64, u64]
    lib.core_head.restype = u64
    lib.core_head.argtypes = [C.c_void_p, u64]
    return lib


class PState(C.Structure):
    _fields_ = [("V", C.c_uint64), ("reset_mark", C.c_uint64),
                ("reset_credit", C.c_uint64)]


def test_split_ownership_allocator_equals_reference(core):
    """The device allocator's state machine (producer V/mark/credit, host
    release cursor L) reproduces the reference RingPair on random
    reserve/release scripts: same offsets, head, tail and occupancy."""
    rng = random.Random(2026)
    for trial in range(300):
        cap = 16 * rng.randint(2, 40)
        ref = oracle.OracleRing(cap, 1 << 20)
        p = PState(0, (1 << 64) - 1, 0)
        L = 0
        fifo = []  # (off, len, skip)
        for _ in range(rng.randint(1, 80)):
            if rng.random() < 0.55:
                length = 16 * rng.randint(1, max(1, cap // 16))
                rc, roff, _ = ref.reserve(length)
                off, skip, kind = C.c_uint64(), C.c_uint64(), C.c_uint32()
                ok = core.core_reserve(C.byref(p), L, cap, length, C.byref(off),
                                       C.byref(skip), C.byref(kind))
                assert bool(ok) == (rc == 0), (trial, length)
                if ok:
                    assert off.value == roff
                    fifo.append((off.value, length, skip.value))
            elif fifo:
                off, length, skip = fifo.pop(0)
                assert ref.release(off, length) == 0
                L += skip + length
            s = ref.state()
            assert core.core_used(C.byref(p), L) == s["used"]
            assert core.core_head(C.byref(p), cap) == s["head"]
            if s["used"]:
                assert core.core_tail(C.byref(p), L, cap) == s["tail"]
