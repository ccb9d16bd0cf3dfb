"""Sink throughput: records.ndjson + records.bin written
from capture-sized payloads held in memory (as the exporter hands staging
batches to the sink), per writer: Python FileSink, NativeFileSink buffered
and O_DIRECT, at several thread counts. One JSON line per configuration.

usage: python scripts/exp_sink.py [--dir D] [--gib 4] [--capture-mib 32]
"""
import argparse
import json
import os
import shutil
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11093_b200 import DType, TensorMeta  # noqa: E402
from paper_2605_11093_b200.sinks import FileSink, NativeFileSink  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dir", default="gpurun_out/sink_tmp")
ap.add_argument("--gib", type=float, default=4.0)
ap.add_argument("--capture-mib", type=int, default=32)
ap.add_argument("--batch", type=int, default=8, help="requests per capture")
ap.add_argument("--threads", default="1,4,8,16")
ap.add_argument("--python", action="store_true", help="also time the Python FileSink")
args = ap.parse_args()

cap = args.capture_mib << 20
payload = bytearray(os.urandom(1 << 20)) * args.capture_mib
B = args.batch
row = cap // B
bf16 = DType.of("bf16")
n_caps = int(args.gib * (1 << 30) // cap)
metas = [TensorMeta(f"resid_post[{i % 32}]", i % 32, i // 32, tuple(range(B)),
                    tuple((0, 1) for _ in range(B)), (1, row // 2), bf16)
         for i in range(n_caps)]
import ctypes as C  # noqa: E402
buf = (C.c_char * len(payload)).from_buffer(payload)
addr = C.addressof(buf)


def run(make, label, threads):
    d = os.path.join(args.dir, label)
    shutil.rmtree(d, ignore_errors=True)
    sink = make(d)
    t0 = time.perf_counter()
    for k in range(0, n_caps, 4):  # 4 captures per staging batch
        sink.write_captures([(m, payload, addr) for m in metas[k:k + 4]])
    close_t = time.perf_counter()
    sink.close()
    t1 = time.perf_counter()
    size = os.path.getsize(os.path.join(d, "records.bin"))
    shutil.rmtree(d, ignore_errors=True)
    print(json.dumps({"sink": label, "threads": threads, "bytes": size,
                      "seconds": t1 - t0, "close_s": t1 - close_t,
                      "gbs": size / (t1 - t0) / 1e9,
                      "direct": getattr(sink, "direct", None)}), flush=True)


os.makedirs(args.dir, exist_ok=True)
for th in [int(x) for x in args.threads.split(",")]:
    run(lambda d: NativeFileSink(d, threads=th), f"native_buffered_t{th}", th)
    run(lambda d: NativeFileSink(d, threads=th, direct=True), f"native_direct_t{th}", th)
if args.python:
    class Py(FileSink):
        def write_captures(self, caps):
            from paper_2605_11093_b200.exporter import split_payload
            for m, p, _ in caps:
                self.write(split_payload(m, p))
    run(lambda d: Py(d), "python_filesink", 1)
