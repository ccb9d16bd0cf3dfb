"""Build the in-tree C-ABI library ``_lib/libring2.so`` for sm_100a.

Plain nvcc, no torch extension machinery: the library exports only the
``extern "C"`` entry points declared in ``include/ring2.h`` and is loaded
with ctypes. The output lives in-tree so it travels to the GPU box.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB = LIB_DIR / "libring2.so"
SOURCES = ["ring2.cu", "stager.cu", "sink.cpp"]
HEADERS = ["ring2_core.h", "ring2_internal.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3,-pthread",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _stale() -> bool:
    if not LIB.exists():
        return True
    built = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + [CSRC / h for h in HEADERS]
    deps.append(ROOT / "include" / "ring2.h")
    return any(p.stat().st_mtime > built for p in deps)


def build(force: bool = False, verbose: bool = False,
          variant: str | None = None) -> Path:
    """Compile the sources to objects and link the shared library.

    ``variant="trace"`` builds ``libring2_trace.so`` with -DTF_TRACE (phase
    timers in the capture kernel) and ``variant="variants"`` builds
    ``libring2_variants.so`` with the rejected TMA / cp.async copy paths, for
    experiments; the product library is always the plain ``libring2.so``
    (hot path only)."""
    lib = LIB if not variant else LIB_DIR / f"libring2_{variant}.so"
    if not force and not variant and not _stale():
        return LIB
    LIB_DIR.mkdir(exist_ok=True)
    nvcc = _nvcc()
    objs = []
    defines = []
    if variant == "variants":  # rejected copy paths (TF_COPY_PATH=tma|stage)
        defines.append("-DTF_COPY_VARIANTS")
    if variant and variant != "variants":
        # e.g. trace_ablN_cM (phase stamps, ablation N, M CTAs/SM) or smem0
        # (no shared-memory speculation) without stamps
        for part in variant.split("_"):
            if part == "trace":
                defines.append("-DTF_TRACE")
            elif part.startswith("abl"):
                defines.append(f"-DTF_ABL={int(part[3:])}")
            elif part == "noctl":  # last-reader commit, no controller CTA (A/B)
                defines.append("-DTF_CONTROLLER_CTA=0")
            elif part.startswith("c"):
                defines.append(f"-DTF_CTAS_PER_SM={int(part[1:])}")
            elif part.startswith("u"):
                defines.append(f"-DTF_UNROLL={int(part[1:])}")
            elif part == "nopreload":  # lazy kernel loading (repro of the hang)
                defines.append("-DTF_NO_PRELOAD")
            elif part == "nostcs":  # plain (evict-normal) ring stores (A/B)
                defines.append("-DTF_ST_CS=0")
            elif part == "nospec0":
                defines.append("-DTF_SPEC_WARP0=0")
            elif part.startswith("smem"):  # trace_smemN: N shared-memory spec segments
                defines.append(f"-DTF_SMEM_SPEC={int(part[4:])}")
    for src in SOURCES:
        obj = LIB_DIR / (Path(src).stem + (f"_{variant}" if variant else "") + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *defines, "-I", str(ROOT / "include"), "-c",
               str(CSRC / src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(res.stderr)
        if not variant:
            (LIB_DIR / (Path(src).stem + ".ptxas.txt")).write_text(res.stderr)
        objs.append(str(obj))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
           *objs, "-o", str(tmp), "-Xcompiler", "-pthread", "-lpthread", "-lz"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), None)
    print(build(force="--force" in sys.argv, verbose=True, variant=var))
