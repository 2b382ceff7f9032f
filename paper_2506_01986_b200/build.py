"""Build libspecmemo.so in-tree with nvcc for sm_100a (no GPU needed).

    python -m paper_2506_01986_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libspecmemo.so")
LIB_TRACE = os.path.join(HERE, "libspecmemo_trace.so")
SOURCES = ["gemm.cu", "attention.cu", "attention_tc.cu", "attention_f32.cu", "epilogue.cu", "decode.cu", "tp.cu", "runtime.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]


def _compile(src: str, verbose: bool, trace: bool = False) -> str:
    obj = os.path.join(CSRC, "build" + ("_trace" if trace else ""), src.replace(".cu", ".o"))
    cmd = [NVCC, *ARCH, *FLAGS, *(["-DSM_TRACE"] if trace else []), "-c", os.path.join(CSRC, src), "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".h"))]
    deps.append(os.path.join(ROOT, "include", "specmemo.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    """trace=True: diagnostic variant libspecmemo_trace.so (-DSM_TRACE: in-kernel clock stamps,
    sm_trace_read); selected at import with SPECMEMO_LIB=<path>."""
    out = LIB_TRACE if trace else LIB
    if not force and not trace and not _stale():
        return LIB
    os.makedirs(os.path.join(CSRC, "build" + ("_trace" if trace else "")), exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, trace), SOURCES))
    tmp = out + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-ldl", "-lpthread", "-lrt"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv))
