"""In-tree build of libep_b200.so (nvcc, sm_100a only).

    python -m paper_2504_11729_b200.build [--force] [--ptxas-v]

Objects go to paper_2504_11729_b200/_build/, the library to
paper_2504_11729_b200/_lib/libep_b200.so (git-ignored, travels to the GPU box
with gpurun). There is no JIT and no fallback: the package refuses to load
without this library.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIB_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIB_DIR, "libep_b200.so")
CHECKED_LIB = os.path.join(LIB_DIR, "libep_b200_checked.so")
INCLUDE = os.path.join(ROOT, "include")

NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2", f"-I{INCLUDE}", f"-I{CSRC}"]
CU_FLAGS = ARCH + COMMON + ["--expt-relaxed-constexpr", "-Xptxas", "-O3"]

SOURCES = ["kern_reference.cu", "kern_decode.cu", "kern_verify.cu", "kern_score.cu", "kern_peer.cu",
           "kern_ingest.cu", "kern_model.cu", "kern_model_persist.cu", "capi.cpp", "plan.cpp", "model.cpp",
           "cache.cpp"]
HEADERS = ["ep_common.cuh", "ep_internal.h", "umma.cuh", "merge.cuh", "model_internal.h"]
PUBLIC_HEADERS = ["ep_attn.h", "ep_model.h"]


def _deps(src: str) -> list[str]:
    hdrs = [os.path.join(CSRC, h) for h in HEADERS if os.path.exists(os.path.join(CSRC, h))]
    return [os.path.join(CSRC, src)] + [os.path.join(INCLUDE, "ep", h) for h in PUBLIC_HEADERS] + hdrs


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(src: str, force: bool, ptxas_v: bool, obj_dir: str = OBJ, checked: bool = False) -> str:
    obj = os.path.join(obj_dir, os.path.splitext(src)[0] + ".o")
    if force or _stale(obj, _deps(src)):
        flags = CU_FLAGS + (["-Xptxas", "-v"] if ptxas_v and src.endswith(".cu") else [])
        if checked:
            flags = flags + ["-DEP_CHECKED"]
        cmd = [NVCC] + flags + ["-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if ptxas_v:
            sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, ptxas_v: bool = False, checked: bool = False) -> str:
    """checked: the -DEP_CHECKED variant (device bounds checks, bounded spins)
    into _build/checked/ and _lib/libep_b200_checked.so."""
    obj_dir = os.path.join(OBJ, "checked") if checked else OBJ
    lib = CHECKED_LIB if checked else LIB
    os.makedirs(obj_dir, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, ptxas_v, obj_dir, checked), srcs))
    if force or _stale(lib, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", lib] + objs + ["-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--ptxas-v", action="store_true")
    ap.add_argument("--checked", action="store_true", help="the -DEP_CHECKED variant (bounds checks)")
    args = ap.parse_args()
    print(build(force=args.force, ptxas_v=args.ptxas_v, checked=args.checked))
