"""Build libmhlmoe.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2602_04870_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build_obj")
LIB = os.path.join(HERE, "libmhlmoe.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["router.cu", "router_sm100.cu", "tma_host.cu", "cluster.cu", "simt.cu", "combine.cu",
              "expert_sm100.cu", "expert_bwd_dx_sm100.cu", "expert_bwd_fused_sm100.cu", "expert_dw_sm100.cu",
              "router_bwd_sm100.cu", "expert_fwd_pair_sm100.cu",
              "router_blk_sm100.cu"]
CXX_SOURCES = ["capi.cpp"]


def _nccl_include() -> str:
    try:
        import nvidia.nccl  # noqa: WPS433 (build-time header location only)
        for p in nvidia.nccl.__path__:
            inc = os.path.join(p, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return inc
    except Exception:
        pass
    return "/usr/include"


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hs.append(os.path.join(ROOT, "include", "mhlmoe.h"))
    return hs


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in [src, *_headers()])


def _compile(src: str, force: bool) -> str:
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src + ".o")
    if not force and not _stale(obj, path):
        return obj
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-I", CSRC, "-I", os.path.join(ROOT, "include"),
              "-I", _nccl_include()]
    if src.endswith(".cu"):
        # MHL_NVCC_DEFS: extra -D flags for A/B builds of kernel variants (rebuild with --force)
        defs = os.environ.get("MHL_NVCC_DEFS", "").split()
        cmd = [NVCC, *ARCH, "-lineinfo", "-Xptxas", "-v", *common, *defs, "-c", path, "-o", obj]
    else:
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-fvisibility=hidden", "-I", CSRC, "-I", os.path.join(ROOT, "include"),
               "-I", _nccl_include(), "-I", os.path.join(CUDA, "include"), "-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    with open(obj + ".ptxas.txt", "w") as f:
        f.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = True) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=max(1, min(8, os.cpu_count() or 1))) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), CU_SOURCES + CXX_SOURCES))
    if force or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcublasLt", "-ldl",
               "-Xlinker", f"-rpath={os.path.join(CUDA, 'lib64')}", "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"[build] {LIB}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
