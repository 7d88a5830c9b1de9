"""Builds libstg.so (the CUDA library behind include/stg.h) in-tree for sm_100a.

    python -m paper_2603_29235_b200.build          # libstg.so (+ the C++ shim)

Objects go to paper_2603_29235_b200/_build/, the library to
paper_2603_29235_b200/libstg.so (git-ignored, travels to the GPU box).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "_build"
LIB = PKG / "libstg.so"
BENCH_LIB = PKG / "libstg_bench.so"
SHIM_LIB = PKG / "libstg_strata.so"
REF_INC = Path("/root/reference/proj/core/include")
JSON_DIR = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_INC = "/usr/local/cuda/include"



def _nccl_dir():
    """The NCCL torch ships with (nvidia/nccl wheel), so libstg and torch.distributed
    share one libnccl.so.2 in a process whichever is loaded first; the system
    NCCL only when the wheel is absent."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        d = Path(list(spec.submodule_search_locations)[0])
        if (d / "lib" / "libnccl.so.2").exists() and (d / "include" / "nccl.h").exists():
            return d
    return None


NCCL_DIR = _nccl_dir()
NCCL_INC = [f"-I{NCCL_DIR / 'include'}"] if NCCL_DIR else []
NCCL_LINK = ([f"-L{NCCL_DIR / 'lib'}", "-l:libnccl.so.2", "-Xlinker", f"-rpath={NCCL_DIR / 'lib'}"]
             if NCCL_DIR else ["-lnccl"])

CU_SOURCES = ["stg_window.cu", "stg_render.cu", "stg_samples.cu", "symtab.cu", "stg_bundle.cu"]
CPP_SOURCES = ["stg_api.cpp", "stg_bundle_host.cpp", "stg_report.cpp"]
HEADERS = ["stg_internal.h", "kernels.cuh", "result.h", "stg_runner.inl", "stg_output.inl", "bundle.h"]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} ... {cmd[-1]}")
    return r


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build(verbose: bool = False) -> Path:
    OUT.mkdir(exist_ok=True)
    hdrs = [CSRC / h for h in HEADERS] + [ROOT / "include" / "stg.h"]
    objs = []
    for src in CU_SOURCES:
        obj = OUT / (Path(src).stem + ".o")
        if _stale(obj, [CSRC / src] + hdrs):
            _run([NVCC, "-std=c++17", "-O3", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC",
                  "-Xptxas", "-v" if verbose else "-O3", "-diag-suppress", "177",
                  *NCCL_INC, f"-I{ROOT / 'include'}", "-c", str(CSRC / src), "-o", str(obj)])
        objs.append(obj)
    for src in CPP_SOURCES:
        obj = OUT / (Path(src).stem + ".o")
        if _stale(obj, [CSRC / src] + hdrs):
            _run(["g++", "-std=c++17", "-O2", "-fPIC", *NCCL_INC, f"-I{ROOT / 'include'}", f"-I{JSON_DIR}", f"-I{CUDA_INC}",
                  "-c", str(CSRC / src), "-o", str(obj)])
        objs.append(obj)
    if _stale(LIB, objs):
        _run([NVCC, "-shared", *ARCH, "-o", str(LIB), *map(str, objs), "-lcudart", *NCCL_LINK])
    # bench-side generator (not part of the product library)
    if _stale(BENCH_LIB, [CSRC / "bench_gen.cu"]):
        _run([NVCC, "-std=c++17", "-O3", *ARCH, "-Xcompiler", "-fPIC", "-shared",
              str(CSRC / "bench_gen.cu"), "-o", str(BENCH_LIB)])
    # C++ drop-in shim over the C-ABI: needs the reference's headers (this
    # container only; the built .so travels to the GPU box)
    if REF_INC.exists() and _stale(SHIM_LIB, [CSRC / "shim" / "strata_stg.cpp", ROOT / "include" / "stg.h", LIB]):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", f"-I{ROOT / 'include'}", f"-I{REF_INC}",
              f"-I{JSON_DIR}", str(CSRC / "shim" / "strata_stg.cpp"), "-o", str(SHIM_LIB),
              f"-L{PKG}", "-lstg", "-Wl,-rpath,$ORIGIN"])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
