"""Native build of the package: the CUDA library (sm_100a) and the host-side
input generators. Outputs are written in-tree next to this file so they travel
with the repository snapshot to the GPU box:

  librl_cddt.so      csrc/*.cu   nvcc -gencode arch=compute_100a,code=sm_100a
  libcddt_synth.so   csrc/synth.c (seeded workload generators, harness side)

All CUDA translation units are compiled with -fmad=false: the CDDT query is an
FP64 restatement of the reference and must not contract multiply-adds
(SURVEY.md §0.5, §8 N2).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import re
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB = PKG / "librl_cddt.so"
SYNTH = PKG / "libcddt_synth.so"
SYNTH_GPU = PKG / "libcddt_synth_gpu.so"
OBJ = PKG / "build"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo", "-fmad=false", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "-Xptxas", "-v",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build librl_cddt.so")


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str], log: Path | None = None) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.write_text(r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ... (exit {r.returncode})")


def build_cuda(force: bool = False, defines: tuple[str, ...] = (), out: Path | None = None) -> Path:
    """Build librl_cddt.so (or, with `defines`, a variant library at `out`)."""
    lib = out or LIB
    cu = sorted(p for p in CSRC.glob("*.cu") if p.name != "synth_gpu.cu")
    hdrs = sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))
    if not force and not _stale(lib, cu + hdrs + [Path(__file__)]):
        return lib
    nvcc = _nvcc()
    if not defines and out is None:
        objdir = OBJ
    else:  # variant libraries keep their own objects
        tag = "_".join(re.sub(r"[^A-Za-z0-9_]", "", d) for d in defines) or Path(out).stem
        objdir = OBJ / ("v_" + tag)
    objdir.mkdir(parents=True, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]

    def one(src: Path) -> Path:
        obj = objdir / (src.stem + ".o")
        if force or _stale(obj, [src] + hdrs + [Path(__file__)]):
            _run([nvcc, *ARCH, *NVCC_FLAGS, *dflags, "-I", str(INCLUDE), "-c", str(src), "-o",
                  str(obj)], objdir / (src.stem + ".ptxas.log"))
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, len(cu))) as ex:
        objs = list(ex.map(one, cu))
    tmp = lib.with_suffix(".so.tmp")
    _run([nvcc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart_static", "-lrt",
          "-ldl", "-lpthread"])
    os.replace(tmp, lib)
    return lib


def build_synth(force: bool = False) -> Path:
    src = CSRC / "synth.c"
    if not force and not _stale(SYNTH, [src]):
        return SYNTH
    tmp = SYNTH.with_suffix(".so.tmp")
    _run(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
          "-o", str(tmp), str(src), "-lm"])
    os.replace(tmp, SYNTH)
    return SYNTH


def build_synth_gpu(force: bool = False) -> Path:
    """Device twin of the query generator (harness side, not the C ABI)."""
    src = CSRC / "synth_gpu.cu"
    if not force and not _stale(SYNTH_GPU, [src]):
        return SYNTH_GPU
    tmp = SYNTH_GPU.with_suffix(".so.tmp")
    _run([_nvcc(), *ARCH, "-std=c++17", "-O3", "-Xcompiler", "-fPIC,-ffp-contract=off",
          "-fmad=false", "-shared", "-o", str(tmp), str(src), "-lcudart_static", "-lrt", "-ldl",
          "-lpthread"])
    os.replace(tmp, SYNTH_GPU)
    return SYNTH_GPU


def build_all(force: bool = False) -> None:
    build_synth(force)
    build_synth_gpu(force)
    build_cuda(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print(LIB, SYNTH)
