"""Build the sm_100a C-ABI library in-tree with nvcc.

Produces ``paper_2604_18348_b200/libadacluster_sm100.so`` (git-ignored, but
it travels to the GPU box with the gpurun snapshot).  The clustering and
selection translation units are compiled with ``--fmad=false`` because they
must reproduce the reference's unfused numpy arithmetic bit-for-bit; the
attention units allow contraction.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "csrc"
LIB = PKG / "libadacluster_sm100.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--extended-lambda",
    "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}", "-Xptxas", "-warn-spills",
] + os.environ.get("AC_NVCC_FLAGS", "").split()  # A/B experiments only (e.g. -DAC_ASG_X_GLOBAL=0)
# translation unit -> extra flags
UNITS = {
    "capi.cu": [],
    "cluster.cu": ["--fmad=false"],
    "select.cu": ["--fmad=false"],
    "tensorops.cu": ["--fmad=false"],
    "attn_simt.cu": [],
    "attn_fa4.cu": [],
    "attn_fa4_d128.cu": [],
    "assign_tc.cu": ["--fmad=false"],
}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _compile(unit: str, flags: list[str], verbose: bool) -> Path:
    src = CSRC / unit
    obj = BUILD / (unit + ".o")
    deps = [src] + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "adacluster_sm100.h"]
    if obj.exists() and obj.stat().st_mtime >= max(p.stat().st_mtime for p in deps):
        return obj
    cmd = [nvcc(), *ARCH, *COMMON, *flags, "-c", str(src), "-o", str(obj)]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {unit}:\n{res.stderr}\n{res.stdout}")
    if verbose and res.stderr:
        sys.stderr.write(res.stderr)
    return obj


def build(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    units = {u: f for u, f in UNITS.items() if (CSRC / u).exists()}
    if force:
        for u in units:
            (BUILD / (u + ".o")).unlink(missing_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(units)) as ex:
        objs = list(ex.map(lambda kv: _compile(kv[0], kv[1], verbose), units.items()))
    newest = max(o.stat().st_mtime for o in objs)
    if force or not LIB.exists() or LIB.stat().st_mtime < newest:
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
        tmp.replace(LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
