"""Build libbamg_b200.so in-tree with nvcc for sm_100a (no JIT cache, no torch ext).

The shared library carries every CUDA kernel of the path plus the extern "C"
boundary declared in include/bamg_b200.h. It links the CUDA runtime statically so
it only needs the driver on the GPU box.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "csrc", "_obj")
LIB = os.path.join(HERE, "libbamg_b200.so")
SOURCES = ["prims.cu", "problem.cu", "schur.cu", "blas.cu", "mg.cu", "driver.cu", "blockmat.cu", "scenegen.cu", "balio.cpp"]
HEADERS = ["common.cuh", "ctx.h", "vcycle.cuh", os.path.join("..", "..", "include", "bamg_b200.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "-diag-suppress", "550,177"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(verbose: bool = False, force: bool = False, defines: list[str] | None = None,
          out: str | None = None) -> str:
    """Compile + link. `defines` / `out`: an A/B variant (extra -D flags) built into
    its own object directory and library path (dev tool; the product is LIB)."""
    defines = list(defines or [])
    lib_path = out or LIB
    obj_dir = OBJ if not defines else os.path.join(CSRC, "_obj_" + "_".join(d.lstrip("-D") for d in defines))
    os.makedirs(obj_dir, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in HEADERS]
    objs, jobs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(obj_dir, os.path.splitext(src)[0] + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = [nvcc(), *ARCH, *FLAGS, *defines, "-c", s, "-o", o]
            jobs.append((src, cmd))

    def run(job):
        src, cmd = job
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{p.stderr}")
        return src, p.stderr

    if jobs:
        with cf.ThreadPoolExecutor(min(len(jobs), os.cpu_count() or 4)) as ex:
            for src, log in ex.map(run, jobs):
                if verbose:
                    print(f"[build] {src}\n{log}", file=sys.stderr)
    if force or jobs or _stale(lib_path, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", lib_path, *objs]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed:\n{p.stderr}")
    return lib_path


if __name__ == "__main__":
    defs = [a for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[len("--out="):] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, defines=defs, out=outs[0] if outs else None))
