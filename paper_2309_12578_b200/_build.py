"""Build libspion.so in-tree (nvcc, sm_100a).  Used by __graft_entry__.build()."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "lib")
SO = os.path.join(OUT_DIR, "libspion.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def _needs(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out_dir: str = OUT_DIR, defines=()) -> str:
    """Compile csrc/*.cu into out_dir/libspion.so; `defines` (e.g. ["-DSPION_PING=0"]) build a
    variant for A/B measurements (tools/build_variant.py)."""
    SO = os.path.join(out_dir, "libspion.so")
    os.makedirs(os.path.join(out_dir, "obj"), exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "spion.h")]
    objs = []
    jobs = []
    for s in srcs:
        o = os.path.join(out_dir, "obj", os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or _needs(o, [s] + hdrs):
            cmd = [NVCC, *ARCH, *FLAGS, *defines, "-Xptxas", "-v", "-c", s, "-o", o]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        return r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for log in ex.map(run, jobs):
            if verbose:
                sys.stderr.write(log)
    if force or jobs or _needs(SO, objs):
        # default visibility only for the extern "C" ABI (see -fvisibility=hidden + SPION_API)
        cmd = [NVCC, *ARCH, "-shared", "-o", SO, *objs, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
