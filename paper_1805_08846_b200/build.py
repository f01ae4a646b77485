"""Build the sm_100a sweep library in-tree: paper_1805_08846_b200/libclawb200.so.

nvcc flags are part of the parity contract: ``--fmad=false`` forbids FMA
contraction and the default ``-prec-div=true -prec-sqrt=true -ftz=false``
keep division/sqrt IEEE round-to-nearest; never
``--use_fast_math``.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libclawb200.so")
BUILD = os.path.join(HERE, "csrc", "build")

# (source, extra flags, object name): solver families compile once per dtype
SOURCES = [("clb_capi.cu", [], "clb_capi.o")] + [
    (f"clb_inst_{fam}.cu", [f"-DCLB_DTYPE={isz}"], f"clb_inst_{fam}_f{8 * isz}.o")
    for fam in ("acoustics", "shallow_water", "advection", "vc_acoustics")
    for isz in (4, 8)
]
HEADERS = ["clb_solvers.cuh", "clb_kernels.cuh", "clb_async.cuh", "clb_controller.cuh",
           "../../include/clawb200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
]


def _nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c
    return "nvcc"


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, variant: str | None = None,
          defines: tuple = ()) -> str:
    """Compile and link the library; `variant` + `defines` build a tuning
    variant libclawb200_<variant>.so from its own object directory."""
    if defines and not variant:
        # knobs (some timing-only and not bit-exact) never go into the default
        # library: its objects' staleness check looks at mtimes, not defines
        raise ValueError("build(defines=...) needs a variant name (libclawb200_<variant>.so)")
    out = OUT if not variant else os.path.join(HERE, f"libclawb200_{variant}.so")
    bdir = BUILD if not variant else os.path.join(CSRC, f"build_{variant}")
    extra_d = [f"-D{d}" for d in defines] if variant else ["-DCLB_DEFAULT_LIB=1"]
    if variant:
        # a variant's objects are rebuilt whenever its define set changes
        os.makedirs(bdir, exist_ok=True)
        stamp = os.path.join(bdir, "defines.txt")
        want = "\n".join(sorted(extra_d))
        old = open(stamp).read() if os.path.exists(stamp) else None
        if old != want:
            force = True
            with open(stamp, "w") as fh:
                fh.write(want)
    os.makedirs(bdir, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS]
    objs = []
    jobs = []
    for src, extra, obj in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(bdir, obj)
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            cmd = [_nvcc(), *NVCC_FLAGS, *extra, *extra_d, "-c", s, "-o", o]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            for cmd, r in ex.map(run, jobs):
                if verbose or r.returncode != 0:
                    sys.stderr.write(r.stdout + r.stderr)
                if r.returncode != 0:
                    raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")
    if force or _stale(out, objs):
        cmd = [_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out, *objs,
               "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {r.stdout}{r.stderr}")
    return out


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("-v", action="store_true")
    ap.add_argument("-f", action="store_true")
    ap.add_argument("--variant")
    ap.add_argument("-D", action="append", default=[])
    a = ap.parse_args()
    print(build(verbose=a.v, force=a.f, variant=a.variant, defines=tuple(a.D)))
