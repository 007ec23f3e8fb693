"""Build liblpb.so in-tree with nvcc for sm_100a (B200).

    python paper_1609_08114_b200/build.py [--verbose] [--force]
(run it by path: importing the package first would load a possibly stale liblpb.so)

Development build (never the product library):
    python paper_1609_08114_b200/build.py --dev
builds devbuild/paper_1609_08114_b200/ (a copy of the package whose liblpb.so is compiled
with -DLPB_DEV_HOOKS -- environment switches for A/B experiments and tests of alternative
paths, lpb_set_profile_buffer -- plus the diagnostic kernels of devsrc/, declared in
include/dev/lpb_selftest.h).  The product liblpb.so reads no environment variable and
exports only include/lpb.h.  Other variants:
    python paper_1609_08114_b200/build.py --variant ab/prof -DLPB_PROFILE
builds a copy of the package under ab/prof/paper_1609_08114_b200/ with extra defines
(scripts/phase_prof.py and scripts/ab_time.py import it from there).

Every .cu under csrc/ is compiled to an object with
    -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false
(-fmad=false: no implicit multiply-add contraction; the kernels write the FMAs the method
needs explicitly with __fma_rn, which keeps them bit-identical to the oracle), then linked
into paper_1609_08114_b200/liblpb.so with the CUDA runtime linked statically, so the library
loads on a machine without a GPU (the symbol-export tests run on CPU).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
DEVSRC = os.path.join(HERE, "devsrc")
OUT = os.path.join(HERE, "liblpb.so")
OBJ = os.path.join(HERE, "build_obj")
DEV_DIR = os.path.join(ROOT, "devbuild", os.path.basename(HERE))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC",
         "-I", os.path.join(ROOT, "include")]


def _stale(obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines: list[str] | None = None,
          out: str = OUT, obj: str = OBJ, dev: bool = False) -> str:
    OUT, OBJ = out, obj
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    if dev:
        srcs += sorted(glob.glob(os.path.join(DEVSRC, "*.cu")))
        defines = ["-DLPB_DEV_HOOKS", *(defines or [])]
    hdrs = (sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) +
            sorted(glob.glob(os.path.join(ROOT, "include", "**", "*.h"), recursive=True)))
    objs = []
    jobs = []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            cmd = [NVCC, *ARCH, *FLAGS, *(defines or []), "-c", s, "-o", o]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        for err in ex.map(run, jobs):
            if verbose and err:
                print(err, file=sys.stderr)
    if force or jobs or not os.path.exists(OUT) or _stale(OUT, objs):
        tmp = OUT + f".tmp{os.getpid()}"
        run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs])
        os.replace(tmp, OUT)
    return OUT


def build_dev(verbose: bool = False, force: bool = False) -> str:
    """The development build (see the module docstring) under devbuild/."""
    import shutil
    os.makedirs(DEV_DIR, exist_ok=True)
    for f in glob.glob(os.path.join(HERE, "*.py")):
        shutil.copy(f, DEV_DIR)
    return build(verbose=verbose, force=force, out=os.path.join(DEV_DIR, "liblpb.so"),
                 obj=os.path.join(DEV_DIR, "build_obj"), dev=True)


if __name__ == "__main__":
    # -D... defines and -X... / --extra nvcc flags (A/B variants); --variant/--verbose/--force
    # are this script's own
    defs = [a for a in sys.argv[1:] if a.startswith("-D") or a.startswith("-X")
            or (a.startswith("--") and a not in ("--variant", "--verbose", "--force", "--dev"))]
    if "--dev" in sys.argv:
        print(build_dev(verbose="--verbose" in sys.argv, force="--force" in sys.argv))
    elif "--variant" in sys.argv:
        import shutil
        vdir = os.path.join(os.path.abspath(sys.argv[sys.argv.index("--variant") + 1]),
                            os.path.basename(HERE))
        os.makedirs(vdir, exist_ok=True)
        for f in glob.glob(os.path.join(HERE, "*.py")):
            shutil.copy(f, vdir)
        print(build(verbose="--verbose" in sys.argv, force=True, defines=defs,
                    out=os.path.join(vdir, "liblpb.so"), obj=os.path.join(vdir, "build_obj"),
                    dev=True))
    else:
        print(build(verbose="--verbose" in sys.argv, force="--force" in sys.argv, defines=defs))
