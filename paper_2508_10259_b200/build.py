"""Build libams.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python paper_2508_10259_b200/build.py [--force]     (or __graft_entry__.build())

Every .cu under csrc/ is compiled with -gencode arch=compute_100a,code=sm_100a
-lineinfo -O3 (no fast-math: the fp32 path is bit-exact), then linked into
paper_2508_10259_b200/libams.so against the NCCL that torch loads (pip
nvidia-nccl-cu12), with an rpath to it.  ptxas register/spill reports go to
build/ptxas_<file>.log.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libams.so")
BUILD = os.path.join(ROOT, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    cands = []
    for base in {sysconfig.get_paths()["purelib"], sysconfig.get_paths()["platlib"]}:
        cands.append(os.path.join(base, "nvidia", "nccl"))
    try:
        import nvidia.nccl  # type: ignore
        cands.insert(0, os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0])
    except Exception:
        pass
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    raise RuntimeError("pip NCCL (nvidia/nccl/include/nccl.h) not found")


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build_id(srcs, hdrs, flags) -> str:
    """Identity of a build: sha256 over the sources, headers and compile flags (nvcc output
    itself is not byte-reproducible -- it embeds temporary file names -- so a hash of the
    .so cannot tie a profile to the code it measured; this can).  Compiled into the
    library (ams_build_id) and recorded next to every ncu capture."""
    import hashlib
    h = hashlib.sha256()
    for f in sorted(srcs + hdrs):
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    h.update(" ".join(flags).encode())
    return h.hexdigest()[:32]


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    inc, lib = nccl_dirs()
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "ams.h")]
    if not force and not _stale(OUT, [*srcs, *hdrs, os.path.abspath(__file__)]):
        return OUT
    common = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-I", os.path.join(ROOT, "include"), "-I", inc, "-Xptxas", "-v"]
    bid = build_id(srcs, hdrs, [*ARCH, "-O3", "-lineinfo", "-std=c++17"])
    common += [f"-DAMS_BUILD_ID=\"{bid}\""]

    def compile_one(src):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        # the object that embeds the build id (ams_capi.cu) is stale whenever the id changes,
        # not only when its own sources change
        stamp = obj + ".build_id"
        id_changed = "AMS_BUILD_ID" in open(src).read() and (
            not os.path.exists(stamp) or open(stamp).read().strip() != bid)
        if force or id_changed or _stale(obj, [src, *hdrs]):
            log = os.path.join(BUILD, "ptxas_" + os.path.basename(src) + ".log")
            cmd = [*common, "-c", src, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            with open(log, "w") as f:
                f.write(r.stdout + r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
            with open(stamp, "w") as f:
                f.write(bid)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(compile_one, srcs))
    if force or _stale(OUT, objs):
        tmp = OUT + f".tmp{os.getpid()}"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-L", lib, "-l:libnccl.so.2",
               "-Xlinker", f"-rpath={lib}"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
        os.replace(tmp, OUT)
    if verbose:
        print(OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
