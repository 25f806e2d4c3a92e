"""Build libpu_unwrap.so in-tree with nvcc for sm_100a.

    python -m paper_2401_09961_b200.build_ext [--force] [-v]

Objects: pu_api.cu (host runtime, element-wise kernels, C ABI) plus one
object per (dtype, internal FFT length) instantiation of the transform
kernels (pu_dct_inst.cu), compiled in parallel and linked into
`_lib/libpu_unwrap.so`.  The library travels with the repository snapshot to
the GPU box (it is git-ignored).
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
# PU_BUILD_LIBDIR / PU_BUILD_DEFS: an alternative build (A/B variants, loaded
# with PU_LIB_PATH=<libdir>/libpu_unwrap.so)
LIBDIR = os.environ.get("PU_BUILD_LIBDIR") or os.path.join(PKG, "_lib")
OBJDIR = os.path.join(LIBDIR, "obj")
LIB = os.path.join(LIBDIR, "libpu_unwrap.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-O2",
          "-Xptxas", "-v"] + os.environ.get("PU_BUILD_DEFS", "").split()

# (dtype, internal FFT length); 0 = runtime plan.  Keep in sync with
# PU_STATIC_LS_F32 / PU_STATIC_LS_F64 in csrc/pu_dct_launch.cuh.
INSTANCES = ([("float", ls) for ls in (0, 512, 1024, 2048, 4096, 8192, 16384)]
             + [("double", ls) for ls in (0, 512, 1024, 2048, 4096, 8192)])
# (dtype, half length) of the 2-CTA cluster transforms (csrc/pu_split.cuh)
SPLIT_INSTANCES = [("double", 8192), ("float", 16384)]


def nvcc():
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libpu_unwrap.so")
    return path


def deps():
    return (sorted(glob.glob(os.path.join(CSRC, "*.cu"))) + sorted(glob.glob(os.path.join(CSRC, "*.cuh")))
            + [os.path.join(INCLUDE, "pu_unwrap.h"), os.path.abspath(__file__)])


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in deps())


def _includes(path, seen=None):
    """Transitive closure of the quoted #includes of `path` (csrc/ and include/)."""
    import re
    seen = set() if seen is None else seen
    if path in seen or not os.path.exists(path):
        return seen
    seen.add(path)
    for name in re.findall(r'^\s*#include\s+"([^"]+)"', open(path).read(), re.M):
        for d in (os.path.dirname(path), CSRC, INCLUDE):
            cand = os.path.join(d, name)
            if os.path.exists(cand):
                _includes(cand, seen)
                break
    return seen


def _obj_fresh(src, obj):
    if not os.path.exists(obj):
        return False
    t = os.path.getmtime(obj)
    return all(os.path.getmtime(p) <= t for p in _includes(src))


def _compile(job):
    src, obj, defs = job
    log = obj + ".log"  # per-object ptxas output, reused while the object is up to date
    if not FORCE and _obj_fresh(src, obj):
        return obj, 0, open(log).read() if os.path.exists(log) else "(up to date)"
    cmd = [nvcc(), *ARCH, *CFLAGS, *defs, f"-I{INCLUDE}", f"-I{CSRC}", "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as fh:
        fh.write(res.stdout + res.stderr)
    return obj, res.returncode, res.stdout + res.stderr


FORCE = False


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    global FORCE
    FORCE = force
    if not force and up_to_date():
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)
    work = [(os.path.join(CSRC, "pu_api.cu"), os.path.join(OBJDIR, "pu_api.o"), []),
            (os.path.join(CSRC, "pu_host.cu"), os.path.join(OBJDIR, "pu_host.o"), []),
            (os.path.join(CSRC, "pu_synth.cu"), os.path.join(OBJDIR, "pu_synth.o"), [])]
    for t, ls in INSTANCES:
        work.append((os.path.join(CSRC, "pu_dct_inst.cu"), os.path.join(OBJDIR, f"pu_dct_{t}_{ls}.o"),
                     [f"-DPU_INST_T={t}", f"-DPU_INST_LS={ls}"]))
    for t, lh in SPLIT_INSTANCES:
        work.append((os.path.join(CSRC, "pu_split_inst.cu"), os.path.join(OBJDIR, f"pu_split_{t}_{lh}.o"),
                     [f"-DPU_INST_T={t}", f"-DPU_INST_LH={lh}"]))
    jobs = jobs or max(1, min(len(work), os.cpu_count() or 1))
    logs = []
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        for obj, rc, out in ex.map(_compile, work):
            logs.append(f"==== {os.path.basename(obj)}\n{out}")
            if rc != 0:
                sys.stderr.write(out)
                raise RuntimeError(f"nvcc failed for {obj} ({rc})")
    with open(os.path.join(LIBDIR, "ptxas.log"), "w") as fh:
        fh.write("\n".join(logs))
    tmp = LIB + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", *[w[1] for w in work], "-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    if verbose:
        sys.stderr.write("\n".join(logs))
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
