"""In-tree build of libsinga_b200.so (nvcc, sm_100a only).

Usage: python -m paper_1603_07846_b200.build [--force] [-j N] [--variant NAME -D MACRO ...]

A variant (A/B experiments, instrumentation) builds into build/<NAME>/ and
links build/<NAME>/libsinga_b200.so; load it with SG_LIB=<path>.
"""

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(HERE, "libsinga_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    site = sysconfig.get_paths()["purelib"]
    base = os.path.join(site, "nvidia", "nccl")
    return os.path.join(base, "include"), os.path.join(base, "lib")


EXTRA = []  # extra nvcc flags of a variant build


def flags():
    inc, _ = nccl_dirs()
    return ARCH + EXTRA + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
                   "-I", CSRC, "-I", os.path.join(ROOT, "include"), "-I", inc, "--expt-relaxed-constexpr"]


def _compile(src, force):
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    deps = [src] + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj, None
    cmd = [NVCC] + flags() + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        return obj, " ".join(cmd) + "\n" + r.stdout + r.stderr
    return obj, None


def build(force=False, jobs=None, verbose=True):
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = jobs or max(1, min(len(srcs), os.cpu_count() or 4))
    objs = []
    with cf.ThreadPoolExecutor(jobs) as ex:
        for obj, err in ex.map(lambda s: _compile(s, force), srcs):
            if err:
                raise RuntimeError("nvcc failed:\n" + err)
            objs.append(obj)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        _, libdir = nccl_dirs()
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + \
            ["-L" + libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + libdir]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        if verbose:
            print("built", LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("--variant", default=None)
    ap.add_argument("-D", action="append", default=[])
    a = ap.parse_args()
    if a.variant:
        EXTRA[:] = ["-D" + d for d in a.D]
        BUILD = os.path.join(ROOT, "build", a.variant, "obj")
        LIB = os.path.join(ROOT, "build", a.variant, "libsinga_b200.so")
    try:
        build(a.force or bool(a.variant), a.j)
    except RuntimeError as e:
        print(e, file=sys.stderr)
        sys.exit(1)
