"""Build the C-ABI library libhq.so in-tree for sm_100a (nvcc, no JIT cache).

    python -m paper_2111_06868_b200.build

Outputs paper_2111_06868_b200/lib/libhq.so.  Kernels are compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo`` so ncu's source page maps
to the code.  NCCL is the torch-bundled NCCL 2.28 (linked with an rpath).
"""
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libhq.so")
# checked variant (-DHQ_DEVICE_CHECKS): mbarrier watchdogs and bounds checks on
# every tensor-core / SIMT global access; tests load it through HQ_LIB
LIB_CHECK = os.path.join(LIBDIR, "libhq_check.so")
INCLUDE = os.path.join(ROOT, "include")

SOURCES = ["hq_apply.cu", "hq_tc.cu", "hq_state_ops.cu", "hq_runtime.cpp", "hq_plan.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    purelib = sysconfig.get_paths()["purelib"]
    base = os.path.join(purelib, "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if not os.path.exists(os.path.join(inc, "nccl.h")):
        raise RuntimeError("nccl.h not found under %s" % inc)
    return inc, lib


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    return "nvcc"


def _stale(lib=LIB):
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "hq.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force=False, verbose=False, checked=False):
    lib = LIB_CHECK if checked else LIB
    if not force and not _stale(lib):
        return lib
    if not force and os.environ.get("HQ_NO_BUILD") and os.path.exists(lib):
        return lib          # use the shipped build as is (GPU-box scripts)
    os.makedirs(LIBDIR, exist_ok=True)
    inc, nlib = _nccl_dirs()
    objdir = os.path.join(LIBDIR, "obj_check" if checked else "obj")
    os.makedirs(objdir, exist_ok=True)
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC, "-I", inc]
    if checked:
        common += ["-DHQ_DEVICE_CHECKS"]
    objs = []
    procs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        if not os.path.exists(path):
            continue
        obj = os.path.join(objdir, src + ".o")
        cmd = [nvcc()] + common + ARCH + ["-lineinfo", "-c", path, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
            cmd += ["--expt-relaxed-constexpr"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT), cmd))
        objs.append(obj)
    for p, cmd in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError("nvcc failed:\n%s\n%s" % (" ".join(cmd), out.decode(errors="replace")))
        if verbose and out:
            sys.stderr.write(out.decode(errors="replace"))
    link = [nvcc(), "-shared"] + ARCH + objs + [
        "-L" + nlib, "-Xlinker", "-l:libnccl.so.2", "-Xlinker", "-rpath=" + nlib, "-o", lib]
    subprocess.check_call(link)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
