"""Build the engine's shared library in-tree: paper_2603_13289_b200/librelaykv_b200.so.

nvcc cross-compiles for sm_100a only (no GPU needed). Incremental: a source
is recompiled when it or any header under csrc/ or include/ is newer than
its object. Usage: python -m paper_2603_13289_b200.build [-j N] [--force]
"""
import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_obj")
LIB = os.path.join(HERE, "librelaykv_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
# Exact kernels must never contract a*b+c into an FMA the reference lacks.
NO_FMAD = {"kernels_exact.cu", "kernels_common.cu"}


def _cxx():
    return "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


def _headers():
    return glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))


def _cmd(src, obj):
    inc = ["-I", CSRC, "-I", os.path.join(ROOT, "include")]
    name = os.path.basename(src)
    if src.endswith(".cu"):
        return [NVCC, *GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr",
                "-fmad=false" if name in NO_FMAD else "-fmad=true",
                *inc, "-c", src, "-o", obj]
    return [_cxx(), "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall", "-Wno-unused-function",
            *inc, "-I", os.path.join(CUDA, "include"), "-c", src, "-o", obj]


def build(jobs=8, force=False, verbose=False):
    if not os.path.exists(NVCC):
        raise RuntimeError(f"nvcc not found at {NVCC}")
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    hdr_mtime = max([os.path.getmtime(h) for h in _headers()] + [0])
    todo, objs = [], []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s) + ".o")
        objs.append(o)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), hdr_mtime):
            todo.append((s, o))

    def run(so):
        s, o = so
        cmd = _cmd(s, o)
        if verbose:
            print(" ".join(cmd), flush=True)
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"compile failed: {os.path.basename(s)}\n{p.stdout}\n{p.stderr}")
        return s

    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        for s in ex.map(run, todo):
            print(f"[build] {os.path.basename(s)}", flush=True)
    if todo or not os.path.exists(LIB):
        link = [NVCC, *GENCODE, "-shared", "-cudart", "static", "-o", LIB + ".tmp", *objs, "-lpthread"]
        p = subprocess.run(link, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed\n{p.stdout}\n{p.stderr}")
        shutil.move(LIB + ".tmp", LIB)
        print(f"[build] linked {os.path.relpath(LIB, ROOT)}", flush=True)
    build_dropin(force)
    return LIB


DROPIN = os.path.join(HERE, "librelaykv_dropin.so")
DROPIN_TEST = os.path.join(HERE, "_bin", "test_dropin")


def build_dropin(force=False):
    """The C++ drop-in (namespace relaykv, cpp/) over the C ABI, and its test binary."""
    src = os.path.join(HERE, "cpp", "relaykv_dropin.cpp")
    hdrs = glob.glob(os.path.join(HERE, "cpp", "include", "relaykv", "*.hpp")) + \
        [os.path.join(ROOT, "include", "relaykv_b200.h")]
    newest = max(os.path.getmtime(f) for f in [src, LIB] + hdrs)
    inc = ["-I", os.path.join(HERE, "cpp", "include"), "-I", os.path.join(ROOT, "include")]
    if force or not os.path.exists(DROPIN) or os.path.getmtime(DROPIN) < newest:
        subprocess.run([_cxx(), "-std=c++20", "-O2", "-fPIC", "-shared", *inc, src, "-o", DROPIN,
                        "-L", HERE, "-lrelaykv_b200", "-Wl,-rpath,$ORIGIN"], check=True)
        print(f"[build] linked {os.path.relpath(DROPIN, ROOT)}", flush=True)
    test_src = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
    oracle_lib = os.path.join(ROOT, "oracle", "build", "liboracle.so")
    if os.path.exists(test_src) and os.path.exists(oracle_lib) and \
            (force or not os.path.exists(DROPIN_TEST) or
             os.path.getmtime(DROPIN_TEST) < max(newest, os.path.getmtime(test_src), os.path.getmtime(DROPIN))):
        os.makedirs(os.path.dirname(DROPIN_TEST), exist_ok=True)
        subprocess.run([_cxx(), "-std=c++20", "-O2", *inc, "-I", os.path.join(ROOT, "oracle", "doctest_shim"),
                        test_src, "-o", DROPIN_TEST, "-L", HERE, "-lrelaykv_dropin", "-lrelaykv_b200",
                        "-L", os.path.dirname(oracle_lib), "-loracle",
                        f"-Wl,-rpath,{HERE}", f"-Wl,-rpath,{os.path.dirname(oracle_lib)}",
                        "-Wl,-rpath,$ORIGIN/..", "-Wl,-rpath,$ORIGIN/../../oracle/build"], check=True)
        print(f"[build] linked {os.path.relpath(DROPIN_TEST, ROOT)}", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=os.cpu_count() or 8)
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args()
    try:
        build(a.j, a.force, a.v)
    except RuntimeError as e:
        print(e, file=sys.stderr)
        sys.exit(1)
