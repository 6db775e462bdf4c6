"""Build the C-ABI shared library libbdattn.so in-tree with nvcc (sm_100a).

    python -m paper_2512_22234_b200.build        # or __graft_entry__.build()

The .so lands next to this file so it travels with the repo snapshot to the
GPU box (it is git-ignored, not gpurun-ignored).  No torch.utils.cpp_extension
and no JIT cache: the library has a plain C ABI and is loaded with ctypes.
"""

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbdattn.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    "-I", os.path.join(ROOT, "include"),
]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def build(verbose=False, force=False):
    srcs = sources()
    deps = srcs + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    if not force and not os.environ.get("BD_NVCC_EXTRA") and os.path.exists(LIB):
        lib_m = os.path.getmtime(LIB)
        if all(os.path.getmtime(d) <= lib_m for d in deps):
            return LIB
    # dev A/B builds: extra nvcc flags (e.g. -DBD_DKDV_SPLIT=0) into a separate
    # object dir and library path; the product build never sets these
    extra = os.environ.get("BD_NVCC_EXTRA", "").split()
    lib = os.environ.get("BD_LIB_OUT", LIB) if extra else LIB
    objdir = os.path.join(HERE, "build" + ("_ab" if extra else ""))
    os.makedirs(objdir, exist_ok=True)
    nvcc = _nvcc()

    def compile_one(s):
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        r = subprocess.run([nvcc, *NVCC_FLAGS, *extra, "-c", s, "-o", o], capture_output=True, text=True)
        log = r.stdout + r.stderr
        with open(o + ".ptxas.txt", "w") as f:
            f.write(log)
        return s, o, r.returncode, log

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, srcs))
    objs = []
    for s, o, rc, log in results:
        if verbose or rc:
            sys.stderr.write(log)
        if rc:
            raise RuntimeError(f"nvcc failed on {s}")
        objs.append(o)
    tmp = lib + ".tmp"
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC", "-o", tmp,
           *objs, "-lcudart_static", "-ldl", "-lrt", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
