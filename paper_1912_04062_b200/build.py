"""Build the sm_100a C-ABI library libskeweig.so in-tree with nvcc (no torch JIT cache).

    python -m paper_1912_04062_b200.build            # incremental
    python -m paper_1912_04062_b200.build --force
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libskeweig.so")
ROOT = os.path.dirname(HERE)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]
SOURCES = ["api.cu", "f2b.cu", "b2t.cu", "tridiag.cu", "bt1.cu", "bse.cu", "coll.cu", "onestep.cu"]
HEADERS = ["common.cuh", "gemm_dmma.cuh", "tma_gemm.cuh", "internal.h"]


def _nccl_flags():
    """NCCL: torch's bundled libnccl (2.28) if present, else the system one."""
    try:
        import nvidia.nccl as nn  # noqa  (namespace package: no __file__)
        d = list(nn.__path__)[0]
        inc = os.path.join(d, "include")
        lib = os.path.join(d, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return ["-I" + inc], ["-L" + lib, "-Xlinker", "-rpath=" + lib, "-l:libnccl.so.2"]
    except Exception:
        pass
    return [], ["-lnccl"]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", f)
                                                        for f in os.listdir(os.path.join(ROOT, "include"))]
    inc_nccl, lib_nccl = _nccl_flags()
    jobs = []
    objs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s.replace(".cu", ".o"))
        objs.append(obj)
        if force or _newer(obj, [src] + hdrs):
            jobs.append([NVCC, *ARCH, *FLAGS, *inc_nccl, "-c", src, "-o", obj])

    def run(cmd):
        if verbose:
            print(" ".join(cmd))
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        return r.stdout + r.stderr

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for out in ex.map(run, jobs):
            if verbose and out.strip():
                print(out)
    if force or jobs or _newer(LIB, objs):
        run([NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-lcudart", *lib_nccl])
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
