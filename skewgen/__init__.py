"""Seeded synthetic input generators shared by the oracle tests, the CUDA-path
tests and bench.py.

This module holds NONE of the method's arithmetic (no reflectors, no
eigen-solves): it only produces input matrices from a counter-based generator,
so that the oracle (``oracle/``) and the CUDA path (``paper_1912_04062_b200``)
consume bit-identical inputs.

Generator (DESIGN.md §Input recipe; SURVEY §8(c) "Generator"; the paper only
says "randomly generated skew-symmetric matrices in double precision",
PAPER.md:797-798, distribution unstated -> reading R12: uniform [-1, 1)):

    key(i, j)  = seed * 0x9E3779B97F4A7C15 + j * n + i          (mod 2**64)
    z          = splitmix64(key)
    a_ij       = 2 * ((z >> 11) * 2**-53) - 1                   (exact in fp64)

for the strictly lower triangle i > j; upper = -lower, diagonal = 0.
``splitmix64(x)`` is the standard SplitMix64 output function applied to
``x + 0x9E3779B97F4A7C15``.

Two implementations of the same specification exist: numpy (here) and a CUDA
kernel (``skewgen/skewgen.cu`` -> ``libskewgen.so``) used for large n in
bench.py. tests/test_generator.py checks them bit for bit.
"""
from .gen import (splitmix64, uniform_pm1, random_skew, random_skew_lower_colmajor,
                  skew_toeplitz, planted_skew, bse_spd, bse_AB, J_matrix)

__all__ = ["splitmix64", "uniform_pm1", "random_skew", "random_skew_lower_colmajor",
           "skew_toeplitz", "planted_skew", "bse_spd", "bse_AB", "J_matrix"]


def build_device_lib(force=False):
    """Compile skewgen.cu -> libskewgen.so (input generation only)."""
    import os
    import subprocess
    here = os.path.dirname(os.path.abspath(__file__))
    src = os.path.join(here, "skewgen.cu")
    lib = os.path.join(here, "libskewgen.so")
    if force or not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(src):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-Xcompiler", "-fPIC", "-shared", "-o", lib + ".tmp", src])
        os.replace(lib + ".tmp", lib)
    return lib


def random_skew_lower_device(A, n, seed, stream=0):
    """Fill the column-major CUDA buffer A (ld = A.stride(1)) with the strictly-lower
    random skew matrix of (n, seed) -- bit-identical to random_skew(n, seed)."""
    import ctypes
    L = ctypes.CDLL(build_device_lib())
    f = L.skewgen_random_skew_lower_device
    f.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p]
    rc = f(ctypes.c_void_p(A.data_ptr()), n, A.stride(1), seed, ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"skewgen device kernel failed: {rc}")
