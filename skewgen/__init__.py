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
                  skew_toeplitz, planted_skew, bse_spd, J_matrix)

__all__ = ["splitmix64", "uniform_pm1", "random_skew", "random_skew_lower_colmajor",
           "skew_toeplitz", "planted_skew", "bse_spd", "J_matrix"]
