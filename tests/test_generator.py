"""Input generator (skewgen) pins: SplitMix64 reference value, exact skew structure, determinism."""
import numpy as np

import skewgen


def test_splitmix64_reference_value():
    # SplitMix64 seeded with 0: first output 0xE220A8397B1DCDAF (Vigna's reference generator)
    assert int(skewgen.splitmix64(np.uint64(0))) == 0xE220A8397B1DCDAF


def test_random_skew_structure_and_determinism():
    A = skewgen.random_skew(100, 3)
    assert np.array_equal(A.T, -A)
    assert np.all(np.diag(A) == 0.0)
    assert np.array_equal(A, skewgen.random_skew(100, 3))
    assert not np.array_equal(A, skewgen.random_skew(100, 4))
    L = np.tril(A, -1)
    assert L.min() >= -1.0 and L.max() < 1.0
    assert skewgen.random_skew(1, 5).shape == (1, 1)


def test_random_skew_entry_formula():
    n, seed = 7, 11
    A = skewgen.random_skew(n, seed)
    i, j = 5, 2
    key = (seed * 0x9E3779B97F4A7C15 + j * n + i) % 2 ** 64
    z = int(skewgen.splitmix64(np.uint64(key)))
    assert A[i, j] == 2.0 * ((z >> 11) * 2.0 ** -53) - 1.0


def test_bse_spd_is_spd():
    M = skewgen.bse_spd(30, 1)
    assert np.array_equal(M, M.T)
    assert np.linalg.eigvalsh(M).min() > 0.9
