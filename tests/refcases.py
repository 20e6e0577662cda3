"""Input recipes of the reference's own hot-path tests, reproduced exactly.

``numpy.random.RandomState(seed)`` yields the same raw 32-bit stream as
``std::mt19937(seed)``, so the helpers of
/root/reference/proj/tests/test_kernels.cpp:13-51 (random_matrix, random_chw,
random_bias, masked_case) produce the reference tests' exact inputs. Masks come
from the oracle's restatement of generate_mask (libstdc++ semantics), pinned
against the compiled reference in tests/test_oracle.py.
"""
from __future__ import annotations

import numpy as np

F = np.float32


class Mt:
    """std::mt19937 raw draws."""

    def __init__(self, seed: int):
        self.rs = np.random.RandomState(seed)

    def __call__(self, n: int | None = None):
        if n is None:
            return int(self.rs.randint(0, 2**32, dtype=np.uint64))
        return self.rs.randint(0, 2**32, size=n, dtype=np.uint64)


def random_matrix(rows: int, cols: int, rng: Mt) -> np.ndarray:
    """test_kernels.cpp:13-17: rng()%2000/999.0f - 1.0f."""
    r = rng(rows * cols) % 2000
    return (r.astype(F) / F(999.0) - F(1.0)).astype(F).reshape(rows, cols)


def random_chw(c: int, h: int, w: int, rng: Mt) -> np.ndarray:
    """test_kernels.cpp:19-23: rng()%1000/999.0f."""
    r = rng(c * h * w) % 1000
    return (r.astype(F) / F(999.0)).astype(F).reshape(c, h, w)


def random_bias(n: int, rng: Mt) -> np.ndarray:
    """test_kernels.cpp:25-29: rng()%200/99.0f - 1.0f."""
    r = rng(n) % 200
    return (r.astype(F) / F(99.0) - F(1.0)).astype(F)


def masked_case(rows, cols, sparsity, block_h, rng: Mt, oracle):
    """test_kernels.cpp:44-51: dense weights, then generate_mask(seed=rng()), apply, encode."""
    from paper_1911_09723_b200 import encode_bcsr

    dense = random_matrix(rows, cols, rng)
    rc, keep = oracle.generate_mask(rows, cols, sparsity, block_h, 1, rng())
    assert rc == 0
    dense = np.where(keep, dense, F(0.0)).astype(F)
    return dense, encode_bcsr(dense, block_h)
