"""Seeded synthetic inputs shared by the tests and bench.py.

This module holds NO arithmetic of the method: it only draws random uint16 matrices in the
boundary encoding (0xFFFF = +inf, finite values <= 0x7FFE).  Both the CUDA path and the
CPU oracle consume what it returns; neither side imports the other.

Recipes: SURVEY.md section 8(d), kernel micro-bench row --
A: uniform [0, 12] with P(inf) in {0, 0.5, 0.992} (the transfer matrices have entries
<= n and density 27% .. 0.77%); B: uniform [0, 600] with P(inf) = 0 (the dense powers
have entries <= n*k); a saturation set with large finite values and a short inner
dimension so that many sums reach 0x7FFF and must come out +inf.
"""
from __future__ import annotations

import numpy as np

INF = 0xFFFF
FINITE_MAX = 0x7FFE
SEED = 17688


def rng(seed: int = SEED, *salt: int) -> np.random.Generator:
    return np.random.default_rng([seed, *salt])


def tropical_matrix(rows: int, cols: int, lo: int = 0, hi: int = 600, p_inf: float = 0.0,
                    seed: int = SEED, salt: int = 0) -> np.ndarray:
    """uint16 matrix, finite entries uniform in [lo, hi], each entry +inf with p_inf."""
    g = rng(seed, salt, rows, cols)
    X = g.integers(lo, hi + 1, size=(rows, cols), dtype=np.int64).astype(np.uint16)
    if p_inf > 0.0:
        X[g.random((rows, cols)) < p_inf] = INF
    return X


def transfer_like(rows: int, cols: int, p_inf: float, seed: int = SEED, salt: int = 0) -> np.ndarray:
    """The A operand recipe: small labels [0, 12] with many +inf."""
    return tropical_matrix(rows, cols, 0, 12, p_inf, seed, salt)


def power_like(rows: int, cols: int, seed: int = SEED, salt: int = 0) -> np.ndarray:
    """The B operand recipe: dense, entries [0, 600]."""
    return tropical_matrix(rows, cols, 0, 600, 0.0, seed, salt)


def saturation_pair(M: int, K: int, N: int, seed: int = SEED, salt: int = 0):
    """Finite entries in [0x3F00, 0x7FFE] so a + b often exceeds 0x7FFE (-> +inf)."""
    A = tropical_matrix(M, K, 0x3F00, FINITE_MAX, 0.1, seed, salt)
    B = tropical_matrix(K, N, 0x3F00, FINITE_MAX, 0.1, seed, salt + 1)
    return A, B
