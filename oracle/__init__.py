"""CPU oracle for arXiv 2409.17688 -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct implementations of what the hot path computes (see
``oracle/oracle.c`` and ``oracle/graph.c`` for the per-function citations).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2409_17688_b200`` never imports it and shares no code with it.

Parity status:
  words / transition matrix / product / powers / periodicity / gamma_2 read-off:
      pinned (Table 1, SPEC hand examples, scipy shortest paths, Table 5, Table 7,
      closed forms, brute force, column DP);
  fingerprint: pinned (splitmix64 published test vectors, linearity);
  power_rows: pinned against the full powers of oracle_power_until_periodic (n <= 9).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRCS = [os.path.join(_HERE, "oracle.c"), os.path.join(_HERE, "graph.c")]

INF = 0xFFFF
FINITE_MAX = 0x7FFE
MAX_K = 256


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (generic x86-64-v2 so the .so runs on any host)."""
    newest = max(os.path.getmtime(s) for s in _SRCS)
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        tmp = _SO + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC",
               "-std=c99", "-Wall", "-o", tmp] + _SRCS
        subprocess.run(cmd, check=True)
        os.replace(tmp, _SO)
    return _SO


class PeriodicResult(ctypes.Structure):
    _fields_ = [("mu", ctypes.c_int32), ("lambda_", ctypes.c_int32),
                ("offset", ctypes.c_int32), ("k_last", ctypes.c_int32),
                ("dense_from", ctypes.c_int32),
                ("diag_min", ctypes.c_uint16 * (MAX_K + 1)),
                ("fingerprint", ctypes.c_uint64 * (MAX_K + 1))]


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        L.oracle_is_correct_word.argtypes = [P, ctypes.c_int]
        L.oracle_words.argtypes = [ctypes.c_int, P]
        L.oracle_words.restype = i64
        L.oracle_can_follow.argtypes = [P, P, ctypes.c_int]
        L.oracle_zero_count.argtypes = [P, ctypes.c_int]
        L.oracle_transition_matrix.argtypes = [ctypes.c_int, P]
        L.oracle_transition_matrix.restype = i64
        for f in (L.oracle_minplus_ijk, L.oracle_minplus_ikj):
            f.argtypes = [P, P, P, i64, i64, i64]
            f.restype = None
        L.oracle_splitmix64.argtypes = [ctypes.c_uint64]
        L.oracle_splitmix64.restype = ctypes.c_uint64
        L.oracle_fingerprint.argtypes = [P, i64, i64]
        L.oracle_fingerprint.restype = ctypes.c_uint64
        L.oracle_fingerprint_cols.argtypes = [P, i64, i64, i64, i64]
        L.oracle_fingerprint_cols.restype = ctypes.c_uint64
        L.oracle_constant_difference.argtypes = [P, P, i64, P]
        L.oracle_power_until_periodic.argtypes = [P, i64, ctypes.c_int, P]
        L.oracle_power_rows.argtypes = [P, i64, i64, ctypes.c_int, P]
        L.oracle_power_rows.restype = None
        L.oracle_gamma2_readoff.argtypes = [P, i64]
        L.oracle_gamma2_readoff.restype = i64
        L.oracle_gamma2_bruteforce.argtypes = [ctypes.c_int, ctypes.c_int]
        L.oracle_gamma2_column_dp.argtypes = [ctypes.c_int, ctypes.c_int]
        L.oracle_gamma2_path_dp.argtypes = [ctypes.c_int, ctypes.c_int]
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


# ---------------------------------------------------------------------------- c1-c3 words
def words(n: int) -> np.ndarray:
    """All correct n-words, lexicographic, as an (N, n) uint8 array."""
    N = lib().oracle_words(n, None)
    out = np.zeros((N, n), dtype=np.uint8)
    lib().oracle_words(n, _ptr(out))
    return out


def count_words(n: int) -> int:
    return int(lib().oracle_words(n, None))


def is_correct_word(w) -> bool:
    a = np.ascontiguousarray(np.asarray(w, dtype=np.uint8))
    r = lib().oracle_is_correct_word(_ptr(a), len(a))
    if r < 0:
        raise ValueError("letter outside {0,1,2}")
    return bool(r)


def can_follow(q, p) -> bool:
    a = np.ascontiguousarray(np.asarray(q, dtype=np.uint8))
    b = np.ascontiguousarray(np.asarray(p, dtype=np.uint8))
    if len(a) != len(b):
        raise ValueError("length mismatch")
    return bool(lib().oracle_can_follow(_ptr(a), _ptr(b), len(a)))


def transition_matrix(n: int) -> np.ndarray:
    """A(D_n) (Algorithm 1), uint16 with 0xFFFF = inf."""
    N = count_words(n)
    A = np.empty((N, N), dtype=np.uint16)
    lib().oracle_transition_matrix(n, _ptr(A))
    return A


# ---------------------------------------------------------------------------- c4 product
def minplus(A: np.ndarray, B: np.ndarray, literal: bool = False) -> np.ndarray:
    """C = A x B over (min,+) with the G6 saturation."""
    A = np.ascontiguousarray(A, dtype=np.uint16)
    B = np.ascontiguousarray(B, dtype=np.uint16)
    M, K = A.shape
    K2, N = B.shape
    assert K == K2
    C = np.empty((M, N), dtype=np.uint16)
    f = lib().oracle_minplus_ijk if literal else lib().oracle_minplus_ikj
    f(_ptr(A), _ptr(B), _ptr(C), M, K, N)
    return C


def splitmix64(t: int) -> int:
    return int(lib().oracle_splitmix64(t))


def fingerprint(X: np.ndarray) -> int:
    X = np.ascontiguousarray(X, dtype=np.uint16)
    return int(lib().oracle_fingerprint(_ptr(X), X.shape[0], X.shape[1]))


def fingerprint_cols(X: np.ndarray, c0: int, c1: int) -> int:
    X = np.ascontiguousarray(X, dtype=np.uint16)
    return int(lib().oracle_fingerprint_cols(_ptr(X), X.shape[0], X.shape[1], c0, c1))


def constant_difference(Y: np.ndarray, X: np.ndarray):
    Y = np.ascontiguousarray(Y, dtype=np.uint16)
    X = np.ascontiguousarray(X, dtype=np.uint16)
    c = ctypes.c_int32(0)
    ok = lib().oracle_constant_difference(_ptr(Y), _ptr(X), Y.size, ctypes.addressof(c))
    return int(c.value) if ok else None


# ---------------------------------------------------------------------------- c5-c7
class Periodic:
    def __init__(self, r: PeriodicResult, rc: int):
        self.rc = rc
        self.mu, self.lam, self.offset = r.mu, r.lambda_, r.offset
        self.k_last, self.dense_from = r.k_last, r.dense_from
        self.diag_min = [int(r.diag_min[k]) for k in range(r.k_last + 1)]
        self.fingerprint = [int(r.fingerprint[k]) for k in range(r.k_last + 1)]
        self._raw = r

    def gamma2(self, m: int) -> int:
        return int(lib().oracle_gamma2_readoff(ctypes.addressof(self._raw), m))


def power_until_periodic(A: np.ndarray, max_k: int = 64) -> Periodic:
    A = np.ascontiguousarray(A, dtype=np.uint16)
    r = PeriodicResult()
    rc = lib().oracle_power_until_periodic(_ptr(A), A.shape[0], max_k, ctypes.addressof(r))
    return Periodic(r, rc)


def power_rows(A: np.ndarray, r: int, kmax: int) -> np.ndarray:
    """Row r of A^1..A^kmax as a (kmax, N) array (row k-1 = row r of A^k)."""
    A = np.ascontiguousarray(A, dtype=np.uint16)
    out = np.empty((kmax, A.shape[0]), dtype=np.uint16)
    lib().oracle_power_rows(_ptr(A), A.shape[0], r, kmax, _ptr(out))
    return out


def powers(A: np.ndarray, K: int) -> dict:
    """Algorithm 2: {i: A^i} for i = 1..K, A^i = A x A^(i-1)."""
    P = {1: np.ascontiguousarray(A, dtype=np.uint16)}
    for i in range(2, K + 1):
        P[i] = minplus(A, P[i - 1])
    return P


def algorithm3(P: dict, K: int):
    """Algorithm 3 verbatim: for i = K down to 1, for j = i-1 down to 1, the
    first pair with A^i - A^j constant gives a = i - j, b = the constant, r0 = j."""
    for i in range(K, 0, -1):
        for j in range(i - 1, 0, -1):
            c = constant_difference(P[i], P[j])
            if c is not None:
                return j, i - j, c
    return None


def algorithm4(P: dict, r0: int, a: int, b: int):
    """Algorithm 4 verbatim: for i = r0 + a down to 1 (while i - a >= 1, reading
    G11), exit at the first i with A^i - A^(i-a) != b; otherwise n0 = i - a."""
    n0 = None
    for i in range(r0 + a, 0, -1):
        if i - a < 1:
            break
        if constant_difference(P[i], P[i - a]) != b:
            break
        n0 = i - a
    return n0


def gamma2(n: int, m: int, max_k: int = 64) -> int:
    """gamma_2(P_n x C_m) from the transfer matrix (Theorems 2 and 3)."""
    return power_until_periodic(transition_matrix(n), max_k).gamma2(m)


def gamma2_bruteforce(n: int, m: int) -> int:
    return int(lib().oracle_gamma2_bruteforce(n, m))


def gamma2_column_dp(n: int, m: int) -> int:
    return int(lib().oracle_gamma2_column_dp(n, m))


def gamma2_path_dp(n: int, m: int) -> int:
    """gamma_2(P_n x C_m) by DP along the path over row subsets of C_m (any n, m <= 8)."""
    return int(lib().oracle_gamma2_path_dp(n, m))


def num_threads() -> int:
    return int(lib().oracle_num_threads())
