"""Write the per-power golden records of the power sequence of A(D_n) -- ORACLE ONLY.

Usage: python tests/golden/make_power_records.py 10 11 12   (n = path order, G1)

Imports nothing but ``oracle/`` (and numpy / hashlib / json).  For each n it runs Algorithm 2
(A^1 = A, A^k = A (x) A^{k-1}, left multiplication G8) with the oracle's skip-inf
triple loop (``oracle.minplus``, pinned to the literal ijk loop, the scipy shortest-path
library pin and the paper's Tables 4/5 in tests/test_oracle.py), until the first repeat
A^k = c (x) A^j (Lemma 1; reading G9), and writes, for every power k:

  fingerprint  H(A^k) = sum_ij s(2i) s(2j+1) x_ij mod 2^64 (oracle.fingerprint_cols over
               column blocks, summed: the fingerprint is additive over columns -- pinned in
               test_oracle.py), as a decimal string;
  diag_min     min_i (A^k)_ii (Algorithm 5);
  inf_count    number of +inf (0xFFFF) entries;
  ref          (t << 16) | x_t of the first finite entry in row-major order t = i*N + j;
  sha256       SHA-256 of the whole N x N matrix as row-major little-endian uint16, boundary
               encoding (0xFFFF = +inf) -- lets a GPU run prove every entry of every power
               equal without the oracle on the GPU box;

plus (mu, lambda, offset) of the first repeat and the constant confirmed by
oracle.constant_difference.

Only the last RING powers are kept in RAM (a power is 2 N^2 bytes: 5.6 GB at n = 12).  For
j still in the ring the repeat test is the oracle's exact constant_difference.  For an
evicted j the script applies a NECESSARY condition of A^k = c (x) A^j: equal inf counts, the
first finite entry at the same position with c = x_k - x_j, and, when both are inf-free,
H(A^k) - H(A^j) = c * S (mod 2^64) with S = H(all-ones); the fingerprint is linear, so a
true repeat always satisfies it.  If an evicted j ever passed it the script would stop
(ring too small) instead of guessing -- so "no repeat with j" is always proven.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

RING = 4
MASK = (1 << 64) - 1


def fingerprint_parallel(X: np.ndarray, threads: int) -> int:
    """H(X) as the sum of oracle.fingerprint_cols over column blocks (ctypes drops the GIL)."""
    N = X.shape[1]
    step = -(-N // threads)
    blocks = [(c, min(N, c + step)) for c in range(0, N, step)]
    with cf.ThreadPoolExecutor(len(blocks)) as ex:
        parts = list(ex.map(lambda b: oracle.fingerprint_cols(X, b[0], b[1]), blocks))
    return sum(parts) & MASK


def ref_entry(X: np.ndarray) -> int:
    flat = X.reshape(-1)
    for t0 in range(0, flat.size, 1 << 24):  # chunked: no N^2-sized index array
        fin = np.flatnonzero(flat[t0:t0 + (1 << 24)] != oracle.INF)
        if fin.size:
            t = t0 + int(fin[0])
            return (t << 16) | int(flat[t])
    return (1 << 63) - 1


def sha256_le16(X: np.ndarray) -> str:
    assert X.dtype == np.uint16 and X.flags["C_CONTIGUOUS"] and sys.byteorder == "little"
    return hashlib.sha256(memoryview(X.reshape(-1)).cast("B")).hexdigest()


def record(X: np.ndarray, k: int, threads: int) -> dict:
    diag = np.diagonal(X)
    return {
        "k": k,
        "fingerprint": str(fingerprint_parallel(X, threads)),
        "diag_min": int(diag.min()),
        "inf_count": int(sum(np.count_nonzero(r == oracle.INF) for r in X)),
        "ref": int(ref_entry(X)),
        "sha256": sha256_le16(X),
    }


def necessary(rk: dict, rj: dict, S: int) -> bool:
    """Necessary condition for A^k = c (x) A^j from the records alone (see module doc)."""
    if rk["inf_count"] != rj["inf_count"]:
        return False
    if (rk["ref"] >> 16) != (rj["ref"] >> 16):
        return False
    if rk["inf_count"] == 0:
        c = (rk["ref"] & 0xFFFF) - (rj["ref"] & 0xFFFF)
        return (int(rk["fingerprint"]) - int(rj["fingerprint"])) & MASK == (c * S) & MASK
    return True


def run(n: int, threads: int, max_k: int = 64) -> dict:
    t0 = time.time()
    A = oracle.transition_matrix(n)
    N = A.shape[0]
    # S = H(all-ones) = (sum_i s(2i)) (sum_j s(2j+1)): the bilinear form factorises; checked
    # against the fingerprint of an all-ones matrix where that is cheap.
    si = sum(oracle.splitmix64(2 * i) for i in range(N)) & MASK
    sj = sum(oracle.splitmix64(2 * j + 1) for j in range(N)) & MASK
    S = (si * sj) & MASK
    if N <= 4096:
        assert S == fingerprint_parallel(np.ones((N, N), dtype=np.uint16), threads)
    # Keep every power when max_k of them fit in 8 GB (n <= 10); else the last RING.
    keep = max_k if 2 * N * N * max_k <= 8 << 30 else RING
    recs = [None, record(A, 1, threads)]
    ring = {1: A}
    out = {"n": n, "N": N, "nnz": int(np.count_nonzero(A != oracle.INF)), "S": str(S)}
    print(f"n={n} N={N} k=1 {time.time() - t0:.1f}s", flush=True)
    X = A
    for k in range(2, max_k + 1):
        X = oracle.minplus(A, X)  # A^k = A (x) A^{k-1}
        rk = record(X, k, threads)
        recs.append(rk)
        hit = None
        for j in range(k - 1, 0, -1):
            if j in ring:
                c = oracle.constant_difference(X, ring[j])
                if c is not None:
                    hit = (j, c)
                    break
            elif necessary(rk, recs[j], S):
                raise RuntimeError(f"n={n}: evicted power {j} passes the necessary test at k={k}; "
                                   f"raise RING")
        ring[k] = X
        if keep < max_k:
            for j in [j for j in ring if j <= k - keep and j != 1]:
                del ring[j]
        print(f"n={n} k={k} diag_min={rk['diag_min']} inf={rk['inf_count']} "
              f"{time.time() - t0:.1f}s", flush=True)
        if hit:
            j, c = hit
            out.update(mu=j, lambda_=k - j, offset=c, k_last=k)
            break
    else:
        raise RuntimeError(f"n={n}: no repeat up to k={max_k}")
    out["powers"] = recs[1:]
    out["seconds"] = round(time.time() - t0, 1)
    out["threads"] = threads
    out["generator"] = "tests/golden/make_power_records.py (oracle only)"
    return out


def main() -> None:
    threads = oracle.num_threads()
    for n in [int(a) for a in sys.argv[1:]] or [10]:
        rec = run(n, threads)
        path = os.path.join(ROOT, "tests", "golden", f"power_records_n{n}.json")
        with open(path, "w") as f:
            json.dump(rec, f, indent=1)
        print(f"wrote {path}: mu={rec['mu']} lambda={rec['lambda_']} b={rec['offset']} "
              f"in {rec['seconds']} s on {threads} threads", flush=True)


if __name__ == "__main__":
    main()
