"""Host models of the bit-level tricks in the device kernels, checked on CPU against the oracle
or against plain definitions (the kernels themselves are checked on the GPU by test_gpu_*):

* k_check_xfer: the can-follow rule on two columns per 32-bit word, with the
  per-column masks U = up ^ dn, B = up & dn precomputed and the per-half nonzero test
  nz2(v) = (((v & 0x7FFF7FFF) + 0x7FFF7FFF) | v) & 0x80008000, against oracle.can_follow for
  every pair of correct words (n <= 6), and the A(D_n) entry test against the oracle's matrix;
* k_bits_transpose: the five shuffle block-swap stages of the 32 x 32 bit transpose;
* k_tile_union: the per-byte nonzero test of a 32-bit word.
"""
import numpy as np
import pytest

import oracle

M32 = 0xFFFFFFFF


def nz2(v):
    return ((((v & 0x7FFF7FFF) + 0x7FFF7FFF) | v) & 0x80008000) & M32


def masks(w):
    """z, o, t bitmasks (bit i = letter i) and the zero count of a word."""
    z = sum(1 << i for i, c in enumerate(w) if c == 0)
    o = sum(1 << i for i, c in enumerate(w) if c == 1)
    t = sum(1 << i for i, c in enumerate(w) if c == 2)
    return z, o, t, bin(z).count("1")


def pair_fail(q, p0, p1, n):
    """The kernel's fail bits for columns p0 (low half) and p1 (high half) against row q."""
    full = (1 << n) - 1
    qz, _, qt, _ = masks(q)
    qz2, qt2 = qz | qz << 16, qt | qt << 16
    cols = []
    for p in (p0, p1):
        pz, po, pt, _ = masks(p)
        up, dn = (pz << 1) & full, pz >> 1
        cols.append((pz, up ^ dn, up & dn, pt, po))
    pz, pu, pb, pt, po = (cols[0][k] | cols[1][k] << 16 for k in range(5))
    ex1 = (pu ^ qz2) & ~(pb & qz2)
    at2 = pb | (pu & qz2)
    f = ((qt2 & ~pz) | (pt & ~ex1) | (po & ~at2)) & M32
    return nz2(f)


@pytest.mark.parametrize("n", [3, 4, 5, 6])
def test_xfer_can_follow_pairs(n):
    W = [tuple(int(c) for c in w) for w in oracle.words(n)]
    rng = np.random.default_rng(n)
    for qi, q in enumerate(W):
        js = range(len(W)) if len(W) <= 60 else rng.choice(len(W), 60, replace=False)
        for j in js:
            p0, p1 = W[j], W[(j * 7 + 3) % len(W)]
            F = pair_fail(q, p0, p1, n)
            assert bool(F & 0x8000) == (not oracle.can_follow(q, p0)), (q, p0)
            assert bool(F & 0x80000000) == (not oracle.can_follow(q, p1)), (q, p1)


@pytest.mark.parametrize("n", [4, 5])
def test_xfer_entry_test_against_matrix(n):
    """err = (~(FIN ^ F) | (FIN & D)) & 0x80008000 is zero exactly on A(D_n)'s entries and
    nonzero for a changed label, a dropped arc and an added arc."""
    A = oracle.transition_matrix(n)
    W = [tuple(int(c) for c in w) for w in oracle.words(n)]

    def err(q, p0, p1, x0, x1):
        F = pair_fail(q, p0, p1, n)
        xx = x0 | x1 << 16
        FIN = nz2(~xx & M32)
        lab = masks(p0)[3] | masks(p1)[3] << 16
        D = nz2(xx ^ lab)
        return (~(FIN ^ F) | (FIN & D)) & 0x80008000

    N = len(W)
    for i in range(0, N, max(1, N // 40)):
        for j in range(0, N - 1, 2):
            x0, x1 = int(A[i, j]), int(A[i, j + 1])
            assert err(W[i], W[j], W[j + 1], x0, x1) == 0
            fin = x0 != 0xFFFF
            wrong = [x0 + 1] if fin else [3]
            wrong.append(0xFFFF if fin else masks(W[j])[3])
            for y in wrong:
                assert err(W[i], W[j], W[j + 1], y, x1) & 0x8000, (i, j, x0, y)


def transpose_model(xs):
    out = list(xs)
    for j in (16, 8, 4, 2, 1):
        m = {16: 0x0000FFFF, 8: 0x00FF00FF, 4: 0x0F0F0F0F, 2: 0x33333333, 1: 0x55555555}[j]
        ys = [out[lane ^ j] for lane in range(32)]
        out = [((x & ~m) | ((y >> j) & m)) & M32 if lane & j else ((x & m) | ((y << j) & ~m)) & M32
               for lane, (x, y) in enumerate(zip(out, ys))]
    return out


def test_bit_transpose_stages():
    rng = np.random.default_rng(5)
    for _ in range(50):
        xs = [int(v) for v in rng.integers(0, 2**32, size=32, dtype=np.uint64)]
        t = transpose_model(xs)
        for r in range(32):
            for c in range(32):
                assert (xs[r] >> c) & 1 == (t[c] >> r) & 1


def test_nonzero_byte_flags():
    rng = np.random.default_rng(9)
    vals = [0, 0x80, 0x01, 0x7F000000, 0x00010000, 0x80808080] + \
        [int(v) for v in rng.integers(0, 2**32, size=200, dtype=np.uint64)]
    for w in vals:
        nz = (((w & 0x7F7F7F7F) + 0x7F7F7F7F) | w) & 0x80808080
        f = ((nz >> 7) & 1) | ((nz >> 14) & 2) | ((nz >> 21) & 4) | ((nz >> 28) & 8)
        assert f == sum(1 << b for b in range(4) if (w >> (8 * b)) & 0xFF)
