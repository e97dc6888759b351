"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU needed).

Each test names the passage it pins (P:L = PAPER.md line, S:L = SPEC.md line).  The oracle
must never be checked against itself: every expected value here is a paper number, a hand
example, a closed form, an independent library routine (scipy), a brute-force search on the
graph, or an algebraic invariant.
"""
import math

import numpy as np
import pytest

import synth
from conftest import golden

INF = 0xFFFF


def word(s):
    return [int(ch) for ch in s]


# ------------------------------------------------------------------------------- c1 words
def test_table1_word_counts(oracle_mod):
    """Table 1: |C_n| for n = 2..13, and the printed memory sizes (G18)."""
    units = {"KB": 1024.0, "MB": 1024.0 ** 2, "GB": 1024.0 ** 3}
    for n, rows, mem in golden("table1_words.txt"):
        n, rows = int(n), int(rows)
        assert oracle_mod.count_words(n) == rows, n
        if n == 7:  # G22: printed 0.69 MB vs 2*558^2 B = 0.59 MiB
            continue
        val, unit = float(mem[:-2]), mem[-2:]
        assert round(2 * rows * rows / units[unit], 2) == pytest.approx(val, abs=0.011), n


def test_words_m2_and_order(oracle_mod):
    """SPEC's m=2 list and lexicographic order 0<1<2 (G5)."""
    spec = [r for r in golden("spec_examples.txt") if r[0] == "words2"][0][1:]
    got = ["".join(map(str, w)) for w in oracle_mod.words(2)]
    assert got == spec
    for n in (3, 5, 7):
        W = oracle_mod.words(n)
        keys = [tuple(w) for w in W]
        assert keys == sorted(keys) and len(set(keys)) == len(keys)


def test_forbidden_patterns_by_hand(oracle_mod):
    """P:136-139 and the S:51-54 examples."""
    assert oracle_mod.is_correct_word(word("00"))
    assert not oracle_mod.is_correct_word(word("11"))   # 11 at the beginning
    assert not oracle_mod.is_correct_word(word("21"))   # 21 at the end
    assert not oracle_mod.is_correct_word(word("020"))  # anywhere
    for bad in ("0200", "01110", "02110", "01120", "02120", "120", "011"):
        assert not oracle_mod.is_correct_word(word(bad)), bad
    for good in ("0000", "2002", "0110", "10", "0210"):
        assert oracle_mod.is_correct_word(word(good)), good
    with pytest.raises(ValueError):
        oracle_mod.is_correct_word([0, 3])


def test_word_reversal_symmetry(oracle_mod):
    """The forbidden sets mirror (020, 111, 212 palindromes; 211 <-> 112; start 11,12 <->
    end 11,21), so C_n is closed under reversal."""
    for n in range(2, 9):
        S = {tuple(w) for w in oracle_mod.words(n)}
        assert {w[::-1] for w in S} == S


# ------------------------------------------------------------------------ c2/c3 matrix
def test_can_follow_examples(oracle_mod):
    """S:72-75."""
    for _, q, p, exp in [r for r in golden("spec_examples.txt") if r[0] == "cf"]:
        assert oracle_mod.can_follow(word(q), word(p)) == bool(int(exp)), (q, p)


def test_matrix_m2_entries(oracle_mod):
    """(22,00)=2, (22,01)=inf, (00,22)=0."""
    A = oracle_mod.transition_matrix(2)
    idx = {"".join(map(str, w)): i for i, w in enumerate(oracle_mod.words(2))}
    for _, q, p, v in [r for r in golden("spec_examples.txt") if r[0] == "a2"]:
        assert A[idx[q], idx[p]] == int(v)


def test_matrix_label_is_zero_count(oracle_mod):
    """every finite entry equals the number of zeros of the column word; the diagonal
    of A(D_n) is finite exactly for words that can follow themselves."""
    for n in (3, 4, 6):
        W = oracle_mod.words(n)
        A = oracle_mod.transition_matrix(n)
        zeros = (W == 0).sum(axis=1)
        fin = A != INF
        assert np.all(A[fin] == np.broadcast_to(zeros[None, :], A.shape)[fin])


def test_closed_walk_is_two_dominating_set(oracle_mod):
    """Theorem 2's correspondence checked on the graph: every closed walk of
    length m in D_n that realises diag_min is a 2-dominating set of that size.  Brute force
    over all closed walks for tiny (n, m), reading the vertex set off the 0-letters."""
    for n, m in ((2, 3), (3, 3), (3, 4), (4, 3)):
        W = oracle_mod.words(n)
        A = oracle_mod.transition_matrix(n)
        N = len(W)
        best = None

        def dominated(cols):
            S = {(i, j) for j, c in enumerate(cols) for i in range(n) if c[i] == 0}
            for i in range(n):
                for j in range(m):
                    if (i, j) in S:
                        continue
                    nb = [(i - 1, j), (i + 1, j), (i, (j + 1) % m), (i, (j - 1) % m)]
                    if sum((a, b) in S for a, b in nb if 0 <= a < n) < 2:
                        return None
            return len(S)

        def rec(path):
            nonlocal best
            if len(path) == m:
                if A[path[-1], path[0]] != INF:
                    size = dominated([W[k] for k in path])
                    assert size is not None, path
                    label = sum(int(A[path[t], path[(t + 1) % m]]) for t in range(m))
                    assert label == size
                    best = size if best is None else min(best, size)
                return
            for nxt in range(N):
                if A[path[-1], nxt] != INF:
                    rec(path + [nxt])

        for s in range(N):
            rec([s])
        assert best == oracle_mod.gamma2_bruteforce(n, m)


# ----------------------------------------------------------------------------- c4 product
def test_product_hand_example(oracle_mod):
    """[[0,1],[inf,2]] x [[3,inf],[0,5]] = [[1,6],[2,7]]."""
    _, a, b, c = [r for r in golden("spec_examples.txt") if r[0] == "mul"][0]
    A = np.array([int(x) for x in a.split(",")], dtype=np.uint16).reshape(2, 2)
    B = np.array([int(x) for x in b.split(",")], dtype=np.uint16).reshape(2, 2)
    C = np.array([int(x) for x in c.split(",")], dtype=np.uint16).reshape(2, 2)
    for literal in (True, False):
        assert np.array_equal(oracle_mod.minplus(A, B, literal), C)


def test_product_identity_and_inf_row(oracle_mod):
    """S:155 (I x A = A with I = 0 on the diagonal, inf elsewhere) and S:157 (an inf row of
    A gives an inf row of A x B)."""
    X = synth.tropical_matrix(37, 37, 0, 600, 0.3, salt=1)
    I = np.full((37, 37), INF, dtype=np.uint16)
    np.fill_diagonal(I, 0)
    assert np.array_equal(oracle_mod.minplus(I, X), X)
    assert np.array_equal(oracle_mod.minplus(X, I), X)
    A = synth.tropical_matrix(20, 37, 0, 12, 0.2, salt=2)
    A[5, :] = INF
    C = oracle_mod.minplus(A, X)
    assert np.all(C[5] == INF)


def test_product_matches_scipy_shortest_paths(oracle_mod):
    """Library pin: for a zero-diagonal weighted adjacency W, W^(2^t) with 2^t >= N-1 is the
    all-pairs shortest-path matrix, which scipy's Dijkstra computes independently (inf for
    unreachable pairs).  Zero-weight edges are encoded as 1e-12 for the csr input."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import shortest_path
    N = 96
    g = synth.rng(synth.SEED, 7)
    W = np.full((N, N), INF, dtype=np.uint16)
    mask = g.random((N, N)) < 0.04
    W[mask] = g.integers(0, 40, size=int(mask.sum()))
    np.fill_diagonal(W, 0)
    dense = np.where(W == INF, 0.0, np.where(W == 0, 1e-12, W.astype(float)))
    np.fill_diagonal(dense, 0.0)
    D = shortest_path(csr_matrix(dense), method="D")
    X = W.copy()
    for _ in range(7):  # 2^7 = 128 >= N - 1
        X = oracle_mod.minplus(X, X)
    expect = np.where(np.isinf(D), INF, np.rint(D)).astype(np.uint16)
    assert (X == INF).sum() > 100  # unreachable pairs exist
    assert np.array_equal(X, expect)


def test_product_literal_equals_skip_inf(oracle_mod):
    """The i-j-k literal loop and the i-k-j skip-inf loop implement one definition."""
    for (M, K, N, p) in ((1, 1, 1, 0.0), (17, 33, 9, 0.5), (64, 129, 31, 0.99), (8, 5, 8, 1.0)):
        A = synth.tropical_matrix(M, K, 0, 30, p, salt=3)
        B = synth.tropical_matrix(K, N, 0, 600, p / 2, salt=4)
        assert np.array_equal(oracle_mod.minplus(A, B, True), oracle_mod.minplus(A, B, False))
    A, B = synth.saturation_pair(40, 3, 50)
    assert np.array_equal(oracle_mod.minplus(A, B, True), oracle_mod.minplus(A, B, False))


def test_product_saturation_boundary(oracle_mod):
    """G6: 0x3FFF+0x3FFF = 0x7FFE stays finite; 0x3FFF+0x4000 = 0x7FFF becomes inf;
    0x7FFE+0 stays finite; a saturated term never beats a finite one."""
    A = np.array([[0x3FFF, INF], [0x3FFF, INF], [0x7FFE, INF], [0x4000, 5]], dtype=np.uint16)
    B = np.array([[0x3FFF, 0x4000, 0], [7, 7, 7]], dtype=np.uint16)
    C = oracle_mod.minplus(A, B, literal=True)
    assert C[0, 0] == 0x7FFE and C[0, 1] == INF and C[2, 2] == 0x7FFE
    assert C[3, 0] == 12 and C[3, 1] == 12 and C[3, 2] == 12 and C[1, 1] == INF


def test_product_associativity(oracle_mod):
    """(A x B) x C = A x (B x C) on random triples."""
    for s in range(3):
        A = synth.tropical_matrix(13, 16, 0, 100, 0.3, salt=10 + s)
        B = synth.tropical_matrix(16, 11, 0, 100, 0.3, salt=20 + s)
        C = synth.tropical_matrix(11, 14, 0, 100, 0.3, salt=30 + s)
        assert np.array_equal(oracle_mod.minplus(oracle_mod.minplus(A, B), C),
                              oracle_mod.minplus(A, oracle_mod.minplus(B, C)))


def test_product_walks_brute_force(oracle_mod):
    """Theorem 1 (Carre): (A^k)_ij = min label over length-k walks i -> j, by
    explicit walk enumeration on a tiny digraph."""
    import itertools
    A = synth.tropical_matrix(5, 5, 0, 9, 0.4, salt=40)
    X = A.copy()
    for k in range(2, 5):
        X = oracle_mod.minplus(A, X)
        for i in range(5):
            for j in range(5):
                best = INF
                for mid in itertools.product(range(5), repeat=k - 1):
                    path = (i,) + mid + (j,)
                    w = [int(A[path[t], path[t + 1]]) for t in range(k)]
                    if INF not in w:
                        best = min(best, sum(w))
                assert X[i, j] == best


# -------------------------------------------------------------------------- fingerprint
def test_splitmix64_vectors(oracle_mod):
    """Published splitmix64 outputs: state 0 -> 0xE220A8397B1DCDAF; seeded 1234567 the first
    two outputs are 6457827717110365317 and 3203168211198807973 (the generator advances its
    state by 0x9E3779B97F4A7C15 per output, so output 2 is h(1234567 + golden))."""
    assert oracle_mod.splitmix64(0) == 0xE220A8397B1DCDAF
    assert oracle_mod.splitmix64(1234567) == 6457827717110365317
    assert oracle_mod.splitmix64((1234567 + 0x9E3779B97F4A7C15) % 2**64) == 3203168211198807973


def test_fingerprint_linear_and_additive(oracle_mod):
    """H(c (x) X) = H(X) + c*S for inf-free X (S = H(all-ones)); H is additive over column
    blocks; a single entry (i, j) gives s(2i)*s(2j+1)*x."""
    X = synth.power_like(23, 29, salt=50)
    S = oracle_mod.fingerprint(np.ones_like(X))
    for c in (1, 3, 14):
        assert oracle_mod.fingerprint(X + c) == (oracle_mod.fingerprint(X) + c * S) % 2**64
    parts = [oracle_mod.fingerprint_cols(X, 0, 7), oracle_mod.fingerprint_cols(X, 7, 20),
             oracle_mod.fingerprint_cols(X, 20, 29)]
    assert sum(parts) % 2**64 == oracle_mod.fingerprint(X)
    Z = np.zeros_like(X)
    Z[4, 5] = 9
    assert oracle_mod.fingerprint(Z) == (9 * oracle_mod.splitmix64(2 * 4) * oracle_mod.splitmix64(2 * 5 + 1)) % 2**64
    Z[4, 5] = 0
    Z[0, 0] = 1  # h(0, 0) = s(0) * s(1)
    assert oracle_mod.fingerprint(Z) == (0xE220A8397B1DCDAF * oracle_mod.splitmix64(1)) % 2**64


# -------------------------------------------------------------------- c5/c6 periodicity
@pytest.mark.parametrize("n", range(2, 10))
def test_table5_recurrence(oracle_mod, n):
    """Table 5: (n0, a, b) = (mu, lambda, b); powers dense from k = 3;
    entries of A^k bounded by n*k."""
    row = {int(r[0]): tuple(map(int, r[1:])) for r in golden("table5_recurrence.txt")}[n]
    r = oracle_mod.power_until_periodic(oracle_mod.transition_matrix(n))
    assert r.rc == 0
    assert (r.mu, r.lam, r.offset) == row
    assert r.k_last == r.mu + r.lam
    assert r.dense_from == 3


@pytest.mark.slow
@pytest.mark.parametrize("n", [10])
def test_table5_recurrence_n10(oracle_mod, n):
    test_table5_recurrence(oracle_mod, n)


@pytest.mark.parametrize("n", range(2, 9))
def test_algorithms_3_and_4_verbatim(oracle_mod, n):
    """NEXT-2: the paper's own Algorithm 3 with K = 50 reproduces Table 4 (r0, a, b)
     and Algorithm 4 from there reproduces Table 5's n0, which equals
    the forward first-repeat mu ("Why first-repeat detection equals Algs 3/4")."""
    t4 = {int(r[0]): tuple(map(int, r[1:])) for r in golden("table4_recurrence.txt")}[n]
    t5 = {int(r[0]): tuple(map(int, r[1:])) for r in golden("table5_recurrence.txt")}[n]
    P = oracle_mod.powers(oracle_mod.transition_matrix(n), 50)
    r0, a, b = oracle_mod.algorithm3(P, 50)
    assert (r0, a, b) == t4
    assert oracle_mod.algorithm4(P, r0, a, b) == t5[0]
    r = oracle_mod.power_until_periodic(P[1])
    assert (r.mu, r.lam, r.offset) == (t5[0], a, b)


def test_periodicity_invariants(oracle_mod):
    """Lemma 1 on the oracle's own powers: A^{k+lambda} = b (x) A^k for several
    k >= mu beyond the first repeat; A^{i+j} = A^i x A^j."""
    A = oracle_mod.transition_matrix(4)
    r = oracle_mod.power_until_periodic(A)
    P = {1: A}
    for k in range(2, r.k_last + 2 * r.lam + 1):
        P[k] = oracle_mod.minplus(A, P[k - 1])
    for k in range(r.mu, r.k_last + r.lam + 1):
        assert oracle_mod.constant_difference(P[k + r.lam], P[k]) == r.offset
    assert oracle_mod.constant_difference(P[r.mu + r.lam - 1], P[r.mu - 1]) is None
    assert np.array_equal(oracle_mod.minplus(P[3], P[4]), P[7])
    assert int(P[r.k_last].max()) <= 4 * r.k_last


def test_periodicity_degenerate(oracle_mod):
    """Degenerate cases: all-inf A repeats at once with offset 0; a zero matrix is
    idempotent; a 1x1 matrix [[c]] has A^2 = c (x) A."""
    r = oracle_mod.power_until_periodic(np.full((5, 5), INF, dtype=np.uint16))
    assert (r.rc, r.mu, r.lam, r.offset, r.dense_from) == (0, 1, 1, 0, 0)
    r = oracle_mod.power_until_periodic(np.zeros((4, 4), dtype=np.uint16))
    assert (r.mu, r.lam, r.offset, r.dense_from) == (1, 1, 0, 1)
    r = oracle_mod.power_until_periodic(np.array([[7]], dtype=np.uint16))
    assert (r.mu, r.lam, r.offset, r.diag_min[2]) == (1, 1, 7, 14)
    # a permutation cycle of length 3 with weight 1 per arc: A^4 = 1 (x) A^... no, period 3
    P = np.full((3, 3), INF, dtype=np.uint16)
    P[0, 1] = P[1, 2] = P[2, 0] = 1
    r = oracle_mod.power_until_periodic(P)
    assert (r.mu, r.lam, r.offset) == (1, 3, 3)


def test_power_rows_match_full_powers(oracle_mod):
    """The row-sampled oracle (vector-matrix products) equals rows of the full powers."""
    A = oracle_mod.transition_matrix(6)
    X = A.copy()
    rows = {r: oracle_mod.power_rows(A, r, 8) for r in (0, 17, 224)}
    for k in range(1, 9):
        if k > 1:
            X = oracle_mod.minplus(A, X)
        for r, R in rows.items():
            assert np.array_equal(R[k - 1], X[r])


# ------------------------------------------------------------------------------ c7 gamma_2
def test_gamma2_bruteforce_matches_diagonal(oracle_mod):
    """Theorem 2: the diagonal read-off equals the exhaustive minimum over
    vertex subsets for every n*m <= 24."""
    for n in range(2, 9):
        r = oracle_mod.power_until_periodic(oracle_mod.transition_matrix(n))
        for m in range(3, 24 // n + 1):
            assert r.gamma2(m) == oracle_mod.gamma2_bruteforce(n, m), (n, m)


def test_example1(oracle_mod):
    """Example 1: a 2-dominating set of P_4 x C_5 with 10 vertices; the
    minimum is therefore <= 10 and the brute force says it is exactly 10."""
    g = oracle_mod.gamma2(4, 5)
    assert g <= 10
    assert g == oracle_mod.gamma2_bruteforce(4, 5) == 10


def test_gamma2_column_dp(oracle_mod):
    """An independent dynamic program over column subsets equals the read-off, including
    read-offs far beyond k_last (Theorem 3)."""
    for n, mmax in ((2, 30), (3, 30), (4, 30), (5, 10)):
        r = oracle_mod.power_until_periodic(oracle_mod.transition_matrix(n))
        for m in range(3, mmax + 1):
            assert r.gamma2(m) == oracle_mod.gamma2_column_dp(n, m), (n, m)


def test_gamma2_path_dp(oracle_mod):
    """A third graph oracle, DP along the path over row subsets of the cycle: equals brute
    force (n*m <= 24), the column DP, and the transfer-matrix read-off for n <= 9, m <= 8."""
    for n in range(1, 9):
        for m in range(3, min(8, 24 // n) + 1):
            assert oracle_mod.gamma2_path_dp(n, m) == oracle_mod.gamma2_bruteforce(n, m), (n, m)
    for n in (2, 3, 4, 5):
        for m in range(3, 9):
            assert oracle_mod.gamma2_path_dp(n, m) == oracle_mod.gamma2_column_dp(n, m), (n, m)
    for n in range(6, 10):
        r = oracle_mod.power_until_periodic(oracle_mod.transition_matrix(n))
        for m in range(3, 9):
            assert oracle_mod.gamma2_path_dp(n, m) == r.gamma2(m), (n, m)


def test_gamma2_closed_forms(oracle_mod):
    """P_2: gamma_2 = m; P_3: ceil(4m/3) (from Table 5 a=6, b=8 and Table 7 all alpha=0);
    C_5 formula of [Garzon2022] quoted at P:504; the n >= 8, 3 | m formula (n+2)m/3 proven
    for 8 <= n <= 12."""
    r2 = oracle_mod.power_until_periodic(oracle_mod.transition_matrix(2))
    r3 = oracle_mod.power_until_periodic(oracle_mod.transition_matrix(3))
    for m in range(3, 200):
        assert r2.gamma2(m) == m
        assert r3.gamma2(m) == -(-4 * m // 3)
    for n in range(2, 10):
        r = oracle_mod.power_until_periodic(oracle_mod.transition_matrix(n))
        assert r.gamma2(5) == (2 * n + 2 if (n > 2 and n % 2 == 0) else 2 * n + 1), n
        if n >= 8:
            for m in range(3, 300, 3):
                assert r.gamma2(m) == (n + 2) * m // 3


def test_gamma2_table7_closed_formula(oracle_mod):
    """P:496-502 + Table 7: gamma_2 = ceil(b m / a) + alpha_k, k = m mod a,
    with the exception rows (G14, G15), for every cycle length 3 <= m <= 120."""
    t5 = {int(r[0]): tuple(map(int, r[1:])) for r in golden("table5_recurrence.txt")}
    rows = golden("table7_alpha.txt")
    alpha = {int(r[0]): (int(r[1]), set() if r[2] == "-" else set(map(int, r[2].split(","))),
                         int(r[3])) for r in rows if r[0] != "exc"}
    exc = {(int(r[1]), int(r[2])): int(r[3]) for r in rows if r[0] == "exc"}
    for n in range(2, 10):
        a, ks, mmin = alpha[n]
        _, a5, b = t5[n]
        assert a == a5
        r = oracle_mod.power_until_periodic(oracle_mod.transition_matrix(n))
        for m in range(3, 121):
            expect = exc.get((n, m))
            if expect is None:
                expect = -(-b * m // a) + (1 if (m % a in ks and m >= mmin) else 0)
            assert r.gamma2(m) == expect, (n, m)
