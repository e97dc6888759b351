"""C-ABI checks that need no GPU: the library loads, exports every declared symbol, the
host-side steps (a1 words / transition matrix, shard ranges, periodicity bookkeeping, read-off)
match the oracle, and argument errors are reported before any device work."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2409_17688_b200 as mp
from paper_2409_17688_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "minplus.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^(?!\s*typedef)\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s*"
                       r"([A-Za-z_][A-Za-z0-9_]*)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_exports_every_declared_symbol():
    decl = declared_functions()
    assert len(decl) >= 20
    L = ctypes.CDLL(_native._build.SO)
    for name in decl:
        assert hasattr(L, name), name
    assert sorted(_native.EXPORTS) == decl


def test_no_cpu_fallback_symbols():
    """The product library must not contain the oracle (no shared code, no CPU path)."""
    L = ctypes.CDLL(_native._build.SO)
    for sym in ("oracle_minplus_ijk", "oracle_minplus_ikj", "oracle_power_until_periodic"):
        assert not hasattr(L, sym)


def test_count_words_table1(oracle_mod):
    for n in range(2, 14):
        assert mp.count_words(n) == oracle_mod.count_words(n)
    with pytest.raises(mp.MinplusError):
        mp.count_words(14)
    with pytest.raises(mp.MinplusError) as e:
        mp.count_words(1)
    assert e.value.status == 1


def test_spmm_width_option():
    """The SpMM CTA width accepts 0 (automatic), +-256, +-512 and +-1024 columns, nothing else."""
    for cols in (256, 512, 1024, -256, -512, -1024, 0):
        mp.set_spmm_width(cols)
    for cols in (-1, 128, 768, 2048, -768):
        with pytest.raises(mp.MinplusError) as e:
            mp.set_spmm_width(cols)
        assert e.value.status == 1


@pytest.mark.parametrize("n", range(2, 11))
def test_transition_matrix_equals_oracle(oracle_mod, n):
    """a1 parity: the bitmask/DFS construction equals the letter-by-letter oracle bit for bit."""
    assert np.array_equal(mp.build_transition_matrix(n), oracle_mod.transition_matrix(n))


def test_transition_matrix_domain_errors():
    for n in (0, 1, 14):
        with pytest.raises(mp.MinplusError) as e:
            mp.build_transition_matrix(n)
        assert e.value.status == 1
    A = np.empty(4, dtype=np.uint16)
    assert _native.lib.build_transition_matrix_into(2, A.ctypes.data, 5) == 1


def test_transition_matrix_n12_structure():
    """n = 12 (the largest case): N = 52929 (Table 1), nnz = 21567085 (re-derived
    by counting), labels <= 12, and no row is all +inf."""
    A = mp.build_transition_matrix(12)
    assert A.shape == (52929, 52929)
    fin = A != 0xFFFF
    assert int(fin.sum()) == 21567085
    assert int(A[fin].max()) <= 12
    assert fin.any(axis=1).all()


def test_shard_ranges_cover():
    for N in (1, 6, 15, 225, 3447, 52929):
        for world in (1, 2, 3, 4, 8):
            spans = [mp.shard_range(N, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == N
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0 and a0 <= a1
            w = spans[0][1] - spans[0][0]
            assert w % 8 == 0 or w == N
    with pytest.raises(mp.MinplusError):
        mp.shard_range(10, 2, 2)


@pytest.mark.parametrize("n", [9, 10, 11, 12, 13])
def test_column_plan_padding(n):
    """Shard quantisation: for every rank of G = 1..8 column shards of the
    symmetric domain of A(D_n), the SpMM column plan pads its shard by less than 64 columns (one
    DPX instruction spans 64), and covers it with at most four CTA widths."""
    N = mp.count_words(n)
    sg = mp.word_reversal(n)
    D = int(np.sum(np.arange(N) <= sg))
    for G in range(1, 9):
        for r in range(G):
            c0, c1 = mp.shard_range(D, G, r)
            p = mp.column_plan(N, c1 - c0)
            assert c1 - c0 <= p["ld"] < max(c1 - c0, 1) + 64, (n, G, r, p)
            assert p["ld"] % 64 == 0 and p["main_cols"] in (256, 512, 1024)
    # a forced width pads to a multiple of it; a negative one keeps the remainder columns
    mp.set_spmm_width(1024)
    try:
        assert mp.column_plan(N, 3328)["ld"] == 4096
    finally:
        mp.set_spmm_width(-1024)
    try:
        p = mp.column_plan(N, 3328)
        assert (p["ld"], p["main_cols"], p["tail_cols"]) == (3328, 1024, 256)
        assert mp.column_plan(N, 960) == {"ld": 960, "main_cols": 1024, "tail_cols": 960}
        assert mp.column_plan(N, 1800) == {"ld": 1856, "main_cols": 1024, "tail_cols": 832}
    finally:
        mp.set_spmm_width(0)


def test_fingerprint_unit_matches_oracle(oracle_mod):
    for N in (1, 5, 37, 200):
        assert mp.fingerprint_unit(N) == oracle_mod.fingerprint(np.ones((N, N), dtype=np.uint16))


def _stats(oracle_mod, X):
    N = X.shape[0]
    fin = np.flatnonzero(X.ravel() != 0xFFFF)
    ref = (int(fin[0]) << 16) | int(X.ravel()[fin[0]]) if len(fin) else 2**63 - 1
    fp = oracle_mod.fingerprint(X)
    return mp.PowerStats(fp - 2**64 if fp >= 2**63 else fp, int((X == 0xFFFF).sum()),
                         int(np.diag(X).min()), ref)


def test_repeat_candidate_logic(oracle_mod):
    """The prefilter passes every true repeat (linearity of H) and rejects differing powers."""
    A = oracle_mod.transition_matrix(4)
    r = oracle_mod.power_until_periodic(A)
    P = {1: A}
    for k in range(2, r.k_last + 1):
        P[k] = oracle_mod.minplus(A, P[k - 1])
    S = mp.fingerprint_unit(A.shape[0])
    st = {k: _stats(oracle_mod, P[k]) for k in P}
    assert mp.repeat_candidate(st[r.k_last], st[r.mu], S) == r.offset
    hits = [(k, j) for k in P for j in range(1, k) if mp.repeat_candidate(st[k], st[j], S) is not None
            and oracle_mod.constant_difference(P[k], P[j]) is not None]
    assert hits == [(r.k_last, r.mu)]
    # all-inf pair: candidate with offset 0
    Z = np.full((3, 3), 0xFFFF, dtype=np.uint16)
    assert mp.repeat_candidate(_stats(oracle_mod, Z), _stats(oracle_mod, Z), 1) == 0


def test_readoff_matches_oracle(oracle_mod):
    """a6 on a result built from oracle values equals the oracle's read-off for m to 500."""
    for n in (3, 5, 7):
        o = oracle_mod.power_until_periodic(oracle_mod.transition_matrix(n))
        r = _native._PeriodicResult()
        r.mu, r.lambda_, r.offset, r.k_last, r.dense_from = o.mu, o.lam, o.offset, o.k_last, o.dense_from
        for k, v in enumerate(o.diag_min):
            r.diag_min[k] = v
        res = _native._result(r)
        for m in range(3, 500):
            assert res.gamma2(m) == o.gamma2(m)
        with pytest.raises(mp.MinplusError):
            res.gamma2(2)


@pytest.mark.parametrize("n", range(2, 10))
def test_word_reversal_is_a_symmetry(n):
    """sigma = word reversal is an involution and A(D_n)[sigma i][sigma j] = A(D_n)[i][j]
    (the reflection of the path)."""
    s = mp.word_reversal(n)
    A = mp.build_transition_matrix(n)
    assert np.array_equal(s[s], np.arange(len(s)))
    assert np.array_equal(A[np.ix_(s, s)], A)


def test_symmetry_hint_domain_errors():
    assert _native.lib.mp_set_symmetry(np.array([1, 2, 0], dtype=np.int32).ctypes.data, 3) == 1  # a 3-cycle
    assert _native.lib.mp_set_symmetry(np.array([0, 5], dtype=np.int32).ctypes.data, 2) == 1     # out of range
    assert _native.lib.mp_set_symmetry(None, 0) == 0
    with pytest.raises(mp.MinplusError):
        _native._check(_native.lib.mp_word_reversal(4, np.zeros(3, dtype=np.int32).ctypes.data, 3))


def test_next4_argument_errors():
    lib = _native.lib
    a = np.zeros((4, 4), dtype=np.uint16)
    assert lib.minplus_closure(None, 4, a.ctypes.data, None) == 1
    assert lib.minplus_closure(a.ctypes.data, 0, a.ctypes.data, None) == 1
    assert lib.minplus_closure(a.ctypes.data, 4, a.ctypes.data, None) == 1  # D overlaps W
    assert lib.minplus_mul_strided_batched_device(None, 4, 16, None, 4, 16, None, 4, 16, 4, 4, 4, 2, None) == 1
    assert lib.minplus_mul_strided_batched_device(a.ctypes.data, 4, 16, a.ctypes.data, 4, 16, 8, 4, 16,
                                                  4, 4, 4, 0, None) == 1  # batch <= 0


def test_argument_errors_before_device():
    with pytest.raises(mp.MinplusError) as e:
        mp.minplus_mul(np.zeros((2, 3)), np.zeros((2, 3)))
    assert e.value.status == 1
    assert _native.lib.minplus_mul(None, None, None, 1, 1, 1) == 1
    a = np.zeros((4, 4), dtype=np.uint16)
    assert _native.lib.minplus_mul(a.ctypes.data, a.ctypes.data, a.ctypes.data, 4, 4, 4) == 1  # aliasing
    g = ctypes.c_int64()
    assert _native.lib.gamma2_cylinder(5, 2, ctypes.byref(g)) == 1
    assert _native.lib.gamma2_cylinder(14, 5, ctypes.byref(g)) == 1
    r = _native._PeriodicResult()
    assert _native.lib.minplus_power_until_periodic(a.ctypes.data, 4, 1, ctypes.byref(r)) == 1
    assert _native.lib.minplus_power_until_periodic(a.ctypes.data, 4, 257, ctypes.byref(r)) == 1
    assert _native.lib.mp_set_grouping(2) == 1 and _native.lib.mp_set_options(3, 0) == 1
    assert _native.lib.mp_set_grouping(-1) == 0


def test_no_gpu_reports_cuda_error():
    """Without an sm_100 device the computing calls fail loudly (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(mp.MinplusError) as e:
        mp.minplus_mul(np.zeros((2, 2)), np.zeros((2, 2)))
    assert e.value.status == 5


def test_gamma2_formula_reproduces_table7(oracle_mod):
    """NEXT-2: the closed formula built from the run (alpha from the boundary values,
    exceptions below n0) reproduces Table 7 and its exception rows (G14, G15)."""
    from conftest import golden
    rows = golden("table7_alpha.txt")
    exc = {(int(x[1]), int(x[2])): int(x[3]) for x in rows if x[0] == "exc"}
    for x in rows:
        if x[0] == "exc":
            continue
        n, a = int(x[0]), int(x[1])
        if n > 9:
            continue
        ks = set() if x[2] == "-" else set(map(int, x[2].split(",")))
        mmin = int(x[3])
        o = oracle_mod.power_until_periodic(oracle_mod.transition_matrix(n))
        r = _native._PeriodicResult()
        r.mu, r.lambda_, r.offset, r.k_last, r.dense_from = o.mu, o.lam, o.offset, o.k_last, o.dense_from
        for k, v in enumerate(o.diag_min):
            r.diag_min[k] = v
        f = _native._result(r).formula()
        assert f["a"] == a
        t4 = {int(x[0]): int(x[1]) for x in golden("table4_recurrence.txt")}
        assert f["r0_k50"] == t4[n]  # Table 4's r0 (Algorithm 3 with K = 50)
        assert {k for k in range(a) if f["alpha"][k] == 1} == ks, n
        assert all(v in (0, 1) for v in f["alpha"])
        expect_exc = {m: g for (nn, m), g in exc.items() if nn == n}
        if mmin:  # n = 7: alpha = 1 only from m = 19 on (G14) -> residues 1,2,4,5 below are exceptions
            expect_exc.update({m: -(-o.offset * m // a) for m in range(3, mmin) if m % a in ks})
        assert f["exceptions"] == expect_exc, (n, f["exceptions"], expect_exc)
