"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle, bit for bit.

Integer results are compared exactly (the north star: "bit-exact on every matrix entry,
period, offset and gamma_2 value").  Sizes span several 128 x 256 x 32 tiles and ragged
tails; the full-size cases (n = 11, 12) are checked on sampled rows of every power, which the
oracle computes by vector-matrix products, plus the paper's tables for the summaries.
"""
import numpy as np
import pytest

import synth
from conftest import golden

pytestmark = pytest.mark.gpu

INF = 0xFFFF


@pytest.fixture(scope="module")
def mp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)
    import paper_2409_17688_b200 as m
    m.set_options("auto", device_budget_bytes=0)
    return m


def use_kernel(mp, kernel):
    """kernel: a sparsity option, or "spmm-greedy" = SpMM with greedily grouped rows."""
    mp.set_options("spmm" if kernel == "spmm-greedy" else kernel)
    mp.set_grouping("greedy" if kernel == "spmm-greedy" else "consecutive" if kernel == "spmm" else "auto")


def reset_kernel(mp):
    mp.set_options("auto")
    mp.set_grouping("auto")


# ----------------------------------------------------------------------------- products
SHAPES = [(1, 1, 1), (1, 300, 257), (300, 1, 5), (129, 33, 1), (127, 257, 1031), (128, 32, 256),
          (129, 97, 257), (300, 517, 301), (1031, 513, 600), (4097, 31, 70), (40, 4097, 300)]


@pytest.mark.parametrize("M,K,N", SHAPES)
@pytest.mark.parametrize("p_inf", [0.0, 0.5, 0.99])
def test_minplus_mul_random(mp, oracle_mod, M, K, N, p_inf):
    A = synth.transfer_like(M, K, p_inf, salt=M + 7 * K)
    B = synth.tropical_matrix(K, N, 0, 600, p_inf / 3, salt=N + 11 * K)
    assert np.array_equal(mp.minplus_mul(A, B), oracle_mod.minplus(A, B))


def test_minplus_mul_all_inf_rows_cols(mp, oracle_mod):
    A = synth.transfer_like(200, 300, 0.3, salt=5)
    B = synth.power_like(300, 260, salt=6)
    A[17, :] = INF
    B[:, 5] = INF
    A[:, 100:140] = INF
    C = mp.minplus_mul(A, B)
    assert np.array_equal(C, oracle_mod.minplus(A, B))
    assert np.all(C[17] == INF) and np.all(C[:, 5] == INF)
    Z = np.full((50, 60), INF, dtype=np.uint16)
    assert np.all(mp.minplus_mul(Z, synth.power_like(60, 70)) == INF)


@pytest.mark.parametrize("K", [1, 2, 3, 40])
def test_minplus_mul_saturation(mp, oracle_mod, K):
    """G6: finite sums >= 0x7FFF become +inf; boundary pairs exact."""
    A, B = synth.saturation_pair(150, K, 270, salt=K)
    C = mp.minplus_mul(A, B)
    assert np.array_equal(C, oracle_mod.minplus(A, B))
    assert (C == INF).any()
    A = np.array([[0x3FFF], [0x3FFF], [0x7FFE], [0]], dtype=np.uint16)
    B = np.array([[0x3FFF, 0x4000, 0, 0x7FFE]], dtype=np.uint16)
    C = mp.minplus_mul(A, B)
    assert C[0, 0] == 0x7FFE and C[1, 1] == INF and C[2, 2] == 0x7FFE and C[3, 3] == 0x7FFE
    assert C[2, 3] == INF


def test_minplus_mul_range_error(mp):
    A = np.zeros((4, 4), dtype=np.uint16)
    A[1, 2] = 0x8000
    with pytest.raises(mp.MinplusError) as e:
        mp.minplus_mul(A, A.copy())
    assert e.value.status == 2


def test_minplus_mul_device_strided(mp, oracle_mod):
    """Device-pointer entry point with ld > cols (torch tensors, int16 storage)."""
    import torch
    A = synth.transfer_like(300, 200, 0.5, salt=9)
    B = synth.power_like(200, 333, salt=10)
    dA = torch.from_numpy(A.view(np.int16)).cuda()
    big = torch.full((200, 400), -1, dtype=torch.int16, device="cuda")
    big[:, :333] = torch.from_numpy(B.view(np.int16)).cuda()
    dB = big[:, :333]
    dC = torch.zeros((300, 512), dtype=torch.int16, device="cuda")[:, :333]
    mp.minplus_mul_device(dA, dB, dC)
    torch.cuda.synchronize()
    got = dC.cpu().numpy().view(np.uint16)
    assert np.array_equal(got, oracle_mod.minplus(A, B))


# ----------------------------------------------------------------- NEXT-4: batched, closure
def test_minplus_mul_batched(mp, oracle_mod):
    """Strided batch: every C_b equals the oracle's product of its own A_b, B_b."""
    import torch
    nb, M, K, N = 3, 130, 70, 300
    As = [synth.transfer_like(M, K, 0.5, salt=900 + b) for b in range(nb)]
    Bs = [synth.power_like(K, N, salt=910 + b) for b in range(nb)]
    dA = torch.from_numpy(np.stack(As).view(np.int16)).cuda()
    dB = torch.from_numpy(np.stack(Bs).view(np.int16)).cuda()
    dC = mp.minplus_mul_batched_device(dA, dB)
    torch.cuda.synchronize()
    got = dC.cpu().numpy().view(np.uint16)
    for b in range(nb):
        assert np.array_equal(got[b], oracle_mod.minplus(As[b], Bs[b])), b


@pytest.mark.parametrize("N,density", [(1, 0.5), (2, 0.5), (96, 0.04), (700, 0.01)])
def test_minplus_closure_all_pairs_shortest_paths(mp, oracle_mod, N, density):
    """(I + W)^(2^t) on the GPU equals scipy's Dijkstra all-pairs shortest paths (an
    independent library) and, for small N, the oracle's repeated squaring."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import shortest_path
    g = synth.rng(synth.SEED, 70 + N)
    W = np.full((N, N), INF, dtype=np.uint16)
    mask = g.random((N, N)) < density
    W[mask] = g.integers(0, 40, size=int(mask.sum()))
    D, t = mp.minplus_closure(W)
    assert 2 ** t >= N - 1
    Wz = W.copy()
    np.fill_diagonal(Wz, 0)
    dense = np.where(Wz == INF, 0.0, np.where(Wz == 0, 1e-12, Wz.astype(float)))
    np.fill_diagonal(dense, 0.0)
    ref = shortest_path(csr_matrix(dense), method="D")
    expect = np.where(np.isinf(ref), INF, np.rint(ref)).astype(np.uint16)
    assert np.array_equal(D, expect)
    if N <= 96:
        X = Wz
        for _ in range(t):
            X = oracle_mod.minplus(X, X)
        assert np.array_equal(D, X)


# ------------------------------------------------------------------- power sequences
@pytest.mark.parametrize("kernel", ["tiles", "spmm", "spmm-greedy"])
@pytest.mark.parametrize("n", range(2, 10))
def test_power_until_periodic_transfer(mp, oracle_mod, n, kernel):
    """Every summary of the run equals the oracle's: (mu, lambda, b), k_last, dense_from,
    diag_min[k] and the fingerprint of every power A^k (a whole-matrix check), and Table 5."""
    A = mp.build_transition_matrix(n)
    use_kernel(mp, kernel)
    try:
        g = mp.minplus_power_until_periodic(A)
    finally:
        reset_kernel(mp)
    o = oracle_mod.power_until_periodic(A)
    assert (g.mu, g.lam, g.offset, g.k_last, g.dense_from) == (o.mu, o.lam, o.offset, o.k_last, o.dense_from)
    assert g.diag_min == o.diag_min
    assert g.fingerprint == o.fingerprint
    row = {int(r[0]): tuple(map(int, r[1:])) for r in golden("table5_recurrence.txt")}[n]
    assert (g.mu, g.lam, g.offset) == row


@pytest.mark.parametrize("sparse", ["dense", "tiles", "spmm", "spmm-greedy"])
def test_power_rows_full_matrices(mp, oracle_mod, sparse):
    """Every entry of every power A^1..A^12 for n = 7 (N = 558, 5 x 3 tiles, ragged)."""
    use_kernel(mp, sparse)
    try:
        A = mp.build_transition_matrix(7)
        rows = np.arange(A.shape[0])
        got = mp.minplus_power_rows(A, rows, 12)
        X = A.copy()
        for k in range(1, 13):
            if k > 1:
                X = oracle_mod.minplus(A, X)
            assert np.array_equal(got[k - 1], X), k
    finally:
        reset_kernel(mp)


@pytest.mark.parametrize("width", [256, 512, 1024])
@pytest.mark.parametrize("sym", [False, True])
def test_spmm_width_full_matrices(mp, oracle_mod, width, sym):
    """Every SpMM CTA width (256 / 512 / 1024 columns; the automatic choice: 256 for n <= 9)
    forced on n = 7 (N = 558: one ragged 1024-column block): every entry of A^1..A^10."""
    A = mp.build_transition_matrix(7)
    use_kernel(mp, "spmm-greedy")
    mp.set_spmm_width(width)
    if sym:
        mp.set_symmetry(mp.word_reversal(7))
    try:
        got = mp.minplus_power_rows(A, np.arange(A.shape[0]), 10)
    finally:
        mp.set_symmetry(None)
        mp.set_spmm_width(0)
        reset_kernel(mp)
    X = A.copy()
    for k in range(1, 11):
        if k > 1:
            X = oracle_mod.minplus(A, X)
        assert np.array_equal(got[k - 1], X), k


@pytest.mark.parametrize("width", [256, 512, 1024])
@pytest.mark.parametrize("n", [2, 5, 8, 9])
def test_spmm_width_power_until_periodic(mp, oracle_mod, n, width):
    """Whole runs with each forced SpMM width (symmetric columns, greedy rows) = the oracle."""
    A = mp.build_transition_matrix(n)
    use_kernel(mp, "spmm-greedy")
    mp.set_spmm_width(width)
    mp.set_symmetry(mp.word_reversal(n))
    try:
        g = mp.minplus_power_until_periodic(A)
    finally:
        mp.set_symmetry(None)
        mp.set_spmm_width(0)
        reset_kernel(mp)
    o = oracle_mod.power_until_periodic(A)
    assert (g.mu, g.lam, g.offset, g.k_last, g.dense_from) == (o.mu, o.lam, o.offset, o.k_last, o.dense_from)
    assert g.diag_min == o.diag_min and g.fingerprint == o.fingerprint


@pytest.mark.parametrize("order", ["sorted", "greedy"])
@pytest.mark.parametrize("sym", [False, True])
@pytest.mark.parametrize("n", [4, 6, 7, 8, 9])
def test_row_reuse_transfer_hint(mp, oracle_mod, n, sym, order, monkeypatch):
    """Row-inclusion reuse (SpMM on each row's extra entries, then one fold pass per level of
    the parent DAG) on A(D_n) announced by the transfer hint, greedy grouping forced so the
    grouped SpMM runs at these sizes, with the rows in the extras order (sorted by their first
    extra columns, the default) or in the windowed greedy tiles (MP_GROUP_ORDER=greedy): every
    entry of A^1..A^8 and the whole periodic record equal the oracle's; a matrix that is not
    A(D_n) is refused."""
    if order == "greedy":
        monkeypatch.setenv("MP_GROUP_ORDER", "greedy")
    A = mp.build_transition_matrix(n)
    o = oracle_mod.power_until_periodic(A)
    use_kernel(mp, "spmm-greedy")
    mp.set_transfer_hint(n)
    mp.set_small_path(False)
    if sym:
        mp.set_symmetry(mp.word_reversal(n))
    try:
        got = mp.minplus_power_rows(A, np.arange(A.shape[0]), 8)
        g = mp.minplus_power_until_periodic(A)
        assert mp.last_profile()["row_levels"] > 1
        bad = A.copy()
        i, j = np.argwhere(A != INF)[3]
        bad[i, j] = INF
        with pytest.raises(mp.MinplusError) as e:
            mp.minplus_power_until_periodic(bad)
        assert e.value.name == "MP_ERR_DOMAIN"
    finally:
        mp.set_symmetry(None)
        mp.set_transfer_hint(0)
        mp.set_small_path(True)
        reset_kernel(mp)
    assert (g.mu, g.lam, g.offset, g.k_last, g.dense_from) == (o.mu, o.lam, o.offset, o.k_last, o.dense_from)
    assert g.diag_min == o.diag_min and g.fingerprint == o.fingerprint
    X = A.copy()
    for k in range(1, 9):
        if k > 1:
            X = oracle_mod.minplus(A, X)
        assert np.array_equal(got[k - 1], X), k


def _fold_rows_model(oracle_mod, n):
    """sum over DAG levels >= 1 of (2 x rows + distinct parents of the level): the parents of a
    word are the words with one letter 0 or 1 turned into a 2, the level
    is 0 without parents, else 1 + the parents' maximum"""
    W = [tuple(w) for w in oracle_mod.words(n).tolist()]
    pos = {w: i for i, w in enumerate(W)}
    par = [[pos[w[:b] + (2,) + w[b + 1:]] for b in range(n) if w[b] != 2 and w[:b] + (2,) + w[b + 1:] in pos]
           for w in W]
    level = [0] * len(W)
    for q in sorted(range(len(W)), key=lambda q: -W[q].count(2)):  # parents have one more 2
        level[q] = 1 + max(level[p] for p in par[q]) if par[q] else 0
    total = 0
    for lv in range(1, max(level) + 1):
        rows = [q for q in range(len(W)) if level[q] == lv]
        total += 2 * len(rows) + len({p for q in rows for p in par[q]})
    return total, max(level) + 1


@pytest.mark.parametrize("n", [5, 7, 8])
def test_fold_bytes_profile(mp, oracle_mod, n):
    """The folds' algorithmic bytes the library reports (mp_profile.fold_bytes, bench.py's k_fold
    roofline numerator) equal the count from a host model of the parent DAG x ld x 2 bytes."""
    A = mp.build_transition_matrix(n)
    use_kernel(mp, "spmm-greedy")
    mp.set_transfer_hint(n)
    mp.set_small_path(False)
    try:
        mp.minplus_power_until_periodic(A)
        p = mp.last_profile()
    finally:
        mp.set_transfer_hint(0)
        mp.set_small_path(True)
        reset_kernel(mp)
    rows, levels = _fold_rows_model(oracle_mod, n)
    assert p["row_levels"] == levels
    assert p["fold_bytes"] == rows * p["ld"] * 2


@pytest.mark.parametrize("main", [-1024, -512, -256, 0])
@pytest.mark.parametrize("N", [100, 700, 960, 1500, 1800])
def test_spmm_remainder_columns(mp, oracle_mod, N, main):
    """Column plans with narrower remainder CTA columns (mp_column_plan: 768 / 512 / 256 / 128
    / 64 wide after the main width; e.g. N = 960 at main 1024 -> 768 + 128 + 64): every entry
    of A^1..A^4 of a random sparse matrix through the SpMM kernel equals the oracle's."""
    A = synth.transfer_like(N, N, 0.97, salt=700 + N)
    use_kernel(mp, "spmm-greedy")
    mp.set_spmm_width(main)
    try:
        got = mp.minplus_power_rows(A, np.arange(N), 4)
        plan = mp.column_plan(N, N)
    finally:
        mp.set_spmm_width(0)
        reset_kernel(mp)
    assert N <= plan["ld"] < N + 64
    X = A.copy()
    for k in range(1, 5):
        if k > 1:
            X = oracle_mod.minplus(A, X)
        assert np.array_equal(got[k - 1], X), k


@pytest.mark.parametrize("kernel", ["dense", "tiles", "spmm", "spmm-greedy", "auto"])
@pytest.mark.parametrize("seed", range(5))
def test_power_until_periodic_random(mp, oracle_mod, seed, kernel):
    """Random sparse matrices (the +inf pattern persists for several powers, exercising the
    exact-compare path with +inf entries), with each product kernel; seed 4 spans three
    grouping windows (1100 rows, ragged)."""
    N = [37, 130, 257, 300, 1100][seed]
    A = synth.transfer_like(N, N, [0.9, 0.95, 0.97, 0.5, 0.97][seed], salt=100 + seed)
    use_kernel(mp, kernel)
    try:
        g = mp.minplus_power_until_periodic(A, max_k=64)
    finally:
        reset_kernel(mp)
    o = oracle_mod.power_until_periodic(A, max_k=64)
    assert o.rc == 0
    assert (g.mu, g.lam, g.offset, g.k_last, g.dense_from) == (o.mu, o.lam, o.offset, o.k_last, o.dense_from)
    assert g.diag_min == o.diag_min and g.fingerprint == o.fingerprint


def test_power_until_periodic_degenerate(mp, oracle_mod):
    for A in (np.full((5, 5), INF, dtype=np.uint16), np.zeros((4, 4), dtype=np.uint16),
              np.array([[7]], dtype=np.uint16)):
        g = mp.minplus_power_until_periodic(A)
        o = oracle_mod.power_until_periodic(A)
        assert (g.mu, g.lam, g.offset, g.dense_from) == (o.mu, o.lam, o.offset, o.dense_from)
        assert g.diag_min == o.diag_min and g.fingerprint == o.fingerprint
    P = np.full((300, 300), INF, dtype=np.uint16)
    for i in range(300):
        P[i, (i + 1) % 300] = 1  # a 300-cycle: period 300 > max_k
    with pytest.raises(mp.MinplusError) as e:
        mp.minplus_power_until_periodic(P, max_k=20)
    assert e.value.status == 4
    for kernel in ("dense", "tiles", "spmm", "auto"):  # entries in (0x7FFE, 0xFFFF): MP_ERR_RANGE
        use_kernel(mp, kernel)
        try:
            B = synth.transfer_like(100, 100, 0.5, salt=3)
            B[7, 9] = 0x8000
            with pytest.raises(mp.MinplusError) as e:
                mp.minplus_power_until_periodic(B)
            assert e.value.status == 2
        finally:
            reset_kernel(mp)


def test_ring_eviction_recompute(mp, oracle_mod):
    """A device budget of 17 power slots (the minimum for a 16-power batch) forces the
    recompute path for evicted A^j: n = 7 has lambda = 18, so the partner of the first repeat
    has left the ring."""
    A = mp.build_transition_matrix(7)
    # Np x ld x 2 B; ld = the SpMM column plan's padded width (mp_column_plan)
    slot = (((A.shape[0] + 127) // 128) * 128) * mp.column_plan(A.shape[0], A.shape[0])["ld"] * 2
    mp.set_options("auto", device_budget_bytes=19 * slot)  # 19 - 2 reserved = 17 ring slots
    try:
        g = mp.minplus_power_until_periodic(A)
    finally:
        mp.set_options("auto", device_budget_bytes=0)
    assert (g.mu, g.lam, g.offset) == (23, 18, 53)


def test_resource_error_reports_bytes(mp):
    """A device budget below the power store's minimum (17 slots for a 16-power batch at this
    size) is MP_ERR_RESOURCE, with the slot size and the budget in the message; the
    next run with the default budget works."""
    A = mp.build_transition_matrix(7)
    slot = (((A.shape[0] + 127) // 128) * 128) * mp.column_plan(A.shape[0], A.shape[0])["ld"] * 2
    mp.set_options("auto", device_budget_bytes=8 * slot)
    try:
        with pytest.raises(mp.MinplusError) as e:
            mp.minplus_power_until_periodic(A)
    finally:
        mp.set_options("auto", device_budget_bytes=0)
    assert e.value.name == "MP_ERR_RESOURCE"
    assert str(slot) in str(e.value) and str(8 * slot) in str(e.value)
    assert mp.minplus_power_until_periodic(A).mu == 23


# --------------------------------------------------------------------------- symmetry
def _random_symmetric(N, p_inf, seed):
    """A random matrix with A[sigma i][sigma j] = A[i][j] for a random involution sigma."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(N)
    sigma = np.arange(N, dtype=np.int32)
    npairs = (N - N // 5) // 2                      # a fifth (about) fixed points
    a, b = perm[:npairs], perm[npairs:2 * npairs]
    sigma[a], sigma[b] = b, a
    A = synth.transfer_like(N, N, p_inf, salt=seed)
    S = A[np.ix_(sigma, sigma)]
    keep = np.arange(N)[:, None] <= np.arange(N)[None, :]  # take the upper triangle's orbit rep.
    B = np.where(keep, A, S)
    B = np.where(B[np.ix_(sigma, sigma)] == B, B, np.minimum(B, B[np.ix_(sigma, sigma)]))
    assert (B[np.ix_(sigma, sigma)] == B).all()
    return B.astype(np.uint16), sigma


@pytest.mark.parametrize("kernel", ["tiles", "spmm", "spmm-greedy"])
@pytest.mark.parametrize("n", range(2, 10))
def test_power_until_periodic_symmetry(mp, oracle_mod, n, kernel):
    """With the word-reversal hint the run computes only the columns g <= sigma(g) and must
    still report the oracle's full-matrix summaries and fingerprints."""
    A = mp.build_transition_matrix(n)
    use_kernel(mp, kernel)
    mp.set_symmetry(mp.word_reversal(n))
    try:
        g = mp.minplus_power_until_periodic(A)
    finally:
        mp.set_symmetry(None)
        reset_kernel(mp)
    o = oracle_mod.power_until_periodic(A)
    assert (g.mu, g.lam, g.offset, g.k_last, g.dense_from) == (o.mu, o.lam, o.offset, o.k_last, o.dense_from)
    assert g.diag_min == o.diag_min and g.fingerprint == o.fingerprint


@pytest.mark.parametrize("kernel", ["dense", "tiles", "spmm"])
@pytest.mark.parametrize("seed", range(3))
def test_symmetry_random(mp, oracle_mod, seed, kernel):
    N = [61, 300, 1031][seed]
    A, sigma = _random_symmetric(N, [0.5, 0.9, 0.97][seed], 300 + seed)
    use_kernel(mp, kernel)
    mp.set_symmetry(sigma)
    try:
        g = mp.minplus_power_until_periodic(A, max_k=64)
        rows = np.array([0, 5, N // 2, N - 1])
        got = mp.minplus_power_rows(A, rows, 6)
    finally:
        mp.set_symmetry(None)
        reset_kernel(mp)
    o = oracle_mod.power_until_periodic(A, max_k=64)
    assert o.rc == 0
    assert (g.mu, g.lam, g.offset, g.k_last, g.dense_from) == (o.mu, o.lam, o.offset, o.k_last, o.dense_from)
    assert g.diag_min == o.diag_min and g.fingerprint == o.fingerprint
    for r_i, r in enumerate(rows):
        assert np.array_equal(got[:, r_i, :], oracle_mod.power_rows(A, int(r), 6)), r


def test_symmetry_power_rows_full(mp, oracle_mod):
    """Every entry of every power A^1..A^12 for n = 7 reassembled from the domain columns."""
    A = mp.build_transition_matrix(7)
    mp.set_symmetry(mp.word_reversal(7))
    try:
        got = mp.minplus_power_rows(A, np.arange(A.shape[0]), 12)
    finally:
        mp.set_symmetry(None)
    X = A.copy()
    for k in range(1, 13):
        if k > 1:
            X = oracle_mod.minplus(A, X)
        assert np.array_equal(got[k - 1], X), k


def test_symmetry_hint_verified(mp):
    """A hint that does not hold is rejected (MP_ERR_DOMAIN), as is a non-involution."""
    A = mp.build_transition_matrix(6)
    N = A.shape[0]
    bad = np.arange(N, dtype=np.int32)
    bad[[3, 4]] = [4, 3]
    mp.set_symmetry(bad)
    try:
        with pytest.raises(mp.MinplusError) as e:
            mp.minplus_power_until_periodic(A)
        assert e.value.status == 1
    finally:
        mp.set_symmetry(None)
    with pytest.raises(mp.MinplusError):
        mp.set_symmetry(np.roll(np.arange(N, dtype=np.int32), 1))


# -------------------------------------------------------------------------- gamma_2
def test_gamma2_cylinder_small(mp, oracle_mod):
    """gamma_2 through the public entry point: brute force (n*m <= 24), column DP, and the
    oracle read-off far beyond k_last."""
    for n in range(2, 9):
        for m in range(3, 24 // n + 1):
            assert mp.gamma2_cylinder(n, m) == oracle_mod.gamma2_bruteforce(n, m), (n, m)
    for n in (2, 3, 4):
        for m in range(3, 31):
            assert mp.gamma2_cylinder(n, m) == oracle_mod.gamma2_column_dp(n, m)
    for n in range(2, 9):
        o = oracle_mod.power_until_periodic(oracle_mod.transition_matrix(n))
        for m in list(range(3, 60)) + [1000, 10**6]:
            assert mp.gamma2_cylinder(n, m) == o.gamma2(m), (n, m)


@pytest.mark.parametrize("sym", [False, True])
@pytest.mark.parametrize("n", [10, 11, 12])
def test_large_n_sampled_rows_and_tables(mp, oracle_mod, n, sym):
    """Full-size cases, in the configuration bench.py times (sym: the word-reversal symmetry,
    only the domain columns computed) and on all columns: sampled rows of every power up to
    k_last against the oracle's vector-matrix recurrence; (mu, lambda, b) against Table 5;
    gamma_2 against the paper's closed formula (Table 7 with the exception rows) for every
    m <= 200 and m = 1000."""
    t5 = {int(r[0]): tuple(map(int, r[1:])) for r in golden("table5_recurrence.txt")}
    A = mp.build_transition_matrix(n)
    N = A.shape[0]
    mp.set_symmetry(mp.word_reversal(n) if sym else None)
    try:
        g = mp.minplus_power_until_periodic(A)
        rows = [0, 1, N // 3, N // 2 + 7, N - 1]
        got = mp.minplus_power_rows(A, rows, g.k_last)
    finally:
        mp.set_symmetry(None)
    assert (g.mu, g.lam, g.offset) == t5[n]
    assert g.dense_from == 3
    if sym:  # every full-matrix fingerprint and diagonal minimum equals the all-columns run's
        full = mp.minplus_power_until_periodic(A)
        assert g.fingerprint == full.fingerprint and g.diag_min == full.diag_min
    for r_i, r in enumerate(rows):
        ref = oracle_mod.power_rows(A, r, g.k_last)
        assert np.array_equal(got[:, r_i, :], ref), r
    rows7 = golden("table7_alpha.txt")
    a, ks, mmin = [(int(x[1]), set() if x[2] == "-" else set(map(int, x[2].split(","))), int(x[3]))
                   for x in rows7 if x[0] == str(n)][0]
    exc = {(int(x[1]), int(x[2])): int(x[3]) for x in rows7 if x[0] == "exc"}
    b = t5[n][2]
    for m in list(range(3, 201)) + [1000]:
        expect = exc.get((n, m), -(-b * m // a) + (1 if (m % a in ks and m >= mmin) else 0))
        assert g.gamma2(m) == expect, (n, m)
    assert mp.gamma2_cylinder(n, 1000) == {10: 4001, 11: 4334, 12: 4668}[n]
    f = g.formula()  # NEXT-2: Table 7 row and the exception (G15) from the run itself
    assert f["a"] == a and {k for k in range(a) if f["alpha"][k] == 1} == ks
    assert f["exceptions"] == {m: v for (nn, m), v in exc.items() if nn == n}
    t4 = {int(x[0]): int(x[1]) for x in golden("table4_recurrence.txt")}
    assert f["r0_k50"] == t4[n]  # Table 4


@pytest.mark.parametrize("sym", [True, False])
@pytest.mark.parametrize("kernel", ["spmm", "spmm-greedy", "tiles"])
def test_gamma2_record_words_source(mp, oracle_mod, kernel, sym):
    """The gamma2_cylinder path builds A(D_n) on the device from the word masks (with SpMM no
    AT2 at all): its whole record -- every power's fingerprint included -- equals the oracle's
    run on the oracle's own transition matrix."""
    mp.shutdown()  # drop the cached records
    use_kernel(mp, kernel)
    mp.set_word_symmetry(sym)
    try:
        for n in range(2, 10):
            g = mp.gamma2_record(n)
            o = oracle_mod.power_until_periodic(oracle_mod.transition_matrix(n))
            assert (g.mu, g.lam, g.offset, g.k_last, g.dense_from) == (o.mu, o.lam, o.offset, o.k_last, o.dense_from)
            assert g.diag_min == o.diag_min and g.fingerprint == o.fingerprint, n
    finally:
        reset_kernel(mp)
        mp.set_word_symmetry(True)
        mp.shutdown()


def test_gamma2_small_cycles_all_paths(mp, oracle_mod):
    """gamma_2(P_n x C_m) for every path order n <= 13 at cycle lengths m <= 8 against the
    DP along the path (a graph oracle independent of the transfer matrix): pins the full-size
    runs n = 10, 11, 12 and the new n = 13 (NEXT-3)."""
    for n in range(2, 14):
        for m in range(3, 9 if n <= 12 else 8):
            assert mp.gamma2_cylinder(n, m) == oracle_mod.gamma2_path_dp(n, m), (n, m)


def test_n13_record(mp):
    """NEXT-3: n = 13 on one B200 (no dense A: 69 GB).  Dense from k = 3
    (P:342); the C_5 formula of [Garzon2022] quoted at P:504 (2n+1 for odd n); the paper's
    conjecture (n+2)m/3 for 3 | m; Lemma 1 via the read-off far beyond k_last."""
    r = mp.gamma2_record(13)
    assert r.dense_from == 3 and r.k_last == r.mu + r.lam
    assert r.gamma2(5) == 27
    for m in range(3, 3000, 3):
        assert r.gamma2(m) == 5 * m
    f = r.formula()
    for m in range(r.mu, r.mu + 200):
        assert r.gamma2(m) == -(-f["b"] * m // f["a"]) + f["alpha"][m % f["a"]]


@pytest.mark.parametrize("pitch", ["host", "dense", "padded"])
@pytest.mark.parametrize("n", [7, 9])
def test_transfer_check_layouts(mp, oracle_mod, n, pitch):
    """The range / transfer-hint check of A on both of its kernels: the vectorised one (rows
    16-byte aligned: host sources are staged with a padded pitch, and a padded device tensor)
    and the general one (a device tensor with lda = N).  A(D_n) passes with the oracle's record;
    a changed label, a dropped arc and an added arc are MP_ERR_DOMAIN; a value in (0x7FFE,
    0xFFFF) is MP_ERR_RANGE."""
    import torch
    A = mp.build_transition_matrix(n)
    N = A.shape[0]
    o = oracle_mod.power_until_periodic(A)
    fin = np.argwhere(A != INF)
    inf = np.argwhere(A == INF)
    cases = []
    for (i, j), v in [(fin[len(fin) // 2], None), (fin[-1], INF), (inf[len(inf) // 3], 3), (fin[1], 0x8000)]:
        B = A.copy()
        B[i, j] = (int(A[i, j]) + 1) if v is None else v
        cases.append((B, "MP_ERR_RANGE" if v == 0x8000 else "MP_ERR_DOMAIN"))

    def run(M):
        if pitch == "host":
            return mp.minplus_power_until_periodic(M)
        ld = N if pitch == "dense" else -(-N // 64) * 64
        d = torch.full((N, ld), -1, dtype=torch.int16, device="cuda")[:, :N]
        d.copy_(torch.from_numpy(M.view(np.int16)))
        return mp.minplus_power_until_periodic_device(d)

    mp.set_transfer_hint(n)
    mp.set_symmetry(mp.word_reversal(n))
    try:
        g = run(A)
        for B, name in cases:
            with pytest.raises(mp.MinplusError) as e:
                run(B)
            assert e.value.name == name
    finally:
        mp.set_symmetry(None)
        mp.set_transfer_hint(0)
    assert (g.mu, g.lam, g.offset) == (o.mu, o.lam, o.offset)
    assert g.diag_min == o.diag_min and g.fingerprint == o.fingerprint


@pytest.mark.parametrize("kernel", ["tiles", "spmm"])
def test_fingerprint_saturating_powers(mp, oracle_mod, kernel):
    """Every power after the first is all-finite here until the sums saturate (G6): A^3 is
    all-finite, A^4 onwards hold +inf.  The tensor-core fingerprint remaps +inf only after a
    power that held +inf, so at A^4 it flags itself void and the statistics kernel hashes that
    power on the CUDA cores: every fingerprint still equals the oracle's."""
    rng = np.random.default_rng(77)
    N = 300
    A = rng.integers(0x2000, 0x2C00, size=(N, N)).astype(np.uint16)
    A[rng.random((N, N)) < 0.002] = INF  # a few +inf in A^1 (remapped: the first power)
    use_kernel(mp, kernel)
    mp.set_symmetry(np.arange(N, dtype=np.int32))  # the identity: every column computed, symmetric path
    try:
        g = mp.minplus_power_until_periodic(A, max_k=16)
    finally:
        mp.set_symmetry(None)
        reset_kernel(mp)
    o = oracle_mod.power_until_periodic(A, max_k=16)
    assert o.rc == 0
    P2 = oracle_mod.minplus(A, A)
    P3 = oracle_mod.minplus(A, P2)
    assert (P3 != INF).all() and (oracle_mod.minplus(A, P3) == INF).any()
    assert (g.mu, g.lam, g.offset, g.k_last, g.dense_from) == (o.mu, o.lam, o.offset, o.k_last, o.dense_from)
    assert g.diag_min == o.diag_min and g.fingerprint == o.fingerprint
