"""The small-N latency path (N <= 256: the whole run in one thread-block-cluster launch) against
the oracle and against the general path, bit for bit (DESIGN.md section 5 "Small-N path")."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)
    import paper_2409_17688_b200 as m
    m.set_options("auto", device_budget_bytes=0)
    m.set_small_path(True)
    return m


def same(g, o):
    assert (g.mu, g.lam, g.offset, g.k_last, g.dense_from) == (o.mu, o.lam, o.offset, o.k_last, o.dense_from)
    assert g.diag_min == o.diag_min and g.fingerprint == o.fingerprint


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6])
def test_transfer_matrices(mp, oracle_mod, n):
    """A(D_n), n <= 6 (N = 6 .. 225; one to four CTAs): the one-launch run = the oracle, and the
    profile says the fused kernel ran."""
    A = oracle_mod.transition_matrix(n)
    g = mp.minplus_power_until_periodic(A)
    assert mp.last_profile()["kernel"] == "small"
    same(g, oracle_mod.power_until_periodic(A))


@pytest.mark.parametrize("seed", range(8))
def test_random_sparse(mp, oracle_mod, seed):
    """Random sparse matrices, ragged N (the +inf pattern persists for several powers: the exact
    compare with +inf entries); the general path gives the same record."""
    N = [1, 7, 63, 64, 65, 129, 200, 256][seed]
    A = synth.transfer_like(N, N, [0.0, 0.6, 0.9, 0.9, 0.93, 0.95, 0.97, 0.97][seed], salt=900 + seed)
    o = oracle_mod.power_until_periodic(A)
    try:
        g = mp.minplus_power_until_periodic(A)
        assert mp.last_profile()["kernel"] == "small"
    except mp.MinplusError as e:
        assert e.name == "MP_ERR_NOT_PERIODIC" and o.rc == 4
        return
    assert o.rc == 0
    same(g, o)
    mp.set_small_path(False)
    try:
        same(mp.minplus_power_until_periodic(A), o)
    finally:
        mp.set_small_path(True)


def test_dense_falls_back(mp, oracle_mod):
    """More finite entries than the kernel's shared memory holds (N = 200, dense): the general
    path runs instead, same answer."""
    A = synth.tropical_matrix(200, 200, lo=1, hi=9, salt=77)
    np.fill_diagonal(A, 0)  # powers converge to the shortest-path matrix: A^k = A^{k+1}
    g = mp.minplus_power_until_periodic(A)
    assert mp.last_profile()["kernel"] != "small"
    same(g, oracle_mod.power_until_periodic(A))


def test_errors(mp, oracle_mod):
    """Range error, a violated symmetry hint, and no repeat within max_k: the same statuses as
    the general path; a valid hint is accepted."""
    A = oracle_mod.transition_matrix(5)
    bad = A.copy()
    bad[3, 4] = 0x8000
    with pytest.raises(mp.MinplusError) as e:
        mp.minplus_power_until_periodic(bad)
    assert e.value.name == "MP_ERR_RANGE"
    mp.set_symmetry(mp.word_reversal(5))
    try:
        same(mp.minplus_power_until_periodic(A), oracle_mod.power_until_periodic(A))
        asym = A.copy()
        i, j = np.argwhere(A != 0xFFFF)[5]
        asym[i, j] = A[i, j] + 1
        with pytest.raises(mp.MinplusError) as e:
            mp.minplus_power_until_periodic(asym)
        assert e.value.name == "MP_ERR_DOMAIN"
    finally:
        mp.set_symmetry(None)
    with pytest.raises(mp.MinplusError) as e:
        mp.minplus_power_until_periodic(A, max_k=10)  # mu + lambda = 38 for n = 5
    assert e.value.name == "MP_ERR_NOT_PERIODIC"


@pytest.mark.parametrize("max_k", [2, 3, 8, 16, 17])
def test_small_max_k(mp, oracle_mod, max_k):
    """Short runs (ADVICE: ring sizing for max_k <= 16) on both paths: a constant matrix repeats
    at once (A^2 = A + c), a transfer matrix does not within max_k."""
    Z = np.zeros((4, 4), dtype=np.uint16)
    for small in (True, False):
        mp.set_small_path(small)
        try:
            g = mp.minplus_power_until_periodic(Z, max_k=max_k)
            assert (g.mu, g.lam, g.offset, g.k_last) == (1, 1, 0, 2)
            A = oracle_mod.transition_matrix(6)
            with pytest.raises(mp.MinplusError) as e:
                mp.minplus_power_until_periodic(A, max_k=max_k)
            assert e.value.name == "MP_ERR_NOT_PERIODIC"
        finally:
            mp.set_small_path(True)


def test_words_source_and_device_entry(mp, oracle_mod):
    """gamma2_cylinder for n <= 6 (words source) and the device entry point on the small path."""
    import torch
    mp.shutdown()
    for n in range(2, 7):
        o = oracle_mod.power_until_periodic(oracle_mod.transition_matrix(n))
        for m in list(range(3, 40)) + [1000]:
            assert mp.gamma2_cylinder(n, m) == o.gamma2(m)
        A = oracle_mod.transition_matrix(n)
        dA = torch.from_numpy(A.view(np.int16)).cuda()
        same(mp.minplus_power_until_periodic_device(dA), o)
