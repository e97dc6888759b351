"""Full-size parity: every power of the benchmarked runs (n = 10, 11, 12) against the oracle.

The golden records ``tests/golden/power_records_n{n}.json`` are written by
``tests/golden/make_power_records.py``, which imports only ``oracle/``: the oracle's skip-inf
triple loop runs Algorithm 2 to the first repeat (Lemma 1) and records,
for every power A^k, its fingerprint, diagonal minimum (Algorithm 5), +inf count, first finite
entry and the SHA-256 of the whole matrix.  Here the CUDA path (through the C ABI) must
reproduce:

* every record field, for the configuration bench.py times (device-resident A, word-reversal
  symmetry, automatic SpMM width and greedy row grouping), for the all-columns run, for the
  tile kernel and for the words source of gamma2_cylinder;
* the SHA-256 of every whole power (the observer hands each A^k over in full), i.e. every entry
  of every power of the benchmarked run equals the oracle's;
* with MP_FULL_PARITY=1 (a long run, logged under profiles/), a streamed element-wise compare:
  each GPU power against the oracle's power computed in lockstep on the host.
"""
import hashlib
import json
import os
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def records(n):
    with open(os.path.join(ROOT, "tests", "golden", f"power_records_n{n}.json")) as f:
        return json.load(f)


def have(n):
    return os.path.exists(os.path.join(ROOT, "tests", "golden", f"power_records_n{n}.json"))


SIZES = [n for n in (10, 11, 12) if have(n)]


@pytest.fixture(scope="module")
def mp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)
    import paper_2409_17688_b200 as m
    m.set_options("auto", device_budget_bytes=0)
    return m


def sha(X):
    assert X.dtype == np.uint16 and X.flags["C_CONTIGUOUS"] and sys.byteorder == "little"
    return hashlib.sha256(memoryview(X.reshape(-1)).cast("B")).hexdigest()


def check_result(g, rec):
    pw = rec["powers"]
    assert (g.mu, g.lam, g.offset, g.k_last) == (rec["mu"], rec["lambda_"], rec["offset"], rec["k_last"])
    assert len(pw) == g.k_last
    assert g.diag_min[1:] == [p["diag_min"] for p in pw]
    assert [str(f) for f in g.fingerprint[1:]] == [p["fingerprint"] for p in pw]
    assert g.dense_from == next(p["k"] for p in pw if p["inf_count"] == 0)


def run_config(mp, A, n, config):
    import torch
    if config == "bench":  # exactly what bench.py times: device-resident A, its stream, hints
        mp.set_symmetry(mp.word_reversal(n))
        mp.set_transfer_hint(n)
        N = A.shape[0]
        ld = -(-N // 64) * 64  # bench.py's row pitch
        dA = torch.full((N, ld), -1, dtype=torch.int16, device="cuda")[:, :N]
        dA.copy_(torch.from_numpy(A.view(np.int16)))
        mp.set_stream(torch.cuda.current_stream())
        try:
            g = mp.minplus_power_until_periodic_device(dA)
            assert mp.last_profile()["row_levels"] > 1  # the row-inclusion reuse ran
            return g
        finally:
            mp.set_stream(None)
            mp.set_symmetry(None)
            mp.set_transfer_hint(0)
    if config == "allcols":
        return mp.minplus_power_until_periodic(A)
    if config == "noreuse":  # the benchmarked options without the row-inclusion reuse
        mp.set_symmetry(mp.word_reversal(n))
        mp.set_transfer_hint(n)
        mp.set_row_reuse(False)
        try:
            g = mp.minplus_power_until_periodic(A)
            assert mp.last_profile()["row_levels"] == 0
            return g
        finally:
            mp.set_row_reuse(True)
            mp.set_symmetry(None)
            mp.set_transfer_hint(0)
    if config in ("nolookahead", "nofptc"):  # the benchmarked options, other code paths: no
        # lookahead power loop / the fingerprint on the CUDA cores instead of the tensor cores
        env = {"nolookahead": {"MP_LOOKAHEAD": "0"}, "nofptc": {"MP_FP_TC": "0"}}[config]
        os.environ.update(env)
        mp.set_symmetry(mp.word_reversal(n))
        mp.set_transfer_hint(n)
        try:
            return mp.minplus_power_until_periodic(A)
        finally:
            for v in env:
                del os.environ[v]
            mp.set_symmetry(None)
            mp.set_transfer_hint(0)
    if config == "tiles":
        mp.set_options("tiles")
        try:
            return mp.minplus_power_until_periodic(A)
        finally:
            mp.set_options("auto")
    raise ValueError(config)


@pytest.mark.parametrize("config", ["bench", "allcols", "tiles", "noreuse", "nolookahead", "nofptc"])
@pytest.mark.parametrize("n", SIZES)
def test_power_records(mp, n, config):
    """Every power's fingerprint and diagonal minimum, (mu, lambda, b) and dense_from equal the
    oracle's golden records; the input A(D_n) from the library's host builder is itself pinned
    by the record of A^1 (its SHA-256)."""
    rec = records(n)
    A = mp.build_transition_matrix(n)
    assert A.shape == (rec["N"], rec["N"]) and sha(A) == rec["powers"][0]["sha256"]
    check_result(run_config(mp, A, n, config), rec)


@pytest.mark.parametrize("n", SIZES)
def test_words_source_records(mp, n):
    """gamma2_cylinder's record (A(D_n) built on the device from the word masks, symmetry on)."""
    mp.shutdown()
    try:
        check_result(mp.gamma2_record(n), records(n))
    finally:
        mp.shutdown()


@pytest.mark.parametrize("n", SIZES)
def test_every_entry_of_every_power(mp, n):
    """The benchmarked configuration with the power observer: the SHA-256 of every whole power
    A^1 .. A^{k_last} (columns the symmetric run does not compute filled in from their mirrors)
    equals the oracle's -- every entry of every power is the oracle's."""
    rec = records(n)
    A = mp.build_transition_matrix(n)
    seen = {}
    mp.set_power_observer(lambda k, X: seen.__setitem__(k, sha(X)))
    try:
        g = run_config(mp, A, n, "bench")
    finally:
        mp.set_power_observer(None)
    check_result(g, rec)
    assert sorted(seen) == list(range(1, g.k_last + 1))
    for p in rec["powers"]:
        assert seen[p["k"]] == p["sha256"], p["k"]


def test_observer_rejects_sharded_runs(mp):
    """A rank holds only its shard: an observer with world > 1 is a domain error."""
    A = mp.build_transition_matrix(4)
    mp.dist_set(0, 2, lambda op, ptr, count: None)
    mp.set_power_observer(lambda k, X: None)
    try:
        with pytest.raises(mp.MinplusError) as e:
            mp.minplus_power_until_periodic(A)
        assert e.value.name == "MP_ERR_DOMAIN"
    finally:
        mp.set_power_observer(None)
        mp.dist_set(0, 1, None)


def test_observer_stop(mp, oracle_mod):
    """fn returning True stops the run with MP_ERR_DOMAIN; the powers it saw are the oracle's."""
    A = oracle_mod.transition_matrix(6)
    P = oracle_mod.powers(A, 5)
    seen = []

    def obs(k, X):
        assert np.array_equal(X, P[k])
        seen.append(k)
        return k == 5
    mp.set_power_observer(obs)
    try:
        with pytest.raises(mp.MinplusError) as e:
            mp.minplus_power_until_periodic(A)
        assert e.value.name == "MP_ERR_DOMAIN"
    finally:
        mp.set_power_observer(None)
    assert seen == [1, 2, 3, 4, 5]


def test_device_entry_strided(mp, oracle_mod):
    """The device entry point on a pitched tensor (lda > N) written asynchronously by torch on
    its current stream, while the library runs on its own stream (the binding orders them)."""
    import torch
    A = oracle_mod.transition_matrix(8)
    N = A.shape[0]
    o = oracle_mod.power_until_periodic(A)
    big = torch.full((N, N + 37), -1, dtype=torch.int16, device="cuda")
    for _ in range(3):
        big.fill_(7)
        dA = big[:, 5:5 + N]
        dA.copy_(torch.from_numpy(A.view(np.int16)).cuda(non_blocking=True))
        g = mp.minplus_power_until_periodic_device(dA)
        assert (g.mu, g.lam, g.offset) == (o.mu, o.lam, o.offset)
        assert g.fingerprint == o.fingerprint and g.diag_min == o.diag_min


@pytest.mark.skipif(os.environ.get("MP_FULL_PARITY") != "1", reason="long: set MP_FULL_PARITY=1")
@pytest.mark.parametrize("n", [11])
def test_streamed_elementwise(mp, oracle_mod, n):
    """Each power of the benchmarked run against the oracle's power computed in lockstep on the
    host (oracle.minplus, A^k = A (x) A^{k-1}), element by element."""
    import time
    A = oracle_mod.transition_matrix(n)
    state = {"prev": None, "oracle_s": 0.0}

    def obs(k, X):
        t = time.time()
        ref = A if k == 1 else oracle_mod.minplus(A, state["prev"])
        state["oracle_s"] += time.time() - t
        bad = np.count_nonzero(X != ref)
        assert bad == 0, (k, bad)
        state["prev"] = ref
        print(f"n={n} k={k} equal ({X.size} entries), oracle {state['oracle_s']:.1f} s", flush=True)
    mp.set_power_observer(obs)
    try:
        g = run_config(mp, A, n, "bench")
    finally:
        mp.set_power_observer(None)
    if have(n):
        check_result(g, records(n))
