"""The column-sharded power run with REAL ranks: 2 and 3 processes on cuda:0, each running the
library's device path on its own shard, the per-power statistics all-reduced by
torch.distributed (gloo on CUDA tensors: NCCL refuses two ranks on one GPU).  No rank's kernels
wait on another's -- the ranks only meet in the host-side all-reduce of a few int64 values per
power -- so one GPU stands in for several without distorting the algorithm (DESIGN.md
section 6).  Every rank must return the oracle's (mu, lambda, b), every diag_min and every
fingerprint."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, cases, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2409_17688_b200 as mp
    mp.dist_set_torch()
    out = []
    try:
        for n, sym, reuse in cases:
            A = mp.build_transition_matrix(n)
            mp.set_symmetry(mp.word_reversal(n) if sym else None)
            mp.set_transfer_hint(n if reuse else 0)
            mp.set_grouping("greedy" if reuse else "auto")
            mp.set_options("spmm" if reuse else "auto")
            g = mp.minplus_power_until_periodic(A)
            p = mp.last_profile()
            out.append(((n, sym, reuse), (g.mu, g.lam, g.offset, g.k_last, g.dense_from), g.diag_min, g.fingerprint,
                        p["local_cols"], p["row_levels"]))
        mp.set_symmetry(None)
        mp.set_transfer_hint(0)
        mp.set_grouping("auto")
        mp.set_options("auto")
        # sharded general products: every rank passes the same operands, gets the whole C
        import synth
        prods = []
        for (M, K, N) in PRODUCTS:
            A = synth.transfer_like(M, K, 0.5, salt=M + K)
            B = synth.power_like(K, N, salt=N + K)
            prods.append(mp.minplus_mul(A, B))
        W = synth.transfer_like(300, 300, 0.98, salt=31)
        prods.append(mp.minplus_closure(W))
        q.put((rank, out, None, prods))
    except Exception as e:  # noqa: BLE001 -- reported to the parent
        q.put((rank, None, repr(e), None))
    finally:
        dist.destroy_process_group()


CASES = [(6, False, False), (8, True, False), (9, True, True), (10, True, True), (10, False, False)]
PRODUCTS = [(5, 7, 3), (300, 200, 517), (129, 1000, 1031)]


@pytest.mark.parametrize("world", [2, 3])
def test_real_ranks_on_one_gpu(oracle_mod, world):
    import torch
    import torch.multiprocessing as tmp
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, CASES, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=900) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, out, err, _ in got:
        assert err is None, (rank, err)
    ref = {}
    for n in sorted({c[0] for c in CASES}):
        o = oracle_mod.power_until_periodic(oracle_mod.transition_matrix(n))
        ref[n] = ((o.mu, o.lam, o.offset, o.k_last, o.dense_from), o.diag_min, o.fingerprint)
    import synth
    refp = []
    for (M, K, N) in PRODUCTS:
        refp.append(oracle_mod.minplus(synth.transfer_like(M, K, 0.5, salt=M + K), synth.power_like(K, N, salt=N + K)))
    W = synth.transfer_like(300, 300, 0.98, salt=31)
    X = W.copy()
    np.fill_diagonal(X, 0)
    t = 0
    while 2 ** t < 299:
        X = oracle_mod.minplus(X, X)
        t += 1
    for rank, _, _, prods in got:  # the sharded general products: whole C on every rank
        for C, R in zip(prods[:-1], refp):
            assert np.array_equal(C, R), rank
        D, tt = prods[-1]
        assert tt == t and np.array_equal(D, X), rank
    for rank, out, _, _ in got:
        cols = {}
        for case, summary, diag, fp, local_cols, levels in out:
            n = case[0]
            assert summary == ref[n][0], (rank, case)
            assert diag == ref[n][1] and fp == ref[n][2], (rank, case)
            if case[2]:
                assert levels > 1, (rank, case)  # the row-inclusion reuse ran on the shard
            cols[case] = local_cols
        assert all(v > 0 for v in cols.values())
