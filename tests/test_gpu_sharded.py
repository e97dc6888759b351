"""The column-sharded (multi-rank) device path, emulated on ONE GPU in one process.

A rank of a G-rank run differs from a 1-GPU run only in (i) its column shard of every power
and (ii) the all-reduce of the per-power statistics and of the exact-compare mismatch count.
Here the library runs as rank r of G with an all-reduce callback that adds the other ranks'
contributions, which the test computes from the oracle's powers (shard statistics with global
indices t = i*N + j).  The shard kernels, the reduction layout and the decision logic are the
real ones; the result must equal the oracle's single-process answer on every rank.  (No
second GPU is involved and no kernels wait on each other.)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

INF = 0xFFFF
I64_MAX = 2**63 - 1


def _i64(u):
    u %= 2**64
    return u - 2**64 if u >= 2**63 else u


def _shard_stats(oracle, X, c0, c1):
    N = X.shape[0]
    if c1 <= c0:
        return 0, 0, INF, I64_MAX
    sub = X[:, c0:c1]
    fp = oracle.fingerprint_cols(X, c0, c1)
    inf = int((sub == INF).sum())
    diag = min([int(X[i, i]) for i in range(c0, c1)] + [INF])
    fin = np.argwhere(sub != INF)
    ref = I64_MAX
    if len(fin):
        i, j = fin[np.lexsort((fin[:, 1], fin[:, 0]))][0]
        ref = (int(i * N + c0 + j) << 16) | int(sub[i, j])
    return fp, inf, diag, ref


@pytest.mark.parametrize("n,world", [(5, 2), (6, 3), (7, 2), (8, 4), (3, 3)])
def test_sharded_run_emulated(oracle_mod, n, world):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)
    import paper_2409_17688_b200 as mp

    A = oracle_mod.transition_matrix(n)
    N = A.shape[0]
    o = oracle_mod.power_until_periodic(A)
    P = {1: A}
    for k in range(2, o.k_last + 1):
        P[k] = oracle_mod.minplus(A, P[k - 1])
    S = mp.fingerprint_unit(N)
    shards = [mp.shard_range(N, world, r) for r in range(world)]
    full = {k: _shard_stats(oracle_mod, P[k], 0, N) for k in P}
    gstats = {k: mp.PowerStats(_i64(full[k][0]), full[k][1], full[k][2], full[k][3]) for k in P}

    for rank in range(world):
        others = [s for r, s in enumerate(shards) if r != rank]
        part = {k: [_shard_stats(oracle_mod, P[k], a, b) for a, b in others] for k in P}
        # the compares the library will request, in order, from the global statistics
        expected = []
        for k in range(1, o.k_last + 1):
            for j in range(k - 1, 0, -1):
                c = mp.repeat_candidate(gstats[k], gstats[j], S)
                if c is not None:
                    expected.append((k, j, c))
                    if oracle_mod.constant_difference(P[k], P[j]) == c:
                        break
        state = {"k": 0, "kb": 1, "cmp": 0}

        class _Dev:
            def __init__(self, ptr, cnt):
                self.__cuda_array_interface__ = {"shape": (cnt,), "typestr": "<i8", "data": (ptr, False),
                                                 "version": 3, "strides": None, "stream": None}

        def allreduce(op, ptr, count):
            t = torch.as_tensor(_Dev(ptr, count), device="cuda")
            vals = [int(v) for v in t.cpu().tolist()]
            if op == 0 and count >= 2:          # SUM {fingerprint, inf count} of a batch of powers
                out = []
                for q in range(count // 2):
                    k = state["k"] + 1 + q
                    got = part.get(k, [])       # powers past k_last: any value (discarded)
                    out += [_i64(vals[2 * q] + sum(p[0] for p in got)), vals[2 * q + 1] + sum(p[1] for p in got)]
                state["kb"] = state["k"] + 1
                state["k"] += count // 2
            elif op == 1 and count >= 2:        # MIN {diag min, first finite entry} of the batch
                out = []
                for q in range(count // 2):
                    got = part.get(state["kb"] + q, [])
                    out += [min([vals[2 * q]] + [p[2] for p in got]), min([vals[2 * q + 1]] + [p[3] for p in got])]
            elif op == 0 and count == 1:        # SUM of exact-compare mismatches
                k, j, c = expected[state["cmp"]]
                state["cmp"] += 1
                assert state["kb"] <= k <= state["k"]
                bad = vals[0]
                for a, b in others:
                    Y, Z = P[k][:, a:b].astype(np.int64), P[j][:, a:b].astype(np.int64)
                    bad += int(((Y == INF) != (Z == INF)).sum() + ((Y != INF) & (Y - Z != c)).sum())
                out = [bad]
            else:
                raise AssertionError((op, count))
            t.copy_(torch.tensor(out, dtype=torch.int64, device="cuda"))
            torch.cuda.synchronize()

        mp.dist_set(rank, world, allreduce)
        try:
            g = mp.minplus_power_until_periodic(A)
        finally:
            mp.dist_set(0, 1, None)
        assert (g.mu, g.lam, g.offset, g.k_last, g.dense_from) == (o.mu, o.lam, o.offset, o.k_last, o.dense_from)
        assert g.diag_min == o.diag_min and g.fingerprint == o.fingerprint
        assert state["cmp"] == len(expected)


def _cols_stats(oracle, X, cols):
    """Statistics of the full matrix restricted to a set of columns (global indices)."""
    N = X.shape[0]
    cols = sorted(set(int(c) for c in cols))
    if not cols:
        return 0, 0, INF, I64_MAX
    fp = sum(oracle.fingerprint_cols(X, c, c + 1) for c in cols) % 2**64
    sub = X[:, cols]
    inf = int((sub == INF).sum())
    diag = min([int(X[c, c]) for c in cols] + [INF])
    ref = I64_MAX
    for jj, c in enumerate(cols):
        fin = np.nonzero(sub[:, jj] != INF)[0]
        if len(fin):
            i = int(fin[0])
            ref = min(ref, (int(i * N + c) << 16) | int(X[i, c]))
    return fp, inf, diag, ref


@pytest.mark.parametrize("n,world", [(5, 2), (7, 3), (8, 2)])
def test_sharded_run_symmetry_emulated(oracle_mod, n, world):
    """As above with the word-reversal symmetry: the ranks shard the domain D = {g <= sigma g}
    and a domain column stands for g and sigma g in every statistic."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)
    import paper_2409_17688_b200 as mp

    A = oracle_mod.transition_matrix(n)
    N = A.shape[0]
    sigma = mp.word_reversal(n)
    D = [g for g in range(N) if g <= sigma[g]]
    o = oracle_mod.power_until_periodic(A)
    P = {1: A}
    for k in range(2, o.k_last + 1):
        P[k] = oracle_mod.minplus(A, P[k - 1])
    shards = [mp.shard_range(len(D), world, r) for r in range(world)]

    def colset(a, b):
        return [D[q] for q in range(a, b)] + [int(sigma[D[q]]) for q in range(a, b)]

    for rank in range(world):
        others = [s for r, s in enumerate(shards) if r != rank]
        part = {k: [_cols_stats(oracle_mod, P[k], colset(a, b)) for a, b in others] for k in P}
        state = {"k": 0, "kb": 1}

        class _Dev:
            def __init__(self, ptr, cnt):
                self.__cuda_array_interface__ = {"shape": (cnt,), "typestr": "<i8", "data": (ptr, False),
                                                 "version": 3, "strides": None, "stream": None}

        def allreduce(op, ptr, count):
            t = torch.as_tensor(_Dev(ptr, count), device="cuda")
            vals = [int(v) for v in t.cpu().tolist()]
            if op == 0 and count >= 2:
                out = []
                for q in range(count // 2):
                    got = part.get(state["k"] + 1 + q, [])
                    out += [_i64(vals[2 * q] + sum(p[0] for p in got)), vals[2 * q + 1] + sum(p[1] for p in got)]
                state["kb"] = state["k"] + 1
                state["k"] += count // 2
            elif op == 1 and count >= 2:
                out = []
                for q in range(count // 2):
                    got = part.get(state["kb"] + q, [])
                    out += [min([vals[2 * q]] + [p[2] for p in got]), min([vals[2 * q + 1]] + [p[3] for p in got])]
            elif op == 0 and count == 1:        # exact-compare mismatches of the other domain shards
                out = [vals[0]]                 # (the decisive compare has none anywhere)
            else:
                raise AssertionError((op, count))
            t.copy_(torch.tensor(out, dtype=torch.int64, device="cuda"))
            torch.cuda.synchronize()

        mp.set_symmetry(sigma)
        mp.dist_set(rank, world, allreduce)
        try:
            g = mp.minplus_power_until_periodic(A)
        finally:
            mp.dist_set(0, 1, None)
            mp.set_symmetry(None)
        assert (g.mu, g.lam, g.offset, g.k_last, g.dense_from) == (o.mu, o.lam, o.offset, o.k_last, o.dense_from)
        assert g.diag_min == o.diag_min and g.fingerprint == o.fingerprint


def test_dist_torch_nccl_world1(oracle_mod):
    """The torch.distributed (NCCL) callback plumbing end to end with a 1-rank group."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2409_17688_b200 as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        mp.dist_set_torch()
        A = oracle_mod.transition_matrix(6)
        o = oracle_mod.power_until_periodic(A)
        for sym in (False, True):
            mp.set_symmetry(mp.word_reversal(6) if sym else None)
            try:
                g = mp.minplus_power_until_periodic(A)
            finally:
                mp.set_symmetry(None)
            assert (g.mu, g.lam, g.offset) == (o.mu, o.lam, o.offset)
            assert g.fingerprint == o.fingerprint and g.diag_min == o.diag_min
    finally:
        mp.dist_set(0, 1, None)
        dist.destroy_process_group()
