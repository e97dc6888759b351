"""The multi-rank (column-sharded) periodicity logic on CPU with torch.distributed/gloo.

Each rank owns the column shard mp.shard_range(N, world, rank) of every power, reduces its
shard statistics exactly as the device driver does (SUM of fingerprint and +inf count, MIN of
diagonal minimum and first finite entry), and runs the library's own candidate test
(mp_repeat_candidate) plus a sharded exact comparison whose mismatch counts are SUM-reduced.
The shard powers come from the oracle (this is a test of the host-side logic, not of the
kernels); the decision must equal the single-process oracle's (mu, lambda, b) on every rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

INF = 0xFFFF
I64_MAX = 2**63 - 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _to_i64(u):
    return u - 2**64 if u >= 2**63 else u


def _shard_stats(oracle, X, c0, c1):
    N = X.shape[0]
    sub = X[:, c0:c1]
    fp = oracle.fingerprint_cols(X, c0, c1) if c1 > c0 else 0
    inf = int((sub == INF).sum())
    diag = min([int(X[i, i]) for i in range(c0, c1)] + [INF])
    ref = I64_MAX
    fin = np.argwhere(sub != INF)
    if len(fin):
        i, j = fin[np.lexsort((fin[:, 1], fin[:, 0]))][0]
        ref = (int(i * N + c0 + j) << 16) | int(sub[i, j])
    return fp, inf, diag, ref


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2409_17688_b200 as mp
        A = oracle.transition_matrix(n)
        N = A.shape[0]
        c0, c1 = mp.shard_range(N, world, rank)
        S = mp.fingerprint_unit(N)
        P = {1: A}
        stats = {}
        found = None
        for k in range(1, 64):
            if k > 1:
                P[k] = oracle.minplus(A, P[k - 1])
            fp, inf, diag, ref = _shard_stats(oracle, P[k], c0, c1)
            s = torch.tensor([_to_i64(fp % 2**64), inf], dtype=torch.int64)
            m = torch.tensor([diag, ref], dtype=torch.int64)
            dist.all_reduce(s, op=dist.ReduceOp.SUM)
            dist.all_reduce(m, op=dist.ReduceOp.MIN)
            st = mp.PowerStats(int(s[0]), int(s[1]), int(m[0]), int(m[1]))
            # the reduced statistics equal the whole-matrix ones
            assert st.fingerprint % 2**64 == oracle.fingerprint(P[k])
            assert st.inf_count == int((P[k] == INF).sum())
            assert st.diag_min == int(np.diag(P[k]).min())
            stats[k] = st
            for j in range(k - 1, 0, -1):
                c = mp.repeat_candidate(stats[k], stats[j], S)
                if c is None:
                    continue
                Y, Z = P[k][:, c0:c1].astype(np.int64), P[j][:, c0:c1].astype(np.int64)
                bad = int(((Y == INF) != (Z == INF)).sum() + ((Y != INF) & (Y - Z != c)).sum())
                b = torch.tensor([bad], dtype=torch.int64)
                dist.all_reduce(b, op=dist.ReduceOp.SUM)
                if int(b[0]) == 0:
                    found = (j, k - j, c)
                    break
            if found:
                break
        q.put((rank, found))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,world", [(4, 2), (5, 2), (3, 3)])
def test_sharded_periodicity_matches_oracle(oracle_mod, n, world):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    got = dict(q.get(timeout=10) for _ in range(world))
    o = oracle_mod.power_until_periodic(oracle_mod.transition_matrix(n))
    for r in range(world):
        assert got[r] == (o.mu, o.lam, o.offset), (r, got)
