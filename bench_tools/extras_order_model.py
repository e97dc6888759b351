"""Host model of the SpMM tile unions under the row-inclusion reuse (DESIGN.md section 5,
"Extras order"): extra(q) = supp(q) minus the supports of q's parents (q with one letter 0 or
1 turned into a 2), then the total size of the 32-row tile unions (= X rows staged per CTA
column) for the windowed greedy tiles (a model of k_tile_greedy) and for the rows sorted by
their first extra columns.  Offline study (builds A(D_n) with the CPU oracle); usage:
python bench_tools/extras_order_model.py 11"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402


def extras(n):
    W = oracle.words(n)
    fin = oracle.transition_matrix(n) != oracle.INF
    key = {tuple(w): i for i, w in enumerate(W.tolist())}
    out = []
    for q, w in enumerate(W.tolist()):
        s = fin[q].copy()
        for b in range(n):
            if w[b] != 2:
                p = key.get(tuple(w[:b] + [2] + w[b + 1:]))
                if p is not None:
                    s &= ~fin[p]
        out.append(np.flatnonzero(s))
    return out


def tile_unions(ext, order, T=32):
    return sum(len(set().union(*[set(ext[q].tolist()) for q in order[t:t + T]])) for t in range(0, len(order), T))


def greedy_windows(ext, T=32, win=256):
    """pass 2 of the builder: per window of `win` rows, tiles grown by the fewest new columns"""
    order = []
    for w0 in range(0, len(ext), win):
        rem = list(range(w0, min(w0 + win, len(ext))))
        while rem:
            u = set()
            for _ in range(min(T, len(rem))):
                i = min(range(len(rem)), key=lambda i: (len(set(ext[rem[i]].tolist()) - u), i))
                q = rem.pop(i)
                u |= set(ext[q].tolist())
                order.append(q)
    return order


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    ext = extras(n)
    N = len(ext)
    first = lambda q, i: int(ext[q][i]) if len(ext[q]) > i else N  # noqa: E731
    print(f"n = {n}: N = {N}, extras = {sum(len(e) for e in ext)}")
    print("lexicographic tiles   ", tile_unions(ext, list(range(N))))
    print("windowed greedy tiles ", tile_unions(ext, greedy_windows(ext)))
    print("sorted (c1)           ", tile_unions(ext, sorted(range(N), key=lambda q: first(q, 0))))
    print("sorted (c1, c2)       ", tile_unions(ext, sorted(range(N), key=lambda q: (first(q, 0), first(q, 1)))))
