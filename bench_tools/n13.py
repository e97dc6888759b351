"""NEXT-3: the power sequence of A(D_13) (N = 131562, 34.6 GB per power; the paper's future
work) on one B200, with the checks the paper allows at n = 13."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2409_17688_b200 as mp  # noqa: E402

torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 13
t = time.time()
r = mp.gamma2_record(n)
dt = time.time() - t
out = {"n": n, "N": mp.count_words(n), "mu": r.mu, "lambda": r.lam, "b": r.offset, "k_last": r.k_last,
       "dense_from": r.dense_from, "diag_min": r.diag_min[1:], "seconds": dt, "profile": mp.last_profile(),
       "formula": r.formula(), "gamma2": {m: r.gamma2(m) for m in list(range(3, 61)) + [1000, 10**6]}}
# checks the paper states for any n: C_5 formula of [Garzon2022], and the conjecture
# gamma_2 = (n+2) m / 3 for n >= 8, 3 | m
out["check_C5"] = r.gamma2(5) == (2 * n + 2 if n % 2 == 0 else 2 * n + 1)
out["check_conjecture"] = all(r.gamma2(m) == (n + 2) * m // 3 for m in range(3, 3000, 3))
print(json.dumps(out), flush=True)
