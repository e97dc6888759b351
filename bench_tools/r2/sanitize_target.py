"""Small runs of every device path for compute-sanitizer (memcheck / racecheck / synccheck):
the grouped SpMM (bulk-copy + mbarrier ring) at every CTA width with and without the word-reversal
symmetry, the remainder CTA columns, the row-inclusion reuse and its fold passes, the tile
kernels, the fused small-N cluster kernel, the observer path and a product."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2409_17688_b200 as mp  # noqa: E402

torch.cuda.set_device(0)
n = int(os.environ.get("MP_SAN_N", "7"))
A = mp.build_transition_matrix(n)
mp.set_small_path(False)
mp.set_options("spmm")
mp.set_grouping("greedy")
for width in (256, 512, 1024, -1024):
    mp.set_spmm_width(width)
    for sym in (False, True):
        mp.set_symmetry(mp.word_reversal(n) if sym else None)
        g = mp.minplus_power_until_periodic(A)
        print("spmm", width, sym, (g.mu, g.lam, g.offset), flush=True)
mp.set_spmm_width(0)
mp.set_transfer_hint(n)
g = mp.minplus_power_until_periodic(A)
print("row reuse", (g.mu, g.lam, g.offset), mp.last_profile()["row_levels"], flush=True)
mp.set_transfer_hint(0)
mp.set_symmetry(None)
mp.set_options("tiles")
g = mp.minplus_power_until_periodic(A)
print("tiles", (g.mu, g.lam, g.offset), flush=True)
mp.set_options("auto")
mp.set_grouping("auto")
mp.set_small_path(True)
g = mp.minplus_power_until_periodic(mp.build_transition_matrix(6))
print("small", (g.mu, g.lam, g.offset), mp.last_profile()["kernel"], flush=True)
mp.set_power_observer(lambda k, X: None)
g = mp.minplus_power_until_periodic(mp.build_transition_matrix(5))
mp.set_power_observer(None)
C = mp.minplus_mul(A[:300], A[:, :200])
print("done", C.shape, flush=True)
