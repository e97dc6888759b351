"""Average k_stats / k_stats_sym time per power (one n = 12 run).  Diagnostic only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2409_17688_b200 as mp  # noqa: E402

torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
A = mp.build_transition_matrix(n)
dA = torch.from_numpy(A.view(np.int16)).cuda()
for sym in (True, False):
    mp.set_symmetry(mp.word_reversal(n) if sym else None)
    for _ in range(2):
        r = mp.minplus_power_until_periodic_device(dA)
    p = mp.last_profile()
    print(f"{sys.argv[2] if len(sys.argv) > 2 else ''} sym={sym} stats ms/power {p['stats_ms'] / (r.k_last - 1):.3f} "
          f"total {p['total_ms']:.1f}", flush=True)
