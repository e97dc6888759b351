"""Repeated power runs at path order n (argv[1]) with device-resident A; prints the setup
and total time of each run (MP_TRACE=1 adds the phase lines).  Diagnostic only."""
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
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    mp.minplus_power_until_periodic_device(dA)
    p = mp.last_profile()
    print(f"run {it}: setup {p['setup_ms']:.1f} ms, stats {p['stats_ms']:.1f} ms, products {p['product_ms']:.1f} ms, "
          f"total {p['total_ms']:.1f} ms", file=sys.stderr, flush=True)
