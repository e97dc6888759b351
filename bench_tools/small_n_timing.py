"""Host wall-clock timing of repeated power runs (device-resident A and host A) for small n,
to separate library time from harness effects.  Diagnostic only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2409_17688_b200 as mp  # noqa: E402

torch.cuda.set_device(0)
for n in [int(a) for a in sys.argv[1:]] or [3, 6, 9]:
    A = mp.build_transition_matrix(n)
    dA = torch.from_numpy(A.view(np.int16)).cuda()
    for use_stream in (False, True):
        mp.set_stream(torch.cuda.current_stream() if use_stream else None)
        for _ in range(3):
            mp.minplus_power_until_periodic_device(dA)
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            t = time.perf_counter()
            mp.minplus_power_until_periodic_device(dA)
            ts.append(time.perf_counter() - t)
        p = mp.last_profile()
        th = []
        for _ in range(10):
            t = time.perf_counter()
            mp.minplus_power_until_periodic(A)
            th.append(time.perf_counter() - t)
        print(f"n={n} torch_stream={use_stream} device-A median {np.median(ts)*1e3:.3f} ms min {min(ts)*1e3:.3f} "
              f"| host-A median {np.median(th)*1e3:.3f} ms | lib total {p['total_ms']:.3f} products {p['product_ms']:.3f} "
              f"stats {p['stats_ms']:.3f} setup {p['setup_ms']:.3f}", flush=True)
