"""Where the small-N step time goes: the device-timed run with and without an L2 flush before
it, and the library's own event split (setup / kernel / result copy)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2409_17688_b200 as mp  # noqa: E402

torch.cuda.set_device(0)
stream = torch.cuda.current_stream()
mp.set_stream(stream)
for n in (3, 6):
    A = mp.build_transition_matrix(n)
    N = A.shape[0]
    mp.set_symmetry(mp.word_reversal(n))
    dA = torch.from_numpy(A.view(np.int16)).cuda()
    flush = torch.empty(512 * 2**20 // 4, dtype=torch.int32, device="cuda")
    for mode in ("noflush", "flush", "flush+sleep"):
        ts, ks = [], []
        for it in range(30):
            if mode != "noflush":
                flush.fill_(it)
            if mode == "flush+sleep":
                torch.cuda._sleep(2_000_000)  # ~1 ms of spin: the flush drains before the run
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            mp.minplus_power_until_periodic_device(dA)
            e1.record(stream)
            torch.cuda.synchronize()
            if it >= 5:
                ts.append(e0.elapsed_time(e1) * 1000)
                ks.append(mp.last_profile()["product_ms"] * 1000)
        print(f"n={n} {mode:12s} step {np.median(ts):7.1f} us  kernel events {np.median(ks):7.1f} us")
    mp.set_symmetry(None)
