"""SURVEY.md section 8(d) kernel micro-benchmark: minplus_mul_device on square N x N x N
products (the dense 128x256x32 tile kernel, staging included).  A: uniform [0, 12] with
P(+inf) in {0, 0.5, 0.992}; B: uniform [0, 600]; generated on the device (seed 17688).
Prints one JSON line per (N, p_inf): ms per product, Gstep/s (N^3 steps) and the fraction of
the 37.2 T steps/s DPX issue peak at 1965 MHz."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2409_17688_b200 as mp  # noqa: E402

PEAK = 148 * 128 * 1965e6
torch.cuda.set_device(0)
sizes = [int(a) for a in sys.argv[1:]] or [1024, 3447, 4096, 8192, 16384, 21294]
g = torch.Generator(device="cuda").manual_seed(17688)
for N in sizes:
    for p_inf in (0.0, 0.5, 0.992):
        A = torch.randint(0, 13, (N, N), generator=g, device="cuda", dtype=torch.int32)
        if p_inf > 0:
            A[torch.rand((N, N), generator=g, device="cuda") < p_inf] = 0xFFFF
        A = A.to(torch.int32).to(torch.uint16) if hasattr(torch, "uint16") else A.to(torch.int16)
        B = torch.randint(0, 601, (N, N), generator=g, device="cuda", dtype=torch.int32).to(A.dtype)
        C = torch.empty_like(A)
        reps = 1 if N >= 16384 else 3
        mp.minplus_mul_device(A, B, C)  # warm-up (allocates the staging buffers)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            mp.minplus_mul_device(A, B, C)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / reps
        steps = float(N) ** 3
        print(json.dumps({"N": N, "p_inf": p_inf, "ms": ms, "gstep_s": steps / ms / 1e6,
                          "frac_of_dpx_peak": steps / (ms * 1e-3) / PEAK}), flush=True)
        del A, B, C
        torch.cuda.empty_cache()
