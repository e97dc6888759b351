"""Average product-kernel time over a few powers (minplus_power_rows, no periodicity search),
for kernel experiments whose results are not meaningful.  Diagnostic only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2409_17688_b200 as mp  # noqa: E402

torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
A = mp.build_transition_matrix(n)
mp.set_symmetry(mp.word_reversal(n))
mp.set_spmm_width(int(os.environ.get("MP_WIDTH", "0")))  # 0: the automatic choice
for _ in range(2):
    mp.minplus_power_rows(A, np.array([0]), 6)
p = mp.last_profile()
print(f"{sys.argv[2] if len(sys.argv) > 2 else ''} n={n} product_ms/launch {p['product_ms'] / p['product_launches']:.3f} "
      f"issued G/launch {p['issued_steps'] / p['product_launches'] / 1e9:.1f}", flush=True)
