"""One power run at path order n (argv[1]) with device-resident A, for a launch list of the
setup kernels under ncu.  Diagnostic only."""
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
r = mp.minplus_power_until_periodic_device(dA)
print(n, r.mu, r.lam, r.offset, mp.last_profile())
