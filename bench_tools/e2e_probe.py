import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2409_17688_b200 as mp
torch.cuda.set_device(0)
n=int(sys.argv[1])
A=mp.build_transition_matrix(n); N=A.shape[0]
mp.set_symmetry(mp.word_reversal(n)); mp.set_transfer_hint(n)
pinned=torch.from_numpy(A.view(np.int16)).pin_memory(); Ah=pinned.numpy().view(np.uint16)
flush=torch.empty(512*2**20//4, dtype=torch.int32, device='cuda')
for mode in ('lib', 'torch'):
    mp.set_stream(None if mode=='lib' else torch.cuda.current_stream())
    for fl in (False, True):
        ts=[]; ws=[]
        for i in range(12):
            if fl: flush.fill_(i)
            e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
            e0.record(); t0=time.perf_counter()
            mp.minplus_power_until_periodic(Ah)
            t1=time.perf_counter(); e1.record(); torch.cuda.synchronize()
            if i>=2: ts.append(e0.elapsed_time(e1)); ws.append((t1-t0)*1e3)
        p=mp.last_profile()
        print(f"n={n} stream={mode:5s} flush={fl!s:5s} events {np.median(ts):7.3f} ms  wall {np.median(ws):7.3f} ms  lib total {p['total_ms']:.3f} setup {p['setup_ms']:.3f}")
