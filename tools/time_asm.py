"""Dev timing helper: python tools/time_asm.py c5[p] [atomic,coloured,tiled,...] [dims...]  (c5p: perturbed variant)"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from fem_inputs import make_config, make_state
from paper_2111_03541_b200 import FemSystem

name = sys.argv[1]
modes = sys.argv[2].split(',') if len(sys.argv) > 2 else ['atomic']
dims = tuple(int(x) for x in sys.argv[3:]) or None
variant = 'perturbed' if name.endswith('p') and name[:-1] in ('c2', 'c3', 'c4', 'c5') else 'structured'
name = name[:-1] if variant == 'perturbed' else name
t0 = time.time(); m, p = make_config(name, variant, dims); st = make_state(name, m, p)
print(f'{name} E={m.n_elems} N={m.n_nodes} gen {time.time()-t0:.1f}s', flush=True)
t0 = time.time(); S = FemSystem(m, p); torch.cuda.synchronize()
print(f'mesh+pattern {time.time()-t0:.1f}s nnz={S.nnz} colours={S.info()}', flush=True)
sd = torch.from_numpy(st).cuda()
for mode in modes:
    for what in ['system', 'matrix', 'residual']:
        f = getattr(S, what)
        for _ in range(3): f(sd, scatter=mode)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        n = 10
        ev[0].record()
        for _ in range(n): f(sd, scatter=mode)
        ev[1].record(); torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / n
        print(f'{mode:9s} {what:8s} {ms:8.3f} ms  {m.n_elems/ms/1e6:8.3f} Gelem/s  {S.nnz/ms/1e6:8.3f} Gnnz/s', flush=True)
print(S.status())
