"""Dev check of the hex sweep path: tiled (sweep) vs coloured on c5 at several sizes and on partitions."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from fem_inputs import make_config, make_state
from paper_2111_03541_b200 import FemSystem
from paper_2111_03541_b200.partition import partition_nodes

def cmp(m, p, st, tag):
    S = FemSystem(m, p)
    sd = torch.from_numpy(st).cuda()
    v1, r1 = [x.clone() for x in S.system(sd, scatter='coloured')]
    S.values.fill_(float("nan")); S.rhs.fill_(float("nan"))
    v2, r2 = S.system(sd, scatter="tiled")
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(3): S.system(sd, scatter='tiled')
    ev[1].record(); torch.cuda.synchronize()
    dv = (v1 - v2).abs().max().item() / v1.abs().max().item()
    dr = (r1 - r2).abs().max().item() / r1.abs().max().item()
    nbad = int(((v1 - v2).abs() > 1e-10 * v1.abs().max()).sum().item())
    print(f'{tag}: E={m.n_elems} tiles={S.info()["n_tiles"]} dv={dv:.2e} dr={dr:.2e} nbad={nbad}/{v1.numel()} '
          f'{ev[0].elapsed_time(ev[1])/3:.3f} ms', flush=True)
    S.close()

for dims in [(7, 5, 6), (16, 16, 16), (13, 17, 70), (64, 64, 64), (128, 128, 128)]:
    m, p = make_config('c5', 'structured', dims)
    cmp(m, p, make_state('c5', m, p), f'c5 {dims}')
m, p = make_config('c5', 'perturbed', (24, 20, 30))
cmp(m, p, make_state('c5', m, p), 'c5 perturbed (24,20,30)')
m, p = make_config('c5', 'structured', (7, 5, 6))
st = make_state('c5', m, p)
for part in partition_nodes(m, 3):
    cmp(part.mesh, p, part.local_state(st), f'part {part.rank} own={part.n_owned}/{part.mesh.n_nodes}')
