import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle
from fem_inputs import make_config, make_state
from paper_2111_03541_b200 import FemSystem
for dims in [(9, 4, 3), (20, 8, 8)]:
    m, p = make_config("c4", "structured", dims)
    st = make_state("c4", m, p)
    S = FemSystem(m, p)
    sd = torch.from_numpy(st).cuda()
    S.system(sd, scatter="tiled"); d = S.rhs.clone()
    for rs in (40, 100, 400):
        x, it, rel = S.solve(-d, rtol=1e-11, max_iter=3000, method="gmres", restart=rs)
        print(dims, S.n_rows, 'restart', rs, 'it', it, 'rel', rel, flush=True)
    x, it, rel = S.solve(-d, rtol=1e-11, max_iter=3000, method="bicgstab")
    print(dims, 'bicgstab it', it, 'rel', rel, flush=True)
    S.close()
