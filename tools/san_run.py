"""Small ordered-mode assemblies for compute-sanitizer: c5 (z-sweep), c2 (hex node tiles), c3 (ordered P2),
c4 (ordered NS), each TILED once; c3 also STORED (element pass + per-slot gather)."""
import sys
import torch
sys.path.insert(0, '.')
from fem_inputs import make_config, make_state
from paper_2111_03541_b200 import FemSystem
for name, dims in [("c5", (6, 5, 7)), ("c2", (5, 4, 3)), ("c3", (4, 2, 2)), ("c4", (5, 3, 2))]:
    m, p = make_config(name, "perturbed", dims)
    S = FemSystem(m, p)
    sd = torch.from_numpy(make_state(name, m, p)).cuda()
    S.system(sd, scatter="tiled")
    S.residual(sd, scatter="tiled")
    if name == "c3":
        S.system(sd, scatter="stored")
    torch.cuda.synchronize()
    print(name, S.status(), flush=True)
    S.close()
