"""Run a few assembly calls of one config/mode (for ncu captures): python tools/run_once.py c5 tiled system 3 [dims]"""
import sys
import torch
sys.path.insert(0, '.')
from fem_inputs import make_config, make_state
from paper_2111_03541_b200 import FemSystem
name, mode, what, reps = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
dims = tuple(int(x) for x in sys.argv[5:]) or None
m, p = make_config(name, 'structured', dims)
S = FemSystem(m, p)
sd = torch.from_numpy(make_state(name, m, p)).cuda()
for _ in range(reps):
    getattr(S, what)(sd, scatter=mode)
torch.cuda.synchronize()
print('ok', S.status())
