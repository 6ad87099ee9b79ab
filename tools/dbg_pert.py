import sys, time
import torch
sys.path.insert(0, '.')
from fem_inputs import make_config, make_state
from paper_2111_03541_b200 import FemSystem
dims = tuple(int(x) for x in sys.argv[1:]) or None
m, p = make_config('c5', 'perturbed', dims)
t0 = time.time(); S = FemSystem(m, p); torch.cuda.synchronize()
print('pattern', time.time() - t0, S.info(), flush=True)
sd = torch.from_numpy(make_state('c5', m, p)).cuda()
for _ in range(3): S.system(sd, scatter='tiled')
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
torch.cuda.synchronize(); ev[0].record()
for _ in range(5): S.system(sd, scatter='tiled')
ev[1].record(); torch.cuda.synchronize()
print('ms', ev[0].elapsed_time(ev[1]) / 5, S.status())
