"""Dev A/B: time a config's tiled system call with and without its boundary terms (facet phase cost).
python tools/time_variants.py [config] [dims...]"""
import sys
import torch
sys.path.insert(0, '.')
from fem_inputs import make_config, make_state
from paper_2111_03541_b200 import FemSystem

name = sys.argv[1] if len(sys.argv) > 1 else 'c5'
dims = tuple(int(x) for x in sys.argv[2:]) or None
m, p = make_config(name, 'structured', dims)
st = torch.from_numpy(make_state(name, m, p)).cuda()
for label, terms in [('all terms', p.terms), ('domain only', p.terms[:1])]:
    p.terms = terms
    S = FemSystem(m, p)
    for _ in range(3): S.system(st, scatter='tiled')
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(10): S.system(st, scatter='tiled')
    e[1].record(); torch.cuda.synchronize()
    print(f'{label:12s} {e[0].elapsed_time(e[1]) / 10:8.3f} ms', flush=True)
    S.close()
