import sys
import numpy as np
import torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from fem_inputs import make_config, make_state
from paper_2111_03541_b200 import FemSystem
from paper_2111_03541_b200.partition import partition_nodes
m, p = make_config('c5', 'structured', (7, 5, 6))
st = make_state('c5', m, p)
for part in partition_nodes(m, 3):
    pm = part.mesh
    S = FemSystem(pm, p, own=part.own)
    sd = torch.from_numpy(part.local_state(st)).cuda()
    v1, r1 = [x.clone() for x in S.system(sd, scatter='coloured')]
    S.values.fill_(float('nan')); S.rhs.fill_(float('nan'))
    v2, r2 = S.system(sd, scatter='tiled')
    torch.cuda.synchronize()
    v1, v2, r1, r2 = [x.cpu().numpy() for x in (v1, v2, r1, r2)]
    n_own = part.n_owned
    lat = np.round(pm.coords * np.array([[7], [5], [6]])).astype(int)
    badr = np.nonzero(~np.isclose(r1, r2, rtol=1e-12, atol=1e-14 * np.abs(r1).max()))[0]
    print('part', part.rank, 'own', n_own, 'local', pm.n_nodes, 'bad rhs rows', len(badr), 'of', len(r1))
    pat = S.export_pattern(slot=False)
    rp = pat['rowptr'].cpu().numpy()
    badrows = set()
    for r in range(len(rp) - 1):
        a, b = rp[r], rp[r + 1]
        if not np.allclose(v1[a:b], v2[a:b], rtol=1e-12, atol=1e-14 * np.abs(v1).max(), equal_nan=False):
            badrows.add(r % n_own)
    nodes = sorted(set(badrows) | set(int(x) % n_own for x in badr))
    print('  bad nodes', len(nodes), [tuple(lat[:, n]) for n in nodes[:20]])
    own_lat = lat[:, :n_own]
    print('  owned box', own_lat.min(axis=1), own_lat.max(axis=1))
    S.close()
