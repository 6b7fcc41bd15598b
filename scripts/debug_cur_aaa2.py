import json, warnings, pickle
import numpy as np, torch
import paper_2601_22344_b200 as rp
from paper_2601_22344_b200.cauchy import tree_bounds_device
ref = pickle.load(open('scripts/tmp_ref_trace.pkl', 'rb'))
arr = np.load('tests/golden/rational.npz'); info = json.load(open('tests/golden/rational.json'))
for c in info['cases']:
    name = c['name']; z = arr[name + '_z']; f = arr[name + '_f']
    rng = rp.RngState(c['seed']); m = z.size
    perm = rng.permutation(m); half = (m + 1) // 2; xi, yi = perm[:half], perm[half:]
    L = rp.loewner_build(z[xi], f[xi], z[yi], f[yi])
    plan = rp.build_plan(z[xi], z[yi], nu=5.0)
    u0 = tree_bounds_device(plan, L).cpu().numpy()
    R = ref[name]
    print(name, 'u0 rel diff', np.max(np.abs(u0 - R['u0']) / np.maximum(R['u0'], 1e-300)), u0.max(), R['u0'].max())
    with warnings.catch_warnings():
        warnings.simplefilter('ignore')
        tr = rp.structured_eliminate(L, 'rplu', min(L.shape) - 1, stop_tol=c['tol'], nu=5.0,
                                     plan=plan, rng=rp.RngState(c['seed'] ^ 0x517CC1B727220A95),
                                     host_steps=False)
    print('  rows', tr.row_indices[:6], R['rows'][:6])
    print('  props', tr.proposals, R['prop'], tr.acceptances, R['acc'], tr.exact_fallbacks, R['fb'])
    print('  bmax', tr.bound_maxes[:4], R['bmax'][:4])
