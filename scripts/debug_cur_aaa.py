import json, warnings
import numpy as np, torch
import paper_2601_22344_b200 as rp
from paper_2601_22344_b200 import rational as R
arr = np.load('tests/golden/rational.npz'); info = json.load(open('tests/golden/rational.json'))
for c in info['cases']:
    name = c['name']; z = arr[name + '_z']; f = arr[name + '_f']
    rng = rp.RngState(c['seed']); m = z.size
    perm = rng.permutation(m); half = (m + 1) // 2; xi, yi = perm[:half], perm[half:]
    L = rp.loewner_build(z[xi], f[xi], z[yi], f[yi])
    plan = rp.build_plan(z[xi], z[yi], nu=5.0)
    with warnings.catch_warnings():
        warnings.simplefilter('ignore')
        tr = rp.structured_eliminate(L, 'rplu', min(L.shape) - 1, stop_tol=c['tol'], nu=5.0,
                                     plan=plan, rng=rp.RngState(c['seed'] ^ 0x517CC1B727220A95),
                                     host_steps=False)
    print(name, 'rank', tr.rank, 'rows', list(xi[tr.row_indices]), 'cols', list(yi[tr.col_indices]))
    print('  ref cur support', c['cur_support_idx'], c['side'])
    Zd = torch.from_numpy(z).cuda(); Fd = torch.from_numpy(f).cuda()
    for side, pick in (("rows", xi[tr.row_indices]), ("cols", yi[tr.col_indices])):
        mask = np.ones(m, bool); mask[pick] = False
        P = torch.from_numpy(np.asarray(pick)).cuda(); O = torch.from_numpy(np.nonzero(mask)[0]).cuda()
        w, Lw, smin = R._loewner_weights(Zd[P], Fd[P], Zd[O], Fd[O])
        Lref = (f[mask][:, None] - f[pick][None, :]) / (z[mask][:, None] - z[pick][None, :])
        print('  ', side, 'L maxdiff', float(np.abs(Lw.cpu().numpy() - Lref).max()), 'smin', smin)
        r = rp.BarycentricRational(Zd[P], Fd[P], w)
        vals, near = r.eval_dev(Zd)
        print('  ', side, 'err', float((vals - Fd).abs().max()), 'near', int(near.sum()))
        s, Vh = np.linalg.svd(Lref)[1:]
        wr = Vh[-1].conj(); wn = w.cpu().numpy(); ph = np.vdot(wn, wr); ph /= abs(ph)
        print('   w diff vs numpy', np.abs(wn * ph - wr / np.linalg.norm(wr)).max())
