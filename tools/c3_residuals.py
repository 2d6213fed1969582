import sys, numpy as np
sys.path.insert(0, '.')
import paper_1203_4031_b200 as fb
from paper_1203_4031_b200 import workloads as W
w = W.c3_heev()
r = fb.feast_he(w.a, w.emin, w.emax, w.m0, fpm=w.fpm())
g = np.load('tests/golden/full_c3.npz')
print('gpu', r.info, r.m0, r.loop, r.m, 'ref scal', g['scal'])
i = np.argsort(-r.res[:r.m])[:6]
print('worst gpu res', [(round(r.e[k], 6), '%.1e' % r.res[k]) for k in i])
print('ref res at same e', ['%.1e' % g['res'][k] for k in i] if 'res' in g.files else g.files)
print('gpu median res %.1e' % np.median(r.res[:r.m]))
