import sys; sys.path.insert(0,'.')
import numpy as np, torch
from oracle import oracle as O
from paper_2403_13806_b200.render import RasterizeOptions, render_device
from paper_2403_13806_b200.device import renderer
from paper_2403_13806_b200.synth import config2
scene, cams = config2(0, n=300_000, n_views=200)
opts = RasterizeOptions(near_limit=0.2)
v = cams[120]
out, st = render_device(scene, v, opts)
fa = renderer().frame_arrays()
ob = O.bin_tiles(scene, v, opts, np.float32)
print('P', st.n_pairs, ob['P'], 'nvis', st.n_visible)
print('ranges eq', np.array_equal(fa['ranges'], ob['ranges']))
pi = fa['pair_items']; ov = ob['vals']
print('vals eq', np.array_equal(pi, ov))
d = np.nonzero(pi != ov)[0]
print('first diffs', d[:10], len(d))
if len(d):
    k = d[0]
    t = np.searchsorted(ob['ranges'][:,1], k, side='right')
    print('tile', t, ob['ranges'][t], 'gpu', pi[max(0,k-3):k+5], 'orc', ov[max(0,k-3):k+5])
order = O.order(scene, v, opts, np.float32)
print('order eq', np.array_equal(fa['items_sorted'][:st.n_visible].astype(np.int64), order))
g = 49545
rec = fa['records'][g]
print('rec d', rec[12:16].view(np.int32), 'oracle proj', [int(O.project(scene, v, opts, np.float32)[k][g]) for k in ('x0','x1','y0','y1')])
# where does g appear
print('gpu count of g', int((pi == g).sum()), 'oracle', int((ov == g).sum()))
