import sys; sys.path.insert(0,'.')
import numpy as np, torch
from oracle import oracle as O
from paper_2403_13806_b200.render import RasterizeOptions, render_device
from paper_2403_13806_b200.synth import config2
scene, cams = config2(0, n=300_000, n_views=200)
opts = RasterizeOptions(near_limit=0.2)
for v in cams[::40]:
    a = torch.zeros(len(scene), device='cuda'); b = torch.zeros(len(scene), device='cuda')
    _, st = render_device(scene, v, opts, color=False, scores=a)
    out, st2 = render_device(scene, v, opts, color=True, scores=b)
    ref = O.views(scene, [v], opts, np.float32, scores=True, images=True)
    ga, gb = a.cpu().numpy(), b.cpu().numpy()
    r = ref['contrib']
    print('view', st.n_pairs, st.overflow, 'score-only mism', int((ga != r).sum()), 'color+score mism', int((gb != r).sum()),
          'img', int((out['rgb'].cpu().numpy() != ref['img_last']).sum()))
    bad = np.nonzero(ga != r)[0][:5]
    print('  ', bad, ga[bad], gb[bad], r[bad])
