"""Two ranks on one GPU (gloo over CUDA tensors): the sharded product paths --
compute_importance(shard=True) (views split + MAX all-reduce, pruning.py:80-92)
and bake_visibility(shard=True) (clusters split + bitset all-gather,
visibility.py:175-210) -- give bit-identical results to one rank.

The ranks never wait on each other inside a kernel (the collectives are host-side
gloo), so sharing one GPU is safe here; NCCL's multi-GPU runs use the same code."""
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q, prec):
    import os
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    import torch
    import torch.distributed as dist

    from conftest import golden, load_cam
    from paper_2403_13806_b200.core import GaussianScene
    from paper_2403_13806_b200.pruning import compute_importance
    from paper_2403_13806_b200.render import RasterizeOptions
    from paper_2403_13806_b200.synth import config2
    from paper_2403_13806_b200.visibility import bake_visibility, cluster_cameras

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        opts = RasterizeOptions(near_limit=0.2, precision=prec)
        scene, cams = config2(0, n=80_000, n_views=9)
        shard = compute_importance(scene, cams, opts, shard=True)
        local = compute_importance(scene, cams, opts)  # the whole camera list on this rank
        d = golden("two_room")
        p = "room5_"
        room = GaussianScene(positions=d[p + "pos"], opacity_logits=d[p + "logit"], sh=d[p + "sh"],
                             log_scales=d[p + "ls"], quaternions=d[p + "quat"], active_sh_degree=int(d[p + "deg"]))
        rcams = [load_cam(d, f"{p}cam{i}_") for i in range(int(d[p + "n_cams"]))]
        cl = cluster_cameras(np.array([c.center for c in rcams]), k=3, seed=0)
        vs = bake_visibility(room, cl, rcams, t_cluster=0.001, aux_per_camera=2, seed=0, options=opts, shard=True)
        vl = bake_visibility(room, cl, rcams, t_cluster=0.001, aux_per_camera=2, seed=0, options=opts)
        q.put((rank, shard.values.tobytes(), local.values.tobytes(), vs.indicators.tobytes(),
               vl.indicators.tobytes(), int((shard.values > 0).sum())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_sharded_scoring_and_bake_two_ranks_equal_one(prec):
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, prec)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, shard, local, vs, vl, nz in res:
        assert shard == local, rank  # MAX merge of two view shards == all views on one rank
        assert vs == vl, rank        # gathered cluster bitsets == baking every cluster locally
        assert nz > 0
    assert res[0][1] == res[1][1] and res[0][3] == res[1][3]
