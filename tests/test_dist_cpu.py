"""Multi-process (gloo, world_size 2, CPU) test of the mapping step's
sharding + all-reduce logic: views are assigned round robin,
every rank accumulates its views' gradients, one SUM all-reduce combines them,
and the result equals the single-process gradient over all views.  The
per-view gradient engine here is the fp64 oracle (the CUDA path's equivalent
is tests/test_gpu_pipeline.py)."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_10070_b200 import inputs
from paper_2312_10070_b200.pipeline import shard_views


def _scene():
    s = inputs.config3(seed=9, n=300, n_views=5)
    s.cam = inputs.Camera(48, 32, 24.0, 24.0, 23.5, 15.5)
    return s


def _view_grad(orc, s, v):
    """Oracle gradient of view v's L1 colour + depth loss (lambda / V)."""
    V = s.views.shape[0]
    p64 = orc.params64(*s.params())
    tp = orc.params64(*s.extra["target_params"])
    view = s.views[v].astype(np.float64)
    tgt = orc.forward(tp, view, s.cam)
    fr = orc.forward(p64, view, s.cam)
    _, gc, gd = orc.loss(s.cam, fr["color"], fr["depth"], tgt["color"], tgt["depth"], None, 1.0 / V, 1.0 / V)
    b = orc.backward(p64, view, s.cam, fr["sorted_idx"], fr["tile_range"], gc, gd)
    return b["g3"]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    s = _scene()
    mine = shard_views(s.views.shape[0], rank, world)
    g = np.zeros((s.n, 16))
    for v in mine:
        g += _view_grad(oracle, s, v)
    t = torch.from_numpy(g)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    out[rank] = t.numpy().copy()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def test_shard_views_round_robin():
    assert shard_views(8, 0, 1) == list(range(8))
    assert shard_views(8, 1, 2) == [1, 3, 5, 7]
    assert shard_views(8, 3, 8) == [3]
    allv = sorted(v for r in range(3) for v in shard_views(8, r, 3))
    assert allv == list(range(8))


def test_gloo_two_rank_allreduce_equals_single_process(orc):
    world = 2
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, start_method="spawn", join=True)
    s = _scene()
    ref = sum(_view_grad(orc, s, v) for v in range(s.views.shape[0]))
    for r in range(world):
        assert np.allclose(out[r], ref, rtol=1e-12, atol=1e-15 * np.abs(ref).max())
