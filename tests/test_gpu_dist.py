"""S8 on its product path (the mapping loss sums
over the keyframes of the sub-map, so views shard across ranks and one SUM
all-reduce of the gradient buffer combines them).

Two processes on the one GPU, each running ``MapStep(rank, world=2)`` with its
DEFAULT all-reduce (``torch.distributed.all_reduce`` on the gradient buffer;
the process group is gloo here because the box has one GPU — gloo reduces the
CUDA tensor through the host, no kernel of one rank waits on the other).
Every rank's result must equal the fp64 oracle's all-view gradient under R23.
A second test makes only rank 0 overflow its pair capacity: the collective
repeat decision of ``step_checked`` must make both ranks re-size and repeat,
so the all-reduces stay paired and the result is still the oracle's.  A third
runs ``bench.py``'s WORLD_SIZE > 1 branch (rank-MAX timing, e2e across ranks)
under torchrun with ``--backend gloo``."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from gpu_helpers import grad_check, oracle_mapping_reference, small_submap

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEED = 8


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _worker(rank, world, port, data_path, out_dir, mode):
    import torch.distributed as dist

    from gpu_helpers import grads_as_g3, zero_upstream_hook
    from paper_2312_10070_b200 import Params
    from paper_2312_10070_b200.pipeline import MapStep
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    d = torch.device("cuda", 0)
    ref = np.load(data_path)
    s = small_submap(seed=SEED)
    V = s.views.shape[0]
    P = Params.from_numpy(*s.params(), device=d)
    views = torch.as_tensor(s.views, device=d)
    tc = {v: torch.as_tensor(ref["tc"][v], device=d) for v in range(V)}
    td = {v: torch.as_tensor(ref["td"][v], device=d) for v in range(V)}
    amb = {v: torch.as_tensor(ref["amb"][v], device=d) for v in range(V)}
    ms = MapStep(P, views, s.cam, tc, td, rank=rank, world=world, device=d,  # default all-reduce
                 ar_chunks=3 if mode == "chunked" else None)
    ms.size()
    if mode == "overflow" and rank == 0:
        for r in ms.lanes:
            r.capacity = 1000  # far below the pair count: this rank's views overflow
    steps = []
    step = ms.step

    def counted(*a, **k):
        steps.append(1)
        return step(*a, **k)
    ms.step = counted
    g = ms.step_checked(hooks={"bwd": zero_upstream_hook(ms, amb)})
    torch.cuda.synchronize()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), g3=grads_as_g3(g), loss=ms.losses.cpu().numpy(),
             mine=np.array(ms.mine), steps=len(steps))
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def reference(tmp_path_factory):
    s = small_submap(seed=SEED)
    ref = oracle_mapping_reference(s)
    V = s.views.shape[0]
    path = str(tmp_path_factory.mktemp("s8") / "ref.npz")
    np.savez(path, tc=np.stack([ref["tc"][v] for v in range(V)]), td=np.stack([ref["td"][v] for v in range(V)]),
             amb=np.stack([ref["amb"][v] for v in range(V)]))
    return ref, path


def _run(reference, tmp_path, mode):
    ref, path = reference
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), path, str(tmp_path), mode), nprocs=world,
                       start_method="spawn", join=True)
    out = [dict(np.load(os.path.join(tmp_path, f"rank{r}.npz"))) for r in range(world)]
    for r in range(world):
        ok, st = grad_check(out[r]["g3"], ref["g3"], ref["m3"])
        assert ok.all(), (mode, r, st)
        mine = out[r]["mine"]
        assert np.array_equal(mine, np.arange(r, 4, world))
        assert np.allclose(out[r]["loss"][:len(mine), :3], ref["loss"][mine], rtol=1e-6, atol=0)
    return out


def test_two_rank_mapstep_allreduce_equals_oracle(reference, tmp_path):
    out = _run(reference, tmp_path, "plain")
    assert all(o["steps"] == 1 for o in out)
    assert np.array_equal(out[0]["g3"], out[1]["g3"])  # one SUM: every rank holds the same buffer


def test_chunked_allreduce_equals_oracle(reference, tmp_path):
    """ar_chunks = 3: S6 in three Gaussian ranges, each range all-reduced (its
    four component slices) on the communication stream after every view
    chained it: the same summed gradient."""
    out = _run(reference, tmp_path, "chunked")
    assert np.array_equal(out[0]["g3"], out[1]["g3"])


def test_overflow_on_one_rank_repeats_on_every_rank(reference, tmp_path):
    out = _run(reference, tmp_path, "overflow")
    assert all(o["steps"] == 2 for o in out)  # the collective decision: both ranks repeated


def test_bench_two_ranks_gloo(tmp_path):
    """bench.py's WORLD_SIZE > 1 branch: per-rank views, the gradient
    all-reduce inside the timed step, MAX over ranks of the step time and of
    the end-to-end step, one JSON line from rank 0."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--backend", "gloo", "--steps", "2", "--warmup", "3", "--small"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["views_per_rank"] == 2 and line["value"] > 0
    assert line["e2e"]["value"] > 0 and "GLOO" in line["config"]["parallelism"]
