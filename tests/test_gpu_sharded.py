"""The view-sharded optimize step through the product path (optim.step with a
process group), world size 2 and 3 (3 ranks over 2 views: a rank without a view), against
the single-GPU step: bit-identical.

Both ranks run on cuda:0 in separate processes with a gloo group; the
collectives are staged through host memory (parallel.Collectives), so the
ranks never wait on each other's kernels.  On an 8-GPU box the same code
runs over NCCL.  Compared after 3 steps: every parameter, the per-rank Adam
shards concatenated (moments, age, grad EMA), the losses.  With and without
a row subset, and with a view count the ranks cannot split evenly.
"""

import os
import socket

import numpy as np
import pytest

from gpu_util import require_gpu

pytestmark = pytest.mark.gpu

GROUPS = ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _scene(n_views):
    from paper_2604_02851_b200 import synth
    W, H = 320, 192
    host = synth.random_field(30_000, 3, W, H, seed=11)
    host.active_count = 29_001  # frozen tail, and shards of unequal length
    tgt = synth.target_model(host, seed=12)
    return host, tgt, synth.ring_poses(n_views, radius=0.8), synth.intrinsics(W, H), synth.light()


def _run(pg, n_views, subset, steps=3, exchange=None):
    import torch
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.optim import OptimizerState, ReferenceView, StepWorkspace, step
    from paper_2604_02851_b200.render import render_device
    host, tgt_h, poses, intr, light = _scene(n_views)
    dm = DeviceModel.from_host(host, 0)
    tgt = DeviceModel.from_host(tgt_h, 0)
    views = [ReferenceView(p, intr, render_device(tgt, p, intr, light), light, np.zeros(3)) for p in poses]
    state = OptimizerState(dm, scene_extent=2.0, process_group=pg)
    ws = StepWorkspace(dm)
    losses = [step(dm, state, views, index_subset=subset, workspace=ws, exchange=exchange) for _ in range(steps)]
    torch.cuda.synchronize()
    return (dm.to_host(), {k: v.copy() for k, v in state.m.items()}, {k: v.copy() for k, v in state.v.items()},
            state.age.copy(), state.grad_ema.copy(), losses, state.step_count)


def _worker(rank, world, port, n_views, use_subset, exchange, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    subset = _subset() if use_subset else None
    m, mm, vv, age, ema, losses, t = _run(dist.group.WORLD, n_views, subset, exchange=exchange)
    out.put((rank, {k: getattr(m, k) for k in GROUPS}, mm, vv, age, ema, losses, t))
    dist.barrier()
    dist.destroy_process_group()


def _subset():
    rng = np.random.default_rng(4)
    return np.sort(rng.choice(30_000, 21_000, replace=False))


@pytest.mark.parametrize("n_views,use_subset,exchange,world", [(4, False, "collectives", 2), (3, True, "collectives", 2),
                                                               (4, False, "p2p", 2), (3, True, "p2p", 2),
                                                               (2, False, "p2p", 3), (5, True, "p2p", 3)])
def test_gpu_sharded_step_bit_identical(n_views, use_subset, exchange, world):
    """exchange="collectives": an all-to-all of the records and an all-gather of
    the parameter rows; "p2p": the chain rule reads the peers' records from
    their memory and Adam stores every updated row into the peers' replicas
    (CUDA IPC -- here two processes on one device)."""
    require_gpu()
    import torch.multiprocessing as mp
    ref = _run(None, n_views, _subset() if use_subset else None)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_views, use_subset, exchange, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    m1, mm1, vv1, age1, ema1, l1, t1 = ref
    for rank, params, mm, vv, age, ema, losses, t in res:
        assert losses == l1, rank
        assert t == t1 == 3
        for k in GROUPS:
            np.testing.assert_array_equal(params[k], getattr(m1, k), err_msg=f"rank {rank} {k}")
    for k in GROUPS:
        np.testing.assert_array_equal(np.concatenate([x[2][k] for x in res]), mm1[k])
        np.testing.assert_array_equal(np.concatenate([x[3][k] for x in res]), vv1[k])
    np.testing.assert_array_equal(np.concatenate([x[4] for x in res]), age1)
    np.testing.assert_array_equal(np.concatenate([x[5] for x in res]), ema1)
