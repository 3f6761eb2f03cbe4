"""World-size-2 view sharding with gloo on CPU (the N>1 host logic).

Two ranks each take their round-robin shard of a reference step's views,
compute per-view gradients with the oracle (the per-view kernel stand-in on
CPU), pack them in the flat layout, and sum them with the same
`parallel.reduce_gradients` the GPU path uses.  The reduced buffer must equal
the single-process sum, and Adam on it must reproduce the reference's
trajectory (ref optim.py:353-407).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import NS, case_model, load_cases

GROUPS = ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _flat(g):
    return np.concatenate([np.asarray(g[k], np.float64).ravel() for k in GROUPS])


def _views(c):
    from oracle import raster as orr
    intr = NS(width=c["W"], height=c["H"], fov_y=c["fov"], near=c["near"])
    cams = [orr.camera(NS(position=p[:3], quaternion=p[3:]), intr) for p in c.a("poses")]
    return list(zip(cams, c.a("gts")))


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import raster as orr
    from paper_2604_02851_b200 import parallel
    c = load_cases("step_cases")[0]
    m = case_model(c, "init_")
    light = dict(direction=c.a("light_dir"), intensity=c.a("light_int"), ambient=c.a("ambient"))
    views = _views(c)
    mine = parallel.shard_views(views, rank, world)
    total = parallel.global_view_count(len(mine), dist.group.WORLD, torch.device("cpu"))
    grad = None
    loss = torch.zeros(1, dtype=torch.float64)
    for cam, gt in mine:
        L, g, _ = orr.backward(m, cam, light, gt, c.a("bg"))
        f = torch.from_numpy(_flat(g))
        grad = f if grad is None else grad + f
        loss += L
    parallel.reduce_gradients(grad, loss, dist.group.WORLD)
    if rank == 0:
        out.put((total, grad.numpy().copy(), float(loss.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_view_sharded_allreduce_matches_single_process_step():
    from oracle import adam as oadam
    from oracle import raster as orr
    c = load_cases("step_cases")[0]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    total, grad, loss = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert total == 3
    # single-process reference sum
    m = case_model(c, "init_")
    light = dict(direction=c.a("light_dir"), intensity=c.a("light_int"), ambient=c.a("ambient"))
    ref = None
    lsum = 0.0
    for cam, gt in _views(c):
        L, g, _ = orr.backward(m, cam, light, gt, c.a("bg"))
        ref = _flat(g) if ref is None else ref + _flat(g)
        lsum += L
    np.testing.assert_allclose(grad, ref, rtol=1e-12, atol=1e-18)
    assert abs(loss / total - c.a("losses")[0]) < 1e-12
    # Adam on the reduced buffer reproduces the reference's first step
    a, B = m.active_count, m.sh_coeffs.shape[2]
    sizes = [a * 3, a * 3, a * 4, a, a * 3 * B]
    shapes = [(a, 3), (a, 3), (a, 4), (a,), (a, 3, B)]
    parts, o = {}, 0
    for k, n, s in zip(GROUPS, sizes, shapes):
        parts[k] = grad[o:o + n].reshape(s)
        o += n
    st = oadam.AdamState(a, B, scene_extent=c["scene_extent"])
    oadam.apply(m, st, parts, total)
    for k in GROUPS:
        np.testing.assert_allclose(getattr(m, k), c.a(f"after0_{k}"), rtol=0, atol=2e-6)


def test_shard_assignment_is_a_partition():
    from paper_2604_02851_b200 import parallel
    views = list(range(8))
    for world in (1, 2, 3, 4, 8):
        shards = [parallel.shard_views(views, r, world) for r in range(world)]
        assert sorted(sum(shards, [])) == views
        assert max(map(len, shards)) - min(map(len, shards)) <= 1
