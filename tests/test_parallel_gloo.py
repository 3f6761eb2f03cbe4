"""The view-sharded step's host logic on CPU, world sizes 2 and 3 over gloo.

`parallel.sharded_step` -- the orchestration optim.step runs on N GPUs
(view slots, the all-to-all of per-row screen-space records, the chain rule
of every view over the rank's row shard in view order, the sharded Adam, the
in-place all-gather of parameter rows, the exact per-view loss sum) -- is
driven here with the CPU oracle's per-view functions standing in for the
kernels (oracle/raster.py screen_grads / chain_rule, oracle/adam.py).  The
N-rank result must be BIT-IDENTICAL to the same kernels at N = 1 (parameters,
losses, and the concatenated Adam shards), and follow the reference's
trajectory (tests/golden step_cases, ref optim.py:353-407).

The sharded OptimizerState bookkeeping (ZeRO-1 shards, resize by gathering,
remapping and re-splitting, device_stats) runs on CPU tensors with gloo and
must equal the unsharded state after the same records.
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


def _case_views(c):
    from oracle import raster as orr
    intr = NS(width=c["W"], height=c["H"], fov_y=c["fov"], near=c["near"])
    return [(orr.camera(NS(position=p[:3], quaternion=p[3:]), intr), gt) for p, gt in zip(c.a("poses"), c.a("gts"))]


class OracleKernels:
    """parallel.sharded_step's kernel interface on the CPU oracle (float64)."""

    def __init__(self, model, light, bg, adam_state, plan, n_views):
        self.m, self.light, self.bg, self.st, self.plan = model, light, bg, adam_state, plan
        self.n = model.means.shape[0]
        self.B = model.sh_coeffs.shape[2]
        self.losses = torch.zeros(n_views, dtype=torch.float64)
        self.grad = None
        self.rows_alloc = max(self.n, plan.padded)

    def records(self, slots):
        return [(torch.zeros((self.rows_alloc, 9), dtype=torch.float64),
                 torch.full((self.rows_alloc,), -1, dtype=torch.int32)) for _ in range(slots)]

    def backward(self, view, rec, i):
        from oracle import raster as orr
        cam, gt = view
        prep = orr.prepare(self.m, cam, self.light, None, True)
        img, _, _ = orr.composite(prep, cam["W"], cam["H"], self.bg)
        gt = np.asarray(gt, np.float64)
        self.losses[i] = float(np.mean(np.abs(img - gt)))
        gc, go, gm, gs = orr.screen_grads(prep, img, gt, cam["W"], cam["H"])
        rows = prep["rows"]
        g = np.concatenate([gc, go[:, None], gm, gs], axis=1)
        rec[0][torch.from_numpy(rows)] = torch.from_numpy(g)
        rec[1][torch.from_numpy(rows)] = 1

    def invisible(self, rec):
        rec[1].fill_(-1)

    def exchange(self, coll, send):
        P = self.plan.padded
        out = []
        for g, v in send:
            rg = torch.empty((P, 9), dtype=g.dtype)
            rv = torch.empty(P, dtype=v.dtype)
            coll.all_to_all(rg, g[:P].contiguous())
            coll.all_to_all(rv, v[:P].contiguous())
            out.append((rg, rv))
        return out

    def shard_view(self, rec, s):
        R = self.plan.R
        return rec[0][s * R:(s + 1) * R], rec[1][s * R:(s + 1) * R], self.plan.row0

    def chain_batch(self, views, recs):
        from oracle import raster as orr
        p = self.plan
        a = int(self.m.active_count)
        if self.grad is None:
            self.grad = dict(means=np.zeros((p.rows, 3)), log_scales=np.zeros((p.rows, 3)),
                             quaternions=np.zeros((p.rows, 4)), logit_opacities=np.zeros(p.rows),
                             sh_coeffs=np.zeros((p.rows, 3, self.B)))
        for (cam, _), rec in zip(views, recs):
            if len(rec) == 2:  # N = 1: records indexed by row
                g, vis, base = rec[0], rec[1], 0
            else:
                g, vis, base = rec
            # the chain rule is row-local: evaluate the view's prep over its
            # visible rows and keep this shard's rows (the prep rows of the
            # single-rank run, so each row's arithmetic is identical)
            prep = orr.prepare(self.m, cam, self.light, None, True)
            rows = prep["rows"]
            mine = (rows >= p.row0) & (rows < p.row0 + p.rows) & (rows < a)
            sg = np.zeros((rows.size, 9))
            sel = rows[mine] - base
            assert (vis[torch.from_numpy(sel)] == 1).all()
            sg[mine] = g[torch.from_numpy(sel)].numpy()
            per = orr.chain_rule(prep, cam, self.light, sg[:, :3], sg[:, 3], sg[:, 4:6], sg[:, 6:9])
            for k in GROUPS:
                self.grad[k][rows[mine] - p.row0] += per[k][mine]

    def sum_losses(self, coll):
        if coll is not None:
            coll.all_reduce_(self.losses)
        t = 0.0
        for x in self.losses.tolist():
            t += x
        return t

    def adam(self, n_views):
        from oracle import adam as oadam
        p = self.plan
        sl = slice(p.row0, p.row0 + p.rows)
        view = NS(**{k: getattr(self.m, k)[sl] for k in GROUPS}, active_count=p.rows)
        oadam.apply(view, self.st, self.grad, n_views)
        self.grad = None

    def gather(self, coll):
        from paper_2604_02851_b200 import parallel
        for k in GROUPS:
            t = torch.from_numpy(getattr(self.m, k))
            v, wb = parallel.padded_rows_view(t, self.plan.padded)
            coll.all_gather_rows(v, self.plan.R)
            if wb is not None:
                wb()


def _run(c, world, rank, coll, steps, n_views):
    from oracle import adam as oadam
    from paper_2604_02851_b200 import parallel
    m = case_model(c, "init_")
    light = dict(direction=c.a("light_dir"), intensity=c.a("light_int"), ambient=c.a("ambient"))
    views = _case_views(c)[:n_views]
    plan = parallel.ShardPlan(world, rank, int(m.active_count))
    st = oadam.AdamState(plan.rows, m.sh_coeffs.shape[2], scene_extent=c["scene_extent"])
    losses = []
    for _ in range(steps):
        kern = OracleKernels(m, light, c.a("bg"), st, plan, len(views))
        L = parallel.sharded_step(kern, views, plan, coll)
        losses.append(L / len(views))
    return m, st, losses


def _worker(rank, world, port, n_views, case, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_02851_b200 import parallel
    c = load_cases("step_cases")[case]
    coll = parallel.Collectives(dist.group.WORLD)
    m, st, losses = _run(c, world, rank, coll, 2, n_views)
    out.put((rank, {k: getattr(m, k).copy() for k in GROUPS},
             {k: st.m[k].copy() for k in GROUPS}, {k: st.v[k].copy() for k in GROUPS},
             st.age.copy(), st.grad_ema.copy(), losses))
    dist.barrier()
    dist.destroy_process_group()


def _spawn(world, n_views, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_views, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world,n_views,case", [(2, 3, 1), (3, 2, 0)])
def test_sharded_step_bit_identical_to_single_rank(world, n_views, case):
    """2 ranks over 3 views (uneven slots; degree 3, 31 active of 40 rows) and
    3 ranks over 2 views (a rank with no view; 40 rows in shards of 14, so the
    parameter gather runs through a padded copy)."""
    c = load_cases("step_cases")[case]
    m1, st1, l1 = _run(c, 1, 0, None, 2, n_views)
    res = _spawn(world, n_views, case)
    for r, params, mm, vv, age, ema, losses in res:
        assert losses == l1  # exact: per-view losses summed in view order
        for k in GROUPS:
            np.testing.assert_array_equal(params[k], getattr(m1, k), err_msg=f"rank {r} {k}")
    # the Adam shards concatenate to the single-rank state, bit for bit
    for k in GROUPS:
        np.testing.assert_array_equal(np.concatenate([x[2][k] for x in res]), st1.m[k])
        np.testing.assert_array_equal(np.concatenate([x[3][k] for x in res]), st1.v[k])
    np.testing.assert_array_equal(np.concatenate([x[4] for x in res]), st1.age)
    np.testing.assert_array_equal(np.concatenate([x[5] for x in res]), st1.grad_ema)


def test_sharded_orchestration_follows_reference_trajectory():
    c = load_cases("step_cases")[1]
    m, _, losses = _run(c, 1, 0, None, 2, 3)
    for it in range(2):
        assert abs(losses[it] - c.a("losses")[it]) < 1e-12
    for k in GROUPS:
        np.testing.assert_allclose(getattr(m, k), c.a(f"after1_{k}"), rtol=0, atol=2e-6)


def _state_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out.put((rank, _state_script(dist.group.WORLD)))
    dist.barrier()
    dist.destroy_process_group()


def _state_script(pg):
    """OptimizerState on CPU tensors: fill, resize through the reference's
    three record kinds, report the full state (gathered when sharded)."""
    from paper_2604_02851_b200.optim import OptimizerState
    rng = np.random.default_rng(3)
    a, B = 13, 4
    model = NS(active_count=a, sh_degree=1)
    st = OptimizerState(model, device="cpu", process_group=pg)
    full_m = {k: rng.normal(size=s) for k, s in
              dict(means=(a, 3), log_scales=(a, 3), quaternions=(a, 4), logit_opacities=(a,),
                   sh_coeffs=(a, 3, B)).items()}
    full_v = {k: np.abs(rng.normal(size=x.shape)) for k, x in full_m.items()}
    age = rng.integers(0, 50, a)
    ema = rng.random(a)
    p = st.plan if pg is not None else None
    sl = slice(p.row0, p.row0 + p.rows) if p is not None else slice(0, a)
    for k in full_m:  # the reference-visible numpy views, written back on the next device use
        st.m[k][...] = full_m[k][sl]
        st.v[k][...] = full_v[k][sl]
    st.age[...] = age[sl]
    st.grad_ema[...] = ema[sl]

    class PermuteRecord:
        def __init__(self, permutation, new_active_count):
            self.permutation, self.new_active_count = permutation, new_active_count

    class AppendRecord:
        def __init__(self, insert_at, count):
            self.insert_at, self.count = insert_at, count

    class PruneRecord:
        def __init__(self, indices):
            self.indices = indices

    st.resize(PermuteRecord(np.array([0, 2, 4, 6, 8, 10, 12, 1, 3, 5, 7, 9, 11]), 9))
    st.resize(AppendRecord(9, 6))
    st.resize(PruneRecord(np.array([1, 4, 14, 20])))
    m, v, age_d, ema_d = st._full()
    return ({k: t.numpy().copy() for k, t in m.items()}, {k: t.numpy().copy() for k, t in v.items()},
            age_d.numpy().copy(), ema_d.numpy().copy(), st.active_count)


def test_sharded_optimizer_state_resize_matches_unsharded():
    ref = _state_script(None)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_state_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ref[4] == 12
    for _, got in res:
        assert got[4] == ref[4]
        for k in GROUPS:
            np.testing.assert_array_equal(got[0][k], ref[0][k])
            np.testing.assert_array_equal(got[1][k], ref[1][k])
        np.testing.assert_array_equal(got[2], ref[2])
        np.testing.assert_array_equal(got[3], ref[3])


def test_shard_plan_partitions_rows_and_views():
    from paper_2604_02851_b200 import parallel
    for a in (0, 1, 7, 40, 1000):
        for world in (1, 2, 3, 8):
            plans = [parallel.ShardPlan(world, r, a) for r in range(world)]
            covered = np.concatenate([np.arange(p.row0, p.row0 + p.rows) for p in plans]) if a else np.array([])
            np.testing.assert_array_equal(covered, np.arange(a))
            assert all(p.padded >= a and p.padded == world * p.R for p in plans)
    views = list(range(8))
    for world in (1, 2, 3, 4, 8):
        shards = [parallel.shard_views(views, r, world) for r in range(world)]
        assert sorted(sum(shards, [])) == views
        assert max(map(len, shards)) - min(map(len, shards)) <= 1
