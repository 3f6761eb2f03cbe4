"""View-sharded optimize step across GPUs.

The reference sums per-view gradients and scales by 1/len(views)
(ref pkg/src/splatstream/optim.py:365-372).  On N GPUs the views are dealt
round-robin (view i to rank i % N) and every rank holds the model.  The
exchange is built on the structure of the backward pass rather than on its
output:

* a view's backward ends in per-row SCREEN-SPACE gradients (9 floats per
  visible row: colour 3, opacity 1, 2D mean 2, 2D covariance 3, plus the
  row's visibility word) -- 40 B per row per view, against the 236 B per
  row (SH degree 3) of the parameter gradient the chain rule turns them into;
* the chain rule is row-local (ref optim.py:174-268).

So the rows are split into N equal shards (ShardPlan) and the step runs

  1. per local view: K1-K6 + the partial sums -> screen-space records over
     all rows (one buffer per view slot);
  2. ONE all-to-all per slot: rank s receives, from every rank, the records
     of its own row shard for every view of the step (SH degree 3, 1M rows,
     8 GPUs: 35 MB per rank instead of a 236 MB all-reduce);
  3. the chain rule of EVERY view of the step over the rank's row shard, in
     view order (ss_chain_views_range) -- per row the same fp32 arithmetic
     in the same order as the single-GPU step, so the sharded gradient is
     bit-identical to the single-GPU one;
  4. Adam on the shard with the shard's float64 moments (ZeRO-1: 1/N of the
     optimizer state and of its HBM traffic per rank);
  5. an in-place all-gather of the updated parameter rows (one per group).

With exchange="p2p" (the default on NCCL groups) steps 2 and 5 are fused
into the kernels over peer memory (PeerWindow: every rank's record buffers
and parameter columns mapped into every rank by CUDA IPC): the chain rule
reads the other ranks' records of its rows straight from their HBM over
NVLink (no all-to-all copy), and Adam stores each updated row into every
replica as it computes it (ss_adam_step_peers); two one-element all-reduces
order the phases (records complete before any rank reads them; every
replica's rows written before any rank's next step reads them).

The per-view losses travel in a V-entry float64 vector (one all-reduce of
entries that are non-zero on exactly one rank, so exact) and are summed in
view order like the reference's `loss_sum`.

`sharded_step` is the orchestration; the compute is a `kernels` object
(optim._DeviceKernels on the GPU; the world-size-2 gloo tests in
tests/test_parallel_gloo.py drive the same orchestration with the CPU
oracle's per-row functions).  Collectives go through `Collectives`: NCCL on
the GPU box; with a gloo group, CUDA tensors are staged through host memory.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class ShardPlan:
    """Rank `rank`'s row shard of `active` rows over `world` ranks: shards of
    R = ceil(active / world) rows (the last ones may be short or empty)."""
    world: int
    rank: int
    active: int

    @property
    def R(self) -> int:
        return -(-self.active // self.world) if self.active > 0 else 0

    @property
    def row0(self) -> int:
        return min(self.rank * self.R, self.active)

    @property
    def rows(self) -> int:
        return max(0, min(self.row0 + self.R, self.active) - self.row0)

    @property
    def padded(self) -> int:
        return self.world * self.R

    def shard(self, rank: int) -> "ShardPlan":
        return ShardPlan(self.world, rank, self.active)


def shard_views(views, rank: int, world: int):
    """The views rank `rank` renders: rank, rank+world, ..."""
    return list(views)[rank::world]


def view_slot(t: int, world: int):
    """(owner rank, slot) of the t-th view of a batch."""
    return t % world, t // world


class Collectives:
    """The step's collectives over a torch.distributed group."""

    def __init__(self, group):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.host_staged = dist.get_backend(group) == "gloo"

    def _staged(self, t):
        return t.cpu() if (self.host_staged and t.is_cuda) else t

    def all_to_all(self, out, inp):
        """Equal splits along dim 0 (world chunks): chunk s of inp goes to
        rank s, chunk s of out comes from rank s."""
        o, i = self._staged(out), self._staged(inp)
        self.dist.all_to_all_single(o, i, group=self.group)
        if o is not out:
            out.copy_(o)

    def barrier(self):
        """A device-ordered barrier: a one-element all-reduce on the stream
        (work queued after it starts only once every rank reached it)."""
        import torch
        t = getattr(self, "_tick", None)
        if t is None:
            dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
            t = self._tick = torch.zeros(1, dtype=torch.int32, device=dev)
        self.all_reduce_(t)

    def all_reduce_(self, t, op="sum"):
        s = self._staged(t)
        self.dist.all_reduce(s, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM,
                             group=self.group)
        if s is not t:
            t.copy_(s)

    def all_gather_rows(self, full, R: int):
        """In place: rows [rank*R, (rank+1)*R) of `full` (dim 0, >= world*R
        rows) from every rank into rows [0, world*R)."""
        out = full[: self.world * R]
        if self.host_staged:
            o = out.cpu() if out.is_cuda else out
            self.dist.all_gather_into_tensor(o, o[self.rank * R:(self.rank + 1) * R].clone(), group=self.group)
            if o is not out:
                out.copy_(o)
        else:  # NCCL gathers in place when the input is the rank's own slice of the output
            self.dist.all_gather_into_tensor(out, out[self.rank * R:(self.rank + 1) * R], group=self.group)


_PEER_OK = {}


def peer_access_ok(group) -> bool:
    """Whether every rank's GPU can map every other rank's memory (CUDA
    peer access; the same device counts): the default exchange is "p2p"
    only then.  Decided once per group, identically on every rank."""
    import torch
    import torch.distributed as dist
    key = id(group)
    if key not in _PEER_OK:
        me = torch.cuda.current_device()
        devs = [None] * dist.get_world_size(group)
        dist.all_gather_object(devs, me, group=group)
        ok = all(d == me or torch.cuda.can_device_access_peer(me, d) for d in devs)
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=torch.device("cuda", me))
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        _PEER_OK[key] = bool(int(flag.item()))
    return _PEER_OK[key]


class PeerWindow:
    """Other ranks' device tensors mapped into this process (CUDA IPC; on an
    NVSwitch box the mapped addresses are the peers' HBM over NVLink): each
    rank shares `tensors` (name -> CUDA tensor) once, every rank gets every
    rank's tensors.  `key` identifies the shared buffers (re-share when a
    buffer is reallocated; every rank reallocates at the same step)."""

    def __init__(self, group, tensors: dict):
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        mine = {k: reduce_tensor(t) for k, t in tensors.items()}
        objs = [None] * self.world
        dist.all_gather_object(objs, mine, group=group)
        self.peers = []
        for r, o in enumerate(objs):
            if r == self.rank:
                self.peers.append(dict(tensors))
            else:
                self.peers.append({k: fn(*args) for k, (fn, args) in o.items()})
        self.key = self.key_of(tensors)

    @staticmethod
    def key_of(tensors: dict):
        return tuple((k, int(t.data_ptr()), tuple(t.shape)) for k, t in sorted(tensors.items()))


def padded_rows_view(t, rows: int):
    """t (dim 0 >= rows) as its first `rows` rows, or a zero-padded copy and a
    write-back callback when t is shorter (all_gather_rows needs world*R rows)."""
    import torch
    if t.shape[0] >= rows:
        return t[:rows], None
    pad = torch.zeros((rows,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]].copy_(t)
    return pad, (lambda: t.copy_(pad[: t.shape[0]]))


def sharded_step(kern, views, plan: ShardPlan, coll=None, batch: int = 16):
    """One optimizer step over `views` (every rank passes the same ready
    list) on this rank; returns the mean loss as the kernels' scalar.

    kern: records(n_slots) -> per-slot record sets; backward(view, slot_recs,
    loss_index); invisible(slot_recs); exchange(coll, send) -> recv;
    chain_batch(views, recs_of_view); losses / sum_losses(coll); adam(n_views);
    gather(coll).  See optim._DeviceKernels."""
    V = len(views)
    N = plan.world
    for b0 in range(0, V, batch):
        idx = list(range(b0, min(V, b0 + batch)))
        slots = -(-len(idx) // N)
        send = kern.records(slots)
        used = set()
        for t, i in enumerate(idx):
            owner, slot = view_slot(t, N)
            if owner == plan.rank:
                kern.backward(views[i], send[slot], i)
                used.add(slot)
        for k in range(slots):
            if k not in used:  # a rank with fewer views than the busiest: nothing visible
                kern.invisible(send[k])
        join = getattr(kern, "join", None)
        if join is not None:  # the backward passes may run on several streams
            join()
        if N > 1:
            recv = kern.exchange(coll, send)
            recs = [kern.shard_view(recv[view_slot(t, N)[1]], view_slot(t, N)[0]) for t in range(len(idx))]
        else:
            recs = [send[t] for t in range(len(idx))]
        kern.chain_batch([views[i] for i in idx], recs)
    loss = kern.sum_losses(coll if N > 1 else None)
    kern.adam(V)
    if N > 1:
        kern.gather(coll)
    return loss
