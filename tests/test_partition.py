"""Host-side logic of the multi-GPU path (-m "not gpu"): edge-balanced
1-D partition boundaries, and the N>1 setup (NCCL unique id distributed out
of band, every rank computing the same partition) on world_size 2 with the
gloo backend."""
import os
import socket

import numpy as np
import pytest

import graphgen as gg
import oracle


def _fb():
    import paper_1903_01665_b200 as fb
    from paper_1903_01665_b200 import _build
    _build.build()
    fb.load()
    return fb


def _check_bounds(row_off, P, b):
    n = len(row_off) - 1
    m = int(row_off[-1])
    assert b[0] == 0 and b[-1] == n and len(b) == P + 1
    assert (np.diff(b) >= 0).all()
    deg = np.diff(row_off.astype(np.int64))
    dmax = int(deg.max()) if n else 0
    arcs = row_off[b[1:]].astype(np.int64) - row_off[b[:-1]].astype(np.int64)
    assert arcs.sum() == m
    assert (np.abs(arcs - m / P) <= dmax + 1).all(), (arcs, m / P, dmax)


@pytest.mark.parametrize("name", ["tiny", "rand-s", "rmat-s", "grid-s"])
@pytest.mark.parametrize("P", [1, 2, 3, 8, 64])
def test_partition_edge_balanced(name, P):
    fb = _fb()
    g = gg.config(name)
    _check_bounds(g.row_off, P, fb.falcon_partition(g.row_off, P))


def test_partition_small_cases():
    fb = _fb()
    ro = np.array([0, 2, 3, 3, 10, 10, 12], np.uint32)
    b = fb.falcon_partition(ro, 3)
    _check_bounds(ro, 3, b)
    assert b.tolist() == [0, 3, 4, 6]   # nearest prefix: 3 | 7 | 2 arcs
    ro = np.zeros(5, np.uint32)         # no arcs: everything on one side, still a cover
    _check_bounds(ro, 4, fb.falcon_partition(ro, 4))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fb = _fb()
    g = gg.config("rmat-s")
    # the NCCL unique id is created on rank 0 and shipped out of band
    obj = [fb.falcon_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    b = fb.falcon_partition(g.row_off, world)
    lo, hi = int(b[rank]), int(b[rank + 1])
    gathered = [None] * world
    dist.all_gather_object(gathered, (obj[0], b.tolist(), lo, hi))
    q.put((rank, gathered))
    dist.destroy_process_group()


def test_gloo_world2_setup():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        g = res[r]
        uids = {x[0] for x in g}
        assert len(uids) == 1 and len(next(iter(uids))) == 128   # one id everywhere
        bounds = {tuple(x[1]) for x in g}
        assert len(bounds) == 1                                   # same partition everywhere
        ranges = sorted((x[2], x[3]) for x in g)
        n = ranges[-1][1]
        assert ranges[0][0] == 0 and ranges[0][1] == ranges[1][0] and n == gg.config("rmat-s").n


def _worker_exchange(rank, world, port, q):
    """Each rank owns one slice of falcon_partition's bounds, relaxes only its
    own rows (numpy, test infrastructure) and exchanges its proposals with a
    real all-reduce(MIN) over gloo each superstep; termination by all-reduce
    (SUM) of `changed` -- the superstep structure of the dense exchange
    (DESIGN.md §7), on CPU."""
    import numpy as np
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fb = _fb()
    g = gg.config("rand-s")
    b = fb.falcon_partition(g.row_off, world)
    lo, hi = int(b[rank]), int(b[rank + 1])
    base, top = int(g.row_off[lo]), int(g.row_off[hi])
    src = np.repeat(np.arange(lo, hi, dtype=np.int64), np.diff(g.row_off[lo:hi + 1].astype(np.int64)))
    dst = g.col[base:top].astype(np.int64)
    w = g.w[base:top].astype(np.int64)
    INF = 2147483647
    d = torch.full((g.n,), INF, dtype=torch.int64)
    d[g.source] = 0
    steps = 0
    while True:
        steps += 1
        dv = d.numpy()
        ok = dv[src] < INF
        prop = np.full(g.n, INF, np.int64)
        np.minimum.at(prop, dst[ok], dv[src[ok]] + w[ok])
        new = torch.minimum(d, torch.from_numpy(prop))
        dist.all_reduce(new, op=dist.ReduceOp.MIN)          # the boundary exchange
        changed = torch.tensor([int((new < d).any())])
        dist.all_reduce(changed)                            # termination
        d = new
        if int(changed.item()) == 0:
            break
    q.put((rank, d[lo:hi].numpy().astype(np.int32), lo, hi, steps))
    dist.destroy_process_group()


def test_gloo_world2_partitioned_exchange():
    import numpy as np
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_exchange, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((x[0], x[1:]) for x in (q.get(timeout=240) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = gg.config("rand-s")
    exp = oracle.sssp(g.row_off, g.col, g.w, g.source)
    got = np.concatenate([res[0][0], res[1][0]])
    assert res[0][1] == 0 and res[0][2] == res[1][1] and res[1][2] == g.n
    assert np.array_equal(got, exp)
    assert res[0][3] == res[1][3] > 1   # both ranks took the same number of supersteps
