"""The per-rank multi-GPU path (SURVEY.md §8(e), §8(b) load / output
conventions), executed by P host threads of one process on one GPU through
the loopback communicator (include/falcon.h falcon_comm_loopback_id): the
same code an NCCL rank runs -- slice loading (FALCON_LOAD_SLICE), the bounds
all-gather, the dense / sparse / fused exchanges, the termination all-reduce,
owned-slice output or FALCON_LOAD_GATHER -- with every NCCL call served
in-process.  Outputs must equal the oracle bit for bit: each rank's owned
slice, or the full array on every rank."""
import threading

import numpy as np
import pytest

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu
_cache = {}


def _g(name):
    if name not in _cache:
        _cache[name] = gg.config(name)
    return _cache[name]


def _ranks(fb, P, G, algos, flags=0, exchange=0, slice_mode=False, source=None):
    """Run `algos` collectively on P loopback ranks; returns per rank
    (owned range, {algo: output}, {algo: partition info})."""
    uid = fb.falcon_comm_loopback_id(P)
    bounds = fb.falcon_partition(G.row_off, P)
    res, errs = [None] * P, []
    src = G.source if source is None else source

    def rank(r):
        try:
            comm = fb.falcon_comm_init(P, r, uid, 0)
            if slice_mode:   # this rank passes only its rows (global column ids)
                lo, hi = int(bounds[r]), int(bounds[r + 1])
                base, top = int(G.row_off[lo]), int(G.row_off[hi])
                ro = (G.row_off[lo:hi + 1] - base).astype(np.uint32)
                g = fb.graph_load_csr(hi - lo, top - base, ro, G.col[base:top], G.w[base:top], device=0,
                                      flags=fb.LOAD_SLICE | flags, comm=comm)
            else:
                g = fb.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0, flags=flags, comm=comm)
            assert (g.n, g.m) == (G.n, G.m)
            fb.falcon_set_option(g, "exchange", exchange)
            outs, infos = {}, {}
            for a in algos:
                out = np.full(g.out_len, -7, np.int32)
                fb.run(g, a, "vertex", out, src)
                outs[a] = out
                infos[a] = fb.graph_partition_info(g)
            res[r] = (fb.graph_owned_range(g), outs, infos)
            fb.graph_free(g)
            fb.falcon_comm_free(comm)
        except Exception as e:   # noqa: BLE001 -- re-raised below
            errs.append((r, e))

    ths = [threading.Thread(target=rank, args=(r,)) for r in range(P)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in ths), "a loopback rank hung"
    if errs:
        raise errs[0][1]
    return res, bounds


def _check_slices(res, bounds, G, algos, gather):
    for a in algos:
        exp = oracle.run(a, G)
        for r, (rng, outs, _) in enumerate(res):
            lo, hi = rng
            assert (lo, hi) == (int(bounds[r]), int(bounds[r + 1]))
            got = outs[a]
            if gather:
                assert np.array_equal(got, exp), f"{a} rank {r}: {np.flatnonzero(got != exp)[:8]}"
            else:
                assert len(got) == hi - lo
                assert np.array_equal(got, exp[lo:hi]), f"{a} rank {r}: {np.flatnonzero(got != exp[lo:hi])[:8]}"
        if not gather:   # the owned ranges tile [0, n)
            rngs = sorted(x[0] for x in res)
            assert rngs[0][0] == 0 and rngs[-1][1] == G.n
            assert all(rngs[i][1] == rngs[i + 1][0] for i in range(len(rngs) - 1))


@pytest.mark.parametrize("name", ["tiny", "rand-s", "rmat-s", "grid-s"])
@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("exchange", [0, 1, 2, 3])
def test_loopback_ranks_owned_slices(gpu_lib, name, P, exchange):
    fb = gpu_lib
    G = _g(name)
    algos = ["sssp", "bfs", "cc"]
    res, bounds = _ranks(fb, P, G, algos, exchange=exchange)
    _check_slices(res, bounds, G, algos, gather=False)
    mode = res[0][2]["sssp"][0]
    assert mode == {0: 3, 1: 1, 2: 2, 3: 3}[exchange]   # auto between loopback ranks = fused


@pytest.mark.parametrize("name", ["tiny", "rand-s", "grid-s"])
@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("gather", [False, True])
def test_loopback_slice_load(gpu_lib, name, P, gather):
    """FALCON_LOAD_SLICE: each rank passes only its rows; with
    FALCON_LOAD_GATHER every rank receives the full array."""
    fb = gpu_lib
    G = _g(name)
    algos = ["sssp", "bfs", "cc"]
    res, bounds = _ranks(fb, P, G, algos, flags=fb.LOAD_GATHER if gather else 0, slice_mode=True)
    _check_slices(res, bounds, G, algos, gather=gather)


def test_loopback_no_host_round_trip_per_superstep(gpu_lib):
    """Fused / dense supersteps: the host looks at the control block once
    every 4 supersteps (SURVEY §8(a) a8 across ranks)."""
    fb = gpu_lib
    G = _g("grid-s")   # hundreds of supersteps
    for exchange in (1, 3):
        res, _ = _ranks(fb, 2, G, ["sssp"], exchange=exchange)
        mode, steps, checks = res[0][2]["sssp"]
        assert steps > 50 and checks <= steps // 4 + 1, (exchange, steps, checks)


def test_loopback_overflow_and_edge_cases(gpu_lib):
    """Overflow certificate across ranks (owned-slice output) and a rank that
    owns no arcs."""
    fb = gpu_lib
    G = gg.from_edges("ovf", 4, np.array([0, 1, 2], np.uint32), np.array([1, 2, 3], np.uint32),
                      np.array([1 << 30] * 3, np.int32), source=0)
    with pytest.raises(fb.FalconError) as ei:
        _ranks(fb, 2, G, ["sssp"], exchange=3)
    assert ei.value.name == "OVERFLOW"
    G2 = gg.from_edges("repro", 3, np.array([0, 1, 2], np.uint32), np.array([1, 2, 0], np.uint32),
                       np.array([1 << 30, (1 << 30) - 2, 5], np.int32), source=0)
    for ex in (1, 2, 3):
        res, bounds = _ranks(fb, 3, G2, ["sssp"], exchange=ex)
        _check_slices(res, bounds, G2, ["sssp"], gather=False)


def test_slice_flags_need_a_rank_communicator(gpu_lib):
    fb = gpu_lib
    G = _g("tiny")
    with pytest.raises(fb.FalconError) as ei:
        fb.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0, flags=fb.LOAD_SLICE)
    assert ei.value.name == "INVALID_ARG"
    comm = fb.falcon_comm_init_simulated(2)
    with pytest.raises(fb.FalconError) as ei:
        fb.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0, flags=fb.LOAD_SLICE, comm=comm)
    assert ei.value.name == "UNSUPPORTED"
