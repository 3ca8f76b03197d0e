"""Thin Python binding of the C ABI in include/falcon.h (libfalcon.so).

Argument marshalling only: every step of the path runs in the library's
sm_100a kernels.  There is no CPU fallback -- if libfalcon.so cannot be loaded
every call raises.  Arrays may be numpy arrays (host) or torch tensors (host
or CUDA); PyTorch is used only for device memory and streams.

Names follow the C ABI: graph_load_csr, graph_free, graph_info, graph_owned_range,
graph_share, falcon_run_many, falcon_sssp, falcon_bfs, falcon_cc, falcon_mst, falcon_set_profiling, falcon_set_delta, falcon_set_option,
falcon_partition, falcon_comm_unique_id, falcon_comm_init,
falcon_comm_init_simulated, falcon_comm_free, falcon_last_error, falcon_version.
"""
from __future__ import annotations

import ctypes
import os

__all__ = ["load", "graph_load_csr", "graph_free", "graph_info", "graph_share", "falcon_run_many", "falcon_mst", "falcon_trim_memory", "graph_exchange_bytes", "falcon_sssp", "falcon_bfs", "falcon_cc",
           "falcon_set_profiling", "falcon_set_delta", "falcon_set_option", "falcon_partition", "falcon_comm_unique_id",
           "falcon_comm_init", "falcon_comm_init_simulated", "falcon_comm_loopback_id", "falcon_comm_free", "graph_owned_range", "graph_partition_info", "LOAD_SLICE", "LOAD_GATHER", "Comm", "falcon_last_error", "falcon_version", "FalconError", "FalconStats",
           "STYLES", "INF", "LIB_PATH"]

INF = 2147483647
STYLE_VERTEX, STYLE_EDGE, STYLE_WORKLIST, STYLE_DELTA = 0, 1, 2, 3
STYLES = {"vertex": STYLE_VERTEX, "edge": STYLE_EDGE, "worklist": STYLE_WORKLIST, "delta": STYLE_DELTA}
LOAD_BUILD_COO = 0x1
LOAD_BUILD_REVERSE = 0x2
LOAD_SLICE = 0x4    # partitioned: this rank passes only its rows (include/falcon.h)
LOAD_GATHER = 0x8   # partitioned: full output on every rank (default: the owned slice)
ALGOS = {"sssp": 0, "bfs": 1, "cc": 2}
STATUS = {0: "OK", 1: "INVALID_ARG", 2: "OUT_OF_RANGE", 3: "NO_MEMORY", 4: "CUDA", 5: "OVERFLOW",
          6: "NOT_CONVERGED", 7: "COMM", 8: "UNSUPPORTED"}

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfalcon.so")
_lib = None


class FalconError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class FalconStats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("vertices_processed", ctypes.c_int64),
                ("edges_relaxed", ctypes.c_int64), ("updates", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("ms", ctypes.c_double),
                ("relax_ms", ctypes.c_double), ("relax_launches", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class _Job(ctypes.Structure):
    _fields_ = [("algo", ctypes.c_int), ("style", ctypes.c_int), ("source", ctypes.c_uint32)]


class _LoadOpts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("cuda_stream", ctypes.c_void_p), ("flags", ctypes.c_uint32),
                ("comm", ctypes.c_void_p)]


def load(build_if_missing: bool = False):
    """Load libfalcon.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if not build_if_missing:
            raise FalconError(4, f"{LIB_PATH} not built: run __graft_entry__.build() "
                                 "(there is no CPU fallback)")
        from . import _build
        _build.build()
    lib = ctypes.CDLL(LIB_PATH)
    p, i64, u32, st = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32, ctypes.c_int
    lib.graph_load_csr.argtypes = [i64, i64, p, p, p, ctypes.POINTER(_LoadOpts), ctypes.POINTER(p)]
    lib.graph_free.argtypes = [p]
    lib.graph_info.argtypes = [p, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    lib.falcon_sssp.argtypes = [p, u32, ctypes.c_int, p, ctypes.POINTER(FalconStats)]
    lib.falcon_bfs.argtypes = [p, u32, ctypes.c_int, p, ctypes.POINTER(FalconStats)]
    lib.falcon_cc.argtypes = [p, ctypes.c_int, p, ctypes.POINTER(FalconStats)]
    lib.falcon_set_profiling.argtypes = [p, ctypes.c_int]
    lib.falcon_set_delta.argtypes = [p, ctypes.c_int32]
    lib.falcon_set_delta.restype = st
    lib.falcon_set_option.argtypes = [p, ctypes.c_char_p, i64]
    lib.falcon_set_option.restype = st
    lib.falcon_partition.argtypes = [i64, p, ctypes.c_int, p]
    lib.falcon_comm_unique_id.argtypes = [p]
    lib.falcon_comm_init.argtypes = [ctypes.c_int, ctypes.c_int, p, ctypes.c_int, ctypes.POINTER(p)]
    lib.falcon_comm_init_simulated.argtypes = [ctypes.c_int, ctypes.POINTER(p)]
    lib.falcon_comm_free.argtypes = [p]
    lib.graph_owned_range.argtypes = [p, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    lib.graph_exchange_bytes.argtypes = [p, ctypes.POINTER(i64)]
    lib.graph_exchange_bytes.restype = st
    lib.falcon_trim_memory.argtypes = [ctypes.POINTER(i64)]
    lib.falcon_trim_memory.restype = st
    lib.falcon_mst.argtypes = [p, ctypes.c_int, ctypes.POINTER(i64), ctypes.POINTER(i64), p,
                               ctypes.POINTER(FalconStats)]
    lib.falcon_mst.restype = st
    lib.graph_share.argtypes = [p, ctypes.POINTER(_LoadOpts), ctypes.POINTER(p)]
    lib.graph_share.restype = st
    lib.falcon_run_many.argtypes = [ctypes.c_int, ctypes.POINTER(p), ctypes.POINTER(_Job), ctypes.POINTER(p),
                                    ctypes.POINTER(FalconStats)]
    lib.falcon_run_many.restype = st
    for f in (lib.falcon_partition, lib.falcon_comm_unique_id, lib.falcon_comm_init, lib.falcon_comm_init_simulated,
              lib.falcon_comm_free, lib.graph_owned_range, lib.falcon_comm_loopback_id, lib.graph_partition_info):
        f.restype = st
    for f in (lib.graph_load_csr, lib.graph_free, lib.graph_info, lib.falcon_sssp, lib.falcon_bfs, lib.falcon_cc,
              lib.falcon_set_profiling):
        f.restype = st
    lib.falcon_last_error.restype = ctypes.c_char_p
    lib.falcon_version.restype = ctypes.c_char_p
    _lib = lib
    return lib


def _ptr(x):
    if x is None:
        return None
    if hasattr(x, "data_ptr"):  # torch tensor (host or CUDA)
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(x.data_ptr())
    if hasattr(x, "ctypes"):  # numpy
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return ctypes.c_void_p(x.ctypes.data)
    if isinstance(x, int):
        return ctypes.c_void_p(x)
    raise TypeError(f"unsupported buffer type {type(x)}")


def _check(rc: int):
    if rc != 0:
        raise FalconError(rc, (load().falcon_last_error() or b"").decode())


def _style(style) -> int:
    if isinstance(style, str):
        return STYLES[style.lower()]
    return int(style)


def _check_dtype(x, kind: str, name: str):
    dt = getattr(x, "dtype", None)
    if dt is None:
        return
    s = str(dt)
    ok = {"u32": ("uint32",), "i32": ("int32",)}[kind]
    if not any(s.endswith(o) for o in ok):
        raise TypeError(f"{name} must be {ok[0]}, got {s}")


def _numel(x):
    if hasattr(x, "numel"):
        return int(x.numel())
    if hasattr(x, "size") and not callable(x.size):
        return int(x.size)
    return None


def _check_len(x, need: int, name: str, exact: bool = False):
    """The C ABI reads / writes `need` elements through the pointer: a shorter
    buffer would be overrun, so refuse it here."""
    k = _numel(x)
    if k is None:
        return
    if k < need or (exact and k != need):
        raise ValueError(f"{name} has {k} elements, needs {'exactly ' if exact else 'at least '}{need}")


class Graph:
    """Owning handle of a falcon_graph_t (freed by graph_free or on GC)."""

    def __init__(self, handle: ctypes.c_void_p, n: int, m: int):
        self.handle = handle
        self.n = n
        self.m = m
        self.out_len = n   # elements an output buffer must hold

    def __del__(self):
        try:
            graph_free(self)
            parent = getattr(self, "_parent", None)
            if parent is not None:
                parent._views -= 1
        except Exception:
            pass

    @property
    def _as_parameter_(self):
        return self.handle


class Comm:
    """Owning handle of a falcon_comm_t (multi-GPU or simulated partitions)."""

    def __init__(self, handle: ctypes.c_void_p, nparts: int, rank: int):
        self.handle = handle
        self.nparts = nparts
        self.rank = rank

    def __del__(self):
        try:
            falcon_comm_free(self)
        except Exception:
            pass


def falcon_partition(row_off, nparts: int):
    """Edge-balanced contiguous vertex ranges: int64[nparts+1] (host only)."""
    import numpy as np
    row_off = np.ascontiguousarray(row_off, np.uint32)
    bounds = np.empty(nparts + 1, np.int64)
    _check(load().falcon_partition(len(row_off) - 1, _ptr(row_off), nparts, _ptr(bounds)))
    return bounds


def falcon_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().falcon_comm_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return buf.raw


def falcon_comm_init(nranks: int, rank: int, unique_id: bytes, device: int) -> Comm:
    out = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(bytes(unique_id), 128)
    _check(load().falcon_comm_init(nranks, rank, ctypes.cast(buf, ctypes.c_void_p), device, ctypes.byref(out)))
    return Comm(out, nranks, rank)


def falcon_comm_loopback_id(nranks: int) -> bytes:
    """Id of an in-process loopback world of nranks ranks (host threads of this
    process; include/falcon.h): pass it to falcon_comm_init from each thread."""
    buf = ctypes.create_string_buffer(128)
    _check(load().falcon_comm_loopback_id(nranks, ctypes.cast(buf, ctypes.c_void_p)))
    return buf.raw


def graph_partition_info(g: "Graph"):
    """(exchange mode 1 dense / 2 sparse / 3 fused, supersteps, host round trips) of the last call."""
    mode, steps, checks = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
    _check(load().graph_partition_info(g.handle, ctypes.byref(mode), ctypes.byref(steps), ctypes.byref(checks)))
    return mode.value, steps.value, checks.value


def falcon_comm_init_simulated(nparts: int) -> Comm:
    out = ctypes.c_void_p()
    _check(load().falcon_comm_init_simulated(nparts, ctypes.byref(out)))
    return Comm(out, nparts, 0)


def falcon_comm_free(comm: Comm):
    if comm is not None and comm.handle:
        load().falcon_comm_free(comm.handle)
        comm.handle = None


def graph_owned_range(g: "Graph"):
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _check(load().graph_owned_range(g.handle, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def graph_load_csr(n: int, m: int, row_off, col, w=None, device: int = -1, stream=None, flags: int = 0,
                   comm: Comm | None = None) -> Graph:
    """graph_load_csr(n, m, row_off u32[n+1], col u32[m], w i32[m] | None, ...)."""
    lib = load()
    _check_dtype(row_off, "u32", "row_off"); _check_dtype(col, "u32", "col")
    _check_len(row_off, n + 1, "row_off")
    _check_len(col, m, "col")
    if w is not None:
        _check_dtype(w, "i32", "w")
        _check_len(w, m, "w")
    if stream is not None and hasattr(stream, "cuda_stream"):
        stream = stream.cuda_stream
    opts = _LoadOpts(device, ctypes.c_void_p(stream) if stream else None, flags,
                     comm.handle if comm is not None else None)
    out = ctypes.c_void_p()
    _check(lib.graph_load_csr(n, m, _ptr(row_off), _ptr(col), _ptr(w), ctypes.byref(opts), ctypes.byref(out)))
    g = Graph(out, n, m)
    g._comm = comm   # keep the communicator alive as long as the graph
    if comm is not None:   # a slice load's n / m are the rank's; the graph's are global
        g.n, g.m = graph_info(g)
        lo, hi = graph_owned_range(g)
        g.out_len = g.n if flags & LOAD_GATHER else hi - lo
    return g


def graph_free(g: Graph):
    if g is not None and g.handle:
        _check(load().graph_free(g.handle))
        g.handle = None


def graph_share(g: Graph, stream=None) -> Graph:
    """A view of g with its own scratch (for concurrent calls); free it before g."""
    if stream is not None and hasattr(stream, "cuda_stream"):
        stream = stream.cuda_stream
    opts = _LoadOpts(-1, ctypes.c_void_p(stream) if stream else None, 0, None)
    out = ctypes.c_void_p()
    _check(load().graph_share(g.handle, ctypes.byref(opts), ctypes.byref(out)))
    v = Graph(out, g.n, g.m)
    v._parent = g   # the parent must outlive the view
    g._views = getattr(g, "_views", 0) + 1
    return v


def falcon_run_many(jobs) -> list:
    """Run jobs concurrently: jobs = [(graph, algo, style, source, out), ...] on
    distinct handles (a graph and its views).  Returns one FalconStats per job."""
    k = len(jobs)
    hs = (ctypes.c_void_p * k)(*[j[0].handle for j in jobs])
    js = (_Job * k)(*[_Job(ALGOS[j[1]], _style(j[2]), int(j[3])) for j in jobs])
    for j in jobs:
        _check_dtype(j[4], "i32", "out")
        _check_len(j[4], j[0].out_len, "out")
    outs = (ctypes.c_void_p * k)(*[_ptr(j[4]) for j in jobs])
    stats = (FalconStats * k)()
    _check(load().falcon_run_many(k, hs, js, outs, stats))
    return list(stats)


def graph_info(g: Graph):
    n, m = ctypes.c_int64(), ctypes.c_int64()
    _check(load().graph_info(g.handle, ctypes.byref(n), ctypes.byref(m)))
    return n.value, m.value


def falcon_sssp(g: Graph, source: int, style, dist_out) -> FalconStats:
    st = FalconStats()
    _check_dtype(dist_out, "i32", "dist_out")
    _check_len(dist_out, g.out_len, "dist_out")
    _check(load().falcon_sssp(g.handle, source, _style(style), _ptr(dist_out), ctypes.byref(st)))
    return st


def falcon_bfs(g: Graph, source: int, style, level_out) -> FalconStats:
    st = FalconStats()
    _check_dtype(level_out, "i32", "level_out")
    _check_len(level_out, g.out_len, "level_out")
    _check(load().falcon_bfs(g.handle, source, _style(style), _ptr(level_out), ctypes.byref(st)))
    return st


def falcon_cc(g: Graph, style, label_out) -> FalconStats:
    st = FalconStats()
    _check_dtype(label_out, "i32", "label_out")
    _check_len(label_out, g.out_len, "label_out")
    _check(load().falcon_cc(g.handle, _style(style), _ptr(label_out), ctypes.byref(st)))
    return st


def graph_exchange_bytes(g: Graph) -> int:
    """Bytes the last call on a partitioned graph moved in boundary exchanges."""
    out = ctypes.c_int64()
    _check(load().graph_exchange_bytes(g.handle, ctypes.byref(out)))
    return out.value


def falcon_trim_memory() -> int:
    """Release the library's cached device memory; returns the bytes released."""
    out = ctypes.c_int64()
    _check(load().falcon_trim_memory(ctypes.byref(out)))
    return out.value


def falcon_mst(g: Graph, style, label_out=None):
    """Minimum spanning forest: returns (total weight, forest edges, FalconStats);
    label_out (optional int32[n]) receives the min-id tree label per vertex."""
    st = FalconStats()
    if label_out is not None:
        _check_dtype(label_out, "i32", "label_out")
        _check_len(label_out, g.out_len, "label_out")
    tot, ne = ctypes.c_int64(), ctypes.c_int64()
    _check(load().falcon_mst(g.handle, _style(style), ctypes.byref(tot), ctypes.byref(ne), _ptr(label_out),
                             ctypes.byref(st)))
    return tot.value, ne.value, st


def falcon_set_profiling(g: Graph, enable: bool):
    _check(load().falcon_set_profiling(g.handle, int(bool(enable))))


def falcon_set_delta(g: Graph, delta: int):
    """Bucket width of the DELTA style (0 = auto: max(1, average weight))."""
    _check(load().falcon_set_delta(g.handle, int(delta)))


def falcon_set_option(g: Graph, name: str, value: int):
    """Tuning option of a loaded graph (include/falcon.h: block_bytes, dense_div,
    pull_div, persist, persist_max).  Results never depend on it."""
    _check(load().falcon_set_option(g.handle, name.encode(), int(value)))


def falcon_last_error() -> str:
    return (load().falcon_last_error() or b"").decode()


def falcon_version() -> str:
    return load().falcon_version().decode()


def run(g: Graph, algo: str, style, out, source: int = 0) -> FalconStats:
    """Dispatch helper: algo in {'sssp','bfs','cc'}."""
    if algo == "sssp":
        return falcon_sssp(g, source, style, out)
    if algo == "bfs":
        return falcon_bfs(g, source, style, out)
    if algo == "cc":
        return falcon_cc(g, style, out)
    raise KeyError(algo)
