"""CPU oracle for the fixpoint min-relaxation path (SSSP / BFS / CC).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_1903_01665_b200`` never imports it, and
the two share no code.

Each function writes out the plain definition of what the paper's fixpoint
reaches (see oracle.c header):

* ``sssp``: dist[v] = min over directed source~>v paths of the weight sum
  (PAPER.md:1664-1693 Alg. "SSSP: iterating over Points"),
  by binary-heap Dijkstra with int64 sums; INF = 2**31-1.
* ``bfs``: level[v] = min number of arcs on a source~>v path
  (Alg. "BFS Algorithm in Falcon for CPU"), FIFO BFS.
* ``cc``: label[v] = min vertex id of v's weakly connected component
  ("propagation based"; SPEC.md:452 min-label convention),
  union-find.

Pins (tests/test_oracle.py): brute-force Bellman-Ford / Floyd-Warshall /
transitive closure on tiny graphs, scipy.sparse.csgraph on medium graphs,
hand-checked SPEC.md examples (tests/golden/), certificates, special cases.
No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

INF = 2147483647
_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile oracle.c (plain C, single-threaded) into liboracle.so."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", tmp, src])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        p = ctypes.c_void_p
        lib.oracle_sssp.argtypes = [ctypes.c_int64, p, p, p, ctypes.c_uint32, p]
        lib.oracle_bfs.argtypes = [ctypes.c_int64, p, p, ctypes.c_uint32, p]
        lib.oracle_cc.argtypes = [ctypes.c_int64, p, p, p]
        lib.oracle_mst.argtypes = [ctypes.c_int64, p, p, p, ctypes.POINTER(ctypes.c_int64),
                                   ctypes.POINTER(ctypes.c_int64), p]
        for f in (lib.oracle_sssp, lib.oracle_bfs, lib.oracle_cc, lib.oracle_mst):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


_ERR = {1: "bad argument or negative weight", 2: "overflow: a finite distance >= INF", 3: "out of memory"}


def sssp(row_off, col, w, source: int) -> np.ndarray:
    row_off = _c(row_off, np.uint32); col = _c(col, np.uint32)
    w = None if w is None else _c(w, np.int32)
    n = len(row_off) - 1
    out = np.empty(n, np.int32)
    rc = _L().oracle_sssp(n, _p(row_off), _p(col), _p(w), source, _p(out))
    if rc:
        raise OracleError(_ERR.get(rc, str(rc)))
    return out


def bfs(row_off, col, source: int) -> np.ndarray:
    row_off = _c(row_off, np.uint32); col = _c(col, np.uint32)
    n = len(row_off) - 1
    out = np.empty(n, np.int32)
    rc = _L().oracle_bfs(n, _p(row_off), _p(col), source, _p(out))
    if rc:
        raise OracleError(_ERR.get(rc, str(rc)))
    return out


def cc(row_off, col) -> np.ndarray:
    row_off = _c(row_off, np.uint32); col = _c(col, np.uint32)
    n = len(row_off) - 1
    out = np.empty(n, np.int32)
    rc = _L().oracle_cc(n, _p(row_off), _p(col), _p(out))
    if rc:
        raise OracleError(_ERR.get(rc, str(rc)))
    return out


def mst(row_off, col, w=None):
    """Minimum spanning forest of the undirected view (Kruskal): returns
    (total weight, number of forest edges, min-id tree label per vertex)."""
    row_off = _c(row_off, np.uint32); col = _c(col, np.uint32)
    w = None if w is None else _c(w, np.int32)
    n = len(row_off) - 1
    label = np.empty(n, np.int32)
    tot, ne = ctypes.c_int64(), ctypes.c_int64()
    rc = _L().oracle_mst(n, _p(row_off), _p(col), _p(w), ctypes.byref(tot), ctypes.byref(ne), _p(label))
    if rc:
        raise OracleError(_ERR.get(rc, str(rc)))
    return tot.value, ne.value, label


def run(algo: str, g) -> np.ndarray:
    """Oracle output for a graphgen.Graph (algo in {'sssp','bfs','cc'})."""
    if algo == "sssp":
        return sssp(g.row_off, g.col, g.w, g.source)
    if algo == "bfs":
        return bfs(g.row_off, g.col, g.source)
    if algo == "cc":
        return cc(g.row_off, g.col)
    raise KeyError(algo)
