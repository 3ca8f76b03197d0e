"""Seeded synthetic graph inputs shared by the oracle and the CUDA path.

Input infrastructure only: it draws graphs and lays them out as CSR; it holds
none of the method's arithmetic (no relaxation, no distances, no labels).
Both ``oracle/`` and ``paper_1903_01665_b200`` consume what it returns.

Recipe: xoshiro256** seeded by splitmix64
(SPEC.md:567), chunked by 2^20 arcs; G(n,m) directed with weights U[1,100]
(SPEC.md:538-546); R-MAT with (a,b,c,d) = (0.476, 0.15, 0.15, 0.224) fitted to
PAPER.md Table 1 (rmat-10M max-degree 1873) and a seeded vertex
relabelling; a W x H road-like lattice with keep probability p (shape of
USA-full); CSR by stable counting sort.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libgraphgen.so")
_lib = None

RMAT_ABCD = (0.476, 0.15, 0.15, 0.224)
GRID_P = 0.6043


def build(force: bool = False) -> str:
    """Compile gen.c into libgraphgen.so (gcc, OpenMP)."""
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC",
                               "-o", tmp, src, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        u64, u32, i64, dbl, p = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
        lib.gg_er.argtypes = [u64, u64, u64, p, p, p]
        lib.gg_er.restype = ctypes.c_int
        lib.gg_rmat.argtypes = [u64, u64, u64, dbl, dbl, dbl, ctypes.c_int, p, p, p]
        lib.gg_rmat.restype = ctypes.c_int
        lib.gg_grid.argtypes = [u64, u64, dbl, u64, p, p, p]
        lib.gg_grid.restype = i64
        lib.gg_csr.argtypes = [u64, u64, p, p, p, p, p, p]
        lib.gg_csr.restype = ctypes.c_int
        lib.gg_pick_source.argtypes = [u64, p, u64]
        lib.gg_pick_source.restype = u32
        lib.gg_xoshiro_first.argtypes = [u64]
        lib.gg_xoshiro_first.restype = u64
        lib.gg_uniform_first.argtypes = [u64, u32]
        lib.gg_uniform_first.restype = u32
        lib.gg_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray | None):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------- edge lists
def er_edges(n: int, m: int, seed: int):
    """Directed G(n,m): m arcs, endpoints uniform, no self loops, duplicates kept."""
    src = np.empty(m, np.uint32); dst = np.empty(m, np.uint32); w = np.empty(m, np.int32)
    if _L().gg_er(n, m, seed, _ptr(src), _ptr(dst), _ptr(w)) != 0:
        raise ValueError("gg_er: bad parameters")
    return src, dst, w


def rmat_edges(n: int, m: int, seed: int, abcd=RMAT_ABCD, relabel: bool = True):
    a, b, c, d = abcd
    if abs(a + b + c + d - 1.0) > 1e-9:
        raise ValueError("R-MAT probabilities must sum to 1")
    src = np.empty(m, np.uint32); dst = np.empty(m, np.uint32); w = np.empty(m, np.int32)
    if _L().gg_rmat(n, m, seed, a, b, c, int(relabel), _ptr(src), _ptr(dst), _ptr(w)) != 0:
        raise ValueError("gg_rmat: bad parameters")
    return src, dst, w


def grid_edges(W: int, H: int, p: float, seed: int):
    lib = _L()
    cnt = lib.gg_grid(W, H, p, seed, None, None, None)
    if cnt < 0:
        raise ValueError("gg_grid: bad parameters")
    src = np.empty(cnt, np.uint32); dst = np.empty(cnt, np.uint32); w = np.empty(cnt, np.int32)
    lib.gg_grid(W, H, p, seed, _ptr(src), _ptr(dst), _ptr(w))
    return src, dst, w


def csr_from_edges(n: int, src, dst, w=None):
    """Stable counting sort by src -> (row_off u32[n+1], col u32[m], w i32[m] | None)."""
    src = np.ascontiguousarray(src, np.uint32); dst = np.ascontiguousarray(dst, np.uint32)
    m = len(src)
    row_off = np.empty(n + 1, np.uint32); col = np.empty(m, np.uint32)
    wout = None
    if w is not None:
        w = np.ascontiguousarray(w, np.int32); wout = np.empty(m, np.int32)
    rc = _L().gg_csr(n, m, _ptr(src), _ptr(dst), _ptr(w), _ptr(row_off), _ptr(col), _ptr(wout))
    if rc != 0:
        raise ValueError(f"gg_csr failed ({rc}): endpoint out of range or m too large")
    return row_off, col, wout


def pick_source(row_off: np.ndarray, seed: int) -> int:
    n = len(row_off) - 1
    return int(_L().gg_pick_source(n, _ptr(np.ascontiguousarray(row_off, np.uint32)), seed))


# ---------------------------------------------------------------- graphs
@dataclass
class Graph:
    name: str
    n: int
    row_off: np.ndarray
    col: np.ndarray
    w: np.ndarray | None
    source: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def m(self) -> int:
        return int(self.row_off[-1]) if self.n >= 0 and len(self.row_off) else 0

    def out_degree(self) -> np.ndarray:
        return np.diff(self.row_off.astype(np.int64))

    def edges(self):
        """(src, dst, w) in CSR order."""
        src = np.repeat(np.arange(self.n, dtype=np.uint32), self.out_degree())
        return src, self.col, self.w


def from_edges(name: str, n: int, src, dst, w=None, source: int | None = None, seed: int = 0) -> Graph:
    row_off, col, wout = csr_from_edges(n, src, dst, w)
    if source is None:
        source = pick_source(row_off, seed) if n > 0 else 0
    return Graph(name, n, row_off, col, wout, source)


def er(n: int, m: int, seed: int, name: str | None = None) -> Graph:
    s, d, w = er_edges(n, m, seed)
    g = from_edges(name or f"er-{n}-{m}", n, s, d, w, seed=seed)
    g.meta = {"generator": "G(n,m) directed", "seed": seed}
    return g


def rmat(n: int, m: int, seed: int, abcd=RMAT_ABCD, relabel: bool = True, name: str | None = None) -> Graph:
    s, d, w = rmat_edges(n, m, seed, abcd, relabel)
    g = from_edges(name or f"rmat-{n}-{m}", n, s, d, w, seed=seed)
    g.meta = {"generator": "R-MAT", "abcd": list(abcd), "relabel": relabel, "seed": seed}
    return g


def grid(W: int, H: int, seed: int, p: float = GRID_P, name: str | None = None, centre_source: bool = False) -> Graph:
    s, d, w = grid_edges(W, H, p, seed)
    n = W * H
    g = from_edges(name or f"grid-{W}x{H}", n, s, d, w, seed=seed)
    if centre_source:
        c = (H // 2) * W + W // 2
        if g.row_off[c + 1] > g.row_off[c]:
            g.source = c
    g.meta = {"generator": "2-D lattice, kept w.p. p, both arcs", "W": W, "H": H, "p": p, "seed": seed}
    return g


# The BASELINE.json configs.
CONFIGS = {
    "tiny": lambda: er(1000, 4000, 1, name="tiny"),
    "rand-25M": lambda: er(25_000_000, 100_000_000, 25, name="rand-25M"),
    "rmat-10M": lambda: rmat(10_000_000, 100_000_000, 10, name="rmat-10M"),
    "grid-24M": lambda: grid(6000, 4000, 24, name="grid-24M"),
    "rand-125M": lambda: er(125_000_000, 500_000_000, 125, name="rand-125M"),
    "rmat-50M": lambda: rmat(50_000_000, 500_000_000, 50, name="rmat-50M"),
}

# The partner graphs of the paper's multi-target experiment (Table 1 sizes,
# PAPER.md:24-35; Tables tab:multigpucc / tab:multigpubfs):
# rand-50M, rmat-20M, and a USA-CTR-shaped road grid (14M vertices / 34M arcs).
PAIR_CONFIGS = {
    "rand-50M": lambda: er(50_000_000, 200_000_000, 50, name="rand-50M"),
    "rmat-20M": lambda: rmat(20_000_000, 200_000_000, 20, name="rmat-20M"),
    "grid-14M": lambda: grid(4000, 3500, 14, name="grid-14M"),
}

# Reduced-scale analogues with the same recipe (for tests that must run fast).
SMALL_CONFIGS = {
    "rand-s": lambda: er(200_000, 800_000, 125, name="rand-s"),
    "rmat-s": lambda: rmat(1 << 17, 1_310_720, 50, name="rmat-s"),
    "grid-s": lambda: grid(300, 200, 24, name="grid-s"),
}


def config(name: str) -> Graph:
    if name in CONFIGS:
        return CONFIGS[name]()
    if name in SMALL_CONFIGS:
        return SMALL_CONFIGS[name]()
    if name in PAIR_CONFIGS:
        return PAIR_CONFIGS[name]()
    raise KeyError(name)


def num_threads() -> int:
    return int(_L().gg_num_threads())
