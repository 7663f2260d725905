"""Deterministic datasets for the nested-parallel benchmarks.

Same dataset vocabulary and the same bytes as the reference generators
(bench/graphs.py of ``dynoptc``), held as contiguous int32 numpy arrays (the
HBM layout the kernels read) instead of Python tuples:

=============  =================================================  ==========
spec           contents                                           reference
=============  =================================================  ==========
``hand``       fixed 10-vertex CSR, BFS distances known            :96-104
``powerlaw:N``  zipf(1.8) out-degrees, forced hub at vertex 0       :139-151
``road:N``     out-degrees 1..8, local targets                     :154-171
``sizes:N``    child-grid sizes, 90% in [0,31], 10% in [256,1024]  :194-201
``rmat:S``     RMAT scale S, edge factor 16 (new: BASELINE.json)   --
``curves:N``   N quadratic Bezier curves (new: BASELINE.json)      --
``ksat3:N``    random 3-SAT, N variables, 4.2 N clauses (SP)       --
``ksat5:N``    random 5-SAT, N variables, 20 N clauses (SP)        --
=============  =================================================  ==========

Streams: every generator draws from ``default_rng(SeedSequence([stream_id,
*keys]))`` with the reference's stream ids (graphs.py:109-114), so a
``powerlaw:150:seed2`` here is byte-identical to the reference's.  RMAT uses a
counter-based integer generator in the native library (csrc/gen.cpp) so that
RMAT-22/26 build in seconds on all host cores and identically on any host.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

UNREACHED = 1 << 30  # distance sentinel (graphs.py:29)

GRAPH_KINDS = ("hand", "powerlaw", "road", "rmat")
SAT_KINDS = {"ksat3": (3, 4.2), "ksat5": (5, 20.0)}  # (k, clause ratio)
DATASET_KINDS = GRAPH_KINDS + ("sizes", "curves") + tuple(SAT_KINDS)

RMAT_EDGE_FACTOR = 16  # Graph500 / BASELINE.json configs
BT_MAX_TESS = 2048     # T2048-C64
BT_CURV_SCALE = 64.0

_STREAM = {"powerlaw": 1, "road": 2, "weights": 3, "sizes": 4, "curves": 5,
           "sat": 6, "sat_eta": 7}


def _rng(stream: str, *keys: int) -> np.random.Generator:
    return np.random.default_rng(
        np.random.SeedSequence([_STREAM[stream], *keys]))


@dataclass(frozen=True, eq=False)
class Graph:
    """Directed CSR graph: ``rowptr`` int32[n+1], ``col`` int32[m]."""
    rowptr: np.ndarray
    col: np.ndarray

    @property
    def n(self) -> int:
        return int(self.rowptr.shape[0]) - 1

    @property
    def m(self) -> int:
        return int(self.col.shape[0])

    def degrees(self) -> np.ndarray:
        return np.diff(self.rowptr)

    def neighbors(self, u: int) -> np.ndarray:
        return self.col[self.rowptr[u]:self.rowptr[u + 1]]


@dataclass(frozen=True)
class DatasetSpec:
    kind: str
    size: int
    seed: int
    text: str


def parse_spec(text: str) -> DatasetSpec:
    """``kind:size:seedN`` or ``hand`` (graphs.py:64-89, same errors).

    For ``rmat`` the size field is the scale (n = 2**size)."""
    kind, *rest = text.split(":")
    if kind not in DATASET_KINDS:
        raise ValueError(f"unknown dataset kind {kind!r} "
                         f"(expected one of {', '.join(DATASET_KINDS)})")
    if kind == "hand":
        if rest:
            raise ValueError("the hand fixture takes no size or seed")
        return DatasetSpec("hand", 10, 0, text)
    if len(rest) != 2:
        raise ValueError(f"dataset spec {text!r} is not kind:size:seedN")
    size_txt, seed_txt = rest
    try:
        size = int(size_txt)
    except ValueError:
        raise ValueError(f"bad dataset size {size_txt!r}") from None
    if not seed_txt.startswith("seed") or not seed_txt[4:].lstrip("-").isdigit():
        raise ValueError(f"bad dataset seed {seed_txt!r} (expected seedN)")
    seed = int(seed_txt[4:])
    if size < 1:
        raise ValueError("dataset size must be at least 1")
    if kind == "rmat" and size > 30:
        raise ValueError("rmat scale must be at most 30")
    return DatasetSpec(kind, size, seed, text)


# ---------------------------------------------------------------------------
# graphs
# ---------------------------------------------------------------------------

# 0 -> 1, 2; 1 -> 3; 2 -> 3, 6; 3 -> 4; 4 -> 5; 5 -> 8; 6 -> 7; 7 -> 8;
# 9 unreachable (graphs.py:96-104)
HAND_EDGES = ((0, 1), (0, 2), (1, 3), (2, 3), (2, 6), (3, 4), (4, 5),
              (5, 8), (6, 7), (7, 8))
HAND_BFS_DISTANCES = (0, 1, 1, 2, 3, 4, 2, 3, 4, UNREACHED)


def _csr(n: int, src: np.ndarray, dst: np.ndarray, sort: bool) -> Graph:
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    if sort:
        order = np.lexsort((dst, src))
        src, dst = src[order], dst[order]
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rowptr, src + 1, 1)
    np.cumsum(rowptr, out=rowptr)
    return Graph(rowptr.astype(np.int32), dst.astype(np.int32))


def hand_graph() -> Graph:
    e = np.array(HAND_EDGES, dtype=np.int64)
    return _csr(10, e[:, 0], e[:, 1], sort=True)


def _from_degrees(degrees: np.ndarray, targets: np.ndarray) -> Graph:
    rowptr = np.concatenate(([0], np.cumsum(degrees, dtype=np.int64)))
    return Graph(rowptr.astype(np.int32), targets.astype(np.int32))


def powerlaw_graph(n: int, seed: int) -> Graph:
    """zipf(1.8) out-degrees clipped to n-1, vertex 0 forced to be a hub
    (graphs.py:139-151); targets uniform."""
    rng = _rng("powerlaw", n, seed)
    degrees = np.minimum(rng.zipf(1.8, size=n), max(n - 1, 0))
    if n > 1:
        degrees[0] = max(int(degrees.max()), min(n - 1, max(8, n // 20)))
    targets = rng.integers(0, n, size=int(degrees.sum()), dtype=np.int64)
    return _from_degrees(degrees, targets)


_ROAD_P = (0.25, 0.20, 0.15, 0.12, 0.10, 0.08, 0.06, 0.04)


def road_graph(n: int, seed: int) -> Graph:
    """Out-degree 1..8 (mean ~3.3), each target 1..49 hops ahead on a ring
    that never folds back onto its source (graphs.py:154-171)."""
    rng = _rng("road", n, seed)
    if n == 1:
        return Graph(np.zeros(2, dtype=np.int32), np.zeros(0, dtype=np.int32))
    degrees = rng.choice(np.arange(1, 9), size=n, p=_ROAD_P)
    hops = rng.integers(1, 50, size=int(degrees.sum()), dtype=np.int64)
    src = np.repeat(np.arange(n, dtype=np.int64), degrees)
    return _from_degrees(degrees, (src + 1 + (hops - 1) % (n - 1)) % n)


def rmat_graph(scale: int, seed: int,
               edge_factor: int = RMAT_EDGE_FACTOR) -> Graph:
    """Graph500 RMAT (a,b,c,d = .57,.19,.19,.05), n = 2**scale, m =
    edge_factor*n, multi-edges and self-loops kept, rows sorted."""
    from .. import _lib
    n = 1 << scale
    m = edge_factor * n
    rowptr = np.empty(n + 1, dtype=np.int32)
    col = np.empty(m, dtype=np.int32)
    _lib.check(_lib.load().dp_rmat_csr(scale, edge_factor, seed,
                                      _lib.ptr(rowptr), _lib.ptr(col), 0))
    return Graph(rowptr, col)


def make_graph(spec: DatasetSpec) -> Graph:
    if spec.kind == "hand":
        return hand_graph()
    if spec.kind == "powerlaw":
        return powerlaw_graph(spec.size, spec.seed)
    if spec.kind == "road":
        return road_graph(spec.size, spec.seed)
    if spec.kind == "rmat":
        return rmat_graph(spec.size, spec.seed)
    raise ValueError(f"dataset kind {spec.kind!r} is not a graph")


def edge_weights(graph: Graph, seed: int) -> np.ndarray:
    """Positive int weights in [1, 9] per (n, m, seed) (graphs.py:184-187)."""
    rng = _rng("weights", graph.n, graph.m, seed)
    return rng.integers(1, 10, size=graph.m).astype(np.int32)


def child_sizes(n: int, seed: int) -> np.ndarray:
    """manylaunch child-grid sizes (graphs.py:194-201)."""
    rng = _rng("sizes", n, seed)
    small = rng.integers(0, 32, size=n)
    large = rng.integers(256, 1025, size=n)
    pick_large = rng.random(n) < 0.10
    return np.where(pick_large, large, small).astype(np.int32)


# ---------------------------------------------------------------------------
# triangle counting input: simple undirected graph, degree-oriented
# ---------------------------------------------------------------------------

def tc_orient(graph: Graph) -> Graph:
    """Drop self-loops, symmetrise, deduplicate, keep u->v iff
    (deg u, u) < (deg v, v); rows ascending."""
    from .. import _lib
    import ctypes
    lib = _lib.load()
    rp = ctypes.c_void_p()
    cp = ctypes.c_void_p()
    mp = ctypes.c_int64()
    _lib.check(lib.dp_tc_orient(_lib.ptr(graph.rowptr), _lib.ptr(graph.col),
                                graph.n, ctypes.byref(rp), ctypes.byref(cp),
                                ctypes.byref(mp), 0))
    try:
        n, m = graph.n, mp.value
        rowptr = np.ctypeslib.as_array(
            ctypes.cast(rp, ctypes.POINTER(ctypes.c_int32)), (n + 1,)).copy()
        col = (np.ctypeslib.as_array(
            ctypes.cast(cp, ctypes.POINTER(ctypes.c_int32)), (m,)).copy()
            if m else np.zeros(0, dtype=np.int32))
    finally:
        lib.dp_free(rp)
        lib.dp_free(cp)
    return Graph(rowptr, col)


def symmetrize(graph: Graph) -> Graph:
    """Undirected simple graph: both directions of every non-loop edge,
    duplicates dropped, rows ascending (graph colouring input)."""
    from .. import _lib
    import ctypes
    lib = _lib.load()
    rp = ctypes.c_void_p()
    cp = ctypes.c_void_p()
    mp = ctypes.c_int64()
    _lib.check(lib.dp_symmetrize(_lib.ptr(graph.rowptr), _lib.ptr(graph.col),
                                 graph.n, ctypes.byref(rp), ctypes.byref(cp),
                                 ctypes.byref(mp), 0))
    try:
        n, m = graph.n, mp.value
        rowptr = np.ctypeslib.as_array(
            ctypes.cast(rp, ctypes.POINTER(ctypes.c_int32)), (n + 1,)).copy()
        col = (np.ctypeslib.as_array(
            ctypes.cast(cp, ctypes.POINTER(ctypes.c_int32)), (m,)).copy()
            if m else np.zeros(0, dtype=np.int32))
    finally:
        lib.dp_free(rp)
        lib.dp_free(cp)
    return Graph(rowptr, col)


def edge_mirror(graph: Graph) -> np.ndarray:
    """mirror[e] = slot of the reverse edge of slot e (symmetric simple CSR
    with sorted rows, e.g. from ``symmetrize``)."""
    from .. import _lib
    mirror = np.empty(max(graph.m, 1), dtype=np.int32)
    _lib.check(_lib.load().dp_edge_mirror(_lib.ptr(graph.rowptr),
                                          _lib.ptr(graph.col), graph.n,
                                          _lib.ptr(mirror), 0))
    return mirror[:graph.m]


def mst_inputs(graph: Graph, seed: int) -> tuple:
    """MST input (MSTF / MSTV): the symmetric simple graph,
    symmetric weights and canonical edge ids.  eid[e] = min(e, mirror[e]) is
    the slot of the (min, max) copy of the undirected edge; its weight is the
    reference rule's draw at that slot (graphs.py:184-187, [1, 9]), shared by
    both copies.  Returns (graph, weight int32[m], eid int32[m])."""
    g = symmetrize(graph)
    eid = np.minimum(np.arange(g.m, dtype=np.int32), edge_mirror(g))
    w = edge_weights(g, seed)[eid] if g.m else np.zeros(0, dtype=np.int32)
    return g, np.ascontiguousarray(w, dtype=np.int32), \
        np.ascontiguousarray(eid, dtype=np.int32)


# ---------------------------------------------------------------------------
# Bezier tessellation input
# ---------------------------------------------------------------------------

def bezier_curves(n: int, seed: int) -> np.ndarray:
    """float32[n, 3, 2] control points, U[0,1)^2."""
    return _rng("curves", n, seed).random((n, 3, 2), dtype=np.float32)


# ---------------------------------------------------------------------------
# survey propagation input: random k-SAT (the paper's RAND-3 / 5-SAT sets,
# PAPER.md:436; generator builder-defined)
# ---------------------------------------------------------------------------

@dataclass(frozen=True, eq=False)
class Formula:
    """k-SAT factor graph.  Clause a owns edges [a*k, (a+1)*k) with
    ``lits[e] = var << 1 | negated``; ``occ_row``/``occ`` list each
    variable's edges in ascending edge order (variable-major CSR)."""
    k: int
    nvars: int
    lits: np.ndarray
    occ_row: np.ndarray
    occ: np.ndarray

    @property
    def nclauses(self) -> int:
        return int(self.lits.shape[0]) // self.k


def random_ksat(nvars: int, k: int, ratio: float, seed: int) -> Formula:
    """round(ratio * nvars) clauses of k distinct variables each, uniform
    signs; stream ``sat`` keyed by (nvars, k, seed)."""
    if nvars < k:
        raise ValueError(f"a {k}-SAT formula needs at least {k} variables")
    rng = _rng("sat", nvars, k, seed)
    m = int(round(ratio * nvars))
    var = rng.integers(0, nvars, size=(m, k), dtype=np.int64)
    while True:  # redraw clauses that repeat a variable
        srt = np.sort(var, axis=1)
        bad = np.flatnonzero((srt[:, 1:] == srt[:, :-1]).any(axis=1))
        if bad.size == 0:
            break
        var[bad] = rng.integers(0, nvars, size=(bad.size, k), dtype=np.int64)
    neg = rng.integers(0, 2, size=(m, k), dtype=np.int64)
    lits = ((var << 1) | neg).reshape(-1).astype(np.int32)
    v = var.reshape(-1)
    occ = np.argsort(v, kind="stable").astype(np.int32)
    occ_row = np.concatenate(([0], np.cumsum(np.bincount(v, minlength=nvars))))
    return Formula(k, nvars, lits, occ_row.astype(np.int32), occ)


def sp_initial_surveys(f: Formula, seed: int) -> np.ndarray:
    """eta0 ~ U[0, 1) per edge, float64 (stream ``sat_eta``)."""
    return _rng("sat_eta", f.nvars, f.k, seed).random(f.lits.shape[0])


def make_formula(spec: DatasetSpec) -> Formula:
    if spec.kind not in SAT_KINDS:
        raise ValueError(f"dataset kind {spec.kind!r} is not a k-SAT formula")
    k, ratio = SAT_KINDS[spec.kind]
    return random_ksat(spec.size, k, ratio, spec.seed)
