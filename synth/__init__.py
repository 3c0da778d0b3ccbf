"""Seeded synthetic inputs for the WBPR hot path (configs C1-C5 of BASELINE.json).

This module holds none of the method's arithmetic: it only draws graphs shaped
like the paper's workloads (§4.1) and formats them as CSR.
Both ``oracle/`` and the CUDA path consume its output; it imports neither.
The recipe for every config is written out in DESIGN.md ("Input recipe").

The heavy generators live in ``synth/gen.c`` (built on first use with gcc,
OpenMP when available) and use a counter-based splitmix64 stream, so a given
(config, seed) always yields identical bytes regardless of thread count.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess
import threading
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_SRCS = (_SRC, os.path.join(_HERE, "ingest.c"))
_LIB = os.path.join(_HERE, "libsynth.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile synth/gen.c + synth/ingest.c into synth/libsynth.so (gcc -O3 -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(f) for f in _SRCS):
        tmp = _LIB + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC", *_SRCS, "-o", tmp]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB)
    return _LIB


def _L():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i32, i64, u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
            lib.synth_random_pairs.argtypes = [i32, i64, u64, P, P, P]
            lib.synth_random_pairs.restype = i64
            lib.synth_grid_count.argtypes = [i32, i32]
            lib.synth_grid_count.restype = i64
            lib.synth_grid.argtypes = [i32, i32, i32, u64, P, P, P]
            lib.synth_grid.restype = i64
            lib.synth_rmat.argtypes = [i32, i32, u64, P, P, P]
            lib.synth_rmat.restype = i64
            lib.synth_bipartite.argtypes = [i32, i32, i64, u64, P, P]
            lib.synth_bipartite.restype = i64
            lib.synth_select_pairs.argtypes = [i32, P, P, i32, i32, u64, P, P]
            lib.synth_select_pairs.restype = i32
            lib.synth_select_hubs.argtypes = [i32, P, P, i32, P, P]
            lib.synth_select_hubs.restype = i32
            lib.synth_shuffle_rows.argtypes = [i64, P, P, P, u64]
            lib.synth_shuffle_rows.restype = None
            lib.synth_rlg_count.argtypes = [i32, i32, i32]
            lib.synth_rlg_count.restype = i64
            lib.synth_rlg.argtypes = [i32, i32, i32, i32, u64, P, P, P]
            lib.synth_rlg.restype = i64
            lib.synth_genrmf_count.argtypes = [i32, i32]
            lib.synth_genrmf_count.restype = i64
            lib.synth_genrmf.argtypes = [i32, i32, i32, i32, u64, P, P, P]
            lib.synth_genrmf.restype = i64
            lib.synth_draw.argtypes = [u64, u64, u64]
            lib.synth_draw.restype = u64
            for f in (lib.ingest_dimacs, lib.ingest_konect):
                f.argtypes = [ctypes.c_char_p, ctypes.POINTER(_IngestResult)]
                f.restype = i32
            lib.ingest_snap.argtypes = [ctypes.c_char_p, i32, ctypes.POINTER(_IngestResult)]
            lib.ingest_snap.restype = i32
            lib.ingest_free.argtypes = [ctypes.POINTER(_IngestResult)]
            lib.ingest_free.restype = None
            lib.synth_set_threads.argtypes = [i32]
            lib.synth_set_threads.restype = None
            # (torchrun exports OMP_NUM_THREADS=1 to every rank: use this rank's share of the cores)
            nt = os.environ.get("WBPR_SYNTH_THREADS")
            if nt is None and os.environ.get("LOCAL_WORLD_SIZE"):
                try:
                    cores = len(os.sched_getaffinity(0))
                except Exception:
                    cores = os.cpu_count() or 1
                nt = max(1, cores // int(os.environ["LOCAL_WORLD_SIZE"]))
            if nt is not None:
                lib.synth_set_threads(int(nt))
            _lib = lib
    return _lib


class _IngestResult(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("m", ctypes.c_int64),
                ("src", ctypes.POINTER(ctypes.c_int32)), ("dst", ctypes.POINTER(ctypes.c_int32)),
                ("cap", ctypes.POINTER(ctypes.c_int32)), ("s", ctypes.c_int64), ("t", ctypes.c_int64),
                ("nL", ctypes.c_int64), ("nR", ctypes.c_int64), ("declared_m", ctypes.c_int64),
                ("self_loops", ctypes.c_int64), ("duplicates", ctypes.c_int64), ("err_line", ctypes.c_int64)]


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclasses.dataclass
class Graph:
    """A max-flow instance in CSR form (the boundary's input format).

    row_off: int64[n+1]; col: int32[m]; cap: int32[m]; edges grouped by source row.
    """
    n: int
    row_off: np.ndarray
    col: np.ndarray
    cap: np.ndarray
    s: int
    t: int
    name: str = ""
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def m(self) -> int:
        return int(self.col.shape[0])

    def edges(self):
        """(src, dst, cap) arrays in CSR order."""
        src = np.repeat(np.arange(self.n, dtype=np.int32), np.diff(self.row_off))
        return src, self.col, self.cap


def csr_from_edges(n: int, src, dst, cap) -> tuple:
    """Group an edge list by source row (stable: keeps the input order within a row)."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int32)
    cap = np.asarray(cap, dtype=np.int32)
    order = np.argsort(src, kind="stable")
    counts = np.bincount(src, minlength=n) if src.size else np.zeros(n, dtype=np.int64)
    row_off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_off[1:])
    return row_off, np.ascontiguousarray(dst[order]), np.ascontiguousarray(cap[order])


def from_edges(n, src, dst, cap, s, t, name="", **meta) -> Graph:
    ro, c, w = csr_from_edges(n, src, dst, cap)
    return Graph(n=int(n), row_off=ro, col=c, cap=w, s=int(s), t=int(t), name=name, meta=dict(meta))


def shuffle_rows(g: Graph, seed: int) -> Graph:
    """Same graph with each CSR row's entries in a seeded random order."""
    col = g.col.copy()
    cap = g.cap.copy()
    _L().synth_shuffle_rows(g.n, _p(g.row_off), _p(col), _p(cap), seed)
    return dataclasses.replace(g, col=col, cap=cap)


# --------------------------------------------------------------------------- C1
def random_graph(n: int = 1024, m: int = 8192, seed: int = 1, s: int = 0, t: Optional[int] = None) -> Graph:
    """C1: m distinct ordered pairs (u != v), uniform by rejection, cap U[1,100]."""
    t = n - 1 if t is None else t
    src = np.empty(m, np.int32)
    dst = np.empty(m, np.int32)
    cap = np.empty(m, np.int32)
    k = _L().synth_random_pairs(n, m, seed, _p(src), _p(dst), _p(cap))
    return from_edges(n, src[:k], dst[:k], cap[:k], s, t, name=f"rand-n{n}-m{m}-seed{seed}", config="C1")


# --------------------------------------------------------------------------- C2
def grid(W: int = 1024, H: int = 1024, random_caps: bool = False, seed: int = 1) -> Graph:
    """C2: W x H 4-neighbour grid (both directions), super S -> column x=0,
    column x=W-1 -> super T; unit or U[1,100] caps; super caps = incident sums."""
    L = _L()
    m = L.synth_grid_count(W, H)
    src = np.empty(m, np.int32)
    dst = np.empty(m, np.int32)
    cap = np.empty(m, np.int32)
    k = L.synth_grid(W, H, 1 if random_caps else 0, seed, _p(src), _p(dst), _p(cap))
    assert k == m
    N = W * H
    return from_edges(N + 2, src, dst, cap, N, N + 1,
                      name=f"grid-{W}x{H}-{'rand' if random_caps else 'unit'}", config="C2",
                      W=W, H=H, random_caps=bool(random_caps))


# --------------------------------------------------------------------------- C3/C5
def rmat_edges(scale: int, edgefactor: int = 16, seed: int = 1):
    """R-MAT (Graph500 0.57/0.19/0.19/0.05), self-loops removed, duplicates
    collapsed, vertex ids permuted, caps U[1,100] drawn after collapsing."""
    M = (1 << scale) * edgefactor
    src = np.empty(M, np.int32)
    dst = np.empty(M, np.int32)
    cap = np.empty(M, np.int32)
    k = _L().synth_rmat(scale, edgefactor, seed, _p(src), _p(dst), _p(cap))
    return src[:k].copy(), dst[:k].copy(), cap[:k].copy()


def select_pairs(n, row_off, col, k=20, nstarts=256, seed=1):
    srcs = np.empty(k, np.int32)
    snks = np.empty(k, np.int32)
    got = _L().synth_select_pairs(n, _p(row_off), _p(col), k, nstarts, seed, _p(srcs), _p(snks))
    return srcs[:got].copy(), snks[:got].copy()


def select_hubs(n, row_off, col, k=20):
    srcs = np.empty(k, np.int32)
    snks = np.empty(k, np.int32)
    _L().synth_select_hubs(n, _p(row_off), _p(col), k, _p(srcs), _p(snks))
    return srcs, snks


def add_super_terminals(n, src, dst, cap, sources, sinks):
    """Super-source S=n -> each source (cap = its out-cap sum); each sink ->
    super-sink T=n+1 (cap = its in-cap sum). P:432; caps per S:382."""
    outc = np.bincount(src, weights=cap, minlength=n).astype(np.int64)
    inc = np.bincount(dst, weights=cap, minlength=n).astype(np.int64)
    S, T = n, n + 1
    sources = np.asarray(sources, np.int32)
    sinks = np.asarray(sinks, np.int32)
    s_caps = np.minimum(outc[sources], 2**31 - 1).astype(np.int32)
    t_caps = np.minimum(inc[sinks], 2**31 - 1).astype(np.int32)
    src2 = np.concatenate([src, np.full(len(sources), S, np.int32), sinks])
    dst2 = np.concatenate([dst, sources, np.full(len(sinks), T, np.int32)])
    cap2 = np.concatenate([cap, s_caps, t_caps])
    return n + 2, src2, dst2, cap2, S, T


def rmat(scale: int = 22, edgefactor: int = 16, seed: int = 1, rule: str = "paper",
         npairs: int = 20, nstarts: int = 256) -> Graph:
    """C3/C5: R-MAT instance with 20 source/sink pairs behind super terminals.

    rule="paper": BFS-chosen pairs with top-quartile depth (reading in
    DESIGN.md); rule="hub20": top-20 out-degree sources, top-20 in-degree sinks."""
    n = 1 << scale
    src, dst, cap = rmat_edges(scale, edgefactor, seed)
    ro, col, _ = csr_from_edges(n, src, dst, cap)
    if rule == "paper":
        so, si = select_pairs(n, ro, col, npairs, nstarts, seed)
    elif rule == "hub20":
        so, si = select_hubs(n, ro, col, npairs)
    else:
        raise ValueError(rule)
    N, src2, dst2, cap2, S, T = add_super_terminals(n, src, dst, cap, so, si)
    return from_edges(N, src2, dst2, cap2, S, T, name=f"rmat{scale}-ef{edgefactor}-{rule}-seed{seed}",
                      config="C3" if scale >= 20 else "C5", scale=scale, rule=rule,
                      sources=so.tolist(), sinks=si.tolist())


# --------------------------------------------------------------------------- C4
def bipartite_edges(nL: int = 1 << 20, nR: int = 1 << 20, nE: int = 1 << 24, seed: int = 1):
    """C4: nE uniform (l, r) draws with duplicates collapsed (0-based ids per side)."""
    l = np.empty(nE, np.int32)
    r = np.empty(nE, np.int32)
    k = _L().synth_bipartite(nL, nR, nE, seed, _p(l), _p(r))
    return l[:k].copy(), r[:k].copy()


# --------------------------------------------------------------------------- tiny
def tiny_random(n: int, m: int, cap_max: int, seed: int, self_loops: bool = True,
                zero_caps: bool = True, s: int = 0, t: Optional[int] = None) -> Graph:
    """Tiny adversarial instance for brute-force pins: parallel, antiparallel
    and (optionally) self-loop edges, caps in [0 or 1, cap_max]."""
    rng = np.random.default_rng(seed)
    t = n - 1 if t is None else t
    src = rng.integers(0, n, size=m).astype(np.int32)
    dst = rng.integers(0, n, size=m).astype(np.int32)
    if not self_loops:
        bad = src == dst
        dst[bad] = (dst[bad] + 1 + rng.integers(0, n - 1, size=int(bad.sum()))) % n
    lo = 0 if zero_caps else 1
    cap = rng.integers(lo, cap_max + 1, size=m).astype(np.int32)
    g = from_edges(n, src, dst, cap, s, t, name=f"tiny-n{n}-m{m}-seed{seed}")
    return shuffle_rows(g, seed + 7)


# --------------------------------------------------------------------------- batch
@dataclasses.dataclass
class Batch:
    """Disjoint union of k instances (A10): vertex range [vbase[i], vbase[i+1])."""
    union: Graph
    vbase: np.ndarray
    s: np.ndarray
    t: np.ndarray
    parts: List[Graph]


def disjoint_union(parts: Sequence[Graph]) -> Batch:
    vbase = np.zeros(len(parts) + 1, np.int64)
    for i, g in enumerate(parts):
        vbase[i + 1] = vbase[i] + g.n
    N = int(vbase[-1])
    ro = np.zeros(N + 1, np.int64)
    eb = 0
    cols, caps = [], []
    for i, g in enumerate(parts):
        b = int(vbase[i])
        ro[b + 1:b + g.n + 1] = g.row_off[1:] + eb
        eb += g.m
        cols.append(g.col + np.int32(b))
        caps.append(g.cap)
    U = Graph(n=N, row_off=ro, col=np.concatenate(cols) if cols else np.zeros(0, np.int32),
              cap=np.concatenate(caps) if caps else np.zeros(0, np.int32), s=-1, t=-1, name=f"union{len(parts)}")
    s = np.array([int(vbase[i]) + g.s for i, g in enumerate(parts)], np.int64)
    t = np.array([int(vbase[i]) + g.t for i, g in enumerate(parts)], np.int64)
    return Batch(union=U, vbase=vbase, s=s, t=t, parts=list(parts))


def c5_batch(count: int = 64, scale: int = 18, first_seed: int = 1000, rule: str = "paper", lo: int = 0,
             hi: Optional[int] = None) -> List[Graph]:
    """C5 instances [lo, hi) of the 64-instance batch: instance i uses seed first_seed+i."""
    hi = count if hi is None else hi
    return [rmat(scale, 16, first_seed + i, rule) for i in range(lo, hi)]


# --------------------------------------------------------------------------- DIMACS-shaped (NEXT #4)
def washington_rlg(levels: int = 512, width: int = 512, deg: int = 3, capmax: int = 10000, seed: int = 1) -> Graph:
    """Washington random level graph (DIMACS 1st challenge shape, "S0"):
    default 512 x 512 x 3 -> 262,146 vertices, 785,920 arcs."""
    L = _L()
    m = L.synth_rlg_count(levels, width, deg)
    src, dst, cap = (np.empty(m, np.int32) for _ in range(3))
    k = L.synth_rlg(levels, width, deg, capmax, seed, _p(src), _p(dst), _p(cap))
    assert k == m
    N = levels * width
    return from_edges(N + 2, src, dst, cap, N, N + 1, name=f"rlg-{levels}x{width}x{deg}", config="S0")


def genrmf(a: int = 128, b: int = 128, c1: int = 1, c2: int = 10000, seed: int = 1) -> Graph:
    """Genrmf (DIMACS 1st challenge shape, "S1"): b frames of a x a grids;
    default a = b = 128 -> 2,097,152 vertices, 10,403,840 arcs."""
    L = _L()
    m = L.synth_genrmf_count(a, b)
    src, dst, cap = (np.empty(m, np.int32) for _ in range(3))
    k = L.synth_genrmf(a, b, c1, c2, seed, _p(src), _p(dst), _p(cap))
    assert k == m
    n = a * a * b
    return from_edges(n, src, dst, cap, 0, n - 1, name=f"genrmf-{a}x{b}", config="S1")


# --------------------------------------------------------------------------- dataset files (NEXT #4)
class IngestError(ValueError):
    """A dataset file that does not parse (code, 1-based line)."""

    MESSAGES = {-1: "cannot open or read the file", -2: "no 'p max' problem line",
                -3: "no source or no sink designated", -4: "malformed line",
                -5: "vertex id out of range", -6: "capacity out of range", -7: "out of memory"}

    def __init__(self, path, code, line):
        self.code, self.line = int(code), int(line)
        super().__init__(f"{path}: {self.MESSAGES.get(self.code, 'error')}"
                         + (f" at line {self.line}" if self.line else "") + f" (code {self.code})")


def _ingest(fn, path, *args):
    r = _IngestResult()
    rc = fn(os.fsencode(path), *args, ctypes.byref(r))
    if rc != 0:
        raise IngestError(path, rc, r.err_line)
    try:
        m = int(r.m)

        def take(ptr):
            if m == 0 or not ptr:
                return np.zeros(0, np.int32)
            return np.ctypeslib.as_array(ptr, shape=(m,)).copy()
        out = dict(n=int(r.n), src=take(r.src), dst=take(r.dst), cap=take(r.cap) if r.cap else None,
                   s=int(r.s), t=int(r.t), nL=int(r.nL), nR=int(r.nR), declared_m=int(r.declared_m),
                   self_loops=int(r.self_loops), duplicates=int(r.duplicates))
    finally:
        _L().ingest_free(ctypes.byref(r))
    return out


def read_dimacs(path: str) -> Graph:
    """DIMACS max-flow file (`p max N M`, `n ID s|t`, `a U V CAP`, 1-based) -> Graph with its
    designated s and t (the Washington / Genrmf networks of Table 1).
    meta['declared_m'] is the problem line's arc count (a mismatch is reported, not fatal)."""
    d = _ingest(_L().ingest_dimacs, path)
    return from_edges(d["n"], d["src"], d["dst"], d["cap"], d["s"], d["t"], name=os.path.basename(path),
                      config="dimacs", declared_m=d["declared_m"], arc_count_mismatch=d["declared_m"] != len(d["src"]))


def write_dimacs(g: Graph, path: str, comment: str = "") -> None:
    """Serialise a Graph as a DIMACS max-flow file (round-trip partner of read_dimacs)."""
    src, dst, cap = g.edges()
    with open(path, "w") as f:
        if comment:
            f.write(f"c {comment}\n")
        f.write(f"p max {g.n} {g.m}\nn {g.s + 1} s\nn {g.t + 1} t\n")
        body = np.stack([src.astype(np.int64) + 1, dst.astype(np.int64) + 1, cap.astype(np.int64)], axis=1)
        np.savetxt(f, body, fmt="a %d %d %d")


def read_snap(path: str, cap: int = 1):
    """SNAP edge list -> (n, src, dst, cap): ids remapped densely in order of first appearance,
    self-loops dropped, duplicate lines merged with their capacities summed;
    capacity `cap` per line ("The edge capacity of graphs in SNAP is set to 1", Table 1)."""
    d = _ingest(_L().ingest_snap, path, int(cap))
    return d["n"], d["src"], d["dst"], d["cap"]


def snap_instance(path: str, npairs: int = 20, nstarts: int = 256, seed: int = 1, cap: int = 1) -> Graph:
    """A SNAP network as the paper's multi-source multi-sink instance: `npairs`
    BFS-selected source/sink pairs (the same rule as C3, `select_pairs`) behind a super-source
    and a super-sink with incident-sum capacities."""
    n, src, dst, c = read_snap(path, cap)
    ro, col, _ = csr_from_edges(n, src, dst, c)
    so, si = select_pairs(n, ro, col, npairs, nstarts, seed)
    N, src2, dst2, cap2, S, T = add_super_terminals(n, src, dst, c, so, si)
    return from_edges(N, src2, dst2, cap2, S, T, name=os.path.basename(path), config="snap",
                      sources=so.tolist(), sinks=si.tolist())


def read_konect(path: str):
    """KONECT bipartite edge list -> (nL, nR, l, r) with 0-based ids per side, weights ignored,
    duplicate pairs collapsed; side sizes = max(header `% E L R`, largest id)."""
    d = _ingest(_L().ingest_konect, path)
    return d["nL"], d["nR"], d["src"], d["dst"]
