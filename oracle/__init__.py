"""CPU ORACLE for the WBPR hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path (``paper_2404_00270_b200``) and neither imports the other; the only
common module is ``synth`` (seeded input generators, no method arithmetic).

Contents (each function cites the passage it follows):
  maxflow()          FIFO push-relabel + gap + optional global relabel, two-phase
                     (oracle/maxflow_oracle.c; §2.2, Alg. 1)
  brute.*            Edmonds-Karp and exhaustive cut enumeration (pins)
  check.*            validity / certificate checks V1-V7
  residual_ref.*     the canonical BCSR / RCSR layouts written out from their
                     definitions (§3.2, Fig. 2(c),(d))
  matching.*         bipartite network per S:304 and matching validity

Parity status: every function here is pinned by tests/test_oracle_*.py
(brute force, closed forms, library routines, invariants); none is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess
import threading
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "maxflow_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle (plain gcc -O2, single-threaded)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.run(["gcc", "-O2", "-shared", "-fPIC", _SRC, "-o", tmp], check=True)
        os.replace(tmp, _LIB)
    return _LIB


def _L():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i32, i64 = ctypes.c_int32, ctypes.c_int64
            lib.oracle_maxflow.argtypes = [i64, i64, P, P, P, i64, i64, i32, i32, i32, P, P, P, P, P]
            lib.oracle_maxflow.restype = ctypes.c_int
            lib.oracle_initial_state.argtypes = [i64, i64, P, P, P, i64, i64, P, P, P, P]
            lib.oracle_initial_state.restype = ctypes.c_int
            _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclasses.dataclass
class OracleResult:
    flow: int            # F* = e(t) after phase 1 (Alg. 1 output)
    cut_capacity: int    # sum of c over input edges S* -> V\S*
    in_S: np.ndarray     # uint8[n], 1 iff v in S* (cannot reach t in G_f)
    edge_flow: np.ndarray  # int64[m] strict flow after phase 2 (None if phase2=False)
    stats: dict
    seconds: float

    def bitmap_words(self) -> np.ndarray:
        """S* packed LSB-first into uint32 words (bit v in word v>>5, position v&31)."""
        n = self.in_S.shape[0]
        nw = (n + 31) // 32
        bits = np.zeros(nw * 32, np.uint8)
        bits[:n] = self.in_S
        return np.packbits(bits, bitorder="little").view("<u4").astype(np.uint32)


def maxflow(n, row_off, col, cap, s, t, gr: bool = True, gap: bool = True, phase2: bool = True) -> OracleResult:
    """Exact max flow / canonical min cut of a CSR instance (see maxflow_oracle.c)."""
    row_off = np.ascontiguousarray(row_off, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    cap = np.ascontiguousarray(cap, np.int32)
    m = col.shape[0]
    flow = np.zeros(1, np.int64)
    cut = np.zeros(1, np.int64)
    in_S = np.zeros(n, np.uint8)
    ef = np.zeros(max(m, 1), np.int64)
    st = np.zeros(6, np.int64)
    t0 = time.perf_counter()
    rc = _L().oracle_maxflow(n, m, _p(row_off), _p(col), _p(cap), s, t, int(gr), int(gap), int(phase2),
                             _p(flow), _p(cut), _p(in_S), _p(ef), _p(st))
    dt = time.perf_counter() - t0
    if rc != 0:
        raise ValueError(f"oracle_maxflow rejected the instance (rc={rc})")
    stats = dict(pushes=int(st[0]), relabels=int(st[1]), global_relabels=int(st[2]), gaps=int(st[3]),
                 phase2_pushes=int(st[4]), phase2_relabels=int(st[5]))
    return OracleResult(int(flow[0]), int(cut[0]), in_S, ef[:m] if phase2 else None, stats, dt)


def maxflow_graph(g, **kw) -> OracleResult:
    return maxflow(g.n, g.row_off, g.col, g.cap, g.s, g.t, **kw)


def initial_state(n, row_off, col, cap, s, t):
    """(excess after preflow, Excess_total, exact labels after preflow, labels before preflow).

    Alg. 1 Step 0 then one reverse BFS from t; see
    oracle_initial_state in maxflow_oracle.c."""
    row_off = np.ascontiguousarray(row_off, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    cap = np.ascontiguousarray(cap, np.int32)
    e = np.zeros(n, np.int64)
    tot = np.zeros(1, np.int64)
    lv = np.zeros(n, np.int64)
    lv0 = np.zeros(n, np.int64)
    rc = _L().oracle_initial_state(n, col.shape[0], _p(row_off), _p(col), _p(cap), s, t, _p(e), _p(tot),
                                   _p(lv), _p(lv0))
    if rc != 0:
        raise ValueError("oracle_initial_state rejected the instance")
    return e, int(tot[0]), lv, lv0
