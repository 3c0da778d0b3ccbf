"""Thin Python binding of libwbpr.so (include/wbpr.h) — argument marshalling only.

Every step of the max-flow path runs in the library's sm_100a kernels; torch is
used for device memory (the caller-allocated workspace, inputs, outputs) and for
the current CUDA stream.  There is no CPU fallback: if the extension is missing
or no GPU is present, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libwbpr.so")

WBPR_LAYOUT_BCSR = 0
WBPR_LAYOUT_RCSR = 1
_LAYOUTS = {"bcsr": 0, "rcsr": 1, 0: 0, 1: 1}

# every symbol include/wbpr.h declares
EXPORTS = (
    "wbpr_default_options", "wbpr_workspace_size", "wbpr_maxflow_solve", "wbpr_maxflow_solve_batch",
    "wbpr_bipartite_workspace_size", "wbpr_bipartite_match", "wbpr_residual_view", "wbpr_build_residual",
    "wbpr_status_string", "wbpr_last_error", "wbpr_version", "wbpr_trace_view", "wbpr_barrier_cost",
)


class WbprError(RuntimeError):
    def __init__(self, status: int, name: str, msg: str):
        super().__init__(f"{name} ({status}): {msg}")
        self.status = status
        self.name = name


class Csr(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("m", ctypes.c_int64), ("row_offsets", ctypes.c_void_p),
                ("col", ctypes.c_void_p), ("cap", ctypes.c_void_p), ("on_host", ctypes.c_int32)]


class Options(ctypes.Structure):
    _fields_ = [("layout", ctypes.c_int32), ("gr_beta", ctypes.c_float), ("gap_mode", ctypes.c_int32),
                ("max_rounds", ctypes.c_int64), ("grid_blocks", ctypes.c_int32), ("timeout_ms", ctypes.c_int32),
                ("push_mode", ctypes.c_int32), ("gr_gamma", ctypes.c_float), ("l2_persist", ctypes.c_int32),
                ("bfs_mode", ctypes.c_int32), ("small_mode", ctypes.c_int32), ("schedule", ctypes.c_int32),
                ("phase2", ctypes.c_int32), ("trace_rounds", ctypes.c_int32), ("batch_groups", ctypes.c_int32),
                ("debug_stop", ctypes.c_int32), ("tiny_mode", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int64) for name in (
        "flow_value", "cut_capacity", "n", "m", "M", "rounds", "global_relabels", "bfs_levels", "pushes",
        "relabels", "arcs_scanned", "bfs_arcs_scanned", "compaction_candidates", "avq_total", "gap_lifts",
        "self_loops_ignored", "bad_edge_index", "excess_total")] + [
        ("build_ms", ctypes.c_float), ("solve_ms", ctypes.c_float), ("extract_ms", ctypes.c_float),
        ("total_ms", ctypes.c_float), ("grid_blocks", ctypes.c_int32), ("block_threads", ctypes.c_int32),
        ("kernel_launches", ctypes.c_int64), ("t_barrier_ns", ctypes.c_int64), ("t_flush_ns", ctypes.c_int64),
        ("t_round_ns", ctypes.c_int64), ("phase_ns", ctypes.c_int64 * 10), ("phase_count", ctypes.c_int64 * 10),
        ("bfs_arcs_bottom_up", ctypes.c_int64), ("tiny_path", ctypes.c_int64)]

    def as_dict(self):
        d = {}
        for f in self._fields_:
            v = getattr(self, f[0])
            d[f[0]] = list(v) if isinstance(v, ctypes.Array) else v
        return d


class Residual(ctypes.Structure):
    _fields_ = [("layout", ctypes.c_int32), ("n", ctypes.c_int64), ("M", ctypes.c_int64), ("Mf", ctypes.c_int64)] + [
        (name, ctypes.c_void_p) for name in ("off", "arc", "mate", "cap0", "roff", "rarc", "bcf", "e", "h", "seg",
                                             "avq")] + [("avq_len", ctypes.c_int64), ("excess_total", ctypes.c_int64)]


_lib = None


def load():
    """Load libwbpr.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("WBPR_LIB", LIB_PATH)   # experiment builds (build.py --variant=...)
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -m paper_2404_00270_b200.build` "
                          "(the CUDA path has no fallback)")
    lib = ctypes.CDLL(path)
    P, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.wbpr_default_options.argtypes = [ctypes.POINTER(Options)]
    lib.wbpr_workspace_size.argtypes = [i64, i64, i32, ctypes.POINTER(Options), ctypes.POINTER(ctypes.c_size_t)]
    lib.wbpr_maxflow_solve.argtypes = [ctypes.POINTER(Csr), i64, i64, ctypes.POINTER(Options), P, ctypes.c_size_t,
                                       P, ctypes.POINTER(Stats), P]
    lib.wbpr_maxflow_solve_batch.argtypes = [ctypes.POINTER(Csr), i32, P, P, P, ctypes.POINTER(Options), P,
                                             ctypes.c_size_t, P, P, P, ctypes.POINTER(Stats), P]
    lib.wbpr_bipartite_workspace_size.argtypes = [i64, i64, i64, ctypes.POINTER(Options),
                                                  ctypes.POINTER(ctypes.c_size_t)]
    lib.wbpr_bipartite_match.argtypes = [i64, i64, i64, P, P, ctypes.POINTER(Options), P, ctypes.c_size_t, P,
                                         ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(Stats), P]
    lib.wbpr_residual_view.argtypes = [P, ctypes.POINTER(Residual)]
    lib.wbpr_build_residual.argtypes = [ctypes.POINTER(Csr), ctypes.POINTER(Options), P, ctypes.c_size_t,
                                        ctypes.POINTER(Stats), P]
    for f in ("wbpr_default_options", "wbpr_workspace_size", "wbpr_maxflow_solve", "wbpr_maxflow_solve_batch",
              "wbpr_bipartite_workspace_size", "wbpr_bipartite_match", "wbpr_residual_view", "wbpr_build_residual"):
        getattr(lib, f).restype = ctypes.c_int32
    lib.wbpr_trace_view.argtypes = [P, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_int64),
                                    ctypes.POINTER(ctypes.c_int32)]
    lib.wbpr_trace_view.restype = ctypes.c_int32
    lib.wbpr_barrier_cost.argtypes = [i32, i32, ctypes.POINTER(ctypes.c_double), P]
    lib.wbpr_barrier_cost.restype = ctypes.c_int32
    lib.wbpr_status_string.argtypes = [i32]
    lib.wbpr_status_string.restype = ctypes.c_char_p
    lib.wbpr_last_error.restype = ctypes.c_char_p
    lib.wbpr_version.restype = ctypes.c_char_p
    _lib = lib
    return lib


def _check(st: int):
    if st != 0:
        L = load()
        raise WbprError(st, L.wbpr_status_string(st).decode(), L.wbpr_last_error().decode())


def options(layout="bcsr", gr_beta: float = 0.0, gap_mode: int = 0, max_rounds: int = 0, grid_blocks: int = 0,
            timeout_ms: int = 0, push_mode: Optional[int] = None, gr_gamma: Optional[float] = None,
            l2_persist: Optional[int] = None, bfs_mode: Optional[int] = None,
            small_mode: Optional[int] = None, schedule: Optional[str] = None,
            phase2: Optional[int] = None, trace_rounds: Optional[int] = None,
            batch_groups: Optional[int] = None, debug_stop: Optional[int] = None,
            tiny_mode: Optional[int] = None) -> Options:
    o = Options()
    _check(load().wbpr_default_options(ctypes.byref(o)))
    o.layout = _LAYOUTS[layout]
    if gr_beta > 0:
        o.gr_beta = gr_beta
    o.gap_mode = gap_mode
    o.max_rounds = max_rounds
    o.grid_blocks = grid_blocks
    if timeout_ms > 0:
        o.timeout_ms = timeout_ms
    if push_mode is not None:
        o.push_mode = push_mode
    if gr_gamma is not None:
        o.gr_gamma = gr_gamma
    if l2_persist is not None:
        o.l2_persist = l2_persist
    if bfs_mode is not None:
        o.bfs_mode = bfs_mode
    if small_mode is not None:
        o.small_mode = small_mode
    if schedule is not None:
        o.schedule = {"vc": 0, "tc": 1, 0: 0, 1: 1}[schedule]
    if phase2 is not None:
        o.phase2 = phase2
    if trace_rounds is not None:
        o.trace_rounds = trace_rounds
    if batch_groups is not None:
        o.batch_groups = batch_groups
    if debug_stop is not None:
        o.debug_stop = debug_stop
    if tiny_mode is not None:
        o.tiny_mode = tiny_mode
    return o


def _torch():
    import torch
    return torch


def _stream_ptr(device):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def workspace_size(n: int, m: int, k: int = 1, opt: Optional[Options] = None) -> int:
    b = ctypes.c_size_t()
    _check(load().wbpr_workspace_size(n, m, k, ctypes.byref(opt or options()), ctypes.byref(b)))
    return b.value


class Workspace:
    """A reusable device workspace (torch uint8 tensor) sized for a solve."""

    def __init__(self, nbytes: int, device="cuda"):
        torch = _torch()
        self.tensor = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        self.nbytes = int(self.tensor.numel())

    @property
    def ptr(self):
        return ctypes.c_void_p(self.tensor.data_ptr())

    def ensure(self, nbytes):
        if nbytes > self.nbytes:
            self.__init__(nbytes, self.tensor.device)
        return self


def _as_csr(row_off, col, cap):
    """Csr struct from torch tensors (all CUDA -> device pointers; all CPU -> host pointers)."""
    torch = _torch()
    ts = [row_off, col, cap]
    for t, dt in zip(ts, (torch.int64, torch.int32, torch.int32)):
        if t.dtype != dt or not t.is_contiguous():
            raise TypeError("row_off int64 / col int32 / cap int32 contiguous tensors expected")
    on_host = not row_off.is_cuda
    if any(t.is_cuda == on_host for t in ts):
        raise TypeError("CSR tensors must all be on the GPU or all on the host")
    c = Csr()
    c.n = row_off.numel() - 1
    c.m = col.numel()
    c.row_offsets = row_off.data_ptr()
    c.col = col.data_ptr() if c.m else 0
    c.cap = cap.data_ptr() if c.m else 0
    c.on_host = 1 if on_host else 0
    return c


def maxflow(row_off, col, cap, s: int, t: int, layout="bcsr", workspace: Optional[Workspace] = None,
            bitmap=None, device=None, **opt):
    """Maximum flow value and canonical min-cut bitmap of (G, s, t).

    row_off int64[n+1], col int32[m], cap int32[m] torch tensors, all on the GPU or all on
    the host (then copied in the call; the bitmap comes back on the host).
    Returns (flow:int, bitmap:Tensor[int32 words], stats:dict)."""
    torch = _torch()
    L = load()
    o = options(layout, **opt)
    c = _as_csr(row_off, col, cap)
    dev = torch.device(device) if device is not None else (row_off.device if row_off.is_cuda else torch.device("cuda"))
    need = workspace_size(c.n, c.m, 1, o)
    ws = (workspace or Workspace(need, dev)).ensure(need)
    words = (c.n + 31) // 32
    if bitmap is None:
        bitmap = torch.empty(words, dtype=torch.int32, device=dev if c.on_host == 0 else "cpu",
                             pin_memory=bool(c.on_host))
    st = Stats()
    with torch.cuda.device(dev):
        _check(L.wbpr_maxflow_solve(ctypes.byref(c), s, t, ctypes.byref(o), ws.ptr, ws.nbytes,
                                    ctypes.c_void_p(bitmap.data_ptr()), ctypes.byref(st), _stream_ptr(dev)))
    return int(st.flow_value), bitmap, st.as_dict()


def maxflow_batch(row_off, col, cap, vbase: Sequence[int], s: Sequence[int], t: Sequence[int], layout="bcsr",
                  workspace: Optional[Workspace] = None, bitmap=None, device=None, **opt):
    """k independent instances as one disjoint-union CSR (A10).
    Returns (flows:np.int64[k], cutcaps:np.int64[k], bitmap, stats)."""
    torch = _torch()
    L = load()
    o = options(layout, **opt)
    c = _as_csr(row_off, col, cap)
    dev = torch.device(device) if device is not None else (row_off.device if row_off.is_cuda else torch.device("cuda"))
    vb = np.ascontiguousarray(vbase, np.int64)
    sa = np.ascontiguousarray(s, np.int64)
    ta = np.ascontiguousarray(t, np.int64)
    k = len(sa)
    need = workspace_size(c.n, c.m, k, o)
    ws = (workspace or Workspace(need, dev)).ensure(need)
    words = (c.n + 31) // 32
    if bitmap is None:
        bitmap = torch.empty(words, dtype=torch.int32, device=dev if c.on_host == 0 else "cpu",
                             pin_memory=bool(c.on_host))
    flows = np.zeros(k, np.int64)
    cuts = np.zeros(k, np.int64)
    st = Stats()
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    with torch.cuda.device(dev):
        _check(L.wbpr_maxflow_solve_batch(ctypes.byref(c), k, P(vb), P(sa), P(ta), ctypes.byref(o), ws.ptr,
                                          ws.nbytes, ctypes.c_void_p(bitmap.data_ptr()), P(flows), P(cuts),
                                          ctypes.byref(st), _stream_ptr(dev)))
    return flows, cuts, bitmap, st.as_dict()


def bipartite_match(nL: int, nR: int, l, r, layout="bcsr", workspace: Optional[Workspace] = None, **opt):
    """Maximum bipartite matching (A9).  l, r: int32 CUDA tensors.
    Returns (size:int, match_of_left:Tensor int32[nL] on the GPU, stats)."""
    torch = _torch()
    L = load()
    o = options(layout, **opt)
    dev = l.device
    E = l.numel()
    b = ctypes.c_size_t()
    _check(L.wbpr_bipartite_workspace_size(nL, nR, E, ctypes.byref(o), ctypes.byref(b)))
    ws = (workspace or Workspace(b.value, dev)).ensure(b.value)
    match = torch.empty(max(nL, 1), dtype=torch.int32, device=dev)
    size = ctypes.c_int64()
    st = Stats()
    with torch.cuda.device(dev):
        _check(L.wbpr_bipartite_match(nL, nR, E, ctypes.c_void_p(l.data_ptr() if E else 0),
                                      ctypes.c_void_p(r.data_ptr() if E else 0), ctypes.byref(o), ws.ptr, ws.nbytes,
                                      ctypes.c_void_p(match.data_ptr()), ctypes.byref(size), ctypes.byref(st),
                                      _stream_ptr(dev)))
    return int(size.value), match[:nL], st.as_dict()


def residual(workspace: Workspace) -> dict:
    """Host copies of the residual state the last build/solve left in `workspace`."""
    torch = _torch()
    v = Residual()
    _check(load().wbpr_residual_view(workspace.ptr, ctypes.byref(v)))
    base = workspace.tensor.data_ptr()
    ws = workspace.tensor

    def grab(ptr, count, dtype):
        if not ptr or count <= 0:
            return np.zeros(0, dtype=np.int64 if dtype == torch.int64 else np.int32)
        off = ptr - base
        nb = count * (8 if dtype == torch.int64 else 4)
        return ws[off:off + nb].view(dtype).cpu().numpy()

    n = v.n
    out = dict(layout=v.layout, n=n, M=v.M, Mf=v.Mf)
    if v.layout == 0:   # gapped: vertex u owns slots [seg[u, 0], seg[u, 1]) of the M-slot space
        arc = grab(v.arc, 2 * v.M, torch.int32).reshape(-1, 2)
        out.update(seg=grab(v.seg, 2 * n, torch.int32).reshape(-1, 2), col=arc[:, 0].copy(), cf=arc[:, 1].copy(),
                   mate=grab(v.mate, v.M, torch.int32), cap0=grab(v.cap0, v.M, torch.int32))
    else:
        farc = grab(v.arc, 2 * v.Mf, torch.int32).reshape(-1, 2)
        rarc = grab(v.rarc, 2 * v.Mf, torch.int32).reshape(-1, 2)
        out.update(foff=grab(v.off, n + 1, torch.int32), fcol=farc[:, 0].copy(), fcf=farc[:, 1].copy(),
                   cap0=grab(v.cap0, v.Mf, torch.int32), roff=grab(v.roff, n + 1, torch.int32),
                   rcol=rarc[:, 0].copy(), fidx=rarc[:, 1].copy(), bcf=grab(v.bcf, v.Mf, torch.int32))
    out["e"] = grab(v.e, n, torch.int64)
    out["h"] = grab(v.h, n, torch.int32)
    if v.avq:   # debug_stop solves: the compacted active-vertex queue and Excess_total
        out["avq"] = grab(v.avq, v.avq_len, torch.int32)
        out["excess_total"] = int(v.excess_total)
    return out


def build_residual(row_off, col, cap, layout="bcsr", workspace: Optional[Workspace] = None):
    """Run construction (A1) only and return (host copies of the layout, stats)."""
    torch = _torch()
    L = load()
    o = options(layout)
    c = _as_csr(row_off, col, cap)
    dev = row_off.device if row_off.is_cuda else torch.device("cuda")
    need = workspace_size(c.n, c.m, 1, o)
    ws = (workspace or Workspace(need, dev)).ensure(need)
    st = Stats()
    with torch.cuda.device(dev):
        _check(L.wbpr_build_residual(ctypes.byref(c), ctypes.byref(o), ws.ptr, ws.nbytes, ctypes.byref(st),
                                     _stream_ptr(dev)))
    return residual(ws), st.as_dict()


TRACE_DTYPE = np.dtype([("round", "<i4"), ("warp", "<i4"), ("busy_ns", "<u4"), ("tasks", "<i4"), ("slots", "<i4"),
                        ("pushes", "<i4"), ("relabels", "<i4"), ("schedule", "<i4")])


def trace(workspace: Workspace) -> np.ndarray:
    """Per-warp workload records of the last traced solve: structured array [rounds, warps]."""
    ptr = ctypes.c_void_p()
    rounds = ctypes.c_int64()
    warps = ctypes.c_int32()
    _check(load().wbpr_trace_view(workspace.ptr, ctypes.byref(ptr), ctypes.byref(rounds), ctypes.byref(warps)))
    off = ptr.value - workspace.tensor.data_ptr()
    nbytes = rounds.value * warps.value * TRACE_DTYPE.itemsize
    raw = workspace.tensor[off:off + nbytes].cpu().numpy()
    return raw.view(TRACE_DTYPE).reshape(rounds.value, warps.value)


def barrier_cost(grid_blocks: int = 0, iters: int = 2000, device=None) -> float:
    """ns of device time per EMPTY grid-synchronous phase of the persistent solve kernel
    (wbpr_barrier_cost): the latency floor per phase."""
    torch = _torch()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    ns = ctypes.c_double()
    with torch.cuda.device(dev):
        _check(load().wbpr_barrier_cost(grid_blocks, iters, ctypes.byref(ns), _stream_ptr(dev)))
    return float(ns.value)


def version() -> str:
    return load().wbpr_version().decode()
