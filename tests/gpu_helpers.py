"""Helpers for the -m gpu parity tests: run the CUDA path through the C-ABI
binding and compare with the oracle on the same seeded synth inputs."""
import numpy as np

import oracle
from oracle import check


def to_dev(g, device="cuda"):
    import torch
    return (torch.from_numpy(np.ascontiguousarray(g.row_off)).to(device),
            torch.from_numpy(np.ascontiguousarray(g.col)).to(device),
            torch.from_numpy(np.ascontiguousarray(g.cap)).to(device))


def gpu_solve(g, layout="bcsr", ws=None, **opt):
    import paper_2404_00270_b200 as W
    ro, col, cap = to_dev(g)
    need = W.workspace_size(g.n, g.m, 1, W.options(layout))
    ws = (ws or W.Workspace(need)).ensure(need)
    F, bm, st = W.maxflow(ro, col, cap, g.s, g.t, layout=layout, workspace=ws, **opt)
    return F, bm.cpu().numpy().view(np.uint32), st, ws


def dense_bcsr(R):
    """The gapped BCSR view (segments [seg[u,0], seg[u,1]) in vertex order, unused slots
    between them) compacted to the dense layout of oracle/residual_ref.bcsr: off, col, cf,
    cap0 and mate re-indexed to dense slots.  Also checks the gap invariants."""
    seg = R["seg"].astype(np.int64)
    b, e = seg[:, 0], seg[:, 1]
    lens = e - b
    assert np.all(lens >= 0)
    assert np.all(b[1:] >= e[:-1]), "segments overlap or are out of vertex order"
    n = seg.shape[0]
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum(lens)
    M = int(off[-1])
    shift = b - off[:-1]                       # gapped slot = dense slot + shift[owner]
    idx = np.repeat(shift, lens) + np.arange(M, dtype=np.int64)
    col = R["col"][idx]
    gm = R["mate"][idx].astype(np.int64)
    mate = gm - shift[col]                     # the reverse arc lives in seg(col)
    return dict(M=M, off=off.astype(np.int32), col=col.copy(), cf=R["cf"][idx].copy(),
                cap0=R["cap0"][idx].copy(), mate=mate.astype(np.int32))


def bits_to_mask(words, n):
    b = np.unpackbits(np.asarray(words, np.uint32).view(np.uint8), bitorder="little")
    return b[:n].astype(np.uint8)


def assert_parity(g, layout="bcsr", ref=None, validate=True, **opt):
    """GPU result == oracle bit-exactly on F, cut capacity and canonical bitmap,
    and the GPU's residual state passes V1-V7 (preflow form)."""
    import paper_2404_00270_b200 as W
    F, words, st, ws = gpu_solve(g, layout, **opt)
    ref = ref or oracle.maxflow_graph(g, phase2=False)
    assert F == ref.flow, (g.name, layout, F, ref.flow)
    assert st["cut_capacity"] == ref.cut_capacity
    assert np.array_equal(words, ref.bitmap_words()), (g.name, layout, "bitmap differs")
    # padding bits beyond n are zero
    if g.n % 32:
        assert (int(words[-1]) >> (g.n % 32)) == 0
    if validate:
        R = W.residual(ws)
        if layout == "bcsr":
            D = dense_bcsr(R)
            f = check.demerge_bcsr(g.n, g.row_off, g.col, g.cap, D["off"], D["col"], D["cf"], D["cap0"], D["mate"])
        else:
            f = check.demerge_rcsr(g.n, g.row_off, g.col, g.cap, R["foff"], R["fcol"], R["fcf"], R["cap0"], R["bcf"])
        check.check_flow(g.n, g.row_off, g.col, g.cap, g.s, g.t, F, bits_to_mask(words, g.n), f,
                         strict=bool(opt.get("phase2", 0)))
    return F, st
