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
            f = check.demerge_bcsr(g.n, g.row_off, g.col, g.cap, R["off"], R["col"], R["cf"], R["cap0"], R["mate"])
        else:
            f = check.demerge_rcsr(g.n, g.row_off, g.col, g.cap, R["foff"], R["fcol"], R["fcf"], R["cap0"], R["bcf"])
        check.check_flow(g.n, g.row_off, g.col, g.cap, g.s, g.t, F, bits_to_mask(words, g.n), f,
                         strict=bool(opt.get("phase2", 0)))
    return F, st
