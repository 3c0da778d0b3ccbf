#!/usr/bin/env python
"""Write synth/c5_sizes.json: (n, m, sha256 of the CSR bytes) of every C5 instance
(64 x R-MAT scale 18, paper-rule terminals, seeds 1000-1063).

Input metadata only (calls synth, never the oracle or the CUDA path): bench.py balances
the instance partition over ranks by m without generating every instance
on every rank, and checks each instance it generates against its hash."""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402


def digest(g):
    h = hashlib.sha256()
    for a in (g.row_off, g.col, g.cap):
        h.update(a.tobytes())
    h.update(f"{g.s},{g.t}".encode())
    return h.hexdigest()[:32]


def main():
    out = {}
    for i in range(64):
        g = synth.rmat(18, 16, 1000 + i, "paper")
        out[str(1000 + i)] = {"n": g.n, "m": g.m, "sha": digest(g)}
        print(i, g.n, g.m, flush=True)
    with open(os.path.join(ROOT, "synth", "c5_sizes.json"), "w") as f:
        json.dump({"recipe": "C5: R-MAT scale 18, edgefactor 16, paper-rule terminals (256 starts), seed 1000+i",
                   "instances": out}, f, indent=1)


if __name__ == "__main__":
    main()
