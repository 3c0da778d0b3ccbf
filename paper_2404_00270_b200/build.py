"""Build libwbpr.so (the C-ABI library, include/wbpr.h) for sm_100a, in-tree.

    python -m paper_2404_00270_b200.build      # or __graft_entry__.build()

Each .cu under csrc/ is compiled with
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xptxas -v
and linked into paper_2404_00270_b200/libwbpr.so (static cudart).
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OUT = os.path.join(HERE, "libwbpr.so")
OBJ = os.path.join(HERE, "build_obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", CSRC, "-I", INCLUDE]


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    return sorted(hs) + [os.path.join(INCLUDE, "wbpr.h")]


def _digest() -> str:
    h = hashlib.sha256()
    for p in _sources() + _headers():
        with open(p, "rb") as f:
            h.update(p.encode() + f.read())
    h.update(" ".join(ARCH + FLAGS + ["-Xptxas", "-v", "ptxas-report"]).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False, defines=(), variant: str = "") -> str:
    """variant/defines: an experiment build (extra -D flags) into libwbpr_<variant>.so,
    loaded when WBPR_LIB points at it; the default build is libwbpr.so."""
    obj_dir = OBJ if not variant else os.path.join(OBJ, variant)
    out = OUT if not variant else os.path.join(HERE, f"libwbpr_{variant}.so")
    os.makedirs(obj_dir, exist_ok=True)
    stamp = os.path.join(obj_dir, "digest")
    dg = _digest() + " ".join(defines)
    if not force and os.path.exists(out) and os.path.exists(stamp) and open(stamp).read() == dg:
        return out

    hdr = hashlib.sha256()
    for p in _headers():
        with open(p, "rb") as f:
            hdr.update(p.encode() + f.read())
    hdr.update(" ".join(ARCH + FLAGS + list(defines)).encode())

    def comp(src):
        obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
        # per-object digest (source + every header + flags): only changed sources recompile
        h = hdr.copy()
        with open(src, "rb") as f:
            h.update(f.read())
        odg = h.hexdigest()
        ostamp = obj + ".digest"
        if (not force and os.path.exists(obj) and os.path.exists(ostamp) and os.path.exists(obj + ".ptxas.txt")
                and open(ostamp).read() == odg):
            return obj, open(obj + ".ptxas.txt").read()
        cmd = [NVCC] + ARCH + FLAGS + list(defines) + ["-Xptxas", "-v", "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        with open(obj + ".ptxas.txt", "w") as f:   # register / spill report, see ptxas_report()
            f.write(r.stderr)
        with open(ostamp, "w") as f:
            f.write(odg)
        return obj, r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(comp, _sources()))
    if verbose:
        for _, err in results:
            sys.stderr.write(err)
    tmp = out + f".tmp{os.getpid()}"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + [o for o, _ in results]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, out)
    with open(stamp, "w") as f:
        f.write(dg)
    return out


def ptxas_report(source: str = "solve.cu", variant: str = "") -> dict:
    """{mangled kernel name: (registers, spill store bytes, spill load bytes)} from the ptxas
    report the last build of `source` left next to its object file."""
    obj_dir = OBJ if not variant else os.path.join(OBJ, variant)
    txt = open(os.path.join(obj_dir, source + ".o.ptxas.txt")).read()
    out, name, spill = {}, None, (0, 0)
    for line in txt.splitlines():
        m = re.search(r"Compiling entry function '(\w+)'", line)
        if m:
            name, spill = m.group(1), (0, 0)
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and name:
            spill = (int(m.group(1)), int(m.group(2)))
            continue
        m = re.search(r"Used (\d+) registers", line)
        if m and name:
            out[name] = (int(m.group(1)),) + spill
            name = None
    return out


if __name__ == "__main__":
    defs = [a for a in sys.argv[1:] if a.startswith("-D")]
    var = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--variant=")), "")
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs, variant=var))
