"""Build libbe.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_1912_01703_b200.build [--debug]

Every .cu/.cpp under csrc/ is compiled with
`-gencode arch=compute_100a,code=sm_100a -lineinfo -O3` and linked into
paper_1912_01703_b200/libbe.so (no torch, no link-time NCCL: NCCL is dlopen'ed).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libbe.so")
BUILD = os.path.join(ROOT, "build", "be")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include():
    try:
        import nvidia.nccl  # type: ignore
        p = os.path.join(list(nvidia.nccl.__path__)[0], "include")
        if os.path.exists(os.path.join(p, "nccl.h")):
            return p
    except Exception:
        pass
    return "/usr/include"


def _flags(debug=False):
    f = ["-std=c++17", "-O3" if not debug else "-O0", "-lineinfo", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=hidden" if False else "-fvisibility=default",
         "-I", os.path.join(ROOT, "include"), "-I", _nccl_include(),
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"] + ARCH
    if debug:
        f += ["-G"] if os.environ.get("BE_DEVICE_DEBUG") else []
    return f


def build(debug=False, verbose=False):
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    headers = sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                     [os.path.join(ROOT, "include", "be.h")])
    hh = hashlib.sha1()
    for h in headers:
        hh.update(open(h, "rb").read())
    flags = _flags(debug)
    hh.update(" ".join(flags).encode())
    hdr_sig = hh.hexdigest()[:12]

    def compile_one(src):
        sig = hashlib.sha1(open(src, "rb").read() + hdr_sig.encode()).hexdigest()[:16]
        obj = os.path.join(BUILD, os.path.basename(src) + "." + sig + ".o")
        if not os.path.exists(obj):
            cmd = [NVCC] + flags + ["-c", src, "-o", obj]
            if src.endswith(".cpp"):
                cmd = [NVCC] + flags + ["-x", "cu", "-c", src, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
            if verbose and (r.stderr.strip()):
                print(r.stderr, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = OUT + ".tmp"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart", "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(debug="--debug" in sys.argv, verbose="-v" in sys.argv))
