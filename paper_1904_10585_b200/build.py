"""Build libpf.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with the repo).

Each .cu is compiled to its own object in parallel (build/obj, rebuilt when the source or any
header is newer), then linked into paper_1904_10585_b200/libpf.so."""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libpf.so")
OBJ = os.path.join(HERE, "..", "build", "obj")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_root() -> str:
    import nvidia.nccl  # the torch-bundled NCCL wheel (headers + libnccl.so.2)
    return os.path.dirname(nvidia.nccl.__file__) if getattr(nvidia.nccl, "__file__", None) else \
        list(nvidia.nccl.__path__)[0]


def _compile(nvcc, src, obj, nccl, verbose):
    cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-c",
           "-o", obj, src, f"-I{nccl}/include"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    return src, r


def build(verbose: bool = False, force: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(HERE, "..", "include", "pf.h")]
    hdr_t = max(os.path.getmtime(h) for h in hdrs)
    os.makedirs(OBJ, exist_ok=True)
    nccl = nccl_root()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    objs, todo = [], []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), hdr_t):
            todo.append((s, o))
    if not todo and os.path.exists(OUT) and all(os.path.getmtime(OUT) >= os.path.getmtime(o)
                                                for o in objs):
        return OUT
    with ThreadPoolExecutor(max_workers=min(len(todo), os.cpu_count() or 4) or 1) as ex:
        res = list(ex.map(lambda so: _compile(nvcc, so[0], so[1], nccl, verbose), todo))
    failed = False
    for src, r in res:
        if r.returncode != 0:
            failed = True
            sys.stderr.write(f"--- {src}\n{r.stdout}{r.stderr}")
        elif verbose:
            sys.stderr.write(r.stderr)
    if failed:
        raise RuntimeError("nvcc failed building libpf.so")
    cmd = [nvcc, *ARCH, "-shared", "-o", OUT, *objs, f"-L{nccl}/lib", "-l:libnccl.so.2",
           f"-Xlinker=-rpath={nccl}/lib"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libpf.so")
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
