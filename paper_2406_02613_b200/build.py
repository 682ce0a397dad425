"""In-tree build of the CUDA library ``_acco_b200.so`` (sm_100a only).

Compiles every ``csrc/*.cu`` (device kernels and host C++ alike) and
``csrc/*.cpp`` (host-only C++) with nvcc
(``-gencode arch=compute_100a,code=sm_100a -lineinfo``) and links one shared
library next to this file, so it travels to the GPU box with the repo snapshot.
NCCL comes from the system (``/usr/include/nccl.h``, soname ``libnccl.so.2``);
inside a torch process the already-loaded torch NCCL satisfies the soname.

Incremental: an object is rebuilt only when its source or any header is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "..", "build", "obj")
LIB = os.path.join(HERE, "_acco_b200.so")
REPO = os.path.dirname(HERE)

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# nlohmann/json (the JSON library the reference parses and dumps with), for
# the config-level entry csrc/run_api.cpp; a header-only library in the image
JSON_INC = os.environ.get(
    "ACCO_JSON_INC", "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = [
    "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fopenmp",
    "--expt-relaxed-constexpr", f"-I{CSRC}", f"-I{os.path.join(REPO, 'include')}",
    "-Xptxas", "-warn-spills",
]


def _newest_header() -> float:
    hs = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
    hs += glob.glob(os.path.join(REPO, "include", "*.h"))
    return max((os.path.getmtime(h) for h in hs), default=0.0)


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    if os.path.exists(obj):
        t = os.path.getmtime(obj)
        if t >= os.path.getmtime(src) and t >= _newest_header():
            return obj
    cmd = [NVCC, *ARCH, *COMMON, "-c", src, "-o", obj]
    if src.endswith(".cpp"):  # host-only translation unit
        cmd[1:1] = ["-x", "c++", f"-I{JSON_INC}", "-Xcompiler", "-std=c++17"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip() and verbose:
        print(r.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    newest = max(os.path.getmtime(o) for o in objs)
    if os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-Xcompiler", "-fopenmp",
           "-L/usr/lib/x86_64-linux-gnu", "-lnccl", "-lgomp"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
