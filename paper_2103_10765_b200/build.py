"""Build libgbm3d.so in-tree: every .cu under csrc/ compiled for sm_100a (nvcc), linked with a
static CUDA runtime so the library has no runtime dependency beyond the driver."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libgbm3d.so")
BUILD = os.path.join(PKG, "build")
# Dev experiments only: GBM3D_NVCC_EXTRA adds nvcc flags and GBM3D_LIB_OUT redirects the output
# (e.g. variants/libgbm3d_x.so, loaded via GBM3D_LIB); the default build ignores both.
EXTRA = os.environ.get("GBM3D_NVCC_EXTRA", "").split()
if os.environ.get("GBM3D_LIB_OUT"):
    LIB = os.path.abspath(os.environ["GBM3D_LIB_OUT"])
    BUILD = "/tmp/gbm3d_objs_" + os.path.basename(LIB)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills",
         "-I", os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return (_sources() + glob.glob(os.path.join(CSRC, "*.cuh"))
            + [os.path.join(ROOT, "include", "gbm3d.h"), os.path.abspath(__file__)])


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in _deps())


def source_id() -> str:
    """Hash of everything the library is built from (sources, header, flags): the build id
    that gbm3d_version() reports and that profiles/ captures are tagged with."""
    import hashlib
    h = hashlib.sha256()
    for p in sorted(_deps()):
        if p.endswith(".py"):
            continue
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(ARCH + FLAGS + EXTRA).encode())
    return h.hexdigest()[:16]


def _compile(src: str, sid: str) -> str:
    obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, *EXTRA, f"-DGBM3D_SRC_ID=\"{sid}\"", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if "spill" in (r.stderr or "") and "0 bytes spill" not in r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    sid = source_id()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda src: _compile(src, sid), srcs))
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
