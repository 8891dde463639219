"""Compile the sm_100a C-ABI library in-tree (no torch extension machinery).

    python -m paper_1908_11807_b200._build        # or __graft_entry__.build()

Produces ``paper_1908_11807_b200/_lib/liblbvh_b200.so`` from
``csrc/*.cu`` with nvcc for ``-gencode arch=compute_100a,code=sm_100a``.
The .so is git-ignored but travels to the GPU box with the snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT_DIR, "liblbvh_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-Xptxas", "-warn-spills", f"-I{os.path.join(ROOT, 'include')}"]
# extra flags for A/B builds of compiler options (e.g. LBVH_NVCC_EXTRA="-Xptxas -O3")
NVCC_FLAGS += os.environ.get("LBVH_NVCC_EXTRA", "").split()


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build liblbvh_b200.so")


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(ROOT, "include", "lbvh_b200.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    cc = nvcc()
    objs = []

    def compile_one(src):
        obj = os.path.join(OUT_DIR, os.path.basename(src).replace(".cu", ".o"))
        cmd = [cc, *ARCH, *NVCC_FLAGS, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{res.stdout}\n{res.stderr}")
        if verbose and res.stderr.strip():
            print(res.stderr, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as pool:
        objs = list(pool.map(compile_one, _sources()))
    tmp = LIB + ".tmp"
    cmd = [cc, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    return LIB


def build_variant(name: str, defines: list, csrc: str = None) -> str:
    """A/B build with extra -D defines (and optionally another source tree,
    e.g. a git checkout of csrc/) into _lib/variants/<name>.so (load it with
    LBVH_LIB=<path>); used only for kernel experiments."""
    vdir = os.path.join(OUT_DIR, "variants", name)
    os.makedirs(vdir, exist_ok=True)
    cc = nvcc()
    objs = []
    for src in (sorted(glob.glob(os.path.join(csrc, "*.cu"))) if csrc else _sources()):
        obj = os.path.join(vdir, os.path.basename(src).replace(".cu", ".o"))
        subprocess.run([cc, *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o",
                        obj], check=True)
        objs.append(obj)
    lib = os.path.join(OUT_DIR, "variants", f"{name}.so")
    subprocess.run([cc, *ARCH, "-shared", "-o", lib, *objs, "-lcudart_static", "-lrt", "-ldl",
                    "-lpthread"], check=True)
    return lib


if __name__ == "__main__":
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        csrc = None
        if "--csrc" in sys.argv:
            j = sys.argv.index("--csrc")
            csrc = sys.argv[j + 1]
            del sys.argv[j:j + 2]
        print(build_variant(sys.argv[i + 1], sys.argv[i + 2:], csrc))
    else:
        print(build(force="--force" in sys.argv, verbose=True))
