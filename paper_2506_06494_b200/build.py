"""Build the sm_100a shared library ``lib/libjgs2.so`` in-tree with nvcc.

The library is the C-ABI boundary (``include/jgs2.h``). It links cuBLAS and
cuSOLVER (used only by the one-time rest-Hessian factorization, never on the
per-sweep path) and the static CUDA runtime.
"""

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libjgs2.so"
SOURCES = ["jgs2.cu", "symbolic.cpp", "fill.cpp"]
HEADERS = sorted(p.name for p in CSRC.glob("*.cuh")) + ["symbolic.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc():
    cand = os.environ.get("NVCC") or shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found; cannot build the sm_100a library")
    return cand


def cuda_lib_dir():
    root = Path(nvcc()).resolve().parent.parent
    for d in (root / "lib64", root / "targets" / "x86_64-linux" / "lib"):
        if (d / "libcublas.so").exists() or (d / "libcublas.so.12").exists():
            return d
    return root / "lib64"


def nccl_dirs():
    """(include dir, lib dir) of the NCCL torch loads (pip nvidia-nccl), so the
    library binds the same libnccl.so.2 as torch.distributed; else the system one."""
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia")
        for root in (spec.submodule_search_locations or []):
            d = Path(root) / "nccl"
            if (d / "include" / "nccl.h").exists() and (d / "lib" / "libnccl.so.2").exists():
                return d / "include", d / "lib"
    except Exception:
        pass
    return Path("/usr/include"), Path("/usr/lib/x86_64-linux-gnu")


def stale():
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [PKG.parent / "include" / "jgs2.h"]
    return any(p.exists() and p.stat().st_mtime > t for p in deps)


def build(force=False, verbose=False):
    if not force and not stale():
        return LIB
    LIBDIR.mkdir(exist_ok=True)
    libdir = cuda_lib_dir()
    tmp = LIB.with_suffix(f".so.tmp{os.getpid()}")
    ninc, nlib = nccl_dirs()
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-Xptxas", "-O3", "-Xcompiler", "-fopenmp", "-I", str(PKG.parent / "include"), "-I", str(ninc),
           *[str(CSRC / s) for s in SOURCES], "-o", str(tmp),
           "-L", str(libdir), f"-Xlinker=-rpath,{libdir}", "-lcusolver", "-lcublas", "-lcusparse",
           "-L", str(nlib), f"-Xlinker=-rpath,{nlib}", "-l:libnccl.so.2", "-lgomp"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{res.stdout}\n{res.stderr}")
    if verbose:
        print(res.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
