"""Builds libosmpm.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""
import hashlib
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libosmpm.so")
SOURCES = ["capi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

def _nccl_dir():
    """The NCCL that torch loads (nvidia-nccl wheel); libosmpm links the same libnccl.so.2 so one copy
    serves torch.distributed and the library's communicator."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        d = list(spec.submodule_search_locations)[0]
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("nccl.h / libnccl.so.2 of the nvidia-nccl wheel not found")


NCCL = _nccl_dir()
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17", "--expt-relaxed-constexpr",
         "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(NCCL, "include"),
         "-L", os.path.join(NCCL, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(NCCL, "lib")]


def source_hash():
    """sha256 (first 16 hex digits) of every source the library is built from (csrc/, include/) and of
    the compiler flags; embedded in the library (osmpm_version) and recorded beside it."""
    h = hashlib.sha256()
    for d in (CSRC, os.path.join(ROOT, "include")):
        for f in sorted(os.listdir(d)):
            h.update(f.encode())
            with open(os.path.join(d, f), "rb") as fh:
                h.update(fh.read())
    h.update(" ".join(FLAGS).encode())
    return h.hexdigest()[:16]


def built_hash():
    try:
        with open(OUT + ".srchash") as fh:
            return fh.read().strip()
    except OSError:
        return None


def build(force=False, verbose=False):
    """Rebuild unless the library on disk was built from exactly the current sources (hash check, not
    timestamps: a snapshot copied to another machine keeps neither order nor mtimes)."""
    hs = source_hash()
    if not force and os.path.exists(OUT) and built_hash() == hs:
        return OUT
    cmd = [NVCC, *FLAGS, f"-DOSMPM_SRC_HASH=\"{hs}\"", *[os.path.join(CSRC, s) for s in SOURCES], "-o", OUT + ".tmp"]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(OUT + ".tmp", OUT)
    with open(OUT + ".srchash", "w") as fh:
        fh.write(hs + "\n")
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose=True))
