"""Build libbagel.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

The library is plain C ABI (include/bagel.h); the Python side loads it with
ctypes.  Static cudart is linked so the library does not depend on which
libcudart torch happens to bundle.

Staleness is decided by CONTENT, not mtimes: the SHA-256 of every source, header
and compiler flag is compiled into the library (``bagel_build_hash()``) and
written next to it; a library whose hash differs from the tree's is rebuilt
(``ensure_built``), and the binding refuses to load one it cannot rebuild.
Translation units compile in parallel (one nvcc per .cu), then link.
"""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libbagel.so")
HASH_FILE = LIB + ".sha256"
OBJ_DIR = os.path.join(PKG, "build")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-I" + os.path.join(ROOT, "include")]
LDFLAGS = ["-shared", "-cudart", "static"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(ROOT, "include", "bagel.h")]


def source_hash() -> str:
    h = hashlib.sha256()
    # flags without the (machine-specific) absolute include path: a library built here must hash
    # the same on the GPU box, where the tree lives elsewhere
    h.update(" ".join(ARCH + [f for f in CFLAGS if not f.startswith("-I")] + LDFLAGS).encode())
    for f in deps():
        h.update(os.path.relpath(f, ROOT).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def built_hash() -> str | None:
    try:
        with open(HASH_FILE) as f:
            return f.read().strip()
    except OSError:
        return None


def up_to_date() -> bool:
    return os.path.exists(LIB) and built_hash() == source_hash()


def build_library(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    digest = source_hash()
    if not force and os.path.exists(LIB) and built_hash() == digest:
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    os.makedirs(OBJ_DIR, exist_ok=True)
    flags = ARCH + CFLAGS + [f"-DBAGEL_SRC_HASH=\"{digest}\""]

    def compile_one(src):
        obj = os.path.join(OBJ_DIR, os.path.basename(src) + f".{os.getpid()}.o")
        cmd = [nvcc] + flags + ["-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        return obj

    n = jobs or min(len(sources()), max(1, os.cpu_count() or 1))
    with ThreadPoolExecutor(max_workers=n) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc] + ARCH + LDFLAGS + objs + ["-o", tmp]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    for o in objs:
        os.remove(o)
    os.replace(tmp, LIB)
    with open(HASH_FILE + f".tmp{os.getpid()}", "w") as f:
        f.write(digest + "\n")
    os.replace(HASH_FILE + f".tmp{os.getpid()}", HASH_FILE)
    return LIB


def ensure_built() -> str:
    """The library for the current sources: rebuilt when its content hash is stale."""
    if up_to_date():
        return LIB
    return build_library(verbose=True)


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose=True))
