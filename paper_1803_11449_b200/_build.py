"""Builds libdhsa_b200.so (sm_100a) in-tree with nvcc.  No JIT cache: the .so sits
next to this file so it travels to the GPU box with the repo snapshot."""

from __future__ import annotations

import os
import shutil
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(_HERE, "csrc")
LIB_PATH = os.path.join(_HERE, "libdhsa_b200.so")
SOURCES = ["dhsa_cabi.cu"]
HEADERS = ["dhsa_device.cuh", os.path.join("..", "..", "include", "dhsa_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
    "-cudart", "static",
    "-diag-suppress", "128",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: libdhsa_b200.so cannot be built (no CPU fallback exists)")


def stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    built = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    return any(os.path.exists(d) and os.path.getmtime(d) > built for d in deps)


def build_variant(out: str, defs) -> str:
    """A tuning variant of the library (extra -D definitions) for A/B runs: tools/ builds them
    under build/variants/ and selects one with DHSA_LIB=<path>."""
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = [_nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defs], "-o", out, *[os.path.join(CSRC, f) for f in SOURCES]]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + proc.stdout + proc.stderr)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile the library.  Safe to call from every rank of a multi-process launch at once: one
    process compiles (file lock), into a temporary file that is renamed into place, so nobody can
    dlopen a half-written library; the others wait and find it fresh."""
    import fcntl

    if not force and not stale():
        return LIB_PATH
    with open(LIB_PATH + ".lock", "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        try:
            if not force and not stale():   # another process built it while this one waited
                return LIB_PATH
            tmp = f"{LIB_PATH}.{os.getpid()}.tmp"
            cmd = [_nvcc(), *NVCC_FLAGS, "-o", tmp, *[os.path.join(CSRC, f) for f in SOURCES]]
            if verbose:
                cmd.insert(1, "-Xptxas")
                cmd.insert(2, "-v")
            proc = subprocess.run(cmd, capture_output=True, text=True)
            if proc.returncode != 0:
                if os.path.exists(tmp):
                    os.remove(tmp)
                raise RuntimeError("nvcc failed:\n" + proc.stdout + proc.stderr)
            os.replace(tmp, LIB_PATH)
            if verbose:
                print(proc.stderr)
        finally:
            fcntl.flock(lock, fcntl.LOCK_UN)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force=True, verbose=True))
