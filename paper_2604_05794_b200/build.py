"""Build libphg_b200.so in-tree for sm_100a (``python -m paper_2604_05794_b200.build``).

-fmad=false keeps every a*b+c as a separately rounded multiply and add, which
is what makes the kernel bit-identical to the numpy reference.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRCS = [os.path.join(HERE, "csrc", f)
        for f in ("phg_trace.cu", "phg_grow.cu", "phg_link.cu", "phg_io.cu", "phg_copy.cu")]
HDRS = [os.path.join(HERE, "csrc", "phg_core.cuh")]
OUT = os.path.join(HERE, "libphg_b200.so")
OUT_CHECKED = os.path.join(HERE, "libphg_b200_checked.so")

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-fmad=false", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
]


def nvcc():
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found")
    return cand


def _compile(args):
    src, obj, flags = args
    cmd = [nvcc(), *flags, "-I", os.path.join(ROOT, "include"), "-c", "-o", obj, src]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return src, r


def build(force=False, verbose=False, checked=False, extra=(), out=None):
    """checked=True: libphg_b200_checked.so with -DPHG_CHECKED (device index checks and
    allocation canaries; loaded with PHG_CHECKED_LIB=1).  The translation units compile in
    parallel (one nvcc per file), then link into the shared library.  `extra` nvcc flags and
    another `out` path build experiment libraries for A/B runs (loaded with PHG_LIB_PATH)."""
    out = out or (OUT_CHECKED if checked else OUT)
    deps = SRCS + HDRS + [os.path.join(ROOT, "include", "phg_b200.h")]
    if (not force and os.path.exists(out)
            and os.path.getmtime(out) >= max(os.path.getmtime(d) for d in deps)):
        return out
    flags = NVCC_FLAGS + (["-DPHG_CHECKED"] if checked else []) + list(extra)
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    objdir = tempfile.mkdtemp(prefix="phg_build_")
    try:
        jobs = [(src, os.path.join(objdir, os.path.basename(src) + ".o"), flags) for src in SRCS]
        with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
            results = list(ex.map(_compile, jobs))
        for src, r in results:
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {os.path.basename(src)} ({r.returncode})")
            if verbose:
                sys.stderr.write(r.stderr)
        tmp_out = out + ".tmp"
        link = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler",
                "-fPIC", "-o", tmp_out, *[j[1] for j in jobs]]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc link failed ({r.returncode})")
        os.replace(tmp_out, out)  # atomic: a loaded library is never half-written
    finally:
        shutil.rmtree(objdir, ignore_errors=True)
    return out


def build_all(force=False):
    """The release and the checked library, concurrently."""
    with ThreadPoolExecutor(max_workers=2) as ex:
        return list(ex.map(lambda c: build(force=force, checked=c), (False, True)))


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv))
