"""Build libsg.so (the C-ABI + sm_100a kernels) in-tree with nvcc.

The library is built next to this file so it travels with the repository
snapshot to the GPU box; nothing is installed into site-packages.
"""

import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libsg.so")

SOURCES = ["sg_runtime.cu", "sg_list.cu", "sg_cc.cu", "sg_gen.cu", "sg_host.cpp", "sg_xfer.cu", "sg_multi.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc():
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found: libsg needs the CUDA toolkit to build")
    return cand


FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3"]
# experiments only: extra -D flags for A/B builds (part of the source hash)
FLAGS += [f for f in os.environ.get("SG_NVCC_DEFS", "").split() if f.startswith("-D")]
LINK = ["-lcudart_static", "-lrt", "-ldl", "-lpthread"]
MARKER = b"SG_SOURCE_HASH="


def _deps(src):
    heads = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))
    return [os.path.join(CSRC, src), os.path.join(INCLUDE, "sg.h")] + heads


def _digest(paths, extra):
    h = hashlib.sha256()
    for p in paths:
        h.update(os.path.basename(p).encode() + b"\0")
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(extra).encode())
    return h.hexdigest()


def source_hash():
    """sha256 over every source, header and flag libsg.so is built from."""
    paths = [os.path.join(CSRC, s) for s in SOURCES]
    paths += sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))
    paths.append(os.path.join(INCLUDE, "sg.h"))
    return _digest(paths, ARCH + FLAGS + LINK)


def embedded_hash(path=LIB):
    """The source hash compiled into a built library, or None."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        return None
    i = data.find(MARKER)
    if i < 0:
        return None
    j = data.find(b";", i)
    return data[i + len(MARKER):j].decode(errors="replace")


def build_native(force=False, verbose=False):
    """Compile every csrc source for sm_100a and link libsg.so; returns its
    path.  A library (or object) is reused only when the source hash
    embedded in it (object: its sidecar) equals the tree's -- a shipped
    binary built from other sources is rebuilt, whatever its mtime."""
    os.makedirs(BUILD, exist_ok=True)
    want = source_hash()
    if not force and embedded_hash() == want:
        return LIB
    nvcc = _nvcc()
    objs = []
    jobs = []
    for src in SOURCES:
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        defs = [f"-DSG_SOURCE_HASH=\"{want}\""] if src == "sg_runtime.cu" else []
        cmd = [nvcc, *ARCH, *FLAGS, *defs, "-I", INCLUDE, "-I", CSRC, "-c", os.path.join(CSRC, src), "-o", obj]
        sidecar = obj + ".sha256"
        key = _digest(_deps(src), cmd[1:-3])
        try:
            with open(sidecar) as f:
                fresh = f.read().strip() == key and os.path.exists(obj)
        except OSError:
            fresh = False
        if force or not fresh:
            jobs.append((cmd, sidecar, key))

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        if verbose and (r.stdout or r.stderr):
            sys.stderr.write(r.stdout + r.stderr)

    def compile_one(job):
        cmd, sidecar, key = job
        run(cmd)
        with open(sidecar, "w") as f:
            f.write(key)

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(compile_one, jobs))
    tmp = LIB + ".tmp"
    run([nvcc, *ARCH, "-shared", "-o", tmp, *objs, *LINK])
    os.replace(tmp, LIB)
    if embedded_hash() != want:
        raise RuntimeError("libsg.so does not carry the expected source hash after the build")
    return LIB


if __name__ == "__main__":
    print(build_native(force="--force" in sys.argv, verbose=True))
