"""Builds libios.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libios.so")
SOURCES = ["stage_kernel.cu", "device.cpp", "graph.cpp", "dp.cpp", "abi.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC,-fvisibility=hidden", "-cudart", "static", "--expt-relaxed-constexpr"]


ID_FILE = LIB + ".buildid"


def source_hash() -> str:
    """Content hash of everything libios.so is compiled from (sources, header, flags, this file).
    It is compiled into the library (ios_build_id()) and stored beside it, so a stale or foreign
    binary is rebuilt whatever the file times say, and tests can check the loaded .so is HEAD's."""
    import hashlib
    h = hashlib.sha256()
    deps = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp", ".h")))
    for p in deps + [os.path.join(HERE, "..", "include", "ios.h"), os.path.abspath(__file__)]:
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(FLAGS).encode())
    return h.hexdigest()[:16]


def _stale(sid: str) -> bool:
    if not os.path.exists(LIB) or not os.path.exists(ID_FILE):
        return True
    with open(ID_FILE) as f:
        return f.read().strip() != sid


def build(force: bool = False, verbose: bool = False) -> str:
    sid = source_hash()
    if not force and not _stale(sid):
        return LIB
    objs = []
    os.makedirs(os.path.join(HERE, "build"), exist_ok=True)
    procs = []
    # the stage kernel's six (dtype, smem-descriptor) instantiations are separate units so they
    # compile in parallel (stage_kernel.cu, IOS_INST_DT / IOS_INST_SD)
    units = [(src, []) for src in SOURCES]
    units += [("stage_kernel.cu", [f"-DIOS_INST_DT={dt}", f"-DIOS_INST_SD={sdv}"]) for dt in range(3) for sdv in range(2)]
    for src, defs in units:
        tag = "".join(d.split("=")[1] for d in defs)
        obj = os.path.join(HERE, "build", src + (f".inst{tag}" if tag else "") + ".o")
        cmd = [NVCC, *FLAGS, *defs, f'-DIOS_BUILD_ID="{sid}"', "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu") and verbose:
            cmd += ["-Xptxas", "-v"]
        procs.append((src, cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    failed = False
    for src, cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out)
        if p.returncode != 0:
            sys.stderr.write(f"\n[build] FAILED: {' '.join(cmd)}\n")
            failed = True
    if failed:
        raise RuntimeError("libios build failed")
    tmp = LIB + ".tmp"
    cmd = [NVCC, *FLAGS, "-shared", "-o", tmp, *objs]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    with open(ID_FILE, "w") as f:
        f.write(sid + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
