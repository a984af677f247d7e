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


def build(force: bool = False, verbose: bool = False, extra_defs=(), out: str = "") -> str:
    """Compile libios.so (or, with extra -D flags, an experiment variant into `out`)."""
    sid = source_hash()
    variant = bool(extra_defs or out)
    if not variant and not force and not _stale(sid):
        return LIB
    lib = out or LIB
    objs = []
    bdir = os.path.join(HERE, "build", os.path.splitext(os.path.basename(lib))[0] if variant else "")
    os.makedirs(bdir, exist_ok=True)
    procs = []
    # the stage kernel's six (dtype, smem-descriptor) instantiations are separate units so they
    # compile in parallel (stage_kernel.cu, IOS_INST_DT / IOS_INST_SD)
    units = [(src, []) for src in SOURCES]
    # (dtype, smem-descriptor, feature class): TF32 / BF16 x {lean, gather, full, trace}; FP32-SIMT x
    # {full, trace} (stage_kernel.cu launch_stage, stage_desc.h KernelFeature)
    # + the cluster split-K classes (F_CSK = 8: lean / gather / full) and the trace class (all features)
    insts = [(dt, sdv, ft) for dt in (0, 1) for sdv in (0, 1) for ft in (0, 1, 3, 8, 9, 11, 15)]
    insts += [(2, sdv, ft) for sdv in (0, 1) for ft in (3, 15)]
    units += [("stage_kernel.cu", [f"-DIOS_INST_DT={dt}", f"-DIOS_INST_SD={sdv}", f"-DIOS_INST_FEAT={ft}"])
              for dt, sdv, ft in insts]
    for src, defs in units:
        tag = "_".join(d.split("=")[1] for d in defs)
        obj = os.path.join(bdir, src + (f".inst{tag}" if tag else "") + ".o")
        cmd = [NVCC, *FLAGS, *defs, *extra_defs, f'-DIOS_BUILD_ID="{sid}"', "-c", os.path.join(CSRC, src), "-o", obj]
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
    tmp = lib + ".tmp"
    cmd = [NVCC, *FLAGS, "-shared", "-o", tmp, *objs]
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib)
    if not variant:
        with open(ID_FILE, "w") as f:
            f.write(sid + "\n")
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
