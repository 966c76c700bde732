"""Build libvoltb200.so in-tree with nvcc for sm_100a (no JIT, no torch
extension cache): the .so travels to the GPU box with the repo snapshot."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libvoltb200.so"
LIB_EXP = PKG / "libvoltb200_exp.so"  # experiment build (A/B switches live); loaded only via VB_LIBRARY
SOURCES = ["capi.cu", "stage.cu", "group.cu", "motion.cu", "summary.cu", "probe.cu", "traces.cu", "unet.cu"]
EXP_SOURCES = ["zncc_mma.cu"]  # measured no-go prototypes, experiment build only
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-O3",
         f"-I{ROOT / 'include'}"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + EXP_SOURCES] + [CSRC / "vb.cuh", CSRC / "tma.cuh", ROOT / "include" / "voltb200.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, experiments: bool = False) -> Path:
    """experiments=True compiles the A/B switches (vb::knob) to read the
    environment (-DVB_EXPERIMENTS); the product build uses the defaults."""
    lib = LIB_EXP if experiments else LIB
    extra = []
    if experiments:  # A/B builds: extra compile-time variants, e.g. -DVB_PAIR_UNROLL=2 (build-time only)
        extra = os.environ.get("VB_EXTRA_NVCC_FLAGS", "").split()
        if os.environ.get("VB_EXP_NAME"):
            lib = PKG / f"libvoltb200_{os.environ['VB_EXP_NAME']}.so"
    if not force and not _stale(lib):
        return lib
    obj_dir = PKG / (("build_" + os.environ.get("VB_EXP_NAME", "exp")) if experiments else "build")
    obj_dir.mkdir(exist_ok=True)
    cc = nvcc()
    procs, objs = [], []
    for src in SOURCES + (EXP_SOURCES if experiments else []):
        obj = obj_dir / (Path(src).stem + ".o")
        objs.append(obj)
        cmd = [cc, *ARCH, *FLAGS, "-c", str(CSRC / src), "-o", str(obj)]
        if experiments:
            cmd += ["-DVB_EXPERIMENTS", *extra]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        procs.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    failed = []
    for src, p in zip(SOURCES + (EXP_SOURCES if experiments else []), procs):
        out, _ = p.communicate()
        if verbose or p.returncode:
            sys.stderr.write(out)
        if p.returncode:
            failed.append(src)
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    tmp = lib.with_suffix(".so.tmp")
    subprocess.run([cc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart", "-ldl"], check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, experiments="--experiments" in sys.argv))
