"""Build the native libraries in-tree for sm_100a (B200).

    python -m paper_2502_12574_b200.build      # or __graft_entry__.build()

Outputs
  paper_2502_12574_b200/libheadinfer.so   -- the C ABI (include/headinfer.h) + kernels
  synth/libsynth.so                       -- seeded input generator twin (test/bench infra)
cudart is linked statically (nvcc default), so the libraries load on a GPU-less host too; no other CUDA
library is linked (the NEXT-4 layer's GEMMs are this library's own tcgen05 kernels, k_gemm.cu).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2502_12574_b200")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "--expt-relaxed-constexpr"]


def _stale(out: str, srcs) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


CUDA_LIB = "/usr/local/cuda/lib64"


def _nvcc_shared(out: str, srcs, extra=(), force=False, verbose=False, libs=()):
    deps = list(srcs) + glob.glob(os.path.join(os.path.dirname(srcs[0]), "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    if not force and not _stale(out, deps):
        return out
    objs = []
    # one object directory per library: variant builds may run concurrently
    bdir = os.path.join(os.path.dirname(out), "build", os.path.splitext(os.path.basename(out))[0])
    os.makedirs(bdir, exist_ok=True)
    procs = []
    for s in srcs:
        o = os.path.join(bdir, os.path.basename(s) + ".o")
        cmd = [NVCC, *ARCH, *COMMON, *extra, "-c", s, "-o", o]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT), s))
        objs.append(o)
    failed = False
    for p, s in procs:
        outp = p.communicate()[0].decode()
        if p.returncode != 0:
            sys.stderr.write(f"nvcc failed for {s}:\n{outp}\n")
            failed = True
        elif verbose and outp:
            sys.stderr.write(outp)
    if failed:
        raise RuntimeError("nvcc compilation failed")
    tmp = out + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lpthread", *libs])
    os.replace(tmp, out)
    return out


HI_LIBS: list = []


def build_variant(name: str, defines) -> str:
    """Experiments: the product sources plus the comparison prefill kernels of csrc/variants/ (mma.sync
    baseline, CTA pair, one tile; selected by HI_FLAG_MMA_SYNC_PREFILL / _PREFILL_2CTA / _PREFILL_TC1),
    with extra -D flags -> build/variants/libheadinfer_<name>.so (loaded when HI_LIB_VARIANT=<name>).
    The product library (build()) does not contain the comparison kernels and rejects their flags."""
    srcs = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")) + glob.glob(os.path.join(PKG, "csrc", "variants", "*.cu")))
    out = os.path.join(PKG, "build", "variants", f"libheadinfer_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    return _nvcc_shared(out, srcs, extra=["-DHI_WITH_VARIANTS"] + [f"-D{d}" for d in defines], force=True,
                        libs=HI_LIBS)


def build(force: bool = False, verbose: bool = False) -> None:
    srcs = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))
    _nvcc_shared(os.path.join(PKG, "libheadinfer.so"), srcs, force=force, verbose=verbose, libs=HI_LIBS)
    ssrc = sorted(glob.glob(os.path.join(ROOT, "synth", "csrc", "*.cu")))
    _nvcc_shared(os.path.join(ROOT, "synth", "libsynth.so"), ssrc, force=force, verbose=verbose)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
