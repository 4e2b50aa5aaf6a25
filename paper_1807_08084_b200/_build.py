"""In-tree build of the native libraries (nvcc for sm_100a, gcc for the host
generator twin).  Called by ``__graft_entry__.build()``; also used lazily by
the bindings so a fresh checkout works after one import on a machine with the
CUDA toolkit.  The built ``.so`` files live next to their sources (git-ignored,
shipped to the GPU box by gpurun)."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
INCLUDE = os.path.join(ROOT, "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
                      "-Xptxas", "-v", "-I", INCLUDE]

TARGETS = {
    # product library: the hot path (K1, K2, K3, R1, host pipeline)
    "libpolsar": dict(
        out=os.path.join(PKG, "libpolsar.so"),
        srcs=[os.path.join(PKG, "csrc", f) for f in ("abi.cu", "inv_det.cu", "window.cu", "nlm.cu", "checksum.cu")],
        deps=[os.path.join(INCLUDE, "polsar.h"), os.path.join(PKG, "csrc", "common.cuh"),
              os.path.join(PKG, "csrc", "alg.cuh"), os.path.join(PKG, "csrc", "window_core.cuh"),
              os.path.join(PKG, "csrc", "window_mma.cuh")],
        cmd=lambda out, srcs: [NVCC] + NVCC_COMMON + srcs + ["-o", out],
    ),
    # seeded input generator, GPU build (support; FMA contraction off so it
    # matches the host twin bit for bit)
    "libpolsar_gen": dict(
        out=os.path.join(PKG, "wishart", "libpolsar_gen.so"),
        srcs=[os.path.join(PKG, "wishart", "wishart_gen.cu")],
        deps=[os.path.join(PKG, "wishart", "wishart_core.h"), os.path.join(INCLUDE, "polsar_gen.h")],
        cmd=lambda out, srcs: [NVCC] + NVCC_COMMON + ["-fmad=false"] + srcs + ["-o", out],
    ),
    # seeded input generator, host twin
    "libpolsar_gen_cpu": dict(
        out=os.path.join(PKG, "wishart", "libpolsar_gen_cpu.so"),
        srcs=[os.path.join(PKG, "wishart", "wishart_gen_cpu.c")],
        deps=[os.path.join(PKG, "wishart", "wishart_core.h"), os.path.join(INCLUDE, "polsar_gen.h")],
        cmd=lambda out, srcs: ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
                               "-fno-fast-math", "-mfma", "-I", INCLUDE] + srcs + ["-o", out, "-lm"],
    ),
}


def _stale(out: str, inputs) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(p) > t for p in inputs)


def build_target(name: str, force: bool = False, verbose: bool = False) -> str:
    t = TARGETS[name]
    if force or _stale(t["out"], t["srcs"] + t["deps"] + [__file__]):
        tmp = t["out"] + ".tmp"
        cmd = t["cmd"](tmp, t["srcs"])
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"build of {name} failed:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
        if verbose:
            print(res.stdout + res.stderr)
        os.replace(tmp, t["out"])
    return t["out"]


def build_all(force: bool = False, verbose: bool = False):
    return {name: build_target(name, force, verbose) for name in TARGETS}


if __name__ == "__main__":
    import sys
    build_all(force="--force" in sys.argv, verbose=True)
