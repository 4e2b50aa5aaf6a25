#!/usr/bin/env python
"""Accuracy of the window kernels on B200 against the long-double oracle
(R-12, R-19): the full-size c5 image (BASELINE configs[4]) in the
bench's launch configuration, a sample of pixels (corners, tile seams and
random ones) for W of the log-det window sum in each storage / arithmetic
mode, the KL window sum, and the NLM output (normwise over the 9 components,
and W).  Prints a markdown table of median / max relative errors.  Test
infrastructure: it uses the oracle, so it lives in tools/."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1807_08084_b200 as P  # noqa: E402
from paper_1807_08084_b200 import configs, wishart  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    threads = len(os.sched_getaffinity(0))
    cfg = configs.get("c5")
    h, w, R = cfg.height, cfg.width, cfg.radius
    z = wishart.generate(cfg, device=dev)
    rng = np.random.default_rng(11)
    seams = [y * w + x for y in (0, 31, 32, 63, 64, h - 1) for x in (0, 31, 32, 123, 124, w - 1)]
    idx = np.unique(np.concatenate([seams, rng.integers(0, h * w, 3000)])).astype(np.int64)
    zh = z.cpu().numpy()
    print(f"c5 {h}x{w}, R = {R}, L = {cfg.looks}, h = {cfg.h}; {idx.size} sampled pixels; "
          f"oracle in x87 long double on {threads} threads\n")
    print("| kernel | mode | tolerance | median rel. error | max rel. error |")
    print("|---|---|---|---|---|")

    def row(name, mode, tol, e):
        print(f"| {name} | {mode} | {tol} | {np.median(e):.2e} | {e.max():.2e} |", flush=True)

    ref = oracle.window_threaded(zh, h, w, R, cfg.looks, cfg.h, idx, threads)
    ii = torch.as_tensor(idx, device=dev)
    # the library's pass 1 for fp32 storage (compile-time POLSAR_WINDOW_MMA; a
    # -DPOLSAR_WINDOW_MMA=0 build loaded with POLSAR_LIB_OVERRIDE runs the scalar one)
    form = "scalar pass 1" if os.environ.get("POLSAR_LIB_OVERRIDE") else "tensor-core pass 1"
    for plain in (False, True):
        got = P.window_distance(z, h, w, radius=R, looks=cfg.looks, h=cfg.h, plain=plain)[ii].cpu().numpy()
        row("window W", "fp32 storage, fp32 pair det (plain; reported)" if plain else
            f"fp32 storage, fp64 pair det ({form})", "none" if plain else "2e-5", np.abs(got - ref) / ref)
    z64 = z.double()
    got = P.window_distance(z64, h, w, radius=R, looks=cfg.looks, h=cfg.h)[ii].cpu().numpy()
    ref64 = oracle.window_threaded(z64.cpu().numpy(), h, w, R, cfg.looks, cfg.h, idx, threads)
    row("window W", "fp64 storage", "1e-12", np.abs(got - ref64) / ref64)
    refk = oracle.window_kl_threaded(zh, h, w, R, cfg.looks, cfg.h, idx, threads)
    got = P.window_kl(z, h, w, radius=R, looks=cfg.looks, h=cfg.h)[ii].cpu().numpy()
    row("KL window W", f"fp32 storage, fp64 trace products ({form})", "2e-5", np.abs(got - refk) / refk)
    zhat, W = P.nlm_filter(z, h, w, radius=R, looks=cfg.looks, h=cfg.h)
    rz, rw = oracle.nlm_threaded(zh, h, w, R, cfg.looks, cfg.h, idx, threads)
    gz = zhat[:, ii].cpu().numpy().astype(np.float64)
    row("NLM Zhat (normwise)", "fp32 storage", "2e-5",
        np.max(np.abs(gz - rz), axis=0) / np.max(np.abs(rz), axis=0))
    row("NLM W", "fp32 storage", "2e-5", np.abs(W[ii].cpu().numpy() - rw) / rw)


if __name__ == "__main__":
    main()
