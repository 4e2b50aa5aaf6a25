#!/usr/bin/env python
"""Accuracy of Alg. 2 vs Alg. 1 on B200 (the paper's §III-C claim,
PAPER.md:614-665, measured instead of argued).

For each data set and each kernel mode, the normwise inverse error (DESIGN.md
R-10) and the det error against the binary128 oracle, binned by kappa_2.
Outputs a markdown table (median / max per bin).  Test infrastructure: it
uses the oracle, so it lives in tools/, not in the product package.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1807_08084_b200 as P  # noqa: E402
from paper_1807_08084_b200 import configs, wishart  # noqa: E402

BINS = [(0, 1e2), (1e2, 1e3), (1e3, 1e4), (1e4, np.inf)]


def datasets(dev):
    yield "c1 (fp64, L=4, BASELINE Sigma)", wishart.generate(configs.get("c1"), device=dev)
    yield "c2 (fp32, L=4, quadrants)", wishart.generate(configs.get("c2").scaled(512), device=dev)
    c4 = configs.get("c4")
    tab = c4.table()
    rows = [wishart.generate(c4, r, r + 4, device=dev, table=tab) for r in (0, 2500, 5000, 7500)]
    yield "c4 (fp64, L=8, per-row Sigma + 1% kappa=1e6), 640k px", torch.cat(rows, dim=1).contiguous()
    yield "paper-sim (fp64, G G^H, PAPER.md:719-723), 500k", wishart.generate(
        configs.get("ctx_sim").scaled(1, 500000), device=dev)


def main():
    dev = torch.device("cuda:0")
    threads = len(os.sched_getaffinity(0))
    print("| data | kernel | kappa bin | pixels | inverse err median | inverse err max | det err median | det err max |")
    print("|---|---|---|---|---|---|---|---|")
    for name, z in datasets(dev):
        zh = z.cpu().numpy()
        ref = oracle.inv_det_threaded(zh, threads)
        k = oracle.kappa2(zh)
        modes = [("Alg. 2 (default)", "adjugate", False, False),
                 ("Alg. 2 as printed", "adjugate", True, False),
                 ("Alg. 1 (default)", "cholesky", False, False),
                 ("Alg. 1 as printed (l21 fixed)", "cholesky", True, False)]
        if z.dtype == torch.float64:
            modes.insert(1, ("Alg. 2 error-free (POLSAR_F64_EFT)", "adjugate", False, True))
        for kname, algo, plain, eft in modes:
            out, _ = P.inv_det(z, algo=algo, plain=plain, eft=eft)
            got = out.cpu().numpy().astype(np.float64)
            inv = np.max(np.abs(got[:9] - ref[:9]), axis=0) / np.max(np.abs(ref[:9]), axis=0)
            det = np.abs(got[9] - ref[9]) / np.abs(ref[9])
            for lo, hi in BINS:
                m = (k > lo) & (k <= hi)
                if m.sum() == 0:
                    continue
                print(f"| {name} | {kname} | ({lo:g}, {hi:g}] | {int(m.sum())} | {np.median(inv[m]):.2e} | "
                      f"{inv[m].max():.2e} | {np.median(det[m]):.2e} | {det[m].max():.2e} |")


if __name__ == "__main__":
    main()
