#!/usr/bin/env python
"""Why does Alg. 1 (K2) slow down per pixel as the c3 image grows (1.36 ms per
1e8 px at 2500 rows, 1.51 at 10000) while Alg. 2 (K1) stays linear?  Times K2
and K1 on row ranges of one full-size c3 image (same plane stride): data
dependence shows as a difference between ranges of equal size, footprint
dependence as growth with the range size."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1807_08084_b200 as P  # noqa: E402
from paper_1807_08084_b200 import configs, wishart  # noqa: E402
from tools.kbench import timeit  # noqa: E402
from bench import ClockSampler  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    s = torch.cuda.Stream()
    cfg = configs.get("c3")
    W = cfg.width
    res = {}
    with torch.cuda.stream(s):
        z = wishart.generate(cfg, device=dev, stream=s)
        out = torch.empty((11, cfg.n), dtype=z.dtype, device=dev)
        st = torch.empty(cfg.n, dtype=torch.uint8, device=dev)
        order = ((7500, 10000), (0, 2500), (5000, 7500), (2500, 5000), (0, 10000), (0, 2500), (7500, 10000))
        for r0, r1 in order:
            zs, os_, ss = z[:, r0 * W:r1 * W], out[:, r0 * W:r1 * W], st[r0 * W:r1 * W]
            for name, fn in (("k1", P.polsar_inv_det), ("k2", P.polsar_inv_det_cholesky)):
                with ClockSampler(0, period=0.002) as cs:
                    ms = timeit(lambda: fn(zs, os_, ss, stream=s), s, steps=10)
                res[f"{name}_rows{r0}-{r1}_clocks"] = res.get(f"{name}_rows{r0}-{r1}_clocks", []) + [cs.summary()]
                res[f"{name}_rows{r0}-{r1}_ms_per_1e8"] = res.get(f"{name}_rows{r0}-{r1}_ms_per_1e8", []) + [
                    round(ms / ((r1 - r0) * W) * 1e8, 4)]
        del z, out, st
        torch.cuda.empty_cache()
        # the last 2500 rows' data in a fresh 1e8-pixel allocation
        zl = wishart.generate(cfg, 7500, 10000, device=dev, stream=s)
        ol = torch.empty((11, zl.shape[1]), dtype=zl.dtype, device=dev)
        sl = torch.empty(zl.shape[1], dtype=torch.uint8, device=dev)
        for name, fn in (("k1", P.polsar_inv_det), ("k2", P.polsar_inv_det_cholesky)):
            res[f"{name}_fresh_rows7500-10000_ms_per_1e8"] = round(
                timeit(lambda: fn(zl, ol, sl, stream=s), s, steps=10) / zl.shape[1] * 1e8, 4)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
