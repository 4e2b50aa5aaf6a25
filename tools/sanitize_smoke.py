#!/usr/bin/env python
"""Every C-ABI entry point once on small, ragged, misaligned and edge-case
inputs -- the program compute-sanitizer (memcheck / racecheck / synccheck) runs
over (tools/README.md).  Exits non-zero on any CUDA error."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1807_08084_b200 as P  # noqa: E402
from paper_1807_08084_b200 import configs, wishart  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    cfg = configs.get("c2").scaled(3, 333)
    for dt in (torch.float32, torch.float64):
        z = wishart.generate(cfg, device=dev).to(dt)
        n = z.shape[1]
        for plain in (False, True):
            for fn in (P.polsar_inv_det, P.polsar_inv_det_cholesky):
                # aligned, ragged tail
                out = torch.empty((11, n), dtype=dt, device=dev)
                st = torch.empty(n, dtype=torch.uint8, device=dev)
                fn(z, out, st, plain=plain)
                # misaligned planes (offset 1) and an odd plane stride
                zz = torch.empty((9, n + 3), dtype=dt, device=dev)[:, 1:n]
                zz.copy_(z[:, 1:])
                oo = torch.empty((11, n + 3), dtype=dt, device=dev)[:, 1:n]
                fn(zz, oo, None, plain=plain)
        zb = torch.cat([z, z], dim=0).contiguous()
        ob = torch.empty((20, n), dtype=dt, device=dev)
        P.polsar_inv_det_blocks(zb, ob, 2, torch.empty(n, dtype=torch.uint8, device=dev))
        P.polsar_checksum(out, n, 11, 0, st)
    # windows: edge tiles, tiny images, radius 0 and radii larger than the image
    for (h, w, r) in ((37, 45, 11), (1, 1, 0), (5, 3, 11), (70, 33, 14), (40, 260, 3)):
        z = wishart.generate(configs.get("c5").scaled(h, w), device=dev)
        for dt in (torch.float32, torch.float64):
            zz = z.to(dt)
            P.window_distance(zz, h, w, radius=r)
            P.window_distance(zz, h, w, radius=r, plain=True)
            P.nlm_filter(zz, h, w, radius=r)
            if r <= 12:
                P.window_kl(zz, h, w, radius=r)
        # a sub-range of output rows
        P.window_distance(z, h, w, radius=r, row_begin=h // 3, row_end=h - h // 4)
    # host pipeline with many chunks
    z = wishart.generate(configs.get("c2").scaled(20, 1000), device=dev)
    n = z.shape[1]
    zh = z.cpu().pin_memory()
    oh = torch.empty((11, n)).pin_memory()
    sh = torch.empty(n, dtype=torch.uint8).pin_memory()
    ws = torch.empty(1 << 20, dtype=torch.uint8, device=dev)
    P.polsar_inv_det_host(zh, oh, sh, ws, [torch.cuda.Stream() for _ in range(3)])
    torch.cuda.synchronize()
    print("sanitize smoke: ok")


if __name__ == "__main__":
    main()
