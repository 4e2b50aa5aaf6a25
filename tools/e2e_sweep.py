#!/usr/bin/env python
"""polsar_inv_det_host (the bench's e2e path) on the full c3 image from
pinned host buffers, for several staging-workspace sizes (chunk = ws / (3 x
81 B)): pipeline fill / drain against per-chunk overhead."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1807_08084_b200 as P  # noqa: E402
from paper_1807_08084_b200 import configs, wishart  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    cfg = configs.get("c3")
    z = wishart.generate(cfg, device=dev)
    n = z.shape[1]
    zh = torch.empty((9, n), dtype=z.dtype).pin_memory()
    zh.copy_(z)
    del z
    torch.cuda.empty_cache()
    oh = torch.empty((11, n), dtype=zh.dtype).pin_memory()
    sh = torch.empty(n, dtype=torch.uint8).pin_memory()
    streams = [torch.cuda.Stream() for _ in range(3)]
    res = {}
    for gb in [float(x) for x in sys.argv[1:]] or [0.375, 0.75, 1.5, 3.0, 6.0]:
        ws = torch.empty(int(gb * (1 << 30)), dtype=torch.uint8, device=dev)
        P.polsar_inv_det_host(zh, oh, sh, ws, streams)
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(streams[0])
            P.polsar_inv_det_host(zh, oh, sh, ws, streams)
            b.record(streams[2])
            b.synchronize()
            ts.append(a.elapsed_time(b))
        res[f"ws_{gb}GB"] = {"chunk_px": P.polsar_host_chunk_pixels(ws.numel(), 0), "ms": min(ts),
                             "matrices_per_s": n / (min(ts) / 1e3)}
        del ws
        torch.cuda.empty_cache()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
