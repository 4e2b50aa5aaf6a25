#!/usr/bin/env python
"""PCIe bandwidth on the GPU box: H2D alone, D2H alone, and both at once
(separate streams), pinned host buffers, for the chunk sizes the host
pipeline uses.  Context for bench.py's e2e figure."""
import json
import torch


def bw(fn, nbytes, reps=5):
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return nbytes * reps / (a.elapsed_time(b) / 1e3) / 1e9


def main():
    total = 4 << 30
    res = {}
    h = torch.empty(total, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(total, dtype=torch.uint8).pin_memory()
    d = torch.empty(total, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(total, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for chunk_mb in (16, 64, 256):
        c = chunk_mb << 20
        n = total // c

        def h2d():
            with torch.cuda.stream(s1):
                for i in range(n):
                    d[i * c:(i + 1) * c].copy_(h[i * c:(i + 1) * c], non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)

        def d2h():
            with torch.cuda.stream(s2):
                for i in range(n):
                    h2[i * c:(i + 1) * c].copy_(d2[i * c:(i + 1) * c], non_blocking=True)
            torch.cuda.current_stream().wait_stream(s2)

        def both():
            with torch.cuda.stream(s1):
                for i in range(n):
                    d[i * c:(i + 1) * c].copy_(h[i * c:(i + 1) * c], non_blocking=True)
            with torch.cuda.stream(s2):
                for i in range(n):
                    h2[i * c:(i + 1) * c].copy_(d2[i * c:(i + 1) * c], non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)

        res[f"{chunk_mb}MB"] = {"h2d_GBs": bw(h2d, total), "d2h_GBs": bw(d2h, total),
                                "bidir_total_GBs": bw(both, 2 * total)}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
