#!/usr/bin/env python
"""Quick kernel timings for development (not the bench line): K3 on c5 and
K1/K2 on a c3 slice, CUDA events on one stream, printed as JSON."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1807_08084_b200 as P  # noqa: E402
from paper_1807_08084_b200 import configs, wishart  # noqa: E402


def timeit(fn, stream, steps=10, warm=3):
    for _ in range(warm):
        fn()
    stream.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        fn()
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="window,k1")
    ap.add_argument("--rows", type=int, default=2500)
    ap.add_argument("--ref", default="", help="nlm: save outputs here, or compare with them")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    s = torch.cuda.Stream()
    res = {}
    with torch.cuda.stream(s):
        if "window" in a.what:
            c5 = configs.get("c5")
            z = wishart.generate(c5, device=dev, stream=s)
            for plain in (False, True):
                code = P.dtype_code(z.dtype, plain)
                ws = torch.empty(P.polsar_window_workspace_bytes(c5.height, c5.width, c5.radius, code),
                                 dtype=torch.uint8, device=dev)
                out = torch.empty(c5.n, dtype=z.dtype, device=dev)
                ms = timeit(lambda: P.polsar_window_distance(z, c5.width, c5.height, 0, c5.height,
                                                             c5.radius, c5.looks, c5.h, ws, out,
                                                             plain=plain, stream=s), s)
                res[f"window_c5{'_plain' if plain else ''}_ms"] = ms
            z64 = z.double()
            ws = torch.empty(P.polsar_window_workspace_bytes(c5.height, c5.width, c5.radius, 1),
                             dtype=torch.uint8, device=dev)
            out = torch.empty(c5.n, dtype=z64.dtype, device=dev)
            zz = torch.empty((9, c5.n), dtype=z.dtype, device=dev)
            wo = torch.empty(c5.n, dtype=z.dtype, device=dev)
            ws32 = torch.empty(P.polsar_window_workspace_bytes(c5.height, c5.width, c5.radius, 0),
                               dtype=torch.uint8, device=dev)
            res["nlm_c5_ms"] = timeit(lambda: P.polsar_nlm_filter(z, c5.width, c5.height, 0, c5.height,
                                                                  c5.radius, c5.looks, c5.h, ws32, zz, wo,
                                                                  stream=s), s, steps=3)
            res["kl_c5_ms"] = timeit(lambda: P.polsar_window_kl(z, c5.width, c5.height, 0, c5.height,
                                                                c5.radius, c5.looks, c5.h, ws32, wo,
                                                                stream=s), s, steps=3)
            res["kl_c5_fp64_ms"] = timeit(lambda: P.polsar_window_kl(z64, c5.width, c5.height, 0, c5.height,
                                                                     c5.radius, c5.looks, c5.h, ws, out,
                                                                     stream=s), s, steps=3)
            zz64 = torch.empty((9, c5.n), dtype=torch.float64, device=dev)
            res["nlm_c5_fp64_ms"] = timeit(lambda: P.polsar_nlm_filter(z64, c5.width, c5.height, 0, c5.height,
                                                                       c5.radius, c5.looks, c5.h, ws, zz64, out,
                                                                       stream=s), s, steps=3)
            res["window_c5_fp64_ms"] = timeit(lambda: P.polsar_window_distance(
                z64, c5.width, c5.height, 0, c5.height, c5.radius, c5.looks, c5.h, ws, out,
                stream=s), s, steps=3)
        if a.what == "nlm":
            c5 = configs.get("c5")
            z = wishart.generate(c5, device=dev, stream=s)
            zz = torch.empty((9, c5.n), dtype=z.dtype, device=dev)
            wo = torch.empty(c5.n, dtype=z.dtype, device=dev)
            ws32 = torch.empty(P.polsar_window_workspace_bytes(c5.height, c5.width, c5.radius, 0),
                               dtype=torch.uint8, device=dev)
            res["nlm_c5_ms"] = timeit(lambda: P.polsar_nlm_filter(z, c5.width, c5.height, 0, c5.height,
                                                                  c5.radius, c5.looks, c5.h, ws32, zz, wo,
                                                                  stream=s), s, steps=5)
            ref = torch.load(a.ref) if a.ref and os.path.exists(a.ref) else None
            if a.ref and ref is None:
                torch.save({"z": zz.cpu(), "w": wo.cpu()}, a.ref)
            elif ref is not None:
                res["nlm_bit_identical_to_ref"] = bool(torch.equal(ref["z"], zz.cpu()) and torch.equal(ref["w"], wo.cpu()))
        if "c4" in a.what:
            c4 = configs.get("c4").scaled(a.rows)
            z = wishart.generate(c4, device=dev, stream=s)
            out = torch.empty((11, c4.n), dtype=z.dtype, device=dev)
            st = torch.empty(c4.n, dtype=torch.uint8, device=dev)
            for name, fn in (("adj", P.polsar_inv_det), ("chol", P.polsar_inv_det_cholesky)):
                for plain in (False, True):
                    ms = timeit(lambda: fn(z, out, st, plain=plain, stream=s), s, steps=20)
                    key = f"{name}{'_plain' if plain else ''}_c4x{a.rows}"
                    res[key + "_ms"] = round(ms, 4)
                    res[key + "_pct"] = round(c4.n * 161 / ms / 1e6 / 6556.8 * 100, 1)
        if "k1" in a.what:
            c3 = configs.get("c3").scaled(a.rows)
            z = wishart.generate(c3, device=dev, stream=s)
            out = torch.empty((11, c3.n), dtype=z.dtype, device=dev)
            st = torch.empty(c3.n, dtype=torch.uint8, device=dev)
            for name, fn in (("adj", P.polsar_inv_det), ("chol", P.polsar_inv_det_cholesky)):
                ms = timeit(lambda: fn(z, out, st, stream=s), s)
                res[f"{name}_c3x{a.rows}_ms"] = ms
                res[f"{name}_c3x{a.rows}_GBps"] = c3.n * 81 / ms / 1e6
            z64 = z.double()
            out64 = torch.empty((11, c3.n), dtype=torch.float64, device=dev)
            for name, fn in (("adj", P.polsar_inv_det), ("chol", P.polsar_inv_det_cholesky)):
                for plain in (False, True):
                    ms = timeit(lambda: fn(z64, out64, st, plain=plain, stream=s), s)
                    key = f"{name}{'_plain' if plain else ''}_fp64_c3x{a.rows}"
                    res[key + "_ms"] = ms
                    res[key + "_GBps"] = c3.n * 161 / ms / 1e6
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
