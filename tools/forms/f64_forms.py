#!/usr/bin/env python
"""Accuracy and FP64 operation count of candidate fp64 Alg. 2 forms
(tools/forms/f64_forms.c, host emulation of the device arithmetic) against the
binary128 oracle on c4 samples (BASELINE configs[3]; host twin of the
generator) and on kappa-controlled matrices.  Development tool (uses the
oracle; not product code)."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1807_08084_b200 import configs, wishart  # noqa: E402
from tests.test_oracle import rand_kappa  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SO = "/tmp/libf64forms.so"
subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-mfma",
                       os.path.join(HERE, "f64_forms.c"), "-o", SO, "-lm"])
lib = ctypes.CDLL(SO)
P, I64 = ctypes.c_void_p, ctypes.c_int64
lib.form_eval.argtypes = [ctypes.c_int, P, I64, P, I64, I64, P]
NAMES = {0: "round-1 EFT", 1: "2u cofactors, FMA det", 2: "2u cofactors, compensated det",
         3: "plain", 4: "2u cofactors (dot3 diag), compensated det"}


def run(form, z):
    z = np.ascontiguousarray(z, dtype=np.float64)
    n = z.shape[1]
    out = np.empty((11, n))
    ops = ctypes.c_int(0)
    lib.form_eval(form, z.ctypes.data, n, out.ctypes.data, n, n, ctypes.byref(ops))
    return out, ops.value


def err(got, ref):
    inv = np.max(np.abs(got[:9] - ref[:9]), axis=0) / np.max(np.abs(ref[:9]), axis=0)
    det = np.abs(got[9] - ref[9]) / np.abs(ref[9])
    idet = np.abs(got[10] - ref[10]) / np.abs(ref[10])
    return np.maximum(inv, np.maximum(det, idet))


def main():
    cfg = configs.get("c4")
    rng = np.random.default_rng(1)
    idx = np.unique(rng.integers(0, cfg.n, 300_000)).astype(np.int64)
    sets = [("c4 sample 300k", wishart.generate_pixels_cpu(cfg, idx))]
    for k in (1e2, 1e3, 1e4):
        sets.append((f"U diag(1,k^u,k) U^H k={k:g}", rand_kappa(100_000, 5, k)))
    threads = len(os.sched_getaffinity(0))
    print("| data | form | FP64 ops | max err kappa<=1e2 | (1e2,1e3] | (1e3,1e4] | >1e4 |")
    print("|---|---|---|---|---|---|---|")
    for name, z in sets:
        ref = oracle.inv_det_threaded(z, threads)
        kap = oracle.kappa2(z)
        for form in (0, 1, 2, 4, 3):
            got, ops = run(form, z)
            e = err(got, ref)
            cells = []
            for lo, hi in ((0, 1e2), (1e2, 1e3), (1e3, 1e4), (1e4, np.inf)):
                m = (kap > lo) & (kap <= hi)
                cells.append(f"{e[m].max():.2e}" if m.any() else "-")
            print(f"| {name} | {form} {NAMES[form]} | {ops} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main()
