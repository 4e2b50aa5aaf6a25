"""Development aid: where does one window build differ from another (e.g. the
tensor-core pass 1 against a -DPOLSAR_WINDOW_MMA=0 build loaded with
POLSAR_LIB_OVERRIDE)?  Run once per build and compare."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_08084_b200 as P  # noqa: E402
from paper_1807_08084_b200 import configs, wishart  # noqa: E402

h, w, r = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
out = sys.argv[4]
z = wishart.generate(configs.get("c5").scaled(h, w), device="cuda")
got = P.window_distance(z, h, w, radius=r).cpu().numpy().reshape(h, w)
np.save(out, got)
if len(sys.argv) > 5:
    ref = np.load(sys.argv[5])
    rel = np.abs(got - ref) / ref
    print("max rel", rel.max())
    bad = rel > 2e-5
    print("bad count", bad.sum(), "of", bad.size)
    ys, xs = np.nonzero(bad)
    print("bad by x%32", np.bincount(xs % 32, minlength=32))
    print("bad by y%8", np.bincount(ys % 8, minlength=8))
    print("rows with bad", np.unique(ys)[:40])
    print("ratio got/ref sample", (got / ref)[bad][:10])
    print("constant-image check: got-ref at [5,5..12]", (got - ref)[5, 5:13])
