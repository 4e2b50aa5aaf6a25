#!/usr/bin/env python
"""Mean per-kernel metrics of an `ncu --csv --log-file` launch list."""
import collections
import csv
import sys


def main(path):
    hdr = None
    d = collections.defaultdict(list)
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            k = r[hdr.index("Kernel Name")][:70]
            v = r[hdr.index("Metric Value")].replace(",", "")
            try:
                d[(k, r[hdr.index("Metric Name")])].append(float(v))
            except ValueError:
                pass
    for (k, m), v in sorted(d.items()):
        print(f"{k:70s} {m[:45]:45s} n={len(v):3d} mean={sum(v) / len(v):.4g}")


if __name__ == "__main__":
    main(sys.argv[1])
