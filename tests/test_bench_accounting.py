"""bench.py's work accounting (CPU): the window pair counts behind the
reported pairs/s and roofline numbers, against brute-force enumeration of the
clipped (2R+1)^2 window (§II, the search window of the NLM filter)."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def brute(h, w, r, r0, r1):
    ordered, unordered = 0, set()
    for y in range(r0, r1):
        for x in range(w):
            for dy in range(-r, r + 1):
                for dx in range(-r, r + 1):
                    yy, xx = y + dy, x + dx
                    if 0 <= yy < h and 0 <= xx < w:
                        ordered += 1
                        if (dy, dx) != (0, 0):
                            unordered.add(frozenset([(y, x), (yy, xx)]))
    return ordered, len(unordered)


@pytest.mark.parametrize("h,w,r,r0,r1", [(7, 5, 2, 0, 7), (7, 5, 2, 2, 5), (9, 4, 3, 0, 3),
                                         (6, 11, 1, 5, 6), (3, 3, 5, 0, 3), (12, 8, 0, 3, 9)])
def test_pair_counts(bench, h, w, r, r0, r1):
    ordered, unordered = brute(h, w, r, r0, r1)
    assert bench.window_pairs_rows(h, w, r, r0, r1) == ordered
    assert bench.unordered_pairs_rows(h, w, r, r0, r1) == unordered


def test_full_image_halves(bench):
    # whole image: every unordered off-diagonal pair is one of two ordered ones
    h, w, r = 40, 33, 11
    n = h * w
    assert bench.unordered_pairs_rows(h, w, r, 0, h) * 2 == bench.window_pairs_rows(h, w, r, 0, h) - n


def test_default_is_the_whole_baseline_image(bench, monkeypatch):
    """bench.py's default N > 1 line measures BASELINE configs[2] itself: one
    10000 x 40000 image whose pixel rows are split over the ranks (strong
    scaling), so the union of the shards is the 1-GPU image and the output
    checksum is comparable across N."""
    import sys
    from paper_1807_08084_b200 import configs
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "8"])
    args = bench.parse()
    assert args.scaling == "strong" and args.config == "c3"
    cfg = configs.get("c3")
    rows = []
    for rank in range(8):
        H, r0, r1 = bench.rows_for(rank, 8, cfg, args.scaling)
        assert H == cfg.height
        rows.extend(range(r0, r1))
    assert rows == list(range(cfg.height))
    assert "whole image sharded" in bench.workload_name(cfg, args, 8)
