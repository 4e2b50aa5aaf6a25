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


def _run(cmd, env=None):
    import json
    import subprocess
    import sys
    r = subprocess.run([sys.executable] + cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    return [json.loads(l) for l in lines]


def test_reference_arm_line():
    """`bench.py --impl reference` (CPU only: the oracle's storage-precision
    build on the host cores) prints one JSON line with the contract's keys."""
    (line,) = _run(["bench.py", "--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1"])
    assert line["impl"] == "reference" and line["unit"] == "matrices/s" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["gpu_launches"] == 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["config"]["workload"].startswith("c1: BASELINE configs[0]")
    assert line["paper_table2_context"]["simulated_5469354"]["proposed_ms"]["t_avg"] == 231.51


def test_reference_arm_under_torchrun():
    """Under torchrun only rank 0 runs and prints; the other ranks exit 0."""
    import os
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    lines = _run(["-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
                  "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference", "--gpus", "2",
                  "--config", "c1", "--steps", "1", "--warmup", "1"], env=dict(os.environ, OMP_NUM_THREADS="1"))
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2
