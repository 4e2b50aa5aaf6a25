#!/usr/bin/env python
"""Benchmark of the hot path: batched 3x3 Hermitian inverse + determinant
(arXiv 1807.08084, Alg. 2) on B200.

  python bench.py [--gpus N --steps K --warmup W] [--config c3] [--algo adjugate]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
  python bench.py --impl reference ...      # the CPU oracle, as it stands

A step is one pass of the hot path over one batch: the K1 kernel
(polsar_inv_det, Alg. 2) over this rank's pixels -- inverse (9 planes),
det Z, det Z^-1 and the status plane -- with the inputs resident in HBM.
Default workload: BASELINE configs[2] (c3), one 10000 x 40000 fp32 L=4
Wishart image whose pixel rows are sharded over the N GPUs (strong scaling,
"pixel rows sharded over 1/2/4/8 GPUs": rank r owns rows
[floor(r H / N), floor((r+1) H / N)); the checksum of the whole output is
then comparable across N).  --scaling weak gives every rank 10000 rows of an
N*10000-row image instead (its first 10000 rows are the 1-GPU image).
Inputs (14.4 GB) and outputs (17.6 GB) are far larger than the 126 MB L2,
so no flush is needed between steps; smaller shards flush L2 between steps.

Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "matrices/s (inverse+det)"
UNIT = "matrices/s"
FALLBACK_HBM_GBS = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", default="c3")
    p.add_argument("--algo", choices=["adjugate", "cholesky"], default="adjugate")
    p.add_argument("--plain", action="store_true", help="Alg. as printed in storage precision")
    p.add_argument("--scaling", choices=["weak", "strong"], default="strong",
                   help="strong (default): one BASELINE image sharded over the GPUs; weak: a fixed "
                        "image per GPU")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-extras", action="store_true", help="skip the K2 / K3 side measurements")
    p.add_argument("--no-status", action="store_true")
    p.add_argument("--verify", action="store_true", help="sampled oracle check after timing")
    p.add_argument("--kernel", choices=["inv_det", "window", "nlm", "kl"], default="inv_det",
                   help="inv_det (default: the metric of BASELINE.json) or a window kernel on c5")
    p.add_argument("--halo", choices=["regen", "exchange"], default="regen",
                   help="window kernels at N > 1: regenerate halo rows locally or exchange them (NCCL)")
    p.add_argument("--rows", type=int, default=0,
                   help="override rows per GPU (profiling runs only; not a bench line)")
    p.add_argument("--functional-1gpu", action="store_true",
                   help="test only: run every torchrun rank on cuda:0 with gloo (checks the N > 1 host "
                        "logic on a one-GPU box; not a measurement)")
    return p.parse_args()


# ------------------------------------------------------------------ helpers
def read_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def read_traffic(key):
    """dram bytes per launch from the committed ncu summary, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clock and throttle
    reasons during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting", 0x10: "sync_boost"}

    def __init__(self, device_index, period=0.01):
        self.period = period
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz,
                "reasons": [n for b, n in self.REASONS.items() if self.reasons & b],
                "samples": len(s)}


def setup_dist(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    return world, rank, local


def init_ranks(world, local):
    """One process per GPU over NCCL.  (--functional-1gpu: every rank on
    cuda:0 with gloo collectives -- a host-logic check of the N > 1 path on a
    one-GPU box, never a measurement: the ranks share one GPU.)"""
    import torch
    import torch.distributed as dist
    if ARGS.functional_1gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if ARGS.functional_1gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    return dev


def rows_for(rank, world, cfg, scaling):
    from paper_1807_08084_b200 import dist as pdist
    if scaling == "weak":
        return pdist.weak_rows(cfg.height, world, rank)
    return (cfg.height,) + pdist.shard_rows(cfg.height, world, rank)


def bytes_per_matrix(esz, status):
    return 20 * esz + (1 if status else 0)


def workload_name(cfg, args, world):
    base = f"{cfg.name}: BASELINE configs[{cfg.baseline_index}] {cfg.height}x{cfg.width} {cfg.dtype} L={cfg.looks}"
    if args.scaling == "strong":
        return base + f", the whole image sharded by pixel rows over {world} GPU(s)"
    return base + f" per GPU (weak scaling: an image of {world}x{cfg.height} rows)"


# The paper's own timings (Table 2): context
# only -- another machine, precision unstated.
PAPER_TABLE2 = {
    "hardware": "NVIDIA GeForce 940M (3 CUs, 2 GB), OpenCL, precision unstated (PAPER.md:676-687)",
    "replicates": 1000,
    "simulated_5469354": {"cholesky_ms": {"t_min": 498.89, "t_avg": 507.54, "t_max": 556.79, "t_std": 9.34},
                          "proposed_ms": {"t_min": 223.06, "t_avg": 231.51, "t_max": 273.08, "t_std": 6.11},
                          "proposed_matrices_per_s_avg": 5469354 / 0.23151},
    "airsar_270000": {"cholesky_ms": {"t_min": 24.68, "t_avg": 28.35, "t_max": 62.60, "t_std": 2.55},
                      "proposed_ms": {"t_min": 11.18, "t_avg": 12.98, "t_max": 28.59, "t_std": 1.44},
                      "proposed_matrices_per_s_avg": 270000 / 0.01298},
    "source": "PAPER.md:875-878 (Table 2)",
}


def config_dict(cfg, args, world, n, H, status_plane, bpm, flushed):
    """The `config` object both arms print (same workload description)."""
    return {
        "workload": workload_name(cfg, args, world),
        "algo": "Alg. 2 (adjugate)" if args.algo == "adjugate" else "Alg. 1 (Cholesky, l21 fixed)",
        "storage": cfg.dtype, "mode": "plain" if args.plain else "default",
        "pixels_per_gpu": n, "image_rows": H, "status_plane": status_plane,
        "l2": "flushed between steps" if flushed else
              f"inputs+outputs {n * bpm / 1e9:.1f} GB per step >> 126 MB L2 (no flush)",
        "parallelism": f"dp{world} (pixel rows)",
    }


# ------------------------------------------------------------ reference arm
def generate_host_sample(cfg, pixels, threads):
    """The first `pixels` pixels of cfg's image from the generator's host twin
    (bit-identical to the GPU generator), rows split over host threads."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor

    from paper_1807_08084_b200 import wishart
    rows = min(cfg.height, -(-pixels // cfg.width))
    tab = cfg.table()
    bounds = np.linspace(0, rows, max(1, min(threads, rows)) + 1).astype(int)
    with ThreadPoolExecutor(max_workers=len(bounds) - 1) as ex:
        parts = list(ex.map(lambda k: wishart.generate_cpu(cfg, int(bounds[k]), int(bounds[k + 1]), table=tab),
                            range(len(bounds) - 1)))
    return np.ascontiguousarray(np.concatenate(parts, axis=1)[:, :pixels])


def run_reference(args):
    """The CPU oracle (oracle/, as it stands: its storage-precision
    instantiation of the cofactor definition, the -O3 -march=native build) on
    the host cores, on a bounded sample of the same workload per step; rank 0
    only (the other ranks exit without work)."""
    world, rank, _ = setup_dist(args)
    if rank != 0:
        return 0
    import numpy as np

    import oracle
    from paper_1807_08084_b200 import configs

    cfg = configs.get(args.config)
    if args.rows:
        cfg = cfg.scaled(args.rows)
    cores = len(os.sched_getaffinity(0))
    sample = min(cfg.n, 1 << 24)  # 16.8M matrices per step
    z = generate_host_sample(cfg, sample, cores)
    out = np.empty((11, sample), dtype=z.dtype)
    for _ in range(max(args.warmup, 1)):
        oracle.inv_det_plain(z, cores, out=out)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.inv_det_plain(z, cores, out=out)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    value = sample / t
    esz = 4 if cfg.dtype == "float32" else 8
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f32" if esz == 4 else "f64",
        "data": "synthetic (seeded Wishart, host twin generator)",
        "config": dict(config_dict(cfg, args, world, cfg.n, cfg.height * (world if args.scaling == "weak" else 1),
                                   not args.no_status, bytes_per_matrix(esz, not args.no_status), False),
                       sample_pixels_per_step=sample),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"first {sample} pixels of {cfg.name} per step (host twin generator)",
                         "precision": f"{'float' if esz == 4 else 'double'} (the storage precision), "
                                      "gcc -O3 -march=native build of oracle/polsar_oracle.c",
                         "t_step_ms": {"min": min(times) * 1e3, "avg": t * 1e3, "max": max(times) * 1e3,
                                       "std": float(np.std(times)) * 1e3}},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "paper_table2_context": PAPER_TABLE2,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1807_08084_b200 as P
    from paper_1807_08084_b200 import configs, wishart

    world, rank, local = setup_dist(args)
    dev = init_ranks(world, local)

    cfg = configs.get(args.config)
    if cfg.radius:
        raise SystemExit("window configs are measured as an extra; pick c1..c4 for --config")
    if args.rows:
        cfg = cfg.scaled(args.rows)
    H, r0, r1 = rows_for(rank, world, cfg, args.scaling)
    n = (r1 - r0) * cfg.width
    tdt = torch.float32 if cfg.dtype == "float32" else torch.float64
    esz = 4 if tdt == torch.float32 else 8
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        tab = cfg.table(H)
        z = wishart.generate(cfg, r0, r1, device=dev, table=tab, height=H)
        out = torch.empty((11, n), dtype=tdt, device=dev)
        status = None if args.no_status else torch.empty(n, dtype=torch.uint8, device=dev)
    stream.synchronize()
    fn = P.polsar_inv_det if args.algo == "adjugate" else P.polsar_inv_det_cholesky

    l2_flush = None
    if n * bytes_per_matrix(esz, status is not None) < 4 * 126 * 2 ** 20:
        l2_flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device=dev)

    def step():
        fn(z, out, status, plain=args.plain, stream=stream)

    for _ in range(max(args.warmup, 3)):
        step()
    stream.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(dev.index if dev.index is not None else 0)
    with sampler:
        for i in range(args.steps):
            if l2_flush is not None:
                with torch.cuda.stream(stream):
                    l2_flush.sum(dtype=torch.int64)  # a 512 MB read: clean lines, no write-back tail
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        stream.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    per_step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    if l2_flush is None:
        # the K steps back to back: first start to last end on the stream
        t_local = starts[0].elapsed_time(ends[-1]) / 1e3
    else:
        # the L2 flush between steps is not part of a step
        t_local = sum(per_step_ms) / 1e3
    # roofline of the (only) kernel of the step
    bpm = bytes_per_matrix(esz, status is not None)
    achieved = n * bpm / (t_local / args.steps) / 1e9
    peak, peak_src = read_peaks()
    key = f"{cfg.name}:{args.algo}:{'plain' if args.plain else 'default'}"
    traffic = read_traffic(key)

    # SURVEY §8(a) row D, after the timed region: order-independent checksum
    # of all outputs + status counts (NCCL SUM; int64 wraps like uint64) and
    # the kernel time (NCCL MAX over ranks)
    from paper_1807_08084_b200 import dist as pdist
    res = P.polsar_checksum(out, n, 11, r0 * cfg.width, status, stream=stream)
    stream.synchronize()
    res, t_max = pdist.reduce_results(res, t_local)
    checksum = int(res[0].item()) & 0xFFFFFFFFFFFFFFFF
    counts = [int(x) for x in res[1:].tolist()]

    total = H * cfg.width  # every pixel of the image, over all ranks (shards may differ by a row)
    value = total * args.steps / t_max
    ms_per_step = t_max / args.steps * 1e3
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f32" if (args.plain and tdt == torch.float32) else "f64",
        "data": "synthetic (seeded Wishart, BASELINE law)",
        "config": config_dict(cfg, args, world, n, H, status is not None, bpm, l2_flush is not None),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_src, "bytes_per_matrix": bpm,
                     # north_star's "~8 TB/s" nominal HBM3e figure, reported beside the measured peak
                     "frac_of_nominal_8000": achieved / 8000.0},
        "clocks": sampler.summary(),
        "gpu_launches": args.steps,
        "checksum": f"{checksum:016x}", "status_counts": counts,
        "t_step_ms": {"min": min(per_step_ms), "avg": float(np.mean(per_step_ms)),
                      "max": max(per_step_ms), "std": float(np.std(per_step_ms))},
    }

    # ---------------- e2e: the public host-buffer entry point, copies inside
    if not args.no_e2e:
        line["e2e"] = measure_e2e(args, P, torch, dist, world, z, n, tdt, esz, dev, cfg)
    # ---------------- side measurements (same run): K2 and K3
    if not args.no_extras and rank == 0 and world == 1:
        line["extras"] = measure_extras(args, P, torch, z, out, status, stream, dev, esz)
    # ---------------- cpu baseline: the oracle on this host (rank 0, every N;
    # the other ranks wait at the barrier)
    if not args.no_cpu_baseline:
        if rank == 0:
            line["cpu_baseline"] = measure_cpu_baseline(z, cfg)
        if world > 1:
            dist.barrier()
    line["paper_table2_context"] = PAPER_TABLE2
    if args.verify:
        line["verify"] = verify_sample(P, z, out, status, cfg, r0)

    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def e2e_pixels(n, esz, world):
    """Pixels per rank for the host-buffer leg: the whole shard unless the
    pinned host buffers of all local ranks would exceed ~60 % of host RAM
    (an 8-GPU box pins 8 shards at once); the line reports the size used."""
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 64 << 30
    local = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    per_px = 20 * esz + 1
    cap = int(0.6 * avail / max(1, local) / per_px)
    m = min(n, max(cap, 1 << 20))
    return (m // 64) * 64 if m >= 64 else m


def measure_e2e(args, P, torch, dist, world, z, n_full, tdt, esz, dev, cfg):
    n = e2e_pixels(n_full, esz, world)
    if world > 1:  # every rank must move the same amount
        t = torch.tensor([n], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        n = int(t.item())
    zh = torch.empty((9, n), dtype=tdt).pin_memory()
    zh.copy_(z[:, :n])
    oh = torch.empty((11, n), dtype=tdt).pin_memory()
    sh = torch.empty(n, dtype=torch.uint8).pin_memory()
    ws = torch.empty(3 << 28, dtype=torch.uint8, device=dev)  # 0.75 GB: 3M-px chunks (tools/e2e_sweep.py)
    streams = [torch.cuda.Stream(device=dev) for _ in range(3)]
    algo = 0 if args.algo == "adjugate" else 1
    P.polsar_inv_det_host(zh, oh, sh, ws, streams, algo=algo, plain=args.plain)  # warm-up
    times = []
    for _ in range(args.e2e_steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(streams[0])
        P.polsar_inv_det_host(zh, oh, sh, ws, streams, algo=algo, plain=args.plain)
        t1.record(streams[2])
        t1.synchronize()
        times.append(t0.elapsed_time(t1) / 1e3)
    t = sum(times) / len(times)
    if world > 1:
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    del ws
    return {"value": n * world / t, "unit": UNIT, "h2d_bytes_per_step": 9 * n * esz * world,
            "d2h_bytes_per_step": (11 * n * esz + n) * world, "steps": args.e2e_steps,
            "ms_per_step": t * 1e3, "pixels_per_gpu": n,
            "path": "polsar_inv_det_host: pinned host -> 3-slot chunked H2D/kernel/D2H pipeline"}


def _time_kernel(torch, stream, fn, steps, warm=3):
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
    return a.elapsed_time(b) / 1e3 / steps


def _time_kernel_flushed(torch, stream, fn, steps, flush, warm=3):
    """Mean per-launch time with the L2 flushed (a 512 MB read) before every
    launch; only the launch is inside the events."""
    for _ in range(warm):
        fn()
    stream.synchronize()
    ts = []
    for i in range(steps):
        with torch.cuda.stream(stream):
            flush.sum(dtype=torch.int64)  # read 512 MB: evicts with clean lines, no write-back tail
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        ts.append((a, b))
    stream.synchronize()
    return sum(a.elapsed_time(b) for a, b in ts) / 1e3 / steps


def measure_extras(args, P, torch, z, out, status, stream, dev, esz):
    from paper_1807_08084_b200 import configs, wishart
    n = z.shape[1]
    peak, _ = read_peaks()
    bpm = bytes_per_matrix(esz, status is not None)
    res = {}
    steps = max(5, min(args.steps, 20))
    for algo, fn in (("adjugate", P.polsar_inv_det), ("cholesky", P.polsar_inv_det_cholesky)):
        for plain in (False, True):
            t = _time_kernel(torch, stream, lambda: fn(z, out, status, plain=plain, stream=stream), steps)
            gbs = n * bpm / t / 1e9
            res[f"{algo}{'_plain' if plain else ''}"] = {
                "matrices_per_s": n / t, "ms": t * 1e3, "GB/s": gbs, "frac_hbm": gbs / peak}
    # BASELINE configs[1] (c2: 1024^2 fp32, 4 quadrant classes), the paper-scale
    # head-to-head of both kernels; 84 MB fits the 126 MB L2, so it is flushed
    # before every launch (launch-latency bound: ~13 us at the HBM roof)
    c2 = configs.get("c2")
    with torch.cuda.stream(stream):
        z2 = wishart.generate(c2, device=dev)
        o2 = torch.empty((11, c2.n), dtype=z2.dtype, device=dev)
        s2 = torch.empty(c2.n, dtype=torch.uint8, device=dev)
        flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device=dev)
    stream.synchronize()
    for algo, fn in (("adjugate", P.polsar_inv_det), ("cholesky", P.polsar_inv_det_cholesky)):
        t = _time_kernel_flushed(torch, stream, lambda: fn(z2, o2, s2, stream=stream), steps, flush)
        gbs = c2.n * 81 / t / 1e9
        res[f"c2_{algo}"] = {"matrices_per_s": c2.n / t, "ms": t * 1e3, "GB/s": gbs, "frac_hbm": gbs / peak,
                             "mode": "fp32 storage, L2 flushed before each launch"}
    del z2, o2, s2, flush
    torch.cuda.empty_cache()
    # K1 / K2 on BASELINE configs[3] (c4: 4e8 px fp64 storage), 161 B / matrix:
    # POLSAR_F64 (Alg. 2 with ~2u cofactors, compensated Eq. 6), the
    # error-free POLSAR_F64_EFT, and Alg. 1
    c4 = configs.get("c4")
    with torch.cuda.stream(stream):
        z4 = wishart.generate(c4, device=dev)
        o4 = torch.empty((11, c4.n), dtype=z4.dtype, device=dev)
        s4 = torch.empty(c4.n, dtype=torch.uint8, device=dev)
    stream.synchronize()
    for key, fn, mode in (("c4_adjugate", lambda: P.polsar_inv_det(z4, o4, s4, stream=stream),
                           "fp64 storage, POLSAR_F64 (compensated Alg. 2)"),
                          ("c4_adjugate_eft", lambda: P.polsar_inv_det(z4, o4, s4, stream=stream, eft=True),
                           "fp64 storage, POLSAR_F64_EFT (error-free Alg. 2)"),
                          ("c4_cholesky", lambda: P.polsar_inv_det_cholesky(z4, o4, s4, stream=stream),
                           "fp64 storage, Alg. 1")):
        t = _time_kernel(torch, stream, fn, max(3, steps // 2))
        gbs = c4.n * 161 / t / 1e9
        res[key] = {"matrices_per_s": c4.n / t, "ms": t * 1e3, "GB/s": gbs, "frac_hbm": gbs / peak, "mode": mode}
    del z4, o4, s4
    torch.cuda.empty_cache()
    # K5: 3-band block-diagonal pixels of c3's law,
    # 1e8 px (2500 of c3's rows per band), fp32 storage; (27 + 29) * 4 + 1 B / pixel
    cb = configs.get("c3").scaled(2500)
    nb = 3
    with torch.cuda.stream(stream):
        zb = wishart.generate_bands(cb, nb, device=dev)
        ob = torch.empty((9 * nb + 2, cb.n), dtype=zb.dtype, device=dev)
        sb = torch.empty(cb.n, dtype=torch.uint8, device=dev)
    stream.synchronize()
    t = _time_kernel(torch, stream, lambda: P.polsar_inv_det_blocks(zb, ob, nb, sb, stream=stream),
                     max(3, steps // 2))
    bpp = (9 * nb + 9 * nb + 2) * zb.element_size() + 1
    gbs = cb.n * bpp / t / 1e9
    res["blocks_c3_3bands"] = {"pixels_per_s": cb.n / t, "ms": t * 1e3, "GB/s": gbs, "frac_hbm": gbs / peak,
                               "bytes_per_pixel": bpp, "mode": "3 bands x c3 law, 1e8 px, fp32 storage"}
    del zb, ob, sb
    torch.cuda.empty_cache()
    # K3: BASELINE configs[4] window sum on one GPU
    c5 = configs.get("c5")
    with torch.cuda.stream(stream):
        z5 = wishart.generate(c5, device=dev)
        code = P.dtype_code(z5.dtype)
        ws = torch.empty(P.polsar_window_workspace_bytes(c5.height, c5.width, c5.radius, code),
                         dtype=torch.uint8, device=dev)
        w5 = torch.empty(c5.n, dtype=z5.dtype, device=dev)
    stream.synchronize()
    pairs = window_pairs(c5.height, c5.width, c5.radius)
    for plain in (False, True):
        t = _time_kernel(torch, stream, lambda: P.polsar_window_distance(
            z5, c5.width, c5.height, 0, c5.height, c5.radius, c5.looks, c5.h, ws, w5,
            plain=plain, stream=stream), steps)
        res[f"window_c5{'_plain' if plain else ''}"] = {
            "pairs_per_s": pairs / t, "ms": t * 1e3, "pairs": pairs,
            "mode": "fp32 storage, fp32 weight, " + ("fp32 pair det" if plain else "fp64 pair det") +
                    ("" if plain else " (DMMA mixed-discriminant pass 1)")}
    # K6 (KL window) and K4 (NLM filter) on the same c5 input
    t = _time_kernel(torch, stream, lambda: P.polsar_window_kl(
        z5, c5.width, c5.height, 0, c5.height, c5.radius, c5.looks, c5.h, ws, w5, stream=stream), steps)
    res["kl_window_c5"] = {"pairs_per_s": pairs / t, "ms": t * 1e3, "pairs": pairs,
                           "mode": "symmetric Wishart KL, fp32 storage, fp64 trace products (DMMA pass 1)"}
    zn = torch.empty((9, c5.n), dtype=z5.dtype, device=dev)
    t = _time_kernel(torch, stream, lambda: P.polsar_nlm_filter(
        z5, c5.width, c5.height, 0, c5.height, c5.radius, c5.looks, c5.h, ws, zn, w5, stream=stream), steps)
    res["nlm_c5"] = {"pairs_per_s": pairs / t, "ms": t * 1e3, "pairs": pairs,
                     "mode": "NLM output (W and Zhat), fp32 storage, fp64 pair det"}
    return res


def window_pairs(h, w, r):
    def clipped(n):
        import numpy as np
        i = np.arange(n)
        return int(np.sum(np.minimum(n - 1, i + r) - np.maximum(0, i - r) + 1))
    return clipped(h) * clipped(w)


def measure_cpu_baseline(z, cfg):
    """SURVEY §8(d)'s CPU baseline: the oracle's storage-precision
    instantiation of the cofactor definition (float for fp32 storage, double
    for fp64; gcc -O3 -march=native), on this box's host cores and on one
    core, over the first 1e7 pixels of this rank's input (D2H copy); warm-up
    1, then 5 replicates (Table-2 style t_min / t_avg / t_max / t_std).  The
    binary128 verification oracle's rate is reported beside it."""
    import numpy as np

    import oracle
    cores = len(os.sched_getaffinity(0))
    m = int(min(z.shape[1], 10_000_000))
    zs = z[:, :m].cpu().numpy()
    out = np.empty((11, m), dtype=zs.dtype)

    def reps(threads, cols, k):
        zc = zs if cols == m else np.ascontiguousarray(zs[:, :cols])
        o = out if cols == m else np.empty((11, cols), dtype=zs.dtype)
        oracle.inv_det_plain(zc, threads, out=o)  # warm-up (also first-touches o)
        ts = []
        for _ in range(k):
            t0 = time.perf_counter()
            oracle.inv_det_plain(zc, threads, out=o)
            ts.append(time.perf_counter() - t0)
        return ts

    ts = reps(cores, m, 5)
    t = float(np.mean(ts))
    m1 = min(m, 2_000_000)
    ts1 = reps(1, m1, 3)
    mq = min(m, 1 << 20)
    t0 = time.perf_counter()
    oracle.inv_det_threaded(zs[:, :mq], cores)
    tq = time.perf_counter() - t0
    prec = "float" if zs.dtype == np.float32 else "double"
    return {"value": m / t, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"first {m} pixels of this rank's {cfg.name} input (D2H copy), 5 replicates on "
                      f"{cores} threads",
            "precision": f"{prec} (the storage precision), gcc -O3 -march=native build of oracle/polsar_oracle.c",
            "t_ms": {"min": min(ts) * 1e3, "avg": t * 1e3, "max": max(ts) * 1e3, "std": float(np.std(ts)) * 1e3},
            "single_core": {"value": m1 / float(np.mean(ts1)), "sample": f"first {m1} pixels, 3 replicates, 1 thread"},
            "binary128_oracle": {"value": mq / tq, "cores": cores,
                                 "sample": f"first {mq} pixels, 1 pass (the verification oracle, not a baseline)"}}


def verify_sample(P, z, out, status, cfg, r0):
    import numpy as np

    import oracle
    rng = np.random.default_rng(1)
    n = z.shape[1]
    idx = np.unique(rng.integers(0, n, 20000))
    ii = __import__("torch").as_tensor(idx, device=z.device)
    zs = z[:, ii].cpu().numpy()
    ref = oracle.inv_det(zs)
    got = out[:, ii].cpu().numpy().astype(np.float64)
    k = oracle.kappa2(zs)
    m = k <= 1e4
    inv = np.max(np.abs(got[:9] - ref[:9]), axis=0) / np.max(np.abs(ref[:9]), axis=0)
    det = np.abs(got[9] - ref[9]) / np.abs(ref[9])
    return {"pixels": int(idx.size), "kappa_le_1e4": int(m.sum()),
            "max_rel_inv": float(inv[m].max()), "max_rel_det": float(det[m].max())}


# FP64 pipe peak: 64 lanes / clk / SM x 148 SMs x 1.965 GHz
FP64_PEAK_OPS = 64 * 148 * 1.965e9
FP64_OPS_PER_PAIR = {"window": 29, "window_mma": 20, "nlm": 40, "kl": 19}


def run_window(args):
    """Window kernels (BASELINE configs[4], c5) sharded by pixel rows: the
    2048 x 2048 image split over the N GPUs (strong, the default) or rank r
    owning rows [r*2048, (r+1)*2048) of an N*2048-row image (weak); each
    rank's +-R halo rows are regenerated locally (exact: the generator is
    keyed by global pixel) or exchanged with the neighbouring ranks over NCCL
    (--halo exchange, inside the timed step)."""
    import torch
    import torch.distributed as dist

    import paper_1807_08084_b200 as P
    from paper_1807_08084_b200 import configs, wishart
    from paper_1807_08084_b200 import dist as pdist

    world, rank, local = setup_dist(args)
    dev = init_ranks(world, local)
    cfg = configs.get("c5")
    if args.rows:
        cfg = cfg.scaled(args.rows)
    R, W = cfg.radius, cfg.width
    H, r0, r1 = rows_for(rank, world, cfg, args.scaling)
    s0, s1, ob, oe = pdist.halo_slab(r0, r1, H, R)
    if args.halo == "exchange" and world > 1:
        pdist.check_halo_geometry(r1 - r0, R, device=dev)
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        tab = cfg.table(H)
        if args.halo == "regen" or world == 1:
            slab = wishart.generate(cfg, s0, s1, device=dev, table=tab, height=H)
        else:
            slab = torch.zeros((9, (s1 - s0) * W), dtype=torch.float32, device=dev)
            own = wishart.generate(cfg, r0, r1, device=dev, table=tab, height=H)
            slab[:, ob * W:oe * W] = own
        code = P.dtype_code(slab.dtype)
        ws = torch.empty(P.polsar_window_workspace_bytes(s1 - s0, W, R, code), dtype=torch.uint8, device=dev)
        out = torch.empty((oe - ob) * W, dtype=slab.dtype, device=dev)
        outz = torch.empty((9, (oe - ob) * W), dtype=slab.dtype, device=dev)
    stream.synchronize()

    def step():
        if args.halo == "exchange" and world > 1:
            with torch.cuda.stream(stream):
                pdist.exchange_halos(slab, W, ob, oe, R)
        if args.kernel == "window":
            P.polsar_window_distance(slab, W, s1 - s0, ob, oe, R, cfg.looks, cfg.h, ws, out, stream=stream)
        elif args.kernel == "nlm":
            P.polsar_nlm_filter(slab, W, s1 - s0, ob, oe, R, cfg.looks, cfg.h, ws, outz, out, stream=stream)
        else:
            P.polsar_window_kl(slab, W, s1 - s0, ob, oe, R, cfg.looks, cfg.h, ws, out, stream=stream)

    for _ in range(max(args.warmup, 3)):
        step()
    stream.synchronize()
    steps = args.steps
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(dev.index if dev.index is not None else 0)
    with sampler:
        a.record(stream)
        for _ in range(steps):
            step()
        b.record(stream)
        stream.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_local = a.elapsed_time(b) / 1e3
    res = P.polsar_checksum(out, (oe - ob) * W, 1, r0 * W, stream=stream)
    stream.synchronize()
    res, t_max = pdist.reduce_results(res, t_local)
    pairs_rank = window_pairs_rows(H, W, R, r0, r1)
    pairs = window_pairs_rows(H, W, R, 0, H)  # every output row of the image, over all ranks
    ops = FP64_OPS_PER_PAIR[args.kernel]
    # which form the library runs (fixed at compile time: csrc/window.cu, nlm.cu)
    mma = False
    if args.kernel == "nlm":
        symmetric = 1 <= R <= 12
        variant = ("symmetric two-pass (pass 1 + TMA gather, 1024-row bands)" if symmetric else "direct")
    else:
        symmetric = R <= 12
        variant = "symmetric two-pass" if symmetric else "direct"
        # the tensor-core pass 1 (csrc/window_mma.cuh; the product for fp32 storage): each
        # unordered pair is a 20-term fp64 dot product, 20 FMAs on the same FP64 datapath
        # (DMMA.8x8x4 shares the 64 FMA/clk/SM peak); the KL window's two trace
        # products and the -6 are the same 20-term product
        mma = symmetric and cfg.dtype == "float32"
        if mma:
            variant = "symmetric two-pass, pass 1 on the FP64 tensor cores (DMMA)"
            ops = FP64_OPS_PER_PAIR["window_mma"]
    if symmetric:
        # d(i, j) is symmetric: the algorithmic FP64 work is one evaluation per
        # unordered pair, which is what the symmetric kernels do;
        # NLM's gather pass adds no FP64 work (9 FP32 FMAs per ordered pair)
        work_pairs = unordered_pairs_rows(H, W, R, r0, r1)
        ops = FP64_OPS_PER_PAIR["window"] if args.kernel == "nlm" else ops  # (NLM's pass 1 is scalar)
        launches = 2 if mma else 3  # (prep,) forward pass, backward / gather pass
    else:
        work_pairs = pairs_rank
        launches = 2  # prep, window sum
    achieved = ops * work_pairs / (t_local / steps)
    line = {
        "metric": f"pairs/s ({args.kernel} search-window sum, 23x23)", "value": pairs * steps / t_max,
        "unit": "pairs/s", "n_gpus": world, "steps": steps, "warmup": max(args.warmup, 3),
        "ms_per_step": t_max / steps * 1e3, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Wishart, BASELINE law)",
        "config": {"workload": f"c5: BASELINE configs[4] {cfg.height}x{W} float32 L={cfg.looks} R={R}" +
                               (f", sharded by pixel rows over {world} GPU(s)" if args.scaling == "strong"
                                else " per GPU"), "kernel": args.kernel, "halo": args.halo,
                   "l2": "compute-bound; inputs 151 MB staged once per tile",
                   "parallelism": f"dp{world} (pixel rows + {R}-row halos)",
                   "variant": variant},
        "roofline": {"bound": "alu", "achieved": achieved / 1e12, "peak": FP64_PEAK_OPS / 1e12,
                     "unit": "T fp64-ops/s", "frac": achieved / FP64_PEAK_OPS, "traffic": None,
                     "ops_per_pair": ops, "pairs_evaluated": work_pairs,
                     **({"issued_fma_per_pair": mma_issued_per_pair(R),
                         "issued_frac": mma_issued_per_pair(R) * work_pairs / (t_local / steps) / FP64_PEAK_OPS}
                        if mma else {}),
                     "timed": "whole call (prep + all passes), CUDA events on the launch stream",
                     "peak_source": "64 FP64 lanes/clk/SM x 148 SMs x 1.965 GHz (DESIGN.md §6)"},
        "clocks": sampler.summary(), "gpu_launches": launches * steps,
        "checksum": f"{int(res[0].item()) & 0xFFFFFFFFFFFFFFFF:016x}",
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def window_pairs_rows(h, w, r, r0, r1):
    """Clipped window pairs of output rows [r0, r1) of an h x w image."""
    import numpy as np
    ys = np.arange(r0, r1)
    ny = np.minimum(h - 1, ys + r) - np.maximum(0, ys - r) + 1
    xs = np.arange(w)
    nx = np.minimum(w - 1, xs + r) - np.maximum(0, xs - r) + 1
    return int(ny.sum()) * int(nx.sum())


def mma_issued_per_pair(r):
    """DMMA FMAs the tensor-core pass 1 issues per unordered pair of an interior
    pixel: (R+1) window rows x NT 8-pixel blocks x 5 DMMA x 256 FMA per 8 owned
    pixels, over the 2R(R+1) pairs each pixel owns (masked pairs included)."""
    nt = (2 * r + 15) // 8
    return (r + 1) * nt * 5 * 256 / 8 / (2 * r * (r + 1))


def unordered_pairs_rows(h, w, r, r0, r1):
    """Distinct unordered off-diagonal window pairs {i, j} with at least one
    endpoint in output rows [r0, r1): ordered pairs from the output rows minus
    half of those with both endpoints inside them."""
    n = (r1 - r0) * w
    a = window_pairs_rows(h, w, r, r0, r1) - n
    b = window_pairs_rows(r1 - r0, w, r, 0, r1 - r0) - n
    return a - b // 2


ARGS = None


def main():
    global ARGS
    args = parse()
    ARGS = args
    if args.impl == "reference":
        return run_reference(args)
    if args.kernel != "inv_det":
        return run_window(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
