"""The C-ABI calls are asynchronous, allocation-free and stream-ordered, so
they can run on several streams at once and be captured in CUDA graphs
(replaying a captured hot path avoids launch overhead on small batches)."""
import numpy as np
import pytest
import torch

import paper_1807_08084_b200 as P
from paper_1807_08084_b200 import configs, wishart

pytestmark = pytest.mark.gpu


def test_cuda_graph_capture_replay(cuda):
    cfg = configs.get("c1")
    z = wishart.generate(cfg, device=cuda)
    out = torch.empty((11, z.shape[1]), dtype=z.dtype, device=cuda)
    st = torch.empty(z.shape[1], dtype=torch.uint8, device=cuda)
    c5 = configs.get("c5").scaled(64, 96)
    z5 = wishart.generate(c5, device=cuda)
    ws = torch.empty(P.polsar_window_workspace_bytes(64, 96, 11, 0), dtype=torch.uint8, device=cuda)
    w5 = torch.empty(64 * 96, dtype=z5.dtype, device=cuda)
    ref_out, ref_st = P.inv_det(z)
    ref_w = P.window_distance(z5, 64, 96)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up outside capture (cudaFuncSetAttribute etc.)
        P.polsar_inv_det(z, out, st, stream=s)
        P.polsar_window_distance(z5, 96, 64, 0, 64, 11, 4.0, 1.0, ws, w5, stream=s)
    s.synchronize()
    out.zero_()
    w5.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        P.polsar_inv_det(z, out, st, stream=s)
        P.polsar_window_distance(z5, 96, 64, 0, 64, 11, 4.0, 1.0, ws, w5, stream=s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref_out) and torch.equal(st, ref_st)
    assert torch.equal(w5, ref_w)


def test_concurrent_streams_equal_serial(cuda):
    cfg = configs.get("c2").scaled(256)
    z = wishart.generate(cfg, device=cuda)
    n = z.shape[1]
    ref, ref_st = P.inv_det(z)
    out = torch.empty_like(ref)
    st = torch.empty_like(ref_st)
    streams = [torch.cuda.Stream() for _ in range(4)]
    torch.cuda.synchronize()
    bounds = np.linspace(0, n, 5).astype(int) // 4 * 4
    bounds[-1] = n
    for k, s in enumerate(streams):
        lo, hi = int(bounds[k]), int(bounds[k + 1])
        with torch.cuda.stream(s):
            P.polsar_inv_det(z[:, lo:hi], out[:, lo:hi], st[lo:hi], stream=s)
    torch.cuda.synchronize()
    assert torch.equal(out, ref) and torch.equal(st, ref_st)


def test_errors_surface_as_exceptions(cuda):
    z = torch.zeros((9, 16), device=cuda)
    with pytest.raises(ValueError):
        P.polsar_inv_det(z, torch.zeros((11, 8), device=cuda))      # ld mismatch
    with pytest.raises(TypeError):
        P.polsar_inv_det(z, torch.zeros((11, 16), device=cuda, dtype=torch.float64))
    with pytest.raises(P.PolsarError):
        P.polsar_inv_det_blocks(torch.zeros((0, 16), device=cuda), torch.zeros((2, 16), device=cuda), 0)
    # n = 0 is a successful no-op
    P.polsar_inv_det(z, torch.zeros((11, 16), device=cuda), n=0)
