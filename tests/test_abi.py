"""Host-side checks of the C-ABI (no GPU needed): the libraries build for
sm_100a, load, export every symbol the headers declare, and validate
arguments synchronously (EINVAL paths never touch the device)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_1807_08084_b200 import _build, _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\*\s]+?\b(polsar_\w+)\s*\(", src, flags=re.M))
                  - {"polsar_gen_threshold"})


def exported(so):
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True,
                         check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def test_libpolsar_exports_every_declared_symbol():
    so = _build.build_target("libpolsar")
    syms = exported(so)
    names = declared("polsar.h")
    assert set(_lib.SIGNATURES) == set(names)
    for name in names:
        assert name in syms, name


def test_generator_exports():
    gpu = exported(_build.build_target("libpolsar_gen"))
    cpu = exported(_build.build_target("libpolsar_gen_cpu"))
    names = declared("polsar_gen.h")
    assert "polsar_gen_wishart" in names
    assert "polsar_gen_wishart" in gpu
    assert {"polsar_gen_wishart_cpu", "polsar_gen_wishart_pixels_cpu"} <= cpu


def test_sm100a_cubin_only():
    so = _build.build_target("libpolsar")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_loads_and_validates_without_gpu():
    lib = _lib.lib()
    assert lib.polsar_version() >= 0x000100
    # argument errors are reported synchronously, before any CUDA call
    assert lib.polsar_inv_det(None, None, None, -1, 0, 0, None) == 1
    assert lib.polsar_inv_det(None, None, None, 10, 5, 0, None) == 1
    assert b"ld" in lib.polsar_last_error()
    assert lib.polsar_inv_det(None, None, None, 0, 0, 0, None) == 0  # n == 0 no-op
    assert lib.polsar_inv_det_cholesky(None, None, None, 4, 4, 9, None) == 1
    # POLSAR_F64_EFT (4) is an Alg. 2 mode: Alg. 1 and the window family refuse it
    # before any CUDA call
    dummy = ctypes.c_void_p(16)
    assert lib.polsar_inv_det_cholesky(dummy, dummy, None, 4, 4, 4, None) == 3
    assert b"Alg. 2" in lib.polsar_last_error()
    assert lib.polsar_inv_det(dummy, dummy, None, 4, 4, 5, None) == 1  # unknown dtype
    assert lib.polsar_window_distance(None, 0, 4, 4, 0, 5, 11, 4.0, 1.0, None, None, 0, None) == 1
    assert lib.polsar_window_distance(None, 16, 4, 4, 0, 4, 17, 4.0, 1.0, None, None, 0, None) == 1
    assert lib.polsar_window_distance(None, 16, 4, 4, 0, 4, 3, 0.0, 1.0, None, None, 0, None) == 1
    big = 1 << 31  # slab_rows * width = 2^62 > 2^40: refused before any size arithmetic
    assert lib.polsar_window_distance(None, 1 << 62, big, big, 0, 1, 11, 4.0, 1.0, None, None, 0, None) == 1
    assert b"2^40" in lib.polsar_last_error()
    assert lib.polsar_window_kl(None, 1 << 62, big, big, 0, 1, 11, 4.0, 1.0, None, None, 0, None) == 1
    assert lib.polsar_nlm_filter(None, 1 << 62, big, big, 0, 1, 11, 4.0, 1.0, None, None, None, 1 << 31,
                                 0, None) == 1
    assert lib.polsar_window_workspace_bytes(big, big, 11, 0) == 0
    assert lib.polsar_checksum(None, 5, 2, 1, 0, 0, None, None, None) == 1
    assert lib.polsar_inv_det_host(None, None, None, 5, 5, 0, 0, None, 0, None, None, None) == 1
    # c5: the NLM's weight planes over one 1024-row band (+ 2R halo rows), not the image
    assert lib.polsar_window_workspace_bytes(2048, 2048, 11, 0) >= 1046 * 2048 * (4 + 8 + 264 * 4)
    assert lib.polsar_window_workspace_bytes(2048, 2048, 11, 0) < 2048 * 2048 * (264 * 4)
    assert lib.polsar_host_chunk_pixels(3 << 30, 0) % 64 == 0


def test_binding_refuses_cpu_tensors():
    torch = pytest.importorskip("torch")
    import paper_1807_08084_b200 as P
    z = torch.zeros((9, 4))
    with pytest.raises(P.PolsarError):
        P.polsar_inv_det(z, torch.zeros((11, 4)))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1807_08084_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".c", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, flags=re.M), f
                assert not re.search(r'#include\s+[<"][^>"]*oracle', txt), f
                assert "liboracle" not in txt, f


@pytest.mark.parametrize("rows,width,radius", [(1, 1, 11), (1, 50, 4), (5, 300, 12), (130, 7, 1),
                                               (2048, 2048, 11), (37, 53, 3), (3, 3, 0)])
def test_window_workspace_covers_every_form(rows, width, radius):
    """polsar_window_workspace_bytes_for(entry) is the need of the form that
    entry point runs for (dtype, R) -- fixed at compile time, no environment
    switches: the tiles' backward sums of the shared-memory
    forms (32-column tiles of 32 rows, 16 for fp64 KL, 8 for the tensor-core
    pass 1, each (32 + 2R)(TY + R) int64) after the prepass planes; the weight
    planes (pitch rounded to 16 bytes) where the shared-memory form does not
    fit and for the NLM, whose planes cover one band of 512 output rows;
    polsar_window_workspace_bytes >= all of them."""
    lib = _lib.lib()
    up = lambda b: (b + 255) // 256 * 256  # noqa: E731
    n = rows * width
    for dtype, wt in ((0, 4), (1, 8), (2, 4), (3, 8)):
        pitch = (width + 16 // wt - 1) // (16 // wt) * (16 // wt)

        def planes(pre, r_rows):
            m = r_rows * width
            return up(pre) + up(m * 8) + up(2 * radius * (radius + 1) * r_rows * pitch * wt)

        def acc(pre, ty):
            tiles = ((width + 31) // 32) * ((rows + ty - 1) // ty)
            return up(pre) + up(n * 8) + up(tiles * (32 + 2 * radius) * (ty + radius) * 8)
        sym = radius <= 12
        rows_b = min(rows, 1024 + 2 * radius)
        expect = {}
        if not sym:
            expect[0] = [up(n * wt)]
        elif dtype == 0:  # fp32 storage: the tensor-core pass 1 (8-row tiles, no prepass)
            expect[0] = [acc(0, 8)]
        else:
            expect[0] = [acc(n * wt, 32), planes(n * wt, rows)]
        expect[1] = [planes(rows_b * width * wt, rows_b)] if 1 <= radius <= 12 else [up(n * wt)]
        if not sym or dtype == 2:
            expect[2] = [0]
        else:  # the KL window runs the tensor-core pass 1 for both storage precisions
            expect[2] = [acc(0, 8)]
        for e in range(3):
            got = lib.polsar_window_workspace_bytes_for(e, rows, width, radius, dtype)
            assert got in expect[e], (e, dtype, got, expect[e])
            assert lib.polsar_window_workspace_bytes(rows, width, radius, dtype) >= got
        if dtype == 0 and rows * width > 1000 and radius >= 8:  # the window sum needs far less than the NLM
            assert 4 * lib.polsar_window_workspace_bytes_for(0, rows, width, radius, dtype) < expect[1][0]
        # POLSAR_F64_EFT (an inverse/det mode) has no window form
        assert lib.polsar_window_workspace_bytes_for(0, rows, width, radius, 4) == 0


def test_product_reads_no_environment():
    """every kernel form of libpolsar.so is fixed at compile
    time (A/B alternatives are -D builds); its sources never read the
    environment.  (The statically linked CUDA runtime itself still imports
    getenv, for CUDA_VISIBLE_DEVICES and the like.)"""
    csrc = os.path.join(ROOT, "paper_1807_08084_b200", "csrc")
    for f in os.listdir(csrc):
        txt = open(os.path.join(csrc, f)).read()
        assert not re.search(r"\bgetenv\s*\(|\benviron\b|secure_getenv", txt), f
