"""C-ABI library checks that need no GPU: the library builds/loads, exports every
symbol include/b200conv.h declares, validates arguments before touching the
device, and plans one launch per call.  (`-m "not gpu"`.)"""
import ctypes
import os
import re

import pytest
import torch

from paper_2212_00404_b200 import conv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "b200conv.h")


def header_symbols():
    src = open(HEADER).read()
    return re.findall(r"B200CONV_API\s+[\w\s\*]*?\b(conv_\w+)\s*\(", src)


def test_library_exports_every_header_symbol():
    lib = conv.load()
    syms = header_symbols()
    assert len(syms) == 21
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(conv.EXPORTS)
    assert conv.version() == (1 << 16) | 6


def test_status_strings():
    lib = conv.load()
    for st in range(7):
        assert lib.conv_status_string(st)
    assert b"unknown" in lib.conv_status_string(99)


BAD_SHAPES = [  # (C, Wx, Wy, K, M)
    (0, 8, 8, 3, 4), (1, 0, 8, 3, 4), (1, 8, 0, 3, 4), (1, 8, 8, 0, 4), (1, 8, 8, 3, 0),
    (1, 8, 8, 9, 4), (1, 2, 8, 3, 4), (1, 8, 2, 3, 4), (-1, 8, 8, 3, 4),
    (70000, 200, 200, 3, 4),      # C*Wx*Wy overflows int32
]


@pytest.mark.parametrize("C,Wx,Wy,K,M", BAD_SHAPES)
def test_shape_errors_before_any_device_access(C, Wx, Wy, K, M):
    lib = conv.load()
    fake = 0x1000  # never dereferenced: validation rejects first
    assert lib.conv_multi_ex(fake, C, Wx, Wy, fake, K, M, fake, 0, None) == 1
    assert lib.conv_multi(fake, C, Wx, Wy, fake, K, M, fake) == 1
    if C == 1:
        assert lib.conv_single_ex(fake, Wx, Wy, fake, K, M, fake, None) == 1
    p = conv.ConvPlan()
    assert lib.conv_plan_multi(C, Wx, Wy, K, M, 1, ctypes.byref(p)) == 1


def test_null_align_precision_errors():
    lib = conv.load()
    f = 0x1000
    assert lib.conv_single_ex(None, 8, 8, f, 3, 4, f, None) == 2
    assert lib.conv_multi_ex(f, 2, 8, 8, None, 3, 4, f, 1, None) == 2
    assert lib.conv_multi_ex(f, 2, 8, 8, f, 3, 4, None, 1, None) == 2
    assert lib.conv_single_ex(f + 2, 8, 8, f, 3, 4, f, None) == 3          # f32 needs 4-B alignment
    assert lib.conv_multi_ex(f, 2, 8, 8, f + 2, 3, 4, f, 2, None) != 3     # bf16: 2-B is enough
    assert lib.conv_multi_ex(f, 2, 8, 8, f + 1, 3, 4, f, 2, None) == 3
    assert lib.conv_multi_ex(f, 2, 8, 8, f, 3, 4, f, 7, None) == 4
    assert lib.conv_multi_ex(f, 2, 8, 8, f, 3, 4, f, -1, None) == 4
    p = conv.ConvPlan()
    assert lib.conv_plan_multi(2, 8, 8, 3, 4, 9, ctypes.byref(p)) == 4
    assert lib.conv_plan_multi(2, 8, 8, 3, 4, 1, None) == 2


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device path")
def test_no_device_is_reported_not_faked():
    lib = conv.load()
    f = 0x1000
    assert lib.conv_single_ex(f, 8, 8, f, 3, 4, f, None) == 5
    assert lib.conv_multi_ex(f, 2, 8, 8, f, 3, 4, f, 1, None) == 5
    with pytest.raises(conv.ConvError):
        conv.conv_single(f, 8, 8, f, 3, 4, f)


def test_plans_cover_every_config_with_one_launch():
    import synth
    for cfg in synth.SINGLE_SWEEP + [synth.PR1]:
        p = conv.plan_single(cfg["Wx"], cfg["Wy"], cfg["K"], cfg["M"])
        assert p["kernel"] == 0 and p["grid_x"] * p["grid_y"] * p["grid_z"] >= 1
        Ho, Wo = cfg["Wy"] - cfg["K"] + 1, cfg["Wx"] - cfg["K"] + 1
        if p["tile_n"] == -2:
            # KS-L (large K = 3 maps whose output rows are not whole 128-B lines):
            # 64-float flat chunks of 8 (or 4) filter planes P apart, one wave of 2 (3) CTAs/SM
            assert cfg["K"] == 3 and Wo % 32 != 0 and Wo % 2 == 0 and p["tile_m"] in (4, 8)
            assert 1 <= p["grid_x"] <= 3 * 148 and p["smem_bytes"] <= 110 * 1024
            continue
        assert p["tile_n"] > 0, "every other BASELINE single-channel config uses the band kernel"
        # tasks = (row block of tile_n full-width rows) x (group of tile_m filters),
        # dealt to at most one wave of 3 CTAs per SM, at most one 32-slot segment per warp
        assert p["grid_y"] == p["grid_z"] == 1 and 1 <= p["grid_x"] <= 3 * 148
        tasks = -(-Ho // p["tile_n"]) * -(-cfg["M"] // p["tile_m"])
        assert p["grid_x"] <= tasks * -(-(p["tile_n"] * Wo) // 32)          # >= 1 unit per CTA
        assert p["smem_bytes"] <= 227 * 1024
    for cfg in synth.MULTI_LAYERS + [synth.SHARD_SWEEP]:
        for prec, kern in (("fp32", (1,)), ("tf32", (2, 3)), ("bf16", (2, 3))):
            p = conv.plan_multi(cfg["C"], cfg["Wx"], cfg["Wy"], cfg["K"], cfg["M"], prec)
            if cfg["C"] == 3 and cfg["K"] in (3, 5):
                # RGB stem: the channel-summing KS variant, every precision
                assert p["kernel"] == 4 and p["launches"] == 1 and p["cluster_x"] == 1
                continue
            assert p["kernel"] in kern
            assert 1 <= p["cluster_x"] <= 16 and p["launches"] in (1, 2)
            if p["kernel"] == 3:
                # im2col kernel + GEMM; k split reduced inside a cluster
                assert p["launches"] == 2 and p["grid_x"] == p["cluster_x"] and p["tma_f"] & 5 == 5
                aligned = (cfg["C"] * cfg["K"] ** 2 * (2 if prec == "bf16" else 4)) % 16 == 0
                assert aligned, "KM-TC/G needs TMA-able filter rows"
                continue
            if p["launches"] == 1:
                assert p["grid_x"] == p["cluster_x"]           # split reduced inside a cluster
            else:
                assert p["cluster_x"] == 1 and p["grid_x"] > 1  # split reduced via the workspace
            assert p["smem_bytes"] <= 227 * 1024
            Ho, Wo = cfg["Wy"] - cfg["K"] + 1, cfg["Wx"] - cfg["K"] + 1
            px = Ho * (Wo if prec == "fp32" else cfg["Wx"])        # compact (SIMT) / wide (TC)
            assert p["grid_y"] * p["tile_n"] >= px
            assert p["grid_z"] * p["tile_m"] >= cfg["M"]
            if prec != "fp32":
                aligned = (cfg["C"] * cfg["K"] ** 2 * (2 if prec == "bf16" else 4)) % 16 == 0
                assert (p["tma_f"] & 1) == int(aligned)        # bit 0: F tiles by TMA
                assert p["tma_f"] & 2                            # bit 1: I patch by TMA


def test_batched_plans():
    # one launch over all N images: N times the pixel tiles, no split once N fills the SMs
    for prec in ("tf32", "bf16"):
        p1 = conv.plan_multi_batched(1, 256, 28, 28, 3, 256, prec)
        p32 = conv.plan_multi_batched(32, 256, 28, 28, 3, 256, prec)
        assert p32["kernel"] == 2 and p32["launches"] == 1
        if p32["tma_f"] & 32:            # persistent CTAs: one per SM walks the 32 x 6 tiles
            # 8 gather + 2 producer + 1 MMA warps, two epilogue groups of 4 warps
            assert p32["grid_y"] == 148 and p32["block_x"] == 32 * (11 + 8)
        else:
            assert p32["grid_y"] == 32 * (-(-26 * 28 // 128))
        assert p32["cluster_x"] == 1 and p1["kernel"] in (2, 3)
    assert conv.plan_multi_batched(4, 16, 14, 14, 3, 32, "fp32")["kernel"] == 1
    lib = conv.load()
    f = 0x1000
    assert lib.conv_multi_batched_ex(f, 0, 2, 8, 8, f, 3, 4, f, 1, None) == 1      # N < 1
    assert lib.conv_multi_batched_ex(f, 1 << 20, 64, 64, 64, f, 3, 4, f, 1, None) == 1  # overflow


def test_padded_argument_errors():
    lib = conv.load()
    f = 0x1000
    assert lib.conv_multi_pad_ex(f, 1, 2, 8, 8, f, 3, 4, -1, f, 1, None) == 1        # pad < 0
    assert lib.conv_multi_pad_ex(f, 0, 2, 8, 8, f, 3, 4, 1, f, 1, None) == 1         # N < 1
    assert lib.conv_multi_pad_ex(f, 1, 2, 2, 2, f, 7, 4, 1, f, 1, None) == 1         # K > padded map
    assert lib.conv_single_pad_ex(f, 8, 8, f, 3, 4, -2, f, None) == 1
    assert lib.conv_single_pad_ex(0, 8, 8, f, 3, 4, 1, f, None) == 2                  # null
    assert lib.conv_multi_pad_ex(f, 1, 2, 8, 8, f, 3, 4, 1, f, 9, None) == 4         # precision


def test_strided_argument_errors_and_plans():
    lib = conv.load()
    f = 0x1000
    assert lib.conv_multi_strided_ex(f, 1, 2, 8, 8, f, 3, 4, 0, 0, f, 1, None) == 1      # stride < 1
    assert lib.conv_multi_strided_ex(f, 1, 2, 8, 8, f, 3, 4, -1, 2, f, 1, None) == 1     # pad < 0
    assert lib.conv_multi_strided_ex(f, 0, 2, 8, 8, f, 3, 4, 0, 2, f, 1, None) == 1      # N < 1
    assert lib.conv_multi_strided_ex(f, 1, 2, 2, 2, f, 7, 4, 1, 2, f, 1, None) == 1      # K > padded map
    assert lib.conv_single_strided_ex(0, 8, 8, f, 3, 4, 0, 2, f, None) == 2               # null
    assert lib.conv_multi_strided_ex(f, 1, 2, 8, 8, f, 3, 4, 0, 2, f, 9, None) == 4      # precision
    # stride 1 is the padded / unpadded plan; stride > 1 goes to KM-SIMT (fp32) / KM-TC/G (tf32, bf16)
    assert conv.plan_multi_strided(64, 28, 28, 3, 64, 1, 1, "tf32") == conv.plan_multi(64, 30, 30, 3, 64, "tf32")
    for prec, kern in (("fp32", 1), ("tf32", 3), ("bf16", 3)):
        for (C, W, K, M, pad, s) in [(64, 56, 3, 128, 1, 2), (3, 224, 7, 64, 3, 2), (256, 14, 1, 512, 0, 2)]:
            p = conv.plan_multi_strided(C, W, W, K, M, pad, s, prec)
            assert p["kernel"] == kern, (prec, C, W, K, M, pad, s, p)
            Ho = (W + 2 * pad - K) // s + 1
            if kern == 1:
                assert p["grid_y"] * p["tile_n"] >= Ho * Ho        # compact pixel tiles cover the strided map


def test_strided_output_overflow_is_a_shape_error_before_any_device_work():
    lib = conv.load()
    f = 0x1000
    # N*C*Wx*Wy = 2^30 fits, N*M*Ho*Wo = 2^42 does not: rejected before the pad pre-pass
    assert lib.conv_multi_strided_ex(f, 1 << 14, 1, 256, 256, f, 1, 1 << 14, 1, 2, f, 0, None) == 1


@pytest.mark.parametrize("call", [
    lambda: conv.single(torch.zeros(8, 8), torch.zeros(2, 3, 3)),                                 # CPU tensors
    lambda: conv.multi_host(torch.zeros(3, 8, 8), torch.zeros(4, 2, 3, 3)),                       # channels
    lambda: conv.multi_host(torch.zeros(3, 8, 8).bfloat16(), torch.zeros(4, 3, 3, 3).bfloat16()),  # dtype vs fp32
    lambda: conv.single_host(torch.zeros(8, 8, dtype=torch.float64), torch.zeros(2, 3, 3)),       # dtype
    lambda: conv.single_host(torch.zeros(8, 16)[:, ::2], torch.zeros(2, 3, 3)),                   # non-contiguous
    lambda: conv.multi_host(torch.zeros(3, 8, 8), torch.zeros(4, 3, 3, 3), out=torch.zeros(4, 6, 5)),  # out shape
    lambda: conv.single_host(torch.zeros(8, 8), torch.zeros(2, 3, 2)),                            # non-square F
    lambda: conv.single_host(torch.zeros(4, 4), torch.zeros(2, 5, 5)),                            # K > map
])
def test_python_conveniences_validate_before_the_abi(call):
    with pytest.raises((ValueError, TypeError)):
        call()


def test_verify_cli_usage_and_infeasible_exit_codes():
    import subprocess
    import sys
    v = os.path.join(ROOT, "tests", "verify.py")
    run = lambda *a: subprocess.run([sys.executable, v, *a], capture_output=True, text=True).returncode
    assert run("--mode", "multi") == 1                                                  # usage
    assert run("--mode", "single", "--wx", "8", "--wy", "8", "--k", "3", "--m", "2", "--c", "3") == 1
    assert run("--mode", "multi", "--wx", "4", "--wy", "4", "--c", "2", "--k", "5", "--m", "2") == 2
    assert run("--help") == 0


def test_latency_model_reproduces_the_papers_table1_numbers():
    """PAPER.md §2.2: GTX 1080Ti, 258-clock latency, 128 cores x 2
    FMA per clock -> N_FMA = 66,048; 327 B/clk x 258 = 84,366 bytes; 768
    threads per SM fetching one 4-B word; V_s = 768 x 4 x 28 = 86,016."""
    m = conv.latency_model("gtx1080ti")
    assert m["n_fma"] == 66048 and m["volume"] == 84366
    assert m["threads_per_sm"] == 768 and m["v_s"] == 86016 and m["bytes_per_clk"] == 327


def test_latency_model_b200_profile():
    m = conv.latency_model("b200")
    assert m["n_fma"] == 577 * 128                        # 1 FMA per lane per clock (reading Q15)
    assert abs(m["bytes_per_clk"] - 6554e9 / 1965e6) < 1e-6
    assert m["threads_per_sm"] % 128 == 0 and m["v_s"] >= m["volume"]
    assert conv.load().conv_latency_model(7, (ctypes.c_double * 5)()) == 1        # unknown profile
    assert conv.load().conv_latency_model(0, None) == 2                           # null


def test_allgather_argument_errors_before_device_access():
    lib = conv.load()
    f = 0x1000
    peers = (ctypes.c_void_p * 2)(f, f)
    A = lib.conv_multi_allgather_ex
    assert A(f, 4, 8, 8, f, 3, 4, -1, 8, peers, 2, None, 0, None) == 1          # m0 < 0
    assert A(f, 4, 8, 8, f, 3, 4, 6, 8, peers, 2, None, 0, None) == 1           # m0 + M > M_total
    assert A(f, 4, 8, 8, f, 3, 4, 0, 8, peers, 0, None, 0, None) == 1           # no destination
    assert A(f, 4, 8, 8, f, 3, 4, 0, 8, peers, 9, None, 0, None) == 1           # > 8 destinations
    assert A(f, 4, 8, 8, f, 3, 4, 0, 8, None, 2, None, 0, None) == 2            # null peer array
    assert A(f, 4, 8, 8, f, 3, 4, 0, 8, (ctypes.c_void_p * 2)(f, 0), 2, None, 0, None) == 2
    assert A(f, 4, 8, 8, f, 3, 4, 0, 8, peers, 2, None, 5, None) == 4           # precision
