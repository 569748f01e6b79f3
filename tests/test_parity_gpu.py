"""Parity of the CUDA path (through the C ABI) with the fp64 CPU oracle, element
by element, on identical seeded inputs (synth.py).  `-m gpu`.

Acceptance per output (north_star):
    |O_gpu - O_oracle| <= tau * A,   A = sum |I*F| (oracle, on the fp32 inputs)
    tau = 1e-5 (FP32: KS, KM-SIMT), 2e-3 (TF32, KM-TC), 1e-2 (BF16, KM-TC)
and O_gpu == 0 wherever A == 0.  On small-integer inputs every path is
bit-exact (pin P10).  Full BASELINE sizes run in the same launch configuration
bench.py times (same entry points, same plans)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

TAU = {"fp32": 1e-5, "tf32": 2e-3, "bf16": 1e-2}


@pytest.fixture(scope="module")
def conv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2212_00404_b200 import conv as c
    c.load()
    return c


def run_single(conv, I, F):
    Id = torch.from_numpy(I).cuda()
    Fd = torch.from_numpy(F).cuda()
    O = conv.single(Id, Fd)
    torch.cuda.synchronize()
    return O.cpu().numpy().astype(np.float64)


def run_multi(conv, I, F, prec):
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    Id = torch.from_numpy(I).cuda().to(dt)
    Fd = torch.from_numpy(F).cuda().to(dt)
    O = conv.multi(Id, Fd, prec)
    torch.cuda.synchronize()
    return O.cpu().numpy().astype(np.float64)


def assert_parity(Og, Oo, A, tau, what=""):
    assert Og.shape == Oo.shape, (what, Og.shape, Oo.shape)
    err = np.abs(Og - Oo)
    bad = err > tau * A
    if bad.any():
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {bad.sum()} / {bad.size} outputs out of tolerance; first at "
                             f"{tuple(i)}: gpu={Og[tuple(i)]!r} oracle={Oo[tuple(i)]!r} "
                             f"A={A[tuple(i)]!r} max err/A={float((err / np.maximum(A, 1e-300)).max()):.3g}")
    zero = A == 0
    assert np.all(Og[zero] == 0), what
    return float((err / np.where(A > 0, A, 1)).max())


# ------------------------------------------------------------------ single-channel (KS)
def test_pr1_single(conv):
    c = synth.PR1
    I, F = synth.layer_inputs(1, c["Wx"], c["Wy"], c["K"], c["M"])
    Oo, A = oracle.conv_single(I[0], F[:, 0])
    Og = run_single(conv, I[0], F[:, 0])
    assert_parity(Og, Oo, A, TAU["fp32"], "PR1")


def test_golden_through_gpu(conv):
    from conftest import load_golden
    for name in ("p1_single_handworked.txt", "p2_orientation_delta.txt"):
        g = load_golden(name)
        Og = run_single(conv, g["I"][0].astype(np.float32), g["F"][:, 0].astype(np.float32))
        assert np.array_equal(Og, g["O"]), name
    g = load_golden("p3_multi_handworked.txt")
    for prec in ("fp32", "tf32", "bf16"):
        Og = run_multi(conv, g["I"].astype(np.float32), g["F"].astype(np.float32), prec)
        assert np.array_equal(Og, g["O"]), prec


@pytest.mark.parametrize("idx", range(len(synth.SINGLE_SWEEP)))
def test_single_sweep_full_size(conv, idx):
    c = synth.SINGLE_SWEEP[idx]
    I, F = synth.layer_inputs(1, c["Wx"], c["Wy"], c["K"], c["M"], cfg_index=idx)
    Oo, A = oracle.conv_single(I[0], F[:, 0])
    Og = run_single(conv, I[0], F[:, 0])
    assert_parity(Og, Oo, A, TAU["fp32"], c["name"])


SINGLE_EDGE = [  # (Wx, Wy, K, M): ragged, degenerate, generic-K, large maps
    (5, 5, 5, 3), (1, 1, 1, 1), (9, 4, 4, 7), (300, 17, 3, 5), (33, 65, 2, 9), (20, 20, 11, 6),
    (13, 13, 13, 2), (1000, 3, 3, 3), (64, 64, 6, 33), (257, 9, 1, 17),
]


@pytest.mark.parametrize("Wx,Wy,K,M", SINGLE_EDGE)
def test_single_edge_cases(conv, Wx, Wy, K, M):
    I = synth.uniform01(21, (Wy, Wx))
    F = synth.uniform_pm1(22, (M, K, K))
    Oo, A = oracle.conv_single(I, F)
    assert_parity(run_single(conv, I, F), Oo, A, TAU["fp32"], f"single {Wx}x{Wy} K{K} M{M}")


# KS-L (line-aligned flat chunks, conv_single.cu): forced on shapes covering
# every plane alignment period P (1, 2, 4, 8, 16), filter counts that leave
# groups partly empty, tiny and ragged maps
KSL_SHAPES = [(10, 10, 4), (12, 9, 7), (34, 20, 33), (30, 30, 48), (58, 45, 20), (100, 37, 70),
              (224, 224, 12), (66, 130, 9), (14, 14, 32), (16, 16, 64), (40, 200, 130)]


@pytest.mark.parametrize("Wx,Wy,M", KSL_SHAPES)
def test_single_ksl_forced_matches_oracle(conv, monkeypatch, Wx, Wy, M):
    monkeypatch.setenv("B200CONV_KS_FLAT", "1")
    assert conv.plan_single(Wx, Wy, 3, M)["tile_n"] == -2
    I = synth.uniform01(31, (Wy, Wx))
    F = synth.uniform_pm1(32, (M, 3, 3))
    Oo, A = oracle.conv_single(I, F)
    assert_parity(run_single(conv, I, F), Oo, A, TAU["fp32"], f"KS-L {Wx}x{Wy} M{M}")
    Ii, Fi = synth.layer_inputs(1, Wx, Wy, 3, M, kind="ints")
    Oi, _ = oracle.conv_single(Ii[0], Fi[:, 0])
    assert np.array_equal(run_single(conv, Ii[0], Fi[:, 0]), Oi)


# KS with 8-B window loads (TX = 4 lanes on rows that are only 8-B strided:
# Wx = 2 mod 4), K = 1 / 4 / 5 / 7, incl. the large-map row blocks
@pytest.mark.parametrize("Wx,Wy,K,M", [(230, 230, 7, 4), (62, 66, 5, 8), (130, 40, 5, 3), (30, 30, 1, 8),
                                       (226, 100, 1, 16), (54, 70, 4, 5)])
def test_single_8b_window_loads(conv, Wx, Wy, K, M):
    I = synth.uniform01(41, (Wy, Wx))
    F = synth.uniform_pm1(42, (M, K, K))
    Oo, A = oracle.conv_single(I, F)
    assert_parity(run_single(conv, I, F), Oo, A, TAU["fp32"], f"single {Wx}x{Wy} K{K} M{M}")


def test_single_positive_stress_and_ints(conv):
    I, F = synth.layer_inputs(1, 56, 56, 7, 32, kind="positive")
    Oo, A = oracle.conv_single(I[0], F[:, 0])
    assert_parity(run_single(conv, I[0], F[:, 0]), Oo, A, TAU["fp32"], "positive")
    I, F = synth.layer_inputs(1, 56, 56, 5, 32, kind="ints")
    Oo, _ = oracle.conv_single(I[0], F[:, 0])
    assert np.array_equal(run_single(conv, I[0], F[:, 0]), Oo)


# ------------------------------------------------------------------ multi-channel
MULTI = synth.MULTI_LAYERS


@pytest.fixture(scope="module")
def multi_oracle():
    cache = {}

    def get(i, kind="default"):
        key = (i, kind)
        if key not in cache:
            c = MULTI[i]
            I, F = synth.layer_inputs(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], cfg_index=100 + i,
                                      kind=kind)
            Oo, A = oracle.conv_multi(I, F)
            cache[key] = (I, F, Oo, A)
        return cache[key]
    return get


@pytest.mark.parametrize("prec", ["fp32", "tf32", "bf16"])
@pytest.mark.parametrize("i", range(len(MULTI)))
def test_multi_layers_full_size(conv, multi_oracle, i, prec):
    I, F, Oo, A = multi_oracle(i)
    Og = run_multi(conv, I, F, prec)
    assert_parity(Og, Oo, A, TAU[prec], f"{MULTI[i]['name']} {prec}")


@pytest.mark.parametrize("prec", ["fp32", "tf32", "bf16"])
def test_multi_integer_inputs_bit_exact(conv, prec):
    for (C, W, K, M) in [(64, 14, 3, 96), (3, 40, 3, 64), (96, 27, 5, 40), (512, 7, 3, 64)]:
        I, F = synth.layer_inputs(C, W, W, K, M, kind="ints")
        Oo, _ = oracle.conv_multi(I, F)
        Og = run_multi(conv, I, F, prec)
        assert np.array_equal(Og, Oo), (C, W, K, M, prec)


@pytest.mark.parametrize("prec", ["fp32", "tf32", "bf16"])
def test_multi_positive_stress(conv, prec):
    I, F = synth.layer_inputs(256, 14, 14, 3, 64, kind="positive")
    Oo, A = oracle.conv_multi(I, F)
    assert_parity(run_multi(conv, I, F, prec), Oo, A, TAU[prec], f"positive {prec}")


MULTI_EDGE = [  # (C, Wx, Wy, K, M): ragged tiles, odd K*K*C, tiny/degenerate, generic K
    (1, 9, 9, 3, 5), (2, 5, 7, 5, 3), (5, 17, 11, 3, 37), (3, 30, 30, 1, 130), (7, 6, 6, 6, 9),
    (16, 33, 19, 2, 200), (9, 12, 12, 4, 70), (130, 9, 9, 3, 33), (4, 20, 20, 9, 16),
    (1, 1, 1, 1, 1), (33, 3, 3, 3, 257),
]


@pytest.mark.parametrize("prec", ["fp32", "tf32", "bf16"])
@pytest.mark.parametrize("C,Wx,Wy,K,M", MULTI_EDGE)
def test_multi_edge_cases(conv, prec, C, Wx, Wy, K, M):
    I = synth.uniform01(31, (C, Wy, Wx))
    F = synth.uniform_pm1(32, (M, C, K, K))
    Oo, A = oracle.conv_multi(I, F)
    assert_parity(run_multi(conv, I, F, prec), Oo, A, TAU[prec], f"edge {C},{Wx},{Wy},{K},{M} {prec}")


def test_shard_sweep_sampled_full_size(conv):
    """BASELINE configs[4] (14x14 C=512 M=4096 K=3) at full size, sampled outputs."""
    c = synth.SHARD_SWEEP
    I, F = synth.layer_inputs(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], cfg_index=200)
    rng = np.random.default_rng(0)
    Ho = c["Wy"] - c["K"] + 1
    n = c["M"] * Ho * (c["Wx"] - c["K"] + 1)
    idx = np.unique(np.concatenate([rng.integers(0, n, 4000), np.arange(200), np.arange(n - 200, n)]))
    Oo, A = oracle.conv_multi_sampled(I, F, idx)
    for prec in ("fp32", "tf32", "bf16"):
        Og = run_multi(conv, I, F, prec).ravel()[idx]
        assert_parity(Og, Oo, A, TAU[prec], f"shard sweep {prec}")


def test_multi_c1_equals_single_and_determinism(conv):
    I = synth.uniform01(41, (1, 28, 28))
    F = synth.uniform_pm1(42, (16, 1, 3, 3))
    a = run_multi(conv, I, F, "fp32")
    b = run_multi(conv, I, F, "fp32")
    assert np.array_equal(a, b)
    s = run_single(conv, I[0], F[:, 0])
    Oo, A = oracle.conv_single(I[0], F[:, 0])
    assert_parity(a, Oo, A, TAU["fp32"])
    assert_parity(s, Oo, A, TAU["fp32"])
    for prec in ("tf32", "bf16"):
        c = synth.MULTI_LAYERS[6]
        I, F = synth.layer_inputs(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], cfg_index=7)
        assert np.array_equal(run_multi(conv, I, F, prec), run_multi(conv, I, F, prec))


def test_filter_shards_concatenate(conv):
    """Filter-index sharding: F/O slices are contiguous sub-ranges."""
    c = synth.MULTI_LAYERS[1]
    I, F = synth.layer_inputs(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], cfg_index=3)
    Oo, A = oracle.conv_multi(I, F)
    for prec in ("fp32", "tf32", "bf16"):
        parts = [run_multi(conv, I, np.ascontiguousarray(F[a:a + 64]), prec) for a in range(0, c["M"], 64)]
        assert_parity(np.concatenate(parts), Oo, A, TAU[prec], f"shards {prec}")


def test_host_entry_points(conv):
    c = synth.MULTI_LAYERS[0]
    I, F = synth.layer_inputs(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], cfg_index=5)
    Oo, A = oracle.conv_multi(I, F)
    for prec in ("fp32", "tf32"):
        Og = conv.multi_host(torch.from_numpy(I), torch.from_numpy(F), prec).numpy().astype(np.float64)
        assert_parity(Og, Oo, A, TAU[prec], f"host {prec}")
    Og = conv.multi_host(torch.from_numpy(I).bfloat16(), torch.from_numpy(F).bfloat16(), "bf16")
    assert_parity(Og.numpy().astype(np.float64), Oo, A, TAU["bf16"], "host bf16")
    I1, F1 = synth.layer_inputs(1, 56, 56, 3, 64)
    Oo, A = oracle.conv_single(I1[0], F1[:, 0])
    Og = conv.single_host(torch.from_numpy(I1[0]), torch.from_numpy(F1[:, 0])).numpy().astype(np.float64)
    assert_parity(Og, Oo, A, TAU["fp32"], "host single")


def test_host_async_entry_points_two_streams(conv):
    # several calls in flight on two streams, pinned host buffers, one sync at the end
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    cases = []
    for i, (C, W, K, M, prec) in enumerate([(64, 14, 3, 96, "fp32"), (1, 56, 3, 64, "single"),
                                             (32, 28, 3, 128, "bf16"), (512, 7, 3, 512, "tf32"),
                                             (3, 40, 5, 70, "tf32"), (1, 224, 1, 32, "single")]):
        I, F = synth.layer_inputs(C, W, W, K, M, cfg_index=40 + i)
        Oo, A = oracle.conv_multi(I, F)
        dt = torch.bfloat16 if prec == "bf16" else torch.float32
        Ih = torch.from_numpy(I[0] if prec == "single" else I).to(dt).pin_memory()
        Fh = torch.from_numpy(F[:, 0] if prec == "single" else F).to(dt).pin_memory()
        Oh = torch.full((M, W - K + 1, W - K + 1), float("nan")).pin_memory()
        sh = streams[i & 1].cuda_stream
        if prec == "single":
            conv.conv_single_host_async(Ih, W, W, Fh, K, M, Oh, sh)
        else:
            conv.conv_multi_host_async(Ih, C, W, W, Fh, K, M, Oh, prec, sh)
        cases.append((Oh, Oo, A, "fp32" if prec == "single" else prec))
    for st in streams:
        st.synchronize()
    for Oh, Oo, A, prec in cases:
        assert_parity(Oh.numpy().astype(np.float64), Oo, A, TAU[prec], f"host async {prec}")


def test_output_untouched_on_argument_error(conv):
    O = torch.full((4, 6, 6), 7.0, device="cuda")
    I = torch.rand(8, 8, device="cuda")
    F = torch.rand(4, 9, 9, device="cuda")     # K=9 > 8
    with pytest.raises(conv.ConvError):
        conv.conv_single_ex(I, 8, 8, F, 9, 4, O)
    torch.cuda.synchronize()
    assert torch.all(O == 7.0)


def test_sharded_multi_virtual_ranks(conv):
    """sharded_multi on 4 virtual ranks of one GPU concatenates to the full result."""
    from paper_2212_00404_b200.shard import sharded_multi
    c = synth.MULTI_LAYERS[2]
    I, F = synth.layer_inputs(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], cfg_index=9)
    Oo, A = oracle.conv_multi(I, F)
    for prec in ("fp32", "tf32", "bf16"):
        dt = torch.bfloat16 if prec == "bf16" else torch.float32
        Id = torch.from_numpy(I).cuda().to(dt)
        Fd = torch.from_numpy(F).cuda().to(dt)
        parts = [sharded_multi(Id, Fd, prec, world=4, rank=r) for r in range(4)]
        torch.cuda.synchronize()
        Og = torch.cat(parts).cpu().numpy().astype(np.float64)
        assert_parity(Og, Oo, A, TAU[prec], f"virtual shards {prec}")


# KM-TC has two tensor-core paths: the im2col + TMA GEMM pair (KM-TC/G, the
# planner's choice for few-pixel, many-filter layers; B200CONV_GM=2 forces it
# wherever filter rows are TMA-able) and the implicit kernel (everything else,
# and the fallback when no workspace can be had during stream capture).
# Both are covered explicitly, with the split-K variants each one can take.
TC_PATHS = {
    "implicit": {"B200CONV_GM": "0"},
    "implicit-dsmem": {"B200CONV_GM": "0", "B200CONV_TC_DSMEM": "1"},
    "gemm": {"B200CONV_GM": "2"},
    "gemm-nosplit": {"B200CONV_GM": "2", "B200CONV_GM_SPLIT": "1"},
    "gemm-split3": {"B200CONV_GM": "2", "B200CONV_GM_SPLIT": "3"},
    "gemm-dsmem": {"B200CONV_GM": "2", "B200CONV_GM_SPLIT": "5", "B200CONV_GM_DSMEM": "1"},
    "gemm-ws": {"B200CONV_GM": "2", "B200CONV_GM_DSMEM": "0"},
}


@pytest.mark.parametrize("path", sorted(TC_PATHS))
@pytest.mark.parametrize("prec", ["tf32", "bf16"])
@pytest.mark.parametrize("i", [0, 1, 2, 5])
def test_tc_paths_layers(conv, multi_oracle, monkeypatch, path, prec, i):
    for k, v in TC_PATHS[path].items():
        monkeypatch.setenv(k, v)
    I, F, Oo, A = multi_oracle(i)
    assert_parity(run_multi(conv, I, F, prec), Oo, A, TAU[prec], f"{MULTI[i]['name']} {prec} {path}")


@pytest.mark.parametrize("path", sorted(TC_PATHS))
@pytest.mark.parametrize("prec", ["tf32", "bf16"])
def test_tc_paths_edges_and_ints(conv, monkeypatch, path, prec):
    for k, v in TC_PATHS[path].items():
        monkeypatch.setenv(k, v)
    for (C, Wx, Wy, K, M) in MULTI_EDGE:
        I = synth.uniform01(31, (C, Wy, Wx))
        F = synth.uniform_pm1(32, (M, C, K, K))
        Oo, A = oracle.conv_multi(I, F)
        assert_parity(run_multi(conv, I, F, prec), Oo, A, TAU[prec], f"edge {C},{Wx},{Wy},{K},{M} {prec} {path}")
    for (C, W, K, M) in [(64, 14, 3, 96), (96, 27, 5, 40), (512, 7, 3, 64), (16, 40, 3, 300)]:
        I, F = synth.layer_inputs(C, W, W, K, M, kind="ints")
        Oo, _ = oracle.conv_multi(I, F)
        assert np.array_equal(run_multi(conv, I, F, prec), Oo), (C, W, K, M, prec, path)


# KM-SIMT: every thread tile (B200CONV_SIMT_FORCE="tile,split,ws"), with no
# split, a cluster (DSMEM) split and a workspace split; shapes with chunks of
# k-steps that are / are not multiples of 4 (both F-transpose loops), ragged
# pixel and filter tiles, unaligned F rows (C*K*K odd).
SIMT_SHAPES = [(64, 14, 14, 3, 96), (20, 17, 11, 3, 70), (7, 9, 12, 5, 33), (130, 9, 9, 3, 300)]


@pytest.mark.parametrize("tile", range(9))
@pytest.mark.parametrize("split,ws", [(1, 0), (3, 0), (5, 1)])
def test_simt_every_tile_and_split(conv, monkeypatch, tile, split, ws):
    monkeypatch.setenv("B200CONV_SIMT_FORCE", f"{tile},{split},{ws}")
    for (C, Wx, Wy, K, M) in SIMT_SHAPES:
        I = synth.uniform01(41, (C, Wy, Wx))
        F = synth.uniform_pm1(42, (M, C, K, K))
        Oo, A = oracle.conv_multi(I, F)
        assert_parity(run_multi(conv, I, F, "fp32"), Oo, A, TAU["fp32"],
                      f"simt tile {tile} split {split} ws {ws} shape {(C, Wx, Wy, K, M)}")


# KM-TC implicit kernel with every filter-tile width (B200CONV_TC_BN) and a
# forced k split, on shapes with ragged filter / pixel tiles
@pytest.mark.parametrize("bn", [32, 64, 128, 256])
@pytest.mark.parametrize("prec", ["tf32", "bf16"])
def test_tc_every_filter_tile_width(conv, monkeypatch, bn, prec):
    monkeypatch.setenv("B200CONV_GM", "0")
    monkeypatch.setenv("B200CONV_TC_BN", str(bn))
    for split in ("1", "3"):
        monkeypatch.setenv("B200CONV_TC_SPLIT", split)
        for (C, Wx, Wy, K, M) in [(64, 14, 14, 3, 300), (20, 17, 11, 3, 70), (48, 30, 30, 5, 40)]:
            I = synth.uniform01(43, (C, Wy, Wx))
            F = synth.uniform_pm1(44, (M, C, K, K))
            Oo, A = oracle.conv_multi(I, F)
            assert_parity(run_multi(conv, I, F, prec), Oo, A, TAU[prec],
                          f"tc BN {bn} split {split} {prec} shape {(C, Wx, Wy, K, M)}")


# ------------------------------------------------------------------ batched
BATCHED = [  # (N, C, Wx, Wy, K, M): ragged pixel tiles, unaligned planes, split / no split
    (4, 64, 14, 14, 3, 96), (3, 5, 17, 11, 3, 37), (2, 96, 27, 27, 5, 40), (8, 32, 28, 28, 3, 256),
    (5, 130, 9, 9, 3, 33), (16, 16, 7, 7, 1, 20),
]


@pytest.mark.parametrize("prec", ["fp32", "tf32", "bf16"])
@pytest.mark.parametrize("N,C,Wx,Wy,K,M", BATCHED)
def test_batched_matches_oracle_per_image(conv, prec, N, C, Wx, Wy, K, M):
    I = np.stack([synth.uniform01(50 + n, (C, Wy, Wx)) for n in range(N)])
    F = synth.uniform_pm1(60, (M, C, K, K))
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    O = conv.multi_batched(torch.from_numpy(I).cuda().to(dt), torch.from_numpy(F).cuda().to(dt), prec)
    torch.cuda.synchronize()
    Og = O.cpu().numpy().astype(np.float64)
    for n in range(N):
        Oo, A = oracle.conv_multi(I[n], F)
        assert_parity(Og[n], Oo, A, TAU[prec], f"batched n={n} {N},{C},{Wx},{Wy},{K},{M} {prec}")


@pytest.mark.parametrize("prec", ["tf32", "bf16"])
def test_batched_integer_bit_exact_and_equals_unbatched(conv, prec):
    N, C, W, K, M = 6, 48, 20, 3, 136
    I = np.stack([synth.layer_inputs(C, W, W, K, M, cfg_index=70 + n, kind="ints")[0] for n in range(N)])
    F = synth.layer_inputs(C, W, W, K, M, cfg_index=70, kind="ints")[1]
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    Id, Fd = torch.from_numpy(I).cuda().to(dt), torch.from_numpy(F).cuda().to(dt)
    Ob = conv.multi_batched(Id, Fd, prec).cpu().numpy()
    for n in range(N):
        Oo, _ = oracle.conv_multi(I[n], F)
        assert np.array_equal(Ob[n].astype(np.float64), Oo), (n, prec)
        assert np.array_equal(Ob[n], conv.multi(Id[n].contiguous(), Fd, prec).cpu().numpy()), (n, prec)


# ------------------------------------------------------------------ zero padding
PADDED = [  # (N, C, Wx, Wy, K, M, pad): ResNet/VGG "same" 3x3 pad 1, AlexNet 5x5 pad 2, odd shapes
    (1, 64, 14, 14, 3, 96, 1), (2, 96, 27, 27, 5, 64, 2), (3, 5, 9, 7, 3, 17, 1), (1, 3, 32, 32, 3, 64, 1),
    (4, 32, 7, 7, 3, 128, 1), (1, 8, 4, 4, 7, 9, 3),
]


@pytest.mark.parametrize("prec", ["fp32", "tf32", "bf16"])
@pytest.mark.parametrize("N,C,Wx,Wy,K,M,pad", PADDED)
def test_padded_multi_matches_oracle_on_padded_input(conv, prec, N, C, Wx, Wy, K, M, pad):
    I = np.stack([synth.uniform01(80 + n, (C, Wy, Wx)) for n in range(N)])
    F = synth.uniform_pm1(90, (M, C, K, K))
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    O = conv.multi_padded(torch.from_numpy(I).cuda().to(dt), torch.from_numpy(F).cuda().to(dt), pad, prec)
    Og = O.cpu().numpy().astype(np.float64)
    for n in range(N):
        Ip = np.pad(I[n], ((0, 0), (pad, pad), (pad, pad)))        # the definition of zero padding
        Oo, A = oracle.conv_multi(Ip.astype(np.float32), F)
        assert_parity(Og[n], Oo, A, TAU[prec], f"padded n={n} {C},{Wx},{Wy},{K},{M},p{pad} {prec}")


@pytest.mark.parametrize("Wx,Wy,K,M,pad", [(28, 28, 3, 64, 1), (56, 56, 5, 32, 2), (7, 7, 7, 16, 3), (13, 9, 3, 5, 1)])
def test_padded_single_matches_oracle_on_padded_input(conv, Wx, Wy, K, M, pad):
    I = synth.uniform01(95, (Wy, Wx))
    F = synth.uniform_pm1(96, (M, K, K))
    Og = conv.single_padded(torch.from_numpy(I).cuda(), torch.from_numpy(F).cuda(), pad).cpu().numpy()
    Oo, A = oracle.conv_single(np.pad(I, pad).astype(np.float32), F)
    assert_parity(Og.astype(np.float64), Oo, A, TAU["fp32"], f"padded single p{pad}")


# ------------------------------------------------------------------ determinism and stream capture
# every kernel path: KS, KS-C3, KM-SIMT (cluster and workspace splits), KM-TC
# (implicit, split / no split), KM-TC/G (filters on M, split), batched
PATH_CASES = [  # (kind, C, W, K, M, prec)
    ("single", 1, 224, 3, 64, "fp32"), ("multi", 3, 224, 3, 64, "bf16"), ("multi", 128, 28, 3, 128, "fp32"),
    ("multi", 512, 7, 3, 512, "fp32"), ("multi", 256, 28, 3, 256, "tf32"), ("multi", 64, 56, 3, 64, "bf16"),
    ("multi", 512, 7, 3, 512, "bf16"), ("multi", 512, 14, 3, 1024, "tf32"),
]


def _case_tensors(kind, C, W, K, M, prec, seed):
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    I = torch.from_numpy(synth.uniform01(seed, (C, W, W))).cuda().to(dt)
    F = torch.from_numpy(synth.uniform_pm1(seed + 1, (M, C, K, K))).cuda().to(dt)
    if kind == "single":
        I, F = I[0].contiguous(), F[:, 0].contiguous()
    O = torch.empty((M, W - K + 1, W - K + 1), device="cuda")
    return I, F, O


def _call(conv, kind, I, F, O, C, W, K, M, prec, stream):
    if kind == "single":
        conv.conv_single_ex(I, W, W, F, K, M, O, stream)
    else:
        conv.conv_multi_ex(I, C, W, W, F, K, M, O, prec, stream)


def test_every_path_is_run_to_run_deterministic(conv):
    for i, (kind, C, W, K, M, prec) in enumerate(PATH_CASES):
        I, F, O = _case_tensors(kind, C, W, K, M, prec, 300 + 2 * i)
        outs = []
        for _ in range(3):
            O.fill_(float("nan"))
            _call(conv, kind, I, F, O, C, W, K, M, prec, None)
            torch.cuda.synchronize()
            outs.append(O.cpu().numpy().copy())
        assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2]), (kind, C, W, K, M, prec)


def test_every_path_replays_from_a_cuda_graph(conv):
    # capture after a warm-up call (workspaces exist), replay, compare with eager
    s = torch.cuda.Stream()
    for i, (kind, C, W, K, M, prec) in enumerate(PATH_CASES):
        I, F, O = _case_tensors(kind, C, W, K, M, prec, 400 + 2 * i)
        with torch.cuda.stream(s):
            _call(conv, kind, I, F, O, C, W, K, M, prec, s.cuda_stream)
            s.synchronize()
            ref = O.clone()
            O.fill_(float("nan"))
            g = torch.cuda.CUDAGraph()
            g.capture_begin()
            _call(conv, kind, I, F, O, C, W, K, M, prec, s.cuda_stream)
            g.capture_end()
            g.replay()
            g.replay()
            s.synchronize()
        assert torch.equal(O, ref), (kind, C, W, K, M, prec)


# ------------------------------------------------------------------ KS-C3 (C = 3 stems): odd shapes
C3_CASES = [  # (Wx, Wy, K, M): odd planes (BF16 element staging), K = 5, ragged filter groups
    (33, 29, 3, 7), (40, 40, 5, 64), (27, 31, 5, 9), (224, 19, 3, 130), (57, 57, 3, 1),
]


@pytest.mark.parametrize("prec", ["fp32", "tf32", "bf16"])
@pytest.mark.parametrize("Wx,Wy,K,M", C3_CASES)
def test_c3_stem_path_matches_oracle(conv, prec, Wx, Wy, K, M):
    assert conv.plan_multi(3, Wx, Wy, K, M, prec)["kernel"] == 4
    I = synth.uniform01(500 + Wx, (3, Wy, Wx))
    F = synth.uniform_pm1(600 + K, (M, 3, K, K))
    Oo, A = oracle.conv_multi(I, F)
    assert_parity(run_multi(conv, I, F, prec), Oo, A, TAU[prec], f"c3 {Wx}x{Wy} K{K} M{M} {prec}")


# ------------------------------------------------------------------ stride > 1
# O[y][x] = sum I_pad[y*s + r][x*s + c] F[r][c]: the stride-1 valid result of
# the zero-padded input at rows / columns 0, s, 2s, ... (definition of stride)
STRIDED = [  # (N, C, Wx, Wy, K, M, pad, stride): ResNet downsampling 3x3/2 and 1x1/2, a 7x7/2 RGB stem,
    # ragged and odd shapes, unaligned filter rows (C*K*K*elem not a multiple of 16 B), stride 3
    (1, 64, 56, 56, 3, 128, 1, 2), (1, 256, 14, 14, 1, 512, 0, 2), (1, 3, 33, 29, 7, 20, 3, 2),
    (2, 20, 17, 11, 3, 70, 0, 3), (1, 7, 9, 12, 5, 33, 2, 2), (3, 16, 28, 28, 3, 40, 1, 2),
]


def _strided_ref(I, F, pad, s):
    Ip = np.pad(I, ((0, 0), (pad, pad), (pad, pad)))
    Oo, A = oracle.conv_multi(Ip.astype(np.float32), F)
    return Oo[:, ::s, ::s], A[:, ::s, ::s]


@pytest.mark.parametrize("prec", ["fp32", "tf32", "bf16"])
@pytest.mark.parametrize("N,C,Wx,Wy,K,M,pad,s", STRIDED)
def test_strided_multi_matches_oracle(conv, prec, N, C, Wx, Wy, K, M, pad, s):
    I = np.stack([synth.uniform01(70 + n, (C, Wy, Wx)) for n in range(N)])
    F = synth.uniform_pm1(71, (M, C, K, K))
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    O = conv.multi_strided(torch.from_numpy(I).cuda().to(dt), torch.from_numpy(F).cuda().to(dt), s, pad, prec)
    torch.cuda.synchronize()
    Og = O.cpu().numpy().astype(np.float64)
    for n in range(N):
        Oo, A = _strided_ref(I[n], F, pad, s)
        assert_parity(Og[n], Oo, A, TAU[prec], f"strided n={n} {C},{Wx},{Wy},{K},{M},p{pad},s{s} {prec}")


@pytest.mark.parametrize("prec", ["fp32", "tf32", "bf16"])
def test_strided_integer_inputs_bit_exact(conv, prec):
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    for (C, W, K, M, pad, s) in [(64, 30, 3, 96, 1, 2), (3, 40, 7, 24, 3, 2), (9, 13, 5, 17, 0, 3)]:
        I, F = synth.layer_inputs(C, W, W, K, M, kind="ints")
        O = conv.multi_strided(torch.from_numpy(I[None]).cuda().to(dt), torch.from_numpy(F).cuda().to(dt), s, pad,
                               prec)
        Oo, _ = _strided_ref(I, F, pad, s)
        assert np.array_equal(O[0].cpu().numpy().astype(np.float64), Oo), (C, W, K, M, pad, s, prec)


@pytest.mark.parametrize("Wx,Wy,K,M,pad,s", [(224, 224, 7, 32, 3, 2), (28, 28, 3, 64, 1, 2), (13, 9, 3, 5, 0, 3)])
def test_strided_single_matches_oracle(conv, Wx, Wy, K, M, pad, s):
    I = synth.uniform01(72, (Wy, Wx))
    F = synth.uniform_pm1(73, (M, K, K))
    O = conv.single_strided(torch.from_numpy(I).cuda(), torch.from_numpy(F).cuda(), s, pad)
    torch.cuda.synchronize()
    Oo, A = _strided_ref(I[None], F[:, None], pad, s)
    assert_parity(O.cpu().numpy().astype(np.float64), Oo, A, TAU["fp32"], f"single strided {Wx},{Wy},{K},{M},p{pad},s{s}")


def test_strided_stride1_is_the_padded_call(conv):
    I = torch.from_numpy(synth.uniform01(74, (2, 16, 20, 20))).cuda()
    F = torch.from_numpy(synth.uniform_pm1(75, (24, 16, 3, 3))).cuda()
    for prec in ("fp32", "tf32"):
        assert torch.equal(conv.multi_strided(I, F, 1, 1, prec), conv.multi_padded(I, F, 1, prec))


# strict-FP32 batch in ONE KM-SIMT launch (pixel tiles across images): every
# thread tile with a cluster and a workspace split, tiles straddling images
@pytest.mark.parametrize("tile", range(9))
@pytest.mark.parametrize("split,ws", [(1, 0), (3, 0), (5, 1)])
def test_simt_batched_every_tile(conv, monkeypatch, tile, split, ws):
    monkeypatch.setenv("B200CONV_SIMT_FORCE", f"{tile},{split},{ws}")
    N, C, Wx, Wy, K, M = 3, 20, 17, 11, 3, 70
    I = np.stack([synth.uniform01(60 + n, (C, Wy, Wx)) for n in range(N)])
    F = synth.uniform_pm1(61, (M, C, K, K))
    O = conv.multi_batched(torch.from_numpy(I).cuda(), torch.from_numpy(F).cuda(), "fp32")
    torch.cuda.synchronize()
    Og = O.cpu().numpy().astype(np.float64)
    for n in range(N):
        Oo, A = oracle.conv_multi(I[n], F)
        assert_parity(Og[n], Oo, A, TAU["fp32"], f"simt batched tile {tile} split {split} ws {ws} n={n}")


# persistent KM-TC (more tiles than SMs: each CTA walks several tiles, the
# epilogue of one overlapping the next one's loads); integer inputs: equal to
# the one-tile-per-CTA kernel and to the oracle
@pytest.mark.parametrize("prec", ["tf32", "bf16"])
@pytest.mark.parametrize("M", [300, 200, 64, 32])      # filter tiles of 256 (ragged), 128 (ragged), 64, 32
def test_tc_persistent_many_tiles(conv, monkeypatch, prec, M):
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    N, C, W, K = 40, 64, 28, 3                           # 40 x 6 pixel tiles (x filter tiles) > 148
    I, F = synth.layer_inputs(C, W, W, K, M, kind="ints")
    Ib = np.stack([np.roll(I, n, axis=-1) for n in range(N)])
    plan = conv.plan_multi_batched(N, C, W, W, K, M, prec)
    assert plan["tma_f"] & 32, plan
    Id, Fd = torch.from_numpy(Ib).cuda().to(dt), torch.from_numpy(F).cuda().to(dt)
    Op = conv.multi_batched(Id, Fd, prec)
    monkeypatch.setenv("B200CONV_TC_PERSIST", "0")
    O1 = conv.multi_batched(Id, Fd, prec)
    torch.cuda.synchronize()
    assert torch.equal(Op, O1)
    for n in (0, 17, N - 1):
        Oo, _ = oracle.conv_multi(Ib[n], F)
        assert np.array_equal(Op[n].cpu().numpy().astype(np.float64), Oo), n


def test_batched_strided_persistent_replay_from_a_cuda_graph(conv):
    # the batch / stride entry points and the persistent kernel under graph capture
    s = torch.cuda.Stream()
    I = torch.from_numpy(synth.uniform01(90, (40, 64, 28, 28))).cuda()
    F = torch.from_numpy(synth.uniform_pm1(91, (300, 64, 3, 3))).cuda()
    assert conv.plan_multi_batched(40, 64, 28, 28, 3, 300, "tf32")["tma_f"] & 32
    calls = [
        lambda O: conv.conv_multi_batched_ex(I, 40, 64, 28, 28, F, 3, 300, O, "tf32", s.cuda_stream),
        lambda O: conv.conv_multi_strided_ex(I, 40, 64, 28, 28, F, 3, 300, 1, 2, O, "tf32", s.cuda_stream),
        lambda O: conv.conv_multi_strided_ex(I, 40, 64, 28, 28, F, 3, 300, 1, 2, O, "fp32", s.cuda_stream),
    ]
    shapes = [(40, 300, 26, 26), (40, 300, 14, 14), (40, 300, 14, 14)]
    for fn, shp in zip(calls, shapes):
        O = torch.empty(shp, device="cuda")
        with torch.cuda.stream(s):
            fn(O)
            s.synchronize()
            ref = O.clone()
            O.fill_(float("nan"))
            g = torch.cuda.CUDAGraph()
            g.capture_begin()
            fn(O)
            g.capture_end()
            g.replay()
            g.replay()
            s.synchronize()
        assert torch.equal(O, ref), shp
