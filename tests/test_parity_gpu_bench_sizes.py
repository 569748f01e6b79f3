"""Parity at the exact sizes and entry points the bench and the C ABI expose
(`-m gpu`): the north_star calls on the legacy default stream, the persistent
batched tensor-core kernel at the 28x28x256 N = 64 layer on float data, the
bench's padded N = 32 and strided N = 8 rows, and the filter-sharded path run
end to end by two processes (broadcast -> CUDA shard -> all-gather).

Oracle side: oracle.conv_multi / conv_multi_sampled (fp64, Eq. 1,
P:92-98) on the same seeded float32 inputs; zero padding is np.pad of the
input (its definition) and stride s keeps every s-th row / column of the
stride-1 result (its definition).  Tolerances: north_star's tau * A."""
import os
import socket

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


def check(Og, Oo, A, tau, what):
    err = np.abs(np.asarray(Og, np.float64) - Oo)
    bad = err > tau * A
    assert not bad.any(), f"{what}: {int(bad.sum())}/{bad.size} out of tolerance, max err/A " \
                          f"{float((err / np.maximum(A, 1e-300)).max()):.3g}"
    assert np.all(np.asarray(Og)[A == 0] == 0), what


def _dt(prec):
    return torch.bfloat16 if prec == "bf16" else torch.float32


# ---------------------------------------------------------------- (b) default-stream ABI calls
@pytest.mark.parametrize("Wx,Wy,K,M", [(32, 32, 3, 4), (224, 224, 3, 64), (56, 56, 7, 32), (7, 7, 1, 256)])
def test_conv_single_on_the_default_stream(conv, Wx, Wy, K, M):
    """conv_single(I,Wx,Wy,F,K,M,O) — the north_star name, legacy stream 0."""
    I, F = synth.layer_inputs(1, Wx, Wy, K, M, cfg_index=K)
    Id, Fd = torch.from_numpy(I[0]).cuda(), torch.from_numpy(F[:, 0]).cuda()
    O = torch.full((M, Wy - K + 1, Wx - K + 1), float("nan"), device="cuda")
    torch.cuda.synchronize()
    conv.conv_single(Id, Wx, Wy, Fd, K, M, O)
    torch.cuda.synchronize()
    Oo, A = oracle.conv_single(I[0], F[:, 0])
    check(O.cpu().numpy(), Oo, A, TAU["fp32"], f"conv_single {Wx}x{Wy} K{K} M{M}")


@pytest.mark.parametrize("i", [0, 2, 3, 5])
def test_conv_multi_on_the_default_stream(conv, i):
    """conv_multi(I,C,Wx,Wy,F,K,M,O) — strict FP32 on the legacy stream 0."""
    c = synth.MULTI_LAYERS[i]
    I, F = synth.layer_inputs(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], cfg_index=300 + i)
    Id, Fd = torch.from_numpy(I).cuda(), torch.from_numpy(F).cuda()
    O = torch.full((c["M"], c["Wy"] - c["K"] + 1, c["Wx"] - c["K"] + 1), float("nan"), device="cuda")
    torch.cuda.synchronize()
    conv.conv_multi(Id, c["C"], c["Wx"], c["Wy"], Fd, c["K"], c["M"], O)
    torch.cuda.synchronize()
    Oo, A = oracle.conv_multi(I, F)
    check(O.cpu().numpy(), Oo, A, TAU["fp32"], f"conv_multi {c['name']}")


# ---------------------------------------------------------------- (c) persistent KM-TC, 28x28x256 N=64
def _sample_idx(n, k, seed):
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([rng.integers(0, n, k), np.arange(64), np.arange(n - 64, n)]))


@pytest.mark.parametrize("prec", ["tf32", "bf16"])
def test_persistent_tc_28x28x256_n64_float_sampled(conv, prec):
    N, C, W, K, M = 64, 256, 28, 3, 256
    plan = conv.plan_multi_batched(N, C, W, W, K, M, prec)
    assert plan["tma_f"] & 32, plan                       # the persistent kernel the bench times
    I = synth.uniform01(synth.SEED_I + N, (N, C, W, W))
    F = synth.uniform_pm1(synth.SEED_F + N, (M, C, K, K))
    O = conv.multi_batched(torch.from_numpy(I).cuda().to(_dt(prec)), torch.from_numpy(F).cuda().to(_dt(prec)), prec)
    Og = O.cpu().numpy().reshape(N, -1)
    Ho = W - K + 1
    for n in (0, 1, 37, N - 1):
        idx = _sample_idx(M * Ho * Ho, 1500, n)
        Oo, A = oracle.conv_multi_sampled(I[n], F, idx)
        check(Og[n][idx], Oo, A, TAU[prec], f"persistent {prec} image {n}")


# ---------------------------------------------------------------- (d) the bench's padded / strided rows
@pytest.mark.parametrize("prec,N", [("fp32", 1), ("tf32", 1), ("bf16", 1), ("tf32", 32), ("bf16", 32)])
def test_bench_padded_rows_sampled(conv, prec, N):
    C, W, K, M, pad = 256, 28, 3, 256, 1
    I = synth.uniform01(synth.SEED_I + N, (N, C, W, W))
    F = synth.uniform_pm1(synth.SEED_F + N, (M, C, K, K))
    O = conv.multi_padded(torch.from_numpy(I).cuda().to(_dt(prec)), torch.from_numpy(F).cuda().to(_dt(prec)),
                          pad, prec)
    Og = O.cpu().numpy().reshape(N, -1)
    for n in sorted({0, N // 2, N - 1}):
        Ip = np.pad(I[n], ((0, 0), (pad, pad), (pad, pad)))
        idx = _sample_idx(M * W * W, 2000, 7 + n)
        Oo, A = oracle.conv_multi_sampled(Ip, F, idx)
        check(Og[n][idx], Oo, A, TAU[prec], f"padded {prec} N={N} image {n}")


@pytest.mark.parametrize("prec", ["fp32", "tf32", "bf16"])
@pytest.mark.parametrize("N", [1, 8])
def test_bench_strided_rows_sampled(conv, prec, N):
    C, W, K, M, pad, s = 64, 56, 3, 128, 1, 2
    Ho = (W + 2 * pad - K) // s + 1
    I = synth.uniform01(synth.SEED_I + 11 * N, (N, C, W, W))
    F = synth.uniform_pm1(synth.SEED_F + 11 * N, (M, C, K, K))
    O = conv.multi_strided(torch.from_numpy(I).cuda().to(_dt(prec)), torch.from_numpy(F).cuda().to(_dt(prec)),
                           s, pad, prec)
    Og = O.cpu().numpy().reshape(N, -1)
    Hp = W + 2 * pad - K + 1                                # stride-1 output of the padded map
    for n in sorted({0, N - 1}):
        Ip = np.pad(I[n], ((0, 0), (pad, pad), (pad, pad)))
        idx = _sample_idx(M * Ho * Ho, 2000, 11 + n)
        m, r = np.divmod(idx, Ho * Ho)
        y, x = np.divmod(r, Ho)
        Oo, A = oracle.conv_multi_sampled(Ip, F, (m * Hp + y * s) * Hp + x * s)
        check(Og[n][idx], Oo, A, TAU[prec], f"strided {prec} N={N} image {n}")


# ---------------------------------------------------------------- (a) sharded path end to end, 2 processes
def _free_port():
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    p = sk.getsockname()[1]
    sk.close()
    return p


def _shard_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)                   # both ranks on the one GPU of the box
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2212_00404_b200.shard import allgather_output, broadcast_input, sharded_multi
        c = synth.MULTI_LAYERS[1]
        out = {}
        for prec in ("fp32", "tf32", "bf16"):
            I, F = synth.layer_inputs(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], cfg_index=400)
            Id = torch.from_numpy(I).cuda().to(_dt(prec)) if rank == 0 else \
                torch.zeros((c["C"], c["Wy"], c["Wx"]), device="cuda", dtype=_dt(prec))
            broadcast_input(Id, src=0)                          # G0
            Fd = torch.from_numpy(F).cuda().to(_dt(prec))
            Oloc = sharded_multi(Id, Fd, prec)                  # G1: this rank's filters on the CUDA path
            torch.cuda.synchronize()
            Ofull = allgather_output(Oloc, c["M"])              # G2
            torch.cuda.synchronize()
            out[prec] = Ofull.cpu().numpy()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_sharded_path_two_processes_end_to_end():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    c = synth.MULTI_LAYERS[1]
    I, F = synth.layer_inputs(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], cfg_index=400)
    Oo, A = oracle.conv_multi(I, F)
    for prec in ("fp32", "tf32", "bf16"):
        for r in (0, 1):
            check(res[r][prec], Oo, A, TAU[prec], f"rank {r} gathered {prec}")
        assert np.array_equal(res[0][prec], res[1][prec])


@pytest.mark.parametrize("args", [
    ["--mode", "single", "--wx", "224", "--wy", "224", "--k", "3", "--m", "64"],
    ["--mode", "multi", "--wx", "14", "--wy", "14", "--c", "512", "--k", "3", "--m", "4096", "--precision", "bf16"],
    ["--mode", "multi", "--wx", "27", "--wy", "27", "--c", "96", "--k", "5", "--m", "256", "--precision", "tf32"],
])
def test_verify_cli_passes(conv, args):
    import subprocess
    import sys
    v = os.path.join(os.path.dirname(os.path.abspath(__file__)), "verify.py")
    r = subprocess.run([sys.executable, v, *args], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.startswith("PASS"), r.stdout + r.stderr


@pytest.mark.parametrize("prec,layer", [("fp32", 7), ("tf32", 2), ("bf16", 7)])
def test_capture_on_a_fresh_stream_uses_graph_private_scratch(conv, prec, layer):
    """A workspace-needing call captured on a stream that never ran it (its
    buffer cannot grow during capture) gets graph memory-node scratch; two
    such graphs replayed on different streams at once stay correct."""
    c = (list(synth.MULTI_LAYERS) + [synth.SHARD_SWEEP])[layer]
    I, F = synth.layer_inputs(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], cfg_index=500 + layer)
    Id, Fd = torch.from_numpy(I).cuda().to(_dt(prec)), torch.from_numpy(F).cuda().to(_dt(prec))
    ref = conv.multi(Id, Fd, prec)
    shape = tuple(ref.shape)
    outs, graphs, streams = [], [], [torch.cuda.Stream(), torch.cuda.Stream()]
    for st in streams:
        O = torch.full(shape, float("nan"), device="cuda")
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            g.capture_begin()
            conv.conv_multi_ex(Id, c["C"], c["Wx"], c["Wy"], Fd, c["K"], c["M"], O, prec, st.cuda_stream)
            g.capture_end()
        outs.append(O)
        graphs.append(g)
    torch.cuda.synchronize()
    for _ in range(3):
        for st, g in zip(streams, graphs):
            with torch.cuda.stream(st):
                g.replay()
    torch.cuda.synchronize()
    for O in outs:
        assert torch.equal(O, ref)


# ---------------------------------------------------------------- NEXT-2: epilogue-fused all-gather
@pytest.mark.parametrize("prec,layer", [("fp32", 1), ("tf32", 2), ("bf16", 2), ("fp32", 7), ("tf32", 0),
                                        ("bf16", 3), ("tf32", 7), ("bf16", 7)])
def test_allgather_fused_into_the_epilogue(conv, prec, layer):
    """Four virtual ranks on one GPU, each owning M/4 filters, write their rows
    straight into three 'peer' copies of O (conv_multi_allgather_ex): every
    copy must equal the oracle's full O.  Layers cover the peer-aware stores
    (KM-SIMT split-K reduce, KM-TC/G GEMM) and the copy fallback (implicit
    KM-TC, KS-C3)."""
    c = (list(synth.MULTI_LAYERS) + [synth.SHARD_SWEEP])[layer]
    I, F = synth.layer_inputs(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], cfg_index=600 + layer)
    Ho, Wo = c["Wy"] - c["K"] + 1, c["Wx"] - c["K"] + 1
    Id, Fd = torch.from_numpy(I).cuda().to(_dt(prec)), torch.from_numpy(F).cuda().to(_dt(prec))
    peers = [torch.full((c["M"], Ho, Wo), float("nan"), device="cuda") for _ in range(3)]
    world = 4
    Ml = c["M"] // world
    for r in range(world):
        Fl = Fd[r * Ml:(r + 1) * Ml].contiguous()
        conv.conv_multi_allgather_ex(Id, c["C"], c["Wx"], c["Wy"], Fl, c["K"], Ml, r * Ml, c["M"], peers,
                                     None, prec)
    torch.cuda.synchronize()
    if c["M"] * Ho * Wo > 2_000_000:
        idx = _sample_idx(c["M"] * Ho * Wo, 3000, layer)
        Oo, A = oracle.conv_multi_sampled(I, F, idx)
        for P in peers:
            check(P.cpu().numpy().ravel()[idx], Oo, A, TAU[prec], f"allgather peer {prec} {c['name']}")
    else:
        Oo, A = oracle.conv_multi(I, F)
        for P in peers:
            check(P.cpu().numpy(), Oo, A, TAU[prec], f"allgather peer {prec} {c['name']}")
    assert torch.equal(peers[0], peers[1]) and torch.equal(peers[0], peers[2])


def _symm_worker(q, port):
    """world-1 NCCL group: torch symmetric memory for O, the fused call through
    its buffer pointers, and through its multicast address when the device
    offers one (NVSwitch multicast: multimem.st in the epilogue)."""
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    out = {}
    try:
        from paper_2212_00404_b200 import conv
        c = synth.MULTI_LAYERS[1]
        I, F = synth.layer_inputs(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], cfg_index=700)
        Ho = c["Wy"] - c["K"] + 1
        for prec in ("fp32", "tf32"):
            O = symm.empty((c["M"], Ho, Ho), dtype=torch.float32, device="cuda")
            O.fill_(float("nan"))
            hdl = symm.rendezvous(O, dist.group.WORLD)
            base = hdl.buffer_ptrs[0]
            Id, Fd = torch.from_numpy(I).cuda(), torch.from_numpy(F).cuda()
            conv.conv_multi_allgather_ex(Id, c["C"], c["Wx"], c["Wy"], Fd, c["K"], c["M"], 0, c["M"],
                                         [base + (O.data_ptr() - base)], None, prec)
            torch.cuda.synchronize()
            out[prec] = O.cpu().numpy()
            mc = int(getattr(hdl, "multicast_ptr", 0) or 0)
            if mc:
                O.fill_(float("nan"))
                conv.conv_multi_allgather_ex(Id, c["C"], c["Wx"], c["Wy"], Fd, c["K"], c["M"], 0, c["M"],
                                             [O.data_ptr()], mc + (O.data_ptr() - base), prec)
                torch.cuda.synchronize()
                out[prec + "_mc"] = O.cpu().numpy()
        q.put(out)
    except Exception as e:   # reported to the parent
        q.put({"error": repr(e)[:300]})
    finally:
        dist.destroy_process_group()


def test_allgather_through_torch_symmetric_memory():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_symm_worker, args=(q, _free_port()))
    p.start()
    res = q.get(timeout=300)
    p.join(timeout=60)
    assert "error" not in res, res
    c = synth.MULTI_LAYERS[1]
    I, F = synth.layer_inputs(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], cfg_index=700)
    Oo, A = oracle.conv_multi(I, F)
    for k, O in res.items():
        check(O, Oo, A, TAU[k.split("_")[0]], f"symmetric memory {k}")
    print("symmetric-memory paths checked:", sorted(res))
