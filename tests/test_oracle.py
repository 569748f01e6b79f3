"""Pins for the CPU oracle (oracle/conv_oracle.c) — against values the paper and
mathematics fix, never against the oracle itself.  All `-m "not gpu"`.

Each test names the SURVEY.md §8(c) pin it implements.  A plausible oracle bug
fails at least one: swapped filter axes (P2), dropped channel term or wrong
F layout (P3, P5, P9 channel-sum), off-by-one ranges (P1 shape, P4 crop),
wrong sign (P3 has a negative coefficient), transposed operand (P6).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from conftest import load_golden


# --- P1-P3: hand-worked golden examples (tests/golden, cited there) ----------
@pytest.mark.parametrize("name", ["p1_single_handworked.txt", "p2_orientation_delta.txt"])
def test_golden_single(name):
    g = load_golden(name)
    I, F, Oexp = g["I"][0], g["F"][:, 0], g["O"]
    O, A = oracle.conv_single(I, F)
    assert O.shape == Oexp.shape
    assert np.array_equal(O, Oexp)


def test_golden_multi():
    g = load_golden("p3_multi_handworked.txt")
    O, A = oracle.conv_multi(g["I"], g["F"])
    assert np.array_equal(O, g["O"])
    assert np.array_equal(A, g["A"])


# --- P4: delta-filter closed form (shift / crop / channel selection) --------
@pytest.mark.parametrize("C,Wy,Wx,K", [(1, 9, 7, 3), (3, 8, 11, 4), (2, 5, 5, 5), (4, 13, 6, 1)])
def test_delta_filters(C, Wy, Wx, K):
    I = synth.uniform01(11, (C, Wy, Wx))
    taps = [(ch, r, c) for ch in range(C) for r in range(K) for c in range(K)]
    M = len(taps)
    F = np.zeros((M, C, K, K), np.float32)
    for m, (ch, r, c) in enumerate(taps):
        F[m, ch, r, c] = 1.0
    O, A = oracle.conv_multi(I, F)
    Ho, Wo = Wy - K + 1, Wx - K + 1
    for m, (ch, r, c) in enumerate(taps):
        assert np.array_equal(O[m], I[ch, r:r + Ho, c:c + Wo].astype(np.float64))
    # (0,0) delta is the top-left crop
    assert np.array_equal(O[0], I[0, :Ho, :Wo].astype(np.float64))


# --- P5: all-ones / ramp / constant-plane closed forms ----------------------
@pytest.mark.parametrize("C,W,K", [(1, 6, 3), (3, 9, 2), (5, 7, 7), (2, 12, 5)])
def test_all_ones_and_ramp(C, W, K):
    M = 2
    F = np.ones((M, C, K, K), np.float32)
    O, _ = oracle.conv_multi(np.ones((C, W, W), np.float32), F)
    assert np.all(O == C * K * K)
    # ramp I[ch][y][x] = x + W*y  ->  O = C*(K^2 (x + W y) + K^2 (K-1)/2 (1 + W))
    y, x = np.mgrid[0:W, 0:W]
    ramp = np.broadcast_to((x + W * y).astype(np.float32), (C, W, W))
    O, _ = oracle.conv_multi(ramp, F)
    Ho = W - K + 1
    yy, xx = np.mgrid[0:Ho, 0:Ho]
    closed = C * (K * K * (xx + W * yy) + K * K * (K - 1) / 2 * (1 + W))
    assert np.array_equal(O[0], closed) and np.array_equal(O[1], closed)


def test_spec_trivial_examples():
    I = synth.uniform01(3, (1, 6, 5))
    O, _ = oracle.conv_multi(I, np.ones((1, 1, 1, 1), np.float32))        # identity
    assert np.array_equal(O[0], I[0].astype(np.float64))
    a, b = np.float32(0.75), np.float32(-2.5)
    I2 = np.stack([np.full((4, 4), a, np.float32), np.full((4, 4), b, np.float32)])
    O, _ = oracle.conv_multi(I2, np.ones((1, 2, 1, 1), np.float32))       # a + b
    assert np.all(O == float(a) + float(b))
    O, A = oracle.conv_single(synth.uniform01(4, (8, 8)), np.zeros((3, 3, 3), np.float32))
    assert np.all(O == 0) and np.all(A == 0)                              # zero filter


# --- P6: K=1 is a textbook matrix product ------------------------------------
def test_k1_is_matmul():
    C, Wy, Wx, M = 7, 5, 9, 6
    I = synth.uniform01(5, (C, Wy, Wx))
    F = synth.uniform_pm1(6, (M, C, 1, 1))
    O, A = oracle.conv_multi(I, F)
    ref = F.reshape(M, C).astype(np.float64) @ I.reshape(C, -1).astype(np.float64)
    np.testing.assert_allclose(O.reshape(M, -1), ref, rtol=0, atol=1e-12 * A.max())


# --- P7: K = Wx = Wy is a dot product ----------------------------------------
def test_full_window_is_dot():
    C, W, M = 4, 6, 3
    I = synth.uniform01(7, (C, W, W))
    F = synth.uniform_pm1(8, (M, C, W, W))
    O, A = oracle.conv_multi(I, F)
    assert O.shape == (M, 1, 1)
    for m in range(M):
        d = np.dot(F[m].ravel().astype(np.float64), I.ravel().astype(np.float64))
        assert abs(O[m, 0, 0] - d) <= 1e-13 * A[m, 0, 0]


# --- P8: library routine (torch float64 conv2d, cross-correlation) -----------
@pytest.mark.parametrize("C,Wy,Wx,K,M", [(3, 5, 5, 3, 2), (1, 32, 32, 3, 4), (5, 11, 9, 4, 3),
                                         (2, 7, 7, 7, 2), (8, 14, 14, 3, 5)])
def test_matches_torch_conv2d_f64(C, Wy, Wx, K, M):
    I = synth.uniform01(9, (C, Wy, Wx))
    F = synth.uniform_pm1(10, (M, C, K, K))
    O, A = oracle.conv_multi(I, F)
    ref = torch.nn.functional.conv2d(torch.from_numpy(I).double()[None],
                                     torch.from_numpy(F).double())[0].numpy()
    assert np.all(np.abs(O - ref) <= 1e-12 * A)


# --- P9: invariants -----------------------------------------------------------
def test_linearity_and_channel_sum_and_shards():
    C, W, K, M = 3, 10, 3, 4
    I = synth.uniform01(12, (C, W, W))
    I2 = synth.uniform01(13, (C, W, W))
    F = synth.uniform_pm1(14, (M, C, K, K))
    O, A = oracle.conv_multi(I, F)
    # scaling by a power of two is exact
    O4, _ = oracle.conv_multi(4 * I, F)
    assert np.array_equal(O4, 4 * O)
    O4f, _ = oracle.conv_multi(I, 0.5 * F)
    assert np.array_equal(O4f, 0.5 * O)
    # additivity in I
    Os, As = oracle.conv_multi(I + I2, F)
    O2, A2 = oracle.conv_multi(I2, F)
    assert np.all(np.abs(Os - (O + O2)) <= 1e-6 * (A + A2))   # I+I2 is rounded to f32
    # multi == sum over channels of single (north_star)
    acc = np.zeros_like(O)
    for ch in range(C):
        Oc, _ = oracle.conv_single(I[ch], F[:, ch])
        acc += Oc
    assert np.all(np.abs(acc - O) <= 1e-13 * A)
    # C = 1 multi == single bitwise
    Om, _ = oracle.conv_multi(I[:1], F[:, :1])
    Osg, _ = oracle.conv_single(I[0], F[:, 0])
    assert np.array_equal(Om, Osg)
    # filter shards concatenate to the full result
    parts = [oracle.conv_multi(I, F[a:b])[0] for a, b in ((0, 1), (1, 3), (3, 4))]
    assert np.array_equal(np.concatenate(parts), O)
    # A bounds |O|; equals O on nonnegative data
    assert np.all(A >= np.abs(O))
    Op, Ap = oracle.conv_multi(I, np.abs(F))
    assert np.array_equal(Op, Ap)


# --- P10: exactness on small integers (brute force via integer im2col) -------
def test_integer_inputs_exact():
    C, W, K, M = 6, 9, 3, 5
    I, F = synth.layer_inputs(C, W, W, K, M, kind="ints")
    O, _ = oracle.conv_multi(I, F)
    Ii, Fi = I.astype(np.int64), F.astype(np.int64)
    Ho = W - K + 1
    cols = np.stack([Ii[:, r:r + Ho, c:c + Ho] for r in range(K) for c in range(K)], axis=1)
    ref = np.einsum("mk,kyx->myx", Fi.reshape(M, C * K * K), cols.reshape(C * K * K, Ho, Ho))
    assert np.array_equal(O, ref.astype(np.float64))


# --- sampled evaluation == full evaluation ------------------------------------
def test_sampled_matches_full():
    C, W, K, M = 3, 12, 5, 4
    I = synth.uniform01(15, (C, W, W))
    F = synth.uniform_pm1(16, (M, C, K, K))
    O, A = oracle.conv_multi(I, F)
    idx = np.array([0, 1, 17, O.size - 1, 50, 63], dtype=np.int64)
    Os, As = oracle.conv_multi_sampled(I, F, idx)
    assert np.array_equal(Os, O.ravel()[idx]) and np.array_equal(As, A.ravel()[idx])


def test_thread_count_does_not_change_bits():
    I = synth.uniform01(17, (4, 20, 20))
    F = synth.uniform_pm1(18, (9, 4, 3, 3))
    oracle.set_threads(1)
    O1, _ = oracle.conv_multi(I, F)
    oracle.set_threads(4)
    O4, _ = oracle.conv_multi(I, F)
    assert np.array_equal(O1, O4)


@pytest.mark.parametrize("ishape,fshape", [((1, 3, 3), (1, 1, 4, 4)), ((2, 5, 5), (1, 3, 3, 3)),
                                           ((1, 5, 2), (1, 1, 3, 3))])
def test_shape_errors(ishape, fshape):
    with pytest.raises(ValueError):
        oracle.conv_multi(np.zeros(ishape, np.float32), np.zeros(fshape, np.float32))


def test_output_shape_and_degenerate_sizes():
    # K == Wx == Wy is legal (1x1 output); ragged Wx != Wy
    O, _ = oracle.conv_multi(np.ones((2, 3, 3), np.float32), np.ones((5, 2, 3, 3), np.float32))
    assert O.shape == (5, 1, 1) and np.all(O == 18)
    O, _ = oracle.conv_multi(np.ones((1, 4, 9), np.float32), np.ones((2, 1, 4, 4), np.float32))
    assert O.shape == (2, 1, 6)


def test_generator_is_deterministic_and_in_range():
    a = synth.uniform01(1, (1000,))
    b = synth.uniform01(1, (1000,))
    assert np.array_equal(a, b) and a.min() >= 0 and a.max() < 1
    f = synth.uniform_pm1(2, (1000,))
    assert f.min() >= -1 and f.max() < 1 and abs(float(f.mean())) < 0.1
    s = synth.small_ints(3, (1000,))
    assert set(np.unique(s).tolist()) <= set(range(-3, 4))
    # splitmix64 reference value (Vigna's splitmix64.c, seed 0 -> first output)
    assert int(synth.splitmix64(0, 1)[0]) == 0xE220A8397B1DCDAF
