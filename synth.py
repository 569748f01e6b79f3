"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds none of the convolution's arithmetic: it only draws numbers.
Both ``oracle/`` (via tests / bench) and the GPU path are fed the identical
float32 arrays produced here, so no expected value ever comes from the CUDA
path.  Generator: splitmix64 (counter-based, Steele et al. 2014) -> top 24
bits -> uniform k / 2^24, exactly representable in float32.

Recipe:
  * I ~ U[0, 1)   (post-ReLU activations / normalised pixels of the CNN layers
                   the paper evaluates, §4)
  * F ~ U[-1, 1)
  * seed_I = 0x2212, seed_F = 0x0404 + config index
  * stress sets: all-positive F ~ U[0,1) (worst-case tolerance), small integers
    in {-3..3} (exactness pin P10), zeros / deltas only for closed forms.
"""
from __future__ import annotations

import numpy as np

SEED_I = 0x2212
SEED_F = 0x0404

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """n outputs of splitmix64 seeded with `seed`, counters offset..offset+n-1."""
    with np.errstate(over="ignore"):
        i = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, shape) -> np.ndarray:
    """float32 in [0,1): k / 2^24 with k the top 24 bits of splitmix64."""
    n = int(np.prod(shape)) if len(shape) else 1
    k = (splitmix64(seed, n) >> np.uint64(40)).astype(np.int64)
    return (k.astype(np.float32) * np.float32(1.0 / 16777216.0)).reshape(shape)


def uniform_pm1(seed: int, shape) -> np.ndarray:
    """float32 in [-1,1): (2k - 2^24) / 2^24, exact in float32."""
    n = int(np.prod(shape)) if len(shape) else 1
    k = (splitmix64(seed, n) >> np.uint64(40)).astype(np.int64)
    return ((2 * k - 16777216).astype(np.float32) * np.float32(1.0 / 16777216.0)).reshape(shape)


def small_ints(seed: int, shape, lo: int = -3, hi: int = 3) -> np.ndarray:
    """float32 integers uniform in {lo..hi} (exactness stress set, pin P10)."""
    n = int(np.prod(shape)) if len(shape) else 1
    k = (splitmix64(seed, n) >> np.uint64(33)).astype(np.int64)
    return (lo + (k % (hi - lo + 1))).astype(np.float32).reshape(shape)


def layer_inputs(C: int, Wx: int, Wy: int, K: int, M: int, cfg_index: int = 0,
                 kind: str = "default"):
    """(I[C][Wy][Wx], F[M][C][K][K]) float32 for one layer.

    kind: "default" (I~U[0,1), F~U[-1,1)), "positive" (F~U[0,1)),
          "ints" (both in {-3..3})."""
    sI, sF = SEED_I, SEED_F + cfg_index
    if kind == "default":
        return uniform01(sI, (C, Wy, Wx)), uniform_pm1(sF, (M, C, K, K))
    if kind == "positive":
        return uniform01(sI, (C, Wy, Wx)), uniform01(sF, (M, C, K, K))
    if kind == "ints":
        return small_ints(sI, (C, Wy, Wx)), small_ints(sF, (M, C, K, K))
    raise ValueError(kind)


# ----------------------------------------------------------------------------
# The BASELINE.json configurations (workload shapes of PAPER.md §4).
# ----------------------------------------------------------------------------
PR1 = dict(name="single_pr1_32x32_k3_m4", C=1, Wx=32, Wy=32, K=3, M=4)

SINGLE_SWEEP = [
    dict(name=f"single_{w}x{w}_k{k}_m{m}", C=1, Wx=w, Wy=w, K=k, M=m)
    for w in (7, 14, 28, 56, 224) for k in (1, 3, 5, 7) for m in (32, 64, 128, 256)
]

MULTI_LAYERS = [
    dict(name="resnet_28x28_c128_m128_k3", C=128, Wx=28, Wy=28, K=3, M=128),
    dict(name="resnet_14x14_c256_m256_k3", C=256, Wx=14, Wy=14, K=3, M=256),
    dict(name="resnet_7x7_c512_m512_k3", C=512, Wx=7, Wy=7, K=3, M=512),
    dict(name="vgg_224x224_c3_m64_k3", C=3, Wx=224, Wy=224, K=3, M=64),
    dict(name="vgg_56x56_c64_m64_k3", C=64, Wx=56, Wy=56, K=3, M=64),
    dict(name="alexnet_27x27_c96_m256_k5", C=96, Wx=27, Wy=27, K=5, M=256),
    # "the 28x28x256 layer" of north_star
    dict(name="target_28x28_c256_m256_k3", C=256, Wx=28, Wy=28, K=3, M=256),
]

SHARD_SWEEP = dict(name="sweep_14x14_c512_m4096_k3", C=512, Wx=14, Wy=14, K=3, M=4096)
