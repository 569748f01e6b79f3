"""B200-native (sm_100a) hot path of arXiv 2212.00404: direct valid-mode,
stride-1 convolution (§2.1 Eq. 1/Eq. 2), single- and multi-channel.

    from paper_2212_00404_b200 import conv
    O = conv.single(I, F)                 # KS, FP32 CUDA cores
    O = conv.multi(I, F, "tf32")          # KM-TC, tcgen05 / TMEM
    O = conv.multi(I, F, "fp32")          # KM-SIMT, strict FP32

C ABI: include/b200conv.h (libb200conv.so).  Multi-GPU filter sharding:
paper_2212_00404_b200.shard.
"""
from . import conv  # noqa: F401

__all__ = ["conv"]
