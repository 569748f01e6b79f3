"""CPU oracle for arXiv 2212.00404's hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` leg may import this package.  The product package
``paper_2212_00404_b200`` never imports it, and it never imports the product:
the two share no code (the seeded input generator lives in ``synth.py``, which
holds none of the method's arithmetic).

The arithmetic lives in ``conv_oracle.c`` (plain C, fp64 accumulation, no
blocking or reordering): Eq. 1 of PAPER.md §2.1, single-channel
Eq. 2 as its C = 1 case.  This module only compiles it with gcc
(``-O2 -fopenmp -ffp-contract=off``, no fast-math) and marshals numpy arrays.

Parity pins (``tests/test_oracle.py``, ``-m "not gpu"``): hand-worked golden
examples P1-P3 (``tests/golden/``), delta-filter and all-ones closed forms
(P4, P5), K=1 == matrix product and K=Wx=Wy == dot product (P6, P7),
torch float64 conv2d (P8), linearity / channel-sum / shard invariants (P9) and
integer exactness (P10).  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "conv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile conv_oracle.c into liboracle.so (idempotent)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call([
            "gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
            "-fPIC", "-shared", "-o", tmp, _SRC, "-lm",
        ])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            dp = ctypes.POINTER(ctypes.c_double)
            fp = ctypes.POINTER(ctypes.c_float)
            lib.oracle_conv.argtypes = [fp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        fp, ctypes.c_int, ctypes.c_int, dp, dp]
            lib.oracle_conv.restype = ctypes.c_int
            lib.oracle_conv_sampled.argtypes = [fp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                fp, ctypes.c_int, ctypes.c_int,
                                                ctypes.POINTER(ctypes.c_int64), ctypes.c_int64,
                                                dp, dp]
            lib.oracle_conv_sampled.restype = ctypes.c_int
            lib.oracle_set_threads.argtypes = [ctypes.c_int]
            lib.oracle_set_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def _f32(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a


def _ptr(a, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def set_threads(n: int) -> int:
    """Set the OpenMP thread count of the oracle; returns the count in effect."""
    return _load().oracle_set_threads(int(n))


def conv_multi(I, F):
    """Eq. 1: I[C][Wy][Wx] f32, F[M][C][K][K] f32 ->
    (O[M][Ho][Wo] f64, A[M][Ho][Wo] f64) with A = sum |I*F| per output."""
    I = _f32(I)
    F = _f32(F)
    if I.ndim != 3 or F.ndim != 4 or F.shape[1] != I.shape[0] or F.shape[2] != F.shape[3]:
        raise ValueError(f"shape error: I{I.shape} F{F.shape}")
    C, Wy, Wx = I.shape
    M, _, K, _ = F.shape
    if K > Wx or K > Wy or min(C, Wy, Wx, M, K) < 1:
        raise ValueError(f"shape error: K={K} > min(Wx={Wx}, Wy={Wy}) or empty dim")
    Ho, Wo = Wy - K + 1, Wx - K + 1
    O = np.empty((M, Ho, Wo), dtype=np.float64)
    A = np.empty((M, Ho, Wo), dtype=np.float64)
    rc = _load().oracle_conv(_ptr(I, ctypes.c_float), C, Wx, Wy, _ptr(F, ctypes.c_float), K, M,
                             _ptr(O, ctypes.c_double), _ptr(A, ctypes.c_double))
    if rc != 0:
        raise ValueError("oracle shape error")
    return O, A


def conv_single(I, F):
    """Eq. 2: I[Wy][Wx], F[M][K][K] -> (O[M][Ho][Wo], A) in f64."""
    I = _f32(I)
    F = _f32(F)
    if I.ndim != 2 or F.ndim != 3:
        raise ValueError(f"shape error: I{I.shape} F{F.shape}")
    return conv_multi(I[None], F[:, None])


def conv_multi_sampled(I, F, flat_idx):
    """Eq. 1 evaluated only at the flat output indices flat_idx (into O[M][Ho][Wo]).
    Same arithmetic and order as conv_multi, used at full BASELINE sizes."""
    I = _f32(I)
    F = _f32(F)
    C, Wy, Wx = I.shape
    M, _, K, _ = F.shape
    idx = np.ascontiguousarray(flat_idx, dtype=np.int64)
    O = np.empty(idx.shape[0], dtype=np.float64)
    A = np.empty(idx.shape[0], dtype=np.float64)
    rc = _load().oracle_conv_sampled(_ptr(I, ctypes.c_float), C, Wx, Wy, _ptr(F, ctypes.c_float), K, M,
                                     _ptr(idx, ctypes.c_int64), idx.shape[0],
                                     _ptr(O, ctypes.c_double), _ptr(A, ctypes.c_double))
    if rc != 0:
        raise ValueError("oracle shape error")
    return O, A
