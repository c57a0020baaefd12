"""numpy restatement of ``hy_fill_uniform_bf16`` (csrc/gather.cu) -- TEST INFRASTRUCTURE.

value(r, c) = bf16_rne( fp32(offset) + fp32(scale) * u ),
u = float32(splitmix64(key + r*cols + c) >> 40) * 2^-23 - 1,
key = splitmix64(seed ^ splitmix64(tensor_id)).
Every step is exact or a single IEEE fp32 rounding, so the result is bit-identical
to the device kernel (checked in tests/test_oracle.py and tests/test_kernels_gpu.py).
"""

from __future__ import annotations

import numpy as np

_U64 = np.uint64


def splitmix64(x) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + _U64(0x9E3779B97F4A7C15)
        z = (x ^ (x >> _U64(30))) * _U64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> _U64(27))) * _U64(0x94D049BB133111EB)
    return z ^ (z >> _U64(31))


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 to the nearest bf16 (ties to even), returned as fp32."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    lsb = (b >> np.uint32(16)) & np.uint32(1)
    with np.errstate(over="ignore"):
        r = (b + np.uint32(0x7FFF) + lsb) & np.uint32(0xFFFF0000)
    return r.view(np.float32)


def uniform_tensor(seed: int, tensor_id: int, rows: int, cols: int, scale: float,
                   offset: float, chunk: int = 1 << 22) -> np.ndarray:
    """Logical [rows, cols] tensor (no padding, no interleave permutation)."""
    key = splitmix64(np.uint64(seed) ^ splitmix64(np.uint64(tensor_id)))
    n = rows * cols
    out = np.empty(n, dtype=np.float32)
    sc, of = np.float32(scale), np.float32(offset)
    for s in range(0, n, chunk):
        idx = np.arange(s, min(n, s + chunk), dtype=np.uint64)
        with np.errstate(over="ignore"):
            h = splitmix64(key + idx)
        u = (h >> _U64(40)).astype(np.float32) * np.float32(2.0 ** -23) - np.float32(1.0)
        out[s:s + idx.size] = bf16_round(sc * u + of)
    return out.reshape(rows, cols)


def swiglu_physical_rows(rows: int) -> np.ndarray:
    """Logical row held by each physical row of a SwiGLU-interleaved [gate; up]."""
    pr = np.arange(rows)
    g, j = pr // 32, pr % 32
    return np.where(j < 16, 16 * g + j, rows // 2 + 16 * g + (j - 16))
