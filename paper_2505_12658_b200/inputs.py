"""Synthetic request content.

The reference traces carry only counts per request (image token counts, prompt and
output lengths; workload.py:104-126).  A real executor needs content, so each request
gets deterministic prompt token ids and images derived from ``(seed, request id)``.
The same functions feed the CPU oracle in the parity tests, so both sides see
byte-identical inputs.

Images are uint8 HWC pixel arrays of ``gh*patch x gw*patch`` (the grid comes from
``MllmShape.patch_grid``), drawn from a small deterministic store so host-side
generation stays off the critical path.
"""

from __future__ import annotations

from typing import Dict, Tuple

import numpy as np

FNV_OFFSET = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3
STORE_SIZE = 8


def fnv1a64(text: str) -> int:
    h = FNV_OFFSET
    for b in text.encode():
        h ^= b
        h = (h * FNV_PRIME) & 0xFFFFFFFFFFFFFFFF
    return h


def prompt_tokens(seed: int, rid: str, n: int, vocab: int) -> np.ndarray:
    rng = np.random.default_rng([seed & 0xFFFFFFFF, fnv1a64(rid) & 0xFFFFFFFF, 1])
    return rng.integers(0, vocab, size=n, dtype=np.int64).astype(np.int32)


def image_store_index(seed: int, rid: str, image_idx: int) -> int:
    return fnv1a64(f"{seed}/{rid}/{image_idx}") % STORE_SIZE


class ImageStore:
    """Deterministic pixel arrays keyed by (store index, grid)."""

    def __init__(self, seed: int, patch: int):
        self.seed = seed
        self.patch = patch
        self._cache: Dict[Tuple[int, int, int], np.ndarray] = {}

    def pixels(self, index: int, gh: int, gw: int) -> np.ndarray:
        key = (index, gh, gw)
        img = self._cache.get(key)
        if img is None:
            rng = np.random.default_rng([self.seed & 0xFFFFFFFF, 7, index, gh, gw])
            img = rng.integers(0, 256, size=(gh * self.patch, gw * self.patch, 3),
                               dtype=np.uint8)
            self._cache[key] = img
        return img

    def request_image(self, rid: str, image_idx: int, gh: int, gw: int) -> np.ndarray:
        return self.pixels(image_store_index(self.seed, rid, image_idx), gh, gw)
