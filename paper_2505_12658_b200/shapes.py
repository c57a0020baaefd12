"""Model shapes executed on the GPU.

epdsim's ``ModelProfile`` (model_cost.py:31-63) carries only the dimensions its
roofline needs (hidden sizes, head counts, layer counts, kv_head_ratio).  A real
executor needs the rest of the architecture; ``MllmShape`` is that completion, and
``MllmShape.profile()`` gives back the exact ``ModelProfile`` the reference scheduler
is built with, so the scheduler and the executor always describe the same model.

Presets (BASELINE.json configs):
  tiny          config 1: ModelProfile(512, 4, 2, 256, 4, 2), the oracle-sized model
  llava-1.5-7b  config 2/4/5: CLIP ViT-L/14-336 (1024 / 16 heads / 24 layers, [CLS] + 576
                patches, pre-LN, QuickGELU) + 2-layer GELU projector + Llama-2-7B
                (4096 / 32 heads / 32 layers, SwiGLU 11008, vocab 32000)
  qwen2-vl-7b   config 3: 1280 / 16 heads (d 80) / 32 layer ViT with a 2x2 patch merger,
                Qwen2-7B decoder (3584 / 28 q heads / 4 kv heads / 28 layers, 18944 FFN,
                vocab 152064, qkv bias).  Shape-faithful; the vision tower uses learned
                absolute positions instead of 2-D RoPE and the decoder 1-D RoPE instead of
                M-RoPE.
"""

from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass

from ._epdsim import MC


def _ffn_default(hidden: int) -> int:
    return int(math.ceil(8 * hidden / 3 / 128) * 128)


@dataclass(frozen=True)
class MllmShape:
    name: str
    # language tower
    hidden: int
    n_heads: int
    n_kv_heads: int
    n_layers: int
    ffn: int
    vocab: int
    rope_theta: float
    rms_eps: float
    qkv_bias: bool
    # vision tower
    v_hidden: int
    v_heads: int
    v_layers: int
    v_mlp: int
    patch: int
    cls: bool
    pre_ln: bool
    merge: int
    proj_hidden: int
    max_pos: int
    ln_eps: float = 1e-5

    @property
    def head_dim(self) -> int:
        return self.hidden // self.n_heads

    @property
    def v_head_dim(self) -> int:
        return self.v_hidden // self.v_heads

    @property
    def qkv_cols(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    @property
    def k_patch(self) -> int:
        return 3 * self.patch * self.patch

    @property
    def k_pad(self) -> int:
        return int(math.ceil(self.k_patch / 64) * 64)

    @property
    def kv_bytes_per_token(self) -> int:
        return 2 * self.n_kv_heads * self.head_dim * self.n_layers * 2

    @property
    def kv_block_elems(self) -> int:
        return self.n_layers * 2 * self.n_kv_heads * MC.KV_BLOCK_TOKENS * self.head_dim

    @property
    def kv_layer_elems(self) -> int:
        return 2 * self.n_kv_heads * MC.KV_BLOCK_TOKENS * self.head_dim

    @property
    def image_block_elems(self) -> int:
        return MC.IMAGE_BLOCK_TOKENS * self.hidden

    def profile(self):
        """The epdsim ModelProfile the scheduler and the oracle clock use."""
        return MC.ModelProfile(
            lang_hidden=self.hidden, lang_heads=self.n_heads, lang_layers=self.n_layers,
            vision_hidden=self.v_hidden, vision_heads=self.v_heads,
            vision_layers=self.v_layers, kv_head_ratio=self.n_kv_heads / self.n_heads,
            dtype_bytes=2)

    def vit_tokens(self, visual_tokens: int) -> int:
        """ViT sequence length of an image yielding ``visual_tokens`` LLM tokens."""
        return visual_tokens * self.merge * self.merge + (1 if self.cls else 0)

    def patch_grid(self, visual_tokens: int):
        """(gh, gw) patch grid of an image with ``visual_tokens`` output tokens.

        The reference traces carry only token counts (workload.py:104-126); the grid
        is the most square factorisation, scaled by the merge factor."""
        t = visual_tokens
        th = int(math.isqrt(t))
        while t % th:
            th -= 1
        return th * self.merge, (t // th) * self.merge

    def asdict(self) -> dict:
        return dataclasses.asdict(self)

    def weight_bytes(self) -> int:
        H, F, V = self.hidden, self.ffn, self.vocab
        lang = self.n_layers * (H * self.qkv_cols + self.n_heads * self.head_dim * H + 2 * F * H
                                + F * H + 2 * H) + 2 * V * H + H
        Hv = self.v_hidden
        vis = self.v_layers * (4 * Hv * Hv + 2 * Hv * self.v_mlp + 10 * Hv) + Hv * self.k_pad
        vis += self.max_pos * Hv + self.proj_hidden * Hv * self.merge ** 2 + H * self.proj_hidden
        return 2 * (lang + vis)


PRESETS = {
    "tiny": MllmShape(
        name="tiny", hidden=512, n_heads=4, n_kv_heads=4, n_layers=2, ffn=_ffn_default(512),
        vocab=32000, rope_theta=10000.0, rms_eps=1e-5, qkv_bias=False,
        v_hidden=256, v_heads=4, v_layers=2, v_mlp=1024, patch=14, cls=True, pre_ln=True,
        merge=1, proj_hidden=512, max_pos=577),
    "llava-1.5-7b": MllmShape(
        name="llava-1.5-7b", hidden=4096, n_heads=32, n_kv_heads=32, n_layers=32,
        ffn=11008, vocab=32000, rope_theta=10000.0, rms_eps=1e-5, qkv_bias=False,
        v_hidden=1024, v_heads=16, v_layers=24, v_mlp=4096, patch=14, cls=True, pre_ln=True,
        merge=1, proj_hidden=4096, max_pos=577),
    "qwen2-vl-7b": MllmShape(
        name="qwen2-vl-7b", hidden=3584, n_heads=28, n_kv_heads=4, n_layers=28, ffn=18944,
        vocab=152064, rope_theta=1000000.0, rms_eps=1e-6, qkv_bias=True,
        v_hidden=1280, v_heads=16, v_layers=32, v_mlp=5120, patch=14, cls=False, pre_ln=False,
        merge=2, proj_hidden=5120, max_pos=16384, ln_eps=1e-6),
}


def get_shape(name: str) -> MllmShape:
    if name not in PRESETS:
        raise KeyError(f"unknown model shape {name!r}; known: {sorted(PRESETS)}")
    return PRESETS[name]


def with_layers(shape: MllmShape, n_layers: int = None, v_layers: int = None) -> MllmShape:
    """A depth-reduced copy (used only by parity tests that sample a 7B shape)."""
    return dataclasses.replace(shape, n_layers=n_layers or shape.n_layers,
                               v_layers=v_layers or shape.v_layers)
