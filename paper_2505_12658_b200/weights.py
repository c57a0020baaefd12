"""Random-init device weights and the C structs that describe them.

There are no checkpoints offline (BASELINE.json: "random-init bf16").  Every tensor is
synthesised on the device by ``hy_fill_uniform_bf16`` from a counter hash of
``(seed, tensor id, logical index)``; ``oracle/synth.py`` restates the same hash in
numpy, so the CPU oracle rebuilds bit-identical weights without a device copy.

``weight_specs(shape)`` is the single list of tensors (name, logical shape, physical
row stride, scale, offset, layout permutation) both sides consume.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Dict, List

import torch

from . import _lib
from .inputs import fnv1a64
from .shapes import MllmShape

W_SCALE = 0.035     # uniform(-a, a) with std ~0.02 (HF initializer_range)
B_SCALE = 0.02      # biases
NORM_SCALE = 0.1    # norm gains = 1 +- 0.1


@dataclass(frozen=True)
class WeightSpec:
    name: str
    rows: int
    cols: int
    ld: int          # physical row stride (>= cols; zero padded)
    scale: float
    offset: float
    perm: int        # 0 dense, 1 SwiGLU 16-row interleave of [gate; up]

    @property
    def tensor_id(self) -> int:
        return fnv1a64(self.name)


def weight_specs(s: MllmShape) -> List[WeightSpec]:
    H, D, F = s.hidden, s.head_dim, s.ffn
    out: List[WeightSpec] = []

    def w(name, rows, cols, scale=W_SCALE, offset=0.0, perm=0, ld=None):
        out.append(WeightSpec(name, rows, cols, ld or cols, scale, offset, perm))

    # language tower
    w("lang.embed", s.vocab, H)
    for l in range(s.n_layers):
        p = f"lang.{l}."
        w(p + "attn_norm", 1, H, NORM_SCALE, 1.0)
        w(p + "w_qkv", s.qkv_cols, H)
        if s.qkv_bias:
            w(p + "b_qkv", 1, s.qkv_cols, B_SCALE)
        w(p + "w_o", H, s.n_heads * D)
        w(p + "ffn_norm", 1, H, NORM_SCALE, 1.0)
        w(p + "w_gate_up", 2 * F, H, perm=1)
        w(p + "w_down", H, F)
    w("lang.final_norm", 1, H, NORM_SCALE, 1.0)
    w("lang.lm_head", s.vocab, H)
    # vision tower
    Hv = s.v_hidden
    w("vis.w_patch", Hv, s.k_patch, ld=s.k_pad)
    if s.cls:
        w("vis.cls_emb", 1, Hv)
    w("vis.pos_emb", s.max_pos, Hv)
    if s.pre_ln:
        w("vis.pre_ln_w", 1, Hv, NORM_SCALE, 1.0)
        w("vis.pre_ln_b", 1, Hv, B_SCALE)
    for l in range(s.v_layers):
        p = f"vis.{l}."
        w(p + "ln1_w", 1, Hv, NORM_SCALE, 1.0)
        w(p + "ln1_b", 1, Hv, B_SCALE)
        w(p + "w_qkv", 3 * Hv, Hv)
        w(p + "b_qkv", 1, 3 * Hv, B_SCALE)
        w(p + "w_o", Hv, Hv)
        w(p + "b_o", 1, Hv, B_SCALE)
        w(p + "ln2_w", 1, Hv, NORM_SCALE, 1.0)
        w(p + "ln2_b", 1, Hv, B_SCALE)
        w(p + "w_fc1", s.v_mlp, Hv)
        w(p + "b_fc1", 1, s.v_mlp, B_SCALE)
        w(p + "w_fc2", Hv, s.v_mlp)
        w(p + "b_fc2", 1, Hv, B_SCALE)
    if s.merge == 2:
        w("vis.merge_ln_w", 1, Hv, NORM_SCALE, 1.0)
        w("vis.merge_ln_b", 1, Hv, B_SCALE)
    w("proj.w1", s.proj_hidden, Hv * s.merge * s.merge)
    w("proj.b1", 1, s.proj_hidden, B_SCALE)
    w("proj.w2", H, s.proj_hidden)
    w("proj.b2", 1, H, B_SCALE)
    return out


class DeviceWeights:
    """All weights of one model replica on one device, plus its C descriptors."""

    def __init__(self, shape: MllmShape, device: torch.device, seed: int = 0):
        self.shape = shape
        self.device = torch.device(device)
        self.seed = seed
        self.tensors: Dict[str, torch.Tensor] = {}
        lib = _lib.load()
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device).cuda_stream
            for sp in weight_specs(shape):
                t = torch.empty((sp.rows, sp.ld), dtype=torch.bfloat16, device=self.device)
                _lib.check(lib.hy_fill_uniform_bf16(
                    t.data_ptr(), sp.rows, sp.cols, sp.ld, seed & 0xFFFFFFFFFFFFFFFF,
                    sp.tensor_id, sp.scale, sp.offset, sp.perm, stream), sp.name)
                self.tensors[sp.name] = t
            torch.cuda.synchronize(self.device)
        self._build_structs()

    def p(self, name: str) -> int:
        t = self.tensors.get(name)
        return 0 if t is None else t.data_ptr()

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.tensors.values())

    def _build_structs(self) -> None:
        s = self.shape
        L = _lib
        self._lang_layers = (L.HyLangLayerW * s.n_layers)()
        for l in range(s.n_layers):
            pre = f"lang.{l}."
            self._lang_layers[l] = L.HyLangLayerW(
                self.p(pre + "attn_norm"), self.p(pre + "w_qkv"), self.p(pre + "b_qkv"),
                self.p(pre + "w_o"), self.p(pre + "ffn_norm"), self.p(pre + "w_gate_up"),
                self.p(pre + "w_down"))
        self.lang = L.HyLangModel(
            s.hidden, s.n_heads, s.n_kv_heads, s.head_dim, s.n_layers, s.ffn, s.vocab,
            s.rope_theta, s.rms_eps, self.p("lang.embed"), self.p("lang.final_norm"),
            self.p("lang.lm_head"),
            ctypes.cast(self._lang_layers, ctypes.POINTER(L.HyLangLayerW)))
        self._vit_layers = (L.HyVitLayerW * s.v_layers)()
        for l in range(s.v_layers):
            pre = f"vis.{l}."
            self._vit_layers[l] = L.HyVitLayerW(*[self.p(pre + n) for n in (
                "ln1_w", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o", "ln2_w", "ln2_b", "w_fc1",
                "b_fc1", "w_fc2", "b_fc2")])
        self.vit = L.HyVitModel(
            s.v_hidden, s.v_heads, s.v_head_dim, s.v_layers, s.v_mlp, s.patch, s.k_pad,
            int(s.cls), int(s.pre_ln), s.merge, s.hidden, s.proj_hidden, s.max_pos, s.ln_eps,
            self.p("vis.w_patch"), self.p("vis.cls_emb"), self.p("vis.pos_emb"),
            self.p("vis.pre_ln_w"), self.p("vis.pre_ln_b"),
            ctypes.cast(self._vit_layers, ctypes.POINTER(L.HyVitLayerW)),
            self.p("vis.merge_ln_w"), self.p("vis.merge_ln_b"), self.p("proj.w1"),
            self.p("proj.b1"), self.p("proj.w2"), self.p("proj.b2"))
