"""fp32 CPU restatement of the executed multimodal model -- TEST INFRASTRUCTURE ONLY.

Parity status: UNPINNED against the reference for logits -- /root/reference ships no
model code; the paper's numerics lived in FlashAttention/FlashInfer,
which are not vendored.  This module is the builder's own restatement, written
independently of the CUDA path, and is the numeric checker for it.

What it restates (and the reference hooks it plugs under):
  * vision tower per image: patch conv (3 x p x p, CLIP mean/std normalisation),
    [CLS] + learned positions, pre-LN, pre-norm transformer layers (LN -> QKV+bias ->
    softmax attention -> O+bias -> residual, LN -> FC1+bias -> QuickGELU -> FC2+bias ->
    residual), then the projector (Linear-GELU-Linear; 2x2 merger with LN when merge=2).
    This is the work ``vision_work`` prices (model_cost.py:151-168).
  * language tower per request with its own contiguous fp32 KV cache: RMSNorm ->
    QKV (+bias) -> RoPE (rotate-half, inv_freq = theta^(-2i/d)) -> causal attention over
    the cached prefix -> O -> residual, RMSNorm -> SwiGLU FFN -> residual; final RMSNorm
    and lm_head on the rows that emit a token.  Chunked prefill follows the window
    ``[prefill_done, prefill_done + chunk)`` the scheduler hands out (engine.py:366,397),
    decode follows ``(rid, kv_len)`` entries (engine.py:355-361).  This is the work
    ``language_work`` prices (model_cost.py:171-197).
  * the merged sequence of a request is [visual tokens of its images in order] + [prompt
    tokens] (workload.py:91-101 only counts them; the order is the builder's choice).
"""

from __future__ import annotations

import math
import time
from typing import Dict, List, Sequence, Tuple

import numpy as np
import torch

from .synth import uniform_tensor

_QB = 1024  # attention query block (rows per score matrix)

CLIP_MEAN = np.array([0.48145466, 0.4578275, 0.40821073], dtype=np.float32)
CLIP_STD = np.array([0.26862954, 0.26130258, 0.27577711], dtype=np.float32)


def _ln(x, w, b, eps):
    mu = x.mean(-1, keepdim=True)
    var = ((x - mu) ** 2).mean(-1, keepdim=True)
    return (x - mu) / torch.sqrt(var + eps) * w + b


def _rms(x, w, eps):
    return x / torch.sqrt((x * x).mean(-1, keepdim=True) + eps) * w


def _quick_gelu(x):
    return x * torch.sigmoid(1.702 * x)


def _gelu(x):
    return 0.5 * x * (1.0 + torch.erf(x / math.sqrt(2.0)))


class OracleMLLM:
    """Weights are regenerated from the same (seed, tensor name) hash as the device."""

    _weights_cache: Dict = {}

    def __init__(self, shape: Dict, specs: Sequence, seed: int = 0):
        self.s = dict(shape)
        self.seed = seed
        # the synthesised weights are immutable: share them between oracle instances of
        # the same (shape, seed) -- a full-width 7B layer pair takes a while to hash out
        key = (tuple(sorted(self.s.items())), seed)
        w = OracleMLLM._weights_cache.get(key)
        if w is None:
            w = {}
            for sp in specs:
                arr = uniform_tensor(seed, sp.tensor_id, sp.rows, sp.cols, sp.scale, sp.offset)
                t = torch.from_numpy(arr)
                w[sp.name] = t[0] if sp.rows == 1 else t
            OracleMLLM._weights_cache.clear()  # keep at most one model resident
            OracleMLLM._weights_cache[key] = w
        self.w: Dict[str, torch.Tensor] = w
        self.kv: Dict[str, List[Tuple[torch.Tensor, torch.Tensor]]] = {}
        self.image_rows: Dict[str, torch.Tensor] = {}
        self.layer_s = {"vit": 0.0, "lang": 0.0}  # time inside the layer loops (timing only)

    @classmethod
    def random_for_timing(cls, shape: Dict, specs: Sequence, seed: int = 0) -> "OracleMLLM":
        """Same architecture with torch-random weights (fast to build); used only to time
        the CPU baseline, never as a parity reference."""
        o = cls.__new__(cls)
        o.s = dict(shape)
        o.seed = seed
        g = torch.Generator().manual_seed(seed)
        o.w = {}
        for sp in specs:
            t = (torch.rand(sp.rows, sp.cols, generator=g) * 2 - 1) * sp.scale + sp.offset
            o.w[sp.name] = t[0] if sp.rows == 1 else t
        o.kv = {}
        o.image_rows = {}
        o.layer_s = {"vit": 0.0, "lang": 0.0}
        return o

    # ------------------------------------------------------------------ vision
    def im2col(self, pixels: np.ndarray, gh: int, gw: int) -> torch.Tensor:
        p = self.s["patch"]
        x = pixels.astype(np.float32) * np.float32(1.0 / 255.0)
        x = (x - CLIP_MEAN) / CLIP_STD                      # [H, W, 3]
        x = x.reshape(gh, p, gw, p, 3).transpose(0, 2, 4, 1, 3)  # gh, gw, c, ky, kx
        x = x.reshape(gh, gw, 3 * p * p)
        if self.s["merge"] == 2:
            x = x.reshape(gh // 2, 2, gw // 2, 2, -1).transpose(0, 2, 1, 3, 4)
        return torch.from_numpy(np.ascontiguousarray(x.reshape(-1, 3 * p * p)))

    def encode_image(self, pixels: np.ndarray, gh: int, gw: int) -> torch.Tensor:
        s, w = self.s, self.w
        eps = s["ln_eps"]
        Hv, nh = s["v_hidden"], s["v_heads"]
        d = Hv // nh
        x = self.im2col(pixels, gh, gw) @ w["vis.w_patch"].T
        if s["cls"]:
            x = torch.cat([w["vis.cls_emb"][None], x], 0)
        n = x.shape[0]
        # learned positions; tokens beyond the table (images larger than the tower's native
        # 577-token grid, e.g. the 2.9k-token stress images) reuse the last position
        pidx = torch.clamp(torch.arange(n), max=w["vis.pos_emb"].shape[0] - 1)
        x = x + w["vis.pos_emb"][pidx]
        if s["pre_ln"]:
            x = _ln(x, w["vis.pre_ln_w"], w["vis.pre_ln_b"], eps)
        t0 = time.perf_counter()
        for l in range(s["v_layers"]):
            p = f"vis.{l}."
            t = _ln(x, w[p + "ln1_w"], w[p + "ln1_b"], eps)
            qkv = t @ w[p + "w_qkv"].T + w[p + "b_qkv"]
            q, k, v = qkv.split(Hv, -1)
            q = q.view(n, nh, d).transpose(0, 1)
            k = k.view(n, nh, d).transpose(0, 1)
            v = v.view(n, nh, d).transpose(0, 1)
            a = torch.cat([torch.softmax(q[:, i:i + _QB] @ k.transpose(1, 2) / math.sqrt(d),
                                         -1) @ v for i in range(0, n, _QB)], 1)
            a = a.transpose(0, 1).reshape(n, Hv)
            x = x + a @ w[p + "w_o"].T + w[p + "b_o"]
            t = _ln(x, w[p + "ln2_w"], w[p + "ln2_b"], eps)
            f = _quick_gelu(t @ w[p + "w_fc1"].T + w[p + "b_fc1"])
            x = x + f @ w[p + "w_fc2"].T + w[p + "b_fc2"]
        self.layer_s["vit"] += time.perf_counter() - t0
        if s["merge"] == 1:
            v = x[1:] if s["cls"] else x
        else:
            v = _ln(x, w["vis.merge_ln_w"], w["vis.merge_ln_b"], eps).reshape(n // 4, 4 * Hv)
        h = _gelu(v @ w["proj.w1"].T + w["proj.b1"])
        return h @ w["proj.w2"].T + w["proj.b2"]

    def add_image_rows(self, rid: str, rows: torch.Tensor) -> None:
        prev = self.image_rows.get(rid)
        self.image_rows[rid] = rows if prev is None else torch.cat([prev, rows], 0)

    # ------------------------------------------------------------------ language
    def _rope(self, x: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
        d = x.shape[-1]
        half = d // 2
        inv = 1.0 / (self.s["rope_theta"] ** (torch.arange(0, half, dtype=torch.float32) * 2 / d))
        ang = pos.to(torch.float32)[:, None] * inv[None]
        c, sn = torch.cos(ang)[:, None], torch.sin(ang)[:, None]
        x1, x2 = x[..., :half], x[..., half:]
        return torch.cat([x1 * c - x2 * sn, x2 * c + x1 * sn], -1)

    def forward_rows(self, rid: str, x: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
        """Run rows of one request at positions ``pos`` (contiguous, appended to its
        cache); returns the final hidden states [n, H]."""
        s, w = self.s, self.w
        H, nh, nkv = s["hidden"], s["n_heads"], s["n_kv_heads"]
        d = H // nh
        g = nh // nkv
        F = s["ffn"]
        eps = s["rms_eps"]
        n = x.shape[0]
        cache = self.kv.setdefault(rid, [(torch.zeros(0, nkv, d), torch.zeros(0, nkv, d))
                                         for _ in range(s["n_layers"])])
        t0 = time.perf_counter()
        for l in range(s["n_layers"]):
            p = f"lang.{l}."
            t = _rms(x, w[p + "attn_norm"], eps)
            qkv = t @ w[p + "w_qkv"].T
            if s["qkv_bias"]:
                qkv = qkv + w[p + "b_qkv"]
            q = qkv[:, :nh * d].view(n, nh, d)
            k = qkv[:, nh * d:(nh + nkv) * d].view(n, nkv, d)
            v = qkv[:, (nh + nkv) * d:].view(n, nkv, d)
            q = self._rope(q, pos)
            k = self._rope(k, pos)
            K = torch.cat([cache[l][0], k], 0)
            V = torch.cat([cache[l][1], v], 0)
            cache[l] = (K, V)
            L = K.shape[0]
            Kx = K.repeat_interleave(g, 1).transpose(0, 1)   # nh, L, d
            Vx = V.repeat_interleave(g, 1).transpose(0, 1)
            kpos = torch.arange(L)
            qt = q.transpose(0, 1)
            parts = []
            for i in range(0, n, _QB):  # query blocks bound the score matrix's memory
                sc = qt[:, i:i + _QB] @ Kx.transpose(1, 2) / math.sqrt(d)  # nh, b, L
                mask = kpos[None, :] > pos[i:i + _QB, None]
                sc = sc.masked_fill(mask[None], float("-inf"))
                parts.append(torch.softmax(sc, -1) @ Vx)
            a = torch.cat(parts, 1).transpose(0, 1).reshape(n, nh * d)
            x = x + a @ w[p + "w_o"].T
            t = _rms(x, w[p + "ffn_norm"], eps)
            gu = t @ w[p + "w_gate_up"].T
            x = x + (torch.nn.functional.silu(gu[:, :F]) * gu[:, F:]) @ w[p + "w_down"].T
        self.layer_s["lang"] += time.perf_counter() - t0
        return x

    def logits(self, h: torch.Tensor) -> torch.Tensor:
        return _rms(h, self.w["lang.final_norm"], self.s["rms_eps"]) @ self.w["lang.lm_head"].T

    def prefill_chunk(self, rid: str, prompt: np.ndarray, n_visual: int, offset: int,
                      chunk: int) -> torch.Tensor:
        """Window [offset, offset+chunk) of [visual rows] + [prompt]; returns the logits
        of the window's last row."""
        emb = self.w["lang.embed"]
        rows = []
        for t in range(offset, offset + chunk):
            if t < n_visual:
                rows.append(self.image_rows[rid][t])
            else:
                rows.append(emb[int(prompt[t - n_visual])])
        x = torch.stack(rows)
        pos = torch.arange(offset, offset + chunk)
        h = self.forward_rows(rid, x, pos)
        return self.logits(h[-1:])[0]

    def decode(self, rid: str, token: int, kv_len: int) -> torch.Tensor:
        assert self.kv[rid][0][0].shape[0] == kv_len, "oracle cache out of step"
        x = self.w["lang.embed"][int(token)][None]
        h = self.forward_rows(rid, x, torch.tensor([kv_len]))
        return self.logits(h)[0]

    def drop(self, rid: str) -> None:
        self.kv.pop(rid, None)
        self.image_rows.pop(rid, None)
