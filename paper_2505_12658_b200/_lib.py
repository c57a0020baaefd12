"""ctypes binding of libhydra_sm100.so (the C ABI declared in include/hydra_sm100.h).

The library is built in-tree by ``__graft_entry__.build()`` / ``make -C csrc``.
There is no fallback: if the shared object is missing or a call fails, an error is
raised.  Only plain pointers, ints and the POD structs below cross the boundary.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, Structure, c_char_p, c_float, c_int, c_int64, c_longlong,
                    c_size_t, c_uint64, c_ulonglong, c_void_p)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libhydra_sm100.so")
# lab variants (tools/lab: the same sources built with other compile-time budgets) are loaded
# through HY_LIB_PATH; they are still this library, never a fallback
LIB_PATH = os.environ.get("HY_LIB_PATH", LIB_PATH)

HY_ACT_NONE = 0
HY_ACT_QUICK_GELU = 1
HY_ACT_GELU = 2
HY_ACT_SILU = 3
HY_ACT_SWIGLU = 4
HY_TOK_FROM_LAST = -2147483648
KV_BLOCK_TOKENS = 16
IMAGE_BLOCK_TOKENS = 576


class HyError(RuntimeError):
    """A libhydra_sm100 entry point returned a CUDA error code."""


class HyGemmEpilogue(Structure):
    _fields_ = [("bias", c_void_p), ("residual", c_void_p), ("ldr", c_int), ("act", c_int),
                ("row_map", c_void_p), ("out", c_void_p), ("ldc", c_int), ("out_f32", c_int)]


class HyImageDesc(Structure):
    _fields_ = [("pixels", c_void_p), ("row_stride", c_int), ("gh", c_int), ("gw", c_int),
                ("tok_start", c_int), ("patch_start", c_int), ("vis_start", c_int),
                ("pad_", c_int)]


class HyLangLayerW(Structure):
    _fields_ = [("attn_norm", c_void_p), ("w_qkv", c_void_p), ("b_qkv", c_void_p),
                ("w_o", c_void_p), ("ffn_norm", c_void_p), ("w_gate_up", c_void_p),
                ("w_down", c_void_p)]


class HyLangModel(Structure):
    _fields_ = [("hidden", c_int), ("n_heads", c_int), ("n_kv_heads", c_int),
                ("head_dim", c_int), ("n_layers", c_int), ("ffn", c_int), ("vocab", c_int),
                ("rope_theta", c_float), ("rms_eps", c_float), ("embed", c_void_p),
                ("final_norm", c_void_p), ("lm_head", c_void_p),
                ("layers", POINTER(HyLangLayerW))]


class HyKvCache(Structure):
    _fields_ = [("base", c_void_p), ("block_stride", c_longlong), ("layer_stride", c_longlong),
                ("num_blocks", c_int), ("block_table", c_void_p), ("bt_stride", c_int)]


class HyLangBatch(Structure):
    _fields_ = [("n_rows", c_int), ("n_decode", c_int), ("n_prefill", c_int),
                ("tok", c_void_p), ("pos", c_void_p), ("row_slot", c_void_p),
                ("dec_ctx", c_void_p), ("pf_qstart", c_void_p), ("pf_offset", c_void_p),
                ("pf_slot", c_void_p), ("pf_max_q", c_int), ("max_ctx", c_int),
                ("n_out", c_int), ("out_rows", c_void_p), ("out_slot", c_void_p),
                ("out_tokens", c_void_p), ("out_logits", c_void_p)]


class HyVitLayerW(Structure):
    _fields_ = [(n, c_void_p) for n in ("ln1_w", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o",
                                        "ln2_w", "ln2_b", "w_fc1", "b_fc1", "w_fc2", "b_fc2")]


class HyVitModel(Structure):
    _fields_ = [("hidden", c_int), ("n_heads", c_int), ("head_dim", c_int), ("n_layers", c_int),
                ("mlp", c_int), ("patch", c_int), ("k_pad", c_int), ("cls", c_int),
                ("pre_ln", c_int), ("merge", c_int), ("lang_hidden", c_int),
                ("proj_hidden", c_int), ("max_pos", c_int), ("ln_eps", c_float),
                ("w_patch", c_void_p), ("cls_emb", c_void_p), ("pos_emb", c_void_p),
                ("pre_ln_w", c_void_p), ("pre_ln_b", c_void_p), ("layers", POINTER(HyVitLayerW)),
                ("merge_ln_w", c_void_p), ("merge_ln_b", c_void_p), ("w_proj1", c_void_p),
                ("b_proj1", c_void_p), ("w_proj2", c_void_p), ("b_proj2", c_void_p)]


class HyKernelTimer(Structure):
    _fields_ = [("klass", c_int), ("capacity", c_int), ("count", c_int), ("events", c_void_p),
                ("work", c_void_p), ("shape", c_void_p)]


HY_KCLASS_DECODE_ATTN = 1
HY_KCLASS_GEMM = 2
HY_KCLASS_PREFILL_ATTN = 3
HY_KCLASS_VIT_ATTN = 4


class HyVitBatch(Structure):
    _fields_ = [("n_images", c_int), ("n_tokens", c_int), ("n_patches", c_int),
                ("n_visual", c_int), ("max_image_tokens", c_int), ("images", c_void_p),
                ("seg", c_void_p), ("out_row_map", c_void_p), ("image_rows", c_void_p)]


# name -> (restype, argtypes).  Every symbol declared in include/hydra_sm100.h.
_SIGS = {
    "hy_last_error": (c_char_p, []),
    "hy_version": (c_int, []),
    "hy_device_sm_count": (c_int, []),
    "hy_launch_count": (c_longlong, []),
    "hy_set_kernel_timer": (None, [c_void_p]),
    "hy_set_pdl": (c_int, [c_int]),
    "hy_gemm_bf16": (c_int, [c_void_p, c_int, c_void_p, c_int, c_int, c_int, c_int,
                             POINTER(HyGemmEpilogue), c_void_p, c_size_t, c_void_p]),
    "hy_gemm_bf16_mode": (c_int, [c_void_p, c_int, c_void_p, c_int, c_int, c_int, c_int,
                                  POINTER(HyGemmEpilogue), c_void_p, c_size_t, c_int, c_void_p]),
    "hy_rmsnorm": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_int, c_int, c_int, c_float,
                           c_void_p, c_void_p]),
    "hy_layernorm": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int,
                             c_float, c_void_p, c_void_p]),
    "hy_merge_embed": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_int, c_void_p, c_void_p,
                               c_void_p, c_void_p]),
    "hy_rope_kv_append": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_void_p,
                                  c_void_p, c_void_p, c_int, c_void_p, c_longlong, c_float,
                                  c_void_p]),
    "hy_attn_decode_paged": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_void_p,
                                     c_void_p, c_int, c_void_p, c_int, c_void_p, c_longlong,
                                     c_float, c_void_p, c_int, c_void_p, c_size_t, c_void_p]),
    "hy_attn_decode_workspace_bytes": (c_size_t, [c_int, c_int, c_int, c_int]),
    "hy_set_decode_kernel": (c_int, [c_int, c_int]),
    "hy_set_decode_coresident": (c_int, [c_int]),
    "hy_attn_prefill_paged": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p,
                                      c_int, c_int, c_int, c_int, c_void_p, c_int, c_void_p,
                                      c_longlong, c_float, c_void_p, c_int, c_void_p]),
    "hy_attn_varlen": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_int, c_int, c_int, c_float,
                               c_void_p, c_int, c_void_p]),
    "hy_argmax_f32": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p,
                              c_void_p]),
    "hy_im2col_patches": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_void_p,
                                  c_void_p]),
    "hy_copy_blocks": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_longlong,
                               c_void_p]),
    "hy_copy_blocks_tail": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_longlong,
                                    c_longlong, c_longlong, c_void_p]),
    "hy_enable_peer_access": (c_int, [c_int, c_int]),
    "hy_scatter_i32": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    "hy_fill_uniform_bf16": (c_int, [c_void_p, c_longlong, c_longlong, c_longlong, c_ulonglong,
                                     c_ulonglong, c_float, c_float, c_int, c_void_p]),
    "hy_lang_workspace_bytes": (c_size_t, [POINTER(HyLangModel), c_int, c_int, c_int, c_int]),
    "hy_lang_forward": (c_int, [POINTER(HyLangModel), POINTER(HyLangBatch), POINTER(HyKvCache),
                                c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "hy_vit_workspace_bytes": (c_size_t, [POINTER(HyVitModel), c_int, c_int]),
    "hy_vit_forward": (c_int, [POINTER(HyVitModel), POINTER(HyVitBatch), c_void_p, c_size_t,
                               c_void_p]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None


def load() -> ctypes.CDLL:
    """Load (once) and type the shared library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = load().hy_last_error().decode(errors="replace")
        raise HyError(f"{what or 'libhydra_sm100'} failed (cuda error {rc}): {msg}")


def call(name: str, *args) -> int:
    lib = load()
    rc = getattr(lib, name)(*args)
    check(rc, name)
    return rc


def ptr(t) -> int:
    """Device pointer of a torch tensor (0 for None)."""
    return 0 if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
