"""CPU tests of the host-side logic: shapes, synthetic inputs, weight specs, and the
lowering of reference Batches to the C-ABI metadata (no device needed)."""

import types

import numpy as np
import pytest

from paper_2505_12658_b200 import _lib, get_shape, with_layers
from paper_2505_12658_b200._epdsim import C, E, EN
from paper_2505_12658_b200.executor import InstanceRuntime
from paper_2505_12658_b200.inputs import ImageStore, image_store_index, prompt_tokens
from paper_2505_12658_b200.pools import PhysicalCachePool
from paper_2505_12658_b200.weights import weight_specs


def test_shapes_match_reference_profiles():
    assert get_shape("llava-1.5-7b").profile() == E.MODEL_PRESETS["llava-1.5-7b"]
    tiny = get_shape("tiny").profile()
    assert tiny == E.ModelProfile(512, 4, 2, 256, 4, 2)
    q = get_shape("qwen2-vl-7b")
    assert q.profile().kv_bytes_per_token == 57344
    assert q.head_dim == 128 and q.v_head_dim == 80 and q.n_heads // q.n_kv_heads == 7
    s = get_shape("llava-1.5-7b")
    assert s.patch_grid(576) == (24, 24) and s.vit_tokens(576) == 577
    assert q.patch_grid(256) == (32, 32) and q.vit_tokens(256) == 1024
    assert s.kv_block_elems * 2 == 8 << 20                # one KV block = 8 MiB
    assert s.k_pad == 640 and s.ffn == 11008


def test_weight_specs_cover_architecture():
    s = get_shape("llava-1.5-7b")
    specs = weight_specs(s)
    names = [sp.name for sp in specs]
    assert len(names) == len(set(names))
    n_params = sum(sp.rows * sp.cols for sp in specs)
    assert 7.0e9 < n_params < 7.2e9                      # LLaVA-1.5-7B ~7.06B
    gu = [sp for sp in specs if sp.name == "lang.0.w_gate_up"][0]
    assert gu.perm == 1 and gu.rows == 2 * s.ffn
    q = with_layers(get_shape("qwen2-vl-7b"), 1, 1)
    assert any(sp.name == "lang.0.b_qkv" for sp in weight_specs(q))


def test_inputs_deterministic():
    a = prompt_tokens(0, "r1", 35, 32000)
    assert np.array_equal(a, prompt_tokens(0, "r1", 35, 32000))
    assert not np.array_equal(a, prompt_tokens(0, "r2", 35, 32000))
    assert a.dtype == np.int32 and a.min() >= 0 and a.max() < 32000
    st = ImageStore(0, 14)
    px = st.request_image("r1", 0, 24, 24)
    assert px.shape == (336, 336, 3) and px.dtype == np.uint8
    assert np.array_equal(px, ImageStore(0, 14).request_image("r1", 0, 24, 24))
    assert 0 <= image_store_index(0, "r1", 0) < 8


def _fake_runtime(shape):
    rt = types.SimpleNamespace()
    rt.shape = shape
    rt.kv_pool = PhysicalCachePool(16, 1000, max_slots=8)
    rt.image_pool = PhysicalCachePool(576, 10)
    prompts = {}

    def prompt(r):
        if r.rid not in prompts:
            prompts[r.rid] = prompt_tokens(0, r.rid, r.spec.prompt_tokens, shape.vocab)
        return prompts[r.rid]

    rt.prompt = prompt
    return rt


def _req(rid, images, prompt, out):
    spec = E.RequestSpec(rid, 0.0, tuple(images), prompt, out, E.SloSpec(4, 0.08))
    return EN.RequestState(spec=spec, plan=E.plan_stages(spec))


def test_lower_language_batch():
    shape = get_shape("tiny")
    rt = _fake_runtime(shape)
    a = _req("a", [576], 40, 5)          # mid-prefill, window cuts through the image
    b = _req("b", [], 10, 5)             # decoding
    rt.image_pool.allocate("x", 1)       # occupy id 0 so 'a' gets image block 1
    rt.image_pool.allocate("a", 1)
    rt.kv_pool.allocate("a", 40)
    rt.kv_pool.allocate("b", 2)
    a.stage, a.prefill_done = EN.PREFILL, 570
    b.stage, b.kv_len = EN.DECODE, 11
    reqs = {"a": a, "b": b}
    batch = EN.Batch(decode_entries=[("b", 11)], prefill_chunks=[("a", 46)])
    n_rows, nd, npf, max_q, max_ctx, parts, out_rids = InstanceRuntime._lower_language(
        rt, batch, reqs)
    assert (n_rows, nd, npf, max_q) == (47, 1, 1, 46)
    assert max_ctx == 616 and out_rids == ["b", "a"]   # 570 + 46 = 616 = whole prompt
    tok, pos = parts["tok"], parts["pos"]
    assert tok[0] == _lib.HY_TOK_FROM_LAST and pos[0] == 11 and parts["dec_ctx"][0] == 12
    # rows 1..6: image tokens 570..575 of image block 1 -> pool rows 576+570..
    assert tok[1:7].tolist() == [-(1 + 576 + t) for t in range(570, 576)]
    assert tok[7:].tolist() == rt.prompt(a)[:40].tolist()
    assert pos[1:].tolist() == list(range(570, 616))
    assert parts["pf_qstart"].tolist() == [0, 46] and parts["pf_offset"].tolist() == [570]
    assert parts["row_slot"].tolist() == [rt.kv_pool.slot["b"]] + [rt.kv_pool.slot["a"]] * 46
    assert parts["out_rows"].tolist() == [0, 46]


def test_executor_refuses_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2505_12658_b200.cluster import GpuCluster
    spec = C.ClusterSpec(method=C.DisaggregationMethod.parse("EPD:1"))
    with pytest.raises(RuntimeError):
        GpuCluster(spec, get_shape("tiny"), E.DEFAULT_HARDWARE, E.SloSpec(4, 0.08))
