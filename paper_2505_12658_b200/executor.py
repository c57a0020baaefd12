"""S1: the GPU batch executor that replaces ``batch_latency`` (engine.py:500-509).

One ``InstanceRuntime`` per epdsim instance.  It owns the instance's device state:

  * the physical KV pool ``[blocks][layers][K|V][kv_heads][16][d]`` and image pool
    ``[blocks][576][H]`` (bf16), sized from the reference's ``pool_capacities``
    (cluster.py:127-144) so every block the scheduler counts exists on the device;
  * the device block table ``[slots][max_blocks]`` and ``last_tok[slots]``;
  * a language stream L and a vision stream V (dual-stream co-execution, K12);
  * workspaces for ``hy_lang_forward`` / ``hy_vit_forward``.

``run_batch(batch, reqs)`` lowers one ``Batch`` (decode entries, prefill chunks, encode
entries; engine.py:243-265) to the C ABI using the *pre-batch* cursors -- the reference
only advances ``kv_len`` / ``prefill_done`` / ``images_done`` after the batch
(cluster.py:333-366) -- executes it, and returns its latency:

  clock="oracle"  : epdsim's own ``batch_latency`` (decisions stay bit-identical to the
                    reference; the GPU still executes every batch)
  clock="device"  : CUDA-event time of the batch on the device (inputs resident in HBM)
  clock="wall"    : host wall time of the whole call, including the per-batch H2D of
                    the request images from pinned host memory and the D2H of the new
                    tokens (the end-to-end mode)

It never mutates ``batch`` or ``reqs`` (the loop does that in ``_on_batch_done``).
"""

from __future__ import annotations

import dataclasses
import itertools
import os
import time
from typing import Dict, List, Optional, Tuple

import numpy as np
import torch

from . import _lib
from ._epdsim import EN, MC
from .inputs import ImageStore, image_store_index, prompt_tokens
from .pools import PhysicalCachePool
from .shapes import MllmShape
from .weights import DeviceWeights

IMG = MC.IMAGE_BLOCK_TOKENS
KVB = MC.KV_BLOCK_TOKENS
CLOCKS = ("oracle", "device", "wall")
_BATCH_SEQ = itertools.count()  # global batch order, to merge tokens across instances
# programmatic dependent launch per batch: "decode" (decode-only language batches without
# vision work), "novis" (any batch without vision work), "never", "always"
_PDL_POLICY = os.environ.get("HY_PDL_POLICY", "decode")


@dataclasses.dataclass
class _Inflight:
    """A launched batch: what ``complete_batch`` needs to account it."""
    batch: object
    reqs: dict
    clock: str
    model_profile: object
    hw: object
    t_host0: float
    has_lang: bool
    has_vis: bool
    n_out: int
    tok_off: int
    out_rids: list
    cap_logits: object
    host_tokens: object = None  # pinned D2H buffer of the step's tokens (clock="wall")


class _Staging:
    """Pinned host buffer + device buffer pair for per-batch metadata uploads."""

    def __init__(self, device, nbytes: int):
        self.nbytes = nbytes
        self.host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        self.dev = torch.empty(nbytes, dtype=torch.uint8, device=device)

    def ensure(self, device, nbytes: int) -> None:
        if nbytes > self.nbytes:
            n = max(nbytes, 2 * self.nbytes)
            self.__init__(device, n)


class InstanceRuntime:
    def __init__(self, inst, shape: MllmShape, weights: DeviceWeights, *, seed: int,
                 images: ImageStore, resident_inputs: bool = True,
                 max_slots: Optional[int] = None,
                 max_seq_tokens: int = 16384, vit_max_tokens: Optional[int] = None,
                 lang_max_rows: Optional[int] = None, capture: bool = False,
                 pool_bytes_limit: Optional[int] = None):
        self.inst = inst
        self.iid = inst.id
        self.shape = shape
        self.weights = weights
        self.device = weights.device
        self.seed = seed
        self.images = images
        self.resident_inputs = resident_inputs
        self.lib = _lib.load()
        itype = inst.itype
        s = shape
        # --- S2: physical pools replace the count-only pools (same capacities) ---
        kv_cap = inst.kv_pool.capacity_blocks
        img_cap = inst.image_pool.capacity_blocks
        kv_phys, img_phys = kv_cap, img_cap
        if pool_bytes_limit is not None:
            kv_phys = min(kv_cap, pool_bytes_limit // (2 * s.kv_block_elems))
            img_phys = min(img_cap, pool_bytes_limit // (2 * s.image_block_elems))
        # every concurrent KV holder owns >= 1 block, so capacity bounds the slot count
        max_slots = max_slots or max(1, min(kv_cap, 32768))
        self.kv_pool = PhysicalCachePool(KVB, kv_cap, max_slots=max_slots,
                                         physical_blocks=kv_phys)
        self.image_pool = PhysicalCachePool(IMG, img_cap, physical_blocks=img_phys)
        inst.kv_pool = self.kv_pool
        inst.image_pool = self.image_pool
        self.bt_stride = -(-max_seq_tokens // KVB)
        with torch.cuda.device(self.device):
            self.kv = torch.empty((max(kv_phys, 1), s.kv_block_elems), dtype=torch.bfloat16,
                                  device=self.device)
            self.img = torch.empty((max(img_phys, 1) * IMG, s.hidden), dtype=torch.bfloat16,
                                   device=self.device)
            self.block_table = torch.zeros((max_slots, self.bt_stride), dtype=torch.int32,
                                           device=self.device)
            self.last_tok = torch.zeros(max_slots, dtype=torch.int32, device=self.device)
            # the vision tower is the small side of a mixed batch: give its stream the higher
            # priority so its CTAs are scheduled as soon as language-GEMM CTAs retire instead
            # of stretching over the whole batch (HY_VSTREAM_PRIO=0 disables)
            hi = os.environ.get("HY_VSTREAM_PRIO", "1") != "0"
            self.stream_l = torch.cuda.Stream(self.device, priority=0)
            self.stream_v = torch.cuda.Stream(self.device, priority=-1 if hi else 0)
            self.ev_start = torch.cuda.Event(enable_timing=True)
            self.ev_l = torch.cuda.Event(enable_timing=True)
            self.ev_v = torch.cuda.Event(enable_timing=True)
            self.meta = _Staging(self.device, 1 << 20)
            # one metadata / pixel staging pair per vision group of a batch: a group's host
            # buffer is rewritten only by the next batch, after this batch's events completed
            self.vmeta_groups: List[_Staging] = []
            self.pix_groups: List[Optional[_Staging]] = []
            self.tok_log = torch.empty(1 << 20, dtype=torch.int32, device=self.device)
        self._copy_stream = None
        self._waits: List = []
        self.kvc = _lib.HyKvCache(self.kv.data_ptr(), s.kv_block_elems, s.kv_layer_elems,
                                  kv_cap, self.block_table.data_ptr(), self.bt_stride)
        self.can_lang = itype.can_prefill or itype.can_decode
        self.can_vis = itype.can_encode
        tau_t = inst.budgets.token_budget
        tau_e = max(inst.budgets.image_budget, 1)
        self.lang_max_rows = lang_max_rows or (min(tau_t, 16384) + 2048)
        self.lang_ws = None
        self.lang_ws_rows = 0
        self.vit_max_tokens = vit_max_tokens or max(
            s.vit_tokens(IMG) * min(tau_e, 128), s.vit_tokens(IMG))
        self.vit_ws = None
        self._img_dev: Dict[Tuple[int, int, int], torch.Tensor] = {}
        self._prompts: Dict[str, np.ndarray] = {}
        self.tok_cursor = 0
        self.tok_records: List[Tuple[int, List[str]]] = []
        self.generated: Dict[str, List[int]] = {}
        self.launches = 0
        # parity capture: per batch, the pre-batch cursors and the logits of every row
        # that emits a token (tests only; costs a D2H per batch)
        self.capture = capture
        self.exec_log: List[Dict] = []
        self.sampler = None  # profiling.KernelSampler (bench.py)
        self.stats = {"batches": 0, "lang_rows": 0, "decode_rows": 0, "prefill_rows": 0,
                      "images": 0, "device_ms": 0.0, "host_ms": 0.0, "prep_ms": 0.0,
                      "launch_ms": 0.0, "mixed_batches": 0,
                      "vision_critical": 0}

    # ------------------------------------------------------------------ helpers
    def prompt(self, r) -> np.ndarray:
        p = self._prompts.get(r.rid)
        if p is None:
            p = prompt_tokens(self.seed, r.rid, r.spec.prompt_tokens, self.shape.vocab)
            self._prompts[r.rid] = p
        return p

    def forget(self, rid: str) -> None:
        self._prompts.pop(rid, None)

    def _ensure_lang_ws(self, rows: int, n_out: int, n_dec: int, max_ctx: int) -> None:
        need = self.lib.hy_lang_workspace_bytes(self.weights.lang, max(rows, 1), max(n_out, 1),
                                                max(n_dec, 1), max(max_ctx, 1))
        if self.lang_ws is None or self.lang_ws.numel() < need:
            cap = self.lib.hy_lang_workspace_bytes(
                self.weights.lang, max(rows, self.lang_max_rows), max(n_out, 1024),
                max(n_dec, 1024), max(max_ctx, self.bt_stride * KVB))
            # zero-filled on L itself: the forward (and its stream-K arrival counters, which
            # must start at zero) is stream-ordered after the memset
            self.lang_ws = None
            with torch.cuda.stream(self.stream_l):
                self.lang_ws = torch.zeros(max(need, cap), dtype=torch.uint8,
                                           device=self.device)

    def _ensure_vit_ws(self, tokens: int) -> None:
        need = self.lib.hy_vit_workspace_bytes(self.weights.vit, max(tokens, 1), 0)
        if self.vit_ws is None or self.vit_ws.numel() < need:
            # grow geometrically and zero on V, ordered before the ViT forward
            n = max(need, 2 * self.vit_ws.numel() if self.vit_ws is not None else need)
            self.vit_ws = None
            with torch.cuda.stream(self.stream_v):
                self.vit_ws = torch.zeros(n, dtype=torch.uint8, device=self.device)

    def copy_stream(self):
        """The stream migrations INTO this instance run on (pull model), created lazily."""
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream(self.device)
        return self._copy_stream

    def last_events(self):
        """Events that complete with this instance's last launched batch."""
        return (self.ev_l, self.ev_v)

    def wait_before_next_batch(self, event) -> None:
        """Order this instance's next batch after ``event`` (a migration copy)."""
        self._waits.append(event)

    def sync_block_tables(self, stream) -> None:
        """Push block lists of requests whose KV allocation changed to the device."""
        pool = self.kv_pool
        if not pool.dirty:
            return
        idx_parts, val_parts = [], []
        for rid in pool.dirty:
            ids = pool.ids.get(rid)
            if not ids:
                continue
            if len(ids) > self.bt_stride:
                raise ValueError(f"{rid}: {len(ids)} KV blocks exceed the block table "
                                 f"({self.bt_stride}); raise max_seq_tokens")
            base = pool.slot[rid] * self.bt_stride
            idx_parts.append(np.arange(base, base + len(ids), dtype=np.int32))
            val_parts.append(np.asarray(ids, dtype=np.int32))
        pool.dirty.clear()
        if not idx_parts:
            return
        idx = np.concatenate(idx_parts)
        val = np.concatenate(val_parts)
        n = idx.size
        buf = torch.from_numpy(np.concatenate([idx, val]))
        # a pageable H2D may return before its DMA lands: issue it on the stream the
        # scatter runs on, so the scatter is ordered after it
        with torch.cuda.stream(stream):
            dev = buf.to(self.device, non_blocking=False)
        _lib.check(self.lib.hy_scatter_i32(self.block_table.data_ptr(), dev.data_ptr(),
                                           dev.data_ptr() + 4 * n, n, stream.cuda_stream),
                   "hy_scatter_i32")
        self.launches += 1
        self._keep = dev  # allocated on `stream`: its reuse is ordered after the scatter

    # ------------------------------------------------------------------ lowering
    def _lower_language(self, batch, reqs):
        """Build the int32 metadata of the language part of ``batch``."""
        dec = batch.decode_entries
        pf = batch.prefill_chunks
        nd = len(dec)
        kvp = self.kv_pool
        slot = kvp.slot
        toks, poss, slots = [], [], []
        out_rows, out_slot = [], []
        out_rids: List[str] = []
        if nd:
            d_slot = np.fromiter((slot[rid] for rid, _ in dec), dtype=np.int32, count=nd)
            d_pos = np.fromiter((kl for _, kl in dec), dtype=np.int32, count=nd)
            toks.append(np.full(nd, _lib.HY_TOK_FROM_LAST, dtype=np.int32))
            poss.append(d_pos)
            slots.append(d_slot)
            out_rows.append(np.arange(nd, dtype=np.int32))
            out_slot.append(d_slot)
            out_rids.extend(rid for rid, _ in dec)
            dec_ctx = d_pos + 1
            max_ctx = int(dec_ctx.max())
        else:
            dec_ctx = np.zeros(0, dtype=np.int32)
            max_ctx = 0
        qstart = [0]
        offs, pslots = [], []
        row = nd
        max_q = 0
        for rid, c in pf:
            r = reqs[rid]
            o = r.prefill_done
            n_vis = r.plan.visual_tokens
            s_ = slot[rid]
            pos = np.arange(o, o + c, dtype=np.int32)
            tok = np.empty(c, dtype=np.int32)
            n_img_rows = max(0, min(o + c, n_vis) - o)
            if n_img_rows:
                ids = np.asarray(self.image_pool.ids[rid], dtype=np.int64)
                t = pos[:n_img_rows].astype(np.int64)
                tok[:n_img_rows] = -(1 + ids[t // IMG] * IMG + t % IMG)
            if n_img_rows < c:
                tok[n_img_rows:] = self.prompt(r)[pos[n_img_rows:] - n_vis]
            toks.append(tok)
            poss.append(pos)
            slots.append(np.full(c, s_, dtype=np.int32))
            qstart.append(qstart[-1] + c)
            offs.append(o)
            pslots.append(s_)
            if o + c >= r.plan.prefill_total_tokens:
                out_rows.append(np.array([row + c - 1], dtype=np.int32))
                out_slot.append(np.array([s_], dtype=np.int32))
                out_rids.append(rid)
            row += c
            max_q = max(max_q, c)
            max_ctx = max(max_ctx, o + c)
        n_rows = row
        cat = lambda xs: np.concatenate(xs) if xs else np.zeros(0, dtype=np.int32)
        parts = {
            "tok": cat(toks), "pos": cat(poss), "row_slot": cat(slots), "dec_ctx": dec_ctx,
            "pf_qstart": np.asarray(qstart, dtype=np.int32),
            "pf_offset": np.asarray(offs, dtype=np.int32),
            "pf_slot": np.asarray(pslots, dtype=np.int32),
            "out_rows": cat(out_rows), "out_slot": cat(out_slot),
        }
        return n_rows, nd, len(pf), max_q, max_ctx, parts, out_rids

    def _upload(self, staging: _Staging, parts: Dict[str, np.ndarray], stream) -> Dict[str, int]:
        """Pack int32 arrays into the pinned buffer, one async H2D, return device ptrs."""
        offs = {}
        total = 0
        for k, a in parts.items():
            offs[k] = total
            total += (a.nbytes + 255) & ~255
        staging.ensure(self.device, total)
        hv = staging.host.numpy()
        for k, a in parts.items():
            if a.nbytes:
                hv[offs[k]:offs[k] + a.nbytes] = a.view(np.uint8).reshape(-1)
        with torch.cuda.stream(stream):
            staging.dev[:total].copy_(staging.host[:total], non_blocking=True)
        base = staging.dev.data_ptr()
        return {k: (base + offs[k]) if parts[k].size else 0 for k in parts}

    def _device_image(self, index: int, gh: int, gw: int) -> torch.Tensor:
        key = (index, gh, gw)
        t = self._img_dev.get(key)
        if t is None:
            px = self.images.pixels(index, gh, gw)
            t = torch.from_numpy(px).to(self.device)
            self._img_dev[key] = t
        return t

    def _lower_vision(self, batch, reqs, stream):
        s = self.shape
        descs = []
        seg = [0]
        row_maps = []
        pix_host = []
        tok = patch = vis = 0
        max_t = 0
        for rid, k, counts in batch.encode_entries:
            r = reqs[rid]
            ids = np.asarray(self.image_pool.ids[rid], dtype=np.int64)
            all_counts = r.spec.image_token_counts
            off = sum(all_counts[:r.images_done])
            for j in range(k):
                ii = r.images_done + j
                T = all_counts[ii]
                gh, gw = s.patch_grid(T)
                nt = s.vit_tokens(T)
                sidx = image_store_index(self.seed, rid, ii)
                descs.append([sidx, gh, gw, tok, patch, vis])
                v = off + np.arange(T, dtype=np.int64)
                row_maps.append((ids[v // IMG] * IMG + v % IMG).astype(np.int32))
                tok += nt
                patch += gh * gw
                vis += T
                seg.append(tok)
                max_t = max(max_t, nt)
                off += T
        return descs, seg, row_maps, tok, patch, vis, max_t

    # ------------------------------------------------------------------ execute
    def run_batch(self, batch, reqs, clock: str, model_profile=None, hw=None) -> float:
        """Launch one batch, wait for it and return its latency under ``clock``."""
        return self.complete_batch(self.launch_batch(batch, reqs, clock, model_profile, hw))

    def batch_done(self) -> bool:
        """True once the batch in flight (``launch_batch``) has finished on both streams."""
        return self.ev_l.query() and self.ev_v.query()

    def launch_batch(self, batch, reqs, clock: str, model_profile=None, hw=None) -> "_Inflight":
        """Lower and launch one batch on the V/L streams without waiting for it (at most one
        batch in flight per instance: the reference marks the instance busy)."""
        t_host0 = time.perf_counter()
        cap_logits = None
        lib = self.lib
        dev = self.device
        sl, sv = self.stream_l, self.stream_v
        torch.cuda.set_device(dev)
        sl.wait_stream(torch.cuda.current_stream(dev))
        for ev in self._waits:  # migration copies touching this instance's pools
            sl.wait_event(ev)
        self._waits.clear()
        self.ev_start.record(sl)
        sv.wait_event(self.ev_start)
        self.sync_block_tables(sl)
        sampler = self.sampler
        has_lang = bool(batch.decode_entries or batch.prefill_chunks)
        has_vis = bool(batch.encode_entries)
        # PDL for decode-only batches without vision work (hy_set_pdl; HY_PDL_POLICY=never
        # keeps it off, =always on for every batch)
        lib.hy_set_pdl(1 if _PDL_POLICY == "always" or (
            _PDL_POLICY == "decode" and not batch.prefill_chunks and not has_vis) or (
            _PDL_POLICY == "novis" and not has_vis) else 0)
        if sampler is not None:
            sampler.before_batch(solo=not (has_lang and has_vis))
        out_rids: List[str] = []
        n_out = 0
        tok_off = 0
        if has_lang:
            n_rows, nd, npf, max_q, max_ctx, parts, out_rids = self._lower_language(batch, reqs)
            n_out = len(out_rids)
            self._ensure_lang_ws(n_rows, n_out, nd, max_ctx)
            ptrs = self._upload(self.meta, parts, sl)
            if self.tok_cursor + n_out > self.tok_log.numel():
                torch.cuda.synchronize(dev)
                self.collect_tokens(self.generated)  # drain the device token log
            tok_off = self.tok_cursor
            out_tok_ptr = self.tok_log.data_ptr() + 4 * tok_off
            logits_ptr = 0
            if self.capture and n_out:
                cap_logits = torch.empty((n_out, self.shape.vocab), dtype=torch.float32,
                                         device=dev)
                logits_ptr = cap_logits.data_ptr()
            self.stats["prep_ms"] += (time.perf_counter() - t_host0) * 1e3
            lb = _lib.HyLangBatch(n_rows, nd, npf, ptrs["tok"], ptrs["pos"], ptrs["row_slot"],
                                  ptrs["dec_ctx"], ptrs["pf_qstart"], ptrs["pf_offset"],
                                  ptrs["pf_slot"], max_q, max(max_ctx, 1), n_out,
                                  ptrs["out_rows"], ptrs["out_slot"], out_tok_ptr, logits_ptr)
            _lib.check(lib.hy_lang_forward(self.weights.lang, lb, self.kvc, self.img.data_ptr(),
                                           self.last_tok.data_ptr(), self.lang_ws.data_ptr(),
                                           self.lang_ws.numel(), sl.cuda_stream),
                       f"hy_lang_forward[{self.iid}]")
            self.stats["lang_rows"] += n_rows
            self.stats["decode_rows"] += nd
            self.stats["prefill_rows"] += n_rows - nd
        self.stats["launch_ms"] += (time.perf_counter() - t_host0) * 1e3
        if has_vis:
            self._run_vision(batch, reqs, sv)
        self.ev_l.record(sl)
        self.ev_v.record(sv)
        if n_out:
            self.tok_records.append((tok_off, out_rids, next(_BATCH_SEQ)))
            self.tok_cursor += n_out
        host = None
        if clock == "wall" and n_out:
            # end-to-end: read this step's tokens back to the host
            host = torch.empty(n_out, dtype=torch.int32, pin_memory=True)
            with torch.cuda.stream(sl):
                host.copy_(self.tok_log[tok_off:tok_off + n_out], non_blocking=True)
        return _Inflight(batch, reqs, clock, model_profile, hw, t_host0, has_lang, has_vis,
                         n_out, tok_off, out_rids, cap_logits, host)

    def complete_batch(self, h: "_Inflight") -> float:
        """Wait for the batch ``h`` and account it; returns its latency under ``h.clock``."""
        batch, reqs, clock, has_lang, has_vis = h.batch, h.reqs, h.clock, h.has_lang, h.has_vis
        n_out, tok_off, out_rids, cap_logits = h.n_out, h.tok_off, h.out_rids, h.cap_logits
        t_host0, sampler = h.t_host0, self.sampler
        self.ev_v.synchronize()
        self.ev_l.synchronize()
        t_l = self.ev_start.elapsed_time(self.ev_l)
        t_v = self.ev_start.elapsed_time(self.ev_v) if has_vis else 0.0
        dev_ms = max(t_l, t_v)
        if has_vis and has_lang:
            self.stats["mixed_batches"] += 1
            self.stats["vision_critical"] += int(t_v > t_l)
        host_s = time.perf_counter() - t_host0
        if sampler is not None:
            ctx_sum = sum(kl + 1 for _, kl in batch.decode_entries)
            s = self.shape
            keys = sum(c * reqs[rid].prefill_done + c * (c + 1) // 2
                       for rid, c in batch.prefill_chunks)
            vit_sq = sum(s.vit_tokens(T) ** 2 for rid, k, counts in batch.encode_entries
                         for T in reqs[rid].spec.image_token_counts[
                             reqs[rid].images_done:reqs[rid].images_done + k])
            sampler.after_batch(dev_ms, ctx_sum * s.kv_bytes_per_token / s.n_layers,
                                4.0 * s.head_dim * s.n_heads * keys,
                                4.0 * s.v_head_dim * s.v_heads * vit_sq)
        self.stats["batches"] += 1
        if self.capture:
            entry = {
                "decode": list(batch.decode_entries),
                "prefill": [(rid, c, reqs[rid].prefill_done) for rid, c in batch.prefill_chunks],
                "encode": [(rid, k, reqs[rid].images_done) for rid, k, _ in batch.encode_entries],
                "out_rids": list(out_rids),
            }
            if n_out:
                entry["logits"] = cap_logits.cpu().numpy()
                entry["tokens"] = self.tok_log[tok_off:tok_off + n_out].cpu().numpy().copy()
            self.exec_log.append(entry)
        self.stats["device_ms"] += dev_ms
        self.stats["host_ms"] += host_s * 1e3
        if clock == "device":
            return dev_ms * 1e-3
        if clock == "wall":
            return host_s
        return EN.batch_latency(batch, reqs, h.model_profile, h.hw)

    def _run_vision(self, batch, reqs, sv) -> None:
        s = self.shape
        descs, seg, row_maps, n_tok, n_patch, n_vis, max_t = self._lower_vision(batch, reqs, sv)
        # split into sub-batches that fit the workspace
        groups = []
        cur, cur_tok = [], 0
        for i, d in enumerate(descs):
            nt = seg[i + 1] - seg[i]
            if cur and cur_tok + nt > self.vit_max_tokens:
                groups.append(cur)
                cur, cur_tok = [], 0
            cur.append(i)
            cur_tok += nt
        if cur:
            groups.append(cur)
        while len(self.vmeta_groups) < len(groups):
            self.vmeta_groups.append(_Staging(self.device, 1 << 16))
            self.pix_groups.append(None)
        for gi, g in enumerate(groups):
            self._run_vision_group(gi, g, descs, seg, row_maps, sv)
        self.stats["images"] += len(descs)

    def _run_vision_group(self, gi, g, descs, seg, row_maps, sv) -> None:
        s = self.shape
        lib = self.lib
        tok = patch = vis = 0
        max_t = 0
        recs = []
        pix_arrays = []
        for i in g:
            sidx, gh, gw, _, _, _ = descs[i]
            nt = seg[i + 1] - seg[i]
            recs.append((sidx, gh, gw, tok, patch, vis))
            tok += nt
            patch += gh * gw
            vis += row_maps[i].size
            max_t = max(max_t, nt)
        self._ensure_vit_ws(tok)
        # pixels: resident device store, or per-batch H2D from pinned host memory
        arr = (_lib.HyImageDesc * len(g))()
        if self.resident_inputs:
            for j, (sidx, gh, gw, t0, p0, v0) in enumerate(recs):
                im = self._device_image(sidx, gh, gw)
                arr[j] = _lib.HyImageDesc(im.data_ptr(), gw * s.patch * 3, gh, gw, t0, p0, v0, 0)
        else:
            sizes = [gh * gw * s.patch * s.patch * 3 for (_, gh, gw, _, _, _) in recs]
            total = sum((z + 255) & ~255 for z in sizes)
            pix = self.pix_groups[gi]
            if pix is None or pix.nbytes < total:
                pix = self.pix_groups[gi] = _Staging(self.device, max(total, 1 << 20))
            hv = pix.host.numpy()
            off = 0
            offs = []
            for (sidx, gh, gw, _, _, _), z in zip(recs, sizes):
                hv[off:off + z] = self.images.pixels(sidx, gh, gw).reshape(-1)
                offs.append(off)
                off += (z + 255) & ~255
            with torch.cuda.stream(sv):
                pix.dev[:off].copy_(pix.host[:off], non_blocking=True)
            base = pix.dev.data_ptr()
            for j, ((sidx, gh, gw, t0, p0, v0), o) in enumerate(zip(recs, offs)):
                arr[j] = _lib.HyImageDesc(base + o, gw * s.patch * 3, gh, gw, t0, p0, v0, 0)
        desc_bytes = np.frombuffer(bytes(arr), dtype=np.uint8)
        parts = {
            "desc": desc_bytes.view(np.int32),
            "seg": np.asarray([recs[j][3] for j in range(len(recs))] + [tok], dtype=np.int32),
            "rowmap": np.concatenate([row_maps[i] for i in g]),
        }
        ptrs = self._upload(self.vmeta_groups[gi], parts, sv)
        vb = _lib.HyVitBatch(len(g), tok, patch, vis, max_t, ptrs["desc"], ptrs["seg"],
                             ptrs["rowmap"], self.img.data_ptr())
        _lib.check(lib.hy_vit_forward(self.weights.vit, vb, self.vit_ws.data_ptr(),
                                      self.vit_ws.numel(), sv.cuda_stream),
                   f"hy_vit_forward[{self.iid}]")

    def close(self) -> None:
        self.vmeta_groups, self.pix_groups = [], []
        for name in ("kv", "img", "block_table", "last_tok", "lang_ws", "vit_ws", "tok_log",
                     "meta", "_keep"):
            if hasattr(self, name):
                setattr(self, name, None)
        self._img_dev.clear()
        self.exec_log.clear()

    # ------------------------------------------------------------------ results
    def collect_tokens(self, out: Dict[str, List[int]]) -> None:
        """Append every token generated on this instance to ``out[rid]`` in order."""
        if not self.tok_records:
            return
        host = self.tok_log[:self.tok_cursor].cpu().numpy()
        for off, rids, seq in self.tok_records:
            for j, rid in enumerate(rids):
                out.setdefault(rid, []).append((seq, int(host[off + j])))
        self.tok_records.clear()
        self.tok_cursor = 0
