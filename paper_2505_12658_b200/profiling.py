"""Live kernel timing inside the serving loop (for bench.py's roofline numbers).

``KernelSampler`` installs a ``HyKernelTimer`` (include/hydra_sm100.h) on a sample of
batches: the native forward brackets every launch of the chosen kernel class with a
CUDA event pair on the launching stream, so the kernel's duration is measured where it
actually runs -- inside the timed serving region, not in a separate microbenchmark.

Algorithmic work per launch:
  GEMM           2*M*N*K flops (recorded by the library)
  decode attn    bytes = sum_i ctx_i * kv_bytes_per_token_per_layer (K+V of every key
                 read once; epdsim charges 2*B*H*(S+1)*ratio per layer,
                 model_cost.py:195) -- filled in here from the batch
  prefill attn   flops = 4 * d * heads * sum over chunk queries of keys attended (causal,
                 offset by the chunk start)
  ViT attn       flops = 4 * d * heads * sum over images of tokens^2 (block-diagonal)
"""

from __future__ import annotations

import ctypes
from typing import Dict, List

import torch

from . import _lib


class KernelSampler:
    CLASSES = {"gemm": _lib.HY_KCLASS_GEMM, "decode_attn": _lib.HY_KCLASS_DECODE_ATTN,
               "prefill_attn": _lib.HY_KCLASS_PREFILL_ATTN, "vit_attn": _lib.HY_KCLASS_VIT_ATTN}

    def __init__(self, device, every: int = 8, capacity: int = 512):
        self.every = every
        self.capacity = capacity
        self.lib = _lib.load()
        with torch.cuda.device(device):
            self.events = [torch.cuda.Event(enable_timing=True) for _ in range(2 * capacity)]
            s = torch.cuda.current_stream(device)
            for e in self.events:
                e.record(s)  # materialise the cudaEvent_t handles
            s.synchronize()
        self._handles = (ctypes.c_void_p * (2 * capacity))(*[e.cuda_event for e in self.events])
        self._work = (ctypes.c_double * capacity)()
        self._shape = (ctypes.c_longlong * capacity)()
        self.timer = _lib.HyKernelTimer(0, capacity, 0, ctypes.addressof(self._handles),
                                        ctypes.addressof(self._work),
                                        ctypes.addressof(self._shape))
        self.gemm_shapes: Dict[tuple, List[float]] = {}  # (M bin, N, K) -> [ms, flops, n]
        self.n_batches = 0
        self.active = None
        # per class: list of (ms, work) per launch; plus sampled batch device time
        self.samples: Dict[str, List] = {k: [] for k in self.CLASSES}
        # launches from batches where only one tower (one stream) ran: the kernel had the
        # GPU to itself, so these durations are not inflated by the other stream's CTAs
        self.solo_samples: Dict[str, List] = {k: [] for k in self.CLASSES}
        self.solo = False
        # busy time of the class: the union of its launches' [begin, end) intervals per
        # sampled batch.  With the V and L streams running kernels of the same class at
        # once, per-launch durations double-count the overlapped time; the union does not
        self.union_ms: Dict[str, float] = {k: 0.0 for k in self.CLASSES}
        self.batch_ms: Dict[str, float] = {k: 0.0 for k in self.CLASSES}
        self.class_ms: Dict[str, float] = {k: 0.0 for k in self.CLASSES}
        self.order = list(self.CLASSES)

    def before_batch(self, solo: bool = False) -> None:
        """solo: only one tower runs in this batch (no cross-stream contention)."""
        self.solo = solo
        self.n_batches += 1
        self.active = None
        if self.n_batches % self.every:
            return
        name = self.order[(self.n_batches // self.every) % len(self.order)]
        self.active = name
        self.timer.klass = self.CLASSES[name]
        self.timer.count = 0
        self.lib.hy_set_kernel_timer(ctypes.byref(self.timer))

    def after_batch(self, batch_device_ms: float, decode_ctx_bytes: float,
                    prefill_attn_flops: float = 0.0, vit_attn_flops: float = 0.0) -> None:
        """Call after the batch completed (events are final).  The attention works are per
        layer launch (bytes for decode, flops for prefill / ViT attention)."""
        if self.active is None:
            return
        self.lib.hy_set_kernel_timer(None)
        name = self.active
        tot = 0.0
        ivs = []
        for i in range(self.timer.count):
            ms = self.events[2 * i].elapsed_time(self.events[2 * i + 1])
            t0 = self.events[0].elapsed_time(self.events[2 * i]) if i else 0.0
            ivs.append((t0, t0 + ms))
            work = self._work[i]
            if name == "decode_attn":
                work = decode_ctx_bytes
            elif name == "prefill_attn":
                work = prefill_attn_flops
            elif name == "vit_attn":
                work = vit_attn_flops
            self.samples[name].append((ms, work))
            if self.solo:
                self.solo_samples[name].append((ms, work))
            tot += ms
            if name == "gemm" and self._shape[i]:
                sh = self._shape[i]
                M, N, K = sh >> 42, (sh >> 21) & 0x1FFFFF, sh & 0x1FFFFF
                mb = 1 << max(0, (M - 1).bit_length())  # power-of-two bin
                acc = self.gemm_shapes.setdefault((mb, N, K), [0.0, 0.0, 0])
                acc[0] += ms
                acc[1] += work
                acc[2] += 1
        ivs.sort()
        busy, cur0, cur1 = 0.0, None, None
        for x0, x1 in ivs:
            if cur1 is None or x0 > cur1:
                if cur1 is not None:
                    busy += cur1 - cur0
                cur0, cur1 = x0, x1
            else:
                cur1 = max(cur1, x1)
        if cur1 is not None:
            busy += cur1 - cur0
        self.union_ms[name] += busy
        self.batch_ms[name] += batch_device_ms
        self.class_ms[name] += tot
        self.active = None

    def gemm_breakdown(self, top: int = 16) -> List[Dict]:
        """GEMM time by (M rounded up to a power of two, N, K), largest share first."""
        tot = sum(v[0] for v in self.gemm_shapes.values()) or 1.0
        rows = [{"M_bin": k[0], "N": k[1], "K": k[2], "share": v[0] / tot,
                 "tflops": v[1] / v[0] / 1e9 if v[0] > 0 else 0.0, "launches": v[2]}
                for k, v in self.gemm_shapes.items()]
        return sorted(rows, key=lambda r: -r["share"])[:top]

    def summary(self) -> Dict[str, Dict]:
        out = {}
        for name, s in self.samples.items():
            if not s:
                continue
            ms = sum(x for x, _ in s)
            work = sum(w for _, w in s)
            so = self.solo_samples[name]
            so_ms = sum(x for x, _ in so)
            out[name] = {"launches": len(s), "avg_ms": ms / len(s), "total_ms": ms,
                         "work": work, "work_per_ms": work / ms if ms > 0 else 0.0,
                         "union_ms": self.union_ms[name],
                         "work_per_union_ms": (work / self.union_ms[name]
                                               if self.union_ms[name] > 0 else 0.0),
                         "solo_launches": len(so),
                         "solo_work_per_ms": sum(w for _, w in so) / so_ms if so_ms > 0 else 0.0,
                         "share_of_batch_time": (self.class_ms[name] / self.batch_ms[name]
                                                 if self.batch_ms[name] > 0 else 0.0)}
        return out
