"""Paged, batched, multi-layer compressed KV cache on the B200.

This is the storage layout + pager that replaces the reference's per-layer
numpy arrays (``CompressedLayerCache``, pkg/src/tadakv/cache.py:114-213):

* one device pool per layer (``uint8 [pages, page_bytes]``), laid out by
  ``tada_page_layout`` (include/tadakv_b200.h) for that layer's bit width —
  the per-layer precision dispatch of ``PrecisionPlan`` (cache.py:38-63);
* ONE page table ``int32 [batch, pages_per_seq]`` shared by all layers (every
  layer appends the same tokens, so logical pages line up);
* per-(layer, sequence) device counters ``comp_len`` / ``res_len`` that the
  kernels read, so decode steps are CUDA-graph capturable;
* a f32 residual buffer ``[batch, R, heads, head_dim]`` per layer holding the
  newest ``< R`` tokens verbatim (cache.py:154-180).

Appends follow the reference's flush policy exactly (quantization is per
token, so flushing f*R tokens at once == f block flushes; test_cache.py:107-117).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _dev
from ._lib import call, page_layout
from .errors import CapacityError, ConfigError, DataError, ShapeError, StateError
from .quant import QuantizedDeviation, validate_bits

F32 = np.float32


class PagedKVCache:
    """Compressed KV for ``batch`` sequences x ``num_layers`` layers in paged HBM."""

    def __init__(self, num_layers: int, num_kv_heads: int, head_dim: int, plan, residual_length: int,
                 batch: int = 1, page_tokens: int = 64, max_tokens: int | None = None, shuffle_pages: bool = False,
                 seed: int = 0):
        plan = tuple(int(b) for b in (plan.bits_per_layer if hasattr(plan, "bits_per_layer") else plan))
        if len(plan) != num_layers:
            raise ConfigError(f"plan covers {len(plan)} layers but the model has {num_layers}")
        for b in plan:
            validate_bits(b)
        if min(num_layers, num_kv_heads, head_dim, batch, page_tokens) <= 0:
            raise ConfigError("layer/head/dimension/batch counts must be positive")
        if residual_length < 0:
            raise ConfigError(f"residual_length must be non-negative, got {residual_length}")
        self.dev = _dev.device()
        self.L, self.H, self.D, self.B = num_layers, num_kv_heads, head_dim, batch
        self.plan = plan
        self.R = residual_length
        self.P = page_tokens
        self.layouts = [page_layout(page_tokens, num_kv_heads, head_dim, b) for b in plan]
        self.growable = max_tokens is None
        pps = 1 if max_tokens is None else max(1, math.ceil(max_tokens / page_tokens))
        self._pt_host = np.full((batch, pps), -1, dtype=np.int32)
        self.page_table = torch.full((batch, pps), -1, dtype=torch.int32, device=self.dev)
        self._n_pages = 0
        self._cap_pages = 0
        self.pools = [torch.empty((0, lay.page_bytes), dtype=torch.uint8, device=self.dev) for lay in self.layouts]
        self.comp_host = np.zeros((num_layers, batch), dtype=np.int64)
        self.res_host = np.zeros((num_layers, batch), dtype=np.int64)
        self.comp_len = torch.zeros((num_layers, batch), dtype=torch.int32, device=self.dev)
        self.res_len = torch.zeros((num_layers, batch), dtype=torch.int32, device=self.dev)
        rcap = max(self.R, 1)
        self.res_k = [torch.zeros((batch, rcap, num_kv_heads, head_dim), dtype=torch.float32, device=self.dev)
                      for _ in range(num_layers)]
        self.res_v = [torch.zeros_like(t) for t in self.res_k]
        self.err = _dev.ErrFlag()
        self._zeros_b = torch.zeros(batch, dtype=torch.int32, device=self.dev)
        self._ws = None
        if max_tokens is not None:  # pre-size: every page of every sequence up front
            order = np.arange(batch * pps, dtype=np.int32)
            if shuffle_pages:
                np.random.default_rng(seed).shuffle(order)
            self._grow_pools(batch * pps)
            self._pt_host[:, :] = order.reshape(batch, pps)
            self._n_pages = batch * pps
            self.page_table.copy_(torch.from_numpy(self._pt_host))

    # ------------------------------------------------------------------ pager
    def _grow_pools(self, need: int) -> None:
        if need <= self._cap_pages:
            return
        cap = max(need, 2 * self._cap_pages, 4)
        for i, lay in enumerate(self.layouts):
            # one spare page: 16-byte-rounded bulk copies of a tile tail may read a few bytes past a page
            new = torch.empty((cap + 1, lay.page_bytes), dtype=torch.uint8, device=self.dev)
            if self._n_pages:
                new[: self._n_pages].copy_(self.pools[i][: self._n_pages])
            self.pools[i] = new
        self._cap_pages = cap

    def _ensure_pages(self, upto_tokens: int) -> None:
        """Make logical pages [0, ceil(upto/P)) exist for every sequence."""
        need = math.ceil(upto_tokens / self.P)
        if need <= self._pt_host.shape[1] and (need == 0 or (self._pt_host[:, need - 1] >= 0).all()):
            return
        if not self.growable and need > self._pt_host.shape[1]:
            raise CapacityError(f"{upto_tokens} tokens exceed the cache capacity of "
                                f"{self._pt_host.shape[1] * self.P} tokens per sequence")
        if need > self._pt_host.shape[1]:
            grown = np.full((self.B, max(need, 2 * self._pt_host.shape[1])), -1, dtype=np.int32)
            grown[:, : self._pt_host.shape[1]] = self._pt_host
            self._pt_host = grown
        missing = int((self._pt_host[:, :need] < 0).sum())
        self._grow_pools(self._n_pages + missing)
        for b in range(self.B):
            for j in range(need):
                if self._pt_host[b, j] < 0:
                    self._pt_host[b, j] = self._n_pages
                    self._n_pages += 1
        self.page_table = torch.from_numpy(self._pt_host).to(self.dev)

    # ------------------------------------------------------------------ bookkeeping
    def _uniform(self, arr: np.ndarray, layer: int) -> int:
        row = arr[layer]
        if (row != row[0]).any():
            raise StateError("batched call needs every sequence at the same length; use per-sequence caches")
        return int(row[0])

    def lengths(self, layer: int, b: int = 0) -> tuple[int, int]:
        """(compressed tokens, residual tokens) of one (layer, sequence)."""
        return int(self.comp_host[layer, b]), int(self.res_host[layer, b])

    def _add(self, arr: torch.Tensor, host: np.ndarray, layer: int, delta: int) -> None:
        if delta:
            call("tada_lengths_add", arr[layer].data_ptr(), self.B, delta, _dev.stream())
            host[layer] += delta

    def _layout_ptr(self, layer: int):
        import ctypes

        return ctypes.byref(self.layouts[layer])

    # ------------------------------------------------------------------ append (K1)
    def _quant_append(self, layer: int, src_k, src_v, dtype: int, n_tok: int, src_stride: int, dst_offset: int):
        call("tada_quant_append", self._layout_ptr(layer), self.pools[layer].data_ptr(), src_k, src_v, dtype,
             self.B, n_tok, src_stride, self.page_table.data_ptr(), self.page_table.shape[1],
             self.comp_len[layer].data_ptr(), dst_offset, self.err.ptr, _dev.stream())

    def _residual_write(self, layer: int, k: torch.Tensor, v: torch.Tensor, first: int, n_tok: int, pos_offset: int):
        if n_tok <= 0:
            return
        row = self.H * self.D
        esz = k.element_size()
        call("tada_residual_write", self.res_k[layer].data_ptr(), self.res_v[layer].data_ptr(),
             self.res_k[layer].shape[1], self.H, self.D, k.data_ptr() + first * row * esz,
             v.data_ptr() + first * row * esz, _dev.dtype_code(k), self.B, n_tok, k.shape[1],
             self.res_len[layer].data_ptr(), pos_offset, _dev.stream())

    def append(self, layer: int, k: torch.Tensor, v: torch.Tensor) -> None:
        """Append already-rotated keys and values ``[batch, n, heads, head_dim]`` (cache.py:154-180).

        Non-finite inputs set the device error flag; call :meth:`check_errors`
        (the drop-in ``CompressedLayerCache`` pre-checks instead, so it raises
        before mutating, like the reference).
        """
        if k.ndim != 4 or tuple(k.shape[2:]) != (self.H, self.D) or k.shape[0] != self.B:
            raise ShapeError(f"keys must be ({self.B}, tokens, {self.H}, {self.D}), got {tuple(k.shape)}")
        if tuple(v.shape) != tuple(k.shape):
            raise ShapeError(f"values shape {tuple(v.shape)} does not match keys shape {tuple(k.shape)}")
        n = int(k.shape[1])
        if n == 0:
            return
        k = k.contiguous()
        v = v.contiguous()
        if k.dtype not in (torch.float32, torch.bfloat16) or v.dtype != k.dtype:
            k, v = k.float(), v.float()
        dt = _dev.dtype_code(k)
        C = self._uniform(self.comp_host, layer)
        r = self._uniform(self.res_host, layer)
        R = self.R
        if R == 0:
            self._ensure_pages(C + n)
            self._quant_append(layer, k.data_ptr(), v.data_ptr(), dt, n, n, 0)
            self._add(self.comp_len, self.comp_host, layer, n)
            return
        total = r + n
        ncomp = (total // R) * R
        if ncomp == 0:  # no flush: one launch writes the rows and advances res_len
            call("tada_residual_append", self.res_k[layer].data_ptr(), self.res_v[layer].data_ptr(),
                 self.res_k[layer].shape[1], self.H, self.D, k.data_ptr(), v.data_ptr(), dt, self.B, n, n,
                 self.res_len[layer].data_ptr(), _dev.stream())
            self.res_host[layer] += n
            return
        self._ensure_pages(C + ncomp)
        if r:  # the buffered residual rows are the oldest tokens of the flushed blocks
            self._quant_append(layer, self.res_k[layer].data_ptr(), self.res_v[layer].data_ptr(), 0, r,
                               self.res_k[layer].shape[1], 0)
        n_new = ncomp - r
        self._quant_append(layer, k.data_ptr(), v.data_ptr(), dt, n_new, n, r)
        keep = total - ncomp
        self._residual_write(layer, k, v, n_new, keep, -r)
        self._add(self.comp_len, self.comp_host, layer, ncomp)
        self._add(self.res_len, self.res_host, layer, keep - r)

    def _quant_append_rope(self, layer: int, src_k, src_v, dtype: int, n_tok: int, src_stride: int, dst_offset: int,
                           pos: torch.Tensor, table: torch.Tensor):
        call("tada_quant_append_rope", self._layout_ptr(layer), self.pools[layer].data_ptr(), src_k, src_v, dtype,
             self.B, n_tok, src_stride, self.page_table.data_ptr(), self.page_table.shape[1],
             self.comp_len[layer].data_ptr(), dst_offset, pos.data_ptr(), pos.shape[1], table.data_ptr(),
             int(table.shape[0]), self.err.ptr, _dev.stream())

    def _rotate(self, k: torch.Tensor, pos: torch.Tensor, table: torch.Tensor) -> torch.Tensor:
        """[B, n, heads, D] rows -> rotated f32 copy (tada_apply_rope), positions [B, n] (any head count)."""
        kc = k.contiguous()
        out = torch.empty(kc.shape, dtype=torch.float32, device=self.dev)
        n_rows = kc.shape[0] * kc.shape[1]
        if n_rows:
            call("tada_apply_rope", kc.data_ptr(), _dev.dtype_code(kc), n_rows, kc.shape[2], kc.shape[3],
                 pos.contiguous().data_ptr(), table.data_ptr(), int(table.shape[0]), out.data_ptr(), self.err.ptr,
                 _dev.stream())
        return out

    def append_rope(self, layer: int, k: torch.Tensor, v: torch.Tensor, pos: torch.Tensor, n_pos: int,
                    rope) -> None:
        """Append pre-RoPE keys (rotated on the fly) and values ``[batch, n, heads, head_dim]``.

        ``pos``: device int32 ``[batch, n]`` (validated by the caller, max < n_pos).  The rows that reach
        the compressed region go through K1 with the rotation fused (``tada_quant_append_rope``); rows
        that stay in the residual buffer are rotated by ``tada_apply_rope`` first (cache.py:174-180
        policy as in :meth:`append`).  Bit-identical to rotating first and calling :meth:`append`.
        """
        from .rope import rope_table

        if k.ndim != 4 or tuple(k.shape[2:]) != (self.H, self.D) or k.shape[0] != self.B:
            raise ShapeError(f"keys must be ({self.B}, tokens, {self.H}, {self.D}), got {tuple(k.shape)}")
        if tuple(v.shape) != tuple(k.shape):
            raise ShapeError(f"values shape {tuple(v.shape)} does not match keys shape {tuple(k.shape)}")
        n = int(k.shape[1])
        if tuple(pos.shape) != (self.B, n):
            raise ShapeError(f"positions must be ({self.B}, {n}), got {tuple(pos.shape)}")
        if n == 0:
            return
        table = rope_table(rope, n_pos)
        pos = pos.to(device=self.dev, dtype=torch.int32).contiguous()
        k = k.contiguous()
        v = v.contiguous()
        if k.dtype not in (torch.float32, torch.bfloat16) or v.dtype != k.dtype:
            k, v = k.float(), v.float()
        bits = self.layouts[layer].bits
        if not (self.H == 8 and self.D == 128 and bits in (2, 4, 8)):
            self.append(layer, self._rotate(k, pos, table), v.float())  # generic geometry: compose
            return
        dt = _dev.dtype_code(k)
        C = self._uniform(self.comp_host, layer)
        r = self._uniform(self.res_host, layer)
        R = self.R
        if R == 0:
            self._ensure_pages(C + n)
            self._quant_append_rope(layer, k.data_ptr(), v.data_ptr(), dt, n, n, 0, pos, table)
            self._add(self.comp_len, self.comp_host, layer, n)
            return
        total = r + n
        ncomp = (total // R) * R
        if ncomp == 0:  # no flush: rotated rows go to the residual buffer
            self.append(layer, self._rotate(k, pos, table), v.float())
            return
        self._ensure_pages(C + ncomp)
        if r:  # the buffered residual rows (already rotated) are the oldest tokens of the flushed blocks
            self._quant_append(layer, self.res_k[layer].data_ptr(), self.res_v[layer].data_ptr(), 0, r,
                               self.res_k[layer].shape[1], 0)
        n_new = ncomp - r
        self._quant_append_rope(layer, k.data_ptr(), v.data_ptr(), dt, n_new, n, r, pos, table)
        keep = total - ncomp
        if keep:
            k_keep = self._rotate(k[:, n_new:], pos[:, n_new:], table)
            self._residual_write(layer, k_keep, v[:, n_new:].float().contiguous(), 0, keep, -r)
        self._add(self.comp_len, self.comp_host, layer, ncomp)
        self._add(self.res_len, self.res_host, layer, keep - r)

    def check_errors(self) -> None:
        """Raise DataError if any kernel saw a non-finite input since the last check (synchronising)."""
        if self.err.raised():
            raise DataError("cannot quantize non-finite values")

    # ------------------------------------------------------------------ attention (K2 + K3)
    def workspace(self, num_q_heads: int, splits: int) -> torch.Tensor | None:
        from ._lib import load

        nbytes = int(load().tada_decode_attn_workspace_bytes(self.B, num_q_heads, self.D, splits))
        if nbytes == 0:
            return None
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)
        return self._ws

    def suggest_splits(self, layer: int, num_q_heads: int | None = None) -> int:
        """Split-K factor for this layer's kernel (whole waves of resident CTAs on this device)."""
        from ._lib import load

        tokens = int((self.comp_host[layer] + self.res_host[layer]).max())
        if num_q_heads is None:
            return int(load().tada_decode_attn_suggest_splits(self.B, tokens, self.P))
        return int(load().tada_decode_attn_plan_splits(self._layout_ptr(layer), num_q_heads, self.B, tokens))

    def attend(self, layer: int, q: torch.Tensor, out: torch.Tensor | None = None, out_dtype=torch.float32,
               num_splits: int | None = None, mode: int = 0, scale: float | None = None) -> torch.Tensor:
        """Decode attention for one query per sequence: ``q [batch, Hq, D]`` -> ``[batch, Hq, D]``.

        attend_streaming semantics (attention.py:103-151) over compressed then
        residual tokens, GQA map kv = g*H // Hq (attention.py:47-49).
        """
        if q.ndim != 3 or q.shape[0] != self.B or q.shape[2] != self.D or q.shape[1] % self.H:
            raise ShapeError(f"query must be ({self.B}, Hq, {self.D}) with Hq a multiple of {self.H}, got "
                             f"{tuple(q.shape)}")
        if ((self.comp_host[layer] + self.res_host[layer]) == 0).any():
            raise StateError("cannot attend over an empty cache")
        hq = int(q.shape[1])
        if q.dtype not in (torch.float32, torch.bfloat16):
            q = q.float()
        q = q.contiguous()
        splits = num_splits or self.suggest_splits(layer, hq)
        ws = self.workspace(hq, splits)
        if out is None:
            out = torch.empty((self.B, hq, self.D), dtype=out_dtype, device=self.dev)
        sc = np.float32(1.0 / math.sqrt(self.D)) if scale is None else np.float32(scale)
        call("tada_decode_attn", self._layout_ptr(layer), self.pools[layer].data_ptr(), q.data_ptr(),
             _dev.dtype_code(q), self.B, hq, self.page_table.data_ptr(), self.page_table.shape[1],
             self.comp_len[layer].data_ptr(), self.res_len[layer].data_ptr(), self.res_k[layer].data_ptr(),
             self.res_v[layer].data_ptr(), self.res_k[layer].shape[1], float(sc), splits, _dev.ptr(ws),
             out.data_ptr(), _dev.dtype_code(out), mode, _dev.stream())
        return out

    def append_attend(self, layer: int, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                      out: torch.Tensor | None = None, out_dtype=torch.float32, num_splits: int | None = None,
                      mode: int = 0, scale: float | None = None) -> torch.Tensor:
        """One decode step of a layer: :meth:`append` of one token per sequence (``k``, ``v``:
        ``[batch, 1, heads, head_dim]``, rotated) then :meth:`attend` — model.py:280-281.

        When the token stays in the residual buffer (no flush) and the layer runs on the tensor-core
        path, both happen in one call (``tada_decode_attn_append``: K3 attends the new row straight from
        the input and stores it); otherwise this is exactly append() + attend()."""
        from ._lib import load

        fused_ok = (k.ndim == 4 and k.shape[1] == 1 and tuple(v.shape) == tuple(k.shape) and self.R > 0
                    and mode != 1 and k.dtype in (torch.float32, torch.bfloat16) and v.dtype == k.dtype
                    and q.ndim == 3 and q.shape[0] == self.B and q.shape[2] == self.D and q.shape[1] % self.H == 0)
        if fused_ok:
            C = self._uniform(self.comp_host, layer)
            r = self._uniform(self.res_host, layer)
            fused_ok = C > 0 and r + 1 < self.R
        if not fused_ok:
            self.append(layer, k, v)
            return self.attend(layer, q, out=out, out_dtype=out_dtype, num_splits=num_splits, mode=mode, scale=scale)
        hq = int(q.shape[1])
        if q.dtype not in (torch.float32, torch.bfloat16):
            q = q.float()
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
        splits = num_splits or self.suggest_splits(layer, hq)
        ws = self.workspace(hq, splits)
        if out is None:
            out = torch.empty((self.B, hq, self.D), dtype=out_dtype, device=self.dev)
        sc = np.float32(1.0 / math.sqrt(self.D)) if scale is None else np.float32(scale)
        rc = load().tada_decode_attn_append(
            self._layout_ptr(layer), self.pools[layer].data_ptr(), q.data_ptr(), _dev.dtype_code(q), self.B, hq,
            self.page_table.data_ptr(), self.page_table.shape[1], self.comp_len[layer].data_ptr(),
            self.res_len[layer].data_ptr(), self.res_k[layer].data_ptr(), self.res_v[layer].data_ptr(),
            self.res_k[layer].shape[1], float(sc), splits, _dev.ptr(ws), out.data_ptr(), _dev.dtype_code(out), mode,
            k.data_ptr(), v.data_ptr(), _dev.dtype_code(k), r, _dev.stream())
        if rc != 0:  # geometry without the tensor-core path: nothing was enqueued
            self.append(layer, k, v)
            return self.attend(layer, q, out=out, out_dtype=out_dtype, num_splits=num_splits, mode=mode, scale=scale)
        self.res_host[layer] += 1
        return out

    def attend_lse(self, layer: int, q: torch.Tensor, num_splits: int | None = None, mode: int = 0,
                   scale: float | None = None) -> tuple[torch.Tensor, torch.Tensor]:
        """Like :meth:`attend` (f32 out) and also the log-sum-exp ``[batch, Hq]`` of the scaled logits.

        ``(out, lse)`` pairs over disjoint token sets merge exactly (shard.merge_partials).
        """
        if q.ndim != 3 or q.shape[0] != self.B or q.shape[2] != self.D or q.shape[1] % self.H:
            raise ShapeError(f"query must be ({self.B}, Hq, {self.D}) with Hq a multiple of {self.H}, got "
                             f"{tuple(q.shape)}")
        if ((self.comp_host[layer] + self.res_host[layer]) == 0).any():
            raise StateError("cannot attend over an empty cache")
        hq = int(q.shape[1])
        if q.dtype not in (torch.float32, torch.bfloat16):
            q = q.float()
        q = q.contiguous()
        splits = num_splits or self.suggest_splits(layer, hq)
        ws = self.workspace(hq, splits)
        out = torch.empty((self.B, hq, self.D), dtype=torch.float32, device=self.dev)
        lse = torch.empty((self.B, hq), dtype=torch.float32, device=self.dev)
        sc = np.float32(1.0 / math.sqrt(self.D)) if scale is None else np.float32(scale)
        call("tada_decode_attn_lse", self._layout_ptr(layer), self.pools[layer].data_ptr(), q.data_ptr(),
             _dev.dtype_code(q), self.B, hq, self.page_table.data_ptr(), self.page_table.shape[1],
             self.comp_len[layer].data_ptr(), self.res_len[layer].data_ptr(), self.res_k[layer].data_ptr(),
             self.res_v[layer].data_ptr(), self.res_k[layer].shape[1], float(sc), splits, _dev.ptr(ws),
             out.data_ptr(), _dev.dtype_code(out), mode, lse.data_ptr(), _dev.stream())
        return out, lse

    # ------------------------------------------------------------------ export / import (TADAKV1 parity vehicle)
    def export(self, layer: int, b: int = 0) -> dict:
        """Dense reference-layout tensors of one (layer, sequence): means, deviation records, residual rows."""
        C, r = self.lengths(layer, b)
        lay = self.layouts[layer]
        out = {}
        page_row = self.page_table[b].contiguous()
        for side, name in ((0, "k"), (1, "v")):
            mean = torch.empty((C, self.D), dtype=torch.float32, device=self.dev)
            codes = torch.empty(C * self.H * lay.group_bytes, dtype=torch.uint8, device=self.dev)
            scales = torch.empty(C * self.H, dtype=torch.float32, device=self.dev)
            mins = torch.empty(C * self.H, dtype=torch.float32, device=self.dev)
            if C:
                call("tada_gather_compressed", self._layout_ptr(layer), self.pools[layer].data_ptr(),
                     page_row.data_ptr(), C, side, mean.data_ptr(), codes.data_ptr(), scales.data_ptr(),
                     mins.data_ptr(), _dev.stream())
            out[f"{name}_mean"] = mean
            out[f"{name}_dev"] = QuantizedDeviation(lay.bits, C, self.H, self.D, codes, scales, mins)
        out["residual_k"] = self.res_k[layer][b, :r].clone()
        out["residual_v"] = self.res_v[layer][b, :r].clone()
        return out

    def load(self, layer: int, b: int, k_mean, v_mean, k_dev: QuantizedDeviation, v_dev: QuantizedDeviation,
             residual_k, residual_v) -> None:
        """Replace one (layer, sequence)'s contents from dense reference-layout arrays (deserialize path)."""
        C = int(k_mean.shape[0])
        r = int(residual_k.shape[0])
        if self.B != 1:
            raise StateError("load() is only supported on single-sequence caches")
        if r > max(self.R, 1) or (self.R == 0 and r):
            raise CapacityError("residual rows exceed residual_length")
        self._ensure_pages(C)
        for side, mean, rec in ((0, k_mean, k_dev), (1, v_mean, v_dev)):
            codes, scales, mins = rec.device_tensors()
            m = _dev.to_dev(mean, allow_bf16=False)
            if C:
                call("tada_scatter_compressed", self._layout_ptr(layer), self.pools[layer].data_ptr(),
                     self.page_table[b].contiguous().data_ptr(), C, side, m.data_ptr(), codes.data_ptr(),
                     scales.data_ptr(), mins.data_ptr(), _dev.stream())
        if r:
            self.res_k[layer][b, :r].copy_(_dev.to_dev(residual_k, allow_bf16=False))
            self.res_v[layer][b, :r].copy_(_dev.to_dev(residual_v, allow_bf16=False))
        self.comp_host[layer, b] = C
        self.res_host[layer, b] = r
        self.comp_len[layer, b] = C
        self.res_len[layer, b] = r
