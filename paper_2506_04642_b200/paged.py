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
from ._lib import TADA_ERR_CONFIG, call, check, page_layout
from .errors import CapacityError, ConfigError, DataError, ShapeError, StateError
from .quant import QuantizedDeviation, validate_bits

F32 = np.float32
RES_EAGER_ROWS = 4096  # residual rows allocated up front per (layer, sequence); longer residuals grow lazily


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
        # residual rows [B, cap, H, D] per layer: R rows up front (a decode step never allocates), except for
        # very long residual lengths, which grow on demand (_res_reserve) instead of allocating B*R*H*D*4 bytes
        rcap = max(1, min(self.R, RES_EAGER_ROWS))
        self.res_k = [torch.zeros((batch, rcap, num_kv_heads, head_dim), dtype=torch.float32, device=self.dev)
                      for _ in range(num_layers)]
        self.res_v = [torch.zeros_like(t) for t in self.res_k]
        self.err = _dev.ErrFlag()
        self._step_sync = torch.zeros((num_layers, batch), dtype=torch.int32, device=self.dev)  # K3 arrival counters
        # per-layer range words (K1 note_mean / note_scale): stored values beyond the tensor-core kernels' f16
        # operand range route K2 to its exact f32 path for that layer
        self.range = torch.zeros((num_layers, 2), dtype=torch.int32, device=self.dev)
        self._stale = False  # host length mirrors behind the device (after CUDA-graph replays)
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

    def _res_reserve(self, layer: int, rows: int) -> None:
        """Make the layer's residual buffers hold at least ``rows`` rows per sequence (geometric growth)."""
        cap = self.res_k[layer].shape[1]
        if rows <= cap:
            return
        new_cap = max(rows, min(2 * cap, max(self.R, rows)))
        for bufs in (self.res_k, self.res_v):
            grown = torch.zeros((self.B, new_cap, self.H, self.D), dtype=torch.float32, device=self.dev)
            grown[:, :cap].copy_(bufs[layer])
            bufs[layer] = grown

    # ------------------------------------------------------------------ bookkeeping
    def lengths(self, layer: int, b: int = 0) -> tuple[int, int]:
        """(compressed tokens, residual tokens) of one (layer, sequence)."""
        self._refresh()
        return int(self.comp_host[layer, b]), int(self.res_host[layer, b])

    def _refresh(self) -> None:
        """Re-read the device lengths after CUDA-graph replays advanced them (the host mirrors are stale)."""
        if self._stale:
            torch.cuda.current_stream().synchronize()
            self.comp_host[:] = self.comp_len.cpu().numpy()
            self.res_host[:] = self.res_len.cpu().numpy()
            self._stale = False

    def _layout_ptr(self, layer: int):
        import ctypes

        return ctypes.byref(self.layouts[layer])

    def _plan(self, layer: int, n) -> tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
        """Host mirror of the device's per-sequence append plan (seq_plan in tada_common.cuh, the reference's
        flush policy cache.py:154-180 per sequence): (ncomp, from_residual, from_new, residual_after)."""
        r = self.res_host[layer]
        n = np.broadcast_to(np.asarray(n, dtype=np.int64), r.shape)
        if self.R == 0:
            return n.copy(), np.zeros_like(r), n.copy(), r.copy()
        total = r + n
        ncomp = total // self.R * self.R
        cnt_res = np.where(ncomp > 0, np.minimum(r, ncomp), 0)
        return ncomp, cnt_res, ncomp - cnt_res, total - ncomp

    def _seq_counts(self, lengths, n: int):
        """Per-sequence row counts of a ragged append -> (host int64 [B], device int32 [B] or None)."""
        if lengths is None:
            return np.full(self.B, n, dtype=np.int64), None
        cnt = np.asarray(lengths, dtype=np.int64).reshape(-1)
        if cnt.shape != (self.B,) or (cnt < 0).any() or (cnt > n).any():
            raise ShapeError(f"lengths must be {self.B} counts in [0, {n}], got {lengths!r}")
        return cnt, torch.from_numpy(cnt.astype(np.int32)).to(self.dev)

    # ------------------------------------------------------------------ append (K1)
    def _k1_part(self, layer: int, part: int, src_k: int, src_v: int, dtype: int, n_max: int, stride: int,
                 n_new: int, seq_n, rope=None) -> None:
        pos, pos_stride, table, rows = (None, 0, None, 0) if rope is None else rope
        call("tada_quant_append_plan", self._layout_ptr(layer), self.pools[layer].data_ptr(), src_k, src_v, dtype,
             self.B, n_max, stride, self.page_table.data_ptr(), self.page_table.shape[1],
             self.comp_len[layer].data_ptr(), self.res_len[layer].data_ptr(), self.R, n_new, _dev.ptr(seq_n), part,
             _dev.ptr(pos), pos_stride, _dev.ptr(table), rows, self.err.ptr, self.range[layer].data_ptr(), _dev.stream())

    def _append_planned(self, layer: int, k: torch.Tensor, v: torch.Tensor, lengths, rope=None) -> None:
        """Device-planned append of [batch, n, H, D] rows (n_b = lengths[b] of them per sequence): K1 over the
        residual rows each flush compresses, K1 over the new rows it compresses, then the commit kernel
        (raw rows -> residual buffer, lengths advance).  Sequences may be at any mix of lengths."""
        n = int(k.shape[1])
        cnt, seq_n = self._seq_counts(lengths, n)
        if not cnt.any():
            return
        ncomp, cnt_res, cnt_new, res_after = self._plan(layer, cnt)
        C = self.comp_host[layer]
        self._ensure_pages(int((C + ncomp).max()))
        self._res_reserve(layer, int(res_after.max()))
        dt = _dev.dtype_code(k)
        if cnt_res.max() > 0:  # the buffered residual rows are the oldest tokens of the flushed blocks
            self._k1_part(layer, 1, self.res_k[layer].data_ptr(), self.res_v[layer].data_ptr(), 0,
                          int(cnt_res.max()), self.res_k[layer].shape[1], n, seq_n)
        if cnt_new.max() > 0:
            rope_k1 = None if rope is None else (rope[0], rope[0].shape[1], rope[1], int(rope[1].shape[0]))
            self._k1_part(layer, 2, k.data_ptr(), v.data_ptr(), dt, int(cnt_new.max()), n, n, seq_n, rope_k1)
        pos, table = (None, None) if rope is None else rope
        call("tada_append_commit", self.res_k[layer].data_ptr(), self.res_v[layer].data_ptr(),
             self.res_k[layer].shape[1], self.H, self.D, k.data_ptr(), v.data_ptr(), dt, self.B, n, n,
             _dev.ptr(seq_n), self.R, self.comp_len[layer].data_ptr(), self.res_len[layer].data_ptr(), _dev.ptr(pos),
             0 if pos is None else pos.shape[1], _dev.ptr(table), 0 if table is None else int(table.shape[0]),
             self.err.ptr, _dev.stream())
        self.comp_host[layer] += ncomp
        self.res_host[layer] = res_after

    def _check_rows(self, k: torch.Tensor, v: torch.Tensor) -> None:
        if k.ndim != 4 or tuple(k.shape[2:]) != (self.H, self.D) or k.shape[0] != self.B:
            raise ShapeError(f"keys must be ({self.B}, tokens, {self.H}, {self.D}), got {tuple(k.shape)}")
        if tuple(v.shape) != tuple(k.shape):
            raise ShapeError(f"values shape {tuple(v.shape)} does not match keys shape {tuple(k.shape)}")

    def _reflush_loaded(self, layer: int) -> None:
        """A deserialized stream may hold >= R raw rows (the reference accepts it; its next append flushes
        them): move them back through the planner as new rows so every later append sees r < R."""
        r = int(self.res_host[layer].max())
        rk = self.res_k[layer][:, :r].clone()
        rv = self.res_v[layer][:, :r].clone()
        lens = self.res_host[layer].copy()
        self.res_len[layer].zero_()
        self.res_host[layer] = 0
        self._append_planned(layer, rk, rv, lens)

    def append(self, layer: int, k: torch.Tensor, v: torch.Tensor, lengths=None) -> None:
        """Append already-rotated keys and values ``[batch, n, heads, head_dim]`` (cache.py:154-180) to every
        sequence — ``lengths[b]`` of the n rows for sequence b when given (ragged prefill) — with each
        sequence's flush decided on the device from its own residual count.

        Non-finite inputs set the device error flag; call :meth:`check_errors`
        (the drop-in ``CompressedLayerCache`` pre-checks instead, so it raises
        before mutating, like the reference).
        """
        self._check_rows(k, v)
        if int(k.shape[1]) == 0:
            return
        self._refresh()
        k = k.contiguous()
        v = v.contiguous()
        if k.dtype not in (torch.float32, torch.bfloat16) or v.dtype != k.dtype:
            k, v = k.float(), v.float()
        if self.R > 0 and (self.res_host[layer] >= self.R).any():
            self._reflush_loaded(layer)
        self._append_planned(layer, k, v, lengths)

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
                    rope, lengths=None) -> None:
        """Append pre-RoPE keys (rotated on the fly) and values ``[batch, n, heads, head_dim]``.

        ``pos``: device int32 ``[batch, n]`` (validated by the caller, max < n_pos).  Keys that reach the
        compressed region are rotated inside K1 (``tada_quant_append_plan`` with the table), keys that stay
        raw inside the commit kernel: the rotated keys never round-trip through HBM.  Bit-identical to
        rotating first and calling :meth:`append` (append_fused, model.py:167-183).
        """
        from .rope import rope_table

        self._check_rows(k, v)
        n = int(k.shape[1])
        if tuple(pos.shape) != (self.B, n):
            raise ShapeError(f"positions must be ({self.B}, {n}), got {tuple(pos.shape)}")
        if n == 0:
            return
        self._refresh()
        table = rope_table(rope, n_pos)
        pos = pos.to(device=self.dev, dtype=torch.int32).contiguous()
        k = k.contiguous()
        v = v.contiguous()
        if k.dtype not in (torch.float32, torch.bfloat16) or v.dtype != k.dtype:
            k, v = k.float(), v.float()
        bits = self.layouts[layer].bits
        if not (self.H == 8 and self.D == 128 and bits in (2, 4, 8)) or (
                self.R > 0 and (self.res_host[layer] >= self.R).any()):
            self.append(layer, self._rotate(k, pos, table), v.float(), lengths)  # generic geometry: compose
            return
        self._append_planned(layer, k, v, lengths, rope=(pos, table))

    def check_errors(self) -> None:
        """Raise DataError if any kernel saw a non-finite input since the last check (synchronising)."""
        if self.err.raised():
            raise DataError("cannot quantize non-finite values")

    def append_checked(self, layer: int, k: torch.Tensor, v: torch.Tensor, rope=None) -> None:
        """:meth:`append` (or :meth:`append_rope` with ``rope = (pos, n_pos, params)``) that raises DataError
        and leaves the layer unchanged when a kernel saw a non-finite row — the drop-in ``append_tokens``
        contract (cache.py:154-180) without a pre-pass over the input.  K1 flags the rows it compresses; on a
        flag the lengths (device and host) and the residual rows a flush overwrote are restored.  Rows that
        only enter the residual buffer are not inspected, like the reference, which raises when they flush."""
        self._refresh()
        comp, res = self.comp_host[layer].copy(), self.res_host[layer].copy()
        r = int(res.max())
        saved = None
        if self.R > 0 and r > 0:  # a flush rewrites residual rows [0, r_after) in place
            saved = (self.res_k[layer][:, :r].clone(), self.res_v[layer][:, :r].clone())
        if rope is None:
            self.append(layer, k, v)
        else:
            self.append_rope(layer, k, v, *rope)
        if not self.err.raised():
            return
        self.comp_len[layer].copy_(torch.from_numpy(comp.astype(np.int32)))
        self.res_len[layer].copy_(torch.from_numpy(res.astype(np.int32)))
        self.comp_host[layer], self.res_host[layer] = comp, res
        if saved is not None:
            self.res_k[layer][:, :r].copy_(saved[0])
            self.res_v[layer][:, :r].copy_(saved[1])
        raise DataError("cannot quantize non-finite values")

    # ------------------------------------------------------------------ attention (K2 + K3)
    def _out(self, out, hq: int, out_dtype) -> torch.Tensor:
        """The caller's output buffer, validated (the kernels write B*Hq*D elements to it), or a new one."""
        if out is None:
            return torch.empty((self.B, hq, self.D), dtype=out_dtype, device=self.dev)
        if (tuple(out.shape) != (self.B, hq, self.D) or not out.is_contiguous() or out.device != self.dev
                or out.dtype not in (torch.float32, torch.bfloat16)):
            raise ShapeError(f"out must be a contiguous f32/bf16 ({self.B}, {hq}, {self.D}) tensor on {self.dev}, got "
                             f"{tuple(out.shape)} {out.dtype} on {out.device}")
        return out

    def workspace(self, num_q_heads: int, splits: int) -> torch.Tensor | None:
        from ._lib import load

        nbytes = int(load().tada_decode_attn_workspace_bytes(self.B, num_q_heads, self.D, splits))
        if nbytes == 0:
            return None
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)
        return self._ws

    def suggest_splits(self, layer: int, num_q_heads: int | None = None, mode: int = 0) -> int:
        """Split-K factor for this layer's kernel in ``mode`` (whole waves of resident CTAs on this device)."""
        from ._lib import load

        self._refresh()
        tokens = int((self.comp_host[layer] + self.res_host[layer]).max())
        if num_q_heads is None:
            return int(load().tada_decode_attn_suggest_splits(self.B, tokens, self.P))
        return int(load().tada_decode_attn_plan_splits_mode(self._layout_ptr(layer), num_q_heads, self.B, tokens, mode))

    def attend(self, layer: int, q: torch.Tensor, out: torch.Tensor | None = None, out_dtype=torch.float32,
               num_splits: int | None = None, mode: int = 0, scale: float | None = None) -> torch.Tensor:
        """Decode attention for one query per sequence: ``q [batch, Hq, D]`` -> ``[batch, Hq, D]``.

        attend_streaming semantics (attention.py:103-151) over compressed then
        residual tokens, GQA map kv = g*H // Hq (attention.py:47-49).
        """
        if q.ndim != 3 or q.shape[0] != self.B or q.shape[2] != self.D or q.shape[1] % self.H:
            raise ShapeError(f"query must be ({self.B}, Hq, {self.D}) with Hq a multiple of {self.H}, got "
                             f"{tuple(q.shape)}")
        self._refresh()
        if ((self.comp_host[layer] + self.res_host[layer]) == 0).any():
            raise StateError("cannot attend over an empty cache")
        hq = int(q.shape[1])
        if q.dtype not in (torch.float32, torch.bfloat16):
            q = q.float()
        q = q.contiguous()
        splits = num_splits or self.suggest_splits(layer, hq, mode)
        ws = self.workspace(hq, splits)
        out = self._out(out, hq, out_dtype)
        sc = np.float32(1.0 / math.sqrt(self.D)) if scale is None else np.float32(scale)
        call("tada_decode_attn", self._layout_ptr(layer), self.pools[layer].data_ptr(), q.data_ptr(),
             _dev.dtype_code(q), self.B, hq, self.page_table.data_ptr(), self.page_table.shape[1],
             self.comp_len[layer].data_ptr(), self.res_len[layer].data_ptr(), self.res_k[layer].data_ptr(),
             self.res_v[layer].data_ptr(), self.res_k[layer].shape[1], float(sc), splits, _dev.ptr(ws),
             out.data_ptr(), _dev.dtype_code(out), mode, self.range[layer].data_ptr(), _dev.stream())
        return out

    def append_attend(self, layer: int, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                      out: torch.Tensor | None = None, out_dtype=torch.float32, num_splits: int | None = None,
                      mode: int = 0, scale: float | None = None, _capture: bool = False) -> torch.Tensor:
        """One decode step of a layer: :meth:`append` of one token per sequence (``k``, ``v``:
        ``[batch, 1, heads, head_dim]``, rotated) then :meth:`attend` — model.py:280-281 — for sequences at
        any mix of lengths.

        On the tensor-core path this is one call (``tada_decode_step``): each sequence's flush is decided
        on the device (K1 runs over the sequences whose residual fills up), K2 attends the compressed
        tokens, K3 attends the residual rows plus the new row straight from the input, stores it, and
        advances the lengths — no host branch on lengths, so the step is CUDA-graph capturable
        (:class:`DecodeGraph`).  Otherwise this is exactly append() + attend()."""
        from ._lib import load

        fused_ok = (tuple(k.shape) == (self.B, 1, self.H, self.D) and tuple(v.shape) == tuple(k.shape)
                    and k.device == self.dev and v.device == self.dev
                    and mode != 1 and k.dtype in (torch.float32, torch.bfloat16) and v.dtype == k.dtype
                    and q.ndim == 3 and q.shape[0] == self.B and q.shape[2] == self.D and q.shape[1] % self.H == 0)
        if not _capture:
            self._refresh()
            if self.R > 0 and (self.res_host[layer] >= self.R).any():
                fused_ok = False  # a deserialized stream with >= R raw rows: append() re-flushes them first
        if not fused_ok:
            if _capture:
                raise ConfigError("this decode step cannot be captured: it needs the tensor-core path")
            self.append(layer, k, v)
            return self.attend(layer, q, out=out, out_dtype=out_dtype, num_splits=num_splits, mode=mode, scale=scale)
        hq = int(q.shape[1])
        if q.dtype not in (torch.float32, torch.bfloat16):
            q = q.float()
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
        if _capture:  # every sequence may flush at any replay: K1 covers the longest possible residual
            k1_rows = max(self.R - 1, 0)
        else:
            ncomp, cnt_res, _, res_after = self._plan(layer, 1)
            k1_rows = int(cnt_res.max()) if ncomp.any() else -1
            self._ensure_pages(max(1, int((self.comp_host[layer] + ncomp).max())))
            self._res_reserve(layer, int(res_after.max()))
        splits = num_splits or self.suggest_splits(layer, hq, mode)
        ws = self.workspace(hq, splits)
        out = self._out(out, hq, out_dtype)
        sc = np.float32(1.0 / math.sqrt(self.D)) if scale is None else np.float32(scale)
        rc = load().tada_decode_step(
            self._layout_ptr(layer), self.pools[layer].data_ptr(), q.data_ptr(), _dev.dtype_code(q), self.B, hq,
            self.page_table.data_ptr(), self.page_table.shape[1], self.comp_len[layer].data_ptr(),
            self.res_len[layer].data_ptr(), self.res_k[layer].data_ptr(), self.res_v[layer].data_ptr(),
            self.res_k[layer].shape[1], self.R, k.data_ptr(), v.data_ptr(), _dev.dtype_code(k), k1_rows,
            self._step_sync[layer].data_ptr(), float(sc), splits, _dev.ptr(ws), out.data_ptr(), _dev.dtype_code(out),
            mode, self.err.ptr, self.range[layer].data_ptr(), _dev.stream())
        if rc == TADA_ERR_CONFIG and not _capture:  # geometry without the tensor-core path: nothing was enqueued
            self.append(layer, k, v)
            return self.attend(layer, q, out=out, out_dtype=out_dtype, num_splits=num_splits, mode=mode, scale=scale)
        check(rc)
        if not _capture:
            self.comp_host[layer] += ncomp
            self.res_host[layer] = res_after
        return out

    def attend_lse(self, layer: int, q: torch.Tensor, num_splits: int | None = None, mode: int = 0,
                   scale: float | None = None) -> tuple[torch.Tensor, torch.Tensor]:
        """Like :meth:`attend` (f32 out) and also the log-sum-exp ``[batch, Hq]`` of the scaled logits.

        ``(out, lse)`` pairs over disjoint token sets merge exactly (shard.merge_partials).
        """
        if q.ndim != 3 or q.shape[0] != self.B or q.shape[2] != self.D or q.shape[1] % self.H:
            raise ShapeError(f"query must be ({self.B}, Hq, {self.D}) with Hq a multiple of {self.H}, got "
                             f"{tuple(q.shape)}")
        self._refresh()
        if ((self.comp_host[layer] + self.res_host[layer]) == 0).any():
            raise StateError("cannot attend over an empty cache")
        hq = int(q.shape[1])
        if q.dtype not in (torch.float32, torch.bfloat16):
            q = q.float()
        q = q.contiguous()
        splits = num_splits or self.suggest_splits(layer, hq, mode)
        ws = self.workspace(hq, splits)
        out = torch.empty((self.B, hq, self.D), dtype=torch.float32, device=self.dev)
        lse = torch.empty((self.B, hq), dtype=torch.float32, device=self.dev)
        sc = np.float32(1.0 / math.sqrt(self.D)) if scale is None else np.float32(scale)
        call("tada_decode_attn_lse", self._layout_ptr(layer), self.pools[layer].data_ptr(), q.data_ptr(),
             _dev.dtype_code(q), self.B, hq, self.page_table.data_ptr(), self.page_table.shape[1],
             self.comp_len[layer].data_ptr(), self.res_len[layer].data_ptr(), self.res_k[layer].data_ptr(),
             self.res_v[layer].data_ptr(), self.res_k[layer].shape[1], float(sc), splits, _dev.ptr(ws),
             out.data_ptr(), _dev.dtype_code(out), mode, lse.data_ptr(), self.range[layer].data_ptr(), _dev.stream())
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

    def _note_range(self, layer: int, mean: torch.Tensor, scales: torch.Tensor) -> None:
        """The range words K1 keeps (note_mean / note_scale in tada_quant.cu) for values that arrive by import:
        the binary exponent of max |mean| when >= 2^15 and of max scale when >= 2^8, on the device (no sync)."""
        for word, vals, floor in ((0, mean, 32768.0), (1, scales, 256.0)):
            a = torch.nan_to_num(vals.float().abs().max(), nan=3.0e38, posinf=3.0e38)
            e = (torch.frexp(a)[1] - 1).to(torch.int32)
            e = torch.where(a >= floor, e, torch.zeros_like(e))
            self.range[layer, word] = torch.maximum(self.range[layer, word], e)

    def load(self, layer: int, b: int, k_mean, v_mean, k_dev: QuantizedDeviation, v_dev: QuantizedDeviation,
             residual_k, residual_v) -> None:
        """Replace one (layer, sequence)'s contents from dense reference-layout arrays (deserialize path)."""
        C = int(k_mean.shape[0])
        r = int(residual_k.shape[0])
        if self.B != 1:
            raise StateError("load() is only supported on single-sequence caches")
        self._res_reserve(layer, r)  # r may exceed R in a deserialized stream (the reference accepts it)
        self._ensure_pages(C)
        for side, mean, rec in ((0, k_mean, k_dev), (1, v_mean, v_dev)):
            codes, scales, mins = rec.device_tensors()
            m = _dev.to_dev(mean, allow_bf16=False)
            if C:
                call("tada_scatter_compressed", self._layout_ptr(layer), self.pools[layer].data_ptr(),
                     self.page_table[b].contiguous().data_ptr(), C, side, m.data_ptr(), codes.data_ptr(),
                     scales.data_ptr(), mins.data_ptr(), _dev.stream())
                self._note_range(layer, m, scales)
        if r:
            self.res_k[layer][b, :r].copy_(_dev.to_dev(residual_k, allow_bf16=False))
            self.res_v[layer][b, :r].copy_(_dev.to_dev(residual_v, allow_bf16=False))
        self.comp_host[layer, b] = C
        self.res_host[layer, b] = r
        self.comp_len[layer, b] = C
        self.res_len[layer, b] = r


class DecodeGraph:
    """One decode step of every layer of a :class:`PagedKVCache`, captured once as a CUDA graph and replayed.

    The step is ``append_attend`` per layer (``tada_decode_step``: K1 over the sequences whose residual
    fills, K2, K3 with the length bookkeeping), all decisions on the device, so one capture serves every
    later step whatever the per-sequence lengths (ragged batches included).  Inputs are copied into the
    static buffers ``q [L, B, Hq, D]``, ``k`` / ``v`` ``[L, B, 1, H, D]`` before :meth:`replay`; outputs land
    in ``out [L, B, Hq, D]``.  The cache must be pre-sized (``max_tokens``) so no page is allocated during a
    step; the split count per layer is fixed at capture.  After replays the host length mirrors are
    refreshed lazily (one synchronising read) by the next host-side call.
    """

    def __init__(self, store: PagedKVCache, num_q_heads: int, dtype=torch.bfloat16, out_dtype=torch.bfloat16,
                 num_splits: dict | None = None, mode: int = 0):
        if store.growable:
            raise ConfigError("DecodeGraph needs a pre-sized cache (PagedKVCache(max_tokens=...))")
        if store.R > RES_EAGER_ROWS:
            raise ConfigError(f"DecodeGraph needs residual_length <= {RES_EAGER_ROWS}")
        store._refresh()
        if store.R > 0 and (store.res_host >= store.R).any():
            raise StateError("flush the deserialized residual rows (one eager append) before capturing")
        self.store = store
        L, B, H, D = store.L, store.B, store.H, store.D
        dev = store.dev
        self.q = torch.zeros((L, B, num_q_heads, D), dtype=dtype, device=dev)
        self.k = torch.zeros((L, B, 1, H, D), dtype=dtype, device=dev)
        self.v = torch.zeros((L, B, 1, H, D), dtype=dtype, device=dev)
        self.out = torch.zeros((L, B, num_q_heads, D), dtype=out_dtype, device=dev)
        self.splits = [int((num_splits or {}).get(store.plan[i]) or store.suggest_splits(i, num_q_heads))
                       for i in range(L)]
        for i in range(L):  # workspace, residual buffers and kernel attributes exist before capture
            store.workspace(num_q_heads, self.splits[i])
            store._res_reserve(i, max(store.R, 1))
        from ._lib import load

        load().tada_decode_attn_plan_splits(store._layout_ptr(0), num_q_heads, B, 1)
        self.mode = mode
        self.graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(self.graph, stream=side):
                self._step()
        torch.cuda.current_stream().wait_stream(side)

    def _step(self):
        for i in range(self.store.L):
            self.store.append_attend(i, self.q[i], self.k[i], self.v[i], out=self.out[i], num_splits=self.splits[i],
                                     mode=self.mode, _capture=True)

    def replay(self) -> torch.Tensor:
        """Run one captured decode step (on the current stream); returns the static output buffer."""
        self.graph.replay()
        self.store._stale = True
        return self.out
