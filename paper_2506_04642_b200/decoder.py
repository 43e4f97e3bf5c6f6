"""The reference toy decoder run on the GPU around the compressed KV path.

Mirrors ``tadakv.model`` (model.py:196-330): ``_forward_full`` / ``prefill_forward``, ``decode_step`` and
``generate``, batched over sequences of equal length.  The dense layers (embedding, RMSNorm, the
projections, the MLP, the prompt's causal attention) are torch f32 on the GPU (cuBLAS with TF32 off) —
plumbing around the path.  Everything that touches the KV cache is the library:

* prefill and decode keys are rotated inside K1 (``tada_quant_append_rope``; ``tada_apply_rope`` +
  K1 for geometries the fused kernel does not cover), values appended as projected;
* every layer's width comes from the ``PrecisionPlan`` (one ``PagedKVCache`` pool per layer, one shared
  page table) with the residual/flush policy of cache.py:154-180;
* decode attention is K2 + K3 (``tada_decode_attn``).

The query of a decode step is rotated by ``tada_apply_rope`` with the same host-built table.
"""

from __future__ import annotations

import math
from dataclasses import replace

import numpy as np
import torch

from . import _dev
from .cache import ModelConfig, PrecisionPlan
from .errors import CapacityError, ConfigError, DataError, ShapeError, StateError
from .paged import PagedKVCache
from .rope import _positions, rope_table

F32 = np.float32


def expected_weight_shapes(cfg: ModelConfig, vocab_size: int) -> dict[str, tuple[int, ...]]:
    """model.py:41-56."""
    d_model = cfg.num_q_heads * cfg.head_dim
    d_ff = 4 * d_model
    shapes = {"tok_emb": (vocab_size, d_model)}
    for i in range(cfg.num_layers):
        shapes[f"layers.{i}.attn_norm"] = (d_model,)
        shapes[f"layers.{i}.wq"] = (d_model, cfg.num_q_heads * cfg.head_dim)
        shapes[f"layers.{i}.wk"] = (d_model, cfg.num_kv_heads * cfg.head_dim)
        shapes[f"layers.{i}.wv"] = (d_model, cfg.num_kv_heads * cfg.head_dim)
        shapes[f"layers.{i}.wo"] = (cfg.num_q_heads * cfg.head_dim, d_model)
        shapes[f"layers.{i}.ffn_norm"] = (d_model,)
        shapes[f"layers.{i}.w1"] = (d_model, d_ff)
        shapes[f"layers.{i}.w2"] = (d_ff, d_model)
    shapes["final_norm"] = (d_model,)
    shapes["lm_head"] = (d_model, vocab_size)
    return shapes


class ToyDecoder:
    """GPU decoder for a ``tadakv.model.ToyModel``'s weights (model.py:60-87) with a compressed KV cache.

    ``weights``: name -> array of the shapes :func:`expected_weight_shapes` gives (numpy or torch).
    ``mode``: decode-attention kernel (0 auto, 1 exact generic, 2 tensor-core), as in PagedKVCache.attend.
    """

    def __init__(self, weights: dict, cfg: ModelConfig, vocab_size: int, max_seq_len: int = 4096,
                 batch: int = 1, mode: int = 0, page_tokens: int = 64):
        if vocab_size <= 0 or max_seq_len <= 0:
            raise ConfigError("vocab_size and max_seq_len must be positive")
        shapes = expected_weight_shapes(cfg, vocab_size)
        if set(weights) != set(shapes):  # ToyModel.__post_init__ (model.py:69-87) raises ConfigError
            raise ConfigError(f"weight names mismatch: missing {sorted(set(shapes) - set(weights))}, "
                              f"unexpected {sorted(set(weights) - set(shapes))}")
        dev = _dev.device()
        self.w = {}
        for name, shape in shapes.items():
            t = _dev.to_dev(weights[name], allow_bf16=False)
            if tuple(t.shape) != shape:
                raise ConfigError(f"weight {name} has shape {tuple(t.shape)}, expected {shape}")
            self.w[name] = t
        self.cfg, self.vocab_size, self.max_seq_len, self.B, self.mode = cfg, vocab_size, max_seq_len, batch, mode
        self.page_tokens = page_tokens
        self.dev = dev
        self.store: PagedKVCache | None = None
        self.position = 0

    # ------------------------------------------------------------------ building blocks (model.py:153-160)
    @staticmethod
    def _rmsnorm(x: torch.Tensor, w: torch.Tensor, eps: float = 1e-5) -> torch.Tensor:
        ms = torch.mean(x * x, dim=-1, keepdim=True)
        return x / torch.sqrt(ms + F32(eps)) * w

    @staticmethod
    def _silu(x: torch.Tensor) -> torch.Tensor:
        return x / (1.0 + torch.exp(-x))

    def _mm(self, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
        return a @ b

    def _rotate(self, x: torch.Tensor, pos: torch.Tensor, top: int) -> torch.Tensor:
        """[B, n, heads, D] -> rotated f32 (tada_apply_rope); pos [B, n]."""
        return self.store._rotate(x, pos, rope_table(self.cfg.rope, top))

    def _ids(self, token_ids) -> torch.Tensor:
        if isinstance(token_ids, torch.Tensor):
            ids = token_ids.detach().to("cpu", torch.int64)
        else:
            ids = torch.as_tensor(np.asarray(token_ids), dtype=torch.int64)
        if ids.ndim == 1:
            ids = ids.unsqueeze(0)
        if ids.ndim != 2 or ids.shape[0] != self.B:
            raise ShapeError(f"token ids must be ({self.B}, n), got {tuple(ids.shape)}")
        if ids.numel() and (int(ids.min()) < 0 or int(ids.max()) >= self.vocab_size):
            bad = int(ids.min()) if int(ids.min()) < 0 else int(ids.max())
            raise DataError(f"token id {bad} outside vocabulary of size {self.vocab_size}")
        return ids.to(self.dev)

    # ------------------------------------------------------------------ prefill (model.py:196-254)
    def prefill(self, token_ids) -> torch.Tensor:
        """Run the prompt, filling a fresh cache; returns logits ``[B, n, vocab]`` (f32)."""
        ids = self._ids(token_ids)
        B, n = ids.shape
        if n == 0:
            raise DataError("prompt must be non-empty")
        if n > self.max_seq_len:
            raise CapacityError(f"prompt of {n} tokens exceeds max_seq_len {self.max_seq_len}")
        cfg, w = self.cfg, self.w
        self.store = PagedKVCache(cfg.num_layers, cfg.num_kv_heads, cfg.head_dim, cfg.plan.bits_per_layer,
                                  cfg.residual_length, batch=B, page_tokens=self.page_tokens,
                                  max_tokens=self.max_seq_len)
        pos_np = np.tile(np.arange(n), (B, 1))
        pos, top = _positions(pos_np, n, B)
        hq, h, d = cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim
        g = hq // h
        inv_sqrt_d = F32(1.0 / math.sqrt(d))
        causal = torch.triu(torch.full((n, n), float("-inf"), device=self.dev), diagonal=1)
        x = w["tok_emb"][ids]
        for i in range(cfg.num_layers):
            hn = self._rmsnorm(x, w[f"layers.{i}.attn_norm"])
            q = self._mm(hn, w[f"layers.{i}.wq"]).reshape(B, n, hq, d)
            k = self._mm(hn, w[f"layers.{i}.wk"]).reshape(B, n, h, d)
            v = self._mm(hn, w[f"layers.{i}.wv"]).reshape(B, n, h, d).contiguous()
            q_rot = self._rotate(q, pos, top)
            self.store.append_rope(i, k.contiguous(), v, pos, top, cfg.rope)  # the rotated keys stay on chip
            k_rot = self._rotate(k, pos, top)  # the prompt's own raw attention (prefill_attend, attention.py:154-189)
            kv = torch.arange(hq, device=self.dev) // g
            logits = torch.einsum("bqgd,bkgd->bgqk", q_rot, k_rot[:, :, kv]) * inv_sqrt_d + causal
            p = torch.exp(logits - logits.amax(dim=-1, keepdim=True))
            p = p / p.sum(dim=-1, keepdim=True)
            attn = torch.einsum("bgqk,bkgd->bqgd", p, v[:, :, kv])
            x = x + self._mm(attn.reshape(B, n, -1), w[f"layers.{i}.wo"])
            h2 = self._rmsnorm(x, w[f"layers.{i}.ffn_norm"])
            x = x + self._mm(self._silu(self._mm(h2, w[f"layers.{i}.w1"])), w[f"layers.{i}.w2"])
        self.position = n
        return self._mm(self._rmsnorm(x, w["final_norm"]), w["lm_head"])

    def reset(self, cfg: ModelConfig | None = None) -> None:
        """Fresh empty caches (optionally for another plan / residual length of the same geometry):
        ``new_caches`` (model.py:163-164); the device weights are kept."""
        if cfg is not None:
            if (cfg.num_layers, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim) != (
                    self.cfg.num_layers, self.cfg.num_q_heads, self.cfg.num_kv_heads, self.cfg.head_dim):
                raise ConfigError("reset() keeps the weights: the geometry must not change")
            self.cfg = cfg
        c = self.cfg
        self.store = PagedKVCache(c.num_layers, c.num_kv_heads, c.head_dim, c.plan.bits_per_layer, c.residual_length,
                                  batch=self.B, page_tokens=self.page_tokens, max_tokens=self.max_seq_len)
        self.position = 0

    # ------------------------------------------------------------------ decode (model.py:257-289)
    def decode_step(self, token_ids, position: int) -> torch.Tensor:
        """Append one token per sequence at ``position`` and return next-token logits ``[B, vocab]``."""
        if self.store is None:
            self.reset()
        ids = self._ids(np.asarray(token_ids).reshape(self.B, 1))
        if position != self.position:  # model.py:282-286
            raise StateError(f"layer 0 cache holds {self.position} tokens but position is {position}")
        if position >= self.max_seq_len:
            raise CapacityError(f"position {position} exceeds max_seq_len {self.max_seq_len}")
        cfg, w, B = self.cfg, self.w, self.B
        hq, h, d = cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim
        pos, top = _positions(np.full((B, 1), position), 1, B)
        x = w["tok_emb"][ids[:, 0]]
        for i in range(cfg.num_layers):
            hn = self._rmsnorm(x, w[f"layers.{i}.attn_norm"])
            q = self._mm(hn, w[f"layers.{i}.wq"]).reshape(B, 1, hq, d)
            q_rot = self._rotate(q, pos, top)[:, 0]
            k = self._mm(hn, w[f"layers.{i}.wk"]).reshape(B, 1, h, d).contiguous()
            v = self._mm(hn, w[f"layers.{i}.wv"]).reshape(B, 1, h, d).contiguous()
            self.store.append_rope(i, k, v, pos, top, cfg.rope)  # append_fused (model.py:167-183)
            attn = self.store.attend(i, q_rot, out_dtype=torch.float32, mode=self.mode)
            x = x + self._mm(attn.reshape(B, -1), w[f"layers.{i}.wo"])
            h2 = self._rmsnorm(x, w[f"layers.{i}.ffn_norm"])
            x = x + self._mm(self._silu(self._mm(h2, w[f"layers.{i}.w1"])), w[f"layers.{i}.w2"])
        self.position += 1
        return self._mm(self._rmsnorm(x, w["final_norm"]), w["lm_head"])

    # ------------------------------------------------------------------ generate (model.py:292-330)
    def generate(self, prompt_ids, max_new_tokens: int) -> np.ndarray:
        """Greedy generation with the compressed cache; returns ``[B, n + max_new_tokens]`` token ids."""
        ids = self._ids(prompt_ids)
        if ids.shape[1] == 0:
            raise DataError("prompt must be non-empty")
        if max_new_tokens < 0:
            raise ConfigError(f"max_new_tokens must be non-negative, got {max_new_tokens}")
        if ids.shape[1] + max_new_tokens > self.max_seq_len:
            raise CapacityError(f"{ids.shape[1]} prompt + {max_new_tokens} new tokens exceeds "
                                f"max_seq_len {self.max_seq_len}")
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        try:
            logits = self.prefill(ids)[:, -1]
            out = [ids.cpu().numpy()]
            for step in range(max_new_tokens):
                nxt = torch.argmax(logits, dim=-1)
                out.append(nxt.cpu().numpy()[:, None])
                if step + 1 < max_new_tokens:
                    logits = self.decode_step(nxt.cpu().numpy(), self.position)
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev
        self.store.check_errors()
        return np.concatenate(out, axis=1)


def generate(weights: dict, cfg: ModelConfig, vocab_size: int, prompt_ids, max_new_tokens: int, *,
             plan: PrecisionPlan | None = None, residual_length: int | None = None, max_seq_len: int = 4096,
             mode: int = 0) -> list[int]:
    """``tadakv.model.generate`` (model.py:292-330) for one prompt on the GPU."""
    if plan is not None:
        cfg = replace(cfg, plan=plan)
    if residual_length is not None:
        cfg = replace(cfg, residual_length=residual_length)
    dec = ToyDecoder(weights, cfg, vocab_size, max_seq_len=max_seq_len, batch=1, mode=mode)
    return [int(t) for t in dec.generate(np.asarray(prompt_ids)[None, :], max_new_tokens)[0]]
