"""Decode attention over the compressed cache — drop-in for ``tadakv.attention``.

``attend_streaming`` keeps the reference signature (attention.py:103-151) and
runs the split-K flash-decoding kernel (K2) + log-sum-exp combine (K3) in
libtadakv_b200.so.  The reference's ``block`` (tile length) only changes the
float summation order there, so it is validated and accepted; the kernel
picks its own tiles.  ``attend_naive`` (attention.py:66-91) is the same
computation with a single split (no combine), kept for API parity.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev
from .cache import CompressedLayerCache, ModelConfig
from .errors import ConfigError, ShapeError, StateError

F32 = np.float32


@dataclass(frozen=True)
class BlockSpec:
    """Streaming tile length along the token axis (attention.py:28-36)."""

    block_tokens: int = 64

    def __post_init__(self) -> None:
        if self.block_tokens < 1:
            raise ConfigError(f"block_tokens must be >= 1, got {self.block_tokens}")


@dataclass
class AttentionOutput:
    """Per-query-head output with optional score rows (attention.py:39-44)."""

    output: object
    scores: list | None = None


def kv_head_index(q_head: int, num_q_heads: int, num_kv_heads: int) -> int:
    """KV head serving a query head under GQA (attention.py:47-49)."""
    return q_head * num_kv_heads // num_q_heads


def _check_query(q, layer: CompressedLayerCache, cfg: ModelConfig) -> torch.Tensor:
    qd = _dev.to_dev(q)
    if tuple(qd.shape) != (cfg.num_q_heads, cfg.head_dim):
        raise ShapeError(f"query must be ({cfg.num_q_heads}, {cfg.head_dim}), got {tuple(qd.shape)}")
    if (layer.num_kv_heads, layer.head_dim) != (cfg.num_kv_heads, cfg.head_dim):
        raise ShapeError(f"cache geometry ({layer.num_kv_heads}, {layer.head_dim}) does not match "
                         f"config ({cfg.num_kv_heads}, {cfg.head_dim})")
    return qd


def _scores(q: torch.Tensor, layer: CompressedLayerCache, cfg: ModelConfig) -> list:
    """Softmax score rows (return_scores=True); a diagnostic, computed on the device with torch."""
    from .quant import dequantize_tensor

    ex = layer.export_device()
    g = cfg.num_q_heads // cfg.num_kv_heads
    k_hat = ex["k_mean"][:, None, :] - dequantize_tensor(ex["k_dev"])
    k_all = torch.cat([k_hat, ex["residual_k"]])
    sc = float(F32(1.0 / math.sqrt(cfg.head_dim)))
    rows = []
    for h in range(cfg.num_q_heads):
        logits = (k_all[:, h // g, :] @ q[h].float()) * sc
        rows.append(_dev.host(torch.softmax(logits, dim=0)))
    return rows


def _attend(q, layer, cfg, return_scores, splits):
    qd = _check_query(q, layer, cfg)
    if layer.total_tokens == 0:
        raise StateError("cannot attend over an empty cache")
    out = layer.store.attend(0, qd.unsqueeze(0), num_splits=splits, mode=1)[0]
    scores = _scores(qd, layer, cfg) if return_scores else None
    return AttentionOutput(output=out if isinstance(q, torch.Tensor) else _dev.host(out), scores=scores)


def attend_naive(q, layer: CompressedLayerCache, cfg: ModelConfig, return_scores: bool = False) -> AttentionOutput:
    """Single-position attention over the whole cache (attention.py:66-91).  The reference does one pass; the
    device runs the same exact kernel split-K like attend_streaming (only the f32 summation order differs, well
    inside the reference's own 1e-5 streaming-vs-naive bar), so a long cache is not one CTA's work."""
    return _attend(q, layer, cfg, return_scores, splits=None)


def attend_streaming(q, layer: CompressedLayerCache, cfg: ModelConfig, block: BlockSpec = BlockSpec(),
                     return_scores: bool = False) -> AttentionOutput:
    """Tiled online-softmax attention on the B200 (attention.py:103-151)."""
    if not isinstance(block, BlockSpec):
        raise ConfigError("block must be a BlockSpec")
    return _attend(q, layer, cfg, return_scores, splits=None)
