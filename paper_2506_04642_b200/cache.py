"""Compressed KV cache — drop-in for ``tadakv.cache`` (pkg/src/tadakv/cache.py).

``CompressedLayerCache`` keeps the reference's constructor, properties and
attributes, but its state lives in HBM as a one-sequence, one-layer view of
:class:`~paper_2506_04642_b200.paged.PagedKVCache`; appends run the fused
quantize-on-append kernel (K1) and reads of ``k_mean`` / ``k_dev`` / ... export
the paged layout back to the reference's dense layout (numpy / bytes), which is
what makes the TADAKV1 byte-for-byte parity check possible.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev
from ._lib import call
from .errors import ConfigError, DataError, FormatError, ShapeError
from .paged import PagedKVCache
from .quant import ALLOWED_WIDTHS, QuantizedDeviation, validate_bits

F32 = np.float32
CACHE_MAGIC = b"TADAKV1"


@dataclass(frozen=True)
class RopeParams:
    """Rotary geometry carried by ModelConfig (tensor.py:53-66)."""

    head_dim: int
    base: float = 10000.0

    def __post_init__(self) -> None:
        if self.head_dim <= 0 or self.head_dim % 2 != 0:
            raise ConfigError(f"rotary head_dim must be a positive even integer, got {self.head_dim}")
        if self.base <= 0:
            raise ConfigError(f"rotary base must be positive, got {self.base}")


@dataclass(frozen=True)
class PrecisionPlan:
    """Per-layer deviation bit widths for K and V (cache.py:38-63): the per-layer precision dispatch."""

    bits_per_layer: tuple

    def __post_init__(self) -> None:
        if not self.bits_per_layer:
            raise ConfigError("a precision plan needs at least one layer")
        for bits in self.bits_per_layer:
            validate_bits(bits)
        object.__setattr__(self, "bits_per_layer", tuple(int(b) for b in self.bits_per_layer))

    @classmethod
    def uniform(cls, bits: int, num_layers: int) -> "PrecisionPlan":
        return cls(tuple([bits] * num_layers))

    def __len__(self) -> int:
        return len(self.bits_per_layer)

    def __getitem__(self, layer_idx: int) -> int:
        return self.bits_per_layer[layer_idx]

    @property
    def mean_bits(self) -> float:
        return sum(self.bits_per_layer) / len(self.bits_per_layer)


@dataclass(frozen=True)
class ModelConfig:
    """Geometry + cache policy (cache.py:66-95)."""

    num_layers: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    residual_length: int
    rope: RopeParams
    plan: PrecisionPlan

    def __post_init__(self) -> None:
        if min(self.num_layers, self.num_q_heads, self.num_kv_heads, self.head_dim) <= 0:
            raise ConfigError("layer/head/dimension counts must be positive")
        if self.residual_length < 0:
            raise ConfigError(f"residual_length must be non-negative, got {self.residual_length}")
        if self.num_q_heads % self.num_kv_heads != 0:
            raise ConfigError(f"num_q_heads ({self.num_q_heads}) must be a multiple of "
                              f"num_kv_heads ({self.num_kv_heads})")
        if len(self.plan) != self.num_layers:
            raise ConfigError(f"plan covers {len(self.plan)} layers but the model has {self.num_layers}")
        if self.rope.head_dim != self.head_dim:
            raise ConfigError(f"rotary head_dim {self.rope.head_dim} does not match head_dim {self.head_dim}")


def mean_center(x):
    """(tokens, heads, head_dim) -> (mean [tokens, head_dim], dev = mean - x) (cache.py:98-111).

    fp64 head-order sum, /H, RNE to f32 — bit-exact, computed by ``tada_mean_center``.
    """
    is_t = isinstance(x, torch.Tensor)
    xd = _dev.to_dev(x)
    if xd.ndim != 3:
        raise ShapeError(f"expected (tokens, heads, head_dim) input, got shape {tuple(xd.shape)}")
    t, h, d = xd.shape
    mean = torch.empty((t, d), dtype=torch.float32, device=xd.device)
    dev = torch.empty((t, h, d), dtype=torch.float32, device=xd.device)
    if t and h and d:
        call("tada_mean_center", xd.data_ptr(), _dev.dtype_code(xd), t, h, d, mean.data_ptr(), dev.data_ptr(), None,
             _dev.stream())
    return (mean, dev) if is_t else (_dev.host(mean), _dev.host(dev))


class CompressedLayerCache:
    """One layer's compressed KV state in HBM (cache.py:114-213), single writer."""

    def __init__(self, num_kv_heads: int, head_dim: int, bits: int, residual_length: int, page_tokens: int = 64):
        if num_kv_heads <= 0 or head_dim <= 0:
            raise ConfigError("num_kv_heads and head_dim must be positive")
        if residual_length < 0:
            raise ConfigError("residual_length must be non-negative")
        self.num_kv_heads = num_kv_heads
        self.head_dim = head_dim
        self.bits = validate_bits(bits)
        self.residual_length = residual_length
        self.store = PagedKVCache(1, num_kv_heads, head_dim, (bits,), residual_length, batch=1,
                                  page_tokens=page_tokens)

    @classmethod
    def for_layer(cls, cfg: ModelConfig, layer_idx: int) -> "CompressedLayerCache":
        return cls(cfg.num_kv_heads, cfg.head_dim, cfg.plan[layer_idx], cfg.residual_length)

    @property
    def r(self) -> int:
        return self.store.lengths(0)[1]

    @property
    def compressed_tokens(self) -> int:
        return self.store.lengths(0)[0]

    @property
    def total_tokens(self) -> int:
        return self.compressed_tokens + self.r

    def append_tokens(self, k_new, v_new) -> None:
        """Append rotated keys/values (tokens, H, D); flush policy of cache.py:154-180 on the GPU."""
        k = _dev.to_dev(k_new)
        v = _dev.to_dev(v_new)
        expected = (self.num_kv_heads, self.head_dim)
        if k.ndim != 3 or tuple(k.shape[1:]) != expected:
            raise ShapeError(f"keys must be (tokens, {expected[0]}, {expected[1]}), got {tuple(k.shape)}")
        if tuple(v.shape) != tuple(k.shape):
            raise ShapeError(f"values shape {tuple(v.shape)} does not match keys shape {tuple(k.shape)}")
        if k.shape[0] == 0:
            return
        if v.dtype != k.dtype:
            k, v = k.float(), v.float()
        # a non-finite row that K1 compresses raises DataError with the cache unchanged (one flag read, no pre-pass)
        self.store.append_checked(0, k.unsqueeze(0), v.unsqueeze(0))

    # --- reference attributes, exported from the paged layout -------------------------------------------
    def _export(self) -> dict:
        return self.store.export(0, 0)

    def export_device(self) -> dict:
        """Dense device tensors (k_mean, v_mean, k_dev, v_dev, residual_k, residual_v)."""
        return self._export()

    @property
    def k_mean(self) -> np.ndarray:
        return _dev.host(self._export()["k_mean"])

    @property
    def v_mean(self) -> np.ndarray:
        return _dev.host(self._export()["v_mean"])

    @property
    def k_dev(self) -> QuantizedDeviation:
        return self._export()["k_dev"].to_host()

    @property
    def v_dev(self) -> QuantizedDeviation:
        return self._export()["v_dev"].to_host()

    @property
    def residual_k(self) -> np.ndarray:
        return _dev.host(self._export()["residual_k"])

    @property
    def residual_v(self) -> np.ndarray:
        return _dev.host(self._export()["residual_v"])

    def reconstruct_slice(self, head_idx: int, start: int, stop: int):
        """K̂/V̂ of compressed tokens [start, stop) for one head: mean - deq(dev) (cache.py:193-200)."""
        from .quant import dequantize_groups

        ex = self._export()
        groups = torch.arange(start, stop, dtype=torch.int64, device=self.store.dev) * self.num_kv_heads + head_idx
        k_hat = ex["k_mean"][start:stop] - dequantize_groups(ex["k_dev"], groups)
        v_hat = ex["v_mean"][start:stop] - dequantize_groups(ex["v_dev"], groups)
        return _dev.host(k_hat), _dev.host(v_hat)

    def reconstruct(self, head_idx: int):
        """Full (tokens, head_dim) K̂/V̂ for one head, residual rows appended verbatim (cache.py:202-213)."""
        if not 0 <= head_idx < self.num_kv_heads:
            raise ShapeError(f"head index {head_idx} out of range for {self.num_kv_heads} heads")
        k_c, v_c = self.reconstruct_slice(head_idx, 0, self.compressed_tokens)
        rk, rv = self.residual_k, self.residual_v
        return np.concatenate([k_c, rk[:, head_idx, :]]), np.concatenate([v_c, rv[:, head_idx, :]])


def memory_ratio(cfg: ModelConfig, tokens_per_layer: int, include_residual: bool = False) -> float:
    """Accounted bytes vs a 16-bit cache, 1/H + bits/16 + 2/D per layer, averaged (cache.py:216-239)."""
    if tokens_per_layer < 0:
        raise ConfigError(f"tokens_per_layer must be non-negative, got {tokens_per_layer}")
    if tokens_per_layer == 0:
        return 0.0
    total = 0.0
    for bits in cfg.plan.bits_per_layer:
        per_tok = 1.0 / cfg.num_kv_heads + bits / 16.0 + 2.0 / cfg.head_dim
        if include_residual:
            r = tokens_per_layer % cfg.residual_length if cfg.residual_length > 0 else 0
            total += ((tokens_per_layer - r) * per_tok + r * 1.0) / tokens_per_layer
        else:
            total += per_tok
    return total / cfg.num_layers


def actual_bytes_per_token(head_dim: int, num_kv_heads: int, bits: int) -> int:
    """Bytes actually stored per compressed token and side: f32 mean + codes + f32 (scale, min) per head."""
    gb = head_dim * 4 if bits == 16 else (head_dim * bits + 7) // 8
    return 4 * head_dim + num_kv_heads * (gb + 8)


# ---------------------------------------------------------------------- TADAKV1 (cache.py:242-368)


def _f32le(a) -> bytes:
    return np.ascontiguousarray(a).astype("<f4").tobytes()


def serialize_cache(layer: CompressedLayerCache) -> bytes:
    """TADAKV1 byte stream of one layer (cache.py:311-330); bit-exact with the reference."""
    ex = layer._export()
    C, r = layer.store.lengths(0)
    parts = [CACHE_MAGIC, struct.pack("<IIBIQQ", layer.num_kv_heads, layer.head_dim, layer.bits,
                                      layer.residual_length, C, r)]
    parts += [_f32le(_dev.host(ex["k_mean"])), _f32le(_dev.host(ex["v_mean"]))]
    for rec in (ex["k_dev"].to_host(), ex["v_dev"].to_host()):
        parts.append(struct.pack("<BQII", rec.bits, rec.num_tokens, rec.num_heads, rec.group_size))
        parts.append(struct.pack("<Q", len(rec.codes)))
        parts += [rec.codes, _f32le(rec.scales), _f32le(rec.mins)]
    parts += [_f32le(_dev.host(ex["residual_k"])), _f32le(_dev.host(ex["residual_v"]))]
    return b"".join(parts)


class _Cursor:
    def __init__(self, data: bytes):
        self.data, self.pos = data, 0

    def take(self, n: int) -> bytes:
        if self.pos + n > len(self.data):
            raise FormatError("truncated cache stream")
        self.pos += n
        return self.data[self.pos - n: self.pos]

    def fmt(self, f: str):
        return struct.unpack("<" + f, self.take(struct.calcsize("<" + f)))

    def floats(self, n: int) -> np.ndarray:
        return np.frombuffer(self.take(4 * n), dtype="<f4").astype(F32)


def deserialize_cache(data: bytes) -> CompressedLayerCache:
    """Parse TADAKV1 into a device cache; FormatError without partial state (cache.py:333-368)."""
    cur = _Cursor(data)
    magic = cur.take(len(CACHE_MAGIC))
    if magic[:6] != CACHE_MAGIC[:6]:
        raise FormatError(f"bad cache magic {magic!r}")
    if magic != CACHE_MAGIC:
        raise FormatError(f"unsupported cache version {magic!r}")
    heads, head_dim, bits, residual_length, n_comp, n_res = cur.fmt("IIBIQQ")
    if bits not in ALLOWED_WIDTHS:
        raise FormatError(f"unsupported bit width {bits} in cache stream")
    k_mean = cur.floats(n_comp * head_dim).reshape(n_comp, head_dim)
    v_mean = cur.floats(n_comp * head_dim).reshape(n_comp, head_dim)
    recs = []
    for _ in range(2):
        b, t, h, d = cur.fmt("BQII")
        if b not in ALLOWED_WIDTHS:
            raise FormatError(f"unsupported bit width {b} in cache stream")
        (n,) = cur.fmt("Q")
        codes = cur.take(n)
        s = cur.floats(t * h)
        m = cur.floats(t * h)
        recs.append(QuantizedDeviation(bits=b, num_tokens=t, num_heads=h, group_size=d, codes=codes, scales=s, mins=m))
    residual_k = cur.floats(n_res * heads * head_dim).reshape(n_res, heads, head_dim)
    residual_v = cur.floats(n_res * heads * head_dim).reshape(n_res, heads, head_dim)
    if cur.pos != len(data):
        raise FormatError(f"{len(data) - cur.pos} trailing bytes after cache payload")
    for name, rec in (("key", recs[0]), ("value", recs[1])):
        if (rec.bits, rec.num_tokens, rec.num_heads, rec.group_size) != (bits, n_comp, heads, head_dim):
            raise FormatError(f"{name} deviation header disagrees with cache header")
    cache = CompressedLayerCache(heads, head_dim, bits, residual_length)
    cache.store.load(0, 0, k_mean, v_mean, recs[0], recs[1], residual_k, residual_v)
    return cache
