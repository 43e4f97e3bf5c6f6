"""Rotary embedding on the compressed-cache append path — B200 implementation.

Drop-ins for ``tadakv.tensor.apply_rope`` / ``rotate_heads`` (tensor.py:63-105) and
``tadakv.model.append_fused`` (model.py:167-183).

The cos/sin of every (position, pair) are computed here in f64 with numpy exactly as tensor.py:84-88
does and uploaded once as an f32 table; the kernels (``tada_apply_rope``, and K1's fused variant
``tada_quant_append_rope``, which rotates the keys in registers before the cross-head mean) only
multiply and add in f32 with numpy's rounding, so rotated keys and the cache bytes that follow are
bit-identical to the reference.

Host/device convention as in quant.py: numpy inputs give numpy back, torch inputs stay on the GPU.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev
from ._lib import call
from .cache import CompressedLayerCache, RopeParams
from .errors import DataError, ShapeError

F32 = np.float32
F64 = np.float64

_TABLES: dict[tuple, torch.Tensor] = {}


def rope_table(params: RopeParams, n_pos: int) -> torch.Tensor:
    """Device f32 table [n, head_dim/2, 2] of (cos, sin) for positions 0 .. n-1 (n >= n_pos), built like
    tensor.py:84-88 (f64 inverse frequencies and angles, np.cos / np.sin, RNE to f32); cached and grown
    geometrically per (head_dim, base, device)."""
    dev = _dev.device()
    key = (params.head_dim, float(params.base), str(dev))
    t = _TABLES.get(key)
    if t is None or t.shape[0] < n_pos:
        n = max(1024, 1 << max(0, int(n_pos - 1).bit_length()))
        half = params.head_dim // 2
        inv_freq = params.base ** (-2.0 * np.arange(half, dtype=F64) / params.head_dim)
        angles = np.arange(n, dtype=np.int64)[:, None].astype(F64) * inv_freq[None, :]
        table = np.stack([np.cos(angles).astype(F32), np.sin(angles).astype(F32)], axis=-1)
        t = torch.from_numpy(np.ascontiguousarray(table)).to(dev)
        _TABLES[key] = t
    return t


def _positions(positions, n: int, batch: int | None = None) -> tuple[torch.Tensor, int]:
    """Validate like tensor.py:75-80 and return (device int32 positions, max position + 1)."""
    if isinstance(positions, torch.Tensor):
        pos = positions
        if pos.dtype.is_floating_point or pos.dtype == torch.bool:
            raise DataError("positions must be non-negative integers")
        host = pos.detach().cpu().numpy()
    else:
        host = np.asarray(positions)
        if host.dtype == object or not np.issubdtype(host.dtype, np.integer):
            raise DataError("positions must be non-negative integers")
    want = (n,) if batch is None else (batch, n)
    if host.shape != want:
        raise ShapeError(f"need one position per token row, got {host.shape} for {want}")
    if host.size and (host < 0).any():
        raise DataError("positions must be non-negative integers")
    if host.size and host.max() >= 2**31 - 1:
        raise DataError("positions must fit in int32")
    top = int(host.max()) + 1 if host.size else 1
    return torch.from_numpy(np.ascontiguousarray(host, dtype=np.int32)).to(_dev.device()), top


def _rotate(x: torch.Tensor, pos: torch.Tensor, top: int, params: RopeParams) -> torch.Tensor:
    """[tokens, heads, D] device rows -> rotated f32 (tada_apply_rope)."""
    t, h, d = x.shape
    out = torch.empty((t, h, d), dtype=torch.float32, device=x.device)
    if t and h:
        table = rope_table(params, top)
        call("tada_apply_rope", x.data_ptr(), _dev.dtype_code(x), t, h, d, pos.data_ptr(), table.data_ptr(),
             int(table.shape[0]), out.data_ptr(), None, _dev.stream())
    return out


def apply_rope(x, positions, params: RopeParams):
    """Rotate each adjacent (2j, 2j+1) pair of ``x`` [tokens, head_dim] by position * base^(-2j/head_dim)
    (tensor.py:63-89)."""
    is_t = isinstance(x, torch.Tensor)
    xd = _dev.to_dev(x)
    if xd.ndim != 2 or xd.shape[1] != params.head_dim:
        raise ShapeError(f"expected (tokens, {params.head_dim}) input, got {tuple(xd.shape)}")
    pos, top = _positions(positions, int(xd.shape[0]))
    out = _rotate(xd.unsqueeze(1), pos, top, params).squeeze(1)
    return out if is_t else _dev.host(out)


def rotate_heads(x, positions, params: RopeParams):
    """apply_rope on every head of a [tokens, heads, head_dim] tensor (tensor.py:92-105)."""
    is_t = isinstance(x, torch.Tensor)
    xd = _dev.to_dev(x)
    if xd.ndim != 3 or xd.shape[2] != params.head_dim:
        raise ShapeError(f"expected (tokens, heads, {params.head_dim}) input, got {tuple(xd.shape)}")
    pos, top = _positions(positions, int(xd.shape[0]))
    out = _rotate(xd, pos, top, params)
    return out if is_t else _dev.host(out)


def append_rope(cache: CompressedLayerCache, k_pre_rope, v_new, positions, rope: RopeParams) -> None:
    """rotate_heads(k_pre_rope) + cache.append_tokens(., v_new) with the rotation fused into K1."""
    k = _dev.to_dev(k_pre_rope)
    v = _dev.to_dev(v_new)
    expected = (cache.num_kv_heads, cache.head_dim)
    if k.ndim != 3 or tuple(k.shape[1:]) != expected:
        raise ShapeError(f"keys must be (tokens, {expected[0]}, {expected[1]}), got {tuple(k.shape)}")
    if rope.head_dim != cache.head_dim:
        raise ShapeError(f"rope head_dim {rope.head_dim} does not match the cache's {cache.head_dim}")
    pos, top = _positions(positions, int(k.shape[0]))
    if tuple(v.shape) != tuple(k.shape):
        raise ShapeError(f"values shape {tuple(v.shape)} does not match keys shape {tuple(k.shape)}")
    if k.shape[0] == 0:
        return
    if v.dtype != k.dtype:
        k, v = k.float(), v.float()
    # non-finite rows that K1 compresses raise DataError with the cache unchanged (PagedKVCache.append_checked)
    cache.store.append_checked(0, k.unsqueeze(0), v.unsqueeze(0), rope=(pos.unsqueeze(0), top, rope))


def append_fused(cache: CompressedLayerCache, k_pre_rope, x_norm, w_v, positions, rope: RopeParams) -> None:
    """Rotate keys, project values and write both into the cache in one step (model.py:167-183).

    The value projection ``x_norm @ w_v`` is computed where its operands live: host numpy operands (the
    reference API) get numpy's f32 matmul — the reference's own expression (model.py:181), so the cache is
    byte-equal to composing rotate_heads / ``x_norm @ w_v`` / append_tokens by hand (AC8); device tensors
    get an f32 cuBLAS GEMM (TF32 off).  Either way the projection is a library GEMM beside the path; the
    rotated keys exist only in registers of the fused append kernel."""
    if not (_dev.is_torch(x_norm) or _dev.is_torch(w_v)):
        xh = np.ascontiguousarray(x_norm, dtype=np.float32)
        wh = np.ascontiguousarray(w_v, dtype=np.float32)
        if xh.ndim != 2 or wh.ndim != 2 or xh.shape[1] != wh.shape[0]:
            raise ShapeError(f"cannot project {xh.shape} by {wh.shape}")
        if wh.shape[1] != cache.num_kv_heads * cache.head_dim:
            raise ShapeError(f"w_v must have {cache.num_kv_heads * cache.head_dim} columns, got {wh.shape[1]}")
        v = (xh @ wh).reshape(xh.shape[0], cache.num_kv_heads, cache.head_dim)
        append_rope(cache, k_pre_rope, v, positions, rope)
        return
    xn = _dev.to_dev(x_norm, allow_bf16=False)
    wv = _dev.to_dev(w_v, allow_bf16=False)
    if xn.ndim != 2 or wv.ndim != 2 or xn.shape[1] != wv.shape[0]:
        raise ShapeError(f"cannot project {tuple(xn.shape)} by {tuple(wv.shape)}")
    n = int(xn.shape[0])
    if wv.shape[1] != cache.num_kv_heads * cache.head_dim:
        raise ShapeError(f"w_v must have {cache.num_kv_heads * cache.head_dim} columns, got {wv.shape[1]}")
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        v = (xn @ wv).reshape(n, cache.num_kv_heads, cache.head_dim)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    append_rope(cache, k_pre_rope, v, positions, rope)
