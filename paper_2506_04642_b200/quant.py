"""Group-wise asymmetric quantizer with LSB-first packing — B200 implementation.

Drop-in for ``tadakv.quant`` (pkg/src/tadakv/quant.py): same names, argument
meaning, return types and error types.  The arithmetic runs in
libtadakv_b200.so (``tada_quantize_groups`` / ``tada_dequantize_groups`` /
``tada_pack_codes`` / ``tada_unpack_codes``) and is bit-exact with the reference.

Host/device convention: numpy (or list) inputs give the reference's host types
back (``bytes`` codes, numpy scales/mins); torch inputs stay on the GPU
(``codes`` is a uint8 CUDA tensor, scales/mins f32 CUDA tensors).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev
from ._lib import call
from .errors import ConfigError, DataError, FormatError, ShapeError

PACKED_WIDTHS = (2, 4, 8)
PASSTHROUGH_WIDTH = 16
ALLOWED_WIDTHS = PACKED_WIDTHS + (PASSTHROUGH_WIDTH,)
F32 = np.float32


def validate_bits(bits: int) -> int:
    """quant.py:28-31."""
    if bits not in ALLOWED_WIDTHS:
        raise ConfigError(f"bit width must be one of {ALLOWED_WIDTHS}, got {bits}")
    return bits


def bytes_per_group(group_size: int, bits: int) -> int:
    """Packed bytes of one group incl. byte padding (quant.py:34-38)."""
    return group_size * 4 if bits == PASSTHROUGH_WIDTH else (group_size * bits + 7) // 8


def _nbytes(codes) -> int:
    return int(codes.numel()) if isinstance(codes, torch.Tensor) else len(codes)


def _len(a) -> tuple:
    return tuple(a.shape)


@dataclass
class QuantizedDeviation:
    """Packed codes + per-group f32 (scale, min), groups in (token, head) order (quant.py:41-77)."""

    bits: int
    num_tokens: int
    num_heads: int
    group_size: int
    codes: object  # bytes (host) or uint8 CUDA tensor (device)
    scales: object = field(repr=False)
    mins: object = field(repr=False)

    def __post_init__(self) -> None:
        validate_bits(self.bits)
        expected = self.num_groups * bytes_per_group(self.group_size, self.bits)
        if _nbytes(self.codes) != expected:
            raise FormatError(f"packed codes length mismatch: have {_nbytes(self.codes)} bytes, expected {expected}")
        if _len(self.scales) != (self.num_groups,) or _len(self.mins) != (self.num_groups,):
            raise FormatError(
                f"metadata length mismatch: {_len(self.scales)}/{_len(self.mins)} for {self.num_groups} groups"
            )

    @property
    def num_groups(self) -> int:
        return self.num_tokens * self.num_heads

    @property
    def shape(self) -> tuple[int, int, int]:
        return (self.num_tokens, self.num_heads, self.group_size)

    @property
    def on_device(self) -> bool:
        return isinstance(self.codes, torch.Tensor)

    def device_tensors(self):
        """(codes u8, scales f32, mins f32) as CUDA tensors (copied in if host-backed)."""
        dev = _dev.device()
        if self.on_device:
            return self.codes, self.scales, self.mins
        codes = torch.frombuffer(bytearray(self.codes), dtype=torch.uint8) if len(self.codes) else torch.empty(0, dtype=torch.uint8)
        return (
            codes.to(dev),
            torch.from_numpy(np.ascontiguousarray(self.scales, F32)).to(dev),
            torch.from_numpy(np.ascontiguousarray(self.mins, F32)).to(dev),
        )

    def to_host(self) -> "QuantizedDeviation":
        if not self.on_device:
            return self
        return QuantizedDeviation(self.bits, self.num_tokens, self.num_heads, self.group_size,
                                  _dev.host(self.codes).tobytes(), _dev.host(self.scales), _dev.host(self.mins))


def empty_deviation(bits: int, num_heads: int, group_size: int) -> QuantizedDeviation:
    """Zero-token record (quant.py:80-90)."""
    return QuantizedDeviation(validate_bits(bits), 0, num_heads, group_size, b"",
                              np.empty(0, dtype=F32), np.empty(0, dtype=F32))


def _codes_input(codes):
    if isinstance(codes, torch.Tensor):
        return codes, True
    return np.asarray(codes), False


def pack_codes(codes, bits: int):
    """Pack (groups, group_size) codes in [0, 2^bits) — quant.py:93-111 on the GPU."""
    if bits not in PACKED_WIDTHS:
        raise ConfigError(f"packing supports widths {PACKED_WIDTHS}, got {bits}")
    codes, is_t = _codes_input(codes)
    if codes.ndim != 2:
        raise ShapeError(f"expected (groups, group_size) codes, got shape {tuple(codes.shape)}")
    n, d = codes.shape
    dev = _dev.device()
    src = codes.to(device=dev, dtype=torch.uint8).contiguous() if is_t else \
        torch.from_numpy(np.ascontiguousarray(codes.astype(np.uint8))).to(dev)
    out = torch.empty(n * bytes_per_group(d, bits), dtype=torch.uint8, device=dev)
    call("tada_pack_codes", _dev.ptr(src), n, d, bits, _dev.ptr(out), _dev.stream())
    return out if is_t else _dev.host(out).tobytes()


def unpack_codes(data, bits: int, num_groups: int, group_size: int, groups=None):
    """(groups, group_size) uint8 codes from packed bytes, optional group subset (quant.py:114-140)."""
    if bits not in PACKED_WIDTHS:
        raise ConfigError(f"unpacking supports widths {PACKED_WIDTHS}, got {bits}")
    bpg = bytes_per_group(group_size, bits)
    if _nbytes(data) != num_groups * bpg:
        raise FormatError(f"packed codes length mismatch: have {_nbytes(data)} bytes, expected {num_groups * bpg}")
    is_t = isinstance(data, torch.Tensor)
    dev = _dev.device()
    src = data.to(dev).contiguous() if is_t else torch.frombuffer(bytearray(data), dtype=torch.uint8).to(dev) \
        if len(data) else torch.empty(0, dtype=torch.uint8, device=dev)
    sel = None
    n_out = num_groups
    if groups is not None:
        sel = torch.as_tensor(np.asarray(groups, dtype=np.int64) if not isinstance(groups, torch.Tensor) else groups,
                              dtype=torch.int64).to(dev).contiguous()
        n_out = int(sel.numel())
        if n_out and (int(sel.min()) < 0 or int(sel.max()) >= num_groups):
            raise IndexError("group index out of range")
    out = torch.empty((n_out, group_size), dtype=torch.uint8, device=dev)
    call("tada_unpack_codes", _dev.ptr(src), num_groups, group_size, bits, _dev.ptr(sel), n_out, _dev.ptr(out),
         _dev.stream())
    return out if is_t else _dev.host(out)


def _quantize_device(rows: torch.Tensor, bits: int):
    """rows [G, D] (f32/bf16 CUDA) -> (codes u8 [G*gb], scales [G], mins [G]) on device; DataError on non-finite."""
    g, d = rows.shape
    dev = rows.device
    codes = torch.empty(g * bytes_per_group(d, bits), dtype=torch.uint8, device=dev)
    scales = torch.empty(g, dtype=torch.float32, device=dev)
    mins = torch.empty(g, dtype=torch.float32, device=dev)
    err = _dev.ErrFlag()
    call("tada_quantize_groups", _dev.ptr(rows), _dev.dtype_code(rows), g, d, bits, _dev.ptr(codes), _dev.ptr(scales),
         _dev.ptr(mins), err.ptr, _dev.stream())
    if err.raised():
        raise DataError("cannot quantize non-finite values" if bits != PASSTHROUGH_WIDTH
                        else "cannot store non-finite values")
    return codes, scales, mins


def quantize_group(values, bits: int):
    """One group -> (codes int64, scale, min) (quant.py:183-197)."""
    validate_bits(bits)
    if bits == PASSTHROUGH_WIDTH:
        raise ConfigError("width 16 is a pass-through and bypasses group quantization")
    vals = _dev.to_dev(values)
    if vals.ndim != 1 or vals.numel() == 0:
        raise ShapeError(f"expected a non-empty 1-D group, got shape {tuple(vals.shape)}")
    codes, scales, mins = _quantize_device(vals.reshape(1, -1), bits)
    unpacked = unpack_codes(codes, bits, 1, vals.numel())
    return _dev.host(unpacked)[0].astype(np.int64), float(scales.item()), float(mins.item())


def quantize_tensor(dev, bits: int) -> QuantizedDeviation:
    """(tokens, heads, head_dim) -> QuantizedDeviation, one group per (token, head) (quant.py:200-229)."""
    validate_bits(bits)
    is_t = isinstance(dev, torch.Tensor)
    x = _dev.to_dev(dev)
    if x.ndim != 3:
        raise ShapeError(f"expected (tokens, heads, head_dim) input, got shape {tuple(x.shape)}")
    t, h, d = x.shape
    if t * h == 0 or d == 0:
        rec = QuantizedDeviation(bits, t, h, d, b"", np.zeros(t * h, F32), np.zeros(t * h, F32))
        return rec
    codes, scales, mins = _quantize_device(x.reshape(t * h, d), bits)
    if is_t:
        return QuantizedDeviation(bits, t, h, d, codes, scales, mins)
    return QuantizedDeviation(bits, t, h, d, _dev.host(codes).tobytes(), _dev.host(scales), _dev.host(mins))


def dequantize_groups(q: QuantizedDeviation, groups):
    """Selected groups as (len(groups), group_size) f32 (quant.py:232-239)."""
    codes, scales, mins = q.device_tensors()
    dev = codes.device
    sel = torch.as_tensor(np.asarray(groups, dtype=np.int64) if not isinstance(groups, torch.Tensor) else groups,
                          dtype=torch.int64).to(dev).reshape(-1).contiguous()
    n = int(sel.numel())
    if n and (int(sel.min()) < 0 or int(sel.max()) >= q.num_groups):
        raise IndexError("group index out of range")
    out = torch.empty((n, q.group_size), dtype=torch.float32, device=dev)
    if n:
        call("tada_dequantize_groups", _dev.ptr(codes), _dev.ptr(scales), _dev.ptr(mins), q.num_groups, q.group_size,
             q.bits, _dev.ptr(sel), n, _dev.ptr(out), _dev.stream())
    return out if q.on_device else _dev.host(out)


def dequantize_tensor(q: QuantizedDeviation):
    """Full (tokens, heads, head_dim) reconstruction (quant.py:242-245)."""
    codes, scales, mins = q.device_tensors()
    out = torch.empty(q.shape, dtype=torch.float32, device=codes.device)
    if q.num_groups and q.group_size:
        call("tada_dequantize_groups", _dev.ptr(codes), _dev.ptr(scales), _dev.ptr(mins), q.num_groups, q.group_size,
             q.bits, None, 0, _dev.ptr(out), _dev.stream())
    return out if q.on_device else _dev.host(out)


def direct_quantize_baseline(x, bits: int):
    """Quantize raw activations without mean-centering, then reconstruct (quant.py:248-254)."""
    return dequantize_tensor(quantize_tensor(x, bits))


def concat_deviations(a: QuantizedDeviation, b: QuantizedDeviation) -> QuantizedDeviation:
    """Groups of b after those of a (quant.py:257-272)."""
    if (a.bits, a.num_heads, a.group_size) != (b.bits, b.num_heads, b.group_size):
        raise ShapeError(
            f"cannot concatenate deviations with layouts {(a.bits, a.num_heads, a.group_size)} "
            f"and {(b.bits, b.num_heads, b.group_size)}"
        )
    if a.on_device or b.on_device:
        ca, sa, ma = a.device_tensors()
        cb, sb, mb = b.device_tensors()
        return QuantizedDeviation(a.bits, a.num_tokens + b.num_tokens, a.num_heads, a.group_size,
                                  torch.cat([ca, cb]), torch.cat([sa, sb]), torch.cat([ma, mb]))
    return QuantizedDeviation(a.bits, a.num_tokens + b.num_tokens, a.num_heads, a.group_size, a.codes + b.codes,
                              np.concatenate([a.scales, b.scales]), np.concatenate([a.mins, b.mins]))
