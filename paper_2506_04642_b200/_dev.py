"""Device plumbing: tensors in/out of the C ABI (PyTorch owns memory and streams)."""

from __future__ import annotations

import numpy as np
import torch

from ._lib import TADA_BF16, TADA_F32, BackendUnavailable, load


def device() -> torch.device:
    """The CUDA device all kernels run on; raises if there is none (no CPU fallback)."""
    load()
    if not torch.cuda.is_available():
        raise BackendUnavailable("no CUDA device: the TaDA B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def to_dev(x, allow_bf16: bool = True) -> torch.Tensor:
    """numpy / torch -> contiguous CUDA tensor, f32 unless (allowed) bf16 already."""
    dev = device()
    if isinstance(x, torch.Tensor):
        if x.dtype == torch.bfloat16 and allow_bf16:
            return x.to(dev).contiguous()
        return x.to(device=dev, dtype=torch.float32).contiguous()
    arr = np.ascontiguousarray(x, dtype=np.float32)
    return torch.from_numpy(arr).to(dev)


def dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return TADA_F32
    if t.dtype == torch.bfloat16:
        return TADA_BF16
    raise TypeError(f"unsupported dtype {t.dtype}")


def host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


class ErrFlag:
    """Device int32 word kernels OR into on non-finite input (DataError, quant.py:151-152)."""

    def __init__(self):
        self.t = torch.zeros(1, dtype=torch.int32, device=device())

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    def raised(self) -> bool:
        """Synchronising read; clears the flag."""
        v = int(self.t.item())
        if v:
            self.t.zero_()
        return bool(v)
