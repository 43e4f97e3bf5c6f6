"""Multi-GPU sharding of the compressed KV cache — one process per GPU.

The reference is single-process (no collectives), so this module adds the B200-native
partitioning. Nothing crosses NVLink inside K1/K2.

* **Batch axis** (``batch >= world``). Each rank owns a contiguous block of sequences. It holds
  their whole cache, appends their tokens and attends over them locally. The only collective is
  one NCCL ``all_gather`` of the attention outputs.
* **Sequence axis** (``batch < world``, ``world % batch == 0``; config 4's 128k x B=4 on 8 GPUs).
  Each sequence is served by ``parts = world // batch`` ranks. Ownership of tokens is
  interleaved in whole residual blocks: block ``i`` (tokens ``[i*R, (i+1)*R)``) belongs to part
  ``i % parts``.

  Quantization is per token (cache.py:98-111, quant.py:200-207) and the flush policy moves whole
  R-blocks (cache.py:171-180). Each rank's local cache therefore holds exactly the reference's
  representation of its tokens: the compressed blocks, plus the partial newest block as residual
  rows on the rank that owns it.

  Attention over disjoint token sets merges exactly through ``(out, lse)`` pairs. Each rank
  returns its normalised partial and log-sum-exp (``tada_decode_attn_lse``). One all-gather of
  ``[Hq, D+1]`` floats per sequence follows, then ``tada_combine_lse`` — the online-softmax merge
  of attention.py:139-147. No cache byte is read twice, unlike a kv-head split: the cross-head
  mean row is shared by all heads (SURVEY §7 hard part 3).

Sequence parallelism across ranks changes only the float summation order, not the values being
summed.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from .errors import ConfigError, ShapeError


@dataclass(frozen=True)
class ShardPlan:
    """Which sequences / tokens of a ``batch``-sequence decode this rank owns."""

    world: int
    rank: int
    batch: int
    block: int  # token ownership granule on the sequence axis (= residual_length, or 64 if R == 0)

    def __post_init__(self) -> None:
        if self.world < 1 or not 0 <= self.rank < self.world:
            raise ConfigError(f"bad rank {self.rank} for world {self.world}")
        if self.batch < 1 or self.block < 1:
            raise ConfigError("batch and block must be positive")
        if self.batch < self.world and self.world % self.batch:
            raise ConfigError(f"sequence-axis sharding needs world ({self.world}) divisible by batch ({self.batch})")

    @classmethod
    def make(cls, world: int, rank: int, batch: int, residual_length: int) -> "ShardPlan":
        return cls(world, rank, batch, residual_length if residual_length > 0 else 64)

    @property
    def axis(self) -> str:
        return "batch" if self.batch >= self.world else "seq"

    @property
    def parts(self) -> int:
        """Ranks per sequence (1 on the batch axis)."""
        return 1 if self.axis == "batch" else self.world // self.batch

    @property
    def part(self) -> int:
        return 0 if self.axis == "batch" else self.rank % self.parts

    def seq_range(self, rank: int | None = None) -> tuple[int, int]:
        """Global sequence ids [first, stop) served by ``rank`` (balanced contiguous blocks)."""
        r = self.rank if rank is None else rank
        if self.axis == "batch":
            return r * self.batch // self.world, (r + 1) * self.batch // self.world
        s = r // self.parts
        return s, s + 1

    @property
    def local_batch(self) -> int:
        a, b = self.seq_range()
        return b - a

    def owned_spans(self, start_pos: int, n: int) -> list[tuple[int, int]]:
        """Chunk-relative ``[lo, hi)`` spans of an ``n``-token append at ``start_pos`` this rank stores."""
        if self.axis == "batch":
            return [(0, n)] if n else []
        spans = []
        pos, end = start_pos, start_pos + n
        while pos < end:
            blk = pos // self.block
            stop = min(end, (blk + 1) * self.block)
            if blk % self.parts == self.part:
                lo = pos - start_pos
                if spans and spans[-1][1] == lo:
                    spans[-1] = (spans[-1][0], stop - start_pos)
                else:
                    spans.append((lo, stop - start_pos))
            pos = stop
        return spans

    def local_tokens(self, total: int) -> int:
        """How many of a sequence's first ``total`` tokens this rank holds."""
        return sum(hi - lo for lo, hi in self.owned_spans(0, total))


def gather_outputs(local: torch.Tensor, plan: ShardPlan, group=None) -> torch.Tensor:
    """Batch axis: ``[local_batch, ...]`` on every rank -> ``[batch, ...]`` (one NCCL all-gather).

    Ragged blocks (batch % world != 0) are padded to the largest block for the collective.
    """
    import torch.distributed as dist

    if plan.world == 1:
        return local
    width = max(plan.seq_range(r)[1] - plan.seq_range(r)[0] for r in range(plan.world))
    buf = local.new_zeros((width,) + tuple(local.shape[1:]))
    buf[: local.shape[0]].copy_(local)
    out = local.new_empty((plan.world * width,) + tuple(local.shape[1:]))
    dist.all_gather_into_tensor(out, buf, group=group)
    rows = [out[r * width: r * width + (plan.seq_range(r)[1] - plan.seq_range(r)[0])] for r in range(plan.world)]
    return torch.cat(rows)


def exchange_partials(o: torch.Tensor, lse: torch.Tensor, plan: ShardPlan, group=None):
    """Sequence axis: this rank's ``o [Hq, D]`` f32 and ``lse [Hq]`` -> ``([batch, parts, Hq, D], [batch, parts, Hq])``.

    One all-gather of ``Hq*(D+1)`` floats per rank (NCCL on GPU, gloo on CPU).
    """
    import torch.distributed as dist

    if o.ndim != 2 or lse.shape != o.shape[:1]:
        raise ShapeError("partials must be o [Hq, D] and lse [Hq]")
    hq, d = o.shape
    packed = torch.cat([o.float(), lse.float()[:, None]], dim=1).contiguous()
    if plan.world == 1:
        allp = packed[None]
    else:
        allp = packed.new_empty((plan.world * hq, d + 1))
        dist.all_gather_into_tensor(allp, packed, group=group)
    allp = allp.view(plan.batch, plan.parts, hq, d + 1)
    return allp[..., :d], allp[..., d]


def merge_partials(o_parts: torch.Tensor, lse_parts: torch.Tensor, out_dtype=torch.float32) -> torch.Tensor:
    """``[batch, parts, Hq, D]`` + ``[batch, parts, Hq]`` -> ``[batch, Hq, D]`` via ``tada_combine_lse`` (CUDA)."""
    from . import _dev
    from ._lib import call

    b, p, hq, d = o_parts.shape
    o = o_parts.permute(1, 0, 2, 3).contiguous().float()
    lse = lse_parts.permute(1, 0, 2).contiguous().float()
    out = torch.empty((b, hq, d), dtype=out_dtype, device=o.device)
    call("tada_combine_lse", o.data_ptr(), lse.data_ptr(), p, b * hq, d, out.data_ptr(), _dev.dtype_code(out), None,
         _dev.stream())
    return out


class ShardedKVCache:
    """This rank's share of a ``batch``-sequence, ``num_layers``-layer compressed cache.

    Callers pass the GLOBAL per-step tensors (``[batch, n, H, D]`` K/V, ``[batch, Hq, D]`` q)
    on every rank. The store keeps only what it owns, and ``attend`` returns the global
    ``[batch, Hq, D]`` output on every rank.
    """

    def __init__(self, num_layers: int, num_kv_heads: int, head_dim: int, plan_bits, residual_length: int,
                 batch: int, world: int | None = None, rank: int | None = None, group=None, max_tokens: int | None = None,
                 page_tokens: int = 64):
        import torch.distributed as dist

        from .paged import PagedKVCache

        if world is None:
            world = dist.get_world_size(group) if dist.is_initialized() else 1
        if rank is None:
            rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.plan = ShardPlan.make(world, rank, batch, residual_length)
        self.group = group
        self.R = residual_length
        self.pos = 0  # global tokens appended per sequence (uniform batch)
        local_max = None
        if max_tokens is not None:
            local_max = max_tokens if self.plan.axis == "batch" else self.plan.local_tokens(max_tokens) + self.plan.block
        self.store = PagedKVCache(num_layers, num_kv_heads, head_dim, plan_bits, residual_length,
                                  batch=self.plan.local_batch, page_tokens=page_tokens, max_tokens=local_max)
        self.layer_pos = [0] * num_layers

    def append(self, layer: int, k: torch.Tensor, v: torch.Tensor) -> None:
        """Append the global step's ``[batch, n, H, D]`` K/V; this rank stores its sequences / token blocks."""
        if k.shape[0] != self.plan.batch:
            raise ShapeError(f"expected the global batch {self.plan.batch}, got {k.shape[0]}")
        a, b = self.plan.seq_range()
        n = int(k.shape[1])
        start = self.layer_pos[layer]
        for lo, hi in self.plan.owned_spans(start, n):
            self.store.append(layer, k[a:b, lo:hi], v[a:b, lo:hi])
        self.layer_pos[layer] = start + n

    def attend(self, layer: int, q: torch.Tensor, out_dtype=torch.float32, mode: int = 0) -> torch.Tensor:
        """Global ``q [batch, Hq, D]`` -> global attention output ``[batch, Hq, D]`` on every rank."""
        a, b = self.plan.seq_range()
        ql = q[a:b]
        if self.plan.axis == "batch":
            out = self.store.attend(layer, ql, out_dtype=out_dtype, mode=mode)
            return gather_outputs(out, self.plan, self.group)
        c, r = self.store.lengths(layer)
        hq, d = int(q.shape[1]), int(q.shape[2])
        if c + r:
            o, lse = self.store.attend_lse(layer, ql, mode=mode)
            o, lse = o[0], lse[0]
        else:  # this part holds no tokens yet: contributes nothing to the merge
            o = torch.zeros((hq, d), dtype=torch.float32, device=q.device)
            lse = torch.full((hq,), -math.inf, dtype=torch.float32, device=q.device)
        o_parts, lse_parts = exchange_partials(o, lse, self.plan, self.group)
        return merge_partials(o_parts, lse_parts, out_dtype)

