"""paper_2506_04642_b200 — B200-native TaDA KV-cache hot path (arxiv 2506.04642).

Drop-in for the hot-path subset of the reference package ``tadakv``
(pkg/src/tadakv/__init__.py:10-50): quantize / dequantize, mean centering,
the compressed layer cache (append / reconstruct / TADAKV1), decode attention,
the per-layer PrecisionPlan, and rotary keys fused into the append
(apply_rope / rotate_heads / append_fused, tensor.py:63-105, model.py:167-183).  Compute runs in libtadakv_b200.so
(hand-written sm_100a CUDA behind a C ABI, include/tadakv_b200.h); there is no
CPU fallback.  ``PagedKVCache`` is the batched multi-layer production store.
"""

from .attention import AttentionOutput, BlockSpec, attend_naive, attend_streaming, kv_head_index
from .cache import (
    CompressedLayerCache,
    ModelConfig,
    PrecisionPlan,
    RopeParams,
    actual_bytes_per_token,
    deserialize_cache,
    mean_center,
    memory_ratio,
    serialize_cache,
)
from .errors import (
    BudgetInfeasibleError,
    CapacityError,
    ConfigError,
    DataError,
    FormatError,
    ShapeError,
    StateError,
    TadaError,
)
from .decoder import ToyDecoder
from .paged import DecodeGraph, PagedKVCache
from .rope import append_fused, append_rope, apply_rope, rope_table, rotate_heads
from .shard import ShardedKVCache, ShardPlan
from .quant import (
    QuantizedDeviation,
    bytes_per_group,
    concat_deviations,
    dequantize_groups,
    dequantize_tensor,
    direct_quantize_baseline,
    empty_deviation,
    pack_codes,
    quantize_group,
    quantize_tensor,
    unpack_codes,
    validate_bits,
)

__version__ = "0.1.0"

__all__ = [
    "AttentionOutput", "BlockSpec", "BudgetInfeasibleError", "CapacityError", "CompressedLayerCache", "ConfigError",
    "DataError", "DecodeGraph", "FormatError", "ModelConfig", "PagedKVCache", "PrecisionPlan", "QuantizedDeviation", "RopeParams",
    "ShapeError", "ShardPlan", "ToyDecoder", "append_fused", "append_rope", "apply_rope", "rope_table", "rotate_heads", "ShardedKVCache", "StateError", "TadaError", "actual_bytes_per_token", "attend_naive", "attend_streaming",
    "bytes_per_group", "concat_deviations", "dequantize_groups", "dequantize_tensor", "deserialize_cache",
    "direct_quantize_baseline", "empty_deviation", "kv_head_index", "mean_center", "memory_ratio", "pack_codes",
    "quantize_group", "quantize_tensor", "serialize_cache", "unpack_codes", "validate_bits", "__version__",
]
