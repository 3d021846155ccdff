"""B200-native exact top-k decode attention (hot path of arXiv 2502.06766, `topk_kv`).

Drop-in surface (same names as the reference's `topk_kv/__init__.py:19-31`):
    topk_attend, TierAccounting, build_index, knn_search, TopKResult, MipsIndex,
    recall_at_k, and the error taxonomy.
Batched device API (the fast path):
    topk_decode_attention, topk_search, kv_append, TopkDecoder,
    LayerBudget / uniform_budget / linear_budget / entropy_budget / parse_budget_spec (per-layer k),
    sharded_topk_attention / CudaStages (token-range sharding over torch.distributed).
The compute runs in libtkv.so (sm_100a CUDA kernels behind the C ABI in include/tkv.h).
"""

from .ann import DeviceValues, MipsIndex, TopKResult, build_index, knn_search, recall_at_k
from .attention import VALUE_ROW_BYTES, TierAccounting, topk_attend
from .budget import LayerBudget, entropy_budget, linear_budget, parse_budget_spec, uniform_budget
from .decoder import TopkDecoder
from .errors import (
    ConfigError,
    DegenerateError,
    DeviceError,
    DomainError,
    FormatError,
    InfeasibleBudgetError,
    InputError,
    ShapeError,
    TopkKvError,
)
from .ops import Workspace, kv_append, topk_decode_attention, topk_decode_step, topk_search
from .sharded import (CudaStages, DeviceShardedStep, LocalExchange, SymmetricExchange, narrow_k, shard_range,
                      sharded_topk_attention)

__version__ = "0.1.0"

__all__ = [
    "ConfigError", "CudaStages", "DeviceShardedStep", "LocalExchange", "SymmetricExchange", "DegenerateError", "DeviceError", "DeviceValues", "DomainError",
    "FormatError", "InfeasibleBudgetError", "InputError", "LayerBudget", "MipsIndex", "ShapeError",
    "TierAccounting", "TopKResult", "TopkDecoder", "TopkKvError", "VALUE_ROW_BYTES", "Workspace",
    "build_index", "entropy_budget", "knn_search", "kv_append", "linear_budget", "parse_budget_spec",
    "narrow_k", "recall_at_k", "shard_range", "uniform_budget",
    "sharded_topk_attention", "topk_attend", "topk_decode_attention", "topk_decode_step", "topk_search",
]
