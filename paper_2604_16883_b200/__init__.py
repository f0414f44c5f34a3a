"""paper_2604_16883_b200 — B200-native (sm_100a) SinkRouter sink-aware decode
attention behind the reference's operator API.

The compute path is the CUDA library ``_lib/libsinkr_cuda.so`` (C-ABI:
``include/sinkr_cuda.h``); this package is the host-side mirror of the
reference interface (``router.py``), the synthetic planted-sink workload
(``workload.py``) and the multi-GPU plumbing (``sharding.py``).
"""
from .router import (  # noqa: F401
    AppendStepRunner,
    CacheConfig,
    EngineOptions,
    GroupStepInfo,
    KvCache,
    LayerStepResult,
    LoadCounters,
    RouteDecision,
    RoutingConfig,
    StepRunner,
    ThresholdProfile,
    auto_num_splits,
    decode_rank_partial_async,
    dense_attention,
    merge_rank_partials_async,
    online_attention,
    rank_partial_floats,
    fetch_step_info,
    kDefaultBlockSize,
    last_step_stats,
    route,
    routed_decode_async,
    routed_decode_peer_async,
    routed_decode_step,
    set_timing,
    split_ranges,
    splitk_attention,
    SplitkResult,
    threshold_for_length,
)
from .attention import (  # noqa: F401
    QueryGroup,
    SplitPartial,
    attend_chunk,
    attend_chunk_cached,
    merge_partials,
)
from .workload import WorkloadSpec  # noqa: F401

__version__ = "0.1.0"
