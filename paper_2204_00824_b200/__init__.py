"""B200-native (sm_100a) TSDG graph search — the GPU search hot path of
"Graph-based Approximate NN Search: A Revisit" (arXiv 2204.00824) behind the
reference's search API.  See DESIGN.md."""
from .search import (BestFirstParams, GpuIndex, GreedyParams, InvalidArgument,  # noqa: F401
                     SearchResult, SearchStats, TsdgGraph, TsdgRuntimeError, bestfirst_search,
                     large_batch_search, load_tsdg, merge_shards_device, small_batch_search,
                     small_batch_search_one)
