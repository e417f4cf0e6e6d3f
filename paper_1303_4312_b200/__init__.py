"""B200-native (sm_100a) stable parallel merge of arXiv 1303.4312.

The product is ``lib/libcomerge_cuda.so`` (C ABI: include/comerge_cuda.h,
C++ shim: include/comerge/cuda.hpp).  This package is its Python mirror of
the reference API (see ``comerge``).
"""
from .comerge import merge_pieces  # noqa: F401
from .comerge import (BlockAssignment, ComparisonCounter, CoRankStats, MergeOptions,  # noqa: F401
                      MergeReport, co_rank, co_rank_batch, co_rank_counted, merge_pairs, merge_records,
                      co_rank_records, co_rank_batch_records, plan_records, merge_parallel_records, record_dtype, records_workspace_bytes,
                      merge_parallel, merge_parallel_synced, merge_segmented, partition_output,
                      plan, set_kernel_path, sort, sort_pairs, sort_pairs_workspace_bytes,
                      sort_workspace_bytes, stable_merge,
                      workspace_bytes)

__all__ = ["co_rank", "co_rank_counted", "co_rank_batch", "stable_merge", "partition_output",
           "plan", "merge_parallel", "merge_parallel_synced", "merge_pairs", "merge_records", "co_rank_records", "co_rank_batch_records", "plan_records",
           "merge_parallel_records", "record_dtype", "records_workspace_bytes", "merge_segmented",
           "merge_pieces", "sort", "sort_workspace_bytes", "sort_pairs", "sort_pairs_workspace_bytes", "set_kernel_path", "workspace_bytes",
           "MergeReport", "MergeOptions", "CoRankStats", "ComparisonCounter", "BlockAssignment"]
