"""B200-native Twilight (arXiv 2502.02770) select-then-prune decode attention.

Drop-in for the hot path of the reference package ``nucleuskv``: the same
operator names and argument order, on CUDA tensors, backed by hand-written
sm_100a kernels in ``csrc/`` behind the C ABI of ``include/twilight.h``.
The batched entry point is ``TwilightDecoder`` over a ``PagedKVCache``.
There is no CPU fallback: without ``_lib/libtwilight.so`` the ops raise.
"""

from .attention import (MASS_SLACK, DegenerateSelectionError, TokenSelection, attention_weights, frobenius_norm,
                        output_error, sparse_attention, stable_softmax)
from .decode import DecodeBuffers, DecodeStats, PagedKVCache, TwilightDecoder, pages_for
from .pipeline import (PipelineConfig, PruneReport, bypass_config, memory_overhead, model_speedup, run_grouped,
                       run_head)
from .pruner import BinarySearchConfig, PruneOutcome, binary_search_top_p, prune
from .quantcache import (PARAM_BYTES, SUPPORTED_BITS, EstimateResult, PagedQuantKeyCache, PageMetadata,
                         PageMetadataTable, QuantPage, QuantParams, build_cache, build_page_metadata,
                         dequantize_row, estimate_scores, pack_codes, quantize_row, quantize_rows, unpack_codes)
from .selectors import (GroupMap, SelectorConfig, build_selector, group_union, quest_page_scores, resolve_budget,
                        select_channel_pruned, select_full, select_quest, select_sink_window,
                        top_channels_by_magnitude)

from .dynamism import (RUN_COLUMNS, AxisSummary, DynamismStats, SweepRow, TaggedReport, collect_dynamism, sweep_p,
                       tag_decode_stats, write_run_csv)
from .tensorfile import (BadMagicError, DimOverflowError, TensorFileError, TruncatedFileError,
                         VersionMismatchError, load_file_workload, read_tensor, run_file_workload, write_tensor)

__version__ = "0.1.0"

__all__ = [
    "MASS_SLACK", "DegenerateSelectionError", "TokenSelection", "attention_weights", "frobenius_norm",
    "output_error", "sparse_attention", "stable_softmax", "BinarySearchConfig", "PruneOutcome",
    "binary_search_top_p", "prune", "PagedQuantKeyCache", "PageMetadata", "PageMetadataTable", "QuantPage",
    "QuantParams", "EstimateResult", "PARAM_BYTES", "SUPPORTED_BITS", "build_cache", "build_page_metadata",
    "dequantize_row", "estimate_scores", "pack_codes", "quantize_row", "quantize_rows", "unpack_codes",
    "GroupMap", "SelectorConfig", "build_selector", "group_union", "quest_page_scores", "resolve_budget",
    "select_channel_pruned", "select_full", "select_quest", "select_sink_window", "top_channels_by_magnitude",
    "PipelineConfig", "PruneReport", "bypass_config", "memory_overhead", "model_speedup", "run_grouped",
    "run_head", "PagedKVCache", "TwilightDecoder", "DecodeBuffers", "DecodeStats", "pages_for", "__version__",
    "TensorFileError", "BadMagicError", "VersionMismatchError", "TruncatedFileError", "DimOverflowError",
    "read_tensor", "write_tensor", "load_file_workload", "run_file_workload",
    "TaggedReport", "AxisSummary", "DynamismStats", "SweepRow", "collect_dynamism", "sweep_p", "tag_decode_stats",
    "RUN_COLUMNS", "write_run_csv",
]
