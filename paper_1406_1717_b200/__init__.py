"""B200-native sorting-based median filter (arXiv 1406.1717), drop-in for
``medfilt::median_filter<T>`` (/root/reference/proj/include/medfilt/filter.hpp:149-155).

The product is libmedfilt_b200.so (CUDA kernels for sm_100a behind the C ABI of
include/medfilt_gpu.h); this package is its host-side mirror.
"""
from .filter import (Context, CudaError, InvalidArgument, WindowSpec, block_sort_device, fold_checksum, generate_device,
                     generate_trend_f64, kernel_class, make_window_spec, median_filter, median_filter_device,
                     median_filter_rows, median_filter_rows_device, sort_via_median_filter)
from .shard import gather_outputs_device, input_union, shard_outputs, shard_rows

__all__ = [
    "Context", "CudaError", "InvalidArgument", "WindowSpec", "block_sort_device", "fold_checksum",
    "gather_outputs_device", "generate_device", "input_union",
    "generate_trend_f64", "kernel_class", "make_window_spec", "median_filter", "median_filter_device",
    "median_filter_rows", "median_filter_rows_device", "shard_outputs", "shard_rows", "sort_via_median_filter",
]
