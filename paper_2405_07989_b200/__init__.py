"""paper_2405_07989_b200 -- B200-native parallel bounded lexicographic enumeration of
factorization sets Z(n, (g_1..g_d)) (arXiv 2405.07989), as a C-ABI CUDA library
(libfsgpu.so, include/fsgpu.h) with a thin Python binding.
"""
from ._lib import (FS_CONSUMER_ANY, FS_CONSUMER_COUNT, FS_CONSUMER_HIST, FS_CONSUMER_ROWS,  # noqa: F401
                   FS_ORDER_ANY, FS_ORDER_CANONICAL, FS_ORDER_INCREASING, FS_PRED_COORD_GE, FS_PRED_LEN_EQ,
                   FS_PRED_LEN_GE, FS_PRED_LEN_LE, FS_ROWS_BATCH, FS_ROWS_STAGED, FsError)
from .api import (Plan, fs_any, fs_any_ex, fs_count, fs_count_ex, fs_enumerate, fs_enumerate_ex,  # noqa: F401
                  fs_enumerate_filtered, fs_length_set, fs_length_set_ex, hist_len, sort_rows_desc)

__version__ = "1.0.0"
