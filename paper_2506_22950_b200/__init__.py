"""B200-native continuous-sampling decode step of Infinite Sampling (arXiv 2506.22950).

The product is libinfsamp.so (CUDA C++ for sm_100a, C-ABI in include/infsamp.h);
this package is its thin ctypes binding plus a rollout driver.
"""
from ._lib import (  # noqa: F401
    Context, InfsampError, MODES, is_dbg_gemm, is_group_advantages, is_plan, load, make_config,
)
