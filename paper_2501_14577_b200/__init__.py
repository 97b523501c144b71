"""onedf: B200-native (sm_100a) ZETA parallel causal top-k attention (arXiv 2501.14577).

The hot path (Morton encode, segmented radix sort, causal candidate search,
exact top-k, Adaptive Cauchy-Softmax gather, deterministic backward) lives in
hand-written CUDA kernels behind the C ABI ``include/onedf.h``
(``libonedf.so``); this package is its thin Python binding.
"""
from .abi import (DTYPE_BF16, DTYPE_F32, OK, OP_BWD, OP_ENCODE, OP_FWD, OP_SORT, OP_STEP_HOST, OnedfError, Problem,  # noqa: F401
                  onedf_check_device_status, onedf_encode, onedf_max_run_length, onedf_sort,
                  onedf_topk_attn_bwd, onedf_topk_attn_fwd, onedf_topk_attn_step_host, onedf_validate,
                  onedf_version, onedf_workspace_size, status_string)
from .api import (HostStep, Workspace, ZetaTopkAttention, bounds_finish, bounds_partial,  # noqa: F401
                  ZetaProjectedAttention, check_device_status, code_knn, default_chunk, encode, make_problem, overlap,
                  means_floats, project_bwd, project_encode, query_schedule, rank_sum, sort, topk_attn_bwd,
                  topk_attn_fwd,
                  value_dtype, zeta_attention, zeta_projected_attention)

__version__ = "0.1.0"
