"""B200-native per-time-step collision resolution (arXiv 1909.06623, Sec. 3).

The hot path (contacts, D, RPY/drag mobility, D^T + BB reductions, BBPGD
control) is hand-written CUDA for sm_100a in ``csrc/``, exported through the C
ABI in ``include/stokescol.h`` and bound here by ``api.Context`` (argument
marshalling only).  ``synthetic`` draws the seeded paper-shaped inputs.
"""
from .api import Context, ScError, nccl_unique_id, plan_partition, sym_pair_table  # noqa: F401

__all__ = ["Context", "ScError", "nccl_unique_id", "plan_partition", "sym_pair_table"]
