"""LaRoSA (arXiv 2507.01299) decode hot path for B200 (sm_100a).

The product is the C-ABI library ``lib/liblarosa.so`` (include/larosa.h); this package
is its thin Python binding.  See DESIGN.md.
"""
from .larosa import (  # noqa: F401
    LAROSA_GU_BLOCK, LAROSA_LEFT_QT, LAROSA_RIGHT_Q, LarosaError, LayerState, LayerWeights, abi_version,
    compute_k, fold_rotation, layer_workspace_size, lib, make_taps, pack_gate_up, rotate_topk, solve_alpha,
    sparse_gemv, sparse_layer,
)
