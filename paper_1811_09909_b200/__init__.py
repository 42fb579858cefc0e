"""B200-native DtN geometric multigrid for hybridized high-order FEM
(arXiv:1811.09909): MG-V-cycle-preconditioned CG on the trace system, all
steps in hand-written sm_100a CUDA kernels behind the C ABI include/mgdtn.h.

    from paper_1811_09909_b200 import MGSolver, SmootherConfig
"""
from .mgdtn import (MG_HDG, MG_IIPG_H, MG_NIPG_H, MG_SIPG_H, MG_SMOOTH_BLOCK_JACOBI, MG_SMOOTH_CHEBYSHEV, LIB_PATH,
                    LoopbackHub, MGError, MGSolver, Partition, SmootherConfig, load_library,
                    nccl_unique_id, partition_plan, agglomerate_seeds, macro_edge_params, macro_edge_transfer, partition_side_edges, smoother_from_config)

__all__ = ["MGSolver", "SmootherConfig", "MGError", "load_library", "LIB_PATH", "MG_HDG",
           "MG_SIPG_H", "MG_IIPG_H", "MG_NIPG_H", "MG_SMOOTH_BLOCK_JACOBI", "MG_SMOOTH_CHEBYSHEV", "smoother_from_config",
           "Partition", "LoopbackHub", "nccl_unique_id", "partition_plan", "partition_side_edges", "agglomerate_seeds", "macro_edge_params", "macro_edge_transfer"]
