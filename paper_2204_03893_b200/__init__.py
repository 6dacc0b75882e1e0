"""paper_2204_03893_b200 -- loop-free FP64 finite-element reassembly on NVIDIA B200.

The hot path of arXiv 2204.03893 (Voet): per-Newton-iteration reassembly of the k(u)-weighted
mass and conductivity matrices on triangular P1..P4 meshes, as one fused sm_100a kernel behind
the C ABI of include/fea.h (libfea.so).  See DESIGN.md.
"""
from .fea import (FEA_K_EXP, FEA_K_POLY, FEA_K_PWL, FEA_MASS, FEA_STIFF, Context, FeaError, load_library,
                  nccl_unique_id)
from .assembly import Assembler

__all__ = ["Context", "FeaError", "Assembler", "load_library", "nccl_unique_id", "FEA_MASS", "FEA_STIFF",
           "FEA_K_POLY", "FEA_K_EXP", "FEA_K_PWL"]
