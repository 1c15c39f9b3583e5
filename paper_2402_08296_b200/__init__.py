"""B200-native DDM-GNN preconditioner + PCG (drop-in for the reference package
``ddmgnn``'s hot path: hybrid.build_ddm_gnn / apply_ddm_gnn and sparse.pcg/cg).

Compute runs in hand-written CUDA kernels for sm_100a (csrc/) behind the C ABI
declared in include/ddmgnn_b200.h; this package is the host-side mirror of the
reference's Python interface for that path.
"""

from .asm import AsmPreconditioner, apply_asm, build_asm
from .decomp import Decomposition, extend, finish_decomposition, nicolaides, restrict
from .dss import (DssModel, IterationWeights, Mlp, flat_params, init_model, load_model,
                  param_arrays, param_count, save_model)
from .hybrid import DdmGnnPreconditioner, apply_ddm_gnn, build_ddm_gnn, plan_batches
from .sparse import Ic0Preconditioner, SolveReport, cg, fcg, ic0, pcg, validate_csr

__version__ = "0.1.0"

__all__ = [
    "Decomposition", "finish_decomposition", "restrict", "extend", "nicolaides",
    "DssModel", "IterationWeights", "Mlp", "init_model", "load_model", "save_model",
    "param_count", "param_arrays", "flat_params",
    "DdmGnnPreconditioner", "build_ddm_gnn", "apply_ddm_gnn", "plan_batches",
    "SolveReport", "pcg", "fcg", "cg", "validate_csr", "AsmPreconditioner", "build_asm", "apply_asm",
    "Ic0Preconditioner", "ic0",
]
