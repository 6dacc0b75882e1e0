"""User-facing wrapper around one libfea Context: owns the value buffers and the
user <-> library renumbering, and bootstraps NCCL from a torch.distributed process group.

Marshalling only -- all assembly arithmetic happens in libfea's kernels.
"""
from __future__ import annotations

import numpy as np

from .fea import FEA_MASS, FEA_STIFF, Context, nccl_unique_id


class Assembler:
    """Set up once per mesh (Algorithm 2 lines 1-4), then call
    `reassemble(u)` once per Newton iteration (lines 5-12)."""

    def __init__(self, order: int, q_xy, q_w, vert_xy, elem_vert, n_dof: int, elem_dof, *,
                 device: int = 0, reorder: bool = True, which: int = FEA_MASS | FEA_STIFF,
                 coef_m=(0, (1.0,)), coef_c=(0, (1.0,)), rank: int = 0, world: int = 1,
                 process_group=None, tuning: dict | None = None):
        import torch
        self.torch = torch
        self.device = device
        self.which = which
        self.ctx = Context(device=device, rank=rank, world=world)
        self.ctx.set_element(order, q_xy, q_w)
        self.ctx.mesh_upload(vert_xy, elem_vert, n_dof, elem_dof, reorder=reorder)
        self.ctx.set_tuning(4, which)  # plan sized for the matrices actually assembled
        for k, v in (tuning or {}).items():
            self.ctx.set_tuning(k, v)
        self.row_begin, self.n_rows, self.nnz = self.ctx.build_pattern()
        self.ctx.set_coefficient(FEA_MASS, coef_m[0], coef_m[1])
        self.ctx.set_coefficient(FEA_STIFF, coef_c[0], coef_c[1])
        self.lib_to_user = self.ctx.get_dof_perm()
        self.n_dof = int(n_dof)
        dev = torch.device("cuda", device)
        n = max(self.nnz, 1)
        self.mass = torch.empty(n, dtype=torch.float64, device=dev) if which & FEA_MASS else None
        self.stiff = torch.empty(n, dtype=torch.float64, device=dev) if which & FEA_STIFF else None
        if world > 1:
            import torch.distributed as dist
            obj = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=process_group)
            self.ctx.set_nccl(obj[0])

    # -- numbering helpers (host-side marshalling)
    def to_library(self, u_user: np.ndarray) -> np.ndarray:
        return np.ascontiguousarray(np.asarray(u_user, dtype=np.float64)[self.lib_to_user])

    def owned_slice(self, u_lib: np.ndarray) -> np.ndarray:
        return np.ascontiguousarray(u_lib[self.row_begin:self.row_begin + self.n_rows])

    def pattern(self):
        return self.ctx.get_pattern()

    # -- per iteration
    def reassemble(self, u_owned):
        """u_owned: float64 CUDA tensor of this rank's library rows (world 1: all DOFs)."""
        self.ctx.reassemble(u_owned, self.mass, self.stiff)
        return self.mass, self.stiff

    def assemble(self, u_full):
        self.ctx.assemble(u_full, self.mass, self.stiff)
        return self.mass, self.stiff

    def close(self):
        self.ctx.close()
