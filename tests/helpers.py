"""Shared test helpers: run the library (CUDA path, through the C ABI) and the oracle on the
same seeded inputs, in LIBRARY numbering."""
from __future__ import annotations

import numpy as np

import oracle
from fea_inputs import MASS, STIFF


def lib_numbering(mesh, lib_to_user):
    """The mesh with DOFs relabelled user -> library (assembly is permutation-equivariant)."""
    inv = np.empty_like(lib_to_user)
    inv[lib_to_user] = np.arange(lib_to_user.shape[0])
    return inv[mesh.elem_dof].astype(np.int32)


def coef_of(cfg):
    return (cfg.k_kind, tuple(cfg.k_par))


def coefs_of(cfg):
    """(mass, conductivity) coefficients of a config (they differ for E2)."""
    return cfg.coef_m, cfg.coef_c


def oracle_for(mesh, q_xy, q_w, u_user, lib_to_user, m_coef, c_coef, which, r0=0, r1=None, nthreads=1):
    """Oracle M/C rows [r0, r1) in library numbering."""
    import copy
    mlib = copy.copy(mesh)
    mlib.elem_dof = lib_numbering(mesh, lib_to_user)
    u_lib = np.ascontiguousarray(u_user[lib_to_user])
    return oracle.assemble(mlib, q_xy, q_w, u_lib, m_coef=m_coef, c_coef=c_coef, which=which,
                           r0=r0, r1=r1, nthreads=nthreads)


def maxabs_rel(gpu, ref):
    """North-star tolerance measure: max|gpu - ref| / max|ref| (reading 12)."""
    return float(np.abs(gpu - ref).max() / max(np.abs(ref).max(), 1e-300))


def library_assemble(mesh, q_xy, q_w, u_user, order, m_coef, c_coef, which=MASS | STIFF, reorder=True,
                     tuning=None, rank=0, world=1, device=0):
    """Set up a Context, assemble once with the full u (fea_assemble), return numpy results."""
    import torch
    from paper_2204_03893_b200.fea import Context
    ctx = Context(device=device, rank=rank, world=world)
    ctx.set_element(order, q_xy, q_w)
    ctx.mesh_upload(mesh.vert_xy, mesh.elem_vert, mesh.n_dof, mesh.elem_dof, reorder=reorder)
    ctx.set_tuning(4, which)
    for k, v in (tuning or {}).items():
        ctx.set_tuning(k, v)
    rb, nr, nnz = ctx.build_pattern()
    ctx.set_coefficient(MASS, m_coef[0], m_coef[1])
    ctx.set_coefficient(STIFF, c_coef[0], c_coef[1])
    perm = ctx.get_dof_perm()
    u_lib = torch.tensor(u_user[perm], dtype=torch.float64, device=f"cuda:{device}")
    vm = torch.full((max(nnz, 1),), np.nan, dtype=torch.float64, device=u_lib.device) if which & MASS else None
    vc = torch.full((max(nnz, 1),), np.nan, dtype=torch.float64, device=u_lib.device) if which & STIFF else None
    ctx.assemble(u_lib, vm, vc)
    ctx.sync()
    rp, ci = ctx.get_pattern()
    out = dict(ctx=ctx, perm=perm, row_begin=rb, n_rows=nr, nnz=nnz, row_ptr=rp, col_idx=ci,
               M=None if vm is None else vm[:nnz].cpu().numpy(), K=None if vc is None else vc[:nnz].cpu().numpy())
    return out
