"""Interface-only exchange of u between row-partitioned ranks.

CPU (planning-only contexts, one per rank): every rank derives the same interface lists I_t; the
DOFs a rank's kernel reads (the columns of its rows: all DOFs of the elements touching them) are
its own rows or in some I_t; each I_t is owned by t and minimal (every entry is read by another
rank).  GPU (fake world on one device, no NCCL): pack on every rank, concatenate the send buffers
(what ncclAllGather delivers), unpack, assemble: bit-identical to the world-1 values (the per-slot
summation order does not depend on the partition, R22)."""
import numpy as np
import pytest

from fea_inputs import CONFIGS, K_POLY, make_workload, scaled, triangle_rule
from fea_inputs.mesh import random_mesh_from_structured


def _plan(mesh, p, xy, w, rank, world, device=-1, reorder=True):
    from paper_2204_03893_b200.fea import Context
    ctx = Context(device=device, rank=rank, world=world)
    ctx.set_element(p, xy, w)
    ctx.mesh_upload(mesh.vert_xy, mesh.elem_vert, mesh.n_dof, mesh.elem_dof, reorder=reorder)
    ctx.build_pattern()
    return ctx


@pytest.mark.parametrize("p,world", [(1, 2), (2, 3), (3, 4), (4, 2), (1, 7)])
def test_interface_lists_complete_and_minimal(p, world):
    m = random_mesh_from_structured(9, p, seed=900 + p)
    xy, w = triangle_rule(2 * p)
    ctxs = [_plan(m, p, xy, w, r, world) for r in range(world)]
    lists = [c.get_interface() for c in ctxs]
    for off, d in lists[1:]:  # identical on every rank
        assert np.array_equal(off, lists[0][0]) and np.array_equal(d, lists[0][1])
    off, d = lists[0]
    rows = [(c.row_begin, c.row_begin + c.n_rows) for c in ctxs]
    iface = [set(d[off[t]:off[t + 1]].tolist()) for t in range(world)]
    for t in range(world):
        assert all(rows[t][0] <= x < rows[t][1] for x in iface[t])          # owned by t
        assert np.all(np.diff(d[off[t]:off[t + 1]]) > 0)                     # ascending
    needed = []
    for r, c in enumerate(ctxs):
        _, ci = c.get_pattern()
        needed.append(set(np.unique(ci).tolist()))
    union = set().union(*iface)
    for r in range(world):
        halo = {x for x in needed[r] if not rows[r][0] <= x < rows[r][1]}
        assert halo <= union                                                 # complete
    for t in range(world):
        for x in iface[t]:
            assert any(x in needed[s] for s in range(world) if s != t)       # minimal
    assert max(len(s) for s in iface) == ctxs[0].stat(14)
    for c in ctxs:  # interior blocks (assembled during the exchange) come first; some exist
        assert 0 <= c.stat(15) <= c.stat(1)
        c.close()


def test_interior_blocks_on_a_larger_mesh():
    """Overlap (NEXT-3): on a config-sized mesh split over 2 and 4 ranks most blocks are interior
    (all their elements' DOFs owned) and a few are boundary blocks."""
    cfg = scaled(CONFIGS["C2"], 64)
    wl = make_workload(cfg)
    for world in (2, 4):
        for r in range(world):
            c = _plan(wl.mesh, cfg.p, wl.q_xy, wl.q_w, r, world)
            nb, ni = c.stat(1), c.stat(15)
            assert 0 < ni < nb, (world, r, ni, nb)
            c.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name,N,world", [("C1", 20, 3), ("C2", 24, 4), ("C3", 12, 2), ("C5", 8, 3)])
def test_fake_world_interface_exchange_bit_identical(name, N, world):
    import torch
    from paper_2204_03893_b200.fea import FEA_MASS, FEA_STIFF
    cfg = scaled(CONFIGS[name], N)
    wl = make_workload(cfg)
    m = wl.mesh
    coef = (cfg.k_kind, tuple(cfg.k_par))
    dev = "cuda:0"

    def setup(ctx):
        ctx.set_tuning(4, cfg.which)
        ctx.set_tuning(12, 0)  # bit-identity across worlds needs the same element labelling (no v6 skipping)
        ctx.build_pattern()
        ctx.set_coefficient(FEA_MASS, *coef)
        ctx.set_coefficient(FEA_STIFF, *coef)
        return ctx

    from paper_2204_03893_b200.fea import Context
    base = Context(device=0)
    base.set_element(cfg.p, wl.q_xy, wl.q_w)
    base.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof, reorder=cfg.reorder)
    setup(base)
    perm = base.get_dof_perm()
    u = torch.tensor(wl.u0[perm], dtype=torch.float64, device=dev)
    n = max(base.nnz, 1)
    Mb = torch.zeros(n, dtype=torch.float64, device=dev) if cfg.which & FEA_MASS else None
    Kb = torch.zeros(n, dtype=torch.float64, device=dev) if cfg.which & FEA_STIFF else None
    base.assemble(u, Mb, Kb)
    base.sync()

    ctxs = []
    for r in range(world):
        c = Context(device=0, rank=r, world=world)
        c.set_element(cfg.p, wl.q_xy, wl.q_w)
        c.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof, reorder=cfg.reorder)
        ctxs.append(setup(c))
    maxI = ctxs[0].stat(14)
    sends = []
    for c in ctxs:
        s = torch.full((max(maxI, 1),), np.nan, dtype=torch.float64, device=dev)
        c.exchange_pack(u[c.row_begin:c.row_begin + c.n_rows].contiguous(), s)
        sends.append(s[:maxI])
    recv = torch.cat(sends).contiguous() if maxI else torch.zeros(world, dtype=torch.float64, device=dev)
    slot = 0
    for c in ctxs:
        u_full = torch.full((m.n_dof,), np.nan, dtype=torch.float64, device=dev)
        c.exchange_unpack(u[c.row_begin:c.row_begin + c.n_rows].contiguous(), recv, u_full)
        nl = max(c.nnz, 1)
        M = torch.zeros(nl, dtype=torch.float64, device=dev) if Mb is not None else None
        K = torch.zeros(nl, dtype=torch.float64, device=dev) if Kb is not None else None
        c.assemble(u_full, M, K)  # the kernel reads only owned + interface entries (NaN elsewhere)
        c.sync()
        for got, ref in ((M, Mb), (K, Kb)):
            if got is not None:
                assert torch.equal(got[: c.nnz], ref[slot:slot + c.nnz])
        slot += c.nnz
    assert slot == base.nnz
