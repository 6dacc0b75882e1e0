"""Small runs of every libfea kernel, for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Kernels covered: k_reassemble5 (v5, P1 / P2), k_reassemble (v4, forced, P1-P4, generic rule),
k_reassemble6 (v6, P3 / P4: M+K, M only, K only, distinct coefficients), k_tensor / k_tensor4 / k_tensor5
(tensor contractions), k_pack / k_unpack (interface exchange, two ranks run one after the other).
Every result is also checked against the oracle, so a run that the sanitizer lets through is a
correct run too.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from fea_inputs import K_EXP, K_POLY, MASS, STIFF, triangle_rule  # noqa: E402
from fea_inputs.mesh import random_mesh_from_structured  # noqa: E402
from tests.helpers import library_assemble, maxabs_rel, oracle_for  # noqa: E402

TOL = 1e-12
POLY = (K_POLY, (1.0, 0.0, 1.0))


def check(res, ref, which):
    assert np.array_equal(res["row_ptr"], ref.row_ptr) and np.array_equal(res["col_idx"], ref.col_idx)
    if which & MASS:
        assert maxabs_rel(res["M"], ref.M) <= TOL
    if which & STIFF:
        assert maxabs_rel(res["K"], ref.K) <= TOL


def matrix_cases():
    n = 0
    for p, N, kern in ((1, 6, 0), (2, 4, 0), (3, 3, 0), (4, 2, 0), (1, 4, 4), (2, 3, 4), (3, 2, 4), (4, 2, 4)):
        m = random_mesh_from_structured(N, p, seed=10 + p)
        xy, w = triangle_rule(2 * p)
        u = np.random.default_rng(p).uniform(-1, 1, m.n_dof)
        for which, mc, cc in ((MASS | STIFF, POLY, POLY), (MASS, POLY, POLY), (STIFF, POLY, POLY),
                              (MASS | STIFF, (K_EXP, (1.0, 0.5)), POLY)):
            res = library_assemble(m, xy, w, u, p, mc, cc, which=which, tuning={2: kern} if kern else None)
            check(res, oracle_for(m, xy, w, u, res["perm"], mc, cc, which), which)
            res["ctx"].close()
            n += 1
    # a non-native rule (v4 generic path)
    m = random_mesh_from_structured(3, 2, seed=5)
    xy, w = triangle_rule(6)
    u = np.random.default_rng(5).uniform(-1, 1, m.n_dof)
    res = library_assemble(m, xy, w, u, 2, POLY, POLY)
    check(res, oracle_for(m, xy, w, u, res["perm"], POLY, POLY, 3), 3)
    return n + 1


def tensor_cases():
    from paper_2204_03893_b200.fea import Context
    import oracle
    from tests.helpers import lib_numbering
    import copy
    n = 0
    for p, N, tk in ((1, 5, 1), (1, 5, 5), (1, 24, 5), (2, 3, 4), (3, 2, 4)):
        m = random_mesh_from_structured(N, p, seed=20 + p)
        xy, w = triangle_rule(2 * p)
        rng = np.random.default_rng(p)
        u, v = rng.uniform(-1, 1, m.n_dof), rng.uniform(-1, 1, m.n_dof)
        ctx = Context(device=0)
        ctx.set_element(p, xy, w)
        ctx.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof)
        ctx.set_tuning(8, tk)
        _, _, nnz = ctx.build_pattern()
        ctx.set_coefficient(MASS, *POLY)
        ctx.set_coefficient(STIFF, *POLY)
        perm = ctx.get_dof_perm()
        mt = torch.zeros(nnz, dtype=torch.float64, device="cuda:0")
        ct = torch.zeros(nnz, dtype=torch.float64, device="cuda:0")
        ctx.assemble_tensor(torch.tensor(u[perm], device="cuda:0"), torch.tensor(v[perm], device="cuda:0"), mt, ct)
        ctx.sync()
        ml = copy.copy(m)
        ml.elem_dof = lib_numbering(m, perm)
        ref = oracle.assemble_tensor_contraction(ml, xy, w, u[perm], v[perm], m_coef=POLY, c_coef=POLY)
        assert maxabs_rel(mt.cpu().numpy(), ref.M) <= TOL and maxabs_rel(ct.cpu().numpy(), ref.K) <= TOL
        ctx.close()
        n += 1
    return n


def exchange_cases():
    """Two ranks, one after the other: pack -> concatenated send buffers -> unpack -> assemble."""
    from paper_2204_03893_b200.fea import Context
    p, world = 2, 2
    m = random_mesh_from_structured(4, p, seed=33)
    xy, w = triangle_rule(2 * p)
    u = np.random.default_rng(3).uniform(-1, 1, m.n_dof)
    ctxs = []
    for r in range(world):
        c = Context(device=0, rank=r, world=world)
        c.set_element(p, xy, w)
        c.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof)
        c.build_pattern()
        c.set_coefficient(MASS, *POLY)
        c.set_coefficient(STIFF, *POLY)
        ctxs.append(c)
    perm = ctxs[0].get_dof_perm()
    ul = torch.tensor(u[perm], device="cuda:0")
    maxI = ctxs[0].stat(14)
    sends = []
    for c in ctxs:
        s = torch.zeros(max(maxI, 1), dtype=torch.float64, device="cuda:0")
        c.exchange_pack(ul[c.row_begin:c.row_begin + c.n_rows].contiguous(), s)
        sends.append(s[:maxI])
    recv = torch.cat(sends).contiguous()
    for c in ctxs:
        uf = torch.zeros(m.n_dof, dtype=torch.float64, device="cuda:0")
        c.exchange_unpack(ul[c.row_begin:c.row_begin + c.n_rows].contiguous(), recv, uf)
        M = torch.zeros(max(c.nnz, 1), dtype=torch.float64, device="cuda:0")
        K = torch.zeros(max(c.nnz, 1), dtype=torch.float64, device="cuda:0")
        c.assemble(uf, M, K)
        c.sync()
        ref = oracle_for(m, xy, w, u, perm, POLY, POLY, 3, r0=c.row_begin, r1=c.row_begin + c.n_rows)
        assert maxabs_rel(M[:c.nnz].cpu().numpy(), ref.M) <= TOL and maxabs_rel(K[:c.nnz].cpu().numpy(), ref.K) <= TOL
        c.close()
    return world


if __name__ == "__main__":
    n = matrix_cases() + tensor_cases() + exchange_cases()
    torch.cuda.synchronize()
    print(f"sanitize cases ok: {n} runs")
