"""Seeded synthetic meshes and DOF maps -- INPUT DATA, shared by oracle and CUDA path.

Stand-ins for the paper's Gmsh unit-square meshes (Table 1), which are not
available: structured N x N grids of the unit square, each cell split along its SW-NE
diagonal, P_p Lagrange DOFs on the (pN+1)^2 lattice (recipe: DESIGN.md "Inputs").
This module contains no arithmetic of the assembly method; it only produces
  vert_xy  (n_v, 2) float64   vertex coordinates
  elem_vert(n_e, 3) int32     vertices (a, b, c) of each triangle
  elem_dof (n_e, n_p) int32   index sets N_e in the documented local order
  dof_xy   (n_dof, 2) float64 DOF coordinates (only used to evaluate synthetic u fields)

Local node order for order p (reading 7): barycentric lattice nodes
(k0, k1, k2)/p, k0+k1+k2 = p; vertices v0, v1, v2; then the p-1 nodes of edge
e0 = (v1->v2), e1 = (v2->v0), e2 = (v0->v1), each listed from the edge's first vertex;
then interior nodes in lexicographic (k1, k2) order.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def local_nodes(p: int):
    """Barycentric integer triples (k0, k1, k2), sum p, in the documented local order."""
    nodes = [(p, 0, 0), (0, p, 0), (0, 0, p)]
    for t in range(1, p):  # e0: v1 -> v2
        nodes.append((0, p - t, t))
    for t in range(1, p):  # e1: v2 -> v0
        nodes.append((t, 0, p - t))
    for t in range(1, p):  # e2: v0 -> v1
        nodes.append((p - t, t, 0))
    interior = [(p - k1 - k2, k1, k2) for k1 in range(1, p) for k2 in range(1, p) if p - k1 - k2 >= 1]
    interior.sort(key=lambda k: (k[1], k[2]))
    nodes += interior
    assert len(nodes) == (p + 1) * (p + 2) // 2
    return nodes


@dataclass
class Mesh:
    p: int
    vert_xy: np.ndarray
    elem_vert: np.ndarray
    elem_dof: np.ndarray
    n_dof: int
    _dof_xy: np.ndarray | None = None

    @property
    def dof_xy(self) -> np.ndarray:
        """DOF coordinates: affine image of the reference node from the lowest-index
        element containing the DOF (straight edges)."""
        if self._dof_xy is None:
            self._dof_xy = dof_coordinates(self)
        return self._dof_xy

    @property
    def n_e(self) -> int:
        return int(self.elem_vert.shape[0])

    @property
    def n_v(self) -> int:
        return int(self.vert_xy.shape[0])

    @property
    def n_p(self) -> int:
        return int(self.elem_dof.shape[1])


def structured_mesh(N: int, p: int, jitter: float = 0.0, rng: np.random.Generator | None = None,
                    perm_rng: np.random.Generator | None = None) -> Mesh:
    """N x N unit-square grid, SW-NE split (element 2(jN+i) = (v_ij, v_i+1j, v_i+1j+1),
    2(jN+i)+1 = (v_ij, v_i+1j+1, v_ij+1)), P_p DOFs on lattice id J(pN+1)+I.

    jitter: interior vertices moved by U[-jitter*h, jitter*h] per coordinate (h = 1/N),
            drawn from `rng` (x then y for every vertex in id order, boundary draws discarded).
    perm_rng: if given, lattice DOF ids are relabelled by a uniform random permutation
            (for p = 1 the vertex ids are relabelled identically, reading 16).
    """
    assert N >= 1 and 1 <= p <= 4
    nv1 = N + 1
    ii, jj = np.meshgrid(np.arange(nv1), np.arange(nv1), indexing="xy")
    vi = ii.ravel().astype(np.int64)
    vj = jj.ravel().astype(np.int64)
    h = 1.0 / N
    vx = vi * h
    vy = vj * h
    if jitter > 0.0:
        d = rng.uniform(-jitter * h, jitter * h, size=(nv1 * nv1, 2))
        interior = (vi > 0) & (vi < N) & (vj > 0) & (vj < N)
        vx = np.where(interior, vx + d[:, 0], vx)
        vy = np.where(interior, vy + d[:, 1], vy)
    vert_xy = np.stack([vx, vy], axis=1).astype(np.float64)

    ci, cj = np.meshgrid(np.arange(N), np.arange(N), indexing="xy")
    ci = ci.ravel().astype(np.int64)
    cj = cj.ravel().astype(np.int64)
    v00 = cj * nv1 + ci
    v10 = v00 + 1
    v11 = v00 + nv1 + 1
    v01 = v00 + nv1
    n_e = 2 * N * N
    elem_vert = np.empty((n_e, 3), dtype=np.int64)
    elem_vert[0::2] = np.stack([v00, v10, v11], axis=1)
    elem_vert[1::2] = np.stack([v00, v11, v01], axis=1)

    # lattice coordinates of the element vertices (scaled by p)
    L = p * N + 1
    vlat = np.stack([vi * p, vj * p], axis=1)  # (n_v, 2) integer lattice coords
    nodes = local_nodes(p)
    n_p = len(nodes)
    elem_dof = np.empty((n_e, n_p), dtype=np.int64)
    la = vlat[elem_vert[:, 0]]
    lb = vlat[elem_vert[:, 1]]
    lc = vlat[elem_vert[:, 2]]
    for k, (k0, k1, k2) in enumerate(nodes):
        I = (k0 * la[:, 0] + k1 * lb[:, 0] + k2 * lc[:, 0]) // p
        J = (k0 * la[:, 1] + k1 * lb[:, 1] + k2 * lc[:, 1]) // p
        elem_dof[:, k] = J * L + I
    if perm_rng is not None:
        perm = perm_rng.permutation(L * L).astype(np.int64)  # old id -> new id
        elem_dof = perm[elem_dof]
        if p == 1:
            elem_vert = perm[elem_vert]
            new_xy = np.empty_like(vert_xy)
            new_xy[perm] = vert_xy
            vert_xy = new_xy
    return Mesh(p=p, vert_xy=vert_xy, elem_vert=elem_vert.astype(np.int32),
                elem_dof=elem_dof.astype(np.int32), n_dof=int(L * L))


def two_element_mesh() -> Mesh:
    """N=1 unit square: nodes 0=(0,0), 1=(1,0), 2=(0,1), 3=(1,1); T=(0,1,3), (0,3,2)
    (SURVEY.md 8(c) pins; same triangles as the structured generator at N=1 up to node ids)."""
    vert_xy = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    ev = np.array([[0, 1, 3], [0, 3, 2]], dtype=np.int32)
    return Mesh(p=1, vert_xy=vert_xy, elem_vert=ev, elem_dof=ev.copy(), n_dof=4)


def single_element_mesh(a, b, c, p: int = 1) -> Mesh:
    """One triangle with vertices a, b, c and its P_p DOFs numbered in local order."""
    vert_xy = np.array([a, b, c], dtype=np.float64)
    n_p = (p + 1) * (p + 2) // 2
    ev = np.array([[0, 1, 2]], dtype=np.int32)
    ed = np.arange(n_p, dtype=np.int32)[None, :]
    return Mesh(p=p, vert_xy=vert_xy, elem_vert=ev, elem_dof=ed, n_dof=n_p)


def random_mesh_from_structured(N: int, p: int, seed: int, jitter: float = 0.2, permute: bool = True) -> Mesh:
    """Small jittered, randomly renumbered mesh for property tests."""
    ss = np.random.SeedSequence(seed).spawn(2)
    return structured_mesh(N, p, jitter=jitter, rng=np.random.default_rng(ss[0]),
                           perm_rng=np.random.default_rng(ss[1]) if permute else None)


def dof_coordinates(mesh: Mesh) -> np.ndarray:
    p, n_p = mesh.p, mesh.n_p
    flat = mesh.elem_dof.ravel().astype(np.int64)  # element-major: first occurrence = lowest element
    uniq, first = np.unique(flat, return_index=True)
    assert uniq.shape[0] == mesh.n_dof and uniq[0] == 0 and uniq[-1] == mesh.n_dof - 1
    e_of = first // n_p
    k_of = first % n_p
    kk = np.array(local_nodes(p), dtype=np.float64)
    bary = kk[k_of] / p
    ev = mesh.elem_vert[e_of]
    xy = mesh.vert_xy
    return (bary[:, 0:1] * xy[ev[:, 0]] + bary[:, 1:2] * xy[ev[:, 1]] + bary[:, 2:3] * xy[ev[:, 2]])
