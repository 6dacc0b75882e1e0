"""Input-generator invariants (SPEC.md:55-63 structured generator; SURVEY.md 8(d) recipe)."""
import numpy as np
import pytest

from fea_inputs import CONFIGS, local_nodes, make_workload, scaled, structured_mesh
from fea_inputs.mesh import random_mesh_from_structured


def _shoelace_area(m):
    a, b, c = (m.vert_xy[m.elem_vert[:, k]] for k in range(3))
    return 0.5 * np.abs((b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (c[:, 0] - a[:, 0]) * (b[:, 1] - a[:, 1]))


@pytest.mark.parametrize("N,p", [(1, 1), (2, 1), (3, 2), (4, 3), (3, 4)])
def test_counts(N, p):
    m = structured_mesh(N, p)
    assert m.n_e == 2 * N * N and m.n_v == (N + 1) ** 2 and m.n_dof == (p * N + 1) ** 2
    assert m.n_p == (p + 1) * (p + 2) // 2
    assert len(np.unique(m.elem_dof)) == m.n_dof
    assert abs(_shoelace_area(m).sum() - 1.0) < 1e-13


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_shared_dofs_agree_in_position(p):
    """Every element referencing a DOF places it at the same physical point (edge orientation,
    reading 7), also on jittered, renumbered meshes."""
    m = random_mesh_from_structured(5, p, seed=7 + p)
    nodes = np.array(local_nodes(p), dtype=np.float64) / p
    pos = {}
    for e in range(m.n_e):
        a, b, c = (m.vert_xy[v] for v in m.elem_vert[e])
        for k, d in enumerate(m.elem_dof[e]):
            x = nodes[k, 0] * a + nodes[k, 1] * b + nodes[k, 2] * c
            if d in pos:
                assert np.abs(pos[d] - x).max() < 1e-12
            else:
                pos[d] = x
    assert np.abs(m.dof_xy - np.array([pos[d] for d in range(m.n_dof)])).max() < 1e-12


def test_local_node_order_p2_matches_spec():
    """For P2 the documented order is corners then midsides opposite corners."""
    assert local_nodes(2) == [(2, 0, 0), (0, 2, 0), (0, 0, 2), (0, 1, 1), (1, 0, 1), (1, 1, 0)]


def test_jitter_keeps_boundary_and_validity():
    m = structured_mesh(16, 1, jitter=0.2, rng=np.random.default_rng(0))
    assert abs(_shoelace_area(m).sum() - 1.0) < 1e-12
    assert _shoelace_area(m).min() > 0.1 / 16 ** 2


def test_workloads_deterministic():
    for name in ("C1", "C2"):
        w1 = make_workload(CONFIGS[name])
        w2 = make_workload(CONFIGS[name])
        assert np.array_equal(w1.u0, w2.u0) and np.array_equal(w1.mesh.elem_dof, w2.mesh.elem_dof)
    w = make_workload(scaled(CONFIGS["C4"], 8))
    assert sorted(np.unique(w.mesh.elem_dof)) == list(range(81))
    assert not np.array_equal(w.mesh.elem_dof, structured_mesh(8, 1).elem_dof)  # permuted
