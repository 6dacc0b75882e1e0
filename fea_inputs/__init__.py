"""Seeded synthetic inputs (meshes, DOF maps, quadrature rules, u fields).

The ONLY module shared by the oracle (oracle/) and the CUDA path
(paper_2204_03893_b200/): it holds none of the assembly method's arithmetic.
"""
from .configs import CONFIGS, K_EXP, K_POLY, K_PWL, MASS, STIFF, Config, Workload, make_workload, scaled
from .mesh import Mesh, local_nodes, random_mesh_from_structured, single_element_mesh, structured_mesh, two_element_mesh
from .rules import RULE_POINTS, rule_degree_for_order, triangle_rule, triangle_rule_exact
