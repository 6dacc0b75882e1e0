"""The five BASELINE.json configs as seeded synthetic workloads -- INPUT DATA.

Recipe: seeds SeedSequence(20220408 + c).spawn(4) ->
[jitter, u0, permutation, perturbations] with numpy PCG64, config c in 1..5.
Coefficients are *descriptions* (kind, parameters); each side evaluates k itself.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .mesh import Mesh, structured_mesh
from .rules import rule_degree_for_order, triangle_rule

K_POLY = 0  # k(u) = sum_i c_i u^i (Horner), n_par <= 9
K_EXP = 1   # k(u) = c0 * exp(c1 * u)
K_PWL = 2   # piecewise linear through (T_i, k_i) breakpoints, NEXT-4

MASS = 1
STIFF = 2


@dataclass
class Config:
    name: str
    index: int
    N: int
    p: int
    jitter: float
    permute: bool
    u_kind: str
    k_kind: int
    k_par: tuple
    which: int          # MASS | STIFF bitmask
    reassemblies: int
    reorder: bool       # library Morton reorder requested
    description: str = ""
    extra: dict = field(default_factory=dict)
    m_coef: tuple | None = None  # mass coefficient (kind, par) if it differs from k (else k)
    length: float = 1.0          # side of the square domain

    @property
    def coef_c(self) -> tuple:
        return (self.k_kind, tuple(self.k_par))

    @property
    def coef_m(self) -> tuple:
        return self.m_coef if self.m_coef is not None else self.coef_c

    @property
    def n_p(self) -> int:
        return (self.p + 1) * (self.p + 2) // 2

    @property
    def rule_degree(self) -> int:
        return rule_degree_for_order(self.p)

    @property
    def n_matrices(self) -> int:
        return (1 if self.which & MASS else 0) + (1 if self.which & STIFF else 0)


CONFIGS = {
    "C1": Config("C1", 1, 32, 1, 0.0, False, "U01", K_POLY, (1.0, 0.0, 1.0), MASS | STIFF, 1, True,
                 "P1 32x32, 3-pt deg-2, k=1+u^2, u~U[0,1], M+K"),
    "C2": Config("C2", 2, 256, 2, 0.0, False, "sinsin", K_POLY, (1.0, 0.0, 1.0), MASS | STIFF, 5, True,
                 "P2 256x256, 6-pt deg-4, k=1+u^2, u=sin(pi x)sin(pi y)+0.1N(0,1), M+K, 5 reassemblies"),
    "C3": Config("C3", 3, 1024, 3, 0.2, False, "U11", K_EXP, (1.0, 0.5), MASS | STIFF, 1, True,
                 "P3 1024x1024 jittered, 12-pt deg-6, k=exp(0.5u), u~U[-1,1], M+K"),
    "C4": Config("C4", 4, 4096, 1, 0.0, True, "U01", K_POLY, (1.0, 0.0, 1.0), STIFF, 10, True,
                 "P1 4096x4096 permuted then Morton-reordered, deg-2, k=1+u^2, u~U[0,1], K only, 10 reassemblies"),
    "C5": Config("C5", 5, 2048, 4, 0.2, False, "U01", K_POLY, (1.0, 0.0, 0.0, 0.0, 1.0), MASS | STIFF, 1, True,
                 "P4 2048x2048 jittered, 16-pt deg-8, k=1+u^4, u~U[0,1], M+K"),
    # stand-in for the paper's Experiment 2: the (0, 0.2 m)^2
    # square with P2 elements (43 x 43 grid: 7,569 DOFs; the paper's mesh has 7,593 nodes), mass
    # coefficient c rho = 1000 * 2400, conductivity k(T) piecewise linear through (0, 1.5),
    # (200, 0.7), (1000, 0.5), T in degrees C between T_0 = 0 and T_a = 1000
    "E2": Config("E2", 6, 43, 2, 0.0, False, "heat", K_PWL, (0.0, 1.5, 200.0, 0.7, 1000.0, 0.5), MASS | STIFF, 10,
                 True, "Exp. 2 stand-in: P2 43x43 on (0,0.2)^2, 6-pt deg-4, c rho = 2.4e6, k(T) PWL, "
                 "T = 1000 (1 - sin sin) + 10 N(0,1), M+K, 10 reassemblies",
                 m_coef=(K_POLY, (2.4e6,)), length=0.2),
}


def seeds(cfg: Config):
    ss = np.random.SeedSequence(20220408 + cfg.index).spawn(4)
    return [np.random.default_rng(s) for s in ss]  # jitter, u0, permutation, perturbations


def scaled(cfg: Config, N: int) -> Config:
    """Same workload recipe at another grid size (small parity cases)."""
    c = Config(**{**cfg.__dict__})
    c.N = N
    c.name = f"{cfg.name}@N{N}"
    return c


@dataclass
class Workload:
    cfg: Config
    mesh: Mesh
    q_xy: np.ndarray
    q_w: np.ndarray
    u0: np.ndarray
    pert_rng: np.random.Generator

    def u_sequence(self, R: int | None = None):
        """u_0, u_1 = u_0 + 0.01 xi_1, ... (reading 14)."""
        R = self.cfg.reassemblies if R is None else R
        u = self.u0.copy()
        out = [u.copy()]
        for _ in range(R - 1):
            u = u + 0.01 * self.pert_rng.standard_normal(u.shape[0])
            out.append(u.copy())
        return out


def make_workload(cfg: Config) -> Workload:
    r_jit, r_u, r_perm, r_pert = seeds(cfg)
    mesh = structured_mesh(cfg.N, cfg.p, jitter=cfg.jitter, rng=r_jit,
                           perm_rng=r_perm if cfg.permute else None)
    if cfg.length != 1.0:
        mesh.vert_xy = mesh.vert_xy * cfg.length
        mesh._dof_xy = None  # recomputed from the scaled vertices
    q_xy, q_w = triangle_rule(cfg.rule_degree)
    n = mesh.n_dof
    if cfg.u_kind == "U01":
        u0 = r_u.uniform(0.0, 1.0, n)
    elif cfg.u_kind == "U11":
        u0 = r_u.uniform(-1.0, 1.0, n)
    elif cfg.u_kind == "heat":  # hot boundary (T_a = 1000 C), cold centre, a little noise
        xy = mesh.dof_xy / cfg.length
        u0 = 1000.0 * (1.0 - np.sin(np.pi * xy[:, 0]) * np.sin(np.pi * xy[:, 1])) + 10.0 * r_u.standard_normal(n)
    elif cfg.u_kind == "sinsin":
        xy = mesh.dof_xy
        u0 = np.sin(np.pi * xy[:, 0]) * np.sin(np.pi * xy[:, 1]) + 0.1 * r_u.standard_normal(n)
    else:
        raise ValueError(cfg.u_kind)
    return Workload(cfg, mesh, q_xy, q_w, u0.astype(np.float64), r_pert)
