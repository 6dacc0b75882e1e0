"""ctypes binding of oracle/oracle.c (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

Plain argument marshalling; every number comes from oracle.c (Algorithm 1).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c (plain C, -ffp-contract=off: DESIGN.md reading 18)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC",
                               "-std=c99", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(_LIB)
        P = C.c_void_p
        i64 = C.c_int64
        lib.oracle_basis.argtypes = [C.c_int, C.c_int, P, P, P]
        lib.oracle_basis.restype = C.c_int
        lib.oracle_pattern.argtypes = [i64, i64, C.c_int, P, i64, i64, P, P]
        lib.oracle_pattern.restype = C.c_int
        lib.oracle_assemble.argtypes = [C.c_int, C.c_int, P, P, i64, P, i64, P, P, i64, P,
                                        C.c_int, C.c_int, P, C.c_int, C.c_int, P,
                                        i64, i64, P, P, P, P, C.c_int, P]
        lib.oracle_assemble.restype = C.c_int
        lib.oracle_assemble_tensor_contraction.argtypes = [C.c_int, C.c_int, P, P, P, i64, P, P, P, P,
                                                           C.c_int, C.c_int, P, C.c_int, C.c_int, P,
                                                           i64, i64, P, P, P, P]
        lib.oracle_assemble_tensor_contraction.restype = C.c_int
        lib.oracle_k.argtypes = [C.c_int, C.c_int, P, C.c_double]
        lib.oracle_k.restype = C.c_double
        lib.oracle_dk.argtypes = [C.c_int, C.c_int, P, C.c_double]
        lib.oracle_dk.restype = C.c_double
        lib.oracle_max_threads.restype = C.c_int
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def basis(p: int, q_xy: np.ndarray):
    """Phi (n_p, n_q) and J (n_q, n_p, 2) at the rule points (Algorithm 1)."""
    q_xy = _c(q_xy, np.float64)
    nq = q_xy.shape[0]
    n_p = (p + 1) * (p + 2) // 2
    phi = np.zeros((n_p, nq))
    J = np.zeros((nq, n_p, 2))
    rc = _load().oracle_basis(p, nq, _p(q_xy), _p(phi), _p(J))
    assert rc == n_p, rc
    return phi, J


def k_eval(kind: int, par, u: float) -> float:
    par = _c(par, np.float64)
    return float(_load().oracle_k(kind, len(par), _p(par), float(u)))


def dk_eval(kind: int, par, u: float) -> float:
    par = _c(par, np.float64)
    return float(_load().oracle_dk(kind, len(par), _p(par), float(u)))


@dataclass
class OracleCSR:
    row_begin: int
    row_ptr: np.ndarray  # int64, local (starts at 0)
    col_idx: np.ndarray  # int32, global columns
    M: np.ndarray | None = None
    K: np.ndarray | None = None

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def dense(self, which: str, n_cols: int) -> np.ndarray:
        vals = self.M if which == "M" else self.K
        nr = self.row_ptr.shape[0] - 1
        D = np.zeros((nr, n_cols))
        for r in range(nr):
            a, b = self.row_ptr[r], self.row_ptr[r + 1]
            D[r, self.col_idx[a:b]] = vals[a:b]
        return D


def pattern(n_dof: int, elem_dof: np.ndarray, r0: int = 0, r1: int | None = None):
    """Structural CSR pattern of rows [r0, r1) (reading 9)."""
    r1 = n_dof if r1 is None else r1
    ed = _c(elem_dof, np.int32)
    n_e, n_p = ed.shape
    row_ptr = np.zeros(r1 - r0 + 1, dtype=np.int64)
    lib = _load()
    rc = lib.oracle_pattern(n_dof, n_e, n_p, _p(ed), r0, r1, _p(row_ptr), None)
    if rc:
        raise ValueError(f"oracle_pattern failed: {rc}")
    col_idx = np.zeros(max(int(row_ptr[-1]), 1), dtype=np.int32)
    rc = lib.oracle_pattern(n_dof, n_e, n_p, _p(ed), r0, r1, _p(row_ptr), _p(col_idx))
    if rc:
        raise ValueError(f"oracle_pattern failed: {rc}")
    return row_ptr, col_idx[: int(row_ptr[-1])]


def assemble(mesh, q_xy, q_w, u, m_coef=(0, (1.0,)), c_coef=(0, (1.0,)), which: int = 3,
             r0: int = 0, r1: int | None = None, nthreads: int = 1, pat=None) -> OracleCSR:
    """M (which & 1) and C (which & 2) rows [r0, r1); coefficients (kind, params)."""
    n_dof = mesh.n_dof
    r1 = n_dof if r1 is None else r1
    if pat is None:
        pat = pattern(n_dof, mesh.elem_dof, r0, r1)
    row_ptr, col_idx = pat
    q_xy = _c(q_xy, np.float64)
    q_w = _c(q_w, np.float64)
    vxy = _c(mesh.vert_xy, np.float64)
    ev = _c(mesh.elem_vert, np.int32)
    ed = _c(mesh.elem_dof, np.int32)
    u = _c(u, np.float64)
    mp = _c(m_coef[1], np.float64)
    cp = _c(c_coef[1], np.float64)
    nnz = int(row_ptr[-1])
    M = np.zeros(max(nnz, 1)) if which & 1 else None
    K = np.zeros(max(nnz, 1)) if which & 2 else None
    bad = np.zeros(1, dtype=np.int64)
    rc = _load().oracle_assemble(mesh.p, q_xy.shape[0], _p(q_xy), _p(q_w), mesh.n_v, _p(vxy),
                                 ed.shape[0], _p(ev), _p(ed), n_dof, _p(u),
                                 int(m_coef[0]), len(mp), _p(mp), int(c_coef[0]), len(cp), _p(cp),
                                 r0, r1, _p(row_ptr), _p(_c(col_idx, np.int32)), _p(M), _p(K),
                                 int(nthreads), _p(bad))
    if rc == -3:
        raise ValueError(f"degenerate element {int(bad[0])}")
    if rc:
        raise RuntimeError(f"oracle_assemble failed: {rc}")
    return OracleCSR(r0, row_ptr, col_idx, None if M is None else M[:nnz], None if K is None else K[:nnz])


def assemble_tensor_contraction(mesh, q_xy, q_w, u, v, m_coef=None, c_coef=None,
                                r0: int = 0, r1: int | None = None, pat=None):
    """(Mt o2 v) and (Ct o2 v) of PAPER.md:298 (NEXT-1/NEXT-2) with k' of the given coefficient."""
    n_dof = mesh.n_dof
    r1 = n_dof if r1 is None else r1
    if pat is None:
        pat = pattern(n_dof, mesh.elem_dof, r0, r1)
    row_ptr, col_idx = pat
    nnz = int(row_ptr[-1])
    MT = np.zeros(max(nnz, 1)) if m_coef is not None else None
    CT = np.zeros(max(nnz, 1)) if c_coef is not None else None
    mk, mp = (m_coef if m_coef is not None else (0, (0.0,)))
    ck, cp = (c_coef if c_coef is not None else (0, (0.0,)))
    mp = _c(mp, np.float64)
    cp = _c(cp, np.float64)
    q_xy = _c(q_xy, np.float64)
    q_w = _c(q_w, np.float64)
    rc = _load().oracle_assemble_tensor_contraction(
        mesh.p, q_xy.shape[0], _p(q_xy), _p(q_w), _p(_c(mesh.vert_xy, np.float64)), mesh.n_e,
        _p(_c(mesh.elem_vert, np.int32)), _p(_c(mesh.elem_dof, np.int32)), _p(_c(u, np.float64)),
        _p(_c(v, np.float64)), int(mk), len(mp), _p(mp), int(ck), len(cp), _p(cp), r0, r1,
        _p(row_ptr), _p(_c(col_idx, np.int32)), _p(MT), _p(CT))
    if rc:
        raise RuntimeError(f"oracle tensor contraction failed: {rc}")
    return OracleCSR(r0, row_ptr, col_idx, None if MT is None else MT[:nnz], None if CT is None else CT[:nnz])
