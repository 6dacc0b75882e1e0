"""Thin ctypes binding of libfea (include/fea.h): argument marshalling only.

Every step of the hot path runs in libfea's sm_100a kernels.  There is no CPU fallback:
importing this module without the built libfea.so raises, and so does every call on a
machine without a CUDA device.  PyTorch supplies device memory, streams and process groups.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfea.so")

FEA_OK = 0
_STATUS = {0: "FEA_OK", -1: "FEA_E_ARG", -2: "FEA_E_STATE", -3: "FEA_E_MESH", -4: "FEA_E_CUDA",
           -5: "FEA_E_NCCL", -6: "FEA_E_OOM", -7: "FEA_E_UNSUPPORTED"}
FEA_REORDER_NONE, FEA_REORDER_MORTON = 0, 1
FEA_MASS, FEA_STIFF = 1, 2
FEA_K_POLY, FEA_K_EXP, FEA_K_PWL = 0, 1, 2
FEA_TUNE_SMEM_BUDGET, FEA_TUNE_KERNEL, FEA_TUNE_EMAX, FEA_TUNE_PLAN_WHICH = 1, 2, 3, 4
FEA_TUNE_TENSOR_KERNEL = 8

# the exported C symbols (tests check every one of them against include/fea.h)
SYMBOLS = ["fea_create", "fea_set_element", "fea_set_rule", "fea_mesh_upload", "fea_set_tuning", "fea_build_pattern",
           "fea_get_pattern", "fea_get_pattern_rows", "fea_get_dof_perm", "fea_get_elem_perm", "fea_set_coefficient",
           "fea_assemble_mass", "fea_assemble_stiffness", "fea_assemble", "fea_reassemble",
           "fea_reassemble_host", "fea_assemble_tensor", "fea_get_interface", "fea_exchange_pack",
           "fea_exchange_unpack", "fea_nccl_unique_id", "fea_set_nccl", "fea_set_host_transport", "fea_sync",
           "fea_get_stat",
           "fea_last_error", "fea_destroy"]


# fea.h fea_host_allgather_fn: int (*)(const double* send, double* recv, int64_t count, void* user)
HOST_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)


class FeaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load_library():
    """Load libfea.so; raises if it is missing (the product path never falls back)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libfea.so not built ({LIB_PATH}); run `python -m paper_2204_03893_b200.build`")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    P, I, L = C.c_void_p, C.c_int, C.c_int64
    sig = {
        "fea_create": [C.POINTER(P), I, P, I, I],
        "fea_set_element": [P, I, I, P, P],
        "fea_set_rule": [P, I, I, P, P],
        "fea_mesh_upload": [P, L, P, L, P, L, P, I],
        "fea_set_tuning": [P, I, L],
        "fea_build_pattern": [P, P, P, P],
        "fea_get_pattern": [P, P, P],
        "fea_get_pattern_rows": [P, L, L, P, P],
        "fea_get_dof_perm": [P, P],
        "fea_get_elem_perm": [P, P],
        "fea_set_coefficient": [P, I, I, I, P],
        "fea_assemble_mass": [P, P, P],
        "fea_assemble_stiffness": [P, P, P],
        "fea_assemble": [P, P, P, P],
        "fea_reassemble": [P, P, P, P],
        "fea_reassemble_host": [P, P, P, P],
        "fea_assemble_tensor": [P, P, P, P, P],
        "fea_get_interface": [P, P, P],
        "fea_exchange_pack": [P, P, P],
        "fea_exchange_unpack": [P, P, P, P],
        "fea_nccl_unique_id": [P],
        "fea_set_nccl": [P, P],
        "fea_set_host_transport": [P, P, P],
        "fea_sync": [P],
        "fea_get_stat": [P, I, P],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = C.c_int
    lib.fea_last_error.argtypes = [P]
    lib.fea_last_error.restype = C.c_char_p
    lib.fea_destroy.argtypes = [P]
    lib.fea_destroy.restype = None
    _lib = lib
    return lib


def _np_ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _dev_ptr(t, name, n=None):
    """Device pointer of a contiguous float64 CUDA tensor (None -> NULL)."""
    if t is None:
        return None
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise TypeError(f"{name}: expected a contiguous float64 CUDA tensor")
    if n is not None and t.numel() < n:
        raise ValueError(f"{name}: length {t.numel()} < {n}")
    return C.c_void_p(t.data_ptr())


class Context:
    """One libfea context per (process, GPU); calls mirror include/fea.h one to one."""

    def __init__(self, device: int = 0, stream=None, rank: int = 0, world: int = 1):
        self._lib = load_library()
        self.device = device
        if device == -1:  # planning-only context: pattern / plan, no device work
            self.stream = None
            sptr = None
        else:
            import torch
            if not torch.cuda.is_available():
                raise RuntimeError("libfea needs a CUDA device (no CPU fallback)")
            if stream is None:
                stream = torch.cuda.current_stream(device)
            self.stream = stream
            sptr = C.c_void_p(stream.cuda_stream)
        h = C.c_void_p()
        self._check(self._lib.fea_create(C.byref(h), device, sptr, rank, world), None)
        self._h = h
        self.rank, self.world = rank, world
        self.order = self.n_dof = self.nnz = self.n_rows = self.row_begin = None

    # -- plumbing
    def _check(self, st, h="self"):
        if st != FEA_OK:
            msg = ""
            if h is not None and getattr(self, "_h", None):
                msg = (self._lib.fea_last_error(self._h) or b"").decode()
            raise FeaError(st, msg)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.fea_destroy(self._h)
            self._h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- setup (synchronous)
    def set_element(self, order: int, q_xy, q_w):
        q_xy = np.ascontiguousarray(q_xy, dtype=np.float64)
        q_w = np.ascontiguousarray(q_w, dtype=np.float64)
        self._check(self._lib.fea_set_element(self._h, order, q_w.shape[0], _np_ptr(q_xy), _np_ptr(q_w)))
        self.order = order

    def set_rule(self, which: int, q_xy, q_w):
        """A separate quadrature rule for the matrices in `which` (NEXT-4)."""
        xy = np.ascontiguousarray(q_xy, dtype=np.float64)
        w = np.ascontiguousarray(q_w, dtype=np.float64)
        self._check(self._lib.fea_set_rule(self._h, int(which), w.shape[0], _np_ptr(xy), _np_ptr(w)))

    def mesh_upload(self, vert_xy, elem_vert, n_dof: int, elem_dof, reorder: bool = True):
        vxy = np.ascontiguousarray(vert_xy, dtype=np.float64)
        ev = np.ascontiguousarray(elem_vert, dtype=np.int32)
        ed = np.ascontiguousarray(elem_dof, dtype=np.int32)
        self._check(self._lib.fea_mesh_upload(self._h, vxy.shape[0], _np_ptr(vxy), ev.shape[0], _np_ptr(ev),
                                              int(n_dof), _np_ptr(ed), FEA_REORDER_MORTON if reorder else FEA_REORDER_NONE))
        self.n_dof = int(n_dof)
        self.n_e = int(ev.shape[0])

    def set_tuning(self, key: int, value: int):
        self._check(self._lib.fea_set_tuning(self._h, key, int(value)))

    def build_pattern(self):
        rb, nr, nz = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(self._lib.fea_build_pattern(self._h, C.byref(rb), C.byref(nr), C.byref(nz)))
        self.row_begin, self.n_rows, self.nnz = rb.value, nr.value, nz.value
        return self.row_begin, self.n_rows, self.nnz

    def get_pattern(self):
        rp = np.zeros(self.n_rows + 1, dtype=np.int64)
        ci = np.zeros(max(self.nnz, 1), dtype=np.int32)
        self._check(self._lib.fea_get_pattern(self._h, _np_ptr(rp), _np_ptr(ci)))
        return rp, ci[: self.nnz]

    def get_pattern_rows(self, r0: int, r1: int):
        """Local rows [r0, r1): (row_ptr[r0..r1] (not rebased), col_idx of those rows)."""
        rp = np.zeros(r1 - r0 + 1, dtype=np.int64)
        self._check(self._lib.fea_get_pattern_rows(self._h, int(r0), int(r1), _np_ptr(rp), None))
        ci = np.zeros(max(int(rp[-1] - rp[0]), 1), dtype=np.int32)
        self._check(self._lib.fea_get_pattern_rows(self._h, int(r0), int(r1), _np_ptr(rp), _np_ptr(ci)))
        return rp, ci[: int(rp[-1] - rp[0])]

    def get_dof_perm(self):
        p = np.zeros(self.n_dof, dtype=np.int64)
        self._check(self._lib.fea_get_dof_perm(self._h, _np_ptr(p)))
        return p

    def get_elem_perm(self):
        p = np.zeros(self.n_e, dtype=np.int64)
        self._check(self._lib.fea_get_elem_perm(self._h, _np_ptr(p)))
        return p

    def set_coefficient(self, which: int, kind: int, par):
        par = np.ascontiguousarray(par, dtype=np.float64)
        self._check(self._lib.fea_set_coefficient(self._h, which, kind, par.shape[0], _np_ptr(par)))

    def stat(self, key: int) -> int:
        v = C.c_int64()
        self._check(self._lib.fea_get_stat(self._h, key, C.byref(v)))
        return v.value

    # -- per iteration (asynchronous on the ctx stream)
    def assemble(self, u_full, mass_vals=None, stiff_vals=None):
        self._check(self._lib.fea_assemble(self._h, _dev_ptr(u_full, "u_full", self.n_dof),
                                           _dev_ptr(mass_vals, "mass_vals", self.nnz),
                                           _dev_ptr(stiff_vals, "stiff_vals", self.nnz)))

    def assemble_mass(self, u_full, vals):
        self._check(self._lib.fea_assemble_mass(self._h, _dev_ptr(u_full, "u_full", self.n_dof),
                                                _dev_ptr(vals, "vals", self.nnz)))

    def assemble_stiffness(self, u_full, vals):
        self._check(self._lib.fea_assemble_stiffness(self._h, _dev_ptr(u_full, "u_full", self.n_dof),
                                                     _dev_ptr(vals, "vals", self.nnz)))

    def reassemble(self, u_owned, mass_vals=None, stiff_vals=None):
        self._check(self._lib.fea_reassemble(self._h, _dev_ptr(u_owned, "u_owned", self.n_rows),
                                             _dev_ptr(mass_vals, "mass_vals", self.nnz),
                                             _dev_ptr(stiff_vals, "stiff_vals", self.nnz)))

    def assemble_tensor(self, u_full, v_full, mt_vals=None, ct_vals=None):
        """(M o2 v) into mt_vals and (C o2 v) into ct_vals (NEXT-1 / NEXT-2)."""
        self._check(self._lib.fea_assemble_tensor(self._h, _dev_ptr(u_full, "u_full", self.n_dof),
                                                  _dev_ptr(v_full, "v_full", self.n_dof),
                                                  _dev_ptr(mt_vals, "mt_vals", self.nnz),
                                                  _dev_ptr(ct_vals, "ct_vals", self.nnz)))

    def get_interface(self):
        """Interface lists of every rank (NEXT-3): (offsets [world + 1], dofs)."""
        off = np.zeros(self.world + 1, dtype=np.int64)
        self._check(self._lib.fea_get_interface(self._h, _np_ptr(off), None))
        dofs = np.zeros(max(int(off[-1]), 1), dtype=np.int32)
        self._check(self._lib.fea_get_interface(self._h, _np_ptr(off), _np_ptr(dofs)))
        return off, dofs[: int(off[-1])]

    def exchange_pack(self, u_owned, send):
        self._check(self._lib.fea_exchange_pack(self._h, _dev_ptr(u_owned, "u_owned", self.n_rows),
                                                _dev_ptr(send, "send", self.stat(14))))

    def exchange_unpack(self, u_owned, recv, u_full):
        self._check(self._lib.fea_exchange_unpack(self._h, _dev_ptr(u_owned, "u_owned", self.n_rows),
                                                  _dev_ptr(recv, "recv", self.stat(14) * self.world),
                                                  _dev_ptr(u_full, "u_full", self.n_dof)))

    def reassemble_host(self, u_host, mass_host=None, stiff_host=None):
        """Host buffers (numpy float64; pinned torch CPU tensors also accepted via .numpy())."""
        def hp(a, n, name):
            if a is None:
                return None
            if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"] or a.shape[0] < n:
                raise TypeError(f"{name}: expected contiguous float64 of length >= {n}")
            return _np_ptr(a)
        nu = self.n_dof if self.world == 1 else self.n_rows
        self._check(self._lib.fea_reassemble_host(self._h, hp(u_host, nu, "u_host"), hp(mass_host, self.nnz, "mass_host"),
                                                  hp(stiff_host, self.nnz, "stiff_host")))

    def set_nccl(self, uid: bytes):
        b = (C.c_char * 128).from_buffer_copy(uid)
        self._check(self._lib.fea_set_nccl(self._h, b))

    def set_host_transport(self, fn):
        """fn(send: np.ndarray[count], recv: np.ndarray[world * count]) -> None: an allgather of the
        float64 values over any host transport (fea.h fea_set_host_transport); None -> NCCL.  The
        arrays view the library's pinned buffers (valid during the call only)."""
        if fn is None:
            self._htrans = None
            self._check(self._lib.fea_set_host_transport(self._h, None, None))
            return
        world = self.world

        def tramp(send, recv, count, user):
            try:
                s = np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_double)), shape=(count,))
                r = np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_double)), shape=(count * world,))
                fn(s, r)
                return 0
            except Exception:  # reported as FEA_E_NCCL by the library
                import traceback
                traceback.print_exc()
                return 1

        self._htrans = HOST_ALLGATHER(tramp)  # keep the ctypes thunk alive
        self._check(self._lib.fea_set_host_transport(self._h, C.cast(self._htrans, C.c_void_p), None))

    def sync(self):
        self._check(self._lib.fea_sync(self._h))


def nccl_unique_id() -> bytes:
    lib = load_library()
    b = (C.c_char * 128)()
    st = lib.fea_nccl_unique_id(b)
    if st != FEA_OK:
        raise FeaError(st, "ncclGetUniqueId failed")
    return bytes(b)
