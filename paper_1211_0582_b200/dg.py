"""Thin ctypes binding of libdg.so (include/dg.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.  There is no
fallback — if libdg.so is missing or fails to load, importing this module
raises.

Functions keep the C names (dg_create, dg_mesh_upload, ...).  `Solver` is a
small convenience wrapper around them used by the tests and bench.py.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DG_LIB") or os.path.join(_HERE, "libdg.so")  # DG_LIB: profiling build
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "dg.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libdg.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'`")
lib = C.CDLL(LIB_PATH)

DG_OK, DG_ERR_ARG, DG_ERR_ORDER, DG_ERR_MESH, DG_ERR_STATE, DG_ERR_CUDA, DG_ERR_NCCL, DG_ERR_OOM = range(8)
(DG_VARIANT_AUTO, DG_VARIANT_BASIC, DG_VARIANT_MMA, DG_VARIANT_MMA_WS, DG_VARIANT_TC, DG_VARIANT_FUSED,
 DG_VARIANT_FFMA) = 0, 1, 2, 3, 4, 5, 6
DG_SYSTEM_MAXWELL, DG_SYSTEM_ACOUSTICS = 0, 1
DG_PARTITION_RANGES, DG_PARTITION_RCB = 0, 1
STATUS_NAMES = {0: "DG_OK", 1: "DG_ERR_ARG", 2: "DG_ERR_ORDER", 3: "DG_ERR_MESH", 4: "DG_ERR_STATE",
                5: "DG_ERR_CUDA", 6: "DG_ERR_NCCL", 7: "DG_ERR_OOM"}


class dg_config(C.Structure):
    _fields_ = [("order", C.c_int32), ("precision", C.c_int32), ("alpha", C.c_double),
                ("device", C.c_int32), ("stream", C.c_void_p), ("rank", C.c_int32),
                ("nranks", C.c_int32), ("nccl_id", C.c_void_p), ("variant", C.c_int32),
                ("reorder", C.c_int32), ("system", C.c_int32), ("partition", C.c_int32)]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)
_I32 = C.POINTER(C.c_int32)
_I8 = C.POINTER(C.c_int8)

_SIGS = {
    "dg_config_default": (None, [C.POINTER(dg_config)]),
    "dg_create": (C.c_int, [C.POINTER(dg_config), C.POINTER(_P)]),
    "dg_mesh_upload": (C.c_int, [_P, C.c_int64, _D, C.c_int64, _I64, _I32]),
    "dg_local_elements": (C.c_int, [_P, _I64, _I64]),
    "dg_get_sizes": (C.c_int, [_P, _I32, _I32, _I64, _I64]),
    "dg_fields_upload": (C.c_int, [_P, _D]),
    "dg_fields_upload_device": (C.c_int, [_P, _P]),
    "dg_rhs": (C.c_int, [_P, _D]),
    "dg_rhs_device": (C.c_int, [_P, _P]),
    "dg_lserk_step": (C.c_int, [_P, C.c_double, C.c_int32]),
    "dg_group_lserk_step": (C.c_int, [C.POINTER(_P), C.c_int32, C.c_double, C.c_int32]),
    "dg_fields_download": (C.c_int, [_P, _D]),
    "dg_fields_download_device": (C.c_int, [_P, _P]),
    "dg_synchronize": (C.c_int, [_P]),
    "dg_fields_upload_async": (C.c_int, [_P, _D]),
    "dg_fields_download_async": (C.c_int, [_P, _D]),
    "dg_get_maps": (C.c_int, [_P, _I64, _I8, _I64, _I64]),
    "dg_get_nodes": (C.c_int, [_P, _D, _D, _D]),
    "dg_get_reference": (C.c_int, [_P, _D, _D, _D, _D, _D, _D, _D, _D, _I32]),
    "dg_get_geometry": (C.c_int, [_P, _D, _D, _D]),
    "dg_time_stage_kernel": (C.c_int, [_P, C.c_int32, _D]),
    "dg_poison_padding": (C.c_int, [_P]),
    "dg_check_padding": (C.c_int, [_P, _I64]),
    "dg_launches_per_step": (C.c_int, [_P, _I32]),
    "dg_kernel_variant": (C.c_int, [_P, _I32]),
    "dg_last_error": (C.c_char_p, []),
    "dg_version": (C.c_char_p, []),
    "dg_destroy": (None, [_P]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args
    globals()[_name] = _f

EXPORTED = tuple(_SIGS)


class DGError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        msg = dg_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}: {msg}")


def check(status, where=""):
    if status != DG_OK:
        raise DGError(status, where)


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def group_lserk_step(solvers, dt, nsteps=1):
    """dg_group_lserk_step over loopback partition solvers (one per rank, same mesh)."""
    arr = (_P * len(solvers))(*[sv.h for sv in solvers])
    check(dg_group_lserk_step(arr, len(solvers), float(dt), int(nsteps)), "dg_group_lserk_step")


class Solver:
    """Convenience wrapper: one dg_solver.  Host arrays are numpy FP64 in the
    C-ABI layout [nfields][K_local][Np] (6 Maxwell, 4 acoustics); device arrays are
    torch tensors (data_ptr)."""

    def __init__(self, order, precision=8, alpha=1.0, device=0, stream=None, rank=0, nranks=1,
                 nccl_id=None, variant=DG_VARIANT_AUTO, reorder=False, system=DG_SYSTEM_MAXWELL,
                 partition=0):
        cfg = dg_config()
        dg_config_default(C.byref(cfg))
        cfg.order, cfg.precision, cfg.alpha, cfg.device = order, precision, alpha, device
        cfg.stream = stream
        cfg.rank, cfg.nranks, cfg.variant, cfg.reorder = rank, nranks, variant, int(bool(reorder))
        cfg.system = system
        cfg.partition = partition
        self.nfields = 4 if system == DG_SYSTEM_ACOUSTICS else 6
        self._io_refs = []  # host arrays borrowed by pending async copies
        self._id_buf = None
        if nccl_id is not None:
            self._id_buf = C.create_string_buffer(bytes(nccl_id), 128)
            cfg.nccl_id = C.cast(self._id_buf, C.c_void_p)
        h = _P()
        check(dg_create(C.byref(cfg), C.byref(h)), "dg_create")
        self.h = h
        self.order, self.precision = order, precision
        Np, Nfp = C.c_int32(), C.c_int32()
        check(dg_get_sizes(h, C.byref(Np), C.byref(Nfp), None, None), "dg_get_sizes")
        self.Np, self.Nfp = Np.value, Nfp.value
        self.K = 0
        self.K_local = 0

    def close(self):
        if getattr(self, "h", None):
            dg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def mesh_upload(self, VX, EToV, part=None):
        VX = np.ascontiguousarray(VX, dtype=np.float64)
        EToV = np.ascontiguousarray(EToV, dtype=np.int64)
        p = None if part is None else np.ascontiguousarray(part, dtype=np.int32)
        check(dg_mesh_upload(self.h, VX.shape[0], _ptr(VX, _D), EToV.shape[0], _ptr(EToV, _I64), _ptr(p, _I32)),
              "dg_mesh_upload")
        Kl, Kg = C.c_int64(), C.c_int64()
        check(dg_get_sizes(self.h, None, None, C.byref(Kl), C.byref(Kg)), "dg_get_sizes")
        self.K, self.K_local = Kg.value, Kl.value

    def local_elements(self):
        ids = np.zeros(self.K_local, dtype=np.int64)
        check(dg_local_elements(self.h, None, _ptr(ids, _I64)), "dg_local_elements")
        return ids

    def fields_upload(self, f):
        f = np.ascontiguousarray(f, dtype=np.float64)
        assert f.shape == (self.nfields, self.K_local, self.Np), f.shape
        check(dg_fields_upload(self.h, _ptr(f, _D)), "dg_fields_upload")

    def fields_upload_async(self, f):
        """Enqueue an upload from a C-contiguous float64 host array (page-locked for real
        overlap, e.g. torch.empty(..., pin_memory=True).numpy()); `f` must stay alive and
        unchanged until synchronize()."""
        assert f.dtype == np.float64 and f.flags.c_contiguous
        assert f.shape == (self.nfields, self.K_local, self.Np), f.shape
        self._io_refs.append(f)
        check(dg_fields_upload_async(self.h, _ptr(f, _D)), "dg_fields_upload_async")

    def fields_download_async(self, out):
        """Enqueue a download into `out` (float64, C-contiguous); valid after synchronize()."""
        assert out.dtype == np.float64 and out.flags.c_contiguous
        assert out.shape == (self.nfields, self.K_local, self.Np), out.shape
        self._io_refs.append(out)
        check(dg_fields_download_async(self.h, _ptr(out, _D)), "dg_fields_download_async")

    def fields_upload_device(self, t):
        check(dg_fields_upload_device(self.h, C.c_void_p(t.data_ptr())), "dg_fields_upload_device")

    def fields_download(self, out=None):
        if out is None:
            out = np.empty((self.nfields, self.K_local, self.Np))
        assert out.dtype == np.float64 and out.flags.c_contiguous
        assert out.shape == (self.nfields, self.K_local, self.Np), out.shape
        check(dg_fields_download(self.h, _ptr(out, _D)), "dg_fields_download")
        return out

    def fields_download_device(self, t):
        check(dg_fields_download_device(self.h, C.c_void_p(t.data_ptr())), "dg_fields_download_device")

    def rhs(self):
        out = np.empty((self.nfields, self.K_local, self.Np))
        check(dg_rhs(self.h, _ptr(out, _D)), "dg_rhs")
        return out

    def rhs_device(self, t):
        check(dg_rhs_device(self.h, C.c_void_p(t.data_ptr())), "dg_rhs_device")

    def lserk_step(self, dt, nsteps=1):
        check(dg_lserk_step(self.h, float(dt), int(nsteps)), "dg_lserk_step")

    def synchronize(self):
        check(dg_synchronize(self.h), "dg_synchronize")
        self._io_refs = []

    def get_maps(self):
        K, Nfp = self.K, self.Nfp
        EToE = np.zeros((K, 4), np.int64); EToF = np.zeros((K, 4), np.int8)
        vM = np.zeros((K, 4, Nfp), np.int64); vP = np.zeros((K, 4, Nfp), np.int64)
        check(dg_get_maps(self.h, _ptr(EToE, _I64), _ptr(EToF, _I8), _ptr(vM, _I64), _ptr(vP, _I64)), "dg_get_maps")
        return EToE, EToF, vM, vP

    def get_nodes(self):
        x, y, z = (np.zeros((self.K_local, self.Np)) for _ in range(3))
        check(dg_get_nodes(self.h, _ptr(x, _D), _ptr(y, _D), _ptr(z, _D)), "dg_get_nodes")
        return x, y, z

    def get_reference(self):
        Np, Nfp = self.Np, self.Nfp
        r, s, t = (np.zeros(Np) for _ in range(3))
        Dr, Ds, Dt, M = (np.zeros((Np, Np)) for _ in range(4))
        LIFT = np.zeros((Np, 4 * Nfp)); Fmask = np.zeros((4, Nfp), np.int32)
        check(dg_get_reference(self.h, *[_ptr(a, _D) for a in (r, s, t, Dr, Ds, Dt, M, LIFT)], _ptr(Fmask, _I32)),
              "dg_get_reference")
        return dict(r=r, s=s, t=t, Dr=Dr, Ds=Ds, Dt=Dt, M=M, LIFT=LIFT, Fmask=Fmask)

    def get_geometry(self):
        K = self.K
        J = np.zeros(K); G = np.zeros((K, 9)); nrm = np.zeros((K, 4, 4))
        check(dg_get_geometry(self.h, _ptr(J, _D), _ptr(G, _D), _ptr(nrm, _D)), "dg_get_geometry")
        return J, G, nrm

    def time_stage_kernel(self, reps=20):
        ms = C.c_double()
        check(dg_time_stage_kernel(self.h, int(reps), C.byref(ms)), "dg_time_stage_kernel")
        return ms.value

    def poison_padding(self):
        """NaN into every padding word of the device field buffers (test hook)."""
        check(dg_poison_padding(self.h), "dg_poison_padding")

    def check_padding(self):
        """[(padding words no longer NaN, real DOFs not finite)] for u0, u1, res, rhs scratch."""
        c = np.zeros(8, np.int64)
        check(dg_check_padding(self.h, _ptr(c, _I64)), "dg_check_padding")
        return [tuple(int(x) for x in c[2 * i:2 * i + 2]) for i in range(4)]

    def kernel_variant(self):
        """The stage kernel in use (dg_variant; AUTO resolved by the library)."""
        v = C.c_int32()
        check(dg_kernel_variant(self.h, C.byref(v)), "dg_kernel_variant")
        return v.value

    def launches_per_step(self):
        n = C.c_int32()
        check(dg_launches_per_step(self.h, C.byref(n)), "dg_launches_per_step")
        return n.value
