"""Thin Python binding of the C ABI in include/cpm.h (argument marshalling only).

Every function here has the name of the C entry point it calls.  Arrays may be
torch tensors (CUDA or CPU) or numpy arrays; all must be float64, contiguous,
of length n_active.  Device tensors are passed as device pointers on the
current torch stream; host arrays are passed as host pointers and staged by the
library.  There is no fallback: if libcpm.so is missing or a call fails, an
exception is raised.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# CPM_LIB_PATH: another in-tree build of the same library (kernel A/B timing only)
LIB_PATH = os.environ.get("CPM_LIB_PATH") or os.path.join(_HERE, "_lib", "libcpm.so")

SPHERE = 1
TORUS = 2


class CpmError(RuntimeError):
    pass


class _Surface(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("param", ctypes.c_double * 4)]


class _BandInfo(ctypes.Structure):
    _fields_ = [
        ("n_active", ctypes.c_int64),
        ("n_ghost", ctypes.c_int64),
        ("n_tiles", ctypes.c_int64),
        ("n_runs", ctypes.c_int64),
        ("max_box", ctypes.c_int64),
        ("bytes_device", ctypes.c_int64),
        ("h", ctypes.c_double),
        ("lam", ctypes.c_double),
        ("L", ctypes.c_double),
        ("lattice_lo", ctypes.c_int32 * 3),
        ("lattice_hi", ctypes.c_int32 * 3),
        ("zero_fill", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("nranks", ctypes.c_int32),
        ("n_owned", ctypes.c_int64),
        ("n_halo", ctypes.c_int64),
    ]


class _SolveStats(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int32),
        ("converged", ctypes.c_int32),
        ("cycles", ctypes.c_int32),
        ("breakdown", ctypes.c_int32),
        ("resid_est", ctypes.c_double),
        ("resid_true", ctypes.c_double),
        ("bnorm", ctypes.c_double),
        ("seconds", ctypes.c_double),
    ]


class _RdParams(ctypes.Structure):
    _fields_ = [("a", ctypes.c_double), ("b", ctypes.c_double), ("gamma", ctypes.c_double),
                ("mu1", ctypes.c_double), ("mu2", ctypes.c_double), ("dt", ctypes.c_double),
                ("rtol", ctypes.c_double), ("restart", ctypes.c_int32), ("maxit", ctypes.c_int32)]


_ALLRED_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int64)
_ALLTOALLV_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                 ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double),
                                 ctypes.POINTER(ctypes.c_int64))


class _HostTransport(ctypes.Structure):
    _fields_ = [("ctx", ctypes.c_void_p), ("allreduce_sum", _ALLRED_FN), ("alltoallv", _ALLTOALLV_FN)]


_vp = ctypes.c_void_p
_SIGS = {
    "cpm_version": (ctypes.c_char_p, []),
    "cpm_last_error": (ctypes.c_char_p, []),
    "cpm_build_band": (ctypes.c_int, [ctypes.POINTER(_Surface), ctypes.c_double, ctypes.c_int,
                                      ctypes.c_double, _vp, ctypes.POINTER(_vp)]),
    "cpm_band_get_info": (ctypes.c_int, [_vp, ctypes.POINTER(_BandInfo)]),
    "cpm_band_active_coords": (ctypes.c_int, [_vp, _vp]),
    "cpm_band_ghost_coords": (ctypes.c_int, [_vp, _vp]),
    "cpm_band_eval_order": (ctypes.c_int, [_vp, _vp, _vp]),
    "cpm_band_item_rounds": (ctypes.c_int, [_vp, _vp]),
    "cpm_band_free": (None, [_vp]),
    "cpm_apply": (ctypes.c_int, [_vp, ctypes.c_double, _vp, _vp, _vp]),
    "cpm_apply_async": (ctypes.c_int, [_vp, ctypes.c_double, _vp, _vp, _vp]),
    "cpm_apply_sync": (ctypes.c_int, [_vp]),
    "cpm_solve": (ctypes.c_int, [_vp, ctypes.c_double, _vp, _vp, ctypes.c_double, ctypes.c_int,
                                 ctypes.c_int, _vp, ctypes.POINTER(_SolveStats), _vp]),
    "cpm_ras_setup": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_double, _vp, ctypes.POINTER(_vp)]),
    "cpm_ras_apply": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "cpm_ras_free": (None, [_vp]),
    "cpm_eval_sph": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_double, _vp, _vp]),
    "cpm_eval_torus_rhs": (ctypes.c_int, [_vp, _vp, ctypes.c_int, _vp, _vp]),
    "cpm_profile_enable": (ctypes.c_int, [ctypes.c_int]),
    "cpm_profile_reset": (ctypes.c_int, []),
    "cpm_profile_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_int64)]),
    "cpm_kernel_launches": (ctypes.c_int64, []),
    "cpm_comm_unique_id": (ctypes.c_int, [_vp]),
    "cpm_comm_init": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)]),
    "cpm_comm_init_host": (ctypes.c_int, [ctypes.POINTER(_HostTransport), ctypes.c_int, ctypes.c_int,
                                          ctypes.POINTER(_vp)]),
    "cpm_comm_free": (None, [_vp]),
    "cpm_part_create": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, ctypes.POINTER(_vp)]),
    "cpm_part_get_info": (ctypes.c_int, [_vp, _vp]),
    "cpm_part_halo_nodes": (ctypes.c_int, [_vp, _vp]),
    "cpm_part_set_send": (ctypes.c_int, [_vp, _vp, _vp]),
    "cpm_part_apply_local": (ctypes.c_int, [_vp, ctypes.c_double, _vp, _vp, _vp, _vp]),
    "cpm_part_apply": (ctypes.c_int, [_vp, _vp, ctypes.c_double, _vp, _vp, _vp]),
    "cpm_part_solve": (ctypes.c_int, [_vp, _vp, ctypes.c_double, _vp, _vp, ctypes.c_double, ctypes.c_int,
                                      ctypes.c_int, _vp, ctypes.POINTER(_SolveStats), _vp]),
    "cpm_part_ras_setup": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                          _vp, ctypes.POINTER(_vp)]),
    "cpm_ras_get_info": (ctypes.c_int, [_vp, _vp]),
    "cpm_ras_halo_nodes": (ctypes.c_int, [_vp, _vp]),
    "cpm_ras_set_send": (ctypes.c_int, [_vp, _vp, _vp]),
    "cpm_part_ras_apply_local": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "cpm_part_ras_apply": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "cpm_part_free": (None, [_vp]),
    "cpm_rd_step": (ctypes.c_int, [_vp, ctypes.POINTER(_RdParams), _vp, _vp, ctypes.POINTER(_SolveStats),
                                   ctypes.POINTER(_SolveStats), _vp]),
    "cpm_part_rd_step": (ctypes.c_int, [_vp, _vp, ctypes.POINTER(_RdParams), _vp, _vp,
                                        ctypes.POINTER(_SolveStats), ctypes.POINTER(_SolveStats), _vp]),
}

_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libcpm.so (raises if it was not built — no fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise CpmError(f"{path} not found: build it with __graft_entry__.build() "
                       "(python -m paper_2110_06322_b200._build)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def _check(rc: int, what: str):
    if rc != 0:
        msg = load_library().cpm_last_error().decode(errors="replace")
        raise CpmError(f"{what} failed (code {rc}): {msg}")


def _ptr_stream(x, n: int, writable: bool):
    """(pointer, stream) for a float64 torch tensor / numpy array of length n."""
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(x, torch.Tensor):
        if x.dtype != torch.float64 or not x.is_contiguous() or x.numel() != n:
            raise CpmError(f"expected a contiguous float64 tensor of {n} elements, got "
                           f"{x.dtype} {tuple(x.shape)}")
        stream = torch.cuda.current_stream(x.device).cuda_stream if x.is_cuda else None
        return x.data_ptr(), stream
    if isinstance(x, np.ndarray):
        if x.dtype != np.float64 or not x.flags.c_contiguous or x.size != n:
            raise CpmError(f"expected a contiguous float64 array of {n} elements")
        if writable and not x.flags.writeable:
            raise CpmError("output array is read-only")
        return x.ctypes.data, None
    raise CpmError(f"unsupported array type {type(x)}")


@dataclass
class BandInfo:
    n_active: int
    n_ghost: int
    n_tiles: int
    n_runs: int
    max_box: int
    bytes_device: int
    h: float
    lam: float
    L: float
    zero_fill: bool
    n_owned: int
    n_halo: int
    rank: int
    nranks: int


class Band:
    """Owning wrapper of a cpm_band handle."""

    def __init__(self, handle, surface_kind: int, params):
        self._h = handle
        self.surface_kind = surface_kind
        self.params = tuple(params)
        info = _BandInfo()
        _check(load_library().cpm_band_get_info(self._h, ctypes.byref(info)), "cpm_band_get_info")
        self.info = BandInfo(info.n_active, info.n_ghost, info.n_tiles, info.n_runs, info.max_box,
                             info.bytes_device, info.h, info.lam, info.L, bool(info.zero_fill),
                             info.n_owned, info.n_halo, info.rank, info.nranks)

    @property
    def handle(self):
        return self._h

    @property
    def n(self) -> int:
        return self.info.n_active

    def close(self):
        if self._h:
            load_library().cpm_band_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def cpm_build_band(kind: str, h: float, p: int = 3, L: float = 2.0, stream=None, **params) -> Band:
    """cpm_build_band(surface, h, p=3): the lambda-tube band of a sphere or torus."""
    lib = load_library()
    s = _Surface()
    if kind == "sphere":
        s.kind = SPHERE
        s.param[0] = params.get("R", 1.0)
    elif kind == "torus":
        s.kind = TORUS
        s.param[0] = params.get("R", 1.0)
        s.param[1] = params.get("r", 0.4)
    else:
        raise CpmError(f"unknown surface {kind!r}")
    out = _vp()
    _check(lib.cpm_build_band(ctypes.byref(s), float(h), int(p), float(L), stream, ctypes.byref(out)),
           "cpm_build_band")
    return Band(out, s.kind, list(s.param))


def cpm_band_active_coords(band: Band) -> np.ndarray:
    out = np.empty((band.n, 3), dtype=np.int32)
    _check(load_library().cpm_band_active_coords(band.handle, out.ctypes.data), "cpm_band_active_coords")
    return out


def cpm_band_ghost_coords(band: Band) -> np.ndarray:
    out = np.empty((band.info.n_ghost, 3), dtype=np.int32)
    _check(load_library().cpm_band_ghost_coords(band.handle, out.ctypes.data), "cpm_band_ghost_coords")
    return out


def cpm_band_eval_order(band: Band):
    """(tiles[n_tiles, 6] = e0, e1, np, row stride, plane stride, box cells; eoff[e1 of the
    last tile]) — diagnostics of the extend's node order (include/cpm.h)."""
    lib = load_library()
    tiles = np.empty((band.info.n_tiles, 6), dtype=np.int32)
    _check(lib.cpm_band_eval_order(band.handle, tiles.ctypes.data, None), "cpm_band_eval_order")
    ne = int(tiles[-1, 1]) if len(tiles) else 0
    eoff = np.empty(ne, dtype=np.uint32)
    _check(lib.cpm_band_eval_order(band.handle, tiles.ctypes.data, eoff.ctypes.data), "cpm_band_eval_order")
    return tiles, eoff


def cpm_band_item_rounds(band: Band):
    """rounds[n_tiles, 32] (uint64) — the item rounds of an item-order band (include/cpm.h)."""
    out = np.zeros((band.info.n_tiles, 32), dtype=np.uint64)
    _check(load_library().cpm_band_item_rounds(band.handle, out.ctypes.data), "cpm_band_item_rounds")
    return out


def cpm_apply(band: Band, c: float, u, y, stream=None):
    """y = (c I - Delta_S^h) u."""
    pu, su = _ptr_stream(u, band.n, False)
    py, sy = _ptr_stream(y, band.n, True)
    _check(load_library().cpm_apply(band.handle, float(c), pu, py, stream or su or sy), "cpm_apply")
    return y


def cpm_apply_async(band: Band, c: float, u, y, stream=None):
    """Pipelined apply on pinned host buffers (include/cpm.h); y complete after cpm_apply_sync."""
    pu, su = _ptr_stream(u, band.n, False)
    py, sy = _ptr_stream(y, band.n, True)
    _check(load_library().cpm_apply_async(band.handle, float(c), pu, py, stream or su or sy), "cpm_apply_async")
    return y


def cpm_apply_sync(band: Band):
    _check(load_library().cpm_apply_sync(band.handle), "cpm_apply_sync")


@dataclass
class SolveStats:
    iterations: int
    converged: bool
    cycles: int
    breakdown: bool
    resid_est: float
    resid_true: float
    bnorm: float
    seconds: float


def cpm_solve(band: Band, c: float, f, u, rtol: float = 1e-10, restart: int = 30,
              maxit: int = 100000, ras=None, stream=None) -> SolveStats:
    """Solve (c - Delta_S^h) u = f by (F)GMRES(restart); u holds x0 on entry."""
    pf, sf = _ptr_stream(f, band.n, False)
    pu, su = _ptr_stream(u, band.n, True)
    st = _SolveStats()
    _check(load_library().cpm_solve(band.handle, float(c), pf, pu, float(rtol), int(restart), int(maxit),
                                    ras.handle if ras is not None else None, ctypes.byref(st),
                                    stream or sf or su), "cpm_solve")
    return SolveStats(st.iterations, bool(st.converged), st.cycles, bool(st.breakdown), st.resid_est,
                      st.resid_true, st.bnorm, st.seconds)


class Ras:
    def __init__(self, handle, band: Band):
        self._h = handle
        self.band = band

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            load_library().cpm_ras_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def cpm_ras_setup(band: Band, n_sub: int, overlap: int, k_inner: int, c: float, stream=None) -> Ras:
    out = _vp()
    _check(load_library().cpm_ras_setup(band.handle, int(n_sub), int(overlap), int(k_inner), float(c),
                                        stream, ctypes.byref(out)), "cpm_ras_setup")
    return Ras(out, band)


def cpm_ras_apply(ras: Ras, r, z, stream=None):
    pr, sr = _ptr_stream(r, ras.band.n, False)
    pz, sz = _ptr_stream(z, ras.band.n, True)
    _check(load_library().cpm_ras_apply(ras.handle, pr, pz, stream or sr or sz), "cpm_ras_apply")
    return z


def cpm_rd_step(band: Band, u, v, a: float = 0.1, b: float = 0.9, gamma: float = 10.0,
                mu1: float = 1e-3, mu2: float = 1e-2, dt: float = 1e-3, rtol: float = 1e-10,
                restart: int = 50, maxit: int = 100000, stream=None):
    """One IMEX Euler step of the Schnakenberg system (config 4); u, v device tensors,
    updated in place.  Returns the two SolveStats."""
    pu, su = _ptr_stream(u, band.n, True)
    pv, sv = _ptr_stream(v, band.n, True)
    prm = _RdParams(a, b, gamma, mu1, mu2, dt, rtol, restart, maxit)
    s1, s2 = _SolveStats(), _SolveStats()
    _check(load_library().cpm_rd_step(band.handle, ctypes.byref(prm), pu, pv, ctypes.byref(s1),
                                      ctypes.byref(s2), stream or su or sv), "cpm_rd_step")
    return tuple(SolveStats(x.iterations, bool(x.converged), x.cycles, bool(x.breakdown), x.resid_est,
                            x.resid_true, x.bnorm, x.seconds) for x in (s1, s2))


def cpm_part_rd_step(part, comm, u_owned, v_owned, a: float = 0.1, b: float = 0.9, gamma: float = 10.0,
                     mu1: float = 1e-3, mu2: float = 1e-2, dt: float = 1e-3, rtol: float = 1e-10,
                     restart: int = 50, maxit: int = 100000, stream=None):
    """cpm_rd_step on this rank's owned slices (device tensors of n_owned, in place)."""
    pu, su = _ptr_stream(u_owned, part.n_owned, True)
    pv, _ = _ptr_stream(v_owned, part.n_owned, True)
    prm = _RdParams(a, b, gamma, mu1, mu2, dt, rtol, restart, maxit)
    s1, s2 = _SolveStats(), _SolveStats()
    _check(load_library().cpm_part_rd_step(part.handle, comm.handle if comm else None, ctypes.byref(prm),
                                           pu, pv, ctypes.byref(s1), ctypes.byref(s2), stream or su),
           "cpm_part_rd_step")
    return tuple(SolveStats(x.iterations, bool(x.converged), x.cycles, bool(x.breakdown), x.resid_est,
                            x.resid_true, x.bnorm, x.seconds) for x in (s1, s2))


def cpm_eval_sph(band: Band, l: int, m: int, scale: float, out, stream=None):
    po, so = _ptr_stream(out, band.n, True)
    _check(load_library().cpm_eval_sph(band.handle, int(l), int(m), float(scale), po, stream or so),
           "cpm_eval_sph")
    return out


def cpm_eval_torus_rhs(band: Band, coeffs: np.ndarray, out, stream=None):
    co = np.ascontiguousarray(coeffs, dtype=np.float64)
    po, so = _ptr_stream(out, band.n, True)
    _check(load_library().cpm_eval_torus_rhs(band.handle, co.ctypes.data, int(co.shape[0]), po,
                                             stream or so), "cpm_eval_torus_rhs")
    return out


def cpm_profile_enable(on: bool = True):
    _check(load_library().cpm_profile_enable(1 if on else 0), "cpm_profile_enable")


def cpm_profile_reset():
    _check(load_library().cpm_profile_reset(), "cpm_profile_reset")


def cpm_profile_read(name: str):
    ms = ctypes.c_double()
    n = ctypes.c_int64()
    _check(load_library().cpm_profile_read(name.encode(), ctypes.byref(ms), ctypes.byref(n)),
           "cpm_profile_read")
    return ms.value, n.value


def cpm_kernel_launches() -> int:
    return int(load_library().cpm_kernel_launches())


def cpm_version() -> str:
    return load_library().cpm_version().decode()


# ---------------------------------------------------------------- multi-GPU
class _PartInfo(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("lo", ctypes.c_int64),
                ("hi", ctypes.c_int64), ("n_owned", ctypes.c_int64), ("n_halo", ctypes.c_int64),
                ("n_tiles", ctypes.c_int64), ("n_send", ctypes.c_int64), ("n_interior_tiles", ctypes.c_int64)]


class Part:
    """Owning wrapper of a cpm_part handle (this rank's slab of a band)."""

    def __init__(self, handle, band: Band):
        self._h = handle
        self.band = band
        self.refresh()

    def refresh(self):
        inf = _PartInfo()
        _check(load_library().cpm_part_get_info(self._h, ctypes.byref(inf)), "cpm_part_get_info")
        self.rank, self.nranks = inf.rank, inf.nranks
        self.lo, self.hi = inf.lo, inf.hi
        self.n_owned, self.n_halo, self.n_tiles, self.n_send = inf.n_owned, inf.n_halo, inf.n_tiles, inf.n_send
        self.n_interior_tiles = inf.n_interior_tiles

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            load_library().cpm_part_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Comm:
    def __init__(self, handle):
        self._h = handle

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            load_library().cpm_comm_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def cpm_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load_library().cpm_comm_unique_id(buf), "cpm_comm_unique_id")
    return buf.raw


def cpm_comm_init(uid: bytes, rank: int, nranks: int) -> Comm:
    buf = ctypes.create_string_buffer(uid, 128)
    out = _vp()
    _check(load_library().cpm_comm_init(buf, int(rank), int(nranks), ctypes.byref(out)), "cpm_comm_init")
    return Comm(out)


def cpm_comm_init_host(allreduce_sum, alltoallv, rank: int, nranks: int) -> Comm:
    """Host-staged communicator (include/cpm.h cpm_comm_init_host).

    allreduce_sum(buf: np.ndarray) sums buf over the ranks in place;
    alltoallv(send, send_counts, recv, recv_counts) exchanges blocks in rank order
    (numpy views of the library's pinned staging; counts are int64 arrays).
    Both return None (an exception makes the library call fail)."""
    nr = int(nranks)

    def _ar(ctx, buf, n):
        try:
            allreduce_sum(np.ctypeslib.as_array(buf, shape=(int(n),)))
            return 0
        except Exception:  # pragma: no cover - reported through the library error
            import traceback
            traceback.print_exc()
            return 1

    def _a2a(ctx, send, sc, recv, rc):
        try:
            scn = np.ctypeslib.as_array(sc, shape=(nr,)).copy()
            rcn = np.ctypeslib.as_array(rc, shape=(nr,)).copy()
            ns, nrv = int(scn.sum()), int(rcn.sum())
            sv = np.ctypeslib.as_array(send, shape=(ns,)) if ns else np.empty(0)
            rv = np.ctypeslib.as_array(recv, shape=(nrv,)) if nrv else np.empty(0)
            alltoallv(sv, scn, rv, rcn)
            return 0
        except Exception:  # pragma: no cover
            import traceback
            traceback.print_exc()
            return 1

    fa, fb = _ALLRED_FN(_ar), _ALLTOALLV_FN(_a2a)
    tr = _HostTransport(None, fa, fb)
    out = _vp()
    _check(load_library().cpm_comm_init_host(ctypes.byref(tr), int(rank), nr, ctypes.byref(out)),
           "cpm_comm_init_host")
    c = Comm(out)
    c._keep = (fa, fb, tr)  # the library holds the function pointers
    return c


def cpm_part_create(band: Band, rank: int, nranks: int, stream=None) -> Part:
    out = _vp()
    _check(load_library().cpm_part_create(band.handle, int(rank), int(nranks), stream, ctypes.byref(out)),
           "cpm_part_create")
    return Part(out, band)


def cpm_part_halo_nodes(part: Part) -> np.ndarray:
    out = np.empty(part.n_halo, dtype=np.int64)
    _check(load_library().cpm_part_halo_nodes(part.handle, out.ctypes.data if part.n_halo else None),
           "cpm_part_halo_nodes")
    return out


def cpm_part_set_send(part: Part, send_global: np.ndarray, counts: np.ndarray):
    sg = np.ascontiguousarray(send_global, dtype=np.int64)
    ct = np.ascontiguousarray(counts, dtype=np.int64)
    if ct.size != part.nranks or sg.size != int(ct.sum()):
        raise CpmError("cpm_part_set_send: counts must have nranks entries summing to len(send_global)")
    _check(load_library().cpm_part_set_send(part.handle, sg.ctypes.data if sg.size else None, ct.ctypes.data),
           "cpm_part_set_send")
    part.refresh()


def cpm_part_apply_local(part: Part, c: float, u_owned, u_halo, y_owned, stream=None):
    pu, su = _ptr_stream(u_owned, part.n_owned, False)
    ph = None
    if part.n_halo:
        ph, _ = _ptr_stream(u_halo, part.n_halo, False)
    py, _ = _ptr_stream(y_owned, part.n_owned, True)
    _check(load_library().cpm_part_apply_local(part.handle, float(c), pu, ph, py, stream or su),
           "cpm_part_apply_local")
    return y_owned


def cpm_part_apply(part: Part, comm: Comm, c: float, u_owned, y_owned, stream=None):
    pu, su = _ptr_stream(u_owned, part.n_owned, False)
    py, _ = _ptr_stream(y_owned, part.n_owned, True)
    _check(load_library().cpm_part_apply(part.handle, comm.handle if comm else None, float(c), pu, py,
                                         stream or su), "cpm_part_apply")
    return y_owned


def cpm_part_solve(part: Part, comm: Comm, c: float, f_owned, u_owned, rtol: float = 1e-10,
                   restart: int = 30, maxit: int = 100000, ras=None, stream=None) -> SolveStats:
    pf, sf = _ptr_stream(f_owned, part.n_owned, False)
    pu, _ = _ptr_stream(u_owned, part.n_owned, True)
    st = _SolveStats()
    _check(load_library().cpm_part_solve(part.handle, comm.handle if comm else None, float(c), pf, pu,
                                         float(rtol), int(restart), int(maxit),
                                         ras.handle if ras is not None else None, ctypes.byref(st),
                                         stream or sf), "cpm_part_solve")
    return SolveStats(st.iterations, bool(st.converged), st.cycles, bool(st.breakdown), st.resid_est,
                      st.resid_true, st.bnorm, st.seconds)


# ---------------------------------------------------------------- distributed RAS
class _RasInfo(ctypes.Structure):
    _fields_ = [("n_sub", ctypes.c_int32), ("sub0", ctypes.c_int32), ("n_sub_local", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("n_members", ctypes.c_int64),
                ("n_owned", ctypes.c_int64), ("n_halo", ctypes.c_int64), ("n_send", ctypes.c_int64)]


def cpm_ras_get_info(ras) -> dict:
    inf = _RasInfo()
    _check(load_library().cpm_ras_get_info(ras.handle, ctypes.byref(inf)), "cpm_ras_get_info")
    return {f: getattr(inf, f) for f, _ in _RasInfo._fields_}


def cpm_part_ras_setup(part: Part, n_sub: int, overlap: int, k_inner: int, c: float, stream=None) -> Ras:
    out = _vp()
    _check(load_library().cpm_part_ras_setup(part.handle, int(n_sub), int(overlap), int(k_inner), float(c),
                                             stream, ctypes.byref(out)), "cpm_part_ras_setup")
    return Ras(out, part.band)


def cpm_ras_halo_nodes(ras) -> np.ndarray:
    n = cpm_ras_get_info(ras)["n_halo"]
    out = np.empty(n, dtype=np.int64)
    _check(load_library().cpm_ras_halo_nodes(ras.handle, out.ctypes.data if n else None), "cpm_ras_halo_nodes")
    return out


def cpm_ras_set_send(ras, send_global: np.ndarray, counts: np.ndarray):
    sg = np.ascontiguousarray(send_global, dtype=np.int64)
    ct = np.ascontiguousarray(counts, dtype=np.int64)
    if sg.size != int(ct.sum()):
        raise CpmError("cpm_ras_set_send: counts must sum to len(send_global)")
    _check(load_library().cpm_ras_set_send(ras.handle, sg.ctypes.data if sg.size else None, ct.ctypes.data),
           "cpm_ras_set_send")


def cpm_part_ras_apply_local(ras, r_owned, r_halo, z_owned, stream=None):
    inf = cpm_ras_get_info(ras)
    pr, sr = _ptr_stream(r_owned, inf["n_owned"], False)
    ph = None
    if inf["n_halo"]:
        ph, _ = _ptr_stream(r_halo, inf["n_halo"], False)
    pz, _ = _ptr_stream(z_owned, inf["n_owned"], True)
    _check(load_library().cpm_part_ras_apply_local(ras.handle, pr, ph, pz, stream or sr),
           "cpm_part_ras_apply_local")
    return z_owned


def cpm_part_ras_apply(ras, comm: Comm, r_owned, z_owned, stream=None):
    inf = cpm_ras_get_info(ras)
    pr, sr = _ptr_stream(r_owned, inf["n_owned"], False)
    pz, _ = _ptr_stream(z_owned, inf["n_owned"], True)
    _check(load_library().cpm_part_ras_apply(ras.handle, comm.handle if comm else None, pr, pz, stream or sr),
           "cpm_part_ras_apply")
    return z_owned
