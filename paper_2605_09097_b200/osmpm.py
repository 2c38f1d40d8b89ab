"""Thin ctypes binding of libosmpm (include/osmpm.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels of
csrc/.  There is no CPU fallback: importing this module without the built
libosmpm.so raises.  Arrays may be numpy (host) or torch CUDA tensors (device);
outputs are returned in the same memory space as requested.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OSMPM_LIB", os.path.join(_HERE, "libosmpm.so"))  # OSMPM_LIB: A/B builds

OK = 0
HOST, DEVICE = 0, 1
F64, F32 = 0, 1
COARSE_TO_FINE, FINE_TO_COARSE = 0, 1
STATUS = {0: "OK", 1: "INVALID_ARG", 2: "OUT_OF_DOMAIN", 3: "INVERTED_F", 4: "NEWTON_NOT_CONVERGED",
          5: "LINESEARCH_STAGNATION", 6: "SCHWARZ_NOT_CONVERGED", 7: "COUPLING_CONFIG", 8: "CUDA", 9: "NCCL",
          10: "OOM", 11: "STATE"}


class OsmpmError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"osmpm {STATUS.get(code, code)}: {msg}")
        self.code = code


class GridDesc(C.Structure):
    _fields_ = [("dim", C.c_int32), ("origin", C.c_double * 3), ("dx", C.c_double), ("dims", C.c_int64 * 3)]


class Material(C.Structure):
    _fields_ = [("E", C.c_double), ("nu", C.c_double)]


class ParticlesView(C.Structure):
    _fields_ = [("n", C.c_int64), ("space", C.c_int), ("x", C.c_void_p), ("v", C.c_void_p), ("F", C.c_void_p),
                ("B", C.c_void_p), ("m", C.c_void_p), ("V0", C.c_void_p), ("material", C.c_void_p),
                ("is_boundary", C.c_void_p)]


class NewtonSettings(C.Structure):
    _fields_ = [("max_newton", C.c_int32), ("max_cg", C.c_int32), ("fixed_iters", C.c_int32), ("guess", C.c_int32),
                ("newton_rtol", C.c_double), ("newton_atol", C.c_double), ("cg_rtol", C.c_double),
                ("ls_min_alpha", C.c_double), ("energy_noise_rtol", C.c_double), ("cg_variant", C.c_int32),
                ("psd", C.c_int32)]


class SolveStats(C.Structure):
    _fields_ = [("newton_iters", C.c_int32), ("cg_iters", C.c_int32), ("ls_halvings", C.c_int32),
                ("status", C.c_int32), ("grad_norm0", C.c_double), ("grad_norm", C.c_double),
                ("energy", C.c_double), ("negcurv", C.c_int32), ("ls_failures", C.c_int32),
                ("floor_accept", C.c_int32), ("psd_solves", C.c_int32)]


class SchwarzSettings(C.Structure):
    _fields_ = [("eps_conv", C.c_double), ("eps_tol", C.c_double), ("tau_gamma_rel", C.c_double),
                ("k_max", C.c_int32), ("M", C.c_int32), ("parity_fixed_k", C.c_int32),
                ("coarse", NewtonSettings), ("fine", NewtonSettings)]


class SchwarzReport(C.Structure):
    _fields_ = [("iters", C.c_int32), ("fine_substeps", C.c_int32), ("converged", C.c_int32),
                ("n_recv_B", C.c_int32), ("n_recv_S", C.c_int32), ("r_B", C.c_double * 256),
                ("r_S", C.c_double * 256)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (there is no CPU fallback)")
        _lib = C.CDLL(LIB_PATH)
        _lib.osmpm_last_error.restype = C.c_char_p
        _lib.osmpm_version.restype = C.c_char_p
        _lib.osmpm_subdomain_destroy.restype = None
        _lib.osmpm_ctx_destroy.restype = None
        _lib.osmpm_coupler_destroy.restype = None
    return _lib


def _check(rc):
    if rc != OK:
        raise OsmpmError(rc, lib().osmpm_last_error().decode())


def comm_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().osmpm_comm_unique_id(buf))
    return bytes(buf)


def sort_pairs(ctx, keys, vals, nbits):
    """Stable radix sort of (uint32 key, int32 value) pairs on the low nbits bits, in place (numpy or
    torch CUDA arrays)."""
    if _is_torch(keys):
        kp, vp, sp = C.c_void_p(keys.data_ptr()), C.c_void_p(vals.data_ptr()), DEVICE
    else:
        assert keys.dtype == np.uint32 and vals.dtype == np.int32 and keys.flags.c_contiguous and vals.flags.c_contiguous
        kp, vp, sp = keys.ctypes.data_as(C.c_void_p), vals.ctypes.data_as(C.c_void_p), HOST
    _check(lib().osmpm_sort_pairs(ctx._h, kp, vp, C.c_int64(int(keys.shape[0])), C.c_int32(nbits), C.c_int(sp)))


def newton_settings(max_newton=50, max_cg=1000, fixed_iters=0, guess=0, newton_rtol=1e-8, newton_atol=0.0,
                    cg_rtol=1e-8, ls_min_alpha=2.0 ** -20, energy_noise_rtol=1e-13, cg_variant=0,
                    psd=0) -> NewtonSettings:
    return NewtonSettings(max_newton, max_cg, fixed_iters, guess, newton_rtol, newton_atol, cg_rtol, ls_min_alpha,
                          energy_noise_rtol, cg_variant, psd)


# --------------------------------------------------------------------------------------------
# buffer marshalling: numpy -> (pointer, HOST); torch CUDA tensor -> (data_ptr, DEVICE)
# --------------------------------------------------------------------------------------------

def _is_torch(a):
    return type(a).__module__.startswith("torch")


def _ptr(a, dtype=np.float64):
    if a is None:
        return None, None
    if _is_torch(a):
        import torch
        want = {np.float64: torch.float64, np.int32: torch.int32, np.uint8: torch.uint8,
                np.int64: torch.int64}[dtype]
        assert a.dtype == want and a.is_contiguous(), (a.dtype, want)
        return C.c_void_p(a.data_ptr()), (DEVICE if a.is_cuda else HOST)
    assert isinstance(a, np.ndarray) and a.dtype == dtype and a.flags.c_contiguous, (type(a), getattr(a, "dtype", None))
    return a.ctypes.data_as(C.c_void_p), HOST


def _space(*arrays):
    sp = None
    for a in arrays:
        if a is None:
            continue
        _, s = _ptr(a, _dtype_of(a))
        if sp is None:
            sp = s
        elif sp != s:
            raise ValueError("all arrays of one call must live in the same memory space")
    return HOST if sp is None else sp


def _dtype_of(a):
    if _is_torch(a):
        import torch
        return {torch.float64: np.float64, torch.int32: np.int32, torch.uint8: np.uint8, torch.int64: np.int64}[a.dtype]
    return a.dtype.type


def _empty_like_space(shape, dtype, device):
    if device is None:
        return np.zeros(shape, dtype=dtype)
    import torch
    tdt = {np.float64: torch.float64, np.uint8: torch.uint8}[dtype]
    return torch.zeros(shape, dtype=tdt, device=device)


class Context:
    def __init__(self, device=0, stream=None):
        """stream: a cudaStream_t handle (e.g. torch.cuda.current_stream().cuda_stream) the library
        enqueues all its work on, or None for a library-owned stream.  Handle 0 (torch's default
        stream) is passed as cudaStreamLegacy so the work stays ordered with torch's."""
        self._h = C.c_void_p()
        s = None if stream is None else C.c_void_p(stream if stream != 0 else 1)  # 1 == cudaStreamLegacy
        _check(lib().osmpm_ctx_create(C.c_int(device), s, C.byref(self._h)))
        self.device = device
        self._children = []  # weakrefs to subdomains / couplers: destroyed before the context

    def profile(self, enable=True):
        _check(lib().osmpm_profile_enable(self._h, C.c_int(1 if enable else 0)))

    def profile_reset(self):
        _check(lib().osmpm_profile_reset(self._h))

    def kernel_time(self, family):
        n = C.c_int64()
        ms = C.c_double()
        _check(lib().osmpm_kernel_time(self._h, family.encode(), C.byref(n), C.byref(ms)))
        return n.value, ms.value

    def init_comm(self, rank, nranks, uid: bytes):
        """Join the NCCL process group (one rank per GPU); uid from comm_unique_id() on rank 0."""
        assert len(uid) == 128
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().osmpm_ctx_init_comm(self._h, C.c_int(rank), C.c_int(nranks), buf))
        self.rank, self.nranks = rank, nranks

    def set_local_slabs(self, n):
        """Split each rank's share of decomposed subdomains into n slabs on this device."""
        _check(lib().osmpm_ctx_set_local_slabs(self._h, C.c_int(n)))

    def measure_fma_peak(self, precision=F64):
        """CUDA-core FMA throughput in TFLOP/s (osmpm_measure_fma_peak)."""
        t = C.c_double()
        _check(lib().osmpm_measure_fma_peak(self._h, C.c_int(precision), C.byref(t)))
        return t.value

    def launch_count(self):
        n = C.c_int64()
        _check(lib().osmpm_launch_count(self._h, C.byref(n)))
        return n.value

    def close(self):
        if self._h:
            # couplers before subdomains before the context they live on
            kids = [k() for k in self._children]
            for k in sorted((k for k in kids if k is not None), key=lambda o: not isinstance(o, Coupler)):
                k.close()
            self._children = []
            lib().osmpm_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def grid_desc(grid) -> GridDesc:
    g = GridDesc()
    g.dim = grid.dim
    for a in range(3):
        g.origin[a] = grid.origin[a]
        g.dims[a] = grid.dims[a] if a < grid.dim else 1
    g.dx = grid.dx
    return g


class Subdomain:
    """One MPM subdomain (§3.1) living on the context's GPU."""

    def __init__(self, ctx: Context, grid, dt, particles, materials, gravity=(0.0, 0.0, 0.0), precision=F64,
                 decompose=True):
        """decompose: split into x-slabs over the ctx's process group / local slabs (if any)."""
        self.ctx = ctx
        ctx._children.append(weakref.ref(self))
        self.grid = grid
        self.dim = grid.dim
        self._h = C.c_void_p()
        pt = particles
        self._keep = []
        arrays = [pt.x, pt.v, pt.F, pt.B, pt.m, pt.V0]
        ptrs = []
        sp = HOST
        for a in arrays:
            if isinstance(a, np.ndarray):
                a = np.ascontiguousarray(a, dtype=np.float64)
            self._keep.append(a)
            p, s = _ptr(a)
            sp = s
            ptrs.append(p)
        mat = np.ascontiguousarray(pt.mat, dtype=np.int32) if isinstance(pt.mat, np.ndarray) else pt.mat
        bnd = np.ascontiguousarray(pt.boundary, dtype=np.uint8) if isinstance(pt.boundary, np.ndarray) else pt.boundary
        self._keep += [mat, bnd]
        pm, _ = _ptr(mat, np.int32)
        pb, _ = _ptr(bnd, np.uint8)
        n = pt.x.shape[0]
        view = ParticlesView(n, sp, *ptrs, pm, pb)
        mats = (Material * len(materials))(*[Material(float(E), float(nu)) for (E, nu) in materials])
        gvec = (C.c_double * 3)(*[float(g) for g in gravity[:3]])
        gd = grid_desc(grid)
        _check(lib().osmpm_subdomain_create_ex(ctx._h, C.byref(gd), C.c_double(dt), C.byref(view), mats,
                                               C.c_int32(len(materials)), gvec, C.c_int(precision),
                                               C.c_int32(1 if decompose else 0), C.byref(self._h)))
        self._keep = []
        self.n = n
        self.n_nodes = int(np.prod(grid.dims[: grid.dim]))

    # --- configuration -----------------------------------------------------------------------
    def set_gravity(self, g):
        _check(lib().osmpm_set_gravity(self._h, (C.c_double * 3)(*[float(x) for x in g[:3]])))

    def set_dt(self, dt):
        _check(lib().osmpm_set_dt(self._h, C.c_double(dt)))

    def set_particles(self, x=None, v=None, F=None, B=None):
        ps = [_ptr(a)[0] if a is not None else None for a in (x, v, F, B)]
        _check(lib().osmpm_set_particles(self._h, *ps, C.c_int(_space(x, v, F, B))))

    def set_dirichlet(self, node_idx, comp_mask, vel):
        node_idx = np.ascontiguousarray(node_idx, dtype=np.int64)
        comp_mask = np.ascontiguousarray(comp_mask, dtype=np.uint8)
        vel = np.ascontiguousarray(vel, dtype=np.float64)
        _check(lib().osmpm_set_dirichlet(self._h, C.c_int64(node_idx.shape[0]), _ptr(node_idx, np.int64)[0],
                                         _ptr(comp_mask, np.uint8)[0], _ptr(vel)[0], C.c_int(HOST)))

    def set_dirichlet_device(self, node_idx, comp_mask, vel):
        """Dirichlet list from torch CUDA tensors (int64, uint8, float64 (n, d))."""
        _check(lib().osmpm_set_dirichlet(self._h, C.c_int64(int(node_idx.shape[0])), _ptr(node_idx, np.int64)[0],
                                         _ptr(comp_mask, np.uint8)[0], _ptr(vel)[0], C.c_int(DEVICE)))

    # --- hot path ------------------------------------------------------------------------------
    def p2g(self):
        _check(lib().osmpm_p2g(self._h))

    def read_grid(self, device=None):
        d = self.dim
        nn = self.n_nodes
        m = _empty_like_space((nn,), np.float64, device)
        p = _empty_like_space((nn, d), np.float64, device)
        v = _empty_like_space((nn, d), np.float64, device)
        fe = _empty_like_space((nn, d), np.float64, device)
        fs = _empty_like_space((nn, d), np.float64, device)
        act = _empty_like_space((nn,), np.uint8, device)
        sp = HOST if device is None else DEVICE
        _check(lib().osmpm_read_grid(self._h, _ptr(m)[0], _ptr(p)[0], _ptr(v)[0], _ptr(fe)[0], _ptr(fs)[0],
                                     _ptr(act, np.uint8)[0], C.c_int(sp)))
        return dict(m=m, p=p, v=v, fext=fe, fsig=fs, active=act)

    def newton_gradient(self, u):
        g = _empty_like_space(tuple(u.shape), np.float64, None if not _is_torch(u) else u.device)
        E = C.c_double()
        up, sp = _ptr(u)
        _check(lib().osmpm_newton_gradient(self._h, up, _ptr(g)[0], C.byref(E), C.c_int(sp)))
        return g, E.value

    def newton_hvp(self, dvec, out=None):
        y = out if out is not None else _empty_like_space(tuple(dvec.shape), np.float64,
                                                          None if not _is_torch(dvec) else dvec.device)
        dp, sp = _ptr(dvec)
        _check(lib().osmpm_newton_hvp(self._h, dp, _ptr(y)[0], C.c_int(sp)))
        return y

    def newton_diag(self, device=None):
        out = _empty_like_space((self.n_nodes, self.dim), np.float64, device)
        _check(lib().osmpm_newton_diag(self._h, _ptr(out)[0], C.c_int(HOST if device is None else DEVICE)))
        return out

    def implicit_solve(self, settings=None, raise_on_error=True) -> SolveStats:
        st = SolveStats()
        rc = lib().osmpm_implicit_solve(self._h, C.byref(settings or newton_settings()), C.byref(st))
        if raise_on_error:
            _check(rc)
        return st

    def read_grid_velocity(self, device=None):
        out = _empty_like_space((self.n_nodes, self.dim), np.float64, device)
        _check(lib().osmpm_read_grid_velocity(self._h, _ptr(out)[0], C.c_int(HOST if device is None else DEVICE)))
        return out

    def set_grid_velocity(self, v):
        vp, sp = _ptr(v)
        _check(lib().osmpm_set_grid_velocity(self._h, vp, C.c_int(sp)))

    def g2p(self):
        _check(lib().osmpm_g2p(self._h))

    def read_particles(self, device=None, fields=("x", "v", "F", "B")):
        d = self.dim
        n = self.n
        shapes = dict(x=(n, d), v=(n, d), F=(n, d, d), B=(n, d, d))
        out = {k: _empty_like_space(shapes[k], np.float64, device) for k in fields}
        ps = [(_ptr(out[k])[0] if k in out else None) for k in ("x", "v", "F", "B")]
        _check(lib().osmpm_read_particles(self._h, *ps, C.c_int(HOST if device is None else DEVICE)))
        return out

    def read_particles_into(self, x=None, v=None, F=None, B=None):
        """Creation-order particle fields into caller buffers (numpy / pinned or CUDA torch tensors)."""
        ps = [_ptr(a)[0] if a is not None else None for a in (x, v, F, B)]
        _check(lib().osmpm_read_particles(self._h, *ps, C.c_int(_space(x, v, F, B))))

    def info(self):
        n = C.c_int64()
        lo = (C.c_int64 * 3)()
        dims = (C.c_int64 * 3)()
        _check(lib().osmpm_subdomain_info(self._h, C.byref(n), lo, dims))
        return n.value, tuple(lo), tuple(dims)

    def sync(self):
        _check(lib().osmpm_sync(self._h))

    def checkpoint(self):
        _check(lib().osmpm_checkpoint(self._h))

    def restore(self):
        _check(lib().osmpm_restore(self._h))

    def decomp(self):
        """(slabs_total, slabs_local, first_slab, n_local_particles, cuts)"""
        st, sl, fs = C.c_int32(), C.c_int32(), C.c_int32()
        nl = C.c_int64()
        cuts = (C.c_int32 * 4096)()
        _check(lib().osmpm_subdomain_decomp(self._h, C.byref(st), C.byref(sl), C.byref(fs), C.byref(nl), cuts))
        return st.value, sl.value, fs.value, nl.value, [cuts[k] for k in range(st.value - 1)]

    def close(self):
        if self._h:
            if self.ctx._h:
                lib().osmpm_subdomain_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def transmit(src: Subdomain, dst: Subdomain, direction, alpha=0.0, eps_tol=0.0, targets=None, device=None):
    """Pi (FINE_TO_COARSE) or I+T (COARSE_TO_FINE) onto `targets` (dst dense node indices)."""
    d = src.dim
    if targets is None:
        nt = dst.n_nodes
        tp = None
    else:
        targets = np.ascontiguousarray(targets, dtype=np.int64) if isinstance(targets, np.ndarray) else targets
        nt = int(targets.shape[0])
        tp = _ptr(targets, np.int64)[0]
    out = _empty_like_space((nt, d), np.float64, device)
    sp = HOST if device is None else DEVICE
    if targets is not None and _is_torch(targets) != (device is not None):
        raise ValueError("targets and output must share a memory space")
    _check(lib().osmpm_transmit(src._h, dst._h, C.c_int(direction), C.c_double(alpha), C.c_double(eps_tol),
                                C.c_int64(nt), tp, _ptr(out)[0], C.c_int(sp)))
    return out


class Coupler:
    """Schwarz coupler of a coarse and a fine subdomain (Alg. 1)."""

    def __init__(self, coarse: Subdomain, fine: Subdomain, settings: SchwarzSettings):
        self._h = C.c_void_p()
        self.coarse, self.fine = coarse, fine
        fine.ctx._children.append(weakref.ref(self))
        _check(lib().osmpm_coupler_create(coarse._h, fine._h, C.byref(settings), C.byref(self._h)))

    def prepare(self):
        _check(lib().osmpm_schwarz_prepare(self._h))

    def substep(self, m):
        st = SolveStats()
        _check(lib().osmpm_schwarz_substep(self._h, C.c_int32(m), C.byref(st)))
        return st

    def step(self) -> SchwarzReport:
        rep = SchwarzReport()
        _check(lib().osmpm_schwarz_step(self._h, C.byref(rep)))
        return rep

    def close(self):
        if self._h:
            if self.fine._h and self.coarse._h:
                lib().osmpm_coupler_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def schwarz_settings(eps_conv=1e-5, eps_tol=-1.0, tau_gamma_rel=1e-6, k_max=100, M=1, parity_fixed_k=0,
                     coarse=None, fine=None) -> SchwarzSettings:
    return SchwarzSettings(eps_conv, eps_tol, tau_gamma_rel, k_max, M, parity_fixed_k,
                           coarse or newton_settings(), fine or newton_settings())
