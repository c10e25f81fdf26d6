"""TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.

ctypes bindings of the CPU checkers:
  * Oracle3D — oracle/build/liboracle3d.so, the 3D restatement (oracle/sdg3d.cpp)
  * Ref2D    — oracle/_ref/libsdg_ref.so, the unmodified reference library
               (/root/reference/proj/src) behind oracle/ref_harness.cpp

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2008_04356_b200 import types as T

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle3d.so")
REF_SO = os.path.join(HERE, "_ref", "libsdg_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lp = C.POINTER(C.c_long)


def _d(a):
    return a.ctypes.data_as(_dp)


def build(ref: bool = True) -> None:
    """Compiles the oracle (and the reference, when /root/reference is present)."""
    target = "all" if ref else "oracle"
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


_oracle_lib = None
_ref_lib = None


def oracle_lib():
    global _oracle_lib
    if _oracle_lib is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        lib = C.CDLL(ORACLE_SO)
        vp = C.c_void_p
        lib.orc_create.argtypes = [C.POINTER(T.MeshSpec), C.POINTER(T.SolverConfig), C.POINTER(vp)]
        lib.orc_destroy.argtypes = [vp]
        lib.orc_last_error.argtypes = [vp]
        lib.orc_last_error.restype = C.c_char_p
        lib.orc_global_error.restype = C.c_char_p
        lib.orc_n_elements.argtypes = [vp]
        lib.orc_n_elements.restype = C.c_long
        lib.orc_n1.argtypes = [vp]
        lib.orc_n_contexts.argtypes = [vp]
        lib.orc_set_initial_condition.argtypes = [vp, C.c_double]
        lib.orc_set_state.argtypes = [vp, _dp]
        lib.orc_get_state.argtypes = [vp, _dp]
        lib.orc_get_register.argtypes = [vp, _dp]
        lib.orc_compute_residual.argtypes = [vp, C.c_double, _dp, _dp]
        lib.orc_compute_gradients.argtypes = [vp, C.c_double, _dp, _dp]
        lib.orc_step.argtypes = [vp, C.c_double]
        lib.orc_steps.argtypes = [vp, C.c_double, C.c_int]
        lib.orc_suggest_dt.argtypes = [vp, C.c_double, _dp]
        lib.orc_time.argtypes = [vp]
        lib.orc_time.restype = C.c_double
        lib.orc_total_rebuilds.argtypes = [vp]
        lib.orc_total_rebuilds.restype = C.c_long
        lib.orc_ctx_info.argtypes = [vp, C.c_int, _lp, _dp, _dp]
        lib.orc_get_pairing.argtypes = [vp, C.c_int, _ip, _ip]
        lib.orc_get_mapping.argtypes = [vp, C.c_int, _ip]
        lib.orc_integrate_mass_energy.argtypes = [vp, _dp, _dp]
        lib.orc_sample_case.argtypes = [vp, C.c_double, _dp]
        lib.orc_nodes.argtypes = [C.c_int, C.c_int, _dp, _dp]
        lib.orc_basis.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp]
        lib.orc_mortar_ops.argtypes = [C.c_int, C.c_int, C.c_double, _dp, _dp]
        lib.orc_subrange_ops.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, _dp, _dp]
        lib.orc_mortar_intervals.argtypes = [C.c_long, C.c_long, C.c_double, C.c_double, _lp, _lp, _dp]
        lib.orc_displacement.argtypes = [C.c_double, C.c_double, C.c_long, _dp, _lp, _dp]
        lib.orc_moving_index.argtypes = [C.c_long, C.c_long, C.c_int, C.c_long]
        lib.orc_moving_index.restype = C.c_long
        lib.orc_static_index.argtypes = [C.c_long, C.c_long, C.c_int, C.c_long]
        lib.orc_static_index.restype = C.c_long
        lib.orc_pairing.argtypes = [C.c_int, _lp, C.c_long, C.c_long, _ip, C.c_long, C.c_int, C.c_int, C.c_int,
                                    _ip, _ip, _ip, _lp, _ip, _ip, _ip]
        lib.orc_face_flux.argtypes = [C.POINTER(T.Gas), _dp, _dp, C.c_int, C.c_double, _dp, _dp, _dp]
        lib.orc_set_threads.argtypes = [C.c_int]
        lib.orc_n_nc_interfaces.argtypes = [vp]
        lib.orc_nc_rows.argtypes = [vp, C.c_int, C.c_int, _lp, _lp, _dp, _dp]
        _oracle_lib = lib
    return _oracle_lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref_lib
    if _ref_lib is None:
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_field_size.argtypes = [C.c_void_p]
        lib.ref_field_size.restype = C.c_long
        lib.ref_single_rank.argtypes = [C.c_void_p, C.c_double, _dp, C.c_int, C.c_double, C.c_double, C.c_int,
                                        _dp, _dp]
        lib.ref_run.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_int, C.c_int, _dp, _dp]
        lib.ref_run_case.argtypes = [C.c_char_p, _dp]
        lib.ref_convergence.argtypes = [C.c_char_p, _dp, _ip]
        lib.ref_nodes.argtypes = [C.c_int, C.c_int, _dp, _dp]
        lib.ref_basis.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp]
        lib.ref_mortar_ops.argtypes = [C.c_int, C.c_int, C.c_double, _dp, _dp]
        lib.ref_displacement.argtypes = [C.c_double, C.c_double, C.c_long, _dp, _lp, _dp]
        lib.ref_moving_index.argtypes = [C.c_long, C.c_long, C.c_int, C.c_long]
        lib.ref_moving_index.restype = C.c_long
        lib.ref_static_index.argtypes = [C.c_long, C.c_long, C.c_int, C.c_long]
        lib.ref_static_index.restype = C.c_long
        lib.ref_pairing.argtypes = [C.c_int, _lp, C.c_long, C.c_long, _ip, C.c_long, C.c_int, C.c_int, C.c_int,
                                    _ip, _ip, _ip, _lp, _ip, _ip, _ip]
        lib.ref_ctx_state.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_int, C.c_int, _lp, _dp, _ip, _ip]
        lib.ref_face_flux.argtypes = [C.c_double] * 4 + [_dp, _dp, C.c_int, C.c_double, _dp, _dp, _dp]
        _ref_lib = lib
    return _ref_lib


class Oracle3D:
    """Single-rank 3D restatement; field layout U[e][i][j][k][5], gid order."""

    def __init__(self, mesh: T.MeshSpec, cfg: T.SolverConfig):
        self.lib = oracle_lib()
        h = C.c_void_p()
        code = self.lib.orc_create(C.byref(mesh), C.byref(cfg), C.byref(h))
        T.raise_for(code, self.lib.orc_global_error().decode())
        self.h = h
        self.n1 = self.lib.orc_n1(h)
        self.n_elements = self.lib.orc_n_elements(h)
        self.size = self.n_elements * self.n1 ** 3 * T.NVARS
        self.widths = (13, 6) if mesh.mapping == T.MAP_ANNULUS else (10, 4)  # metric doubles per node / face node

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.orc_destroy(self.h)
            self.h = None

    def _check(self, code):
        T.raise_for(code, self.lib.orc_last_error(self.h).decode())

    def set_initial_condition(self, t0=0.0):
        self._check(self.lib.orc_set_initial_condition(self.h, t0))

    def field(self):
        u = np.empty(self.size)
        self._check(self.lib.orc_get_state(self.h, _d(u)))
        return u

    def register(self):
        r = np.empty(self.size)
        self._check(self.lib.orc_get_register(self.h, _d(r)))
        return r

    def set_state(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        assert u.size == self.size
        self._check(self.lib.orc_set_state(self.h, _d(u)))

    def compute_residual(self, t_stage, u=None):
        u = self.field() if u is None else np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros(self.size)
        self._check(self.lib.orc_compute_residual(self.h, t_stage, _d(u), _d(out)))
        return out

    def compute_gradients(self, t_stage, u=None):
        u = self.field() if u is None else np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros(self.n_elements * self.n1 ** 3 * T.NGRAD)
        self._check(self.lib.orc_compute_gradients(self.h, t_stage, _d(u), _d(out)))
        return out

    def step(self, dt, n=1):
        self._check(self.lib.orc_steps(self.h, dt, n))

    def suggest_dt(self, cfl):
        dt = C.c_double()
        self._check(self.lib.orc_suggest_dt(self.h, cfl, C.byref(dt)))
        return dt.value

    def time(self):
        return self.lib.orc_time(self.h)

    def total_rebuilds(self):
        return self.lib.orc_total_rebuilds(self.h)

    def n_contexts(self):
        return self.lib.orc_n_contexts(self.h)

    def ctx_info(self, ctx):
        o = (C.c_long * 5)()
        sd, sg = C.c_double(), C.c_double()
        self._check(self.lib.orc_ctx_info(self.h, ctx, o, C.byref(sd), C.byref(sg)))
        return dict(iface=o[0], on_static=bool(o[1]), n_delta=o[2], conforming=bool(o[3]), n_faces=o[4],
                    s_delta=sd.value, sigma_side=sg.value)

    def n_nc_interfaces(self):
        return self.lib.orc_n_nc_interfaces(self.h)

    def nc_rows(self, iface, direction):
        """Rows of a non-matching interface at the last residual: faces, ranges, displacement."""
        n, d = C.c_long(), C.c_double()
        self._check(self.lib.orc_nc_rows(self.h, iface, direction, C.byref(n), None, None, C.byref(d)))
        faces = np.zeros((n.value, 2), dtype=np.int64)
        ranges = np.zeros((n.value, 4))
        self._check(self.lib.orc_nc_rows(self.h, iface, direction, C.byref(n), faces.ctypes.data_as(_lp), _d(ranges),
                                         C.byref(d)))
        return faces, ranges, d.value

    def pairing(self, role):
        nc = C.c_int()
        self._check(self.lib.orc_get_pairing(self.h, role, C.byref(nc), None))
        cols = np.zeros((max(nc.value, 1), T.TUPLE_INTS), dtype=np.int32)
        self._check(self.lib.orc_get_pairing(self.h, role, C.byref(nc), cols.ctypes.data_as(_ip)))
        return cols[: nc.value]

    def mapping(self, ctx):
        nf = self.ctx_info(ctx)["n_faces"]
        m = np.zeros((2, nf), dtype=np.int32)
        self._check(self.lib.orc_get_mapping(self.h, ctx, m.ctypes.data_as(_ip)))
        return m

    def mass_energy(self, u=None):
        u = self.field() if u is None else np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros(2)
        self._check(self.lib.orc_integrate_mass_energy(self.h, _d(u), _d(out)))
        return out

    def metrics(self):
        """(met [E, N3, 10], fmet [E, 6, N2, 4]) of a curved (SDG_MAP_WARP) mesh."""
        n1 = self.n1
        mw, fw = self.widths
        met = np.zeros((self.n_elements, n1 ** 3, mw))
        fmet = np.zeros((self.n_elements, 6, n1 * n1, fw))
        self.lib.orc_get_metrics.argtypes = [C.c_void_p, _dp, _dp]
        self._check(self.lib.orc_get_metrics(self.h, _d(met), _d(fmet)))
        return met, fmet

    def sample_case(self, t):
        out = np.zeros(self.size)
        self._check(self.lib.orc_sample_case(self.h, t, _d(out)))
        return out


def _pairing_call(fn, faces, n_par, n_perp, ranks, n_delta, on_static, conforming, self_rank):
    faces = np.ascontiguousarray(faces, dtype=np.int64).reshape(-1, 3)
    ranks = np.ascontiguousarray(ranks, dtype=np.int32).reshape(-1)
    nl = faces.shape[0]
    cols = np.zeros((2 * nl + 1, T.TUPLE_INTS), dtype=np.int32)
    lo_hi = (faces[:, 0].max() - faces[:, 0].min() + 1) if nl else 1
    m = np.zeros(2 * lo_hi, dtype=np.int32)
    ncols, nsched = C.c_int(), C.c_int()
    face_lo = C.c_long()
    sched = np.zeros(3 * (2 * nl + 1), dtype=np.int32)
    self_e = np.zeros(3, dtype=np.int32)
    code = fn(nl, faces.ctypes.data_as(_lp), n_par, n_perp, ranks.ctypes.data_as(_ip), n_delta, int(on_static),
              int(conforming), self_rank, C.byref(ncols), cols.ctypes.data_as(_ip), m.ctypes.data_as(_ip),
              C.byref(face_lo), C.byref(nsched), sched.ctypes.data_as(_ip), self_e.ctypes.data_as(_ip))
    return code, dict(cols=cols[: ncols.value], m=m.reshape(2, -1), face_lo=face_lo.value,
                      sched=sched[: 3 * nsched.value].reshape(-1, 3), self_entry=self_e)


def oracle_pairing(*args):
    lib = oracle_lib()
    code, out = _pairing_call(lib.orc_pairing, *args)
    T.raise_for(code, lib.orc_global_error().decode())
    return out


def ref_pairing(*args):
    lib = ref_lib()
    code, out = _pairing_call(lib.ref_pairing, *args)
    T.raise_for(code, lib.ref_last_error().decode())
    return out


def oracle_mortar_ops(degree, kind, sigma):
    n = degree + 1
    f, b = np.zeros((2, n, n)), np.zeros((2, n, n))
    T.raise_for(oracle_lib().orc_mortar_ops(degree, kind, sigma, _d(f), _d(b)), oracle_lib().orc_global_error().decode())
    return f, b


def subrange_ops(degree, kind, lo, hi):
    """Mortar operators of the face sub-range [lo, hi] (non-matching interfaces)."""
    n = degree + 1
    f, b = np.zeros((n, n)), np.zeros((n, n))
    T.raise_for(oracle_lib().orc_subrange_ops(degree, kind, lo, hi, _d(f), _d(b)), oracle_lib().orc_global_error().decode())
    return f, b


def mortar_intervals(n_a, n_b, l_a, delta):
    """Mortars of a non-matching periodic face row: faces [M, 2], ranges [M, 4]."""
    L = oracle_lib()
    n = C.c_long()
    T.raise_for(L.orc_mortar_intervals(n_a, n_b, l_a, delta, C.byref(n), None, None), L.orc_global_error().decode())
    faces = np.zeros((n.value, 2), dtype=np.int64)
    ranges = np.zeros((n.value, 4))
    T.raise_for(L.orc_mortar_intervals(n_a, n_b, l_a, delta, C.byref(n), faces.ctypes.data_as(_lp), _d(ranges)),
                L.orc_global_error().decode())
    return faces, ranges


def ref_mortar_ops(degree, kind, sigma):
    n = degree + 1
    f, b = np.zeros((2, n, n)), np.zeros((2, n, n))
    T.raise_for(ref_lib().ref_mortar_ops(degree, kind, sigma, _d(f), _d(b)), ref_lib().ref_last_error().decode())
    return f, b


def oracle_displacement(delta, l_par, n_faces):
    d, nd, sd = C.c_double(), C.c_long(), C.c_double()
    oracle_lib().orc_displacement(delta, l_par, n_faces, C.byref(d), C.byref(nd), C.byref(sd))
    return d.value, nd.value, sd.value


def ref_displacement(delta, l_par, n_faces):
    d, nd, sd = C.c_double(), C.c_long(), C.c_double()
    ref_lib().ref_displacement(delta, l_par, n_faces, C.byref(d), C.byref(nd), C.byref(sd))
    return d.value, nd.value, sd.value


class RefSpec(C.Structure):
    """Mirror of ref_spec in oracle/ref_harness.cpp (2D problem)."""
    _fields_ = [
        ("width", C.c_double), ("height", C.c_double), ("ny", C.c_int), ("n_bands", C.c_int),
        ("band_nx", C.c_int * 16), ("band_frac", C.c_double * 16), ("band_vg", C.c_double * 16),
        ("periodic_x", C.c_int), ("periodic_y", C.c_int),
        ("degree", C.c_int), ("node_kind", C.c_int),
        ("gamma", C.c_double), ("R", C.c_double), ("mu", C.c_double), ("Pr", C.c_double),
        ("case_kind", C.c_int), ("fs", C.c_double * 4), ("dw", C.c_double * 4), ("vx", C.c_double * 8),
    ]


def ref_spec(bands, ny, degree, node_kind=T.NODES_GAUSS, width=2.0, height=2.0, periodic=(True, True),
             gamma=1.4, R=1.0, mu=0.0, Pr=0.72, case="density_wave", fs=(1.0, 1.0, 0.5, 1.0),
             dw=(0.1, 1.0, 1.0, 1.0), vx=None) -> RefSpec:
    s = RefSpec()
    s.width, s.height, s.ny, s.n_bands = width, height, ny, len(bands)
    for i, (nx, frac, vg) in enumerate(bands):
        s.band_nx[i], s.band_frac[i], s.band_vg[i] = nx, frac, vg
    s.periodic_x, s.periodic_y = int(periodic[0]), int(periodic[1])
    s.degree, s.node_kind = degree, node_kind
    s.gamma, s.R, s.mu, s.Pr = gamma, R, mu, Pr
    s.case_kind = {"freestream": 0, "density_wave": 1, "vortex": 2}[case]
    for i in range(4):
        s.fs[i], s.dw[i] = fs[i], dw[i]
    if vx is not None:
        for i in range(8):
            s.vx[i] = vx[i]
    return s


class Ref2D:
    """The unmodified reference (2D) through oracle/ref_harness.cpp."""

    def __init__(self, spec: RefSpec):
        self.lib = ref_lib()
        self.spec = spec
        self.size = self.lib.ref_field_size(C.byref(spec))

    def _check(self, code):
        T.raise_for(code, self.lib.ref_last_error().decode())

    def residual(self, t0, t_stage, u=None):
        out = np.zeros(self.size)
        up = _d(np.ascontiguousarray(u, dtype=np.float64)) if u is not None else None
        self._check(self.lib.ref_single_rank(C.byref(self.spec), t0, up, 0, t_stage, 0.0, 0, _d(out), None))
        return out

    def gradients(self, t0, t_stage, u=None):
        out = np.zeros(self.size // 4 * 6)
        up = _d(np.ascontiguousarray(u, dtype=np.float64)) if u is not None else None
        self._check(self.lib.ref_single_rank(C.byref(self.spec), t0, up, 1, t_stage, 0.0, 0, _d(out), None))
        return out

    def steps(self, t0, dt, n, u=None):
        out = np.zeros(self.size)
        aux = np.zeros(2)
        up = _d(np.ascontiguousarray(u, dtype=np.float64)) if u is not None else None
        self._check(self.lib.ref_single_rank(C.byref(self.spec), t0, up, 2, 0.0, dt, n, _d(out), _d(aux)))
        return out, aux[0], int(aux[1])

    def initial(self, t0):
        return self.steps(t0, 0.0, 0)[0]

    def suggest_dt(self, cfl, t0=0.0):
        aux = np.zeros(2)
        self._check(self.lib.ref_single_rank(C.byref(self.spec), t0, None, 3, cfl, 0.0, 0, _d(np.zeros(1)), _d(aux)))
        return aux[0]

    def run(self, dt, n_steps, ranks=1, backend=0):
        out = np.zeros(self.size)
        wall = C.c_double()
        self._check(self.lib.ref_run(C.byref(self.spec), dt, n_steps, ranks, backend, _d(out), C.byref(wall)))
        return out, wall.value
