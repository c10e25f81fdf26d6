"""ctypes binding of the C-ABI (include/sdg_gpu.h) and a Python mirror of the
reference's per-rank solver interface (`sdg::RankSolver`,
/root/reference/proj/src/solver.hpp:64-98), so tests read like the
reference's own (proj/tests/test_solver.cpp).

There is no CPU fallback: loading fails loudly when the CUDA library is
missing, and every call goes to the device.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import types as T

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SDG_GPU_LIB", os.path.join(HERE, "libsdg_gpu.so"))

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lp = C.POINTER(C.c_long)
_vp = C.c_void_p

_lib = None


def build() -> None:
    """Compiles csrc/ for sm_100a into libsdg_gpu.so (nvcc cross-compiles without a GPU)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "csrc")], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA extension missing: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        L.sdg_create.argtypes = [C.POINTER(T.MeshSpec), C.POINTER(T.SolverConfig), C.c_int, C.c_int, C.c_int,
                                 C.c_void_p, C.POINTER(_vp)]
        L.sdg_create_inproc.argtypes = [C.POINTER(T.MeshSpec), C.POINTER(T.SolverConfig), C.c_int, C.c_int,
                                        C.c_int, C.c_char_p, C.POINTER(_vp)]
        L.sdg_destroy.argtypes = [_vp]
        L.sdg_last_error.argtypes = [_vp]
        L.sdg_last_error.restype = C.c_char_p
        L.sdg_global_error.restype = C.c_char_p
        L.sdg_nccl_unique_id.argtypes = [C.c_void_p]
        L.sdg_nccl_selfcheck.argtypes = [C.c_int, C.c_long]
        L.sdg_init_rank_maps.argtypes = [_vp]
        L.sdg_set_initial_condition.argtypes = [_vp, C.c_double]
        L.sdg_n1.argtypes = [_vp]
        L.sdg_n_local_elements.argtypes = [_vp]
        L.sdg_n_local_elements.restype = C.c_long
        L.sdg_n_global_elements.argtypes = [_vp]
        L.sdg_n_global_elements.restype = C.c_long
        L.sdg_local_element_ids.argtypes = [_vp, _lp]
        L.sdg_set_state.argtypes = [_vp, _dp]
        L.sdg_get_state.argtypes = [_vp, _dp]
        L.sdg_get_register.argtypes = [_vp, _dp]
        L.sdg_state_device_ptr.argtypes = [_vp, C.POINTER(_dp)]
        L.sdg_step.argtypes = [_vp, C.c_double]
        L.sdg_steps.argtypes = [_vp, C.c_double, C.c_int]
        L.sdg_steps_async.argtypes = [_vp, C.c_double, C.c_int]
        L.sdg_synchronize.argtypes = [_vp]
        L.sdg_rk_stage.argtypes = [_vp, C.c_int, C.c_double, C.c_double]
        L.sdg_rk_coefficients.argtypes = [_dp, _dp, _dp]
        L.sdg_update_interfaces.argtypes = [_vp, C.c_double, _dp]
        L.sdg_compute_residual.argtypes = [_vp, C.c_double, C.c_void_p, C.c_void_p]
        L.sdg_compute_residual_host.argtypes = [_vp, C.c_double, _dp, _dp]
        L.sdg_compute_gradients_host.argtypes = [_vp, C.c_double, _dp, _dp]
        L.sdg_suggest_dt.argtypes = [_vp, C.c_double, _dp]
        L.sdg_time.argtypes = [_vp, _dp, _ip]
        L.sdg_total_rebuilds.argtypes = [_vp]
        L.sdg_total_rebuilds.restype = C.c_long
        L.sdg_n_contexts.argtypes = [_vp]
        L.sdg_ctx_info.argtypes = [_vp, C.c_int, _lp, _dp, _dp]
        L.sdg_get_pairing.argtypes = [_vp, C.c_int, _ip, _ip]
        L.sdg_n_nc_interfaces.argtypes = [_vp]
        L.sdg_nc_rows.argtypes = [_vp, C.c_int, C.c_int, _lp, _lp, _dp, _dp]
        L.sdg_get_mapping.argtypes = [_vp, C.c_int, _ip]
        L.sdg_pairing_device.argtypes = [C.c_int, _lp, C.c_long, C.c_long, _ip, C.c_long, C.c_int, C.c_int,
                                         C.c_int, _ip, _ip, _ip, _lp, _ip, _ip, _ip]
        L.sdg_plan_json.argtypes = [C.POINTER(T.MeshSpec), C.c_int, C.c_int, C.c_double, C.c_char_p, C.c_long, _lp]
        L.sdg_metrics_host.argtypes = [C.POINTER(T.MeshSpec), C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, _lp]
        L.sdg_subrange_ops.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, _dp, _dp]
        L.sdg_mortar_intervals.argtypes = [C.c_long, C.c_long, C.c_double, C.c_double, _lp, _lp, _dp]
        L.sdg_mortar_intervals_device.argtypes = [C.c_long, C.c_long, C.c_double, C.c_double, _lp, _lp, _dp]
        L.sdg_interface_project_device.argtypes = [C.c_int, C.c_int, _lp, _lp, C.c_double, C.c_double, C.c_double,
                                                   C.c_double, C.c_int, C.c_int, _dp, _dp, _dp, _lp]
        L.sdg_interface_flux_device.argtypes = [C.POINTER(T.Gas), C.c_int, C.c_int, _lp, _lp, C.c_double, C.c_double,
                                                C.c_double, C.c_double, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _lp]
        L.sdg_interface_lift_device.argtypes = [C.POINTER(T.Gas), C.c_int, C.c_int, _lp, _lp, C.c_double, C.c_double,
                                                C.c_double, C.c_double, _dp, _dp, _dp, _dp, _dp, _lp]
        L.sdg_diagnostics.argtypes = [_vp, C.c_double, C.c_int, _dp]
        L.sdg_write_snapshot.argtypes = [_vp, C.c_char_p, C.c_double]
        L.sdg_read_snapshot.argtypes = [_vp, C.c_char_p, _dp]
        L.sdg_trace_json.argtypes = [_vp, C.c_char_p, C.c_long, _lp]
        L.sdg_inject_collective.argtypes = [_vp]
        L.sdg_stream.argtypes = [_vp]
        L.sdg_stream.restype = C.c_void_p
        L.sdg_kernel_launches.argtypes = [_vp]
        L.sdg_kernel_launches.restype = C.c_long
        L.sdg_enable_kernel_timing.argtypes = [_vp, C.c_int]
        L.sdg_kernel_timing.argtypes = [_vp, C.c_char_p, C.c_int, _dp, _lp, C.c_int, _ip]
        _lib = L
    return _lib


EXPORTED = [
    "sdg_create", "sdg_create_inproc", "sdg_destroy", "sdg_last_error", "sdg_global_error", "sdg_nccl_unique_id", "sdg_nccl_selfcheck", "sdg_init_rank_maps",
    "sdg_set_initial_condition", "sdg_n1", "sdg_n_local_elements", "sdg_n_global_elements",
    "sdg_local_element_ids", "sdg_set_state", "sdg_get_state", "sdg_get_register", "sdg_state_device_ptr",
    "sdg_step", "sdg_steps", "sdg_steps_async", "sdg_synchronize", "sdg_rk_stage", "sdg_rk_coefficients",
    "sdg_update_interfaces", "sdg_compute_residual",
    "sdg_compute_residual_host", "sdg_compute_gradients_host", "sdg_suggest_dt", "sdg_time",
    "sdg_total_rebuilds", "sdg_n_contexts", "sdg_ctx_info", "sdg_get_pairing", "sdg_get_mapping",
    "sdg_n_nc_interfaces", "sdg_nc_rows",
    "sdg_pairing_device", "sdg_plan_json", "sdg_metrics_host", "sdg_subrange_ops",
    "sdg_mortar_intervals", "sdg_mortar_intervals_device",
    "sdg_interface_project_device", "sdg_interface_flux_device", "sdg_interface_lift_device",
    "sdg_diagnostics", "sdg_write_snapshot", "sdg_read_snapshot",
    "sdg_trace_json", "sdg_inject_collective", "sdg_stream", "sdg_kernel_launches", "sdg_enable_kernel_timing", "sdg_kernel_timing",
]


def _d(a):
    return a.ctypes.data_as(_dp)


def rk_coefficients():
    """(a, b, c) of the 5-stage low-storage RK scheme (lsrk.cpp:7-29)."""
    a, b, c = np.zeros(5), np.zeros(5), np.zeros(5)
    lib().sdg_rk_coefficients(_d(a), _d(b), _d(c))
    return a, b, c


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    T.raise_for(lib().sdg_nccl_unique_id(buf), lib().sdg_global_error().decode())
    return buf.raw


def nccl_selfcheck(device: int = 0, n_doubles: int = 1 << 20) -> None:
    """Every NCCL call of the transport on a one-rank communicator (sdg_nccl_selfcheck)."""
    T.raise_for(lib().sdg_nccl_selfcheck(device, n_doubles), lib().sdg_global_error().decode())


class RankSolver:
    """One rank's share of the mesh on one GPU (mirror of sdg::RankSolver)."""

    def __init__(self, mesh: T.MeshSpec, cfg: T.SolverConfig, n_ranks: int = 1, rank: int = 0, device: int = 0,
                 nccl_id: bytes | None = None, init_rank_maps: bool = True, inproc_hub: str | None = None):
        self.lib = lib()
        h = _vp()
        if inproc_hub is not None:
            code = self.lib.sdg_create_inproc(C.byref(mesh), C.byref(cfg), n_ranks, rank, device,
                                              inproc_hub.encode(), C.byref(h))
        else:
            idp = C.create_string_buffer(nccl_id, 128) if nccl_id else None
            code = self.lib.sdg_create(C.byref(mesh), C.byref(cfg), n_ranks, rank, device, idp, C.byref(h))
        T.raise_for(code, self.lib.sdg_global_error().decode())
        self.h = h
        self.n1 = self.lib.sdg_n1(h)
        self.n_elements = self.lib.sdg_n_local_elements(h)
        self.size = self.n_elements * self.n1 ** 3 * T.NVARS
        if init_rank_maps:
            self.init_rank_maps()

    def close(self):
        if getattr(self, "h", None):
            self.lib.sdg_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def _check(self, code):
        T.raise_for(code, self.lib.sdg_last_error(self.h).decode())

    # --- reference interface -------------------------------------------------
    def init_rank_maps(self):
        self._check(self.lib.sdg_init_rank_maps(self.h))

    def set_initial_condition(self, t0: float = 0.0):
        self._check(self.lib.sdg_set_initial_condition(self.h, t0))

    def field(self) -> np.ndarray:
        u = np.empty(self.size)
        self._check(self.lib.sdg_get_state(self.h, _d(u)))
        return u

    def register(self) -> np.ndarray:
        r = np.empty(self.size)
        self._check(self.lib.sdg_get_register(self.h, _d(r)))
        return r

    def set_state(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        if u.size != self.size:
            raise T.ConfigError("state size mismatch")
        self._check(self.lib.sdg_set_state(self.h, _d(u)))

    def step(self, dt: float, n: int = 1):
        self._check(self.lib.sdg_steps(self.h, dt, n))

    def steps_async(self, dt: float, n: int):
        self._check(self.lib.sdg_steps_async(self.h, dt, n))

    def rk_stage(self, s: int, t: float, dt: float):
        """One stage of the low-storage RK step starting at t (lsrk_step, lsrk.hpp:20-21)."""
        self._check(self.lib.sdg_rk_stage(self.h, s, t, dt))

    def update_interfaces(self, t_stage: float) -> np.ndarray:
        """RankSolver::update_interfaces (solver.cpp:156-176); returns the per-context
        operators [ctx][fwd lower, fwd upper, bwd lower, bwd upper][n][n]."""
        n = self.lib.sdg_n1(self.h)
        ops = np.zeros((max(self.n_contexts(), 1), 4, n, n))
        self._check(self.lib.sdg_update_interfaces(self.h, t_stage, _d(ops)))
        return ops[: self.n_contexts()]

    def synchronize(self):
        self._check(self.lib.sdg_synchronize(self.h))

    def compute_residual(self, t_stage: float, u=None) -> np.ndarray:
        u = self.field() if u is None else np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros(self.size)
        self._check(self.lib.sdg_compute_residual_host(self.h, t_stage, _d(u), _d(out)))
        return out

    def compute_residual_device(self, t_stage: float, d_u: int, d_dudt: int):
        self._check(self.lib.sdg_compute_residual(self.h, t_stage, C.c_void_p(d_u), C.c_void_p(d_dudt)))

    def compute_gradients(self, t_stage: float, u=None) -> np.ndarray:
        u = self.field() if u is None else np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros(self.n_elements * self.n1 ** 3 * T.NGRAD)
        self._check(self.lib.sdg_compute_gradients_host(self.h, t_stage, _d(u), _d(out)))
        return out

    def suggest_dt(self, cfl: float) -> float:
        dt = C.c_double()
        self._check(self.lib.sdg_suggest_dt(self.h, cfl, C.byref(dt)))
        return dt.value

    def time(self) -> float:
        t = C.c_double()
        self.lib.sdg_time(self.h, C.byref(t), None)
        return t.value

    def step_index(self) -> int:
        s = C.c_int()
        self.lib.sdg_time(self.h, None, C.byref(s))
        return s.value

    def total_rebuilds(self) -> int:
        return self.lib.sdg_total_rebuilds(self.h)

    def n_contexts(self) -> int:
        return self.lib.sdg_n_contexts(self.h)

    def ctx_info(self, ctx: int) -> dict:
        o = (C.c_long * 5)()
        sd, sg = C.c_double(), C.c_double()
        self._check(self.lib.sdg_ctx_info(self.h, ctx, o, C.byref(sd), C.byref(sg)))
        return dict(iface=o[0], on_static=bool(o[1]), n_delta=o[2], conforming=bool(o[3]), n_faces=o[4],
                    s_delta=sd.value, sigma_side=sg.value)

    def n_nc_interfaces(self) -> int:
        return self.lib.sdg_n_nc_interfaces(self.h)

    def nc_rows(self, iface: int, direction: int):
        """Device rows of a non-matching interface at the last stage: faces [M, 2]
        (A face, B face), ranges [M, 4] (a_lo, a_hi, b_lo, b_hi), displacement."""
        n, d = C.c_long(), C.c_double()
        self._check(self.lib.sdg_nc_rows(self.h, iface, direction, C.byref(n), None, None, C.byref(d)))
        faces = np.zeros((n.value, 2), dtype=np.int64)
        ranges = np.zeros((n.value, 4))
        self._check(self.lib.sdg_nc_rows(self.h, iface, direction, C.byref(n), faces.ctypes.data_as(_lp), _d(ranges),
                                         C.byref(d)))
        return faces, ranges, d.value

    def pairing(self, role: int) -> np.ndarray:
        nc = C.c_int()
        self._check(self.lib.sdg_get_pairing(self.h, role, C.byref(nc), None))
        cols = np.zeros((max(nc.value, 1), T.TUPLE_INTS), dtype=np.int32)
        self._check(self.lib.sdg_get_pairing(self.h, role, C.byref(nc), cols.ctypes.data_as(_ip)))
        return cols[: nc.value]

    def mapping(self, ctx: int) -> np.ndarray:
        nf = self.ctx_info(ctx)["n_faces"]
        m = np.zeros((2, nf), dtype=np.int32)
        self._check(self.lib.sdg_get_mapping(self.h, ctx, m.ctypes.data_as(_ip)))
        return m

    def local_element_ids(self) -> np.ndarray:
        g = np.zeros(self.n_elements, dtype=np.int64)
        self.lib.sdg_local_element_ids(self.h, g.ctypes.data_as(_lp))
        return g

    def diagnostics(self, t: float, exact: bool = True) -> dict:
        """Device integrals and error norms (diagnostics.cpp:31-87)."""
        out = np.zeros(14)
        self._check(self.lib.sdg_diagnostics(self.h, t, int(exact), _d(out)))
        return dict(mass=out[0], energy=out[1], volume=out[2], l2=out[3:8].copy(), linf=out[8:13].copy(),
                    max_deviation=out[13])

    def write_snapshot(self, path: str, time: float | None = None):
        self._check(self.lib.sdg_write_snapshot(self.h, path.encode(), self.time() if time is None else time))

    def read_snapshot(self, path: str) -> float:
        t = C.c_double()
        self._check(self.lib.sdg_read_snapshot(self.h, path.encode(), C.byref(t)))
        return t.value

    def trace(self) -> dict:
        """Communication trace of this rank (TraceRow, transport.hpp:28-37)."""
        import json
        n = C.c_long()
        self._check(self.lib.sdg_trace_json(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        self._check(self.lib.sdg_trace_json(self.h, buf, n.value + 1, C.byref(n)))
        return json.loads(buf.value.decode())

    def inject_collective(self):
        self._check(self.lib.sdg_inject_collective(self.h))

    # --- instrumentation -------------------------------------------------------
    def stream(self) -> int:
        return self.lib.sdg_stream(self.h) or 0

    def state_device_ptr(self) -> int:
        p = _dp()
        self.lib.sdg_state_device_ptr(self.h, C.byref(p))
        return C.cast(p, C.c_void_p).value

    def kernel_launches(self) -> int:
        return self.lib.sdg_kernel_launches(self.h)

    def enable_kernel_timing(self, on: bool = True):
        self.lib.sdg_enable_kernel_timing(self.h, int(on))

    def kernel_timing(self) -> dict:
        names = C.create_string_buffer(512)
        ms = np.zeros(16)
        cnt = np.zeros(16, dtype=np.int64)
        n = C.c_int()
        self._check(self.lib.sdg_kernel_timing(self.h, names, 512, _d(ms), cnt.ctypes.data_as(_lp), 16, C.byref(n)))
        keys = names.value.decode().split(",")
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(keys[: n.value])}


def run_inproc(mesh: T.MeshSpec, cfg: T.SolverConfig, n_ranks: int, body, device: int = 0, hub: str = "sdg"):
    """Runs `body(solver)` on n_ranks in-process ranks (one host thread each) that
    share `device`; returns the per-rank results.  Collective calls happen
    inside `body` on every rank in the same order."""
    import threading
    out = [None] * n_ranks
    err = [None] * n_ranks

    def worker(r):
        try:
            s = RankSolver(mesh, cfg, n_ranks=n_ranks, rank=r, device=device, inproc_hub=hub, init_rank_maps=False)
            s.init_rank_maps()
            out[r] = body(s)
            s.close()
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err[r] = e

    ths = [threading.Thread(target=worker, args=(r,)) for r in range(n_ranks)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out


def gather_global(parts, n_elements_global: int, n1: int) -> np.ndarray:
    """Scatters per-rank (gids, local field) pairs into the global element order."""
    per = n1 ** 3 * T.NVARS
    g = np.full(n_elements_global * per, np.nan)
    for gids, u in parts:
        u = u.reshape(-1, per)
        for q, gid in enumerate(gids):
            g[gid * per:(gid + 1) * per] = u[q]
    return g


def plan(mesh: T.MeshSpec, n_ranks: int, rank: int, delta: float = 0.0) -> dict:
    """Host-only partition / message plan of one rank (no GPU): see sdg_plan_json."""
    import json
    n = C.c_long()
    T.raise_for(lib().sdg_plan_json(C.byref(mesh), n_ranks, rank, delta, None, 0, C.byref(n)),
                lib().sdg_global_error().decode())
    buf = C.create_string_buffer(n.value + 1)
    T.raise_for(lib().sdg_plan_json(C.byref(mesh), n_ranks, rank, delta, buf, n.value + 1, C.byref(n)),
                lib().sdg_global_error().decode())
    return json.loads(buf.value.decode())


def metrics_host(mesh: T.MeshSpec, degree: int, node_kind: int, n_ranks: int = 1, rank: int = 0):
    """Host-only curved metrics of one rank (no GPU): (met [E, N3, 10], fmet [E, 6, N2, 4])."""
    n = C.c_long()
    L = lib()
    T.raise_for(L.sdg_metrics_host(C.byref(mesh), degree, node_kind, n_ranks, rank, None, None, C.byref(n)),
                L.sdg_global_error().decode())
    n1 = degree + 1
    mw, fw = (13, 6) if mesh.mapping == T.MAP_ANNULUS else (10, 4)
    met = np.zeros((n.value, n1 ** 3, mw))
    fmet = np.zeros((n.value, 6, n1 * n1, fw))
    T.raise_for(L.sdg_metrics_host(C.byref(mesh), degree, node_kind, n_ranks, rank, _d(met), _d(fmet), C.byref(n)),
                L.sdg_global_error().decode())
    return met, fmet


def subrange_ops(degree: int, node_kind: int, lo: float, hi: float):
    """Face <-> mortar operators (fwd, bwd), n x n each, of a mortar on face sub-range [lo, hi]."""
    n1 = degree + 1
    fwd, bwd = np.zeros((n1, n1)), np.zeros((n1, n1))
    L = lib()
    T.raise_for(L.sdg_subrange_ops(degree, node_kind, lo, hi, _d(fwd), _d(bwd)), L.sdg_global_error().decode())
    return fwd, bwd


def mortar_intervals(n_a: int, n_b: int, l_a: float, delta: float, device: bool = False):
    """Mortars of a non-matching periodic face row: (faces [M, 2] = (A face, B face),
    ranges [M, 4] = (a_lo, a_hi, b_lo, b_hi)), in A order (by A face, then along it).
    device=True runs the device kernel (needs a GPU)."""
    L = lib()
    fn = L.sdg_mortar_intervals_device if device else L.sdg_mortar_intervals
    n = C.c_long()
    T.raise_for(fn(n_a, n_b, l_a, delta, C.byref(n), None, None), L.sdg_global_error().decode())
    faces = np.zeros((n.value, 2), dtype=np.int64)
    ranges = np.zeros((n.value, 4))
    T.raise_for(fn(n_a, n_b, l_a, delta, C.byref(n), faces.ctypes.data_as(_lp), _d(ranges)), L.sdg_global_error().decode())
    return faces, ranges


def interface_project_device(degree: int, node_kind: int, nfy, nfz, l_y: float, l_z: float, d_y: float, d_z: float,
                             src, from_side: int = 0):
    """Non-matching planar interface on the device: src [nfy[from]][nfz[from]][n][n][nc]
    -> (mortars [My * Mz, n, n, nc], target faces [nfy[to], nfz[to], n, n, nc])."""
    src = np.ascontiguousarray(src, dtype=np.float64)
    n1, nc = degree + 1, src.shape[-1]
    to = 1 - from_side
    fy = np.array(nfy, dtype=np.int64)
    fz = np.array(nfz, dtype=np.int64)
    assert src.shape == (fy[from_side], fz[from_side], n1, n1, nc)
    my = len(mortar_intervals(int(fy[0]), int(fy[1]), l_y, d_y)[0])
    mz = len(mortar_intervals(int(fz[0]), int(fz[1]), l_z, d_z)[0])
    mortar = np.zeros((my * mz, n1, n1, nc))
    dst = np.zeros((fy[to], fz[to], n1, n1, nc))
    nm = C.c_long()
    L = lib()
    T.raise_for(L.sdg_interface_project_device(degree, node_kind, fy.ctypes.data_as(_lp), fz.ctypes.data_as(_lp), l_y,
                                               l_z, d_y, d_z, nc, from_side, _d(src), _d(mortar), _d(dst),
                                               C.byref(nm)), L.sdg_global_error().decode())
    assert nm.value == my * mz
    return mortar, dst


def interface_flux_device(gas, degree: int, node_kind: int, nfy, nfz, l_y: float, l_z: float, d_y: float,
                          d_z: float, u_a, u_b, g_a=None, g_b=None):
    """Surface flux of a non-matching planar interface (normal +x, A below, B above)
    on the device: -> (mortar fluxes [My * Mz, n, n, 5], flux on A's faces, flux on
    B's faces), u_* [nfy[s], nfz[s], n, n, 5], optional gradients g_* [..., 12]."""
    n1 = degree + 1
    fy = np.array(nfy, dtype=np.int64)
    fz = np.array(nfz, dtype=np.int64)
    u = [np.ascontiguousarray(x, dtype=np.float64) for x in (u_a, u_b)]
    g = [None if x is None else np.ascontiguousarray(x, dtype=np.float64) for x in (g_a, g_b)]
    for s in (0, 1):
        assert u[s].shape == (fy[s], fz[s], n1, n1, 5)
        assert g[s] is None or g[s].shape == (fy[s], fz[s], n1, n1, 12)
    my = len(mortar_intervals(int(fy[0]), int(fy[1]), l_y, d_y)[0])
    mz = len(mortar_intervals(int(fz[0]), int(fz[1]), l_z, d_z)[0])
    fm = np.zeros((my * mz, n1, n1, 5))
    fa = np.zeros((fy[0], fz[0], n1, n1, 5))
    fb = np.zeros((fy[1], fz[1], n1, n1, 5))
    nm = C.c_long()
    L = lib()
    gp = [None if x is None else _d(x) for x in g]
    T.raise_for(L.sdg_interface_flux_device(C.byref(gas), degree, node_kind, fy.ctypes.data_as(_lp),
                                            fz.ctypes.data_as(_lp), l_y, l_z, d_y, d_z, _d(u[0]), _d(u[1]), gp[0],
                                            gp[1], _d(fm), _d(fa), _d(fb), C.byref(nm)),
                L.sdg_global_error().decode())
    assert nm.value == my * mz
    return fm, fa, fb


def interface_lift_device(gas, degree: int, node_kind: int, nfy, nfz, l_y: float, l_z: float, d_y: float,
                          d_z: float, u_a, u_b):
    """Lifting mean of a non-matching planar interface on the device: -> (mortar
    means [My * Mz, n, n, 4] of (u, v, w, T), their projections onto A's and B's faces)."""
    n1 = degree + 1
    fy = np.array(nfy, dtype=np.int64)
    fz = np.array(nfz, dtype=np.int64)
    u = [np.ascontiguousarray(x, dtype=np.float64) for x in (u_a, u_b)]
    for s in (0, 1):
        assert u[s].shape == (fy[s], fz[s], n1, n1, 5)
    my = len(mortar_intervals(int(fy[0]), int(fy[1]), l_y, d_y)[0])
    mz = len(mortar_intervals(int(fz[0]), int(fz[1]), l_z, d_z)[0])
    lm = np.zeros((my * mz, n1, n1, 4))
    la = np.zeros((fy[0], fz[0], n1, n1, 4))
    lb = np.zeros((fy[1], fz[1], n1, n1, 4))
    nm = C.c_long()
    L = lib()
    T.raise_for(L.sdg_interface_lift_device(C.byref(gas), degree, node_kind, fy.ctypes.data_as(_lp),
                                            fz.ctypes.data_as(_lp), l_y, l_z, d_y, d_z, _d(u[0]), _d(u[1]), _d(lm),
                                            _d(la), _d(lb), C.byref(nm)),
                L.sdg_global_error().decode())
    assert nm.value == my * mz
    return lm, la, lb


def pairing_device(faces, n_par, n_perp, ranks, n_delta, on_static, conforming, self_rank):
    """Device pairing kernel on a caller-given face set (rebuild_index_arrays contract)."""
    faces = np.ascontiguousarray(faces, dtype=np.int64).reshape(-1, 3)
    ranks = np.ascontiguousarray(ranks, dtype=np.int32).reshape(-1)
    nl = faces.shape[0]
    cols = np.zeros((2 * nl + 1, T.TUPLE_INTS), dtype=np.int32)
    w = (faces[:, 0].max() - faces[:, 0].min() + 1) if nl else 1
    m = np.zeros(2 * w, dtype=np.int32)
    ncols, nsched = C.c_int(), C.c_int()
    face_lo = C.c_long()
    sched = np.zeros(3 * (2 * nl + 1), dtype=np.int32)
    self_e = np.zeros(3, dtype=np.int32)
    code = lib().sdg_pairing_device(nl, faces.ctypes.data_as(_lp), n_par, n_perp, ranks.ctypes.data_as(_ip), n_delta,
                                    int(on_static), int(conforming), self_rank, C.byref(ncols),
                                    cols.ctypes.data_as(_ip), m.ctypes.data_as(_ip), C.byref(face_lo),
                                    C.byref(nsched), sched.ctypes.data_as(_ip), self_e.ctypes.data_as(_ip))
    T.raise_for(code, lib().sdg_global_error().decode())
    return dict(cols=cols[: ncols.value], m=m.reshape(2, -1), face_lo=face_lo.value,
                sched=sched[: 3 * nsched.value].reshape(-1, 3), self_entry=self_e)
