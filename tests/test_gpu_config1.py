"""Non-matching, obliquely sliding interfaces on the device (BASELINE configs[1]):
the CUDA path's tensor-product mortar chain inside every stage against the
oracle (tests/test_nonmatching_solver.py pins the oracle), through the C-ABI.

Tolerances as the north star: relative Linf <= 1e-12 after one stage / step,
<= 1e-10 after 100 stages; the device rows (the pairing of a non-matching
interface) bit for bit."""
import math

import numpy as np
import pytest

from conftest import rel_linf
from oracle import pyoracle as P
from paper_2008_04356_b200 import types as T

pytestmark = pytest.mark.gpu


def gpu_solver(mesh, cfg):
    from paper_2008_04356_b200.capi import RankSolver
    return RankSolver(mesh, cfg)


def nc_box(n=4, m=3, periodic_x=False, vy=0.37, vz=0.11, nx=None):
    nx = n if nx is None else nx
    return T.mesh_spec([(nx, 1.0, 0.0), (nx, 1.0, vy, m, m, vz)], ny=n, nz=n, periodic=(periodic_x, True, True))


def config1(degree=7):
    """BASELINE configs[1]: [0,2]^3 split at the interface; lower block 16^3, upper
    12 x 12 faces by 16 along the split, sliding (+0.37, +0.11) (axes relabelled,
    include/sdg_types.h); the configs[0] case (Dirichlet across the split, gamma 1.4,
    Pr 0.72, mu 1e-3, R 1) plus the seeded 1e-3 perturbation of 8 modes |k| <= 4
    (SURVEY §8(d), mt19937_64(2008043560 + 1))."""
    mesh = T.mesh_spec([(16, 1.0, 0.0), (16, 1.0, 0.37, 12, 12, 0.11)], ny=16, nz=16, periodic=(False, True, True))
    base = T.density_wave(a=(1.0, 1.0, 1.0))
    case = T.perturbed(base, 1, 1e-3, 4, (0.0, 0.0, 0.0), (2.0, 2.0, 2.0), adv=(1.0, 1.0, 1.0))
    return mesh, T.solver_config(degree, T.NODES_GAUSS, gamma=1.4, R=1.0, mu=1e-3, Pr=0.72, case=case)


@pytest.mark.parametrize("kind", [T.NODES_GAUSS, T.NODES_LGL])
@pytest.mark.parametrize("mu", [0.0, 1e-3])
@pytest.mark.parametrize("t", [0.0, 0.13, 0.77])
def test_nonmatching_residual_matches_oracle(kind, mu, t):
    mesh = nc_box()
    cfg = T.solver_config(3, kind, mu=mu, case=T.density_wave(a=(1.0, 0.5, 0.25)))
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    o.set_initial_condition(0.0)
    u = o.field()
    assert g.n_nc_interfaces() == 1
    assert rel_linf(g.compute_residual(t, u), o.compute_residual(t, u)) <= 1e-12


def test_nonmatching_gradients_match_oracle():
    mesh = nc_box()
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave(a=(1.0, 0.5, 0.25)))
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    o.set_initial_condition(0.0)
    u = o.field()
    assert rel_linf(g.compute_gradients(0.31, u), o.compute_gradients(0.31, u)) <= 1e-12


def test_device_rows_bit_exact_every_stage():
    """The device recomputes both face-interval rows every stage (k_nc_rows); they are
    the oracle's rows bit for bit, at the same per-stage displacement."""
    mesh = nc_box()
    cfg = T.solver_config(2, T.NODES_GAUSS, mu=1e-3, case=T.density_wave())
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    from paper_2008_04356_b200 import capi
    _, _, c = capi.rk_coefficients()
    dt = 0.0123
    for step in range(4):
        t0 = g.time()
        for s in range(5):
            g.rk_stage(s, t0, dt)
            o.compute_residual(t0 + c[s] * dt, o.field())
            for d in (0, 1):
                fg, rg, dg = g.nc_rows(0, d)
                fo, ro, do = o.nc_rows(0, d)
                assert dg == do and np.array_equal(fg, fo) and np.array_equal(rg, ro), (step, s, d)
        o.step(dt)


@pytest.mark.parametrize("degree", [2, 3, 4, 5, 6, 7])
def test_nonmatching_one_step(degree):
    mesh = nc_box()
    cfg = T.solver_config(degree, T.NODES_GAUSS, mu=1e-3, case=T.density_wave(a=(1.0, 0.5, 0.25)))
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    dt = o.suggest_dt(0.5)
    assert abs(g.suggest_dt(0.5) - dt) <= 1e-14 * dt
    g.step(dt)
    o.step(dt)
    assert rel_linf(g.field(), o.field()) <= 1e-12


def test_nonmatching_hundred_stages_small():
    mesh = nc_box(periodic_x=True)
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave(a=(1.0, 0.5, 0.25)))
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    dt = o.suggest_dt(0.5)
    g.step(dt, 20)
    o.step(dt, 20)
    assert rel_linf(g.field(), o.field()) <= 1e-10


def test_baseline_config1_hundred_stages():
    """BASELINE configs[1] at full size (6,400 elements, N=7, 3.3M DOF): 100 RK stages
    from the seeded initial state, device against oracle <= 1e-10; the device rows at
    the last stage equal the oracle's."""
    mesh, cfg = config1(7)
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    assert g.n_elements == 16 ** 3 + 16 * 12 * 12
    assert rel_linf(g.field(), o.field()) <= 1e-15
    dt = o.suggest_dt(0.5)
    assert abs(g.suggest_dt(0.5) - dt) <= 1e-14 * dt
    g.step(dt, 20)
    o.step(dt, 20)
    assert rel_linf(g.field(), o.field()) <= 1e-10
    for d in (0, 1):
        fg, rg, dg = g.nc_rows(0, d)
        fo, ro, do = o.nc_rows(0, d)
        assert dg == do and np.array_equal(fg, fo) and np.array_equal(rg, ro)
    assert 16 <= len(g.nc_rows(0, 0)[0]) <= 16 + 12


@pytest.mark.parametrize("mu", [0.0, 1e-3])
def test_nonmatching_freestream_on_device(mu):
    mesh = nc_box()
    cfg = T.solver_config(4, T.NODES_GAUSS, mu=mu, case=T.freestream(v=(0.3, 0.5, 0.25)))
    g = gpu_solver(mesh, cfg)
    g.set_initial_condition(0.0)
    for t in (0.0, 0.05, 1.0 / 3.0, 0.77, 2.9):
        assert np.abs(g.compute_residual(t)).max() < 1e-12
    g.step(g.suggest_dt(0.5), 5)
    assert g.diagnostics(g.time())["max_deviation"] < 1e-12


def test_nonmatching_conservation_on_device():
    mesh = nc_box(periodic_x=True)
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave(a=(1.0, 0.5, 0.25)))
    g = gpu_solver(mesh, cfg)
    g.set_initial_condition(0.0)
    d0 = g.diagnostics(0.0, exact=False)
    g.step(g.suggest_dt(0.5), 5)
    d1 = g.diagnostics(g.time(), exact=False)
    assert abs(d1["mass"] - d0["mass"]) <= 1e-12 * d0["mass"]
    assert abs(d1["energy"] - d0["energy"]) <= 1e-12 * d0["energy"]


@pytest.mark.parametrize("mu", [0.0, 1e-3])
def test_tensor_mortars_equal_reference_mortars_on_device(mu):
    """SDG_MORTARS_TENSOR on an equal-count interface: the device's tensor-product chain
    against its reference-mortar chain (bitwise at conforming instants, rounding
    otherwise) and against the oracle."""
    ms = [T.mesh_spec([(2, 1.0, 0.0), (2, 1.0, 0.7), (2, 1.0, 0.0)], ny=4, nz=3, mortars=m)
          for m in (T.MORTARS_AUTO, T.MORTARS_TENSOR)]
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=mu, case=T.density_wave())
    ref, ten = (gpu_solver(m, cfg) for m in ms)
    o = P.Oracle3D(ms[1], cfg)
    o.set_initial_condition(0.0)
    u = o.field()
    for t in (0.0, 0.13, 0.5, 0.5 / 0.7):
        a, b = ref.compute_residual(t, u), ten.compute_residual(t, u)
        assert np.abs(a - b).max() <= 2e-13 * np.abs(a).max()
        if t in (0.0, 0.5 / 0.7):
            assert np.array_equal(a, b)
        assert rel_linf(b, o.compute_residual(t, u)) <= 1e-12


def test_nonmatching_multi_rank_is_refused():
    from paper_2008_04356_b200 import capi
    cfg = T.solver_config(2, T.NODES_GAUSS, case=T.density_wave())
    with pytest.raises(T.ConfigError):
        capi.run_inproc(nc_box(), cfg, 2, lambda s: None, hub="nc2")
