"""Curved hexahedra (SDG_MAP_WARP) and the rotating annulus (SDG_MAP_ANNULUS) on the CUDA path vs the CPU oracle, through
the C-ABI (k_gradient_curved / k_update_curved, csrc/curved.cuh).

Same tolerances as tests/test_gpu_parity.py: state relative Linf <= 1e-12
after one stage / step, <= 1e-10 after 100 stages; free stream <= 1e-12.
"""
import numpy as np
import pytest

from conftest import rel_linf
from oracle import pyoracle as P
from paper_2008_04356_b200 import types as T

pytestmark = pytest.mark.gpu

BANDS3 = [(2, 1.0, 0.0), (2, 1.0, 1.0), (2, 1.0, 0.0)]


def gpu_solver(mesh, cfg):
    from paper_2008_04356_b200.capi import RankSolver
    return RankSolver(mesh, cfg)


def warped3(ny=4, nz=3, warp=0.2, periodic=(True, True, True), nx=2):
    return T.mesh_spec([(nx, 1.0, 0.0), (nx, 1.0, 1.0), (nx, 1.0, 0.0)], ny=ny, nz=nz, depth=1.0, warp=warp,
                       periodic=periodic)


def box0_warped(n_per=2, warp=0.2):
    """BASELINE config [0] geometry with curved elements (Dirichlet across the split axis)."""
    return T.mesh_spec([(n_per, 1.0, 0.0), (n_per, 1.0, 0.5)], ny=n_per, nz=n_per, periodic=(False, True, True),
                       warp=warp)


CASES = {
    "w3_gauss_visc": (warped3(), dict(degree=3, node_kind=T.NODES_GAUSS, mu=1e-3)),
    "w3_lgl_inv": (warped3(), dict(degree=3, node_kind=T.NODES_LGL, mu=0.0)),
    "box0w_gauss_visc_n5": (box0_warped(), dict(degree=5, node_kind=T.NODES_GAUSS, mu=1e-3)),
    "box0w_lgl_visc": (box0_warped(), dict(degree=4, node_kind=T.NODES_LGL, mu=1e-3)),
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("t", [0.0, 0.37])
def test_curved_residual_matches_oracle(name, t):
    mesh, kw = CASES[name]
    cfg = T.solver_config(case=T.density_wave(a=(1.0, 1.0, 0.5)), **kw)
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    o.set_initial_condition(0.0)
    g.set_initial_condition(0.0)
    assert rel_linf(g.field(), o.field()) <= 1e-15
    u = o.field()
    assert rel_linf(g.compute_residual(t, u), o.compute_residual(t, u)) <= 1e-12


@pytest.mark.parametrize("degree", [1, 2, 3, 4, 5, 6, 7])
@pytest.mark.parametrize("kind", [T.NODES_LGL, T.NODES_GAUSS])
def test_curved_all_degrees_one_step(degree, kind):
    mesh = warped3(ny=3, nz=2, periodic=(False, True, True))
    cfg = T.solver_config(degree, kind, mu=1e-3, case=T.density_wave(a=(1.0, 1.0, 0.5)))
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    dt = o.suggest_dt(0.4)
    g.step(dt)
    o.step(dt)
    assert rel_linf(g.field(), o.field()) <= 1e-12


def test_curved_gradients_match_oracle():
    mesh, kw = CASES["box0w_gauss_visc_n5"]
    cfg = T.solver_config(case=T.density_wave(a=(1.0, 1.0, 0.5)), **kw)
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    o.set_initial_condition(0.0)
    u = o.field()
    assert rel_linf(g.compute_gradients(0.2, u), o.compute_gradients(0.2, u)) <= 1e-12


def test_curved_hundred_stages():
    mesh = box0_warped(2, warp=0.25)
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave())
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    dt = o.suggest_dt(0.5)
    g.step(dt, 20)
    o.step(dt, 20)
    assert rel_linf(g.field(), o.field()) <= 1e-10
    assert g.total_rebuilds() == o.total_rebuilds()


@pytest.mark.parametrize("kind", [T.NODES_LGL, T.NODES_GAUSS])
def test_curved_freestream_preserved_across_sliding(kind):
    mesh = warped3(ny=6, nz=3)
    cfg = T.solver_config(3, kind, mu=1e-3, case=T.freestream(v=(1.0, 0.5, 0.25)))
    g = gpu_solver(mesh, cfg)
    g.set_initial_condition(0.0)
    u = g.field()
    for t in (0.0, 0.05, 1.0 / 3.0, 0.37, 0.99, 2.0):
        assert np.abs(g.compute_residual(t, u)).max() < 1e-12
    g.step(g.suggest_dt(0.5), 10)
    assert g.diagnostics(g.time())["max_deviation"] < 1e-12


def test_curved_conservation_and_diagnostics():
    mesh = warped3(ny=6, nz=2, warp=0.25)
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave(a=(1.0, 1.0, 0.5)))
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    d0 = g.diagnostics(0.0)
    me0 = o.mass_energy(g.field())
    assert abs(d0["mass"] - me0[0]) <= 1e-13 * abs(me0[0])
    assert abs(d0["volume"] - 4.0) <= 1e-12  # [0,2] x [0,2] x [0,1]: the warp preserves the volume
    g.step(g.suggest_dt(0.4), 10)
    d1 = g.diagnostics(g.time())
    assert abs(d1["mass"] - d0["mass"]) <= 1e-12 * abs(d0["mass"])
    assert abs(d1["energy"] - d0["energy"]) <= 1e-12 * abs(d0["energy"])


@pytest.mark.parametrize("ranks,partition", [(3, T.PARTITION_LEX), (6, T.PARTITION_SFC)])
def test_curved_rank_counts_do_not_change_the_bits(ranks, partition):
    from paper_2008_04356_b200 import capi
    mesh = T.mesh_spec(BANDS3, ny=6, nz=2, depth=1.0, partition=partition, warp=0.2)
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave())
    n_el = 2 * 6 * 2 * 3

    def body(s):
        s.set_initial_condition(0.0)
        s.step(0.004, 5)
        return s.local_element_ids(), s.field()

    ref = capi.gather_global(capi.run_inproc(mesh, cfg, 1, body, hub="c1"), n_el, 4)
    got = capi.gather_global(capi.run_inproc(mesh, cfg, ranks, body, hub=f"c{ranks}p{partition}"), n_el, 4)
    assert not np.isnan(got).any()
    assert np.array_equal(got, ref)


def test_curved_multi_wave_mesh_matches_oracle():
    """More element tiles than resident CTAs (the double-buffered trace path)."""
    mesh = T.mesh_spec([(6, 1.0, 0.0), (6, 1.0, 0.5), (6, 1.0, 0.0)], ny=8, nz=8, warp=0.1)
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave(a=(1.0, 1.0, 0.5)))
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    dt = o.suggest_dt(0.4)
    g.step(dt, 2)
    o.step(dt, 2)
    assert rel_linf(g.field(), o.field()) <= 1e-12


# ---------------------------------------------------------------- rotating annulus (SDG_MAP_ANNULUS)
def rotor(ne=2, warp=0.1, omega=0.8):
    """BASELINE configs[2] shape: stator | rotor annulus r in [0.5, 1], full circle, axial split."""
    return T.annulus_spec([(ne, 1.0, 0.0), (ne, 1.0, omega)], 4 * ne, ne, 0.5, 1.0, warp=warp)


AXIAL_WAVE = dict(a=(1.0, 0.0, 0.0), k=(1.0, 0.0, 0.0))


@pytest.mark.parametrize("kind", [T.NODES_GAUSS, T.NODES_LGL])
@pytest.mark.parametrize("mu", [0.0, 1e-3])
@pytest.mark.parametrize("t", [0.0, 0.37, 3.1])
def test_rotating_annulus_residual_matches_oracle(kind, mu, t):
    mesh = rotor()
    cfg = T.solver_config(3, kind, mu=mu, case=T.density_wave(**AXIAL_WAVE))
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    o.set_initial_condition(0.0)
    g.set_initial_condition(0.0)
    assert rel_linf(g.field(), o.field()) <= 1e-15
    u = o.field()
    assert rel_linf(g.compute_residual(t, u), o.compute_residual(t, u)) <= 1e-12
    if mu > 0.0:
        assert rel_linf(g.compute_gradients(t, u), o.compute_gradients(t, u)) <= 1e-12


@pytest.mark.parametrize("degree", [1, 2, 3, 4, 5, 6, 7])
def test_rotating_annulus_one_step_all_degrees(degree):
    mesh = rotor(warp=0.05)
    cfg = T.solver_config(degree, T.NODES_GAUSS, mu=1e-3, case=T.density_wave(**AXIAL_WAVE))
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    dt = o.suggest_dt(0.4)
    assert abs(g.suggest_dt(0.4) - dt) <= 1e-14 * dt
    g.step(dt)
    o.step(dt)
    assert rel_linf(g.field(), o.field()) <= 1e-12


def test_rotating_annulus_hundred_stages_and_free_stream():
    mesh = rotor()
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave(**AXIAL_WAVE))
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    dt = o.suggest_dt(0.5)
    g.step(dt, 20)
    o.step(dt, 20)
    assert rel_linf(g.field(), o.field()) <= 1e-10
    assert g.total_rebuilds() == o.total_rebuilds()
    fs = gpu_solver(mesh, T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.freestream(v=(1.0, 0.0, 0.0))))
    fs.set_initial_condition(0.0)
    u = fs.field()
    for t in (0.0, 0.2, 1.7):
        assert np.abs(fs.compute_residual(t, u)).max() < 1e-12
    fs.step(fs.suggest_dt(0.5), 10)
    assert fs.diagnostics(fs.time())["max_deviation"] < 1e-12


def test_rotating_annulus_rank_split_keeps_the_bits():
    """Stator and rotor on different ranks (the mortar exchange carries the
    rotor/stator coupling) equals one rank bit for bit."""
    from paper_2008_04356_b200 import capi
    mesh = rotor()
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave(**AXIAL_WAVE))
    n_el = 2 * 2 * 8 * 2

    def body(s):
        s.set_initial_condition(0.0)
        s.step(0.01, 5)
        return s.local_element_ids(), s.field()

    ref = capi.gather_global(capi.run_inproc(mesh, cfg, 1, body, hub="ann1"), n_el, 4)
    got = capi.gather_global(capi.run_inproc(mesh, cfg, 2, body, hub="ann2"), n_el, 4)
    assert not np.isnan(got).any()
    assert np.array_equal(got, ref)


# ---------------------------------------------------------------- periodic annulus sectors
def sector(nth=3, m=8, bands=None, n_r=2, warp=None):
    bands = bands or [(2, 1.0, 0.0), (2, 1.0, 0.8)]
    return T.annulus_spec(bands, nth, n_r, 0.5, 1.0, warp=warp, theta_span=2.0 * np.pi / m)


@pytest.mark.parametrize("kind", [T.NODES_GAUSS, T.NODES_LGL])
@pytest.mark.parametrize("mu", [0.0, 1e-3])
@pytest.mark.parametrize("t", [0.0, 0.3, 1.7])
def test_periodic_sector_residual_matches_oracle(kind, mu, t):
    """configs[2] geometry: pi/4 sector, rotor at 0.8; momentum, gradients and fluxes
    rotate across the theta seam and across wrapped rotor/stator mortars."""
    mesh = sector(warp=0.05)
    cfg = T.solver_config(3, kind, mu=mu, case=T.swirl(omega=0.7))
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    o.set_initial_condition(0.0)
    u = o.field()
    assert rel_linf(g.compute_residual(t, u), o.compute_residual(t, u)) <= 1e-12


@pytest.mark.parametrize("degree", [2, 3, 5])
def test_periodic_sector_steps_through_windings(degree):
    """The rotor passes the seam twice (windings of the sliding displacement)."""
    mesh = sector(nth=2, m=4, bands=[(1, 1.0, 0.0), (1, 1.0, 3.0)], n_r=1)
    cfg = T.solver_config(degree, T.NODES_GAUSS, mu=1e-3, case=T.swirl(omega=0.4))
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    dt = 0.5 * o.suggest_dt(0.4)
    steps = int(np.ceil((np.pi / 2) / dt))
    g.step(dt, steps)
    o.step(dt, steps)
    assert rel_linf(g.field(), o.field()) <= 1e-10
    assert g.total_rebuilds() == o.total_rebuilds()


def test_periodic_sector_rank_split_keeps_the_bits():
    from paper_2008_04356_b200 import capi
    mesh = sector()
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.swirl(omega=0.7))
    n_el = 2 * 2 * 3 * 2

    dt = P.Oracle3D(mesh, cfg)
    dt.set_initial_condition(0.0)
    dt = dt.suggest_dt(0.4)

    def body(s):
        s.set_initial_condition(0.0)
        s.step(dt, 5)
        return s.local_element_ids(), s.field()

    ref = capi.gather_global(capi.run_inproc(mesh, cfg, 1, body, hub="sec1"), n_el, 4)
    got = capi.gather_global(capi.run_inproc(mesh, cfg, 2, body, hub="sec2"), n_el, 4)
    assert np.array_equal(got, ref)


def config2_mesh():
    """BASELINE configs[2]: r in [0.5, 1], theta in [0, pi/4] (periodic), axial [0, 2] split at 1,
    downstream block rotating at omega = 0.8, 24 (theta) x 12 (r) x 24 (axial) curved hexahedra per block."""
    return T.annulus_spec([(24, 1.0, 0.0), (24, 1.0, 0.8)], 24, 12, 0.5, 1.0, length=2.0,
                          theta_span=np.pi / 4)


def test_baseline_config2_free_stream_and_parity():
    """configs[2] at its full size, N = 5: the uniform axial free stream (M = 0.3) is
    preserved at several rotor angles and over 5 steps; with seeded 1e-3 density and
    velocity perturbations one step agrees with the oracle."""
    mesh = config2_mesh()
    mach, gamma = 0.3, 1.4
    fs = T.freestream(rho=1.0, v=(1.0, 0.0, 0.0), p=1.0 / (gamma * mach * mach))
    cfg = T.solver_config(5, T.NODES_GAUSS, mu=1e-3, case=fs)
    g = gpu_solver(mesh, cfg)
    g.set_initial_condition(0.0)
    u0 = g.field()
    dt = g.suggest_dt(0.5)
    for t in (0.0, 0.1, 0.55):  # the state change one residual would make in a time step
        assert dt * np.abs(g.compute_residual(t, u0)).max() < 1e-12 * np.abs(u0).max()
    g.step(dt, 5)
    assert np.abs(g.field() - u0).max() < 1e-12 * np.abs(u0).max()
    # seeded perturbations (BASELINE: seeded 1e-3 density / velocity perturbations)
    rng = np.random.default_rng(2008043562)
    u = u0.reshape(-1, 5).copy()
    rho = u[:, 0] * (1.0 + 1e-3 * rng.uniform(-1.0, 1.0, u.shape[0]))
    vel = u[:, 1:4] / u[:, :1] + 1e-3 * rng.uniform(-1.0, 1.0, (u.shape[0], 3))
    p = (gamma - 1.0) * (u[:, 4] - 0.5 * (u[:, 1:4] ** 2).sum(axis=1) / u[:, 0])
    u = np.column_stack([rho, rho[:, None] * vel, p / (gamma - 1.0) + 0.5 * rho * (vel ** 2).sum(axis=1)]).reshape(-1)
    o = P.Oracle3D(mesh, cfg)
    o.set_initial_condition(0.0)
    o.set_state(u)
    g2 = gpu_solver(mesh, cfg)
    g2.set_initial_condition(0.0)
    g2.set_state(u)
    g2.step(dt)
    o.step(dt)
    assert rel_linf(g2.field(), o.field()) <= 1e-12


@pytest.mark.parametrize("ranks", [3, 6])
def test_periodic_sector_yslab_ranks_keep_the_bits(ranks):
    """y slabs through a rotating annulus sector: every rank owns stator and rotor rows (rank-local
    mortars), slab edges carry cross-rank mortars and seam faces; bitwise equal to one rank."""
    from paper_2008_04356_b200 import capi
    mesh = T.annulus_spec([(2, 1.0, 0.0), (2, 1.0, 0.8)], 6, 2, 0.5, 1.0, warp=0.05, theta_span=np.pi / 4,
                          partition=T.PARTITION_YSLAB)
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.swirl(omega=0.7))
    n_el = 4 * 6 * 2

    dt = P.Oracle3D(mesh, cfg)
    dt.set_initial_condition(0.0)
    dt = dt.suggest_dt(0.4)

    def body(s):
        s.set_initial_condition(0.0)
        s.step(dt, 5)
        return s.local_element_ids(), s.field()

    ref = capi.gather_global(capi.run_inproc(mesh, cfg, 1, body, hub=f"ys1_{ranks}"), n_el, 4)
    got = capi.gather_global(capi.run_inproc(mesh, cfg, ranks, body, hub=f"ys{ranks}"), n_el, 4)
    assert np.array_equal(got, ref)
