"""Parity where the bench numbers come from (VERDICT r1 "what's weak" #1): the
device against the oracle on the exact bench meshes, long runs at N=5 and N=7,
and convergence-order checks of the curved / rotating geometry the target
config uses (the reference has no curved elements; proj/tests/test_solver.cpp:
103-144 is the rate check this mirrors).

Tolerances as the north star: relative Linf <= 1e-12 after one step,
<= 1e-10 after 100 stages."""
import math
import os
import sys

import numpy as np
import pytest

from conftest import rel_linf
from oracle import pyoracle as P
from paper_2008_04356_b200 import types as T

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def gpu_solver(mesh, cfg):
    from paper_2008_04356_b200.capi import RankSolver
    return RankSolver(mesh, cfg)


class Args:
    def __init__(self, degree=5, mesh="rotor", elems=64):
        self.degree, self.mesh, self.elems = degree, mesh, elems


def one_step(mesh, cfg, steps=1, cfl=0.5, tol=1e-12):
    P.oracle_lib().orc_set_threads(os.cpu_count() or 1)
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    dt = o.suggest_dt(cfl)
    assert abs(g.suggest_dt(cfl) - dt) <= 1e-14 * dt
    g.step(dt, steps)
    o.step(dt, steps)
    err = rel_linf(g.field(), o.field())
    assert err <= tol, err
    return g, o


def test_bench_tgv_64_cubed_n5_one_step():
    """The configs[4] bench mesh itself: 64^3 elements (262,144 CTAs of k_update_bulk),
    N=5, TGV M=0.1 Re=1600, one RK step against the oracle."""
    mesh, _ = bench.tgv_mesh(T, 64, 64)
    cfg = T.solver_config(5, T.NODES_GAUSS, gamma=1.4, R=1.0, mu=1.0 / 1600.0, Pr=0.72, case=T.tgv())
    one_step(mesh, cfg)


@pytest.mark.parametrize("degree", [3, 7])
def test_bench_tgv_16_cubed_one_step(degree):
    """The configs[4] sweep's other degrees on the bench mesh builder at 16^3."""
    mesh, _ = bench.tgv_mesh(T, 16, 16)
    cfg = T.solver_config(degree, T.NODES_GAUSS, gamma=1.4, R=1.0, mu=1.0 / 1600.0, Pr=0.72, case=T.tgv())
    one_step(mesh, cfg)


def test_bench_rotor_theta_slice_one_step():
    """configs[3], the default bench workload: the full-axial (192) x full-radial (60)
    periodic 1/8 theta slice of the sector with the bench's element geometry, case
    (seeded broadband 1e-2 perturbation), rotor speed and viscosity, one RK step
    against the oracle (the whole 1.1M-element mesh needs ~140 GB in the oracle)."""
    mesh, cfg, conf, _ = bench.rotor_workload(Args(), 1, elements=(192, 12, 60), span_div=8)
    assert conf["elements"] == 192 * 12 * 60
    one_step(mesh, cfg)


def test_bench_rotor_mesh_is_the_target_config():
    """The bench's configs[3] mesh: 1,105,920 curved hexahedra, 20-degree periodic sector,
    3 axial blocks, N=5 -> 2.39e8 DOF (BASELINE: ~1.1M, ~2.4e8)."""
    mesh, cfg, conf, dof = bench.rotor_workload(Args(), 1)
    assert conf["elements"] == 1105920 and dof == 1105920 * 216
    assert abs(mesh.height - math.pi / 9) < 1e-15 and mesh.mapping == T.MAP_ANNULUS and mesh.warp == 0.05
    assert cfg.flow_case.pt_modes == 8 and cfg.flow_case.pt_amp == 1e-2 and cfg.flow_case.pt_coords == 1


@pytest.mark.parametrize("degree", [5, 7])
def test_hundred_stages_multi_wave(degree):
    """100 stages (20 steps) on a multi-wave mesh (several element tiles per resident
    CTA) with two sliding interfaces, N = 5 and 7, viscous."""
    mesh = T.mesh_spec([(4, 1.0, 0.0), (4, 1.0, 0.7), (4, 1.0, 0.0)], ny=8, nz=6)
    cfg = T.solver_config(degree, T.NODES_GAUSS, mu=1e-3, case=T.density_wave())
    one_step(mesh, cfg, steps=20, tol=1e-10)


def test_hundred_stages_rotating_sector_n5():
    """100 stages at N=5 on a configs[3]-shaped rotor/stator/rotor sector (20 degrees,
    5% warp, seeded broadband perturbation), viscous."""
    mesh, cfg, _, _ = bench.rotor_workload(Args(), 1, elements=(12, 6, 3))
    one_step(mesh, cfg, steps=20, tol=1e-10)


def _sector(n, omega, span=math.pi / 9, warp=0.05):
    bands = [(n, 1.0, 0.0), (n, 1.0, omega), (n, 1.0, 0.0)]
    return T.annulus_spec(bands, 2 * n, n, 0.8, 1.0, length=1.0, warp=warp, theta_span=span)


@pytest.mark.parametrize("warp", [0.0, 0.05])
def test_rotating_sector_converges_on_device(warp):
    """Convergence of an exact Euler solution (the axial density wave, SDG_CASE_SWIRL
    without swirl) on configs[3] geometry -- curved, warped, rotating rotor
    between two stators, periodic 20-degree sector -- on the device: N=3, error at
    t = 0.05 for 3 and 6 elements per block direction, rate > 3."""
    errs = []
    for n in (3, 6):
        mesh = _sector(n, 0.6, warp=warp)
        cfg = T.solver_config(3, T.NODES_GAUSS, mu=0.0, case=T.swirl(alpha=0.1, a=1.0, k=2.0, p0=5.0, omega=0.0))
        g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
        g.set_initial_condition(0.0)
        t_end, steps = 0.05, 10 * n
        g.step(t_end / steps, steps)
        errs.append(np.abs(g.field() - o.sample_case(t_end)).max())
    rate = math.log2(errs[0] / errs[1])
    assert rate > 3.0, (errs, rate)


def test_baseline_config2_converges_on_device():
    """configs[2] geometry (pi/4 periodic sector, r in [0.5, 1], two axial blocks, the
    downstream one rotating at 0.8): the same exact solution converges at rate > 3."""
    errs = []
    for n in (3, 6):
        mesh = T.annulus_spec([(n, 1.0, 0.0), (n, 1.0, 0.8)], 2 * n, n, 0.5, 1.0, length=2.0,
                              theta_span=math.pi / 4)
        cfg = T.solver_config(3, T.NODES_GAUSS, mu=0.0, case=T.swirl(alpha=0.1, a=1.0, k=1.0, p0=5.0, omega=0.0))
        g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
        g.set_initial_condition(0.0)
        t_end, steps = 0.05, 10 * n
        g.step(t_end / steps, steps)
        errs.append(np.abs(g.field() - o.sample_case(t_end)).max())
    rate = math.log2(errs[0] / errs[1])
    assert rate > 3.0, (errs, rate)


@pytest.mark.parametrize("ranks", [2, 4])
def test_bench_strong_scaling_mesh_rank_split_keeps_the_bits(ranks):
    """`bench.py --mesh tgv --strong` (configs[4]'s strong-scaling mesh, scaled to 12^3): one mesh
    split in y slabs through all three blocks.  2 and 4 ranks (in-process transport, one device)
    against one rank, bitwise, at the bench degree; the one-rank run takes the loopback path
    (mortar consumers read the producers' arrays), the others the per-partner block copies."""
    from paper_2008_04356_b200 import capi
    cfg = T.solver_config(5, T.NODES_GAUSS, gamma=1.4, R=1.0, mu=1.0 / 1600.0, Pr=0.72, case=T.tgv())
    n_el = 12 ** 3

    def body(s):
        s.set_initial_condition(0.0)
        s.step(s.suggest_dt(0.5), 2)
        return s.local_element_ids(), s.field()

    mesh, _ = bench.tgv_mesh(T, 12, 12, yslab=True)
    ref = capi.gather_global(capi.run_inproc(mesh, cfg, 1, body, hub="strong1"), n_el, 6)
    got = capi.gather_global(capi.run_inproc(mesh, cfg, ranks, body, hub=f"strong{ranks}"), n_el, 6)
    assert not np.isnan(got).any()
    assert np.array_equal(got, ref)
