"""Curved hexahedra (SDG_MAP_WARP) and the rotating annulus (SDG_MAP_ANNULUS) in the CPU oracle.

The reference has affine elements only (ElementMetrics, proj/src/mesh.cpp:102-111),
so the curved restatement is pinned by properties rather than by reference
outputs:
  * on an affine geometry the curved code path reproduces the affine path
    (which is itself pinned to the reference, tests/test_oracle_pins.py);
  * the discrete metric identities hold to rounding (conservative curl form);
  * free-stream preservation across sliding interfaces at several offsets
    (3D form of proj/tests/test_solver.cpp:78-101 on curved elements);
  * conservation of mass and energy over 10 steps (test_solver.cpp:282-299);
  * convergence of the advected density wave under refinement.
"""
import numpy as np
import pytest

from conftest import rel_linf
from oracle import pyoracle as P
from paper_2008_04356_b200 import types as T

BANDS3 = [(2, 1.0, 0.0), (2, 1.0, 1.0), (2, 1.0, 0.0)]


def _basis(degree, kind):
    n = degree + 1
    lib = P.oracle_lib()
    x, w, D, fl, fr = (np.zeros(n), np.zeros(n), np.zeros(n * n), np.zeros(n), np.zeros(n))
    assert lib.orc_nodes(degree, kind, P._d(x), P._d(w)) == 0
    assert lib.orc_basis(degree, kind, P._d(D), P._d(fl), P._d(fr)) == 0
    return x, w, D.reshape(n, n), fl, fr


@pytest.mark.parametrize("kind", [T.NODES_GAUSS, T.NODES_LGL])
@pytest.mark.parametrize("mu", [0.0, 1e-3])
def test_curved_path_on_affine_geometry_matches_affine(kind, mu):
    """warp = 0: metrics equal the affine ones up to rounding, so residual,
    BR1 gradients and two RK steps agree with the affine (reference-pinned) path."""
    per = (False, True, True)
    cfg = T.solver_config(3, kind, mu=mu, case=T.density_wave(a=(1.0, 1.0, 0.5)))
    a = P.Oracle3D(T.mesh_spec(BANDS3, ny=4, nz=3, depth=1.0, periodic=per), cfg)
    c = P.Oracle3D(T.mesh_spec(BANDS3, ny=4, nz=3, depth=1.0, periodic=per, warp=0.0), cfg)
    a.set_initial_condition(0.0)
    c.set_initial_condition(0.0)
    assert rel_linf(c.field(), a.field()) == 0.0
    for t in (0.0, 0.37):
        assert rel_linf(c.compute_residual(t), a.compute_residual(t)) < 1e-13
    if mu > 0.0:
        assert rel_linf(c.compute_gradients(0.37), a.compute_gradients(0.37)) < 1e-13
    dt = a.suggest_dt(0.5)
    a.step(dt, 2)
    c.step(dt, 2)
    assert rel_linf(c.field(), a.field()) < 1e-13


@pytest.mark.parametrize("kind", [T.NODES_GAUSS, T.NODES_LGL])
@pytest.mark.parametrize("degree", [3, 5])
def test_discrete_metric_identities(kind, degree):
    """sum_d [ l(+1)/w (n sJ)+ - l(-1)/w (n sJ)- - Dhat Ja^d ] = 0 at every node:
    the condition for free-stream preservation of the weak-form DGSEM."""
    n = degree + 1
    x, w, D, fl, fr = _basis(degree, kind)
    Dh = (w[None, :] * D.T) / w[:, None]
    m = T.mesh_spec(BANDS3, ny=4, nz=3, depth=1.0, warp=0.3)
    o = P.Oracle3D(m, T.solver_config(degree, kind, case=T.freestream()))
    met, fmet = o.metrics()
    E = met.shape[0]
    Ja = met[:, :, :9].reshape(E, n, n, n, 3, 3)
    NS = (fmet[:, :, :, :3] * fmet[:, :, :, 3:4]).reshape(E, 6, n, n, 3)
    lw0, lw1 = fl / w, fr / w
    res = -np.einsum("im,emjkc->eijkc", Dh, Ja[..., 0, :])
    res -= np.einsum("jm,eimkc->eijkc", Dh, Ja[..., 1, :])
    res -= np.einsum("km,eijmc->eijkc", Dh, Ja[..., 2, :])
    res += lw1[None, :, None, None, None] * NS[:, 1, None] - lw0[None, :, None, None, None] * NS[:, 0, None]
    res += lw1[None, None, :, None, None] * NS[:, 3, :, None] - lw0[None, None, :, None, None] * NS[:, 2, :, None]
    res += lw1[None, None, None, :, None] * NS[:, 5, :, :, None] - lw0[None, None, None, :, None] * NS[:, 4, :, :, None]
    assert np.abs(res).max() < 1e-14 * np.abs(Ja).max() * 100
    # unit normals, positive Jacobians, genuinely curved geometry
    assert np.allclose(np.linalg.norm(fmet[..., :3], axis=-1), 1.0, atol=1e-15)
    assert (met[:, :, 9] > 0).all()
    assert np.ptp(met[:, :, 9]) > 0.1 * met[:, :, 9].mean()


def test_sliding_faces_stay_planar():
    """The warp vanishes on band boundaries (BASELINE configs[3]: interface faces
    left unwarped): x-faces on the interfaces have normal e_x and sJ = hy hz / 4."""
    m = T.mesh_spec(BANDS3, ny=4, nz=3, depth=1.0, warp=0.3)
    o = P.Oracle3D(m, T.solver_config(3, T.NODES_GAUSS, case=T.freestream()))
    _, fmet = o.metrics()
    hy, hz = 2.0 / 4, 1.0 / 3
    # band 1 (moving) occupies gids 24..47; its x- faces (side 0) of ix = 0 sit on interface 0
    for g in range(24, 24 + 12):
        f = fmet[g, 0]
        assert np.abs(f[:, 0] - 1.0).max() < 1e-15 and np.abs(f[:, 1:3]).max() < 1e-15
        assert np.abs(f[:, 3] - 0.25 * hy * hz).max() < 1e-15


@pytest.mark.parametrize("kind", [T.NODES_GAUSS, T.NODES_LGL])
@pytest.mark.parametrize("mu", [0.0, 1e-3])
def test_freestream_preservation_curved_sliding(kind, mu):
    """3D curved form of proj/tests/test_solver.cpp:86-92 (7 interface offsets)."""
    mesh = T.mesh_spec(BANDS3, ny=6, nz=3, depth=1.0, warp=0.2)
    o = P.Oracle3D(mesh, T.solver_config(3, kind, mu=mu, case=T.freestream(v=(1.0, 0.5, 0.25))))
    o.set_initial_condition(0.0)
    for t in (0.0, 0.05, 1.0 / 3.0, 0.37, 0.99, 2.0, 5.0 + 1e-9):
        assert np.abs(o.compute_residual(t)).max() < 1e-12


def test_conservation_curved_sliding():
    """3D curved form of proj/tests/test_solver.cpp:282-299 (J-weighted quadrature)."""
    mesh = T.mesh_spec(BANDS3, ny=6, nz=2, depth=1.0, warp=0.25)
    o = P.Oracle3D(mesh, T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave(a=(1.0, 1.0, 0.5))))
    o.set_initial_condition(0.0)
    before = o.mass_energy()
    o.step(o.suggest_dt(0.4), 10)
    after = o.mass_energy()
    assert np.all(np.abs(after - before) / np.abs(before) < 1e-12)


def test_density_wave_converges_on_curved_mesh():
    """Inviscid density wave on a warped periodic box: the L_inf error after a
    fixed time drops at (close to) the design order N+1 under h-refinement."""
    errs = []
    for ne in (2, 4):
        mesh = T.mesh_spec([(ne, 1.0, 0.0), (ne, 1.0, 0.4)], ny=2 * ne, nz=2 * ne, warp=0.15)
        o = P.Oracle3D(mesh, T.solver_config(3, T.NODES_GAUSS, case=T.density_wave(a=(1.0, 1.0, 0.5))))
        o.set_initial_condition(0.0)
        t_end = 0.1
        dt0 = o.suggest_dt(0.25)
        steps = int(np.ceil(t_end / dt0))
        o.step(t_end / steps, steps)
        errs.append(np.abs(o.field() - o.sample_case(t_end)).max())
    rate = np.log2(errs[0] / errs[1])
    assert rate > 3.0, (errs, rate)


# ---------------------------------------------------------------- rotating annulus (SDG_MAP_ANNULUS)
ROTOR = [(2, 1.0, 0.0), (2, 1.0, 0.8)]  # stator | rotor at omega = 0.8 (BASELINE configs[2])


@pytest.mark.parametrize("kind", [T.NODES_GAUSS, T.NODES_LGL])
@pytest.mark.parametrize("mu", [0.0, 1e-3])
@pytest.mark.parametrize("warp", [None, 0.1])
def test_rotating_annulus_preserves_free_stream(kind, mu, warp):
    """Axial free stream through a stator/rotor annulus: the contravariant grid
    velocity is a discrete curl, so the discrete GCL holds and the uniform state
    is a steady solution at every rotor angle (configs[2]: free-stream preservation)."""
    m = T.annulus_spec(ROTOR, 8, 2, 0.5, 1.0, warp=warp)
    o = P.Oracle3D(m, T.solver_config(3, kind, mu=mu, case=T.freestream(v=(1.0, 0.0, 0.0))))
    o.set_initial_condition(0.0)
    for t in (0.0, 0.1, 0.37, 1.3, 7.9):
        assert np.abs(o.compute_residual(t)).max() < 1e-12
    o.step(o.suggest_dt(0.5), 5)
    assert np.abs(o.field() - o.sample_case(o.time())).max() < 1e-12


def test_rotating_annulus_metrics():
    """Grid velocity per unit omega: (vg/omega) . n on the faces is bounded by the
    tip radius and vanishes on the axial-normal (sliding) faces; metrics satisfy
    the discrete identities including the grid-velocity (GCL) identity."""
    degree = 4
    n = degree + 1
    m = T.annulus_spec(ROTOR, 8, 2, 0.5, 1.0, warp=0.1)
    o = P.Oracle3D(m, T.solver_config(degree, T.NODES_GAUSS, case=T.freestream()))
    met, fmet = o.metrics()
    assert met.shape[2] == 13 and fmet.shape[3] == 6
    # band-boundary x faces (ix = 0 side 0, ix = 1 side 1 in each 2 x 8 x 2 band) are planar: vg . e_x = 0
    for b in range(2):
        lo = 32 * b
        assert np.abs(fmet[lo:lo + 16, 0, :, 4]).max() < 1e-14
        assert np.abs(fmet[lo + 16:lo + 32, 1, :, 4]).max() < 1e-14
    assert np.abs(fmet[:, :, :, 4]).max() <= 1.0 + 0.1 * 0.25 + 1e-12  # |vg| / omega <= r, warped r <= 1 + A hz
    x, w, D, fl, fr = _basis(degree, T.NODES_GAUSS)
    Dh = (w[None, :] * D.T) / w[:, None]
    E = met.shape[0]
    V = met[:, :, 10:13].reshape(E, n, n, n, 3)
    S = (fmet[:, :, :, 3] * fmet[:, :, :, 4]).reshape(E, 6, n, n)
    lw0, lw1 = fl / w, fr / w
    res = -np.einsum("im,emjk->eijk", Dh, V[..., 0]) - np.einsum("jm,eimk->eijk", Dh, V[..., 1]) \
        - np.einsum("km,eijm->eijk", Dh, V[..., 2])
    res += lw1[None, :, None, None] * S[:, 1, None] - lw0[None, :, None, None] * S[:, 0, None]
    res += lw1[None, None, :, None] * S[:, 3, :, None] - lw0[None, None, :, None] * S[:, 2, :, None]
    res += lw1[None, None, None, :] * S[:, 5, :, :, None] - lw0[None, None, None, :] * S[:, 4, :, :, None]
    assert np.abs(res).max() < 1e-13


def test_rotating_annulus_density_wave_converges():
    """Axial density wave (an exact solution independent of theta and r) through
    the rotating annulus: error drops at ~ the design order under refinement."""
    errs = []
    for ne in (2, 4):
        m = T.annulus_spec([(ne, 1.0, 0.0), (ne, 1.0, 0.8)], 4 * ne, ne, 0.5, 1.0, warp=0.1)
        o = P.Oracle3D(m, T.solver_config(3, T.NODES_GAUSS, case=T.density_wave(a=(1.0, 0.0, 0.0),
                                                                                k=(1.0, 0.0, 0.0))))
        o.set_initial_condition(0.0)
        dt = o.suggest_dt(0.3)
        st = int(np.ceil(0.2 / dt))
        o.step(0.2 / st, st)
        errs.append(np.abs(o.field() - o.sample_case(0.2)).max())
    assert np.log2(errs[0] / errs[1]) > 3.0, errs


def test_annulus_config_errors():
    with pytest.raises(T.ConfigError):  # periodic sector that does not divide the full circle
        P.Oracle3D(T.mesh_spec(ROTOR, ny=8, nz=2, height=1.0, depth=0.5, z0=0.5, periodic=(False, True, False),
                               mapping=T.MAP_ANNULUS), T.solver_config(2))
    with pytest.raises(T.ConfigError):  # inner radius 0
        P.Oracle3D(T.annulus_spec(ROTOR, 8, 2, 0.0, 1.0), T.solver_config(2))


# ---------------------------------------------------------------- periodic annulus sectors
def _sector_pair(nth=3, m=8, bands=ROTOR, n_r=2):
    full = T.annulus_spec(bands, m * nth, n_r, 0.5, 1.0)
    sec = T.annulus_spec(bands, nth, n_r, 0.5, 1.0, theta_span=2.0 * np.pi / m)
    assert sec.periodic_y == 1
    return full, sec


@pytest.mark.parametrize("kind", [T.NODES_GAUSS, T.NODES_LGL])
@pytest.mark.parametrize("mu", [0.0, 1e-3])
def test_periodic_sector_reproduces_full_annulus(kind, mu):
    """A pi/4 sector with rotational periodicity (momentum, gradients and fluxes
    rotated across the theta seam and across wrapped rotor/stator mortars) equals
    the first sector of the full annulus for an axisymmetric swirling state; the
    invariant curl form makes the metrics rotation covariant, so the two
    discretisations coincide up to rounding."""
    m, nth = 8, 3
    full, sec = _sector_pair(nth, m)
    cfg = T.solver_config(3, kind, mu=mu, case=T.swirl(omega=0.7))
    of, osr = P.Oracle3D(full, cfg), P.Oracle3D(sec, cfg)
    of.set_initial_condition(0.0)
    osr.set_initial_condition(0.0)
    n3 = 4 ** 3

    def first(u):
        return u.reshape(2, 2, m * nth, 2, n3 * 5)[:, :, :nth].reshape(-1)

    assert np.array_equal(first(of.field()), osr.field())
    for t in (0.0, 0.05, 0.3, 1.7):
        rf, rs = first(of.compute_residual(t)), osr.compute_residual(t)
        assert np.abs(rf - rs).max() <= 1e-12 * np.abs(rf).max()
    dt = of.suggest_dt(0.4)
    of.step(dt, 5)
    osr.step(dt, 5)
    assert rel_linf(osr.field(), first(of.field())) <= 1e-12


def test_periodic_sector_windings():
    """The rotor passes the sector seam several times (windings of the sliding
    displacement): the sector still follows the full annulus."""
    m, nth = 4, 2
    full, sec = _sector_pair(nth, m, bands=[(1, 1.0, 0.0), (1, 1.0, 3.0)], n_r=1)
    cfg = T.solver_config(2, T.NODES_GAUSS, mu=1e-3, case=T.swirl(omega=0.4))
    of, osr = P.Oracle3D(full, cfg), P.Oracle3D(sec, cfg)
    of.set_initial_condition(0.0)
    osr.set_initial_condition(0.0)
    n3 = 3 ** 3
    dt = 0.5 * of.suggest_dt(0.4)
    steps = int(np.ceil(3.0 * (np.pi / 2) / 3.0 / dt))  # about three sector passes
    of.step(dt, steps)
    osr.step(dt, steps)
    first = of.field().reshape(2, m * nth, n3 * 5)[:, :nth].reshape(-1)
    assert rel_linf(osr.field(), first) <= 1e-11
