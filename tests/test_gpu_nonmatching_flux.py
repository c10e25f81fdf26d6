"""Non-matching sliding interfaces (BASELINE configs[1]): the two-sided surface flux
on the device (sdg_interface_flux_device).  Both sides' traces and gradients go to
the tensor-product mortars, the Roe + central viscous flux is evaluated at the
mortar nodes and L2-projected back to both sides.  Checked against the oracle's
face flux (oracle/sdg3d.cpp face_flux, the reference's face_numerical_flux,
solver.cpp:308-321) at every mortar node on numpy-assembled mortar traces, then
for conservation, free-stream preservation and the conforming limit."""
import itertools

import numpy as np
import pytest

from oracle import pyoracle as P
from paper_2008_04356_b200 import capi
from paper_2008_04356_b200 import types as T

pytestmark = pytest.mark.gpu

GAS_VISC = T.Gas(1.4, 287.0, 1e-3, 0.72)
GAS_EULER = T.Gas(1.4, 287.0, 0.0, 0.72)


def _states(rng, shape):
    """Physical conserved states: rho ~ 1 +- 0.1, |v| <= 0.3, p ~ 1 +- 0.1."""
    rho = 1.0 + 0.1 * rng.uniform(-1, 1, shape)
    v = 0.3 * rng.uniform(-1, 1, shape + (3,))
    p = 1.0 + 0.1 * rng.uniform(-1, 1, shape)
    u = np.empty(shape + (5,))
    u[..., 0] = rho
    u[..., 1:4] = rho[..., None] * v
    u[..., 4] = p / 0.4 + 0.5 * rho * (v ** 2).sum(-1)
    return u


def _rows_ops(degree, kind, n_a, n_b, l_a, d):
    faces, ranges = capi.mortar_intervals(n_a, n_b, l_a, d)
    ops = [[capi.subrange_ops(degree, kind, r[2 * s], r[2 * s + 1]) for r in ranges] for s in (0, 1)]
    return faces, ops


def _oracle_flux(gas, degree, kind, nfy, nfz, l_y, l_z, d_y, d_z, u, g):
    n = degree + 1
    fy, oy = _rows_ops(degree, kind, nfy[0], nfy[1], l_y, d_y)
    fz, oz = _rows_ops(degree, kind, nfz[0], nfz[1], l_z, d_z)

    def to_mortar(s, src, ky, kz):
        return np.einsum("ki,lj,ijc->klc", oy[s][ky][0], oz[s][kz][0], src[s][fy[ky, s], fz[kz, s]])

    lib = P.oracle_lib()
    fm = np.zeros((len(fy) * len(fz), n, n, 5))
    out = [np.zeros((nfy[s], nfz[s], n, n, 5)) for s in (0, 1)]
    f = np.zeros(5)
    for ky, kz in itertools.product(range(len(fy)), range(len(fz))):
        mu = [to_mortar(s, u, ky, kz) for s in (0, 1)]
        mg = [to_mortar(s, g, ky, kz) for s in (0, 1)] if g is not None else None
        m = ky * len(fz) + kz
        for i, j in itertools.product(range(n), range(n)):
            um, up = np.ascontiguousarray(mu[0][i, j]), np.ascontiguousarray(mu[1][i, j])
            gm = gp = None
            if mg is not None:
                gm, gp = P._d(np.ascontiguousarray(mg[0][i, j])), P._d(np.ascontiguousarray(mg[1][i, j]))
            assert lib.orc_face_flux(C_gas(gas), P._d(um), P._d(up), 0, 0.0, gm, gp, P._d(f)) == 0
            fm[m, i, j] = f
        for s in (0, 1):
            out[s][fy[ky, s], fz[kz, s]] += np.einsum("ik,jl,klc->ijc", oy[s][ky][1], oz[s][kz][1], fm[m])
    return fm, out[0], out[1]


def C_gas(gas):
    import ctypes
    return ctypes.byref(gas)


def _face_integral(f, degree, kind, l_y, l_z):
    x, w = np.zeros(degree + 1), np.zeros(degree + 1)
    assert P.oracle_lib().orc_nodes(degree, kind, P._d(x), P._d(w)) == 0
    return (l_y / 2) * (l_z / 2) * np.einsum("i,j,abijc->c", w, w, f)


@pytest.mark.parametrize("viscous", [False, True])
@pytest.mark.parametrize("kind", [T.NODES_GAUSS, T.NODES_LGL])
def test_config1_interface_flux_matches_oracle(viscous, kind):
    """configs[1] interface: 16 x 16 faces (A) against 12 x 12 (B), displaced by
    (0.37, 0.11) t at t = 1.3.  N = 5 keeps the per-node oracle loop to seconds
    (the transfer at N = 7 is covered in test_gpu_nonmatching.py)."""
    degree, n = 5, 6
    nfy, nfz = [16, 12], [16, 12]
    l = [2.0 / 16, 2.0 / 12]
    d_y, d_z = 0.37 * 1.3, 0.11 * 1.3
    rng = np.random.default_rng(20080435 + viscous + 2 * kind)
    u = [_states(rng, (nfy[s], nfz[s], n, n)) for s in (0, 1)]
    g = [0.1 * rng.standard_normal((nfy[s], nfz[s], n, n, 12)) for s in (0, 1)] if viscous else None
    gas = GAS_VISC if viscous else GAS_EULER
    fm, fa, fb = capi.interface_flux_device(gas, degree, kind, nfy, nfz, l[0], l[0], d_y, d_z, u[0], u[1],
                                            *(g if viscous else (None, None)))
    rm, ra, rb = _oracle_flux(gas, degree, kind, nfy, nfz, l[0], l[0], d_y, d_z, u, g)
    scale = np.abs(rm).max()
    assert np.abs(fm - rm).max() <= 1e-12 * scale
    assert np.abs(fa - ra).max() <= 1e-12 * scale
    assert np.abs(fb - rb).max() <= 1e-12 * scale
    # conservation: what leaves A through the interface enters B, per variable
    ia = _face_integral(fa, degree, kind, l[0], l[0])
    ib = _face_integral(fb, degree, kind, l[1], l[1])
    assert np.abs(ia - ib).max() <= 1e-12 * max(1.0, np.abs(ia).max())


def test_interface_flux_free_stream():
    """A uniform state on both sides: every face node of both sides carries the
    physical flux F(u) . e_x exactly (to rounding); the viscous part vanishes."""
    degree, n, kind = 7, 8, T.NODES_GAUSS
    nfy, nfz = [16, 12], [16, 12]
    rho, v, p = 1.2, np.array([0.3, -0.2, 0.1]), 0.9
    state = np.array([rho, *(rho * v), p / 0.4 + 0.5 * rho * v @ v])
    u = [np.broadcast_to(state, (nfy[s], nfz[s], n, n, 5)).copy() for s in (0, 1)]
    g = [np.zeros((nfy[s], nfz[s], n, n, 12)) for s in (0, 1)]
    _, fa, fb = capi.interface_flux_device(GAS_VISC, degree, kind, nfy, nfz, 2.0 / 16, 2.0 / 16, 0.481, 0.143,
                                           u[0], u[1], g[0], g[1])
    phys = np.array([rho * v[0], rho * v[0] * v[0] + p, rho * v[0] * v[1], rho * v[0] * v[2],
                     (state[4] + p) * v[0]])
    for f in (fa, fb):
        assert np.abs(f - phys).max() <= 1e-13 * np.abs(phys).max()


def test_interface_flux_conforming_limit_is_pointwise_face_flux():
    """Equal counts and zero displacement: every mortar is a whole face on both
    sides, so the interface flux is the oracle's face flux node by node."""
    degree, n, kind = 3, 4, T.NODES_GAUSS
    nf = [4, 4]
    rng = np.random.default_rng(7)
    u = [_states(rng, (4, 4, n, n)) for _ in (0, 1)]
    g = [0.1 * rng.standard_normal((4, 4, n, n, 12)) for _ in (0, 1)]
    _, fa, fb = capi.interface_flux_device(GAS_VISC, degree, kind, nf, nf, 0.5, 0.5, 0.0, 0.0, u[0], u[1], g[0], g[1])
    lib = P.oracle_lib()
    f = np.zeros(5)
    for idx in itertools.product(range(4), range(4), range(n), range(n)):
        um, up = np.ascontiguousarray(u[0][idx]), np.ascontiguousarray(u[1][idx])
        gm, gp = np.ascontiguousarray(g[0][idx]), np.ascontiguousarray(g[1][idx])
        assert lib.orc_face_flux(C_gas(GAS_VISC), P._d(um), P._d(up), 0, 0.0, P._d(gm), P._d(gp), P._d(f)) == 0
        assert np.abs(fa[idx] - f).max() <= 1e-13 * np.abs(f).max()
        assert np.abs(fb[idx] - f).max() <= 1e-13 * np.abs(f).max()


def test_interface_flux_rejects_nonphysical_state():
    degree, n = 3, 4
    u = [_states(np.random.default_rng(1), (2, 2, n, n)) for _ in (0, 1)]
    for s in (0, 1):
        u[s][..., 4] = -1.0  # negative energy -> negative Roe-averaged enthalpy
    with pytest.raises(Exception):
        capi.interface_flux_device(GAS_EULER, degree, T.NODES_GAUSS, [2, 2], [2, 2], 1.0, 1.0, 0.3, 0.0, u[0], u[1])


def _prim4(u, gas):
    v = u[..., 1:4] / u[..., :1]
    p = (gas.gamma - 1.0) * (u[..., 4] - 0.5 * (u[..., 1:4] ** 2).sum(-1) / u[..., 0])
    return np.concatenate([v, (p / (u[..., 0] * gas.R))[..., None]], axis=-1)


@pytest.mark.parametrize("kind", [T.NODES_GAUSS, T.NODES_LGL])
def test_config1_interface_lift_matches_numpy(kind):
    """The lifting mean on the configs[1] interface (N = 7): both sides' traces to
    the mortars, mean of the primitive (u, v, w, T) there (the oracle's
    run_lifting, oracle/sdg3d.cpp, after solver.cpp:597-727), projected back."""
    degree, n = 7, 8
    nfy, nfz = [16, 12], [16, 12]
    l = 2.0 / 16
    d_y, d_z = 0.37 * 1.3, 0.11 * 1.3
    rng = np.random.default_rng(31 + kind)
    u = [_states(rng, (nfy[s], nfz[s], n, n)) for s in (0, 1)]
    lm, la, lb = capi.interface_lift_device(GAS_VISC, degree, kind, nfy, nfz, l, l, d_y, d_z, u[0], u[1])
    fy, oy = _rows_ops(degree, kind, nfy[0], nfy[1], l, d_y)
    fz, oz = _rows_ops(degree, kind, nfz[0], nfz[1], l, d_z)
    ref = [np.zeros((nfy[s], nfz[s], n, n, 4)) for s in (0, 1)]
    for ky, kz in itertools.product(range(len(fy)), range(len(fz))):
        mu = [np.einsum("ki,lj,ijc->klc", oy[s][ky][0], oz[s][kz][0], u[s][fy[ky, s], fz[kz, s]]) for s in (0, 1)]
        mean = 0.5 * (_prim4(mu[0], GAS_VISC) + _prim4(mu[1], GAS_VISC))
        m = ky * len(fz) + kz
        assert np.abs(lm[m] - mean).max() <= 1e-12 * np.abs(mean).max()
        for s in (0, 1):
            ref[s][fy[ky, s], fz[kz, s]] += np.einsum("ik,jl,klc->ijc", oy[s][ky][1], oz[s][kz][1], mean)
    for got, want in zip((la, lb), ref):
        assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()


def test_interface_lift_uniform_state_is_exact():
    degree, n = 5, 6
    nfy, nfz = [16, 12], [16, 12]
    state = np.array([1.2, 0.36, -0.24, 0.12, 0.9 / 0.4 + 0.5 * 1.2 * 0.14])
    u = [np.broadcast_to(state, (nfy[s], nfz[s], n, n, 5)).copy() for s in (0, 1)]
    _, la, lb = capi.interface_lift_device(GAS_VISC, degree, T.NODES_GAUSS, nfy, nfz, 0.125, 0.125, 0.481, 0.143,
                                           u[0], u[1])
    want = _prim4(state, GAS_VISC)
    for f in (la, lb):
        assert np.abs(f - want).max() <= 1e-13 * np.abs(want).max()


def test_equal_counts_flux_is_reference_mortar_chain():
    """Equal counts, displacement along y only: the interface flux equals the
    reference's mortar chain built from the oracle-restated pieces: the static side
    A's halves fwd(sigma)[sub] of face i, the moving side B's fwd(-sigma)[1 - sub] of
    face moving_index(i, n_delta, sub) (mortar.cpp:136-150), face_numerical_flux at
    the mortar nodes, and bwd(sigma)[sub] / bwd(-sigma)[1 - sub] back (solver.cpp:156-176)."""
    degree, n, kind = 3, 4, T.NODES_GAUSS
    nf, l, d = 4, 0.5, 0.3
    rng = np.random.default_rng(11)
    u = [_states(rng, (nf, nf, n, n)) for _ in (0, 1)]
    g = [0.1 * rng.standard_normal((nf, nf, n, n, 12)) for _ in (0, 1)]
    _, fa, fb = capi.interface_flux_device(GAS_VISC, degree, kind, [nf, nf], [nf, nf], l, l, d, 0.0, u[0], u[1],
                                           g[0], g[1])
    _, n_delta, s_delta = P.oracle_displacement(d, l, nf)
    sigma = 2.0 * s_delta - 1.0
    fwd_a, bwd_a = P.oracle_mortar_ops(degree, kind, sigma)
    fwd_b, bwd_b = P.oracle_mortar_ops(degree, kind, -sigma)
    lib = P.oracle_lib()
    ea, eb = np.zeros_like(fa), np.zeros_like(fb)
    f = np.zeros(5)
    for i in range(nf):
        for sub in (0, 1):
            j = lib.orc_moving_index(i, n_delta, sub, nf)
            mu = [np.einsum("ki,zijc->zkjc", fwd_a[sub], u[0][i]), np.einsum("ki,zijc->zkjc", fwd_b[1 - sub], u[1][j])]
            mg = [np.einsum("ki,zijc->zkjc", fwd_a[sub], g[0][i]), np.einsum("ki,zijc->zkjc", fwd_b[1 - sub], g[1][j])]
            fm = np.zeros((nf, n, n, 5))
            for idx in itertools.product(range(nf), range(n), range(n)):
                args = [np.ascontiguousarray(x[idx]) for x in (mu[0], mu[1], mg[0], mg[1])]
                assert lib.orc_face_flux(C_gas(GAS_VISC), P._d(args[0]), P._d(args[1]), 0, 0.0, P._d(args[2]),
                                         P._d(args[3]), P._d(f)) == 0
                fm[idx] = f
            ea[i] += np.einsum("ik,zkjc->zijc", bwd_a[sub], fm)
            eb[j] += np.einsum("ik,zkjc->zijc", bwd_b[1 - sub], fm)
    scale = np.abs(ea).max()
    assert np.abs(fa - ea).max() <= 1e-12 * scale
    assert np.abs(fb - eb).max() <= 1e-12 * scale
