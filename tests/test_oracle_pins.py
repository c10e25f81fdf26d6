"""Pins the 3D CPU oracle (oracle/sdg3d.cpp) to the reference.

* against the reference's own golden vectors and known-answer tests
  (proj/tests/test_partition.cpp, test_mortar.cpp, test_mesh.cpp, test_solver.cpp);
* against the UNMODIFIED reference library (oracle/_ref) when it is built here,
  through the z-invariant embedding of its 2D problems;
* against the committed reference fixtures in tests/golden/ (made by
  tests/golden/make_golden.py), which do not need /root/reference.
"""
import os

import numpy as np
import pytest

import embed
from conftest import rel_linf
from oracle import pyoracle as P
from paper_2008_04356_b200 import types as T

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
needs_ref = pytest.mark.skipif(not P.ref_available(), reason="oracle/_ref not built (no /root/reference)")
BANDS3 = [(2, 1.0, 0.0), (2, 1.0, 1.0), (2, 1.0, 0.0)]


# ---------------------------------------------------------------- golden vectors
def test_appendix_a_worked_example():
    """proj/tests/test_partition.cpp:110-150 (Appendix A)."""
    faces = [(5, 4, 1), (6, 4, 2), (7, 5, 1), (8, 3, 2), (9, 3, 1)]
    ranks = np.full((3, 6), 9, dtype=np.int32)
    for (ip, iq, r) in [(1, 1, 7), (2, 1, 7), (3, 1, 4), (4, 1, 4), (1, 2, 7), (2, 2, 4), (3, 2, 4), (4, 2, 4)]:
        ranks[iq, ip] = r
    out = P.oracle_pairing(faces, 6, 3, ranks, 1, True, False, 0)
    cols = out["cols"]
    assert list(cols[:, 0]) == [4, 4, 4, 4, 4, 4, 7, 7, 7, 7]
    assert list(cols[:, 2]) == [3, 4, 4, 4, 5, 5, 3, 3, 3, 4]
    assert list(cols[:, 3]) == [2, 1, 2, 2, 1, 1, 1, 1, 2, 1]
    assert list(cols[:, 4]) == [1, 1, 0, 1, 0, 1, 0, 1, 0, 0]
    assert list(cols[:, 5]) == [8, 5, 6, 6, 7, 7, 9, 9, 8, 5]
    assert out["face_lo"] == 5
    assert list(out["m"][0] + 1) == [10, 3, 5, 9, 7]
    assert list(out["m"][1] + 1) == [2, 4, 6, 1, 8]
    assert out["sched"].tolist() == [[4, 0, 6], [7, 6, 4]]
    assert out["self_entry"][2] == 0


def test_pairing_idempotent_and_conforming_order():
    """proj/tests/test_partition.cpp:152-182."""
    ranks = np.full(4, 3, dtype=np.int32)
    out = P.oracle_pairing([(0, 2, 0), (1, 0, 0), (2, 3, 0), (3, 1, 0)], 4, 1, ranks, 0, True, True, 0)
    cols = out["cols"]
    assert len(cols) == 4 and set(cols[:, 4]) == {1}
    assert all(cols[i - 1, 2] < cols[i, 2] for i in range(1, 4))


def test_both_endpoints_agree():
    """Stamp check, proj/tests/test_partition.cpp:184-227."""
    nf, nd = 8, 3
    faces = [(i, i, 0) for i in range(nf)]
    st = P.oracle_pairing(faces, nf, 1, np.ones(nf, np.int32), nd, True, False, 0)
    mv = P.oracle_pairing(faces, nf, 1, np.zeros(nf, np.int32), nd, False, False, 1)
    assert st["sched"].tolist() == [[1, 0, 16]] and mv["sched"].tolist() == [[0, 0, 16]]
    assert np.array_equal(st["cols"][:, 2:5], mv["cols"][:, 2:5])


def test_index_relation_known_answers():
    """proj/tests/test_mortar.cpp:446-459."""
    L = P.oracle_lib()
    assert L.orc_moving_index(3, 1, 0, 100) == 1
    assert L.orc_moving_index(3, 1, 1, 100) == 2
    assert L.orc_moving_index(7, 0, 1, 100) == 7
    assert L.orc_moving_index(0, 2, 0, 6) == 3
    rng = np.random.default_rng(53)
    for _ in range(200):
        i, n = int(rng.integers(0, 100)), int(rng.integers(0, 301))
        for sub in (0, 1):
            assert L.orc_static_index(L.orc_moving_index(i, n, sub, 100), n, sub, 100) == i


def test_displacement_known_answers():
    """proj/tests/test_mesh.cpp:70-98."""
    d, nd, sd = P.oracle_displacement(0.4, 1.0, 100)
    assert nd == 0 and abs(sd - 0.4) < 1e-13
    d, nd, sd = P.oracle_displacement(1.1, 1.0, 100)
    assert nd == 1 and abs(sd - 0.1) < 1e-12
    d, nd, sd = P.oracle_displacement(1.0, 1.0, 100)
    assert nd == 1 and sd == 0.0
    for delta in (0.07, 0.5, 1.23, 1.999):
        a = P.oracle_displacement(delta, 1.0 / 3.0, 6)
        b = P.oracle_displacement(delta + 6 * (1.0 / 3.0), 1.0 / 3.0, 6)
        assert a[1] == b[1] and abs(a[2] - b[2]) < 1e-10


def test_mortar_operator_identities():
    """proj/tests/test_mortar.cpp:49-169: identity at sigma=-1, N=1 sigma=0 values,
    projection == interpolation, partition of unity, round trip, conservation."""
    f, b = P.oracle_mortar_ops(4, T.NODES_LGL, -1.0)
    assert np.allclose(f[1], np.eye(5), atol=1e-12) and np.allclose(b[1], np.eye(5), atol=1e-12)
    f, _ = P.oracle_mortar_ops(1, T.NODES_LGL, 0.0)
    assert np.allclose(f[1], [[0.5, 0.5], [0.0, 1.0]], atol=1e-13)
    with pytest.raises(T.ConfigError):
        P.oracle_mortar_ops(4, T.NODES_LGL, 1.0)
    rng = np.random.default_rng(23)
    for deg in range(1, 9):
        x = np.zeros(deg + 1)
        w = np.zeros(deg + 1)
        P.oracle_lib().orc_nodes(deg, T.NODES_LGL, P._d(x), P._d(w))
        for _ in range(5):
            s = float(rng.uniform(-0.999, 0.999))
            f, b = P.oracle_mortar_ops(deg, T.NODES_LGL, s)
            coef = rng.uniform(-1, 1, deg + 1)
            nodal = np.polyval(coef, x)
            lo = f[0] @ nodal
            up = f[1] @ nodal
            assert np.allclose(lo, np.polyval(coef, -1 + 0.5 * (1 + s) * (x + 1)), rtol=1e-12, atol=1e-12)
            assert np.allclose(up, np.polyval(coef, s + 0.5 * (1 - s) * (x + 1)), rtol=1e-12, atol=1e-12)
            assert np.allclose(b[0] @ lo + b[1] @ up, nodal, atol=1e-11)
            assert np.allclose(b[0] @ np.full(deg + 1, 4.2) + b[1] @ np.full(deg + 1, 4.2), 4.2, atol=1e-12)


def test_mortar_operators_match_reference_fixture():
    z = np.load(os.path.join(GOLDEN, "ref_mortar_ops.npz"))
    for kind in (T.NODES_LGL, T.NODES_GAUSS):
        for deg in range(1, 8):
            for i, s in enumerate(z["sigma"]):
                f, b = P.oracle_mortar_ops(deg, kind, float(s))
                assert np.abs(f - z[f"fwd_{kind}_{deg}"][i]).max() <= 2e-15
                assert np.abs(b - z[f"bwd_{kind}_{deg}"][i]).max() <= 2e-15


@needs_ref
@pytest.mark.parametrize("kind", [T.NODES_LGL, T.NODES_GAUSS])
def test_nodes_and_basis_bit_exact_with_reference(kind):
    for deg in range(1, 9):
        n = deg + 1
        xo, wo, xr, wr = (np.zeros(n) for _ in range(4))
        P.oracle_lib().orc_nodes(deg, kind, P._d(xo), P._d(wo))
        P.ref_lib().ref_nodes(deg, kind, P._d(xr), P._d(wr))
        assert np.array_equal(xo, xr) and np.array_equal(wo, wr)
        Do, flo, fro, Dr, flr, frr = np.zeros(n * n), np.zeros(n), np.zeros(n), np.zeros(n * n), np.zeros(n), np.zeros(n)
        P.oracle_lib().orc_basis(deg, kind, P._d(Do), P._d(flo), P._d(fro))
        P.ref_lib().ref_basis(deg, kind, P._d(Dr), P._d(flr), P._d(frr))
        assert np.array_equal(Do, Dr) and np.array_equal(flo, flr) and np.array_equal(fro, frr)


@needs_ref
def test_displacement_and_pairing_bit_exact_with_reference():
    rng = np.random.default_rng(7)
    for _ in range(500):
        l, nf = float(rng.uniform(0.05, 1.0)), int(rng.integers(1, 40))
        delta = float(rng.uniform(-3, 3)) * l * nf
        assert P.oracle_displacement(delta, l, nf) == P.ref_displacement(delta, l, nf)
    for trial in range(30):
        n_par, n_perp = int(rng.integers(2, 9)), int(rng.integers(1, 4))
        ranks = rng.integers(0, 5, size=(n_perp, n_par)).astype(np.int32)
        sel = rng.permutation(n_par * n_perp)[: int(rng.integers(1, n_par * n_perp + 1))]
        faces = [(100 + i, int(s % n_par), int(s // n_par)) for i, s in enumerate(sel)]
        for on_static in (True, False):
            for conf in (True, False):
                nd = int(rng.integers(0, n_par))
                a = P.oracle_pairing(faces, n_par, n_perp, ranks, nd, on_static, conf, 2)
                b = P.ref_pairing(faces, n_par, n_perp, ranks, nd, on_static, conf, 2)
                for k in a:
                    assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), (trial, k)


# ---------------------------------------------------------------- z-invariant embedding
def _embedded(name):
    z = np.load(os.path.join(GOLDEN, f"ref2d_{name}.npz"))
    return z


FIXT = {
    # name: (bands, ny, degree, kind, mu, periodic_x, case)
    "dw_lgl3_inv": (BANDS3, 6, 3, T.NODES_LGL, 0.0, True, "density_wave"),
    "dw_gauss3_visc": (BANDS3, 6, 3, T.NODES_GAUSS, 1e-3, True, "density_wave"),
    "dw_gauss5_visc_dirichlet": ([(2, 1.0, 0.0), (2, 1.0, 0.5)], 2, 5, T.NODES_GAUSS, 1e-3, False, "density_wave"),
    "fs_lgl4_inv": (BANDS3, 6, 4, T.NODES_LGL, 0.0, True, "freestream"),
}


@pytest.mark.parametrize("name", sorted(FIXT))
def test_oracle_embeds_reference_fixture(name):
    bands, ny, deg, kind, mu, px, case = FIXT[name]
    z = _embedded(name)
    nz = 2
    o = P.Oracle3D(embed.mesh3d(bands, ny, nz, periodic_x=px), T.solver_config(deg, kind, mu=mu, case=embed.case3d(case)))
    o.set_initial_condition(0.0)
    n = deg + 1
    u0 = o.field()
    assert embed.max_layer_diff(u0, z["u0"], bands, ny, nz, n) == 0.0
    r = o.compute_residual(float(z["t_res"]), u0)
    scale = max(np.abs(z["residual"]).max(), 1.0)
    assert embed.max_layer_diff(r, z["residual"], bands, ny, nz, n) <= 1e-12 * scale
    assert np.abs(embed.w_component(r)).max() <= 1e-12 * scale
    o = P.Oracle3D(embed.mesh3d(bands, ny, nz, periodic_x=px), T.solver_config(deg, kind, mu=mu, case=embed.case3d(case)))
    o.set_initial_condition(0.0)
    o.step(float(z["dt"]), int(z["n_steps"]))
    u = o.field()
    assert embed.max_layer_diff(u, z["u_end"], bands, ny, nz, n) <= 1e-12 * np.abs(z["u_end"]).max()
    assert o.total_rebuilds() == int(z["rebuilds"])


@needs_ref
@pytest.mark.parametrize("kind", [T.NODES_LGL, T.NODES_GAUSS])
@pytest.mark.parametrize("mu", [0.0, 1e-3])
def test_oracle_embeds_live_reference(kind, mu):
    ny, nz, deg = 6, 2, 3
    ref = P.Ref2D(P.ref_spec(BANDS3, ny, deg, kind, mu=mu, case="density_wave"))
    o = P.Oracle3D(embed.mesh3d(BANDS3, ny, nz), T.solver_config(deg, kind, mu=mu, case=embed.case3d("density_wave")))
    o.set_initial_condition(0.0)
    u0 = o.field()
    n = deg + 1
    for t in (0.0, 0.05, 1.0 / 3.0, 0.99):
        r2 = ref.residual(0.0, t)
        assert embed.max_layer_diff(o.compute_residual(t, u0), r2, BANDS3, ny, nz, n) <= 1e-12 * np.abs(r2).max()
    if mu > 0:
        g2 = ref.gradients(0.0, 0.21)
        g3 = o.compute_gradients(0.21, u0).reshape(-1, n, n, n, 12)
        for iz in range(nz):
            layer = []
            g = 0
            for nx, _, _ in BANDS3:
                for e in range(nx * ny):
                    layer.append(g3[(g + e) * nz + iz][:, :, 0][..., [0, 1, 3, 4, 9, 10]])
                g += nx * ny
            assert np.abs(np.array(layer).reshape(-1) - g2).max() <= 1e-11 * np.abs(g2).max()


@needs_ref
def test_rebuild_count_matches_reference():
    """proj/tests/test_solver.cpp:326-336: 16 rebuilds for 150 steps of 0.005."""
    ref = P.Ref2D(P.ref_spec(BANDS3, 6, 2, T.NODES_LGL, case="freestream"))
    _, _, reb = ref.steps(0.0, 0.005, 150)
    assert reb == 16
    o = P.Oracle3D(embed.mesh3d(BANDS3, 6, 1), T.solver_config(2, T.NODES_LGL, case=embed.case3d("freestream")))
    o.set_initial_condition(0.0)
    o.step(0.005, 150)
    assert o.total_rebuilds() == 16


@needs_ref
def test_reference_reproduces_its_shipped_freestream_report():
    """proj/out/freestream/report.csv:2 — dt and Linf(rho) of the shipped run."""
    cfg = "/root/reference/proj/configs/freestream.cfg"
    if not os.path.exists(cfg):
        pytest.skip("reference configs not present")
    out = np.zeros(12)
    code = P.ref_lib().ref_run_case(cfg.encode(), P._d(out))
    assert code == 0
    assert out[2] == 0.006437725221731195
    assert out[1] == 200
    assert abs(out[7] - 1.998401444325282e-15) < 1e-30


# ---------------------------------------------------------------- 3D properties
def test_freestream_preservation_3d_sliding():
    """3D form of proj/tests/test_solver.cpp:86-92 (7 offsets)."""
    mesh = T.mesh_spec(BANDS3, ny=6, nz=3, depth=1.0)
    for kind in (T.NODES_LGL, T.NODES_GAUSS):
        o = P.Oracle3D(mesh, T.solver_config(3, kind, mu=1e-3, case=T.freestream(v=(1.0, 0.5, 0.25))))
        o.set_initial_condition(0.0)
        for t in (0.0, 0.05, 1.0 / 3.0, 0.37, 0.99, 2.0, 5.0 + 1e-9):
            assert np.abs(o.compute_residual(t)).max() < 1e-12


def test_conservation_3d_sliding():
    """3D form of proj/tests/test_solver.cpp:282-299."""
    mesh = T.mesh_spec(BANDS3, ny=6, nz=2, depth=1.0)
    o = P.Oracle3D(mesh, T.solver_config(3, T.NODES_LGL, case=T.density_wave(a=(1.0, 1.0, 0.5))))
    o.set_initial_condition(0.0)
    before = o.mass_energy()
    o.step(o.suggest_dt(0.4), 10)
    after = o.mass_energy()
    assert np.all(np.abs(after - before) / np.abs(before) < 1e-12)


def test_positivity_violation_raises_in_oracle():
    o = P.Oracle3D(T.mesh_spec(BANDS3, ny=3, nz=1), T.solver_config(2, T.NODES_LGL, case=T.freestream()))
    o.set_initial_condition(0.0)
    u = o.field()
    u[0] = -1.0
    o.set_state(u)
    with pytest.raises(T.InvalidStateError):
        o.step(1e-6)


def test_invalid_configs_rejected():
    with pytest.raises(T.ConfigError):
        P.Oracle3D(T.mesh_spec([(2, 1.0, 0.5), (2, 1.0, 1.0)], ny=2, nz=1), T.solver_config(2))
    with pytest.raises(T.ConfigError):
        P.Oracle3D(T.mesh_spec([(2, 1.0, -1.0), (2, 1.0, 0.0)], ny=2, nz=1), T.solver_config(2))
    with pytest.raises(T.ConfigError):
        P.Oracle3D(T.mesh_spec([(2, 1.0, 0.0)], ny=2, nz=1), T.solver_config(0))
