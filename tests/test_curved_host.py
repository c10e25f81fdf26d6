"""Host-side curved metrics of the product (csrc/host.cpp compute_metrics, through
the C-ABI sdg_metrics_host; no GPU) against the oracle's independent
restatement (oracle/sdg3d.cpp build_metrics), and their rank independence."""
import numpy as np
import pytest

from oracle import pyoracle as P
from paper_2008_04356_b200 import capi
from paper_2008_04356_b200 import types as T

BANDS3 = [(2, 1.0, 0.0), (2, 1.0, 1.0), (2, 1.0, 0.0)]


@pytest.mark.parametrize("kind", [T.NODES_GAUSS, T.NODES_LGL])
@pytest.mark.parametrize("degree", [1, 3, 5, 7])
def test_product_metrics_match_oracle(kind, degree):
    mesh = T.mesh_spec(BANDS3, ny=4, nz=3, depth=1.0, warp=0.25, periodic=(False, True, True))
    met, fmet = capi.metrics_host(mesh, degree, kind)
    o = P.Oracle3D(mesh, T.solver_config(degree, kind, case=T.freestream()))
    omet, ofmet = o.metrics()
    assert met.shape == omet.shape and fmet.shape == ofmet.shape
    assert np.abs(met - omet).max() <= 1e-15 * np.abs(omet).max()
    assert np.abs(fmet - ofmet).max() <= 1e-15 * np.abs(ofmet).max()


def test_face_slots_hold_identical_bits():
    """Both slots of every conforming face (incl. periodic wrap) carry the same
    normal and sJ, so both elements evaluate the face flux identically."""
    mesh = T.mesh_spec([(3, 1.0, 0.0), (2, 0.5, 0.0)], ny=3, nz=2, warp=0.3)  # two static bands: conforming
    met, fmet = capi.metrics_host(mesh, 3, T.NODES_GAUSS)
    nx = [3, 2]
    off = [0, 3 * 3 * 2]

    def gid(b, ix, iy, iz):
        return off[b] + (ix * 3 + iy) * 2 + iz

    checked = 0
    for b in range(2):
        for ix in range(nx[b]):
            for iy in range(3):
                for iz in range(2):
                    g = gid(b, ix, iy, iz)
                    # +y and +z neighbours (periodic)
                    assert np.array_equal(fmet[g, 3], fmet[gid(b, ix, (iy + 1) % 3, iz), 2])
                    assert np.array_equal(fmet[g, 5], fmet[gid(b, ix, iy, (iz + 1) % 2), 4])
                    # +x neighbour: same band, next band, or the periodic wrap
                    if ix + 1 < nx[b]:
                        nb = gid(b, ix + 1, iy, iz)
                    else:
                        nb = gid((b + 1) % 2, 0, iy, iz)
                    assert np.array_equal(fmet[g, 1], fmet[nb, 0])
                    checked += 3
    assert checked == 3 * 30


def test_metrics_independent_of_rank_count():
    mesh = T.mesh_spec(BANDS3, ny=4, nz=3, depth=1.0, warp=0.2, partition=T.PARTITION_SFC)
    met1, fmet1 = capi.metrics_host(mesh, 3, T.NODES_GAUSS)
    for n_ranks in (2, 3, 5):
        for r in range(n_ranks):
            gids = np.array(capi.plan(mesh, n_ranks, r)["elements"])
            met, fmet = capi.metrics_host(mesh, 3, T.NODES_GAUSS, n_ranks, r)
            assert np.array_equal(met, met1[gids])
            assert np.array_equal(fmet, fmet1[gids])


def test_invalid_mapping_rejected():
    mesh = T.mesh_spec(BANDS3, ny=2, nz=2, warp=0.2)
    mesh.mapping = 7
    with pytest.raises(T.ConfigError):
        capi.metrics_host(mesh, 2, T.NODES_GAUSS)
    with pytest.raises(T.ConfigError):
        capi.metrics_host(T.mesh_spec(BANDS3, ny=4, nz=3, warp=5.0), 3, T.NODES_GAUSS)  # folded mapping
    with pytest.raises(T.ConfigError):
        capi.metrics_host(T.mesh_spec(BANDS3, ny=4, nz=3), 3, T.NODES_GAUSS)  # affine: no stored metrics


@pytest.mark.parametrize("kind", [T.NODES_GAUSS, T.NODES_LGL])
@pytest.mark.parametrize("degree", [2, 5])
@pytest.mark.parametrize("warp", [None, 0.1])
def test_product_annulus_metrics_match_oracle(kind, degree, warp):
    """SDG_MAP_ANNULUS: metrics plus the contravariant grid velocity (per node) and
    (vg / omega) . n (per face node) of the product host agree with the oracle."""
    mesh = T.annulus_spec([(2, 1.0, 0.0), (2, 1.0, 0.8)], 8, 2, 0.5, 1.0, warp=warp)
    met, fmet = capi.metrics_host(mesh, degree, kind)
    o = P.Oracle3D(mesh, T.solver_config(degree, kind, case=T.freestream()))
    omet, ofmet = o.metrics()
    assert met.shape == omet.shape and met.shape[2] == 13 and fmet.shape[3] == 6
    assert np.abs(met - omet).max() <= 1e-15 * np.abs(omet).max()
    assert np.abs(fmet - ofmet).max() <= 1e-15 * np.abs(ofmet).max()
    for r in range(3):
        gids = np.array(capi.plan(mesh, 3, r)["elements"])
        m3, f3 = capi.metrics_host(mesh, degree, kind, 3, r)
        assert np.array_equal(m3, met[gids]) and np.array_equal(f3, fmet[gids])


def test_sector_metrics_rotate_across_the_seam():
    """Periodic annulus sector: the two slots of a seam face are not copied from one side; each
    side's face metrics are its own, and (invariant curl form) they are exact rotations of each
    other by the sector angle: n(theta = 0) = R(-alpha) n(theta = alpha)."""
    alpha = np.pi / 4
    mesh = T.annulus_spec([(2, 1.0, 0.0), (2, 1.0, 0.8)], 3, 2, 0.5, 1.0, theta_span=alpha)
    assert mesh.periodic_y == 1
    met, fmet = capi.metrics_host(mesh, 3, T.NODES_GAUSS)
    c, s = np.cos(-alpha), np.sin(-alpha)
    n_theta, n_r = 3, 2
    for b in range(2):
        for ix in range(2):
            for ir in range(n_r):
                lo = b * 2 * n_theta * n_r + (ix * n_theta + 0) * n_r + ir            # theta row 0, side YM (2)
                hi = b * 2 * n_theta * n_r + (ix * n_theta + n_theta - 1) * n_r + ir  # last row, side YP (3)
                n_lo, n_hi = fmet[lo, 2, :, :3], fmet[hi, 3, :, :3]
                rot = np.stack([n_hi[:, 0], c * n_hi[:, 1] + s * n_hi[:, 2], -s * n_hi[:, 1] + c * n_hi[:, 2]], axis=1)
                assert np.abs(rot - n_lo).max() < 1e-14
                assert np.abs(fmet[lo, 2, :, 3] - fmet[hi, 3, :, 3]).max() < 1e-15 * fmet[lo, 2, :, 3].max()
