"""Non-matching sliding interfaces (BASELINE configs[1]) on the device: the interval
kernel against the host row construction (bitwise), and the tensor-product mortar
transfer of a 16 x 16 / 12 x 12 interface against a numpy assembly of the same
host operators, with its conservation and constant-preservation properties."""
import itertools

import numpy as np
import pytest

from oracle import pyoracle as P
from paper_2008_04356_b200 import capi
from paper_2008_04356_b200 import types as T

pytestmark = pytest.mark.gpu

ROWS = [(4, 4), (16, 12), (12, 16), (5, 7), (1, 1), (3, 1), (1, 3), (8, 8), (7, 5), (16, 16), (600, 451)]


@pytest.mark.parametrize("n_a,n_b", ROWS)
def test_device_intervals_match_host_bitwise(n_a, n_b):
    rng = np.random.default_rng(n_a + 7 * n_b)
    l_a = 2.0 / n_a
    for d in list(rng.uniform(-5.0, 5.0, 10)) + [0.0, 0.37, 0.11, l_a, -2.0, 2.0 / n_b, 1e-17]:
        hf, hr = capi.mortar_intervals(n_a, n_b, l_a, d)
        df, dr = capi.mortar_intervals(n_a, n_b, l_a, d, device=True)
        assert np.array_equal(hf, df) and np.array_equal(hr, dr)


def _nodes(degree, kind):
    x, w = np.zeros(degree + 1), np.zeros(degree + 1)
    assert P.oracle_lib().orc_nodes(degree, kind, P._d(x), P._d(w)) == 0
    return x, w


def _numpy_transfer(degree, kind, nfy, nfz, l_y, l_z, d_y, d_z, src, frm):
    to = 1 - frm
    n = degree + 1
    rows = [capi.mortar_intervals(nfy[0], nfy[1], l_y, d_y), capi.mortar_intervals(nfz[0], nfz[1], l_z, d_z)]

    def ops(r):
        s = (0, 1) if frm == 0 else (2, 3)
        t = (0, 1) if to == 0 else (2, 3)
        return [(capi.subrange_ops(degree, kind, rr[s[0]], rr[s[1]])[0],
                 capi.subrange_ops(degree, kind, rr[t[0]], rr[t[1]])[1]) for rr in r]

    oy, oz = ops(rows[0][1]), ops(rows[1][1])
    fy, fz = rows[0][0], rows[1][0]
    mortar = np.zeros((len(fy) * len(fz), n, n, src.shape[-1]))
    dst = np.zeros((nfy[to], nfz[to], n, n, src.shape[-1]))
    for ky, kz in itertools.product(range(len(fy)), range(len(fz))):
        m = np.einsum("ki,lj,ijc->klc", oy[ky][0], oz[kz][0], src[fy[ky, frm], fz[kz, frm]])
        mortar[ky * len(fz) + kz] = m
        dst[fy[ky, to], fz[kz, to]] += np.einsum("ik,jl,klc->ijc", oy[ky][1], oz[kz][1], m)
    return mortar, dst


@pytest.mark.parametrize("kind", [T.NODES_GAUSS, T.NODES_LGL])
@pytest.mark.parametrize("frm", [0, 1])
def test_config1_interface_transfer(kind, frm):
    """configs[1]: 16 x 16 faces (A, lower block) against 12 x 12 (B, upper block) on
    [0, 2]^2, N = 7, displaced by (0.37, 0.11) t at t = 1.3 (an oblique, non-aligned
    position); five conserved variables per node."""
    degree, n = 7, 8
    nfy, nfz = [16, 12], [16, 12]
    l_y = l_z = 2.0 / 16
    d_y, d_z = 0.37 * 1.3, 0.11 * 1.3
    rng = np.random.default_rng(2008043561 + frm)
    src = rng.standard_normal((nfy[frm], nfz[frm], n, n, 5))
    mortar, dst = capi.interface_project_device(degree, kind, nfy, nfz, l_y, l_z, d_y, d_z, src, frm)
    ref_m, ref_d = _numpy_transfer(degree, kind, nfy, nfz, l_y, l_z, d_y, d_z, src, frm)
    assert np.abs(mortar - ref_m).max() <= 1e-13 * np.abs(ref_m).max()
    assert np.abs(dst - ref_d).max() <= 1e-13 * np.abs(ref_d).max()
    # conservation of the integral over the interface, per variable
    _, w = _nodes(degree, kind)
    h = [(2.0 / 16) ** 2 / 4, (2.0 / 12) ** 2 / 4]
    int_src = h[frm] * np.einsum("i,j,abijc->c", w, w, src)
    int_dst = h[1 - frm] * np.einsum("i,j,abijc->c", w, w, dst)
    assert np.abs(int_src - int_dst).max() < 1e-12
    # constants are carried exactly (to rounding)
    _, ones = capi.interface_project_device(degree, kind, nfy, nfz, l_y, l_z, d_y, d_z,
                                            np.ones((nfy[frm], nfz[frm], n, n, 1)), frm)
    assert np.abs(ones - 1.0).max() < 1e-13


def test_equal_counts_transfer_is_reference_mortar_chain():
    """Equal counts, displacement along y only: every mortar is the reference's
    hanging-node pair along y times the identity along z, so the A -> B transfer of a
    face field equals applying the reference's (oracle-restated) fwd/bwd operators."""
    degree, n, kind = 3, 4, T.NODES_GAUSS
    nf = 4
    l = 2.0 / nf
    d = 0.3
    rng = np.random.default_rng(5)
    src = rng.standard_normal((nf, nf, n, n, 2))
    _, dst = capi.interface_project_device(degree, kind, [nf, nf], [nf, nf], l, l, d, 0.0, src, 0)
    _, n_delta, s_delta = P.oracle_displacement(d, l, nf)
    sigma = 2.0 * s_delta - 1.0
    fa, _ = P.oracle_mortar_ops(degree, kind, sigma)     # static side, halves (lower, upper)
    _, bb = P.oracle_mortar_ops(degree, kind, -sigma)    # moving side
    expect = np.zeros_like(dst)
    for i in range(nf):
        for sub in (0, 1):
            j = P.oracle_lib().orc_moving_index(i, n_delta, sub, nf)
            m = np.einsum("ki,zijc->zkjc", fa[sub], src[i])
            expect[j] += np.einsum("ik,zkjc->zijc", bb[1 - sub], m)   # moving side swaps halves
    assert np.abs(dst - expect).max() <= 1e-13 * np.abs(expect).max()
