"""ctypes mirrors of include/sdg_types.h plus builders for the problem description.

The builders follow the reference's setup vocabulary (bands, ny/nz, band_vg,
case kinds) — /root/reference/proj/src/config.cpp:132-212 maps the same keys
into MeshSpec/CaseDef.
"""
from __future__ import annotations

import ctypes as C
import math

SDG_MAX_BANDS = 16
NVARS = 5
NGRAD = 12
TUPLE_INTS = 7

OK, ERR_CONFIG, ERR_INVALID_STATE, ERR_PROTOCOL, ERR_CUDA, ERR_NCCL = range(6)
NODES_LGL, NODES_GAUSS = 0, 1
MORTARS_AUTO, MORTARS_TENSOR = 0, 1
CASE_FREESTREAM, CASE_DENSITY_WAVE, CASE_VORTEX, CASE_TGV, CASE_SWIRL = range(5)


class BandSpec(C.Structure):
    _fields_ = [("nx", C.c_int), ("width_frac", C.c_double), ("vg_y", C.c_double), ("ny", C.c_int), ("nz", C.c_int),
                ("vg_z", C.c_double)]


class MeshSpec(C.Structure):
    _fields_ = [
        ("x0", C.c_double), ("y0", C.c_double), ("z0", C.c_double),
        ("width", C.c_double), ("height", C.c_double), ("depth", C.c_double),
        ("ny", C.c_int), ("nz", C.c_int),
        ("n_bands", C.c_int),
        ("bands", BandSpec * SDG_MAX_BANDS),
        ("periodic_x", C.c_int), ("periodic_y", C.c_int), ("periodic_z", C.c_int),
        ("partition", C.c_int),
        ("mapping", C.c_int), ("warp", C.c_double),
        ("mortars", C.c_int), ("pad_", C.c_int),
    ]


class Gas(C.Structure):
    _fields_ = [("gamma", C.c_double), ("R", C.c_double), ("mu", C.c_double), ("Pr", C.c_double)]


class Case(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("fs_rho", C.c_double), ("fs_v", C.c_double * 3), ("fs_p", C.c_double),
        ("dw_alpha", C.c_double), ("dw_a", C.c_double * 3), ("dw_k", C.c_double * 3), ("dw_p0", C.c_double),
        ("vx_eps", C.c_double), ("vx_rc", C.c_double), ("vx_rho_inf", C.c_double), ("vx_v_inf", C.c_double),
        ("vx_theta", C.c_double), ("vx_ma_inf", C.c_double), ("vx_center", C.c_double * 2),
        ("tgv_rho0", C.c_double), ("tgv_v0", C.c_double), ("tgv_mach", C.c_double),
        ("sw_omega", C.c_double),
        ("pt_modes", C.c_int), ("pt_coords", C.c_int), ("pt_amp", C.c_double),
        ("pt_x0", C.c_double * 3), ("pt_len", C.c_double * 3), ("pt_adv", C.c_double * 3),
        ("pt_k", (C.c_double * 3) * 8), ("pt_a", C.c_double * 8), ("pt_phi", C.c_double * 8),
    ]


class SolverConfig(C.Structure):
    _fields_ = [("degree", C.c_int), ("node_kind", C.c_int), ("gas", Gas), ("flow_case", Case)]


class SdgError(RuntimeError):
    code = ERR_CONFIG


class ConfigError(SdgError):
    """Mirror of sdg::ConfigError (proj/src/errors.hpp:9-11)."""
    code = ERR_CONFIG


class InvalidStateError(SdgError):
    """Mirror of sdg::InvalidStateError (proj/src/errors.hpp:14-16)."""
    code = ERR_INVALID_STATE


class ProtocolError(SdgError):
    """Mirror of sdg::ProtocolError (proj/src/errors.hpp:19-21)."""
    code = ERR_PROTOCOL


class DeviceError(SdgError):
    code = ERR_CUDA


ERRORS = {ERR_CONFIG: ConfigError, ERR_INVALID_STATE: InvalidStateError, ERR_PROTOCOL: ProtocolError,
          ERR_CUDA: DeviceError, ERR_NCCL: DeviceError}


def raise_for(code: int, msg: str) -> None:
    if code != OK:
        raise ERRORS.get(code, SdgError)(msg)


PARTITION_LEX, PARTITION_SFC, PARTITION_YSLAB = 0, 1, 2
MAP_BOX, MAP_WARP, MAP_ANNULUS = 0, 1, 2


def mesh_spec(bands, ny, nz, width=2.0, height=2.0, depth=2.0, x0=0.0, y0=0.0, z0=0.0,
              periodic=(True, True, True), partition=PARTITION_LEX, warp=None, mapping=None,
              mortars=0) -> MeshSpec:
    """bands: list of (nx, width_frac, vg_y[, ny, nz, vg_z]) tuples, stacked along x
    (ny / nz = 0: the mesh-wide counts; bands with other counts meet at a
    non-matching sliding interface; vg_z: slide along z).  warp: None for
    affine hexahedra, else the amplitude of the curved SDG_MAP_WARP mapping
    (include/sdg_types.h; 0.0 gives the curved code path on an affine geometry)."""
    if not 1 <= len(bands) <= SDG_MAX_BANDS:
        raise ConfigError("mesh needs 1..16 bands")
    m = MeshSpec()
    m.x0, m.y0, m.z0 = x0, y0, z0
    m.width, m.height, m.depth = width, height, depth
    m.ny, m.nz = ny, nz
    m.n_bands = len(bands)
    for i, b in enumerate(bands):
        b = tuple(b)
        nx, frac, vg = b[0], (b[1] if len(b) > 1 else 1.0), (b[2] if len(b) > 2 else 0.0)
        m.bands[i].nx, m.bands[i].width_frac, m.bands[i].vg_y = int(nx), float(frac), float(vg)
        m.bands[i].ny = int(b[3]) if len(b) > 3 else 0
        m.bands[i].nz = int(b[4]) if len(b) > 4 else 0
        m.bands[i].vg_z = float(b[5]) if len(b) > 5 else 0.0
    m.periodic_x, m.periodic_y, m.periodic_z = (int(bool(p)) for p in periodic)
    m.partition = int(partition)
    m.mapping = (MAP_BOX if warp is None else MAP_WARP) if mapping is None else int(mapping)
    m.warp = 0.0 if warp is None else float(warp)
    m.mortars = int(mortars)
    return m


def annulus_spec(bands, n_theta, n_r, r_in, r_out, length=2.0, warp=None, theta_span=2.0 * math.pi,
                 partition=PARTITION_LEX, periodic_theta=None) -> MeshSpec:
    """Rotor/stator annulus (SDG_MAP_ANNULUS): bands (nx, width_frac, omega) stacked
    along the axis x over [0, length], n_theta elements around, n_r radially in
    [r_in, r_out]; radial walls and axial ends Dirichlet.  theta is periodic by
    default when the span divides the full circle (a sector 2 pi / m is
    rotationally periodic: vectors rotate by the sector angle across its seam)."""
    if periodic_theta is None:
        m = 2.0 * math.pi / theta_span
        periodic_theta = abs(m - round(m)) < 1e-9
    return mesh_spec(bands, ny=n_theta, nz=n_r, width=length, height=theta_span, depth=r_out - r_in,
                     z0=r_in, periodic=(False, periodic_theta, False), partition=partition, warp=warp,
                     mapping=MAP_ANNULUS)


def freestream(rho=1.0, v=(1.0, 0.5, 0.0), p=1.0) -> Case:
    c = Case()
    c.kind = CASE_FREESTREAM
    c.fs_rho, c.fs_p = rho, p
    for i in range(3):
        c.fs_v[i] = v[i]
    return c


def density_wave(alpha=0.1, a=(1.0, 1.0, 1.0), k=(1.0, 1.0, 1.0), p0=1.0) -> Case:
    c = Case()
    c.kind = CASE_DENSITY_WAVE
    c.dw_alpha, c.dw_p0 = alpha, p0
    for i in range(3):
        c.dw_a[i], c.dw_k[i] = a[i], k[i]
    return c


def vortex(eps=1.0, rc=1.0, rho_inf=1.0, v_inf=1.0, theta=math.atan(0.5), ma_inf=0.3, center=(0.0, 0.0)) -> Case:
    c = Case()
    c.kind = CASE_VORTEX
    c.vx_eps, c.vx_rc, c.vx_rho_inf, c.vx_v_inf, c.vx_theta, c.vx_ma_inf = eps, rc, rho_inf, v_inf, theta, ma_inf
    c.vx_center[0], c.vx_center[1] = center
    return c


def tgv(rho0=1.0, v0=1.0, mach=0.1) -> Case:
    c = Case()
    c.kind = CASE_TGV
    c.tgv_rho0, c.tgv_v0, c.tgv_mach = rho0, v0, mach
    return c


def swirl(alpha=0.1, a=1.0, k=1.0, p0=5.0, omega=0.5) -> Case:
    """Axial density wave with rigid swirl about x (include/sdg_types.h SDG_CASE_SWIRL)."""
    c = Case()
    c.kind = CASE_SWIRL
    c.dw_alpha, c.dw_p0, c.sw_omega = alpha, p0, omega
    c.dw_a[0], c.dw_k[0] = a, k
    return c


class MT19937_64:
    """std::mt19937_64 (the 64-bit Mersenne Twister of C++11 <random>), so the seeded
    inputs of SURVEY §8(d) -- mt19937_64(2008043560 + config index) -- are the same
    numbers a C++ harness would draw."""
    N, M = 312, 156
    MATRIX_A, UPPER, LOWER = 0xB5026F5AA96619E9, 0xFFFFFFFF80000000, 0x7FFFFFFF
    MASK = (1 << 64) - 1

    def __init__(self, seed: int):
        self.mt = [0] * self.N
        self.mt[0] = seed & self.MASK
        for i in range(1, self.N):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & self.MASK
        self.idx = self.N

    def __call__(self) -> int:
        if self.idx >= self.N:
            mt = self.mt
            for i in range(self.N):
                x = (mt[i] & self.UPPER) | (mt[(i + 1) % self.N] & self.LOWER)
                xa = x >> 1
                if x & 1:
                    xa ^= self.MATRIX_A
                mt[i] = mt[(i + self.M) % self.N] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & self.MASK

    def uniform(self) -> float:
        """[0, 1) with 53 random bits."""
        return (self() >> 11) * (1.0 / 9007199254740992.0)


SEED_BASE = 2008043560


def seeded_modes(config_index: int, kmax: int, n_modes: int = 8):
    """The 8 Fourier modes of SURVEY §8(d): draw with mt19937_64(2008043560 + i), per
    mode k in {-kmax..kmax}^3 minus 0 (k_d = draw mod (2 kmax + 1) - kmax, redrawn
    while k = 0), a ~ U(-1, 1), phi ~ U[0, 2 pi); a normalised to sum |a| = 1.
    Returns (k [n,3], a [n], phi [n])."""
    rng = MT19937_64(SEED_BASE + config_index)
    ks, a, phi = [], [], []
    for _ in range(n_modes):
        while True:
            k = [int(rng() % (2 * kmax + 1)) - kmax for _ in range(3)]
            if any(k):
                break
        ks.append(k)
        a.append(2.0 * rng.uniform() - 1.0)
        phi.append(2.0 * math.pi * rng.uniform())
    s = sum(abs(x) for x in a)
    return ks, [x / s for x in a], phi


def perturbed(case: Case, config_index: int, amp: float, kmax: int, x0, length, adv=(0.0, 0.0, 0.0),
              cylindrical: bool = False) -> Case:
    """`case` plus the seeded density perturbation of SURVEY §8(d) (include/sdg_types.h
    sdg_case.pt_*): amp * sum_m a_m sin(2 pi k_m . xh + phi_m), xh = (c - x0) / length with
    c the point advected by `adv` (cylindrical: (x, theta, r) about the x axis)."""
    ks, a, phi = seeded_modes(config_index, kmax)
    c = Case()
    C.pointer(c)[0] = case
    c.pt_modes, c.pt_coords, c.pt_amp = len(ks), 1 if cylindrical else 0, amp
    for d in range(3):
        c.pt_x0[d], c.pt_len[d], c.pt_adv[d] = x0[d], length[d], adv[d]
    for m in range(len(ks)):
        for d in range(3):
            c.pt_k[m][d] = ks[m][d]
        c.pt_a[m], c.pt_phi[m] = a[m], phi[m]
    return c


def solver_config(degree, node_kind=NODES_GAUSS, gamma=1.4, R=1.0, mu=0.0, Pr=0.72, case=None) -> SolverConfig:
    s = SolverConfig()
    s.degree, s.node_kind = degree, node_kind
    s.gas.gamma, s.gas.R, s.gas.mu, s.gas.Pr = gamma, R, mu, Pr
    s.flow_case = case if case is not None else freestream()
    return s
