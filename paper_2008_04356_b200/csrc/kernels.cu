// sm_100a kernels of the sliding-mesh DGSEM right-hand side (fp64).
//
// Dataflow per RK stage (viscous):
//   k_gradient  (element): U + neighbour traces -> BR1 lift* -> volume gradient ->
//                          viscous normal flux Fv.n on every conforming side
//                          (the 12-component gradient trace only on sliding /
//                          Dirichlet sides, which need it unprojected)
//   mortar kernels         face -> mortar transfer, two-sided mortar flux,
//                          L2 back projection (only sliding faces)
//   k_update    (element): U + neighbour traces + Fv.n -> Roe + viscous face flux,
//                          recomputed gradient, volume flux + weak divergence,
//                          surface lift, low-storage RK update, admissibility,
//                          and the face traces of the NEW state for the next stage.
// Each conforming face flux is evaluated by both of its elements with the
// same instruction sequence on the same operands (minus side first), so both
// sides see identical bits — the orientation rule of solver.cpp:323-341.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

namespace sdg {
namespace {

template <int N1>
struct Dim {
  static constexpr int N2 = N1 * N1;
  static constexpr int N3 = N2 * N1;
  // elements per CTA: keep CTAs at 200-512 threads
  static constexpr int EPB = N1 == 2 ? 32 : N1 == 3 ? 8 : N1 == 4 ? 4 : N1 <= 6 ? 2 : 1;
  static constexpr int THREADS = EPB * N3;
  // shared operator table (doubles); N1 = 8 appends D-hat transposed (load_tables, dhat_k)
  static constexpr int TAB = ((N1 * N1 + 6 * N1 + (N1 == 8 ? N1 * N1 : 0)) + 1) & ~1;
};

__device__ __forceinline__ double sel3(int d, double a, double b, double c) { return d == 0 ? a : (d == 1 ? b : c); }

// Rotation of a (y, z) pair about the x axis by the angle with cosine c and sine s
// (theta -> theta + angle with Y = r sin theta, Z = r cos theta; annulus sectors).
__device__ __forceinline__ void rot_yz(double c, double s, double& y, double& z) {
  const double a = c * y + s * z, b = -s * y + c * z;
  y = a;
  z = b;
}

// ----------------------------------------------------------------------------
// Canonical quantities that two kernels must reproduce bit-identically are
// written with explicit rounding intrinsics (no contraction freedom).
// ----------------------------------------------------------------------------

// Shared-memory bank rotation of the face contractions.  A face node's line of N1
// values is read in the rotated order m -> (m + rot) mod N1, with rot a fixed function
// of the face node (side, a, b), so that the 16 threads of a half-warp (consecutive
// face nodes it = side * N2 + a * N1 + b) hit 16 different 8-byte banks of a
// [row][node] element block.  Unrotated, the lines along j and k collide 2-way at
// N+1 = 6, 4-way at 4 and up to 8-way at 8 (line starts are multiples of N+1).
// The rotation is part of the canonical trace: every kernel that prolongs a
// state uses the same order, so all of them produce the same bits.
// N+1 = 6 has no closed form (36 face nodes per side do not tile half-warps);
// its table comes from a per-half-warp search (tools/bank_rotation.py).
__device__ const unsigned char kFaceRot6[216] = {
    0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0,  // side 0
    1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0,  // side 1
    3, 3, 3, 3, 2, 2, 3, 3, 0, 0, 0, 0, 1, 1, 0, 0, 0, 0, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 1,  // side 2
    1, 1, 1, 1, 0, 0, 1, 1, 0, 0, 0, 0, 1, 1, 1, 1, 0, 0, 1, 1, 0, 0, 0, 0, 1, 1, 0, 0, 0, 0, 1, 1, 1, 1, 0, 0,  // side 3
    0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0,  // side 4
    1, 1, 1, 1, 1, 0, 1, 0, 5, 2, 5, 2, 0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0, 0,  // side 5
};

template <int N1>
__device__ __forceinline__ int face_rot(int side, int a, int b) {
  const int dir = side >> 1;
  if constexpr (N1 == 4) {
    return dir == 0 ? 0 : a;
  } else if constexpr (N1 == 8) {
    return dir == 0 ? 0 : (dir == 1 ? (a & 1) : (b >> 1) + 4 * (a & 1));
  } else if constexpr (N1 == 6) {
    return kFaceRot6[side * 36 + a * 6 + b];
  } else {
    return 0;
  }
}

// Rotated line index (m + rot) mod N1 for 0 <= m, rot < N1.
template <int N1>
__device__ __forceinline__ int rot_index(int m, int rot) {
  const int r = m + rot;
  return r >= N1 ? r - N1 : r;
}

// The same rotation for the volume contractions of node threads (thread t = node
// (i, j, k) reads its lines along i and j): only N+1 = 6 needs it, where a half-warp
// that straddles two i-planes (36 nodes each) hits the banks of the previous plane's
// tail.  Those threads start their lines one node later.
template <int N1>
__device__ __forceinline__ int node_rot(int t) {
  if constexpr (N1 == 6) {
    return (t & ~15) < 36 * (t / 36) ? 1 : 0;
  } else {
    return 0;
  }
}

// Face trace of one variable along the face normal (solver.cpp:208-232).
template <int N1>
__device__ __forceinline__ double prolong1(const double* __restrict__ s, const double* __restrict__ ell, int dir,
                                           int a, int b, int rot) {
  constexpr int N2 = N1 * N1;
  const int base = dir == 0 ? a * N1 + b : (dir == 1 ? a * N2 + b : (a * N1 + b) * N1);
  const int stride = dir == 0 ? N2 : (dir == 1 ? N1 : 1);
  double acc = 0.0;
#pragma unroll
  for (int m = 0; m < N1; ++m) {
    const int mr = rot_index<N1>(m, rot);
    acc = __fma_rn(ell[mr], s[base + mr * stride], acc);
  }
  return acc;
}

// Call-free reciprocal / square root for the face-flux hot loop: the MUFU seed
// refined by Newton steps (~1 ulp; the correctly rounded library versions
// branch to out-of-line slow paths whose call ABI makes ptxas spill the
// kernel's live state).  Arguments are positive and normal on every
// admissible state; anything else yields NaN, which the admissibility checks
// report.
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = __fma_rn(y, __fma_rn(-x, y, 1.0), y);
  y = __fma_rn(y, __fma_rn(-x, y, 1.0), y);
  return __fma_rn(y, __fma_rn(-x, y, 1.0), y);
}

__device__ __forceinline__ double sqrt_nr(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double hx = 0.5 * x;
  r = r * __fma_rn(-hx * r, r, 1.5);
  r = r * __fma_rn(-hx * r, r, 1.5);
  const double s = x * r;
  const double v = __fma_rn(0.5 * r, __fma_rn(-s, s, x), s);
  return x > 0.0 ? v : (x == 0.0 ? 0.0 : __longlong_as_double(0x7ff8000000000000ll));
}

// (v1, v2, v3, T) of a conserved state (state.hpp:47-84).
__device__ __forceinline__ void prim4(const double* u, const GasD& g, double* q) {
  const double ir = rcp_nr(u[0]);
  q[0] = __dmul_rn(u[1], ir);
  q[1] = __dmul_rn(u[2], ir);
  q[2] = __dmul_rn(u[3], ir);
  const double m2 = __fma_rn(u[3], u[3], __fma_rn(u[2], u[2], __dmul_rn(u[1], u[1])));
  const double p = __dmul_rn(g.gm1, __fma_rn(-__dmul_rn(0.5, m2), ir, u[4]));
  q[3] = __dmul_rn(p, __dmul_rn(ir, g.inv_R));
}

__device__ __forceinline__ double pressure(const double* u, double ir, const GasD& g) {
  const double m2 = u[1] * u[1] + u[2] * u[2] + u[3] * u[3];
  return g.gm1 * (u[4] - 0.5 * m2 * ir);
}

__device__ __forceinline__ double entropy_fix(double lam, double lam_l, double lam_r) {
  const double delta = fmax(0.0, fmax(lam - lam_l, lam_r - lam));
  const double a = fabs(lam);
  return a < 2.0 * delta ? lam * lam * rcp_nr(4.0 * delta) + delta : a;
}

// Roe flux, Harten-Hyman fix on acoustic waves, eigenvalues shifted by the
// normal grid speed; axis normal e_dir (flux.cpp:68-133, 3D: second shear wave).
// Returns false when the Roe-averaged c^2 is not positive.
__device__ __forceinline__ bool roe_flux(const double* ul, const double* ur, int dir, double vg, const GasD& g,
                                         double* f) {
  const double rl = ul[0], rr = ur[0];
  const double irl = rcp_nr(rl), irr = rcp_nr(rr);
  const double mnl = sel3(dir, ul[1], ul[2], ul[3]), mal = sel3(dir, ul[2], ul[3], ul[1]),
               mbl = sel3(dir, ul[3], ul[1], ul[2]);
  const double mnr = sel3(dir, ur[1], ur[2], ur[3]), mar = sel3(dir, ur[2], ur[3], ur[1]),
               mbr = sel3(dir, ur[3], ur[1], ur[2]);
  const double unl = mnl * irl, ual = mal * irl, ubl = mbl * irl;
  const double unr = mnr * irr, uar = mar * irr, ubr = mbr * irr;
  const double pl = g.gm1 * (ul[4] - 0.5 * (mnl * unl + mal * ual + mbl * ubl));
  const double pr = g.gm1 * (ur[4] - 0.5 * (mnr * unr + mar * uar + mbr * ubr));
  const double hl = (ul[4] + pl) * irl, hr = (ur[4] + pr) * irr;
  const double cl = sqrt_nr(g.gamma * pl * irl), cr = sqrt_nr(g.gamma * pr * irr);

  const double sl = sqrt_nr(rl), sr = sqrt_nr(rr);
  const double inv = rcp_nr(sl + sr);
  const double un = (sl * unl + sr * unr) * inv;
  const double ua = (sl * ual + sr * uar) * inv;
  const double ub = (sl * ubl + sr * ubr) * inv;
  const double h = (sl * hl + sr * hr) * inv;
  const double q2 = un * un + ua * ua + ub * ub;
  const double c2 = g.gm1 * (h - 0.5 * q2);
  if (!(c2 > 0.0)) return false;
  const double c = sqrt_nr(c2);
  const double ic2 = rcp_nr(c2);
  const double rho = sl * sr;

  const double dp = pr - pl, dun = unr - unl, dua = uar - ual, dub = ubr - ubl, drho = rr - rl;
  const double a1 = (dp - rho * c * dun) * 0.5 * ic2;
  const double a2 = drho - dp * ic2;
  const double a3 = rho * dua;
  const double a3b = rho * dub;
  const double a4 = (dp + rho * c * dun) * 0.5 * ic2;

  const double l1 = entropy_fix(un - c - vg, unl - cl - vg, unr - cr - vg);
  const double l2 = fabs(un - vg);
  const double l4 = entropy_fix(un + c - vg, unl + cl - vg, unr + cr - vg);
  const double w1 = l1 * a1, w2 = l2 * a2, w4 = l4 * a4;
  const double d0 = w1 + w2 + w4;
  const double dn = w1 * (un - c) + w2 * un + w4 * (un + c);
  const double da = d0 * ua + l2 * a3;
  const double db = d0 * ub + l2 * a3b;
  const double dE = w1 * (h - un * c) + w2 * 0.5 * q2 + l2 * a3 * ua + l2 * a3b * ub + w4 * (h + un * c);

  // Physical normal fluxes minus vg_n U (flux.cpp:44-54).
  const double f0 = 0.5 * ((rl * unl - vg * rl) + (rr * unr - vg * rr) - d0);
  const double fn = 0.5 * ((mnl * unl + pl - vg * mnl) + (mnr * unr + pr - vg * mnr) - dn);
  const double fa = 0.5 * ((mal * unl - vg * mal) + (mar * unr - vg * mar) - da);
  const double fb = 0.5 * ((mbl * unl - vg * mbl) + (mbr * unr - vg * mbr) - db);
  const double fE = 0.5 * (((ul[4] + pl) * unl - vg * ul[4]) + ((ur[4] + pr) * unr - vg * ur[4]) - dE);
  f[0] = f0;
  f[1] = sel3(dir, fn, fb, fa);
  f[2] = sel3(dir, fa, fn, fb);
  f[3] = sel3(dir, fb, fa, fn);
  f[4] = fE;
  return true;
}

// Viscous flux along direction dir, components 1..4 (flux.cpp:23-42).
__device__ __forceinline__ void fv_dir(const double* u, const double* gr, int dir, const GasD& g, double* o) {
  const double ir = rcp_nr(u[0]);
  const double v0 = u[1] * ir, v1 = u[2] * ir, v2 = u[3] * ir;
  const double div = gr[0] + gr[4] + gr[8];
  const double t00 = 2.0 * g.mu * gr[0] + g.lam * div;
  const double t11 = 2.0 * g.mu * gr[4] + g.lam * div;
  const double t22 = 2.0 * g.mu * gr[8] + g.lam * div;
  const double t01 = g.mu * (gr[1] + gr[3]);
  const double t02 = g.mu * (gr[2] + gr[6]);
  const double t12 = g.mu * (gr[5] + gr[7]);
  const double r0 = sel3(dir, t00, t01, t02), r1 = sel3(dir, t01, t11, t12), r2 = sel3(dir, t02, t12, t22);
  const double dT = sel3(dir, gr[9], gr[10], gr[11]);
  o[0] = r0;
  o[1] = r1;
  o[2] = r2;
  o[3] = r0 * v0 + r1 * v1 + r2 * v2 + g.kcond * dT;
}

// face_numerical_flux with both viscous normal fluxes given (solver.cpp:308-321).
__device__ __forceinline__ bool face_flux_fv(const double* um, const double* up, int dir, double vg,
                                             const double* fvm, const double* fvp, const GasD& g, double* f) {
  const bool ok = roe_flux(um, up, dir, vg, g, f);
  if (fvm != nullptr) {
#pragma unroll
    for (int v = 0; v < 4; ++v) f[1 + v] -= 0.5 * (fvm[v] + fvp[v]);
  }
  return ok;
}

// Seeded density perturbation of include/sdg_types.h (sdg_case.pt_*).
__device__ double case_perturbation(const sdg_case& cs, const double* x, double t) {
  const double two_pi = 6.283185307179586476925286766559;
  double c[3] = {x[0] - cs.pt_adv[0] * t, x[1] - cs.pt_adv[1] * t, x[2] - cs.pt_adv[2] * t};
  if (cs.pt_coords == 1) {
    const double th = atan2(c[1], c[2]), r = sqrt(c[1] * c[1] + c[2] * c[2]);
    c[1] = th;
    c[2] = r;
  }
  double xh[3];
  for (int d = 0; d < 3; ++d) xh[d] = (c[d] - cs.pt_x0[d]) / cs.pt_len[d];
  double acc = 0.0;
  for (int m = 0; m < cs.pt_modes; ++m)
    acc += cs.pt_a[m] * sin(two_pi * (cs.pt_k[m][0] * xh[0] + cs.pt_k[m][1] * xh[1] + cs.pt_k[m][2] * xh[2]) + cs.pt_phi[m]);
  return cs.pt_amp * acc;
}

// Exact solutions (exact_solutions.cpp:7-35; TGV in BASELINE axes).
__device__ void eval_case(const sdg_case& cs, const double* x, double t, const GasD& g, double* u) {
  const double pi = 3.14159265358979323846;
  double rho, v0, v1, v2, p;
  switch (cs.kind) {
    case SDG_CASE_DENSITY_WAVE: {
      const double* k = cs.dw_k;
      const double* a = cs.dw_a;
      const double ph = pi * (k[0] * x[0] + k[1] * x[1] + k[2] * x[2] - (k[0] * a[0] + k[1] * a[1] + k[2] * a[2]) * t);
      rho = 2.0 + cs.dw_alpha * sin(ph);
      v0 = a[0];
      v1 = a[1];
      v2 = a[2];
      p = cs.dw_p0;
      break;
    }
    case SDG_CASE_VORTEX: {
      const double ui = cs.vx_v_inf * cos(cs.vx_theta), vi = cs.vx_v_inf * sin(cs.vx_theta);
      const double xb = x[0] - cs.vx_center[0] - ui * t, yb = x[1] - cs.vx_center[1] - vi * t;
      const double r2 = (xb * xb + yb * yb) / (cs.vx_rc * cs.vx_rc);
      const double s = cs.vx_eps * exp(0.5 * (1.0 - r2));
      v0 = ui - cs.vx_v_inf * s * yb / cs.vx_rc;
      v1 = vi + cs.vx_v_inf * s * xb / cs.vx_rc;
      v2 = 0.0;
      const double tr = 1.0 - 0.5 * g.gm1 * cs.vx_eps * cs.vx_eps * cs.vx_ma_inf * cs.vx_ma_inf * exp(1.0 - r2);
      rho = cs.vx_rho_inf * pow(tr, 1.0 / g.gm1);
      const double pinf = cs.vx_rho_inf * cs.vx_v_inf * cs.vx_v_inf / (g.gamma * cs.vx_ma_inf * cs.vx_ma_inf);
      p = pinf * pow(tr, g.gamma / g.gm1);
      break;
    }
    case SDG_CASE_TGV: {
      const double X = x[1], Y = x[2], Z = x[0];
      const double V0 = cs.tgv_v0, r0 = cs.tgv_rho0;
      rho = r0;
      v0 = 0.0;
      v1 = V0 * sin(X) * cos(Y) * cos(Z);
      v2 = -V0 * cos(X) * sin(Y) * cos(Z);
      const double p0 = r0 * V0 * V0 / (g.gamma * cs.tgv_mach * cs.tgv_mach);
      p = p0 + r0 * V0 * V0 / 16.0 * (cos(2.0 * X) + cos(2.0 * Y)) * (cos(2.0 * Z) + 2.0);
      break;
    }
    case SDG_CASE_SWIRL: {
      const double om = cs.sw_omega;
      rho = 2.0 + cs.dw_alpha * sin(pi * cs.dw_k[0] * (x[0] - cs.dw_a[0] * t));
      v0 = cs.dw_a[0];
      v1 = om * x[2];
      v2 = -om * x[1];
      p = cs.dw_p0 + om * om * (x[1] * x[1] + x[2] * x[2]);
      break;
    }
    default:
      rho = cs.fs_rho;
      v0 = cs.fs_v[0];
      v1 = cs.fs_v[1];
      v2 = cs.fs_v[2];
      p = cs.fs_p;
  }
  if (cs.pt_modes > 0) rho += case_perturbation(cs, x, t);
  u[0] = rho;
  u[1] = rho * v0;
  u[2] = rho * v1;
  u[3] = rho * v2;
  u[4] = p / g.gm1 + 0.5 * rho * (v0 * v0 + v1 * v1 + v2 * v2);
}

// sin(pi t), exactly 0 at integer t (the warp vanishes on band boundaries).
__device__ __forceinline__ double sinpi_exact(double t) {
  double r = fmod(t, 2.0);
  if (r < 0.0) r += 2.0;
  return (r == 0.0 || r == 1.0) ? 0.0 : sinpi(r);
}

// Physical position of reference point (xi, eta, zeta) of an element at time t
// (mesh.cpp:118-122; SDG_MAP_WARP adds the curved warp of include/sdg_types.h).
__device__ __forceinline__ void map_position(const ElemConsts& C, const int* crd, double xi, double eta, double zeta,
                                             double t, double* x) {
  const BandD& B = C.bands[crd[0]];
  x[0] = (B.x_lo + crd[1] * B.hx) + 0.5 * (xi + 1.0) * B.hx;
  x[1] = (C.y0 + crd[2] * B.hy) + 0.5 * (eta + 1.0) * B.hy;
  x[2] = (C.z0 + crd[3] * B.hz) + 0.5 * (zeta + 1.0) * B.hz;
  if (C.mapping != SDG_MAP_BOX) {
    const double tx = (crd[1] + 0.5 * (xi + 1.0)) / B.nxd, ty = (crd[2] + 0.5 * (eta + 1.0)) / C.ny,
                 tz = (crd[3] + 0.5 * (zeta + 1.0)) / C.nz;
    const double sp = sinpi_exact(tx), sy = sinpi_exact(2.0 * ty), sz = sinpi_exact(2.0 * tz);
    x[0] += C.warp * B.hx * sp * sy * sz;
    if (C.mapping != SDG_MAP_ANNULUS) x[1] += C.warp * B.hy * sp * sz;  // annulus: no theta warp
    x[2] += C.warp * B.hz * sp * sy;
  }
  x[1] += B.vg * t;
  x[2] += B.vgz * t;
  if (C.mapping == SDG_MAP_ANNULUS) {  // (x, theta, r) -> (x, r sin theta, r cos theta)
    double sn, cs;
    sincos(x[1], &sn, &cs);
    const double r = x[2];
    x[1] = r * sn;
    x[2] = r * cs;
  }
}

// Physical position of face node (a, b) of `side` at time t.
template <int N1>
__device__ __forceinline__ void face_position(const ElemConsts& C, const int* crd, int side, int a, int b, double t,
                                              double* x) {
  const int dir = side >> 1;
  const double pm = (side & 1) ? 1.0 : -1.0;
  const double xi = dir == 0 ? pm : C.x[a];
  const double eta = dir == 1 ? pm : (dir == 0 ? C.x[a] : C.x[b]);
  const double zeta = dir == 2 ? pm : C.x[b];
  map_position(C, crd, xi, eta, zeta, t, x);
}

// Viscous stress tensor (tau_00, tau_01, tau_02, tau_11, tau_12, tau_22) and heat flux
// k dT/dx_d of a node from its BR1 gradient g[3 q + d] = d q / d x_d, q = (v1, v2, v3, T)
// (viscous_flux, flux.cpp:23-42).
__device__ __forceinline__ void visc_terms(const double* g, const GasD& gas, double* o) {
  const double div = g[0] + g[4] + g[8];
  const double mu = gas.mu, lam = gas.lam;
  o[0] = 2.0 * mu * g[0] + lam * div;
  o[1] = mu * (g[1] + g[3]);
  o[2] = mu * (g[2] + g[6]);
  o[3] = 2.0 * mu * g[4] + lam * div;
  o[4] = mu * (g[5] + g[7]);
  o[5] = 2.0 * mu * g[8] + lam * div;
  o[6] = gas.kcond * g[9];
  o[7] = gas.kcond * g[10];
  o[8] = gas.kcond * g[11];
}

template <int N1>
__device__ __forceinline__ void load_tables(const ElemConsts& C, double* tab) {
  // tab: dhat[N1*N1] | fl | fr | liftw0 | liftw1 | inv_w | (unused)
  for (int q = threadIdx.x; q < N1 * N1; q += blockDim.x) tab[q] = C.dhat[(q / N1) * kMaxN1 + q % N1];
  for (int q = threadIdx.x; q < N1; q += blockDim.x) {
    tab[N1 * N1 + q] = C.fl[q];
    tab[N1 * N1 + N1 + q] = C.fr[q];
    tab[N1 * N1 + 2 * N1 + q] = C.liftw[0][q];
    tab[N1 * N1 + 3 * N1 + q] = C.liftw[1][q];
    tab[N1 * N1 + 4 * N1 + q] = C.inv_w[q];
  }
  if constexpr (N1 == 8) {  // D-hat transposed for the lines along k (dhat_k)
    for (int q = threadIdx.x; q < N1 * N1; q += blockDim.x) tab[N1 * N1 + 6 * N1 + q] = C.dhat[(q % N1) * kMaxN1 + q / N1];
  }
}

// D-hat(k, m) for a node thread's line along k.  Rows of 8 doubles put the 8 values of k in a
// half-warp on 2 banks (8 k + m mod 16), a 4-way conflict; N1 = 8 reads the transposed copy
// (m * 8 + k: consecutive).  Rows of 4 and 6 doubles spread over distinct banks.
template <int N1>
__device__ __forceinline__ double dhat_k(const double* tab, int k, int m) {
  if constexpr (N1 == 8) return tab[N1 * N1 + 6 * N1 + m * N1 + k];
  else return tab[k * N1 + m];
}


// Flat, coalesced load of EPB consecutive elements into SoA shared memory su[v][node].
template <int N1>
__device__ __forceinline__ void load_state(const double* __restrict__ U, int e0, int E, double* smem_elems,
                                           int per_elem) {
  constexpr int N3 = Dim<N1>::N3, EPB = Dim<N1>::EPB;
  const int n_el = min(EPB, E - e0);
  const double* src = U + static_cast<size_t>(e0) * 5 * N3;
  for (int f = threadIdx.x; f < n_el * 5 * N3; f += blockDim.x) {
    const int le = f / (5 * N3), r = f - le * 5 * N3;
    smem_elems[le * per_elem + (r % 5) * N3 + r / 5] = __ldg(src + f);
  }
}

// ----------------------------------------------------------------------------
// Face traces of U (first stage of a step / residual entry).
// ----------------------------------------------------------------------------
template <int N1>
__global__ void __launch_bounds__(Dim<N1>::THREADS) k_prolong(const __grid_constant__ ElemConsts C, FieldPtrs P) {
  constexpr int N2 = Dim<N1>::N2, N3 = Dim<N1>::N3, EPB = Dim<N1>::EPB, TAB = Dim<N1>::TAB;
  extern __shared__ double smem[];
  double* tab = smem;
  double* elems = smem + TAB;
  constexpr int PER = 5 * N3;
  load_tables<N1>(C, tab);
  const int e0 = P.e_first + blockIdx.x * EPB;
  load_state<N1>(P.U, e0, P.E, elems, PER);
  __syncthreads();
  const int le = threadIdx.x / N3, t = threadIdx.x % N3, e = e0 + le;
  if (e >= P.E) return;
  const double* su = elems + le * PER;
  for (int it = t; it < 6 * N2; it += N3) {
    const int s = it / N2, f = it % N2, a = f / N1, b = f % N1;
    const double* ell = tab + N1 * N1 + (s & 1) * N1;
    double* dst = P.trace + (static_cast<size_t>(e) * 6 + s) * N2 * 5 + f * 5;
#pragma unroll
    for (int v = 0; v < 5; ++v) dst[v] = prolong1<N1>(su + v * N3, ell, s >> 1, a, b, face_rot<N1>(s, a, b));
  }
}

// ----------------------------------------------------------------------------
// Shared face phase: BR1 surface values lift*[s][c][f] on all six sides
// (run_lifting, solver.cpp:606-723), and optionally the own traces.
// ----------------------------------------------------------------------------
template <int N1>
__device__ __forceinline__ void face_lift_phase(const ElemConsts& C, const FieldPtrs& P, const double* tab,
                                                const double* su, int e, double t_stage, double* sLift,
                                                double* sTr) {
  constexpr int N2 = Dim<N1>::N2, N3 = Dim<N1>::N3;
  const int t = threadIdx.x % N3;
  for (int it = t; it < 6 * N2; it += N3) {
    const int s = it / N2, f = it % N2, a = f / N1, b = f % N1;
    const double* ell = tab + N1 * N1 + (s & 1) * N1;
    double own[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) own[v] = prolong1<N1>(su + v * N3, ell, s >> 1, a, b, face_rot<N1>(s, a, b));
    if (sTr != nullptr) {
#pragma unroll
      for (int v = 0; v < 5; ++v) sTr[(s * N2 + f) * 5 + v] = own[v];
    }
    const int slot = e * 6 + s;
    const int typ = P.side_type[slot], idx = P.side_idx[slot];
    double lift[4];
    if (typ == kConforming) {
      const double* nb = P.trace + static_cast<size_t>(idx) * N2 * 5 + f * 5;
      double other[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) other[v] = nb[v];
      if (C.sec_s != 0.0 && P.side_rot[slot] != 0)  // periodic annulus sector seam
        rot_yz(C.sec_c, P.side_rot[slot] * C.sec_s, other[2], other[3]);
      double qa[4], qb[4];
      prim4(own, C.gas, qa);
      prim4(other, C.gas, qb);
#pragma unroll
      for (int c = 0; c < 4; ++c) lift[c] = __dmul_rn(0.5, __dadd_rn(qa[c], qb[c]));
    } else if (typ == kSliding) {
      const double* sl = P.slide_lift + (static_cast<size_t>(idx) * N2 + f) * 4;
#pragma unroll
      for (int c = 0; c < 4; ++c) lift[c] = sl[c];
    } else {
      double x[3], ext[5];
      face_position<N1>(C, P.coords + 4 * e, s, a, b, t_stage, x);
      eval_case(C.flow_case, x, t_stage, C.gas, ext);
      prim4(ext, C.gas, lift);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) sLift[(s * 4 + c) * N2 + f] = lift[c];
  }
}

// Volume BR1 gradient of (v1, v2, v3, T) at one node (assemble_gradients, solver.cpp:729-768).
template <int N1>
__device__ __forceinline__ void node_gradient(const double* tab, const double* sq, const double* sLift,
                                              const BandD& B, int i, int j, int k, double* g) {
  constexpr int N2 = Dim<N1>::N2, N3 = Dim<N1>::N3;
  const double* dh = tab;
  const double* fl = tab + N1 * N1;
  const double* fr = fl + N1;
  const double* iw = fl + 4 * N1;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double* q = sq + c * N3;
    double vx = 0.0, vy = 0.0, vz = 0.0;
#pragma unroll
    for (int m = 0; m < N1; ++m) {
      vx += dh[i * N1 + m] * q[(m * N1 + j) * N1 + k];
      vy += dh[j * N1 + m] * q[(i * N1 + m) * N1 + k];
      vz += dh[k * N1 + m] * q[(i * N1 + j) * N1 + m];
    }
    const double sx = (sLift[(1 * 4 + c) * N2 + j * N1 + k] * fr[i] - sLift[(0 * 4 + c) * N2 + j * N1 + k] * fl[i]) * iw[i];
    const double sy = (sLift[(3 * 4 + c) * N2 + i * N1 + k] * fr[j] - sLift[(2 * 4 + c) * N2 + i * N1 + k] * fl[j]) * iw[j];
    const double sz = (sLift[(5 * 4 + c) * N2 + i * N1 + j] * fr[k] - sLift[(4 * 4 + c) * N2 + i * N1 + j] * fl[k]) * iw[k];
    g[3 * c + 0] = B.cdir[0] * (sx - vx);
    g[3 * c + 1] = B.cdir[1] * (sy - vy);
    g[3 * c + 2] = B.cdir[2] * (sz - vz);
  }
}

// Same, with q stored node-major at pitch 6 (two 128-bit loads per node).
template <int N1>
__device__ __forceinline__ void node_gradient_pk(const double* tab, const double* q6, const double* sLift,
                                                 const BandD& B, int i, int j, int k, double* g) {
  constexpr int N2 = N1 * N1;
  const double* dh = tab;
  const double* fl = tab + N1 * N1;
  const double* fr = fl + N1;
  const double* iw = fl + 4 * N1;
  double vx[4] = {0, 0, 0, 0}, vy[4] = {0, 0, 0, 0}, vz[4] = {0, 0, 0, 0};
#pragma unroll
  for (int m = 0; m < N1; ++m) {
    const double cx = dh[i * N1 + m], cy = dh[j * N1 + m], cz = dh[k * N1 + m];
    const double* px = q6 + ((m * N1 + j) * N1 + k) * 6;
    const double* py = q6 + ((i * N1 + m) * N1 + k) * 6;
    const double* pz = q6 + ((i * N1 + j) * N1 + m) * 6;
    const double2 x01 = *reinterpret_cast<const double2*>(px), x23 = *reinterpret_cast<const double2*>(px + 2);
    const double2 y01 = *reinterpret_cast<const double2*>(py), y23 = *reinterpret_cast<const double2*>(py + 2);
    const double2 z01 = *reinterpret_cast<const double2*>(pz), z23 = *reinterpret_cast<const double2*>(pz + 2);
    vx[0] += cx * x01.x; vx[1] += cx * x01.y; vx[2] += cx * x23.x; vx[3] += cx * x23.y;
    vy[0] += cy * y01.x; vy[1] += cy * y01.y; vy[2] += cy * y23.x; vy[3] += cy * y23.y;
    vz[0] += cz * z01.x; vz[1] += cz * z01.y; vz[2] += cz * z23.x; vz[3] += cz * z23.y;
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double sx = (sLift[(1 * 4 + c) * N2 + j * N1 + k] * fr[i] - sLift[(0 * 4 + c) * N2 + j * N1 + k] * fl[i]) * iw[i];
    const double sy = (sLift[(3 * 4 + c) * N2 + i * N1 + k] * fr[j] - sLift[(2 * 4 + c) * N2 + i * N1 + k] * fl[j]) * iw[j];
    const double sz = (sLift[(5 * 4 + c) * N2 + i * N1 + j] * fr[k] - sLift[(4 * 4 + c) * N2 + i * N1 + j] * fl[k]) * iw[k];
    g[3 * c + 0] = B.cdir[0] * (sx - vx[c]);
    g[3 * c + 1] = B.cdir[1] * (sy - vy[c]);
    g[3 * c + 2] = B.cdir[2] * (sz - vz[c]);
  }
}

// Same, with lift*(s, c, f) at nb[s * nbs + off + f * 4 + c] (in place over Fv.n slots).
template <int N1>
__device__ __forceinline__ void node_gradient_nb(const double* tab, const double* sq, const double* nb, int nbs,
                                                 int off, const BandD& B, int i, int j, int k, double* g) {
  constexpr int N3 = N1 * N1 * N1;
  const double* dh = tab;
  const double* fl = tab + N1 * N1;
  const double* fr = fl + N1;
  const double* iw = fl + 4 * N1;
  const double* lx0 = nb + 0 * nbs + off + (j * N1 + k) * 4;
  const double* lx1 = nb + 1 * nbs + off + (j * N1 + k) * 4;
  const double* ly0 = nb + 2 * nbs + off + (i * N1 + k) * 4;
  const double* ly1 = nb + 3 * nbs + off + (i * N1 + k) * 4;
  const double* lz0 = nb + 4 * nbs + off + (i * N1 + j) * 4;
  const double* lz1 = nb + 5 * nbs + off + (i * N1 + j) * 4;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double* q = sq + c * N3;
    double vx = 0.0, vy = 0.0, vz = 0.0;
#pragma unroll
    for (int m = 0; m < N1; ++m) {
      vx += dh[i * N1 + m] * q[(m * N1 + j) * N1 + k];
      vy += dh[j * N1 + m] * q[(i * N1 + m) * N1 + k];
      vz += dh[k * N1 + m] * q[(i * N1 + j) * N1 + m];
    }
    const double sx = (lx1[c] * fr[i] - lx0[c] * fl[i]) * iw[i];
    const double sy = (ly1[c] * fr[j] - ly0[c] * fl[j]) * iw[j];
    const double sz = (lz1[c] * fr[k] - lz0[c] * fl[k]) * iw[k];
    g[3 * c + 0] = B.cdir[0] * (sx - vx);
    g[3 * c + 1] = B.cdir[1] * (sy - vy);
    g[3 * c + 2] = B.cdir[2] * (sz - vz);
  }
}

// ----------------------------------------------------------------------------
// k_gradient: lift* -> gradient -> Fv.n (conforming sides) / gradient traces
// (sliding and Dirichlet sides).  Also serves compute_gradients (grad_out).
// ----------------------------------------------------------------------------
template <int N1>
__global__ void __launch_bounds__(Dim<N1>::THREADS) k_gradient(const __grid_constant__ ElemConsts C, FieldPtrs P,
                                                               StageArgs A) {
  constexpr int N2 = Dim<N1>::N2, N3 = Dim<N1>::N3, EPB = Dim<N1>::EPB, TAB = Dim<N1>::TAB;
  constexpr int PER = 5 * N3 + 4 * N3 + 12 * N3 + 30 * N2 + 24 * N2;
  extern __shared__ double smem[];
  double* tab = smem;
  load_tables<N1>(C, tab);
  const int e0 = P.e_first + blockIdx.x * EPB;
  load_state<N1>(P.U, e0, P.E, smem + TAB, PER);
  const int le = threadIdx.x / N3, t = threadIdx.x % N3, e = e0 + le;
  const bool active = e < P.E;
  double* su = smem + TAB + le * PER;
  double* sq = su + 5 * N3;
  double* sG = sq + 4 * N3;
  double* sTr = sG + 12 * N3;
  double* sLift = sTr + 30 * N2;
  __syncthreads();
  if (active) {
    double u[5], q[4];
#pragma unroll
    for (int v = 0; v < 5; ++v) u[v] = su[v * N3 + t];
    prim4(u, C.gas, q);
#pragma unroll
    for (int c = 0; c < 4; ++c) sq[c * N3 + t] = q[c];
    face_lift_phase<N1>(C, P, tab, su, e, A.t_stage, sLift, sTr);
  }
  __syncthreads();
  if (active) {
    const int i = t / N2, j = (t / N1) % N1, k = t % N1;
    double g[12];
    node_gradient<N1>(tab, sq, sLift, C.bands[P.coords[4 * e]], i, j, k, g);
#pragma unroll
    for (int c = 0; c < 12; ++c) sG[c * N3 + t] = g[c];
    if (P.grad_out != nullptr) {
      double* go = P.grad_out + (static_cast<size_t>(e) * N3 + t) * 12;
#pragma unroll
      for (int c = 0; c < 12; ++c) go[c] = g[c];
    }
  }
  __syncthreads();
  if (!active) return;
  for (int it = t; it < 6 * N2; it += N3) {
    const int s = it / N2, f = it % N2, a = f / N1, b = f % N1;
    const double* ell = tab + N1 * N1 + (s & 1) * N1;
    double gt[12];
#pragma unroll
    for (int c = 0; c < 12; ++c) gt[c] = prolong1<N1>(sG + c * N3, ell, s >> 1, a, b, face_rot<N1>(s, a, b));
    const int slot = e * 6 + s;
    const int typ = P.side_type[slot], idx = P.side_idx[slot];
    if (typ == kConforming) {
      double fv[4];
      fv_dir(sTr + (s * N2 + f) * 5, gt, s >> 1, C.gas, fv);
      double* dst = P.fvn + (static_cast<size_t>(slot) * N2 + f) * 4;
#pragma unroll
      for (int c = 0; c < 4; ++c) dst[c] = fv[c];
    } else {
      double* dst = (typ == kSliding ? P.slide_g : P.dir_g) + (static_cast<size_t>(idx) * N2 + f) * 12;
#pragma unroll
      for (int c = 0; c < 12; ++c) dst[c] = gt[c];
    }
  }
}

__device__ __forceinline__ void record_error(ErrRec* err, int flag, int step, int stage, long long elem,
                                             long long node, const double* vals) {
  if (atomicCAS(&err->flag, 0, flag) == 0) {
    err->step = step;
    err->stage = stage;
    err->elem = elem;
    err->node = node;
    for (int v = 0; v < 5; ++v) err->vals[v] = vals ? vals[v] : 0.0;
  }
}

// ----------------------------------------------------------------------------
// k_update: the whole rest of the stage for one element (see file header).
// ----------------------------------------------------------------------------
template <int N1, bool VISC>
__global__ void __launch_bounds__(Dim<N1>::THREADS) k_update(const __grid_constant__ ElemConsts C, FieldPtrs P,
                                                             StageArgs A) {
  constexpr int N2 = Dim<N1>::N2, N3 = Dim<N1>::N3, EPB = Dim<N1>::EPB, TAB = Dim<N1>::TAB;
  constexpr int PER = 5 * N3 + 5 * N3 + 24 * N2 + 30 * N2;
  extern __shared__ double smem[];
  double* tab = smem;
  load_tables<N1>(C, tab);
  const int e0 = P.e_first + blockIdx.x * EPB;
  load_state<N1>(P.U, e0, P.E, smem + TAB, PER);
  const int le = threadIdx.x / N3, t = threadIdx.x % N3, e = e0 + le;
  const bool active = e < P.E;
  double* su = smem + TAB + le * PER;
  double* sF = su + 5 * N3;
  double* sLift = sF + 5 * N3;
  double* sFlux = sLift + 24 * N2;
  const int i = t / N2, j = (t / N1) % N1, k = t % N1;
  const BandD& B = C.bands[active ? P.coords[4 * e] : 0];
  __syncthreads();

  // Phase 1: numerical flux on all six sides -> sFlux[s][v][f]; lift* -> sLift.
  if (active) {
    if (VISC) {
      double u[5], q[4];
#pragma unroll
      for (int v = 0; v < 5; ++v) u[v] = su[v * N3 + t];
      prim4(u, C.gas, q);
#pragma unroll
      for (int c = 0; c < 4; ++c) sF[c * N3 + t] = q[c];
    }
    for (int it = t; it < 6 * N2; it += N3) {
      const int s = it / N2, f = it % N2, a = f / N1, b = f % N1, dir = s >> 1;
      const double* ell = tab + N1 * N1 + (s & 1) * N1;
      double own[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) own[v] = prolong1<N1>(su + v * N3, ell, dir, a, b, face_rot<N1>(s, a, b));
      const int slot = e * 6 + s;
      const int typ = P.side_type[slot], idx = P.side_idx[slot];
      double flux[5], lift[4];
      bool ok = true;
      if (typ == kConforming) {
        const double* nb = P.trace + static_cast<size_t>(idx) * N2 * 5 + f * 5;
        double other[5];
#pragma unroll
        for (int v = 0; v < 5; ++v) other[v] = nb[v];
        const double vg = dir == 1 ? B.vg : (dir == 2 ? B.vgz : 0.0);
        const double* um = (s & 1) ? own : other;
        const double* up = (s & 1) ? other : own;
        if (VISC) {
          double qa[4], qb[4];
          prim4(own, C.gas, qa);
          prim4(other, C.gas, qb);
#pragma unroll
          for (int c = 0; c < 4; ++c) lift[c] = __dmul_rn(0.5, __dadd_rn(qa[c], qb[c]));
          double fa[4], fb[4];
          const double* pa = P.fvn + (static_cast<size_t>(slot) * N2 + f) * 4;
          const double* pb = P.fvn + (static_cast<size_t>(idx) * N2 + f) * 4;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            fa[c] = pa[c];
            fb[c] = pb[c];
          }
          ok = face_flux_fv(um, up, dir, vg, (s & 1) ? fa : fb, (s & 1) ? fb : fa, C.gas, flux);
        } else {
          ok = roe_flux(um, up, dir, vg, C.gas, flux);
        }
      } else if (typ == kSliding) {
        const double* sf = P.slide_flux + (static_cast<size_t>(idx) * N2 + f) * 5;
#pragma unroll
        for (int v = 0; v < 5; ++v) flux[v] = sf[v];
        if (VISC) {
          const double* sl = P.slide_lift + (static_cast<size_t>(idx) * N2 + f) * 4;
#pragma unroll
          for (int c = 0; c < 4; ++c) lift[c] = sl[c];
        }
      } else {
        double x[3], ext[5];
        face_position<N1>(C, P.coords + 4 * e, s, a, b, A.t_stage, x);
        eval_case(C.flow_case, x, A.t_stage, C.gas, ext);
        const double vg = dir == 1 ? B.vg : (dir == 2 ? B.vgz : 0.0);
        const double* um = (s & 1) ? own : ext;
        const double* up = (s & 1) ? ext : own;
        if (VISC) {
          prim4(ext, C.gas, lift);
          const double* gd = P.dir_g + (static_cast<size_t>(idx) * N2 + f) * 12;
          double gg[12];
#pragma unroll
          for (int c = 0; c < 12; ++c) gg[c] = gd[c];
          double fm[4], fp[4];
          fv_dir(um, gg, dir, C.gas, fm);
          fv_dir(up, gg, dir, C.gas, fp);
          ok = face_flux_fv(um, up, dir, vg, fm, fp, C.gas, flux);
        } else {
          ok = roe_flux(um, up, dir, vg, C.gas, flux);
        }
      }
      if (!ok) record_error(P.err, 2, A.step, A.stage, e, -1 - it, own);
#pragma unroll
      for (int v = 0; v < 5; ++v) sFlux[(s * 5 + v) * N2 + f] = flux[v];
      if (VISC) {
#pragma unroll
        for (int c = 0; c < 4; ++c) sLift[(s * 4 + c) * N2 + f] = lift[c];
      }
    }
  }
  __syncthreads();

  // Phase 2: pointwise volume flux (ALE convective minus viscous), flux.cpp:7-42.
  double F[3][5];
  double u[5];
  if (active) {
#pragma unroll
    for (int v = 0; v < 5; ++v) u[v] = su[v * N3 + t];
    const double ir = rcp_nr(u[0]);
    const double vv[3] = {u[1] * ir, u[2] * ir, u[3] * ir};
    const double p = pressure(u, ir, C.gas);
    const double vgv[3] = {0.0, B.vg, B.vgz};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      F[d][0] = u[0] * vv[d];
      F[d][1] = u[1] * vv[d] + (d == 0 ? p : 0.0);
      F[d][2] = u[2] * vv[d] + (d == 1 ? p : 0.0);
      F[d][3] = u[3] * vv[d] + (d == 2 ? p : 0.0);
      F[d][4] = (u[4] + p) * vv[d];
#pragma unroll
      for (int v = 0; v < 5; ++v) F[d][v] -= vgv[d] * u[v];
    }
    if (VISC) {
      double g[12];
      node_gradient<N1>(tab, sF, sLift, B, i, j, k, g);
      const double div = g[0] + g[4] + g[8];
      const double mu = C.gas.mu, lam = C.gas.lam;
      const double tau[3][3] = {{2.0 * mu * g[0] + lam * div, mu * (g[1] + g[3]), mu * (g[2] + g[6])},
                                {mu * (g[1] + g[3]), 2.0 * mu * g[4] + lam * div, mu * (g[5] + g[7])},
                                {mu * (g[2] + g[6]), mu * (g[5] + g[7]), 2.0 * mu * g[8] + lam * div}};
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        F[d][1] -= tau[d][0];
        F[d][2] -= tau[d][1];
        F[d][3] -= tau[d][2];
        F[d][4] -= tau[d][0] * vv[0] + tau[d][1] * vv[1] + tau[d][2] * vv[2] + C.gas.kcond * g[9 + d];
      }
    }
  }

  // Phase 3: weak divergence sum_m D-hat(i,m) F(m) per direction (volume_kernel, solver.cpp:372-383).
  double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const double* dh = tab;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    __syncthreads();
    if (active) {
#pragma unroll
      for (int v = 0; v < 5; ++v) sF[v * N3 + t] = F[d][v] * B.sj[d];
    }
    __syncthreads();
    if (active) {
      const int ia = d == 0 ? i : (d == 1 ? j : k);
      const int base = d == 0 ? j * N1 + k : (d == 1 ? i * N2 + k : (i * N1 + j) * N1);
      const int stride = d == 0 ? N2 : (d == 1 ? N1 : 1);
#pragma unroll
      for (int m = 0; m < N1; ++m) {
        const double c = dh[ia * N1 + m];
#pragma unroll
        for (int v = 0; v < 5; ++v) acc[v] += c * sF[v * N3 + base + m * stride];
      }
    }
  }

  // Phase 4: surface lift (apply_all_faces, solver.cpp:547-582), sides X-,X+,Y-,Y+,Z-,Z+.
  double du[5];
  if (active) {
#pragma unroll
    for (int v = 0; v < 5; ++v) du[v] = acc[v] * B.inv_jac;
    const double* lw = tab + N1 * N1 + 2 * N1;
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int dir = s >> 1;
      const int ia = dir == 0 ? i : (dir == 1 ? j : k);
      const int f = dir == 0 ? j * N1 + k : (dir == 1 ? i * N1 + k : i * N1 + j);
      const double c = ((s & 1) ? -1.0 : 1.0) * B.cdir[dir] * lw[(s & 1) * N1 + ia];
      if (c != 0.0) {
#pragma unroll
        for (int v = 0; v < 5; ++v) du[v] += c * sFlux[(s * 5 + v) * N2 + f];
      }
    }
  }
  __syncthreads();
  if (active) {
#pragma unroll
    for (int v = 0; v < 5; ++v) sF[v * N3 + t] = du[v];
  }
  __syncthreads();

  // Phase 5: flat coalesced RK update (solver.cpp:912-917) or residual store.
  const int n_el = min(EPB, P.E - e0);
  const size_t gbase = static_cast<size_t>(e0) * 5 * N3;
  constexpr int PERB = 5 * N3 + 5 * N3 + 24 * N2 + 30 * N2;
  double* elems = smem + TAB;
  if (A.mode == 1) {
    for (int fI = threadIdx.x; fI < n_el * 5 * N3; fI += blockDim.x) {
      const int l = fI / (5 * N3), r = fI - l * 5 * N3;
      P.out[gbase + fI] = elems[l * PERB + 5 * N3 + (r % 5) * N3 + r / 5];
    }
    return;
  }
  for (int fI = threadIdx.x; fI < n_el * 5 * N3; fI += blockDim.x) {
    const int l = fI / (5 * N3), r = fI - l * 5 * N3;
    double* us = elems + l * PERB + (r % 5) * N3 + r / 5;
    const double d = us[5 * N3];
    const double rg = A.rk_a * P.reg[gbase + fI] + A.dt * d;
    const double un = *us + A.rk_b * rg;
    P.reg[gbase + fI] = rg;
    P.U[gbase + fI] = un;
    *us = un;
  }
  __syncthreads();
  if (!active) return;
  // Admissibility (check_admissible, solver.cpp:892-906).
  {
    double w[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) w[v] = su[v * N3 + t];
    const double p = pressure(w, rcp_nr(w[0]), C.gas);
    bool ok = w[0] > 0.0 && p > 0.0;
#pragma unroll
    for (int v = 0; v < 5; ++v) ok = ok && isfinite(w[v]);
    if (!ok) record_error(P.err, 2, A.step, A.stage, e, t, w);
  }
  // Face traces of the new state for the next stage.
  for (int it = t; it < 6 * N2; it += N3) {
    const int s = it / N2, f = it % N2, a = f / N1, b = f % N1;
    const double* ell = tab + N1 * N1 + (s & 1) * N1;
    double* dst = P.trace_out + (static_cast<size_t>(e) * 6 + s) * N2 * 5 + f * 5;
#pragma unroll
    for (int v = 0; v < 5; ++v) dst[v] = prolong1<N1>(su + v * N3, ell, s >> 1, a, b, face_rot<N1>(s, a, b));
  }
}

// ----------------------------------------------------------------------------
// CFL time step (suggest_dt, solver.cpp:929-947): min over elements via an
// order-preserving atomicMin on the bits of positive doubles.
// ----------------------------------------------------------------------------
template <int N1>
__global__ void __launch_bounds__(Dim<N1>::THREADS) k_suggest_dt(const __grid_constant__ ElemConsts C, FieldPtrs P,
                                                                 double cfl, int degree, unsigned long long* out) {
  constexpr int N3 = Dim<N1>::N3, EPB = Dim<N1>::EPB;
  __shared__ double red[Dim<N1>::THREADS];
  const int le = threadIdx.x / N3, t = threadIdx.x % N3, e = blockIdx.x * EPB + le;
  double lm = 0.0;
  if (e < P.E) {
    const double* u = P.U + (static_cast<size_t>(e) * N3 + t) * 5;
    const BandD& B = C.bands[P.coords[4 * e]];
    const bool ann = C.mapping == SDG_MAP_ANNULUS;
    const double ir = 1.0 / u[0];
    const double a = u[1] * ir, b = u[2] * ir - (ann ? 0.0 : B.vg), c = u[3] * ir - (ann ? 0.0 : B.vgz);
    const double p = pressure(u, ir, C.gas);
    lm = sqrt(a * a + b * b + c * c) + sqrt(C.gas.gamma * p * ir);
    if (ann) lm += fabs(B.vg) * (C.z0 + B.hz * C.nz);  // tip speed of a rotating band
  }
  red[threadIdx.x] = lm;
  __syncthreads();
  if (t == 0 && e < P.E) {
    double m = 0.0;
    for (int q = 0; q < N3; ++q) m = fmax(m, red[le * N3 + q]);
    const BandD& B = C.bands[P.coords[4 * e]];
    const double h = C.mapping == SDG_MAP_ANNULUS ? fmin(B.hx, fmin(B.hy * C.z0, B.hz)) : fmin(B.hx, fmin(B.hy, B.hz));
    const double dt = cfl * h / (m * (2.0 * degree + 1.0));
    atomicMin(out, static_cast<unsigned long long>(__double_as_longlong(dt)));
  }
}

// ----------------------------------------------------------------------------
// Device pairing (paper §4.4 / Appendix A; partition.cpp:85-169; solver.cpp:156-206):
// per interface side the displacement (bit-exact scalar chain of mesh.cpp:9-25),
// the mortar tuples, their nested sort by (partner, iface, i_par, i_perp, i_sub)
// and the inverse map m.  The 5-key order restricted to one partner equals the
// order of the dense key d = base[iface] + (i_par*n_perp + i_perp)*2 + i_sub, so
// the sort is a per-partner counting pass over the dense key range.
// One CTA per role.
// ----------------------------------------------------------------------------
constexpr int kPairThreads = 1024;
constexpr int kPairPartners = 16;

__device__ __forceinline__ long long pmod(long long a, long long n) {
  const long long r = a % n;
  return r < 0 ? r + n : r;
}

__global__ void __launch_bounds__(kPairThreads) k_pairing(const __grid_constant__ PairingArgs A, PairingPtrs P) {
  const int role = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kPairThreads / 32;
  __shared__ long long s_nd[kMaxCtx];
  __shared__ int s_conf[kMaxCtx];
  __shared__ int cnt[kPairPartners], base[kPairPartners], carry[kPairPartners];
  __shared__ int wcnt[kPairPartners][NW];
  __shared__ int s_bad;
  if (tid < kPairPartners) {
    cnt[tid] = 0;
    carry[tid] = 0;
  }
  if (tid == 0) s_bad = 0;
  if (tid < A.n_ctx) {
    const CtxD& c = A.ctx[tid];
    const double delta = __dadd_rn(A.delta_base[tid], __dmul_rn(c.vg_rel, __dsub_rn(A.t_stage, A.time)));
    const double period = __dmul_rn(c.l_par, static_cast<double>(c.n_par));
    double d = fmod(delta, period);
    if (d < 0.0) d = __dadd_rn(d, period);
    const double ratio = __ddiv_rn(d, c.l_par);
    long long nd = static_cast<long long>(floor(ratio));
    double sd = __dsub_rn(ratio, static_cast<double>(nd));
    if (nd >= c.n_par) {
      nd = 0;
      sd = 0.0;
    }
    s_nd[tid] = nd;
    s_conf[tid] = sd == 0.0;
    if (role == 0) {
      P.ctx_state[2 * tid] = static_cast<int>(nd);
      P.ctx_state[2 * tid + 1] = sd == 0.0;
      P.ctx_sdelta[tid] = sd;
    }
  }
  int* pres = P.pres[role];
  int* payload = P.payload[role];
  for (long long d = tid; d < A.dense_size; d += kPairThreads) pres[d] = -1;
  for (int r = 0; r < A.role_nctx[role]; ++r) {
    const CtxD& c = A.ctx[A.role_ctx[role][r]];
    for (int q = tid; q < 2 * c.n_faces; q += kPairThreads) P.m[2 * c.face_off + q] = -1;
  }
  __syncthreads();
  // Tuples (append_mortar_tuples): dense key, partner and passive payload.
  for (int r = 0; r < A.role_nctx[role]; ++r) {
    const int ci = A.role_ctx[role][r];
    const CtxD& c = A.ctx[ci];
    const long long nd = s_nd[ci];
    const int conf = s_conf[ci];
    for (int q = tid; q < 2 * c.n_faces; q += kPairThreads) {
      const int f = q >> 1, sub = q & 1;
      if (conf && sub == 0) continue;
      const long long fpar = P.ctx_face_par[c.face_off + f], fperp = P.ctx_face_perp[c.face_off + f];
      long long ipar;
      int partner;
      if (c.on_static) {
        ipar = fpar;
        partner = P.partner_map[c.map_off + fperp * c.n_par + pmod(fpar - nd + sub - 1, c.n_par)];
      } else {
        ipar = pmod(fpar + nd - sub + 1, c.n_par);
        partner = P.partner_map[c.map_off + fperp * c.n_par + ipar];
      }
      if (partner < 0 || partner >= kPairPartners) {
        s_bad = 1;
        continue;
      }
      const long long d = A.iface_base[c.iface] + (ipar * c.n_perp + fperp) * 2 + sub;
      pres[d] = partner;
      payload[d] = (ci << 24) | f;
      atomicAdd(&cnt[partner], 1);
    }
  }
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int p = 0; p < kPairPartners; ++p) {
      base[p] = acc;
      acc += cnt[p];
    }
    P.n_mortars[role] = acc;
    if (s_bad || (A.expect_mortars[role] >= 0 && A.expect_mortars[role] != acc)) {
      if (atomicCAS(&P.err->flag, 0, 3) == 0) {
        P.err->elem = role;
        P.err->node = acc;
      }
    }
  }
  __syncthreads();
  // Positions (sort_index_array + build_mapping): one coalesced pass over the dense
  // key range in chunks of the block; per partner, rank = running carry + warp
  // offset + lane prefix from ballots.
  const unsigned lt = (1u << lane) - 1u;
  for (long long c0 = 0; c0 < A.dense_size; c0 += kPairThreads) {
    const long long d = c0 + tid;
    const int p = d < A.dense_size ? pres[d] : -1;
    if (lane < kPairPartners) wcnt[lane][warp] = 0;
    __syncwarp();
    const unsigned peers = __match_any_sync(0xffffffffu, p);
    const int my_pref = __popc(peers & lt);
    if (p >= 0 && my_pref == 0) wcnt[p][warp] = __popc(peers);
    __syncthreads();
    if (p >= 0) {
      int off = base[p] + carry[p] + my_pref;
      for (int w = 0; w < warp; ++w) off += wcnt[p][w];
      const int pos = off;
      int ifc = 0;
      for (int x = 1; x < A.n_ifaces; ++x)
        if (d >= A.iface_base[x]) ifc = x;
      long long rest = d - A.iface_base[ifc];
      const int sub = static_cast<int>(rest & 1);
      rest >>= 1;
      const long long np = A.iface_nperp[ifc];
      const int iperp = static_cast<int>(rest % np), ipar = static_cast<int>(rest / np);
      const int pl = payload[d];
      const int ci = pl >> 24, f = pl & 0xffffff;
      int* col = P.cols[role] + 7 * pos;
      col[0] = p;
      col[1] = ifc;
      col[2] = ipar;
      col[3] = iperp;
      col[4] = sub;
      col[5] = f;
      col[6] = ci;
      const CtxD& c = A.ctx[ci];
      P.m[2 * c.face_off + sub * c.n_faces + f] = pos;
    }
    __syncthreads();
    if (tid < kPairPartners) {
      int tot = 0;
      for (int w = 0; w < NW; ++w) tot += wcnt[tid][w];
      carry[tid] += tot;
    }
    __syncthreads();
  }
}

// ----------------------------------------------------------------------------
// Mortar kernels (fill_mortar_solution / send_gradient_phase / run_lifting /
// mortar_flux_phase / mortar_apply_phase; solver.cpp:234-252, 657-714, 806-831,
// 442-526).  The 1D operators act along the sliding axis j for every k line.
// ----------------------------------------------------------------------------
template <int N1>
__device__ __forceinline__ void load_ops(const MortarOps& ops, int n_ctx, double* s_ops) {
  for (int q = threadIdx.x; q < n_ctx * 2 * N1 * N1; q += blockDim.x) {
    const int c = q / (2 * N1 * N1), r = q % (2 * N1 * N1), h = r / (N1 * N1), x = r % (N1 * N1);
    s_ops[q] = ops.op[c][h][x];
  }
}

// Windings k of a mortar column of a periodic annulus sector (its moving partner sits at
// the static location + k * sector angle).
__device__ __forceinline__ int mortar_wind(const MortarPtrs& P, const int* cols, int mc) {
  const int ci = cols[7 * mc + 6];
  const int raw = cols[7 * mc + 2] - P.ctx_state[2 * ci] + cols[7 * mc + 4] - 1;
  return P.wind[ci] + (raw < 0 ? 1 : 0);
}

template <int N1, int NC>
__global__ void k_mortar_fill(const __grid_constant__ MortarOps ops, int n_ctx, MortarPtrs P, const double* src,
                              double* dst0, double* dst1) {
  constexpr int N2 = N1 * N1;
  __shared__ double s_ops[kMaxCtx * 2 * N1 * N1];
  load_ops<N1>(ops, n_ctx, s_ops);
  __syncthreads();
  const int item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= P.S * 2 * N2) return;
  const int ks = item / (2 * N2), sub = (item / N2) & 1, node = item % N2, jm = node / N1, kk = node % N1;
  const int ci = P.slide_ctx[ks], f = P.slide_f[ks];
  if (ci < 0) return;  // a face of a non-matching interface (tensor-product chain)
  const int conf = P.ctx_state[2 * ci + 1];
  if (conf && sub == 0) return;
  const int role = P.ctx_role[ci];
  const int mi = P.m[2 * P.ctx_face_off[ci] + sub * P.ctx_nf[ci] + f];
  const double* s = NC == 5 ? src + (static_cast<size_t>(P.slide_elem[ks]) * 6 + P.slide_side[ks]) * N2 * NC
                            : src + static_cast<size_t>(ks) * N2 * NC;
  double* d = (role == 0 ? dst0 : dst1) + (static_cast<size_t>(mi) * N2 + node) * NC;
  if (conf) {
#pragma unroll
    for (int c = 0; c < NC; ++c) d[c] = s[node * NC + c];
    return;
  }
  const int half = role == 0 ? sub : 1 - sub;
  const double* op = s_ops + (ci * 2 + half) * N2 + jm * N1;
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
#pragma unroll
  for (int jj = 0; jj < N1; ++jj) {
    const double w = op[jj];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] += w * s[(jj * N1 + kk) * NC + c];
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) d[c] = acc[c];
}

template <int N1>
__global__ void k_mortar_lift(GasD g, MortarPtrs P, int max_mortars) {
  constexpr int N2 = N1 * N1;
  const int item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= max_mortars * N2 || item / N2 >= P.n_mortars[0]) return;
  const size_t q = static_cast<size_t>(item);
  double a[4], b[4], th[5];
#pragma unroll
  for (int v = 0; v < 5; ++v) th[v] = P.u_theirs[q * 5 + v];
  if (P.sector) {  // the moving partner's state at the static location: R(-k alpha)
    double sn, cs;
    sincos(-mortar_wind(P, P.cols_static, item / N2) * P.alpha, &sn, &cs);
    rot_yz(cs, sn, th[2], th[3]);
  }
  prim4(P.u_mine[0] + q * 5, g, a);
  prim4(th, g, b);
#pragma unroll
  for (int c = 0; c < 4; ++c) P.lift[0][q * 4 + c] = __dmul_rn(0.5, __dadd_rn(a[c], b[c]));
}

template <int N1, int NC>
__global__ void k_mortar_backproject(const __grid_constant__ MortarOps ops, int n_ctx, MortarPtrs P,
                                     const double* src0, const double* src1, double* dst) {
  constexpr int N2 = N1 * N1;
  __shared__ double s_ops[kMaxCtx * 2 * N1 * N1];
  load_ops<N1>(ops, n_ctx, s_ops);
  __syncthreads();
  const int item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= P.S * N2) return;
  const int ks = item / N2, node = item % N2, jj = node / N1, kk = node % N1;
  const int ci = P.slide_ctx[ks], f = P.slide_f[ks];
  if (ci < 0) return;  // a face of a non-matching interface (tensor-product chain)
  const int conf = P.ctx_state[2 * ci + 1];
  const int role = P.ctx_role[ci];
  const double* src = role == 0 ? src0 : src1;
  const int* mrow = P.m + 2 * P.ctx_face_off[ci];
  const int nf = P.ctx_nf[ci];
  double* d = dst + (static_cast<size_t>(ks) * N2 + node) * NC;
  // Periodic annulus sector, moving role: each mortar's values (computed by the static side at
  // its location) rotate by R(+k alpha) to the moving element; (y, z) at OY, OY + 1.
  constexpr int OY = NC == 4 ? 1 : 2;
  const bool rot = P.sector && role == 1;
  if (conf) {
    const double* s = src + (static_cast<size_t>(mrow[nf + f]) * N2 + node) * NC;
    double o[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) o[c] = s[c];
    if (rot) {
      double sn, cs;
      sincos(mortar_wind(P, P.cols_moving, mrow[nf + f]) * P.alpha, &sn, &cs);
      rot_yz(cs, sn, o[OY], o[OY + 1]);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) d[c] = o[c];
    return;
  }
  double out[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) out[c] = 0.0;
#pragma unroll
  for (int sub = 0; sub < 2; ++sub) {
    const int half = role == 0 ? sub : 1 - sub;
    const double* op = s_ops + (ci * 2 + half) * N2 + jj * N1;
    const double* s = src + static_cast<size_t>(mrow[sub * nf + f]) * N2 * NC;
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.0;
#pragma unroll
    for (int jm = 0; jm < N1; ++jm) {
      const double w = op[jm];
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[c] += w * s[(jm * N1 + kk) * NC + c];
    }
    if (rot) {
      double sn, cs;
      sincos(mortar_wind(P, P.cols_moving, mrow[sub * nf + f]) * P.alpha, &sn, &cs);
      rot_yz(cs, sn, acc[OY], acc[OY + 1]);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) out[c] += acc[c];
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) d[c] = out[c];
}

template <int N1, bool VISC>
__global__ void k_mortar_flux(GasD g, MortarPtrs P, int max_mortars, ErrRec* err) {
  constexpr int N2 = N1 * N1;
  const int item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= max_mortars * N2) return;
  const int mc = item / N2;
  if (mc >= P.n_mortars[0]) return;
  const int ci = P.cols_static[7 * mc + 6];
  const bool static_left = P.ctx_static_left[ci] != 0;
  const size_t q = static_cast<size_t>(item);
  const double* mine = P.u_mine[0] + q * 5;
  double th[5];
#pragma unroll
  for (int v = 0; v < 5; ++v) th[v] = P.u_theirs[q * 5 + v];
  double sn = 0.0, cs = 1.0;
  if (P.sector) {  // the moving partner's values at the static location: R(-k alpha)
    sincos(-mortar_wind(P, P.cols_static, mc) * P.alpha, &sn, &cs);
    rot_yz(cs, sn, th[2], th[3]);
  }
  const double* theirs = th;
  double f[5];
  bool ok;
  if (VISC) {
    double fm[4], ft[4];
    fv_dir(mine, P.g_mine[0] + q * 12, 0, g, fm);
    fv_dir(P.u_theirs + q * 5, P.g_theirs + q * 12, 0, g, ft);  // Fv . e_x in the partner's frame ...
    if (P.sector) rot_yz(cs, sn, ft[1], ft[2]);                // ... rotated (e_x is the rotation axis)
    ok = static_left ? face_flux_fv(mine, theirs, 0, 0.0, fm, ft, g, f)
                     : face_flux_fv(theirs, mine, 0, 0.0, ft, fm, g, f);
  } else {
    ok = static_left ? roe_flux(mine, theirs, 0, 0.0, g, f) : roe_flux(theirs, mine, 0, 0.0, g, f);
  }
  if (!ok) record_error(err, 2, -1, -1, -1, mc, mine);
#pragma unroll
  for (int v = 0; v < 5; ++v) P.flux[0][q * 5 + v] = f[v];
}


// ----------------------------------------------------------------------------
// Diagnostics: quadrature integrals of mass and energy and the L2 / Linf
// error against the exact case state (diagnostics.cpp:31-87).  Each block
// reduces in a fixed tree and writes its partials; the host sums the
// partials in block order, so results are run-to-run reproducible.
// ----------------------------------------------------------------------------
template <int N1>
__global__ void __launch_bounds__(256) k_diag(const __grid_constant__ ElemConsts C, FieldPtrs P, double t,
                                              int with_exact, double* partial) {
  constexpr int N2 = N1 * N1, N3 = N2 * N1;
  double a[kDiagVals];
#pragma unroll
  for (int q = 0; q < kDiagVals; ++q) a[q] = 0.0;
  const long long nodes = static_cast<long long>(P.E) * N3;
  for (long long nd = blockIdx.x * 256LL + threadIdx.x; nd < nodes; nd += 256LL * gridDim.x) {
    const int e = static_cast<int>(nd / N3), r = static_cast<int>(nd % N3);
    const int i = r / N2, j = (r / N1) % N1, k = r % N1;
    const int* crd = P.coords + 4 * e;
    const BandD& B = C.bands[crd[0]];
    const int mw = C.mapping == SDG_MAP_ANNULUS ? 13 : 10;  // device layout met[e][c][node] (curved.cuh)
    const double wq = C.w[i] * C.w[j] * C.w[k] *
                      (C.mapping != SDG_MAP_BOX ? 1.0 / P.met[(static_cast<size_t>(e) * mw + 9) * N3 + r] : B.jac);
    const double* u = P.U + nd * 5;
    a[0] += wq * u[0];
    a[1] += wq * u[4];
    a[2] += wq;
    if (with_exact) {
      double x[3], ex[5];
      map_position(C, crd, C.x[i], C.x[j], C.x[k], t, x);
      eval_case(C.flow_case, x, t, C.gas, ex);
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        const double d = u[v] - ex[v];
        a[3 + v] += wq * d * d;
        a[8 + v] = fmax(a[8 + v], fabs(d));
      }
    }
  }
  __shared__ double red[8][kDiagVals];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < kDiagVals; ++q) {
    double v = a[q];
    for (int o = 16; o > 0; o >>= 1) {
      const double y = __shfl_down_sync(0xffffffffu, v, o);
      v = (q >= 8 && q < 13) ? fmax(v, y) : v + y;
    }
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < kDiagVals) {
    const int q = threadIdx.x;
    double v = red[0][q];
    for (int w = 1; w < 8; ++w) v = (q >= 8 && q < 13) ? fmax(v, red[w][q]) : v + red[w][q];
    partial[static_cast<size_t>(blockIdx.x) * kDiagVals + q] = v;
  }
}

template <int N1>
int smem_gradient() {
  constexpr int N2 = N1 * N1, N3 = N2 * N1;
  return (Dim<N1>::TAB + Dim<N1>::EPB * (21 * N3 + 54 * N2)) * 8;
}
template <int N1>
int smem_update() {
  constexpr int N2 = N1 * N1, N3 = N2 * N1;
  return (Dim<N1>::TAB + Dim<N1>::EPB * (10 * N3 + 54 * N2)) * 8;
}
template <int N1>
int smem_prolong() {
  return (Dim<N1>::TAB + Dim<N1>::EPB * 5 * Dim<N1>::N3) * 8;
}

inline void check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw DeviceError(SDG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ============================================================================
// Persistent, TMA-pipelined element kernels (even N+1: every per-element and
// per-face-slot block is a multiple of 16 bytes, as cp.async.bulk requires).
//
// Each CTA owns a strided sequence of element tiles.  One thread issues, per
// tile, cp.async.bulk copies of everything the tile reads from HBM — the
// element state, the RK register, its own Fv.n slots and, per side, the
// neighbour's trace + Fv.n slot (or the sliding face's back-projected flux +
// lift*) — into one of two shared-memory stages, completing on an mbarrier,
// while the CTA computes the previous tile from the other stage.  Outputs
// (new state, register, face traces, Fv.n) are assembled in shared memory and
// written back with cp.async.bulk stores.  The compute phases are those of
// k_gradient / k_update above.
// ============================================================================
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void consumer_sync(int n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

constexpr int kCodeShift = 29;

// Element tiles of the persistent TMA gradient kernel (k_gradient_ws): one element
// per tile, eight at N = 1.
template <int N1>
struct Tma {
  static constexpr int N2 = N1 * N1, N3 = N2 * N1;
  static constexpr int EPB = N1 == 2 ? 8 : 1;
};

// Side codes of one tile (8 ints per element) into shared memory, asynchronously.
template <int N1>
__device__ __forceinline__ void prefetch_codes(const FieldPtrs& P, int tile, int* dst) {
  using D = Tma<N1>;
  const int e0 = P.e_first + tile * D::EPB;
  const int n = min(D::EPB, P.E - e0);
  for (int q = 0; q < n * 2; ++q) cp_async16(dst + 4 * q, P.side_code + 8 * e0 + 4 * q);
  cp_async_commit();
}

// Prolongation of one variable from an AoS [node][5] element block (same rotated order as prolong1).
template <int N1>
__device__ __forceinline__ double prolong_aos(const double* __restrict__ s, int v, const double* __restrict__ ell,
                                              int dir, int a, int b, int rot) {
  constexpr int N2 = N1 * N1;
  const int base = dir == 0 ? a * N1 + b : (dir == 1 ? a * N2 + b : (a * N1 + b) * N1);
  const int stride = dir == 0 ? N2 : (dir == 1 ? N1 : 1);
  double acc = 0.0;
#pragma unroll
  for (int m = 0; m < N1; ++m) {
    const int mr = rot_index<N1>(m, rot);
    acc = __fma_rn(ell[mr], s[(base + mr * stride) * 5 + v], acc);
  }
  return acc;
}

// XOR swizzle of the node index inside the [row][node] blocks q and g of k_gradient_ws
// (N+1 = 4 and 8, where a node row is a whole number of half-warps): lines along
// j and k start at multiples of N+1, so unswizzled all 16 lines of a half-warp of line
// tasks fall on 4 (N+1 = 4) or 2 (N+1 = 8) banks.  With the swizzle node rows, lines in
// all three directions and face-node prolongations are conflict-free.
template <int N1>
__device__ __forceinline__ int swz(int n) {
  if constexpr (N1 == 8) {
    const int i = n >> 6, j = (n >> 3) & 7;
    return n ^ ((i & 1) << 3) ^ j;
  } else if constexpr (N1 == 4) {
    const int i = n >> 4;
    return n ^ (i << 2) ^ i;
  } else {
    return n;
  }
}

// BR1 gradient by line tasks: task (d, c, line) loads q along the line once and
// produces g[3c+d] on all N1 nodes of that line; D-hat, l(+-1) and 1/w enter as
// compile-time-indexed kernel-parameter (constant bank) operands
// (assemble_gradients, solver.cpp:729-768).  lift(s, c, f) = lift[s * ls + f * lf + c * lc].
template <int N1>
__device__ __forceinline__ void gradient_lines(const ElemConsts& C, const BandD& B, const double* __restrict__ q,
                                               const double* __restrict__ lift, int ls, const int* lfs, int lc,
                                               double* __restrict__ g, int t, int nt) {
  constexpr int N2 = N1 * N1, N3 = N2 * N1;
  for (int task = t; task < 12 * N2; task += nt) {
    const int d = task / (4 * N2), rem = task - d * 4 * N2, c = rem / N2, f = rem - c * N2;
    const int a = f / N1, b = f - a * N1;
    const int base = d == 0 ? a * N1 + b : (d == 1 ? a * N2 + b : (a * N1 + b) * N1);
    const int stride = d == 0 ? N2 : (d == 1 ? N1 : 1);
    double x[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) x[m] = q[c * N3 + swz<N1>(base + m * stride)];
    const double lm = lift[(2 * d) * ls + f * lfs[2 * d] + c * lc];
    const double lp = lift[(2 * d + 1) * ls + f * lfs[2 * d + 1] + c * lc];
    const double cd = B.cdir[d];
    double* out = g + (3 * c + d) * N3;
#pragma unroll
    for (int o = 0; o < N1; ++o) {
      double vol = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) vol += C.dhat[o * kMaxN1 + m] * x[m];
      const double surf = (lp * C.fr[o] - lm * C.fl[o]) * C.inv_w[o];
      out[swz<N1>(base + o * stride)] = cd * (surf - vol);
    }
  }
}

// Components of the gradient trace that Fv.n along `dir` needs (flux.cpp:23-42):
// the divergence, the row/column of the velocity gradient and dT/d(dir).
__host__ __device__ constexpr int fv_comp(int dir, int q) {
  // dir 0: {0,1,2,3,4,6,8,9}  dir 1: {0,1,3,4,5,7,8,10}  dir 2: {0,2,4,5,6,7,8,11}
  return dir == 0 ? (q < 5 ? q : (q == 5 ? 6 : (q == 6 ? 8 : 9)))
                  : dir == 1 ? (q == 0 ? 0 : q == 1 ? 1 : q == 2 ? 3 : q == 3 ? 4 : q == 4 ? 5 : q == 5 ? 7 : q == 6 ? 8 : 10)
                             : (q == 0 ? 0 : q == 1 ? 2 : q == 2 ? 4 : q == 3 ? 5 : q == 4 ? 6 : q == 5 ? 7 : q == 6 ? 8 : 11);
}

template <int N1, int DIR>
__device__ __forceinline__ void fvn_item(const ElemConsts& C, const double* gS, const double* ell, int a, int b,
                                         int rot, const double* own, double* out) {
  constexpr int N2 = N1 * N1, N3 = N2 * N1;
  const int base = DIR == 0 ? a * N1 + b : (DIR == 1 ? a * N2 + b : (a * N1 + b) * N1);
  constexpr int stride = DIR == 0 ? N2 : (DIR == 1 ? N1 : 1);
  double gt[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) gt[q] = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int c = fv_comp(DIR, q);
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < N1; ++m) {
      const int mr = rot_index<N1>(m, rot);
      acc = __fma_rn(ell[mr], gS[c * N3 + swz<N1>(base + mr * stride)], acc);
    }
    gt[c] = acc;
  }
  fv_dir(own, gt, DIR, C.gas, out);
}

// ============================================================================
// v5 element kernels.  Differences from the kernels above:
//  * the element's own face traces are staged by TMA (the slots the previous
//    k_update wrote) instead of being recomputed — the own trace is then the
//    very bits every neighbour reads;
//  * side codes and the band index come from the cp.async-prefetched copy in
//    shared memory (three rotating buffers), no global loads in the tile loop;
//  * the RK register is single-buffered (own mbarrier, loaded during the tile);
//  * new face traces are written in place over the consumed own-trace stage
//    and bulk-stored; prolongation directions are compile-time.
// ============================================================================
template <int N1>
struct T5 {
  static constexpr int N2 = N1 * N1, N3 = N2 * N1;
  static constexpr int EPB = Tma<N1>::EPB;
  static constexpr int THREADS = EPB * N3;
  static constexpr int MINB = N1 == 2 ? 3 : (N1 == 8 ? 1 : (N1 == 4 ? 4 : 2));
  static constexpr int TAB = Dim<N1>::TAB;
  static constexpr int EL = 5 * N3, TS = 5 * N2, FS = 4 * N2, NB = TS + FS;
  // update stage: U | reg | own traces | own Fv.n | neighbour (trace|flux, Fv.n|lift)
  static constexpr int U_STAGE = EPB * (2 * EL + 6 * TS + 6 * FS + 6 * NB);
  static constexpr int U_SMEM = (TAB + 2 * U_STAGE + EPB * 5 * N3) * 8 + 64;
  // gradient stage: U | own traces | neighbour (trace|lift)
  static constexpr int G_STAGE = EPB * (EL + 12 * TS);
  static constexpr int G_SMEM = (TAB + 2 * G_STAGE + EPB * 4 * N3 + EPB * 12 * N3 + EPB * 6 * FS) * 8 + 64;
};

template <int N1>
__device__ __forceinline__ void issue_gradient_loads5(const FieldPtrs& P, int tile, const int* codes, double* st,
                                                      uint64_t* bar) {
  using D = T5<N1>;
  const int e0 = P.e_first + tile * D::EPB;
  const int n = min(D::EPB, P.E - e0);
  uint32_t bytes = n * (D::EL + 6u * D::TS) * 8u;
  for (int le = 0; le < n; ++le)
    for (int s = 0; s < 6; ++s) {
      const int typ = codes[8 * le + s] >> kCodeShift;
      if (typ == kConforming) bytes += D::TS * 8u;
      else if (typ == kSliding) bytes += D::FS * 8u;
    }
  mbar_arrive_expect_tx(bar, bytes);
  bulk_g2s(st, P.U + static_cast<size_t>(e0) * D::EL, n * D::EL * 8u, bar);
  bulk_g2s(st + D::EPB * D::EL, P.trace + static_cast<size_t>(e0) * 6 * D::TS, n * 6u * D::TS * 8u, bar);
  double* sNb = st + D::EPB * (D::EL + 6 * D::TS);
  for (int le = 0; le < n; ++le)
    for (int s = 0; s < 6; ++s) {
      const int code = codes[8 * le + s];
      const int typ = code >> kCodeShift, idx = code & ((1 << kCodeShift) - 1);
      double* nb = sNb + (le * 6 + s) * D::TS;
      if (typ == kConforming) bulk_g2s(nb, P.trace + static_cast<size_t>(idx) * D::TS, D::TS * 8u, bar);
      else if (typ == kSliding) bulk_g2s(nb, P.slide_lift + static_cast<size_t>(idx) * D::FS, D::FS * 8u, bar);
    }
}

// ---------------------------------------------------------------------------
// Warp-specialised k_gradient: the same phases as k_gradient5 on
// the consumer warps (EPB*N3 threads rounded up to whole warps, synchronised by
// named barrier 1), plus one producer warp that owns every asynchronous copy:
// side-code prefetch, the TMA stage loads (full[s] barriers), and the bulk
// store of the tile's Fv.n once the consumers have released the tile
// (empty[s]), followed by the wFv-free signal the next tile's phase 3 waits on.
// No consumer thread ever waits on a copy it did not need.
template <int N1>
struct GWs {
  static constexpr int CONSUMERS = (T5<N1>::THREADS + 31) / 32 * 32;
  static constexpr int THREADS = CONSUMERS + 32;
};


template <int N1>
__global__ void __launch_bounds__(GWs<N1>::THREADS, T5<N1>::MINB) k_gradient_ws(const __grid_constant__ ElemConsts C,
                                                                              FieldPtrs P, StageArgs A) {
  using D = T5<N1>;
  constexpr int N2 = D::N2, N3 = D::N3, EPB = D::EPB, NC = GWs<N1>::CONSUMERS;
  extern __shared__ __align__(128) double smem[];
  double* tab = smem;
  double* stage0 = smem + D::TAB;
  double* wQ = stage0 + 2 * D::G_STAGE;  // EPB x 4 N3
  double* wG = wQ + EPB * 4 * N3;        // EPB x 12 N3
  double* wFv = wG + EPB * 12 * N3;      // EPB x 6 FS
  uint64_t* full = reinterpret_cast<uint64_t*>(wFv + EPB * 6 * D::FS);
  uint64_t* empty = full + 2;
  uint64_t* fv_free = full + 4;
  __shared__ __align__(16) int codes[3][8 * EPB];
  __shared__ int lstr[EPB][6];
  load_tables<N1>(C, tab);
  const int tiles = (P.E - P.e_first + EPB - 1) / EPB;
  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&empty[0], 1);
    mbar_init(&empty[1], 1);
    mbar_init(fv_free, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x >= NC) {
    // ---------------- producer warp (one elected lane)
    if (threadIdx.x != NC) return;
    int tile = blockIdx.x;
    if (tile < tiles) {
      prefetch_codes<N1>(P, tile, codes[0]);
      cp_async_wait_all();
      issue_gradient_loads5<N1>(P, tile, codes[0], stage0, &full[0]);
      if (tile + gridDim.x < tiles) prefetch_codes<N1>(P, tile + gridDim.x, codes[1]);
    }
    for (int it = 0; tile < tiles; ++it, tile += gridDim.x) {
      const int next = tile + gridDim.x;
      if (next < tiles) {
        cp_async_wait_all();  // codes of `next`
        fence_proxy_async();
        issue_gradient_loads5<N1>(P, next, codes[(it + 1) % 3], stage0 + ((it + 1) & 1) * D::G_STAGE,
                                  &full[(it + 1) & 1]);
        if (next + gridDim.x < tiles) prefetch_codes<N1>(P, next + gridDim.x, codes[(it + 2) % 3]);
      }
      mbar_wait(&empty[it & 1], (it >> 1) & 1);  // tile consumed, its Fv.n assembled in wFv
      const int e0 = P.e_first + tile * EPB;
      bulk_s2g(P.fvn + static_cast<size_t>(e0) * 6 * D::FS, wFv, min(EPB, P.E - e0) * 6u * D::FS * 8u);
      bulk_commit();
      bulk_wait_read0();
      mbar_arrive(fv_free);
    }
    bulk_wait0();
    return;
  }
  // ---------------- consumer warps
  const int le = threadIdx.x / N3, t = threadIdx.x % N3;
  int tile = blockIdx.x;
  for (int it = 0; tile < tiles; ++it, tile += gridDim.x) {
    const int sidx = it & 1;
    double* st = stage0 + sidx * D::G_STAGE;
    const int e0 = P.e_first + tile * EPB;
    const int n_el = min(EPB, P.E - e0);
    const int e = e0 + le;
    const bool active = le < n_el;
    mbar_wait(&full[sidx], (it >> 1) & 1);
    const int* myc = codes[it % 3] + 8 * le;
    double* sU = st + le * D::EL;
    double* sTr = st + EPB * D::EL + le * 6 * D::TS;
    double* sNb = st + EPB * (D::EL + 6 * D::TS) + le * 6 * D::TS;
    double* q = wQ + le * 4 * N3;
    double* gS = wG + le * 12 * N3;
    double* fvo = wFv + le * 6 * D::FS;
    const BandD& B = C.bands[active ? myc[6] : 0];
    // Phase 1: q; lift* in place over the neighbour slot (stride 5), sliding lift* stays at stride 4.
    if (active) {
      double u[5], qq[4];
#pragma unroll
      for (int v = 0; v < 5; ++v) u[v] = sU[t * 5 + v];
      prim4(u, C.gas, qq);
#pragma unroll
      for (int c = 0; c < 4; ++c) q[c * N3 + swz<N1>(t)] = qq[c];
      for (int itm = t; itm < 6 * N2; itm += N3) {
        const int s = itm / N2, f = itm - s * N2;
        const int typ = myc[s] >> kCodeShift;
        double* nb = sNb + s * D::TS;
        if (typ == kSliding) {
          if (f == 0) lstr[le][s] = 4;
          continue;
        }
        double lift[4];
        const double* own = sTr + s * D::TS + f * 5;
        if (typ == kConforming) {
          double ow[5], other[5], qa[4], qb[4];
#pragma unroll
          for (int v = 0; v < 5; ++v) {
            ow[v] = own[v];
            other[v] = nb[f * 5 + v];
          }
          prim4(ow, C.gas, qa);
          prim4(other, C.gas, qb);
#pragma unroll
          for (int c = 0; c < 4; ++c) lift[c] = __dmul_rn(0.5, __dadd_rn(qa[c], qb[c]));
        } else {
          const int a = f / N1, b = f - (f / N1) * N1;
          double x[3], ext[5];
          face_position<N1>(C, P.coords + 4 * e, s, a, b, A.t_stage, x);
          eval_case(C.flow_case, x, A.t_stage, C.gas, ext);
          prim4(ext, C.gas, lift);
        }
        if (f == 0) lstr[le][s] = 5;
#pragma unroll
        for (int c = 0; c < 4; ++c) nb[f * 5 + c] = lift[c];
      }
    }
    consumer_sync(NC);
    if (active) gradient_lines<N1>(C, B, q, sNb, D::TS, lstr[le], 1, gS, t, N3);
    if (it > 0) mbar_wait(fv_free, (it - 1) & 1);  // the previous tile's Fv.n store has read wFv
    consumer_sync(NC);
    if (active && P.grad_out != nullptr) {
      double* go = P.grad_out + (static_cast<size_t>(e) * N3 + t) * 12;
#pragma unroll
      for (int c = 0; c < 12; ++c) go[c] = gS[c * N3 + swz<N1>(t)];
    }
    if (active && P.visc != nullptr) {  // stress and heat flux of the node for k_update_cv (coalesced rows [c][node])
      double g[12], vs[9];
#pragma unroll
      for (int c = 0; c < 12; ++c) g[c] = gS[c * N3 + swz<N1>(t)];
      visc_terms(g, C.gas, vs);
      double* vo = P.visc + static_cast<size_t>(e) * 9 * N3 + t;
#pragma unroll
      for (int c = 0; c < 9; ++c) vo[c * N3] = vs[c];
    }
    // Phase 3: Fv.n on conforming sides; full gradient traces on sliding / Dirichlet sides.
    if (active) {
      for (int itm = t; itm < 6 * N2; itm += N3) {
        const int s = itm / N2, f = itm - s * N2, a = f / N1, b = f - a * N1, dir = s >> 1;
        const double* ell = tab + N1 * N1 + (s & 1) * N1;
        const int code = myc[s];
        const int typ = code >> kCodeShift, idx = code & ((1 << kCodeShift) - 1);
        if (typ == kConforming) {
          double fv[4];
          const double* own = sTr + s * D::TS + f * 5;
          const int rot = (N1 == 4 || N1 == 8) ? 0 : face_rot<N1>(s, a, b);  // swizzled blocks need no rotation
          if (dir == 0) fvn_item<N1, 0>(C, gS, ell, a, b, rot, own, fv);
          else if (dir == 1) fvn_item<N1, 1>(C, gS, ell, a, b, rot, own, fv);
          else fvn_item<N1, 2>(C, gS, ell, a, b, rot, own, fv);
          double2* fq = reinterpret_cast<double2*>(fvo + s * D::FS + f * 4);  // [f][4]: 128-bit stores, no 4-way conflict
          fq[0] = make_double2(fv[0], fv[1]);
          fq[1] = make_double2(fv[2], fv[3]);
        } else {
          double* dst = (typ == kSliding ? P.slide_g : P.dir_g) + (static_cast<size_t>(idx) * N2 + f) * 12;
#pragma unroll
          for (int c = 0; c < 12; ++c) {
            const int base = dir == 0 ? a * N1 + b : (dir == 1 ? a * N2 + b : (a * N1 + b) * N1);
            const int stride = dir == 0 ? N2 : (dir == 1 ? N1 : 1);
            double acc = 0.0;
#pragma unroll
            for (int m = 0; m < N1; ++m) acc = __fma_rn(ell[m], gS[c * N3 + swz<N1>(base + m * stride)], acc);
            dst[c] = acc;
          }
        }
      }
    }
    fence_proxy_async();
    consumer_sync(NC);
    if (threadIdx.x == 0) mbar_arrive(&empty[sidx]);
  }
}

template <int N1>
bool gws_t(const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, int n_sm, cudaStream_t st) {
  if constexpr (N1 % 2 != 0) {
    return false;
  } else {
    using D = T5<N1>;
    const int tiles = (p.E - p.e_first + D::EPB - 1) / D::EPB;
    auto kern = k_gradient_ws<N1>;
    static int occ = -1;
    if (occ < 0) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, D::G_SMEM);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, GWs<N1>::THREADS, D::G_SMEM);
      if (occ < 1) occ = 1;
    }
    kern<<<std::min(tiles, n_sm * occ), GWs<N1>::THREADS, D::G_SMEM, st>>>(c, p, a);
    check_launch("k_gradient_ws");
    return true;
  }
}


template <class K>
void set_smem(K kernel, int bytes) {
  static_assert(sizeof(K) > 0, "");
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

template <int N1>
void prolong_t(const ElemConsts& c, const FieldPtrs& p, cudaStream_t st) {
  const int blocks = (p.E - p.e_first + Dim<N1>::EPB - 1) / Dim<N1>::EPB;
  const int sm = smem_prolong<N1>();
  set_smem(k_prolong<N1>, sm);
  k_prolong<N1><<<blocks, Dim<N1>::THREADS, sm, st>>>(c, p);
  check_launch("k_prolong");
}
template <int N1>
void gradient_t(const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st) {
  const int blocks = (p.E - p.e_first + Dim<N1>::EPB - 1) / Dim<N1>::EPB;
  const int sm = smem_gradient<N1>();
  set_smem(k_gradient<N1>, sm);
  k_gradient<N1><<<blocks, Dim<N1>::THREADS, sm, st>>>(c, p, a);
  check_launch("k_gradient");
}
template <int N1>
void update_t(const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st) {
  const int blocks = (p.E - p.e_first + Dim<N1>::EPB - 1) / Dim<N1>::EPB;
  const int sm = smem_update<N1>();
  if (c.gas.viscous) {
    set_smem(k_update<N1, true>, sm);
    k_update<N1, true><<<blocks, Dim<N1>::THREADS, sm, st>>>(c, p, a);
  } else {
    set_smem(k_update<N1, false>, sm);
    k_update<N1, false><<<blocks, Dim<N1>::THREADS, sm, st>>>(c, p, a);
  }
  check_launch("k_update");
}

template <int N1>
void mortar_fill_t(int nc, const double* src, double* const dst[2], const MortarOps& ops, const MortarPtrs& p,
                   cudaStream_t st) {
  const int items = p.S * 2 * N1 * N1;
  if (items == 0) return;
  const int bs = 128, blocks = (items + bs - 1) / bs;
  int n_ctx = kMaxCtx;
  if (nc == 5) k_mortar_fill<N1, 5><<<blocks, bs, 0, st>>>(ops, n_ctx, p, src, dst[0], dst[1]);
  else k_mortar_fill<N1, 12><<<blocks, bs, 0, st>>>(ops, n_ctx, p, src, dst[0], dst[1]);
  check_launch("k_mortar_fill");
}
template <int N1>
void mortar_back_t(int nc, const double* const src[2], double* dst, const MortarOps& ops, const MortarPtrs& p,
                   cudaStream_t st) {
  const int items = p.S * N1 * N1;
  if (items == 0) return;
  const int bs = 128, blocks = (items + bs - 1) / bs;
  if (nc == 4) k_mortar_backproject<N1, 4><<<blocks, bs, 0, st>>>(ops, kMaxCtx, p, src[0], src[1], dst);
  else k_mortar_backproject<N1, 5><<<blocks, bs, 0, st>>>(ops, kMaxCtx, p, src[0], src[1], dst);
  check_launch("k_mortar_backproject");
}

#include "curved.cuh"

#define SDG_DISPATCH(n1, CALL)                          \
  switch (n1) {                                         \
    case 2: { constexpr int NN = 2; CALL; break; }      \
    case 3: { constexpr int NN = 3; CALL; break; }      \
    case 4: { constexpr int NN = 4; CALL; break; }      \
    case 5: { constexpr int NN = 5; CALL; break; }      \
    case 6: { constexpr int NN = 6; CALL; break; }      \
    case 7: { constexpr int NN = 7; CALL; break; }      \
    case 8: { constexpr int NN = 8; CALL; break; }      \
    default: throw ConfigError("unsupported N+1");      \
  }

}  // namespace

void launch_prolong(int n1, const ElemConsts& c, const FieldPtrs& p, cudaStream_t st) {
  if (p.E <= p.e_first) return;
  SDG_DISPATCH(n1, (prolong_t<NN>(c, p, st)));
}
void launch_gradient(int n1, const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st) {
  if (p.E <= p.e_first) return;
  SDG_DISPATCH(n1, (gradient_t<NN>(c, p, a, st)));
}
void launch_update(int n1, const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st) {
  if (p.E <= p.e_first) return;
  SDG_DISPATCH(n1, (update_t<NN>(c, p, a, st)));
}
bool launch_gradient_tma(int n1, const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, int n_sm,
                         cudaStream_t st) {
  if (p.E <= p.e_first) return true;
  bool ok = false;
  SDG_DISPATCH(n1, (ok = gws_t<NN>(c, p, a, n_sm, st)));
  return ok;
}
// Curved elements: the bulk-loaded kernels for even N+1 (every block a multiple of
// 16 bytes, as cp.async.bulk needs), the plain-load ones otherwise.
void launch_gradient_curved(int n1, const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st) {
  if (p.E <= p.e_first) return;
  bool done = false;
  SDG_DISPATCH(n1, (done = gradient_curved_b_t<NN>(c, p, a, st)));
  if (!done) SDG_DISPATCH(n1, (gradient_curved_t<NN>(c, p, a, st)));
}
void launch_update_curved(int n1, const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st) {
  if (p.E <= p.e_first) return;
  bool done = false;
  SDG_DISPATCH(n1, (done = update_curved_b_t<NN>(c, p, a, st)));
  if (!done) SDG_DISPATCH(n1, (update_curved_t<NN>(c, p, a, st)));
}
bool launch_update_affine_b(int n1, const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st) {
  if (p.E <= p.e_first) return true;
  bool done = false;
  SDG_DISPATCH(n1, (done = update_affine_b_t<NN>(c, p, a, st)));
  return done;
}
// ---------------------------------------------------------------------------
// Non-matching face rows (BASELINE configs[1]): the mortars of one periodic row,
// side A n_a faces of length l_a, side B n_b faces, B displaced by delta; the
// device form of merge_intervals (csrc/host.cpp), bit for bit.  One block: pass 1
// counts each B face's pieces (1 + A edges strictly inside), pass 2 writes them
// at the block-scanned offsets, rotated so the list is ordered by A face (the B
// order runs along the row from B's edge 0, so sorting by A face is the rotation
// that starts at the first piece past A's period).  Explicit _rn arithmetic keeps
// the displacement split and the local coordinates free of contraction.
// ---------------------------------------------------------------------------
constexpr int kIvThreads = 512;

struct IvEdge {
  long long I;
  double F;
};

__device__ __forceinline__ IvEdge iv_edge(long long j, long long n_a, long long n_b, long long nd, double sd) {
  const long long jj = j % n_b, wraps = j / n_b, num = jj * n_a;
  IvEdge e;
  e.I = nd + num / n_b + wraps * n_a;
  e.F = __dadd_rn(sd, __ddiv_rn(static_cast<double>(num % n_b), static_cast<double>(n_b)));
  if (e.F >= 1.0) {
    e.F = __dsub_rn(e.F, 1.0);
    e.I += 1;
  }
  return e;
}

__device__ __forceinline__ long long iv_block_scan(long long v, long long* sh, long long& total) {
  const int tid = threadIdx.x;
  sh[tid] = v;
  __syncthreads();
  for (int off = 1; off < kIvThreads; off <<= 1) {
    const long long add = tid >= off ? sh[tid - off] : 0;
    __syncthreads();
    sh[tid] += add;
    __syncthreads();
  }
  const long long incl = sh[tid];
  total = sh[kIvThreads - 1];
  __syncthreads();
  return incl - v;
}

__device__ __forceinline__ void mortar_intervals_row(long long n_a, long long n_b, double l_a, double delta,
                                                     long long* faces, double* ranges, long long* n_out,
                                                     long long* sh) {
  const double period = __dmul_rn(l_a, static_cast<double>(n_a));
  double d = fmod(delta, period);
  if (d < 0.0) d = __dadd_rn(d, period);
  const double ratio = __ddiv_rn(d, l_a);
  long long nd = static_cast<long long>(floor(ratio));
  double sd = __dsub_rn(ratio, static_cast<double>(nd));
  if (nd >= n_a) {
    nd = 0;
    sd = 0.0;
  }
  const double q = __ddiv_rn(static_cast<double>(n_a), static_cast<double>(n_b));
  // pass 1: total pieces M and r = pieces starting before A's period end
  long long M = 0, R = 0;
  for (long long base = 0; base < n_b; base += kIvThreads) {
    const long long j = base + threadIdx.x;
    long long cnt = 0, before = 0;
    if (j < n_b) {
      const IvEdge e0 = iv_edge(j, n_a, n_b, nd, sd), e1 = iv_edge(j + 1, n_a, n_b, nd, sd);
      const long long m_first = e0.I + 1, m_last = e1.F == 0.0 ? e1.I - 1 : e1.I;
      cnt = m_last - m_first + 2;
      // piece starts: e0.I, then m_first..m_last; count those < n_a
      before = (e0.I < n_a ? 1 : 0) + max(0LL, min(m_last, n_a - 1) - m_first + 1);
    }
    long long tc, tb;
    iv_block_scan(cnt, sh, tc);
    iv_block_scan(before, sh, tb);
    M += tc;
    R += tb;
  }
  if (threadIdx.x == 0) *n_out = M;
  if (faces == nullptr) return;
  long long run = 0;
  for (long long base = 0; base < n_b; base += kIvThreads) {
    const long long j = base + threadIdx.x;
    long long cnt = 0;
    IvEdge e0{0, 0.0}, e1{0, 0.0};
    long long m_first = 0, m_last = -1;
    if (j < n_b) {
      e0 = iv_edge(j, n_a, n_b, nd, sd);
      e1 = iv_edge(j + 1, n_a, n_b, nd, sd);
      m_first = e0.I + 1;
      m_last = e1.F == 0.0 ? e1.I - 1 : e1.I;
      cnt = m_last - m_first + 2;
    }
    long long tc;
    const long long off = run + iv_block_scan(cnt, sh, tc);
    run += tc;
    if (j >= n_b) continue;
    long long p_int = e0.I;
    double a_lo = e0.F == 0.0 ? -1.0 : __dsub_rn(__dmul_rn(2.0, e0.F), 1.0), b_lo = -1.0;
    for (long long m = m_first, k = off; m <= m_last + 1; ++m, ++k) {
      double a_hi, b_hi;
      if (m <= m_last) {
        a_hi = 1.0;
        const double dr = __dadd_rn(static_cast<double>(e1.I - m), e1.F);
        b_hi = __dsub_rn(1.0, __dmul_rn(2.0, __ddiv_rn(dr, q)));
      } else {
        a_hi = e1.F == 0.0 ? 1.0 : __dsub_rn(__dmul_rn(2.0, e1.F), 1.0);
        b_hi = 1.0;
      }
      const long long o = ((k - R) % M + M) % M;
      faces[2 * o] = ((p_int % n_a) + n_a) % n_a;
      faces[2 * o + 1] = j;
      ranges[4 * o] = a_lo;
      ranges[4 * o + 1] = a_hi;
      ranges[4 * o + 2] = b_lo;
      ranges[4 * o + 3] = b_hi;
      a_lo = -1.0;
      b_lo = b_hi;
      p_int = m;
    }
  }
}

__global__ void __launch_bounds__(kIvThreads) k_mortar_intervals(long long n_a, long long n_b, double l_a, double delta,
                                                                 long long* faces, double* ranges, long long* n_out) {
  __shared__ long long sh[kIvThreads];
  mortar_intervals_row(n_a, n_b, l_a, delta, faces, ranges, n_out, sh);
}

// Both rows (y and z) of a non-matching interface in one launch, one block per row.
__global__ void __launch_bounds__(kIvThreads) k_mortar_intervals2(const __grid_constant__ IvRows rows) {
  __shared__ long long sh[kIvThreads];
  const IvRow& r = rows.row[blockIdx.x];
  mortar_intervals_row(r.n_a, r.n_b, r.l_a, r.delta, r.faces, r.ranges, r.n_out, sh);
}

void launch_mortar_intervals2(const IvRows& rows, cudaStream_t st) {
  k_mortar_intervals2<<<2, kIvThreads, 0, st>>>(rows);
  check_launch("k_mortar_intervals2");
}

void launch_mortar_intervals(long long n_a, long long n_b, double l_a, double delta, long long* faces,
                             double* ranges, long long* n_out, cudaStream_t st) {
  k_mortar_intervals<<<1, kIvThreads, 0, st>>>(n_a, n_b, l_a, delta, faces, ranges, n_out);
  check_launch("k_mortar_intervals");
}

// ---------------------------------------------------------------------------
// Non-matching planar interface transfer: mortars are tensor products of a y row
// and a z row of intervals.  Face data layout [fy][fz][i][j][nc] (i along y).
// k_nc_to_mortar: mortar (ky, kz) = (Fy[ky] x Fz[kz]) applied to its source face.
// k_nc_to_face: target face (fy, fz) = sum over its mortars (rows in CSR, fixed
// order) of (By[ky] x Bz[kz]) applied to the mortar data.  One block per item.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void nc_to_mortar_body(long long blk, int n, int nc, const double* __restrict__ src,
                                                  long long nfz, const long long* __restrict__ iv_y,
                                                  const long long* __restrict__ iv_z, int col, long long mz,
                                                  const double* __restrict__ Fy, const double* __restrict__ Fz,
                                                  double* __restrict__ mortar) {
  extern __shared__ double sm[];
  const long long ky = blk / mz, kz = blk % mz;
  const long long fy = iv_y[2 * ky + col], fz = iv_z[2 * kz + col];
  const int per = n * n * nc;
  double* u = sm;
  double* t = sm + per;
  const double* face = src + (fy * nfz + fz) * per;
  for (int x = threadIdx.x; x < per; x += blockDim.x) u[x] = face[x];
  __syncthreads();
  const double* fy_op = Fy + ky * n * n;
  const double* fz_op = Fz + kz * n * n;
  for (int x = threadIdx.x; x < per; x += blockDim.x) {  // t[k][j][c] = sum_i Fy[k][i] u[i][j][c]
    const int c = x % nc, j = (x / nc) % n, k = x / (nc * n);
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc = fma(fy_op[k * n + i], u[(i * n + j) * nc + c], acc);
    t[x] = acc;
  }
  __syncthreads();
  double* out = mortar + blk * static_cast<long long>(per);
  for (int x = threadIdx.x; x < per; x += blockDim.x) {  // out[k][l][c] = sum_j Fz[l][j] t[k][j][c]
    const int c = x % nc, l = (x / nc) % n, k = x / (nc * n);
    double acc = 0.0;
    for (int j = 0; j < n; ++j) acc = fma(fz_op[l * n + j], t[(k * n + j) * nc + c], acc);
    out[x] = acc;
  }
}

__global__ void k_nc_to_mortar(int n, int nc, const double* __restrict__ src, long long nfz,
                               const long long* __restrict__ iv_y, const long long* __restrict__ iv_z, int col,
                               long long mz, const double* __restrict__ Fy, const double* __restrict__ Fz,
                               double* __restrict__ mortar) {
  nc_to_mortar_body(blockIdx.x, n, nc, src, nfz, iv_y, iv_z, col, mz, Fy, Fz, mortar);
}

// Several face -> mortar transfers of one interface in one launch (blockIdx.y = job).
__global__ void k_nc_to_mortar_batch(int n, const long long* __restrict__ iv_y, const long long* __restrict__ iv_z,
                                     long long mz, const __grid_constant__ NcMortarJobs jobs) {
  const NcMortarJob& j = jobs.job[blockIdx.y];
  nc_to_mortar_body(blockIdx.x, n, j.nc, j.src, j.src_nfz, iv_y, iv_z, j.col, mz, j.Fy, j.Fz, j.out);
}

__device__ __forceinline__ void nc_to_face_body(long long blk, int n, int nc, const double* __restrict__ mortar,
                                                long long mz, long long nfz, const int* __restrict__ off_y,
                                                const int* __restrict__ idx_y, const int* __restrict__ off_z,
                                                const int* __restrict__ idx_z, const double* __restrict__ By,
                                                const double* __restrict__ Bz, double* __restrict__ dst) {
  extern __shared__ double sm[];
  const long long fy = blk / nfz, fz = blk % nfz;
  const int per = n * n * nc;
  double* m = sm;
  double* t = sm + per;
  double acc_local[8];  // up to 8 outputs per thread (per <= 8 * blockDim)
  const int reps = (per + blockDim.x - 1) / blockDim.x;
  for (int r = 0; r < reps; ++r) acc_local[r] = 0.0;
  for (int a = off_y[fy]; a < off_y[fy + 1]; ++a)
    for (int b = off_z[fz]; b < off_z[fz + 1]; ++b) {
      const long long ky = idx_y[a], kz = idx_z[b];
      const double* src = mortar + (ky * mz + kz) * static_cast<long long>(per);
      __syncthreads();
      for (int x = threadIdx.x; x < per; x += blockDim.x) m[x] = src[x];
      __syncthreads();
      const double* by = By + ky * n * n;
      const double* bz = Bz + kz * n * n;
      for (int x = threadIdx.x; x < per; x += blockDim.x) {  // t[i][l][c] = sum_k By[i][k] m[k][l][c]
        const int c = x % nc, l = (x / nc) % n, i = x / (nc * n);
        double acc = 0.0;
        for (int k = 0; k < n; ++k) acc = fma(by[i * n + k], m[(k * n + l) * nc + c], acc);
        t[x] = acc;
      }
      __syncthreads();
      for (int r = 0, x = threadIdx.x; x < per; ++r, x += blockDim.x) {  // += sum_l Bz[j][l] t[i][l][c]
        const int c = x % nc, j = (x / nc) % n, i = x / (nc * n);
        double acc = 0.0;
        for (int l = 0; l < n; ++l) acc = fma(bz[j * n + l], t[(i * n + l) * nc + c], acc);
        acc_local[r] += acc;
      }
    }
  double* out = dst + blk * static_cast<long long>(per);
  for (int r = 0, x = threadIdx.x; x < per; ++r, x += blockDim.x) out[x] = acc_local[r];
}

__global__ void k_nc_to_face(int n, int nc, const double* __restrict__ mortar, long long mz, long long nfz,
                             const int* __restrict__ off_y, const int* __restrict__ idx_y,
                             const int* __restrict__ off_z, const int* __restrict__ idx_z,
                             const double* __restrict__ By, const double* __restrict__ Bz, double* __restrict__ dst) {
  nc_to_face_body(blockIdx.x, n, nc, mortar, mz, nfz, off_y, idx_y, off_z, idx_z, By, Bz, dst);
}

// Mortar -> face projections onto several face sets in one launch (blockIdx.y = job;
// blocks past a job's face count exit before any barrier).
__global__ void k_nc_to_face_batch(int n, int nc, const double* __restrict__ mortar, long long mz,
                                   const __grid_constant__ NcFaceJobs jobs) {
  const NcFaceJob& j = jobs.job[blockIdx.y];
  if (blockIdx.x >= j.nfy * j.nfz) return;
  nc_to_face_body(blockIdx.x, n, nc, mortar, mz, j.nfz, j.off_y, j.idx_y, j.off_z, j.idx_z, j.By, j.Bz, j.dst);
}

static int nc_threads(int per) { return std::min(1024, (per + 31) / 32 * 32); }

void launch_nc_to_mortar_batch(int n, const long long* iv_y, const long long* iv_z, long long my, long long mz,
                               const NcMortarJobs& jobs, cudaStream_t st) {
  int per = 0;
  for (int k = 0; k < jobs.n; ++k) per = std::max(per, n * n * jobs.job[k].nc);
  if (per > 1024) throw DeviceError(SDG_ERR_CONFIG, "nc transfer: n*n*nc exceeds 1024");
  if (my * mz == 0 || jobs.n == 0) return;
  // No serial loop here (one mortar per block): narrow blocks keep more mortars resident per SM.
  k_nc_to_mortar_batch<<<dim3(static_cast<unsigned>(my * mz), jobs.n), 128, 2 * per * sizeof(double),
                         st>>>(n, iv_y, iv_z, mz, jobs);
  check_launch("k_nc_to_mortar_batch");
}

void launch_nc_to_face_batch(int n, int nc, const double* mortar, long long mz, const NcFaceJobs& jobs,
                             cudaStream_t st) {
  const int per = n * n * nc;
  if (per > 1024) throw DeviceError(SDG_ERR_CONFIG, "nc transfer: n*n*nc exceeds 1024");
  long long faces = 0;
  for (int k = 0; k < jobs.n; ++k) faces = std::max(faces, jobs.job[k].nfy * jobs.job[k].nfz);
  if (faces == 0) return;
  k_nc_to_face_batch<<<dim3(static_cast<unsigned>(faces), jobs.n), nc_threads(per), 2 * per * sizeof(double), st>>>(
      n, nc, mortar, mz, jobs);
  check_launch("k_nc_to_face_batch");
}

void launch_nc_transfer(int n, int nc, const double* src, long long src_nfz, const long long* iv_y,
                        const long long* iv_z, int src_col, long long my, long long mz, const double* Fy,
                        const double* Fz, double* mortar, long long dst_nfy, long long dst_nfz, const int* off_y,
                        const int* idx_y, const int* off_z, const int* idx_z, const double* By, const double* Bz,
                        double* dst, cudaStream_t st) {
  // One thread per output value of a face / mortar (up to 1024): the CSR gather of
  // k_nc_to_face is a serial loop over a face's mortars, so the per-mortar
  // contraction must be as wide as the face.
  const int per = n * n * nc, threads = std::min(1024, (per + 31) / 32 * 32);
  if (per > 1024) throw DeviceError(SDG_ERR_CONFIG, "nc transfer: n*n*nc exceeds 1024");
  const size_t shm = 2 * per * sizeof(double);
  if (my * mz > 0) {
    k_nc_to_mortar<<<static_cast<unsigned>(my * mz), threads, shm, st>>>(n, nc, src, src_nfz, iv_y, iv_z, src_col, mz,
                                                                        Fy, Fz, mortar);
    check_launch("k_nc_to_mortar");
  }
  if (dst_nfy * dst_nfz > 0) {
    k_nc_to_face<<<static_cast<unsigned>(dst_nfy * dst_nfz), threads, shm, st>>>(n, nc, mortar, mz, dst_nfz, off_y,
                                                                                idx_y, off_z, idx_z, By, Bz, dst);
    check_launch("k_nc_to_face");
  }
}

// Two-sided numerical flux at the nodes of the tensor-product mortars of a
// non-matching planar interface with normal e_dir, side A on the minus side:
// face_numerical_flux (solver.cpp:308-321) on both sides' mortar traces, the
// viscous normal fluxes from the mortar gradients when given (ga/gb non-null).
// One thread per mortar node; *bad counts nodes with a non-positive Roe c^2.
__global__ void k_nc_mortar_flux(long long nodes, GasD g, int dir, double vg, const double* __restrict__ ua,
                                 const double* __restrict__ ub, const double* __restrict__ ga,
                                 const double* __restrict__ gb, double* __restrict__ flux, int* bad) {
  const long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (q >= nodes) return;
  double um[5], up[5], f[5];
#pragma unroll
  for (int v = 0; v < 5; ++v) {
    um[v] = ua[q * 5 + v];
    up[v] = ub[q * 5 + v];
  }
  double fvm[4], fvp[4];
  const bool vis = ga != nullptr && g.viscous;
  if (vis) {
    fv_dir(um, ga + q * 12, dir, g, fvm);
    fv_dir(up, gb + q * 12, dir, g, fvp);
  }
  if (!face_flux_fv(um, up, dir, vg, vis ? fvm : nullptr, fvp, g, f)) atomicAdd(bad, 1);
#pragma unroll
  for (int v = 0; v < 5; ++v) flux[q * 5 + v] = f[v];
}

// The lifting mean at the mortar nodes of a non-matching interface: the mean of
// both sides' primitive (u, v, w, T) (run_lifting, solver.cpp:597-727).
__global__ void k_nc_mortar_lift(long long nodes, GasD g, const double* __restrict__ ua, const double* __restrict__ ub,
                                 double* __restrict__ lift) {
  const long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (q >= nodes) return;
  double a[4], b[4];
  prim4(ua + q * 5, g, a);
  prim4(ub + q * 5, g, b);
#pragma unroll
  for (int c = 0; c < 4; ++c) lift[q * 4 + c] = __dmul_rn(0.5, __dadd_rn(a[c], b[c]));
}

void launch_nc_mortar_lift(long long nodes, const GasD& g, const double* ua, const double* ub, double* lift,
                           cudaStream_t st) {
  if (nodes <= 0) return;
  const int threads = 128;
  k_nc_mortar_lift<<<static_cast<unsigned>((nodes + threads - 1) / threads), threads, 0, st>>>(nodes, g, ua, ub, lift);
  check_launch("k_nc_mortar_lift");
}

void launch_nc_mortar_flux(long long nodes, const GasD& g, int dir, double vg, const double* ua, const double* ub,
                           const double* ga, const double* gb, double* flux, int* bad, cudaStream_t st) {
  if (nodes <= 0) return;
  const int threads = 128;
  k_nc_mortar_flux<<<static_cast<unsigned>((nodes + threads - 1) / threads), threads, 0, st>>>(nodes, g, dir, vg, ua,
                                                                                              ub, ga, gb, flux, bad);
  check_launch("k_nc_mortar_flux");
}

// ---------------------------------------------------------------------------
// Non-matching / oblique interfaces inside the stage (BASELINE configs[1]).
// Face data are read from / written to the resident arrays through per-face
// slot tables (trace slots 6e + side, or compact sliding indices), so no
// gather copies are needed; the tensor-product contractions are those of
// nc_to_mortar_body / nc_to_face_body above.
// ---------------------------------------------------------------------------
// Both rows of one interface recomputed on the device every stage and compared
// with the rows the host built its operators from: a mismatch is a protocol error.
__global__ void __launch_bounds__(kIvThreads) k_nc_rows(const __grid_constant__ NcStage S, int iface, ErrRec* err) {
  __shared__ long long sh[kIvThreads];
  __shared__ int bad;
  const int d = blockIdx.x;
  if (threadIdx.x == 0) bad = 0;
  mortar_intervals_row(S.n_a[d], S.n_b[d], S.l_a[d], S.delta[d], S.d_faces[d], S.d_ranges[d], S.d_n + d, sh);
  __syncthreads();
  const long long m = d == 0 ? S.my : S.mz;
  if (S.d_n[d] != m) bad = 1;
  for (long long k = threadIdx.x; k < m; k += blockDim.x) {
    if (S.d_faces[d][2 * k] != S.h_faces[d][2 * k] || S.d_faces[d][2 * k + 1] != S.h_faces[d][2 * k + 1]) bad = 1;
    for (int q = 0; q < 4; ++q)
      if (S.d_ranges[d][4 * k + q] != S.h_ranges[d][4 * k + q]) bad = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0 && bad && atomicCAS(&err->flag, 0, 4) == 0) {
    err->elem = iface;
    err->node = d;
  }
}

// Face -> mortar for both sides (blockIdx.y = side): mortar (ky, kz) of side s is
// (F_y[s][ky] x F_z[s][kz]) applied to its face, located by the DEVICE rows.
__global__ void k_nc_fill(int n, int nc, const double* __restrict__ src, const __grid_constant__ NcStage S,
                          const int* __restrict__ tab0, const int* __restrict__ tab1, double* __restrict__ out0,
                          double* __restrict__ out1) {
  extern __shared__ double sm[];
  const int s = blockIdx.y;
  const long long blk = blockIdx.x, ky = blk / S.mz, kz = blk % S.mz;
  const long long fy = S.d_faces[0][2 * ky + s], fz = S.d_faces[1][2 * kz + s];
  const int* tab = s ? tab1 : tab0;
  const int per = n * n * nc;
  double* u = sm;
  double* t = sm + per;
  const double* face = src + static_cast<long long>(tab[fy * S.nfz[s] + fz]) * per;
  for (int x = threadIdx.x; x < per; x += blockDim.x) u[x] = face[x];
  __syncthreads();
  const double* fy_op = S.F[s][0] + ky * n * n;
  const double* fz_op = S.F[s][1] + kz * n * n;
  for (int x = threadIdx.x; x < per; x += blockDim.x) {  // t[k][j][c] = sum_i Fy[k][i] u[i][j][c]
    const int c = x % nc, j = (x / nc) % n, k = x / (nc * n);
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc = fma(fy_op[k * n + i], u[(i * n + j) * nc + c], acc);
    t[x] = acc;
  }
  __syncthreads();
  double* o = (s ? out1 : out0) + blk * static_cast<long long>(per);
  for (int x = threadIdx.x; x < per; x += blockDim.x) {  // o[k][l][c] = sum_j Fz[l][j] t[k][j][c]
    const int c = x % nc, l = (x / nc) % n, k = x / (nc * n);
    double acc = 0.0;
    for (int j = 0; j < n; ++j) acc = fma(fz_op[l * n + j], t[(k * n + j) * nc + c], acc);
    o[x] = acc;
  }
}

// Mortar -> face for both sides (blocks over the faces of A, then of B): each face
// sums (B_y[s][ky] x B_z[s][kz]) applied to its mortars in the fixed CSR order.
__global__ void k_nc_project(int n, int nc, const double* __restrict__ mortar, const __grid_constant__ NcStage S,
                             const int* __restrict__ tab0, const int* __restrict__ tab1, double* __restrict__ dst) {
  extern __shared__ double sm[];
  const long long nf0 = S.nfy[0] * S.nfz[0];
  const int s = blockIdx.x < nf0 ? 0 : 1;
  const long long f = s ? blockIdx.x - nf0 : blockIdx.x;
  const long long fy = f / S.nfz[s], fz = f % S.nfz[s];
  const int per = n * n * nc;
  double* m = sm;
  double* t = sm + per;
  double acc_local[8];
  const int reps = (per + blockDim.x - 1) / blockDim.x;
  for (int r = 0; r < reps; ++r) acc_local[r] = 0.0;
  const int *offy = S.off[s][0], *offz = S.off[s][1], *idy = S.idx[s][0], *idz = S.idx[s][1];
  for (int a = offy[fy]; a < offy[fy + 1]; ++a)
    for (int b = offz[fz]; b < offz[fz + 1]; ++b) {
      const long long ky = idy[a], kz = idz[b];
      const double* src = mortar + (ky * S.mz + kz) * static_cast<long long>(per);
      __syncthreads();
      for (int x = threadIdx.x; x < per; x += blockDim.x) m[x] = src[x];
      __syncthreads();
      const double* by = S.B[s][0] + ky * n * n;
      const double* bz = S.B[s][1] + kz * n * n;
      for (int x = threadIdx.x; x < per; x += blockDim.x) {  // t[i][l][c] = sum_k By[i][k] m[k][l][c]
        const int c = x % nc, l = (x / nc) % n, i = x / (nc * n);
        double acc = 0.0;
        for (int k = 0; k < n; ++k) acc = fma(by[i * n + k], m[(k * n + l) * nc + c], acc);
        t[x] = acc;
      }
      __syncthreads();
      for (int r = 0, x = threadIdx.x; x < per; ++r, x += blockDim.x) {  // += sum_l Bz[j][l] t[i][l][c]
        const int c = x % nc, j = (x / nc) % n, i = x / (nc * n);
        double acc = 0.0;
        for (int l = 0; l < n; ++l) acc = fma(bz[j * n + l], t[(i * n + l) * nc + c], acc);
        acc_local[r] += acc;
      }
    }
  double* out = dst + static_cast<long long>((s ? tab1 : tab0)[f]) * per;
  for (int r = 0, x = threadIdx.x; x < per; ++r, x += blockDim.x) out[x] = acc_local[r];
}

// Two-sided Roe (+ central viscous) flux at the mortar nodes, A on the minus side,
// normal +x, vg_n = 0 (tangential sliding); failures go to the stage's error record.
__global__ void k_nc_flux(long long nodes, GasD g, const double* __restrict__ ua, const double* __restrict__ ub,
                          const double* __restrict__ ga, const double* __restrict__ gb, double* __restrict__ flux,
                          ErrRec* err) {
  const long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (q >= nodes) return;
  double um[5], up[5], f[5];
#pragma unroll
  for (int v = 0; v < 5; ++v) {
    um[v] = ua[q * 5 + v];
    up[v] = ub[q * 5 + v];
  }
  double fvm[4], fvp[4];
  const bool vis = ga != nullptr && g.viscous;
  if (vis) {
    fv_dir(um, ga + q * 12, 0, g, fvm);
    fv_dir(up, gb + q * 12, 0, g, fvp);
  }
  if (!face_flux_fv(um, up, 0, 0.0, vis ? fvm : nullptr, fvp, g, f)) record_error(err, 2, -1, -1, -1, -1, um);
#pragma unroll
  for (int v = 0; v < 5; ++v) flux[q * 5 + v] = f[v];
}

void launch_nc_rows(const NcStage& S, int iface, ErrRec* err, cudaStream_t st) {
  k_nc_rows<<<2, kIvThreads, 0, st>>>(S, iface, err);
  check_launch("k_nc_rows");
}
void launch_nc_fill(int n, int nc, const double* src, const NcStage& S, const int* const tab[2], double* const out[2],
                    cudaStream_t st) {
  const int per = n * n * nc;
  if (per > 1024) throw DeviceError(SDG_ERR_CONFIG, "nc fill: n*n*nc exceeds 1024");
  if (S.my * S.mz == 0) return;
  k_nc_fill<<<dim3(static_cast<unsigned>(S.my * S.mz), 2), 128, 2 * per * sizeof(double), st>>>(
      n, nc, src, S, tab[0], tab[1], out[0], out[1]);
  check_launch("k_nc_fill");
}
void launch_nc_project(int n, int nc, const double* mortar, const NcStage& S, const int* const tab[2], double* dst,
                       cudaStream_t st) {
  const int per = n * n * nc;
  if (per > 1024) throw DeviceError(SDG_ERR_CONFIG, "nc projection: n*n*nc exceeds 1024");
  const long long faces = S.nfy[0] * S.nfz[0] + S.nfy[1] * S.nfz[1];
  k_nc_project<<<static_cast<unsigned>(faces), nc_threads(per), 2 * per * sizeof(double), st>>>(n, nc, mortar, S,
                                                                                              tab[0], tab[1], dst);
  check_launch("k_nc_project");
}
void launch_nc_flux(long long nodes, const GasD& g, const double* ua, const double* ub, const double* ga,
                    const double* gb, double* flux, ErrRec* err, cudaStream_t st) {
  if (nodes <= 0) return;
  k_nc_flux<<<static_cast<unsigned>((nodes + 127) / 128), 128, 0, st>>>(nodes, g, ua, ub, ga, gb, flux, err);
  check_launch("k_nc_flux");
}

void launch_pairing(const PairingArgs& a, const PairingPtrs& p, cudaStream_t st) {
  k_pairing<<<2, kPairThreads, 0, st>>>(a, p);
  check_launch("k_pairing");
}
void launch_mortar_fill(int n1, int nc, const double* src, double* const dst[2], const MortarOps& ops,
                        const MortarPtrs& p, cudaStream_t st) {
  SDG_DISPATCH(n1, (mortar_fill_t<NN>(nc, src, dst, ops, p, st)));
}
void launch_mortar_lift(int n1, const GasD& g, const MortarPtrs& p, int max_mortars, cudaStream_t st) {
  const int items = max_mortars * n1 * n1;
  if (items == 0) return;
  const int bs = 128, blocks = (items + bs - 1) / bs;
  SDG_DISPATCH(n1, (k_mortar_lift<NN><<<blocks, bs, 0, st>>>(g, p, max_mortars)));
  check_launch("k_mortar_lift");
}
void launch_mortar_backproject(int n1, int nc, const double* const src[2], double* dst, const MortarOps& ops,
                               const MortarPtrs& p, cudaStream_t st) {
  SDG_DISPATCH(n1, (mortar_back_t<NN>(nc, src, dst, ops, p, st)));
}
void launch_mortar_flux(int n1, const GasD& g, int viscous, const MortarPtrs& p, int max_mortars, ErrRec* err,
                        cudaStream_t st) {
  const int items = max_mortars * n1 * n1;
  if (items == 0) return;
  const int bs = 128, blocks = (items + bs - 1) / bs;
  if (viscous) {
    SDG_DISPATCH(n1, (k_mortar_flux<NN, true><<<blocks, bs, 0, st>>>(g, p, max_mortars, err)));
  } else {
    SDG_DISPATCH(n1, (k_mortar_flux<NN, false><<<blocks, bs, 0, st>>>(g, p, max_mortars, err)));
  }
  check_launch("k_mortar_flux");
}
int launch_diagnostics(int n1, const ElemConsts& c, const FieldPtrs& p, double t, int with_exact, double* partial,
                       int max_blocks, cudaStream_t st) {
  const long long nodes = static_cast<long long>(p.E) * n1 * n1 * n1;
  const int blocks = static_cast<int>(std::max(1LL, std::min<long long>(max_blocks, (nodes + 255) / 256)));
  SDG_DISPATCH(n1, (k_diag<NN><<<blocks, 256, 0, st>>>(c, p, t, with_exact, partial)));
  check_launch("k_diag");
  return blocks;
}
void launch_suggest_dt(int n1, const ElemConsts& c, const FieldPtrs& p, double cfl, int degree,
                       unsigned long long* out, cudaStream_t st) {
  if (p.E == 0) return;
  SDG_DISPATCH(n1, (k_suggest_dt<NN><<<(p.E + Dim<NN>::EPB - 1) / Dim<NN>::EPB, Dim<NN>::THREADS, 0, st>>>(
                        c, p, cfl, degree, out)));
  check_launch("k_suggest_dt");
}

}  // namespace sdg
