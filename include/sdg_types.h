/*
 * sdg_types.h — plain-C problem description shared by the B200 C-ABI
 * (include/sdg_gpu.h) and the CPU oracle (oracle/sdg3d.h).
 *
 * This is the 3D generalisation of the reference's setup types:
 *   - BandSpec / MeshSpec           /root/reference/proj/src/mesh.hpp:12-26
 *   - GasModel                      /root/reference/proj/src/state.hpp:29-44
 *   - CaseDef (+ exact solutions)   /root/reference/proj/src/cases.hpp:11-28,
 *                                   /root/reference/proj/src/exact_solutions.hpp:9-42
 *   - NodeKind                      /root/reference/proj/src/nodal_basis.hpp:11
 *   - error classes                 /root/reference/proj/src/errors.hpp:9-21
 *
 * Geometry convention (the reference's 2D axes, extended by z):
 *   bands (sliding blocks) are stacked along x, the sliding interfaces are
 *   x-normal planes, a moving band translates rigidly along +y (the
 *   interface-parallel index i_par = iy), z is the second tangential axis
 *   (i_perp = iz).  BASELINE.json's configs are mapped by relabelling:
 *   BASELINE z (split axis) -> x, BASELINE x (slide axis) -> y,
 *   BASELINE y -> z.
 *
 * State layout (host and device, fp64):
 *   U[e][i][j][k][v], i along x, j along y, k along z (k fastest),
 *   v in {rho, rho*v1, rho*v2, rho*v3, rho*E}.
 */
#ifndef SDG_TYPES_H
#define SDG_TYPES_H

#ifdef __cplusplus
extern "C" {
#endif

#define SDG_MAX_BANDS 16
#define SDG_NVARS 5
#define SDG_PT_MAX_MODES 8
#define SDG_NGRAD 12 /* (v1, v2, v3, T) x (d/dx, d/dy, d/dz): g[3*q + dir] */

/* Status codes of every C entry point (0 = success). The C++ facade maps
 * 1..3 to the reference's ConfigError / InvalidStateError / ProtocolError. */
enum {
  SDG_OK = 0,
  SDG_ERR_CONFIG = 1,
  SDG_ERR_INVALID_STATE = 2,
  SDG_ERR_PROTOCOL = 3,
  SDG_ERR_CUDA = 4,
  SDG_ERR_NCCL = 5
};

enum { SDG_NODES_LGL = 0, SDG_NODES_GAUSS = 1 };

enum {
  SDG_CASE_FREESTREAM = 0,
  SDG_CASE_DENSITY_WAVE = 1,
  SDG_CASE_VORTEX = 2, /* isentropic vortex in the x-y plane, z-invariant */
  SDG_CASE_TGV = 3,    /* Taylor-Green vortex in BASELINE axes (see above) */
  SDG_CASE_SWIRL = 4   /* axial density wave with rigid swirl about the x axis (annulus tests) */
};

/* One band (block) of structured, axis-aligned hexahedra (BandSpec, mesh.hpp:12-17). */
typedef struct {
  int nx;            /* elements along x */
  double width_frac; /* relative width, normalised over all bands */
  double vg_y;       /* rigid translation speed along +y (0 = static) */
  /* Per-band element counts along y and z; 0 uses the mesh-wide ny / nz (the
   * reference's BandSpec::ny override).  Bands with different counts meet at
   * a non-matching sliding interface (BASELINE configs[1]); the reference
   * requires equal counts (mesh.cpp:75-77). */
  int ny, nz;
  /* Rigid translation speed along +z (the second tangential direction of the
   * x-normal interfaces; BASELINE configs[1] slides obliquely).  SDG_MAP_BOX only. */
  double vg_z;
} sdg_band_spec;

typedef struct {
  double x0, y0, z0;
  double width, height, depth; /* extents along x, y, z */
  int ny, nz;                  /* elements along y and z (all bands) */
  int n_bands;
  sdg_band_spec bands[SDG_MAX_BANDS];
  int periodic_x, periodic_y, periodic_z;
  /* Element order inside a band for the rank split: 0 = contiguous (ix, iy, iz)
   * lexicographic blocks (proj/src/partition.cpp:48-81), 1 = Morton
   * space-filling curve, 2 = slabs along y through all bands (every rank owns
   * an equal share of every band and both sides of the sliding interfaces;
   * the reference's rule of one side per rank is lifted, which the per-kind
   * exchange rounds allow). */
  int partition;
  /* Geometry of the elements: SDG_MAP_BOX (affine hexahedra, the reference's
   * ElementMetrics, proj/src/mesh.cpp:102-111) or SDG_MAP_WARP (curved
   * hexahedra: the box mapped by a smooth sinusoidal warp inside every band,
   * see below), with `warp` the amplitude as a fraction of the element size. */
  int mapping;
  double warp;
  /* Mortars of the sliding interfaces: SDG_MORTARS_AUTO uses the reference's
   * (solver.cpp:156-526) wherever the face counts match and the slide is along y,
   * and the tensor-product (non-matching) mortars otherwise; SDG_MORTARS_TENSOR
   * routes every sliding interface through the tensor-product path (SDG_MAP_BOX),
   * which at equal counts must reproduce the reference's mortars. */
  int mortars;
  int pad_;
} sdg_mesh_spec;

enum { SDG_MORTARS_AUTO = 0, SDG_MORTARS_TENSOR = 1 };

/* SDG_MAP_WARP: a box point (x, y, z) of band b maps to
 *   X = x + A*hx*sp(tx)*s2(ty)*s2(tz),  Y = y + A*hy*sp(tx)*s2(tz),  Z = z + A*hz*sp(tx)*s2(ty)
 * with tx = (ix + (xi+1)/2)/nx_b, ty = (iy + (eta+1)/2)/ny, tz = (iz + (zeta+1)/2)/nz,
 * sp(t) = sin(pi t), s2(t) = sin(2 pi t) (both exactly 0 at integer multiples of
 * their half period), A = warp.  The warp vanishes on every band boundary, so
 * sliding interfaces stay planar and unwarped (BASELINE configs[3]: "interface
 * faces left unwarped"), and it is periodic in y and z.  A moving band carries
 * its warp rigidly (+vg t along y), so the metric terms are time-invariant.
 * Metrics are the conservative curl form (Kopriva 2006) of the degree-N LGL
 * interpolant of the mapping, evaluated at the solution nodes. */
enum { SDG_MAP_BOX = 0, SDG_MAP_WARP = 1, SDG_MAP_ANNULUS = 2 };

/* SDG_MAP_ANNULUS (BASELINE configs[2]/[3]: rotor/stator annulus): the warped
 * box point (xw, yw, zw) above (A = warp, 0 for none) maps to cylindrical
 * coordinates about the x axis,
 *   X = xw,  Y = r sin(theta),  Z = r cos(theta),  theta = yw (+ vg t),  r = zw,
 * so y is the angle (radians) and z the radius (z0 > 0).  A moving band
 * ROTATES rigidly at angular velocity vg_y about the x axis (the sliding
 * interfaces are x-normal annuli, the pairing runs along theta as before).  A
 * periodic y direction spans the full circle (height = 2 pi) or a rotationally
 * periodic sector 2 pi / m: vectors crossing the sector seam (momentum, Fv.n,
 * gradients, the moving side's mortar data) rotate by the sector angle.
 * Metric terms rotate with the band, Ja(t) = R(vg t) Ja(0); the contravariant
 * grid velocity Ja^d . vg is the discrete curl of I^N(omega r^2/2 grad_xi X),
 * so the discrete geometric conservation law holds exactly (free stream). */

typedef struct {
  double gamma, R, mu, Pr;
} sdg_gas;

typedef struct {
  int kind;
  /* freestream */
  double fs_rho, fs_v[3], fs_p;
  /* density wave: rho = 2 + alpha*sin(pi*(k.x - (k.a) t)), v = a, p = p0 */
  double dw_alpha, dw_a[3], dw_k[3], dw_p0;
  /* isentropic vortex (x-y plane) */
  double vx_eps, vx_rc, vx_rho_inf, vx_v_inf, vx_theta, vx_ma_inf, vx_center[2];
  /* Taylor-Green vortex: reference density, velocity, Mach number */
  double tgv_rho0, tgv_v0, tgv_mach;
  /* swirl: rho = 2 + dw_alpha sin(pi dw_k[0] (x - dw_a[0] t)), v = (dw_a[0], sw_omega Z, -sw_omega Y),
   * p = dw_p0 + sw_omega^2 (Y^2 + Z^2): axisymmetric, so periodic under any rotation about x */
  double sw_omega;
  /* Seeded perturbation added to the density of the case above (SURVEY §8d,
   * BASELINE configs[1] and [3]): rho += pt_amp * sum_m pt_a[m] sin(2 pi k_m . xh + pt_phi[m]),
   * xh = (c - pt_x0) / pt_len per direction with c the point x - pt_adv t (pt_coords 0)
   * or its cylindrical coordinates about the x axis (x, theta = atan2(Y, Z), r) (pt_coords 1,
   * annulus meshes: periodic across a sector seam).  Velocity and pressure are the
   * case's, so with the case's uniform velocity as pt_adv the perturbed density wave /
   * free stream stays an exact Euler solution.  pt_modes = 0: none. */
  int pt_modes, pt_coords;
  double pt_amp;
  double pt_x0[3], pt_len[3], pt_adv[3];
  double pt_k[SDG_PT_MAX_MODES][3], pt_a[SDG_PT_MAX_MODES], pt_phi[SDG_PT_MAX_MODES];
} sdg_case;

typedef struct {
  int degree;
  int node_kind;
  sdg_gas gas;
  sdg_case flow_case;
} sdg_solver_config;

/* One column of the paper's index array A, 7 ints:
 * partner_rank, i_iface, i_par, i_perp, i_sub, i_face, ctx_tag. */
#define SDG_TUPLE_INTS 7

#ifdef __cplusplus
}
#endif
#endif
