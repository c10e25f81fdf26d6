// Device-side data structures and launch wrappers of the B200 path.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/sdg_types.h"
#include "host.hpp"

namespace sdg {

struct GasD {
  double gamma, gm1, R, inv_R, mu, lam, kcond;
  int viscous;
};

struct BandD {
  double x_lo, hx, hy, hz, vg;
  double vgz;      // translation speed along +z (oblique sliding, affine only)
  double jac, inv_jac;
  double cdir[3];  // sJ_d / J
  double sj[3];    // sJ_d
  double nxd;      // elements along x (curved mapping)
};

// Per-run constants, passed by value (__grid_constant__) to every element kernel.
struct ElemConsts {
  double dhat[kMaxN1 * kMaxN1];  // D-hat(i,m) = w_m D(m,i) / w_i  (solver.cpp:38-41)
  double fl[kMaxN1], fr[kMaxN1];  // l_j(-1), l_j(+1)
  double liftw[2][kMaxN1];        // l_j(-+1) / w_j
  double inv_w[kMaxN1];
  double w[kMaxN1];
  double x[kMaxN1];
  BandD bands[SDG_MAX_BANDS];
  GasD gas;
  double y0, z0;
  sdg_case flow_case;
  int mapping, ny, nz, pad;  // SDG_MAP_BOX / SDG_MAP_WARP / SDG_MAP_ANNULUS (include/sdg_types.h)
  double warp;
  double sec_c, sec_s;       // cos / sin of the periodic annulus sector angle (side_rot)
};

// Deferred admissibility / protocol error record (written by the first failing thread).
struct ErrRec {
  int flag;  // 0 none, 2 invalid state, 3 protocol
  int step, stage, pad;
  long long elem, node;
  double vals[5];
};

// Pointers of the resident fields and face arrays.
struct FieldPtrs {
  double* U;
  double* reg;
  double* out;         // dudt (residual mode)
  double* trace;       // (6E + H) slots x N2 x 5   face traces of U (read: stage s)
  double* trace_out;   // the other trace buffer (written: traces of the stage s+1 state)
  double* fvn;         // (6E + H) slots x N2 x 4   viscous normal flux (mom x,y,z, energy)
  const double* slide_lift;  // S x N2 x 4
  const double* slide_flux;  // S x N2 x 5
  double* slide_g;           // S x N2 x 12
  double* dir_g;             // ND x N2 x 12
  const int8_t* side_type;   // E x 6
  const int* side_idx;       // E x 6
  const int* coords;         // E x 4 (band, ix, iy, iz)
  const int* side_code;      // E x 8: idx | type << 29 for the 6 sides, [6] = band, [7] pad (32 B/element)
  double* grad_out;          // optional E x N3 x 12
  const double* met;         // curved: E x N3 x 10 (Ja^d_c at 3d + c, 1/J)
  const double* fmet;        // curved: 6E x N2 x 4 (unit +xi normal, sJ) per local side
  const int8_t* side_rot;    // E x 6: neighbour vectors rotate by side_rot * sector angle (annulus sectors)
  double* visc;              // curved, viscous, even N+1: E x 9 x N3 (tau_00 01 02 11 12 22, k dT/dx_d), written by
                             // the gradient kernel and read by k_update_cv in place of a second gradient evaluation
  ErrRec* err;
  int E;        // element kernels process local elements [e_first, E)
  int e_first;  // (interior / boundary split for exchange overlap; 0 = all)
};

struct StageArgs {
  double t_stage, dt, rk_a, rk_b;
  int mode;  // 0: RK update (+ trace output), 1: residual into out
  int step, stage;
  // Annulus: cos / sin of each band's rotation angle vg * t_stage, evaluated once on the host
  // (every element of a band shares it; conforming faces never join two bands).
  double rot_c[SDG_MAX_BANDS], rot_s[SDG_MAX_BANDS];
};

// ---- mortar side ----
// Interface-side context as the device sees it.
struct CtxD {
  int iface, on_static, role, n_faces;  // n_faces = local faces of this side
  int face_off;                         // offset into ctx_faces / slide ids
  int map_off;                          // offset into the partner rank map
  long long n_par, n_perp;
  int static_is_left;
  double l_par, vg_rel;
};

struct PairingArgs {
  int n_ctx;
  CtxD ctx[kMaxCtx];
  int role_ctx[2][kMaxCtx];
  int role_nctx[2];
  long long iface_base[kMaxCtx];  // dense-key base per interface (same for both roles)
  long long iface_nperp[kMaxCtx];
  long long dense_size;
  int n_ifaces;
  int self_rank;
  double delta_base[kMaxCtx];
  double time, t_stage;
  int expect_mortars[2];           // host-side count per role, checked on the device
};

struct PairingPtrs {
  const int* ctx_face_par;   // per ctx face: i_par (static frame for static, moving index for moving)
  const int* ctx_face_perp;
  const int* ctx_face_slide; // compact sliding index of the ctx face
  const int* partner_map;    // concatenated partner-side rank maps
  int* pres[2];              // dense scratch per role
  int* payload[2];
  int* cols[2];              // SDG_TUPLE_INTS per column
  int* m;                    // per ctx: 2 x n_faces (offset 2*face_off)
  int* ctx_state;            // per ctx: n_delta, conforming
  double* ctx_sdelta;
  int* n_mortars;            // 2
  ErrRec* err;
};

struct MortarOps {
  double op[kMaxCtx][2][kMaxN1 * kMaxN1];
};

struct MortarPtrs {
  const double* trace;
  double* u_mine[2];
  double* u_theirs;     // static role
  double* lift[2];
  double* g_mine[2];
  double* g_theirs;     // static role
  double* flux[2];
  double* slide_lift;
  double* slide_flux;
  const double* slide_g;
  const int* slide_elem;   // S: element
  const int* slide_side;   // S: side
  const int* slide_ctx;    // S: ctx id
  const int* slide_f;      // S: face index within ctx
  const int* m;            // per ctx 2 x n_faces at 2*face_off
  const int* ctx_face_off; // n_ctx
  const int* ctx_nf;       // n_ctx
  const int* ctx_role;     // n_ctx (0 static, 1 moving)
  const int* ctx_state;    // per ctx: n_delta, conforming
  const int* n_mortars;    // 2
  const int* cols_static;  // ctx of each static mortar: cols[7*c + 6]
  const int* cols_moving;  // moving role's columns
  const int* ctx_static_left;
  int S;
  // Periodic annulus sector: a mortar's moving partner sits at the static location + k alpha,
  // k = wind[ctx] + (i_par - n_delta + i_sub - 1 < 0): static-role kernels rotate the partner's
  // values by R(-k alpha), the moving role's back projection by R(+k alpha).
  int sector;
  double alpha;
  int wind[kMaxCtx];
};

// ---- launch wrappers (kernels.cu) ----
void launch_prolong(int n1, const ElemConsts& c, const FieldPtrs& p, cudaStream_t st);
void launch_gradient(int n1, const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st);
void launch_update(int n1, const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st);
// The warp-specialised persistent TMA gradient kernel for affine elements (even N+1);
// false when not applicable (the plain launch_gradient then runs).
bool launch_gradient_tma(int n1, const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, int n_sm,
                         cudaStream_t st);
// Curved-element kernels (SDG_MAP_WARP / SDG_MAP_ANNULUS; csrc/curved.cuh).
void launch_gradient_curved(int n1, const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st);
void launch_update_curved(int n1, const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st);
// Affine update in the bulk-loaded, non-persistent structure of curved.cuh (even N+1;
// false when not applicable: the plain launch_update then runs).
bool launch_update_affine_b(int n1, const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st);
void launch_pairing(const PairingArgs& a, const PairingPtrs& p, cudaStream_t st);
// Mortars of one non-matching periodic face row (device merge_intervals, host.cpp).
void launch_mortar_intervals(long long n_a, long long n_b, double l_a, double delta, long long* faces,
                             double* ranges, long long* n_out, cudaStream_t st);
// Non-matching planar interface: source faces -> tensor-product mortars -> target faces.
void launch_nc_transfer(int n, int nc, const double* src, long long src_nfz, const long long* iv_y,
                        const long long* iv_z, int src_col, long long my, long long mz, const double* Fy,
                        const double* Fz, double* mortar, long long dst_nfy, long long dst_nfz, const int* off_y,
                        const int* idx_y, const int* off_z, const int* idx_z, const double* By, const double* Bz,
                        double* dst, cudaStream_t st);
// The y and z rows of one interface in one launch (separate output buffers).
struct IvRow {
  long long n_a, n_b;
  double l_a, delta;
  long long* faces;
  double* ranges;
  long long* n_out;
};
struct IvRows {
  IvRow row[2];
};
void launch_mortar_intervals2(const IvRows& rows, cudaStream_t st);
// Batched transfers of one non-matching interface (up to 4 face -> mortar jobs, up to
// 2 mortar -> face jobs per launch).
struct NcMortarJob {
  const double* src;
  long long src_nfz;
  int col, nc;
  const double *Fy, *Fz;
  double* out;
};
struct NcMortarJobs {
  NcMortarJob job[4];
  int n;
};
struct NcFaceJob {
  long long nfy, nfz;
  const int *off_y, *idx_y, *off_z, *idx_z;
  const double *By, *Bz;
  double* dst;
};
struct NcFaceJobs {
  NcFaceJob job[2];
  int n;
};
void launch_nc_to_mortar_batch(int n, const long long* iv_y, const long long* iv_z, long long my, long long mz,
                               const NcMortarJobs& jobs, cudaStream_t st);
void launch_nc_to_face_batch(int n, int nc, const double* mortar, long long mz, const NcFaceJobs& jobs,
                             cudaStream_t st);
// Two-sided Riemann (+ viscous) flux at the mortar nodes of a non-matching interface.
void launch_nc_mortar_flux(long long nodes, const GasD& g, int dir, double vg, const double* ua, const double* ub,
                           const double* ga, const double* gb, double* flux, int* bad, cudaStream_t st);
void launch_nc_mortar_lift(long long nodes, const GasD& g, const double* ua, const double* ub, double* lift,
                           cudaStream_t st);
// One non-matching / oblique interface at one stage, as the in-stage kernels see it.
// Rows per direction d (0: y, 1: z): the host's (h_*, from which its operators were
// built) and the device's (d_*, recomputed by k_nc_rows and used for indexing).
// Side s = 0 (A, the left band's x+ faces) / 1 (B, the right band's x- faces).
struct NcStage {
  long long nfy[2], nfz[2];  // faces per side
  long long my, mz;          // mortars per direction
  long long n_a[2], n_b[2];  // row parameters per direction
  double l_a[2], delta[2];
  const long long* h_faces[2];
  const double* h_ranges[2];
  long long* d_faces[2];
  double* d_ranges[2];
  long long* d_n;                    // 2
  const double* F[2][2];             // [side][dir]: forward (face -> mortar) n x n per row
  const double* B[2][2];             // [side][dir]: backward (mortar -> face) n x n per row
  const int* off[2][2];              // [side][dir]: CSR offsets over the side's face rows
  const int* idx[2][2];              // [side][dir]: CSR row indices
};
void launch_nc_rows(const NcStage& S, int iface, ErrRec* err, cudaStream_t st);
void launch_nc_fill(int n, int nc, const double* src, const NcStage& S, const int* const tab[2], double* const out[2],
                    cudaStream_t st);
void launch_nc_project(int n, int nc, const double* mortar, const NcStage& S, const int* const tab[2], double* dst,
                       cudaStream_t st);
void launch_nc_flux(long long nodes, const GasD& g, const double* ua, const double* ub, const double* ga,
                    const double* gb, double* flux, ErrRec* err, cudaStream_t st);
void launch_mortar_fill(int n1, int ncomp, const double* src, double* const dst[2], const MortarOps& ops,
                        const MortarPtrs& p, cudaStream_t st);
void launch_mortar_lift(int n1, const GasD& g, const MortarPtrs& p, int max_mortars, cudaStream_t st);
void launch_mortar_backproject(int n1, int ncomp, const double* const src[2], double* dst, const MortarOps& ops,
                               const MortarPtrs& p, cudaStream_t st);
void launch_mortar_flux(int n1, const GasD& g, int viscous, const MortarPtrs& p, int max_mortars, ErrRec* err,
                        cudaStream_t st);
// Diagnostics (diagnostics.cpp:31-87): per-block partial sums of mass, energy,
// volume and squared errors, and maxima of |errors| — kDiagVals per block.
constexpr int kDiagVals = 14;
int launch_diagnostics(int n1, const ElemConsts& c, const FieldPtrs& p, double t, int with_exact, double* partial,
                       int max_blocks, cudaStream_t st);
void launch_suggest_dt(int n1, const ElemConsts& c, const FieldPtrs& p, double cfl, int degree,
                       unsigned long long* out, cudaStream_t st);

}  // namespace sdg
