/*
 * TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
 *
 * sdg3d.h — C API of the 3D CPU oracle: a plain restatement of the reference's
 * sliding-mesh DGSEM right-hand side (/root/reference/proj/src/solver.cpp) in
 * three dimensions.  Only tests/, __graft_entry__.smoke() and bench.py's CPU
 * baseline leg may load it; the B200 product never links or calls it.
 *
 * Parity pinning: the restatement is checked against the reference library
 * itself (oracle/_ref, built from /root/reference/proj/src by oracle/Makefile)
 * through the z-invariant embedding (a 3D run with w = 0 and z-constant data
 * reproduces the 2D reference on every z layer), the reference's golden
 * vectors (Appendix-A pairing, mortar operator identities, shipped CSVs) and
 * the free-stream / conservation properties.  See tests/test_oracle_*.py.
 */
#ifndef SDG3D_ORACLE_H
#define SDG3D_ORACLE_H

#include <stddef.h>

#include "../include/sdg_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_solver orc_solver;

/* Single-rank solver over the whole mesh (the reference's results are
 * bitwise independent of the rank count, proj/tests/test_runner.cpp:32-50). */
int orc_create(const sdg_mesh_spec* mesh, const sdg_solver_config* cfg, orc_solver** out);
void orc_destroy(orc_solver* s);
const char* orc_last_error(const orc_solver* s);
const char* orc_global_error(void);
int orc_set_threads(int n);

long orc_n_elements(const orc_solver* s);
int orc_n1(const orc_solver* s);
int orc_n_contexts(const orc_solver* s);

int orc_set_initial_condition(orc_solver* s, double t0);
int orc_set_state(orc_solver* s, const double* u);
int orc_get_state(const orc_solver* s, double* u);
int orc_get_register(const orc_solver* s, double* reg);
int orc_compute_residual(orc_solver* s, double t_stage, const double* u, double* dudt);
int orc_compute_gradients(orc_solver* s, double t_stage, const double* u, double* grad);
int orc_step(orc_solver* s, double dt);
int orc_steps(orc_solver* s, double dt, int n);
/* One RK stage of a step (stage in 0..4); orc_step == 5 stages + bookkeeping. */
int orc_suggest_dt(const orc_solver* s, double cfl, double* dt);
double orc_time(const orc_solver* s);
long orc_total_rebuilds(const orc_solver* s);

/* Interface context state after the last update (one per (iface, side)):
 * out[0]=iface, out[1]=on_static, out[2]=n_delta, out[3]=conforming,
 * out[4]=n_faces_local; sd = s_delta, sig = sigma_side. */
int orc_ctx_info(const orc_solver* s, int ctx, long* out5, double* s_delta, double* sigma_side);
/* Sorted index array A of one role (0 = static, 1 = moving): ncols and
 * SDG_TUPLE_INTS ints per column.  cols may be NULL to query ncols. */
int orc_get_pairing(const orc_solver* s, int role, int* ncols, int* cols);
/* m(i_sub, i_face) of one context: 2 rows of n_faces_local ints. */
int orc_get_mapping(const orc_solver* s, int ctx, int* m);

/* Curved metrics (SDG_MAP_WARP): met E x N3 x 10 (Ja^d_c at [3d+c], 1/J),
 * fmet E x 6 x N2 x 4 (unit +xi normal, sJ).  ConfigError for affine meshes. */
int orc_get_metrics(const orc_solver* s, double* met, double* fmet);

/* Mass and energy integrals (proj/src/diagnostics.cpp:31-50). */
int orc_integrate_mass_energy(const orc_solver* s, const double* u, double* out2);
/* Exact case solution sampled at the nodes at time t (full field). */
int orc_sample_case(const orc_solver* s, double t, double* u);

/* ---- standalone restatements used by the golden-vector tests ---- */
int orc_nodes(int degree, int kind, double* nodes, double* weights);
/* D (n*n row-major), l(-1), l(+1). */
int orc_basis(int degree, int kind, double* diff, double* face_left, double* face_right);
/* fwd/bwd: [2][n][n] (Lower, Upper), row-major. */
int orc_mortar_ops(int degree, int kind, double sigma, double* fwd, double* bwd);
/* Non-matching interfaces (BASELINE configs[1]): mortar operators of a face
 * sub-range [lo, hi] (n*n each) and the mortars of one periodic face row,
 * faces 2 and ranges 4 per mortar (see include/sdg_gpu.h sdg_mortar_intervals). */
int orc_subrange_ops(int degree, int kind, double lo, double hi, double* fwd, double* bwd);
/* Non-matching / oblique interfaces: the rows (y: dir 0, z: dir 1) of the last
 * residual evaluation, as sdg_nc_rows on the device. */
int orc_n_nc_interfaces(const orc_solver* s);
int orc_nc_rows(const orc_solver* s, int iface, int dir, long* n_out, long* faces, double* ranges, double* delta);
int orc_mortar_intervals(long n_a, long n_b, double l_a, double delta, long* n_out, long* faces, double* ranges);
int orc_displacement(double delta, double l_par, long n_faces, double* d, long* n_delta,
                     double* s_delta);
long orc_moving_index(long i_par, long n_delta, int i_sub, long n_faces);
long orc_static_index(long i_moving, long n_delta, int i_sub, long n_faces);
/* rebuild_index_arrays (proj/src/partition.cpp:143-152) for one face set:
 * faces: n_faces_local x (i_face, i_par, i_perp); partner_ranks: n_perp*n_par,
 * row-major by i_perp.  Outputs cols (SDG_TUPLE_INTS per column), m rows
 * (2 x (hi-lo+1)), face_lo, and the schedule (partner, offset, count)
 * triples plus the self entry. */
int orc_pairing(int n_local, const long* faces, long n_par, long n_perp,
                const int* partner_ranks, long n_delta, int on_static, int conforming,
                int self_rank, int* ncols, int* cols, int* m_rows, long* face_lo,
                int* nsched, int* sched, int* self_entry);

/* Roe + viscous face flux (3D), exposed for unit tests. */
int orc_face_flux(const sdg_gas* gas, const double* um, const double* up, int dir,
                  double vg_n, const double* gm, const double* gp, double* out);

#ifdef __cplusplus
}
#endif
#endif
