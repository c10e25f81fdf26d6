/*
 * sdg_gpu.h — the C-ABI drop-in boundary of the B200 sliding-mesh DGSEM
 * right-hand side.  Plain pointers and sizes only; every entry point returns
 * an SDG_* status code (include/sdg_types.h) and leaves a message readable
 * through sdg_last_error().
 *
 * Each entry point replaces one member of the reference's per-rank solver
 * class `sdg::RankSolver` (/root/reference/proj/src/solver.hpp:64-98) or one
 * of the setup calls its runner makes (/root/reference/proj/src/runner.cpp:33-55):
 *
 *   sdg_create                 Mesh(MeshSpec) mesh.hpp:79 + assign_ranks partition.hpp:26
 *                              + build_local_domain face_topology.hpp:60 + NodeSet/
 *                              build_basis_operators nodal_basis.hpp:26,59 +
 *                              RankSolver::RankSolver solver.hpp:66-67
 *   sdg_init_rank_maps         RankSolver::init_rank_maps            solver.hpp:70
 *   sdg_set_initial_condition  RankSolver::set_initial_condition     solver.hpp:72
 *   sdg_set_state/get_state    RankSolver::field() (mutable span)    solver.hpp:80-81
 *   sdg_step                   RankSolver::step                      solver.hpp:75
 *   sdg_compute_residual[_host] RankSolver::compute_residual         solver.hpp:85
 *   sdg_compute_gradients_host RankSolver::compute_gradients + gradients() solver.hpp:89-90
 *   sdg_suggest_dt             RankSolver::suggest_dt                solver.hpp:92
 *   sdg_time                   RankSolver::time / step_index         solver.hpp:77-78
 *   sdg_ctx_info               RankSolver::side_ctx                  solver.hpp:94
 *   sdg_total_rebuilds         RankSolver::total_rebuilds            solver.hpp:95
 *   sdg_get_pairing/mapping    RoleArrays::cols / InterfaceSideCtx::m solver.hpp:17,30 (read back
 *                              from the device, where the pairing is recomputed every stage)
 *   sdg_pairing_device         rebuild_index_arrays + build_schedule partition.hpp:100-115
 *                              (run by the device pairing kernel on caller-given faces)
 *
 * The interface-displacement update (RankSolver::update_interfaces,
 * solver.cpp:156-176) runs inside every stage: the host advances delta_base
 * exactly as solver.cpp:922-926 and assembles the long-double mortar
 * operators; the device recomputes displacement and pairing bit-exactly.
 *
 * Conventions: host pointers are borrowed for the call only; device buffers
 * are owned by the context.  All work is enqueued on the context's stream;
 * sdg_step / sdg_get_state / sdg_synchronize synchronise and report a deferred
 * InvalidStateError (admissibility is checked on the device after every
 * stage, solver.cpp:892-906).  Not thread-safe per context; one host thread
 * per GPU.  Collective-style calls must be entered by all ranks in lock-step.
 */
#ifndef SDG_GPU_H
#define SDG_GPU_H

#include <stddef.h>

#include "sdg_types.h"

/* The library is built with -fvisibility=hidden: only these entry points are
 * exported, so it links next to the reference's own sdg_core (namespace sdg). */
#if defined(__GNUC__)
#define SDG_API __attribute__((visibility("default")))
#else
#define SDG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sdg_ctx sdg_ctx;

#define SDG_NCCL_ID_BYTES 128

/* n_ranks/rank: one process (or host thread) per GPU.  nccl_id: the
 * ncclUniqueId bytes shared by all ranks (NULL when n_ranks == 1). */
SDG_API int sdg_create(const sdg_mesh_spec* mesh, const sdg_solver_config* cfg, int n_ranks, int rank,
               int device, const void* nccl_id, sdg_ctx** out);
/* Several ranks in one process sharing devices (one host thread per rank):
 * the ranks named by the same `hub` exchange through event-ordered device
 * copies instead of NCCL — the analogue of the reference's InProcHub
 * (transport.hpp:83-120), used to test the multi-rank path on one GPU. */
SDG_API int sdg_create_inproc(const sdg_mesh_spec* mesh, const sdg_solver_config* cfg, int n_ranks, int rank, int device,
                      const char* hub, sdg_ctx** out);
SDG_API void sdg_destroy(sdg_ctx* ctx);
SDG_API const char* sdg_last_error(const sdg_ctx* ctx);
SDG_API const char* sdg_global_error(void);
/* Fills SDG_NCCL_ID_BYTES bytes (rank 0 calls it and broadcasts). */
SDG_API int sdg_nccl_unique_id(void* out);
/* A one-rank NCCL communicator on `device` driven through every call of the transport
 * (transport.hpp:39-81's role): init, the all-gathers of init_rank_maps, min / sum
 * all-reduces, one grouped send + receive round of n_doubles to the rank itself.
 * SDG_OK when every result is exact. */
SDG_API int sdg_nccl_selfcheck(int device, long n_doubles);

SDG_API int sdg_init_rank_maps(sdg_ctx* ctx);
SDG_API int sdg_set_initial_condition(sdg_ctx* ctx, double t0);

SDG_API int sdg_n1(const sdg_ctx* ctx);
SDG_API long sdg_n_local_elements(const sdg_ctx* ctx);
SDG_API long sdg_n_global_elements(const sdg_ctx* ctx);
SDG_API int sdg_local_element_ids(const sdg_ctx* ctx, long* gids);

/* Local field, layout U[e][i][j][k][5] in local element order. */
SDG_API int sdg_set_state(sdg_ctx* ctx, const double* host_u);
SDG_API int sdg_get_state(sdg_ctx* ctx, double* host_u);
SDG_API int sdg_get_register(sdg_ctx* ctx, double* host_reg);
/* Device pointer of the resident field (valid until sdg_destroy). */
SDG_API int sdg_state_device_ptr(sdg_ctx* ctx, double** d_u);

SDG_API int sdg_step(sdg_ctx* ctx, double dt);
/* n steps enqueued without host synchronisation, then one synchronise. */
SDG_API int sdg_steps(sdg_ctx* ctx, double dt, int n_steps);
/* Same, but returns without synchronising (timing / overlap). */
SDG_API int sdg_steps_async(sdg_ctx* ctx, double dt, int n_steps);
SDG_API int sdg_synchronize(sdg_ctx* ctx);

/* One stage s (0..4) of the low-storage RK step that starts at time t = sdg_time
 * (lsrk_step, lsrk.hpp:20-21, as RankSolver::step drives it, solver.cpp:908-927):
 * reg = a_s reg + dt R(u, t + c_s dt); u += b_s reg; admissibility checked on the
 * device.  Stages run in order; stage 4 completes the step (time, step index,
 * interface offsets).  Five calls are bitwise one sdg_step.  Does not synchronise. */
SDG_API int sdg_rk_stage(sdg_ctx* ctx, int s, double t, double dt);
/* The scheme's coefficients a, b, c (5 each; LowStorageRK, lsrk.cpp:7-29); any may be NULL. */
SDG_API int sdg_rk_coefficients(double* a, double* b, double* c);
/* RankSolver::update_interfaces (solver.cpp:156-176): the displacement of every
 * interface side at t_stage, sigma and the long-double mortar operators on the
 * host, the rotor/stator pairing on the device (read back with sdg_ctx_info /
 * sdg_get_pairing / sdg_get_mapping).  ops (may be NULL) receives per side
 * context 4 n x n row-major operators: forward lower, forward upper, backward
 * lower, backward upper (MortarOperators, mortar.hpp). Every stage of sdg_step
 * runs this itself. */
SDG_API int sdg_update_interfaces(sdg_ctx* ctx, double t_stage, double* ops);

SDG_API int sdg_compute_residual(sdg_ctx* ctx, double t_stage, const double* d_u, double* d_dudt);
SDG_API int sdg_compute_residual_host(sdg_ctx* ctx, double t_stage, const double* h_u, double* h_dudt);
/* BR1 gradients g[e][node][12], g[3*q + dir], q in (v1, v2, v3, T). */
SDG_API int sdg_compute_gradients_host(sdg_ctx* ctx, double t_stage, const double* h_u, double* h_grad);

SDG_API int sdg_suggest_dt(sdg_ctx* ctx, double cfl, double* dt);
SDG_API int sdg_time(const sdg_ctx* ctx, double* t, int* step_index);
SDG_API long sdg_total_rebuilds(const sdg_ctx* ctx);
SDG_API int sdg_n_contexts(const sdg_ctx* ctx);
/* out5: iface, on_static, n_delta, conforming, n_faces_local (device-computed
 * at the last stage); s_delta, sigma_side. */
SDG_API int sdg_ctx_info(sdg_ctx* ctx, int ctx_id, long* out5, double* s_delta, double* sigma_side);
/* Sorted A columns of one role (0 static, 1 moving), SDG_TUPLE_INTS each. */
SDG_API int sdg_get_pairing(sdg_ctx* ctx, int role, int* ncols, int* cols);
SDG_API int sdg_get_mapping(sdg_ctx* ctx, int ctx_id, int* m);

/* Non-matching / obliquely sliding interfaces (BASELINE configs[1]; per-band ny / nz
 * or vg_z in sdg_band_spec).  Their pairing is the pair of face-interval rows (y, z)
 * recomputed on the device every stage; sdg_nc_rows reads back the device row of
 * direction dir (0: y, 1: z) of the last stage: per mortar the A face and B face
 * (faces[2k..]) and the sub-ranges (a_lo, a_hi, b_lo, b_hi) (ranges[4k..]), and the
 * displacement of side B it was built for (delta).  faces / ranges may be NULL to
 * query *n_out. */
SDG_API int sdg_n_nc_interfaces(const sdg_ctx* ctx);
SDG_API int sdg_nc_rows(sdg_ctx* ctx, int iface, int dir, long* n_out, long* faces, double* ranges, double* delta);

/* The device pairing kernel on an arbitrary face set (same contract as
 * rebuild_index_arrays + build_schedule, partition.cpp:143-169). */
SDG_API int sdg_pairing_device(int n_local, const long* faces, long n_par, long n_perp, const int* partner_ranks,
                       long n_delta, int on_static, int conforming, int self_rank, int* ncols, int* cols,
                       int* m_rows, long* face_lo, int* nsched, int* sched, int* self_entry);

/* Host-only building blocks of non-matching sliding interfaces (BASELINE
 * configs[1]; the reference requires equal face counts, proj/src/mesh.cpp:75-77):
 * sdg_subrange_ops: face <-> mortar L2 operators (n x n each, row-major) of a
 * mortar covering the face sub-range [lo, hi] of [-1, 1]; the reference's
 * build_mortar_operators (mortar.cpp:79-134) is the pair [-1, sigma], [sigma, 1],
 * reproduced bit for bit.
 * sdg_mortar_intervals: the mortars of one periodic face row where side A has
 * n_a faces of length l_a and side B n_b faces over the same period, displaced
 * by delta: per mortar (A face, B face) in faces[2k..] and (a_lo, a_hi, b_lo,
 * b_hi) in ranges[4k..], in A order (by A face, then along it).  With n_a == n_b this
 * is the reference's pairing (moving_index, sigma / -sigma, mortar.cpp:136-150).
 * faces/ranges may be NULL to query *n_out (at most n_a + n_b). */
SDG_API int sdg_subrange_ops(int degree, int node_kind, double lo, double hi, double* fwd, double* bwd);
SDG_API int sdg_mortar_intervals(long n_a, long n_b, double l_a, double delta, long* n_out, long* faces, double* ranges);
/* The same row computed by the device kernel (one block; bitwise equal to the host). */
SDG_API int sdg_mortar_intervals_device(long n_a, long n_b, double l_a, double delta, long* n_out, long* faces,
                                double* ranges);
/* A non-matching planar interface on the device: side A has nfy[0] x nfz[0]
 * faces of size l_y x l_z, side B nfy[1] x nfz[1] faces over the same periodic
 * rectangle, displaced by (d_y, d_z).  The data of side `from` (0 = A, 1 = B),
 * src[fy][fz][n][n][nc], is carried to the tensor-product mortars (row ky of y
 * by row kz of z, mortar_out[ky][kz][n][n][nc], n = degree + 1) and projected
 * onto the other side's faces (dst).  mortar_out / dst may be NULL; *n_mortars
 * receives the mortar count. */
SDG_API int sdg_interface_project_device(int degree, int node_kind, const long* nfy, const long* nfz, double l_y,
                                 double l_z, double d_y, double d_z, int nc, int from, const double* src,
                                 double* mortar_out, double* dst, long* n_mortars);

/* The surface flux of a non-matching planar interface with normal +x, side A
 * (nfy[0] x nfz[0] faces) below and side B (nfy[1] x nfz[1]) above, displaced by
 * (d_y, d_z): both sides' traces u_a / u_b ([fy][fz][n][n][5]) and, when the gas
 * is viscous and both are non-NULL, gradients g_a / g_b ([..][12], d(u,v,w)/dx_j
 * then dT/dx_j) go to the tensor-product mortars; the two-sided Roe + central
 * viscous flux (face_numerical_flux, solver.cpp:308-321) is evaluated at the
 * mortar nodes (flux_mortar[M][n][n][5], may be NULL) and L2-projected back onto
 * both sides' faces (flux_a, flux_b; the flux along +x on both).  With equal
 * counts this is the reference's mortar chain (solver.cpp:156-176). */
SDG_API int sdg_interface_flux_device(const sdg_gas* gas, int degree, int node_kind, const long* nfy, const long* nfz,
                              double l_y, double l_z, double d_y, double d_z, const double* u_a, const double* u_b,
                              const double* g_a, const double* g_b, double* flux_mortar, double* flux_a,
                              double* flux_b, long* n_mortars);

/* The same interface's lifting mean: the mean of both sides' primitive
 * (u, v, w, T) at the mortar nodes (lift_mortar[M][n][n][4], may be NULL; run_lifting,
 * solver.cpp:597-727), L2-projected back onto both sides' faces (lift_a, lift_b). */
SDG_API int sdg_interface_lift_device(const sdg_gas* gas, int degree, int node_kind, const long* nfy, const long* nfz,
                              double l_y, double l_z, double d_y, double d_z, const double* u_a, const double* u_b,
                              double* lift_mortar, double* lift_a, double* lift_b, long* n_mortars);

/* Diagnostics on the device (integrate_mass_energy / error_norms /
 * max_freestream_deviation, diagnostics.cpp:31-87): out[14] = mass, energy,
 * volume, L2 error[5], Linf error[5], max deviation; the errors are against the
 * exact case state at time t when with_exact != 0 (else zero). */
SDG_API int sdg_diagnostics(sdg_ctx* ctx, double t, int with_exact, double* out);
/* SDGFLD1 snapshot of the global field (write_snapshot / read_snapshot,
 * snapshot.cpp:10-56) with a 3D header; collective over ranks. */
SDG_API int sdg_write_snapshot(sdg_ctx* ctx, const char* path, double time);
SDG_API int sdg_read_snapshot(sdg_ctx* ctx, const char* path, double* time);

/* Host-only partition / message plan of one rank (no GPU needed): JSON with the
 * local elements, the conforming halo peers and face keys in send order, and
 * the per-partner mortar blocks of both roles at interface displacement
 * `delta` (init_rank_maps + build_schedule, solver.cpp:95-133,
 * partition.cpp:154-169).  *len receives the full length. */
SDG_API int sdg_plan_json(const sdg_mesh_spec* mesh, int n_ranks, int rank, double delta, char* buf, long cap, long* len);

/* Host-only curved metric terms of one rank's elements (no GPU needed), as
 * uploaded by sdg_create for an SDG_MAP_WARP mesh: met n_local x N3 x 10
 * (Ja^d_c at [3d + c], 1/J), fmet n_local x 6 x N2 x 4 (unit +xi normal, sJ);
 * SDG_MAP_ANNULUS: 13 per node (+ contravariant grid velocity per unit omega)
 * and 6 per face node (+ (vg / omega) . n, pad).
 * The reference's metrics are affine (ElementMetrics, proj/src/mesh.cpp:102-111).
 * met/fmet may be NULL to query *n_local; elements in sdg_local_element_ids order. */
SDG_API int sdg_metrics_host(const sdg_mesh_spec* mesh, int degree, int node_kind, int n_ranks, int rank, double* met,
                     double* fmet, long* n_local);

/* Communication trace of this rank (TraceRow, transport.hpp:28-37): JSON rows
 * [step, stage, src, dst, bytes, kind, is_send], step -1 = init; kinds follow
 * MsgKind (transport.hpp:13-24).  sdg_inject_collective is the audit's
 * negative-test hook (RankSolver::inject_collective, solver.cpp:961-964). */
SDG_API int sdg_trace_json(sdg_ctx* ctx, char* buf, long cap, long* len);
SDG_API int sdg_inject_collective(sdg_ctx* ctx);

/* Instrumentation: the cudaStream_t the context enqueues on, the number of
 * kernels this library launched, and per-kernel-class CUDA-event timing of
 * the next sdg_steps_async call (ms, summed over launches). */
SDG_API void* sdg_stream(sdg_ctx* ctx);
SDG_API long sdg_kernel_launches(const sdg_ctx* ctx);
SDG_API int sdg_enable_kernel_timing(sdg_ctx* ctx, int on);
/* names: comma-separated kernel classes; ms/launches per class. */
SDG_API int sdg_kernel_timing(sdg_ctx* ctx, char* names, int names_cap, double* ms, long* launches, int cap,
                      int* n_classes);

#ifdef __cplusplus
}
#endif
#endif
