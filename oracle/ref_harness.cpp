// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
//
// C shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It exposes
// the reference's own entry points to the Python tests so the 3D restatement
// (oracle/sdg3d.cpp) and the golden fixtures in tests/golden/ can be pinned to
// the reference's bits.  Nothing here re-implements reference logic.
#include <algorithm>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "config.hpp"
#include "diagnostics.hpp"
#include "driver.hpp"
#include "errors.hpp"
#include "face_topology.hpp"
#include "flux.hpp"
#include "lsrk.hpp"
#include "mesh.hpp"
#include "mortar.hpp"
#include "nodal_basis.hpp"
#include "partition.hpp"
#include "runner.hpp"
#include "solver.hpp"
#include "transport.hpp"

using namespace sdg;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const InvalidStateError& e) {
    g_err = e.what();
    return 2;
  } catch (const ProtocolError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // namespace

extern "C" {

// 2D problem description mirroring MeshSpec/CaseDef (mesh.hpp:12-26, cases.hpp:11-28).
struct ref_spec {
  double width, height;
  int ny;
  int n_bands;
  int band_nx[16];
  double band_frac[16];
  double band_vg[16];
  int periodic_x, periodic_y;
  int degree, node_kind;  // 0 lgl, 1 gauss
  double gamma, R, mu, Pr;
  int case_kind;  // 0 freestream, 1 density wave, 2 vortex
  double fs[4];   // rho, vx, vy, p
  double dw[4];   // alpha, ax, ay, p0
  double vx[8];   // eps, rc, rho_inf, v_inf, theta, ma_inf, cx, cy
};

static MeshSpec mesh_of(const ref_spec& s) {
  MeshSpec m;
  m.width = s.width;
  m.height = s.height;
  m.ny = s.ny;
  m.periodic_x = s.periodic_x != 0;
  m.periodic_y = s.periodic_y != 0;
  for (int b = 0; b < s.n_bands; ++b) m.bands.push_back({s.band_nx[b], s.band_frac[b], s.band_vg[b], 0});
  return m;
}

static SolverConfig cfg_of(const ref_spec& s) {
  SolverConfig c;
  c.gas.gamma = s.gamma;
  c.gas.R = s.R;
  c.gas.mu = s.mu;
  c.gas.Pr = s.Pr;
  c.flow_case.kind = static_cast<CaseDef::Kind>(s.case_kind);
  c.flow_case.fs = {s.fs[0], {s.fs[1], s.fs[2]}, s.fs[3]};
  c.flow_case.dw = {s.dw[0], {s.dw[1], s.dw[2]}, s.dw[3]};
  c.flow_case.vx.eps = s.vx[0];
  c.flow_case.vx.rc = s.vx[1];
  c.flow_case.vx.rho_inf = s.vx[2];
  c.flow_case.vx.v_inf = s.vx[3];
  c.flow_case.vx.theta = s.vx[4];
  c.flow_case.vx.ma_inf = s.vx[5];
  c.flow_case.vx.center0 = {s.vx[6], s.vx[7]};
  return c;
}

static NodeKind kind_of(int k) { return k == 1 ? NodeKind::LegendreGauss : NodeKind::LegendreGaussLobatto; }

const char* ref_last_error(void) { return g_err.c_str(); }

long ref_field_size(const ref_spec* s) {
  const Mesh mesh(mesh_of(*s));
  const long n = s->degree + 1;
  return static_cast<long>(mesh.n_elements()) * n * n * kNumVars;
}

// Single-rank RankSolver (the SingleRank fixture of proj/tests/test_solver.cpp:28-48):
// set_initial_condition(t0), optionally overwrite the field, then
//   mode 0: compute_residual(t_stage) -> out
//   mode 1: compute_gradients(t_stage) -> out (6 per node)
//   mode 2: n_steps steps of dt -> out = field; aux[0] = time, aux[1] = rebuilds
//   mode 3: suggest_dt(cfl = t_stage) -> aux[0]
// u_in may be NULL.  On a single rank the element order equals the global id.
int ref_single_rank(const ref_spec* s, double t0, const double* u_in, int mode, double t_stage, double dt,
                    int n_steps, double* out, double* aux) {
  return guard([&] {
    const Mesh mesh(mesh_of(*s));
    const NodeSet ns(s->degree, kind_of(s->node_kind));
    const BasisOperators basis = build_basis_operators(ns);
    const Ownership own = assign_ranks(mesh, 1);
    InProcHub hub(1);
    InProcTransport tr(hub, 0);
    RankSolver solver(mesh, own, build_local_domain(mesh, own, 0), ns, basis, cfg_of(*s), tr);
    solver.init_rank_maps();
    solver.set_initial_condition(t0);
    if (u_in) std::copy(u_in, u_in + solver.field().size(), solver.field().begin());
    if (mode == 0) {
      std::vector<double> dudt(solver.field().size(), 0.0);
      solver.compute_residual(t_stage, solver.field(), dudt);
      std::copy(dudt.begin(), dudt.end(), out);
    } else if (mode == 1) {
      solver.compute_gradients(t_stage, solver.field());
      std::copy(solver.gradients().begin(), solver.gradients().end(), out);
    } else if (mode == 2) {
      for (int k = 0; k < n_steps; ++k) solver.step(dt);
      std::copy(solver.field().begin(), solver.field().end(), out);
      if (aux) {
        aux[0] = solver.time();
        aux[1] = static_cast<double>(solver.total_rebuilds());
      }
    } else {
      if (aux) aux[0] = solver.suggest_dt(t_stage);
    }
  });
}

// Multi-rank run through the reference runner (runner.cpp:297-303); field in gid order.
int ref_run(const ref_spec* s, double dt, int n_steps, int ranks, int backend, double* field_out,
            double* wall_out) {
  return guard([&] {
    const Mesh mesh(mesh_of(*s));
    const NodeSet ns(s->degree, kind_of(s->node_kind));
    const BasisOperators basis = build_basis_operators(ns);
    RunnerOptions opts;
    opts.n_ranks = ranks;
    opts.backend = backend == 1 ? Backend::Proc : Backend::InProc;
    opts.dt = dt;
    opts.n_steps = n_steps;
    const RunOutput r = run_simulation(mesh, ns, basis, cfg_of(*s), opts);
    std::copy(r.field.data.begin(), r.field.data.end(), field_out);
    if (wall_out) *wall_out = r.wall_max;
  });
}

// run_case on a shipped config file (driver.cpp:42-91), no outputs written.
// out: t_end, n_steps, dt, l2[4], linf_rho, mass_drift, energy_drift, wall, pid
int ref_run_case(const char* path, double* out) {
  return guard([&] {
    RunConfig cfg = RunConfig::from_file(path);
    cfg.ranks = 1;
    const CaseReport r = run_case(cfg, false);
    out[0] = r.t_end;
    out[1] = static_cast<double>(r.n_steps);
    out[2] = r.dt;
    for (int v = 0; v < 4; ++v) out[3 + v] = r.norms.l2[v];
    out[7] = r.norms.linf[0];
    out[8] = r.mass_drift;
    out[9] = r.energy_drift;
    out[10] = r.wall;
    out[11] = r.pid;
  });
}

// convergence_study on a shipped config (driver.cpp:93-152); rows of
// (degree, level, n_elements, h, l2_rho, order).  *n_rows in: capacity, out: rows.
int ref_convergence(const char* path, double* rows, int* n_rows) {
  return guard([&] {
    RunConfig cfg = RunConfig::from_file(path);
    cfg.ranks = 1;
    const auto r = convergence_study(cfg, false);
    const int cap = *n_rows;
    *n_rows = static_cast<int>(r.size());
    for (int i = 0; i < std::min(cap, *n_rows); ++i) {
      rows[6 * i + 0] = r[i].degree;
      rows[6 * i + 1] = r[i].level;
      rows[6 * i + 2] = r[i].n_elements;
      rows[6 * i + 3] = r[i].h;
      rows[6 * i + 4] = r[i].l2_rho;
      rows[6 * i + 5] = r[i].order;
    }
  });
}

int ref_nodes(int degree, int kind, double* nodes, double* weights) {
  return guard([&] {
    const NodeSet ns(degree, kind_of(kind));
    std::copy(ns.nodes().begin(), ns.nodes().end(), nodes);
    std::copy(ns.weights().begin(), ns.weights().end(), weights);
  });
}

int ref_basis(int degree, int kind, double* diff, double* fl, double* fr) {
  return guard([&] {
    const NodeSet ns(degree, kind_of(kind));
    const BasisOperators b = build_basis_operators(ns);
    const int n = ns.count();
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) diff[i * n + j] = b.diff(i, j);
    std::copy(b.face_left.begin(), b.face_left.end(), fl);
    std::copy(b.face_right.begin(), b.face_right.end(), fr);
  });
}

int ref_mortar_ops(int degree, int kind, double sigma, double* fwd, double* bwd) {
  return guard([&] {
    const NodeSet ns(degree, kind_of(kind));
    const MortarOperators ops = build_mortar_operators(ns, sigma);
    const int n = ns.count();
    for (int h = 0; h < 2; ++h)
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          fwd[(h * n + i) * n + j] = ops.to_mortar[h](i, j);
          bwd[(h * n + i) * n + j] = ops.to_face[h](i, j);
        }
  });
}

int ref_displacement(double delta, double l_par, long n_faces, double* d, long* n_delta, double* s_delta) {
  const InterfaceState st = displacement_state(delta, l_par, n_faces);
  *d = st.delta;
  *n_delta = st.n_delta;
  *s_delta = st.s_delta;
  return 0;
}

long ref_moving_index(long i_par, long n_delta, int i_sub, long n_faces) {
  return moving_index(i_par, n_delta, i_sub, n_faces);
}
long ref_static_index(long i_moving, long n_delta, int i_sub, long n_faces) {
  return static_index(i_moving, n_delta, i_sub, n_faces);
}

// rebuild_index_arrays + build_schedule (partition.cpp:143-169).
int ref_pairing(int n_local, const long* faces, long n_par, long n_perp, const int* partner_ranks, long n_delta,
                int on_static, int conforming, int self_rank, int* ncols, int* cols, int* m_rows, long* face_lo,
                int* nsched, int* sched, int* self_entry) {
  return guard([&] {
    std::vector<LocalInterfaceFace> fs(n_local);
    for (int f = 0; f < n_local; ++f) fs[f] = {faces[3 * f], faces[3 * f + 1], faces[3 * f + 2]};
    RankMaps maps;
    RankMap& mp = on_static ? maps.moving_side : maps.static_side;
    mp.n_par = n_par;
    mp.n_perp = n_perp;
    mp.ranks.assign(partner_ranks, partner_ranks + n_par * n_perp);
    IndexArrayA a;
    MappingM m;
    rebuild_index_arrays(fs, maps, n_delta, n_par, on_static != 0, conforming != 0, a, m);
    *ncols = static_cast<int>(a.cols.size());
    for (size_t i = 0; i < a.cols.size(); ++i) {
      int* o = cols + i * 7;
      o[0] = a.cols[i].partner_rank;
      o[1] = a.cols[i].i_iface;
      o[2] = static_cast<int>(a.cols[i].i_par);
      o[3] = static_cast<int>(a.cols[i].i_perp);
      o[4] = a.cols[i].i_sub;
      o[5] = static_cast<int>(a.cols[i].i_face);
      o[6] = a.cols[i].ctx_tag;
    }
    *face_lo = m.face_lo;
    const size_t w = m.rows[0].size();
    for (size_t q = 0; q < w; ++q) {
      m_rows[q] = m.rows[0][q];
      m_rows[w + q] = m.rows[1][q];
    }
    ScheduleEntry self;
    const auto sc = build_schedule(a.cols, self_rank, self);
    *nsched = static_cast<int>(sc.size());
    for (size_t i = 0; i < sc.size(); ++i) {
      sched[3 * i] = sc[i].partner;
      sched[3 * i + 1] = sc[i].offset;
      sched[3 * i + 2] = sc[i].count;
    }
    self_entry[0] = self.partner;
    self_entry[1] = self.offset;
    self_entry[2] = self.count;
  });
}

// Pairing actually used by a single-rank solver at stage time t_stage after
// set_initial_condition(t0): statics (role 0) / movings (role 1) columns.
// Exercised through compute_gradients' update_interfaces; read via side_ctx.
int ref_ctx_state(const ref_spec* s, double t0, double t_stage, int iface, int on_static, long* out3,
                  double* s_delta, int* m_rows, int* n_faces_local) {
  return guard([&] {
    const Mesh mesh(mesh_of(*s));
    const NodeSet ns(s->degree, kind_of(s->node_kind));
    const BasisOperators basis = build_basis_operators(ns);
    const Ownership own = assign_ranks(mesh, 1);
    InProcHub hub(1);
    InProcTransport tr(hub, 0);
    RankSolver solver(mesh, own, build_local_domain(mesh, own, 0), ns, basis, cfg_of(*s), tr);
    solver.init_rank_maps();
    solver.set_initial_condition(t0);
    std::vector<double> dudt(solver.field().size(), 0.0);
    solver.compute_residual(t_stage, solver.field(), dudt);
    const InterfaceSideCtx* c = solver.side_ctx(iface, on_static != 0);
    if (!c) throw ConfigError("no such interface side");
    out3[0] = c->st.n_delta;
    out3[1] = c->conforming ? 1 : 0;
    out3[2] = c->rebuild_count;
    *s_delta = c->st.s_delta;
    *n_faces_local = static_cast<int>(c->faces.size());
    const size_t w = c->m.rows[0].size();
    for (size_t q = 0; q < w; ++q) {
      m_rows[q] = c->m.rows[0][q];
      m_rows[w + q] = c->m.rows[1][q];
    }
  });
}

// 2D Roe + viscous flux (flux.cpp:68-133 + solver.cpp:308-321), normal e_dir.
int ref_face_flux(double gamma, double R, double mu, double Pr, const double* um, const double* up, int dir,
                  double vg_n, const double* gm, const double* gp, double* out) {
  return guard([&] {
    GasModel gas{gamma, R, mu, Pr};
    const Vec2 normal = dir == 0 ? Vec2{1.0, 0.0} : Vec2{0.0, 1.0};
    const State a{um[0], um[1], um[2], um[3]}, b{up[0], up[1], up[2], up[3]};
    State f = roe_flux(a, b, normal, vg_n, gas);
    if (gas.viscous() && gm && gp) {
      const PrimGrad pgm{{gm[0], gm[1]}, {gm[2], gm[3]}, {gm[4], gm[5]}};
      const PrimGrad pgp{{gp[0], gp[1]}, {gp[2], gp[3]}, {gp[4], gp[5]}};
      const FluxPair fm = viscous_flux(a, pgm, gas);
      const FluxPair fp = viscous_flux(b, pgp, gas);
      for (int v = 0; v < kNumVars; ++v)
        f[v] -= 0.5 * ((fm.fx[v] + fp.fx[v]) * normal[0] + (fm.fy[v] + fp.fy[v]) * normal[1]);
    }
    for (int v = 0; v < 4; ++v) out[v] = f[v];
  });
}

}  // extern "C"
