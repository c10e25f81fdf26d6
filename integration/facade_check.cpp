// facade_check — TEST INFRASTRUCTURE for integration/gpu_rank_solver.hpp.
//
// Built by integration/Makefile against the UNMODIFIED reference sources
// (their headers, and their objects compiled by oracle/Makefile into
// oracle/_ref) plus the product's libsdg_gpu.so: the reference's own
// RankSolver and the device path behind the facade run side by side in one
// program on the same reference setup objects.
//
//   facade_check spec   no GPU: prints the descriptors the facade derives from
//                       reference MeshSpec / SolverConfig objects (JSON lines)
//   facade_check run    GPU: reference RankSolver vs facade on 2D cases:
//                       residual, gradients, dt, 10 steps, rk_stage, operators,
//                       rebuild counts, a 2-rank run; exit code 0 iff all pass
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "gpu_rank_solver.hpp"
#include "lsrk.hpp"

using namespace sdg;

namespace {

MeshSpec three_band(int nx, int ny, double vg, bool periodic_x = true) {
  MeshSpec s;
  s.width = 2.0;
  s.height = 2.0;
  s.ny = ny;
  s.bands = {{nx, 1.0, 0.0}, {nx, 1.0, vg}, {nx, 1.0, 0.0}};
  s.periodic_x = periodic_x;
  return s;
}

MeshSpec box0_2d(int n) {  // BASELINE configs[0] 2D analog
  MeshSpec s;
  s.width = 2.0;
  s.height = 2.0;
  s.ny = n;
  s.bands = {{n, 1.0, 0.0}, {n, 1.0, 0.5}};
  s.periodic_x = false;
  return s;
}

SolverConfig density_wave(double mu) {
  SolverConfig c;
  c.gas.R = 1.0;
  c.gas.mu = mu;
  c.flow_case.kind = CaseDef::Kind::DensityWave;
  c.flow_case.dw = {0.1, {1.0, 1.0}, 1.0};
  return c;
}

SolverConfig vortex() {
  SolverConfig c;
  c.gas.R = 1.0;
  c.flow_case.kind = CaseDef::Kind::Vortex;
  return c;
}

void print_spec(const char* name, const sdg_mesh_spec& m, const sdg_solver_config& c) {
  std::printf("{\"name\": \"%s\", \"x0\": %.17g, \"y0\": %.17g, \"width\": %.17g, \"height\": %.17g, \"depth\": %.17g, "
              "\"ny\": %d, \"nz\": %d, \"n_bands\": %d, \"bands\": [",
              name, m.x0, m.y0, m.width, m.height, m.depth, m.ny, m.nz, m.n_bands);
  for (int b = 0; b < m.n_bands; ++b)
    std::printf("%s[%d, %.17g, %.17g, %d, %d, %.17g]", b ? ", " : "", m.bands[b].nx, m.bands[b].width_frac,
                m.bands[b].vg_y, m.bands[b].ny, m.bands[b].nz, m.bands[b].vg_z);
  std::printf("], \"periodic\": [%d, %d, %d], \"partition\": %d, \"mapping\": %d, \"degree\": %d, \"node_kind\": %d, "
              "\"gas\": [%.17g, %.17g, %.17g, %.17g], \"case\": %d, \"dw\": [%.17g, %.17g, %.17g, %.17g, %.17g, %.17g], "
              "\"vx\": [%.17g, %.17g, %.17g, %.17g, %.17g, %.17g, %.17g, %.17g]}\n",
              m.periodic_x, m.periodic_y, m.periodic_z, m.partition, m.mapping, c.degree, c.node_kind, c.gas.gamma,
              c.gas.R, c.gas.mu, c.gas.Pr, c.flow_case.kind, c.flow_case.dw_alpha, c.flow_case.dw_a[0],
              c.flow_case.dw_a[1], c.flow_case.dw_k[0], c.flow_case.dw_k[1], c.flow_case.dw_p0, c.flow_case.vx_eps,
              c.flow_case.vx_rc, c.flow_case.vx_rho_inf, c.flow_case.vx_v_inf, c.flow_case.vx_theta,
              c.flow_case.vx_ma_inf, c.flow_case.vx_center[0], c.flow_case.vx_center[1]);
}

int spec_mode() {
  MeshSpec a = three_band(2, 6, 1.0);
  a.bands[1].ny = 0;
  print_spec("three_band", gpu::to_mesh_spec(a), gpu::to_solver_config(NodeSet(3, NodeKind::LegendreGauss), density_wave(1e-3)));
  print_spec("box0", gpu::to_mesh_spec(box0_2d(4)), gpu::to_solver_config(NodeSet(5, NodeKind::LegendreGaussLobatto), vortex()));
  return 0;
}

double rel_linf(std::span<const double> a, std::span<const double> b) {
  double d = 0.0, s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    d = std::max(d, std::abs(a[i] - b[i]));
    s = std::max(s, std::abs(b[i]));
  }
  return d / std::max(s, 1e-300);
}

// The reference's single-rank setup (proj/tests/test_solver.cpp:28-48) and the
// facade built from the same Mesh / NodeSet / BasisOperators / Ownership.
struct Pair {
  Mesh mesh;
  NodeSet ns;
  BasisOperators basis;
  Ownership own;
  InProcHub hub_ref, hub_gpu;
  InProcTransport tr_ref, tr_gpu;
  RankSolver ref;
  gpu::GpuRankSolver dev;
  Pair(const MeshSpec& spec, int degree, NodeKind kind, const SolverConfig& cfg)
      : mesh(spec), ns(degree, kind), basis(build_basis_operators(ns)), own(assign_ranks(mesh, 1)), hub_ref(1),
        hub_gpu(1), tr_ref(hub_ref, 0), tr_gpu(hub_gpu, 0),
        ref(mesh, own, build_local_domain(mesh, own, 0), ns, basis, cfg, tr_ref),
        dev(mesh, own, build_local_domain(mesh, own, 0), ns, basis, cfg, tr_gpu, 0) {
    ref.init_rank_maps();
    dev.init_rank_maps();
  }
};

int failures = 0;
void expect(bool ok, const std::string& what, double v) {
  std::printf("%s %s (%.3e)\n", ok ? "PASS" : "FAIL", what.c_str(), v);
  if (!ok) ++failures;
}

void run_case(const char* name, const MeshSpec& spec, int degree, NodeKind kind, const SolverConfig& cfg) {
  const std::string tag = std::string(name) + ": ";
  {  // residual and gradients at three stage times
    Pair p(spec, degree, kind, cfg);
    p.ref.set_initial_condition(0.0);
    p.dev.set_initial_condition(0.0);
    expect(rel_linf(p.dev.field(), p.ref.field()) <= 1e-15, tag + "initial condition", rel_linf(p.dev.field(), p.ref.field()));
    const std::vector<double> u(p.ref.field().begin(), p.ref.field().end());
    for (double t : {0.0, 0.05, 0.37}) {
      std::vector<double> r0(u.size()), r1(u.size());
      p.ref.compute_residual(t, u, r0);
      p.dev.compute_residual(t, u, r1);
      double scale = 1.0;
      for (double v : r0) scale = std::max(scale, std::abs(v));
      double d = 0.0;
      for (size_t i = 0; i < u.size(); ++i) d = std::max(d, std::abs(r0[i] - r1[i]));
      expect(d <= 1e-12 * scale, tag + "residual t=" + std::to_string(t), d / scale);
      if (cfg.gas.viscous()) {
        p.ref.compute_gradients(t, u);
        p.dev.compute_gradients(t, u);
        double gs = 1.0, gd = 0.0;
        for (size_t i = 0; i < p.ref.gradients().size(); ++i) {
          gs = std::max(gs, std::abs(p.ref.gradients()[i]));
          gd = std::max(gd, std::abs(p.ref.gradients()[i] - p.dev.gradients()[i]));
        }
        expect(gd <= 1e-11 * gs, tag + "gradients t=" + std::to_string(t), gd / gs);
      }
    }
  }
  {  // dt and 10 RK steps, rebuild counts
    Pair p(spec, degree, kind, cfg);
    p.ref.set_initial_condition(0.0);
    p.dev.set_initial_condition(0.0);
    const double dt = p.ref.suggest_dt(0.5);
    const double dg = p.dev.suggest_dt(0.5);
    expect(std::abs(dt - dg) <= 1e-14 * dt, tag + "suggest_dt", std::abs(dt - dg) / dt);
    for (int s = 0; s < 10; ++s) {
      p.ref.step(dt);
      p.dev.step(dt);
    }
    expect(rel_linf(p.dev.field(), p.ref.field()) <= 1e-12, tag + "10 steps", rel_linf(p.dev.field(), p.ref.field()));
    expect(p.dev.total_rebuilds() == p.ref.total_rebuilds(), tag + "rebuild count " + std::to_string(p.ref.total_rebuilds()),
           static_cast<double>(p.dev.total_rebuilds() - p.ref.total_rebuilds()));
    expect(p.dev.time() == p.ref.time() && p.dev.step_index() == p.ref.step_index(), tag + "time / step index", 0.0);
  }
  {  // lsrk_step with the reference's residual vs five device rk_stage calls
    Pair p(spec, degree, kind, cfg);
    p.ref.set_initial_condition(0.0);
    p.dev.set_initial_condition(0.0);
    const double dt = p.ref.suggest_dt(0.5);
    std::vector<double> u(p.ref.field().begin(), p.ref.field().end()), reg(u.size(), 0.0);
    for (int k = 0; k < 3; ++k) {
      const double t = p.dev.time();
      lsrk_step(u, reg, t, dt, [&](double ts, std::span<const double> uu, std::span<double> du) {
        p.ref.compute_residual(ts, uu, du);
      });
      for (int s = 0; s < 5; ++s) p.dev.rk_stage(s, t, dt);
    }
    expect(rel_linf(p.dev.field(), u) <= 1e-12, tag + "rk_stage x15 vs lsrk_step(RankSolver::compute_residual) x3",
           rel_linf(p.dev.field(), u));
    Pair q(spec, degree, kind, cfg);
    q.ref.set_initial_condition(0.0);
    for (int k = 0; k < 3; ++k) q.ref.step(dt);
    expect(rel_linf(p.dev.field(), q.ref.field()) <= 1e-12, tag + "rk_stage x15 vs RankSolver::step x3",
           rel_linf(p.dev.field(), q.ref.field()));
  }
  {  // update_interfaces: operators equal the reference's bits
    Pair p(spec, degree, kind, cfg);
    p.ref.set_initial_condition(0.0);
    p.dev.set_initial_condition(0.0);
    const std::vector<double> u(p.ref.field().begin(), p.ref.field().end());
    std::vector<double> r(u.size());
    const double t = 0.37;
    p.ref.compute_residual(t, u, r);  // runs the reference's update_interfaces(t)
    const std::vector<double> ops = p.dev.update_interfaces(t);
    const int n = degree + 1, nc = sdg_n_contexts(p.dev.handle());
    bool same = true;
    int compared = 0;
    for (int c = 0; c < nc; ++c) {
      long info[5];
      double sd, sig;
      gpu::check(sdg_ctx_info(p.dev.handle(), c, info, &sd, &sig), p.dev.handle());
      const InterfaceSideCtx* rc = p.ref.side_ctx(static_cast<int>(info[0]), info[1] != 0);
      if (rc == nullptr) {
        same = false;
        continue;
      }
      same = same && rc->st.n_delta == info[2] && rc->conforming == (info[3] != 0) && rc->st.s_delta == sd &&
             rc->sigma_side == sig;
      if (rc->conforming) continue;
      for (int h = 0; h < 2; ++h) {
        same = same && std::memcmp(rc->ops.to_mortar[h].data(), ops.data() + (c * 4 + h) * n * n, sizeof(double) * n * n) == 0;
        same = same && std::memcmp(rc->ops.to_face[h].data(), ops.data() + (c * 4 + 2 + h) * n * n, sizeof(double) * n * n) == 0;
      }
      ++compared;
    }
    expect(same && (compared > 0 || nc == 0), tag + "update_interfaces: state and operators bit-exact (" +
           std::to_string(compared) + " contexts)", same ? 0.0 : 1.0);
  }
}

// Two ranks of the reference (threads, InProcHub) against two facade ranks on
// one device (the device path's in-process hub): fields agree rank by rank.
void run_two_ranks() {
  const MeshSpec spec = three_band(2, 6, 1.0);
  const SolverConfig cfg = density_wave(1e-3);
  Mesh mesh(spec);
  NodeSet ns(3, NodeKind::LegendreGauss);
  BasisOperators basis = build_basis_operators(ns);
  Ownership own = assign_ranks(mesh, 2);
  InProcHub hr(2), hg(2);
  std::vector<double> err(2, 1.0);
  std::vector<std::string> msg(2);
  auto worker = [&](int r) {
    try {
      InProcTransport tr(hr, r), tg(hg, r);
      RankSolver ref(mesh, own, build_local_domain(mesh, own, r), ns, basis, cfg, tr);
      gpu::GpuRankSolver dev(mesh, own, build_local_domain(mesh, own, r), ns, basis, cfg, tg, 0, "facade2");
      ref.init_rank_maps();
      dev.init_rank_maps();
      ref.set_initial_condition(0.0);
      dev.set_initial_condition(0.0);
      for (int s = 0; s < 5; ++s) {
        ref.step(0.004);
        dev.step(0.004);
      }
      err[r] = rel_linf(dev.field(), ref.field());
    } catch (const std::exception& e) {
      msg[r] = e.what();
    }
  };
  std::thread a(worker, 0), b(worker, 1);
  a.join();
  b.join();
  for (int r = 0; r < 2; ++r)
    expect(err[r] <= 1e-12, "two ranks: rank " + std::to_string(r) + " after 5 steps" + (msg[r].empty() ? "" : " [" + msg[r] + "]"),
           err[r]);
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "";
  if (mode == "spec") return spec_mode();
  if (mode != "run") {
    std::fprintf(stderr, "usage: facade_check spec|run\n");
    return 2;
  }
  try {
    run_case("three bands, Gauss N=3, viscous", three_band(2, 6, 1.0), 3, NodeKind::LegendreGauss, density_wave(1e-3));
    run_case("three bands, LGL N=4, inviscid", three_band(2, 6, 1.0), 4, NodeKind::LegendreGaussLobatto, density_wave(0.0));
    run_case("configs[0] 2D analog, Gauss N=3, viscous, Dirichlet x", box0_2d(4), 3, NodeKind::LegendreGauss, density_wave(1e-3));
    run_case("vortex, static mesh, Gauss N=5", three_band(3, 6, 0.0), 5, NodeKind::LegendreGauss, vortex());
    run_two_ranks();
    // Error mapping: an inadmissible state raises the reference's InvalidStateError.
    Pair p(three_band(2, 3, 1.0), 2, NodeKind::LegendreGaussLobatto, density_wave(0.0));
    p.dev.set_initial_condition(0.0);
    p.dev.field()[0] = -1.0;
    bool thrown = false;
    try {
      p.dev.step(1e-6);
    } catch (const InvalidStateError&) {
      thrown = true;
    }
    expect(thrown, "inadmissible state raises sdg::InvalidStateError", thrown ? 0.0 : 1.0);
  } catch (const std::exception& e) {
    std::printf("FAIL exception: %s\n", e.what());
    return 1;
  }
  std::printf("%s: %d failures\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
