// gpu_rank_solver.hpp — the reference-side binding of the B200 path.
//
// A maintainer drops this header into the reference's source tree
// (/root/reference/proj/src, next to solver.hpp) and links
// paper_2008_04356_b200/libsdg_gpu.so.  `sdg::gpu::GpuRankSolver` has the public
// surface of `sdg::RankSolver` (proj/src/solver.hpp:64-98) and the same
// constructor arguments (solver.hpp:66-67), so the runner (runner.cpp:33-55)
// and the tests (proj/tests/test_solver.cpp:28-48) switch by changing one
// type.  It is compiled against the reference's own headers by
// integration/Makefile and exercised by integration/facade_check.cpp.
//
// The reference is 2D; the device path is 3D.  A 2D problem is embedded as
// one periodic z layer of elements (nz = 1) with w = 0, which the device path
// reproduces on every z node layer (the embedding tests, tests/embed.py).  The
// facade converts fields between the reference layout U[e][i][j][4] (local
// element order of LocalDomain::elements) and the device layout
// U[e][i][j][k][5] (sdg_local_element_ids order).
//
// Errors: status codes are rethrown as the reference's ConfigError /
// InvalidStateError / ProtocolError (errors.hpp:9-21).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "errors.hpp"
#include "mesh.hpp"
#include "nodal_basis.hpp"
#include "partition.hpp"
#include "sdg_gpu.h"  // -I<repo>/include
#include "solver.hpp"
#include "transport.hpp"

namespace sdg::gpu {

inline void check(int code, const sdg_ctx* c) {
  if (code == SDG_OK) return;
  const std::string m = c ? sdg_last_error(c) : sdg_global_error();
  switch (code) {
    case SDG_ERR_CONFIG: throw ConfigError(m);
    case SDG_ERR_INVALID_STATE: throw InvalidStateError(m);
    case SDG_ERR_PROTOCOL: throw ProtocolError(m);
    default: throw std::runtime_error("device error: " + m);
  }
}

// MeshSpec (mesh.hpp:19-26) -> the 3D descriptor: one periodic z layer whose
// depth is the largest element size, so the time step (min of hx, hy;
// diagnostics.cpp:89-112) is unchanged.  Partition 0 is assign_ranks'
// (partition.cpp:17-83).
inline sdg_mesh_spec to_mesh_spec(const MeshSpec& s) {
  if (s.bands.empty() || s.bands.size() > SDG_MAX_BANDS) throw ConfigError("mesh needs 1..16 bands");
  sdg_mesh_spec m{};
  m.x0 = s.x0;
  m.y0 = s.y0;
  m.z0 = 0.0;
  m.width = s.width;
  m.height = s.height;
  m.ny = s.ny;
  m.nz = 1;
  m.n_bands = static_cast<int>(s.bands.size());
  double frac = 0.0, hmax = 0.0;
  for (const auto& b : s.bands) frac += b.width_frac;
  for (size_t b = 0; b < s.bands.size(); ++b) {
    m.bands[b].nx = s.bands[b].nx;
    m.bands[b].width_frac = s.bands[b].width_frac;
    m.bands[b].vg_y = s.bands[b].vg_y;
    m.bands[b].ny = s.bands[b].ny;  // 0: the mesh-wide ny, as BandSpec::ny
    m.bands[b].nz = 0;
    m.bands[b].vg_z = 0.0;
    const int ny = s.bands[b].ny > 0 ? s.bands[b].ny : s.ny;
    hmax = std::max({hmax, s.width * s.bands[b].width_frac / frac / s.bands[b].nx, s.height / ny});
  }
  m.depth = hmax;
  m.periodic_x = s.periodic_x ? 1 : 0;
  m.periodic_y = s.periodic_y ? 1 : 0;
  m.periodic_z = 1;
  m.partition = 0;
  m.mapping = SDG_MAP_BOX;
  m.warp = 0.0;
  return m;
}

// SolverConfig (solver.hpp) + NodeSet -> degree, nodes, gas and case.  The
// cases keep their 2D formulas (exact_solutions.cpp:7-35) with w = 0.
inline sdg_solver_config to_solver_config(const NodeSet& ns, const SolverConfig& cfg) {
  sdg_solver_config c{};
  c.degree = ns.degree();
  c.node_kind = ns.kind() == NodeKind::LegendreGauss ? SDG_NODES_GAUSS : SDG_NODES_LGL;
  c.gas = {cfg.gas.gamma, cfg.gas.R, cfg.gas.mu, cfg.gas.Pr};
  const CaseDef& k = cfg.flow_case;
  sdg_case& f = c.flow_case;
  switch (k.kind) {
    case CaseDef::Kind::Freestream:
      f.kind = SDG_CASE_FREESTREAM;
      f.fs_rho = k.fs.rho;
      f.fs_v[0] = k.fs.v[0];
      f.fs_v[1] = k.fs.v[1];
      f.fs_p = k.fs.p;
      break;
    case CaseDef::Kind::DensityWave:  // rho = 2 + alpha sin(pi (x + y - (a1 + a2) t))
      f.kind = SDG_CASE_DENSITY_WAVE;
      f.dw_alpha = k.dw.alpha;
      f.dw_a[0] = k.dw.a[0];
      f.dw_a[1] = k.dw.a[1];
      f.dw_k[0] = 1.0;
      f.dw_k[1] = 1.0;
      f.dw_p0 = k.dw.p0;
      break;
    case CaseDef::Kind::Vortex:
      f.kind = SDG_CASE_VORTEX;
      f.vx_eps = k.vx.eps;
      f.vx_rc = k.vx.rc;
      f.vx_rho_inf = k.vx.rho_inf;
      f.vx_v_inf = k.vx.v_inf;
      f.vx_theta = k.vx.theta;
      f.vx_ma_inf = k.vx.ma_inf;
      f.vx_center[0] = k.vx.center0[0];
      f.vx_center[1] = k.vx.center0[1];
      break;
  }
  return c;
}

// RankSolver's public surface on the device.
class GpuRankSolver {
 public:
  // Same arguments as RankSolver::RankSolver (solver.hpp:66-67), plus the
  // device.  Several ranks: one process (or host thread) per GPU; the NCCL
  // unique id travels through the reference transport's init-phase allgather
  // (transport.hpp:59-61), the one collective the audit allows.  `inproc_hub`
  // (optional) instead runs every rank of this process on one device through
  // the device path's in-process hub (InProcHub's analogue, transport.hpp:83-120).
  GpuRankSolver(const Mesh& mesh, const Ownership& own, LocalDomain dom, const NodeSet& ns,
                const BasisOperators& basis, const SolverConfig& cfg, Transport& transport, int device = -1,
                const char* inproc_hub = nullptr)
      : mesh_(&mesh), dom_(std::move(dom)), ns_(&ns), cfg_(cfg), transport_(&transport) {
    (void)basis;  // the device path builds its operators from the node set (nodal_basis.cpp:72-182)
    cfg.gas.validate();
    const sdg_mesh_spec ms = to_mesh_spec(mesh.spec());
    const sdg_solver_config sc = to_solver_config(ns, cfg);
    const int n_ranks = transport.size(), rank = transport.rank();
    if (own.n_ranks != n_ranks) throw ConfigError("ownership and transport disagree on the rank count");
    const int dev = device >= 0 ? device : (inproc_hub ? 0 : rank);
    if (n_ranks == 1) {
      check(sdg_create(&ms, &sc, 1, 0, dev, nullptr, &ctx_), nullptr);
    } else if (inproc_hub) {
      check(sdg_create_inproc(&ms, &sc, n_ranks, rank, dev, inproc_hub, &ctx_), nullptr);
    } else {
      constexpr int kWords = SDG_NCCL_ID_BYTES / sizeof(double);
      std::vector<double> mine;
      if (rank == 0) {
        char id[SDG_NCCL_ID_BYTES];
        check(sdg_nccl_unique_id(id), nullptr);
        mine.resize(kWords);
        std::memcpy(mine.data(), id, SDG_NCCL_ID_BYTES);
      }
      const auto all = transport.allgather(mine);
      if (all.empty() || all[0].size() != static_cast<size_t>(kWords)) throw ProtocolError("NCCL id exchange failed");
      check(sdg_create(&ms, &sc, n_ranks, rank, dev, all[0].data(), &ctx_), nullptr);
    }
    n1_ = sdg_n1(ctx_);
    // The device partition must be the reference's ownership; map local orders.
    std::vector<long> gids(sdg_n_local_elements(ctx_));
    sdg_local_element_ids(ctx_, gids.data());
    if (gids.size() != dom_.elements.size()) throw ConfigError("device partition differs from the ownership");
    std::unordered_map<long, int> ref_of;
    for (size_t q = 0; q < dom_.elements.size(); ++q) ref_of[dom_.elements[q].gid] = static_cast<int>(q);
    perm_.resize(gids.size());
    for (size_t q = 0; q < gids.size(); ++q) {
      const auto it = ref_of.find(gids[q]);
      if (it == ref_of.end()) throw ConfigError("device partition differs from the ownership");
      perm_[q] = it->second;
    }
    field_.assign(dom_.elements.size() * n1_ * n1_ * 4, 0.0);
    dev_.resize(dom_.elements.size() * static_cast<size_t>(n1_) * n1_ * n1_ * 5);
  }
  ~GpuRankSolver() { sdg_destroy(ctx_); }
  GpuRankSolver(const GpuRankSolver&) = delete;
  GpuRankSolver& operator=(const GpuRankSolver&) = delete;

  void init_rank_maps() { check(sdg_init_rank_maps(ctx_), ctx_); }
  void set_initial_condition(double t0) {
    check(sdg_set_initial_condition(ctx_, t0), ctx_);
    host_valid_ = dirty_ = false;
  }
  void step(double dt) {
    push();
    check(sdg_step(ctx_, dt), ctx_);
    host_valid_ = false;
  }
  // lsrk_step (lsrk.hpp:20-21) one stage at a time on the device.
  void rk_stage(int s, double t, double dt) {
    push();
    check(sdg_rk_stage(ctx_, s, t, dt), ctx_);
    if (s == 4) check(sdg_synchronize(ctx_), ctx_);
    host_valid_ = false;
  }
  // The private RankSolver::update_interfaces (solver.hpp:127), exported for
  // stage-by-stage checks: per side context the lower/upper forward and
  // backward operators (MortarOperators, mortar.hpp).
  std::vector<double> update_interfaces(double t_stage) {
    std::vector<double> ops(static_cast<size_t>(std::max(1, sdg_n_contexts(ctx_))) * 4 * n1_ * n1_);
    check(sdg_update_interfaces(ctx_, t_stage, ops.data()), ctx_);
    return ops;
  }

  double time() const {
    double t = 0.0;
    sdg_time(ctx_, &t, nullptr);
    return t;
  }
  int step_index() const {
    int s = 0;
    sdg_time(ctx_, nullptr, &s);
    return s;
  }
  const LocalDomain& domain() const { return dom_; }
  // field(): the reference layout, read back from the device on demand; the
  // mutable overload marks it for upload before the next device call.
  std::span<const double> field() const {
    pull();
    return field_;
  }
  std::span<double> field() {
    pull();
    dirty_ = true;
    return field_;
  }

  void compute_residual(double t_stage, std::span<const double> u, std::span<double> dudt) {
    if (u.size() != field_.size() || dudt.size() != field_.size()) throw ConfigError("compute_residual: size mismatch");
    push();
    to_device_layout(u, dev_);
    std::vector<double> r(dev_.size());
    check(sdg_compute_residual_host(ctx_, t_stage, dev_.data(), r.data()), ctx_);
    from_device_layout(r, dudt);
  }
  // BR1 gradients of (v1, v2, T), 6 per node, g[2c + dir] (solver.cpp:729-791).
  void compute_gradients(double t_stage, std::span<const double> u) {
    if (u.size() != field_.size()) throw ConfigError("compute_gradients: size mismatch");
    push();
    to_device_layout(u, dev_);
    const size_t nodes = dev_.size() / 5;
    std::vector<double> g3(nodes * SDG_NGRAD);
    check(sdg_compute_gradients_host(ctx_, t_stage, dev_.data(), g3.data()), ctx_);
    const int n = n1_;
    grad_.assign(dom_.elements.size() * n * n * 6, 0.0);
    const int q_of[3] = {0, 1, 3};  // (v1, v2, T) among the device's (v1, v2, v3, T)
    for (size_t q = 0; q < perm_.size(); ++q)
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          const double* s = g3.data() + (((q * n + i) * n + j) * n) * SDG_NGRAD;  // z node 0
          double* d = grad_.data() + ((static_cast<size_t>(perm_[q]) * n + i) * n + j) * 6;
          for (int c = 0; c < 3; ++c)
            for (int dir = 0; dir < 2; ++dir) d[2 * c + dir] = s[3 * q_of[c] + dir];
        }
  }
  std::span<const double> gradients() const { return grad_; }

  double suggest_dt(double cfl) const {
    const_cast<GpuRankSolver*>(this)->push();
    double dt = 0.0;
    check(sdg_suggest_dt(ctx_, cfl, &dt), ctx_);
    return dt;
  }
  long total_rebuilds() const { return sdg_total_rebuilds(ctx_); }
  void inject_collective() { check(sdg_inject_collective(ctx_), ctx_); }
  sdg_ctx* handle() const { return ctx_; }

 private:
  void pull() const {
    if (host_valid_ || dirty_) return;
    check(sdg_get_state(ctx_, dev_.data()), ctx_);
    from_device_layout(dev_, field_);
    host_valid_ = true;
  }
  void push() {
    if (!dirty_) return;
    to_device_layout(field_, dev_);
    check(sdg_set_state(ctx_, dev_.data()), ctx_);
    dirty_ = false;
    host_valid_ = true;
  }
  // 2D (rho, rho v1, rho v2, rho E) -> 3D (rho, rho v1, rho v2, 0, rho E) on every z node.
  void to_device_layout(std::span<const double> u2, std::vector<double>& u3) const {
    const int n = n1_;
    for (size_t q = 0; q < perm_.size(); ++q)
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          const double* s = u2.data() + ((static_cast<size_t>(perm_[q]) * n + i) * n + j) * 4;
          for (int k = 0; k < n; ++k) {
            double* d = u3.data() + (((q * n + i) * n + j) * n + k) * 5;
            d[0] = s[0];
            d[1] = s[1];
            d[2] = s[2];
            d[3] = 0.0;
            d[4] = s[3];
          }
        }
  }
  // 3D -> 2D from the first z node layer (all layers agree to rounding).
  void from_device_layout(const std::vector<double>& u3, std::span<double> u2) const {
    const int n = n1_;
    for (size_t q = 0; q < perm_.size(); ++q)
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          const double* s = u3.data() + (((q * n + i) * n + j) * n) * 5;
          double* d = u2.data() + ((static_cast<size_t>(perm_[q]) * n + i) * n + j) * 4;
          d[0] = s[0];
          d[1] = s[1];
          d[2] = s[2];
          d[3] = s[4];
        }
  }

  const Mesh* mesh_;
  LocalDomain dom_;
  const NodeSet* ns_;
  SolverConfig cfg_;
  Transport* transport_;
  sdg_ctx* ctx_ = nullptr;
  int n1_ = 0;
  std::vector<int> perm_;  // device local element q -> reference local element
  mutable std::vector<double> field_, dev_;
  std::vector<double> grad_;
  mutable bool host_valid_ = false;
  bool dirty_ = false;
};

}  // namespace sdg::gpu
