// GpuRankSolver: the per-rank, per-GPU context behind the C-ABI.
//
// Mirrors the public surface of sdg::RankSolver (/root/reference/proj/src/solver.hpp:64-98):
// construction from mesh / partition / basis / gas / case, the one init-time
// rank-map exchange, initial condition, step, compute_residual,
// compute_gradients, suggest_dt, side_ctx and total_rebuilds.  Fields live on
// the device for the lifetime of the context; every stage is a fixed sequence
// of kernel launches on one stream.
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <deque>
#include <functional>
#include <map>
#include <mutex>
#include <memory>
#include <sstream>
#include <tuple>
#include <string>
#include <vector>

#include "../../include/sdg_gpu.h"
#include "kernels.cuh"

namespace sdg {

namespace {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(SDG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw DeviceError(SDG_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void alloc(size_t count) {
    if (p) cudaFree(p);
    p = nullptr;
    n = count;
    if (count) cuda_check(cudaMalloc(&p, count * sizeof(T)), "cudaMalloc");
  }
  void upload(const std::vector<T>& v, cudaStream_t st) {
    alloc(v.size());
    if (!v.empty()) cuda_check(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st), "upload");
  }
  void zero(cudaStream_t st) {
    if (n) cuda_check(cudaMemsetAsync(p, 0, n * sizeof(T), st), "memset");
  }
};


// ----------------------------------------------------------------------------
// Rank-to-rank transport behind one interface (the reference's Transport,
// transport.hpp:43-80): NCCL over NVLink between processes / GPUs, or an
// in-process hub for several ranks sharing one GPU (the analogue of the
// reference's InProcHub, used to exercise the multi-rank data path on a single
// device).  Every rank issues the same sequence of calls.
// ----------------------------------------------------------------------------
struct Xfer {
  int partner;
  double* ptr;  // send: source, recv: destination (device)
  size_t count;
};

struct Comm {
  virtual ~Comm() = default;
  virtual void allgather_ints(const std::vector<int>& mine, std::vector<std::vector<int>>& all, cudaStream_t st) = 0;
  // One grouped round: all sends and receives of this rank.
  virtual void exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, cudaStream_t st) = 0;
  // op: 0 sum, 1 max, 2 min (host values, every rank gets the result).
  virtual void allreduce(double* vals, int n, int op, cudaStream_t st) = 0;
};

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  int n_ranks;
  NcclComm(const void* id_bytes, int n, int rank) : n_ranks(n) {
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, sizeof(id));
    nccl_check(ncclCommInitRank(&comm, n, id, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm) ncclCommDestroy(comm);
  }
  void allgather_ints(const std::vector<int>& mine, std::vector<std::vector<int>>& all, cudaStream_t st) override {
    DevBuf<int> d_cnt, d_all_cnt;
    d_cnt.alloc(1);
    d_all_cnt.alloc(n_ranks);
    const int cnt = static_cast<int>(mine.size());
    cuda_check(cudaMemcpyAsync(d_cnt.p, &cnt, sizeof(int), cudaMemcpyHostToDevice, st), "h2d");
    nccl_check(ncclAllGather(d_cnt.p, d_all_cnt.p, 1, ncclInt32, comm, st), "allgather sizes");
    std::vector<int> counts(n_ranks);
    cuda_check(cudaMemcpyAsync(counts.data(), d_all_cnt.p, n_ranks * sizeof(int), cudaMemcpyDeviceToHost, st), "d2h");
    cuda_check(cudaStreamSynchronize(st), "sync");
    const int mx = std::max(1, *std::max_element(counts.begin(), counts.end()));
    std::vector<int> padded(mx, 0);
    std::copy(mine.begin(), mine.end(), padded.begin());
    DevBuf<int> d_mine, d_all;
    d_mine.upload(padded, st);
    d_all.alloc(static_cast<size_t>(mx) * n_ranks);
    nccl_check(ncclAllGather(d_mine.p, d_all.p, mx, ncclInt32, comm, st), "allgather maps");
    std::vector<int> h(static_cast<size_t>(mx) * n_ranks);
    cuda_check(cudaMemcpyAsync(h.data(), d_all.p, h.size() * sizeof(int), cudaMemcpyDeviceToHost, st), "d2h");
    cuda_check(cudaStreamSynchronize(st), "sync");
    all.assign(n_ranks, {});
    for (int r = 0; r < n_ranks; ++r) all[r].assign(h.begin() + r * mx, h.begin() + r * mx + counts[r]);
  }
  void exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, cudaStream_t st) override {
    if (sends.empty() && recvs.empty()) return;
    nccl_check(ncclGroupStart(), "group start");
    for (const auto& x : sends) nccl_check(ncclSend(x.ptr, x.count, ncclFloat64, x.partner, comm, st), "send");
    for (const auto& x : recvs) nccl_check(ncclRecv(x.ptr, x.count, ncclFloat64, x.partner, comm, st), "recv");
    nccl_check(ncclGroupEnd(), "group end");
  }
  void allreduce(double* vals, int n, int op, cudaStream_t st) override {
    DevBuf<double> d;
    d.alloc(n);
    cuda_check(cudaMemcpyAsync(d.p, vals, n * sizeof(double), cudaMemcpyHostToDevice, st), "h2d");
    const ncclRedOp_t o = op == 0 ? ncclSum : (op == 1 ? ncclMax : ncclMin);
    nccl_check(ncclAllReduce(d.p, d.p, n, ncclFloat64, o, comm, st), "allreduce");
    cuda_check(cudaMemcpyAsync(vals, d.p, n * sizeof(double), cudaMemcpyDeviceToHost, st), "d2h");
    cuda_check(cudaStreamSynchronize(st), "sync");
  }
};

struct InProcHub {
  int n;
  std::mutex mu;
  std::condition_variable cv;
  long gen = 0;
  int arrived = 0;
  struct Msg {
    const double* ptr;
    size_t count;
    cudaEvent_t ready;
  };
  std::vector<std::deque<Msg>> box;  // n*n channels (src*n + dst), FIFO as transport.cpp:46-75
  std::vector<std::vector<int>> ints;
  std::vector<std::vector<double>> vals;
  explicit InProcHub(int n_) : n(n_), box(static_cast<size_t>(n_) * n_), ints(n_), vals(n_) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

std::mutex g_hubs_mu;
std::map<std::string, std::weak_ptr<InProcHub>> g_hubs;

struct InProcComm : Comm {
  std::shared_ptr<InProcHub> hub;
  int rank;
  cudaEvent_t ev = nullptr;
  InProcComm(const std::string& name, int n, int r) : rank(r) {
    std::lock_guard<std::mutex> lk(g_hubs_mu);
    auto& w = g_hubs[name];
    hub = w.lock();
    if (!hub) {
      hub = std::make_shared<InProcHub>(n);
      w = hub;
    }
    if (hub->n != n) throw ConfigError("in-process hub rank count mismatch");
    cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
  }
  ~InProcComm() override {
    if (ev) cudaEventDestroy(ev);
  }
  void allgather_ints(const std::vector<int>& mine, std::vector<std::vector<int>>& all, cudaStream_t) override {
    {
      std::lock_guard<std::mutex> lk(hub->mu);
      hub->ints[rank] = mine;
    }
    hub->barrier();
    {
      std::lock_guard<std::mutex> lk(hub->mu);
      all = hub->ints;
    }
    hub->barrier();
  }
  void exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, cudaStream_t st) override {
    cuda_check(cudaEventRecord(ev, st), "event record");
    {
      std::lock_guard<std::mutex> lk(hub->mu);
      for (const auto& x : sends) hub->box[static_cast<size_t>(rank) * hub->n + x.partner].push_back({x.ptr, x.count, ev});
    }
    hub->barrier();
    for (const auto& x : recvs) {
      InProcHub::Msg m;
      {
        std::lock_guard<std::mutex> lk(hub->mu);
        auto& q = hub->box[static_cast<size_t>(x.partner) * hub->n + rank];
        if (q.empty()) throw ProtocolError("in-process receive without a matching send");
        m = q.front();
        q.pop_front();
      }
      if (m.count != x.count) throw ProtocolError("message length mismatch");
      cuda_check(cudaStreamWaitEvent(st, m.ready, 0), "wait event");
      cuda_check(cudaMemcpyAsync(x.ptr, m.ptr, x.count * sizeof(double), cudaMemcpyDeviceToDevice, st), "d2d");
    }
    // Senders may reuse their buffers only after every receiver has copied.
    cuda_check(cudaStreamSynchronize(st), "sync");
    hub->barrier();
  }
  void allreduce(double* v, int n, int op, cudaStream_t) override {
    {
      std::lock_guard<std::mutex> lk(hub->mu);
      hub->vals[rank].assign(v, v + n);
    }
    hub->barrier();
    {
      std::lock_guard<std::mutex> lk(hub->mu);
      for (int q = 0; q < n; ++q) {
        double a = hub->vals[0][q];
        for (int r = 1; r < hub->n; ++r) {
          const double b = hub->vals[r][q];
          a = op == 0 ? a + b : (op == 1 ? std::max(a, b) : std::min(a, b));
        }
        v[q] = a;
      }
    }
    hub->barrier();
  }
};

// Carpenter-Kennedy 5-stage 2N-storage RK4 (proj/src/lsrk.cpp:7-29).
const double RK_A[5] = {0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
                        -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0};
const double RK_B[5] = {1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
                        1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
                        2277821191437.0 / 14882151754819.0};
const double RK_C[5] = {0.0, 1432997174477.0 / 9575080441755.0, 2526269341429.0 / 6820363962896.0,
                        2006345519317.0 / 3224310063776.0, 2802321613138.0 / 2924317926251.0};

// Interface-side context on the host (InterfaceSideCtx, solver.hpp:16-42).
struct SideCtx {
  int iface = 0;
  bool on_static = true;
  std::vector<int> slides;  // compact sliding indices, sorted by (i_par, i_perp)
  std::vector<int> static_map, moving_map;  // rank maps (r, r~), n_perp x n_par
  double delta_base = 0.0;
  long wraps = 0;  // periods subtracted from delta_base (annulus sector windings)
  long wind = 0;   // windings at the stage: displacement = d + wind * period
  Displacement st;
  double sigma_side = -1.0;
  bool conforming = true;
  long last_n = -1;
  bool last_conf = true, topo_valid = false;
  long rebuilds = 0;
  double ops_sigma = 2.0;  // sigma the cached operators were built for
  std::vector<double> fwd, bwd;
  // per-partner mortar counts of this side (for the NCCL blocks)
};

// Message kinds of the trace (transport.hpp:13-24; this protocol sends Fv.n
// instead of the primary's LiftConf / FluxConf replies).
enum MsgKind { MK_INIT = 1, MK_SOL_CONF = 2, MK_SOL_MORTAR = 3, MK_LIFT_MORTAR = 5, MK_FVN_CONF = 6,
               MK_GRAD_MORTAR = 7, MK_FLUX_MORTAR = 9, MK_DIAG = 10 };
const char* kKernelClasses[] = {"prolong", "pairing", "mortar", "gradient", "update", "copy", "halo"};
enum KClass { KC_PROLONG, KC_PAIRING, KC_MORTAR, KC_GRADIENT, KC_UPDATE, KC_COPY, KC_HALO, KC_N };

}  // namespace

class GpuRankSolver {
 public:
  GpuRankSolver(const sdg_mesh_spec& ms, const sdg_solver_config& cfg, int n_ranks, int rank, int device,
                const void* nccl_id, const char* inproc_hub = nullptr);
  ~GpuRankSolver();

  void init_rank_maps();
  void set_initial_condition(double t0);
  void set_state(const double* h);
  void get_state(double* h);
  void get_register(double* h);
  void steps(double dt, int n, bool sync);
  void rk_stage(int s, double t, double dt);
  void update_interfaces(double t_stage, double* ops);
  void synchronize();
  void compute_residual(double t_stage, const double* d_u, double* d_dudt);
  void compute_gradients(double t_stage, const double* d_u, double* d_grad);
  double suggest_dt(double cfl);
  void diagnostics(double t, int with_exact, double* out);
  void write_snapshot(const char* path, double time);
  double read_snapshot(const char* path);
  long total_rebuilds() const {
    long t = 0;
    for (const auto& s : sides_) t += s.rebuilds;
    return t;
  }
  void ctx_info(int c, long* out5, double* sd, double* sig);
  void nc_rows(int i, int dir, long* n_out, long* faces, double* ranges, double* delta);
  int n_nc() const { return static_cast<int>(nc_.size()); }
  void get_pairing(int role, int* ncols, int* cols);
  void get_mapping(int c, int* m);

  int n1() const { return n_; }
  int device() const { return device_; }
  long n_local() const { return E_; }
  long n_global() const { return mesh_.n_elements; }
  const std::vector<long>& gids() const { return topo_.gids; }
  int n_contexts() const { return static_cast<int>(sides_.size()); }
  double time() const { return time_; }
  int step_index() const { return step_index_; }
  double* d_state() { return U_.p; }
  cudaStream_t stream() const { return stream_; }
  long launches() const { return launches_; }
  void enable_timing(bool on) { timing_ = on; }
  std::vector<std::pair<double, long>> timing_totals();

  std::string err;
  std::string trace_json() const;
  void inject_collective();

 private:
  struct TraceRow {
    int step, stage, src, dst;
    long long count;
    int kind;
    bool is_send;
  };
  std::vector<TraceRow> comm_trace_;
  void record(int kind, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs);
  void build_consts();
  void build_sides();
  void upload_topology();
  void stage(double t_stage, int mode, double rk_a, double rk_b, double dt, double* out, const double* u_override);
  void update_interfaces_host(double t_stage);
  void run_pairing(double t_stage);
  void mortar_exchange(double* const src[2], double* dst_static, int ncomp, bool moving_to_static, int kind);
  void halo_exchange(double* arr, int ncomp, int kind, const std::function<void()>& overlap_work = {});
  void comm_round(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, bool join,
                  const std::function<void()>& overlap_work = {});
  void join_comm();
  void element_kernel(bool update, const FieldPtrs& fp, const StageArgs& a, int e_first, int e_end, int n_sm);
  StageArgs stage_args(double t_stage, double dt, double rk_a, double rk_b, int mode) const;
  void find_interior_run();
  FieldPtrs field_ptrs(double* U, double* out);
  MortarPtrs mortar_ptrs();
  void check_error();
  void mark(int cls, bool begin);
  void reset_clock(double t0);
  void snapshot_barrier(double& flag);

  MeshGeom mesh_;
  Partition part_;
  LocalTopology topo_;
  Basis basis_;
  sdg_solver_config cfg_;
  ElemConsts consts_{};
  int n_ = 0, n2_ = 0, n3_ = 0;
  int E_ = 0, S_ = 0, ND_ = 0;
  int rank_ = 0, n_ranks_ = 1, device_ = 0;
  bool lifting_ = false;
  cudaStream_t stream_ = nullptr;
  std::unique_ptr<Comm> comm_;
  // Exchange overlap: every comm round runs on comm_stream_ in issue order; the
  // conforming halo rounds are joined only after the element kernel has processed the
  // interior run [int_lo_, int_hi_) (elements with no remote or sliding side).
  cudaStream_t comm_stream_ = nullptr;
  cudaEvent_t ev_ready_ = nullptr, ev_comm_ = nullptr;
  int int_lo_ = 0, int_hi_ = 0;
  bool overlap_ = false;
  int sm_reserve_ = 0;  // SMs left free for the NCCL kernels while the interior run computes

  DevBuf<double> U_, reg_, dudt_, trace_[2], fvn_, slide_lift_, slide_flux_, slide_g_, dir_g_, grad_, visc_;
  // Curved elements (SDG_MAP_WARP): per-node metrics and per-side face metrics (host.cpp compute_metrics).
  bool curved_ = false;
  DevBuf<double> met_, fmet_;
  DevBuf<int8_t> side_type_, side_rot_;
  DevBuf<int> side_idx_, coords_, side_code_;
  int n_sm_ = 148;
  DevBuf<ErrRec> err_;
  ErrRec* err_host_ = nullptr;
  DevBuf<unsigned long long> dt_min_;
  DevBuf<double> diag_partial_;
  DevBuf<double> send_buf_;
  DevBuf<int> send_slots_;

  // mortar / pairing
  std::vector<SideCtx> sides_;
  std::vector<int> role_ids_[2];
  PairingArgs pargs_{};
  DevBuf<int> face_par_, face_perp_, face_slide_, partner_map_, pres_[2], payload_[2], cols_[2], m_, ctx_state_,
      n_mortars_;
  DevBuf<double> ctx_sdelta_;
  DevBuf<int> slide_elem_, slide_side_, slide_ctx_, slide_f_, ctx_face_off_, ctx_nf_, ctx_role_, ctx_static_left_;
  DevBuf<double> u_mine_[2], u_theirs_, mlift_[2], g_mine_[2], g_theirs_, mflux_[2];
  int max_mortars_[2] = {0, 0};
  int expect_mortars_[2] = {0, 0};
  MortarOps fwd_ops_{}, bwd_ops_{};
  // per role: mortar blocks per partner (partner, offset, count) + self
  std::vector<std::array<int, 3>> sched_[2];
  std::array<int, 3> self_[2] = {{0, 0, 0}, {0, 0, 0}};

  // Non-matching / oblique interfaces (BASELINE configs[1]; tensor-product mortars).
  struct NcRuntime {
    int iface = 0;                     // index into mesh_.nc_ifaces
    double dy_base = 0.0, dz_base = 0.0;  // relative displacement of side B at time_ (per step)
    double dy = 0.0, dz = 0.0;         // at the current stage
    long long max_m[2] = {0, 0};       // row capacity per direction
    DevBuf<int> slot[2], kidx[2];      // per side: face (fy * nfz + fz) -> trace slot / sliding index
    DevBuf<long long> d_faces[2], d_n;
    DevBuf<double> d_ranges[2];
    DevBuf<double> mu[2], mg[2], mlift, mflux;  // mortar data [M][n2][nc]
    NcStage S{};                       // tables of the current stage
    size_t blob_off = 0, blob_bytes = 0;  // this interface's part of the per-stage upload
  };
  std::vector<NcRuntime> nc_;
  DevBuf<unsigned char> nc_blob_;      // per-stage rows / operators / CSR of all NC interfaces
  std::vector<unsigned char*> nc_pinned_;  // pinned staging ring for nc_blob_
  std::vector<cudaEvent_t> nc_pinned_ev_;
  int nc_ring_ = 0;
  void build_nc();
  void nc_prepare(double t_stage);
  void nc_fill(bool grad);
  void nc_lift();
  void nc_flux();

  double time_ = 0.0;
  int step_index_ = 0, stage_index_ = 0;
  int next_stage_ = 0;  // the RK stage rk_stage expects next
  bool traces_valid_ = false;
  int cur_trace_ = 0;  // traces of the current state live in trace_[cur_trace_]
  long launches_ = 0;
  bool timing_ = false;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> events_;
  cudaEvent_t pending_start_ = nullptr;
  double class_ms_[KC_N] = {};
  long class_n_[KC_N] = {};
};

GpuRankSolver::GpuRankSolver(const sdg_mesh_spec& ms, const sdg_solver_config& cfg, int n_ranks, int rank,
                             int device, const void* nccl_id, const char* inproc_hub)
    : mesh_(ms), part_(assign_ranks(mesh_, n_ranks)), topo_(build_topology(mesh_, part_, rank)),
      basis_(cfg.degree, cfg.node_kind), cfg_(cfg), rank_(rank), n_ranks_(n_ranks), device_(device) {
  const auto& g = cfg.gas;
  if (!(g.gamma > 1.0) || !(g.R > 0.0) || !(g.mu >= 0.0) || !(g.Pr > 0.0))
    throw ConfigError("gas model requires gamma > 1, R > 0, mu >= 0, Pr > 0");
  if (rank < 0 || rank >= n_ranks) throw ConfigError("rank outside [0, n_ranks)");
  n_ = basis_.n;
  n2_ = n_ * n_;
  n3_ = n2_ * n_;
  E_ = static_cast<int>(topo_.gids.size());
  S_ = static_cast<int>(topo_.sliding.size());
  ND_ = static_cast<int>(topo_.dirichlet.size());
  lifting_ = g.mu > 0.0;
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  cuda_check(cudaDeviceGetAttribute(&n_sm_, cudaDevAttrMultiProcessorCount, device), "device attribute");
  if (n_ranks > 1) {
    if (inproc_hub) comm_ = std::make_unique<InProcComm>(inproc_hub, n_ranks, rank);
    else if (nccl_id) comm_ = std::make_unique<NcclComm>(nccl_id, n_ranks, rank);
    else throw ConfigError("multi-rank context needs an NCCL unique id or an in-process hub name");
    // Highest priority: the NCCL kernels of an overlapped round take the SM slots the
    // element kernel's CTAs free first, instead of queueing behind the whole grid.
    int lo_prio = 0, hi_prio = 0;
    cuda_check(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio), "stream priority range");
    cuda_check(cudaStreamCreateWithPriority(&comm_stream_, cudaStreamNonBlocking, hi_prio), "cudaStreamCreate");
    cuda_check(cudaEventCreateWithFlags(&ev_ready_, cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&ev_comm_, cudaEventDisableTiming), "event");
    sm_reserve_ = inproc_hub ? 0 : 8;
  }
  if (n_ranks > 1 && !mesh_.nc_ifaces.empty())
    throw ConfigError("non-matching / obliquely sliding interfaces run on a single rank");
  build_consts();
  upload_topology();
  find_interior_run();
  build_sides();
  build_nc();
  cuda_check(cudaMallocHost(&err_host_, sizeof(ErrRec)), "cudaMallocHost");
  cuda_check(cudaStreamSynchronize(stream_), "setup sync");
}

GpuRankSolver::~GpuRankSolver() {
  if (stream_) cudaStreamSynchronize(stream_);
  for (auto& ev : events_) {
    cudaEventDestroy(ev.second.first);
    cudaEventDestroy(ev.second.second);
  }
  if (comm_stream_) cudaStreamSynchronize(comm_stream_);
  comm_.reset();
  if (ev_ready_) cudaEventDestroy(ev_ready_);
  if (ev_comm_) cudaEventDestroy(ev_comm_);
  if (comm_stream_) cudaStreamDestroy(comm_stream_);
  for (auto* p : nc_pinned_) cudaFreeHost(p);
  for (auto ev : nc_pinned_ev_) cudaEventDestroy(ev);
  if (err_host_) cudaFreeHost(err_host_);
  if (stream_) cudaStreamDestroy(stream_);
}

// Interior run of this rank (host.cpp interior_run).  With the contiguous band-block
// partition it is everything but the first and last planes of the rank's block.
void GpuRankSolver::find_interior_run() {
  int_lo_ = int_hi_ = 0;
  overlap_ = false;
  if (n_ranks_ == 1 || std::getenv("SDG_NO_OVERLAP")) return;
  const auto run = interior_run(topo_);
  int_lo_ = run[0];
  int_hi_ = run[1];
  overlap_ = int_hi_ > int_lo_;
}

void GpuRankSolver::build_consts() {
  const int n = n_;
  for (int i = 0; i < n; ++i) {
    for (int m = 0; m < n; ++m) consts_.dhat[i * kMaxN1 + m] = basis_.w[m] * basis_.D[m * n + i] / basis_.w[i];
    consts_.fl[i] = basis_.fl[i];
    consts_.fr[i] = basis_.fr[i];
    consts_.liftw[0][i] = basis_.fl[i] / basis_.w[i];
    consts_.liftw[1][i] = basis_.fr[i] / basis_.w[i];
    consts_.inv_w[i] = 1.0 / basis_.w[i];
    consts_.w[i] = basis_.w[i];
    consts_.x[i] = basis_.x[i];
  }
  for (size_t b = 0; b < mesh_.bands.size(); ++b) {
    const BandGeom& bg = mesh_.bands[b];
    BandD& d = consts_.bands[b];
    d.x_lo = bg.x_lo;
    d.hx = bg.hx;
    d.hy = bg.hy;
    d.hz = bg.hz;
    d.vg = bg.vg;
    d.vgz = bg.vgz;
    const double jac = 0.125 * bg.hx * bg.hy * bg.hz;
    d.jac = jac;
    d.inv_jac = 1.0 / jac;
    d.sj[0] = 0.25 * bg.hy * bg.hz;
    d.sj[1] = 0.25 * bg.hx * bg.hz;
    d.sj[2] = 0.25 * bg.hx * bg.hy;
    for (int q = 0; q < 3; ++q) d.cdir[q] = d.sj[q] / jac;
    d.nxd = bg.nx;
  }
  consts_.mapping = mesh_.spec.mapping;
  consts_.ny = mesh_.spec.ny;
  consts_.nz = mesh_.spec.nz;
  consts_.warp = mesh_.spec.mapping != SDG_MAP_BOX ? mesh_.spec.warp : 0.0;
  consts_.sec_c = std::cos(sector_angle(mesh_));
  consts_.sec_s = std::sin(sector_angle(mesh_));
  const auto& g = cfg_.gas;
  consts_.gas = {g.gamma, g.gamma - 1.0, g.R, 1.0 / g.R, g.mu, -2.0 / 3.0 * g.mu,
                 g.gamma * g.R * g.mu / ((g.gamma - 1.0) * g.Pr), g.mu > 0.0 ? 1 : 0};
  consts_.y0 = mesh_.spec.y0;
  consts_.z0 = mesh_.spec.z0;
  consts_.flow_case = cfg_.flow_case;
}

void GpuRankSolver::upload_topology() {
  const size_t slots = static_cast<size_t>(6) * E_ + topo_.n_halo;
  U_.alloc(static_cast<size_t>(E_) * n3_ * 5);
  reg_.alloc(U_.n);
  dudt_.alloc(U_.n);
  U_.zero(stream_);
  reg_.zero(stream_);
  for (auto& t : trace_) {
    t.alloc(slots * n2_ * 5);
    t.zero(stream_);
  }
  fvn_.alloc(slots * n2_ * 4);
  fvn_.zero(stream_);
  slide_lift_.alloc(static_cast<size_t>(S_) * n2_ * 4);
  slide_flux_.alloc(static_cast<size_t>(S_) * n2_ * 5);
  slide_g_.alloc(static_cast<size_t>(S_) * n2_ * 12);
  dir_g_.alloc(static_cast<size_t>(ND_) * n2_ * 12);
  side_type_.upload(topo_.side_type, stream_);
  side_rot_.upload(topo_.side_rot, stream_);
  side_idx_.upload(topo_.side_idx, stream_);
  {
    std::vector<int> code(static_cast<size_t>(E_) * 8, 0);
    for (int e = 0; e < E_; ++e)
      for (int q = 0; q < 6; ++q) {
        const int idx = topo_.side_idx[6 * e + q];
        if (idx < 0 || idx >= (1 << 29)) throw ConfigError("face index exceeds the side-code range");
        code[8 * e + q] = idx | (static_cast<int>(topo_.side_type[6 * e + q]) << 29);
      }
    for (int e = 0; e < E_; ++e) code[8 * e + 6] = topo_.coords[4 * e];  // band of the element
    side_code_.upload(code, stream_);
  }
  coords_.upload(topo_.coords, stream_);
  curved_ = mesh_.spec.mapping != SDG_MAP_BOX;
  if (curved_) {
    CurvedMetrics cm = compute_metrics(mesh_, basis_, topo_);
    // Device layout: per element structure-of-arrays, met[e][c][node] and
    // fmet[e][side][c][f] (curved.cuh), so a warp's threads read consecutive words.
    // Transposed block by block in place (1.1M-element meshes carry ~36 GB of metrics).
    const int mw = cm.mw, fw = cm.fw;
    std::vector<double> tmp(std::max<size_t>(static_cast<size_t>(n3_) * mw, static_cast<size_t>(n2_) * fw));
    for (int e = 0; e < E_; ++e) {
      double* blk = cm.met.data() + static_cast<size_t>(e) * n3_ * mw;
      for (int g = 0; g < n3_; ++g)
        for (int c = 0; c < mw; ++c) tmp[static_cast<size_t>(c) * n3_ + g] = blk[static_cast<size_t>(g) * mw + c];
      std::copy(tmp.begin(), tmp.begin() + static_cast<size_t>(n3_) * mw, blk);
      for (int sd = 0; sd < 6; ++sd) {
        double* fb = cm.fmet.data() + (static_cast<size_t>(e) * 6 + sd) * n2_ * fw;
        for (int f = 0; f < n2_; ++f)
          for (int c = 0; c < fw; ++c) tmp[static_cast<size_t>(c) * n2_ + f] = fb[static_cast<size_t>(f) * fw + c];
        std::copy(tmp.begin(), tmp.begin() + static_cast<size_t>(n2_) * fw, fb);
      }
    }
    met_.upload(cm.met, stream_);
    fmet_.upload(cm.fmet, stream_);
    cuda_check(cudaStreamSynchronize(stream_), "metric upload");
  }
  // Viscous stresses and heat flux per node, handed from the gradient kernel to the
  // update kernel (bulk-loaded kernels, even N+1; curved.cuh k_update_cv).
  if (cfg_.gas.mu > 0.0 && n_ % 2 == 0) visc_.alloc(static_cast<size_t>(E_) * n3_ * 9);
  err_.alloc(1);
  err_.zero(stream_);
  dt_min_.alloc(1);
  // Halo send slots (concatenated over peers).
  std::vector<int> send;
  for (const auto& p : topo_.peers) send.insert(send.end(), p.send_slots.begin(), p.send_slots.end());
  send_slots_.upload(send, stream_);
  send_buf_.alloc(send.size() * n2_ * 5);
}

// Interface-side contexts (solver.cpp:73-90) and the device pairing tables.
void GpuRankSolver::build_sides() {
  const int ni = static_cast<int>(mesh_.ifaces.size());
  for (int ic = 0; ic < ni; ++ic)
    for (const bool left : {true, false}) {
      SideCtx c;
      c.iface = ic;
      for (int k = 0; k < S_; ++k) {
        const auto& r = topo_.sliding[k];
        if (!r.nc && r.iface == ic && (r.side == 1) == left) c.slides.push_back(k);
      }
      if (c.slides.empty()) continue;
      c.on_static = mesh_.ifaces[ic].static_is_left == left;
      std::sort(c.slides.begin(), c.slides.end(), [&](int a, int b) {
        const auto &ra = topo_.sliding[a], &rb = topo_.sliding[b];
        return ra.i_par != rb.i_par ? ra.i_par < rb.i_par : ra.i_perp < rb.i_perp;
      });
      c.fwd.assign(2 * n2_, 0.0);
      c.bwd.assign(2 * n2_, 0.0);
      sides_.push_back(std::move(c));
    }
  if (sides_.size() > static_cast<size_t>(kMaxCtx)) throw ConfigError("too many interface sides");
  // Per-sliding-face lookup tables.
  std::vector<int> s_elem(S_), s_side(S_), s_ctx(S_, -1), s_f(S_, -1);
  std::vector<int> off(sides_.size()), nf(sides_.size()), role(sides_.size()), sleft(sides_.size());
  std::vector<int> fpar, fperp, fslide;
  int o = 0;
  for (size_t c = 0; c < sides_.size(); ++c) {
    const auto& sc = sides_[c];
    off[c] = o;
    nf[c] = static_cast<int>(sc.slides.size());
    role[c] = sc.on_static ? 0 : 1;
    sleft[c] = mesh_.ifaces[sc.iface].static_is_left ? 1 : 0;
    role_ids_[role[c]].push_back(static_cast<int>(c));
    for (int f = 0; f < nf[c]; ++f) {
      const int k = sc.slides[f];
      s_ctx[k] = static_cast<int>(c);
      s_f[k] = f;
      fpar.push_back(static_cast<int>(topo_.sliding[k].i_par));
      fperp.push_back(static_cast<int>(topo_.sliding[k].i_perp));
      fslide.push_back(k);
    }
    o += nf[c];
    max_mortars_[role[c]] += 2 * nf[c];
  }
  for (int k = 0; k < S_; ++k) {
    s_elem[k] = topo_.sliding[k].elem;
    s_side[k] = topo_.sliding[k].side;
  }
  slide_elem_.upload(s_elem, stream_);
  slide_side_.upload(s_side, stream_);
  slide_ctx_.upload(s_ctx, stream_);
  slide_f_.upload(s_f, stream_);
  ctx_face_off_.upload(off, stream_);
  ctx_nf_.upload(nf, stream_);
  ctx_role_.upload(role, stream_);
  ctx_static_left_.upload(sleft, stream_);
  face_par_.upload(fpar, stream_);
  face_perp_.upload(fperp, stream_);
  face_slide_.upload(fslide, stream_);
  m_.alloc(2 * static_cast<size_t>(std::max(o, 1)));
  ctx_state_.alloc(2 * kMaxCtx);
  ctx_state_.zero(stream_);
  ctx_sdelta_.alloc(kMaxCtx);
  n_mortars_.alloc(2);
  n_mortars_.zero(stream_);
  // Dense key space of the pairing sort.
  pargs_.n_ctx = static_cast<int>(sides_.size());
  pargs_.n_ifaces = ni;
  long long base = 0;
  for (int ic = 0; ic < ni; ++ic) {
    pargs_.iface_base[ic] = base;
    pargs_.iface_nperp[ic] = mesh_.ifaces[ic].n_perp;
    base += 2LL * mesh_.ifaces[ic].n_faces * mesh_.ifaces[ic].n_perp;
  }
  pargs_.dense_size = base;
  pargs_.self_rank = rank_;
  for (int r = 0; r < 2; ++r) {
    pargs_.role_nctx[r] = static_cast<int>(role_ids_[r].size());
    for (size_t q = 0; q < role_ids_[r].size(); ++q) pargs_.role_ctx[r][q] = role_ids_[r][q];
    pres_[r].alloc(std::max<long long>(base, 1));
    payload_[r].alloc(std::max<long long>(base, 1));
    cols_[r].alloc(7 * static_cast<size_t>(std::max(max_mortars_[r], 1)));
    const size_t nodes = static_cast<size_t>(std::max(max_mortars_[r], 1)) * n2_;
    u_mine_[r].alloc(nodes * 5);
    mlift_[r].alloc(nodes * 4);
    g_mine_[r].alloc(nodes * 12);
    mflux_[r].alloc(nodes * 5);
  }
  const size_t snodes = static_cast<size_t>(std::max(max_mortars_[0], 1)) * n2_;
  u_theirs_.alloc(snodes * 5);
  g_theirs_.alloc(snodes * 12);
  for (size_t c = 0; c < sides_.size(); ++c) {
    const auto& ifc = mesh_.ifaces[sides_[c].iface];
    CtxD& d = pargs_.ctx[c];
    d.iface = sides_[c].iface;
    d.on_static = sides_[c].on_static ? 1 : 0;
    d.role = role[c];
    d.n_faces = nf[c];
    d.face_off = off[c];
    d.n_par = ifc.n_faces;
    d.n_perp = ifc.n_perp;
    d.static_is_left = ifc.static_is_left ? 1 : 0;
    d.l_par = ifc.l_par;
    d.vg_rel = ifc.vg_rel;
  }
}

// The one init-time collective (init_rank_maps, solver.cpp:95-133): every rank
// contributes (iface, side, i_par, i_perp) of its interface faces; the owner
// maps r, r~ follow, and each side keeps the map of its partner side.
void GpuRankSolver::init_rank_maps() {
  std::vector<int> mine;
  for (const auto& c : sides_)
    for (int k : c.slides) {
      mine.push_back(c.iface);
      mine.push_back(c.on_static ? 0 : 1);
      mine.push_back(static_cast<int>(topo_.sliding[k].i_par));
      mine.push_back(static_cast<int>(topo_.sliding[k].i_perp));
    }
  std::vector<std::vector<int>> all(n_ranks_);
  if (n_ranks_ == 1) {
    all[0] = mine;
  } else {
    for (int r = 0; r < n_ranks_; ++r)
      if (r != rank_) comm_trace_.push_back({-1, 0, rank_, r, static_cast<long long>(mine.size()), MK_INIT, true});
    comm_->allgather_ints(mine, all, stream_);
  }
  const int ni = static_cast<int>(mesh_.ifaces.size());
  std::vector<std::vector<int>> smap(ni), mmap(ni);
  for (int ic = 0; ic < ni; ++ic) {
    const size_t sz = static_cast<size_t>(mesh_.ifaces[ic].n_faces * mesh_.ifaces[ic].n_perp);
    smap[ic].assign(sz, -1);
    mmap[ic].assign(sz, -1);
  }
  for (int r = 0; r < n_ranks_; ++r)
    for (size_t q = 0; q + 3 < all[r].size(); q += 4) {
      const int ic = all[r][q];
      const bool is_static = all[r][q + 1] == 0;
      const long np = mesh_.ifaces[ic].n_faces;
      const size_t slot = static_cast<size_t>(all[r][q + 3]) * np + all[r][q + 2];
      int& owner = (is_static ? smap[ic] : mmap[ic])[slot];
      if (owner != -1) throw ProtocolError("interface face claimed by two ranks");
      owner = r;
    }
  for (int ic = 0; ic < ni; ++ic)
    for (const auto* mp : {&smap[ic], &mmap[ic]})
      for (int r : *mp)
        if (r < 0) throw ProtocolError("interface face without an owner");
  std::vector<int> concat;
  for (size_t c = 0; c < sides_.size(); ++c) {
    auto& sc = sides_[c];
    sc.static_map = smap[sc.iface];
    sc.moving_map = mmap[sc.iface];
    pargs_.ctx[c].map_off = static_cast<int>(concat.size());
    const auto& partner = sc.on_static ? sc.moving_map : sc.static_map;
    concat.insert(concat.end(), partner.begin(), partner.end());
  }
  if (concat.empty()) concat.push_back(0);
  partner_map_.upload(concat, stream_);
  cuda_check(cudaStreamSynchronize(stream_), "rank maps");
}

void GpuRankSolver::set_initial_condition(double t0) {
  std::vector<double> h(static_cast<size_t>(E_) * n3_ * 5);
  const int n = n_;
  for (int e = 0; e < E_; ++e) {
    const int b = topo_.coords[4 * e], ix = topo_.coords[4 * e + 1], iy = topo_.coords[4 * e + 2],
              iz = topo_.coords[4 * e + 3];
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        for (int k = 0; k < n; ++k) {
          double x[3];
          map_point(mesh_, b, ix, iy, iz, basis_.x[i], basis_.x[j], basis_.x[k], t0, x);
          eval_case_host(cfg_.flow_case, cfg_.gas, x, t0, h.data() + ((static_cast<size_t>(e) * n3_) + (i * n + j) * n + k) * 5);
        }
  }
  cuda_check(cudaMemcpyAsync(U_.p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, stream_), "h2d");
  reset_clock(t0);
  traces_valid_ = false;
  cuda_check(cudaStreamSynchronize(stream_), "set_initial_condition");
}

// Time, step counter, RK register and interface offsets of a run starting at t0.
void GpuRankSolver::reset_clock(double t0) {
  time_ = t0;
  step_index_ = 0;
  next_stage_ = 0;
  reg_.zero(stream_);
  for (auto& c : sides_) {
    c.delta_base = mesh_.ifaces[c.iface].vg_rel * t0;
    c.wraps = 0;
    c.topo_valid = false;
  }
  for (auto& r : nc_) {
    r.dy_base = mesh_.nc_ifaces[r.iface].vy_rel * t0;
    r.dz_base = mesh_.nc_ifaces[r.iface].vz_rel * t0;
  }
}

void GpuRankSolver::set_state(const double* h) {
  cuda_check(cudaMemcpyAsync(U_.p, h, U_.n * sizeof(double), cudaMemcpyHostToDevice, stream_), "set_state");
  cuda_check(cudaStreamSynchronize(stream_), "set_state");
  traces_valid_ = false;
}
void GpuRankSolver::get_state(double* h) {
  cuda_check(cudaMemcpyAsync(h, U_.p, U_.n * sizeof(double), cudaMemcpyDeviceToHost, stream_), "get_state");
  synchronize();
}
void GpuRankSolver::get_register(double* h) {
  cuda_check(cudaMemcpyAsync(h, reg_.p, reg_.n * sizeof(double), cudaMemcpyDeviceToHost, stream_), "get_register");
  synchronize();
}

FieldPtrs GpuRankSolver::field_ptrs(double* U, double* out) {
  FieldPtrs p{};
  p.U = U;
  p.reg = reg_.p;
  p.out = out;
  p.trace = trace_[cur_trace_].p;
  p.trace_out = trace_[cur_trace_ ^ 1].p;
  p.fvn = fvn_.p;
  p.slide_lift = slide_lift_.p;
  p.slide_flux = slide_flux_.p;
  p.slide_g = slide_g_.p;
  p.dir_g = dir_g_.p;
  p.side_type = side_type_.p;
  p.side_idx = side_idx_.p;
  p.coords = coords_.p;
  p.side_code = side_code_.p;
  p.grad_out = nullptr;
  p.met = met_.p;
  p.fmet = fmet_.p;
  p.visc = visc_.p;
  p.side_rot = side_rot_.p;
  p.err = err_.p;
  p.E = E_;
  return p;
}

MortarPtrs GpuRankSolver::mortar_ptrs() {
  MortarPtrs p{};
  p.trace = trace_[cur_trace_].p;
  for (int r = 0; r < 2; ++r) {
    p.u_mine[r] = u_mine_[r].p;
    p.lift[r] = mlift_[r].p;
    p.g_mine[r] = g_mine_[r].p;
    p.flux[r] = mflux_[r].p;
  }
  p.u_theirs = u_theirs_.p;
  p.g_theirs = g_theirs_.p;
  p.slide_lift = slide_lift_.p;
  p.slide_flux = slide_flux_.p;
  p.slide_g = slide_g_.p;
  p.slide_elem = slide_elem_.p;
  p.slide_side = slide_side_.p;
  p.slide_ctx = slide_ctx_.p;
  p.slide_f = slide_f_.p;
  p.m = m_.p;
  p.ctx_face_off = ctx_face_off_.p;
  p.ctx_nf = ctx_nf_.p;
  p.ctx_role = ctx_role_.p;
  p.ctx_state = ctx_state_.p;
  p.n_mortars = n_mortars_.p;
  p.cols_static = cols_[0].p;
  p.cols_moving = cols_[1].p;
  p.ctx_static_left = ctx_static_left_.p;
  p.S = S_;
  p.alpha = sector_angle(mesh_);
  p.sector = p.alpha != 0.0;
  for (size_t c = 0; c < sides_.size(); ++c) p.wind[c] = static_cast<int>(sides_[c].wind);
  return p;
}

void GpuRankSolver::mark(int cls, bool begin) {
  if (!timing_) return;
  if (begin) {
    cudaEvent_t a;
    cudaEventCreate(&a);
    cudaEventRecord(a, stream_);
    pending_start_ = a;
  } else {
    cudaEvent_t b;
    cudaEventCreate(&b);
    cudaEventRecord(b, stream_);
    events_.push_back({cls, {pending_start_, b}});
  }
}

std::vector<std::pair<double, long>> GpuRankSolver::timing_totals() {
  cuda_check(cudaStreamSynchronize(stream_), "timing sync");
  for (auto& ev : events_) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev.second.first, ev.second.second);
    class_ms_[ev.first] += ms;
    class_n_[ev.first] += 1;
    cudaEventDestroy(ev.second.first);
    cudaEventDestroy(ev.second.second);
  }
  events_.clear();
  std::vector<std::pair<double, long>> out;
  for (int c = 0; c < KC_N; ++c) out.push_back({class_ms_[c], class_n_[c]});
  for (int c = 0; c < KC_N; ++c) {
    class_ms_[c] = 0.0;
    class_n_[c] = 0;
  }
  return out;
}

// ---------------------------------------------------------------------------
// Non-matching / oblique interfaces (BASELINE configs[1]).  Per stage the host
// displaces side B by (dy, dz), merges the face rows (merge_intervals) and builds
// the long-double sub-range operators of every row and the face -> row CSR
// lists; one upload carries them.  The device recomputes both rows
// (k_nc_rows, checked against the host's: a mismatch is a ProtocolError) and
// indexes the faces through its own rows.  Chain (the reference's mortar chain,
// solver.cpp:234-252, 597-727, 442-526, on tensor-product mortars): traces ->
// mortars -> lifting mean -> back to both sides (slide_lift); gradients ->
// mortars -> two-sided Roe + viscous flux -> back to both sides (slide_flux).
// The element kernels read slide_lift / slide_flux exactly as for the
// reference's mortars.
// ---------------------------------------------------------------------------
void GpuRankSolver::build_nc() {
  const int ni = static_cast<int>(mesh_.nc_ifaces.size());
  if (ni == 0) return;
  nc_.resize(ni);
  size_t blob = 0;
  for (int i = 0; i < ni; ++i) {
    NcRuntime& r = nc_[i];
    const NcIfaceGeom& f = mesh_.nc_ifaces[i];
    r.iface = i;
    std::vector<int> slot[2], kidx[2];
    for (int s = 0; s < 2; ++s) {
      slot[s].assign(f.nfy[s] * f.nfz[s], -1);
      kidx[s].assign(f.nfy[s] * f.nfz[s], -1);
    }
    for (int k = 0; k < S_; ++k) {
      const SlidingFaceRec& rec = topo_.sliding[k];
      if (!rec.nc || rec.iface != i) continue;
      const int s = rec.side == 1 ? 0 : 1;  // A: the left band's x+ faces
      const long face = rec.i_par * f.nfz[s] + rec.i_perp;
      slot[s][face] = 6 * rec.elem + rec.side;
      kidx[s][face] = k;
    }
    for (int s = 0; s < 2; ++s) {
      for (int v : slot[s])
        if (v < 0) throw ConfigError("non-matching interface side is not complete on this rank");
      r.slot[s].upload(slot[s], stream_);
      r.kidx[s].upload(kidx[s], stream_);
    }
    r.max_m[0] = f.nfy[0] + f.nfy[1];
    r.max_m[1] = f.nfz[0] + f.nfz[1];
    for (int d = 0; d < 2; ++d) {
      r.d_faces[d].alloc(2 * r.max_m[d]);
      r.d_ranges[d].alloc(4 * r.max_m[d]);
    }
    r.d_n.alloc(2);
    const size_t nodes = static_cast<size_t>(r.max_m[0] * r.max_m[1]) * n2_;
    for (int s = 0; s < 2; ++s) {
      r.mu[s].alloc(nodes * 5);
      if (lifting_) r.mg[s].alloc(nodes * 12);
    }
    r.mlift.alloc(nodes * 4);
    r.mflux.alloc(nodes * 5);
    // Upload capacity: host rows, operators (F, B per side and row) and CSR.
    size_t bytes = 0;
    for (int d = 0; d < 2; ++d) {
      const long long m = r.max_m[d];
      const long long nf = d == 0 ? std::max(f.nfy[0], f.nfy[1]) : std::max(f.nfz[0], f.nfz[1]);
      bytes += m * 2 * sizeof(long long) + m * 4 * sizeof(double);
      bytes += 2 * 2 * m * n2_ * sizeof(double);
      bytes += 2 * ((nf + 1 + m) * sizeof(int) + 8);
    }
    r.blob_off = blob;
    r.blob_bytes = bytes + 256;  // + alignment of the 20 tables
    blob += r.blob_bytes;
  }
  nc_blob_.alloc(blob);
  for (int k = 0; k < 4; ++k) {
    unsigned char* p = nullptr;
    cuda_check(cudaMallocHost(&p, blob), "cudaMallocHost");
    nc_pinned_.push_back(p);
    cudaEvent_t ev;
    cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
    nc_pinned_ev_.push_back(ev);
  }
}

void GpuRankSolver::nc_prepare(double t_stage) {
  const int slot = nc_ring_;
  nc_ring_ = (nc_ring_ + 1) % static_cast<int>(nc_pinned_.size());
  cuda_check(cudaEventSynchronize(nc_pinned_ev_[slot]), "nc staging reuse");
  unsigned char* host = nc_pinned_[slot];
  const int nn = n2_;
  for (auto& r : nc_) {
    const NcIfaceGeom& f = mesh_.nc_ifaces[r.iface];
    r.dy = r.dy_base + f.vy_rel * (t_stage - time_);
    r.dz = r.dz_base + f.vz_rel * (t_stage - time_);
    NcStage& S = r.S;
    S = NcStage{};
    size_t off = r.blob_off;
    auto take = [&](size_t bytes) {
      off = (off + 7) & ~static_cast<size_t>(7);
      const size_t o = off;
      off += bytes;
      if (off > r.blob_off + r.blob_bytes) throw ProtocolError("non-matching interface tables overflow");
      return o;
    };
    for (int s = 0; s < 2; ++s) {
      S.nfy[s] = f.nfy[s];
      S.nfz[s] = f.nfz[s];
    }
    std::map<std::pair<double, double>, int> cache;
    std::vector<double> opsF, opsB;
    for (int d = 0; d < 2; ++d) {
      const long n_a = d == 0 ? f.nfy[0] : f.nfz[0], n_b = d == 0 ? f.nfy[1] : f.nfz[1];
      const double l_a = d == 0 ? f.ly[0] : f.lz[0], delta = d == 0 ? r.dy : r.dz;
      const std::vector<MortarInterval> rows = merge_intervals(n_a, n_b, l_a, delta);
      const long long m = static_cast<long long>(rows.size());
      if (m > r.max_m[d]) throw ProtocolError("non-matching interface row exceeds its capacity");
      (d == 0 ? S.my : S.mz) = m;
      S.n_a[d] = n_a;
      S.n_b[d] = n_b;
      S.l_a[d] = l_a;
      S.delta[d] = delta;
      const size_t o_faces = take(m * 2 * sizeof(long long)), o_rng = take(m * 4 * sizeof(double));
      auto* hf = reinterpret_cast<long long*>(host + o_faces);
      auto* hr = reinterpret_cast<double*>(host + o_rng);
      for (long long k = 0; k < m; ++k) {
        hf[2 * k] = rows[k].face_a;
        hf[2 * k + 1] = rows[k].face_b;
        hr[4 * k] = rows[k].a_lo;
        hr[4 * k + 1] = rows[k].a_hi;
        hr[4 * k + 2] = rows[k].b_lo;
        hr[4 * k + 3] = rows[k].b_hi;
      }
      S.h_faces[d] = reinterpret_cast<const long long*>(nc_blob_.p + o_faces);
      S.h_ranges[d] = reinterpret_cast<const double*>(nc_blob_.p + o_rng);
      S.d_faces[d] = r.d_faces[d].p;
      S.d_ranges[d] = r.d_ranges[d].p;
      for (int s = 0; s < 2; ++s) {
        const size_t oF = take(m * nn * sizeof(double)), oB = take(m * nn * sizeof(double));
        auto* F = reinterpret_cast<double*>(host + oF);
        auto* B = reinterpret_cast<double*>(host + oB);
        for (long long k = 0; k < m; ++k) {
          const double lo = s == 0 ? rows[k].a_lo : rows[k].b_lo, hi = s == 0 ? rows[k].a_hi : rows[k].b_hi;
          // Distinct sub-ranges of a row repeat with the face-count ratio: build each once.
          auto it = cache.find({lo, hi});
          if (it == cache.end()) {
            const int id = static_cast<int>(opsF.size() / nn);
            opsF.resize(opsF.size() + nn);
            opsB.resize(opsB.size() + nn);
            build_subrange_ops(basis_, lo, hi, opsF.data() + static_cast<size_t>(id) * nn,
                               opsB.data() + static_cast<size_t>(id) * nn);
            it = cache.emplace(std::make_pair(lo, hi), id).first;
          }
          std::copy_n(opsF.data() + static_cast<size_t>(it->second) * nn, nn, F + k * nn);
          std::copy_n(opsB.data() + static_cast<size_t>(it->second) * nn, nn, B + k * nn);
        }
        S.F[s][d] = reinterpret_cast<const double*>(nc_blob_.p + oF);
        S.B[s][d] = reinterpret_cast<const double*>(nc_blob_.p + oB);
        // Face -> rows CSR of this side, rows in ascending order (a fixed summation order).
        const long nf = s == 0 ? n_a : n_b;
        const size_t oO = take((nf + 1) * sizeof(int)), oI = take(m * sizeof(int));
        int* O = reinterpret_cast<int*>(host + oO);
        int* I = reinterpret_cast<int*>(host + oI);
        std::fill(O, O + nf + 1, 0);
        for (long long k = 0; k < m; ++k) ++O[(s == 0 ? rows[k].face_a : rows[k].face_b) + 1];
        for (long q = 0; q < nf; ++q) O[q + 1] += O[q];
        std::vector<int> fill(O, O + nf);
        for (long long k = 0; k < m; ++k) I[fill[s == 0 ? rows[k].face_a : rows[k].face_b]++] = static_cast<int>(k);
        S.off[s][d] = reinterpret_cast<const int*>(nc_blob_.p + oO);
        S.idx[s][d] = reinterpret_cast<const int*>(nc_blob_.p + oI);
      }
    }
    S.d_n = r.d_n.p;
  }
  const size_t total = nc_blob_.n;
  cuda_check(cudaMemcpyAsync(nc_blob_.p, host, total, cudaMemcpyHostToDevice, stream_), "nc tables h2d");
  cuda_check(cudaEventRecord(nc_pinned_ev_[slot], stream_), "event record");
  mark(KC_PAIRING, true);
  for (auto& r : nc_) launch_nc_rows(r.S, r.iface, err_.p, stream_);
  mark(KC_PAIRING, false);
  launches_ += static_cast<long>(nc_.size());
}

// Face -> mortar of both sides: the traces (grad = false) or the gradient traces.
void GpuRankSolver::nc_fill(bool grad) {
  if (nc_.empty() || (grad && !lifting_)) return;
  mark(KC_MORTAR, true);
  for (auto& r : nc_) {
    if (grad) {
      const int* tab[2] = {r.kidx[0].p, r.kidx[1].p};
      double* out[2] = {r.mg[0].p, r.mg[1].p};
      launch_nc_fill(n_, 12, slide_g_.p, r.S, tab, out, stream_);
    } else {
      const int* tab[2] = {r.slot[0].p, r.slot[1].p};
      double* out[2] = {r.mu[0].p, r.mu[1].p};
      launch_nc_fill(n_, 5, trace_[cur_trace_].p, r.S, tab, out, stream_);
    }
    launches_++;
  }
  mark(KC_MORTAR, false);
}

// Lifting mean at the mortar nodes, projected back onto both sides (slide_lift).
void GpuRankSolver::nc_lift() {
  if (nc_.empty()) return;
  mark(KC_MORTAR, true);
  for (auto& r : nc_) {
    const long long nodes = r.S.my * r.S.mz * n2_;
    launch_nc_mortar_lift(nodes, consts_.gas, r.mu[0].p, r.mu[1].p, r.mlift.p, stream_);
    const int* tab[2] = {r.kidx[0].p, r.kidx[1].p};
    launch_nc_project(n_, 4, r.mlift.p, r.S, tab, slide_lift_.p, stream_);
    launches_ += 2;
  }
  mark(KC_MORTAR, false);
}

// Two-sided flux at the mortar nodes, projected back onto both sides (slide_flux).
void GpuRankSolver::nc_flux() {
  if (nc_.empty()) return;
  mark(KC_MORTAR, true);
  for (auto& r : nc_) {
    const long long nodes = r.S.my * r.S.mz * n2_;
    launch_nc_flux(nodes, consts_.gas, r.mu[0].p, r.mu[1].p, lifting_ ? r.mg[0].p : nullptr,
                   lifting_ ? r.mg[1].p : nullptr, r.mflux.p, err_.p, stream_);
    const int* tab[2] = {r.kidx[0].p, r.kidx[1].p};
    launch_nc_project(n_, 5, r.mflux.p, r.S, tab, slide_flux_.p, stream_);
    launches_ += 2;
  }
  mark(KC_MORTAR, false);
}

// Device rows of the last stage (the pairing of a non-matching interface).
void GpuRankSolver::nc_rows(int i, int dir, long* n_out, long* faces, double* ranges, double* delta) {
  if (i < 0 || i >= static_cast<int>(nc_.size()) || dir < 0 || dir > 1)
    throw ConfigError("no such non-matching interface / direction");
  const NcRuntime& r = nc_[i];
  long long n[2] = {0, 0};
  cuda_check(cudaMemcpyAsync(n, r.d_n.p, sizeof(n), cudaMemcpyDeviceToHost, stream_), "d2h");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  *n_out = static_cast<long>(n[dir]);
  if (delta) *delta = dir == 0 ? r.dy : r.dz;
  if (faces == nullptr || ranges == nullptr || n[dir] <= 0) return;
  std::vector<long long> f(2 * n[dir]);
  cuda_check(cudaMemcpyAsync(f.data(), r.d_faces[dir].p, f.size() * sizeof(long long), cudaMemcpyDeviceToHost, stream_),
             "d2h");
  cuda_check(cudaMemcpyAsync(ranges, r.d_ranges[dir].p, 4 * n[dir] * sizeof(double), cudaMemcpyDeviceToHost, stream_),
             "d2h");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  for (size_t q = 0; q < f.size(); ++q) faces[q] = static_cast<long>(f[q]);
}

// update_interfaces (solver.cpp:156-176) on the host: displacement, sigma,
// long-double operators, topology-change bookkeeping and the per-partner
// mortar blocks used to size the NCCL messages.
void GpuRankSolver::update_interfaces_host(double t_stage) {
  bool changed[2] = {false, false};
  for (size_t c = 0; c < sides_.size(); ++c) {
    SideCtx& sc = sides_[c];
    const IfaceGeom& f = mesh_.ifaces[sc.iface];
    const double delta = sc.delta_base + f.vg_rel * (t_stage - time_);
    sc.st = displacement(delta, f.l_par, f.n_faces);
    sc.conforming = sc.st.conforming();
    {  // windings: delta = d + wind * period (displacement() wraps d into [0, period))
      const double period = f.l_par * static_cast<double>(f.n_faces);
      double dd = std::fmod(delta, period);
      if (dd < 0.0) dd += period;
      sc.wind = sc.wraps + std::lround((delta - dd) / period);
      if (dd / f.l_par >= static_cast<double>(f.n_faces)) sc.wind += 1;
    }
    const double sigma = 2.0 * sc.st.s_delta - 1.0;
    sc.sigma_side = sc.on_static ? sigma : -sigma;
    if (!sc.conforming && sc.sigma_side != sc.ops_sigma) {
      build_mortar_ops(basis_, sc.sigma_side, sc.fwd.data(), sc.bwd.data());
      sc.ops_sigma = sc.sigma_side;
    }
    for (int h = 0; h < 2; ++h)
      for (int q = 0; q < n2_; ++q) {
        fwd_ops_.op[c][h][(q / n_) * n_ + q % n_] = sc.fwd[h * n2_ + q];
        bwd_ops_.op[c][h][(q / n_) * n_ + q % n_] = sc.bwd[h * n2_ + q];
      }
    if (!sc.topo_valid || sc.st.n_delta != sc.last_n || sc.conforming != sc.last_conf) {
      sc.topo_valid = true;
      sc.last_n = sc.st.n_delta;
      sc.last_conf = sc.conforming;
      sc.rebuilds++;
      changed[sc.on_static ? 0 : 1] = true;
    }
  }
  // Per-partner block sizes (build_schedule, partition.cpp:154-169) on a topology change.
  for (int r = 0; r < 2; ++r) {
    if (!changed[r]) continue;
    std::map<int, int> cnt;
    int total = 0;
    for (int c : role_ids_[r]) {
      const SideCtx& sc = sides_[c];
      const IfaceGeom& f = mesh_.ifaces[sc.iface];
      const auto& pmap = sc.on_static ? sc.moving_map : sc.static_map;
      for (int k : sc.slides) {
        const long ip = topo_.sliding[k].i_par, iq = topo_.sliding[k].i_perp;
        for (int sub = sc.conforming ? 1 : 0; sub < 2; ++sub) {
          const long par = sc.on_static ? moving_index(ip, sc.st.n_delta, sub, f.n_faces)
                                        : static_index(ip, sc.st.n_delta, sub, f.n_faces);
          cnt[pmap[static_cast<size_t>(iq) * f.n_faces + par]]++;
          total++;
        }
      }
    }
    expect_mortars_[r] = total;
    sched_[r].clear();
    self_[r] = {rank_, 0, 0};
    int offp = 0;
    for (const auto& kv : cnt) {
      if (kv.first == rank_) self_[r] = {rank_, offp, kv.second};
      else sched_[r].push_back({kv.first, offp, kv.second});
      offp += kv.second;
    }
  }
}

void GpuRankSolver::run_pairing(double t_stage) {
  PairingArgs a = pargs_;
  for (size_t c = 0; c < sides_.size(); ++c) a.delta_base[c] = sides_[c].delta_base;
  a.time = time_;
  a.t_stage = t_stage;
  a.expect_mortars[0] = expect_mortars_[0];
  a.expect_mortars[1] = expect_mortars_[1];
  PairingPtrs p{};
  p.ctx_face_par = face_par_.p;
  p.ctx_face_perp = face_perp_.p;
  p.ctx_face_slide = face_slide_.p;
  p.partner_map = partner_map_.p;
  for (int r = 0; r < 2; ++r) {
    p.pres[r] = pres_[r].p;
    p.payload[r] = payload_[r].p;
    p.cols[r] = cols_[r].p;
  }
  p.m = m_.p;
  p.ctx_state = ctx_state_.p;
  p.ctx_sdelta = ctx_sdelta_.p;
  p.n_mortars = n_mortars_.p;
  p.err = err_.p;
  mark(KC_PAIRING, true);
  launch_pairing(a, p, stream_);
  mark(KC_PAIRING, false);
  launches_++;
}

// Mortar block exchange between the two roles (send_solution_phase etc.):
// moving_to_static: src[1] blocks -> dst (static "theirs"); otherwise src[0]
// blocks -> dst (moving array).  Self blocks are device copies, remote
// blocks grouped NCCL send/recv in ascending partner order.
void GpuRankSolver::mortar_exchange(double* const src[2], double* dst, int nc, bool moving_to_static, int kind) {
  const int from = moving_to_static ? 1 : 0, to = 1 - from;
  const size_t node = static_cast<size_t>(n2_) * nc;
  const auto& sf = self_[from];
  const auto& st = self_[to];
  if (sf[2] > 0) {
    if (sf[2] != st[2]) throw ProtocolError("loopback mortar block size mismatch");
    mark(KC_COPY, true);
    cuda_check(cudaMemcpyAsync(dst + st[1] * node, src[from] + sf[1] * node, sf[2] * node * sizeof(double),
                               cudaMemcpyDeviceToDevice, stream_),
               "self mortar copy");
    mark(KC_COPY, false);
  }
  if (n_ranks_ == 1) return;
  std::vector<Xfer> sends, recvs;
  for (const auto& e : sched_[from]) sends.push_back({e[0], src[from] + e[1] * node, e[2] * node});
  for (const auto& e : sched_[to]) recvs.push_back({e[0], dst + e[1] * node, e[2] * node});
  record(kind, sends, recvs);
  mark(KC_HALO, true);
  comm_round(sends, recvs, true);
  mark(KC_HALO, false);
}

// One grouped exchange on the comm stream, after everything stream_ has enqueued so far.
// join: stream_ waits for it at once; otherwise join_comm() later.
// overlap_work is enqueued on stream_ after the data-ready point and before the round is
// issued, so it runs concurrently with the exchange even when the transport blocks the host.
void GpuRankSolver::comm_round(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, bool join,
                               const std::function<void()>& overlap_work) {
  cuda_check(cudaEventRecord(ev_ready_, stream_), "event record");
  if (overlap_work) overlap_work();
  cuda_check(cudaStreamWaitEvent(comm_stream_, ev_ready_, 0), "wait event");
  comm_->exchange(sends, recvs, comm_stream_);
  cuda_check(cudaEventRecord(ev_comm_, comm_stream_), "event record");
  if (join) join_comm();
}

// stream_ waits for every comm round issued so far (they run in order on comm_stream_).
void GpuRankSolver::join_comm() {
  if (comm_stream_) cuda_check(cudaStreamWaitEvent(stream_, ev_comm_, 0), "wait event");
}

// Per-launch arguments of the element kernels; on an annulus, every band's rotation
// (cos, sin)(vg * t_stage) is evaluated here once instead of by every thread.
StageArgs GpuRankSolver::stage_args(double t_stage, double dt, double rk_a, double rk_b, int mode) const {
  StageArgs a{};
  a.t_stage = t_stage;
  a.dt = dt;
  a.rk_a = rk_a;
  a.rk_b = rk_b;
  a.mode = mode;
  a.step = step_index_;
  a.stage = stage_index_;
  const bool rot = mesh_.spec.mapping == SDG_MAP_ANNULUS;
  for (int b = 0; b < SDG_MAX_BANDS; ++b) {
    const double phi = rot && b < static_cast<int>(mesh_.bands.size()) ? consts_.bands[b].vg * t_stage : 0.0;
    a.rot_c[b] = std::cos(phi);
    a.rot_s[b] = std::sin(phi);
  }
  return a;
}

// k_gradient / k_update over local elements [e_first, e_end).
void GpuRankSolver::element_kernel(bool update, const FieldPtrs& fp0, const StageArgs& a, int e_first, int e_end,
                                   int n_sm) {
  if (e_end <= e_first) return;
  FieldPtrs fp = fp0;
  fp.e_first = e_first;
  fp.E = e_end;
  mark(update ? KC_UPDATE : KC_GRADIENT, true);
  // Affine elements (even N+1): the update in the bulk-loaded, non-persistent structure
  // of curved.cuh at 4 CTAs/SM, the gradient in the warp-specialised persistent kernel
  // (DESIGN.md §4); the plain kernels for odd N+1.
  if (curved_) {
    if (update) launch_update_curved(n_, consts_, fp, a, stream_);
    else launch_gradient_curved(n_, consts_, fp, a, stream_);
  } else if (update) {
    if (!launch_update_affine_b(n_, consts_, fp, a, stream_)) launch_update(n_, consts_, fp, a, stream_);
  } else {
    if (!launch_gradient_tma(n_, consts_, fp, a, n_sm, stream_)) launch_gradient(n_, consts_, fp, a, stream_);
  }
  mark(update ? KC_UPDATE : KC_GRADIENT, false);
  launches_++;
}

// Conforming halo exchange of face data (traces or Fv.n): gather the local
// slots facing each peer, then grouped NCCL send/recv straight into the halo
// slots (contiguous per peer by construction).
__global__ void k_gather_slots(const double* src, const int* slots, int n_slots, int per_slot, double* dst) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<long long>(n_slots) * per_slot) return;
  const int s = static_cast<int>(i / per_slot), q = static_cast<int>(i % per_slot);
  dst[i] = src[static_cast<size_t>(slots[s]) * per_slot + q];
}

void GpuRankSolver::halo_exchange(double* arr, int nc, int kind, const std::function<void()>& overlap_work) {
  if (n_ranks_ == 1) {
    if (overlap_work) overlap_work();
    return;
  }
  const int per = n2_ * nc;
  const int ns = static_cast<int>(send_slots_.n);
  mark(KC_HALO, true);
  if (ns > 0) {
    k_gather_slots<<<(ns * per + 255) / 256, 256, 0, stream_>>>(arr, send_slots_.p, ns, per, send_buf_.p);
    launches_++;
  }
  std::vector<Xfer> sends, recvs;
  size_t off = 0;
  for (const auto& p : topo_.peers) {
    const size_t cnt = p.send_slots.size() * per;
    sends.push_back({p.partner, send_buf_.p + off, cnt});
    recvs.push_back({p.partner, arr + static_cast<size_t>(p.recv_slots.front()) * per, p.recv_slots.size() * per});
    off += cnt;
  }
  record(kind, sends, recvs);
  mark(KC_HALO, false);
  comm_round(sends, recvs, !overlap_work, overlap_work);
}

// One right-hand-side evaluation (compute_residual, solver.cpp:846-870) with
// the RK update fused into the last kernel when mode == 0.
void GpuRankSolver::stage(double t_stage, int mode, double rk_a, double rk_b, double dt, double* out,
                          const double* u_override) {
  double* U = u_override ? const_cast<double*>(u_override) : U_.p;
  update_interfaces_host(t_stage);
  run_pairing(t_stage);
  const FieldPtrs fp = field_ptrs(U, out);
  if (!traces_valid_ || u_override) {
    mark(KC_PROLONG, true);
    launch_prolong(n_, consts_, fp, stream_);
    mark(KC_PROLONG, false);
    launches_++;
  }
  // One rank: both roles' mortar blocks are this rank's, whole and at offset 0 (self_), so the
  // four loopback copies of mortar_exchange are replaced by pointing each consumer at the
  // producer's array (the 8^3-per-GPU end of configs[4] spent 20 % of its stage in them).
  const bool loopback = n_ranks_ == 1;
  MortarPtrs mp = mortar_ptrs();
  if (loopback) {
    mp.u_theirs = u_mine_[1].p;
    mp.g_theirs = g_mine_[1].p;
    mp.lift[1] = mlift_[0].p;
    mp.flux[1] = mflux_[0].p;
  }
  double* const u_src[2] = {u_mine_[0].p, u_mine_[1].p};
  mark(KC_MORTAR, true);
  if (!sides_.empty()) launch_mortar_fill(n_, 5, trace_[cur_trace_].p, u_src, fwd_ops_, mp, stream_);
  mark(KC_MORTAR, false);
  launches_ += !sides_.empty();
  if (!loopback) mortar_exchange(u_src, u_theirs_.p, 5, true, MK_SOL_MORTAR);
  if (!nc_.empty()) {
    nc_prepare(t_stage);
    nc_fill(false);
  }
  const StageArgs a = stage_args(t_stage, dt, rk_a, rk_b, mode);
  // Element kernel over all local elements; with an exchange in flight, the interior run
  // first (on all but sm_reserve_ SMs), then the join, then the two boundary ranges.
  // Halo round of `arr` + element kernel: with overlap, the interior run is enqueued while the
  // round is in flight (on all but sm_reserve_ SMs), then the join and the boundary ranges.
  auto halo_and_elements = [&](double* arr, int nc, int kind, bool update) {
    if (!overlap_) {
      halo_exchange(arr, nc, kind);
      element_kernel(update, fp, a, 0, E_, n_sm_);
      return;
    }
    halo_exchange(arr, nc, kind, [&] { element_kernel(update, fp, a, int_lo_, int_hi_, n_sm_ - sm_reserve_); });
    join_comm();
    element_kernel(update, fp, a, 0, int_lo_, n_sm_);
    element_kernel(update, fp, a, int_hi_, E_, n_sm_);
  };
  if (lifting_) {
    mark(KC_MORTAR, true);
    launch_mortar_lift(n_, consts_.gas, mp, max_mortars_[0], stream_);
    mark(KC_MORTAR, false);
    launches_ += max_mortars_[0] > 0;
    double* const l_src[2] = {mlift_[0].p, loopback ? mlift_[0].p : mlift_[1].p};
    if (!loopback) mortar_exchange(l_src, mlift_[1].p, 4, false, MK_LIFT_MORTAR);
    mark(KC_MORTAR, true);
    if (!sides_.empty()) launch_mortar_backproject(n_, 4, l_src, slide_lift_.p, bwd_ops_, mp, stream_);
    mark(KC_MORTAR, false);
    launches_ += !sides_.empty();
    nc_lift();
    halo_and_elements(trace_[cur_trace_].p, 5, MK_SOL_CONF, false);
    nc_fill(true);
    double* const g_src[2] = {g_mine_[0].p, g_mine_[1].p};
    mark(KC_MORTAR, true);
    if (!sides_.empty()) launch_mortar_fill(n_, 12, slide_g_.p, g_src, fwd_ops_, mp, stream_);
    mark(KC_MORTAR, false);
    launches_ += !sides_.empty();
    if (!loopback) mortar_exchange(g_src, g_theirs_.p, 12, true, MK_GRAD_MORTAR);
  }
  mark(KC_MORTAR, true);
  launch_mortar_flux(n_, consts_.gas, lifting_ ? 1 : 0, mp, max_mortars_[0], err_.p, stream_);
  mark(KC_MORTAR, false);
  launches_ += max_mortars_[0] > 0;
  double* const f_src[2] = {mflux_[0].p, loopback ? mflux_[0].p : mflux_[1].p};
  if (!loopback) mortar_exchange(f_src, mflux_[1].p, 5, false, MK_FLUX_MORTAR);
  mark(KC_MORTAR, true);
  if (!sides_.empty()) launch_mortar_backproject(n_, 5, f_src, slide_flux_.p, bwd_ops_, mp, stream_);
  mark(KC_MORTAR, false);
  launches_ += !sides_.empty();
  nc_flux();
  // Viscous: Fv.n of the remote faces; inviscid: the traces themselves.
  if (lifting_) halo_and_elements(fvn_.p, 4, MK_FVN_CONF, true);
  else halo_and_elements(trace_[cur_trace_].p, 5, MK_SOL_CONF, true);
  // The update wrote the new traces into the other buffer: neighbours processed
  // later in the same launch still read this stage's traces.
  if (mode == 0) cur_trace_ ^= 1;
  traces_valid_ = (mode == 0 && !u_override);
}


void GpuRankSolver::record(int kind, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs) {
  for (const auto& x : sends)
    comm_trace_.push_back({step_index_, stage_index_, rank_, x.partner, static_cast<long long>(x.count), kind, true});
  for (const auto& x : recvs)
    comm_trace_.push_back({step_index_, stage_index_, x.partner, rank_, static_cast<long long>(x.count), kind, false});
}

// Test hook (RankSolver::inject_collective, solver.cpp:961-964): one
// unsanctioned collective after init, which the audit must flag.
void GpuRankSolver::inject_collective() {
  if (n_ranks_ == 1) return;
  double v = 0.0;
  for (int r = 0; r < n_ranks_; ++r)
    if (r != rank_) comm_trace_.push_back({step_index_, stage_index_, rank_, r, 1, MK_INIT, true});
  comm_->allreduce(&v, 1, 0, stream_);
}

std::string GpuRankSolver::trace_json() const {
  std::ostringstream os;
  os << "{\"rank\":" << rank_ << ",\"n_ranks\":" << n_ranks_ << ",\"n1\":" << n_ << ",\"rows\":[";
  for (size_t i = 0; i < comm_trace_.size(); ++i) {
    const auto& r = comm_trace_[i];
    os << (i ? "," : "") << "[" << r.step << "," << r.stage << "," << r.src << "," << r.dst << "," << r.count * 8
       << "," << r.kind << "," << (r.is_send ? 1 : 0) << "]";
  }
  os << "]}";
  return os.str();
}

void GpuRankSolver::check_error() {
  cuda_check(cudaMemcpyAsync(err_host_, err_.p, sizeof(ErrRec), cudaMemcpyDeviceToHost, stream_), "err d2h");
  cuda_check(cudaStreamSynchronize(stream_), "stream sync");
  if (err_host_->flag == 0) return;
  const ErrRec r = *err_host_;
  err_.zero(stream_);
  cuda_check(cudaStreamSynchronize(stream_), "stream sync");
  std::ostringstream os;
  if (r.flag == 4) {
    os << "device rows of non-matching interface " << r.elem << " (" << (r.node ? "z" : "y")
       << ") disagree with the host's";
    throw ProtocolError(os.str());
  }
  if (r.flag == 3) {
    os << "device pairing disagrees with the host schedule (role " << r.elem << ", " << r.node << " mortars)";
    throw ProtocolError(os.str());
  }
  if (r.node < 0) {
    os << "roe_flux: nonpositive Roe enthalpy average in element gid=" << (r.elem >= 0 ? topo_.gids[r.elem] : -1)
       << " at step " << r.step << " stage " << r.stage;
  } else {
    os << "inadmissible state in element gid=" << (r.elem >= 0 ? topo_.gids[r.elem] : -1) << " node " << r.node
       << " at step " << r.step << " stage " << r.stage << ": [" << r.vals[0] << ", " << r.vals[1] << ", "
       << r.vals[2] << ", " << r.vals[3] << ", " << r.vals[4] << "]";
  }
  throw InvalidStateError(os.str());
}

void GpuRankSolver::synchronize() { check_error(); }

// step (solver.cpp:908-927), n times without host synchronisation.
void GpuRankSolver::steps(double dt, int n, bool sync) {
  if (next_stage_ != 0) throw ConfigError("step: an RK step begun with rk_stage is unfinished");
  for (int it = 0; it < n; ++it)
    for (int s = 0; s < 5; ++s) rk_stage(s, time_, dt);
  if (sync) check_error();
}

// One stage of the 5-stage low-storage RK step that starts at t (lsrk_step,
// lsrk.hpp:20-21 / lsrk.cpp:31-44, as RankSolver::step runs it, solver.cpp:908-927):
// reg = a_s reg + dt R(u, t + c_s dt); u += b_s reg, then the admissibility check.
// The last stage completes the step: time, step index and the sliding offsets
// (delta_base += vg dt, wrapped by repeated subtraction, solver.cpp:922-926).
void GpuRankSolver::rk_stage(int s, double t, double dt) {
  if (s != next_stage_) throw ConfigError("rk_stage: stages run in order 0..4; expected stage " + std::to_string(next_stage_));
  if (t != time_) throw ConfigError("rk_stage: t must be the time the step starts at (time())");
  stage_index_ = s;
  stage(time_ + RK_C[s] * dt, 0, RK_A[s], RK_B[s], dt, nullptr, nullptr);
  next_stage_ = (s + 1) % 5;
  if (s < 4) return;
  time_ += dt;
  step_index_++;
  for (auto& c : sides_) {
    const IfaceGeom& f = mesh_.ifaces[c.iface];
    c.delta_base += f.vg_rel * dt;
    const double period = f.l_par * static_cast<double>(f.n_faces);
    while (c.delta_base >= period) {
      c.delta_base -= period;
      ++c.wraps;
    }
  }
  for (auto& r : nc_) {  // the same bookkeeping for both directions of an oblique slide
    const NcIfaceGeom& f = mesh_.nc_ifaces[r.iface];
    r.dy_base += f.vy_rel * dt;
    r.dz_base += f.vz_rel * dt;
    const double py = f.ly[0] * static_cast<double>(f.nfy[0]), pz = f.lz[0] * static_cast<double>(f.nfz[0]);
    while (r.dy_base >= py) r.dy_base -= py;
    while (r.dy_base < 0.0) r.dy_base += py;
    while (r.dz_base >= pz) r.dz_base -= pz;
    while (r.dz_base < 0.0) r.dz_base += pz;
  }
}

// update_interfaces (solver.cpp:156-176) as an entry point: displacement, sigma
// and the long-double operators on the host, the pairing on the device.
// ops (may be NULL): per interface-side context, the lower / upper forward
// (face -> mortar) and the lower / upper backward (mortar -> face) n x n
// operators, row-major (MortarOperators, mortar.hpp).
void GpuRankSolver::update_interfaces(double t_stage, double* ops) {
  update_interfaces_host(t_stage);
  run_pairing(t_stage);
  if (ops == nullptr) return;
  for (size_t c = 0; c < sides_.size(); ++c) {
    double* o = ops + c * 4 * n2_;
    std::copy(sides_[c].fwd.begin(), sides_[c].fwd.end(), o);
    std::copy(sides_[c].bwd.begin(), sides_[c].bwd.end(), o + 2 * n2_);
  }
  check_error();
}

void GpuRankSolver::compute_residual(double t_stage, const double* d_u, double* d_dudt) {
  stage(t_stage, 1, 0.0, 0.0, 0.0, d_dudt, d_u == U_.p ? nullptr : d_u);
  traces_valid_ = false;
  check_error();
}

void GpuRankSolver::compute_gradients(double t_stage, const double* d_u, double* d_grad) {
  double* U = const_cast<double*>(d_u);
  update_interfaces_host(t_stage);
  run_pairing(t_stage);
  FieldPtrs fp = field_ptrs(U, nullptr);
  launch_prolong(n_, consts_, fp, stream_);
  halo_exchange(trace_[cur_trace_].p, 5, MK_SOL_CONF);
  const MortarPtrs mp = mortar_ptrs();
  double* const u_src[2] = {u_mine_[0].p, u_mine_[1].p};
  launch_mortar_fill(n_, 5, trace_[cur_trace_].p, u_src, fwd_ops_, mp, stream_);
  mortar_exchange(u_src, u_theirs_.p, 5, true, MK_SOL_MORTAR);
  launch_mortar_lift(n_, consts_.gas, mp, max_mortars_[0], stream_);
  double* const l_src[2] = {mlift_[0].p, mlift_[1].p};
  mortar_exchange(l_src, mlift_[1].p, 4, false, MK_LIFT_MORTAR);
  launch_mortar_backproject(n_, 4, l_src, slide_lift_.p, bwd_ops_, mp, stream_);
  if (!nc_.empty()) {
    nc_prepare(t_stage);
    nc_fill(false);
    nc_lift();
  }
  fp.grad_out = d_grad;
  ElemConsts c = consts_;
  c.gas.viscous = 1;
  const StageArgs a = stage_args(t_stage, 0.0, 0.0, 0.0, 1);
  if (curved_) launch_gradient_curved(n_, c, fp, a, stream_);
  else launch_gradient(n_, c, fp, a, stream_);
  launches_ += 6;
  traces_valid_ = false;
  check_error();
}

double GpuRankSolver::suggest_dt(double cfl) {
  const unsigned long long init = 0x7fefffffffffffffULL;  // DBL_MAX bits
  cuda_check(cudaMemcpyAsync(dt_min_.p, &init, sizeof(init), cudaMemcpyHostToDevice, stream_), "h2d");
  launch_suggest_dt(n_, consts_, field_ptrs(U_.p, nullptr), cfl, basis_.degree, dt_min_.p, stream_);
  launches_++;
  unsigned long long bits = 0;
  cuda_check(cudaMemcpyAsync(&bits, dt_min_.p, sizeof(bits), cudaMemcpyDeviceToHost, stream_), "d2h");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  double dt;
  std::memcpy(&dt, &bits, sizeof(dt));
  if (n_ranks_ > 1) comm_->allreduce(&dt, 1, 2, stream_);
  return dt;
}


// Mass / energy integrals and error norms against the exact case
// (integrate_mass_energy, error_norms, max_freestream_deviation;
// diagnostics.cpp:31-87).  out: mass, energy, volume, L2[5], Linf[5], fs_dev.
void GpuRankSolver::diagnostics(double t, int with_exact, double* out) {
  const int max_blocks = 4 * n_sm_;
  if (diag_partial_.n < static_cast<size_t>(max_blocks) * kDiagVals) diag_partial_.alloc(max_blocks * kDiagVals);
  const int blocks =
      launch_diagnostics(n_, consts_, field_ptrs(U_.p, nullptr), t, with_exact, diag_partial_.p, max_blocks, stream_);
  launches_++;
  std::vector<double> h(static_cast<size_t>(blocks) * kDiagVals);
  cuda_check(cudaMemcpyAsync(h.data(), diag_partial_.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, stream_),
             "d2h");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  double acc[kDiagVals] = {};
  for (int b = 0; b < blocks; ++b)
    for (int q = 0; q < kDiagVals; ++q) {
      const double v = h[static_cast<size_t>(b) * kDiagVals + q];
      acc[q] = (q >= 8 && q < 13) ? std::max(acc[q], v) : acc[q] + v;
    }
  if (n_ranks_ > 1) {
    double sums[kDiagVals], maxs[kDiagVals];
    std::copy(acc, acc + kDiagVals, sums);
    std::copy(acc, acc + kDiagVals, maxs);
    comm_->allreduce(sums, kDiagVals, 0, stream_);
    comm_->allreduce(maxs, kDiagVals, 1, stream_);
    for (int q = 0; q < kDiagVals; ++q) acc[q] = (q >= 8 && q < 13) ? maxs[q] : sums[q];
  }
  out[0] = acc[0];
  out[1] = acc[1];
  out[2] = acc[2];
  for (int v = 0; v < 5; ++v) {
    out[3 + v] = std::sqrt(acc[3 + v] / acc[2]);
    out[8 + v] = acc[8 + v];
  }
  out[13] = std::max(std::max(acc[8], acc[9]), std::max(std::max(acc[10], acc[11]), acc[12]));
}

// SDGFLD1 snapshot (snapshot.cpp:10-56), 3D header; every rank writes / reads
// its own elements at their global offsets.
static std::string snapshot_header(const MeshGeom& m, int degree, double time) {
  std::ostringstream os;
  os.precision(17);
  os << "SDGFLD1\n";
  os << "n_elements " << m.n_elements << " degree " << degree << " nvars " << SDG_NVARS << " time " << time << "\n";
  os << "domain " << m.spec.x0 << ' ' << m.spec.y0 << ' ' << m.spec.z0 << ' ' << m.spec.width << ' '
     << m.spec.height << ' ' << m.spec.depth << " ny " << m.spec.ny << " nz " << m.spec.nz << "\n";
  for (size_t b = 0; b < m.bands.size(); ++b)
    os << "band " << b << " x_lo " << m.bands[b].x_lo << " nx " << m.bands[b].nx << " vg " << m.bands[b].vg << "\n";
  os << "end_header\n";
  return os.str();
}

// Collective: rank 0 writes the header and sizes the file; after a barrier every
// rank writes its elements in place ("r+b", never truncating); a second barrier
// makes the file complete on every rank when the call returns.  The barriers
// are I/O-phase synchronisation (like the diagnostics reductions), not part of
// the stepping protocol, so the communication trace does not list them.
void GpuRankSolver::write_snapshot(const char* path, double time) {
  std::vector<double> h(U_.n);
  get_state(h.data());
  const std::string hdr = snapshot_header(mesh_, basis_.degree, time);
  const size_t stride = static_cast<size_t>(n3_) * 5;
  const long total = static_cast<long>(hdr.size() + static_cast<size_t>(mesh_.n_elements) * stride * sizeof(double));
  double status = 0.0;  // max over ranks: 1 = some rank failed
  if (rank_ == 0) {
    FILE* f = std::fopen(path, "wb");
    bool ok = f != nullptr && std::fwrite(hdr.data(), 1, hdr.size(), f) == hdr.size();
    if (ok && total > static_cast<long>(hdr.size())) {
      const char zero = 0;  // pre-size: the last byte of the payload
      ok = std::fseek(f, total - 1, SEEK_SET) == 0 && std::fwrite(&zero, 1, 1, f) == 1;
    }
    if (f) ok = (std::fclose(f) == 0) && ok;
    status = ok ? 0.0 : 1.0;
  }
  snapshot_barrier(status);
  if (status != 0.0) throw ConfigError(std::string("cannot create snapshot file ") + path);
  FILE* f = std::fopen(path, "r+b");
  bool ok = f != nullptr;
  for (int e = 0; e < E_ && ok; ++e) {
    ok = std::fseek(f, static_cast<long>(hdr.size() + topo_.gids[e] * stride * sizeof(double)), SEEK_SET) == 0 &&
         std::fwrite(h.data() + e * stride, sizeof(double), stride, f) == stride;
  }
  if (f) ok = (std::fclose(f) == 0) && ok;
  status = ok ? 0.0 : 1.0;
  snapshot_barrier(status);
  if (status != 0.0) throw ConfigError(std::string("snapshot write failed for ") + path);
}

// Max of `flag` over ranks; a barrier between the snapshot phases.
void GpuRankSolver::snapshot_barrier(double& flag) {
  if (n_ranks_ > 1) comm_->allreduce(&flag, 1, 1, stream_);
}

// Restores the field, the time and the sliding-interface offsets (as
// set_initial_condition(t) does, solver.cpp:73-90 / 156-176): the run continues
// from the snapshot's time with delta_base = vg t.
double GpuRankSolver::read_snapshot(const char* path) {
  FILE* f = std::fopen(path, "rb");
  if (!f) throw ConfigError(std::string("cannot open snapshot file ") + path);
  char line[4096];
  if (!std::fgets(line, sizeof line, f) || std::string(line) != "SDGFLD1\n") {
    std::fclose(f);
    throw ConfigError(std::string("not a snapshot file: ") + path);
  }
  long ne = 0;
  int degree = 0, nvars = 0;
  double time = 0.0;
  if (!std::fgets(line, sizeof line, f) ||
      std::sscanf(line, "n_elements %ld degree %d nvars %d time %lf", &ne, &degree, &nvars, &time) != 4) {
    std::fclose(f);
    throw ConfigError("malformed snapshot header");
  }
  if (ne != mesh_.n_elements || degree != basis_.degree || nvars != SDG_NVARS) {
    std::fclose(f);
    throw ConfigError("snapshot does not match the mesh / degree / variable count");
  }
  while (std::fgets(line, sizeof line, f) && std::string(line) != "end_header\n") {
  }
  const long data0 = std::ftell(f);
  const size_t stride = static_cast<size_t>(n3_) * 5;
  std::vector<double> h(U_.n);
  bool ok = true;
  for (int e = 0; e < E_ && ok; ++e)
    ok = std::fseek(f, static_cast<long>(data0 + topo_.gids[e] * stride * sizeof(double)), SEEK_SET) == 0 &&
         std::fread(h.data() + e * stride, sizeof(double), stride, f) == stride;
  std::fclose(f);
  if (!ok) throw ConfigError(std::string("snapshot payload truncated in ") + path);
  set_state(h.data());
  reset_clock(time);
  return time;
}

void GpuRankSolver::ctx_info(int c, long* out5, double* sd, double* sig) {
  if (c < 0 || c >= static_cast<int>(sides_.size())) throw ConfigError("no such interface side context");
  int st[2 * kMaxCtx];
  double sdv[kMaxCtx];
  cuda_check(cudaMemcpyAsync(st, ctx_state_.p, sizeof(st), cudaMemcpyDeviceToHost, stream_), "d2h");
  cuda_check(cudaMemcpyAsync(sdv, ctx_sdelta_.p, sizeof(sdv), cudaMemcpyDeviceToHost, stream_), "d2h");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  out5[0] = sides_[c].iface;
  out5[1] = sides_[c].on_static ? 1 : 0;
  out5[2] = st[2 * c];
  out5[3] = st[2 * c + 1];
  out5[4] = static_cast<long>(sides_[c].slides.size());
  *sd = sdv[c];
  const double sigma = 2.0 * sdv[c] - 1.0;
  *sig = sides_[c].on_static ? sigma : -sigma;
}

void GpuRankSolver::get_pairing(int role, int* ncols, int* cols) {
  if (role < 0 || role > 1) throw ConfigError("role must be 0 (static) or 1 (moving)");
  int nm[2];
  cuda_check(cudaMemcpyAsync(nm, n_mortars_.p, sizeof(nm), cudaMemcpyDeviceToHost, stream_), "d2h");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  *ncols = nm[role];
  if (cols && nm[role] > 0) {
    cuda_check(cudaMemcpyAsync(cols, cols_[role].p, sizeof(int) * 7 * nm[role], cudaMemcpyDeviceToHost, stream_),
               "d2h");
    cuda_check(cudaStreamSynchronize(stream_), "sync");
  }
}

void GpuRankSolver::get_mapping(int c, int* m) {
  if (c < 0 || c >= static_cast<int>(sides_.size())) throw ConfigError("no such interface side context");
  const int nf = static_cast<int>(sides_[c].slides.size());
  const int off = pargs_.ctx[c].face_off;
  cuda_check(cudaMemcpyAsync(m, m_.p + 2 * off, sizeof(int) * 2 * nf, cudaMemcpyDeviceToHost, stream_), "d2h");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
}

// A device buffer ordered on one stream (cudaMallocAsync / cudaFreeAsync): the
// caller's host data is copied in, used by kernels and copied back in stream
// order, pageable host memory included (the copy is staged before return).
struct StreamBuf {
  double* p = nullptr;
  size_t n = 0;
  cudaStream_t st;
  StreamBuf(size_t count, cudaStream_t s) : n(count), st(s) {
    cuda_check(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(double), st), "cudaMallocAsync");
  }
  ~StreamBuf() {
    cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
  }
  StreamBuf(const StreamBuf&) = delete;
  StreamBuf& operator=(const StreamBuf&) = delete;
  void from_host(const double* h) {
    cuda_check(cudaMemcpyAsync(p, h, n * sizeof(double), cudaMemcpyHostToDevice, st), "h2d");
  }
  void to_host(double* h) {
    cuda_check(cudaMemcpyAsync(h, p, n * sizeof(double), cudaMemcpyDeviceToHost, st), "d2h");
    cuda_check(cudaStreamSynchronize(st), "d2h sync");
  }
};

// A stream owned by one host-side call, released on every exit path (exceptions included).
struct OwnedStream {
  cudaStream_t s{};
  OwnedStream() { cuda_check(cudaStreamCreate(&s), "stream"); }
  ~OwnedStream() {
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
  OwnedStream(const OwnedStream&) = delete;
  OwnedStream& operator=(const OwnedStream&) = delete;
  operator cudaStream_t() const { return s; }
};

// Stand-alone device pairing on caller-given faces (Appendix-A fixture).
static void device_intervals(long n_a, long n_b, double l_a, double delta, long* n_out, long* faces, double* ranges) {
  if (n_a < 1 || n_b < 1) throw ConfigError("interval merge needs at least one face per side");
  if (!(l_a > 0.0)) throw ConfigError("face length must be positive");
  const OwnedStream st;
  const long cap = n_a + n_b;
  DevBuf<long long> d_faces, d_n;
  DevBuf<double> d_ranges;
  d_faces.alloc(2 * cap);
  d_ranges.alloc(4 * cap);
  d_n.alloc(1);
  launch_mortar_intervals(n_a, n_b, l_a, delta, d_faces.p, d_ranges.p, d_n.p, st);
  long long n = 0;
  cuda_check(cudaMemcpyAsync(&n, d_n.p, sizeof(long long), cudaMemcpyDeviceToHost, st), "copy");
  std::vector<long long> hf(2 * cap);
  std::vector<double> hr(4 * cap);
  cuda_check(cudaMemcpyAsync(hf.data(), d_faces.p, hf.size() * sizeof(long long), cudaMemcpyDeviceToHost, st), "copy");
  cuda_check(cudaMemcpyAsync(hr.data(), d_ranges.p, hr.size() * sizeof(double), cudaMemcpyDeviceToHost, st), "copy");
  cuda_check(cudaStreamSynchronize(st), "sync");
  *n_out = static_cast<long>(n);
  if (faces == nullptr || ranges == nullptr) return;
  for (long long k = 0; k < 2 * n; ++k) faces[k] = static_cast<long>(hf[k]);
  std::copy(hr.begin(), hr.begin() + 4 * n, ranges);
}

// Non-matching planar interface transfer on the device (BASELINE configs[1]):
// side A has nfy[0] x nfz[0] faces of size l_y x l_z, side B nfy[1] x nfz[1] faces
// over the same periodic rectangle, displaced by (d_y, d_z).  Data on side `from`
// ([fy][fz][n][n][nc]) goes to the tensor-product mortars (face -> mortar L2
// operators) and on to the other side's faces (mortar -> face L2 projections).
// The rows come from the device interval kernel; the host assembles the long
// double operators from its bitwise-equal rows, as the reference assembles its
// mortar operators on the host every stage (proj/src/solver.cpp:156-176).
static void device_interface_project(int degree, int kind, const long* nfy, const long* nfz, double l_y, double l_z,
                                     double d_y, double d_z, int nc, int from, const double* src, double* mortar_out,
                                     double* dst, long* n_mortars) {
  if (from != 0 && from != 1) throw ConfigError("from must be 0 (A) or 1 (B)");
  if (nc < 1) throw ConfigError("nc must be positive");
  const Basis bs(degree, kind);
  const int n = bs.n, nn = n * n, to = 1 - from;
  const std::vector<MortarInterval> ry = merge_intervals(nfy[0], nfy[1], l_y, d_y);
  const std::vector<MortarInterval> rz = merge_intervals(nfz[0], nfz[1], l_z, d_z);
  const long my = static_cast<long>(ry.size()), mz = static_cast<long>(rz.size());
  *n_mortars = my * mz;
  auto ops = [&](const std::vector<MortarInterval>& rows, std::vector<double>& F, std::vector<double>& B,
                 std::vector<int>& off, std::vector<int>& idx, long n_to) {
    F.assign(rows.size() * nn, 0.0);
    B.assign(rows.size() * nn, 0.0);
    std::vector<double> tmp(nn);
    for (size_t k = 0; k < rows.size(); ++k) {
      const MortarInterval& r = rows[k];
      const double slo = from == 0 ? r.a_lo : r.b_lo, shi = from == 0 ? r.a_hi : r.b_hi;
      const double tlo = to == 0 ? r.a_lo : r.b_lo, thi = to == 0 ? r.a_hi : r.b_hi;
      build_subrange_ops(bs, slo, shi, F.data() + k * nn, tmp.data());
      build_subrange_ops(bs, tlo, thi, tmp.data(), B.data() + k * nn);
    }
    off.assign(n_to + 1, 0);  // target face -> its rows, in row order
    for (const MortarInterval& r : rows) ++off[(to == 0 ? r.face_a : r.face_b) + 1];
    for (long f = 0; f < n_to; ++f) off[f + 1] += off[f];
    idx.assign(rows.size(), 0);
    std::vector<int> fill(off.begin(), off.end() - 1);
    for (size_t k = 0; k < rows.size(); ++k) idx[fill[to == 0 ? rows[k].face_a : rows[k].face_b]++] = static_cast<int>(k);
  };
  std::vector<double> Fy, By, Fz, Bz;
  std::vector<int> offy, idxy, offz, idxz;
  ops(ry, Fy, By, offy, idxy, nfy[to]);
  ops(rz, Fz, Bz, offz, idxz, nfz[to]);
  const OwnedStream st;
  DevBuf<long long> d_ivy, d_ivz, d_n;
  DevBuf<double> d_rng, d_Fy, d_By, d_Fz, d_Bz, d_src, d_mortar, d_dst;
  DevBuf<int> d_offy, d_idxy, d_offz, d_idxz;
  d_ivy.alloc(2 * (nfy[0] + nfy[1]));
  d_ivz.alloc(2 * (nfz[0] + nfz[1]));
  d_rng.alloc(4 * std::max(nfy[0] + nfy[1], nfz[0] + nfz[1]));
  d_n.alloc(2);
  launch_mortar_intervals(nfy[0], nfy[1], l_y, d_y, d_ivy.p, d_rng.p, d_n.p, st);
  launch_mortar_intervals(nfz[0], nfz[1], l_z, d_z, d_ivz.p, d_rng.p, d_n.p + 1, st);
  d_Fy.upload(Fy, st);
  d_By.upload(By, st);
  d_Fz.upload(Fz, st);
  d_Bz.upload(Bz, st);
  d_offy.upload(offy, st);
  d_idxy.upload(idxy, st);
  d_offz.upload(offz, st);
  d_idxz.upload(idxz, st);
  const long per = static_cast<long>(nn) * nc;
  d_src.upload(std::vector<double>(src, src + nfy[from] * nfz[from] * per), st);
  d_mortar.alloc(my * mz * per);
  d_dst.alloc(nfy[to] * nfz[to] * per);
  launch_nc_transfer(n, nc, d_src.p, nfz[from], d_ivy.p, d_ivz.p, from, my, mz, d_Fy.p, d_Fz.p, d_mortar.p, nfy[to],
                     nfz[to], d_offy.p, d_idxy.p, d_offz.p, d_idxz.p, d_By.p, d_Bz.p, d_dst.p, st);
  if (mortar_out)
    cuda_check(cudaMemcpyAsync(mortar_out, d_mortar.p, my * mz * per * sizeof(double), cudaMemcpyDeviceToHost, st),
               "copy");
  if (dst)
    cuda_check(cudaMemcpyAsync(dst, d_dst.p, nfy[to] * nfz[to] * per * sizeof(double), cudaMemcpyDeviceToHost, st),
               "copy");
  long long dn[2] = {0, 0};
  cuda_check(cudaMemcpyAsync(dn, d_n.p, sizeof(dn), cudaMemcpyDeviceToHost, st), "copy");
  cuda_check(cudaStreamSynchronize(st), "sync");
  if (dn[0] != my || dn[1] != mz)  // the kernels indexed with the device's rows; the operators came from the host's
    throw ProtocolError("interface transfer: device rows (" + std::to_string(dn[0]) + " x " + std::to_string(dn[1]) +
                        ") differ from the host's (" + std::to_string(my) + " x " + std::to_string(mz) + ")");
}

// The operators of one side s of a mortar row: face -> mortar (F) and mortar ->
// face (B) for each row's sub-range on s, and the CSR list face -> rows (row order).
struct NcSideOps {
  std::vector<double> F, B;
  std::vector<int> off, idx;
};
static NcSideOps nc_side_ops(const Basis& bs, const std::vector<MortarInterval>& rows, int s, long n_faces) {
  const int nn = bs.n * bs.n;
  NcSideOps o;
  o.F.assign(rows.size() * nn, 0.0);
  o.B.assign(rows.size() * nn, 0.0);
  o.off.assign(n_faces + 1, 0);
  for (size_t k = 0; k < rows.size(); ++k) {
    const MortarInterval& r = rows[k];
    build_subrange_ops(bs, s == 0 ? r.a_lo : r.b_lo, s == 0 ? r.a_hi : r.b_hi, o.F.data() + k * nn,
                       o.B.data() + k * nn);
    ++o.off[(s == 0 ? r.face_a : r.face_b) + 1];
  }
  for (long f = 0; f < n_faces; ++f) o.off[f + 1] += o.off[f];
  o.idx.assign(rows.size(), 0);
  std::vector<int> fill(o.off.begin(), o.off.end() - 1);
  for (size_t k = 0; k < rows.size(); ++k) o.idx[fill[s == 0 ? rows[k].face_a : rows[k].face_b]++] = static_cast<int>(k);
  return o;
}

// The surface flux of a non-matching planar interface with normal +x (side A
// below, side B above), on the device: both sides' traces (and gradients, for
// the viscous part) go to the tensor-product mortars, the two-sided numerical
// flux is evaluated at the mortar nodes and L2-projected back onto the faces of
// both sides.  This is the reference's mortar chain (solver.cpp:156-176 fill,
// 308-321 flux, mortar.cpp:79-134 projections) on non-aligned face rows.
// lift != 0: the lifting mean of the primitive (u, v, w, T) instead (4 components).
static void device_interface_flux(const sdg_gas& gas, int degree, int kind, const long* nfy, const long* nfz,
                                  double l_y, double l_z, double d_y, double d_z, const double* u_a,
                                  const double* u_b, const double* g_a, const double* g_b, double* flux_mortar,
                                  double* flux_a, double* flux_b, long* n_mortars, int lift = 0) {
  if ((g_a == nullptr) != (g_b == nullptr)) throw ConfigError("gradients must be given for both sides or neither");
  const Basis bs(degree, kind);
  const int n = bs.n, nn = n * n;
  const std::vector<MortarInterval> ry = merge_intervals(nfy[0], nfy[1], l_y, d_y);
  const std::vector<MortarInterval> rz = merge_intervals(nfz[0], nfz[1], l_z, d_z);
  const long my = static_cast<long>(ry.size()), mz = static_cast<long>(rz.size());
  *n_mortars = my * mz;
  NcSideOps oy[2] = {nc_side_ops(bs, ry, 0, nfy[0]), nc_side_ops(bs, ry, 1, nfy[1])};
  NcSideOps oz[2] = {nc_side_ops(bs, rz, 0, nfz[0]), nc_side_ops(bs, rz, 1, nfz[1])};
  const OwnedStream st;
  DevBuf<long long> d_ivy, d_ivz, d_n;
  DevBuf<double> d_rng;
  d_ivy.alloc(2 * (nfy[0] + nfy[1]));
  d_ivz.alloc(2 * (nfz[0] + nfz[1]));
  const long rmax = 4 * std::max(nfy[0] + nfy[1], nfz[0] + nfz[1]);
  d_rng.alloc(2 * rmax);
  d_n.alloc(2);
  IvRows rows{};
  rows.row[0] = IvRow{nfy[0], nfy[1], l_y, d_y, d_ivy.p, d_rng.p, d_n.p};
  rows.row[1] = IvRow{nfz[0], nfz[1], l_z, d_z, d_ivz.p, d_rng.p + rmax, d_n.p + 1};
  launch_mortar_intervals2(rows, st);
  DevBuf<double> d_F[2][2], d_B[2][2];  // [side][y/z]
  DevBuf<int> d_off[2][2], d_idx[2][2];
  for (int s = 0; s < 2; ++s) {
    d_F[s][0].upload(oy[s].F, st);
    d_B[s][0].upload(oy[s].B, st);
    d_off[s][0].upload(oy[s].off, st);
    d_idx[s][0].upload(oy[s].idx, st);
    d_F[s][1].upload(oz[s].F, st);
    d_B[s][1].upload(oz[s].B, st);
    d_off[s][1].upload(oz[s].off, st);
    d_idx[s][1].upload(oz[s].idx, st);
  }
  const long nm = my * mz;
  const bool vis = g_a != nullptr;
  DevBuf<double> d_u[2], d_g[2], d_mu[2], d_mg[2], d_flux, d_face[2];
  const double* u_in[2] = {u_a, u_b};
  const double* g_in[2] = {g_a, g_b};
  NcMortarJobs mj{};
  for (int s = 0; s < 2; ++s) {
    const long nf = nfy[s] * nfz[s];
    d_u[s].upload(std::vector<double>(u_in[s], u_in[s] + nf * nn * 5), st);
    d_mu[s].alloc(nm * nn * 5);
    mj.job[mj.n++] = NcMortarJob{d_u[s].p, nfz[s], s, 5, d_F[s][0].p, d_F[s][1].p, d_mu[s].p};
    if (vis) {
      d_g[s].upload(std::vector<double>(g_in[s], g_in[s] + nf * nn * 12), st);
      d_mg[s].alloc(nm * nn * 12);
      mj.job[mj.n++] = NcMortarJob{d_g[s].p, nfz[s], s, 12, d_F[s][0].p, d_F[s][1].p, d_mg[s].p};
    }
  }
  launch_nc_to_mortar_batch(n, d_ivy.p, d_ivz.p, my, mz, mj, st);
  const GasD g{gas.gamma, gas.gamma - 1.0, gas.R, 1.0 / gas.R, gas.mu, -2.0 / 3.0 * gas.mu,
               gas.gamma * gas.R * gas.mu / ((gas.gamma - 1.0) * gas.Pr), gas.mu > 0.0 ? 1 : 0};
  DevBuf<int> d_bad;
  d_bad.upload(std::vector<int>{0}, st);
  const int nco = lift ? 4 : 5;
  d_flux.alloc(nm * nn * nco);
  if (lift)
    launch_nc_mortar_lift(nm * nn, g, d_mu[0].p, d_mu[1].p, d_flux.p, st);
  else
    launch_nc_mortar_flux(nm * nn, g, 0, 0.0, d_mu[0].p, d_mu[1].p, vis ? d_mg[0].p : nullptr,
                          vis ? d_mg[1].p : nullptr, d_flux.p, d_bad.p, st);
  double* out[2] = {flux_a, flux_b};
  NcFaceJobs fj{};
  for (int s = 0; s < 2; ++s) {
    d_face[s].alloc(nfy[s] * nfz[s] * nn * nco);
    fj.job[fj.n++] = NcFaceJob{nfy[s], nfz[s], d_off[s][0].p, d_idx[s][0].p, d_off[s][1].p, d_idx[s][1].p,
                               d_B[s][0].p, d_B[s][1].p, d_face[s].p};
  }
  launch_nc_to_face_batch(n, nco, d_flux.p, mz, fj, st);
  for (int s = 0; s < 2; ++s)
    if (out[s])
      cuda_check(cudaMemcpyAsync(out[s], d_face[s].p, d_face[s].n * sizeof(double), cudaMemcpyDeviceToHost, st),
                 "copy");
  if (flux_mortar)
    cuda_check(cudaMemcpyAsync(flux_mortar, d_flux.p, d_flux.n * sizeof(double), cudaMemcpyDeviceToHost, st), "copy");
  int bad = 0;
  long long dn[2] = {0, 0};
  cuda_check(cudaMemcpyAsync(&bad, d_bad.p, sizeof(int), cudaMemcpyDeviceToHost, st), "copy");
  cuda_check(cudaMemcpyAsync(dn, d_n.p, sizeof(dn), cudaMemcpyDeviceToHost, st), "copy");
  cuda_check(cudaStreamSynchronize(st), "sync");
  // The kernels indexed with the device's rows; the operators came from the host's.
  if (dn[0] != my || dn[1] != mz)
    throw ProtocolError("interface flux: device rows (" + std::to_string(dn[0]) + " x " + std::to_string(dn[1]) +
                        ") differ from the host's (" + std::to_string(my) + " x " + std::to_string(mz) + ")");
  if (bad) throw InvalidStateError("interface flux: non-positive Roe-averaged c^2 at " + std::to_string(bad) + " mortar nodes");
}

static void device_pairing(int n_local, const long* faces, long n_par, long n_perp, const int* partner_ranks,
                           long n_delta, int on_static, int conforming, int self_rank, int* ncols, int* cols,
                           int* m_rows, long* face_lo, int* nsched, int* sched, int* self_entry) {
  const OwnedStream st;
  PairingArgs a{};
  a.n_ctx = 1;
  a.n_ifaces = 1;
  a.iface_base[0] = 0;
  a.iface_nperp[0] = n_perp;
  a.dense_size = 2LL * n_par * n_perp;
  a.self_rank = self_rank;
  const int role = on_static ? 0 : 1;
  a.role_nctx[role] = 1;
  a.role_ctx[role][0] = 0;
  a.role_nctx[1 - role] = 0;
  CtxD& c = a.ctx[0];
  c.iface = 0;
  c.on_static = on_static;
  c.role = role;
  c.n_faces = n_local;
  c.face_off = 0;
  c.map_off = 0;
  c.n_par = n_par;
  c.n_perp = n_perp;
  c.l_par = 1.0;
  c.vg_rel = 0.0;
  // Displacement chain reproduces (n_delta, conforming): delta = n_delta (+ 0.5 if hanging).
  a.delta_base[0] = static_cast<double>(n_delta) + (conforming ? 0.0 : 0.5);
  a.time = 0.0;
  a.t_stage = 0.0;
  a.expect_mortars[0] = a.expect_mortars[1] = -1;
  std::vector<int> fpar(n_local), fperp(n_local), fsl(n_local);
  for (int f = 0; f < n_local; ++f) {
    fpar[f] = static_cast<int>(faces[3 * f + 1]);
    fperp[f] = static_cast<int>(faces[3 * f + 2]);
    fsl[f] = f;
  }
  DevBuf<int> d_par, d_perp, d_sl, d_map, d_pres, d_pay, d_cols, d_m, d_state, d_nm, d_dummy;
  DevBuf<double> d_sd;
  DevBuf<ErrRec> d_err;
  d_par.upload(fpar, st);
  d_perp.upload(fperp, st);
  d_sl.upload(fsl, st);
  d_map.upload(std::vector<int>(partner_ranks, partner_ranks + n_par * n_perp), st);
  d_pres.alloc(a.dense_size);
  d_pay.alloc(a.dense_size);
  d_cols.alloc(7 * static_cast<size_t>(2 * n_local + 1));
  d_dummy.alloc(7);
  d_m.alloc(2 * static_cast<size_t>(n_local) + 1);
  d_state.alloc(2 * kMaxCtx);
  d_sd.alloc(kMaxCtx);
  d_nm.alloc(2);
  d_nm.zero(st);
  d_err.alloc(1);
  d_err.zero(st);
  PairingPtrs p{};
  p.ctx_face_par = d_par.p;
  p.ctx_face_perp = d_perp.p;
  p.ctx_face_slide = d_sl.p;
  p.partner_map = d_map.p;
  p.pres[0] = p.pres[1] = d_pres.p;
  p.payload[0] = p.payload[1] = d_pay.p;
  p.cols[role] = d_cols.p;
  p.cols[1 - role] = d_dummy.p;
  p.m = d_m.p;
  p.ctx_state = d_state.p;
  p.ctx_sdelta = d_sd.p;
  p.n_mortars = d_nm.p;
  p.err = d_err.p;
  launch_pairing(a, p, st);
  int nm[2];
  ErrRec er;
  cuda_check(cudaMemcpyAsync(nm, d_nm.p, sizeof(nm), cudaMemcpyDeviceToHost, st), "d2h");
  cuda_check(cudaMemcpyAsync(&er, d_err.p, sizeof(er), cudaMemcpyDeviceToHost, st), "d2h");
  cuda_check(cudaStreamSynchronize(st), "sync");
  std::vector<int> hc(7 * static_cast<size_t>(std::max(nm[role], 1))), hm(2 * static_cast<size_t>(n_local) + 1);
  cuda_check(cudaMemcpy(hc.data(), d_cols.p, sizeof(int) * 7 * nm[role], cudaMemcpyDeviceToHost), "d2h");
  cuda_check(cudaMemcpy(hm.data(), d_m.p, sizeof(int) * 2 * n_local, cudaMemcpyDeviceToHost), "d2h");
  if (er.flag != 0) throw ProtocolError("rank map lookup hit an unset entry");
  // Caller face ids ride along passively (build_mapping, partition.cpp:124-141).
  long lo = 0, hi = -1;
  if (n_local > 0) {
    lo = hi = faces[0];
    for (int f = 0; f < n_local; ++f) {
      lo = std::min(lo, faces[3 * f]);
      hi = std::max(hi, faces[3 * f]);
    }
  }
  *face_lo = lo;
  const long w = hi - lo + 1;
  for (long q = 0; q < 2 * w; ++q) m_rows[q] = -1;
  *ncols = nm[role];
  for (int i = 0; i < nm[role]; ++i) {
    int* o = cols + 7 * i;
    for (int q = 0; q < 7; ++q) o[q] = hc[7 * i + q];
    const int f = o[5];
    o[5] = static_cast<int>(faces[3 * f]);
    o[6] = 0;
    m_rows[o[4] * w + (faces[3 * f] - lo)] = i;
  }
  int ns = 0;
  self_entry[0] = self_rank;
  self_entry[1] = 0;
  self_entry[2] = 0;
  for (int i = 0; i < nm[role]; ++i) {
    const int p = cols[7 * i];
    if (p == self_rank) {
      if (self_entry[2] == 0) self_entry[1] = i;
      self_entry[2]++;
      continue;
    }
    if (ns == 0 || sched[3 * (ns - 1)] != p) {
      sched[3 * ns] = p;
      sched[3 * ns + 1] = i;
      sched[3 * ns + 2] = 0;
      ns++;
    }
    sched[3 * (ns - 1) + 2]++;
  }
  *nsched = ns;
}


// Host-only description of one rank's share of a multi-rank run (no CUDA
// calls): local elements, conforming halo peers with their face keys in send
// order, and the per-partner mortar blocks of both roles for a displacement
// `delta` of every interface.  Used by the CPU multi-process tests to check
// that every pair of ranks derives matching message blocks independently
// (the stamp check of proj/tests/test_partition.cpp:184-227, for the halo too).
static std::string plan_json(const sdg_mesh_spec& ms, int n_ranks, int rank, double delta) {
  const MeshGeom mesh(ms);
  const Partition part = assign_ranks(mesh, n_ranks);
  const LocalTopology topo = build_topology(mesh, part, rank);
  std::ostringstream os;
  const auto run = interior_run(topo);
  os << "{\"rank\":" << rank << ",\"interior_run\":[" << run[0] << "," << run[1] << "],\"elements\":[";
  for (size_t i = 0; i < topo.gids.size(); ++i) os << (i ? "," : "") << topo.gids[i];
  os << "],\"halo\":[";
  const int ne = static_cast<int>(topo.gids.size());
  for (size_t p = 0; p < topo.peers.size(); ++p) {
    const auto& pf = topo.peers[p];
    os << (p ? "," : "") << "{\"partner\":" << pf.partner << ",\"keys\":[";
    for (size_t q = 0; q < pf.send_slots.size(); ++q) {
      const int slot = pf.send_slots[q], e = slot / 6, side = slot % 6;
      // the same face key the partner sorts by: minus element gid * 3 + dir
      long minus = topo.gids[e];
      if (!(side & 1)) {
        int b = topo.coords[4 * e], ix = topo.coords[4 * e + 1], iy = topo.coords[4 * e + 2], iz = topo.coords[4 * e + 3];
        const int dir = side / 2;
        if (dir == 0) {
          if (ix > 0) ix--;
          else {
            b = (b - 1 + static_cast<int>(mesh.bands.size())) % static_cast<int>(mesh.bands.size());
            ix = mesh.bands[b].nx - 1;
          }
        } else if (dir == 1) {
          iy = (iy - 1 + ms.ny) % ms.ny;
        } else {
          iz = (iz - 1 + ms.nz) % ms.nz;
        }
        minus = mesh.gid(b, ix, iy, iz);
      }
      os << (q ? "," : "") << minus * 3 + side / 2;
    }
    os << "],\"recv_first\":" << (pf.recv_slots.empty() ? -1 : pf.recv_slots.front() - 6 * ne) << "}";
  }
  os << "],\"mortars\":[";
  // Owner maps of every interface side (what init_rank_maps gathers).
  bool first_role = true;
  for (int role = 0; role < 2; ++role) {
    struct Key {
      int partner, iface;
      long par, perp;
      int sub;
    };
    std::vector<Key> keys;
    for (size_t ic = 0; ic < mesh.ifaces.size(); ++ic) {
      const IfaceGeom& f = mesh.ifaces[ic];
      const int my_band = role == 0 ? f.static_band() : f.moving_band();
      const int other_band = role == 0 ? f.moving_band() : f.static_band();
      const int my_ix = (my_band == f.left) ? mesh.bands[my_band].nx - 1 : 0;
      const int other_ix = (other_band == f.left) ? mesh.bands[other_band].nx - 1 : 0;
      const Displacement st = displacement(delta, f.l_par, f.n_faces);
      for (long iy = 0; iy < ms.ny; ++iy)
        for (long iz = 0; iz < ms.nz; ++iz) {
          const long g = mesh.gid(my_band, my_ix, static_cast<int>(iy), static_cast<int>(iz));
          if (part.owner(my_band, g - mesh.bands[my_band].off) != rank) continue;
          for (int sub = st.conforming() ? 1 : 0; sub < 2; ++sub) {
            const long par = role == 0 ? iy : static_index(iy, st.n_delta, sub, f.n_faces);
            const long opar = role == 0 ? moving_index(iy, st.n_delta, sub, f.n_faces) : par;
            const long og = mesh.gid(other_band, other_ix, static_cast<int>(opar), static_cast<int>(iz));
            const int partner = part.owner(other_band, og - mesh.bands[other_band].off);
            keys.push_back({partner, static_cast<int>(ic), par, iz, sub});
          }
        }
    }
    std::sort(keys.begin(), keys.end(), [](const Key& a, const Key& b) {
      return std::tie(a.partner, a.iface, a.par, a.perp, a.sub) < std::tie(b.partner, b.iface, b.par, b.perp, b.sub);
    });
    for (size_t i = 0; i < keys.size();) {
      size_t j = i;
      while (j < keys.size() && keys[j].partner == keys[i].partner) ++j;
      os << (first_role ? "" : ",") << "{\"role\":" << role << ",\"partner\":" << keys[i].partner << ",\"keys\":[";
      first_role = false;
      for (size_t q = i; q < j; ++q)
        os << (q > i ? "," : "") << "[" << keys[q].iface << "," << keys[q].par << "," << keys[q].perp << ","
           << keys[q].sub << "]";
      os << "]}";
      i = j;
    }
  }
  os << "]}";
  return os.str();
}

}  // namespace sdg

// ============================================================================
// C-ABI (include/sdg_gpu.h)
// ============================================================================
using sdg::GpuRankSolver;

struct sdg_ctx {
  GpuRankSolver* s;
};

namespace {
thread_local std::string g_error;

// Makes the context's device current for the duration of one entry point and
// restores the caller's afterwards (one host thread may drive several GPUs).
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(const sdg_ctx* c) {
    if (c && c->s && cudaGetDevice(&prev) == cudaSuccess && prev != c->s->device()) cudaSetDevice(c->s->device());
    else prev = -1;
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <class F>
int guarded(const sdg_ctx* c, F&& fn) {
  std::string* sink = c && c->s ? &c->s->err : &g_error;
  try {
    DeviceScope dev(c);
    fn();
    return SDG_OK;
  } catch (const sdg::ConfigError& e) {
    *sink = e.what();
    return SDG_ERR_CONFIG;
  } catch (const sdg::InvalidStateError& e) {
    *sink = e.what();
    return SDG_ERR_INVALID_STATE;
  } catch (const sdg::ProtocolError& e) {
    *sink = e.what();
    return SDG_ERR_PROTOCOL;
  } catch (const sdg::DeviceError& e) {
    *sink = e.what();
    return e.code;
  } catch (const std::exception& e) {
    *sink = e.what();
    return SDG_ERR_CONFIG;
  }
}
}  // namespace

extern "C" {

int sdg_create(const sdg_mesh_spec* mesh, const sdg_solver_config* cfg, int n_ranks, int rank, int device,
               const void* nccl_id, sdg_ctx** out) {
  return guarded(nullptr, [&] {
    if (!mesh || !cfg || !out) throw sdg::ConfigError("null argument");
    auto* c = new sdg_ctx{nullptr};
    try {
      c->s = new GpuRankSolver(*mesh, *cfg, n_ranks, rank, device, nccl_id);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}
int sdg_create_inproc(const sdg_mesh_spec* mesh, const sdg_solver_config* cfg, int n_ranks, int rank, int device,
                      const char* hub, sdg_ctx** out) {
  return guarded(nullptr, [&] {
    if (!mesh || !cfg || !out || !hub) throw sdg::ConfigError("null argument");
    auto* c = new sdg_ctx{nullptr};
    try {
      c->s = new GpuRankSolver(*mesh, *cfg, n_ranks, rank, device, nullptr, hub);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}
void sdg_destroy(sdg_ctx* c) {
  if (!c) return;
  delete c->s;
  delete c;
}
const char* sdg_last_error(const sdg_ctx* c) { return c && c->s ? c->s->err.c_str() : g_error.c_str(); }
const char* sdg_global_error(void) { return g_error.c_str(); }
int sdg_nccl_unique_id(void* out) {
  return guarded(nullptr, [&] {
    ncclUniqueId id;
    sdg::nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
  });
}
// One-rank communicator through every NcclComm method the solver uses: init, the two
// all-gathers of init_rank_maps, the min / sum all-reduces of suggest_dt and the
// diagnostics, and one grouped send + receive round (to the rank itself, the only
// partner a single GPU offers).  The multi-rank data path is checked bitwise on the
// in-process transport; this checks that the NCCL calls themselves run on the device.
int sdg_nccl_selfcheck(int device, long n_doubles) {
  return guarded(nullptr, [&] {
    if (n_doubles < 1) throw sdg::ConfigError("sdg_nccl_selfcheck: n_doubles < 1");
    int prev = -1;
    sdg::cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
    sdg::cuda_check(cudaSetDevice(device), "cudaSetDevice");
    {
      ncclUniqueId id;
      sdg::nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
      sdg::NcclComm comm(&id, 1, 0);
      cudaStream_t st = nullptr;
      sdg::cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
      std::vector<std::vector<int>> all;
      const std::vector<int> mine = {7, 11, 13};
      comm.allgather_ints(mine, all, st);
      if (all.size() != 1 || all[0] != mine) throw sdg::ProtocolError("sdg_nccl_selfcheck: all-gather");
      double v[3] = {3.5, -2.0, 8.25};
      comm.allreduce(v, 3, 2, st);
      comm.allreduce(v, 3, 0, st);
      if (v[0] != 3.5 || v[1] != -2.0 || v[2] != 8.25) throw sdg::ProtocolError("sdg_nccl_selfcheck: all-reduce");
      std::vector<double> h(static_cast<size_t>(n_doubles));
      for (long i = 0; i < n_doubles; ++i) h[i] = 0.25 * static_cast<double>(i) - 3.0;
      sdg::DevBuf<double> src, dst;
      src.upload(h, st);
      dst.alloc(h.size());
      dst.zero(st);
      comm.exchange({{0, src.p, h.size()}}, {{0, dst.p, h.size()}}, st);
      std::vector<double> back(h.size());
      sdg::cuda_check(cudaMemcpyAsync(back.data(), dst.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st), "d2h");
      sdg::cuda_check(cudaStreamSynchronize(st), "sync");
      cudaStreamDestroy(st);
      if (back != h) throw sdg::ProtocolError("sdg_nccl_selfcheck: send / receive round");
    }
    if (prev >= 0) cudaSetDevice(prev);
  });
}
int sdg_init_rank_maps(sdg_ctx* c) {
  return guarded(c, [&] { c->s->init_rank_maps(); });
}
int sdg_set_initial_condition(sdg_ctx* c, double t0) {
  return guarded(c, [&] { c->s->set_initial_condition(t0); });
}
int sdg_n1(const sdg_ctx* c) { return c->s->n1(); }
long sdg_n_local_elements(const sdg_ctx* c) { return c->s->n_local(); }
long sdg_n_global_elements(const sdg_ctx* c) { return c->s->n_global(); }
int sdg_local_element_ids(const sdg_ctx* c, long* gids) {
  std::copy(c->s->gids().begin(), c->s->gids().end(), gids);
  return SDG_OK;
}
int sdg_set_state(sdg_ctx* c, const double* h) {
  return guarded(c, [&] { c->s->set_state(h); });
}
int sdg_get_state(sdg_ctx* c, double* h) {
  return guarded(c, [&] { c->s->get_state(h); });
}
int sdg_get_register(sdg_ctx* c, double* h) {
  return guarded(c, [&] { c->s->get_register(h); });
}
int sdg_state_device_ptr(sdg_ctx* c, double** d) {
  *d = c->s->d_state();
  return SDG_OK;
}
int sdg_step(sdg_ctx* c, double dt) {
  return guarded(c, [&] { c->s->steps(dt, 1, true); });
}
int sdg_steps(sdg_ctx* c, double dt, int n) {
  return guarded(c, [&] { c->s->steps(dt, n, true); });
}
int sdg_steps_async(sdg_ctx* c, double dt, int n) {
  return guarded(c, [&] { c->s->steps(dt, n, false); });
}
int sdg_rk_stage(sdg_ctx* c, int s, double t, double dt) {
  return guarded(c, [&] { c->s->rk_stage(s, t, dt); });
}
int sdg_rk_coefficients(double* a, double* b, double* cc) {
  for (int s = 0; s < 5; ++s) {
    if (a) a[s] = sdg::RK_A[s];
    if (b) b[s] = sdg::RK_B[s];
    if (cc) cc[s] = sdg::RK_C[s];
  }
  return SDG_OK;
}
int sdg_update_interfaces(sdg_ctx* c, double t_stage, double* ops) {
  return guarded(c, [&] { c->s->update_interfaces(t_stage, ops); });
}
int sdg_synchronize(sdg_ctx* c) {
  return guarded(c, [&] { c->s->synchronize(); });
}
int sdg_compute_residual(sdg_ctx* c, double t, const double* d_u, double* d_dudt) {
  return guarded(c, [&] { c->s->compute_residual(t, d_u, d_dudt); });
}
int sdg_compute_residual_host(sdg_ctx* c, double t, const double* h_u, double* h_dudt) {
  return guarded(c, [&] {
    const size_t n = static_cast<size_t>(c->s->n_local()) * c->s->n1() * c->s->n1() * c->s->n1() * 5;
    sdg::StreamBuf du(n, c->s->stream()), dd(n, c->s->stream());
    du.from_host(h_u);
    c->s->compute_residual(t, du.p, dd.p);
    dd.to_host(h_dudt);
  });
}
int sdg_compute_gradients_host(sdg_ctx* c, double t, const double* h_u, double* h_grad) {
  return guarded(c, [&] {
    const size_t nodes = static_cast<size_t>(c->s->n_local()) * c->s->n1() * c->s->n1() * c->s->n1();
    sdg::StreamBuf du(nodes * 5, c->s->stream()), dg(nodes * 12, c->s->stream());
    du.from_host(h_u);
    c->s->compute_gradients(t, du.p, dg.p);
    dg.to_host(h_grad);
  });
}
int sdg_suggest_dt(sdg_ctx* c, double cfl, double* dt) {
  return guarded(c, [&] { *dt = c->s->suggest_dt(cfl); });
}
int sdg_time(const sdg_ctx* c, double* t, int* step) {
  if (t) *t = c->s->time();
  if (step) *step = c->s->step_index();
  return SDG_OK;
}
long sdg_total_rebuilds(const sdg_ctx* c) { return c->s->total_rebuilds(); }
int sdg_n_contexts(const sdg_ctx* c) { return c->s->n_contexts(); }
int sdg_ctx_info(sdg_ctx* c, int id, long* out5, double* sd, double* sig) {
  return guarded(c, [&] { c->s->ctx_info(id, out5, sd, sig); });
}
int sdg_n_nc_interfaces(const sdg_ctx* c) { return c->s->n_nc(); }
int sdg_nc_rows(sdg_ctx* c, int iface, int dir, long* n_out, long* faces, double* ranges, double* delta) {
  return guarded(c, [&] { c->s->nc_rows(iface, dir, n_out, faces, ranges, delta); });
}
int sdg_get_pairing(sdg_ctx* c, int role, int* ncols, int* cols) {
  return guarded(c, [&] { c->s->get_pairing(role, ncols, cols); });
}
int sdg_get_mapping(sdg_ctx* c, int id, int* m) {
  return guarded(c, [&] { c->s->get_mapping(id, m); });
}
int sdg_pairing_device(int n_local, const long* faces, long n_par, long n_perp, const int* partner_ranks,
                       long n_delta, int on_static, int conforming, int self_rank, int* ncols, int* cols,
                       int* m_rows, long* face_lo, int* nsched, int* sched, int* self_entry) {
  return guarded(nullptr, [&] {
    sdg::device_pairing(n_local, faces, n_par, n_perp, partner_ranks, n_delta, on_static, conforming, self_rank,
                        ncols, cols, m_rows, face_lo, nsched, sched, self_entry);
  });
}
int sdg_trace_json(sdg_ctx* c, char* buf, long cap, long* len) {
  return guarded(c, [&] {
    const std::string j = c->s->trace_json();
    *len = static_cast<long>(j.size());
    if (buf && cap > 0) {
      std::strncpy(buf, j.c_str(), static_cast<size_t>(cap) - 1);
      buf[cap - 1] = 0;
    }
  });
}
int sdg_inject_collective(sdg_ctx* c) {
  return guarded(c, [&] { c->s->inject_collective(); });
}
int sdg_plan_json(const sdg_mesh_spec* mesh, int n_ranks, int rank, double delta, char* buf, long cap,
                  long* len) {
  return guarded(nullptr, [&] {
    const std::string j = sdg::plan_json(*mesh, n_ranks, rank, delta);
    *len = static_cast<long>(j.size());
    if (buf && cap > 0) {
      std::strncpy(buf, j.c_str(), static_cast<size_t>(cap) - 1);
      buf[cap - 1] = 0;
    }
  });
}
int sdg_metrics_host(const sdg_mesh_spec* mesh, int degree, int node_kind, int n_ranks, int rank, double* met,
                     double* fmet, long* n_local) {
  return guarded(nullptr, [&] {
    if (n_ranks < 1 || rank < 0 || rank >= n_ranks) throw sdg::ConfigError("rank outside [0, n_ranks)");
    const sdg::MeshGeom m(*mesh);
    if (mesh->mapping == SDG_MAP_BOX) throw sdg::ConfigError("metrics are stored for curved meshes only");
    const sdg::Partition part = sdg::assign_ranks(m, n_ranks);
    const sdg::LocalTopology topo = sdg::build_topology(m, part, rank);
    *n_local = static_cast<long>(topo.gids.size());
    if (met == nullptr || fmet == nullptr) return;
    const sdg::Basis basis(degree, node_kind);
    const sdg::CurvedMetrics cm = sdg::compute_metrics(m, basis, topo);
    std::copy(cm.met.begin(), cm.met.end(), met);
    std::copy(cm.fmet.begin(), cm.fmet.end(), fmet);
  });
}
int sdg_subrange_ops(int degree, int node_kind, double lo, double hi, double* fwd, double* bwd) {
  return guarded(nullptr, [&] {
    if (node_kind != SDG_NODES_GAUSS && node_kind != SDG_NODES_LGL) throw sdg::ConfigError("unknown node kind");
    sdg::build_subrange_ops(sdg::Basis(degree, node_kind), lo, hi, fwd, bwd);
  });
}
int sdg_mortar_intervals(long n_a, long n_b, double l_a, double delta, long* n_out, long* faces, double* ranges) {
  return guarded(nullptr, [&] {
    const std::vector<sdg::MortarInterval> iv = sdg::merge_intervals(n_a, n_b, l_a, delta);
    *n_out = static_cast<long>(iv.size());
    if (faces == nullptr || ranges == nullptr) return;
    for (size_t k = 0; k < iv.size(); ++k) {
      faces[2 * k] = iv[k].face_a;
      faces[2 * k + 1] = iv[k].face_b;
      ranges[4 * k] = iv[k].a_lo;
      ranges[4 * k + 1] = iv[k].a_hi;
      ranges[4 * k + 2] = iv[k].b_lo;
      ranges[4 * k + 3] = iv[k].b_hi;
    }
  });
}
int sdg_mortar_intervals_device(long n_a, long n_b, double l_a, double delta, long* n_out, long* faces,
                                double* ranges) {
  return guarded(nullptr, [&] { sdg::device_intervals(n_a, n_b, l_a, delta, n_out, faces, ranges); });
}
int sdg_interface_project_device(int degree, int node_kind, const long* nfy, const long* nfz, double l_y,
                                 double l_z, double d_y, double d_z, int nc, int from, const double* src,
                                 double* mortar_out, double* dst, long* n_mortars) {
  return guarded(nullptr, [&] {
    sdg::device_interface_project(degree, node_kind, nfy, nfz, l_y, l_z, d_y, d_z, nc, from, src, mortar_out, dst,
                                  n_mortars);
  });
}
int sdg_interface_flux_device(const sdg_gas* gas, int degree, int node_kind, const long* nfy, const long* nfz,
                              double l_y, double l_z, double d_y, double d_z, const double* u_a, const double* u_b,
                              const double* g_a, const double* g_b, double* flux_mortar, double* flux_a,
                              double* flux_b, long* n_mortars) {
  return guarded(nullptr, [&] {
    if (gas == nullptr) throw sdg::ConfigError("gas is NULL");
    sdg::device_interface_flux(*gas, degree, node_kind, nfy, nfz, l_y, l_z, d_y, d_z, u_a, u_b, g_a, g_b,
                               flux_mortar, flux_a, flux_b, n_mortars);
  });
}
int sdg_interface_lift_device(const sdg_gas* gas, int degree, int node_kind, const long* nfy, const long* nfz,
                              double l_y, double l_z, double d_y, double d_z, const double* u_a, const double* u_b,
                              double* lift_mortar, double* lift_a, double* lift_b, long* n_mortars) {
  return guarded(nullptr, [&] {
    if (gas == nullptr) throw sdg::ConfigError("gas is NULL");
    sdg::device_interface_flux(*gas, degree, node_kind, nfy, nfz, l_y, l_z, d_y, d_z, u_a, u_b, nullptr, nullptr,
                               lift_mortar, lift_a, lift_b, n_mortars, 1);
  });
}
int sdg_diagnostics(sdg_ctx* c, double t, int with_exact, double* out) {
  return guarded(c, [&] { c->s->diagnostics(t, with_exact, out); });
}
int sdg_write_snapshot(sdg_ctx* c, const char* path, double time) {
  return guarded(c, [&] { c->s->write_snapshot(path, time); });
}
int sdg_read_snapshot(sdg_ctx* c, const char* path, double* time) {
  return guarded(c, [&] {
    const double t = c->s->read_snapshot(path);
    if (time) *time = t;
  });
}
void* sdg_stream(sdg_ctx* c) { return c->s->stream(); }
long sdg_kernel_launches(const sdg_ctx* c) { return c->s->launches(); }
int sdg_enable_kernel_timing(sdg_ctx* c, int on) {
  c->s->enable_timing(on != 0);
  return SDG_OK;
}
int sdg_kernel_timing(sdg_ctx* c, char* names, int names_cap, double* ms, long* launches, int cap, int* n_classes) {
  return guarded(c, [&] {
    const auto t = c->s->timing_totals();
    std::string nm;
    for (int k = 0; k < static_cast<int>(t.size()); ++k) {
      if (k) nm += ",";
      nm += sdg::kKernelClasses[k];
      if (k < cap) {
        ms[k] = t[k].first;
        launches[k] = t[k].second;
      }
    }
    *n_classes = static_cast<int>(t.size());
    if (names && names_cap > 0) {
      std::strncpy(names, nm.c_str(), names_cap - 1);
      names[names_cap - 1] = 0;
    }
  });
}

}  // extern "C"
