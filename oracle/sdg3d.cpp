// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
//
// 3D CPU restatement of the reference's sliding-mesh DGSEM right-hand side and
// low-storage RK step.  Every phase follows the reference's phase order and
// arithmetic (citations are /root/reference/proj/src/<file>:<line>); the third
// direction (z, index k, faces ZMinus/ZPlus) is added uniformly and the
// interface-perpendicular index i_perp = iz is carried through the pairing
// exactly as partition.cpp already provides for it.
//
// Build: oracle/Makefile (g++ -O2 -ffp-contract=off -fopenmp).  Element loops
// are OpenMP-parallel without reductions, so results are bitwise independent
// of the thread count.
#include "sdg3d.h"

#include <algorithm>
#include <functional>
#include <array>
#include <cmath>
#include <cstring>
#include <exception>
#include <limits>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace orc {

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidStateError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ProtocolError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

constexpr int NV = SDG_NVARS;
constexpr int NG = SDG_NGRAD;
using State = std::array<double, NV>;

enum Side { XM = 0, XP = 1, YM = 2, YP = 3, ZM = 4, ZP = 5 };

// ---------------------------------------------------------------------------
// Nodes and basis: proj/src/nodal_basis.cpp:89-182 (Newton on Legendre
// polynomials from Chebyshev guesses, symmetrised; barycentric Lagrange;
// D with diagonal = -sum of the off-diagonal row).
// ---------------------------------------------------------------------------
static void legendre(int n, double x, double& p_out, double& dp_out) {
  if (n == 0) {
    p_out = 1.0;
    dp_out = 0.0;
    return;
  }
  double pm1 = 1.0, p = x, dpm1 = 0.0, dp = 1.0;
  for (int k = 1; k < n; ++k) {
    const double pp1 = ((2.0 * k + 1.0) * x * p - k * pm1) / (k + 1.0);
    const double dpp1 = dpm1 + (2.0 * k + 1.0) * p;
    pm1 = p;
    p = pp1;
    dpm1 = dp;
    dp = dpp1;
  }
  p_out = p;
  dp_out = dp;
}

struct Nodes {
  int degree = 0, kind = SDG_NODES_LGL;
  std::vector<double> x, w, bary;
  int count() const { return degree + 1; }

  Nodes() = default;
  Nodes(int deg, int knd) : degree(deg), kind(knd) {
    if (deg < 1 || deg > 15) throw ConfigError("polynomial degree outside [1,15]");
    const int n = deg + 1;
    x.assign(n, 0.0);
    w.assign(n, 0.0);
    const double pi = 3.14159265358979323846;
    if (kind == SDG_NODES_LGL) {
      x.front() = -1.0;
      x.back() = 1.0;
      for (int j = 1; j <= (n - 1) / 2; ++j) {
        double xx = -std::cos(pi * j / deg);
        for (int it = 0; it < 50; ++it) {
          double p, dp;
          legendre(deg, xx, p, dp);
          const double d2p = (2.0 * xx * dp - deg * (deg + 1.0) * p) / (1.0 - xx * xx);
          const double step = dp / d2p;
          xx -= step;
          if (std::abs(step) < 1e-15) break;
        }
        x[j] = xx;
        x[deg - j] = -xx;
      }
      if (n % 2 == 1) x[deg / 2] = 0.0;
      for (int j = 0; j < n; ++j) {
        double p, dp;
        legendre(deg, x[j], p, dp);
        w[j] = 2.0 / (deg * (deg + 1.0) * p * p);
      }
    } else {
      for (int j = 0; j <= (n - 1) / 2; ++j) {
        double xx = -std::cos(pi * (2.0 * j + 1.0) / (2.0 * n));
        for (int it = 0; it < 50; ++it) {
          double p, dp;
          legendre(n, xx, p, dp);
          const double step = p / dp;
          xx -= step;
          if (std::abs(step) < 1e-15) break;
        }
        x[j] = xx;
        x[deg - j] = -xx;
      }
      if (n % 2 == 1) x[deg / 2] = 0.0;
      for (int j = 0; j < n; ++j) {
        double p, dp;
        legendre(n, x[j], p, dp);
        w[j] = 2.0 / ((1.0 - x[j] * x[j]) * dp * dp);
      }
    }
    bary.assign(n, 1.0);
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k)
        if (k != j) bary[j] *= x[j] - x[k];
    for (double& b : bary) b = 1.0 / b;
  }

  void lagrange_all(double xx, double* out) const {
    const int n = count();
    for (int k = 0; k < n; ++k)
      if (xx == x[k]) {
        for (int j = 0; j < n; ++j) out[j] = (j == k) ? 1.0 : 0.0;
        return;
      }
    double den = 0.0;
    for (int k = 0; k < n; ++k) {
      out[k] = bary[k] / (xx - x[k]);
      den += out[k];
    }
    for (int k = 0; k < n; ++k) out[k] /= den;
  }
};

struct Basis {
  std::vector<double> D, fl, fr;  // D row-major n*n
};

static Basis make_basis(const Nodes& ns) {
  const int n = ns.count();
  Basis b;
  b.D.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i) {
    double diag = 0.0;
    for (int j = 0; j < n; ++j) {
      if (i == j) continue;
      const double d = (ns.bary[j] / ns.bary[i]) / (ns.x[i] - ns.x[j]);
      b.D[i * n + j] = d;
      diag -= d;
    }
    b.D[i * n + i] = diag;
  }
  b.fl.assign(n, 0.0);
  b.fr.assign(n, 0.0);
  ns.lagrange_all(-1.0, b.fl.data());
  ns.lagrange_all(1.0, b.fr.data());
  return b;
}

// ---------------------------------------------------------------------------
// Mortar operators: proj/src/mortar.cpp:12-134.  L2 projection between a face
// and its two mortars for a hanging node at sigma, assembled in long double
// (Gauss quadrature with n points, Cholesky solves) and rounded once.
// ---------------------------------------------------------------------------
using ld = long double;

static void ld_lagrange(const std::vector<ld>& xs, const std::vector<ld>& bw, ld x, ld* out) {
  const int n = static_cast<int>(xs.size());
  for (int k = 0; k < n; ++k)
    if (x == xs[k]) {
      for (int j = 0; j < n; ++j) out[j] = (j == k) ? 1.0L : 0.0L;
      return;
    }
  ld den = 0.0L;
  for (int k = 0; k < n; ++k) {
    out[k] = bw[k] / (x - xs[k]);
    den += out[k];
  }
  for (int k = 0; k < n; ++k) out[k] /= den;
}

static void ld_spd_solve(std::vector<ld> a, std::vector<ld>& b, int n) {
  for (int j = 0; j < n; ++j) {
    ld d = a[j * n + j];
    for (int k = 0; k < j; ++k) d -= a[j * n + k] * a[j * n + k];
    if (d <= 0.0L) throw ConfigError("mortar mass matrix not positive definite");
    const ld ljj = std::sqrt(d);
    a[j * n + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      ld s = a[i * n + j];
      for (int k = 0; k < j; ++k) s -= a[i * n + k] * a[j * n + k];
      a[i * n + j] = s / ljj;
    }
  }
  for (int c = 0; c < n; ++c) {
    for (int i = 0; i < n; ++i) {
      ld s = b[i * n + c];
      for (int k = 0; k < i; ++k) s -= a[i * n + k] * b[k * n + c];
      b[i * n + c] = s / a[i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      ld s = b[i * n + c];
      for (int k = i + 1; k < n; ++k) s -= a[k * n + i] * b[k * n + c];
      b[i * n + c] = s / a[i * n + i];
    }
  }
}

// fwd/bwd: [2][n*n] row-major; half 0 = Lower [-1, sigma], 1 = Upper [sigma, 1].
static void mortar_ops(const Nodes& ns, double sigma, double* fwd, double* bwd) {
  if (!(sigma >= -1.0 && sigma < 1.0)) throw ConfigError("mortar position sigma must lie in [-1, 1)");
  const int n = ns.count();
  const Nodes gauss(ns.degree, SDG_NODES_GAUSS);
  std::vector<ld> xs(ns.x.begin(), ns.x.end()), bw(n, 1.0L);
  for (int j = 0; j < n; ++j) {
    for (int k = 0; k < n; ++k)
      if (k != j) bw[j] *= xs[j] - xs[k];
    bw[j] = 1.0L / bw[j];
  }
  std::vector<ld> mass(n * n, 0.0L), lq(n), lx(n);
  for (int q = 0; q < n; ++q) {
    ld_lagrange(xs, bw, gauss.x[q], lq.data());
    const ld wq = gauss.w[q];
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) mass[i * n + j] += wq * lq[i] * lq[j];
  }
  const ld frac[2] = {0.5L * (1.0L + sigma), 0.5L * (1.0L - sigma)};
  for (int h = 0; h < 2; ++h) {
    std::vector<ld> s(n * n, 0.0L);
    for (int q = 0; q < n; ++q) {
      const ld z = gauss.x[q];
      const ld xi = (h == 0) ? -1.0L + frac[0] * (z + 1.0L) : static_cast<ld>(sigma) + frac[1] * (z + 1.0L);
      ld_lagrange(xs, bw, xi, lx.data());
      ld_lagrange(xs, bw, z, lq.data());
      const ld wq = gauss.w[q];
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) s[i * n + j] += wq * lx[i] * lq[j];
    }
    std::vector<ld> st(n * n), sw(n * n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        st[i * n + j] = s[j * n + i];
        sw[i * n + j] = frac[h] * s[i * n + j];
      }
    ld_spd_solve(mass, st, n);
    ld_spd_solve(mass, sw, n);
    for (int i = 0; i < n * n; ++i) {
      fwd[h * n * n + i] = static_cast<double>(st[i]);
      bwd[h * n * n + i] = static_cast<double>(sw[i]);
    }
  }
}

// General sub-range mortar (non-matching interfaces, BASELINE configs[1]): the same
// construction as mortar_ops with the mortar on face coordinates [lo, hi].
static void subrange_ops(const Nodes& ns, double lo, double hi, double* fwd, double* bwd) {
  if (!(lo >= -1.0 && lo < hi && hi <= 1.0)) throw ConfigError("mortar sub-range must satisfy -1 <= lo < hi <= 1");
  const int n = ns.count();
  const Nodes gauss(ns.degree, SDG_NODES_GAUSS);
  std::vector<ld> xs(ns.x.begin(), ns.x.end()), bw(n, 1.0L);
  for (int j = 0; j < n; ++j) {
    for (int k = 0; k < n; ++k)
      if (k != j) bw[j] *= xs[j] - xs[k];
    bw[j] = 1.0L / bw[j];
  }
  std::vector<ld> mass(n * n, 0.0L), lq(n), lx(n), s(n * n, 0.0L);
  for (int q = 0; q < n; ++q) {
    ld_lagrange(xs, bw, gauss.x[q], lq.data());
    const ld wq = gauss.w[q];
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) mass[i * n + j] += wq * lq[i] * lq[j];
  }
  const ld frac = 0.5L * (static_cast<ld>(hi) - static_cast<ld>(lo));
  for (int q = 0; q < n; ++q) {
    const ld z = gauss.x[q];
    ld_lagrange(xs, bw, static_cast<ld>(lo) + frac * (z + 1.0L), lx.data());
    ld_lagrange(xs, bw, z, lq.data());
    const ld wq = gauss.w[q];
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) s[i * n + j] += wq * lx[i] * lq[j];
  }
  std::vector<ld> st(n * n), sw(n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      st[i * n + j] = s[j * n + i];
      sw[i * n + j] = frac * s[i * n + j];
    }
  ld_spd_solve(mass, st, n);
  ld_spd_solve(mass, sw, n);
  for (int i = 0; i < n * n; ++i) {
    fwd[i] = static_cast<double>(st[i]);
    bwd[i] = static_cast<double>(sw[i]);
  }
}

// ---------------------------------------------------------------------------
// Interface kinematics and index algebra: proj/src/mesh.cpp:9-25,
// proj/src/mortar.cpp:136-150.
// ---------------------------------------------------------------------------
struct Disp {
  double delta = 0.0;
  long n_delta = 0;
  double s_delta = 0.0;
  bool conforming() const { return s_delta == 0.0; }
};

static Disp displacement(double delta, double l_par, long n_faces) {
  const double period = l_par * static_cast<double>(n_faces);
  double d = std::fmod(delta, period);
  if (d < 0.0) d += period;
  const double ratio = d / l_par;
  Disp st;
  st.delta = d;
  st.n_delta = static_cast<long>(std::floor(ratio));
  st.s_delta = ratio - static_cast<double>(st.n_delta);
  if (st.n_delta >= n_faces) {
    st.n_delta = 0;
    st.s_delta = 0.0;
    st.delta = 0.0;
  }
  return st;
}

static long moving_index(long i_par, long n_delta, int i_sub, long n_faces) {
  const long raw = i_par - n_delta + i_sub - 1;
  return ((raw % n_faces) + n_faces) % n_faces;
}
static long static_index(long i_moving, long n_delta, int i_sub, long n_faces) {
  const long raw = i_moving + n_delta - i_sub + 1;
  return ((raw % n_faces) + n_faces) % n_faces;
}

// Non-matching periodic face rows (BASELINE configs[1]; the reference needs equal
// counts, proj/src/mesh.cpp:75-77).  Side A: n_a faces of length l_a; side B: n_b
// faces over the same period, displaced by delta.  In A units, B edge j is
// n_delta + k_j + (s + r_j / n_b) with j n_a = k_j n_b + r_j and (n_delta, s) the
// reference's displacement split, so the equal-count limit keeps the reference's
// s bits; A-local coordinate of a B edge 2F - 1 (sigma), B-local coordinate of an
// A edge 1 - 2 (distance to B's right edge) / q (-sigma at equal counts).
// Restated pairwise: every (A face, B face) overlap, instead of the product's sweep.
struct Interval {
  long fa, fb, cp, lo_i;
  double lo_f, r[4];
};
static std::vector<Interval> intervals(long n_a, long n_b, double l_a, double delta) {
  if (n_a < 1 || n_b < 1 || !(l_a > 0.0)) throw ConfigError("bad face rows");
  const Disp d = displacement(delta, l_a, n_a);
  const double q = static_cast<double>(n_a) / static_cast<double>(n_b);
  auto edge = [&](long j, long& I, double& F) {  // B edge j (0 <= j <= n_b), unwrapped
    const long jj = j % n_b, wraps = j / n_b;
    I = d.n_delta + (jj * n_a) / n_b + wraps * n_a;
    F = d.s_delta + static_cast<double>((jj * n_a) % n_b) / static_cast<double>(n_b);
    if (F >= 1.0) {
      F -= 1.0;
      I += 1;
    }
  };
  auto less = [](long i1, double f1, long i2, double f2) { return i1 < i2 || (i1 == i2 && f1 < f2); };
  std::vector<Interval> out;
  for (long i = 0; i < n_a; ++i)
    for (long j = 0; j < n_b; ++j) {
      long I0, I1;
      double F0, F1;
      edge(j, I0, F0);
      edge(j + 1, I1, F1);
      for (long cp = 0; cp < 2; ++cp) {  // A face i and its copy one period on
        const long ai = i + cp * n_a;
        // overlap [max(ai, e_j), min(ai + 1, e_{j+1})]
        const bool lo_is_b = less(ai, 0.0, I0, F0) || (ai == I0 && F0 == 0.0);
        const long lo_i = lo_is_b ? I0 : ai;
        const double lo_f = lo_is_b ? F0 : 0.0;
        const bool hi_is_b = less(I1, F1, ai + 1, 0.0) || (I1 == ai + 1 && F1 == 0.0);
        const long hi_i = hi_is_b ? I1 : ai + 1;
        const double hi_f = hi_is_b ? F1 : 0.0;
        if (!less(lo_i, lo_f, hi_i, hi_f)) continue;
        Interval iv;
        iv.fa = i;
        iv.fb = j;
        iv.cp = cp;
        iv.lo_i = lo_i;
        iv.lo_f = lo_f;
        iv.r[0] = lo_is_b ? (F0 == 0.0 ? -1.0 : 2.0 * F0 - 1.0) : -1.0;
        iv.r[1] = hi_is_b ? (F1 == 0.0 ? 1.0 : 2.0 * F1 - 1.0) : 1.0;
        iv.r[2] = lo_is_b ? -1.0 : 1.0 - 2.0 * ((static_cast<double>(I1 - ai) + F1) / q);
        iv.r[3] = hi_is_b ? 1.0 : 1.0 - 2.0 * ((static_cast<double>(I1 - (ai + 1)) + F1) / q);
        out.push_back(iv);
      }
    }
  // A order: by A face, then along it -- the copy one period on (the part of the face
  // before B's edge 0) first, then by the exact start (integer, fraction).
  std::sort(out.begin(), out.end(), [](const Interval& x, const Interval& y) {
    if (x.fa != y.fa) return x.fa < y.fa;
    if (x.cp != y.cp) return x.cp > y.cp;
    return x.lo_i != y.lo_i ? x.lo_i < y.lo_i : x.lo_f < y.lo_f;
  });
  return out;
}

// ---------------------------------------------------------------------------
// Pairing (paper §4.4 / Appendix A): proj/src/partition.cpp:85-169.
// ---------------------------------------------------------------------------
struct RankMap {
  long n_par = 0, n_perp = 1;
  std::vector<int> ranks;
  int at(long i_par, long i_perp) const {
    const long ip = ((i_par % n_par) + n_par) % n_par;
    return ranks[static_cast<size_t>(i_perp) * n_par + ip];
  }
};

struct Tuple {
  int partner = 0, iface = 0;
  long i_par = 0, i_perp = 0;
  int i_sub = 0;
  long i_face = 0;
  int ctx = 0;
};

struct LocalFace {
  long i_face, i_par, i_perp;
};

static void append_tuples(const std::vector<LocalFace>& faces, const RankMap& partner_map,
                          long n_delta, long n_faces, bool on_static, bool conforming,
                          int iface, int ctx, std::vector<Tuple>& out) {
  for (const auto& f : faces)
    for (int i_sub = conforming ? 1 : 0; i_sub < 2; ++i_sub) {
      Tuple t;
      t.iface = iface;
      t.i_sub = i_sub;
      t.i_perp = f.i_perp;
      t.i_face = f.i_face;
      t.ctx = ctx;
      if (on_static) {
        t.i_par = f.i_par;
        t.partner = partner_map.at(moving_index(f.i_par, n_delta, i_sub, n_faces), f.i_perp);
      } else {
        t.i_par = static_index(f.i_par, n_delta, i_sub, n_faces);
        t.partner = partner_map.at(t.i_par, f.i_perp);
      }
      if (t.partner < 0) throw ProtocolError("rank map lookup hit an unset entry");
      out.push_back(t);
    }
}

static void sort_tuples(std::vector<Tuple>& cols) {
  std::sort(cols.begin(), cols.end(), [](const Tuple& a, const Tuple& b) {
    if (a.partner != b.partner) return a.partner < b.partner;
    if (a.iface != b.iface) return a.iface < b.iface;
    if (a.i_par != b.i_par) return a.i_par < b.i_par;
    if (a.i_perp != b.i_perp) return a.i_perp < b.i_perp;
    return a.i_sub < b.i_sub;
  });
}

struct Sched {
  int partner, offset, count;
};

static std::vector<Sched> make_schedule(const std::vector<Tuple>& cols, int self, Sched& self_entry) {
  std::vector<Sched> s;
  self_entry = {self, 0, 0};
  for (int i = 0; i < static_cast<int>(cols.size()); ++i) {
    const int p = cols[i].partner;
    if (p == self) {
      if (self_entry.count == 0) self_entry.offset = i;
      self_entry.count++;
      continue;
    }
    if (s.empty() || s.back().partner != p) s.push_back({p, i, 0});
    s.back().count++;
  }
  return s;
}

// ---------------------------------------------------------------------------
// Physics: proj/src/state.hpp:29-93, proj/src/flux.cpp:7-133, extended to 3D
// (second tangent and shear wave in the Roe dissipation).
// ---------------------------------------------------------------------------
struct Gas {
  double gamma, R, mu, Pr;
  double lambda() const { return -2.0 / 3.0 * mu; }
  double conductivity() const { return gamma * R * mu / ((gamma - 1.0) * Pr); }
  bool viscous() const { return mu > 0.0; }
};

static inline double pressure(const double* u, const Gas& g) {
  return (g.gamma - 1.0) * (u[4] - 0.5 * (u[1] * u[1] + u[2] * u[2] + u[3] * u[3]) / u[0]);
}
static inline double temperature(const double* u, const Gas& g) { return pressure(u, g) / (u[0] * g.R); }

static inline void prim4(const double* s, const Gas& g, double* out) {
  out[0] = s[1] / s[0];
  out[1] = s[2] / s[0];
  out[2] = s[3] / s[0];
  out[3] = temperature(s, g);
}

static State from_primitive(double rho, double v1, double v2, double v3, double p, const Gas& g) {
  if (!(rho > 0.0) || !(p > 0.0)) throw InvalidStateError("primitive state requires rho > 0 and p > 0");
  const double rhoe = p / (g.gamma - 1.0) + 0.5 * rho * (v1 * v1 + v2 * v2 + v3 * v3);
  return {rho, rho * v1, rho * v2, rho * v3, rhoe};
}

// ALE convective flux along direction d (flux.cpp:7-21).
static inline void ale_flux(const double* u, const double* vg, const Gas& g, double f[3][NV]) {
  const double rho = u[0];
  const double v[3] = {u[1] / rho, u[2] / rho, u[3] / rho};
  const double p = pressure(u, g);
  for (int d = 0; d < 3; ++d) {
    f[d][0] = u[0] * v[d];
    f[d][1] = u[1] * v[d] + (d == 0 ? p : 0.0);
    f[d][2] = u[2] * v[d] + (d == 1 ? p : 0.0);
    f[d][3] = u[3] * v[d] + (d == 2 ? p : 0.0);
    f[d][4] = (u[4] + p) * v[d];
    for (int c = 0; c < NV; ++c) f[d][c] -= vg[d] * u[c];
  }
}

// Viscous flux from primitive gradients g[3*q + dir] (flux.cpp:23-42).
static inline void viscous_flux(const double* u, const double* gr, const Gas& g, double f[3][NV]) {
  const double v[3] = {u[1] / u[0], u[2] / u[0], u[3] / u[0]};
  const double mu = g.mu, lam = g.lambda();
  const double div = gr[0] + gr[4] + gr[8];
  double tau[3][3];
  tau[0][0] = 2.0 * mu * gr[0] + lam * div;
  tau[1][1] = 2.0 * mu * gr[4] + lam * div;
  tau[2][2] = 2.0 * mu * gr[8] + lam * div;
  tau[0][1] = tau[1][0] = mu * (gr[1] + gr[3]);
  tau[0][2] = tau[2][0] = mu * (gr[2] + gr[6]);
  tau[1][2] = tau[2][1] = mu * (gr[5] + gr[7]);
  const double k = g.conductivity();
  for (int d = 0; d < 3; ++d) {
    const double qd = -k * gr[9 + d];
    f[d][0] = 0.0;
    f[d][1] = tau[d][0];
    f[d][2] = tau[d][1];
    f[d][3] = tau[d][2];
    f[d][4] = tau[d][0] * v[0] + tau[d][1] * v[1] + tau[d][2] * v[2] - qd;
  }
}

static inline void normal_flux(const double* u, int dir, double vg_n, const Gas& g, double* f) {
  const double rho = u[0];
  const double v[3] = {u[1] / rho, u[2] / rho, u[3] / rho};
  const double p = pressure(u, g);
  const double vn = v[dir];
  f[0] = rho * vn - vg_n * u[0];
  for (int d = 0; d < 3; ++d) f[1 + d] = u[1 + d] * vn + p * (d == dir ? 1.0 : 0.0) - vg_n * u[1 + d];
  f[4] = (u[4] + p) * vn - vg_n * u[4];
}

static inline double entropy_fixed_abs(double lam, double lam_l, double lam_r) {
  const double delta = std::max(0.0, std::max(lam - lam_l, lam_r - lam));
  const double a = std::abs(lam);
  if (a < 2.0 * delta) return lam * lam / (4.0 * delta) + delta;
  return a;
}

// Roe flux with Harten-Hyman fix on the acoustic waves, eigenvalues shifted by
// the normal grid speed (flux.cpp:68-133) — axis-aligned normal e_dir,
// tangents e_{dir+1}, e_{dir+2}.
static void roe_flux(const double* ul, const double* ur, int dir, double vg_n, const Gas& g, double* f) {
  const int t1 = (dir + 1) % 3, t2 = (dir + 2) % 3;
  const double rho_l = ul[0];
  const double vl[3] = {ul[1] / rho_l, ul[2] / rho_l, ul[3] / rho_l};
  const double p_l = pressure(ul, g);
  const double h_l = (ul[4] + p_l) / rho_l;
  const double un_l = vl[dir], ut1_l = vl[t1], ut2_l = vl[t2];
  const double c_l = std::sqrt(g.gamma * p_l / rho_l);

  const double rho_r = ur[0];
  const double vr[3] = {ur[1] / rho_r, ur[2] / rho_r, ur[3] / rho_r};
  const double p_r = pressure(ur, g);
  const double h_r = (ur[4] + p_r) / rho_r;
  const double un_r = vr[dir], ut1_r = vr[t1], ut2_r = vr[t2];
  const double c_r = std::sqrt(g.gamma * p_r / rho_r);

  const double sl = std::sqrt(rho_l), sr = std::sqrt(rho_r);
  const double inv = 1.0 / (sl + sr);
  const double un = (sl * un_l + sr * un_r) * inv;
  const double ut1 = (sl * ut1_l + sr * ut1_r) * inv;
  const double ut2 = (sl * ut2_l + sr * ut2_r) * inv;
  const double h = (sl * h_l + sr * h_r) * inv;
  const double q2 = un * un + ut1 * ut1 + ut2 * ut2;
  const double c2 = (g.gamma - 1.0) * (h - 0.5 * q2);
  if (!(c2 > 0.0)) throw InvalidStateError("roe_flux: nonpositive Roe enthalpy average");
  const double c = std::sqrt(c2);
  const double rho = sl * sr;

  const double dp = p_r - p_l;
  const double dun = un_r - un_l;
  const double dut1 = ut1_r - ut1_l;
  const double dut2 = ut2_r - ut2_l;
  const double drho = rho_r - rho_l;
  const double alpha1 = (dp - rho * c * dun) / (2.0 * c2);
  const double alpha2 = drho - dp / c2;
  const double alpha3 = rho * dut1;
  const double alpha3b = rho * dut2;
  const double alpha4 = (dp + rho * c * dun) / (2.0 * c2);

  const double a1 = entropy_fixed_abs(un - c - vg_n, un_l - c_l - vg_n, un_r - c_r - vg_n);
  const double a2 = std::abs(un - vg_n);
  const double a4 = entropy_fixed_abs(un + c - vg_n, un_l + c_l - vg_n, un_r + c_r - vg_n);

  const double d0 = a1 * alpha1 + a2 * alpha2 + a4 * alpha4;
  const double dn = a1 * alpha1 * (un - c) + a2 * alpha2 * un + a4 * alpha4 * (un + c);
  const double dt1 = (a1 * alpha1 + a2 * alpha2 + a4 * alpha4) * ut1 + a2 * alpha3;
  const double dt2 = (a1 * alpha1 + a2 * alpha2 + a4 * alpha4) * ut2 + a2 * alpha3b;
  const double dE = a1 * alpha1 * (h - un * c) + a2 * alpha2 * 0.5 * q2 + a2 * alpha3 * ut1 +
                    a2 * alpha3b * ut2 + a4 * alpha4 * (h + un * c);

  double fl[NV], fr[NV];
  normal_flux(ul, dir, vg_n, g, fl);
  normal_flux(ur, dir, vg_n, g, fr);
  f[0] = 0.5 * (fl[0] + fr[0] - d0);
  f[1 + dir] = 0.5 * (fl[1 + dir] + fr[1 + dir] - dn);
  f[1 + t1] = 0.5 * (fl[1 + t1] + fr[1 + t1] - dt1);
  f[1 + t2] = 0.5 * (fl[1 + t2] + fr[1 + t2] - dt2);
  f[4] = 0.5 * (fl[4] + fr[4] - dE);
}

// face_numerical_flux (solver.cpp:308-321): Roe minus the BR1 central viscous flux.
static void face_flux(const double* um, const double* up, int dir, double vg_n, const double* gm,
                      const double* gp, const Gas& g, double* f) {
  roe_flux(um, up, dir, vg_n, g, f);
  if (g.viscous() && gm != nullptr && gp != nullptr) {
    double fm[3][NV], fp[3][NV];
    viscous_flux(um, gm, g, fm);
    viscous_flux(up, gp, g, fp);
    for (int v = 0; v < NV; ++v) f[v] -= 0.5 * (fm[dir][v] + fp[dir][v]);
  }
}

// ---------------------------------------------------------------------------
// Curved hexahedra (SDG_MAP_WARP, include/sdg_types.h).  The reference has
// affine elements only (ElementMetrics, mesh.cpp:102-111); these are the
// rotation-invariant forms of its flux functions for a general unit normal n,
// which reduce to roe_flux / face_flux above for n = e_dir.
// ---------------------------------------------------------------------------

// sin(pi t), exactly 0 at integer t.
static double sinpi_exact(double t) {
  double r = std::fmod(t, 2.0);
  if (r < 0.0) r += 2.0;
  if (r == 0.0 || r == 1.0) return 0.0;
  return std::sin(3.14159265358979323846 * r);
}

static long double sinpi_ld(long double t) {
  long double r = std::fmod(t, 2.0L);
  if (r < 0.0L) r += 2.0L;
  if (r == 0.0L || r == 1.0L) return 0.0L;
  return std::sin(3.14159265358979323846264338327950288L * r);
}

static inline void normal_flux_n(const double* u, const double* n, double vg_n, const Gas& g, double* f) {
  const double rho = u[0];
  const double v[3] = {u[1] / rho, u[2] / rho, u[3] / rho};
  const double p = pressure(u, g);
  const double vn = v[0] * n[0] + v[1] * n[1] + v[2] * n[2];
  f[0] = rho * vn - vg_n * u[0];
  for (int d = 0; d < 3; ++d) f[1 + d] = u[1 + d] * vn + p * n[d] - vg_n * u[1 + d];
  f[4] = (u[4] + p) * vn - vg_n * u[4];
}

// Roe flux along the unit normal n (flux.cpp:68-133 in vector form: the two
// shear waves carry rho * (dv - dun n)).
static void roe_flux_n(const double* ul, const double* ur, const double* n, double vg_n, const Gas& g, double* f) {
  const double rho_l = ul[0], rho_r = ur[0];
  const double vl[3] = {ul[1] / rho_l, ul[2] / rho_l, ul[3] / rho_l};
  const double vr[3] = {ur[1] / rho_r, ur[2] / rho_r, ur[3] / rho_r};
  const double p_l = pressure(ul, g), p_r = pressure(ur, g);
  const double h_l = (ul[4] + p_l) / rho_l, h_r = (ur[4] + p_r) / rho_r;
  const double c_l = std::sqrt(g.gamma * p_l / rho_l), c_r = std::sqrt(g.gamma * p_r / rho_r);
  const double un_l = vl[0] * n[0] + vl[1] * n[1] + vl[2] * n[2];
  const double un_r = vr[0] * n[0] + vr[1] * n[1] + vr[2] * n[2];

  const double sl = std::sqrt(rho_l), sr = std::sqrt(rho_r);
  const double inv = 1.0 / (sl + sr);
  double v[3];
  for (int d = 0; d < 3; ++d) v[d] = (sl * vl[d] + sr * vr[d]) * inv;
  const double h = (sl * h_l + sr * h_r) * inv;
  const double un = v[0] * n[0] + v[1] * n[1] + v[2] * n[2];
  const double q2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
  const double c2 = (g.gamma - 1.0) * (h - 0.5 * q2);
  if (!(c2 > 0.0)) throw InvalidStateError("roe_flux: nonpositive Roe enthalpy average");
  const double c = std::sqrt(c2);
  const double rho = sl * sr;

  const double dp = p_r - p_l, dun = un_r - un_l, drho = rho_r - rho_l;
  double dvt[3];
  for (int d = 0; d < 3; ++d) dvt[d] = (vr[d] - vl[d]) - dun * n[d];
  const double alpha1 = (dp - rho * c * dun) / (2.0 * c2);
  const double alpha2 = drho - dp / c2;
  const double alpha4 = (dp + rho * c * dun) / (2.0 * c2);
  const double a1 = entropy_fixed_abs(un - c - vg_n, un_l - c_l - vg_n, un_r - c_r - vg_n);
  const double a2 = std::abs(un - vg_n);
  const double a4 = entropy_fixed_abs(un + c - vg_n, un_l + c_l - vg_n, un_r + c_r - vg_n);
  const double w1 = a1 * alpha1, w2 = a2 * alpha2, w4 = a4 * alpha4;
  const double d0 = w1 + w2 + w4;
  double dm[3];
  for (int d = 0; d < 3; ++d) dm[d] = d0 * v[d] + (w4 - w1) * c * n[d] + a2 * rho * dvt[d];
  const double dE = w1 * (h - un * c) + w2 * 0.5 * q2 + w4 * (h + un * c) +
                    a2 * rho * (v[0] * dvt[0] + v[1] * dvt[1] + v[2] * dvt[2]);
  double fl[NV], fr[NV];
  normal_flux_n(ul, n, vg_n, g, fl);
  normal_flux_n(ur, n, vg_n, g, fr);
  f[0] = 0.5 * (fl[0] + fr[0] - d0);
  for (int d = 0; d < 3; ++d) f[1 + d] = 0.5 * (fl[1 + d] + fr[1 + d] - dm[d]);
  f[4] = 0.5 * (fl[4] + fr[4] - dE);
}

// face_numerical_flux (solver.cpp:308-321) along n: Roe minus the BR1 central
// viscous normal flux 0.5 (Fv- + Fv+) . n.
static void face_flux_n(const double* um, const double* up, const double* n, double vg_n, const double* gm,
                        const double* gp, const Gas& g, double* f) {
  roe_flux_n(um, up, n, vg_n, g, f);
  if (g.viscous() && gm != nullptr && gp != nullptr) {
    double fm[3][NV], fp[3][NV];
    viscous_flux(um, gm, g, fm);
    viscous_flux(up, gp, g, fp);
    for (int v = 0; v < NV; ++v)
      f[v] -= 0.5 * ((fm[0][v] * n[0] + fm[1][v] * n[1] + fm[2][v] * n[2]) +
                     (fp[0][v] * n[0] + fp[1][v] * n[1] + fp[2][v] * n[2]));
  }
}

// ---------------------------------------------------------------------------
// Exact solutions / cases: proj/src/exact_solutions.cpp:7-35, cases.hpp:18-25.
// ---------------------------------------------------------------------------
// The seeded density perturbation (include/sdg_types.h sdg_case.pt_*):
// A sum_m a_m sin(2 pi k_m . xh + phi_m), xh the advected point normalised per direction.
static double perturbation(const sdg_case& cs, const double* x, double t) {
  const double two_pi = 6.283185307179586476925286766559;
  double c[3];
  for (int d = 0; d < 3; ++d) c[d] = x[d] - cs.pt_adv[d] * t;
  if (cs.pt_coords == 1) {  // (x, theta, r) about the x axis, theta measured from +Z towards +Y
    const double th = std::atan2(c[1], c[2]), r = std::sqrt(c[1] * c[1] + c[2] * c[2]);
    c[1] = th;
    c[2] = r;
  }
  double arg[SDG_PT_MAX_MODES];
  double acc = 0.0;
  for (int m = 0; m < cs.pt_modes; ++m) {
    arg[m] = 0.0;
    for (int d = 0; d < 3; ++d) arg[m] += cs.pt_k[m][d] * ((c[d] - cs.pt_x0[d]) / cs.pt_len[d]);
    acc += cs.pt_a[m] * std::sin(two_pi * arg[m] + cs.pt_phi[m]);
  }
  return cs.pt_amp * acc;
}

static State eval_base(const sdg_case& cs, const double* x, double t, const Gas& g);
// The case state plus its seeded density perturbation (velocity and pressure kept).
static State eval_case(const sdg_case& cs, const double* x, double t, const Gas& g) {
  State u = eval_base(cs, x, t, g);
  if (cs.pt_modes <= 0) return u;
  if (cs.pt_modes > SDG_PT_MAX_MODES) throw ConfigError("perturbation: 0..8 modes");
  const double v1 = u[1] / u[0], v2 = u[2] / u[0], v3 = u[3] / u[0];
  return from_primitive(u[0] + perturbation(cs, x, t), v1, v2, v3, pressure(u.data(), g), g);
}

static State eval_base(const sdg_case& cs, const double* x, double t, const Gas& g) {
  const double pi = 3.14159265358979323846;
  switch (cs.kind) {
    case SDG_CASE_FREESTREAM:
      return from_primitive(cs.fs_rho, cs.fs_v[0], cs.fs_v[1], cs.fs_v[2], cs.fs_p, g);
    case SDG_CASE_DENSITY_WAVE: {
      const double* k = cs.dw_k;
      const double* a = cs.dw_a;
      const double phase =
          pi * (k[0] * x[0] + k[1] * x[1] + k[2] * x[2] - (k[0] * a[0] + k[1] * a[1] + k[2] * a[2]) * t);
      const double rho = 2.0 + cs.dw_alpha * std::sin(phase);
      return from_primitive(rho, a[0], a[1], a[2], cs.dw_p0, g);
    }
    case SDG_CASE_VORTEX: {
      const double u_inf = cs.vx_v_inf * std::cos(cs.vx_theta);
      const double v_inf = cs.vx_v_inf * std::sin(cs.vx_theta);
      const double xb = x[0] - cs.vx_center[0] - u_inf * t;
      const double yb = x[1] - cs.vx_center[1] - v_inf * t;
      const double r2 = (xb * xb + yb * yb) / (cs.vx_rc * cs.vx_rc);
      const double s = cs.vx_eps * std::exp(0.5 * (1.0 - r2));
      const double v1 = u_inf - cs.vx_v_inf * s * yb / cs.vx_rc;
      const double v2 = v_inf + cs.vx_v_inf * s * xb / cs.vx_rc;
      const double tr = 1.0 - 0.5 * (g.gamma - 1.0) * cs.vx_eps * cs.vx_eps * cs.vx_ma_inf *
                                  cs.vx_ma_inf * std::exp(1.0 - r2);
      const double rho = cs.vx_rho_inf * std::pow(tr, 1.0 / (g.gamma - 1.0));
      const double p_inf = cs.vx_rho_inf * cs.vx_v_inf * cs.vx_v_inf / (g.gamma * cs.vx_ma_inf * cs.vx_ma_inf);
      const double pres = p_inf * std::pow(tr, g.gamma / (g.gamma - 1.0));
      return from_primitive(rho, v1, v2, 0.0, pres, g);
    }
    case SDG_CASE_TGV: {
      // BASELINE frame (X, Y, Z) = (y, z, x); see include/sdg_types.h.
      const double X = x[1], Y = x[2], Z = x[0];
      const double V0 = cs.tgv_v0, r0 = cs.tgv_rho0;
      const double uX = V0 * std::sin(X) * std::cos(Y) * std::cos(Z);
      const double uY = -V0 * std::cos(X) * std::sin(Y) * std::cos(Z);
      const double p0 = r0 * V0 * V0 / (g.gamma * cs.tgv_mach * cs.tgv_mach);
      const double p = p0 + r0 * V0 * V0 / 16.0 * (std::cos(2.0 * X) + std::cos(2.0 * Y)) * (std::cos(2.0 * Z) + 2.0);
      return from_primitive(r0, 0.0, uX, uY, p, g);
    }
    case SDG_CASE_SWIRL: {
      // Axial density wave with rigid swirl about x (include/sdg_types.h).
      const double om = cs.sw_omega;
      const double rho = 2.0 + cs.dw_alpha * std::sin(pi * cs.dw_k[0] * (x[0] - cs.dw_a[0] * t));
      const double p = cs.dw_p0 + om * om * (x[1] * x[1] + x[2] * x[2]);
      return from_primitive(rho, cs.dw_a[0], om * x[2], -om * x[1], p, g);
    }
  }
  throw ConfigError("unknown case kind");
}

// ---------------------------------------------------------------------------
// Mesh (proj/src/mesh.cpp:27-122) and local domain (face_topology.cpp:55-150),
// 3D: bands along x, ny x nz elements per band cross-section.
// ---------------------------------------------------------------------------
struct Band {
  double x_lo, x_hi, hx, hy, hz, vg;
  int nx, off;
  int ny = 0, nz = 0;  // per-band counts (BandSpec::ny, mesh.hpp:16; nz its 3D analogue)
  double vgz = 0.0;    // translation along +z (oblique sliding)
};
struct Iface {
  int left, right;
  bool static_is_left;
  double l_par;
  long n_faces, n_perp;
  double vg_rel;
};
struct Elem {
  int band, ix, iy, iz;
};
// Non-matching / obliquely sliding interface (BASELINE configs[1]): side A = the
// left band's x+ faces, B = the right band's x- faces, B displaced by
// (vy_rel, vz_rel) t.  Mortars: every pair of a y-row interval and a z-row
// interval (intervals() above), with the sub-range operators of both sides.
struct NcIface {
  int left = 0, right = 0;
  long nfy[2] = {0, 0}, nfz[2] = {0, 0};
  double ly[2] = {0, 0}, lz[2] = {0, 0};
  double vy_rel = 0.0, vz_rel = 0.0;
  std::vector<int> elem[2], side[2];  // per side, face fy * nfz + fz -> (element, side)
  double dy_base = 0.0, dz_base = 0.0;
  // current stage
  double dy = 0.0, dz = 0.0;
  std::vector<Interval> rows[2];
  std::vector<double> F[2][2], B[2][2];  // [side][dir]: per row n x n
  std::vector<double> u[2], g[2];        // mortar traces / gradients per side
};
struct InteriorFace {
  int em, ep, dir;
  int seam = 0;  // annulus sector: the face crosses the theta seam (minus at theta ~ alpha, plus at ~ 0)
};
struct BoundaryFace {
  int e, side;
};
struct SlidingFace {
  int e, side;
  long i_par, i_perp;
};

struct Ctx {
  int iface = 0;
  bool on_static = true;
  std::vector<SlidingFace> faces;
  RankMap static_map, moving_map;
  std::vector<int> m[2];
  double delta_base = 0.0;
  Disp st;
  double sigma_side = -1.0;
  bool conforming = true;
  std::vector<double> fwd, bwd;  // [2][n*n]
  long last_n = -1;
  bool last_conf = true, topo_valid = false;
  long rebuilds = 0;
  long wraps = 0;  // periods subtracted from delta_base so far (annulus sector windings)
  long K = 0;      // windings of the moving band at the stage: displacement = d + K * period
  int half(int i_sub) const { return on_static ? i_sub : 1 - i_sub; }
};

struct Role {
  std::vector<Tuple> cols;
  std::vector<Sched> sched;
  Sched self{0, 0, 0};
  int n_mortars = 0;
  std::vector<double> u_mine, u_theirs, flux, lift, g_mine, g_theirs;
};

}  // namespace orc

using namespace orc;

struct orc_solver {
  sdg_mesh_spec spec;
  Gas gas;
  sdg_case flow_case;
  Nodes ns;
  Basis basis;
  int n = 0, n2 = 0, n3 = 0;
  std::vector<double> wdiff;  // D-hat(i,m) = w_m D(m,i) / w_i
  std::vector<Band> bands;
  std::vector<Iface> ifaces;
  std::vector<Elem> elems;
  std::vector<InteriorFace> interior;
  std::vector<BoundaryFace> dirichlet;
  std::vector<std::vector<SlidingFace>> sliding;
  std::vector<NcIface> ncs;
  std::vector<Ctx> ctxs;
  std::vector<int> static_ids, moving_ids;
  Role statics, movings;
  bool lifting = false;

  std::vector<double> field, reg, dudt, grad, trace, fflux, gtrace, lift;
  // Curved elements (SDG_MAP_WARP): per node Ja^d_c (9, [3*d + c]) and 1/J;
  // per side face node the unit normal along +xi_dir and the surface Jacobian sJ.
  // SDG_MAP_ANNULUS adds per node the contravariant grid velocity per unit
  // angular speed V^d (3) and per face node vg.n per unit angular speed.
  bool curved = false, annulus = false;
  // Periodic annulus sector of angle alpha (< 2 pi): vectors crossing the theta seam rotate by alpha.
  bool sector = false;
  double alpha = 0.0;
  int mw = 10, fw = 4;  // doubles per node / per face node
  std::vector<double> met, fmet;
  double t_cur = 0.0;   // stage time of the residual being evaluated (band rotation)
  double time = 0.0;
  int step_index = 0, stage_index = 0;
  std::string err;

  int nz() const { return spec.nz; }
  int ny() const { return spec.ny; }
  long gid(int b, int ix, int iy, int iz) const {
    return bands[b].off + (static_cast<long>(ix) * bands[b].ny + iy) * bands[b].nz + iz;
  }
  size_t node(int e, int i, int j, int k) const { return ((static_cast<size_t>(e) * n + i) * n + j) * n + k; }
  double* tr(int e, int side) { return trace.data() + (static_cast<size_t>(e) * 6 + side) * n2 * NV; }
  double* ff(int e, int side) { return fflux.data() + (static_cast<size_t>(e) * 6 + side) * n2 * NV; }
  double* gt(int e, int side) { return gtrace.data() + (static_cast<size_t>(e) * 6 + side) * n2 * NG; }
  double* lf(int e, int side) { return lift.data() + (static_cast<size_t>(e) * 6 + side) * n2 * 4; }
  const double* mt(int e, int nd) const { return met.data() + (static_cast<size_t>(e) * n3 + nd) * mw; }
  const double* fm(int e, int side) const { return fmet.data() + (static_cast<size_t>(e) * 6 + side) * n2 * fw; }
  // Rotation of a rotating annulus band at the stage time: theta -> theta + phi,
  // (Y, Z) -> (c Y + s Z, -s Y + c Z) with Y = r sin(theta), Z = r cos(theta).
  void band_rot(int e, double& c, double& s) const {
    const double phi = annulus ? bands[elems[e].band].vg * t_cur : 0.0;
    c = std::cos(phi);
    s = std::sin(phi);
  }
  static void rot3(double c, double s, const double* v, double* o) {
    o[0] = v[0];
    o[1] = c * v[1] + s * v[2];
    o[2] = -s * v[1] + c * v[2];
  }
  // Rotation by k sector angles (periodic annulus sectors): state momentum,
  // primitive velocity, velocity-gradient tensor R G R^T and temperature gradient.
  void sector_rot(int k, double& c, double& s) const {
    c = std::cos(k * alpha);
    s = std::sin(k * alpha);
  }
  void rot_state(int k, const double* u, double* o) const {
    double c, s;
    sector_rot(k, c, s);
    o[0] = u[0];
    rot3(c, s, u + 1, o + 1);
    o[4] = u[4];
  }
  void rot_prim(int k, const double* q, double* o) const {
    double c, s;
    sector_rot(k, c, s);
    rot3(c, s, q, o);
    o[3] = q[3];
  }
  void rot_grad(int k, const double* g, double* o) const {
    // G_qd = g[3q + d] (q velocity component, d direction): G' = R G R^T; grad T' = R grad T.
    double c, s;
    sector_rot(k, c, s);
    double t[9];
    for (int d = 0; d < 3; ++d) {  // each column (over q)
      const double col[3] = {g[d], g[3 + d], g[6 + d]};
      double r[3];
      rot3(c, s, col, r);
      t[d] = r[0];
      t[3 + d] = r[1];
      t[6 + d] = r[2];
    }
    for (int q = 0; q < 3; ++q) rot3(c, s, t + 3 * q, o + 3 * q);  // each row (over d)
    rot3(c, s, g + 9, o + 9);
  }
  // The moving role's mortar data (computed by the static side in its frame) moved to the
  // moving elements' positions: each mortar block rotated by +k alpha.  comps: first
  // rotated component (0: primitive velocity, 1: momentum); nc values per node.
  std::vector<double> to_moving_frame(const Role& role, const std::vector<double>& data, int nc, int comps) const {
    std::vector<double> out(data);
    if (!sector) return out;
    for (int m = 0; m < role.n_mortars; ++m) {
      const int k = mortar_k(role.cols[m]);
      double c, s;
      sector_rot(k, c, s);
      for (int q = 0; q < n2; ++q) {
        double* v = out.data() + (static_cast<size_t>(m) * n2 + q) * nc + comps;  // (x, y, z) components
        const double in[3] = {v[0], v[1], v[2]};
        double r[3];
        rot3(c, s, in, r);
        v[0] = r[0];
        v[1] = r[1];
        v[2] = r[2];
      }
    }
    return out;
  }
  // Windings k of a mortar column (its moving partner sits at the static location + k alpha).
  int mortar_k(const Tuple& t) const {
    const Ctx& c = ctxs[t.ctx];
    const long raw = t.i_par - c.st.n_delta + t.i_sub - 1;
    return static_cast<int>(c.K + (raw < 0 ? 1 : 0));
  }
  // Ja^d_c of node nd at t_cur (rotated with the band).
  void ja_at(int e, int nd, double* o9) const {
    double c, s;
    band_rot(e, c, s);
    for (int d = 0; d < 3; ++d) rot3(c, s, mt(e, nd) + 3 * d, o9 + 3 * d);
  }
  // Unit +xi normal of face node f at t_cur, and vg . n.
  void normal_at(int e, int side, int f, double* n3o, double& vgn) const {
    const double* q = fm(e, side) + f * fw;
    if (!annulus) {
      for (int c = 0; c < 3; ++c) n3o[c] = q[c];
      vgn = bands[elems[e].band].vg * q[1];
      return;
    }
    double c, s;
    band_rot(e, c, s);
    rot3(c, s, q, n3o);
    vgn = bands[elems[e].band].vg * q[4];
  }

  void physical(int e, double xi, double eta, double zeta, double t, double* x) const {
    const Elem& el = elems[e];
    const Band& b = bands[el.band];
    const double ox = b.x_lo + el.ix * b.hx;
    const double oy = spec.y0 + el.iy * b.hy;
    const double oz = spec.z0 + el.iz * b.hz;
    if (!curved) {
      x[0] = ox + 0.5 * (xi + 1.0) * b.hx;
      x[1] = oy + 0.5 * (eta + 1.0) * b.hy + b.vg * t;
      x[2] = oz + 0.5 * (zeta + 1.0) * b.hz + b.vgz * t;
      return;
    }
    // SDG_MAP_WARP (include/sdg_types.h).
    const double tx = (el.ix + 0.5 * (xi + 1.0)) / b.nx;
    const double ty = (el.iy + 0.5 * (eta + 1.0)) / spec.ny;
    const double tz = (el.iz + 0.5 * (zeta + 1.0)) / spec.nz;
    const double sp = sinpi_exact(tx), sy = sinpi_exact(2.0 * ty), sz = sinpi_exact(2.0 * tz);
    const double A = spec.warp;
    x[0] = (ox + 0.5 * (xi + 1.0) * b.hx) + A * b.hx * sp * sy * sz;
    x[1] = (oy + 0.5 * (eta + 1.0) * b.hy) + (annulus ? 0.0 : A * b.hy * sp * sz) + b.vg * t;  // annulus: no theta warp
    x[2] = (oz + 0.5 * (zeta + 1.0) * b.hz) + A * b.hz * sp * sy;
    if (annulus) {
      // SDG_MAP_ANNULUS: (x, theta, r) -> (x, r sin theta, r cos theta); the band's
      // rotation is the + vg t already in theta.
      const double th = x[1], r = x[2];
      x[1] = r * std::sin(th);
      x[2] = r * std::cos(th);
    }
  }
  // Mapped position minus the mapped element centre, long double (metrics only).
  void relative_position(int e, double xi, double eta, double zeta, ld* x) const {
    const Elem& el = elems[e];
    const Band& b = bands[el.band];
    const ld h[3] = {b.hx, b.hy, b.hz};
    const ld r[3] = {0.5L * xi, 0.5L * eta, 0.5L * zeta};
    const ld t[3] = {(el.ix + 0.5L * (xi + 1.0L)) / b.nx, (el.iy + 0.5L * (eta + 1.0L)) / spec.ny,
                     (el.iz + 0.5L * (zeta + 1.0L)) / spec.nz};
    const ld tc[3] = {(el.ix + 0.5L) / b.nx, (el.iy + 0.5L) / spec.ny, (el.iz + 0.5L) / spec.nz};
    const ld A = spec.warp;
    const ld sp = sinpi_ld(t[0]), sy = sinpi_ld(2.0L * t[1]), sz = sinpi_ld(2.0L * t[2]);
    const ld cp = sinpi_ld(tc[0]), cy = sinpi_ld(2.0L * tc[1]), cz = sinpi_ld(2.0L * tc[2]);
    x[0] = r[0] * h[0] + A * h[0] * (sp * sy * sz - cp * cy * cz);
    x[1] = r[1] * h[1] + A * h[1] * (sp * sz - cp * cz);
    x[2] = r[2] * h[2] + A * h[2] * (sp * sy - cp * cy);
    if (annulus) {
      // Polar map about the x axis, minus the mapped centre.
      const ld th = spec.y0 + h[1] * (el.iy + 0.5L * (eta + 1.0L));  // theta faces stay meridional planes
      const ld rr = spec.z0 + h[2] * (el.iz + 0.5L * (zeta + 1.0L)) + A * h[2] * sp * sy;
      const ld thc = center_angle(e);
      const ld rc = spec.z0 + h[2] * (el.iz + 0.5L) + A * h[2] * cp * cy;
      x[1] = rr * std::sin(th) - rc * std::sin(thc);
      x[2] = rr * std::cos(th) - rc * std::cos(thc);
    }
  }
  // Angle of an annulus element's centre at t = 0.
  ld center_angle(int e) const {
    const Elem& el = elems[e];
    const Band& b = bands[el.band];
    const ld tc[3] = {(el.ix + 0.5L) / b.nx, (el.iy + 0.5L) / spec.ny, (el.iz + 0.5L) / spec.nz};
    (void)tc;
    return spec.y0 + static_cast<ld>(b.hy) * (el.iy + 0.5L);
  }
  // Absolute radius of a reference point (annulus grid-velocity potential).
  ld radius(int e, double xi, double eta, double zeta) const {
    const Elem& el = elems[e];
    const Band& b = bands[el.band];
    const ld h[3] = {b.hx, b.hy, b.hz};
    const ld t[3] = {(el.ix + 0.5L * (xi + 1.0L)) / b.nx, (el.iy + 0.5L * (eta + 1.0L)) / spec.ny,
                     (el.iz + 0.5L * (zeta + 1.0L)) / spec.nz};
    const ld sp = sinpi_ld(t[0]), sy = sinpi_ld(2.0L * t[1]);
    return spec.z0 + h[2] * (el.iz + 0.5L * (zeta + 1.0L)) + static_cast<ld>(spec.warp) * h[2] * sp * sy;
  }
  void face_node_position(int e, int side, int p, int q, double t, double* x) const {
    const double a = ns.x[p], c = ns.x[q];
    switch (side) {
      case XM: physical(e, -1.0, a, c, t, x); break;
      case XP: physical(e, 1.0, a, c, t, x); break;
      case YM: physical(e, a, -1.0, c, t, x); break;
      case YP: physical(e, a, 1.0, c, t, x); break;
      case ZM: physical(e, a, c, -1.0, t, x); break;
      default: physical(e, a, c, 1.0, t, x); break;
    }
  }

  void build(const sdg_mesh_spec& s, const sdg_solver_config& cfg);
  void build_metrics();
  void update_interfaces(double t_stage);
  void rebuild_role(Role& role, const std::vector<int>& ids);
  void prolong(const double* u);
  void fill_mortar_solution();
  void exchange_solution();
  void run_lifting(double t_stage, const double* u);
  void assemble_gradients(const double* u);
  void assemble_gradients_curved(const double* u);
  void prolong_gradients(int e);
  void send_gradients();
  void interior_flux();
  void volume(const double* u, double* out);
  void mortar_flux();
  void mortar_apply();
  void dirichlet_flux(double t_stage);
  void apply_faces(double* out);
  void residual(double t_stage, const double* u, double* out);
  void nc_update(double t_stage);
  void nc_lift();
  void nc_flux();
  void check_admissible(const double* u) const;
  void step(double dt);
  double suggest_dt(double cfl) const;
};

static thread_local std::string g_err;

// Mesh construction: proj/src/mesh.cpp:27-92, 3D extents and z periodicity.
void orc_solver::build(const sdg_mesh_spec& s, const sdg_solver_config& cfg) {
  spec = s;
  gas = {cfg.gas.gamma, cfg.gas.R, cfg.gas.mu, cfg.gas.Pr};
  if (!(gas.gamma > 1.0) || !(gas.R > 0.0) || !(gas.mu >= 0.0) || !(gas.Pr > 0.0))
    throw ConfigError("gas model requires gamma > 1, R > 0, mu >= 0, Pr > 0");
  flow_case = cfg.flow_case;
  ns = Nodes(cfg.degree, cfg.node_kind);
  basis = make_basis(ns);
  n = ns.count();
  n2 = n * n;
  n3 = n2 * n;
  wdiff.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int m = 0; m < n; ++m) wdiff[i * n + m] = ns.w[m] * basis.D[m * n + i] / ns.w[i];

  if (s.n_bands < 1 || s.n_bands > SDG_MAX_BANDS) throw ConfigError("mesh needs 1..16 bands");
  if (s.ny < 1 || s.nz < 1) throw ConfigError("mesh needs ny, nz >= 1");
  if (!(s.width > 0.0) || !(s.height > 0.0) || !(s.depth > 0.0)) throw ConfigError("mesh extents must be positive");
  double frac_sum = 0.0;
  for (int b = 0; b < s.n_bands; ++b) {
    if (s.bands[b].nx < 1) throw ConfigError("band element count nx must be >= 1");
    if (!(s.bands[b].width_frac > 0.0)) throw ConfigError("band width fraction must be positive");
    frac_sum += s.bands[b].width_frac;
  }
  const int nb = s.n_bands;
  bands.resize(nb);
  double x = s.x0, acc = 0.0;
  int off = 0;
  for (int b = 0; b < nb; ++b) {
    Band& bd = bands[b];
    bd.x_lo = x;
    acc += s.bands[b].width_frac;
    bd.x_hi = (b == nb - 1) ? s.x0 + s.width : s.x0 + s.width * acc / frac_sum;
    x = bd.x_hi;
    bd.nx = s.bands[b].nx;
    bd.ny = s.bands[b].ny > 0 ? s.bands[b].ny : s.ny;
    bd.nz = s.bands[b].nz > 0 ? s.bands[b].nz : s.nz;
    if (s.bands[b].ny < 0 || s.bands[b].nz < 0) throw ConfigError("band ny / nz must be >= 0");
    bd.hx = (bd.x_hi - bd.x_lo) / bd.nx;
    bd.hy = s.height / bd.ny;
    bd.hz = s.depth / bd.nz;
    bd.vg = s.bands[b].vg_y;
    bd.vgz = s.bands[b].vg_z;
    bd.off = off;
    off += bd.nx * bd.ny * bd.nz;
    if (bd.vg < 0.0 || bd.vgz < 0.0) throw ConfigError("moving bands must translate toward +y / +z");
    if (bd.vg != 0.0 && !s.periodic_y)
      throw ConfigError("a moving band requires periodicity along the movement direction");
    if (bd.vgz != 0.0 && !s.periodic_z) throw ConfigError("a band moving along z requires periodicity along z");
    if ((bd.ny != s.ny || bd.nz != s.nz || bd.vgz != 0.0 || s.mortars != 0) && s.mapping != SDG_MAP_BOX)
      throw ConfigError("per-band ny / nz and sliding along z need affine hexahedra (SDG_MAP_BOX)");
  }
  const int n_pairs = s.periodic_x ? nb : nb - 1;
  for (int p = 0; p < n_pairs; ++p) {
    const int left = p, right = (p + 1) % nb;
    if (nb == 1 && left == right) continue;
    const Band& bl = bands[left];
    const Band& br = bands[right];
    if (bl.ny != br.ny || bl.nz != br.nz || bl.vgz != 0.0 || br.vgz != 0.0 || s.mortars == SDG_MORTARS_TENSOR) {
      if (bl.ny == br.ny && bl.nz == br.nz && bl.vg == br.vg && bl.vgz == br.vgz) continue;
      NcIface f;
      f.left = left;
      f.right = right;
      f.nfy[0] = bl.ny;
      f.nfz[0] = bl.nz;
      f.nfy[1] = br.ny;
      f.nfz[1] = br.nz;
      f.ly[0] = bl.hy;
      f.lz[0] = bl.hz;
      f.ly[1] = br.hy;
      f.lz[1] = br.hz;
      f.vy_rel = br.vg - bl.vg;
      f.vz_rel = br.vgz - bl.vgz;
      for (int sd = 0; sd < 2; ++sd) {
        f.elem[sd].assign(f.nfy[sd] * f.nfz[sd], -1);
        f.side[sd].assign(f.nfy[sd] * f.nfz[sd], -1);
      }
      ncs.push_back(std::move(f));
      continue;
    }
    if (bl.vg == br.vg) continue;
    if (bl.vg != 0.0 && br.vg != 0.0) throw ConfigError("sliding interface requires one static side");
    Iface f;
    f.left = left;
    f.right = right;
    f.static_is_left = (bl.vg == 0.0);
    f.l_par = bl.hy;
    f.n_faces = bl.ny;
    f.n_perp = bl.nz;
    f.vg_rel = f.static_is_left ? br.vg : bl.vg;
    ifaces.push_back(f);
  }

  // Elements in global id order (single rank owns everything).
  for (int b = 0; b < nb; ++b)
    for (int ix = 0; ix < bands[b].nx; ++ix)
      for (int iy = 0; iy < bands[b].ny; ++iy)
        for (int iz = 0; iz < bands[b].nz; ++iz) elems.push_back({b, ix, iy, iz});
  const int ne = static_cast<int>(elems.size());

  // Faces (face_topology.cpp:55-150): y and z within the band (periodic or
  // Dirichlet), x across bands (conforming, sliding, or Dirichlet).
  sliding.assign(ifaces.size(), {});
  for (int e = 0; e < ne; ++e) {
    const Elem& el = elems[e];
    const Band& bd = bands[el.band];
    // y
    if (el.iy + 1 == bd.ny && !s.periodic_y) dirichlet.push_back({e, YP});
    else interior.push_back({e, static_cast<int>(gid(el.band, el.ix, (el.iy + 1) % bd.ny, el.iz)), 1,
                             (el.iy + 1 == bd.ny) ? 1 : 0});
    if (el.iy == 0 && !s.periodic_y) dirichlet.push_back({e, YM});
    // z
    if (el.iz + 1 == bd.nz && !s.periodic_z) dirichlet.push_back({e, ZP});
    else interior.push_back({e, static_cast<int>(gid(el.band, el.ix, el.iy, (el.iz + 1) % bd.nz)), 2});
    if (el.iz == 0 && !s.periodic_z) dirichlet.push_back({e, ZM});
    // x
    for (const bool plus : {true, false}) {
      int ob = -1, oix = 0;
      int iface = -1, nci = -1;
      bool exists = true;
      if (plus && el.ix + 1 < bd.nx) {
        ob = el.band;
        oix = el.ix + 1;
      } else if (!plus && el.ix > 0) {
        ob = el.band;
        oix = el.ix - 1;
      } else {
        int other = plus ? el.band + 1 : el.band - 1;
        if (other < 0 || other >= nb) {
          if (!s.periodic_x) exists = false;
          other = (other + nb) % nb;
        }
        if (exists) {
          if (nb == 1) {
            ob = el.band;
            oix = plus ? 0 : bd.nx - 1;
          } else {
            const int left = plus ? el.band : other;
            const int right = plus ? other : el.band;
            for (size_t i = 0; i < ifaces.size(); ++i)
              if (ifaces[i].left == left && ifaces[i].right == right) iface = static_cast<int>(i);
            for (size_t i = 0; i < ncs.size(); ++i)
              if (ncs[i].left == left && ncs[i].right == right) nci = static_cast<int>(i);
            ob = other;
            oix = plus ? 0 : bands[other].nx - 1;
          }
        }
      }
      if (!exists) {
        dirichlet.push_back({e, plus ? XP : XM});
        continue;
      }
      if (iface >= 0) {
        sliding[iface].push_back({e, plus ? XP : XM, el.iy, el.iz});
        continue;
      }
      if (nci >= 0) {
        NcIface& f = ncs[nci];
        const int sd = plus ? 0 : 1;  // A: the left band's x+ faces
        f.elem[sd][el.iy * f.nfz[sd] + el.iz] = e;
        f.side[sd][el.iy * f.nfz[sd] + el.iz] = plus ? XP : XM;
        continue;
      }
      if (plus) interior.push_back({e, static_cast<int>(gid(ob, oix, el.iy, el.iz)), 0});
    }
  }

  // Interface-side contexts (solver.cpp:73-90); faces ordered by (i_par, i_perp).
  for (size_t ic = 0; ic < ifaces.size(); ++ic)
    for (const bool left_side : {true, false}) {
      Ctx c;
      c.iface = static_cast<int>(ic);
      for (const auto& sf : sliding[ic])
        if ((sf.side == XP) == left_side) c.faces.push_back(sf);
      if (c.faces.empty()) continue;
      c.on_static = (ifaces[ic].static_is_left == left_side);
      std::sort(c.faces.begin(), c.faces.end(), [](const SlidingFace& a, const SlidingFace& b) {
        if (a.i_par != b.i_par) return a.i_par < b.i_par;
        return a.i_perp < b.i_perp;
      });
      // Rank maps (init_rank_maps, solver.cpp:95-133): one rank owns all.
      for (RankMap* mp : {&c.static_map, &c.moving_map}) {
        mp->n_par = ifaces[ic].n_faces;
        mp->n_perp = ifaces[ic].n_perp;
        mp->ranks.assign(static_cast<size_t>(mp->n_par * mp->n_perp), 0);
      }
      c.fwd.assign(2 * n2, 0.0);
      c.bwd.assign(2 * n2, 0.0);
      const int id = static_cast<int>(ctxs.size());
      (c.on_static ? static_ids : moving_ids).push_back(id);
      ctxs.push_back(std::move(c));
    }

  lifting = gas.viscous();
  const size_t nn = static_cast<size_t>(ne) * n3 * NV;
  field.assign(nn, 0.0);
  reg.assign(nn, 0.0);
  dudt.assign(nn, 0.0);
  grad.assign(static_cast<size_t>(ne) * n3 * NG, 0.0);
  trace.assign(static_cast<size_t>(ne) * 6 * n2 * NV, 0.0);
  fflux.assign(static_cast<size_t>(ne) * 6 * n2 * NV, 0.0);
  gtrace.assign(static_cast<size_t>(ne) * 6 * n2 * NG, 0.0);
  lift.assign(static_cast<size_t>(ne) * 6 * n2 * 4, 0.0);
  if (s.mapping != SDG_MAP_BOX && s.mapping != SDG_MAP_WARP && s.mapping != SDG_MAP_ANNULUS)
    throw ConfigError("unknown mesh mapping");
  curved = s.mapping != SDG_MAP_BOX;
  annulus = s.mapping == SDG_MAP_ANNULUS;
  if (annulus) {
    if (!(s.z0 > 0.0)) throw ConfigError("annulus needs a positive inner radius (z0 > 0)");
    if (s.periodic_z) throw ConfigError("annulus: the radial direction cannot be periodic");
    if (s.periodic_y && std::abs(s.height - 2.0 * 3.14159265358979323846) > 1e-12) {
      const double m = 2.0 * 3.14159265358979323846 / s.height;
      if (!(std::abs(m - std::round(m)) < 1e-9) || m < 1.5)
        throw ConfigError("annulus: a periodic sector must divide the full circle (height = 2 pi / m)");
      sector = true;
      alpha = s.height;
    }
    mw = 13;
    fw = 6;
  }
  if (curved) {
    if (!std::isfinite(s.warp)) throw ConfigError("warp amplitude must be finite");
    build_metrics();
  }
}

// Metric terms of the curved mapping: conservative curl form (Kopriva 2006)
//   Ja^i_n = -e_i . curl_xi( I^N( X_l grad_xi X_m ) ),  (n, m, l) cyclic,
// on the degree-N LGL interpolant of the mapping, then interpolated to the
// solution nodes; J = det(dX/dxi) of the interpolant.  Assembled in long
// double on coordinates relative to the element centre and rounded once, so
// the discrete metric identities hold to the rounding of the stored terms
// (free-stream preservation).  Face metrics (unit
// normal along +xi_d and sJ) come from the Ja^d of the LGL face layer, which
// depends on the face's geometry only; the minus element's values are copied
// to the plus element so that both see identical bits.
void orc_solver::build_metrics() {
  const Nodes lgl(ns.degree, SDG_NODES_LGL);
  const Basis bl = make_basis(lgl);
  std::vector<double> Ld(static_cast<size_t>(n) * n);  // L[s][p] = l_p(x_s), LGL -> solution nodes
  for (int a = 0; a < n; ++a) lgl.lagrange_all(ns.x[a], Ld.data() + a * n);
  const std::vector<ld> L(Ld.begin(), Ld.end());
  const std::vector<ld> DL(bl.D.begin(), bl.D.end());
  const int ne = static_cast<int>(elems.size());
  met.assign(static_cast<size_t>(ne) * n3 * mw, 0.0);
  fmet.assign(static_cast<size_t>(ne) * 6 * n2 * fw, 0.0);
  auto idx = [&](int p, int q, int r) { return (p * n + q) * n + r; };
  // d/dxi_d of a grid function on the LGL grid.
  auto deriv = [&](const ld* f, int d, ld* out) {
    for (int p = 0; p < n; ++p)
      for (int q = 0; q < n; ++q)
        for (int r = 0; r < n; ++r) {
          ld acc = 0.0L;
          for (int m = 0; m < n; ++m) {
            const ld dm = DL[(d == 0 ? p : (d == 1 ? q : r)) * n + m];
            acc += dm * f[d == 0 ? idx(m, q, r) : (d == 1 ? idx(p, m, r) : idx(p, q, m))];
          }
          out[idx(p, q, r)] = acc;
        }
  };
  // LGL grid -> solution nodes, one direction at a time.
  auto interp3 = [&](const ld* f, ld* out) {
    std::vector<ld> t1(n3), t2(n3);
    for (int a = 0; a < n; ++a)
      for (int q = 0; q < n; ++q)
        for (int r = 0; r < n; ++r) {
          ld acc = 0.0L;
          for (int p = 0; p < n; ++p) acc += L[a * n + p] * f[idx(p, q, r)];
          t1[idx(a, q, r)] = acc;
        }
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b)
        for (int r = 0; r < n; ++r) {
          ld acc = 0.0L;
          for (int q = 0; q < n; ++q) acc += L[b * n + q] * t1[idx(a, q, r)];
          t2[idx(a, b, r)] = acc;
        }
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b)
        for (int c = 0; c < n; ++c) {
          ld acc = 0.0L;
          for (int r = 0; r < n; ++r) acc += L[c * n + r] * t2[idx(a, b, r)];
          out[idx(a, b, c)] = acc;
        }
  };
  std::exception_ptr first;
#pragma omp parallel for schedule(static)
  for (int e = 0; e < ne; ++e) try {
    std::vector<ld> X(3 * n3), dX(9 * n3), V(3 * n3), dV(n3), JaL(9 * n3, 0.0L), Ja(9 * n3), dXs(9 * n3);
    // Coordinates relative to the element centre, in long double (the curl
    // form is translation invariant; the two elements of a face then see the
    // same face geometry up to an exact translation).
    for (int p = 0; p < n; ++p)
      for (int q = 0; q < n; ++q)
        for (int r = 0; r < n; ++r) {
          ld x[3];
          relative_position(e, lgl.x[p], lgl.x[q], lgl.x[r], x);
          for (int c = 0; c < 3; ++c) X[c * n3 + idx(p, q, r)] = x[c];
        }
    for (int d = 0; d < 3; ++d)
      for (int c = 0; c < 3; ++c) deriv(X.data() + c * n3, d, dX.data() + (3 * d + c) * n3);
    for (int nn = 0; nn < 3; ++nn) {
      const int m = (nn + 1) % 3, l = (nn + 2) % 3;
      // Invariant curl form (Kopriva 2006): V = (X_l grad X_m - X_m grad X_l) / 2 is an
      // antisymmetric bilinear form, so the metrics are covariant under rotations
      // (a periodic annulus sector reproduces its part of the full annulus).
      for (int d = 0; d < 3; ++d)
        for (int g = 0; g < n3; ++g)
          V[d * n3 + g] = 0.5L * (X[l * n3 + g] * dX[(3 * d + m) * n3 + g] - X[m * n3 + g] * dX[(3 * d + l) * n3 + g]);
      // Ja^i_nn = -(curl V)_i, (curl V)_i = d_{i+1} V_{i+2} - d_{i+2} V_{i+1}.
      for (int i = 0; i < 3; ++i) {
        const int i1 = (i + 1) % 3, i2 = (i + 2) % 3;
        ld* out = JaL.data() + (3 * i + nn) * n3;
        deriv(V.data() + i2 * n3, i1, dV.data());
        for (int g = 0; g < n3; ++g) out[g] = -dV[g];
        deriv(V.data() + i1 * n3, i2, dV.data());
        for (int g = 0; g < n3; ++g) out[g] += dV[g];
      }
    }
    for (int c = 0; c < 9; ++c) {
      interp3(JaL.data() + c * n3, Ja.data() + c * n3);
      interp3(dX.data() + c * n3, dXs.data() + c * n3);
    }
    // Annulus: contravariant grid velocity per unit angular speed,
    // V^d = Ja^d . (vg / omega) = [curl_xi I^N(psi grad_xi X)]_d with psi = r^2 / 2
    // (vg / omega = curl(psi e_x) = (0, Z, -Y)), discretely divergence free.
    std::vector<ld> VL(3 * n3, 0.0L), Vs(3 * n3, 0.0L);
    if (annulus) {
      std::vector<ld> At(3 * n3);
      for (int p = 0; p < n; ++p)
        for (int q = 0; q < n; ++q)
          for (int r = 0; r < n; ++r) {
            const ld rr = radius(e, lgl.x[p], lgl.x[q], lgl.x[r]);
            for (int k = 0; k < 3; ++k) At[k * n3 + idx(p, q, r)] = 0.5L * rr * rr * dX[(3 * k + 0) * n3 + idx(p, q, r)];
          }
      for (int i = 0; i < 3; ++i) {
        const int i1 = (i + 1) % 3, i2 = (i + 2) % 3;
        deriv(At.data() + i2 * n3, i1, dV.data());
        for (int g = 0; g < n3; ++g) VL[i * n3 + g] = dV[g];
        deriv(At.data() + i1 * n3, i2, dV.data());
        for (int g = 0; g < n3; ++g) VL[i * n3 + g] -= dV[g];
        interp3(VL.data() + i * n3, Vs.data() + i * n3);
      }
    }
    for (int g = 0; g < n3; ++g) {
      double* o = met.data() + (static_cast<size_t>(e) * n3 + g) * mw;
      if (annulus)
        for (int i = 0; i < 3; ++i) o[10 + i] = static_cast<double>(Vs[i * n3 + g]);
      for (int c = 0; c < 9; ++c) o[c] = static_cast<double>(Ja[c * n3 + g]);
      // dXs[(3 d + c)] = dX_c / dxi_d; J = det.
      const ld a00 = dXs[0 * n3 + g], a01 = dXs[1 * n3 + g], a02 = dXs[2 * n3 + g];
      const ld a10 = dXs[3 * n3 + g], a11 = dXs[4 * n3 + g], a12 = dXs[5 * n3 + g];
      const ld a20 = dXs[6 * n3 + g], a21 = dXs[7 * n3 + g], a22 = dXs[8 * n3 + g];
      const ld jac = a00 * (a11 * a22 - a12 * a21) - a01 * (a10 * a22 - a12 * a20) + a02 * (a10 * a21 - a11 * a20);
      if (!(jac > 0.0)) throw ConfigError("curved mapping has a non-positive Jacobian (warp too large)");
      o[9] = static_cast<double>(1.0L / jac);
    }
    for (int side = 0; side < 6; ++side) {
      const int d = side / 2, layer = (side & 1) ? n - 1 : 0;
      double* o = fmet.data() + (static_cast<size_t>(e) * 6 + side) * n2 * fw;
      for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
          ld ns3[4];
          for (int c = 0; c < (annulus ? 4 : 3); ++c) {
            const ld* f = c < 3 ? JaL.data() + (3 * d + c) * n3 : VL.data() + d * n3;
            ld acc = 0.0L;
            for (int u = 0; u < n; ++u) {
              ld inner = 0.0L;
              for (int v = 0; v < n; ++v) {
                const int g = d == 0 ? idx(layer, u, v) : (d == 1 ? idx(u, layer, v) : idx(u, v, layer));
                inner += L[b * n + v] * f[g];
              }
              acc += L[a * n + u] * inner;
            }
            ns3[c] = acc;
          }
          const ld sj = std::sqrt(ns3[0] * ns3[0] + ns3[1] * ns3[1] + ns3[2] * ns3[2]);
          double* q = o + (a * n + b) * fw;
          for (int c = 0; c < 3; ++c) q[c] = static_cast<double>(ns3[c] / sj);
          q[3] = static_cast<double>(sj);
          if (annulus) q[4] = static_cast<double>(ns3[3] / sj);  // (vg / omega) . n
        }
    }
  } catch (...) {
#pragma omp critical
    if (!first) first = std::current_exception();
  }
  if (first) std::rethrow_exception(first);
  for (const auto& f : interior) {
    if (sector && f.seam) continue;  // the two slots differ by the sector rotation
    const double* src = fm(f.em, 2 * f.dir + 1);
    std::copy(src, src + n2 * fw, fmet.data() + (static_cast<size_t>(f.ep) * 6 + 2 * f.dir) * n2 * fw);
  }
}

// update_interfaces (solver.cpp:156-176).
void orc_solver::update_interfaces(double t_stage) {
  bool st_topo = false, mv_topo = false;
  for (auto& c : ctxs) {
    const Iface& f = ifaces[c.iface];
    const double delta = c.delta_base + f.vg_rel * (t_stage - time);
    c.st = displacement(delta, f.l_par, f.n_faces);
    c.conforming = c.st.conforming();
    {  // windings of the moving band: delta = d + K * period (displacement() wraps d to [0, period))
      const double period = f.l_par * static_cast<double>(f.n_faces);
      double dd = std::fmod(delta, period);
      if (dd < 0.0) dd += period;
      c.K = c.wraps + std::lround((delta - dd) / period);
      if (dd / f.l_par >= static_cast<double>(f.n_faces)) c.K += 1;  // d rounded up to the period
    }
    const double sigma = 2.0 * c.st.s_delta - 1.0;
    c.sigma_side = c.on_static ? sigma : -sigma;
    if (!c.conforming) mortar_ops(ns, c.sigma_side, c.fwd.data(), c.bwd.data());
    if (!c.topo_valid || c.st.n_delta != c.last_n || c.conforming != c.last_conf) {
      c.topo_valid = true;
      c.last_n = c.st.n_delta;
      c.last_conf = c.conforming;
      c.rebuilds++;
      (c.on_static ? st_topo : mv_topo) = true;
    }
  }
  if (st_topo) rebuild_role(statics, static_ids);
  if (mv_topo) rebuild_role(movings, moving_ids);
}

// rebuild_role (solver.cpp:178-206).
void orc_solver::rebuild_role(Role& role, const std::vector<int>& ids) {
  role.cols.clear();
  auto local_faces = [&](const Ctx& c) {
    std::vector<LocalFace> fs(c.faces.size());
    for (size_t f = 0; f < c.faces.size(); ++f) fs[f] = {static_cast<long>(f), c.faces[f].i_par, c.faces[f].i_perp};
    return fs;
  };
  for (const int id : ids) {
    const Ctx& c = ctxs[id];
    append_tuples(local_faces(c), c.on_static ? c.moving_map : c.static_map, c.st.n_delta,
                  ifaces[c.iface].n_faces, c.on_static, c.conforming, c.iface, id, role.cols);
  }
  sort_tuples(role.cols);
  for (const int id : ids) {
    Ctx& c = ctxs[id];
    const long nf = static_cast<long>(c.faces.size());
    c.m[0].assign(nf, -1);
    c.m[1].assign(nf, -1);
    for (int i = 0; i < static_cast<int>(role.cols.size()); ++i)
      if (role.cols[i].ctx == id) c.m[role.cols[i].i_sub][role.cols[i].i_face] = i;
  }
  role.sched = make_schedule(role.cols, 0, role.self);
  role.n_mortars = static_cast<int>(role.cols.size());
  const size_t nodes = static_cast<size_t>(role.n_mortars) * n2;
  role.u_mine.assign(nodes * NV, 0.0);
  role.u_theirs.assign(nodes * NV, 0.0);
  role.flux.assign(nodes * NV, 0.0);
  role.lift.assign(nodes * 4, 0.0);
  role.g_mine.assign(nodes * NG, 0.0);
  role.g_theirs.assign(nodes * NG, 0.0);
}

// Face traces U(+-1) per side (solver.cpp:208-232), sums in normal-index order.
void orc_solver::prolong(const double* u) {
  const int ne = static_cast<int>(elems.size());
  const double* fl = basis.fl.data();
  const double* fr = basis.fr.data();
#pragma omp parallel for schedule(static)
  for (int e = 0; e < ne; ++e) {
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b)
        for (int v = 0; v < NV; ++v) {
          double xm = 0.0, xp = 0.0, ym = 0.0, yp = 0.0, zm = 0.0, zp = 0.0;
          for (int m = 0; m < n; ++m) {
            const double px = u[node(e, m, a, b) * NV + v];  // x-line at (j,k) = (a,b)
            xm += fl[m] * px;
            xp += fr[m] * px;
            const double py = u[node(e, a, m, b) * NV + v];  // y-line at (i,k) = (a,b)
            ym += fl[m] * py;
            yp += fr[m] * py;
            const double pz = u[node(e, a, b, m) * NV + v];  // z-line at (i,j) = (a,b)
            zm += fl[m] * pz;
            zp += fr[m] * pz;
          }
          const int fn = a * n + b;
          tr(e, XM)[fn * NV + v] = xm;
          tr(e, XP)[fn * NV + v] = xp;
          tr(e, YM)[fn * NV + v] = ym;
          tr(e, YP)[fn * NV + v] = yp;
          tr(e, ZM)[fn * NV + v] = zm;
          tr(e, ZP)[fn * NV + v] = zp;
        }
  }
}

// Face -> mortar transfer along the sliding axis (j) for every k line
// (apply_line, mortar.cpp:152-173); nc components per node.
static void face_to_mortar(const double* op, int n, const double* in, double* out, int nc) {
  for (int k = 0; k < n; ++k)
    for (int i = 0; i < n; ++i)
      for (int c = 0; c < nc; ++c) {
        double acc = 0.0;
        for (int j = 0; j < n; ++j) acc += op[i * n + j] * in[(j * n + k) * nc + c];
        out[(i * n + k) * nc + c] = acc;
      }
}

// fill_mortar_solution (solver.cpp:234-252).
void orc_solver::fill_mortar_solution() {
  for (auto& c : ctxs) {
    Role& role = c.on_static ? statics : movings;
    for (size_t f = 0; f < c.faces.size(); ++f) {
      const double* line = tr(c.faces[f].e, c.faces[f].side);
      if (c.conforming) {
        std::copy(line, line + n2 * NV, role.u_mine.data() + static_cast<size_t>(c.m[1][f]) * n2 * NV);
      } else {
        for (int s = 0; s < 2; ++s)
          face_to_mortar(c.fwd.data() + c.half(s) * n2, n, line,
                         role.u_mine.data() + static_cast<size_t>(c.m[s][f]) * n2 * NV, NV);
      }
    }
  }
}

// send_solution_phase self loop-back (solver.cpp:273-280).
void orc_solver::exchange_solution() {
  if (movings.self.count > 0) {
    if (movings.self.count != statics.self.count) throw ProtocolError("loopback mortar block size mismatch");
    std::copy_n(movings.u_mine.begin() + static_cast<size_t>(movings.self.offset) * n2 * NV,
                static_cast<size_t>(movings.self.count) * n2 * NV,
                statics.u_theirs.begin() + static_cast<size_t>(statics.self.offset) * n2 * NV);
  }
}

// Mortar -> face back projection of two sub-mortars (solver.cpp:688-714, 495-526).
static void mortar_to_face(const Ctx& c, int n, const double* role_data, size_t f, int nc, double* out) {
  const int n2 = n * n;
  for (int q = 0; q < n2 * nc; ++q) out[q] = 0.0;
  for (int s = 0; s < 2; ++s) {
    const double* op = c.bwd.data() + c.half(s) * n2;
    const double* src = role_data + static_cast<size_t>(c.m[s][f]) * n2 * nc;
    for (int k = 0; k < n; ++k)
      for (int i = 0; i < n; ++i)
        for (int cc = 0; cc < nc; ++cc) {
          double acc = 0.0;
          for (int j = 0; j < n; ++j) acc += op[i * n + j] * src[(j * n + k) * nc + cc];
          out[(i * n + k) * nc + cc] += acc;
        }
  }
}

// run_lifting (solver.cpp:597-727).
void orc_solver::run_lifting(double t_stage, const double* u) {
  const int nif = static_cast<int>(interior.size());
#pragma omp parallel for schedule(static)
  for (int fi = 0; fi < nif; ++fi) {
    const InteriorFace& f = interior[fi];
    const int sm = 2 * f.dir + 1, sp = 2 * f.dir;
    const double* um = tr(f.em, sm);
    const double* up = tr(f.ep, sp);
    double* lm = lf(f.em, sm);
    double* lp = lf(f.ep, sp);
    const bool seam = sector && f.seam;
    for (int k = 0; k < n2; ++k) {
      double a[4], b[4];
      prim4(um + k * NV, gas, a);
      prim4(up + k * NV, gas, b);
      if (seam) {  // the plus element's values at theta ~ 0 seen from theta ~ alpha, and back
        double br[4], lmv[4];
        rot_prim(1, b, br);
        for (int c = 0; c < 4; ++c) lmv[c] = 0.5 * (a[c] + br[c]);
        rot_prim(-1, lmv, lp + k * 4);
        for (int c = 0; c < 4; ++c) lm[k * 4 + c] = lmv[c];
        continue;
      }
      for (int c = 0; c < 4; ++c) lm[k * 4 + c] = lp[k * 4 + c] = 0.5 * (a[c] + b[c]);
    }
  }
  // Sliding mortars: the static side computes the mean, moving receives it.
  if (statics.n_mortars > 0) {
    const size_t nodes = static_cast<size_t>(statics.n_mortars) * n2;
    for (size_t q = 0; q < nodes; ++q) {
      double a[4], b[4], th[NV];
      prim4(statics.u_mine.data() + q * NV, gas, a);
      // the moving partner's state at the static location (periodic sector: R(-k alpha))
      if (sector) rot_state(-mortar_k(statics.cols[q / n2]), statics.u_theirs.data() + q * NV, th);
      else std::copy_n(statics.u_theirs.data() + q * NV, NV, th);
      prim4(th, gas, b);
      for (int c = 0; c < 4; ++c) statics.lift[q * 4 + c] = 0.5 * (a[c] + b[c]);
    }
    if (statics.self.count > 0)
      std::copy_n(statics.lift.begin() + static_cast<size_t>(statics.self.offset) * n2 * 4,
                  static_cast<size_t>(statics.self.count) * n2 * 4,
                  movings.lift.begin() + static_cast<size_t>(movings.self.offset) * n2 * 4);
  }
  const std::vector<double> mv_lift = to_moving_frame(movings, movings.lift, 4, 0);
  for (const auto& c : ctxs) {
    const double* data = c.on_static ? statics.lift.data() : mv_lift.data();
    for (size_t f = 0; f < c.faces.size(); ++f) {
      double* lout = lf(c.faces[f].e, c.faces[f].side);
      if (c.conforming) {
        std::copy_n(data + static_cast<size_t>(c.m[1][f]) * n2 * 4, n2 * 4, lout);
        continue;
      }
      mortar_to_face(c, n, data, f, 4, lout);
    }
  }
  nc_lift();
  for (const auto& df : dirichlet) {
    double* lout = lf(df.e, df.side);
    for (int p = 0; p < n; ++p)
      for (int q = 0; q < n; ++q) {
        double x[3];
        face_node_position(df.e, df.side, p, q, t_stage, x);
        const State ext = eval_case(flow_case, x, t_stage, gas);
        prim4(ext.data(), gas, lout + (p * n + q) * 4);
      }
  }
  assemble_gradients(u);
  send_gradients();
}

// assemble_gradients (solver.cpp:729-791): BR1 gradients of (v1, v2, v3, T).
void orc_solver::assemble_gradients(const double* u) {
  if (curved) {
    assemble_gradients_curved(u);
    return;
  }
  const int ne = static_cast<int>(elems.size());
  const double* w = ns.w.data();
  const double* fl = basis.fl.data();
  const double* fr = basis.fr.data();
#pragma omp parallel
  {
    std::vector<double> q(static_cast<size_t>(n3) * 4);
#pragma omp for schedule(static)
    for (int e = 0; e < ne; ++e) {
      const Band& b = bands[elems[e].band];
      const double jac = 0.125 * b.hx * b.hy * b.hz;
      const double cx = (0.25 * b.hy * b.hz) / jac;
      const double cy = (0.25 * b.hx * b.hz) / jac;
      const double cz = (0.25 * b.hx * b.hy) / jac;
      for (int nd = 0; nd < n3; ++nd) prim4(u + (static_cast<size_t>(e) * n3 + nd) * NV, gas, q.data() + nd * 4);
      const double* sxm = lf(e, XM);
      const double* sxp = lf(e, XP);
      const double* sym = lf(e, YM);
      const double* syp = lf(e, YP);
      const double* szm = lf(e, ZM);
      const double* szp = lf(e, ZP);
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
          for (int k = 0; k < n; ++k) {
            double* g = grad.data() + node(e, i, j, k) * NG;
            for (int c = 0; c < 4; ++c) {
              double vx = 0.0, vy = 0.0, vz = 0.0;
              for (int m = 0; m < n; ++m) {
                vx += wdiff[i * n + m] * q[((m * n + j) * n + k) * 4 + c];
                vy += wdiff[j * n + m] * q[((i * n + m) * n + k) * 4 + c];
                vz += wdiff[k * n + m] * q[((i * n + j) * n + m) * 4 + c];
              }
              const double sx = (sxp[(j * n + k) * 4 + c] * fr[i] - sxm[(j * n + k) * 4 + c] * fl[i]) / w[i];
              const double sy = (syp[(i * n + k) * 4 + c] * fr[j] - sym[(i * n + k) * 4 + c] * fl[j]) / w[j];
              const double sz = (szp[(i * n + j) * 4 + c] * fr[k] - szm[(i * n + j) * 4 + c] * fl[k]) / w[k];
              g[3 * c + 0] = cx * (sx - vx);
              g[3 * c + 1] = cy * (sy - vy);
              g[3 * c + 2] = cz * (sz - vz);
            }
          }
      prolong_gradients(e);
    }
  }
}

// Prolong gradients to the faces (solver.cpp:770-790).
void orc_solver::prolong_gradients(int e) {
  const double* fl = basis.fl.data();
  const double* fr = basis.fr.data();
      for (int a = 0; a < n; ++a)
        for (int bb = 0; bb < n; ++bb)
          for (int c = 0; c < NG; ++c) {
            double xm = 0.0, xp = 0.0, ym = 0.0, yp = 0.0, zm = 0.0, zp = 0.0;
            for (int m = 0; m < n; ++m) {
              const double px = grad[node(e, m, a, bb) * NG + c];
              xm += fl[m] * px;
              xp += fr[m] * px;
              const double py = grad[node(e, a, m, bb) * NG + c];
              ym += fl[m] * py;
              yp += fr[m] * py;
              const double pz = grad[node(e, a, bb, m) * NG + c];
              zm += fl[m] * pz;
              zp += fr[m] * pz;
            }
            const int fn = a * n + bb;
            gt(e, XM)[fn * NG + c] = xm;
            gt(e, XP)[fn * NG + c] = xp;
            gt(e, YM)[fn * NG + c] = ym;
            gt(e, YP)[fn * NG + c] = yp;
            gt(e, ZM)[fn * NG + c] = zm;
            gt(e, ZP)[fn * NG + c] = zp;
          }
}

// Curved BR1 gradient, conservative weak form (the metric inside the derivative):
//   J g_c = sum_d [ (l_i(+1)/w_i) q*+ (n sJ)+_c - (l_i(-1)/w_i) q*- (n sJ)-_c
//                   - sum_m Dhat(i,m) Ja^d_c(m) q(m) ],
// with (n sJ) the +xi_d normal of the side; for affine metrics this is
// assemble_gradients above (solver.cpp:729-768).
void orc_solver::assemble_gradients_curved(const double* u) {
  const int ne = static_cast<int>(elems.size());
  const double* w = ns.w.data();
  const double* fl = basis.fl.data();
  const double* fr = basis.fr.data();
#pragma omp parallel
  {
    std::vector<double> q(static_cast<size_t>(n3) * 4);
#pragma omp for schedule(static)
    for (int e = 0; e < ne; ++e) {
      for (int nd = 0; nd < n3; ++nd) prim4(u + (static_cast<size_t>(e) * n3 + nd) * NV, gas, q.data() + nd * 4);
      std::vector<double> ja(static_cast<size_t>(n3) * 9), ns4(static_cast<size_t>(6) * n2 * 4);
      for (int nd = 0; nd < n3; ++nd) ja_at(e, nd, ja.data() + nd * 9);
      for (int sd = 0; sd < 6; ++sd)
        for (int f = 0; f < n2; ++f) {
          double vgn;
          double* o = ns4.data() + (sd * n2 + f) * 4;
          normal_at(e, sd, f, o, vgn);
          o[3] = fm(e, sd)[f * fw + 3];
        }
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
          for (int k = 0; k < n; ++k) {
            const int nd = (i * n + j) * n + k;
            const int ia[3] = {i, j, k};
            const int fidx[3] = {j * n + k, i * n + k, i * n + j};
            double* g = grad.data() + node(e, i, j, k) * NG;
            const double ij = mt(e, nd)[9];
            for (int c = 0; c < 4; ++c)
              for (int kk = 0; kk < 3; ++kk) {
                double vol = 0.0;
                for (int m = 0; m < n; ++m) {
                  const int mx = (m * n + j) * n + k, my = (i * n + m) * n + k, mz = (i * n + j) * n + m;
                  vol += wdiff[i * n + m] * ja[mx * 9 + 0 + kk] * q[mx * 4 + c] +
                         wdiff[j * n + m] * ja[my * 9 + 3 + kk] * q[my * 4 + c] +
                         wdiff[k * n + m] * ja[mz * 9 + 6 + kk] * q[mz * 4 + c];
                }
                double surf = 0.0;
                for (int d = 0; d < 3; ++d) {
                  const int f = fidx[d];
                  const double* np = ns4.data() + ((2 * d + 1) * n2 + f) * 4;
                  const double* nm = ns4.data() + ((2 * d) * n2 + f) * 4;
                  surf += (lf(e, 2 * d + 1)[f * 4 + c] * np[kk] * np[3] * fr[ia[d]] -
                           lf(e, 2 * d)[f * 4 + c] * nm[kk] * nm[3] * fl[ia[d]]) / w[ia[d]];
                }
                g[3 * c + kk] = ij * (surf - vol);
              }
          }
      prolong_gradients(e);
    }
  }
}

// send_gradient_phase mortar part + loop-back (solver.cpp:806-843).
void orc_solver::send_gradients() {
  for (auto& c : ctxs) {
    Role& role = c.on_static ? statics : movings;
    for (size_t f = 0; f < c.faces.size(); ++f) {
      const double* g = gt(c.faces[f].e, c.faces[f].side);
      if (c.conforming) {
        std::copy_n(g, n2 * NG, role.g_mine.begin() + static_cast<size_t>(c.m[1][f]) * n2 * NG);
        continue;
      }
      for (int s = 0; s < 2; ++s)
        face_to_mortar(c.fwd.data() + c.half(s) * n2, n, g,
                       role.g_mine.data() + static_cast<size_t>(c.m[s][f]) * n2 * NG, NG);
    }
  }
  if (movings.self.count > 0)
    std::copy_n(movings.g_mine.begin() + static_cast<size_t>(movings.self.offset) * n2 * NG,
                static_cast<size_t>(movings.self.count) * n2 * NG,
                statics.g_theirs.begin() + static_cast<size_t>(statics.self.offset) * n2 * NG);
}

// interior_face_phase (solver.cpp:323-341): minus-side oriented, vg_n from the minus element.
void orc_solver::interior_flux() {
  const int nif = static_cast<int>(interior.size());
  // Exceptions may not leave an OpenMP region: keep the first, rethrow after.
  std::exception_ptr first;
#pragma omp parallel for schedule(static)
  for (int fi = 0; fi < nif; ++fi) try {
    const InteriorFace& f = interior[fi];
    const int sm = 2 * f.dir + 1, sp = 2 * f.dir;
    const double* um = tr(f.em, sm);
    const double* up = tr(f.ep, sp);
    const Band& bm = bands[elems[f.em].band];
    const double vg_n = f.dir == 1 ? bm.vg : (f.dir == 2 ? bm.vgz : 0.0);
    double* om = ff(f.em, sm);
    double* op = ff(f.ep, sp);
    for (int k = 0; k < n2; ++k) {
      const double* gm = lifting ? gt(f.em, sm) + k * NG : nullptr;
      const double* gp = lifting ? gt(f.ep, sp) + k * NG : nullptr;
      if (curved && sector && f.seam) {
        // theta seam of a periodic sector: the plus element's trace and gradient rotated
        // into the minus element's frame; the plus side gets the flux rotated back.
        double nrm[3], vgn, upr[NV], gpr[NG];
        normal_at(f.em, sm, k, nrm, vgn);
        rot_state(1, up + k * NV, upr);
        if (gp) rot_grad(1, gp, gpr);
        face_flux_n(um + k * NV, upr, nrm, vgn, gm, gp ? gpr : nullptr, gas, om + k * NV);
        rot_state(-1, om + k * NV, op + k * NV);
        continue;
      }
      if (curved) {
        // +xi normal of the face (identical in both slots); vg_n = vg . n.
        double nrm[3], vgn;
        normal_at(f.em, sm, k, nrm, vgn);
        face_flux_n(um + k * NV, up + k * NV, nrm, vgn, gm, gp, gas, om + k * NV);
      } else
      face_flux(um + k * NV, up + k * NV, f.dir, vg_n, gm, gp, gas, om + k * NV);
      for (int v = 0; v < NV; ++v) op[k * NV + v] = om[k * NV + v];
    }
  } catch (...) {
#pragma omp critical
    if (!first) first = std::current_exception();
  }
  if (first) std::rethrow_exception(first);
}

// volume_kernel (solver.cpp:343-385): one accumulator per (node, var) over m
// for all three directions, then times 1/J.
void orc_solver::volume(const double* u, double* out) {
  const int ne = static_cast<int>(elems.size());
#pragma omp parallel
  {
    std::vector<double> fx(static_cast<size_t>(n3) * NV), fy(fx.size()), fz(fx.size());
#pragma omp for schedule(static)
    for (int e = 0; e < ne; ++e) {
      const Band& b = bands[elems[e].band];
      const double vg[3] = {0.0, annulus ? 0.0 : b.vg, annulus ? 0.0 : b.vgz};
      const double jac = 0.125 * b.hx * b.hy * b.hz;
      const double sjx = 0.25 * b.hy * b.hz, sjy = 0.25 * b.hx * b.hz, sjz = 0.25 * b.hx * b.hy;
      for (int nd = 0; nd < n3; ++nd) {
        const double* s = u + (static_cast<size_t>(e) * n3 + nd) * NV;
        double f[3][NV];
        ale_flux(s, vg, gas, f);
        if (lifting) {
          double fv[3][NV];
          viscous_flux(s, grad.data() + (static_cast<size_t>(e) * n3 + nd) * NG, gas, fv);
          for (int d = 0; d < 3; ++d)
            for (int v = 0; v < NV; ++v) f[d][v] -= fv[d][v];
        }
        if (curved) {
          // Contravariant flux Ja^d . F (the affine sJ_d F_d below).  Annulus: F holds
          // no grid velocity (vg = 0 above) and the rotating band's ALE term is
          // omega V^d u with the contravariant grid velocity V^d.
          double ja[9];
          ja_at(e, nd, ja);
          double wv[3] = {0.0, 0.0, 0.0};
          if (annulus)
            for (int d = 0; d < 3; ++d) wv[d] = b.vg * mt(e, nd)[10 + d];
          for (int v = 0; v < NV; ++v) {
            fx[nd * NV + v] = ja[0] * f[0][v] + ja[1] * f[1][v] + ja[2] * f[2][v] - wv[0] * s[v];
            fy[nd * NV + v] = ja[3] * f[0][v] + ja[4] * f[1][v] + ja[5] * f[2][v] - wv[1] * s[v];
            fz[nd * NV + v] = ja[6] * f[0][v] + ja[7] * f[1][v] + ja[8] * f[2][v] - wv[2] * s[v];
          }
          continue;
        }
        for (int v = 0; v < NV; ++v) {
          fx[nd * NV + v] = f[0][v] * sjx;
          fy[nd * NV + v] = f[1][v] * sjy;
          fz[nd * NV + v] = f[2][v] * sjz;
        }
      }
      const double inv_jac = 1.0 / jac;
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
          for (int k = 0; k < n; ++k) {
            double* o = out + node(e, i, j, k) * NV;
            for (int v = 0; v < NV; ++v) {
              double acc = 0.0;
              for (int m = 0; m < n; ++m)
                acc += wdiff[i * n + m] * fx[((m * n + j) * n + k) * NV + v] +
                       wdiff[j * n + m] * fy[((i * n + m) * n + k) * NV + v] +
                       wdiff[k * n + m] * fz[((i * n + j) * n + m) * NV + v];
              o[v] = acc * (curved ? mt(e, (i * n + j) * n + k)[9] : inv_jac);
            }
          }
    }
  }
}

// mortar_flux_phase (solver.cpp:442-479): static side, normal = x, vg_n = 0.
void orc_solver::mortar_flux() {
  if (statics.n_mortars == 0) return;
  for (int c = 0; c < statics.n_mortars; ++c) {
    const Ctx& cx = ctxs[statics.cols[c].ctx];
    const bool static_left = ifaces[cx.iface].static_is_left;
    for (int k = 0; k < n2; ++k) {
      const size_t q = static_cast<size_t>(c) * n2 + k;
      const double* mine = statics.u_mine.data() + q * NV;
      const double* theirs = statics.u_theirs.data() + q * NV;
      const double* gm = lifting ? statics.g_mine.data() + q * NG : nullptr;
      const double* gt_ = lifting ? statics.g_theirs.data() + q * NG : nullptr;
      double thr[NV], gtr[NG];
      if (sector) {  // the moving partner's values at the static location: R(-k alpha)
        const int kk = -mortar_k(statics.cols[c]);
        rot_state(kk, theirs, thr);
        theirs = thr;
        if (gt_) {
          rot_grad(kk, gt_, gtr);
          gt_ = gtr;
        }
      }
      double* o = statics.flux.data() + q * NV;
      if (static_left) face_flux(mine, theirs, 0, 0.0, gm, gt_, gas, o);
      else face_flux(theirs, mine, 0, 0.0, gt_, gm, gas, o);
    }
  }
  if (statics.self.count > 0)
    std::copy_n(statics.flux.begin() + static_cast<size_t>(statics.self.offset) * n2 * NV,
                static_cast<size_t>(statics.self.count) * n2 * NV,
                movings.flux.begin() + static_cast<size_t>(movings.self.offset) * n2 * NV);
}

// mortar_apply_phase (solver.cpp:495-526).
void orc_solver::mortar_apply() {
  const std::vector<double> mv_flux = to_moving_frame(movings, movings.flux, NV, 1);
  for (const auto& c : ctxs) {
    const double* data = c.on_static ? statics.flux.data() : mv_flux.data();
    for (size_t f = 0; f < c.faces.size(); ++f) {
      double* o = ff(c.faces[f].e, c.faces[f].side);
      if (c.conforming) {
        std::copy_n(data + static_cast<size_t>(c.m[1][f]) * n2 * NV, n2 * NV, o);
        continue;
      }
      mortar_to_face(c, n, data, f, NV, o);
    }
  }
}

// dirichlet_phase (solver.cpp:528-545).
void orc_solver::dirichlet_flux(double t_stage) {
  for (const auto& df : dirichlet) {
    const double* mine = tr(df.e, df.side);
    double* o = ff(df.e, df.side);
    const int dir = df.side / 2;
    const bool plus = (df.side % 2) == 1;
    const Band& bd = bands[elems[df.e].band];
    const double vg_n = dir == 1 ? bd.vg : (dir == 2 ? bd.vgz : 0.0);
    for (int p = 0; p < n; ++p)
      for (int q = 0; q < n; ++q) {
        const int k = p * n + q;
        double x[3];
        face_node_position(df.e, df.side, p, q, t_stage, x);
        const State ext = eval_case(flow_case, x, t_stage, gas);
        const double* g = lifting ? gt(df.e, df.side) + k * NG : nullptr;
        if (curved) {
          double nrm[3], vgn;
          normal_at(df.e, df.side, k, nrm, vgn);
          if (plus) face_flux_n(mine + k * NV, ext.data(), nrm, vgn, g, g, gas, o + k * NV);
          else face_flux_n(ext.data(), mine + k * NV, nrm, vgn, g, g, gas, o + k * NV);
          continue;
        }
        if (plus) face_flux(mine + k * NV, ext.data(), dir, vg_n, g, g, gas, o + k * NV);
        else face_flux(ext.data(), mine + k * NV, dir, vg_n, g, g, gas, o + k * NV);
      }
  }
}

// apply_all_faces (solver.cpp:547-582): sides in order X-, X+, Y-, Y+, Z-, Z+.
void orc_solver::apply_faces(double* out) {
  const int ne = static_cast<int>(elems.size());
  const double* w = ns.w.data();
#pragma omp parallel for schedule(static)
  for (int e = 0; e < ne; ++e) {
    const Band& b = bands[elems[e].band];
    const double jac = 0.125 * b.hx * b.hy * b.hz;
    const double cdir[3] = {(0.25 * b.hy * b.hz) / jac, (0.25 * b.hx * b.hz) / jac, (0.25 * b.hx * b.hy) / jac};
    for (int side = 0; side < 6; ++side) {
      const double* line = ff(e, side);
      const int dir = side / 2;
      const bool plus = side % 2 == 1;
      const double sgn = plus ? -1.0 : 1.0;
      const double* lift_v = plus ? basis.fr.data() : basis.fl.data();
      for (int a = 0; a < n; ++a) {
        const double c = sgn * cdir[dir] * lift_v[a] / w[a];
        if (c == 0.0) continue;
        for (int p = 0; p < n; ++p)
          for (int q = 0; q < n; ++q) {
            int i, j, k;
            if (dir == 0) { i = a; j = p; k = q; }
            else if (dir == 1) { i = p; j = a; k = q; }
            else { i = p; j = q; k = a; }
            double* o = out + node(e, i, j, k) * NV;
            // Curved: (sJ / J) of the face node and the volume node.
            const double cc = curved ? sgn * (lift_v[a] / w[a]) * fm(e, side)[(p * n + q) * fw + 3] *
                                           mt(e, (i * n + j) * n + k)[9]
                                     : c;
            for (int v = 0; v < NV; ++v) o[v] += cc * line[(p * n + q) * NV + v];
          }
      }
    }
  }
}

// compute_residual (solver.cpp:846-870), single rank.
void orc_solver::residual(double t_stage, const double* u, double* out) {
  t_cur = t_stage;
  update_interfaces(t_stage);
  prolong(u);
  fill_mortar_solution();
  exchange_solution();
  nc_update(t_stage);
  if (lifting) run_lifting(t_stage, u);
  interior_flux();
  volume(u, out);
  mortar_flux();
  mortar_apply();
  nc_flux();
  dirichlet_flux(t_stage);
  apply_faces(out);
}

// ---------------------------------------------------------------------------
// Non-matching / oblique interfaces: the reference's mortar chain (fill
// solver.cpp:234-252, lifting mean :597-727, flux :442-479, apply :495-526) on
// the tensor-product mortars of a y row and a z row of face intervals.
// ---------------------------------------------------------------------------
// (Fy x Fz) applied to one face's n x n x nc block: out[k][l] = sum_ij Fy[k][i] Fz[l][j] in[i][j].
static void tensor_apply(const double* fy, const double* fz, int n, const double* in, double* out, int nc) {
  for (int k = 0; k < n; ++k)
    for (int l = 0; l < n; ++l)
      for (int c = 0; c < nc; ++c) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < n; ++j) acc += fy[k * n + i] * fz[l * n + j] * in[(i * n + j) * nc + c];
        out[(k * n + l) * nc + c] = acc;
      }
}

// Displacement, rows and operators of the stage; the mortar traces of both sides.
void orc_solver::nc_update(double t_stage) {
  for (auto& f : ncs) {
    f.dy = f.dy_base + f.vy_rel * (t_stage - time);
    f.dz = f.dz_base + f.vz_rel * (t_stage - time);
    f.rows[0] = intervals(f.nfy[0], f.nfy[1], f.ly[0], f.dy);
    f.rows[1] = intervals(f.nfz[0], f.nfz[1], f.lz[0], f.dz);
    for (int d = 0; d < 2; ++d)
      for (int sd = 0; sd < 2; ++sd) {
        const size_t m = f.rows[d].size();
        f.F[sd][d].assign(m * n2, 0.0);
        f.B[sd][d].assign(m * n2, 0.0);
        for (size_t k = 0; k < m; ++k) {
          const double* r = f.rows[d][k].r;
          subrange_ops(ns, r[2 * sd], r[2 * sd + 1], f.F[sd][d].data() + k * n2, f.B[sd][d].data() + k * n2);
        }
      }
    const size_t my = f.rows[0].size(), mz = f.rows[1].size();
    for (int sd = 0; sd < 2; ++sd) {
      f.u[sd].assign(my * mz * n2 * NV, 0.0);
      for (size_t ky = 0; ky < my; ++ky)
        for (size_t kz = 0; kz < mz; ++kz) {
          const long fy = sd ? f.rows[0][ky].fb : f.rows[0][ky].fa, fz = sd ? f.rows[1][kz].fb : f.rows[1][kz].fa;
          const size_t face = fy * f.nfz[sd] + fz;
          tensor_apply(f.F[sd][0].data() + ky * n2, f.F[sd][1].data() + kz * n2, n, tr(f.elem[sd][face], f.side[sd][face]),
                       f.u[sd].data() + (ky * mz + kz) * n2 * NV, NV);
        }
    }
  }
}

// Mortar data back onto both sides' faces (the sum over each face's mortars).
static void nc_project(const NcIface& f, int n, const std::vector<double>& mortar, int nc,
                       const std::function<double*(int, size_t)>& face_out) {
  const int n2 = n * n;
  const size_t my = f.rows[0].size(), mz = f.rows[1].size();
  std::vector<double> tmp(static_cast<size_t>(n2) * nc);
  for (int sd = 0; sd < 2; ++sd) {
    for (size_t face = 0; face < static_cast<size_t>(f.nfy[sd] * f.nfz[sd]); ++face)
      std::fill_n(face_out(sd, face), n2 * nc, 0.0);
    for (size_t ky = 0; ky < my; ++ky)
      for (size_t kz = 0; kz < mz; ++kz) {
        const long fy = sd ? f.rows[0][ky].fb : f.rows[0][ky].fa, fz = sd ? f.rows[1][kz].fb : f.rows[1][kz].fa;
        tensor_apply(f.B[sd][0].data() + ky * n2, f.B[sd][1].data() + kz * n2, n,
                     mortar.data() + (ky * mz + kz) * n2 * nc, tmp.data(), nc);
        double* o = face_out(sd, fy * f.nfz[sd] + fz);
        for (int q = 0; q < n2 * nc; ++q) o[q] += tmp[q];
      }
  }
}

// Lifting mean of the primitives at the mortar nodes, back onto both sides.
void orc_solver::nc_lift() {
  for (auto& f : ncs) {
    const size_t nodes = f.u[0].size() / NV;
    std::vector<double> lm(nodes * 4);
    for (size_t q = 0; q < nodes; ++q) {
      double a[4], b[4];
      prim4(f.u[0].data() + q * NV, gas, a);
      prim4(f.u[1].data() + q * NV, gas, b);
      for (int c = 0; c < 4; ++c) lm[q * 4 + c] = 0.5 * (a[c] + b[c]);
    }
    nc_project(f, n, lm, 4, [&](int sd, size_t face) { return lf(f.elem[sd][face], f.side[sd][face]); });
  }
}

// Two-sided Roe + central viscous flux at the mortar nodes (normal +x, vg_n = 0,
// A on the minus side), back onto both sides.
void orc_solver::nc_flux() {
  for (auto& f : ncs) {
    const size_t my = f.rows[0].size(), mz = f.rows[1].size(), nodes = my * mz * n2;
    if (lifting)
      for (int sd = 0; sd < 2; ++sd) {
        f.g[sd].assign(nodes * NG, 0.0);
        for (size_t ky = 0; ky < my; ++ky)
          for (size_t kz = 0; kz < mz; ++kz) {
            const long fy = sd ? f.rows[0][ky].fb : f.rows[0][ky].fa, fz = sd ? f.rows[1][kz].fb : f.rows[1][kz].fa;
            const size_t face = fy * f.nfz[sd] + fz;
            tensor_apply(f.F[sd][0].data() + ky * n2, f.F[sd][1].data() + kz * n2, n,
                         gt(f.elem[sd][face], f.side[sd][face]), f.g[sd].data() + (ky * mz + kz) * n2 * NG, NG);
          }
      }
    std::vector<double> fl(nodes * NV);
    for (size_t q = 0; q < nodes; ++q)
      face_flux(f.u[0].data() + q * NV, f.u[1].data() + q * NV, 0, 0.0, lifting ? f.g[0].data() + q * NG : nullptr,
                lifting ? f.g[1].data() + q * NG : nullptr, gas, fl.data() + q * NV);
    nc_project(f, n, fl, NV, [&](int sd, size_t face) { return ff(f.elem[sd][face], f.side[sd][face]); });
  }
}

// check_admissible (solver.cpp:892-906).
void orc_solver::check_admissible(const double* u) const {
  const size_t nodes = elems.size() * static_cast<size_t>(n3);
  for (size_t q = 0; q < nodes; ++q) {
    const double* s = u + q * NV;
    const bool ok = s[0] > 0.0 && pressure(s, gas) > 0.0 && std::isfinite(s[0]) && std::isfinite(s[1]) &&
                    std::isfinite(s[2]) && std::isfinite(s[3]) && std::isfinite(s[4]);
    if (!ok) {
      std::ostringstream os;
      os << "inadmissible state in element gid=" << q / n3 << " node " << q % n3 << " at step " << step_index
         << " stage " << stage_index << ": [" << s[0] << ", " << s[1] << ", " << s[2] << ", " << s[3] << ", "
         << s[4] << "]";
      throw InvalidStateError(os.str());
    }
  }
}

// Carpenter-Kennedy 5-stage 2N-storage RK4 (proj/src/lsrk.cpp:7-29).
static const double RK_A[5] = {0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
                               -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0};
static const double RK_B[5] = {1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
                               1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
                               2277821191437.0 / 14882151754819.0};
static const double RK_C[5] = {0.0, 1432997174477.0 / 9575080441755.0, 2526269341429.0 / 6820363962896.0,
                               2006345519317.0 / 3224310063776.0, 2802321613138.0 / 2924317926251.0};

// step (solver.cpp:908-927).
void orc_solver::step(double dt) {
  const size_t nn = field.size();
  for (int s = 0; s < 5; ++s) {
    stage_index = s;
    residual(time + RK_C[s] * dt, field.data(), dudt.data());
    const double as = RK_A[s], bs = RK_B[s];
    double* f = field.data();
    double* r = reg.data();
    const double* d = dudt.data();
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < nn; ++i) {
      r[i] = as * r[i] + dt * d[i];
      f[i] += bs * r[i];
    }
    check_admissible(field.data());
  }
  time += dt;
  step_index++;
  for (auto& f : ncs) {  // both directions of an oblique slide, wrapped like delta_base
    f.dy_base += f.vy_rel * dt;
    f.dz_base += f.vz_rel * dt;
    const double py = f.ly[0] * static_cast<double>(f.nfy[0]), pz = f.lz[0] * static_cast<double>(f.nfz[0]);
    while (f.dy_base >= py) f.dy_base -= py;
    while (f.dy_base < 0.0) f.dy_base += py;
    while (f.dz_base >= pz) f.dz_base -= pz;
    while (f.dz_base < 0.0) f.dz_base += pz;
  }
  for (auto& c : ctxs) {
    const Iface& f = ifaces[c.iface];
    c.delta_base += f.vg_rel * dt;
    const double period = f.l_par * static_cast<double>(f.n_faces);
    while (c.delta_base >= period) {
      c.delta_base -= period;
      ++c.wraps;
    }
  }
}

// suggest_dt (solver.cpp:929-947).
double orc_solver::suggest_dt(double cfl) const {
  double dt = std::numeric_limits<double>::max();
  for (size_t e = 0; e < elems.size(); ++e) {
    const Band& b = bands[elems[e].band];
    const double vg[3] = {0.0, annulus ? 0.0 : b.vg, annulus ? 0.0 : b.vgz};
    double lmax = 0.0;
    for (int nd = 0; nd < n3; ++nd) {
      const double* s = field.data() + (e * n3 + nd) * NV;
      const double v1 = s[1] / s[0] - vg[0], v2 = s[2] / s[0] - vg[1], v3 = s[3] / s[0] - vg[2];
      lmax = std::max(lmax, std::sqrt(v1 * v1 + v2 * v2 + v3 * v3) + std::sqrt(gas.gamma * pressure(s, gas) / s[0]));
    }
    // Annulus: the angular spacing times the inner radius, and the tip speed.
    if (annulus) lmax += std::abs(b.vg) * (spec.z0 + spec.depth);
    const double h = annulus ? std::min(b.hx, std::min(b.hy * spec.z0, b.hz)) : std::min(b.hx, std::min(b.hy, b.hz));
    dt = std::min(dt, cfl * h / (lmax * (2.0 * ns.degree + 1.0)));
  }
  return dt;
}

// ---------------------------------------------------------------------------
// C API
// ---------------------------------------------------------------------------
template <class F>
static int guard(orc_solver* s, F&& fn) {
  try {
    fn();
    return SDG_OK;
  } catch (const ConfigError& e) {
    (s ? s->err : g_err) = e.what();
    return SDG_ERR_CONFIG;
  } catch (const InvalidStateError& e) {
    (s ? s->err : g_err) = e.what();
    return SDG_ERR_INVALID_STATE;
  } catch (const ProtocolError& e) {
    (s ? s->err : g_err) = e.what();
    return SDG_ERR_PROTOCOL;
  } catch (const std::exception& e) {
    (s ? s->err : g_err) = e.what();
    return SDG_ERR_CONFIG;
  }
}

extern "C" {

int orc_create(const sdg_mesh_spec* mesh, const sdg_solver_config* cfg, orc_solver** out) {
  return guard(nullptr, [&] {
    auto* s = new orc_solver();
    try {
      s->build(*mesh, *cfg);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}
void orc_destroy(orc_solver* s) { delete s; }
const char* orc_last_error(const orc_solver* s) { return s ? s->err.c_str() : g_err.c_str(); }
const char* orc_global_error(void) { return g_err.c_str(); }
int orc_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}
long orc_n_elements(const orc_solver* s) { return static_cast<long>(s->elems.size()); }
int orc_n1(const orc_solver* s) { return s->n; }
int orc_n_contexts(const orc_solver* s) { return static_cast<int>(s->ctxs.size()); }

// set_initial_condition (solver.cpp:135-154).
int orc_set_initial_condition(orc_solver* s, double t0) {
  return guard(s, [&] {
    s->time = t0;
    s->step_index = 0;
    const int n = s->n;
    for (size_t e = 0; e < s->elems.size(); ++e)
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
          for (int k = 0; k < n; ++k) {
            double x[3];
            s->physical(static_cast<int>(e), s->ns.x[i], s->ns.x[j], s->ns.x[k], t0, x);
            const State u = eval_case(s->flow_case, x, t0, s->gas);
            std::copy(u.begin(), u.end(), s->field.begin() + s->node(static_cast<int>(e), i, j, k) * NV);
          }
    for (auto& c : s->ctxs) {
      c.delta_base = s->ifaces[c.iface].vg_rel * t0;
      c.topo_valid = false;
    }
    for (auto& f : s->ncs) {
      f.dy_base = f.vy_rel * t0;
      f.dz_base = f.vz_rel * t0;
    }
    std::fill(s->reg.begin(), s->reg.end(), 0.0);
  });
}
int orc_sample_case(const orc_solver* s, double t, double* u) {
  return guard(const_cast<orc_solver*>(s), [&] {
    const int n = s->n;
    for (size_t e = 0; e < s->elems.size(); ++e)
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
          for (int k = 0; k < n; ++k) {
            double x[3];
            s->physical(static_cast<int>(e), s->ns.x[i], s->ns.x[j], s->ns.x[k], t, x);
            const State st = eval_case(s->flow_case, x, t, s->gas);
            std::copy(st.begin(), st.end(), u + s->node(static_cast<int>(e), i, j, k) * NV);
          }
  });
}
int orc_set_state(orc_solver* s, const double* u) {
  std::copy(u, u + s->field.size(), s->field.begin());
  return SDG_OK;
}
int orc_get_state(const orc_solver* s, double* u) {
  std::copy(s->field.begin(), s->field.end(), u);
  return SDG_OK;
}
int orc_get_register(const orc_solver* s, double* r) {
  std::copy(s->reg.begin(), s->reg.end(), r);
  return SDG_OK;
}
int orc_compute_residual(orc_solver* s, double t_stage, const double* u, double* dudt) {
  return guard(s, [&] { s->residual(t_stage, u, dudt); });
}
int orc_compute_gradients(orc_solver* s, double t_stage, const double* u, double* grad) {
  return guard(s, [&] {
    s->update_interfaces(t_stage);
    s->prolong(u);
    s->fill_mortar_solution();
    s->exchange_solution();
    s->nc_update(t_stage);
    s->run_lifting(t_stage, u);
    std::copy(s->grad.begin(), s->grad.end(), grad);
  });
}
int orc_step(orc_solver* s, double dt) {
  return guard(s, [&] { s->step(dt); });
}
int orc_steps(orc_solver* s, double dt, int n) {
  return guard(s, [&] {
    for (int i = 0; i < n; ++i) s->step(dt);
  });
}
int orc_suggest_dt(const orc_solver* s, double cfl, double* dt) {
  *dt = s->suggest_dt(cfl);
  return SDG_OK;
}
double orc_time(const orc_solver* s) { return s->time; }
long orc_total_rebuilds(const orc_solver* s) {
  long t = 0;
  for (const auto& c : s->ctxs) t += c.rebuilds;
  return t;
}
int orc_ctx_info(const orc_solver* s, int ctx, long* out5, double* s_delta, double* sigma_side) {
  if (ctx < 0 || ctx >= static_cast<int>(s->ctxs.size())) return SDG_ERR_CONFIG;
  const Ctx& c = s->ctxs[ctx];
  out5[0] = c.iface;
  out5[1] = c.on_static ? 1 : 0;
  out5[2] = c.st.n_delta;
  out5[3] = c.conforming ? 1 : 0;
  out5[4] = static_cast<long>(c.faces.size());
  *s_delta = c.st.s_delta;
  *sigma_side = c.sigma_side;
  return SDG_OK;
}
int orc_get_pairing(const orc_solver* s, int role, int* ncols, int* cols) {
  const Role& r = role == 0 ? s->statics : s->movings;
  *ncols = static_cast<int>(r.cols.size());
  if (cols)
    for (size_t i = 0; i < r.cols.size(); ++i) {
      const Tuple& t = r.cols[i];
      int* o = cols + i * SDG_TUPLE_INTS;
      o[0] = t.partner;
      o[1] = t.iface;
      o[2] = static_cast<int>(t.i_par);
      o[3] = static_cast<int>(t.i_perp);
      o[4] = t.i_sub;
      o[5] = static_cast<int>(t.i_face);
      o[6] = t.ctx;
    }
  return SDG_OK;
}
int orc_get_mapping(const orc_solver* s, int ctx, int* m) {
  if (ctx < 0 || ctx >= static_cast<int>(s->ctxs.size())) return SDG_ERR_CONFIG;
  const Ctx& c = s->ctxs[ctx];
  const size_t nf = c.faces.size();
  for (int r = 0; r < 2; ++r)
    for (size_t f = 0; f < nf; ++f) m[r * nf + f] = c.m[r].empty() ? -1 : c.m[r][f];
  return SDG_OK;
}
int orc_get_metrics(const orc_solver* s, double* met, double* fmet) {
  return guard(const_cast<orc_solver*>(s), [&] {
    if (!s->curved) throw ConfigError("metrics are stored for curved meshes only");
    std::copy(s->met.begin(), s->met.end(), met);
    std::copy(s->fmet.begin(), s->fmet.end(), fmet);
  });
}

// integrate_mass_energy (diagnostics.cpp:31-50).
int orc_integrate_mass_energy(const orc_solver* s, const double* u, double* out2) {
  const int n = s->n;
  double m = 0.0, en = 0.0;
  for (size_t e = 0; e < s->elems.size(); ++e) {
    const Band& b = s->bands[s->elems[e].band];
    const double jac = 0.125 * b.hx * b.hy * b.hz;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        for (int k = 0; k < n; ++k) {
          const double* p = u + s->node(static_cast<int>(e), i, j, k) * NV;
          const double wj = s->ns.w[i] * s->ns.w[j] * s->ns.w[k] *
                            (s->curved ? 1.0 / s->mt(static_cast<int>(e), (i * n + j) * n + k)[9] : jac);
          m += wj * p[0];
          en += wj * p[4];
        }
  }
  out2[0] = m;
  out2[1] = en;
  return SDG_OK;
}

int orc_nodes(int degree, int kind, double* nodes, double* weights) {
  return guard(nullptr, [&] {
    const Nodes ns(degree, kind);
    std::copy(ns.x.begin(), ns.x.end(), nodes);
    std::copy(ns.w.begin(), ns.w.end(), weights);
  });
}
int orc_basis(int degree, int kind, double* diff, double* face_left, double* face_right) {
  return guard(nullptr, [&] {
    const Nodes ns(degree, kind);
    const Basis b = make_basis(ns);
    std::copy(b.D.begin(), b.D.end(), diff);
    std::copy(b.fl.begin(), b.fl.end(), face_left);
    std::copy(b.fr.begin(), b.fr.end(), face_right);
  });
}
int orc_mortar_ops(int degree, int kind, double sigma, double* fwd, double* bwd) {
  return guard(nullptr, [&] {
    const Nodes ns(degree, kind);
    mortar_ops(ns, sigma, fwd, bwd);
  });
}
int orc_subrange_ops(int degree, int kind, double lo, double hi, double* fwd, double* bwd) {
  return guard(nullptr, [&] { subrange_ops(Nodes(degree, kind), lo, hi, fwd, bwd); });
}
int orc_n_nc_interfaces(const orc_solver* s) { return static_cast<int>(s->ncs.size()); }
int orc_nc_rows(const orc_solver* s, int iface, int dir, long* n_out, long* faces, double* ranges, double* delta) {
  return guard(const_cast<orc_solver*>(s), [&] {
    if (iface < 0 || iface >= static_cast<int>(s->ncs.size()) || dir < 0 || dir > 1)
      throw ConfigError("no such non-matching interface / direction");
    const NcIface& f = s->ncs[iface];
    const auto& rows = f.rows[dir];
    *n_out = static_cast<long>(rows.size());
    if (delta) *delta = dir == 0 ? f.dy : f.dz;
    if (!faces || !ranges) return;
    for (size_t k = 0; k < rows.size(); ++k) {
      faces[2 * k] = rows[k].fa;
      faces[2 * k + 1] = rows[k].fb;
      for (int c = 0; c < 4; ++c) ranges[4 * k + c] = rows[k].r[c];
    }
  });
}
int orc_mortar_intervals(long n_a, long n_b, double l_a, double delta, long* n_out, long* faces, double* ranges) {
  return guard(nullptr, [&] {
    const std::vector<Interval> iv = intervals(n_a, n_b, l_a, delta);
    *n_out = static_cast<long>(iv.size());
    if (!faces || !ranges) return;
    for (size_t k = 0; k < iv.size(); ++k) {
      faces[2 * k] = iv[k].fa;
      faces[2 * k + 1] = iv[k].fb;
      for (int c = 0; c < 4; ++c) ranges[4 * k + c] = iv[k].r[c];
    }
  });
}
int orc_displacement(double delta, double l_par, long n_faces, double* d, long* n_delta, double* s_delta) {
  const Disp st = displacement(delta, l_par, n_faces);
  *d = st.delta;
  *n_delta = st.n_delta;
  *s_delta = st.s_delta;
  return SDG_OK;
}
long orc_moving_index(long i_par, long n_delta, int i_sub, long n_faces) {
  return moving_index(i_par, n_delta, i_sub, n_faces);
}
long orc_static_index(long i_moving, long n_delta, int i_sub, long n_faces) {
  return static_index(i_moving, n_delta, i_sub, n_faces);
}
int orc_pairing(int n_local, const long* faces, long n_par, long n_perp, const int* partner_ranks,
                long n_delta, int on_static, int conforming, int self_rank, int* ncols, int* cols,
                int* m_rows, long* face_lo, int* nsched, int* sched, int* self_entry) {
  return guard(nullptr, [&] {
    std::vector<LocalFace> fs(n_local);
    for (int f = 0; f < n_local; ++f) fs[f] = {faces[3 * f], faces[3 * f + 1], faces[3 * f + 2]};
    RankMap mp;
    mp.n_par = n_par;
    mp.n_perp = n_perp;
    mp.ranks.assign(partner_ranks, partner_ranks + n_par * n_perp);
    std::vector<Tuple> tc;
    append_tuples(fs, mp, n_delta, n_par, on_static != 0, conforming != 0, 0, 0, tc);
    sort_tuples(tc);
    *ncols = static_cast<int>(tc.size());
    for (size_t i = 0; i < tc.size(); ++i) {
      int* o = cols + i * SDG_TUPLE_INTS;
      o[0] = tc[i].partner;
      o[1] = tc[i].iface;
      o[2] = static_cast<int>(tc[i].i_par);
      o[3] = static_cast<int>(tc[i].i_perp);
      o[4] = tc[i].i_sub;
      o[5] = static_cast<int>(tc[i].i_face);
      o[6] = tc[i].ctx;
    }
    // build_mapping (partition.cpp:124-141).
    long lo = 0, hi = -1;
    if (!fs.empty()) {
      lo = hi = fs.front().i_face;
      for (const auto& f : fs) {
        lo = std::min(lo, f.i_face);
        hi = std::max(hi, f.i_face);
      }
    }
    *face_lo = lo;
    const long w = hi - lo + 1;
    for (long q = 0; q < 2 * w; ++q) m_rows[q] = -1;
    for (int i = 0; i < static_cast<int>(tc.size()); ++i) m_rows[tc[i].i_sub * w + (tc[i].i_face - lo)] = i;
    Sched self;
    const auto sc = make_schedule(tc, self_rank, self);
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
int orc_face_flux(const sdg_gas* gas, const double* um, const double* up, int dir, double vg_n, const double* gm,
                  const double* gp, double* out) {
  return guard(nullptr, [&] {
    const Gas g{gas->gamma, gas->R, gas->mu, gas->Pr};
    face_flux(um, up, dir, vg_n, gm, gp, g, out);
  });
}

}  // extern "C"
