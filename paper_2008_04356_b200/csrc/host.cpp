// Host setup for the B200 path (see host.hpp).
#include "host.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <string>
#include <thread>
#include <tuple>

namespace sdg {

// ---------------------------------------------------------------- mesh
MeshGeom::MeshGeom(const sdg_mesh_spec& s) : spec(s) {
  if (s.n_bands < 1 || s.n_bands > SDG_MAX_BANDS) throw ConfigError("mesh needs 1..16 bands");
  if (s.mapping != SDG_MAP_BOX && s.mapping != SDG_MAP_WARP && s.mapping != SDG_MAP_ANNULUS)
    throw ConfigError("unknown mesh mapping");
  if (s.mapping != SDG_MAP_BOX && !std::isfinite(s.warp)) throw ConfigError("warp amplitude must be finite");
  if (s.mapping == SDG_MAP_ANNULUS) {
    if (!(s.z0 > 0.0)) throw ConfigError("annulus needs a positive inner radius (z0 > 0)");
    if (s.periodic_z) throw ConfigError("annulus: the radial direction cannot be periodic");
    if (s.periodic_y && std::abs(s.height - 2.0 * 3.14159265358979323846) > 1e-12)
    {
      const double mm = 2.0 * 3.14159265358979323846 / s.height;
      if (!(std::abs(mm - std::round(mm)) < 1e-9) || mm < 1.5)
        throw ConfigError("annulus: a periodic sector must divide the full circle (height = 2 pi / m)");
    }
  }
  if (s.ny < 1 || s.nz < 1) throw ConfigError("mesh needs ny >= 1 and nz >= 1");
  if (!(s.width > 0.0) || !(s.height > 0.0) || !(s.depth > 0.0))
    throw ConfigError("mesh extents must be positive");
  double frac_sum = 0.0;
  for (int b = 0; b < s.n_bands; ++b) {
    if (s.bands[b].nx < 1) throw ConfigError("band element count nx must be >= 1");
    if (!(s.bands[b].width_frac > 0.0)) throw ConfigError("band width fraction must be positive");
    if (s.bands[b].ny < 0 || s.bands[b].nz < 0) throw ConfigError("band ny / nz must be >= 0 (0 = the mesh-wide count)");
    frac_sum += s.bands[b].width_frac;
  }
  const int nb = s.n_bands;
  double x = s.x0, acc = 0.0;
  bool uniform = true;
  for (int b = 0; b < nb; ++b) {
    BandGeom g{};
    g.x_lo = x;
    acc += s.bands[b].width_frac;
    g.x_hi = (b == nb - 1) ? s.x0 + s.width : s.x0 + s.width * acc / frac_sum;
    x = g.x_hi;
    g.nx = s.bands[b].nx;
    g.ny = s.bands[b].ny > 0 ? s.bands[b].ny : s.ny;
    g.nz = s.bands[b].nz > 0 ? s.bands[b].nz : s.nz;
    g.hx = (g.x_hi - g.x_lo) / g.nx;
    g.hy = s.height / g.ny;
    g.hz = s.depth / g.nz;
    g.vg = s.bands[b].vg_y;
    g.vgz = s.bands[b].vg_z;
    g.off = n_elements;
    g.n_elements = static_cast<long>(g.nx) * g.ny * g.nz;
    n_elements += g.n_elements;
    if (g.vg < 0.0 || g.vgz < 0.0) throw ConfigError("moving bands must translate toward +y / +z");
    if (!std::isfinite(g.vg) || !std::isfinite(g.vgz)) throw ConfigError("band velocities must be finite");
    if (g.vg != 0.0 && !s.periodic_y)
      throw ConfigError("a moving band requires periodicity along the movement direction");
    if (g.vgz != 0.0 && !s.periodic_z)
      throw ConfigError("a band moving along z requires periodicity along z");
    uniform = uniform && g.ny == s.ny && g.nz == s.nz && g.vgz == 0.0;
    bands.push_back(g);
  }
  if (s.mortars != SDG_MORTARS_AUTO && s.mortars != SDG_MORTARS_TENSOR) throw ConfigError("unknown mortar kind");
  if ((!uniform || s.mortars == SDG_MORTARS_TENSOR) && s.mapping != SDG_MAP_BOX)
    throw ConfigError("per-band ny / nz, sliding along z and tensor-product mortars need affine hexahedra (SDG_MAP_BOX)");
  const int n_pairs = s.periodic_x ? nb : nb - 1;
  for (int p = 0; p < n_pairs; ++p) {
    const int l = p, r = (p + 1) % nb;
    if (nb == 1) continue;
    const BandGeom &L = bands[l], &R = bands[r];
    const bool matching = L.ny == R.ny && L.nz == R.nz;
    if (!matching || L.vgz != 0.0 || R.vgz != 0.0 || s.mortars == SDG_MORTARS_TENSOR) {
      // Non-matching and / or oblique: the tensor-product mortar path.
      if (matching && L.vg == R.vg && L.vgz == R.vgz) continue;  // conforming, moving together
      NcIfaceGeom f{};
      f.left = l;
      f.right = r;
      f.nfy[0] = L.ny;
      f.nfz[0] = L.nz;
      f.nfy[1] = R.ny;
      f.nfz[1] = R.nz;
      f.ly[0] = L.hy;
      f.lz[0] = L.hz;
      f.ly[1] = R.hy;
      f.lz[1] = R.hz;
      f.vy_rel = R.vg - L.vg;
      f.vz_rel = R.vgz - L.vgz;
      nc_ifaces.push_back(f);
      continue;
    }
    if (L.vg == R.vg) continue;
    if (L.vg != 0.0 && R.vg != 0.0)
      throw ConfigError("sliding interface requires one static side");
    IfaceGeom f{};
    f.left = l;
    f.right = r;
    f.static_is_left = L.vg == 0.0;
    f.l_par = L.hy;
    f.n_faces = L.ny;
    f.n_perp = L.nz;
    f.vg_rel = f.static_is_left ? R.vg : L.vg;
    ifaces.push_back(f);
  }
  if (ifaces.size() * 2 > static_cast<size_t>(kMaxCtx)) throw ConfigError("at most 4 sliding interfaces");
  if (nc_ifaces.size() > static_cast<size_t>(kMaxNcIfaces))
    throw ConfigError("at most " + std::to_string(kMaxNcIfaces) + " non-matching interfaces");
}

void MeshGeom::locate(long g, int& b, int& ix, int& iy, int& iz) const {
  b = 0;
  while (b + 1 < static_cast<int>(bands.size()) && g >= bands[b + 1].off) ++b;
  long loc = g - bands[b].off;
  const int ny = bands[b].ny, nz = bands[b].nz;
  iz = static_cast<int>(loc % nz);
  loc /= nz;
  iy = static_cast<int>(loc % ny);
  ix = static_cast<int>(loc / ny);
}

// ---------------------------------------------------------------- partition
int Partition::owner(int band, long local) const {
  const long o = order_of[band].empty() ? local : order_of[band][local];
  for (const auto& blk : band_blocks[band])
    if (o >= blk.start && o < blk.start + blk.count) return blk.rank;
  throw ProtocolError("ownership lookup outside any block");
}

namespace {
unsigned long long spread3(unsigned long long v) {  // 21 bits -> every third bit
  v &= 0x1fffff;
  v = (v | v << 32) & 0x1f00000000ffffULL;
  v = (v | v << 16) & 0x1f0000ff0000ffULL;
  v = (v | v << 8) & 0x100f00f00f00f00fULL;
  v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
  v = (v | v << 2) & 0x1249249249249249ULL;
  return v;
}

// Morton (Z-order) space-filling curve over a band's (ix, iy, iz) elements.
void sfc_order(const MeshGeom& mesh, int b, std::vector<long>& lex_of, std::vector<long>& order_of) {
  const long ny = mesh.bands[b].ny, nz = mesh.bands[b].nz, ne = mesh.bands[b].n_elements;
  std::vector<std::pair<unsigned long long, long>> key(ne);
  for (long l = 0; l < ne; ++l) {
    const long ix = l / (ny * nz), iy = (l / nz) % ny, iz = l % nz;
    key[l] = {spread3(ix) << 2 | spread3(iy) << 1 | spread3(iz), l};
  }
  std::sort(key.begin(), key.end());
  lex_of.resize(ne);
  order_of.resize(ne);
  for (long o = 0; o < ne; ++o) {
    lex_of[o] = key[o].second;
    order_of[key[o].second] = o;
  }
}
}  // namespace

Partition assign_ranks(const MeshGeom& mesh, int n_ranks) {
  const int nb = static_cast<int>(mesh.bands.size());
  if (n_ranks < 1) throw ConfigError("rank count must be positive");
  Partition p;
  p.n_ranks = n_ranks;
  p.band_blocks.resize(nb);
  p.lex_of.resize(nb);
  p.order_of.resize(nb);
  if (mesh.spec.partition == 1 && n_ranks > 1)
    for (int b = 0; b < nb; ++b) sfc_order(mesh, b, p.lex_of[b], p.order_of[b]);
  else if (mesh.spec.partition < 0 || mesh.spec.partition > 2)
    throw ConfigError("partition must be 0 (lexicographic blocks), 1 (space-filling curve) or 2 (y slabs)");
  if (mesh.spec.partition == 2 && n_ranks > 1) {
    // Slabs along the sliding direction through all bands: every rank owns the same share of
    // every band, so any rank count balances exactly when it divides ny.  A rank then owns
    // both sides of the sliding interfaces (rank-local mortars, the self block); mortars cross
    // ranks only where a slab edge meets the sliding displacement.  Element order inside a
    // band: iy major.
    const int ny = mesh.spec.ny, nz = mesh.spec.nz;
    if (n_ranks > ny) throw ConfigError("y-slab partition needs n_ranks <= ny");
    for (const auto& B : mesh.bands)
      if (B.ny != ny || B.nz != nz) throw ConfigError("y-slab partition needs the same ny / nz in every band");
    for (int b = 0; b < nb; ++b) {
      const int nx = mesh.bands[b].nx;
      auto& lo = p.lex_of[b];
      auto& ord = p.order_of[b];
      lo.resize(static_cast<size_t>(nx) * ny * nz);
      ord.resize(lo.size());
      long o = 0;
      for (int iy = 0; iy < ny; ++iy)
        for (int ix = 0; ix < nx; ++ix)
          for (int iz = 0; iz < nz; ++iz, ++o) {
            const long lex = (static_cast<long>(ix) * ny + iy) * nz + iz;
            lo[o] = lex;
            ord[lex] = o;
          }
      for (int r = 0; r < n_ranks; ++r) {
        const long y0 = static_cast<long>(ny) * r / n_ranks, y1 = static_cast<long>(ny) * (r + 1) / n_ranks;
        p.band_blocks[b].push_back({r, y0 * nx * nz, (y1 - y0) * nx * nz});
      }
    }
    return p;
  }
  if (n_ranks == 1) {
    for (int b = 0; b < nb; ++b) p.band_blocks[b].push_back({0, 0, mesh.bands[b].n_elements});
    return p;
  }
  if (n_ranks < nb) {
    if (n_ranks != 2) throw ConfigError("rank count below band count is only supported for 2 ranks");
    bool st = false, mv = false;
    for (const auto& b : mesh.bands) (b.vg != 0.0 ? mv : st) = true;
    if (!st || !mv) throw ConfigError("2 ranks over more bands requires both static and moving bands");
    for (int b = 0; b < nb; ++b) p.band_blocks[b].push_back({mesh.bands[b].vg != 0.0 ? 1 : 0, 0, mesh.bands[b].n_elements});
    return p;
  }
  const double total = static_cast<double>(mesh.n_elements);
  std::vector<int> per(nb, 1);
  int assigned = nb;
  std::vector<std::pair<double, int>> rem;
  for (int b = 0; b < nb; ++b) {
    const double share = static_cast<double>(mesh.bands[b].n_elements) / total * n_ranks;
    const int extra = std::max(0, static_cast<int>(std::floor(share)) - 1);
    per[b] += extra;
    assigned += extra;
    rem.emplace_back(share - std::floor(share), b);
  }
  std::sort(rem.begin(), rem.end(), [](const auto& a, const auto& c) {
    return a.first != c.first ? a.first > c.first : a.second < c.second;
  });
  for (int i = 0; assigned < n_ranks; ++i, ++assigned) per[rem[i % nb].second]++;
  int next = 0;
  for (int b = 0; b < nb; ++b) {
    const long ne = mesh.bands[b].n_elements;
    const long r = std::min<long>(per[b], ne);
    long start = 0;
    for (long k = 0; k < r; ++k) {
      const long count = ne / r + (k < ne % r ? 1 : 0);
      p.band_blocks[b].push_back({next++, start, count});
      start += count;
    }
    next += static_cast<int>(std::max<long>(0, per[b] - r));
  }
  return p;
}

// ---------------------------------------------------------------- topology
namespace {
struct Nbr {
  int kind;  // 0 conforming, 1 sliding, 2 dirichlet
  int band, ix, iy, iz, side, iface;
  bool nc = false;  // iface indexes MeshGeom::nc_ifaces
};

// Neighbour across `side` (3D form of face_topology.cpp:14-46 + 64-121).
Nbr neighbour(const MeshGeom& m, int b, int ix, int iy, int iz, int side) {
  const auto& s = m.spec;
  const int dir = side / 2;
  const bool plus = side & 1;
  const int opp = side ^ 1;
  const int ny = m.bands[b].ny, nz = m.bands[b].nz;
  if (dir == 1) {
    if (plus && iy + 1 == ny && !s.periodic_y) return {2, 0, 0, 0, 0, 0, -1};
    if (!plus && iy == 0 && !s.periodic_y) return {2, 0, 0, 0, 0, 0, -1};
    return {0, b, ix, plus ? (iy + 1) % ny : (iy - 1 + ny) % ny, iz, opp, -1};
  }
  if (dir == 2) {
    if (plus && iz + 1 == nz && !s.periodic_z) return {2, 0, 0, 0, 0, 0, -1};
    if (!plus && iz == 0 && !s.periodic_z) return {2, 0, 0, 0, 0, 0, -1};
    return {0, b, ix, iy, plus ? (iz + 1) % nz : (iz - 1 + nz) % nz, opp, -1};
  }
  const int nb = static_cast<int>(m.bands.size());
  const int nx = m.bands[b].nx;
  if (plus && ix + 1 < nx) return {0, b, ix + 1, iy, iz, opp, -1};
  if (!plus && ix > 0) return {0, b, ix - 1, iy, iz, opp, -1};
  int other = plus ? b + 1 : b - 1;
  if (other < 0 || other >= nb) {
    if (!s.periodic_x) return {2, 0, 0, 0, 0, 0, -1};
    other = (other + nb) % nb;
  }
  if (nb == 1) return {0, b, plus ? 0 : nx - 1, iy, iz, opp, -1};
  const int left = plus ? b : other, right = plus ? other : b;
  for (size_t i = 0; i < m.ifaces.size(); ++i)
    if (m.ifaces[i].left == left && m.ifaces[i].right == right)
      return {1, other, 0, iy, iz, opp, static_cast<int>(i)};
  for (size_t i = 0; i < m.nc_ifaces.size(); ++i)
    if (m.nc_ifaces[i].left == left && m.nc_ifaces[i].right == right)
      return {1, other, 0, iy, iz, opp, static_cast<int>(i), true};
  return {0, other, plus ? 0 : m.bands[other].nx - 1, iy, iz, opp, -1};
}
}  // namespace

double sector_angle(const MeshGeom& mesh) {
  const auto& s = mesh.spec;
  if (s.mapping != SDG_MAP_ANNULUS || !s.periodic_y) return 0.0;
  return std::abs(s.height - 2.0 * 3.14159265358979323846) > 1e-12 ? s.height : 0.0;
}

LocalTopology build_topology(const MeshGeom& mesh, const Partition& part, int rank) {
  LocalTopology t;
  t.rank = rank;
  const int nb = static_cast<int>(mesh.bands.size());
  std::map<long, int> local_of;
  for (int b = 0; b < nb; ++b)
    for (const auto& blk : part.band_blocks[b]) {
      if (blk.rank != rank) continue;
      for (long o = blk.start; o < blk.start + blk.count; ++o) t.gids.push_back(mesh.bands[b].off + part.lex(b, o));
    }
  // Local order: elements whose six neighbours are all on this rank first (stable), then
  // the rank-boundary elements, so the element kernels can run the interior as one range
  // while the halo exchange is in flight (interior_run).
  if (part.n_ranks > 1) {
    std::vector<long> inner, outer;
    for (const long g : t.gids) {
      int b, ix, iy, iz;
      mesh.locate(g, b, ix, iy, iz);
      bool remote = false;
      for (int s = 0; s < 6 && !remote; ++s) {
        const Nbr n = neighbour(mesh, b, ix, iy, iz, s);
        if (n.kind == 0) {
          const long ng = mesh.gid(n.band, n.ix, n.iy, n.iz);
          remote = part.owner(n.band, ng - mesh.bands[n.band].off) != rank;
        }
      }
      (remote ? outer : inner).push_back(g);
    }
    t.gids = inner;
    t.gids.insert(t.gids.end(), outer.begin(), outer.end());
  }
  for (size_t q = 0; q < t.gids.size(); ++q) local_of[t.gids[q]] = static_cast<int>(q);
  const int ne = static_cast<int>(t.gids.size());
  t.coords.resize(4 * ne);
  t.side_type.assign(6 * ne, kConforming);
  t.side_rot.assign(6 * ne, 0);
  const bool sector = sector_angle(mesh) != 0.0;
  t.side_idx.assign(6 * ne, -1);
  struct Remote {
    int partner;
    long key;
    int slot;
  };
  std::vector<Remote> remote;
  for (int e = 0; e < ne; ++e) {
    int b, ix, iy, iz;
    mesh.locate(t.gids[e], b, ix, iy, iz);
    t.coords[4 * e] = b;
    t.coords[4 * e + 1] = ix;
    t.coords[4 * e + 2] = iy;
    t.coords[4 * e + 3] = iz;
    for (int s = 0; s < 6; ++s) {
      const Nbr n = neighbour(mesh, b, ix, iy, iz, s);
      const int slot = 6 * e + s;
      if (n.kind == 2) {
        t.side_type[slot] = kDirichlet;
        t.side_idx[slot] = static_cast<int>(t.dirichlet.size());
        t.dirichlet.push_back({e, s});
      } else if (n.kind == 1) {
        t.side_type[slot] = kSliding;
        t.side_idx[slot] = static_cast<int>(t.sliding.size());
        t.sliding.push_back({n.iface, e, s, iy, iz, n.nc});
      } else {
        const long ng = mesh.gid(n.band, n.ix, n.iy, n.iz);
        const int owner = part.owner(n.band, ng - mesh.bands[n.band].off);
        t.side_type[slot] = kConforming;
        if (sector && s == 2 && iy == 0) t.side_rot[slot] = -1;
        if (sector && s == 3 && iy + 1 == mesh.bands[b].ny) t.side_rot[slot] = 1;
        if (owner == rank) {
          t.side_idx[slot] = 6 * local_of.at(ng) + n.side;
        } else {
          // Key of the face: minus element's global id and direction.
          const long minus = (s & 1) ? t.gids[e] : ng;
          remote.push_back({owner, minus * 3 + s / 2, slot});
        }
      }
    }
  }
  std::sort(remote.begin(), remote.end(), [](const Remote& a, const Remote& c) {
    return std::tie(a.partner, a.key) < std::tie(c.partner, c.key);
  });
  for (const auto& r : remote) {
    if (t.peers.empty() || t.peers.back().partner != r.partner) t.peers.push_back({r.partner, {}, {}});
    const int h = t.n_halo++;
    t.side_idx[r.slot] = 6 * ne + h;
    t.peers.back().send_slots.push_back(r.slot);
    t.peers.back().recv_slots.push_back(6 * ne + h);
  }
  return t;
}

// ---------------------------------------------------------------- curved geometry
namespace {
// sin(pi t), exactly 0 at integer t (the warp must vanish on band boundaries
// and be exactly periodic).
template <class R>
R sinpi_exact(R t) {
  R r = std::fmod(t, R(2));
  if (r < R(0)) r += R(2);
  if (r == R(0) || r == R(1)) return R(0);
  return std::sin(R(3.14159265358979323846264338327950288L) * r);
}
}  // namespace

// SDG_MAP_WARP position (include/sdg_types.h) at time t; the box position when affine.
void map_point(const MeshGeom& m, int b, int ix, int iy, int iz, double xi, double eta, double zeta, double t,
               double* x) {
  const BandGeom& B = m.bands[b];
  const double bx = (B.x_lo + ix * B.hx) + 0.5 * (xi + 1.0) * B.hx;
  const double by = (m.spec.y0 + iy * B.hy) + 0.5 * (eta + 1.0) * B.hy;
  const double bz = (m.spec.z0 + iz * B.hz) + 0.5 * (zeta + 1.0) * B.hz;
  if (m.spec.mapping == SDG_MAP_BOX) {
    x[0] = bx;
    x[1] = by + B.vg * t;
    x[2] = bz + B.vgz * t;
    return;
  }
  const double tx = (ix + 0.5 * (xi + 1.0)) / B.nx, ty = (iy + 0.5 * (eta + 1.0)) / m.spec.ny,
               tz = (iz + 0.5 * (zeta + 1.0)) / m.spec.nz;
  const double sp = sinpi_exact(tx), sy = sinpi_exact(2.0 * ty), sz = sinpi_exact(2.0 * tz);
  const double A = m.spec.warp;
  x[0] = bx + A * B.hx * sp * sy * sz;
  x[1] = by + (m.spec.mapping == SDG_MAP_ANNULUS ? 0.0 : A * B.hy * sp * sz) + B.vg * t;  // annulus: no theta warp
  x[2] = bz + A * B.hz * sp * sy;
  if (m.spec.mapping == SDG_MAP_ANNULUS) {  // (x, theta, r) -> (x, r sin theta, r cos theta)
    const double th = x[1], r = x[2];
    x[1] = r * std::sin(th);
    x[2] = r * std::cos(th);
  }
}

namespace {
using ldm = long double;
// Angle of an annulus element's centre at t = 0.
ldm center_angle(const MeshGeom& m, int b, int ix, int iy, int iz) {
  (void)ix;
  (void)iz;
  return m.spec.y0 + static_cast<ldm>(m.bands[b].hy) * (iy + 0.5L);
}

// Mapped position minus the mapped element centre, long double.  Two elements
// sharing a face see its geometry up to an exact translation.
void relative_point(const MeshGeom& m, int b, int ix, int iy, int iz, double xi, double eta, double zeta, ldm* x) {
  const BandGeom& B = m.bands[b];
  const ldm h[3] = {B.hx, B.hy, B.hz};
  const ldm t[3] = {(ix + 0.5L * (xi + 1.0L)) / B.nx, (iy + 0.5L * (eta + 1.0L)) / m.spec.ny,
                    (iz + 0.5L * (zeta + 1.0L)) / m.spec.nz};
  const ldm tc[3] = {(ix + 0.5L) / B.nx, (iy + 0.5L) / m.spec.ny, (iz + 0.5L) / m.spec.nz};
  const ldm A = m.spec.warp;
  const ldm sp = sinpi_exact<ldm>(t[0]), sy = sinpi_exact<ldm>(2.0L * t[1]), sz = sinpi_exact<ldm>(2.0L * t[2]);
  const ldm cp = sinpi_exact<ldm>(tc[0]), cy = sinpi_exact<ldm>(2.0L * tc[1]), cz = sinpi_exact<ldm>(2.0L * tc[2]);
  x[0] = 0.5L * xi * h[0] + A * h[0] * (sp * sy * sz - cp * cy * cz);
  x[1] = 0.5L * eta * h[1] + A * h[1] * (sp * sz - cp * cz);
  x[2] = 0.5L * zeta * h[2] + A * h[2] * (sp * sy - cp * cy);
  if (m.spec.mapping == SDG_MAP_ANNULUS) {
    const ldm th = m.spec.y0 + h[1] * (iy + 0.5L * (eta + 1.0L));  // theta faces stay meridional planes
    const ldm rr = m.spec.z0 + h[2] * (iz + 0.5L * (zeta + 1.0L)) + A * h[2] * sp * sy;
    const ldm thc = center_angle(m, b, ix, iy, iz);
    const ldm rc = m.spec.z0 + h[2] * (iz + 0.5L) + A * h[2] * cp * cy;
    x[1] = rr * std::sin(th) - rc * std::sin(thc);
    x[2] = rr * std::cos(th) - rc * std::cos(thc);
  }
}

// Absolute radius (annulus grid-velocity potential psi = r^2 / 2), long double.
ldm radius_point(const MeshGeom& m, int b, int ix, int iy, int iz, double xi, double eta, double zeta) {
  const BandGeom& B = m.bands[b];
  const ldm tx = (ix + 0.5L * (xi + 1.0L)) / B.nx, ty = (iy + 0.5L * (eta + 1.0L)) / m.spec.ny;
  const ldm sp = sinpi_exact<ldm>(tx), sy = sinpi_exact<ldm>(2.0L * ty);
  return m.spec.z0 + static_cast<ldm>(B.hz) * (iz + 0.5L * (zeta + 1.0L)) + static_cast<ldm>(m.spec.warp) * B.hz * sp * sy;
}

// Metric terms of one element (conservative curl form, Kopriva 2006):
//   Ja^i_c = -e_i . curl_xi( X_l grad_xi X_m ),  (c, m, l) cyclic,
// on the degree-N LGL interpolant, in long double.  JaL: LGL grid values
// [9][n^3] ([3 i + c]), dXL: dX_c/dxi_d [9][n^3] ([3 d + c]).
struct ElemMetricBuilder {
  int n, n3;
  Basis lgl;
  std::vector<ldm> DL, L;  // LGL differentiation; LGL -> solution interpolation L[s][p]
  ElemMetricBuilder(const Basis& sol) : n(sol.n), n3(sol.n * sol.n * sol.n), lgl(sol.degree, SDG_NODES_LGL) {
    DL.assign(lgl.D.begin(), lgl.D.end());
    std::vector<double> row(n);
    L.resize(static_cast<size_t>(n) * n);
    for (int a = 0; a < n; ++a) {
      lgl.lagrange(sol.x[a], row.data());
      for (int p = 0; p < n; ++p) L[a * n + p] = row[p];
    }
  }
  int idx(int p, int q, int r) const { return (p * n + q) * n + r; }
  void deriv(const ldm* f, int d, ldm* out) const {
    for (int p = 0; p < n; ++p)
      for (int q = 0; q < n; ++q)
        for (int r = 0; r < n; ++r) {
          const int row = d == 0 ? p : (d == 1 ? q : r);
          ldm acc = 0.0L;
          for (int m = 0; m < n; ++m)
            acc += DL[row * n + m] * f[d == 0 ? idx(m, q, r) : (d == 1 ? idx(p, m, r) : idx(p, q, m))];
          out[idx(p, q, r)] = acc;
        }
  }
  void interp3(const ldm* f, ldm* out) const {
    std::vector<ldm> t1(n3), t2(n3);
    for (int a = 0; a < n; ++a)
      for (int q = 0; q < n; ++q)
        for (int r = 0; r < n; ++r) {
          ldm acc = 0.0L;
          for (int p = 0; p < n; ++p) acc += L[a * n + p] * f[idx(p, q, r)];
          t1[idx(a, q, r)] = acc;
        }
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b)
        for (int r = 0; r < n; ++r) {
          ldm acc = 0.0L;
          for (int q = 0; q < n; ++q) acc += L[b * n + q] * t1[idx(a, q, r)];
          t2[idx(a, b, r)] = acc;
        }
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b)
        for (int c = 0; c < n; ++c) {
          ldm acc = 0.0L;
          for (int r = 0; r < n; ++r) acc += L[c * n + r] * t2[idx(a, b, r)];
          out[idx(a, b, c)] = acc;
        }
  }
  // Annulus: contravariant grid velocity per unit omega on the LGL grid,
  // VL^i = [curl_xi I^N(psi grad_xi X_0)]_i with psi = r^2 / 2 (vg / omega = curl(psi e_x)).
  void grid_velocity(const MeshGeom& m, int b, int ix, int iy, int iz, const std::vector<ldm>& dXL,
                     std::vector<ldm>& VL) const {
    std::vector<ldm> At(3 * n3), dV(n3);
    VL.assign(3 * n3, 0.0L);
    for (int p = 0; p < n; ++p)
      for (int q = 0; q < n; ++q)
        for (int r = 0; r < n; ++r) {
          const ldm rr = radius_point(m, b, ix, iy, iz, lgl.x[p], lgl.x[q], lgl.x[r]);
          for (int k = 0; k < 3; ++k) At[k * n3 + idx(p, q, r)] = 0.5L * rr * rr * dXL[(3 * k) * n3 + idx(p, q, r)];
        }
    for (int i = 0; i < 3; ++i) {
      const int i1 = (i + 1) % 3, i2 = (i + 2) % 3;
      deriv(At.data() + i2 * n3, i1, dV.data());
      for (int g = 0; g < n3; ++g) VL[i * n3 + g] = dV[g];
      deriv(At.data() + i1 * n3, i2, dV.data());
      for (int g = 0; g < n3; ++g) VL[i * n3 + g] -= dV[g];
    }
  }
  void build(const MeshGeom& m, int b, int ix, int iy, int iz, std::vector<ldm>& JaL, std::vector<ldm>& dXL) const {
    std::vector<ldm> X(3 * n3), V(3 * n3), dV(n3);
    JaL.assign(9 * n3, 0.0L);
    dXL.assign(9 * n3, 0.0L);
    for (int p = 0; p < n; ++p)
      for (int q = 0; q < n; ++q)
        for (int r = 0; r < n; ++r) {
          ldm x[3];
          relative_point(m, b, ix, iy, iz, lgl.x[p], lgl.x[q], lgl.x[r], x);
          for (int c = 0; c < 3; ++c) X[c * n3 + idx(p, q, r)] = x[c];
        }
    for (int d = 0; d < 3; ++d)
      for (int c = 0; c < 3; ++c) deriv(X.data() + c * n3, d, dXL.data() + (3 * d + c) * n3);
    for (int c = 0; c < 3; ++c) {
      const int mm = (c + 1) % 3, l = (c + 2) % 3;
      for (int d = 0; d < 3; ++d)
        for (int g = 0; g < n3; ++g)  // invariant form: rotation covariant (periodic annulus sectors)
          V[d * n3 + g] = 0.5L * (X[l * n3 + g] * dXL[(3 * d + mm) * n3 + g] - X[mm * n3 + g] * dXL[(3 * d + l) * n3 + g]);
      for (int i = 0; i < 3; ++i) {
        const int i1 = (i + 1) % 3, i2 = (i + 2) % 3;
        ldm* out = JaL.data() + (3 * i + c) * n3;
        deriv(V.data() + i2 * n3, i1, dV.data());
        for (int g = 0; g < n3; ++g) out[g] = -dV[g];
        deriv(V.data() + i1 * n3, i2, dV.data());
        for (int g = 0; g < n3; ++g) out[g] += dV[g];
      }
    }
  }
  // Unit +xi_d normal and sJ at the solution face nodes of `side`, from the
  // face's own geometry only: the normal component of the curl needs the
  // tangential derivatives on the face layer alone.  A face's two slots are
  // filled from the same element and side, so they hold identical bits.
  void face(const MeshGeom& m, int b, int ix, int iy, int iz, int side, double* out, int fw) const {
    const int d = side / 2;
    const double lay = (side & 1) ? 1.0 : -1.0;
    const int p1 = d == 0 ? 1 : 0, p2 = d == 2 ? 1 : 2;  // face index (a, b) runs along (p1, p2)
    const int n2 = n * n;
    std::vector<ldm> X(3 * n2), D1(3 * n2), D2(3 * n2), V1(n2), V2(n2), J(3 * n2);
    for (int u = 0; u < n; ++u)
      for (int v = 0; v < n; ++v) {
        double r[3];
        r[d] = lay;
        r[p1] = lgl.x[u];
        r[p2] = lgl.x[v];
        ldm x[3];
        relative_point(m, b, ix, iy, iz, r[0], r[1], r[2], x);
        for (int c = 0; c < 3; ++c) X[c * n2 + u * n + v] = x[c];
      }
    auto du = [&](const ldm* f, ldm* o) {
      for (int u = 0; u < n; ++u)
        for (int v = 0; v < n; ++v) {
          ldm acc = 0.0L;
          for (int q = 0; q < n; ++q) acc += DL[u * n + q] * f[q * n + v];
          o[u * n + v] = acc;
        }
    };
    auto dv = [&](const ldm* f, ldm* o) {
      for (int u = 0; u < n; ++u)
        for (int v = 0; v < n; ++v) {
          ldm acc = 0.0L;
          for (int q = 0; q < n; ++q) acc += DL[v * n + q] * f[u * n + q];
          o[u * n + v] = acc;
        }
    };
    for (int c = 0; c < 3; ++c) {
      du(X.data() + c * n2, D1.data() + c * n2);
      dv(X.data() + c * n2, D2.data() + c * n2);
    }
    // (curl V)_d = d_{p1} V_{p2} - d_{p2} V_{p1} for d = 0, 2 and its negative for d = 1.
    const ldm sgn = d == 1 ? -1.0L : 1.0L;
    std::vector<ldm> a1(n2), a2(n2);
    for (int c = 0; c < 3; ++c) {
      const int mm = (c + 1) % 3, l = (c + 2) % 3;
      for (int g = 0; g < n2; ++g) {
        V1[g] = 0.5L * (X[l * n2 + g] * D1[mm * n2 + g] - X[mm * n2 + g] * D1[l * n2 + g]);
        V2[g] = 0.5L * (X[l * n2 + g] * D2[mm * n2 + g] - X[mm * n2 + g] * D2[l * n2 + g]);
      }
      du(V2.data(), a1.data());
      dv(V1.data(), a2.data());
      for (int g = 0; g < n2; ++g) J[c * n2 + g] = -sgn * (a1[g] - a2[g]);
    }
    // Annulus: normal grid velocity per unit omega, sJ (vg / omega) . n = [curl_xi (psi grad_xi X_0)]_d.
    const bool ann = m.spec.mapping == SDG_MAP_ANNULUS;
    std::vector<ldm> W(n2, 0.0L);
    if (ann) {
      for (int u = 0; u < n; ++u)
        for (int v = 0; v < n; ++v) {
          double r[3];
          r[d] = lay;
          r[p1] = lgl.x[u];
          r[p2] = lgl.x[v];
          const ldm rr = radius_point(m, b, ix, iy, iz, r[0], r[1], r[2]);
          V1[u * n + v] = 0.5L * rr * rr * D1[u * n + v];  // psi dX_0/dxi_p1
          V2[u * n + v] = 0.5L * rr * rr * D2[u * n + v];  // psi dX_0/dxi_p2
        }
      du(V2.data(), a1.data());
      dv(V1.data(), a2.data());
      for (int g = 0; g < n2; ++g) W[g] = sgn * (a1[g] - a2[g]);
    }
    for (int a = 0; a < n; ++a)
      for (int bb = 0; bb < n; ++bb) {
        ldm v[4];
        for (int c = 0; c < (ann ? 4 : 3); ++c) {
          const ldm* src = c < 3 ? J.data() + c * n2 : W.data();
          ldm acc = 0.0L;
          for (int u = 0; u < n; ++u) {
            ldm inner = 0.0L;
            for (int w = 0; w < n; ++w) inner += L[bb * n + w] * src[u * n + w];
            acc += L[a * n + u] * inner;
          }
          v[c] = acc;
        }
        const ldm sj = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
        double* q = out + (a * n + bb) * fw;
        for (int c = 0; c < 3; ++c) q[c] = static_cast<double>(v[c] / sj);
        q[3] = static_cast<double>(sj);
        if (ann) {
          q[4] = static_cast<double>(v[3] / sj);
          q[5] = 0.0;
        }
      }
  }
};
}  // namespace

CurvedMetrics compute_metrics(const MeshGeom& m, const Basis& sol, const LocalTopology& topo) {
  const int n = sol.n, n2 = n * n, n3 = n2 * n;
  const int ne = static_cast<int>(topo.gids.size());
  CurvedMetrics out;
  const bool ann = m.spec.mapping == SDG_MAP_ANNULUS;
  out.mw = ann ? 13 : 10;
  out.fw = ann ? 6 : 4;
  const int mw = out.mw, fw = out.fw;
  out.met.assign(static_cast<size_t>(ne) * n3 * mw, 0.0);
  out.fmet.assign(static_cast<size_t>(ne) * 6 * n2 * fw, 0.0);
  const ElemMetricBuilder mb(sol);
  // Elements are independent: split them over the host threads (setup only).
  auto work = [&](int e_lo, int e_hi, std::string* err) {
    try {
      std::vector<ldm> JaL, dXL, Ja(9 * n3), dX(9 * n3), VL, Vs(3 * n3);
      for (int e = e_lo; e < e_hi; ++e) {
        const int* c = topo.coords.data() + 4 * e;
        mb.build(m, c[0], c[1], c[2], c[3], JaL, dXL);
        for (int q = 0; q < 9; ++q) {
          mb.interp3(JaL.data() + q * n3, Ja.data() + q * n3);
          mb.interp3(dXL.data() + q * n3, dX.data() + q * n3);
        }
        if (ann) {
          mb.grid_velocity(m, c[0], c[1], c[2], c[3], dXL, VL);
          for (int i = 0; i < 3; ++i) mb.interp3(VL.data() + i * n3, Vs.data() + i * n3);
        }
        for (int g = 0; g < n3; ++g) {
          double* o = out.met.data() + (static_cast<size_t>(e) * n3 + g) * mw;
          if (ann)
            for (int i = 0; i < 3; ++i) o[10 + i] = static_cast<double>(Vs[i * n3 + g]);
          for (int q = 0; q < 9; ++q) o[q] = static_cast<double>(Ja[q * n3 + g]);
          const ldm a00 = dX[0 * n3 + g], a01 = dX[1 * n3 + g], a02 = dX[2 * n3 + g];
          const ldm a10 = dX[3 * n3 + g], a11 = dX[4 * n3 + g], a12 = dX[5 * n3 + g];
          const ldm a20 = dX[6 * n3 + g], a21 = dX[7 * n3 + g], a22 = dX[8 * n3 + g];
          const ldm jac = a00 * (a11 * a22 - a12 * a21) - a01 * (a10 * a22 - a12 * a20) + a02 * (a10 * a21 - a11 * a20);
          if (!(jac > 0.0L)) throw ConfigError("curved mapping has a non-positive Jacobian (warp too large)");
          o[9] = static_cast<double>(1.0L / jac);
        }
        for (int side = 0; side < 6; ++side) {
          double* o = out.fmet.data() + (static_cast<size_t>(e) * 6 + side) * n2 * fw;
          const Nbr nb = neighbour(m, c[0], c[1], c[2], c[3], side);
          const bool seam = topo.side_rot[6 * e + side] != 0;  // the two slots differ by the sector rotation
          if ((side & 1) == 0 && nb.kind == 0 && !seam) {
            // Minus side of a conforming face: the face's metrics are those of the
            // minus element (whose plus side it is), bit for bit, on every rank.
            mb.face(m, nb.band, nb.ix, nb.iy, nb.iz, nb.side, o, fw);
          } else {
            mb.face(m, c[0], c[1], c[2], c[3], side, o, fw);
          }
        }
      }
    } catch (const std::exception& ex) {
      *err = ex.what();
    }
  };
  const int nt = std::max(1, std::min<int>(static_cast<int>(std::thread::hardware_concurrency()), (ne + 63) / 64));
  std::vector<std::thread> pool;
  std::vector<std::string> errs(nt);
  for (int t = 0; t < nt; ++t)
    pool.emplace_back(work, static_cast<int>(static_cast<long>(ne) * t / nt),
                      static_cast<int>(static_cast<long>(ne) * (t + 1) / nt), &errs[t]);
  for (auto& th : pool) th.join();
  for (const auto& e : errs)
    if (!e.empty()) throw ConfigError(e);
  return out;
}

// ---------------------------------------------------------------- basis
namespace {
void legendre_pd(int n, double x, double& p, double& dp) {
  if (n == 0) {
    p = 1.0;
    dp = 0.0;
    return;
  }
  double p0 = 1.0, p1 = x, d0 = 0.0, d1 = 1.0;
  for (int k = 1; k < n; ++k) {
    const double p2 = ((2.0 * k + 1.0) * x * p1 - k * p0) / (k + 1.0);
    const double d2 = d0 + (2.0 * k + 1.0) * p1;
    p0 = p1;
    p1 = p2;
    d0 = d1;
    d1 = d2;
  }
  p = p1;
  dp = d1;
}
}  // namespace

Basis::Basis(int deg, int knd) : degree(deg), kind(knd), n(deg + 1) {
  if (deg < 1 || deg > kMaxN1 - 1)
    throw ConfigError("polynomial degree " + std::to_string(deg) + " outside the device range [1,7]");
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  const double pi = 3.14159265358979323846;
  for (int j = 0; j <= (n - 1) / 2; ++j) {
    if (kind == SDG_NODES_LGL) {
      if (j == 0) {
        x[0] = -1.0;
        x[n - 1] = 1.0;
        continue;
      }
      double r = -std::cos(pi * j / deg);
      for (int it = 0; it < 50; ++it) {
        double p, dp;
        legendre_pd(deg, r, p, dp);
        const double step = dp / ((2.0 * r * dp - deg * (deg + 1.0) * p) / (1.0 - r * r));
        r -= step;
        if (std::abs(step) < 1e-15) break;
      }
      x[j] = r;
      x[deg - j] = -r;
    } else {
      double r = -std::cos(pi * (2.0 * j + 1.0) / (2.0 * n));
      for (int it = 0; it < 50; ++it) {
        double p, dp;
        legendre_pd(n, r, p, dp);
        const double step = p / dp;
        r -= step;
        if (std::abs(step) < 1e-15) break;
      }
      x[j] = r;
      x[deg - j] = -r;
    }
  }
  if (n % 2 == 1) x[deg / 2] = 0.0;
  for (int j = 0; j < n; ++j) {
    double p, dp;
    if (kind == SDG_NODES_LGL) {
      legendre_pd(deg, x[j], p, dp);
      w[j] = 2.0 / (deg * (deg + 1.0) * p * p);
    } else {
      legendre_pd(n, x[j], p, dp);
      w[j] = 2.0 / ((1.0 - x[j] * x[j]) * dp * dp);
    }
  }
  bary.assign(n, 1.0);
  for (int j = 0; j < n; ++j) {
    for (int k = 0; k < n; ++k)
      if (k != j) bary[j] *= x[j] - x[k];
    bary[j] = 1.0 / bary[j];
  }
  D.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i) {
    double diag = 0.0;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      D[i * n + j] = (bary[j] / bary[i]) / (x[i] - x[j]);
      diag -= D[i * n + j];
    }
    D[i * n + i] = diag;
  }
  fl.assign(n, 0.0);
  fr.assign(n, 0.0);
  lagrange(-1.0, fl.data());
  lagrange(1.0, fr.data());
}

void Basis::lagrange(double xx, double* out) const {
  for (int k = 0; k < n; ++k)
    if (xx == x[k]) {
      for (int j = 0; j < n; ++j) out[j] = j == k ? 1.0 : 0.0;
      return;
    }
  double den = 0.0;
  for (int k = 0; k < n; ++k) den += (out[k] = bary[k] / (xx - x[k]));
  for (int k = 0; k < n; ++k) out[k] /= den;
}

// ---------------------------------------------------------------- mortar operators
namespace {
using ld = long double;

struct LdLagrange {
  std::vector<ld> x, b;
  explicit LdLagrange(const std::vector<double>& nodes) : x(nodes.begin(), nodes.end()), b(nodes.size(), 1.0L) {
    const int n = static_cast<int>(x.size());
    for (int j = 0; j < n; ++j) {
      for (int k = 0; k < n; ++k)
        if (k != j) b[j] *= x[j] - x[k];
      b[j] = 1.0L / b[j];
    }
  }
  void eval(ld xx, ld* out) const {
    const int n = static_cast<int>(x.size());
    for (int k = 0; k < n; ++k)
      if (xx == x[k]) {
        for (int j = 0; j < n; ++j) out[j] = j == k ? 1.0L : 0.0L;
        return;
      }
    ld den = 0.0L;
    for (int k = 0; k < n; ++k) den += (out[k] = b[k] / (xx - x[k]));
    for (int k = 0; k < n; ++k) out[k] /= den;
  }
};

// In-place Cholesky of SPD a (n x n), then solve a X = rhs (n x n) column by column.
void chol_solve(std::vector<ld> a, std::vector<ld>& rhs, int n) {
  for (int j = 0; j < n; ++j) {
    ld d = a[j * n + j];
    for (int k = 0; k < j; ++k) d -= a[j * n + k] * a[j * n + k];
    if (d <= 0.0L) throw ConfigError("mortar mass matrix not positive definite");
    a[j * n + j] = std::sqrt(d);
    for (int i = j + 1; i < n; ++i) {
      ld s = a[i * n + j];
      for (int k = 0; k < j; ++k) s -= a[i * n + k] * a[j * n + k];
      a[i * n + j] = s / a[j * n + j];
    }
  }
  for (int c = 0; c < n; ++c) {
    for (int i = 0; i < n; ++i) {
      ld s = rhs[i * n + c];
      for (int k = 0; k < i; ++k) s -= a[i * n + k] * rhs[k * n + c];
      rhs[i * n + c] = s / a[i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      ld s = rhs[i * n + c];
      for (int k = i + 1; k < n; ++k) s -= a[k * n + i] * rhs[k * n + c];
      rhs[i * n + c] = s / a[i * n + i];
    }
  }
}
}  // namespace

namespace {
// Face <-> mortar operators for mortars covering sub-ranges of one face, sharing the
// face mass matrix (n-point Gauss quadrature, exact for the degree-2N integrands).
struct SubrangeBuilder {
  const Basis& bs;
  Basis gauss;
  LdLagrange lag;
  std::vector<ld> mass;
  explicit SubrangeBuilder(const Basis& b) : bs(b), gauss(b.degree, SDG_NODES_GAUSS), lag(b.x), mass(b.n * b.n, 0.0L) {
    const int n = bs.n;
    std::vector<ld> la(n);
    for (int q = 0; q < n; ++q) {
      lag.eval(gauss.x[q], la.data());
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) mass[i * n + j] += static_cast<ld>(gauss.w[q]) * la[i] * la[j];
    }
  }
  // Mortar on face coordinates [lo, hi]: fwd = M^-1 S^T (face -> mortar), bwd =
  // (hi - lo)/2 M^-1 S (mortar -> face), S_ij = int l_i(xi(z)) l_j(z) dz.
  void build(double lo, double hi, double* fwd, double* bwd) const {
    const int n = bs.n;
    const ld frac = 0.5L * (static_cast<ld>(hi) - static_cast<ld>(lo));
    std::vector<ld> s(n * n, 0.0L), la(n), lb(n);
    for (int q = 0; q < n; ++q) {
      const ld z = gauss.x[q];
      const ld xi = static_cast<ld>(lo) + frac * (z + 1.0L);
      lag.eval(xi, la.data());
      lag.eval(z, lb.data());
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) s[i * n + j] += static_cast<ld>(gauss.w[q]) * la[i] * lb[j];
    }
    std::vector<ld> f(n * n), bk(n * n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        f[i * n + j] = s[j * n + i];
        bk[i * n + j] = frac * s[i * n + j];
      }
    chol_solve(mass, f, n);
    chol_solve(mass, bk, n);
    for (int i = 0; i < n * n; ++i) {
      fwd[i] = static_cast<double>(f[i]);
      bwd[i] = static_cast<double>(bk[i]);
    }
  }
};
}  // namespace

// The reference's two mortars of a hanging node are the sub-ranges [-1, sigma] and
// [sigma, 1] (proj/src/mortar.cpp:79-134); the general builder reproduces its bits
// (-1 + (1 + sigma)/2 (z + 1) and sigma + (1 - sigma)/2 (z + 1) are the same roundings).
void build_mortar_ops(const Basis& bs, double sigma, double* fwd, double* bwd) {
  if (!(sigma >= -1.0 && sigma < 1.0)) throw ConfigError("mortar position sigma must lie in [-1, 1)");
  const SubrangeBuilder sb(bs);
  const int nn = bs.n * bs.n;
  sb.build(-1.0, sigma, fwd, bwd);
  sb.build(sigma, 1.0, fwd + nn, bwd + nn);
}

void build_subrange_ops(const Basis& bs, double lo, double hi, double* fwd, double* bwd) {
  if (!(lo >= -1.0 && lo < hi && hi <= 1.0)) throw ConfigError("mortar sub-range must satisfy -1 <= lo < hi <= 1");
  SubrangeBuilder(bs).build(lo, hi, fwd, bwd);
}

// Non-matching periodic face rows (BASELINE configs[1]).  Side A has n_a faces of
// length l_a, side B n_b faces over the same period, displaced by delta.  The
// displacement splits exactly as the reference's (proj/src/mesh.cpp:9-25) into
// n_delta + s in A units; B edge j sits at n_delta + k_j + (s + r_j / n_b) with
// j n_a = k_j n_b + r_j, so equal counts give edges n_delta + j + s with the
// reference's own s bits, and local coordinates 2s - 1 (= sigma) on A and
// 1 - 2s (= -sigma, proj/src/solver.cpp:162-163) on B.
std::vector<MortarInterval> merge_intervals(long n_a, long n_b, double l_a, double delta) {
  if (n_a < 1 || n_b < 1) throw ConfigError("interval merge needs at least one face per side");
  if (!(l_a > 0.0)) throw ConfigError("face length must be positive");
  const Displacement st = displacement(delta, l_a, n_a);
  const double q = static_cast<double>(n_a) / static_cast<double>(n_b);  // B face length in A units
  std::vector<long> ei(n_b + 1);
  std::vector<double> ef(n_b + 1);
  for (long j = 0; j < n_b; ++j) {
    const long num = j * n_a;
    long I = st.n_delta + num / n_b;
    double f = st.s_delta + static_cast<double>(num % n_b) / static_cast<double>(n_b);
    if (f >= 1.0) {
      f -= 1.0;
      ++I;
    }
    ei[j] = I;
    ef[j] = f;
  }
  ei[n_b] = ei[0] + n_a;
  ef[n_b] = ef[0];
  std::vector<MortarInterval> out;
  out.reserve(static_cast<size_t>(n_a + n_b));
  long n_before = 0;  // pieces starting before A's period end
  for (long j = 0; j < n_b; ++j) {
    // Breakpoints inside B face j: its left edge, the A edges strictly inside, its right edge.
    const long m_first = ei[j] + 1;
    const long m_last = ef[j + 1] == 0.0 ? ei[j + 1] - 1 : ei[j + 1];
    auto b_local = [&](long m) { return 1.0 - 2.0 * ((static_cast<double>(ei[j + 1] - m) + ef[j + 1]) / q); };
    long p_int = ei[j];
    double a_lo = ef[j] == 0.0 ? -1.0 : 2.0 * ef[j] - 1.0, b_lo = -1.0;
    for (long m = m_first; m <= m_last + 1; ++m) {
      if (p_int < n_a) ++n_before;
      MortarInterval iv;
      iv.face_a = ((p_int % n_a) + n_a) % n_a;
      iv.face_b = j;
      iv.a_lo = a_lo;
      iv.b_lo = b_lo;
      if (m <= m_last) {  // piece ends at A edge m
        iv.a_hi = 1.0;
        iv.b_hi = b_local(m);
        a_lo = -1.0;
        b_lo = iv.b_hi;
        p_int = m;
      } else {            // piece ends at B's right edge
        iv.a_hi = ef[j + 1] == 0.0 ? 1.0 : 2.0 * ef[j + 1] - 1.0;
        iv.b_hi = 1.0;
      }
      out.push_back(iv);
    }
  }
  // The walk runs along the row from B's edge 0 (inside A face n_delta); A order starts
  // with the pieces past A's period end (faces 0 .. n_delta), so it is a rotation.
  // (Not a sort by a_lo: a sub-ulp s makes 2s - 1 round to -1 and would tie.)
  std::rotate(out.begin(), out.begin() + n_before, out.end());
  return out;
}

// ---------------------------------------------------------------- kinematics
Displacement displacement(double delta, double l_par, long n_faces) {
  const double period = l_par * static_cast<double>(n_faces);
  double d = std::fmod(delta, period);
  if (d < 0.0) d += period;
  const double ratio = d / l_par;
  Displacement st;
  st.delta = d;
  st.n_delta = static_cast<long>(std::floor(ratio));
  st.s_delta = ratio - static_cast<double>(st.n_delta);
  if (st.n_delta >= n_faces) st = Displacement{};
  return st;
}

long moving_index(long i_par, long n_delta, int i_sub, long n_faces) {
  const long r = (i_par - n_delta + i_sub - 1) % n_faces;
  return r < 0 ? r + n_faces : r;
}
long static_index(long i_moving, long n_delta, int i_sub, long n_faces) {
  const long r = (i_moving + n_delta - i_sub + 1) % n_faces;
  return r < 0 ? r + n_faces : r;
}

}  // namespace sdg

namespace sdg {
// Seeded density perturbation of include/sdg_types.h (sdg_case.pt_*).
static double case_perturbation(const sdg_case& cs, const double* x, double t) {
  const double two_pi = 6.283185307179586476925286766559;
  double c[3] = {x[0] - cs.pt_adv[0] * t, x[1] - cs.pt_adv[1] * t, x[2] - cs.pt_adv[2] * t};
  if (cs.pt_coords == 1) {
    const double th = std::atan2(c[1], c[2]), r = std::sqrt(c[1] * c[1] + c[2] * c[2]);
    c[1] = th;
    c[2] = r;
  }
  double xh[3];
  for (int d = 0; d < 3; ++d) xh[d] = (c[d] - cs.pt_x0[d]) / cs.pt_len[d];
  double acc = 0.0;
  for (int m = 0; m < cs.pt_modes; ++m)
    acc += cs.pt_a[m] * std::sin(two_pi * (cs.pt_k[m][0] * xh[0] + cs.pt_k[m][1] * xh[1] + cs.pt_k[m][2] * xh[2]) + cs.pt_phi[m]);
  return cs.pt_amp * acc;
}

void eval_case_host(const sdg_case& cs, const sdg_gas& g, const double* x, double t, double* u) {
  const double pi = 3.14159265358979323846;
  const double gm1 = g.gamma - 1.0;
  double rho, v0, v1, v2, p;
  switch (cs.kind) {
    case SDG_CASE_DENSITY_WAVE: {
      const double* k = cs.dw_k;
      const double* a = cs.dw_a;
      const double ph = pi * (k[0] * x[0] + k[1] * x[1] + k[2] * x[2] - (k[0] * a[0] + k[1] * a[1] + k[2] * a[2]) * t);
      rho = 2.0 + cs.dw_alpha * std::sin(ph);
      v0 = a[0];
      v1 = a[1];
      v2 = a[2];
      p = cs.dw_p0;
      break;
    }
    case SDG_CASE_VORTEX: {
      const double ui = cs.vx_v_inf * std::cos(cs.vx_theta), vi = cs.vx_v_inf * std::sin(cs.vx_theta);
      const double xb = x[0] - cs.vx_center[0] - ui * t, yb = x[1] - cs.vx_center[1] - vi * t;
      const double r2 = (xb * xb + yb * yb) / (cs.vx_rc * cs.vx_rc);
      const double s = cs.vx_eps * std::exp(0.5 * (1.0 - r2));
      v0 = ui - cs.vx_v_inf * s * yb / cs.vx_rc;
      v1 = vi + cs.vx_v_inf * s * xb / cs.vx_rc;
      v2 = 0.0;
      const double tr =
          1.0 - 0.5 * gm1 * cs.vx_eps * cs.vx_eps * cs.vx_ma_inf * cs.vx_ma_inf * std::exp(1.0 - r2);
      rho = cs.vx_rho_inf * std::pow(tr, 1.0 / gm1);
      const double pinf = cs.vx_rho_inf * cs.vx_v_inf * cs.vx_v_inf / (g.gamma * cs.vx_ma_inf * cs.vx_ma_inf);
      p = pinf * std::pow(tr, g.gamma / gm1);
      break;
    }
    case SDG_CASE_TGV: {
      const double X = x[1], Y = x[2], Z = x[0];
      const double V0 = cs.tgv_v0, r0 = cs.tgv_rho0;
      rho = r0;
      v0 = 0.0;
      v1 = V0 * std::sin(X) * std::cos(Y) * std::cos(Z);
      v2 = -V0 * std::cos(X) * std::sin(Y) * std::cos(Z);
      const double p0 = r0 * V0 * V0 / (g.gamma * cs.tgv_mach * cs.tgv_mach);
      p = p0 + r0 * V0 * V0 / 16.0 * (std::cos(2.0 * X) + std::cos(2.0 * Y)) * (std::cos(2.0 * Z) + 2.0);
      break;
    }
    case SDG_CASE_SWIRL: {
      const double pi = 3.14159265358979323846;
      const double om = cs.sw_omega;
      rho = 2.0 + cs.dw_alpha * std::sin(pi * cs.dw_k[0] * (x[0] - cs.dw_a[0] * t));
      v0 = cs.dw_a[0];
      v1 = om * x[2];
      v2 = -om * x[1];
      p = cs.dw_p0 + om * om * (x[1] * x[1] + x[2] * x[2]);
      break;
    }
    case SDG_CASE_FREESTREAM:
      rho = cs.fs_rho;
      v0 = cs.fs_v[0];
      v1 = cs.fs_v[1];
      v2 = cs.fs_v[2];
      p = cs.fs_p;
      break;
    default:
      throw ConfigError("unknown case kind");
  }
  if (cs.pt_modes < 0 || cs.pt_modes > SDG_PT_MAX_MODES) throw ConfigError("perturbation: 0..8 modes");
  if (cs.pt_modes > 0) rho += case_perturbation(cs, x, t);
  if (!(rho > 0.0) || !(p > 0.0)) throw InvalidStateError("primitive state requires rho > 0 and p > 0");
  u[0] = rho;
  u[1] = rho * v0;
  u[2] = rho * v1;
  u[3] = rho * v2;
  u[4] = p / gm1 + 0.5 * rho * (v0 * v0 + v1 * v1 + v2 * v2);
}
std::array<int, 2> interior_run(const LocalTopology& topo) {
  const int E = static_cast<int>(topo.gids.size());
  int best_lo = 0, best_len = 0, run_lo = 0;
  for (int e = 0; e <= E; ++e) {
    bool interior = e < E;
    for (int s = 0; interior && s < 6; ++s) {
      const size_t k = static_cast<size_t>(e) * 6 + s;
      // Mortar data are complete before the element kernels (the mortar rounds are joined
      // at once); only remote conforming neighbours arrive with the overlapped halo round.
      if (topo.side_type[k] == kConforming && topo.side_idx[k] >= 6 * E) interior = false;
    }
    if (!interior) {
      if (e - run_lo > best_len) {
        best_len = e - run_lo;
        best_lo = run_lo;
      }
      run_lo = e + 1;
    }
  }
  return {best_lo, best_lo + best_len};
}

}  // namespace sdg
