// Host-side setup of the B200 path: mesh geometry, rank partition, local face
// tables in the flat form the kernels consume, nodal basis, long-double mortar
// operator assembly and the scalar displacement chain.  Everything here is
// per-run or per-stage scalar work; the per-node work lives in kernels.cu.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sdg_types.h"

namespace sdg {

// Error classes of the boundary (reference: proj/src/errors.hpp:9-21).
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidStateError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ProtocolError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
  int code;
  DeviceError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

constexpr int kMaxN1 = 8;       // N <= 7 on the device path
constexpr int kMaxCtx = 8;      // interface sides per rank (4 interfaces)
constexpr int kMaxPartners = 32;
constexpr int kMaxNcIfaces = 4;  // non-matching / oblique interfaces per mesh

enum SideType : int8_t { kConforming = 0, kSliding = 1, kDirichlet = 2 };

struct BandGeom {
  double x_lo, x_hi, hx, hy, hz, vg;
  int nx;
  long off;  // first global element id
  long n_elements;
  int ny, nz;   // per-band counts (BandSpec::ny, mesh.hpp:16; nz the 3D analogue)
  double vgz;   // translation speed along +z (oblique sliding, SDG_MAP_BOX only)
};

struct IfaceGeom {
  int left, right;
  bool static_is_left;
  double l_par;
  long n_faces, n_perp;
  double vg_rel;
  int static_band() const { return static_is_left ? left : right; }
  int moving_band() const { return static_is_left ? right : left; }
};

// A non-matching and/or obliquely sliding planar interface (BASELINE configs[1];
// the reference requires equal face counts, mesh.cpp:75-77, and motion along y
// only, mesh.hpp:12-17).  Side A = the left band's x+ faces, side B = the right
// band's x- faces; B is displaced by (vy_rel, vz_rel) t relative to A.  Its
// mortars are the tensor products of the y and z rows of face intervals
// (merge_intervals), recomputed every stage.
struct NcIfaceGeom {
  int left, right;
  long nfy[2], nfz[2];  // faces per side along y and z
  double ly[2], lz[2];  // face sizes
  double vy_rel, vz_rel;
};

// Structured multi-band hexahedral mesh (3D form of proj/src/mesh.cpp:27-92).
struct MeshGeom {
  sdg_mesh_spec spec;
  std::vector<BandGeom> bands;
  std::vector<IfaceGeom> ifaces;      // the reference's sliding interfaces (equal counts, y motion)
  std::vector<NcIfaceGeom> nc_ifaces; // non-matching / oblique ones
  long n_elements = 0;

  explicit MeshGeom(const sdg_mesh_spec& s);
  long gid(int b, int ix, int iy, int iz) const {
    return bands[b].off + (static_cast<long>(ix) * bands[b].ny + iy) * bands[b].nz + iz;
  }
  void locate(long g, int& b, int& ix, int& iy, int& iz) const;
};

// Contiguous blocks of each band per rank (proj/src/partition.cpp:17-83):
// largest-remainder rank counts per band, no rank on both sides of a sliding
// interface, 2 ranks over >2 bands -> static / moving split.
struct Partition {
  int n_ranks = 1;
  struct Block {
    int rank;
    long start, count;  // range of the band's element order (lexicographic or SFC)
  };
  std::vector<std::vector<Block>> band_blocks;
  // Element order of each band: lex_of[b][o] = band-local lexicographic index of
  // position o, order_of[b][lex] the inverse (empty = identity).
  std::vector<std::vector<long>> lex_of, order_of;
  int owner(int band, long local) const;  // local = lexicographic index
  long lex(int band, long o) const { return lex_of[band].empty() ? o : lex_of[band][o]; }
};
Partition assign_ranks(const MeshGeom& mesh, int n_ranks);

struct SlidingFaceRec {
  int iface;  // index into MeshGeom::ifaces, or MeshGeom::nc_ifaces when nc
  int elem;   // local element
  int side;   // 0 (x-) or 1 (x+)
  long i_par, i_perp;
  bool nc = false;
};

// Flat per-rank topology consumed by the kernels.
struct LocalTopology {
  int rank = 0;
  std::vector<long> gids;            // local element -> global id
  std::vector<int> coords;           // 4 per element: band, ix, iy, iz
  std::vector<int8_t> side_type;     // 6 per element
  // Periodic annulus sector (SDG_MAP_ANNULUS, height 2 pi / m): per side, the neighbour's
  // vectors reach this element's frame after a rotation by side_rot * sector angle
  // (-1 on the theta-minus side of the first theta row, +1 on the theta-plus side of the last).
  std::vector<int8_t> side_rot;
  std::vector<int> side_idx;         // conforming: neighbour trace slot; sliding: sliding index; dirichlet: index
  std::vector<std::array<int, 2>> dirichlet;  // (elem, side)
  std::vector<SlidingFaceRec> sliding;        // compact sliding index -> record
  int n_halo = 0;                             // halo trace slots after the 6*E local ones
  struct PeerFaces {
    int partner;
    std::vector<int> send_slots;  // local trace slots (e*6+side), in global key order
    std::vector<int> recv_slots;  // halo slots, same order
  };
  std::vector<PeerFaces> peers;   // ascending partner
};
LocalTopology build_topology(const MeshGeom& mesh, const Partition& part, int rank);
// Sector angle of a rotationally periodic annulus sector, 0 otherwise.
double sector_angle(const MeshGeom& mesh);
// Longest run [lo, hi) of local elements with no remote conforming and no sliding side: the
// elements whose kernels can run while the halo exchange is in flight.
std::array<int, 2> interior_run(const LocalTopology& topo);

// Nodal basis (proj/src/nodal_basis.cpp:89-182, same published algorithm).
struct Basis;
// Mapped position (SDG_MAP_WARP, include/sdg_types.h; the box otherwise) of a
// reference point of element (b, ix, iy, iz) at time t.
void map_point(const MeshGeom& m, int b, int ix, int iy, int iz, double xi, double eta, double zeta, double t,
               double* x);
// Curved metric terms of the local elements (SDG_MAP_WARP): met E x N3 x 10
// (Ja^d_c at [3d + c], 1/J), fmet 6E x N2 x 4 (unit +xi_dir normal, sJ) per local
// side; a conforming face carries the minus element's values in both slots.
struct CurvedMetrics {
  std::vector<double> met, fmet;
  int mw = 10, fw = 4;  // doubles per node (Ja 9, 1/J [, V 3 annulus]) / per face node (n 3, sJ [, vg.n/omega, pad])
};
CurvedMetrics compute_metrics(const MeshGeom& m, const Basis& sol, const LocalTopology& topo);

struct Basis {
  int degree = 0, kind = SDG_NODES_GAUSS, n = 0;
  std::vector<double> x, w, bary, D, fl, fr;
  Basis() = default;
  Basis(int degree, int kind);
  void lagrange(double xx, double* out) const;
};

// Face<->mortar L2 projections for hanging node sigma (proj/src/mortar.cpp:79-134),
// long double assembly.  fwd/bwd [2][n*n] row-major (Lower, Upper).
void build_mortar_ops(const Basis& b, double sigma, double* fwd, double* bwd);
// General sub-range [lo, hi] of one face (non-matching interfaces): fwd/bwd n*n.
void build_subrange_ops(const Basis& b, double lo, double hi, double* fwd, double* bwd);

struct Displacement {
  double delta = 0.0;
  long n_delta = 0;
  double s_delta = 0.0;
  bool conforming() const { return s_delta == 0.0; }
};
Displacement displacement(double delta, double l_par, long n_faces);  // proj/src/mesh.cpp:9-25

// Pairing restatement on the host, used only to size the per-partner NCCL
// blocks (the device computes A/m itself): counts of mortars per partner.
long moving_index(long i_par, long n_delta, int i_sub, long n_faces);
long static_index(long i_moving, long n_delta, int i_sub, long n_faces);

// One mortar of a non-matching periodic face row: the A face and B face it
// joins and its extent in each face's reference coordinate.
struct MortarInterval {
  long face_a = 0, face_b = 0;
  double a_lo = -1.0, a_hi = 1.0, b_lo = -1.0, b_hi = 1.0;
};
// Intersection of A's n_a faces of length l_a with B's n_b faces over the same
// period, B displaced by delta; in A order (by A face, then along the face).
std::vector<MortarInterval> merge_intervals(long n_a, long n_b, double l_a, double delta);

}  // namespace sdg

namespace sdg {
// Exact case state at x, t (exact_solutions.cpp:7-35, cases.hpp:18-25), host side.
void eval_case_host(const sdg_case& cs, const sdg_gas& gas, const double* x, double t, double* u);
}  // namespace sdg
