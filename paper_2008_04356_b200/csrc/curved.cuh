// Curved hexahedra (SDG_MAP_WARP, include/sdg_types.h): element kernels with
// per-node metric terms.  Included by kernels.cu inside its anonymous
// namespace (shares the flux helpers, tables and loaders defined there).
//
// The reference has affine elements only (ElementMetrics, mesh.cpp:102-111);
// these kernels generalise its phases as follows:
//   volume term   (1/J) sum_d Dhat (Ja^d . F)               (volume_kernel, solver.cpp:343-385)
//   BR1 gradient  J g_c = sum_d [surface q* (n sJ)_c - Dhat (Ja^d_c q)]   (assemble_gradients, :729-768)
//   face flux     Roe / viscous along the face's unit normal n, vg_n = vg . n   (flux.cpp:68-133)
//   surface lift  +- (l(+-1)/w) (sJ / J) F*                  (apply_all_faces, :547-582)
// Device layout (solver.cu upload_topology), per element structure-of-arrays so
// that the threads of a warp read consecutive words: met[e][c][node], c < MW
// (Ja^d_c at c = 3d + c', 1/J at 9 [, V^d at 10 + d]); fmet[e][side][c][f], c < FW
// (unit normal along +xi_dir at c < 3, sJ at 3 [, (vg / omega) . n at 4]).
// Both slots of a conforming face hold identical bits (host.cpp compute_metrics),
// so both elements evaluate the face flux identically, as in the affine kernels.

// Metric widths: per node Ja (9), 1/J [, V^d (3): annulus grid velocity per unit omega];
// per face node unit normal (3), sJ [, (vg / omega) . n, pad: annulus].
template <bool ROT>
struct MWidth {
  static constexpr int MW = ROT ? 13 : 10, FW = ROT ? 6 : 4;
};

// Opt a kernel in to more than 48 KB of dynamic shared memory; a failure (more than the
// 227 KB a CTA may use) is reported instead of surfacing as a failed launch.
template <class K>
void set_smem_checked(K kernel, cudaFuncAttribute attr, int bytes) {
  const cudaError_t e = cudaFuncSetAttribute(kernel, attr, bytes);
  if (e != cudaSuccess)
    throw DeviceError(SDG_ERR_CUDA, std::string("cudaFuncSetAttribute(") + std::to_string(bytes) +
                                        " B shared): " + cudaGetErrorString(e));
}

template <int N1, bool ROT>
struct CDim {
  static constexpr int N2 = N1 * N1;
  static constexpr int N3 = N2 * N1;
  static constexpr int MW = MWidth<ROT>::MW, FW = MWidth<ROT>::FW;
  static constexpr int EPB = N1 <= 4 ? Dim<N1>::EPB : 1;
  static constexpr int THREADS = EPB * N3;
  static constexpr int PER_GRAD = (21 + MW) * N3 + (54 + 6 * FW) * N2;  // U, q, metrics, gradient | traces, lift*, face metrics
  static constexpr int PER_UPD = (10 + MW) * N3 + (54 + 6 * FW) * N2;   // U, staging, metrics | lift*, face flux, face metrics
};

// Rigid rotation of an annulus band at the stage time (SDG_MAP_ANNULUS): theta -> theta + phi,
// (Y, Z) -> (c Y + s Z, -s Y + c Z).  Metric vectors rotate with the band: Ja(t) = R Ja(0), n(t) = R n(0).
struct Rot {
  double c, s;
};
__device__ __forceinline__ Rot band_rotation(bool rot, const StageArgs& A, int band) {
  return rot ? Rot{A.rot_c[band], A.rot_s[band]} : Rot{1.0, 0.0};  // (cos, sin)(vg t_stage), solver.cu stage_args
}
__device__ __forceinline__ void rotate_yz(const Rot& r, double& y, double& z) {
  const double a = r.c * y + r.s * z, b = -r.s * y + r.c * z;
  y = a;
  z = b;
}
// Unit normal of a face node at the stage time and vg . n.
// sfm: one element's face metrics [side][c][f].
template <int N2, int FW, bool ROT>
__device__ __forceinline__ void face_normal(const double* sfm, int s, int f, const Rot& r, const BandD& B, double* n,
                                            double& vgn) {
  const double* q = sfm + s * FW * N2 + f;
  n[0] = q[0];
  n[1] = q[N2];
  n[2] = q[2 * N2];
  if (ROT) {
    rotate_yz(r, n[1], n[2]);
    vgn = B.vg * q[4 * N2];
  } else {
    vgn = B.vg * n[1];
  }
}
__device__ __forceinline__ double face_sj(const double* sfm, int s, int f, int n2, int fw) {
  return sfm[(s * fw + 3) * n2 + f];
}

// Flat, coalesced load of EPB consecutive elements' node-major NC-vectors into
// SoA shared memory dst[le * per + c * N3 + node].
template <int N1, int EPB, int NC>
__device__ __forceinline__ void load_soa(const double* __restrict__ src, int e0, int E, double* dst, int per) {
  constexpr int N3 = N1 * N1 * N1;
  const int n_el = min(EPB, E - e0);
  const double* s = src + static_cast<size_t>(e0) * NC * N3;
  for (int f = threadIdx.x; f < n_el * NC * N3; f += blockDim.x) {
    const int le = f / (NC * N3), r = f - le * NC * N3;
    dst[le * per + (r % NC) * N3 + r / NC] = __ldg(s + f);
  }
}

// W contiguous doubles per element of EPB consecutive elements (metrics, face metrics).
template <int W, int EPB>
__device__ __forceinline__ void load_flat(const double* __restrict__ src, int e0, int E, double* dst, int per) {
  const int n_el = min(EPB, E - e0);
  const double* s = src + static_cast<size_t>(e0) * W;
  for (int f = threadIdx.x; f < n_el * W; f += blockDim.x) {
    const int le = f / W;
    dst[le * per + (f - le * W)] = __ldg(s + f);
  }
}

// Roe flux along the unit normal n, Harten-Hyman fix on the acoustic waves,
// eigenvalues shifted by vg_n (flux.cpp:68-133 in rotation-invariant vector
// form: the shear waves carry rho (dv - dun n)).  False when c^2 <= 0.
__device__ __forceinline__ bool roe_flux_n(const double* ul, const double* ur, const double* n, double vgn,
                                           const GasD& g, double* f) {
  const double rl = ul[0], rr = ur[0];
  const double irl = rcp_nr(rl), irr = rcp_nr(rr);
  const double vl0 = ul[1] * irl, vl1 = ul[2] * irl, vl2 = ul[3] * irl;
  const double vr0 = ur[1] * irr, vr1 = ur[2] * irr, vr2 = ur[3] * irr;
  const double pl = g.gm1 * (ul[4] - 0.5 * (ul[1] * vl0 + ul[2] * vl1 + ul[3] * vl2));
  const double pr = g.gm1 * (ur[4] - 0.5 * (ur[1] * vr0 + ur[2] * vr1 + ur[3] * vr2));
  const double hl = (ul[4] + pl) * irl, hr = (ur[4] + pr) * irr;
  const double cl = sqrt_nr(g.gamma * pl * irl), cr = sqrt_nr(g.gamma * pr * irr);
  const double unl = vl0 * n[0] + vl1 * n[1] + vl2 * n[2];
  const double unr = vr0 * n[0] + vr1 * n[1] + vr2 * n[2];

  const double sl = sqrt_nr(rl), sr = sqrt_nr(rr);
  const double inv = rcp_nr(sl + sr);
  const double v0 = (sl * vl0 + sr * vr0) * inv, v1 = (sl * vl1 + sr * vr1) * inv, v2 = (sl * vl2 + sr * vr2) * inv;
  const double h = (sl * hl + sr * hr) * inv;
  const double un = v0 * n[0] + v1 * n[1] + v2 * n[2];
  const double q2 = v0 * v0 + v1 * v1 + v2 * v2;
  const double c2 = g.gm1 * (h - 0.5 * q2);
  if (!(c2 > 0.0)) return false;
  const double c = sqrt_nr(c2);
  const double ic2 = rcp_nr(c2);
  const double rho = sl * sr;

  const double dp = pr - pl, dun = unr - unl, drho = rr - rl;
  const double dt0 = (vr0 - vl0) - dun * n[0], dt1 = (vr1 - vl1) - dun * n[1], dt2 = (vr2 - vl2) - dun * n[2];
  const double a1 = (dp - rho * c * dun) * 0.5 * ic2;
  const double a2 = drho - dp * ic2;
  const double a4 = (dp + rho * c * dun) * 0.5 * ic2;
  const double l1 = entropy_fix(un - c - vgn, unl - cl - vgn, unr - cr - vgn);
  const double l2 = fabs(un - vgn);
  const double l4 = entropy_fix(un + c - vgn, unl + cl - vgn, unr + cr - vgn);
  const double w1 = l1 * a1, w2 = l2 * a2, w4 = l4 * a4;
  const double d0 = w1 + w2 + w4;
  const double wc = (w4 - w1) * c, lr = l2 * rho;
  const double dm0 = d0 * v0 + wc * n[0] + lr * dt0;
  const double dm1 = d0 * v1 + wc * n[1] + lr * dt1;
  const double dm2 = d0 * v2 + wc * n[2] + lr * dt2;
  const double dE = w1 * (h - un * c) + w2 * 0.5 * q2 + w4 * (h + un * c) + lr * (v0 * dt0 + v1 * dt1 + v2 * dt2);

  f[0] = 0.5 * ((rl * unl - vgn * rl) + (rr * unr - vgn * rr) - d0);
  f[1] = 0.5 * ((ul[1] * unl + pl * n[0] - vgn * ul[1]) + (ur[1] * unr + pr * n[0] - vgn * ur[1]) - dm0);
  f[2] = 0.5 * ((ul[2] * unl + pl * n[1] - vgn * ul[2]) + (ur[2] * unr + pr * n[1] - vgn * ur[2]) - dm1);
  f[3] = 0.5 * ((ul[3] * unl + pl * n[2] - vgn * ul[3]) + (ur[3] * unr + pr * n[2] - vgn * ur[3]) - dm2);
  f[4] = 0.5 * (((ul[4] + pl) * unl - vgn * ul[4]) + ((ur[4] + pr) * unr - vgn * ur[4]) - dE);
  return true;
}

// Viscous normal flux Fv . n, components 1..4 (flux.cpp:23-42 contracted with n).
__device__ __forceinline__ void fv_n(const double* u, const double* gr, const double* n, const GasD& g, double* o) {
  const double ir = rcp_nr(u[0]);
  const double v0 = u[1] * ir, v1 = u[2] * ir, v2 = u[3] * ir;
  const double div = gr[0] + gr[4] + gr[8];
  const double t00 = 2.0 * g.mu * gr[0] + g.lam * div;
  const double t11 = 2.0 * g.mu * gr[4] + g.lam * div;
  const double t22 = 2.0 * g.mu * gr[8] + g.lam * div;
  const double t01 = g.mu * (gr[1] + gr[3]);
  const double t02 = g.mu * (gr[2] + gr[6]);
  const double t12 = g.mu * (gr[5] + gr[7]);
  const double r0 = t00 * n[0] + t01 * n[1] + t02 * n[2];
  const double r1 = t01 * n[0] + t11 * n[1] + t12 * n[2];
  const double r2 = t02 * n[0] + t12 * n[1] + t22 * n[2];
  const double dT = gr[9] * n[0] + gr[10] * n[1] + gr[11] * n[2];
  o[0] = r0;
  o[1] = r1;
  o[2] = r2;
  o[3] = r0 * v0 + r1 * v1 + r2 * v2 + g.kcond * dT;
}

// Curved BR1 gradient at one node, conservative weak form:
//   g_c = (1/J) sum_d [ lw1 q*+ (n sJ)+_c - lw0 q*- (n sJ)-_c - sum_m Dhat(ia, m) Ja^d_c(m) q(m) ].
// sq [4][N3], sJa [10][N3] (Ja^d_c at 3d + c), sLift [6][4][N2], sfm [6][N2][4].
template <int N1, int FW, bool ROT>
__device__ __forceinline__ void node_gradient_curved(const double* tab, const double* sq, const double* sJa,
                                                     const double* sLift, const double* sfm, int i, int j, int k,
                                                     const Rot& rot, double* g) {
  constexpr int N2 = N1 * N1, N3 = N2 * N1;
  const double* dh = tab;
  const double* lw = tab + N1 * N1 + 2 * N1;  // liftw[0][.], liftw[1][.]
  double acc[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) acc[q] = 0.0;
  const int rv = node_rot<N1>((i * N1 + j) * N1 + k);
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int ia = d == 0 ? i : (d == 1 ? j : k);
    const int base = d == 0 ? j * N1 + k : (d == 1 ? i * N2 + k : (i * N1 + j) * N1);
    const int stride = d == 0 ? N2 : (d == 1 ? N1 : 1);
    // Bank rotation (node_rot, 0 or 1) of the lines along i and j: nodes rv, .., N1-1, then node 0 if rv.
    const int r = d == 2 ? 0 : rv;
    const int b0 = base + r * stride, bl = base + (r ? 0 : (N1 - 1) * stride);
    const double* dq = dh + ia * N1 + r;
    const double dl = dh[ia * N1 + (r ? 0 : N1 - 1)];
#pragma unroll
    for (int m = 0; m < N1; ++m) {
      const double c = d == 2 ? dhat_k<N1>(tab, ia, m) : (m < N1 - 1 ? dq[m] : dl);
      const int nd = m < N1 - 1 ? b0 + m * stride : bl;
      const double ja0 = sJa[(3 * d + 0) * N3 + nd], ja1 = sJa[(3 * d + 1) * N3 + nd],
                   ja2 = sJa[(3 * d + 2) * N3 + nd];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double cq = c * sq[q * N3 + nd];
        acc[3 * q + 0] += cq * ja0;
        acc[3 * q + 1] += cq * ja1;
        acc[3 * q + 2] += cq * ja2;
      }
    }
  }
  // The surface terms go into the same accumulators (volume minus surface): 12 live values, not 24.
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int ia = d == 0 ? i : (d == 1 ? j : k);
    const int f = d == 0 ? j * N1 + k : (d == 1 ? i * N1 + k : i * N1 + j);
    const double* np = sfm + (2 * d + 1) * FW * N2 + f;  // [c][f]
    const double* nm = sfm + (2 * d) * FW * N2 + f;
    const double sp = lw[N1 + ia] * np[3 * N2], sm = lw[ia] * nm[3 * N2];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double lp = sLift[((2 * d + 1) * 4 + q) * N2 + f] * sp;
      const double lm = sLift[((2 * d) * 4 + q) * N2 + f] * sm;
#pragma unroll
      for (int kk = 0; kk < 3; ++kk) acc[3 * q + kk] += lm * nm[kk * N2] - lp * np[kk * N2];
    }
  }
  const double nij = -sJa[9 * N3 + (i * N1 + j) * N1 + k];
#pragma unroll
  for (int q = 0; q < 12; ++q) g[q] = nij * acc[q];
  if (ROT) {  // computed with the t = 0 metrics: g(t) = R g
#pragma unroll
    for (int q = 0; q < 4; ++q) rotate_yz(rot, g[3 * q + 1], g[3 * q + 2]);
  }
}

// ----------------------------------------------------------------------------
// k_gradient_curved: lift* -> curved gradient -> Fv.n (conforming sides) /
// gradient traces (sliding and Dirichlet sides); grad_out for compute_gradients.
// ----------------------------------------------------------------------------
template <int N1, bool ROT>
__global__ void __launch_bounds__(CDim<N1, ROT>::THREADS) k_gradient_curved(const __grid_constant__ ElemConsts C,
                                                                            FieldPtrs P, const __grid_constant__ StageArgs A) {
  using D = CDim<N1, ROT>;
  constexpr int N2 = N1 * N1, N3 = N2 * N1, EPB = D::EPB, TAB = Dim<N1>::TAB, PER = D::PER_GRAD;
  constexpr int MW = D::MW, FW = D::FW;
  extern __shared__ double smem[];
  double* tab = smem;
  load_tables<N1>(C, tab);
  const int e0 = P.e_first + blockIdx.x * EPB;
  double* base = smem + TAB;
  load_soa<N1, EPB, 5>(P.U, e0, P.E, base, PER);
  load_flat<MW * N3, EPB>(P.met, e0, P.E, base + 9 * N3, PER);
  load_flat<6 * FW * N2, EPB>(P.fmet, e0, P.E, base + (21 + MW) * N3 + 54 * N2, PER);
  const int le = threadIdx.x / N3, t = threadIdx.x % N3, e = e0 + le;
  const bool active = e < P.E;
  double* su = base + le * PER;
  double* sq = su + 5 * N3;
  double* sJa = sq + 4 * N3;
  double* sG = sJa + MW * N3;
  double* sTr = sG + 12 * N3;
  double* sLift = sTr + 30 * N2;
  double* sfm = sLift + 24 * N2;
  const int band = active ? P.coords[4 * e] : 0;
  const BandD& B = C.bands[band];
  const Rot rot = band_rotation(ROT, A, band);
  __syncthreads();
  if (active) {
    double u[5], q[4];
#pragma unroll
    for (int v = 0; v < 5; ++v) u[v] = su[v * N3 + t];
    prim4(u, C.gas, q);
#pragma unroll
    for (int c = 0; c < 4; ++c) sq[c * N3 + t] = q[c];
    face_lift_phase<N1>(C, P, tab, su, e, A.t_stage, sLift, sTr);
  }
  __syncthreads();
  if (active) {
    const int i = t / N2, j = (t / N1) % N1, k = t % N1;
    double g[12];
    node_gradient_curved<N1, FW, ROT>(tab, sq, sJa, sLift, sfm, i, j, k, rot, g);
#pragma unroll
    for (int c = 0; c < 12; ++c) sG[c * N3 + t] = g[c];
    if (P.grad_out != nullptr) {
      double* go = P.grad_out + (static_cast<size_t>(e) * N3 + t) * 12;
#pragma unroll
      for (int c = 0; c < 12; ++c) go[c] = g[c];
    }
  }
  __syncthreads();
  if (!active) return;
  for (int it = t; it < 6 * N2; it += N3) {
    const int s = it / N2, f = it % N2, a = f / N1, b = f % N1;
    const double* ell = tab + N1 * N1 + (s & 1) * N1;
    double gt[12];
#pragma unroll
    for (int c = 0; c < 12; ++c) gt[c] = prolong1<N1>(sG + c * N3, ell, s >> 1, a, b, face_rot<N1>(s, a, b));
    const int slot = e * 6 + s;
    const int typ = P.side_type[slot], idx = P.side_idx[slot];
    if (typ == kConforming) {
      double fv[4], nrm[3], vgn;
      face_normal<N2, FW, ROT>(sfm, s, f, rot, B, nrm, vgn);
      fv_n(sTr + (s * N2 + f) * 5, gt, nrm, C.gas, fv);
      double* dst = P.fvn + (static_cast<size_t>(slot) * N2 + f) * 4;
#pragma unroll
      for (int c = 0; c < 4; ++c) dst[c] = fv[c];
    } else {
      double* dst = (typ == kSliding ? P.slide_g : P.dir_g) + (static_cast<size_t>(idx) * N2 + f) * 12;
#pragma unroll
      for (int c = 0; c < 12; ++c) dst[c] = gt[c];
    }
  }
}

// ----------------------------------------------------------------------------
// k_update_curved: face fluxes, curved gradient, contravariant volume flux and
// weak divergence, surface lift, low-storage RK update, admissibility and the
// traces of the new state (the phases of k_update with metric terms).
// ----------------------------------------------------------------------------
template <int N1, bool VISC, bool ROT>
__global__ void __launch_bounds__(CDim<N1, ROT>::THREADS) k_update_curved(const __grid_constant__ ElemConsts C,
                                                                          FieldPtrs P, const __grid_constant__ StageArgs A) {
  using D = CDim<N1, ROT>;
  constexpr int N2 = N1 * N1, N3 = N2 * N1, EPB = D::EPB, TAB = Dim<N1>::TAB, PER = D::PER_UPD;
  constexpr int MW = D::MW, FW = D::FW;
  extern __shared__ double smem[];
  double* tab = smem;
  load_tables<N1>(C, tab);
  const int e0 = P.e_first + blockIdx.x * EPB;
  double* elems = smem + TAB;
  load_soa<N1, EPB, 5>(P.U, e0, P.E, elems, PER);
  load_flat<MW * N3, EPB>(P.met, e0, P.E, elems + 10 * N3, PER);
  load_flat<6 * FW * N2, EPB>(P.fmet, e0, P.E, elems + (10 + MW) * N3 + 54 * N2, PER);
  const int le = threadIdx.x / N3, t = threadIdx.x % N3, e = e0 + le;
  const bool active = e < P.E;
  double* su = elems + le * PER;
  double* sF = su + 5 * N3;
  double* sJa = sF + 5 * N3;
  double* sLift = sJa + MW * N3;
  double* sFlux = sLift + 24 * N2;
  double* sfm = sFlux + 30 * N2;
  const int i = t / N2, j = (t / N1) % N1, k = t % N1;
  const int band = active ? P.coords[4 * e] : 0;
  const BandD& B = C.bands[band];
  const Rot rot = band_rotation(ROT, A, band);
  __syncthreads();

  // Phase 1: numerical flux along each face node's normal -> sFlux[s][v][f]; lift* -> sLift.
  if (active) {
    if (VISC) {
      double u[5], q[4];
#pragma unroll
      for (int v = 0; v < 5; ++v) u[v] = su[v * N3 + t];
      prim4(u, C.gas, q);
#pragma unroll
      for (int c = 0; c < 4; ++c) sF[c * N3 + t] = q[c];
    }
    for (int it = t; it < 6 * N2; it += N3) {
      const int s = it / N2, f = it % N2, a = f / N1, b = f % N1, dir = s >> 1;
      const double* ell = tab + N1 * N1 + (s & 1) * N1;
      double own[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) own[v] = prolong1<N1>(su + v * N3, ell, dir, a, b, face_rot<N1>(s, a, b));
      double nrm[3], vgn;
      face_normal<N2, FW, ROT>(sfm, s, f, rot, B, nrm, vgn);
      const int slot = e * 6 + s;
      const int typ = P.side_type[slot], idx = P.side_idx[slot];
      double flux[5], lift[4];
      bool ok = true;
      if (typ == kConforming) {
        const double* nb = P.trace + static_cast<size_t>(idx) * N2 * 5 + f * 5;
        double other[5], fvo[4];
#pragma unroll
        for (int v = 0; v < 5; ++v) other[v] = nb[v];
        const int kr = ROT ? P.side_rot[slot] : 0;  // periodic annulus sector seam
        if (kr != 0) rot_yz(C.sec_c, kr * C.sec_s, other[2], other[3]);
        const double* um = (s & 1) ? own : other;
        const double* up = (s & 1) ? other : own;
        ok = roe_flux_n(um, up, nrm, vgn, C.gas, flux);
        if (VISC) {
          double qa[4], qb[4];
          prim4(own, C.gas, qa);
          prim4(other, C.gas, qb);
#pragma unroll
          for (int c = 0; c < 4; ++c) lift[c] = __dmul_rn(0.5, __dadd_rn(qa[c], qb[c]));
          const double* pa = P.fvn + (static_cast<size_t>(slot) * N2 + f) * 4;
#pragma unroll
          for (int c = 0; c < 4; ++c) fvo[c] = P.fvn[(static_cast<size_t>(idx) * N2 + f) * 4 + c];
          if (kr != 0) rot_yz(C.sec_c, kr * C.sec_s, fvo[1], fvo[2]);
          const double* pb = fvo;
          const double* fm = (s & 1) ? pa : pb;
          const double* fp = (s & 1) ? pb : pa;
#pragma unroll
          for (int c = 0; c < 4; ++c) flux[1 + c] -= 0.5 * (fm[c] + fp[c]);
        }
      } else if (typ == kSliding) {
        const double* sf = P.slide_flux + (static_cast<size_t>(idx) * N2 + f) * 5;
#pragma unroll
        for (int v = 0; v < 5; ++v) flux[v] = sf[v];
        if (VISC) {
          const double* sl = P.slide_lift + (static_cast<size_t>(idx) * N2 + f) * 4;
#pragma unroll
          for (int c = 0; c < 4; ++c) lift[c] = sl[c];
        }
      } else {
        double x[3], ext[5];
        face_position<N1>(C, P.coords + 4 * e, s, a, b, A.t_stage, x);
        eval_case(C.flow_case, x, A.t_stage, C.gas, ext);
        const double* um = (s & 1) ? own : ext;
        const double* up = (s & 1) ? ext : own;
        ok = roe_flux_n(um, up, nrm, vgn, C.gas, flux);
        if (VISC) {
          prim4(ext, C.gas, lift);
          const double* gd = P.dir_g + (static_cast<size_t>(idx) * N2 + f) * 12;
          double gg[12];
#pragma unroll
          for (int c = 0; c < 12; ++c) gg[c] = gd[c];
          double fm[4], fp[4];
          fv_n(um, gg, nrm, C.gas, fm);
          fv_n(up, gg, nrm, C.gas, fp);
#pragma unroll
          for (int c = 0; c < 4; ++c) flux[1 + c] -= 0.5 * (fm[c] + fp[c]);
        }
      }
      if (!ok) record_error(P.err, 2, A.step, A.stage, e, -1 - it, own);
#pragma unroll
      for (int v = 0; v < 5; ++v) sFlux[(s * 5 + v) * N2 + f] = flux[v];
      if (VISC) {
#pragma unroll
        for (int c = 0; c < 4; ++c) sLift[(s * 4 + c) * N2 + f] = lift[c];
      }
    }
  }
  __syncthreads();

  // Phase 2: pointwise flux (ALE convective minus viscous) -> contravariant Ja^d . F.
  double Ft[3][5];
  if (active) {
    double u[5], F[3][5];
#pragma unroll
    for (int v = 0; v < 5; ++v) u[v] = su[v * N3 + t];
    const double ir = rcp_nr(u[0]);
    const double vv[3] = {u[1] * ir, u[2] * ir, u[3] * ir};
    const double p = pressure(u, ir, C.gas);
    const double vgv[3] = {0.0, ROT ? 0.0 : B.vg, ROT ? 0.0 : B.vgz};  // annulus: grid velocity enters through V^d below
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      F[d][0] = u[0] * vv[d];
      F[d][1] = u[1] * vv[d] + (d == 0 ? p : 0.0);
      F[d][2] = u[2] * vv[d] + (d == 1 ? p : 0.0);
      F[d][3] = u[3] * vv[d] + (d == 2 ? p : 0.0);
      F[d][4] = (u[4] + p) * vv[d];
#pragma unroll
      for (int v = 0; v < 5; ++v) F[d][v] -= vgv[d] * u[v];
    }
    if (VISC) {
      double g[12];
      node_gradient_curved<N1, FW, ROT>(tab, sF, sJa, sLift, sfm, i, j, k, rot, g);
      const double div = g[0] + g[4] + g[8];
      const double mu = C.gas.mu, lam = C.gas.lam;
      const double tau[3][3] = {{2.0 * mu * g[0] + lam * div, mu * (g[1] + g[3]), mu * (g[2] + g[6])},
                                {mu * (g[1] + g[3]), 2.0 * mu * g[4] + lam * div, mu * (g[5] + g[7])},
                                {mu * (g[2] + g[6]), mu * (g[5] + g[7]), 2.0 * mu * g[8] + lam * div}};
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        F[d][1] -= tau[d][0];
        F[d][2] -= tau[d][1];
        F[d][3] -= tau[d][2];
        F[d][4] -= tau[d][0] * vv[0] + tau[d][1] * vv[1] + tau[d][2] * vv[2] + C.gas.kcond * g[9 + d];
      }
    }
    if (ROT) {  // Ja(t) . F = Ja(0) . (R^T F)
#pragma unroll
      for (int v = 0; v < 5; ++v) rotate_yz(Rot{rot.c, -rot.s}, F[1][v], F[2][v]);
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double ja0 = sJa[(3 * d) * N3 + t], ja1 = sJa[(3 * d + 1) * N3 + t], ja2 = sJa[(3 * d + 2) * N3 + t];
      const double wv = ROT ? B.vg * sJa[(10 + d) * N3 + t] : 0.0;  // contravariant grid velocity
#pragma unroll
      for (int v = 0; v < 5; ++v) Ft[d][v] = ja0 * F[0][v] + ja1 * F[1][v] + ja2 * F[2][v] - wv * u[v];
    }
  }

  // Phase 3: weak divergence sum_m Dhat(i,m) Ft(m) per direction.
  double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const double* dh = tab;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    __syncthreads();
    if (active) {
#pragma unroll
      for (int v = 0; v < 5; ++v) sF[v * N3 + t] = Ft[d][v];
    }
    __syncthreads();
    if (active) {
      const int ia = d == 0 ? i : (d == 1 ? j : k);
      const int base = d == 0 ? j * N1 + k : (d == 1 ? i * N2 + k : (i * N1 + j) * N1);
      const int stride = d == 0 ? N2 : (d == 1 ? N1 : 1);
#pragma unroll
      for (int m = 0; m < N1; ++m) {
        const double c = dh[ia * N1 + m];
#pragma unroll
        for (int v = 0; v < 5; ++v) acc[v] += c * sF[v * N3 + base + m * stride];
      }
    }
  }

  // Phase 4: surface lift with (sJ of the face node) / (J of the volume node).
  double du[5];
  if (active) {
    const double ij = sJa[9 * N3 + t];
#pragma unroll
    for (int v = 0; v < 5; ++v) du[v] = acc[v] * ij;
    const double* lw = tab + N1 * N1 + 2 * N1;
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int dir = s >> 1;
      const int ia = dir == 0 ? i : (dir == 1 ? j : k);
      const int f = dir == 0 ? j * N1 + k : (dir == 1 ? i * N1 + k : i * N1 + j);
      const double l = lw[(s & 1) * N1 + ia];
      if (l != 0.0) {
        const double c = ((s & 1) ? -1.0 : 1.0) * l * face_sj(sfm, s, f, N2, FW) * ij;
#pragma unroll
        for (int v = 0; v < 5; ++v) du[v] += c * sFlux[(s * 5 + v) * N2 + f];
      }
    }
  }
  __syncthreads();
  if (active) {
#pragma unroll
    for (int v = 0; v < 5; ++v) sF[v * N3 + t] = du[v];
  }
  __syncthreads();

  // Phase 5: flat coalesced RK update (solver.cpp:912-917) or residual store.
  const int n_el = min(EPB, P.E - e0);
  const size_t gbase = static_cast<size_t>(e0) * 5 * N3;
  if (A.mode == 1) {
    for (int fI = threadIdx.x; fI < n_el * 5 * N3; fI += blockDim.x) {
      const int l = fI / (5 * N3), r = fI - l * 5 * N3;
      P.out[gbase + fI] = elems[l * PER + 5 * N3 + (r % 5) * N3 + r / 5];
    }
    return;
  }
  for (int fI = threadIdx.x; fI < n_el * 5 * N3; fI += blockDim.x) {
    const int l = fI / (5 * N3), r = fI - l * 5 * N3;
    double* us = elems + l * PER + (r % 5) * N3 + r / 5;
    const double d = us[5 * N3];
    const double rg = A.rk_a * P.reg[gbase + fI] + A.dt * d;
    const double un = *us + A.rk_b * rg;
    P.reg[gbase + fI] = rg;
    P.U[gbase + fI] = un;
    *us = un;
  }
  __syncthreads();
  if (!active) return;
  {
    double w[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) w[v] = su[v * N3 + t];
    const double p = pressure(w, rcp_nr(w[0]), C.gas);
    bool ok = w[0] > 0.0 && p > 0.0;
#pragma unroll
    for (int v = 0; v < 5; ++v) ok = ok && isfinite(w[v]);
    if (!ok) record_error(P.err, 2, A.step, A.stage, e, t, w);
  }
  for (int it = t; it < 6 * N2; it += N3) {
    const int s = it / N2, f = it % N2, a = f / N1, b = f % N1;
    const double* ell = tab + N1 * N1 + (s & 1) * N1;
    double* dst = P.trace_out + (static_cast<size_t>(e) * 6 + s) * N2 * 5 + f * 5;
#pragma unroll
    for (int v = 0; v < 5; ++v) dst[v] = prolong1<N1>(su + v * N3, ell, s >> 1, a, b, face_rot<N1>(s, a, b));
  }
}

template <int N1, bool ROT>
void gradient_curved_r(const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st) {
  using D = CDim<N1, ROT>;
  const int blocks = (p.E - p.e_first + D::EPB - 1) / D::EPB;
  const int sm = (Dim<N1>::TAB + D::EPB * D::PER_GRAD) * 8;
  set_smem_checked(k_gradient_curved<N1, ROT>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  k_gradient_curved<N1, ROT><<<blocks, D::THREADS, sm, st>>>(c, p, a);
  check_launch("k_gradient_curved");
}
template <int N1>
void gradient_curved_t(const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st) {
  if (c.mapping == SDG_MAP_ANNULUS) gradient_curved_r<N1, true>(c, p, a, st);
  else gradient_curved_r<N1, false>(c, p, a, st);
}
template <int N1, bool ROT>
void update_curved_r(const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st) {
  using D = CDim<N1, ROT>;
  const int blocks = (p.E - p.e_first + D::EPB - 1) / D::EPB;
  const int sm = (Dim<N1>::TAB + D::EPB * D::PER_UPD) * 8;
  auto kern = c.gas.viscous ? k_update_curved<N1, true, ROT> : k_update_curved<N1, false, ROT>;
  set_smem_checked(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  kern<<<blocks, D::THREADS, sm, st>>>(c, p, a);
  check_launch("k_update_curved");
}
template <int N1>
void update_curved_t(const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st) {
  if (c.mapping == SDG_MAP_ANNULUS) update_curved_r<N1, true>(c, p, a, st);
  else update_curved_r<N1, false>(c, p, a, st);
}

// ============================================================================
// Bulk-loaded element kernels (even N+1: every per-element and per-slot block is
// a multiple of 16 bytes).  One thread issues cp.async.bulk copies of what the
// element tile stages in shared memory, completing on one mbarrier, so the
// tile's global reads are in flight together instead of as dependent load chains
// (ncu: 50% long-scoreboard stalls in the plain-load kernels above); what only
// one thread reads is loaded by that thread meanwhile.  Own traces come from
// the trace buffer, so both elements of a face use the same stored bits.
// ============================================================================
// Elements per CTA (shared memory: <= 227 KB per CTA).
template <int N1>
struct BulkEpb {
  static constexpr int EPB = N1 == 2 ? 16 : (N1 <= 4 ? Dim<N1>::EPB : 1);
};

// Exterior state of a Dirichlet face node (the exact case at the node's position).  Kept out
// of line: its position mapping and transcendental code would otherwise set the register
// budget of the whole kernel, though only boundary elements run it.
template <int N1>
__device__ __noinline__ void dirichlet_state(const ElemConsts& C, const int* crd, int side, int a, int b, double t,
                                             double* ext) {
  double x[3];
  face_position<N1>(C, crd, side, a, b, t, x);
  eval_case(C.flow_case, x, t, C.gas, ext);
}

// ============================================================================
// k_gradient_cv: lift* -> curved gradient -> Fv.n (conforming sides) / gradient
// traces (sliding and Dirichlet sides), the node's viscous stress for k_update_cv
// (N = 5: 55 KB of shared memory and <= 72 registers, 4 CTAs per SM).
//   * the node's state is read by its own thread (it is only needed for the
//     primitive variables), not staged;
//   * only the metric rows the gradient uses are staged: Ja and 1/J of the node
//     metrics, unit normal and sJ of the face metrics (compact [side][4][f]);
//   * the gradient is accumulated in one set of 12 registers (volume minus surface).
// Shared memory per element: met (Ja, 1/J) | q  (later the gradient [12][node]) |
// face metrics | own traces | neighbour trace / lift* (later Fv.n) | lift*.
// ============================================================================
template <int N1, bool ROT>
struct CG {
  static constexpr int N2 = N1 * N1, N3 = N2 * N1;
  static constexpr int MWG = MWidth<ROT>::MW, FWG = MWidth<ROT>::FW;  // row counts in global memory
  static constexpr int EPB = BulkEpb<N1>::EPB;
  static constexpr int THREADS = EPB * N3;
  static constexpr int TAB = Dim<N1>::TAB;
  static constexpr int EL = 5 * N3, ML = 10 * N3, SQ = 4 * N3, FMC = 6 * 4 * N2, TS = 5 * N2, FS = 4 * N2;
  static constexpr int PER = ML + SQ + FMC + 6 * TS + 6 * TS + 6 * FS;
  static constexpr int KF = (6 * N2 + N3 - 1) / N3;
#ifndef SDG_CG_MINB
#define SDG_CG_MINB 4
#endif
  static constexpr int MINB = N1 == 6 ? SDG_CG_MINB : 1;
  static constexpr int SMEM = (TAB + EPB * PER) * 8 + 16;
  static_assert(12 * N3 <= ML + SQ, "gradient aliases metrics + q");
  static_assert(N1 % 2 == 0, "bulk path needs even N+1");
  static_assert(SMEM <= 227 * 1024, "shared memory per CTA");
};

template <int N1, bool ROT>
__device__ __forceinline__ void cg_issue_loads(const FieldPtrs& P, int e0, int n, double* base, uint64_t* bar) {
  using D = CG<N1, ROT>;
  constexpr int N2 = D::N2;
  uint32_t bytes = n * (D::ML + D::FMC + 6 * D::TS) * 8u;
  for (int le = 0; le < n; ++le) {
    const int e = e0 + le;
    double* b = base + le * D::PER;
    bulk_g2s(b, P.met + static_cast<size_t>(e) * D::MWG * D::N3, D::ML * 8u, bar);
    for (int sd = 0; sd < 6; ++sd)  // [side][c][f]: normal and sJ rows of every side
      bulk_g2s(b + D::ML + D::SQ + sd * 4 * N2, P.fmet + (static_cast<size_t>(e) * 6 + sd) * D::FWG * N2, 4 * N2 * 8u,
               bar);
    bulk_g2s(b + D::ML + D::SQ + D::FMC, P.trace + static_cast<size_t>(e) * 6 * D::TS, 6 * D::TS * 8u, bar);
  }
  constexpr int MASK = (1 << kCodeShift) - 1;
  for (int le = 0; le < n; ++le) {
    const int e = e0 + le;
    const int4 c0 = *reinterpret_cast<const int4*>(P.side_code + 8 * e);
    const int2 c1 = *reinterpret_cast<const int2*>(P.side_code + 8 * e + 4);
    const int code[6] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y};
    double* nb = base + le * D::PER + D::ML + D::SQ + D::FMC + 6 * D::TS;
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int typ = code[s] >> kCodeShift, idx = code[s] & MASK;
      if (typ == kConforming) {
        bulk_g2s(nb + s * D::TS, P.trace + static_cast<size_t>(idx) * D::TS, D::TS * 8u, bar);
        bytes += D::TS * 8u;
      } else if (typ == kSliding) {
        bulk_g2s(nb + s * D::TS, P.slide_lift + static_cast<size_t>(idx) * D::FS, D::FS * 8u, bar);
        bytes += D::FS * 8u;
      }
    }
  }
  mbar_arrive_expect_tx(bar, bytes);
}

template <int N1, bool ROT>
__global__ void __launch_bounds__(CG<N1, ROT>::THREADS, CG<N1, ROT>::MINB) k_gradient_cv(
    const __grid_constant__ ElemConsts C, FieldPtrs P, const __grid_constant__ StageArgs A) {
  using D = CG<N1, ROT>;
  constexpr int N2 = D::N2, N3 = D::N3, EPB = D::EPB, PER = D::PER, KF = D::KF;
  extern __shared__ __align__(128) double smem[];
  double* tab = smem;
  double* base = smem + D::TAB;
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + EPB * PER);
  const int e0 = P.e_first + blockIdx.x * EPB;
  const int n_el = min(EPB, P.E - e0);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
    cg_issue_loads<N1, ROT>(P, e0, n_el, base, bar);
  }
  const int le = threadIdx.x / N3, t = threadIdx.x % N3, e = e0 + le;
  const bool active = le < n_el;
  double* sM = base + le * PER;   // [c][node], c < 10
  double* sq = sM + D::ML;        // [c][node], c < 4
  double* sfm = sq + D::SQ;       // [side][c][f], c < 4
  double* sTr = sfm + D::FMC;     // [side][f][5]
  double* sNb = sTr + 6 * D::TS;  // [side]: trace [f][5] or lift* [f][4]
  double* sLift = sNb + 6 * D::TS;
  double* sG = sM;                // [c][node], c < 12, once every node's gradient is computed
  // While the bulk copies are in flight: this node's state and this thread's side types.  Nothing
  // before the wait depends on another load's result (the band is used after it), so every
  // thread's loads leave at once.
  const int band_ld = active ? P.side_code[8 * e + 6] : 0;
  double u[5];
  int typs[KF], rots[KF];
  if (active) {
    const double* up = P.U + (static_cast<size_t>(e) * N3 + t) * 5;
#pragma unroll
    for (int v = 0; v < 5; ++v) u[v] = __ldg(up + v);
  }
#pragma unroll
  for (int kf = 0; kf < KF; ++kf) {
    const int it = t + kf * N3;
    const bool on = active && it < 6 * N2;
    typs[kf] = on ? P.side_type[e * 6 + it / N2] : 0;
    rots[kf] = (ROT && on) ? P.side_rot[e * 6 + it / N2] : 0;
  }
  // Elements whose six sides are all conforming need only Fv.n on their faces: the stress and
  // heat flux are linear in the gradient, so their 9 components are prolonged instead of
  // the gradient's 12.  Sliding / Dirichlet sides need the gradient trace itself.
  bool allconf = false;
  load_tables<N1>(C, tab);
  if constexpr (EPB == 1) {
    // One element per CTA: the barrier before the wait doubles as the vote over the side types.
    bool mine = true;
#pragma unroll
    for (int kf = 0; kf < KF; ++kf) mine = mine && (t + kf * N3 >= 6 * N2 || typs[kf] == kConforming);
    allconf = __syncthreads_and(mine) != 0;  // barrier init visible, tables loaded
  } else {
    if (active) {
      constexpr int MASK = (1 << kCodeShift) - 1;
      const int4 c0 = __ldg(reinterpret_cast<const int4*>(P.side_code + 8 * e));
      const int2 c1 = __ldg(reinterpret_cast<const int2*>(P.side_code + 8 * e + 4));
      const int any = (c0.x | c0.y | c0.z | c0.w | c1.x | c1.y) & ~MASK;
      const int all = (c0.x & c0.y & c0.z & c0.w & c1.x & c1.y) & ~MASK;
      allconf = any == (kConforming << kCodeShift) && all == (kConforming << kCodeShift);
    }
    __syncthreads();  // barrier init visible, tables loaded
  }
  mbar_wait(bar, 0);
  const Rot rot = band_rotation(ROT, A, band_ld);
  if (active) {
    double q[4];
    prim4(u, C.gas, q);
#pragma unroll
    for (int c = 0; c < 4; ++c) sq[c * N3 + t] = q[c];
    // BR1 surface values lift* (run_lifting, solver.cpp:606-723).
#pragma unroll
    for (int kf = 0; kf < KF; ++kf) {
      const int it = t + kf * N3;
      if (it >= 6 * N2) break;
      const int s = it / N2, f = it - s * N2, a = f / N1, b = f % N1;
      const int typ = typs[kf];
      double lift[4];
      if (typ == kConforming) {
        double other[5], qa[4], qb[4];
#pragma unroll
        for (int v = 0; v < 5; ++v) other[v] = sNb[it * 5 + v];
        if constexpr (ROT) {  // periodic annulus sector seam
          if (rots[kf] != 0) rot_yz(C.sec_c, rots[kf] * C.sec_s, other[2], other[3]);
        }
        prim4(sTr + it * 5, C.gas, qa);
        prim4(other, C.gas, qb);
#pragma unroll
        for (int c = 0; c < 4; ++c) lift[c] = __dmul_rn(0.5, __dadd_rn(qa[c], qb[c]));
      } else if (typ == kSliding) {
#pragma unroll
        for (int c = 0; c < 4; ++c) lift[c] = sNb[s * D::TS + f * 4 + c];
      } else {
        double ext[5];
        dirichlet_state<N1>(C, P.coords + 4 * e, s, a, b, A.t_stage, ext);
        prim4(ext, C.gas, lift);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) sLift[(s * 4 + c) * N2 + f] = lift[c];
    }
  }
  __syncthreads();
  double g[12];
  if (active) {
    const int i = t / N2, j = (t / N1) % N1, k = t % N1;
    node_gradient_curved<N1, 4, ROT>(tab, sq, sM, sLift, sfm, i, j, k, rot, g);
    if (P.grad_out != nullptr) {
      double* go = P.grad_out + (static_cast<size_t>(e) * N3 + t) * 12;
#pragma unroll
      for (int c = 0; c < 12; ++c) go[c] = g[c];
    }
    double vs[9];
    visc_terms(g, C.gas, vs);
    if (P.visc != nullptr) {  // stress and heat flux of the node for k_update_cv (coalesced rows [c][node])
      double* vo = P.visc + static_cast<size_t>(e) * 9 * N3 + t;
#pragma unroll
      for (int c = 0; c < 9; ++c) vo[c * N3] = vs[c];
    }
    if (allconf) {
#pragma unroll
      for (int c = 0; c < 9; ++c) g[c] = vs[c];
    }
  }
  __syncthreads();  // every node's gradient is computed: metrics and q are dead
  if (active) {
    if (allconf) {
#pragma unroll
      for (int c = 0; c < 9; ++c) sG[c * N3 + t] = g[c];
    } else {
#pragma unroll
      for (int c = 0; c < 12; ++c) sG[c * N3 + t] = g[c];
    }
  }
  __syncthreads();
  // Fv.n of the 6 sides staged in the dead neighbour-trace region [side][f][4]
  // (zero on sliding / Dirichlet sides) and bulk-stored as one contiguous block.
  double* sOut = sNb;
  if (active) {
#pragma unroll
    for (int kf = 0; kf < KF; ++kf) {
      const int it = t + kf * N3;
      if (it >= 6 * N2) break;
      const int s = it / N2, f = it - s * N2, a = f / N1, b = f % N1;
      const double* ell = tab + N1 * N1 + (s & 1) * N1;
      const double* fm = sfm + s * 4 * N2 + f;
      double nrm[3] = {fm[0], fm[N2], fm[2 * N2]};
      if (ROT) rotate_yz(rot, nrm[1], nrm[2]);
      double fv[4] = {0.0, 0.0, 0.0, 0.0};
      if (allconf) {  // Fv.n from the prolonged stress and heat flux (flux.cpp:23-42 contracted with n)
        double vt[9];
#pragma unroll
        for (int c = 0; c < 9; ++c) vt[c] = prolong1<N1>(sG + c * N3, ell, s >> 1, a, b, face_rot<N1>(s, a, b));
        const double* uo = sTr + it * 5;
        const double ir = rcp_nr(uo[0]);
        fv[0] = vt[0] * nrm[0] + vt[1] * nrm[1] + vt[2] * nrm[2];
        fv[1] = vt[1] * nrm[0] + vt[3] * nrm[1] + vt[4] * nrm[2];
        fv[2] = vt[2] * nrm[0] + vt[4] * nrm[1] + vt[5] * nrm[2];
        fv[3] = (fv[0] * uo[1] + fv[1] * uo[2] + fv[2] * uo[3]) * ir + vt[6] * nrm[0] + vt[7] * nrm[1] + vt[8] * nrm[2];
        double2* so = reinterpret_cast<double2*>(sOut + it * 4);  // [f][4]: 128-bit stores, no 4-way conflict
        so[0] = make_double2(fv[0], fv[1]);
        so[1] = make_double2(fv[2], fv[3]);
        continue;
      }
      double gt[12];
#pragma unroll
      for (int c = 0; c < 12; ++c) gt[c] = prolong1<N1>(sG + c * N3, ell, s >> 1, a, b, face_rot<N1>(s, a, b));
      const int typ = typs[kf];
      if (typ == kConforming) {
        fv_n(sTr + it * 5, gt, nrm, C.gas, fv);
      } else {
        const int idx = P.side_idx[e * 6 + s];
        double* dst = (typ == kSliding ? P.slide_g : P.dir_g) + (static_cast<size_t>(idx) * N2 + f) * 12;
#pragma unroll
        for (int c = 0; c < 12; ++c) dst[c] = gt[c];
      }
      double2* so = reinterpret_cast<double2*>(sOut + it * 4);
      so[0] = make_double2(fv[0], fv[1]);
      so[1] = make_double2(fv[2], fv[3]);
    }
    fence_proxy_async();
  }
  __syncthreads();
  if (active && t == 0) {
    bulk_s2g(P.fvn + static_cast<size_t>(e) * 6 * D::FS, sOut, 6 * D::FS * 8u);
    bulk_commit();
    bulk_wait_read0();
  }
}

// ============================================================================
// k_update_cv: the update kernel of curved and (AFF) affine elements (even N+1).
//   * The node's viscous stress and heat flux come from the gradient kernel (P.visc),
//     so the BR1 gradient is evaluated once per stage, not again here.
//   * What only one thread reads is loaded by that thread while the tile's bulk
//     copies are in flight: a face node's own trace, Fv.n and face metrics.
//     State, node metrics, stresses and the neighbour slots are bulk-copied onto
//     one mbarrier.
//   * The three contravariant flux directions are staged at once over the node's
//     own metric / stress columns (thread-local aliasing: no barrier between the
//     pointwise flux and the staging), so one CTA barrier separates the face and
//     pointwise phases from the weak divergence.
//   * The RK register is L2-prefetched with the tile and fetched into registers
//     before that barrier.
// Shared memory per element: U | met, visc (later 3 x 5 staged fluxes) | face flux
// | face sJ | neighbour slots (later dudt, then the new traces).
// ============================================================================
template <int N1, bool ROT, bool VISC, bool AFF = false>
struct CV {
  static constexpr int N2 = N1 * N1, N3 = N2 * N1;
  static constexpr int MW = MWidth<ROT>::MW, FW = MWidth<ROT>::FW;
  static constexpr int EPB = BulkEpb<N1>::EPB;
  static constexpr int THREADS = EPB * N3;
  static constexpr int TAB = Dim<N1>::TAB;
  static constexpr int EL = 5 * N3, ML = AFF ? 0 : MW * N3, VL = VISC ? 9 * N3 : 0;
  // Directions staged at once for the weak divergence: all three (15 rows), or two and then
  // the third (10 rows, two more barriers) where that buys another resident CTA: affine N = 7,
  // 104 instead of 125 KB -> 2 CTAs/SM at 64 registers, 18.1 -> 16.7 ms at 64^3 elements
  // (affine N = 5 at 4 CTAs x 72 registers lost: 5.47 -> 5.68 ms; profiles/r2l_ab.txt).
  static constexpr int PASSES = (AFF && N1 == 8) ? 2 : 1;
  static constexpr int FROWS = PASSES == 1 ? 15 : 10;
  static constexpr int MV = (ML + VL > FROWS * N3 ? ML + VL : FROWS * N3);
  static constexpr int TS = 5 * N2, FS = 4 * N2, NB = TS + (VISC ? FS : 0);
  static constexpr int FX = 6 * TS, SJ = AFF ? 0 : 6 * N2;
  static constexpr int NBR = 6 * NB > EL ? 6 * NB : EL;
  static constexpr int PER = EL + MV + FX + SJ + NBR;
  static constexpr int KF = (6 * N2 + N3 - 1) / N3;  // face nodes per thread
  static constexpr int FM = 6 * FW * N2;
#ifndef SDG_CV_MINB
#define SDG_CV_MINB 3
#endif
#ifndef SDG_CVA_MINB
#define SDG_CVA_MINB 3  // affine: 58 KB per CTA
#endif
#ifndef SDG_CVA_MINB8
#define SDG_CVA_MINB8 2
#endif
#ifndef SDG_CVA_MINB4
#define SDG_CVA_MINB4 2
#endif
  static constexpr int MINB = N1 == 6   ? (AFF ? SDG_CVA_MINB : SDG_CV_MINB)
                              : N1 == 8 ? (AFF ? SDG_CVA_MINB8 : 1)
                              : N1 == 4 ? (AFF ? SDG_CVA_MINB4 : 1)
                                        : 1;
  // (Registers: the file is split over the SM's four schedulers, 16K each.  3 CTAs of 7 warps put 6
  // warps on one scheduler -> at most 85 registers per thread; __launch_bounds__ makes ptxas stop at 80.
  // A 96-register build -- 21 warps x 96 x 32 fits the SM's 64K as a whole -- ran 2 CTAs per SM.)
  static constexpr int SMEM = (TAB + EPB * PER) * 8 + 16;
  static_assert(N1 % 2 == 0, "bulk path needs even N+1");
  static_assert(SMEM <= 227 * 1024, "shared memory per CTA");
  static_assert(6 * TS <= NBR, "new traces fit the neighbour region");
};

template <int N1, bool ROT, bool VISC, bool AFF>
__device__ __forceinline__ void cv_issue_loads(const FieldPtrs& P, int e0, int n, double* base, uint64_t* bar) {
  using D = CV<N1, ROT, VISC, AFF>;
  uint32_t bytes = n * (D::EL + D::ML + D::VL) * 8u;
  for (int le = 0; le < n; ++le) {
    const int e = e0 + le;
    double* b = base + le * D::PER;
    bulk_g2s(b, P.U + static_cast<size_t>(e) * D::EL, D::EL * 8u, bar);
    if (!AFF) bulk_g2s(b + D::EL, P.met + static_cast<size_t>(e) * D::ML, D::ML * 8u, bar);
    if (VISC) bulk_g2s(b + D::EL + D::ML, P.visc + static_cast<size_t>(e) * D::VL, D::VL * 8u, bar);
  }
  constexpr int MASK = (1 << kCodeShift) - 1;
  for (int le = 0; le < n; ++le) {
    const int e = e0 + le;
    const int4 c0 = *reinterpret_cast<const int4*>(P.side_code + 8 * e);
    const int2 c1 = *reinterpret_cast<const int2*>(P.side_code + 8 * e + 4);
    const int code[6] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y};
    double* nb = base + le * D::PER + D::EL + D::MV + D::FX + D::SJ;
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int typ = code[s] >> kCodeShift, idx = code[s] & MASK;
      double* d = nb + s * D::NB;
      if (typ == kConforming) {
        bulk_g2s(d, P.trace + static_cast<size_t>(idx) * D::TS, D::TS * 8u, bar);
        bytes += D::TS * 8u;
        if (VISC) {
          bulk_g2s(d + D::TS, P.fvn + static_cast<size_t>(idx) * D::FS, D::FS * 8u, bar);
          bytes += D::FS * 8u;
        }
      } else if (typ == kSliding) {
        bulk_g2s(d, P.slide_flux + static_cast<size_t>(idx) * D::TS, D::TS * 8u, bar);
        bytes += D::TS * 8u;
      }
    }
  }
  mbar_arrive_expect_tx(bar, bytes);
}

template <int N1, bool VISC, bool ROT, bool AFF = false>
__global__ void __launch_bounds__(CV<N1, ROT, VISC, AFF>::THREADS, CV<N1, ROT, VISC, AFF>::MINB) k_update_cv(
    const __grid_constant__ ElemConsts C, FieldPtrs P, const __grid_constant__ StageArgs A) {
  using D = CV<N1, ROT, VISC, AFF>;
  constexpr int FW = D::FW, KF = D::KF;
  constexpr int N2 = D::N2, N3 = D::N3, EPB = D::EPB, PER = D::PER, THREADS = D::THREADS;
  extern __shared__ __align__(128) double smem[];
  double* tab = smem;
  double* base = smem + D::TAB;
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + EPB * PER);
  const int e0 = P.e_first + blockIdx.x * EPB;
  const int n_el = min(EPB, P.E - e0);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
    cv_issue_loads<N1, ROT, VISC, AFF>(P, e0, n_el, base, bar);
    if (A.mode == 0 && A.rk_a != 0.0) bulk_prefetch_l2(P.reg + static_cast<size_t>(e0) * D::EL, n_el * D::EL * 8u);
  }
  const int le = threadIdx.x / N3, t = threadIdx.x % N3, e = e0 + le;
  const bool active = le < n_el;
  double* sU = base + le * PER;
  double* sM = sU + D::EL;           // [c][node], c < MW
  double* sV = sM + D::ML;           // [c][node], c < 9
  double* sF3 = sM;                  // [d][v][node] once the node's own columns are consumed
  double* sFlux = sM + D::MV;        // [side][v][f]
  double* sSJ = sFlux + D::FX;       // [side][f]
  double* sNb = sSJ + D::SJ;         // [side]: trace [f][5] | Fv.n [f][4]  (sliding: flux [f][5])
  double* sD = sNb;                  // dudt [node][5], after the face phase
  const int i = t / N2, j = (t / N1) % N1, k = t % N1;
  const int band_ld = active ? P.side_code[8 * e + 6] : 0;  // used after the wait: no load below depends on it

  // This thread's face nodes: own trace, own Fv.n, unit normal, sJ and vg.n straight from
  // global memory (nobody else reads them), in flight together with the bulk copies.
  // (sFlux and sSJ are no bulk-copy destinations: the own Fv.n waits in the flux slots this
  // thread overwrites later, sJ goes straight to its place.)
  double own[KF][5], nrm[KF][3], vgn[KF];
  int typs[KF], rots[KF];
#pragma unroll
  for (int kf = 0; kf < KF; ++kf) {
    const int it = t + kf * N3;
    typs[kf] = 0;
    rots[kf] = 0;
    if (active && it < 6 * N2) {
      const int s = it / N2, f = it - s * N2;
      typs[kf] = P.side_type[e * 6 + s];
      if (ROT) rots[kf] = P.side_rot[e * 6 + s];
      const double* tr = P.trace + (static_cast<size_t>(e) * 6 * N2 + it) * 5;
#pragma unroll
      for (int v = 0; v < 5; ++v) own[kf][v] = __ldg(tr + v);
      if (VISC) {
        const double2* fp = reinterpret_cast<const double2*>(P.fvn + (static_cast<size_t>(e) * 6 * N2 + it) * 4);
        const double2 a0 = __ldg(fp), a1 = __ldg(fp + 1);
        sFlux[(s * 5 + 1) * N2 + f] = a0.x;
        sFlux[(s * 5 + 2) * N2 + f] = a0.y;
        sFlux[(s * 5 + 3) * N2 + f] = a1.x;
        sFlux[(s * 5 + 4) * N2 + f] = a1.y;
      }
      if constexpr (!AFF) {
        const double* fm = P.fmet + static_cast<size_t>(e) * D::FM + s * FW * N2 + f;  // [side][c][f]
        nrm[kf][0] = __ldg(fm);
        nrm[kf][1] = __ldg(fm + N2);
        nrm[kf][2] = __ldg(fm + 2 * N2);
        sSJ[it] = __ldg(fm + 3 * N2);
        if (ROT) vgn[kf] = __ldg(fm + 4 * N2);  // (vg / omega) . n; times the band's omega after the wait
      }
    }
  }
  load_tables<N1>(C, tab);
  __syncthreads();  // barrier init visible, tables loaded
  mbar_wait(bar, 0);
  const BandD& B = C.bands[band_ld];
  const Rot rot = band_rotation(ROT, A, band_ld);

  // Phase 1: numerical flux along each face node's normal -> sFlux, sJ -> sSJ.
  if (active) {
#pragma unroll
    for (int kf = 0; kf < KF; ++kf) {
      const int it = t + kf * N3;
      if (it >= 6 * N2) break;
      const int s = it / N2, f = it - s * N2, a = f / N1, b = f % N1;
      double* n = nrm[kf];
      const int dir = s >> 1;
      if constexpr (AFF) {
        vgn[kf] = dir == 1 ? B.vg : (dir == 2 ? B.vgz : 0.0);
      } else if (ROT) {
        rotate_yz(rot, n[1], n[2]);
        vgn[kf] *= B.vg;
      } else {
        vgn[kf] = B.vg * n[1];
      }
      const double* nb = sNb + s * D::NB;
      const int typ = typs[kf];
      double flux[5];
      bool ok = true;
      if (typ == kConforming) {
        double other[5];
#pragma unroll
        for (int v = 0; v < 5; ++v) other[v] = nb[f * 5 + v];
        double fvo[4];
        if (VISC) {  // [f][4]: two 128-bit loads (stride-4 64-bit loads collide 4-way)
          const double2* fq = reinterpret_cast<const double2*>(nb + D::TS + f * 4);
          const double2 f0 = fq[0], f1 = fq[1];
          fvo[0] = f0.x;
          fvo[1] = f0.y;
          fvo[2] = f1.x;
          fvo[3] = f1.y;
        }
        if constexpr (ROT) {  // periodic annulus sector seam: the neighbour's vectors in this sector's frame
          if (rots[kf] != 0) {
            const double sn = rots[kf] * C.sec_s;
            rot_yz(C.sec_c, sn, other[2], other[3]);
            if (VISC) rot_yz(C.sec_c, sn, fvo[1], fvo[2]);
          }
        }
        const double* um = (s & 1) ? own[kf] : other;
        const double* up = (s & 1) ? other : own[kf];
        if constexpr (AFF) ok = roe_flux(um, up, dir, vgn[kf], C.gas, flux);
        else ok = roe_flux_n(um, up, n, vgn[kf], C.gas, flux);
        if (VISC) {
          double ofv[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) ofv[c] = sFlux[(s * 5 + 1 + c) * N2 + f];
          const double* fm = (s & 1) ? ofv : fvo;
          const double* fp = (s & 1) ? fvo : ofv;
#pragma unroll
          for (int c = 0; c < 4; ++c) flux[1 + c] -= 0.5 * (fm[c] + fp[c]);
        }
      } else if (typ == kSliding) {
#pragma unroll
        for (int v = 0; v < 5; ++v) flux[v] = nb[f * 5 + v];
      } else {
        double ext[5];
        dirichlet_state<N1>(C, P.coords + 4 * e, s, a, b, A.t_stage, ext);
        const double* um = (s & 1) ? own[kf] : ext;
        const double* up = (s & 1) ? ext : own[kf];
        if constexpr (AFF) ok = roe_flux(um, up, dir, vgn[kf], C.gas, flux);
        else ok = roe_flux_n(um, up, n, vgn[kf], C.gas, flux);
        if (VISC) {
          const int idx = P.side_idx[e * 6 + s];
          const double* gd = P.dir_g + (static_cast<size_t>(idx) * N2 + f) * 12;
          double gg[12];
#pragma unroll
          for (int c = 0; c < 12; ++c) gg[c] = gd[c];
          double fm[4], fp[4];
          if constexpr (AFF) {
            fv_dir(um, gg, dir, C.gas, fm);
            fv_dir(up, gg, dir, C.gas, fp);
          } else {
            fv_n(um, gg, n, C.gas, fm);
            fv_n(up, gg, n, C.gas, fp);
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) flux[1 + c] -= 0.5 * (fm[c] + fp[c]);
        }
      }
      if (!ok) record_error(P.err, 2, A.step, A.stage, e, -1 - it, own[kf]);
#pragma unroll
      for (int v = 0; v < 5; ++v) sFlux[(s * 5 + v) * N2 + f] = flux[v];
    }
  }

  // Phase 2: pointwise flux (ALE convective minus viscous) -> contravariant Ja^d . F, staged
  // over this node's own metric / stress columns.
  double ij = 0.0;
  double ft2[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // third direction, staged in a second pass (PASSES == 2)
  if (active) {
    double u[5], F[3][5];
#pragma unroll
    for (int v = 0; v < 5; ++v) u[v] = sU[t * 5 + v];
    const double ir = rcp_nr(u[0]);
    const double vv[3] = {u[1] * ir, u[2] * ir, u[3] * ir};
    const double p = pressure(u, ir, C.gas);
    const double vgv[3] = {0.0, ROT ? 0.0 : B.vg, ROT ? 0.0 : B.vgz};  // annulus: grid velocity enters through V^d below
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      F[d][0] = u[0] * vv[d];
      F[d][1] = u[1] * vv[d] + (d == 0 ? p : 0.0);
      F[d][2] = u[2] * vv[d] + (d == 1 ? p : 0.0);
      F[d][3] = u[3] * vv[d] + (d == 2 ? p : 0.0);
      F[d][4] = (u[4] + p) * vv[d];
#pragma unroll
      for (int v = 0; v < 5; ++v) F[d][v] -= vgv[d] * u[v];
    }
    if (VISC) {
      const double* vs = sV + t;
      const double t00 = vs[0], t01 = vs[N3], t02 = vs[2 * N3], t11 = vs[3 * N3], t12 = vs[4 * N3], t22 = vs[5 * N3];
      const double tau[3][3] = {{t00, t01, t02}, {t01, t11, t12}, {t02, t12, t22}};
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        F[d][1] -= tau[d][0];
        F[d][2] -= tau[d][1];
        F[d][3] -= tau[d][2];
        F[d][4] -= tau[d][0] * vv[0] + tau[d][1] * vv[1] + tau[d][2] * vv[2] + vs[(6 + d) * N3];
      }
    }
    if (ROT && !AFF) {  // Ja(t) . F = Ja(0) . (R^T F)
#pragma unroll
      for (int v = 0; v < 5; ++v) rotate_yz(Rot{rot.c, -rot.s}, F[1][v], F[2][v]);
    }
    double Ft[3][5];
    if constexpr (AFF) {  // contravariant flux sJ_d F_d (volume_kernel, solver.cpp:357-370)
      ij = B.inv_jac;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
#pragma unroll
        for (int v = 0; v < 5; ++v) Ft[d][v] = F[d][v] * B.sj[d];
      }
    } else {
      const double* ja = sM + t;  // [c][node]
      ij = ja[9 * N3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double wv = ROT ? B.vg * ja[(10 + d) * N3] : 0.0;  // contravariant grid velocity
        const double j0 = ja[(3 * d) * N3], j1 = ja[(3 * d + 1) * N3], j2 = ja[(3 * d + 2) * N3];
#pragma unroll
        for (int v = 0; v < 5; ++v) Ft[d][v] = j0 * F[0][v] + j1 * F[1][v] + j2 * F[2][v] - wv * u[v];
      }
    }
    // Every read of this node's columns precedes these stores in program order.
#pragma unroll
    for (int d = 0; d < (D::PASSES == 1 ? 3 : 2); ++d) {
#pragma unroll
      for (int v = 0; v < 5; ++v) sF3[(d * 5 + v) * N3 + t] = Ft[d][v];
    }
    if constexpr (D::PASSES == 2) {
#pragma unroll
      for (int v = 0; v < 5; ++v) ft2[v] = Ft[2][v];
    }
  }
  // RK register of this thread's flat positions (L2-prefetched), in flight across the barrier.
  constexpr int KR = 5;
  double rv[KR];
  const size_t gbase = static_cast<size_t>(e0) * 5 * N3;
  if (A.mode == 0) {
#pragma unroll
    for (int q = 0; q < KR; ++q) {
      const int fI = threadIdx.x + q * THREADS;
      rv[q] = (A.rk_a != 0.0 && fI < n_el * 5 * N3) ? P.reg[gbase + fI] : 0.0;
    }
  }
  __syncthreads();

  // Phase 3: weak divergence sum_m Dhat(i,m) Ft_d(m) over the three directions;
  // Phase 4: surface lift with (sJ of the face node) / (J of the volume node).
  double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const double* dh = tab;
  const int nrot = node_rot<N1>(t);
  if (active) {
#pragma unroll
    for (int d = 0; d < (D::PASSES == 1 ? 3 : 2); ++d) {
      const int ia = d == 0 ? i : (d == 1 ? j : k);
      const int bse = d == 0 ? j * N1 + k : (d == 1 ? i * N2 + k : (i * N1 + j) * N1);
      const int stride = d == 0 ? N2 : (d == 1 ? N1 : 1);
      // Bank rotation (node_rot, 0 or 1) of the lines along i and j: nodes r, .., N1-1, then node 0 if r.
      const int r = d == 2 ? 0 : nrot;
      const int b0 = bse + r * stride, bl = bse + (r ? 0 : (N1 - 1) * stride);
      const double* dq = dh + ia * N1 + r;
      const double dl = dh[ia * N1 + (r ? 0 : N1 - 1)];
#pragma unroll
      for (int m = 0; m < N1; ++m) {
        const double c = d == 2 ? dhat_k<N1>(tab, ia, m) : (m < N1 - 1 ? dq[m] : dl);
        const int nd = m < N1 - 1 ? b0 + m * stride : bl;
#pragma unroll
        for (int v = 0; v < 5; ++v) acc[v] += c * sF3[(d * 5 + v) * N3 + nd];
      }
    }
  }
  if constexpr (D::PASSES == 2) {
    __syncthreads();  // the first two directions are consumed
    if (active) {
#pragma unroll
      for (int v = 0; v < 5; ++v) sF3[v * N3 + t] = ft2[v];
    }
    __syncthreads();
    if (active) {
      const int bse = (i * N1 + j) * N1;
#pragma unroll
      for (int m = 0; m < N1; ++m) {
        const double c = dhat_k<N1>(tab, k, m);
#pragma unroll
        for (int v = 0; v < 5; ++v) acc[v] += c * sF3[v * N3 + bse + m];
      }
    }
  }
  if (active) {
    double du[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) du[v] = acc[v] * ij;
    const double* lw = tab + N1 * N1 + 2 * N1;
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int dir = s >> 1;
      const int ia = dir == 0 ? i : (dir == 1 ? j : k);
      const int f = dir == 0 ? j * N1 + k : (dir == 1 ? i * N1 + k : i * N1 + j);
      const double l = lw[(s & 1) * N1 + ia];
      if (l != 0.0) {
        const double c = AFF ? ((s & 1) ? -1.0 : 1.0) * B.cdir[dir] * l : ((s & 1) ? -1.0 : 1.0) * l * sSJ[s * N2 + f] * ij;
#pragma unroll
        for (int v = 0; v < 5; ++v) du[v] += c * sFlux[(s * 5 + v) * N2 + f];
      }
    }
#pragma unroll
    for (int v = 0; v < 5; ++v) sD[t * 5 + v] = du[v];  // AoS, like the global state
  }
  __syncthreads();

  // Phase 5: flat coalesced RK update (solver.cpp:912-917) or residual store.
  if (A.mode == 1) {
    for (int fI = threadIdx.x; fI < n_el * 5 * N3; fI += THREADS) {
      const int l = fI / (5 * N3), r = fI - l * 5 * N3;
      P.out[gbase + fI] = base[l * PER + D::EL + D::MV + D::FX + D::SJ + r];
    }
    return;
  }
#pragma unroll
  for (int q = 0; q < KR; ++q) {
    const int fI = threadIdx.x + q * THREADS;
    if (fI < n_el * 5 * N3) {
      const int l = fI / (5 * N3), r = fI - l * 5 * N3;
      double* us = base + l * PER + r;
      const double dd = base[l * PER + D::EL + D::MV + D::FX + D::SJ + r];
      const double rg = A.rk_a * rv[q] + A.dt * dd;
      const double un = *us + A.rk_b * rg;
      P.reg[gbase + fI] = rg;
      P.U[gbase + fI] = un;
      *us = un;
    }
  }
  __syncthreads();
  // Admissibility (check_admissible, solver.cpp:892-906), then the traces of the
  // new state staged in the dead neighbour region [side][f][5] and bulk-stored.
  double* sOut = sNb;
  if (active) {
    double w[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) w[v] = sU[t * 5 + v];
    const double p = pressure(w, rcp_nr(w[0]), C.gas);
    bool ok = w[0] > 0.0 && p > 0.0;
#pragma unroll
    for (int v = 0; v < 5; ++v) ok = ok && isfinite(w[v]);
    if (!ok) record_error(P.err, 2, A.step, A.stage, e, t, w);
#pragma unroll
    for (int kf = 0; kf < KF; ++kf) {
      const int it = t + kf * N3;
      if (it >= 6 * N2) break;
      const int s = it / N2, f = it - s * N2, a = f / N1, b = f % N1;
      const double* ell = tab + N1 * N1 + (s & 1) * N1;
#pragma unroll
      for (int v = 0; v < 5; ++v) sOut[it * 5 + v] = prolong_aos<N1>(sU, v, ell, s >> 1, a, b, face_rot<N1>(s, a, b));
    }
    fence_proxy_async();
  }
  __syncthreads();
  if (active && t == 0) {
    bulk_s2g(P.trace_out + static_cast<size_t>(e) * 6 * D::TS, sOut, 6 * D::TS * 8u);
    bulk_commit();
    bulk_wait_read0();
  }
}

template <int N1>
bool update_affine_b_t(const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st) {
  if constexpr (N1 % 2 != 0) {
    return false;
  } else {
    if (c.gas.viscous && p.visc == nullptr) throw ProtocolError("k_update_cv needs the stress buffer of the gradient kernel");
    if (c.gas.viscous) {
      using D = CV<N1, false, true, true>;
      const int blocks = (p.E - p.e_first + D::EPB - 1) / D::EPB;
      set_smem_checked(k_update_cv<N1, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, D::SMEM);
      k_update_cv<N1, true, false, true><<<blocks, D::THREADS, D::SMEM, st>>>(c, p, a);
    } else {
      using D = CV<N1, false, false, true>;
      const int blocks = (p.E - p.e_first + D::EPB - 1) / D::EPB;
      set_smem_checked(k_update_cv<N1, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, D::SMEM);
      k_update_cv<N1, false, false, true><<<blocks, D::THREADS, D::SMEM, st>>>(c, p, a);
    }
    check_launch("k_update_cv (affine)");
    return true;
  }
}

template <int N1, bool ROT>
void gradient_curved_b_r(const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st) {
  using D = CG<N1, ROT>;
  const int blocks = (p.E - p.e_first + D::EPB - 1) / D::EPB;
  set_smem_checked(k_gradient_cv<N1, ROT>, cudaFuncAttributeMaxDynamicSharedMemorySize, D::SMEM);
  k_gradient_cv<N1, ROT><<<blocks, D::THREADS, D::SMEM, st>>>(c, p, a);
  check_launch("k_gradient_cv");
}
template <int N1>
bool gradient_curved_b_t(const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st) {
  if constexpr (N1 % 2 != 0) {
    return false;
  } else {
    if (c.mapping == SDG_MAP_ANNULUS) gradient_curved_b_r<N1, true>(c, p, a, st);
    else gradient_curved_b_r<N1, false>(c, p, a, st);
    return true;
  }
}
template <int N1, bool ROT>
void update_curved_b_r(const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st) {
  if (c.gas.viscous && p.visc == nullptr) throw ProtocolError("k_update_cv needs the stress buffer of the gradient kernel");
  if (c.gas.viscous) {
    using D = CV<N1, ROT, true>;
    const int blocks = (p.E - p.e_first + D::EPB - 1) / D::EPB;
    set_smem_checked(k_update_cv<N1, true, ROT>, cudaFuncAttributeMaxDynamicSharedMemorySize, D::SMEM);
    k_update_cv<N1, true, ROT><<<blocks, D::THREADS, D::SMEM, st>>>(c, p, a);
  } else {
    using D = CV<N1, ROT, false>;
    const int blocks = (p.E - p.e_first + D::EPB - 1) / D::EPB;
    set_smem_checked(k_update_cv<N1, false, ROT>, cudaFuncAttributeMaxDynamicSharedMemorySize, D::SMEM);
    k_update_cv<N1, false, ROT><<<blocks, D::THREADS, D::SMEM, st>>>(c, p, a);
  }
  check_launch("k_update_cv");
}
template <int N1>
bool update_curved_b_t(const ElemConsts& c, const FieldPtrs& p, const StageArgs& a, cudaStream_t st) {
  if constexpr (N1 % 2 != 0) {
    return false;
  } else {
    if (c.mapping == SDG_MAP_ANNULUS) update_curved_b_r<N1, true>(c, p, a, st);
    else update_curved_b_r<N1, false>(c, p, a, st);
    return true;
  }
}
