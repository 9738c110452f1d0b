// sb_device.cuh -- device-side geometry and the MAC stencil rows shared by
// every kernel (smoother colour passes, residual->restriction, apply_M).
//
// Layout: every array of a level (cells, the d face
// components, node/edge arrays) lives in ONE pitched box
//     [P0][P1][P2],  P_a = n_a + (axis a is a wall),  P2 rounded up to 4,
// so a point (i0,i1,i2) has the same linear index in all of them and stencil
// neighbours are fixed offsets.  2D grids use internal axes (1,2) with
// n0 = 1.  Entries outside an array's own extent (pads) are never written
// and stay 0, as do wall-normal boundary faces; reductions can therefore run
// over the whole box.
#pragma once
#include <cstdint>

namespace sb {

enum { BC_PER = 0, BC_NOSLIP = 1, BC_FREESLIP = 2 };
enum { F_LAP = 0, F_STRESS = 1, F_BULK = 2 };

struct LevelDev {
  int n[3];          // cells per internal axis (axis 0: this slab's planes when distributed)
  int dist0;         // axis 0 is slab-distributed: neighbours come from 2 ghost planes, no wrap
  int bclo[3], bchi[3];
  int s0, s1;        // strides of axes 0 and 1 (axis 2 is contiguous); boxes < 2^31 points
  int mue_derived;   // mu_e equals edge_mean(mu_c) to roundoff on this level (checked at setup)
  int beta_const;    // every non-wall 1/rho_face of the level equals beta_val (checked at setup)
  double beta_val;
  double h, inv_h, inv_h2, theta;
  const double* mu_c;
  const double* gam_c;
  const double* mu_e[3];   // edge array whose staggered pair excludes axis e
  const double* rho_f[3];
  const double* beta_f[3]; // 1/rho_face, 0 on wall boundary faces
};

__host__ __device__ __forceinline__ bool per(const LevelDev& L, int a) { return L.bclo[a] == BC_PER; }
// PA (compile-time boundary pattern): 1 = every axis of the level is periodic
// (wall logic compiled out), 0 = any boundary conditions (runtime checks),
// 2 + m = only the axes in bit mask m may be walls (PA_W2: walls along the
// contiguous axis 2 only -- C2's y and C4's z walls).
constexpr int PA_W2 = 2 + 4;
template <int PA>
__host__ __device__ __forceinline__ bool perq(const LevelDev& L, int a) {
  if (PA == 1) return true;
  if (PA >= 2 && !(((PA - 2) >> a) & 1)) return true;
  return L.bclo[a] == BC_PER;
}

template <int AX>
__device__ __forceinline__ int stride(const LevelDev& L) {
  return AX == 0 ? L.s0 : (AX == 1 ? L.s1 : 1);
}

// index shift to the +1 / -1 neighbour along AX of coordinate c (periodic wrap)
// periodic wrap along AX, except along a slab-distributed axis 0 (ghosts)
template <int AX, int PA = false>
__device__ __forceinline__ bool wraps(const LevelDev& L) {
  return perq<PA>(L, AX) && !(AX == 0 && L.dist0);
}
template <int AX, int PA = false>
__device__ __forceinline__ int dplus(const LevelDev& L, int c) {
  return (wraps<AX, PA>(L) && c == L.n[AX] - 1) ? -(L.n[AX] - 1) * stride<AX>(L) : stride<AX>(L);
}
template <int AX, int PA = false>
__device__ __forceinline__ int dminus(const LevelDev& L, int c) {
  return (wraps<AX, PA>(L) && c == 0) ? (L.n[AX] - 1) * stride<AX>(L) : -stride<AX>(L);
}

// Programmatic dependent launch: the solve's kernels are
// launched with programmatic stream serialization (launch_k, sb_kernels.h),
// so a kernel's CTAs are scheduled while its predecessor drains.
// griddepcontrol.wait holds them until the predecessor grid has completed and
// its writes are visible; it must be the first, unconditional statement of
// every kernel so the ordering stays transitive.  Then the kernel lets its
// own dependent launch early.  Both are no-ops for ordinary launches.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ double ld(const double* p, int i) { return __ldg(p + i); }

__host__ __device__ constexpr int edge_of(int a, int b) { return 3 - a - b; }

// Edge (3D) / node (2D) viscosity as the mean of the four cells around it,
// averaged first along the lower axis of the edge plane, then the higher
// (operators.py:90-104 average_cell_to_node_edge, :133-145 _avg_to_stagger,
// periodic branch).  dlo / dhi: index offsets of the -1 neighbour along the
// lower / higher axis (wraps applied).
__device__ __forceinline__ double edge_mean(const double* mu, int i, int dlo, int dhi) {
  const double a = 0.5 * (__ldg(mu + i) + __ldg(mu + i + dlo));
  const double b = 0.5 * (__ldg(mu + i + dhi) + __ldg(mu + i + dlo + dhi));
  return 0.5 * (a + b);
}

// (D u)(c) * h accumulated in axis order: ((d0 + d1) + d2)  (operators.py:182-188)
template <int DIM, int PA = false>
__device__ __forceinline__ double div_sum(const LevelDev& L, const double* const* u, int c,
                                          const int* ci) {
  double acc = 0.0;
  bool first = true;
#pragma unroll
  for (int b = 3 - DIM; b < 3; ++b) {
    int dp = (b == 0) ? dplus<0, PA>(L, ci[0]) : (b == 1 ? dplus<1, PA>(L, ci[1]) : dplus<2, PA>(L, ci[2]));
    // on a wall axis the high face of cell c is c+1 (<= n), never wrapped
    double d = u[b][c + dp] - u[b][c];
    acc = first ? d : acc + d;
    first = false;
  }
  return acc;
}

// The 7-point u_A neighbourhood of a face: centre and +/- neighbour along each
// axis (periodic wraps already applied).  Gathered from global memory
// (gather_ua) or from a shared-memory tile (the fused sweep kernels).
struct UA7 {
  double c, p[3], m[3];
};

// CG: load through L2 only (ld.global.cg).  The wavefront sweep kernels
// (sb_wave.cu) read iterate values that other SMs wrote earlier in the same
// launch; L1 is not coherent across SMs, so those loads bypass it.
template <bool CG>
__device__ __forceinline__ double ldu(const double* p, int i) { return CG ? __ldcg(p + i) : p[i]; }

template <int DIM, int A, int PA = false, bool CG = false>
__device__ __forceinline__ UA7 gather_ua(const LevelDev& L, const double* ua, int f, const int* ci) {
  UA7 s;
  s.c = ldu<CG>(ua, f);
#pragma unroll
  for (int b = 3 - DIM; b < 3; ++b) {
    const int dp = b == 0 ? dplus<0, PA>(L, ci[0]) : (b == 1 ? dplus<1, PA>(L, ci[1]) : dplus<2, PA>(L, ci[2]));
    const int dm = b == 0 ? dminus<0, PA>(L, ci[0]) : (b == 1 ? dminus<1, PA>(L, ci[1]) : dminus<2, PA>(L, ci[2]));
    // on a wall axis B != A the +/- neighbours are only read away from the wall
    const bool wallB = b != A && !perq<PA>(L, b);
    s.p[b] = (wallB && ci[b] == L.n[b] - 1) ? 0.0 : ldu<CG>(ua, f + dp);
    s.m[b] = (wallB && ci[b] == 0) ? 0.0 : ldu<CG>(ua, f + dm);
  }
  return s;
}

// Operand accessors for the face row.  Every array a face row reads, at the
// offsets it reads them: mu_c at f and f-e_A, mu_e(A,B) at f and f+e_B, u_B at
// (f | f+e_B) (- e_A), rho_A and rhs at f, plus the u_A neighbourhood.
// GAcc gathers from global memory with periodic wraps; the streaming sweep
// kernels (sb_sweep.cu) provide a shared-memory accessor with the same API.
// NC: the u_B operands go through the read-only (non-coherent) path.  The
// single-CTA coarse-level kernel updates u inside the launch and reads it
// back after __syncthreads, so it instantiates NC = false (plain loads).
// DE: the edge viscosities are derived from mu_c (edge_mean; on a wall the
// two-cell boundary mean) instead of read from the mu_e arrays -- only on
// levels whose mu_e matched that derivation at setup (LevelDev::mue_derived,
// k_check_mue); mu_c's neighbours come from L1/L2, so the face row streams
// one coefficient array instead of three.
// ZM: bit B set = component B is known to be identically zero (the first
// sweep of a V-cycle level starts from x = 0, multigrid.py:409-439), so its
// loads are replaced by the value they would return.
template <int DIM, int A, int PA = false, bool NC = true, bool DE = false, int ZM = 0>
struct GAcc {
  const LevelDev& L;
  const double* const* u;
  int f;
  const int* ci;
  int dmA;
  double mf, mfa;      // DE: mu_c at f, f - e_A (loaded once)
  double me[3][2];     // DE: derived edge viscosities [B][hi edge]
  __device__ __forceinline__ GAcc(const LevelDev& L_, const double* const* u_, int f_, const int* ci_)
      : L(L_), u(u_), f(f_), ci(ci_) {
    dmA = (A == 0) ? dminus<0, PA>(L, ci[0]) : (A == 1 ? dminus<1, PA>(L, ci[1]) : dminus<2, PA>(L, ci[2]));
    if (DE) {
      // every mu_c operand of the row loaded once: f, f-e_A, f-+e_B, f-+e_B-e_A
      mf = ld(L.mu_c, f);
      mfa = ld(L.mu_c, f + dmA);
      const double mA = 0.5 * (mf + mfa);  // lower-axis-first mean along A (both orders start so)
#pragma unroll
      for (int B = 3 - DIM; B < 3; ++B) {
        if (B == A) continue;
        const int pB = B == 0 ? dplus<0, PA>(L, ci[0]) : (B == 1 ? dplus<1, PA>(L, ci[1]) : dplus<2, PA>(L, ci[2]));
        const int mB = B == 0 ? dminus<0, PA>(L, ci[0]) : (B == 1 ? dminus<1, PA>(L, ci[1]) : dminus<2, PA>(L, ci[2]));
        // wall along B: the boundary edge (jj = 0 / n_B) is the mean of the two
        // cells on its side -- _avg_to_stagger copies the boundary cell, so both
        // averaging orders reduce to 0.5 (mu_c(f) + mu_c(f - e_A))
        const bool wB = !perq<PA>(L, B);
        const bool wlo = wB && ci[B] == 0, whi = wB && ci[B] == L.n[B] - 1;
        if (wlo) {
          me[B][0] = mA;
        } else {
          const double fbm = ld(L.mu_c, f + mB), fbma = ld(L.mu_c, f + mB + dmA);
          // edge_mean order: lower plane axis first (see edge_mean)
          me[B][0] = A < B ? 0.5 * (mA + 0.5 * (fbm + fbma)) : 0.5 * (0.5 * (mf + fbm) + 0.5 * (mfa + fbma));
        }
        if (whi) {
          me[B][1] = mA;
        } else {
          const double fbp = ld(L.mu_c, f + pB), fbpa = ld(L.mu_c, f + pB + dmA);
          me[B][1] = A < B ? 0.5 * (0.5 * (fbp + fbpa) + mA) : 0.5 * (0.5 * (fbp + mf) + 0.5 * (fbpa + mfa));
        }
      }
    }
  }
  template <int B>
  __device__ __forceinline__ int eB() const {
    return B == 0 ? dplus<0, PA>(L, ci[0]) : (B == 1 ? dplus<1, PA>(L, ci[1]) : dplus<2, PA>(L, ci[2]));
  }
  __device__ __forceinline__ double mu(bool lo) const {
    if (DE) return lo ? mfa : mf;
    return ld(L.mu_c, lo ? f + dmA : f);
  }
  __device__ __forceinline__ double gam(bool lo) const { return ld(L.gam_c, lo ? f + dmA : f); }
  template <int B>
  __device__ __forceinline__ double mue(bool hi) const {
    if (!DE) return ld(L.mu_e[edge_of(A, B)], hi ? f + eB<B>() : f);
    return me[B][hi ? 1 : 0];
  }
  template <int B>
  __device__ __forceinline__ double ub(bool hi, bool lowA) const {
    if (ZM & (1 << B)) return 0.0;
    const int e = hi ? f + eB<B>() : f;
    return NC ? ld(u[B], lowA ? e + dmA : e) : u[B][lowA ? e + dmA : e];
  }
  __device__ __forceinline__ double rho() const { return ld(L.rho_f[A], f); }
  // (D u) h at the cells c_hi = f / c_lo = f - e_A (stress+bulk form only)
  __device__ __forceinline__ double divh(bool lo) const {
    if (!lo) return div_sum<DIM, PA>(L, u, f, ci);
    int clo[3] = {ci[0], ci[1], ci[2]};
    clo[A] = (perq<PA>(L, A) && ci[A] == 0 && !(A == 0 && L.dist0)) ? L.n[A] - 1 : ci[A] - 1;
    return div_sum<DIM, PA>(L, u, f + dmA, clo);
  }
};

// One tangential flux of row A across the edge at B-position jj (lo edge
// jj = cB, hi edge jj = cB+1) and the matching diagonal weight
// (operators.py:267-300, 331-340; diag :424-434).  u_hi/u_lo are u_A on the
// two sides of the edge along B.
template <int FORM, int A, int B, int PA, class ACC>
__device__ __forceinline__ void tang_flux(const LevelDev& L, const ACC& acc, int cB, bool hi_edge, double u_hi,
                                          double u_lo, double& flux, double& w) {
  const int nB = L.n[B];
  const bool pB = perq<PA>(L, B);
  const int jj = hi_edge ? cB + 1 : cB;
  const double mue = acc.template mue<B>(hi_edge);
  double tang;
  int side = -1;  // 0: low wall, 1: high wall
  if (!pB && jj == 0) {
    side = 0;
    tang = 2.0 * (u_hi - 0.0) * L.inv_h;
  } else if (!pB && jj == nB) {
    side = 1;
    tang = 2.0 * (0.0 - u_lo) * L.inv_h;
  } else {
    tang = (u_hi - u_lo) * L.inv_h;
  }
  double ft = tang;
  if (FORM != F_LAP) {
    const double cross = (acc.template ub<B>(hi_edge, false) - acc.template ub<B>(hi_edge, true)) * L.inv_h;
    ft = tang + cross;
  }
  ft = mue * ft;
  w = mue;
  if (side >= 0) {  // only reachable on a wall axis
    const int kind = side == 0 ? L.bclo[B] : L.bchi[B];
    if (kind == BC_FREESLIP) {
      ft = 0.0;
      w = 0.0;
    } else {
      w = mue * 2.0;
    }
  }
  flux = ft;
}

// (A u)_A at unknown face f (coords ci) from the u_A neighbourhood s and the
// accessor, plus the smoother diagonal of that row.
// operators.py:303-360 (row form multigrid.py:343-383), diag operators.py:408-439.
template <int DIM, int FORM, int A, int PA, class ACC>
__device__ __forceinline__ double face_row_t(const LevelDev& L, const UA7& s, const ACC& acc, const int* ci,
                                             double& diag) {
  const double uf = s.c, up = s.p[A], um = s.m[A];
  const double mu_hi = acc.mu(false), mu_lo = acc.mu(true);
  const double nc_hi = FORM == F_LAP ? mu_hi : 2.0 * mu_hi;
  const double nc_lo = FORM == F_LAP ? mu_lo : 2.0 * mu_lo;
  double fn_hi = nc_hi * (up - uf) * L.inv_h;
  double fn_lo = nc_lo * (uf - um) * L.inv_h;
  double ncd_hi = nc_hi, ncd_lo = nc_lo;
  if (FORM == F_BULK) {
    const double bk_hi = acc.gam(false) - (2.0 / 3.0) * mu_hi;
    const double bk_lo = acc.gam(true) - (2.0 / 3.0) * mu_lo;
    fn_hi = fn_hi + bk_hi * (acc.divh(false) * L.inv_h);
    fn_lo = fn_lo + bk_lo * (acc.divh(true) * L.inv_h);
    ncd_hi = nc_hi + bk_hi;
    ncd_lo = nc_lo + bk_lo;
  }
  double res = (fn_hi - fn_lo) * L.inv_h;
  double dg = L.theta == 0.0 ? 0.0 : L.theta * acc.rho();
  dg = dg + (ncd_hi + ncd_lo) * L.inv_h2;
#pragma unroll
  for (int B = 3 - DIM; B < 3; ++B) {
    if (B == A) continue;
    double f_lo, f_hi, w_lo, w_hi;
    const int cB = ci[B];
    if (B == 0) {
      tang_flux<FORM, A, 0, PA>(L, acc, cB, false, uf, s.m[0], f_lo, w_lo);
      tang_flux<FORM, A, 0, PA>(L, acc, cB, true, s.p[0], uf, f_hi, w_hi);
    } else if (B == 1) {
      tang_flux<FORM, A, 1, PA>(L, acc, cB, false, uf, s.m[1], f_lo, w_lo);
      tang_flux<FORM, A, 1, PA>(L, acc, cB, true, s.p[1], uf, f_hi, w_hi);
    } else {
      tang_flux<FORM, A, 2, PA>(L, acc, cB, false, uf, s.m[2], f_lo, w_lo);
      tang_flux<FORM, A, 2, PA>(L, acc, cB, true, s.p[2], uf, f_hi, w_hi);
    }
    res = res + (f_hi - f_lo) * L.inv_h;
    dg = dg + (w_lo + w_hi) * L.inv_h2;
  }
  diag = dg;
  const double tr = L.theta == 0.0 ? 0.0 : (L.theta * acc.rho()) * uf;
  return tr - res;
}

template <int DIM, int FORM, int A, int PA = false, bool NC = true, bool DE = false, int ZM = 0>
__device__ __forceinline__ double face_row_core(const LevelDev& L, const UA7& s, const double* const* u, int f,
                                                const int* ci, double& diag) {
  return face_row_t<DIM, FORM, A, PA>(L, s, GAcc<DIM, A, PA, NC, DE, ZM>(L, u, f, ci), ci, diag);
}

template <int DIM, int FORM, int A, int PA = false, bool NC = true, bool CG = false, bool DE = false>
__device__ __forceinline__ double face_row(const LevelDev& L, const double* const* u, int f, const int* ci,
                                           double& diag) {
  return face_row_core<DIM, FORM, A, PA, NC, DE>(L, gather_ua<DIM, A, PA, CG>(L, u[A], f, ci), u, f, ci, diag);
}

// beta = 1/rho_face accessor for the cell row: beta_a at the low face (c) or
// the high face (c + e_a, wrapped) of cell c.
template <int PA = false>
struct GBeta {
  const LevelDev& L;
  int c;
  const int* ci;
  __device__ __forceinline__ GBeta(const LevelDev& L_, int c_, const int* ci_) : L(L_), c(c_), ci(ci_) {}
  template <int AX>
  __device__ __forceinline__ double beta(bool hi) const {
    // constant density (LevelDev::beta_const): the level's single 1/rho_face
    // value, 0 on wall faces like the stored array -- no beta stream at all
    if (L.beta_const) {
      const bool wall = !perq<PA>(L, AX) && (hi ? ci[AX] == L.n[AX] - 1 : ci[AX] == 0);
      return wall ? 0.0 : L.beta_val;
    }
    return ld(L.beta_f[AX], hi ? c + dplus<AX, PA>(L, ci[AX]) : c);
  }
};

// (L_rho phi)(c) and its diagonal from the 7-point phi neighbourhood s
// (operators.py:206-215, 396-405).
template <int DIM, int PA, class BA>
__device__ __forceinline__ double cell_row_t(const LevelDev& L, const UA7& s, const BA& ba, const int* ci,
                                             double& diag) {
  const double pc = s.c;
  double acc = 0.0, dacc = 0.0;
  bool first = true;
#pragma unroll
  for (int a = 3 - DIM; a < 3; ++a) {
    const int n = L.n[a];
    const bool p = perq<PA>(L, a);
    double b_lo, b_hi;
    if (a == 0) {
      b_lo = ba.template beta<0>(false);
      b_hi = ba.template beta<0>(true);
    } else if (a == 1) {
      b_lo = ba.template beta<1>(false);
      b_hi = ba.template beta<1>(true);
    } else {
      b_lo = ba.template beta<2>(false);
      b_hi = ba.template beta<2>(true);
    }
    double g_lo = 0.0, g_hi = 0.0;
    if (p || ci[a] > 0) g_lo = ((pc - s.m[a]) * L.inv_h) * b_lo;
    if (p || ci[a] < n - 1) g_hi = ((s.p[a] - pc) * L.inv_h) * b_hi;
    const double d = g_hi - g_lo;
    acc = first ? d : acc + d;
    dacc = dacc - (b_lo + b_hi);
    first = false;
  }
  diag = dacc * L.inv_h2;
  return acc * L.inv_h;
}

template <int DIM, int PA = false>
__device__ __forceinline__ double cell_row_core(const LevelDev& L, const UA7& s, int c, const int* ci,
                                                double& diag) {
  return cell_row_t<DIM, PA>(L, s, GBeta<PA>(L, c, ci), ci, diag);
}

template <int DIM, int PA = false, bool CG = false>
__device__ __forceinline__ UA7 gather_cell(const LevelDev& L, const double* phi, int c, const int* ci) {
  UA7 s;
  s.c = ldu<CG>(phi, c);
#pragma unroll
  for (int a = 3 - DIM; a < 3; ++a) {
    const int dp = a == 0 ? dplus<0, PA>(L, ci[0]) : (a == 1 ? dplus<1, PA>(L, ci[1]) : dplus<2, PA>(L, ci[2]));
    const int dm = a == 0 ? dminus<0, PA>(L, ci[0]) : (a == 1 ? dminus<1, PA>(L, ci[1]) : dminus<2, PA>(L, ci[2]));
    const bool wall = !perq<PA>(L, a);
    s.p[a] = (wall && ci[a] == L.n[a] - 1) ? 0.0 : ldu<CG>(phi, c + dp);
    s.m[a] = (wall && ci[a] == 0) ? 0.0 : ldu<CG>(phi, c + dm);
  }
  return s;
}

template <int DIM, int PA = false, bool CG = false>
__device__ __forceinline__ double cell_row(const LevelDev& L, const double* phi, int c, const int* ci,
                                           double& diag) {
  return cell_row_core<DIM, PA>(L, gather_cell<DIM, PA, CG>(L, phi, c, ci), c, ci, diag);
}

}  // namespace sb
