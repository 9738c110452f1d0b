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
  int n[3];          // cells per internal axis
  int bclo[3], bchi[3];
  long long s0, s1;  // strides of axes 0 and 1 (axis 2 is contiguous)
  double h, inv_h, inv_h2, theta;
  const double* mu_c;
  const double* gam_c;
  const double* mu_e[3];   // edge array whose staggered pair excludes axis e
  const double* rho_f[3];
  const double* beta_f[3]; // 1/rho_face, 0 on wall boundary faces
};

__host__ __device__ __forceinline__ bool per(const LevelDev& L, int a) { return L.bclo[a] == BC_PER; }

template <int AX>
__device__ __forceinline__ long long stride(const LevelDev& L) {
  return AX == 0 ? L.s0 : (AX == 1 ? L.s1 : 1LL);
}

// index shift to the +1 / -1 neighbour along AX of coordinate c (periodic wrap)
template <int AX>
__device__ __forceinline__ long long dplus(const LevelDev& L, int c) {
  return (L.bclo[AX] == BC_PER && c == L.n[AX] - 1) ? -(long long)(L.n[AX] - 1) * stride<AX>(L)
                                                     : stride<AX>(L);
}
template <int AX>
__device__ __forceinline__ long long dminus(const LevelDev& L, int c) {
  return (L.bclo[AX] == BC_PER && c == 0) ? (long long)(L.n[AX] - 1) * stride<AX>(L)
                                           : -stride<AX>(L);
}

__device__ __forceinline__ double ld(const double* p, long long i) { return __ldg(p + i); }

__host__ __device__ constexpr int edge_of(int a, int b) { return 3 - a - b; }

// (D u)(c) * h accumulated in axis order: ((d0 + d1) + d2)  (operators.py:182-188)
template <int DIM>
__device__ __forceinline__ double div_sum(const LevelDev& L, const double* const* u, long long c,
                                          const int* ci) {
  double acc = 0.0;
  bool first = true;
#pragma unroll
  for (int b = 3 - DIM; b < 3; ++b) {
    long long dp = (b == 0) ? dplus<0>(L, ci[0]) : (b == 1 ? dplus<1>(L, ci[1]) : dplus<2>(L, ci[2]));
    // on a wall axis the high face of cell c is c+1 (<= n), never wrapped
    double d = u[b][c + dp] - u[b][c];
    acc = first ? d : acc + d;
    first = false;
  }
  return acc;
}

// One tangential flux of row A across the edge at B-position jj, and the
// matching diagonal weight w (operators.py:267-300, 331-340; diag :424-434).
// f is the face index, cA/cB its coordinates, am_d the index shift to the
// A-neighbour cell below (wrapped).
template <int FORM, int A, int B>
__device__ __forceinline__ void tang_flux(const LevelDev& L, const double* const* u, long long f,
                                          int cB, int jj, long long am_d, double& flux, double& w) {
  const long long sB = stride<B>(L);
  const int nB = L.n[B];
  const bool pB = per(L, B);
  // edge index: same point with B-coordinate jj (wrapped jj==nB -> 0 on periodic axes)
  int jw = (pB && jj == nB) ? 0 : jj;
  long long e = f + (long long)(jw - cB) * sB;
  double mue = ld(L.mu_e[edge_of(A, B)], e);
  double tang;
  int side = -1;  // 0: low wall, 1: high wall
  if (!pB && jj == 0) {
    side = 0;
    tang = 2.0 * (u[A][e] - 0.0) * L.inv_h;
  } else if (!pB && jj == nB) {
    side = 1;
    tang = 2.0 * (0.0 - u[A][e - sB]) * L.inv_h;
  } else {
    long long em = (pB && jw == 0) ? e + (long long)(nB - 1) * sB : e - sB;
    tang = (u[A][e] - u[A][em]) * L.inv_h;
  }
  double ft = tang;
  if (FORM != F_LAP) {
    double cross = (u[B][e] - u[B][e + am_d]) * L.inv_h;
    ft = tang + cross;
  }
  ft = mue * ft;
  w = mue;
  if (side >= 0) {
    int kind = side == 0 ? L.bclo[B] : L.bchi[B];
    if (kind == BC_FREESLIP) {
      ft = 0.0;
      w = 0.0;
    } else {
      w = mue * 2.0;
    }
  }
  flux = ft;
}

// (A u)_A at unknown face f (coords ci) and the smoother diagonal of that row.
// operators.py:303-360 (row form multigrid.py:343-383), diag operators.py:408-439.
template <int DIM, int FORM, int A>
__device__ __forceinline__ double face_row(const LevelDev& L, const double* const* u, long long f,
                                           const int* ci, double& diag) {
  const long long dpA = (A == 0) ? dplus<0>(L, ci[0]) : (A == 1 ? dplus<1>(L, ci[1]) : dplus<2>(L, ci[2]));
  const long long dmA = (A == 0) ? dminus<0>(L, ci[0]) : (A == 1 ? dminus<1>(L, ci[1]) : dminus<2>(L, ci[2]));
  const double uf = u[A][f];
  const double up = u[A][f + dpA];
  const double um = u[A][f + dmA];
  // cells c_hi = f, c_lo = f + dmA share the face's index (uniform strides)
  const double mu_hi = ld(L.mu_c, f), mu_lo = ld(L.mu_c, f + dmA);
  double nc_hi = FORM == F_LAP ? mu_hi : 2.0 * mu_hi;
  double nc_lo = FORM == F_LAP ? mu_lo : 2.0 * mu_lo;
  double fn_hi = nc_hi * (up - uf) * L.inv_h;
  double fn_lo = nc_lo * (uf - um) * L.inv_h;
  double ncd_hi = nc_hi, ncd_lo = nc_lo;
  if (FORM == F_BULK) {
    const double g_hi = ld(L.gam_c, f), g_lo = ld(L.gam_c, f + dmA);
    const double bk_hi = g_hi - (2.0 / 3.0) * mu_hi;
    const double bk_lo = g_lo - (2.0 / 3.0) * mu_lo;
    int clo[3] = {ci[0], ci[1], ci[2]};
    clo[A] = (per(L, A) && ci[A] == 0) ? L.n[A] - 1 : ci[A] - 1;
    fn_hi = fn_hi + bk_hi * (div_sum<DIM>(L, u, f, ci) * L.inv_h);
    fn_lo = fn_lo + bk_lo * (div_sum<DIM>(L, u, f + dmA, clo) * L.inv_h);
    ncd_hi = nc_hi + bk_hi;
    ncd_lo = nc_lo + bk_lo;
  }
  double res = (fn_hi - fn_lo) * L.inv_h;
  double dg = L.theta == 0.0 ? 0.0 : L.theta * ld(L.rho_f[A], f);
  dg = dg + (ncd_hi + ncd_lo) * L.inv_h2;
#pragma unroll
  for (int B = 3 - DIM; B < 3; ++B) {
    if (B == A) continue;
    double f_lo, f_hi, w_lo, w_hi;
    const int cB = ci[B];
    if (B == 0) {
      tang_flux<FORM, A, 0>(L, u, f, cB, cB, dmA, f_lo, w_lo);
      tang_flux<FORM, A, 0>(L, u, f, cB, cB + 1, dmA, f_hi, w_hi);
    } else if (B == 1) {
      tang_flux<FORM, A, 1>(L, u, f, cB, cB, dmA, f_lo, w_lo);
      tang_flux<FORM, A, 1>(L, u, f, cB, cB + 1, dmA, f_hi, w_hi);
    } else {
      tang_flux<FORM, A, 2>(L, u, f, cB, cB, dmA, f_lo, w_lo);
      tang_flux<FORM, A, 2>(L, u, f, cB, cB + 1, dmA, f_hi, w_hi);
    }
    res = res + (f_hi - f_lo) * L.inv_h;
    dg = dg + (w_lo + w_hi) * L.inv_h2;
  }
  diag = dg;
  double tr = L.theta == 0.0 ? 0.0 : (L.theta * ld(L.rho_f[A], f)) * uf;
  return tr - res;
}

// (L_rho phi)(c) and its diagonal (operators.py:206-215, 396-405).
template <int DIM>
__device__ __forceinline__ double cell_row(const LevelDev& L, const double* phi, long long c,
                                           const int* ci, double& diag) {
  const double pc = phi[c];
  double acc = 0.0, dacc = 0.0;
  bool first = true;
#pragma unroll
  for (int a = 3 - DIM; a < 3; ++a) {
    const long long s = a == 0 ? L.s0 : (a == 1 ? L.s1 : 1LL);
    const int n = L.n[a];
    const bool p = per(L, a);
    const double* beta = L.beta_f[a];
    // low face of c is c (index c); high face c+1 (wrapped)
    double g_lo = 0.0, g_hi = 0.0;
    const long long lo_nb = (p && ci[a] == 0) ? (long long)(n - 1) * s : -s;  // cell below
    const long long hi_f = (p && ci[a] == n - 1) ? -(long long)(n - 1) * s : s; // face above / cell above
    const double b_lo = ld(beta, c);
    const double b_hi = ld(beta, c + hi_f);
    if (p || ci[a] > 0) g_lo = ((pc - phi[c + lo_nb]) * L.inv_h) * b_lo;
    if (p || ci[a] < n - 1) g_hi = ((phi[c + hi_f] - pc) * L.inv_h) * b_hi;
    double d = g_hi - g_lo;
    acc = first ? d : acc + d;
    dacc = dacc - (b_lo + b_hi);
    first = false;
  }
  diag = dacc * L.inv_h2;
  return acc * L.inv_h;
}

}  // namespace sb
