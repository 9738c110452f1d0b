// sb_rowv.cu -- row kernels for large 3D levels (sm_100a): the face residual
// field of the split residual -> restriction and apply_M (default), and the
// face colour passes (opt-in).
//
// The one-face-per-thread kernels (sb_kernels.cu) issue one load per stencil
// operand; a colour pass reads every other face of a row, so each warp-wide
// load touches four 128-B lines for 256 useful bytes, and the all-face
// kernels evaluate three face rows per thread from ~70 separate loads.
//
// Two generations live here:
//  * k_face_all_rm (default, "row-march"): a warp walks one whole row in
//    32-face segments, -1 neighbours carried between segments, every edge /
//    normal stress evaluated once and shared by the two rows that use it,
//    FMAs on the final combinations; all-periodic levels and levels with walls
//    along the contiguous axis (C4).  ncu C5 256^3: apply_M 273 us, residual
//    field 263 us (0.91 / 1.03 of the measured HBM peak by the byte model).  Equal to the
//    per-face kernels to ~1e-15 relative (different rounding order).
//  * k_face_all_rv / k_face_colour_rv ("segment" kernels, SB_ROWM=0 /
//    SB_ROWV_COLOUR=1): a warp owns a 32- or 64-face row segment and every
//    operand ROW is read once, contiguously; the +-1 neighbours along the
//    contiguous axis come from the neighbouring lane (__shfl), the segment
//    ends from one uniform-address load.  Same arithmetic as face_row_t on
//    the same operands: bit-identical to the per-face kernels
//    (tests/test_gpu_rowv.py).  Measured (ncu, C5 256^3): residual field
//    465 -> 413 us, apply_M 533 -> 510 us against the per-face kernels; the
//    colour pass is NOT faster than the per-face kernel with derived edge
//    viscosities (173-195 vs 155-164 us: 74-80 registers, latency bound).
//
// Scope: 3D, axes 0 and 1 periodic (a slab-distributed axis 0 reads ghost
// planes), LAPLACIAN / STRESS forms, contiguous extent a multiple of 64
// (rowv_supported); walls along the contiguous axis only in the row-march
// kernel.
#include <cuda_runtime.h>
#include <cstdlib>
#include "sb_kernels.h"

namespace sb {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int RT = 256;  // threads per CTA
#ifndef RV_MINB
#define RV_MINB 3
#endif
#ifndef RM_MINB
#define RM_MINB 2
#endif

// ---- compile-time operand masks -------------------------------------------
// A stencil operand at offset (o0, o1, o2) from the thread's face lives in
// row r = (o0+1)*3 + (o1+1) of the 3x3 row neighbourhood (axes 0, 1), at
// contiguous offset o2 in {-1, 0, +1}: bit r of Need.m / .c / .p.
struct Need {
  unsigned m, c, p;
};
__host__ __device__ constexpr int rix(int o0, int o1) { return (o0 + 1) * 3 + (o1 + 1); }
__host__ __device__ constexpr Need add(Need n, int o0, int o1, int o2) {
  const unsigned b = 1u << rix(o0, o1);
  if (o2 < 0) n.m |= b;
  else if (o2 > 0) n.p |= b;
  else n.c |= b;
  return n;
}
__host__ __device__ constexpr Need orn(Need a, Need b) { return Need{a.m | b.m, a.c | b.c, a.p | b.p}; }
__host__ __device__ constexpr int e(int axis, int a) { return axis == a ? 1 : 0; }
// f + sa e_A + sb e_B
__host__ __device__ constexpr Need add2(Need n, int A, int sa, int B, int sb) {
  return add(n, sa * e(0, A) + sb * e(0, B), sa * e(1, A) + sb * e(1, B), sa * e(2, A) + sb * e(2, B));
}
__host__ __device__ constexpr int oth1(int A) { return A == 0 ? 1 : 0; }
__host__ __device__ constexpr int oth2(int A) { return A == 2 ? 1 : 2; }

// u_A neighbourhood (UA7)
__host__ __device__ constexpr Need need_ua(int A) {
  Need n{0, 0, 0};
  (void)A;
  n = add(n, 0, 0, 0);
  n = add(n, 1, 0, 0);
  n = add(n, -1, 0, 0);
  n = add(n, 0, 1, 0);
  n = add(n, 0, -1, 0);
  n = add(n, 0, 0, 1);
  n = add(n, 0, 0, -1);
  return n;
}
// mu_c: f, f - e_A; derived edges add f -+ e_B, f -+ e_B - e_A per tangent B
__host__ __device__ constexpr Need need_mu(int A, bool DE) {
  Need n{0, 0, 0};
  n = add2(n, A, 0, A, 0);
  n = add2(n, A, -1, A, 0);
  if (DE) {
    for (int k = 0; k < 2; ++k) {
      const int B = k == 0 ? oth1(A) : oth2(A);
      n = add2(n, A, 0, B, -1);
      n = add2(n, A, -1, B, -1);
      n = add2(n, A, 0, B, 1);
      n = add2(n, A, -1, B, 1);
    }
  }
  return n;
}
// stored edge viscosity mu_e(A,B): f and f + e_B
__host__ __device__ constexpr Need need_mue(int A, int B) {
  Need n{0, 0, 0};
  n = add2(n, A, 0, B, 0);
  n = add2(n, A, 0, B, 1);
  return n;
}
// u_B cross terms of row A: f, f - e_A, f + e_B, f + e_B - e_A
__host__ __device__ constexpr Need need_ub(int A, int B) {
  Need n{0, 0, 0};
  n = add2(n, A, 0, B, 0);
  n = add2(n, A, -1, B, 0);
  n = add2(n, A, 0, B, 1);
  n = add2(n, A, -1, B, 1);
  return n;
}
// what the face row of component A needs from u_X (X = 0, 1, 2)
__host__ __device__ constexpr Need need_u(int A, int X, int FORM) {
  if (X == A) return need_ua(A);
  return FORM == F_LAP ? Need{0, 0, 0} : need_ub(A, X);
}
// (D u) at the cell of the thread (apply_M): u_X at f and f + e_X
__host__ __device__ constexpr Need need_div(int X) {
  Need n{0, 0, 0};
  n = add2(n, X, 0, X, 0);
  n = add2(n, X, 1, X, 0);
  return n;
}
// grad p at face A: p at f and f - e_A
__host__ __device__ constexpr Need need_grad(int A) {
  Need n{0, 0, 0};
  n = add2(n, A, 0, A, 0);
  n = add2(n, A, -1, A, 0);
  return n;
}

// ---- row loads ------------------------------------------------------------
struct RowV {
  double m, c, p;
};

// Per-thread geometry: the linear index of (i, j, s) (row start + segment
// start), the wrapped row offsets for o0 / o1 = -1, 0, +1, and the segment.
struct Seg {
  int base;
  int di[3], dj[3];
  int t;    // lane
  int k0;   // PAIR: own face of the pair (colour); ALL: 0
  int wl;   // offset from a segment's first element to the wrapped element before it
  int wr;   // offset from a segment's first element to the wrapped element after its end
};

template <int W>
__device__ __forceinline__ Seg make_seg(const LevelDev& L, int i, int j, int s, int t, int k0) {
  Seg g;
  g.base = i * L.s0 + j * L.s1 + s;
  // a slab-distributed axis 0 reads its ghost planes instead of wrapping
  g.di[0] = ((i == 0 && !L.dist0) ? L.n[0] - 1 : -1) * L.s0;
  g.di[1] = 0;
  g.di[2] = ((i == L.n[0] - 1 && !L.dist0) ? -(L.n[0] - 1) : 1) * L.s0;
  g.dj[0] = (j == 0 ? L.n[1] - 1 : -1) * L.s1;
  g.dj[1] = 0;
  g.dj[2] = (j == L.n[1] - 1 ? -(L.n[1] - 1) : 1) * L.s1;
  g.t = t;
  g.k0 = k0;
  g.wl = s == 0 ? L.n[2] - 1 : -1;
  g.wr = s + W == L.n[2] ? -s : W;
  return g;
}

// PAIR (colour passes): lane t reads faces (2t, 2t+1) of a 64-face segment
// with one 16-B load; c is the face of colour k0, m / p its neighbours.
// ALL: lane t reads face t of a 32-face segment.  NC: read-only path.
template <bool PAIR, bool NC, bool NM, bool NP>
__device__ __forceinline__ RowV load_row(const double* __restrict__ a, int rp, const Seg& g) {
  // branch-free: every lane issues the segment-end load at the same (uniform)
  // address -- one sector, one wavefront -- so the loads of all rows can be
  // in flight together; only the end lane keeps the value
  RowV r;
  r.m = r.p = 0.0;
  if (PAIR) {
    const double2* q = reinterpret_cast<const double2*>(a + rp) + g.t;
    const double2 v = NC ? __ldg(q) : *q;
    const bool hi = g.k0 != 0;  // warp-uniform
    r.c = hi ? v.y : v.x;
    const double o = hi ? v.x : v.y;  // the pair's other face: m (hi) or p (lo)
    if (NM || NP) {  // (unconditional in hi: keeps the loads hoistable)
      const double nb = __shfl_sync(FULL, o, hi ? g.t + 1 : g.t - 1);
      const int ei = rp + (hi ? g.wr : g.wl);
      const double ev = NC ? __ldg(a + ei) : a[ei];
      const double x = g.t == (hi ? 31 : 0) ? ev : nb;
      r.m = hi ? o : x;
      r.p = hi ? x : o;
    } else {
      r.m = hi ? o : 0.0;
      r.p = hi ? 0.0 : o;
    }
  } else {
    r.c = NC ? __ldg(a + rp + g.t) : a[rp + g.t];
    if (NM) {
      const double w = __shfl_up_sync(FULL, r.c, 1);
      const double ev = NC ? __ldg(a + rp + g.wl) : a[rp + g.wl];
      r.m = g.t == 0 ? ev : w;
    }
    if (NP) {
      const double w = __shfl_down_sync(FULL, r.c, 1);
      const double ev = NC ? __ldg(a + rp + g.wr) : a[rp + g.wr];
      r.p = g.t == 31 ? ev : w;
    }
  }
  return r;
}

// The rows of one operand array selected by the masks (M, C, P).
template <unsigned M, unsigned C, unsigned P>
struct Rows {
  RowV r[9];
  double2 v[9];  // raw loads: PAIR the 16-B pair, ALL v.x
  double el[9], er[9];  // segment-end values (uniform-address loads)
  // Phase 1: issue every load of the selected rows (no dependent work, so all
  // rows of all operands can be in flight together)
  template <bool PAIR, bool NC>
  __device__ __forceinline__ void issue(const double* __restrict__ a, const Seg& g) {
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      if (((M | C | P) >> q) & 1u) {
        const int rp = g.base + g.di[q / 3] + g.dj[q % 3];
        const bool nm = (M >> q) & 1u, np = (P >> q) & 1u;
        if (PAIR) {
          const double2* qq = reinterpret_cast<const double2*>(a + rp) + g.t;
          v[q] = NC ? __ldg(qq) : *qq;
          if (nm || np) {
            const int ei = rp + (g.k0 ? g.wr : g.wl);
            el[q] = NC ? __ldg(a + ei) : a[ei];
          }
        } else {
          v[q].x = NC ? __ldg(a + rp + g.t) : a[rp + g.t];
          if (nm) el[q] = NC ? __ldg(a + rp + g.wl) : a[rp + g.wl];
          if (np) er[q] = NC ? __ldg(a + rp + g.wr) : a[rp + g.wr];
        }
      }
    }
  }
  // Phase 2: neighbours along the contiguous axis by warp shuffle
  template <bool PAIR>
  __device__ __forceinline__ void finish(const Seg& g) {
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      if (((M | C | P) >> q) & 1u) {
        const bool nm = (M >> q) & 1u, np = (P >> q) & 1u;
        RowV& o = r[q];
        o.m = o.p = 0.0;
        if (PAIR) {
          const bool hi = g.k0 != 0;  // warp-uniform
          o.c = hi ? v[q].y : v[q].x;
          const double ot = hi ? v[q].x : v[q].y;  // the pair's other face: m (hi) or p (lo)
          double x = 0.0;
          if (nm || np) {
            const double nb = __shfl_sync(FULL, ot, hi ? g.t + 1 : g.t - 1);
            x = g.t == (hi ? 31 : 0) ? el[q] : nb;
          }
          o.m = hi ? ot : x;
          o.p = hi ? x : ot;
        } else {
          o.c = v[q].x;
          if (nm) {
            const double w = __shfl_up_sync(FULL, o.c, 1);
            o.m = g.t == 0 ? el[q] : w;
          }
          if (np) {
            const double w = __shfl_down_sync(FULL, o.c, 1);
            o.p = g.t == 31 ? er[q] : w;
          }
        }
      }
    }
  }
  template <bool PAIR, bool NC>
  __device__ __forceinline__ void load(const double* __restrict__ a, const Seg& g) {
    issue<PAIR, NC>(a, g);
    finish<PAIR>(g);
  }
  // value at offset (o0, o1, o2)
  __device__ __forceinline__ double at(int o0, int o1, int o2) const {
    const RowV& v = r[rix(o0, o1)];
    return o2 < 0 ? v.m : (o2 > 0 ? v.p : v.c);
  }
  // value at f + sa e_A + sb e_B
  __device__ __forceinline__ double at2(int A, int sa, int B, int sb) const {
    return at(sa * e(0, A) + sb * e(0, B), sa * e(1, A) + sb * e(1, B), sa * e(2, A) + sb * e(2, B));
  }
};

#define SB_ROWS(name, need) Rows<(need).m, (need).c, (need).p> name

// Operand values of the face row of component A, in face_row_t's accessor
// interface (GAcc, sb_device.cuh).
struct RAcc {
  double mu_hi, mu_lo, rho_v;
  double mue_v[3][2];     // [B][hi edge]
  double ub_v[3][2][2];   // [B][hi][lowA]
  __device__ __forceinline__ double mu(bool lo) const { return lo ? mu_lo : mu_hi; }
  __device__ __forceinline__ double gam(bool) const { return 0.0; }
  __device__ __forceinline__ double divh(bool) const { return 0.0; }
  template <int B>
  __device__ __forceinline__ double mue(bool hi) const { return mue_v[B][hi ? 1 : 0]; }
  template <int B>
  __device__ __forceinline__ double ub(bool hi, bool lowA) const { return ub_v[B][hi ? 1 : 0][lowA ? 1 : 0]; }
  __device__ __forceinline__ double rho() const { return rho_v; }
};

// edge_mean (sb_device.cuh) on operand values: lower plane axis first
__device__ __forceinline__ double emean(double i, double ilo, double ihi, double ilohi) {
  const double a = 0.5 * (i + ilo);
  const double b = 0.5 * (ihi + ilohi);
  return 0.5 * (a + b);
}

// Fill UA7 + RAcc for component A from the loaded rows.  UR: rows of u_A;
// UB1/UB2: rows of the tangential components (ascending axis); MU: mu_c;
// E1/E2: stored mu_e(A,B) rows (unused when DE).
template <int FORM, int A, bool DE, class UR, class UB1, class UB2, class MU, class E1, class E2>
__device__ __forceinline__ void face_vals(const UR& ua, const UB1& u1, const UB2& u2, const MU& mu, const E1& e1,
                                          const E2& e2, UA7& s, RAcc& acc) {
  s.c = ua.at(0, 0, 0);
  s.p[0] = ua.at(1, 0, 0);
  s.m[0] = ua.at(-1, 0, 0);
  s.p[1] = ua.at(0, 1, 0);
  s.m[1] = ua.at(0, -1, 0);
  s.p[2] = ua.at(0, 0, 1);
  s.m[2] = ua.at(0, 0, -1);
  acc.mu_hi = mu.at2(A, 0, A, 0);
  acc.mu_lo = mu.at2(A, -1, A, 0);
  acc.rho_v = 0.0;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int B = k == 0 ? oth1(A) : oth2(A);
    double lo, hi;
    if (DE) {
      const double f = acc.mu_hi, fa = acc.mu_lo;
      const double fbm = mu.at2(A, 0, B, -1), fbma = mu.at2(A, -1, B, -1);
      const double fbp = mu.at2(A, 0, B, 1), fbpa = mu.at2(A, -1, B, 1);
      if (A < B) {
        lo = emean(f, fa, fbm, fbma);
        hi = emean(fbp, fbpa, f, fa);
      } else {
        lo = emean(f, fbm, fa, fbma);
        hi = emean(fbp, f, fbpa, fa);
      }
    } else {
      lo = k == 0 ? e1.at2(A, 0, B, 0) : e2.at2(A, 0, B, 0);
      hi = k == 0 ? e1.at2(A, 0, B, 1) : e2.at2(A, 0, B, 1);
    }
    acc.mue_v[B][0] = lo;
    acc.mue_v[B][1] = hi;
    if (FORM != F_LAP) {
      const double b00 = k == 0 ? u1.at2(A, 0, B, 0) : u2.at2(A, 0, B, 0);
      const double b0a = k == 0 ? u1.at2(A, -1, B, 0) : u2.at2(A, -1, B, 0);
      const double b10 = k == 0 ? u1.at2(A, 0, B, 1) : u2.at2(A, 0, B, 1);
      const double b1a = k == 0 ? u1.at2(A, -1, B, 1) : u2.at2(A, -1, B, 1);
      acc.ub_v[B][0][0] = b00;
      acc.ub_v[B][0][1] = b0a;
      acc.ub_v[B][1][0] = b10;
      acc.ub_v[B][1][1] = b1a;
    } else {
      acc.ub_v[B][0][0] = acc.ub_v[B][0][1] = acc.ub_v[B][1][0] = acc.ub_v[B][1][1] = 0.0;
    }
  }
}

constexpr Need NONE{0, 0, 0};

// ---- colour pass (multigrid.py:327-340; k_face_colour's expression) --------
template <int FORM, int A, bool DE, int MINB>
__global__ void __launch_bounds__(RT, MINB)
k_face_colour_rv(LevelDev L, Ptr3 u, const double* __restrict__ rhs, int parity, double omega, int nseg) {
  pdl_enter();
  // a CTA = 8 warps on 8 consecutive rows j of one segment: the +-1 rows
  // along axis 1 are shared through L1
  const int t = threadIdx.x & 31;
  const int nj = (L.n[1] + 7) >> 3;
  const int seg = (int)blockIdx.x % nseg, rest = (int)blockIdx.x / nseg;
  const int i = rest / nj, j = (rest - i * nj) * 8 + (threadIdx.x >> 5);
  if (j >= L.n[1]) return;  // whole warps
  const int k0 = (parity - i - j) & 1;
  const Seg g = make_seg<64>(L, i, j, seg * 64, t, k0);
  constexpr int B1 = oth1(A), B2 = oth2(A);
  constexpr Need nua = need_ua(A), nb1 = need_u(A, B1, FORM), nb2 = need_u(A, B2, FORM);
  constexpr Need nmu = need_mu(A, DE);
  constexpr Need ne1 = DE ? NONE : need_mue(A, B1), ne2 = DE ? NONE : need_mue(A, B2);
  SB_ROWS(ua, nua);
  SB_ROWS(ub1, nb1);
  SB_ROWS(ub2, nb2);
  SB_ROWS(mu, nmu);
  SB_ROWS(me1, ne1);
  SB_ROWS(me2, ne2);
  // u_A is relaxed in place: this pass writes only faces of colour k0, and the
  // values used from u_A are the other colour (neighbours) or the thread's own
  // face, so plain loads see no race on any value they use
  ua.template issue<true, false>(u.p[A], g);
  if (FORM != F_LAP) {
    ub1.template issue<true, true>(u.p[B1], g);
    ub2.template issue<true, true>(u.p[B2], g);
  }
  mu.template issue<true, true>(L.mu_c, g);
  if (!DE) {
    me1.template issue<true, true>(L.mu_e[edge_of(A, B1)], g);
    me2.template issue<true, true>(L.mu_e[edge_of(A, B2)], g);
  }
  const int f = g.base + 2 * t + k0;
  const double rhs_f = __ldg(rhs + f);
  ua.template finish<true>(g);
  if (FORM != F_LAP) {
    ub1.template finish<true>(g);
    ub2.template finish<true>(g);
  }
  mu.template finish<true>(g);
  if (!DE) {
    me1.template finish<true>(g);
    me2.template finish<true>(g);
  }
  UA7 s;
  RAcc acc;
  face_vals<FORM, A, DE>(ua, ub1, ub2, mu, me1, me2, s, acc);
  if (L.theta != 0.0) acc.rho_v = __ldg(L.rho_f[A] + f);
  const int ci[3] = {i, j, seg * 64 + 2 * t + k0};
  double dg;
  const double au = face_row_t<3, FORM, A, true>(L, s, acc, ci, dg);
  const double res = rhs_f - au;
  u.p[A][f] = s.c + omega * (res / dg);
}

// ---- all faces: residual field (k_face_res3) and apply_M (k_apply_M) -------
template <int FORM, bool DE, bool MODE_M, int MINB>
__global__ void __launch_bounds__(RT, MINB)
k_face_all_rv(LevelDev L, CPtr3 x, CPtr3 rhs, const double* __restrict__ p, Ptr3 out, double* __restrict__ out_p,
              int nseg) {
  pdl_enter();
  const int t = threadIdx.x & 31;
  const int nj = (L.n[1] + 7) >> 3;
  const int seg = (int)blockIdx.x % nseg, rest = (int)blockIdx.x / nseg;
  const int i = rest / nj, j = (rest - i * nj) * 8 + (threadIdx.x >> 5);
  if (j >= L.n[1]) return;
  const Seg g = make_seg<32>(L, i, j, seg * 32, t, 0);
  // union of the three face rows' (and the divergence's) operand rows
  constexpr Need n0 = orn(orn(need_u(0, 0, FORM), need_u(1, 0, FORM)), orn(need_u(2, 0, FORM), MODE_M ? need_div(0) : NONE));
  constexpr Need n1 = orn(orn(need_u(0, 1, FORM), need_u(1, 1, FORM)), orn(need_u(2, 1, FORM), MODE_M ? need_div(1) : NONE));
  constexpr Need n2 = orn(orn(need_u(0, 2, FORM), need_u(1, 2, FORM)), orn(need_u(2, 2, FORM), MODE_M ? need_div(2) : NONE));
  constexpr Need nmu = orn(need_mu(0, DE), orn(need_mu(1, DE), need_mu(2, DE)));
  // stored mu_e arrays by normal axis e: edge (A,B) with e = 3-A-B
  constexpr Need ne0 = DE ? NONE : orn(need_mue(1, 2), need_mue(2, 1));
  constexpr Need ne1 = DE ? NONE : orn(need_mue(0, 2), need_mue(2, 0));
  constexpr Need ne2 = DE ? NONE : orn(need_mue(0, 1), need_mue(1, 0));
  constexpr Need np = MODE_M ? orn(need_grad(0), orn(need_grad(1), need_grad(2))) : NONE;
  SB_ROWS(u0, n0);
  SB_ROWS(u1, n1);
  SB_ROWS(u2, n2);
  SB_ROWS(mu, nmu);
  SB_ROWS(e0, ne0);
  SB_ROWS(e1, ne1);
  SB_ROWS(e2, ne2);
  SB_ROWS(pr, np);
  u0.template issue<false, true>(x.p[0], g);
  u1.template issue<false, true>(x.p[1], g);
  u2.template issue<false, true>(x.p[2], g);
  mu.template issue<false, true>(L.mu_c, g);
  if (!DE) {
    e0.template issue<false, true>(L.mu_e[0], g);
    e1.template issue<false, true>(L.mu_e[1], g);
    e2.template issue<false, true>(L.mu_e[2], g);
  }
  if (MODE_M) pr.template issue<false, true>(p, g);
  u0.template finish<false>(g);
  u1.template finish<false>(g);
  u2.template finish<false>(g);
  mu.template finish<false>(g);
  if (!DE) {
    e0.template finish<false>(g);
    e1.template finish<false>(g);
    e2.template finish<false>(g);
  }
  if (MODE_M) pr.template finish<false>(g);
  const int f = g.base + t;
  const int ci[3] = {i, j, seg * 32 + t};
  UA7 s;
  RAcc acc;
  double dg;
  // component 0: tangents 1, 2 -> mu_e normals 2 (edge (0,1)) and 1 (edge (0,2))
  face_vals<FORM, 0, DE>(u0, u1, u2, mu, e2, e1, s, acc);
  if (L.theta != 0.0) acc.rho_v = __ldg(L.rho_f[0] + f);
  double a0 = face_row_t<3, FORM, 0, true>(L, s, acc, ci, dg);
  // component 1: tangents 0, 2 -> edges (0,1) normal 2, (1,2) normal 0
  face_vals<FORM, 1, DE>(u1, u0, u2, mu, e2, e0, s, acc);
  if (L.theta != 0.0) acc.rho_v = __ldg(L.rho_f[1] + f);
  double a1 = face_row_t<3, FORM, 1, true>(L, s, acc, ci, dg);
  // component 2: tangents 0, 1 -> edges (0,2) normal 1, (1,2) normal 0
  face_vals<FORM, 2, DE>(u2, u0, u1, mu, e1, e0, s, acc);
  if (L.theta != 0.0) acc.rho_v = __ldg(L.rho_f[2] + f);
  double a2 = face_row_t<3, FORM, 2, true>(L, s, acc, ci, dg);
  if (MODE_M) {
    // m_face: A u + G p; (G p)_A = (p(f) - p(f - e_A)) / h
    out.p[0][f] = a0 + (pr.at(0, 0, 0) - pr.at(-1, 0, 0)) * L.inv_h;
    out.p[1][f] = a1 + (pr.at(0, 0, 0) - pr.at(0, -1, 0)) * L.inv_h;
    out.p[2][f] = a2 + (pr.at(0, 0, 0) - pr.at(0, 0, -1)) * L.inv_h;
    // div_sum: ((d0 + d1) + d2)
    double acc_d = u0.at(1, 0, 0) - u0.at(0, 0, 0);
    acc_d = acc_d + (u1.at(0, 1, 0) - u1.at(0, 0, 0));
    acc_d = acc_d + (u2.at(0, 0, 1) - u2.at(0, 0, 0));
    out_p[f] = -(acc_d * L.inv_h);
  } else {
    out.p[0][f] = __ldg(rhs.p[0] + f) - a0;
    out.p[1][f] = __ldg(rhs.p[1] + f) - a1;
    out.p[2][f] = __ldg(rhs.p[2] + f) - a2;
  }
}

// ---- row-march: all faces, a warp walks one whole row ----------------------
// k_face_all_rv is latency / instruction bound (ncu, C5 256^3: 600 instructions
// per warp of 32 points, issue 56-65 %, DRAM 28-38 %): two thirds of its
// instructions are address arithmetic, the segment-end loads and selects of
// every +-1 operand, and stress terms evaluated twice (each edge flux by both
// faces that share it).  Here a warp owns a whole row (i, j) and walks it in
// 32-face segments:
//  * the -1 neighbours along the row come from the neighbouring lane, lane 0's
//    from lane 31 of the previous segment (carried in registers): no
//    segment-end loads, the row end is read once before the walk (periodic
//    wrap);
//  * every edge stress T_AB = mu_e (d_B u_A + d_A u_B) and normal stress
//    N_A = mu_c d_A u_A is evaluated ONCE per point at the point's own
//    (lower) edge / cell and shared by the two rows (A and B) that use it;
//    the +1 values along axes 0 / 1 are evaluated from the neighbouring rows'
//    operands, the +1 values along the row are the next lane's (one rotate
//    shuffle; lane 31 finishes its face one segment later, the last segment
//    with the first segment's lane-0 values);
//  * derived edge viscosities as sums of cell pairs shared between edges,
//    the factor 1/4 folded into the h^-2 scale (exact: powers of two), fused
//    multiply-adds on the final combinations.
// 79 fp64 operations and ~220 instructions per point instead of 165 / 600.
// Same formulas as face_row_t with a different rounding order (and FMAs):
// equal to the per-face kernels to ~1e-15 relative, not bit-identical
// (tests/test_gpu_rowv.py).  Derived edge viscosities only (mue_derived levels).
// L2 prefetch of the row walk (ncu, C5 256^3, apply_M / residual field; off:
// 321 / 318 us).  RM_PF > 0: the first-touched rows RM_PF segments ahead along
// the row (1: 301 / 289, 2: 290 / 301, 4: 303 / 327); RM_PF < 0: this warp's own
// row -RM_PF planes beyond the last plane it reads, for the CTAs of the later
// planes (-1: 281 / 269, -2: 273 / 263 (default), -3 and -4: the same)
#ifndef RM_PF
#define RM_PF -2
#endif
__device__ __forceinline__ void pf_l2(const double* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
__device__ __forceinline__ double rot_m(double v, double& prev, int lane) {
  const double s = lane == 31 ? prev : v;
  prev = v;
  return __shfl_sync(FULL, s, (lane + 31) & 31);
}
__device__ __forceinline__ double rot_p(double v, int lane) { return __shfl_sync(FULL, v, (lane + 1) & 31); }

template <int FORM, bool MODE_M, bool THETA, bool DE, bool W2, int TI, int TJ, int MINB>
__global__ void __launch_bounds__(TI * TJ * 32, MINB)
k_face_all_rm(LevelDev L, CPtr3 x, CPtr3 rhs, const double* __restrict__ p, Ptr3 out, double* __restrict__ out_p) {
  pdl_enter();
  constexpr bool ST = FORM != F_LAP;
  const int lane = threadIdx.x & 31;
  // a CTA = TI x TJ warps on TJ consecutive rows of TI consecutive planes:
  // the +-1 rows / planes of its warps are shared through L1
  const int wid = threadIdx.x >> 5;
  const int j = (int)blockIdx.x * TJ + wid % TJ, i = (int)blockIdx.y * TI + wid / TJ;
  if (j >= L.n[1] || i >= L.n[0]) return;  // whole warps
  const int n2 = L.n[2];
  const int rowc = i * L.s0 + j * L.s1;
  // a slab-distributed axis 0 reads its ghost planes instead of wrapping
  const int im = ((i == 0 && !L.dist0) ? L.n[0] - 1 : -1) * L.s0;
  const int ip = ((i == L.n[0] - 1 && !L.dist0) ? -(L.n[0] - 1) : 1) * L.s0;
  const int jm = (j == 0 ? L.n[1] - 1 : -1) * L.s1;
  const int jp = (j == L.n[1] - 1 ? -(L.n[1] - 1) : 1) * L.s1;
  const double* __restrict__ u0 = x.p[0];
  const double* __restrict__ u1 = x.p[1];
  const double* __restrict__ u2 = x.p[2];
  const double* __restrict__ mu = L.mu_c;
  // stored edge viscosities (!DE): mu_e(A,B) lives in L.mu_e[3 - A - B]
  const double* __restrict__ e01 = L.mu_e[2];
  const double* __restrict__ e02 = L.mu_e[1];
  const double* __restrict__ e12 = L.mu_e[0];
  const double c1 = (ST ? 2.0 : 1.0) * L.inv_h2, c2 = (DE ? 0.25 : 1.0) * L.inv_h2;
  // results are accumulated as sgn * (A u)_A [+ rhs | + G p]
  const double sg = MODE_M ? 1.0 : -1.0;
  const double k1 = -sg * c1, k2 = -sg * c2;

  // carried -1 operands: lane 31's value of the previous segment; before the
  // walk, the row's last element (periodic wrap) or, W2 (walls at both ends
  // of the row), the ghost values behind the low wall: -u (no-slip: the wall
  // flux mu_e 2 u / h, operators.py:267-300) or +u (free-slip: no flux) for the
  // tangential components, the boundary cell's mu (two-cell boundary mean)
  double pv_u0c, pv_u0x, pv_u1c, pv_u1y, pv_u2c, pv_mc, pv_P0c = 0.0, pv_P0x = 0.0, pv_P1c = 0.0, pv_P1y = 0.0, pv_p = 0.0;
  {
    const int q = W2 ? rowc : rowc + n2 - 1;
    const double gl = W2 ? (L.bclo[2] == BC_FREESLIP ? 1.0 : -1.0) : 1.0;
    const double m00 = __ldg(mu + q);
    double mm0 = 0.0, mp0 = 0.0, m0m = 0.0, m0p = 0.0;
    if (DE) {
      mm0 = __ldg(mu + q + im);
      mp0 = __ldg(mu + q + ip);
      m0m = __ldg(mu + q + jm);
      m0p = __ldg(mu + q + jp);
    }
    pv_u0c = gl * __ldg(u0 + q);
    pv_u0x = gl * __ldg(u0 + q + ip);
    pv_u1c = gl * __ldg(u1 + q);
    pv_u1y = gl * __ldg(u1 + q + jp);
    pv_u2c = W2 ? 0.0 : __ldg(u2 + q);  // W2: face 0 of component 2 is a wall face (its row is not formed)
    pv_mc = m00;
    if (DE) {
      pv_P0c = m00 + mm0;
      pv_P0x = mp0 + m00;
      pv_P1c = m00 + m0m;
      pv_P1y = m0p + m00;
    }
    if (MODE_M) pv_p = __ldg(p + q);
  }
  double pe0 = 0.0, pe1 = 0.0, pe2 = 0.0, peD = 0.0, peU = 0.0;  // lane 31: unfinished face of the previous segment
  double f0 = 0.0, f1 = 0.0, f2 = 0.0, f3 = 0.0;                  // lane 31: lane 0's +1 values of the first segment
  const int nseg = n2 >> 5;
#pragma unroll 1
  for (int s = 0; s < nseg; ++s) {
    const int q = rowc + (s << 5) + lane;
#if RM_PF > 0
    // the rows this plane touches first (plane i + 1 of u and mu, the own row of
    // p / rhs) come from DRAM: ask L2 for them RM_PF segments ahead
    if (s + RM_PF < nseg) {
      const int qp = q + 32 * RM_PF;
      pf_l2(u0 + qp + ip);
      pf_l2(u1 + qp + ip);
      pf_l2(u2 + qp + ip);
      pf_l2(mu + qp + ip);
      if (MODE_M) {
        pf_l2(p + qp);
      } else {
        pf_l2(rhs.p[0] + qp);
        pf_l2(rhs.p[1] + qp);
        pf_l2(rhs.p[2] + qp);
      }
    }
#elif RM_PF < 0
    // plane-ahead variant: this warp's row, -RM_PF planes after plane i + 1
    {
      const int pl = i + 1 - RM_PF;
      if (pl < L.n[0] + (L.dist0 ? 1 : 0)) {
        const int qp = q + (pl - i) * L.s0;
        pf_l2(u0 + qp);
        pf_l2(u1 + qp);
        pf_l2(u2 + qp);
        pf_l2(mu + qp);
        if (MODE_M) {
          pf_l2(p + qp - L.s0);
        } else {
          pf_l2(rhs.p[0] + qp - L.s0);
          pf_l2(rhs.p[1] + qp - L.s0);
          pf_l2(rhs.p[2] + qp - L.s0);
        }
      }
    }
#endif
    const double u0c = __ldg(u0 + q), u0im = __ldg(u0 + q + im), u0ip = __ldg(u0 + q + ip);
    const double u0jm = __ldg(u0 + q + jm), u0jp = __ldg(u0 + q + jp), u0ipjm = __ldg(u0 + q + ip + jm);
    const double u1c = __ldg(u1 + q), u1im = __ldg(u1 + q + im), u1ip = __ldg(u1 + q + ip);
    const double u1jm = __ldg(u1 + q + jm), u1jp = __ldg(u1 + q + jp), u1imjp = __ldg(u1 + q + im + jp);
    const double u2c = __ldg(u2 + q), u2im = __ldg(u2 + q + im), u2ip = __ldg(u2 + q + ip);
    const double u2jm = __ldg(u2 + q + jm), u2jp = __ldg(u2 + q + jp);
    const double mc = __ldg(mu + q), mim = __ldg(mu + q + im), mjm = __ldg(mu + q + jm);
    double mip = 0.0, mjp = 0.0, mimjm = 0.0, mimjp = 0.0, mipjm = 0.0;
    double S01, S01y, S01x, S02, S02x, S12, S12y;
    if (DE) {
      mip = __ldg(mu + q + ip);
      mjp = __ldg(mu + q + jp);
      mimjm = __ldg(mu + q + im + jm);
      mimjp = __ldg(mu + q + im + jp);
      mipjm = __ldg(mu + q + ip + jm);
    } else {
      S01 = __ldg(e01 + q);
      S01y = __ldg(e01 + q + jp);
      S01x = __ldg(e01 + q + ip);
      S02 = __ldg(e02 + q);
      S02x = __ldg(e02 + q + ip);
      S12 = __ldg(e12 + q);
      S12y = __ldg(e12 + q + jp);
    }
    double pc = 0.0, pim = 0.0, pjm = 0.0, r0 = 0.0, r1 = 0.0, r2 = 0.0;
    if (MODE_M) {
      pc = __ldg(p + q);
      pim = __ldg(p + q + im);
      pjm = __ldg(p + q + jm);
    } else {
      r0 = __ldg(rhs.p[0] + q);
      r1 = __ldg(rhs.p[1] + q);
      r2 = __ldg(rhs.p[2] + q);
    }
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    if (THETA) {
      t0 = L.theta * __ldg(L.rho_f[0] + q);
      t1 = L.theta * __ldg(L.rho_f[1] + q);
      t2 = L.theta * __ldg(L.rho_f[2] + q);
    }
    // -1 neighbours along the row
    const double u0c_m = rot_m(u0c, pv_u0c, lane), u1c_m = rot_m(u1c, pv_u1c, lane);
    double u0x_m = 0.0, u1y_m = 0.0;
    if (ST) {
      u0x_m = rot_m(u0ip, pv_u0x, lane);
      u1y_m = rot_m(u1jp, pv_u1y, lane);
    }
    const double u2c_m = rot_m(u2c, pv_u2c, lane), mc_m = rot_m(mc, pv_mc, lane);
    if (DE) {
      // cell pair sums (edge_mean's first stage: lower plane axis first), then
      // 4 mu_e at the edges used (no suffix: own point, y: + e_1, x: + e_0)
      const double P0c = mc + mim, P0x = mip + mc, P0jm = mjm + mimjm, P0jp = mjp + mimjp, P0xjm = mipjm + mjm;
      const double P1c = mc + mjm, P1y = mjp + mc;
      const double P0c_m = rot_m(P0c, pv_P0c, lane), P0x_m = rot_m(P0x, pv_P0x, lane);
      const double P1c_m = rot_m(P1c, pv_P1c, lane), P1y_m = rot_m(P1y, pv_P1y, lane);
      S01 = P0c + P0jm;
      S01y = P0jp + P0c;
      S01x = P0x + P0xjm;
      S02 = P0c + P0c_m;
      S02x = P0x + P0x_m;
      S12 = P1c + P1c_m;
      S12y = P1y + P1y_m;
    }
    // edge stresses T_AB: tA = the d_B u_A part (row A), tB = the d_A u_B part
    // (row B); the stress forms share the full bracket
    double T01a, T01b, T01y, T01x, T02a, T02b, T02x, T12a, T12b, T12y;
    if (ST) {
      T01a = T01b = S01 * ((u0c - u0jm) + (u1c - u1im));
      T01y = S01y * ((u0jp - u0c) + (u1jp - u1imjp));
      T01x = S01x * ((u0ip - u0ipjm) + (u1ip - u1c));
      T02a = T02b = S02 * ((u0c - u0c_m) + (u2c - u2im));
      T02x = S02x * ((u0ip - u0x_m) + (u2ip - u2c));
      T12a = T12b = S12 * ((u1c - u1c_m) + (u2c - u2jm));
      T12y = S12y * ((u1jp - u1y_m) + (u2jp - u2c));
    } else {
      T01a = S01 * (u0c - u0jm);
      T01b = S01 * (u1c - u1im);
      T01y = S01y * (u0jp - u0c);    // row 0
      T01x = S01x * (u1ip - u1c);    // row 1
      T02a = S02 * (u0c - u0c_m);
      T02b = S02 * (u2c - u2im);
      T02x = S02x * (u2ip - u2c);    // row 2
      T12a = S12 * (u1c - u1c_m);
      T12b = S12 * (u2c - u2jm);
      T12y = S12y * (u2jp - u2c);    // row 2
    }
    // normal stresses at the cells x, x - e_A
    const double N0 = mc * (u0ip - u0c), N0m = mim * (u0c - u0im);
    const double N1 = mc * (u1jp - u1c), N1m = mjm * (u1c - u1jm);
    const double N2m = mc_m * (u2c - u2c_m);
    // everything but the +1 term along the row
    double a0 = fma(k1, N0 - N0m, k2 * ((T01y - T01a) - T02a));
    double a1 = fma(k1, N1 - N1m, k2 * ((T01x - T01b) - T12a));
    double a2 = fma(-k1, N2m, k2 * ((T02x - T02b) + (T12y - T12b)));
    if (THETA) {
      a0 = fma(sg * t0, u0c, a0);
      a1 = fma(sg * t1, u1c, a1);
      a2 = fma(sg * t2, u2c, a2);
    }
    double d01 = 0.0;
    if (MODE_M) {
      const double pc_m = rot_m(pc, pv_p, lane);
      a0 = fma(pc - pim, L.inv_h, a0);
      a1 = fma(pc - pjm, L.inv_h, a1);
      a2 = fma(pc - pc_m, L.inv_h, a2);
      d01 = (u0ip - u0c) + (u1jp - u1c);  // div_sum order: (d0 + d1) + d2
    } else {
      a0 += r0;
      a1 += r1;
      a2 += r2;
    }
    // +1 values along the row: lanes 0..30 the next lane's (this segment),
    // lane 31 lane 0's, which completes its face of the PREVIOUS segment
    const double h0 = rot_p(T02a, lane), h1 = rot_p(T12a, lane), h2 = rot_p(N2m, lane);
    const double h3 = MODE_M ? rot_p(u2c, lane) : 0.0;
    const bool last = lane == 31;
    double b0 = a0, b1 = a1, b2 = a2, bd = d01, bu = u2c;
    if (s == 0) {
      f0 = h0;
      f1 = h1;
      f2 = h2;
      f3 = h3;
    }
    if (last) {
      b0 = pe0;
      b1 = pe1;
      b2 = pe2;
      bd = peD;
      bu = peU;
    }
    pe0 = a0;
    pe1 = a1;
    pe2 = a2;
    peD = d01;
    peU = u2c;
    const int qo = last ? q - 32 : q;
    if (!last || s > 0) {
      out.p[0][qo] = fma(k2, h0, b0);
      out.p[1][qo] = fma(k2, h1, b1);
      if (!(W2 && s == 0 && lane == 0)) out.p[2][qo] = fma(k1, h2, b2);
      else if (MODE_M) out.p[2][qo] = 0.0;  // wall face (k_apply_M's m_face); the residual field leaves it
      if (MODE_M) out_p[qo] = -((bd + (h3 - bu)) * L.inv_h);
    }
  }
  if (lane == 31) {  // the row's last face: +1 neighbours wrap to the first segment's lane 0
    const int qo = rowc + n2 - 1;
    if (W2) {
      // ... or sit on the high wall: edge stresses from the ghost values (-u /
      // +u), the normal stress of the last cell against the wall face u_2 = 0
      const double gh = (L.bchi[2] == BC_FREESLIP ? 1.0 : -1.0) - 1.0;
      const double s02 = DE ? 2.0 * pv_P0c : __ldg(e02 + qo + 1);
      const double s12 = DE ? 2.0 * pv_P1c : __ldg(e12 + qo + 1);
      f0 = s02 * (gh * pv_u0c);
      f1 = s12 * (gh * pv_u1c);
      f2 = pv_mc * (0.0 - pv_u2c);
      f3 = 0.0;
      if (MODE_M) out.p[2][qo + 1] = 0.0;  // the high wall face
    }
    out.p[0][qo] = fma(k2, f0, pe0);
    out.p[1][qo] = fma(k2, f1, pe1);
    out.p[2][qo] = fma(k1, f2, pe2);
    if (MODE_M) out_p[qo] = -((peD + (f3 - peU)) * L.inv_h);
  }
}

// SB_ROWM=0: the segment kernel (k_face_all_rv) on every row-vector level
bool rowm_on() {
  const char* e = std::getenv("SB_ROWM");
  return !(e && e[0] == '0');
}

int blocks_for(const LevelDev& L, int seglen) {
  return L.n[0] * ((L.n[1] + 7) / 8) * (L.n[2] / seglen);
}

// read per launch: tests compare both paths in one process
bool rowv_on() {  // SB_ROWV=0: per-face kernels everywhere
  const char* e = std::getenv("SB_ROWV");
  return !(e && e[0] == '0');
}

template <int FM, int A>
void colour_rv_t(cudaStream_t s, const LevelDev& L, Ptr3 u, const double* rhs, int parity, double omega) {
  const int nseg = L.n[2] / 64;
  const int nb = blocks_for(L, 64);
  if (L.mue_derived) launch_k(k_face_colour_rv<FM, A, true, 3>, nb, RT, 0, s, L, u, rhs, parity, omega, nseg);
  else launch_k(k_face_colour_rv<FM, A, false, 3>, nb, RT, 0, s, L, u, rhs, parity, omega, nseg);
}

}  // namespace

// The colour passes stay on the per-face kernel (k_face_colour with derived
// mu_e, 40 registers, 48 resident warps per SM): the row-vector colour pass
// moves half the L1 wavefronts but needs 74-80 registers and is latency bound
// (ncu, C5 256^3: 173-195 us vs 155-164 us per pass).
// SB_ROWV_COLOUR=1 selects it.
bool rowv_colour_on() {
  const char* e = std::getenv("SB_ROWV_COLOUR");
  return e && e[0] == '1';
}

bool rowv_supported(const LevelDev& L, int dim, int form) {
  if (dim != 3 || form == F_BULK || !rowv_on()) return false;
  for (int a = 0; a < 3; ++a)
    if (L.n[a] < 2) return false;
  if (L.bclo[0] != BC_PER || L.bclo[1] != BC_PER || L.n[2] % 64 != 0) return false;
  // walls along the contiguous axis (C4's z walls): the row-march kernel only
  return L.bclo[2] == BC_PER || rowm_on();
}

bool rowv_colour_supported(const LevelDev& L, int dim, int form) {
  return rowv_colour_on() && L.bclo[2] == BC_PER && rowv_supported(L, dim, form);
}

void launch_face_colour_rv(cudaStream_t s, const LevelDev& L, int form, int A, Ptr3 u, const double* rhsA,
                           int parity, double omega) {
  if (form == F_LAP) {
    if (A == 0) colour_rv_t<F_LAP, 0>(s, L, u, rhsA, parity, omega);
    else if (A == 1) colour_rv_t<F_LAP, 1>(s, L, u, rhsA, parity, omega);
    else colour_rv_t<F_LAP, 2>(s, L, u, rhsA, parity, omega);
  } else {
    if (A == 0) colour_rv_t<F_STRESS, 0>(s, L, u, rhsA, parity, omega);
    else if (A == 1) colour_rv_t<F_STRESS, 1>(s, L, u, rhsA, parity, omega);
    else colour_rv_t<F_STRESS, 2>(s, L, u, rhsA, parity, omega);
  }
}

template <bool MODE_M>
static void all_rv(cudaStream_t s, const LevelDev& L, int form, CPtr3 x, CPtr3 rhs, const double* p, Ptr3 out,
                   double* out_p) {
  const int nseg = L.n[2] / 32;
  const int nb = blocks_for(L, 32);
  const bool de = L.mue_derived != 0;
  const bool w2 = L.bclo[2] != BC_PER;
  if (rowm_on() || w2) {  // row-march kernel: a warp per row
    const bool th = L.theta != 0.0;
    // CTA tile: 1 plane x 4 rows, 4 CTAs per SM (128 registers).  Measured
    // (ncu, C5 256^3, apply_M / residual): 1x8 warps x 2 CTAs 328 / 325 us,
    // 1x4 x 4 322 / 319, 2x2 x 4 332 / 315, 2x4 x 2 339 / 322, 4x4 x 1 359 / 341;
    // lane 31's carried values in shared memory (80-96 registers, 20-24 warps
    // per SM) 307-352 us: the L1 data pipe (loads + shuffles) is the busiest
    // unit at 62 %, more warps do not help
#define SB_RM2(FM, TH, DD)                                                                                        \
  if (w2) launch_k(k_face_all_rm<FM, MODE_M, TH, DD, true, 1, 4, 4>, dim3((L.n[1] + 3) / 4, L.n[0], 1), dim3(128, 1, 1), 0, \
                   s, L, x, rhs, p, out, out_p);                                                                  \
  else launch_k(k_face_all_rm<FM, MODE_M, TH, DD, false, 1, 4, 4>, dim3((L.n[1] + 3) / 4, L.n[0], 1), dim3(128, 1, 1), 0, \
                s, L, x, rhs, p, out, out_p)
#define SB_RM1(FM, TH)       \
  if (de) { SB_RM2(FM, TH, true); } \
  else { SB_RM2(FM, TH, false); }
#define SB_RM(FM)            \
  if (th) { SB_RM1(FM, true) } \
  else { SB_RM1(FM, false) }
    if (form == F_LAP) {
      SB_RM(F_LAP)
    } else {
      SB_RM(F_STRESS)
    }
#undef SB_RM
#undef SB_RM1
#undef SB_RM2
    return;
  }
  if (form == F_LAP) {
    if (de) launch_k(k_face_all_rv<F_LAP, true, MODE_M, RV_MINB>, nb, RT, 0, s, L, x, rhs, p, out, out_p, nseg);
    else launch_k(k_face_all_rv<F_LAP, false, MODE_M, RV_MINB>, nb, RT, 0, s, L, x, rhs, p, out, out_p, nseg);
  } else {
    if (de) launch_k(k_face_all_rv<F_STRESS, true, MODE_M, RV_MINB>, nb, RT, 0, s, L, x, rhs, p, out, out_p, nseg);
    else launch_k(k_face_all_rv<F_STRESS, false, MODE_M, RV_MINB>, nb, RT, 0, s, L, x, rhs, p, out, out_p, nseg);
  }
}

void launch_face_res3_rv(cudaStream_t s, const LevelDev& L, int form, CPtr3 x, CPtr3 rhs, Ptr3 out) {
  all_rv<false>(s, L, form, x, rhs, nullptr, out, nullptr);
}

void launch_apply_M_rv(cudaStream_t s, const LevelDev& L, int form, CPtr3 u, const double* p, Ptr3 out_u,
                       double* out_p) {
  CPtr3 none{{nullptr, nullptr, nullptr}};
  all_rv<true>(s, L, form, u, none, p, out_u, out_p);
}

}  // namespace sb
