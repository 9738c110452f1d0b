// sb_sweep.cu -- fused two-colour Gauss-Seidel sweeps (2.5D streaming, sm_100a).
//
// One kernel performs BOTH colour passes of one component (multigrid.py:334-340
// for a face component, :321-324 for cells) out of place: it reads the
// current iterate x (never modified during the launch) and writes the swept
// iterate to a second buffer.  A CTA owns a TJ x TK tile of the (axis-1,
// axis-2) plane and marches along axis 0 over a chunk of planes.  Every
// operand (the iterate, the other velocity components, mu_c, mu_e, rho, rhs,
// 1/rho) is staged plane by plane into a per-array shared-memory ring with
// cp.async (LDGSTS), one plane ahead of use, so the relaxation phases read
// shared memory only:
//
//   step p:  prefetch the next plane of every operand
//            R_p   = old plane p with its RED unknowns relaxed   (tile + ring 1)
//            black = relax the BLACK unknowns of plane p-1 from R_{p-2..p}
//            write plane p-1 (both colours) to the output buffer
//
// Red faces never neighbour red faces (even periodic extents), so R_p depends
// on old values only and the ring recomputed by neighbouring CTAs is
// bit-identical; black reads only red neighbours and its own old value.  The
// result equals the reference's sequential red-then-black pass to the bit,
// while every array streams from HBM once per component sweep (64 B per face
// instead of 2 x 56 B for two colour passes).  Levels with an
// odd periodic extent, 2D grids and the stress+bulk form use the per-colour
// kernels instead.
#include <cuda_runtime.h>
#include <algorithm>
#include "sb_kernels.h"

namespace sb {
extern long long g_kernel_launches;

namespace {

constexpr int NT = 256;
constexpr int TJ = 8, TK = 32;
constexpr int RJ = TJ + 4, RK = TK + 4;  // staged planes: halo 2
constexpr int QJ = TJ + 2, QK = TK + 2;  // relaxed planes: halo 1
constexpr int PL = RJ * RK;              // doubles per staged plane
constexpr int QL = QJ * QK;
constexpr int RED_PER_ROW = QK / 2;      // 17

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

__device__ __forceinline__ int wrapc(int x, int n) {
  x %= n;
  return x < 0 ? x + n : x;
}
__device__ __forceinline__ int pmod(int x, int m) {
  x %= m;
  return x < 0 ? x + m : x;
}

struct Ext {
  int e[3];
  bool p[3];
};

// absolute coordinate -> array coordinate (wrapped), or -1 outside a wall axis
__device__ __forceinline__ int acoord(const Ext& E, const LevelDev& L, int a, int x) {
  if (E.p[a]) return wrapc(x, L.n[a]);
  return (x >= 0 && x < E.e[a]) ? x : -1;
}

// Per-CTA in-plane offset tables: tab[cls][t] = ja*s1 + ka of staged position
// t (halo 2, wraps applied) or -1 outside the array.  cls bit 0: the array has
// n1+1 entries along axis 1 (wall), bit 1: n2+1 along axis 2.  Plane-independent,
// so staging a plane is a table lookup + cp.async per element.
__device__ __forceinline__ void build_tabs(const LevelDev& L, int (*tab)[PL], int j0, int k0) {
  for (int t = threadIdx.x; t < 4 * PL; t += NT) {
    const int cls = t / PL, u = t - cls * PL;
    const int jj = u / RK, kk = u - jj * RK;
    int j = j0 - 2 + jj, k = k0 - 2 + kk;
    const int e1 = L.n[1] + ((cls & 1) && L.bclo[1] != BC_PER ? 1 : 0);
    const int e2 = L.n[2] + ((cls & 2) && L.bclo[2] != BC_PER ? 1 : 0);
    bool ok = true;
    if (L.bclo[1] == BC_PER) j = j < 0 ? j + L.n[1] : (j >= L.n[1] ? j - L.n[1] : j);
    else ok = ok && j >= 0 && j < e1;
    if (L.bclo[2] == BC_PER) k = k < 0 ? k + L.n[2] : (k >= L.n[2] ? k - L.n[2] : k);
    else ok = ok && k >= 0 && k < e2;
    tab[cls][u] = ok ? j * L.s1 + k : -1;
  }
}

// stage plane q (halo 2) of x into a shared slot; outside the array -> 0
__device__ __forceinline__ void stage(const LevelDev& L, const Ext& E, const int* tab, const double* x,
                                     double* slot, int q) {
  int qa = q;
  if (E.p[0]) qa = q < 0 ? q + L.n[0] : (q >= L.n[0] ? q - L.n[0] : q);
  else if (q < 0 || q >= E.e[0]) qa = -1;
  if (qa < 0) {
    for (int t = threadIdx.x; t < PL; t += NT) slot[t] = 0.0;
    return;
  }
  const double* xp = x + qa * L.s0;
  for (int t = threadIdx.x; t < PL; t += NT) {
    const int o = tab[t];
    if (o >= 0) cp_async8(slot + t, xp + o);
    else slot[t] = 0.0;
  }
}

template <int AX>
__host__ __device__ constexpr int cls_of_face() { return (AX == 1 ? 1 : 0) | (AX == 2 ? 2 : 0); }

// A staged operand: ring of NS planes; at step p its window is planes
// [p-1+LO, p+HI] and plane p+1+HI is in flight.
template <int LO, int HI>
struct Ring {
  static constexpr int NS = HI - LO + 3;
  double* base;
  const double* src;
  __device__ __forceinline__ double* slot(int q) const { return base + pmod(q, NS) * PL; }
};

// in-plane offset of +e_ax in the staged layout (axis 0 is the plane axis)
template <int AX>
__device__ __forceinline__ constexpr int inplane() { return AX == 1 ? RK : (AX == 2 ? 1 : 0); }

// Shared-memory accessor with the GAcc interface (sb_device.cuh) for a face
// of component A on plane pp at staged-layout index o.
template <int A, class RUB1, class RUB2, class RMU, class RME1, class RME2>
struct SAcc {
  static constexpr int B1 = A == 0 ? 1 : 0, B2 = A == 2 ? 1 : 2;
  const RUB1& ub1;
  const RUB2& ub2;
  const RMU& rmu;
  const RME1& me1;
  const RME2& me2;
  const double* rho0;
  int pp, o;
  // value of ring R at (plane pp + dp, index o + di)
  template <class R>
  __device__ __forceinline__ double at(const R& r, int dp, int di) const {
    return r.slot(pp + dp)[o + di];
  }
  __device__ __forceinline__ double mu(bool lo) const {
    return lo ? (A == 0 ? at(rmu, -1, 0) : at(rmu, 0, -inplane<A>())) : at(rmu, 0, 0);
  }
  __device__ __forceinline__ double gam(bool) const { return 0.0; }  // stress+bulk not staged
  __device__ __forceinline__ double divh(bool) const { return 0.0; }
  template <int B>
  __device__ __forceinline__ double mue(bool hi) const {
    const int dp = (hi && B == 0) ? 1 : 0, di = hi ? inplane<B>() : 0;
    return B == B1 ? at(me1, dp, di) : at(me2, dp, di);
  }
  template <int B>
  __device__ __forceinline__ double ub(bool hi, bool lowA) const {
    const int dp = ((hi && B == 0) ? 1 : 0) + ((lowA && A == 0) ? -1 : 0);
    const int di = (hi ? inplane<B>() : 0) - (lowA ? inplane<A>() : 0);
    return B == B1 ? at(ub1, dp, di) : at(ub2, dp, di);
  }
  __device__ __forceinline__ double rho() const { return rho0[o]; }
};

template <int AX, int BB>
struct LoOf {  // window low offset of u_B / mu_c for component AX (A==0 reads plane -1)
  static constexpr int v = AX == 0 ? -1 : 0;
};

template <int FORM, int A, bool TH>
__global__ void __launch_bounds__(NT)
k_face_sweep2(LevelDev L, CPtr3 u, double* __restrict__ unew, const double* __restrict__ rhs, double omega,
              int chunk) {
  constexpr int B1 = A == 0 ? 1 : 0, B2 = A == 2 ? 1 : 2;
  constexpr int LA = A == 0 ? -1 : 0;
  extern __shared__ double smem[];
  __shared__ int tab[4][PL];
  Ring<0, 1> rx;                            // u_A (old), red window [p-1, p+1]
  Ring<LA, B1 == 0 ? 1 : 0> rb1;            // u_B1
  Ring<LA, 0> rb2;                          // u_B2 (B2 is never axis 0)
  Ring<LA, 0> rmu;                          // mu_c
  Ring<0, B1 == 0 ? 1 : 0> re1;             // mu_e(A, B1)
  Ring<0, 0> re2;                           // mu_e(A, B2)
  Ring<0, 0> rrhs;                          // rhs_A
  Ring<0, 0> rrho;                          // rho_A (theta > 0)
  double* sp = smem;
  rx.base = sp; sp += decltype(rx)::NS * PL;
  rb1.base = sp; sp += decltype(rb1)::NS * PL;
  rb2.base = sp; sp += decltype(rb2)::NS * PL;
  rmu.base = sp; sp += decltype(rmu)::NS * PL;
  re1.base = sp; sp += decltype(re1)::NS * PL;
  re2.base = sp; sp += decltype(re2)::NS * PL;
  rrhs.base = sp; sp += decltype(rrhs)::NS * PL;
  rrho.base = sp; if (TH) sp += decltype(rrho)::NS * PL;
  double* sr = sp;  // 3 relaxed planes (halo 1)
  rx.src = u.p[A];
  rb1.src = u.p[B1];
  rb2.src = u.p[B2];
  rmu.src = L.mu_c;
  re1.src = L.mu_e[edge_of(A, B1)];
  re2.src = L.mu_e[edge_of(A, B2)];
  rrhs.src = rhs;
  rrho.src = L.rho_f[A];

  Ext E;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    E.p[a] = per(L, a);
    E.e[a] = L.n[a] + ((a == A && !E.p[a]) ? 1 : 0);
  }
  // staging extents: face arrays of B carry +1 along their own wall axis; the
  // other operands are cell/edge shaped -- the pitched box covers them all, so
  // stage with the extents of the array actually read.
  Ext EB1 = E, EB2 = E, EC = E, EE1 = E, EE2 = E;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    EB1.e[a] = L.n[a] + ((a == B1 && !E.p[a]) ? 1 : 0);
    EB2.e[a] = L.n[a] + ((a == B2 && !E.p[a]) ? 1 : 0);
    EC.e[a] = L.n[a];
    EE1.e[a] = L.n[a] + (((a == A || a == B1) && !E.p[a]) ? 1 : 0);
    EE2.e[a] = L.n[a] + (((a == A || a == B2) && !E.p[a]) ? 1 : 0);
  }
  const int off = E.p[A] ? 0 : 1;  // interior-relative parity offset (multigrid.py:335-339)
  const int k0 = blockIdx.x * TK, j0 = blockIdx.y * TJ;
  const int i0 = blockIdx.z * chunk, i1 = min(i0 + chunk, E.e[0]) - 1;
  auto unknown = [&](const int* ca) { return E.p[A] || (ca[A] != 0 && ca[A] != L.n[A]); };

  build_tabs(L, tab, j0, k0);
  __syncthreads();
  // table class per operand: which of axes 1/2 it is staggered along
  constexpr int cA = cls_of_face<A>(), cB1 = cls_of_face<B1>(), cB2 = cls_of_face<B2>();
  auto stage_plane = [&](int q, auto& r, const Ext& Ex, int cls) { stage(L, Ex, tab[cls], r.src, r.slot(q), q); };
  // prologue: window of step i0-1
  for (int q = i0 - 2 + 0; q <= i0 - 1 + 1; ++q) stage_plane(q, rx, E, cA);
  for (int q = i0 - 2 + LA; q <= i0 - 1 + (B1 == 0 ? 1 : 0); ++q) stage_plane(q, rb1, EB1, cB1);
  for (int q = i0 - 2 + LA; q <= i0 - 1; ++q) stage_plane(q, rb2, EB2, cB2);
  for (int q = i0 - 2 + LA; q <= i0 - 1; ++q) stage_plane(q, rmu, EC, 0);
  for (int q = i0 - 2; q <= i0 - 1 + (B1 == 0 ? 1 : 0); ++q) stage_plane(q, re1, EE1, cA | cB1);
  for (int q = i0 - 2; q <= i0 - 1; ++q) stage_plane(q, re2, EE2, cA | cB2);
  for (int q = i0 - 2; q <= i0 - 1; ++q) stage_plane(q, rrhs, E, cA);
  if (TH)
    for (int q = i0 - 2; q <= i0 - 1; ++q) stage_plane(q, rrho, E, cA);
  cp_commit();

  for (int p = i0 - 1; p <= i1 + 1; ++p) {
    // prefetch the newest plane of every window for step p+1
    stage_plane(p + 2, rx, E, cA);
    stage_plane(p + 1 + (B1 == 0 ? 1 : 0), rb1, EB1, cB1);
    stage_plane(p + 1, rb2, EB2, cB2);
    stage_plane(p + 1, rmu, EC, 0);
    stage_plane(p + 1 + (B1 == 0 ? 1 : 0), re1, EE1, cA | cB1);
    stage_plane(p + 1, re2, EE2, cA | cB2);
    stage_plane(p + 1, rrhs, E, cA);
    if (TH) stage_plane(p + 1, rrho, E, cA);
    cp_commit();
    cp_wait1();
    __syncthreads();
    // ---- R_p: relax the red unknowns of plane p on the tile + ring 1 ----
    double* R = sr + pmod(p, 3) * QL;
    {
      const double* O0 = rx.slot(p - 1);
      const double* O1 = rx.slot(p);
      const double* O2 = rx.slot(p + 1);
      for (int q = threadIdx.x; q < QL; q += NT) {  // start from the old plane
        const int jj = q / QK, kk = q - jj * QK;
        R[q] = O1[(jj + 1) * RK + (kk + 1)];
      }
      __syncthreads();
      const int pa = acoord(E, L, 0, p);
      if (pa >= 0) {
        for (int q = threadIdx.x; q < QJ * RED_PER_ROW; q += NT) {  // lanes on red faces only
          const int jj = q / RED_PER_ROW, m = q - jj * RED_PER_ROW;
          const int j = j0 - 1 + jj;
          const int kk = ((off - p - j - (k0 - 1)) & 1) + 2 * m;
          const int k = k0 - 1 + kk;
          const int ca[3] = {pa, acoord(E, L, 1, j), acoord(E, L, 2, k)};
          if (ca[1] < 0 || ca[2] < 0 || !unknown(ca)) continue;
          const int o = (jj + 1) * RK + (kk + 1);
          UA7 s;
          s.c = O1[o];
          s.p[0] = O2[o];
          s.m[0] = O0[o];
          s.p[1] = O1[o + RK];
          s.m[1] = O1[o - RK];
          s.p[2] = O1[o + 1];
          s.m[2] = O1[o - 1];
          const SAcc<A, decltype(rb1), decltype(rb2), decltype(rmu), decltype(re1), decltype(re2)> acc{
              rb1, rb2, rmu, re1, re2, rrho.slot(p), p, o};
          double dg;
          const double au = face_row_t<3, FORM, A, false>(L, s, acc, ca, dg);
          const double res = rrhs.slot(p)[o] - au;
          R[jj * QK + kk] = s.c + omega * (res / dg);
        }
      }
    }
    __syncthreads();
    // ---- black unknowns of plane p-1 (tile) from R_{p-2}, R_{p-1}, R_p ----
    const int pb = p - 1;
    if (pb >= i0 && pb <= i1) {
      double* Rm = sr + pmod(pb, 3) * QL;
      const double* Rlo = sr + pmod(pb - 1, 3) * QL;
      const double* Rhi = sr + pmod(pb + 1, 3) * QL;
      const int pa = acoord(E, L, 0, pb);
      for (int q = threadIdx.x; q < TJ * (TK / 2); q += NT) {
        const int jj = q / (TK / 2), m = q - jj * (TK / 2);
        const int j = j0 + jj;
        const int k = k0 + ((1 + off - pb - j - k0) & 1) + 2 * m;  // black: parity 1
        const int ca[3] = {pa, j, k};
        if (j >= E.e[1] || k >= E.e[2] || !unknown(ca)) continue;
        const int oq = (jj + 1) * QK + (k - k0 + 1);
        UA7 s;
        s.c = Rm[oq];
        s.p[0] = Rhi[oq];
        s.m[0] = Rlo[oq];
        s.p[1] = Rm[oq + QK];
        s.m[1] = Rm[oq - QK];
        s.p[2] = Rm[oq + 1];
        s.m[2] = Rm[oq - 1];
        const int o = (jj + 2) * RK + (k - k0 + 2);
        const SAcc<A, decltype(rb1), decltype(rb2), decltype(rmu), decltype(re1), decltype(re2)> acc{
            rb1, rb2, rmu, re1, re2, rrho.slot(pb), pb, o};
        double dg;
        const double au = face_row_t<3, FORM, A, false>(L, s, acc, ca, dg);
        const double res = rrhs.slot(pb)[o] - au;
        Rm[oq] = s.c + omega * (res / dg);
      }
      __syncthreads();
      for (int q = threadIdx.x; q < TJ * TK; q += NT) {  // write plane pb, coalesced along k
        const int jj = q / TK, kk = q - jj * TK;
        const int j = j0 + jj, k = k0 + kk;
        if (j < E.e[1] && k < E.e[2]) unew[pa * L.s0 + j * L.s1 + k] = Rm[(jj + 1) * QK + kk + 1];
      }
    }
  }
}

// beta accessor over staged rings: beta_a at the low / high face of cell (pp, o)
template <class R0, class R1, class R2>
struct SBeta {
  const R0& b0;
  const R1& b1;
  const R2& b2;
  int pp, o;
  template <int AX>
  __device__ __forceinline__ double beta(bool hi) const {
    if (AX == 0) return b0.slot(pp + (hi ? 1 : 0))[o];
    if (AX == 1) return b1.slot(pp)[o + (hi ? RK : 0)];
    return b2.slot(pp)[o + (hi ? 1 : 0)];
  }
};

__global__ void __launch_bounds__(NT)
k_cell_sweep2(LevelDev L, const double* __restrict__ phi, double* __restrict__ pnew,
              const double* __restrict__ rhs, double omega, int chunk) {
  extern __shared__ double smem[];
  __shared__ int tab[4][PL];
  Ring<0, 1> rx;    // phi (old)
  Ring<0, 1> rb0;   // beta_0 (reads plane +1)
  Ring<0, 0> rb1;   // beta_1
  Ring<0, 0> rb2;   // beta_2
  Ring<0, 0> rrhs;
  double* sp = smem;
  rx.base = sp; sp += decltype(rx)::NS * PL;
  rb0.base = sp; sp += decltype(rb0)::NS * PL;
  rb1.base = sp; sp += decltype(rb1)::NS * PL;
  rb2.base = sp; sp += decltype(rb2)::NS * PL;
  rrhs.base = sp; sp += decltype(rrhs)::NS * PL;
  double* sr = sp;
  rx.src = phi;
  rb0.src = L.beta_f[0];
  rb1.src = L.beta_f[1];
  rb2.src = L.beta_f[2];
  rrhs.src = rhs;
  Ext E, F0, F1, F2;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    E.p[a] = per(L, a);
    E.e[a] = L.n[a];
  }
  F0 = F1 = F2 = E;
  if (!E.p[0]) F0.e[0] += 1;
  if (!E.p[1]) F1.e[1] += 1;
  if (!E.p[2]) F2.e[2] += 1;
  const int k0 = blockIdx.x * TK, j0 = blockIdx.y * TJ;
  const int i0 = blockIdx.z * chunk, i1 = min(i0 + chunk, E.e[0]) - 1;
  build_tabs(L, tab, j0, k0);
  __syncthreads();
  auto stage_plane = [&](int q, auto& r, const Ext& Ex, int cls) { stage(L, Ex, tab[cls], r.src, r.slot(q), q); };
  for (int q = i0 - 2; q <= i0; ++q) stage_plane(q, rx, E, 0);
  for (int q = i0 - 2; q <= i0; ++q) stage_plane(q, rb0, F0, 0);
  for (int q = i0 - 2; q <= i0 - 1; ++q) stage_plane(q, rb1, F1, 1);
  for (int q = i0 - 2; q <= i0 - 1; ++q) stage_plane(q, rb2, F2, 2);
  for (int q = i0 - 2; q <= i0 - 1; ++q) stage_plane(q, rrhs, E, 0);
  cp_commit();

  for (int p = i0 - 1; p <= i1 + 1; ++p) {
    stage_plane(p + 2, rx, E, 0);
    stage_plane(p + 2, rb0, F0, 0);
    stage_plane(p + 1, rb1, F1, 1);
    stage_plane(p + 1, rb2, F2, 2);
    stage_plane(p + 1, rrhs, E, 0);
    cp_commit();
    cp_wait1();
    __syncthreads();
    double* R = sr + pmod(p, 3) * QL;
    {
      const double* O0 = rx.slot(p - 1);
      const double* O1 = rx.slot(p);
      const double* O2 = rx.slot(p + 1);
      for (int q = threadIdx.x; q < QL; q += NT) {
        const int jj = q / QK, kk = q - jj * QK;
        R[q] = O1[(jj + 1) * RK + (kk + 1)];
      }
      __syncthreads();
      const int pa = acoord(E, L, 0, p);
      if (pa >= 0) {
        for (int q = threadIdx.x; q < QJ * RED_PER_ROW; q += NT) {
          const int jj = q / RED_PER_ROW, m = q - jj * RED_PER_ROW;
          const int j = j0 - 1 + jj;
          const int kk = ((-p - j - (k0 - 1)) & 1) + 2 * m;
          const int k = k0 - 1 + kk;
          const int ca[3] = {pa, acoord(E, L, 1, j), acoord(E, L, 2, k)};
          if (ca[1] < 0 || ca[2] < 0) continue;
          const int o = (jj + 1) * RK + (kk + 1);
          UA7 s;
          s.c = O1[o];
          s.p[0] = O2[o];
          s.m[0] = O0[o];
          s.p[1] = O1[o + RK];
          s.m[1] = O1[o - RK];
          s.p[2] = O1[o + 1];
          s.m[2] = O1[o - 1];
          const SBeta<decltype(rb0), decltype(rb1), decltype(rb2)> ba{rb0, rb1, rb2, p, o};
          double dg;
          const double lp = cell_row_t<3, false>(L, s, ba, ca, dg);
          const double res = rrhs.slot(p)[o] - lp;
          R[jj * QK + kk] = s.c + omega * res / dg;
        }
      }
    }
    __syncthreads();
    const int pb = p - 1;
    if (pb >= i0 && pb <= i1) {
      double* Rm = sr + pmod(pb, 3) * QL;
      const double* Rlo = sr + pmod(pb - 1, 3) * QL;
      const double* Rhi = sr + pmod(pb + 1, 3) * QL;
      for (int q = threadIdx.x; q < TJ * (TK / 2); q += NT) {
        const int jj = q / (TK / 2), m = q - jj * (TK / 2);
        const int j = j0 + jj;
        const int k = k0 + ((1 - pb - j - k0) & 1) + 2 * m;
        if (j >= E.e[1] || k >= E.e[2]) continue;
        const int ca[3] = {pb, j, k};
        const int oq = (jj + 1) * QK + (k - k0 + 1);
        UA7 s;
        s.c = Rm[oq];
        s.p[0] = Rhi[oq];
        s.m[0] = Rlo[oq];
        s.p[1] = Rm[oq + QK];
        s.m[1] = Rm[oq - QK];
        s.p[2] = Rm[oq + 1];
        s.m[2] = Rm[oq - 1];
        const int o = (jj + 2) * RK + (k - k0 + 2);
        const SBeta<decltype(rb0), decltype(rb1), decltype(rb2)> ba{rb0, rb1, rb2, pb, o};
        double dg;
        const double lp = cell_row_t<3, false>(L, s, ba, ca, dg);
        const double res = rrhs.slot(pb)[o] - lp;
        Rm[oq] = s.c + omega * res / dg;
      }
      __syncthreads();
      for (int q = threadIdx.x; q < TJ * TK; q += NT) {
        const int jj = q / TK, kk = q - jj * TK;
        const int j = j0 + jj, k = k0 + kk;
        if (j < E.e[1] && k < E.e[2]) pnew[pb * L.s0 + j * L.s1 + k] = Rm[(jj + 1) * QK + kk + 1];
      }
    }
  }
}

inline dim3 sweep_grid(int e0, int e1, int e2, int ctas_per_sm, int& chunk) {
  const int gx = (e2 + TK - 1) / TK, gy = (e1 + TJ - 1) / TJ;
  const int cols = gx * gy;
  int nch = std::max(1, std::min(e0 / 16, (148 * ctas_per_sm + cols - 1) / cols));
  chunk = (e0 + nch - 1) / nch;
  nch = (e0 + chunk - 1) / chunk;
  return dim3(gx, gy, nch);
}

template <int FORM, int A, bool TH>
size_t face_smem() {
  constexpr int B1 = A == 0 ? 1 : 0;
  constexpr int LA = A == 0 ? -1 : 0;
  const int slots = Ring<0, 1>::NS + Ring<LA, B1 == 0 ? 1 : 0>::NS + 2 * Ring<LA, 0>::NS +
                    Ring<0, B1 == 0 ? 1 : 0>::NS + Ring<0, 0>::NS * (TH ? 3 : 2);
  return (size_t)(slots * PL + 3 * QL) * sizeof(double);
}

template <int FORM, int A, bool TH>
void launch_face_t(cudaStream_t s, const LevelDev& L, CPtr3 u, double* unew, const double* rhsA, double omega) {
  static bool configured = false;
  const size_t sm = face_smem<FORM, A, TH>();
  if (!configured) {
    cudaFuncSetAttribute(k_face_sweep2<FORM, A, TH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    configured = true;
  }
  int e[3];
  for (int a = 0; a < 3; ++a) e[a] = L.n[a] + ((a == A && L.bclo[a] != BC_PER) ? 1 : 0);
  int chunk;
  const dim3 g = sweep_grid(e[0], e[1], e[2], sm > 100 * 1024 ? 1 : 2, chunk);
  k_face_sweep2<FORM, A, TH><<<g, NT, sm, s>>>(L, u, unew, rhsA, omega, chunk);
}

template <int FORM, int A>
void launch_face_a(cudaStream_t s, const LevelDev& L, CPtr3 u, double* unew, const double* rhsA, double omega) {
  if (L.theta > 0.0) launch_face_t<FORM, A, true>(s, L, u, unew, rhsA, omega);
  else launch_face_t<FORM, A, false>(s, L, u, unew, rhsA, omega);
}

}  // namespace

bool sweep2_supported(const LevelDev& L, int dim, int form) {
  if (dim != 3 || form == F_BULK || L.dist0) return false;
  for (int a = 0; a < 3; ++a)
    if (L.n[a] < 8 || (L.bclo[a] == BC_PER && (L.n[a] & 1))) return false;
  return true;
}

void launch_face_sweep2(cudaStream_t s, const LevelDev& L, int form, int A, CPtr3 u, double* unew,
                        const double* rhsA, double omega) {
  ++g_kernel_launches;
  if (form == F_LAP) {
    if (A == 0) launch_face_a<F_LAP, 0>(s, L, u, unew, rhsA, omega);
    else if (A == 1) launch_face_a<F_LAP, 1>(s, L, u, unew, rhsA, omega);
    else launch_face_a<F_LAP, 2>(s, L, u, unew, rhsA, omega);
  } else {
    if (A == 0) launch_face_a<F_STRESS, 0>(s, L, u, unew, rhsA, omega);
    else if (A == 1) launch_face_a<F_STRESS, 1>(s, L, u, unew, rhsA, omega);
    else launch_face_a<F_STRESS, 2>(s, L, u, unew, rhsA, omega);
  }
}

void launch_cell_sweep2(cudaStream_t s, const LevelDev& L, const double* phi, double* pnew, const double* rhs,
                        double omega) {
  ++g_kernel_launches;
  static bool configured = false;
  const size_t sm = (size_t)((Ring<0, 1>::NS * 2 + Ring<0, 0>::NS * 3) * PL + 3 * QL) * sizeof(double);
  if (!configured) {
    cudaFuncSetAttribute(k_cell_sweep2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    configured = true;
  }
  int chunk;
  const dim3 g = sweep_grid(L.n[0], L.n[1], L.n[2], 3, chunk);
  k_cell_sweep2<<<g, NT, sm, s>>>(L, phi, pnew, rhs, omega, chunk);
}

}  // namespace sb
