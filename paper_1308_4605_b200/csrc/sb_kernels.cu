// sb_kernels.cu -- sm_100a fp64 kernels of the preconditioned MAC-Stokes solve.
//
// Every kernel here is HBM-bound stencil / streaming work (0.5-1 flop per
// byte, far below the fp64 ridge), so the design rules are coalesced
// contiguous-axis access, on-chip reuse of stencil neighbours (L1/L2), grids
// sized to the 148 SMs and deterministic reductions.  Arithmetic follows the
// reference's operation order (see sb_device.cuh) so results agree with the
// NumPy reference to a few ulp.
#include <cuda_runtime.h>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include "sb_kernels.h"

namespace sb {

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SB_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

namespace {

constexpr int kThreads = 256;
constexpr int kSMs = 148;

inline int grid_for(long long total, int per_block = kThreads, int max_blocks = kSMs * 16) {
  long long b = (total + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

// 3D launch over a box: x -> axis 2 (contiguous), y -> axis 1, z -> axis 0.
// No div/mod in the kernels; one point per thread.
__device__ __forceinline__ bool box_point(const Box& b, int* ci) {
  ci[2] = b.lo[2] + (int)(blockIdx.x * blockDim.x + threadIdx.x);
  ci[1] = b.lo[1] + (int)(blockIdx.y * blockDim.y + threadIdx.y);
  ci[0] = b.lo[0] + (int)blockIdx.z;
  return ci[2] <= b.hi[2] && ci[1] <= b.hi[1];
}

struct L3 {
  dim3 g, b;
};
inline L3 cfg3(int e0, int e1, int e2) {
  int bx = 32;
  while (bx > 1 && bx / 2 >= e2) bx >>= 1;
  int by = kThreads / bx;
  while (by > 1 && by / 2 >= e1) by >>= 1;
  L3 c;
  c.b = dim3(bx, by, 1);
  c.g = dim3((e2 + bx - 1) / bx, (e1 + by - 1) / by, e0);
  return c;
}
inline L3 cfg3(const Box& b) {
  return cfg3(b.hi[0] - b.lo[0] + 1, b.hi[1] - b.lo[1] + 1, b.hi[2] - b.lo[2] + 1);
}

inline unsigned box_count(const Box& b) {
  return (unsigned)(b.hi[0] - b.lo[0] + 1) * (unsigned)(b.hi[1] - b.lo[1] + 1) *
         (unsigned)(b.hi[2] - b.lo[2] + 1);
}

__device__ __forceinline__ int lin(const LevelDev& L, const int* ci) {
  return ci[0] * L.s0 + ci[1] * L.s1 + ci[2];
}

// unknown faces of component A (wall axis A: 1..n_A-1)
__host__ __device__ inline Box face_box(const LevelDev& L, int dim, int A) {
  Box b;
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = 0;
    b.hi[a] = L.n[a] - 1;
  }
  if (L.bclo[A] != BC_PER) {
    b.lo[A] = 1;
    b.hi[A] = L.n[A] - 1;
  }
  (void)dim;
  return b;
}
__host__ __device__ inline Box cell_box(const LevelDev& L) {
  Box b;
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = 0;
    b.hi[a] = L.n[a] - 1;
  }
  return b;
}

template <int DIM, int A>
struct Others;  // the tangential axes of component A, ascending
template <> struct Others<3, 0> { static constexpr int B1 = 1, B2 = 2; };
template <> struct Others<3, 1> { static constexpr int B1 = 0, B2 = 2; };
template <> struct Others<3, 2> { static constexpr int B1 = 0, B2 = 1; };
template <> struct Others<2, 1> { static constexpr int B1 = 2, B2 = -1; };
template <> struct Others<2, 2> { static constexpr int B1 = 1, B2 = -1; };

// ---------------------------------------------------------------------------
// colour passes (multigrid.py:318-340)
// ---------------------------------------------------------------------------

// One GS colour pass of component A.  Thread t owns the t-th same-colour face
// of a row along the contiguous axis.  TWO_PHASE (odd periodic extents, where
// same-colour faces couple through the wrap): phase 0 stores the new values in
// tmp, phase 1 copies them in -- exactly the reference's compute-all-then-
// update-masked order.
//
// Z (first sweep of a V-cycle level, x = 0 on entry): 1 = the components after
// A are still zero (their loads are skipped); 2 = also u_A itself (first colour
// of A: no u loads at all); 3 = as 2 and the pass also stores the zero of the
// other-colour partner face (k ^ 1), which replaces the level's zero fill on
// all-periodic pad-free levels (every block entry is then written).  Same
// arithmetic on the same values as the plain pass: bit-identical.
// L2 prefetch distance of the colour passes in planes (ncu, C5 256^3, finest face
// pass of components 0 / 1 / 2: off 157 / 158 / 161 us, 1: 142 / 138 / 144,
// 2: 140 / 137 / 143, 4: 141 / 136 / 144)
#ifndef FC_PF
#define FC_PF 2
#endif
// this thread's column FC_PF planes ahead of plane i0 (see k_face_colour)
__device__ __forceinline__ void pf_plane(const double* p, int idx) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p + idx));
}
template <int A>
__host__ __device__ constexpr int later_mask() { return A == 0 ? 6 : (A == 1 ? 4 : 0); }

template <int DIM, int FORM, int A, int PHASE, int PA, bool DE = false, int Z = 0>
__global__ void __launch_bounds__(kThreads)
k_face_colour(LevelDev L, Ptr3 u, const double* __restrict__ rhs, double* tmp, int parity,
              double omega, Box b, unsigned half2, unsigned total) {
  pdl_enter();
  const int off = (L.bclo[A] == BC_PER) ? 0 : 1;
  {
    int ci[3];
    const int tt = (int)(blockIdx.x * blockDim.x + threadIdx.x);
    ci[1] = b.lo[1] + (int)(blockIdx.y * blockDim.y + threadIdx.y);
    ci[0] = b.lo[0] + (int)blockIdx.z;
    if (ci[1] > b.hi[1]) return;
    const int k = b.lo[2] + ((parity + off - ci[0] - ci[1] - b.lo[2]) & 1) + 2 * tt;
    if (k > b.hi[2]) return;
    ci[2] = k;
    const int f = lin(L, ci);
    if (PHASE == 1) {
      u.p[A][f] = tmp[f];
      return;
    }
    const double* uc[3] = {u.p[0], u.p[1], u.p[2]};
    double dg;
    if (Z >= 2) {
      constexpr int ZM = later_mask<A>() | (1 << A);
#if FC_PF > 0
      // zero-first pass: only the arrays it reads (mu_c, rhs, the components
      // relaxed before A) are worth asking for
      if (DIM == 3 && DE && ci[0] + FC_PF <= b.hi[0]) {
        const int fp = f + FC_PF * L.s0;
        pf_plane(L.mu_c, fp);
        pf_plane(rhs, fp);
        if (A > 0) pf_plane(uc[0], fp);
        if (A > 1) pf_plane(uc[1], fp);
      }
#endif
      UA7 s0;
      s0.c = 0.0;
#pragma unroll
      for (int q = 0; q < 3; ++q) s0.p[q] = s0.m[q] = 0.0;
      const double au = face_row_core<DIM, FORM, A, PA, true, DE, ZM>(L, s0, uc, f, ci, dg);
      const double res = __ldg(rhs + f) - au;
      u.p[A][f] = s0.c + omega * (res / dg);
      if (Z == 3) u.p[A][(k & 1) ? f - 1 : f + 1] = 0.0;
      return;
    }
    constexpr int ZM = Z == 1 ? later_mask<A>() : 0;
#if FC_PF > 0
    // planes are scheduled in ascending order (blockIdx.z): ask L2 for this
    // thread's column FC_PF planes ahead, where later CTAs read it first.  Only
    // the derived-mu_e row, which is latency / L1 bound (C5: 157-161 -> 137-143 us
    // per finest pass); the stored-mu_e row already saturates HBM and the
    // extra requests cost it 3 % (C4: 198 / 198 / 181 -> 197 / 204 / 187 us)
    if (DIM == 3 && DE && Z <= 1 && ci[0] + FC_PF <= b.hi[0]) {
      const int fp = f + FC_PF * L.s0;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(uc[0] + fp));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(uc[1] + fp));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(uc[2] + fp));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(L.mu_c + fp));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(rhs + fp));
    }
#endif
    const double au =
        face_row_core<DIM, FORM, A, PA, true, DE, ZM>(L, gather_ua<DIM, A, PA>(L, uc[A], f, ci), uc, f, ci, dg);
    const double res = __ldg(rhs + f) - au;
    const double nv = uc[A][f] + omega * (res / dg);
    if (PHASE == 2) tmp[f] = nv;
    else u.p[A][f] = nv;
  }
}

template <int DIM, int PHASE, int PA, int Z = 0>
__global__ void __launch_bounds__(kThreads)
k_cell_colour(LevelDev L, double* phi, const double* __restrict__ rhs, double* tmp, int parity,
              double omega, Box b, unsigned half2, unsigned total) {
  pdl_enter();
  {
    int ci[3];
    const int tt = (int)(blockIdx.x * blockDim.x + threadIdx.x);
    ci[1] = b.lo[1] + (int)(blockIdx.y * blockDim.y + threadIdx.y);
    ci[0] = b.lo[0] + (int)blockIdx.z;
    if (ci[1] > b.hi[1]) return;
    const int k = b.lo[2] + ((parity - ci[0] - ci[1] - b.lo[2]) & 1) + 2 * tt;
    if (k > b.hi[2]) return;
    ci[2] = k;
    const int c = lin(L, ci);
    if (PHASE == 1) {
      phi[c] = tmp[c];
      return;
    }
    double dg;
    if (Z >= 2) {  // first colour of a V-cycle level from phi = 0 (see k_face_colour)
      UA7 s0;
      s0.c = 0.0;
#pragma unroll
      for (int q = 0; q < 3; ++q) s0.p[q] = s0.m[q] = 0.0;
      const double lp = cell_row_core<DIM, PA>(L, s0, c, ci, dg);
      const double res = __ldg(rhs + c) - lp;
      phi[c] = s0.c + omega * res / dg;
      if (Z == 3) phi[(k & 1) ? c - 1 : c + 1] = 0.0;
      return;
    }
#if FC_PF > 0
    // as k_face_colour: this column, FC_PF planes ahead (C4, streamed 1/rho:
    // 136 -> 121 us per finest pass; C5, constant 1/rho: 64 -> 63 us)
    if (DIM == 3 && ci[0] + FC_PF <= b.hi[0]) {
      const int cp = c + FC_PF * L.s0;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(phi + cp));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(rhs + cp));
      if (!L.beta_const) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(L.beta_f[0] + cp));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(L.beta_f[1] + cp));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(L.beta_f[2] + cp));
      }
    }
#endif
    const double lp = cell_row<DIM, PA>(L, phi, c, ci, dg);
    const double res = __ldg(rhs + c) - lp;
    const double nv = phi[c] + omega * res / dg;
    if (PHASE == 2) tmp[c] = nv;
    else phi[c] = nv;
  }
}

// ---------------------------------------------------------------------------
// residual -> restriction (multigrid.py:195-233, 177-182, 403-406)
// ---------------------------------------------------------------------------

template <int DIM, int FORM, int A, int PA, bool NC = true>
__device__ __forceinline__ double face_resid_at(const LevelDev& L, const double* const* u,
                                                const double* rhs, const int* ci) {
  const int f = lin(L, ci);
  double dg;
  const double au = face_row<DIM, FORM, A, PA, NC>(L, u, f, ci, dg);
  return (NC ? __ldg(rhs + f) : rhs[f]) - au;
}

// Tangential 2^(d-1) mean of fine residuals at fine normal index fa, coarse
// tangential indices in C (mean along B1 first, then B2: multigrid.py:112-119).
template <int DIM, int FORM, int A, int PA, bool NC = true>
__device__ __forceinline__ double tmean_resid(const LevelDev& Lf, const double* const* u, const double* rhs,
                                              const int* C, int fa) {
  using O = Others<DIM, A>;
  int fi[3] = {2 * C[0], 2 * C[1], 2 * C[2]};
  if (DIM == 2) fi[0] = 0;
  fi[A] = fa;
  if (DIM == 3) {
    double p[2];
#pragma unroll 1
    for (int t2 = 0; t2 < 2; ++t2) {
      int q0[3] = {fi[0], fi[1], fi[2]}, q1[3] = {fi[0], fi[1], fi[2]};
      q0[O::B2] += t2;
      q1[O::B2] += t2;
      q1[O::B1] += 1;
      const double m0 = face_resid_at<DIM, FORM, A, PA, NC>(Lf, u, rhs, q0);
      const double m1 = face_resid_at<DIM, FORM, A, PA, NC>(Lf, u, rhs, q1);
      p[t2] = 0.5 * (m0 + m1);
    }
    return 0.5 * (p[0] + p[1]);
  }
  int q1[3] = {fi[0], fi[1], fi[2]};
  q1[O::B1] += 1;
  const double m0 = face_resid_at<DIM, FORM, A, PA, NC>(Lf, u, rhs, fi);
  const double m1 = face_resid_at<DIM, FORM, A, PA, NC>(Lf, u, rhs, q1);
  return 0.5 * (m0 + m1);
}

// Small levels: one thread per coarse face, all 3 (or 2D: 3) normal offsets
// evaluated by that thread (fine residuals on odd normal planes computed twice;
// parallelism matters more than redundancy below ~32^3).
template <int DIM, int FORM, int A, int PA>
__global__ void __launch_bounds__(kThreads)
k_face_rr_s(LevelDev Lf, LevelDev Lc, CPtr3 u, const double* __restrict__ rhs, double* __restrict__ coarse,
            Box cb, unsigned total) {
  pdl_enter();
  int C[3];
  if (!box_point(cb, C)) return;
  double tv[3];
#pragma unroll 1
  for (int o = -1; o <= 1; ++o) {
    int fa = 2 * C[A] + o;
    if (fa < 0 && !(A == 0 && Lf.dist0)) fa += Lf.n[A];
    tv[o + 1] = tmean_resid<DIM, FORM, A, PA>(Lf, u.p, rhs, C, fa);
  }
  coarse[lin(Lc, C)] = (0.25 * tv[0] + 0.5 * tv[1]) + 0.25 * tv[2];
}

// Fused residual -> restriction, each fine residual evaluated once.
// A == 2 (contiguous axis): lanes run along coarse K; t(2K-1) is the previous
// lane's t(2K+1) (warp shuffle), lane 0 evaluates it itself.
template <int DIM, int FORM, int PA>
__global__ void __launch_bounds__(kThreads)
k_face_rr_c(LevelDev Lf, LevelDev Lc, CPtr3 u, const double* __restrict__ rhs, double* __restrict__ coarse,
            Box cb) {
  pdl_enter();
  constexpr int A = 2;
  int C[3];
  C[2] = cb.lo[2] + (int)(blockIdx.x * blockDim.x + threadIdx.x);
  C[1] = cb.lo[1] + (int)(blockIdx.y * blockDim.y + threadIdx.y);
  C[0] = cb.lo[0] + (int)blockIdx.z;
  const bool ok = C[2] <= cb.hi[2] && C[1] <= cb.hi[1];
  int Cs[3] = {C[0], ok ? C[1] : cb.lo[1], ok ? C[2] : cb.lo[2]};
  const double t0 = tmean_resid<DIM, FORM, A, PA>(Lf, u.p, rhs, Cs, 2 * Cs[A]);
  const double t1 = tmean_resid<DIM, FORM, A, PA>(Lf, u.p, rhs, Cs, 2 * Cs[A] + 1);
  double tm = __shfl_up_sync(0xffffffffu, t1, 1);
  const int lane = threadIdx.x & 31;
  if (lane == 0 || Cs[A] == cb.lo[A]) {
    int fa = 2 * Cs[A] - 1;
    if (fa < 0 && !(A == 0 && Lf.dist0)) fa += Lf.n[A];
    tm = tmean_resid<DIM, FORM, A, PA>(Lf, u.p, rhs, Cs, fa);
  }
  if (ok) coarse[lin(Lc, C)] = (0.25 * tm + 0.5 * t0) + 0.25 * t1;
}

// A in {0, 1}: lanes along coarse axis 2 (coalesced), each thread marches a
// chunk of coarse indices along A, carrying t(2C+1) into the next t(2C-1).
template <int DIM, int FORM, int A, int PA>
__global__ void __launch_bounds__(kThreads)
k_face_rr_m(LevelDev Lf, LevelDev Lc, CPtr3 u, const double* __restrict__ rhs, double* __restrict__ coarse,
            Box cb, int chunk) {
  pdl_enter();
  constexpr int T = (A == 0) ? 1 : 0;  // the other non-contiguous axis
  int C[3];
  C[2] = cb.lo[2] + (int)(blockIdx.x * blockDim.x + threadIdx.x);
  if (DIM == 3) {
    C[T] = cb.lo[T] + (int)(blockIdx.y * blockDim.y + threadIdx.y);
    if (C[T] > cb.hi[T]) return;
  } else {
    C[0] = 0;
  }
  if (C[2] > cb.hi[2]) return;
  const int a0 = cb.lo[A] + (int)blockIdx.z * chunk;
  const int a1 = min(a0 + chunk - 1, cb.hi[A]);
  C[A] = a0;
  int fa = 2 * a0 - 1;
  if (fa < 0 && !(A == 0 && Lf.dist0)) fa += Lf.n[A];
  double tm = tmean_resid<DIM, FORM, A, PA>(Lf, u.p, rhs, C, fa);
#pragma unroll 1
  for (int c = a0; c <= a1; ++c) {
    C[A] = c;
    const double t0 = tmean_resid<DIM, FORM, A, PA>(Lf, u.p, rhs, C, 2 * c);
    const double t1 = tmean_resid<DIM, FORM, A, PA>(Lf, u.p, rhs, C, 2 * c + 1);
    coarse[lin(Lc, C)] = (0.25 * tm + 0.5 * t0) + 0.25 * t1;
    tm = t1;
  }
}

template <int DIM, int PA, bool NC = true>
__device__ __forceinline__ double cell_resid_at(const LevelDev& L, const double* phi,
                                                const double* rhs, const int* ci) {
  const int c = lin(L, ci);
  double dg;
  const double lp = cell_row<DIM, PA>(L, phi, c, ci, dg);
  return (NC ? __ldg(rhs + c) : rhs[c]) - lp;
}

// mean of the 2^d fine residuals of coarse cell C (multigrid.py:177-182)
template <int DIM, int PA, bool NC = true>
__device__ __forceinline__ double cell_rr_at(const LevelDev& Lf, const double* phi, const double* rhs,
                                             const int* C) {
  if (DIM == 3) {
    double s[2];
#pragma unroll 1
    for (int k = 0; k < 2; ++k) {
      double q[2];
#pragma unroll 1
      for (int j = 0; j < 2; ++j) {
        int a0[3] = {2 * C[0], 2 * C[1] + j, 2 * C[2] + k};
        int a1[3] = {2 * C[0] + 1, 2 * C[1] + j, 2 * C[2] + k};
        q[j] = 0.5 * (cell_resid_at<3, PA, NC>(Lf, phi, rhs, a0) + cell_resid_at<3, PA, NC>(Lf, phi, rhs, a1));
      }
      s[k] = 0.5 * (q[0] + q[1]);
    }
    return 0.5 * (s[0] + s[1]);
  }
  double q[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    int a0[3] = {0, 2 * C[1], 2 * C[2] + k};
    int a1[3] = {0, 2 * C[1] + 1, 2 * C[2] + k};
    q[k] = 0.5 * (cell_resid_at<2, PA, NC>(Lf, phi, rhs, a0) + cell_resid_at<2, PA, NC>(Lf, phi, rhs, a1));
  }
  return 0.5 * (q[0] + q[1]);
}

template <int DIM, int PA>
__global__ void __launch_bounds__(kThreads)
k_cell_rr(LevelDev Lf, LevelDev Lc, const double* phi, const double* __restrict__ rhs,
          double* __restrict__ coarse, Box cb, unsigned total) {
  pdl_enter();
  int C[3];
  if (!box_point(cb, C)) return;
  coarse[lin(Lc, C)] = cell_rr_at<DIM, PA>(Lf, phi, rhs, C);
}

// ---------------------------------------------------------------------------
// prolongation + add (multigrid.py:185-192, 236-295, 431-436)
// ---------------------------------------------------------------------------

__device__ __forceinline__ void tang_pair(const LevelDev& Lc, int ax, int fine_i, int& J, int& nb) {
  J = fine_i >> 1;
  nb = (fine_i & 1) ? J + 1 : J - 1;
  const int n = Lc.n[ax];
  if (ax == 0 && Lc.dist0) {
    // ghost planes hold the neighbouring slabs' values
  } else if (Lc.bclo[ax] == BC_PER) {
    if (nb < 0) nb += n;
    if (nb >= n) nb -= n;
  } else {
    nb = nb < 0 ? 0 : (nb > n - 1 ? n - 1 : nb);
  }
}

template <bool NC>
__device__ __forceinline__ double ldc(const double* p, int i) { return NC ? __ldg(p + i) : p[i]; }

// fine face F of component A += bilinear prolongation of the coarse field
// (multigrid.py:236-295): tangential (3/4, 1/4) weights, normal midpoint mean
template <int DIM, int A, bool NC = true>
__device__ __forceinline__ void face_pa_at(const LevelDev& Lf, const LevelDev& Lc, const double* coarse,
                                           double* fine, const int* F) {
  using O = Others<DIM, A>;
  int J1, n1, J2 = 0, n2 = 0;
  tang_pair(Lc, O::B1, F[O::B1], J1, n1);
  if (DIM == 3) tang_pair(Lc, O::B2, F[O::B2], J2, n2);
  auto T = [&](int I) -> double {
    int c[3] = {0, 0, 0};
    c[A] = I;
    if (DIM == 3) {
      c[O::B1] = J1; c[O::B2] = J2;
      const double x00 = ldc<NC>(coarse, lin(Lc, c));
      c[O::B1] = n1;
      const double x10 = ldc<NC>(coarse, lin(Lc, c));
      c[O::B1] = J1; c[O::B2] = n2;
      const double x01 = ldc<NC>(coarse, lin(Lc, c));
      c[O::B1] = n1;
      const double x11 = ldc<NC>(coarse, lin(Lc, c));
      const double ta = 0.75 * x00 + 0.25 * x10;
      const double tb = 0.75 * x01 + 0.25 * x11;
      return 0.75 * ta + 0.25 * tb;
    } else {
      c[O::B1] = J1;
      const double x0 = ldc<NC>(coarse, lin(Lc, c));
      c[O::B1] = n1;
      const double x1 = ldc<NC>(coarse, lin(Lc, c));
      return 0.75 * x0 + 0.25 * x1;
    }
  };
  const int I = F[A] >> 1;
  double v;
  if ((F[A] & 1) == 0) {
    v = T(I);
  } else {
    int I2 = I + 1;
    if (Lc.bclo[A] == BC_PER && I2 == Lc.n[A] && !(A == 0 && Lc.dist0)) I2 = 0;
    v = 0.5 * (T(I) + T(I2));
  }
  const int f = lin(Lf, F);
  fine[f] = fine[f] + v;
}

// The two coarse neighbours used by the fine faces 2J (J-1) and 2J+1 (J+1)
// along tangential axis ax (tang_pair for both parities at once).
__device__ __forceinline__ void tang_nbrs(const LevelDev& Lc, int ax, int J, int& jm, int& jp) {
  jm = J - 1;
  jp = J + 1;
  const int n = Lc.n[ax];
  if (ax == 0 && Lc.dist0) {
    // ghost planes hold the neighbouring slabs' values
  } else if (Lc.bclo[ax] == BC_PER) {
    if (jm < 0) jm += n;
    if (jp >= n) jp -= n;
  } else {
    jm = jm < 0 ? 0 : jm;
    jp = jp > n - 1 ? n - 1 : jp;
  }
}

// Prolongation + add, one thread per coarse position C = (I along A, J1, J2):
// the 2^d fine faces (2I+{0,1}, 2J1+{0,1}, 2J2+{0,1}) from 2 x 3^(d-1) coarse
// values (instead of up to 8 per fine face).  Same expressions, same order as
// face_pa_at, so bit-identical.
template <int DIM, int A>
__global__ void __launch_bounds__(kThreads)
k_face_pa8(LevelDev Lf, LevelDev Lc, const double* __restrict__ coarse, double* __restrict__ fine, Box cb) {
  pdl_enter();
  using O = Others<DIM, A>;
  int C[3];
  if (!box_point(cb, C)) return;
  const int I = C[A];
  int I2 = I + 1;
  if (Lc.bclo[A] == BC_PER && I2 == Lc.n[A] && !(A == 0 && Lc.dist0)) I2 = 0;
  int jm1, jp1, jm2 = 0, jp2 = 0;
  tang_nbrs(Lc, O::B1, C[O::B1], jm1, jp1);
  if (DIM == 3) tang_nbrs(Lc, O::B2, C[O::B2], jm2, jp2);
  double T[2][2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    int c[3] = {C[0], C[1], C[2]};
    c[A] = a ? I2 : I;
    if (DIM == 3) {
      const int b1[3] = {jm1, C[O::B1], jp1}, b2[3] = {jm2, C[O::B2], jp2};
      double x[3][3];
#pragma unroll
      for (int u = 0; u < 3; ++u)
#pragma unroll
        for (int v = 0; v < 3; ++v) {
          c[O::B1] = b1[u];
          c[O::B2] = b2[v];
          x[u][v] = __ldg(coarse + lin(Lc, c));
        }
#pragma unroll
      for (int p1 = 0; p1 < 2; ++p1)
#pragma unroll
        for (int p2 = 0; p2 < 2; ++p2) {
          const int n1 = p1 ? 2 : 0, n2 = p2 ? 2 : 0;
          const double ta = 0.75 * x[1][1] + 0.25 * x[n1][1];
          const double tb = 0.75 * x[1][n2] + 0.25 * x[n1][n2];
          T[a][p1][p2] = 0.75 * ta + 0.25 * tb;
        }
    } else {
      const int b1[3] = {jm1, C[O::B1], jp1};
      double x[3];
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        c[O::B1] = b1[u];
        x[u] = __ldg(coarse + lin(Lc, c));
      }
#pragma unroll
      for (int p1 = 0; p1 < 2; ++p1) {
        T[a][p1][0] = 0.75 * x[1] + 0.25 * x[p1 ? 2 : 0];
        T[a][p1][1] = T[a][p1][0];
      }
    }
  }
  const bool wallA = Lf.bclo[A] != BC_PER;
#if FC_PF > 0
  if (DIM == 3 && C[0] + 1 <= cb.hi[0]) {  // the 8 fine faces of the next coarse plane (2 fine planes ahead)
#pragma unroll
    for (int pa = 0; pa < 2; ++pa)
#pragma unroll
      for (int p1 = 0; p1 < 2; ++p1) {
        int F[3] = {0, 0, 0};
        F[A] = 2 * I + pa;
        F[O::B1] = 2 * C[O::B1] + p1;
        F[O::B2] = 2 * C[O::B2];
        pf_plane(fine, lin(Lf, F) + 2 * Lf.s0);  // both p2 faces share the 16 bytes when B2 is contiguous
        if (O::B2 != 2) {
          F[O::B2] += 1;
          pf_plane(fine, lin(Lf, F) + 2 * Lf.s0);
        }
      }
  }
#endif
#pragma unroll
  for (int pa = 0; pa < 2; ++pa) {
    if (wallA && pa == 0 && I == 0) continue;  // fine wall face, not an unknown
#pragma unroll
    for (int p1 = 0; p1 < 2; ++p1)
#pragma unroll
      for (int p2 = 0; p2 < (DIM == 3 ? 2 : 1); ++p2) {
        int F[3] = {0, 0, 0};
        F[A] = 2 * I + pa;
        F[O::B1] = 2 * C[O::B1] + p1;
        if (DIM == 3) F[O::B2] = 2 * C[O::B2] + p2;
        const double v = pa == 0 ? T[0][p1][p2] : 0.5 * (T[0][p1][p2] + T[1][p1][p2]);
        const int f = lin(Lf, F);
        fine[f] = fine[f] + v;
      }
  }
}

template <int DIM, bool NC = true>
__device__ __forceinline__ void cell_pa_at(const LevelDev& Lf, const LevelDev& Lc, const double* coarse,
                                           double* fine, const int* F) {
  int C[3] = {DIM == 3 ? F[0] >> 1 : 0, F[1] >> 1, F[2] >> 1};
  const int f = lin(Lf, F);
  fine[f] = fine[f] + ldc<NC>(coarse, lin(Lc, C));
}

template <int DIM>
__global__ void __launch_bounds__(kThreads)
k_cell_pa(LevelDev Lf, LevelDev Lc, const double* __restrict__ coarse, double* __restrict__ fine,
          Box fb, unsigned total) {
  pdl_enter();
  int F[3];
  if (!box_point(fb, F)) return;
  cell_pa_at<DIM>(Lf, Lc, coarse, fine, F);
}

// ---------------------------------------------------------------------------
// full operators and preconditioner glue
// ---------------------------------------------------------------------------

__device__ __forceinline__ bool in_face(const LevelDev& L, int A, const int* ci) {
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    const int ext = L.n[b] + ((b == A && L.bclo[A] != BC_PER) ? 1 : 0);
    if (ci[b] >= ext) return false;
  }
  return true;
}
__device__ __forceinline__ bool is_wall_face(const LevelDev& L, int A, const int* ci) {
  return L.bclo[A] != BC_PER && (ci[A] == 0 || ci[A] == L.n[A]);
}
__device__ __forceinline__ bool in_cell(const LevelDev& L, const int* ci) {
  return ci[0] < L.n[0] && ci[1] < L.n[1] && ci[2] < L.n[2];
}

// (G q)_A at face f (operators.py:191-198): (q(f) - q(f-1))/h, wall faces 0
template <int A>
__device__ __forceinline__ double grad_at(const LevelDev& L, const double* q, int f, const int* ci) {
  const int dm = A == 0 ? dminus<0>(L, ci[0]) : (A == 1 ? dminus<1>(L, ci[1]) : dminus<2>(L, ci[2]));
  return (__ldg(q + f) - __ldg(q + f + dm)) * L.inv_h;
}

template <int DIM, int FORM, int A, int PA, bool DE>
__device__ __forceinline__ void m_face(const LevelDev& L, const double* const* u, const double* p,
                                       double* out, const int* ci) {
  if (!in_face(L, A, ci)) return;
  const int f = lin(L, ci);
  if (is_wall_face(L, A, ci)) {
    out[f] = 0.0;
    return;
  }
  double dg;
  const double au = face_row<DIM, FORM, A, PA, true, false, DE>(L, u, f, ci, dg);
  out[f] = au + grad_at<A>(L, p, f, ci);
}

template <int DIM, int FORM, int PA, bool DE = false>
__global__ void __launch_bounds__(kThreads)
k_apply_M(LevelDev L, CPtr3 u, const double* __restrict__ p, Ptr3 out_u, double* __restrict__ out_p,
          Box b, unsigned total) {
  pdl_enter();
  {
    int ci[3];
    if (!box_point(b, ci)) return;
    if (DIM == 3) m_face<3, FORM, 0, PA, DE>(L, u.p, p, out_u.p[0], ci);
    m_face<DIM, FORM, 1, PA, DE>(L, u.p, p, out_u.p[1], ci);
    m_face<DIM, FORM, 2, PA, DE>(L, u.p, p, out_u.p[2], ci);
    if (in_cell(L, ci)) {
      const int c = lin(L, ci);
      out_p[c] = -(div_sum<DIM, PA>(L, u.p, c, ci) * L.inv_h);
    }
  }
}

template <int DIM, int FORM, int A>
__device__ __forceinline__ void r_face(const LevelDev& L, const double* const* x, const double* const* rhs,
                                       const double* q, double* out, const int* ci) {
  if (!in_face(L, A, ci)) return;
  const int f = lin(L, ci);
  if (is_wall_face(L, A, ci)) {
    out[f] = 0.0;
    return;
  }
  double v;
  if (rhs[A] != nullptr) {
    v = __ldg(rhs[A] + f);
    if (q != nullptr) v = v - grad_at<A>(L, q, f, ci);
    if (x[A] != nullptr) {
      double dg;
      v = v - face_row<DIM, FORM, A>(L, x, f, ci, dg);
    }
  } else {
    double dg;
    v = face_row<DIM, FORM, A>(L, x, f, ci, dg);
  }
  out[f] = v;
}

template <int DIM, int FORM>
__global__ void __launch_bounds__(kThreads)
k_face_residual(LevelDev L, CPtr3 x, CPtr3 rhs, const double* __restrict__ q, Ptr3 out, Box b,
                unsigned total) {
  pdl_enter();
  {
    int ci[3];
    if (!box_point(b, ci)) return;
    if (DIM == 3) r_face<3, FORM, 0>(L, x.p, rhs.p, q, out.p[0], ci);
    r_face<DIM, FORM, 1>(L, x.p, rhs.p, q, out.p[1], ci);
    r_face<DIM, FORM, 2>(L, x.p, rhs.p, q, out.p[2], ci);
  }
}

// Residual of all face components into memory (rhs - A x; the fused
// residual->restriction's face_resid_at expression), for the split
// residual / restriction path on large levels: one face row per thread at
// full occupancy instead of the latency-bound marching kernels.
template <int DIM, int FORM, int PA, bool DE = false>
__global__ void __launch_bounds__(kThreads)
k_face_res3(LevelDev L, CPtr3 x, CPtr3 rhs, Ptr3 out, Box b) {
  pdl_enter();
  int ci[3];
  if (!box_point(b, ci)) return;
  const int f = lin(L, ci);
#pragma unroll
  for (int A = 3 - DIM; A < 3; ++A) {
    if (!in_face(L, A, ci) || is_wall_face(L, A, ci)) continue;
    double au;
    double dg;
    if (A == 0) au = face_row<DIM, FORM, (DIM == 3 ? 0 : 1), PA, true, false, DE>(L, x.p, f, ci, dg);
    else if (A == 1) au = face_row<DIM, FORM, 1, PA, true, false, DE>(L, x.p, f, ci, dg);
    else au = face_row<DIM, FORM, 2, PA, true, false, DE>(L, x.p, f, ci, dg);
    out.p[A][f] = __ldg(rhs.p[A] + f) - au;
  }
}

// Face restriction of a residual field (multigrid.py:195-233): the tangential
// 2^(d-1) mean on the three fine normal planes, weights (1/4, 1/2, 1/4).
template <int DIM, int A>
__global__ void __launch_bounds__(kThreads)
k_face_restrict(LevelDev Lf, LevelDev Lc, const double* __restrict__ r, double* __restrict__ coarse, Box cb) {
  pdl_enter();
  using O = Others<DIM, A>;
  int C[3];
  if (!box_point(cb, C)) return;
  double tv[3];
#pragma unroll
  for (int o = -1; o <= 1; ++o) {
    int fa = 2 * C[A] + o;
    if (fa < 0 && !(A == 0 && Lf.dist0)) fa += Lf.n[A];
    int fi[3] = {2 * C[0], 2 * C[1], 2 * C[2]};
    if (DIM == 2) fi[0] = 0;
    fi[A] = fa;
    if (DIM == 3) {
      double p[2];
#pragma unroll
      for (int t2 = 0; t2 < 2; ++t2) {
        int q0[3] = {fi[0], fi[1], fi[2]};
        q0[O::B2] += t2;
        int q1[3] = {q0[0], q0[1], q0[2]};
        q1[O::B1] += 1;
        p[t2] = 0.5 * (__ldg(r + lin(Lf, q0)) + __ldg(r + lin(Lf, q1)));
      }
      tv[o + 1] = 0.5 * (p[0] + p[1]);
    } else {
      int q1[3] = {fi[0], fi[1], fi[2]};
      q1[O::B1] += 1;
      tv[o + 1] = 0.5 * (__ldg(r + lin(Lf, fi)) + __ldg(r + lin(Lf, q1)));
    }
  }
  coarse[lin(Lc, C)] = (0.25 * tv[0] + 0.5 * tv[1]) + 0.25 * tv[2];
}

template <int DIM, int PA>
__global__ void __launch_bounds__(kThreads)
k_cell_res(LevelDev L, const double* x, const double* __restrict__ rhs, double* __restrict__ out, Box b) {
  pdl_enter();
  int ci[3];
  if (!box_point(b, ci)) return;
#if FC_PF > 0
  if (DIM == 3 && ci[0] + FC_PF <= b.hi[0]) {
    const int cp = lin(L, ci) + FC_PF * L.s0;
    pf_plane(x, cp);
    pf_plane(rhs, cp);
    if (!L.beta_const) {
      pf_plane(L.beta_f[0], cp);
      pf_plane(L.beta_f[1], cp);
      pf_plane(L.beta_f[2], cp);
    }
  }
#endif
  out[lin(L, ci)] = cell_resid_at<DIM, PA>(L, x, rhs, ci);
}

// cell restriction of a residual field (multigrid.py:177-182), cell_rr_at's order
template <int DIM>
__global__ void __launch_bounds__(kThreads)
k_cell_restrict(LevelDev Lf, LevelDev Lc, const double* __restrict__ r, double* __restrict__ coarse, Box cb) {
  pdl_enter();
  int C[3];
  if (!box_point(cb, C)) return;
  double out;
  if (DIM == 3) {
    double s[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      double q[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        int a0[3] = {2 * C[0], 2 * C[1] + j, 2 * C[2] + k};
        int a1[3] = {2 * C[0] + 1, 2 * C[1] + j, 2 * C[2] + k};
        q[j] = 0.5 * (__ldg(r + lin(Lf, a0)) + __ldg(r + lin(Lf, a1)));
      }
      s[k] = 0.5 * (q[0] + q[1]);
    }
    out = 0.5 * (s[0] + s[1]);
  } else {
    double q[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      int a0[3] = {0, 2 * C[1], 2 * C[2] + k};
      int a1[3] = {0, 2 * C[1] + 1, 2 * C[2] + k};
      q[k] = 0.5 * (__ldg(r + lin(Lf, a0)) + __ldg(r + lin(Lf, a1)));
    }
    out = 0.5 * (q[0] + q[1]);
  }
  coarse[lin(Lc, C)] = out;
}

template <int DIM>
__global__ void __launch_bounds__(kThreads)
k_cell_residual(LevelDev L, const double* x, const double* rhs, double* out, Box b, unsigned total) {
  pdl_enter();
  {
    int ci[3];
    if (!box_point(b, ci)) return;
    const int c = lin(L, ci);
    double dg;
    const double lp = cell_row<DIM>(L, x, c, ci, dg);
    out[c] = rhs != nullptr ? __ldg(rhs + c) - lp : lp;
  }
}

template <int DIM>
__global__ void __launch_bounds__(kThreads)
k_div_add(LevelDev L, CPtr3 u, const double* __restrict__ rp, double* __restrict__ out, Box b,
          unsigned total) {
  pdl_enter();
  {
    int ci[3];
    if (!box_point(b, ci)) return;
    const int c = lin(L, ci);
#if FC_PF > 0
    if (DIM == 3 && ci[0] + FC_PF <= b.hi[0]) {
      const int cp = c + FC_PF * L.s0;
      pf_plane(u.p[0], cp);
      pf_plane(u.p[1], cp);
      pf_plane(u.p[2], cp);
      pf_plane(rp, cp);
    }
#endif
    out[c] = div_sum<DIM>(L, u.p, c, ci) * L.inv_h + __ldg(rp + c);
  }
}

__device__ __forceinline__ double schur_v(const LevelDev& L, int form, int c) {
  const double mu = __ldg(L.mu_c + c);
  if (form == F_LAP) return mu;
  if (form == F_STRESS) return 2.0 * mu;
  return __ldg(L.gam_c + c) + (4.0 / 3.0) * mu;
}

template <int A>
__device__ __forceinline__ void glue_face(const LevelDev& L, double* xu, const double* phi, const int* ci) {
  if (!in_face(L, A, ci) || is_wall_face(L, A, ci)) return;
  const int f = lin(L, ci);
  const double beta = L.beta_const ? L.beta_val : __ldg(L.beta_f[A] + f);  // non-wall face
  xu[f] = xu[f] - grad_at<A>(L, phi, f, ci) * beta;
}

template <int DIM>
__global__ void __launch_bounds__(kThreads)
k_p1_glue(LevelDev L, int form, Ptr3 xu, const double* __restrict__ phi, const double* __restrict__ bc,
          double* __restrict__ xp, double sign, Box b, unsigned total) {
  pdl_enter();
  {
    int ci[3];
    if (!box_point(b, ci)) return;
#if FC_PF > 0
    if (DIM == 3 && ci[0] + FC_PF <= b.hi[0]) {
      const int cp = lin(L, ci) + FC_PF * L.s0;
      pf_plane(xu.p[0], cp);
      pf_plane(xu.p[1], cp);
      pf_plane(xu.p[2], cp);
      pf_plane(phi, cp);
      pf_plane(bc, cp);
      pf_plane(L.mu_c, cp);
    }
#endif
    if (DIM == 3) glue_face<0>(L, xu.p[0], phi, ci);
    glue_face<1>(L, xu.p[1], phi, ci);
    glue_face<2>(L, xu.p[2], phi, ci);
    if (in_cell(L, ci)) {
      const int c = lin(L, ci);
      const double s = schur_v(L, form, c) * __ldg(bc + c) - L.theta * __ldg(phi + c);
      xp[c] = s * sign;
    }
  }
}

__global__ void __launch_bounds__(kThreads)
k_schur(LevelDev L, int form, const double* __restrict__ r, const double* __restrict__ phi,
        double* __restrict__ out, double sign, Box b, unsigned total) {
  pdl_enter();
  {
    int ci[3];
    if (!box_point(b, ci)) return;
    const int c = lin(L, ci);
    double s;
    if (phi != nullptr) s = (-L.theta) * __ldg(phi + c) + schur_v(L, form, c) * __ldg(r + c);
    else s = schur_v(L, form, c) * __ldg(r + c);
    out[c] = s * sign;
  }
}

template <int A>
__device__ __forceinline__ void subg_face(const LevelDev& L, const double* ru, const double* q, double* out,
                                          const int* ci) {
  if (!in_face(L, A, ci)) return;
  const int f = lin(L, ci);
  if (is_wall_face(L, A, ci)) {
    out[f] = 0.0;
    return;
  }
  out[f] = __ldg(ru + f) - grad_at<A>(L, q, f, ci);
}

template <int DIM>
__global__ void __launch_bounds__(kThreads)
k_face_sub_grad(LevelDev L, CPtr3 ru, const double* __restrict__ q, Ptr3 out, Box b, unsigned total) {
  pdl_enter();
  {
    int ci[3];
    if (!box_point(b, ci)) return;
    if (DIM == 3) subg_face<0>(L, ru.p[0], q, out.p[0], ci);
    subg_face<1>(L, ru.p[1], q, out.p[1], ci);
    subg_face<2>(L, ru.p[2], q, out.p[2], ci);
  }
}

// ---------------------------------------------------------------------------
// setup: coefficient coarsening (multigrid.py:112-169), 1/rho, checks
// ---------------------------------------------------------------------------

template <int DIM>
__global__ void k_coarsen_cellmean(LevelDev Lf, LevelDev Lc, const double* __restrict__ fine,
                                   double* __restrict__ coarse, Box cb, unsigned total) {
  pdl_enter();
  {
    int C[3];
    if (!box_point(cb, C)) return;
    auto at = [&](int i, int j, int k) {
      int q[3] = {DIM == 3 ? 2 * C[0] + i : 0, 2 * C[1] + j, 2 * C[2] + k};
      return __ldg(fine + lin(Lf, q));
    };
    double out;
    if (DIM == 3) {
      double s[2];
      for (int k = 0; k < 2; ++k) {
        double q0 = 0.5 * (at(0, 0, k) + at(1, 0, k));
        double q1 = 0.5 * (at(0, 1, k) + at(1, 1, k));
        s[k] = 0.5 * (q0 + q1);
      }
      out = 0.5 * (s[0] + s[1]);
    } else {
      double q0 = 0.5 * (at(0, 0, 0) + at(0, 1, 0));
      double q1 = 0.5 * (at(0, 0, 1) + at(0, 1, 1));
      out = 0.5 * (q0 + q1);
    }
    coarse[lin(Lc, C)] = out;
  }
}

// rho_face: inject along A, then 2-mean along the other axes in ascending order
template <int DIM, int A>
__global__ void k_coarsen_face(LevelDev Lf, LevelDev Lc, const double* __restrict__ fine,
                               double* __restrict__ coarse, Box cb, unsigned total) {
  pdl_enter();
  using O = Others<DIM, A>;
  {
    int C[3];
    if (!box_point(cb, C)) return;
    int q[3] = {2 * C[0], 2 * C[1], 2 * C[2]};
    double out;
    if (DIM == 3) {
      double p[2];
      for (int t2 = 0; t2 < 2; ++t2) {
        int a[3] = {q[0], q[1], q[2]};
        a[O::B2] += t2;
        const double m0 = __ldg(fine + lin(Lf, a));
        a[O::B1] += 1;
        const double m1 = __ldg(fine + lin(Lf, a));
        p[t2] = 0.5 * (m0 + m1);
      }
      out = 0.5 * (p[0] + p[1]);
    } else {
      int a[3] = {q[0], q[1], q[2]};
      const double m0 = __ldg(fine + lin(Lf, a));
      a[O::B1] += 1;
      const double m1 = __ldg(fine + lin(Lf, a));
      out = 0.5 * (m0 + m1);
    }
    coarse[lin(Lc, C)] = out;
  }
}

// mu_edge with normal axis e: inject on the staggered pair, 2-mean along e (3D)
template <int DIM>
__global__ void k_coarsen_edge(LevelDev Lf, LevelDev Lc, int e, const double* __restrict__ fine,
                               double* __restrict__ coarse, Box cb, unsigned total) {
  pdl_enter();
  {
    int C[3];
    if (!box_point(cb, C)) return;
    int q[3] = {2 * C[0], 2 * C[1], 2 * C[2]};
    if (DIM == 2) q[0] = 0;
    double out;
    if (DIM == 3) {
      const double m0 = __ldg(fine + lin(Lf, q));
      q[e] += 1;
      const double m1 = __ldg(fine + lin(Lf, q));
      out = 0.5 * (m0 + m1);
    } else {
      out = __ldg(fine + lin(Lf, q));
    }
    coarse[lin(Lc, C)] = out;
  }
}

// beta = 1/rho_face (0 on wall faces); flag |= 1 on rho_face <= 0 (operators.py:209-210);
// cflag |= 1 when a non-wall rho_face differs from *ref (the level is not constant-density)
__global__ void k_beta(LevelDev L, int A, const double* __restrict__ rho, double* __restrict__ beta,
                       int* flag, int* cflag, const double* ref, Box b, unsigned total) {
  pdl_enter();
  {
    int ci[3];
    if (!box_point(b, ci)) return;
    const int f = lin(L, ci);
    const double r = rho[f];
    if (!(r > 0.0)) atomicOr(flag, 1);
    const bool wall = L.bclo[A] != BC_PER && (ci[A] == 0 || ci[A] == L.n[A]);
    beta[f] = wall ? 0.0 : 1.0 / r;
    if (cflag && !wall && !(r == __ldg(ref))) atomicOr(cflag, 1);
  }
}

template <int DIM, int FORM, int A>
__device__ __forceinline__ void chk_face(const LevelDev& L, const int* ci, int* flags) {
  if (!in_face(L, A, ci) || is_wall_face(L, A, ci)) return;
  // the diagonal only reads coefficients; pass a zero field for u
  double dg;
  const double* none[3] = {L.mu_c, L.mu_c, L.mu_c};
  (void)face_row<DIM, FORM, A>(L, none, lin(L, ci), ci, dg);
  if (dg == 0.0) atomicOr(flags, 1);
}

template <int DIM, int FORM>
__global__ void k_check_diag(LevelDev L, int* flags, Box b, unsigned total) {
  pdl_enter();
  {
    int ci[3];
    if (!box_point(b, ci)) return;
    if (DIM == 3) chk_face<3, FORM, 0>(L, ci, flags);
    chk_face<DIM, FORM, 1>(L, ci, flags);
    chk_face<DIM, FORM, 2>(L, ci, flags);
    if (in_cell(L, ci)) {
      double dg;
      (void)cell_row<DIM>(L, L.mu_c, lin(L, ci), ci, dg);
      if (dg == 0.0) atomicOr(flags + 1, 1);  // cell diagonal: its own int (ranks max-reduce the flags)
    }
  }
}

// The smoother diagonals as arrays (helmholtz_diagonal / lrho_diagonal,
// operators.py:396-439): the same register-computed diagonal the colour passes
// divide by; wall-normal boundary faces are set to one as in the reference.
template <int DIM, int FORM, int A>
__device__ __forceinline__ void wr_face_diag(const LevelDev& L, const int* ci, double* out) {
  if (!in_face(L, A, ci)) return;
  const int f = lin(L, ci);
  if (is_wall_face(L, A, ci)) {
    out[f] = 1.0;
    return;
  }
  double dg;
  const double* none[3] = {L.mu_c, L.mu_c, L.mu_c};
  (void)face_row<DIM, FORM, A>(L, none, f, ci, dg);
  out[f] = dg;
}

template <int DIM, int FORM>
__global__ void k_write_diag(LevelDev L, Ptr3 fd, double* cd, Box b, unsigned total) {
  pdl_enter();
  {
    int ci[3];
    if (!box_point(b, ci)) return;
    if (fd.p[2] != nullptr) {
      if (DIM == 3) wr_face_diag<3, FORM, 0>(L, ci, fd.p[0]);
      wr_face_diag<DIM, FORM, 1>(L, ci, fd.p[1]);
      wr_face_diag<DIM, FORM, 2>(L, ci, fd.p[2]);
    }
    if (cd != nullptr && in_cell(L, ci)) {
      double dg;
      (void)cell_row<DIM>(L, L.mu_c, lin(L, ci), ci, dg);
      cd[lin(L, ci)] = dg;
    }
  }
}

// div / grad as the reference's public functions compute them (operators.py:
// 182-198), bit for bit: div = ((d0 + d1) + d2) / h reading the stored
// boundary faces, grad = (p[i] - p[i-1]) / h with wall-normal faces 0.
template <int DIM>
__global__ void k_div(LevelDev L, CPtr3 u, double* out, Box b, unsigned total) {
  pdl_enter();
  {
    int ci[3];
    if (!box_point(b, ci)) return;
    const int c = lin(L, ci);
    const double* uu[3] = {u.p[0], u.p[1], u.p[2]};
    out[c] = div_sum<DIM>(L, uu, c, ci) / L.h;
  }
}

template <int A>
__device__ __forceinline__ void grad_face(const LevelDev& L, const double* p, double* out, const int* ci) {
  if (!in_face(L, A, ci)) return;
  const int f = lin(L, ci);
  if (is_wall_face(L, A, ci)) {
    out[f] = 0.0;
    return;
  }
  const int dm = A == 0 ? dminus<0>(L, ci[0]) : (A == 1 ? dminus<1>(L, ci[1]) : dminus<2>(L, ci[2]));
  out[f] = (__ldg(p + f) - __ldg(p + f + dm)) / L.h;
}

template <int DIM>
__global__ void k_grad(LevelDev L, const double* p, Ptr3 out, Box b, unsigned total) {
  pdl_enter();
  {
    int ci[3];
    if (!box_point(b, ci)) return;
    if (DIM == 3) grad_face<0>(L, p, out.p[0], ci);
    grad_face<1>(L, p, out.p[1], ci);
    grad_face<2>(L, p, out.p[2], ci);
  }
}

// The reference's edge (3D) / node (2D) viscosity at index ci of edge array e,
// for any boundary conditions: _avg_to_stagger along the lower plane axis,
// then the higher (operators.py:90-104, :133-145) -- periodic and interior
// positions average 0.5 (x[j] + x[j-1]), a wall boundary copies its cell.
template <int DIM>
__device__ double edge_ref(const LevelDev& L, int e, const int* ci) {
  const int al = DIM == 2 ? 1 : (e == 0 ? 1 : 0);
  const int ah = DIM == 2 ? 2 : (e == 2 ? 1 : 2);
  const bool pl = L.bclo[al] == BC_PER, ph = L.bclo[ah] == BC_PER;
  const int jl = ci[al], jh = ci[ah], nl = L.n[al], nh = L.n[ah];
  // a slab-distributed axis 0 reads its ghost plane -1 instead of wrapping
  auto wrapa = [&](int j, int n, int ax) { return (j < 0 && !(ax == 0 && L.dist0)) ? j + n : j; };
  auto cell = [&](int cl, int ch) {
    int c[3] = {ci[0], ci[1], ci[2]};
    c[al] = cl;
    c[ah] = ch;
    return __ldg(L.mu_c + lin(L, c));
  };
  auto arr1 = [&](int ch) {
    if (!pl && jl == 0) return cell(0, ch);
    if (!pl && jl == nl) return cell(nl - 1, ch);
    return 0.5 * (cell(jl, ch) + cell(wrapa(jl - 1, nl, al), ch));
  };
  if (!ph && jh == 0) return arr1(0);
  if (!ph && jh == nh) return arr1(nh - 1);
  return 0.5 * (arr1(jh) + arr1(wrapa(jh - 1, nh, ah)));
}

// ---- device-side coefficient averaging (operators.py:81-104, :133-145) ----
// rho_face[A] = 0.5 (rho[i] + rho[i-1]) along A (periodic wrap), wall
// boundary faces copy the adjacent cell -- to_stagger_mean's expression.
__global__ void k_cell_to_face(LevelDev L, int A, const double* __restrict__ cell, double* __restrict__ face, Box b) {
  pdl_enter();
  int ci[3];
  if (!box_point(b, ci)) return;
  const int f = lin(L, ci);
  const int sA = A == 0 ? L.s0 : (A == 1 ? L.s1 : 1);
  double v;
  if (L.bclo[A] != BC_PER) {
    if (ci[A] == 0) v = __ldg(cell + f);
    else if (ci[A] == L.n[A]) v = __ldg(cell + f - sA);
    else v = 0.5 * (__ldg(cell + f) + __ldg(cell + f - sA));
  } else {
    const int lo = ci[A] == 0 ? f + (L.n[A] - 1) * sA : f - sA;
    v = 0.5 * (__ldg(cell + f) + __ldg(cell + lo));
  }
  face[f] = v;
}

// mu_e (edge with normal axis e; 2D: the node array) = scale * edge_ref:
// to_stagger_mean along the lower plane axis, then the upper (make_coef), then
// rescale's multiplication (operators.py:532-550) -- the host's operation order.
template <int DIM>
__device__ double edge_ref(const LevelDev& L, int e, const int* ci);
template <int DIM>
__global__ void k_cell_to_edge(LevelDev L, int e, double* __restrict__ out, double scale, Box b) {
  pdl_enter();
  int ci[3];
  if (!box_point(b, ci)) return;
  out[lin(L, ci)] = scale * edge_ref<DIM>(L, e, ci);
}

__global__ void k_scale(double* __restrict__ x, double scale, long long n) {
  pdl_enter();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    x[i] = scale * x[i];
}

// Does every edge (3D) / node (2D) viscosity of a level equal edge_ref to
// roundoff?  The reference builds mu_e exactly that way (operators.py:90-104)
// and rescale multiplies both by c (operators.py:532-550), so on the finest
// level they agree to a few ulp; coarse levels inject mu_e
// (multigrid.py:150-169) and do not.  flag |= 1 on any edge further apart
// than 4e-15 relative.  b: the cell box extended by one along wall axes.
template <int DIM>
__global__ void k_check_mue(LevelDev L, int* flag, Box b) {
  pdl_enter();
  int ci[3];
  if (!box_point(b, ci)) return;
  const int i = lin(L, ci);
  bool bad = false;
#pragma unroll
  for (int e = 0; e < (DIM == 3 ? 3 : 1); ++e) {
    const int ax = DIM == 2 ? 0 : e;  // the edge's own (cell-centred) axis
    if (ci[ax] >= L.n[ax]) continue;
    const double d = edge_ref<DIM>(L, e, ci);
    const double v = __ldg(L.mu_e[e] + i);
    bad |= !(fabs(d - v) <= 4e-15 * fabs(v));
  }
  if (bad) atomicOr(flag, 1);
}

__global__ void k_box_fill(LevelDev L, double* x, double v, Box b, unsigned total) {
  pdl_enter();
  {
    int ci[3];
    if (!box_point(b, ci)) return;
    x[lin(L, ci)] = v;
  }
}

// Inhomogeneous tangential wall velocity (operators.py:267-291 with BoundaryValues):
// the one-sided wall gradient 2(u - lo)/h (low wall) / 2(hi - u)/h (high wall)
// differs from the homogeneous one by -/+ 2 v/h, times mu_e at the wall edge,
// so row A of the face adjacent to wall (B, side) moves by -2 mu_e v / h^2.
// Free-slip walls zero the flux (no contribution); wall-normal boundary rows
// of A stay zero.  plane: C-order over the face extents of A with B dropped.
__global__ void k_wall_tangent(LevelDev L, int A, int B, int side, const double* __restrict__ plane,
                               double* out, Box b, int e1, int e2) {
  pdl_enter();
  int ci[3];
  if (!box_point(b, ci)) return;
  if (L.bclo[A] != BC_PER && (ci[A] == 0 || ci[A] == L.n[A])) return;
  int q[3] = {ci[0], ci[1], ci[2]};
  q[B] = 0;
  const double v = plane[((long long)q[0] * e1 + q[1]) * e2 + q[2]];
  const int f = lin(L, ci);
  const int st = B == 0 ? L.s0 : (B == 1 ? L.s1 : 1);
  const double mue = L.mu_e[edge_of(A, B)][side ? f + st : f];
  out[f] = out[f] - (mue * (2.0 * v * L.inv_h)) * L.inv_h;
}

// block partials of sum(x) and sum(|x|) (homogenize's flux compatibility check)
__global__ void __launch_bounds__(kThreads)
k_sum_abs_partial(const double* __restrict__ x, long long n, double* __restrict__ partials, int stride) {
  pdl_enter();
  __shared__ double acc[2][kThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v = 0.0, va = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const double t = __ldg(x + e);
    v += t;
    va += fabs(t);
  }
  for (int o = 16; o > 0; o >>= 1) {
    v += __shfl_down_sync(0xffffffffu, v, o);
    va += __shfl_down_sync(0xffffffffu, va, o);
  }
  if (lane == 0) {
    acc[0][warp] = v;
    acc[1][warp] = va;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0, sa = 0.0;
    for (int k = 0; k < kThreads / 32; ++k) {
      s += acc[0][k];
      sa += acc[1][k];
    }
    partials[blockIdx.x] = s;
    partials[stride + blockIdx.x] = sa;
  }
}

__global__ void k_box_sub_mean(LevelDev L, double* x, const double* sum, double inv_count, Box b,
                               unsigned total) {
  pdl_enter();
  const double m = sum[0] * inv_count;
  {
    int ci[3];
    if (!box_point(b, ci)) return;
    const int i = lin(L, ci);
    x[i] = x[i] - m;
  }
}

__global__ void k_add_scalar(double* y, const double* x) {
  pdl_enter(); *y += *x; }
__global__ void k_neg_copy(double* y, const double* x) {
  pdl_enter();
  *y = -*x;
}
__global__ void k_max_scalar(double* y, const double* x, int neg) {
  pdl_enter();
  const double v = neg ? -*x : *x;
  if (v > *y) *y = v;
}

__global__ void k_box_axpy(LevelDev L, double* y, const double* __restrict__ x, Box b, unsigned total) {
  pdl_enter();
  {
    int ci[3];
    if (!box_point(b, ci)) return;
    const int i = lin(L, ci);
    y[i] = y[i] + x[i];
  }
}

// ---------------------------------------------------------------------------
// flat-vector kernels for GMRES (deterministic two-stage reductions)
// ---------------------------------------------------------------------------

constexpr int kRedBlocks = kSMs * 8;   // partial-sum slots per reduction (8 CTAs/SM)
constexpr int kMaxVec = 128;           // max basis vectors in one multi-dot
constexpr int kVecChunk = 120;         // vectors per launch when a basis is longer (launch_cgs2 / launch_combo)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// partials[i*kRedBlocks + block] = sum over this block's elements of V_i . w
// (each thread keeps two double2 of w in registers: 2 x 16 B loads in flight per V_i)
__global__ void __launch_bounds__(kThreads)
k_multi_dot(const double* __restrict__ V, long long vstride, int nv, const double* __restrict__ w,
            long long n2, double* __restrict__ partials) {
  pdl_enter();
  __shared__ double acc[kMaxVec][kThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < nv * (kThreads / 32); i += blockDim.x) acc[i / (kThreads / 32)][i % (kThreads / 32)] = 0.0;
  __syncthreads();
  const double2* w2 = reinterpret_cast<const double2*>(w);
  const long long step = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e - threadIdx.x < n2; e += 2 * step) {
    const long long e1 = e + step;
    const bool ok0 = e < n2, ok1 = e1 < n2;
    const double2 w0 = ok0 ? __ldg(w2 + e) : make_double2(0.0, 0.0);
    const double2 wv1 = ok1 ? __ldg(w2 + e1) : make_double2(0.0, 0.0);
    for (int i = 0; i < nv; ++i) {
      const double2* v2 = reinterpret_cast<const double2*>(V + i * vstride);
      const double2 a = ok0 ? __ldg(v2 + e) : make_double2(0.0, 0.0);
      const double2 b = ok1 ? __ldg(v2 + e1) : make_double2(0.0, 0.0);
      double s = warp_sum((a.x * w0.x + a.y * w0.y) + (b.x * wv1.x + b.y * wv1.y));
      if (lane == 0) acc[i][warp] += s;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < kThreads / 32; ++k) s += acc[i][k];
    partials[i * kRedBlocks + blockIdx.x] = s;
  }
}

// w -= sum_i h_i V_i ; then partials of V_i . w (mode 0) or w . w (mode 1).
// The second read of V_i (mode 0) follows the first within the same thread
// and hits L1/L2; DRAM sees each V_i once.
__global__ void __launch_bounds__(kThreads)
k_update_dot(const double* __restrict__ V, long long vstride, int nv, const double* __restrict__ h,
             double* __restrict__ w, long long n2, double* __restrict__ partials, int mode) {
  pdl_enter();
  __shared__ double acc[kMaxVec][kThreads / 32];
  __shared__ double hs[kMaxVec];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nacc = mode == 0 ? nv : 1;
  for (int i = threadIdx.x; i < nacc * (kThreads / 32); i += blockDim.x) acc[i / (kThreads / 32)][i % (kThreads / 32)] = 0.0;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) hs[i] = h[i];
  __syncthreads();
  double2* w2 = reinterpret_cast<double2*>(w);
  const long long step = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e - threadIdx.x < n2; e += 2 * step) {
    const long long e1 = e + step;
    const bool ok0 = e < n2, ok1 = e1 < n2;
    double2 w0 = ok0 ? w2[e] : make_double2(0.0, 0.0);
    double2 wv1 = ok1 ? w2[e1] : make_double2(0.0, 0.0);
    for (int i = 0; i < nv; ++i) {
      const double2* v2 = reinterpret_cast<const double2*>(V + i * vstride);
      const double2 a = ok0 ? __ldg(v2 + e) : make_double2(0.0, 0.0);
      const double2 b = ok1 ? __ldg(v2 + e1) : make_double2(0.0, 0.0);
      const double hi = hs[i];
      w0.x -= hi * a.x;
      w0.y -= hi * a.y;
      wv1.x -= hi * b.x;
      wv1.y -= hi * b.y;
    }
    if (ok0) w2[e] = w0;
    if (ok1) w2[e1] = wv1;
    if (mode == 0) {
      for (int i = 0; i < nv; ++i) {
        const double2* v2 = reinterpret_cast<const double2*>(V + i * vstride);
        const double2 a = ok0 ? __ldg(v2 + e) : make_double2(0.0, 0.0);
        const double2 b = ok1 ? __ldg(v2 + e1) : make_double2(0.0, 0.0);
        double s = warp_sum((a.x * w0.x + a.y * w0.y) + (b.x * wv1.x + b.y * wv1.y));
        if (lane == 0) acc[i][warp] += s;
      }
    } else {
      double s = warp_sum((w0.x * w0.x + w0.y * w0.y) + (wv1.x * wv1.x + wv1.y * wv1.y));
      if (lane == 0) acc[0][warp] += s;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nacc; i += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < kThreads / 32; ++k) s += acc[i][k];
    partials[i * kRedBlocks + blockIdx.x] = s;
  }
}

// Delayed-reorthogonalisation Arnoldi, pass A: finish the previous basis
// vector and project the new operator output on the whole basis in ONE read
// of the basis.  q_k = (s_k - sum_{i<k} c_i Q_i) * inv_gamma is written over
// the provisional s_k (slot k); partials of Q_i . w for i <= k.
__global__ void __launch_bounds__(kThreads)
k_dcgs_a(double* __restrict__ Q, long long vstride, int k, const double* __restrict__ c, double inv_gamma,
         const double* __restrict__ w, long long n2, double* __restrict__ partials) {
  pdl_enter();
  __shared__ double acc[kMaxVec][kThreads / 32];
  __shared__ double cs[kMaxVec];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nv = k + 1;
  for (int i = threadIdx.x; i < nv * (kThreads / 32); i += blockDim.x) acc[i / (kThreads / 32)][i % (kThreads / 32)] = 0.0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) cs[i] = c[i];
  __syncthreads();
  const double2* w2 = reinterpret_cast<const double2*>(w);
  double2* s2 = reinterpret_cast<double2*>(Q + k * vstride);
  const long long step = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e - threadIdx.x < n2; e += 2 * step) {
    const long long e1 = e + step;
    const bool ok0 = e < n2, ok1 = e1 < n2;
    const double2 w0 = ok0 ? __ldg(w2 + e) : make_double2(0.0, 0.0);
    const double2 wv1 = ok1 ? __ldg(w2 + e1) : make_double2(0.0, 0.0);
    double2 q0 = ok0 ? s2[e] : make_double2(0.0, 0.0);
    double2 q1 = ok1 ? s2[e1] : make_double2(0.0, 0.0);
    for (int i = 0; i < k; ++i) {
      const double2* v2 = reinterpret_cast<const double2*>(Q + i * vstride);
      const double2 a = ok0 ? __ldg(v2 + e) : make_double2(0.0, 0.0);
      const double2 b = ok1 ? __ldg(v2 + e1) : make_double2(0.0, 0.0);
      const double ci = cs[i];
      q0.x -= ci * a.x;
      q0.y -= ci * a.y;
      q1.x -= ci * b.x;
      q1.y -= ci * b.y;
      const double sdot = warp_sum((a.x * w0.x + a.y * w0.y) + (b.x * wv1.x + b.y * wv1.y));
      if (lane == 0) acc[i][warp] += sdot;
    }
    if (k > 0) {
      q0.x *= inv_gamma;
      q0.y *= inv_gamma;
      q1.x *= inv_gamma;
      q1.y *= inv_gamma;
      if (ok0) s2[e] = q0;
      if (ok1) s2[e1] = q1;
    }
    const double sdot = warp_sum((q0.x * w0.x + q0.y * w0.y) + (q1.x * wv1.x + q1.y * wv1.y));
    if (lane == 0) acc[k][warp] += sdot;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    double s = 0.0;
    for (int kk = 0; kk < kThreads / 32; ++kk) s += acc[i][kk];
    partials[i * kRedBlocks + blockIdx.x] = s;
  }
}

// pass B: w' = w - sum_i d_i Q_i written to `out`, partials of Q_i . w' (slots
// 0..nv-1) and ||w'||^2 (slot nv).  The second read of Q_i hits L1/L2.
__global__ void __launch_bounds__(kThreads)
k_dcgs_b(const double* __restrict__ Q, long long vstride, int nv, const double* __restrict__ d,
         const double* __restrict__ w, double* __restrict__ out, long long n2, double* __restrict__ partials) {
  pdl_enter();
  __shared__ double acc[kMaxVec + 1][kThreads / 32];
  __shared__ double ds[kMaxVec];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (nv + 1) * (kThreads / 32); i += blockDim.x) acc[i / (kThreads / 32)][i % (kThreads / 32)] = 0.0;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) ds[i] = d[i];
  __syncthreads();
  const double2* w2 = reinterpret_cast<const double2*>(w);
  double2* o2 = reinterpret_cast<double2*>(out);
  const long long step = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e - threadIdx.x < n2; e += 2 * step) {
    const long long e1 = e + step;
    const bool ok0 = e < n2, ok1 = e1 < n2;
    double2 w0 = ok0 ? __ldg(w2 + e) : make_double2(0.0, 0.0);
    double2 wv1 = ok1 ? __ldg(w2 + e1) : make_double2(0.0, 0.0);
    for (int i = 0; i < nv; ++i) {
      const double2* v2 = reinterpret_cast<const double2*>(Q + i * vstride);
      const double2 a = ok0 ? __ldg(v2 + e) : make_double2(0.0, 0.0);
      const double2 b = ok1 ? __ldg(v2 + e1) : make_double2(0.0, 0.0);
      const double di = ds[i];
      w0.x -= di * a.x;
      w0.y -= di * a.y;
      wv1.x -= di * b.x;
      wv1.y -= di * b.y;
    }
    if (ok0) o2[e] = w0;
    if (ok1) o2[e1] = wv1;
    for (int i = 0; i < nv; ++i) {
      const double2* v2 = reinterpret_cast<const double2*>(Q + i * vstride);
      const double2 a = ok0 ? __ldg(v2 + e) : make_double2(0.0, 0.0);
      const double2 b = ok1 ? __ldg(v2 + e1) : make_double2(0.0, 0.0);
      const double sdot = warp_sum((a.x * w0.x + a.y * w0.y) + (b.x * wv1.x + b.y * wv1.y));
      if (lane == 0) acc[i][warp] += sdot;
    }
    const double nn = warp_sum((w0.x * w0.x + w0.y * w0.y) + (wv1.x * wv1.x + wv1.y * wv1.y));
    if (lane == 0) acc[nv][warp] += nn;
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= nv; i += blockDim.x) {
    double s = 0.0;
    for (int kk = 0; kk < kThreads / 32; ++kk) s += acc[i][kk];
    partials[i * kRedBlocks + blockIdx.x] = s;
  }
}

// pass B with the basis values of the current tile stashed in shared memory:
// every Q_i streams from HBM exactly once (the dots re-read the stash).
constexpr int kStashThreads = 128;
__global__ void __launch_bounds__(kStashThreads)
k_dcgs_b_stash(const double* __restrict__ Q, long long vstride, int nv, const double* __restrict__ d,
               const double* __restrict__ w, double* __restrict__ out, long long n2, double* __restrict__ partials) {
  pdl_enter();
  extern __shared__ double2 stash[];  // [nv][kStashThreads]
  __shared__ double acc[kMaxVec + 1][kStashThreads / 32];
  __shared__ double ds[kMaxVec];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (nv + 1) * (kStashThreads / 32); i += blockDim.x)
    acc[i / (kStashThreads / 32)][i % (kStashThreads / 32)] = 0.0;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) ds[i] = d[i];
  __syncthreads();
  const double2* w2 = reinterpret_cast<const double2*>(w);
  double2* o2 = reinterpret_cast<double2*>(out);
  const long long step = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e - threadIdx.x < n2; e += step) {
    const bool ok = e < n2;
    double2 wv = ok ? __ldg(w2 + e) : make_double2(0.0, 0.0);
    for (int i = 0; i < nv; ++i) {
      const double2 a = ok ? __ldg(reinterpret_cast<const double2*>(Q + i * vstride) + e) : make_double2(0.0, 0.0);
      stash[i * kStashThreads + threadIdx.x] = a;
      const double di = ds[i];
      wv.x -= di * a.x;
      wv.y -= di * a.y;
    }
    if (ok) o2[e] = wv;
    for (int i = 0; i < nv; ++i) {
      const double2 a = stash[i * kStashThreads + threadIdx.x];
      const double sdot = warp_sum(a.x * wv.x + a.y * wv.y);
      if (lane == 0) acc[i][warp] += sdot;
    }
    const double nn = warp_sum(wv.x * wv.x + wv.y * wv.y);
    if (lane == 0) acc[nv][warp] += nn;
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= nv; i += blockDim.x) {
    double s = 0.0;
    for (int kk = 0; kk < kStashThreads / 32; ++kk) s += acc[i][kk];
    partials[i * kRedBlocks + blockIdx.x] = s;
  }
}

// pass B, L2-resident variant: a bounded grid (2 CTAs/SM) so the tile of the
// basis read by the update loop is still in L2 (126 MB) when the dot loop
// re-reads it; the update loop is unrolled for memory-level parallelism.
constexpr int kL2Blocks = kSMs * 2;
__global__ void __launch_bounds__(kThreads)
k_dcgs_b_l2(const double* __restrict__ Q, long long vstride, int nv, const double* __restrict__ d,
            const double* __restrict__ w, double* __restrict__ out, long long n2, double* __restrict__ partials) {
  pdl_enter();
  __shared__ double acc[kMaxVec + 1][kThreads / 32];
  __shared__ double ds[kMaxVec];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (nv + 1) * (kThreads / 32); i += blockDim.x) acc[i / (kThreads / 32)][i % (kThreads / 32)] = 0.0;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) ds[i] = d[i];
  __syncthreads();
  const double2* w2 = reinterpret_cast<const double2*>(w);
  double2* o2 = reinterpret_cast<double2*>(out);
  const long long step = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e - threadIdx.x < n2; e += step) {
    const bool ok = e < n2;
    double2 wv = ok ? __ldg(w2 + e) : make_double2(0.0, 0.0);
    int i = 0;
    for (; i + 8 <= nv; i += 8) {
      double2 a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        a[u] = ok ? __ldg(reinterpret_cast<const double2*>(Q + (i + u) * vstride) + e) : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        wv.x -= ds[i + u] * a[u].x;
        wv.y -= ds[i + u] * a[u].y;
      }
    }
    for (; i < nv; ++i) {
      const double2 a = ok ? __ldg(reinterpret_cast<const double2*>(Q + i * vstride) + e) : make_double2(0.0, 0.0);
      wv.x -= ds[i] * a.x;
      wv.y -= ds[i] * a.y;
    }
    if (ok) o2[e] = wv;
    i = 0;
    for (; i + 8 <= nv; i += 8) {
      double2 a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        a[u] = ok ? __ldg(reinterpret_cast<const double2*>(Q + (i + u) * vstride) + e) : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double sdot = warp_sum(a[u].x * wv.x + a[u].y * wv.y);
        if (lane == 0) acc[i + u][warp] += sdot;
      }
    }
    for (; i < nv; ++i) {
      const double2 a = ok ? __ldg(reinterpret_cast<const double2*>(Q + i * vstride) + e) : make_double2(0.0, 0.0);
      const double sdot = warp_sum(a.x * wv.x + a.y * wv.y);
      if (lane == 0) acc[i][warp] += sdot;
    }
    const double nn = warp_sum(wv.x * wv.x + wv.y * wv.y);
    if (lane == 0) acc[nv][warp] += nn;
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= nv; i += blockDim.x) {
    double s = 0.0;
    for (int kk = 0; kk < kThreads / 32; ++kk) s += acc[i][kk];
    partials[i * kRedBlocks + blockIdx.x] = s;
  }
}

// Gram variant, pass A: like k_dcgs_a, plus the dots Q_l . s_k (l < k) and
// s_k . s_k of the provisional vector, from which the host extends the Gram
// matrix of the basis.  Partial slots: [0..k] Q.w with the finished q_k,
// [k+1..2k] Q_l . s_k, [2k+1] s_k . s_k.
__global__ void __launch_bounds__(kThreads)
k_dcgs_a_g(double* __restrict__ Q, long long vstride, int k, const double* __restrict__ c, double inv_gamma,
           const double* __restrict__ w, long long n2, double* __restrict__ partials) {
  pdl_enter();
  __shared__ double acc[2 * kMaxVec + 2][kThreads / 32];
  __shared__ double cs[kMaxVec];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nslot = 2 * k + 2;
  for (int i = threadIdx.x; i < nslot * (kThreads / 32); i += blockDim.x) acc[i / (kThreads / 32)][i % (kThreads / 32)] = 0.0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) cs[i] = c[i];
  __syncthreads();
  const double2* w2 = reinterpret_cast<const double2*>(w);
  double2* s2 = reinterpret_cast<double2*>(Q + k * vstride);
  const long long step = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e - threadIdx.x < n2; e += 2 * step) {
    const long long e1 = e + step;
    const bool ok0 = e < n2, ok1 = e1 < n2;
    const double2 w0 = ok0 ? __ldg(w2 + e) : make_double2(0.0, 0.0);
    const double2 wv1 = ok1 ? __ldg(w2 + e1) : make_double2(0.0, 0.0);
    const double2 sa = ok0 ? s2[e] : make_double2(0.0, 0.0);
    const double2 sb = ok1 ? s2[e1] : make_double2(0.0, 0.0);
    double2 q0 = sa, q1 = sb;
    for (int i = 0; i < k; ++i) {
      const double2* v2 = reinterpret_cast<const double2*>(Q + i * vstride);
      const double2 a = ok0 ? __ldg(v2 + e) : make_double2(0.0, 0.0);
      const double2 b = ok1 ? __ldg(v2 + e1) : make_double2(0.0, 0.0);
      const double ci = cs[i];
      q0.x -= ci * a.x;
      q0.y -= ci * a.y;
      q1.x -= ci * b.x;
      q1.y -= ci * b.y;
      const double dw = warp_sum((a.x * w0.x + a.y * w0.y) + (b.x * wv1.x + b.y * wv1.y));
      const double dsv = warp_sum((a.x * sa.x + a.y * sa.y) + (b.x * sb.x + b.y * sb.y));
      if (lane == 0) {
        acc[i][warp] += dw;
        acc[k + 1 + i][warp] += dsv;
      }
    }
    if (k > 0) {
      q0.x *= inv_gamma;
      q0.y *= inv_gamma;
      q1.x *= inv_gamma;
      q1.y *= inv_gamma;
      if (ok0) s2[e] = q0;
      if (ok1) s2[e1] = q1;
    }
    const double dq = warp_sum((q0.x * w0.x + q0.y * w0.y) + (q1.x * wv1.x + q1.y * wv1.y));
    const double ss = warp_sum((sa.x * sa.x + sa.y * sa.y) + (sb.x * sb.x + sb.y * sb.y));
    if (lane == 0) {
      acc[k][warp] += dq;
      acc[2 * k + 1][warp] += ss;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nslot; i += blockDim.x) {
    double s = 0.0;
    for (int kk = 0; kk < kThreads / 32; ++kk) s += acc[i][kk];
    partials[i * kRedBlocks + blockIdx.x] = s;
  }
}

// Same as k_dcgs_a_g, register-chunked: every thread owns CH double2 of each
// vector per step, so the two warp reductions per basis vector are amortised
// over 2*CH elements (instead of 4) and CH independent loads are in flight.
template <int CH>
__global__ void __launch_bounds__(kThreads)
k_dcgs_a_g2(double* __restrict__ Q, long long vstride, int k, const double* __restrict__ c, double inv_gamma,
            const double* __restrict__ w, long long n2, double* __restrict__ partials,
            const double* __restrict__ /*means: A/B variant without the deferral*/, long long /*bb*/,
            double* __restrict__ /*wout*/, long long /*gh*/) {
  pdl_enter();
  __shared__ double acc[2 * kMaxVec + 2][kThreads / 32];
  __shared__ double cs[kMaxVec];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nslot = 2 * k + 2;
  for (int i = threadIdx.x; i < nslot * (kThreads / 32); i += blockDim.x) acc[i / (kThreads / 32)][i % (kThreads / 32)] = 0.0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) cs[i] = c[i];
  __syncthreads();
  const double2* w2 = reinterpret_cast<const double2*>(w);
  double2* s2 = reinterpret_cast<double2*>(Q + k * vstride);
  const long long span = (long long)blockDim.x * CH;
  for (long long base = blockIdx.x * span; base < n2; base += (long long)gridDim.x * span) {
    double2 wv[CH], sv[CH], q[CH];
    bool ok[CH];
#pragma unroll
    for (int t = 0; t < CH; ++t) {
      const long long e = base + t * blockDim.x + threadIdx.x;
      ok[t] = e < n2;
      wv[t] = ok[t] ? __ldg(w2 + e) : make_double2(0.0, 0.0);
      sv[t] = ok[t] ? s2[e] : make_double2(0.0, 0.0);
      q[t] = sv[t];
    }
    for (int i = 0; i < k; ++i) {
      const double2* v2 = reinterpret_cast<const double2*>(Q + i * vstride);
      double2 a[CH];
#pragma unroll
      for (int t = 0; t < CH; ++t) a[t] = ok[t] ? __ldg(v2 + base + t * blockDim.x + threadIdx.x) : make_double2(0.0, 0.0);
      const double ci = cs[i];
      double dw = 0.0, dsv = 0.0;
#pragma unroll
      for (int t = 0; t < CH; ++t) {
        q[t].x -= ci * a[t].x;
        q[t].y -= ci * a[t].y;
        dw += a[t].x * wv[t].x + a[t].y * wv[t].y;
        dsv += a[t].x * sv[t].x + a[t].y * sv[t].y;
      }
      dw = warp_sum(dw);
      dsv = warp_sum(dsv);
      if (lane == 0) {
        acc[i][warp] += dw;
        acc[k + 1 + i][warp] += dsv;
      }
    }
    double dq = 0.0, ss = 0.0;
#pragma unroll
    for (int t = 0; t < CH; ++t) {
      if (k > 0) {
        q[t].x *= inv_gamma;
        q[t].y *= inv_gamma;
        if (ok[t]) s2[base + t * blockDim.x + threadIdx.x] = q[t];
      }
      dq += q[t].x * wv[t].x + q[t].y * wv[t].y;
      ss += sv[t].x * sv[t].x + sv[t].y * sv[t].y;
    }
    dq = warp_sum(dq);
    ss = warp_sum(ss);
    if (lane == 0) {
      acc[k][warp] += dq;
      acc[2 * k + 1][warp] += ss;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nslot; i += blockDim.x) {
    double s = 0.0;
    for (int kk = 0; kk < kThreads / 32; ++kk) s += acc[i][kk];
    partials[i * kRedBlocks + blockIdx.x] = s;
  }
}

// Butterfly transpose-reduction of V (power of two, <= 32) per-lane values
// across the warp: V-1 + (5 - log2 V) shuffles instead of 5 V.  On return
// v[0] of lane L holds the warp sum of value (L & (V-1)).
template <int V>
__device__ __forceinline__ double warp_sum_many(double* v, int lane) {
#pragma unroll
  for (int w = V, s = 1; w > 1; w >>= 1, s <<= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int j = 0; j < w / 2; ++j) {
      const double keep = up ? v[2 * j + 1] : v[2 * j];
      const double send = up ? v[2 * j] : v[2 * j + 1];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  double r = v[0];
#pragma unroll
  for (int s = V; s < 32; s <<= 1) r += __shfl_xor_sync(0xffffffffu, r, s);
  return r;
}

// Pass A with the basis read G vectors at a time: G*CH independent 16-B loads
// per thread in flight, and the 2G dot products of a group reduced across the
// warp by one transpose-reduction (2G-1 + 5-log2(2G) shuffles instead of 10G).
// q_j = (s - sum_i c_i Q_i) * inv_gamma keeps the ascending-i update order.
// MEANS: the null-space projection deferred from P^-1 is applied to w on
// load (w - means[b] on the b-th block of bb double2, pass B's expression), so
// d = Q^T (projected w) is exactly what pass B subtracts: the Gram identity
// c' = d - G d then holds to roundoff even when the means dominate w (near a
// breakdown, where Q^T 1 = O(eps) would otherwise leak into d).
//
// W1 (one-pass Arnoldi, sb_solver.cu gmres): also ||w||^2 (slot 2k+2) and w
// (projected by the means) stored to wout = basis slot k+1 -- the next
// step's unfinished vector, whose pending projection the next pass A applies,
// so no second stream over the basis.  gh: slab blocks keep their first / last
// gh double2 (ghost planes) at 0, the means are not applied there.
template <int CH, int G, int MB = 2, bool MEANS = false, bool W1 = false>
__global__ void __launch_bounds__(kThreads, MB)
k_dcgs_a_g3(double* __restrict__ Q, long long vstride, int k, const double* __restrict__ c, double inv_gamma,
            const double* __restrict__ w, long long n2, double* __restrict__ partials,
            const double* __restrict__ means = nullptr, long long bb = 0, double* __restrict__ wout = nullptr,
            long long gh = 0) {
  pdl_enter();
  __shared__ double acc[2 * kMaxVec + 2][kThreads / 32];
  __shared__ double cs[kMaxVec];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nslot = 2 * k + 2 + (W1 ? 1 : 0);
  for (int i = threadIdx.x; i < nslot * (kThreads / 32); i += blockDim.x) acc[i / (kThreads / 32)][i % (kThreads / 32)] = 0.0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) cs[i] = c[i];
  __syncthreads();
  const double2* w2 = reinterpret_cast<const double2*>(w);
  double2* s2 = reinterpret_cast<double2*>(Q + k * vstride);
  const long long span = (long long)blockDim.x * CH;
  for (long long base = blockIdx.x * span; base < n2; base += (long long)gridDim.x * span) {
    double2 wv[CH], sv[CH], q[CH];
    bool ok[CH];
    // when the chunk [base, base + span) crosses at most one block boundary
    // (span <= bb, every production size): its two candidate means, chosen per
    // element by one compare; tiny vectors take the per-element block index
    long long bnd = 0;
    double m_lo = 0.0, m_hi = 0.0;
    int b_lo = 0;
    const bool chunked = span <= bb;
    if (MEANS && chunked) {
      b_lo = (base >= bb) + (base >= 2 * bb) + (base >= 3 * bb);
      bnd = (long long)(b_lo + 1) * bb;
      m_lo = __ldg(means + b_lo);
      m_hi = b_lo < 3 ? __ldg(means + b_lo + 1) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < CH; ++t) {
      const long long e = base + t * blockDim.x + threadIdx.x;
      ok[t] = e < n2;
      wv[t] = ok[t] ? __ldg(w2 + e) : make_double2(0.0, 0.0);
      if (MEANS && ok[t]) {
        const int bf = chunked ? (e < bnd ? b_lo : b_lo + 1) : (e >= bb) + (e >= 2 * bb) + (e >= 3 * bb);
        double m = chunked ? (e < bnd ? m_lo : m_hi) : __ldg(means + bf);
        if (gh) {
          const int bi = bf;
          const long long la = e - bi * bb;
          if (la < gh || la >= bb - gh) m = 0.0;
        }
        wv[t].x = wv[t].x - m;
        wv[t].y = wv[t].y - m;
      }
      sv[t] = ok[t] ? s2[e] : make_double2(0.0, 0.0);
      q[t] = sv[t];
    }
    int i = 0;
    for (; i + G <= k; i += G) {
      double2 a[G][CH];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const double2* v2 = reinterpret_cast<const double2*>(Q + (i + g) * vstride);
#pragma unroll
        for (int t = 0; t < CH; ++t)
          a[g][t] = ok[t] ? __ldg(v2 + base + t * blockDim.x + threadIdx.x) : make_double2(0.0, 0.0);
      }
      double dv[2 * G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const double ci = cs[i + g];
        double dw = 0.0, dsv = 0.0;
#pragma unroll
        for (int t = 0; t < CH; ++t) {
          q[t].x -= ci * a[g][t].x;
          q[t].y -= ci * a[g][t].y;
          dw += a[g][t].x * wv[t].x + a[g][t].y * wv[t].y;
          dsv += a[g][t].x * sv[t].x + a[g][t].y * sv[t].y;
        }
        dv[2 * g] = dw;
        dv[2 * g + 1] = dsv;
      }
      const double r = warp_sum_many<2 * G>(dv, lane);
      if (lane < 2 * G) {
        const int g = lane >> 1;
        acc[(lane & 1) ? k + 1 + i + g : i + g][warp] += r;
      }
    }
    for (; i < k; ++i) {
      const double2* v2 = reinterpret_cast<const double2*>(Q + i * vstride);
      double2 a[CH];
#pragma unroll
      for (int t = 0; t < CH; ++t) a[t] = ok[t] ? __ldg(v2 + base + t * blockDim.x + threadIdx.x) : make_double2(0.0, 0.0);
      const double ci = cs[i];
      double dv[2] = {0.0, 0.0};
#pragma unroll
      for (int t = 0; t < CH; ++t) {
        q[t].x -= ci * a[t].x;
        q[t].y -= ci * a[t].y;
        dv[0] += a[t].x * wv[t].x + a[t].y * wv[t].y;
        dv[1] += a[t].x * sv[t].x + a[t].y * sv[t].y;
      }
      const double r = warp_sum_many<2>(dv, lane);
      if (lane < 2) acc[lane ? k + 1 + i : i][warp] += r;
    }
    if (W1) {
      double dv[4] = {0.0, 0.0, 0.0, 0.0};
      double2* o2 = reinterpret_cast<double2*>(wout);
#pragma unroll
      for (int t = 0; t < CH; ++t) {
        if (k > 0) {
          q[t].x *= inv_gamma;
          q[t].y *= inv_gamma;
          if (ok[t]) s2[base + t * blockDim.x + threadIdx.x] = q[t];
        }
        if (ok[t]) o2[base + t * blockDim.x + threadIdx.x] = wv[t];
        dv[0] += q[t].x * wv[t].x + q[t].y * wv[t].y;
        dv[1] += sv[t].x * sv[t].x + sv[t].y * sv[t].y;
        dv[2] += wv[t].x * wv[t].x + wv[t].y * wv[t].y;
      }
      const double r = warp_sum_many<4>(dv, lane);
      if (lane < 3) acc[lane == 0 ? k : (lane == 1 ? 2 * k + 1 : 2 * k + 2)][warp] += r;
    } else {
      double dv[2] = {0.0, 0.0};
#pragma unroll
      for (int t = 0; t < CH; ++t) {
        if (k > 0) {
          q[t].x *= inv_gamma;
          q[t].y *= inv_gamma;
          if (ok[t]) s2[base + t * blockDim.x + threadIdx.x] = q[t];
        }
        dv[0] += q[t].x * wv[t].x + q[t].y * wv[t].y;
        dv[1] += sv[t].x * sv[t].x + sv[t].y * sv[t].y;
      }
      const double r = warp_sum_many<2>(dv, lane);
      if (lane < 2) acc[lane ? 2 * k + 1 : k][warp] += r;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nslot; i += blockDim.x) {
    double s = 0.0;
    for (int kk = 0; kk < kThreads / 32; ++kk) s += acc[i][kk];
    partials[i * kRedBlocks + blockIdx.x] = s;
  }
}

// ---------------------------------------------------------------------------
// Pass A with the basis staged by the TMA (cp.async.bulk, sm_100a).
//
// k_dcgs_a_g3 keeps G*CH 16-byte basis loads per thread in registers (120
// registers, 16 resident warps per SM) and reaches 6.1 TB/s where pass B, at
// 47 registers, reaches 6.8 TB/s (ncu): pass A is short of bytes in flight.
// Here thread 0 streams each basis vector's chunk (CH * 256 double2 = 16 KB)
// into an S-deep shared-memory ring with one bulk copy per stage
// (cp.async.bulk.shared::cluster.global, completion on an mbarrier); the
// CTA's threads wait on the stage's mbarrier, read their own elements with
// conflict-free 16-byte shared loads and, after a __syncthreads, thread 0
// refills the stage with the chunk S steps ahead -- across chunk boundaries,
// so the ring never drains.  w and s_j of a chunk come through the ring too
// (then live in registers while the basis streams past).  Same
// element-to-thread mapping, same accumulation order: bit-identical to
// k_dcgs_a_g3<4, 2>.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  const unsigned a = smem_u32(bar);
  unsigned ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(phase)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

constexpr int kTmaCH = 4;      // double2 per thread per chunk (as k_dcgs_a_g3<4, 2>)
constexpr int kTmaStages = 4;  // ring depth: 4 x 16 KB per CTA

template <bool MEANS>
__global__ void __launch_bounds__(kThreads, 2)
k_dcgs_a_tma(double* __restrict__ Q, long long vstride, int k, const double* __restrict__ c, double inv_gamma,
             const double* __restrict__ w, long long n2, double* __restrict__ partials,
             const double* __restrict__ means, long long bb) {
  pdl_enter();
  constexpr int CH = kTmaCH, S = kTmaStages, G = 2;
  extern __shared__ __align__(128) unsigned char dsm[];
  double2* const ring = reinterpret_cast<double2*>(dsm);  // [S][kThreads * CH]
  __shared__ unsigned long long full[S];
  __shared__ double acc[2 * kMaxVec + 2][kThreads / 32];
  __shared__ double cs[kMaxVec];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nslot = 2 * k + 2;
  for (int i = threadIdx.x; i < nslot * (kThreads / 32); i += blockDim.x) acc[i / (kThreads / 32)][i % (kThreads / 32)] = 0.0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) cs[i] = c[i];
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double2* s2 = reinterpret_cast<double2*>(Q + k * vstride);
  const long long span = (long long)blockDim.x * CH;
  const long long gstep = (long long)gridDim.x * span;
  const long long first = blockIdx.x * span;
  const long long nchunk = first < n2 ? (n2 - first + gstep - 1) / gstep : 0;
  // stage loads of this CTA, in order: per chunk w, s_j, Q_0 .. Q_{k-1}
  const int kk = k + 2;
  const long long total = nchunk * kk;
  // producer (thread 0): stage load number L
  auto issue = [&](long long L) {
    const long long ci = L / kk;
    const int r = (int)(L - ci * kk);
    const long long base = first + ci * gstep;
    const unsigned bytes = (unsigned)((n2 - base < span ? n2 - base : span) * sizeof(double2));
    const int slot = (int)(L % S);
    const double* src = r == 0 ? w : (r == 1 ? Q + (long long)k * vstride : Q + (long long)(r - 2) * vstride);
    mbar_expect_tx(&full[slot], bytes);
    bulk_g2s(ring + (long long)slot * span, reinterpret_cast<const double2*>(src) + base, bytes, &full[slot]);
  };
  long long Lp = 0, Lc = 0;
  if (threadIdx.x == 0)
    for (; Lp < S && Lp < total; ++Lp) issue(Lp);
  for (long long base = first; base < n2; base += gstep) {
    double2 wv[CH], sv[CH], q[CH];
    bool ok[CH];
    long long bnd = 0;
    double m_lo = 0.0, m_hi = 0.0;
    int b_lo = 0;
    const bool chunked = span <= bb;
    if (MEANS && chunked) {
      b_lo = (base >= bb) + (base >= 2 * bb) + (base >= 3 * bb);
      bnd = (long long)(b_lo + 1) * bb;
      m_lo = __ldg(means + b_lo);
      m_hi = b_lo < 3 ? __ldg(means + b_lo + 1) : 0.0;
    }
    // w and s_j of the chunk arrive through the ring like the basis
    mbar_wait(&full[Lc % S], (unsigned)((Lc / S) & 1));
    mbar_wait(&full[(Lc + 1) % S], (unsigned)(((Lc + 1) / S) & 1));
    const double2* stw = ring + (Lc % S) * span + threadIdx.x;
    const double2* sts = ring + ((Lc + 1) % S) * span + threadIdx.x;
#pragma unroll
    for (int t = 0; t < CH; ++t) {
      const long long e = base + t * blockDim.x + threadIdx.x;
      ok[t] = e < n2;
      wv[t] = ok[t] ? stw[t * blockDim.x] : make_double2(0.0, 0.0);
      if (MEANS && ok[t]) {
        const int bf = chunked ? (e < bnd ? b_lo : b_lo + 1) : (e >= bb) + (e >= 2 * bb) + (e >= 3 * bb);
        const double m = chunked ? (e < bnd ? m_lo : m_hi) : __ldg(means + bf);
        wv[t].x = wv[t].x - m;
        wv[t].y = wv[t].y - m;
      }
      sv[t] = ok[t] ? sts[t * blockDim.x] : make_double2(0.0, 0.0);
      q[t] = sv[t];
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int g = 0; g < 2 && Lp < total; ++g, ++Lp) issue(Lp);
    Lc += 2;
    int i = 0;
    for (; i + G <= k; i += G) {
      const double2* st[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const long long L = Lc + g;
        mbar_wait(&full[L % S], (unsigned)((L / S) & 1));
        st[g] = ring + (L % S) * span + threadIdx.x;
      }
      double dv[2 * G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const double ci = cs[i + g];
        double dw = 0.0, dsv = 0.0;
#pragma unroll
        for (int t = 0; t < CH; ++t) {
          const double2 a = ok[t] ? st[g][t * blockDim.x] : make_double2(0.0, 0.0);
          q[t].x -= ci * a.x;
          q[t].y -= ci * a.y;
          dw += a.x * wv[t].x + a.y * wv[t].y;
          dsv += a.x * sv[t].x + a.y * sv[t].y;
        }
        dv[2 * g] = dw;
        dv[2 * g + 1] = dsv;
      }
      __syncthreads();  // every thread has read its elements: the two stages can be refilled
      if (threadIdx.x == 0)
        for (int g = 0; g < G && Lp < total; ++g, ++Lp) issue(Lp);
      Lc += G;
      const double r = warp_sum_many<2 * G>(dv, lane);
      if (lane < 2 * G) {
        const int g = lane >> 1;
        acc[(lane & 1) ? k + 1 + i + g : i + g][warp] += r;
      }
    }
    for (; i < k; ++i) {
      double2 a[CH];
      mbar_wait(&full[Lc % S], (unsigned)((Lc / S) & 1));
      const double2* st = ring + (Lc % S) * span;
#pragma unroll
      for (int t = 0; t < CH; ++t) a[t] = ok[t] ? st[t * blockDim.x + threadIdx.x] : make_double2(0.0, 0.0);
      __syncthreads();
      if (threadIdx.x == 0 && Lp < total) issue(Lp++);
      ++Lc;
      const double ci = cs[i];
      double dv[2] = {0.0, 0.0};
#pragma unroll
      for (int t = 0; t < CH; ++t) {
        q[t].x -= ci * a[t].x;
        q[t].y -= ci * a[t].y;
        dv[0] += a[t].x * wv[t].x + a[t].y * wv[t].y;
        dv[1] += a[t].x * sv[t].x + a[t].y * sv[t].y;
      }
      const double r = warp_sum_many<2>(dv, lane);
      if (lane < 2) acc[lane ? k + 1 + i : i][warp] += r;
    }
    double dv[2] = {0.0, 0.0};
#pragma unroll
    for (int t = 0; t < CH; ++t) {
      if (k > 0) {
        q[t].x *= inv_gamma;
        q[t].y *= inv_gamma;
        if (ok[t]) s2[base + t * blockDim.x + threadIdx.x] = q[t];
      }
      dv[0] += q[t].x * wv[t].x + q[t].y * wv[t].y;
      dv[1] += sv[t].x * sv[t].x + sv[t].y * sv[t].y;
    }
    const double r = warp_sum_many<2>(dv, lane);
    if (lane < 2) acc[lane ? 2 * k + 1 : k][warp] += r;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nslot; i += blockDim.x) {
    double s = 0.0;
    for (int kk = 0; kk < kThreads / 32; ++kk) s += acc[i][kk];
    partials[i * kRedBlocks + blockIdx.x] = s;
  }
}

// Gram variant, pass B: w' = w - sum_i d_i Q_i written to `out`, ||w'||^2 only
// (one streaming read of the basis).  means (nullable): the null-space
// projection of w deferred from P^-1 -- w - means[b] on the b-th block of
// bb double2 (the k_box_sub_mean expression, so w' is unchanged to the bit).
// GH (slab blocks): the first and last gh double2 of each block are ghost
// planes and keep 0 (a separate instantiation: the single-domain kernel's code
// generation -- 47 registers, 5 CTAs/SM -- is unchanged).
template <bool GH>
__global__ void __launch_bounds__(kThreads)
k_dcgs_b_g(const double* __restrict__ Q, long long vstride, int nv, const double* __restrict__ d,
           const double* __restrict__ w, double* __restrict__ out, long long n2, double* __restrict__ partials,
           const double* __restrict__ means, long long bb, long long gh) {
  pdl_enter();
  __shared__ double acc[kThreads / 32];
  __shared__ double ds[kMaxVec];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < kThreads / 32) acc[threadIdx.x] = 0.0;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) ds[i] = d[i];
  const double m0 = means ? means[0] : 0.0, m1 = means ? means[1] : 0.0;
  const double m2 = means ? means[2] : 0.0, m3 = means ? means[3] : 0.0;
  __syncthreads();
  const double2* w2 = reinterpret_cast<const double2*>(w);
  double2* o2 = reinterpret_cast<double2*>(out);
  const long long step = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e - threadIdx.x < n2; e += 2 * step) {
    const long long e1 = e + step;
    const bool ok0 = e < n2, ok1 = e1 < n2;
    double2 w0 = ok0 ? __ldg(w2 + e) : make_double2(0.0, 0.0);
    double2 wv1 = ok1 ? __ldg(w2 + e1) : make_double2(0.0, 0.0);
    if (means) {
      const int b0 = (e >= bb) + (e >= 2 * bb) + (e >= 3 * bb);
      const int b1 = (e1 >= bb) + (e1 >= 2 * bb) + (e1 >= 3 * bb);
      double ma = b0 == 0 ? m0 : (b0 == 1 ? m1 : (b0 == 2 ? m2 : m3));
      double mb = b1 == 0 ? m0 : (b1 == 1 ? m1 : (b1 == 2 ? m2 : m3));
      if (GH) {  // slab blocks: the ghost planes at both block ends stay 0
        const long long la = e - b0 * bb, lb = e1 - b1 * bb;
        if (la < gh || la >= bb - gh) ma = 0.0;
        if (lb < gh || lb >= bb - gh) mb = 0.0;
      }
      if (ok0) {
        w0.x = w0.x - ma;
        w0.y = w0.y - ma;
      }
      if (ok1) {
        wv1.x = wv1.x - mb;
        wv1.y = wv1.y - mb;
      }
    }
    for (int i = 0; i < nv; ++i) {
      const double2* v2 = reinterpret_cast<const double2*>(Q + i * vstride);
      const double2 a = ok0 ? __ldg(v2 + e) : make_double2(0.0, 0.0);
      const double2 b = ok1 ? __ldg(v2 + e1) : make_double2(0.0, 0.0);
      const double di = ds[i];
      w0.x -= di * a.x;
      w0.y -= di * a.y;
      wv1.x -= di * b.x;
      wv1.y -= di * b.y;
    }
    if (ok0) o2[e] = w0;
    if (ok1) o2[e1] = wv1;
    const double nn = warp_sum((w0.x * w0.x + w0.y * w0.y) + (wv1.x * wv1.x + wv1.y * wv1.y));
    if (lane == 0) acc[warp] += nn;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int kk = 0; kk < kThreads / 32; ++kk) s += acc[kk];
    partials[blockIdx.x] = s;
  }
}

// out[i] = sum_b partials[i*kRedBlocks + b], fixed-order tree (deterministic)
__global__ void k_finalize(const double* __restrict__ partials, double* __restrict__ out, int nblocks) {
  pdl_enter();
  __shared__ double s[kThreads];
  const int i = blockIdx.x;
  double v = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) v += partials[i * kRedBlocks + b];
  s[threadIdx.x] = v;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[i] = s[0];
}

__global__ void __launch_bounds__(kThreads)
k_sum_partial(const double* __restrict__ x, long long n, double* __restrict__ partials) {
  pdl_enter();
  __shared__ double acc[kThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    v += __ldg(x + e);
  v = warp_sum(v);
  if (lane == 0) acc[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < kThreads / 32; ++k) s += acc[k];
    partials[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kThreads)
k_sub_norm(const double* __restrict__ a, const double* __restrict__ b, long long n,
           double* __restrict__ partials) {
  pdl_enter();
  __shared__ double acc[kThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const double d = __ldg(a + e) - __ldg(b + e);
    v += d * d;
  }
  v = warp_sum(v);
  if (lane == 0) acc[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < kThreads / 32; ++k) s += acc[k];
    partials[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kThreads)
k_scale_div(const double2* __restrict__ w, double d, double2* __restrict__ out, long long n2) {
  pdl_enter();
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n2;
       e += (long long)gridDim.x * blockDim.x) {
    double2 v = w[e];
    out[e] = make_double2(v.x / d, v.y / d);
  }
}

__global__ void __launch_bounds__(kThreads)
k_combo(double2* out, const double2* x, const double* __restrict__ V, long long vstride, int nv,
        const double* __restrict__ y, long long n2) {
  pdl_enter();
  __shared__ double ys[kMaxVec];
  for (int i = threadIdx.x; i < nv; i += blockDim.x) ys[i] = y[i];
  __syncthreads();
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n2;
       e += (long long)gridDim.x * blockDim.x) {
    double sx = 0.0, sy = 0.0;
    for (int i = 0; i < nv; ++i) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(V + i * vstride) + e);
      sx += ys[i] * v.x;
      sy += ys[i] * v.y;
    }
    const double2 xv = x[e];
    out[e] = make_double2(xv.x + sx, xv.y + sy);
  }
}

__global__ void __launch_bounds__(kThreads)
k_sub(const double2* __restrict__ a, const double2* __restrict__ b, double2* __restrict__ out, long long n2) {
  pdl_enter();
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n2;
       e += (long long)gridDim.x * blockDim.x) {
    const double2 x = a[e], y = b[e];
    out[e] = make_double2(x.x - y.x, x.y - y.y);
  }
}

// ---------------------------------------------------------------------------
// coarse-level tail of a V-cycle in ONE CTA (multigrid.py:391-439 below the
// chain's top level).  Levels of <= 16^3 cells are launch-latency bound: each
// colour pass / transfer is 1-2 us of work behind 3-5 us of launch and drain.
// Here every pass is a block-strided loop followed by __syncthreads, the
// iterate and right-hand sides are re-read with plain (coherent) loads, and
// the operation order is the multi-kernel V-cycle's, so results are
// identical to it.
// ---------------------------------------------------------------------------

constexpr int kCoarseThreads = 512;

__device__ __forceinline__ void cz_fill(double* x, long long n) {
  for (long long i = threadIdx.x; i < n; i += blockDim.x) x[i] = 0.0;
}

// one colour pass of component A on chain level C (k_face_colour's mapping)
template <int DIM, int FORM, int A, int PA>
__device__ void cf_colour(const CoarseLv& C, double omega, int parity) {
  const LevelDev& L = C.d;
  const Box b = face_box(L, DIM, A);
  const int off = (L.bclo[A] == BC_PER) ? 0 : 1;
  const int e1 = b.hi[1] - b.lo[1] + 1;
  const int half2 = (b.hi[2] - b.lo[2] + 2) / 2;
  const int total = (b.hi[0] - b.lo[0] + 1) * e1 * half2;
  double* const* x = C.x;
  const double* uc[3] = {x[0], x[1], x[2]};
  const double* rhs = C.rhs[A];
  for (int phase = 0; phase < (C.two_phase ? 2 : 1); ++phase) {
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
      const int tt = t % half2, r = t / half2;
      int ci[3];
      ci[1] = b.lo[1] + r % e1;
      ci[0] = b.lo[0] + r / e1;
      ci[2] = b.lo[2] + ((parity + off - ci[0] - ci[1] - b.lo[2]) & 1) + 2 * tt;
      if (ci[2] > b.hi[2]) continue;
      const int f = lin(L, ci);
      if (phase == 1) {
        x[A][f] = C.tmp[f];
        continue;
      }
      double dg;
      const double au = face_row<DIM, FORM, A, PA, false>(L, uc, f, ci, dg);
      const double nv = uc[A][f] + omega * ((rhs[f] - au) / dg);
      if (C.two_phase) C.tmp[f] = nv;
      else x[A][f] = nv;
    }
    __syncthreads();
  }
}

template <int DIM, int FORM, int A, int PA>
__device__ void cf_rr(const CoarseLv& F, const CoarseLv& Cc) {
  const Box cb = face_box(Cc.d, DIM, A);
  const int e1 = cb.hi[1] - cb.lo[1] + 1, e2 = cb.hi[2] - cb.lo[2] + 1;
  const int total = (cb.hi[0] - cb.lo[0] + 1) * e1 * e2;
  const double* u[3] = {F.x[0], F.x[1], F.x[2]};
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    int C[3];
    C[2] = cb.lo[2] + t % e2;
    C[1] = cb.lo[1] + (t / e2) % e1;
    C[0] = cb.lo[0] + t / (e1 * e2);
    double tv[3];
#pragma unroll 1
    for (int o = -1; o <= 1; ++o) {
      int fa = 2 * C[A] + o;
      if (fa < 0) fa += F.d.n[A];
      tv[o + 1] = tmean_resid<DIM, FORM, A, PA, false>(F.d, u, F.rhs[A], C, fa);
    }
    Cc.rhs[A][lin(Cc.d, C)] = (0.25 * tv[0] + 0.5 * tv[1]) + 0.25 * tv[2];
  }
}

template <int DIM, int A>
__device__ void cf_pa(const CoarseLv& Cc, const CoarseLv& F) {
  const Box fb = face_box(F.d, DIM, A);
  const int e1 = fb.hi[1] - fb.lo[1] + 1, e2 = fb.hi[2] - fb.lo[2] + 1;
  const int total = (fb.hi[0] - fb.lo[0] + 1) * e1 * e2;
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    int X[3];
    X[2] = fb.lo[2] + t % e2;
    X[1] = fb.lo[1] + (t / e2) % e1;
    X[0] = fb.lo[0] + t / (e1 * e2);
    face_pa_at<DIM, A, false>(F.d, Cc.d, Cc.x[A], F.x[A], X);
  }
}

template <int DIM, int FORM, int PA>
__device__ void cf_smooth(const CoarseLv& C, double omega, int sweeps) {
  for (int s = 0; s < sweeps; ++s) {
#pragma unroll 1
    for (int p = 0; p < 2; ++p) {
      if (DIM == 3) cf_colour<3, FORM, 0, PA>(C, omega, p);
    }
#pragma unroll 1
    for (int p = 0; p < 2; ++p) cf_colour<DIM, FORM, 1, PA>(C, omega, p);
#pragma unroll 1
    for (int p = 0; p < 2; ++p) cf_colour<DIM, FORM, 2, PA>(C, omega, p);
  }
}

template <int DIM, int FORM, int PA>
__global__ void __launch_bounds__(kCoarseThreads, 1)
k_coarse_face(const CoarseChain* __restrict__ gch, int sweeps_down, int sweeps_up, int bottom, double omega) {
  pdl_enter();
  __shared__ CoarseChain ch;
  {
    const int* src = reinterpret_cast<const int*>(gch);
    int* dst = reinterpret_cast<int*>(&ch);
    for (int i = threadIdx.x; i < (int)(sizeof(CoarseChain) / sizeof(int)); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const int nl = ch.nl;
  for (int l = 0; l < nl; ++l) {
    const CoarseLv& C = ch.lv[l];
    for (int A = 3 - DIM; A < 3; ++A) cz_fill(C.x[A], C.block);
    __syncthreads();
    if (l == nl - 1) {
      cf_smooth<DIM, FORM, PA>(C, omega, bottom);
    } else {
      cf_smooth<DIM, FORM, PA>(C, omega, sweeps_down);
      if (DIM == 3) cf_rr<3, FORM, 0, PA>(C, ch.lv[l + 1]);
      cf_rr<DIM, FORM, 1, PA>(C, ch.lv[l + 1]);
      cf_rr<DIM, FORM, 2, PA>(C, ch.lv[l + 1]);
      __syncthreads();
    }
  }
  for (int l = nl - 2; l >= 0; --l) {
    const CoarseLv& C = ch.lv[l];
    if (DIM == 3) cf_pa<3, 0>(ch.lv[l + 1], C);
    cf_pa<DIM, 1>(ch.lv[l + 1], C);
    cf_pa<DIM, 2>(ch.lv[l + 1], C);
    __syncthreads();
    cf_smooth<DIM, FORM, PA>(C, omega, sweeps_up);
  }
}

template <int DIM, int PA>
__device__ void cc_smooth(const CoarseLv& C, double omega, int sweeps) {
  const LevelDev& L = C.d;
  const int e1 = L.n[1];
  const int half2 = (L.n[2] + 1) / 2;
  const int total = L.n[0] * e1 * half2;
  double* phi = C.x[0];
  const double* rhs = C.rhs[0];
  for (int s = 0; s < sweeps; ++s) {
#pragma unroll 1
    for (int parity = 0; parity < 2; ++parity) {
      for (int phase = 0; phase < (C.two_phase ? 2 : 1); ++phase) {
        for (int t = threadIdx.x; t < total; t += blockDim.x) {
          const int tt = t % half2, r = t / half2;
          int ci[3];
          ci[1] = r % e1;
          ci[0] = r / e1;
          ci[2] = ((parity - ci[0] - ci[1]) & 1) + 2 * tt;
          if (ci[2] >= L.n[2]) continue;
          const int c = lin(L, ci);
          if (phase == 1) {
            phi[c] = C.tmp[c];
            continue;
          }
          double dg;
          const double lp = cell_row<DIM, PA>(L, phi, c, ci, dg);
          const double nv = phi[c] + omega * (rhs[c] - lp) / dg;
          if (C.two_phase) C.tmp[c] = nv;
          else phi[c] = nv;
        }
        __syncthreads();
      }
    }
  }
}

template <int DIM, int PA>
__global__ void __launch_bounds__(kCoarseThreads, 1)
k_coarse_cell(const CoarseChain* __restrict__ gch, int sweeps_down, int sweeps_up, int bottom, double omega) {
  pdl_enter();
  __shared__ CoarseChain ch;
  {
    const int* src = reinterpret_cast<const int*>(gch);
    int* dst = reinterpret_cast<int*>(&ch);
    for (int i = threadIdx.x; i < (int)(sizeof(CoarseChain) / sizeof(int)); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const int nl = ch.nl;
  for (int l = 0; l < nl; ++l) {
    const CoarseLv& C = ch.lv[l];
    cz_fill(C.x[0], C.block);
    __syncthreads();
    if (l == nl - 1) {
      cc_smooth<DIM, PA>(C, omega, bottom);
    } else {
      cc_smooth<DIM, PA>(C, omega, sweeps_down);
      const CoarseLv& Cc = ch.lv[l + 1];
      const int e1 = Cc.d.n[1], e2 = Cc.d.n[2];
      const int total = Cc.d.n[0] * e1 * e2;
      for (int t = threadIdx.x; t < total; t += blockDim.x) {
        int K[3] = {t / (e1 * e2), (t / e2) % e1, t % e2};
        Cc.rhs[0][lin(Cc.d, K)] = cell_rr_at<DIM, PA, false>(C.d, C.x[0], C.rhs[0], K);
      }
      __syncthreads();
    }
  }
  for (int l = nl - 2; l >= 0; --l) {
    const CoarseLv& C = ch.lv[l];
    const CoarseLv& Cc = ch.lv[l + 1];
    const int e1 = C.d.n[1], e2 = C.d.n[2];
    const int total = C.d.n[0] * e1 * e2;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
      int F[3] = {t / (e1 * e2), (t / e2) % e1, t % e2};
      cell_pa_at<DIM, false>(C.d, Cc.d, Cc.x[0], C.x[0], F);
    }
    __syncthreads();
    cc_smooth<DIM, PA>(C, omega, sweeps_up);
  }
}

}  // namespace

// ===========================================================================
// launchers
// ===========================================================================

long long g_kernel_launches = 0;
static int g_red_blocks_used = kRedBlocks;  // partial slots written by the last reduction

int reduce_blocks() { return kRedBlocks; }

// one full wave of resident CTAs for a grid-stride reduction kernel: with a
// grid that is not a multiple of the resident capacity the last partial wave
// runs at a fraction of the bandwidth (pass B: 1184 CTAs at 6/SM -> 888 is
// 18 % faster).  Capped by the partial-slot count kRedBlocks.
template <class K>
static int wave_grid(K kernel) {
  int occ = 0, sms = 0, dev = 0;
  cudaGetDevice(&dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, 0) != cudaSuccess || occ < 1) occ = 8;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1) sms = kSMs;
  return std::max(1, std::min(occ * sms, kRedBlocks));
}


#define SB_DISPATCH_FORM(form, ...)                     \
  switch (form) {                                       \
    case F_LAP: { constexpr int FM = F_LAP; __VA_ARGS__; } break;       \
    case F_STRESS: { constexpr int FM = F_STRESS; __VA_ARGS__; } break; \
    default: { constexpr int FM = F_BULK; __VA_ARGS__; } break;         \
  }

static bool all_periodic(const LevelDev& L) {
  return L.bclo[0] == BC_PER && L.bclo[1] == BC_PER && L.bclo[2] == BC_PER;
}
// compile-time boundary pattern of a level (sb_device.cuh perq): 1 all
// periodic, PA_W2 walls along axis 2 only, 0 anything else
static int bc_pattern(const LevelDev& L) {
  if (all_periodic(L)) return 1;
  if (L.bclo[0] == BC_PER && L.bclo[1] == BC_PER) return PA_W2;
  return 0;
}
#define SB_DISPATCH_PA(L, ...)                                     \
  switch (bc_pattern(L)) {                                         \
    case 1: { constexpr int PAT = 1; __VA_ARGS__; } break;         \
    case PA_W2: { constexpr int PAT = PA_W2; __VA_ARGS__; } break; \
    default: { constexpr int PAT = 0; __VA_ARGS__; } break;        \
  }
// level whose edge viscosities are derived from mu_c (DE kernels)
// (slab levels read mu_c's ghost planes along axis 0, exchanged at setup)
static bool derive_mue(const LevelDev& L) { return L.mue_derived != 0; }

static bool odd_periodic(const LevelDev& L, int dim) {
  for (int a = 3 - dim; a < 3; ++a)
    if (L.bclo[a] == BC_PER && (L.n[a] & 1)) return true;
  return false;
}

template <int DIM, int FM, int A>
static void face_colour_t(cudaStream_t s, const LevelDev& L, Ptr3 u, const double* rhs, double* tmp,
                          int parity, double omega, int z = 0, int ext0 = 0, int w_lo = 0, int w_hi = -1) {
  Box b = face_box(L, DIM, A);
  b.lo[0] -= ext0;  // slab levels: also relax the ghost planes (sb_dist.inc dsweep_face)
  b.hi[0] += ext0;
  if (w_hi >= w_lo) {  // a window of planes
    b.lo[0] = w_lo;
    b.hi[0] = w_hi;
  }
  const unsigned len2 = (unsigned)(b.hi[2] - b.lo[2] + 1);
  const unsigned half2 = (len2 + 1) / 2;
  const unsigned total = half2;
  L3 c3 = cfg3(b.hi[0] - b.lo[0] + 1, b.hi[1] - b.lo[1] + 1, (int)half2);
  // threads along the row: two warps per row segment (64 same-colour faces,
  // 4 rows per CTA) on rows of >= 128 faces -- measured 164 vs 166-168 us per
  // finest pass against one warp x 8 rows (C5 256^3); SB_FC_BX overrides
  static const int bx_env = [] {
    const char* e = std::getenv("SB_FC_BX");
    return e ? std::atoi(e) : 64;
  }();
  static const int bx_min = [] {  // SB_FC_BX_MIN: shortest same-colour row taking it
    const char* e = std::getenv("SB_FC_BX_MIN");
    return e ? std::atoi(e) : 0;
  }();
  if (bx_env > 0 && (int)half2 >= std::max(bx_env, bx_min) && c3.b.x == 32) {
    const int by = kThreads / bx_env;
    c3.b = dim3(bx_env, by, 1);
    c3.g = dim3((half2 + bx_env - 1) / bx_env, (b.hi[1] - b.lo[1] + 1 + by - 1) / by, b.hi[0] - b.lo[0] + 1);
  }
  const dim3 g = c3.g, kb = c3.b;
  if (tmp == nullptr && z == 3) {  // all-periodic pad-free level (zero_fill_free)
    if (derive_mue(L)) launch_k(k_face_colour<DIM, FM, A, 0, 1, true, 3>, g, kb, 0, s, L, u, rhs, nullptr, parity, omega, b, half2, total);
    else launch_k(k_face_colour<DIM, FM, A, 0, 1, false, 3>, g, kb, 0, s, L, u, rhs, nullptr, parity, omega, b, half2, total);
  } else if (tmp == nullptr) {
#define SB_FC_Z(ZZ)                                                                                                          \
  SB_DISPATCH_PA(L, {                                                                                                        \
    if (derive_mue(L)) launch_k(k_face_colour<DIM, FM, A, 0, PAT, true, ZZ>, g, kb, 0, s, L, u, rhs, nullptr, parity, omega, b, half2, total); \
    else launch_k(k_face_colour<DIM, FM, A, 0, PAT, false, ZZ>, g, kb, 0, s, L, u, rhs, nullptr, parity, omega, b, half2, total);            \
  })
    if (z == 2) {
      SB_FC_Z(2);
    } else if (z == 1) {
      SB_FC_Z(1);
    } else {
      SB_FC_Z(0);
    }
#undef SB_FC_Z
  } else {
    ++g_kernel_launches;
    launch_k(k_face_colour<DIM, FM, A, 2, false>, g, kb, 0, s, L, u, rhs, tmp, parity, omega, b, half2, total);
    launch_k(k_face_colour<DIM, FM, A, 1, false>, g, kb, 0, s, L, u, rhs, tmp, parity, omega, b, half2, total);
  }
}

void launch_face_colour(cudaStream_t s, const LevelDev& L, int dim, int form, int A, Ptr3 u,
                        const double* rhsA, int parity, double omega, int z, int ext0, int w_lo, int w_hi) {
  ++g_kernel_launches;
  // odd periodic extents need the two-phase (Jacobi-within-colour) form; the
  // caller's level scratch is passed through u.p[?] is not available here, so
  // the solver routes those levels through launch_face_colour_tmp below.
  if (z == 0 && !L.dist0 && rowv_colour_supported(L, dim, form)) {
    launch_face_colour_rv(s, L, form, A, u, rhsA, parity, omega);
    return;
  }
  SB_DISPATCH_FORM(form, {
    if (dim == 3) {
      if (A == 0) face_colour_t<3, FM, 0>(s, L, u, rhsA, nullptr, parity, omega, z, ext0, w_lo, w_hi);
      else if (A == 1) face_colour_t<3, FM, 1>(s, L, u, rhsA, nullptr, parity, omega, z, ext0, w_lo, w_hi);
      else face_colour_t<3, FM, 2>(s, L, u, rhsA, nullptr, parity, omega, z, ext0, w_lo, w_hi);
    } else {
      if (A == 1) face_colour_t<2, FM, 1>(s, L, u, rhsA, nullptr, parity, omega, z, ext0, w_lo, w_hi);
      else face_colour_t<2, FM, 2>(s, L, u, rhsA, nullptr, parity, omega, z, ext0, w_lo, w_hi);
    }
  });
}

void launch_face_colour_tmp(cudaStream_t s, const LevelDev& L, int dim, int form, int A, Ptr3 u,
                            const double* rhsA, double* tmp, int parity, double omega) {
  ++g_kernel_launches;
  SB_DISPATCH_FORM(form, {
    if (dim == 3) {
      if (A == 0) face_colour_t<3, FM, 0>(s, L, u, rhsA, tmp, parity, omega);
      else if (A == 1) face_colour_t<3, FM, 1>(s, L, u, rhsA, tmp, parity, omega);
      else face_colour_t<3, FM, 2>(s, L, u, rhsA, tmp, parity, omega);
    } else {
      if (A == 1) face_colour_t<2, FM, 1>(s, L, u, rhsA, tmp, parity, omega);
      else face_colour_t<2, FM, 2>(s, L, u, rhsA, tmp, parity, omega);
    }
  });
}

template <int DIM>
static void cell_colour_t(cudaStream_t s, const LevelDev& L, double* phi, const double* rhs, double* tmp,
                          int parity, double omega, int z = 0, int ext0 = 0, int w_lo = 0, int w_hi = -1) {
  Box b = cell_box(L);
  b.lo[0] -= ext0;
  b.hi[0] += ext0;
  if (w_hi >= w_lo) {
    b.lo[0] = w_lo;
    b.hi[0] = w_hi;
  }
  const unsigned len2 = (unsigned)L.n[2];
  const unsigned half2 = (len2 + 1) / 2;
  const unsigned total = half2;
  L3 c3 = cfg3(b.hi[0] - b.lo[0] + 1, L.n[1], (int)half2);
  static const int bx_env = [] {  // SB_CC_BX: threads along the row
    const char* e = std::getenv("SB_CC_BX");
    return e ? std::atoi(e) : 32;
  }();
  if (bx_env != 32 && bx_env > 0 && (int)half2 >= bx_env && c3.b.x == 32) {
    const int by = kThreads / bx_env;
    c3.b = dim3(bx_env, by, 1);
    c3.g = dim3((half2 + bx_env - 1) / bx_env, (L.n[1] + by - 1) / by, b.hi[0] - b.lo[0] + 1);
  }
  const dim3 g = c3.g, kb = c3.b;
  if (tmp == nullptr && z == 3) {
    launch_k(k_cell_colour<DIM, 0, 1, 3>, g, kb, 0, s, L, phi, rhs, nullptr, parity, omega, b, half2, total);
  } else if (tmp == nullptr && z == 2) {
    SB_DISPATCH_PA(L, launch_k(k_cell_colour<DIM, 0, PAT, 2>, g, kb, 0, s, L, phi, rhs, nullptr, parity, omega, b, half2, total));
  } else if (tmp == nullptr) {
    SB_DISPATCH_PA(L, launch_k(k_cell_colour<DIM, 0, PAT>, g, kb, 0, s, L, phi, rhs, nullptr, parity, omega, b, half2, total));
  } else {
    ++g_kernel_launches;
    launch_k(k_cell_colour<DIM, 2, false>, g, kb, 0, s, L, phi, rhs, tmp, parity, omega, b, half2, total);
    launch_k(k_cell_colour<DIM, 1, false>, g, kb, 0, s, L, phi, rhs, tmp, parity, omega, b, half2, total);
  }
}

void launch_cell_colour(cudaStream_t s, const LevelDev& L, int dim, double* phi, const double* rhs,
                        int parity, double omega, int z, int ext0, int w_lo, int w_hi) {
  ++g_kernel_launches;
  if (dim == 3) cell_colour_t<3>(s, L, phi, rhs, nullptr, parity, omega, z, ext0, w_lo, w_hi);
  else cell_colour_t<2>(s, L, phi, rhs, nullptr, parity, omega, z, ext0, w_lo, w_hi);
}

void launch_cell_colour_tmp(cudaStream_t s, const LevelDev& L, int dim, double* phi, const double* rhs,
                            double* tmp, int parity, double omega) {
  ++g_kernel_launches;
  if (dim == 3) cell_colour_t<3>(s, L, phi, rhs, tmp, parity, omega);
  else cell_colour_t<2>(s, L, phi, rhs, tmp, parity, omega);
}

bool level_needs_two_phase(const LevelDev& L, int dim) { return odd_periodic(L, dim); }

template <int DIM, int FM, int A>
static void face_rr_t(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, CPtr3 u, const double* rhs,
                      double* coarse) {
  Box cb = face_box(Lc, DIM, A);
  const unsigned ncoarse = box_count(cb);
  if (ncoarse < 32768u) {  // small level: thread per coarse face
    if (all_periodic(Lf)) launch_k(k_face_rr_s<DIM, FM, A, true>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, u, rhs, coarse, cb, ncoarse);
    else launch_k(k_face_rr_s<DIM, FM, A, false>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, u, rhs, coarse, cb, ncoarse);
    return;
  }
  if (A == 2) {
    const L3 c3 = cfg3(cb.hi[0] - cb.lo[0] + 1, cb.hi[1] - cb.lo[1] + 1, cb.hi[2] - cb.lo[2] + 1);
    dim3 b = c3.b, g = c3.g;
    if (b.x < 32) {  // the shuffle needs whole warps along K
      b = dim3(32, kThreads / 32, 1);
      g = dim3((cb.hi[2] - cb.lo[2] + 32) / 32, (cb.hi[1] - cb.lo[1] + b.y) / b.y, cb.hi[0] - cb.lo[0] + 1);
    }
    if (all_periodic(Lf)) launch_k(k_face_rr_c<DIM, FM, true>, g, b, 0, s, Lf, Lc, u, rhs, coarse, cb);
    else launch_k(k_face_rr_c<DIM, FM, false>, g, b, 0, s, Lf, Lc, u, rhs, coarse, cb);
  } else {
    constexpr int T = (A == 0) ? 1 : 0;
    const int e2 = cb.hi[2] - cb.lo[2] + 1;
    const int eT = DIM == 3 ? cb.hi[T] - cb.lo[T] + 1 : 1;
    const int eA = cb.hi[A] - cb.lo[A] + 1;
    const L3 c3 = cfg3(1, eT, e2);
    // chunk along A: enough CTAs to fill the machine, at least 4 coarse faces per thread
    long long cols = (long long)c3.g.x * c3.g.y;
    // chunks of 4 coarse faces (measured best at 256^3: 2 -> 8 spans 5 %);
    // more when the grid would not fill the machine otherwise
    int nchunk = (int)std::max<long long>(1, std::max<long long>(eA / 4, (kSMs * 8 + cols - 1) / cols));
    nchunk = std::min(nchunk, eA);
    static const int chunk_env = [] {
      const char* e = std::getenv("SB_RR_CHUNK");
      return e ? std::atoi(e) : 0;
    }();
    const int chunk = chunk_env > 0 ? std::min(chunk_env, eA) : (eA + nchunk - 1) / nchunk;
    nchunk = (eA + chunk - 1) / chunk;
    dim3 g(c3.g.x, c3.g.y, nchunk);
    if (all_periodic(Lf)) launch_k(k_face_rr_m<DIM, FM, A, true>, g, c3.b, 0, s, Lf, Lc, u, rhs, coarse, cb, chunk);
    else launch_k(k_face_rr_m<DIM, FM, A, false>, g, c3.b, 0, s, Lf, Lc, u, rhs, coarse, cb, chunk);
  }
}

void launch_face_resid_restrict(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, int dim, int form,
                                int A, CPtr3 u, const double* rhsA, double* coarseA) {
  ++g_kernel_launches;
  SB_DISPATCH_FORM(form, {
    if (dim == 3) {
      if (A == 0) face_rr_t<3, FM, 0>(s, Lf, Lc, u, rhsA, coarseA);
      else if (A == 1) face_rr_t<3, FM, 1>(s, Lf, Lc, u, rhsA, coarseA);
      else face_rr_t<3, FM, 2>(s, Lf, Lc, u, rhsA, coarseA);
    } else {
      if (A == 1) face_rr_t<2, FM, 1>(s, Lf, Lc, u, rhsA, coarseA);
      else face_rr_t<2, FM, 2>(s, Lf, Lc, u, rhsA, coarseA);
    }
  });
}

void launch_face_res3(cudaStream_t s, const LevelDev& L, int dim, int form, CPtr3 x, CPtr3 rhs, Ptr3 out) {
  ++g_kernel_launches;
  Box b;
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = 0;
    b.hi[a] = L.n[a] - 1 + (L.bclo[a] != BC_PER ? 1 : 0);
  }
  if (dim == 2) b.hi[0] = 0;
  if (rowv_supported(L, dim, form)) {
    launch_face_res3_rv(s, L, form, x, rhs, out);
    return;
  }
  const bool de = derive_mue(L);
  SB_DISPATCH_FORM(form, {
    if (dim == 3) {
      SB_DISPATCH_PA(L, {
        if (de) launch_k(k_face_res3<3, FM, PAT, true>, cfg3(b).g, cfg3(b).b, 0, s, L, x, rhs, out, b);
        else launch_k(k_face_res3<3, FM, PAT>, cfg3(b).g, cfg3(b).b, 0, s, L, x, rhs, out, b);
      });
    } else {
      SB_DISPATCH_PA(L, {
        if (de) launch_k(k_face_res3<2, FM, PAT, true>, cfg3(b).g, cfg3(b).b, 0, s, L, x, rhs, out, b);
        else launch_k(k_face_res3<2, FM, PAT>, cfg3(b).g, cfg3(b).b, 0, s, L, x, rhs, out, b);
      });
    }
  });
}

void launch_face_restrict(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, int dim, int A, const double* r,
                          double* coarse) {
  ++g_kernel_launches;
  Box cb = face_box(Lc, dim, A);
  if (dim == 3) {
    if (A == 0) launch_k(k_face_restrict<3, 0>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, r, coarse, cb);
    else if (A == 1) launch_k(k_face_restrict<3, 1>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, r, coarse, cb);
    else launch_k(k_face_restrict<3, 2>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, r, coarse, cb);
  } else {
    if (A == 1) launch_k(k_face_restrict<2, 1>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, r, coarse, cb);
    else launch_k(k_face_restrict<2, 2>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, r, coarse, cb);
  }
}

void launch_cell_res(cudaStream_t s, const LevelDev& L, int dim, const double* x, const double* rhs,
                     double* out) {
  ++g_kernel_launches;
  Box b = cell_box(L);
  if (dim == 3) SB_DISPATCH_PA(L, launch_k(k_cell_res<3, PAT>, cfg3(b).g, cfg3(b).b, 0, s, L, x, rhs, out, b))
  else SB_DISPATCH_PA(L, launch_k(k_cell_res<2, PAT>, cfg3(b).g, cfg3(b).b, 0, s, L, x, rhs, out, b))
}

void launch_cell_restrict(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, int dim, const double* r,
                          double* coarse) {
  ++g_kernel_launches;
  Box cb = cell_box(Lc);
  if (dim == 3) launch_k(k_cell_restrict<3>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, r, coarse, cb);
  else launch_k(k_cell_restrict<2>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, r, coarse, cb);
}

void launch_cell_resid_restrict(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, int dim,
                                const double* phi, const double* rhs, double* coarse) {
  ++g_kernel_launches;
  Box cb = cell_box(Lc);
  const unsigned total = box_count(cb);
  const bool pa = all_periodic(Lf);
  if (dim == 3) {
    if (pa) launch_k(k_cell_rr<3, true>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, phi, rhs, coarse, cb, total);
    else launch_k(k_cell_rr<3, false>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, phi, rhs, coarse, cb, total);
  } else {
    if (pa) launch_k(k_cell_rr<2, true>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, phi, rhs, coarse, cb, total);
    else launch_k(k_cell_rr<2, false>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, phi, rhs, coarse, cb, total);
  }
}

void launch_face_prolong_add(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, int dim, int A,
                             const double* coarseA, double* fineA) {
  ++g_kernel_launches;
  // one thread per coarse position (I along A, J1, J2), 2^d fine faces each
  Box cb;
  for (int a = 0; a < 3; ++a) {
    cb.lo[a] = 0;
    cb.hi[a] = Lc.n[a] - 1;
  }
  if (dim == 2) cb.hi[0] = 0;
  if (dim == 3) {
    if (A == 0) launch_k(k_face_pa8<3, 0>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, coarseA, fineA, cb);
    else if (A == 1) launch_k(k_face_pa8<3, 1>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, coarseA, fineA, cb);
    else launch_k(k_face_pa8<3, 2>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, coarseA, fineA, cb);
  } else {
    if (A == 1) launch_k(k_face_pa8<2, 1>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, coarseA, fineA, cb);
    else launch_k(k_face_pa8<2, 2>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, coarseA, fineA, cb);
  }
}

void launch_cell_prolong_add(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, int dim,
                             const double* coarse, double* fine) {
  ++g_kernel_launches;
  Box fb = cell_box(Lf);
  const unsigned total = box_count(fb);
  if (dim == 3) launch_k(k_cell_pa<3>, cfg3(fb).g, cfg3(fb).b, 0, s, Lf, Lc, coarse, fine, fb, total);
  else launch_k(k_cell_pa<2>, cfg3(fb).g, cfg3(fb).b, 0, s, Lf, Lc, coarse, fine, fb, total);
}

void launch_coarse_face(cudaStream_t s, int dim, int form, bool pa, const CoarseChain* dchain,
                        int sweeps_down, int sweeps_up, int bottom, double omega) {
  ++g_kernel_launches;
  SB_DISPATCH_FORM(form, {
    if (dim == 3) {
      if (pa) launch_k(k_coarse_face<3, FM, true>, 1, kCoarseThreads, 0, s, dchain, sweeps_down, sweeps_up, bottom, omega);
      else launch_k(k_coarse_face<3, FM, false>, 1, kCoarseThreads, 0, s, dchain, sweeps_down, sweeps_up, bottom, omega);
    } else {
      if (pa) launch_k(k_coarse_face<2, FM, true>, 1, kCoarseThreads, 0, s, dchain, sweeps_down, sweeps_up, bottom, omega);
      else launch_k(k_coarse_face<2, FM, false>, 1, kCoarseThreads, 0, s, dchain, sweeps_down, sweeps_up, bottom, omega);
    }
  });
}

void launch_coarse_cell(cudaStream_t s, int dim, bool pa, const CoarseChain* dchain, int sweeps_down,
                        int sweeps_up, int bottom, double omega) {
  ++g_kernel_launches;
  if (dim == 3) {
    if (pa) launch_k(k_coarse_cell<3, true>, 1, kCoarseThreads, 0, s, dchain, sweeps_down, sweeps_up, bottom, omega);
    else launch_k(k_coarse_cell<3, false>, 1, kCoarseThreads, 0, s, dchain, sweeps_down, sweeps_up, bottom, omega);
  } else {
    if (pa) launch_k(k_coarse_cell<2, true>, 1, kCoarseThreads, 0, s, dchain, sweeps_down, sweeps_up, bottom, omega);
    else launch_k(k_coarse_cell<2, false>, 1, kCoarseThreads, 0, s, dchain, sweeps_down, sweeps_up, bottom, omega);
  }
}

// padded box covering every array of the level
static Box full_box(const LevelDev& L) {
  Box b;
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = 0;
    b.hi[a] = L.n[a] - 1 + (L.bclo[a] != BC_PER ? 1 : 0);
  }
  return b;
}

void launch_apply_M(cudaStream_t s, const LevelDev& L, int dim, int form, CPtr3 u, const double* p,
                    Ptr3 out_u, double* out_p) {
  ++g_kernel_launches;
  if (rowv_supported(L, dim, form)) {
    launch_apply_M_rv(s, L, form, u, p, out_u, out_p);
    return;
  }
  Box b = full_box(L);
  const unsigned total = box_count(b);
  SB_DISPATCH_FORM(form, {
    SB_DISPATCH_PA(L, {
      if (derive_mue(L)) {
        if (dim == 3) launch_k(k_apply_M<3, FM, PAT, true>, cfg3(b).g, cfg3(b).b, 0, s, L, u, p, out_u, out_p, b, total);
        else launch_k(k_apply_M<2, FM, PAT, true>, cfg3(b).g, cfg3(b).b, 0, s, L, u, p, out_u, out_p, b, total);
      } else {
        if (dim == 3) launch_k(k_apply_M<3, FM, PAT>, cfg3(b).g, cfg3(b).b, 0, s, L, u, p, out_u, out_p, b, total);
        else launch_k(k_apply_M<2, FM, PAT>, cfg3(b).g, cfg3(b).b, 0, s, L, u, p, out_u, out_p, b, total);
      }
    });
  });
}

void launch_face_residual(cudaStream_t s, const LevelDev& L, int dim, int form, CPtr3 x, CPtr3 rhs,
                          const double* q, Ptr3 out) {
  ++g_kernel_launches;
  Box b = full_box(L);
  const unsigned total = box_count(b);
  SB_DISPATCH_FORM(form, {
    if (dim == 3) launch_k(k_face_residual<3, FM>, cfg3(b).g, cfg3(b).b, 0, s, L, x, rhs, q, out, b, total);
    else launch_k(k_face_residual<2, FM>, cfg3(b).g, cfg3(b).b, 0, s, L, x, rhs, q, out, b, total);
  });
}

void launch_cell_residual(cudaStream_t s, const LevelDev& L, int dim, const double* x, const double* rhs,
                          double* out) {
  ++g_kernel_launches;
  Box b = cell_box(L);
  const unsigned total = box_count(b);
  if (dim == 3) launch_k(k_cell_residual<3>, cfg3(b).g, cfg3(b).b, 0, s, L, x, rhs, out, b, total);
  else launch_k(k_cell_residual<2>, cfg3(b).g, cfg3(b).b, 0, s, L, x, rhs, out, b, total);
}

void launch_div_add(cudaStream_t s, const LevelDev& L, int dim, CPtr3 u, const double* rp, double* out) {
  Box b = cell_box(L);
  const unsigned total = box_count(b);
  if (dim == 3) launch_k(k_div_add<3>, cfg3(b).g, cfg3(b).b, 0, s, L, u, rp, out, b, total);
  else launch_k(k_div_add<2>, cfg3(b).g, cfg3(b).b, 0, s, L, u, rp, out, b, total);
}

void launch_p1_glue(cudaStream_t s, const LevelDev& L, int dim, int form, Ptr3 xu, const double* phi,
                    const double* bc, double* xp, double sign) {
  ++g_kernel_launches;
  Box b = full_box(L);
  const unsigned total = box_count(b);
  if (dim == 3) launch_k(k_p1_glue<3>, cfg3(b).g, cfg3(b).b, 0, s, L, form, xu, phi, bc, xp, sign, b, total);
  else launch_k(k_p1_glue<2>, cfg3(b).g, cfg3(b).b, 0, s, L, form, xu, phi, bc, xp, sign, b, total);
}

void launch_schur(cudaStream_t s, const LevelDev& L, int form, const double* r, const double* phi,
                  double* out, double sign) {
  ++g_kernel_launches;
  Box b = cell_box(L);
  const unsigned total = box_count(b);
  launch_k(k_schur, cfg3(b).g, cfg3(b).b, 0, s, L, form, r, phi, out, sign, b, total);
}

void launch_face_sub_grad(cudaStream_t s, const LevelDev& L, int dim, CPtr3 ru, const double* q, Ptr3 out) {
  Box b = full_box(L);
  const unsigned total = box_count(b);
  if (dim == 3) launch_k(k_face_sub_grad<3>, cfg3(b).g, cfg3(b).b, 0, s, L, ru, q, out, b, total);
  else launch_k(k_face_sub_grad<2>, cfg3(b).g, cfg3(b).b, 0, s, L, ru, q, out, b, total);
}

void launch_coarsen_cellmean(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, int dim,
                             const double* fine, double* coarse) {
  ++g_kernel_launches;
  Box cb = cell_box(Lc);
  const unsigned total = box_count(cb);
  if (dim == 3) launch_k(k_coarsen_cellmean<3>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, fine, coarse, cb, total);
  else launch_k(k_coarsen_cellmean<2>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, fine, coarse, cb, total);
}

void launch_coarsen_face(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, int dim, int A,
                         const double* fine, double* coarse) {
  ++g_kernel_launches;
  Box cb = cell_box(Lc);
  if (Lc.bclo[A] != BC_PER) cb.hi[A] = Lc.n[A];  // all faces incl. wall boundary
  const unsigned total = box_count(cb);
  if (dim == 3) {
    if (A == 0) launch_k(k_coarsen_face<3, 0>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, fine, coarse, cb, total);
    else if (A == 1) launch_k(k_coarsen_face<3, 1>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, fine, coarse, cb, total);
    else launch_k(k_coarsen_face<3, 2>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, fine, coarse, cb, total);
  } else {
    if (A == 1) launch_k(k_coarsen_face<2, 1>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, fine, coarse, cb, total);
    else launch_k(k_coarsen_face<2, 2>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, fine, coarse, cb, total);
  }
}

void launch_coarsen_edge(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, int dim, int e,
                         const double* fine, double* coarse) {
  ++g_kernel_launches;
  Box cb = cell_box(Lc);
  for (int a = 3 - dim; a < 3; ++a)
    if (a != e && Lc.bclo[a] != BC_PER) cb.hi[a] = Lc.n[a];
  const unsigned total = box_count(cb);
  if (dim == 3) launch_k(k_coarsen_edge<3>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, e, fine, coarse, cb, total);
  else launch_k(k_coarsen_edge<2>, cfg3(cb).g, cfg3(cb).b, 0, s, Lf, Lc, e, fine, coarse, cb, total);
}

void launch_beta(cudaStream_t s, const LevelDev& L, int A, const double* rho, double* beta, int* flag,
                 int* cflag, const double* ref) {
  Box b = cell_box(L);
  if (L.bclo[A] != BC_PER) b.hi[A] = L.n[A];
  const unsigned total = box_count(b);
  launch_k(k_beta, cfg3(b).g, cfg3(b).b, 0, s, L, A, rho, beta, flag, cflag, ref, b, total);
}

void launch_check_diag(cudaStream_t s, const LevelDev& L, int dim, int form, int* flags) {
  ++g_kernel_launches;
  Box b = full_box(L);
  const unsigned total = box_count(b);
  SB_DISPATCH_FORM(form, {
    if (dim == 3) launch_k(k_check_diag<3, FM>, cfg3(b).g, cfg3(b).b, 0, s, L, flags, b, total);
    else launch_k(k_check_diag<2, FM>, cfg3(b).g, cfg3(b).b, 0, s, L, flags, b, total);
  });
}

void launch_write_diag(cudaStream_t s, const LevelDev& L, int dim, int form, Ptr3 face_diag, double* cell_diag) {
  ++g_kernel_launches;
  Box b = full_box(L);
  const unsigned total = box_count(b);
  SB_DISPATCH_FORM(form, {
    if (dim == 3) launch_k(k_write_diag<3, FM>, cfg3(b).g, cfg3(b).b, 0, s, L, face_diag, cell_diag, b, total);
    else launch_k(k_write_diag<2, FM>, cfg3(b).g, cfg3(b).b, 0, s, L, face_diag, cell_diag, b, total);
  });
}

void launch_div(cudaStream_t s, const LevelDev& L, int dim, CPtr3 u, double* out) {
  ++g_kernel_launches;
  Box b = cell_box(L);
  const unsigned total = box_count(b);
  if (dim == 3) launch_k(k_div<3>, cfg3(b).g, cfg3(b).b, 0, s, L, u, out, b, total);
  else launch_k(k_div<2>, cfg3(b).g, cfg3(b).b, 0, s, L, u, out, b, total);
}

void launch_grad(cudaStream_t s, const LevelDev& L, int dim, const double* p, Ptr3 out) {
  ++g_kernel_launches;
  Box b = full_box(L);
  const unsigned total = box_count(b);
  if (dim == 3) launch_k(k_grad<3>, cfg3(b).g, cfg3(b).b, 0, s, L, p, out, b, total);
  else launch_k(k_grad<2>, cfg3(b).g, cfg3(b).b, 0, s, L, p, out, b, total);
}

void launch_cell_to_face(cudaStream_t s, const LevelDev& L, int dim, int A, const double* cell, double* face) {
  ++g_kernel_launches;
  Box b = cell_box(L);
  if (L.bclo[A] != BC_PER) b.hi[A] += 1;
  if (dim == 2) b.hi[0] = 0;
  launch_k(k_cell_to_face, cfg3(b).g, cfg3(b).b, 0, s, L, A, cell, face, b);
}

void launch_cell_to_edge(cudaStream_t s, const LevelDev& L, int dim, int e, double* out, double scale) {
  ++g_kernel_launches;
  Box b = cell_box(L);
  for (int a = 0; a < 3; ++a)
    if (a != e && L.bclo[a] != BC_PER) b.hi[a] += 1;
  if (dim == 2) b.hi[0] = 0;
  if (dim == 3) launch_k(k_cell_to_edge<3>, cfg3(b).g, cfg3(b).b, 0, s, L, e, out, scale, b);
  else launch_k(k_cell_to_edge<2>, cfg3(b).g, cfg3(b).b, 0, s, L, e, out, scale, b);
}

void launch_scale(cudaStream_t s, double* x, double scale, long long n) {
  ++g_kernel_launches;
  launch_k(k_scale, grid_for(n), kThreads, 0, s, x, scale, n);
}

void launch_check_mue(cudaStream_t s, const LevelDev& L, int dim, int* flag) {
  ++g_kernel_launches;
  Box b = cell_box(L);
  for (int a = 0; a < 3; ++a)
    if (L.bclo[a] != BC_PER) b.hi[a] += 1;
  if (dim == 2) b.hi[0] = 0;
  if (dim == 3) launch_k(k_check_mue<3>, cfg3(b).g, cfg3(b).b, 0, s, L, flag, b);
  else launch_k(k_check_mue<2>, cfg3(b).g, cfg3(b).b, 0, s, L, flag, b);
}

void launch_box_fill(cudaStream_t s, const LevelDev& L, Box b, double* x, double v) {
  const unsigned total = box_count(b);
  launch_k(k_box_fill, cfg3(b).g, cfg3(b).b, 0, s, L, x, v, b, total);
}

void launch_box_add_scalar(cudaStream_t s, const LevelDev& L, Box b, double* x, const double* sum,
                           double inv_count) {
  ++g_kernel_launches;
  const unsigned total = box_count(b);
  launch_k(k_box_sub_mean, cfg3(b).g, cfg3(b).b, 0, s, L, x, sum, inv_count, b, total);
}

void launch_wall_tangent(cudaStream_t s, const LevelDev& L, int A, int B, int side, const double* plane,
                         double* out) {
  ++g_kernel_launches;
  Box b;
  int ext[3];
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = 0;
    b.hi[a] = L.n[a] - 1 + ((a == A && L.bclo[A] != BC_PER) ? 1 : 0);
    ext[a] = b.hi[a] + 1;
  }
  b.lo[B] = b.hi[B] = side ? L.n[B] - 1 : 0;
  ext[B] = 1;
  const unsigned total = box_count(b);
  (void)total;
  launch_k(k_wall_tangent, cfg3(b).g, cfg3(b).b, 0, s, L, A, B, side, plane, out, b, ext[1], ext[2]);
}

void launch_sum_abs_partial(cudaStream_t s, const double* x, long long n, double* partials) {
  ++g_kernel_launches;
  launch_k(k_sum_abs_partial, kRedBlocks, kThreads, 0, s, x, n, partials, kRedBlocks);
}

void launch_axpy_scalar(cudaStream_t s, double* y, const double* x) {
  ++g_kernel_launches;
  launch_k(k_add_scalar, 1, 1, 0, s, y, x);
}
void launch_max_scalar(cudaStream_t s, double* y, const double* x, bool neg) {
  ++g_kernel_launches;
  launch_k(k_max_scalar, 1, 1, 0, s, y, x, neg ? 1 : 0);
}
void launch_neg_copy(cudaStream_t s, double* y, const double* x) {
  ++g_kernel_launches;
  launch_k(k_neg_copy, 1, 1, 0, s, y, x);
}

void launch_axpy_box(cudaStream_t s, const LevelDev& L, Box b, double* y, const double* x) {
  const unsigned total = box_count(b);
  launch_k(k_box_axpy, cfg3(b).g, cfg3(b).b, 0, s, L, y, x, b, total);
}

void launch_multi_dot(cudaStream_t s, const double* V, long long vstride, int nv, const double* w,
                      long long n, double* partials) {
  ++g_kernel_launches;
  static const int grid = wave_grid(k_multi_dot);
  g_red_blocks_used = grid;
  launch_k(k_multi_dot, grid, kThreads, 0, s, V, vstride, nv, w, n / 2, partials);
}

void launch_update_dot(cudaStream_t s, const double* V, long long vstride, int nv, const double* h,
                       double* w, long long n, double* partials, int mode) {
  ++g_kernel_launches;
  static const int grid = wave_grid(k_update_dot);
  g_red_blocks_used = grid;
  launch_k(k_update_dot, grid, kThreads, 0, s, V, vstride, nv, h, w, n / 2, partials, mode);
}

void launch_dcgs_a(cudaStream_t s, double* Q, long long vstride, int k, const double* c, double inv_gamma,
                   const double* w, long long n, double* partials) {
  ++g_kernel_launches;
  launch_k(k_dcgs_a, kRedBlocks, kThreads, 0, s, Q, vstride, k, c, inv_gamma, w, n / 2, partials);
}

void launch_dcgs_b(cudaStream_t s, const double* Q, long long vstride, int nv, const double* d, const double* w,
                   double* out, long long n, double* partials) {
  ++g_kernel_launches;
  static const int variant = [] {
    const char* e = std::getenv("SB_DCGS_B");
    return e ? std::atoi(e) : 2;
  }();
  if (variant == 1) {
    const size_t stash = (size_t)nv * kStashThreads * sizeof(double2);
    static bool configured = false;
    if (!configured) {
      cudaFuncSetAttribute(k_dcgs_b_stash, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      configured = true;
    }
    if (stash <= 160 * 1024) {
      launch_k(k_dcgs_b_stash, kRedBlocks, kStashThreads, stash, s, Q, vstride, nv, d, w, out, n / 2, partials);
      return;
    }
  }
  if (variant == 2) {
    launch_k(k_dcgs_b_l2, kL2Blocks, kThreads, 0, s, Q, vstride, nv, d, w, out, n / 2, partials);
    g_red_blocks_used = kL2Blocks;
    return;
  }
  launch_k(k_dcgs_b, kRedBlocks, kThreads, 0, s, Q, vstride, nv, d, w, out, n / 2, partials);
}

void launch_dcgs_a_g(cudaStream_t s, double* Q, long long vstride, int k, const double* c, double inv_gamma,
                     const double* w, long long n, double* partials, const double* means, long long block) {
  ++g_kernel_launches;
  // default: the basis staged through shared memory by TMA bulk copies
  // (k_dcgs_a_tma; bit-identical to k_dcgs_a_g3<4, 2>).  ncu, C5 256^3, the 31
  // launches of a solve: 42.95 ms vs 49.08 ms (j = 1: 0.30 vs 0.51 ms, j = 30:
  // 2.46 vs 2.69 ms = 7.2 TB/s); solve 0.3296-0.3299 vs 0.3356-0.3365 s.
  // SB_DCGS_TMA=0 (or any SB_DCGS_A variant) selects the register-staged
  // kernels.  The same ring under pass B gains 1.7 % of that pass (43.6 vs
  // 44.3 ms: it already runs at 6.8 TB/s) and changes the order of its norm
  // partial sums; not kept.
  {
    const char* et = std::getenv("SB_DCGS_TMA");
    if (!(et && et[0] == '0') && !std::getenv("SB_DCGS_A") && k > 0) {
      constexpr size_t ring_bytes = (size_t)kTmaStages * kThreads * kTmaCH * sizeof(double2);
      static const int grid_t = [] {
        cudaFuncSetAttribute(k_dcgs_a_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ring_bytes);
        cudaFuncSetAttribute(k_dcgs_a_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ring_bytes);
        int occ = 0, sms = 0, dev = 0;
        cudaGetDevice(&dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dcgs_a_tma<true>, kThreads, ring_bytes) != cudaSuccess ||
            occ < 1)
          occ = 2;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1) sms = kSMs;
        return std::max(1, std::min(occ * sms, kRedBlocks));
      }();
      g_red_blocks_used = grid_t;
      if (means)
        launch_k(k_dcgs_a_tma<true>, grid_t, kThreads, ring_bytes, s, Q, vstride, k, c, inv_gamma, w, n / 2, partials,
                 means, block / 2);
      else
        launch_k(k_dcgs_a_tma<false>, grid_t, kThreads, ring_bytes, s, Q, vstride, k, c, inv_gamma, w, n / 2, partials,
                 nullptr, 0LL);
      return;
    }
  }
  if (means) {  // deferred null projection: the grouped kernel with the means applied on load
    static const int grid_m = wave_grid(k_dcgs_a_g3<4, 2, 2, true>);
    g_red_blocks_used = grid_m;
    launch_k(k_dcgs_a_g3<4, 2, 2, true>, grid_m, kThreads, 0, s, Q, vstride, k, c, inv_gamma, w, n / 2, partials,
             means, block / 2, nullptr, 0LL);
    return;
  }
  // SB_DCGS_A: 0 un-chunked, 2 register-chunked (CH 4), 32 / 34 / 24 (default)
  // / 323 / 343 grouped
  // basis reads (CH 2 or 4 double2 per thread, G 2 or 4 vectors per group;
  // a trailing 3: three resident CTAs per SM)
  // read per launch (not cached) so tests can switch variants in-process
  const char* ev = std::getenv("SB_DCGS_A");
  const int variant = ev ? std::atoi(ev) : 24;
#define SB_DCGS_A_LAUNCH(KER)                                                        \
  {                                                                                 \
    static const int grid_a = wave_grid(KER);                                       \
    g_red_blocks_used = grid_a;                                                     \
    launch_k(KER, grid_a, kThreads, 0, s, Q, vstride, k, c, inv_gamma, w, n / 2, partials, nullptr, 0LL, nullptr, \
             0LL);                                                                  \
  }
  switch (variant) {
    case 0: launch_k(k_dcgs_a_g, kRedBlocks, kThreads, 0, s, Q, vstride, k, c, inv_gamma, w, n / 2, partials); break;
    case 32: SB_DCGS_A_LAUNCH((k_dcgs_a_g3<2, 2>)); break;
    case 34: SB_DCGS_A_LAUNCH((k_dcgs_a_g3<2, 4>)); break;
    case 343: SB_DCGS_A_LAUNCH((k_dcgs_a_g3<2, 4, 3>)); break;
    case 323: SB_DCGS_A_LAUNCH((k_dcgs_a_g3<2, 2, 3>)); break;
    case 2: SB_DCGS_A_LAUNCH(k_dcgs_a_g2<4>); break;
    default: SB_DCGS_A_LAUNCH((k_dcgs_a_g3<4, 2>)); break;
  }
#undef SB_DCGS_A_LAUNCH
}

void launch_arnoldi1(cudaStream_t s, double* Q, long long vstride, int k, const double* c, double inv_gamma,
                     const double* w, long long n, double* partials, const double* means, long long block,
                     long long ghost) {
  ++g_kernel_launches;
  double* wout = Q + (long long)(k + 1) * vstride;
  if (means) {
    static const int grid_m = wave_grid(k_dcgs_a_g3<4, 2, 2, true, true>);
    g_red_blocks_used = grid_m;
    launch_k(k_dcgs_a_g3<4, 2, 2, true, true>, grid_m, kThreads, 0, s, Q, vstride, k, c, inv_gamma, w, n / 2,
             partials, means, block / 2, wout, ghost / 2);
  } else {
    static const int grid_p = wave_grid(k_dcgs_a_g3<4, 2, 2, false, true>);
    g_red_blocks_used = grid_p;
    launch_k(k_dcgs_a_g3<4, 2, 2, false, true>, grid_p, kThreads, 0, s, Q, vstride, k, c, inv_gamma, w, n / 2,
             partials, nullptr, 0LL, wout, 0LL);
  }
}

void launch_dcgs_b_g(cudaStream_t s, const double* Q, long long vstride, int nv, const double* d, const double* w,
                     double* out, long long n, double* partials, const double* means, long long block,
                     long long ghost) {
  ++g_kernel_launches;
  static const int grid_b = wave_grid(k_dcgs_b_g<false>);
  static const int grid_bg = wave_grid(k_dcgs_b_g<true>);
  if (ghost) {
    g_red_blocks_used = grid_bg;
    launch_k(k_dcgs_b_g<true>, grid_bg, kThreads, 0, s, Q, vstride, nv, d, w, out, n / 2, partials, means,
             block / 2, ghost / 2);
  } else {
    g_red_blocks_used = grid_b;
    launch_k(k_dcgs_b_g<false>, grid_b, kThreads, 0, s, Q, vstride, nv, d, w, out, n / 2, partials, means,
             block / 2, ghost / 2);
  }
}

__global__ void k_block_means(const double* __restrict__ sums, int4 slot, double inv_count, double* __restrict__ means) {
  pdl_enter();
  if (threadIdx.x == 0) {
    means[0] = slot.x >= 0 ? sums[slot.x] * inv_count : 0.0;
    means[1] = slot.y >= 0 ? sums[slot.y] * inv_count : 0.0;
    means[2] = slot.z >= 0 ? sums[slot.z] * inv_count : 0.0;
    means[3] = slot.w >= 0 ? sums[slot.w] * inv_count : 0.0;
  }
}

void launch_block_means(cudaStream_t s, const double* sums, const int* slot, double inv_count, double* means) {
  ++g_kernel_launches;
  launch_k(k_block_means, 1, 32, 0, s, sums, make_int4(slot[0], slot[1], slot[2], slot[3]), inv_count, means);
}

void launch_finalize(cudaStream_t s, const double* partials, int nv, double* out) {
  launch_k(k_finalize, nv, kThreads, 0, s, partials, out, g_red_blocks_used);
  g_red_blocks_used = kRedBlocks;
}

void launch_sum_partial(cudaStream_t s, const double* x, long long n, double* partials) {
  ++g_kernel_launches;
  static const int grid = wave_grid(k_sum_partial);
  g_red_blocks_used = grid;
  launch_k(k_sum_partial, grid, kThreads, 0, s, x, n, partials);
}

void launch_sub_norm(cudaStream_t s, const double* a, const double* b, long long n, double* partials) {
  ++g_kernel_launches;
  static const int grid = wave_grid(k_sub_norm);
  g_red_blocks_used = grid;
  launch_k(k_sub_norm, grid, kThreads, 0, s, a, b, n, partials);
}

void launch_scale_div(cudaStream_t s, const double* w, double d, double* out, long long n) {
  ++g_kernel_launches;
  launch_k(k_scale_div, grid_for(n / 2), kThreads, 0, s, reinterpret_cast<const double2*>(w), d,
                                                    reinterpret_cast<double2*>(out), n / 2);
}

void launch_combo(cudaStream_t s, double* out, const double* x, const double* V, long long vstride, int nv,
                  const double* y, long long n) {
  // the kernels stage <= kMaxVec coefficients in shared memory: longer
  // combinations (GMRES restart >= 128) run in chunks, out accumulating
  for (int c0 = 0; c0 < nv || c0 == 0; c0 += kVecChunk) {
    const int nc = std::min(kVecChunk, nv - c0);
    ++g_kernel_launches;
    launch_k(k_combo, grid_for(n / 2), kThreads, 0, s, reinterpret_cast<double2*>(out),
             reinterpret_cast<const double2*>(c0 == 0 ? x : out), V + (long long)c0 * vstride, vstride, nc, y + c0,
             n / 2);
  }
}

// Textbook CGS2 Arnoldi step on nv basis vectors (krylov.py:111-115 with MGS
// replaced): h1 = V^T w, w -= V h1, h2 = V^T w, w -= V h2,
// nrm2 = ||w||^2.  Up to kVecChunk vectors the update and the next reduction
// share one read of the basis; a longer basis (restart >= 128) is processed in
// chunks of kVecChunk vectors -- the dots of a pass all see the same w, the
// updates accumulate.
void launch_cgs2(cudaStream_t s, const double* V, long long vstride, int nv, double* w, long long n,
                 double* partials, double* h1, double* h2, double* nrm2) {
  if (nv <= kVecChunk) {
    launch_multi_dot(s, V, vstride, nv, w, n, partials);
    launch_finalize(s, partials, nv, h1);
    launch_update_dot(s, V, vstride, nv, h1, w, n, partials, 0);
    launch_finalize(s, partials, nv, h2);
    launch_update_dot(s, V, vstride, nv, h2, w, n, partials, 1);
    launch_finalize(s, partials, 1, nrm2);
    return;
  }
  for (int pass = 0; pass < 2; ++pass) {
    double* h = pass == 0 ? h1 : h2;
    for (int c0 = 0; c0 < nv; c0 += kVecChunk) {
      const int nc = std::min(kVecChunk, nv - c0);
      launch_multi_dot(s, V + (long long)c0 * vstride, vstride, nc, w, n, partials);
      launch_finalize(s, partials, nc, h + c0);
    }
    for (int c0 = 0; c0 < nv; c0 += kVecChunk) {
      const int nc = std::min(kVecChunk, nv - c0);
      launch_update_dot(s, V + (long long)c0 * vstride, vstride, nc, h + c0, w, n, partials, 1);
      if (pass == 1 && c0 + nc == nv) launch_finalize(s, partials, 1, nrm2);  // ||w||^2 after the last update
      else g_red_blocks_used = kRedBlocks;
    }
  }
}

void launch_sub(cudaStream_t s, const double* a, const double* b, double* out, long long n) {
  launch_k(k_sub, grid_for(n / 2), kThreads, 0, s, reinterpret_cast<const double2*>(a),
                                             reinterpret_cast<const double2*>(b),
                                             reinterpret_cast<double2*>(out), n / 2);
}

}  // namespace sb
