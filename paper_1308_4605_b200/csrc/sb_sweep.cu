// sb_sweep.cu -- fused two-colour Gauss-Seidel sweeps (2.5D streaming, sm_100a).
//
// One kernel performs BOTH colour passes of one component (multigrid.py:334-340
// for a face component, :321-324 for cells) out of place: it reads the
// current iterate x (never modified during the launch) and writes the swept
// iterate to a second buffer.  A CTA owns a TJ x TK tile of the (axis-1,
// axis-2) plane and marches along axis 0 over a chunk of planes:
//
//   step p:  prefetch old plane p+2 (cp.async, ring of 4 planes, halo 2)
//            R_p   = old plane p with its RED unknowns relaxed   (tile + ring 1)
//            black = relax the BLACK unknowns of plane p-1 from R_{p-2..p}
//            write plane p-1 (both colours) to the output buffer
//
// Red faces never neighbour red faces (even periodic extents), so R_p depends
// on old values only and the redundant ring computed by neighbouring CTAs is
// bit-identical; black reads only red neighbours and its own old value.  The
// result therefore equals the reference's sequential red-then-black pass to the
// bit, while every array streams through HBM once per component sweep (64 B per
// face instead of 2 x 56 B for two colour passes).  Levels with an
// odd periodic extent, 2D grids and the stress+bulk form use the per-colour
// kernels instead.
#include <cuda_runtime.h>
#include <algorithm>
#include "sb_kernels.h"

namespace sb {
extern long long g_kernel_launches;

namespace {

constexpr int NT = 256;
constexpr int TJ = 16, TK = 32;
constexpr int RJ = TJ + 4, RK = TK + 4;  // old planes: halo 2
constexpr int QJ = TJ + 2, QK = TK + 2;  // relaxed planes: halo 1
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

struct Ext {
  int e[3];
  bool p[3];
};

// absolute coordinate -> array coordinate (wrapped), or -1 if outside a wall axis
__device__ __forceinline__ int acoord(const Ext& E, const LevelDev& L, int a, int x) {
  if (E.p[a]) return wrapc(x, L.n[a]);
  return (x >= 0 && x < E.e[a]) ? x : -1;
}

// stage plane q (ring-2 halo) of x into a shared slot
__device__ __forceinline__ void stage(const LevelDev& L, const Ext& E, const double* x, double* slot, int q,
                                     int j0, int k0) {
  const int qa = acoord(E, L, 0, q);
  for (int t = threadIdx.x; t < RJ * RK; t += NT) {
    const int jj = t / RK, kk = t - jj * RK;
    const int ja = acoord(E, L, 1, j0 - 2 + jj), ka = acoord(E, L, 2, k0 - 2 + kk);
    if (qa >= 0 && ja >= 0 && ka >= 0) cp_async8(slot + t, x + qa * L.s0 + ja * L.s1 + ka);
    else slot[t] = 0.0;
  }
}

__device__ __forceinline__ int mod3(int p) { return ((p % 3) + 3) % 3; }

template <int FORM, int A>
__global__ void __launch_bounds__(NT)
k_face_sweep2(LevelDev L, CPtr3 u, double* __restrict__ unew, const double* __restrict__ rhs, double omega,
              int chunk) {
  __shared__ double so[4][RJ * RK];
  __shared__ double sr[3][QJ * QK];
  Ext E;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    E.p[a] = per(L, a);
    E.e[a] = L.n[a] + ((a == A && !E.p[a]) ? 1 : 0);
  }
  const int off = E.p[A] ? 0 : 1;  // interior-relative parity offset (multigrid.py:335-339)
  const int k0 = blockIdx.x * TK, j0 = blockIdx.y * TJ;
  const int i0 = blockIdx.z * chunk, i1 = min(i0 + chunk, E.e[0]) - 1;
  const double* ua = u.p[A];
  auto unknown = [&](const int* ca) {  // array coordinates of a face of A
    if (!E.p[A] && (ca[A] == 0 || ca[A] == L.n[A])) return false;
    return true;
  };

  stage(L, E, ua, so[(i0 - 2) & 3], i0 - 2, j0, k0);
  stage(L, E, ua, so[(i0 - 1) & 3], i0 - 1, j0, k0);
  stage(L, E, ua, so[i0 & 3], i0, j0, k0);
  cp_commit();
  stage(L, E, ua, so[(i0 + 1) & 3], i0 + 1, j0, k0);
  cp_commit();

  for (int p = i0 - 1; p <= i1 + 1; ++p) {
    if (p + 2 <= i1 + 2) stage(L, E, ua, so[(p + 2) & 3], p + 2, j0, k0);
    cp_commit();
    cp_wait1();
    __syncthreads();
    // ---- R_p: relax the red unknowns of plane p on the tile + ring 1 ----
    {
      double* R = sr[mod3(p)];
      const double* O0 = so[(p - 1) & 3];
      const double* O1 = so[p & 3];
      const double* O2 = so[(p + 1) & 3];
      const int pa = acoord(E, L, 0, p);
      for (int q = threadIdx.x; q < QJ * QK; q += NT) {  // start from the old plane
        const int jj = q / QK, kk = q - jj * QK;
        R[q] = O1[(jj + 1) * RK + (kk + 1)];
      }
      __syncthreads();
      if (pa >= 0) {
        for (int q = threadIdx.x; q < QJ * RED_PER_ROW; q += NT) {  // lanes on red faces only
          const int jj = q / RED_PER_ROW, m = q - jj * RED_PER_ROW;
          const int j = j0 - 1 + jj;
          const int kk = ((off - p - j - (k0 - 1)) & 1) + 2 * m;
          const int k = k0 - 1 + kk;
          int ca[3] = {pa, acoord(E, L, 1, j), acoord(E, L, 2, k)};
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
          const int f = ca[0] * L.s0 + ca[1] * L.s1 + ca[2];
          double dg;
          const double au = face_row_core<3, FORM, A>(L, s, u.p, f, ca, dg);
          const double res = __ldg(rhs + f) - au;
          R[jj * QK + kk] = s.c + omega * (res / dg);
        }
      }
    }
    __syncthreads();
    // ---- black unknowns of plane p-1 (tile) from R_{p-2}, R_{p-1}, R_p ----
    const int pb = p - 1;
    if (pb >= i0 && pb <= i1) {
      double* Rm = sr[mod3(pb)];
      const double* Rlo = sr[mod3(pb - 1)];
      const double* Rhi = sr[mod3(pb + 1)];
      const int pa = acoord(E, L, 0, pb);
      for (int q = threadIdx.x; q < TJ * (TK / 2); q += NT) {
        const int jj = q / (TK / 2), m = q - jj * (TK / 2);
        const int j = j0 + jj;
        const int k = k0 + ((1 + off - pb - j - k0) & 1) + 2 * m;  // black: parity 1
        const int ca[3] = {pa, j, k};
        if (j >= E.e[1] || k >= E.e[2] || !unknown(ca)) continue;
        const int o = (jj + 1) * QK + (k - k0 + 1);
        UA7 s;
        s.c = Rm[o];
        s.p[0] = Rhi[o];
        s.m[0] = Rlo[o];
        s.p[1] = Rm[o + QK];
        s.m[1] = Rm[o - QK];
        s.p[2] = Rm[o + 1];
        s.m[2] = Rm[o - 1];
        const int f = ca[0] * L.s0 + ca[1] * L.s1 + ca[2];
        double dg;
        const double au = face_row_core<3, FORM, A>(L, s, u.p, f, ca, dg);
        const double res = __ldg(rhs + f) - au;
        Rm[o] = s.c + omega * (res / dg);
      }
      __syncthreads();
      // write plane pb (both colours) -- coalesced along k
      for (int q = threadIdx.x; q < TJ * TK; q += NT) {
        const int jj = q / TK, kk = q - jj * TK;
        const int j = j0 + jj, k = k0 + kk;
        if (j < E.e[1] && k < E.e[2]) unew[pa * L.s0 + j * L.s1 + k] = Rm[(jj + 1) * QK + kk + 1];
      }
    }
  }
}

template <int DIM>
__global__ void __launch_bounds__(NT)
k_cell_sweep2(LevelDev L, const double* __restrict__ phi, double* __restrict__ pnew,
              const double* __restrict__ rhs, double omega, int chunk) {
  __shared__ double so[4][RJ * RK];
  __shared__ double sr[3][QJ * QK];
  Ext E;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    E.p[a] = per(L, a);
    E.e[a] = L.n[a];
  }
  const int k0 = blockIdx.x * TK, j0 = blockIdx.y * TJ;
  const int i0 = blockIdx.z * chunk, i1 = min(i0 + chunk, E.e[0]) - 1;

  stage(L, E, phi, so[(i0 - 2) & 3], i0 - 2, j0, k0);
  stage(L, E, phi, so[(i0 - 1) & 3], i0 - 1, j0, k0);
  stage(L, E, phi, so[i0 & 3], i0, j0, k0);
  cp_commit();
  stage(L, E, phi, so[(i0 + 1) & 3], i0 + 1, j0, k0);
  cp_commit();

  for (int p = i0 - 1; p <= i1 + 1; ++p) {
    if (p + 2 <= i1 + 2) stage(L, E, phi, so[(p + 2) & 3], p + 2, j0, k0);
    cp_commit();
    cp_wait1();
    __syncthreads();
    {
      double* R = sr[mod3(p)];
      const double* O0 = so[(p - 1) & 3];
      const double* O1 = so[p & 3];
      const double* O2 = so[(p + 1) & 3];
      const int pa = acoord(E, L, 0, p);
      for (int q = threadIdx.x; q < QJ * QK; q += NT) {
        const int jj = q / QK, kk = q - jj * QK;
        R[q] = O1[(jj + 1) * RK + (kk + 1)];
      }
      __syncthreads();
      if (pa >= 0) {
        for (int q = threadIdx.x; q < QJ * RED_PER_ROW; q += NT) {
          const int jj = q / RED_PER_ROW, m = q - jj * RED_PER_ROW;
          const int j = j0 - 1 + jj;
          const int kk = ((-p - j - (k0 - 1)) & 1) + 2 * m;
          const int k = k0 - 1 + kk;
          int ca[3] = {pa, acoord(E, L, 1, j), acoord(E, L, 2, k)};
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
          const int c = ca[0] * L.s0 + ca[1] * L.s1 + ca[2];
          double dg;
          const double lp = cell_row_core<3>(L, s, c, ca, dg);
          const double res = __ldg(rhs + c) - lp;
          R[jj * QK + kk] = s.c + omega * res / dg;
        }
      }
    }
    __syncthreads();
    const int pb = p - 1;
    if (pb >= i0 && pb <= i1) {
      double* Rm = sr[mod3(pb)];
      const double* Rlo = sr[mod3(pb - 1)];
      const double* Rhi = sr[mod3(pb + 1)];
      for (int q = threadIdx.x; q < TJ * (TK / 2); q += NT) {
        const int jj = q / (TK / 2), m = q - jj * (TK / 2);
        const int j = j0 + jj;
        const int k = k0 + ((1 - pb - j - k0) & 1) + 2 * m;
        if (j >= E.e[1] || k >= E.e[2]) continue;
        const int ca[3] = {pb, j, k};
        const int o = (jj + 1) * QK + (k - k0 + 1);
        UA7 s;
        s.c = Rm[o];
        s.p[0] = Rhi[o];
        s.m[0] = Rlo[o];
        s.p[1] = Rm[o + QK];
        s.m[1] = Rm[o - QK];
        s.p[2] = Rm[o + 1];
        s.m[2] = Rm[o - 1];
        const int c = ca[0] * L.s0 + ca[1] * L.s1 + ca[2];
        double dg;
        const double lp = cell_row_core<3>(L, s, c, ca, dg);
        const double res = __ldg(rhs + c) - lp;
        Rm[o] = s.c + omega * res / dg;
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

inline dim3 sweep_grid(int e0, int e1, int e2, int& chunk) {
  const int gx = (e2 + TK - 1) / TK, gy = (e1 + TJ - 1) / TJ;
  const int cols = gx * gy;
  int nch = std::max(1, std::min(e0 / 16, (148 * 4 + cols - 1) / cols));
  if (nch < 1) nch = 1;
  chunk = (e0 + nch - 1) / nch;
  nch = (e0 + chunk - 1) / chunk;
  return dim3(gx, gy, nch);
}

}  // namespace

bool sweep2_supported(const LevelDev& L, int dim, int form) {
  if (dim != 3 || form == F_BULK) return false;
  for (int a = 0; a < 3; ++a)
    if (L.n[a] < 8 || (L.bclo[a] == BC_PER && (L.n[a] & 1))) return false;
  return true;
}

void launch_face_sweep2(cudaStream_t s, const LevelDev& L, int form, int A, CPtr3 u, double* unew,
                        const double* rhsA, double omega) {
  ++g_kernel_launches;
  int e[3];
  for (int a = 0; a < 3; ++a) e[a] = L.n[a] + ((a == A && L.bclo[a] != BC_PER) ? 1 : 0);
  int chunk;
  const dim3 g = sweep_grid(e[0], e[1], e[2], chunk);
  if (form == F_LAP) {
    if (A == 0) k_face_sweep2<F_LAP, 0><<<g, NT, 0, s>>>(L, u, unew, rhsA, omega, chunk);
    else if (A == 1) k_face_sweep2<F_LAP, 1><<<g, NT, 0, s>>>(L, u, unew, rhsA, omega, chunk);
    else k_face_sweep2<F_LAP, 2><<<g, NT, 0, s>>>(L, u, unew, rhsA, omega, chunk);
  } else {
    if (A == 0) k_face_sweep2<F_STRESS, 0><<<g, NT, 0, s>>>(L, u, unew, rhsA, omega, chunk);
    else if (A == 1) k_face_sweep2<F_STRESS, 1><<<g, NT, 0, s>>>(L, u, unew, rhsA, omega, chunk);
    else k_face_sweep2<F_STRESS, 2><<<g, NT, 0, s>>>(L, u, unew, rhsA, omega, chunk);
  }
}

void launch_cell_sweep2(cudaStream_t s, const LevelDev& L, const double* phi, double* pnew, const double* rhs,
                        double omega) {
  ++g_kernel_launches;
  int chunk;
  const dim3 g = sweep_grid(L.n[0], L.n[1], L.n[2], chunk);
  k_cell_sweep2<3><<<g, NT, 0, s>>>(L, phi, pnew, rhs, omega, chunk);
}

}  // namespace sb
