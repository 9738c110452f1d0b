// sb_wave.cu -- red-black Gauss-Seidel sweeps as ONE wavefront launch per
// component, with the black pass served from L2 (sm_100a).
//
// A colour pass of a 256^3 level streams every operand of the face row from
// HBM (56 B per face); the two passes of a sweep stream them twice because a
// level's operands (~1.2 GB) exceed the 126 MB L2.  Here both passes of one
// component run in a single persistent launch, ordered as a wavefront along
// axis 0:
//
//     R0 R1 R2 | R3 B1 | R4 B2 | ... | R(n-1) B(n-3) | B(n-2) B(n-1) B0
//
// (R p = red faces of plane p, B p = black faces; lookahead K = 2 shown, 8 by
// default, SB_WAVE_K; the periodic
// wrap makes B0 wait for R(n-1)).  CTAs take (step, row-tile) work items from
// an atomic counter in that order; a black item waits until the red items of
// planes p-1, p, p+1 are complete (per-plane counters, release/acquire).
// Black therefore runs a few planes behind red, while that window's operands
// (~40 MB at 256^3) are still in L2, so each operand crosses HBM about once
// per component sweep instead of twice.
//
// Bit-identical to the per-colour kernels: red reads old values only, black
// reads the relaxed red values, each face's update is the same expression.
// Hazards: black p overwrites values that red p-1..p+1 read, and reads what
// they write -- both covered by the wait.  Iterate loads use ld.global.cg
// (L2 only): values written by other SMs during the launch are never served
// from a stale L1 line.  Items are handed out in order and a waiting item
// only depends on earlier items, which are held by running CTAs, so the
// scheme cannot deadlock whatever the number of resident CTAs.
//
// Used on 3D levels without odd periodic extents, outside slab decomposition,
// for the Laplacian / stress forms and the cell (pressure) sweeps.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdlib>
#include <vector>
#include "sb_kernels.h"

namespace sb {
extern long long g_kernel_launches;

namespace {

constexpr int WT = 256;       // threads per CTA
int wave_ctas() {  // resident CTAs per SM requested (SB_WAVE_CTAS, default 6)
  const char* e = std::getenv("SB_WAVE_CTAS");
  const int v = e ? std::atoi(e) : 6;
  return 148 * std::max(1, std::min(v, 8));
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct WaveGeom {
  Box b;          // unknowns of the swept array (face box of A / cell box)
  int off;        // colour offset of the interior-relative parity
  int rows;       // axis-1 rows per work item
  int tiles;      // work items per (plane, colour)
  int np;         // planes along axis 0
  int per0;       // axis 0 periodic
  int nsteps;
};

// relaxed value of the face/cell at coordinates ci (index f); the update is
// the per-colour kernels' expression (k_face_colour / k_cell_colour)
template <int DIM, int FORM, int A, bool PA, bool CELL, bool CG>
__device__ __forceinline__ double wave_relax(const LevelDev& L, const Ptr3& u, const double* __restrict__ rhs,
                                            double omega, int f, const int* ci) {
  double dg;
  if (CELL) {
    const double* phi = u.p[0];
    const double lp = cell_row<DIM, PA, CG>(L, phi, f, ci, dg);
    const double res = __ldg(rhs + f) - lp;
    return ldu<CG>(phi, f) + omega * res / dg;
  }
  const double* uc[3] = {u.p[0], u.p[1], u.p[2]};
  const double au = face_row<DIM, FORM, A, PA, true, CG>(L, uc, f, ci, dg);
  const double res = __ldg(rhs + f) - au;
  return ldu<CG>(uc[A], f) + omega * (res / dg);
}

// One work item: the same-colour unknowns of rows [r0, r0 + rows) of a plane
// (rows * half2 <= 2 * WT), up to two per thread, both relaxed before either
// is stored so their loads overlap.  (rr, kk): the thread's row / slot
// offsets, fixed for the launch.
template <int DIM, int FORM, int A, bool PA, bool CELL, bool CG>
__device__ __forceinline__ void wave_item(const LevelDev& L, const Ptr3& u, const double* __restrict__ rhs,
                                          double omega, const WaveGeom& G, int plane, int tile, int colour,
                                          const int* rr, const int* kk) {
  const Box& b = G.b;
  const int r0 = b.lo[1] + tile * G.rows;
  double* out = CELL ? u.p[0] : u.p[A];
  int f[2];
  bool ok[2];
  double nv[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    int ci[3];
    ci[0] = b.lo[0] + plane;
    ci[1] = r0 + rr[h];
    ci[2] = b.lo[2] + ((colour + G.off - ci[0] - ci[1] - b.lo[2]) & 1) + 2 * kk[h];
    ok[h] = rr[h] < G.rows && ci[1] <= b.hi[1] && ci[2] <= b.hi[2];
    f[h] = ci[0] * L.s0 + ci[1] * L.s1 + ci[2];
    nv[h] = ok[h] ? wave_relax<DIM, FORM, A, PA, CELL, CG>(L, u, rhs, omega, f[h], ci) : 0.0;
  }
  if (ok[0]) out[f[0]] = nv[0];
  if (ok[1]) out[f[1]] = nv[1];
}

// Persistent CTAs take work items (step, row tile) from the counter in step
// order, one barrier per item: the next item index is fetched while the
// current one runs.  Black items wait (thread 0 spinning) until every red
// item of planes p-1, p, p+1 has signalled completion.
template <int DIM, int FORM, int A, bool PA, bool CELL>
__global__ void __launch_bounds__(WT)
k_wave(LevelDev L, Ptr3 u, const double* __restrict__ rhs, double omega, WaveGeom G,
       const int* __restrict__ steps, int* ctr) {
  __shared__ int s_next[2];
  const int total = G.nsteps * G.tiles;
  int* done = ctr + 1;
  const int half2 = (G.b.hi[2] - G.b.lo[2] + 2) / 2;
  int rr[2], kk[2];
  for (int h = 0; h < 2; ++h) {
    const int t = threadIdx.x + WT * h;
    rr[h] = t / half2;
    kk[h] = t - rr[h] * half2;
  }
  if (threadIdx.x == 0) s_next[0] = atomicAdd(ctr, 1);
  __syncthreads();
  for (int k = 0;; k ^= 1) {
    const int it = s_next[k];
    if (it >= total) return;
    const int st = __ldg(steps + it / G.tiles);
    const int tile = it % G.tiles;
    const int plane = st >> 1, colour = st & 1;
    if (threadIdx.x == 0) s_next[k ^ 1] = atomicAdd(ctr, 1);
    if (colour == 1) {
      if (threadIdx.x == 0) {
        for (int d = -1; d <= 1; ++d) {
          int q = plane + d;
          if (q < 0 || q >= G.np) {
            if (!G.per0) continue;
            q = q < 0 ? q + G.np : q - G.np;
          }
          while (ld_acquire(done + q) < G.tiles) __nanosleep(64);
        }
      }
      __syncthreads();
      // red values written by other SMs: read through L2 only
      wave_item<DIM, FORM, A, PA, CELL, true>(L, u, rhs, omega, G, plane, tile, 1, rr, kk);
      __syncthreads();
    } else {
      // red items read values nobody writes before they complete (L1 allowed)
      wave_item<DIM, FORM, A, PA, CELL, false>(L, u, rhs, omega, G, plane, tile, 0, rr, kk);
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) atomicAdd(done + plane, 1);
    }
  }
}

bool all_per(const LevelDev& L) { return L.bclo[0] == BC_PER && L.bclo[1] == BC_PER && L.bclo[2] == BC_PER; }

WaveGeom geom(const LevelDev& L, bool cell, int A, int nsteps) {
  WaveGeom G;
  for (int a = 0; a < 3; ++a) {
    G.b.lo[a] = 0;
    G.b.hi[a] = L.n[a] - 1;
  }
  G.off = 0;
  if (!cell && L.bclo[A] != BC_PER) {
    G.b.lo[A] = 1;
    G.b.hi[A] = L.n[A] - 1;
    G.off = 1;
  }
  const int e1 = G.b.hi[1] - G.b.lo[1] + 1;
  const int half2 = (G.b.hi[2] - G.b.lo[2] + 2) / 2;
  // rows per item: as many as fit 2 * WT unknowns (a row is never split)
  G.rows = std::max(1, std::min(e1, 2 * WT / std::max(half2, 1)));
  G.tiles = (e1 + G.rows - 1) / G.rows;
  G.np = G.b.hi[0] - G.b.lo[0] + 1;
  G.per0 = L.bclo[0] == BC_PER;
  G.nsteps = nsteps;
  return G;
}

template <int DIM, int FM, int A>
void face_wave_t(cudaStream_t s, const LevelDev& L, Ptr3 u, const double* rhs, double omega, const int* steps,
                 int nsteps, int* ctr) {
  const WaveGeom G = geom(L, false, A, nsteps);
  const int grid = std::min(wave_ctas(), nsteps * G.tiles);
  (void)cudaMemsetAsync(ctr, 0, sizeof(int) * (G.np + 1), s);
  if (all_per(L)) k_wave<DIM, FM, A, true, false><<<grid, WT, 0, s>>>(L, u, rhs, omega, G, steps, ctr);
  else k_wave<DIM, FM, A, false, false><<<grid, WT, 0, s>>>(L, u, rhs, omega, G, steps, ctr);
}

}  // namespace

// The step order of one component sweep (see the file comment): plane p,
// colour c encoded as 2p + c.  np planes along axis 0, periodic or not.
std::vector<int> wave_steps(int np, bool per0, int K) {
  // K: red lookahead (planes)
  std::vector<int> s;
  auto R = [&](int p) { s.push_back(2 * p); };
  auto B = [&](int p) { s.push_back(2 * p + 1); };
  if (np < 3) {
    for (int p = 0; p < np; ++p) R(p);
    for (int p = 0; p < np; ++p) B(p);
    return s;
  }
  const int r0 = std::min(np, K + 1);
  for (int p = 0; p < r0; ++p) R(p);
  if (per0) {
    for (int j = 1; j < np; ++j) {
      if (j + K < np) R(j + K);
      B(j);
    }
    B(0);
  } else {
    for (int j = 0; j < np; ++j) {
      if (j + K + 1 < np) R(j + K + 1);
      B(j);
    }
  }
  return s;
}

bool wave_supported(const LevelDev& L, int dim, int form) {
  if (dim != 3 || form == F_BULK || L.dist0) return false;
  if ((L.n[2] + 2) / 2 > 2 * WT) return false;  // a row of same-colour unknowns fits one item
  for (int a = 0; a < 3; ++a)
    if (L.bclo[a] == BC_PER && (L.n[a] & 1)) return false;
  return true;
}

void launch_face_wave(cudaStream_t s, const LevelDev& L, int form, int A, Ptr3 u, const double* rhsA,
                      double omega, const int* steps, int nsteps, int* ctr) {
  ++g_kernel_launches;
  if (form == F_LAP) {
    if (A == 0) face_wave_t<3, F_LAP, 0>(s, L, u, rhsA, omega, steps, nsteps, ctr);
    else if (A == 1) face_wave_t<3, F_LAP, 1>(s, L, u, rhsA, omega, steps, nsteps, ctr);
    else face_wave_t<3, F_LAP, 2>(s, L, u, rhsA, omega, steps, nsteps, ctr);
  } else {
    if (A == 0) face_wave_t<3, F_STRESS, 0>(s, L, u, rhsA, omega, steps, nsteps, ctr);
    else if (A == 1) face_wave_t<3, F_STRESS, 1>(s, L, u, rhsA, omega, steps, nsteps, ctr);
    else face_wave_t<3, F_STRESS, 2>(s, L, u, rhsA, omega, steps, nsteps, ctr);
  }
}

void launch_cell_wave(cudaStream_t s, const LevelDev& L, double* phi, const double* rhs, double omega,
                      const int* steps, int nsteps, int* ctr) {
  ++g_kernel_launches;
  const WaveGeom G = geom(L, true, 0, nsteps);
  const int grid = std::min(wave_ctas(), nsteps * G.tiles);
  (void)cudaMemsetAsync(ctr, 0, sizeof(int) * (G.np + 1), s);
  Ptr3 u{{phi, nullptr, nullptr}};
  if (all_per(L)) k_wave<3, F_LAP, 0, true, true><<<grid, WT, 0, s>>>(L, u, rhs, omega, G, steps, ctr);
  else k_wave<3, F_LAP, 0, false, true><<<grid, WT, 0, s>>>(L, u, rhs, omega, G, steps, ctr);
}

}  // namespace sb
