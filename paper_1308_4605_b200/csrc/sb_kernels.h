// sb_kernels.h -- host-side launchers for the sm_100a kernels (sb_kernels.cu).
#pragma once
#include <cuda_runtime.h>
#include <vector>
#include "sb_device.cuh"

namespace sb {

// Kernel launch with programmatic stream serialization (see pdl_enter);
// SB_PDL=0 falls back to plain stream order.
bool pdl_enabled();
template <typename... KA, typename... AA>
inline void launch_k(void (*k)(KA...), dim3 g, dim3 b, size_t smem, cudaStream_t s, AA&&... a) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, static_cast<AA&&>(a)...);
}

struct Ptr3 { double* p[3]; };
struct CPtr3 { const double* p[3]; };

// Sub-box of a level: lo/hi inclusive per internal axis.
struct Box { int lo[3], hi[3]; };

// The coarse-level tail of a V-cycle (levels of <= kCoarseCells cells) run by
// one CTA: level 0 of the chain receives its right-hand side from the fine
// levels' residual->restriction and returns its correction in x.
constexpr int kCoarseMaxLevels = 10;
constexpr long long kCoarseCells = 1024;   // 2D (32^2)
constexpr long long kCoarseCells3 = 512;   // 3D (8^3)
struct CoarseLv {
  LevelDev d;
  double* x[3];      // iterate (face components; cell uses x[0])
  double* rhs[3];
  double* tmp;       // two-phase scratch (odd periodic extents)
  long long block;   // elements per array of the level
  int two_phase;
  int pad_;
};
struct CoarseChain {
  int nl, pad_[3];
  CoarseLv lv[kCoarseMaxLevels];
};

// colour passes (multigrid.py:318-340)
// z: first-sweep-from-zero variants (k_face_colour): 0 plain, 1 later
// components zero, 2 also the relaxed array zero, 3 as 2 + store the partner's
// zero (replaces the zero fill; all-periodic pad-free levels only).
// ext0: also relax ext0 ghost planes on each side of axis 0 (slab levels)
// w_lo..w_hi (w_hi >= w_lo): only these axis-0 planes (slab levels relax their
// boundary planes first so the halo exchange overlaps the interior)
void launch_face_colour(cudaStream_t s, const LevelDev& L, int dim, int form, int A, Ptr3 u,
                        const double* rhsA, int parity, double omega, int z = 0, int ext0 = 0, int w_lo = 0,
                        int w_hi = -1);
void launch_cell_colour(cudaStream_t s, const LevelDev& L, int dim, double* phi, const double* rhs,
                        int parity, double omega, int z = 0, int ext0 = 0, int w_lo = 0, int w_hi = -1);
// two-phase variants for levels with an odd periodic extent (same-colour
// cells couple through the wrap): compute all, then update (reference order)
void launch_face_colour_tmp(cudaStream_t s, const LevelDev& L, int dim, int form, int A, Ptr3 u,
                            const double* rhsA, double* tmp, int parity, double omega);
void launch_cell_colour_tmp(cudaStream_t s, const LevelDev& L, int dim, double* phi, const double* rhs,
                            double* tmp, int parity, double omega);
bool level_needs_two_phase(const LevelDev& L, int dim);
// row-vector kernels for large all-periodic 3D levels (sb_rowv.cu; the callers
// are launch_face_colour / launch_face_res3 / launch_apply_M, which count the launch)
bool rowv_supported(const LevelDev& L, int dim, int form);         // residual field, apply_M
bool rowv_colour_supported(const LevelDev& L, int dim, int form);  // colour passes (opt-in)
void launch_face_colour_rv(cudaStream_t s, const LevelDev& L, int form, int A, Ptr3 u, const double* rhsA,
                           int parity, double omega);
void launch_face_res3_rv(cudaStream_t s, const LevelDev& L, int form, CPtr3 x, CPtr3 rhs, Ptr3 out);
void launch_apply_M_rv(cudaStream_t s, const LevelDev& L, int form, CPtr3 u, const double* p, Ptr3 out_u,
                       double* out_p);
// fused residual -> restriction (multigrid.py:403-406 + :177-233)
void launch_face_resid_restrict(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, int dim,
                                int form, int A, CPtr3 u, const double* rhsA, double* coarseA);
void launch_cell_resid_restrict(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, int dim,
                                const double* phi, const double* rhs, double* coarse);
// split residual / restriction (large levels): residual field to memory, then restrict
void launch_face_res3(cudaStream_t s, const LevelDev& L, int dim, int form, CPtr3 x, CPtr3 rhs, Ptr3 out);
void launch_face_restrict(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, int dim, int A, const double* r,
                          double* coarse);
void launch_cell_res(cudaStream_t s, const LevelDev& L, int dim, const double* x, const double* rhs,
                     double* out);
void launch_cell_restrict(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, int dim, const double* r,
                          double* coarse);
// prolongation + add (multigrid.py:185-192, :236-295, :431-436)
void launch_face_prolong_add(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, int dim, int A,
                             const double* coarseA, double* fineA);
void launch_cell_prolong_add(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, int dim,
                             const double* coarse, double* fine);
// one-CTA coarse tail (sb_kernels.cu k_coarse_face / k_coarse_cell); dchain in device memory
void launch_coarse_face(cudaStream_t s, int dim, int form, bool all_periodic, const CoarseChain* dchain,
                        int sweeps_down, int sweeps_up, int bottom, double omega);
void launch_coarse_cell(cudaStream_t s, int dim, bool all_periodic, const CoarseChain* dchain,
                        int sweeps_down, int sweeps_up, int bottom, double omega);
// full-level operators
void launch_apply_M(cudaStream_t s, const LevelDev& L, int dim, int form, CPtr3 u, const double* p,
                    Ptr3 out_u, double* out_p);
// out_A = (rhs_A - G q_A) - (A x)_A   (q or x may be null -> term dropped)
void launch_face_residual(cudaStream_t s, const LevelDev& L, int dim, int form, CPtr3 x,
                          CPtr3 rhs, const double* q, Ptr3 out);
void launch_cell_residual(cudaStream_t s, const LevelDev& L, int dim, const double* x,
                          const double* rhs, double* out);  // rhs may be null -> out = L x
// preconditioner glue (precond.py:118-152, schur.py:59-78)
void launch_div_add(cudaStream_t s, const LevelDev& L, int dim, CPtr3 u, const double* rp, double* out);
void launch_p1_glue(cudaStream_t s, const LevelDev& L, int dim, int form, Ptr3 xu, const double* phi,
                    const double* bc, double* xp, double sign);
void launch_schur(cudaStream_t s, const LevelDev& L, int form, const double* r, const double* phi,
                  double* out, double sign);
void launch_face_sub_grad(cudaStream_t s, const LevelDev& L, int dim, CPtr3 ru, const double* q, Ptr3 out);
// setup: coarsening (multigrid.py:112-169), inverse densities, checks
void launch_coarsen_cellmean(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, int dim,
                             const double* fine, double* coarse);
void launch_coarsen_face(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, int dim, int A,
                         const double* fine, double* coarse);
void launch_coarsen_edge(cudaStream_t s, const LevelDev& Lf, const LevelDev& Lc, int dim, int e,
                         const double* fine, double* coarse);
// cflag (nullable): |= 1 unless every non-wall rho_face equals *ref (constant-density level)
void launch_beta(cudaStream_t s, const LevelDev& L, int A, const double* rho, double* beta, int* flag,
                 int* cflag = nullptr, const double* ref = nullptr);
void launch_check_diag(cudaStream_t s, const LevelDev& L, int dim, int form, int* flags);
// the smoother diagonals as arrays (face: Ptr3 with p[2] != null; cell: nullable)
// the reference's public div / grad (operators.py:182-198), bit-exact
void launch_div(cudaStream_t s, const LevelDev& L, int dim, CPtr3 u, double* out);
void launch_grad(cudaStream_t s, const LevelDev& L, int dim, const double* p, Ptr3 out);
void launch_write_diag(cudaStream_t s, const LevelDev& L, int dim, int form, Ptr3 face_diag, double* cell_diag);
// device-side make_coefficients + rescale: rho_face[A] from rho_cell, mu_e[e]
// = scale * edge mean of L.mu_c (unscaled at the call), x *= scale
void launch_cell_to_face(cudaStream_t s, const LevelDev& L, int dim, int A, const double* cell, double* face);
void launch_cell_to_edge(cudaStream_t s, const LevelDev& L, int dim, int e, double* out, double scale);
void launch_scale(cudaStream_t s, double* x, double scale, long long n);
// all-periodic level: flag |= 1 unless mu_e == edge_mean(mu_c) to roundoff everywhere
void launch_check_mue(cudaStream_t s, const LevelDev& L, int dim, int* flag);
// box utilities
void launch_box_fill(cudaStream_t s, const LevelDev& L, Box b, double* x, double v);
void launch_box_add_scalar(cudaStream_t s, const LevelDev& L, Box b, double* x, const double* sum,
                           double inv_count);  // x -= sum*inv_count
void launch_axpy_box(cudaStream_t s, const LevelDev& L, Box b, double* y, const double* x);  // y += x
void launch_axpy_scalar(cudaStream_t s, double* y, const double* x);  // *y += *x (one thread)
void launch_max_scalar(cudaStream_t s, double* y, const double* x, bool neg);  // *y = max(*y, +-*x)
void launch_neg_copy(cudaStream_t s, double* y, const double* x);             // *y = -*x
// inhomogeneous walls (operators.py:267-291, 484-512)
void launch_wall_tangent(cudaStream_t s, const LevelDev& L, int A, int B, int side, const double* plane,
                         double* out);  // out_A -= 2 mu_e v / h^2 on the rows next to wall (B, side)
void launch_sum_abs_partial(cudaStream_t s, const double* x, long long n, double* partials);  // sum, sum|x|

// flat-vector kernels (GMRES; whole padded box, pads are zero)
int reduce_blocks();
void launch_multi_dot(cudaStream_t s, const double* V, long long vstride, int nv, const double* w,
                      long long n, double* partials);
void launch_update_dot(cudaStream_t s, const double* V, long long vstride, int nv, const double* h,
                       double* w, long long n, double* partials, int mode);  // mode 0: dots, 1: norm
void launch_finalize(cudaStream_t s, const double* partials, int nv, double* out);
// Gram-matrix variant of the delayed-reorthogonalisation passes
// means (nullable): the deferred null projection applied to w on load (as pass B)
void launch_dcgs_a_g(cudaStream_t s, double* Q, long long vstride, int k, const double* c, double inv_gamma,
                     const double* w, long long n, double* partials, const double* means = nullptr,
                     long long block = 0);
// One-pass Arnoldi (Gram variant without pass B): pass A plus ||w||^2 (slot
// 2k+2) and the (means-projected) w stored to basis slot k+1; ghost: elements
// kept 0 at each block end (slab blocks)
void launch_arnoldi1(cudaStream_t s, double* Q, long long vstride, int k, const double* c, double inv_gamma,
                     const double* w, long long n, double* partials, const double* means = nullptr,
                     long long block = 0, long long ghost = 0);
// means (nullable): per-block values subtracted from w first (deferred null projection,
// blocks of `block` elements, at most 4)
void launch_dcgs_b_g(cudaStream_t s, const double* Q, long long vstride, int nv, const double* d, const double* w,
                     double* out, long long n, double* partials, const double* means = nullptr,
                     long long block = 0, long long ghost = 0);  // ghost: elements kept 0 at each block end
// means[b] = sums[slot[b]] * inv_count (0 where slot[b] < 0), b < 4
void launch_block_means(cudaStream_t s, const double* sums, const int* slot, double inv_count, double* means);
// delayed-reorthogonalisation Arnoldi passes (see sb_solver.cu gmres())
void launch_dcgs_a(cudaStream_t s, double* Q, long long vstride, int k, const double* c, double inv_gamma,
                   const double* w, long long n, double* partials);
void launch_dcgs_b(cudaStream_t s, const double* Q, long long vstride, int nv, const double* d, const double* w,
                   double* out, long long n, double* partials);
void launch_sum_partial(cudaStream_t s, const double* x, long long n, double* partials);
void launch_scale_div(cudaStream_t s, const double* w, double d, double* out, long long n);
void launch_combo(cudaStream_t s, double* out, const double* x, const double* V, long long vstride,
                  int nv, const double* y, long long n);
// CGS2 Arnoldi step (any number of basis vectors; chunked above 120)
void launch_cgs2(cudaStream_t s, const double* V, long long vstride, int nv, double* w, long long n,
                 double* partials, double* h1, double* h2, double* nrm2);  // out = x + sum y_i V_i (y on device)
void launch_sub(cudaStream_t s, const double* a, const double* b, double* out, long long n);  // out=a-b
void launch_sub_norm(cudaStream_t s, const double* a, const double* b, long long n, double* partials);

}  // namespace sb
