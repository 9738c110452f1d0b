/*
 * stokesb200.h -- C ABI of the B200 (sm_100a) preconditioned MAC-Stokes solve.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `stokesmg` 0.1.0 (/root/reference/pkg/src/stokesmg).  The reference is pure
 * Python with duck-typed seams and no FFI; each entry point below replaces one
 * of those seams (file:line cited per function).  A maintainer binds it with
 * ctypes exactly as INTEGRATION.md shows; this package's own Python mirror
 * (paper_1308_4605_b200/_lib.py) is that binding.
 *
 * Conventions
 *  - fp64 everywhere.  Array arguments are the reference's C-order NumPy
 *    layouts: cells `cells`, face component a `GridSpec.face_shape(a)`
 *    (grid.py:84-89), node/edge arrays `node_edge_shape((a,b))` in the order
 *    of `edge_planes` (grid.py:229-233).  Pointers may be host or device
 *    (CUDA unified addressing decides); the library copies them into its own
 *    pitched device layout and back.
 *  - Wall-normal boundary faces are ignored on input and written as 0.
 *  - A context owns one CUDA stream and all device memory; it is not
 *    thread-safe.  Every call is stream-ordered and returns when its results
 *    are visible to the caller (host outputs are synchronised).
 *  - Return codes: SB_OK, SB_EINVAL (the reference raises ValueError),
 *    SB_EDOM (ZeroDivisionError: zero smoother diagonal), SB_ECUDA / SB_ENOMEM
 *    (runtime failure).  sb_last_error() gives the message of the last failure
 *    on the calling thread.
 */
#ifndef STOKESB200_H
#define STOKESB200_H

#ifdef __cplusplus
extern "C" {
#endif

#define SB_OK 0
#define SB_EINVAL 22
#define SB_EDOM 33
#define SB_ENOMEM 12
#define SB_ECUDA 99

/* grid.py:24-32 BoundaryCondition */
#define SB_BC_PERIODIC 0
#define SB_BC_NO_SLIP 1
#define SB_BC_FREE_SLIP 2

/* operators.py:29-37 ViscousForm */
#define SB_FORM_LAPLACIAN 0
#define SB_FORM_STRESS 1
#define SB_FORM_STRESS_BULK 2

/* precond.py:27-41 PrecondKind */
#define SB_P1 1
#define SB_P2 2
#define SB_P3 3
#define SB_P4 4
#define SB_P5 5
#define SB_IDENTITY 0

/* multigrid.py:391 vcycle kind */
#define SB_KIND_CELL 0
#define SB_KIND_FACE 1

/* gmres status (krylov.py:136-145) */
#define SB_STATUS_CONVERGED 0
#define SB_STATUS_BREAKDOWN 1
#define SB_STATUS_MAXITER 2

typedef struct sb_ctx sb_ctx;

/* multigrid.py:33-46 SmootherParams */
typedef struct {
  double omega;
  int sweeps_down;
  int sweeps_up;
  int bottom_sweeps;
} sb_smoother;

/* precond.py:44-53 PrecondConfig + schur.py:37-44 SchurConfig */
typedef struct {
  int kind;            /* SB_P1..SB_P5, SB_IDENTITY */
  int velocity_cycles; /* >= 1 */
  int schur_sign;      /* -1 (SchurSign.MINUS) or +1 (PLUS) */
  int pressure_cycles; /* >= 1 */
} sb_precond;

/* krylov.py:22-38 GmresConfig */
typedef struct {
  int restart;
  int max_iters;
  double rtol;
  double atol;
  int track_true_residual;
} sb_gmres;

/* krylov.py:40-47 HistoryEntry */
typedef struct {
  int iteration;
  long long scalar_vcycles;
  double resid_precond;
  double resid_true;
  int restart;
} sb_history_row;

/* Per-kernel-class device time of the last solve (CUDA events), for the
 * roofline report.  Filled only when profiling was enabled on the context. */
typedef struct {
  double smoother_face_ms;   /* face colour passes, all levels */
  double smoother_cell_ms;   /* cell colour passes, all levels */
  double smoother_face_bytes; /* algorithmic bytes of those passes */
  double smoother_cell_bytes;
  long long smoother_face_launches;
  long long smoother_cell_launches;
  double fine_face_ms;       /* finest-level face colour passes only */
  double fine_face_bytes;
  long long fine_face_launches;
} sb_kernel_stats;

/* Create a context for one grid (grid.py:40 GridSpec).
 *  dim 2|3, cells[dim], spacing h, bc[2*dim] = (lo, hi) per axis,
 *  viscous_form SB_FORM_*.  Returns NULL on failure (see sb_last_error). */
sb_ctx* sb_create(int dim, const int* cells, double h, const int* bc, int viscous_form);
void sb_destroy(sb_ctx* ctx);
const char* sb_last_error(void);

/* Upload a CoefficientSet (operators.py:45-78) and build the multigrid
 * hierarchy on the device: coarsen_coefficients per level
 * (multigrid.py:92-169), inverse face densities and zero-diagonal /
 * non-positive-density checks (multigrid.py:70-89, operators.py:209-210).
 * rho_face[dim], mu_edge[1 or 3] (edge_planes order), gamma_cell may be NULL. */
int sb_set_coefficients(sb_ctx* ctx, double theta, const double* const* rho_face,
                        const double* mu_cell, const double* const* mu_edge,
                        const double* gamma_cell);
/* Device-side make_coefficients (operators.py:107-125; averaging :81-104)
 * followed by rescale with factor `scale` (operators.py:532-550, applied as
 * cli.py:340-343 does; scale = 1 for none): only the cell arrays cross the
 * boundary, the face densities and node/edge viscosities are averaged on the
 * device, then as sb_set_coefficients.  Equal to the host path to the bit.
 * gamma_cell may be NULL. */
int sb_set_cell_coefficients(sb_ctx* ctx, double theta, const double* rho_cell, const double* mu_cell,
                             const double* gamma_cell, double scale);

/* operators.py:363-365 apply_M:  (A u + G p, -D u). */
int sb_apply_M(sb_ctx* ctx, const double* const* u, const double* p,
               double* const* out_u, double* out_p);

/* operators.py:348-360 apply_A on a face field.  Like the reference, the
 * wall-normal boundary faces of u (and of sb_apply_M's u) are read as given:
 * a boundary lift there enters the interior rows. */
int sb_apply_A(sb_ctx* ctx, const double* const* u, double* const* out_u);

/* operators.py:348-360 apply_A(u, coeff, bvals) with BoundaryValues
 * (operators.py:224-264): tangential[(axis*2 + side)*3 + comp] is the C-order
 * plane tangential_values(axis, side, comp) (comp's face array with `axis`
 * dropped; reference axis/comp numbering), NULL = zero.  The normal values
 * are the boundary faces of u (boundary_lift, operators.py:471). */
int sb_apply_A_affine(sb_ctx* ctx, const double* const* u, const double* const* tangential,
                      double* const* out_u);

/* operators.py:484-512 homogenize(bvals, coeff, rhs): out = (rhs.u - A(u_b; bvals),
 * rhs.p + div u_b), u_b = boundary_lift.  normal[axis*2 + side] is the plane
 * normal_values(axis, side) (cells with `axis` dropped), NULL = zero;
 * tangential as sb_apply_A_affine.  SB_EINVAL "incompatible boundary data: ..."
 * when the net boundary flux does not match the divergence source (:505). */
int sb_homogenize(sb_ctx* ctx, const double* const* normal, const double* const* tangential,
                  const double* const* rhs_u, const double* rhs_p, double* const* out_u, double* out_p);

/* operators.py:206-215 apply_Lrho on a cell field. */
int sb_apply_Lrho(sb_ctx* ctx, const double* p, double* out_p);

/* multigrid.py:442-460 mg_solve (n_cycles = 1 is multigrid.py:391 vcycle).
 * kind SB_KIND_CELL: rhs[0]/out[0] are cell arrays; SB_KIND_FACE: dim face arrays. */
int sb_mg_solve(sb_ctx* ctx, int kind, const sb_smoother* sm, int n_cycles,
                const double* const* rhs, double* const* out);

/* precond.py:111-156 Preconditioner.apply (incl. null projection :163-168).
 * *scalar_vcycles is advanced by the V-cycles spent (precond.py:94, :101). */
int sb_precond_apply(sb_ctx* ctx, const sb_precond* pc, const sb_smoother* sm,
                     const double* const* r_u, const double* r_p,
                     double* const* x_u, double* x_p, long long* scalar_vcycles);

/* krylov.py:164-214 gmres_solve on an already homogenised / rescaled rhs.
 * rows[max_rows] receives the ConvergenceHistory; *status SB_STATUS_*. */
int sb_gmres_solve(sb_ctx* ctx, const sb_precond* pc, const sb_gmres* gc,
                   const sb_smoother* sm, const double* const* b_u, const double* b_p,
                   double* const* x_u, double* x_p, sb_history_row* rows, int max_rows,
                   int* n_rows, int* status, long long* scalar_vcycles);

/* ---- introspection / component-level entry points (parity tests) ---- */

/* number of multigrid levels (multigrid.py:92-104) and the cells of one level */
int sb_num_levels(sb_ctx* ctx);
int sb_level_cells(sb_ctx* ctx, int level, int* cells);

/* Per-level operand specialisations chosen at sb_set_coefficients (bit mask;
 * -1 on a bad level).  Both are exact restatements of the uploaded arrays:
 *  SB_LEVEL_MUE_DERIVED: all-periodic level whose mu_edge equals the
 *    four-cell mean of mu_cell (operators.py:90-104) to 4e-15 relative; the
 *    face rows compute it instead of reading mu_edge (SB_MUE_DERIVED=0: off).
 *  SB_LEVEL_CONST_RHO: every non-wall rho_face of the level is the same value;
 *    the cell rows use its 1/rho instead of reading the 1/rho_face arrays
 *    (bit-identical; SB_CONST_BETA=0: off). */
#define SB_LEVEL_MUE_DERIVED 1
#define SB_LEVEL_CONST_RHO 2
int sb_level_flags(sb_ctx* ctx, int level);

/* download the coarsened coefficients of one level (multigrid.py:127-169) */
int sb_get_level_coefficients(sb_ctx* ctx, int level, double* const* rho_face,
                              double* mu_cell, double* const* mu_edge, double* gamma_cell);

/* one smoother sweep in place on a level (multigrid.py:318-340) */
int sb_smooth(sb_ctx* ctx, int kind, int level, double omega, double* const* x,
              const double* const* rhs);

/* residual -> restriction onto level+1 (multigrid.py:403-406 + :177-233) */
int sb_residual_restrict(sb_ctx* ctx, int kind, int level, const double* const* x,
                         const double* const* rhs, double* const* coarse);

/* fine (level) += prolong(coarse (level+1)) (multigrid.py:185-192, :282-295, :431-436) */
int sb_prolong_add(sb_ctx* ctx, int kind, int level, const double* const* coarse,
                   double* const* fine);

/* ---- the reference's remaining public operators (geometry only unless noted;
 * a context needs no coefficients for these) ---- */
/* div(u) -> cell, reading the stored boundary faces (operators.py:182-188) */
int sb_div(sb_ctx* ctx, const double* const* u, double* out);
/* grad(p) -> faces, wall-normal faces 0 (operators.py:191-198) */
int sb_grad(sb_ctx* ctx, const double* p, double* const* out);
/* lap_pressure(p) = div(grad(p)) (operators.py:201-203) */
int sb_lap_pressure(sb_ctx* ctx, const double* p, double* out);
/* pure restriction level -> level+1 (multigrid.py:177-182, :214-233) */
int sb_restrict(sb_ctx* ctx, int kind, int level, const double* const* fine, double* const* coarse);
/* pure prolongation level+1 -> level (multigrid.py:185-192, :282-295) */
int sb_prolong(sb_ctx* ctx, int kind, int level, const double* const* coarse, double* const* fine);
/* needs coefficients: the smoother diagonal of a level as arrays
 * (helmholtz_diagonal / lrho_diagonal, operators.py:396-439; wall-normal
 * boundary faces 1) */
int sb_diagonal(sb_ctx* ctx, int kind, int level, double* const* out);
/* needs coefficients: S~^-1 r = -theta phi + V r with phi the caller's Poisson
 * solve of r, or V r when phi is NULL (apply_schur_inv, schur.py:59-78) */
int sb_schur_inv(sb_ctx* ctx, const double* r, const double* phi, double* out);

/* ---- restarted GMRES on flat vectors with a caller-supplied operator: the
 * reference's gmres_kernel(apply_op, b, restart, max_iters, target,
 * breakdown_tol, callback) seam (krylov.py:81-146).  Host arrays of length n;
 * the basis and orthogonalisation live on the device, apply(in, out, user)
 * computes out = op(in) on host arrays, callback(k, x_k, r_P, restart_flag,
 * user) (nullable) sees every iterate.  status: SB_STATUS_*; iterations = k. */
typedef void (*sb_apply_fn)(const double* in, double* out, void* user);
typedef void (*sb_iter_fn)(int k, const double* x, double resid_precond, int restart_flag, void* user);
int sb_gmres_flat(long long n, const double* b, int restart, int max_iters, double target, double breakdown_tol,
                  sb_apply_fn apply, sb_iter_fn callback, void* user, double* x_out, int* status, int* iterations);

/* ---- measurement ---- */
void sb_set_profiling(sb_ctx* ctx, int enabled);
int sb_get_kernel_stats(sb_ctx* ctx, sb_kernel_stats* out);
/* kernels launched by this context since creation (graph nodes counted per replay) */
long long sb_launch_count(sb_ctx* ctx);
/* enable / disable CUDA-graph replay of the preconditioner (default on) */
void sb_set_graphs(sb_ctx* ctx, int enabled);
/* device bytes currently allocated by the context */
long long sb_device_bytes(sb_ctx* ctx);
/* run the context's work on a caller-owned CUDA stream (cudaStream_t; NULL
 * restores the context's own stream), e.g. torch's current stream so that
 * CUDA events recorded there bracket the solve */
int sb_set_stream(sb_ctx* ctx, void* stream);

/* page-locked host buffers (the Python API recycles them for returned arrays) */
void* sb_host_alloc(long long bytes);
void sb_host_free(void* ptr);

/* ---- slab-decomposed multi-GPU solve ----------
 * The global 3D grid is cut along axis 0 (must be periodic) into
 * nranks x nslab slabs; a process owns nslab consecutive slabs.  nranks > 1:
 * one slab per process, one GPU per process, NCCL halo exchange / allreduce /
 * allgather (communicator from sb_nccl_unique_id on rank 0, broadcast by the
 * caller).  nranks == 1 with nslab > 1 runs the same decomposition on one GPU
 * (exchanges are device copies).  nranks == 1, nslab == 1 with a non-NULL
 * nccl_id creates a 1-rank communicator: every exchange / reduction / gather
 * takes the NCCL branch (self send/recv), i.e. exactly the code each rank runs
 * at N > 1.  nranks > 1 with nccl_id == NULL is SB_EINVAL.
 * Array arguments hold THIS RANK's planes [rank*n0r, (rank+1)*n0r) of the
 * reference layouts (n0r = N0 / nranks).  Replaces the same seams as
 * sb_set_coefficients / sb_apply_M / sb_precond_apply / sb_gmres_solve
 * (operators.py:107, :363; precond.py:111; krylov.py:164). */
typedef struct sb_dist sb_dist;
int sb_nccl_id_bytes(void);
int sb_nccl_unique_id(unsigned char* out);
sb_dist* sb_dist_create(const int* cells, double h, const int* bc, int viscous_form, int nranks, int rank,
                        int nslab, const unsigned char* nccl_id);
void sb_dist_destroy(sb_dist* dist);
/* the CUDA stream the distributed context launches on (cudaStream_t) */
void* sb_dist_stream(sb_dist* dist);
/* order the context after the caller's stream on entry to every public call
 * (set_coefficients / apply_M / precond_apply / gmres_solve) and the caller's
 * stream after the context on exit; NULL = no join (the default) */
void sb_dist_set_stream(sb_dist* dist, void* stream);
/* 1 when the context routes its exchanges through an NCCL communicator */
int sb_dist_uses_nccl(sb_dist* dist);
/* measurement: CUDA events around every slab colour pass of the next solves
 * (eager launches while enabled; sb_kernel_stats as for sb_ctx), and the
 * kernels launched by this context (graph nodes counted per replay) */
void sb_dist_set_profiling(sb_dist* dist, int enabled);
int sb_dist_get_kernel_stats(sb_dist* dist, sb_kernel_stats* out);
long long sb_dist_launch_count(sb_dist* dist);
/* out[6] = {distributed levels, agglomerated levels, planes per slab, slabs in this process,
 *          bit l: distributed level l derives mu_e from mu_c, bit l: level l has constant 1/rho} */
int sb_dist_info(sb_dist* dist, int* out);
int sb_dist_set_coefficients(sb_dist* dist, double theta, const double* const* rho_face, const double* mu_cell,
                             const double* const* mu_edge, const double* gamma_cell);
int sb_dist_apply_M(sb_dist* dist, const double* const* u, const double* p, double* const* out_u, double* out_p);
int sb_dist_precond_apply(sb_dist* dist, const sb_precond* pc, const sb_smoother* sm, const double* const* r_u,
                          const double* r_p, double* const* x_u, double* x_p);
int sb_dist_gmres_solve(sb_dist* dist, const sb_precond* pc, const sb_gmres* gc, const sb_smoother* sm,
                        const double* const* b_u, const double* b_p, double* const* x_u, double* x_p,
                        sb_history_row* rows, int max_rows, int* n_rows, int* status, long long* scalar_vcycles);

#ifdef __cplusplus
}
#endif
#endif /* STOKESB200_H */
