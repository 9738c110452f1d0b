// sb_solver.cu -- host orchestration and the C ABI (include/stokesb200.h).
//
// One sb_ctx per grid: it owns a CUDA stream, the device multigrid hierarchy
// (coefficients per level, work buffers), the level-0 Krylov / preconditioner
// vectors and the GMRES basis.  The preconditioner application P^{-1}
// (two V-cycles plus glue, ~30 launches per level) is captured once into a
// CUDA graph and replayed every GMRES iteration; the Arnoldi step is three
// fused multi-vector kernels (CGS2) with one host sync per iteration for the
// Hessenberg column.
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <stdexcept>
#include <utility>
#include "../../include/stokesb200.h"
#include "sb_kernels.h"

namespace sb {
extern long long g_kernel_launches;
}

using namespace sb;

namespace {

thread_local std::string g_err;

struct CudaErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ArgErr : std::runtime_error {
  int code;
  ArgErr(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess)                                                          \
      throw CudaErr(std::string(#x) + ": " + cudaGetErrorString(e_));               \
  } while (0)

constexpr int kMaxVec = 128;
constexpr int kMaxLevels = 24;
constexpr int kFlagInts = 16 + 2 * kMaxLevels;
// GMRES: ||w'||^2 below this fraction of ||w||^2 (or ||c'||^2 > ||w'||^2 / 2)
// finishes the Arnoldi step explicitly (direct second pass, sb_solver.cu gmres)
constexpr double kDirectRel = 1e-10;
// one-pass Arnoldi: gam_{j+1}^2 below this fraction of ||w||^2 finishes the
// step explicitly (the implicit norm then carries < ~1e-10 relative error)
constexpr double kOnePassRel = 1e-6;  // dflags: 16 setup-check slots + mu_e / constant-rho flags per level

struct Level {
  LevelDev d{};
  int P[3]{};
  long long block = 0;
  bool two_phase = false;
  double *mu_c = nullptr, *gam_c = nullptr, *mu_e[3]{}, *rho_f[3]{}, *beta_f[3]{};
  double *fx[3]{}, *frhs[3]{}, *cx = nullptr, *crhs = nullptr, *tmp = nullptr;
  bool split_rr = false;                      // residual to memory, then restrict (large levels)
  double *fres[3]{}, *cres = nullptr;
};

struct ProfEv {
  cudaEvent_t a, b;
  int cls;       // 0 face, 1 cell
  bool fine;
  double bytes;
};

}  // namespace

struct sb_ctx {
  int dim = 3, form = 1, off = 0;
  int n[3]{};         // internal cells
  int bc[3][2]{};     // internal bcs
  double h = 1.0;
  cudaStream_t st = nullptr;
  cudaStream_t own_st = nullptr;
  std::vector<Level> lv;
  std::vector<void*> allocs;
  long long bytes = 0;
  bool have_coef = false;
  double theta = 0.0;
  int flag_rho = 0, flag_face = 0, flag_cell = 0;
  std::vector<int> null_comps;  // internal axes
  // null-space projection deferred from P^-1 into the Arnoldi pass B (pad-free
  // all-periodic level 0 only: the pass subtracts per-block means from every
  // element of a block, pads included)
  bool defer_nulls = false;
  double* cscratch = nullptr;  // cell-layout scratch (sb_set_cell_coefficients: rho_cell)
  int* dflags = nullptr;
  double* dpart = nullptr;
  double* dsmall = nullptr;   // [h1 kMaxVec][h2 kMaxVec][misc 64][y kMaxVec]
  double* hsmall = nullptr;   // pinned mirror
  double* dbig = nullptr;     // restart >= kMaxVec: [h1 M][h2 M][y M]
  double* hbig = nullptr;     // pinned mirror
  int bigcap = 0;
  long long vlen = 0;         // vector length (nblk * block)
  double *vb = nullptr, *vz0 = nullptr, *vx = nullptr, *vw = nullptr, *vMv = nullptr, *vt = nullptr;
  double* basis = nullptr;
  int basis_cap = 0;
  double *sc0 = nullptr, *sc1 = nullptr, *scR = nullptr, *scC = nullptr;
  double *sf0[3]{}, *sf1[3]{}, *sfR[3]{}, *sfC[3]{};
  double* splane = nullptr;   // staging for one wall plane of BoundaryValues
  // one-CTA coarse tail of the V-cycles (levels >= coarse_ls; -1 = off)
  int coarse_ls = -1;
  CoarseChain* dchain_face = nullptr;
  CoarseChain* dchain_cell = nullptr;
  bool scratch = false, scratch_mg = false;
  // graph cache
  cudaGraphExec_t gexec = nullptr;
  long long gnodes = 0;
  sb_precond gpc{};
  sb_smoother gsm{};
  bool use_graphs = true;
  bool profiling = false;
  std::vector<ProfEv> prof;
  std::vector<cudaEvent_t> evpool;
  size_t evnext = 0;
  long long launches_base = 0;  // g_kernel_launches at creation
  long long direct_norms = 0;   // GMRES steps that took the direct subdiagonal norm (near breakdown)
  long long graph_launches = 0; // kernel nodes replayed through graphs
  sb_kernel_stats stats{};
};

namespace {

double* dalloc(sb_ctx* c, long long n) {
  void* p = nullptr;
  if (n < 1) n = 1;
  cudaError_t e = cudaMalloc(&p, (size_t)n * sizeof(double));
  if (e != cudaSuccess) throw ArgErr(SB_ENOMEM, std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
  CK(cudaMemsetAsync(p, 0, (size_t)n * sizeof(double), c->st));
  c->allocs.push_back(p);
  c->bytes += n * (long long)sizeof(double);
  return (double*)p;
}

bool can_coarsen(const int* n, int dim) {
  for (int a = 3 - dim; a < 3; ++a)
    if (n[a] < 4 || (n[a] & 1)) return false;
  return true;
}

void make_level(sb_ctx* c, const int* n, double h) {
  Level L;
  for (int a = 0; a < 3; ++a) {
    L.d.n[a] = n[a];
    L.d.bclo[a] = c->bc[a][0];
    L.d.bchi[a] = c->bc[a][1];
    L.P[a] = n[a] + (c->bc[a][0] != BC_PER ? 1 : 0);
  }
  L.P[2] = (L.P[2] + 3) / 4 * 4;
  L.d.s1 = L.P[2];
  L.d.s0 = (long long)L.P[1] * L.P[2];
  L.block = (long long)L.P[0] * L.P[1] * L.P[2];
  L.d.h = h;
  L.d.inv_h = 1.0 / h;
  L.d.inv_h2 = 1.0 / (h * h);
  L.d.theta = 0.0;
  L.two_phase = level_needs_two_phase(L.d, c->dim);
  // split residual / restriction on levels with >= SB_RR_SPLIT cells (default
  // 64^3; 0 = always fused): full-occupancy residual kernel + light restriction
  const long long split_min = [] {
    const char* e = std::getenv("SB_RR_SPLIT");
    return e ? std::atoll(e) : 262144LL;
  }();
  {
    long long cells = 1;
    for (int a = 3 - c->dim; a < 3; ++a) cells *= n[a];
    L.split_rr = split_min > 0 && cells >= split_min && can_coarsen(n, c->dim);
  }
  c->lv.push_back(L);
}

void alloc_level(sb_ctx* c, Level& L, bool first) {
  const long long B = L.block;
  L.mu_c = dalloc(c, B);
  L.gam_c = dalloc(c, B);
  for (int a = 3 - c->dim; a < 3; ++a) {
    L.rho_f[a] = dalloc(c, B);
    L.beta_f[a] = dalloc(c, B);
  }
  if (c->dim == 3) {
    for (int e = 0; e < 3; ++e) L.mu_e[e] = dalloc(c, B);
  } else {
    L.mu_e[0] = dalloc(c, B);
  }
  if (!first) {
    for (int a = 3 - c->dim; a < 3; ++a) {
      L.fx[a] = dalloc(c, B);
      L.frhs[a] = dalloc(c, B);
    }
    L.cx = dalloc(c, B);
    L.crhs = dalloc(c, B);
  }
  if (L.two_phase) L.tmp = dalloc(c, B);
  if (L.split_rr) {
    for (int a = 3 - c->dim; a < 3; ++a) L.fres[a] = dalloc(c, B);
    L.cres = dalloc(c, B);
  }
  L.d.mu_c = L.mu_c;
  L.d.gam_c = L.gam_c;
  for (int a = 0; a < 3; ++a) {
    L.d.mu_e[a] = L.mu_e[a];
    L.d.rho_f[a] = L.rho_f[a];
    L.d.beta_f[a] = L.beta_f[a];
  }
}

// extents (internal axes) of an array kind: -1 cell, A face A, 10+e edge e
void extents(const sb_ctx* c, const Level& L, int kind, int* ext) {
  for (int a = 0; a < 3; ++a) ext[a] = L.d.n[a];
  auto wall = [&](int a) { return c->bc[a][0] != BC_PER; };
  if (kind >= 0 && kind < 3) {
    if (wall(kind)) ext[kind] += 1;
  } else if (kind >= 10) {
    const int e = kind - 10;
    for (int a = 3 - c->dim; a < 3; ++a)
      if (a != e && wall(a)) ext[a] += 1;
  }
}

// a reference array whose rows fill the box exactly (no pads along axes 1, 2)
// moves as one linear copy; otherwise a pitched 3D copy
bool dense_rows(const Level& L, const int* ext) { return ext[2] == L.P[2] && ext[1] == L.P[1]; }

void copy_in(sb_ctx* c, const Level& L, int kind, const double* src, double* dst) {
  int ext[3];
  extents(c, L, kind, ext);
  if (dense_rows(L, ext)) {
    CK(cudaMemcpyAsync(dst, src, (size_t)ext[0] * ext[1] * ext[2] * 8, cudaMemcpyDefault, c->st));
    return;
  }
  cudaMemcpy3DParms p;
  std::memset(&p, 0, sizeof(p));
  p.srcPtr = make_cudaPitchedPtr((void*)src, (size_t)ext[2] * 8, (size_t)ext[2], (size_t)ext[1]);
  p.dstPtr = make_cudaPitchedPtr((void*)dst, (size_t)L.P[2] * 8, (size_t)L.P[2], (size_t)L.P[1]);
  p.extent = make_cudaExtent((size_t)ext[2] * 8, (size_t)ext[1], (size_t)ext[0]);
  p.kind = cudaMemcpyDefault;
  CK(cudaMemcpy3DAsync(&p, c->st));
}

void copy_out(sb_ctx* c, const Level& L, int kind, const double* src, double* dst) {
  int ext[3];
  extents(c, L, kind, ext);
  if (dense_rows(L, ext)) {
    CK(cudaMemcpyAsync(dst, src, (size_t)ext[0] * ext[1] * ext[2] * 8, cudaMemcpyDefault, c->st));
    return;
  }
  cudaMemcpy3DParms p;
  std::memset(&p, 0, sizeof(p));
  p.srcPtr = make_cudaPitchedPtr((void*)src, (size_t)L.P[2] * 8, (size_t)L.P[2], (size_t)L.P[1]);
  p.dstPtr = make_cudaPitchedPtr((void*)dst, (size_t)ext[2] * 8, (size_t)ext[2], (size_t)ext[1]);
  p.extent = make_cudaExtent((size_t)ext[2] * 8, (size_t)ext[1], (size_t)ext[0]);
  p.kind = cudaMemcpyDefault;
  CK(cudaMemcpy3DAsync(&p, c->st));
}

// zero the wall-normal boundary faces of a face array (they are not unknowns)
void zero_wall_faces(sb_ctx* c, const Level& L, int A, double* x) {
  if (c->bc[A][0] == BC_PER) return;
  Box b;
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = 0;
    b.hi[a] = L.d.n[a] - 1;
  }
  b.lo[A] = b.hi[A] = 0;
  launch_box_fill(c->st, L.d, b, x, 0.0);
  b.lo[A] = b.hi[A] = L.d.n[A];
  launch_box_fill(c->st, L.d, b, x, 0.0);
}

// one plane (index j along axis B) of an array kind, from a C-order plane
// holding the kind's extents with axis B dropped (BoundaryValues layouts)
void copy_plane_in(sb_ctx* c, const Level& L, int kind, int B, int j, const double* src, double* dst) {
  int ext[3];
  extents(c, L, kind, ext);
  ext[B] = 1;
  const long long st = B == 0 ? (long long)L.d.s0 : (B == 1 ? (long long)L.d.s1 : 1LL);
  cudaMemcpy3DParms p;
  std::memset(&p, 0, sizeof(p));
  p.srcPtr = make_cudaPitchedPtr((void*)src, (size_t)ext[2] * 8, (size_t)ext[2], (size_t)ext[1]);
  p.dstPtr = make_cudaPitchedPtr((void*)(dst + j * st), (size_t)L.P[2] * 8, (size_t)L.P[2], (size_t)L.P[1]);
  p.extent = make_cudaExtent((size_t)ext[2] * 8, (size_t)ext[1], (size_t)ext[0]);
  p.kind = cudaMemcpyDefault;
  CK(cudaMemcpy3DAsync(&p, c->st));
}

// tangential wall velocities of BoundaryValues (operators.py:267-291):
// tangential[(axis*2 + side)*3 + comp] in reference axes, NULL = zero
void wall_tangent(sb_ctx* c, const double* const* tangential, double* const* out) {
  const Level& L = c->lv[0];
  if (!c->splane) c->splane = dalloc(c, L.block);
  for (int rb = 0; rb < c->dim; ++rb) {
    const int B = rb + c->off;
    for (int side = 0; side < 2; ++side) {
      if (c->bc[B][side] != BC_NOSLIP) continue;  // periodic: none; free slip: flux zeroed
      for (int ra = 0; ra < c->dim; ++ra) {
        const double* src = ra == rb ? nullptr : tangential[(rb * 2 + side) * 3 + ra];
        if (!src) continue;
        const int A = ra + c->off;
        int ext[3];
        extents(c, L, A, ext);
        ext[B] = 1;
        CK(cudaMemcpyAsync(c->splane, src, (size_t)ext[0] * ext[1] * ext[2] * 8, cudaMemcpyDefault, c->st));
        launch_wall_tangent(c->st, L.d, A, B, side, c->splane, out[A]);
      }
    }
  }
}

void sync(sb_ctx* c) {
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->st));
}

void ensure_scratch(sb_ctx* c) {
  if (c->scratch) return;
  const long long B = c->lv[0].block;
  c->sc0 = dalloc(c, B);
  c->sc1 = dalloc(c, B);
  for (int a = 3 - c->dim; a < 3; ++a) {
    c->sf0[a] = dalloc(c, B);
    c->sf1[a] = dalloc(c, B);
  }
  c->scratch = true;
}
void ensure_scratch_mg(sb_ctx* c) {
  if (c->scratch_mg) return;
  const long long B = c->lv[0].block;
  c->scR = dalloc(c, B);
  c->scC = dalloc(c, B);
  for (int a = 3 - c->dim; a < 3; ++a) {
    c->sfR[a] = dalloc(c, B);
    c->sfC[a] = dalloc(c, B);
  }
  c->scratch_mg = true;
}
void ensure_vectors(sb_ctx* c) {
  if (c->vb) return;
  c->vlen = (long long)(c->dim + 1) * c->lv[0].block;
  c->vb = dalloc(c, c->vlen);
  c->vz0 = dalloc(c, c->vlen);
  c->vx = dalloc(c, c->vlen);
  c->vw = dalloc(c, c->vlen);
  c->vMv = dalloc(c, c->vlen);
  c->vt = dalloc(c, c->vlen);
}

// vector block pointers (reference component r -> internal axis r + off)
double* vcomp(sb_ctx* c, double* v, int A) { return v + (long long)(A - c->off) * c->lv[0].block; }
double* vpres(sb_ctx* c, double* v) { return v + (long long)c->dim * c->lv[0].block; }

void check_ready(sb_ctx* c) {
  if (!c->have_coef) throw ArgErr(SB_EINVAL, "coefficients not set (call sb_set_coefficients)");
}
void check_mg(sb_ctx* c, int kind, bool need_levels = true) {
  check_ready(c);
  if (need_levels && c->lv.size() < 2) throw ArgErr(SB_EINVAL, "grid cannot be coarsened; need even counts >= 4");
  if (kind == SB_KIND_CELL) {
    if (c->flag_rho) throw ArgErr(SB_EINVAL, "face density must be positive");
    if (c->flag_cell) throw ArgErr(SB_EDOM, "zero diagonal in pressure operator");
  } else if (c->flag_face) {
    throw ArgErr(SB_EDOM, "zero diagonal in velocity operator (theta = 0 with mu = 0 row)");
  }
}

// ---- profiling ---------------------------------------------------------------

cudaEvent_t next_event(sb_ctx* c) {
  if (c->evnext == c->evpool.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    c->evpool.push_back(e);
  }
  return c->evpool[c->evnext++];
}

double face_pass_bytes(const sb_ctx* c, const Level& L) {
  double per;
  if (c->dim == 3) per = c->form == F_LAP ? 40.0 : 56.0;
  else per = c->form == F_LAP ? 32.0 : 40.0;
  if (c->form == F_BULK) per += 8.0;
  if (c->theta > 0) per += 4.0;
  return per * (double)L.d.n[0] * L.d.n[1] * L.d.n[2];
}
double cell_pass_bytes(const sb_ctx* c, const Level& L) {
  // phi + 1/2 rhs + 1/2 write, plus the d arrays of 1/rho_face -- which a
  // constant-density level does not stream (LevelDev::beta_const), so they are
  // not credited there
  const double per = 16.0 + (L.d.beta_const ? 0.0 : 8.0 * c->dim);
  return per * (double)L.d.n[0] * L.d.n[1] * L.d.n[2];
}

// ---- multigrid ---------------------------------------------------------------

// One smoother sweep on level l, in place on cur[].
// zs (first sweep of a V-cycle level, x = 0 on entry): 0 plain, 1 the level
// was zero-filled, 2 the level was not (zero_fill_free: the first colour pass
// stores both colours).  Only the per-colour kernels take the zero variants.
void sweep_face(sb_ctx* c, int l, double** cur, const double* const* rhs, double omega, int zs = 0) {
  Level& L = c->lv[l];
  for (int A = 3 - c->dim; A < 3; ++A) {
    for (int parity = 0; parity < 2; ++parity) {
      cudaEvent_t ea = nullptr;
      if (c->profiling) {
        ea = next_event(c);
        CK(cudaEventRecord(ea, c->st));
      }
      int z = 0;
      Ptr3 u{{cur[0], cur[1], cur[2]}};
      if (L.two_phase) {
        launch_face_colour_tmp(c->st, L.d, c->dim, c->form, A, u, rhs[A], L.tmp, parity, omega);
      } else {
        z = zs == 0 ? 0 : (parity == 0 ? (zs == 2 ? 3 : 2) : 1);
        launch_face_colour(c->st, L.d, c->dim, c->form, A, u, rhs[A], parity, omega, z);
      }
      if (c->profiling) {
        cudaEvent_t eb = next_event(c);
        CK(cudaEventRecord(eb, c->st));
        // zero-aware passes: 8 B less per skipped component, the partner store
        // of z = 3 adds 4 B; the roofline (fine) average takes plain passes only
        double bytes = face_pass_bytes(c, L);
        if (z != 0) {
          int nz = 0;
          for (int B = 3 - c->dim; B < 3; ++B) nz += (B > A || (B == A && z >= 2)) ? 1 : 0;
          bytes -= (8.0 * nz - (z == 3 ? 4.0 : 0.0)) * (double)L.d.n[0] * L.d.n[1] * L.d.n[2];
        }
        c->prof.push_back({ea, eb, 0, l == 0 && z == 0, bytes});
      }
    }
  }
}

void sweep_cell(sb_ctx* c, int l, double*& cur, const double* rhs, double omega, int zs = 0) {
  Level& L = c->lv[l];
  for (int parity = 0; parity < 2; ++parity) {
    cudaEvent_t ea = nullptr;
    if (c->profiling) {
      ea = next_event(c);
      CK(cudaEventRecord(ea, c->st));
    }
    int z = 0;
    if (L.two_phase) {
      launch_cell_colour_tmp(c->st, L.d, c->dim, cur, rhs, L.tmp, parity, omega);
    } else {
      z = (zs == 0 || parity == 1) ? 0 : (zs == 2 ? 3 : 2);
      launch_cell_colour(c->st, L.d, c->dim, cur, rhs, parity, omega, z);
    }
    if (c->profiling) {
      cudaEvent_t eb = next_event(c);
      CK(cudaEventRecord(eb, c->st));
      const double pts = (double)L.d.n[0] * L.d.n[1] * L.d.n[2];
      const double bytes = cell_pass_bytes(c, L) - (z == 0 ? 0.0 : (z == 3 ? 4.0 : 8.0) * pts);
      c->prof.push_back({ea, eb, 1, l == 0, bytes});
    }
  }
}

// multigrid.py:409-439 -- x is written (zero initial guess)
double chain_face_bytes(sb_ctx* c, const sb_smoother& sm) {
  double b = 0;
  const int last = (int)c->lv.size() - 1;
  for (int l = c->coarse_ls; l <= last; ++l) {
    const int sw = l == last ? sm.bottom_sweeps : sm.sweeps_down + sm.sweeps_up;
    b += 2.0 * c->dim * sw * face_pass_bytes(c, c->lv[l]);
  }
  return b;
}
double chain_cell_bytes(sb_ctx* c, const sb_smoother& sm) {
  double b = 0;
  const int last = (int)c->lv.size() - 1;
  for (int l = c->coarse_ls; l <= last; ++l) {
    const int sw = l == last ? sm.bottom_sweeps : sm.sweeps_down + sm.sweeps_up;
    b += 2.0 * sw * cell_pass_bytes(c, c->lv[l]);
  }
  return b;
}

// the coarse tail in one launch when level l is the chain's top level and the
// buffers are the level's own (the V-cycle recursion's)
bool coarse_tail(sb_ctx* c, int l, int kind, const double* const* rhs, double* const* x, const sb_smoother& sm) {
  if (l != c->coarse_ls || l <= 0) return false;
  Level& L = c->lv[l];
  if (kind == SB_KIND_FACE) {
    for (int A = 3 - c->dim; A < 3; ++A)
      if (rhs[A] != L.frhs[A] || x[A] != L.fx[A]) return false;
  } else if (rhs[0] != L.crhs || x[0] != L.cx) {
    return false;
  }
  cudaEvent_t ea = nullptr;
  if (c->profiling) {
    ea = next_event(c);
    CK(cudaEventRecord(ea, c->st));
  }
  bool pa = true;
  for (int a = 0; a < 3; ++a) pa = pa && c->bc[a][0] == BC_PER;
  if (kind == SB_KIND_FACE)
    launch_coarse_face(c->st, c->dim, c->form, pa, c->dchain_face, sm.sweeps_down, sm.sweeps_up, sm.bottom_sweeps,
                       sm.omega);
  else
    launch_coarse_cell(c->st, c->dim, pa, c->dchain_cell, sm.sweeps_down, sm.sweeps_up, sm.bottom_sweeps, sm.omega);
  if (c->profiling) {
    cudaEvent_t eb = next_event(c);
    CK(cudaEventRecord(eb, c->st));
    c->prof.push_back({ea, eb, kind == SB_KIND_FACE ? 0 : 1, false,
                       kind == SB_KIND_FACE ? chain_face_bytes(c, sm) : chain_cell_bytes(c, sm)});
  }
  return true;
}

// How the first sweep of a V-cycle level treats its x = 0 start: 0 plain
// passes after the zero fill (row-vector / two-phase
// levels, SB_ZERO_FIRST=0), 1 zero-aware passes after the zero fill, 2
// zero-aware passes without it -- all-periodic levels whose block has no pads
// or ghosts, where the first colour pass stores every entry (bulk-form face
// rows read the divergence of all components, so they keep the fill).
static bool zero_first_on() {  // read per call: tests compare both paths in one process
  const char* e = std::getenv("SB_ZERO_FIRST");
  return !(e && e[0] == '0');
}
int first_sweep_mode(sb_ctx* c, const Level& L, int kind) {
  if (!zero_first_on() || L.two_phase) return 0;
  if (kind == SB_KIND_FACE && rowv_colour_supported(L.d, c->dim, c->form)) return 0;
  bool pa = L.d.dist0 == 0 && (L.d.n[2] % 4) == 0;
  for (int a = 3 - c->dim; a < 3; ++a) pa = pa && c->bc[a][0] == BC_PER && L.P[a] == L.d.n[a];
  if (kind == SB_KIND_FACE && c->form == F_BULK) pa = false;
  return pa ? 2 : 1;
}

void vcycle_face(sb_ctx* c, int l, const double* const* rhs, double* const* x, const sb_smoother& sm) {
  if (coarse_tail(c, l, SB_KIND_FACE, rhs, x, sm)) return;
  Level& L = c->lv[l];
  double* cur[3] = {x[0], x[1], x[2]};
  const int zs = first_sweep_mode(c, L, SB_KIND_FACE);
  if (zs != 2)
    for (int A = 3 - c->dim; A < 3; ++A) CK(cudaMemsetAsync(cur[A], 0, L.block * 8, c->st));
  const int last = (int)c->lv.size() - 1;
  if (l == last) {
    for (int s = 0; s < sm.bottom_sweeps; ++s) sweep_face(c, l, cur, rhs, sm.omega, s == 0 ? zs : 0);
  } else {
    for (int s = 0; s < sm.sweeps_down; ++s) sweep_face(c, l, cur, rhs, sm.omega, s == 0 ? zs : 0);
    Level& Lc = c->lv[l + 1];
    CPtr3 xc{{cur[0], cur[1], cur[2]}};
    if (L.split_rr) {
      CPtr3 rr{{rhs[0], rhs[1], rhs[2]}};
      Ptr3 res{{L.fres[0], L.fres[1], L.fres[2]}};
      launch_face_res3(c->st, L.d, c->dim, c->form, xc, rr, res);
      for (int A = 3 - c->dim; A < 3; ++A) launch_face_restrict(c->st, L.d, Lc.d, c->dim, A, L.fres[A], Lc.frhs[A]);
    } else {
      for (int A = 3 - c->dim; A < 3; ++A)
        launch_face_resid_restrict(c->st, L.d, Lc.d, c->dim, c->form, A, xc, rhs[A], Lc.frhs[A]);
    }
    vcycle_face(c, l + 1, Lc.frhs, Lc.fx, sm);
    for (int A = 3 - c->dim; A < 3; ++A)
      launch_face_prolong_add(c->st, L.d, Lc.d, c->dim, A, Lc.fx[A], cur[A]);
    for (int s = 0; s < sm.sweeps_up; ++s) sweep_face(c, l, cur, rhs, sm.omega);
  }
}

void vcycle_cell(sb_ctx* c, int l, const double* rhs, double* x, const sb_smoother& sm) {
  {
    const double* r3[3] = {rhs, nullptr, nullptr};
    double* x3[3] = {x, nullptr, nullptr};
    if (coarse_tail(c, l, SB_KIND_CELL, r3, x3, sm)) return;
  }
  Level& L = c->lv[l];
  double* cur = x;
  const int zs = first_sweep_mode(c, L, SB_KIND_CELL);
  if (zs != 2) CK(cudaMemsetAsync(cur, 0, L.block * 8, c->st));
  const int last = (int)c->lv.size() - 1;
  if (l == last) {
    for (int s = 0; s < sm.bottom_sweeps; ++s) sweep_cell(c, l, cur, rhs, sm.omega, s == 0 ? zs : 0);
  } else {
    for (int s = 0; s < sm.sweeps_down; ++s) sweep_cell(c, l, cur, rhs, sm.omega, s == 0 ? zs : 0);
    Level& Lc = c->lv[l + 1];
    if (L.split_rr) {
      launch_cell_res(c->st, L.d, c->dim, cur, rhs, L.cres);
      launch_cell_restrict(c->st, L.d, Lc.d, c->dim, L.cres, Lc.crhs);
    } else {
      launch_cell_resid_restrict(c->st, L.d, Lc.d, c->dim, cur, rhs, Lc.crhs);
    }
    vcycle_cell(c, l + 1, Lc.crhs, Lc.cx, sm);
    launch_cell_prolong_add(c->st, L.d, Lc.d, c->dim, Lc.cx, cur);
    for (int s = 0; s < sm.sweeps_up; ++s) sweep_cell(c, l, cur, rhs, sm.omega);
  }
}

// multigrid.py:442-460 on level-0 device buffers
void mg_face(sb_ctx* c, int ncyc, const double* const* rhs, double* const* out, const sb_smoother& sm) {
  vcycle_face(c, 0, rhs, out, sm);
  if (ncyc <= 1) return;
  ensure_scratch_mg(c);
  const Level& L = c->lv[0];
  Box fb;
  for (int k = 1; k < ncyc; ++k) {
    CPtr3 xo{{out[0], out[1], out[2]}}, rr{{rhs[0], rhs[1], rhs[2]}};
    Ptr3 R{{c->sfR[0], c->sfR[1], c->sfR[2]}};
    launch_face_residual(c->st, L.d, c->dim, c->form, xo, rr, nullptr, R);
    vcycle_face(c, 0, c->sfR, c->sfC, sm);
    for (int A = 3 - c->dim; A < 3; ++A) {
      for (int a = 0; a < 3; ++a) {
        fb.lo[a] = 0;
        fb.hi[a] = L.d.n[a] - 1 + ((a == A && c->bc[A][0] != BC_PER) ? 1 : 0);
      }
      launch_axpy_box(c->st, L.d, fb, out[A], c->sfC[A]);
    }
  }
}

void mg_cell(sb_ctx* c, int ncyc, const double* rhs, double* out, const sb_smoother& sm) {
  vcycle_cell(c, 0, rhs, out, sm);
  if (ncyc <= 1) return;
  ensure_scratch_mg(c);
  const Level& L = c->lv[0];
  Box cb;
  for (int a = 0; a < 3; ++a) {
    cb.lo[a] = 0;
    cb.hi[a] = L.d.n[a] - 1;
  }
  for (int k = 1; k < ncyc; ++k) {
    launch_cell_residual(c->st, L.d, c->dim, out, rhs, c->scR);
    vcycle_cell(c, 0, c->scR, c->scC, sm);
    launch_axpy_box(c->st, L.d, cb, out, c->scC);
  }
}

// ---- reductions ----------------------------------------------------------------

// small device/host scratch: [h1: 3*kMaxVec][h2: kMaxVec][misc 64][y kMaxVec]
double* dh1(sb_ctx* c) { return c->dsmall; }
double* dh2(sb_ctx* c) { return c->dsmall + 3 * kMaxVec; }
double* dmisc(sb_ctx* c) { return c->dsmall + 4 * kMaxVec; }
double* dy(sb_ctx* c) { return c->dsmall + 4 * kMaxVec + 64; }
double* hh1(sb_ctx* c) { return c->hsmall; }
double* hh2(sb_ctx* c) { return c->hsmall + 3 * kMaxVec; }
double* hmisc(sb_ctx* c) { return c->hsmall + 4 * kMaxVec; }
double* hy(sb_ctx* c) { return c->hsmall + 4 * kMaxVec + 64; }

// device sum of a full block into dmisc[slot]
void block_sum(sb_ctx* c, const double* x, long long n, int slot) {
  launch_sum_partial(c->st, x, n, c->dpart);
  launch_finalize(c->st, c->dpart, 1, dmisc(c) + slot);
}

// ||x||^2 of a flat vector into dmisc[slot]
void vec_norm2(sb_ctx* c, const double* x, int slot) {
  launch_multi_dot(c->st, x, 0, 1, x, c->vlen, c->dpart);
  launch_finalize(c->st, c->dpart, 1, dmisc(c) + slot);
}

double fetch_misc(sb_ctx* c, int slot) {
  CK(cudaMemcpyAsync(hmisc(c) + slot, dmisc(c) + slot, 8, cudaMemcpyDeviceToHost, c->st));
  sync(c);
  return hmisc(c)[slot];
}

// ---- preconditioner (precond.py:111-168) ------------------------------------------

long long precond_cost(const sb_ctx* c, const sb_precond& pc) {
  const long long v = (long long)c->dim * pc.velocity_cycles, p = pc.pressure_cycles;
  const bool th = c->theta > 0;
  switch (pc.kind) {
    case SB_P1: return v + p;
    case SB_P2: case SB_P3: case SB_P4: return v + (th ? p : 0);
    case SB_P5: return 2 * v + (th ? p : 0);
    default: return 0;
  }
}

void project_nulls(sb_ctx* c, double* x) {
  const Level& L = c->lv[0];
  Box cb;
  for (int a = 0; a < 3; ++a) {
    cb.lo[a] = 0;
    cb.hi[a] = L.d.n[a] - 1;
  }
  const double ncell = (double)L.d.n[0] * L.d.n[1] * L.d.n[2];
  double* xp = vpres(c, x);
  block_sum(c, xp, L.block, 0);
  launch_box_add_scalar(c->st, L.d, cb, xp, dmisc(c) + 0, 1.0 / ncell);
  int slot = 1;
  for (int A : c->null_comps) {
    double* xa = vcomp(c, x, A);
    block_sum(c, xa, L.block, slot);
    // null components are periodic along A: every stored face is an unknown
    launch_box_add_scalar(c->st, L.d, cb, xa, dmisc(c) + slot, 1.0 / ncell);
    ++slot;
  }
}

double* dmeans(sb_ctx* c) { return dmisc(c) + 32; }

// The sums of project_nulls only, and the per-block means the deferred
// subtraction uses (Arnoldi pass B or finish_projection); same slots.
void project_sums(sb_ctx* c, double* x) {
  const Level& L = c->lv[0];
  const double ncell = (double)L.d.n[0] * L.d.n[1] * L.d.n[2];
  int slot[4] = {-1, -1, -1, -1};
  block_sum(c, vpres(c, x), L.block, 0);
  slot[c->dim] = 0;
  int k = 1;
  for (int A : c->null_comps) {
    block_sum(c, vcomp(c, x, A), L.block, k);
    slot[A - c->off] = k++;
  }
  launch_block_means(c->st, dmisc(c), slot, 1.0 / ncell, dmeans(c));
}

// the subtraction half of project_nulls, after project_sums (bit-identical result)
void finish_projection(sb_ctx* c, double* x) {
  if (!c->defer_nulls) return;
  const Level& L = c->lv[0];
  Box cb;
  for (int a = 0; a < 3; ++a) {
    cb.lo[a] = 0;
    cb.hi[a] = L.d.n[a] - 1;
  }
  const double ncell = (double)L.d.n[0] * L.d.n[1] * L.d.n[2];
  launch_box_add_scalar(c->st, L.d, cb, vpres(c, x), dmisc(c) + 0, 1.0 / ncell);
  int slot = 1;
  for (int A : c->null_comps) launch_box_add_scalar(c->st, L.d, cb, vcomp(c, x, A), dmisc(c) + slot++, 1.0 / ncell);
}

// x = P^{-1} r on level-0 vectors (all device, stream-ordered, graph-capturable);
// with defer_nulls the null-space means are computed but not yet subtracted
void precond_dev(sb_ctx* c, const sb_precond& pc, const sb_smoother& sm, double* r, double* x) {
  const Level& L = c->lv[0];
  const int d = c->dim, o = c->off;
  const double sign = pc.schur_sign < 0 ? -1.0 : 1.0;
  const double* ru[3] = {nullptr, nullptr, nullptr};
  double* xu[3] = {nullptr, nullptr, nullptr};
  for (int A = o; A < 3; ++A) {
    ru[A] = vcomp(c, r, A);
    xu[A] = vcomp(c, x, A);
  }
  double* rp = vpres(c, r);
  double* xp = vpres(c, x);
  if (pc.kind == SB_IDENTITY) {
    CK(cudaMemcpyAsync(x, r, c->vlen * 8, cudaMemcpyDeviceToDevice, c->st));
    return;
  }
  ensure_scratch(c);
  const bool th = c->theta > 0;
  CPtr3 cxu{{xu[0], xu[1], xu[2]}};
  switch (pc.kind) {
    case SB_P1: {
      mg_face(c, pc.velocity_cycles, ru, xu, sm);
      launch_div_add(c->st, L.d, d, cxu, rp, c->sc0);
      mg_cell(c, pc.pressure_cycles, c->sc0, c->sc1, sm);
      Ptr3 pxu{{xu[0], xu[1], xu[2]}};
      launch_p1_glue(c->st, L.d, d, c->form, pxu, c->sc1, c->sc0, xp, sign);
      break;
    }
    case SB_P2: {
      mg_face(c, pc.velocity_cycles, ru, xu, sm);
      launch_div_add(c->st, L.d, d, cxu, rp, c->sc0);
      if (th) mg_cell(c, pc.pressure_cycles, c->sc0, c->sc1, sm);
      launch_schur(c->st, L.d, c->form, c->sc0, th ? c->sc1 : nullptr, xp, sign);
      break;
    }
    case SB_P3: {
      if (th) mg_cell(c, pc.pressure_cycles, rp, c->sc1, sm);
      launch_schur(c->st, L.d, c->form, rp, th ? c->sc1 : nullptr, xp, sign);
      CPtr3 cru{{ru[0], ru[1], ru[2]}};
      Ptr3 f0{{c->sf0[0], c->sf0[1], c->sf0[2]}};
      launch_face_sub_grad(c->st, L.d, d, cru, xp, f0);
      mg_face(c, pc.velocity_cycles, c->sf0, xu, sm);
      break;
    }
    case SB_P4: {
      mg_face(c, pc.velocity_cycles, ru, xu, sm);
      if (th) mg_cell(c, pc.pressure_cycles, rp, c->sc1, sm);
      launch_schur(c->st, L.d, c->form, rp, th ? c->sc1 : nullptr, xp, sign);
      break;
    }
    case SB_P5: {
      mg_face(c, pc.velocity_cycles, ru, c->sf1, sm);
      CPtr3 cs1{{c->sf1[0], c->sf1[1], c->sf1[2]}};
      launch_div_add(c->st, L.d, d, cs1, rp, c->sc0);
      if (th) mg_cell(c, pc.pressure_cycles, c->sc0, c->sc1, sm);
      launch_schur(c->st, L.d, c->form, c->sc0, th ? c->sc1 : nullptr, xp, sign);
      CPtr3 cru{{ru[0], ru[1], ru[2]}};
      Ptr3 f0{{c->sf0[0], c->sf0[1], c->sf0[2]}};
      launch_face_residual(c->st, L.d, d, c->form, cs1, cru, xp, f0);
      mg_face(c, pc.velocity_cycles, c->sf0, xu, sm);
      for (int A = o; A < 3; ++A) {
        Box fb;
        for (int a = 0; a < 3; ++a) {
          fb.lo[a] = 0;
          fb.hi[a] = L.d.n[a] - 1 + ((a == A && c->bc[A][0] != BC_PER) ? 1 : 0);
        }
        launch_axpy_box(c->st, L.d, fb, xu[A], c->sf1[A]);
      }
      break;
    }
    default:
      throw ArgErr(SB_EINVAL, "unknown preconditioner kind");
  }
  if (c->defer_nulls) project_sums(c, x);
  else project_nulls(c, x);
}

void drop_graph(sb_ctx* c) {
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  c->gexec = nullptr;
}

// vw = P^{-1} vMv, through the cached CUDA graph when enabled
void precond_apply_graph(sb_ctx* c, const sb_precond& pc, const sb_smoother& sm) {
  if (!c->use_graphs || c->profiling) {
    precond_dev(c, pc, sm, c->vMv, c->vw);
    return;
  }
  const bool same = c->gexec && std::memcmp(&c->gpc, &pc, sizeof(pc)) == 0 &&
                    std::memcmp(&c->gsm, &sm, sizeof(sm)) == 0;
  if (!same) {
    drop_graph(c);
    ensure_scratch(c);
    if (pc.velocity_cycles > 1 || pc.pressure_cycles > 1) ensure_scratch_mg(c);
    const long long before = g_kernel_launches;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
    try {
      precond_dev(c, pc, sm, c->vMv, c->vw);
    } catch (...) {
      cudaStreamEndCapture(c->st, &g);
      if (g) cudaGraphDestroy(g);
      g_kernel_launches = before;
      throw;
    }
    CK(cudaStreamEndCapture(c->st, &g));
    g_kernel_launches = before;
    size_t nn = 0;
    CK(cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    CK(cudaGraphGetNodes(g, nodes.data(), &nn));
    long long nk = 0;
    for (auto& nd : nodes) {
      cudaGraphNodeType t;
      CK(cudaGraphNodeGetType(nd, &t));
      if (t == cudaGraphNodeTypeKernel) ++nk;
    }
    CK(cudaGraphInstantiate(&c->gexec, g, 0));
    CK(cudaGraphDestroy(g));
    c->gnodes = nk;
    c->gpc = pc;
    c->gsm = sm;
  }
  CK(cudaGraphLaunch(c->gexec, c->st));
  c->graph_launches += c->gnodes;
}

// ---- GMRES (krylov.py:81-214) -----------------------------------------------------

void solve_upper(const std::vector<double>& H, int ld, const double* g, int n, double* y) {
  for (int i = n - 1; i >= 0; --i) {
    double s = 0.0;
    for (int k = i + 1; k < n; ++k) s += H[i * ld + k] * y[k];
    y[i] = (g[i] - s) / H[i * ld + i];
  }
}

void apply_M_vec(sb_ctx* c, const double* x, double* out) {
  const Level& L = c->lv[0];
  CPtr3 u{{nullptr, nullptr, nullptr}};
  Ptr3 o{{nullptr, nullptr, nullptr}};
  for (int A = c->off; A < 3; ++A) {
    u.p[A] = vcomp(c, (double*)x, A);
    o.p[A] = vcomp(c, out, A);
  }
  launch_apply_M(c->st, L.d, c->dim, c->form, u, vpres(c, (double*)x), o, vpres(c, out));
}

// upload a host/device vector in the reference layout into a level-0 vector
// keep_walls: read the wall-normal boundary faces as given (operators.apply_M);
// otherwise zero them (vectors of the packed unknown space, grid.py:373)
void vec_in(sb_ctx* c, const double* const* u, const double* p, double* v, bool keep_walls = false) {
  const Level& L = c->lv[0];
  for (int r = 0; r < c->dim; ++r) {
    const int A = r + c->off;
    copy_in(c, L, A, u[r], vcomp(c, v, A));
    if (!keep_walls) zero_wall_faces(c, L, A, vcomp(c, v, A));
  }
  copy_in(c, L, -1, p, vpres(c, v));
}
void vec_out(sb_ctx* c, const double* v, double* const* u, double* p) {
  const Level& L = c->lv[0];
  for (int r = 0; r < c->dim; ++r) {
    const int A = r + c->off;
    copy_out(c, L, A, vcomp(c, (double*)v, A), u[r]);
  }
  copy_out(c, L, -1, vpres(c, (double*)v), p);
}

void ensure_basis(sb_ctx* c, int m) {
  if (c->basis_cap >= m + 1) return;
  if (c->basis) {
    for (auto it = c->allocs.begin(); it != c->allocs.end(); ++it)
      if (*it == c->basis) {
        c->allocs.erase(it);
        break;
      }
    CK(cudaFree(c->basis));
    c->bytes -= (long long)c->basis_cap * c->vlen * 8;
    c->basis = nullptr;
  }
  c->basis = dalloc(c, (long long)(m + 1) * c->vlen);
  c->basis_cap = m + 1;
}

void prof_reset(sb_ctx* c) {
  c->prof.clear();
  c->evnext = 0;
}

void prof_collect(sb_ctx* c) {
  sb_kernel_stats s{};
  for (auto& e : c->prof) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e.a, e.b));
    if (e.cls == 0) {
      s.smoother_face_ms += ms;
      s.smoother_face_bytes += e.bytes;
      s.smoother_face_launches++;
      if (e.fine) {
        s.fine_face_ms += ms;
        s.fine_face_bytes += e.bytes;
        s.fine_face_launches++;
      }
    } else {
      s.smoother_cell_ms += ms;
      s.smoother_cell_bytes += e.bytes;
      s.smoother_cell_launches++;
    }
  }
  c->stats = s;
}

int gmres(sb_ctx* c, const sb_precond& pc, const sb_gmres& gc, const sb_smoother& sm,
          const double* const* bu, const double* bp, double* const* xu, double* xpo,
          sb_history_row* rows, int max_rows, int* n_rows, int* status, long long* vcyc) {
  if (pc.kind != SB_IDENTITY) {
    check_mg(c, SB_KIND_FACE);
    if (pc.kind == SB_P1 || c->theta > 0) check_mg(c, SB_KIND_CELL);
  } else {
    check_ready(c);
  }
  const int m = gc.restart;
  if (m < 1) throw ArgErr(SB_EINVAL, "restart must be >= 1");
  // restart >= kMaxVec: the delayed-reorthogonalisation kernels keep one
  // partial sum per basis vector in shared memory, so a longer basis takes the
  // textbook CGS2 step in chunks (launch_cgs2); the reference's GmresConfig
  // has no upper bound (krylov.py:23-38)
  const bool big = m >= kMaxVec;
  const int bigM = (m + 2 + 3) / 4 * 4;
  if (big && c->bigcap < bigM) {
    if (c->hbig) cudaFreeHost(c->hbig);
    c->hbig = nullptr;
    c->dbig = dalloc(c, 3LL * bigM);
    CK(cudaMallocHost(&c->hbig, (size_t)3 * bigM * 8));
    c->bigcap = bigM;
  }
  ensure_vectors(c);
  ensure_basis(c, m);
  if (c->profiling) prof_reset(c);
  const long long vl = c->vlen;
  int nr = 0;
  auto add_row = [&](int it, double rp, double rt, bool rf) {
    if (nr < max_rows) rows[nr] = sb_history_row{it, *vcyc, rp, rt, rf ? 1 : 0};
    ++nr;
  };
  vec_in(c, bu, bp, c->vb);
  vec_norm2(c, c->vb, 0);
  const double bnorm = std::sqrt(fetch_misc(c, 0));
  // z0 = P^{-1} b
  CK(cudaMemcpyAsync(c->vMv, c->vb, vl * 8, cudaMemcpyDeviceToDevice, c->st));
  precond_apply_graph(c, pc, sm);
  finish_projection(c, c->vw);
  *vcyc += precond_cost(c, pc);
  CK(cudaMemcpyAsync(c->vz0, c->vw, vl * 8, cudaMemcpyDeviceToDevice, c->st));
  vec_norm2(c, c->vz0, 0);
  const double rp0 = std::sqrt(fetch_misc(c, 0));
  add_row(0, rp0, bnorm, false);
  CK(cudaMemsetAsync(c->vx, 0, vl * 8, c->st));
  auto finish = [&](int st) {
    vec_out(c, c->vx, xu, xpo);
    sync(c);
    *status = st;
    *n_rows = nr;
    if (c->profiling) prof_collect(c);
    return SB_OK;
  };
  if (rp0 <= gc.atol || rp0 == 0.0) return finish(SB_STATUS_CONVERGED);
  const double target = gc.rtol * rp0 + gc.atol;
  const double bd_tol = std::max(gc.atol, 1e-14 * rp0);

  std::vector<double> H((m + 1) * m), Horig((m + 1) * m), cs(m), sn(m), g(m + 1), y(m + 1), cpend(m + 1);
  static const bool cgs2 = [] {
    const char* e = std::getenv("SB_ORTHO");
    return e && std::strcmp(e, "cgs2") == 0;
  }();
  // default: Gram variant; SB_ORTHO=dcgs re-reads the basis for c', =cgs2 three passes
  static const bool gram = [] {
    const char* e = std::getenv("SB_ORTHO");
    return !(e && (std::strcmp(e, "dcgs") == 0 || std::strcmp(e, "cgs2") == 0));
  }();
  // SB_ORTHO=gram1: one-pass Gram Arnoldi (opt-in).  It removes pass B (C5
  // 256^3 launch list 336 -> 321 ms) but its pending coefficients t = d + c'
  // are first order (||t|| / gam_{j+1} = ||w|| / ||r||, growing along a cycle),
  // so every implicit step carries ~eps ||w|| / ||r|| of cancellation error:
  // harmless at rtol 1e-9, but the Krylov relation is no longer accurate to
  // the 1e-14 breakdown threshold (krylov.py:138, 198) -- a Krylov-exhaustion
  // solve runs to maxiter instead of breaking down.  The default two-pass Gram
  // variant keeps the pending correction second order (cpend = c').
  static const bool one_pass = [] {
    const char* e = std::getenv("SB_ORTHO");
    return e && std::strcmp(e, "gram1") == 0;
  }();
  std::vector<double> G((m + 1) * (m + 1), 0.0), tv(m + 1);
  const bool cgs2_l = cgs2 || big, gram_l = gram && !big;
  double* const yd = big ? c->dbig + 2 * c->bigcap : dy(c);  // least-squares solution y on the device
  double* const yh = big ? c->hbig + 2 * c->bigcap : hy(c);
  double gam = 1.0;
  int k = 0;
  bool first = true;
  const double* r = c->vz0;
  double beta = rp0;
  while (true) {
    if (!first) {
      vec_norm2(c, r, 0);
      beta = std::sqrt(fetch_misc(c, 0));
    }
    if (beta == 0.0) return finish(SB_STATUS_CONVERGED);
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(Horig.begin(), Horig.end(), 0.0);
    std::fill(G.begin(), G.end(), 0.0);
    gam = 1.0;  // q_0 = r / beta is final: no pending correction
    std::fill(cs.begin(), cs.end(), 0.0);
    std::fill(sn.begin(), sn.end(), 0.0);
    std::fill(g.begin(), g.end(), 0.0);
    double* V = c->basis;
    launch_scale_div(c->st, r, beta, V, vl);
    g[0] = beta;
    int j = 0;
    int ydim = 0;  // columns in the last least-squares solve
    while (j < m && k < gc.max_iters) {
      apply_M_vec(c, V + (long long)j * vl, c->vMv);
      precond_apply_graph(c, pc, sm);
      // the Gram pass B subtracts the deferred null-space means while it
      // streams w (P^-1 M Q has zero means in exact arithmetic, so pass A's
      // dots with the basis are unaffected); the other variants project here
      if (!gram_l) finish_projection(c, c->vw);
      *vcyc += precond_cost(c, pc);
      ++k;
      double hn;
      if (cgs2_l) {
        // CGS2 Arnoldi (parity-safe replacement of MGS)
        const int nv = j + 1;
        double* h1d = big ? c->dbig : dh1(c);
        double* h2d = big ? c->dbig + c->bigcap : dh2(c);
        launch_cgs2(c->st, V, vl, nv, c->vw, vl, c->dpart, h1d, h2d, dmisc(c) + 1);
        const double *h1h, *h2h;
        if (big) {
          CK(cudaMemcpyAsync(c->hbig, c->dbig, (size_t)2 * c->bigcap * 8, cudaMemcpyDeviceToHost, c->st));
          h1h = c->hbig;
          h2h = c->hbig + c->bigcap;
        } else {
          h1h = hh1(c);
          h2h = hh2(c);
        }
        CK(cudaMemcpyAsync(c->hsmall, c->dsmall, (4 * kMaxVec + 2) * 8, cudaMemcpyDeviceToHost, c->st));
        sync(c);
        for (int i = 0; i <= j; ++i) H[i * m + j] = h1h[i] + h2h[i];
        hn = std::sqrt(hmisc(c)[1]);
      } else {
        // CGS2 with delayed reorthogonalisation: two passes over the basis.
        // Slot j holds s_j = gam_j q_j + Q_j cpend; w = P^-1 M s_j.
        //  A: q_j = (s_j - Q_j cpend)/gam_j written in place, d = [Q_j q_j]^T w
        //  B: w' = w - Q_{j+1} d -> slot j+1, c' = Q_{j+1}^T w', ||w'||^2
        // Using P^-1 M Q_j = Q_{j+1} Horig (Arnoldi relation):
        //  H[:j+1, j] = (d - Horig cpend + c')/gam_j,
        //  H[j+1, j]  = sqrt(||w'||^2 - ||c'||^2)/gam_j, and slot j+1 becomes
        //  s_{j+1} = w' with cpend = c', gam_{j+1} = sqrt(||w'||^2 - ||c'||^2).
        // gram: c' = d - G d from the Gram matrix G = Q^T Q, maintained from the
        // extra dots of pass A, so pass B streams the basis once (no re-read).
        for (int i = 0; i < j; ++i) hy(c)[i] = cpend[i];
        if (j > 0) CK(cudaMemcpyAsync(dh2(c), hy(c), j * 8, cudaMemcpyHostToDevice, c->st));
        double cc = 0.0, ww;
        if (one_pass) {
          // One pass over the basis per iteration.  Pass A finishes q_j, forms
          // d = Q_{j+1}^T w, the Gram extension and ||w||^2, and stores w
          // (projected by the deferred means) into slot j+1 as the unfinished
          // s_{j+1} = gam_{j+1} q_{j+1} + Q_{j+1} t with t = d + c' (c' = d - G d,
          // the CGS2 correction), gam_{j+1}^2 = ||w||^2 - 2 t.d + t^T G t.  The
          // next pass A applies t while it streams the basis, so the separate
          // pass B (w' = w - Q d) disappears.  Near a breakdown (gam_{j+1}^2 <
          // kOnePassRel ||w||^2) the step is finished explicitly: two streamed
          // CGS passes on slot j+1 and a direct norm (krylov.py:114).
          double* sj1 = V + (long long)(j + 1) * vl;
          launch_arnoldi1(c->st, V, vl, j, dh2(c), 1.0 / gam, c->vw, vl, c->dpart,
                          c->defer_nulls ? dmeans(c) : nullptr, c->lv[0].block);
          launch_finalize(c->st, c->dpart, 2 * j + 3, dh1(c));
          CK(cudaMemcpyAsync(c->hsmall, c->dsmall, (2 * j + 3) * 8, cudaMemcpyDeviceToHost, c->st));
          sync(c);
          const double* dd = hh1(c);
          const double* sd = hh1(c) + j + 1;
          const double ss = hh1(c)[2 * j + 1];
          const double wwf = hh1(c)[2 * j + 2];
          double cgc = 0.0, csd = 0.0;
          for (int l = 0; l < j; ++l) {
            double gcl = 0.0;
            for (int t = 0; t < j; ++t) gcl += G[l * (m + 1) + t] * cpend[t];
            const double gjl = (sd[l] - gcl) / gam;
            G[j * (m + 1) + l] = gjl;
            G[l * (m + 1) + j] = gjl;
            cgc += cpend[l] * gcl;
            csd += cpend[l] * sd[l];
          }
          G[j * (m + 1) + j] = j == 0 ? ss : (ss - 2.0 * csd + cgc) / (gam * gam);
          std::vector<double> cp(j + 1);
          for (int i = 0; i <= j; ++i) {
            double gd = 0.0;
            for (int t = 0; t <= j; ++t) gd += G[i * (m + 1) + t] * dd[t];
            cp[i] = dd[i] - gd;
            tv[i] = dd[i] + cp[i];
          }
          double td = 0.0, tgt = 0.0;
          for (int i = 0; i <= j; ++i) {
            double gt = 0.0;
            for (int t = 0; t <= j; ++t) gt += G[i * (m + 1) + t] * tv[t];
            td += tv[i] * dd[i];
            tgt += tv[i] * gt;
          }
          const double r2 = wwf - 2.0 * td + tgt;
          const bool direct = !(r2 > kOnePassRel * wwf);
          double gnext;
          if (direct) {
            for (int i = 0; i <= j; ++i) hy(c)[i] = dd[i];
            CK(cudaMemcpyAsync(dy(c), hy(c), (j + 1) * 8, cudaMemcpyHostToDevice, c->st));
            launch_update_dot(c->st, V, vl, j + 1, dy(c), sj1, vl, c->dpart, 0);
            launch_finalize(c->st, c->dpart, j + 1, dy(c) + kMaxVec);
            launch_update_dot(c->st, V, vl, j + 1, dy(c) + kMaxVec, sj1, vl, c->dpart, 1);
            launch_finalize(c->st, c->dpart, 1, dmisc(c) + 1);
            CK(cudaMemcpyAsync(hy(c), dy(c) + kMaxVec, (j + 1) * 8, cudaMemcpyDeviceToHost, c->st));
            gnext = std::sqrt(fetch_misc(c, 1));  // synchronises
            for (int i = 0; i <= j; ++i) cp[i] = hy(c)[i];
            ++c->direct_norms;
          } else {
            gnext = std::sqrt(r2);
          }
          for (int i = 0; i <= j; ++i) {
            double e = 0.0;
            for (int t = 0; t < j; ++t) e += Horig[i * m + t] * cpend[t];
            H[i * m + j] = ((dd[i] - e) + cp[i]) / gam;
          }
          hn = gnext / gam;
          static const bool trace1 = [] {
            const char* e = std::getenv("SB_GMRES_TRACE");
            return e && e[0] == '1';
          }();
          if (trace1)
            std::fprintf(stderr, "gmres1 k=%d j=%d ww=%.6e r2=%.6e gnext=%.6e gam=%.6e hn=%.6e direct=%d\n", k, j,
                         wwf, r2, gnext, gam, hn, (int)direct);
          for (int i = 0; i <= j; ++i) Horig[i * m + j] = H[i * m + j];
          Horig[(j + 1) * m + j] = hn;
          for (int i = 0; i <= j; ++i) cpend[i] = direct ? 0.0 : dd[i] + cp[i];
          gam = gnext;
        } else {
        if (gram) {
          launch_dcgs_a_g(c->st, V, vl, j, dh2(c), 1.0 / gam, c->vw, vl, c->dpart,
                          c->defer_nulls ? dmeans(c) : nullptr, c->lv[0].block);
          launch_finalize(c->st, c->dpart, 2 * j + 2, dh1(c));
          launch_dcgs_b_g(c->st, V, vl, j + 1, dh1(c), c->vw, V + (long long)(j + 1) * vl, vl, c->dpart,
                          c->defer_nulls ? dmeans(c) : nullptr, c->lv[0].block);
          launch_finalize(c->st, c->dpart, 1, dh2(c) + kMaxVec - 1);
          CK(cudaMemcpyAsync(c->hsmall, c->dsmall, (4 * kMaxVec) * 8, cudaMemcpyDeviceToHost, c->st));
          sync(c);
          const double* dd = hh1(c);
          const double* sd = hh1(c) + j + 1;  // Q_l . s_j
          const double ss = hh1(c)[2 * j + 1];
          // extend G with the finished q_j = (s_j - Q_j cpend)/gam
          double cgc = 0.0, csd = 0.0;
          for (int l = 0; l < j; ++l) {
            double gcl = 0.0;
            for (int t = 0; t < j; ++t) gcl += G[l * (m + 1) + t] * cpend[t];
            const double gjl = (sd[l] - gcl) / gam;
            G[j * (m + 1) + l] = gjl;
            G[l * (m + 1) + j] = gjl;
            cgc += cpend[l] * gcl;
            csd += cpend[l] * sd[l];
          }
          G[j * (m + 1) + j] = j == 0 ? ss : (ss - 2.0 * csd + cgc) / (gam * gam);
          for (int i = 0; i <= j; ++i) {
            double gd = 0.0;
            for (int t = 0; t <= j; ++t) gd += G[i * (m + 1) + t] * dd[t];
            hh2(c)[i] = dd[i] - gd;  // c'
          }
          ww = hh2(c)[kMaxVec - 1];
        } else {
          launch_dcgs_a(c->st, V, vl, j, dh2(c), 1.0 / gam, c->vw, vl, c->dpart);
          launch_finalize(c->st, c->dpart, j + 1, dh1(c));
          launch_dcgs_b(c->st, V, vl, j + 1, dh1(c), c->vw, V + (long long)(j + 1) * vl, vl, c->dpart);
          launch_finalize(c->st, c->dpart, j + 2, dh2(c));
          CK(cudaMemcpyAsync(c->hsmall, c->dsmall, (4 * kMaxVec) * 8, cudaMemcpyDeviceToHost, c->st));
          sync(c);
          ww = hh2(c)[j + 1];
        }
        double dd = 0.0;
        for (int i = 0; i <= j; ++i) {
          cc += hh2(c)[i] * hh2(c)[i];
          dd += hh1(c)[i] * hh1(c)[i];
        }
        // Near a breakdown (w nearly in span(Q)) the delayed scheme loses its
        // accuracy: ||w'||^2 - ||c'||^2 cancels, and the Gram c' = d - G d
        // carries an absolute error ~eps ||d|| that can exceed ||w'|| itself.
        // Then finish the step explicitly: c' = Q^T w' re-read from the basis
        // (gram) and s_{j+1} = w' - Q c' with its norm taken directly, as the
        // reference's ||w|| (krylov.py:114).  Nothing stays pending.
        const bool direct = cc > 0.5 * ww || ww < kDirectRel * (dd + ww);
        double gnext;
        if (direct) {
          double* sj = V + (long long)(j + 1) * vl;
          if (gram) {
            launch_multi_dot(c->st, V, vl, j + 1, sj, vl, c->dpart);
            launch_finalize(c->st, c->dpart, j + 1, dy(c));
          } else {
            for (int i = 0; i <= j; ++i) hy(c)[i] = hh2(c)[i];
            CK(cudaMemcpyAsync(dy(c), hy(c), (j + 1) * 8, cudaMemcpyHostToDevice, c->st));
          }
          launch_update_dot(c->st, V, vl, j + 1, dy(c), sj, vl, c->dpart, 1);
          launch_finalize(c->st, c->dpart, 1, dmisc(c) + 1);
          CK(cudaMemcpyAsync(hy(c), dy(c), (j + 1) * 8, cudaMemcpyDeviceToHost, c->st));
          gnext = std::sqrt(fetch_misc(c, 1));  // synchronises
          for (int i = 0; i <= j; ++i) hh2(c)[i] = hy(c)[i];
          ++c->direct_norms;
        } else {
          gnext = std::sqrt(std::max(ww - cc, 0.0));
        }
        for (int i = 0; i <= j; ++i) {
          double e = 0.0;
          for (int t = 0; t < j; ++t) e += Horig[i * m + t] * cpend[t];
          H[i * m + j] = ((hh1(c)[i] - e) + hh2(c)[i]) / gam;
        }
        hn = gnext / gam;
        static const bool trace = [] {
          const char* e = std::getenv("SB_GMRES_TRACE");
          return e && e[0] == '1';
        }();
        if (trace)
          std::fprintf(stderr, "gmres k=%d j=%d ww=%.6e cc=%.6e gnext=%.6e gam=%.6e hn=%.6e direct=%d\n", k, j, ww,
                       cc, gnext, gam, hn, (int)direct);
        for (int i = 0; i <= j; ++i) Horig[i * m + j] = H[i * m + j];
        Horig[(j + 1) * m + j] = hn;
        for (int i = 0; i <= j; ++i) cpend[i] = direct ? 0.0 : hh2(c)[i];
        gam = gnext;
        }  // two-pass Gram / DCGS
      }
      H[(j + 1) * m + j] = hn;
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * H[i * m + j] + sn[i] * H[(i + 1) * m + j];
        H[(i + 1) * m + j] = -sn[i] * H[i * m + j] + cs[i] * H[(i + 1) * m + j];
        H[i * m + j] = t;
      }
      const double den = std::hypot(H[j * m + j], H[(j + 1) * m + j]);
      if (den == 0.0) {
        cs[j] = 1.0;
        sn[j] = 0.0;
      } else {
        cs[j] = H[j * m + j] / den;
        sn[j] = H[(j + 1) * m + j] / den;
      }
      H[j * m + j] = den;
      H[(j + 1) * m + j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      const double rp = std::fabs(g[j + 1]);
      const bool conv = rp <= target;
      const bool brk = !conv && hn <= bd_tol;
      ydim = j + 1;
      double rt = NAN;
      if (gc.track_true_residual || conv || brk) {
        solve_upper(H, m, g.data(), ydim, y.data());
        std::memcpy(yh, y.data(), ydim * 8);
        CK(cudaMemcpyAsync(yd, yh, ydim * 8, cudaMemcpyHostToDevice, c->st));
      }
      if (gc.track_true_residual) {
        launch_combo(c->st, c->vt, c->vx, V, vl, ydim, yd, vl);
        apply_M_vec(c, c->vt, c->vMv);
        launch_sub_norm(c->st, c->vb, c->vMv, vl, c->dpart);
        launch_finalize(c->st, c->dpart, 1, dmisc(c) + 2);
        rt = std::sqrt(fetch_misc(c, 2));
      }
      add_row(k, rp, rt, j == 0 && !first);
      if (conv || brk) {
        launch_combo(c->st, c->vx, c->vx, V, vl, ydim, yd, vl);
        return finish(conv ? SB_STATUS_CONVERGED : SB_STATUS_BREAKDOWN);
      }
      if (cgs2_l) launch_scale_div(c->st, c->vw, hn, V + (long long)(j + 1) * vl, vl);
      ++j;
    }
    // x = x + V[:j] y  (the last iteration's least-squares solution)
    solve_upper(H, m, g.data(), ydim, y.data());
    std::memcpy(yh, y.data(), ydim * 8);
    CK(cudaMemcpyAsync(yd, yh, ydim * 8, cudaMemcpyHostToDevice, c->st));
    launch_combo(c->st, c->vx, c->vx, V, vl, ydim, yd, vl);
    first = false;
    if (k >= gc.max_iters) return finish(SB_STATUS_MAXITER);
    // r = z0 - P^{-1} M x
    apply_M_vec(c, c->vx, c->vMv);
    precond_apply_graph(c, pc, sm);
    finish_projection(c, c->vw);
    *vcyc += precond_cost(c, pc);
    launch_sub(c->st, c->vz0, c->vw, c->vt, vl);
    r = c->vt;
  }
}

template <class F>
int guard(F&& f) {
  try {
    return f();
  } catch (const ArgErr& e) {
    g_err = e.what();
    return e.code;
  } catch (const CudaErr& e) {
    g_err = e.what();
    return SB_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SB_ECUDA;
  }
}


// Coarsen the level-0 coefficients (already on the device) down the hierarchy,
// derive 1/rho_face, run the zero-diagonal / positive-density checks and the
// velocity null space (multigrid.py:92-169, :70-89; operators.py:368-388).
// choose the coarse tail (first level >= 1 with <= kCoarseCells cells) and
// upload its level table; SB_COARSE_KERNEL=0 keeps every level multi-kernel
void upload_chains(sb_ctx* c) {
  const bool enabled = [] {
    const char* e = std::getenv("SB_COARSE_KERNEL");
    return !(e && e[0] == '0');
  }();
  c->coarse_ls = -1;
  const int nlev = (int)c->lv.size();
  if (!enabled || c->lv[0].d.dist0 || nlev < 2) return;
  int ls = -1;
  // largest level of the tail: 3D 8^3, 2D 32^2 (the 16^3 / 64^2 levels run
  // faster as multi-kernel passes: C5 256^3 0.3407 -> 0.3386 s, C3 128^3
  // 0.0907 -> 0.0862 s, C2 256^2 8.19 -> 6.89 ms); SB_COARSE_CELLS overrides
  const long long max_cells = [&] {
    const char* e = std::getenv("SB_COARSE_CELLS");
    return e ? std::atoll(e) : (c->dim == 3 ? kCoarseCells3 : kCoarseCells);
  }();
  for (int l = 1; l < nlev; ++l) {
    long long cells = 1;
    for (int a = 3 - c->dim; a < 3; ++a) cells *= c->lv[l].d.n[a];
    if (cells <= max_cells) {
      ls = l;
      break;
    }
  }
  if (ls < 0 || nlev - ls > kCoarseMaxLevels) return;
  CoarseChain hf{}, hc{};
  hf.nl = hc.nl = nlev - ls;
  for (int l = ls; l < nlev; ++l) {
    const Level& L = c->lv[l];
    CoarseLv& f = hf.lv[l - ls];
    CoarseLv& k = hc.lv[l - ls];
    f.d = k.d = L.d;
    for (int a = 0; a < 3; ++a) {
      f.x[a] = L.fx[a];
      f.rhs[a] = L.frhs[a];
    }
    k.x[0] = L.cx;
    k.rhs[0] = L.crhs;
    f.tmp = k.tmp = L.tmp;
    f.block = k.block = L.block;
    f.two_phase = k.two_phase = L.two_phase ? 1 : 0;
  }
  const long long nd = (long long)(sizeof(CoarseChain) + 7) / 8;
  if (!c->dchain_face) c->dchain_face = reinterpret_cast<CoarseChain*>(dalloc(c, nd));
  if (!c->dchain_cell) c->dchain_cell = reinterpret_cast<CoarseChain*>(dalloc(c, nd));
  CK(cudaMemcpyAsync(c->dchain_face, &hf, sizeof(hf), cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->dchain_cell, &hc, sizeof(hc), cudaMemcpyHostToDevice, c->st));
  CK(cudaStreamSynchronize(c->st));
  c->coarse_ls = ls;
}

void build_from_level0(sb_ctx* c) {
    for (size_t l = 0; l + 1 < c->lv.size(); ++l) {
      Level& F = c->lv[l];
      Level& C = c->lv[l + 1];
      launch_coarsen_cellmean(c->st, F.d, C.d, c->dim, F.mu_c, C.mu_c);
      launch_coarsen_cellmean(c->st, F.d, C.d, c->dim, F.gam_c, C.gam_c);
      for (int A = c->off; A < 3; ++A) launch_coarsen_face(c->st, F.d, C.d, c->dim, A, F.rho_f[A], C.rho_f[A]);
      if (c->dim == 3) {
        for (int e = 0; e < 3; ++e) launch_coarsen_edge(c->st, F.d, C.d, 3, e, F.mu_e[e], C.mu_e[e]);
      } else {
        launch_coarsen_edge(c->st, F.d, C.d, 2, 0, F.mu_e[0], C.mu_e[0]);
      }
    }
    CK(cudaMemsetAsync(c->dflags, 0, 4 * kFlagInts, c->st));
    int hf[4] = {0, 0, 0, 0};
    const int nl = (int)c->lv.size();
    if (nl > kMaxLevels) throw ArgErr(SB_EINVAL, "too many multigrid levels");
    // constant-density levels (cflag slot 16 + kMaxLevels + l): the cell rows
    // use one 1/rho_face value instead of streaming the d beta arrays.  The
    // reference face: the first interior face of component `off`.
    std::vector<double> href(nl, 0.0);
    for (int l = 0; l < nl; ++l) {
      Level& L = c->lv[l];
      const int a0 = c->off;
      const long long st0 = a0 == 0 ? L.d.s0 : (a0 == 1 ? L.d.s1 : 1);
      const double* ref = L.rho_f[a0] + (c->bc[a0][0] != BC_PER ? st0 : 0);
      for (int A = c->off; A < 3; ++A)
        launch_beta(c->st, L.d, A, L.rho_f[A], L.beta_f[A], c->dflags + 2, c->dflags + 16 + kMaxLevels + l, ref);
      CK(cudaMemcpyAsync(&href[l], ref, 8, cudaMemcpyDeviceToHost, c->st));
    }
    for (size_t l = 0; l < c->lv.size(); ++l) launch_check_diag(c->st, c->lv[l].d, c->dim, c->form, c->dflags);
    // levels whose edge viscosities are the four-cell mean of mu_c: the face
    // rows derive them instead of streaming mu_e.  SB_MUE_DERIVED: 1 (default)
    // all-periodic levels and 3D levels with walls along the contiguous axis
    // only, 2 every wall-bounded level too (two-cell boundary means;
    // bit-compatible), 0 never
    const int derive_mode = [] {  // read per upload: tests compare the paths in one process
      const char* e = std::getenv("SB_MUE_DERIVED");
      return e ? std::atoi(e) : 1;
    }();
    // default: all-periodic levels and 3D levels whose only walls are along
    // the contiguous axis (C4) -- with the L2 prefetch of the derived-edge row
    // the walled row now beats the stored one (C4 256^3: 182 / 196 / 178 vs
    // 195 / 198 / 180 us per finest pass, solve 2.18 vs 2.22 s)
    const bool per_01 = c->bc[0][0] == BC_PER && c->bc[1][0] == BC_PER;
    const bool per_all = per_01 && c->bc[2][0] == BC_PER;
    const bool derive_on = derive_mode == 2 || (derive_mode == 1 && (per_all || (c->dim == 3 && per_01)));
    if (derive_on)
      for (int l = 0; l < nl; ++l) launch_check_mue(c->st, c->lv[l].d, c->dim, c->dflags + 16 + l);
    int hm[kFlagInts - 16];
    CK(cudaMemcpyAsync(hf, c->dflags, 16, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(hm, c->dflags + 16, 4 * (kFlagInts - 16), cudaMemcpyDeviceToHost, c->st));
    sync(c);
    const bool const_on = [] {  // SB_CONST_BETA=0: always stream the beta arrays
      const char* e = std::getenv("SB_CONST_BETA");
      return !(e && e[0] == '0');
    }();
    bool changed = false;
    for (int l = 0; l < nl; ++l) {
      LevelDev& d = c->lv[l].d;
      const int de = (derive_on && hm[l] == 0) ? 1 : 0;
      const int bc = (const_on && hm[kMaxLevels + l] == 0 && href[l] > 0.0) ? 1 : 0;
      const double bv = bc ? 1.0 / href[l] : 0.0;  // k_beta's expression
      changed |= de != d.mue_derived || bc != d.beta_const || bv != d.beta_val;
      d.mue_derived = de;
      d.beta_const = bc;
      d.beta_val = bv;
    }
    // the captured P^-1 graph and the coarse chains hold the LevelDev values
    if (changed) drop_graph(c);
    upload_chains(c);
    c->flag_face = hf[0] & 1;
    c->flag_cell = hf[1] & 1;
    c->flag_rho = hf[2] & 1;
    // operators.py:368-388 velocity_null_components
    c->null_comps.clear();
    if (c->theta == 0.0) {
      for (int A = c->off; A < 3; ++A) {
        if (c->bc[A][0] != BC_PER) continue;
        bool ok = true;
        for (int B = c->off; B < 3; ++B) {
          if (B == A) continue;
          const bool pb = c->bc[B][0] == BC_PER;
          const bool fs = c->bc[B][0] == BC_FREESLIP && c->bc[B][1] == BC_FREESLIP;
          if (!(pb || fs)) ok = false;
        }
        if (ok) c->null_comps.push_back(A);
      }
    }
}

}  // namespace

// ====================================================================================
// C ABI
// ====================================================================================

extern "C" {

const char* sb_last_error(void) { return g_err.c_str(); }

sb_ctx* sb_create(int dim, const int* cells, double h, const int* bc, int viscous_form) {
  sb_ctx* c = nullptr;
  int rc = guard([&]() -> int {
    if (dim != 2 && dim != 3) throw ArgErr(SB_EINVAL, "dim must be 2 or 3");
    if (!(h > 0)) throw ArgErr(SB_EINVAL, "grid spacing must be positive");
    if (viscous_form < 0 || viscous_form > 2) throw ArgErr(SB_EINVAL, "bad viscous form");
    c = new sb_ctx();
    c->dim = dim;
    c->form = viscous_form;
    c->off = 3 - dim;
    c->h = h;
    c->n[0] = 1;
    c->bc[0][0] = c->bc[0][1] = BC_PER;
    for (int r = 0; r < dim; ++r) {
      const int A = r + c->off;
      if (cells[r] < 2) throw ArgErr(SB_EINVAL, "cell counts must be >= 2");
      c->n[A] = cells[r];
      c->bc[A][0] = bc[2 * r];
      c->bc[A][1] = bc[2 * r + 1];
      if ((c->bc[A][0] == BC_PER) != (c->bc[A][1] == BC_PER))
        throw ArgErr(SB_EINVAL, "periodic must hold on both sides of an axis");
    }
    CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    c->own_st = c->st;
    int n[3] = {c->n[0], c->n[1], c->n[2]};
    double hh = h;
    make_level(c, n, hh);
    if (can_coarsen(n, dim)) {
      while (can_coarsen(n, dim)) {
        for (int a = c->off; a < 3; ++a) n[a] /= 2;
        hh *= 2.0;
        make_level(c, n, hh);
      }
    }
    for (size_t l = 0; l < c->lv.size(); ++l) alloc_level(c, c->lv[l], l == 0);
    {
      // pad-free level 0 (every axis periodic, contiguous extent a multiple of 4)
      const Level& L0 = c->lv[0];
      bool padfree = true;
      for (int a = 0; a < 3; ++a) padfree &= c->bc[a][0] == BC_PER && L0.P[a] == L0.d.n[a];
      const char* e = std::getenv("SB_DEFER_NULLS");
      c->defer_nulls = padfree && !(e && e[0] == '0');
    }
    int* fl = nullptr;
    CK(cudaMalloc(&fl, 4 * kFlagInts));
    c->allocs.push_back(fl);
    c->dflags = fl;
    c->dpart = dalloc(c, (long long)(2 * kMaxVec + 2) * reduce_blocks());
    c->dsmall = dalloc(c, 8 * kMaxVec);
    CK(cudaMallocHost(&c->hsmall, 8 * kMaxVec * 8));
    c->launches_base = g_kernel_launches;
    sync(c);
    return SB_OK;
  });
  if (rc != SB_OK) {
    if (c) sb_destroy(c);
    return nullptr;
  }
  return c;
}

void sb_destroy(sb_ctx* c) {
  if (!c) return;
  drop_graph(c);
  if (c->st) cudaStreamSynchronize(c->st);
  for (void* p : c->allocs) cudaFree(p);
  for (auto e : c->evpool) cudaEventDestroy(e);
  if (c->hsmall) cudaFreeHost(c->hsmall);
  if (c->hbig) cudaFreeHost(c->hbig);
  if (c->own_st) cudaStreamDestroy(c->own_st);
  delete c;
}

int sb_set_coefficients(sb_ctx* c, double theta, const double* const* rho_face, const double* mu_cell,
                        const double* const* mu_edge, const double* gamma_cell) {
  return guard([&]() -> int {
    if (!(theta >= 0)) throw ArgErr(SB_EINVAL, "theta must be >= 0");
    // the captured P^-1 graph holds buffer pointers and theta (kernel
    // parameters, null-space components); new coefficient VALUES in the same
    // buffers replay correctly, so only a theta change invalidates it
    if (!c->have_coef || theta != c->theta) drop_graph(c);
    c->theta = theta;
    for (auto& L : c->lv) L.d.theta = theta;
    Level& L0 = c->lv[0];
    copy_in(c, L0, -1, mu_cell, L0.mu_c);
    if (gamma_cell) copy_in(c, L0, -1, gamma_cell, L0.gam_c);
    else CK(cudaMemsetAsync(L0.gam_c, 0, L0.block * 8, c->st));
    for (int r = 0; r < c->dim; ++r) copy_in(c, L0, r + c->off, rho_face[r], L0.rho_f[r + c->off]);
    if (c->dim == 3) {
      // edge_planes order (0,1),(0,2),(1,2) -> normal axis 2,1,0
      copy_in(c, L0, 12, mu_edge[0], L0.mu_e[2]);
      copy_in(c, L0, 11, mu_edge[1], L0.mu_e[1]);
      copy_in(c, L0, 10, mu_edge[2], L0.mu_e[0]);
    } else {
      copy_in(c, L0, 10, mu_edge[0], L0.mu_e[0]);
    }
    build_from_level0(c);
    c->have_coef = true;
    return SB_OK;
  });
}

// Device-side make_coefficients (operators.py:107-125: face densities and
// node/edge viscosities averaged from the cells, :81-104) followed by rescale
// (operators.py:532-550 / cli.py:340-343: theta, mu, mu_e, gamma times
// `scale`; the edge means are formed from the unscaled mu and then scaled, the
// host's operation order, so every array equals the host path's to the bit).
// Uploads 2-3 cell arrays instead of 2 + d + (1|3).
int sb_set_cell_coefficients(sb_ctx* c, double theta, const double* rho_cell, const double* mu_cell,
                             const double* gamma_cell, double scale) {
  return guard([&]() -> int {
    if (!(theta >= 0)) throw ArgErr(SB_EINVAL, "theta must be >= 0");
    if (!(scale > 0)) throw ArgErr(SB_EINVAL, "scale must be > 0");
    const double th = scale * theta;
    if (!c->have_coef || th != c->theta) drop_graph(c);
    c->theta = th;
    for (auto& L : c->lv) L.d.theta = th;
    Level& L0 = c->lv[0];
    if (!c->cscratch) c->cscratch = dalloc(c, L0.block);
    copy_in(c, L0, -1, rho_cell, c->cscratch);
    for (int A = c->off; A < 3; ++A) launch_cell_to_face(c->st, L0.d, c->dim, A, c->cscratch, L0.rho_f[A]);
    copy_in(c, L0, -1, mu_cell, L0.mu_c);
    if (c->dim == 3) {
      for (int e = 0; e < 3; ++e) launch_cell_to_edge(c->st, L0.d, 3, e, L0.mu_e[e], scale);
    } else {
      launch_cell_to_edge(c->st, L0.d, 2, 0, L0.mu_e[0], scale);
    }
    launch_scale(c->st, L0.mu_c, scale, L0.block);
    if (gamma_cell) {
      copy_in(c, L0, -1, gamma_cell, L0.gam_c);
      launch_scale(c->st, L0.gam_c, scale, L0.block);
    } else {
      CK(cudaMemsetAsync(L0.gam_c, 0, L0.block * 8, c->st));
    }
    build_from_level0(c);
    c->have_coef = true;
    return SB_OK;
  });
}

int sb_apply_M(sb_ctx* c, const double* const* u, const double* p, double* const* out_u, double* out_p) {
  return guard([&]() -> int {
    check_ready(c);
    ensure_vectors(c);
    vec_in(c, u, p, c->vt, true);
    apply_M_vec(c, c->vt, c->vMv);
    vec_out(c, c->vMv, out_u, out_p);
    sync(c);
    return SB_OK;
  });
}

int sb_apply_A_affine(sb_ctx* c, const double* const* u, const double* const* tangential,
                      double* const* out_u) {
  return guard([&]() -> int {
    check_ready(c);
    ensure_scratch(c);
    const Level& L = c->lv[0];
    // wall-normal boundary faces are read as given (the boundary lift), as
    // the reference's apply_A does
    for (int r = 0; r < c->dim; ++r) copy_in(c, L, r + c->off, u[r], c->sf0[r + c->off]);
    CPtr3 x{{c->sf0[0], c->sf0[1], c->sf0[2]}}, none{{nullptr, nullptr, nullptr}};
    Ptr3 o{{c->sf1[0], c->sf1[1], c->sf1[2]}};
    launch_face_residual(c->st, L.d, c->dim, c->form, x, none, nullptr, o);
    if (tangential) wall_tangent(c, tangential, c->sf1);
    for (int r = 0; r < c->dim; ++r) copy_out(c, L, r + c->off, c->sf1[r + c->off], out_u[r]);
    sync(c);
    return SB_OK;
  });
}

int sb_apply_A(sb_ctx* c, const double* const* u, double* const* out_u) {
  return sb_apply_A_affine(c, u, nullptr, out_u);
}

// operators.py:484-512 homogenize
int sb_homogenize(sb_ctx* c, const double* const* normal, const double* const* tangential,
                  const double* const* rhs_u, const double* rhs_p, double* const* out_u, double* out_p) {
  return guard([&]() -> int {
    check_ready(c);
    ensure_scratch(c);
    const Level& L = c->lv[0];
    // u_b = boundary_lift(bvals) (operators.py:471-481)
    for (int r = 0; r < c->dim; ++r) {
      const int A = r + c->off;
      CK(cudaMemsetAsync(c->sf0[A], 0, L.block * 8, c->st));
      if (c->bc[A][0] == BC_PER || !normal) continue;
      for (int side = 0; side < 2; ++side)
        if (normal[2 * r + side]) copy_plane_in(c, L, A, A, side ? L.d.n[A] : 0, normal[2 * r + side], c->sf0[A]);
    }
    CK(cudaMemsetAsync(c->sc0, 0, L.block * 8, c->st));
    {
      CPtr3 ub{{c->sf0[0], c->sf0[1], c->sf0[2]}};
      Ptr3 o{{c->sf1[0], c->sf1[1], c->sf1[2]}};
      launch_apply_M(c->st, L.d, c->dim, c->form, ub, c->sc0, o, c->sc1);  // A u_b, -div(u_b)
    }
    if (tangential) wall_tangent(c, tangential, c->sf1);
    // compatibility of the boundary flux with the divergence source (:495-509)
    copy_in(c, L, -1, rhs_p, c->sc0);
    const int rb = reduce_blocks();
    launch_sum_abs_partial(c->st, c->sc1, L.block, c->dpart);
    launch_sum_abs_partial(c->st, c->sc0, L.block, c->dpart + 2 * rb);
    launch_finalize(c->st, c->dpart, 4, dmisc(c));
    CK(cudaMemcpyAsync(hmisc(c), dmisc(c), 4 * 8, cudaMemcpyDeviceToHost, c->st));
    sync(c);
    const double* hs = hmisc(c);
    const double hd = std::pow(c->h, (double)c->dim);
    const double flux = -hs[0] * hd;         // sum(div u_b) h^d
    const double source = -hs[2] * hd;
    const double scale = std::max(1.0, std::max(hs[1] * hd, hs[3] * hd));
    if (std::fabs(flux - source) > 1e-10 * scale) {
      char msg[160];
      std::snprintf(msg, sizeof msg, "incompatible boundary data: net boundary flux %g != divergence-source integral %g",
                    flux, source);
      throw ArgErr(SB_EINVAL, msg);
    }
    // (rhs.u - A u_b, rhs.p - (-div u_b)) over the full arrays
    for (int r = 0; r < c->dim; ++r) {
      const int A = r + c->off;
      copy_in(c, L, A, rhs_u[r], c->sf0[A]);
      launch_sub(c->st, c->sf0[A], c->sf1[A], c->sf0[A], L.block);
      copy_out(c, L, A, c->sf0[A], out_u[r]);
    }
    launch_sub(c->st, c->sc0, c->sc1, c->sc0, L.block);
    copy_out(c, L, -1, c->sc0, out_p);
    sync(c);
    return SB_OK;
  });
}

int sb_apply_Lrho(sb_ctx* c, const double* p, double* out_p) {
  return guard([&]() -> int {
    check_ready(c);
    if (c->flag_rho) throw ArgErr(SB_EINVAL, "face density must be positive");
    ensure_scratch(c);
    const Level& L = c->lv[0];
    copy_in(c, L, -1, p, c->sc0);
    launch_cell_residual(c->st, L.d, c->dim, c->sc0, nullptr, c->sc1);
    copy_out(c, L, -1, c->sc1, out_p);
    sync(c);
    return SB_OK;
  });
}

int sb_mg_solve(sb_ctx* c, int kind, const sb_smoother* sm, int n_cycles, const double* const* rhs,
                double* const* out) {
  return guard([&]() -> int {
    if (kind != SB_KIND_CELL && kind != SB_KIND_FACE) throw ArgErr(SB_EINVAL, "kind must be 'cell' or 'face'");
    if (n_cycles < 1) throw ArgErr(SB_EINVAL, "need at least one cycle");
    check_mg(c, kind);
    ensure_scratch(c);
    const Level& L = c->lv[0];
    if (kind == SB_KIND_CELL) {
      copy_in(c, L, -1, rhs[0], c->sc0);
      mg_cell(c, n_cycles, c->sc0, c->sc1, *sm);
      copy_out(c, L, -1, c->sc1, out[0]);
    } else {
      for (int r = 0; r < c->dim; ++r) {
        const int A = r + c->off;
        copy_in(c, L, A, rhs[r], c->sf0[A]);
        zero_wall_faces(c, L, A, c->sf0[A]);
      }
      mg_face(c, n_cycles, c->sf0, c->sf1, *sm);
      for (int r = 0; r < c->dim; ++r) copy_out(c, L, r + c->off, c->sf1[r + c->off], out[r]);
    }
    sync(c);
    return SB_OK;
  });
}

int sb_precond_apply(sb_ctx* c, const sb_precond* pc, const sb_smoother* sm, const double* const* r_u,
                     const double* r_p, double* const* x_u, double* x_p, long long* scalar_vcycles) {
  return guard([&]() -> int {
    if (pc->kind != SB_IDENTITY) {
      check_mg(c, SB_KIND_FACE);
      if (pc->kind == SB_P1 || c->theta > 0) check_mg(c, SB_KIND_CELL);
    } else {
      check_ready(c);
    }
    ensure_vectors(c);
    vec_in(c, r_u, r_p, c->vMv);
    precond_apply_graph(c, *pc, *sm);
    finish_projection(c, c->vw);
    vec_out(c, c->vw, x_u, x_p);
    sync(c);
    if (scalar_vcycles) *scalar_vcycles += precond_cost(c, *pc);
    return SB_OK;
  });
}

int sb_gmres_solve(sb_ctx* c, const sb_precond* pc, const sb_gmres* gc, const sb_smoother* sm,
                   const double* const* b_u, const double* b_p, double* const* x_u, double* x_p,
                   sb_history_row* rows, int max_rows, int* n_rows, int* status, long long* scalar_vcycles) {
  return guard([&]() -> int {
    long long dummy = 0;
    return gmres(c, *pc, *gc, *sm, b_u, b_p, x_u, x_p, rows, max_rows, n_rows, status,
                 scalar_vcycles ? scalar_vcycles : &dummy);
  });
}

int sb_level_flags(sb_ctx* c, int level) {
  if (!c || level < 0 || level >= (int)c->lv.size()) return -1;
  const LevelDev& d = c->lv[level].d;
  return (d.mue_derived ? SB_LEVEL_MUE_DERIVED : 0) | (d.beta_const ? SB_LEVEL_CONST_RHO : 0);
}

int sb_num_levels(sb_ctx* c) { return (int)c->lv.size(); }

int sb_level_cells(sb_ctx* c, int level, int* cells) {
  if (level < 0 || level >= (int)c->lv.size()) {
    g_err = "level out of range";
    return SB_EINVAL;
  }
  for (int r = 0; r < c->dim; ++r) cells[r] = c->lv[level].d.n[r + c->off];
  return SB_OK;
}

int sb_get_level_coefficients(sb_ctx* c, int level, double* const* rho_face, double* mu_cell,
                              double* const* mu_edge, double* gamma_cell) {
  return guard([&]() -> int {
    check_ready(c);
    if (level < 0 || level >= (int)c->lv.size()) throw ArgErr(SB_EINVAL, "level out of range");
    const Level& L = c->lv[level];
    if (mu_cell) copy_out(c, L, -1, L.mu_c, mu_cell);
    if (gamma_cell) copy_out(c, L, -1, L.gam_c, gamma_cell);
    if (rho_face)
      for (int r = 0; r < c->dim; ++r) copy_out(c, L, r + c->off, L.rho_f[r + c->off], rho_face[r]);
    if (mu_edge) {
      if (c->dim == 3) {
        copy_out(c, L, 12, L.mu_e[2], mu_edge[0]);
        copy_out(c, L, 11, L.mu_e[1], mu_edge[1]);
        copy_out(c, L, 10, L.mu_e[0], mu_edge[2]);
      } else {
        copy_out(c, L, 10, L.mu_e[0], mu_edge[0]);
      }
    }
    sync(c);
    return SB_OK;
  });
}

// level-l staging buffers for the component entry points
static void level_bufs(sb_ctx* c, int l, int kind, double** x, double** rhs) {
  Level& L = c->lv[l];
  ensure_scratch(c);
  for (int a = 0; a < 3; ++a) {
    if (kind == SB_KIND_FACE) {
      x[a] = l == 0 ? c->sf0[a] : L.fx[a];
      rhs[a] = l == 0 ? c->sf1[a] : L.frhs[a];
    } else {
      x[a] = l == 0 ? c->sc0 : L.cx;
      rhs[a] = l == 0 ? c->sc1 : L.crhs;
    }
  }
}

int sb_smooth(sb_ctx* c, int kind, int level, double omega, double* const* x, const double* const* rhs) {
  return guard([&]() -> int {
    check_mg(c, kind, false);  // one sweep needs no coarse level (smooth_face on any grid)
    if (level < 0 || level >= (int)c->lv.size()) throw ArgErr(SB_EINVAL, "level out of range");
    double *bx[3], *br[3];
    level_bufs(c, level, kind, bx, br);
    const Level& L = c->lv[level];
    if (kind == SB_KIND_FACE) {
      for (int r = 0; r < c->dim; ++r) {
        const int A = r + c->off;
        copy_in(c, L, A, x[r], bx[A]);
        copy_in(c, L, A, rhs[r], br[A]);
      }
      double* cur[3] = {bx[0], bx[1], bx[2]};
      sweep_face(c, level, cur, br, omega);
      for (int r = 0; r < c->dim; ++r) copy_out(c, L, r + c->off, cur[r + c->off], x[r]);
    } else {
      copy_in(c, L, -1, x[0], bx[0]);
      copy_in(c, L, -1, rhs[0], br[0]);
      double* cur = bx[0];
      sweep_cell(c, level, cur, br[0], omega);
      copy_out(c, L, -1, cur, x[0]);
    }
    sync(c);
    return SB_OK;
  });
}

int sb_residual_restrict(sb_ctx* c, int kind, int level, const double* const* x, const double* const* rhs,
                         double* const* coarse) {
  return guard([&]() -> int {
    check_mg(c, kind);
    if (level < 0 || level + 1 >= (int)c->lv.size()) throw ArgErr(SB_EINVAL, "level out of range");
    double *bx[3], *br[3];
    level_bufs(c, level, kind, bx, br);
    const Level& L = c->lv[level];
    Level& C = c->lv[level + 1];
    if (kind == SB_KIND_FACE) {
      for (int r = 0; r < c->dim; ++r) {
        const int A = r + c->off;
        copy_in(c, L, A, x[r], bx[A]);
        copy_in(c, L, A, rhs[r], br[A]);
      }
      CPtr3 xc{{bx[0], bx[1], bx[2]}};
      for (int A = c->off; A < 3; ++A)
        launch_face_resid_restrict(c->st, L.d, C.d, c->dim, c->form, A, xc, br[A], C.frhs[A]);
      for (int r = 0; r < c->dim; ++r) copy_out(c, C, r + c->off, C.frhs[r + c->off], coarse[r]);
    } else {
      copy_in(c, L, -1, x[0], bx[0]);
      copy_in(c, L, -1, rhs[0], br[0]);
      launch_cell_resid_restrict(c->st, L.d, C.d, c->dim, bx[0], br[0], C.crhs);
      copy_out(c, C, -1, C.crhs, coarse[0]);
    }
    sync(c);
    return SB_OK;
  });
}

int sb_prolong_add(sb_ctx* c, int kind, int level, const double* const* coarse, double* const* fine) {
  return guard([&]() -> int {
    check_ready(c);
    if (level < 0 || level + 1 >= (int)c->lv.size()) throw ArgErr(SB_EINVAL, "level out of range");
    double *bx[3], *br[3];
    level_bufs(c, level, kind, bx, br);
    const Level& L = c->lv[level];
    Level& C = c->lv[level + 1];
    if (kind == SB_KIND_FACE) {
      for (int r = 0; r < c->dim; ++r) {
        const int A = r + c->off;
        copy_in(c, C, A, coarse[r], C.fx[A]);
        copy_in(c, L, A, fine[r], bx[A]);
        launch_face_prolong_add(c->st, L.d, C.d, c->dim, A, C.fx[A], bx[A]);
        copy_out(c, L, A, bx[A], fine[r]);
      }
    } else {
      copy_in(c, C, -1, coarse[0], C.cx);
      copy_in(c, L, -1, fine[0], bx[0]);
      launch_cell_prolong_add(c->st, L.d, C.d, c->dim, C.cx, bx[0]);
      copy_out(c, L, -1, bx[0], fine[0]);
    }
    sync(c);
    return SB_OK;
  });
}

// ---- the reference's remaining public operators (operators.py:182-198,
// :396-439; multigrid.py:177-295; schur.py:59-78) on the device ----------------

static void zero_block(sb_ctx* c, const Level& L, double* p) { CK(cudaMemsetAsync(p, 0, (size_t)L.block * 8, c->st)); }

int sb_div(sb_ctx* c, const double* const* u, double* out) {
  return guard([&]() -> int {
    ensure_scratch(c);
    const Level& L = c->lv[0];
    for (int r = 0; r < c->dim; ++r) copy_in(c, L, r + c->off, u[r], c->sf0[r + c->off]);
    launch_div(c->st, L.d, c->dim, CPtr3{{c->sf0[0], c->sf0[1], c->sf0[2]}}, c->sc0);
    copy_out(c, L, -1, c->sc0, out);
    sync(c);
    return SB_OK;
  });
}

int sb_grad(sb_ctx* c, const double* p, double* const* out) {
  return guard([&]() -> int {
    ensure_scratch(c);
    const Level& L = c->lv[0];
    copy_in(c, L, -1, p, c->sc0);
    launch_grad(c->st, L.d, c->dim, c->sc0, Ptr3{{c->sf0[0], c->sf0[1], c->sf0[2]}});
    for (int r = 0; r < c->dim; ++r) copy_out(c, L, r + c->off, c->sf0[r + c->off], out[r]);
    sync(c);
    return SB_OK;
  });
}

// lap_pressure = div(grad(p)) (operators.py:201-203), the same two steps
int sb_lap_pressure(sb_ctx* c, const double* p, double* out) {
  return guard([&]() -> int {
    ensure_scratch(c);
    const Level& L = c->lv[0];
    copy_in(c, L, -1, p, c->sc0);
    launch_grad(c->st, L.d, c->dim, c->sc0, Ptr3{{c->sf0[0], c->sf0[1], c->sf0[2]}});
    launch_div(c->st, L.d, c->dim, CPtr3{{c->sf0[0], c->sf0[1], c->sf0[2]}}, c->sc1);
    copy_out(c, L, -1, c->sc1, out);
    sync(c);
    return SB_OK;
  });
}

int sb_diagonal(sb_ctx* c, int kind, int level, double* const* out) {
  return guard([&]() -> int {
    check_ready(c);
    if (kind != SB_KIND_CELL && kind != SB_KIND_FACE) throw ArgErr(SB_EINVAL, "kind must be 'cell' or 'face'");
    if (level < 0 || level >= (int)c->lv.size()) throw ArgErr(SB_EINVAL, "level out of range");
    double *bx[3], *br[3];
    level_bufs(c, level, kind, bx, br);
    const Level& L = c->lv[level];
    if (kind == SB_KIND_FACE) {
      launch_write_diag(c->st, L.d, c->dim, c->form, Ptr3{{bx[0], bx[1], bx[2]}}, nullptr);
      for (int r = 0; r < c->dim; ++r) copy_out(c, L, r + c->off, bx[r + c->off], out[r]);
    } else {
      launch_write_diag(c->st, L.d, c->dim, c->form, Ptr3{{nullptr, nullptr, nullptr}}, bx[0]);
      copy_out(c, L, -1, bx[0], out[0]);
    }
    sync(c);
    return SB_OK;
  });
}

// S~^-1 r = -theta phi + V r (phi = the Poisson solve of r; NULL: steady, V r)
int sb_schur_inv(sb_ctx* c, const double* r, const double* phi, double* out) {
  return guard([&]() -> int {
    check_ready(c);
    ensure_scratch(c);
    const Level& L = c->lv[0];
    copy_in(c, L, -1, r, c->sc0);
    if (phi) copy_in(c, L, -1, phi, c->sc1);
    launch_schur(c->st, L.d, c->form, c->sc0, phi ? c->sc1 : nullptr, c->sf0[2], 1.0);
    copy_out(c, L, -1, c->sf0[2], out);
    sync(c);
    return SB_OK;
  });
}

// pure restriction / prolongation between levels `level` and `level + 1`
int sb_restrict(sb_ctx* c, int kind, int level, const double* const* fine, double* const* coarse) {
  return guard([&]() -> int {
    if (kind != SB_KIND_CELL && kind != SB_KIND_FACE) throw ArgErr(SB_EINVAL, "kind must be 'cell' or 'face'");
    if (level < 0 || level + 1 >= (int)c->lv.size()) throw ArgErr(SB_EINVAL, "level out of range");
    double *fx[3], *fr[3], *cx[3], *cr[3];
    level_bufs(c, level, kind, fx, fr);
    level_bufs(c, level + 1, kind, cx, cr);
    const Level& L = c->lv[level];
    const Level& C = c->lv[level + 1];
    if (kind == SB_KIND_FACE) {
      for (int r = 0; r < c->dim; ++r) {
        const int A = r + c->off;
        copy_in(c, L, A, fine[r], fx[A]);
        zero_block(c, C, cr[A]);  // coarse wall faces stay 0
        launch_face_restrict(c->st, L.d, C.d, c->dim, A, fx[A], cr[A]);
        copy_out(c, C, A, cr[A], coarse[r]);
      }
    } else {
      copy_in(c, L, -1, fine[0], fx[0]);
      launch_cell_restrict(c->st, L.d, C.d, c->dim, fx[0], cr[0]);
      copy_out(c, C, -1, cr[0], coarse[0]);
    }
    sync(c);
    return SB_OK;
  });
}

int sb_prolong(sb_ctx* c, int kind, int level, const double* const* coarse, double* const* fine) {
  return guard([&]() -> int {
    if (kind != SB_KIND_CELL && kind != SB_KIND_FACE) throw ArgErr(SB_EINVAL, "kind must be 'cell' or 'face'");
    if (level < 0 || level + 1 >= (int)c->lv.size()) throw ArgErr(SB_EINVAL, "level out of range");
    double *fx[3], *fr[3], *cx[3], *cr[3];
    level_bufs(c, level, kind, fx, fr);
    level_bufs(c, level + 1, kind, cx, cr);
    const Level& L = c->lv[level];
    const Level& C = c->lv[level + 1];
    if (kind == SB_KIND_FACE) {
      for (int r = 0; r < c->dim; ++r) {
        const int A = r + c->off;
        copy_in(c, C, A, coarse[r], cx[A]);
        zero_block(c, L, fx[A]);
        launch_face_prolong_add(c->st, L.d, C.d, c->dim, A, cx[A], fx[A]);
        copy_out(c, L, A, fx[A], fine[r]);
      }
    } else {
      copy_in(c, C, -1, coarse[0], cx[0]);
      zero_block(c, L, fx[0]);
      launch_cell_prolong_add(c->st, L.d, C.d, c->dim, cx[0], fx[0]);
      copy_out(c, L, -1, fx[0], fine[0]);
    }
    sync(c);
    return SB_OK;
  });
}

void sb_set_profiling(sb_ctx* c, int enabled) { c->profiling = enabled != 0; }

int sb_get_kernel_stats(sb_ctx* c, sb_kernel_stats* out) {
  *out = c->stats;
  return SB_OK;
}

long long sb_launch_count(sb_ctx* c) { return (g_kernel_launches - c->launches_base) + c->graph_launches; }

void sb_set_graphs(sb_ctx* c, int enabled) {
  c->use_graphs = enabled != 0;
  if (!c->use_graphs) drop_graph(c);
}

long long sb_device_bytes(sb_ctx* c) { return c->bytes; }

void* sb_host_alloc(long long bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, (size_t)bytes) != cudaSuccess) {
    g_err = "cudaMallocHost failed";
    return nullptr;
  }
  return p;
}

void sb_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int sb_set_stream(sb_ctx* c, void* stream) {
  return guard([&]() -> int {
    sync(c);
    cudaStream_t s = stream ? (cudaStream_t)stream : c->own_st;
    if (s != c->st) drop_graph(c);
    c->st = s;
    return SB_OK;
  });
}

}  // extern "C"

// slab-decomposed multi-GPU path (shares this translation unit)
#include "sb_dist.inc"

// gmres_kernel seam: flat vectors, host operator callback (shares this translation unit)
#include "sb_flat.inc"
