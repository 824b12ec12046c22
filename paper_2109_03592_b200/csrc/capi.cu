// C ABI (include/sbx.h): context lifetime, data upload/re-layout, operator
// entry points and the two PCG drivers (EXACT: the reference's pcg loop with
// device operators; FAST: fused kernels with device-resident scalars).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "cg.cuh"
#include "pressure.cuh"
#include "kernels.cuh"
#include "sbx_internal.h"

namespace sbx {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

}  // namespace sbx

using namespace sbx;

#define SBX_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t _e = (call);                                                        \
    if (_e != cudaSuccess) {                                                        \
      set_error(std::string(#call) + ": " + cudaGetErrorString(_e));                \
      return SBX_E_CUDA;                                                            \
    }                                                                               \
  } while (0)

#define SBX_TRY(call)                     \
  do {                                    \
    sbx_status _s = (sbx_status)(call);   \
    if (_s != SBX_OK) return _s;          \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct sbx_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  cudaStream_t caller = nullptr;  // stream the caller's inputs were produced on
  cudaEvent_t order_ev = nullptr;
  OpDev op;
  int64_t global_count = 0;
  bool interior_clean = false;  // every element-interior node: unmasked singleton
  bool has_mask = false;
  std::vector<void*> allocs;
  int64_t device_bytes = 0;
  // host copies kept for re-layout queries
  // scratch
  double* work[10] = {};  // nodes-sized
  double* partials = nullptr;
  int64_t partials_len = 0;
  double* dscal = nullptr;   // 16 device doubles
  uint32_t* dcount = nullptr;
  double* hscal = nullptr;   // pinned 16 doubles
  // Jacobi diagonal cache
  double* ddiag = nullptr;
  double* ddinv = nullptr;
  double diag_h1 = NAN, diag_h2 = NAN;
  double* h1f = nullptr;  // per-node coefficients (sbx_ctx_set_coeff_fields)
  double* h2f = nullptr;
  // fast CG
  std::unique_ptr<CgEngine> cg;
  // consistent-Poisson pressure operator (built on first use)
  std::unique_ptr<PressureEngine> pe;
  // distributed (filled by sbx_ctx_create_box_dist)
  std::vector<int64_t> local_elements;
  bool dist = false;
  bool connected = false;
  int nranks = 1, rank = 0;
  DistDev dd;
  void* window = nullptr;
  std::vector<int64_t> recv_base_for_src;  // per source rank, -1 if not a neighbour
  std::vector<void*> peer_windows;
  double* dgllx = nullptr;  // GLL nodes on the device (advect)
  // timing
  bool timing = false;
  // a multi-GPU exchange timed out: the per-phase sequence counters of the
  // ranks are out of step, so every later call is refused (recreate the
  // context on every rank)
  bool poisoned = false;
};

namespace {

sbx_status dalloc(sbx_ctx* c, void** p, size_t bytes) {
  if (bytes == 0) bytes = 8;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) {
    set_error(std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? SBX_E_NOMEM : SBX_E_CUDA;
  }
  c->allocs.push_back(*p);
  c->device_bytes += (int64_t)bytes;
  return SBX_OK;
}

template <typename T>
sbx_status dupload(sbx_ctx* c, T** out, const T* host, int64_t count) {
  void* p = nullptr;
  SBX_TRY(dalloc(c, &p, sizeof(T) * (size_t)count));
  if (host && count > 0)
    SBX_CUDA(cudaMemcpyAsync(p, host, sizeof(T) * (size_t)count, cudaMemcpyHostToDevice,
                             c->stream));
  *out = static_cast<T*>(p);
  return SBX_OK;
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

sbx_status work(sbx_ctx* c, int slot, double** out) {
  if (!c->work[slot]) {
    void* p = nullptr;
    SBX_TRY(dalloc(c, &p, sizeof(double) * (size_t)c->op.nodes));
    c->work[slot] = static_cast<double*>(p);
  }
  *out = c->work[slot];
  return SBX_OK;
}

// Input/output staging: device pointers pass through, host pointers are copied
// through a context work buffer.
struct In {
  const double* d = nullptr;
};
sbx_status stage_in(sbx_ctx* c, const double* p, int slot, const double** out) {
  if (is_device_ptr(p)) {
    *out = p;
    return SBX_OK;
  }
  double* w = nullptr;
  SBX_TRY(work(c, slot, &w));
  SBX_CUDA(cudaMemcpyAsync(w, p, sizeof(double) * (size_t)c->op.nodes, cudaMemcpyHostToDevice,
                           c->stream));
  *out = w;
  return SBX_OK;
}

// Every entry point runs on the context's own (capturable, non-blocking)
// stream, ordered after all work already queued on the caller's stream
// (default: the legacy default stream, i.e. torch's default stream).
sbx_status enter(sbx_ctx* c) {
  if (c->poisoned) {
    set_error("context unusable after a multi-GPU exchange timeout; recreate it on every rank");
    return SBX_E_COMM;
  }
  SBX_CUDA(cudaSetDevice(c->device));
  SBX_CUDA(cudaEventRecord(c->order_ev, c->caller));
  SBX_CUDA(cudaStreamWaitEvent(c->stream, c->order_ev, 0));
  return SBX_OK;
}

sbx_status finish(sbx_ctx* c) {
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    set_error(std::string("kernel execution: ") + cudaGetErrorString(e));
    return SBX_E_CUDA;
  }
  if (c->dist && c->dd.status) {
    // an exchange kernel (halo or scalar all-reduce) timed out on this rank
    int st = 0;
    SBX_CUDA(cudaMemcpy(&st, c->dd.status, sizeof(int), cudaMemcpyDeviceToHost));
    if (st) {
      c->poisoned = true;
      set_error("multi-GPU exchange timed out (a peer rank stopped responding); "
                "the context is unusable, recreate it on every rank");
      return SBX_E_COMM;
    }
  }
  return SBX_OK;
}

// Boundary CSR: all groups except element-interior unmasked singletons.
sbx_status build_boundary_csr(sbx_ctx* c, const int64_t* offsets, const int64_t* nodes,
                              const double* mask) {
  const int n = c->op.n;
  const int64_t n3 = (int64_t)n * n * n, N = c->op.nodes, G = c->global_count;
  if (offsets[0] != 0 || offsets[G] != N) {
    set_error("gather-scatter map: group_offsets must start at 0 and end at E*n^3");
    return SBX_E_SHAPE;
  }
  if (N >= (int64_t)INT32_MAX) {
    set_error("gather-scatter map: more than 2^31-1 local nodes per device");
    return SBX_E_SHAPE;
  }
  std::vector<uint8_t> seen(N, 0);
  auto on_boundary = [&](int64_t a) {
    const int64_t l = a % n3;
    const int i = (int)(l % n), j = (int)((l / n) % n), k = (int)(l / ((int64_t)n * n));
    return i == 0 || j == 0 || k == 0 || i == n - 1 || j == n - 1 || k == n - 1;
  };
  std::vector<int32_t> off;
  std::vector<int32_t> idx;
  off.reserve(G / 2 + 2);
  idx.reserve(N * 6 / 10 + 16);
  off.push_back(0);
  bool clean = true;
  std::vector<uint8_t> mult8(N, 0);
  std::vector<double> inv_mult(N, 0.0);
  for (int64_t g = 0; g < G; ++g) {
    const int64_t lo = offsets[g], hi = offsets[g + 1];
    if (hi <= lo || lo < 0 || hi > N) {
      set_error("gather-scatter map: empty or out-of-range group " + std::to_string(g));
      return SBX_E_SHAPE;
    }
    bool keep = hi - lo > 1;
    for (int64_t q = lo; q < hi; ++q) {
      const int64_t a = nodes[q];
      if (a < 0 || a >= N || seen[a]) {
        set_error("gather-scatter map: group_nodes is not a permutation of the local nodes");
        return SBX_E_SHAPE;
      }
      seen[a] = 1;
      const bool masked = mask && mask[a] == 0.0;
      if (masked || on_boundary(a)) keep = true;
      if (!on_boundary(a) && (masked || hi - lo > 1)) clean = false;
      mult8[a] = (uint8_t)std::min<int64_t>(hi - lo, 255);
      inv_mult[a] = 1.0 / (double)(int32_t)(hi - lo);
    }
    if (!keep) continue;
    for (int64_t q = lo; q < hi; ++q) {
      const int64_t a = nodes[q];
      const bool masked = mask && mask[a] == 0.0;
      idx.push_back(masked ? ~(int32_t)a : (int32_t)a);
    }
    off.push_back((int32_t)idx.size());
  }
  c->interior_clean = clean;
  c->op.nB = (int64_t)off.size() - 1;
  c->op.nBcopies = (int64_t)idx.size();
  int32_t *doff = nullptr, *didx = nullptr;
  SBX_TRY(dupload(c, &doff, off.data(), (int64_t)off.size()));
  SBX_TRY(dupload(c, &didx, idx.data(), (int64_t)idx.size()));
  c->op.b_off = doff;
  c->op.b_idx = didx;
  uint8_t* dm8 = nullptr;
  double* dim = nullptr;
  SBX_TRY(dupload(c, &dm8, mult8.data(), N));
  SBX_TRY(dupload(c, &dim, inv_mult.data(), N));
  c->op.mult8 = dm8;
  c->op.inv_mult = dim;
  SBX_CUDA(cudaStreamSynchronize(c->stream));  // host vectors die here
  return SBX_OK;
}

sbx_status ctx_init_common(sbx_ctx* c, int device) {
  c->device = device;
  SBX_CUDA(cudaSetDevice(device));
  SBX_CUDA(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
  c->stream = c->own_stream;
  SBX_CUDA(cudaEventCreateWithFlags(&c->order_ev, cudaEventDisableTiming));
  void* p = nullptr;
  SBX_TRY(dalloc(c, &p, 64 * sizeof(double)));
  c->dscal = static_cast<double*>(p);
  SBX_TRY(dalloc(c, &p, 64 * sizeof(uint32_t)));
  c->dcount = static_cast<uint32_t*>(p);
  SBX_CUDA(cudaMemsetAsync(c->dcount, 0, 64 * sizeof(uint32_t), c->stream));
  SBX_CUDA(cudaMallocHost(&c->hscal, 64 * sizeof(double)));
  return SBX_OK;
}

sbx_status ensure_partials(sbx_ctx* c, int64_t count) {
  if (c->partials_len >= count) return SBX_OK;
  void* p = nullptr;
  SBX_TRY(dalloc(c, &p, sizeof(double) * (size_t)count));
  c->partials = static_cast<double*>(p);
  c->partials_len = count;
  return SBX_OK;
}

// Trilinear-element data for the fused CG kernel's on-the-fly metrics: the
// per-element map coefficients and the GLL nodes / weights.
sbx_status upload_trilinear(sbx_ctx* c, int degree, const double* corners, int64_t E) {
  std::vector<double> tl(E * 24);
  trilinear_coeffs(E, corners, tl.data());
  double* dtl = nullptr;
  SBX_TRY(dupload(c, &dtl, tl.data(), E * 24));
  c->op.tl = dtl;
  double* dcr = nullptr;  // the corners themselves (EXACT pressure geometry)
  SBX_TRY(dupload(c, &dcr, corners, E * 24));
  c->op.corners = dcr;
  SBX_TRY(sbx_gll_basis(degree, c->op.Xh, c->op.Wh, nullptr));
  return SBX_OK;
}


// Structured-box hint of sbx_problem_desc: verify on the device that the
// caller's map and mask are the lattice's (and the geometry the corners'
// trilinear metric); if so switch the context to the lattice gather-scatter
// (no CSR) and, with verified corners, the trilinear K1.  *lattice = false
// (and nothing changed) when the hint is absent or does not match.
sbx_status try_box_hint(sbx_ctx* c, const sbx_problem_desc* d, bool* lattice) {
  *lattice = false;
  const int64_t E = c->op.E, N = c->op.nodes;
  if (d->box[0] <= 0 || d->box[1] <= 0 || d->box[2] <= 0 || !d->mask) return SBX_OK;
  if ((int64_t)d->box[0] * d->box[1] * d->box[2] != E) return SBX_OK;
  if (std::getenv("SBX_HOST_SETUP") || N >= (int64_t)INT32_MAX) return SBX_OK;
  OpDev probe = c->op;
  probe.ex = d->box[0];
  probe.ey = d->box[1];
  probe.ez = d->box[2];
  int64_t G = 1;
  const int n = c->op.n;
  for (int q = 0; q < 3; ++q) {
    probe.per[q] = d->periodic[q] ? 1 : 0;
    if (probe.per[q] && d->box[q] < 2) return SBX_OK;  // lattice gs needs 2 cells
    const int64_t span = (int64_t)d->box[q] * (n - 1);
    G *= probe.per[q] ? span : span + 1;
  }
  if (G != d->global_count || d->group_offsets[0] != 0 || d->group_offsets[G] != N)
    return SBX_OK;
  int* flag = reinterpret_cast<int*>(c->dcount) + 8;
  SBX_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), c->stream));
  {
    int64_t *doff = nullptr, *didx = nullptr;
    SBX_CUDA(cudaMalloc(&doff, sizeof(int64_t) * (size_t)(G + 1)));
    SBX_CUDA(cudaMalloc(&didx, sizeof(int64_t) * (size_t)N));
    SBX_CUDA(cudaMemcpyAsync(doff, d->group_offsets, sizeof(int64_t) * (size_t)(G + 1),
                             cudaMemcpyHostToDevice, c->stream));
    SBX_CUDA(cudaMemcpyAsync(didx, d->group_nodes, sizeof(int64_t) * (size_t)N,
                             cudaMemcpyHostToDevice, c->stream));
    SBX_CUDA(launch_validate_box(probe, G, doff, didx, c->op.mask, flag, c->stream));
    SBX_CUDA(cudaStreamSynchronize(c->stream));
    cudaFree(doff);
    cudaFree(didx);
  }
  int bad = 0;
  SBX_CUDA(cudaMemcpy(&bad, flag, sizeof(int), cudaMemcpyDeviceToHost));
  if (bad) return SBX_OK;
  // the map / mask are the lattice's: lattice gather-scatter, no CSR
  double* im = nullptr;
  uint8_t* m8 = nullptr;
  SBX_TRY(dupload<double>(c, &im, nullptr, N));
  SBX_TRY(dupload<uint8_t>(c, &m8, nullptr, N));
  SBX_CUDA(launch_lattice_fields(probe, nullptr, im, m8, c->stream));
  c->op = probe;
  c->op.box = true;
  c->op.lat = true;
  c->op.inv_mult = im;
  c->op.mult8 = m8;
  c->op.nB = 0;
  c->op.nBcopies = 0;
  c->interior_clean = true;
  *lattice = true;
  // geometry from the corners (trilinear K1) only if it is bitwise the
  // caller's g1..g6 / bm
  if (d->corners) {
    std::vector<double> x(n), w(n);
    SBX_TRY(sbx_gll_basis(n - 1, x.data(), w.data(), nullptr));
    double* dcr = nullptr;
    SBX_CUDA(cudaMalloc(&dcr, sizeof(double) * (size_t)E * 24));
    SBX_CUDA(cudaMemcpyAsync(dcr, d->corners, sizeof(double) * (size_t)E * 24,
                             cudaMemcpyHostToDevice, c->stream));
    SBX_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), c->stream));
    SBX_CUDA(launch_validate_geom(dcr, E, n, x.data(), w.data(), c->op.G, c->op.bm, flag,
                                  c->stream));
    SBX_CUDA(cudaStreamSynchronize(c->stream));
    cudaFree(dcr);
    SBX_CUDA(cudaMemcpy(&bad, flag, sizeof(int), cudaMemcpyDeviceToHost));
    if (!bad) SBX_TRY(upload_trilinear(c, n - 1, d->corners, E));
  }
  return SBX_OK;
}

// Upload the problem (reference layout host arrays) and re-lay it out.
sbx_status ctx_upload(sbx_ctx* c, const sbx_problem_desc* d) {
  const int n = d->degree + 1;
  c->op.E = d->elem_count;
  c->op.n = n;
  c->op.nodes = d->elem_count * (int64_t)n * n * n;
  c->global_count = d->global_count;
  for (int q = 0; q < n * n; ++q) c->op.Dh[q] = d->deriv[q];
  double* dD = nullptr;
  SBX_TRY(dupload(c, &dD, d->deriv, (int64_t)n * n));
  c->op.Dd = dD;
  const int64_t N = c->op.nodes;
  // geometry: stage each SoA array once and pack to [E][6][n^3]
  double* G = nullptr;
  SBX_TRY(dupload<double>(c, &G, nullptr, 6 * N));
  {
    double* tmp[6] = {};
    for (int q = 0; q < 6; ++q) {
      SBX_CUDA(cudaMalloc(&tmp[q], sizeof(double) * (size_t)std::max<int64_t>(N, 1)));
      SBX_CUDA(cudaMemcpyAsync(tmp[q], d->g[q], sizeof(double) * (size_t)N,
                               cudaMemcpyHostToDevice, c->stream));
    }
    OpDev tmpop = c->op;
    SBX_CUDA(launch_pack_geometry(tmpop, tmp, G, c->stream));
    SBX_CUDA(cudaStreamSynchronize(c->stream));
    for (int q = 0; q < 6; ++q) cudaFree(tmp[q]);
  }
  c->op.G = G;
  if (d->bm) {
    double* bm = nullptr;
    SBX_TRY(dupload(c, &bm, d->bm, N));
    c->op.bm = bm;
  }
  if (d->mask) {
    double* m = nullptr;
    SBX_TRY(dupload(c, &m, d->mask, N));
    c->op.mask = m;
    c->has_mask = true;
  }
  bool lattice = false;
  SBX_TRY(try_box_hint(c, d, &lattice));
  if (!lattice) SBX_TRY(build_boundary_csr(c, d->group_offsets, d->group_nodes, d->mask));
  SBX_TRY(ensure_partials(c, std::max<int64_t>(c->op.E, 4096)));
  c->cg.reset(new CgEngine());
  return SBX_OK;
}

sbx_status check_ctx(const sbx_ctx* c) {
  if (!c) {
    set_error("null context");
    return SBX_E_INVALID;
  }
  return SBX_OK;
}

// ---- scalar helpers for the EXACT driver ---------------------------------
sbx_status dot_exact(sbx_ctx* c, const double* a, const double* b, bool weighted, double* out) {
  SBX_CUDA(launch_dot_exact(c->op, a, b, weighted ? c->op.inv_mult : nullptr, c->partials,
                            c->dscal, c->stream));
  SBX_CUDA(cudaMemcpyAsync(c->hscal, c->dscal, sizeof(double), cudaMemcpyDeviceToHost,
                           c->stream));
  SBX_TRY(finish(c));
  *out = c->hscal[0];
  return SBX_OK;
}

// gather-scatter of a device field: local boundary CSR, plus the peer
// exchange and interface groups on a distributed context
sbx_status gs_dev(sbx_ctx* c, double* f, bool apply_mask) {
  if (c->dist) {
    if (!c->connected) {
      set_error("distributed context used before sbx_ctx_dist_connect");
      return SBX_E_COMM;
    }
    SBX_CUDA(launch_dist_gs(c->op, c->dd, f, apply_mask && c->has_mask, c->stream));
  } else {
    SBX_CUDA(launch_gs(c->op, f, apply_mask && c->has_mask, c->stream));
  }
  return SBX_OK;
}

sbx_status apply_dev(sbx_ctx* c, const double* x, double* q, double h1, double h2,
                     bool exact, bool flip, bool use_mask) {
  SBX_CUDA(launch_axhelm(c->op, x, q, h1, h2, exact, flip, c->stream));
  return gs_dev(c, q, use_mask);
}

sbx_status ensure_diag(sbx_ctx* c, double h1, double h2) {
  if (c->ddiag && c->diag_h1 == h1 && c->diag_h2 == h2) return SBX_OK;
  if (!c->ddiag) {
    void* p = nullptr;
    SBX_TRY(dalloc(c, &p, sizeof(double) * (size_t)c->op.nodes));
    c->ddiag = static_cast<double*>(p);
    SBX_TRY(dalloc(c, &p, sizeof(double) * (size_t)c->op.nodes));
    c->ddinv = static_cast<double*>(p);
  }
  SBX_CUDA(launch_axhelm_diag(c->op, h1, h2, c->ddiag, c->stream));
  SBX_TRY(gs_dev(c, c->ddiag, false));
  SBX_CUDA(launch_recip(c->op.nodes, c->ddiag, c->ddinv, c->stream));
  c->diag_h1 = h1;
  c->diag_h2 = h2;
  return SBX_OK;
}

sbx_status ensure_diag_if(sbx_ctx* c, const sbx_pcg_config* cfg) {
  if (cfg->precond == SBX_PRECOND_JACOBI) return ensure_diag(c, cfg->h1, cfg->h2);
  return SBX_OK;
}

// ---- EXACT PCG: krylov.cpp:7-91 statement by statement ------------------
sbx_status pcg_exact(sbx_ctx* c, const double* b, double* x, const sbx_pcg_config* cfg,
                     sbx_pcg_result* res) {
  const int64_t N = c->op.nodes;
  cudaStream_t s = c->stream;
  auto push = [&](double v) {
    if (cfg->history && res->history_length < cfg->history_capacity)
      cfg->history[res->history_length] = v;
    ++res->history_length;
  };
  double bb;
  SBX_TRY(dot_exact(c, b, b, true, &bb));
  if (bb == 0.0) {
    SBX_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * (size_t)N, s));
    res->converged = 1;
    return finish(c);
  }
  const double bnorm = std::sqrt(bb);
  double *r, *z, *q, *p;
  SBX_TRY(work(c, 2, &r));
  SBX_TRY(work(c, 3, &z));
  SBX_TRY(work(c, 4, &q));
  SBX_TRY(work(c, 5, &p));
  SBX_CUDA(cudaMemcpyAsync(r, b, sizeof(double) * (size_t)N, cudaMemcpyDeviceToDevice, s));
  // zero-guess test (krylov.cpp:22-28): any x != 0
  SBX_CUDA(launch_dot_fast(N, x, x, nullptr, c->partials, c->dcount, c->dscal, s));
  SBX_CUDA(cudaMemcpyAsync(c->hscal, c->dscal, sizeof(double), cudaMemcpyDeviceToHost, s));
  SBX_TRY(finish(c));
  // x.x == 0 can underflow for tiny nonzero entries; confirm with an exact scan
  bool zero_guess = c->hscal[0] == 0.0;
  if (zero_guess) {
    std::vector<double> hx(N);
    SBX_CUDA(cudaMemcpy(hx.data(), x, sizeof(double) * (size_t)N, cudaMemcpyDeviceToHost));
    for (double v : hx)
      if (v != 0.0) {
        zero_guess = false;
        break;
      }
  }
  if (!zero_guess) {
    SBX_TRY(apply_dev(c, x, q, cfg->h1, cfg->h2, true, false, true));
    SBX_CUDA(launch_axpy(N, -1.0, q, r, s));
  }
  const bool jacobi = cfg->precond == SBX_PRECOND_JACOBI;
  if (jacobi) SBX_TRY(ensure_diag(c, cfg->h1, cfg->h2));
  auto precond = [&](const double* in, double* out) -> sbx_status {
    if (jacobi)
      SBX_CUDA(launch_div(N, in, c->ddiag, out, s));
    else
      SBX_CUDA(cudaMemcpyAsync(out, in, sizeof(double) * (size_t)N, cudaMemcpyDeviceToDevice, s));
    return SBX_OK;
  };
  SBX_TRY(precond(b, z));
  double bmb;
  SBX_TRY(dot_exact(c, b, z, true, &bmb));
  SBX_TRY(precond(r, z));
  double rz, rr;
  SBX_TRY(dot_exact(c, r, z, true, &rz));
  SBX_TRY(dot_exact(c, r, r, true, &rr));
  double rnorm = std::sqrt(rr);
  push(rnorm / bnorm);
  SBX_CUDA(cudaMemcpyAsync(p, z, sizeof(double) * (size_t)N, cudaMemcpyDeviceToDevice, s));
  for (int it = 0; it < cfg->max_iterations; ++it) {
    res->rel_residual = rnorm / bnorm;
    res->rel_residual_precond = bmb > 0.0 ? std::sqrt(std::max(rz, 0.0) / bmb) : 0.0;
    if (res->rel_residual <= cfg->tolerance && res->rel_residual_precond <= cfg->tolerance) {
      res->converged = 1;
      return finish(c);
    }
    SBX_TRY(apply_dev(c, p, q, cfg->h1, cfg->h2, true, false, true));
    double pq;
    SBX_TRY(dot_exact(c, p, q, true, &pq));
    if (!std::isfinite(pq) || pq <= 0.0) {
      res->error_iteration = it;
      set_error("pcg: breakdown (p'Ap = " + std::to_string(pq) + ") at iteration " +
                std::to_string(it));
      return SBX_E_BREAKDOWN;
    }
    const double alpha = rz / pq;
    SBX_CUDA(launch_axpy(N, alpha, p, x, s));
    SBX_CUDA(launch_axpy(N, -alpha, q, r, s));
    SBX_TRY(precond(r, z));
    double rz_new;
    SBX_TRY(dot_exact(c, r, z, true, &rz_new));
    SBX_TRY(dot_exact(c, r, r, true, &rr));
    rnorm = std::sqrt(rr);
    if (!std::isfinite(rnorm) || !std::isfinite(rz_new)) {
      res->error_iteration = it;
      set_error("pcg: residual diverged (NaN/Inf) at iteration " + std::to_string(it));
      return SBX_E_NAN;
    }
    push(rnorm / bnorm);
    ++res->iterations;
    const double beta = rz_new / rz;
    rz = rz_new;
    SBX_CUDA(launch_scale(N, beta, p, s));
    SBX_CUDA(launch_axpy(N, 1.0, z, p, s));
  }
  res->rel_residual = rnorm / bnorm;
  res->rel_residual_precond = bmb > 0.0 ? std::sqrt(std::max(rz, 0.0) / bmb) : 0.0;
  res->converged = res->rel_residual <= cfg->tolerance &&
                   res->rel_residual_precond <= cfg->tolerance;
  return finish(c);
}

}  // namespace

// =========================================================================
extern "C" {

const char* sbx_last_error(void) { return g_last_error.c_str(); }
const char* sbx_version(void) { return "sbx 0.1 (sm_100a)"; }

sbx_status sbx_gll_basis(int degree, double* nodes, double* weights, double* deriv) {
  const int rc = gll_basis(degree, nodes, weights, deriv);
  if (rc) set_error("build_gll_basis: degree must be in [1,32], got " + std::to_string(degree));
  return (sbx_status)rc;
}

sbx_status sbx_box_corners(int ex, int ey, int ez, const double origin[3],
                           const double lengths[3], double* corners) {
  const int rc = box_corners(ex, ey, ez, origin, lengths, corners);
  if (rc) set_error("build_box_mesh: element counts must be >= 1 and extents positive");
  return (sbx_status)rc;
}

sbx_status sbx_deform_corners(int64_t elem_count, double amplitude, double* corners) {
  deform_corners(elem_count, amplitude, corners);
  return SBX_OK;
}

sbx_status sbx_geometric_factors(int64_t elem_count, int degree, const double* corners,
                                 double* g1, double* g2, double* g3, double* g4, double* g5,
                                 double* g6, double* bm, double* jac, int64_t* bad_elem) {
  double* const g[6] = {g1, g2, g3, g4, g5, g6};
  int64_t bad = -1;
  const int rc = geometric_factors(elem_count, degree, corners, g, bm, jac, &bad);
  if (bad_elem) *bad_elem = bad;
  if (rc == SBX_E_MESH)
    set_error("build_geometric_factors: nonpositive Jacobian in element " + std::to_string(bad));
  else if (rc)
    set_error("build_geometric_factors: bad degree");
  return (sbx_status)rc;
}

sbx_status sbx_gather_scatter(int ex, int ey, int ez, const int periodic[3], int degree,
                              int64_t* gid, int64_t* group_offsets, int64_t* group_nodes,
                              int32_t* mult, double* inv_mult, int64_t* global_count) {
  const int rc = gather_scatter(ex, ey, ez, periodic, degree, gid, group_offsets, group_nodes,
                                mult, inv_mult, global_count);
  if (rc) set_error("build_gather_scatter: degree must be >= 1");
  return (sbx_status)rc;
}

sbx_status sbx_dirichlet_mask(int ex, int ey, int ez, const int periodic[3], int degree,
                              double* mask) {
  return (sbx_status)dirichlet_mask(ex, ey, ez, periodic, degree, mask);
}

sbx_status sbx_partition_rcb(int64_t elem_count, const double* corners, int ranks,
                             int32_t* rank_of) {
  const int rc = partition_rcb(elem_count, corners, ranks, rank_of);
  if (rc)
    set_error("partition_rcb: ranks (" + std::to_string(ranks) + ") must be in [1, " +
              std::to_string(elem_count) + "]");
  return (sbx_status)rc;
}

sbx_status sbx_ctx_create(const sbx_problem_desc* desc, int device, sbx_ctx** out) {
  if (!desc || !out || !desc->deriv || !desc->group_offsets || !desc->group_nodes) {
    set_error("sbx_ctx_create: null argument");
    return SBX_E_INVALID;
  }
  for (int q = 0; q < 6; ++q)
    if (!desc->g[q]) {
      set_error("sbx_ctx_create: null geometric factor");
      return SBX_E_INVALID;
    }
  if (desc->degree < 1 || desc->degree > kMaxDegree) {
    set_error("sbx_ctx_create: degree must be in [1,32]");
    return SBX_E_CONFIG;
  }
  if (desc->elem_count < 1) {
    set_error("sbx_ctx_create: elem_count must be >= 1");
    return SBX_E_SHAPE;
  }
  *out = nullptr;
  auto* c = new sbx_ctx();
  sbx_status st = ctx_init_common(c, device);
  if (st == SBX_OK) st = ctx_upload(c, desc);
  if (st != SBX_OK) {
    sbx_ctx_destroy(c);
    return st;
  }
  *out = c;
  return SBX_OK;
}

// Device-side setup of a structured box: geometry, mask
// and multiplicities are built by kernels (setup_dev.cu) from the element
// corners; the gather-scatter runs on the lattice, so no map is built or
// uploaded.  Bitwise equal to the host builders (tests/test_gpu_setup.py).
static sbx_status ctx_setup_box_device(sbx_ctx* c, const sbx_box_desc* d, const double* corners) {
  const int64_t E = (int64_t)d->ex * d->ey * d->ez;
  const int n = d->degree + 1;
  const int64_t N = E * n * n * n;
  if (N >= (int64_t)INT32_MAX) {
    set_error("sbx_ctx_create_box: more than 2^31-1 local nodes per device");
    return SBX_E_SHAPE;
  }
  OpDev& op = c->op;
  op.E = E;
  op.n = n;
  op.nodes = N;
  std::vector<double> x(n), w(n), deriv(n * n);
  SBX_TRY(sbx_gll_basis(d->degree, x.data(), w.data(), deriv.data()));
  for (int q = 0; q < n * n; ++q) op.Dh[q] = deriv[q];
  double* dD = nullptr;
  SBX_TRY(dupload(c, &dD, deriv.data(), (int64_t)n * n));
  op.Dd = dD;
  // corners -> packed G and bm (temporary device copy of the corners)
  double* dcr = nullptr;
  SBX_CUDA(cudaMalloc(&dcr, sizeof(double) * (size_t)E * 24));
  SBX_CUDA(cudaMemcpyAsync(dcr, corners, sizeof(double) * (size_t)E * 24,
                           cudaMemcpyHostToDevice, c->stream));
  double *G = nullptr, *bm = nullptr;
  SBX_TRY(dupload<double>(c, &G, nullptr, 6 * N));
  SBX_TRY(dupload<double>(c, &bm, nullptr, N));
  unsigned long long* dbad = reinterpret_cast<unsigned long long*>(c->dcount);
  SBX_CUDA(cudaMemsetAsync(dbad, 0xff, sizeof(unsigned long long), c->stream));
  SBX_CUDA(launch_geom_box(dcr, E, n, x.data(), w.data(), G, bm, dbad, c->stream));
  unsigned long long hbad = 0;
  SBX_CUDA(cudaMemcpyAsync(&hbad, dbad, sizeof(hbad), cudaMemcpyDeviceToHost, c->stream));
  SBX_CUDA(cudaMemsetAsync(c->dcount, 0, 64 * sizeof(uint32_t), c->stream));
  SBX_CUDA(cudaStreamSynchronize(c->stream));
  cudaFree(dcr);
  if (hbad != ~0ull) {
    set_error("build_geometric_factors: nonpositive Jacobian in element " +
              std::to_string(hbad));
    return SBX_E_MESH;
  }
  op.G = G;
  op.bm = bm;
  // lattice: box dims, mask, multiplicities
  op.box = true;
  op.lat = true;
  op.ex = d->ex;
  op.ey = d->ey;
  op.ez = d->ez;
  int64_t gcount = 1;
  for (int q = 0; q < 3; ++q) {
    op.per[q] = d->periodic[q] ? 1 : 0;
    const int64_t span = (int64_t)(q == 0 ? d->ex : q == 1 ? d->ey : d->ez) * d->degree;
    gcount *= op.per[q] ? span : span + 1;
  }
  c->global_count = gcount;
  double *mask = nullptr, *im = nullptr;
  uint8_t* m8 = nullptr;
  SBX_TRY(dupload<double>(c, &mask, nullptr, N));
  SBX_TRY(dupload<double>(c, &im, nullptr, N));
  SBX_TRY(dupload<uint8_t>(c, &m8, nullptr, N));
  SBX_CUDA(launch_lattice_fields(op, mask, im, m8, c->stream));
  op.mask = mask;
  op.inv_mult = im;
  op.mult8 = m8;
  c->has_mask = true;
  c->interior_clean = true;  // element-interior nodes: unmasked singletons
  op.nB = 0;
  op.nBcopies = 0;
  SBX_TRY(upload_trilinear(c, d->degree, corners, E));
  SBX_TRY(ensure_partials(c, std::max<int64_t>(E, 4096)));
  c->cg.reset(new CgEngine());
  SBX_CUDA(cudaStreamSynchronize(c->stream));
  return SBX_OK;
}

sbx_status sbx_ctx_create_box(const sbx_box_desc* d, int device, sbx_ctx** out) {
  if (!d || !out) {
    set_error("sbx_ctx_create_box: null argument");
    return SBX_E_INVALID;
  }
  if (d->degree < 1 || d->degree > kMaxDegree) {
    set_error("build_gll_basis: degree must be in [1,32], got " + std::to_string(d->degree));
    return SBX_E_CONFIG;
  }
  const int64_t E = (int64_t)d->ex * d->ey * d->ez;
  const int n = d->degree + 1;
  const int64_t N = E * n * n * n;
  std::vector<double> corners(E * 24);
  SBX_TRY(sbx_box_corners(d->ex, d->ey, d->ez, d->origin, d->lengths, corners.data()));
  if (d->deform_amplitude != 0.0) deform_corners(E, d->deform_amplitude, corners.data());
  // device-side setup unless disabled (SBX_HOST_SETUP) or the lattice
  // gather-scatter does not apply (a periodic direction with one element)
  static const bool host_setup = std::getenv("SBX_HOST_SETUP") != nullptr;
  bool lattice_ok = true;
  const int counts[3] = {d->ex, d->ey, d->ez};
  for (int q = 0; q < 3; ++q)
    if (d->periodic[q] && counts[q] < 2) lattice_ok = false;
  if (!host_setup && lattice_ok) {
    *out = nullptr;
    auto* c = new sbx_ctx();
    sbx_status st = ctx_init_common(c, device);
    if (st == SBX_OK) st = ctx_setup_box_device(c, d, corners.data());
    if (st != SBX_OK) {
      sbx_ctx_destroy(c);
      return st;
    }
    *out = c;
    return SBX_OK;
  }
  std::vector<double> deriv(n * n);
  SBX_TRY(sbx_gll_basis(d->degree, nullptr, nullptr, deriv.data()));
  std::vector<std::vector<double>> g(7, std::vector<double>(N));
  int64_t bad = -1;
  SBX_TRY(sbx_geometric_factors(E, d->degree, corners.data(), g[0].data(), g[1].data(),
                                g[2].data(), g[3].data(), g[4].data(), g[5].data(), g[6].data(),
                                nullptr, &bad));
  std::vector<int64_t> offsets(N + 1), nodes(N);
  int64_t G = 0;
  SBX_TRY(sbx_gather_scatter(d->ex, d->ey, d->ez, d->periodic, d->degree, nullptr,
                             offsets.data(), nodes.data(), nullptr, nullptr, &G));
  std::vector<double> mask(N);
  SBX_TRY(sbx_dirichlet_mask(d->ex, d->ey, d->ez, d->periodic, d->degree, mask.data()));
  sbx_problem_desc pd{};
  pd.elem_count = E;
  pd.degree = d->degree;
  pd.deriv = deriv.data();
  for (int q = 0; q < 6; ++q) pd.g[q] = g[q].data();
  pd.bm = g[6].data();
  pd.mask = mask.data();
  pd.global_count = G;
  pd.group_offsets = offsets.data();
  pd.group_nodes = nodes.data();
  SBX_TRY(sbx_ctx_create(&pd, device, out));
  SBX_TRY(upload_trilinear(*out, d->degree, corners.data(), E));
  // structured element-centric gather-scatter (needs >= 2 cells per periodic axis)
  if (lattice_ok) {
    (*out)->op.box = true;
    (*out)->op.ex = d->ex;
    (*out)->op.ey = d->ey;
    (*out)->op.ez = d->ez;
    for (int q = 0; q < 3; ++q) (*out)->op.per[q] = d->periodic[q] ? 1 : 0;
  }
  return SBX_OK;
}

void sbx_ctx_destroy(sbx_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->dd.trace) {
    // SBX_TRACE=<prefix>: per-iteration timeline of this rank, one line per
    // iteration: it K1start K1end ifaceStart ifaceWaited K2start K2xchg K2xchgDone (ns)
    std::vector<unsigned long long> h((size_t)kTraceIters * 8);
    if (cudaMemcpy(h.data(), c->dd.trace, h.size() * 8, cudaMemcpyDeviceToHost) == cudaSuccess) {
      const std::string path = std::string(std::getenv("SBX_TRACE") ? std::getenv("SBX_TRACE")
                                                                     : "sbx_trace") +
                               ".rank" + std::to_string(c->rank);
      if (FILE* f = std::fopen(path.c_str(), "w")) {
        for (int it = 0; it < kTraceIters; ++it) {
          if (!h[(size_t)it * 8]) continue;
          std::fprintf(f, "%d", it);
          for (int q = 0; q < 7; ++q) std::fprintf(f, " %llu", h[(size_t)it * 8 + q]);
          std::fprintf(f, "\n");
        }
        std::fclose(f);
      }
    }
  }
  c->cg.reset();
  c->pe.reset();
  for (void* p : c->peer_windows) cudaIpcCloseMemHandle(p);
  if (c->window) cudaFree(c->window);
  for (void* p : c->allocs) cudaFree(p);
  if (c->hscal) cudaFreeHost(c->hscal);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  if (c->order_ev) cudaEventDestroy(c->order_ev);
  delete c;
}

sbx_status sbx_ctx_info(const sbx_ctx* c, int64_t* E, int32_t* n1d, int64_t* nodes,
                        int64_t* G, int64_t* bytes) {
  SBX_TRY(check_ctx(c));
  if (E) *E = c->op.E;
  if (n1d) *n1d = c->op.n;
  if (nodes) *nodes = c->op.nodes;
  if (G) *G = c->global_count;
  if (bytes) *bytes = c->device_bytes;
  return SBX_OK;
}

sbx_status sbx_ctx_features(const sbx_ctx* c, uint32_t* f) {
  SBX_TRY(check_ctx(c));
  if (!f) {
    set_error("sbx_ctx_features: null output");
    return SBX_E_INVALID;
  }
  *f = (c->op.lat ? SBX_FEAT_LATTICE_GS : 0u) | (c->op.box ? SBX_FEAT_BOX_K2 : 0u) |
       (c->op.tl ? SBX_FEAT_TRILINEAR : 0u);
  return SBX_OK;
}

sbx_status sbx_ctx_set_stream(sbx_ctx* c, void* stream) {
  SBX_TRY(check_ctx(c));
  c->caller = static_cast<cudaStream_t>(stream);
  return SBX_OK;
}

sbx_status sbx_ctx_copy_array(const sbx_ctx* c, int which, double* out) {
  SBX_TRY(check_ctx(c));
  const int64_t N = c->op.nodes;
  const int n3 = c->op.n * c->op.n * c->op.n;
  cudaSetDevice(c->device);
  auto copy = [&](const double* src, int64_t count) -> sbx_status {
    if (!src) {
      set_error("sbx_ctx_copy_array: array not present");
      return SBX_E_INVALID;
    }
    SBX_CUDA(cudaMemcpy(out, src, sizeof(double) * (size_t)count, cudaMemcpyDefault));
    return SBX_OK;
  };
  switch (which) {
    case 0: return copy(c->op.mask, N);
    case 1: return copy(c->op.inv_mult, N);
    case 2: return copy(c->op.bm, N);
    case 9: return copy(c->op.Dd, (int64_t)c->op.n * c->op.n);
    default:
      if (which >= 3 && which <= 8) {
        std::vector<double> G(6 * N);
        SBX_CUDA(cudaMemcpy(G.data(), c->op.G, sizeof(double) * 6 * (size_t)N,
                            cudaMemcpyDeviceToHost));
        std::vector<double> h(N);
        const int comp = which - 3;
        for (int64_t e = 0; e < c->op.E; ++e)
          std::memcpy(&h[e * n3], &G[(e * 6 + comp) * n3], sizeof(double) * n3);
        SBX_CUDA(cudaMemcpy(out, h.data(), sizeof(double) * (size_t)N, cudaMemcpyDefault));
        return SBX_OK;
      }
      set_error("sbx_ctx_copy_array: unknown array id");
      return SBX_E_INVALID;
  }
}

sbx_status sbx_ctx_set_coeff_fields(sbx_ctx* c, const double* h1f, const double* h2f) {
  SBX_TRY(check_ctx(c));
  if (c->dist && (h1f || h2f)) {
    set_error("sbx_ctx_set_coeff_fields: per-node coefficients are single-process only");
    return SBX_E_CONFIG;
  }
  if (h2f && !c->op.bm) {
    set_error("sbx_ctx_set_coeff_fields: h2 fields need the mass factors (bm)");
    return SBX_E_SHAPE;
  }
  SBX_TRY(enter(c));
  const size_t bytes = sizeof(double) * (size_t)c->op.nodes;
  auto put = [&](const double* src, double** dst) -> sbx_status {
    if (!src) return SBX_OK;
    if (!*dst) {
      void* p = nullptr;
      SBX_TRY(dalloc(c, &p, bytes));
      *dst = static_cast<double*>(p);
    }
    SBX_CUDA(cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyDefault, c->stream));
    return SBX_OK;
  };
  SBX_TRY(put(h1f, &c->h1f));
  SBX_TRY(put(h2f, &c->h2f));
  c->op.h1f = h1f ? c->h1f : nullptr;
  c->op.h2f = h2f ? c->h2f : nullptr;
  c->diag_h1 = c->diag_h2 = NAN;  // the cached Jacobi diagonal no longer applies
  return finish(c);
}

sbx_status sbx_axhelm(sbx_ctx* c, const double* u, double* w, double h1, double h2,
                      uint32_t flags) {
  SBX_TRY(check_ctx(c));
  if (!u || !w) {
    set_error("sbx_axhelm: null field");
    return SBX_E_INVALID;
  }
  if (h2 != 0.0 && !c->op.bm) {
    set_error("axhelm: h2 != 0 needs the mass factors (bm)");
    return SBX_E_SHAPE;
  }
  SBX_TRY(enter(c));
  const double* du = nullptr;
  SBX_TRY(stage_in(c, u, 0, &du));
  const bool wdev = is_device_ptr(w);
  double* dw = w;
  if (!wdev) SBX_TRY(work(c, 1, &dw));
  SBX_CUDA(launch_axhelm(c->op, du, dw, h1, h2, flags & SBX_FLAG_EXACT,
                         flags & SBX_FLAG_FLIP_T, c->stream));
  if (!wdev)
    SBX_CUDA(cudaMemcpyAsync(w, dw, sizeof(double) * (size_t)c->op.nodes, cudaMemcpyDeviceToHost,
                             c->stream));
  return finish(c);
}

sbx_status sbx_axhelm_diagonal(sbx_ctx* c, double h1, double h2, int assembled, double* diag) {
  SBX_TRY(check_ctx(c));
  if (!diag) {
    set_error("sbx_axhelm_diagonal: null output");
    return SBX_E_INVALID;
  }
  SBX_TRY(enter(c));
  const bool ddev = is_device_ptr(diag);
  double* dd = diag;
  if (!ddev) SBX_TRY(work(c, 1, &dd));
  SBX_CUDA(launch_axhelm_diag(c->op, h1, h2, dd, c->stream));
  if (assembled) SBX_TRY(gs_dev(c, dd, false));
  if (!ddev)
    SBX_CUDA(cudaMemcpyAsync(diag, dd, sizeof(double) * (size_t)c->op.nodes,
                             cudaMemcpyDeviceToHost, c->stream));
  return finish(c);
}

sbx_status sbx_gs_sum(sbx_ctx* c, double* f) {
  SBX_TRY(check_ctx(c));
  if (!f) {
    set_error("sbx_gs_sum: null field");
    return SBX_E_INVALID;
  }
  SBX_TRY(enter(c));
  const bool dev = is_device_ptr(f);
  double* df = f;
  if (!dev) {
    SBX_TRY(work(c, 1, &df));
    SBX_CUDA(cudaMemcpyAsync(df, f, sizeof(double) * (size_t)c->op.nodes,
                             cudaMemcpyHostToDevice, c->stream));
  }
  SBX_TRY(gs_dev(c, df, false));
  if (!dev)
    SBX_CUDA(cudaMemcpyAsync(f, df, sizeof(double) * (size_t)c->op.nodes, cudaMemcpyDeviceToHost,
                             c->stream));
  return finish(c);
}

sbx_status sbx_apply(sbx_ctx* c, const double* x, double* q, double h1, double h2,
                     uint32_t flags) {
  SBX_TRY(check_ctx(c));
  if (!x || !q) {
    set_error("sbx_apply: null field");
    return SBX_E_INVALID;
  }
  if (h2 != 0.0 && !c->op.bm) {
    set_error("apply: h2 != 0 needs the mass factors (bm)");
    return SBX_E_SHAPE;
  }
  SBX_TRY(enter(c));
  const double* dx = nullptr;
  SBX_TRY(stage_in(c, x, 0, &dx));
  const bool qdev = is_device_ptr(q);
  double* dq = q;
  if (!qdev) SBX_TRY(work(c, 1, &dq));
  SBX_TRY(apply_dev(c, dx, dq, h1, h2, flags & SBX_FLAG_EXACT, flags & SBX_FLAG_FLIP_T,
                    !(flags & SBX_FLAG_NO_MASK)));
  if (!qdev)
    SBX_CUDA(cudaMemcpyAsync(q, dq, sizeof(double) * (size_t)c->op.nodes, cudaMemcpyDeviceToHost,
                             c->stream));
  return finish(c);
}

sbx_status sbx_dot(sbx_ctx* c, const double* a, const double* b, int weighted, uint32_t flags,
                   double* result) {
  SBX_TRY(check_ctx(c));
  if (!a || !b || !result) {
    set_error("sbx_dot: null argument");
    return SBX_E_INVALID;
  }
  SBX_TRY(enter(c));
  const double *da = nullptr, *db = nullptr;
  SBX_TRY(stage_in(c, a, 0, &da));
  SBX_TRY(stage_in(c, b, 1, &db));
  if (flags & SBX_FLAG_EXACT) {
    if (c->dist) {
      set_error("sbx_dot: the reference-order (EXACT) dot is single-process");
      return SBX_E_CONFIG;
    }
    return dot_exact(c, da, db, weighted != 0, result);
  }
  SBX_CUDA(launch_dot_fast(c->op.nodes, da, db, weighted ? c->op.inv_mult : nullptr,
                           c->partials, c->dcount, c->dscal, c->stream));
  if (c->dist) SBX_CUDA(launch_dist_allreduce(c->dd, 3, c->dscal, c->dscal, 1, c->stream));
  SBX_CUDA(cudaMemcpyAsync(c->hscal, c->dscal, sizeof(double), cudaMemcpyDeviceToHost,
                           c->stream));
  SBX_TRY(finish(c));
  *result = c->hscal[0];
  return SBX_OK;
}

void sbx_pcg_config_default(sbx_pcg_config* cfg) {
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->tolerance = 1e-8;
  cfg->max_iterations = 500;
  cfg->precond = SBX_PRECOND_JACOBI;
  cfg->mode = SBX_MODE_FAST;
  cfg->h1 = 1.0;
  cfg->h2 = 0.0;
}

sbx_status sbx_pcg(sbx_ctx* c, const double* b, double* x, const sbx_pcg_config* cfg,
                   sbx_pcg_result* res) {
  SBX_TRY(check_ctx(c));
  if (!b || !x || !cfg || !res) {
    set_error("sbx_pcg: null argument");
    return SBX_E_INVALID;
  }
  if (cfg->h2 != 0.0 && !c->op.bm) {
    set_error("pcg: h2 != 0 needs the mass factors (bm)");
    return SBX_E_SHAPE;
  }
  SBX_TRY(enter(c));
  std::memset(res, 0, sizeof(*res));
  res->error_iteration = -1;
  const int64_t N = c->op.nodes;
  const double* db = nullptr;
  SBX_TRY(stage_in(c, b, 0, &db));
  const bool xdev = is_device_ptr(x);
  double* dx = x;
  if (!xdev) {
    SBX_TRY(work(c, 1, &dx));
    SBX_CUDA(cudaMemcpyAsync(dx, x, sizeof(double) * (size_t)N, cudaMemcpyHostToDevice,
                             c->stream));
  }
  sbx_status st;
  if (c->dist && cfg->mode != SBX_MODE_FAST) {
    set_error("pcg: the EXACT (reference-order) mode is single-process; use FAST with >1 rank");
    return SBX_E_CONFIG;
  }
  if (c->dist && !c->connected) {
    set_error("distributed context used before sbx_ctx_dist_connect");
    return SBX_E_COMM;
  }
  // per-node coefficients: the fused kernels take scalars only, so the solve
  // runs in the reference order (still on the device)
  const bool fields = c->op.h1f || c->op.h2f;
  if (cfg->mode == SBX_MODE_FAST && !fields) {
    if (cfg->precond == SBX_PRECOND_JACOBI) SBX_TRY(ensure_diag(c, cfg->h1, cfg->h2));
    CgRun run;
    run.op = &c->op;
    run.stream = c->stream;
    run.b = db;
    run.x = dx;
    run.dinv = cfg->precond == SBX_PRECOND_JACOBI ? c->ddinv : nullptr;
    run.h1 = cfg->h1;
    run.h2 = cfg->h2;
    run.tol = cfg->tolerance;
    run.max_it = cfg->max_iterations;
    run.history = cfg->history;
    run.history_capacity = cfg->history_capacity;
    run.interior_clean = c->interior_clean;
    run.timing = c->timing;
    run.dist = c->dist ? &c->dd : nullptr;
    const int rc = c->cg->solve(run, res);
    st = (sbx_status)rc;
    if (rc == kCgFallback) {
      // FAST schedule preconditions not met (see cg.cu): reference-order path
      std::memset(res, 0, sizeof(*res));
      res->error_iteration = -1;
      st = pcg_exact(c, db, dx, cfg, res);
    } else if (st == SBX_E_CUDA) set_error(c->cg->error());
    else if (st == SBX_E_BREAKDOWN)
      set_error("pcg: breakdown (p'Ap <= 0 or non-finite) at iteration " +
                std::to_string(res->error_iteration));
    else if (st == SBX_E_NAN)
      set_error("pcg: residual diverged (NaN/Inf) at iteration " +
                std::to_string(res->error_iteration));
    else if (st == SBX_E_SHAPE || st == SBX_E_COMM || st == SBX_E_CONFIG)
      set_error(c->cg->error());
    if (st == SBX_E_COMM) c->poisoned = true;
  } else {
    st = pcg_exact(c, db, dx, cfg, res);
  }
  if (!xdev && (st == SBX_OK || st == SBX_E_BREAKDOWN || st == SBX_E_NAN)) {
    SBX_CUDA(cudaMemcpyAsync(x, dx, sizeof(double) * (size_t)N, cudaMemcpyDeviceToHost,
                             c->stream));
    sbx_status f = finish(c);
    if (st == SBX_OK) st = f;
  }
  return st;
}

sbx_status sbx_debug_cg_k1(sbx_ctx* c, const double* u, double* w, double h1, double h2) {
  SBX_TRY(check_ctx(c));
  if (!u || !w) {
    set_error("sbx_debug_cg_k1: null field");
    return SBX_E_INVALID;
  }
  if (c->dist) {
    set_error("sbx_debug_cg_k1: single-process contexts only (K1 pushes the halo)");
    return SBX_E_CONFIG;
  }
  if (c->op.h1f || c->op.h2f) {
    set_error("sbx_debug_cg_k1: the fused K1 takes scalar h1 / h2 (per-node fields are set)");
    return SBX_E_CONFIG;
  }
  if (h2 != 0.0 && !c->op.bm) {
    set_error("sbx_debug_cg_k1: h2 != 0 needs the mass factors (bm)");
    return SBX_E_SHAPE;
  }
  SBX_TRY(enter(c));
  const double* du = nullptr;
  SBX_TRY(stage_in(c, u, 0, &du));
  const bool wdev = is_device_ptr(w);
  double* dw = w;
  if (!wdev) SBX_TRY(work(c, 1, &dw));
  const int rc = c->cg->debug_k1(c->op, c->stream, du, dw, h1, h2);
  if (rc != SBX_OK) {
    set_error(c->cg->error());
    return (sbx_status)rc;
  }
  if (!wdev)
    SBX_CUDA(cudaMemcpyAsync(w, dw, sizeof(double) * (size_t)c->op.nodes, cudaMemcpyDeviceToHost,
                             c->stream));
  return finish(c);
}

// ---- consistent-Poisson pressure operator ------------
sbx_status sbx_pressure_basis(int degree, double* nodes, double* weights, double* interp) {
  const int rc = pressure_basis(degree, nodes, weights, interp);
  if (rc)
    set_error("build_pressure_basis: velocity degree must be >= 3 (no interior pressure grid "
              "below that), got " + std::to_string(degree));
  return (sbx_status)rc;
}

static sbx_status pressure_enter(sbx_ctx* c) {
  SBX_TRY(check_ctx(c));
  if (c->dist) {
    set_error("pressure operator: single-process contexts only");
    return SBX_E_CONFIG;
  }
  SBX_TRY(enter(c));
  if (!c->pe) c->pe.reset(new PressureEngine());
  const int rc = c->pe->setup(c->op, c->stream);
  if (rc != SBX_OK) {
    set_error(c->pe->error());
    return (sbx_status)rc;
  }
  return SBX_OK;
}

sbx_status sbx_pressure_info(sbx_ctx* c, int64_t* pnodes, int32_t* m1d) {
  SBX_TRY(pressure_enter(c));
  if (pnodes) *pnodes = c->pe->pnodes();
  if (m1d) *m1d = c->pe->m1d();
  return finish(c);
}

// pressure-grid vectors share the velocity-size work buffers (E m^3 < E n^3)
static sbx_status stage_p(sbx_ctx* c, const double* p, int64_t count, int slot,
                          const double** out) {
  if (is_device_ptr(p)) {
    *out = p;
    return SBX_OK;
  }
  double* w = nullptr;
  SBX_TRY(work(c, slot, &w));
  SBX_CUDA(cudaMemcpyAsync(w, p, sizeof(double) * (size_t)count, cudaMemcpyHostToDevice,
                           c->stream));
  *out = w;
  return SBX_OK;
}

sbx_status sbx_gradient_from_pressure(sbx_ctx* c, const double* p, double* gx, double* gy,
                                      double* gz, uint32_t flags) {
  if (!p || !gx || !gy || !gz) {
    set_error("sbx_gradient_from_pressure: null field");
    return SBX_E_INVALID;
  }
  SBX_TRY(pressure_enter(c));
  const double* dp = nullptr;
  SBX_TRY(stage_p(c, p, c->pe->pnodes(), 0, &dp));
  double* outs[3] = {gx, gy, gz};
  double* d[3];
  for (int q = 0; q < 3; ++q) {
    d[q] = outs[q];
    if (!is_device_ptr(outs[q])) SBX_TRY(work(c, 1 + q, &d[q]));
  }
  const int grc = (flags & SBX_FLAG_EXACT) ? c->pe->grad_exact(dp, d, c->stream)
                                            : c->pe->grad(dp, d, c->stream);
  if (grc != SBX_OK) {
    set_error(c->pe->error());
    return (sbx_status)grc;
  }
  for (int q = 0; q < 3; ++q)
    if (d[q] != outs[q])
      SBX_CUDA(cudaMemcpyAsync(outs[q], d[q], sizeof(double) * (size_t)c->op.nodes,
                               cudaMemcpyDeviceToHost, c->stream));
  return finish(c);
}

sbx_status sbx_divergence_to_pressure(sbx_ctx* c, const double* ux, const double* uy,
                                      const double* uz, double* out, uint32_t flags) {
  if (!ux || !uy || !uz || !out) {
    set_error("sbx_divergence_to_pressure: null field");
    return SBX_E_INVALID;
  }
  SBX_TRY(pressure_enter(c));
  const double* in[3] = {ux, uy, uz};
  const double* d[3];
  for (int q = 0; q < 3; ++q) SBX_TRY(stage_in(c, in[q], q, &d[q]));
  const bool odev = is_device_ptr(out);
  double* o = out;
  if (!odev) SBX_TRY(work(c, 3, &o));
  const int drc = (flags & SBX_FLAG_EXACT) ? c->pe->div_exact(d, o, c->stream)
                                            : c->pe->div(d, o, c->stream);
  if (drc != SBX_OK) {
    set_error(c->pe->error());
    return (sbx_status)drc;
  }
  if (!odev)
    SBX_CUDA(cudaMemcpyAsync(out, o, sizeof(double) * (size_t)c->pe->pnodes(),
                             cudaMemcpyDeviceToHost, c->stream));
  return finish(c);
}

sbx_status sbx_pressure_apply(sbx_ctx* c, const double* p, double* out, uint32_t flags) {
  if (!p || !out) {
    set_error("sbx_pressure_apply: null field");
    return SBX_E_INVALID;
  }
  SBX_TRY(pressure_enter(c));
  const double* dp = nullptr;
  SBX_TRY(stage_p(c, p, c->pe->pnodes(), 0, &dp));
  const bool odev = is_device_ptr(out);
  double* o = out;
  if (!odev) SBX_TRY(work(c, 1, &o));
  const int arc = (flags & SBX_FLAG_EXACT) ? c->pe->apply_exact(dp, o, c->stream)
                                            : c->pe->apply(dp, o, c->stream);
  if (arc != SBX_OK) {
    set_error(c->pe->error());
    return (sbx_status)arc;
  }
  if (!odev)
    SBX_CUDA(cudaMemcpyAsync(out, o, sizeof(double) * (size_t)c->pe->pnodes(),
                             cudaMemcpyDeviceToHost, c->stream));
  return finish(c);
}

sbx_status sbx_pressure_diagonal(sbx_ctx* c, double* diag, uint32_t flags) {
  if (!diag) {
    set_error("sbx_pressure_diagonal: null output");
    return SBX_E_INVALID;
  }
  SBX_TRY(pressure_enter(c));
  const bool ex = flags & SBX_FLAG_EXACT;
  const int rc = ex ? c->pe->ensure_diag_exact(c->stream) : c->pe->ensure_diag(c->stream);
  if (rc != SBX_OK) {
    set_error(c->pe->error());
    return (sbx_status)rc;
  }
  SBX_CUDA(cudaMemcpyAsync(diag, ex ? c->pe->diag_exact() : c->pe->diag(),
                           sizeof(double) * (size_t)c->pe->pnodes(), cudaMemcpyDefault,
                           c->stream));
  return finish(c);
}

sbx_status sbx_pressure_pcg(sbx_ctx* c, const double* b, double* x, const sbx_pcg_config* cfg,
                            sbx_pcg_result* res) {
  if (!b || !x || !cfg || !res) {
    set_error("sbx_pressure_pcg: null argument");
    return SBX_E_INVALID;
  }
  SBX_TRY(pressure_enter(c));
  const int64_t Np = c->pe->pnodes();
  const double* db = nullptr;
  SBX_TRY(stage_p(c, b, Np, 0, &db));
  const bool xdev = is_device_ptr(x);
  double* dx = x;
  if (!xdev) {
    SBX_TRY(work(c, 1, &dx));
    SBX_CUDA(cudaMemcpyAsync(dx, x, sizeof(double) * (size_t)Np, cudaMemcpyHostToDevice,
                             c->stream));
  }
  const int rc = cfg->mode == SBX_MODE_EXACT ? c->pe->solve_exact(c->stream, db, dx, *cfg, res)
                                             : c->pe->solve(c->stream, db, dx, *cfg, res);
  sbx_status st = (sbx_status)rc;
  if (st == SBX_E_BREAKDOWN)
    set_error("pcg: breakdown (p'Ap <= 0 or non-finite) at iteration " +
              std::to_string(res->error_iteration));
  else if (st == SBX_E_NAN)
    set_error("pcg: residual diverged (NaN/Inf) at iteration " +
              std::to_string(res->error_iteration));
  else if (st != SBX_OK)
    set_error(c->pe->error());
  if (!xdev && (st == SBX_OK || st == SBX_E_BREAKDOWN || st == SBX_E_NAN)) {
    SBX_CUDA(cudaMemcpyAsync(x, dx, sizeof(double) * (size_t)Np, cudaMemcpyDeviceToHost,
                             c->stream));
    const sbx_status f = finish(c);
    if (st == SBX_OK) st = f;
  }
  return st;
}

sbx_status sbx_projection_reset(sbx_ctx* c, int depth) {
  SBX_TRY(pressure_enter(c));
  c->pe->proj_reset(depth);
  return finish(c);
}

sbx_status sbx_projection_size(sbx_ctx* c, int32_t* size) {
  SBX_TRY(pressure_enter(c));
  if (size) *size = c->pe->proj_size();
  return finish(c);
}

sbx_status sbx_projection_guess(sbx_ctx* c, const double* b, double* guess, double* deflated,
                                uint32_t flags) {
  if (!b || !guess) {
    set_error("sbx_projection_guess: null field");
    return SBX_E_INVALID;
  }
  SBX_TRY(pressure_enter(c));
  const int64_t Np = c->pe->pnodes();
  const double* db = nullptr;
  SBX_TRY(stage_p(c, b, Np, 0, &db));
  double* dg = guess;
  const bool gdev = is_device_ptr(guess);
  if (!gdev) SBX_TRY(work(c, 1, &dg));
  double* dd = deflated;
  const bool ddev = !deflated || is_device_ptr(deflated);
  if (!ddev) SBX_TRY(work(c, 2, &dd));
  const int rc = c->pe->proj_guess(c->stream, db, dg, dd, flags & SBX_FLAG_EXACT);
  if (rc != SBX_OK) {
    set_error(c->pe->error());
    return (sbx_status)rc;
  }
  if (!gdev)
    SBX_CUDA(cudaMemcpyAsync(guess, dg, sizeof(double) * (size_t)Np, cudaMemcpyDeviceToHost,
                             c->stream));
  if (!ddev)
    SBX_CUDA(cudaMemcpyAsync(deflated, dd, sizeof(double) * (size_t)Np, cudaMemcpyDeviceToHost,
                             c->stream));
  return finish(c);
}

sbx_status sbx_projection_append(sbx_ctx* c, const double* x, uint32_t flags) {
  if (!x) {
    set_error("sbx_projection_append: null field");
    return SBX_E_INVALID;
  }
  SBX_TRY(pressure_enter(c));
  const double* dx = nullptr;
  SBX_TRY(stage_p(c, x, c->pe->pnodes(), 0, &dx));
  const int rc = c->pe->proj_append(c->stream, dx, flags & SBX_FLAG_EXACT);
  if (rc != SBX_OK) {
    set_error(c->pe->error());
    return (sbx_status)rc;
  }
  return finish(c);
}

sbx_status sbx_advect(sbx_ctx* c, const double* const u[3], const double* const cv[3],
                      double* const out[3]) {
  SBX_TRY(check_ctx(c));
  if (!u || !cv || !out) {
    set_error("sbx_advect: null argument");
    return SBX_E_INVALID;
  }
  for (int q = 0; q < 3; ++q)
    if (!u[q] || !cv[q] || !out[q]) {
      set_error("sbx_advect: null field");
      return SBX_E_INVALID;
    }
  if (!c->op.corners || !c->op.bm) {
    set_error("advect: needs the element corners and the mass factors (a box context or a "
              "verified structured-box hint)");
    return SBX_E_CONFIG;
  }
  SBX_TRY(enter(c));
  const double* du[3];
  const double* dc[3];
  double* dout[3];
  for (int q = 0; q < 3; ++q) {
    SBX_TRY(stage_in(c, u[q], q, &du[q]));
    SBX_TRY(stage_in(c, cv[q], 3 + q, &dc[q]));
    dout[q] = out[q];
    if (!is_device_ptr(out[q])) SBX_TRY(work(c, 6 + q, &dout[q]));
  }
  // GLL nodes on the device (the derivative matrix is op.Dd)
  if (!c->dgllx) {
    void* p = nullptr;
    SBX_TRY(dalloc(c, &p, sizeof(double) * 33));
    c->dgllx = static_cast<double*>(p);
    SBX_CUDA(cudaMemcpyAsync(c->dgllx, c->op.Xh, sizeof(double) * c->op.n,
                             cudaMemcpyHostToDevice, c->stream));
  }
  SBX_CUDA(launch_advect(c->op.E, c->op.n, c->op.corners, c->op.Dd, c->dgllx, c->op.bm, du, dc,
                         dout, c->stream));
  for (int q = 0; q < 3; ++q)
    if (dout[q] != out[q])
      SBX_CUDA(cudaMemcpyAsync(out[q], dout[q], sizeof(double) * (size_t)c->op.nodes,
                               cudaMemcpyDeviceToHost, c->stream));
  return finish(c);
}

// Batched solve of count <= 3 right-hand sides with one operator: the three
// velocity components of FlowSolver::solve_velocity_star (stepper.cpp:
// 188-238), each with its own initial guess in x[d] and its own convergence.
sbx_status sbx_pcg_multi(sbx_ctx* c, int count, const double* const* b, double* const* x,
                         const sbx_pcg_config* cfg, sbx_pcg_result* res) {
  SBX_TRY(check_ctx(c));
  if (!b || !x || !cfg || !res || count < 1 || count > kMaxComp) {
    set_error("sbx_pcg_multi: null argument or count not in [1, 3]");
    return SBX_E_INVALID;
  }
  for (int q = 0; q < count; ++q)
    if (!b[q] || !x[q]) {
      set_error("sbx_pcg_multi: null field");
      return SBX_E_INVALID;
    }
  if (cfg->h2 != 0.0 && !c->op.bm) {
    set_error("pcg: h2 != 0 needs the mass factors (bm)");
    return SBX_E_SHAPE;
  }
  auto one = [&](int q) -> sbx_status {
    sbx_pcg_config cq = *cfg;
    if (cfg->history) cq.history = cfg->history + (size_t)q * cfg->history_capacity;
    return sbx_pcg(c, b[q], x[q], &cq, &res[q]);
  };
  if (cfg->mode != SBX_MODE_FAST || c->dist || count == 1 || c->op.h1f || c->op.h2f) {
    // reference order (or one rhs, or per-node coefficients): the components
    // one after the other, as solve_velocity_star does
    for (int q = 0; q < count; ++q) SBX_TRY(one(q));
    return SBX_OK;
  }
  SBX_TRY(enter(c));
  const int64_t N = c->op.nodes;
  SBX_TRY(ensure_diag_if(c, cfg));
  const double* db[kMaxComp];
  double* dx[kMaxComp];
  bool xdev[kMaxComp];
  for (int q = 0; q < count; ++q) {
    SBX_TRY(stage_in(c, b[q], q, &db[q]));
    xdev[q] = is_device_ptr(x[q]);
    dx[q] = x[q];
    if (!xdev[q]) {
      SBX_TRY(work(c, 3 + q, &dx[q]));
      SBX_CUDA(cudaMemcpyAsync(dx[q], x[q], sizeof(double) * (size_t)N, cudaMemcpyHostToDevice,
                               c->stream));
    }
  }
  CgRun runs[kMaxComp];
  for (int q = 0; q < count; ++q) {
    CgRun& r = runs[q];
    r.op = &c->op;
    r.stream = c->stream;
    r.b = db[q];
    r.x = dx[q];
    r.dinv = cfg->precond == SBX_PRECOND_JACOBI ? c->ddinv : nullptr;
    r.h1 = cfg->h1;
    r.h2 = cfg->h2;
    r.tol = cfg->tolerance;
    r.max_it = cfg->max_iterations;
    r.history = cfg->history ? cfg->history + (size_t)q * cfg->history_capacity : nullptr;
    r.history_capacity = cfg->history_capacity;
    r.interior_clean = c->interior_clean;
  }
  const int rc = c->cg->solve_multi(runs, count, res);
  if (rc == kCgFallback) {
    // no batched kernels here (or a right-hand side the fused schedule cannot
    // take): nothing was written; solve the components one by one
    for (int q = 0; q < count; ++q) SBX_TRY(one(q));
    return SBX_OK;
  }
  sbx_status st = (sbx_status)rc;
  if (st == SBX_E_CUDA) set_error(c->cg->error());
  else if (st == SBX_E_BREAKDOWN || st == SBX_E_NAN)
    set_error("pcg (batched): breakdown or NaN/Inf in a component");
  for (int q = 0; q < count; ++q)
    if (!xdev[q])
      SBX_CUDA(cudaMemcpyAsync(x[q], dx[q], sizeof(double) * (size_t)N, cudaMemcpyDeviceToHost,
                               c->stream));
  const sbx_status f = finish(c);
  return st == SBX_OK ? f : st;
}

sbx_status sbx_ctx_enable_timing(sbx_ctx* c, int enable) {
  SBX_TRY(check_ctx(c));
  c->timing = enable != 0;
  return SBX_OK;
}

sbx_status sbx_ctx_kernel_time(const sbx_ctx* c, const char* name, double* total_ms,
                               int64_t* launches) {
  SBX_TRY(check_ctx(c));
  if (!c->cg) return SBX_E_INVALID;
  return (sbx_status)c->cg->kernel_time(name, total_ms, launches);
}

sbx_status sbx_ctx_local_elements(const sbx_ctx* c, int64_t* ids) {
  SBX_TRY(check_ctx(c));
  if (c->local_elements.empty()) {
    for (int64_t e = 0; e < c->op.E; ++e) ids[e] = e;
  } else {
    std::memcpy(ids, c->local_elements.data(), sizeof(int64_t) * c->local_elements.size());
  }
  return SBX_OK;
}

}  // extern "C"

// ---- multi-GPU entry points: see dist.cu -----------------------------------

// =========================================================== multi-GPU =====
#include "dist_plan.h"

namespace {

struct DistBlob {
  cudaIpcMemHandle_t handle;
  int64_t recv_total;                 // size of one receive-buffer parity region
  int64_t recv_base_for_src[kMaxRanks];  // where rank q's block lands in it (-1: none)
};

sbx_status upload_dist(sbx_ctx* c, const DistPlan& P, const sbx_box_desc* d) {
  const int n = P.n;
  const int64_t EL = (int64_t)P.loc_elems.size();
  const int64_t NL = P.nodes_local();
  c->op.E = EL;
  c->op.n = n;
  c->op.nodes = NL;
  c->global_count = 0;
  // local geometry from the local elements' corners (deformed like the box)
  std::vector<double> all(P.E * 24);
  SBX_TRY(sbx_box_corners(d->ex, d->ey, d->ez, d->origin, d->lengths, all.data()));
  if (d->deform_amplitude != 0.0) deform_corners(P.E, d->deform_amplitude, all.data());
  std::vector<double> loc(EL * 24);
  for (int64_t le = 0; le < EL; ++le)
    std::memcpy(&loc[le * 24], &all[P.loc_elems[le] * 24], 24 * sizeof(double));
  all.clear();
  all.shrink_to_fit();
  SBX_TRY(upload_trilinear(c, d->degree, loc.data(), EL));
  std::vector<double> deriv(n * n);
  SBX_TRY(sbx_gll_basis(d->degree, nullptr, nullptr, deriv.data()));
  for (int q = 0; q < n * n; ++q) c->op.Dh[q] = deriv[q];
  double* dD = nullptr;
  SBX_TRY(dupload(c, &dD, deriv.data(), (int64_t)n * n));
  c->op.Dd = dD;
  std::vector<std::vector<double>> g(7, std::vector<double>(NL));
  int64_t bad = -1;
  SBX_TRY(sbx_geometric_factors(EL, d->degree, loc.data(), g[0].data(), g[1].data(),
                                g[2].data(), g[3].data(), g[4].data(), g[5].data(), g[6].data(),
                                nullptr, &bad));
  double* G = nullptr;
  SBX_TRY(dupload<double>(c, &G, nullptr, 6 * NL));
  {
    double* tmp[6] = {};
    for (int q = 0; q < 6; ++q) {
      SBX_CUDA(cudaMalloc(&tmp[q], sizeof(double) * (size_t)NL));
      SBX_CUDA(cudaMemcpyAsync(tmp[q], g[q].data(), sizeof(double) * (size_t)NL,
                               cudaMemcpyHostToDevice, c->stream));
    }
    SBX_CUDA(launch_pack_geometry(c->op, tmp, G, c->stream));
    SBX_CUDA(cudaStreamSynchronize(c->stream));
    for (int q = 0; q < 6; ++q) cudaFree(tmp[q]);
  }
  c->op.G = G;
  double *bm = nullptr, *mask = nullptr, *im = nullptr;
  SBX_TRY(dupload(c, &bm, g[6].data(), NL));
  SBX_TRY(dupload(c, &mask, P.mask.data(), NL));
  SBX_TRY(dupload(c, &im, P.inv_mult.data(), NL));
  c->op.bm = bm;
  c->op.mask = mask;
  c->op.inv_mult = im;
  c->has_mask = true;
  c->interior_clean = true;  // by construction of the plan
  int32_t *boff = nullptr, *bidx = nullptr, *n27 = nullptr;
  SBX_TRY(dupload(c, &boff, P.b_off.data(), (int64_t)P.b_off.size()));
  SBX_TRY(dupload(c, &bidx, P.b_idx.data(), (int64_t)P.b_idx.size()));
  SBX_TRY(dupload(c, &n27, P.nbr27.data(), (int64_t)P.nbr27.size()));
  int64_t* ge = nullptr;
  SBX_TRY(dupload(c, &ge, P.loc_elems.data(), EL));
  c->op.b_off = boff;
  c->op.b_idx = bidx;
  c->op.nB = (int64_t)P.b_off.size() - 1;
  c->op.nBcopies = (int64_t)P.b_idx.size();
  c->op.box = true;
  c->op.table = true;
  c->op.ex = d->ex;
  c->op.ey = d->ey;
  c->op.ez = d->ez;
  for (int q = 0; q < 3; ++q) c->op.per[q] = d->periodic[q] ? 1 : 0;
  c->op.nbr27 = n27;
  c->op.gelem = ge;
  // exchange plan on the device
  DistDev& D = c->dd;
  D.nranks = P.nranks;
  D.rank = P.rank;
  D.nodes_local = NL;
  D.nnbr = (int)P.nbr.size();
  std::vector<int32_t> sidx;
  D.send_off[0] = 0;
  for (int qi = 0; qi < D.nnbr; ++qi) {
    D.nbr[qi] = P.nbr[qi];
    sidx.insert(sidx.end(), P.send_idx[qi].begin(), P.send_idx[qi].end());
    D.send_off[qi + 1] = (int64_t)sidx.size();
  }
  int32_t *dsidx = nullptr, *ioff = nullptr, *icode = nullptr;
  SBX_TRY(dupload(c, &dsidx, sidx.data(), (int64_t)sidx.size()));
  SBX_TRY(dupload(c, &ioff, P.if_off.data(), (int64_t)P.if_off.size()));
  SBX_TRY(dupload(c, &icode, P.if_code.data(), (int64_t)P.if_code.size()));
  D.send_idx = dsidx;
  D.if_off = ioff;
  D.if_code = icode;
  int32_t *eo = nullptr, *en = nullptr, *eq = nullptr, *ep = nullptr;
  SBX_TRY(dupload(c, &eo, P.esend_off.data(), (int64_t)P.esend_off.size()));
  SBX_TRY(dupload(c, &en, P.esend_node.data(), (int64_t)P.esend_node.size()));
  SBX_TRY(dupload(c, &eq, P.esend_q.data(), (int64_t)P.esend_q.size()));
  SBX_TRY(dupload(c, &ep, P.esend_pos.data(), (int64_t)P.esend_pos.size()));
  D.esend_off = eo;
  D.esend_node = en;
  D.esend_q = eq;
  D.esend_pos = ep;
  D.n_if = (int64_t)P.if_off.size() - 1;
  D.nbr27 = n27;
  D.gelem = ge;
  D.recv_total = P.recv_total;
  D.send_total = D.send_off[D.nnbr];
  for (int qi = 0; qi < D.nnbr; ++qi) D.recv_base[qi] = P.recv_base[qi];
  D.recv_base[D.nnbr] = P.recv_total;
  void* p = nullptr;
  SBX_TRY(dalloc(c, &p, 4 * sizeof(unsigned long long)));
  D.seq = static_cast<unsigned long long*>(p);
  SBX_TRY(dalloc(c, &p, 4 * sizeof(unsigned int)));
  D.counter = static_cast<unsigned int*>(p);
  SBX_TRY(dalloc(c, &p, 2 * sizeof(unsigned int)));
  D.gbar = static_cast<unsigned int*>(p);
  SBX_CUDA(cudaMemsetAsync(D.gbar, 0, 2 * sizeof(unsigned int), c->stream));
  SBX_TRY(dalloc(c, &p, sizeof(int)));
  D.status = static_cast<int*>(p);
  SBX_CUDA(cudaMemsetAsync(D.seq, 0, 4 * sizeof(unsigned long long), c->stream));
  SBX_CUDA(cudaMemsetAsync(D.counter, 0, 4 * sizeof(unsigned int), c->stream));
  SBX_CUDA(cudaMemsetAsync(D.status, 0, sizeof(int), c->stream));
  // peer window (exported over CUDA IPC; own allocation, not via dalloc's list
  // so it is freed after the peers close their mappings)
  const size_t wbytes =
      kWinRecv + sizeof(double) * (size_t)std::max<int64_t>(4 * D.recv_total, 2);
  SBX_CUDA(cudaMalloc(&c->window, wbytes));
  SBX_CUDA(cudaMemsetAsync(c->window, 0, wbytes, c->stream));
  char* wb = static_cast<char*>(c->window);
  D.flags = reinterpret_cast<unsigned long long*>(wb + kWinFlags);
  D.mbox = reinterpret_cast<double*>(wb + kWinMbox);
  D.recvb = reinterpret_cast<double*>(wb + kWinRecv);
  // per source rank: offset of its block in my receive buffer (-1: none)
  c->recv_base_for_src.assign(kMaxRanks, -1);
  for (int qi = 0; qi < D.nnbr; ++qi) c->recv_base_for_src[P.nbr[qi]] = D.recv_base[qi];
  SBX_TRY(ensure_partials(c, std::max<int64_t>(EL, 4096)));
  c->cg.reset(new CgEngine());
  SBX_CUDA(cudaStreamSynchronize(c->stream));
  return SBX_OK;
}

}  // namespace

extern "C" {

sbx_status sbx_ctx_create_box_dist(const sbx_box_desc* d, const int32_t* rank_of, int nranks,
                                   int rank, int device, sbx_ctx** out) {
  if (!d || !rank_of || !out) {
    set_error("sbx_ctx_create_box_dist: null argument");
    return SBX_E_INVALID;
  }
  *out = nullptr;
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) {
    set_error("sbx_ctx_create_box_dist: 1 <= nranks <= 8 and 0 <= rank < nranks");
    return SBX_E_CONFIG;
  }
  const int counts[3] = {d->ex, d->ey, d->ez};
  for (int q = 0; q < 3; ++q)
    if (d->periodic[q] && counts[q] < 2) {
      set_error("sbx_ctx_create_box_dist: periodic directions need >= 2 elements");
      return SBX_E_CONFIG;
    }
  if (d->degree < 1 || d->degree > kMaxTemplN || !dist_k1_supported(d->degree + 1)) {
    set_error("sbx_ctx_create_box_dist: the distributed solver needs an odd degree N <= 13 "
              "(its fused K1 pipeline must fit shared memory), got N=" +
              std::to_string(d->degree));
    return SBX_E_CONFIG;
  }
  auto plan = std::make_unique<DistPlan>();
  int rc = build_dist_plan(d->ex, d->ey, d->ez, d->periodic, d->degree, rank_of, nranks, rank,
                           *plan);
  if (rc != SBX_OK) return (sbx_status)rc;
  auto* c = new sbx_ctx();
  sbx_status st = ctx_init_common(c, device);
  c->dist = true;
  c->nranks = nranks;
  c->rank = rank;
  c->local_elements = plan->loc_elems;
  if (st == SBX_OK) st = upload_dist(c, *plan, d);
  if (st != SBX_OK) {
    sbx_ctx_destroy(c);
    return st;
  }
  *out = c;
  return SBX_OK;
}

size_t sbx_ctx_dist_blob_size(int nranks) {
  (void)nranks;
  return sizeof(DistBlob);
}

sbx_status sbx_ctx_dist_blob(sbx_ctx* c, uint8_t* blob) {
  SBX_TRY(check_ctx(c));
  if (!c->dist || !blob) {
    set_error("sbx_ctx_dist_blob: not a distributed context");
    return SBX_E_INVALID;
  }
  SBX_CUDA(cudaSetDevice(c->device));
  DistBlob b;
  std::memset(&b, 0, sizeof(b));
  SBX_CUDA(cudaIpcGetMemHandle(&b.handle, c->window));
  b.recv_total = c->dd.recv_total;
  for (int q = 0; q < kMaxRanks; ++q) b.recv_base_for_src[q] = c->recv_base_for_src[q];
  std::memcpy(blob, &b, sizeof(b));
  return SBX_OK;
}

sbx_status sbx_ctx_dist_connect(sbx_ctx* c, const uint8_t* blobs) {
  SBX_TRY(check_ctx(c));
  if (!c->dist || !blobs) {
    set_error("sbx_ctx_dist_connect: not a distributed context");
    return SBX_E_INVALID;
  }
  SBX_CUDA(cudaSetDevice(c->device));
  DistDev& D = c->dd;
  for (int q = 0; q < c->nranks; ++q) {
    DistBlob b;
    std::memcpy(&b, blobs + (size_t)q * sizeof(DistBlob), sizeof(DistBlob));
    char* base = nullptr;
    if (q == c->rank) {
      base = static_cast<char*>(c->window);
    } else {
      void* p = nullptr;
      SBX_CUDA(cudaIpcOpenMemHandle(&p, b.handle, cudaIpcMemLazyEnablePeerAccess));
      c->peer_windows.push_back(p);
      base = static_cast<char*>(p);
    }
    D.pflags[q] = reinterpret_cast<unsigned long long*>(base + kWinFlags);
    D.pmbox[q] = reinterpret_cast<double*>(base + kWinMbox);
    D.precv[q] = reinterpret_cast<double*>(base + kWinRecv);
    D.precv_total[q] = b.recv_total;
    D.pbase_for_me[q] = b.recv_base_for_src[c->rank];
    if (q != c->rank) {
      // a neighbour must hold a send block for me, and I for it
      bool i_send = false;
      for (int qi = 0; qi < D.nnbr; ++qi)
        if (D.nbr[qi] == q) i_send = true;
      if (i_send != (b.recv_base_for_src[c->rank] >= 0)) {
        set_error("sbx_ctx_dist_connect: inconsistent exchange plans between ranks");
        return SBX_E_COMM;
      }
    }
  }
  // device copy of the exchange state for the fused kernels (K1 epilogue
  // sends, K2 scalar step)
  if (std::getenv("SBX_TRACE")) {
    void* tp = nullptr;
    SBX_TRY(dalloc(c, &tp, sizeof(unsigned long long) * kTraceIters * 8));
    SBX_CUDA(cudaMemset(tp, 0, sizeof(unsigned long long) * kTraceIters * 8));
    D.trace = static_cast<unsigned long long*>(tp);
  }
  void* p = nullptr;
  SBX_TRY(dalloc(c, &p, sizeof(DistDev)));
  SBX_CUDA(cudaMemcpy(p, &c->dd, sizeof(DistDev), cudaMemcpyHostToDevice));
  c->op.dd = static_cast<const DistDev*>(p);
  c->connected = true;
  return SBX_OK;
}

}  // extern "C"
