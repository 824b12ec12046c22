// Standalone operator kernels (sm_100a): axhelm, its diagonal, gather-scatter,
// reference-order and tree dot products, BLAS-1 updates.
//
// EXACT variants keep the reference's floating-point evaluation order with
// explicitly rounded operations (__dmul_rn / __dadd_rn, no FMA contraction),
// so their output is bitwise equal to sembox built for x86-64.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "ax_core.cuh"
#include "ax_tma.cuh"
#include "ax_dmma.cuh"
#include "kernels.cuh"
#include "sbx_internal.h"

namespace sbx {

namespace {

// axhelm (operators.cpp:215-263).  bm non-null adds the mass term; the exact
// variant is always given bm when present (the reference evaluates h2*bm*u
// even for h2 == 0), and adds (0*u) when absent -- same value incl. sign of 0.
template <int n, bool EXACT>
__global__ void __launch_bounds__(AxCfg<n>::threads)
    ax_kernel(const double* __restrict__ u, const double* __restrict__ G,
              const double* __restrict__ bm, double* __restrict__ w, int64_t E, double h1,
              double h2, double tsign, DParam<n> Dp) {
  using C = AxCfg<n>;
  extern __shared__ double sm[];
  double* sD = sm;
  const int t = threadIdx.x;
  const int slot = t / C::nn, ij = t % C::nn, i = ij % n, j = ij / n;
  double* su = sm + n * C::DS + slot * 3 * C::TILE;
  ax_stage_D<n>(sD, Dp);
  const int64_t e = (int64_t)blockIdx.x * C::EPB + slot;
  const bool valid = e < E;
  const int64_t base = e * C::n3;
  double uc[n];
#pragma unroll
  for (int k = 0; k < n; ++k) {
    uc[k] = valid ? __ldg(u + base + k * C::nn + ij) : 0.0;
    su[k * C::SP + j * C::SR + i] = uc[k];
  }
  double acc[n];
  ax_column<n, EXACT>(uc, su, su + C::TILE, su + 2 * C::TILE, sD,
                      G + (valid ? e : 0) * 6 * C::n3 + ij, valid, i, j, h1, tsign, Dp, acc);
  if (!valid) return;
#pragma unroll
  for (int k = 0; k < n; ++k) {
    double out;
    if constexpr (EXACT) {
      const double hb = bm ? dmul(h2, __ldg(bm + base + k * C::nn + ij)) : 0.0;
      out = dadd(acc[k], dmul(hb, uc[k]));
    } else {
      out = bm ? fma(h2 * __ldg(bm + base + k * C::nn + ij), uc[k], acc[k]) : acc[k];
    }
    w[base + k * C::nn + ij] = out;
  }
}

// Runtime-n fallback for 16 <= N <= 32 (n > 16): one element per CTA, every
// thread loops over nodes; reference evaluation order in both modes.
// Also the kernel for per-node coefficients h1f / h2f (any n): h1 and h2 read
// at each node exactly where operators.cpp:242, 258 read them.
__global__ void ax_generic_kernel(const double* __restrict__ u, const double* __restrict__ G,
                                  const double* __restrict__ bm, const double* __restrict__ D,
                                  double* __restrict__ w, int n, double h1, double h2,
                                  double tsign, const double* __restrict__ h1f = nullptr,
                                  const double* __restrict__ h2f = nullptr) {
  extern __shared__ double sm[];
  const int n3 = n * n * n;
  double* su = sm;
  double* sr = su + n3;
  double* ss = sr + n3;
  double* st = ss + n3;
  const int64_t e = blockIdx.x;
  const int64_t base = e * n3;
  const double* Ge = G + e * 6 * n3;
  for (int a = threadIdx.x; a < n3; a += blockDim.x) su[a] = u[base + a];
  __syncthreads();
  for (int a = threadIdx.x; a < n3; a += blockDim.x) {
    const int i = a % n, j = (a / n) % n, k = a / (n * n);
    double r = 0.0, s = 0.0, t = 0.0;
    for (int l = 0; l < n; ++l) {
      r = dadd(r, dmul(D[i * n + l], su[(k * n + j) * n + l]));
      s = dadd(s, dmul(D[j * n + l], su[(k * n + l) * n + i]));
      t = dadd(t, dmul(D[k * n + l], su[(l * n + j) * n + i]));
    }
    const double g1 = Ge[a], g2 = Ge[n3 + a], g3 = Ge[2 * n3 + a], g4 = Ge[3 * n3 + a],
                 g5 = Ge[4 * n3 + a], g6 = Ge[5 * n3 + a];
    const double hh = h1f ? h1f[base + a] : h1;
    sr[a] = dmul(dadd(dadd(dmul(g1, r), dmul(g4, s)), dmul(g5, t)), hh);
    ss[a] = dmul(dadd(dadd(dmul(g2, s), dmul(g4, r)), dmul(g6, t)), hh);
    st[a] = dmul(dadd(dadd(dmul(g3, t), dmul(g5, r)), dmul(g6, s)), hh);
  }
  __syncthreads();
  for (int a = threadIdx.x; a < n3; a += blockDim.x) {
    const int i = a % n, j = (a / n) % n, k = a / (n * n);
    double acc = 0.0;
    for (int l = 0; l < n; ++l) {
      const double t1 = dmul(D[l * n + i], sr[(k * n + j) * n + l]);
      const double t2 = dmul(D[l * n + j], ss[(k * n + l) * n + i]);
      const double t3 = dmul(dmul(tsign, D[l * n + k]), st[(l * n + j) * n + i]);
      acc = dadd(acc, dadd(dadd(t1, t2), t3));
    }
    const double hb = bm ? dmul(h2f ? h2f[base + a] : h2, bm[base + a]) : 0.0;
    w[base + a] = dadd(acc, dmul(hb, su[a]));
  }
}

// Standalone FAST axhelm on the persistent TMA pipeline (ax_tma.cuh): stages
// the packed G, u [, bm] per element; w = h1*DᵀGDu (+ h2*bm*u).  64 / 72
// algorithmic B/node (Poisson / Helmholtz).
template <bool HAS_BM>
struct AxPol {
  static constexpr int NV = HAS_BM ? 2 : 1;
  static constexpr int BMQ = HAS_BM ? 1 : -1;
  struct Args {
    const double* u;
    const double* bm;
    double* w;
    double h2;
  };
  __device__ static bool init_ptrs(Args&) { return true; }
  __device__ static bool init_scalars(Args&) { return true; }
  __device__ static double* partials_of(const Args&, double* partials) { return partials; }
  __device__ static const int32_t* send_index(const Args&) { return nullptr; }
  __device__ static void element_done(Args&, int, int64_t, int, int, int, int, int) {}
  __device__ static const double* vec(const Args& a, int q) { return q == 0 ? a.u : a.bm; }
  __device__ static void pro(const Args& a, const double (&v)[NV], int64_t, double& u,
                             double& hb) {
    u = v[0];
    hb = HAS_BM ? a.h2 * v[NV - 1] : 0.0;
  }
  __device__ static double hb_of(const Args& a, double bm) { return a.h2 * bm; }
  __device__ static void epi(const Args& a, double acc, double u, double hb, int64_t idx,
                             double&) {
    a.w[idx] = HAS_BM ? fma(hb, u, acc) : acc;
  }
  __device__ static void finish(const Args&, double, double*, double*, bool*) {}
};

template <int n, bool HAS_BM>
cudaError_t launch_ax_tma(const OpDev& op, const double* u, double* w, double h1, double h2,
                          double tsign, cudaStream_t s) {
  using Pol = AxPol<HAS_BM>;
  using Ch = TmaChoice<n, Pol::NV>;
  if constexpr (!Ch::ok) {
    return cudaErrorNotSupported;
  } else {
    using L = TmaLayout<n, Pol::NV, Ch::GROUPS, Ch::S>;
    auto kern = ax_tma_kernel<n, Pol, Ch::GROUPS, Ch::S>;
    static std::atomic<bool> attr_set[64];  // per device (distinct contexts may race: idempotent)
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
      cudaError_t err =
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::smem);
      if (err != cudaSuccess) return err;
      attr_set[dev & 63] = true;
    }
    static std::atomic<int> sms[64];
    if (!sms[dev & 63]) {
      int v = 0;
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
      sms[dev & 63] = v;
    }
    DParam<n> Dp;
    for (int q = 0; q < n * n; ++q) Dp.d[q] = op.Dh[q];
    QParam<n> Qp{};
    typename Pol::Args a{u, op.bm, w, h2};
    const int64_t NG = (op.E + TmaGeom<n>::EPG - 1) / TmaGeom<n>::EPG;
    const int nsm = sms[dev & 63];
    int64_t grid = nsm > 0 ? nsm : 148;
    if (grid > NG) grid = NG;
    kern<<<(unsigned)grid, L::threads, L::smem, s>>>(a, op.G, op.E, h1, tsign, Dp, nullptr, Qp);
    return cudaGetLastError();
  }
}

inline bool al16(const void* p) { return p == nullptr || ((uintptr_t)p & 15) == 0; }

// n = 8: the operator on the FP64 tensor cores (ax_dmma.cuh), stored geometry
template <bool HAS_BM>
cudaError_t launch_ax_dmma(const OpDev& op, const double* u, double* w, double h1, double h2,
                           double tsign, cudaStream_t s) {
  using L = AxDmmaLayout<HAS_BM>;
  auto kern = ax_dmma_kernel<HAS_BM>;
  static std::atomic<bool> attr_set[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    cudaError_t err =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::smem);
    if (err != cudaSuccess) return err;
    attr_set[dev & 63] = true;
  }
  static std::atomic<int> sms[64];
  if (!sms[dev & 63]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms[dev & 63] = v;
  }
  DParam<8> Dp;
  for (int q = 0; q < 64; ++q) Dp.d[q] = op.Dh[q];
  const int nsm = sms[dev & 63];
  int64_t grid = nsm > 0 ? nsm : 148;
  if (grid > op.E) grid = op.E;
  kern<<<(unsigned)grid, L::threads, L::smem, s>>>(u, op.G, op.bm, w, op.E, h1, h2, tsign, Dp);
  return cudaGetLastError();
}

template <int n, bool EXACT>
cudaError_t launch_ax_t(const OpDev& op, const double* u, double* w, double h1, double h2,
                        double tsign, cudaStream_t s) {
  using C = AxCfg<n>;
  static const bool no_tma = std::getenv("SBX_NO_TMA") != nullptr;
  if (!EXACT && !no_tma && n % 2 == 0 && al16(u) && al16(w) && al16(op.G) &&
      (h2 == 0.0 || al16(op.bm))) {
    static const bool fma_ax = std::getenv("SBX_K1_FMA") != nullptr;
    if constexpr (n == 8) {
      if (!fma_ax)
        return h2 != 0.0 ? launch_ax_dmma<true>(op, u, w, h1, h2, tsign, s)
                         : launch_ax_dmma<false>(op, u, w, h1, h2, tsign, s);
    }
    const cudaError_t e = h2 != 0.0 ? launch_ax_tma<n, true>(op, u, w, h1, h2, tsign, s)
                                    : launch_ax_tma<n, false>(op, u, w, h1, h2, tsign, s);
    if (e != cudaErrorNotSupported) return e;
  }
  static std::atomic<bool> attr_set[64];  // per device (distinct contexts may race: idempotent)
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    cudaError_t err = cudaFuncSetAttribute(ax_kernel<n, EXACT>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)C::smem);
    if (err != cudaSuccess) return err;
    attr_set[dev & 63] = true;
  }
  DParam<n> Dp;
  for (int q = 0; q < n * n; ++q) Dp.d[q] = op.Dh[q];
  const int64_t blocks = (op.E + C::EPB - 1) / C::EPB;
  // bm is read only when the mass term is active (h2 != 0), or always in the
  // exact variant (the reference evaluates h2*bm*u even for h2 == 0).
  const double* bm = (EXACT || h2 != 0.0) ? op.bm : nullptr;
  ax_kernel<n, EXACT><<<(unsigned)blocks, C::threads, C::smem, s>>>(u, op.G, bm, w, op.E, h1,
                                                                    h2, tsign, Dp);
  return cudaGetLastError();
}

// ---- axhelm diagonal (operators.cpp:272-298), reference order -------------
__global__ void ax_diag_kernel(const double* __restrict__ G, const double* __restrict__ bm,
                               const double* __restrict__ D, int n, int64_t nodes, double h1,
                               double h2, double* __restrict__ diag,
                               const double* __restrict__ h1f, const double* __restrict__ h2f) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= nodes) return;
  const int n3 = n * n * n;
  const int64_t e = a / n3;
  const int loc = (int)(a - e * n3);
  const int i = loc % n, j = (loc / n) % n, k = loc / (n * n);
  const double* Ge = G + e * 6 * n3;
  double s = 0.0;
  for (int l = 0; l < n; ++l) {
    s = dadd(s, dmul(dmul(D[l * n + i], D[l * n + i]), Ge[(k * n + j) * n + l]));
    s = dadd(s, dmul(dmul(D[l * n + j], D[l * n + j]), Ge[n3 + (k * n + l) * n + i]));
    s = dadd(s, dmul(dmul(D[l * n + k], D[l * n + k]), Ge[2 * n3 + (l * n + j) * n + i]));
  }
  s = dadd(s, dmul(dmul(dmul(2.0, D[i * n + i]), D[j * n + j]), Ge[3 * n3 + loc]));
  s = dadd(s, dmul(dmul(dmul(2.0, D[i * n + i]), D[k * n + k]), Ge[4 * n3 + loc]));
  s = dadd(s, dmul(dmul(dmul(2.0, D[j * n + j]), D[k * n + k]), Ge[5 * n3 + loc]));
  const double b = bm ? bm[a] : 0.0;
  diag[a] = dadd(dmul(h1f ? h1f[a] : h1, s), dmul(h2f ? h2f[a] : h2, b));
}

// ---- gather-scatter over the boundary CSR (gather.cpp:85-98) --------------
// One thread per group; copies summed from 0.0 in group order, so the result
// is bitwise the reference's.  Masked copies (index ~a) get s*0.0 when
// apply_mask (HelmholtzOperator::apply multiplies by the 0/1 mask, and
// s*1.0 == s bitwise).
__global__ void gs_kernel(const int32_t* __restrict__ off, const int32_t* __restrict__ idx,
                          int64_t nB, double* __restrict__ f, int apply_mask) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nB) return;
  const int lo = off[g], hi = off[g + 1];
  if (hi - lo == 1) {
    const int32_t c = idx[lo];
    if (apply_mask && c < 0) f[~c] = dmul(f[~c], 0.0);
    return;
  }
  double s = 0.0;
  for (int c = lo; c < hi; ++c) {
    const int32_t a = idx[c];
    s = dadd(s, f[a < 0 ? ~a : a]);
  }
  for (int c = lo; c < hi; ++c) {
    const int32_t a = idx[c];
    if (a >= 0)
      f[a] = s;
    else
      f[~a] = apply_mask ? dmul(s, 0.0) : s;
  }
}

// ---- reference-order dot (field.cpp:13-22, 59-81) -------------------------
__global__ void dot_elem_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                const double* __restrict__ w, int64_t E, int nper,
                                double* __restrict__ partial) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int64_t base = e * nper;
  double p = 0.0;
  if (w)
    for (int q = 0; q < nper; ++q) p = dadd(p, dmul(dmul(a[base + q], b[base + q]), w[base + q]));
  else
    for (int q = 0; q < nper; ++q) p = dadd(p, dmul(a[base + q], b[base + q]));
  partial[e] = p;
}

__global__ void serial_sum_kernel(const double* __restrict__ partial, int64_t E,
                                  double* __restrict__ out) {
  double s = 0.0;
  for (int64_t e = 0; e < E; ++e) s = dadd(s, partial[e]);
  *out = s;
}

// ---- deterministic tree dot ---------------------------------------------
constexpr int kDotThreads = 256;
constexpr int kDotMaxBlocks = 1184;  // 8 per SM on 148 SMs

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  v = threadIdx.x < nw ? sh[threadIdx.x] : 0.0;
  if (wid == 0) v = warp_sum(v);
  __syncthreads();
  return v;
}

__global__ void __launch_bounds__(kDotThreads)
    dot_fast_kernel(int64_t N, const double* __restrict__ a, const double* __restrict__ b,
                    const double* __restrict__ w, double* __restrict__ partials,
                    uint32_t* __restrict__ counter, double* __restrict__ out) {
  __shared__ double sh[32];
  __shared__ bool last;
  double v = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < N;
       q += (int64_t)gridDim.x * blockDim.x)
    v += w ? a[q] * b[q] * w[q] : a[q] * b[q];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = v;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    double s = 0.0;
    for (int q = threadIdx.x; q < (int)gridDim.x; q += blockDim.x) s += partials[q];
    s = block_sum(s, sh);
    if (threadIdx.x == 0) {
      *out = s;
      *counter = 0;
    }
  }
}

// ---- BLAS-1 (field.cpp:32-57), reference rounding -------------------------
__global__ void axpy_kernel(int64_t N, double alpha, const double* __restrict__ x,
                            double* __restrict__ y) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < N;
       q += (int64_t)gridDim.x * blockDim.x)
    y[q] = dadd(y[q], dmul(alpha, x[q]));
}
__global__ void scale_kernel(int64_t N, double alpha, double* __restrict__ y) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < N;
       q += (int64_t)gridDim.x * blockDim.x)
    y[q] = dmul(y[q], alpha);
}
__global__ void div_kernel(int64_t N, const double* __restrict__ r, const double* __restrict__ d,
                           double* __restrict__ z) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < N;
       q += (int64_t)gridDim.x * blockDim.x)
    z[q] = __ddiv_rn(r[q], d[q]);
}
__global__ void mul_kernel(int64_t N, const double* __restrict__ a, double* __restrict__ b) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < N;
       q += (int64_t)gridDim.x * blockDim.x)
    b[q] = dmul(b[q], a[q]);
}
__global__ void recip_kernel(int64_t N, const double* __restrict__ d, double* __restrict__ o) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < N;
       q += (int64_t)gridDim.x * blockDim.x)
    o[q] = __ddiv_rn(1.0, d[q]);
}

// SoA g1..g6 (reference layout) -> packed [E][6][n^3]
__global__ void pack_geometry_kernel(const double* __restrict__ g1, const double* __restrict__ g2,
                                     const double* __restrict__ g3, const double* __restrict__ g4,
                                     const double* __restrict__ g5, const double* __restrict__ g6,
                                     int64_t nodes, int n3, double* __restrict__ G) {
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < nodes;
       a += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = a / n3, l = a - e * n3;
    double* o = G + e * 6 * n3 + l;
    o[0] = g1[a];
    o[n3] = g2[a];
    o[2 * n3] = g3[a];
    o[3 * n3] = g4[a];
    o[4 * n3] = g5[a];
    o[5 * n3] = g6[a];
  }
}

inline unsigned grid_for(int64_t N, int threads) {
  int64_t b = (N + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  if (b < 1) b = 1;
  return (unsigned)b;
}

}  // namespace

cudaError_t launch_axhelm(const OpDev& op, const double* u, double* w, double h1, double h2,
                          bool exact, bool flip, cudaStream_t s) {
  const double tsign = flip ? -1.0 : 1.0;
  if (op.E == 0) return cudaSuccess;
  const int N = op.n - 1;
  if (N > kMaxTemplN || op.h1f || op.h2f) {  // (per-node coefficients: the reference order)
    const int n3 = op.n * op.n * op.n;
    const size_t smem = (size_t)4 * n3 * sizeof(double);
    cudaError_t err = cudaFuncSetAttribute(
        ax_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    const double* bm = (exact || h2 != 0.0 || op.h2f) ? op.bm : nullptr;
    ax_generic_kernel<<<(unsigned)op.E, 256, smem, s>>>(u, op.G, bm, op.Dd, w, op.n, h1, h2,
                                                        tsign, op.h1f, op.h2f);
    return cudaGetLastError();
  }
#define SBX_AX_CASE(NN)                                                                  \
  case NN:                                                                               \
    return exact ? launch_ax_t<NN + 1, true>(op, u, w, h1, h2, tsign, s)                 \
                 : launch_ax_t<NN + 1, false>(op, u, w, h1, h2, tsign, s);
  switch (N) {
    SBX_AX_CASE(1)
    SBX_AX_CASE(2)
    SBX_AX_CASE(3)
    SBX_AX_CASE(4)
    SBX_AX_CASE(5)
    SBX_AX_CASE(6)
    SBX_AX_CASE(7)
    SBX_AX_CASE(8)
    SBX_AX_CASE(9)
    SBX_AX_CASE(10)
    SBX_AX_CASE(11)
    SBX_AX_CASE(12)
    SBX_AX_CASE(13)
    SBX_AX_CASE(14)
    SBX_AX_CASE(15)
    default:
      return cudaErrorInvalidValue;
  }
#undef SBX_AX_CASE
}

cudaError_t launch_axhelm_diag(const OpDev& op, double h1, double h2, double* diag,
                               cudaStream_t s) {
  if (op.nodes == 0) return cudaSuccess;
  ax_diag_kernel<<<(unsigned)((op.nodes + 255) / 256), 256, 0, s>>>(
      op.G, op.bm, op.Dd, op.n, op.nodes, h1, h2, diag, op.h1f, op.h2f);
  return cudaGetLastError();
}

cudaError_t launch_gs(const OpDev& op, double* f, bool apply_mask, cudaStream_t s) {
  if (op.lat) return launch_gs_box(op, f, apply_mask, s);
  if (op.nB == 0) return cudaSuccess;
  gs_kernel<<<(unsigned)((op.nB + 255) / 256), 256, 0, s>>>(op.b_off, op.b_idx, op.nB, f,
                                                            apply_mask ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_dot_exact_n(int64_t E, int nper, const double* a, const double* b,
                               double* partials, double* out, cudaStream_t s) {
  dot_elem_kernel<<<(unsigned)((E + 127) / 128), 128, 0, s>>>(a, b, nullptr, E, nper, partials);
  serial_sum_kernel<<<1, 1, 0, s>>>(partials, E, out);
  return cudaGetLastError();
}

cudaError_t launch_dot_exact(const OpDev& op, const double* a, const double* b,
                             const double* w, double* partials, double* out, cudaStream_t s) {
  const int nper = op.n * op.n * op.n;
  dot_elem_kernel<<<(unsigned)((op.E + 127) / 128), 128, 0, s>>>(a, b, w, op.E, nper, partials);
  serial_sum_kernel<<<1, 1, 0, s>>>(partials, op.E, out);
  return cudaGetLastError();
}

cudaError_t launch_dot_fast(int64_t N, const double* a, const double* b, const double* w,
                            double* partials, uint32_t* counter, double* out, cudaStream_t s) {
  int64_t blocks = (N + kDotThreads * 4 - 1) / (kDotThreads * 4);
  if (blocks > kDotMaxBlocks) blocks = kDotMaxBlocks;
  if (blocks < 1) blocks = 1;
  dot_fast_kernel<<<(unsigned)blocks, kDotThreads, 0, s>>>(N, a, b, w, partials, counter, out);
  return cudaGetLastError();
}

cudaError_t launch_axpy(int64_t N, double alpha, const double* x, double* y, cudaStream_t s) {
  axpy_kernel<<<grid_for(N, 256), 256, 0, s>>>(N, alpha, x, y);
  return cudaGetLastError();
}
cudaError_t launch_scale(int64_t N, double alpha, double* y, cudaStream_t s) {
  scale_kernel<<<grid_for(N, 256), 256, 0, s>>>(N, alpha, y);
  return cudaGetLastError();
}
cudaError_t launch_div(int64_t N, const double* r, const double* d, double* z, cudaStream_t s) {
  div_kernel<<<grid_for(N, 256), 256, 0, s>>>(N, r, d, z);
  return cudaGetLastError();
}
cudaError_t launch_mul(int64_t N, const double* a, double* b, cudaStream_t s) {
  mul_kernel<<<grid_for(N, 256), 256, 0, s>>>(N, a, b);
  return cudaGetLastError();
}
cudaError_t launch_recip(int64_t N, const double* d, double* dinv, cudaStream_t s) {
  recip_kernel<<<grid_for(N, 256), 256, 0, s>>>(N, d, dinv);
  return cudaGetLastError();
}
cudaError_t launch_pack_geometry(const OpDev& op, const double* const* g, double* G,
                                 cudaStream_t s) {
  const int n3 = op.n * op.n * op.n;
  pack_geometry_kernel<<<grid_for(op.nodes, 256), 256, 0, s>>>(g[0], g[1], g[2], g[3], g[4],
                                                               g[5], op.nodes, n3, G);
  return cudaGetLastError();
}

}  // namespace sbx
