// Consistent-Poisson pressure operator E = Div M^-1 QQ^T Grad on the
// P_N / P_N-2 staggered grid, and its PCG, for sm_100a.
//
//   gradient_from_pressure   operators.cpp:365-410   p_grad_kernel
//   divergence_to_pressure   operators.cpp:327-363   p_div_kernel
//   apply_pressure_operator  stepper.cpp:240-248     grad -> gs + inv_bdiag -> div
//   pressure_operator_diagonal stepper.cpp:250-275   p_diag_kernel (closed form)
//   solve_pressure_update's pcg stepper.cpp:277-348  the fused loop below
//
// Both element operators are sums of nine 3-D tensor contractions between the
// GL (m = N-1 points) and GLL (n = N+1) grids: along the derivative direction
// the 1-D operator is I D (m x n; interpolation after the GLL derivative) or
// its transpose, along the other two the interpolation I or I^T.  The
// pressure geometry (GL weight x detJ x dr/dx) is never stored: at a GL node it
// is w_ijk adj(J), the adjugate rows c1 x c2, c2 x c0, c0 x c1 of the
// element's trilinear map (the detJ of wdetj and the 1/detJ of dr/dx
// cancel), formed from the 24 map coefficients the CG kernels already use.
// One CTA per element; the contractions run out of shared memory (FAST mode:
// the reference's numbers to rounding, tests/test_gpu_pressure.py).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>

#include "kernels.cuh"
#include "pressure.cuh"
#include "sbx_internal.h"
#include "tma.cuh"

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace sbx {

namespace {

// one of three component pointers (a runtime index into a local pointer
// array would put the array in local memory)
template <class T>
__device__ __forceinline__ T* pick3(T* a, T* b, T* c, int i) {
  return i == 0 ? a : (i == 1 ? b : c);
}


constexpr int kPThreads = 128;

// 1-D operators in device memory, staged into shared memory per CTA:
// It, Ct (n x m: I^T, (I D)^T), I, CI (m x n: I, I D), GL weights w[m], nodes x[m]
template <int n>
struct PMat {
  static constexpr int m = n - 2;
  static constexpr int OFF_IT = 0, OFF_CT = n * m, OFF_I = 2 * n * m, OFF_CI = 3 * n * m;
  static constexpr int OFF_W = 4 * n * m, OFF_X = 4 * n * m + m;
  static constexpr int SIZE = 4 * n * m + 2 * m;
};

__device__ __forceinline__ void pcross(const double (&x)[3], const double (&y)[3],
                                       double (&o)[3]) {
  o[0] = x[1] * y[2] - x[2] * y[1];
  o[1] = x[2] * y[0] - x[0] * y[2];
  o[2] = x[0] * y[1] - x[1] * y[0];
}

// w_q * adj(J) at GL node (qi, qj, qk) of element e: F[pd*3 + comp] =
// wdetj * dr_pd/dx_comp (operators.cpp:180-214 with the det cancelled)
__device__ __forceinline__ void gl_metric(const double* __restrict__ tl, const double* sX,
                                          const double* sW, int qi, int qj, int qk,
                                          double (&F)[9]) {
  const double r = sX[qi], s = sX[qj], t = sX[qk];
  double c0[3], c1[3], c2[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const double S0 = tl[q], S1 = tl[3 + q], S2 = tl[6 + q], S01 = tl[9 + q], S02 = tl[12 + q],
                 S12 = tl[15 + q], S012 = tl[18 + q];
    c0[q] = S0 + S01 * s + S02 * t + S012 * s * t;
    c1[q] = S1 + S01 * r + S12 * t + S012 * r * t;
    c2[q] = S2 + S02 * r + S12 * s + S012 * r * s;
  }
  double a0[3], a1[3], a2[3];
  pcross(c1, c2, a0);
  pcross(c2, c0, a1);
  pcross(c0, c1, a2);
  const double w = sW[qi] * sW[qj] * sW[qk];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    F[q] = w * a0[q];
    F[3 + q] = w * a1[q];
    F[6 + q] = w * a2[q];
  }
}

template <int n>
struct PGradSmem {
  static constexpr int m = n - 2, m3 = m * m * m;
  static constexpr int T_D = 3 * m3;          // t_pd = F[pd][comp] p
  static constexpr int A_D = 3 * m * m * n;   // after the z pass
  static constexpr int B_D = 2 * m * n * n;   // after the y pass
  static constexpr size_t bytes = sizeof(double) * (PMat<n>::SIZE + T_D + A_D + B_D);
};

// CG prologue of the pressure loop, fused into the gradient: z = M r with the
// mean deflation of pressure_precond (z = r/diag - mu), p = z + beta p_old,
// x += alpha_prev p_old; p is written and is the operand.
struct PCgArgs {
  const double* r;
  const double* dinv;  // null: no preconditioner (deflation only)
  double* p;
  double* x;
  const CgScalars* sc;
};

// gradient_from_pressure: p (E m^3) -> g0, g1, g2 (E n^3 each)
template <int n, bool CG>
__global__ void __launch_bounds__(kPThreads)
    p_grad_kernel(const double* __restrict__ pin, int64_t E, const double* __restrict__ TL,
                  const double* __restrict__ mats, double* __restrict__ g0,
                  double* __restrict__ g1, double* __restrict__ g2, PCgArgs cg) {
  using S = PGradSmem<n>;
  using PM = PMat<n>;
  constexpr int m = n - 2, m3 = m * m * m, n3 = n * n * n;
  constexpr int QPT = (m3 + kPThreads - 1) / kPThreads;  // GL nodes per thread
  extern __shared__ double psm[];
  double* sM = psm;
  double* sT = sM + PM::SIZE;
  double* sA = sT + S::T_D;
  double* sB = sA + S::A_D;
  if (CG && cg.sc->done) return;
  for (int q = threadIdx.x; q < PM::SIZE; q += blockDim.x) sM[q] = mats[q];
  double beta = 0.0, ap = 0.0, mu = 0.0;
  int first = 1;
  if constexpr (CG) {
    beta = cg.sc->beta;
    ap = cg.sc->alpha_prev;
    mu = cg.sc->mu;
    first = cg.sc->first;
  }
  __syncthreads();
  const double* sIt = sM + PM::OFF_IT;
  const double* sCt = sM + PM::OFF_CT;
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    // per owned GL node: the operand p and the nine metric factors
    double pv[QPT], F[QPT][9];
#pragma unroll
    for (int u = 0; u < QPT; ++u) {
      const int q = threadIdx.x + u * kPThreads;
      pv[u] = 0.0;
      if (q < m3) {
        const int qi = q % m, qj = (q / m) % m, qk = q / (m * m);
        gl_metric(TL + e * 24, sM + PM::OFF_X, sM + PM::OFF_W, qi, qj, qk, F[u]);
        const int64_t a = e * m3 + q;
        if constexpr (CG) {
          const double rv = cg.r[a];
          const double z = (cg.dinv ? rv * cg.dinv[a] : rv) - mu;
          double pn = z;
          if (!first) {
            const double po = cg.p[a];
            pn = fma(beta, po, z);
            cg.x[a] = fma(ap, po, cg.x[a]);
          }
          cg.p[a] = pn;
          pv[u] = pn;
        } else {
          pv[u] = pin[a];
        }
      }
    }
    for (int comp = 0; comp < 3; ++comp) {
      __syncthreads();  // previous component's passes are done with sT / sA / sB
#pragma unroll
      for (int u = 0; u < QPT; ++u) {
        const int q = threadIdx.x + u * kPThreads;
        if (q < m3) {
#pragma unroll
          for (int pd = 0; pd < 3; ++pd) sT[pd * m3 + q] = F[u][pd * 3 + comp] * pv[u];
        }
      }
      __syncthreads();
      // z pass: A_pd[kz][jj][ii] = sum_kk Mz_pd[kz][kk] t_pd[kk][jj][ii]
      for (int idx = threadIdx.x; idx < 3 * m * m * n; idx += blockDim.x) {
        const int pd = idx / (m * m * n), rem = idx - pd * (m * m * n);
        const int kz = rem / (m * m), jjii = rem - kz * (m * m);
        const double* Mz = (pd == 2 ? sCt : sIt) + kz * m;
        const double* t = sT + pd * m3 + jjii;
        double acc = 0.0;
#pragma unroll
        for (int kk = 0; kk < m; ++kk) acc = fma(Mz[kk], t[kk * m * m], acc);
        sA[idx] = acc;
      }
      __syncthreads();
      // y pass: B0 = Iy A0 ; B12 = Cy A1 + Iy A2   ([kz][jy][ii])
      for (int idx = threadIdx.x; idx < 2 * m * n * n; idx += blockDim.x) {
        const int which = idx / (m * n * n), rem = idx - which * (m * n * n);
        const int kz = rem / (n * m), jy = (rem / m) % n, ii = rem % m;
        const double* It = sIt + jy * m;
        const double* Ct = sCt + jy * m;
        double acc = 0.0;
        if (which == 0) {
          const double* a0 = sA + kz * m * m + ii;
#pragma unroll
          for (int jj = 0; jj < m; ++jj) acc = fma(It[jj], a0[jj * m], acc);
        } else {
          const double* a1 = sA + m * m * n + kz * m * m + ii;
          const double* a2 = sA + 2 * m * m * n + kz * m * m + ii;
#pragma unroll
          for (int jj = 0; jj < m; ++jj) {
            acc = fma(Ct[jj], a1[jj * m], acc);
            acc = fma(It[jj], a2[jj * m], acc);
          }
        }
        sB[idx] = acc;
      }
      __syncthreads();
      // x pass: g = Cx B0 + Ix B12, written straight to global
      double* out = pick3(g0, g1, g2, comp) + e * n3;
      for (int idx = threadIdx.x; idx < n3; idx += blockDim.x) {
        const int ix = idx % n, kzjy = idx / n;
        const double* Ct = sCt + ix * m;
        const double* It = sIt + ix * m;
        const double* b0 = sB + kzjy * m;
        const double* b12 = sB + m * n * n + kzjy * m;
        double acc = 0.0;
#pragma unroll
        for (int ii = 0; ii < m; ++ii) {
          acc = fma(Ct[ii], b0[ii], acc);
          acc = fma(It[ii], b12[ii], acc);
        }
        out[idx] = acc;
      }
    }
    __syncthreads();
  }
}

template <int n>
struct PDivSmem {
  static constexpr int m = n - 2;
  static constexpr int V_D = n * n * n;
  static constexpr int X_D = 2 * n * n * m;
  static constexpr int Y_D = 3 * n * m * m;
  static constexpr size_t bytes = sizeof(double) * (PMat<n>::SIZE + V_D + X_D + Y_D);
};

// divergence_to_pressure: v0, v1, v2 (E n^3) -> q (E m^3).  With `pdot`
// (the CG loop): per-CTA partials of p'q into partials[], and the last CTA
// forms alpha = rz / p'q (breakdown test as krylov.cpp:61-64).
template <int n, bool CG>
__global__ void __launch_bounds__(kPThreads)
    p_div_kernel(const double* __restrict__ v0, const double* __restrict__ v1,
                 const double* __restrict__ v2, int64_t E, const double* __restrict__ TL,
                 const double* __restrict__ mats, double* __restrict__ qout,
                 const double* __restrict__ pdot, double* __restrict__ partials,
                 CgScalars* __restrict__ sc) {
  using S = PDivSmem<n>;
  using PM = PMat<n>;
  constexpr int m = n - 2, m3 = m * m * m, n3 = n * n * n;
  constexpr int QPT = (m3 + kPThreads - 1) / kPThreads;
  extern __shared__ double psm[];
  __shared__ double red[32];
  __shared__ bool is_last;
  double* sM = psm;
  double* sV = sM + PM::SIZE;
  double* sX = sV + S::V_D;
  double* sY = sX + S::X_D;
  if (CG && sc->done) return;
  for (int q = threadIdx.x; q < PM::SIZE; q += blockDim.x) sM[q] = mats[q];
  __syncthreads();
  const double* sI = sM + PM::OFF_I;
  const double* sCI = sM + PM::OFF_CI;
  double pq = 0.0;
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    double acc[QPT], F[QPT][9];
#pragma unroll
    for (int u = 0; u < QPT; ++u) {
      const int q = threadIdx.x + u * kPThreads;
      acc[u] = 0.0;
      if (q < m3)
        gl_metric(TL + e * 24, sM + PM::OFF_X, sM + PM::OFF_W, q % m, (q / m) % m, q / (m * m),
                  F[u]);
    }
    for (int comp = 0; comp < 3; ++comp) {
      __syncthreads();
      const double* vin = pick3(v0, v1, v2, comp) + e * n3;
      for (int idx = threadIdx.x; idx < n3; idx += blockDim.x) sV[idx] = vin[idx];
      __syncthreads();
      // x pass: X0 = CIx v, X12 = Ix v   ([k][j][a])
      for (int idx = threadIdx.x; idx < 2 * n * n * m; idx += blockDim.x) {
        const int which = idx / (n * n * m), rem = idx - which * (n * n * m);
        const int kj = rem / m, a = rem % m;
        const double* Mx = (which == 0 ? sCI : sI) + a * n;
        const double* v = sV + kj * n;
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < n; ++i) s = fma(Mx[i], v[i], s);
        sX[idx] = s;
      }
      __syncthreads();
      // y pass: Y0 = Iy X0, Y1 = CIy X12, Y2 = Iy X12   ([k][b][a])
      for (int idx = threadIdx.x; idx < 3 * n * m * m; idx += blockDim.x) {
        const int which = idx / (n * m * m), rem = idx - which * (n * m * m);
        const int k = rem / (m * m), b = (rem / m) % m, a = rem % m;
        const double* My = (which == 1 ? sCI : sI) + b * n;
        const double* x = sX + (which == 0 ? 0 : n * n * m) + k * n * m + a;
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < n; ++j) s = fma(My[j], x[j * m], s);
        sY[idx] = s;
      }
      __syncthreads();
      // z pass at the thread's own GL nodes: R_p = Mz_p Y_p, then the metric
#pragma unroll
      for (int u = 0; u < QPT; ++u) {
        const int q = threadIdx.x + u * kPThreads;
        if (q < m3) {
          const int ba = q % (m * m), c = q / (m * m);
          const double* Iz = sI + c * n;
          const double* CIz = sCI + c * n;
          double r0 = 0.0, r1 = 0.0, r2 = 0.0;
#pragma unroll
          for (int k = 0; k < n; ++k) {
            r0 = fma(Iz[k], sY[k * m * m + ba], r0);
            r1 = fma(Iz[k], sY[n * m * m + k * m * m + ba], r1);
            r2 = fma(CIz[k], sY[2 * n * m * m + k * m * m + ba], r2);
          }
          acc[u] = fma(F[u][0 * 3 + comp], r0,
                       fma(F[u][1 * 3 + comp], r1, fma(F[u][2 * 3 + comp], r2, acc[u])));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < QPT; ++u) {
      const int q = threadIdx.x + u * kPThreads;
      if (q < m3) {
        const int64_t a = e * m3 + q;
        qout[a] = acc[u];
        if (CG) pq = fma(pdot[a], acc[u], pq);
      }
    }
  }
  if constexpr (CG) {
    pq = [&] {
      double v = pq;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
      __syncthreads();
      if (lane == 0) red[wid] = v;
      __syncthreads();
      v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
      if (wid == 0)
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      return v;
    }();
    if (threadIdx.x == 0) partials[blockIdx.x] = pq;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      is_last = atomicAdd(&sc->counter[0], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last || threadIdx.x != 0) return;
    __threadfence();
    double tot = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) tot += partials[b];
    sc->counter[0] = 0;
    sc->pq = tot;
    if (!isfinite(tot) || tot <= 0.0) {
      sc->status = 5;
      sc->err_it = sc->it;
      sc->done = 1;
    } else {
      sc->alpha = sc->rz / tot;
    }
  }
}

// ---- pencil kernels (n <= 10): each thread owns a 1-D pencil of a pass, its
// inputs in registers, the 1-D operator as compile-time constant-bank operands
// (kernel parameters), every component of a pass in flight at once
// (CP = 3) or one component per pass (CP = 1, less shared memory).
#ifndef SBX_PENCIL_MINB
#define SBX_PENCIL_MINB 1  // resident CTAs per SM the pencil kernels are compiled for (A/B knob)
#endif
#ifndef SBX_PENCIL_THREADS
#define SBX_PENCIL_THREADS 192  // threads per CTA of the pencil kernels (A/B: 128 / 192 / 256 -> 14.2 / 13.7 / 18.0 ms per pressure iteration at 64^3)
#endif

template <int n>
struct PMatK {
  static constexpr int m = n - 2;
  double It[n * m], Ct[n * m];  // I^T, (I D)^T   [n][m]
  double I[m * n], CI[m * n];   // I, I D         [m][n]
  double w[m], x[m];            // GL weights, nodes
};

template <int n, int CP>
struct PGrad2 {
  static constexpr int m = n - 2, m2 = m * m, m3 = m2 * m;
  static constexpr int F_D = 9 * m3, P_D = m3, A_D = 3 * CP * n * m2, B_D = 2 * CP * n * n * m;
  static constexpr size_t bytes = sizeof(double) * (F_D + P_D + A_D + B_D);
};

template <int n, int CP, bool CG>
__global__ void __launch_bounds__(SBX_PENCIL_THREADS, SBX_PENCIL_MINB)
    p_grad2_kernel(const double* __restrict__ pin, int64_t E, const double* __restrict__ TL,
                   PMatK<n> M, double* __restrict__ g0, double* __restrict__ g1,
                   double* __restrict__ g2, PCgArgs cg) {
  using S = PGrad2<n, CP>;
  constexpr int m = n - 2, m2 = m * m, m3 = m2 * m, n3 = n * n * n;
  extern __shared__ double psm[];
  double* sF = psm;          // [9][m3]: F[pd*3 + comp]
  double* sp = sF + S::F_D;  // [m3]
  double* sA = sp + S::P_D;  // [CP][3][n][m][m]  (kz, jj, ii)
  double* sB = sA + S::A_D;  // [CP][2][n][n][m]  (kz, jy, ii)
  // GL nodes / weights in shared memory (compile-time indices into the
  // parameter; a runtime index would copy it to local memory)
  __shared__ double sGx[n], sGw[n];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < m; ++q) {
      sGx[q] = M.x[q];
      sGw[q] = M.w[q];
    }
  }
  __syncthreads();
  if (CG && cg.sc->done) return;
  double beta = 0.0, ap = 0.0, mu = 0.0;
  int first = 1;
  if constexpr (CG) {
    beta = cg.sc->beta;
    ap = cg.sc->alpha_prev;
    mu = cg.sc->mu;
    first = cg.sc->first;
  }
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    __syncthreads();
    for (int q = threadIdx.x; q < m3; q += blockDim.x) {
      double F[9];
      gl_metric(TL + e * 24, sGx, sGw, q % m, (q / m) % m, q / m2, F);
#pragma unroll
      for (int c = 0; c < 9; ++c) sF[c * m3 + q] = F[c];
      const int64_t a = e * m3 + q;
      double pv;
      if constexpr (CG) {
        const double rv = cg.r[a];
        const double z = (cg.dinv ? rv * cg.dinv[a] : rv) - mu;
        pv = z;
        if (!first) {
          const double po = cg.p[a];
          pv = fma(beta, po, z);
          cg.x[a] = fma(ap, po, cg.x[a]);
        }
        cg.p[a] = pv;
      } else {
        pv = pin[a];
      }
      sp[q] = pv;
    }
    for (int c0 = 0; c0 < 3; c0 += CP) {
      __syncthreads();
      // z pass: pencil (jj, ii) of field (comp, pd): A = Mz t, Mz = Ct (pd = 2) or It
      for (int job = threadIdx.x; job < CP * 3 * m2; job += blockDim.x) {
        const int cl = job / (3 * m2), pd = (job / m2) % 3, jjii = job % m2;
        const int comp = c0 + cl;
        double t[m];
#pragma unroll
        for (int kk = 0; kk < m; ++kk)
          t[kk] = sF[(pd * 3 + comp) * m3 + kk * m2 + jjii] * sp[kk * m2 + jjii];
        double* A = sA + (cl * 3 + pd) * n * m2 + jjii;
        if (pd == 2) {
#pragma unroll
          for (int kz = 0; kz < n; ++kz) {
            double acc = 0.0;
#pragma unroll
            for (int kk = 0; kk < m; ++kk) acc = fma(M.Ct[kz * m + kk], t[kk], acc);
            A[kz * m2] = acc;
          }
        } else {
#pragma unroll
          for (int kz = 0; kz < n; ++kz) {
            double acc = 0.0;
#pragma unroll
            for (int kk = 0; kk < m; ++kk) acc = fma(M.It[kz * m + kk], t[kk], acc);
            A[kz * m2] = acc;
          }
        }
      }
      __syncthreads();
      // y pass: pencil (kz, ii): B0 = Iy A0, B12 = Cy A1 + Iy A2
      for (int job = threadIdx.x; job < CP * n * m; job += blockDim.x) {
        const int cl = job / (n * m), kz = (job / m) % n, ii = job % m;
        const double* A = sA + cl * 3 * n * m2 + kz * m2 + ii;
        double a0[m], a1[m], a2[m];
#pragma unroll
        for (int jj = 0; jj < m; ++jj) {
          a0[jj] = A[jj * m];
          a1[jj] = A[n * m2 + jj * m];
          a2[jj] = A[2 * n * m2 + jj * m];
        }
        double* B = sB + cl * 2 * n * n * m + kz * n * m + ii;
#pragma unroll
        for (int jy = 0; jy < n; ++jy) {
          double b0 = 0.0, b12 = 0.0;
#pragma unroll
          for (int jj = 0; jj < m; ++jj) {
            b0 = fma(M.It[jy * m + jj], a0[jj], b0);
            b12 = fma(M.Ct[jy * m + jj], a1[jj], b12);
            b12 = fma(M.It[jy * m + jj], a2[jj], b12);
          }
          B[jy * m] = b0;
          B[n * n * m + jy * m] = b12;
        }
      }
      __syncthreads();
      // x pass: pencil (kz, jy): g = Cx B0 + Ix B12, a row of n outputs
      for (int job = threadIdx.x; job < CP * n * n; job += blockDim.x) {
        const int cl = job / (n * n), row = job % (n * n);
        const double* B = sB + cl * 2 * n * n * m + row * m;
        double b0[m], b12[m];
#pragma unroll
        for (int ii = 0; ii < m; ++ii) {
          b0[ii] = B[ii];
          b12[ii] = B[n * n * m + ii];
        }
        double* out = pick3(g0, g1, g2, c0 + cl) + e * n3 + row * n;
#pragma unroll
        for (int ix = 0; ix < n; ++ix) {
          double acc = 0.0;
#pragma unroll
          for (int ii = 0; ii < m; ++ii) {
            acc = fma(M.Ct[ix * m + ii], b0[ii], acc);
            acc = fma(M.It[ix * m + ii], b12[ii], acc);
          }
          out[ix] = acc;
        }
      }
    }
  }
}

template <int n, int CP>
struct PDiv2 {
  static constexpr int m = n - 2, m2 = m * m, m3 = m2 * m, n3 = n * n * n;
  static constexpr int F_D = 9 * m3, V_D = 2 * 3 * n3, X_D = 2 * CP * n * n * m,
                       Y_D = 3 * CP * n * m2, Q_D = 3 * m3;
  static constexpr size_t bytes = sizeof(double) * (F_D + V_D + X_D + Y_D + Q_D);
};

template <int n, int CP, bool CG>
__global__ void __launch_bounds__(SBX_PENCIL_THREADS, SBX_PENCIL_MINB)
    p_div2_kernel(const double* __restrict__ v0, const double* __restrict__ v1,
                  const double* __restrict__ v2, int64_t E, const double* __restrict__ TL,
                  PMatK<n> M, double* __restrict__ qout, const double* __restrict__ pdot,
                  double* __restrict__ partials, CgScalars* __restrict__ sc) {
  using S = PDiv2<n, CP>;
  constexpr int m = n - 2, m2 = m * m, m3 = m2 * m, n3 = n * n * n;
  extern __shared__ double psm[];
  __shared__ double red[32];
  __shared__ bool is_last;
  double* sF = psm;           // [9][m3]
  double* sVb = sF + S::F_D;  // [2][3][n3]: this element's fields, the next one's in flight
  double* sX = sVb + S::V_D;  // [CP][2][n][n][m]   (k, j, a)
  double* sY = sX + S::X_D;  // [CP][3][n][m][m]   (k, b, a)
  double* sQ = sY + S::Y_D;  // [3][m3] per-component contributions
  // GL nodes / weights in shared memory (compile-time indices into the
  // parameter; a runtime index would copy it to local memory)
  __shared__ double sGx[n], sGw[n];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < m; ++q) {
      sGx[q] = M.x[q];
      sGw[q] = M.w[q];
    }
  }
  __syncthreads();
  if (CG && sc->done) return;
  double pq = 0.0;
  // the three fields of an element, copied asynchronously one element ahead
  auto prefetch = [&](int64_t ee, double* dst) {
    if (ee < E)
      for (int q = threadIdx.x; q < 3 * n3; q += blockDim.x)
        cp_async8(dst + q, pick3(v0, v1, v2, q / n3) + ee * n3 + q % n3, true);
    cp_async_commit();
  };
  prefetch(blockIdx.x, sVb);
  int buf = 0;
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x, buf ^= 1) {
    __syncthreads();  // the previous element is done with the other buffer
    prefetch(e + gridDim.x, sVb + (buf ^ 1) * 3 * n3);
    for (int q = threadIdx.x; q < m3; q += blockDim.x) {
      double F[9];
      gl_metric(TL + e * 24, sGx, sGw, q % m, (q / m) % m, q / m2, F);
#pragma unroll
      for (int c = 0; c < 9; ++c) sF[c * m3 + q] = F[c];
    }
    cp_async_wait<1>();  // this element's fields have landed (the next may still fly)
    double* sV = sVb + buf * 3 * n3;
    for (int c0 = 0; c0 < 3; c0 += CP) {
      __syncthreads();
      // x pass: row (k, j) of component: X0 = CIx v, X12 = Ix v
      for (int job = threadIdx.x; job < CP * n * n; job += blockDim.x) {
        const int cl = job / (n * n), row = job % (n * n);
        const double* v = sV + (c0 + cl) * n3 + row * n;
        double vr[n];
#pragma unroll
        for (int i = 0; i < n; ++i) vr[i] = v[i];
        double* X = sX + cl * 2 * n * n * m + row * m;
#pragma unroll
        for (int a = 0; a < m; ++a) {
          double x0 = 0.0, x12 = 0.0;
#pragma unroll
          for (int i = 0; i < n; ++i) {
            x0 = fma(M.CI[a * n + i], vr[i], x0);
            x12 = fma(M.I[a * n + i], vr[i], x12);
          }
          X[a] = x0;
          X[n * n * m + a] = x12;
        }
      }
      __syncthreads();
      // y pass: pencil (k, a): Y0 = Iy X0, Y1 = CIy X12, Y2 = Iy X12
      for (int job = threadIdx.x; job < CP * n * m; job += blockDim.x) {
        const int cl = job / (n * m), k = (job / m) % n, a = job % m;
        const double* X = sX + cl * 2 * n * n * m + k * n * m + a;
        double x0[n], x12[n];
#pragma unroll
        for (int j = 0; j < n; ++j) {
          x0[j] = X[j * m];
          x12[j] = X[n * n * m + j * m];
        }
        double* Y = sY + cl * 3 * n * m2 + k * m2 + a;
#pragma unroll
        for (int b = 0; b < m; ++b) {
          double y0 = 0.0, y1 = 0.0, y2 = 0.0;
#pragma unroll
          for (int j = 0; j < n; ++j) {
            y0 = fma(M.I[b * n + j], x0[j], y0);
            y1 = fma(M.CI[b * n + j], x12[j], y1);
            y2 = fma(M.I[b * n + j], x12[j], y2);
          }
          Y[b * m] = y0;
          Y[n * m2 + b * m] = y1;
          Y[2 * n * m2 + b * m] = y2;
        }
      }
      __syncthreads();
      // z pass: pencil (b, a) of component: R_p = Mz_p Y_p, times the metric
      for (int job = threadIdx.x; job < CP * m2; job += blockDim.x) {
        const int cl = job / m2, ba = job % m2, comp = c0 + cl;
        const double* Y = sY + cl * 3 * n * m2 + ba;
        double y0[n], y1[n], y2[n];
#pragma unroll
        for (int k = 0; k < n; ++k) {
          y0[k] = Y[k * m2];
          y1[k] = Y[n * m2 + k * m2];
          y2[k] = Y[2 * n * m2 + k * m2];
        }
#pragma unroll
        for (int c = 0; c < m; ++c) {
          double r0 = 0.0, r1 = 0.0, r2 = 0.0;
#pragma unroll
          for (int k = 0; k < n; ++k) {
            r0 = fma(M.I[c * n + k], y0[k], r0);
            r1 = fma(M.I[c * n + k], y1[k], r1);
            r2 = fma(M.CI[c * n + k], y2[k], r2);
          }
          const int q = c * m2 + ba;
          sQ[comp * m3 + q] = fma(sF[(0 * 3 + comp) * m3 + q], r0,
                                  fma(sF[(1 * 3 + comp) * m3 + q], r1,
                                      sF[(2 * 3 + comp) * m3 + q] * r2));
        }
      }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < m3; q += blockDim.x) {
      const double v = (sQ[q] + sQ[m3 + q]) + sQ[2 * m3 + q];
      const int64_t a = e * m3 + q;
      qout[a] = v;
      if (CG) pq = fma(pdot[a], v, pq);
    }
  }
  if constexpr (CG) {
    double v = pq;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    if (wid == 0)
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) partials[blockIdx.x] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      is_last = atomicAdd(&sc->counter[0], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last || threadIdx.x != 0) return;
    __threadfence();
    double tot = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) tot += partials[b];
    sc->counter[0] = 0;
    sc->pq = tot;
    if (!isfinite(tot) || tot <= 0.0) {
      sc->status = 5;
      sc->err_it = sc->it;
      sc->done = 1;
    } else {
      sc->alpha = sc->rz / tot;
    }
  }
}

// pressure_operator_diagonal (stepper.cpp:250-275) in closed form: the
// gradient of the unit vector at GL node q restricted to its element is
// g_comp(a) = sum_pd F[pd][comp](q) prod_dir M_{pd,dir}[a_dir][q_dir]
// (M = (I D)^T along pd, I^T elsewhere); diag(q) = sum_comp,a g^2 inv_bdiag(a).
template <int n>
__global__ void __launch_bounds__(kPThreads)
    p_diag_kernel(int64_t E, const double* __restrict__ TL, const double* __restrict__ mats,
                  const double* __restrict__ inv_bdiag, double* __restrict__ diag) {
  using PM = PMat<n>;
  constexpr int m = n - 2, m3 = m * m * m, n3 = n * n * n;
  extern __shared__ double psm[];
  double* sM = psm;
  double* sB = sM + PM::SIZE;  // inv_bdiag of the element
  for (int q = threadIdx.x; q < PM::SIZE; q += blockDim.x) sM[q] = mats[q];
  const double* sIt = sM + PM::OFF_IT;
  const double* sCt = sM + PM::OFF_CT;
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    __syncthreads();
    for (int a = threadIdx.x; a < n3; a += blockDim.x) sB[a] = inv_bdiag[e * n3 + a];
    __syncthreads();
    for (int q = threadIdx.x; q < m3; q += blockDim.x) {
      const int qi = q % m, qj = (q / m) % m, qk = q / (m * m);
      double F[9];
      gl_metric(TL + e * 24, sM + PM::OFF_X, sM + PM::OFF_W, qi, qj, qk, F);
      double s = 0.0;
      for (int ak = 0; ak < n; ++ak) {
        const double iz = sIt[ak * m + qk], cz = sCt[ak * m + qk];
        for (int aj = 0; aj < n; ++aj) {
          const double iy = sIt[aj * m + qj], cy = sCt[aj * m + qj];
          const double yz0 = iy * iz, yz1 = cy * iz, yz2 = iy * cz;
          for (int ai = 0; ai < n; ++ai) {
            const double ix = sIt[ai * m + qi], cx = sCt[ai * m + qi];
            const double X0 = cx * yz0, X1 = ix * yz1, X2 = ix * yz2;
            const double w = sB[(ak * n + aj) * n + ai];
#pragma unroll
            for (int comp = 0; comp < 3; ++comp) {
              const double g = fma(F[comp], X0, fma(F[3 + comp], X1, F[6 + comp] * X2));
              s = fma(g * g, w, s);
            }
          }
        }
      }
      diag[e * m3 + q] = s;
    }
  }
}

// The rest of a pressure CG iteration: r -= alpha q, then the sums the
// deflated preconditioner needs (z = r/diag - mu with mu = mean(r/diag)):
// S1 = r'(r/diag), S2 = sum r/diag, S3 = sum r, S4 = r'r; rz = S1 - mu S3.
// The last CTA takes the scalar step (krylov.cpp:66-88) and sets the WHILE
// condition.
__global__ void p_update_kernel(int64_t Np, double* __restrict__ r,
                                const double* __restrict__ q, const double* __restrict__ dinv,
                                double* __restrict__ partials, CgScalars* __restrict__ sc,
                                double* __restrict__ hist, int64_t hist_cap,
                                cudaGraphConditionalHandle cond, int use_cond) {
  __shared__ double red[4][32];
  __shared__ bool is_last;
  if (sc->done) {
    if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
    return;
  }
  const double alpha = sc->alpha;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < Np;
       a += (int64_t)gridDim.x * blockDim.x) {
    const double rv = fma(-alpha, q[a], r[a]);
    r[a] = rv;
    const double z = dinv ? rv * dinv[a] : rv;
    s[0] = fma(rv, z, s[0]);
    s[1] += z;
    s[2] += rv;
    s[3] = fma(rv, rv, s[3]);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double v = s[c];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[c][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[threadIdx.x][w];
    partials[4 * (int64_t)blockIdx.x + threadIdx.x] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    is_last = atomicAdd(&sc->counter[1], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!is_last || threadIdx.x != 0) return;
  __threadfence();
  double S[4] = {0.0, 0.0, 0.0, 0.0};
  for (int b = 0; b < (int)gridDim.x; ++b)
    for (int c = 0; c < 4; ++c) S[c] += partials[4 * (int64_t)b + c];
  sc->counter[1] = 0;
  const double mu = S[1] / (double)Np;
  const double rz_new = S[0] - mu * S[2];
  const double rnorm = sqrt(S[3]);
  const int it = sc->it;
  if (!isfinite(rnorm) || !isfinite(rz_new)) {
    sc->status = 6;
    sc->err_it = it;
    sc->done = 1;
  } else {
    const double rel = rnorm / sc->bnorm;
    if (hist && it + 1 < hist_cap) hist[it + 1] = rel;
    sc->it = it + 1;
    sc->beta = rz_new / sc->rz;
    sc->rz = rz_new;
    sc->rr = S[3];
    sc->mu = mu;
    sc->alpha_prev = alpha;
    sc->first = 0;
    sc->rel = rel;
    sc->relp = sc->bmb > 0.0 ? sqrt(fmax(rz_new, 0.0) / sc->bmb) : 0.0;
    if (sc->rel <= sc->tol && sc->relp <= sc->tol) {
      sc->converged = 1;
      sc->done = 1;
    } else if (sc->it >= sc->max_it) {
      sc->done = 1;
    }
  }
  if (use_cond) cudaGraphSetConditional(cond, sc->done ? 0 : 1);
}

// Initial sums over (b, r): [b'b, b'(b/d), sum b/d, sum b, r'(r/d), sum r/d,
// sum r, r'r] (d = 1 without a preconditioner) -> out[8], fixed order.
__global__ void p_init_kernel(int64_t Np, const double* __restrict__ b,
                              const double* __restrict__ r, const double* __restrict__ dinv,
                              double* __restrict__ partials, uint32_t* counter,
                              double* __restrict__ out) {
  __shared__ double red[8][32];
  __shared__ bool is_last;
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < Np;
       a += (int64_t)gridDim.x * blockDim.x) {
    const double bv = b[a], rv = r[a], di = dinv ? dinv[a] : 1.0;
    const double zb = bv * di, zr = rv * di;
    s[0] = fma(bv, bv, s[0]);
    s[1] = fma(bv, zb, s[1]);
    s[2] += zb;
    s[3] += bv;
    s[4] = fma(rv, zr, s[4]);
    s[5] += zr;
    s[6] += rv;
    s[7] = fma(rv, rv, s[7]);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    double v = s[c];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[c][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < 8) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[threadIdx.x][w];
    partials[8 * (int64_t)blockIdx.x + threadIdx.x] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    is_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!is_last || threadIdx.x >= 8) return;
  __threadfence();
  double v = 0.0;
  for (int bl = 0; bl < (int)gridDim.x; ++bl) v += partials[8 * (int64_t)bl + threadIdx.x];
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) *counter = 0;
}

__global__ void p_finish_kernel(int64_t Np, const double* __restrict__ p, double* __restrict__ x,
                                const CgScalars* __restrict__ sc) {
  if (sc->first || sc->status == 5) return;
  const double a = sc->alpha;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Np;
       q += (int64_t)gridDim.x * blockDim.x)
    x[q] = fma(a, p[q], x[q]);
}

template <class K>
cudaError_t set_smem(K kern, size_t bytes) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

unsigned pgrid(int64_t E) {
  int64_t g = E < 148 * 16 ? E : 148 * 16;
  return (unsigned)(g < 1 ? 1 : g);
}

// the pencil kernels' 1-D operators as a kernel parameter (constant bank)
template <int n>
PMatK<n> pmatk(const PresDev& P) {
  constexpr int m = n - 2;
  PMatK<n> M;
  const double* h = P.hmats;
  for (int q = 0; q < n * m; ++q) {
    M.It[q] = h[PMat<n>::OFF_IT + q];
    M.Ct[q] = h[PMat<n>::OFF_CT + q];
    M.I[q] = h[PMat<n>::OFF_I + q];
    M.CI[q] = h[PMat<n>::OFF_CI + q];
  }
  for (int q = 0; q < m; ++q) {
    M.w[q] = h[PMat<n>::OFF_W + q];
    M.x[q] = h[PMat<n>::OFF_X + q];
  }
  return M;
}

// components per pass of the pencil kernels (all three while they fit)
template <int n>
constexpr int pencil_cp() {
  return PGrad2<n, 3>::bytes <= 64 * 1024 && PDiv2<n, 3>::bytes <= 96 * 1024 ? 3 : 1;
}

template <int n>
cudaError_t grad_t(const PresDev& P, const double* p, double* const g[3], const PCgArgs* cg,
                   cudaStream_t s) {
  if constexpr (n < 4) {
    return cudaErrorInvalidValue;
  } else if constexpr (n <= 10) {
    constexpr int CP = pencil_cp<n>();
    const size_t sm = PGrad2<n, CP>::bytes;
    const PMatK<n> M = pmatk<n>(P);
    if (cg) {
      cudaError_t e = set_smem(p_grad2_kernel<n, CP, true>, sm);
      if (e != cudaSuccess) return e;
      p_grad2_kernel<n, CP, true><<<pgrid(P.E), SBX_PENCIL_THREADS, sm, s>>>(nullptr, P.E, P.tl, M, g[0], g[1],
                                                              g[2], *cg);
    } else {
      cudaError_t e = set_smem(p_grad2_kernel<n, CP, false>, sm);
      if (e != cudaSuccess) return e;
      p_grad2_kernel<n, CP, false><<<pgrid(P.E), SBX_PENCIL_THREADS, sm, s>>>(p, P.E, P.tl, M, g[0], g[1],
                                                               g[2], PCgArgs{});
    }
    return cudaGetLastError();
  } else {
    const size_t sm = PGradSmem<n>::bytes;
    if (cg) {
      cudaError_t e = set_smem(p_grad_kernel<n, true>, sm);
      if (e != cudaSuccess) return e;
      p_grad_kernel<n, true><<<pgrid(P.E), kPThreads, sm, s>>>(nullptr, P.E, P.tl, P.mats, g[0],
                                                              g[1], g[2], *cg);
    } else {
      cudaError_t e = set_smem(p_grad_kernel<n, false>, sm);
      if (e != cudaSuccess) return e;
      p_grad_kernel<n, false><<<pgrid(P.E), kPThreads, sm, s>>>(p, P.E, P.tl, P.mats, g[0],
                                                               g[1], g[2], PCgArgs{});
    }
    return cudaGetLastError();
  }
}

template <int n>
cudaError_t div_t(const PresDev& P, const double* const v[3], double* q, const double* pdot,
                  double* partials, CgScalars* sc, cudaStream_t s) {
  if constexpr (n < 4) {
    return cudaErrorInvalidValue;
  } else if constexpr (n <= 10) {
    constexpr int CP = pencil_cp<n>();
    const size_t sm = PDiv2<n, CP>::bytes;
    const PMatK<n> M = pmatk<n>(P);
    if (sc) {
      cudaError_t e = set_smem(p_div2_kernel<n, CP, true>, sm);
      if (e != cudaSuccess) return e;
      p_div2_kernel<n, CP, true><<<pgrid(P.E), SBX_PENCIL_THREADS, sm, s>>>(v[0], v[1], v[2], P.E, P.tl, M, q,
                                                             pdot, partials, sc);
    } else {
      cudaError_t e = set_smem(p_div2_kernel<n, CP, false>, sm);
      if (e != cudaSuccess) return e;
      p_div2_kernel<n, CP, false><<<pgrid(P.E), SBX_PENCIL_THREADS, sm, s>>>(v[0], v[1], v[2], P.E, P.tl, M, q,
                                                              nullptr, nullptr, nullptr);
    }
    return cudaGetLastError();
  } else {
    const size_t sm = PDivSmem<n>::bytes;
    if (sc) {
      cudaError_t e = set_smem(p_div_kernel<n, true>, sm);
      if (e != cudaSuccess) return e;
      p_div_kernel<n, true><<<pgrid(P.E), kPThreads, sm, s>>>(v[0], v[1], v[2], P.E, P.tl,
                                                             P.mats, q, pdot, partials, sc);
    } else {
      cudaError_t e = set_smem(p_div_kernel<n, false>, sm);
      if (e != cudaSuccess) return e;
      p_div_kernel<n, false><<<pgrid(P.E), kPThreads, sm, s>>>(v[0], v[1], v[2], P.E, P.tl,
                                                              P.mats, q, nullptr, nullptr,
                                                              nullptr);
    }
    return cudaGetLastError();
  }
}

template <int n>
cudaError_t diag_t(const PresDev& P, const double* inv_bdiag, double* diag, cudaStream_t s) {
  if constexpr (n < 4) {
    return cudaErrorInvalidValue;
  } else {
    const size_t sm = sizeof(double) * (PMat<n>::SIZE + n * n * n);
    cudaError_t e = set_smem(p_diag_kernel<n>, sm);
    if (e != cudaSuccess) return e;
    p_diag_kernel<n><<<pgrid(P.E), kPThreads, sm, s>>>(P.E, P.tl, P.mats, inv_bdiag, diag);
    return cudaGetLastError();
  }
}

#define SBX_P_SWITCH(NVAL, CALL)                                               \
  switch (NVAL) {                                                              \
    case 4: CALL(4); break;                                                    \
    case 5: CALL(5); break;                                                    \
    case 6: CALL(6); break;                                                    \
    case 7: CALL(7); break;                                                    \
    case 8: CALL(8); break;                                                    \
    case 9: CALL(9); break;                                                    \
    case 10: CALL(10); break;                                                  \
    case 11: CALL(11); break;                                                  \
    case 12: CALL(12); break;                                                  \
    case 13: CALL(13); break;                                                  \
    case 14: CALL(14); break;                                                  \
    case 15: CALL(15); break;                                                  \
    case 16: CALL(16); break;                                                  \
    default: err = cudaErrorInvalidValue;                                      \
  }

}  // namespace

cudaError_t launch_p_grad(const PresDev& P, const double* p, double* const g[3],
                          cudaStream_t s) {
  cudaError_t err = cudaSuccess;
#define CALLG(NN) err = grad_t<NN>(P, p, g, nullptr, s)
  SBX_P_SWITCH(P.n, CALLG)
#undef CALLG
  return err;
}

cudaError_t launch_p_div(const PresDev& P, const double* const v[3], double* q,
                         cudaStream_t s) {
  cudaError_t err = cudaSuccess;
#define CALLD(NN) err = div_t<NN>(P, v, q, nullptr, nullptr, nullptr, s)
  SBX_P_SWITCH(P.n, CALLD)
#undef CALLD
  return err;
}

cudaError_t launch_p_diag(const PresDev& P, const double* inv_bdiag, double* diag,
                          cudaStream_t s) {
  cudaError_t err = cudaSuccess;
#define CALLP(NN) err = diag_t<NN>(P, inv_bdiag, diag, s)
  SBX_P_SWITCH(P.n, CALLP)
#undef CALLP
  return err;
}

// One pressure-CG iteration (FAST): grad with the fused p / x update, gs +
// inverse mass, div with p'q and alpha, r update with the deflated
// preconditioner's sums and the scalar step.
cudaError_t launch_p_iteration(const PresDev& P, const PIterArgs& A,
                               cudaGraphConditionalHandle cond, int use_cond, cudaStream_t s) {
  cudaError_t err = cudaSuccess;
  PCgArgs cg{A.r, A.dinv, A.p, A.x, A.sc};
#define CALLI(NN) err = grad_t<NN>(P, nullptr, A.g, &cg, s)
  SBX_P_SWITCH(P.n, CALLI)
#undef CALLI
  if (err != cudaSuccess) return err;
  err = launch_gs3_scale(*A.op, A.g, A.inv_bdiag, s, A.v);
  if (err != cudaSuccess) return err;
#define CALLJ(NN) err = div_t<NN>(P, A.v, A.q, A.p, A.partials, A.sc, s)
  SBX_P_SWITCH(P.n, CALLJ)
#undef CALLJ
  if (err != cudaSuccess) return err;
  int64_t blocks = (P.Np + 1023) / 1024;
  if (blocks > 1184) blocks = 1184;
  if (blocks < 1) blocks = 1;
  p_update_kernel<<<(unsigned)blocks, 256, 0, s>>>(P.Np, A.r, A.q, A.dinv, A.partials, A.sc,
                                                   A.hist, A.hist_cap, cond, use_cond);
  return cudaGetLastError();
}

cudaError_t launch_p_init(const PresDev& P, const double* b, const double* r, const double* dinv,
                          double* partials, uint32_t* counter, double* out, cudaStream_t s) {
  int64_t blocks = (P.Np + 1023) / 1024;
  if (blocks > 1184) blocks = 1184;
  if (blocks < 1) blocks = 1;
  p_init_kernel<<<(unsigned)blocks, 256, 0, s>>>(P.Np, b, r, dinv, partials, counter, out);
  return cudaGetLastError();
}

cudaError_t launch_p_finish(const PresDev& P, const double* p, double* x, const CgScalars* sc,
                            cudaStream_t s) {
  int64_t blocks = (P.Np + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  p_finish_kernel<<<(unsigned)blocks, 256, 0, s>>>(P.Np, p, x, sc);
  return cudaGetLastError();
}


// ======================================================= host engine ======
namespace {

__global__ void inv_mass_kernel(int64_t N, const double* __restrict__ mask,
                                const double* __restrict__ bdiag, double* __restrict__ out) {
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < N;
       a += (int64_t)gridDim.x * blockDim.x)
    out[a] = (mask ? mask[a] : 1.0) / bdiag[a];
}

__global__ void nonzero_kernel(int64_t N, const double* __restrict__ x, int* flag) {
  bool nz = false;
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < N;
       a += (int64_t)gridDim.x * blockDim.x)
    nz |= (x[a] != 0.0);
  if (__syncthreads_or(nz) && threadIdx.x == 0) *flag = 1;
}

__global__ void sub_kernel(int64_t N, const double* __restrict__ b, const double* __restrict__ q,
                           double* __restrict__ r) {
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < N;
       a += (int64_t)gridDim.x * blockDim.x)
    r[a] = b[a] - q[a];
}

unsigned sgrid(int64_t N) {
  int64_t b = (N + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace

#define PE_CUDA(call)                                                         \
  do {                                                                        \
    cudaError_t _e = (call);                                                  \
    if (_e != cudaSuccess) {                                                  \
      err_ = std::string(#call) + ": " + cudaGetErrorString(_e);              \
      return SBX_E_CUDA;                                                      \
    }                                                                         \
  } while (0)

PressureEngine::~PressureEngine() {
  if (exec_) cudaGraphExecDestroy(exec_);
  if (graph_) cudaGraphDestroy(graph_);
  for (auto& e : basis_) {
    cudaFree(e.first);
    cudaFree(e.second);
  }
  for (double* v : pool_) cudaFree(v);
  for (double* v : {mats_, inv_bdiag_, pdiag_, pdinv_, g_[0], g_[1], g_[2], v_[0], v_[1], v_[2],
                    r_, p_, q_,
                    partials_, hist_, sums_, xmats_, pdiag_x_, zx_, scal_})
    cudaFree(v);
  cudaFree(counter_);
  cudaFree(flag_);
  cudaFree(sc_);
  if (hsc_) cudaFreeHost(hsc_);
}

int PressureEngine::setup(const OpDev& op, cudaStream_t s) {
  if (ready_ && op_ == &op) return SBX_OK;
  const int n = op.n, N = n - 1, m = n - 2;
  if (N < 3 || n > 16) {
    err_ = "pressure operator: needs 3 <= N <= 15 (build_pressure_basis, basis.cpp:114-119)";
    return SBX_E_CONFIG;
  }
  if (!op.tl) {
    err_ = "pressure operator: needs the element corners (a box context or a verified "
           "structured-box hint)";
    return SBX_E_CONFIG;
  }
  op_ = &op;
  P_.n = n;
  P_.m = m;
  P_.E = op.E;
  P_.Np = op.E * (int64_t)m * m * m;
  P_.tl = op.tl;
  // 1-D operators: [I^T | (I D)^T | I | I D | w | x]
  std::vector<double> gx(m), gw(m), I((size_t)m * n);
  if (pressure_basis(N, gx.data(), gw.data(), I.data()) != SBX_OK) {
    err_ = "pressure operator: bad degree";
    return SBX_E_CONFIG;
  }
  const double* D = op.Dh;
  std::vector<double> mats(4 * n * m + 2 * m);
  for (int a = 0; a < m; ++a)
    for (int l = 0; l < n; ++l) {
      double ci = 0.0;
      for (int j = 0; j < n; ++j) ci += I[(size_t)a * n + j] * D[j * n + l];
      mats[0 * n * m + l * m + a] = I[(size_t)a * n + l];  // It[l][a]
      mats[1 * n * m + l * m + a] = ci;                    // Ct[l][a] = (I D)[a][l]
      mats[2 * n * m + a * n + l] = I[(size_t)a * n + l];  // I[a][l]
      mats[3 * n * m + a * n + l] = ci;                    // CI[a][l]
    }
  for (int a = 0; a < m; ++a) {
    mats[4 * n * m + a] = gw[a];
    mats[4 * n * m + m + a] = gx[a];
  }
  // EXACT-mode operands: D, interp_v2p, its transpose, GL nodes / weights
  {
    std::vector<double> xm((size_t)n * n + 2 * (size_t)m * n + 2 * m);
    for (int q = 0; q < n * n; ++q) xm[q] = D[q];
    for (int a = 0; a < m; ++a)
      for (int j = 0; j < n; ++j) {
        xm[(size_t)n * n + (size_t)a * n + j] = I[(size_t)a * n + j];
        xm[(size_t)n * n + (size_t)m * n + (size_t)j * m + a] = I[(size_t)a * n + j];
      }
    for (int a = 0; a < m; ++a) {
      xm[(size_t)n * n + 2 * (size_t)m * n + a] = gx[a];
      xm[(size_t)n * n + 2 * (size_t)m * n + m + a] = gw[a];
    }
    PE_CUDA(cudaMalloc(&xmats_, sizeof(double) * xm.size()));
    PE_CUDA(cudaMemcpyAsync(xmats_, xm.data(), sizeof(double) * xm.size(),
                            cudaMemcpyHostToDevice, s));
    PE_CUDA(cudaStreamSynchronize(s));
    X_.n = n;
    X_.m = m;
    X_.E = op.E;
    X_.corners = op.corners;
    X_.d = xmats_;
    X_.iv = xmats_ + n * n;
    X_.ivt = xmats_ + n * n + m * n;
    X_.glx = xmats_ + n * n + 2 * m * n;
    X_.glw = X_.glx + m;
  }
  PE_CUDA(cudaMalloc(&mats_, sizeof(double) * mats.size()));
  PE_CUDA(cudaMemcpyAsync(mats_, mats.data(), sizeof(double) * mats.size(),
                          cudaMemcpyHostToDevice, s));
  P_.mats = mats_;
  hmats_ = mats;
  P_.hmats = hmats_.data();
  // inv_bdiag = mask / gs_sum(bm)   (FlowSolver constructor, stepper.cpp:79-84)
  if (!op.bm) {
    err_ = "pressure operator: needs the mass factors (bm)";
    return SBX_E_CONFIG;
  }
  PE_CUDA(cudaMalloc(&inv_bdiag_, sizeof(double) * op.nodes));
  double* bd = nullptr;
  PE_CUDA(cudaMalloc(&bd, sizeof(double) * op.nodes));
  PE_CUDA(cudaMemcpyAsync(bd, op.bm, sizeof(double) * op.nodes, cudaMemcpyDeviceToDevice, s));
  PE_CUDA(launch_gs(op, bd, false, s));
  inv_mass_kernel<<<sgrid(op.nodes), 256, 0, s>>>(op.nodes, op.mask, bd, inv_bdiag_);
  PE_CUDA(cudaGetLastError());
  PE_CUDA(cudaStreamSynchronize(s));
  cudaFree(bd);
  PE_CUDA(cudaMalloc(&sc_, sizeof(CgScalars)));
  PE_CUDA(cudaMemset(sc_, 0, sizeof(CgScalars)));
  PE_CUDA(cudaMallocHost(&hsc_, sizeof(CgScalars)));
  PE_CUDA(cudaMalloc(&sums_, 8 * sizeof(double)));
  PE_CUDA(cudaMalloc(&counter_, 4 * sizeof(uint32_t)));
  PE_CUDA(cudaMemset(counter_, 0, 4 * sizeof(uint32_t)));
  PE_CUDA(cudaMalloc(&flag_, sizeof(int)));
  PE_CUDA(cudaMalloc(&partials_, sizeof(double) * 8 * 148 * 16));
  for (int c = 0; c < 3; ++c) {
    PE_CUDA(cudaMalloc(&g_[c], sizeof(double) * op.nodes));
    PE_CUDA(cudaMalloc(&v_[c], sizeof(double) * op.nodes));
  }
  ready_ = true;
  return SBX_OK;
}

int PressureEngine::ensure_diag(cudaStream_t s) {
  if (pdiag_) return SBX_OK;
  PE_CUDA(cudaMalloc(&pdiag_, sizeof(double) * P_.Np));
  PE_CUDA(cudaMalloc(&pdinv_, sizeof(double) * P_.Np));
  PE_CUDA(launch_p_diag(P_, inv_bdiag_, pdiag_, s));
  PE_CUDA(launch_recip(P_.Np, pdiag_, pdinv_, s));
  return SBX_OK;
}

int PressureEngine::grad(const double* p, double* const g[3], cudaStream_t s) {
  PE_CUDA(launch_p_grad(P_, p, g, s));
  return SBX_OK;
}

int PressureEngine::div(const double* const v[3], double* q, cudaStream_t s) {
  PE_CUDA(launch_p_div(P_, v, q, s));
  return SBX_OK;
}

int PressureEngine::apply(const double* p, double* q, cudaStream_t s) {
  PE_CUDA(launch_p_grad(P_, p, g_, s));
  PE_CUDA(launch_gs3_scale(*op_, g_, inv_bdiag_, s, v_));
  PE_CUDA(launch_p_div(P_, v_, q, s));
  return SBX_OK;
}

int PressureEngine::grad_exact(const double* p, double* const g[3], cudaStream_t s) {
  if (!X_.corners) {
    err_ = "EXACT pressure operators need the element corners";
    return SBX_E_CONFIG;
  }
  PE_CUDA(launch_p_grad_exact(X_, p, g, s));
  return SBX_OK;
}

int PressureEngine::div_exact(const double* const v[3], double* q, cudaStream_t s) {
  if (!X_.corners) {
    err_ = "EXACT pressure operators need the element corners";
    return SBX_E_CONFIG;
  }
  PE_CUDA(launch_p_div_exact(X_, v, q, s));
  return SBX_OK;
}

// apply_pressure_operator (stepper.cpp:240-248) in the reference order:
// gs_sum_inplace per component, then field_pointwise_mul(inv_bdiag)
int PressureEngine::apply_exact(const double* p, double* q, cudaStream_t s) {
  int rc = grad_exact(p, g_, s);
  if (rc != SBX_OK) return rc;
  for (int c = 0; c < 3; ++c) {
    PE_CUDA(launch_gs(*op_, g_[c], false, s));
    PE_CUDA(launch_mul(op_->nodes, inv_bdiag_, g_[c], s));
  }
  return div_exact(g_, q, s);
}

int PressureEngine::ensure_diag_exact(cudaStream_t s) {
  if (pdiag_x_) return SBX_OK;
  if (!X_.corners) {
    err_ = "EXACT pressure operators need the element corners";
    return SBX_E_CONFIG;
  }
  PE_CUDA(cudaMalloc(&pdiag_x_, sizeof(double) * P_.Np));
  PE_CUDA(launch_p_diag_exact(X_, inv_bdiag_, pdiag_x_, s));
  return SBX_OK;
}

// pcg (krylov.cpp:7-91) statement by statement with the pressure operator,
// field_dot and pressure_precond (stepper.cpp:277-308), every operation in the
// reference's order: bitwise equal residual history and solution.
int PressureEngine::solve_exact(cudaStream_t s, const double* b, double* x,
                                const sbx_pcg_config& cfg, sbx_pcg_result* res) {
  const bool jacobi = cfg.precond == SBX_PRECOND_JACOBI;
  if (jacobi) {
    const int rc = ensure_diag_exact(s);
    if (rc != SBX_OK) return rc;
  }
  if (ensure_work(cfg.max_iterations) != SBX_OK) return SBX_E_CUDA;
  if (!zx_) {
    PE_CUDA(cudaMalloc(&zx_, sizeof(double) * P_.Np));
    PE_CUDA(cudaMalloc(&scal_, 4 * sizeof(double)));
  }
  const int64_t Np = P_.Np;
  const int m3 = P_.m * P_.m * P_.m;
  std::memset(res, 0, sizeof(*res));
  res->error_iteration = -1;
  auto push = [&](double v) {
    if (cfg.history && res->history_length < cfg.history_capacity)
      cfg.history[res->history_length] = v;
    ++res->history_length;
  };
  auto dot = [&](const double* a, const double* c, double* out) -> int {
    PE_CUDA(launch_dot_exact_n(P_.E, m3, a, c, partials_, scal_, s));
    PE_CUDA(cudaMemcpyAsync(out, scal_, sizeof(double), cudaMemcpyDeviceToHost, s));
    PE_CUDA(cudaStreamSynchronize(s));
    return SBX_OK;
  };
  auto precond = [&](const double* in, double* out) -> int {
    if (jacobi)
      PE_CUDA(launch_div(Np, in, pdiag_x_, out, s));
    else
      PE_CUDA(cudaMemcpyAsync(out, in, sizeof(double) * Np, cudaMemcpyDeviceToDevice, s));
    PE_CUDA(launch_deflate_exact(Np, out, scal_ + 1, s));
    return SBX_OK;
  };
  double bb;
  if (dot(b, b, &bb)) return SBX_E_CUDA;
  if (bb == 0.0) {
    PE_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * Np, s));
    PE_CUDA(cudaStreamSynchronize(s));
    res->converged = 1;
    return SBX_OK;
  }
  const double bnorm = std::sqrt(bb);
  double *r = r_, *z = zx_, *q = q_, *p = p_;
  PE_CUDA(cudaMemcpyAsync(r, b, sizeof(double) * Np, cudaMemcpyDeviceToDevice, s));
  PE_CUDA(cudaMemsetAsync(flag_, 0, sizeof(int), s));
  nonzero_kernel<<<sgrid(Np), 256, 0, s>>>(Np, x, flag_);
  int nz = 0;
  PE_CUDA(cudaMemcpyAsync(&nz, flag_, sizeof(int), cudaMemcpyDeviceToHost, s));
  PE_CUDA(cudaStreamSynchronize(s));
  if (nz) {
    const int rc = apply_exact(x, q, s);
    if (rc != SBX_OK) return rc;
    PE_CUDA(launch_axpy(Np, -1.0, q, r, s));
  }
  if (precond(b, z)) return SBX_E_CUDA;
  double bmb;
  if (dot(b, z, &bmb)) return SBX_E_CUDA;
  if (precond(r, z)) return SBX_E_CUDA;
  double rz, rr;
  if (dot(r, z, &rz) || dot(r, r, &rr)) return SBX_E_CUDA;
  double rnorm = std::sqrt(rr);
  push(rnorm / bnorm);
  PE_CUDA(cudaMemcpyAsync(p, z, sizeof(double) * Np, cudaMemcpyDeviceToDevice, s));
  for (int it = 0; it < cfg.max_iterations; ++it) {
    res->rel_residual = rnorm / bnorm;
    res->rel_residual_precond = bmb > 0.0 ? std::sqrt(std::max(rz, 0.0) / bmb) : 0.0;
    if (res->rel_residual <= cfg.tolerance && res->rel_residual_precond <= cfg.tolerance) {
      res->converged = 1;
      return SBX_OK;
    }
    const int rc = apply_exact(p, q, s);
    if (rc != SBX_OK) return rc;
    double pq;
    if (dot(p, q, &pq)) return SBX_E_CUDA;
    if (!std::isfinite(pq) || pq <= 0.0) {
      res->error_iteration = it;
      return SBX_E_BREAKDOWN;
    }
    const double alpha = rz / pq;
    PE_CUDA(launch_axpy(Np, alpha, p, x, s));
    PE_CUDA(launch_axpy(Np, -alpha, q, r, s));
    if (precond(r, z)) return SBX_E_CUDA;
    double rz_new;
    if (dot(r, z, &rz_new) || dot(r, r, &rr)) return SBX_E_CUDA;
    rnorm = std::sqrt(rr);
    if (!std::isfinite(rnorm) || !std::isfinite(rz_new)) {
      res->error_iteration = it;
      return SBX_E_NAN;
    }
    push(rnorm / bnorm);
    ++res->iterations;
    const double beta = rz_new / rz;
    rz = rz_new;
    PE_CUDA(launch_scale(Np, beta, p, s));
    PE_CUDA(launch_axpy(Np, 1.0, z, p, s));
  }
  res->rel_residual = rnorm / bnorm;
  res->rel_residual_precond = bmb > 0.0 ? std::sqrt(std::max(rz, 0.0) / bmb) : 0.0;
  res->converged = res->rel_residual <= cfg.tolerance &&
                   res->rel_residual_precond <= cfg.tolerance;
  PE_CUDA(cudaStreamSynchronize(s));
  return SBX_OK;
}

// ---- ProjectionHistory (krylov.cpp:93-124), plain field_dot ----------------
int PressureEngine::pdot(cudaStream_t s, const double* a, const double* b, bool exact,
                         double* out) {
  if (!scal_) PE_CUDA(cudaMalloc(&scal_, 4 * sizeof(double)));
  if (exact)
    PE_CUDA(launch_dot_exact_n(P_.E, P_.m * P_.m * P_.m, a, b, partials_, scal_, s));
  else
    PE_CUDA(launch_dot_fast(P_.Np, a, b, nullptr, partials_, counter_ + 1, scal_, s));
  PE_CUDA(cudaMemcpyAsync(out, scal_, sizeof(double), cudaMemcpyDeviceToHost, s));
  PE_CUDA(cudaStreamSynchronize(s));
  return SBX_OK;
}

int PressureEngine::proj_reset(int depth) {
  for (auto& e : basis_) {
    pool_.push_back(e.first);
    pool_.push_back(e.second);
  }
  basis_.clear();
  depth_ = depth;
  return SBX_OK;
}

int PressureEngine::proj_guess(cudaStream_t s, const double* b, double* guess, double* deflated,
                               bool exact) {
  const int64_t Np = P_.Np;
  PE_CUDA(cudaMemsetAsync(guess, 0, sizeof(double) * Np, s));
  if (deflated && deflated != b)
    PE_CUDA(cudaMemcpyAsync(deflated, b, sizeof(double) * Np, cudaMemcpyDeviceToDevice, s));
  for (const auto& xy : basis_) {
    double alpha;
    if (pdot(s, xy.first, b, exact, &alpha)) return SBX_E_CUDA;
    PE_CUDA(launch_axpy(Np, alpha, xy.first, guess, s));
    if (deflated) PE_CUDA(launch_axpy(Np, -alpha, xy.second, deflated, s));
  }
  PE_CUDA(cudaStreamSynchronize(s));
  return SBX_OK;
}

int PressureEngine::proj_append(cudaStream_t s, const double* x, bool exact) {
  if (depth_ <= 0) return SBX_OK;
  const int64_t Np = P_.Np;
  auto fresh = [&](double** v) -> int {
    if (!pool_.empty()) {
      *v = pool_.back();
      pool_.pop_back();
      return SBX_OK;
    }
    PE_CUDA(cudaMalloc(v, sizeof(double) * Np));
    return SBX_OK;
  };
  double *v = nullptr, *w = nullptr;
  if (fresh(&v) || fresh(&w)) return SBX_E_CUDA;
  PE_CUDA(cudaMemcpyAsync(v, x, sizeof(double) * Np, cudaMemcpyDeviceToDevice, s));
  const int rc = exact ? apply_exact(x, w, s) : apply(x, w, s);
  if (rc != SBX_OK) return rc;
  double scale;
  if (pdot(s, v, w, exact, &scale)) return SBX_E_CUDA;
  for (const auto& xy : basis_) {
    double c;
    if (pdot(s, xy.first, w, exact, &c)) return SBX_E_CUDA;
    PE_CUDA(launch_axpy(Np, -c, xy.first, v, s));
    PE_CUDA(launch_axpy(Np, -c, xy.second, w, s));
  }
  double d;
  if (pdot(s, v, w, exact, &d)) return SBX_E_CUDA;
  if (!(d > scale * 1e-24) || !std::isfinite(d)) {  // linearly dependent
    pool_.push_back(v);
    pool_.push_back(w);
    return SBX_OK;
  }
  const double inv = 1.0 / std::sqrt(d);
  PE_CUDA(launch_scale(Np, inv, v, s));
  PE_CUDA(launch_scale(Np, inv, w, s));
  basis_.push_back({v, w});
  while ((int)basis_.size() > depth_) {
    pool_.push_back(basis_.front().first);
    pool_.push_back(basis_.front().second);
    basis_.pop_front();
  }
  PE_CUDA(cudaStreamSynchronize(s));
  return SBX_OK;
}

int PressureEngine::ensure_work(int max_it) {
  if (!r_) {
    PE_CUDA(cudaMalloc(&r_, sizeof(double) * P_.Np));
    PE_CUDA(cudaMalloc(&p_, sizeof(double) * P_.Np));
    PE_CUDA(cudaMalloc(&q_, sizeof(double) * P_.Np));
  }
  if (hist_len_ < (int64_t)max_it + 1) {
    cudaFree(hist_);
    hist_len_ = (int64_t)max_it + 1;
    PE_CUDA(cudaMalloc(&hist_, sizeof(double) * hist_len_));
    if (exec_) cudaGraphExecDestroy(exec_);
    exec_ = nullptr;
  }
  return SBX_OK;
}

int PressureEngine::build_graph(cudaStream_t s, double* x, const double* dinv) {
  if (exec_) cudaGraphExecDestroy(exec_);
  if (graph_) cudaGraphDestroy(graph_);
  exec_ = nullptr;
  graph_ = nullptr;
  PE_CUDA(cudaGraphCreate(&graph_, 0));
  cudaGraphConditionalHandle handle;
  PE_CUDA(cudaGraphConditionalHandleCreate(&handle, graph_, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams params = {};
  params.type = cudaGraphNodeTypeConditional;
  params.conditional.handle = handle;
  params.conditional.type = cudaGraphCondTypeWhile;
  params.conditional.size = 1;
  cudaGraphNode_t node;
  PE_CUDA(cudaGraphAddNode(&node, graph_, nullptr, 0, &params));
  cudaGraph_t body = params.conditional.phGraph_out[0];
  PE_CUDA(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0,
                                        cudaStreamCaptureModeRelaxed));
  PIterArgs A{op_, inv_bdiag_, r_, dinv, p_, x, q_, {g_[0], g_[1], g_[2]},
              {v_[0], v_[1], v_[2]}, partials_, sc_, hist_, hist_len_};
  cudaError_t e = cudaSuccess;
  for (int u = 0; u < 2 && e == cudaSuccess; ++u) e = launch_p_iteration(P_, A, handle, 1, s);
  cudaGraph_t captured = nullptr;
  const cudaError_t e2 = cudaStreamEndCapture(s, &captured);
  PE_CUDA(e);
  PE_CUDA(e2);
  PE_CUDA(cudaGraphInstantiate(&exec_, graph_, 0));
  gkey_[0] = x;
  gkey_[1] = dinv;
  gkey_[2] = hist_;
  gkey_[3] = s;
  return SBX_OK;
}

// pcg (krylov.cpp:7-91) on the pressure operator with the plain dot and the
// deflated preconditioner (stepper.cpp:277-308), FAST schedule: the deflated
// inner products come from one reduction pass (r'z = r'(r/d) - mean(r/d) sum r).
int PressureEngine::solve(cudaStream_t s, const double* b, double* x, const sbx_pcg_config& cfg,
                          sbx_pcg_result* res) {
  const bool jacobi = cfg.precond == SBX_PRECOND_JACOBI;
  if (jacobi && ensure_diag(s) != SBX_OK) return SBX_E_CUDA;
  if (ensure_work(cfg.max_iterations) != SBX_OK) return SBX_E_CUDA;
  const double* dinv = jacobi ? pdinv_ : nullptr;
  const int64_t Np = P_.Np;
  // r = b - E x0, the apply skipped for a zero guess (krylov.cpp:19-32)
  PE_CUDA(cudaMemsetAsync(flag_, 0, sizeof(int), s));
  nonzero_kernel<<<sgrid(Np), 256, 0, s>>>(Np, x, flag_);
  int nz = 0;
  PE_CUDA(cudaMemcpyAsync(&nz, flag_, sizeof(int), cudaMemcpyDeviceToHost, s));
  PE_CUDA(cudaStreamSynchronize(s));
  if (nz) {
    if (apply(x, q_, s) != SBX_OK) return SBX_E_CUDA;
    sub_kernel<<<sgrid(Np), 256, 0, s>>>(Np, b, q_, r_);
  } else {
    PE_CUDA(cudaMemcpyAsync(r_, b, sizeof(double) * Np, cudaMemcpyDeviceToDevice, s));
  }
  PE_CUDA(launch_p_init(P_, b, r_, dinv, partials_, counter_, sums_, s));
  double h[8];
  PE_CUDA(cudaMemcpyAsync(h, sums_, sizeof(h), cudaMemcpyDeviceToHost, s));
  PE_CUDA(cudaStreamSynchronize(s));
  std::memset(res, 0, sizeof(*res));
  res->error_iteration = -1;
  const double bb = h[0];
  if (bb == 0.0) {
    PE_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * Np, s));
    PE_CUDA(cudaStreamSynchronize(s));
    res->converged = 1;
    return SBX_OK;
  }
  const double npd = (double)Np;
  const double bmb = h[1] - (h[2] / npd) * h[3];
  const double mu = h[5] / npd;
  const double rz = h[4] - mu * h[6];
  const double rr = h[7];
  CgScalars c{};
  c.bnorm = std::sqrt(bb);
  c.bmb = bmb;
  c.rz = rz;
  c.rr = rr;
  c.mu = mu;
  c.tol = cfg.tolerance;
  c.rel = std::sqrt(rr) / c.bnorm;
  c.relp = bmb > 0.0 ? std::sqrt(std::max(rz, 0.0) / bmb) : 0.0;
  c.max_it = cfg.max_iterations;
  c.first = 1;
  c.err_it = -1;
  c.nranks = 1;
  if (c.rel <= cfg.tolerance && c.relp <= cfg.tolerance) {
    c.converged = 1;
    c.done = 1;
  } else if (cfg.max_iterations <= 0) {
    c.done = 1;
  }
  *hsc_ = c;
  PE_CUDA(cudaMemcpyAsync(sc_, hsc_, sizeof(CgScalars), cudaMemcpyHostToDevice, s));
  PE_CUDA(cudaMemcpyAsync(hist_, &c.rel, sizeof(double), cudaMemcpyHostToDevice, s));
  if (!c.done) {
    if (!exec_ || gkey_[0] != x || gkey_[1] != dinv || gkey_[2] != hist_ || gkey_[3] != s) {
      const int rc = build_graph(s, x, dinv);
      if (rc != SBX_OK) return rc;
    }
    PE_CUDA(cudaGraphLaunch(exec_, s));
    PE_CUDA(launch_p_finish(P_, p_, x, sc_, s));
  }
  PE_CUDA(cudaMemcpyAsync(hsc_, sc_, sizeof(CgScalars), cudaMemcpyDeviceToHost, s));
  PE_CUDA(cudaStreamSynchronize(s));
  const CgScalars& o = *hsc_;
  res->iterations = o.it;
  res->converged = o.converged;
  res->rel_residual = o.rel;
  res->rel_residual_precond = o.relp;
  res->history_length = (int64_t)o.it + 1;
  if (cfg.history && cfg.history_capacity > 0) {
    const int64_t cnt = std::min<int64_t>(res->history_length, cfg.history_capacity);
    PE_CUDA(cudaMemcpy(cfg.history, hist_, sizeof(double) * cnt, cudaMemcpyDeviceToHost));
  }
  if (o.status == 5 || o.status == 6) {
    res->error_iteration = o.err_it;
    return o.status;
  }
  return SBX_OK;
}

}  // namespace sbx
