// Element tensor-product core of axhelm shared by the standalone operator
// kernel (ops.cu) and the fused CG kernel (cg.cu).
//
// Thread layout: one thread per (i, j) column of an element, looping over k
// (the paper's shared-memory axhelm, re-tiled for sm_100a:
// several elements per CTA, padded smem rows against bank conflicts, D[k][l]
// read from the kernel-parameter constant bank with compile-time indices, the
// thread's own t-column kept in registers across both sweeps).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace sbx {

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

template <int n>
struct DParam {
  double d[n * n];
};

template <int n>
struct AxCfg {
  static constexpr int nn = n * n;
  static constexpr int n3 = n * n * n;
  static constexpr int EPB = (256 / nn) > 0 ? 256 / nn : 1;  // elements per CTA
  static constexpr int threads = EPB * nn;
  static constexpr int SR = (n % 2 == 0) ? n + 1 : n;  // padded smem row stride
  static constexpr int SP = n * SR;                     // plane stride
  static constexpr int TILE = n * SP;
  static constexpr int DS = SR;
  static constexpr size_t smem = (size_t)(3 * EPB * TILE + n * DS) * sizeof(double);
};

// Stage D (padded rows) into shared memory.
template <int n>
__device__ __forceinline__ void ax_stage_D(double* sD, const DParam<n>& Dp) {
  using C = AxCfg<n>;
  for (int q = threadIdx.x; q < n * n; q += blockDim.x) sD[(q / n) * C::DS + q % n] = Dp.d[q];
}

// Given the thread's column uc[k] = u(i,j,k) (already written to su by the
// caller for every k), compute acc[k] = sum_l D^T G D u  at (i,j,k) without
// the mass term.  Contains two __syncthreads (all CTA threads must call it).
// EXACT keeps the reference's evaluation order (operators.cpp:224-260).
template <int n, bool EXACT>
__device__ __forceinline__ void ax_column(const double (&uc)[n], double* su, double* sr,
                                          double* ss, const double* sD,
                                          const double* __restrict__ Ge, bool valid, int i,
                                          int j, double h1, double tsign, const DParam<n>& Dp,
                                          double (&acc)[n]) {
  using C = AxCfg<n>;
  __syncthreads();
  double wt[n];
#pragma unroll
  for (int k = 0; k < n; ++k) {
    double r = 0.0, s = 0.0, tt = 0.0;
#pragma unroll
    for (int l = 0; l < n; ++l) {
      const double dil = sD[i * C::DS + l], djl = sD[j * C::DS + l];
      const double ur = su[k * C::SP + j * C::SR + l], us = su[k * C::SP + l * C::SR + i];
      if constexpr (EXACT) {
        r = dadd(r, dmul(dil, ur));
        s = dadd(s, dmul(djl, us));
        tt = dadd(tt, dmul(Dp.d[k * n + l], uc[l]));
      } else {
        r = fma(dil, ur, r);
        s = fma(djl, us, s);
        tt = fma(Dp.d[k * n + l], uc[l], tt);
      }
    }
    double g[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) g[c] = valid ? __ldg(Ge + c * C::n3 + k * C::nn) : 0.0;
    double wr, ws, wtk;
    if constexpr (EXACT) {
      wr = dmul(dadd(dadd(dmul(g[0], r), dmul(g[3], s)), dmul(g[4], tt)), h1);
      ws = dmul(dadd(dadd(dmul(g[1], s), dmul(g[3], r)), dmul(g[5], tt)), h1);
      wtk = dmul(dadd(dadd(dmul(g[2], tt), dmul(g[4], r)), dmul(g[5], s)), h1);
    } else {
      wr = h1 * fma(g[0], r, fma(g[3], s, g[4] * tt));
      ws = h1 * fma(g[1], s, fma(g[3], r, g[5] * tt));
      wtk = h1 * fma(g[2], tt, fma(g[4], r, g[5] * s));
    }
    sr[k * C::SP + j * C::SR + i] = wr;
    ss[k * C::SP + j * C::SR + i] = ws;
    wt[k] = wtk;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < n; ++k) {
    double a = 0.0;
#pragma unroll
    for (int l = 0; l < n; ++l) {
      const double a1v = sr[k * C::SP + j * C::SR + l];
      const double a2v = ss[k * C::SP + l * C::SR + i];
      if constexpr (EXACT) {
        const double t1 = dmul(sD[l * C::DS + i], a1v);
        const double t2 = dmul(sD[l * C::DS + j], a2v);
        const double t3 = dmul(dmul(tsign, Dp.d[l * n + k]), wt[l]);
        a = dadd(a, dadd(dadd(t1, t2), t3));
      } else {
        a = fma(sD[l * C::DS + i], a1v, a);
        a = fma(sD[l * C::DS + j], a2v, a);
        a = fma(tsign * Dp.d[l * n + k], wt[l], a);
      }
    }
    acc[k] = a;
  }
}

}  // namespace sbx
