// K1 for n = 10 (N = 9) on the FP64 tensor cores (sm_100a).
//
// At n = 10 a plane is 10 x 10, which does not tile 8 x 8 the way n = 8 does
// (ax_dmma.cuh), and the FMA kernel (ax_tma_kernel, one thread per (i, j)
// column) is bound by shared-memory traffic (~80 loads per node) at 2 groups
// per SM.  Here each of the six tensor contractions of axhelm is ONE GEMM over
// the whole element, with the contracted index l as K:
//
//   ur[(k,j)][i]   = sum_l U[(k,j)][l] D[i][l]      M = 100 (k,j), N = 10 i
//   us[j][(k,i)]   = sum_l D[j][l] U[k][l][i]       M = 10 j,      N = 100 (k,i)
//   ut[k][(j,i)]   = sum_l D[k][l] U[l][(j,i)]      M = 10 k,      N = 100 (j,i)
//
// and the transposed three for the second sweep, each as m8n8k4 DMMA tiles
// (M, N padded to multiples of 8, K = 10 padded to 12 with zero D fragments;
// operand addresses outside the element are clamped to finite data whose
// products are discarded or multiplied by zero).  A TEAM of two warps owns an
// element: tiles alternate between the warps, the trilinear metric runs
// column by column (one lane per (i, j) column, all 10 k), and every phase
// ends at the team's named barrier.  ur, us, ut live in three 1000-double
// tiles: two overlay the staged p_old and x (dead after the prologue), one is
// the team's scratch; the second sweep accumulates w's t-part in place over
// ut, then adds the s-part and finally the r-part, whose accumulator
// fragments go straight to the epilogue (w, p'Ap).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "ax_dmma.cuh"

namespace sbx {

#ifndef SBX_DMMA10_UNROLL
#define SBX_DMMA10_UNROLL 1  // tile-loop unroll (measured: 1 with 6 teams >= 13 with 4)
#endif
constexpr int kD10Unroll = SBX_DMMA10_UNROLL;
#ifndef SBX_DMMA10_TEAMS
#define SBX_DMMA10_TEAMS 6  // two-warp teams per CTA at most
#endif

template <int NV, int TEAMS, int NSLOT, bool OVL>
struct Dmma10Layout {
  static constexpr int G_D = 24;    // the element's trilinear map coefficients
  static constexpr int V_D = 1000;  // one staged vector
  static constexpr int SLOT_D = G_D + NV * V_D;
  static constexpr int S = NSLOT;
  // per-team scratch tile for ut (OVL: none -- ut overlays the staged 1/diag,
  // dead after the prologue like p_old and x)
  static constexpr int T_D = OVL ? 0 : 1000;
  static constexpr size_t BAR_BYTES = 1024;
  static constexpr int AUX_D = 128;  // D (10 x 10, row-major), GLL x[10], w[10]
  static constexpr size_t smem =
      BAR_BYTES + sizeof(double) * (size_t)(AUX_D + S * SLOT_D + TEAMS * T_D);
  static constexpr int threads = TEAMS * 64;
  static_assert(NV >= 3, "the sr / ss tiles overlay the staged p_old and x");
};

template <int NV, bool OVL>
struct Dmma10Choice {
  static constexpr size_t BUDGET = 225 * 1024;
  static constexpr size_t slot_b = sizeof(double) * (24 + (size_t)NV * 1000);
  static constexpr size_t fixed_b(int t) {
    return 1024 + sizeof(double) * (128 + (OVL ? 0 : (size_t)t * 1000));
  }
  static constexpr int slots_for(int t) {
    return fixed_b(t) >= BUDGET ? 0 : (int)((BUDGET - fixed_b(t)) / slot_b);
  }
  static constexpr int pick() {
    for (int t = SBX_DMMA10_TEAMS; t >= 1; --t)
      if (slots_for(t) >= t + 1) return t;
    return 0;
  }
  static constexpr int TEAMS = pick();
  static constexpr int S = TEAMS ? (slots_for(TEAMS) > 16 ? 16 : slots_for(TEAMS)) : 1;
  static constexpr bool ok = TEAMS >= 1;
};

// ut may overlay staged vector 3 when that is 1/diag (CgK1Pol with Jacobi)
template <class Pol>
constexpr bool dmma10_ovl() {
  return Pol::NV >= 4 && Pol::BMQ != 3;
}

// Pol: CgK1Pol (cg.cu), as for k1_dmma_kernel.
template <class Pol, int TEAMS, int NSLOT>
__global__ void __launch_bounds__(Dmma10Layout<Pol::NV, TEAMS, NSLOT, dmma10_ovl<Pol>()>::threads, 1)
    k1_dmma10_kernel(typename Pol::Args args, const double* __restrict__ TL, int64_t E, double h1,
                     DParam<10> Dp, double* __restrict__ partials, QParam<10> Qp) {
  constexpr bool OVL = dmma10_ovl<Pol>();
  using L = Dmma10Layout<Pol::NV, TEAMS, NSLOT, OVL>;
  constexpr int NV = Pol::NV;
  constexpr int S = L::S;
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ double red_sm[32];
  __shared__ bool last_flag;
  typename Pol::Args args_l = args;
  partials = Pol::partials_of(args, partials);
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
  int* tag = reinterpret_cast<int*>(full + S);
  static_assert(S * 8 + S * 4 <= L::BAR_BYTES, "barrier area");
  double* sD = reinterpret_cast<double*>(smraw + L::BAR_BYTES);  // D[i][l]
  double* sQ = sD + 100;                                          // x[10], w[10]
  double* slots = sD + L::AUX_D;
  double* scratch = slots + S * L::SLOT_D;

  const int64_t M = E > (int64_t)blockIdx.x ? (E - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      tag[s] = -1;
    }
    mbar_fence_init();
  }
  // (compile-time indices into the by-value parameters only)
  if (threadIdx.x < 32) {
    const int l = threadIdx.x;
#pragma unroll
    for (int q = 0; q < 128; q += 32) {
      double v = 0.0;
#pragma unroll
      for (int t = 0; t < 32; ++t)
        if (q + t < 100 && l == t) v = Dp.d[q + t];
      if (q + l < 100) sD[q + l] = v;
    }
    if (l == 0) {
#pragma unroll
      for (int q = 0; q < 10; ++q) {
        sQ[q] = Qp.x[q];
        sQ[10 + q] = Qp.w[q];
      }
    }
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  if (!Pol::init_ptrs(args_l)) return;

  double red = 0.0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int team = warp >> 1, h = warp & 1, t64 = threadIdx.x & 63;
  auto issue = [&](int64_t m) {
    const int s = (int)(m % S);
    const int64_t e = blockIdx.x + m * gridDim.x;
    double* slot = slots + s * L::SLOT_D;
    *reinterpret_cast<volatile int*>(&tag[s]) = (int)m;
    mbar_expect_tx(&full[s], 24 * 8 + NV * 1000 * 8);
    tma_load_1d(slot, TL + e * 24, 24 * 8, &full[s]);
#pragma unroll
    for (int q = 0; q < NV; ++q)
      tma_load_1d(slot + L::G_D + q * L::V_D, Pol::vec(args_l, q) + e * 1000, 1000 * 8,
                  &full[s]);
  };
  constexpr int kIssuer = L::threads > 32 ? 32 : 0;
  if (threadIdx.x == kIssuer)
    for (int64_t m = 0; m < M && m < S; ++m) issue(m);
  if (!Pol::init_scalars(args_l)) {
    if (threadIdx.x == kIssuer)
      for (int64_t m = 0; m < M && m < S; ++m) mbar_wait(&full[m], 0u);
    Pol::finish(args_l, 0.0, partials, red_sm, &last_flag);  // (the ticket records why)
    return;
  }

  const int r4 = lane >> 2, c4 = lane & 3;
  // D fragments, zero outside the 10 x 10 matrix (the K = 12 padding):
  //   fA[s]     = D(8h + r4, 4s + c4): A of us / ut (row j or k), B of ur (col i)
  //   fAT[t][s] = D(4s + c4, 8t + r4): A of the second sweep's t / s parts
  //               (row k or j = 8t + r4), B of its r part (col i, t = h)
  auto dv = [&](int row, int col) { return (row < 10 && col < 10) ? sD[row * 10 + col] : 0.0; };
  double fA[3], fAT[2][3];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    fA[s] = dv(8 * h + r4, 4 * s + c4);
    fAT[0][s] = dv(4 * s + c4, r4);
    fAT[1][s] = dv(4 * s + c4, 8 + r4);
  }
  double fAh[3];  // fAT[h] (a register array is indexed at compile time only)
#pragma unroll
  for (int s = 0; s < 3; ++s) fAh[s] = h ? fAT[1][s] : fAT[0][s];
  int lk[3];  // the K index of this lane's operand, clamped into the element
#pragma unroll
  for (int s = 0; s < 3; ++s) lk[s] = (4 * s + c4) < 10 ? 4 * s + c4 : 9;
  double* const Tteam = scratch + team * L::T_D;
  const int bar = 1 + team;

  for (int64_t m = team; m < M; m += TEAMS) {
    const int s = (int)(m % S);
    const int64_t e = blockIdx.x + m * gridDim.x;
    while (*reinterpret_cast<volatile int*>(&tag[s]) != (int)m) __nanosleep(20);
    mbar_wait(&full[s], (uint32_t)((m / S) & 1));
    const int32_t* soff = Pol::send_index(args_l);  // multi-GPU send CSR, or null
    const int nsend = soff ? __ldg(soff + e + 1) - __ldg(soff + e) : 0;
    double* slot = slots + s * L::SLOT_D;
    double* V = slot + L::G_D;
    double* U = V;             // p          (overlays r)
    double* R = V + L::V_D;    // ur -> sr   (overlays p_old)
    double* Sx = V + 2 * L::V_D;  // us -> ss (overlays x)
    double* Tt = OVL ? V + 3 * L::V_D : Tteam;  // ut -> st -> w's t and s parts
    const int64_t ebase = e * 1000;
    // ---- prologue: z = r/diag, p = z + beta p_old, x += alpha_prev p_old
    for (int q = t64; q < 500; q += 64) {
      const int off = 2 * q;
      double va[NV], vb[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const double2 t = lds2(V + v * L::V_D + off);
        va[v] = t.x;
        vb[v] = t.y;
      }
      double u0, u1, hb0, hb1;
      Pol::pro2(args_l, va, vb, ebase + off, u0, u1, hb0, hb1);
      sts2(U + off, u0, u1);
    }
    named_bar_sync(bar, 64);
    // ---- first sweep: ur (cols i of tile h), us and ut (rows of tile h) --
#pragma unroll kD10Unroll
    for (int mt = 0; mt < 13; ++mt) {
      const int rr = 8 * mt + r4;
      const int ra = rr < 100 ? rr : 99;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int s3 = 0; s3 < 3; ++s3) dmma884(c0, c1, U[ra * 10 + lk[s3]], fA[s3]);
      const int io = 8 * h + 2 * c4;
      if (rr < 100 && io < 10) sts2(R + rr * 10 + io, c0, c1);
    }
#pragma unroll kD10Unroll
    for (int ct = 0; ct < 13; ++ct) {
      const int cb = (8 * ct + r4) < 100 ? 8 * ct + r4 : 99;
      const int kb = cb / 10, ib = cb - 10 * kb;
      double s0 = 0.0, s1 = 0.0, t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int s3 = 0; s3 < 3; ++s3) {
        dmma884(s0, s1, fA[s3], U[kb * 100 + lk[s3] * 10 + ib]);
        dmma884(t0, t1, fA[s3], U[lk[s3] * 100 + cb]);
      }
      const int row = 8 * h + r4, co = 8 * ct + 2 * c4;
      if (row < 10 && co < 100) {
        const int k = co / 10, i = co - 10 * k;
        sts2(Sx + k * 100 + row * 10 + i, s0, s1);
        sts2(Tt + row * 100 + co, t0, t1);
      }
    }
    named_bar_sync(bar, 64);
    // ---- trilinear metric, one lane per (i, j) column ---------------------
    for (int col = t64; col < 100; col += 64) {
      const int j = col / 10, i = col - 10 * j;
      const double* Gs = slot;
      const double ri = sQ[i], sj = sQ[j];
      const double wij = h1 * (sQ[10 + i] * sQ[10 + j]);
      double A[3], B[3], Cc[3], Ev[3], P0[3], P1[3], P2[3], qa, qb, qc;
      {
        auto cross = [](const double (&x)[3], const double (&y)[3], double (&o)[3]) {
          o[0] = fma(x[1], y[2], -x[2] * y[1]);
          o[1] = fma(x[2], y[0], -x[0] * y[2]);
          o[2] = fma(x[0], y[1], -x[1] * y[0]);
        };
        double a0[3], b0[3], a1[3], b1[3], c2[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double S0 = Gs[c], S1 = Gs[3 + c], S2 = Gs[6 + c], S01 = Gs[9 + c],
                       S02 = Gs[12 + c], S12 = Gs[15 + c], S012 = Gs[18 + c];
          a0[c] = fma(S01, sj, S0);
          b0[c] = fma(S012, sj, S02);
          a1[c] = fma(S01, ri, S1);
          b1[c] = fma(S012, ri, S12);
          c2[c] = fma(fma(S012, sj, S02), ri, fma(S12, sj, S2));
        }
        cross(a1, c2, A);
        cross(b1, c2, B);
        cross(c2, a0, Cc);
        cross(c2, b0, Ev);
        double u1[3], u2[3];
        cross(a0, a1, P0);
        cross(a0, b1, u1);
        cross(b0, a1, u2);
        cross(b0, b1, P2);
#pragma unroll
        for (int c = 0; c < 3; ++c) P1[c] = u1[c] + u2[c];
        qa = fma(a0[0], A[0], fma(a0[1], A[1], a0[2] * A[2]));
        qb = fma(a0[0], B[0], fma(a0[1], B[1], fma(a0[2], B[2], fma(b0[0], A[0],
             fma(b0[1], A[1], b0[2] * A[2])))));
        qc = fma(b0[0], B[0], fma(b0[1], B[1], b0[2] * B[2]));
      }
#pragma unroll
      for (int k = 0; k < 10; ++k) {
        const int off = k * 100 + col;
        const double r = R[off], sv = Sx[off], tt = Tt[off];
        const double t = Qp.x[k], wk = Qp.w[k];
        double r0[3], r1[3], r2[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          r0[c] = fma(B[c], t, A[c]);
          r1[c] = fma(Ev[c], t, Cc[c]);
          r2[c] = fma(fma(P2[c], t, P1[c]), t, P0[c]);
        }
        const double det = fma(fma(qc, t, qb), t, qa);
        const double f = (wij * wk) * fast_rcp(det);
        double v[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c] = fma(r, r0[c], fma(sv, r1[c], tt * r2[c]));
        R[off] = f * fma(r0[0], v[0], fma(r0[1], v[1], r0[2] * v[2]));
        Sx[off] = f * fma(r1[0], v[0], fma(r1[1], v[1], r1[2] * v[2]));
        Tt[off] = f * fma(r2[0], v[0], fma(r2[1], v[1], r2[2] * v[2]));
        if ((k & 1) == 1) asm volatile("" ::: "memory");
      }
    }
    named_bar_sync(bar, 64);
    // ---- second sweep, t part: W[k][(j,i)] = sum_l D(l,k) st[l][(j,i)],
    // in place over st (a warp owns whole column tiles, both row tiles, and
    // every lane's loads of a tile feed its DMMAs before any lane stores)
#pragma unroll kD10Unroll
    for (int ct = h; ct < 13; ct += 2) {
      const int cb = (8 * ct + r4) < 100 ? 8 * ct + r4 : 99;
      double b[3];
#pragma unroll
      for (int s3 = 0; s3 < 3; ++s3) b[s3] = Tt[lk[s3] * 100 + cb];
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
      for (int s3 = 0; s3 < 3; ++s3) {
        dmma884(a0, a1, fAT[0][s3], b[s3]);
        dmma884(a2, a3, fAT[1][s3], b[s3]);
      }
      const int co = 8 * ct + 2 * c4;
      if (co < 100) {
        sts2(Tt + r4 * 100 + co, a0, a1);
        if (8 + r4 < 10) sts2(Tt + (8 + r4) * 100 + co, a2, a3);
      }
    }
    named_bar_sync(bar, 64);
    // ---- s part: W[k][j][i] += sum_l D(l,j) ss[k][l][i] (rows j of tile h)
#pragma unroll kD10Unroll
    for (int ct = 0; ct < 13; ++ct) {
      const int row = 8 * h + r4, co = 8 * ct + 2 * c4;
      const bool v = row < 10 && co < 100;
      int woff = 0;
      double c0 = 0.0, c1 = 0.0;
      if (v) {
        const int k = co / 10, i = co - 10 * k;
        woff = k * 100 + row * 10 + i;
        const double2 t = lds2(Tt + woff);
        c0 = t.x;
        c1 = t.y;
      }
      const int cb = (8 * ct + r4) < 100 ? 8 * ct + r4 : 99;
      const int kb = cb / 10, ib = cb - 10 * kb;
#pragma unroll
      for (int s3 = 0; s3 < 3; ++s3) dmma884(c0, c1, fAh[s3], Sx[kb * 100 + lk[s3] * 10 + ib]);
      if (v) sts2(Tt + woff, c0, c1);
    }
    named_bar_sync(bar, 64);
    // ---- r part + epilogue: w[(k,j)][i] = W + sum_l sr[(k,j)][l] D(l,i) ---
#pragma unroll kD10Unroll
    for (int mt = 0; mt < 13; ++mt) {
      const int rr = 8 * mt + r4;
      const int ra = rr < 100 ? rr : 99;
      const int io = 8 * h + 2 * c4;
      const bool v = rr < 100 && io < 10;
      const int off = rr * 10 + io;
      double c0 = 0.0, c1 = 0.0;
      if (v) {
        const double2 t = lds2(Tt + off);
        c0 = t.x;
        c1 = t.y;
      }
#pragma unroll
      for (int s3 = 0; s3 < 3; ++s3) dmma884(c0, c1, R[ra * 10 + lk[s3]], fAh[s3]);
      if (v) {
        const double2 u = lds2(U + off);
        double hb0 = 0.0, hb1 = 0.0;
        if constexpr (Pol::BMQ >= 0) {
          const double2 bm = lds2(V + Pol::BMQ * L::V_D + off);
          hb0 = Pol::hb_of(args_l, bm.x);
          hb1 = Pol::hb_of(args_l, bm.y);
        }
        Pol::epi2(args_l, c0, c1, u.x, u.y, hb0, hb1, ebase + off, red);
      }
    }
    Pol::element_done(args_l, nsend, e, 1, 1000, t64, 64, bar);
    fence_proxy_async_smem();
    named_bar_sync(bar, 64);
    if (t64 == 0 && m + S < M) issue(m + S);  // refill the slot just released
  }
  Pol::finish(args_l, red, partials, red_sm, &last_flag);
}

}  // namespace sbx
