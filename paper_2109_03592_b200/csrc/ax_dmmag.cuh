// K1 on the FP64 tensor cores for an even n that does not tile 8 x 8 planes
// (used at n = 6, N = 5): the whole-element GEMM scheme of ax_dmma10.cuh
// with n as a template parameter.  A team of W = ceil(n / 8) warps owns an
// element; the six contractions of axhelm are GEMMs over the element with the
// contracted index as K (padded to a multiple of 4 with zero D fragments),
// m8n8k4 DMMA tiles; the trilinear metric runs one lane per (i, j) column.
// At n = 6 the metric comes from the element's trilinear map (24 doubles)
// instead of the six stored factors, so K1 streams 56 B per node instead of
// 104 -- the reason for this kernel: the FMA pipeline could not afford the
// on-the-fly metric at n = 6 (SBX_TRI_MINN), the tensor cores can.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "ax_dmma.cuh"

namespace sbx {

#ifndef SBX_DMMAG_MAXT
#define SBX_DMMAG_MAXT 384  // threads per CTA at most (168 registers each)
#endif

template <int n>
struct DmmaGGeom {
  static constexpr int NN = n * n, N3 = n * n * n;
  static constexpr int W = (n + 7) / 8;     // warps per team: tiles along an n-dimension
  static constexpr int KS = (n + 3) / 4;    // k4 steps
  static constexpr int RT = (NN + 7) / 8;   // tiles along an n^2-dimension
  static_assert(n % 2 == 0, "pairs of nodes (16-byte accesses)");
};

template <int n, int NV, int TEAMS, int NSLOT, bool OVL>
struct DmmaGLayout {
  using T = DmmaGGeom<n>;
  static constexpr int G_D = 24;
  static constexpr int V_D = T::N3;
  static constexpr int SLOT_D = G_D + NV * V_D;
  static constexpr int S = NSLOT;
  static constexpr int T_D = OVL ? 0 : T::N3;  // per-team scratch for ut (OVL: over 1/diag)
  static constexpr size_t BAR_BYTES = 1024;
  static constexpr int AUX_D = ((n * n + 2 * n + 1) / 2) * 2;  // D, GLL x[n], w[n]
  static constexpr size_t smem =
      BAR_BYTES + sizeof(double) * (size_t)(AUX_D + S * SLOT_D + TEAMS * T_D);
  static constexpr int threads = TEAMS * T::W * 32;
  static_assert(NV >= 3, "the sr / ss tiles overlay the staged p_old and x");
};

template <int n, int NV, bool OVL>
struct DmmaGChoice {
  using T = DmmaGGeom<n>;
  static constexpr size_t BUDGET = 225 * 1024;
  static constexpr size_t slot_b = sizeof(double) * (24 + (size_t)NV * T::N3);
  static constexpr size_t fixed_b(int t) {
    return 1024 + sizeof(double) * (DmmaGLayout<n, NV, 1, 1, OVL>::AUX_D +
                                    (OVL ? 0 : (size_t)t * T::N3));
  }
  static constexpr int slots_for(int t) {
    return fixed_b(t) >= BUDGET ? 0 : (int)((BUDGET - fixed_b(t)) / slot_b);
  }
  static constexpr int pick() {
    for (int t = SBX_DMMAG_MAXT / (T::W * 32); t >= 1; --t)
      if (t <= 15 && slots_for(t) >= t + 1) return t;  // (named barriers 1..15)
    return 0;
  }
  static constexpr int TEAMS = pick();
  static constexpr int S = TEAMS ? (slots_for(TEAMS) > 16 ? 16 : slots_for(TEAMS)) : 1;
  static constexpr bool ok = TEAMS >= 1;
};

template <class Pol>
constexpr bool dmmag_ovl() {
  return Pol::NV >= 4 && Pol::BMQ != 3;
}

template <int n, class Pol, int TEAMS, int NSLOT>
__global__ void __launch_bounds__(DmmaGLayout<n, Pol::NV, TEAMS, NSLOT, dmmag_ovl<Pol>()>::threads,
                                  1)
    k1_dmmag_kernel(typename Pol::Args args, const double* __restrict__ TL, int64_t E, double h1,
                    DParam<n> Dp, double* __restrict__ partials, QParam<n> Qp) {
  constexpr bool OVL = dmmag_ovl<Pol>();
  using T = DmmaGGeom<n>;
  using L = DmmaGLayout<n, Pol::NV, TEAMS, NSLOT, OVL>;
  constexpr int NV = Pol::NV;
  constexpr int S = L::S;
  constexpr int NN = T::NN, N3 = T::N3, W = T::W, KS = T::KS, RT = T::RT, TT = W * 32;
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ double red_sm[32];
  __shared__ bool last_flag;
  typename Pol::Args args_l = args;
  partials = Pol::partials_of(args, partials);
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
  int* tag = reinterpret_cast<int*>(full + S);
  static_assert(S * 8 + S * 4 <= L::BAR_BYTES, "barrier area");
  double* sD = reinterpret_cast<double*>(smraw + L::BAR_BYTES);  // D[i][l]
  double* sQ = sD + NN;                                           // x[n], w[n]
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
    for (int q = 0; q < ((NN + 31) / 32) * 32; q += 32) {
      double v = 0.0;
#pragma unroll
      for (int t = 0; t < 32; ++t)
        if (q + t < NN && l == t) v = Dp.d[q + t];
      if (q + l < NN) sD[q + l] = v;
    }
    if (l == 0) {
#pragma unroll
      for (int q = 0; q < n; ++q) {
        sQ[q] = Qp.x[q];
        sQ[n + q] = Qp.w[q];
      }
    }
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  if (!Pol::init_ptrs(args_l)) return;

  double red = 0.0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int team = warp / W, h = warp % W, tt = threadIdx.x % TT;
  auto issue = [&](int64_t m) {
    const int s = (int)(m % S);
    const int64_t e = blockIdx.x + m * gridDim.x;
    double* slot = slots + s * L::SLOT_D;
    *reinterpret_cast<volatile int*>(&tag[s]) = (int)m;
    mbar_expect_tx(&full[s], 24 * 8 + NV * N3 * 8);
    tma_load_1d(slot, TL + e * 24, 24 * 8, &full[s]);
#pragma unroll
    for (int q = 0; q < NV; ++q)
      tma_load_1d(slot + L::G_D + q * L::V_D, Pol::vec(args_l, q) + e * N3, N3 * 8, &full[s]);
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
  // D fragments, zero outside the n x n matrix (the K padding):
  //   fA[s]     = D(8h + r4, 4s + c4): A of us / ut (row j or k), B of ur (col i)
  //   fAT[t][s] = D(4s + c4, 8t + r4): A of the second sweep's t / s parts
  //               (row k or j = 8t + r4), B of its r part (col i, t = h)
  auto dv = [&](int row, int col) { return (row < n && col < n) ? sD[row * n + col] : 0.0; };
  double fA[KS], fAT[W][KS], fAh[KS];
  int lk[KS];  // the K index of this lane's operand, clamped into the element
#pragma unroll
  for (int s = 0; s < KS; ++s) {
    fA[s] = dv(8 * h + r4, 4 * s + c4);
#pragma unroll
    for (int t = 0; t < W; ++t) fAT[t][s] = dv(4 * s + c4, 8 * t + r4);
    fAh[s] = dv(4 * s + c4, 8 * h + r4);
    lk[s] = (4 * s + c4) < n ? 4 * s + c4 : n - 1;
  }
  double* const Tteam = scratch + team * L::T_D;
  const int bar = 1 + team;
  auto team_sync = [&]() {
    if constexpr (W == 1)
      __syncwarp();
    else
      named_bar_sync(bar, TT);
  };

  for (int64_t m = team; m < M; m += TEAMS) {
    const int s = (int)(m % S);
    const int64_t e = blockIdx.x + m * gridDim.x;
    while (*reinterpret_cast<volatile int*>(&tag[s]) != (int)m) __nanosleep(20);
    mbar_wait(&full[s], (uint32_t)((m / S) & 1));
    const int32_t* soff = Pol::send_index(args_l);  // multi-GPU send CSR, or null
    const int nsend = soff ? __ldg(soff + e + 1) - __ldg(soff + e) : 0;
    double* slot = slots + s * L::SLOT_D;
    double* V = slot + L::G_D;
    double* U = V;                // p          (overlays r)
    double* R = V + L::V_D;       // ur -> sr   (overlays p_old)
    double* Sx = V + 2 * L::V_D;  // us -> ss   (overlays x)
    double* Tt = OVL ? V + 3 * L::V_D : Tteam;  // ut -> st -> w's t and s parts
    const int64_t ebase = e * N3;
    // ---- prologue: z = r/diag, p = z + beta p_old, x += alpha_prev p_old
    for (int q = tt; q < N3 / 2; q += TT) {
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
    team_sync();
    // ---- first sweep: ur (cols i of tile h), us and ut (rows of tile h) --
    for (int mt = 0; mt < RT; ++mt) {
      const int rr = 8 * mt + r4;
      const int ra = rr < NN ? rr : NN - 1;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int s3 = 0; s3 < KS; ++s3) dmma884(c0, c1, U[ra * n + lk[s3]], fA[s3]);
      const int io = 8 * h + 2 * c4;
      if (rr < NN && io < n) sts2(R + rr * n + io, c0, c1);
    }
    for (int ct = 0; ct < RT; ++ct) {
      const int cb = (8 * ct + r4) < NN ? 8 * ct + r4 : NN - 1;
      const int kb = cb / n, ib = cb - n * kb;
      double s0 = 0.0, s1 = 0.0, t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int s3 = 0; s3 < KS; ++s3) {
        dmma884(s0, s1, fA[s3], U[kb * NN + lk[s3] * n + ib]);
        dmma884(t0, t1, fA[s3], U[lk[s3] * NN + cb]);
      }
      const int row = 8 * h + r4, co = 8 * ct + 2 * c4;
      if (row < n && co < NN) {
        const int k = co / n, i = co - n * k;
        sts2(Sx + k * NN + row * n + i, s0, s1);
        sts2(Tt + row * NN + co, t0, t1);
      }
    }
    team_sync();
    // ---- trilinear metric, one lane per (i, j) column ---------------------
    // (column constants: the adjugate rows are polynomials in t along a column)
    struct ColC {
      double A[3], B[3], Cc[3], Ev[3], P0[3], P1[3], P2[3], qa, qb, qc, wij;
    };
    auto col_consts = [&](int col, ColC& c) {
      const int j = col / n, i = col - n * j;
      const double* Gs = slot;
      const double ri = sQ[i], sj = sQ[j];
      c.wij = h1 * (sQ[n + i] * sQ[n + j]);
      auto cross = [](const double (&x)[3], const double (&y)[3], double (&o)[3]) {
        o[0] = fma(x[1], y[2], -x[2] * y[1]);
        o[1] = fma(x[2], y[0], -x[0] * y[2]);
        o[2] = fma(x[0], y[1], -x[1] * y[0]);
      };
      double a0[3], b0[3], a1[3], b1[3], c2[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const double S0 = Gs[q], S1 = Gs[3 + q], S2 = Gs[6 + q], S01 = Gs[9 + q],
                     S02 = Gs[12 + q], S12 = Gs[15 + q], S012 = Gs[18 + q];
        a0[q] = fma(S01, sj, S0);
        b0[q] = fma(S012, sj, S02);
        a1[q] = fma(S01, ri, S1);
        b1[q] = fma(S012, ri, S12);
        c2[q] = fma(fma(S012, sj, S02), ri, fma(S12, sj, S2));
      }
      cross(a1, c2, c.A);
      cross(b1, c2, c.B);
      cross(c2, a0, c.Cc);
      cross(c2, b0, c.Ev);
      double u1[3], u2[3];
      cross(a0, a1, c.P0);
      cross(a0, b1, u1);
      cross(b0, a1, u2);
      cross(b0, b1, c.P2);
#pragma unroll
      for (int q = 0; q < 3; ++q) c.P1[q] = u1[q] + u2[q];
      c.qa = fma(a0[0], c.A[0], fma(a0[1], c.A[1], a0[2] * c.A[2]));
      c.qb = fma(a0[0], c.B[0], fma(a0[1], c.B[1], fma(a0[2], c.B[2], fma(b0[0], c.A[0],
             fma(b0[1], c.A[1], b0[2] * c.A[2])))));
      c.qc = fma(b0[0], c.B[0], fma(b0[1], c.B[1], b0[2] * c.B[2]));
    };
    auto metric_node = [&](const ColC& c, int off, double t, double wk) {
      const double r = R[off], sv = Sx[off], tv = Tt[off];
      double r0[3], r1[3], r2[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        r0[q] = fma(c.B[q], t, c.A[q]);
        r1[q] = fma(c.Ev[q], t, c.Cc[q]);
        r2[q] = fma(fma(c.P2[q], t, c.P1[q]), t, c.P0[q]);
      }
      const double det = fma(fma(c.qc, t, c.qb), t, c.qa);
      const double f = (c.wij * wk) * fast_rcp(det);
      double v[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) v[q] = fma(r, r0[q], fma(sv, r1[q], tv * r2[q]));
      R[off] = f * fma(r0[0], v[0], fma(r0[1], v[1], r0[2] * v[2]));
      Sx[off] = f * fma(r1[0], v[0], fma(r1[1], v[1], r1[2] * v[2]));
      Tt[off] = f * fma(r2[0], v[0], fma(r2[1], v[1], r2[2] * v[2]));
    };
    // whole columns while every lane has one; a remainder that fits one round
    // when split by plane (n = 6: 4 columns x 6 planes on 24 lanes) goes node
    // by node instead of leaving the last round with 4 busy lanes
    constexpr int FULL = NN / TT, LEFT = NN - FULL * TT;
    constexpr bool SPLIT = LEFT > 0 && LEFT * n <= TT;
    constexpr int COLS = SPLIT ? FULL * TT : NN;
    for (int col = tt; col < COLS; col += TT) {
      ColC c;
      col_consts(col, c);
#pragma unroll
      for (int k = 0; k < n; ++k) {
        metric_node(c, k * NN + col, Qp.x[k], Qp.w[k]);
        if ((k & 1) == 1) asm volatile("" ::: "memory");
      }
    }
    if constexpr (SPLIT) {
      if (tt < LEFT * n) {
        const int col = COLS + tt / n, k = tt - n * (tt / n);
        ColC c;
        col_consts(col, c);
        metric_node(c, k * NN + col, sQ[k], sQ[n + k]);
      }
    }
    team_sync();
    // ---- second sweep, t part: W[k][(j,i)] = sum_l D(l,k) st[l][(j,i)], in
    // place over st (a warp owns whole column tiles, every row tile, and all
    // lanes' loads of a tile feed its DMMAs before any lane stores)
    for (int ct = h; ct < RT; ct += W) {
      const int cb = (8 * ct + r4) < NN ? 8 * ct + r4 : NN - 1;
      double b[KS];
#pragma unroll
      for (int s3 = 0; s3 < KS; ++s3) b[s3] = Tt[lk[s3] * NN + cb];
      double acc[W][2];
#pragma unroll
      for (int t = 0; t < W; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
      for (int s3 = 0; s3 < KS; ++s3)
#pragma unroll
        for (int t = 0; t < W; ++t) dmma884(acc[t][0], acc[t][1], fAT[t][s3], b[s3]);
      const int co = 8 * ct + 2 * c4;
      if (co < NN) {
#pragma unroll
        for (int t = 0; t < W; ++t)
          if (8 * t + r4 < n) sts2(Tt + (8 * t + r4) * NN + co, acc[t][0], acc[t][1]);
      }
    }
    team_sync();
    // ---- s part: W[k][j][i] += sum_l D(l,j) ss[k][l][i] (rows j of tile h)
    for (int ct = 0; ct < RT; ++ct) {
      const int row = 8 * h + r4, co = 8 * ct + 2 * c4;
      const bool v = row < n && co < NN;
      int woff = 0;
      double c0 = 0.0, c1 = 0.0;
      if (v) {
        const int k = co / n, i = co - n * k;
        woff = k * NN + row * n + i;
        const double2 t = lds2(Tt + woff);
        c0 = t.x;
        c1 = t.y;
      }
      const int cb = (8 * ct + r4) < NN ? 8 * ct + r4 : NN - 1;
      const int kb = cb / n, ib = cb - n * kb;
#pragma unroll
      for (int s3 = 0; s3 < KS; ++s3) dmma884(c0, c1, fAh[s3], Sx[kb * NN + lk[s3] * n + ib]);
      if (v) sts2(Tt + woff, c0, c1);
    }
    team_sync();
    // ---- r part + epilogue: w[(k,j)][i] = W + sum_l sr[(k,j)][l] D(l,i) ---
    for (int mt = 0; mt < RT; ++mt) {
      const int rr = 8 * mt + r4;
      const int ra = rr < NN ? rr : NN - 1;
      const int io = 8 * h + 2 * c4;
      const bool v = rr < NN && io < n;
      const int off = rr * n + io;
      double c0 = 0.0, c1 = 0.0;
      if (v) {
        const double2 t = lds2(Tt + off);
        c0 = t.x;
        c1 = t.y;
      }
#pragma unroll
      for (int s3 = 0; s3 < KS; ++s3) dmma884(c0, c1, R[ra * n + lk[s3]], fAh[s3]);
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
    Pol::element_done(args_l, nsend, e, 1, N3, tt, TT, bar);
    fence_proxy_async_smem();
    team_sync();
    if (tt == 0 && m + S < M) issue(m + S);  // refill the slot just released
  }
  Pol::finish(args_l, red, partials, red_sm, &last_flag);
}

}  // namespace sbx
