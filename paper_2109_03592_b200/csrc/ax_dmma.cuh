// K1 for n = 8 (N = 7) on the FP64 tensor cores: the r- and s-direction
// contractions of both sweeps as DMMA (mma.sync.aligned.m8n8k4 f64), the
// t-direction on the FMA pipe out of registers, the trilinear metric in
// between (sm_100a).
//
// Same pipeline as ax_tma_kernel (persistent, one CTA per SM, a producer warp
// streaming each element's trilinear map and its r, p_old, x [, 1/diag]
// [, bm] columns into per-group slots with 1-D TMA bulk copies), but a
// consumer group is ONE warp per element, and its thread ownership is the
// DMMA accumulator fragment:
//
//   lane -> row j = lane/4 of every 8x8 (j, i) plane, columns i = 2(lane%4)
//   and 2(lane%4)+1, all eight k planes: 16 nodes = two (i, j) columns.
//
// Per plane k the warp forms  ur(j,i) = sum_l u(k,j,l) D(i,l)   [A = u tile,
// B = D^T fragment],  us(j,i) = sum_l D(j,l) u(k,l,i)   [A = D fragment,
// B = u tile]  (2 DMMAs each, K = 8 as two k4 steps), and ut from the
// thread's own columns in registers (8 FMAs per node with compile-time
// D(k,l) constant-bank operands).  The second sweep accumulates
// sum_l D(l,i) sr(k,j,l) + sum_l D(l,j) ss(k,l,i) into ONE fragment (4 DMMAs
// per plane) and adds the t-term from registers.  Per node that is 16 FP64
// FMAs for the contractions instead of 48, and 4 shared-memory loads per
// plane per lane instead of ~28.
//
// Shared-memory tiles (u, sr, ss: 8 planes x 8 x 8, rows of 8 doubles with
// an XOR swizzle of the column by 4 on rows 2,3,6,7) are laid out so that
// every access is bank-conflict free: the fragment loads (row = lane/4,
// col = lane%4 (+4)) and (row = lane%4 (+4), col = lane/4) as 8-byte loads
// by half-warps, and the fragment stores (row = lane/4, cols 2(lane%4),+1)
// as 16-byte stores by quarter-warps.  The three tiles overlay the slot's
// staged r, p_old, x vectors once the warp has read them (bm, when staged,
// lies beyond them and is re-read in the epilogue).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "ax_core.cuh"
#include "ax_tma.cuh"
#include "tma.cuh"

namespace sbx {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// plane-local tile index of (row, col), 8x8 doubles, swizzled (see above)
__device__ __forceinline__ int dtix(int row, int col) {
  return row * 8 + (col ^ (((row >> 1) & 1) << 2));
}

__device__ __forceinline__ void sts2(double* p, double a, double b) {
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}

#ifndef SBX_DMMA_SELF
// 1: the consumer warps refill the ring themselves (a warp that releases slot
// s issues the loads of the unit S ahead into it), so all 8 warps of a
// 256-thread CTA compute; 0: a dedicated producer warp (A/B knob)
#define SBX_DMMA_SELF 1
#endif

template <int NV, int GROUPS, int NSLOT>
struct DmmaLayout {
  static constexpr int n3 = 512;
  static constexpr int G_D = 24;  // the element's trilinear map coefficients
  static constexpr int V_D = 512;
  static constexpr int SLOT_D = G_D + NV * V_D;
  static constexpr int S = NSLOT;
  static constexpr size_t BAR_BYTES = 1024;
  static constexpr int AUX_D = 64 + 16;  // D (row-major) and GLL x[8], w[8]
  static constexpr size_t smem = BAR_BYTES + sizeof(double) * (size_t)(AUX_D + S * SLOT_D);
  // self-refilling ring (SBX_DMMA_SELF): no producer warp
  static constexpr int threads = GROUPS * 32 + (SBX_DMMA_SELF ? 0 : 32);
  static_assert(NV >= 3, "the u / sr / ss tiles overlay three staged vectors");
};

#ifndef SBX_DMMA_MAXG
// consumer warps: 256 threads in all -> up to 255 registers per thread
#define SBX_DMMA_MAXG (SBX_DMMA_SELF ? 8 : 7)
#endif
#ifndef SBX_CONS_SUSPEND
#define SBX_CONS_SUSPEND 0  // consumers wait for their slot suspended (A/B knob)
#endif

// Slots are a shared ring (not owned per warp): as many as fit, each unit m
// (element) goes to slot m % S and warp m % GROUPS.  A consumer first waits
// for the slot's unit tag to read m -- the producer writes it only after the
// slot's previous unit was released -- so its parity wait on the full barrier
// can never match a phase two back.
template <int NV>
struct DmmaChoice {
  static constexpr size_t BUDGET = 225 * 1024;
  using L1 = DmmaLayout<NV, 1, 1>;
  static constexpr size_t FIXED = L1::BAR_BYTES + sizeof(double) * L1::AUX_D;
  static constexpr int fit = (int)((BUDGET - FIXED) / (sizeof(double) * L1::SLOT_D));
  static constexpr int S = fit > 16 ? 16 : fit;
  static constexpr int GROUPS = (S - 1) < SBX_DMMA_MAXG ? (S - 1) : SBX_DMMA_MAXG;
  static constexpr bool ok = GROUPS >= 1;
};

// Pol: the CG K1 policy of cg.cu (CgK1Pol): vec(q), pro(), epi(), hb_of(),
// finish(), send_index(), element_done(); BMQ = index of bm (or -1).
template <class Pol, int GROUPS, int NSLOT>
__global__ void __launch_bounds__(DmmaLayout<Pol::NV, GROUPS, NSLOT>::threads, 1)
    k1_dmma_kernel(typename Pol::Args args, const double* __restrict__ TL, int64_t E, double h1,
                   DParam<8> Dp, double* __restrict__ partials, QParam<8> Qp) {
  using L = DmmaLayout<Pol::NV, GROUPS, NSLOT>;
  constexpr int n = 8;
  constexpr int NV = Pol::NV;
  constexpr int S = L::S;
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ double red_sm[32];
  __shared__ bool last_flag;
  typename Pol::Args args_l = args;
  partials = Pol::partials_of(args, partials);
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
  uint64_t* empty = full + S;
  int* meta = reinterpret_cast<int*>(empty + S);
  int* tag = meta + S;  // unit index the slot currently holds (-1: none yet)
  static_assert(S * 16 + S * 8 <= L::BAR_BYTES, "barrier area");
  double* sD = reinterpret_cast<double*>(smraw + L::BAR_BYTES);  // D[i][l], row-major
  double* sQ = sD + 64;                                           // x[8], w[8]
  double* slots = sD + L::AUX_D;

  const int64_t M = E > (int64_t)blockIdx.x ? (E - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      tag[s] = -1;
    }
    mbar_fence_init();
  }
  // (compile-time indices only: a runtime index into a by-value kernel
  // parameter makes the compiler copy it to local memory, and every later
  // access -- the metric's Qp.x[k], Qp.w[k] -- becomes a local load)
  if (threadIdx.x < 32) {
    const int l = threadIdx.x;
#pragma unroll
    for (int q = 0; q < 64; q += 32) {
      double v = 0.0;
#pragma unroll
      for (int t = 0; t < 32; ++t)
        if (l == t) v = Dp.d[q + t];
      sD[q + l] = v;
    }
    if (l == 0) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        sQ[q] = Qp.x[q];
        sQ[8 + q] = Qp.w[q];
      }
    }
  }
  __syncthreads();
  // (launched programmatically after the update kernel: the set-up above
  // overlaps its tail; r and the scalars are read only from here on)
  pdl_wait();
  pdl_trigger();
  if (!Pol::init_ptrs(args_l)) return;

  double red = 0.0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // arm slot m % S for unit m and start its loads (one thread)
  auto issue = [&](int64_t m) {
    const int s = (int)(m % S);
    const int64_t e = blockIdx.x + m * gridDim.x;
    double* slot = slots + s * L::SLOT_D;
    *reinterpret_cast<volatile int*>(&tag[s]) = (int)m;
    mbar_expect_tx(&full[s], 24 * 8 + NV * 512 * 8);
    tma_load_1d(slot, TL + e * 24, 24 * 8, &full[s]);
#pragma unroll
    for (int q = 0; q < NV; ++q)
      tma_load_1d(slot + L::G_D + q * L::V_D, Pol::vec(args_l, q) + e * 512, 512 * 8, &full[s]);
  };
  // the first loads (thread 32: thread 0 takes the multi-GPU exchange below)
  constexpr int kIssuer = L::threads > 32 ? 32 : 0;
  if (SBX_DMMA_SELF && threadIdx.x == kIssuer)
    for (int64_t m = 0; m < M && m < S; ++m) issue(m);
  // the scalars (multi-GPU: after the r'z / r'r exchange, which the loads
  // just started overlap); a solve found finished drains the loads first
  if (!Pol::init_scalars(args_l)) {
    if (SBX_DMMA_SELF && threadIdx.x == kIssuer)
      for (int64_t m = 0; m < M && m < S; ++m) mbar_wait(&full[m], 0u);
    Pol::finish(args_l, 0.0, partials, red_sm, &last_flag);  // (the ticket records why)
    return;
  }
  if (!SBX_DMMA_SELF && warp == GROUPS) {
    // ---------------- producer warp: one lane drives the TMA ring ----------
    if (lane == 0) {
      constexpr int PD = 4;
      __shared__ int32_t sring[PD][2];
      const int32_t* soff = Pol::send_index(args_l);
      auto pf = [&](int64_t mm) {
        if (mm < M) {
          const int64_t e0 = blockIdx.x + mm * gridDim.x;
          cp_async4(&sring[mm % PD][0], soff + e0);
          cp_async4(&sring[mm % PD][1], soff + e0 + 1);
        }
        cp_async_commit();
      };
      if (soff)
        for (int d = 0; d < PD - 1; ++d) pf(d);
      for (int64_t m = 0; m < M; ++m) {
        const int s = (int)(m % S);
        if (m >= S) mbar_wait_backoff(&empty[s], (uint32_t)((m / S - 1) & 1));
        const int64_t e = blockIdx.x + m * gridDim.x;
        if (soff) {
          pf(m + PD - 1);
          cp_async_wait<PD - 1>();
          meta[s] = sring[m % PD][1] - sring[m % PD][0];
        } else {
          meta[s] = 0;
        }
        (void)e;
        issue(m);
      }
    }
  } else {
    // ---------------- consumer warps: one element per warp -----------------
    const int g = warp;
    const int jr = lane >> 2, q4 = lane & 3, i0 = 2 * q4;
    // D fragments: dA[h] = D(jr, q4 + 4h), dB[h] = D(q4 + 4h, jr)
    const double dA0 = sD[jr * 8 + q4], dA1 = sD[jr * 8 + q4 + 4];
    const double dB0 = sD[q4 * 8 + jr], dB1 = sD[(q4 + 4) * 8 + jr];
    const double sj = sQ[jr], ri0 = sQ[i0], ri1 = sQ[i0 + 1];
    const double wj = h1 * sQ[8 + jr];
    const double wij0 = wj * sQ[8 + i0], wij1 = wj * sQ[8 + i0 + 1];
    for (int64_t m = g; m < M; m += GROUPS) {
      const int s = (int)(m % S);
      const int64_t e = blockIdx.x + m * gridDim.x;
      while (*reinterpret_cast<volatile int*>(&tag[s]) != (int)m) __nanosleep(20);
      if (SBX_CONS_SUSPEND)
        mbar_wait_backoff(&full[s], (uint32_t)((m / S) & 1));
      else
        mbar_wait(&full[s], (uint32_t)((m / S) & 1));
      int nsend;
      if constexpr (SBX_DMMA_SELF) {
        const int32_t* soff = Pol::send_index(args_l);  // multi-GPU send CSR, or null
        nsend = soff ? __ldg(soff + e + 1) - __ldg(soff + e) : 0;
      } else {
        nsend = meta[s];
      }
      double* slot = slots + s * L::SLOT_D;
      double* V = slot + L::G_D;
      double* tu = V;          // u tile   (overlays r)
      double* tr = V + 512;    // sr tile  (overlays p_old)
      double* ts = V + 1024;   // ss tile  (overlays x)
      const int64_t ebase = e * 512;
      // ---- prologue: z = r/diag, p = z + beta p_old, x += alpha_prev p_old
      double uc0[n], uc1[n];
#pragma unroll
      for (int k = 0; k < n; ++k) {
        const int off = k * 64 + jr * 8 + i0;
        double va[NV], vb[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          const double2 t = lds2(V + q * L::V_D + off);
          va[q] = t.x;
          vb[q] = t.y;
        }
        double u0, u1, h0, h1v;
        Pol::pro2(args_l, va, vb, ebase + off, u0, u1, h0, h1v);
        uc0[k] = u0;
        uc1[k] = u1;
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < n; ++k) sts2(tu + k * 64 + dtix(jr, i0), uc0[k], uc1[k]);
      __syncwarp();
      // ---- column constants of the trilinear metric (two columns) --------
      // Gs: S0, S1, S2, S01, S02, S12, S012 (xyz each)
      const double* Gs = slot;
      double A0[3], B0[3], C0[3], E0[3], P00[3], P10[3], P20[3];
      double A1[3], B1[3], C1[3], E1[3], P01[3], P11[3], P21[3];
      double q00, q10, q20, q01, q11, q21;
      {
        auto cross = [](const double (&x)[3], const double (&y)[3], double (&o)[3]) {
          o[0] = fma(x[1], y[2], -x[2] * y[1]);
          o[1] = fma(x[2], y[0], -x[0] * y[2]);
          o[2] = fma(x[0], y[1], -x[1] * y[0]);
        };
        double a0[3], b0[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          a0[c] = fma(Gs[9 + c], sj, Gs[c]);
          b0[c] = fma(Gs[18 + c], sj, Gs[12 + c]);
        }
        auto column = [&](double ri, double (&A)[3], double (&B)[3], double (&Cc)[3],
                          double (&Ev)[3], double (&P0)[3], double (&P1)[3], double (&P2)[3],
                          double& qa, double& qb, double& qc) {
          double a1[3], b1[3], c2[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double S0 = Gs[c], S1 = Gs[3 + c], S2 = Gs[6 + c], S01 = Gs[9 + c],
                         S02 = Gs[12 + c], S12 = Gs[15 + c], S012 = Gs[18 + c];
            (void)S0;
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
        };
        column(ri0, A0, B0, C0, E0, P00, P10, P20, q00, q10, q20);
        column(ri1, A1, B1, C1, E1, P01, P11, P21, q01, q11, q21);
      }
      // ---- first sweep + metric --------------------------------------------
      // t-direction of the thread's own columns first, so the column values
      // die here and the t-derivatives die plane by plane below
      double ut0[n], ut1[n];
#pragma unroll
      for (int k = 0; k < n; ++k) {
        double t0 = 0.0, t1 = 0.0;
#pragma unroll
        for (int l = 0; l < n; ++l) {
          t0 = fma(Dp.d[k * n + l], uc0[l], t0);
          t1 = fma(Dp.d[k * n + l], uc1[l], t1);
        }
        ut0[k] = t0;
        ut1[k] = t1;
      }
      double wt0[n], wt1[n];
#pragma unroll
      for (int k = 0; k < n; ++k) {
        const double* up = tu + k * 64;
        double cr0 = 0.0, cr1 = 0.0, cs0 = 0.0, cs1 = 0.0;
        dmma884(cr0, cr1, up[dtix(jr, q4)], dA0);
        dmma884(cr0, cr1, up[dtix(jr, q4 + 4)], dA1);
        dmma884(cs0, cs1, dA0, up[dtix(q4, jr)]);
        dmma884(cs0, cs1, dA1, up[dtix(q4 + 4, jr)]);
        const double t0 = ut0[k], t1 = ut1[k];
        const double t = Qp.x[k], wk = Qp.w[k];
        auto metric = [&](double r, double sv, double tt, const double (&A)[3],
                          const double (&B)[3], const double (&Cc)[3], const double (&Ev)[3],
                          const double (&P0)[3], const double (&P1)[3], const double (&P2)[3],
                          double qa, double qb, double qc, double wij, double& o_r,
                          double& o_s, double& o_t) {
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
          o_r = f * fma(r0[0], v[0], fma(r0[1], v[1], r0[2] * v[2]));
          o_s = f * fma(r1[0], v[0], fma(r1[1], v[1], r1[2] * v[2]));
          o_t = f * fma(r2[0], v[0], fma(r2[1], v[1], r2[2] * v[2]));
        };
        double sr0, ss0, sr1, ss1;
        metric(cr0, cs0, t0, A0, B0, C0, E0, P00, P10, P20, q00, q10, q20, wij0, sr0, ss0,
               wt0[k]);
        metric(cr1, cs1, t1, A1, B1, C1, E1, P01, P11, P21, q01, q11, q21, wij1, sr1, ss1,
               wt1[k]);
        sts2(tr + k * 64 + dtix(jr, i0), sr0, sr1);
        sts2(ts + k * 64 + dtix(jr, i0), ss0, ss1);
        if ((k & 1) == 1) asm volatile("" ::: "memory");
      }
      __syncwarp();
      // ---- second sweep + epilogue ----------------------------------------
      // t-terms of the thread's own columns first (the wt die here)
      double ct0[n], ct1[n];
#pragma unroll
      for (int k = 0; k < n; ++k) {
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int l = 0; l < n; ++l) {
          c0 = fma(Dp.d[l * n + k], wt0[l], c0);
          c1 = fma(Dp.d[l * n + k], wt1[l], c1);
        }
        ct0[k] = c0;
        ct1[k] = c1;
      }
#pragma unroll
      for (int k = 0; k < n; ++k) {
        const double* rp = tr + k * 64;
        const double* sp = ts + k * 64;
        double a0 = 0.0, a1 = 0.0;
        dmma884(a0, a1, rp[dtix(jr, q4)], dB0);
        dmma884(a0, a1, rp[dtix(jr, q4 + 4)], dB1);
        dmma884(a0, a1, dB0, sp[dtix(q4, jr)]);
        dmma884(a0, a1, dB1, sp[dtix(q4 + 4, jr)]);
        const double c0 = ct0[k], c1 = ct1[k];
        const double2 u = lds2(tu + k * 64 + dtix(jr, i0));
        const int off = k * 64 + jr * 8 + i0;
        double hb0 = 0.0, hb1 = 0.0;
        if constexpr (Pol::BMQ >= 0) {
          const double2 bm = lds2(V + Pol::BMQ * L::V_D + off);
          hb0 = Pol::hb_of(args_l, bm.x);
          hb1 = Pol::hb_of(args_l, bm.y);
        }
        Pol::epi2(args_l, a0 + c0, a1 + c1, u.x, u.y, hb0, hb1, ebase + off, red);
        if ((k & 1) == 1) asm volatile("" ::: "memory");
      }
      Pol::element_done(args_l, nsend, e, 1, 512, lane, 32, 1 + g);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (SBX_DMMA_SELF) {
          if (m + S < M) issue(m + S);  // refill the slot just released
        } else {
          mbar_arrive(&empty[s]);
        }
      }
    }
  }
  Pol::finish(args_l, red, partials, red_sm, &last_flag);
}

// ---- standalone axhelm at n = 8 on the FP64 tensor cores (stored geometry) --
// The same warp-per-element DMMA scheme for the operator alone (the BASELINE
// configs[1] microbench): each slot holds the element's packed G [6][512],
// u [, bm]; per plane the two columns' six factors are read into registers,
// and after a __syncwarp the plane's sr / ss values overwrite the g1 / g2
// planes just consumed (the u tile overlays u).  w = h1 D^T G D u + h2 bm u.
template <bool HAS_BM>
struct AxDmmaLayout {
  static constexpr int NV = HAS_BM ? 2 : 1;
  static constexpr int SLOT_D = 6 * 512 + NV * 512;
  static constexpr size_t BAR_BYTES = 1024;
  static constexpr int AUX_D = 64;
  static constexpr size_t BUDGET = 225 * 1024;
  static constexpr int fit =
      (int)((BUDGET - BAR_BYTES - sizeof(double) * AUX_D) / (sizeof(double) * SLOT_D));
  static constexpr int S = fit > 16 ? 16 : fit;
  static constexpr int GROUPS = (S - 1) < 8 ? (S - 1) : 8;
  static constexpr size_t smem = BAR_BYTES + sizeof(double) * (size_t)(AUX_D + S * SLOT_D);
  static constexpr int threads = GROUPS * 32;
};

template <bool HAS_BM>
__global__ void __launch_bounds__(AxDmmaLayout<HAS_BM>::threads, 1)
    ax_dmma_kernel(const double* __restrict__ U, const double* __restrict__ G,
                   const double* __restrict__ BM, double* __restrict__ W, int64_t E, double h1,
                   double h2, double tsign, DParam<8> Dp) {
  using L = AxDmmaLayout<HAS_BM>;
  constexpr int n = 8, S = L::S, GROUPS = L::GROUPS, NV = L::NV;
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
  int* tag = reinterpret_cast<int*>(full + S);
  static_assert(S * 8 + S * 4 <= L::BAR_BYTES, "barrier area");
  double* sD = reinterpret_cast<double*>(smraw + L::BAR_BYTES);
  double* slots = sD + L::AUX_D;
  const int64_t M = E > (int64_t)blockIdx.x ? (E - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      tag[s] = -1;
    }
    mbar_fence_init();
  }
  if (threadIdx.x < 32) {
    const int l = threadIdx.x;
#pragma unroll
    for (int q = 0; q < 64; q += 32) {
      double v = 0.0;
#pragma unroll
      for (int t = 0; t < 32; ++t)
        if (l == t) v = Dp.d[q + t];
      sD[q + l] = v;
    }
  }
  __syncthreads();
  auto issue = [&](int64_t m) {
    const int s = (int)(m % S);
    const int64_t e = blockIdx.x + m * gridDim.x;
    double* slot = slots + s * L::SLOT_D;
    *reinterpret_cast<volatile int*>(&tag[s]) = (int)m;
    mbar_expect_tx(&full[s], (6 + NV) * 512 * 8);
    tma_load_1d(slot, G + e * 6 * 512, 6 * 512 * 8, &full[s]);
    tma_load_1d(slot + 6 * 512, U + e * 512, 512 * 8, &full[s]);
    if (HAS_BM) tma_load_1d(slot + 7 * 512, BM + e * 512, 512 * 8, &full[s]);
  };
  if (threadIdx.x == 0)
    for (int64_t m = 0; m < M && m < S; ++m) issue(m);
  const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int jr = lane >> 2, q4 = lane & 3, i0 = 2 * q4;
  const double dA0 = sD[jr * 8 + q4], dA1 = sD[jr * 8 + q4 + 4];
  const double dB0 = sD[q4 * 8 + jr], dB1 = sD[(q4 + 4) * 8 + jr];
  for (int64_t m = g; m < M; m += GROUPS) {
    const int s = (int)(m % S);
    const int64_t e = blockIdx.x + m * gridDim.x;
    while (*reinterpret_cast<volatile int*>(&tag[s]) != (int)m) __nanosleep(20);
    mbar_wait(&full[s], (uint32_t)((m / S) & 1));
    double* slot = slots + s * L::SLOT_D;
    double* Gs = slot;               // g1..g6, [6][512]; g1 / g2 planes become sr / ss
    double* tu = slot + 6 * 512;     // u -> u tile
    const int64_t ebase = e * 512;
    double uc0[n], uc1[n];
#pragma unroll
    for (int k = 0; k < n; ++k) {
      const double2 t = lds2(tu + k * 64 + jr * 8 + i0);
      uc0[k] = t.x;
      uc1[k] = t.y;
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < n; ++k) sts2(tu + k * 64 + dtix(jr, i0), uc0[k], uc1[k]);
    __syncwarp();
    double ut0[n], ut1[n];
#pragma unroll
    for (int k = 0; k < n; ++k) {
      double t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int l = 0; l < n; ++l) {
        t0 = fma(Dp.d[k * n + l], uc0[l], t0);
        t1 = fma(Dp.d[k * n + l], uc1[l], t1);
      }
      ut0[k] = t0;
      ut1[k] = t1;
    }
    double wt0[n], wt1[n];
#pragma unroll
    for (int k = 0; k < n; ++k) {
      const double* up = tu + k * 64;
      double cr0 = 0.0, cr1 = 0.0, cs0 = 0.0, cs1 = 0.0;
      dmma884(cr0, cr1, up[dtix(jr, q4)], dA0);
      dmma884(cr0, cr1, up[dtix(jr, q4 + 4)], dA1);
      dmma884(cs0, cs1, dA0, up[dtix(q4, jr)]);
      dmma884(cs0, cs1, dA1, up[dtix(q4 + 4, jr)]);
      // the plane's six factors of both columns (node (i0 | i0+1, jr, k))
      const int off = k * 64 + jr * 8 + i0;
      double2 gg[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) gg[c] = lds2(Gs + c * 512 + off);
      __syncwarp();  // every lane has read plane k of g1 / g2: overwrite it
      const double sr0 = h1 * fma(gg[0].x, cr0, fma(gg[3].x, cs0, gg[4].x * ut0[k]));
      const double ss0 = h1 * fma(gg[1].x, cs0, fma(gg[3].x, cr0, gg[5].x * ut0[k]));
      wt0[k] = h1 * fma(gg[2].x, ut0[k], fma(gg[4].x, cr0, gg[5].x * cs0));
      const double sr1 = h1 * fma(gg[0].y, cr1, fma(gg[3].y, cs1, gg[4].y * ut1[k]));
      const double ss1 = h1 * fma(gg[1].y, cs1, fma(gg[3].y, cr1, gg[5].y * ut1[k]));
      wt1[k] = h1 * fma(gg[2].y, ut1[k], fma(gg[4].y, cr1, gg[5].y * cs1));
      sts2(Gs + k * 64 + dtix(jr, i0), sr0, sr1);
      sts2(Gs + 512 + k * 64 + dtix(jr, i0), ss0, ss1);
    }
    __syncwarp();
    double ct0[n], ct1[n];
#pragma unroll
    for (int k = 0; k < n; ++k) {
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int l = 0; l < n; ++l) {
        c0 = fma(tsign * Dp.d[l * n + k], wt0[l], c0);
        c1 = fma(tsign * Dp.d[l * n + k], wt1[l], c1);
      }
      ct0[k] = c0;
      ct1[k] = c1;
    }
#pragma unroll
    for (int k = 0; k < n; ++k) {
      const double* rp = Gs + k * 64;
      const double* sp = Gs + 512 + k * 64;
      double a0 = 0.0, a1 = 0.0;
      dmma884(a0, a1, rp[dtix(jr, q4)], dB0);
      dmma884(a0, a1, rp[dtix(jr, q4 + 4)], dB1);
      dmma884(a0, a1, dB0, sp[dtix(q4, jr)]);
      dmma884(a0, a1, dB1, sp[dtix(q4 + 4, jr)]);
      double w0 = a0 + ct0[k], w1 = a1 + ct1[k];
      const int off = k * 64 + jr * 8 + i0;
      if constexpr (HAS_BM) {
        const double2 u = lds2(tu + k * 64 + dtix(jr, i0));
        const double2 b = lds2(slot + 7 * 512 + off);
        w0 = fma(h2 * b.x, u.x, w0);
        w1 = fma(h2 * b.y, u.y, w1);
      }
      stg2(W + ebase + off, w0, w1);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0 && m + S < M) issue(m + S);
  }
}

}  // namespace sbx
