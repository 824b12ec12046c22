// Peer-window exchange kernels for the distributed PCG (included by cg.cu).
//
// A sender stores raw copy values straight into its neighbours' receive
// buffers over NVLink (IPC-mapped peer pointers), fences them at system scope
// once per storing thread, and releases a per-(phase, source) sequence flag in
// every peer's window; the receiver acquires the flags, then reads its own
// receive buffer.  Scalars travel in
// per-source mailboxes and are summed in rank order, so every rank computes
// bit-identical CG scalars.  Waits are bounded (kSpinTimeoutNs) and report a
// communication error instead of hanging.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace sbx {
namespace {

constexpr unsigned long long kSpinTimeoutNs = 20ull * 1000 * 1000 * 1000;

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Publication rule: local values are made visible at GPU scope (__threadfence;
// every peer access to this rank's memory goes through this GPU's L2).  A
// thread that stored into PEER memory (halo values over NVLink) takes one
// system-scope fence (__threadfence_system) after its last such store, before
// its CTA's ticket -- once per storing thread per kernel, not per store.  ONE
// thread then releases the flags (dist_release: a system fence, whose
// cumulativity orders every write it has observed -- including its own stores
// into peer mailboxes -- before the relaxed flag stores).  Readers acquire the
// flag with ld.acquire.sys.
__device__ __forceinline__ void dist_fence() { __threadfence(); }

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

// SBX_TRACE stamp: slot c of iteration it (one thread calls it).  Single GPU
// (SBX_TRACE1): the same slots in g_trace1 (0 K1 start, 1 K1 last CTA, 4 K2
// start, 5 K2 last CTA).
__device__ unsigned long long* g_trace1 = nullptr;
__device__ __forceinline__ void trace_stamp(const DistDev* D, int it, int c) {
  if (D && D->trace)
    D->trace[(it % kTraceIters) * 8 + c] = globaltimer();
  else if (!D && g_trace1)
    g_trace1[(it % kTraceIters) * 8 + c] = globaltimer();
}

// Release `phase` with sequence v to every other rank: ONE system-scope fence
// (it orders every write this thread has made or observed -- the mailboxes,
// and through the CTA tickets the halo stores the other threads fenced --
// before what follows), then relaxed system-scope flag stores: the PTX
// release pattern, paid once instead of once per peer (st.release.sys fences
// before each store, ~1 us apiece over NVLink).
__device__ __forceinline__ void dist_release(const DistDev& D, int phase, unsigned long long v) {
  __threadfence_system();
  for (int q = 0; q < D.nranks; ++q)
    if (q != D.rank) st_relaxed_sys(D.pflags[q] + phase * kMaxRanks + D.rank, v);
}

// Wait until every other rank released `phase` with sequence >= expected.
__device__ bool dist_wait_all(const DistDev& D, int phase, unsigned long long expected) {
  const unsigned long long t0 = globaltimer();
  for (int q = 0; q < D.nranks; ++q) {
    if (q == D.rank) continue;
    const unsigned long long* f = D.flags + phase * kMaxRanks + q;
    while (ld_acquire_sys(f) < expected) {
      if (globaltimer() - t0 > kSpinTimeoutNs) return false;
      __nanosleep(64);
    }
  }
  return true;
}

// Stores this rank's send values (w at the send lists) into the neighbours'
// receive buffers, its scalars into every rank's mailbox, then releases the
// phase flag on every rank.  slot: receive-buffer slot (0 loop, 1 standalone).
__global__ void dist_put_kernel(DistDev D, int phase, int slot, const double* __restrict__ w,
                                const double* __restrict__ scal, int nscal) {
  __shared__ bool last;
  const unsigned long long s = ld_volatile_u64(D.seq + phase);
  const int64_t par = (int64_t)((s + 1) & 1);
  const int64_t total = D.send_off[D.nnbr];
  // push into the neighbours' receive buffers over NVLink
  bool stored = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int qi = 0;
    while (i >= D.send_off[qi + 1]) ++qi;
    const int q = D.nbr[qi];
    D.precv[q][(slot * 2 + par) * D.precv_total[q] + D.pbase_for_me[q] + (i - D.send_off[qi])] =
        w[D.send_idx[i]];
    stored = true;
  }
  if (stored) __threadfence_system();  // this thread's remote stores, before the ticket
  dist_fence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(D.counter + phase, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  dist_fence();
  D.counter[phase] = 0;
  for (int q = 0; q < D.nranks; ++q)
    for (int c = 0; c < nscal; ++c)
      D.pmbox[q][mbox_index(phase, (int)par, D.rank, c)] = scal[c];
  dist_release(D, phase, s + 1);
  D.seq[phase] = s + 1;
}

// Rank-order sum of mailbox entry c of `phase`.
__device__ __forceinline__ double mbox_sum(const DistDev& D, int phase, int par, int c) {
  double v = 0.0;
  for (int q = 0; q < D.nranks; ++q) {
    const volatile double* m = D.mbox + mbox_index(phase, par, q, c);
    v += *m;
  }
  return v;
}

// Interface groups [t0, n_if) step dt: sum every copy in canonical order
// (local copies from f, remote ones from the receive buffer `par` of `slot`)
// and write the sum to the local copies (s*0 for masked ones when
// apply_mask).  Local copies are read through L2 (ld.global.cg): in the fused
// CG update kernel other SMs read these lines afterwards with cp.async, and no
// stale L1 line may be left behind.
// A thread's first interface group, its copy codes loaded ahead (they are
// static tables: the fused update kernel loads them before the halo wait).
struct IfacePre {
  static constexpr int kMax = 8;  // copies of a node: at most 8 elements
  int lo = 0, cnt = -1;            // cnt < 0: no group; > kMax: not preloaded
  int32_t code[kMax];
};

__device__ __forceinline__ IfacePre iface_preload(const DistDev& D, int64_t g) {
  IfacePre p;
  if (g < D.n_if) {
    p.lo = D.if_off[g];
    p.cnt = D.if_off[g + 1] - p.lo;
#pragma unroll
    for (int c = 0; c < IfacePre::kMax; ++c)
      if (c < p.cnt) p.code[c] = D.if_code[p.lo + c];
  }
  return p;
}

__device__ __forceinline__ void dist_iface_groups(const DistDev& D, int slot, int64_t par,
                                                  double* f, int apply_mask, int64_t t0,
                                                  int64_t dt, const IfacePre* pre = nullptr) {
  const double* rb = D.recvb + (int64_t)(slot * 2 + par) * D.recv_total;
  const int64_t NL = D.nodes_local;
  if (pre && pre->cnt >= 0 && pre->cnt <= IfacePre::kMax) {
    double v[IfacePre::kMax];
#pragma unroll
    for (int c = 0; c < IfacePre::kMax; ++c) {
      if (c < pre->cnt) {
        const int32_t code = pre->code[c];
        v[c] = code >= NL ? __ldcv(rb + (code - NL)) : __ldcg(f + (code < 0 ? ~code : code));
      }
    }
    double sum = 0.0;
#pragma unroll
    for (int c = 0; c < IfacePre::kMax; ++c)
      if (c < pre->cnt) sum += v[c];
#pragma unroll
    for (int c = 0; c < IfacePre::kMax; ++c) {
      if (c < pre->cnt) {
        const int32_t code = pre->code[c];
        if (code >= NL) continue;
        if (code >= 0)
          f[code] = sum;
        else
          f[~code] = apply_mask ? __dmul_rn(sum, 0.0) : sum;
      }
    }
    t0 += dt;
  }
  for (int64_t g = t0; g < D.n_if; g += dt) {
    const int lo = D.if_off[g], hi = D.if_off[g + 1];
    double sum = 0.0;
    for (int c = lo; c < hi; ++c) {
      const int32_t code = D.if_code[c];
      double v;
      if (code >= NL) {
        v = __ldcv(rb + (code - NL));
      } else {
        v = __ldcg(f + (code < 0 ? ~code : code));
      }
      sum += v;
    }
    for (int c = lo; c < hi; ++c) {
      const int32_t code = D.if_code[c];
      if (code >= NL) continue;
      if (code >= 0)
        f[code] = sum;
      else
        f[~code] = apply_mask ? __dmul_rn(sum, 0.0) : sum;
    }
  }
}

// Grid-wide barrier of a kernel whose CTAs are all resident (the persistent
// CG update kernel: grid <= #SMs, one CTA per SM).  gbar[0] counts arrivals,
// gbar[1] is the generation; bounded like the exchange waits.
__device__ __forceinline__ bool grid_barrier(unsigned int* gbar) {
  __shared__ int ok;
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* gen = gbar + 1;
    const unsigned int g0 = *gen;
    __threadfence();
    ok = 1;
    if (atomicAdd(gbar, 1u) == gridDim.x - 1) {
      gbar[0] = 0;
      __threadfence();
      atomicAdd(gbar + 1, 1u);
    } else {
      const unsigned long long t0 = globaltimer();
      unsigned int v;
      for (int spin = 0;; ++spin) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gbar + 1) : "memory");
        if (v != g0) break;
        if ((spin & 255) == 255 && globaltimer() - t0 > kSpinTimeoutNs) {
          ok = 0;
          break;
        }
      }
      __threadfence();
    }
  }
  __syncthreads();
  return ok != 0;
}

// Interface groups: wait for the halo, sum every copy in canonical order
// (local copies from f, remote ones from the receive buffer) and write the sum
// to the local copies (s*0 for masked ones when apply_mask).  In the CG loop
// (sc != null) block 0 also forms alpha = rz / sum_q pq_q and tests breakdown.
// (The fused CG loop does this inside the update kernel: k2_dist_prologue.)
__global__ void dist_iface_kernel(DistDev D, int phase, int slot, double* __restrict__ f,
                                  int apply_mask, CgScalars* __restrict__ sc) {
  __shared__ bool ok;
  if (sc && sc->done) return;
  if (threadIdx.x == 0) {
    if (sc && blockIdx.x == 0) trace_stamp(&D, sc->it, 2);
    ok = dist_wait_all(D, phase, ld_volatile_u64(D.seq + phase));
    if (!ok) *D.status = 1;
    if (sc && blockIdx.x == 0) trace_stamp(&D, sc->it, 3);
  }
  __syncthreads();
  if (!ok) {
    if (sc && blockIdx.x == 0 && threadIdx.x == 0) {
      sc->status = 8;
      sc->done = 1;
    }
    return;
  }
  if (sc && blockIdx.x == 0 && threadIdx.x == 0) {
    const double pq = mbox_sum(D, phase, (int)(ld_volatile_u64(D.seq + phase) & 1), 0);
    sc->pq = pq;
    if (!isfinite(pq) || pq <= 0.0) {
      sc->status = 5;
      sc->err_it = sc->it;
      sc->done = 1;
    } else {
      sc->alpha = sc->rz / pq;
    }
  }
  // remote copies were pushed into this rank's receive buffer
  dist_iface_groups(D, slot, (int64_t)(ld_volatile_u64(D.seq + phase) & 1), f, apply_mask,
                    (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                    (int64_t)gridDim.x * blockDim.x);
}

// Start of the fused multi-GPU CG update kernel (replaces dist_iface_kernel
// in the loop): every CTA waits for the halo and the p'Ap partials of phase 0,
// forms alpha = rz / sum_q pq_q itself (rank order: identical bits in every
// CTA and on every rank), assembles its share of the interface groups into w,
// and passes a grid barrier before any CTA reads w.  Returns false when the
// iteration must stop (exchange timeout, breakdown); block 0 records why.
__device__ bool k2_dist_prologue(const DistDev& D, double* w, CgScalars* __restrict__ sc,
                                 cudaGraphConditionalHandle cond, int use_cond,
                                 double& alpha) {
  __shared__ int st_sm;
  __shared__ double al_sm;
  const int it = sc->it;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // this thread's first interface group: codes loaded while thread 0 waits
  const IfacePre pre = iface_preload(D, t0);
  // phase 0 of this iteration (K1 advanced the sequence at its end)
  const unsigned long long s = ld_volatile_u64(D.seq);
  if (threadIdx.x == 0) {
    const double pq_loc = sc->pq_loc;
    if (blockIdx.x == 0) {
      trace_stamp(&D, it, 2);
      // K1 has completed, so the halo it pushed is visible system-wide:
      // publish this rank's p'Ap and release phase 0 to every peer
      for (int q = 0; q < D.nranks; ++q)
        if (q != D.rank) D.pmbox[q][mbox_index(0, (int)(s & 1), D.rank, 0)] = pq_loc;
      dist_release(D, 0, s);
    }
    int st = dist_wait_all(D, 0, s) ? 0 : 8;
    double a = 0.0, pq = 0.0;
    if (!st) {
      // rank order; this rank's own term from sc (identical in every CTA)
      for (int q = 0; q < D.nranks; ++q)
        pq += q == D.rank ? pq_loc
                          : *(const volatile double*)(D.mbox + mbox_index(0, (int)(s & 1), q, 0));
      if (!isfinite(pq) || pq <= 0.0)
        st = 5;
      else
        a = sc->rz / pq;
    }
    if (blockIdx.x == 0) {
      trace_stamp(&D, it, 3);
      if (st) {
        if (st == 8) *D.status = 1;
        sc->status = st;
        if (st == 5) sc->err_it = it;
        sc->done = 1;
        if (use_cond) cudaGraphSetConditional(cond, 0);
      } else {
        sc->pq = pq;
        sc->alpha = a;
      }
    }
    st_sm = st;
    al_sm = a;
  }
  __syncthreads();
  if (st_sm) return false;
  alpha = al_sm;
  dist_iface_groups(D, 0, (int64_t)(s & 1), w, 1, t0, (int64_t)gridDim.x * blockDim.x, &pre);
  if (!grid_barrier(D.gbar)) {
    if (threadIdx.x == 0) {
      *D.status = 1;
      sc->status = 8;
      sc->done = 1;
      if (use_cond) cudaGraphSetConditional(cond, 0);
    }
    return false;
  }
  // the assembled values are read next by TMA (async proxy) and cp.async
  asm volatile("fence.proxy.async.global;" ::: "memory");
  if (blockIdx.x == 0 && threadIdx.x == 0) trace_stamp(&D, it, 4);
  return true;
}

// Scalar all-reduce (rank order) of `count` doubles; one thread.
__global__ void dist_allreduce_kernel(DistDev D, int phase, const double* __restrict__ in,
                                      double* __restrict__ out, int count) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const unsigned long long s = ld_volatile_u64(D.seq + phase);
  for (int q = 0; q < D.nranks; ++q)
    for (int c = 0; c < count; ++c)
      D.pmbox[q][mbox_index(phase, (int)((s + 1) & 1), D.rank, c)] = in[c];
  dist_release(D, phase, s + 1);
  D.seq[phase] = s + 1;
  if (!dist_wait_all(D, phase, s + 1)) {
    *D.status = 1;
    for (int c = 0; c < count; ++c) out[c] = nan("");
    return;
  }
  for (int c = 0; c < count; ++c) out[c] = mbox_sum(D, phase, (int)((s + 1) & 1), c);
}

// The distributed scalar step of one iteration (krylov.cpp:51-57, 70-84 with
// rank-order sums): computed at the start of the next K1 by thread 0 of EVERY
// CTA from the same mailboxes, so every CTA (and every rank) holds identical
// values; written to the scalars by the last CTA of that K1 (or, when the
// solve ends there, by block 0).
struct DistStep {
  double beta, rz, rr, rel, relp, alpha_prev;
  int it_before, it, done, converged, status, pending;
};
__device__ __forceinline__ DistStep& dist_step_smem() {
  __shared__ DistStep st;
  return st;
}

__device__ __forceinline__ void dist_step_commit(CgScalars* __restrict__ sc, const DistStep& o) {
  if (o.status) {
    sc->status = o.status;
    if (o.status == 6) sc->err_it = o.it_before;
    sc->done = 1;
  } else {
    if (sc->hist && o.it_before + 1 < sc->hist_cap) sc->hist[o.it_before + 1] = o.rel;
    sc->it = o.it;
    sc->beta = o.beta;
    sc->rz = o.rz;
    sc->rr = o.rr;
    sc->alpha_prev = o.alpha_prev;
    sc->first = 0;
    sc->rel = o.rel;
    sc->relp = o.relp;
    if (o.converged) sc->converged = 1;
    if (o.done) sc->done = 1;
  }
  sc->xpend = 0;
}

// Start of a distributed K1 (all threads call it): when the update kernel
// left r'z / r'r partials (sc->xpend), publish this rank's (block 0: phase-1
// mailboxes + release), wait for every peer's, sum in rank order and take the
// scalar step.  Returns 0: no step pending (first iteration), 1: stepped,
// iterate; 2: the solve is finished.  Nothing here writes the scalars: every
// CTA reads them at its start, so they change only in the last CTA of the
// kernel (its ticket follows every CTA's head), which records the step --
// also when the solve is finished and the CTAs skip the iteration; the
// update kernel that follows then sees done and ends the graph loop.
__device__ int k1_dist_head(const DistDev& D, CgScalars* __restrict__ sc) {
  __shared__ int res;
  DistStep& st = dist_step_smem();
  if (threadIdx.x == 0) {
    int r = 0;
    st.pending = 0;
    if (sc->xpend) {
      DistStep o{};
      o.it_before = o.it = sc->it;
      const unsigned long long s = ld_volatile_u64(D.seq + 1);
      const int par = (int)(s & 1);
      const double rz_loc = sc->rz_loc, rr_loc = sc->rr_loc;
      const bool lead = blockIdx.x == 0 && blockIdx.y == 0;
      if (lead) {
        for (int q = 0; q < D.nranks; ++q) {
          if (q == D.rank) continue;
          D.pmbox[q][mbox_index(1, par, D.rank, 0)] = rz_loc;
          D.pmbox[q][mbox_index(1, par, D.rank, 1)] = rr_loc;
        }
        dist_release(D, 1, s);
      }
      if (!dist_wait_all(D, 1, s)) {
        o.status = 8;
        o.done = 1;
        if (lead) *D.status = 1;
      } else {
        if (lead) trace_stamp(&D, o.it_before + 1, 6);
        double rz_new = 0.0, rr_new = 0.0;
        for (int q = 0; q < D.nranks; ++q) {
          const volatile double* m = D.mbox + mbox_index(1, par, q, 0);
          rz_new += q == D.rank ? rz_loc : m[0];
        }
        for (int q = 0; q < D.nranks; ++q) {
          const volatile double* m = D.mbox + mbox_index(1, par, q, 1);
          rr_new += q == D.rank ? rr_loc : m[0];
        }
        const double rnorm = sqrt(rr_new);
        if (!isfinite(rnorm) || !isfinite(rz_new)) {
          o.status = 6;
          o.done = 1;
        } else {
          o.rel = rnorm / sc->bnorm;
          o.it = o.it_before + 1;
          o.beta = rz_new / sc->rz;
          o.rz = rz_new;
          o.rr = rr_new;
          o.alpha_prev = sc->alpha;
          o.relp = sc->bmb > 0.0 ? sqrt(fmax(rz_new, 0.0) / sc->bmb) : 0.0;
          if (o.rel <= sc->tol && o.relp <= sc->tol) {
            o.converged = 1;
            o.done = 1;
          } else if (o.it >= sc->max_it) {
            o.done = 1;
          }
        }
      }
      o.pending = 1;
      st = o;
      r = o.done ? 2 : 1;
    }
    res = r;
  }
  __syncthreads();
  return res;
}

// Sends of one element-step from the Ax epilogue: the group's threads store
// the interface values of its element(s) straight into the neighbours'
// receive buffers (phase 0, slot 0) over NVLink.  Called by every thread of a
// consumer group; group-uniform control flow.  Returns whether this thread
// stored anything.
__device__ __forceinline__ bool dist_send_elements(const DistDev* __restrict__ D, int par,
                                                   const double* __restrict__ w, int64_t e0,
                                                   int cnt, int n3, int lt, int tg) {
  // (each storing thread fences at system scope once, at the end of K1,
  // before the last-CTA ticket; released by dist_release_phase0)
  bool stored = false;
  for (int el = 0; el < cnt; ++el) {
    const int64_t e = e0 + el;
    const int lo = D->esend_off[e], hi = D->esend_off[e + 1];
    for (int c = lo + lt; c < hi; c += tg) {
      const int q = D->nbr[D->esend_q[c]];
      D->precv[q][(int64_t)par * D->precv_total[q] + D->pbase_for_me[q] + D->esend_pos[c]] =
          w[e * n3 + D->esend_node[c]];
      stored = true;
    }
  }
  return stored;
}


}  // namespace
}  // namespace sbx
