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

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
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
// thread then releases a flag with st.release.sys, whose cumulativity orders
// every write it has observed -- including its own stores into peer mailboxes
// -- before the flag.  Readers acquire the flag with ld.acquire.sys.
__device__ __forceinline__ void dist_fence() { __threadfence(); }

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

// SBX_TRACE stamp: slot c of iteration it (one thread calls it)
__device__ __forceinline__ void trace_stamp(const DistDev* D, int it, int c) {
  if (D && D->trace) D->trace[(it % kTraceIters) * 8 + c] = globaltimer();
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
  for (int q = 0; q < D.nranks; ++q)
    if (q != D.rank) st_release_sys(D.pflags[q] + phase * kMaxRanks + D.rank, s + 1);
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

// Interface groups: wait for the halo, sum every copy in canonical order
// (local copies from f, remote ones from the receive buffer) and write the sum
// to the local copies (s*0 for masked ones when apply_mask).  In the CG loop
// (sc != null) block 0 also forms alpha = rz / sum_q pq_q and tests breakdown.
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
  const int64_t par = (int64_t)(ld_volatile_u64(D.seq + phase) & 1);
  // remote copies were pushed into this rank's receive buffer
  const double* rb = D.recvb + (int64_t)(slot * 2 + par) * D.recv_total;
  const int64_t NL = D.nodes_local;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < D.n_if;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int lo = D.if_off[g], hi = D.if_off[g + 1];
    double sum = 0.0;
    for (int c = lo; c < hi; ++c) {
      const int32_t code = D.if_code[c];
      double v;
      if (code >= NL) {
        v = __ldcv(rb + (code - NL));
      } else {
        v = f[code < 0 ? ~code : code];
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

// Scalar all-reduce (rank order) of `count` doubles; one thread.
__global__ void dist_allreduce_kernel(DistDev D, int phase, const double* __restrict__ in,
                                      double* __restrict__ out, int count) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const unsigned long long s = ld_volatile_u64(D.seq + phase);
  for (int q = 0; q < D.nranks; ++q)
    for (int c = 0; c < count; ++c)
      D.pmbox[q][mbox_index(phase, (int)((s + 1) & 1), D.rank, c)] = in[c];
  for (int q = 0; q < D.nranks; ++q)
    if (q != D.rank) st_release_sys(D.pflags[q] + phase * kMaxRanks + D.rank, s + 1);
  D.seq[phase] = s + 1;
  if (!dist_wait_all(D, phase, s + 1)) {
    *D.status = 1;
    for (int c = 0; c < count; ++c) out[c] = nan("");
    return;
  }
  for (int c = 0; c < count; ++c) out[c] = mbox_sum(D, phase, (int)((s + 1) & 1), c);
}

// End of a distributed CG iteration, run by ONE thread (the last CTA of the
// update kernel): all-reduce r'z, r'r (phase 1) through the mailboxes, then
// the scalar logic of update_tail (beta, history, convergence, NaN) and the
// WHILE condition.
__device__ void dist_scalar_step(const DistDev& D, CgScalars* __restrict__ sc, double rz_loc,
                                 double rr_loc, double* __restrict__ hist, int64_t hist_cap,
                                 cudaGraphConditionalHandle cond, int use_cond) {
  const int phase = 1;
  const unsigned long long s = ld_volatile_u64(D.seq + phase);
  const double mine[2] = {rz_loc, rr_loc};
  trace_stamp(&D, sc->it, 5);
  for (int q = 0; q < D.nranks; ++q)
    for (int c = 0; c < 2; ++c)
      D.pmbox[q][mbox_index(phase, (int)((s + 1) & 1), D.rank, c)] = mine[c];
  for (int q = 0; q < D.nranks; ++q)
    if (q != D.rank) st_release_sys(D.pflags[q] + phase * kMaxRanks + D.rank, s + 1);
  D.seq[phase] = s + 1;
  if (!dist_wait_all(D, phase, s + 1)) {
    *D.status = 1;
    sc->status = 8;
    sc->done = 1;
    if (use_cond) cudaGraphSetConditional(cond, 0);
    return;
  }
  trace_stamp(&D, sc->it, 6);
  const double rz_new = mbox_sum(D, phase, (int)((s + 1) & 1), 0);
  const double rr_new = mbox_sum(D, phase, (int)((s + 1) & 1), 1);
  const double rnorm = sqrt(rr_new);
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
    sc->rr = rr_new;
    sc->alpha_prev = sc->alpha;
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

// Release of phase 0 by the last CTA of K1 (one thread): this rank's p'Ap
// partial into every rank's mailbox, then the flags.
__device__ void dist_release_phase0(const DistDev& D, double pq_loc) {
  const unsigned long long s = ld_volatile_u64(D.seq);
  const int par = (int)((s + 1) & 1);
  for (int q = 0; q < D.nranks; ++q) D.pmbox[q][mbox_index(0, par, D.rank, 0)] = pq_loc;
  for (int q = 0; q < D.nranks; ++q)
    if (q != D.rank) st_release_sys(D.pflags[q] + D.rank, s + 1);
  D.seq[0] = s + 1;
}

}  // namespace
}  // namespace sbx
