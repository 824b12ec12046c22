// Multi-GPU C ABI: exchange plan (host, testable without a GPU) and the
// distributed context (one process per GPU, peer windows over CUDA IPC).
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <vector>

#include "dist_plan.h"
#include "sbx_internal.h"

struct sbx_dist_plan {
  sbx::DistPlan p;
};

using namespace sbx;

extern "C" {

sbx_status sbx_dist_plan_create(const sbx_box_desc* d, const int32_t* rank_of, int nranks,
                                int rank, sbx_dist_plan** out) {
  if (!d || !rank_of || !out) {
    set_error("sbx_dist_plan_create: null argument");
    return SBX_E_INVALID;
  }
  *out = nullptr;
  auto* h = new sbx_dist_plan();
  const int rc = build_dist_plan(d->ex, d->ey, d->ez, d->periodic, d->degree, rank_of, nranks,
                                 rank, h->p);
  if (rc != SBX_OK) {
    delete h;
    return (sbx_status)rc;
  }
  *out = h;
  return SBX_OK;
}

void sbx_dist_plan_destroy(sbx_dist_plan* h) { delete h; }

sbx_status sbx_dist_plan_sizes(const sbx_dist_plan* h, int64_t* s) {
  if (!h || !s) return SBX_E_INVALID;
  const DistPlan& p = h->p;
  int64_t sends = 0;
  for (const auto& v : p.send_idx) sends += (int64_t)v.size();
  s[0] = (int64_t)p.loc_elems.size();
  s[1] = p.nodes_local();
  s[2] = (int64_t)p.b_off.size() - 1;
  s[3] = (int64_t)p.b_idx.size();
  s[4] = (int64_t)p.if_off.size() - 1;
  s[5] = (int64_t)p.if_code.size();
  s[6] = (int64_t)p.nbr.size();
  s[7] = p.recv_total;
  s[8] = sends;
  return SBX_OK;
}

// 0 loc_elems (i64) | 1 b_off, 2 b_idx, 3 if_off, 4 if_code, 5 nbr (i32) |
// 6 send counts (i64 per neighbour) | 7 send_idx concatenated (i32) |
// 8 recv_count, 9 recv_base (i64) | 10 nbr27 (i32) | 11 inv_mult, 12 mask (f64)
// | 13 if_gid (i64)
sbx_status sbx_dist_plan_array(const sbx_dist_plan* h, int which, void* out) {
  if (!h || !out) return SBX_E_INVALID;
  const DistPlan& p = h->p;
  auto cp = [&](const void* src, size_t bytes) {
    if (bytes) std::memcpy(out, src, bytes);
    return SBX_OK;
  };
  switch (which) {
    case 0: return cp(p.loc_elems.data(), p.loc_elems.size() * 8);
    case 1: return cp(p.b_off.data(), p.b_off.size() * 4);
    case 2: return cp(p.b_idx.data(), p.b_idx.size() * 4);
    case 3: return cp(p.if_off.data(), p.if_off.size() * 4);
    case 4: return cp(p.if_code.data(), p.if_code.size() * 4);
    case 5: return cp(p.nbr.data(), p.nbr.size() * 4);
    case 6: {
      auto* o = static_cast<int64_t*>(out);
      for (size_t q = 0; q < p.send_idx.size(); ++q) o[q] = (int64_t)p.send_idx[q].size();
      return SBX_OK;
    }
    case 7: {
      auto* o = static_cast<int32_t*>(out);
      for (const auto& v : p.send_idx) {
        if (!v.empty()) std::memcpy(o, v.data(), v.size() * 4);
        o += v.size();
      }
      return SBX_OK;
    }
    case 8: return cp(p.recv_count.data(), p.recv_count.size() * 8);
    case 9: return cp(p.recv_base.data(), p.recv_base.size() * 8);
    case 10: return cp(p.nbr27.data(), p.nbr27.size() * 4);
    case 11: return cp(p.inv_mult.data(), p.inv_mult.size() * 8);
    case 12: return cp(p.mask.data(), p.mask.size() * 8);
    case 13: return cp(p.if_gid.data(), p.if_gid.size() * 8);
    default:
      set_error("sbx_dist_plan_array: unknown array id");
      return SBX_E_INVALID;
  }
}

}  // extern "C"

// ---- distributed context: device side in dist_ctx.cu -----------------------
