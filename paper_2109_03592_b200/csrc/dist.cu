// Multi-GPU (one process per GPU) context: placeholder until the NCCL
// exchange plan lands.
#include "sbx_internal.h"

extern "C" {
sbx_status sbx_comm_unique_id(uint8_t id[128]) {
  (void)id;
  sbx::set_error("multi-GPU support not built");
  return SBX_E_COMM;
}
sbx_status sbx_ctx_create_box_dist(const sbx_box_desc*, const int32_t*, int, int,
                                   const uint8_t[128], int, sbx_ctx** out) {
  *out = nullptr;
  sbx::set_error("multi-GPU support not built");
  return SBX_E_COMM;
}
}
