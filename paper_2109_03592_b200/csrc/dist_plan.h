// Host-side exchange plan of the distributed gather-scatter (one rank's view).
//
// Elements of a structured box are partitioned by partition_rcb (mesh.cpp:
// 168-226); a rank keeps its elements in ascending global order.  A lattice
// node whose copies live on several ranks forms an "interface group"; every
// rank owning a copy sums ALL copies in the reference's canonical order
// (ascending global (element, local index)), taking remote copies from a
// receive buffer, so every copy on every rank gets the bits the
// single-process gs_sum_inplace (gather.cpp:85-98) would produce.
// Exchanged values are raw copy values (not partial sums), neighbour-major,
// groups ascending by gid, copies in canonical order -- both sides derive the
// same layout from the global lattice without communication.
#pragma once

#include <cstdint>
#include <vector>

namespace sbx {

struct DistPlan {
  int nranks = 1, rank = 0;
  int ex = 0, ey = 0, ez = 0, degree = 0, n = 0;
  int per[3] = {0, 0, 0};
  int64_t E = 0;                        // global elements
  std::vector<int64_t> loc_elems;       // global ids of this rank's elements, ascending
  std::vector<int32_t> g2l;             // global element -> local id or -1
  // non-interface groups that contain element-boundary or masked nodes (the
  // local part of the boundary CSR); copies in canonical order, ~a = masked
  std::vector<int32_t> b_off, b_idx;
  // interface groups, ascending gid; codes: local node a (>= 0) or ~a when
  // masked; remote copy: nodes_local + position in the receive buffer
  std::vector<int64_t> if_gid;
  std::vector<int32_t> if_off, if_code;
  // neighbours (ascending rank) and per-neighbour send lists / receive counts
  std::vector<int> nbr;
  std::vector<std::vector<int32_t>> send_idx;
  std::vector<int64_t> recv_count, recv_base;  // recv_base: offset of nbr q's block
  int64_t recv_total = 0;
  // the same sends regrouped by local element (for sending from the Ax
  // epilogue): per entry the node within the element, the neighbour index and
  // the position inside that neighbour's block
  std::vector<int32_t> esend_off, esend_node, esend_q, esend_pos;
  // 27-neighbourhood of every local element: local id, -1 outside the
  // domain, -2 on another rank ((dx+1) + 3(dy+1) + 9(dz+1))
  std::vector<int32_t> nbr27;
  std::vector<double> inv_mult;         // 1/global multiplicity per local node
  std::vector<double> mask;             // Dirichlet mask per local node
  int64_t nodes_local() const { return (int64_t)loc_elems.size() * n * n * n; }
};

// Build rank `rank`'s plan.  Returns SBX_OK or an sbx_status error code.
int build_dist_plan(int ex, int ey, int ez, const int* periodic, int degree,
                    const int32_t* rank_of, int nranks, int rank, DistPlan& plan);

}  // namespace sbx
