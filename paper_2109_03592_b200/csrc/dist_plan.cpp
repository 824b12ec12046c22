// Exchange plan of the distributed gather-scatter (see dist_plan.h).
#include "dist_plan.h"

#include <algorithm>
#include <map>

#include "lattice.h"
#include "sbx_internal.h"

namespace sbx {

namespace {
struct IfaceGroup {
  int64_t gid;
  int m;
  int64_t elem[8];
  int lidx[8];
  int owner[8];
  bool masked;
};
}  // namespace

int build_dist_plan(int ex, int ey, int ez, const int* periodic, int degree,
                    const int32_t* rank_of, int nranks, int rank, DistPlan& P) {
  if (degree < 1 || degree > kMaxDegree) {
    set_error("dist plan: degree must be in [1,32]");
    return SBX_E_CONFIG;
  }
  if (nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("dist plan: bad rank / rank count");
    return SBX_E_CONFIG;
  }
  Lattice L;
  L.init(ex, ey, ez, periodic, degree);
  const int n = degree + 1, N = degree;
  const int64_t n3 = (int64_t)n * n * n;
  const int64_t E = (int64_t)ex * ey * ez;
  P = DistPlan();
  P.nranks = nranks;
  P.rank = rank;
  P.ex = ex;
  P.ey = ey;
  P.ez = ez;
  P.degree = degree;
  P.n = n;
  for (int d = 0; d < 3; ++d) P.per[d] = periodic[d] ? 1 : 0;
  P.E = E;
  P.g2l.assign(E, -1);
  for (int64_t e = 0; e < E; ++e) {
    if (rank_of[e] < 0 || rank_of[e] >= nranks) {
      set_error("dist plan: rank_of entry out of range");
      return SBX_E_CONFIG;
    }
    if (rank_of[e] == rank) {
      P.g2l[e] = (int32_t)P.loc_elems.size();
      P.loc_elems.push_back(e);
    }
  }
  if (P.loc_elems.empty()) {
    set_error("dist plan: rank owns no elements");
    return SBX_E_CONFIG;
  }
  const int64_t NL = P.nodes_local();
  if (NL >= (int64_t)INT32_MAX - 1) {
    set_error("dist plan: more than 2^31 local nodes");
    return SBX_E_SHAPE;
  }
  P.inv_mult.assign(NL, 1.0);
  P.mask.assign(NL, 1.0);
  const int counts[3] = {ex, ey, ez};
  std::vector<IfaceGroup> iface;
  P.b_off.push_back(0);
  for (size_t le = 0; le < P.loc_elems.size(); ++le) {
    const int64_t e = P.loc_elems[le];
    const int64_t cell[3] = {e % ex, (e / ex) % ey, e / ((int64_t)ex * ey)};
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
          const int loc[3] = {i, j, k};
          const bool bnd = i == 0 || j == 0 || k == 0 || i == N || j == N || k == N;
          if (!bnd) continue;  // element interior: unmasked singleton
          const int64_t a = (int64_t)le * n3 + (k * n + j) * n + i;
          int64_t g[3];
          bool masked = false;
          for (int d = 0; d < 3; ++d) {
            g[d] = L.coord(d, cell[d], loc[d]);
            if (!L.per[d] && (g[d] == 0 || g[d] == (int64_t)counts[d] * N)) masked = true;
          }
          int64_t celem[8];
          int clid[8];
          const int m = L.copies(g[0], g[1], g[2], celem, clid);
          P.inv_mult[a] = 1.0 / (double)m;
          P.mask[a] = masked ? 0.0 : 1.0;
          bool remote = false;
          int first_local = -1;
          for (int c = 0; c < m; ++c) {
            const bool mine = rank_of[celem[c]] == rank;
            if (!mine) remote = true;
            if (mine && first_local < 0) first_local = c;
          }
          // emit the group once, from its first local copy
          const int l = (k * n + j) * n + i;
          if (!(celem[first_local] == e && clid[first_local] == l)) continue;
          if (!remote) {
            for (int c = 0; c < m; ++c) {
              const int32_t la = (int32_t)(P.g2l[celem[c]] * n3 + clid[c]);
              P.b_idx.push_back(masked ? ~la : la);
            }
            P.b_off.push_back((int32_t)P.b_idx.size());
          } else {
            IfaceGroup G;
            G.gid = g[0] + L.gdim[0] * (g[1] + L.gdim[1] * g[2]);
            G.m = m;
            G.masked = masked;
            for (int c = 0; c < m; ++c) {
              G.elem[c] = celem[c];
              G.lidx[c] = clid[c];
              G.owner[c] = rank_of[celem[c]];
            }
            iface.push_back(G);
          }
        }
  }
  std::sort(iface.begin(), iface.end(),
            [](const IfaceGroup& a, const IfaceGroup& b) { return a.gid < b.gid; });
  // neighbours
  std::vector<char> isn(nranks, 0);
  for (const auto& G : iface)
    for (int c = 0; c < G.m; ++c)
      if (G.owner[c] != rank) isn[G.owner[c]] = 1;
  std::vector<int> qidx(nranks, -1);
  for (int q = 0; q < nranks; ++q)
    if (isn[q]) {
      qidx[q] = (int)P.nbr.size();
      P.nbr.push_back(q);
    }
  const size_t NQ = P.nbr.size();
  P.send_idx.assign(NQ, {});
  P.recv_count.assign(NQ, 0);
  // receive positions: for each neighbour, its copies of the shared groups in
  // (gid, canonical copy) order
  std::vector<std::vector<int64_t>> pos(iface.size());
  for (size_t gi = 0; gi < iface.size(); ++gi) pos[gi].assign(iface[gi].m, -1);
  for (size_t qi = 0; qi < NQ; ++qi) {
    const int q = P.nbr[qi];
    for (size_t gi = 0; gi < iface.size(); ++gi) {
      const IfaceGroup& G = iface[gi];
      bool shares = false;
      for (int c = 0; c < G.m; ++c)
        if (G.owner[c] == q) shares = true;
      if (!shares) continue;
      for (int c = 0; c < G.m; ++c) {
        if (G.owner[c] == rank)
          P.send_idx[qi].push_back((int32_t)(P.g2l[G.elem[c]] * n3 + G.lidx[c]));
        else if (G.owner[c] == q)
          pos[gi][c] = P.recv_count[qi]++;
      }
    }
  }
  {
    // regroup the send lists by local element
    const size_t EL = P.loc_elems.size();
    std::vector<int32_t> cnt(EL + 1, 0);
    for (size_t qi = 0; qi < NQ; ++qi)
      for (int32_t a : P.send_idx[qi]) ++cnt[a / n3 + 1];
    for (size_t e = 0; e < EL; ++e) cnt[e + 1] += cnt[e];
    P.esend_off = cnt;
    const size_t tot = (size_t)cnt[EL];
    P.esend_node.assign(tot, 0);
    P.esend_q.assign(tot, 0);
    P.esend_pos.assign(tot, 0);
    std::vector<int32_t> fill(cnt.begin(), cnt.end() - 1);
    for (size_t qi = 0; qi < NQ; ++qi)
      for (size_t i = 0; i < P.send_idx[qi].size(); ++i) {
        const int32_t a = P.send_idx[qi][i];
        const int32_t slot = fill[a / n3]++;
        P.esend_node[slot] = (int32_t)(a % n3);
        P.esend_q[slot] = (int32_t)qi;
        P.esend_pos[slot] = (int32_t)i;
      }
  }
  P.recv_base.assign(NQ, 0);
  for (size_t qi = 1; qi < NQ; ++qi) P.recv_base[qi] = P.recv_base[qi - 1] + P.recv_count[qi - 1];
  P.recv_total = NQ ? P.recv_base[NQ - 1] + P.recv_count[NQ - 1] : 0;
  P.if_off.push_back(0);
  for (size_t gi = 0; gi < iface.size(); ++gi) {
    const IfaceGroup& G = iface[gi];
    P.if_gid.push_back(G.gid);
    for (int c = 0; c < G.m; ++c) {
      if (G.owner[c] == rank) {
        const int32_t la = (int32_t)(P.g2l[G.elem[c]] * n3 + G.lidx[c]);
        P.if_code.push_back(G.masked ? ~la : la);
      } else {
        P.if_code.push_back((int32_t)(NL + P.recv_base[qidx[G.owner[c]]] + pos[gi][c]));
      }
    }
    P.if_off.push_back((int32_t)P.if_code.size());
  }
  // 27-neighbourhood
  P.nbr27.assign(P.loc_elems.size() * 27, -1);
  for (size_t le = 0; le < P.loc_elems.size(); ++le) {
    const int64_t e = P.loc_elems[le];
    const int64_t cell[3] = {e % ex, (e / ex) % ey, e / ((int64_t)ex * ey)};
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int dd[3] = {dx, dy, dz};
          int64_t c2[3];
          bool inside = true;
          for (int d = 0; d < 3; ++d) {
            c2[d] = cell[d] + dd[d];
            if (c2[d] < 0 || c2[d] >= counts[d]) {
              if (L.per[d])
                c2[d] = (c2[d] + counts[d]) % counts[d];
              else
                inside = false;
            }
          }
          int32_t code = -1;
          if (inside) {
            const int64_t g = c2[0] + ex * (c2[1] + (int64_t)ey * c2[2]);
            code = P.g2l[g] >= 0 ? P.g2l[g] : -2;
          }
          P.nbr27[le * 27 + (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1)] = code;
        }
  }
  return SBX_OK;
}

}  // namespace sbx
