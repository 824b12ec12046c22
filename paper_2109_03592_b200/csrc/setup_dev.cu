// Device-side setup of a structured-box context: the
// geometric factors, the Dirichlet mask, the multiplicities, and the
// gather-scatter over the node lattice, built on the GPU instead of on the
// host and uploaded.
//
// * geom_box_kernel: one thread per node, the node metric of the element's
//   trilinear map (metric.h, shared with the host builder; this file is
//   compiled with -fmad=false so every operation rounds as in the reference,
//   operators.cpp:123-178) written straight into the packed [E][6][n^3]
//   layout the kernels stream, plus bm; the first element with detJ <= 0 is
//   reported like the host builder's MeshError.
// * lattice_fields_kernel: mask (operators.cpp:433-455), inv_mult and the
//   clamped multiplicity per node from the lattice coordinates
//   (gather.cpp:15-46 read backwards, lattice.h).
// * gs_box_kernel: gs_sum_inplace (gather.cpp:85-98) without a CSR: the
//   thread of a group's FIRST copy (ascending local index) sums the copies
//   from 0.0 in the reference order and writes every copy; bitwise equal to
//   the CSR gs_kernel.  Masked copies get s*0.0 when the mask is applied.
// * check_rhs_box_kernel: the fused CG's continuity / mask precondition on
//   the right-hand side, per node against its partner copies.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "lattice.h"
#include "metric.h"

namespace sbx {

namespace {

struct GllParam {
  double x[33];
  double w[33];
};

__global__ void geom_box_kernel(const double* __restrict__ corners, int64_t E, int n,
                                GllParam q, double* __restrict__ G, double* __restrict__ bm,
                                unsigned long long* __restrict__ bad) {
  const int n3 = n * n * n;
  const int64_t nodes = E * n3;
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < nodes;
       a += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = a / n3;
    const int l = (int)(a - e * n3);
    const int i = l % n, j = (l / n) % n, k = l / (n * n);
    double cr[24];
#pragma unroll
    for (int c = 0; c < 24; ++c) cr[c] = __ldg(corners + e * 24 + c);
    Metric m;
    const double wq = q.w[i] * q.w[j] * q.w[k];
    if (!node_metric(cr, q.x[i], q.x[j], q.x[k], wq, m)) {
      atomicMin(bad, (unsigned long long)e);
      continue;
    }
    double* Ge = G + e * 6 * (int64_t)n3 + l;
#pragma unroll
    for (int c = 0; c < 6; ++c) Ge[c * n3] = m.g[c];
    if (bm) bm[a] = m.wdet;
  }
}

struct BoxLat {
  int ex, ey, ez;
  int per[3];
  int N;
};

__device__ __forceinline__ Lattice make_lattice(const BoxLat& b) {
  Lattice L;
  const int p[3] = {b.per[0], b.per[1], b.per[2]};
  L.init(b.ex, b.ey, b.ez, p, b.N);
  return L;
}

// lattice coordinates of local node a
__device__ __forceinline__ void node_coords(const Lattice& L, const BoxLat& b, int64_t a,
                                            int64_t g[3], bool& boundary) {
  const int n = b.N + 1, n3 = n * n * n;
  const int64_t e = a / n3;
  const int l = (int)(a - e * n3);
  const int loc[3] = {l % n, (l / n) % n, l / (n * n)};
  const int64_t cell[3] = {e % b.ex, (e / b.ex) % b.ey, e / ((int64_t)b.ex * b.ey)};
  boundary = false;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    g[d] = L.coord(d, cell[d], loc[d]);
    if (loc[d] == 0 || loc[d] == b.N) boundary = true;
  }
}

__device__ __forceinline__ bool lattice_masked(const Lattice& L, const int64_t g[3]) {
  bool m = false;
#pragma unroll
  for (int d = 0; d < 3; ++d)
    if (!L.per[d] && (g[d] == 0 || g[d] == (int64_t)L.counts[d] * L.N)) m = true;
  return m;
}

__global__ void lattice_fields_kernel(BoxLat b, int64_t nodes, double* __restrict__ mask,
                                      double* __restrict__ inv_mult,
                                      uint8_t* __restrict__ mult8) {
  const Lattice L = make_lattice(b);
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < nodes;
       a += (int64_t)gridDim.x * blockDim.x) {
    int64_t g[3];
    bool boundary;
    node_coords(L, b, a, g, boundary);
    int m = 1;
#pragma unroll
    for (int d = 0; d < 3; ++d) m *= L.opts(d, g[d]).count;
    if (mask) mask[a] = lattice_masked(L, g) ? 0.0 : 1.0;
    if (inv_mult) inv_mult[a] = 1.0 / (double)m;
    if (mult8) mult8[a] = (uint8_t)m;
  }
}

// ---- per-solve lattice kernels: 32-bit, one thread per element column -----
// (thread = (element e, column (i, j)); only the column's element-boundary
// nodes do work: all k when i or j is on a face, else k = 0 and k = N)

// copies of one lattice direction (32-bit Lattice::opts)
struct Ax32 {
  int cnt;
  int cell[2];
  int loc[2];
};

__device__ __forceinline__ Ax32 axis32(int g, int count, int N, bool per) {
  Ax32 o;
  const int q = g / N, r = g - q * N;
  if (r != 0) {
    o.cnt = 1;
    o.cell[0] = q;
    o.loc[0] = r;
    return o;
  }
  o.cnt = 0;
  if (per) {
    o.cell[0] = q;
    o.loc[0] = 0;
    o.cell[1] = (q - 1 + count) % count;
    o.loc[1] = N;
    o.cnt = 2;
  } else {
    if (g > 0) {
      o.cell[o.cnt] = q - 1;
      o.loc[o.cnt++] = N;
    }
    if (q < count) {
      o.cell[o.cnt] = q;
      o.loc[o.cnt++] = 0;
    }
  }
  return o;
}

struct Col32 {
  int e, i, j, cx, cy, cz;
};

__device__ __forceinline__ Col32 col_of(const BoxLat& b, int n, int col) {
  Col32 c;
  const int nn = n * n;
  c.e = col / nn;
  const int ij = col - c.e * nn;
  c.j = ij / n;
  c.i = ij - c.j * n;
  const int exy = b.ex * b.ey;
  c.cz = c.e / exy;
  const int rxy = c.e - c.cz * exy;
  c.cy = rxy / b.ex;
  c.cx = rxy - c.cy * b.ex;
  return c;
}

// lattice coordinate along d of local index loc in cell c (periodic wrap)
__device__ __forceinline__ int gcoord(int c, int loc, int count, int N, bool per) {
  const int g = c * N + loc;
  return (per && g == count * N) ? 0 : g;
}

// All copies of node (col, k) in ascending local index (the reference's
// group order): returns the count; idx[] = e * n^3 + local index.
__device__ __forceinline__ int copies32(const BoxLat& b, int n, const Col32& c, int k,
                                        int (&idx)[8], bool& masked) {
  const int N = n - 1, n3 = n * n * n;
  const int gx = gcoord(c.cx, c.i, b.ex, N, b.per[0]);
  const int gy = gcoord(c.cy, c.j, b.ey, N, b.per[1]);
  const int gz = gcoord(c.cz, k, b.ez, N, b.per[2]);
  masked = (!b.per[0] && (gx == 0 || gx == b.ex * N)) ||
           (!b.per[1] && (gy == 0 || gy == b.ey * N)) ||
           (!b.per[2] && (gz == 0 || gz == b.ez * N));
  const Ax32 ox = axis32(gx, b.ex, N, b.per[0]);
  const Ax32 oy = axis32(gy, b.ey, N, b.per[1]);
  const Ax32 oz = axis32(gz, b.ez, N, b.per[2]);
  int m = 0;
  for (int z = 0; z < oz.cnt; ++z)
    for (int y = 0; y < oy.cnt; ++y)
      for (int x = 0; x < ox.cnt; ++x) {
        const int e = ox.cell[x] + b.ex * (oy.cell[y] + b.ey * oz.cell[z]);
        idx[m++] = e * n3 + (oz.loc[z] * n + oy.loc[y]) * n + ox.loc[x];
      }
  for (int x = 1; x < m; ++x)  // <= 8 copies; already sorted unless a periodic wrap
    for (int y = x; y > 0 && idx[y - 1] > idx[y]; --y) {
      const int t = idx[y - 1];
      idx[y - 1] = idx[y];
      idx[y] = t;
    }
  return m;
}

__global__ void gs_box_kernel(BoxLat b, int n, int cols, double* __restrict__ f,
                              int apply_mask) {
  const int N = n - 1, n3 = n * n * n;
  for (int col = blockIdx.x * blockDim.x + threadIdx.x; col < cols;
       col += gridDim.x * blockDim.x) {
    const Col32 c = col_of(b, n, col);
    const bool face = c.i == 0 || c.i == N || c.j == 0 || c.j == N;
    for (int k = 0; k < n; k += (face || k == N) ? 1 : N) {
      const int a = c.e * n3 + (k * n + c.j) * n + c.i;
      int idx[8];
      bool masked;
      const int m = copies32(b, n, c, k, idx, masked);
      masked = masked && apply_mask;
      if (m == 1) {
        if (masked) f[a] = __dmul_rn(f[a], 0.0);
        continue;
      }
      if (idx[0] != a) continue;  // the group's first copy does the work
      double sum = 0.0;
      for (int q = 0; q < m; ++q) sum = __dadd_rn(sum, f[idx[q]]);
      const double v = masked ? __dmul_rn(sum, 0.0) : sum;
      for (int q = 0; q < m; ++q) f[idx[q]] = v;
    }
  }
}

// gs_sum of three fields, then the pointwise scale (every node, the element
// interiors included): apply_pressure_operator's gradient step
// (stepper.cpp:242-245).  Reference copy order, as gs_box_kernel.
__global__ void gs3_scale_box_kernel(BoxLat b, int n, int cols, double* __restrict__ f0,
                                     double* __restrict__ f1, double* __restrict__ f2,
                                     const double* __restrict__ scale) {
  const int N = n - 1, n3 = n * n * n;
  for (int col = blockIdx.x * blockDim.x + threadIdx.x; col < cols;
       col += gridDim.x * blockDim.x) {
    const Col32 c = col_of(b, n, col);
    const bool face = c.i == 0 || c.i == N || c.j == 0 || c.j == N;
    for (int k = 0; k < n; ++k) {
      const int a = c.e * n3 + (k * n + c.j) * n + c.i;
      if (!face && k != 0 && k != N) {
        const double w = scale[a];
        f0[a] *= w;
        f1[a] *= w;
        f2[a] *= w;
        continue;
      }
      int idx[8];
      bool masked;
      const int m = copies32(b, n, c, k, idx, masked);
      if (idx[0] != a) continue;  // the group's first copy does the work
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      for (int q = 0; q < m; ++q) {
        s0 = __dadd_rn(s0, f0[idx[q]]);
        s1 = __dadd_rn(s1, f1[idx[q]]);
        s2 = __dadd_rn(s2, f2[idx[q]]);
      }
      for (int q = 0; q < m; ++q) {
        const double w = scale[idx[q]];
        f0[idx[q]] = __dmul_rn(s0, w);
        f1[idx[q]] = __dmul_rn(s1, w);
        f2[idx[q]] = __dmul_rn(s2, w);
      }
    }
  }
}

// Out of place: v_c = scale * gs_sum(g_c).  Every thread sums its own node's
// copies (the same copies in the same reference order for every copy, so
// every copy gets the same bits as the in-place kernel) -- no serial owner
// loop, the partner loads of all copies in flight at once.  The copies are the
// product of at most two options per axis; with each axis's options in
// ascending cell order, the (z, y, x) nesting visits them in ascending
// element index -- the reference's order -- with compile-time indices only
// (no local-memory index array, no sort).
__device__ __forceinline__ Ax32 axis32_sorted(int g, int count, int N, bool per) {
  Ax32 o = axis32(g, count, N, per);
  if (o.cnt == 2 && o.cell[1] < o.cell[0]) {
    const int c = o.cell[0], l = o.loc[0];
    o.cell[0] = o.cell[1];
    o.loc[0] = o.loc[1];
    o.cell[1] = c;
    o.loc[1] = l;
  }
  return o;
}

__global__ void gs3_scale_box_oop_kernel(BoxLat b, int n, int cols,
                                         const double* __restrict__ f0,
                                         const double* __restrict__ f1,
                                         const double* __restrict__ f2,
                                         const double* __restrict__ scale,
                                         double* __restrict__ v0, double* __restrict__ v1,
                                         double* __restrict__ v2) {
  const int N = n - 1, n3 = n * n * n;
  for (int col = blockIdx.x * blockDim.x + threadIdx.x; col < cols;
       col += gridDim.x * blockDim.x) {
    const Col32 c = col_of(b, n, col);
    const bool face = c.i == 0 || c.i == N || c.j == 0 || c.j == N;
    // the x / y options are the column's, the same for every k
    const Ax32 ox = axis32_sorted(gcoord(c.cx, c.i, b.ex, N, b.per[0]), b.ex, N, b.per[0]);
    const Ax32 oy = axis32_sorted(gcoord(c.cy, c.j, b.ey, N, b.per[1]), b.ey, N, b.per[1]);
    for (int k = 0; k < n; ++k) {
      const int a = c.e * n3 + (k * n + c.j) * n + c.i;
      const double w = scale[a];
      if (!face && k != 0 && k != N) {
        v0[a] = __dmul_rn(f0[a], w);
        v1[a] = __dmul_rn(f1[a], w);
        v2[a] = __dmul_rn(f2[a], w);
        continue;
      }
      const Ax32 oz = axis32_sorted(gcoord(c.cz, k, b.ez, N, b.per[2]), b.ez, N, b.per[2]);
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int z = 0; z < 2; ++z) {
#pragma unroll
        for (int y = 0; y < 2; ++y) {
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            if (z < oz.cnt && y < oy.cnt && x < ox.cnt) {
              const int e = ox.cell[x] + b.ex * (oy.cell[y] + b.ey * oz.cell[z]);
              const int q = e * n3 + (oz.loc[z] * n + oy.loc[y]) * n + ox.loc[x];
              s0 = __dadd_rn(s0, f0[q]);
              s1 = __dadd_rn(s1, f1[q]);
              s2 = __dadd_rn(s2, f2[q]);
            }
          }
        }
      }
      if (ox.cnt * oy.cnt * oz.cnt == 1) {  // a singleton: gs leaves it alone (no 0.0 + x)
        s0 = f0[a];
        s1 = f1[a];
        s2 = f2[a];
      }
      v0[a] = __dmul_rn(s0, w);
      v1[a] = __dmul_rn(s1, w);
      v2[a] = __dmul_rn(s2, w);
    }
  }
}

__global__ void mul3_kernel(int64_t N, double* __restrict__ f0, double* __restrict__ f1,
                            double* __restrict__ f2, const double* __restrict__ scale) {
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < N;
       a += (int64_t)gridDim.x * blockDim.x) {
    const double w = scale[a];
    f0[a] = __dmul_rn(f0[a], w);
    f1[a] = __dmul_rn(f1[a], w);
    f2[a] = __dmul_rn(f2[a], w);
  }
}

// Continuity: every copy equals its face neighbours' copies (the copies of a
// node are connected by face steps, so pairwise face equality is equality of
// all copies); masked copies are zero.
__global__ void check_rhs_box_kernel(BoxLat b, int n, int cols, const double* __restrict__ f,
                                     int* flag) {
  const int N = n - 1, n3 = n * n * n;
  bool bad = false;
  for (int col = blockIdx.x * blockDim.x + threadIdx.x; col < cols;
       col += gridDim.x * blockDim.x) {
    const Col32 c = col_of(b, n, col);
    const bool face = c.i == 0 || c.i == N || c.j == 0 || c.j == N;
    // partner across the +x / +y / +z face (loc == N), with the wrap
    const int ex1 = (c.cx + 1 < b.ex) ? 1 : (b.per[0] ? 1 - b.ex : 0);
    const int ey1 = (c.cy + 1 < b.ey) ? b.ex : (b.per[1] ? (1 - b.ey) * b.ex : 0);
    const int exy = b.ex * b.ey;
    const int ez1 = (c.cz + 1 < b.ez) ? exy : (b.per[2] ? (1 - b.ez) * exy : 0);
    const bool mx = !b.per[0] && ((c.cx == 0 && c.i == 0) || (c.cx == b.ex - 1 && c.i == N));
    const bool my = !b.per[1] && ((c.cy == 0 && c.j == 0) || (c.cy == b.ey - 1 && c.j == N));
    for (int k = 0; k < n; k += (face || k == N) ? 1 : N) {
      const int l = (k * n + c.j) * n + c.i;
      const double v = f[c.e * n3 + l];
      const bool mz = !b.per[2] && ((c.cz == 0 && k == 0) || (c.cz == b.ez - 1 && k == N));
      if ((mx || my || mz) && v != 0.0) bad = true;
      if (c.i == N && ex1 != 0 && f[(c.e + ex1) * n3 + l - N] != v) bad = true;
      if (c.j == N && ey1 != 0 && f[(c.e + ey1) * n3 + l - N * n] != v) bad = true;
      if (k == N && ez1 != 0 && f[(c.e + ez1) * n3 + l - N * n * n] != v) bad = true;
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
}

// The caller's map (group_offsets / group_nodes, gather.hpp:14-29) against
// the lattice: one thread per group (= lattice point, gid order).
__global__ void validate_map_kernel(BoxLat b, int64_t G, int64_t nodes,
                                    const int64_t* __restrict__ off,
                                    const int64_t* __restrict__ idx, int* flag) {
  const Lattice L = make_lattice(b);
  const int n = b.N + 1;
  const int64_t n3 = (int64_t)n * n * n;
  bool bad = false;
  for (int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < G;
       gid += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g0 = gid % L.gdim[0], g1 = (gid / L.gdim[0]) % L.gdim[1],
                  g2 = gid / (L.gdim[0] * L.gdim[1]);
    int64_t el[8];
    int li[8];
    const int m = L.copies(g0, g1, g2, el, li);
    const int64_t lo = off[gid], hi = off[gid + 1];
    if (hi - lo != m || lo < 0 || hi > nodes) {
      bad = true;
      continue;
    }
    for (int c = 0; c < m; ++c)
      if (idx[lo + c] != el[c] * n3 + li[c]) bad = true;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
}

__global__ void validate_mask_kernel(BoxLat b, int64_t nodes, const double* __restrict__ mask,
                                     int* flag) {
  const Lattice L = make_lattice(b);
  bool bad = false;
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < nodes;
       a += (int64_t)gridDim.x * blockDim.x) {
    int64_t g[3];
    bool boundary;
    node_coords(L, b, a, g, boundary);
    const double want = lattice_masked(L, g) ? 0.0 : 1.0;
    // bitwise (-0.0 is not the reference's 0.0)
    if (__double_as_longlong(mask[a]) != __double_as_longlong(want)) bad = true;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
}

// The caller's packed geometry against the corners' trilinear metric, bitwise.
__global__ void validate_geom_kernel(const double* __restrict__ corners, int64_t E, int n,
                                     GllParam q, const double* __restrict__ G,
                                     const double* __restrict__ bm, int* flag) {
  const int n3 = n * n * n;
  const int64_t nodes = E * n3;
  bool bad = false;
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < nodes;
       a += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = a / n3;
    const int l = (int)(a - e * n3);
    const int i = l % n, j = (l / n) % n, k = l / (n * n);
    double cr[24];
#pragma unroll
    for (int c = 0; c < 24; ++c) cr[c] = __ldg(corners + e * 24 + c);
    Metric m;
    const double wq = q.w[i] * q.w[j] * q.w[k];
    if (!node_metric(cr, q.x[i], q.x[j], q.x[k], wq, m)) {
      bad = true;
      continue;
    }
    const double* Ge = G + e * 6 * (int64_t)n3 + l;
#pragma unroll
    for (int c = 0; c < 6; ++c)
      if (__double_as_longlong(Ge[c * n3]) != __double_as_longlong(m.g[c])) bad = true;
    if (bm && __double_as_longlong(bm[a]) != __double_as_longlong(m.wdet)) bad = true;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
}

unsigned grid_for(int64_t work) {
  int64_t b = (work + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  if (b < 1) b = 1;
  return (unsigned)b;
}

BoxLat box_lat(const OpDev& op) {
  return BoxLat{op.ex, op.ey, op.ez, {op.per[0], op.per[1], op.per[2]}, op.n - 1};
}

}  // namespace

cudaError_t launch_geom_box(const double* corners, int64_t E, int n, const double* x,
                            const double* w, double* G, double* bm, unsigned long long* bad,
                            cudaStream_t s) {
  GllParam q{};
  for (int i = 0; i < n; ++i) {
    q.x[i] = x[i];
    q.w[i] = w[i];
  }
  geom_box_kernel<<<grid_for(E * n * n * n), 256, 0, s>>>(corners, E, n, q, G, bm, bad);
  return cudaGetLastError();
}

cudaError_t launch_lattice_fields(const OpDev& op, double* mask, double* inv_mult,
                                  uint8_t* mult8, cudaStream_t s) {
  lattice_fields_kernel<<<grid_for(op.nodes), 256, 0, s>>>(box_lat(op), op.nodes, mask,
                                                           inv_mult, mult8);
  return cudaGetLastError();
}

cudaError_t launch_gs_box(const OpDev& op, double* f, bool apply_mask, cudaStream_t s) {
  const int cols = (int)(op.E * op.n * op.n);
  gs_box_kernel<<<grid_for(cols), 256, 0, s>>>(box_lat(op), op.n, cols, f, apply_mask ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_check_rhs_box(const OpDev& op, const double* f, int* flag, cudaStream_t s) {
  const int cols = (int)(op.E * op.n * op.n);
  check_rhs_box_kernel<<<grid_for(cols), 256, 0, s>>>(box_lat(op), op.n, cols, f, flag);
  return cudaGetLastError();
}

cudaError_t launch_validate_box(const OpDev& op, int64_t G, const int64_t* offsets,
                                const int64_t* group_nodes, const double* mask, int* flag,
                                cudaStream_t s) {
  if (offsets && group_nodes)
    validate_map_kernel<<<grid_for(G), 256, 0, s>>>(box_lat(op), G, op.nodes, offsets,
                                                     group_nodes, flag);
  if (mask) validate_mask_kernel<<<grid_for(op.nodes), 256, 0, s>>>(box_lat(op), op.nodes, mask,
                                                                    flag);
  return cudaGetLastError();
}

cudaError_t launch_validate_geom(const double* corners, int64_t E, int n, const double* x,
                                 const double* w, const double* G, const double* bm, int* flag,
                                 cudaStream_t s) {
  GllParam q{};
  for (int i = 0; i < n; ++i) {
    q.x[i] = x[i];
    q.w[i] = w[i];
  }
  validate_geom_kernel<<<grid_for(E * n * n * n), 256, 0, s>>>(corners, E, n, q, G, bm, flag);
  return cudaGetLastError();
}

cudaError_t launch_gs3_scale(const OpDev& op, double* const g[3], const double* scale,
                             cudaStream_t s, double* const* out) {
  if (op.lat && out) {
    const int cols = (int)(op.E * op.n * op.n);
    gs3_scale_box_oop_kernel<<<grid_for(cols), 256, 0, s>>>(box_lat(op), op.n, cols, g[0], g[1],
                                                            g[2], scale, out[0], out[1], out[2]);
    return cudaGetLastError();
  }
  if (out) {
    for (int c = 0; c < 3; ++c) {
      const cudaError_t e = cudaMemcpyAsync(out[c], g[c], sizeof(double) * op.nodes,
                                            cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return e;
    }
    return launch_gs3_scale(op, out, scale, s, nullptr);
  }
  if (op.lat) {
    const int cols = (int)(op.E * op.n * op.n);
    gs3_scale_box_kernel<<<grid_for(cols), 256, 0, s>>>(box_lat(op), op.n, cols, g[0], g[1],
                                                        g[2], scale);
    return cudaGetLastError();
  }
  for (int c = 0; c < 3; ++c) {
    const cudaError_t e = launch_gs(op, g[c], false, s);
    if (e != cudaSuccess) return e;
  }
  mul3_kernel<<<grid_for(op.nodes), 256, 0, s>>>(op.nodes, g[0], g[1], g[2], scale);
  return cudaGetLastError();
}

}  // namespace sbx
