// EXACT (reference evaluation order) pressure operators: bitwise equal to
// sembox's gradient_from_pressure / divergence_to_pressure (operators.cpp:
// 327-410 with interp3 / contract_dir / ref_derivatives, :60-121), the GL
// pressure geometry of build_pressure_geometry (:180-214, formed on the fly
// from the element corners with the same TrilinearMap / det3 / inv3
// expressions, metric.h) and pressure_operator_diagonal (stepper.cpp:250-275).
//
// Compiled with -fmad=false: every `s += a * b` rounds the product and the sum
// separately, as the reference (x86-64, no FMA contraction) does.  Each output
// entry is one thread's sequential sum in the reference's loop order, so the
// parallel schedule does not change a bit.  One CTA per element.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "metric.h"

namespace sbx {

namespace {

constexpr int kXThreads = 128;

struct ExactMats {
  const double* d;     // GLL derivative, n x n (d[i*n + l] = l_l'(x_i))
  const double* iv;    // interp_v2p, m x n
  const double* ivt;   // its transpose, n x m
  const double* glx;   // GL nodes [m]
  const double* glw;   // GL weights [m]
};

// wdetj and drdx[9] at GL node (i, j, k) of an element (operators.cpp:180-214)
__device__ __forceinline__ void pgeom(const double* cr, const ExactMats& M, int i, int j, int k,
                                      double& wdetj, double (&drdx)[9]) {
  const double r = M.glx[i], s = M.glx[j], t = M.glx[k];
  const double sh[3][2] = {{0.5 * (1 - r), 0.5 * (1 + r)},
                           {0.5 * (1 - s), 0.5 * (1 + s)},
                           {0.5 * (1 - t), 0.5 * (1 + t)}};
  double J[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int v = 0; v < 8; ++v) {
    const int b0 = v & 1, b1 = (v >> 1) & 1, b2 = (v >> 2) & 1;
    const double d0 = b0 ? 0.5 : -0.5, d1 = b1 ? 0.5 : -0.5, d2 = b2 ? 0.5 : -0.5;
    const double gr[3] = {d0 * sh[1][b1] * sh[2][b2], sh[0][b0] * d1 * sh[2][b2],
                          sh[0][b0] * sh[1][b1] * d2};
    for (int p = 0; p < 3; ++p) {
      const double xp = cr[v * 3 + p];
      J[p * 3 + 0] += xp * gr[0];
      J[p * 3 + 1] += xp * gr[1];
      J[p * 3 + 2] += xp * gr[2];
    }
  }
  const double det = J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
                     J[2] * (J[3] * J[7] - J[4] * J[6]);
  const double id = 1.0 / det;
  drdx[0] = (J[4] * J[8] - J[5] * J[7]) * id;
  drdx[1] = (J[2] * J[7] - J[1] * J[8]) * id;
  drdx[2] = (J[1] * J[5] - J[2] * J[4]) * id;
  drdx[3] = (J[5] * J[6] - J[3] * J[8]) * id;
  drdx[4] = (J[0] * J[8] - J[2] * J[6]) * id;
  drdx[5] = (J[2] * J[3] - J[0] * J[5]) * id;
  drdx[6] = (J[3] * J[7] - J[4] * J[6]) * id;
  drdx[7] = (J[1] * J[6] - J[0] * J[7]) * id;
  drdx[8] = (J[0] * J[4] - J[1] * J[3]) * id;
  wdetj = M.glw[i] * M.glw[j] * M.glw[k] * det;
}

// contract_dir (operators.cpp:80-110): one output entry, sequential sum
__device__ __forceinline__ double cdir(const double* in, const double* mat, int nb, int na,
                                      int dim0, int dim1, int dir, int idx) {
  double s = 0.0;
  if (dir == 0) {
    const int a = idx % nb, kj = idx / nb;  // out[(k*dim0 + j)*nb + a]
    for (int i = 0; i < na; ++i) s += mat[a * na + i] * in[kj * na + i];
  } else if (dir == 1) {
    const int i = idx % dim0, a = (idx / dim0) % nb, k = idx / (dim0 * nb);
    for (int j = 0; j < na; ++j) s += mat[a * na + j] * in[(k * na + j) * dim0 + i];
  } else {
    const int i = idx % dim0, j = (idx / dim0) % dim1, a = idx / (dim0 * dim1);
    for (int k = 0; k < na; ++k) s += mat[a * na + k] * in[(k * dim1 + j) * dim0 + i];
  }
  return s;
}

// interp3 (operators.cpp:112-121): in (na^3) -> out (nb^3), through t1, t2
__device__ void interp3_cta(const double* in, double* t1, double* t2, double* out,
                            const double* mat, int nb, int na) {
  for (int q = threadIdx.x; q < nb * na * na; q += blockDim.x)
    t1[q] = cdir(in, mat, nb, na, na, na, 0, q);
  __syncthreads();
  for (int q = threadIdx.x; q < nb * nb * na; q += blockDim.x)
    t2[q] = cdir(t1, mat, nb, na, nb, na, 1, q);
  __syncthreads();
  for (int q = threadIdx.x; q < nb * nb * nb; q += blockDim.x)
    out[q] = cdir(t2, mat, nb, na, nb, nb, 2, q);
  __syncthreads();
}

// shared memory: tmp / gl [m^3], t1, t2 [n^2 m], vel [n^3], ur/us/ut [3 n^3]
__host__ __device__ inline size_t exact_smem_doubles(int n) {
  const int m = n - 2;
  return (size_t)m * m * m + 2 * (size_t)n * n * m + (size_t)n * n * n + 3 * (size_t)n * n * n;
}

// gradient_from_pressure (operators.cpp:365-410), one CTA per element
__global__ void __launch_bounds__(kXThreads)
    p_grad_exact_kernel(const double* __restrict__ p, int64_t E, int n,
                        const double* __restrict__ corners, ExactMats M, double* __restrict__ g0,
                        double* __restrict__ g1, double* __restrict__ g2) {
  const int m = n - 2, m3 = m * m * m, n3 = n * n * n;
  extern __shared__ double xs[];
  double* tmp = xs;
  double* t1 = tmp + m3;
  double* t2 = t1 + n * n * m;
  double* vel = t2 + n * n * m;
  double* acc = vel + n3;  // [3][n^3] outputs of the element
  double* outs[3] = {g0, g1, g2};
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    for (int q = threadIdx.x; q < 3 * n3; q += blockDim.x) acc[q] = 0.0;
    __syncthreads();
    for (int comp = 0; comp < 3; ++comp)
      for (int pd = 0; pd < 3; ++pd) {
        for (int q = threadIdx.x; q < m3; q += blockDim.x) {
          double wdetj, drdx[9];
          pgeom(corners + e * 24, M, q % m, (q / m) % m, q / (m * m), wdetj, drdx);
          tmp[q] = wdetj * drdx[pd * 3 + comp] * p[e * m3 + q];
        }
        __syncthreads();
        interp3_cta(tmp, t1, t2, vel, M.ivt, n, m);
        for (int q = threadIdx.x; q < n3; q += blockDim.x) {
          const int i = q % n, j = (q / n) % n, k = q / (n * n);
          double s = 0.0;
          if (pd == 0)
            for (int l = 0; l < n; ++l) s += M.d[l * n + i] * vel[(k * n + j) * n + l];
          else if (pd == 1)
            for (int l = 0; l < n; ++l) s += M.d[l * n + j] * vel[(k * n + l) * n + i];
          else
            for (int l = 0; l < n; ++l) s += M.d[l * n + k] * vel[(l * n + j) * n + i];
          acc[comp * n3 + q] += s;
        }
        __syncthreads();
      }
    for (int q = threadIdx.x; q < 3 * n3; q += blockDim.x) outs[q / n3][e * n3 + q % n3] = acc[q];
    __syncthreads();
  }
}

// divergence_to_pressure (operators.cpp:327-363), one CTA per element
__global__ void __launch_bounds__(kXThreads)
    p_div_exact_kernel(const double* __restrict__ u0, const double* __restrict__ u1,
                       const double* __restrict__ u2, int64_t E, int n,
                       const double* __restrict__ corners, ExactMats M,
                       double* __restrict__ out) {
  const int m = n - 2, m3 = m * m * m, n3 = n * n * n;
  extern __shared__ double xs[];
  double* gl = xs;
  double* t1 = gl + m3;
  double* t2 = t1 + n * n * m;
  double* in = t2 + n * n * m;
  double* ref = in + n3;  // ur, us, ut
  const double* us[3] = {u0, u1, u2};
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    double o[(14 * 14 * 14 + kXThreads - 1) / kXThreads];  // the thread's GL outputs
    const int per = (m3 + kXThreads - 1) / kXThreads;
    for (int u = 0; u < per; ++u) o[u] = 0.0;
    for (int comp = 0; comp < 3; ++comp) {
      for (int q = threadIdx.x; q < n3; q += blockDim.x) in[q] = us[comp][e * n3 + q];
      __syncthreads();
      // ref_derivatives (operators.cpp:60-76)
      for (int q = threadIdx.x; q < n3; q += blockDim.x) {
        const int i = q % n, j = (q / n) % n, k = q / (n * n);
        double r = 0.0, s = 0.0, t = 0.0;
        for (int l = 0; l < n; ++l) {
          r += M.d[i * n + l] * in[(k * n + j) * n + l];
          s += M.d[j * n + l] * in[(k * n + l) * n + i];
          t += M.d[k * n + l] * in[(l * n + j) * n + i];
        }
        ref[q] = r;
        ref[n3 + q] = s;
        ref[2 * n3 + q] = t;
      }
      __syncthreads();
      for (int pp = 0; pp < 3; ++pp) {
        interp3_cta(ref + pp * n3, t1, t2, gl, M.iv, m, n);
        for (int u = 0; u < per; ++u) {
          const int q = threadIdx.x + u * kXThreads;
          if (q < m3) {
            double wdetj, drdx[9];
            pgeom(corners + e * 24, M, q % m, (q / m) % m, q / (m * m), wdetj, drdx);
            o[u] += wdetj * drdx[pp * 3 + comp] * gl[q];
          }
        }
        __syncthreads();
      }
    }
    for (int u = 0; u < per; ++u) {
      const int q = threadIdx.x + u * kXThreads;
      if (q < m3) out[e * m3 + q] = o[u];
    }
    __syncthreads();
  }
}

// pressure_operator_diagonal (stepper.cpp:250-275): per element, the exact
// gradient of every GL unit vector, sum over d, a of v*v*inv_bdiag
__global__ void __launch_bounds__(kXThreads)
    p_diag_exact_kernel(int64_t E, int n, const double* __restrict__ corners, ExactMats M,
                        const double* __restrict__ inv_bdiag, double* __restrict__ diag) {
  const int m = n - 2, m3 = m * m * m, n3 = n * n * n;
  extern __shared__ double xs[];
  double* tmp = xs;
  double* t1 = tmp + m3;
  double* t2 = t1 + n * n * m;
  double* vel = t2 + n * n * m;
  double* acc = vel + n3;
  __shared__ double red[kXThreads];
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    for (int qu = 0; qu < m3; ++qu) {
      for (int q = threadIdx.x; q < 3 * n3; q += blockDim.x) acc[q] = 0.0;
      __syncthreads();
      for (int comp = 0; comp < 3; ++comp)
        for (int pd = 0; pd < 3; ++pd) {
          for (int q = threadIdx.x; q < m3; q += blockDim.x) {
            double wdetj, drdx[9];
            pgeom(corners + e * 24, M, q % m, (q / m) % m, q / (m * m), wdetj, drdx);
            tmp[q] = wdetj * drdx[pd * 3 + comp] * (q == qu ? 1.0 : 0.0);
          }
          __syncthreads();
          interp3_cta(tmp, t1, t2, vel, M.ivt, n, m);
          for (int q = threadIdx.x; q < n3; q += blockDim.x) {
            const int i = q % n, j = (q / n) % n, k = q / (n * n);
            double s = 0.0;
            if (pd == 0)
              for (int l = 0; l < n; ++l) s += M.d[l * n + i] * vel[(k * n + j) * n + l];
            else if (pd == 1)
              for (int l = 0; l < n; ++l) s += M.d[l * n + j] * vel[(k * n + l) * n + i];
            else
              for (int l = 0; l < n; ++l) s += M.d[l * n + k] * vel[(l * n + j) * n + i];
            acc[comp * n3 + q] += s;
          }
          __syncthreads();
        }
      // s = sum_d sum_a v*v*inv_bdiag, sequential (thread 0)
      if (threadIdx.x == 0) {
        double s = 0.0;
        for (int d = 0; d < 3; ++d)
          for (int a = 0; a < n3; ++a) {
            const double v = acc[d * n3 + a];
            s += v * v * inv_bdiag[e * n3 + a];
          }
        diag[e * m3 + qu] = s;
      }
      __syncthreads();
    }
  }
  (void)red;
}

// mean deflation of pressure_precond (stepper.cpp:278-283): mean = sequential
// sum / size; z -= mean.  One thread for the sum (reference order).
__global__ void deflate_sum_kernel(int64_t N, const double* __restrict__ z,
                                   double* __restrict__ mean) {
  double s = 0.0;
  for (int64_t a = 0; a < N; ++a) s += z[a];
  *mean = s / (double)N;
}

__global__ void deflate_sub_kernel(int64_t N, double* __restrict__ z,
                                   const double* __restrict__ mean) {
  const double mu = *mean;
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < N;
       a += (int64_t)gridDim.x * blockDim.x)
    z[a] -= mu;
}

// advect (operators.cpp:412-431) with grad_velocity (:300-325): per
// component the reference derivatives, dr/dx at the GLL node (the
// TrilinearMap Jacobian's inverse, as build_geometric_factors forms drdx),
// out = bm (c . grad u).  Reference operation order (this file is -fmad=false).
__global__ void __launch_bounds__(kXThreads)
    advect_kernel(const double* __restrict__ u0, const double* __restrict__ u1,
                  const double* __restrict__ u2, const double* __restrict__ c0,
                  const double* __restrict__ c1, const double* __restrict__ c2,
                  const double* __restrict__ bm, int64_t E, int n,
                  const double* __restrict__ corners, const double* __restrict__ D,
                  const double* __restrict__ gllx, double* __restrict__ o0,
                  double* __restrict__ o1, double* __restrict__ o2) {
  const int n3 = n * n * n;
  extern __shared__ double xs[];
  double* in = xs;         // u0 | u1 | u2 of the element
  double* sD = in + 3 * n3;
  double* sX = sD + n * n;
  double* scr = sX + n;    // the element's 24 corner coordinates
  const double* us[3] = {u0, u1, u2};
  double* outs[3] = {o0, o1, o2};
  for (int q = threadIdx.x; q < n * n; q += blockDim.x) sD[q] = D[q];
  for (int q = threadIdx.x; q < n; q += blockDim.x) sX[q] = gllx[q];
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    __syncthreads();
    for (int q = threadIdx.x; q < 3 * n3; q += blockDim.x)
      in[q] = us[q / n3][e * n3 + q % n3];
    if (threadIdx.x < 24) scr[threadIdx.x] = corners[e * 24 + threadIdx.x];
    __syncthreads();
    for (int q = threadIdx.x; q < n3; q += blockDim.x) {
      const int i = q % n, j = (q / n) % n, k = q / (n * n);
      // drdx at GLL node (i, j, k): inv3 of the TrilinearMap Jacobian, once
      // per node for the three components
      const double r = sX[i], s = sX[j], t = sX[k];
      const double sh[3][2] = {{0.5 * (1 - r), 0.5 * (1 + r)},
                               {0.5 * (1 - s), 0.5 * (1 + s)},
                               {0.5 * (1 - t), 0.5 * (1 + t)}};
      double J[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int b0 = v & 1, b1 = (v >> 1) & 1, b2 = (v >> 2) & 1;
        const double d0 = b0 ? 0.5 : -0.5, d1 = b1 ? 0.5 : -0.5, d2 = b2 ? 0.5 : -0.5;
        const double gr[3] = {d0 * sh[1][b1] * sh[2][b2], sh[0][b0] * d1 * sh[2][b2],
                              sh[0][b0] * sh[1][b1] * d2};
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          const double xp = scr[v * 3 + p];
          J[p * 3 + 0] += xp * gr[0];
          J[p * 3 + 1] += xp * gr[1];
          J[p * 3 + 2] += xp * gr[2];
        }
      }
      const double det = J[0] * (J[4] * J[8] - J[5] * J[7]) -
                         J[1] * (J[3] * J[8] - J[5] * J[6]) + J[2] * (J[3] * J[7] - J[4] * J[6]);
      const double id = 1.0 / det;
      const double R[9] = {(J[4] * J[8] - J[5] * J[7]) * id, (J[2] * J[7] - J[1] * J[8]) * id,
                           (J[1] * J[5] - J[2] * J[4]) * id, (J[5] * J[6] - J[3] * J[8]) * id,
                           (J[0] * J[8] - J[2] * J[6]) * id, (J[2] * J[3] - J[0] * J[5]) * id,
                           (J[3] * J[7] - J[4] * J[6]) * id, (J[1] * J[6] - J[0] * J[7]) * id,
                           (J[0] * J[4] - J[1] * J[3]) * id};
      const int64_t a = e * n3 + q;
      const double cv0 = c0[a], cv1 = c1[a], cv2 = c2[a], b = bm[a];
      for (int comp = 0; comp < 3; ++comp) {
        const double* u = in + comp * n3;
        double dr = 0.0, ds = 0.0, dt = 0.0;
        for (int l = 0; l < n; ++l) {
          dr += sD[i * n + l] * u[(k * n + j) * n + l];
          ds += sD[j * n + l] * u[(k * n + l) * n + i];
          dt += sD[k * n + l] * u[(l * n + j) * n + i];
        }
        double g[3];
#pragma unroll
        for (int qq = 0; qq < 3; ++qq) g[qq] = R[0 + qq] * dr + R[3 + qq] * ds + R[6 + qq] * dt;
        outs[comp][a] = b * (cv0 * g[0] + cv1 * g[1] + cv2 * g[2]);
      }
    }
  }
}

unsigned egrid(int64_t E) { return (unsigned)(E < 148 * 8 ? (E < 1 ? 1 : E) : 148 * 8); }

}  // namespace

cudaError_t launch_p_grad_exact(const PresExact& X, const double* p, double* const g[3],
                                cudaStream_t s) {
  const size_t sm = sizeof(double) * exact_smem_doubles(X.n);
  cudaError_t e = cudaFuncSetAttribute(p_grad_exact_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  ExactMats M{X.d, X.iv, X.ivt, X.glx, X.glw};
  p_grad_exact_kernel<<<egrid(X.E), kXThreads, sm, s>>>(p, X.E, X.n, X.corners, M, g[0], g[1],
                                                        g[2]);
  return cudaGetLastError();
}

cudaError_t launch_p_div_exact(const PresExact& X, const double* const u[3], double* out,
                               cudaStream_t s) {
  const size_t sm = sizeof(double) * exact_smem_doubles(X.n);
  cudaError_t e = cudaFuncSetAttribute(p_div_exact_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  ExactMats M{X.d, X.iv, X.ivt, X.glx, X.glw};
  p_div_exact_kernel<<<egrid(X.E), kXThreads, sm, s>>>(u[0], u[1], u[2], X.E, X.n, X.corners,
                                                       M, out);
  return cudaGetLastError();
}

cudaError_t launch_p_diag_exact(const PresExact& X, const double* inv_bdiag, double* diag,
                                cudaStream_t s) {
  const size_t sm = sizeof(double) * exact_smem_doubles(X.n);
  cudaError_t e = cudaFuncSetAttribute(p_diag_exact_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  ExactMats M{X.d, X.iv, X.ivt, X.glx, X.glw};
  p_diag_exact_kernel<<<egrid(X.E), kXThreads, sm, s>>>(X.E, X.n, X.corners, M, inv_bdiag,
                                                        diag);
  return cudaGetLastError();
}

cudaError_t launch_advect(int64_t E, int n, const double* corners, const double* D,
                          const double* gllx, const double* bm, const double* const u[3],
                          const double* const c[3], double* const out[3], cudaStream_t s) {
  const size_t sm = sizeof(double) * (3 * (size_t)n * n * n + (size_t)n * n + n + 24);
  cudaError_t e = cudaFuncSetAttribute(advect_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  advect_kernel<<<egrid(E), kXThreads, sm, s>>>(u[0], u[1], u[2], c[0], c[1], c[2], bm, E, n,
                                                corners, D, gllx, out[0], out[1], out[2]);
  return cudaGetLastError();
}

cudaError_t launch_deflate_exact(int64_t N, double* z, double* mean_scratch, cudaStream_t s) {
  deflate_sum_kernel<<<1, 1, 0, s>>>(N, z, mean_scratch);
  int64_t b = (N + 255) / 256;
  if (b > 148 * 8) b = 148 * 8;
  deflate_sub_kernel<<<(unsigned)(b < 1 ? 1 : b), 256, 0, s>>>(N, z, mean_scratch);
  return cudaGetLastError();
}

}  // namespace sbx
