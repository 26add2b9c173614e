// BCD half-sweep: exact per-row minimisers of the MF objective.
//
// Replaces _half_sweep (mfg/mfsolver.py:53-75), which assembles the per-row
// normal matrices lam*I + 2*sum_{j in Omega_i} o_j o_j^T with a pattern SpMM
// over k(k+1)/2 pair-product columns (materialising (m, k, k) fp64 normals
// and (m, k(k+1)/2) pair products on the host) and then runs a batched LU
// solve. Here one CTA owns one row at a time: the gathered factor rows are
// staged through shared memory in chunks of kC entries, the Gram matrix is
// accumulated in fp64 register tiles (4x4 per thread, upper triangle only)
// into shared memory, and the SPD system is solved in place by Cholesky.
// Nothing of size (m, k, k) ever exists, so config 5 (n ~ 1e6, k = 64) runs.
// Arithmetic is fp64 for both storage types.
#include "common.cuh"
#include "engine.cuh"

namespace mfg {
namespace {

constexpr int kNT = 128;
constexpr int kC = 16;         // entries staged per chunk
constexpr int kSmemMaxK = 128; // Gram in shared memory up to this k

template <typename TS>
__global__ void __launch_bounds__(kNT)
k_bcd(mfg_layout lay, int k, const TS* __restrict__ vals, const TS* __restrict__ other, int ldo,
      double lam, TS* __restrict__ out, int ldout, double* __restrict__ gscratch, int use_global,
      int* __restrict__ bad) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x;
  const int kp = k + 1;                         // padded leading dimension
  double* stage = sm;                           // [kC][kp]
  double* sa = stage + kC * kp;                 // [kC]
  double* bvec = sa + kC;                       // [k]
  double* yvec = bvec + k;                      // [k]
  double* G = use_global ? gscratch + (size_t)blockIdx.x * k * k : yvec + k;  // [k][k]
  const int nt4 = (k + 3) / 4;                  // 4x4 tiles per dim
  for (int i = blockIdx.x; i < lay.nrows; i += gridDim.x) {
    const int e0 = lay.ptr[i], e1 = lay.ptr[i + 1];
    for (int x = tid; x < k * k; x += kNT) G[x] = 0.0;
    for (int x = tid; x < k; x += kNT) bvec[x] = 0.0;
    __syncthreads();
    for (int c0 = e0; c0 < e1; c0 += kC) {
      const int cn = min(kC, e1 - c0);
      for (int x = tid; x < kC * k; x += kNT) {
        const int c = x / k, d = x - c * k;
        double v = 0.0;
        if (c < cn) v = (double)other[(int64_t)lay.idx[c0 + c] * ldo + d];
        stage[c * kp + d] = v;
      }
      if (tid < kC) sa[tid] = tid < cn ? (double)vals[c0 + tid] : 0.0;
      __syncthreads();
      // Gram tiles (upper triangle incl. diagonal)
      for (int t = tid; t < nt4 * nt4; t += kNT) {
        const int tp = t / nt4, tq = t - tp * nt4;
        if (tq < tp) continue;
        double accv[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) accv[a][b] = 0.0;
        for (int c = 0; c < cn; ++c) {
          double xp[4], xq[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const int p = tp * 4 + a, q = tq * 4 + a;
            xp[a] = p < k ? stage[c * kp + p] : 0.0;
            xq[a] = q < k ? stage[c * kp + q] : 0.0;
          }
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) accv[a][b] = fma(xp[a], xq[b], accv[a][b]);
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int p = tp * 4 + a, q = tq * 4 + b;
            if (p < k && q < k && q >= p) G[p * k + q] += accv[a][b];
          }
      }
      for (int d = tid; d < k; d += kNT) {
        double s = 0.0;
        for (int c = 0; c < cn; ++c) s = fma(sa[c], stage[c * kp + d], s);
        bvec[d] += s;
      }
      __syncthreads();
    }
    // N = lam I + 2 G (upper), rhs = 2 b
    for (int x = tid; x < k * k; x += kNT) {
      const int p = x / k, q = x - p * k;
      if (q >= p) G[x] = 2.0 * G[x] + (p == q ? lam : 0.0);
    }
    for (int x = tid; x < k; x += kNT) bvec[x] *= 2.0;
    __syncthreads();
    // Cholesky N = U^T U, U upper, in place (right-looking)
    for (int j = 0; j < k; ++j) {
      if (tid == 0) {
        const double djj = G[j * k + j];
        if (!(djj > 0.0)) atomicOr(bad, 1);
        G[j * k + j] = sqrt(djj);
      }
      __syncthreads();
      const double ujj = G[j * k + j];
      for (int q = j + 1 + tid; q < k; q += kNT) G[j * k + q] /= ujj;
      __syncthreads();
      const int rem = k - j - 1;
      for (int x = tid; x < rem * rem; x += kNT) {
        const int p = j + 1 + x / rem, q = j + 1 + x % rem;
        if (q >= p) G[p * k + q] -= G[j * k + p] * G[j * k + q];
      }
      __syncthreads();
    }
    // U^T y = rhs
    for (int j = 0; j < k; ++j) {
      if (tid == 0) yvec[j] = bvec[j] / G[j * k + j];
      __syncthreads();
      const double yj = yvec[j];
      for (int q = j + 1 + tid; q < k; q += kNT) bvec[q] -= G[j * k + q] * yj;
      __syncthreads();
    }
    // U w = y  (w stored into bvec)
    for (int j = k - 1; j >= 0; --j) {
      if (tid == 0) bvec[j] = yvec[j] / G[j * k + j];
      __syncthreads();
      const double wj = bvec[j];
      for (int p = tid; p < j; p += kNT) yvec[p] -= G[p * k + j] * wj;
      __syncthreads();
    }
    for (int d = tid; d < k; d += kNT) out[(int64_t)i * ldout + d] = (TS)bvec[d];
    __syncthreads();
  }
}

size_t smem_bytes(int k, bool global) {
  const int kp = k + 1;
  size_t n = (size_t)kC * kp + kC + 2 * (size_t)k;
  if (!global) n += (size_t)k * k;
  return n * sizeof(double);
}

int grid_for_rows(int nrows) {
  int g = nrows;
  if (g > kNumSMs * 8) g = kNumSMs * 8;
  if (g < 1) g = 1;
  return g;
}

template <typename TS>
int do_bcd(const mfg_layout* lay, int k, const void* vals, const void* other, int ldo, double lam,
           void* out, int ldout, void* ws, size_t wsb, cudaStream_t stream) {
  if (lay->nrows == 0 || k == 0) return MFG_OK;
  const bool global = k > kSmemMaxK;
  const int grid = global ? 2 * kNumSMs : grid_for_rows(lay->nrows);
  Carver c(ws, wsb);
  int* bad = c.take<int>(1);
  double* gs = global ? c.take<double>((size_t)grid * k * k) : nullptr;
  MFG_REQUIRE(c.ok, "bcd workspace too small");
  const size_t smem = smem_bytes(k, global);
  if (smem > 48 * 1024)
    MFG_CUDA_CHECK(cudaFuncSetAttribute(k_bcd<TS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
  MFG_CUDA_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), stream));
  k_bcd<TS><<<grid, kNT, smem, stream>>>(*lay, k, (const TS*)vals, (const TS*)other, ldo, lam,
                                         (TS*)out, ldout, gs, global ? 1 : 0, bad);
  MFG_LAUNCH_CHECK();
  return MFG_OK;
}

}  // namespace

size_t bcd_workspace(const mfg_layout* lay, int k) {
  Sizer s;
  s.take<int>(1);
  if (k > kSmemMaxK) s.take<double>((size_t)2 * kNumSMs * k * k);
  return s.off + 512;
}

int bcd_dispatch(int dtype, const mfg_layout* lay, int k, const void* vals, const void* other,
                 int ldo, double lam, void* out, int ldout, void* ws, size_t wsb,
                 cudaStream_t stream) {
  if (dtype == MFG_F64)
    return do_bcd<double>(lay, k, vals, other, ldo, lam, out, ldout, ws, wsb, stream);
  return do_bcd<float>(lay, k, vals, other, ldo, lam, out, ldout, ws, wsb, stream);
}

}  // namespace mfg
