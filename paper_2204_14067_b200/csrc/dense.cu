// Dense fp64 contractions of the lifting step on the fp64 tensor cores.
//
// The lifting step's dense work is tall-skinny: Grams of factor / basis
// blocks (m x p with m up to 1e6 and p up to ~1500: inner_product's
// L_a^T L_b and R_a^T R_b, mfg/operators.py:67-81; the CholeskyQR Gram B^T B
// and the Rayleigh-Ritz projection q^T S q, mfg/kernels.py:76-105,
// mfg/eigensolver.py:81-92; H^T V / W^T U in ShiftedOperator.apply,
// mfg/operators.py:102-118) and tall-times-small products (W (H^T V),
// q P, S q P, M^T U / sigma). Both run here on mma.sync.m8n8k4.f64 (DMMA):
//   * k_gemm_tn: C = alpha A^T B. 64 x 64 tiles of C per CTA (4 warps, each
//     32 x 32 = 4 x 4 DMMA tiles), rows of A/B (the contraction) streamed
//     through shared memory 16 at a time with a register prefetch of the
//     next chunk. The contraction is split over S row slices so that tall
//     blocks with few tiles still fill the GPU; the CTA that finishes a
//     tile's last slice (arrival counter) adds the S partial tiles in slice
//     order, so results are bitwise reproducible with no second launch.
//   * k_gemm_nn: C = alpha A B + beta C, 64 x 64 tiles of C, the (short)
//     contraction streamed 16 at a time.
// DMMA fragment conventions (PTX m8n8k4 .f64): A (8x4 row) a0 = A[lane/4][lane%4],
// B (4x8 col) b0 = B[lane%4][lane/4], C/D (8x8) d{0,1} = D[lane/4][2(lane%4)+{0,1}].
#include "common.cuh"
#include "engine.cuh"

namespace mfg {
namespace {

constexpr int kT = 64;       // C tile
constexpr int kKC = 16;      // contraction chunk
constexpr int kLdW = 72;     // shared row stride (doubles) of 64-wide chunks: 4 rows -> alternating bank halves
constexpr int kLdN = 20;     // shared row stride of the 16-wide A chunk of k_gemm_nn

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// C (p x q) = alpha * A^T B over rows [r0, r1) of slice blockIdx.z; S == 1
// writes C, else the slice's partial tile goes to part[z][tile][64 x 64] and
// the last-arriving slice of the tile (cnt[tile], zero at rest) sums them.
__global__ void __launch_bounds__(128) k_gemm_tn(int m, int p, int q, const double* __restrict__ A,
                                                 int lda, const double* __restrict__ B, int ldb,
                                                 double alpha, double* __restrict__ C, int ldc,
                                                 double* __restrict__ part, unsigned* __restrict__ cnt,
                                                 int S, int rps) {
  __shared__ __align__(16) double sA[kKC][kLdW];
  __shared__ __align__(16) double sB[kKC][kLdW];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int wy = w >> 1, wx = w & 1;
  const int p0 = blockIdx.x * kT, q0 = blockIdx.y * kT;
  const int r0 = blockIdx.z * rps;
  const int r1 = min(m, r0 + rps);
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // each thread moves 8 doubles of A and 8 of B per chunk: row rr = x / 64
  double ra[8], rb[8];
  auto fetch = [&](int r) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int x = tid + 128 * u;
      const int rr = x >> 6, cc = x & 63;
      const int row = r + rr;
      ra[u] = (row < r1 && p0 + cc < p) ? A[(int64_t)row * lda + p0 + cc] : 0.0;
      rb[u] = (row < r1 && q0 + cc < q) ? B[(int64_t)row * ldb + q0 + cc] : 0.0;
    }
  };
  if (r0 < r1) fetch(r0);
  for (int r = r0; r < r1; r += kKC) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int x = tid + 128 * u;
      sA[x >> 6][x & 63] = ra[u];
      sB[x >> 6][x & 63] = rb[u];
    }
    __syncthreads();
    if (r + kKC < r1) fetch(r + kKC);
#pragma unroll
    for (int s = 0; s < kKC / 4; ++s) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sA[4 * s + tq][wy * 32 + 8 * i + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sB[4 * s + tq][wx * 32 + 8 * j + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }
  const size_t tile = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
  const size_t per = (size_t)gridDim.x * gridDim.y * kT * kT;
  double* dst = S > 1 ? part + blockIdx.z * per + tile * kT * kT : nullptr;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int lr = wy * 32 + 8 * i + g, lc = wx * 32 + 8 * j + 2 * tq + h;
        if (dst) {
          dst[lr * kT + lc] = acc[i][j][h];
        } else if (p0 + lr < p && q0 + lc < q) {
          C[(int64_t)(p0 + lr) * ldc + q0 + lc] = alpha * acc[i][j][h];
        }
      }
  if (S == 1) return;
  __shared__ int s_last;
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  __syncthreads();
  if (tid == 0) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt + tile) : "memory");
    s_last = old == (unsigned)(S - 1);
  }
  __syncthreads();
  if (!s_last) return;
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  for (int e = tid; e < kT * kT; e += 128) {
    const int r = p0 + e / kT, c = q0 + e % kT;
    if (r >= p || c >= q) continue;
    const double* src = part + tile * kT * kT + e;
    double s = 0.0;
    for (int z = 0; z < S; ++z) s += __ldcg(src + z * per);
    C[(int64_t)r * ldc + c] = alpha * s;
  }
  if (tid == 0) cnt[tile] = 0u;   // at rest for the next call
}

// C (m x q) = alpha * A (m x p) B (p x q) + beta * Cin (Cin may be C itself)
__global__ void __launch_bounds__(128) k_gemm_nn(int m, int p, int q, const double* __restrict__ A,
                                                 int lda, const double* __restrict__ B, int ldb,
                                                 double alpha, double beta, double* C, int ldc,
                                                 const double* Cin, int ldcin) {
  __shared__ __align__(16) double sA[kT][kLdN];
  __shared__ __align__(16) double sB[kKC][kLdW];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int wy = w >> 1, wx = w & 1;
  const int i0 = blockIdx.x * kT, j0 = blockIdx.y * kT;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double ra[8], rb[8];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int x = tid + 128 * u;
      // A chunk 64 x 16: row x / 16, col x % 16
      const int ar = x >> 4, ac = x & 15;
      ra[u] = (i0 + ar < m && k0 + ac < p) ? A[(int64_t)(i0 + ar) * lda + k0 + ac] : 0.0;
      // B chunk 16 x 64: row x / 64, col x % 64
      const int br = x >> 6, bc = x & 63;
      rb[u] = (k0 + br < p && j0 + bc < q) ? B[(int64_t)(k0 + br) * ldb + j0 + bc] : 0.0;
    }
  };
  fetch(0);
  for (int k0 = 0; k0 < p; k0 += kKC) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int x = tid + 128 * u;
      sA[x >> 4][x & 15] = ra[u];
      sB[x >> 6][x & 63] = rb[u];
    }
    __syncthreads();
    if (k0 + kKC < p) fetch(k0 + kKC);
#pragma unroll
    for (int s = 0; s < kKC / 4; ++s) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sA[wy * 32 + 8 * i + g][4 * s + tq];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sB[4 * s + tq][wx * 32 + 8 * j + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = i0 + wy * 32 + 8 * i + g, c = j0 + wx * 32 + 8 * j + 2 * tq + h;
        if (r < m && c < q) {
          double* o = C + (int64_t)r * ldc + c;
          const double v = alpha * acc[i][j][h];
          *o = beta == 0.0 ? v : fma(beta, Cin[(int64_t)r * ldcin + c], v);
        }
      }
}

int slices_for(int m, int ntiles) {
  // fill ~2 CTAs per SM; at least 64 contraction rows per slice
  int s = (2 * kNumSMs + ntiles - 1) / ntiles;
  const int maxs = (m + 63) / 64;
  if (s > maxs) s = maxs;
  if (s < 1) s = 1;
  return s;
}

}  // namespace

// workspace: a fixed region of kMaxTiles arrival counters (zero before the
// first use; the kernel leaves them zero -- fixed, so calls of different
// shapes sharing one workspace never overlay partials on counters), then
// the S partial tiles
constexpr int kMaxTiles = 16384;
constexpr size_t kCntBytes = (size_t)kMaxTiles * 4;

size_t gemm_tn_workspace(int m, int p, int q) {
  const int ntx = (p + kT - 1) / kT, nty = (q + kT - 1) / kT;
  const int S = ntx * nty <= kMaxTiles ? slices_for(m, ntx * nty) : 1;
  return S > 1 ? kCntBytes + (size_t)S * ntx * nty * kT * kT * sizeof(double) : 0;
}

int gemm_tn(int m, int p, int q, const double* A, int lda, const double* B, int ldb, double alpha,
            double* C, int ldc, void* ws, size_t wsb, cudaStream_t stream) {
  MFG_REQUIRE(m >= 0 && p >= 0 && q >= 0, "negative size");
  MFG_REQUIRE(lda >= p && ldb >= q && ldc >= q, "leading dimension too small");
  if (p == 0 || q == 0) return MFG_OK;
  const int ntx = (p + kT - 1) / kT, nty = (q + kT - 1) / kT;
  if (m == 0) {
    MFG_CUDA_CHECK(cudaMemset2DAsync(C, (size_t)ldc * 8, 0, (size_t)q * 8, p, stream));
    return MFG_OK;
  }
  const int S = ntx * nty <= kMaxTiles ? slices_for(m, ntx * nty) : 1;
  const int rps = (((m + S - 1) / S) + kKC - 1) / kKC * kKC;
  const int Sr = (m + rps - 1) / rps;
  const size_t coff = kCntBytes;
  if (Sr > 1) MFG_REQUIRE(ws && wsb >= coff + (size_t)Sr * ntx * nty * kT * kT * sizeof(double),
                          "gemm_tn workspace too small");
  dim3 grid(ntx, nty, Sr);
  k_gemm_tn<<<grid, 128, 0, stream>>>(m, p, q, A, lda, B, ldb, alpha, C, ldc,
                                      Sr > 1 ? (double*)((char*)ws + coff) : nullptr,
                                      (unsigned*)ws, Sr, rps);
  MFG_LAUNCH_CHECK();
  return MFG_OK;
}

int gemm_nn(int m, int p, int q, const double* A, int lda, const double* B, int ldb, double alpha,
            double beta, double* C, int ldc, cudaStream_t stream, const double* Cin, int ldcin) {
  if (!Cin) {
    Cin = C;
    ldcin = ldc;
  }
  MFG_REQUIRE(m >= 0 && p >= 0 && q >= 0, "negative size");
  MFG_REQUIRE(lda >= p && ldb >= q && ldc >= q, "leading dimension too small");
  if (m == 0 || q == 0) return MFG_OK;
  if (p == 0 && beta == 0.0) {
    MFG_CUDA_CHECK(cudaMemset2DAsync(C, (size_t)ldc * 8, 0, (size_t)q * 8, m, stream));
    return MFG_OK;
  }
  dim3 grid((m + kT - 1) / kT, (q + kT - 1) / kT);
  k_gemm_nn<<<grid, 128, 0, stream>>>(m, p, q, A, lda, B, ldb, alpha, beta, C, ldc, Cin, ldcin);
  MFG_LAUNCH_CHECK();
  return MFG_OK;
}

}  // namespace mfg
