// Calibration microbenchmark: random factor-row gathers on B200, LSU vs TMA.
// Table of R rows x k fp32 (ld = k, unpadded, as the sweep stores factors);
// N row ids (uniform or Zipf). Every gathered row is summed into a register.
//   ldg : the sweep's 8-lane groups, one LDG.128 per lane per row (lanes past
//         the row alias chunk 0), 8 rows per group in flight.
//   tma : per warp a ring of NS stages x 32 rows; lanes 0..7 each issue one
//         cp.async.bulk.tensor.2d ... tile::gather4 (4 rows -> shared memory,
//         completion on the stage's mbarrier); the 8-lane groups then read
//         their 8 rows with LDS.128. The gathers bypass the LSU / L1 tag path.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo
//        tools/tma_gather_bench.cu -o tools/tma_gather_bench -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <int K>
__global__ void __launch_bounds__(128) ldg8(const float* __restrict__ T, const int* __restrict__ idx, int n,
                                            float* out, double* chk) {
  constexpr int NC = K / 4;  // 16-byte chunks per row
  const int q = threadIdx.x & 7;
  const int grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int ngrp = (gridDim.x * blockDim.x) >> 3;
  const int cq = q < NC ? q : 0;
  float acc = 0.f;
  for (int base = grp * 8; base < n; base += ngrp * 8) {
    const int my = base + q < n ? idx[base + q] : 0;
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = __shfl_sync(0xffffffffu, my, u, 8);
      v[u] = reinterpret_cast<const float4*>(T + (size_t)j * K)[cq];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += (q < NC) ? (v[u].x + v[u].y + v[u].z + v[u].w) : 0.f;
  }
  if (acc == 12345.f) out[grp] = acc;
  if (chk) atomicAdd(chk, (double)acc);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_gather4(float* dst, const CUtensorMap* map, int c0, int r0, int r1, int r2, int r3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

template <int K, int NS>
__global__ void __launch_bounds__(128) tma8(const __grid_constant__ CUtensorMap map, const int* __restrict__ idx,
                                            int n, float* out, double* chk) {
  constexpr int NC = K / 4;
  constexpr int ROWB = K * 4;
  constexpr int SLOT = (4 * K + 31) / 32 * 32;  // floats per gather4 slot (128-byte aligned)
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = lane & 7, g = lane >> 3;
  float* ring = reinterpret_cast<float*>(smem) + (size_t)warp * NS * 8 * SLOT;
  __shared__ __align__(8) uint64_t bars[4][NS];
  uint64_t* bar = bars[warp];
  if (lane == 0)
    for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int gw = blockIdx.x * 4 + warp, nw = gridDim.x * 4;
  const int nb = (n + 31) / 32;  // 32-row batches
  auto issue = [&](int b, int s) {
    const int base = b * 32;
    const int my = base + lane < n ? idx[base + lane] : 0;
    const int j0 = __shfl_sync(0xffffffffu, my, (lane & 7) * 4 + 0);
    const int j1 = __shfl_sync(0xffffffffu, my, (lane & 7) * 4 + 1);
    const int j2 = __shfl_sync(0xffffffffu, my, (lane & 7) * 4 + 2);
    const int j3 = __shfl_sync(0xffffffffu, my, (lane & 7) * 4 + 3);
    if (lane == 0) mbar_expect(&bar[s], 32 * ROWB);
    __syncwarp();
    if (lane < 8) tma_gather4(ring + (size_t)s * 8 * SLOT + lane * SLOT, &map, 0, j0, j1, j2, j3, &bar[s]);
  };
  float acc = 0.f;
  int it = 0;
  // prologue: fill NS stages
  for (int s = 0; s < NS; ++s) {
    const int b = gw + s * nw;
    if (b < nb) issue(b, s);
  }
  for (int b = gw; b < nb; b += nw, ++it) {
    const int s = it % NS;
    mbar_wait(&bar[s], (it / NS) & 1);
    const float* st = ring + (size_t)s * 8 * SLOT + g * 2 * SLOT;
    const int cq = q < NC ? q : 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float4 v = reinterpret_cast<const float4*>(st + (u >> 2) * SLOT + (u & 3) * K)[cq];
      acc += (q < NC) ? (v.x + v.y + v.z + v.w) : 0.f;
    }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const int bn = b + NS * nw;
    if (bn < nb) issue(bn, s);
  }
  if (acc == 12345.f) out[gw * 32 + lane] = acc;
  if (chk) atomicAdd(chk, (double)acc);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <typename F>
float timeit(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  launch();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < 20; ++i) launch();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 20;
}

template <int K>
void run(int R, int n, double zipf) {
  std::vector<int> h(n);
  std::mt19937 rng(1);
  if (zipf <= 0) { std::uniform_int_distribution<int> d(0, R - 1); for (auto& x : h) x = d(rng); }
  else {
    std::vector<double> cw(R); double s = 0;
    for (int i = 0; i < R; ++i) { s += 1.0 / pow(i + 1.0, zipf); cw[i] = s; }
    std::uniform_real_distribution<double> d(0, s);
    std::vector<int> perm(R); for (int i = 0; i < R; ++i) perm[i] = i; std::shuffle(perm.begin(), perm.end(), rng);
    for (auto& x : h) x = perm[std::lower_bound(cw.begin(), cw.end(), d(rng)) - cw.begin()];
  }
  float *T, *out; int* idx;
  CK(cudaMalloc(&T, (size_t)R * K * 4)); CK(cudaMemset(T, 0, (size_t)R * K * 4));
  CK(cudaMalloc(&idx, (size_t)n * 4)); CK(cudaMemcpy(idx, h.data(), (size_t)n * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&out, 64 << 20));
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr));
  CUtensorMap map;
  cuuint64_t gdim[2] = {(cuuint64_t)K, (cuuint64_t)R};
  cuuint64_t gstr[1] = {(cuuint64_t)K * 4};
  cuuint32_t box[2] = {(cuuint32_t)K, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, T, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) { printf("encode failed %d\n", (int)cr); exit(1); }
  const double rows = n;
  printf("K=%d R=%d n=%d zipf=%.2f table=%.2f MB\n", K, R, n, zipf, R * K * 4 / 1e6);
  for (int bps : {2, 4, 6}) {  // 128-thread CTAs per SM
    const int grid = 148 * bps;
    float t = timeit([&] { ldg8<K><<<grid, 128>>>(T, idx, n, out, nullptr); });
    printf("  ldg8  CTAs/SM %d       : %8.1f us  %6.1f G rows/s\n", bps, t * 1e3, rows / t / 1e6);
  }
  auto tma_run = [&](auto ns_c, int bps) {
    constexpr int NS = decltype(ns_c)::value;
    const size_t sm = (size_t)4 * NS * 8 * ((4 * K + 31) / 32 * 32) * 4;
    if (sm > 227 * 1024) return;
    CK(cudaFuncSetAttribute(tma8<K, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const int grid = 148 * bps;
    float t = timeit([&] { tma8<K, NS><<<grid, 128, sm>>>(map, idx, n, out, nullptr); });
    CK(cudaGetLastError());
    printf("  tma8  CTAs/SM %d NS=%d : %8.1f us  %6.1f G rows/s  (smem %zu B/CTA)\n", bps, NS, t * 1e3,
           rows / t / 1e6, sm);
  };
  for (int bps : {2, 4}) {
    tma_run(std::integral_constant<int, 2>{}, bps);
    tma_run(std::integral_constant<int, 4>{}, bps);
  }
  tma_run(std::integral_constant<int, 8>{}, 2);
  // correctness: row j holds (j % 97) in every element; both kernels must sum
  // K * sum_e (idx_e % 97)
  {
    std::vector<float> tv((size_t)R * K);
    for (int j = 0; j < R; ++j) for (int c = 0; c < K; ++c) tv[(size_t)j * K + c] = (float)(j % 97);
    CK(cudaMemcpy(T, tv.data(), tv.size() * 4, cudaMemcpyHostToDevice));
    double want = 0; for (int e = 0; e < n; ++e) want += (double)K * (h[e] % 97);
    double* chk; CK(cudaMalloc(&chk, 8));
    double got[2];
    CK(cudaMemset(chk, 0, 8)); ldg8<K><<<296, 128>>>(T, idx, n, out, chk); CK(cudaMemcpy(&got[0], chk, 8, cudaMemcpyDeviceToHost));
    const size_t sm = (size_t)4 * 2 * 8 * ((4 * K + 31) / 32 * 32) * 4;
    CK(cudaFuncSetAttribute(tma8<K, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    CK(cudaMemset(chk, 0, 8)); tma8<K, 2><<<296, 128, sm>>>(map, idx, n, out, chk); CK(cudaMemcpy(&got[1], chk, 8, cudaMemcpyDeviceToHost));
    printf("  check: want %.0f ldg8 %.0f tma8 %.0f -> %s\n", want, got[0], got[1],
           (fabs(got[0] - want) < 1e-6 * want && fabs(got[1] - want) < 1e-6 * want) ? "OK" : "MISMATCH");
    cudaFree(chk);
  }
  cudaFree(T); cudaFree(idx); cudaFree(out);
}

int main(int argc, char** argv) {
  const int R = argc > 1 ? atoi(argv[1]) : 6040;
  const int n = argc > 2 ? atoi(argv[2]) : 2000000;
  const double zipf = argc > 3 ? atof(argv[3]) : 1.0;
  run<20>(R, n, zipf);
  run<40>(R, n, zipf);
  run<64>(R, n, zipf);
  return 0;
}
