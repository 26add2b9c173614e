// Calibration: cost of each ingredient of the grouped sweep loop on B200.
// Flat entry stream (idx, val) of n entries; factor tables of 128-B rows.
// MODE 0: gathers only (indices broadcast via smem from per-lane loads)
// MODE 1: + value stream load + R store
// MODE 2: + dot + 8-lane transposed reduce
// MODE 3: + accumulate (full loop body)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ float reduce8(float (&v)[8]) {
  const int q = threadIdx.x & 7;
#pragma unroll
  for (int s = 4; s >= 1; s >>= 1) {
    const bool upper = (q & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float send = upper ? v[i] : v[i + s];
      const float keep = upper ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

template <int MODE>
__global__ void __launch_bounds__(256) loop(const float* __restrict__ T, const float* __restrict__ Wr,
                                            const int* __restrict__ idx, const float* __restrict__ val,
                                            float* __restrict__ R, float* __restrict__ out, int n, int chunk) {
  __shared__ __align__(16) int s_col[32][8];
  __shared__ __align__(16) float s_r[32][8];
  const int q = threadIdx.x & 7, g = threadIdx.x >> 3;
  const int grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const long E0 = (long)grp * chunk, E1 = min(E0 + chunk, (long)n);
  float4 w = reinterpret_cast<const float4*>(Wr + (size_t)(grp % 1000) * 32)[q];
  float acc[4] = {0, 0, 0, 0};
  float sink = 0.f;
  for (long Eb = E0; Eb < E0 + chunk; Eb += 8) {
    const long e = Eb + q;
    const bool v = e < E1;
    const int col = v ? idx[e] : 0;
    float a = 0.f;
    if (MODE >= 1) a = v ? val[e] : 0.f;
    __syncwarp();
    s_col[g][q] = col;
    __syncwarp();
    const int4 c0 = reinterpret_cast<const int4*>(s_col[g])[0];
    const int4 c1 = reinterpret_cast<const int4*>(s_col[g])[1];
    const int cols[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    float4 h[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) h[i] = reinterpret_cast<const float4*>(T + (size_t)cols[i] * 32)[q];
    if (MODE == 0 || MODE == 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) sink += h[i].x + h[i].y + h[i].z + h[i].w;
      if (MODE == 1 && v) R[e] = a + sink;
      continue;
    }
    float p[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) p[i] = w.x * h[i].x + w.y * h[i].y + w.z * h[i].z + w.w * h[i].w;
    const float dot = reduce8(p);
    const float r = v ? dot - a : 0.f;
    if (v) R[e] = r;
    if (MODE == 3) {
      __syncwarp();
      s_r[g][q] = r;
      __syncwarp();
      const float4 r0 = reinterpret_cast<const float4*>(s_r[g])[0];
      const float4 r1 = reinterpret_cast<const float4*>(s_r[g])[1];
      const float rr[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        acc[0] += rr[i] * h[i].x; acc[1] += rr[i] * h[i].y; acc[2] += rr[i] * h[i].z; acc[3] += rr[i] * h[i].w;
      }
    } else {
      sink += r;
    }
  }
  if (sink == 12345.f || acc[0] == 12345.f) out[grp] = sink + acc[1];
}

int main(int argc, char** argv) {
  const int R = 6040, n = 2000000;
  std::vector<int> hidx(n);
  std::mt19937 rng(1);
  std::vector<double> cw(R); double s = 0;
  for (int i = 0; i < R; ++i) { s += 1.0 / (i + 1.0); cw[i] = s; }
  std::uniform_real_distribution<double> d(0, s);
  for (auto& x : hidx) x = std::lower_bound(cw.begin(), cw.end(), d(rng)) - cw.begin();
  // rows: sort indices within runs of 270 (CSR-like)
  for (int i = 0; i + 270 <= n; i += 270) std::sort(hidx.begin() + i, hidx.begin() + i + 270);
  float *T, *W, *val, *Rr, *out; int* idx;
  cudaMalloc(&T, R * 128); cudaMemset(T, 0, R * 128);
  cudaMalloc(&W, 1000 * 128); cudaMemset(W, 0, 1000 * 128);
  cudaMalloc(&idx, n * 4); cudaMemcpy(idx, hidx.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&val, n * 4); cudaMemset(val, 0, n * 4);
  cudaMalloc(&Rr, n * 4); cudaMalloc(&out, 64 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int chunk : {64, 128, 256}) {
    const int groups = (n + chunk - 1) / chunk;
    const int grid = (groups + 31) / 32;
    auto run = [&](auto kern, const char* name) {
      kern<<<grid, 256>>>(T, W, idx, val, Rr, out, n, chunk);
      cudaEventRecord(a);
      for (int i = 0; i < 20; ++i) kern<<<grid, 256>>>(T, W, idx, val, Rr, out, n, chunk);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("chunk %3d %-28s %7.1f us\n", chunk, name, ms / 20 * 1e3);
    };
    run(loop<0>, "gathers+idx");
    run(loop<1>, "+val+Rstore");
    run(loop<2>, "+dot+reduce");
    run(loop<3>, "+acc (full)");
  }
  cudaError_t e = cudaGetLastError(); printf("%s\n", cudaGetErrorString(e));
  return 0;
}
