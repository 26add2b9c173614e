// Calibration microbenchmark: throughput of random row gathers on B200.
// Table of R rows x 32 fp32 (128 B rows); N random row indices; variants:
//   G=8 lanes per row (one LDG.128 per lane), U rows in flight per group;
//   G=32 lanes per row (LDG.32); sum into a register, write one float per group.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include <cmath>
#include <cuda_runtime.h>

template <int U>
__global__ void g8(const float* __restrict__ T, const int* __restrict__ idx, int n, float* out) {
  const int q = threadIdx.x & 7;
  const int grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int ngrp = (gridDim.x * blockDim.x) >> 3;
  float acc = 0.f;
  for (int base = grp * U; base < n; base += ngrp * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = (base + u < n) ? idx[base + u] : 0;
      v[u] = reinterpret_cast<const float4*>(T + (size_t)j * 32)[q];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 12345.f) out[grp] = acc;
}

template <int U>
__global__ void g32(const float* __restrict__ T, const int* __restrict__ idx, int n, float* out) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (int base = w * U; base < n; base += nw * U) {
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = (base + u < n) ? idx[base + u] : 0;
      v[u] = T[(size_t)j * 32 + lane];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 12345.f) out[w] = acc;
}

template <typename K>
float timeit(K kern, int grid, int block, const float* T, const int* idx, int n, float* out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  kern<<<grid, block>>>(T, idx, n, out);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) kern<<<grid, block>>>(T, idx, n, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 10;
}

int main(int argc, char** argv) {
  const int R = argc > 1 ? atoi(argv[1]) : 6040;
  const int n = argc > 2 ? atoi(argv[2]) : 2000000;
  const double zipf = argc > 3 ? atof(argv[3]) : 0.0;
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
  cudaMalloc(&T, (size_t)R * 128); cudaMemset(T, 0, (size_t)R * 128);
  cudaMalloc(&idx, (size_t)n * 4); cudaMemcpy(idx, h.data(), (size_t)n * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&out, 64 << 20);
  const double bytes = (double)n * 128;
  printf("R=%d n=%d zipf=%.2f table=%.1f MB\n", R, n, zipf, R * 128 / 1e6);
  for (int wps : {8, 16, 32, 64}) {
    const int grid = 148 * wps / 8;  // blocks of 256 threads
    float t;
    t = timeit(g8<4>, grid, 256, T, idx, n, out);  printf("warps/SM %2d g8  U=4 : %7.1f us %7.1f GB/s\n", wps, t * 1e3, bytes / t / 1e6);
    t = timeit(g8<8>, grid, 256, T, idx, n, out);  printf("warps/SM %2d g8  U=8 : %7.1f us %7.1f GB/s\n", wps, t * 1e3, bytes / t / 1e6);
    t = timeit(g8<16>, grid, 256, T, idx, n, out); printf("warps/SM %2d g8  U=16: %7.1f us %7.1f GB/s\n", wps, t * 1e3, bytes / t / 1e6);
    t = timeit(g32<8>, grid, 256, T, idx, n, out); printf("warps/SM %2d g32 U=8 : %7.1f us %7.1f GB/s\n", wps, t * 1e3, bytes / t / 1e6);
    t = timeit(g32<32>, grid, 256, T, idx, n, out); printf("warps/SM %2d g32 U=32: %7.1f us %7.1f GB/s\n", wps, t * 1e3, bytes / t / 1e6);
  }
  return 0;
}
