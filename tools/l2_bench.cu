// L2 -> SM read bandwidth microbenchmark (DESIGN.md §3 bound table).
//
// Every CTA streams its slice of a buffer of S bytes with 16-byte loads, R
// times; for S well below the 126 MB L2 the bytes come from L2 (L1 is
// bypassed with ld.global.cg so they are not L1 hits), for S far above it
// from HBM. Reported: bytes delivered to the SMs / kernel time (CUDA events,
// best of 5), for several sizes and CTA counts.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_bench tools/l2_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) k_read(const int4* __restrict__ p, size_t n16, int reps,
                                              int* out) {
  int4 acc = make_int4(0, 0, 0, 0);
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t nth = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    // rotate the start per rep so a CTA does not re-read its own (L1) lines
    const size_t off = (tid + (size_t)r * 7919 * 32) % n16;
#pragma unroll 4
    for (size_t i = 0; i < n16; i += nth) {
      size_t j = off + i;
      if (j >= n16) j -= n16;
      int4 v;
      asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "l"(p + j));
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x7fffffff) out[0] = 1;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const size_t big = (size_t)4 << 30;
  char* buf;
  int* out;
  cudaMalloc(&buf, big);
  cudaMalloc(&out, 4);
  cudaMemset(buf, 1, big);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  printf("{\"sms\": %d, \"clock_khz\": %d, \"runs\": [\n", sms, clk);
  const size_t sizes[] = {(size_t)8 << 20, (size_t)24 << 20, (size_t)48 << 20, (size_t)80 << 20,
                          (size_t)2 << 30};
  bool first = true;
  for (size_t S : sizes) {
    for (int per_sm : {2, 4, 8}) {
      const int threads = 512;
      const int grid = sms * per_sm / 2;  // 512-thread CTAs, per_sm/2 CTAs per SM
      const size_t n16 = S / 16;
      const size_t target = (size_t)16 << 30;  // ~16 GB moved per launch
      int reps = (int)(target / S);
      if (reps < 1) reps = 1;
      k_read<<<grid, threads>>>((const int4*)buf, n16, 1, out);
      cudaDeviceSynchronize();
      float best = 1e30f;
      for (int t = 0; t < 5; ++t) {
        cudaEventRecord(a);
        k_read<<<grid, threads>>>((const int4*)buf, n16, reps, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      const double bytes = (double)S * reps;
      printf("%s  {\"bytes_buffer\": %zu, \"warps_per_sm\": %d, \"GBps\": %.1f, \"B_per_sm_clk\": %.1f}",
             first ? "" : ",\n", S, per_sm * 8, bytes / (best * 1e-3) / 1e9,
             bytes / (best * 1e-3) / (clk * 1e3) / sms);
      first = false;
    }
  }
  printf("\n]}\n");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "%s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
