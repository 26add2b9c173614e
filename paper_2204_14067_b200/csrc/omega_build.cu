// Omega build on the device: validation, (row, col) sort, duplicate
// rejection, CSR pointers, CSC view, and the flat-chunk scheduling metadata.
//
// Replaces ObservationSet.from_coo (mfg/data.py:70-102) and the scipy
// transposes a_csr_t / csr_t (mfg/data.py:113-119, 156-158). The sort is a
// CUB LSD radix sort of the 64-bit key row*n+col; with no duplicates the
// sorted order is unique, so the result is bit-identical to np.lexsort. The
// CSC permutation is a *stable* radix sort of the sorted column indices, so
// rows stay ascending inside each column exactly like scipy's csr_tocsc.
#include <cub/cub.cuh>

#include "common.cuh"

namespace mfg {

namespace {

__global__ void k_range_and_keys(int64_t nnz, int32_t m, int32_t n,
                                 const int64_t* __restrict__ rows,
                                 const int64_t* __restrict__ cols,
                                 uint64_t* __restrict__ keys,
                                 int32_t* __restrict__ iota,
                                 int32_t* __restrict__ flags) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rows[e], c = cols[e];
    bool bad = false;
    if (r < 0 || r >= m) { atomicOr(&flags[0], 1); bad = true; }
    if (c < 0 || c >= n) { atomicOr(&flags[1], 1); bad = true; }
    keys[e] = bad ? 0ull : (uint64_t)r * (uint64_t)n + (uint64_t)c;
    iota[e] = (int32_t)e;
  }
}

__global__ void k_dups_and_split(int64_t nnz, int32_t n,
                                 const uint64_t* __restrict__ keys,
                                 const int32_t* __restrict__ order,
                                 const double* __restrict__ vals_in,
                                 int32_t* __restrict__ rows_out,
                                 int32_t* __restrict__ cols_out,
                                 double* __restrict__ vals_out,
                                 unsigned long long* __restrict__ dup_min) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = keys[e];
    rows_out[e] = (int32_t)(key / (uint64_t)n);
    cols_out[e] = (int32_t)(key % (uint64_t)n);
    vals_out[e] = vals_in[order[e]];
    if (e + 1 < nnz && keys[e + 1] == key) atomicMin(dup_min, (unsigned long long)e);
  }
}

// ptr[q] = first e with row_of[e] >= q (row_of sorted ascending).
__global__ void k_pointers(int64_t nnz, int32_t nrows,
                           const int32_t* __restrict__ row_of,
                           int32_t* __restrict__ ptr) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e <= nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t prev = e == 0 ? -1 : row_of[e - 1];
    const int32_t cur = e == nnz ? nrows : row_of[e];
    for (int32_t q = prev + 1; q <= cur; ++q) ptr[q] = (int32_t)e;
  }
}

__global__ void k_gather_i32(int64_t nnz, const int32_t* __restrict__ perm,
                             const int32_t* __restrict__ src,
                             int32_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = src[perm[e]];
}

__global__ void k_iota(int64_t nnz, int32_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = (int32_t)e;
}

__global__ void k_nonempty_flags(int32_t nrows, const int32_t* __restrict__ ptr,
                                 int32_t* __restrict__ flag) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nrows;
       i += gridDim.x * blockDim.x)
    flag[i] = ptr[i + 1] > ptr[i] ? 1 : 0;
}

__global__ void k_rank_lists(int32_t nrows, const int32_t* __restrict__ flag,
                             const int32_t* __restrict__ rank,
                             int32_t* __restrict__ nzrows,
                             int32_t* __restrict__ empty_rows,
                             int32_t* __restrict__ counts) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nrows;
       i += gridDim.x * blockDim.x) {
    if (flag[i]) nzrows[rank[i]] = i;
    else empty_rows[i - rank[i]] = i;
    if (i == nrows - 1) {
      counts[0] = rank[i] + flag[i];
      counts[1] = nrows - counts[0];
    }
  }
}

// one warp per 32-entry batch
__global__ void k_batches(int64_t nnz, const int32_t* __restrict__ row_of,
                          const int32_t* __restrict__ rank_of_row,
                          uint32_t* __restrict__ bmask,
                          int32_t* __restrict__ brank) {
  const int64_t nb = (nnz + 31) / 32;
  const int lane = threadIdx.x & 31;
  for (int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; b < nb;
       b += (int64_t)gridDim.x * blockDim.x / 32) {
    const int64_t e = b * 32 + lane;
    bool start = false;
    int32_t r = 0;
    if (e < nnz) {
      r = row_of[e];
      start = (e == 0) || (row_of[e - 1] != r);
    }
    const uint32_t mask = __ballot_sync(0xffffffffu, start);
    if (lane == 0) {
      bmask[b] = mask;
      brank[b] = rank_of_row[r];
    }
  }
}

inline int grid_for(int64_t n, int nt = 256) {
  int64_t g = (n + nt - 1) / nt;
  if (g < 1) g = 1;
  if (g > kNumSMs * 32) g = kNumSMs * 32;
  return (int)g;
}

int end_bit_for(uint64_t maxval) {
  int b = 1;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

size_t cub_pairs_u64(int64_t nnz) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (int32_t*)nullptr, (int32_t*)nullptr, (int)nnz, 0, 64);
  return bytes;
}
size_t cub_pairs_i32(int64_t nnz) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (int32_t*)nullptr, (int32_t*)nullptr,
                                  (int32_t*)nullptr, (int32_t*)nullptr, (int)nnz, 0, 32);
  return bytes;
}
size_t cub_scan_i32(int32_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  return bytes;
}

template <typename C>
void carve_build(C& c, int64_t nnz, int32_t m, int32_t n) {
  const int64_t nz = nnz > 0 ? nnz : 1;
  c.template take<uint64_t>(nz);             // keys
  c.template take<uint64_t>(nz);             // keys sorted
  c.template take<int32_t>(nz);              // iota
  c.template take<int32_t>(nz);              // order
  c.template take<int32_t>(4);               // flags
  c.template take<unsigned long long>(1);    // dup min
  size_t t = cub_pairs_u64(nz);
  size_t t2 = cub_pairs_i32(nz);
  c.template take<char>(t > t2 ? t : t2);    // cub temp
}

template <typename C>
void carve_layout(C& c, int64_t nnz, int32_t nrows) {
  const int32_t nr = nrows > 0 ? nrows : 1;
  c.template take<int32_t>(nr);  // flags
  c.template take<int32_t>(nr);  // ranks
  c.template take<int32_t>(2);   // counts
  c.template take<char>(cub_scan_i32(nr));
}

}  // namespace

}  // namespace mfg

using namespace mfg;

extern "C" size_t mfg_omega_build_workspace(int64_t nnz, int32_t m, int32_t n) {
  Sizer s;
  carve_build(s, nnz, m, n);
  return s.off;
}

extern "C" int mfg_omega_build(int32_t m, int32_t n, int64_t nnz,
                               const int64_t* rows_in, const int64_t* cols_in,
                               const double* vals_in, int32_t* rows_out,
                               int32_t* cols_out, double* vals_out, int32_t* ptr,
                               int32_t* csc_ptr, int32_t* csc_rows,
                               int32_t* csc_cols, int32_t* csc_perm,
                               int64_t* dup_pos_host, int32_t* range_err_host,
                               void* workspace, size_t ws_bytes, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (dup_pos_host) *dup_pos_host = -1;
  if (range_err_host) *range_err_host = 0;
  MFG_REQUIRE(m >= 0 && n >= 0 && nnz >= 0, "negative dimension");
  if (nnz >= (int64_t)INT32_MAX) {
    set_error("|Omega| >= 2^31 is not supported by the int32 index layout");
    return MFG_ERR_CAPACITY;
  }
  Carver c(workspace, ws_bytes);
  const int64_t nz = nnz > 0 ? nnz : 1;
  uint64_t* keys = c.take<uint64_t>(nz);
  uint64_t* keys_s = c.take<uint64_t>(nz);
  int32_t* iota = c.take<int32_t>(nz);
  int32_t* order = c.take<int32_t>(nz);
  int32_t* flags = c.take<int32_t>(4);
  unsigned long long* dmin = c.take<unsigned long long>(1);
  size_t t1 = cub_pairs_u64(nz), t2 = cub_pairs_i32(nz);
  size_t tbytes = t1 > t2 ? t1 : t2;
  char* temp = c.take<char>(tbytes);
  MFG_REQUIRE(c.ok, "omega build workspace too small");

  if (nnz == 0) {
    MFG_CUDA_CHECK(cudaMemsetAsync(ptr, 0, sizeof(int32_t) * (m + 1), stream));
    MFG_CUDA_CHECK(cudaMemsetAsync(csc_ptr, 0, sizeof(int32_t) * (n + 1), stream));
    return MFG_OK;
  }
  MFG_CUDA_CHECK(cudaMemsetAsync(flags, 0, sizeof(int32_t) * 4, stream));
  MFG_CUDA_CHECK(cudaMemsetAsync(dmin, 0xff, sizeof(unsigned long long), stream));
  const int g = grid_for(nnz);
  k_range_and_keys<<<g, 256, 0, stream>>>(nnz, m, n, rows_in, cols_in, keys, iota, flags);
  MFG_LAUNCH_CHECK();
  int32_t hflags[2] = {0, 0};
  MFG_CUDA_CHECK(cudaMemcpyAsync(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost, stream));
  MFG_CUDA_CHECK(cudaStreamSynchronize(stream));
  if (hflags[0] || hflags[1]) {
    if (range_err_host) *range_err_host = hflags[0] ? 1 : 2;
    set_error(hflags[0] ? "row index out of range" : "column index out of range");
    return MFG_ERR_DATASET;
  }
  const int ebits = end_bit_for((uint64_t)m * (uint64_t)n - 1);
  size_t tb = tbytes;
  MFG_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(temp, tb, keys, keys_s, iota, order, (int)nnz,
                                                 0, ebits, stream));
  g_launches.fetch_add(1);
  k_dups_and_split<<<g, 256, 0, stream>>>(nnz, n, keys_s, order, vals_in, rows_out, cols_out,
                                          vals_out, dmin);
  MFG_LAUNCH_CHECK();
  unsigned long long hd = 0;
  MFG_CUDA_CHECK(cudaMemcpyAsync(&hd, dmin, sizeof(hd), cudaMemcpyDeviceToHost, stream));
  MFG_CUDA_CHECK(cudaStreamSynchronize(stream));
  if (hd != ~0ull) {
    if (dup_pos_host) *dup_pos_host = (int64_t)hd;
    set_error("duplicate entry");
    return MFG_ERR_DATASET;
  }
  k_pointers<<<grid_for(nnz + 1), 256, 0, stream>>>(nnz, m, rows_out, ptr);
  MFG_LAUNCH_CHECK();
  // CSC: stable sort of the (row-major sorted) column indices.
  k_iota<<<g, 256, 0, stream>>>(nnz, iota);
  MFG_LAUNCH_CHECK();
  const int cbits = end_bit_for(n > 0 ? (uint64_t)(n - 1) : 0);
  tb = tbytes;
  MFG_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(temp, tb, cols_out, csc_cols, iota, csc_perm,
                                                 (int)nnz, 0, cbits, stream));
  g_launches.fetch_add(1);
  k_gather_i32<<<g, 256, 0, stream>>>(nnz, csc_perm, rows_out, csc_rows);
  MFG_LAUNCH_CHECK();
  k_pointers<<<grid_for(nnz + 1), 256, 0, stream>>>(nnz, n, csc_cols, csc_ptr);
  MFG_LAUNCH_CHECK();
  return MFG_OK;
}

extern "C" size_t mfg_layout_workspace(int64_t nnz, int32_t nrows) {
  Sizer s;
  carve_layout(s, nnz, nrows);
  return s.off;
}

extern "C" int mfg_layout_build(int32_t nrows, int64_t nnz, const int32_t* ptr,
                                const int32_t* row_of, uint32_t* bmask, int32_t* brank,
                                int32_t* nzrows, int32_t* empty_rows,
                                int32_t* n_nonempty_host, int32_t* n_empty_host,
                                void* workspace, size_t ws_bytes, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (nrows == 0) {
    *n_nonempty_host = 0;
    *n_empty_host = 0;
    return MFG_OK;
  }
  Carver c(workspace, ws_bytes);
  int32_t* flag = c.take<int32_t>(nrows);
  int32_t* rank = c.take<int32_t>(nrows);
  int32_t* counts = c.take<int32_t>(2);
  size_t tb = cub_scan_i32(nrows);
  char* temp = c.take<char>(tb);
  MFG_REQUIRE(c.ok, "layout workspace too small");
  k_nonempty_flags<<<grid_for(nrows), 256, 0, stream>>>(nrows, ptr, flag);
  MFG_LAUNCH_CHECK();
  MFG_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(temp, tb, flag, rank, (int)nrows, stream));
  g_launches.fetch_add(1);
  k_rank_lists<<<grid_for(nrows), 256, 0, stream>>>(nrows, flag, rank, nzrows, empty_rows, counts);
  MFG_LAUNCH_CHECK();
  if (nnz > 0) {
    const int64_t nb = (nnz + 31) / 32;
    k_batches<<<grid_for(nb * 32), 256, 0, stream>>>(nnz, row_of, rank, bmask, brank);
    MFG_LAUNCH_CHECK();
  }
  int32_t hc[2];
  MFG_CUDA_CHECK(cudaMemcpyAsync(hc, counts, sizeof(hc), cudaMemcpyDeviceToHost, stream));
  MFG_CUDA_CHECK(cudaStreamSynchronize(stream));
  *n_nonempty_host = hc[0];
  *n_empty_host = hc[1];
  return MFG_OK;
}
