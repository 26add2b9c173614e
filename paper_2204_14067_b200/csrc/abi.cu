// extern "C" entry points of libmfg_b200.so (see include/mfg_b200.h).
#include <mutex>
#include <string>

#include "common.cuh"
#include "engine.cuh"

namespace mfg {

namespace {
thread_local std::string g_err;

template <typename TO, typename TI>
__global__ void k_convert(int64_t n, const TI* __restrict__ in, TO* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (TO)in[i];
}

template <typename T>
__global__ void k_gather(int64_t n, const int32_t* __restrict__ perm, const T* __restrict__ src,
                         T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = src[perm[i]];
}

// 4 entries per thread and iteration: the 4 random loads are in flight together
__global__ void __launch_bounds__(256)
k_gather4_f32(int64_t n4, const int4* __restrict__ perm, const float* __restrict__ src,
              float4* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int4 p = perm[i];
    float4 v;
    v.x = src[p.x]; v.y = src[p.y]; v.z = src[p.z]; v.w = src[p.w];
    out[i] = v;
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
k_dot(int64_t n, const T* __restrict__ x, const T* __restrict__ y, double* __restrict__ bp,
      unsigned int* __restrict__ counter, double* __restrict__ out) {
  __shared__ double sm[8];
  double v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v += (double)x[i] * (double)y[i];
  const double s = block_sum<256>(v, sm);
  if (threadIdx.x == 0) bp[blockIdx.x] = s;
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last) {
    // the last block adds the block partials: each thread a fixed strided
    // subset, then the fixed block tree (deterministic; a single thread
    // walking up to 2368 partials took ~70 us)
    __threadfence();
    const volatile double* b = bp;
    double t = 0.0;
    for (unsigned int i = threadIdx.x; i < gridDim.x; i += 256) t += b[i];
    const double tot = block_sum<256>(t, sm);
    if (threadIdx.x == 0) {
      *out = tot;
      *counter = 0u;
    }
  }
}

inline int grid1(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g < 1) g = 1;
  if (g > kNumSMs * 16) g = kNumSMs * 16;
  return (int)g;
}
}  // namespace

void set_error(const std::string& msg) { g_err = msg; }

}  // namespace mfg

using namespace mfg;

extern "C" const char* mfg_last_error(void) { return g_err.c_str(); }
extern "C" int mfg_version(void) { return 100; }
extern "C" int64_t mfg_launch_count(void) { return g_launches.load(); }

extern "C" int mfg_gather(int dtype, int64_t nnz, const int32_t* perm, const void* src, void* out,
                          void* stream) {
  if (nnz == 0) return MFG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == MFG_F64) {
    k_gather<double><<<grid1(nnz), 256, 0, s>>>(nnz, perm, (const double*)src, (double*)out);
  } else if (((uintptr_t)perm | (uintptr_t)out) % 16 == 0 && nnz >= 4) {
    const int64_t n4 = nnz / 4;
    k_gather4_f32<<<grid1(n4), 256, 0, s>>>(n4, (const int4*)perm, (const float*)src, (float4*)out);
    if (nnz % 4) {
      MFG_LAUNCH_CHECK();
      k_gather<float><<<1, 32, 0, s>>>(nnz % 4, perm + n4 * 4, (const float*)src, (float*)out + n4 * 4);
    }
  } else {
    k_gather<float><<<grid1(nnz), 256, 0, s>>>(nnz, perm, (const float*)src, (float*)out);
  }
  MFG_LAUNCH_CHECK();
  return MFG_OK;
}

extern "C" int mfg_convert(int dtype_out, int dtype_in, int64_t count, const void* src, void* out,
                           void* stream) {
  if (count == 0) return MFG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype_out == MFG_F32 && dtype_in == MFG_F64)
    k_convert<float, double><<<grid1(count), 256, 0, s>>>(count, (const double*)src, (float*)out);
  else if (dtype_out == MFG_F64 && dtype_in == MFG_F32)
    k_convert<double, float><<<grid1(count), 256, 0, s>>>(count, (const float*)src, (double*)out);
  else if (dtype_out == MFG_F64)
    k_convert<double, double><<<grid1(count), 256, 0, s>>>(count, (const double*)src, (double*)out);
  else
    k_convert<float, float><<<grid1(count), 256, 0, s>>>(count, (const float*)src, (float*)out);
  MFG_LAUNCH_CHECK();
  return MFG_OK;
}

extern "C" int mfg_sweep_ld(int dtype, int compute_f64, int k) {
  return sweep_ld(dtype, compute_f64, k);
}

extern "C" size_t mfg_sweep_workspace(const mfg_layout* csr, const mfg_layout* csc, int k) {
  return sweep_workspace(csr, csc, k);
}

extern "C" int mfg_sweep(int dtype, int compute_f64, const mfg_layout* csr, const mfg_layout* csc,
                         int k, const void* vals_csr, const void* vals_csc, const void* W, int ldw,
                         const void* H, int ldh, void* R, void* RH, void* RtW, double out_scale,
                         double* sums, void* workspace, size_t ws_bytes, void* stream) {
  MFG_REQUIRE(csr && csc, "null layout");
  MFG_REQUIRE(k >= 1, "k must be >= 1");
  MFG_REQUIRE(csr->nrows == csc->ncols && csr->ncols == csc->nrows && csr->nnz == csc->nnz,
              "CSR/CSC layouts disagree");
  return sweep_dispatch(dtype, compute_f64, csr, csc, k, vals_csr, vals_csc, W, ldw, H, ldh, R,
                        RH, RtW, out_scale, sums, workspace, ws_bytes, (cudaStream_t)stream);
}

extern "C" int mfg_sweep_sharded(int dtype, int compute_f64, const mfg_layout* rows_csr,
                                 const mfg_layout* cols_csc, int k, const void* vals_rows,
                                 const void* vals_cols, const void* W_rows, const void* W_full,
                                 int ldw, const void* H_cols, const void* H_full, int ldh, void* R,
                                 void* RH, void* RtW, double out_scale, double* sums,
                                 void* workspace, size_t ws_bytes, void* stream) {
  MFG_REQUIRE(rows_csr && cols_csc, "null layout");
  MFG_REQUIRE(k >= 1, "k must be >= 1");
  MFG_REQUIRE(W_rows && W_full && H_cols && H_full, "null factor");
  MFG_REQUIRE(rows_csr->ncols >= cols_csc->nrows && cols_csc->ncols >= rows_csr->nrows,
              "shard layouts do not fit the factor replicas");
  return sweep_dispatch(dtype, compute_f64, rows_csr, cols_csc, k, vals_rows, vals_cols, W_rows,
                        ldw, H_cols, ldh, R, RH, RtW, out_scale, sums, workspace, ws_bytes,
                        (cudaStream_t)stream, W_full, H_full);
}

extern "C" int mfg_sweep_host(int dtype, int compute_f64, const mfg_layout* csr,
                              const mfg_layout* csc, int k, const void* vals_csr,
                              const void* vals_csc, const void* W_host, const void* H_host,
                              void* W, int ldw, void* H, int ldh, void* R, void* out,
                              void* out_host, double out_scale, void* workspace, size_t ws_bytes,
                              void* stream) {
  MFG_REQUIRE(csr && csc, "null layout");
  MFG_REQUIRE(W_host && H_host && W && H && out, "null buffer");
  MFG_REQUIRE(k >= 1 && ldw >= k && ldh >= k, "need k >= 1 and ldw, ldh >= k");
  MFG_REQUIRE(dtype == MFG_F32 || dtype == MFG_F64, "dtype must be MFG_F32 or MFG_F64");
  const size_t es = dtype == MFG_F32 ? 4 : 8;
  const cudaStream_t st = (cudaStream_t)stream;
  const size_t m = (size_t)csr->nrows, n = (size_t)csc->nrows;
  auto h2d = [&](void* dst, int ld, const void* src, size_t rows) -> cudaError_t {
    if (rows == 0) return cudaSuccess;
    if ((size_t)ld == (size_t)k)
      return cudaMemcpyAsync(dst, src, rows * k * es, cudaMemcpyHostToDevice, st);
    return cudaMemcpy2DAsync(dst, ld * es, src, k * es, k * es, rows, cudaMemcpyHostToDevice, st);
  };
  // W and H adjacent on both sides (SweepPlan.pinned_factors): one copy
  if ((size_t)ldw == (size_t)k && (size_t)ldh == (size_t)k &&
      static_cast<const char*>(H_host) == static_cast<const char*>(W_host) + m * k * es &&
      static_cast<char*>(H) == static_cast<char*>(W) + m * k * es) {
    if (m + n) MFG_CUDA_CHECK(cudaMemcpyAsync(W, W_host, (m + n) * k * es, cudaMemcpyHostToDevice, st));
  } else {
    MFG_CUDA_CHECK(h2d(W, ldw, W_host, m));
    MFG_CUDA_CHECK(h2d(H, ldh, H_host, n));
  }
  char* o = static_cast<char*>(out);
  const int rc = mfg_sweep(dtype, compute_f64, csr, csc, k, vals_csr, vals_csc, W, ldw, H, ldh, R,
                           o + 32, o + 32 + m * k * es, out_scale, reinterpret_cast<double*>(o),
                           workspace, ws_bytes, stream);
  if (rc != MFG_OK) return rc;
  if (out_host)
    MFG_CUDA_CHECK(cudaMemcpyAsync(out_host, out, 32 + (m + n) * k * es, cudaMemcpyDeviceToHost, st));
  return MFG_OK;
}

extern "C" size_t mfg_sddmm_workspace(const mfg_layout* lay, int k) {
  return sddmm_workspace(lay, k);
}

extern "C" int mfg_sddmm(int dtype, int compute_f64, const mfg_layout* lay, int k, const void* L,
                         int ldl, const double* scale, const void* Rt, int ldr, const void* A,
                         const void* G, double out_mult, void* out, double* sums, void* workspace,
                         size_t ws_bytes, void* stream) {
  MFG_REQUIRE(lay, "null layout");
  MFG_REQUIRE(k >= 0, "k must be >= 0");
  if (k == 0) {
    // p = 0: r = -A
    k = 0;
  }
  return sddmm_dispatch(dtype, compute_f64, lay, k, L, ldl, scale, Rt, ldr, A, G, out_mult, out,
                        sums, workspace, ws_bytes, (cudaStream_t)stream);
}

extern "C" size_t mfg_spmm_workspace(const mfg_layout* lay, int p) {
  return spmm_workspace(lay, p);
}

extern "C" int mfg_spmm(int dtype, const mfg_layout* lay, int p, const void* vals, const void* X,
                        int ldx, double alpha, double beta, void* Y, int ldy, void* workspace,
                        size_t ws_bytes, void* stream) {
  MFG_REQUIRE(lay, "null layout");
  MFG_REQUIRE(p >= 0, "p must be >= 0");
  return spmm_dispatch(dtype, lay, p, vals, X, ldx, alpha, beta, Y, ldy, workspace, ws_bytes,
                       (cudaStream_t)stream);
}

extern "C" size_t mfg_bcd_workspace(const mfg_layout* lay, int k) {
  return bcd_workspace(lay, k);
}

extern "C" int mfg_bcd_half_sweep(int dtype, const mfg_layout* lay, int k, const void* vals,
                                  const void* other, int ldo, double lam, void* out, int ldout,
                                  void* workspace, size_t ws_bytes, void* stream) {
  MFG_REQUIRE(lay, "null layout");
  MFG_REQUIRE(lam > 0.0, "lam must be positive");
  return bcd_dispatch(dtype, lay, k, vals, other, ldo, lam, out, ldout, workspace, ws_bytes,
                      (cudaStream_t)stream);
}

extern "C" size_t mfg_gemm_tn_workspace(int m, int p, int q) { return gemm_tn_workspace(m, p, q); }

extern "C" int mfg_gemm_tn(int m, int p, int q, const double* A, int lda, const double* B, int ldb,
                           double alpha, double* C, int ldc, void* workspace, size_t ws_bytes,
                           void* stream) {
  return gemm_tn(m, p, q, A, lda, B, ldb, alpha, C, ldc, workspace, ws_bytes, (cudaStream_t)stream);
}

extern "C" int mfg_gemm_nn(int m, int p, int q, const double* A, int lda, const double* B, int ldb,
                           double alpha, double beta, double* C, int ldc, void* stream) {
  return gemm_nn(m, p, q, A, lda, B, ldb, alpha, beta, C, ldc, (cudaStream_t)stream);
}

extern "C" size_t mfg_qr_workspace(int m, int p) { return qr_workspace(m, p); }

extern "C" int mfg_qr(int m, int p, const double* B, int ldb, double* Q, int ldq, double* diag,
                      void* workspace, size_t ws_bytes, void* stream) {
  return qr_factor(m, p, B, ldb, Q, ldq, diag, workspace, ws_bytes, (cudaStream_t)stream);
}

extern "C" int mfg_bcd_status(const void* workspace, int* flag_host, void* stream) {
  MFG_REQUIRE(workspace && flag_host, "null workspace or flag");
  // the half-sweep's non-SPD flag is the workspace's first word (bcd.cu do_bcd)
  MFG_CUDA_CHECK(cudaMemcpyAsync(flag_host, workspace, sizeof(int), cudaMemcpyDeviceToHost,
                                 (cudaStream_t)stream));
  return MFG_OK;
}

extern "C" int mfg_dot(int dtype, int64_t count, const void* x, const void* y, double* out,
                       void* workspace, size_t ws_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  Carver c(workspace, ws_bytes);
  const int g = grid1(count);
  double* bp = c.take<double>(g);
  unsigned int* counter = c.take<unsigned int>(1);
  MFG_REQUIRE(c.ok, "dot workspace too small (needs 64 KiB)");
  MFG_CUDA_CHECK(cudaMemsetAsync(counter, 0, sizeof(unsigned int), s));
  if (dtype == MFG_F64)
    k_dot<double><<<g, 256, 0, s>>>(count, (const double*)x, (const double*)y, bp, counter, out);
  else
    k_dot<float><<<g, 256, 0, s>>>(count, (const float*)x, (const float*)y, bp, counter, out);
  MFG_LAUNCH_CHECK();
  return MFG_OK;
}
