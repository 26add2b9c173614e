// Internal dispatch entry points shared between the kernel files and abi.cu.
#pragma once

#include <cuda_runtime.h>

#include "../../include/mfg_b200.h"

namespace mfg {

size_t sweep_workspace(const mfg_layout* csr, const mfg_layout* csc, int k);
int sweep_dispatch(int dtype, int compute_f64, const mfg_layout* csr, const mfg_layout* csc,
                   int k, const void* vals_csr, const void* vals_csc, const void* W, int ldw,
                   const void* H, int ldh, void* R, void* RH, void* RtW, double out_scale,
                   double* sums, void* ws, size_t wsb, cudaStream_t stream,
                   const void* Wg = nullptr, const void* Hg = nullptr);

size_t sddmm_workspace(const mfg_layout* lay, int k);
int sweep_ld(int dtype, int compute_f64, int k);
size_t gemm_tn_workspace(int m, int p, int q);
int gemm_tn(int m, int p, int q, const double* A, int lda, const double* B, int ldb, double alpha,
            double* C, int ldc, void* ws, size_t wsb, cudaStream_t stream);
int gemm_nn(int m, int p, int q, const double* A, int lda, const double* B, int ldb, double alpha,
            double beta, double* C, int ldc, cudaStream_t stream, const double* Cin = nullptr,
            int ldcin = 0);
size_t qr_workspace(int m, int p);
int qr_factor(int m, int p, const double* B, int ldb, double* Q, int ldq, double* diag, void* ws,
              size_t wsb, cudaStream_t stream);
int sddmm_dispatch(int dtype, int compute_f64, const mfg_layout* lay, int k, const void* L,
                   int ldl, const double* scale, const void* Rt, int ldr, const void* A,
                   const void* G, double out_mult, void* out, double* sums, void* ws, size_t wsb,
                   cudaStream_t stream);

size_t spmm_workspace(const mfg_layout* lay, int p);
int spmm_dispatch(int dtype, const mfg_layout* lay, int p, const void* vals, const void* X,
                  int ldx, double alpha, double beta, void* Y, int ldy, void* ws, size_t wsb,
                  cudaStream_t stream);

size_t bcd_workspace(const mfg_layout* lay, int k);
int bcd_dispatch(int dtype, const mfg_layout* lay, int k, const void* vals, const void* other,
                 int ldo, double lam, void* out, int ldout, void* ws, size_t wsb,
                 cudaStream_t stream);

// CUDA-event timing of the dominant kernel(s) (mfg_profile_enable)
void prof_begin(cudaStream_t s);
void prof_end(cudaStream_t s);

}  // namespace mfg
