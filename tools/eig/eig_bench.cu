// syevd vs syevdx (top-k subset) vs syevj at Ritz sizes, fp64.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#define CK(x) do { auto e = (x); if (e != 0) { printf("err %d at %s:%d\n", (int)e, __FILE__, __LINE__); exit(1); } } while (0)
int main() {
  cusolverDnHandle_t h; CK(cusolverDnCreate(&h));
  for (int n : {288, 576, 1024, 1400}) {
    std::vector<double> A(n * n);
    srand(1);
    for (int i = 0; i < n; ++i) for (int j = 0; j <= i; ++j) { double v = rand() / (double)RAND_MAX - 0.5; A[i * n + j] = A[j * n + i] = v; }
    double *dA, *dA0, *dW; int* info;
    CK(cudaMalloc(&dA, sizeof(double) * n * n)); CK(cudaMalloc(&dA0, sizeof(double) * n * n));
    CK(cudaMalloc(&dW, sizeof(double) * n)); CK(cudaMalloc(&info, sizeof(int)));
    CK(cudaMemcpy(dA0, A.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice));
    int lw = 0; CK(cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, &lw));
    int m = 0, lwx = 0;
    int il = n - n / 4 + 1, iu = n;
    CK(cusolverDnDsyevdx_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, dA, n, 0, 0, il, iu, &m, dW, &lwx));
    syevjInfo_t sj; CK(cusolverDnCreateSyevjInfo(&sj)); CK(cusolverDnXsyevjSetTolerance(sj, 1e-14));
    int lwj = 0; CK(cusolverDnDsyevj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, &lwj, sj));
    int lmax = lw > lwx ? lw : lwx; if (lwj > lmax) lmax = lwj;
    double* work; CK(cudaMalloc(&work, sizeof(double) * lmax));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float t[3] = {0, 0, 0};
    for (int rep = 0; rep < 6; ++rep) {
      for (int alg = 0; alg < 3; ++alg) {
        CK(cudaMemcpy(dA, dA0, sizeof(double) * n * n, cudaMemcpyDeviceToDevice));
        cudaDeviceSynchronize(); cudaEventRecord(a);
        if (alg == 0) CK(cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, work, lw, info));
        else if (alg == 1) CK(cusolverDnDsyevdx(h, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, dA, n, 0, 0, il, iu, &m, dW, work, lwx, info));
        else CK(cusolverDnDsyevj(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, work, lwj, info, sj));
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (rep > 0) t[alg] += ms / 5;
      }
    }
    printf("n=%5d syevd %7.2f ms  syevdx(top n/4) %7.2f ms  syevj %7.2f ms\n", n, t[0], t[1], t[2]);
  }
  return 0;
}
