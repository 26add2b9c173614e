/* A pure C client of libmfg_b200 (no Python, no torch): what a reference-side
 * caller binding the C ABI does. Builds Omega from COO on the device, builds
 * both layouts' scheduling metadata, runs one fp64 sweep (mfg_sweep) and one
 * end-to-end sweep from host factors (mfg_sweep_host), and checks R, R.H,
 * R^T.W and sum r^2 against a direct host computation. Exit code 0 = pass.
 * Built and run by tests/test_abi_client.py (gpu). */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "../include/mfg_b200.h"

#define CK(x)                                                                     \
  do {                                                                            \
    int _s = (int)(x);                                                            \
    if (_s) {                                                                     \
      fprintf(stderr, "%s failed (%d): %s\n", #x, _s, mfg_last_error());          \
      return 1;                                                                   \
    }                                                                             \
  } while (0)
#define CU(x)                                                                     \
  do {                                                                            \
    cudaError_t _e = (x);                                                         \
    if (_e != cudaSuccess) {                                                      \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(_e));                    \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

static void* dalloc(size_t bytes) {
  void* p = NULL;
  if (cudaMalloc(&p, bytes ? bytes : 16) != cudaSuccess) return NULL;
  cudaMemset(p, 0, bytes ? bytes : 16);
  return p;
}

static double urand(unsigned long long* s) {
  *s = *s * 6364136223846793005ULL + 1442695040888963407ULL;
  return (double)((*s >> 11) & ((1ULL << 53) - 1)) / (double)(1ULL << 53);
}

static int build_layout(mfg_layout* L, int32_t nrows, int32_t ncols, int64_t nnz,
                        const int32_t* ptr, const int32_t* idx, const int32_t* row_of) {
  const int64_t nb = (nnz + 31) / 32 > 0 ? (nnz + 31) / 32 : 1;
  uint32_t* bmask = dalloc(nb * 4);
  int32_t* brank = dalloc(nb * 4);
  int32_t* nzrows = dalloc((nrows > 0 ? nrows : 1) * 4);
  int32_t* empty = dalloc((nrows > 0 ? nrows : 1) * 4);
  size_t wsb = mfg_layout_workspace(nnz, nrows);
  void* ws = dalloc(wsb);
  int32_t nne = 0, ne = 0;
  CK(mfg_layout_build(nrows, nnz, ptr, row_of, bmask, brank, nzrows, empty, &nne, &ne, ws, wsb,
                      NULL));
  CU(cudaDeviceSynchronize());
  memset(L, 0, sizeof(*L));
  L->nrows = nrows; L->ncols = ncols; L->nnz = nnz; L->ptr = ptr; L->idx = idx;
  L->row_of = row_of; L->bmask = bmask; L->brank = brank; L->nzrows = nzrows;
  L->n_nonempty = nne; L->empty_rows = empty; L->n_empty = ne;
  return 0;
}

int main(void) {
  const int32_t m = 97, n = 131, k = 8;
  unsigned long long seed = 12345;
  /* COO with ~30% density, unsorted, no duplicates */
  int64_t cap = (int64_t)m * n, nnz = 0;
  int64_t* rows = malloc(cap * 8);
  int64_t* cols = malloc(cap * 8);
  double* vals = malloc(cap * 8);
  for (int32_t j = n - 1; j >= 0; --j)
    for (int32_t i = 0; i < m; ++i)
      if (urand(&seed) < 0.3) { rows[nnz] = i; cols[nnz] = j; vals[nnz] = 5.0 * urand(&seed); ++nnz; }
  double* w = malloc((size_t)m * k * 8);
  double* h = malloc((size_t)n * k * 8);
  for (int64_t t = 0; t < (int64_t)m * k; ++t) w[t] = urand(&seed) - 0.5;
  for (int64_t t = 0; t < (int64_t)n * k; ++t) h[t] = urand(&seed) - 0.5;

  /* Omega build (device sort, dedupe, CSR + CSC) */
  int64_t *d_rin = dalloc(nnz * 8), *d_cin = dalloc(nnz * 8);
  double* d_vin = dalloc(nnz * 8);
  CU(cudaMemcpy(d_rin, rows, nnz * 8, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_cin, cols, nnz * 8, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_vin, vals, nnz * 8, cudaMemcpyHostToDevice));
  const int64_t pad = nnz + 64; /* entry streams are read up to 64 past nnz */
  int32_t *r_out = dalloc(pad * 4), *c_out = dalloc(pad * 4), *ptr = dalloc((m + 1) * 4);
  double* v_out = dalloc(pad * 8);
  int32_t *cptr = dalloc((n + 1) * 4), *crows = dalloc(pad * 4), *ccols = dalloc(pad * 4);
  int32_t* cperm = dalloc(pad * 4);
  size_t wsb = mfg_omega_build_workspace(nnz, m, n);
  void* ws = dalloc(wsb);
  int64_t dup = -1;
  int32_t rerr = 0;
  CK(mfg_omega_build(m, n, nnz, d_rin, d_cin, d_vin, r_out, c_out, v_out, ptr, cptr, crows, ccols,
                     cperm, &dup, &rerr, ws, wsb, NULL));
  double* v_csc = dalloc(pad * 8);
  CK(mfg_gather(MFG_F64, nnz, cperm, v_out, v_csc, NULL));
  mfg_layout csr, csc;
  if (build_layout(&csr, m, n, nnz, ptr, c_out, r_out)) return 1;
  if (build_layout(&csc, n, m, nnz, cptr, crows, ccols)) return 1;

  /* one sweep from device factors */
  double *dw = dalloc((size_t)m * k * 8), *dh = dalloc((size_t)n * k * 8);
  CU(cudaMemcpy(dw, w, (size_t)m * k * 8, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(dh, h, (size_t)n * k * 8, cudaMemcpyHostToDevice));
  double *dR = dalloc(nnz * 8), *dRH = dalloc((size_t)m * k * 8), *dRtW = dalloc((size_t)n * k * 8);
  double* dsums = dalloc(3 * 8);
  size_t swb = mfg_sweep_workspace(&csr, &csc, k);
  void* sws = dalloc(swb);
  CK(mfg_sweep(MFG_F64, 0, &csr, &csc, k, v_out, v_csc, dw, k, dh, k, dR, dRH, dRtW, 1.0, dsums,
               sws, swb, NULL));
  CU(cudaDeviceSynchronize());

  /* host reference: R in (row, col) order, R.H, R^T.W, sum r^2 */
  int32_t* hr = malloc(nnz * 4);
  int32_t* hc = malloc(nnz * 4);
  double* hv = malloc(nnz * 8);
  double* R = malloc(nnz * 8);
  double* RH = calloc((size_t)m * k, 8);
  double* RtW = calloc((size_t)n * k, 8);
  double sums[3];
  CU(cudaMemcpy(hr, r_out, nnz * 4, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(hc, c_out, nnz * 4, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(hv, v_out, nnz * 8, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(R, dR, nnz * 8, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(sums, dsums, 24, cudaMemcpyDeviceToHost));
  double* gRH = malloc((size_t)m * k * 8);
  double* gRtW = malloc((size_t)n * k * 8);
  CU(cudaMemcpy(gRH, dRH, (size_t)m * k * 8, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(gRtW, dRtW, (size_t)n * k * 8, cudaMemcpyDeviceToHost));
  double sq = 0.0, err = 0.0;
  for (int64_t e = 0; e < nnz; ++e) {
    if (e > 0 && ((int64_t)hr[e] * n + hc[e]) <= ((int64_t)hr[e - 1] * n + hc[e - 1])) {
      fprintf(stderr, "CSR not sorted at %lld\n", (long long)e);
      return 1;
    }
    double p = 0.0;
    for (int d = 0; d < k; ++d) p += w[(size_t)hr[e] * k + d] * h[(size_t)hc[e] * k + d];
    const double r = p - hv[e];
    sq += r * r;
    err = fmax(err, fabs(r - R[e]));
    for (int d = 0; d < k; ++d) {
      RH[(size_t)hr[e] * k + d] += r * h[(size_t)hc[e] * k + d];
      RtW[(size_t)hc[e] * k + d] += r * w[(size_t)hr[e] * k + d];
    }
  }
  for (int64_t t = 0; t < (int64_t)m * k; ++t) err = fmax(err, fabs(RH[t] - gRH[t]));
  for (int64_t t = 0; t < (int64_t)n * k; ++t) err = fmax(err, fabs(RtW[t] - gRtW[t]));
  const double sq_rel = fabs(sums[0] - sq) / sq;
  printf("nnz %lld  max |err| %.3e  sum r^2 rel %.3e\n", (long long)nnz, err, sq_rel);
  if (!(err < 1e-11) || !(sq_rel < 1e-12)) return 2;

  /* end to end from host factors: [sums | RH | RtW] in one host buffer */
  const size_t outb = 32 + ((size_t)m + n) * k * 8;
  void* dout = dalloc(outb);
  void* hout = NULL;
  CU(cudaMallocHost(&hout, outb));
  CK(mfg_sweep_host(MFG_F64, 0, &csr, &csc, k, v_out, v_csc, w, h, dw, k, dh, k, dR, dout, hout,
                    1.0, sws, swb, NULL));
  CU(cudaDeviceSynchronize());
  if (memcmp((char*)hout + 32, gRH, (size_t)m * k * 8) != 0 ||
      memcmp((char*)hout + 32 + (size_t)m * k * 8, gRtW, (size_t)n * k * 8) != 0) {
    fprintf(stderr, "mfg_sweep_host differs from mfg_sweep\n");
    return 3;
  }
  /* argument errors map to MFG_ERR_ARG with a message */
  if (mfg_sweep(MFG_F64, 0, &csr, &csr, k, v_out, v_csc, dw, k, dh, k, dR, dRH, dRtW, 1.0, dsums,
                sws, swb, NULL) != MFG_ERR_ARG) {
    fprintf(stderr, "mismatched layouts not rejected\n");
    return 4;
  }
  printf("abi client ok (%s)\n", mfg_last_error());
  return 0;
}
