// Tall-skinny Householder QR with the |R_jj| column screening of
// orthonormalize (mfg/kernels.py:76-105: np.linalg.qr, then columns with
// |R_jj| <= tol ||B||_F are dropped), on our own kernels.
//
// The reference's LAPACK geqrf/orgqr is a column-by-column Householder QR;
// cuSOLVER's version of it ran config 1's blocks (2000 x 300) at ~9 GF/s in
// 8-column panel kernels (`geqr2_smem_domino_fast`: 4.9 s of a 20 s run).
// Here the block is factored 32 columns at a time:
//   * block classical Gram-Schmidt with re-orthogonalisation (BCGS2): the
//     panel is projected off the finished columns (P -= Q (Q^T P), both
//     products on the DMMA kernels of dense.cu), factored, projected and
//     factored again -- "twice is enough": Q is orthonormal to O(eps) and
//     |diag R| = |diag R2| |diag R1| matches Householder's to O(eps ||B||);
//   * the panel itself is factored by TSQR on Householder reflectors:
//     k_qr_chunk holds up to 256 rows x 32 columns of the panel in shared
//     memory (column-major), runs the 32 reflector steps there (dlarfg /
//     dlarf arithmetic, fixed reduction trees), writes the chunk's R and
//     overwrites the reflectors with the explicit chunk Q (dorg2r order);
//     the stacked R factors (32 rows per chunk) recurse through the same
//     kernel until one chunk is left, and k_chunk_mul multiplies the chunk
//     Q's down the tree. Orthogonal transformations only, so a panel that is
//     rank deficient after the projection still gives an orthonormal Q and
//     tiny |R_jj| for the dependent columns -- the property the screening
//     needs and CholeskyQR lacks (its R_jj resolve only sqrt(eps) ||B||).
// Everything is one stream-ordered sequence of launches behind one ABI call;
// no host synchronisation, bitwise reproducible.
#include "common.cuh"
#include "engine.cuh"

namespace mfg {
namespace {

constexpr int kNB = 32;            // panel width
constexpr int kCH = 256;           // rows of a chunk (one row per thread)
constexpr size_t kQrSmem = (size_t)kNB * kCH * sizeof(double);   // parked columns

struct ChunkSplit {
  int nch, base, rem;
};

// rows split evenly over nch chunks of at most kCH and at least nb rows
inline ChunkSplit split_rows(int rows, int nb) {
  int nch = (rows + kCH - 1) / kCH;
  const int cap = rows / nb;   // >= 1: rows >= nb
  if (nch > cap) nch = cap;
  if (nch < 1) nch = 1;
  return {nch, rows / nch, rows % nch};
}

// lane L ends with the warp's sum of red[L] in red[0] (31 shuffles, fixed tree)
__device__ __forceinline__ void transpose_reduce(double (&red)[kNB], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const double send = up ? red[i] : red[i + s];
      const double keep = up ? red[i + s] : red[i];
      red[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
}

// Householder QR of chunk blockIdx.x of A (rows x nb, row-major, lda): R
// (nb x nb upper, zeros below) to Rst[chunk], explicit Q (chunk rows x nb) to
// Q (row-major, ldq). diag_out (top level only): |R_cc| (* diag_mul[c]).
// One row per thread, held in registers as a window that slides with the
// step: slot s is column j + s (slots past the panel are zero), so every
// step runs the same code (a fully unrolled version is 24k instructions and
// stalls on instruction fetch). Step j reduces, in one round, x^T x and
// x^T a_c for the sub-diagonal part x of column j (per-warp transpose
// reduction, 8 partials per slot through shared memory, summed by every
// warp); the dlarfg scalars follow from x^T x, and v^T a_c = a_jc + scale
// x^T a_c with v = [1; scale x], so a step costs one block barrier. Finished
// columns (R above the diagonal, reflectors below) are parked in shared
// memory, one column-major slab, and come back in the dorg2r pass, which
// slides the window the other way.
__global__ void __launch_bounds__(kCH) k_qr_chunk(int nb, const double* __restrict__ A, int lda,
                                                  int base, int rem, double* __restrict__ Rst,
                                                  double* __restrict__ Q, int ldq,
                                                  double* __restrict__ diag_out,
                                                  const double* __restrict__ diag_mul) {
  extern __shared__ __align__(16) double sV[];        // [kNB][kCH] finished columns
  __shared__ double spart[2][kCH / 32][kNB];
  __shared__ double stotw[kCH / 32][kNB];
  __shared__ double srow[2][kNB];
  __shared__ double stau[kNB];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int ch = blockIdx.x;
  const int r0 = ch * base + min(ch, rem);
  const int rows = base + (ch < rem ? 1 : 0);
  const bool live = tid < rows;
  double a[kNB];
  {
    const double* src = A + (int64_t)(r0 + (live ? tid : 0)) * lda;
#pragma unroll
    for (int c = 0; c < kNB; ++c) a[c] = (live && c < nb) ? src[c] : 0.0;
  }
#pragma unroll 1
  for (int j = 0; j < nb; ++j) {
    const int par = j & 1;
    const double x = tid > j ? a[0] : 0.0;
    double red[kNB];
#pragma unroll
    for (int c = 0; c < kNB; ++c) red[c] = x * a[c];
    transpose_reduce(red, lane);
    spart[par][w][lane] = red[0];
    if (tid == j) {
#pragma unroll
      for (int c = 0; c < kNB; ++c) srow[par][c] = a[c];
    }
    __syncthreads();
    {
      double t = 0.0;
#pragma unroll
      for (int i = 0; i < kCH / 32; ++i) t += spart[par][i][lane];
      stotw[w][lane] = t;
    }
    __syncwarp();
    const double xn2 = stotw[w][0], alpha = srow[par][0];
    double beta = alpha, tau = 0.0, scale = 0.0;
    if (xn2 > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    const double vr = tid > j ? x * scale : (tid == j ? 1.0 : 0.0);
    const double done = tid > j ? vr : (tid == j ? beta : a[0]);
    sV[j * kCH + tid] = done;
    if (tid == 0) stau[j] = tau;
    // slide the window: slot s <- slot s + 1, updated by the reflector
#pragma unroll
    for (int c = 1; c < kNB; ++c) {
      const double t = tau * fma(scale, stotw[w][c], srow[par][c]);
      a[c - 1] = fma(-t, vr, a[c]);
    }
    a[kNB - 1] = 0.0;
    __syncwarp();
  }
  __syncthreads();
  for (int e = tid; e < nb * nb; e += kCH) {
    const int r = e / nb, c = e - r * nb;
    Rst[(size_t)ch * nb * nb + e] = c >= r ? sV[c * kCH + r] : 0.0;
  }
  if (diag_out && tid < nb) {
    const double d = fabs(sV[tid * kCH + tid]);
    diag_out[tid] = diag_mul ? d * diag_mul[tid] : d;
  }
  // explicit Q, last reflector first (dorg2r): slot s is column j + 1 + s
#pragma unroll
  for (int c = 0; c < kNB; ++c) a[c] = 0.0;
  __syncthreads();
#pragma unroll 1
  for (int j = nb - 1; j >= 0; --j) {
    const int par = j & 1;
    const double tau = stau[j];
    const double v = tid > j ? sV[j * kCH + tid] : 0.0;
    const double vr = tid > j ? v : (tid == j ? 1.0 : 0.0);
    // (tau == 0 runs the same code: t = 0, the window just slides -- one
    // barrier per step on every path keeps the double buffers safe)
    double red[kNB];
#pragma unroll
    for (int c = 0; c < kNB; ++c) red[c] = v * a[c];
    transpose_reduce(red, lane);
    spart[par][w][lane] = red[0];
    if (tid == j) {
#pragma unroll
      for (int c = 0; c < kNB; ++c) srow[par][c] = a[c];
    }
    __syncthreads();
    {
      double t = 0.0;
#pragma unroll
      for (int i = 0; i < kCH / 32; ++i) t += spart[par][i][lane];
      stotw[w][lane] = t;
    }
    __syncwarp();
#pragma unroll
    for (int c = kNB - 1; c >= 1; --c) {
      const double t = tau * (srow[par][c - 1] + stotw[w][c - 1]);
      a[c] = fma(-t, vr, a[c - 1]);
    }
    __syncwarp();
    a[0] = tid > j ? -tau * v : (tid == j ? 1.0 - tau : 0.0);
  }
  if (live) {
    double* dst = Q + (int64_t)(r0 + tid) * ldq;
#pragma unroll
    for (int c = 0; c < kNB; ++c)
      if (c < nb) dst[c] = a[c];
  }
}

// out[chunk rows] = Qloc[chunk rows] (rows x nb, ld nb) * M[chunk] (nb x nb,
// ld nb): one row per thread; out may alias Qloc (a thread reads its whole
// row before it writes).
__global__ void __launch_bounds__(kCH) k_chunk_mul(int nb, const double* Qloc, int base, int rem,
                                                   const double* __restrict__ M, double* out,
                                                   int ldo) {
  __shared__ double sM[kNB][kNB];
  const int tid = threadIdx.x;
  const int ch = blockIdx.x;
  const int r0 = ch * base + min(ch, rem);
  const int rows = base + (ch < rem ? 1 : 0);
  for (int e = tid; e < kNB * kNB; e += kCH) {
    const int r = e / kNB, c = e % kNB;
    sM[r][c] = (r < nb && c < nb) ? M[((size_t)ch * nb + r) * nb + c] : 0.0;
  }
  __syncthreads();
  if (tid >= rows) return;
  const double* src = Qloc + (size_t)(r0 + tid) * nb;
  double a[kNB];
#pragma unroll
  for (int k = 0; k < kNB; ++k) a[k] = k < nb ? src[k] : 0.0;
  double* dst = out + (int64_t)(r0 + tid) * ldo;
  for (int c = 0; c < nb; ++c) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < kNB; ++k) acc = fma(a[k], sM[k][c], acc);
    dst[c] = acc;
  }
}

// bytes of the TSQR tree buffers of a rows x nb panel
template <typename C>
void tree_buffers(C& c, int rows, int nb, double** qloc, double** rst, int* nchs, int* rws,
                  int* levels) {
  int L = 0;
  for (;;) {
    const ChunkSplit sp = split_rows(rows, nb);
    qloc[L] = c.template take<double>((size_t)rows * nb);
    rst[L] = c.template take<double>((size_t)sp.nch * nb * nb);
    nchs[L] = sp.nch;
    rws[L] = rows;
    ++L;
    if (sp.nch == 1) break;
    rows = sp.nch * nb;
  }
  *levels = L;
}

constexpr int kMaxLevels = 12;

struct QrPlan {
  double* gemm_ws;
  size_t gemm_wsb;
  double* panel;   // m x 32
  double* proj;    // p x 32
  double* dtmp;    // 32
  double* qloc[kMaxLevels];
  double* rst[kMaxLevels];
  int nch[kMaxLevels], rows[kMaxLevels], levels;
};

size_t gemm_ws_max(int m, int p) {
  size_t g = 0;
  for (int j0 = kNB; j0 < p; j0 += kNB) {
    const size_t b = gemm_tn_workspace(m, j0, min(kNB, p - j0));
    if (b > g) g = b;
  }
  // never hand out the front of a shared workspace: gemm_tn's arrival
  // counters live in its first 64 KiB and must stay zero at rest
  if (g < 65536) g = 65536;
  return g;
}

template <typename C>
void carve(C& c, int m, int p, QrPlan& pl) {
  pl.gemm_wsb = gemm_ws_max(m, p);
  pl.gemm_ws = (double*)c.template take<char>(pl.gemm_wsb);
  pl.panel = c.template take<double>((size_t)m * kNB);
  pl.proj = c.template take<double>((size_t)p * kNB);
  pl.dtmp = c.template take<double>(kNB);
  tree_buffers(c, m, min(kNB, p), pl.qloc, pl.rst, pl.nch, pl.rows, &pl.levels);
}

// TSQR of P (m x nb, ldp): explicit Q to Qout (ldq), |diag R| (* mul) to dout
int tsqr(const QrPlan& pl, int m, int nb, const double* P, int ldp, double* Qout, int ldq,
         double* dout, const double* dmul, cudaStream_t s) {
  // the tree of an nb-wide panel (nb <= the width the buffers were carved for)
  int rws[kMaxLevels], L = 0, rows = m;
  for (;;) {
    const ChunkSplit sp = split_rows(rows, nb);
    rws[L] = rows;
    ++L;
    if (sp.nch == 1) break;
    rows = sp.nch * nb;
    MFG_REQUIRE(L < kMaxLevels, "tsqr: too many levels");
  }
  MFG_REQUIRE(L <= pl.levels, "tsqr: tree deeper than planned");
  const double* in = P;
  int ldin = ldp;
  for (int l = 0; l < L; ++l) {
    const ChunkSplit sp = split_rows(rws[l], nb);
    const bool top = l == L - 1;
    double* q = (l == 0 && top) ? Qout : pl.qloc[l];
    const int ld = (l == 0 && top) ? ldq : nb;
    k_qr_chunk<<<sp.nch, kCH, kQrSmem, s>>>(nb, in, ldin, sp.base, sp.rem, pl.rst[l], q, ld,
                                            top ? dout : nullptr, top ? dmul : nullptr);
    MFG_LAUNCH_CHECK();
    in = pl.rst[l];
    ldin = nb;
  }
  for (int l = L - 2; l >= 0; --l) {
    const ChunkSplit sp = split_rows(rws[l], nb);
    k_chunk_mul<<<sp.nch, kCH, 0, s>>>(nb, pl.qloc[l], sp.base, sp.rem, pl.qloc[l + 1],
                                       l == 0 ? Qout : pl.qloc[l], l == 0 ? ldq : nb);
    MFG_LAUNCH_CHECK();
  }
  return MFG_OK;
}

}  // namespace

size_t qr_workspace(int m, int p) {
  if (m <= 0 || p <= 0 || p > m) return 0;
  Sizer s;
  QrPlan pl;
  carve(s, m, p, pl);
  return s.off;
}

// Q (m x p, ldq) and diag (p: |R_jj|) of the QR factorisation of B (m x p,
// ldb), m >= p >= 1. The front of the workspace is the gemm_tn workspace
// (arrival counters zero at rest).
int qr_factor(int m, int p, const double* B, int ldb, double* Q, int ldq, double* diag, void* ws,
              size_t wsb, cudaStream_t s) {
  MFG_REQUIRE(m >= 1 && p >= 1 && p <= m, "qr: need m >= p >= 1");
  MFG_REQUIRE(ldb >= p && ldq >= p, "qr: leading dimension too small");
  MFG_REQUIRE(B && Q && diag && ws, "qr: null pointer");
  MFG_CUDA_CHECK(cudaFuncSetAttribute(k_qr_chunk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kQrSmem));
  Carver c(ws, wsb);
  QrPlan pl;
  carve(c, m, p, pl);
  MFG_REQUIRE(c.ok, "qr workspace too small");
  for (int j0 = 0; j0 < p; j0 += kNB) {
    const int nb = min(kNB, p - j0);
    double* qj = Q + j0;
    if (j0 == 0) {
      if (int e = tsqr(pl, m, nb, B, ldb, qj, ldq, diag, nullptr, s)) return e;
      continue;
    }
    // pass 1: panel = B_j - Q (Q^T B_j) over the finished columns, factor
    if (int e = gemm_tn(m, j0, nb, Q, ldq, B + j0, ldb, 1.0, pl.proj, kNB, pl.gemm_ws,
                        pl.gemm_wsb, s))
      return e;
    if (int e = gemm_nn(m, j0, nb, Q, ldq, pl.proj, kNB, -1.0, 1.0, pl.panel, kNB, s, B + j0, ldb))
      return e;
    if (int e = tsqr(pl, m, nb, pl.panel, kNB, qj, ldq, pl.dtmp, nullptr, s)) return e;
    // pass 2: the same on the pass-1 Q
    if (int e = gemm_tn(m, j0, nb, Q, ldq, qj, ldq, 1.0, pl.proj, kNB, pl.gemm_ws, pl.gemm_wsb, s))
      return e;
    if (int e = gemm_nn(m, j0, nb, Q, ldq, pl.proj, kNB, -1.0, 1.0, pl.panel, kNB, s, qj, ldq))
      return e;
    if (int e = tsqr(pl, m, nb, pl.panel, kNB, qj, ldq, diag + j0, pl.dtmp, s)) return e;
  }
  return MFG_OK;
}

}  // namespace mfg
