// SpMM over Omega for the lifting operator: Y = alpha * S X + beta * Y.
//
// Replaces scipy csr_matvecs in ShiftedOperator.apply / apply_t /
// project_rows (mfg/operators.py:108,117,135) and certify_epsilon's g_apply
// (mfg/proxlift.py:239-243). Same flat-chunk schedule as the sweep (one warp
// per nnz chunk, carries for rows crossing chunk boundaries, deterministic
// epilogue), lanes over the p block columns: each entry gathers one X row
// with coalesced 128-byte accesses and does S FMAs per lane; no cross-lane
// reductions are needed. gridDim.y tiles p in 32*S-column slabs; S (1..8
// columns per lane) is picked per call so that the block takes as few
// passes over the entry stream as possible: a pass costs ~8 ms at config 4
// whatever its width, so p = 160 in one 5-column pass instead of 128 + 32
// takes 10.5 instead of 17.9 ms. Per (row, column) the additions keep their
// order, so results do not depend on S.
#include "common.cuh"
#include "engine.cuh"

namespace mfg {
namespace {

constexpr int kThreads = 256;
constexpr int kWpb = kThreads / 32;
constexpr int kS = 4;        // columns per lane of the chunk-size rule (pick_cb; kept from the
                             // fixed 128-column slabs so that chunk boundaries, and with them
                             // the carry order, are unchanged)
constexpr int kMaxS = 8;     // at most 256 columns per pass

template <typename T>
struct SpPass {
  mfg_layout lay;
  const T* vals;
  const T* X;
  int ldx;
  T* Y;
  int ldy;
  double alpha, beta;
  int p;
  int cb;
  int nchunks;
  T* carry_vec;        // [2*nchunks][p]
  int32_t* carry_row;  // [2*nchunks]
};

// S: columns per lane; G: entries whose gathers are issued together (G * S = 32 loads in flight)
template <typename T, int S, int G>
__global__ void __launch_bounds__(kThreads) k_spmm(SpPass<T> P) {
  __shared__ int32_t s_col[kWpb][32];
  __shared__ T s_val[kWpb][32];
  const int wib = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int chunk = blockIdx.x * kWpb + wib;
  if (chunk >= P.nchunks) return;
  const int d0 = blockIdx.y * 32 * S;
  const int64_t nnz = P.lay.nnz;
  const int64_t E0 = (int64_t)chunk * P.cb * 32;
  const int64_t E1 = min(E0 + (int64_t)P.cb * 32, nnz);
  const int64_t b0 = E0 / 32;
  const bool start_cross = (P.lay.bmask[b0] & 1u) == 0u;
  const bool end_cross = (E1 < nnz) && ((P.lay.bmask[E1 / 32] & 1u) == 0u);
  int rank = P.lay.brank[b0];
  int row = P.lay.nzrows[rank];
  bool first_row = true, used_first = false, used_last = false;
  int row_first = -1, row_last = -1;
  T acc[S];
#pragma unroll
  for (int s = 0; s < S; ++s) acc[s] = T(0);
  const T alpha = (T)P.alpha, beta = (T)P.beta;

  auto flush = [&](bool is_last) {
    const bool cs = first_row && start_cross;
    const bool ce = is_last && end_cross;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int d = d0 + lane + 32 * s;
      if (d < P.p) {
        if (cs) P.carry_vec[(int64_t)(2 * chunk) * P.p + d] = acc[s];
        else if (ce) P.carry_vec[(int64_t)(2 * chunk + 1) * P.p + d] = acc[s];
        else {
          T* y = P.Y + (int64_t)row * P.ldy + d;
          *y = beta == T(0) ? alpha * acc[s] : alpha * acc[s] + beta * *y;
        }
      }
      acc[s] = T(0);
    }
    if (cs) { used_first = true; row_first = row; }
    else if (ce) { used_last = true; row_last = row; }
  };

  const int nb = (int)((E1 - E0 + 31) / 32);
  for (int bi = 0; bi < nb; ++bi) {
    const int64_t Eb = E0 + (int64_t)bi * 32;
    const int nvalid = (int)min((int64_t)32, E1 - Eb);
    const uint32_t mask = P.lay.bmask[Eb / 32] & (bi == 0 ? ~1u : ~0u);
    __syncwarp();
    if (lane < nvalid) {
      s_col[wib][lane] = P.lay.idx[Eb + lane];
      s_val[wib][lane] = P.vals[Eb + lane];
    } else {
      s_col[wib][lane] = 0;
      s_val[wib][lane] = T(0);
    }
    __syncwarp();
#pragma unroll
    for (int g = 0; g < 32; g += G) {
      T x[G][S];
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const int j = s_col[wib][g + u];
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const int d = d0 + lane + 32 * s;
          x[u][s] = (g + u < nvalid && d < P.p) ? P.X[(int64_t)j * P.ldx + d] : T(0);
        }
      }
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const int t = g + u;
        if (t < nvalid) {
          if ((mask >> t) & 1u) {
            flush(false);
            first_row = false;
            ++rank;
            row = P.lay.nzrows[rank];
          }
          const T v = s_val[wib][t];
#pragma unroll
          for (int s = 0; s < S; ++s) acc[s] += v * x[u][s];
        }
      }
    }
  }
  flush(true);
  if (lane == 0 && blockIdx.y == 0) {
    P.carry_row[2 * chunk] = used_first ? row_first : -1;
    P.carry_row[2 * chunk + 1] = used_last ? row_last : -1;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_spmm_epilogue(SpPass<T> P) {
  const int lane = threadIdx.x & 31;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwg = (gridDim.x * blockDim.x) >> 5;
  const int nslots = 2 * P.nchunks;
  const T alpha = (T)P.alpha, beta = (T)P.beta;
  for (int q = 2 * wg + 1; q < nslots; q += 2 * nwg) {
    const int row = P.carry_row[q];
    if (row < 0) continue;
    for (int d0 = 0; d0 < P.p; d0 += 32) {
      const int d = d0 + lane;
      T v = T(0);
      if (d < P.p) v = P.carry_vec[(int64_t)q * P.p + d];
      for (int nx = q + 1; nx < nslots; ++nx) {
        const int r2 = P.carry_row[nx];
        if (r2 < 0) continue;
        if (r2 != row) break;
        if (d < P.p) v += P.carry_vec[(int64_t)nx * P.p + d];
      }
      if (d < P.p) {
        T* y = P.Y + (int64_t)row * P.ldy + d;
        *y = beta == T(0) ? alpha * v : alpha * v + beta * *y;
      }
    }
  }
  for (int i = wg; i < P.lay.n_empty; i += nwg) {
    const int row = P.lay.empty_rows[i];
    for (int d = lane; d < P.p; d += 32) {
      T* y = P.Y + (int64_t)row * P.ldy + d;
      *y = beta == T(0) ? T(0) : beta * *y;
    }
  }
}

int pick_cb(int64_t nnz, int slabs) {
  int64_t target = (int64_t)kNumSMs * 16 / (slabs > 0 ? slabs : 1);
  if (target < kNumSMs) target = kNumSMs;
  int64_t cb = (nnz / 32 + target - 1) / target;
  if (cb < 2) cb = 2;
  if (cb > 32) cb = 32;
  return (int)cb;
}

template <typename T>
int do_spmm(const mfg_layout* lay, int p, const void* vals, const void* X, int ldx, double alpha,
            double beta, void* Y, int ldy, void* ws, size_t wsb, cudaStream_t stream) {
  SpPass<T> P{};
  P.lay = *lay;
  P.vals = (const T*)vals; P.X = (const T*)X; P.ldx = ldx; P.Y = (T*)Y; P.ldy = ldy;
  P.alpha = alpha; P.beta = beta; P.p = p;
  const int slabs = (p + 32 * kS - 1) / (32 * kS);
  P.cb = pick_cb(lay->nnz, slabs);
  P.nchunks = (int)((lay->nnz + (int64_t)P.cb * 32 - 1) / ((int64_t)P.cb * 32));
  Carver c(ws, wsb);
  const int nch = P.nchunks > 0 ? P.nchunks : 1;
  P.carry_vec = c.take<T>((size_t)2 * nch * p);
  P.carry_row = c.take<int32_t>((size_t)2 * nch);
  MFG_REQUIRE(c.ok, "spmm workspace too small");
  if (p == 0 || lay->nrows == 0) return MFG_OK;
  if (P.nchunks > 0) {
    // fewest passes of at most 32 * kMaxS columns, then the narrowest S that covers them
    const int npass = (p + 32 * kMaxS - 1) / (32 * kMaxS);
    const int S = ((p + npass - 1) / npass + 31) / 32;
    dim3 grid((P.nchunks + kWpb - 1) / kWpb, (p + 32 * S - 1) / (32 * S));
    switch (S) {
      case 1: k_spmm<T, 1, 8><<<grid, kThreads, 0, stream>>>(P); break;
      case 2: k_spmm<T, 2, 8><<<grid, kThreads, 0, stream>>>(P); break;
      case 3: k_spmm<T, 3, 8><<<grid, kThreads, 0, stream>>>(P); break;
      case 4: k_spmm<T, 4, 8><<<grid, kThreads, 0, stream>>>(P); break;
      case 5: k_spmm<T, 5, 4><<<grid, kThreads, 0, stream>>>(P); break;
      case 6: k_spmm<T, 6, 4><<<grid, kThreads, 0, stream>>>(P); break;
      case 7: k_spmm<T, 7, 4><<<grid, kThreads, 0, stream>>>(P); break;
      default: k_spmm<T, 8, 4><<<grid, kThreads, 0, stream>>>(P); break;
    }
    MFG_LAUNCH_CHECK();
  }
  k_spmm_epilogue<T><<<2 * kNumSMs, 256, 0, stream>>>(P);
  MFG_LAUNCH_CHECK();
  return MFG_OK;
}

}  // namespace

size_t spmm_workspace(const mfg_layout* lay, int p) {
  const int slabs = (p + 32 * kS - 1) / (32 * kS);
  const int cb = pick_cb(lay->nnz, slabs);
  int64_t nch = (lay->nnz + (int64_t)cb * 32 - 1) / ((int64_t)cb * 32);
  if (nch < 1) nch = 1;
  Sizer s;
  s.take<double>((size_t)2 * nch * (p > 0 ? p : 1));
  s.take<int32_t>((size_t)2 * nch);
  return s.off + 512;
}

int spmm_dispatch(int dtype, const mfg_layout* lay, int p, const void* vals, const void* X,
                  int ldx, double alpha, double beta, void* Y, int ldy, void* ws, size_t wsb,
                  cudaStream_t stream) {
  if (dtype == MFG_F64)
    return do_spmm<double>(lay, p, vals, X, ldx, alpha, beta, Y, ldy, ws, wsb, stream);
  return do_spmm<float>(lay, p, vals, X, ldx, alpha, beta, Y, ldy, ws, wsb, stream);
}

}  // namespace mfg
