// The Omega sweep: fused SDDMM + SpMM over one or both orientations of Omega.
//
// Work decomposition ("flat chunks"): the nnz stream of a layout is cut into
// chunks of `cb` 32-entry batches; one warp owns one chunk, regardless of row
// boundaries, so Zipf-skewed degree distributions are load-balanced by
// construction. Rows that cross a chunk boundary emit partial sums into two
// carry slots per chunk; a deterministic epilogue adds the carries of each
// row in chunk order, zero-fills empty rows, and reduces the per-warp fp64
// partial sums in a fixed order. No floating-point atomics anywhere, so the
// results are bitwise reproducible run to run.
//
// Per 32-entry batch (lanes over the k factor dimensions, d = lane + 32 s):
//   1. lane t loads (col_t, A_t) coalesced; cols are broadcast through smem;
//   2. for every slot t the warp gathers the *whole* factor row other[col_t]
//      with one coalesced 128-byte access per 32 dimensions (the L1-wavefront
//      optimal way to gather rows), keeping all 32 rows in registers;
//   3. lane-partials p_t = <self_row(t), other[col_t]> restricted to the
//      lane's dimensions; a butterfly transpose-reduction (31 shuffles for 32
//      entries) leaves dot_t in lane t; r_t = dot_t - A_t is stored coalesced;
//   4. the SpMM accumulation acc += r_t * other[col_t] reuses the registers of
//      step 2, and is flushed (coalesced k-vector store) at each row change.
// This replaces pair_values (mfg/data.py:253-263, an einsum over gathered
// rows) and scipy csr_matvecs (grad.csr @ block, mfg/operators.py:108,117).
#include <cstdlib>
#include <vector>

#ifndef MFG_FFMA2
#define MFG_FFMA2 1
#endif
#ifndef MFG_FFMA2_VMAX
#define MFG_FFMA2_VMAX 4
#endif
#ifndef MFG_G8_MINB4
#define MFG_G8_MINB4 4   // 128-thread CTAs per SM, 16-byte lane slices (<= 128 registers;
                         // 5 x 102 spills and measured slower)
#endif
#ifndef MFG_G8_MINB8
#define MFG_G8_MINB8 4   // 32-byte lane slices (<= 128 registers)
#endif

#include "common.cuh"

#ifndef MFG_SMEM_REDUCE
#define MFG_SMEM_REDUCE 1  // fp32: partial-dot transpose through shared memory instead of the
                           // butterfly (11 fewer instructions per batch; c3/c4 -1.4%)
#endif
#ifndef MFG_UNROLL_U
#define MFG_UNROLL_U 0  // unroll the 4 group-batches of a ring block
#endif
#include "engine.cuh"

namespace mfg {

std::atomic<int64_t> g_launches{0};

// Optional per-launch CUDA-event timing of the dominant (main sweep) kernel,
// recorded on the launching stream. Enabled by mfg_profile_enable().
struct KernelProfiler {
  std::vector<cudaEvent_t> start, stop;
  size_t used = 0;
  bool on = false;
};
KernelProfiler g_prof;
long long* g_probe = nullptr;  // device buffer for per-worker clock stamps (diagnostics)

void prof_begin(cudaStream_t s) {
  if (g_prof.on && g_prof.used < g_prof.start.size()) cudaEventRecord(g_prof.start[g_prof.used], s);
}
void prof_end(cudaStream_t s) {
  if (g_prof.on && g_prof.used < g_prof.start.size()) {
    cudaEventRecord(g_prof.stop[g_prof.used], s);
    ++g_prof.used;
  }
}

namespace {

constexpr int kThreads = 256;
constexpr int kWarpsPerBlock = kThreads / 32;
// grouped sweep CTA: 16 eight-lane workers (4 warps). Smaller CTAs than the
// other kernels: finer occupancy steps and shorter CTA-level tails (c4 -2%).
constexpr int kGThreads = 128;
template <typename TS, typename TC, int V>
__host__ __device__ constexpr int g8_min_blocks() {
  return sizeof(TC) == 4 ? (V * sizeof(TS) == 16 ? MFG_G8_MINB4 : MFG_G8_MINB8) : 2;
}

// Fixed-pattern butterfly: lane l ends with sum over lanes of v[l].
template <typename T>
__device__ __forceinline__ T transpose_reduce(T (&v)[32]) {
  const int lane = lane_id();
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const T send = upper ? v[i] : v[i + s];
      const T keep = upper ? v[i + s] : v[i];
      v[i] = keep + shfl_xor(send, s);
    }
  }
  return v[0];
}

template <typename TS, typename TC>
struct Pass {
  mfg_layout lay;
  const TS* vals;       // A (may be null -> 0)
  const TS* G;          // optional gradient values (SDDMM reductions)
  const TS* self;       // row factor
  int lds;
  const double* scale;  // optional per-dim scale of self
  const TS* other;      // gathered factor
  int ldo;
  TS* R;                // optional residual output (layout order)
  double r_mult;        // R = r_mult * r
  TS* out;              // optional SpMM output (nrows x k)
  int ldout;
  double out_scale;
  int cb;               // batches per chunk
  int nchunks;
  TC* carry_vec;        // [2*nchunks][cstride]
  int32_t* carry_row;   // [2*nchunks]
  int cstride;          // carry vector stride (k, or the padded kp of the grouped kernel)
  int32_t* row_cnt;     // [nrows] arrival counters (fused finisher; zero at rest)
  long long* probe;     // optional [nchunks][4] clock64 stamps (diagnostics)
  double* part;         // [3][nchunks] per-warp partial sums (or null)
  int want_sq;          // accumulate sum r^2 into part[0]
};

template <typename TS, typename TC>
__device__ __forceinline__ TC ld_self(const Pass<TS, TC>& P, int row, int d, int k) {
  if (d >= k) return TC(0);
  TC v = (TC)P.self[(int64_t)row * P.lds + d];
  if (P.scale) v *= (TC)P.scale[d];
  return v;
}

// Process one chunk. S = dimension slices held in registers (k <= 32*S when
// !MULTI; with MULTI, k is processed in 32*S-wide dimension chunks, the
// accumulator lives in shared memory across batches and the gathered rows are
// re-read (L1/L2-resident) for the accumulation).
template <typename TS, typename TC, int S, bool ACC, bool MULTI>
__device__ void run_chunk(const Pass<TS, TC>& P, int chunk, int k, int32_t* s_col,
                          TC* s_r, TC* s_acc) {
  const int lane = lane_id();
  const int64_t nnz = P.lay.nnz;
  const int64_t E0 = (int64_t)chunk * P.cb * 32;
  if (E0 >= nnz) return;
  const int64_t E1 = min(E0 + (int64_t)P.cb * 32, nnz);
  const int nkc = MULTI ? (k + 32 * S - 1) / (32 * S) : 1;
  const int64_t b0 = E0 / 32;
  const bool start_cross = (P.lay.bmask[b0] & 1u) == 0u;
  const bool end_cross = (E1 < nnz) && ((P.lay.bmask[E1 / 32] & 1u) == 0u);

  int rank = P.lay.brank[b0];
  int row = P.lay.nzrows[rank];
  bool first_row = true;
  bool used_first = false, used_last = false;
  int row_first = -1, row_last = -1;

  TC acc[S];
#pragma unroll
  for (int s = 0; s < S; ++s) acc[s] = TC(0);
  if (MULTI && ACC) {
    for (int d = lane; d < k; d += 32) s_acc[d] = TC(0);
  }
  double sq = 0.0, s1 = 0.0, s2 = 0.0;

  // flush the accumulated vector of `frow` (dims slice kc)
  auto flush = [&](int frow, bool is_first, bool is_last, int kc) {
    const bool cross_start = is_first && start_cross;
    const bool cross_end = is_last && end_cross;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int d = kc * 32 * S + lane + 32 * s;
      if (d < k) {
        const TC v = MULTI ? s_acc[d] : acc[s];
        if (cross_start) {
          P.carry_vec[(int64_t)(2 * chunk) * k + d] = v;
        } else if (cross_end) {
          P.carry_vec[(int64_t)(2 * chunk + 1) * k + d] = v;
        } else {
          P.out[(int64_t)frow * P.ldout + d] = (TS)(v * (TC)P.out_scale);
        }
      }
    }
    if (cross_start) { used_first = true; row_first = frow; }
    else if (cross_end) { used_last = true; row_last = frow; }
  };

  const int nb = (int)((E1 - E0 + 31) / 32);
  for (int bi = 0; bi < nb; ++bi) {
    const int64_t Eb = E0 + (int64_t)bi * 32;
    const int nvalid = (int)min((int64_t)32, E1 - Eb);
    const int64_t e = Eb + lane;
    const bool valid = lane < nvalid;
    const uint32_t mask = P.lay.bmask[Eb / 32] & (bi == 0 ? ~1u : ~0u);
    int col = 0;
    TC a = TC(0), gval = TC(0);
    if (valid) {
      col = P.lay.idx[e];
      if (P.vals) a = (TC)P.vals[e];
      if (P.G) gval = (TC)P.G[e];
    }
    __syncwarp();
    s_col[lane] = col;
    __syncwarp();

    const int rank_b = rank, row_b = row;  // state at batch start (for loop 2)
    TC p[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) p[t] = TC(0);
    TS h[32][S];

    for (int kc = 0; kc < nkc; ++kc) {
      // issue all gathers for this dimension chunk
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        const int j = s_col[t];
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const int d = kc * 32 * S + lane + 32 * s;
          h[t][s] = (t < nvalid && d < k) ? P.other[(int64_t)j * P.ldo + d] : TS(0);
        }
      }
      // lane partial dot products, reloading self at row changes
      int rk = rank_b, rw = row_b;
      TC w[S];
#pragma unroll
      for (int s = 0; s < S; ++s) w[s] = ld_self(P, rw, kc * 32 * S + lane + 32 * s, k);
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        if (t < nvalid) {
          if ((mask >> t) & 1u) {
            ++rk;
            rw = P.lay.nzrows[rk];
#pragma unroll
            for (int s = 0; s < S; ++s) w[s] = ld_self(P, rw, kc * 32 * S + lane + 32 * s, k);
          }
#pragma unroll
          for (int s = 0; s < S; ++s) p[t] += w[s] * (TC)h[t][s];
        }
      }
    }
    const TC dot = transpose_reduce(p);
    const TC r = valid ? dot - a : TC(0);
    if (valid) {
      if (P.R) P.R[e] = (TS)(r * (TC)P.r_mult);
      if (P.want_sq) sq += (double)r * (double)r;
      if (P.G) {
        s1 += (double)gval * ((double)r - 0.5 * (double)gval);
        s2 += (double)gval * (double)dot;
      }
    }

    if (ACC && P.out) {
      __syncwarp();
      s_r[lane] = r;
      __syncwarp();
      for (int kc = 0; kc < nkc; ++kc) {
        if (MULTI) {
#pragma unroll
          for (int s = 0; s < S; ++s) {
            const int d = kc * 32 * S + lane + 32 * s;
            acc[s] = d < k ? s_acc[d] : TC(0);
          }
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const int j = s_col[t];
#pragma unroll
            for (int s = 0; s < S; ++s) {
              const int d = kc * 32 * S + lane + 32 * s;
              h[t][s] = (t < nvalid && d < k) ? P.other[(int64_t)j * P.ldo + d] : TS(0);
            }
          }
        }
        int rk = rank_b, rw = row_b;
        bool fr = first_row;
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          if (t < nvalid) {
            if ((mask >> t) & 1u) {
              if (MULTI) {
#pragma unroll
                for (int s = 0; s < S; ++s) {
                  const int d = kc * 32 * S + lane + 32 * s;
                  if (d < k) s_acc[d] = acc[s];
                }
              }
              flush(rw, fr, false, kc);
              fr = false;
              ++rk;
              rw = P.lay.nzrows[rk];
#pragma unroll
              for (int s = 0; s < S; ++s) acc[s] = TC(0);
            }
            const TC rt = s_r[t];
#pragma unroll
            for (int s = 0; s < S; ++s) acc[s] += rt * (TC)h[t][s];
          }
        }
        if (MULTI) {
#pragma unroll
          for (int s = 0; s < S; ++s) {
            const int d = kc * 32 * S + lane + 32 * s;
            if (d < k) s_acc[d] = acc[s];
          }
        }
        if (kc == nkc - 1) {
          rank = rk;
          row = rw;
          first_row = fr;
        }
      }
    } else {
      // advance row state without accumulation (uniform across the warp)
      rank += __popc(mask & (nvalid == 32 ? 0xffffffffu : ((1u << nvalid) - 1u)));
      row = P.lay.nzrows[rank];
      first_row = false;
    }
  }
  if (ACC && P.out) {
    // final row of the chunk
    for (int kc = 0; kc < nkc; ++kc) flush(row, first_row, true, kc);
    if (lane == 0) {
      P.carry_row[2 * chunk] = used_first ? row_first : -1;
      P.carry_row[2 * chunk + 1] = used_last ? row_last : -1;
    }
  }
  if (P.part) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sq += __shfl_xor_sync(0xffffffffu, sq, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) {
      P.part[chunk] = sq;
      P.part[P.nchunks + chunk] = s1;
      P.part[2 * P.nchunks + chunk] = s2;
    }
  }
}

// Out-of-line row flush (row ends are rare relative to entries): either a
// direct coalesced store of the k-vector or a carry slot for a row that
// crosses a chunk boundary.
template <typename TS, typename TC>
__device__ __noinline__ void flush_row(TS* out, int ldout, double out_scale, TC* carry_vec,
                                       int64_t slot, int k, int frow, TC a0, TC a1) {
  const int lane = threadIdx.x & 31;
  const int d0 = lane, d1 = lane + 32;
  if (slot >= 0) {
    if (d0 < k) carry_vec[slot * k + d0] = a0;
    if (d1 < k) carry_vec[slot * k + d1] = a1;
  } else {
    if (d0 < k) out[(int64_t)frow * ldout + d0] = (TS)(a0 * (TC)out_scale);
    if (d1 < k) out[(int64_t)frow * ldout + d1] = (TS)(a1 * (TC)out_scale);
  }
}

template <typename T>
__device__ __forceinline__ void ld4(const T* p, T (&o)[4]);
template <>
__device__ __forceinline__ void ld4<float>(const float* p, float (&o)[4]) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
template <>
__device__ __forceinline__ void ld4<double>(const double* p, double (&o)[4]) {
  const double2 a = reinterpret_cast<const double2*>(p)[0];
  const double2 b = reinterpret_cast<const double2*>(p)[1];
  o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
}

// Fast path (k <= 32*S): branch-free inner loops for batches that contain no
// row start (the common case), next-batch index/value prefetch, vectorised
// shared-memory broadcasts, and no per-slot validity tests (padding slots
// gather row 0 and contribute r = 0).
template <typename TS, typename TC, int S, bool ACC>
__device__ __forceinline__ void run_chunk_fast(const Pass<TS, TC>& P, int chunk, int k,
                                               int32_t* s_col, TC* s_r, int32_t* s_row) {
  static_assert(S == 1 || S == 2, "S in {1,2}");
  const int lane = lane_id();
  const int64_t nnz = P.lay.nnz;
  const int64_t E0 = (int64_t)chunk * P.cb * 32;
  if (E0 >= nnz) return;
  const int64_t E1 = min(E0 + (int64_t)P.cb * 32, nnz);
  const int nb = (int)((E1 - E0 + 31) / 32);
  const int32_t* __restrict__ idx = P.lay.idx;
  const uint32_t* __restrict__ bm = P.lay.bmask;
  const int32_t* __restrict__ nzrows = P.lay.nzrows;
  const TS* __restrict__ vals = P.vals;
  const TS* __restrict__ Gv = P.G;
  const TS* __restrict__ other = P.other;
  const TS* __restrict__ self = P.self;
  const double* __restrict__ scale = P.scale;
  const int ldo = P.ldo, lds = P.lds;
  const int64_t b0 = E0 / 32;
  const bool start_cross = (bm[b0] & 1u) == 0u;
  const bool end_cross = (E1 < nnz) && ((bm[E1 / 32] & 1u) == 0u);
  int rank = P.lay.brank[b0];
  int row = nzrows[rank];
  bool first_row = true;
  int row_first = -1, row_last = -1;

  TC w[S];
  auto load_w = [&](int rw) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int d = lane + 32 * s;
      TC v = TC(0);
      if (d < k) {
        v = (TC)self[(int64_t)rw * lds + d];
        if (scale) v *= (TC)scale[d];
      }
      w[s] = v;
    }
  };
  load_w(row);
  TC acc[S];
#pragma unroll
  for (int s = 0; s < S; ++s) acc[s] = TC(0);
  double sq = 0.0, s1 = 0.0, s2 = 0.0;

  auto flush = [&](int frow, bool is_first, bool is_last) {
    int64_t slot = -1;
    if (is_first && start_cross) { slot = 2 * (int64_t)chunk; row_first = frow; }
    else if (is_last && end_cross) { slot = 2 * (int64_t)chunk + 1; row_last = frow; }
    flush_row<TS, TC>(P.out, P.ldout, P.out_scale, P.carry_vec, slot, k, frow, acc[0],
                      S > 1 ? acc[S - 1] : TC(0));
  };

  int col_n = 0;
  TC a_n = TC(0), g_n = TC(0);
  uint32_t mask_n = 0u;
  auto fetch = [&](int bi) {
    const int64_t e = E0 + (int64_t)bi * 32 + lane;
    const bool v = e < E1;
    col_n = v ? idx[e] : 0;
    a_n = (v && vals) ? (TC)vals[e] : TC(0);
    g_n = (v && Gv) ? (TC)Gv[e] : TC(0);
    mask_n = bm[b0 + bi];
  };
  fetch(0);

  for (int bi = 0; bi < nb; ++bi) {
    const int col = col_n;
    const TC a = a_n, gval = g_n;
    const uint32_t mask = mask_n & (bi == 0 ? ~1u : ~0u);
    const int64_t Eb = E0 + (int64_t)bi * 32;
    const int nvalid = (int)min((int64_t)32, E1 - Eb);
    if (bi + 1 < nb) fetch(bi + 1);
    __syncwarp();
    s_col[lane] = col;
    __syncwarp();

    TS h[32][S];
#pragma unroll
    for (int t4 = 0; t4 < 32; t4 += 4) {
      const int4 j4 = *reinterpret_cast<const int4*>(s_col + t4);
      const int jj[4] = {j4.x, j4.y, j4.z, j4.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const int d = lane + 32 * s;
          h[t4 + u][s] = d < k ? other[(int64_t)jj[u] * ldo + d] : TS(0);
        }
      }
    }
    TC p[32];
    const int row_b = row;
    const bool fr_b = first_row;
    if (mask == 0u) {
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        TC v = w[0] * (TC)h[t][0];
        if (S > 1) v += w[S - 1] * (TC)h[t][S - 1];
        p[t] = v;
      }
    } else {
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        if ((mask >> t) & 1u) {
          ++rank;
          row = nzrows[rank];
          load_w(row);
          s_row[t] = row;
        }
        TC v = w[0] * (TC)h[t][0];
        if (S > 1) v += w[S - 1] * (TC)h[t][S - 1];
        p[t] = v;
      }
    }
    const TC dot = transpose_reduce(p);
    const bool valid = lane < nvalid;
    const TC r = valid ? dot - a : TC(0);
    if (valid) {
      if (P.R) P.R[Eb + lane] = (TS)(r * (TC)P.r_mult);
      if (P.want_sq) sq += (double)r * (double)r;
      if (Gv) {
        s1 += (double)gval * ((double)r - 0.5 * (double)gval);
        s2 += (double)gval * (double)dot;
      }
    }
    if (ACC) {
      __syncwarp();
      s_r[lane] = r;
      __syncwarp();
      if (mask == 0u) {
#pragma unroll
        for (int t4 = 0; t4 < 32; t4 += 4) {
          TC r4[4];
          ld4<TC>(s_r + t4, r4);
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int s = 0; s < S; ++s) acc[s] += r4[u] * (TC)h[t4 + u][s];
        }
      } else {
        int rw = row_b;
        bool fr = fr_b;
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          if ((mask >> t) & 1u) {
            flush(rw, fr, false);
            fr = false;
            rw = s_row[t];
#pragma unroll
            for (int s = 0; s < S; ++s) acc[s] = TC(0);
          }
          const TC rt = s_r[t];
#pragma unroll
          for (int s = 0; s < S; ++s) acc[s] += rt * (TC)h[t][s];
        }
        first_row = fr;
      }
    } else if (mask != 0u) {
      first_row = false;
    }
  }
  if (ACC) {
    flush(row, first_row, true);
    if (lane == 0) {
      P.carry_row[2 * chunk] = row_first;
      P.carry_row[2 * chunk + 1] = row_last;
    }
  }
  if (P.part) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sq += __shfl_xor_sync(0xffffffffu, sq, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) {
      P.part[chunk] = sq;
      P.part[P.nchunks + chunk] = s1;
      P.part[2 * P.nchunks + chunk] = s2;
    }
  }
}

template <typename TS, typename TC, int S, bool ACC, bool MULTI>
__global__ void __launch_bounds__(kThreads)
k_sweep(Pass<TS, TC> P0, Pass<TS, TC> P1, int nw0, int nw_total, int k) {
  __shared__ __align__(16) int32_t s_col[kWarpsPerBlock][32];
  __shared__ __align__(16) TC s_r[kWarpsPerBlock][32];
  __shared__ int32_t s_row[kWarpsPerBlock][32];
  extern __shared__ __align__(16) unsigned char s_dyn[];
  const int wib = threadIdx.x >> 5;
  TC* s_acc = MULTI ? reinterpret_cast<TC*>(s_dyn) + (size_t)wib * k : nullptr;
  const int gw = blockIdx.x * kWarpsPerBlock + wib;
  if (gw >= nw_total) return;
  if constexpr (!MULTI) {
    if (gw < nw0) run_chunk_fast<TS, TC, S, ACC>(P0, gw, k, s_col[wib], s_r[wib], s_row[wib]);
    else run_chunk_fast<TS, TC, S, ACC>(P1, gw - nw0, k, s_col[wib], s_r[wib], s_row[wib]);
  } else {
    if (gw < nw0) run_chunk<TS, TC, S, ACC, MULTI>(P0, gw, k, s_col[wib], s_r[wib], s_acc);
    else run_chunk<TS, TC, S, ACC, MULTI>(P1, gw - nw0, k, s_col[wib], s_r[wib], s_acc);
  }
}

// ---------------------------------------------------------------------------
// v3 "grouped" sweep: 8-lane groups act as independent mini-warps, each
// owning a flat chunk of entries. Factor rows are zero-padded to kp = 8*V
// elements, so lane q of a group holds dims [qV, qV+V) and ONE 16-byte vector
// load per lane gathers a whole 128-byte row across the group (one L1
// wavefront per entry, the minimum). Per 8-entry group-batch: 8 row gathers,
// lane-partial dots, a 3-step butterfly (7 shuffles per 8 entries) that
// leaves entry q's dot in lane q, then the SpMM accumulation from the same
// registers. Row ends are rare and handled by an out-of-line flush.

// Lane q's slice of a factor row is V elements in 16-byte chunks: chunk c
// holds elements [c*8E + qE, c*8E + qE + E), E = 16 / sizeof(TS). One
// LDG.128 instruction per chunk then covers 128 contiguous bytes of a row
// across the 8-lane group (each sector fetched once), where a contiguous
// 32-byte slice per lane would touch every sector with two instructions.
template <typename TS>
__host__ __device__ constexpr int chunk_elems() { return 16 / (int)sizeof(TS); }

template <typename TS, int V>
__device__ __forceinline__ int dim_of(int q, int v) {
  constexpr int E = chunk_elems<TS>();
  return (v / E) * 8 * E + q * E + (v % E);
}

// p = row base + q*E; chunks whose bit in `live` is clear are zero-filled
// (their dims are >= k: padding or, unpadded, the next row's data).
template <typename TS, typename TC, int V>
__device__ __forceinline__ void ldrow(const TS* p, TS (&o)[V], unsigned live) {
  constexpr int E = chunk_elems<TS>();
#pragma unroll
  for (int c = 0; c < V / E; ++c) {
    if ((live >> c) & 1u) {
      if constexpr (sizeof(TS) == 4) {
        const float4 x = *reinterpret_cast<const float4*>(p + c * 8 * E);
        o[4 * c] = x.x; o[4 * c + 1] = x.y; o[4 * c + 2] = x.z; o[4 * c + 3] = x.w;
      } else {
        const double2 x = *reinterpret_cast<const double2*>(p + c * 8 * E);
        o[2 * c] = x.x; o[2 * c + 1] = x.y;
      }
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) o[c * E + e] = TS(0);
    }
  }
}

// cp.async (LDGSTS) 16-byte copy global -> shared, cached in L1 (.ca).
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// 8-lane transposed butterfly: lane q (of its group) ends with sum_lanes v[q].
template <typename T>
__device__ __forceinline__ T reduce8(T (&v)[8]) {
  const int q = threadIdx.x & 7;
#pragma unroll
  for (int s = 4; s >= 1; s >>= 1) {
    const bool upper = (q & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const T send = upper ? v[i] : v[i + s];
      const T keep = upper ? v[i + s] : v[i];
      v[i] = keep + shfl_xor(send, s);
    }
  }
  return v[0];
}

// Lane-partial dot w . h over the lane's V dims. fp32: packed FFMA2 on
// (even, odd) dim pairs, then one add (V/2 + 1 issues instead of V).
template <typename TS, typename TC, int V>
__device__ __forceinline__ TC dotv(const TC (&w)[V], const TS (&h)[V]) {
  if constexpr (MFG_FFMA2 && sizeof(TS) == 4 && sizeof(TC) == 4 && V % 2 == 0 && V <= MFG_FFMA2_VMAX) {
    float2 s = __fmul2_rn(make_float2(w[0], w[1]), make_float2(h[0], h[1]));
#pragma unroll
    for (int j = 2; j < V; j += 2)
      s = __ffma2_rn(make_float2(w[j], w[j + 1]), make_float2(h[j], h[j + 1]), s);
    return s.x + s.y;
  } else {
    TC v = TC(0);
#pragma unroll
    for (int j = 0; j < V; ++j) v += w[j] * (TC)h[j];
    return v;
  }
}

// acc += r * h over the lane's V dims (packed FFMA2 for fp32).
template <typename TS, typename TC, int V>
__device__ __forceinline__ void axpyv(TC (&acc)[V], TC r, const TS (&h)[V]) {
  if constexpr (MFG_FFMA2 && sizeof(TS) == 4 && sizeof(TC) == 4 && V % 2 == 0 && V <= MFG_FFMA2_VMAX) {
    const float2 rr = make_float2(r, r);
#pragma unroll
    for (int j = 0; j < V; j += 2) {
      const float2 t = __ffma2_rn(rr, make_float2(h[j], h[j + 1]), make_float2(acc[j], acc[j + 1]));
      acc[j] = t.x; acc[j + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < V; ++j) acc[j] += r * (TC)h[j];
  }
}

template <typename TC, int V>
struct AccV {
  TC a[V];
};

template <typename TS, typename TC, int V>
__device__ __noinline__ void flush_group(TS* out, int ldout, double out_scale, TC* carry_vec,
                                         int64_t slot, int k, int kp, int frow, AccV<TC, V> acc) {
  const int q = threadIdx.x & 7;
  if (slot >= 0) {
    TC* c = carry_vec + slot * kp + q * V;
#pragma unroll
    for (int v = 0; v < V; ++v) c[v] = acc.a[v];
  } else {
    TS* o = out + (int64_t)frow * ldout;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int d = dim_of<TS, V>(q, v);
      if (d < k) o[d] = (TS)(acc.a[v] * (TC)out_scale);
    }
  }
}

// A worker deposited its piece of a row that crosses chunk boundaries into
// carry slot `slot`. The worker that deposits the row's last piece sums all
// pieces in slot order (first chunk a: slot 2a+1; chunks a+1..b: slot 2c)
// and writes the output row, so no epilogue pass is needed and the result
// is independent of arrival order.
template <typename TS, typename TC, int V>
__device__ __noinline__ void finish_row(TS* out, int ldout, double out_scale, TC* carry_vec,
                                        int32_t* row_cnt, const int32_t* ptr, int64_t CB,
                                        int k, int kp, int frow) {
  const int lane = threadIdx.x & 31;
  const int q = lane & 7;
  const unsigned gmask = 0xFFu << (lane & 24);
  // Ordering (PTX memory model): every lane's carry stores -> its
  // fence.acq_rel.gpu (run by the caller, all lanes) -> warp barrier -> the
  // group leader's acq_rel increment of the row's arrival counter. All
  // increments are release RMWs on one location, so the finisher's acq_rel
  // RMW synchronises with every earlier depositor; its lanes then pass an
  // acquire fence before reading the pieces through L2 (ld.cg). The fences
  // are MEMBAR.GPU without the CCTL.IVALL that __threadfence() adds, so the
  // SM's L1 (the gathered factor rows) survives a row crossing.
  int old = 0;
  if (q == 0) {
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(old) : "l"(row_cnt + frow) : "memory");
  }
  old = __shfl_sync(gmask, old, lane & 24);
  const int64_t a = (int64_t)ptr[frow] / CB;
  const int64_t b = (int64_t)(ptr[frow + 1] - 1) / CB;
  if (old != (int)(b - a)) return;
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  TC acc[V];
  {
    const TC* c = carry_vec + (2 * a + 1) * kp + q * V;
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = __ldcg(c + v);
  }
  // pieces of chunks a+1..b: issue 8 pieces' loads at a time (independent,
  // in flight together), then add them in slot order (deterministic)
  int64_t ch = a + 1;
  for (; ch + 8 <= b + 1; ch += 8) {
    TC t[8][V];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const TC* c = carry_vec + (2 * (ch + u)) * kp + q * V;
#pragma unroll
      for (int v = 0; v < V; ++v) t[u][v] = __ldcg(c + v);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] += t[u][v];
  }
  for (; ch <= b; ++ch) {
    const TC* c = carry_vec + (2 * ch) * kp + q * V;
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] += __ldcg(c + v);
  }
  TS* o = out + (int64_t)frow * ldout;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int d = dim_of<TS, V>(q, v);
    if (d < k) o[d] = (TS)(acc[v] * (TC)out_scale);
  }
  if (q == 0) row_cnt[frow] = 0;
}

// Lean grouped worker. Preconditions (checked by the launcher): chunk size
// CB is a multiple of 32 entries; idx / row_of / vals are readable up to
// nnz + 64 entries (the Omega arrays are allocated with that padding), so
// the prefetch loads need no bounds guards. Entry offsets are 32-bit.
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Returns the group's fp64 sum r^2 (all 8 lanes hold it; 0 unless want_sq).
template <typename TS, typename TC, int V>
__device__ __forceinline__ double run_group(const Pass<TS, TC>& P, int chunk, int k, int kp,
                                            int32_t* s_ring, TS* s_vring, TC* s_r) {
  const int q = threadIdx.x & 7;
  const int nnz = (int)P.lay.nnz;
  const int CB = P.cb * 8;
  const int E0 = chunk * CB;
  const bool active = chunk < P.nchunks && E0 < nnz;
  const int E1 = active ? min(E0 + CB, nnz) : E0;
  const int32_t* __restrict__ pidx = P.lay.idx + E0 + q;
  const int32_t* __restrict__ prow = P.lay.row_of + E0 + q;
  const TS* __restrict__ pval = P.vals + E0 + q;
  const uint32_t* __restrict__ pbm = P.lay.bmask + (E0 >> 5);
  constexpr int E = chunk_elems<TS>();
  const TS* __restrict__ self = P.self + q * E;
  // Chunks whose dims are all >= k are not loaded (bit c of livem clear).
  // With one chunk per lane (16-byte slices) the all-padding lanes instead
  // gather lane 0's chunk of the same row: no extra sectors, no predication
  // or register zeroing, and their products vanish because their self-row
  // slice is held at zero. Measured: aliasing wins at one chunk only.
  constexpr bool kAlias = V == E;
  unsigned livem = 0;
#pragma unroll
  for (int c = 0; c < V / E; ++c) livem |= (c * 8 * E + q * E < k ? 1u : 0u) << c;
  const bool live = (livem & 1u) != 0;
  const char* __restrict__ obase =
      reinterpret_cast<const char*>(P.other + (kAlias && !live ? 0 : q * E));
  const uint32_t ostride = (uint32_t)P.ldo * (uint32_t)sizeof(TS);
  const int64_t sstride = P.lds;
  const int nvalid_all = E1 - E0;  // entries of this worker
  bool start_cross = false, end_cross = false;
  int row = 0;
  long long t_start = gtimer();
  if (active) {
    start_cross = (pbm[0] & 1u) == 0u;
    row = P.lay.row_of[E0];
    end_cross = (E1 < nnz) && (((P.lay.bmask[E1 >> 5] >> (E1 & 31)) & 1u) == 0u);
  }
  bool first_row = true;
  int row_first = -1, row_last = -1;
  TC w[V];
  // all-padding lanes hold w = 0 (with ld = k their slice is the next row)
  auto load_w = [&](int rw) {
    TS t[V];
    ldrow<TS, TC, V>(self + (int64_t)rw * sstride, t, livem);
#pragma unroll
    for (int v = 0; v < V; ++v) w[v] = (TC)t[v];
  };
  if (active) load_w(row);
  else {
#pragma unroll
    for (int v = 0; v < V; ++v) w[v] = TC(0);
  }
  long long t_init = 0, t_loop = 0;
  if (P.probe) {
    asm volatile("" ::"f"((float)w[0]));
    t_init = gtimer();
  }
  AccV<TC, V> acc;
#pragma unroll
  for (int v = 0; v < V; ++v) acc.a[v] = TC(0);
  double sq = 0.0;
  auto flush = [&](int frow, bool is_first, bool is_last) {
    int64_t slot = -1;
    if (is_first && start_cross) { slot = 2 * (int64_t)chunk; row_first = frow; }
    else if (is_last && end_cross) { slot = 2 * (int64_t)chunk + 1; row_last = frow; }
    flush_group<TS, TC, V>(P.out, P.ldout, P.out_scale, P.carry_vec, slot, k, kp, frow, acc);
  };

  // Prefetch ring in shared memory, filled with cp.async one 32-entry block
  // ahead: per block the group's 32 column ids, row ids and values (8 x 16 B
  // chunks each; lane q copies chunk q of each stream). The step loop then
  // needs no unrolling (I-cache) and the ring costs no registers.
  const int nblk = P.cb / 4;  // warp-uniform
  constexpr int VPC = 16 / (int)sizeof(TS);  // values per 16-byte chunk
  auto fetch_block = [&](int b) {
    if (b * 32 >= nvalid_all) return;  // never read past this worker's end (+pad)
    const int slot = b & 1;
    const int o = b * 32;
    cp_async16(s_ring + slot * 32 + q * 4, pidx - q + o + q * 4);
    cp_async16(s_ring + 64 + slot * 32 + q * 4, prow - q + o + q * 4);
    if (VPC == 4) {
      cp_async16(s_vring + slot * 32 + q * 4, pval - q + o + q * 4);
    } else {
      cp_async16(s_vring + slot * 32 + q * 4, pval - q + o + q * 4);
      cp_async16(s_vring + slot * 32 + q * 4 + 2, pval - q + o + q * 4 + 2);
    }
  };
  // zero the ring: inactive workers (padding groups of the last warp) and
  // blocks past a worker's end must gather valid rows (index 0)
#pragma unroll
  for (int z = 0; z < 16; ++z) s_ring[q * 16 + z] = 0;
#pragma unroll
  for (int z = 0; z < 8; ++z) s_vring[q * 8 + z] = TS(0);
  __syncwarp();
  fetch_block(0);
  cp_async_commit();
  uint32_t mw_next = nvalid_all > 0 ? pbm[0] : 0u;
  for (int b = 0; b < nblk; ++b) {
    fetch_block(b + 1 < nblk ? b + 1 : nblk);
    cp_async_commit();
    cp_async_wait<1>();   // block b landed (own copies)
    __syncwarp();         // ... and the other lanes' copies of this group
    uint32_t m = mw_next;
    if (b + 1 < nblk && (b + 1) * 32 < nvalid_all) mw_next = pbm[b + 1];
    const int left = nvalid_all - b * 32;
    if (left < 32) m &= left <= 0 ? 0u : ((1u << left) - 1u);
    if (b == 0) m &= ~1u;
    const int slot = b & 1;
#if MFG_UNROLL_U
#pragma unroll
#endif
    for (int u = 0; u < 4; ++u) {
      const int o = b * 32 + u * 8;
      const uint32_t bits = (m >> (8 * u)) & 0xFFu;
      const bool valid = o + q < nvalid_all;
      const int* rc = s_ring + slot * 32 + u * 8;        // this group-batch's cols
      const int* rr = s_ring + 64 + slot * 32 + u * 8;   // ... rows
      const TC a = (TC)s_vring[slot * 32 + u * 8 + q];
      int cols[8];
      {
        const int4 x0 = reinterpret_cast<const int4*>(rc)[0];
        const int4 x1 = reinterpret_cast<const int4*>(rc)[1];
        cols[0] = x0.x; cols[1] = x0.y; cols[2] = x0.z; cols[3] = x0.w;
        cols[4] = x1.x; cols[5] = x1.y; cols[6] = x1.z; cols[7] = x1.w;
      }
      // the self row of the batch's first row start is loaded before the
      // gathers, so its latency overlaps theirs instead of serialising the
      // dots behind it
      int i0 = -1, row0 = 0;
      TS w0[V];
      if (bits) {
        i0 = __ffs(bits) - 1;
        row0 = rr[i0];
        ldrow<TS, TC, V>(self + (int64_t)row0 * sstride, w0, livem);
      }
      TS h[8][V];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        ldrow<TS, TC, V>(reinterpret_cast<const TS*>(obase + (uint64_t)(uint32_t)cols[i] * ostride), h[i],
                         kAlias ? 1u : livem);
      TC p[8];
    const int row_b = row;
    const bool fr_b = first_row;
    // single-row-start specialisation: one-chunk lane slices only (with two
    // chunks, V = 8 fp32, the extra live registers spill)
    const bool one_start = kAlias && bits != 0u && (bits & (bits - 1u)) == 0u;
    if (bits == 0u) {
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = dotv<TS, TC, V>(w, h[i]);
    } else if (one_start) {
      // one row start at i0: entries >= i0 use the new row (branch-free)
      TC wn[V];
#pragma unroll
      for (int v = 0; v < V; ++v) wn[v] = (TC)w0[v];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        TC ws[V];
#pragma unroll
        for (int v = 0; v < V; ++v) ws[v] = i < i0 ? w[v] : wn[v];
        p[i] = dotv<TS, TC, V>(ws, h[i]);
      }
      row = row0;
#pragma unroll
      for (int v = 0; v < V; ++v) w[v] = wn[v];
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if ((bits >> i) & 1u) {
          if (i == i0) {
            row = row0;
#pragma unroll
            for (int v = 0; v < V; ++v) w[v] = (TC)w0[v];
          } else {
            row = rr[i];
            load_w(row);
          }
        }
        p[i] = dotv<TS, TC, V>(w, h[i]);
      }
    }
    TC dot;
    if constexpr (MFG_SMEM_REDUCE && sizeof(TC) == 4) {
      // transpose through shared memory: lane q writes its partials of the 8
      // entries down column q, then sums row q (entry q) in fixed order
      TC* s_p = s_r + 8;
#pragma unroll
      for (int i = 0; i < 8; ++i) s_p[i * 8 + q] = p[i];
      __syncwarp();
      TC t[8];
      ld4<TC>(s_p + q * 8, *reinterpret_cast<TC(*)[4]>(&t[0]));
      ld4<TC>(s_p + q * 8 + 4, *reinterpret_cast<TC(*)[4]>(&t[4]));
      dot = ((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7]));
    } else {
      dot = reduce8(p);
    }
    const TC r = valid ? dot - a : TC(0);
    if (valid) {
      if (P.R) P.R[E0 + o + q] = (TS)r;
      sq += (double)r * (double)r;
    }
    __syncwarp();
    s_r[q] = r;
    __syncwarp();
    TC r8[8];
    ld4<TC>(s_r, *reinterpret_cast<TC(*)[4]>(&r8[0]));
    ld4<TC>(s_r + 4, *reinterpret_cast<TC(*)[4]>(&r8[4]));
    if (bits == 0u) {
#pragma unroll
      for (int i = 0; i < 8; ++i) axpyv<TS, TC, V>(acc.a, r8[i], h[i]);
    } else if (one_start) {
      // entries < i0 finish the current row, the rest start the new one
#pragma unroll
      for (int i = 0; i < 8; ++i) axpyv<TS, TC, V>(acc.a, i < i0 ? r8[i] : TC(0), h[i]);
      flush(row_b, fr_b, false);
      first_row = false;
#pragma unroll
      for (int j = 0; j < V; ++j) acc.a[j] = TC(0);
#pragma unroll
      for (int i = 0; i < 8; ++i) axpyv<TS, TC, V>(acc.a, i < i0 ? TC(0) : r8[i], h[i]);
    } else {
      int rw = row_b;
      bool fr = fr_b;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if ((bits >> i) & 1u) {
          flush(rw, fr, false);
          fr = false;
          rw = rr[i];
#pragma unroll
          for (int j = 0; j < V; ++j) acc.a[j] = TC(0);
        }
        axpyv<TS, TC, V>(acc.a, r8[i], h[i]);
      }
      first_row = fr;
    }
    }
  }
  cp_async_wait<0>();
  if (P.probe) {
    asm volatile("" ::"f"((float)acc.a[0]));
    t_loop = gtimer();
  }
  if (active) {
    flush(row, first_row, true);
    if (q == 0 && !P.row_cnt) {
      P.carry_row[2 * chunk] = row_first;
      P.carry_row[2 * chunk + 1] = row_last;
    }
  }
  if (P.row_cnt) {
    // Deferred crossing notification: every lane fences its own carry
    // stores (one MEMBAR.GPU per warp, no L1 invalidation) before the group
    // leaders' release increments in finish_row; the worker depositing a
    // row's last piece finishes it.
    __syncwarp();
    const bool any = __any_sync(0xffffffffu, row_first >= 0 || row_last >= 0);
    if (any) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      __syncwarp();
      const int64_t CB64 = CB;
      if (row_first >= 0)
        finish_row<TS, TC, V>(P.out, P.ldout, P.out_scale, P.carry_vec, P.row_cnt, P.lay.ptr,
                              CB64, k, kp, row_first);
      if (row_last >= 0)
        finish_row<TS, TC, V>(P.out, P.ldout, P.out_scale, P.carry_vec, P.row_cnt, P.lay.ptr,
                              CB64, k, kp, row_last);
    }
  }
  if (P.probe && active && q == 0) {
    long long* pr = P.probe + 10 * (int64_t)chunk;
    pr[0] = t_start;
    pr[1] = t_init;
    pr[2] = t_loop;
    pr[3] = gtimer();
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  return P.want_sq ? sq : 0.0;
}


struct SumJob {
  const double* part;  // [3][np]
  int np;
  const void* W;       // optional dense norms
  int64_t wcount;
  const void* H;
  int64_t hcount;
  int is_f64;
  double* block_part;  // [gridDim.x][5]
  unsigned int* counter;
  double* sums;        // [5] out: sq, s1, s2, |W|^2, |H|^2 (first 3 used by callers)
};

// One warp per head slot. Heads are the used odd slots (a row's last
// chunk-crossing); the run of slots carrying the same row follows in slot
// order (unused slots = -1), and is summed in that fixed order.
template <typename TS, typename TC>
__device__ void carry_head(const Pass<TS, TC>& P, int k, int q) {
  const int lane = lane_id();
  const int nslots = 2 * P.nchunks;
  const int cs = P.cstride;
  const int row = P.carry_row[q];
  if (row < 0) return;
  int end = q + 1;
  while (end < nslots) {
    const int sidx = end + lane;
    const int r2 = sidx < nslots ? P.carry_row[sidx] : -2;
    const bool stop = (sidx >= nslots) || (r2 >= 0 && r2 != row);
    const unsigned b = __ballot_sync(0xffffffffu, stop);
    if (b) { end += __ffs(b) - 1; break; }
    end += 32;
  }
  if (end > nslots) end = nslots;
  for (int d0 = 0; d0 < k; d0 += 32) {
    const int d = d0 + lane;
    TC v = TC(0);
    if (d < k) {
#pragma unroll 4
      for (int sl = q; sl < end; ++sl) {
        if (P.carry_row[sl] == row) v += P.carry_vec[(int64_t)sl * cs + d];
      }
      P.out[(int64_t)row * P.ldout + d] = (TS)(v * (TC)P.out_scale);
    }
  }
}

template <typename TS, typename TC>
__device__ void empty_rows_zero(const Pass<TS, TC>& P, int k, int warp_global, int nwarps_grid) {
  const int lane = lane_id();
  for (int i = warp_global; i < P.lay.n_empty; i += nwarps_grid) {
    const int row2 = P.lay.empty_rows[i];
    for (int d = lane; d < k; d += 32) P.out[(int64_t)row2 * P.ldout + d] = TS(0);
  }
}

__device__ __forceinline__ double ldv(const void* p, int64_t i, int is_f64) {
  return is_f64 ? static_cast<const double*>(p)[i] : (double)static_cast<const float*>(p)[i];
}

template <typename TS, typename TC>
__global__ void __launch_bounds__(256)
k_epilogue(Pass<TS, TC> P0, int has0, Pass<TS, TC> P1, int has1, int k, SumJob J) {
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwg = (gridDim.x * blockDim.x) >> 5;
  // carries: warp wg owns head slot 2*wg+1 of each pass (grid sized for it)
  if (has0 && P0.out) {
    for (int q = 2 * wg + 1; q < 2 * P0.nchunks; q += 2 * nwg) carry_head(P0, k, q);
    empty_rows_zero(P0, k, wg, nwg);
  }
  if (has1 && P1.out) {
    for (int q = 2 * wg + 1; q < 2 * P1.nchunks; q += 2 * nwg) carry_head(P1, k, q);
    empty_rows_zero(P1, k, wg, nwg);
  }
  if (!J.block_part) return;
  __shared__ double sm[8];
  double v[5] = {0, 0, 0, 0, 0};
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < J.np; i += nth) {
    v[0] += J.part[i];
    v[1] += J.part[J.np + i];
    v[2] += J.part[2 * J.np + i];
  }
  if (J.W)
    for (int64_t i = tid; i < J.wcount; i += nth) {
      const double x = ldv(J.W, i, J.is_f64);
      v[3] += x * x;
    }
  if (J.H)
    for (int64_t i = tid; i < J.hcount; i += nth) {
      const double x = ldv(J.H, i, J.is_f64);
      v[4] += x * x;
    }
  for (int c = 0; c < 5; ++c) {
    const double s = block_sum<256>(v[c], sm);
    if (threadIdx.x == 0) J.block_part[blockIdx.x * 5 + c] = s;
  }
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int done = atomicAdd(J.counter, 1u);
    last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    __threadfence();
    const volatile double* bp = J.block_part;
    for (int c = 0; c < 5; ++c) {
      double t = 0.0;
      for (unsigned int b = threadIdx.x; b < gridDim.x; b += blockDim.x) t += bp[b * 5 + c];
      const double tot = block_sum<256>(t, sm);
      if (threadIdx.x == 0) J.sums[c] = tot;
    }
    if (threadIdx.x == 0) *J.counter = 0u;
  }
}

struct FusedRed {
  const void* W;
  int64_t wcount;
  const void* H;
  int64_t hcount;
  int is_f64;
  double* block_part;    // [gridDim.x][3]
  unsigned int* counter; // zero at rest (the last block re-zeroes it)
  double* sums;          // out: sum r^2, |W|^2, |H|^2
};

__device__ __forceinline__ double ldv2(const void* p, int64_t i, int is_f64) {
  return is_f64 ? static_cast<const double*>(p)[i] : (double)static_cast<const float*>(p)[i];
}

template <typename TS, typename TC>
__device__ __forceinline__ void sweep_tail(const Pass<TS, TC>& P0, const Pass<TS, TC>& P1, int k,
                                           const FusedRed& F, double sq, int lblk);

template <typename TS, typename TC, int V>
__global__ void __launch_bounds__(kGThreads, g8_min_blocks<TS, TC, V>())
k_sweep_g8f(Pass<TS, TC> P0, Pass<TS, TC> P1, int nb0, int nb1, int k, int kp, FusedRed F) {
  __shared__ __align__(16) int32_t s_ring[kGThreads / 8][128];   // [cols|rows][2 slots][32]
  __shared__ __align__(16) TS s_vring[kGThreads / 8][64];        // [2 slots][32]
  // per worker: r of the batch [8] (+ the 8 x 8 partial-dot transpose)
  __shared__ __align__(16) TC s_r[kGThreads / 8][(MFG_SMEM_REDUCE && sizeof(TC) == 4) ? 72 : 8];
  __shared__ int s_ticket;
  const int gl = threadIdx.x >> 3;
  // diagnostics: block entry stamps after the per-worker records
  if (P0.probe && threadIdx.x == 0)
    P0.probe[10 * (int64_t)(P0.nchunks + P1.nchunks) + 2 * blockIdx.x] = gtimer();
  // Pass affinity by SM: CTAs on the first nb0/(nb0+nb1) of the SMs take
  // CSR work blocks, the others CSC, so each SM's L1 holds one gathered
  // factor (H or W) instead of both. Blocks are handed out by tickets; a CTA
  // whose pass is exhausted takes the other pass (the counts always fit:
  // grid = nb0 + nb1). The last block re-zeroes the tickets.
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const int pref = (int)smid * (nb0 + nb1) < kNumSMs * nb0 ? 0 : 1;
    unsigned int* tick = F.counter + 1 + gridDim.x;
    int t = (int)atomicAdd(&tick[pref], 1u);
    int pass = pref;
    if (t >= (pref ? nb1 : nb0)) {
      pass = 1 - pref;
      t = (int)atomicAdd(&tick[pass], 1u);
    }
    s_ticket = (pass << 30) | t;
  }
  __syncthreads();
  double sq = 0.0;
  {
    const bool second = (s_ticket >> 30) != 0;
    const int wk = (s_ticket & ((1 << 30) - 1)) * (kGThreads / 8) + gl;  // worker in its pass
    // one inlined copy of the worker (I-cache): select the orientation's pass
    const Pass<TS, TC>& P = second ? P1 : P0;
    if (((wk & ~3) < P.nchunks))  // warp-uniform
      sq = run_group<TS, TC, V>(P, wk, k, kp, s_ring[gl], s_vring[gl], s_r[gl]);
  }
  // fixed-order reductions: partial slots follow the logical work block,
  // not the (dynamically ticketed) CTA
  const int lblk = (s_ticket >> 30) ? nb0 + (s_ticket & ((1 << 30) - 1)) : s_ticket;
  sweep_tail(P0, P1, k, F, sq, lblk);
}

// Kernel-wide tail of the fused sweep: zero the empty rows, and reduce
// sum r^2 (per-group sums) and the dense norms |W|^2, |H|^2 in fp64.
template <typename TS, typename TC>
__device__ __forceinline__ void sweep_tail(const Pass<TS, TC>& P0, const Pass<TS, TC>& P1, int k,
                                           const FusedRed& F, double sq, int lblk) {
  const int lane = threadIdx.x & 31;
  // fold the 4 groups' sums (each group's lanes hold its sum)
  sq += __shfl_xor_sync(0xffffffffu, sq, 8);
  sq += __shfl_xor_sync(0xffffffffu, sq, 16);
  const int wg = (lblk * kGThreads + threadIdx.x) >> 5;
  const int nwg = (gridDim.x * kGThreads) >> 5;
  empty_rows_zero(P0, k, wg, nwg);
  empty_rows_zero(P1, k, wg, nwg);
  // per-warp fp64 partials of the dense norms (fixed slices)
  const int64_t gl0 = (int64_t)wg * 32 + lane, gstride = (int64_t)nwg * 32;
  double w2 = 0.0, h2 = 0.0;
  for (int64_t i = gl0; i < F.wcount; i += gstride) { const double x = ldv2(F.W, i, F.is_f64); w2 += x * x; }
  for (int64_t i = gl0; i < F.hcount; i += gstride) { const double x = ldv2(F.H, i, F.is_f64); h2 += x * x; }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    w2 += __shfl_xor_sync(0xffffffffu, w2, o);
    h2 += __shfl_xor_sync(0xffffffffu, h2, o);
  }
  // One-level last-arriver fold: the CTA sums its warps' partials in shared
  // memory (fixed order) and publishes them; the last CTA to arrive sums the
  // block partials with all its threads (fixed assignment + fixed tree).
  __shared__ double s_part[kGThreads / 32][3];
  __shared__ int s_last;
  double* bp = F.block_part;   // [gridDim.x][3] block partials
  const int wib = threadIdx.x >> 5;
  if (lane == 0) {
    s_part[wib][0] = sq;
    s_part[wib][1] = w2;
    s_part[wib][2] = h2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b0 = 0.0, b1 = 0.0, b2 = 0.0;
#pragma unroll
    for (int w = 0; w < kGThreads / 32; ++w) {
      b0 += s_part[w][0];
      b1 += s_part[w][1];
      b2 += s_part[w][2];
    }
    bp[3 * lblk] = b0;
    bp[3 * lblk + 1] = b1;
    bp[3 * lblk + 2] = b2;
    // release RMW (all CTAs' increments form one release sequence); the last
    // arriver's acq_rel RMW synchronises with every earlier block partial
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(old) : "l"(F.counter) : "memory");
    s_last = old == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  double u0 = 0.0, u1 = 0.0, u2 = 0.0;
  for (unsigned int b2 = threadIdx.x; b2 < gridDim.x; b2 += kGThreads) {
    u0 += __ldcg(bp + 3 * b2);
    u1 += __ldcg(bp + 3 * b2 + 1);
    u2 += __ldcg(bp + 3 * b2 + 2);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    u0 += __shfl_xor_sync(0xffffffffu, u0, o);
    u1 += __shfl_xor_sync(0xffffffffu, u1, o);
    u2 += __shfl_xor_sync(0xffffffffu, u2, o);
  }
  __syncthreads();  // s_part reuse
  if (lane == 0) {
    s_part[wib][0] = u0;
    s_part[wib][1] = u1;
    s_part[wib][2] = u2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double v0 = 0.0, v1 = 0.0, v2 = 0.0;
#pragma unroll
    for (int w = 0; w < kGThreads / 32; ++w) {
      v0 += s_part[w][0];
      v1 += s_part[w][1];
      v2 += s_part[w][2];
    }
    F.sums[0] = v0;
    F.sums[1] = v1;
    F.sums[2] = v2;
    *F.counter = 0u;
    F.counter[1 + gridDim.x] = 0u;  // pass tickets
    F.counter[2 + gridDim.x] = 0u;
    if (P0.probe) P0.probe[10 * (int64_t)(P0.nchunks + P1.nchunks) + 2 * lblk + 1] = gtimer();
  }
}

constexpr int kEpiBlocksMax = 32 * kNumSMs;

int epi_blocks(int nch0, int nch1) {
  const int heads = nch0 > nch1 ? nch0 : nch1;
  int b = (heads + 7) / 8;
  if (b < 2 * kNumSMs) b = 2 * kNumSMs;
  if (b > kEpiBlocksMax) b = kEpiBlocksMax;
  return b;
}

int pick_cb(int64_t nnz) {
  // target >= ~16 warps per SM of chunks, batches in [2, 32]
  int64_t target_chunks = (int64_t)kNumSMs * 16;
  int64_t cb = (nnz / 32 + target_chunks - 1) / target_chunks;
  if (cb < 2) cb = 2;
  if (cb > 32) cb = 32;
  return (int)cb;
}

int chunks_of(int64_t nnz, int cb) {
  return (int)((nnz + (int64_t)cb * 32 - 1) / ((int64_t)cb * 32));
}

// Grouped (v3) kernel: padded factor width for k, or 0 if not eligible.
int grouped_kp(int k, int elem_bytes) {
  if (elem_bytes == 4) return k <= 32 ? 32 : (k <= 64 ? 64 : 0);
  return k <= 16 ? 16 : (k <= 32 ? 32 : 0);
}

int pick_cb_g(int64_t nnz) {
  // Target worker count per orientation (default: one resident wave for both
  // passes, 16 warps x 4 groups per SM). Longer chunks amortise the
  // per-worker fixed costs (schedule lookup chain, crossing-row notification).
  static const int64_t env_target = [] {
    const char* e = getenv("MFG_WORKERS_PER_SM");
    return e ? (int64_t)atoi(e) : (int64_t)32;
  }();
  const int64_t target = (int64_t)kNumSMs * env_target;
  int64_t cb = (nnz + 8 * target - 1) / (8 * target);
  if (cb < 4) cb = 4;
  if (cb > 512) cb = 512;
  return (int)((cb + 3) & ~3);
}

int chunks_of_g(int64_t nnz, int cb) {
  return (int)((nnz + (int64_t)cb * 8 - 1) / ((int64_t)cb * 8));
}

template <typename C>
void carve_pass(C& c, const mfg_layout* lay, int k, bool acc, bool part) {
  if (!lay) return;
  // room for either schedule: warp chunks (stride k) or group chunks (stride kp)
  const int cb = pick_cb(lay->nnz);
  int64_t nch = chunks_of(lay->nnz, cb) > 0 ? chunks_of(lay->nnz, cb) : 1;
  const int kp = grouped_kp(k, 4) ? grouped_kp(k, 4) : k;
  const int64_t nchg = chunks_of_g(lay->nnz, pick_cb_g(lay->nnz)) + 4;
  const size_t carry = (size_t)2 * (nch * k > nchg * kp ? nch * k : nchg * kp);
  if (nchg > nch) nch = nchg;
  if (acc) {
    c.template take<double>(carry);  // carry vecs (sized for fp64)
    c.template take<int32_t>((size_t)2 * nch);
  }
  if (part) c.template take<double>((size_t)3 * nch);
}

template <typename C>
void carve_epi(C& c) {
  c.template take<double>((size_t)kEpiBlocksMax * 5);
  c.template take<unsigned int>(1);
  c.template take<double>(5);
}

template <typename TS, typename TC>
bool setup_pass(Pass<TS, TC>& P, Carver& c, const mfg_layout* lay, int k, bool acc, bool part,
                int kp_grouped = 0) {
  P.lay = *lay;
  if (kp_grouped) {
    P.cb = pick_cb_g(lay->nnz);
    P.nchunks = chunks_of_g(lay->nnz, P.cb);
    P.cstride = kp_grouped;
  } else {
    P.cb = pick_cb(lay->nnz);
    P.nchunks = chunks_of(lay->nnz, P.cb);
    P.cstride = k;
  }
  const int nch = P.nchunks > 0 ? P.nchunks : 1;
  P.carry_vec = nullptr;
  P.carry_row = nullptr;
  P.part = nullptr;
  if (acc) {
    P.carry_vec = reinterpret_cast<TC*>(c.take<double>((size_t)2 * nch * P.cstride));
    P.carry_row = c.take<int32_t>((size_t)2 * nch);
  }
  if (part) P.part = c.take<double>((size_t)3 * nch);
  return c.ok;
}


// CTAs of the grouped kernel: one per kGThreads/8 workers of each pass.
int grouped_blocks(int nchunks) { return (nchunks + kGThreads / 8 - 1) / (kGThreads / 8); }
int grouped_grid(int n0, int n1) {
  const int g = grouped_blocks(n0) + grouped_blocks(n1);
  return g < 1 ? 1 : g;
}

template <typename TS, typename TC>
int launch_grouped(const Pass<TS, TC>& P0, const Pass<TS, TC>& P1, int k, int kp,
                   const FusedRed& F, cudaStream_t stream) {
  const int nb0 = grouped_blocks(P0.nchunks), nb1 = grouped_blocks(P1.nchunks);
  const int grid = grouped_grid(P0.nchunks, P1.nchunks);
  if (grid != nb0 + nb1) return MFG_ERR_ARG;  // empty passes are not launched here
  const int V = kp / 8;
  constexpr bool f32 = sizeof(TS) == 4, mixed = sizeof(TS) != sizeof(TC);
  auto go = [&](auto kern) { kern<<<grid, kGThreads, 0, stream>>>(P0, P1, nb0, nb1, k, kp, F); };
  if constexpr (f32 && !mixed) {
    if (V == 4) go(k_sweep_g8f<TS, TC, 4>);
    else go(k_sweep_g8f<TS, TC, 8>);
  } else if constexpr (f32) {
    go(k_sweep_g8f<TS, TC, 4>);
  } else {
    if (V == 2) go(k_sweep_g8f<TS, TC, 2>);
    else go(k_sweep_g8f<TS, TC, 4>);
  }
  MFG_LAUNCH_CHECK();
  return MFG_OK;
}

template <typename TS, typename TC, bool ACC>
int launch_main(const Pass<TS, TC>& P0, const Pass<TS, TC>& P1, int n0, int n1, int k,
                cudaStream_t stream) {
  const int nwt = n0 + n1;
  if (nwt == 0) return MFG_OK;
  const int grid = (nwt + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const bool f32s = sizeof(TS) == 4;
  if (k <= 32) {
    k_sweep<TS, TC, 1, ACC, false><<<grid, kThreads, 0, stream>>>(P0, P1, n0, nwt, k);
  } else if (k <= 64 && f32s) {
    k_sweep<TS, TC, 2, ACC, false><<<grid, kThreads, 0, stream>>>(P0, P1, n0, nwt, k);
  } else {
    const size_t smem = ACC ? (size_t)kWarpsPerBlock * k * sizeof(TC) : 0;
    if (smem > 48 * 1024) {
      cudaFuncSetAttribute(k_sweep<TS, TC, 1, ACC, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    k_sweep<TS, TC, 1, ACC, true><<<grid, kThreads, smem, stream>>>(P0, P1, n0, nwt, k);
  }
  MFG_LAUNCH_CHECK();
  return MFG_OK;
}

template <typename TS, typename TC>
// W / H: the self rows of the CSR / CSC pass (and the rows the norms cover);
// Wg / Hg: the factors the CSC / CSR pass gathers from. One Omega: Wg = W,
// Hg = H. A rank's shards (mfg_sweep_sharded): W = its row block of W,
// H = its column block of H, Wg / Hg = the full replicas.
int do_sweep(const mfg_layout* csr, const mfg_layout* csc, int k, const void* vals_csr,
             const void* vals_csc, const void* W, int ldw, const void* H, int ldh, void* R,
             void* RH, void* RtW, double out_scale, double* sums, void* ws, size_t wsb,
             cudaStream_t stream, const void* Wg = nullptr, const void* Hg = nullptr) {
  if (!Wg) Wg = W;
  if (!Hg) Hg = H;
  Carver c(ws, wsb);
  // persistent, zero-at-rest state first (fixed offsets for every path)
  int32_t* cnt0 = c.take<int32_t>((size_t)csr->nrows + 1);
  int32_t* cnt1 = c.take<int32_t>((size_t)csc->nrows + 1);
  const int ggrid = grouped_grid(chunks_of_g(csr->nnz, pick_cb_g(csr->nnz)),
                                 chunks_of_g(csc->nnz, pick_cb_g(csc->nnz)));
  unsigned int* fcounter = c.take<unsigned int>((size_t)ggrid + 3);  // fold, per-block, 2 tickets
  Pass<TS, TC> P0{}, P1{};
  const bool acc0 = RH != nullptr, acc1 = RtW != nullptr;
  // grouped v3 kernel: zero-padded factors of width kp, all outputs wanted
  int kpg = grouped_kp(k, (int)sizeof(TS));
  if (sizeof(TS) != sizeof(TC) && kpg > 32) kpg = 0;  // fp64 compute on fp32: V = 4 only
  // factor layouts of the grouped kernel: zero-padded to kp, or unpadded
  // (ld = k) when rows are whole 16-byte chunks (k * sizeof(TS) % 16 == 0)
  const bool ld_ok = kpg && ((ldw == kpg && ldh == kpg) ||
                             (ldw == k && ldh == k && ((size_t)k * sizeof(TS)) % 16 == 0));
  const bool grouped = ld_ok && acc0 && acc1 && csr->nnz > 0;
  if (!setup_pass(P0, c, csr, k, acc0, true, grouped ? kpg : 0)) goto small;
  if (!setup_pass(P1, c, csc, k, acc1, false, grouped ? kpg : 0)) goto small;
  {
    P0.vals = (const TS*)vals_csr; P0.G = nullptr; P0.self = (const TS*)W; P0.lds = ldw;
    P0.scale = nullptr; P0.other = (const TS*)Hg; P0.ldo = ldh; P0.R = (TS*)R; P0.r_mult = 1.0;
    P0.out = (TS*)RH; P0.ldout = k; P0.out_scale = out_scale; P0.want_sq = 1;
    P1.vals = (const TS*)vals_csc; P1.G = nullptr; P1.self = (const TS*)H; P1.lds = ldh;
    P1.scale = nullptr; P1.other = (const TS*)Wg; P1.ldo = ldw; P1.R = nullptr; P1.r_mult = 1.0;
    P1.out = (TS*)RtW; P1.ldout = k; P1.out_scale = out_scale; P1.want_sq = 0;
    SumJob J{};
    {
      const size_t gb = grouped ? (size_t)grouped_grid(P0.nchunks, P1.nchunks) * (3 + 3 * (kGThreads / 32)) : 0;
      J.block_part = c.take<double>(gb > (size_t)kEpiBlocksMax * 5 ? gb : (size_t)kEpiBlocksMax * 5);
    }
    J.counter = c.take<unsigned int>(1);
    double* tmp = c.take<double>(5);
    if (!c.ok) goto small;
    J.part = P0.part; J.np = P0.nchunks;
    // norms over the ld-strided buffers: padding columns must be zero
    J.W = W; J.wcount = (int64_t)csr->nrows * ldw;
    J.H = H; J.hcount = (int64_t)csc->nrows * ldh;
    J.is_f64 = sizeof(TS) == 8;
    J.sums = tmp;
    if (ldw < k || ldh < k) { set_error("sweep requires ldw, ldh >= k"); return MFG_ERR_ARG; }
    const int n0 = csr->nnz ? P0.nchunks : 0;
    const int n1 = (acc1 && csc->nnz) ? P1.nchunks : 0;
    int st;
    // counter must start at zero: the epilogue's last block re-zeroes it.
    if (!grouped) MFG_CUDA_CHECK(cudaMemsetAsync(J.counter, 0, sizeof(unsigned int), stream));
    prof_begin(stream);
    if (grouped) {
      P0.row_cnt = cnt0;
      P1.row_cnt = cnt1;
      P0.probe = P1.probe = nullptr;
      if (g_probe) {
        P0.probe = g_probe;
        P1.probe = g_probe + 10 * (int64_t)P0.nchunks;
      }
      FusedRed F{};
      F.W = W; F.wcount = J.wcount; F.H = H; F.hcount = J.hcount; F.is_f64 = J.is_f64;
      // the last block writes [sum r^2, |W|^2, |H|^2] straight into the caller's
      // sums (no trailing device-to-device copy node in the sweep)
      F.block_part = J.block_part; F.counter = fcounter; F.sums = sums;
      st = launch_grouped<TS, TC>(P0, P1, k, kpg, F, stream);
      prof_end(stream);
      return st;
    }
    if (acc0 || acc1) st = launch_main<TS, TC, true>(P0, P1, n0, n1, k, stream);
    else st = launch_main<TS, TC, false>(P0, P1, n0, 0, k, stream);
    prof_end(stream);
    if (st != MFG_OK) return st;
    if (n0 == 0) {  // no entries: partials are zero
      MFG_CUDA_CHECK(cudaMemsetAsync(P0.part, 0, sizeof(double) * 3, stream));
      J.np = 1;
    }
    k_epilogue<TS, TC><<<epi_blocks(acc0 ? P0.nchunks : 0, acc1 ? P1.nchunks : 0), 256, 0, stream>>>(
        P0, acc0 ? 1 : 0, P1, acc1 ? 1 : 0, k, J);
    MFG_LAUNCH_CHECK();
    // sums = [sq, |W|^2, |H|^2]
    MFG_CUDA_CHECK(cudaMemcpyAsync(sums, tmp, sizeof(double), cudaMemcpyDeviceToDevice, stream));
    MFG_CUDA_CHECK(cudaMemcpyAsync(sums + 1, tmp + 3, 2 * sizeof(double),
                                   cudaMemcpyDeviceToDevice, stream));
    return MFG_OK;
  }
small:
  set_error("sweep workspace too small");
  return MFG_ERR_ARG;
}

template <typename TS, typename TC>
int do_sddmm(const mfg_layout* lay, int k, const void* L, int ldl, const double* scale,
             const void* Rt, int ldr, const void* A, const void* G, double out_mult, void* out,
             double* sums, void* ws, size_t wsb, cudaStream_t stream) {
  Carver c(ws, wsb);
  Pass<TS, TC> P{};
  if (!setup_pass(P, c, lay, k, false, true)) {
    set_error("sddmm workspace too small");
    return MFG_ERR_ARG;
  }
  P.vals = (const TS*)A; P.G = (const TS*)G; P.self = (const TS*)L; P.lds = ldl; P.scale = scale;
  P.other = (const TS*)Rt; P.ldo = ldr; P.R = (TS*)out; P.r_mult = out_mult; P.out = nullptr;
  P.ldout = 0; P.out_scale = 1.0; P.want_sq = 1;
  SumJob J{};
  J.block_part = c.take<double>((size_t)kEpiBlocksMax * 5);
  J.counter = c.take<unsigned int>(1);
  double* tmp = c.take<double>(5);
  if (!c.ok) {
    set_error("sddmm workspace too small");
    return MFG_ERR_ARG;
  }
  J.part = P.part; J.np = P.nchunks; J.is_f64 = sizeof(TS) == 8; J.sums = tmp;
  MFG_CUDA_CHECK(cudaMemsetAsync(J.counter, 0, sizeof(unsigned int), stream));
  const int n0 = lay->nnz ? P.nchunks : 0;
  int st = launch_main<TS, TC, false>(P, P, n0, 0, k, stream);
  if (st != MFG_OK) return st;
  if (n0 == 0) {
    MFG_CUDA_CHECK(cudaMemsetAsync(P.part, 0, sizeof(double) * 3, stream));
    J.np = 1;
  }
  k_epilogue<TS, TC><<<2 * kNumSMs, 256, 0, stream>>>(P, 0, P, 0, k, J);
  MFG_LAUNCH_CHECK();
  if (sums)
    MFG_CUDA_CHECK(cudaMemcpyAsync(sums, tmp, 3 * sizeof(double), cudaMemcpyDeviceToDevice, stream));
  return MFG_OK;
}

}  // namespace

size_t sweep_workspace(const mfg_layout* csr, const mfg_layout* csc, int k) {
  Sizer s;
  s.take<int32_t>((size_t)csr->nrows + 1);
  s.take<int32_t>((size_t)csc->nrows + 1);
  const int64_t gg = grouped_grid(chunks_of_g(csr->nnz, pick_cb_g(csr->nnz)),
                                  chunks_of_g(csc->nnz, pick_cb_g(csc->nnz)));
  s.take<unsigned int>((size_t)gg + 3);
  carve_pass(s, csr, k, true, true);
  carve_pass(s, csc, k, true, false);
  carve_epi(s);
  const int64_t g = grouped_grid(chunks_of_g(csr->nnz, pick_cb_g(csr->nnz)),
                                 chunks_of_g(csc->nnz, pick_cb_g(csc->nnz)));
  s.take<double>((size_t)g * (3 + 3 * (kGThreads / 32)));
  return s.off + 1024;
}

int sweep_ld(int dtype, int compute_f64, int k) {
  const int es = dtype == MFG_F64 ? 8 : 4;
  int kp = grouped_kp(k, es);
  if (dtype != MFG_F64 && compute_f64 && kp > 32) kp = 0;
  if (!kp) return k;
  return (k * es) % 16 == 0 ? k : kp;
}

size_t sddmm_workspace(const mfg_layout* lay, int k) {
  Sizer s;
  carve_pass(s, lay, k, false, true);
  carve_epi(s);
  return s.off + 1024;
}

int sweep_dispatch(int dtype, int compute_f64, const mfg_layout* csr, const mfg_layout* csc,
                   int k, const void* vals_csr, const void* vals_csc, const void* W, int ldw,
                   const void* H, int ldh, void* R, void* RH, void* RtW, double out_scale,
                   double* sums, void* ws, size_t wsb, cudaStream_t stream, const void* Wg,
                   const void* Hg) {
  if (dtype == MFG_F64)
    return do_sweep<double, double>(csr, csc, k, vals_csr, vals_csc, W, ldw, H, ldh, R, RH, RtW,
                                     out_scale, sums, ws, wsb, stream, Wg, Hg);
  if (compute_f64)
    return do_sweep<float, double>(csr, csc, k, vals_csr, vals_csc, W, ldw, H, ldh, R, RH, RtW,
                                    out_scale, sums, ws, wsb, stream, Wg, Hg);
  return do_sweep<float, float>(csr, csc, k, vals_csr, vals_csc, W, ldw, H, ldh, R, RH, RtW,
                                 out_scale, sums, ws, wsb, stream, Wg, Hg);
}

int sddmm_dispatch(int dtype, int compute_f64, const mfg_layout* lay, int k, const void* L,
                   int ldl, const double* scale, const void* Rt, int ldr, const void* A,
                   const void* G, double out_mult, void* out, double* sums, void* ws, size_t wsb,
                   cudaStream_t stream) {
  if (dtype == MFG_F64)
    return do_sddmm<double, double>(lay, k, L, ldl, scale, Rt, ldr, A, G, out_mult, out, sums, ws,
                                     wsb, stream);
  if (compute_f64)
    return do_sddmm<float, double>(lay, k, L, ldl, scale, Rt, ldr, A, G, out_mult, out, sums, ws,
                                    wsb, stream);
  return do_sddmm<float, float>(lay, k, L, ldl, scale, Rt, ldr, A, G, out_mult, out, sums, ws,
                                 wsb, stream);
}

}  // namespace mfg

extern "C" int mfg_profile_enable(int max_records) {
  using mfg::g_prof;
  for (auto e : g_prof.start) cudaEventDestroy(e);
  for (auto e : g_prof.stop) cudaEventDestroy(e);
  g_prof.start.clear();
  g_prof.stop.clear();
  g_prof.used = 0;
  g_prof.on = max_records > 0;
  for (int i = 0; i < max_records; ++i) {
    cudaEvent_t a, b;
    MFG_CUDA_CHECK(cudaEventCreate(&a));
    MFG_CUDA_CHECK(cudaEventCreate(&b));
    g_prof.start.push_back(a);
    g_prof.stop.push_back(b);
  }
  return MFG_OK;
}

extern "C" int mfg_profile_collect(double* total_ms, int* count) {
  using mfg::g_prof;
  double t = 0.0;
  for (size_t i = 0; i < g_prof.used; ++i) {
    MFG_CUDA_CHECK(cudaEventSynchronize(g_prof.stop[i]));
    float ms = 0.f;
    MFG_CUDA_CHECK(cudaEventElapsedTime(&ms, g_prof.start[i], g_prof.stop[i]));
    t += ms;
  }
  *total_ms = t;
  *count = (int)g_prof.used;
  g_prof.used = 0;
  return MFG_OK;
}

extern "C" int mfg_set_probe(void* dev_buffer) {
  mfg::g_probe = static_cast<long long*>(dev_buffer);
  return MFG_OK;
}
