// BCD half-sweep: exact per-row minimisers of the MF objective.
//
// Replaces _half_sweep (mfg/mfsolver.py:53-75), which assembles the per-row
// normal matrices lam*I + 2*sum_{j in Omega_i} o_j o_j^T with a pattern SpMM
// over k(k+1)/2 pair-product columns (materialising (m, k, k) fp64 normals
// and (m, k(k+1)/2) pair products on the host) and then runs a batched LU
// solve. Here one CTA owns one row at a time: the gathered factor rows are
// staged through shared memory in chunks of kC entries, the Gram matrix is
// accumulated in fp64 register tiles (4x4 per thread, upper triangle only)
// into shared memory, and the SPD system is solved in place by Cholesky.
// Nothing of size (m, k, k) ever exists, so config 5 (n ~ 1e6, k = 64) runs.
// Arithmetic is fp64 for both storage types.
#include <cub/cub.cuh>

#include "common.cuh"
#include "engine.cuh"

namespace mfg {
namespace {

constexpr int kNT = 128;
constexpr int kC = 16;         // entries staged per chunk (packed/dual kernel)
#ifndef MFG_BCD_KCS
#define MFG_BCD_KCS 32
#endif
constexpr int kCS = MFG_BCD_KCS;  // entries per chunk of the small-k shared-memory path (fewer
                                  // gather round trips and barriers per row)

// Small-k shared-memory path (entry groups, see k_bcd): at most NT/2 upper
// 4x4 tiles. Only it stages kCS entries per chunk and keeps the group
// partials; larger k keeps kC-entry chunks and no partials buffer, since
// the shared-memory footprint sets how many CTAs fit on an SM there.
__host__ __device__ constexpr bool small_k_path(int k, int nt = kNT) {
  return 2 * (((k + 3) / 4) * ((k + 3) / 4 + 1) / 2) <= nt;
}
constexpr int kSmemMaxK = 128; // Gram in shared memory up to this k
constexpr int kNB = 32;        // panel width of the blocked Cholesky (global path)

// Row scheduling: the rows of a half-sweep cost ~ d_i k^2 and are Zipf-
// skewed (c2: the heaviest row is 6x the mean per-CTA load of a static
// round-robin split; ncu showed the busiest SM active 2.7x the average).
// CTAs therefore take rows from a ticket counter in decreasing-degree order
// (longest first), so the heavy rows start at once and the light ones fill
// in behind them. Which CTA solves a row does not change its arithmetic.
// Double-buffered shared ticket: the barrier of the next take orders this
// take's reads before the buffer is written again.
// Heavy rows (d > S) of the shared-memory path are cut into segments of S
// entries; items[u] = (position in the row order, segment, segments, first
// item of the row) for u < info[1]; info[0] = number of split rows.
struct SplitPlan {
  const int4* items = nullptr;
  const int* info = nullptr;
  int* done = nullptr;        // per split row: segments finished (zero at rest)
  double* part = nullptr;     // per item: packed upper Gram + rhs
  int S = 0;
};

__device__ __forceinline__ int take_row(int* ticket, int* s_t, int& par) {
  if (threadIdx.x == 0) s_t[par] = atomicAdd(ticket, 1);
  __syncthreads();
  const int t = s_t[par];
  par ^= 1;
  return t;
}

// 5 CTAs per SM at 128 threads (<= 102 registers): the split-row logic
// otherwise raises the allocation to 124 registers and costs a CTA per SM
#ifndef MFG_BCD_SK_MINB
#define MFG_BCD_SK_MINB 5
#endif
// MINB: CTAs per SM the register allocation must allow. k <= kTinyK takes
// the small-k instantiation with 8 (64 registers); its gathers need more
// warps in flight, and the smaller Gram tiles leave the registers to spare
// (profiles/r1i_bcd_minb_ab.log: c2 k=20 -10%; at k=30/40 8 CTAs cost 10-23%).
constexpr int kTinyK = 24;
template <typename TS, int NT = kNT, bool SK = false, int MINB = (SK ? MFG_BCD_SK_MINB : 5)>
__global__ void __launch_bounds__(NT, NT == kNT ? MINB : 1)
k_bcd(mfg_layout lay, int k, const TS* __restrict__ vals, const TS* __restrict__ other, int ldo,
      double lam, TS* __restrict__ out, int ldout, double* __restrict__ gscratch, int use_global,
      int* __restrict__ bad, int min_d, const int* __restrict__ order, int* __restrict__ ticket,
      SplitPlan sp) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x;
  const int kp = k + 1;                         // padded leading dimension
  // global path: the Cholesky panel [kNB][k] reuses the staging area, and
  // the Gram stages as many entries per chunk as that area holds (fewer
  // read-modify-write passes over the global Gram)
  // SK: the small-k instantiation (entry groups); the others keep the plain
  // tile loop, whose register allocation the groups' accumulators would crowd
  const int kcs = SK ? kCS : kC;
  const int region0 = use_global ? (kNB * k > kC * kp + kC ? kNB * k : kC * kp + kC) : kcs * kp + kcs;
  const int region = use_global && 32 * (64 + 4 * (NT / 16)) > region0 ? 32 * (64 + 4 * (NT / 16))
                                                                      : region0;
  const int kc = use_global ? max(kC, min(64, region / (kp + 1))) : kcs;  // entries per chunk
  double* stage = sm;                           // [kc][kp]
  double* sa = stage + kc * kp;                 // [kc]
  double* bvec = sm + region;                   // [k]
  double* yvec = bvec + k;                      // [k]
  double* G = use_global ? gscratch + (size_t)blockIdx.x * k * k : yvec + k;  // [k][k]
  const int nt4 = (k + 3) / 4;                  // 4x4 tiles per dim
  __shared__ int s_t[2];
  __shared__ int s_last;
  int par = 0;
  const int nhr = sp.items ? sp.info[0] : 0;   // split (heavy) rows: a prefix of the order
  const int nhi = sp.items ? sp.info[1] : 0;   // their segment items, taken first
  const int pslot = k * (k + 1) / 2 + k;       // packed upper Gram + rhs per segment
  // Small k (at most NT/2 upper 4x4 tiles): EG groups of T threads each take
  // every EG-th entry of the row for one tile, accumulating in registers
  // across all chunks; the groups' partials are summed once per row in group
  // order (fixed). With k = 20 that is 8 threads per tile instead of 1.
  const int T = nt4 * (nt4 + 1) / 2;
  const int EG = SK ? NT / T : 1;
  int my_tp = 0, my_tq = 0, my_g = EG;      // my_g == EG: idle in the Gram
  if (EG > 1 && tid < EG * T) {
    my_g = tid / T;
    int rem = tid - my_g * T;
    while (rem >= nt4 - my_tp) { rem -= nt4 - my_tp; ++my_tp; }
    my_tq = my_tp + rem;
  }
  double* red = G + k * k;                  // [EG][T][16] group partials (EG > 1)
  for (;;) {
    const int u = take_row(ticket, s_t, par);
    int i, seg = 0, nseg = 1, ibase = 0, hidx = -1, s0, s1;
    if (u < nhi) {
      const int4 it = sp.items[u];   // (position in order, segment, segments, first item)
      hidx = it.x; seg = it.y; nseg = it.z; ibase = it.w;
      i = order[hidx];
    } else {
      const int t = u - nhi + nhr;
      if (t >= lay.nrows) break;
      i = order[t];
    }
    const int e0 = lay.ptr[i], e1 = lay.ptr[i + 1];
    if (e1 - e0 < min_d) break;   // rows in decreasing degree: the rest are the packed/dual kernel's
    s0 = e0 + seg * sp.S;
    s1 = nseg > 1 ? min(e1, s0 + sp.S) : e1;
    if (!use_global)                 // the global path writes every upper entry once
      for (int x = tid; x < k * k; x += NT) G[x] = 0.0;
    for (int x = tid; x < k; x += NT) bvec[x] = 0.0;
    __syncthreads();
    double eacc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) eacc[a][b] = 0.0;
    if (!use_global) {
      for (int c0 = s0; c0 < s1; c0 += kc) {
        const int cn = min(kc, s1 - c0);
        for (int x = tid; x < kc * k; x += NT) {
          const int c = x / k, d = x - c * k;
          double v = 0.0;
          if (c < cn) v = (double)other[(int64_t)lay.idx[c0 + c] * ldo + d];
          stage[c * kp + d] = v;
        }
        for (int c = tid; c < kc; c += NT) sa[c] = c < cn ? (double)vals[c0 + c] : 0.0;
        __syncthreads();
        if constexpr (SK) {
          if (my_g < EG) {
            for (int c = my_g; c < cn; c += EG) {
              double xp[4], xq[4];
#pragma unroll
              for (int a = 0; a < 4; ++a) {
                const int p = my_tp * 4 + a, q = my_tq * 4 + a;
                xp[a] = p < k ? stage[c * kp + p] : 0.0;
                xq[a] = q < k ? stage[c * kp + q] : 0.0;
              }
#pragma unroll
              for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) eacc[a][b] = fma(xp[a], xq[b], eacc[a][b]);
            }
          }
        } else
        // Gram tiles (upper triangle incl. diagonal)
        for (int t = tid; t < nt4 * nt4; t += NT) {
          const int tp = t / nt4, tq = t - tp * nt4;
          if (tq < tp) continue;
          double accv[4][4];
  #pragma unroll
          for (int a = 0; a < 4; ++a)
  #pragma unroll
            for (int b = 0; b < 4; ++b) accv[a][b] = 0.0;
          for (int c = 0; c < cn; ++c) {
            double xp[4], xq[4];
  #pragma unroll
            for (int a = 0; a < 4; ++a) {
              const int p = tp * 4 + a, q = tq * 4 + a;
              xp[a] = p < k ? stage[c * kp + p] : 0.0;
              xq[a] = q < k ? stage[c * kp + q] : 0.0;
            }
  #pragma unroll
            for (int a = 0; a < 4; ++a)
  #pragma unroll
              for (int b = 0; b < 4; ++b) accv[a][b] = fma(xp[a], xq[b], accv[a][b]);
          }
  #pragma unroll
          for (int a = 0; a < 4; ++a)
  #pragma unroll
            for (int b = 0; b < 4; ++b) {
              const int p = tp * 4 + a, q = tq * 4 + b;
              if (p < k && q < k && q >= p) G[p * k + q] += accv[a][b];
            }
        }
        for (int d = tid; d < k; d += NT) {
          double s = 0.0;
          for (int c = 0; c < cn; ++c) s = fma(sa[c], stage[c * kp + d], s);
          bvec[d] += s;
        }
        __syncthreads();
      }
      if constexpr (SK) {
        if (my_g < EG) {
          double* rp = red + ((size_t)my_g * T + (tid - my_g * T)) * 16;
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) rp[a * 4 + b] = eacc[a][b];
        }
        __syncthreads();
        if (my_g == 0) {
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              double v = 0.0;
              for (int gg = 0; gg < EG; ++gg) v += red[((size_t)gg * T + tid) * 16 + a * 4 + b];
              const int p = my_tp * 4 + a, q = my_tq * 4 + b;
              if (p < k && q < k && q >= p) G[p * k + q] = v;
            }
        }
        __syncthreads();
      }
      if (nseg > 1) {
        // Heavy row split into segments: publish this segment's partial Gram
        // and rhs; the CTA finishing the row's last segment sums all partials
        // in segment order (fixed, so the result does not depend on which
        // CTA ran which segment) and solves.
        double* slot = sp.part + (size_t)u * pslot;
        for (int x = tid; x < k * k; x += NT) {
          const int pp = x / k, qq = x - pp * k;
          if (qq >= pp) slot[pp * k - pp * (pp - 1) / 2 + (qq - pp)] = G[x];
        }
        for (int x = tid; x < k; x += NT) slot[k * (k + 1) / 2 + x] = bvec[x];
        __threadfence();
        __syncthreads();
        if (tid == 0) s_last = atomicAdd(&sp.done[hidx], 1) == nseg - 1;
        __syncthreads();
        if (!s_last) continue;
        __threadfence();
        for (int x = tid; x < k * k; x += NT) {
          const int pp = x / k, qq = x - pp * k;
          if (qq < pp) continue;
          const int off = pp * k - pp * (pp - 1) / 2 + (qq - pp);
          double acc = 0.0;
          for (int sg = 0; sg < nseg; ++sg) acc += __ldcg(sp.part + (size_t)(ibase + sg) * pslot + off);
          G[x] = acc;
        }
        for (int x = tid; x < k; x += NT) {
          double acc = 0.0;
          for (int sg = 0; sg < nseg; ++sg)
            acc += __ldcg(sp.part + (size_t)(ibase + sg) * pslot + k * (k + 1) / 2 + x);
          bvec[x] = acc;
        }
        if (tid == 0) sp.done[hidx] = 0;   // at rest for the next call
        __syncthreads();
      }
    } else {
      // Heavy rows, k beyond shared memory: GEMM-shaped Gram. Each 64 x 32
      // tile of G (4x4 register tiles, 128 threads) accumulates over all of
      // the row's entries, streamed through shared memory 32 at a time, and
      // is written once -- no read-modify-write of the global Gram per chunk.
      for (int e = e0; e < e1; ++e) {
        const double a = (double)vals[e];
        const TS* hrow = other + (int64_t)lay.idx[e] * ldo;
        for (int d = tid; d < k; d += NT) bvec[d] = fma(a, (double)hrow[d], bvec[d]);
      }
      constexpr int TX = NT / 16;          // thread columns; 16 thread rows
      constexpr int TQ = 4 * TX;           // tile: 64 x TQ
      double* sP = stage;                 // [32][64]
      double* sQ = stage + 32 * 64;       // [32][TQ]
      const int ty = tid / TX, tx = tid % TX;
      for (int pb = 0; pb < k; pb += 64) {
        for (int qb = pb; qb < k; qb += TQ) {
          double acc[4][4];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
          for (int c0 = e0; c0 < e1; c0 += 32) {
            const int cn = min(32, e1 - c0);
            __syncthreads();   // the previous chunk's reads are done
            for (int x = tid; x < 32 * (64 + TQ); x += NT) {
              const int c = x / (64 + TQ), j = x - c * (64 + TQ);
              double v = 0.0;
              const int dim = j < 64 ? pb + j : qb + (j - 64);
              if (c < cn && dim < k) v = (double)other[(int64_t)lay.idx[c0 + c] * ldo + dim];
              if (j < 64) sP[c * 64 + j] = v;
              else sQ[c * TQ + (j - 64)] = v;
            }
            __syncthreads();
            for (int c = 0; c < cn; ++c) {
              double xp[4], xq[4];
#pragma unroll
              for (int a = 0; a < 4; ++a) {
                xp[a] = sP[c * 64 + ty * 4 + a];
                xq[a] = sQ[c * TQ + tx * 4 + a];
              }
#pragma unroll
              for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = fma(xp[a], xq[b], acc[a][b]);
            }
          }
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const int pp = pb + ty * 4 + a, qq = qb + tx * 4 + b;
              if (pp < k && qq < k && qq >= pp) G[(int64_t)pp * k + qq] = acc[a][b];
            }
        }
      }
      __syncthreads();
    }
    // N = lam I + 2 G (upper), rhs = 2 b
    for (int x = tid; x < k * k; x += NT) {
      const int p = x / k, q = x - p * k;
      if (q >= p) G[x] = 2.0 * G[x] + (p == q ? lam : 0.0);
    }
    for (int x = tid; x < k; x += NT) bvec[x] *= 2.0;
    __syncthreads();
    // Cholesky N = U^T U, U upper, in place (right-looking)
    if (!use_global) {
      for (int j = 0; j < k; ++j) {
        if (tid == 0) {
          const double djj = G[j * k + j];
          if (!(djj > 0.0)) atomicOr(bad, 1);
          G[j * k + j] = sqrt(djj);
        }
        __syncthreads();
        const double ujj = G[j * k + j];
        for (int q = j + 1 + tid; q < k; q += NT) G[j * k + q] /= ujj;
        __syncthreads();
        const int rem = k - j - 1;
        for (int x = tid; x < rem * rem; x += NT) {
          const int p = j + 1 + x / rem, q = j + 1 + x % rem;
          if (q >= p) G[p * k + q] -= G[j * k + p] * G[j * k + q];
        }
        __syncthreads();
      }
    } else {
      // Blocked right-looking Cholesky on the global scratch: a panel of
      // kNB rows of U is factored in shared memory, then the trailing
      // matrix takes one rank-kNB update (4x4 register tiles), so each
      // trailing entry is read and written once per panel instead of once
      // per column.
      double* P = stage;  // [kNB][k]
      for (int jb = 0; jb < k; jb += kNB) {
        const int w = min(kNB, k - jb);
        const int wc = k - jb;
        for (int x = tid; x < w * wc; x += NT) {
          const int r = x / wc, c = jb + x - r * wc;
          P[r * k + c] = G[(int64_t)(jb + r) * k + c];
        }
        __syncthreads();
        for (int j = 0; j < w; ++j) {
          const int jj = jb + j;
          if (tid == 0) {
            const double djj = P[j * k + jj];
            if (!(djj > 0.0)) atomicOr(bad, 1);
            P[j * k + jj] = sqrt(djj);
          }
          __syncthreads();
          const double ujj = P[j * k + jj];
          for (int q = jj + 1 + tid; q < k; q += NT) P[j * k + q] /= ujj;
          __syncthreads();
          const int nr = w - j - 1;
          for (int x = tid; x < nr * wc; x += NT) {
            const int r = j + 1 + x / wc, q = jb + x % wc;
            if (q >= jb + r) P[r * k + q] -= P[j * k + jb + r] * P[j * k + q];
          }
          __syncthreads();
        }
        for (int x = tid; x < w * wc; x += NT) {
          const int r = x / wc, c = jb + x - r * wc;
          if (c >= jb + r) G[(int64_t)(jb + r) * k + c] = P[r * k + c];
        }
        // trailing update G[p][q] -= sum_r P[r][p] P[r][q], p, q >= jb + w
        const int t0 = jb + w, n = k - t0;
        const int nt = (n + 3) / 4;
        for (int t = tid; t < nt * nt; t += NT) {
          const int tp = t / nt, tq = t - tp * nt;
          if (tq < tp) continue;
          double acc[4][4];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
          for (int r = 0; r < w; ++r) {
            double xp[4], xq[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              const int p = t0 + tp * 4 + a, q = t0 + tq * 4 + a;
              xp[a] = p < k ? P[r * k + p] : 0.0;
              xq[a] = q < k ? P[r * k + q] : 0.0;
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int b = 0; b < 4; ++b) acc[a][b] = fma(xp[a], xq[b], acc[a][b]);
          }
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const int p = t0 + tp * 4 + a, q = t0 + tq * 4 + b;
              if (p < k && q < k && q >= p) G[(int64_t)p * k + q] -= acc[a][b];
            }
        }
        __syncthreads();
      }
    }
    // U^T y = rhs
    for (int j = 0; j < k; ++j) {
      if (tid == 0) yvec[j] = bvec[j] / G[j * k + j];
      __syncthreads();
      const double yj = yvec[j];
      for (int q = j + 1 + tid; q < k; q += NT) bvec[q] -= G[j * k + q] * yj;
      __syncthreads();
    }
    // U w = y  (w stored into bvec)
    for (int j = k - 1; j >= 0; --j) {
      if (tid == 0) bvec[j] = yvec[j] / G[j * k + j];
      __syncthreads();
      const double wj = bvec[j];
      for (int p = tid; p < j; p += NT) yvec[p] -= G[p * k + j] * wj;
      __syncthreads();
    }
    for (int d = tid; d < k; d += NT) out[(int64_t)i * ldout + d] = (TS)bvec[d];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Packed / dual BCD (k > kSmemMaxK): the normal matrix is stored packed
// (lower triangle, s(s+1)/2 doubles) in shared memory, s = min(d_i, k), so
// k up to ~210 stays on chip. Rows with fewer entries than k use the
// push-through identity
//   (lam I_k + 2 H^T H)^{-1} 2 H^T a = 2 H^T (lam I_d + 2 H H^T)^{-1} a,
// i.e. a d x d solve instead of k x k (H = the row's gathered factor rows).
__device__ __forceinline__ int tri(int p, int q) { return p * (p + 1) / 2 + q; }

template <typename TS>
__global__ void __launch_bounds__(kNT)
k_bcd_packed(mfg_layout lay, int k, const TS* __restrict__ vals, const TS* __restrict__ other,
             int ldo, double lam, TS* __restrict__ out, int ldout, int smax, int* __restrict__ bad,
             const int* __restrict__ order, int* __restrict__ ticket) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x;
  const int kp = k + 1;
  double* L = sm;                                     // [smax*(smax+1)/2]
  double* stA = L + (size_t)smax * (smax + 1) / 2;    // [kC][kp]
  double* stB = stA + kC * kp;                        // [kC][kp]
  double* vec = stB + kC * kp;                        // [max(k, smax)] rhs / solution
  double* aux = vec + (k > smax ? k : smax);          // [max(k, smax)]
  __shared__ int s_t[2];
  int par = 0;
  for (;;) {
    const int t = take_row(ticket, s_t, par);
    if (t >= lay.nrows) break;
    const int i = order[t];
    const int e0 = lay.ptr[i], e1 = lay.ptr[i + 1];
    const int d = e1 - e0;
    if (d == 0) {
      for (int x = tid; x < k; x += kNT) out[(int64_t)i * ldout + x] = TS(0);
      continue;
    }
    const bool dual = d < k;
    const int sdim = dual ? d : k;
    if (sdim > smax) continue;   // system larger than the shared-memory budget: global kernel
    const int npk = sdim * (sdim + 1) / 2;
    for (int x = tid; x < npk; x += kNT) L[x] = 0.0;
    for (int x = tid; x < sdim; x += kNT) vec[x] = 0.0;
    __syncthreads();
    auto stage = [&](double* st, int c0, int cn) {
      for (int x = tid; x < kC * k; x += kNT) {
        const int c = x / k, dd = x - c * k;
        st[c * kp + dd] = c < cn ? (double)other[(int64_t)lay.idx[e0 + c0 + c] * ldo + dd] : 0.0;
      }
    };
    if (!dual) {
      // primal: L += sum_c h_c h_c^T (lower), vec += sum_c a_c h_c
      for (int c0 = 0; c0 < d; c0 += kC) {
        const int cn = min(kC, d - c0);
        stage(stA, c0, cn);
        if (tid < kC) aux[tid] = tid < cn ? (double)vals[e0 + c0 + tid] : 0.0;
        __syncthreads();
        for (int x = tid; x < npk; x += kNT) {
          const int p = (int)((sqrtf(8.f * x + 1.f) - 1.f) * 0.5f);
          int pp = p;
          if (tri(pp + 1, 0) <= x) ++pp;
          if (tri(pp, 0) > x) --pp;
          const int q = x - tri(pp, 0);
          double acc = 0.0;
          for (int c = 0; c < cn; ++c) acc = fma(stA[c * kp + pp], stA[c * kp + q], acc);
          L[x] += acc;
        }
        for (int dd = tid; dd < k; dd += kNT) {
          double acc = 0.0;
          for (int c = 0; c < cn; ++c) acc = fma(aux[c], stA[c * kp + dd], acc);
          vec[dd] += acc;
        }
        __syncthreads();
      }
    } else {
      // dual: L[p][q] = h_p . h_q over the row's d entries (block pairs)
      for (int q0 = 0; q0 < d; q0 += kC) {
        const int qn = min(kC, d - q0);
        stage(stB, q0, qn);
        for (int p0 = q0; p0 < d; p0 += kC) {
          const int pn = min(kC, d - p0);
          stage(stA, p0, pn);
          __syncthreads();
          for (int x = tid; x < kC * kC; x += kNT) {
            const int pi = x / kC, qi = x - pi * kC;
            const int p = p0 + pi, q = q0 + qi;
            if (pi < pn && qi < qn && q <= p) {
              double acc = 0.0;
              for (int dd = 0; dd < k; ++dd) acc = fma(stA[pi * kp + dd], stB[qi * kp + dd], acc);
              L[tri(p, q)] = acc;
            }
          }
          __syncthreads();
        }
      }
      for (int x = tid; x < d; x += kNT) vec[x] = (double)vals[e0 + x];
      __syncthreads();
    }
    // N = lam I + 2 G (primal), or lam I_d + 2 H H^T (dual); rhs = 2b or a
    for (int x = tid; x < npk; x += kNT) {
      int p = (int)((sqrtf(8.f * x + 1.f) - 1.f) * 0.5f);
      if (tri(p + 1, 0) <= x) ++p;
      if (tri(p, 0) > x) --p;
      const int q = x - tri(p, 0);
      L[x] = 2.0 * L[x] + (p == q ? lam : 0.0);
    }
    if (!dual)
      for (int x = tid; x < sdim; x += kNT) vec[x] *= 2.0;
    __syncthreads();
    // packed right-looking Cholesky N = L L^T
    for (int j = 0; j < sdim; ++j) {
      if (tid == 0) {
        const double djj = L[tri(j, j)];
        if (!(djj > 0.0)) atomicOr(bad, 1);
        L[tri(j, j)] = sqrt(djj);
      }
      __syncthreads();
      const double ljj = L[tri(j, j)];
      for (int p = j + 1 + tid; p < sdim; p += kNT) L[tri(p, j)] /= ljj;
      __syncthreads();
      const int rem = sdim - j - 1;
      const int ntr = rem * (rem + 1) / 2;
      for (int x = tid; x < ntr; x += kNT) {
        int a = (int)((sqrtf(8.f * x + 1.f) - 1.f) * 0.5f);
        if (tri(a + 1, 0) <= x) ++a;
        if (tri(a, 0) > x) --a;
        const int b = x - tri(a, 0);
        const int p = j + 1 + a, q = j + 1 + b;
        L[tri(p, q)] -= L[tri(p, j)] * L[tri(q, j)];
      }
      __syncthreads();
    }
    // L y = rhs
    for (int j = 0; j < sdim; ++j) {
      if (tid == 0) vec[j] /= L[tri(j, j)];
      __syncthreads();
      const double yj = vec[j];
      for (int p = j + 1 + tid; p < sdim; p += kNT) vec[p] -= L[tri(p, j)] * yj;
      __syncthreads();
    }
    // L^T x = y
    for (int j = sdim - 1; j >= 0; --j) {
      if (tid == 0) vec[j] /= L[tri(j, j)];
      __syncthreads();
      const double xj = vec[j];
      for (int p = tid; p < j; p += kNT) vec[p] -= L[tri(j, p)] * xj;
      __syncthreads();
    }
    if (!dual) {
      for (int x = tid; x < k; x += kNT) out[(int64_t)i * ldout + x] = (TS)vec[x];
    } else {
      // w = 2 H^T y
      for (int x = tid; x < k; x += kNT) aux[x] = 0.0;
      __syncthreads();
      for (int c0 = 0; c0 < d; c0 += kC) {
        const int cn = min(kC, d - c0);
        stage(stA, c0, cn);
        __syncthreads();
        for (int dd = tid; dd < k; dd += kNT) {
          double acc = 0.0;
          for (int c = 0; c < cn; ++c) acc = fma(vec[c0 + c], stA[c * kp + dd], acc);
          aux[dd] += acc;
        }
        __syncthreads();
      }
      for (int x = tid; x < k; x += kNT) out[(int64_t)i * ldout + x] = (TS)(2.0 * aux[x]);
    }
    __syncthreads();
  }
}

size_t smem_packed(int k, int smax) {
  const int kp = k + 1;
  const int v = k > smax ? k : smax;
  return ((size_t)smax * (smax + 1) / 2 + 2 * (size_t)kC * kp + 2 * (size_t)v) * sizeof(double);
}

constexpr int kNTG = 512;      // threads of the global (heavy-row) path: 16 warps per SM

size_t smem_bytes(int k, bool global) {
  const int kp = k + 1;
  const bool small = !global && small_k_path(k);
  size_t region = small ? (size_t)kCS * kp + kCS : (size_t)kC * kp + kC;
  if (global) {
    if ((size_t)kNB * k > region) region = (size_t)kNB * k;
    const size_t gt = 32 * (64 + 4 * (kNTG / 16));
    if (gt > region) region = gt;
  }
  size_t n = region + 2 * (size_t)k;
  if (!global) n += (size_t)k * k;
  if (small) n += 16 * (size_t)kNT;   // the entry groups' partials
  return n * sizeof(double);
}

int grid_for_rows(int nrows) {
  int g = nrows;
  if (g > kNumSMs * 8) g = kNumSMs * 8;
  if (g < 1) g = 1;
  return g;
}

__global__ void k_row_degrees(const int32_t* __restrict__ ptr, int n, unsigned* __restrict__ key,
                              int* __restrict__ row) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    key[i] = (unsigned)(ptr[i + 1] - ptr[i]);
    row[i] = i;
  }
}

size_t sort_temp_bytes(int n) {
  size_t b = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, b, (unsigned*)nullptr, (unsigned*)nullptr,
                                            (int*)nullptr, (int*)nullptr, n);
  return b;
}

// Scheduling workspace: row order (decreasing degree) and two tickets.
struct RowSched {
  int* order = nullptr;
  int* ticket = nullptr;   // [2], zeroed per call
  const unsigned* deg = nullptr;   // degrees in that order
};

template <typename C>
void take_sched(C& c, int n, RowSched* rs, unsigned** kin, unsigned** kout, int* *rin, void** tmp,
                size_t* tmpb) {
  *kin = c.template take<unsigned>(n);
  *kout = c.template take<unsigned>(n);
  *rin = c.template take<int>(n);
  rs->order = c.template take<int>(n);
  rs->ticket = c.template take<int>(2);
  *tmpb = sort_temp_bytes(n);
  *tmp = c.template take<char>(*tmpb);
}

int build_sched(const mfg_layout* lay, Carver& c, RowSched* rs, cudaStream_t stream) {
  const int n = lay->nrows;
  unsigned *kin, *kout;
  int* rin;
  void* tmp;
  size_t tmpb;
  take_sched(c, n, rs, &kin, &kout, &rin, &tmp, &tmpb);
  MFG_REQUIRE(c.ok, "bcd workspace too small");
  k_row_degrees<<<(n + 255) / 256, 256, 0, stream>>>(lay->ptr, n, kin, rin);
  MFG_LAUNCH_CHECK();
  MFG_CUDA_CHECK(cub::DeviceRadixSort::SortPairsDescending(tmp, tmpb, kin, kout, rin, rs->order, n,
                                                           0, 32, stream));
  MFG_CUDA_CHECK(cudaMemsetAsync(rs->ticket, 0, 2 * sizeof(int), stream));
  rs->deg = kout;
  return MFG_OK;
}

// Items of the split heavy rows from the sorted degrees (heavy rows are a
// prefix of at most nnz/S <= grid rows; one 1024-thread block covers 2048).
__global__ void __launch_bounds__(1024) k_split_items(const unsigned* __restrict__ deg, int n, int S,
                                                      int4* __restrict__ items, int* __restrict__ info) {
  using Scan = cub::BlockScan<int, 1024>;
  __shared__ typename Scan::TempStorage ts;
  __shared__ int nh;
  if (threadIdx.x == 0) nh = 0;
  const int t0 = 2 * threadIdx.x;
  int c[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int t = t0 + j;
    const long long d = t < n ? (long long)deg[t] : 0;
    c[j] = d > S ? (int)((d + S - 1) / S) : 0;
  }
  int off, agg;
  Scan(ts).ExclusiveSum(c[0] + c[1], off, agg);
  __syncthreads();
  atomicAdd(&nh, (c[0] > 0) + (c[1] > 0));
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int base = off + (j ? c[0] : 0);
    for (int sg = 0; sg < c[j]; ++sg) items[base + sg] = make_int4(t0 + j, sg, c[j], base);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    info[0] = nh;
    info[1] = agg;
  }
}

int split_len(int64_t nnz, int grid) {
  const int64_t s = (nnz + grid - 1) / grid;
  return (int)(s < 256 ? 256 : s);
}

template <typename C>
void take_split(C& c, int grid, int k, SplitPlan* sp, int4** items, int** info) {
  *items = c.template take<int4>((size_t)2 * grid);
  *info = c.template take<int>(2);
  sp->done = c.template take<int>(grid);
  sp->part = c.template take<double>((size_t)2 * grid * (k * (k + 1) / 2 + k));
}

int build_split(const mfg_layout* lay, Carver& c, const RowSched& rs, int grid, int k, SplitPlan* sp,
                cudaStream_t stream) {
  int4* items;
  int* info;
  take_split(c, grid, k, sp, &items, &info);
  MFG_REQUIRE(c.ok, "bcd workspace too small");
  sp->S = split_len(lay->nnz, grid);
  MFG_CUDA_CHECK(cudaMemsetAsync(sp->done, 0, sizeof(int) * grid, stream));
  k_split_items<<<1, 1024, 0, stream>>>(rs.deg, lay->nrows, sp->S, items, info);
  MFG_LAUNCH_CHECK();
  sp->items = items;
  sp->info = info;
  return MFG_OK;
}


// ---------------------------------------------------------------------------
// Warp-per-row BCD with the Gram on the fp64 tensor cores (round 2, k <= 64).
//
// One warp owns one row (or one segment of a heavy row) at a time and takes
// it from a warp-granular ticket (longest first, as above), so a short row
// costs no CTA barriers. The row's Gram G = X^T X (X = the d gathered factor
// rows, d x k) is accumulated by mma.sync.m8n8k4.f64 (DMMA) over 8 x 8 tiles
// of G, upper tile pairs (P <= Q) only: for 4 entries e0..e0+3 the A
// fragment of tile P (X^T: 8 dims x 4 entries) and the B fragment of tile Q
// (X: 4 entries x 8 dims) are the same per-lane value x[T] =
// X[e0 + lane%4][8T + lane/4], so one gathered value per lane and tile feeds
// every pair; the accumulators stay in registers for the whole row (k = 40:
// 15 pairs, 30 doubles per lane). The right-hand side sum_e a_e x_e is a
// per-lane fp64 FMA reduced over the 4 lanes of each dim in fixed order.
// The normal matrix lam I + 2 G then goes to the warp's shared-memory slab
// and is factored by an in-warp right-looking Cholesky; the two triangular
// solves keep the vector in registers (lane l owns dims l, l + 32).
// Heavy rows are cut into segments of S entries (S ~ nnz / 8192, so no
// segment outlasts the sweep) whose packed partial Grams are summed in
// segment order by the warp that finishes the row's last segment -- the
// result does not depend on which warp ran which segment.
// fp64 arithmetic throughout; per-row results are bitwise reproducible.

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int kDmMaxK = 64;            // k handled by the DMMA kernel (8 tiles)
// warps per CTA: 4 up to k = 40; 3 for k = 41..64, where a warp's slab is up
// to 37.9 KB (two CTAs = 6 warps fill an SM's shared memory) and the 2 NP
// accumulators take up to 144 registers
__host__ __device__ constexpr int dm_warps(int nt) { return nt <= 5 ? 4 : 3; }
#ifndef MFG_BCD_DM_MINB
#define MFG_BCD_DM_MINB 4              // CTAs per SM (128 registers)
#endif
#ifndef MFG_BCD_DM_MINB5
#define MFG_BCD_DM_MINB5 4             // ... for k = 33..40 (3: 168 registers, measured slower)
#endif

// the warp's slab: N padded to K8 = 8 ceil(k/8) dims with row stride
// ld = K8 (+8 when K8 % 16 == 0, so the 4 rows of a DMMA fragment load fall
// in alternating bank halves), then the rhs
__host__ __device__ inline int dm_ld(int k) {
  const int k8 = 8 * ((k + 7) / 8);
  return k8 % 16 == 8 ? k8 : k8 + 8;
}
size_t dm_smem_per_warp(int k) {
  const int k8 = 8 * ((k + 7) / 8);
  return ((size_t)k8 * dm_ld(k) + 2 * k8) * sizeof(double);
}

// CTAs per SM of an instantiation (NT = 5: 3 CTAs with 168 registers was
// slower than 4 with 128 at c4, CSR 11.7 -> 12.4 ms, CSC 19.4 -> 22.0 ms)
template <int NT>
__host__ __device__ constexpr int dm_minb() {
  return NT >= 6 ? 2 : (NT >= 5 ? MFG_BCD_DM_MINB5 : MFG_BCD_DM_MINB);
}

template <typename TS, int NT>
__global__ void __launch_bounds__(32 * dm_warps(NT), dm_minb<NT>())
k_bcd_dm(mfg_layout lay, int k, const TS* __restrict__ vals, const TS* __restrict__ other, int ldo,
         double lam, TS* __restrict__ out, int ldout, int* __restrict__ bad,
         const int* __restrict__ order, int* __restrict__ ticket, SplitPlan sp) {
  constexpr int NP = NT * (NT + 1) / 2;
  // 4-entry steps per chunk: the prefetched fragments f[SB][NT] compete with
  // the 2 NP accumulators for registers (NT = 5: SB = 4 spilled 120 bytes)
  constexpr int SB = NT <= 3 ? (sizeof(TS) == 4 ? 8 : 4) : (NT == 4 ? 4 : 2);
  constexpr int CH = 4 * SB;
  extern __shared__ __align__(16) double smw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  constexpr int K8 = 8 * NT;
  const int kl = dm_ld(k);
  double* G = smw + (size_t)wib * ((size_t)K8 * kl + 2 * K8);
  double* bv = G + (size_t)K8 * kl;
  double* rv = bv + K8;                 // 1 / U_jj
  const int g = lane >> 2, tq = lane & 3;
  const int nhr = sp.items ? sp.info[0] : 0;
  const int nhi = sp.items ? sp.info[1] : 0;
  const int pslot = k * (k + 1) / 2 + k;
  for (;;) {
    int u = 0;
    if (lane == 0) u = atomicAdd(ticket, 1);
    u = __shfl_sync(0xffffffffu, u, 0);
    int i, seg = 0, nseg = 1, ibase = 0, hidx = -1;
    if (u < nhi) {
      const int4 it = sp.items[u];
      hidx = it.x; seg = it.y; nseg = it.z; ibase = it.w;
      i = order[hidx];
    } else {
      const int t = u - nhi + nhr;
      if (t >= lay.nrows) break;
      i = order[t];
    }
    const int e0 = lay.ptr[i], e1 = lay.ptr[i + 1];
    const int s0 = e0 + seg * sp.S;
    const int s1 = nseg > 1 ? min(e1, s0 + sp.S) : e1;
    double acc[NP][2];
#pragma unroll
    for (int p = 0; p < NP; ++p) acc[p][0] = acc[p][1] = 0.0;
    double bp[NT];
#pragma unroll
    for (int T = 0; T < NT; ++T) bp[T] = 0.0;
    for (int c0 = s0; c0 < s1; c0 += CH) {
      const int cn = min(CH, s1 - c0);
      int colv = 0;
      double av = 0.0;
      if (lane < cn) {
        colv = lay.idx[c0 + lane];
        av = (double)vals[c0 + lane];
      }
      TS f[SB][NT];
#pragma unroll
      for (int s = 0; s < SB; ++s) {
        const int src = 4 * s + tq;
        const int col = __shfl_sync(0xffffffffu, colv, src & 31);
        const TS* rowp = other + (int64_t)col * ldo;
#pragma unroll
        for (int T = 0; T < NT; ++T) {
          const int d = 8 * T + g;
          f[s][T] = (src < cn && d < k) ? rowp[d] : TS(0);
        }
      }
#pragma unroll
      for (int s = 0; s < SB; ++s) {
        if (4 * s >= cn) break;   // warp-uniform
        const double a = __shfl_sync(0xffffffffu, av, (4 * s + tq) & 31);
        double x[NT];
#pragma unroll
        for (int T = 0; T < NT; ++T) {
          x[T] = (double)f[s][T];
          bp[T] = fma(a, x[T], bp[T]);
        }
        int pi = 0;
#pragma unroll
        for (int P = 0; P < NT; ++P)
#pragma unroll
          for (int Q = P; Q < NT; ++Q) {
            dmma884(acc[pi][0], acc[pi][1], x[P], x[Q]);
            ++pi;
          }
      }
    }
    // rhs: sum the 4 lanes of each dim (fixed order)
#pragma unroll
    for (int T = 0; T < NT; ++T) {
      bp[T] += __shfl_xor_sync(0xffffffffu, bp[T], 1);
      bp[T] += __shfl_xor_sync(0xffffffffu, bp[T], 2);
    }
    // The normal matrix N = lam I + 2 G on the warp's slab, padded to K8 =
    // 8 NT dims with an identity block (padded rhs and solution are zero).
    // Whole rows: N (upper tiles; diagonal tiles whole) straight from the
    // fragments. Segments of heavy rows publish the raw G instead.
    {
      const bool whole = nseg == 1;
      int pi = 0;
#pragma unroll
      for (int P = 0; P < NT; ++P)
#pragma unroll
        for (int Q = P; Q < NT; ++Q) {
          const int p = 8 * P + g;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int q = 8 * Q + 2 * tq + h;
            double v = acc[pi][h];
            if (whole) v = 2.0 * v + (p == q ? (p < k ? lam : 1.0) : 0.0);
            G[p * kl + q] = v;
          }
          ++pi;
        }
    }
    if (tq == 0) {
#pragma unroll
      for (int T = 0; T < NT; ++T) bv[8 * T + g] = bp[T];
    }
    __syncwarp();
    if (nseg > 1) {
      // publish this segment's packed upper Gram + rhs; the warp that
      // deposits the row's last segment sums all of them in segment order
      double* slot = sp.part + (size_t)u * pslot;
      for (int pp = 0; pp < k; ++pp)
        for (int qq = pp + lane; qq < k; qq += 32)
          slot[pp * k - pp * (pp - 1) / 2 + (qq - pp)] = G[pp * kl + qq];
      for (int x = lane; x < k; x += 32) slot[k * (k + 1) / 2 + x] = bv[x];
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      __syncwarp();
      int old = 0;
      if (lane == 0)
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                     : "=r"(old) : "l"(sp.done + hidx) : "memory");
      old = __shfl_sync(0xffffffffu, old, 0);
      if (old != nseg - 1) continue;
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      for (int pp = 0; pp < k; ++pp)
        for (int qq = pp + lane; qq < k; qq += 32) {
          const int off = pp * k - pp * (pp - 1) / 2 + (qq - pp);
          double a = 0.0;
          for (int sg = 0; sg < nseg; ++sg) a += __ldcg(sp.part + (size_t)(ibase + sg) * pslot + off);
          G[pp * kl + qq] = 2.0 * a + (pp == qq ? lam : 0.0);
        }
      for (int x = lane; x < k; x += 32) {
        double a = 0.0;
        for (int sg = 0; sg < nseg; ++sg)
          a += __ldcg(sp.part + (size_t)(ibase + sg) * pslot + k * (k + 1) / 2 + x);
        bv[x] = a;
      }
      for (int pp = k + lane; pp < K8; pp += 32) G[pp * kl + pp] = 1.0;   // identity padding
      if (lane == 0) sp.done[hidx] = 0;   // at rest for the next call
      __syncwarp();
    }
    // Blocked right-looking Cholesky N = U^T U in place (U upper), panels of
    // 8 rows: the panel is factored by lanes over columns (at most 7 row
    // updates per column), then the trailing matrix takes the panel's
    // rank-8 update on the tensor cores (two DMMA per 8 x 8 tile pair,
    // A = -U[panel rows][tile P], B = U[panel rows][tile Q], C = N tile).
#pragma unroll 1
    for (int b = 0; b < NT; ++b) {
      const int jb = 8 * b;
#pragma unroll 1
      for (int jj = 0; jj < 8; ++jj) {
        const int j = jb + jj;
        const double djj = G[j * kl + j];
        if (!(djj > 0.0) && lane == 0) atomicOr(bad, 1);
        const double ujj = sqrt(djj);
        const double rinv = 1.0 / ujj;
        __syncwarp();
        if (lane == 0) {
          G[j * kl + j] = ujj;
          rv[j] = rinv;
        }
        for (int q = j + 1 + lane; q < K8; q += 32) G[j * kl + q] *= rinv;
        __syncwarp();
        for (int q = j + 1 + lane; q < K8; q += 32) {
          const double gjq = G[j * kl + q];
#pragma unroll
          for (int pp = 1; pp < 8; ++pp) {
            const int p = j + pp;
            if (jj + pp < 8 && p <= q) G[p * kl + q] -= G[j * kl + p] * gjq;
          }
        }
        __syncwarp();
      }
      if (b + 1 < NT) {
        double xa[NT][2];
#pragma unroll
        for (int P = 0; P < NT; ++P)
          if (P > b) {
#pragma unroll
            for (int s = 0; s < 2; ++s) xa[P][s] = G[(jb + 4 * s + tq) * kl + 8 * P + g];
          }
#pragma unroll
        for (int P = 0; P < NT; ++P)
#pragma unroll
          for (int Q = 0; Q < NT; ++Q)
            if (P > b && Q >= P) {
              double* c = G + (8 * P + g) * kl + 8 * Q + 2 * tq;
              double c0 = c[0], c1 = c[1];
              dmma884(c0, c1, -xa[P][0], xa[Q][0]);
              dmma884(c0, c1, -xa[P][1], xa[Q][1]);
              c[0] = c0;
              c[1] = c1;
            }
        __syncwarp();
      }
    }
    // U^T y = b (forward; lane l owns dims l, l + 32), then U w = y by rows
    // (w_j = (y_j - U[j][j+1:] . w[j+1:]) / U_jj, a warp dot per row)
    double y0 = lane < K8 ? 2.0 * bv[lane] : 0.0;
    double y1 = lane + 32 < K8 ? 2.0 * bv[lane + 32] : 0.0;
#pragma unroll 1
    for (int j = 0; j < K8; ++j) {
      const double own = j < 32 ? y0 : y1;
      const double yj = __shfl_sync(0xffffffffu, own, j & 31) * rv[j];
      if (lane == (j & 31)) { if (j < 32) y0 = yj; else y1 = yj; }
      if (lane > j && lane < K8) y0 -= G[j * kl + lane] * yj;
      if (lane + 32 > j && lane + 32 < K8) y1 -= G[j * kl + lane + 32] * yj;
    }
    double w0 = 0.0, w1 = 0.0;
#pragma unroll 1
    for (int j = K8 - 1; j >= 0; --j) {
      double s = 0.0;
      if (lane > j && lane < K8) s = G[j * kl + lane] * w0;
      if (lane + 32 > j && lane + 32 < K8) s = fma(G[j * kl + lane + 32], w1, s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      const double own = j < 32 ? y0 : y1;
      const double wj = (__shfl_sync(0xffffffffu, own, j & 31) - s) * rv[j];
      if (lane == (j & 31)) { if (j < 32) w0 = wj; else w1 = wj; }
    }
    if (lane < k) out[(int64_t)i * ldout + lane] = (TS)w0;
    if (lane + 32 < k) out[(int64_t)i * ldout + lane + 32] = (TS)w1;
    __syncwarp();   // the slab is rewritten by the next row
  }
}

// Warp-granular split plan: every row with more than S entries becomes
// ceil(d / S) items (in the longest-first order, so split rows are a prefix
// of it); items[] = (position in the order, segment, segments, first item).
__global__ void k_seg_counts(const unsigned* __restrict__ deg, int n, int S, int* __restrict__ cnt) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) {
    const long long d = deg[t];
    cnt[t] = d > S ? (int)((d + S - 1) / S) : 0;
  }
}

__global__ void k_seg_fill(const int* __restrict__ cnt, const int* __restrict__ off, int n,
                           int4* __restrict__ items, int* __restrict__ info) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n || cnt[t] == 0) return;
  const int base = off[t], c = cnt[t];
  for (int sg = 0; sg < c; ++sg) items[base + sg] = make_int4(t, sg, c, base);
  if (t + 1 == n || cnt[t + 1] == 0) {   // last split row: the prefix ends here
    info[0] = t + 1;
    info[1] = base + c;
  }
}

int dm_split_len(int64_t nnz) {
  const int64_t s = (nnz + 8191) / 8192;
  return (int)(s < 512 ? 512 : s);
}

size_t dm_scan_temp_bytes(int n) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const int*)nullptr, (int*)nullptr, n);
  return b;
}

template <typename C>
void take_dm_split(C& c, int64_t nnz, int n, int k, SplitPlan* sp, int** cnt, int** off,
                   int4** items, int** info, void** tmp, size_t* tmpb) {
  const int S = dm_split_len(nnz);
  const size_t nitems = (size_t)(2 * (nnz / S) + 2);
  *cnt = c.template take<int>(n > 0 ? n : 1);
  *off = c.template take<int>(n > 0 ? n : 1);
  *items = c.template take<int4>(nitems);
  *info = c.template take<int>(2);
  sp->done = c.template take<int>(nitems);
  sp->part = c.template take<double>(nitems * (size_t)(k * (k + 1) / 2 + k));
  *tmpb = dm_scan_temp_bytes(n > 0 ? n : 1);
  *tmp = c.template take<char>(*tmpb);
}

int build_dm_split(const mfg_layout* lay, Carver& c, const RowSched& rs, int k, SplitPlan* sp,
                   cudaStream_t stream) {
  const int n = lay->nrows;
  int *cnt, *off, *info;
  int4* items;
  void* tmp;
  size_t tmpb;
  take_dm_split(c, lay->nnz, n, k, sp, &cnt, &off, &items, &info, &tmp, &tmpb);
  MFG_REQUIRE(c.ok, "bcd workspace too small");
  sp->S = dm_split_len(lay->nnz);
  const size_t nitems = (size_t)(2 * (lay->nnz / sp->S) + 2);
  MFG_CUDA_CHECK(cudaMemsetAsync(sp->done, 0, sizeof(int) * nitems, stream));
  MFG_CUDA_CHECK(cudaMemsetAsync(info, 0, 2 * sizeof(int), stream));
  k_seg_counts<<<(n + 255) / 256, 256, 0, stream>>>(rs.deg, n, sp->S, cnt);
  MFG_LAUNCH_CHECK();
  MFG_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp, tmpb, cnt, off, n, stream));
  k_seg_fill<<<(n + 255) / 256, 256, 0, stream>>>(cnt, off, n, items, info);
  MFG_LAUNCH_CHECK();
  sp->items = items;
  sp->info = info;
  return MFG_OK;
}

bool dm_path(int k) {
  static const bool off = [] {
    const char* e = getenv("MFG_BCD_NO_DMMA");
    return e && e[0] && e[0] != '0';
  }();
  return !off && k >= 1 && k <= kDmMaxK;
}

template <typename TS>
int launch_dm(const mfg_layout* lay, int k, const TS* vals, const TS* other, int ldo, double lam,
              TS* out, int ldout, int* bad, const RowSched& rs, const SplitPlan& sp,
              cudaStream_t stream) {
  const int nt = (k + 7) / 8;
  const int wpc = dm_warps(nt);
  const size_t smem = dm_smem_per_warp(k) * wpc;
  int grid = (lay->nrows + wpc - 1) / wpc;
  const int full = kNumSMs * (nt >= 6 ? 2 : (nt >= 5 ? MFG_BCD_DM_MINB5 : MFG_BCD_DM_MINB));
  if (grid > full) grid = full;
  if (grid < 1) grid = 1;
  auto go = [&](auto kern) -> int {
    if (smem > 48 * 1024)
      MFG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, 32 * wpc, smem, stream>>>(*lay, k, vals, other, ldo, lam, out, ldout, bad,
                                                rs.order, rs.ticket, sp);
    MFG_LAUNCH_CHECK();
    return MFG_OK;
  };
  switch (nt) {
    case 1: return go(k_bcd_dm<TS, 1>);
    case 2: return go(k_bcd_dm<TS, 2>);
    case 3: return go(k_bcd_dm<TS, 3>);
    case 4: return go(k_bcd_dm<TS, 4>);
    case 5: return go(k_bcd_dm<TS, 5>);
    case 6: return go(k_bcd_dm<TS, 6>);
    case 7: return go(k_bcd_dm<TS, 7>);
    case 8: return go(k_bcd_dm<TS, 8>);
    default: break;
  }
  set_error("bcd: DMMA path supports k <= 64");
  return MFG_ERR_ARG;
}

template <typename TS>
int do_bcd(const mfg_layout* lay, int k, const void* vals, const void* other, int ldo, double lam,
           void* out, int ldout, void* ws, size_t wsb, cudaStream_t stream) {
  if (lay->nrows == 0 || k == 0) return MFG_OK;
  if (dm_path(k)) {
    Carver c(ws, wsb);
    int* bad = c.take<int>(1);
    MFG_REQUIRE(c.ok, "bcd workspace too small");
    RowSched rs;
    if (int st = build_sched(lay, c, &rs, stream)) return st;
    SplitPlan sp;
    if (int st = build_dm_split(lay, c, rs, k, &sp, stream)) return st;
    MFG_CUDA_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), stream));
    return launch_dm<TS>(lay, k, (const TS*)vals, (const TS*)other, ldo, lam, (TS*)out, ldout, bad,
                         rs, sp, stream);
  }
  if (k > kSmemMaxK && smem_packed(k, k) <= 220 * 1024) {
    Carver c(ws, wsb);
    int* bad = c.take<int>(1);
    MFG_REQUIRE(c.ok, "bcd workspace too small");
    RowSched rs;
    if (int st = build_sched(lay, c, &rs, stream)) return st;
    const size_t smem = smem_packed(k, k);
    MFG_CUDA_CHECK(cudaFuncSetAttribute(k_bcd_packed<TS>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    MFG_CUDA_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), stream));
    k_bcd_packed<TS><<<grid_for_rows(lay->nrows), kNT, smem, stream>>>(
        *lay, k, (const TS*)vals, (const TS*)other, ldo, lam, (TS*)out, ldout, k, bad, rs.order,
        rs.ticket);
    MFG_LAUNCH_CHECK();
    return MFG_OK;
  }
  const bool global = k > kSmemMaxK;
  const int grid = global ? kNumSMs : grid_for_rows(lay->nrows);
  Carver c(ws, wsb);
  int* bad = c.take<int>(1);
  // k beyond the on-chip primal: rows with few entries still fit on chip as
  // d x d dual systems (d <= smax); only the heavier rows take the global
  // k x k path (its Gram and Cholesky live in global scratch)
  int smax = 0;
  if (global)
    while (smax + 1 <= k && smem_packed(k, smax + 1) <= 220 * 1024) ++smax;
  double* gs = global ? c.take<double>((size_t)grid * k * k) : nullptr;
  MFG_REQUIRE(c.ok, "bcd workspace too small");
  RowSched rs;
  if (int st = build_sched(lay, c, &rs, stream)) return st;
  SplitPlan sp;
  if (!global)
    if (int st = build_split(lay, c, rs, grid, k, &sp, stream)) return st;
  const size_t smem = smem_bytes(k, global);
  if (smem > 48 * 1024) {
    MFG_CUDA_CHECK(cudaFuncSetAttribute(k_bcd<TS, kNT, false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    MFG_CUDA_CHECK(cudaFuncSetAttribute(k_bcd<TS, kNT, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    MFG_CUDA_CHECK(cudaFuncSetAttribute(k_bcd<TS, kNT, true, 8>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    MFG_CUDA_CHECK(cudaFuncSetAttribute(k_bcd<TS, kNTG>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  MFG_CUDA_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), stream));
  if (smax >= 1) {
    const size_t psm = smem_packed(k, smax);
    MFG_CUDA_CHECK(cudaFuncSetAttribute(k_bcd_packed<TS>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm));
    k_bcd_packed<TS><<<grid_for_rows(lay->nrows), kNT, psm, stream>>>(
        *lay, k, (const TS*)vals, (const TS*)other, ldo, lam, (TS*)out, ldout, smax, bad, rs.order,
        rs.ticket);
    MFG_LAUNCH_CHECK();
  }
  if (global)
    k_bcd<TS, kNTG><<<grid, kNTG, smem, stream>>>(*lay, k, (const TS*)vals, (const TS*)other, ldo,
                                                 lam, (TS*)out, ldout, gs, 1, bad,
                                                 smax >= 1 ? smax + 1 : 0, rs.order, rs.ticket + 1,
                                                 SplitPlan{});
  else
  {
    auto kern = k <= kTinyK      ? k_bcd<TS, kNT, true, 8>
                : small_k_path(k) ? k_bcd<TS, kNT, true>
                                  : k_bcd<TS, kNT, false>;
    kern<<<grid, kNT, smem, stream>>>(*lay, k, (const TS*)vals, (const TS*)other, ldo, lam,
                                      (TS*)out, ldout, gs, 0, bad, 0, rs.order, rs.ticket, sp);
  }
  MFG_LAUNCH_CHECK();
  return MFG_OK;
}

}  // namespace

size_t bcd_workspace(const mfg_layout* lay, int k) {
  Sizer s;
  s.take<int>(1);
  if (k > kSmemMaxK) s.take<double>((size_t)2 * kNumSMs * k * k);
  RowSched rs;
  unsigned *kin, *kout;
  int* rin;
  void* tmp;
  size_t tmpb;
  take_sched(s, lay ? lay->nrows : 0, &rs, &kin, &kout, &rin, &tmp, &tmpb);
  if (k <= kSmemMaxK && lay) {
    SplitPlan sp;
    int4* items;
    int* info;
    take_split(s, grid_for_rows(lay->nrows), k, &sp, &items, &info);
  }
  if (dm_path(k) && lay) {   // the DMMA path's plan (sized on its own, after the shared prefix)
    Sizer s2;
    s2.take<int>(1);
    RowSched rs2;
    unsigned *kin2, *kout2;
    int* rin2;
    void* tmp2;
    size_t tmpb2;
    take_sched(s2, lay->nrows, &rs2, &kin2, &kout2, &rin2, &tmp2, &tmpb2);
    SplitPlan sp;
    int *cnt, *off, *info;
    int4* items;
    void* tmp;
    size_t tmpb;
    take_dm_split(s2, lay->nnz, lay->nrows, k, &sp, &cnt, &off, &items, &info, &tmp, &tmpb);
    if (s2.off > s.off) s.off = s2.off;
  }
  return s.off + 512;
}

int bcd_dispatch(int dtype, const mfg_layout* lay, int k, const void* vals, const void* other,
                 int ldo, double lam, void* out, int ldout, void* ws, size_t wsb,
                 cudaStream_t stream) {
  if (dtype == MFG_F64)
    return do_bcd<double>(lay, k, vals, other, ldo, lam, out, ldout, ws, wsb, stream);
  return do_bcd<float>(lay, k, vals, other, ldo, lam, out, ldout, ws, wsb, stream);
}

}  // namespace mfg
