// The shared-memory staged Omega sweep (fp32).
//
// The all-gather sweep (sweep.cu, k_sweep_g8f) moves one k-wide factor row
// through L2 per entry and orientation; at c4/c5 it runs at the L2->SM
// throughput cap, at c2 at the L2 gather latency. This kernel instead cuts
// the gathered factor into blocks of S rows that fit one SM's shared memory
// (rows ranked by degree, so the Zipf head lands in the first blocks), and
// reorders each orientation's entry stream by (block, output row, col):
//
//   stream = [block 0 entries | block 1 | ... | cold entries], each segment
//            32-entry aligned, sorted by output row inside a segment.
//
// A persistent CTA per SM walks its tiles (a tile = up to 64 chunks of one
// segment, one chunk per 8-lane worker); on a block change it stages the
// block's S rows into shared memory with cp.async, and its workers then
// gather factor rows with LDS.128 instead of LDG.128. Segments whose rows are
// too sparse to amortise staging (cold) gather from global memory as before.
//
// A worker's run of entries with the same output row inside its chunk is a
// "piece": the piece's partial R.H vector is stored once to a piece buffer,
// and k_staged_fold adds the pieces of every output row in a fixed order
// (stream order), then applies out_scale. Everything is deterministic: the
// tile -> CTA assignment is static, and no floating-point atomics are used.
//
// Replaces the same reference calls as mfg_sweep: pair_values /
// residual_on_omega (mfg/data.py:253-280), grad.csr @ H and grad.csr_t @ W
// (mfg/operators.py:108,117; mfg/mfsolver.py:74), loss_quad (data.py:291)
// and FactorPair.frob_sq (operators.py:53-55).
#include <cstdlib>

#include "common.cuh"

#ifndef MFG_UNROLL_U
#define MFG_UNROLL_U 0  // unroll the 4 group-batches of a ring block
#endif
#include "engine.cuh"

namespace mfg {
namespace {

// CTA shape per lane-slice width: V = 4 (k <= 32) runs 512 threads (64
// eight-lane workers, <= 128 registers); V = 8 (k <= 64) runs 256 threads:
// the two-chunk slices need ~220 registers, and the register file is split
// over the 4 schedulers (10 warps would cap a thread at 168 and spill).
template <int V>
__host__ __device__ constexpr int s_threads() { return V == 4 ? 512 : 256; }
// per worker ring: cols | vals | pos, each [2 slots][32 entries]
constexpr int kRingWords = 3 * 64;
constexpr int kSmemDyn = 227 * 1024 - 1024;  // dynamic; static s_part/s_last take the rest
template <int V>
__host__ __device__ constexpr int s_smem_fixed() {
  return (s_threads<V>() / 8) * (kRingWords * 4 + 8 * 4) + 64;
}

__host__ __device__ inline int row_bytes(int k) { return ((k * 4 + 15) / 16) * 16; }

struct SPassDev {
  const int32_t* sidx;
  const int32_t* prow;     // piece -> output row (+2 padding)
  const float* svals;
  const int32_t* spos;
  const uint32_t* bmask;
  const int32_t* members;
  int S;
  const float* self;
  int lds;
  const float* other;
  int ldo;
  float* R;
  float* vpart;
};

struct SArgs {
  SPassDev p[2];
  const int4* chunks;     // E0, E1, piece0, pass
  const int4* tiles;      // pass, block, chunk begin, chunk end
  const int* tile_nblk;   // 32-entry blocks per chunk of the tile
  int ntiles;
  double* tile_part;      // [ntiles] sum r^2 of each tile (pass 0; 0 for pass 1)
  int k, rbe;             // rbe = row_bytes(k) / 4 floats
  // reductions
  const float* W; int64_t wcount;
  const float* H; int64_t hcount;
  double* block_part;     // [grid][2] |W|^2, |H|^2 slices
  unsigned int* counter;  // [0] finished CTAs, [1] tile tickets; zero at rest
  double* sums;           // sum r^2, |W|^2, |H|^2
};

__device__ __forceinline__ void cp_async16a(void* sdst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

// Lane q of a worker holds its dims in 16-byte chunks: chunk c covers
// elements [c*32 + 4q, +4) (one LDS/LDG.128 per chunk reads 128 contiguous
// bytes of a row across the 8 lanes). V = 4 (k <= 32) or 8 (k <= 64).
template <int V, bool SMEM>
__device__ __forceinline__ void grow(const float* g, uint32_t s, float (&o)[V], unsigned live) {
#pragma unroll
  for (int c = 0; c < V / 4; ++c) {
    if ((live >> c) & 1u) {
      const float4 x = SMEM ? lds128(s + c * 128) : *reinterpret_cast<const float4*>(g + c * 32);
      o[4 * c] = x.x; o[4 * c + 1] = x.y; o[4 * c + 2] = x.z; o[4 * c + 3] = x.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) o[4 * c + e] = 0.f;
    }
  }
}

template <int V>
__device__ __forceinline__ void grow_g(const float* g, float (&o)[V], unsigned live) {
  grow<V, false>(g, 0u, o, live);
}

__device__ __forceinline__ float reduce8f(float (&v)[8]) {
  const int q = threadIdx.x & 7;
#pragma unroll
  for (int s = 4; s >= 1; s >>= 1) {
    const bool upper = (q & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float send = upper ? v[i] : v[i + s];
      const float keep = upper ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

template <int V>
__device__ __forceinline__ float dot8(const float (&w)[V], const float (&h)[V]) {
  float2 s = __fmul2_rn(make_float2(w[0], w[1]), make_float2(h[0], h[1]));
#pragma unroll
  for (int j = 2; j < V; j += 2) s = __ffma2_rn(make_float2(w[j], w[j + 1]), make_float2(h[j], h[j + 1]), s);
  return s.x + s.y;
}

template <int V>
__device__ __forceinline__ void axpy8(float (&acc)[V], float r, const float (&h)[V]) {
  const float2 rr = make_float2(r, r);
#pragma unroll
  for (int j = 0; j < V; j += 2) {
    const float2 t = __ffma2_rn(rr, make_float2(h[j], h[j + 1]), make_float2(acc[j], acc[j + 1]));
    acc[j] = t.x; acc[j + 1] = t.y;
  }
}

template <int V>
__device__ __forceinline__ void store_piece(float* p, const float (&acc)[V], unsigned live) {
#pragma unroll
  for (int c = 0; c < V / 4; ++c)
    if ((live >> c) & 1u)
      *reinterpret_cast<float4*>(p + c * 32) = make_float4(acc[4 * c], acc[4 * c + 1], acc[4 * c + 2], acc[4 * c + 3]);
}

// One worker (8 lanes) over one chunk [E0, E1) of a segment. nblk 32-entry
// blocks are iterated by every worker of the warp (uniform trip count);
// entries past E1 are masked. Returns the worker's sum r^2 (all 8 lanes).
//
// Self rows are prefetched one piece ahead from the plan's piece -> row
// table: at every piece change w <- wn, and the load of the row after next
// is issued, so the self-row latency overlaps a whole piece of entries
// instead of stalling the batch where the row starts.
template <int V, bool SMEM>
__device__ __forceinline__ double run_piece_worker(const SPassDev& P, int E0, int E1, int piece,
                                                   int nblk, int k, int rbe, uint32_t sblk,
                                                   int32_t* s_ring, float* s_r) {
  const int q = threadIdx.x & 7;
  const int nvalid_all = E1 - E0;
  const bool active = nvalid_all > 0;
  unsigned livem = 0;
#pragma unroll
  for (int c = 0; c < V / 4; ++c) livem |= (c * 32 + q * 4 < k ? 1u : 0u) << c;
  // One-chunk slices (V = 4): lanes whose dims are all >= k read lane 0's
  // chunk (no extra bytes) against a zero self slice.
  constexpr bool kAlias = V == 4;
  const bool live0 = (livem & 1u) != 0;
  const int qoff = (kAlias && !live0) ? 0 : q * 4;        // element offset of the lane's chunk
  const float* __restrict__ self = P.self + q * 4;
  const int64_t lds = P.lds;
  const uint32_t gstride_s = (uint32_t)rbe * 4u;          // bytes per staged row
  const uint32_t sbase = sblk + (uint32_t)qoff * 4u;
  const float* __restrict__ gbase = P.other + qoff;
  const int64_t ldo = P.ldo;
  const int32_t* __restrict__ pidx = P.sidx + E0;
  const float* __restrict__ pval = P.svals + E0;
  const uint32_t* __restrict__ pbm = P.bmask + (E0 >> 5);
  const int32_t* __restrict__ ppos = P.spos + E0;
  const int32_t* __restrict__ prow = P.prow;
  float* __restrict__ R = P.R;
  // ring layout: [0,64) cols, [64,128) vals, [128,192) pos
  float* s_vring = reinterpret_cast<float*>(s_ring + 64);

  float w[V], wn[V];
  int rnext = 0;
  if (active) {
    grow_g<V>(self + (int64_t)prow[piece] * lds, w, livem);
    grow_g<V>(self + (int64_t)prow[piece + 1] * lds, wn, livem);
    rnext = prow[piece + 2];
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) { w[v] = 0.f; wn[v] = 0.f; }
  }
  // piece change: the prefetched row becomes current, the next one is issued
  auto advance = [&]() {
#pragma unroll
    for (int v = 0; v < V; ++v) w[v] = wn[v];
    grow_g<V>(self + (int64_t)rnext * lds, wn, livem);
    rnext = prow[piece + 2];
  };
  float acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = 0.f;
  double sq = 0.0;
  float* __restrict__ vp = P.vpart + q * 4;
  auto flush = [&]() {
    store_piece<V>(vp + (int64_t)piece * rbe, acc, livem);
    ++piece;
  };

  auto fetch_block = [&](int b) {
    if (b * 32 >= nvalid_all) return;
    const int slot = b & 1;
    const int o = b * 32 + q * 4;
    cp_async16a(s_ring + slot * 32 + q * 4, pidx + o);
    cp_async16a(s_vring + slot * 32 + q * 4, pval + o);
    if (R) cp_async16a(s_ring + 128 + slot * 32 + q * 4, ppos + o);
  };
#pragma unroll
  for (int z = 0; z < 24; ++z) s_ring[q * 24 + z] = 0;
  __syncwarp();
  fetch_block(0);
  cp_commit();
  uint32_t mw_next = active ? pbm[0] : 0u;
  for (int b = 0; b < nblk; ++b) {
    fetch_block(b + 1 < nblk ? b + 1 : nblk);
    cp_commit();
    cp_wait<1>();
    __syncwarp();
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
      const int pos = R ? s_ring[128 + slot * 32 + u * 8 + q] : 0;
      const int* rc = s_ring + slot * 32 + u * 8;
      const float a = s_vring[slot * 32 + u * 8 + q];
      int cols[8];
      {
        const int4 x0 = reinterpret_cast<const int4*>(rc)[0];
        const int4 x1 = reinterpret_cast<const int4*>(rc)[1];
        cols[0] = x0.x; cols[1] = x0.y; cols[2] = x0.z; cols[3] = x0.w;
        cols[4] = x1.x; cols[5] = x1.y; cols[6] = x1.z; cols[7] = x1.w;
      }
      float h[8][V];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (SMEM) grow<V, true>(nullptr, sbase + (uint32_t)cols[i] * gstride_s, h[i], kAlias ? 1u : livem);
        else grow_g<V>(gbase + (int64_t)cols[i] * ldo, h[i], kAlias ? 1u : livem);
      }
      float p[8];
      const int i0 = bits ? __ffs(bits) - 1 : 8;
      const bool one_start = kAlias && bits != 0u && (bits & (bits - 1u)) == 0u;
      // dots; w_old is needed by the accumulation split below only through acc
      if (bits == 0u) {
#pragma unroll
        for (int i = 0; i < 8; ++i) p[i] = dot8<V>(w, h[i]);
      } else if (one_start) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float ws[V];
#pragma unroll
          for (int v = 0; v < V; ++v) ws[v] = i < i0 ? w[v] : wn[v];
          p[i] = dot8<V>(ws, h[i]);
        }
      } else {
        // several row starts: walk them (the first uses the prefetched row,
        // later ones wait for the row issued at the previous start)
        float wc[V], wq[V];
#pragma unroll
        for (int v = 0; v < V; ++v) { wc[v] = w[v]; wq[v] = wn[v]; }
        int rq = rnext, pc = piece;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if ((bits >> i) & 1u) {
#pragma unroll
            for (int v = 0; v < V; ++v) wc[v] = wq[v];
            grow_g<V>(self + (int64_t)rq * lds, wq, livem);
            ++pc;
            rq = prow[pc + 2];
          }
          p[i] = dot8<V>(wc, h[i]);
        }
      }
      const float dot = reduce8f(p);
      const float r = valid ? dot - a : 0.f;
      if (valid) {
        if (R) R[pos] = r;
        sq += (double)r * (double)r;
      }
      __syncwarp();
      s_r[q] = r;
      __syncwarp();
      float r8[8];
      {
        const float4 x0 = reinterpret_cast<const float4*>(s_r)[0];
        const float4 x1 = reinterpret_cast<const float4*>(s_r)[1];
        r8[0] = x0.x; r8[1] = x0.y; r8[2] = x0.z; r8[3] = x0.w;
        r8[4] = x1.x; r8[5] = x1.y; r8[6] = x1.z; r8[7] = x1.w;
      }
      if (bits == 0u) {
#pragma unroll
        for (int i = 0; i < 8; ++i) axpy8<V>(acc, r8[i], h[i]);
      } else if (one_start) {
#pragma unroll
        for (int i = 0; i < 8; ++i) axpy8<V>(acc, i < i0 ? r8[i] : 0.f, h[i]);
        flush();
        advance();
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) axpy8<V>(acc, i < i0 ? 0.f : r8[i], h[i]);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if ((bits >> i) & 1u) {
            flush();
            advance();
#pragma unroll
            for (int j = 0; j < V; ++j) acc[j] = 0.f;
          }
          axpy8<V>(acc, r8[i], h[i]);
        }
      }
    }
  }
  cp_wait<0>();
  if (active) flush();
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  return sq;
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n}\n" ::"r"(bar), "r"(parity) : "memory");
}

template <int V>
__global__ void __launch_bounds__(s_threads<V>(), 1) k_sweep_staged(SArgs A) {
  constexpr int NT = s_threads<V>();
  constexpr int G = NT / 8;
  extern __shared__ __align__(128) unsigned char smem[];
  int32_t* ring = reinterpret_cast<int32_t*>(smem);                       // [G][256]
  float* sr = reinterpret_cast<float*>(smem + G * kRingWords * 4);         // [G][8]
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(smem + G * (kRingWords * 4 + 32));
  unsigned char* blk = smem + s_smem_fixed<V>();
  const uint32_t sblk = (uint32_t)__cvta_generic_to_shared(blk);
  const uint32_t sbar = (uint32_t)__cvta_generic_to_shared(mbar);
  const int g = threadIdx.x >> 3;
  const int rbe = A.rbe;
  const uint32_t rb = (uint32_t)rbe * 4u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase = 0;
  int staged_pass = -1, staged_block = -1;
  __shared__ int s_tile;
  __shared__ double s_wsq[NT / 32];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  // Tiles are handed out in stream order by a ticket counter, so CTAs that
  // drew cheap tiles take more (the per-tile cost varies with row starts,
  // staging and cold gathers far more than any static model predicts).
  // sum r^2 is folded per tile in fixed worker order and stored by tile
  // index, so the result does not depend on which CTA ran which tile.
  for (;;) {
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(A.counter + 1, 1u);
    __syncthreads();  // also: every worker is done with the previous tile
    const int t = s_tile;
    if (t >= A.ntiles) break;
    const int4 tile = A.tiles[t];
    const int pass = tile.x, block = tile.y;
    const SPassDev& P = pass ? A.p[1] : A.p[0];
    if (block >= 0 && (pass != staged_pass || block != staged_block)) {
      // Stage the block's S rows: one bulk copy (cp.async.bulk, TMA engine)
      // per row, completion counted in bytes on the CTA's mbarrier.
      if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     ::"r"(sbar), "r"((uint32_t)P.S * rb) : "memory");
      __syncthreads();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const int32_t* mem = P.members + (int64_t)block * P.S;
      for (int s = threadIdx.x; s < P.S; s += NT) {
        const float* src = P.other + (int64_t)mem[s] * P.ldo;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(sblk + (uint32_t)s * rb), "l"(src), "r"(rb), "r"(sbar) : "memory");
      }
      mbar_wait(sbar, phase);
      phase ^= 1u;
      staged_pass = pass;
      staged_block = block;
    }
    const int nblk = A.tile_nblk[t];
    const int c = tile.z + g;
    int4 ch = make_int4(0, 0, 0, 0);
    if (c < tile.w) ch = A.chunks[c];
    const bool warp_live = __any_sync(0xffffffffu, c < tile.w);
    double sq = 0.0;
    if (warp_live) {
      if (block >= 0)
        sq = run_piece_worker<V, true>(P, ch.x, ch.y, ch.z, nblk, A.k, rbe, sblk, ring + g * kRingWords,
                                       sr + g * 8);
      else
        sq = run_piece_worker<V, false>(P, ch.x, ch.y, ch.z, nblk, A.k, rbe, sblk, ring + g * kRingWords,
                                        sr + g * 8);
    }
    // the 4 workers of the warp (each worker's lanes hold its sum)
    sq += __shfl_xor_sync(0xffffffffu, sq, 8);
    sq += __shfl_xor_sync(0xffffffffu, sq, 16);
    if (lane == 0) s_wsq[wib] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double ts = 0.0;
      for (int w = 0; w < NT / 32; ++w) ts += s_wsq[w];
      A.tile_part[t] = pass == 0 ? ts : 0.0;
    }
  }
  // dense norms over fixed slices
  const int64_t gt = (int64_t)blockIdx.x * NT + threadIdx.x, gs = (int64_t)gridDim.x * NT;
  double w2 = 0.0, h2 = 0.0;
  for (int64_t i = gt; i < A.wcount; i += gs) { const double x = A.W[i]; w2 += x * x; }
  for (int64_t i = gt; i < A.hcount; i += gs) { const double x = A.H[i]; h2 += x * x; }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    w2 += __shfl_xor_sync(0xffffffffu, w2, o);
    h2 += __shfl_xor_sync(0xffffffffu, h2, o);
  }
  __shared__ double s_part[NT / 32][3];
  __shared__ int s_last;
  if (lane == 0) { s_part[wib][1] = w2; s_part[wib][2] = h2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b1 = 0.0, b2 = 0.0;
    for (int w = 0; w < NT / 32; ++w) { b1 += s_part[w][1]; b2 += s_part[w][2]; }
    double* bp = A.block_part + 2 * blockIdx.x;
    bp[0] = b1; bp[1] = b2;
    asm volatile("fence.release.gpu;" ::: "memory");
    s_last = atomicAdd(A.counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  double u0 = 0.0, u1 = 0.0, u2 = 0.0;
  for (int t = threadIdx.x; t < A.ntiles; t += NT) u0 += __ldcg(A.tile_part + t);
  for (unsigned b = threadIdx.x; b < gridDim.x; b += NT) {
    u1 += __ldcg(A.block_part + 2 * b);
    u2 += __ldcg(A.block_part + 2 * b + 1);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    u0 += __shfl_xor_sync(0xffffffffu, u0, o);
    u1 += __shfl_xor_sync(0xffffffffu, u1, o);
    u2 += __shfl_xor_sync(0xffffffffu, u2, o);
  }
  __syncthreads();
  if (lane == 0) { s_part[wib][0] = u0; s_part[wib][1] = u1; s_part[wib][2] = u2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double v0 = 0.0, v1 = 0.0, v2 = 0.0;
    for (int w = 0; w < NT / 32; ++w) { v0 += s_part[w][0]; v1 += s_part[w][1]; v2 += s_part[w][2]; }
    A.sums[0] = v0; A.sums[1] = v1; A.sums[2] = v2;
    A.counter[0] = 0u;
    A.counter[1] = 0u;
  }
}

// Output rows from their pieces: out[i] = out_scale * sum of the pieces of
// row i in stream order (zero for rows without entries). 8 lanes per row,
// lane q adds the 16-byte chunks q and q + 8 of every piece.
struct FoldPass {
  const int32_t* pptr;
  const int32_t* plist;
  const float* vpart;
  float* out;
  int nrows;
};

__global__ void __launch_bounds__(256) k_staged_fold(FoldPass F0, FoldPass F1, int k, int rbe,
                                                     float out_scale) {
  const int q = threadIdx.x & 7;
  const int nchk = rbe / 4;
  const int64_t grow0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int64_t gstride = ((int64_t)gridDim.x * blockDim.x) >> 3;
  for (int64_t gr = grow0; gr < (int64_t)F0.nrows + F1.nrows; gr += gstride) {
    const bool second = gr >= F0.nrows;
    const FoldPass& F = second ? F1 : F0;
    const int i = (int)(second ? gr - F0.nrows : gr);
    const int p0 = F.pptr[i], p1 = F.pptr[i + 1];
    float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
    const bool c0 = q < nchk, c1 = q + 8 < nchk;
    // 8 pieces per round: lane u of the group loads piece id u, the ids are
    // broadcast in the group, all 16 chunk loads are in flight together,
    // then added in piece order (deterministic)
    const unsigned gmask = 0xFFu << (threadIdx.x & 24);
    const int gbase = threadIdx.x & 24;
    for (int p = p0; p < p1; p += 8) {
      const int n = min(8, p1 - p);
      const int myid = q < n ? F.plist[p + q] : 0;
      float4 t0[8], t1[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int id = __shfl_sync(gmask, myid, gbase + u);
        const float4* base = reinterpret_cast<const float4*>(F.vpart + (int64_t)id * rbe);
        const bool ok = u < n;
        t0[u] = (ok && c0) ? __ldcg(base + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        t1[u] = (ok && c1) ? __ldcg(base + q + 8) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a0.x += t0[u].x; a0.y += t0[u].y; a0.z += t0[u].z; a0.w += t0[u].w;
        a1.x += t1[u].x; a1.y += t1[u].y; a1.z += t1[u].z; a1.w += t1[u].w;
      }
    }
    float* o = F.out + (int64_t)i * k;
    const float v0[4] = {a0.x, a0.y, a0.z, a0.w}, v1[4] = {a1.x, a1.y, a1.z, a1.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int d0 = q * 4 + e, d1 = 32 + q * 4 + e;
      if (d0 < k) o[d0] = v0[e] * out_scale;
      if (d1 < k) o[d1] = v1[e] * out_scale;
    }
  }
}

}  // namespace

int staged_workers(int k) {
  if (k < 1 || k > 64) return 0;
  return (k <= 32 ? s_threads<4>() : s_threads<8>()) / 8;
}

int staged_block_rows(int k) {
  if (k < 1 || k > 64) return 0;
  return (kSmemDyn - (k <= 32 ? s_smem_fixed<4>() : s_smem_fixed<8>())) / row_bytes(k);
}

size_t staged_workspace(const mfg_staged_plan* pl) {
  Sizer s;
  s.take<float>((size_t)(pl->pass[0].npieces + 1) * (row_bytes(pl->k) / 4));
  s.take<float>((size_t)(pl->pass[1].npieces + 1) * (row_bytes(pl->k) / 4));
  s.take<double>((size_t)2 * (pl->grid + 1));
  s.take<double>((size_t)pl->ntiles + 1);
  s.take<unsigned int>(4);
  s.take<double>(4);
  return s.off;
}

int staged_sweep(const mfg_staged_plan* pl, const float* W, int ldw, const float* H, int ldh,
                 float* R, float* RH, float* RtW, double out_scale, double* sums, void* ws,
                 size_t wsb, cudaStream_t stream) {
  const int k = pl->k;
  MFG_REQUIRE(k >= 1 && k <= 64, "staged sweep: k must be in [1, 64]");
  MFG_REQUIRE(ldw >= k && ldh >= k && (ldw % 4) == 0 && (ldh % 4) == 0,
              "staged sweep: ldw, ldh must be >= k and multiples of 4 (16-byte rows)");
  MFG_REQUIRE(RH && RtW && sums, "staged sweep: RH, RtW and sums are required");
  MFG_REQUIRE(!R || pl->pass[0].spos, "staged sweep: R requested from a plan built without positions");
  MFG_REQUIRE(pl->grid >= 1 && pl->grid <= 4 * kNumSMs, "staged sweep: bad grid");
  const int S = staged_block_rows(k);
  MFG_REQUIRE(pl->pass[0].S >= 1 && pl->pass[1].S >= 1 &&
                  (pl->l1 || (pl->pass[0].S <= S && pl->pass[1].S <= S)),
              "staged sweep: block rows exceed the shared-memory capacity for this k");
  const int rbe = row_bytes(k) / 4;
  Carver c(ws, wsb);
  float* vp0 = c.take<float>((size_t)(pl->pass[0].npieces + 1) * rbe);
  float* vp1 = c.take<float>((size_t)(pl->pass[1].npieces + 1) * rbe);
  double* bp = c.take<double>((size_t)2 * (pl->grid + 1));
  double* tp = c.take<double>((size_t)pl->ntiles + 1);
  unsigned int* counter = c.take<unsigned int>(4);
  double* tmp = c.take<double>(4);
  MFG_REQUIRE(c.ok, "staged sweep workspace too small");
  SArgs A{};
  for (int p = 0; p < 2; ++p) {
    const mfg_staged_pass& sp = pl->pass[p];
    SPassDev& d = A.p[p];
    d.sidx = sp.sidx; d.prow = sp.prow; d.svals = sp.svals; d.spos = p == 0 ? sp.spos : nullptr;
    d.bmask = sp.bmask; d.members = sp.members; d.S = sp.S;
    d.self = p == 0 ? W : H; d.lds = p == 0 ? ldw : ldh;
    d.other = p == 0 ? H : W; d.ldo = p == 0 ? ldh : ldw;
    d.R = p == 0 ? R : nullptr;
    d.vpart = p == 0 ? vp0 : vp1;
  }
  if (!R) A.p[0].spos = nullptr;
  A.chunks = reinterpret_cast<const int4*>(pl->chunks);
  A.tiles = reinterpret_cast<const int4*>(pl->tiles);
  A.tile_nblk = pl->tile_nblk;
  A.ntiles = pl->ntiles;
  A.tile_part = tp;
  A.k = k;
  A.rbe = rbe;
  A.W = W; A.wcount = (int64_t)pl->pass[0].nrows * ldw;
  A.H = H; A.hcount = (int64_t)pl->pass[1].nrows * ldh;
  A.block_part = bp;
  A.counter = counter;
  A.sums = tmp;
  // nothing staged (L1-blocked plans): request only the rings, so the SM's
  // unified L1/shared storage is left to the L1 cache
  bool any_staged = false;
  for (int t = 0; t < 2; ++t) any_staged |= pl->pass[t].nblocks > 0 && !pl->l1;
  const int smem = any_staged ? kSmemDyn : (k <= 32 ? s_smem_fixed<4>() : s_smem_fixed<8>());
  auto go = [&](auto kern) -> int {
    MFG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    MFG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        any_staged ? 100 : 0));
    kern<<<pl->grid, k <= 32 ? s_threads<4>() : s_threads<8>(), smem, stream>>>(A);
    MFG_LAUNCH_CHECK();
    return MFG_OK;
  };
  prof_begin(stream);  // the timed region covers both kernels of the sweep
  int st = k <= 32 ? go(k_sweep_staged<4>) : go(k_sweep_staged<8>);
  if (st != MFG_OK) return st;
  static const bool skip_fold = getenv("MFG_STAGED_SKIP_FOLD") != nullptr;  // diagnostics only
  if (skip_fold) {
    prof_end(stream);
    MFG_CUDA_CHECK(cudaMemcpyAsync(sums, tmp, 3 * sizeof(double), cudaMemcpyDeviceToDevice, stream));
    return MFG_OK;
  }
  FoldPass F0{pl->pass[0].pptr, pl->pass[0].plist, vp0, RH, pl->pass[0].nrows};
  FoldPass F1{pl->pass[1].pptr, pl->pass[1].plist, vp1, RtW, pl->pass[1].nrows};
  int64_t rows = (int64_t)F0.nrows + F1.nrows;
  int fgrid = (int)((rows * 8 + 255) / 256);
  if (fgrid > 8 * kNumSMs) fgrid = 8 * kNumSMs;
  if (fgrid < 1) fgrid = 1;
  k_staged_fold<<<fgrid, 256, 0, stream>>>(F0, F1, k, rbe, (float)out_scale);
  MFG_LAUNCH_CHECK();
  prof_end(stream);
  MFG_CUDA_CHECK(cudaMemcpyAsync(sums, tmp, 3 * sizeof(double), cudaMemcpyDeviceToDevice, stream));
  return MFG_OK;
}

}  // namespace mfg
