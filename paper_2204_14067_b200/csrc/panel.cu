// The piece sweep: every entry of a pass belongs to a *piece* -- a run of one
// self row's entries -- and 4- or 8-lane groups walk pieces; the gathered
// factor rows of the hot pieces come from shared-memory panels.
//
// The sweep's two passes (CSR: r = w_i.h_j - a, R.H; CSC: the same residual,
// R^T.W; mfg/data.py:253-263, mfg/operators.py:108,117) gather one k-wide
// factor row per entry. With every gather served by L2 the sweep is bound by
// the L2->SM crossbar (K4). Gather counts are Zipf-skewed, so most
// gathers go to a few thousand rows: this file runs those entries from
// *panels* -- sets of PR gathered rows held in one SM's shared memory (200 KB)
// -- with k_panel4 (rows of one 32-dim block, k <= 40) or k_panel (k = 64),
// and the remaining (cold) entries as pieces on global loads with k_cold4 (or,
// for k = 64, through the gather kernel in sweep.cu).
//
// Layout (built once per Omega and k by panel.py):
//   panel_ids [NP][PR]   global gathered-row id of each panel slot (-1: none)
//   pieces    [NPC]      {self row, first record block, length, output slot}:
//                        a run of entries of one self row inside one panel (hot)
//                        or of its cold entries, at most Lmax entries; listed by
//                        decreasing length (hot pieces: per panel and chunk)
//   recs                 hot: record blocks of 16 entries (96 B): 16 x u16 panel-
//                        local rows, then 16 x f32 A values; cold: 128 B blocks of
//                        16 x u32 gathered-row ids, 16 x f32 A. A piece owns whole
//                        blocks (zero padded). Inside a hot piece the entries are
//                        ordered so that the 4 entries of a batch fall into
//                        different 32-byte bank windows of the tail array where
//                        possible.
//   plist     [NL]       {pass, panel, first piece, end piece}, panel-major
//   cta_start [CTAs]     the list element each CTA starts at (work-proportional)
//   frows / fbeg / fcnt  self rows that own slots and their slot ranges; slots are
//                        numbered in (self row, panel, run) order, cold pieces last
//
// k_panel (8-lane groups; k_panel4 below is the 4-lane version): persistent
// CTAs (one per SM) walk the panel list cyclically from their start element; a
// CTA loads a panel that still has pieces with cp.async, then its warps take
// rounds of 4 pieces (one per 8-lane group) from the element's global ticket,
// the next round's descriptors and self rows loading during the current one.
// Records stream through a per-group cp.async ring. Per 4 entries a group
// issues 4 conflict-free LDS.128 of the rows' first 128 bytes (lane q holds
// dims [4q, 4q+4) of 32-dim blocks), one LDS.128 of the 4 entries' tail chunks
// (k = 40: dims 32..39, lane q holds chunk q&1 of entry q>>1), a transposed
// 8-lane butterfly that leaves entry q>>1's dot in lanes 2(q>>1), 2(q>>1)+1,
// and the accumulation of r * row in registers. A piece writes its partial
// output vector to its slot; k_panel_fold sums a self row's slots in slot
// order, so the result does not depend on which CTA ran which piece (bitwise
// reproducible for a given layout).
#include <stdlib.h>

#include "common.cuh"
#include "engine.cuh"

namespace mfg {

namespace {

constexpr int kPT = 640;               // threads per CTA (20 warps, <= 102 registers)
constexpr int kPanelBytes = 211 * 1024; // the panel
constexpr int kBlockBytes = 96;         // a record block: 16 x u16 local rows, 16 x f32 values
constexpr int kRingBytes = (kPT / 32) * 4 * 2 * kBlockBytes;  // per 8-lane group: 2 blocks
constexpr int kPanelSmem = kPanelBytes + kRingBytes;

struct PanelPass {
  const float* self;        // self rows (W in the CSR pass, H in the CSC pass)
  const float* gath;        // gathered table
  const int32_t* panel_ids;
  const int4* pieces;
  const int4* recs;         // record blocks, 6 int4 each
  float* rhot;              // residuals in record order (nullable)
  float* po;                // piece outputs [slot][KP]
  double* psq;              // per-slot sum r^2 (nullable)
  int lds, ldg;
};

struct PanelArgs {
  PanelPass p[2];
  const int4* plist;        // {pass, panel, first piece, end piece}
  const int32_t* cta_start; // [gridDim.x] first list element of each CTA
  int n_list;
  int PR;
  int* counters;            // [n_list] piece tickets, [n_list] finished CTAs (zero at rest)
};

__device__ __forceinline__ void cp16(void* sdst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ float4 lds128(unsigned a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds64(unsigned a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ float lds32(unsigned a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ float dot4(const float4& a, const float4& b) {
  float2 s = __fmul2_rn(make_float2(a.x, a.y), make_float2(b.x, b.y));
  s = __ffma2_rn(make_float2(a.z, a.w), make_float2(b.z, b.w), s);
  return s.x + s.y;
}

__device__ __forceinline__ void axpy4(float4& acc, float r, const float4& x) {
  const float2 rr = make_float2(r, r);
  const float2 lo = __ffma2_rn(rr, make_float2(x.x, x.y), make_float2(acc.x, acc.y));
  const float2 hi = __ffma2_rn(rr, make_float2(x.z, x.w), make_float2(acc.z, acc.w));
  acc.x = lo.x; acc.y = lo.y; acc.z = hi.x; acc.w = hi.y;
}

// NB: 32-dim blocks per row (k = 40: 1, k = 64: 2); KT: 16-byte tail chunks
// (k = 40: 2; 0 when the row is whole blocks).
template <int NB, int KT>
__global__ void __launch_bounds__(kPT, 1) k_panel(const PanelArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int KC = NB * 8 + KT;       // 16-byte chunks per row
  constexpr int KP = KC * 4;            // floats per row / per piece output
  constexpr int KTD = KT > 0 ? KT : 1;
  float* s_main = reinterpret_cast<float*>(smem_raw);
  float* s_tail = s_main + (size_t)A.PR * NB * 32;
  __shared__ int s_left;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int q = lane & 7, g = lane >> 3;
  const int ei = q >> 1;                // the entry of a 4-batch this lane finishes
  // this group's record ring: 2 slots of one 96-byte block (16 records = 4 batches)
  unsigned char* ring = smem_raw + kPanelBytes + (warp * 4 + g) * 2 * kBlockBytes;
  // 32-bit shared addresses and per-lane constants of the batch loop
  const unsigned a_main = (unsigned)__cvta_generic_to_shared(s_main) + q * 16;
  const unsigned a_tail = (unsigned)__cvta_generic_to_shared(s_tail) + (q % KTD) * 16;
  const unsigned a_ring = (unsigned)__cvta_generic_to_shared(ring);
  const bool t_hi = (ei >> 1) != 0;     // the tail entry's local row: upper word of the pair
  const int t_sh = (ei & 1) * 16;       // ... and its half
  const bool b2 = (q & 4) != 0, b1 = (q & 2) != 0, even = (q & 1) == 0;
  const int gb = lane & 24;
  int cur_key = -1;
  int li = A.cta_start[blockIdx.x];
  for (int step = 0; step < A.n_list; ++step, li = li + 1 == A.n_list ? 0 : li + 1) {
    const int4 it = A.plist[li];        // {pass, panel, first piece, end piece}
    const int npc = it.w - it.z;
    __syncthreads();                    // everyone is done with the previous panel
    if (tid == 0) s_left = npc - *reinterpret_cast<volatile int*>(A.counters + li);
    __syncthreads();
    if (s_left <= 0) continue;          // this panel's pieces are all taken
    const PanelPass& P = A.p[it.x];
    const int key = it.x * 65536 + it.y;
    if (key != cur_key) {               // consecutive elements may share a panel (column chunks)
      cur_key = key;
      const int32_t* ids = P.panel_ids + (size_t)it.y * A.PR;
      const int total = A.PR * KC;
      for (int c = tid; c < total; c += kPT) {
        const int r = c / KC, ch = c - r * KC;
        const int gid = ids[r];
        float* dst = ch < NB * 8 ? s_main + (size_t)r * NB * 32 + ch * 4
                                 : s_tail + (size_t)r * KT * 4 + (ch - NB * 8) * 4;
        if (gid >= 0) cp16(dst, P.gath + (size_t)gid * P.ldg + ch * 4);
        else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      cp_commit();
      cp_wait<0>();
    }
    __syncthreads();
    float* const rhot = P.rhot;
    const bool st_r = rhot != nullptr && even;   // even lanes store their pair's residual
    const bool want_sq = P.psq != nullptr;
    // Warps take 4 consecutive pieces (one per 8-lane group) from the panel's
    // list (sorted by decreasing length) through a global ticket, one round
    // ahead: the next round's descriptors and self rows load during this one.
    auto take = [&]() {
      int v = 0;
      if (lane == 0) v = atomicAdd(A.counters + li, 4);
      return __shfl_sync(0xffffffffu, v, 0);
    };
    auto load_desc = [&](int t0) {
      int4 d = make_int4(0, 0, 0, -1);  // {self row, first block, length, slot}; slot < 0: none
      if (t0 + g < npc) d = P.pieces[it.z + t0 + g];
      return d;
    };
    int t_cur = take();
    int4 pc = load_desc(t_cur);
    float4 hm[NB], ht = make_float4(0.f, 0.f, 0.f, 0.f);
    {
      const float* srow = P.self + (size_t)pc.x * P.lds;
#pragma unroll
      for (int b = 0; b < NB; ++b) hm[b] = *reinterpret_cast<const float4*>(srow + b * 32 + q * 4);
      if (KT > 0) ht = *reinterpret_cast<const float4*>(srow + NB * 32 + (q % KTD) * 4);
    }
    while (t_cur < npc) {
      const int t_nxt = take();
      const int4 pcn = load_desc(t_nxt);
      float4 hmn[NB], htn = make_float4(0.f, 0.f, 0.f, 0.f);
      const int len = pc.z;
      const int lim = len - ei;         // batch b holds this lane's entry iff 4 b < lim
      float* rh = rhot + (size_t)pc.y * 16 + ei;
      float4 am[NB], at = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int b = 0; b < NB; ++b) am[b] = make_float4(0.f, 0.f, 0.f, 0.f);
      double sq = 0.0;
      const int nb = (len + 3) >> 2;    // batches of 4 entries
      const int nblk = (nb + 3) >> 2;   // record blocks of 4 batches
      int nbw = nb;
      nbw = max(nbw, __shfl_xor_sync(0xffffffffu, nbw, 8));
      nbw = max(nbw, __shfl_xor_sync(0xffffffffu, nbw, 16));
      const int nblkw = (nbw + 3) >> 2;
      const int4* rp = P.recs + (size_t)pc.y * 6;
      const int jmax = max(nblk - 1, 0);
      if (q < 6) cp16(ring + q * 16, rp + q);  // block 0 -> slot 0
      cp_commit();
      for (int j = 0; j < nblkw; ++j) {
        {
          const int jn = min(j + 1, jmax);     // clamped: short pieces re-read their last block
          if (q < 6) cp16(ring + ((j + 1) & 1) * kBlockBytes + q * 16, rp + jn * 6 + q);
          cp_commit();
        }
        cp_wait<1>();
        __syncwarp();
        if (j == 0) {
          // the next round's self rows (its descriptors were requested a block ago)
          const float* srow = P.self + (size_t)pcn.x * P.lds;
#pragma unroll
          for (int b = 0; b < NB; ++b) hmn[b] = *reinterpret_cast<const float4*>(srow + b * 32 + q * 4);
          if (KT > 0) htn = *reinterpret_cast<const float4*>(srow + NB * 32 + (q % KTD) * 4);
        }
        const unsigned rs = a_ring + (j & 1) * kBlockBytes;
#pragma unroll 1
        for (int bb = 0; bb < 4; ++bb) {
          const int b = j * 4 + bb;
          if (b >= nbw) break;
          // this batch's records: 4 u16 local rows, and this lane's entry's value
          const uint2 lw = lds64(rs + bb * 8);
          const float a_mine = lds32(rs + 32 + (bb * 4 + ei) * 4);
          const unsigned l0 = lw.x & 0xffffu, l1 = lw.x >> 16, l2 = lw.y & 0xffffu, l3 = lw.y >> 16;
          const unsigned lt = ((t_hi ? lw.y : lw.x) >> t_sh) & 0xffffu;
          float4 m[4][NB];
#pragma unroll
          for (int x = 0; x < NB; ++x) {
            m[0][x] = lds128(a_main + l0 * (NB * 128) + x * 128);
            m[1][x] = lds128(a_main + l1 * (NB * 128) + x * 128);
            m[2][x] = lds128(a_main + l2 * (NB * 128) + x * 128);
            m[3][x] = lds128(a_main + l3 * (NB * 128) + x * 128);
          }
          float4 tt = make_float4(0.f, 0.f, 0.f, 0.f);
          if (KT > 0) tt = lds128(a_tail + lt * (KT * 16));
          float p[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            p[i] = dot4(m[i][0], hm[0]);
#pragma unroll
            for (int x = 1; x < NB; ++x) p[i] += dot4(m[i][x], hm[x]);
          }
          // transposed butterfly over the group's 8 lanes: entry q>>1 ends in
          // lanes 2(q>>1), 2(q>>1)+1 (fixed tree: deterministic)
          float k0 = b2 ? p[2] : p[0], k1 = b2 ? p[3] : p[1];
          const float s0 = b2 ? p[0] : p[2], s1 = b2 ? p[1] : p[3];
          k0 += __shfl_xor_sync(0xffffffffu, s0, 4);
          k1 += __shfl_xor_sync(0xffffffffu, s1, 4);
          float kk = b1 ? k1 : k0;
          const float ss = b1 ? k0 : k1;
          kk += __shfl_xor_sync(0xffffffffu, ss, 2);
          if (KT > 0) kk += dot4(tt, ht);
          kk += __shfl_xor_sync(0xffffffffu, kk, 1);
          const bool valid = b * 4 < lim;
          const float r = valid ? kk - a_mine : 0.f;
          const float r0 = __shfl_sync(0xffffffffu, r, gb);
          const float r1 = __shfl_sync(0xffffffffu, r, gb + 2);
          const float r2 = __shfl_sync(0xffffffffu, r, gb + 4);
          const float r3 = __shfl_sync(0xffffffffu, r, gb + 6);
#pragma unroll
          for (int x = 0; x < NB; ++x) {
            axpy4(am[x], r0, m[0][x]);
            axpy4(am[x], r1, m[1][x]);
            axpy4(am[x], r2, m[2][x]);
            axpy4(am[x], r3, m[3][x]);
          }
          if (KT > 0) axpy4(at, r, tt);
          if (st_r && valid) rh[b * 4] = r;
          if (want_sq) sq = fma((double)r, (double)r, sq);   // odd lanes duplicate their pair's r
        }
        __syncwarp();                  // slot j & 1 is refilled by the next iteration
      }
      cp_wait<0>();                    // drain the clamped copy before the ring is reused
      if (nblkw == 0) {
        const float* srow = P.self + (size_t)pcn.x * P.lds;
#pragma unroll
        for (int b = 0; b < NB; ++b) hmn[b] = *reinterpret_cast<const float4*>(srow + b * 32 + q * 4);
        if (KT > 0) htn = *reinterpret_cast<const float4*>(srow + NB * 32 + (q % KTD) * 4);
      }
      // the tail accumulators of lanes q = c, c+2, c+4, c+6 (entries 0..3) sum to chunk c
      if (KT > 0) {
#pragma unroll
        for (int o = 2; o <= 4; o <<= 1) {
          at.x += __shfl_xor_sync(0xffffffffu, at.x, o);
          at.y += __shfl_xor_sync(0xffffffffu, at.y, o);
          at.z += __shfl_xor_sync(0xffffffffu, at.z, o);
          at.w += __shfl_xor_sync(0xffffffffu, at.w, o);
        }
      }
      if (want_sq) {
        if (!even) sq = 0.0;
        sq += __shfl_xor_sync(0xffffffffu, sq, 2);
        sq += __shfl_xor_sync(0xffffffffu, sq, 4);
      }
      if (pc.w >= 0) {
        float* o = P.po + (size_t)pc.w * KP;
#pragma unroll
        for (int b = 0; b < NB; ++b) *reinterpret_cast<float4*>(o + b * 32 + q * 4) = am[b];
        if (KT > 0 && q < KT) *reinterpret_cast<float4*>(o + NB * 32 + q * 4) = at;
        if (want_sq && q == 0) P.psq[pc.w] = sq;
      }
      __syncwarp();
      pc = pcn;
      t_cur = t_nxt;
#pragma unroll
      for (int b = 0; b < NB; ++b) hm[b] = hmn[b];
      ht = htn;
    }
  }
  // the last CTA leaves the tickets zero for the next launch
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const int d = atomicAdd(A.counters + A.n_list, 1);
    if (d == (int)gridDim.x - 1) {
      for (int i = 0; i <= A.n_list; ++i) A.counters[i] = 0;
    }
  }
}

// ---- 4-lane groups (rows of one 32-dim block, k <= 40) --------------------
// The same walk with a row on 4 lanes (8 groups, i.e. 8 pieces, per warp and
// 32 entries per warp batch): a lane holds two 16-byte chunks of each of the 4
// rows of a batch, so the reduce-scatter / all-gather of the 4 dots costs 7
// shuffles per 32 entries instead of 8 per 16 -- shuffles share the shared-
// memory data pipe that bounds this kernel -- and the batch costs ~110
// instructions per 32 entries. Even groups read chunks [0,4) then [4,8) of
// their rows, odd groups the opposite halves, so the two rows of a quarter
// warp never share banks.
constexpr int kPT4 = 512;                 // 16 warps, <= 128 registers
constexpr int kRing4Stride = 2 * kBlockBytes + 16;   // per group; 52 words: the 8 groups' slots fall in distinct banks
constexpr int kRing4Bytes = (kPT4 / 32) * 8 * kRing4Stride;
constexpr int kPanel4Bytes = 200 * 1024;
static_assert(kPanel4Bytes + kRing4Bytes + 64 <= 232448, "k_panel4 shared memory");
constexpr int kPanel4Smem = kPanel4Bytes + kRing4Bytes;

template <int KT>
__global__ void __launch_bounds__(kPT4, 1) k_panel4(const PanelArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int KC = 8 + KT;
  constexpr int KP = KC * 4;
  float* s_main = reinterpret_cast<float*>(smem_raw);
  float* s_tail = s_main + (size_t)A.PR * 32;
  __shared__ int s_left;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int q = lane & 3, g = lane >> 2;
  const int cA = q + 4 * (g & 1), cB = q + 4 * ((g & 1) ^ 1);   // this lane's two main chunks
  const int e_mine = (q >> 1) + 2 * (q & 1);                    // the entry this lane finishes
  unsigned char* ring = smem_raw + kPanel4Bytes + (warp * 8 + g) * kRing4Stride;
  const unsigned a_mA = (unsigned)__cvta_generic_to_shared(s_main) + cA * 16;
  const unsigned a_mB = (unsigned)__cvta_generic_to_shared(s_main) + cB * 16;
  const unsigned a_tail = (unsigned)__cvta_generic_to_shared(s_tail) + (q & 1) * 16;
  const unsigned a_ring = (unsigned)__cvta_generic_to_shared(ring);
  const bool hi1 = (q & 2) != 0, odd = (q & 1) != 0;
  const bool gpar = (g & 1) != 0;       // odd groups load their tails in the opposite order
  const int gb = lane & 28;
  int cur_key = -1;
  int li = A.cta_start[blockIdx.x];
  for (int step = 0; step < A.n_list; ++step, li = li + 1 == A.n_list ? 0 : li + 1) {
    const int4 it = A.plist[li];        // {pass, panel, first piece, end piece}
    const int npc = it.w - it.z;
    __syncthreads();                    // everyone is done with the previous panel
    if (tid == 0) s_left = npc - *reinterpret_cast<volatile int*>(A.counters + li);
    __syncthreads();
    if (s_left <= 0) continue;          // this panel's pieces are all taken
    const PanelPass& P = A.p[it.x];
    const int key = it.x * 65536 + it.y;
    if (key != cur_key) {               // consecutive elements may share a panel (column chunks)
      cur_key = key;
      const int32_t* ids = P.panel_ids + (size_t)it.y * A.PR;
      const int total = A.PR * KC;
      for (int c = tid; c < total; c += kPT4) {
        const int r = c / KC, ch = c - r * KC;
        const int gid = ids[r];
        float* dst = ch < 8 ? s_main + (size_t)r * 32 + ch * 4
                            : s_tail + (size_t)r * KT * 4 + (ch - 8) * 4;
        if (gid >= 0) cp16(dst, P.gath + (size_t)gid * P.ldg + ch * 4);
        else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      cp_commit();
      cp_wait<0>();
    }
    __syncthreads();
    float* const rhot = P.rhot;
    const bool want_sq = P.psq != nullptr;
    auto take = [&]() {
      int v = 0;
      if (lane == 0) v = atomicAdd(A.counters + li, 8);
      return __shfl_sync(0xffffffffu, v, 0);
    };
    auto load_desc = [&](int t0) {
      int4 d = make_int4(0, 0, 0, -1);  // {self row, first block, length, slot}; slot < 0: none
      if (t0 + g < npc) d = P.pieces[it.z + t0 + g];
      return d;
    };
    auto load_self = [&](const int4& d, float4& xa, float4& xb, float4& xt) {
      const float* srow = P.self + (size_t)d.x * P.lds;
      xa = *reinterpret_cast<const float4*>(srow + cA * 4);
      xb = *reinterpret_cast<const float4*>(srow + cB * 4);
      if (KT > 0) xt = *reinterpret_cast<const float4*>(srow + 32 + (q & 1) * 4);
    };
    int t_cur = take();
    int4 pc = load_desc(t_cur);
    float4 hA, hB, ht = make_float4(0.f, 0.f, 0.f, 0.f);
    load_self(pc, hA, hB, ht);
    while (t_cur < npc) {
      const int t_nxt = take();
      const int4 pcn = load_desc(t_nxt);
      float4 hAn, hBn, htn = make_float4(0.f, 0.f, 0.f, 0.f);
      const int len = pc.z;
      const int lim = len - e_mine;     // batch b holds this lane's entry iff 4 b < lim
      float* rh = rhot + (size_t)pc.y * 16 + e_mine;
      float4 aA = make_float4(0.f, 0.f, 0.f, 0.f), aB = aA, at = aA;
      double sq = 0.0;
      const int nb = (len + 3) >> 2;
      const int nblk = (nb + 3) >> 2;
      int nbw = nb;
      nbw = max(nbw, __shfl_xor_sync(0xffffffffu, nbw, 4));
      nbw = max(nbw, __shfl_xor_sync(0xffffffffu, nbw, 8));
      nbw = max(nbw, __shfl_xor_sync(0xffffffffu, nbw, 16));
      const int nblkw = (nbw + 3) >> 2;
      const int4* rp = P.recs + (size_t)pc.y * 6;
      const int jmax = max(nblk - 1, 0);
      // the group's 4 lanes copy a 96-byte block as 6 chunks: lanes 0, 1 take two
      auto fetch = [&](int slot, int jb) {
        cp16(ring + slot * kBlockBytes + q * 16, rp + jb * 6 + q);
        if (q < 2) cp16(ring + slot * kBlockBytes + (q + 4) * 16, rp + jb * 6 + q + 4);
      };
      fetch(0, 0);
      cp_commit();
      for (int j = 0; j < nblkw; ++j) {
        fetch((j + 1) & 1, min(j + 1, jmax));   // clamped: short pieces re-read their last block
        cp_commit();
        cp_wait<1>();
        __syncwarp();
        if (j == 0) load_self(pcn, hAn, hBn, htn);
        const unsigned rs = a_ring + (j & 1) * kBlockBytes;
#pragma unroll 1
        for (int bb = 0; bb < 4; ++bb) {
          const int b = j * 4 + bb;
          if (b >= nbw) break;
          const uint2 lw = lds64(rs + bb * 8);
          const float a_mine = lds32(rs + 32 + (bb * 4 + e_mine) * 4);
          const unsigned l0 = lw.x & 0xffffu, l1 = lw.x >> 16, l2 = lw.y & 0xffffu, l3 = lw.y >> 16;
          const float4 mA0 = lds128(a_mA + l0 * 128), mB0 = lds128(a_mB + l0 * 128);
          const float4 mA1 = lds128(a_mA + l1 * 128), mB1 = lds128(a_mB + l1 * 128);
          const float4 mA2 = lds128(a_mA + l2 * 128), mB2 = lds128(a_mB + l2 * 128);
          const float4 mA3 = lds128(a_mA + l3 * 128), mB3 = lds128(a_mB + l3 * 128);
          // tail chunk q&1 of entries q>>1 (lo) and (q>>1) + 2 (hi). The layout
          // build orders a batch's entries by bank window (local row mod 4), so an
          // even group reading its lo pair while the odd group of the same quarter
          // warp reads its hi pair touches 4 different windows.
          float4 tA = make_float4(0.f, 0.f, 0.f, 0.f), tB = tA;
          if (KT > 0) {
            const unsigned llo = hi1 ? l1 : l0, lhi = hi1 ? l3 : l2;
            tA = lds128(a_tail + (gpar ? lhi : llo) * (KT * 16));
            tB = lds128(a_tail + (gpar ? llo : lhi) * (KT * 16));
          }
          const float p0 = dot4(mA0, hA) + dot4(mB0, hB);
          const float p1 = dot4(mA1, hA) + dot4(mB1, hB);
          const float p2 = dot4(mA2, hA) + dot4(mB2, hB);
          const float p3 = dot4(mA3, hA) + dot4(mB3, hB);
          // reduce-scatter over the 4 lanes: lanes with q&2 keep entries {1,3},
          // the others {0,2}; then q&1 picks the upper one (fixed tree)
          float klo = hi1 ? p1 : p0, khi = hi1 ? p3 : p2;
          const float slo = hi1 ? p0 : p1, shi = hi1 ? p2 : p3;
          klo += __shfl_xor_sync(0xffffffffu, slo, 2);
          khi += __shfl_xor_sync(0xffffffffu, shi, 2);
          if (KT > 0) {
            const float dA = dot4(tA, ht), dB = dot4(tB, ht);
            klo += gpar ? dB : dA;
            khi += gpar ? dA : dB;
          }
          float kk = odd ? khi : klo;
          const float ss = odd ? klo : khi;
          kk += __shfl_xor_sync(0xffffffffu, ss, 1);
          const bool valid = b * 4 < lim;
          const float r = valid ? kk - a_mine : 0.f;
          // entry e lives in lane (e & 1) * 2 + (e >> 1) of the group
          const float r0 = __shfl_sync(0xffffffffu, r, gb);
          const float r1 = __shfl_sync(0xffffffffu, r, gb + 2);
          const float r2 = __shfl_sync(0xffffffffu, r, gb + 1);
          const float r3 = __shfl_sync(0xffffffffu, r, gb + 3);
          axpy4(aA, r0, mA0); axpy4(aB, r0, mB0);
          axpy4(aA, r1, mA1); axpy4(aB, r1, mB1);
          axpy4(aA, r2, mA2); axpy4(aB, r2, mB2);
          axpy4(aA, r3, mA3); axpy4(aB, r3, mB3);
          if (KT > 0) {
            const float rlo = hi1 ? r1 : r0, rhi = hi1 ? r3 : r2;
            axpy4(at, gpar ? rhi : rlo, tA);
            axpy4(at, gpar ? rlo : rhi, tB);
          }
          if (rhot != nullptr && valid) rh[b * 4] = r;
          if (want_sq) sq = fma((double)r, (double)r, sq);
        }
        __syncwarp();
      }
      cp_wait<0>();
      if (nblkw == 0) load_self(pcn, hAn, hBn, htn);
      if (KT > 0) {   // lanes q and q ^ 2 hold the same tail chunk
        at.x += __shfl_xor_sync(0xffffffffu, at.x, 2);
        at.y += __shfl_xor_sync(0xffffffffu, at.y, 2);
        at.z += __shfl_xor_sync(0xffffffffu, at.z, 2);
        at.w += __shfl_xor_sync(0xffffffffu, at.w, 2);
      }
      if (want_sq) {
        sq += __shfl_xor_sync(0xffffffffu, sq, 1);
        sq += __shfl_xor_sync(0xffffffffu, sq, 2);
      }
      if (pc.w >= 0) {
        float* o = P.po + (size_t)pc.w * KP;
        *reinterpret_cast<float4*>(o + cA * 4) = aA;
        *reinterpret_cast<float4*>(o + cB * 4) = aB;
        if (KT > 0 && q < KT) *reinterpret_cast<float4*>(o + 32 + q * 4) = at;
        if (want_sq && q == 0) P.psq[pc.w] = sq;
      }
      __syncwarp();
      pc = pcn;
      t_cur = t_nxt;
      hA = hAn; hB = hBn; ht = htn;
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const int d = atomicAdd(A.counters + A.n_list, 1);
    if (d == (int)gridDim.x - 1) {
      for (int i = 0; i <= A.n_list; ++i) A.counters[i] = 0;
    }
  }
}

// ---- cold entries: the same piece walk on global loads --------------------
// Entries whose gathered row is not panelled, or whose piece is too short, are
// cut into pieces per self row as well (a self row's cold entries in their
// original order, at most Lmax each) and walked by 4-lane groups with the
// batch loop of k_panel4 -- the rows come through L2 / L1 (`ld.global.nc`)
// instead of shared memory, 10 LDG.128 per lane and batch in flight. Record
// blocks hold global row ids: 16 x u32, then 16 x f32 (128 B). Warps take
// rounds of 8 pieces from one ticket per pass; there is no CTA-wide step.
constexpr int kCT = 512;
constexpr int kColdBlock = 128;
constexpr int kColdRingStride = 2 * kColdBlock + 16;   // 68 words: 8 groups on distinct banks
constexpr int kColdSmem = (kCT / 32) * 8 * kColdRingStride;

struct ColdArgs {
  PanelPass p[2];
  float* out[2];            // RH / RtW: rows whose only slot is a cold piece are written here
  float scale;
  int npieces[2];
  int* counters;            // [2] piece tickets, [1] finished CTAs (zero at rest)
};

__device__ __forceinline__ float4 ldg128(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}

template <int KT>
__global__ void __launch_bounds__(kCT, 1) k_cold4(const ColdArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int KP = (8 + KT) * 4;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int q = lane & 3, g = lane >> 2;
  const int cA = q, cB = q + 4;         // this lane's two main chunks
  const int e_mine = (q >> 1) + 2 * (q & 1);
  unsigned char* ring = smem_raw + (warp * 8 + g) * kColdRingStride;
  const unsigned a_ring = (unsigned)__cvta_generic_to_shared(ring);
  const bool hi1 = (q & 2) != 0, odd = (q & 1) != 0;
  const int gb = lane & 28;
  for (int pass = 0; pass < 2; ++pass) {
    const PanelPass& P = A.p[pass];
    const int npc = A.npieces[pass];
    if (npc <= 0) continue;
    float* const rhot = P.rhot;
    const bool want_sq = P.psq != nullptr;
    const float* const gath = P.gath;
    const int ldg = P.ldg;
    auto take = [&]() {
      int v = 0;
      if (lane == 0) v = atomicAdd(A.counters + pass, 8);
      return __shfl_sync(0xffffffffu, v, 0);
    };
    auto load_desc = [&](int t0) {
      int4 d = make_int4(0, 0, 0, -1);  // {self row, first block, length, slot}; slot < 0: none
      if (t0 + g < npc) d = P.pieces[t0 + g];
      return d;
    };
    auto load_self = [&](const int4& d, float4& xa, float4& xb, float4& xt) {
      const float* srow = P.self + (size_t)d.x * P.lds;
      xa = *reinterpret_cast<const float4*>(srow + cA * 4);
      xb = *reinterpret_cast<const float4*>(srow + cB * 4);
      if (KT > 0) xt = *reinterpret_cast<const float4*>(srow + 32 + (q & 1) * 4);
    };
    int t_cur = take();
    int4 pc = load_desc(t_cur);
    float4 hA, hB, ht = make_float4(0.f, 0.f, 0.f, 0.f);
    load_self(pc, hA, hB, ht);
    while (t_cur < npc) {
      const int t_nxt = take();
      const int4 pcn = load_desc(t_nxt);
      float4 hAn, hBn, htn = make_float4(0.f, 0.f, 0.f, 0.f);
      const int len = pc.z & 0x3fffffff;
      const bool direct = (pc.z >> 30) != 0;   // the row's only slot: write the output row itself
      const int lim = len - e_mine;
      float* rh = rhot + (size_t)pc.y * 16 + e_mine;
      float4 aA = make_float4(0.f, 0.f, 0.f, 0.f), aB = aA, at = aA;
      double sq = 0.0;
      const int nb = (len + 3) >> 2;
      const int nblk = (nb + 3) >> 2;
      int nbw = nb;
      nbw = max(nbw, __shfl_xor_sync(0xffffffffu, nbw, 4));
      nbw = max(nbw, __shfl_xor_sync(0xffffffffu, nbw, 8));
      nbw = max(nbw, __shfl_xor_sync(0xffffffffu, nbw, 16));
      const int nblkw = (nbw + 3) >> 2;
      const int4* rp = P.recs + (size_t)pc.y * 8;
      const int jmax = max(nblk - 1, 0);
      auto fetch = [&](int slot, int jb) {   // 8 chunks of a 128-byte block on 4 lanes
        cp16(ring + slot * kColdBlock + q * 16, rp + jb * 8 + q);
        cp16(ring + slot * kColdBlock + (q + 4) * 16, rp + jb * 8 + q + 4);
      };
      fetch(0, 0);
      cp_commit();
      for (int j = 0; j < nblkw; ++j) {
        fetch((j + 1) & 1, min(j + 1, jmax));
        cp_commit();
        cp_wait<1>();
        __syncwarp();
        if (j == 0) load_self(pcn, hAn, hBn, htn);
        const unsigned rs = a_ring + (j & 1) * kColdBlock;
#pragma unroll 1
        for (int bb = 0; bb < 4; ++bb) {
          const int b = j * 4 + bb;
          if (b >= nbw) break;
          uint4 iw;
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(iw.x), "=r"(iw.y), "=r"(iw.z), "=r"(iw.w) : "r"(rs + bb * 16));
          const float a_mine = lds32(rs + 64 + (bb * 4 + e_mine) * 4);
          const float* g0 = gath + (size_t)iw.x * ldg;
          const float* g1 = gath + (size_t)iw.y * ldg;
          const float* g2 = gath + (size_t)iw.z * ldg;
          const float* g3 = gath + (size_t)iw.w * ldg;
          const float4 mA0 = ldg128(g0 + cA * 4), mB0 = ldg128(g0 + cB * 4);
          const float4 mA1 = ldg128(g1 + cA * 4), mB1 = ldg128(g1 + cB * 4);
          const float4 mA2 = ldg128(g2 + cA * 4), mB2 = ldg128(g2 + cB * 4);
          const float4 mA3 = ldg128(g3 + cA * 4), mB3 = ldg128(g3 + cB * 4);
          float4 tA = make_float4(0.f, 0.f, 0.f, 0.f), tB = tA;
          if (KT > 0) {
            tA = ldg128((hi1 ? g1 : g0) + 32 + (q & 1) * 4);
            tB = ldg128((hi1 ? g3 : g2) + 32 + (q & 1) * 4);
          }
          const float p0 = dot4(mA0, hA) + dot4(mB0, hB);
          const float p1 = dot4(mA1, hA) + dot4(mB1, hB);
          const float p2 = dot4(mA2, hA) + dot4(mB2, hB);
          const float p3 = dot4(mA3, hA) + dot4(mB3, hB);
          float klo = hi1 ? p1 : p0, khi = hi1 ? p3 : p2;
          const float slo = hi1 ? p0 : p1, shi = hi1 ? p2 : p3;
          klo += __shfl_xor_sync(0xffffffffu, slo, 2);
          khi += __shfl_xor_sync(0xffffffffu, shi, 2);
          if (KT > 0) {
            klo += dot4(tA, ht);
            khi += dot4(tB, ht);
          }
          float kk = odd ? khi : klo;
          const float ss = odd ? klo : khi;
          kk += __shfl_xor_sync(0xffffffffu, ss, 1);
          const bool valid = b * 4 < lim;
          const float r = valid ? kk - a_mine : 0.f;
          const float r0 = __shfl_sync(0xffffffffu, r, gb);
          const float r1 = __shfl_sync(0xffffffffu, r, gb + 2);
          const float r2 = __shfl_sync(0xffffffffu, r, gb + 1);
          const float r3 = __shfl_sync(0xffffffffu, r, gb + 3);
          axpy4(aA, r0, mA0); axpy4(aB, r0, mB0);
          axpy4(aA, r1, mA1); axpy4(aB, r1, mB1);
          axpy4(aA, r2, mA2); axpy4(aB, r2, mB2);
          axpy4(aA, r3, mA3); axpy4(aB, r3, mB3);
          if (KT > 0) {
            axpy4(at, hi1 ? r1 : r0, tA);
            axpy4(at, hi1 ? r3 : r2, tB);
          }
          if (rhot != nullptr && valid) rh[b * 4] = r;
          if (want_sq) sq = fma((double)r, (double)r, sq);
        }
        __syncwarp();
      }
      cp_wait<0>();
      if (nblkw == 0) load_self(pcn, hAn, hBn, htn);
      if (KT > 0) {
        at.x += __shfl_xor_sync(0xffffffffu, at.x, 2);
        at.y += __shfl_xor_sync(0xffffffffu, at.y, 2);
        at.z += __shfl_xor_sync(0xffffffffu, at.z, 2);
        at.w += __shfl_xor_sync(0xffffffffu, at.w, 2);
      }
      if (want_sq) {
        sq += __shfl_xor_sync(0xffffffffu, sq, 1);
        sq += __shfl_xor_sync(0xffffffffu, sq, 2);
      }
      if (pc.w >= 0) {
        float* o = P.po + (size_t)pc.w * KP;
        if (direct) {
          o = A.out[pass] + (size_t)pc.x * KP;
          const float sc = A.scale;
          aA.x *= sc; aA.y *= sc; aA.z *= sc; aA.w *= sc;
          aB.x *= sc; aB.y *= sc; aB.z *= sc; aB.w *= sc;
          at.x *= sc; at.y *= sc; at.z *= sc; at.w *= sc;
        }
        *reinterpret_cast<float4*>(o + cA * 4) = aA;
        *reinterpret_cast<float4*>(o + cB * 4) = aB;
        if (KT > 0 && q < KT) *reinterpret_cast<float4*>(o + 32 + q * 4) = at;
        if (want_sq && q == 0) P.psq[pc.w] = sq;
      }
      __syncwarp();
      pc = pcn;
      t_cur = t_nxt;
      hA = hAn; hB = hBn; ht = htn;
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const int d = atomicAdd(A.counters + 2, 1);
    if (d == (int)gridDim.x - 1) {
      A.counters[0] = 0;
      A.counters[1] = 0;
      A.counters[2] = 0;
    }
  }
}

// out[row] += scale * sum of the row's piece outputs, in slot order (assign:
// out[row] = ..., when every entry of the row is in a piece).
// Threads are (sub-range, row, 16-byte chunk): a block takes 256 / (KC * S)
// self rows, each row's slots cut into S contiguous sub-ranges whose partial
// sums are added in sub-range order (a fixed tree). Light rows (few slots)
// run with S = 1 (no shared memory, no barrier), heavy rows with one row per
// block, so a row with thousands of slots does not serialise on one thread.
__global__ void __launch_bounds__(256)
k_panel_fold(int n_rows, int n_row_blocks, int S, const int32_t* __restrict__ frows,
             const int32_t* __restrict__ fbeg, const int32_t* __restrict__ fcnt,
             const float* __restrict__ po, int KC, int k, float* __restrict__ out, int ldout,
             float scale, int assign) {
  __shared__ float4 s_part[256];
  {
    const int rpb = 256 / (KC * S);
    const int cpb = rpb * KC;
    const int sub = threadIdx.x / cpb, c = threadIdx.x - sub * cpb;
    const int rr = c / KC, ch = c - rr * KC;
    const int f = blockIdx.x * rpb + rr;
    const bool on = sub < S && f < n_rows;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (on) {
      const int s0 = fbeg[f], n = fcnt[f];
      const int per = (n + S - 1) / S;
      const int a = s0 + min(sub * per, n), b = s0 + min((sub + 1) * per, n);
      const float4* src = reinterpret_cast<const float4*>(po) + ch;
      int s = a;
      for (; s + 8 <= b; s += 8) {
        float4 t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) t[u] = __ldcs(src + (size_t)(s + u) * KC);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          acc.x += t[u].x; acc.y += t[u].y; acc.z += t[u].z; acc.w += t[u].w;
        }
      }
      if (s < b) {
        float4 t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          t[u] = s + u < b ? __ldcs(src + (size_t)(s + u) * KC) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (s + u < b) { acc.x += t[u].x; acc.y += t[u].y; acc.z += t[u].z; acc.w += t[u].w; }
        }
      }
    }
    if (S > 1) {
      s_part[threadIdx.x] = acc;
      __syncthreads();
      if (on && sub == 0) {
        for (int u = 1; u < S; ++u) {
          const float4 p = s_part[u * cpb + c];
          acc.x += p.x; acc.y += p.y; acc.z += p.z; acc.w += p.w;
        }
      }
    }
    if (on && sub == 0) {
      const float tot[4] = {acc.x, acc.y, acc.z, acc.w};
      float* o = out + (size_t)frows[f] * ldout + ch * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (ch * 4 + e < k) o[e] = assign ? scale * tot[e] : o[e] + scale * tot[e];
    }
  }
}

// sums[0] += sum of the per-slot r^2: 64 blocks over fixed contiguous chunks
// (fixed tree inside a block), the last-arriving block adds the 64 block sums
// in block order -- bitwise reproducible. ws: [64 doubles | arrival counter].
constexpr int kSqBlocks = 64;
__global__ void __launch_bounds__(256)
k_panel_sq(int n, const double* __restrict__ psq, double* __restrict__ bp, unsigned int* counter,
           double* sums) {
  __shared__ double s_red[8];
  __shared__ bool last;
  const int per = (n + kSqBlocks - 1) / kSqBlocks;
  const int a = min((int)blockIdx.x * per, n), b = min(a + per, n);
  double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
  int i = a + threadIdx.x;
  for (; i + 768 < b; i += 1024) {
    v0 += psq[i]; v1 += psq[i + 256]; v2 += psq[i + 512]; v3 += psq[i + 768];
  }
  for (; i < b; i += 256) v0 += psq[i];
  const double s = block_sum<256>((v0 + v1) + (v2 + v3), s_red);
  if (threadIdx.x == 0) {
    bp[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    const volatile double* vb = bp;
    double t = 0.0;
    for (int j = 0; j < kSqBlocks; ++j) t += vb[j];
    sums[0] += t;
    *counter = 0u;
  }
}

template <int NB, int KT>
int launch_panel(const PanelArgs& A, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    MFG_CUDA_CHECK(cudaFuncSetAttribute(k_panel<NB, KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        kPanelSmem));
    configured = true;
  }
  k_panel<NB, KT><<<kNumSMs, kPT, kPanelSmem, stream>>>(A);
  MFG_LAUNCH_CHECK();
  return MFG_OK;
}

template <int KT>
int launch_panel4(const PanelArgs& A, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    MFG_CUDA_CHECK(cudaFuncSetAttribute(k_panel4<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        kPanel4Smem));
    configured = true;
  }
  k_panel4<KT><<<kNumSMs, kPT4, kPanel4Smem, stream>>>(A);
  MFG_LAUNCH_CHECK();
  return MFG_OK;
}

bool panel_shape(int ld, int* nb, int* kt) {
  if (ld == 40) { *nb = 1; *kt = 2; return true; }
  if (ld == 32) { *nb = 1; *kt = 0; return true; }
  if (ld == 64) { *nb = 2; *kt = 0; return true; }
  return false;
}

}  // namespace
}  // namespace mfg

using namespace mfg;

extern "C" int mfg_panel_rows(int ld) {
  int nb, kt;
  if (!panel_shape(ld, &nb, &kt)) return 0;
  // rows of one 32-dim block run on 4-lane groups (k_panel4), k = 64 on 8-lane groups
  return ((nb == 1 ? kPanel4Bytes : kPanelBytes) / ((nb * 8 + kt) * 16)) & ~1;
}

extern "C" int mfg_panel_sweep(int ld, int n_list, const int32_t* plist, const int32_t* cta_start,
                               const mfg_panel_pass* csr, const mfg_panel_pass* csc,
                               const void* W, const void* H, int32_t* counters, void* stream) {
  int nb, kt;
  MFG_REQUIRE(panel_shape(ld, &nb, &kt), "panel sweep: unsupported factor row width");
  MFG_REQUIRE(csr && csc && plist && cta_start && counters, "panel sweep: null argument");
  if (n_list <= 0) return MFG_OK;
  PanelArgs A;
  const mfg_panel_pass* pp[2] = {csr, csc};
  for (int i = 0; i < 2; ++i) {
    PanelPass& P = A.p[i];
    P.self = (const float*)(i == 0 ? W : H);
    P.gath = (const float*)(i == 0 ? H : W);
    P.panel_ids = pp[i]->panel_ids;
    P.pieces = (const int4*)pp[i]->pieces;
    P.recs = (const int4*)pp[i]->recs;
    P.rhot = (float*)pp[i]->r_hot;
    P.po = (float*)pp[i]->piece_out;
    P.psq = (double*)pp[i]->piece_sq;
    P.lds = ld;
    P.ldg = ld;
  }
  A.plist = (const int4*)plist;
  A.cta_start = cta_start;
  A.n_list = n_list;
  A.PR = mfg_panel_rows(ld);
  A.counters = counters;
  cudaStream_t s = (cudaStream_t)stream;
  if (getenv("MFG_PANEL_GL8")) {   // A/B: the 8-lane-group kernel for every width
    if (nb == 1 && kt == 2) return launch_panel<1, 2>(A, s);
    if (nb == 1 && kt == 0) return launch_panel<1, 0>(A, s);
  }
  if (nb == 1 && kt == 2) return launch_panel4<2>(A, s);
  if (nb == 1 && kt == 0) return launch_panel4<0>(A, s);
  return launch_panel<2, 0>(A, s);
}

extern "C" int mfg_panel_ctas(void) { return kNumSMs; }

extern "C" int mfg_panel_fold(int ld, int k, const mfg_panel_pass* pass, void* out, int ldout,
                              double out_scale, int assign, double* sums, void* sq_ws,
                              void* stream) {
  int nb, kt;
  MFG_REQUIRE(panel_shape(ld, &nb, &kt), "panel fold: unsupported factor row width");
  MFG_REQUIRE(pass && out, "panel fold: null argument");
  if (pass->n_frows <= 0) return MFG_OK;
  const int KC = nb * 8 + kt;
  cudaStream_t st = (cudaStream_t)stream;
  const int nl = pass->n_light, nh = pass->n_frows - pass->n_light;
  MFG_REQUIRE(nl >= 0 && nh >= 0, "panel fold: bad light/heavy split");
  if (nl > 0) {
    const int rpb = 256 / KC;
    const int nrb = (nl + rpb - 1) / rpb;
    k_panel_fold<<<nrb, 256, 0, st>>>(nl, nrb, 1, pass->frows, pass->fbeg, pass->fcnt,
                                      (const float*)pass->piece_out, KC, k, (float*)out, ldout,
                                      (float)out_scale, assign);
    MFG_LAUNCH_CHECK();
  }
  if (nh > 0) {
    const int S = 256 / KC;   // one row per block
    k_panel_fold<<<nh, 256, 0, st>>>(nh, nh, S, pass->frows + nl, pass->fbeg + nl,
                                     pass->fcnt + nl, (const float*)pass->piece_out, KC, k,
                                     (float*)out, ldout, (float)out_scale, assign);
    MFG_LAUNCH_CHECK();
  }
  if (pass->piece_sq != nullptr && sums != nullptr) {
    MFG_REQUIRE(sq_ws != nullptr, "panel fold: sum r^2 needs its workspace");
    double* bp = (double*)sq_ws;
    k_panel_sq<<<kSqBlocks, 256, 0, st>>>(pass->n_pieces, (const double*)pass->piece_sq, bp,
                                          (unsigned int*)(bp + kSqBlocks), sums);
    MFG_LAUNCH_CHECK();
  }
  return MFG_OK;
}

/* The cold pieces of both passes on global loads (k_cold4). The passes'
 * structs carry the cold piece table, the cold record blocks (16 x u32 row
 * ids, 16 x f32 values), the residual buffer in record order, and the same
 * piece_out / piece_sq arrays as the panel passes (slots are shared).      */
extern "C" int mfg_cold_sweep(int ld, const mfg_panel_pass* csr, const mfg_panel_pass* csc,
                              const void* W, const void* H, void* RH, void* RtW, double out_scale,
                              int32_t* counters, void* stream) {
  int nb, kt;
  MFG_REQUIRE(panel_shape(ld, &nb, &kt) && nb == 1, "cold sweep: unsupported factor row width");
  MFG_REQUIRE(csr && csc && counters, "cold sweep: null argument");
  if (csr->n_pieces <= 0 && csc->n_pieces <= 0) return MFG_OK;
  ColdArgs A;
  const mfg_panel_pass* pp[2] = {csr, csc};
  for (int i = 0; i < 2; ++i) {
    PanelPass& P = A.p[i];
    P.self = (const float*)(i == 0 ? W : H);
    P.gath = (const float*)(i == 0 ? H : W);
    P.panel_ids = nullptr;
    P.pieces = (const int4*)pp[i]->pieces;
    P.recs = (const int4*)pp[i]->recs;
    P.rhot = (float*)pp[i]->r_hot;
    P.po = (float*)pp[i]->piece_out;
    P.psq = (double*)pp[i]->piece_sq;
    P.lds = ld;
    P.ldg = ld;
    A.npieces[i] = pp[i]->n_pieces;
  }
  A.out[0] = (float*)RH;
  A.out[1] = (float*)RtW;
  A.scale = (float)out_scale;
  A.counters = counters;
  cudaStream_t s = (cudaStream_t)stream;
  if (kt == 2) k_cold4<2><<<kNumSMs, kCT, kColdSmem, s>>>(A);
  else k_cold4<0><<<kNumSMs, kCT, kColdSmem, s>>>(A);
  MFG_LAUNCH_CHECK();
  return MFG_OK;
}
