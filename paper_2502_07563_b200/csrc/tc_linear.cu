// tcgen05 / TMEM / TMA kernels for the LASP-2 linear-attention path (bf16 in,
// fp32 accumulate), sm_100a only.
//
// All operand tiles are 128 tokens x 128 features of bf16, loaded by TMA as two
// 64-column SWIZZLE_128B boxes (16 KB each). The same smem image serves as a
// K-major operand when the contraction runs over features (Q K^T, Q S) and as
// an MN-major operand when it runs over tokens (K^T V, P V), so no tile is ever
// transposed in software. dim < 128 (e.g. cfg1's d=64) is handled by TMA
// zero-fill of the out-of-range feature columns.
//
// Kernels
//   tc_segment_states : M_seg = X_seg^T Y_seg          (lasp2.py:130-147, per segment)
//   tc_causal_chunk   : O = mask(Q K^T) V + Q S_j,  S_{j+1} = S_j + K_j^T V_j
//                       (oracle.py:50-62 blocked; lasp2.py:219-243 inter term
//                       folded in through the initial state)
//   tc_apply_state    : O (+)= X M or X M^T            (lasp2.py:150-165)
#include <cuda.h>

#include "kernels.h"
#include "tc_common.cuh"

namespace lasp {
namespace tc {


constexpr int kSegStages = 3;
constexpr uint32_t kSegSmem = kSegStages * 2 * kTileBytes + 1024 + 256;

__global__ void __launch_bounds__(192, 1)
    tc_segment_states_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_y,
                             float* __restrict__ out, int64_t tokens, int dim, int nseg) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSegStages * 2 * kTileBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kSegStages;
  uint64_t* acc_full = bars + 2 * kSegStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kSegStages + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seg = blockIdx.x;
  const int slot = blockIdx.y;
  int64_t lo, hi;
  seg_range(seg, nseg, tokens, &lo, &hi);
  const int nblk = (int)((hi - lo + kTile - 1) / kTile);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSegStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<128>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    if (elect_one()) {
      prefetch_tmap(&tm_x);
      prefetch_tmap(&tm_y);
      for (int b = 0; b < nblk; ++b) {
        const int s = b % kSegStages, u = b / kSegStages;
        if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
        uint8_t* xs = ring + s * 2 * kTileBytes;
        uint8_t* ys = xs + kTileBytes;
        const int nbox = dim > 64 ? 2 : 1;
        mbar_arrive_expect_tx(&full[s], 2 * nbox * kBoxBytes);
        const int row = (int)(lo + (int64_t)b * kTile);
        for (int bx = 0; bx < nbox; ++bx) {
          tma_load_3d(xs + bx * kBoxBytes, &tm_x, &full[s], 64 * bx, row, slot);
          tma_load_3d(ys + bx * kBoxBytes, &tm_y, &full[s], 64 * bx, row, slot);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16_f32(128, 128, 1, 1);
    for (int b = 0; b < nblk; ++b) {
      const int s = b % kSegStages, u = b / kSegStages;
      mbar_wait(&full[s], u & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t xs = smem_u32(ring + s * 2 * kTileBytes), ys = xs + kTileBytes;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_bf16_ss(tmem, desc_mnmajor(xs, kk), desc_mnmajor(ys, kk), idesc, (b > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&empty[s]);
        if (b == nblk - 1) mma_commit(acc_full);
      }
      __syncwarp();
    }
  } else {
    const int qd = warp & 3;
    const uint32_t row = qd * 32 + lane;
    mbar_wait(acc_full, 0);
    tc_fence_after();
    float* ob = out + ((int64_t)slot * nseg + seg) * (int64_t)dim * dim;
#pragma unroll 1
    for (int c0 = 0; c0 < 128; c0 += 32) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem + ((qd * 32) << 16) + c0, r);
      tmem_ld_wait();
      if ((int)row < dim) {
        float* orow = ob + (int64_t)row * dim + c0;
        if (c0 + 32 <= dim && (dim & 3) == 0) {  // 16-byte stores: 8 per 32 columns instead of 32
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(orow + i) = make_float4(__uint_as_float(r[i]), __uint_as_float(r[i + 1]),
                                                               __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c0 + i < dim) orow[i] = __uint_as_float(r[i]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<128>(tmem);
}

// ============================================================================
// Causal chunk kernel family (tcgen05, one 128-token block per step)
// ============================================================================
constexpr int kRing = 5;  // tile slots for the q'/k'/v' stream
constexpr uint32_t kCausalSmem = (kRing + 2) * kTileBytes + 1024 + 256;

struct CausalArgs {
  const float* seg_states;  // [slots][nseg][dim][dim] exclusive segment states (or null)
  const float* base;        // [slots][dim][dim] rank-level state (or null)
  // backward-triple only: forward states for the dQ role (run in reverse by subtraction)
  const float* fwd_seg;     // [slots][nseg][dim][dim] exclusive prefixes of K^T V
  const float* fwd_total;   // [slots][dim][dim] chunk total of K^T V
  const float* fwd_base;    // [slots][dim][dim] M_{1:t-1} (or null)
  float* g_out;             // kMode 3: [slots][nseg][dim][dim] segment states X^T q' (unscanned)
  int64_t tokens;
  int dim;
  int nseg;
  int reverse;
  int transpose_state;
  // fused peer-exchange consumer (kModes 0 / 1): the rank-level base is folded in the
  // prologue from this epoch's receive half [T][slots][dim][dim] once flags[xlo, xhi)
  // carry xepoch (ascending for a prefix, descending when xdesc); replaces `base`
  const float* xrecv = nullptr;
  const unsigned long long* xflags = nullptr;
  int xlo = 0, xhi = 0, xdesc = 0;
  unsigned long long xepoch = 0;
  const unsigned long long* xepoch_dev = nullptr;  // device epoch: recv half (e & 1) * xhalf, flags >= e
  int64_t xhalf = 0;
  float* base_out = nullptr;  // the folded base of each slot (written by its segment-0 CTA), or null
  const float* seg_total = nullptr;  // kMode 4: [slots][dim][dim] chunk total of the (suffix-scanned) seg_states
};

__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

struct TileMaps {
  CUtensorMap m[7];
};

// The dK/dV pair (kMode 1) prefetches the multicast tile of block j + 1 into L2 while it loads block j:
// its 5-slot ring holds only ~1.7 blocks and the MMA warp waited for tiles (cfg3: 2.31 -> 2.14 ms with
// every tile prefetched, 1.4 % better again without the private tile; distance 2 was worse). The
// HBM-bound kModes 0 / 3 got slower with any distance (1: +5 / +10 %), so they do not prefetch. The
// opt-in single-launch backward (kMode 2, chain-bound like the pair) gains too (4.00 -> 3.89 ms).
#ifndef LASP2_L2PF
#define LASP2_L2PF 1
#endif
#ifndef LASP2_L2PF_TRIPLE
#define LASP2_L2PF_TRIPLE 1
#endif
template <int kMode>
constexpr int kL2Prefetch = kMode == 1 ? LASP2_L2PF : (kMode == 2 || kMode == 4) ? LASP2_L2PF_TRIPLE : 0;

#ifdef LASP2_MMA_PROBE  // diagnostic: the MMA warp ignores the epilogue (TMA + MMA only; garbage results)
constexpr bool kMmaProbe = true;
#else
constexpr bool kMmaProbe = false;
#endif

constexpr int kCausalThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue

// Per-CTA role: which maps feed q', k', v' and receive the output, how the
// running state is seeded and updated, and which causal mask P gets.
struct Role {
  int qi, ki, vi, oi;   // indices into TileMaps
  int reverse;          // block order (1: last block first)
  int transpose;        // seed the state transposed
  int subtract;         // state -= k'^T v' before the block (dQ run in reverse)
  int mask;             // 1 keep col <= row, 2 keep col >= row, 3 keep col < row
  int mcast;            // kMode 1: which ring position (1 or 2) this CTA multicasts
  int neg;              // kMode 4 dK / dV: TMEM holds minus the state, the output is drained negated
};

// kMode 0: causal_chunk(q, k, v) -> o; maps [q, k, v, o].
// kMode 1: 2-CTA cluster per segment, masked backward dK (rank 0) and dV (rank 1);
//          maps [V, K, dO, Q, dK, dV]; dO and Q TMA-multicast to both CTAs and ring
//          slots released by multicast tcgen05.commit (empty barriers count 2).
// kMode 2: three CTAs per segment (blockIdx.x = 3*seg + role): dK, dV and dQ of the
//          masked backward; maps [Q, K, V, dO, dQ, dK, dV]. The three CTAs stream
//          the same four tiles in the same (reverse) order at the same time, so L2
//          serves the re-reads: HBM sees Q, K, V, dO once. dQ is the causal
//          forward form run backwards: TMEM holds T = -S, seeded with minus the
//          segment-END state; each block adds K^T V (so T becomes minus the
//          block-start state) and the state image is written as -T.
// kMode 4: kMode 2's three roles with every role walking its segment forwards, so the
//          three stream the same tiles in the same order with no subtract-form chain.
//          dK / dV use the suffix INCLUSIVE of the current block, G_{>=j} = G_{>j} + Q_j^T dO_j:
//          dK_j = V_j G_{>=j}^T - strict(V_j dO_j^T) Q_j and dV_j = K_j G_{>=j} - strict(K_j Q_j^T) dO_j
//          (strict: keep col < row), so with T = -G in TMEM (seeded with -(R + G_{>=seg}), then
//          T += k'^T v' per block like the forward form) the output is minus the forward-form chain
//          with mask 3, drained negated. Seeds: dQ fwd_base + fwd_seg[seg]; dK / dV base +
//          (seg > 0 ? seg_states[seg - 1] : seg_total), seg_states the exclusive suffix scan.
// kMode 3: kMode 0 plus one more tile per block, X (maps[4]), and the segment
//          state G = X^T q' accumulated in TMEM [384,512) (O single-buffered):
//          the masked backward's dQ pass (q' = dO, k' = V, v' = K) also yields
//          the dM segment states (X = Q), so Q^T dO needs no pass of its own.
template <int kMode>
__device__ __forceinline__ Role causal_role(uint32_t role, const CausalArgs& a) {
  if (kMode == 0 || kMode == 3) return Role{0, 1, 2, 3, a.reverse, a.transpose_state, 0, a.reverse ? 2 : 1, 0, 0};
  if (kMode == 1)
    // ring positions are shared by both CTAs: 0 private (V | K), 1 = dO, 2 = Q; rank 1 swaps k'/v' at the MMA
    return role == 0 ? Role{0, 2, 3, 4, 1, 1, 0, 2, 1, 0} : Role{1, 2, 3, 5, 1, 0, 0, 2, 2, 0};
  if (kMode == 4) {  // every role walks its segment forwards (see the kMode 4 note above)
    if (role == 0) return Role{2, 3, 0, 5, 0, 1, 0, 3, 0, 1};  // dK = V G_{>=j}^T - strict(V dO^T) Q
    if (role == 1) return Role{1, 0, 3, 6, 0, 0, 0, 3, 0, 1};  // dV = K G_{>=j} - strict(K Q^T) dO
    return Role{3, 2, 1, 4, 0, 1, 0, 1, 0, 0};                 // dQ = causal(dO, V, K; S^T)
  }
  if (role == 0) return Role{2, 3, 0, 5, 1, 1, 0, 2, 0, 0};  // dK = anti-causal(V, dO, Q; G^T)
  if (role == 1) return Role{1, 0, 3, 6, 1, 0, 0, 2, 0, 0};  // dV = anti-causal(K, Q, dO; G)
  return Role{3, 2, 1, 4, 1, 1, 1, 1, 0, 0};                 // dQ = causal(dO, V, K; S^T), reversed
}

template <int kMode>
__global__ void __launch_bounds__(kCausalThreads, 1)
    tc_causal_chunk_kernel(const __grid_constant__ TileMaps tm, CausalArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;                                // kRing x 32 KB
  uint8_t* pimg = smem + kRing * kTileBytes;           // P tile / O staging
  uint8_t* simg = pimg + kTileBytes;                   // bf16 state image
  uint64_t* bars = reinterpret_cast<uint64_t*>(simg + kTileBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kRing;
  uint64_t* s_full = bars + 2 * kRing + 0;
  uint64_t* st_full = bars + 2 * kRing + 1;
  uint64_t* p_ready = bars + 2 * kRing + 2;
  uint64_t* sst_ready = bars + 2 * kRing + 3;
  uint64_t* o_full = bars + 2 * kRing + 4;   // [2]
  uint64_t* o_empty = bars + 2 * kRing + 6;  // [2]
  uint64_t* g_full = bars + 2 * kRing + 8;   // kMode 3
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kRing + 9);
  constexpr int kTPB = kMode == 3 ? 4 : 3;   // ring tiles per block: q', k', v' (+ X)
  // kMode 1: P goes back to TMEM as bf16 over the S columns it came from (each column half packs into
  // the first half of its own columns: [0,32) and [64,96)) and feeds a TS-mode P.v' MMA; the next
  // block's S MMA is issued after that P.v' MMA, and tcgen05 MMAs execute in issue order.
  constexpr bool kPT = kMode == 1 || kMode == 4;
  constexpr bool kOneO = kMode == 3;  // TMEM [384,512) holds G (kMode 3), else the second O buffer

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifndef LASP2_TRACE
  unsigned long long t_begin = 0;  // per-CTA globaltimer span when the debug buffer is set (tools/cta_span_probe.py)
  if (g_trace != nullptr && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
#endif
#ifdef LASP2_SPAN  // A/B diagnostic build: 8 globaltimer stamps per CTA (tools/cta_phase_probe.py)
  auto span = [&](int i) {
    if (g_trace != nullptr) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      g_trace[16 * (blockIdx.y * gridDim.x + blockIdx.x) + i] = t;
    }
  };
  if (threadIdx.x == 0) span(0);
#else
  auto span = [](int) {};
#endif
  constexpr bool kTriple = kMode == 2 || kMode == 4;
  const uint32_t role_id = kMode == 1 ? cluster_ctarank() : kTriple ? blockIdx.x % 3 : 0u;
  const int seg = kMode == 1 ? (int)(blockIdx.x >> 1) : kTriple ? (int)(blockIdx.x / 3) : (int)blockIdx.x;
  const Role R = causal_role<kMode>(role_id, a);
  const int slot = blockIdx.y;
  int64_t lo, hi;
  seg_range(seg, a.nseg, a.tokens, &lo, &hi);
  const int nblk = (int)((hi - lo + kTile - 1) / kTile);
  const int nbox = a.dim > 64 ? 2 : 1;
  const int kfeat = (a.dim + 15) / 16;  // k-steps of feature contractions

  if (threadIdx.x == 0) {
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kMode == 1 ? 2 : 1);
    }
    for (int i = 0; i < 9; ++i) mbar_init(&s_full[i], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  if constexpr (kMode == 1) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) span(1);
  pdl_wait();
  pdl_launch_dependents();
  // TMEM: S [0,128) (kModes 1 / 4: P packed in place), O[0] [128,256), running state [256,384),
  // O[1] (kMode 3: G) [384,512)
  const uint32_t t_s = tmem, t_st = tmem + 256, t_g = tmem + 384;
  auto t_o = [&](int b) { return tmem + (b ? 384u : 128u); };
  auto o_buf = [&](int jj) { return kOneO ? 0 : (jj & 1); };
  auto release = [&](int s) {
    if constexpr (kMode == 1) mma_commit_mc(&empty[s], 0x3); else mma_commit(&empty[s]);
  };

  if (warp == 0) {
    // ---------------- TMA producer: ring order per block = q', k', v' ----------------
    if (elect_one()) {
      const CUtensorMap* maps[4] = {&tm.m[R.qi], &tm.m[R.ki], &tm.m[R.vi], &tm.m[4]};
      for (int w = 0; w < kTPB; ++w) prefetch_tmap(maps[w]);
      const uint32_t bytes = nbox * kBoxBytes;
      for (int jj = 0; jj < nblk; ++jj) {
        const int j = R.reverse ? nblk - 1 - jj : jj;
#ifdef LASP2_CHAIN_PROBE  // diagnostic: every block re-reads the segment's first tiles (L2-resident)
        const int row = (int)lo + 0 * j;
#else
        const int row = (int)(lo + (int64_t)j * kTile);
#endif
        if (kL2Prefetch<kMode> > 0) {  // the tiles this CTA loads, blocks ahead
          for (int w = 0; w < kTPB; ++w) {
            if (kMode == 1 && w != 0 && R.mcast != w) continue;
            // the pair prefetches only its multicast tile (the private one: +1.4 % at cfg3)
            const int dist = (kMode == 1 && w == 0) ? 0 : kL2Prefetch<kMode>;
            if (dist <= 0 || jj + dist >= nblk) continue;
            const int jp = R.reverse ? nblk - 1 - (jj + dist) : jj + dist;
            const int prow = (int)(lo + (int64_t)jp * kTile);
            for (int bx = 0; bx < nbox; ++bx) tma_prefetch_3d(maps[w], 64 * bx, prow, slot);
          }
        }
        for (int w = 0; w < kTPB; ++w) {
          const int t = kTPB * jj + w, s = t % kRing, u = t / kRing;
          if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
          uint8_t* dst = ring + s * kTileBytes;
          mbar_arrive_expect_tx(&full[s], bytes);
          if (kMode != 1 || w == 0) {
            for (int bx = 0; bx < nbox; ++bx) tma_load_3d(dst + bx * kBoxBytes, maps[w], &full[s], 64 * bx, row, slot);
          } else if (R.mcast == w) {  // kMode 1: rank 0 multicasts dO, rank 1 multicasts Q
            for (int bx = 0; bx < nbox; ++bx)
              tma_load_3d_mc(dst + bx * kBoxBytes, maps[w], &full[s], 64 * bx, row, slot, 0x3);
          }
        }
      }
      if constexpr (kMode == 1) {  // drain: both CTAs' final releases of every used slot have arrived here
        const int total = kTPB * nblk;
        for (int s = 0; s < kRing && s < total; ++s) {
          const int uses = (total - s + kRing - 1) / kRing;
          mbar_wait(&empty[s], (uses - 1) & 1);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t id_qk = idesc_bf16_f32(128, 128, 0, 0);  // S = Q K^T
    constexpr uint32_t id_qs = idesc_bf16_f32(128, 128, 0, 1);  // O = Q S
    constexpr uint32_t id_kv = idesc_bf16_f32(128, 128, 1, 1);  // S += K^T V
    constexpr uint32_t id_pv = idesc_bf16_f32(128, 128, 0, 1);  // O += P V
    const uint32_t simg_a = smem_u32(simg), pimg_a = smem_u32(pimg);
    const bool swap = kMode == 1 && R.mcast == 2;  // kMode 1 rank 1: ring positions of k', v' swapped
    Tracer tr;
    for (int jj = 0; jj < nblk; ++jj) {
      const int t0 = kTPB * jj;
      const int sq = t0 % kRing, sb = (t0 + 1) % kRing, sc = (t0 + 2) % kRing;
      const int sk = swap ? sc : sb, sv = swap ? sb : sc;
      const int tk = swap ? t0 + 2 : t0 + 1, tv = swap ? t0 + 1 : t0 + 2;
      const int ob = o_buf(jj);
      const uint32_t qa = smem_u32(ring + sq * kTileBytes);
      const uint32_t ka = smem_u32(ring + sk * kTileBytes);
      const uint32_t va = smem_u32(ring + sv * kTileBytes);
      if (lane == 0) tr(10, jj);
      mbar_wait(&full[sq], (t0 / kRing) & 1);
      mbar_wait(&full[sk], (tk / kRing) & 1);
      if (lane == 0) tr(11, jj);
      if (!kMmaProbe && jj > 0) mbar_wait(p_ready, (jj - 1) & 1);  // S tile drained by the epilogue
      tc_fence_after();
      if (lane == 0) tr(12, jj);
      if (elect_one()) {
        if (kfeat == 8) {  // d = 128: fully unrolled issue (the runtime-bound loop reloaded a spilled TMEM address per step)
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) mma_bf16_ss(t_s, desc_kmajor(qa, kk), desc_kmajor(ka, kk), id_qk, kk > 0);
        } else {
          for (int kk = 0; kk < kfeat; ++kk) mma_bf16_ss(t_s, desc_kmajor(qa, kk), desc_kmajor(ka, kk), id_qk, kk > 0);
        }
        mma_commit(s_full);
      }
      __syncwarp();
      if (R.subtract) {  // T = -S: T += k'^T v' first; the epilogue then images -T for this block
        mbar_wait(&full[sv], (tv / kRing) & 1);
        if (jj == 0) mbar_wait(sst_ready, 0);  // the seed (tcgen05.st of -S_end) has landed
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_bf16_ss(t_st, desc_mnmajor(ka, kk), desc_mnmajor(va, kk), id_kv, 1u);
          mma_commit(st_full);
          release(sk);
        }
        __syncwarp();
      }
      if (!kMmaProbe) mbar_wait(sst_ready, (jj + (R.subtract ? 1 : 0)) & 1);  // subtract form: arrival 0 is the seed
      if (lane == 0) tr(13, jj);
      if (!kMmaProbe && (kOneO ? jj >= 1 : jj >= 2)) mbar_wait(&o_empty[ob], (kOneO ? jj - 1 : (jj >> 1) - 1) & 1);
      tc_fence_after();
      if (lane == 0) tr(14, jj);
      if (elect_one()) {
        if (kfeat == 8) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_bf16_ss(t_o(ob), desc_kmajor(qa, kk), desc_mnmajor(simg_a, kk), id_qs, kk > 0);
        } else {
          for (int kk = 0; kk < kfeat; ++kk)
            mma_bf16_ss(t_o(ob), desc_kmajor(qa, kk), desc_mnmajor(simg_a, kk), id_qs, kk > 0);
        }
        if constexpr (kMode != 3) release(sq);
      }
      __syncwarp();
      if constexpr (kMode == 3) {  // G += X^T q' (token contraction, both MN-major views)
        const int sx = (t0 + 3) % kRing;
        mbar_wait(&full[sx], ((t0 + 3) / kRing) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t xa = smem_u32(ring + sx * kTileBytes);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_bf16_ss(t_g, desc_mnmajor(xa, kk), desc_mnmajor(qa, kk), id_kv, (jj > 0 || kk > 0) ? 1u : 0u);
          release(sq);
          release(sx);
          if (jj == nblk - 1) mma_commit(g_full);
        }
        __syncwarp();
      }
      if (!R.subtract) {
        mbar_wait(&full[sv], (tv / kRing) & 1);
        tc_fence_after();
        if (lane == 0) tr(15, jj);
        if (elect_one()) {
          if (jj < nblk - 1) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) mma_bf16_ss(t_st, desc_mnmajor(ka, kk), desc_mnmajor(va, kk), id_kv, 1u);
            mma_commit(st_full);
          }
          release(sk);
        }
        __syncwarp();
      }
      if (!kMmaProbe) mbar_wait(p_ready, jj & 1);
      tc_fence_after();
      if (lane == 0) tr(16, jj);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if constexpr (kPT)
            mma_bf16_ts(t_o(ob), t_s + kk * 8 + (kk >= 4 ? 32 : 0), desc_mnmajor(va, kk), id_pv, 1u);
          else
            mma_bf16_ss(t_o(ob), desc_kmajor(pimg_a, kk), desc_mnmajor(va, kk), id_pv, 1u);
        }
        release(sv);
        mma_commit(&o_full[ob]);
      }
      __syncwarp();
    }
    if (lane == 0) tr.flush(0);
    if (kMmaProbe) {  // every MMA complete before TMEM is released (no epilogue waits on them)
      if (elect_one()) mma_commit(g_full);
      __syncwarp();
      mbar_wait(g_full, 0);
    }
  } else {
    // -------- epilogue: 8 warps; warp w owns TMEM lanes 32*(w%4).. and columns [64*half, +64) --------
    const int qd = warp & 3;
    const int half = (warp - 2) >> 2;
    const int cb = 64 * half;
    const uint32_t row = qd * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    const int et = threadIdx.x - 64;
    constexpr uint32_t kEpi = kCausalThreads - 64;
    const int dim = a.dim;
    const int64_t dd = (int64_t)dim * dim;
    const CUtensorMap* tm_o = &tm.m[R.oi];
    Tracer tr;
    // initial state (optionally transposed); rows/cols beyond dim are zero
    //   forward form : base + seg_states[seg]                (state at the segment start)
    //   subtract form: fwd_base + fwd prefix of segment seg+1 (state at the segment end)
    {
      const float *st, *bs;
      if (R.subtract) {
        st = seg + 1 < a.nseg ? a.fwd_seg + ((int64_t)slot * a.nseg + seg + 1) * dd : a.fwd_total + (int64_t)slot * dd;
        bs = a.fwd_base ? a.fwd_base + (int64_t)slot * dd : nullptr;
      } else if (kMode == 4 && !R.neg) {  // dQ: forward prefix at the segment start
        st = a.fwd_seg ? a.fwd_seg + ((int64_t)slot * a.nseg + seg) * dd : nullptr;
        bs = a.fwd_base ? a.fwd_base + (int64_t)slot * dd : nullptr;
      } else if (kMode == 4) {  // dK / dV: suffix inclusive of the segment (seg_states: exclusive suffix scan)
        st = seg > 0 ? a.seg_states + ((int64_t)slot * a.nseg + seg - 1) * dd : a.seg_total + (int64_t)slot * dd;
        bs = a.base ? a.base + (int64_t)slot * dd : nullptr;
      } else {
        st = a.seg_states ? a.seg_states + ((int64_t)slot * a.nseg + seg) * dd : nullptr;
        bs = a.base ? a.base + (int64_t)slot * dd : nullptr;
      }
      const bool fold = a.xrecv != nullptr && a.xhi > a.xlo;
      if (et == 0) span(12);  // epilogue start
      // device-resident epoch (graph replays): the producer's scan_put, earlier on this stream, set it
      const unsigned long long xep =
          a.xepoch_dev != nullptr ? *(volatile const unsigned long long*)a.xepoch_dev : a.xepoch;
      const float* xrecv = a.xepoch_dev != nullptr ? a.xrecv + (int64_t)(xep & 1) * a.xhalf : a.xrecv;
      if (a.xrecv != nullptr && a.xflags != nullptr) {  // wait for the ranks this fold needs (TMA / MMA run ahead)
        if (et == 0) {
          for (int j = a.xlo; j < a.xhi; ++j) {
            const long long t0 = clock64();
            while (ld_acquire_sys_u64(a.xflags + j) < xep) {
              __nanosleep(64);
              if (clock64() - t0 > (1ll << 36)) __trap();  // a peer never arrived: fail loudly
            }
          }
        }
        named_bar_sync(1, kEpi);
      }
      const int64_t xstride = (int64_t)gridDim.y * dd;  // one rank's [slots][dim][dim] in the receive half
      const float* xb = xrecv + (int64_t)slot * dd;
      float* bo = (a.base_out != nullptr && seg == 0 && (kMode != 1 || R.mcast == 1)) ? a.base_out + (int64_t)slot * dd
                                                                                        : nullptr;
      // every load of a 32-column chunk is issued before any store (base_out), so the
      // chunk costs one memory latency, not one per element (the stores may alias as
      // far as the compiler knows)
      const bool rowok = (int)row < dim;
      int c0_cur = cb;
      // nc: states written by earlier launches (read-only here): L1-cached loads, so a
      // thread's 8 float4 of one row cost one L2 request, not eight. Peer buffers use .cg.
      auto load32 = [&](const float* base, float* dst, bool nc) {  // dst[i] = element (row, c0 + i) of base
        if (!R.transpose && rowok && c0_cur + 32 <= dim) {
          const float4* p4 = reinterpret_cast<const float4*>(base + (int64_t)row * dim + c0_cur);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 f = nc ? __ldg(p4 + u) : __ldcg(p4 + u);
            dst[4 * u] = f.x;
            dst[4 * u + 1] = f.y;
            dst[4 * u + 2] = f.z;
            dst[4 * u + 3] = f.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int c = c0_cur + i;
            const float* e = base + (R.transpose ? (int64_t)c * dim + row : (int64_t)row * dim + c);
            dst[i] = (rowok && c < dim) ? (nc ? __ldg(e) : __ldcg(e)) : 0.f;
          }
        }
      };
#pragma unroll 1
      for (int c0 = cb; c0 < cb + 64; c0 += 32) {
        c0_cur = c0;
        float v[32], t[32];
        if (fold) {  // first term copied, the rest in rank order (numerics.py:71-116)
          const int first = a.xdesc ? a.xhi - 1 : a.xlo;
          load32(xb + first * xstride, v, false);
          if (a.xdesc) {
            for (int j = a.xhi - 2; j >= a.xlo; --j) {
              load32(xb + j * xstride, t, false);
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] += t[i];
            }
          } else {
            for (int j = a.xlo + 1; j < a.xhi; ++j) {
              load32(xb + j * xstride, t, false);
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] += t[i];
            }
          }
        } else if (bs) {
          load32(bs, v, true);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
        if (bo != nullptr) {  // the folded base alone (M_{1:t-1} for the cache), zeros when nothing was folded
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int c = c0 + i;
            if (rowok && c < dim) bo[R.transpose ? (int64_t)c * dim + row : (int64_t)row * dim + c] = fold ? v[i] : 0.f;
          }
        }
        if (st) {
          load32(st, t, true);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += t[i];
        }
        if (et == 0) span(8 + (c0 - cb) / 16);  // 8 / 10: chunk loaded
        if (R.neg) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = -v[i];
        }
        uint32_t r[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(R.subtract ? -v[i] : v[i]);
        tmem_st_32x32b_x32(t_st + lane_off + c0, r);
        if (!R.subtract) st_row32_bf16(simg, row, c0, v);
        if (et == 0) span(9 + (c0 - cb) / 16);  // 9 / 11: chunk stored
      }
      tmem_st_wait();
      fence_proxy_async_smem();
      tc_fence_before();
      named_bar_sync(1, kEpi);
      if (et == 0) mbar_arrive(sst_ready);  // forward form: image of block 0; subtract form: seed landed
      if (et == 0) span(2);
    }
    for (int jj = 0; jj < (kMmaProbe ? 0 : nblk); ++jj) {
      const int j = R.reverse ? nblk - 1 - jj : jj;
      const int ob = o_buf(jj);
      // ---- subtract form: this block's (post-subtraction) state image comes first
      if (R.subtract) {
        mbar_wait(st_full, jj & 1);
        tc_fence_after();
        tmem_cols_to_image<0, true>(t_st + lane_off, simg, row, cb, 64);
        fence_proxy_async_smem();
        tc_fence_before();
        named_bar_sync(1, kEpi);
        if (et == 0) mbar_arrive(sst_ready);
      }
      // ---- P = mask(S) -> smem (after the previous O tile left the staging buffer)
      if (et == 0) tr(20, jj);
      mbar_wait(s_full, jj & 1);
      tc_fence_after();
      if (et == 0) tr(21, jj);
      if constexpr (kPT) {  // P -> TMEM over S (S_j completed after P.v'_{j-1}, in issue order)
        if (et == 0) tr(22, jj);
#ifndef LASP2_EPI_PROBE  // diagnostic build: the epilogue only signals (garbage results; timing of the MMA / TMA chain)
        if (R.mask == 2)
          tmem_cols_to_tmem_bf16<2, true>(t_s + lane_off, t_s + lane_off, row, cb, 64);
        else if (R.mask == 3)
          tmem_cols_to_tmem_bf16<3, true>(t_s + lane_off, t_s + lane_off, row, cb, 64);
        else
          tmem_cols_to_tmem_bf16<1, true>(t_s + lane_off, t_s + lane_off, row, cb, 64);
#endif
        tmem_st_wait();
      } else {
        if (jj > 0 && et == 0) tma_store_wait_read<0>();
        named_bar_sync(1, kEpi);
        if (et == 0) tr(22, jj);
        if (R.mask == 2)
          tmem_cols_to_image<2>(t_s + lane_off, pimg, row, cb, 64);
        else
          tmem_cols_to_image<1>(t_s + lane_off, pimg, row, cb, 64);
        fence_proxy_async_smem();
      }
      tc_fence_before();
      named_bar_sync(1, kEpi);
      if (et == 0) mbar_arrive(p_ready);
      if (et == 0) tr(23, jj);
      if (et == 0 && jj == 0) span(3);
      // ---- forward form: next block's state image
      if (!R.subtract && jj < nblk - 1) {
        mbar_wait(st_full, jj & 1);
        tc_fence_after();
        if (et == 0) tr(24, jj);
#ifndef LASP2_EPI_PROBE
        tmem_cols_to_image<0>(t_st + lane_off, simg, row, cb, 64);
#endif
        fence_proxy_async_smem();
        tc_fence_before();
        named_bar_sync(1, kEpi);
        if (et == 0) mbar_arrive(sst_ready);
        if (et == 0) tr(25, jj);
      }
      // ---- O tile -> staging -> TMA store
      mbar_wait(&o_full[ob], (kOneO ? jj : jj >> 1) & 1);
      tc_fence_after();
      if (et == 0) tr(26, jj);
      if (kPT && jj > 0) {  // staging is O-only here: the previous O store must have left it
        if (et == 0) tma_store_wait_read<0>();
        named_bar_sync(1, kEpi);
      }
#ifndef LASP2_EPI_PROBE
      if (R.neg)
        tmem_cols_to_image<0, true>(t_o(ob) + lane_off, pimg, row, cb, 64);
      else
        tmem_cols_to_image<0>(t_o(ob) + lane_off, pimg, row, cb, 64);
#endif
      fence_proxy_async_smem();
      tc_fence_before();
      named_bar_sync(1, kEpi);
      if (et == 0) {
        mbar_arrive(&o_empty[ob]);
#ifdef LASP2_CHAIN_PROBE
        const int orow = (int)lo + 0 * j;
#else
        const int orow = (int)(lo + (int64_t)j * kTile);
#endif
        for (int bx = 0; bx < nbox; ++bx) tma_store_3d(tm_o, pimg + bx * kBoxBytes, 64 * bx, orow, slot);
        tma_store_commit();
        tr(27, jj);
        if (jj == 0) span(4);
      }
    }
    if (et == 0) span(5);
    if constexpr (kMode == 3) {  // segment state G -> fp32 [slot][seg][dim][dim]
      if (nblk > 0) {
        mbar_wait(g_full, 0);
        tc_fence_after();
        float* gb = a.g_out + ((int64_t)slot * a.nseg + seg) * dd + (int64_t)row * dim;
#pragma unroll 1
        for (int c0 = cb; c0 < cb + 64; c0 += 32) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_g + lane_off + c0, r);
          tmem_ld_wait();
          if ((int)row < dim && c0 < dim) {
            if (c0 + 32 <= dim) {
#pragma unroll
              for (int i = 0; i < 32; i += 4)
                *reinterpret_cast<float4*>(gb + c0 + i) = make_float4(__uint_as_float(r[i]), __uint_as_float(r[i + 1]),
                                                                      __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (c0 + i < dim) gb[c0 + i] = __uint_as_float(r[i]);
            }
          }
        }
      }
    }
    if (et == 0) tma_store_wait_all<0>();
    if (et == 0) tr.flush(1);
    if (et == 0) span(6);
  }
  tc_fence_before();
  if constexpr (kMode == 1) cluster_sync(); else __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
  if (threadIdx.x == 0) span(7);
#if !defined(LASP2_TRACE) && !defined(LASP2_SPAN)
  if (g_trace != nullptr && threadIdx.x == 0) {
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    const uint32_t cta = blockIdx.y * gridDim.x + blockIdx.x;
    g_trace[2 * cta] = t_begin;
    g_trace[2 * cta + 1] = t_end;
  }
#endif
}

// ============================================================================
// apply_state: O (+)= X M  (transpose=0) or X M^T (transpose=1); with NX = 3 the
// sum of three such products into one accumulator (one rounding): the hybrid
// stack's dX = dQ W_Q^T + dK W_K^T + dV W_V^T. M is per slot (m_stride = dim^2)
// or one weight shared by every slot (m_stride = 0).
// ============================================================================
template <int NX>
struct ApplyCfg {
  static constexpr int kRing = NX == 1 ? 4 : 3;
  static constexpr int kStages = NX == 1 ? 2 : 1;
  static constexpr uint32_t kSmem = (kRing + NX + kStages) * kTileBytes + 1024 + 256;
};
constexpr uint32_t kApplySmem = ApplyCfg<1>::kSmem;

struct ApplyMaps {
  CUtensorMap x[3];
};

template <int NX>
__global__ void __launch_bounds__(192, 1)
    tc_apply_state_kernel(const __grid_constant__ ApplyMaps tmx, const __grid_constant__ CUtensorMap tm_o,
                          const float* m0, const float* m1, const float* m2, int64_t m_stride,
                          __nv_bfloat16* out, int64_t tokens, int dim, int transpose, int accumulate,
                          int blocks_per_cta) {
  using C = ApplyCfg<NX>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint8_t* mimg = ring + C::kRing * kTileBytes;  // [NX]
  uint8_t* stage = mimg + NX * kTileBytes;       // [kStages] x 32 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(stage + C::kStages * kTileBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::kRing;
  uint64_t* acc_full = bars + 2 * C::kRing;       // [2]
  uint64_t* acc_empty = bars + 2 * C::kRing + 2;  // [2]
  uint64_t* m_ready = bars + 2 * C::kRing + 4;
  uint64_t* o_full = bars + 2 * C::kRing + 5;  // [2] accumulate: the old O tile landed in stage[buf]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::kRing + 7);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = blockIdx.y;
  const int64_t nblk_all = (tokens + kTile - 1) / kTile;
  const int64_t b0 = (int64_t)blockIdx.x * blocks_per_cta;
  const int64_t b1 = lmin(nblk_all, b0 + blocks_per_cta);
  const int nblk = (int)lmax(0, b1 - b0);
  const int nbox = dim > 64 ? 2 : 1;
  const int kfeat = (dim + 15) / 16;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::kRing; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 7; ++i) mbar_init(&acc_full[i], 1);  // acc_full, acc_empty, m_ready, o_full
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    if (elect_one()) {
      for (int i = 0; i < NX; ++i) prefetch_tmap(&tmx.x[i]);
      prefetch_tmap(&tm_o);
      for (int b = 0; b < nblk; ++b) {
        const int row = (int)((b0 + b) * kTile);
        for (int i = 0; i < NX; ++i) {
          const int t = NX * b + i, s = t % C::kRing, u = t / C::kRing;
          if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
          uint8_t* dst = ring + s * kTileBytes;
          mbar_arrive_expect_tx(&full[s], nbox * kBoxBytes);
          for (int bx = 0; bx < nbox; ++bx) tma_load_3d(dst + bx * kBoxBytes, &tmx.x[i], &full[s], 64 * bx, row, slot);
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_bf16_f32(128, 128, 0, transpose ? 0 : 1);
    mbar_wait(m_ready, 0);
    for (int b = 0; b < nblk; ++b) {
      const int buf = b & 1;
      if (b >= 2) mbar_wait(&acc_empty[buf], ((b >> 1) - 1) & 1);
      for (int i = 0; i < NX; ++i) {
        const int t = NX * b + i, s = t % C::kRing, u = t / C::kRing;
        mbar_wait(&full[s], u & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t xa = smem_u32(ring + s * kTileBytes), ma = smem_u32(mimg + i * kTileBytes);
          for (int kk = 0; kk < kfeat; ++kk) {
            const uint64_t bdesc = transpose ? desc_kmajor(ma, kk) : desc_mnmajor(ma, kk);
            mma_bf16_ss(tmem + buf * 128, desc_kmajor(xa, kk), bdesc, idesc, (i > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&empty[s]);
          if (i == NX - 1) mma_commit(&acc_full[buf]);
        }
        __syncwarp();
      }
    }
  } else {
    const int qd = warp & 3;
    const uint32_t row = qd * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    const int et = threadIdx.x - 64;
    const int64_t dd = (int64_t)dim * dim;
    // state / weight images: rows = first index of M, contiguous = second index
    const float* ms[3] = {m0, m1, m2};
#pragma unroll 1
    for (int i = 0; i < NX; ++i) {
      const float* mb = ms[i] + (int64_t)slot * m_stride;
#pragma unroll 1
      for (int c0 = 0; c0 < 128; c0 += 32) {
        float v[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int c = c0 + k;
          v[k] = ((int)row < dim && c < dim) ? mb[(int64_t)row * dim + c] : 0.f;
        }
        st_row32_bf16(mimg + i * kTileBytes, row, c0, v);
      }
    }
    (void)dd;
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (et == 0) mbar_arrive(m_ready);
    // accumulate (NX = 1): the old O tile of block b is TMA-loaded into stage[buf] (once the
    // store of block b-2 has read it) and added from shared memory, coalesced like the stores
    auto load_old = [&](int b) {
      const int buf = b & 1;
      if (b >= 2) tma_store_wait_read<0>();  // the store of block b-2 (the latest group) has read stage[buf]
      mbar_arrive_expect_tx(&o_full[buf], nbox * kBoxBytes);
      const int orow = (int)((b0 + b) * kTile);
      for (int bx = 0; bx < nbox; ++bx)
        tma_load_3d(stage + buf * kTileBytes + bx * kBoxBytes, &tm_o, &o_full[buf], 64 * bx, orow, slot);
    };
    const bool acc_old = NX == 1 && accumulate;
    if (acc_old && et == 0 && nblk > 0) load_old(0);
    for (int b = 0; b < nblk; ++b) {
      const int buf = b & 1, sbuf = C::kStages == 2 ? buf : 0;
      if (acc_old && et == 0 && b + 1 < nblk) load_old(b + 1);
      mbar_wait(&acc_full[buf], (b >> 1) & 1);
      tc_fence_after();
      if (acc_old) mbar_wait(&o_full[buf], (b >> 1) & 1);
      else if (et == 0) {
        if (C::kStages == 2 && b >= 2) tma_store_wait_read<1>();
        if (C::kStages == 1 && b >= 1) tma_store_wait_read<0>();
      }
      named_bar_sync(1, 128);
      uint8_t* st = stage + sbuf * kTileBytes;
#pragma unroll 1
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem + buf * 128 + lane_off + c0, r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = __uint_as_float(r[k]);
        if (acc_old) ld_row32_add_bf16(st, row, c0, v);
        st_row32_bf16(st, row, c0, v);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      named_bar_sync(1, 128);
      if (et == 0) {
        mbar_arrive(&acc_empty[buf]);
        const int orow = (int)((b0 + b) * kTile);
        for (int bx = 0; bx < nbox; ++bx) tma_store_3d(&tm_o, st + bx * kBoxBytes, 64 * bx, orow, slot);
        tma_store_commit();
      }
    }
    if (et == 0) tma_store_wait_all<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<256>(tmem);
}

// ============================================================================
// Fused unmasked-backward kernels (8 epilogue warps, 64 columns each):
//   MODE 0 (state_apply): seg[slot][g] = X0_g^T X1_g and out0 = X1 M^T
//          -> dM segments (Q^T dO) and dQ = dO M^T reading Q, dO once
//   MODE 1 (apply2)     : out0 = X0 M^T, out1 = X1 M
//          -> dK = V dM^T and dV = K dM from one bf16 image of dM
// (reference lasp2.py:256-267)
// ============================================================================
constexpr int kFusedThreads = 320;
constexpr int kFusedStages = 2;  // each stage holds the two input tiles of one block
constexpr uint32_t kFusedSmem = (2 * kFusedStages + 3) * kTileBytes + 1024 + 256;

template <int MODE>
__global__ void __launch_bounds__(kFusedThreads, 1)
    tc_fused_apply_kernel(const __grid_constant__ CUtensorMap tm_x0, const __grid_constant__ CUtensorMap tm_x1,
                          const __grid_constant__ CUtensorMap tm_o0, const __grid_constant__ CUtensorMap tm_o1,
                          const float* __restrict__ m, float* __restrict__ seg_out, int64_t tokens, int dim, int nseg,
                          int blocks_per_cta) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;                                    // [stage][2] tiles
  uint8_t* mimg = ring + 2 * kFusedStages * kTileBytes;   // bf16 state image
  uint8_t* stg = mimg + kTileBytes;                        // [2] output staging
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg + 2 * kTileBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kFusedStages;
  uint64_t* acc_full = bars + 2 * kFusedStages;       // [2]
  uint64_t* acc_empty = bars + 2 * kFusedStages + 2;  // [2]
  uint64_t* m_ready = bars + 2 * kFusedStages + 4;
  uint64_t* g_full = bars + 2 * kFusedStages + 5;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kFusedStages + 6);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = blockIdx.y;
  int64_t b0, b1;
  if (MODE == 0) {
    int64_t lo, hi;
    seg_range(blockIdx.x, nseg, tokens, &lo, &hi);
    b0 = lo / kTile;
    b1 = (hi + kTile - 1) / kTile;
  } else {
    const int64_t nblk_all = (tokens + kTile - 1) / kTile;
    b0 = (int64_t)blockIdx.x * blocks_per_cta;
    b1 = lmin(nblk_all, b0 + blocks_per_cta);
  }
  const int nblk = (int)lmax(0, b1 - b0);
  const int nbox = dim > 64 ? 2 : 1;
  const int kfeat = (dim + 15) / 16;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kFusedStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 6; ++i) mbar_init(&acc_full[i], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();
  // MODE 0: G [0,128), out0[2] at 128/256.  MODE 1: out0[2] at 0/128, out1[2] at 256/384.
  auto t_out0 = [&](int b) { return tmem + (MODE == 0 ? 128u + 128u * b : 128u * b); };
  auto t_out1 = [&](int b) { return tmem + 256u + 128u * b; };

  if (warp == 0) {
    if (elect_one()) {
      prefetch_tmap(&tm_x0);
      prefetch_tmap(&tm_x1);
      for (int b = 0; b < nblk; ++b) {
        const int s = b % kFusedStages, u = b / kFusedStages;
        if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
        uint8_t* d0 = ring + (2 * s) * kTileBytes;
        uint8_t* d1 = d0 + kTileBytes;
        mbar_arrive_expect_tx(&full[s], 2 * nbox * kBoxBytes);
        const int row = (int)((b0 + b) * kTile);
        for (int bx = 0; bx < nbox; ++bx) {
          tma_load_3d(d0 + bx * kBoxBytes, &tm_x0, &full[s], 64 * bx, row, slot);
          tma_load_3d(d1 + bx * kBoxBytes, &tm_x1, &full[s], 64 * bx, row, slot);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t id_g = idesc_bf16_f32(128, 128, 1, 1);    // X0^T X1
    constexpr uint32_t id_mt = idesc_bf16_f32(128, 128, 0, 0);   // X M^T (B = image K-major)
    constexpr uint32_t id_m = idesc_bf16_f32(128, 128, 0, 1);    // X M   (B = image MN-major)
    const uint32_t ma = smem_u32(mimg);
    mbar_wait(m_ready, 0);
    for (int b = 0; b < nblk; ++b) {
      const int s = b % kFusedStages, u = b / kFusedStages;
      const int buf = b & 1;
      mbar_wait(&full[s], u & 1);
      if (b >= 2) mbar_wait(&acc_empty[buf], ((b >> 1) - 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t x0 = smem_u32(ring + (2 * s) * kTileBytes), x1 = x0 + kTileBytes;
        if (MODE == 0) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_bf16_ss(tmem, desc_mnmajor(x0, kk), desc_mnmajor(x1, kk), id_g, (b > 0 || kk > 0) ? 1u : 0u);
          for (int kk = 0; kk < kfeat; ++kk)
            mma_bf16_ss(t_out0(buf), desc_kmajor(x1, kk), desc_kmajor(ma, kk), id_mt, kk > 0);
        } else {
          for (int kk = 0; kk < kfeat; ++kk)
            mma_bf16_ss(t_out0(buf), desc_kmajor(x0, kk), desc_kmajor(ma, kk), id_mt, kk > 0);
          for (int kk = 0; kk < kfeat; ++kk)
            mma_bf16_ss(t_out1(buf), desc_kmajor(x1, kk), desc_mnmajor(ma, kk), id_m, kk > 0);
        }
        mma_commit(&empty[s]);
        mma_commit(&acc_full[buf]);
        if (MODE == 0 && b == nblk - 1) mma_commit(g_full);
      }
      __syncwarp();
    }
  } else {
    const int qd = warp & 3;
    const int half = (warp - 2) >> 2;
    const int cb = 64 * half;
    const uint32_t row = qd * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    const int et = threadIdx.x - 64;
    constexpr uint32_t kEpi = kFusedThreads - 64;
    const int64_t dd = (int64_t)dim * dim;
    const float* mb = m + (int64_t)slot * dd;
#pragma unroll 1
    for (int c0 = cb; c0 < cb + 64; c0 += 32) {
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int c = c0 + i;
        v[i] = ((int)row < dim && c < dim) ? mb[(int64_t)row * dim + c] : 0.f;
      }
      st_row32_bf16(mimg, row, c0, v);
    }
    fence_proxy_async_smem();
    named_bar_sync(1, kEpi);
    if (et == 0) mbar_arrive(m_ready);
    for (int b = 0; b < nblk; ++b) {
      const int buf = b & 1;
      mbar_wait(&acc_full[buf], (b >> 1) & 1);
      tc_fence_after();
      if (et == 0) {
        if (MODE == 0 && b >= 2) tma_store_wait_read<1>();
        if (MODE == 1 && b >= 1) tma_store_wait_read<0>();
      }
      named_bar_sync(1, kEpi);
      if (MODE == 0) {
        tmem_cols_to_image<0>(t_out0(buf) + lane_off, stg + buf * kTileBytes, row, cb, 64);
      } else {
        tmem_cols_to_image<0>(t_out0(buf) + lane_off, stg, row, cb, 64);
        tmem_cols_to_image<0>(t_out1(buf) + lane_off, stg + kTileBytes, row, cb, 64);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      named_bar_sync(1, kEpi);
      if (et == 0) {
        mbar_arrive(&acc_empty[buf]);
        const int orow = (int)((b0 + b) * kTile);
        if (MODE == 0) {
          for (int bx = 0; bx < nbox; ++bx)
            tma_store_3d(&tm_o0, stg + buf * kTileBytes + bx * kBoxBytes, 64 * bx, orow, slot);
        } else {
          for (int bx = 0; bx < nbox; ++bx) {
            tma_store_3d(&tm_o0, stg + bx * kBoxBytes, 64 * bx, orow, slot);
            tma_store_3d(&tm_o1, stg + kTileBytes + bx * kBoxBytes, 64 * bx, orow, slot);
          }
        }
        tma_store_commit();
      }
    }
    if (MODE == 0 && nblk > 0) {  // segment state G -> fp32 [slot][seg][dim][dim]
      mbar_wait(g_full, 0);
      tc_fence_after();
      float* ob = seg_out + ((int64_t)slot * nseg + blockIdx.x) * dd;
#pragma unroll 1
      for (int c0 = cb; c0 < cb + 64; c0 += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem + lane_off + c0, r);
        tmem_ld_wait();
        if ((int)row < dim) {
          float* orow = ob + (int64_t)row * dim + c0;
          if (c0 + 32 <= dim && (dim & 3) == 0) {
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              *reinterpret_cast<float4*>(orow + i) = make_float4(
                  __uint_as_float(r[i]), __uint_as_float(r[i + 1]), __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c0 + i < dim) orow[i] = __uint_as_float(r[i]);
          }
        }
      }
    }
    if (et == 0) tma_store_wait_all<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// ============================================================================
// Debug probe: D = op(A) op(B)^T for one 128x128x128 tile, to pin descriptor
// conventions on hardware (a_mn / b_mn select MN-major interpretation).
// ============================================================================
__global__ void __launch_bounds__(128, 1)
    tc_probe_gemm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                         float* __restrict__ d, int a_mn, int b_mn) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* at = smem;
  uint8_t* bt = smem + kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * kTileBytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bars[0], 2 * kTileBytes);
    tma_load_3d(at, &tm_a, &bars[0], 0, 0, 0);
    tma_load_3d(at + kBoxBytes, &tm_a, &bars[0], 64, 0, 0);
    tma_load_3d(bt, &tm_b, &bars[0], 0, 0, 0);
    tma_load_3d(bt + kBoxBytes, &tm_b, &bars[0], 64, 0, 0);
  }
  mbar_wait(&bars[0], 0);
  if (a_mn == 2) {  // TS mode: row r of A (this thread) packed bf16x2 along K into TMEM columns [128, 192)
    const uint32_t r = warp * 32 + lane;
    uint32_t pk[64];
#pragma unroll
    for (int c = 0; c < 64; ++c)
      pk[c] = *reinterpret_cast<const uint32_t*>(at + sw128_offset(r, 2 * c));
    const uint32_t lane_base = tmem + ((warp * 32) << 16) + 128;
    tmem_st_32x32b_x32(lane_base, *reinterpret_cast<uint32_t(*)[32]>(pk));
    tmem_st_32x32b_x32(lane_base + 32, *reinterpret_cast<uint32_t(*)[32]>(pk + 32));
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, 128, a_mn == 1 ? 1 : 0, b_mn);
    const uint32_t aa = smem_u32(at), ba = smem_u32(bt);
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t bd = b_mn ? desc_mnmajor(ba, kk) : desc_kmajor(ba, kk);
      if (a_mn == 2) {
        mma_bf16_ts(tmem, tmem + 128 + kk * 8, bd, idesc, kk > 0);
      } else {
        const uint64_t ad = a_mn ? desc_mnmajor(aa, kk) : desc_kmajor(aa, kk);
        mma_bf16_ss(tmem, ad, bd, idesc, kk > 0);
      }
    }
    mma_commit(&bars[1]);
  }
  __syncwarp();
  mbar_wait(&bars[1], 0);
  tc_fence_after();
  const uint32_t row = warp * 32 + lane;
  for (int c0 = 0; c0 < 128; c0 += 32) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(tmem + ((warp * 32) << 16) + c0, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; ++i) d[row * 128 + c0 + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

}  // namespace tc

// ============================================================================
// Host side: tensor maps + launchers
// ============================================================================
bool tc_supported(int dim, int64_t tokens) { return dim >= 8 && dim <= 128 && dim % 8 == 0 && tokens >= 1; }

cudaError_t tc_segment_states(const void* x, const void* y, float* out, int64_t slots, int64_t tokens, int dim,
                              int nseg, cudaStream_t s) {
  CUtensorMap mx, my;
  cudaError_t e;
  if ((e = make_tmap_3d(&mx, x, slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = make_tmap_3d(&my, y, slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = set_smem_once((const void*)tc::tc_segment_states_kernel, tc::kSegSmem)) != cudaSuccess) return e;
  dim3 grid(nseg, (unsigned)slots);
  return launch_pdl(tc::tc_segment_states_kernel, grid, dim3(192), tc::kSegSmem, s, 1, mx, my, out, tokens, dim, nseg);
}

namespace {
void set_xfold(tc::CausalArgs* a, const XFold* x) {
  if (x == nullptr) return;
  a->base = nullptr;
  a->xrecv = x->recv;
  a->xflags = x->flags;
  a->xlo = x->lo;
  a->xhi = x->hi;
  a->xdesc = x->descending;
  a->xepoch = x->epoch;
  a->base_out = x->base_out;
  a->xepoch_dev = x->epoch_dev;
  a->xhalf = x->half_elems;
}
}  // namespace

cudaError_t tc_causal_chunk(const void* q, const void* k, const void* v, const float* seg_states, const float* base,
                            void* out, int64_t slots, int64_t tokens, int dim, int nseg, int reverse,
                            int transpose_state, cudaStream_t s, const XFold* xfold) {
  tc::TileMaps tm;
  cudaError_t e;
  const void* ptrs[4] = {q, k, v, out};
  for (int i = 0; i < 4; ++i)
    if ((e = make_tmap_3d(&tm.m[i], ptrs[i], slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = set_smem_once((const void*)tc::tc_causal_chunk_kernel<0>, tc::kCausalSmem)) != cudaSuccess) return e;
  tc::CausalArgs a{seg_states, base, nullptr, nullptr, nullptr, nullptr, tokens, dim, nseg, reverse, transpose_state};
  set_xfold(&a, xfold);
  dim3 grid(nseg, (unsigned)slots);
  return launch_pdl(tc::tc_causal_chunk_kernel<0>, grid, dim3(tc::kCausalThreads), tc::kCausalSmem, s, 1, tm, a);
}

// Masked backward dQ = causal(dO, V, K; S^T) plus the dM segment states Q_g^T dO_g in one pass.
cudaError_t tc_dq_chunk(const void* q, const void* k, const void* v, const void* d_out, const float* fwd_seg,
                        const float* fwd_base, float* g_out, void* dq, int64_t slots, int64_t tokens, int dim,
                        int nseg, cudaStream_t s) {
  tc::TileMaps tm;
  cudaError_t e;
  const void* ptrs[5] = {d_out, v, k, dq, q};
  for (int i = 0; i < 5; ++i)
    if ((e = make_tmap_3d(&tm.m[i], ptrs[i], slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = set_smem_once((const void*)tc::tc_causal_chunk_kernel<3>, tc::kCausalSmem)) != cudaSuccess) return e;
  tc::CausalArgs a{fwd_seg, fwd_base, nullptr, nullptr, nullptr, g_out, tokens, dim, nseg, 0, 1};
  dim3 grid(nseg, (unsigned)slots);
  return launch_pdl(tc::tc_causal_chunk_kernel<3>, grid, dim3(tc::kCausalThreads), tc::kCausalSmem, s, 1, tm, a);
}

// Masked backward dK and dV in one pass over (Q, K, V, dO): 2-CTA clusters.
cudaError_t tc_dkdv_pair(const void* q, const void* k, const void* v, const void* d_out, const float* seg_states,
                         const float* base, void* dk, void* dv, int64_t slots, int64_t tokens, int dim, int nseg,
                         cudaStream_t s, const XFold* xfold) {
  tc::TileMaps tm;
  cudaError_t e;
  const void* ptrs[6] = {v, k, d_out, q, dk, dv};
  for (int i = 0; i < 6; ++i)
    if ((e = make_tmap_3d(&tm.m[i], ptrs[i], slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = set_smem_once((const void*)tc::tc_causal_chunk_kernel<1>, tc::kCausalSmem)) != cudaSuccess) return e;
  tc::CausalArgs a{seg_states, base, nullptr, nullptr, nullptr, nullptr, tokens, dim, nseg, 1, 0};
  set_xfold(&a, xfold);
  return launch_pdl(tc::tc_causal_chunk_kernel<1>, dim3(2 * nseg, (unsigned)slots), dim3(tc::kCausalThreads),
                    tc::kCausalSmem, s, 2, tm, a);
}

// Masked backward dQ, dK, dV in one launch: three CTAs per segment sharing tiles through L2.
cudaError_t tc_backward_triple(const void* q, const void* k, const void* v, const void* d_out, const float* fwd_seg,
                               const float* fwd_total, const float* fwd_base, const float* bwd_seg,
                               const float* bwd_base, void* dq, void* dk, void* dv, int64_t slots, int64_t tokens,
                               int dim, int nseg, cudaStream_t s, const float* bwd_total) {
  tc::TileMaps tm;
  cudaError_t e;
  const void* ptrs[7] = {q, k, v, d_out, dq, dk, dv};
  for (int i = 0; i < 7; ++i)
    if ((e = make_tmap_3d(&tm.m[i], ptrs[i], slots, tokens, dim)) != cudaSuccess) return e;
  dim3 grid(3 * nseg, (unsigned)slots);
  if (bwd_total != nullptr) {  // forward-order triple (kMode 4)
    if ((e = set_smem_once((const void*)tc::tc_causal_chunk_kernel<4>, tc::kCausalSmem)) != cudaSuccess) return e;
    tc::CausalArgs a{bwd_seg, bwd_base, fwd_seg, nullptr, fwd_base, nullptr, tokens, dim, nseg, 0, 0};
    a.seg_total = bwd_total;
    return launch_pdl(tc::tc_causal_chunk_kernel<4>, grid, dim3(tc::kCausalThreads), tc::kCausalSmem, s, 1, tm, a);
  }
  if ((e = set_smem_once((const void*)tc::tc_causal_chunk_kernel<2>, tc::kCausalSmem)) != cudaSuccess) return e;
  tc::CausalArgs a{bwd_seg, bwd_base, fwd_seg, fwd_total, fwd_base, nullptr, tokens, dim, nseg, 1, 0};
  return launch_pdl(tc::tc_causal_chunk_kernel<2>, grid, dim3(tc::kCausalThreads), tc::kCausalSmem, s, 1, tm, a);
}

cudaError_t tc_apply_multi(const void* const* xs, const float* const* ms, int nx, int64_t m_stride, void* out,
                           int64_t slots, int64_t tokens, int dim, int transpose, int accumulate, int sm_count,
                           cudaStream_t s) {
  tc::ApplyMaps tm;
  CUtensorMap mo;
  cudaError_t e;
  for (int i = 0; i < nx; ++i)
    if ((e = make_tmap_3d(&tm.x[i], xs[i], slots, tokens, dim)) != cudaSuccess) return e;
  for (int i = nx; i < 3; ++i) tm.x[i] = tm.x[0];
  if ((e = make_tmap_3d(&mo, out, slots, tokens, dim)) != cudaSuccess) return e;
  const int64_t nblk = (tokens + tc::kTile - 1) / tc::kTile;
  // exactly one wave (one CTA per SM): ctas_per_slot * slots <= sm_count
  int64_t ctas = sm_count / slots;
  if (ctas < 1) ctas = 1;
  if (ctas > nblk) ctas = nblk;
  const int bpc = (int)((nblk + ctas - 1) / ctas);
  ctas = (nblk + bpc - 1) / bpc;
  dim3 grid((unsigned)ctas, (unsigned)slots);
  const float* m1 = nx > 1 ? ms[1] : ms[0];
  const float* m2 = nx > 2 ? ms[2] : ms[0];
  if (nx == 1) {
    if ((e = set_smem_once((const void*)tc::tc_apply_state_kernel<1>, tc::ApplyCfg<1>::kSmem)) != cudaSuccess)
      return e;
    return launch_pdl(tc::tc_apply_state_kernel<1>, grid, dim3(192), tc::ApplyCfg<1>::kSmem, s, 1, tm, mo, ms[0],
                      m1, m2, m_stride, (__nv_bfloat16*)out, tokens, dim, transpose, accumulate, bpc);
  }
  if ((e = set_smem_once((const void*)tc::tc_apply_state_kernel<3>, tc::ApplyCfg<3>::kSmem)) != cudaSuccess) return e;
  return launch_pdl(tc::tc_apply_state_kernel<3>, grid, dim3(192), tc::ApplyCfg<3>::kSmem, s, 1, tm, mo, ms[0], m1,
                    m2, m_stride, (__nv_bfloat16*)out, tokens, dim, transpose, 0, bpc);
}

cudaError_t tc_apply_state(const void* x, const float* m, void* out, int64_t slots, int64_t tokens, int dim,
                           int transpose, int accumulate, int sm_count, cudaStream_t s) {
  const void* xs[1] = {x};
  const float* ms[1] = {m};
  return tc_apply_multi(xs, ms, 1, (int64_t)dim * dim, out, slots, tokens, dim, transpose, accumulate, sm_count, s);
}

// Unmasked backward, fused: dM segment states (Q^T dO) and dQ = dO M^T in one pass.
cudaError_t tc_state_apply(const void* x0, const void* x1, const float* m, float* seg_out, void* out, int64_t slots,
                           int64_t tokens, int dim, int nseg, cudaStream_t s) {
  CUtensorMap m0, m1, mo;
  cudaError_t e;
  if ((e = make_tmap_3d(&m0, x0, slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = make_tmap_3d(&m1, x1, slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = make_tmap_3d(&mo, out, slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = set_smem_once((const void*)tc::tc_fused_apply_kernel<0>, tc::kFusedSmem)) != cudaSuccess) return e;
  dim3 grid(nseg, (unsigned)slots);
  return launch_pdl(tc::tc_fused_apply_kernel<0>, grid, dim3(tc::kFusedThreads), tc::kFusedSmem, s, 1, m0, m1, mo, mo,
                    m, seg_out, tokens, dim, nseg, 0);
}

// Unmasked backward dK = V dM^T and dV = K dM in one pass.
cudaError_t tc_apply2(const void* x0, const void* x1, const float* m, void* out0, void* out1, int64_t slots,
                      int64_t tokens, int dim, int sm_count, cudaStream_t s) {
  CUtensorMap m0, m1, mo0, mo1;
  cudaError_t e;
  if ((e = make_tmap_3d(&m0, x0, slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = make_tmap_3d(&m1, x1, slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = make_tmap_3d(&mo0, out0, slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = make_tmap_3d(&mo1, out1, slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = set_smem_once((const void*)tc::tc_fused_apply_kernel<1>, tc::kFusedSmem)) != cudaSuccess) return e;
  const int64_t nblk = (tokens + tc::kTile - 1) / tc::kTile;
  int64_t ctas = sm_count / slots;
  if (ctas < 1) ctas = 1;
  if (ctas > nblk) ctas = nblk;
  const int bpc = (int)((nblk + ctas - 1) / ctas);
  ctas = (nblk + bpc - 1) / bpc;
  dim3 grid((unsigned)ctas, (unsigned)slots);
  return launch_pdl(tc::tc_fused_apply_kernel<1>, grid, dim3(tc::kFusedThreads), tc::kFusedSmem, s, 1, m0, m1, mo0,
                    mo1, m, (float*)nullptr, tokens, dim, 1, bpc);
}

cudaError_t tc_set_trace(unsigned long long* buf) {
  return cudaMemcpyToSymbol(tc::g_trace, &buf, sizeof(buf));
}

cudaError_t tc_probe_gemm(const void* a, const void* b, float* d, int a_mn, int b_mn, cudaStream_t s) {
  CUtensorMap ma, mb;
  cudaError_t e;
  if ((e = make_tmap_3d(&ma, a, 1, 128, 128)) != cudaSuccess) return e;
  if ((e = make_tmap_3d(&mb, b, 1, 128, 128)) != cudaSuccess) return e;
  const uint32_t smem = 2 * tc::kTileBytes + 1024 + 64;
  e = cudaFuncSetAttribute(tc::tc_probe_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  tc::tc_probe_gemm_kernel<<<1, 128, smem, s>>>(ma, mb, d, a_mn, b_mn);
  return cudaGetLastError();
}

}  // namespace lasp
