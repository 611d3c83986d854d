// tcgen05 flash-style causal softmax attention for LASP-2H (bf16 in, fp32
// accumulate), sm_100a only.
//
// Queries are the rank's chunk at global rows row_offset + [q0, ...); keys /
// values are the full gathered sequence, read straight from the rank-major
// all_gather layout through a 4-D TMA map {d, row-in-chunk, slot, rank}. Only
// key blocks at or below the diagonal are visited (causal); the diagonal block
// is masked by global position exactly as softmax_probs (oracle.py:111-133).
//
// tc_softmax_fwd2_kernel (forward): two 128-query tiles per CTA, P back
//   to TMEM and O += P V as a TS-mode MMA accumulating in TMEM (see its header).
// tc_softmax_bwd3_kernel (backward): one CTA per 128-key block, keys as the
//   MMA rows, P^T / dS^T back to TMEM for TS-mode dK / dV, dQ reduced into an fp32
//   accumulator with TMA bulk reduce-adds (see its header).
// Output O / l in bf16, LSE (natural log) in fp32.
#include <type_traits>

#include "kernels.h"
#include "tc_common.cuh"

namespace lasp {
namespace tc {

constexpr int kSmFwdThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 softmax (2 per TMEM lane quarter)

struct SmFwdArgs {
  float* lse;
  int64_t qtok;
  int64_t kvtok;
  int64_t chunk;
  int64_t row_offset;
  int dim;
  int causal;
  float scale_log2;  // log2(e) / sqrt(d)
  int64_t kv_start;  // the call's key j is key kv_start + j of the rank-major layout (multiple of 128)
};

__device__ __forceinline__ void kv_coords(int64_t key0, int64_t chunk, int* row, int* rank) {
  *rank = (int)(key0 / chunk);
  *row = (int)(key0 % chunk);
}

// ============================================================================
// Forward, two query tiles per CTA (A = rows [256p, 256p+128), B = the next
// 128). Each tile has its own softmax group of four warps (one query row per
// thread, all 128 key columns: no cross-warp row exchange) and its own TMEM
// S and O; K_j / V_j are loaded once for both tiles. Per key block j:
//   S_t = Q_t K_j^T                      (SS-mode MMA, TMEM)
//   P_t = exp2(S_t*scale*log2e - m_t)    bf16 written back over S_t in TMEM
//   O_t += P_t V_j                       (TS-mode MMA: A = P_t from TMEM)
// The MMA warp interleaves the tiles (PV_A, S_A, PV_B, S_B), so one tile's
// softmax runs while the tensor core works on the other. O stays in TMEM; the
// running max is raised lazily (only when a block max exceeds it by more than
// 2^8), and only then are O rows rescaled in place.
// ============================================================================
constexpr int kF2Ring = 5;
constexpr uint32_t kSmFwd2Smem = (2 + kF2Ring) * kTileBytes + 1024 + 256;
constexpr float kLazyRescale = 8.f;  // log2 of the largest unnormalised P
// Share of the exponentials evaluated by ex2_poly on the FMA pipe: pairs
// i >= kPolyFrom of every 16 columns. Measured at N=32K (profiles/r01b_softmax_poly.log):
// 0 % 1177 TFLOP/s, 25 % 1139, 37.5 % 986, 50 % 885 — the softmax warps are
// issue-bound, not SFU-bound, on sm_100, so the default keeps every exp2 on the SFU.
#ifndef LASP2_POLY_FROM
#define LASP2_POLY_FROM 16
#endif
constexpr int kPolyFrom = LASP2_POLY_FROM;

// 10 warps: three share an SMSP's 16K registers, so 168 per thread is the cap
__global__ void __launch_bounds__(kSmFwdThreads, 1)
    tc_softmax_fwd2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                           SmFwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* qimg = smem;  // [2] Q tiles, reused as O staging at the end
  uint8_t* ring = qimg + 2 * kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + kF2Ring * kTileBytes);
  uint64_t* full = bars;              // [kF2Ring]
  uint64_t* empty = bars + kF2Ring;   // [kF2Ring]
  uint64_t* q_full = bars + 2 * kF2Ring;
  uint64_t* s_full = q_full + 1;   // [2] per tile
  uint64_t* p_ready = q_full + 3;  // [2]
  uint64_t* o_full = q_full + 5;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 7);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = blockIdx.y;
  const int npairs = gridDim.x;
  const int pair = npairs - 1 - (int)blockIdx.x;  // longest (causal) pairs first
  const int ntiles = (int)((a.qtok + kTile - 1) / kTile);
  const bool has_b = 2 * pair + 1 < ntiles;
  auto nkb_of = [&](int tile) {
    const int64_t q0 = (int64_t)tile * kTile;
    const int64_t end = a.causal ? lmin(a.kvtok, a.row_offset + q0 + kTile) : a.kvtok;
    return (int)((end + kTile - 1) / kTile);
  };
  const int nkb_a = nkb_of(2 * pair), nkb_b = has_b ? nkb_of(2 * pair + 1) : 0;
  const int nkb = nkb_a > nkb_b ? nkb_a : nkb_b;
  const int nbox = a.dim > 64 ? 2 : 1;
  const int kfeat = (a.dim + 15) / 16;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kF2Ring; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 7; ++i) mbar_init(&q_full[i], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S_A 0, S_B 128 (P_t over S_t[0,64)), O_A 256, O_B 384
  auto s_col = [](int t) { return 128u * t; };
  auto o_col = [](int t) { return 256u + 128u * t; };

  if (warp == 0) {
    if (elect_one()) {
      prefetch_tmap(&tm_q);
      prefetch_tmap(&tm_k);
      prefetch_tmap(&tm_v);
      mbar_arrive_expect_tx(q_full, (has_b ? 2 : 1) * nbox * kBoxBytes);
      for (int t = 0; t < (has_b ? 2 : 1); ++t)
        for (int bx = 0; bx < nbox; ++bx)
          tma_load_3d(qimg + t * kTileBytes + bx * kBoxBytes, &tm_q, q_full, 64 * bx, (2 * pair + t) * kTile, slot);
      for (int j = 0; j < nkb; ++j) {
        int row, rank;
        kv_coords((int64_t)j * kTile + a.kv_start, a.chunk, &row, &rank);
        for (int w = 0; w < 2; ++w) {
          const int t = 2 * j + w, s = t % kF2Ring, u = t / kF2Ring;
          if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
          uint8_t* dst = ring + s * kTileBytes;
          mbar_arrive_expect_tx(&full[s], nbox * kBoxBytes);
          const CUtensorMap* m = w == 0 ? &tm_k : &tm_v;
          for (int bx = 0; bx < nbox; ++bx) tma_load_4d(dst + bx * kBoxBytes, m, &full[s], 64 * bx, row, slot, rank);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t id_qk = idesc_bf16_f32(128, 128, 0, 0);
    constexpr uint32_t id_pv = idesc_bf16_f32(128, 128, 0, 1);
    Tracer tr(blockIdx.x == 0 && blockIdx.y == 0);
    mbar_wait(q_full, 0);
    for (int j = 0; j <= nkb; ++j) {
      for (int t = 0; t < 2; ++t) {
        const int nkb_t = t ? nkb_b : nkb_a;
        if (j >= 1 && j - 1 < nkb_t) {  // O_t += P_t V_{j-1}
          const int jb = j - 1, tv = 2 * jb + 1, sv = tv % kF2Ring;
          mbar_wait(&p_ready[t], jb & 1);
          mbar_wait(&full[sv], (tv / kF2Ring) & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t va = smem_u32(ring + sv * kTileBytes);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              mma_bf16_ts(tmem + o_col(t), tmem + s_col(t) + kk * 8, desc_mnmajor(va, kk), id_pv,
                          (jb > 0 || kk > 0) ? 1u : 0u);
            mma_commit(&o_full[t]);
            if (t == 1 || jb >= nkb_b) mma_commit(&empty[sv]);  // last reader of V_{j-1}
          }
          __syncwarp();
          if (lane == 0) tr(50 + 2 * t, jb);
        }
        if (j < nkb_t) {  // S_t = Q_t K_j^T (after PV_t(j-1), which read P_t from these columns)
          const int tk = 2 * j, sk = tk % kF2Ring;
          mbar_wait(&full[sk], (tk / kF2Ring) & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t qa = smem_u32(qimg + t * kTileBytes), ka = smem_u32(ring + sk * kTileBytes);
            for (int kk = 0; kk < kfeat; ++kk)
              mma_bf16_ss(tmem + s_col(t), desc_kmajor(qa, kk), desc_kmajor(ka, kk), id_qk, kk > 0);
            mma_commit(&s_full[t]);
            if (t == 1 || j >= nkb_b) mma_commit(&empty[sk]);  // last reader of K_j
          }
          __syncwarp();
          if (lane == 0) tr(51 + 2 * t, j);
        }
      }
    }
    if (lane == 0) tr.flush(0);
  } else {
    // ---------------- softmax groups: warps 2-5 tile A, 6-9 tile B ----------------
    const int t = (warp - 2) >> 2;
    const int nkb_t = t == 0 ? nkb_a : nkb_b;
    const uint32_t qd = warp & 3;
    const uint32_t row = qd * 32 + lane;
    const uint32_t lane_off = (qd * 32) << 16;
    const int gt = threadIdx.x - 64 - 128 * t;  // thread index within the group
    const int64_t q0 = (int64_t)(2 * pair + t) * kTile;
    const int64_t gq = a.row_offset + q0 + row;  // global query position
    const uint32_t ts = tmem + s_col(t) + lane_off, to = tmem + o_col(t) + lane_off;
    float m_run = -INFINITY, l_run = 0.f;
    Tracer tr(blockIdx.x == 0 && blockIdx.y == 0 && gt == 0);
    if (t == 0 || has_b) {
      for (int j = 0; j < nkb_t; ++j) {
        const int64_t k0 = (int64_t)j * kTile;
        int lim = (int)lmin(kTile, a.kvtok - k0);
        if (a.causal) lim = (int)lmin((int64_t)lim, gq - k0 + 1);
        const bool full_blk = __all_sync(0xffffffffu, lim >= kTile);
        mbar_wait(&s_full[t], j & 1);
        tc_fence_after();
        tr(60 + 2 * t, j);
        uint32_t sr[128];
#pragma unroll
        for (int c = 0; c < 128; c += 32) tmem_ld_32x32b_x32(ts + c, *reinterpret_cast<uint32_t(*)[32]>(sr + c));
        tmem_ld_wait();
        // row max as 8 independent chains of 3-input max (two new columns per FMNMX3)
        float mx[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) mx[u] = -INFINITY;
        if (full_blk) {
#pragma unroll
          for (int i = 0; i < 128; i += 2)
            mx[(i >> 1) & 7] = fmax3(mx[(i >> 1) & 7], __uint_as_float(sr[i]), __uint_as_float(sr[i + 1]));
        } else {
#pragma unroll
          for (int i = 0; i < 128; ++i)
            if (i < lim) mx[i & 7] = fmaxf(mx[i & 7], __uint_as_float(sr[i]));
        }
        const float bm = fmaxf(fmax3(mx[0], mx[1], mx[2]), fmax3(fmax3(mx[3], mx[4], mx[5]), mx[6], mx[7]));
        const float mc = bm * a.scale_log2;
        const bool need = mc > m_run + kLazyRescale;
        const float m_new = need ? mc : m_run;
        const float corr = (need && m_run != -INFINITY) ? ex2_approx(m_run - m_new) : (need ? 0.f : 1.f);
        float ps[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // row sum as 4 independent pair chains
        // full blocks (all but the diagonal one) get a mask-free copy of the loop
        auto exp_block = [&](auto full_tag) {
          constexpr bool kFull = decltype(full_tag)::value;
#pragma unroll
        for (int c = 0; c < 128; c += 16) {
          uint32_t pk[8];
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const bool ok0 = kFull || c + i < lim, ok1 = kFull || c + i + 1 < lim;
            float x0, x1;  // x = s * scale * log2(e) - m for two columns in one FFMA2
            ffma2_bc(x0, x1, __uint_as_float(sr[c + i]), __uint_as_float(sr[c + i + 1]), a.scale_log2, -m_new);
            // this share of the exponentials runs on the FMA pipe; evaluated unconditionally
            // and selected after, so the compiler interleaves elements instead of branching
            const bool poly = i >= kPolyFrom;
            const float e0 = poly ? ex2_poly(x0) : ex2_approx(x0);
            const float e1 = poly ? ex2_poly(x1) : ex2_approx(x1);
            const float p0 = ok0 ? e0 : 0.f;
            const float p1 = ok1 ? e1 : 0.f;
            const int ch = 2 * ((i >> 1) & 3);
            fadd2(ps[ch], ps[ch + 1], p0, p1);
            pk[i >> 1] = pack_bf16x2(p0, p1);
          }
          tmem_st_32x32b_x8(ts + (c >> 1), pk);
        }
        };
        if (full_blk)
          exp_block(std::true_type{});
        else
          exp_block(std::false_type{});
        const float psum = ((ps[0] + ps[1]) + (ps[2] + ps[3])) + ((ps[4] + ps[5]) + (ps[6] + ps[7]));
        if (j > 0 && __any_sync(0xffffffffu, need)) {  // raise this warp's rows' max: rescale O in TMEM
          mbar_wait(&o_full[t], (j - 1) & 1);  // PV_t(j-1) complete
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < 128; c += 32) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(to + c, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * corr);
            tmem_st_32x32b_x32(to + c, r);
          }
        }
        l_run = l_run * corr + psum;
        m_run = m_new;
        tmem_st_wait();
        tc_fence_before();
        named_bar_sync(1 + t, 128);
        if (gt == 0) mbar_arrive(&p_ready[t]);
        tr(61 + 2 * t, j);
      }
      tr.flush(1 + t);
      // epilogue: O / l -> bf16 -> staging (this tile's Q image) -> TMA store
      mbar_wait(&o_full[t], (nkb_t - 1) & 1);
      tc_fence_after();
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      uint8_t* stg = qimg + t * kTileBytes;
#pragma unroll 1
      for (int c = 0; c < 128; c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(to + c, r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * inv;
        st_row32_bf16(stg, row, c, v);
      }
      if (q0 + row < a.qtok)
        a.lse[(int64_t)slot * a.qtok + q0 + row] = (m_run + __log2f(l_run)) * 0.69314718055994531f;
      fence_proxy_async_smem();
      named_bar_sync(1 + t, 128);
      if (gt == 0) {
        for (int bx = 0; bx < nbox; ++bx) tma_store_3d(&tm_o, stg + bx * kBoxBytes, 64 * bx, (int)q0, slot);
        tma_store_commit();
        tma_store_wait_all<0>();
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// Shared by the backward kernels below.
constexpr int kSmBwdThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9: one query row x 64 columns each

struct SmBwdArgs {
  const float* lse;    // [slots][qtok] natural log
  const float* delta;  // [slots][qtok]
  float* dq_acc;       // [slots][qtok][dim] fp32, zeroed
  float* dk_full;      // rank-major contributions
  float* dv_full;
  int64_t qtok;
  int64_t kvtok;
  int64_t chunk;
  int64_t grad_rank_stride;
  int64_t row_offset;
  int dim;
  int causal;
  float scale;       // 1/sqrt(d)
  float scale_log2;  // log2(e)/sqrt(d)
  int64_t kv_start;  // as SmFwdArgs::kv_start (dk/dv land at the absolute key)
};

// P and dS of this thread's row (64 columns from c0) as packed bf16 pairs -> SW128 image
__device__ __forceinline__ void store_row64_packed(uint8_t* img, uint32_t row, int c0, const uint32_t* pk) {
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const uint32_t off = sw128_offset(row, c0 + 8 * u);
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(img + off)), "r"(pk[4 * u]),
                 "r"(pk[4 * u + 1]), "r"(pk[4 * u + 2]), "r"(pk[4 * u + 3])
                 : "memory");
  }
}

// ============================================================================
// Backward v3 (default): one CTA per (128-key block, slot) with the KEYS as the
// MMA rows (TMEM lanes), so P^T and dS^T are produced per key row and go back
// to TMEM as the A operands of TS-mode MMAs. Per visible query block i:
//   S^T = K Q_i^T -> R0,  dP^T = V dO_i^T -> R1                 (SS)
//   P^T = exp2(S^T*scale*log2e - lse_i*log2e),  dS^T = P^T o (dP^T - D_i)
//        both bf16 -> R0 (over S^T, columns [64h, 64h+32) / [64h+32, 64h+64) of half h:
//        each column half rewrites only columns it has read) and dS^T also -> smem
//        image [key][query]
//   dQ_i = dS K -> R1  (SS: the image read MN-major as A, K read MN-major as B)
//   dK += dS^T Q_i, dV += P^T dO_i                                (TS: A from R0)
// dQ_i is issued first so that its drain overlaps dK_i / dV_i. dQ_i leaves TMEM
// through the epilogue warps: staged in fp32 (columns 0-63 in their own buffer,
// 64-127 over the dS image, which dQ_i has finished reading) and added into the
// fp32 accumulator with TMA bulk reduce-adds (scattered red.global.add.v4 cost
// 6 ms more at N = 32K). TMEM: R0 [0,128), R1 [128,256), dV [256,384), dK [384,512).
// ============================================================================
constexpr int kQRing3 = 3;  // Q_i, dO_i, Q_{i+1} (dO_{i+1} lands in Q_i's slot once dK_i is done)
constexpr uint32_t kSmBwd3Smem = (2 + kQRing3 + 2) * kTileBytes + 1024 + 256 + 1024;  // + lse2 / delta stats

__global__ void __launch_bounds__(kSmBwdThreads, 1)
    tc_softmax_bwd3_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                           const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                           const __grid_constant__ CUtensorMap tm_dq, SmBwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* kimg = smem;
  uint8_t* vimg = kimg + kTileBytes;
  uint8_t* ring = vimg + kTileBytes;  // [kQRing3]: Q_i, dO_i, Q_{i+1}, ...
  uint8_t* dsimg = ring + kQRing3 * kTileBytes;
  uint8_t* stg = dsimg + kTileBytes;  // dQ columns 0-63 (fp32, two 32-column SW128 boxes)
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg + kTileBytes);
  uint64_t* full = bars;               // [kQRing3]
  uint64_t* empty = bars + kQRing3;    // [kQRing3]
  uint64_t* kv_full = bars + 2 * kQRing3;
  uint64_t* s_full = kv_full + 1;      // S^T_i in R0 (one extra final phase: every MMA complete)
  uint64_t* dp_full = kv_full + 2;     // dP^T_i in R1
  uint64_t* pds_ready = kv_full + 3;   // P^T_i / dS^T_i in R1 and the dS image (one arrival per half)
  uint64_t* dq_full = kv_full + 4;     // dQ_i in R1
  uint64_t* r1_free = kv_full + 5;     // dQ_i read out (one arrival per half)
  uint64_t* r0_free = kv_full + 6;     // S^T_i read out (one arrival per half)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(kv_full + 7);
  // per column half: lse*log2e of its 64 query columns, then delta of the same columns
  float* stats = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);  // [2][128]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = blockIdx.x, slot = blockIdx.y;
  const int64_t k0 = (int64_t)kb * kTile;
  const int nqb_all = (int)((a.qtok + kTile - 1) / kTile);
  int qb0 = 0;
  if (a.causal) {
    const int64_t first = k0 - a.row_offset;  // first local query row that can see key k0
    qb0 = first <= 0 ? 0 : (int)(first / kTile);
    if (first >= a.qtok) qb0 = nqb_all;
  }
  const int nq = nqb_all - qb0;
  const int nbox = a.dim > 64 ? 2 : 1;
  const int kfeat = (a.dim + 15) / 16;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kQRing3; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 7; ++i) mbar_init(&kv_full[i], (i == 3 || i == 5 || i == 6) ? 2 : 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_r0 = tmem, t_r1 = tmem + 128, t_dv = tmem + 256, t_dk = tmem + 384;

  if (warp == 0) {
    if (elect_one() && nq > 0) {
      prefetch_tmap(&tm_q);
      prefetch_tmap(&tm_do);
      int row, rank;
      kv_coords(k0 + a.kv_start, a.chunk, &row, &rank);
      mbar_arrive_expect_tx(kv_full, 2 * nbox * kBoxBytes);
      for (int bx = 0; bx < nbox; ++bx) {
        tma_load_4d(kimg + bx * kBoxBytes, &tm_k, kv_full, 64 * bx, row, slot, rank);
        tma_load_4d(vimg + bx * kBoxBytes, &tm_v, kv_full, 64 * bx, row, slot, rank);
      }
      for (int i = 0; i < nq; ++i) {
        const int qrow = (qb0 + i) * kTile;
        for (int w = 0; w < 2; ++w) {
          const int t = 2 * i + w, s = t % kQRing3, u = t / kQRing3;
          if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
          uint8_t* dst = ring + s * kTileBytes;
          mbar_arrive_expect_tx(&full[s], nbox * kBoxBytes);
          const CUtensorMap* m = w == 0 ? &tm_q : &tm_do;
          for (int bx = 0; bx < nbox; ++bx) tma_load_3d(dst + bx * kBoxBytes, m, &full[s], 64 * bx, qrow, slot);
        }
      }
    }
  } else if (warp == 1) {
    if (nq > 0) {
      constexpr uint32_t id_kk = idesc_bf16_f32(128, 128, 0, 0);  // S^T, dP^T (both K-major)
      constexpr uint32_t id_ts = idesc_bf16_f32(128, 128, 0, 1);  // dK, dV (A in TMEM, B MN-major)
      constexpr uint32_t id_mm = idesc_bf16_f32(128, 128, 1, 1);  // dQ (A = dS image, B = K, both MN-major)
      const uint32_t ka = smem_u32(kimg), va = smem_u32(vimg), dsa = smem_u32(dsimg);
      auto slot_addr = [&](int t) { return smem_u32(ring + (t % kQRing3) * kTileBytes); };
      auto issue_s = [&](int i) {  // S^T_i = K Q_i^T -> R0
        mbar_wait(&full[(2 * i) % kQRing3], ((2 * i) / kQRing3) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t qa = slot_addr(2 * i);
          for (int kk = 0; kk < kfeat; ++kk) mma_bf16_ss(t_r0, desc_kmajor(ka, kk), desc_kmajor(qa, kk), id_kk, kk > 0);
          mma_commit(s_full);
        }
        __syncwarp();
      };
      auto issue_dp = [&](int i) {  // dP^T_i = V dO_i^T -> R1
        mbar_wait(&full[(2 * i + 1) % kQRing3], ((2 * i + 1) / kQRing3) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t doa = slot_addr(2 * i + 1);
          for (int kk = 0; kk < kfeat; ++kk)
            mma_bf16_ss(t_r1, desc_kmajor(va, kk), desc_kmajor(doa, kk), id_kk, kk > 0);
          mma_commit(dp_full);
        }
        __syncwarp();
      };
      Tracer tr;
      mbar_wait(kv_full, 0);
      for (int i = 0; i < nq; ++i) {
        if (lane == 0) tr(10, i);
        issue_s(i);  // R0: after dK_{i-1} / dV_{i-1} (its readers) in issue order
        if (lane == 0) tr(11, i);
        if (i > 0) mbar_wait(r1_free, (i - 1) & 1);  // dQ_{i-1} read out of R1
        issue_dp(i);
        if (lane == 0) tr(12, i);
        mbar_wait(pds_ready, i & 1);
        if (lane == 0) tr(13, i);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t qa = slot_addr(2 * i), doa = slot_addr(2 * i + 1);
          // dQ_i first (into R1, whose dP^T_i the softmax warps have read): its drain overlaps dK / dV
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) mma_bf16_ss(t_r1, desc_mnmajor(dsa, kk), desc_mnmajor(ka, kk), id_mm, kk > 0);
          mma_commit(dq_full);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {  // dK before dV: Q_i's slot (where dO_{i+1} lands) frees earlier
            const uint32_t pc = (uint32_t)((kk >> 2) * 64 + 32 + (kk & 3) * 8);
            mma_bf16_ts(t_dk, t_r0 + pc, desc_mnmajor(qa, kk), id_ts, (i > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&empty[(2 * i) % kQRing3]);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t pc = (uint32_t)((kk >> 2) * 64 + (kk & 3) * 8);
            mma_bf16_ts(t_dv, t_r0 + pc, desc_mnmajor(doa, kk), id_ts, (i > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&empty[(2 * i + 1) % kQRing3]);
          if (i == nq - 1) mma_commit(s_full);  // final phase: dK / dV complete
        }
        __syncwarp();
        if (lane == 0) tr(14, i);
      }
      if (lane == 0) tr.flush(0);
    }
  } else {
    // 8 warps: warp w reads TMEM lanes 32*(w%4) (keys for R0 / R1 scores, queries for dQ)
    // and the column half h = (w-2)/4 (queries of the scores, features of dQ)
    const int h = (warp - 2) >> 2;
    const int qd = warp & 3;
    const int cb = 64 * h;
    const uint32_t row = qd * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    const int eh = threadIdx.x - 64 - 128 * h;
    const uint32_t bar_id = 1 + h;
    const int64_t key = k0 + row;            // this thread's key (score rows)
    const bool key_ok = key < a.kvtok;
    Tracer tr;
    // stats of query block i: thread eh of half h loads lse (eh < 64) or delta (eh >= 64) of
    // column 64h + eh % 64 one block ahead into a register, and stores it into the half's smem
    // row once every thread of the half has finished with the current block's
    float* my_stats = stats + 128 * h;
    auto stat_load = [&](int i) -> float {
      if (i >= nq) return 0.f;
      const int64_t qb = (int64_t)(qb0 + i) * kTile + 64 * h + (eh & 63);
      if (qb >= a.qtok) return 0.f;
      const int64_t idx = (int64_t)slot * a.qtok + qb;
      return eh < 64 ? __ldg(a.lse + idx) * 1.4426950408889634f : __ldg(a.delta + idx);
    };
    // dQ_j out of R1 (this half's 64 features of query row `row`), staged fp32 and reduced:
    // half 0 into stg (after its previous reduce has read it), half 1 over the dS image
    auto drain_dq = [&](int j) {
      mbar_wait(dq_full, j & 1);
      tc_fence_after();
      uint32_t q0[32], q1[32];
      tmem_ld_32x32b_x32(t_r1 + lane_off + cb, q0);
      tmem_ld_32x32b_x32(t_r1 + lane_off + cb + 32, q1);
      tmem_ld_wait();
      tc_fence_before();
      if (h == 0 && j > 0 && eh == 0) tma_store_wait_read<0>();
      named_bar_sync(bar_id, 128);
      if (eh == 0) mbar_arrive(r1_free);
      if (eh == 0 && h == 0) tr(25, j);
      uint8_t* st0 = (h == 0 ? stg : dsimg);
      uint8_t* st1 = st0 + kBoxBytes;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t off = row * 128 + (uint32_t)((u ^ (row & 7)) * 16);
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(st0 + off)),
                     "f"(__uint_as_float(q0[4 * u]) * a.scale), "f"(__uint_as_float(q0[4 * u + 1]) * a.scale),
                     "f"(__uint_as_float(q0[4 * u + 2]) * a.scale), "f"(__uint_as_float(q0[4 * u + 3]) * a.scale)
                     : "memory");
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(st1 + off)),
                     "f"(__uint_as_float(q1[4 * u]) * a.scale), "f"(__uint_as_float(q1[4 * u + 1]) * a.scale),
                     "f"(__uint_as_float(q1[4 * u + 2]) * a.scale), "f"(__uint_as_float(q1[4 * u + 3]) * a.scale)
                     : "memory");
      }
      fence_proxy_async_smem();
      named_bar_sync(bar_id, 128);
      if (eh == 0) {
        const int qrow = (qb0 + j) * kTile;
        if (cb < a.dim) tma_reduce_add_3d(&tm_dq, st0, cb, qrow, slot);
        if (cb + 32 < a.dim) tma_reduce_add_3d(&tm_dq, st1, cb + 32, qrow, slot);
        tma_store_commit();
      }
      if (eh == 0 && h == 0) tr(26, j);
    };
    float nxt = stat_load(0);
    my_stats[eh] = nxt;
    nxt = stat_load(1);
    for (int i = 0; i < nq; ++i) {
      const int64_t qbase = (int64_t)(qb0 + i) * kTile;  // local query row of column 0
      // visible query columns of this key row: [cmin, cmax)
      int cmin = 0;
      if (a.causal) cmin = (int)lmax(0, lmin(kTile, key - a.row_offset - qbase));  // key <= row_offset + query
      const int cmax = key_ok ? (int)lmin(kTile, a.qtok - qbase) : 0;
      // ---- S^T_i -> registers, R0 released for S^T_{i+1}
      mbar_wait(s_full, i & 1);
      if (eh == 0 && h == 0) tr(20, i);
      tc_fence_after();
      uint32_t rs[32], rt[32];
      tmem_ld_32x32b_x32(t_r0 + lane_off + cb, rs);
      tmem_ld_32x32b_x32(t_r0 + lane_off + cb + 32, rt);
      tmem_ld_wait();
      named_bar_sync(bar_id, 128);  // publishes this block's stats (written last iteration)
      // ---- P^T = exp2(S^T * scale*log2e - lse*log2e), this half's 64 query columns; the
      // causal / ragged mask is resolved per warp: rows entirely inside or outside the
      // visible columns skip the per-element tests (only diagonal and tail blocks pay them)
      uint32_t ppk[32];
      const bool all_in = __all_sync(0xffffffffu, cmin <= cb && cmax >= cb + 64);
      const bool all_out = __all_sync(0xffffffffu, cmin >= cb + 64 || cmax <= cb);
      if (all_out) {
#pragma unroll
        for (int e = 0; e < 32; ++e) ppk[e] = 0u;
      } else if (all_in) {
#pragma unroll
        for (int c = 0; c < 64; c += 4) {
          const float4 l4 = *reinterpret_cast<const float4*>(my_stats + c);  // smem broadcast
          const uint32_t* src = c < 32 ? rs + c : rt + (c - 32);
          ppk[c >> 1] = pack_bf16x2(ex2_approx(fmaf(__uint_as_float(src[0]), a.scale_log2, -l4.x)),
                                    ex2_approx(fmaf(__uint_as_float(src[1]), a.scale_log2, -l4.y)));
          ppk[(c >> 1) + 1] = pack_bf16x2(ex2_approx(fmaf(__uint_as_float(src[2]), a.scale_log2, -l4.z)),
                                          ex2_approx(fmaf(__uint_as_float(src[3]), a.scale_log2, -l4.w)));
        }
      } else {
#pragma unroll
        for (int c = 0; c < 64; c += 4) {
          const int col = cb + c;
          const float4 l4 = *reinterpret_cast<const float4*>(my_stats + c);
          const uint32_t* src = c < 32 ? rs + c : rt + (c - 32);
          float p[4];
          const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const bool ok = col + e >= cmin && col + e < cmax;
            p[e] = ok ? ex2_approx(fmaf(__uint_as_float(src[e]), a.scale_log2, -lv[e])) : 0.f;
          }
          ppk[c >> 1] = pack_bf16x2(p[0], p[1]);
          ppk[(c >> 1) + 1] = pack_bf16x2(p[2], p[3]);
        }
      }
      tmem_st_32x32b_x32(t_r0 + lane_off + cb, ppk);  // P^T packed over this half's S^T columns
      if (eh == 0 && h == 0) tr(21, i);
      // ---- dS^T = P^T o (dP^T - D)
      uint32_t dpk[32];
      mbar_wait(dp_full, i & 1);
      if (eh == 0 && h == 0) tr(22, i);
      tc_fence_after();
      tmem_ld_32x32b_x32(t_r1 + lane_off + cb, rs);
      tmem_ld_32x32b_x32(t_r1 + lane_off + cb + 32, rt);
      tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < 64; c += 4) {
        const float4 d4 = *reinterpret_cast<const float4*>(my_stats + 64 + c);
        const uint32_t* src = c < 32 ? rs + c : rt + (c - 32);
        const uint32_t p01 = ppk[c >> 1], p23 = ppk[(c >> 1) + 1];
        const float p0 = __uint_as_float(p01 << 16), p1 = __uint_as_float(p01 & 0xFFFF0000u);
        const float p2 = __uint_as_float(p23 << 16), p3 = __uint_as_float(p23 & 0xFFFF0000u);
        dpk[c >> 1] = pack_bf16x2(p0 * (__uint_as_float(src[0]) - d4.x), p1 * (__uint_as_float(src[1]) - d4.y));
        dpk[(c >> 1) + 1] = pack_bf16x2(p2 * (__uint_as_float(src[2]) - d4.z), p3 * (__uint_as_float(src[3]) - d4.w));
      }
      tmem_st_32x32b_x32(t_r0 + lane_off + cb + 32, dpk);  // dS^T packed next to P^T
      if (eh == 0 && h == 0) tr(27, i);
      // the image's previous readers: dQ_{i-1} (drained last iteration) and half 1's reduce of the
      // dQ_{i-1} columns staged over it
      if (i > 0) {
        if (h == 1 && eh == 0) tma_store_wait_read<0>();
        named_bar_sync(3, 256);
      }
      if (eh == 0 && h == 0) tr(28, i);
      store_row64_packed(dsimg, row, cb, dpk);
      tmem_st_wait();
      fence_proxy_async_smem();
      tc_fence_before();
      named_bar_sync(bar_id, 128);
      if (eh == 0) mbar_arrive(pds_ready);
      if (eh == 0 && h == 0) tr(23, i);
      // block i+1's stats (published by the half barrier before its P phase)
      my_stats[eh] = nxt;
      nxt = stat_load(i + 2);
      drain_dq(i);  // while dK_i / dV_i run
    }
    if (eh == 0) tma_store_wait_all<0>();
    if (eh == 0 && h == 0) tr.flush(1);
    // dK / dV rows of this key block (one key per thread, this half's 64 columns) -> fp32 contributions
    if (nq > 0) mbar_wait(s_full, nq & 1);  // the final commit: every MMA complete
    tc_fence_after();
    if (key_ok) {
      const int64_t ka = key + a.kv_start;
      const int64_t off = (ka / a.chunk) * a.grad_rank_stride + ((int64_t)slot * a.chunk + ka % a.chunk) * a.dim;
      float* dkr = a.dk_full + off;
      float* dvr = a.dv_full + off;
      if (nq == 0) {
        for (int c = cb; c < cb + 64 && c < a.dim; c += 4) {
          *reinterpret_cast<float4*>(dkr + c) = make_float4(0.f, 0.f, 0.f, 0.f);
          *reinterpret_cast<float4*>(dvr + c) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      } else {
#pragma unroll 1
        for (int c0 = cb; c0 < cb + 64; c0 += 32) {
          uint32_t rk[32], rv[32];
          tmem_ld_32x32b_x32(t_dk + lane_off + c0, rk);
          tmem_ld_32x32b_x32(t_dv + lane_off + c0, rv);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            if (c0 + e < a.dim) {
              *reinterpret_cast<float4*>(dkr + c0 + e) =
                  make_float4(__uint_as_float(rk[e]) * a.scale, __uint_as_float(rk[e + 1]) * a.scale,
                              __uint_as_float(rk[e + 2]) * a.scale, __uint_as_float(rk[e + 3]) * a.scale);
              *reinterpret_cast<float4*>(dvr + c0 + e) =
                  make_float4(__uint_as_float(rv[e]), __uint_as_float(rv[e + 1]), __uint_as_float(rv[e + 2]),
                              __uint_as_float(rv[e + 3]));
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

__global__ void dq_finalize_kernel(const float* __restrict__ acc, __nv_bfloat16* __restrict__ dq, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dq[i] = __float2bfloat16_rn(acc[i]);
}

}  // namespace tc

cudaError_t tc_set_trace_softmax(unsigned long long* buf) {
  return cudaMemcpyToSymbol(tc::g_trace, &buf, sizeof(buf));
}

bool tc_softmax_supported(int dim, int64_t kv_chunk) {
  return dim >= 8 && dim <= 128 && dim % 8 == 0 && kv_chunk % 128 == 0;
}

cudaError_t tc_softmax_forward(const void* q, const void* kf, const void* vf, void* out, float* lse, int64_t slots,
                               int64_t qtok, int64_t kvtok, int dim, int causal, int64_t row_offset, int64_t kv_chunk,
                               int64_t kv_rank_stride, cudaStream_t s, int64_t kv_start) {
  CUtensorMap mq, mk, mv, mo;
  cudaError_t e;
  const int64_t ranks = (kv_start + kvtok + kv_chunk - 1) / kv_chunk;
  if ((e = make_tmap_3d(&mq, q, slots, qtok, dim)) != cudaSuccess) return e;
  if ((e = make_tmap_4d(&mk, kf, ranks, slots, kv_chunk, dim, kv_rank_stride)) != cudaSuccess) return e;
  if ((e = make_tmap_4d(&mv, vf, ranks, slots, kv_chunk, dim, kv_rank_stride)) != cudaSuccess) return e;
  if ((e = make_tmap_3d(&mo, out, slots, qtok, dim)) != cudaSuccess) return e;
  tc::SmFwdArgs a{lse, qtok, kvtok, kv_chunk, row_offset, dim, causal, 1.4426950408889634f / sqrtf((float)dim),
                  kv_start};
  if ((e = set_smem_once((const void*)tc::tc_softmax_fwd2_kernel, tc::kSmFwd2Smem)) != cudaSuccess) return e;
  dim3 grid((unsigned)((qtok + 255) / 256), (unsigned)slots);
  tc::tc_softmax_fwd2_kernel<<<grid, tc::kSmFwdThreads, tc::kSmFwd2Smem, s>>>(mq, mk, mv, mo, a);
  return cudaGetLastError();
}

int64_t tc_softmax_bwd_scratch(int64_t slots, int64_t qtok, int dim) {
  return slots * qtok * (dim + 1) * 4 + 256;
}

// scratch: delta [slots][qtok] fp32, dq_acc [slots][qtok][dim] fp32
cudaError_t tc_softmax_backward(const void* q, const void* kf, const void* vf, const void* o, const float* lse,
                                const void* d_out, void* dq, float* dk_full, float* dv_full, void* scratch,
                                int64_t slots, int64_t qtok, int64_t kvtok, int dim, int causal, int64_t row_offset,
                                int64_t kv_chunk, int64_t kv_rank_stride, int64_t grad_rank_stride, cudaStream_t s,
                                int64_t kv_start) {
  float* delta = reinterpret_cast<float*>(scratch);
  float* dq_acc = delta + ((slots * qtok + 63) / 64) * 64;
  cudaError_t e = softmax_delta_bf16(o, d_out, delta, slots * qtok, dim, s);
  if (e != cudaSuccess) return e;
  CUtensorMap mq, mdo, mk, mv;
  const int64_t ranks = (kv_start + kvtok + kv_chunk - 1) / kv_chunk;
  if ((e = make_tmap_3d(&mq, q, slots, qtok, dim)) != cudaSuccess) return e;
  if ((e = make_tmap_3d(&mdo, d_out, slots, qtok, dim)) != cudaSuccess) return e;
  if ((e = make_tmap_4d(&mk, kf, ranks, slots, kv_chunk, dim, kv_rank_stride)) != cudaSuccess) return e;
  if ((e = make_tmap_4d(&mv, vf, ranks, slots, kv_chunk, dim, kv_rank_stride)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(dq_acc, 0, (size_t)slots * qtok * dim * 4, s)) != cudaSuccess) return e;
  tc::SmBwdArgs a{lse, delta, dq_acc, dk_full, dv_full, qtok, kvtok, kv_chunk, grad_rank_stride, row_offset, dim,
                  causal, 1.f / sqrtf((float)dim), 1.4426950408889634f / sqrtf((float)dim), kv_start};
  dim3 grid((unsigned)((kvtok + 127) / 128), (unsigned)slots);
  CUtensorMap mdq;
  if ((e = make_tmap_3d_f32(&mdq, dq_acc, slots, qtok, dim)) != cudaSuccess) return e;
  if ((e = set_smem_once((const void*)tc::tc_softmax_bwd3_kernel, tc::kSmBwd3Smem)) != cudaSuccess) return e;
  tc::tc_softmax_bwd3_kernel<<<grid, tc::kSmBwdThreads, tc::kSmBwd3Smem, s>>>(mq, mdo, mk, mv, mdq, a);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int64_t n = slots * qtok * dim;
  tc::dq_finalize_kernel<<<(unsigned)lmin(148 * 16, (n + 255) / 256), 256, 0, s>>>(dq_acc, (__nv_bfloat16*)dq, n);
  return cudaGetLastError();
}

}  // namespace lasp
