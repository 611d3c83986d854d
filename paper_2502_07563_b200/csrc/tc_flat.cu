// Persistent two-phase kernels of the unmasked LASP-2 layer on a world of one
// rank (T = 1), where the state all_gather is the identity and the whole layer
// is two streaming passes per direction (lasp2.py:208-216, :256-267):
//
//   forward  (KIND 0)  phase 1: M = K^T V             (partial states)
//                      phase 2: O = Q M
//   backward (KIND 1)  phase 1: dM = Q^T dO,  dQ = dO M^T
//                      phase 2: dK = V dM^T,  dV = K dM
//
// The (slot, 128-token block) space is flattened and split evenly over one CTA
// per SM (all 148, not slots x floor(148/slots)); a CTA's range may cross slot
// boundaries, so a phase is a sequence of "pieces" (maximal runs inside one
// slot). Phase 1 leaves one partial state per piece; an in-kernel grid
// barrier, an ordered reduction of the partials (ascending token order, split
// over every thread of the grid) and a second barrier produce the slot totals,
// which phase 2 applies. The TMA warp streams phase-2 tiles into the ring
// while the barriers run, so the phase boundary costs no load ramp and the
// layer needs no scan / fold launches.
//
// Warp roles as in tc_linear.cu: warp 0 TMA, warp 1 MMA (one elected thread),
// warps 2-9 epilogue (two warps per TMEM lane quarter, 64 columns each).
#include <cuda.h>

#include "kernels.h"
#include "tc_common.cuh"

namespace lasp {
namespace tc {

constexpr int kFlatThreads = 320;
constexpr uint32_t kFlatEpi = kFlatThreads - 64;
constexpr int kFlatRing = 4;  // tile slots (a block takes one or two)
constexpr uint32_t kFlatSmem = (kFlatRing + 3) * kTileBytes + 1024 + 512;

struct FlatMaps {
  CUtensorMap p1_in0, p1_in1, p1_out0, p2_in0, p2_in1, p2_out0, p2_out1;
};

struct FlatArgs {
  const float* m_in;  // KIND 1: forward state M [slots][dim][dim] (phase-1 operand)
  float* total;       // phase-1 result = phase-2 state [slots][dim][dim]
  float* part;        // [grid][kmax][dim][dim] per-piece partial states
  unsigned* gbar;     // {arrivals, CTAs past barrier 2}; zero before first use, left reusable
  unsigned* done;     // phase-2 producers finished (reset to 0 by the last one)
  unsigned* ctr;      // [slots] phase-2 blocks handed out per slot (reset to 0 by the last producer)
  int64_t tokens;
  int dim;
  int slots;
  int kmax;
  int phases;  // bit 0: phase 1 + reduction (total = this rank's chunk state); bit 1: phase 2 (state = total)
  FlatXchg x;  // x.nranks > 0 (phases 3): fused peer exchange between the phases, total = the full sum
};

template <int KIND>
struct FlatTraits {
  // phase 1
  static constexpr int p1_nin = 2;
  static constexpr int p1_nout = KIND == 0 ? 0 : 1;
  static constexpr bool p1_img = KIND == 1;
  // phase 2
  static constexpr int p2_nin = KIND == 0 ? 1 : 2;
  static constexpr int p2_nout = KIND == 0 ? 1 : 2;
  // TMEM columns
  __device__ static uint32_t g_col(int g) { return KIND == 0 ? 128u * g : (g ? 384u : 0u); }
  __device__ static uint32_t p1_out(int buf) { return 128u + 128u * buf; }
  __device__ static uint32_t p2_out0(int buf) { return KIND == 0 ? 256u + 128u * buf : 128u * buf; }
  __device__ static uint32_t p2_out1(int buf) { return 256u + 128u * buf; }
};

// Even split of F flat blocks over n CTAs: CTA c owns [flat_lo(c), flat_lo(c + 1)).
__device__ __forceinline__ int64_t flat_lo(int64_t c, int64_t F, int64_t n) { return c * F / n; }

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barriers among the epilogue warps of every CTA (all CTAs are
// co-resident: one per SM, cooperative launch). gbar[0] counts arrivals over
// the launch's barriers (targets n and 2n: one red.add and an acquire spin
// each); gbar[1] counts CTAs past the last barrier of the launch, and the last
// of those re-arms both words for the next launch, off the critical path.
__device__ __forceinline__ void grid_barrier(unsigned* gbar, unsigned target, int et) {
  named_bar_sync(1, kFlatEpi);
  if (et == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gbar) : "memory");
    const long long t0 = clock64();
    while (ld_acquire_u32(gbar) < target) {
      __nanosleep(32);
      if (clock64() - t0 > (1ll << 36)) __trap();  // a CTA never arrived: fail loudly, do not hang
    }
  }
  named_bar_sync(1, kFlatEpi);
}

__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// flag / ack words after ONE fence.sc.sys by the storing thread (fence + relaxed stores form the
// release pattern; st.release.sys per word would pay a system-scope fence each: ~2 us per word)
__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// one thread: every word of w[0..n) reaches `want` (a peer that never arrives traps, not hangs)
__device__ __forceinline__ void wait_words(const unsigned long long* w, int n, unsigned long long want) {
  for (int j = 0; j < n; ++j) {
    const long long t0 = clock64();
    while (ld_acquire_sys_u64(w + j) < want) {
      __nanosleep(64);
      if (clock64() - t0 > (1ll << 36)) __trap();
    }
  }
}

__device__ __forceinline__ void grid_barrier_rearm(unsigned* gbar, unsigned n, int et) {
  if (et == 0 && atomicAdd(gbar + 1, 1u) == n - 1) {  // every CTA has left both barriers
    gbar[0] = 0;
    gbar[1] = 0;
    __threadfence();
  }
}

__device__ __forceinline__ void st_shared_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(smem_u32(p)), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_shared_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

constexpr int kRecs = 16;        // phase-2 block records (producer -> MMA / epilogue)
constexpr unsigned kGrab = 2;    // phase-2 blocks per counter grab

template <int KIND>
__global__ void __launch_bounds__(kFlatThreads, 1) tc_flat_kernel(const __grid_constant__ FlatMaps tm, FlatArgs a) {
  using Tr = FlatTraits<KIND>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint8_t* mimg = ring + kFlatRing * kTileBytes;  // bf16 state image
  uint8_t* stg = mimg + kTileBytes;               // [2] output staging
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg + 2 * kTileBytes);
  uint64_t* full = bars;                       // [kFlatRing]
  uint64_t* empty = bars + kFlatRing;          // [kFlatRing]
  uint64_t* acc_full = bars + 2 * kFlatRing;   // [2]
  uint64_t* acc_empty = acc_full + 2;          // [2]
  uint64_t* g_full = acc_full + 4;             // [2]
  uint64_t* g_empty = acc_full + 6;            // [2]
  uint64_t* m_ready = acc_full + 8;
  uint64_t* recs = acc_full + 9;               // [kRecs] (seq << 32) | flat block (0xffffffff: end)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(recs + kRecs);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nb = (a.tokens + kTile - 1) / kTile;  // blocks per slot
  const int64_t F = nb * a.slots;
  const int64_t f0 = flat_lo(blockIdx.x, F, gridDim.x), f1 = flat_lo(blockIdx.x + 1, F, gridDim.x);
  const int nblk = (int)(f1 - f0);
  const bool run1 = a.phases & 1, run2 = a.phases & 2;
  const int nblk1 = run1 ? nblk : 0;  // phase-1 blocks of this CTA
  const int slot0 = (int)(f0 / nb);
  const int nbox = a.dim > 64 ? 2 : 1;
  const int kfeat = (a.dim + 15) / 16;
  auto piece_start = [&](int b) { return b == 0 || (f0 + b) % nb == 0; };
  auto piece_end = [&](int b) { return b == nblk - 1 || (f0 + b + 1) % nb == 0; };

  if (threadIdx.x == 0) {
    for (int i = 0; i < kFlatRing; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 9; ++i) mbar_init(&acc_full[i], 1);
    for (int i = 0; i < kRecs; ++i) recs[i] = ~0ull;
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    // phase 1: the static range [f0, f1). Phase 2: dynamic — 2-block grabs from a
    // home slot's counter, then from the following slots, until every slot is
    // exhausted (phase-2 blocks are independent, so any CTA computes the same bits).
    if (elect_one()) {
      uint32_t tcount = 0;
      auto slot_wait = [&]() {
        const int s = tcount % kFlatRing;
        const uint32_t u = tcount / kFlatRing;
        if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
        return s;
      };
      auto load = [&](const CUtensorMap* m, int64_t f) {
        const int s = slot_wait();
        uint8_t* dst = ring + s * kTileBytes;
        mbar_arrive_expect_tx(&full[s], nbox * kBoxBytes);
        const int row = (int)((f % nb) * kTile), sl = (int)(f / nb);
        for (int bx = 0; bx < nbox; ++bx) tma_load_3d(dst + bx * kBoxBytes, m, &full[s], 64 * bx, row, sl);
        ++tcount;
      };
      if (run1) {
        prefetch_tmap(&tm.p1_in0);
        prefetch_tmap(&tm.p1_in1);
      }
      for (int b = 0; b < nblk1; ++b) {
        load(&tm.p1_in0, f0 + b);
        load(&tm.p1_in1, f0 + b);
      }
      if (run2) {
        prefetch_tmap(&tm.p2_in0);
        if (Tr::p2_nin > 1) prefetch_tmap(&tm.p2_in1);
        uint32_t seq = 0;
        int s = (int)lmin(((f0 + f1) / 2) / nb, a.slots - 1), exhausted = 0;
        while (exhausted < a.slots) {
          unsigned got = (unsigned)nb;
          if (*(volatile unsigned*)(a.ctr + s) < (unsigned)nb) got = atomicAdd(a.ctr + s, kGrab);
          if (got >= (unsigned)nb) {
            ++exhausted;
            s = s + 1 == a.slots ? 0 : s + 1;
            continue;
          }
          exhausted = 0;  // found work here: the scan restarts after this slot drains
          const unsigned hi = got + kGrab < (unsigned)nb ? got + kGrab : (unsigned)nb;
          for (unsigned j = got; j < hi; ++j) {
            const int64_t f = (int64_t)s * nb + j;
            // the record is visible to whoever waits on this block's first tile
            const int rs = tcount % kFlatRing;
            if (tcount >= kFlatRing) mbar_wait(&empty[rs], ((tcount / kFlatRing) - 1) & 1);
            st_shared_u64(recs + seq % kRecs, ((uint64_t)seq << 32) | (uint32_t)f);
            load(&tm.p2_in0, f);
            if (Tr::p2_nin > 1) load(&tm.p2_in1, f);
            ++seq;
          }
        }
        const int rs = slot_wait();  // end record: one ring position, released by a plain arrive
        st_shared_u64(recs + seq % kRecs, ((uint64_t)seq << 32) | 0xffffffffu);
        mbar_arrive(&full[rs]);
        ++tcount;
        // the last CTA to finish grabbing re-arms the counters for the next launch
        __threadfence();
        if (atomicAdd(a.done, 1u) == gridDim.x - 1) {
          for (int i = 0; i < a.slots; ++i) a.ctr[i] = 0;
          *a.done = 0;
          __threadfence();
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t id_g = idesc_bf16_f32(128, 128, 1, 1);   // X0^T X1 (token contraction)
    constexpr uint32_t id_mt = idesc_bf16_f32(128, 128, 0, 0);  // X M^T
    constexpr uint32_t id_m = idesc_bf16_f32(128, 128, 0, 1);   // X M
    const uint32_t ma = smem_u32(mimg);
    uint32_t tcount = 0, bcount = 0, iv = 0, pc = 0;
    auto wait_tile = [&](uint32_t t) {
      mbar_wait(&full[t % kFlatRing], (t / kFlatRing) & 1);
      return smem_u32(ring + (t % kFlatRing) * kTileBytes);
    };
    auto acc_slot = [&]() {
      const int buf = bcount & 1;
      if (bcount >= 2) mbar_wait(&acc_empty[buf], ((bcount >> 1) - 1) & 1);
      return buf;
    };
    for (int b = 0; b < nblk1; ++b) {
      const bool ps = piece_start(b), pe = piece_end(b);
      const uint32_t x0 = wait_tile(tcount), x1 = wait_tile(tcount + 1);
      if (Tr::p1_img && ps) mbar_wait(m_ready, iv++ & 1);
      if (ps && pc >= 2) mbar_wait(&g_empty[pc & 1], ((pc >> 1) - 1) & 1);
      const int buf = Tr::p1_nout ? acc_slot() : 0;
      tc_fence_after();
      if (elect_one()) {
        const uint32_t g = tmem + Tr::g_col(pc & 1);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_bf16_ss(g, desc_mnmajor(x0, kk), desc_mnmajor(x1, kk), id_g, (!ps || kk > 0) ? 1u : 0u);
        if (Tr::p1_nout)  // KIND 1: dQ = dO M^T
          for (int kk = 0; kk < kfeat; ++kk)
            mma_bf16_ss(tmem + Tr::p1_out(buf), desc_kmajor(x1, kk), desc_kmajor(ma, kk), id_mt, kk > 0);
        mma_commit(&empty[tcount % kFlatRing]);
        mma_commit(&empty[(tcount + 1) % kFlatRing]);
        if (Tr::p1_nout) mma_commit(&acc_full[buf]);
        if (pe) mma_commit(&g_full[pc & 1]);
      }
      __syncwarp();
      tcount += 2;
      if (Tr::p1_nout) ++bcount;
      if (pe) ++pc;
    }
    int cur = -1;
    for (uint32_t b = 0; run2; ++b) {
      const uint32_t x0 = wait_tile(tcount);
      const int f = (int)(uint32_t)ld_shared_u64(recs + b % kRecs);
      if (f < 0) break;
      const uint32_t x1 = Tr::p2_nin > 1 ? wait_tile(tcount + 1) : 0u;
      const int s = (int)(f / nb);
      if (s != cur) {
        mbar_wait(m_ready, iv++ & 1);
        cur = s;
      }
      const int buf = acc_slot();
      tc_fence_after();
      if (elect_one()) {
        if (KIND == 0) {  // O = Q M
          for (int kk = 0; kk < kfeat; ++kk)
            mma_bf16_ss(tmem + Tr::p2_out0(buf), desc_kmajor(x0, kk), desc_mnmajor(ma, kk), id_m, kk > 0);
        } else {  // dK = V dM^T, dV = K dM
          for (int kk = 0; kk < kfeat; ++kk)
            mma_bf16_ss(tmem + Tr::p2_out0(buf), desc_kmajor(x0, kk), desc_kmajor(ma, kk), id_mt, kk > 0);
          for (int kk = 0; kk < kfeat; ++kk)
            mma_bf16_ss(tmem + Tr::p2_out1(buf), desc_kmajor(x1, kk), desc_mnmajor(ma, kk), id_m, kk > 0);
        }
        mma_commit(&empty[tcount % kFlatRing]);
        if (Tr::p2_nin > 1) mma_commit(&empty[(tcount + 1) % kFlatRing]);
        mma_commit(&acc_full[buf]);
      }
      __syncwarp();
      tcount += Tr::p2_nin;
      ++bcount;
    }
  } else {
    // ---------------- epilogue warps ----------------
    const int qd = warp & 3;
    const int cb = 64 * ((warp - 2) >> 2);
    const uint32_t row = qd * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    const int et = threadIdx.x - 64;
    const int dim = a.dim;
    const int64_t dd = (int64_t)dim * dim;
    uint32_t bcount = 0, pc = 0;
    // phase timestamps (globaltimer ns) of every CTA when a debug buffer is set
    unsigned long long* const tbuf = g_trace;
    auto trace = [&](int i) {
      if (tbuf != nullptr && et == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        tbuf[blockIdx.x * 8 + i] = t;
      }
    };
    trace(0);
    // next state, loaded coalesced: unit u = et + 256 i covers image row u >> 5,
    // columns 4 (u & 31) .. +3 (zero outside dim x dim)
    float4 nxt[16];

    auto load_state = [&](const float* src, int sl) {
      const float* p = src + (int64_t)sl * dd;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int u = et + 256 * i, r = u >> 5, c = (u & 31) * 4;
        nxt[i] = (r < dim && c < dim) ? __ldcg(reinterpret_cast<const float4*>(p + (int64_t)r * dim + c))
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    auto build_image = [&]() {  // nxt -> bf16 image, then release the MMA warp
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int u = et + 256 * i, r = u >> 5, c = (u & 31) * 4;
        const uint32_t w0 = pack_bf16x2(nxt[i].x, nxt[i].y), w1 = pack_bf16x2(nxt[i].z, nxt[i].w);
        asm volatile("st.shared.v2.b32 [%0], {%1,%2};" ::"r"(smem_u32(mimg + sw128_offset(r, c))), "r"(w0), "r"(w1)
                     : "memory");
      }
      fence_proxy_async_smem();
      named_bar_sync(1, kFlatEpi);
      if (et == 0) mbar_arrive(m_ready);
    };
    // drain one accumulator (64 of this thread's columns) into a staging image
    auto stage_out = [&](uint32_t col, uint8_t* img) { tmem_cols_to_image<0>(tmem + col + lane_off, img, row, cb, 64); };
    auto store_tile = [&](const CUtensorMap* m, uint8_t* img, int64_t f) {
      const int orow = (int)((f % nb) * kTile), sl = (int)(f / nb);
      for (int bx = 0; bx < nbox; ++bx) tma_store_3d(m, img + bx * kBoxBytes, 64 * bx, orow, sl);
    };

    // ---- phase 1 (static range) ----
    if (Tr::p1_img && nblk1 > 0) {
      load_state(a.m_in, slot0);
      build_image();
      if (slot0 + 1 < a.slots && (f1 - 1) / nb > slot0) load_state(a.m_in, slot0 + 1);
    }
    for (int b = 0; b < nblk1; ++b) {
      const bool pe = piece_end(b);
      if (Tr::p1_nout) {
        const int buf = bcount & 1;
        mbar_wait(&acc_full[buf], (bcount >> 1) & 1);
        tc_fence_after();
        if (Tr::p1_img && pe && b + 1 < nblk) {  // MMAs on the old image are done: swap in the next slot's
          build_image();
          const int nsl = (int)((f0 + b + 1) / nb) + 1;
          if (nsl < a.slots && (f1 - 1) / nb >= nsl) load_state(a.m_in, nsl);
        }
        if (b >= 2 && et == 0) tma_store_wait_read<1>();
        named_bar_sync(1, kFlatEpi);
        uint8_t* st = stg + buf * kTileBytes;
        stage_out(Tr::p1_out(buf), st);
        fence_proxy_async_smem();
        tc_fence_before();
        named_bar_sync(1, kFlatEpi);
        if (et == 0) {
          mbar_arrive(&acc_empty[buf]);
          store_tile(&tm.p1_out0, st, f0 + b);
          tma_store_commit();
        }
        ++bcount;
      }
      if (pe) {  // piece done: G -> part[cta][piece]
        mbar_wait(&g_full[pc & 1], (pc >> 1) & 1);
        tc_fence_after();
        const int k = (int)((f0 + b) / nb) - slot0;
        float* ob = a.part + ((int64_t)blockIdx.x * a.kmax + k) * dd + (int64_t)row * dim;
#pragma unroll 1
        for (int c0 = cb; c0 < cb + 64; c0 += 32) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem + Tr::g_col(pc & 1) + lane_off + c0, r);
          tmem_ld_wait();
          if ((int)row < dim && c0 < dim) {
            if (c0 + 32 <= dim) {
#pragma unroll
              for (int i = 0; i < 32; i += 4)
                *reinterpret_cast<float4*>(ob + c0 + i) = make_float4(
                    __uint_as_float(r[i]), __uint_as_float(r[i + 1]), __uint_as_float(r[i + 2]),
                    __uint_as_float(r[i + 3]));
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (c0 + i < dim) ob[c0 + i] = __uint_as_float(r[i]);
            }
          }
        }
        tc_fence_before();
        named_bar_sync(1, kFlatEpi);
        if (et == 0) mbar_arrive(&g_empty[pc & 1]);
        ++pc;
      }
    }

    // ---- slot totals: ordered sum of the partials over the whole grid ----
    trace(1);
    if (run1) grid_barrier(a.gbar, gridDim.x, et);
    trace(2);
    // fused exchange: this launch's epoch (every CTA reads it before CTA 0 advances it after the
    // last barrier); before storing into the peers' half of this epoch, every reader must have
    // acknowledged the exchange two epochs back (the same half)
    const bool xchg = run1 && run2 && a.x.nranks > 0;
    unsigned long long xe = 0;
    int64_t xoff4 = 0;  // float4 offset of this epoch's half in a receive buffer
    if (xchg) {
      xe = *(volatile const unsigned long long*)a.x.epoch_dev + 1;
      xoff4 = (int64_t)(xe & 1) * a.x.nranks * ((int64_t)a.slots * dd / 4);
      if (et == 0 && xe > 2) wait_words(a.x.acks, a.x.nranks, xe - 2);
      named_bar_sync(1, kFlatEpi);
    }
    if (run1) {
      // slot s = flat blocks [s*nb, (s+1)*nb) is covered by CTAs c_lo..c_hi (every CTA owns
      // >= 1 block since grid <= F); c_lo's piece index is s - slot0(c_lo), later CTAs' is 0.
      // float4 units, ~2 per thread; all partial loads of a unit are issued before the adds.
      const int64_t n = gridDim.x;
      const int64_t nthr = n * kFlatEpi;
      const int64_t E4 = (int64_t)a.slots * dd / 4, dd4 = dd / 4;
      const int64_t cstride = (int64_t)a.kmax * dd4;  // float4s between consecutive CTAs' pieces
      const float4* part4 = reinterpret_cast<const float4*>(a.part);
      // each thread owns units e and e + nthr (~2 per thread at cfg sizes): both units'
      // partial loads are issued before their adds
      auto unit_src = [&](int64_t e, int64_t* c_lo, int64_t* c_hi, int64_t* first) {
        const int s = (int)(e / dd4);
        const int64_t r = e - (int64_t)s * dd4;
        const int64_t fs = (int64_t)s * nb, fe = fs + nb;
        *c_lo = ((fs + 1) * n - 1) / F;
        *c_hi = (fe * n - 1) / F;
        *first = *c_lo * cstride + (s - flat_lo(*c_lo, F, n) / nb) * dd4 + r;
        return r;
      };
      for (int64_t e = (int64_t)blockIdx.x * kFlatEpi + et; e < E4; e += 2 * nthr) {
        const bool two = e + nthr < E4;
        int64_t lo0, hi0, first0, lo1 = 0, hi1 = -1, first1 = 0;
        const int64_t r0 = unit_src(e, &lo0, &hi0, &first0);
        const int64_t r1 = two ? unit_src(e + nthr, &lo1, &hi1, &first1) : 0;
        float4 acc0 = __ldcg(part4 + first0);  // copy-first, ascending (numerics.py:71-90)
        float4 acc1 = two ? __ldcg(part4 + first1) : make_float4(0.f, 0.f, 0.f, 0.f);
        const int64_t span = lmax(hi0 - lo0, hi1 - lo1);
        for (int64_t j0 = 1; j0 <= span; j0 += 8) {
          float4 v0[8], v1[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int64_t c0 = lo0 + j0 + j, c1 = lo1 + j0 + j;
            v0[j] = c0 <= hi0 ? __ldcg(part4 + c0 * cstride + r0) : make_float4(0.f, 0.f, 0.f, 0.f);
            v1[j] = c1 <= hi1 ? __ldcg(part4 + c1 * cstride + r1) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (lo0 + j0 + j <= hi0) {
              acc0.x += v0[j].x;
              acc0.y += v0[j].y;
              acc0.z += v0[j].z;
              acc0.w += v0[j].w;
            }
            if (lo1 + j0 + j <= hi1) {
              acc1.x += v1[j].x;
              acc1.y += v1[j].y;
              acc1.z += v1[j].z;
              acc1.w += v1[j].w;
            }
          }
        }
        reinterpret_cast<float4*>(a.total)[e] = acc0;
        if (two) reinterpret_cast<float4*>(a.total)[e + nthr] = acc1;
        if (xchg) {  // this rank's slot of every rank's receive half: P2P stores over NVLink
          const int64_t mine = xoff4 + (int64_t)a.x.rank * E4;
          for (int r = 0; r < a.x.nranks; ++r) {
            float4* dst = reinterpret_cast<float4*>(a.x.recv_peers[r]) + mine;
            dst[e] = acc0;
            if (two) dst[e + nthr] = acc1;
          }
        }
      }
      if (xchg) {  // every thread's peer stores, then one system-scope fence per CTA (cumulative over
                   // the CTA barrier); the last CTA to get here releases this rank's flag on every rank
        named_bar_sync(1, kFlatEpi);
        if (et == 0) {
          __threadfence_system();
          unsigned* xput = a.gbar + 4;
          if (atomicAdd(xput, 1u) == gridDim.x - 1) {
            *xput = 0;  // re-armed for the next exchange (nobody else touches it in this launch)
            __threadfence_system();
            for (int r = 0; r < a.x.nranks; ++r) st_relaxed_sys_u64(a.x.flag_peers[r] + a.x.rank, xe);
          }
        }
      }
    }
    trace(3);
    if (run1 && run2 && !xchg) grid_barrier(a.gbar, 2 * gridDim.x, et);  // every slot total is complete
    if (xchg) {
      trace(7);  // puts fenced (this rank's flag released by the last CTA)
      // each CTA waits for every rank's flag, folds the full sum over its own elements
      // (ascending, copy-first: numerics.py:119-121, as lasp2_fold_states FULL) into total, and
      // after a grid barrier CTA 0 acknowledges the epoch to every writer and advances the epoch
      if (et == 0) wait_words(a.x.flags, a.x.nranks, xe);
      named_bar_sync(1, kFlatEpi);
      const int64_t E4 = (int64_t)a.slots * dd / 4;
      const float4* rv = reinterpret_cast<const float4*>(a.x.recv) + xoff4;
      const int64_t step = (int64_t)gridDim.x * kFlatEpi;
      // two elements per round, every load of a round issued before its adds (the fold is a few
      // L2 latencies, not one per element and rank)
      for (int64_t e = (int64_t)blockIdx.x * kFlatEpi + et; e < E4; e += 2 * step) {
        const bool two = e + step < E4;
        float4 acc[2];
        acc[0] = __ldcg(rv + e);
        acc[1] = two ? __ldcg(rv + e + step) : make_float4(0.f, 0.f, 0.f, 0.f);
        for (int r0 = 1; r0 < a.x.nranks; r0 += 8) {
          float4 v[2][8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int u = 0; u < 2; ++u)
              v[u][j] = (r0 + j < a.x.nranks && (u == 0 || two))
                            ? __ldcg(rv + (int64_t)(r0 + j) * E4 + e + u * step)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (r0 + j < a.x.nranks) {
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                acc[u].x += v[u][j].x;
                acc[u].y += v[u][j].y;
                acc[u].z += v[u][j].z;
                acc[u].w += v[u][j].w;
              }
            }
          }
        }
        reinterpret_cast<float4*>(a.total)[e] = acc[0];
        if (two) reinterpret_cast<float4*>(a.total)[e + step] = acc[1];
      }
      grid_barrier(a.gbar, 2 * gridDim.x, et);  // every total folded, every read of the half done
      if (blockIdx.x == 0 && et == 0) {
        __threadfence_system();
        for (int r = 0; r < a.x.nranks; ++r) st_relaxed_sys_u64(a.x.ack_peers[r] + a.x.rank, xe);
        *a.x.epoch_dev = xe;
      }
    }
    // re-arm: each CTA counts itself past barrier 1 (and 2, 3), the last resets both words; a
    // phase-1-only launch needs no second barrier (its totals are read by later launches)
    if (run1) grid_barrier_rearm(a.gbar, gridDim.x, et);
    trace(4);

    // ---- phase 2 (dynamic blocks, in the producer's record order) ----
    int cur = -1;
    for (uint32_t b = 0; run2; ++b) {
      uint64_t r;
      while ((uint32_t)((r = ld_shared_u64(recs + b % kRecs)) >> 32) != b) __nanosleep(20);
      const int f = (int)(uint32_t)r;
      if (f < 0) break;
      const int s = (int)(f / nb);
      if (s != cur) {  // the previous block's MMAs are complete (its acc_full was awaited)
        load_state(a.total, s);
        build_image();
        cur = s;
      }
      const int buf = bcount & 1;
      mbar_wait(&acc_full[buf], (bcount >> 1) & 1);
      tc_fence_after();
      if (et == 0) {
        if (Tr::p2_nout == 1 && b >= 2) tma_store_wait_read<1>();
        if (Tr::p2_nout == 2 && b >= 1) tma_store_wait_read<0>();
        if (Tr::p1_nout && b == 0) tma_store_wait_read<0>();  // phase-1 stores still reading staging
      }
      named_bar_sync(1, kFlatEpi);
      if (Tr::p2_nout == 1) {
        stage_out(Tr::p2_out0(buf), stg + buf * kTileBytes);
      } else {
        stage_out(Tr::p2_out0(buf), stg);
        stage_out(Tr::p2_out1(buf), stg + kTileBytes);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      named_bar_sync(1, kFlatEpi);
      if (et == 0) {
        mbar_arrive(&acc_empty[buf]);
        if (Tr::p2_nout == 1) {
          store_tile(&tm.p2_out0, stg + buf * kTileBytes, f);
        } else {
          store_tile(&tm.p2_out0, stg, f);
          store_tile(&tm.p2_out1, stg + kTileBytes, f);
        }
        tma_store_commit();
      }
      ++bcount;
    }
    trace(5);
    if (et == 0) tma_store_wait_all<0>();
    trace(6);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace tc

// ============================================================================
// Host side
// ============================================================================
namespace {

int flat_grid(int64_t slots, int64_t tokens, int sm_count) {
  const int64_t F = slots * ((tokens + tc::kTile - 1) / tc::kTile);
  return (int)lmax(1, lmin(F, sm_count));
}

int flat_kmax(int64_t slots, int64_t tokens, int grid) {
  const int64_t nb = (tokens + tc::kTile - 1) / tc::kTile, F = slots * nb;
  const int64_t bpc = (F + grid - 1) / grid;
  return (int)((bpc + nb - 1) / nb + 1);
}

template <int KIND>
cudaError_t launch_flat(const tc::FlatMaps& tm, const tc::FlatArgs& a, int grid, cudaStream_t s) {
  auto kernel = tc::tc_flat_kernel<KIND>;
  cudaError_t e = set_smem_once((const void*)kernel, tc::kFlatSmem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(tc::kFlatThreads);
  cfg.dynamicSmemBytes = tc::kFlatSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeCooperative;  // grid barrier: every CTA must be resident
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  // phase 2 alone has no grid barrier (dynamic counters, re-armed by the last grabber):
  // a plain launch starts 2-3 us sooner than a cooperative one (C = 16K: 29.4 -> 27.4 us)
  cfg.numAttrs = a.phases == 2 ? 1 : 2;
  return cudaLaunchKernelEx(&cfg, kernel, tm, a);
}

// workspace: [0, 256) barrier words; [256, hdr) per-slot phase-2 counters;
// then partial states [grid][kmax][dim][dim] f32, then a [slots][dim][dim] total
int64_t flat_header(int64_t slots) { return 256 + ((slots * 4 + 255) / 256) * 256; }

tc::FlatArgs flat_args(void* workspace, const float* m_in, float* total, int64_t slots, int64_t tokens, int dim,
                       int grid, int phases = 3, const FlatXchg* x = nullptr) {
  uint8_t* ws = (uint8_t*)workspace;
  const int kmax = flat_kmax(slots, tokens, grid);
  float* part = (float*)(ws + flat_header(slots));
  if (total == nullptr) total = part + (int64_t)grid * kmax * dim * dim;
  return tc::FlatArgs{m_in, total, part, (unsigned*)ws, (unsigned*)ws + 2, (unsigned*)(ws + 256),
                      tokens, dim, (int)slots, kmax, phases,
                      x ? *x : FlatXchg{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0}};
}

}  // namespace

cudaError_t tc_set_trace_flat(unsigned long long* buf) { return cudaMemcpyToSymbol(tc::g_trace, &buf, sizeof(buf)); }

int64_t tc_flat_workspace_bytes(int64_t slots, int64_t tokens, int dim, int sm_count) {
  const int grid = flat_grid(slots, tokens, sm_count);
  const int64_t dd = (int64_t)dim * dim;
  return flat_header(slots) + ((int64_t)grid * flat_kmax(slots, tokens, grid) + slots) * dd * (int64_t)sizeof(float);
}

// Unmasked forward of one rank of a world of one: m_full = K^T V, O = Q m_full.
// phases 1 / 2 split it around a state all_gather (T > 1): phase 1 writes this
// rank's chunk state K^T V to m_full; phase 2 computes O = Q m_full from the
// folded state the caller put there.
cudaError_t tc_flat_forward(const void* q, const void* k, const void* v, void* out, float* m_full, void* workspace,
                            int64_t slots, int64_t tokens, int dim, int sm_count, cudaStream_t s, int phases,
                            const FlatXchg* x) {
  tc::FlatMaps tm;
  cudaError_t e;
  // a phase-only call leaves the other phase's tensors null: their maps are never used,
  // so they alias a tensor that is present
  const void* any = k ? k : q;
  if (!k) k = any;
  if (!v) v = any;
  if (!q) q = any;
  if (!out) out = const_cast<void*>(any);
  if ((e = make_tmap_3d(&tm.p1_in0, k, slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = make_tmap_3d(&tm.p1_in1, v, slots, tokens, dim)) != cudaSuccess) return e;
  tm.p1_out0 = tm.p1_in0;  // unused
  if ((e = make_tmap_3d(&tm.p2_in0, q, slots, tokens, dim)) != cudaSuccess) return e;
  tm.p2_in1 = tm.p2_in0;  // unused
  if ((e = make_tmap_3d(&tm.p2_out0, out, slots, tokens, dim)) != cudaSuccess) return e;
  tm.p2_out1 = tm.p2_out0;  // unused
  const int grid = flat_grid(slots, tokens, sm_count);
  return launch_flat<0>(tm, flat_args(workspace, nullptr, m_full, slots, tokens, dim, grid, phases, x), grid, s);
}

// Unmasked backward of one rank of a world of one:
// dM = Q^T dO, dQ = dO M^T, dK = V dM^T, dV = K dM (dM kept in the workspace, or in
// dm when given). phases 1 / 2 split it around the dM all_gather: phase 1 writes dQ
// and this rank's Q^T dO to dm; phase 2 computes dK, dV from the folded dm.
cudaError_t tc_flat_backward(const void* q, const void* k, const void* v, const void* d_out, const float* m_full,
                             void* dq, void* dk, void* dv, void* workspace, int64_t slots, int64_t tokens, int dim,
                             int sm_count, cudaStream_t s, float* dm, int phases, const FlatXchg* x) {
  tc::FlatMaps tm;
  cudaError_t e;
  const void* any = q ? q : v;  // phase-only calls: see tc_flat_forward
  if (!q) q = any;
  if (!d_out) d_out = any;
  if (!dq) dq = const_cast<void*>(any);
  if (!v) v = any;
  if (!k) k = any;
  if (!dk) dk = const_cast<void*>(any);
  if (!dv) dv = const_cast<void*>(any);
  if ((e = make_tmap_3d(&tm.p1_in0, q, slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = make_tmap_3d(&tm.p1_in1, d_out, slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = make_tmap_3d(&tm.p1_out0, dq, slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = make_tmap_3d(&tm.p2_in0, v, slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = make_tmap_3d(&tm.p2_in1, k, slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = make_tmap_3d(&tm.p2_out0, dk, slots, tokens, dim)) != cudaSuccess) return e;
  if ((e = make_tmap_3d(&tm.p2_out1, dv, slots, tokens, dim)) != cudaSuccess) return e;
  const int grid = flat_grid(slots, tokens, sm_count);
  return launch_flat<1>(tm, flat_args(workspace, m_full, dm, slots, tokens, dim, grid, phases, x), grid, s);
}

}  // namespace lasp
