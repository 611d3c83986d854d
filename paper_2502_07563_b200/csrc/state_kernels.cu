// Ordered state reductions and synthetic-input generation.
//
// scan  : per-rank exclusive prefix / suffix over segment states (the
//         in-GPU analogue of LASP-2's prefix over chunks).
// fold  : reduction of the rank-ordered gathered states with the reference's
//         fold-order contract (numerics.py:71-121): a non-empty fold copies its
//         first term and adds the rest in order (ascending for prefix/full,
//         descending for suffix); an empty fold is zeros.
// gen   : bit-exact SplitMix64 counter-hash port of datagen.gen_data
//         (datagen.py:14-57), so the bench can build 2M-token inputs on device.
#include <type_traits>
#include "kernels.h"
#include "tc_common.cuh"

namespace lasp {

// In place: seg[s] <- sum_{s' < s} seg[s'] (reverse: sum_{s' > s}); total <- sum_all.
// One thread per (slot, element); the segment loop is sequential, so the
// order of additions is fixed (ascending / descending).
template <typename A>
__global__ void scan_states_kernel(A* __restrict__ seg, A* __restrict__ total, int64_t slots, int nseg, int64_t dd,
                                   int reverse) {
  ptx::pdl_wait();
  ptx::pdl_launch_dependents();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= slots * dd) return;
  const int64_t slot = idx / dd, el = idx % dd;
  A* base = seg + slot * nseg * dd + el;
  A run = A(0);
  // batches of 8 independent loads keep the (latency-bound) column walk in flight
  for (int i0 = 0; i0 < nseg; i0 += 8) {
    A vals[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u;
      if (i < nseg) vals[u] = base[(int64_t)(reverse ? nseg - 1 - i : i) * dd];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u;
      if (i < nseg) {
        base[(int64_t)(reverse ? nseg - 1 - i : i) * dd] = run;
        run = (i == 0) ? vals[u] : run + vals[u];
      }
    }
  }
  if (total) total[slot * dd + el] = run;
}

// fp32 scan, four consecutive elements per thread (16-byte loads / stores), same order
__global__ void scan_states_f4_kernel(float4* __restrict__ seg, float4* __restrict__ total, int64_t slots, int nseg,
                                      int64_t dd4, int reverse) {
  ptx::pdl_wait();
  ptx::pdl_launch_dependents();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= slots * dd4) return;
  const int64_t slot = idx / dd4, el = idx % dd4;
  float4* base = seg + slot * nseg * dd4 + el;
  float4 run = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i0 = 0; i0 < nseg; i0 += 8) {
    float4 vals[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u;
      if (i < nseg) vals[u] = __ldcg(base + (int64_t)(reverse ? nseg - 1 - i : i) * dd4);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u;
      if (i < nseg) {
        base[(int64_t)(reverse ? nseg - 1 - i : i) * dd4] = run;
        if (i == 0) {
          run = vals[u];
        } else {
          run.x += vals[u].x;
          run.y += vals[u].y;
          run.z += vals[u].z;
          run.w += vals[u].w;
        }
      }
    }
  }
  if (total) total[slot * dd4 + el] = run;
}

// ---- fused state exchange over peer memory -------------------
// scan_put: the scan above, and the chunk total (this rank's M_t / dM_t, the
// all_gather payload) is stored straight into slot `rank` of every rank's
// receive buffer [2][nranks][slots*dd] (double-buffered by epoch parity) —
// P2P stores over NVLink when the buffers are symmetric-memory peers, plain
// stores in the one-GPU threads world. The last block to finish (device-wide
// counter, re-armed by that block) releases one epoch-stamped flag per rank at
// system scope after a system fence, so a reader that acquires flag[rank]
// sees every element of the slot. Back-pressure: before the put of epoch e the
// caller waits (exchange_wait on its own acks) until every reader has
// acknowledged epoch e-2 (exchange_ack after its fold), so a rank that runs
// ahead (a forward-only loop needs nothing from its successors) never
// clobbers the half another rank has not folded yet. The wait is its own
// one-thread kernel: spinning inside the put's grid could starve the other
// ranks' kernels of SM slots when ranks share one GPU.
// flag / ack words are stored relaxed after one fence.sc.sys by the storing thread (the fence
// and the relaxed stores form the release pattern; st.release.sys would fence once per word)
__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ void wait_epochs(const unsigned long long* flags, int lo, int hi, unsigned long long epoch) {
  for (int j = lo; j < hi; ++j) {
    const long long t0 = clock64();
    while (ld_acquire_sys_u64(flags + j) < epoch) {
      __nanosleep(64);
      if (clock64() - t0 > (1ll << 36)) __trap();  // a peer never arrived: fail loudly, do not hang
    }
  }
}

template <typename A>
__global__ void scan_put_kernel(A* __restrict__ seg, A* __restrict__ total, int64_t slots, int nseg, int64_t dd,
                                int reverse, A* const* __restrict__ peer_recv,
                                unsigned long long* const* __restrict__ peer_flags, int rank, int nranks,
                                unsigned long long epoch, unsigned* __restrict__ done,
                                unsigned long long* __restrict__ epoch_dev) {
  ptx::pdl_wait();
  ptx::pdl_launch_dependents();
  // device-resident epoch (graph replays advance it): this exchange is *epoch_dev + 1, stored
  // back by the last block, after every block has read the old value
  if (epoch_dev != nullptr) epoch = *(volatile unsigned long long*)epoch_dev + 1;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = slots * dd;
  const int64_t off = ((int64_t)(epoch & 1) * nranks + rank) * n;
  if (idx < n) {
    const int64_t slot = idx / dd, el = idx % dd;
    A* base = seg + slot * nseg * dd + el;
    A run = A(0);
    for (int i0 = 0; i0 < nseg; i0 += 8) {
      A vals[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u;
        if (i < nseg) vals[u] = base[(int64_t)(reverse ? nseg - 1 - i : i) * dd];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u;
        if (i < nseg) {
          base[(int64_t)(reverse ? nseg - 1 - i : i) * dd] = run;
          run = (i == 0) ? vals[u] : run + vals[u];
        }
      }
    }
    if (total) total[idx] = run;
    for (int r = 0; r < nranks; ++r) peer_recv[r][off + idx] = run;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(done, 1u) == gridDim.x - 1) {
    *done = 0;  // every block has stored and fenced: re-arm for the next exchange
    if (epoch_dev != nullptr) *epoch_dev = epoch;
    __threadfence_system();
    for (int r = 0; r < nranks; ++r) st_relaxed_sys_u64(peer_flags[r] + rank, epoch);
  }
}

// the epoch a peer kernel works on: the host value, or *epoch_dev + offset (signed)
__device__ __forceinline__ long long effective_epoch(unsigned long long epoch, const unsigned long long* epoch_dev) {
  return epoch_dev != nullptr ? (long long)*(volatile const unsigned long long*)epoch_dev + (long long)epoch
                              : (long long)epoch;
}

// Block until flags[lo..hi) all carry `epoch` (or a later one). One thread; a
// peer that never arrives traps after ~2^36 cycles instead of hanging the GPU.
__global__ void exchange_wait_kernel(const unsigned long long* __restrict__ flags, int lo, int hi,
                                     unsigned long long epoch, const unsigned long long* __restrict__ epoch_dev) {
  const long long e = effective_epoch(epoch, epoch_dev);
  if (e > 0) wait_epochs(flags, lo, hi, (unsigned long long)e);
}

// After this rank's fold of `epoch` (stream order): acks[rank] = epoch on every rank.
__global__ void exchange_ack_kernel(unsigned long long* const* __restrict__ peer_acks, int rank, int nranks,
                                    unsigned long long epoch, const unsigned long long* __restrict__ epoch_dev) {
  const unsigned long long e = (unsigned long long)effective_epoch(epoch, epoch_dev);
  __threadfence_system();
  for (int r = 0; r < nranks; ++r) st_relaxed_sys_u64(peer_acks[r] + rank, e);
}

// fold of the receive half of the current device epoch: recv + (e & 1) * half_elems
template <typename A>
__global__ void exchange_fold_kernel(const A* __restrict__ recv, int64_t half_elems,
                                     const unsigned long long* __restrict__ epoch_dev, A* __restrict__ out,
                                     int nstates, int64_t elems, int mode, int bound) {
  const unsigned long long e = *(volatile const unsigned long long*)epoch_dev;
  const A* gathered = recv + (int64_t)(e & 1) * half_elems;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= elems) return;
  A acc = A(0);
  const int lo = mode == 1 ? bound : 0, hi = mode == 1 ? nstates : (mode == 2 ? nstates : bound);
  if (hi > lo) {
    if (mode == 1) {  // descending from the last (numerics.py:93-116)
      acc = gathered[(int64_t)(hi - 1) * elems + idx];
      for (int i = hi - 2; i >= lo; --i) acc += gathered[(int64_t)i * elems + idx];
    } else {  // ascending from the first (numerics.py:71-90)
      acc = gathered[idx];
      for (int i = 1; i < hi; ++i) acc += gathered[(int64_t)i * elems + idx];
    }
  }
  out[idx] = acc;
}

// gathered: [nstates][elems]. mode 0 = prefix(bound), 1 = suffix(bound), 2 = full.
template <typename A>
__global__ void fold_states_kernel(const A* __restrict__ gathered, A* __restrict__ out, int nstates, int64_t elems,
                                   int mode, int bound) {
  ptx::pdl_wait();
  ptx::pdl_launch_dependents();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= elems) return;
  // the same copy-first order as before, loads in batches of 8 so a fold over T
  // states costs ~T/8 memory latencies instead of T
  A acc = A(0);
  if (mode == 1) {  // suffix: states[bound:], seeded by the last, descending
    if (bound < nstates) {
      acc = gathered[(int64_t)(nstates - 1) * elems + idx];
      for (int i0 = nstates - 2; i0 >= bound; i0 -= 8) {
        A v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 - u >= bound) v[u] = gathered[(int64_t)(i0 - u) * elems + idx];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 - u >= bound) acc += v[u];
      }
    }
  } else {  // prefix: states[:bound], seeded by the first, ascending
    const int upto = mode == 2 ? nstates : bound;
    if (upto > 0) {
      acc = gathered[idx];
      for (int i0 = 1; i0 < upto; i0 += 8) {
        A v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 + u < upto) v[u] = gathered[(int64_t)(i0 + u) * elems + idx];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 + u < upto) acc += v[u];
      }
    }
  }
  out[idx] = acc;
}

// fp32 fold, four consecutive elements per thread (16-byte loads): the same per-element
// order as fold_states_kernel, a quarter of the threads and load instructions
__global__ void fold_states_f4_kernel(const float4* __restrict__ gathered, float4* __restrict__ out, int nstates,
                                      int64_t elems4, int mode, int bound) {
  ptx::pdl_wait();
  ptx::pdl_launch_dependents();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= elems4) return;
  auto add = [](float4& a, const float4& b) {
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
  };
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const int lo = mode == 1 ? bound : 0, hi = mode == 1 ? nstates : (mode == 2 ? nstates : bound);
  if (hi > lo) {
    float4 v[8];
    if (mode == 1) {  // descending from the last
      acc = __ldcg(gathered + (int64_t)(hi - 1) * elems4 + idx);
      for (int i0 = hi - 2; i0 >= lo; i0 -= 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 - u >= lo) v[u] = __ldcg(gathered + (int64_t)(i0 - u) * elems4 + idx);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 - u >= lo) add(acc, v[u]);
      }
    } else {  // ascending from the first
      acc = __ldcg(gathered + idx);
      for (int i0 = 1; i0 < hi; i0 += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 + u < hi) v[u] = __ldcg(gathered + (int64_t)(i0 + u) * elems4 + idx);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 + u < hi) add(acc, v[u]);
      }
    }
  }
  out[idx] = acc;
}

// ---- SplitMix64 (datagen.py:22-27) ----
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = z + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// out[slot][r][c] = 2*u - 1, u = (mix(mix(h0^r)^c) >> 11) * 2^-53,
// h0 = mix(seed ^ tag_word[slot]); the f64 value is rounded once to T.
template <typename T>
__global__ void gen_slots_kernel(uint64_t seed, const uint64_t* __restrict__ tag_words, T* __restrict__ out,
                                 int64_t slots, int64_t rows, int64_t cols, int64_t row0) {
  const int64_t n = slots * rows * cols;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t slot = idx / (rows * cols);
    const int64_t rc = idx % (rows * cols);
    const uint64_t r = (uint64_t)(rc / cols + row0), c = (uint64_t)(rc % cols);
    const uint64_t h0 = mix64(seed ^ tag_words[slot]);
    const uint64_t h = mix64(mix64(h0 ^ r) ^ c);
    const double u = (double)(h >> 11) * 0x1.0p-53;
    const double val = 2.0 * u - 1.0;
    out[idx] = (T)val;
  }
}
template <>
__global__ void gen_slots_kernel<__nv_bfloat16>(uint64_t seed, const uint64_t* __restrict__ tag_words,
                                                __nv_bfloat16* __restrict__ out, int64_t slots, int64_t rows,
                                                int64_t cols, int64_t row0) {
  const int64_t n = slots * rows * cols;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t slot = idx / (rows * cols);
    const int64_t rc = idx % (rows * cols);
    const uint64_t r = (uint64_t)(rc / cols + row0), c = (uint64_t)(rc % cols);
    const uint64_t h0 = mix64(seed ^ tag_words[slot]);
    const uint64_t h = mix64(mix64(h0 ^ r) ^ c);
    const double u = (double)(h >> 11) * 0x1.0p-53;
    // f64 -> f32 -> bf16 (round-to-nearest-even at each step), SURVEY §8d
    out[idx] = __float2bfloat16_rn((float)(2.0 * u - 1.0));
  }
}

template <typename A>
cudaError_t scan_states(void* seg, void* total, int64_t slots, int nseg, int dim, int reverse, cudaStream_t s) {
  const int64_t dd = (int64_t)dim * dim;
  const int64_t n = slots * dd;
  if (std::is_same<A, float>::value && dd % 4 == 0 &&
      ((reinterpret_cast<uintptr_t>(seg) | reinterpret_cast<uintptr_t>(total)) & 15) == 0) {
    const int64_t n4 = n / 4;
    return launch_pdl(scan_states_f4_kernel, dim3((unsigned)((n4 + 127) / 128)), dim3(128), 0, s, 1, (float4*)seg,
                      (float4*)total, slots, nseg, dd / 4, reverse);
  }
  return launch_pdl(scan_states_kernel<A>, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, 1, (A*)seg, (A*)total,
                    slots, nseg, dd, reverse);
}

template <typename A>
cudaError_t scan_put(void* seg, void* total, int64_t slots, int nseg, int dim, int reverse, const void* peer_recv,
                     const void* peer_flags, int rank, int nranks, unsigned long long epoch, unsigned* done,
                     cudaStream_t s, void* epoch_dev) {
  const int64_t dd = (int64_t)dim * dim;
  const int64_t n = slots * dd;
  return launch_pdl(scan_put_kernel<A>, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, 1, (A*)seg, (A*)total,
                    slots, nseg, dd, reverse, (A* const*)peer_recv, (unsigned long long* const*)peer_flags, rank,
                    nranks, epoch, done, (unsigned long long*)epoch_dev);
}

cudaError_t exchange_wait(const void* flags, int lo, int hi, unsigned long long epoch, cudaStream_t s,
                          const void* epoch_dev) {
  if (hi <= lo) return cudaSuccess;
  exchange_wait_kernel<<<1, 1, 0, s>>>((const unsigned long long*)flags, lo, hi, epoch,
                                       (const unsigned long long*)epoch_dev);
  return cudaGetLastError();
}

cudaError_t exchange_ack(const void* peer_acks, int rank, int nranks, unsigned long long epoch, cudaStream_t s,
                         const void* epoch_dev) {
  exchange_ack_kernel<<<1, 1, 0, s>>>((unsigned long long* const*)peer_acks, rank, nranks, epoch,
                                      (const unsigned long long*)epoch_dev);
  return cudaGetLastError();
}

template <typename A>
cudaError_t exchange_fold(const void* recv, int64_t half_elems, const void* epoch_dev, void* out, int nstates,
                          int64_t elems, int mode, int bound, cudaStream_t s) {
  exchange_fold_kernel<A><<<(unsigned)((elems + 255) / 256), 256, 0, s>>>(
      (const A*)recv, half_elems, (const unsigned long long*)epoch_dev, (A*)out, nstates, elems, mode, bound);
  return cudaGetLastError();
}
template cudaError_t exchange_fold<float>(const void*, int64_t, const void*, void*, int, int64_t, int, int,
                                          cudaStream_t);
template cudaError_t exchange_fold<double>(const void*, int64_t, const void*, void*, int, int64_t, int, int,
                                           cudaStream_t);

template <typename A>
cudaError_t fold_states(const void* gathered, void* out, int nstates, int64_t elems, int mode, int bound,
                        cudaStream_t s) {
  if (std::is_same<A, float>::value && elems % 4 == 0 &&
      ((reinterpret_cast<uintptr_t>(gathered) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) {
    const int64_t e4 = elems / 4;
    return launch_pdl(fold_states_f4_kernel, dim3((unsigned)((e4 + 127) / 128)), dim3(128), 0, s, 1,
                      (const float4*)gathered, (float4*)out, nstates, e4, mode, bound);
  }
  return launch_pdl(fold_states_kernel<A>, dim3((unsigned)((elems + 255) / 256)), dim3(256), 0, s, 1,
                    (const A*)gathered, (A*)out, nstates, elems, mode, bound);
}

template <typename T>
cudaError_t gen_slots(uint64_t seed, const uint64_t* tag_words, void* out, int64_t slots, int64_t rows, int64_t cols,
                      int64_t row0, cudaStream_t s) {
  const int64_t n = slots * rows * cols;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  gen_slots_kernel<T><<<(unsigned)blocks, 256, 0, s>>>(seed, tag_words, (T*)out, slots, rows, cols, row0);
  return cudaGetLastError();
}

template cudaError_t scan_states<float>(void*, void*, int64_t, int, int, int, cudaStream_t);
template cudaError_t scan_states<double>(void*, void*, int64_t, int, int, int, cudaStream_t);
template cudaError_t scan_put<float>(void*, void*, int64_t, int, int, int, const void*, const void*, int, int,
                                     unsigned long long, unsigned*, cudaStream_t, void*);
template cudaError_t scan_put<double>(void*, void*, int64_t, int, int, int, const void*, const void*, int, int,
                                      unsigned long long, unsigned*, cudaStream_t, void*);
template cudaError_t fold_states<float>(const void*, void*, int, int64_t, int, int, cudaStream_t);
template cudaError_t fold_states<double>(const void*, void*, int, int64_t, int, int, cudaStream_t);
template cudaError_t gen_slots<float>(uint64_t, const uint64_t*, void*, int64_t, int64_t, int64_t, int64_t, cudaStream_t);
template cudaError_t gen_slots<double>(uint64_t, const uint64_t*, void*, int64_t, int64_t, int64_t, int64_t, cudaStream_t);
template cudaError_t gen_slots<__nv_bfloat16>(uint64_t, const uint64_t*, void*, int64_t, int64_t, int64_t,
                                              int64_t, cudaStream_t);

}  // namespace lasp
