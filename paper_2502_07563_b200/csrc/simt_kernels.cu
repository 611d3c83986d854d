// Validation-mode kernels (CUDA cores, exact fp32 / fp64 FMA arithmetic).
//
// These implement the same host-level algorithm as the tcgen05 fast path
// (segment states -> ordered scan -> gathered-state fold -> chunk kernel) so
// the host program is identical across precisions; only the arithmetic unit
// differs. fp64 inputs reproduce the reference's own f64 tolerances
// (pkg/tests/test_lasp2.py:17-19); fp32 is the north star's "fp32 validation
// mode" (<=1e-4 normalised). They also serve bf16 shapes the tensor-core
// kernels do not cover (dim not in {64,128}).
#include "common.cuh"
#include "kernels.h"

namespace lasp {

constexpr int kSimtThreads = 256;
constexpr int kSimtBT = 16;  // tokens per sub-block inside a segment

// ---------------------------------------------------------------------------
// seg_states[slot][seg][a][c] = sum_{i in seg} x[i][a] * y[i][c]
// (reference chunk_state lasp2.py:130-137 / chunk_state_grad lasp2.py:140-147,
// restricted to one segment of the rank's chunk).
// ---------------------------------------------------------------------------
template <typename T, typename A>
__global__ void __launch_bounds__(kSimtThreads) simt_segment_states_kernel(const T* __restrict__ x,
                                                                           const T* __restrict__ y,
                                                                           A* __restrict__ out, int64_t tokens,
                                                                           int dim, int nseg) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* xs = reinterpret_cast<A*>(smem_raw);
  A* ys = xs + kSimtBT * dim;
  const int seg = blockIdx.x;
  const int64_t slot = blockIdx.y;
  int64_t lo, hi;
  seg_range(seg, nseg, tokens, &lo, &hi);
  const T* xb = x + slot * tokens * dim;
  const T* yb = y + slot * tokens * dim;
  A* ob = out + (slot * nseg + seg) * (int64_t)dim * dim;
  const int dd = dim * dim;
  const int per = (dd + kSimtThreads - 1) / kSimtThreads;
  // Each thread owns up to 64 accumulators (dim <= 128 -> dd/256 <= 64).
  A acc[64];
#pragma unroll
  for (int e = 0; e < 64; ++e) acc[e] = A(0);
  for (int64_t t0 = lo; t0 < hi; t0 += kSimtBT) {
    const int n = (int)lmin(kSimtBT, hi - t0);
    for (int idx = threadIdx.x; idx < kSimtBT * dim; idx += blockDim.x) {
      const int r = idx / dim, c = idx % dim;
      xs[idx] = r < n ? load_as<A>(xb + (t0 + r) * dim + c) : A(0);
      ys[idx] = r < n ? load_as<A>(yb + (t0 + r) * dim + c) : A(0);
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 64; ++e) {
      if (e >= per) break;
      const int el = threadIdx.x + e * kSimtThreads;
      if (el < dd) {
        const int a = el / dim, c = el % dim;
        A s = acc[e];
        for (int r = 0; r < n; ++r) s += xs[r * dim + a] * ys[r * dim + c];
        acc[e] = s;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int e = 0; e < 64; ++e) {
    if (e >= per) break;
    const int el = threadIdx.x + e * kSimtThreads;
    if (el < dd) ob[el] = acc[e];
  }
}

// ---------------------------------------------------------------------------
// Causal linear attention over one rank's chunk, segment-parallel.
//   forward : out_s = q_s S_s + sum_{i<=s, i in seg} (q_s.k_i) v_i
//             S_s  = base + seg_states[seg] + sum_{i<s in seg} k_i^T v_i
//   reverse : same with i>=s and the state running from the segment's end.
// transpose_state loads S^T instead of S (used by the dQ / dK passes).
// (reference causal_linear_forward oracle.py:50-62; intra + inter split
// lasp2.py:219-243; backward identities oracle.py:77-108.)
// ---------------------------------------------------------------------------
template <typename T, typename A>
__global__ void __launch_bounds__(kSimtThreads) simt_causal_chunk_kernel(
    const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v, const A* __restrict__ seg_states,
    const A* __restrict__ base, T* __restrict__ out, int64_t tokens, int dim, int nseg, int reverse,
    int transpose_state) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* S = reinterpret_cast<A*>(smem_raw);      // [dim][dim]
  A* qs = S + dim * dim;                      // [BT][dim]
  A* ks = qs + kSimtBT * dim;                 // [BT][dim]
  A* vs = ks + kSimtBT * dim;                 // [BT][dim]
  A* sc = vs + kSimtBT * dim;                 // [BT][BT]
  const int seg = blockIdx.x;
  const int64_t slot = blockIdx.y;
  int64_t lo, hi;
  seg_range(seg, nseg, tokens, &lo, &hi);
  const int dd = dim * dim;
  const A* st = seg_states ? seg_states + (slot * nseg + seg) * (int64_t)dd : nullptr;
  const A* bs = base ? base + slot * (int64_t)dd : nullptr;
  for (int el = threadIdx.x; el < dd; el += blockDim.x) {
    const int a = el / dim, c = el % dim;
    const int src = transpose_state ? c * dim + a : el;
    A s = A(0);
    if (bs) s += bs[src];
    if (st) s += st[src];
    S[el] = s;
  }
  const int64_t off = slot * tokens * dim;
  const int64_t nsub = (hi - lo + kSimtBT - 1) / kSimtBT;
  for (int64_t sb = 0; sb < nsub; ++sb) {
    const int64_t t0 = reverse ? lo + (nsub - 1 - sb) * kSimtBT : lo + sb * kSimtBT;
    const int n = (int)lmin(kSimtBT, hi - t0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < kSimtBT * dim; idx += blockDim.x) {
      const int r = idx / dim, c = idx % dim;
      const bool ok = r < n;
      const int64_t g = off + (t0 + r) * dim + c;
      qs[idx] = ok ? load_as<A>(q + g) : A(0);
      ks[idx] = ok ? load_as<A>(k + g) : A(0);
      vs[idx] = ok ? load_as<A>(v + g) : A(0);
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < kSimtBT * kSimtBT; idx += blockDim.x) {
      const int s = idx / kSimtBT, i = idx % kSimtBT;
      const bool keep = reverse ? (i >= s) : (i <= s);
      A acc = A(0);
      if (keep)
        for (int a = 0; a < dim; ++a) acc += qs[s * dim + a] * ks[i * dim + a];
      sc[idx] = acc;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < kSimtBT * dim; idx += blockDim.x) {
      const int s = idx / dim, c = idx % dim;
      if (s >= n) continue;
      A inter = A(0);
      for (int a = 0; a < dim; ++a) inter += qs[s * dim + a] * S[a * dim + c];
      A intra = A(0);
      for (int i = 0; i < kSimtBT; ++i) intra += sc[s * kSimtBT + i] * vs[i * dim + c];
      store_as<T, A>(out + off + (t0 + s) * dim + c, intra + inter);
    }
    __syncthreads();
    for (int el = threadIdx.x; el < dd; el += blockDim.x) {
      const int a = el / dim, c = el % dim;
      A s = S[el];
      for (int r = 0; r < n; ++r) s += ks[r * dim + a] * vs[r * dim + c];
      S[el] = s;
    }
  }
}

// out = x M (transpose=0) or x M^T (transpose=1), optionally += out.
// (reference apply_state / apply_state_t, lasp2.py:150-165)
template <typename T, typename A>
__global__ void __launch_bounds__(kSimtThreads) simt_apply_state_kernel(const T* __restrict__ x,
                                                                        const A* __restrict__ m, T* out,
                                                                        int64_t tokens, int dim, int transpose,
                                                                        int accumulate, int64_t m_stride) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* M = reinterpret_cast<A*>(smem_raw);  // [dim][dim] as used: M[a][c]
  A* xs = M + dim * dim;                  // [BT][dim]
  const int64_t slot = blockIdx.y;
  const int dd = dim * dim;
  const A* mb = m + slot * m_stride;  // m_stride 0: one weight shared by every slot
  for (int el = threadIdx.x; el < dd; el += blockDim.x) {
    const int a = el / dim, c = el % dim;
    M[el] = transpose ? mb[c * dim + a] : mb[el];
  }
  const int64_t off = slot * tokens * dim;
  for (int64_t t0 = (int64_t)blockIdx.x * kSimtBT * 8; t0 < lmin(tokens, ((int64_t)blockIdx.x + 1) * kSimtBT * 8);
       t0 += kSimtBT) {
    const int n = (int)lmin(kSimtBT, tokens - t0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < kSimtBT * dim; idx += blockDim.x) {
      const int r = idx / dim, c = idx % dim;
      xs[idx] = r < n ? load_as<A>(x + off + (t0 + r) * dim + c) : A(0);
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < n * dim; idx += blockDim.x) {
      const int s = idx / dim, c = idx % dim;
      A acc = A(0);
      for (int a = 0; a < dim; ++a) acc += xs[s * dim + a] * M[a * dim + c];
      T* o = out + off + (t0 + s) * dim + c;
      if (accumulate) acc += load_as<A>(o);
      store_as<T, A>(o, acc);
    }
  }
}

// ---------------------------------------------------------------------------
// Softmax attention for one chunk of queries against full-length keys/values
// (reference softmax_probs / softmax_chunk_forward / softmax_chunk_backward,
// oracle.py:111-158). One CTA per query row; online softmax with an fp32/fp64
// running max. lse[row] = max + log(sum) of the scaled scores.
// ---------------------------------------------------------------------------
template <typename A> __device__ __forceinline__ A dev_exp(A x);
template <> __device__ __forceinline__ float dev_exp<float>(float x) { return expf(x); }
template <> __device__ __forceinline__ double dev_exp<double>(double x) { return exp(x); }
template <typename A> __device__ __forceinline__ A dev_log(A x);
template <> __device__ __forceinline__ float dev_log<float>(float x) { return logf(x); }
template <> __device__ __forceinline__ double dev_log<double>(double x) { return log(x); }
template <typename A> __device__ __forceinline__ A dev_rsqrt(int d);
template <> __device__ __forceinline__ float dev_rsqrt<float>(int d) { return 1.0f / sqrtf((float)d); }
template <> __device__ __forceinline__ double dev_rsqrt<double>(int d) { return 1.0 / sqrt((double)d); }

template <typename A>
__device__ __forceinline__ A block_reduce_sum(A v, A* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  A t = A(0);
  if (threadIdx.x < (blockDim.x >> 5)) t = red[threadIdx.x];
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  A r = red[0];
  __syncthreads();
  return r;
}
template <typename A>
__device__ __forceinline__ A block_reduce_max(A v, A* red) {
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  A t = -INFINITY;
  if (threadIdx.x < (blockDim.x >> 5)) t = red[threadIdx.x];
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1) t = max(t, __shfl_xor_sync(0xffffffffu, t, o));
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  A r = red[0];
  __syncthreads();
  return r;
}

// Full-length key/value tensors may be stored rank-major, exactly as the
// collectives produce them: key j of slot lives at
//   (j / chunk) * rank_stride + slot * chunk * dim + (j % chunk) * dim.
// chunk == kvtok with rank_stride == 0 is the plain [slots][kvtok][dim] layout.
// `start` offsets a key range inside that layout: the call's key j is key start + j.
struct KvLayout {
  int64_t chunk;
  int64_t rank_stride;
  int64_t start;
  __device__ __forceinline__ int64_t row(int64_t slot, int64_t j, int dim) const {
    const int64_t a = j + start;
    return (a / chunk) * rank_stride + (slot * chunk + (a % chunk)) * dim;
  }
};

constexpr int kSmThreads = 128;
constexpr int kSmKeys = 128;  // keys scored per pass (one per thread)

template <typename T, typename A>
__global__ void __launch_bounds__(kSmThreads) simt_softmax_fwd_kernel(const T* __restrict__ q,
                                                                      const T* __restrict__ kf,
                                                                      const T* __restrict__ vf, T* __restrict__ out,
                                                                      A* __restrict__ lse, int64_t qtok,
                                                                      int64_t kvtok, int dim, int causal,
                                                                      int64_t row_offset, KvLayout kl) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* qrow = reinterpret_cast<A*>(smem_raw);  // [dim]
  A* p = qrow + dim;                         // [kSmKeys]
  A* red = p + kSmKeys;                      // [32]
  const int64_t row = blockIdx.x, slot = blockIdx.y;
  const T* qb = q + (slot * qtok + row) * dim;
  for (int c = threadIdx.x; c < dim; c += blockDim.x) qrow[c] = load_as<A>(qb + c);
  __syncthreads();
  const A scale = dev_rsqrt<A>(dim);
  const int64_t limit = causal ? lmin(kvtok, row_offset + row + 1) : kvtok;
  A run_max = -INFINITY, run_sum = A(0);
  // each thread accumulates output columns c = threadIdx.x + j*blockDim.x (dim <= 128 -> 1 column)
  A acc = A(0);
  for (int64_t j0 = 0; j0 < limit; j0 += kSmKeys) {
    const int n = (int)lmin(kSmKeys, limit - j0);
    A s = -INFINITY;
    if (threadIdx.x < n) {
      const T* kr = kf + kl.row(slot, j0 + threadIdx.x, dim);
      A d = A(0);
      for (int a = 0; a < dim; ++a) d += qrow[a] * load_as<A>(kr + a);
      s = d * scale;
    }
    const A m_new = max(run_max, block_reduce_max<A>(s, red));
    const A e = threadIdx.x < n ? dev_exp<A>(s - m_new) : A(0);
    p[threadIdx.x] = e;
    const A corr = run_max == -INFINITY ? A(0) : dev_exp<A>(run_max - m_new);
    const A bsum = block_reduce_sum<A>(e, red);
    run_sum = run_sum * corr + bsum;
    run_max = m_new;
    if (threadIdx.x < dim) {
      A a2 = acc * corr;
      for (int j = 0; j < n; ++j) a2 += p[j] * load_as<A>(vf + kl.row(slot, j0 + j, dim) + threadIdx.x);
      acc = a2;
    }
    __syncthreads();
  }
  if (threadIdx.x < dim) store_as<T, A>(out + (slot * qtok + row) * dim + threadIdx.x, acc / run_sum);
  if (threadIdx.x == 0) lse[slot * qtok + row] = run_max + dev_log<A>(run_sum);  // f64 data: f64 lse
}

// delta[row] = sum_c dO[row][c] * O[row][c]  (== rowsum(dP o P), oracle.py:155)
template <typename T, typename A>
__global__ void simt_softmax_delta_kernel(const T* __restrict__ o, const T* __restrict__ d_out, A* __restrict__ delta,
                                          int64_t rows, int dim) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.y + threadIdx.y;
  if (r >= rows) return;
  A s = A(0);
  for (int c = threadIdx.x; c < dim; c += 32) s += load_as<A>(o + r * dim + c) * load_as<A>(d_out + r * dim + c);
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (threadIdx.x == 0) delta[r] = s;
}

// probabilities recomputed from the saved log-sum-exp (fp32 lse for all precisions
// would lose f64 accuracy, so the f64 path recomputes the row statistics exactly).
template <typename T, typename A>
__device__ __forceinline__ void row_stats(const A* qrow, const T* kf, int64_t slot, KvLayout kl, int64_t limit,
                                          int dim, A scale, A* red, A* out_max, A* out_sum) {
  A m = -INFINITY;
  for (int64_t j = threadIdx.x; j < limit; j += blockDim.x) {
    const T* kr = kf + kl.row(slot, j, dim);
    A d = A(0);
    for (int a = 0; a < dim; ++a) d += qrow[a] * load_as<A>(kr + a);
    m = max(m, d * scale);
  }
  m = block_reduce_max<A>(m, red);
  A s = A(0);
  for (int64_t j = threadIdx.x; j < limit; j += blockDim.x) {
    const T* kr = kf + kl.row(slot, j, dim);
    A d = A(0);
    for (int a = 0; a < dim; ++a) d += qrow[a] * load_as<A>(kr + a);
    s += dev_exp<A>(d * scale - m);
  }
  s = block_reduce_sum<A>(s, red);
  *out_max = m;
  *out_sum = s;
}

// delta[row] = sum_j P[row][j] dP[row][j], dP[row][j] = dO[row] . v_j, exactly
// as the reference forms it (oracle.py:155). Equal to dO . O in exact
// arithmetic, but when |dP| is large next to dP - delta (deep stacks of
// unnormalised linear layers feeding a softmax layer) the two roundings differ
// far beyond f64 tolerance, so the f32/f64 validation path keeps the
// reference's grouping. P comes from the exact row statistics (mx, sm).
template <typename T, typename A>
__global__ void __launch_bounds__(kSmThreads) simt_softmax_delta_exact_kernel(
    const T* __restrict__ q, const T* __restrict__ kf, const T* __restrict__ vf, const T* __restrict__ d_out,
    const A* __restrict__ mx, const A* __restrict__ sm, A* __restrict__ delta, int64_t qtok, int64_t kvtok, int dim,
    int causal, int64_t row_offset, KvLayout kl) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* qrow = reinterpret_cast<A*>(smem_raw);  // [dim]
  A* drow = qrow + dim;                      // [dim]
  A* red = drow + dim;                       // [32]
  const int64_t row = blockIdx.x, slot = blockIdx.y, r = slot * qtok + row;
  for (int c = threadIdx.x; c < dim; c += blockDim.x) {
    qrow[c] = load_as<A>(q + r * dim + c);
    drow[c] = load_as<A>(d_out + r * dim + c);
  }
  __syncthreads();
  const A scale = dev_rsqrt<A>(dim), m = mx[r], ssum = sm[r];
  const int64_t limit = causal ? lmin(kvtok, row_offset + row + 1) : kvtok;
  A acc = A(0);
  for (int64_t j = threadIdx.x; j < limit; j += blockDim.x) {
    const T* kr = kf + kl.row(slot, j, dim);
    const T* vr = vf + kl.row(slot, j, dim);
    A sdot = A(0), dp = A(0);
    for (int a = 0; a < dim; ++a) {
      sdot += qrow[a] * load_as<A>(kr + a);
      dp += drow[a] * load_as<A>(vr + a);
    }
    acc += dev_exp<A>(sdot * scale - m) / ssum * dp;
  }
  acc = block_reduce_sum<A>(acc, red);
  if (threadIdx.x == 0) delta[r] = acc;
}

// Row statistics from the forward's log-sum-exp (max = lse, sum = 1): P over a key
// sub-range normalised by the whole key set, as the balanced LASP-2H schedule needs.
template <typename A>
__global__ void stats_from_lse_kernel(const A* __restrict__ lse, A* __restrict__ mx, A* __restrict__ sm, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    mx[i] = lse[i];
    sm[i] = A(1);
  }
}

// dq[row] = scale * sum_j dS[row][j] k_j, dS = P (dP - delta)   (oracle.py:150-157)
template <typename T, typename A>
__global__ void __launch_bounds__(kSmThreads) simt_softmax_bwd_dq_kernel(
    const T* __restrict__ q, const T* __restrict__ kf, const T* __restrict__ vf, const T* __restrict__ d_out,
    const A* __restrict__ delta, T* __restrict__ dq, int64_t qtok, int64_t kvtok, int dim, int causal,
    int64_t row_offset, KvLayout kl, const A* __restrict__ mx_in, const A* __restrict__ sm_in) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* qrow = reinterpret_cast<A*>(smem_raw);
  A* dorow = qrow + dim;
  A* ds = dorow + dim;  // [kSmKeys]
  A* red = ds + kSmKeys;
  const int64_t row = blockIdx.x, slot = blockIdx.y;
  for (int c = threadIdx.x; c < dim; c += blockDim.x) {
    qrow[c] = load_as<A>(q + (slot * qtok + row) * dim + c);
    dorow[c] = load_as<A>(d_out + (slot * qtok + row) * dim + c);
  }
  __syncthreads();
  const A scale = dev_rsqrt<A>(dim);
  const int64_t limit = causal ? lmin(kvtok, row_offset + row + 1) : kvtok;
  A mx, sm;
  if (mx_in != nullptr) {  // statistics of the full key set (a key sub-range of a larger softmax)
    mx = mx_in[slot * qtok + row];
    sm = sm_in[slot * qtok + row];
  } else {
    row_stats<T, A>(qrow, kf, slot, kl, limit, dim, scale, red, &mx, &sm);
  }
  const A dl = delta[slot * qtok + row];
  A acc = A(0);
  for (int64_t j0 = 0; j0 < limit; j0 += kSmKeys) {
    const int n = (int)lmin(kSmKeys, limit - j0);
    if (threadIdx.x < n) {
      const T* kr = kf + kl.row(slot, j0 + threadIdx.x, dim);
      const T* vr = vf + kl.row(slot, j0 + threadIdx.x, dim);
      A sdot = A(0), pdot = A(0);
      for (int a = 0; a < dim; ++a) {
        sdot += qrow[a] * load_as<A>(kr + a);
        pdot += dorow[a] * load_as<A>(vr + a);
      }
      const A pr = dev_exp<A>(sdot * scale - mx) / sm;
      ds[threadIdx.x] = pr * (pdot - dl);
    }
    __syncthreads();
    if (threadIdx.x < dim)
      for (int j = 0; j < n; ++j) acc += ds[j] * load_as<A>(kf + kl.row(slot, j0 + j, dim) + threadIdx.x);
    __syncthreads();
  }
  if (threadIdx.x < dim) store_as<T, A>(dq + (slot * qtok + row) * dim + threadIdx.x, acc * scale);
}

// Per-query-row statistics (max, sum) for the key-major dK/dV pass.
template <typename T, typename A>
__global__ void __launch_bounds__(kSmThreads) simt_softmax_rowstats_kernel(const T* __restrict__ q,
                                                                           const T* __restrict__ kf, A* __restrict__ mx,
                                                                           A* __restrict__ sm, int64_t qtok,
                                                                           int64_t kvtok, int dim, int causal,
                                                                           int64_t row_offset, KvLayout kl) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* qrow = reinterpret_cast<A*>(smem_raw);
  A* red = qrow + dim;
  const int64_t row = blockIdx.x, slot = blockIdx.y;
  for (int c = threadIdx.x; c < dim; c += blockDim.x) qrow[c] = load_as<A>(q + (slot * qtok + row) * dim + c);
  __syncthreads();
  const A scale = dev_rsqrt<A>(dim);
  const int64_t limit = causal ? lmin(kvtok, row_offset + row + 1) : kvtok;
  A m, s;
  row_stats<T, A>(qrow, kf, slot, kl, limit, dim, scale, red, &m, &s);
  if (threadIdx.x == 0) {
    mx[slot * qtok + row] = m;
    sm[slot * qtok + row] = s;
  }
}

// dk_full[j] = scale * sum_i dS[i][j] q_i ; dv_full[j] = sum_i P[i][j] dO_i  (oracle.py:151-157)
template <typename T, typename A, typename G>
__global__ void __launch_bounds__(kSmThreads) simt_softmax_bwd_dkdv_kernel(
    const T* __restrict__ q, const T* __restrict__ kf, const T* __restrict__ vf, const T* __restrict__ d_out,
    const A* __restrict__ delta, const A* __restrict__ mx, const A* __restrict__ sm, G* __restrict__ dk_full,
    G* __restrict__ dv_full, int64_t qtok, int64_t kvtok, int dim, int causal, int64_t row_offset, KvLayout kl,
    KvLayout gl) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* krow = reinterpret_cast<A*>(smem_raw);
  A* vrow = krow + dim;
  A* pv = vrow + dim;    // [kSmKeys] probabilities
  A* dsv = pv + kSmKeys;  // [kSmKeys] dS
  const int64_t j = blockIdx.x, slot = blockIdx.y;
  for (int c = threadIdx.x; c < dim; c += blockDim.x) {
    krow[c] = load_as<A>(kf + kl.row(slot, j, dim) + c);
    vrow[c] = load_as<A>(vf + kl.row(slot, j, dim) + c);
  }
  __syncthreads();
  const A scale = dev_rsqrt<A>(dim);
  // query rows i (local) with global position row_offset+i >= j see key j
  const int64_t i_start = causal ? lmax(0, j - row_offset) : 0;
  A acc_k = A(0), acc_v = A(0);
  for (int64_t i0 = i_start; i0 < qtok; i0 += kSmKeys) {
    const int n = (int)lmin(kSmKeys, qtok - i0);
    if (threadIdx.x < n) {
      const int64_t i = i0 + threadIdx.x;
      const T* qr = q + (slot * qtok + i) * dim;
      const T* dr = d_out + (slot * qtok + i) * dim;
      A sdot = A(0), pdot = A(0);
      for (int a = 0; a < dim; ++a) {
        sdot += load_as<A>(qr + a) * krow[a];
        pdot += load_as<A>(dr + a) * vrow[a];
      }
      const int64_t r = slot * qtok + i;
      const A pr = dev_exp<A>(sdot * scale - mx[r]) / sm[r];
      pv[threadIdx.x] = pr;
      dsv[threadIdx.x] = pr * (pdot - delta[r]);
    }
    __syncthreads();
    if (threadIdx.x < dim) {
      for (int t = 0; t < n; ++t) {
        const int64_t r = slot * qtok + i0 + t;
        acc_k += dsv[t] * load_as<A>(q + r * dim + threadIdx.x);
        acc_v += pv[t] * load_as<A>(d_out + r * dim + threadIdx.x);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x < dim) {
    dk_full[gl.row(slot, j, dim) + threadIdx.x] = (G)(acc_k * scale);
    dv_full[gl.row(slot, j, dim) + threadIdx.x] = (G)acc_v;
  }
}

// ---------------------------------------------------------------------------
// Host launchers (called from capi.cu).
// ---------------------------------------------------------------------------
template <typename T, typename A>
cudaError_t simt_segment_states(const void* x, const void* y, void* out, int64_t slots, int64_t tokens, int dim,
                                int nseg, cudaStream_t s) {
  const size_t smem = 2 * kSimtBT * dim * sizeof(A);
  dim3 grid(nseg, (unsigned)slots);
  simt_segment_states_kernel<T, A><<<grid, kSimtThreads, smem, s>>>((const T*)x, (const T*)y, (A*)out, tokens, dim,
                                                                    nseg);
  return cudaGetLastError();
}

template <typename T, typename A>
cudaError_t simt_causal_chunk(const void* q, const void* k, const void* v, const void* seg_states, const void* base,
                              void* out, int64_t slots, int64_t tokens, int dim, int nseg, int reverse,
                              int transpose_state, cudaStream_t s) {
  const size_t smem = (size_t)(dim * dim + 3 * kSimtBT * dim + kSimtBT * kSimtBT) * sizeof(A);
  auto kern = simt_causal_chunk_kernel<T, A>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(nseg, (unsigned)slots);
  kern<<<grid, kSimtThreads, smem, s>>>((const T*)q, (const T*)k, (const T*)v, (const A*)seg_states,
                                        (const A*)base, (T*)out, tokens, dim, nseg, reverse, transpose_state);
  return cudaGetLastError();
}

template <typename T, typename A>
cudaError_t simt_apply_state(const void* x, const void* m, void* out, int64_t slots, int64_t tokens, int dim,
                             int transpose, int accumulate, cudaStream_t s, int64_t m_stride) {
  if (m_stride < 0) m_stride = (int64_t)dim * dim;
  const size_t smem = (size_t)(dim * dim + kSimtBT * dim) * sizeof(A);
  auto kern = simt_apply_state_kernel<T, A>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t per_cta = kSimtBT * 8;
  dim3 grid((unsigned)((tokens + per_cta - 1) / per_cta), (unsigned)slots);
  kern<<<grid, kSimtThreads, smem, s>>>((const T*)x, (const A*)m, (T*)out, tokens, dim, transpose, accumulate,
                                         m_stride);
  return cudaGetLastError();
}

template <typename T, typename A>
cudaError_t simt_softmax_forward(const void* q, const void* kf, const void* vf, void* out, void* lse, int64_t slots,
                                 int64_t qtok, int64_t kvtok, int dim, int causal, int64_t row_offset, int64_t kv_chunk,
                                 int64_t kv_rank_stride, cudaStream_t s, int64_t kv_start) {
  const KvLayout kl{kv_chunk, kv_rank_stride, kv_start};
  const size_t smem = (size_t)(dim + kSmKeys + 32) * sizeof(A);
  dim3 grid((unsigned)qtok, (unsigned)slots);
  simt_softmax_fwd_kernel<T, A><<<grid, kSmThreads, smem, s>>>((const T*)q, (const T*)kf, (const T*)vf, (T*)out,
                                                               (A*)lse, qtok, kvtok, dim, causal, row_offset, kl);
  return cudaGetLastError();
}

template <typename T, typename A, typename G>
cudaError_t simt_softmax_backward(const void* q, const void* kf, const void* vf, const void* o, const void* d_out,
                                  void* dq, void* dk_full, void* dv_full, void* scratch, int64_t slots, int64_t qtok,
                                  int64_t kvtok, int dim, int causal, int64_t row_offset, int64_t kv_chunk,
                                  int64_t kv_rank_stride, int64_t grad_rank_stride, cudaStream_t s, const void* lse,
                                  int64_t kv_start) {
  const KvLayout kl{kv_chunk, kv_rank_stride, kv_start}, gl{kv_chunk, grad_rank_stride, kv_start};
  A* delta = reinterpret_cast<A*>(scratch);
  A* mx = delta + slots * qtok;
  A* sm = mx + slots * qtok;
  const int64_t rows = slots * qtok;
  dim3 gq((unsigned)qtok, (unsigned)slots);
  if (lse != nullptr) {
    // the keys are a sub-range of the softmax: P from the forward's lse, delta = rowsum(dO o O)
    // over the whole key set (reference grouping needs every key, this call sees only its range)
    stats_from_lse_kernel<A><<<(unsigned)((rows + 255) / 256), 256, 0, s>>>((const A*)lse, mx, sm, rows);
    simt_softmax_delta_kernel<T, A><<<(unsigned)((rows + 7) / 8), dim3(32, 8), 0, s>>>((const T*)o, (const T*)d_out,
                                                                                      delta, rows, dim);
  } else {
    // delta formed from P and dP (reference grouping, oracle.py:155), exact row statistics
    simt_softmax_rowstats_kernel<T, A><<<gq, kSmThreads, (size_t)(dim + 32) * sizeof(A), s>>>(
        (const T*)q, (const T*)kf, mx, sm, qtok, kvtok, dim, causal, row_offset, kl);
    simt_softmax_delta_exact_kernel<T, A><<<gq, kSmThreads, (size_t)(2 * dim + 32) * sizeof(A), s>>>(
        (const T*)q, (const T*)kf, (const T*)vf, (const T*)d_out, mx, sm, delta, qtok, kvtok, dim, causal, row_offset,
        kl);
  }
  simt_softmax_bwd_dq_kernel<T, A><<<gq, kSmThreads, (size_t)(2 * dim + kSmKeys + 32) * sizeof(A), s>>>(
      (const T*)q, (const T*)kf, (const T*)vf, (const T*)d_out, delta, (T*)dq, qtok, kvtok, dim, causal,
      row_offset, kl, lse != nullptr ? mx : nullptr, sm);
  dim3 gk((unsigned)kvtok, (unsigned)slots);
  simt_softmax_bwd_dkdv_kernel<T, A, G><<<gk, kSmThreads, (size_t)(2 * dim + 2 * kSmKeys) * sizeof(A), s>>>(
      (const T*)q, (const T*)kf, (const T*)vf, (const T*)d_out, delta, mx, sm, (G*)dk_full, (G*)dv_full, qtok,
      kvtok, dim, causal, row_offset, kl, gl);
  return cudaGetLastError();
}

cudaError_t softmax_delta_bf16(const void* o, const void* d_out, float* delta, int64_t rows, int dim,
                               cudaStream_t s) {
  simt_softmax_delta_kernel<__nv_bfloat16, float><<<(unsigned)((rows + 7) / 8), dim3(32, 8), 0, s>>>(
      (const __nv_bfloat16*)o, (const __nv_bfloat16*)d_out, delta, rows, dim);
  return cudaGetLastError();
}

// explicit instantiations: (io, accumulate) = (f32,f32), (f64,f64) -- the validation modes;
// bfloat16 runs on the tcgen05 kernels only
#define LASP_INST(T, A)                                                                                         \
  template cudaError_t simt_segment_states<T, A>(const void*, const void*, void*, int64_t, int64_t, int, int,   \
                                                 cudaStream_t);                                                 \
  template cudaError_t simt_causal_chunk<T, A>(const void*, const void*, const void*, const void*, const void*, \
                                               void*, int64_t, int64_t, int, int, int, int, cudaStream_t);      \
  template cudaError_t simt_apply_state<T, A>(const void*, const void*, void*, int64_t, int64_t, int, int, int, \
                                              cudaStream_t, int64_t);                                           \
  template cudaError_t simt_softmax_forward<T, A>(const void*, const void*, const void*, void*, void*, int64_t, \
                                                  int64_t, int64_t, int, int, int64_t, int64_t, int64_t,         \
                                                  cudaStream_t, int64_t);
LASP_INST(float, float)
LASP_INST(double, double)
template cudaError_t simt_softmax_backward<float, float, float>(const void*, const void*, const void*, const void*,
                                                                const void*, void*, void*, void*, void*, int64_t,
                                                                int64_t, int64_t, int, int, int64_t, int64_t, int64_t,
                                                                int64_t, cudaStream_t, const void*, int64_t);
template cudaError_t simt_softmax_backward<double, double, double>(const void*, const void*, const void*,
                                                                   const void*, const void*, void*, void*, void*,
                                                                   void*, int64_t, int64_t, int64_t, int, int,
                                                                   int64_t, int64_t, int64_t, int64_t, cudaStream_t,
                                                                   const void*, int64_t);

}  // namespace lasp
