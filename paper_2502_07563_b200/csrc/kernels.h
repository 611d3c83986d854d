// Internal launcher declarations (C++ side of the C-ABI in capi.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lasp {

// validation-mode SIMT kernels, (io, accumulate) in {(f32,f32), (f64,f64), (bf16,f32)}
template <typename T, typename A>
cudaError_t simt_segment_states(const void* x, const void* y, void* out, int64_t slots, int64_t tokens, int dim,
                                int nseg, cudaStream_t s);
template <typename T, typename A>
cudaError_t simt_causal_chunk(const void* q, const void* k, const void* v, const void* seg_states, const void* base,
                              void* out, int64_t slots, int64_t tokens, int dim, int nseg, int reverse,
                              int transpose_state, cudaStream_t s);
template <typename T, typename A>
cudaError_t simt_apply_state(const void* x, const void* m, void* out, int64_t slots, int64_t tokens, int dim,
                             int transpose, int accumulate, cudaStream_t s, int64_t m_stride = -1);
template <typename T, typename A>
cudaError_t simt_softmax_forward(const void* q, const void* kf, const void* vf, void* out, void* lse, int64_t slots,
                                 int64_t qtok, int64_t kvtok, int dim, int causal, int64_t row_offset, int64_t kv_chunk,
                                 int64_t kv_rank_stride, cudaStream_t s, int64_t kv_start = 0);
template <typename T, typename A, typename G>
cudaError_t simt_softmax_backward(const void* q, const void* kf, const void* vf, const void* o, const void* d_out,
                                  void* dq, void* dk_full, void* dv_full, void* scratch, int64_t slots, int64_t qtok,
                                  int64_t kvtok, int dim, int causal, int64_t row_offset, int64_t kv_chunk,
                                  int64_t kv_rank_stride, int64_t grad_rank_stride, cudaStream_t s,
                                  const void* lse = nullptr, int64_t kv_start = 0);

// shared state reductions / datagen
template <typename A>
cudaError_t scan_states(void* seg, void* total, int64_t slots, int nseg, int dim, int reverse, cudaStream_t s);
template <typename A>
cudaError_t scan_put(void* seg, void* total, int64_t slots, int nseg, int dim, int reverse, const void* peer_recv,
                     const void* peer_flags, int rank, int nranks, unsigned long long epoch, unsigned* done,
                     cudaStream_t s, void* epoch_dev = nullptr);
// epoch_dev != null: the epoch is *epoch_dev + (signed) epoch, read on the device
cudaError_t exchange_wait(const void* flags, int lo, int hi, unsigned long long epoch, cudaStream_t s,
                          const void* epoch_dev = nullptr);
cudaError_t exchange_ack(const void* peer_acks, int rank, int nranks, unsigned long long epoch, cudaStream_t s,
                         const void* epoch_dev = nullptr);
template <typename A>
cudaError_t exchange_fold(const void* recv, int64_t half_elems, const void* epoch_dev, void* out, int nstates,
                          int64_t elems, int mode, int bound, cudaStream_t s);
template <typename A>
cudaError_t fold_states(const void* gathered, void* out, int nstates, int64_t elems, int mode, int bound,
                        cudaStream_t s);
template <typename T>
cudaError_t gen_slots(uint64_t seed, const uint64_t* tag_words, void* out, int64_t slots, int64_t rows, int64_t cols,
                      int64_t row0, cudaStream_t s);

// tcgen05 fast path (bf16 in, fp32 states)
bool tc_supported(int dim, int64_t tokens);
cudaError_t tc_segment_states(const void* x, const void* y, float* out, int64_t slots, int64_t tokens, int dim,
                              int nseg, cudaStream_t s);
// In-kernel consumer of the fused peer state exchange (lasp2_scan_put): the
// rank-level base is folded from this epoch's receive half once the flags of
// ranks [lo, hi) carry `epoch` (see CausalArgs in tc_linear.cu).
struct XFold {
  const float* recv;                // [T][slots][dim][dim] (with epoch_dev: [2][T][...], half by epoch parity)
  const unsigned long long* flags;  // [T]
  int lo, hi, descending;
  unsigned long long epoch;
  float* base_out;                  // folded base per slot, or null
  const unsigned long long* epoch_dev = nullptr;  // device-resident epoch (graph-capturable exchange)
  int64_t half_elems = 0;           // elements of one receive half
};
cudaError_t tc_causal_chunk(const void* q, const void* k, const void* v, const float* seg_states, const float* base,
                            void* out, int64_t slots, int64_t tokens, int dim, int nseg, int reverse,
                            int transpose_state, cudaStream_t s,
                            const XFold* xfold = nullptr);
cudaError_t tc_dq_chunk(const void* q, const void* k, const void* v, const void* d_out, const float* fwd_seg,
                        const float* fwd_base, float* g_out, void* dq, int64_t slots, int64_t tokens, int dim,
                        int nseg, cudaStream_t s);
cudaError_t tc_dkdv_pair(const void* q, const void* k, const void* v, const void* d_out, const float* seg_states,
                         const float* base, void* dk, void* dv, int64_t slots, int64_t tokens, int dim, int nseg,
                         cudaStream_t s, const XFold* xfold = nullptr);
cudaError_t tc_apply_state(const void* x, const float* m, void* out, int64_t slots, int64_t tokens, int dim,
                           int transpose, int accumulate, int sm_count, cudaStream_t s);
// out (+)= sum_i xs[i] op(ms[i]) for nx in {1, 3} (accumulate only with nx = 1); m_stride =
// dim^2 for per-slot states, 0 for one weight shared by every slot
cudaError_t tc_apply_multi(const void* const* xs, const float* const* ms, int nx, int64_t m_stride, void* out,
                           int64_t slots, int64_t tokens, int dim, int transpose, int accumulate, int sm_count,
                           cudaStream_t s);
bool tc_softmax_supported(int dim, int64_t kv_chunk);
cudaError_t tc_softmax_forward(const void* q, const void* kf, const void* vf, void* out, float* lse, int64_t slots,
                               int64_t qtok, int64_t kvtok, int dim, int causal, int64_t row_offset, int64_t kv_chunk,
                               int64_t kv_rank_stride, cudaStream_t s, int64_t kv_start = 0);
int64_t tc_softmax_bwd_scratch(int64_t slots, int64_t qtok, int dim);
cudaError_t tc_softmax_backward(const void* q, const void* kf, const void* vf, const void* o, const float* lse,
                                const void* d_out, void* dq, float* dk_full, float* dv_full, void* scratch,
                                int64_t slots, int64_t qtok, int64_t kvtok, int dim, int causal, int64_t row_offset,
                                int64_t kv_chunk, int64_t kv_rank_stride, int64_t grad_rank_stride, cudaStream_t s,
                                int64_t kv_start = 0);
cudaError_t softmax_delta_bf16(const void* o, const void* d_out, float* delta, int64_t rows, int dim,
                               cudaStream_t s);
cudaError_t tc_backward_triple(const void* q, const void* k, const void* v, const void* d_out, const float* fwd_seg,
                               const float* fwd_total, const float* fwd_base, const float* bwd_seg,
                               const float* bwd_base, void* dq, void* dk, void* dv, int64_t slots, int64_t tokens,
                               int dim, int nseg, cudaStream_t s, const float* bwd_total = nullptr);
cudaError_t tc_state_apply(const void* x0, const void* x1, const float* m, float* seg_out, void* out, int64_t slots,
                           int64_t tokens, int dim, int nseg, cudaStream_t s);
cudaError_t tc_apply2(const void* x0, const void* x1, const float* m, void* out0, void* out1, int64_t slots,
                      int64_t tokens, int dim, int sm_count, cudaStream_t s);
int64_t tc_flat_workspace_bytes(int64_t slots, int64_t tokens, int dim, int sm_count);
// Fused state exchange of the unmasked world kernels (T > 1, one GPU per rank): the phase-1
// reduction stores this rank's chunk state into every rank's receive buffer, the kernel waits
// for every rank's flag, folds the full sum and runs phase 2 in the same launch.
struct FlatXchg {
  float* const* recv_peers;                // [T] receive buffers [2][T][slots][dim][dim]
  unsigned long long* const* flag_peers;   // [T] flag arrays [T]
  unsigned long long* const* ack_peers;    // [T] ack arrays [T]
  const float* recv;                       // this rank's receive buffer
  const unsigned long long* flags;         // this rank's flags
  const unsigned long long* acks;          // this rank's acks (written by the readers)
  unsigned long long* epoch_dev;           // device epoch: this exchange is *epoch_dev + 1
  int rank, nranks;
};
cudaError_t tc_flat_forward(const void* q, const void* k, const void* v, void* out, float* m_full, void* workspace,
                            int64_t slots, int64_t tokens, int dim, int sm_count, cudaStream_t s, int phases = 3,
                            const FlatXchg* x = nullptr);
cudaError_t tc_flat_backward(const void* q, const void* k, const void* v, const void* d_out, const float* m_full,
                             void* dq, void* dk, void* dv, void* workspace, int64_t slots, int64_t tokens, int dim,
                             int sm_count, cudaStream_t s, float* dm = nullptr, int phases = 3,
                             const FlatXchg* x = nullptr);
cudaError_t tc_set_trace(unsigned long long* buf);
cudaError_t tc_set_trace_flat(unsigned long long* buf);
cudaError_t tc_set_trace_softmax(unsigned long long* buf);
cudaError_t tc_probe_gemm(const void* a, const void* b, float* d, int a_mn, int b_mn, cudaStream_t s);

}  // namespace lasp
