// extern "C" entry points declared in include/lasp2_b200.h.
//
// Validation and dtype dispatch only: argument errors return
// LASP2_ERR_INVALID, CUDA failures LASP2_ERR_CUDA, and lasp2_last_error()
// carries the message. No exception crosses this boundary.
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is dlopen'd (below)
#include <stdio.h>
#include <string.h>

#include <string>

#include "../../include/lasp2_b200.h"
#include "common.cuh"
#include "kernels.h"

namespace {

thread_local std::string g_err;

int fail(int code, const char* msg) {
  g_err = msg;
  return code;
}
int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) {
    g_err.clear();
    return LASP2_OK;
  }
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", where, cudaGetErrorString(e));
  g_err = buf;
  return LASP2_ERR_CUDA;
}
int sm_count_current() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}
bool valid_dtype(int dt) { return dt == LASP2_F32 || dt == LASP2_F64 || dt == LASP2_BF16; }
bool use_tc(int dtype, int dim, int64_t tokens) { return dtype == LASP2_BF16 && lasp::tc_supported(dim, tokens); }
// bfloat16 runs on the tcgen05 kernels only; there is no second bf16 backend.
bool bf16_ok(int dtype, int dim, int64_t tokens) { return dtype != LASP2_BF16 || use_tc(dtype, dim, tokens); }
#define BF16_ENVELOPE "bfloat16 needs the tcgen05 envelope: 8 <= dim <= 128 and dim % 8 == 0 (float32 / float64 run any shape)"

cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#define CHECK(cond, msg) \
  if (!(cond)) return fail(LASP2_ERR_INVALID, msg)

}  // namespace

extern "C" {

int lasp2_version(void) { return 100; }

const char* lasp2_last_error(void) { return g_err.c_str(); }

int lasp2_num_segments(int dtype, int64_t slots, int64_t tokens, int dim, int sm_count) {
  if (slots < 1 || tokens < 1) return 1;
  if (sm_count < 1) sm_count = 148;
  const int64_t nblk = (tokens + LASP_BLOCK_TOKENS - 1) / LASP_BLOCK_TOKENS;
  // tcgen05 kernels run one CTA per SM: fill one wave exactly. SIMT kernels
  // are shorter-lived: two CTAs per SM.
  const int64_t waves = use_tc(dtype, dim, tokens) ? 1 : 2;
  int64_t nseg = (waves * sm_count) / slots;
  if (nseg < 1) nseg = 1;
  if (nseg > nblk) nseg = nblk;
  if (nseg > 65535) nseg = 65535;
  return (int)nseg;
}

int lasp2_segment_states(int dtype, const void* x, const void* y, void* seg_states, int64_t slots, int64_t tokens,
                         int dim, int nseg, void* stream) {
  CHECK(valid_dtype(dtype), "segment_states: unknown dtype");
  CHECK(x && y && seg_states, "segment_states: null pointer");
  CHECK(slots >= 1 && tokens >= 1 && dim >= 1 && dim <= 128, "segment_states: bad shape (1 <= dim <= 128)");
  CHECK(nseg >= 1 && nseg <= (tokens + LASP_BLOCK_TOKENS - 1) / LASP_BLOCK_TOKENS, "segment_states: bad nseg");
  cudaError_t e;
  CHECK(bf16_ok(dtype, dim, tokens), BF16_ENVELOPE);
  if (use_tc(dtype, dim, tokens))
    e = lasp::tc_segment_states(x, y, (float*)seg_states, slots, tokens, dim, nseg, S(stream));
  else if (dtype == LASP2_F32)
    e = lasp::simt_segment_states<float, float>(x, y, seg_states, slots, tokens, dim, nseg, S(stream));
  else if (dtype == LASP2_F64)
    e = lasp::simt_segment_states<double, double>(x, y, seg_states, slots, tokens, dim, nseg, S(stream));
  else
    e = cudaErrorInvalidValue;  // unreachable: bf16_ok() above
  return cuda_status(e, "segment_states");
}

int lasp2_scan_segments(int dtype, void* seg_states, void* chunk_total, int64_t slots, int nseg, int dim, int reverse,
                        void* stream) {
  CHECK(valid_dtype(dtype), "scan_segments: unknown dtype");
  CHECK(seg_states, "scan_segments: null pointer");
  CHECK(slots >= 1 && nseg >= 1 && dim >= 1, "scan_segments: bad shape");
  cudaError_t e = dtype == LASP2_F64 ? lasp::scan_states<double>(seg_states, chunk_total, slots, nseg, dim, reverse,
                                                                 S(stream))
                                     : lasp::scan_states<float>(seg_states, chunk_total, slots, nseg, dim, reverse,
                                                                S(stream));
  return cuda_status(e, "scan_segments");
}

int lasp2_scan_put(int dtype, void* seg_states, void* chunk_total, int64_t slots, int nseg, int dim, int reverse,
                   const void* peer_recv, const void* peer_flags, int rank, int nranks, uint64_t epoch, void* done,
                   void* epoch_dev, void* stream) {
  CHECK(valid_dtype(dtype), "scan_put: unknown dtype");
  CHECK(seg_states && peer_recv && peer_flags && done, "scan_put: null pointer");
  CHECK(slots >= 1 && nseg >= 1 && dim >= 1, "scan_put: bad shape");
  CHECK(nranks >= 1 && rank >= 0 && rank < nranks, "scan_put: rank outside [0, nranks)");
  CHECK(epoch >= 1 || epoch_dev, "scan_put: epochs start at 1");
  cudaError_t e = dtype == LASP2_F64
                      ? lasp::scan_put<double>(seg_states, chunk_total, slots, nseg, dim, reverse, peer_recv,
                                               peer_flags, rank, nranks, epoch, (unsigned*)done, S(stream), epoch_dev)
                      : lasp::scan_put<float>(seg_states, chunk_total, slots, nseg, dim, reverse, peer_recv,
                                              peer_flags, rank, nranks, epoch, (unsigned*)done, S(stream), epoch_dev);
  return cuda_status(e, "scan_put");
}

int lasp2_exchange_wait(const void* flags, int lo, int hi, uint64_t epoch, const void* epoch_dev, void* stream) {
  CHECK(flags, "exchange_wait: null pointer");
  CHECK(lo >= 0 && hi >= lo, "exchange_wait: bad range");
  return cuda_status(lasp::exchange_wait(flags, lo, hi, epoch, S(stream), epoch_dev), "exchange_wait");
}

int lasp2_exchange_ack(const void* peer_acks, int rank, int nranks, uint64_t epoch, const void* epoch_dev,
                       void* stream) {
  CHECK(peer_acks, "exchange_ack: null pointer");
  CHECK(nranks >= 1 && rank >= 0 && rank < nranks, "exchange_ack: rank outside [0, nranks)");
  return cuda_status(lasp::exchange_ack(peer_acks, rank, nranks, epoch, S(stream), epoch_dev), "exchange_ack");
}

int lasp2_exchange_fold(int dtype, const void* recv, int64_t half_elems, const void* epoch_dev, void* out,
                        int nstates, int64_t elems, int mode, int bound, void* stream) {
  CHECK(valid_dtype(dtype), "exchange_fold: unknown dtype");
  CHECK(recv && epoch_dev && out, "exchange_fold: null pointer");
  CHECK(nstates >= 1 && elems >= 1 && half_elems >= (int64_t)nstates * elems, "exchange_fold: bad shape");
  CHECK(mode >= 0 && mode <= 2, "exchange_fold: bad mode");
  CHECK(mode == LASP2_FOLD_FULL || (bound >= 0 && bound <= nstates), "exchange_fold: bound outside [0, nstates]");
  cudaError_t e = dtype == LASP2_F64
                      ? lasp::exchange_fold<double>(recv, half_elems, epoch_dev, out, nstates, elems, mode, bound,
                                                    S(stream))
                      : lasp::exchange_fold<float>(recv, half_elems, epoch_dev, out, nstates, elems, mode, bound,
                                                   S(stream));
  return cuda_status(e, "exchange_fold");
}

int lasp2_fold_states(int dtype, const void* gathered, void* out, int nstates, int64_t elems, int mode, int bound,
                      void* stream) {
  CHECK(valid_dtype(dtype), "fold_states: unknown dtype");
  CHECK(gathered && out, "fold_states: null pointer");
  CHECK(nstates >= 1 && elems >= 1, "fold_states: bad shape");
  CHECK(mode >= 0 && mode <= 2, "fold_states: bad mode");
  CHECK(mode == LASP2_FOLD_FULL || (bound >= 0 && bound <= nstates), "fold_states: bound outside [0, nstates]");
  cudaError_t e = dtype == LASP2_F64
                      ? lasp::fold_states<double>(gathered, out, nstates, elems, mode, bound, S(stream))
                      : lasp::fold_states<float>(gathered, out, nstates, elems, mode, bound, S(stream));
  return cuda_status(e, "fold_states");
}

int lasp2_causal_chunk(int dtype, const void* q, const void* k, const void* v, const void* seg_states,
                       const void* base, void* out, int64_t slots, int64_t tokens, int dim, int nseg, int reverse,
                       int transpose_state, void* stream) {
  CHECK(valid_dtype(dtype), "causal_chunk: unknown dtype");
  CHECK(q && k && v && out, "causal_chunk: null pointer");
  CHECK(slots >= 1 && tokens >= 1 && dim >= 1 && dim <= 128, "causal_chunk: bad shape (1 <= dim <= 128)");
  CHECK(nseg >= 1 && nseg <= (tokens + LASP_BLOCK_TOKENS - 1) / LASP_BLOCK_TOKENS, "causal_chunk: bad nseg");
  CHECK(nseg == 1 || seg_states, "causal_chunk: nseg > 1 needs segment states");
  cudaError_t e;
  CHECK(bf16_ok(dtype, dim, tokens), BF16_ENVELOPE);
  if (use_tc(dtype, dim, tokens))
    e = lasp::tc_causal_chunk(q, k, v, (const float*)seg_states, (const float*)base, out, slots, tokens, dim, nseg,
                              reverse, transpose_state, S(stream));
  else if (dtype == LASP2_F32)
    e = lasp::simt_causal_chunk<float, float>(q, k, v, seg_states, base, out, slots, tokens, dim, nseg, reverse,
                                              transpose_state, S(stream));
  else if (dtype == LASP2_F64)
    e = lasp::simt_causal_chunk<double, double>(q, k, v, seg_states, base, out, slots, tokens, dim, nseg, reverse,
                                                transpose_state, S(stream));
  else
    e = cudaErrorInvalidValue;  // unreachable: bf16_ok() above
  return cuda_status(e, "causal_chunk");
}

int lasp2_causal_chunk_x(const void* q, const void* k, const void* v, const void* seg_states, const void* xrecv,
                         const void* xflags, int lo, int hi, int descending, uint64_t epoch, const void* epoch_dev,
                         int64_t half_elems, void* base_out, void* out, int64_t slots, int64_t tokens, int dim,
                         int nseg, int reverse, int transpose_state, void* stream) {
  CHECK(q && k && v && out && xrecv, "causal_chunk_x: null pointer");
  CHECK(slots >= 1 && tokens >= 1 && dim >= 1 && dim <= 128, "causal_chunk_x: bad shape (1 <= dim <= 128)");
  CHECK(nseg >= 1 && nseg <= (tokens + LASP_BLOCK_TOKENS - 1) / LASP_BLOCK_TOKENS, "causal_chunk_x: bad nseg");
  CHECK(nseg == 1 || seg_states, "causal_chunk_x: nseg > 1 needs segment states");
  CHECK(lo >= 0 && hi >= lo, "causal_chunk_x: bad rank range");
  CHECK(use_tc(LASP2_BF16, dim, tokens), "causal_chunk_x: bf16 tensor-core path only (fold, then lasp2_causal_chunk)");
  const lasp::XFold x{(const float*)xrecv, (const unsigned long long*)xflags, lo, hi, descending, epoch,
                      (float*)base_out, (const unsigned long long*)epoch_dev, half_elems};
  return cuda_status(lasp::tc_causal_chunk(q, k, v, (const float*)seg_states, nullptr, out, slots, tokens, dim, nseg,
                                           reverse, transpose_state, S(stream), &x),
                     "causal_chunk_x");
}

int lasp2_dkdv_chunk_x(const void* q, const void* k, const void* v, const void* d_out, const void* seg_states,
                       const void* xrecv, const void* xflags, int lo, int hi, uint64_t epoch, const void* epoch_dev,
                       int64_t half_elems, void* dk, void* dv, int64_t slots, int64_t tokens, int dim, int nseg,
                       void* stream) {
  CHECK(q && k && v && d_out && dk && dv && xrecv, "dkdv_chunk_x: null pointer");
  CHECK(slots >= 1 && tokens >= 1 && dim >= 1 && dim <= 128, "dkdv_chunk_x: bad shape (1 <= dim <= 128)");
  CHECK(nseg >= 1 && nseg <= (tokens + LASP_BLOCK_TOKENS - 1) / LASP_BLOCK_TOKENS, "dkdv_chunk_x: bad nseg");
  CHECK(nseg == 1 || seg_states, "dkdv_chunk_x: nseg > 1 needs segment states");
  CHECK(lo >= 0 && hi >= lo, "dkdv_chunk_x: bad rank range");
  CHECK(use_tc(LASP2_BF16, dim, tokens), "dkdv_chunk_x: bf16 tensor-core path only (fold, then lasp2_dkdv_chunk)");
  const lasp::XFold x{(const float*)xrecv, (const unsigned long long*)xflags, lo, hi, 1, epoch, nullptr,
                      (const unsigned long long*)epoch_dev, half_elems};
  return cuda_status(lasp::tc_dkdv_pair(q, k, v, d_out, (const float*)seg_states, nullptr, dk, dv, slots, tokens, dim,
                                        nseg, S(stream), &x),
                     "dkdv_chunk_x");
}

int lasp2_dq_chunk(int dtype, const void* q, const void* k, const void* v, const void* d_out, const void* fwd_seg,
                   const void* fwd_base, void* g_seg, void* dq, int64_t slots, int64_t tokens, int dim, int nseg,
                   void* stream) {
  CHECK(valid_dtype(dtype), "dq_chunk: unknown dtype");
  CHECK(q && k && v && d_out && g_seg && dq, "dq_chunk: null pointer");
  CHECK(slots >= 1 && tokens >= 1 && dim >= 1 && dim <= 128, "dq_chunk: bad shape (1 <= dim <= 128)");
  CHECK(nseg >= 1 && nseg <= (tokens + LASP_BLOCK_TOKENS - 1) / LASP_BLOCK_TOKENS, "dq_chunk: bad nseg");
  CHECK(nseg == 1 || fwd_seg, "dq_chunk: nseg > 1 needs segment states");
  CHECK(bf16_ok(dtype, dim, tokens), BF16_ENVELOPE);
  if (use_tc(dtype, dim, tokens))
    return cuda_status(lasp::tc_dq_chunk(q, k, v, d_out, (const float*)fwd_seg, (const float*)fwd_base,
                                         (float*)g_seg, dq, slots, tokens, dim, nseg, S(stream)),
                       "dq_chunk");
  int st = lasp2_segment_states(dtype, q, d_out, g_seg, slots, tokens, dim, nseg, stream);
  if (st != LASP2_OK) return st;
  return lasp2_causal_chunk(dtype, d_out, v, k, fwd_seg, fwd_base, dq, slots, tokens, dim, nseg, 0, 1, stream);
}

int lasp2_dkdv_chunk(int dtype, const void* q, const void* k, const void* v, const void* d_out, const void* seg_states,
                     const void* base, void* dk, void* dv, int64_t slots, int64_t tokens, int dim, int nseg,
                     void* stream) {
  CHECK(valid_dtype(dtype), "dkdv_chunk: unknown dtype");
  CHECK(q && k && v && d_out && dk && dv, "dkdv_chunk: null pointer");
  CHECK(slots >= 1 && tokens >= 1 && dim >= 1 && dim <= 128, "dkdv_chunk: bad shape (1 <= dim <= 128)");
  CHECK(nseg >= 1 && nseg <= (tokens + LASP_BLOCK_TOKENS - 1) / LASP_BLOCK_TOKENS, "dkdv_chunk: bad nseg");
  CHECK(nseg == 1 || seg_states, "dkdv_chunk: nseg > 1 needs segment states");
  CHECK(bf16_ok(dtype, dim, tokens), BF16_ENVELOPE);
  if (use_tc(dtype, dim, tokens))
    return cuda_status(lasp::tc_dkdv_pair(q, k, v, d_out, (const float*)seg_states, (const float*)base, dk, dv, slots,
                                          tokens, dim, nseg, S(stream)),
                       "dkdv_chunk");
  int st = lasp2_causal_chunk(dtype, v, d_out, q, seg_states, base, dk, slots, tokens, dim, nseg, 1, 1, stream);
  if (st != LASP2_OK) return st;
  return lasp2_causal_chunk(dtype, k, q, d_out, seg_states, base, dv, slots, tokens, dim, nseg, 1, 0, stream);
}

int lasp2_backward_chunk(int dtype, const void* q, const void* k, const void* v, const void* d_out,
                         const void* fwd_seg, const void* fwd_total, const void* fwd_base, const void* bwd_seg,
                         const void* bwd_base, void* dq, void* dk, void* dv, int64_t slots, int64_t tokens, int dim,
                         int nseg, void* stream) {
  CHECK(valid_dtype(dtype), "backward_chunk: unknown dtype");
  CHECK(q && k && v && d_out && dq && dk && dv && fwd_total, "backward_chunk: null pointer");
  CHECK(slots >= 1 && tokens >= 1 && dim >= 1 && dim <= 128, "backward_chunk: bad shape (1 <= dim <= 128)");
  CHECK(nseg >= 1 && nseg <= (tokens + LASP_BLOCK_TOKENS - 1) / LASP_BLOCK_TOKENS, "backward_chunk: bad nseg");
  CHECK(nseg == 1 || (fwd_seg && bwd_seg), "backward_chunk: nseg > 1 needs segment states");
  CHECK(bf16_ok(dtype, dim, tokens), BF16_ENVELOPE);
  if (use_tc(dtype, dim, tokens))
    return cuda_status(lasp::tc_backward_triple(q, k, v, d_out, (const float*)fwd_seg, (const float*)fwd_total,
                                                (const float*)fwd_base, (const float*)bwd_seg, (const float*)bwd_base,
                                                dq, dk, dv, slots, tokens, dim, nseg, S(stream)),
                       "backward_chunk");
  int st = lasp2_causal_chunk(dtype, d_out, v, k, fwd_seg, fwd_base, dq, slots, tokens, dim, nseg, 0, 1, stream);
  if (st != LASP2_OK) return st;
  return lasp2_dkdv_chunk(dtype, q, k, v, d_out, bwd_seg, bwd_base, dk, dv, slots, tokens, dim, nseg, stream);
}

int lasp2_backward_chunk_fwd(int dtype, const void* q, const void* k, const void* v, const void* d_out,
                             const void* fwd_seg, const void* fwd_base, const void* bwd_seg, const void* bwd_total,
                             const void* bwd_base, void* dq, void* dk, void* dv, int64_t slots, int64_t tokens,
                             int dim, int nseg, void* stream) {
  CHECK(valid_dtype(dtype), "backward_chunk_fwd: unknown dtype");
  CHECK(q && k && v && d_out && dq && dk && dv && bwd_total, "backward_chunk_fwd: null pointer");
  CHECK(slots >= 1 && tokens >= 1 && dim >= 1 && dim <= 128, "backward_chunk_fwd: bad shape (1 <= dim <= 128)");
  CHECK(nseg >= 1 && nseg <= (tokens + LASP_BLOCK_TOKENS - 1) / LASP_BLOCK_TOKENS, "backward_chunk_fwd: bad nseg");
  CHECK(nseg == 1 || (fwd_seg && bwd_seg), "backward_chunk_fwd: nseg > 1 needs segment states");
  CHECK(bf16_ok(dtype, dim, tokens), BF16_ENVELOPE);
  if (use_tc(dtype, dim, tokens))
    return cuda_status(lasp::tc_backward_triple(q, k, v, d_out, (const float*)fwd_seg, nullptr, (const float*)fwd_base,
                                                (const float*)bwd_seg, (const float*)bwd_base, dq, dk, dv, slots,
                                                tokens, dim, nseg, S(stream), (const float*)bwd_total),
                       "backward_chunk_fwd");
  int st = lasp2_causal_chunk(dtype, d_out, v, k, fwd_seg, fwd_base, dq, slots, tokens, dim, nseg, 0, 1, stream);
  if (st != LASP2_OK) return st;
  return lasp2_dkdv_chunk(dtype, q, k, v, d_out, bwd_seg, bwd_base, dk, dv, slots, tokens, dim, nseg, stream);
}

int lasp2_apply_state(int dtype, const void* x, const void* m, void* out, int64_t slots, int64_t tokens, int dim,
                      int transpose, int accumulate, void* stream) {
  CHECK(valid_dtype(dtype), "apply_state: unknown dtype");
  CHECK(x && m && out, "apply_state: null pointer");
  CHECK(slots >= 1 && tokens >= 1 && dim >= 1 && dim <= 128, "apply_state: bad shape (1 <= dim <= 128)");
  cudaError_t e;
  CHECK(bf16_ok(dtype, dim, tokens), BF16_ENVELOPE);
  if (use_tc(dtype, dim, tokens))
    e = lasp::tc_apply_state(x, (const float*)m, out, slots, tokens, dim, transpose, accumulate, sm_count_current(),
                             S(stream));
  else if (dtype == LASP2_F32)
    e = lasp::simt_apply_state<float, float>(x, m, out, slots, tokens, dim, transpose, accumulate, S(stream));
  else if (dtype == LASP2_F64)
    e = lasp::simt_apply_state<double, double>(x, m, out, slots, tokens, dim, transpose, accumulate, S(stream));
  else
    e = cudaErrorInvalidValue;  // unreachable: bf16_ok() above
  return cuda_status(e, "apply_state");
}

int lasp2_project(int dtype, const void* const* xs, const void* const* ws, int nx, void* out, int64_t slots,
                  int64_t tokens, int dim, int transpose, int accumulate, void* stream) {
  CHECK(valid_dtype(dtype), "project: unknown dtype");
  CHECK(xs && ws && out, "project: null pointer");
  CHECK(nx == 1 || nx == 3, "project: nx must be 1 or 3");
  for (int i = 0; i < nx; ++i) CHECK(xs[i] && ws[i], "project: null input or weight");
  CHECK(slots >= 1 && tokens >= 1 && dim >= 1 && dim <= 128, "project: bad shape (1 <= dim <= 128)");
  CHECK(nx == 1 || !accumulate, "project: accumulate needs nx == 1");
  CHECK(bf16_ok(dtype, dim, tokens), BF16_ENVELOPE);
  cudaError_t e = cudaSuccess;
  if (use_tc(dtype, dim, tokens)) {
    e = lasp::tc_apply_multi(xs, reinterpret_cast<const float* const*>(ws), nx, 0, out, slots, tokens, dim, transpose,
                             accumulate, sm_count_current(), S(stream));
  } else {
    // validation dtypes: one pass per input, the later ones accumulating in the data dtype
    for (int i = 0; i < nx && e == cudaSuccess; ++i) {
      const int acc = i > 0 ? 1 : accumulate;
      e = dtype == LASP2_F64
              ? lasp::simt_apply_state<double, double>(xs[i], ws[i], out, slots, tokens, dim, transpose, acc,
                                                       S(stream), 0)
              : lasp::simt_apply_state<float, float>(xs[i], ws[i], out, slots, tokens, dim, transpose, acc, S(stream),
                                                     0);
    }
  }
  return cuda_status(e, "project");
}

int lasp2_state_apply(int dtype, const void* q, const void* d_out, const void* m, void* seg_states, void* dq,
                      int64_t slots, int64_t tokens, int dim, int nseg, void* stream) {
  CHECK(valid_dtype(dtype), "state_apply: unknown dtype");
  CHECK(q && d_out && m && seg_states && dq, "state_apply: null pointer");
  CHECK(slots >= 1 && tokens >= 1 && dim >= 1 && dim <= 128, "state_apply: bad shape (1 <= dim <= 128)");
  CHECK(nseg >= 1 && nseg <= (tokens + LASP_BLOCK_TOKENS - 1) / LASP_BLOCK_TOKENS, "state_apply: bad nseg");
  CHECK(bf16_ok(dtype, dim, tokens), BF16_ENVELOPE);
  if (use_tc(dtype, dim, tokens))
    return cuda_status(lasp::tc_state_apply(q, d_out, (const float*)m, (float*)seg_states, dq, slots, tokens, dim, nseg,
                                            S(stream)),
                       "state_apply");
  int st = lasp2_segment_states(dtype, q, d_out, seg_states, slots, tokens, dim, nseg, stream);
  if (st != LASP2_OK) return st;
  return lasp2_apply_state(dtype, d_out, m, dq, slots, tokens, dim, 1, 0, stream);
}

int lasp2_apply_state2(int dtype, const void* v, const void* k, const void* dm, void* dk, void* dv, int64_t slots,
                       int64_t tokens, int dim, void* stream) {
  CHECK(valid_dtype(dtype), "apply_state2: unknown dtype");
  CHECK(v && k && dm && dk && dv, "apply_state2: null pointer");
  CHECK(slots >= 1 && tokens >= 1 && dim >= 1 && dim <= 128, "apply_state2: bad shape (1 <= dim <= 128)");
  CHECK(bf16_ok(dtype, dim, tokens), BF16_ENVELOPE);
  if (use_tc(dtype, dim, tokens))
    return cuda_status(lasp::tc_apply2(v, k, (const float*)dm, dk, dv, slots, tokens, dim, sm_count_current(),
                                       S(stream)),
                       "apply_state2");
  int st = lasp2_apply_state(dtype, v, dm, dk, slots, tokens, dim, 1, 0, stream);
  if (st != LASP2_OK) return st;
  return lasp2_apply_state(dtype, k, dm, dv, slots, tokens, dim, 0, 0, stream);
}

// ---- unmasked layer on a world of one rank (lasp2.py:208-216, :256-267 with T = 1) ----
namespace {
int64_t simt_local_ws(int dtype, int64_t slots, int64_t tokens, int dim) {
  const int64_t nseg = lasp2_num_segments(dtype, slots, tokens, dim, sm_count_current());
  const int64_t elt = dtype == LASP2_F64 ? 8 : 4;
  return (slots * nseg + slots) * (int64_t)dim * dim * elt;
}
}  // namespace

int64_t lasp2_local_workspace_bytes(int dtype, int64_t slots, int64_t tokens, int dim, int sm_count) {
  if (!valid_dtype(dtype) || slots < 1 || tokens < 1 || dim < 1 || dim > 128) return -1;
  if (sm_count < 1) sm_count = sm_count_current();
  if (use_tc(dtype, dim, tokens)) return lasp::tc_flat_workspace_bytes(slots, tokens, dim, sm_count);
  return simt_local_ws(dtype, slots, tokens, dim);
}

int lasp2_nomask_forward_local(int dtype, const void* q, const void* k, const void* v, void* out, void* m_full,
                               void* workspace, int64_t workspace_bytes, int64_t slots, int64_t tokens, int dim,
                               void* stream) {
  CHECK(valid_dtype(dtype), "nomask_forward_local: unknown dtype");
  CHECK(q && k && v && out && m_full && workspace, "nomask_forward_local: null pointer");
  CHECK(slots >= 1 && tokens >= 1 && dim >= 1 && dim <= 128, "nomask_forward_local: bad shape (1 <= dim <= 128)");
  const int sms = sm_count_current();
  CHECK(workspace_bytes >= lasp2_local_workspace_bytes(dtype, slots, tokens, dim, sms),
        "nomask_forward_local: workspace too small (lasp2_local_workspace_bytes)");
  CHECK(bf16_ok(dtype, dim, tokens), BF16_ENVELOPE);
  if (use_tc(dtype, dim, tokens))
    return cuda_status(lasp::tc_flat_forward(q, k, v, out, (float*)m_full, workspace, slots, tokens, dim, sms,
                                             S(stream)),
                       "nomask_forward_local");
  const int nseg = lasp2_num_segments(dtype, slots, tokens, dim, sms);
  int st = lasp2_segment_states(dtype, k, v, workspace, slots, tokens, dim, nseg, stream);
  if (st == LASP2_OK) st = lasp2_scan_segments(dtype, workspace, m_full, slots, nseg, dim, 0, stream);
  if (st == LASP2_OK) st = lasp2_apply_state(dtype, q, m_full, out, slots, tokens, dim, 0, 0, stream);
  return st;
}

int lasp2_nomask_backward_local(int dtype, const void* q, const void* k, const void* v, const void* d_out,
                                const void* m_full, void* dq, void* dk, void* dv, void* workspace,
                                int64_t workspace_bytes, int64_t slots, int64_t tokens, int dim, void* stream) {
  CHECK(valid_dtype(dtype), "nomask_backward_local: unknown dtype");
  CHECK(q && k && v && d_out && m_full && dq && dk && dv && workspace, "nomask_backward_local: null pointer");
  CHECK(slots >= 1 && tokens >= 1 && dim >= 1 && dim <= 128, "nomask_backward_local: bad shape (1 <= dim <= 128)");
  const int sms = sm_count_current();
  CHECK(workspace_bytes >= lasp2_local_workspace_bytes(dtype, slots, tokens, dim, sms),
        "nomask_backward_local: workspace too small (lasp2_local_workspace_bytes)");
  CHECK(bf16_ok(dtype, dim, tokens), BF16_ENVELOPE);
  if (use_tc(dtype, dim, tokens))
    return cuda_status(lasp::tc_flat_backward(q, k, v, d_out, (const float*)m_full, dq, dk, dv, workspace, slots,
                                              tokens, dim, sms, S(stream)),
                       "nomask_backward_local");
  const int nseg = lasp2_num_segments(dtype, slots, tokens, dim, sms);
  const int64_t elt = dtype == LASP2_F64 ? 8 : 4;
  void* dm = (uint8_t*)workspace + slots * nseg * (int64_t)dim * dim * elt;
  int st = lasp2_state_apply(dtype, q, d_out, m_full, workspace, dq, slots, tokens, dim, nseg, stream);
  if (st == LASP2_OK) st = lasp2_scan_segments(dtype, workspace, dm, slots, nseg, dim, 0, stream);
  if (st == LASP2_OK) st = lasp2_apply_state2(dtype, v, k, dm, dk, dv, slots, tokens, dim, stream);
  return st;
}

int lasp2_nomask_forward_phase(int dtype, const void* q, const void* k, const void* v, void* out, void* m,
                               void* workspace, int64_t workspace_bytes, int64_t slots, int64_t tokens, int dim,
                               int phase, void* stream) {
  CHECK(valid_dtype(dtype), "nomask_forward_phase: unknown dtype");
  CHECK(phase >= 1 && phase <= 3, "nomask_forward_phase: phase must be 1, 2 or 3");
  CHECK(m && workspace && ((phase & 1) ? (k && v) : true) && ((phase & 2) ? (q && out) : true),
        "nomask_forward_phase: null pointer");
  CHECK(slots >= 1 && tokens >= 1 && dim >= 1 && dim <= 128, "nomask_forward_phase: bad shape (1 <= dim <= 128)");
  const int sms = sm_count_current();
  CHECK(workspace_bytes >= lasp2_local_workspace_bytes(dtype, slots, tokens, dim, sms),
        "nomask_forward_phase: workspace too small (lasp2_local_workspace_bytes)");
  CHECK(bf16_ok(dtype, dim, tokens), BF16_ENVELOPE);
  if (use_tc(dtype, dim, tokens))
    return cuda_status(lasp::tc_flat_forward(q, k, v, out, (float*)m, workspace, slots, tokens, dim, sms, S(stream),
                                             phase),
                       "nomask_forward_phase");
  int st = LASP2_OK;
  if (phase & 1) {
    const int nseg = lasp2_num_segments(dtype, slots, tokens, dim, sms);
    st = lasp2_segment_states(dtype, k, v, workspace, slots, tokens, dim, nseg, stream);
    if (st == LASP2_OK) st = lasp2_scan_segments(dtype, workspace, m, slots, nseg, dim, 0, stream);
  }
  if (st == LASP2_OK && (phase & 2)) st = lasp2_apply_state(dtype, q, m, out, slots, tokens, dim, 0, 0, stream);
  return st;
}

static lasp::FlatXchg flat_xchg(const void* recv, const void* recv_table, const void* flags, const void* flag_table,
                                const void* acks, const void* ack_table, int rank, int nranks, void* epoch_dev) {
  return lasp::FlatXchg{(float* const*)recv_table, (unsigned long long* const*)flag_table,
                        (unsigned long long* const*)ack_table, (const float*)recv, (const unsigned long long*)flags,
                        (const unsigned long long*)acks, (unsigned long long*)epoch_dev, rank, nranks};
}

int lasp2_nomask_forward_x(const void* q, const void* k, const void* v, void* out, void* m, void* workspace,
                           int64_t workspace_bytes, int64_t slots, int64_t tokens, int dim, const void* recv,
                           const void* recv_table, const void* flags, const void* flag_table, const void* acks,
                           const void* ack_table, int rank, int nranks, void* epoch_dev, void* stream) {
  CHECK(q && k && v && out && m && workspace, "nomask_forward_x: null pointer");
  CHECK(recv && recv_table && flags && flag_table && acks && ack_table && epoch_dev, "nomask_forward_x: null exchange");
  CHECK(nranks >= 1 && rank >= 0 && rank < nranks, "nomask_forward_x: bad rank / nranks");
  CHECK(slots >= 1 && tokens >= 1 && dim >= 1 && dim <= 128 && dim % 4 == 0, "nomask_forward_x: bad shape");
  CHECK(use_tc(LASP2_BF16, dim, tokens), "nomask_forward_x: bf16 tensor-core path only");
  const int sms = sm_count_current();
  CHECK(workspace_bytes >= lasp2_local_workspace_bytes(LASP2_BF16, slots, tokens, dim, sms),
        "nomask_forward_x: workspace too small (lasp2_local_workspace_bytes)");
  const lasp::FlatXchg x = flat_xchg(recv, recv_table, flags, flag_table, acks, ack_table, rank, nranks, epoch_dev);
  return cuda_status(lasp::tc_flat_forward(q, k, v, out, (float*)m, workspace, slots, tokens, dim, sms, S(stream), 3,
                                           &x),
                     "nomask_forward_x");
}

int lasp2_nomask_backward_x(const void* q, const void* k, const void* v, const void* d_out, const void* m_full,
                            void* dm, void* dq, void* dk, void* dv, void* workspace, int64_t workspace_bytes,
                            int64_t slots, int64_t tokens, int dim, const void* recv, const void* recv_table,
                            const void* flags, const void* flag_table, const void* acks, const void* ack_table,
                            int rank, int nranks, void* epoch_dev, void* stream) {
  CHECK(q && k && v && d_out && m_full && dm && dq && dk && dv && workspace, "nomask_backward_x: null pointer");
  CHECK(recv && recv_table && flags && flag_table && acks && ack_table && epoch_dev, "nomask_backward_x: null exchange");
  CHECK(nranks >= 1 && rank >= 0 && rank < nranks, "nomask_backward_x: bad rank / nranks");
  CHECK(slots >= 1 && tokens >= 1 && dim >= 1 && dim <= 128 && dim % 4 == 0, "nomask_backward_x: bad shape");
  CHECK(use_tc(LASP2_BF16, dim, tokens), "nomask_backward_x: bf16 tensor-core path only");
  const int sms = sm_count_current();
  CHECK(workspace_bytes >= lasp2_local_workspace_bytes(LASP2_BF16, slots, tokens, dim, sms),
        "nomask_backward_x: workspace too small (lasp2_local_workspace_bytes)");
  const lasp::FlatXchg x = flat_xchg(recv, recv_table, flags, flag_table, acks, ack_table, rank, nranks, epoch_dev);
  return cuda_status(lasp::tc_flat_backward(q, k, v, d_out, (const float*)m_full, dq, dk, dv, workspace, slots, tokens,
                                            dim, sms, S(stream), (float*)dm, 3, &x),
                     "nomask_backward_x");
}

int lasp2_nomask_backward_phase(int dtype, const void* q, const void* k, const void* v, const void* d_out,
                                const void* m_full, void* dm, void* dq, void* dk, void* dv, void* workspace,
                                int64_t workspace_bytes, int64_t slots, int64_t tokens, int dim, int phase,
                                void* stream) {
  CHECK(valid_dtype(dtype), "nomask_backward_phase: unknown dtype");
  CHECK(phase >= 1 && phase <= 3, "nomask_backward_phase: phase must be 1, 2 or 3");
  CHECK(dm && workspace && ((phase & 1) ? (q && d_out && m_full && dq) : true) &&
            ((phase & 2) ? (k && v && dk && dv) : true),
        "nomask_backward_phase: null pointer");
  CHECK(slots >= 1 && tokens >= 1 && dim >= 1 && dim <= 128, "nomask_backward_phase: bad shape (1 <= dim <= 128)");
  const int sms = sm_count_current();
  CHECK(workspace_bytes >= lasp2_local_workspace_bytes(dtype, slots, tokens, dim, sms),
        "nomask_backward_phase: workspace too small (lasp2_local_workspace_bytes)");
  CHECK(bf16_ok(dtype, dim, tokens), BF16_ENVELOPE);
  if (use_tc(dtype, dim, tokens))
    return cuda_status(lasp::tc_flat_backward(q, k, v, d_out, (const float*)m_full, dq, dk, dv, workspace, slots,
                                              tokens, dim, sms, S(stream), (float*)dm, phase),
                       "nomask_backward_phase");
  int st = LASP2_OK;
  if (phase & 1) {
    const int nseg = lasp2_num_segments(dtype, slots, tokens, dim, sms);
    st = lasp2_state_apply(dtype, q, d_out, m_full, workspace, dq, slots, tokens, dim, nseg, stream);
    if (st == LASP2_OK) st = lasp2_scan_segments(dtype, workspace, dm, slots, nseg, dim, 0, stream);
  }
  if (st == LASP2_OK && (phase & 2)) st = lasp2_apply_state2(dtype, v, k, dm, dk, dv, slots, tokens, dim, stream);
  return st;
}

static int softmax_forward_impl(int dtype, const void* q, const void* k_full, const void* v_full, void* out,
                                void* lse, int64_t slots, int64_t q_tokens, int64_t kv_tokens, int dim, int causal,
                                int64_t row_offset, int64_t kv_chunk, int64_t kv_rank_stride, int64_t kv_start,
                                void* stream) {
  CHECK(valid_dtype(dtype), "softmax_forward: unknown dtype");
  CHECK(q && k_full && v_full && out && lse, "softmax_forward: null pointer");
  CHECK(slots >= 1 && q_tokens >= 1 && kv_tokens >= 1 && dim >= 1 && dim <= 128, "softmax_forward: bad shape");
  CHECK(row_offset >= 0 && (!causal || row_offset < kv_tokens), "softmax_forward: bad row_offset");
  CHECK(kv_chunk >= 1 && kv_start >= 0, "softmax_forward: bad kv_chunk / kv_start");
  const bool tc = dtype == LASP2_BF16 && lasp::tc_softmax_supported(dim, kv_chunk);
  CHECK(dtype != LASP2_BF16 || tc,
        "softmax_forward: bfloat16 needs the tcgen05 envelope: 8 <= dim <= 128, dim % 8 == 0 and kv_chunk % 128 == 0 "
        "(float32 / float64 run any shape)");
  CHECK(!tc || kv_start % 128 == 0, "softmax_forward: the bf16 path needs kv_start % 128 == 0");
  cudaError_t e;
  if (tc)
    e = lasp::tc_softmax_forward(q, k_full, v_full, out, (float*)lse, slots, q_tokens, kv_tokens, dim, causal,
                                 row_offset, kv_chunk, kv_rank_stride, S(stream), kv_start);
  else if (dtype == LASP2_F32)
    e = lasp::simt_softmax_forward<float, float>(q, k_full, v_full, out, lse, slots, q_tokens, kv_tokens, dim,
                                                 causal, row_offset, kv_chunk, kv_rank_stride, S(stream), kv_start);
  else if (dtype == LASP2_F64)
    e = lasp::simt_softmax_forward<double, double>(q, k_full, v_full, out, lse, slots, q_tokens, kv_tokens, dim,
                                                   causal, row_offset, kv_chunk, kv_rank_stride, S(stream), kv_start);
  else
    e = cudaErrorInvalidValue;  // unreachable: bf16_ok() above
  return cuda_status(e, "softmax_forward");
}

int lasp2h_softmax_forward(int dtype, const void* q, const void* k_full, const void* v_full, void* out, void* lse,
                           int64_t slots, int64_t q_tokens, int64_t kv_tokens, int dim, int causal, int64_t row_offset,
                           int64_t kv_chunk, int64_t kv_rank_stride, void* stream) {
  return softmax_forward_impl(dtype, q, k_full, v_full, out, lse, slots, q_tokens, kv_tokens, dim, causal, row_offset,
                              kv_chunk, kv_rank_stride, 0, stream);
}

int lasp2h_softmax_forward_range(int dtype, const void* q, const void* k_full, const void* v_full, void* out,
                                 void* lse, int64_t slots, int64_t q_tokens, int64_t kv_tokens, int dim, int causal,
                                 int64_t row_offset, int64_t kv_chunk, int64_t kv_rank_stride, int64_t kv_start,
                                 void* stream) {
  return softmax_forward_impl(dtype, q, k_full, v_full, out, lse, slots, q_tokens, kv_tokens, dim, causal, row_offset,
                              kv_chunk, kv_rank_stride, kv_start, stream);
}

int64_t lasp2h_softmax_scratch_bytes(int dtype, int64_t slots, int64_t q_tokens, int64_t kv_tokens, int dim) {
  (void)kv_tokens;
  const int64_t eb = dtype == LASP2_F64 ? 8 : 4;
  int64_t n = 3 * slots * q_tokens * eb + 256;
  if (dtype == LASP2_BF16) {
    const int64_t t = lasp::tc_softmax_bwd_scratch(slots, q_tokens, dim) + 256;
    if (t > n) n = t;
  }
  return n;
}

static int softmax_backward_impl(bool range, int dtype, const void* q, const void* k_full, const void* v_full, const void* out,
                            const void* lse, const void* d_out, void* dq, void* dk_full, void* dv_full, void* scratch,
                            int64_t slots, int64_t q_tokens, int64_t kv_tokens, int dim, int causal,
                            int64_t row_offset, int64_t kv_chunk, int64_t kv_rank_stride, int64_t grad_rank_stride,
                            int64_t kv_start, void* stream) {
  CHECK(!range || lse, "softmax_backward_range: needs the forward's lse of the whole key set");
  const void* lse_range = range ? lse : nullptr;
  CHECK(valid_dtype(dtype), "softmax_backward: unknown dtype");
  CHECK(q && k_full && v_full && out && d_out && dq && dk_full && dv_full && scratch,
        "softmax_backward: null pointer");
  CHECK(slots >= 1 && q_tokens >= 1 && kv_tokens >= 1 && dim >= 1 && dim <= 128, "softmax_backward: bad shape");
  CHECK(row_offset >= 0 && (!causal || row_offset < kv_tokens), "softmax_backward: bad row_offset");
  CHECK(kv_chunk >= 1 && kv_start >= 0, "softmax_backward: bad kv_chunk / kv_start");
  const bool tc = dtype == LASP2_BF16 && lasp::tc_softmax_supported(dim, kv_chunk);
  CHECK(dtype != LASP2_BF16 || tc,
        "softmax_backward: bfloat16 needs the tcgen05 envelope: 8 <= dim <= 128, dim % 8 == 0 and kv_chunk % 128 == 0 "
        "(float32 / float64 run any shape)");
  CHECK(!tc || kv_start % 128 == 0, "softmax_backward: the bf16 path needs kv_start % 128 == 0");
  cudaError_t e;
  if (tc) {
    CHECK(lse, "softmax_backward: the bf16 path needs the forward's lse");
    e = lasp::tc_softmax_backward(q, k_full, v_full, out, (const float*)lse, d_out, dq, (float*)dk_full,
                                  (float*)dv_full, scratch, slots, q_tokens, kv_tokens, dim, causal, row_offset,
                                  kv_chunk, kv_rank_stride, grad_rank_stride, S(stream), kv_start);
  } else if (dtype == LASP2_F32)
    e = lasp::simt_softmax_backward<float, float, float>(q, k_full, v_full, out, d_out, dq, dk_full, dv_full, scratch,
                                                         slots, q_tokens, kv_tokens, dim, causal, row_offset,
                                                         kv_chunk, kv_rank_stride, grad_rank_stride, S(stream), lse_range,
                                                         kv_start);
  else if (dtype == LASP2_F64)
    e = lasp::simt_softmax_backward<double, double, double>(q, k_full, v_full, out, d_out, dq, dk_full, dv_full,
                                                            scratch, slots, q_tokens, kv_tokens, dim, causal,
                                                            row_offset, kv_chunk, kv_rank_stride, grad_rank_stride,
                                                            S(stream), lse_range, kv_start);
  else
    e = cudaErrorInvalidValue;  // unreachable: bf16_ok() above
  return cuda_status(e, "softmax_backward");
}
int lasp2h_softmax_backward(int dtype, const void* q, const void* k_full, const void* v_full, const void* out,
                            const void* lse, const void* d_out, void* dq, void* dk_full, void* dv_full, void* scratch,
                            int64_t slots, int64_t q_tokens, int64_t kv_tokens, int dim, int causal,
                            int64_t row_offset, int64_t kv_chunk, int64_t kv_rank_stride, int64_t grad_rank_stride,
                            void* stream) {
  return softmax_backward_impl(false, dtype, q, k_full, v_full, out, lse, d_out, dq, dk_full, dv_full, scratch, slots,
                               q_tokens, kv_tokens, dim, causal, row_offset, kv_chunk, kv_rank_stride,
                               grad_rank_stride, 0, stream);
}

int lasp2h_softmax_backward_range(int dtype, const void* q, const void* k_full, const void* v_full, const void* out,
                                  const void* lse, const void* d_out, void* dq, void* dk_full, void* dv_full,
                                  void* scratch, int64_t slots, int64_t q_tokens, int64_t kv_tokens, int dim,
                                  int causal, int64_t row_offset, int64_t kv_chunk, int64_t kv_rank_stride,
                                  int64_t grad_rank_stride, int64_t kv_start, void* stream) {
  return softmax_backward_impl(true, dtype, q, k_full, v_full, out, lse, d_out, dq, dk_full, dv_full, scratch, slots,
                               q_tokens, kv_tokens, dim, causal, row_offset, kv_chunk, kv_rank_stride,
                               grad_rank_stride, kv_start, stream);
}


int lasp2_gen_slots(int dtype, uint64_t seed, const uint64_t* tag_words_device, void* out, int64_t slots, int64_t rows,
                    int64_t cols, int64_t row_offset, void* stream) {
  CHECK(valid_dtype(dtype), "gen_slots: unknown dtype");
  CHECK(tag_words_device && out, "gen_slots: null pointer");
  CHECK(slots >= 1 && rows >= 1 && cols >= 1 && row_offset >= 0, "gen_slots: shape must be positive");
  cudaError_t e;
  if (dtype == LASP2_F32)
    e = lasp::gen_slots<float>(seed, tag_words_device, out, slots, rows, cols, row_offset, S(stream));
  else if (dtype == LASP2_F64)
    e = lasp::gen_slots<double>(seed, tag_words_device, out, slots, rows, cols, row_offset, S(stream));
  else
    e = lasp::gen_slots<__nv_bfloat16>(seed, tag_words_device, out, slots, rows, cols, row_offset, S(stream));
  return cuda_status(e, "gen_slots");
}

int lasp2_debug_trace(void* buffer) {
  cudaError_t e = lasp::tc_set_trace((unsigned long long*)buffer);
  if (e == cudaSuccess) e = lasp::tc_set_trace_softmax((unsigned long long*)buffer);
  if (e == cudaSuccess) e = lasp::tc_set_trace_flat((unsigned long long*)buffer);
  return cuda_status(e, "debug_trace");
}

int lasp2_debug_probe_gemm(const void* a, const void* b, void* d, int a_mn, int b_mn, void* stream) {
  CHECK(a && b && d, "probe_gemm: null pointer");
  return cuda_status(lasp::tc_probe_gemm(a, b, (float*)d, a_mn, b_mn, S(stream)), "probe_gemm");
}

}  // extern "C"

// ---- collectives on a caller-provided stream ---------------------
// NCCL is resolved at run time from libnccl.so.2 — the instance torch.distributed
// already loaded when there is one, so a communicator can be shared with it —
// and the library links no NCCL at build time.
namespace {
struct Nccl {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclReduceScatter) reduce_scatter = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl x;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) return x;
    x.get_unique_id = (decltype(x.get_unique_id))dlsym(h, "ncclGetUniqueId");
    x.comm_init_rank = (decltype(x.comm_init_rank))dlsym(h, "ncclCommInitRank");
    x.comm_destroy = (decltype(x.comm_destroy))dlsym(h, "ncclCommDestroy");
    x.all_gather = (decltype(x.all_gather))dlsym(h, "ncclAllGather");
    x.reduce_scatter = (decltype(x.reduce_scatter))dlsym(h, "ncclReduceScatter");
    x.group_start = (decltype(x.group_start))dlsym(h, "ncclGroupStart");
    x.group_end = (decltype(x.group_end))dlsym(h, "ncclGroupEnd");
    x.error_string = (decltype(x.error_string))dlsym(h, "ncclGetErrorString");
    x.ok = x.get_unique_id && x.comm_init_rank && x.comm_destroy && x.all_gather && x.reduce_scatter &&
           x.group_start && x.group_end && x.error_string;
    return x;
  }();
  return n;
}

int nccl_status(ncclResult_t r, const char* where) {
  if (r == ncclSuccess) {
    g_err.clear();
    return LASP2_OK;
  }
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", where, nccl().error_string(r));
  g_err = buf;
  return LASP2_ERR_COMM;
}

bool nccl_type(int dtype, ncclDataType_t* t) {
  switch (dtype) {
    case LASP2_F32: *t = ncclFloat32; return true;
    case LASP2_F64: *t = ncclFloat64; return true;
    case LASP2_BF16: *t = ncclBfloat16; return true;
    default: return false;
  }
}
}  // namespace

#define NCCL_READY(name) CHECK(nccl().ok, name ": libnccl.so.2 not found")

int lasp2_nccl_unique_id(void* id_out) {
  NCCL_READY("nccl_unique_id");
  CHECK(id_out, "nccl_unique_id: null pointer");
  return nccl_status(nccl().get_unique_id(reinterpret_cast<ncclUniqueId*>(id_out)), "nccl_unique_id");
}

int lasp2_nccl_comm_init(void** comm_out, int nranks, const void* id, int rank) {
  NCCL_READY("nccl_comm_init");
  CHECK(comm_out && id, "nccl_comm_init: null pointer");
  CHECK(nranks >= 1 && rank >= 0 && rank < nranks, "nccl_comm_init: bad rank / nranks");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  const int st = nccl_status(nccl().comm_init_rank(&c, nranks, uid, rank), "nccl_comm_init");
  *comm_out = c;
  return st;
}

int lasp2_nccl_comm_destroy(void* comm) {
  NCCL_READY("nccl_comm_destroy");
  CHECK(comm, "nccl_comm_destroy: null communicator");
  return nccl_status(nccl().comm_destroy((ncclComm_t)comm), "nccl_comm_destroy");
}

int lasp2_state_allgather(void* comm, int dtype, const void* state, void* gathered, int64_t count, void* stream) {
  NCCL_READY("state_allgather");
  ncclDataType_t t;
  CHECK(nccl_type(dtype, &t), "state_allgather: unknown dtype");
  CHECK(comm && state && gathered, "state_allgather: null pointer");
  CHECK(count >= 1, "state_allgather: count must be positive");
  return nccl_status(nccl().all_gather(state, gathered, (size_t)count, t, (ncclComm_t)comm, S(stream)),
                     "state_allgather");
}

int lasp2h_kv_allgather(void* comm, int dtype, const void* k_chunk, const void* v_chunk, void* k_full, void* v_full,
                        int64_t count, void* stream) {
  NCCL_READY("kv_allgather");
  ncclDataType_t t;
  CHECK(nccl_type(dtype, &t), "kv_allgather: unknown dtype");
  CHECK(comm && k_chunk && v_chunk && k_full && v_full, "kv_allgather: null pointer");
  CHECK(count >= 1, "kv_allgather: count must be positive");
  int st = nccl_status(nccl().all_gather(k_chunk, k_full, (size_t)count, t, (ncclComm_t)comm, S(stream)),
                       "kv_allgather (K)");
  if (st != LASP2_OK) return st;
  return nccl_status(nccl().all_gather(v_chunk, v_full, (size_t)count, t, (ncclComm_t)comm, S(stream)),
                     "kv_allgather (V)");
}

int lasp2h_grad_reduce_scatter(void* comm, int dtype, const void* contrib, void* out, int64_t recv_count,
                               void* stream) {
  NCCL_READY("grad_reduce_scatter");
  ncclDataType_t t;
  CHECK(nccl_type(dtype, &t), "grad_reduce_scatter: unknown dtype");
  CHECK(comm && contrib && out, "grad_reduce_scatter: null pointer");
  CHECK(recv_count >= 1, "grad_reduce_scatter: count must be positive");
  return nccl_status(
      nccl().reduce_scatter(contrib, out, (size_t)recv_count, t, ncclSum, (ncclComm_t)comm, S(stream)),
      "grad_reduce_scatter");
}
