/*
 * lasp2_b200.h — C ABI of the B200-native LASP-2 / LASP-2H hot path.
 *
 * Plain pointers and sizes only. Every entry point is stream-ordered and
 * asynchronous: it enqueues work on `stream` (a cudaStream_t passed as void*,
 * NULL = legacy default stream) and returns a status code; no entry point
 * allocates caller-visible memory, frees caller memory or synchronises.
 * Errors never cross the ABI as exceptions: a non-zero status is returned and
 * lasp2_last_error() describes it (thread-local).
 *
 * Tensor layout (reference shards.py:13-39): per-rank tensors
 * are BHND row-major, i.e. `slots` = B*H independent (tokens x dim) matrices
 * stored back to back. Memory states are (slots, dim, dim) row-major with
 * state[a][c] = sum_i x[i][a] * y[i][c]  (reference lasp2.py:130-137).
 *
 * Precision follows the data dtype (reference WorldConfig.element_bytes,
 * comm.py:78-79):
 *   LASP2_F64  : f64 in/out, f64 states       (reference-precision validation)
 *   LASP2_F32  : f32 in/out, f32 states       (fp32 validation mode)
 *   LASP2_BF16 : bf16 in/out, f32 states      (tcgen05/TMEM/TMA fast path)
 *
 * Each function names the reference interface it replaces (file:line under
 * the reference's pkg/src/laspsim/).
 */
#ifndef LASP2_B200_H
#define LASP2_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum lasp2_dtype { LASP2_F32 = 0, LASP2_F64 = 1, LASP2_BF16 = 2 };
enum lasp2_status { LASP2_OK = 0, LASP2_ERR_INVALID = 1, LASP2_ERR_CUDA = 2, LASP2_ERR_UNSUPPORTED = 3,
                    LASP2_ERR_COMM = 4 };
enum lasp2_fold_mode { LASP2_FOLD_PREFIX = 0, LASP2_FOLD_SUFFIX = 1, LASP2_FOLD_FULL = 2 };

/* ABI version (major*100 + minor). */
int lasp2_version(void);
/* Description of the last error on this thread ("" if none). */
const char* lasp2_last_error(void);

/* Number of sequence segments the kernels split one rank's chunk into for
 * `slots` slots of `tokens` tokens on a device with `sm_count` SMs. Segment
 * boundaries are whole 128-token blocks. Host helper, no device work. */
int lasp2_num_segments(int dtype, int64_t slots, int64_t tokens, int dim, int sm_count);

/* seg_states[slot][s] = X_s^T Y_s over segment s of the rank's chunk.
 * Replaces chunk_state (lasp2.py:130-137) with (x,y)=(K,V) and chunk_state_grad
 * (lasp2.py:140-147) with (x,y)=(Q,dO), split into `nseg` segments. */
int lasp2_segment_states(int dtype, const void* x, const void* y, void* seg_states, int64_t slots, int64_t tokens,
                         int dim, int nseg, void* stream);

/* In place exclusive scan over segments (reverse=0: prefix, 1: suffix) and the
 * chunk total (the rank's M_t / dM_t, the AllGather payload; `chunk_total`
 * may be NULL). First-term-copy fold order as numerics.py:71-116. */
int lasp2_scan_segments(int dtype, void* seg_states, void* chunk_total, int64_t slots, int nseg, int dim, int reverse,
                        void* stream);

/* Fused state exchange over peer memory (replaces the NCCL
 * AllGather of RankContext.all_gather, comm.py:367-412, for the state payload).
 * lasp2_scan_put = lasp2_scan_segments plus: the chunk total is stored into
 * slot `rank` of half (epoch & 1) of every rank's receive buffer
 * ([2][nranks][slots*dim*dim], states dtype; `peer_recv` is a DEVICE array of
 * nranks pointers, one per rank, e.g. symmetric-memory peer addresses over
 * NVLink) and, once every element is stored, flag[rank] of every rank
 * (`peer_flags`, device array of nranks pointers to uint64[nranks]) is set to
 * `epoch` with a system-scope release. `done` is a zeroed uint32 the launch
 * re-arms. Epochs start at 1 and grow per exchange. lasp2_exchange_wait
 * blocks the stream until flags[lo..hi) (a uint64 array) carry `epoch`; after
 * waiting on this rank's flags, half (epoch & 1) of the receive buffer is
 * folded with lasp2_fold_states exactly like an all_gather result, and
 * lasp2_exchange_ack then sets acks[rank] = epoch on every rank (`peer_acks`,
 * device array of nranks pointers to uint64[nranks]). Before a put of epoch
 * e > 2 the caller waits on its own acks[0..nranks) for e - 2, so no reader
 * still needs the half being overwritten.
 * Device-resident epoch (`epoch_dev`, a zeroed uint64 per rank and exchange; NULL =
 * the host `epoch` above): lasp2_scan_put uses *epoch_dev + 1 and stores it back,
 * the other calls use *epoch_dev + (int64_t)epoch (an offset: 0 for this
 * exchange's flags and acks, -1 for the back-pressure wait before the next put),
 * and lasp2_exchange_fold folds half (*epoch_dev & 1). Every value is read on the
 * device, so a captured CUDA graph advances the exchange on each replay. */
int lasp2_scan_put(int dtype, void* seg_states, void* chunk_total, int64_t slots, int nseg, int dim, int reverse,
                   const void* peer_recv, const void* peer_flags, int rank, int nranks, uint64_t epoch, void* done,
                   void* epoch_dev, void* stream);
int lasp2_exchange_wait(const void* flags, int lo, int hi, uint64_t epoch, const void* epoch_dev, void* stream);
int lasp2_exchange_ack(const void* peer_acks, int rank, int nranks, uint64_t epoch, const void* epoch_dev,
                       void* stream);
/* lasp2_fold_states over half (*epoch_dev & 1) of a receive buffer whose halves are
 * half_elems apart. */
int lasp2_exchange_fold(int dtype, const void* recv, int64_t half_elems, const void* epoch_dev, void* out,
                        int nstates, int64_t elems, int mode, int bound, void* stream);

/* out = ordered fold of `nstates` gathered states, each `elems` elements,
 * stored rank-major ([nstates][elems], the all_gather layout):
 *   PREFIX(bound): states[0:bound] ascending  = prefix_sum_states (numerics.py:71-90)
 *   SUFFIX(bound): states[bound:] descending  = suffix_sum_states (numerics.py:93-116)
 *   FULL         : all ascending              = sum_states        (numerics.py:119-121) */
int lasp2_fold_states(int dtype, const void* gathered, void* out, int nstates, int64_t elems, int mode, int bound,
                      void* stream);

/* Causal linear attention over one rank's chunk with the inter-chunk state
 * folded in:  out_s = q_s S_s + sum_{i<=s} (q_s.k_i) v_i, where
 * S_s = base + seg_states[seg(s)] + sum_{i<s, same segment} k_i^T v_i.
 * reverse=1 runs the anti-causal form (i>=s, states from the chunk end);
 * transpose_state=1 uses S^T. `base` / `seg_states` may be NULL (zero).
 * Replaces intra_forward (lasp2.py:168-174, oracle.py:50-62) plus the inter
 * term `out += apply_state(q, m_prefix)` (lasp2.py:238-240); with permuted
 * operands it also computes the masked backward's dQ/dK/dV (lasp2.py:270-285). */
int lasp2_causal_chunk(int dtype, const void* q, const void* k, const void* v, const void* seg_states,
                       const void* base, void* out, int64_t slots, int64_t tokens, int dim, int nseg, int reverse,
                       int transpose_state, void* stream);

/* bf16 lasp2_causal_chunk / lasp2_dkdv_chunk that consume a fused peer
 * exchange (lasp2_scan_put) in their prologue instead of a folded `base`: each
 * CTA waits until the uint64 flags[lo..hi) carry `epoch`, folds those ranks'
 * states from the receive half `xrecv` ([T][slots][dim][dim]: ascending with
 * the first term copied, descending for dK/dV's suffix — numerics.py:71-116)
 * and seeds its state with it. base_out (causal_chunk_x, may be NULL)
 * receives the folded base ([slots][dim][dim], the cache's M_{1:t-1}). The
 * caller acknowledges the epoch afterwards (lasp2_exchange_ack). This removes
 * the wait and fold launches between the collective and its consumer.
 * xflags = NULL: no wait — `xrecv` is a complete rank-major all_gather result
 * already ordered before `stream` (the NCCL path: the prefix / suffix fold of
 * the gathered states fused into the consumer's prologue, no fold launch).
 * epoch_dev != NULL: the epoch is *epoch_dev (device-resident, see lasp2_scan_put)
 * and `xrecv` is the whole receive buffer, the half (epoch & 1) half_elems apart. */
int lasp2_causal_chunk_x(const void* q, const void* k, const void* v, const void* seg_states, const void* xrecv,
                         const void* xflags, int lo, int hi, int descending, uint64_t epoch, const void* epoch_dev,
                         int64_t half_elems, void* base_out, void* out, int64_t slots, int64_t tokens, int dim,
                         int nseg, int reverse, int transpose_state, void* stream);
int lasp2_dkdv_chunk_x(const void* q, const void* k, const void* v, const void* d_out, const void* seg_states,
                       const void* xrecv, const void* xflags, int lo, int hi, uint64_t epoch, const void* epoch_dev,
                       int64_t half_elems, void* dk, void* dv, int64_t slots, int64_t tokens, int dim, int nseg,
                       void* stream);

/* Masked backward dQ of one rank's chunk plus the dM segment states, one pass:
 *   dq_s = sum_{i<=s} (do_s.v_i) k_i + do_s S_s^T,  S_s = fwd_base + fwd_seg[seg(s)]
 *          + sum_{i<s, same segment} k_i^T v_i   (lasp2.py:198, :277-279)
 *   g_seg[slot][g] = Q_g^T dO_g  (chunk_state_grad per segment, lasp2.py:140-147;
 *          unscanned, the caller's lasp2_scan_segments turns it into suffixes).
 * Replaces the dq half of intra_backward and chunk_state_grad; the bf16 path
 * reads dO, V, K and Q once (one tcgen05 pass instead of two). */
int lasp2_dq_chunk(int dtype, const void* q, const void* k, const void* v, const void* d_out, const void* fwd_seg,
                   const void* fwd_base, void* g_seg, void* dq, int64_t slots, int64_t tokens, int dim, int nseg,
                   void* stream);

/* Masked backward dK and dV of one rank's chunk in one pass:
 *   dk_s = sum_{i>=s} (v_s.do_i) q_i + v_s G_s^T,  dv_s = sum_{i>=s} (k_s.q_i) do_i + k_s G_s
 * with G_s = base + seg_states[seg(s)] + sum_{i>s, same segment} q_i^T do_i
 * (seg_states = exclusive suffix of Q^T dO segment states, base = suffix fold of
 * the gathered dM). Replaces the dk/dv halves of intra_backward
 * (lasp2.py:199-202) plus lasp2.py:280-284. The bf16 path runs 2-CTA clusters
 * that TMA-multicast Q and dO to both SMs (4 tile reads per block, not 6). */
int lasp2_dkdv_chunk(int dtype, const void* q, const void* k, const void* v, const void* d_out, const void* seg_states,
                     const void* base, void* dk, void* dv, int64_t slots, int64_t tokens, int dim, int nseg,
                     void* stream);

/* The whole masked backward of one rank's chunk in one launch (lasp2.py:270-285):
 *   dq = causal(dO, V, K; state S^T),  S = fwd_base + fwd_seg (exclusive K^T V
 *        segment prefixes; fwd_total is the chunk total), i.e. lasp2.py:277-279;
 *   dk, dv as lasp2_dkdv_chunk with G from bwd_seg / bwd_base (lasp2.py:280-284).
 * The bf16 path runs three CTAs per segment (dQ, dK, dV) that stream Q, K, V, dO
 * in the same order so L2 absorbs the re-reads; dQ walks its segment backwards
 * from the segment-end state, subtracting K^T V per block. */
int lasp2_backward_chunk(int dtype, const void* q, const void* k, const void* v, const void* d_out,
                         const void* fwd_seg, const void* fwd_total, const void* fwd_base, const void* bwd_seg,
                         const void* bwd_base, void* dq, void* dk, void* dv, int64_t slots, int64_t tokens, int dim,
                         int nseg, void* stream);

/* The same backward with every CTA walking its segment forwards (the bf16 path:
 * three CTAs per segment streaming Q, K, V, dO in the same order, no subtract
 * form): dK / dV use the suffix INCLUSIVE of the current block,
 *   dk_j = v_j G_{>=j}^T - strict(V_j dO_j^T) Q_j,  dv_j = k_j G_{>=j} - strict(K_j Q_j^T) dO_j,
 * seeded per segment with bwd_base + (seg > 0 ? bwd_seg[seg-1] : bwd_total), where
 * bwd_seg is the exclusive suffix scan of the Q^T dO segment states (as
 * lasp2_scan_segments(reverse=1) leaves it) and bwd_total its chunk total; dq as
 * lasp2_backward_chunk (fwd_seg exclusive K^T V prefixes, fwd_base M_{1:t-1}).
 * Replaces intra_backward + both inter terms (lasp2.py:270-285) in one launch. */
int lasp2_backward_chunk_fwd(int dtype, const void* q, const void* k, const void* v, const void* d_out,
                             const void* fwd_seg, const void* fwd_base, const void* bwd_seg, const void* bwd_total,
                             const void* bwd_base, void* dq, void* dk, void* dv, int64_t slots, int64_t tokens,
                             int dim, int nseg, void* stream);

/* out (+)= x M (transpose=0) or x M^T (transpose=1) per slot.
 * Replaces apply_state / apply_state_t (lasp2.py:150-165). */
int lasp2_apply_state(int dtype, const void* x, const void* m, void* out, int64_t slots, int64_t tokens, int dim,
                      int transpose, int accumulate, void* stream);

/* Hybrid-stack projections (replaces the W_Q/K/V GEMMs of hybrid.py:136-151):
 * out (+)= sum_{i<nx} xs[i] op(ws[i]) per (batch, head) slot, op = W (transpose 0)
 * or W^T (transpose 1), every ws[i] one [dim][dim] weight in the states dtype
 * (f32 for bf16 data) shared by all slots; xs[i] / out [slots][tokens][dim].
 * nx = 1 (accumulate allowed) or 3 (the chain-rule dX = dQ W_Q^T + dK W_K^T +
 * dV W_V^T with one rounding). bf16: tcgen05 kernels. */
int lasp2_project(int dtype, const void* const* xs, const void* const* ws, int nx, void* out, int64_t slots,
                  int64_t tokens, int dim, int transpose, int accumulate, void* stream);

/* Unmasked backward, fused (lasp2.py:256-267): seg_states[slot][g] = Q_g^T dO_g
 * (the dM segments, scanned by lasp2_scan_segments) and dq = dO M^T, reading Q and
 * dO once. `m` = the forward's M_{1:T} (states dtype). */
int lasp2_state_apply(int dtype, const void* q, const void* d_out, const void* m, void* seg_states, void* dq,
                      int64_t slots, int64_t tokens, int dim, int nseg, void* stream);

/* Unmasked backward dk = v dM^T and dv = k dM in one pass (lasp2.py:265-266). */
int lasp2_apply_state2(int dtype, const void* v, const void* k, const void* dm, void* dk, void* dv, int64_t slots,
                       int64_t tokens, int dim, void* stream);

/* Unmasked layer on a world of ONE rank (T = 1: the state all_gather is the
 * identity and sum_states of one state is a copy). Replaces
 * _forward_nomask_rank (lasp2.py:208-216) and _backward_nomask_rank
 * (lasp2.py:256-267) for sp_size == 1.
 *   forward : m_full = K^T V (states dtype), out = q m_full
 *   backward: dM = Q^T dO; dq = dO m_full^T; dk = v dM^T; dv = k dM
 * bf16 runs one persistent launch per direction over all SMs (cooperative:
 * it needs the whole GPU while it runs; in-kernel grid barrier + ordered
 * reduction of per-CTA partial states). `workspace` must hold
 * lasp2_local_workspace_bytes(...) bytes and be ZERO-FILLED before its first
 * use; every call leaves it reusable. One workspace per concurrently running
 * call. f32/f64 compose lasp2_segment_states / scan / apply entry points. */
int64_t lasp2_local_workspace_bytes(int dtype, int64_t slots, int64_t tokens, int dim, int sm_count);
int lasp2_nomask_forward_local(int dtype, const void* q, const void* k, const void* v, void* out, void* m_full,
                               void* workspace, int64_t workspace_bytes, int64_t slots, int64_t tokens, int dim,
                               void* stream);
int lasp2_nomask_backward_local(int dtype, const void* q, const void* k, const void* v, const void* d_out,
                                const void* m_full, void* dq, void* dk, void* dv, void* workspace,
                                int64_t workspace_bytes, int64_t slots, int64_t tokens, int dim, void* stream);

/* The same persistent kernels split around the state all_gather of a world
 * of T > 1 ranks (the unmasked rank programs, lasp2.py:208-216, :256-267):
 *   forward  phase 1: m = K^T V, this rank's chunk state M_t (the payload);
 *            phase 2: out = Q m, m = the folded M_{1:T} (sum_states).
 *   backward phase 1: dq = dO m_full^T and dm = Q^T dO (this rank's dM_t);
 *            phase 2: dk = V dm^T, dv = K dm, dm = the folded dM_{1:T}.
 * One launch per phase over all SMs (phase 1 with its in-kernel ordered
 * reduction, phase 2 dynamically scheduled); same workspace contract as the
 * _local entries; phase 3 = both (the world-of-one call). */
int lasp2_nomask_forward_phase(int dtype, const void* q, const void* k, const void* v, void* out, void* m,
                               void* workspace, int64_t workspace_bytes, int64_t slots, int64_t tokens, int dim,
                               int phase, void* stream);
int lasp2_nomask_backward_phase(int dtype, const void* q, const void* k, const void* v, const void* d_out,
                                const void* m_full, void* dm, void* dq, void* dk, void* dv, void* workspace,
                                int64_t workspace_bytes, int64_t slots, int64_t tokens, int dim, int phase,
                                void* stream);

/* The unmasked layer of one rank of a T-rank world as ONE launch per direction,
 * the state all_gather fused in (the peer exchange of
 * lasp2_scan_put, bf16, one GPU per rank): phase 1 as lasp2_nomask_*_phase;
 * the in-kernel reduction that produces this rank's chunk state stores it
 * straight into slot `rank` of every rank's receive half (recv_table: T peer
 * addresses of [2][T][slots][dim][dim] fp32, half = epoch parity) after every
 * reader acknowledged the exchange two epochs back; the last CTA to have fenced
 * its stores releases this rank's flag on every rank (flag_table), every CTA
 * waits for all T flags, the full sum is folded in ascending rank order
 * (numerics.py:119-121) into m / dm, and after a grid barrier the epoch is
 * acknowledged to every writer (ack_table) and *epoch_dev advanced; then
 * phase 2. Replaces
 * chunk_state + all_gather + sum_states + apply_state of _forward_nomask_rank
 * (lasp2.py:208-216) and its backward (lasp2.py:256-267). Every rank's kernel
 * must be able to run concurrently (one GPU per rank, or time-sliced
 * processes): a peer that never arrives traps after ~2^36 cycles. */
int lasp2_nomask_forward_x(const void* q, const void* k, const void* v, void* out, void* m, void* workspace,
                           int64_t workspace_bytes, int64_t slots, int64_t tokens, int dim, const void* recv,
                           const void* recv_table, const void* flags, const void* flag_table, const void* acks,
                           const void* ack_table, int rank, int nranks, void* epoch_dev, void* stream);
int lasp2_nomask_backward_x(const void* q, const void* k, const void* v, const void* d_out, const void* m_full,
                            void* dm, void* dq, void* dk, void* dv, void* workspace, int64_t workspace_bytes,
                            int64_t slots, int64_t tokens, int dim, const void* recv, const void* recv_table,
                            const void* flags, const void* flag_table, const void* acks, const void* ack_table,
                            int rank, int nranks, void* epoch_dev, void* stream);

/* LASP-2H softmax attention of one chunk of queries (global rows
 * [row_offset, row_offset+q_tokens)) against full-length keys/values.
 * Full-length tensors may be rank-major as the collectives produce them:
 * key j of slot s is at element (j / kv_chunk) * kv_rank_stride +
 * (s * kv_chunk + j % kv_chunk) * dim (kv_chunk = kv_tokens, stride 0 is the
 * plain [slots][kv_tokens][dim] layout). The dk/dv contributions use the
 * same indexing with grad_rank_stride, so a [T][2][slots][chunk][dim] buffer
 * feeds one reduce-scatter.
 * out = softmax(q k^T / sqrt(d), causal by global position) v; lse (states
 * dtype: f64 for f64 data, else f32; [slots][q_tokens]) receives the row
 * log-sum-exp (natural log). Replaces
 * softmax_chunk_forward (oracle.py:136-139) as called by _cp_forward_rank
 * (standard_sp.py:44-49). */
int lasp2h_softmax_forward(int dtype, const void* q, const void* k_full, const void* v_full, void* out, void* lse,
                           int64_t slots, int64_t q_tokens, int64_t kv_tokens, int dim, int causal, int64_t row_offset,
                           int64_t kv_chunk, int64_t kv_rank_stride, void* stream);
/* The same over the key range [kv_start, kv_start + kv_tokens) of the
 * rank-major layout (k_full / v_full still point at rank 0; kv_tokens need not
 * be a multiple of kv_chunk; row_offset is relative to kv_start; the bf16 path
 * needs kv_start % 128 == 0). The balanced LASP-2H schedule's half-chunk
 * splits; no reference counterpart. */
int lasp2h_softmax_forward_range(int dtype, const void* q, const void* k_full, const void* v_full, void* out,
                                 void* lse, int64_t slots, int64_t q_tokens, int64_t kv_tokens, int dim, int causal,
                                 int64_t row_offset, int64_t kv_chunk, int64_t kv_rank_stride, int64_t kv_start,
                                 void* stream);

/* Gradients of <d_out, softmax_chunk_forward(...)>: dq for the chunk and this
 * chunk's full-length dk/dv contributions (accumulate dtype: f32 for bf16/f32,
 * f64 for f64). `scratch` must hold lasp2h_softmax_scratch_bytes() bytes.
 * Replaces softmax_chunk_backward (oracle.py:142-158) as called by
 * _cp_backward_rank (standard_sp.py:64-68). */
int lasp2h_softmax_backward(int dtype, const void* q, const void* k_full, const void* v_full, const void* out,
                            const void* lse, const void* d_out, void* dq, void* dk_full, void* dv_full, void* scratch,
                            int64_t slots, int64_t q_tokens, int64_t kv_tokens, int dim, int causal,
                            int64_t row_offset, int64_t kv_chunk, int64_t kv_rank_stride, int64_t grad_rank_stride,
                            void* stream);

/* The same over a key SUB-RANGE of a larger softmax (the balanced LASP-2H
 * schedule splits one query chunk's keys between two ranks): P uses the
 * forward's lse of the whole key set and delta = rowsum(dO o O) with the
 * final O, so partial dQ and dK/dV contributions of disjoint ranges add up
 * to the full gradients. Identical to lasp2h_softmax_backward on the bf16
 * tensor-core path; the f32/f64 path would otherwise renormalise over its
 * range. lse must be given (states dtype). The keys are [kv_start, kv_start +
 * kv_tokens) of the rank-major layout as in lasp2h_softmax_forward_range (dk /
 * dv land at the absolute key index). */
int lasp2h_softmax_backward_range(int dtype, const void* q, const void* k_full, const void* v_full, const void* out,
                                  const void* lse, const void* d_out, void* dq, void* dk_full, void* dv_full,
                                  void* scratch, int64_t slots, int64_t q_tokens, int64_t kv_tokens, int dim,
                                  int causal, int64_t row_offset, int64_t kv_chunk, int64_t kv_rank_stride,
                                  int64_t grad_rank_stride, int64_t kv_start, void* stream);
int64_t lasp2h_softmax_scratch_bytes(int dtype, int64_t slots, int64_t q_tokens, int64_t kv_tokens, int dim);

/* Deterministic inputs: out[slot] = rows [row_offset, row_offset+rows) of
 * gen_data(seed, *, cols, tag_slot) where tag_words[slot] is the 64-bit blake2b
 * word of the slot's tag. Bit-exact port of gen_data / gen_slots
 * (datagen.py:33-71); bf16 rounds f64->f32->bf16. row_offset lets each rank
 * generate only its own chunk of the full sequence. */
int lasp2_gen_slots(int dtype, uint64_t seed, const uint64_t* tag_words_device, void* out, int64_t slots, int64_t rows,
                    int64_t cols, int64_t row_offset, void* stream);

/* Test hook: d (f32 128x128) = op(a) op(b)^T for bf16 128x128 tiles with the
 * UMMA descriptor convention of the fast path (a_mn / b_mn select MN-major;
 * a_mn = 2 stages A in TMEM and runs the TS-mode MMA). */
int lasp2_debug_probe_gemm(const void* a, const void* b, void* d, int a_mn, int b_mn, void* stream);

/* Test hook: record a clock64() timeline of CTA (0,0) of the causal kernels into
 * `buffer` (4096 x {event, block, clock} uint64; NULL disables). */
int lasp2_debug_trace(void* buffer);

/* ---- collectives on the caller's stream ----
 * NCCL over NVLink; libnccl.so.2 is resolved at run time (the instance
 * torch.distributed loaded, if any), so `comm` may be an ncclComm_t created
 * here or by the host framework. LASP2_ERR_COMM + lasp2_last_error() on an
 * NCCL failure; LASP2_ERR_INVALID if the library is absent. */
/* ncclGetUniqueId into 128 bytes at id_out (rank 0 shares them out of band). */
int lasp2_nccl_unique_id(void* id_out);
/* ncclCommInitRank: *comm_out = communicator of `nranks` ranks, this one `rank`. */
int lasp2_nccl_comm_init(void** comm_out, int nranks, const void* id, int rank);
int lasp2_nccl_comm_destroy(void* comm);
/* The state AllGather of every LASP-2 pass (RankContext.all_gather,
 * comm.py:367-412, as called at lasp2.py:211/226/232/260/276): `count`
 * elements of this rank's chunk state (pack_slots payload, shards.py:24-29)
 * -> gathered [nranks][count], rank-major (what lasp2_fold_states reads).
 * dtype = the element type moved (LASP2_F32 states for bf16/f32 data). */
int lasp2_state_allgather(void* comm, int dtype, const void* state, void* gathered, int64_t count, void* stream);
/* LASP-2H K and V AllGathers (standard_sp.py:40-41, two launches as in the
 * reference ledger): `count` = slots*chunk*dim elements per rank -> the
 * rank-major [nranks][slots][chunk][dim] layout the softmax kernels read. */
int lasp2h_kv_allgather(void* comm, int dtype, const void* k_chunk, const void* v_chunk, void* k_full, void* v_full,
                        int64_t count, void* stream);
/* LASP-2H dK/dV exchange: ReduceScatter (sum) of the rank-major
 * [nranks][2][slots][chunk][dim] contributions -> this rank's
 * [2][slots][chunk][dim] (replaces the stacked all_gather + ascending sum of
 * standard_sp.py:69-75; recv_count = 2*slots*chunk*dim). */
int lasp2h_grad_reduce_scatter(void* comm, int dtype, const void* contrib, void* out, int64_t recv_count,
                               void* stream);

#ifdef __cplusplus
}
#endif

#endif /* LASP2_B200_H */
