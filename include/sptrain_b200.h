/*
 * sptrain_b200 — C-ABI of the B200-native ALST (arXiv 2506.13996) sequence-parallel layer step.
 *
 * The reference's public surface for this path is the C++ namespace `sptrain`
 * (/root/reference/proj/include/sptrain/*.hpp) plus the operations SPEC.md specifies on top of it
 * (plan_head_shards, seq_to_head, head_to_seq, replicate_kv, ulysses_attention, tiled_mlp,
 * tiled_logits_loss, cross_entropy, preshift/shard/pad, all_to_all, all_reduce_sum).  Each entry
 * point below names the reference interface it replaces.  Plain pointers and sizes only; every
 * device pointer is caller-owned; `stream` is a cudaStream_t (NULL = legacy default stream).
 * Errors: every call returns spt_status (the errors.hpp:12-72 taxonomy) and sets a thread-local
 * message readable with spt_last_error().  There is no CPU fallback: without a usable sm_100a
 * device the compute entry points fail with SPT_ERR_CUDA.
 *
 * Integration notes (ctypes / C++ bindings): see INTEGRATION.md.
 */
#ifndef SPTRAIN_B200_H
#define SPTRAIN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* errors.hpp:12-72 -> status codes */
typedef enum {
    SPT_OK = 0,
    SPT_ERR_SHAPE = 1,       /* errors.hpp:19 ShapeError */
    SPT_ERR_VALIDATION = 2,  /* errors.hpp:13 ValidationError (labels, position ids, head plans) */
    SPT_ERR_COLLECTIVE = 3,  /* errors.hpp:25 CollectiveError */
    SPT_ERR_PROTOCOL = 4,    /* errors.hpp:31 ProtocolError (NCCL async error / timeout) */
    SPT_ERR_OOM = 5,         /* errors.hpp:55 SimulatedOomError (ledger budget) or cudaMalloc failure */
    SPT_ERR_CUDA = 6,        /* CUDA runtime / driver failure, missing device */
    SPT_ERR_CONFIG = 7,      /* errors.hpp:68 ConfigError */
    SPT_ERR_DETERMINISM = 8, /* errors.hpp:37 DeterminismError */
    SPT_ERR_INTERNAL = 9
} spt_status;

const char* spt_last_error(void);
/* Run-time tuning switches for A/B experiments (GEMM: gemm_1sm, gemm_pair_mn, gemm_bn, epi_tstore, gemm_raster,
 * gemm_group_m, gemm_colgroup; attention: attn_fwd_bk128, attn_fwd_hybrid, attn_fwd_tmem, attn_kv_group,
 * attn_dkdv_kt, attn_dkdv_pair, attn_dq_tmem, attn_bwd; engine: mlp_bwd_group, rope_fused).  The defaults are the
 * measured-best configuration (DESIGN.md §4 lists every switch with its evidence); unknown names are an error. */
spt_status spt_tuning_set(const char* name, int32_t value);
const char* spt_version(void);

/* ============================ host-only logic (no GPU needed) ============================ */

/* SPEC.md:286-292 HeadShardPlan */
typedef struct {
    int32_t sp_degree;
    int32_t q_heads;
    int32_t kv_heads;
    int32_t q_heads_per_rank;
    int32_t kv_heads_per_rank;
    int32_t kv_replication; /* r */
} spt_head_shard_plan;

/* SPEC.md:296-305 plan_head_shards. Rejects Hq % P != 0 ("q_heads not divisible by SP degree"),
 * Hkv >= P with Hkv % P != 0, and P % Hkv != 0 when Hkv < P, with SPT_ERR_VALIDATION. */
spt_status spt_plan_head_shards(int32_t q_heads, int32_t kv_heads, int32_t sp_degree, spt_head_shard_plan* out);
/* Global head indices rank `rank` owns after seq_to_head. kind 0 = q heads, 1 = kv heads. */
spt_status spt_plan_heads_of(const spt_head_shard_plan* plan, int32_t rank, int32_t kind, int32_t* out_heads,
                             int32_t capacity, int32_t* n_out);

/* SPEC.md:512-519 preshift_labels: out[i] = labels[i+1], out[s-1] = -100. */
spt_status spt_preshift_labels(const int64_t* labels, int64_t s, int64_t* out);
/* SPEC.md:531-535 pad_to_multiple: returns the padded length; fills the tail (token 0, label -100,
 * isolated position run) into the caller's buffers when they have room for it (cap >= padded). */
spt_status spt_pad_to_multiple(int64_t* input_ids, int64_t* position_ids, int64_t* shift_labels, int64_t s,
                               int32_t sp_degree, int64_t cap, int64_t* padded_len);
/* SPEC.md:243-251 derive_block_causal_mask_predicate, host validation + start index per token. */
spt_status spt_block_causal_starts(const int64_t* position_ids, int64_t s, int64_t* starts_out);

/* All-to-all schedule of the Ulysses reshard for one rank.
 * direction 0 = seq_to_head of fused QKV, 1 = head_to_seq of O, 2 = seq_to_head of dO,
 * 3 = head_to_seq of dQKV.  Element counts (bf16) per peer, in rank order. */
spt_status spt_a2a_counts(const spt_head_shard_plan* plan, int64_t s_loc, int32_t head_dim, int32_t direction,
                          int64_t* send_counts, int64_t* recv_counts);

/* ================================ memest ================================ */
typedef struct {
    double weights_bytes, optimizer_bytes, master_weights_bytes, grads_bytes, total_bytes; /* 2/8/4/4 B per param */
    double device_bytes_per_gpu; /* fixed share on one GPU (ZeRO-3 divides by world size; optimizer offload
                                    moves optimizer + master weights to host) */
    double host_bytes_per_gpu;
} spt_memest_fixed;
/* estimate_fixed: 8e9 params -> 144 GiB total (PAPER §2.1). */
spt_status spt_memest_fixed_bytes(double param_count, int32_t world_size, int32_t zero3, int32_t offload_optimizer,
                                  spt_memest_fixed* out);
/* estimate_logits: seqlen * vocab * bytes (4 for fp32). */
double spt_memest_logits_bytes(double seqlen, double vocab, double bytes);
/* estimate_activation_ckpt: device bytes per GPU without offload, host bytes per node with it. */
spt_status spt_memest_activation_ckpt_bytes(double seqlen, double hidden, double layers, double bytes, int32_t sp,
                                            int32_t gpus_per_node, double* device_bytes, double* host_bytes_per_node);
/* estimate_4d_mask / estimate_position_ids. */
double spt_memest_4d_mask_bytes(double seqlen, double bytes);
double spt_memest_position_ids_bytes(double seqlen, double bytes);
/* This engine's per-rank device bytes: weights, grads, logits tile workspace, checkpoints and the per-token
 * activation coefficients (act_bytes_per_token: per local token; act_bytes_per_seq_token: per GLOBAL token,
 * e.g. the full-sequence Q/K/V of the local heads), calibrated from the measured ledger. */
typedef struct {
    int32_t hidden, q_heads, kv_heads, head_dim, intermediate;
    int64_t vocab;
    int32_t n_layers, sp, ckpt_offload;
    double act_bytes_per_token, act_bytes_per_seq_token;
    int32_t embed; /* 1: token embedding table [vocab][hidden] in front of the stack (weights + grads) */
} spt_memest_engine;
spt_status spt_memest_engine_device_bytes(const spt_memest_engine* cfg, double seqlen, double* out);
/* max_seqlen_solver: largest multiple of `granularity` whose estimate fits device_budget
 * (bisection); SPT_ERR_OOM (infeasibility report in spt_last_error) when none does. */
spt_status spt_max_seqlen_solver(const spt_memest_engine* cfg, double device_budget_bytes, int64_t granularity,
                                 int64_t* out);

/* ==================================== device kernels ==================================== */

/* matmul on tcgen05: C[m,n] = alpha * sum_k A(m,k) B(n,k) (+ residual | + C).
 * A(m,k) = A[m*lda+k] if !a_mn_major else A[k*lda+m]; same for B. c_f32: C is fp32 else bf16.
 * accumulate: fp32 C += result. residual: bf16 [M, ldr] added (bf16 output only). N % 64 == 0. */
spt_status spt_gemm_bf16(const void* A, int64_t lda, int32_t a_mn_major, const void* B, int64_t ldb,
                         int32_t b_mn_major, void* C, int64_t ldc, int32_t c_f32, int32_t accumulate,
                         const void* residual, int64_t ldr, int64_t M, int64_t N, int64_t K, float alpha, void* stream);

/* RMSNorm. y = x * rstd * gamma, rstd fp32 [n]. */
spt_status spt_rmsnorm_fwd(const void* x, const void* gamma, void* y, float* rstd, int64_t n, int64_t h, float eps,
                           void* stream);
/* dx = dres + d(rmsnorm)(dy);  dgamma_accum (fp32 [h]) += sum_t dy*xhat, deterministic two-stage.
 * dres may be NULL. workspace: spt_rmsnorm_bwd_workspace(n, h) bytes. */
size_t spt_rmsnorm_bwd_workspace(int64_t n, int64_t h);
spt_status spt_rmsnorm_bwd(const void* x, const void* gamma, const float* rstd, const void* dy, const void* dres,
                           void* dx, float* dgamma_accum, void* workspace, int64_t n, int64_t h, void* stream);

/* seq_to_head send side (K1): qkv [s_loc, heads_in, d] -> send [P][s_loc][heads_out][d] with
 * send[j][t][a] = qkv[t][head_map[j*heads_out + a]] (kv replication = repeated head ids).
 * head_map is a DEVICE int32 array of P*heads_out entries. */
spt_status spt_reshard_pack(const void* src, int64_t s_loc, int32_t heads_in, int32_t head_dim, int32_t P,
                            int32_t heads_out, const int32_t* head_map, void* dst, void* stream);
/* K1 with RoPE fused: as spt_reshard_pack, with source heads < n_rot (q and k heads)
 * rotated on the way (positions: DEVICE int64 position_ids [s_loc] or pos_offset + t; base theta); bitwise
 * equal to spt_rope followed by spt_reshard_pack.  head_dim % 16 == 0 and head_dim in {32, 64, 128}. */
spt_status spt_reshard_pack_rope(const void* src, int64_t s_loc, int32_t heads_in, int32_t head_dim, int32_t P,
                                 int32_t heads_out, const int32_t* head_map, void* dst, int32_t n_rot,
                                 const int64_t* position_ids, int64_t pos_offset, float theta,
                                 const void* cos_sin_table, void* stream);
/* RoPE angle table for positions [0, npos): (cos, sin) fp32 pairs [npos][head_dim / 2], bit-identical to the
 * angles the kernels compute themselves (npos * head_dim * 4 bytes).  Optional argument of
 * spt_reshard_pack_rope (NULL: computed in-kernel); the layer engine builds one at creation. */
spt_status spt_rope_table(void* cos_sin_table, int64_t npos, int32_t head_dim, float theta, void* stream);
/* head_to_seq receive side (K2): recv [P][s_loc][heads_in][d] -> out [s_loc][heads_out][d];
 * out[t][h] = sum over the (src rank, slot) pairs listed for h, in rank order (replicate_kv backward,
 * SPEC.md:326).  gather: DEVICE int32 [heads_out][max_src] of (rank*heads_in + slot), -1 = unused. */
spt_status spt_reshard_unpack(const void* recv, int64_t s_loc, int32_t heads_in, int32_t head_dim, int32_t P,
                              int32_t heads_out, const int32_t* gather, int32_t max_src, void* dst, void* stream);

/* Inner attention callback: causal GQA flash attention over the full
 * sequence for the local heads.  qkv: [s][hq + 2*hkv][d] bf16 (q heads, k heads, v heads);
 * seg_start: DEVICE int32 [s] start of each token's packed run, or NULL for plain causal.
 * o: [s][hq][d] bf16, lse: [hq][s] fp32. */
spt_status spt_attn_fwd(const void* qkv, int64_t s, int32_t hq, int32_t hkv, int32_t head_dim,
                        const int32_t* seg_start, float scale, void* o, float* lse, void* stream);
/* Deterministic backward: dqkv [s][hq + 2*hkv][d] bf16.  workspace: spt_attn_bwd_workspace bytes. */
size_t spt_attn_bwd_workspace(int64_t s, int32_t hq, int32_t hkv, int32_t head_dim);
spt_status spt_attn_bwd(const void* qkv, const void* o, const float* lse, const void* dout, int64_t s, int32_t hq,
                        int32_t hkv, int32_t head_dim, const int32_t* seg_start, float scale, void* dqkv,
                        void* workspace, void* stream);

/* RoPE in place on the first n_rot heads of x [n][heads][head_dim] bf16;
 * position_ids: DEVICE int64 [n] or NULL (positions pos_offset + t); inverse = 1 for the backward. */
spt_status spt_rope(void* x, int64_t n, int32_t heads, int32_t n_rot, int32_t head_dim, const int64_t* position_ids,
                    int64_t pos_offset, float theta, int32_t inverse, void* stream);

/* Label pre-pass of cross_entropy: count of non-ignored labels (int64, added to
 * *count_accum) and a device error flag set to 1 when a label is outside [0,V) U {-100}. */
spt_status spt_label_stats(const int64_t* labels, int64_t n, int64_t vocab, int64_t* count_accum, int32_t* err_flag,
                           void* stream);
/* position_ids -> run starts (int32) + device error flag for malformed runs. */
spt_status spt_segment_starts(const int64_t* position_ids, int64_t n, int32_t* starts, int32_t* err_flag,
                              void* stream);

/* Token embedding.  input_ids: DEVICE int64 [n]; table: [vocab][h]
 * bf16; x: [n][h] bf16.  err_flag (device int32) is set to 3 when an id is outside [0, vocab).
 * Backward: dtable [vocab][h] fp32 (+)= per-id sums of dx rows, each summed in ascending token order
 * (deterministic, no atomics); accumulate = 0 overwrites (rows with no token become 0).
 * workspace: spt_embed_bwd_workspace(n, vocab) bytes. */
spt_status spt_embed_fwd(const int64_t* input_ids, int64_t n, int64_t vocab, int64_t h, const void* table, void* x,
                         int32_t* err_flag, void* stream);
size_t spt_embed_bwd_workspace(int64_t n, int64_t vocab);
spt_status spt_embed_bwd(const int64_t* input_ids, int64_t n, int64_t vocab, int64_t h, const void* dx, float* dtable,
                         int32_t accumulate, int32_t* err_flag, void* workspace, void* stream);

/* tiled_logits_loss fused fwd+bwd: for each tile of `tile_n` tokens,
 * logits = x W^T (fp32, [tile_n, V] workspace only), CE (sum, count), dlogits scaled by
 * *grad_scale_dev (1/global count, device scalar), dx = dlogits W (bf16), dW (fp32) +=
 * dlogits^T x in ascending tile order.  loss_sum_accum (fp64 device scalar) += sum of NLL.
 * dw_accumulate: 0 overwrites dW with the first tile's contribution. */
size_t spt_flce_workspace(int64_t tile_n, int64_t vocab);
spt_status spt_flce(const void* x, const void* w, const int64_t* labels, int64_t n, int64_t h, int64_t vocab,
                    int64_t tile_n, const float* grad_scale_dev, double* loss_sum_accum, void* dx, float* dw,
                    int32_t dw_accumulate, int32_t* err_flag, void* workspace, void* stream);

/* tiled_mlp. wgu: [2I, h] bf16 with gate/up rows interleaved in blocks of 32
 * (rows 64j..64j+31 = W_gate[32j..], rows 64j+32..64j+63 = W_up[32j..]); wd: [h, I].
 * Forward: y = x_res + W_d(silu(W_g x) * W_u x) per tile (x_res may be NULL).  Backward recomputes
 * gate/up per tile and accumulates dwgu / dwd (fp32) in ascending tile order. */
size_t spt_mlp_workspace(int64_t tile_n, int64_t inter);
spt_status spt_mlp_fwd(const void* x, const void* wgu, const void* wd, const void* x_res, void* y, int64_t n, int64_t h,
                       int64_t inter, int64_t tile_n, void* workspace, void* stream);
spt_status spt_mlp_bwd(const void* x, const void* wgu, const void* wd, const void* dy, void* dx, float* dwgu,
                       float* dwd, int32_t accumulate, int64_t n, int64_t h, int64_t inter, int64_t tile_n,
                       void* workspace, void* stream);

/* ===================================== communicator ===================================== */

/* ProcessGroup.  Three transports (spt_comm_world reports which):
 *   0 loopback: P virtual ranks on one GPU driven by one host thread (the in-process SPMD of SPEC.md:183);
 *   1 NCCL:     one process per GPU, grouped ncclSend/ncclRecv + ncclAllReduce (the library baseline);
 *   2 peer:     one process (or thread) per GPU, buffers mapped into every peer over NVLink/NVSwitch (CUDA
 *               IPC): the Ulysses pack/unpack kernels store into / load from the peers' buffers themselves,
 *               ordered by device-side barriers; all-reduce sums in ascending rank order.
 * Collectives are stream-ordered.  A barrier that waits longer than the group's timeout (default 300 s,
 * spt_comm_set_timeout_ms) flags the group; the next host read (spt_layer_step / read_loss / spt_comm_check /
 * spt_comm_wait) then fails with SPT_ERR_PROTOCOL (a dead or stalled rank), and an NCCL step
 * that does not finish within the deadline aborts the communicator with SPT_ERR_PROTOCOL. */
typedef struct spt_comm spt_comm;
spt_status spt_comm_unique_id(uint8_t out_id[128]);
spt_status spt_comm_init_rank(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device, spt_comm** out);
spt_status spt_comm_init_loopback(int32_t nranks, int32_t device, spt_comm** out);
/* Peer group bootstrap: `exchange` all-gathers `bytes` from every rank into out[nranks * bytes] in rank order
 * (torch.distributed, MPI, a TCP store, or threads of one process) and returns 0 on success.  It is called
 * collectively by spt_comm_init_peer, spt_comm_connect and spt_layer_create (which map the symmetric
 * allocations made since the previous call). */
typedef int32_t (*spt_allgather_fn)(const void* in, void* out, size_t bytes, void* user);
spt_status spt_comm_init_peer(int32_t nranks, int32_t rank, int32_t device, spt_allgather_fn exchange, void* user,
                              spt_comm** out);
spt_status spt_comm_set_timeout_ms(spt_comm* comm, int64_t ms);
spt_status spt_comm_world(spt_comm* comm, int32_t* nranks, int32_t* rank, int32_t* transport);
/* SPT_ERR_PROTOCOL if a barrier of this group timed out (no sync). */
spt_status spt_comm_check(spt_comm* comm);
/* Wait for `stream` with the group's deadline (the host watchdog); SPT_ERR_PROTOCOL on expiry or timeout. */
spt_status spt_comm_wait(spt_comm* comm, void* stream);
/* Communication buffer: peer mode a symmetric allocation (every rank must make the same calls in the same
 * order, then spt_comm_connect), otherwise plain device memory.  Zero-filled. */
spt_status spt_comm_alloc(spt_comm* comm, size_t bytes, void** out);
spt_status spt_comm_free(spt_comm* comm, void* ptr);
spt_status spt_comm_connect(spt_comm* comm);
spt_status spt_comm_barrier(spt_comm* comm, void* stream);
spt_status spt_comm_destroy(spt_comm* comm);
/* CommStats as JSON: per collective call count and bytes sent per rank. */
spt_status spt_comm_stats_json(spt_comm* comm, char* buf, size_t cap);

/* SPEC.md:155-163 all_reduce_sum, in place.  bufs: one buffer per LOCAL rank (loopback: every virtual rank's,
 * summed in rank order into all of them; NCCL / peer: bufs[0], from spt_comm_alloc in peer mode). */
spt_status spt_all_reduce_f32(spt_comm* comm, void* const* bufs, int64_t n, void* stream);
spt_status spt_all_reduce_f64(spt_comm* comm, void* const* bufs, int64_t n, void* stream);
spt_status spt_all_reduce_i64(spt_comm* comm, void* const* bufs, int64_t n, void* stream);
/* SPEC.md:145-153 all_to_all: recv[j] on rank i = send[i] from rank j, bytes_per_peer each; one [P][bytes]
 * buffer per local rank (peer mode: send from spt_comm_alloc). */
spt_status spt_all_to_all(spt_comm* comm, const void* const* send, void* const* recv, size_t bytes_per_peer,
                          void* stream);

/* SPEC.md:307-315 seq_to_head (K1 with the all-to-all fused) for one layer's projections.
 * kind 0: x = fused qkv [s_loc][Hq + 2 Hkv][d] -> out [s][q_loc + 2 kv_loc][d] (replicate_kv: repeated kv head);
 * kind 1: x = q-shaped [s_loc][Hq][d] (dO) -> out [s][q_loc][d].
 * x / out: one pointer per LOCAL rank.  Peer mode: out from spt_comm_alloc (the peers store into it).  NCCL:
 * scratch = spt_reshard_scratch_bytes staging bytes, else NULL. */
size_t spt_reshard_scratch_bytes(const spt_head_shard_plan* plan, int32_t kind, int64_t s_loc, int32_t head_dim);
spt_status spt_seq_to_head(spt_comm* comm, const spt_head_shard_plan* plan, int32_t kind, const void* const* x,
                           int64_t s_loc, int32_t head_dim, void* const* out, void* scratch, void* stream);
/* SPEC.md:317-326 head_to_seq (K2 with the all-to-all fused), the exact inverse.
 * kind 0: x = o_head [s][q_loc][d] -> out [s_loc][Hq][d];
 * kind 1: x = dqkv_head [s][q_loc + 2 kv_loc][d] -> out [s_loc][Hq + 2 Hkv][d] with the replicas of a kv head
 *         summed in fp32 in rank order (replicate_kv backward).
 * Peer mode: x from spt_comm_alloc (the peers load from it). */
spt_status spt_head_to_seq(spt_comm* comm, const spt_head_shard_plan* plan, int32_t kind, const void* const* x,
                           int64_t s_loc, int32_t head_dim, void* const* out, void* scratch, void* stream);

/* SPEC.md:333-341 ulysses_attention as one collective op: seq_to_head -> tcgen05 attention on this rank's heads over
 * the whole sequence (s = s_loc * P; causal, or block-causal from seg = run starts of the FULL sequence, identical
 * on every rank) -> head_to_seq.  Arrays hold one pointer per LOCAL rank (loopback: every virtual rank's):
 *   qkv [s_loc][Hq + 2 Hkv][d] in, out [s_loc][Hq][d] out;
 *   qkv_head [s][q_loc + 2 kv_loc][d], o_head [s][q_loc][d] (peer mode: spt_comm_alloc) and lse [q_loc][s] fp32 are
 *   filled for the backward, which the caller keeps them for.
 * scratch: NCCL staging of spt_reshard_scratch_bytes(plan, 0, s_loc, d) bytes, else NULL.  Errors are those of the
 * three ops it composes. */
spt_status spt_ulysses_attention_fwd(spt_comm* comm, const spt_head_shard_plan* plan, const void* const* qkv,
                                     int64_t s_loc, int32_t head_dim, const int32_t* seg, float scale,
                                     void* const* qkv_head, void* const* o_head, float* const* lse, void* const* out,
                                     void* scratch, void* stream);
/* Backward: dout [s_loc][Hq][d] -> dqkv [s_loc][Hq + 2 Hkv][d] (replicas of a kv head summed in fp32, rank order,
 * SPEC.md:326); do_head [s][q_loc][d] and dqkv_head [s][q_loc + 2 kv_loc][d] head-side buffers (peer mode:
 * spt_comm_alloc), ws one spt_attn_bwd_workspace(s, q_loc, kv_loc, d) buffer per local rank. */
spt_status spt_ulysses_attention_bwd(spt_comm* comm, const spt_head_shard_plan* plan, const void* const* qkv_head,
                                     const void* const* o_head, const float* const* lse, const void* const* dout,
                                     int64_t s_loc, int32_t head_dim, const int32_t* seg, float scale,
                                     void* const* do_head, void* const* dqkv_head, void* const* ws,
                                     void* const* dqkv, void* scratch, void* stream);

/* ================================= layer step engine ================================= */

/* ModelConfig for one layer + lm_head; head_dim explicit. */
typedef struct {
    int32_t hidden;
    int32_t q_heads;
    int32_t kv_heads;
    int32_t head_dim;
    int32_t intermediate;
    int64_t vocab;
    int64_t seq_len;   /* global sequence length (sum over ranks), bs = 1 */
    int32_t mlp_tiles; /* > 0: that many TiledMLP tiles; -1: ceil(s_loc / hidden); 0: fewest tiles whose
                          intermediates fit 2 GiB (16384-token tiles at Llama-3-8B shapes) */
    int64_t loss_tile; /* tokens per logits tile, 0 -> auto */
    float rms_eps;     /* 0 -> 1e-5 */
    int32_t packed;    /* 1: block-causal attention from position_ids */
    float lr;          /* >0: plain SGD update of the bf16 weights at the end of the step */
    int32_t n_layers;  /* decoder layers (0 -> 1); > 1 turns on per-layer activation checkpointing
                          (layer inputs saved, each layer re-run in backward) */
    int32_t ckpt_offload; /* 1: checkpoints in pinned host memory, copied on a side stream
                             (checkpoint_offload); implies checkpointing */
    float rope_theta;     /* > 0: rotary position embedding on q and k (Llama rotate_half convention, base
                             theta; positions = position_ids when packed, else the global token index).
                             0 = off, the reference's model (SPEC.md:261 omits RoPE) */
    int32_t embed;        /* 1: token embedding table "emb" [vocab][hidden] in front of the stack (SPEC.md:205,
                             :223); the step's x argument is then int64 input_ids [local_ranks * s_loc], ids
                             outside [0, vocab) are a validation error, and grad "emb" is the per-id sum of the
                             stack's input gradient (deterministic) */
    int32_t verify_replay; /* 1 (with checkpointing): every checkpoint replay in the backward is fingerprinted
                              against the recorded forward (autograd.hpp:26-30); a mismatch makes the step
                              fail with SPT_ERR_DETERMINISM (errors.hpp:36-40).  Costs one read of each
                              replayed layer's output. */
} spt_layer_config;

typedef struct spt_layer spt_layer;
spt_status spt_layer_create(const spt_layer_config* cfg, spt_comm* comm, spt_layer** out);
spt_status spt_layer_destroy(spt_layer* layer);
/* name in {g1, wqkv, wo, g2, wg, wu, wd, g3, wlm} (per-layer names address layer 0; "layers.<i>.<name>"
 * addresses layer i); data = bf16 bits in [out, in] row-major. */
spt_status spt_layer_set_param(spt_layer* layer, const char* name, const void* data, int32_t data_on_host);
/* Number of bf16 elements spt_layer_set_param copies for `name` (the caller's buffer must hold that many);
 * SPT_ERR_VALIDATION for an unknown name (like spt_layer_set_param). */
spt_status spt_layer_param_numel(spt_layer* layer, const char* name, int64_t* numel);
/* One fwd+bwd step.  x: bf16 [local_ranks * s_loc, hidden] (loopback: the whole sequence),
 * shift_labels / position_ids: int64 [local_ranks * s_loc] (already pre-shifted).
 * inputs_on_host: 1 -> host buffers (copied in inside the call), 0 -> device buffers.
 * loss_out / count_out are host scalars (global mean loss and global valid count). */
spt_status spt_layer_step(spt_layer* layer, const void* x, const int64_t* shift_labels, const int64_t* position_ids,
                          int32_t inputs_on_host, float* loss_out, int64_t* count_out, void* stream);
/* Same step, but leaves loss/count on the device (no host sync); read with spt_layer_read_loss. */
spt_status spt_layer_step_async(spt_layer* layer, const void* x, const int64_t* shift_labels,
                                const int64_t* position_ids, int32_t inputs_on_host, void* stream);
spt_status spt_layer_read_loss(spt_layer* layer, float* loss_out, int64_t* count_out, void* stream);
/* Pipelined per-step results: enqueue a D2H of the step's (loss, count, error flags) into slot [0, 64) of a
 * pinned ring without synchronising, and read a slot after the stream has passed it.  With host inputs,
 * spt_layer_step_async copies them on a separate stream into a double-buffered staging area, so the H2D of
 * step i+1 overlaps step i when steps are enqueued back to back. */
spt_status spt_layer_loss_async(spt_layer* layer, int32_t slot, void* stream);
spt_status spt_layer_loss_slot(spt_layer* layer, int32_t slot, float* loss_out, int64_t* count_out);
/* Gradient accumulation over a window of micro-steps: each micro-step accumulates the grads of
 * the loss SUM (first_micro_step = 1 starts a new window); finish all-reduces the accumulated grads over the
 * SP group, divides them by the window's global valid count, applies the update (lr > 0) and returns the
 * window's mean loss and count.  Pair with sp_over_dp iteration. */
/* CUDA graph of one step with DEVICE inputs at fixed addresses (their contents may change between replays):
 * capture runs one eager step, then records the next into a graph on `stream` (non-default, profiling off);
 * launch replays it (the ~100 kernels of a step without per-launch host work).  Read results as after
 * spt_layer_step_async. */
spt_status spt_layer_graph_capture(spt_layer* layer, const void* x, const int64_t* shift_labels,
                                   const int64_t* position_ids, void* stream);
spt_status spt_layer_graph_launch(spt_layer* layer, void* stream);
spt_status spt_layer_step_accumulate(spt_layer* layer, const void* x, const int64_t* shift_labels,
                                     const int64_t* position_ids, int32_t inputs_on_host, int32_t first_micro_step,
                                     void* stream);
spt_status spt_layer_finish_accumulation(spt_layer* layer, float* loss_out, int64_t* count_out, void* stream);
/* fp32 weight gradient (SP-group all-reduced) copied to host [out, in]. */
spt_status spt_layer_get_grad(spt_layer* layer, const char* name, float* host_out);
/* d loss / d x (bf16 bits, same layout as x) copied to host. */
spt_status spt_layer_get_dx(spt_layer* layer, void* host_out);
/* MemoryLedger::summary_json (ledger.hpp:85) of the device tier + cudaMemGetInfo cross-check. */
spt_status spt_layer_memory_json(spt_layer* layer, char* buf, size_t cap);
/* MemoryLedger::timeline_csv (ledger.hpp:85, ledger.cpp:149-157): one row per tracked allocation / release,
 * "ordinal,kind,tier,tag,delta_bytes,device_live,host_live".  SPT_ERR_SHAPE if cap is too small. */
spt_status spt_layer_memory_timeline_csv(spt_layer* layer, char* buf, size_t cap);
/* Per-phase CUDA-event timings of the last step (ms) as JSON (requires spt_layer_set_profiling(1)). */
spt_status spt_layer_set_profiling(spt_layer* layer, int32_t on);
spt_status spt_layer_timing_json(spt_layer* layer, char* buf, size_t cap);
/* Number of CUDA kernels this library launched since load (gpu_launches evidence). */
int64_t spt_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SPTRAIN_B200_H */
