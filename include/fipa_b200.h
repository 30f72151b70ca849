/*
 * fipa_b200.h -- C ABI of the B200-native FlashIPA layer (libfipa_b200.so).
 *
 * This is the drop-in boundary for the reference's FlashIPA hot path.  Every entry point
 * below replaces one reference interface (paths relative to /root/reference/proj):
 *
 *   fipa_config / fipa_config_validate   IpaConfig + validate      include/fipa/ipa.hpp:14-32,
 *                                                                   src/ipa.cpp:12-21
 *   fipa_layer_create                    (IpaConfig, IpaWeights) pair held by the Python
 *                                        Model                      python/bindings.cpp:82-101
 *   fipa_layer_init_weights              IpaWeights::init(cfg, Rng(seed))
 *                                                                   src/ipa.cpp:172-193
 *   fipa_layer_set_weights / _get_weights  IpaWeights fields        include/fipa/ipa.hpp:37-50
 *   fipa_layer_save_weights              save_weights               src/model_io.cpp:121-141
 *   fipa_layer_load_weights              load_weights               src/model_io.cpp:143-196
 *   fipa_layer_forward (device buffers)  flash_ipa_forward          src/flash_ipa.cpp:141-218
 *   fipa_layer_forward_host (host f64)   Model.flash                python/bindings.cpp:122-135
 *   fipa_last_error + status codes       ValueError / NumericError / IoError
 *                                                                   include/fipa/error.hpp:10-28
 *   fipa_layer_forward_train /           no reference counterpart: the reference is inference-only
 *   fipa_layer_backward / _grad_host     (proj/SPEC.md:8); the gradient of flash_ipa_forward
 *                                        (src/flash_ipa.cpp:141-218), checked against finite
 *                                        differences of the reference (tests/test_oracle.py)
 *
 * Differences from the reference, all additive: a leading batch axis B (each sample is an
 * independent reference call with its own mask), caller-owned device buffers + a CUDA stream,
 * and a precision switch: FIPA_PREC_BF16 runs the tcgen05 tensor-core path (bf16 operands, fp32
 * accumulation), FIPA_PREC_F32 / F64 the fp32-accuracy path, also on the tcgen05 tensor cores
 * (3xTF32: kind::tf32 MMAs over hi/lo operand splits).  There is no CPU fallback: without a
 * B200 every compute entry point returns FIPA_ERR_CUDA.
 *
 * Threading: a layer handle may be used from several threads on distinct streams for
 * forward calls (weights are read-only during forward); weight mutation is not thread-safe.
 */
#ifndef FIPA_B200_H
#define FIPA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (0 = success).  fipa_last_error() returns the thread's last message. */
#define FIPA_OK 0
#define FIPA_ERR_VALUE 1   /* reference ValueError: bad shapes / config / arguments   */
#define FIPA_ERR_NUMERIC 2 /* reference NumericError                                  */
#define FIPA_ERR_IO 3      /* reference IoError: weights file problems                */
#define FIPA_ERR_CUDA 4    /* CUDA runtime / launch failure, or no usable GPU         */
#define FIPA_ERR_OTHER 9

#define FIPA_PREC_BF16 0 /* tcgen05 path: bf16 operands, fp32 accumulation; f64 master weights */
#define FIPA_PREC_F32 1  /* fp32-accuracy path (3xTF32 tensor cores); master weights rounded to f32 */
#define FIPA_PREC_F64 2  /* reference "f64" models: f64 master weights, fp32-accuracy compute      */

/* Hyper-parameters (IpaConfig).  Names follow the reference: d_in = c_s, d_z = c_z,
 * c = c_hidden, n_query = qk-points, n_value = v-points, rank = z_factor_rank. */
typedef struct fipa_config {
    uint64_t d_in, d_z, heads, c, n_query, n_value, rank;
    int32_t precision;        /* FIPA_PREC_BF16 | FIPA_PREC_F32 | FIPA_PREC_F64      */
    int32_t enforce_head_cap; /* reference default 1: max(qk_width, v_width) <= 256   */
} fipa_config;

/* Host weights in the reference IpaWeights layout, float64, row-major:
 *   w_q w_k w_v [d_in, H*c]; w_qp w_kp [d_in, H*Nq*3]; w_vp [d_in, H*Nv*3];
 *   w_bias [H, d_z]; gamma_raw [H]; w_out [H*(d_z+c+4Nv), d_in]; b_out [d_in]. */
typedef struct fipa_host_weights {
    const double *w_q, *w_k, *w_v, *w_qp, *w_kp, *w_vp, *w_bias, *gamma_raw, *w_out, *b_out;
    double w_l, w_c;
} fipa_host_weights;

typedef struct fipa_layer fipa_layer;

const char* fipa_last_error(void);

int fipa_config_validate(const fipa_config* cfg);
/* Lifted widths of the reference (IpaConfig::qk_width / v_width). */
uint64_t fipa_config_qk_width(const fipa_config* cfg);
uint64_t fipa_config_v_width(const fipa_config* cfg);

/* Creates the layer on the current CUDA device with IpaWeights::init(cfg, Rng(0)). */
int fipa_layer_create(const fipa_config* cfg, fipa_layer** out);
void fipa_layer_destroy(fipa_layer* layer);

int fipa_layer_init_weights(fipa_layer* layer, uint64_t seed);
int fipa_layer_set_weights(fipa_layer* layer, const fipa_host_weights* w);
/* Copies the master weights out; w[10] point to caller buffers sized as above, scal[2] = {w_l, w_c}. */
int fipa_layer_get_weights(const fipa_layer* layer, double* const* w, double* scal);
int fipa_layer_save_weights(const fipa_layer* layer, const char* path);
int fipa_layer_load_weights(fipa_layer* layer, const char* path);

/* Device workspace needed by fipa_layer_forward for a [B, L] batch. */
size_t fipa_layer_workspace_size(const fipa_layer* layer, int64_t B, int64_t L);

/* Forward over device buffers (float32 unless noted), enqueued on `stream` (cudaStream_t):
 *   s [B,L,d_in]  z1,z2 [B,L,rank,d_z]  rot [B,L,3,3] (row-major, y = R x + t)  trans [B,L,3]
 *   mask [B,L] uint8 (1 = valid) or NULL     out [B,L,d_in]
 * Masked rows of `out` are zero; a fully masked sample yields all zeros. */
int fipa_layer_forward(fipa_layer* layer, int64_t B, int64_t L, const float* s, const float* z1,
                       const float* z2, const float* rot, const float* trans, const uint8_t* mask,
                       float* out, void* workspace, size_t workspace_bytes, void* stream);

/* The reference's `fully_masked` output of flash_ipa_forward (include/fipa/flash_ipa.hpp:53-57,
 * src/flash_ipa.cpp:156-158): flags [B,L] uint8 (device), 1 on every row of a sample that has no
 * valid residue (mask NULL = all valid: all flags 0).  Enqueued on `stream`. */
int fipa_fully_masked(int64_t B, int64_t L, const uint8_t* mask, uint8_t* flags, void* stream);
/* Same over host buffers (synchronous, current device). */
int fipa_fully_masked_host(int64_t B, int64_t L, const uint8_t* mask, uint8_t* flags);

/* Same forward over HOST float64 buffers (the reference / Python calling convention), synchronous.
 * Pipelined over the batch: chunks of whole samples; the float64 <-> float32 conversion (host
 * cores), the copies (two copy streams) and the kernels of neighbouring chunks overlap. */
int fipa_layer_forward_host(fipa_layer* layer, int64_t B, int64_t L, const double* s,
                            const double* z1, const double* z2, const double* rot,
                            const double* trans, const uint8_t* mask, double* out);

/* Same over HOST float32 buffers (additive: no float64 round trip; float32 out). */
int fipa_layer_forward_host_f32(fipa_layer* layer, int64_t B, int64_t L, const float* s, const float* z1,
                                const float* z2, const float* rot, const float* trans, const uint8_t* mask, float* out);

/* ------------------------------------------------------------ quadratic-memory arm (f3)
 * The reference's dense forward (reference_forward, src/ipa.cpp:244-310; Python Model.reference,
 * python/bindings.cpp:187-189): materialises the pair tensor z [B,L,L,d_z] and the logits /
 * attention [B,H,L,L] on the GPU in fp32 -- the O(L^2) baseline the linear-memory path replaces
 * (paper Fig. 2).  Same buffers and conventions as fipa_layer_forward; any precision. */
size_t fipa_layer_reference_workspace_size(const fipa_layer* layer, int64_t B, int64_t L);
int fipa_layer_reference_forward(fipa_layer* layer, int64_t B, int64_t L, const float* s, const float* z1,
                                 const float* z2, const float* rot, const float* trans, const uint8_t* mask,
                                 float* out, void* workspace, size_t workspace_bytes, void* stream);
int fipa_layer_reference_host(fipa_layer* layer, int64_t B, int64_t L, const double* s, const double* z1,
                              const double* z2, const double* rot, const double* trans, const uint8_t* mask,
                              double* out);

/* ------------------------------------------------------------ generic attention
 * include/fipa/attention_kernel.hpp:17-41: softmax(q k^T) v, no internal scaling (callers fold
 * it into q or k), key mask [L] (1 = valid) or NULL, rows without a valid key are zeros.
 * q, k [H, L, d_qk]; v, out [H, L, d_v]; fp32 device buffers.
 *   fipa_naive_attention   naive_attention   src/attention_kernel.cpp:192-211 (logits [H,L,L]
 *                          in the workspace: fipa_naive_attention_workspace_size bytes)
 *   fipa_flash_attention   flash_attention   src/attention_kernel.cpp:213-243 (O(L) memory)
 *   fipa_attention_host    python/bindings.cpp:153-165 (host float64 in/out, naive != 0 selects
 *                          the dense path; runs synchronously on `device`) */
size_t fipa_naive_attention_workspace_size(int64_t H, int64_t L);
int fipa_naive_attention(int64_t H, int64_t L, int64_t dqk, int64_t dv, const float* q, const float* k,
                         const float* v, const uint8_t* mask, float* out, void* workspace, size_t workspace_bytes,
                         void* stream);
int fipa_flash_attention(int64_t H, int64_t L, int64_t dqk, int64_t dv, const float* q, const float* k,
                         const float* v, const uint8_t* mask, float* out, void* stream);
int fipa_attention_host(int64_t H, int64_t L, int64_t dqk, int64_t dv, const double* q, const double* k,
                        const double* v, const uint8_t* mask, double* out, int naive, int device);

/* Byte offsets of the forward's intermediates inside the workspace (for parity tests and
 * for a caller-driven backward), -1 when absent for this precision, in the order:
 *   0 trans_c (recentred translations, f32 [B,L,3])   1 s_bf16 (bf16 [B,L,d_in])
 *   2 proj (f32 [B,L,n_proj])    3 q_hat   4 k_hat ([B*H,L,dqk_pad])   5 v_hat ([B*H,L,dv_pad])
 *   6 colbias (f32 [B*H,L])      7 lse (f32 [B*H,L])                  8 feat ([B,L,H*seg])
 * q/k/v/feat are bf16 for FIPA_PREC_BF16 and f32 for FIPA_PREC_F32.  dims[4] receives
 * {n_proj, dqk_pad, dv_pad, H*seg}.  Returns the number of offsets written (9). */
int fipa_layer_workspace_layout(const fipa_layer* layer, int64_t B, int64_t L, int64_t* offsets,
                                int64_t* dims);

/* ---------------------------------------------------------------------------- training
 * Training forward: identical outputs to fipa_layer_forward, but over a workspace of
 * fipa_layer_train_workspace_size bytes in which it keeps what fipa_layer_backward needs (the
 * normalised attention output).  FIPA_PREC_BF16 only (tcgen05 path; z_factor_rank 3-4 through the
 * materialised backward, whose workspace grows with L^2). */
size_t fipa_layer_train_workspace_size(const fipa_layer* layer, int64_t B, int64_t L);
int fipa_layer_forward_train(fipa_layer* layer, int64_t B, int64_t L, const float* s, const float* z1,
                             const float* z2, const float* rot, const float* trans, const uint8_t* mask,
                             float* out, void* workspace, size_t workspace_bytes, void* stream);
/* Total number of weight scalars (w_q .. b_out in reference order). */
uint64_t fipa_layer_num_weights(const fipa_layer* layer);
/* Backward of the last fipa_layer_forward_train on the same workspace and inputs: gradients of
 * sum(out * dout) (device float32, same shapes as the inputs): ds [B,L,d_in], dz1/dz2
 * [B,L,rank,d_z], drot [B,L,3,3] and dtrans [B,L,3] (either may be NULL), dweights
 * [fipa_layer_num_weights] = w_q|w_k|w_v|w_qp|w_kp|w_vp|w_bias|gamma_raw|w_out|b_out flattened
 * row-major.  Masked residues receive zero gradients. */
int fipa_layer_backward(fipa_layer* layer, int64_t B, int64_t L, const float* s, const float* z1,
                        const float* z2, const float* rot, const float* trans, const uint8_t* mask,
                        const float* dout, float* ds, float* dz1, float* dz2, float* drot, float* dtrans,
                        float* dweights, void* workspace, size_t workspace_bytes, void* stream);
/* Forward + backward over HOST float64 buffers (copies in, runs, copies out, synchronises).
 * Any gradient output may be NULL. */
int fipa_layer_grad_host(fipa_layer* layer, int64_t B, int64_t L, const double* s, const double* z1,
                         const double* z2, const double* rot, const double* trans, const uint8_t* mask,
                         const double* dout, double* out, double* ds, double* dz1, double* dz2,
                         double* drot, double* dtrans, double* dweights);
/* Same over HOST float32 buffers (additive: no float64 round trip). */
int fipa_layer_grad_host_f32(fipa_layer* layer, int64_t B, int64_t L, const float* s, const float* z1,
                             const float* z2, const float* rot, const float* trans, const uint8_t* mask,
                             const float* dout, float* out, float* ds, float* dz1, float* dz2, float* drot,
                             float* dtrans, float* dweights);
/* Byte offsets of the training intermediates in a train workspace (offsets[FIPA_TRAIN_LAYOUT_SLOTS]),
 * -1 when absent:
 *   0 o_hat (f32 [B,L,H,dv_pad])  1 do_hat (bf16 [B*H,L,dv_pad])  2 D (f32 [B*H,L])
 *   3 dq_acc 4 dk_acc 5 dv_acc (f32 [B,L,H,acc_ld])  6 dproj (bf16 [B*L,nproj_ld])
 *   7 dfeat (bf16 [B*L,feat_ld])  8 dk16 9 dv16 (bf16 [B,L,H,acc_ld]: the fused backward's bf16
 *   dK / dV, every column; dk_acc / dv_acc then hold only the 32-column chunks with point /
 *   translation columns.  -1 for z_factor_rank 3-4)  10 dq16 (likewise for dQ when it comes from
 *   the materialised-dS GEMM; the streaming dQ kernel writes dq_acc whole).  dims[3] receives
 *   {acc_ld, nproj_ld, feat_ld}.  Returns FIPA_TRAIN_LAYOUT_SLOTS. */
#define FIPA_TRAIN_LAYOUT_SLOTS 11
int fipa_layer_train_workspace_layout(const fipa_layer* layer, int64_t B, int64_t L, int64_t* offsets,
                                      int64_t* dims);
int fipa_layer_backward_launches(const fipa_layer* layer);

/* ------------------------------------------------------------ multi-GPU (query-row sharding)
 * One process per GPU.  A sequence of G*L residues is split into G contiguous blocks of L rows
 * (rank r owns rows [r*L, (r+1)*L)); the packed key/value rows are all-gathered over NCCL and each
 * rank returns the output rows of its block.  NCCL is loaded at run time (libnccl.so.2).
 * Reference counterpart: none -- the reference is single-process. */
typedef struct fipa_comm fipa_comm;
#define FIPA_ERR_COMM 5 /* NCCL failure / NCCL unavailable */
int fipa_comm_unique_id(uint8_t out[128]);
int fipa_comm_create(int world, int rank, const uint8_t id[128], int device, fipa_comm** out);
void fipa_comm_destroy(fipa_comm* comm);
/* In-place sum of a device float buffer over the communicator's ranks, on `stream`: the
 * data-parallel (batch-sharded) training step's weight-gradient all-reduce. */
int fipa_comm_all_reduce_f32(fipa_comm* comm, float* buf, size_t n, void* stream);
size_t fipa_layer_sharded_workspace_size(const fipa_layer* layer, int64_t B, int64_t L_local, int world);
int fipa_layer_forward_sharded(fipa_layer* layer, fipa_comm* comm, int64_t B, int64_t L_local, const float* s,
                               const float* z1, const float* z2, const float* rot, const float* trans,
                               const uint8_t* mask, float* out, void* workspace, size_t workspace_bytes,
                               void* stream);
/* Collective-agnostic building blocks of the same path (any all-reduce / all-gather may join them):
 *   1. fipa_layer_shard_centroid_sums: device float sums[B*4] = per-sample {sum t, count} of the
 *      local valid rows; the caller all-reduces (sums) them across ranks.
 *   2. fipa_layer_shard_pack: recentre with the global sums, project and pack the local rows into
 *      the workspace (a fipa_layer_workspace_size(B, L_local) buffer); *khat / *vhat point at the
 *      local packed rows (k_bytes / v_bytes each); the caller all-gathers them rank-major.
 *   3. fipa_layer_shard_attend: local queries against the gathered keys -> out [B, L_local, d_in]. */
int fipa_layer_shard_centroid_sums(fipa_layer* layer, int64_t B, int64_t L_local, const float* trans,
                                   const uint8_t* mask, float* sums, void* stream);
int fipa_layer_shard_pack(fipa_layer* layer, int64_t B, int64_t L_local, const float* s, const float* z1,
                          const float* z2, const float* rot, const float* trans, const uint8_t* mask,
                          const float* sums, void* workspace, size_t workspace_bytes, void* stream,
                          void** khat, size_t* k_bytes, void** vhat, size_t* v_bytes);
int fipa_layer_shard_attend(fipa_layer* layer, int64_t B, int64_t L_local, int world, const float* s,
                            const float* z1, const float* z2, const float* rot, const float* trans,
                            const uint8_t* mask, const void* khat_all, const void* vhat_all, float* out,
                            void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------ sharded training
 * Rank r of G owns residues [r L, (r+1) L); L % 256 == 0 when G > 1.  The forward keeps the fp32
 * O_hat / lse of the local queries and the gathered k_hat / v_hat; the backward computes dQ for
 * the local queries and PARTIAL dK / dV for all G L keys, reduce-scatters them (fp32) to their
 * owners, all-reduces the per-sample translation-gradient sums and the weight gradients.
 * Reference counterpart: none (the reference is single-process and inference-only). */
size_t fipa_layer_sharded_train_workspace_size(const fipa_layer* layer, int64_t B, int64_t L_local, int world);
int fipa_layer_forward_train_sharded(fipa_layer* layer, fipa_comm* comm, int64_t B, int64_t L_local, const float* s,
                                     const float* z1, const float* z2, const float* rot, const float* trans,
                                     const uint8_t* mask, float* out, void* workspace, size_t workspace_bytes,
                                     void* stream);
int fipa_layer_backward_sharded(fipa_layer* layer, fipa_comm* comm, int64_t B, int64_t L_local, const float* s,
                                const float* z1, const float* z2, const float* rot, const float* trans,
                                const uint8_t* mask, const float* dout, float* ds, float* dz1, float* dz2, float* drot,
                                float* dtrans, float* dweights, void* workspace, size_t workspace_bytes,
                                void* stream);
/* Collective-agnostic blocks of the same training step (a fipa_layer_train_workspace_size(B, L_local)
 * workspace per rank):
 *   forward:  shard_centroid_sums -> all-reduce -> shard_pack_train -> rank-major all-gather of
 *             k/v -> shard_attend_train
 *   backward: shard_backward(stage 1) -> reduce-scatter dk_part / dv_part ([G][B][L][H][448] f32,
 *             rank-major) into dk_own / dv_own ([B][L][H][448]) -> shard_backward(stage 2) ->
 *             all-reduce dt_sums [B*4] -> shard_backward(stage 3) -> all-reduce dweights. */
int fipa_layer_shard_pack_train(fipa_layer* layer, int64_t B, int64_t L_local, const float* s, const float* z1,
                                const float* z2, const float* rot, const float* trans, const uint8_t* mask,
                                const float* sums, void* workspace, size_t workspace_bytes, void* stream,
                                void** khat, size_t* k_bytes, void** vhat, size_t* v_bytes);
int fipa_layer_shard_attend_train(fipa_layer* layer, int64_t B, int64_t L_local, int world, const float* s,
                                  const float* z1, const float* z2, const float* rot, const float* trans,
                                  const uint8_t* mask, const void* khat_all, const void* vhat_all, float* out,
                                  void* workspace, size_t workspace_bytes, void* stream);
int fipa_layer_shard_backward(fipa_layer* layer, int stage, int world, int64_t B, int64_t L_local, const float* s,
                              const float* z1, const float* z2, const float* rot, const float* trans,
                              const uint8_t* mask, const float* dout, const void* khat_all, const void* vhat_all,
                              float* dk_part, float* dv_part, const float* dk_own, const float* dv_own,
                              float* dt_sums, float* ds, float* dz1, float* dz2, float* drot, float* dtrans,
                              float* dweights, void* workspace, size_t workspace_bytes, void* stream);

/* -------------------------------------------------------------------------- trunk
 * BASELINE cfg3: n_layers FlashIPA layers with residual and per-layer backbone frame update
 * (FrameFlow-style; the reference has no trunk -- the definition is oracle/fipa_oracle.py
 * trunk_forward):  s <- s + layer_l(s, z, T);  u = s.W_bb,l + b_bb,l;
 * T <- compose(T, (R(normalised (1, u0, u1, u2)), u[3:6])) (proj/src/geometry.cpp:78-90, 107-132).
 * Layer l has IpaWeights::init(cfg, Rng(seed + l)); fipa_trunk_layer returns a borrowed layer
 * handle (get/set/save/load weights through the layer API; fipa_layer_destroy on it is a no-op). */
typedef struct fipa_trunk fipa_trunk;
int fipa_trunk_create(const fipa_config* cfg, int n_layers, uint64_t seed, fipa_trunk** out);
void fipa_trunk_destroy(fipa_trunk* trunk);
int fipa_trunk_num_layers(const fipa_trunk* trunk);
fipa_layer* fipa_trunk_layer(fipa_trunk* trunk, int layer);
int fipa_trunk_get_backbone(const fipa_trunk* trunk, int layer, double* w /* [d_in*6] */, double* b /* [6] */);
int fipa_trunk_set_backbone(fipa_trunk* trunk, int layer, const double* w, const double* b);
size_t fipa_trunk_workspace_size(const fipa_trunk* trunk, int64_t B, int64_t L);
/* Device buffers as in fipa_layer_forward; outputs s_out [B,L,d_in], rot_out [B,L,3,3],
 * trans_out [B,L,3] (may alias the inputs). */
int fipa_trunk_forward(fipa_trunk* trunk, int64_t B, int64_t L, const float* s, const float* z1, const float* z2,
                       const float* rot, const float* trans, const uint8_t* mask, float* s_out, float* rot_out,
                       float* trans_out, void* workspace, size_t workspace_bytes, void* stream);
int fipa_trunk_forward_launches(const fipa_trunk* trunk);
/* Kernels of one fipa_trunk_forward at (B, L), sample chains and micro-batch chains included. */
int fipa_trunk_step_launches(const fipa_trunk* trunk, int64_t B, int64_t L);

/* ----------------------------------------------------------- pair-factor producer (§8 f2)
 * knn_distogram (proj/src/pair_features.cpp:10-64): translations [B,L,3] -> features
 * [B,L,k,n_bins+pe_dim]: the k nearest other residues (float64 distances, ties to the lower
 * index), one-hot distance bins clipped into the end bins, and the sinusoidal encoding of the
 * offset j-i (positional_encoding, pair_features.cpp:66-81).  Reference defaults: k 20, n_bins 22,
 * d_min 2, d_max 22, pe_dim 16.  Errors as the reference (ValueError on invalid specs).
 * build_factors (pair_features.cpp:83-97): z1 = features.w1, z2 = features.w2 ([rows,f] x [f,r*d_z]);
 * precision FIPA_PREC_BF16 uses the tcgen05 GEMM, otherwise fp32. */
int fipa_knn_distogram(int64_t B, int64_t L, const float* trans, uint64_t k, uint64_t n_bins, double d_min,
                       double d_max, uint64_t pe_dim, float* out, void* stream);
/* Same over float64 device buffers: the translations are never rounded, so the neighbour choice
 * and bins are bit-exact with the reference's float64 path (pair_features.cpp:29-45);
 * fipa_knn_distogram_host runs this variant. */
int fipa_knn_distogram_f64(int64_t B, int64_t L, const double* trans, uint64_t k, uint64_t n_bins, double d_min,
                           double d_max, uint64_t pe_dim, double* out, void* stream);
int fipa_knn_distogram_host(int64_t B, int64_t L, const double* trans, uint64_t k, uint64_t n_bins, double d_min,
                            double d_max, uint64_t pe_dim, double* out);
size_t fipa_build_factors_workspace_size(int64_t rows, uint64_t f, uint64_t n);
int fipa_build_factors(int64_t rows, uint64_t f, const float* features, uint64_t r, uint64_t d_z, const float* w1,
                       const float* w2, float* z1, float* z2, int precision, void* workspace, size_t workspace_bytes,
                       void* stream);
int fipa_build_factors_host(int64_t rows, uint64_t f, const double* features, uint64_t r, uint64_t d_z,
                            const double* w1, const double* w2, double* z1, double* z2, int precision);

/* Number of kernels fipa_layer_forward launches per call for this configuration (one sample
 * chain). */
int fipa_layer_forward_launches(const fipa_layer* layer);
/* Kernels of one device call at (B, L) with the layer's tuning, micro-batch chains included:
 * train = 0 the forward, 1 the training forward + backward (the measured step; CUPTI counts of
 * tools/count_launches.py agree: 16 and 39 at B=8 L=1024). */
int fipa_layer_step_launches(const fipa_layer* layer, int64_t B, int64_t L, int train);

/* Kernel-selection / tuning knobs of a layer.  Fixed per layer: seeded once at creation from
 * the FIPA_* environment variables named below (A/B experiments; defaults = the measured-best
 * choices), changed only by fipa_layer_set_tuning -- never read on the launch path.  Not
 * thread-safe against concurrent compute calls on the same layer.
 *   attn_impl  inference attention kernel: 0 automatic, 1 CTA pair, 2 two-pass, 3 single CTA
 *              (FIPA_ATTN_IMPL = pair | pass | 1sm; a sharded forward never takes 3)
 *   fused_pack 1: fused projection + pack kernel (FIPA_FUSED_PACK=0 -> GEMM + pack kernel)
 *   bwd_ds     materialised-dS backward: -1 automatic (L <= 8192, dS <= 2 GiB), 0 off, 1 on
 *              within that cap (FIPA_BWD_DS)
 *   bwd_ring   attention-backward ring plan {nst1, nst2, nab, kb1}, zeros = automatic, and
 *   bwd_slice  its B2 slice rows (16 / 32, 0 = any) (FIPA_BWD_RING "nst1,nst2,nab,kb1[,slice]")
 *   pass_ring  two-pass attention rings {kb, kst, vkeys, vst}, zeros = automatic (FIPA_PASS_RING)
 *   f32_tc     1: FIPA_PREC_F32/F64 run on the tensor cores (3xTF32 projections, attention and
 *              output projection); 0: the fp32 CUDA-core kernels (FIPA_F32_TC=0)
 *   graphs     1: the device entry points (forward, training forward, backward) replay a CUDA graph
 *              captured on their first call with the same shapes and buffers; 0: kernel-by-kernel
 *              launches (FIPA_GRAPHS=0) */
typedef struct fipa_tuning {
    int32_t attn_impl, fused_pack, bwd_ds;
    int32_t bwd_ring[4], pass_ring[4];
    int32_t f32_tc;
    int32_t bwd_slice;
    int32_t graphs;
    int32_t micro; /* bf16 device calls: interleaved sample chunks on forked streams (1 = one chain) */
    int32_t shard_chunks; /* query-row sharding: head chunks of the overlapped K/V gather (0 auto, 1 off) */
    int32_t ds_cap_mb;    /* materialised-dS workspace cap in MiB (query chunks beyond it); default 2048 */
} fipa_tuning;
int fipa_layer_get_tuning(const fipa_layer* layer, fipa_tuning* out);
int fipa_layer_set_tuning(fipa_layer* layer, const fipa_tuning* in);

/* Optional per-stage device timing (CUDA events on the forward's stream).  After enabling,
 * every forward records stage times; fipa_layer_stage_times copies up to n values (ms) in the
 * order recenter, cast, projection, pack, attention, output and returns the count. */
int fipa_layer_set_timing(fipa_layer* layer, int enable);
int fipa_layer_stage_times(const fipa_layer* layer, float* ms, int n);
/* Backward stage times (ms) in the order dout, dfeat, dw_out, prep, attn_kv, attn_q, unpack,
 * recenter, ds, dW, scatter; same enable switch. */
int fipa_layer_bwd_stage_times(const fipa_layer* layer, float* ms, int n);

#ifdef __cplusplus
}
#endif

#endif /* FIPA_B200_H */
