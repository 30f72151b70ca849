// Launch entry points of every sm_100a kernel in the library (host-callable).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <utility>

#include <cstdint>

namespace fipa_b200 {

// Hot-path kernels are launched with programmatic stream serialization (each waits in
// griddepcontrol.wait before touching global memory): the launch of kernel k+1 is processed while
// kernel k's CTAs drain, -0.6% per training step (0.876 -> 0.871 ms).  The dependents are released
// at CTA exit: an explicit early griddepcontrol.launch_dependents (FIPA_PDL_EARLY_TRIGGER) let the
// waiting CTAs crowd the tail and measured 6% slower.  FIPA_PDL=0 (read once) disables it.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}


// SM count of the current device (cached per device, thread-safe); grids of the persistent
// kernels are sized from it.
int device_sm_count();

// ------------------------------------------------------------------ GEMM
// C[M,N] = alpha * A[M,K] . B[K,N] (+ bias[N]) (+ beta*C), rows with row_mask==0 zeroed.
//   a_mn_major = false: A stored row-major [M, K] (lda >= K)
//   a_mn_major = true : A stored row-major [K, M] (lda >= M)      (i.e. A^T given)
//   b_mn_major = false: B stored row-major [N, K] (ldb >= K)      (i.e. B^T given, "K-major")
//   b_mn_major = true : B stored row-major [K, N] (ldb >= N)
// bf16 operands, fp32 accumulation in TMEM (tcgen05.mma kind::f16), TMA-fed.
struct GemmArgs {
    const __nv_bfloat16* A = nullptr;
    const __nv_bfloat16* B = nullptr;
    void* C = nullptr;
    int64_t lda = 0, ldb = 0, ldc = 0;
    int M = 0, N = 0, K = 0;
    bool a_mn_major = false;
    bool b_mn_major = false;
    bool out_bf16 = false;
    bool accumulate = false;  // C += result (fp32 output only)
    int split_k = 1;          // >1: K split over gridDim.z, fp32 C accumulated atomically (zero it first)
    float alpha = 1.0f;
    const float* bias = nullptr;        // [N] or null
    const uint8_t* row_mask = nullptr;  // [M] or null: rows with 0 are written as 0
    // Batched: `batch` independent products z = 0..batch-1 over dense operand stacks (A_z at
    // A + z * (rows of A) * lda, likewise B); C_z at C + (z / batch_h) * ldc_b + (z % batch_h) * ldc_h
    // (plain fp32 C only: no accumulate / split-K / row mask)
    int batch = 1, batch_h = 1;
    int64_t ldc_h = 0, ldc_b = 0;
    // Batched fp32 C only: also write every column as bf16 to C16 (same element strides), and to
    // C only the 32-column chunks flagged in c16_f32_chunks (bit k: columns [32k, 32k + 32))
    __nv_bfloat16* C16 = nullptr;
    uint32_t c16_f32_chunks = 0;
};
void launch_gemm_bf16(const GemmArgs& args, cudaStream_t stream);

// C[M,N] = A[M,K] . B[N,K]^T (+ bias) with masked rows zeroed, fp32 operands (K-major, row
// strides lda / ldb), tcgen05 kind::tf32.  For fp32 accuracy pass split3 operands (K = 3 parts).
struct GemmF32Args {
    const float* A = nullptr;
    const float* B = nullptr;
    float* C = nullptr;
    int64_t lda = 0, ldb = 0, ldc = 0;
    int M = 0, N = 0, K = 0;
    const float* bias = nullptr;
    const uint8_t* row_mask = nullptr;
};
void launch_gemm_tf32(const GemmF32Args& args, cudaStream_t stream);
// split3: out[r, part*ld_part + c] = part_sel(in[r, c]) for parts p = 0, 1, 2, where bit p of
// lo_mask selects lo(x) = x - tf32(x) instead of hi(x) = tf32(x); columns c in [cols, ld_part)
// are written as 0.  planar = true writes part p to out + p * plane instead (row stride ld_part).
// hi/lo split with transpose: in [BH][L][D] -> out [2][BH][D][Lp] (planes `plane` floats apart)
void launch_split_t(const float* in, int BH, int L, int D, float* out, int Lp, int64_t plane, cudaStream_t stream);
void launch_split3(const float* in, int64_t rows, int cols, int64_t ld_in, float* out, int ld_part, int64_t ld_out,
                   int lo_mask, int nparts, cudaStream_t stream, int64_t plane = 0);

// ------------------------------------------------------- FlashIPA layer
// Sizes of one layer configuration (host side, shared with the kernels).
struct LayerDims {
    int d_in, d_z, heads, c, n_query, n_value, rank;
    int n_proj;      // H*(3c + 6Nq + 3Nv): fused projection width
    int zq;          // start of the pair-factor columns: round_up(c + 3Nq + 21, 8)
    int dqk_used;    // zq + r*d_z                (lifted query/key width, see pack.cu)
    int dqk_mma;     // dqk_used rounded up to 16  (MMA K extent of Q.K^T)
    int dqk_pad;     // dqk_used rounded up to 64  (row stride of q_hat / k_hat: 128-byte blocks)
    int dv_used;     // c + r*d_z + 6 + 3Nv       (v | z2 | t_hi | t_lo | R v_p)
    int dv_mma;      // dv_used rounded up to 16   (MMA N extent of P.V)
    int dv_pad;      // dv_used rounded up to 64   (row stride of v_hat)
    int dv_tc;       // value columns accumulated by the tensor cores (multiple of 16, <= 416)
    int dv_simt;     // dv_used - dv_tc trailing value columns accumulated on CUDA cores
    int seg;         // d_z + c + 4Nv             (per-head feature block)
    int feat;        // H*seg
    int din_ld;      // d_in rounded up to 8  (row stride of bf16 GEMM operands, TMA needs 16 B)
    int feat_ld;     // feat rounded up to 8  (row stride of the feature buffer)
};

struct PackArgs {
    const float* proj;     // [BL, n_proj]  s . W_fused (reference column order)
    const float* z1;       // [BL, r, d_z]
    const float* z2;       // [BL, r, d_z]
    const float* rot;      // [BL, 9] row-major
    const float* trans;    // [BL, 3] (already recentred per sample)
    const uint8_t* mask;   // [BL] or null
    const float* head_g;   // [H]  gamma_h * w_l * w_c
    const float* wl_bias;  // [H, d_z]  w_l * w_bias
    float k_scale;         // w_l / sqrt(c)
    void* qhat;            // [B*H, L, dqk_pad]
    void* khat;            // [B*H, L, dqk_pad]
    void* vhat;            // [B*H, L, dv_pad]
    float* colbias;        // [B*H, L]  -g/2 * sum_p |T_j k_p|^2 (natural units), -inf masked
    int B, L;
    bool out_f32;          // write fp32 rows (SIMT f32 path) instead of bf16
};
void launch_pack(const LayerDims& d, const PackArgs& a, cudaStream_t stream);

// Fused projection + pack (proj_pack.cu), bf16 path.  w_heads: head-major bf16 weight copy
// [H * NH, din_ld] (per head: q | k | v | q_p | k_p | v_p columns, padded to NH rows).
struct ProjPackArgs {
    const __nv_bfloat16* s_bf16;   // [BL, din_ld]
    const __nv_bfloat16* w_heads;  // [H * NH, din_ld]
    const float* z1;
    const float* z2;
    const __nv_bfloat16* z1q;      // [BL, r d_z] bf16(log2(e) z1)  (launch_cast_inputs)
    const __nv_bfloat16* z2b;      // [BL, r d_z] bf16(z2)
    const float* rot;
    const float* trans;            // recentred
    const uint8_t* mask;
    const float* head_g;
    const float* wl_bias;
    float k_scale;
    float* proj;                   // [BL, n_proj]: only the point columns are written (write_points)
    bool write_points = true;      // the backward reads them; inference may skip
    float* colbias;
    __nv_bfloat16* qhat;
    __nv_bfloat16* khat;
    __nv_bfloat16* vhat;
    int B, L;
};
bool proj_pack_supported(const LayerDims& d);
int proj_pack_head_width(const LayerDims& d);
void launch_proj_pack(const LayerDims& d, const ProjPackArgs& a, cudaStream_t stream);

struct AttnArgs {
    const __nv_bfloat16* qhat;
    const __nv_bfloat16* khat;
    const __nv_bfloat16* vhat;
    const float* colbias;
    const float* z1;
    const float* rot;
    const float* trans;
    __nv_bfloat16* feat;   // [BL, feat]
    float* lse;            // [B*H, L] natural-log LSE of the shifted logits
    float* o_save;         // [B, L, H, dv_pad] normalised O_hat (fp32, residue-major) for the backward, or null
    int B, L;              // L = query rows (local rows when sharded)
    // Keys (query-row sharding): khat/vhat hold Lk keys as kgroups shards of kchunk rows,
    // [kgroups][B*H][kchunk][pad] (shard g = keys g*kchunk ..).  0 = unsharded (Lk = L).
    int Lk = 0, kchunk = 0;
    int pass_ring[4] = {0, 0, 0, 0};  // two-pass kernel: forced ring (kb, kst, vkeys, vst), 0 = automatic
    int h0 = 0, hc = 0;  // CTA-pair kernel: heads [h0, h0 + hc) of every sample only (hc = 0: all)
};
// tcgen05 attention forward with the K4 epilogue fused (split / pair contraction /
// inverse frame / norms) writing bf16 features.
void launch_attn_fwd_tc(const LayerDims& d, const AttnArgs& a, cudaStream_t stream);
// CTA-pair version (tcgen05 cta_group::2, 256 query rows per pair, streamed K/V rings).
bool attn_fwd_2sm_supported(const LayerDims& d);
void launch_attn_fwd_2sm(const LayerDims& d, const AttnArgs& a, cudaStream_t stream);
// Two-pass CTA-pair version for lifted rows wider than the 2-SM kernel's TMEM/smem budget
// (z_factor_rank 3-4): value columns split over two passes, K streamed in column-block groups.
bool attn_fwd_pass_supported(const LayerDims& d);
void launch_attn_fwd_pass(const LayerDims& d, const AttnArgs& a, cudaStream_t stream);

// ------------------------------------------------------------- backward
struct AttnBwdArgs {
    const __nv_bfloat16* qhat;
    const __nv_bfloat16* khat;
    const __nv_bfloat16* vhat;
    const __nv_bfloat16* dohat;  // [B*H, L, dv_pad]
    const float* lse;            // [B*H, L]
    const float* Dvec;           // [B*H, L]
    float* dq_acc;               // [B, L, H, acc_ld] (residue-major) = dS . K_hat
    float* dk_acc;               //                  = dS^T . Q_hat
    float* dv_acc;               //                  = P^T . dO_hat
    int acc_ld;
    int B, L;                    // L = local query rows
    // Query-row sharding: khat / vhat hold all Lk = G*kchunk keys gathered rank-major
    // [G][B*H][kchunk][pad]; dk_acc / dv_acc then receive PARTIAL sums for all keys, rank-major
    // [G][B][kchunk][H][acc_ld] (ready for a reduce-scatter).  0 = unsharded (Lk = L).
    int Lk = 0, kchunk = 0;
    // Optional materialised dS [B*H][L keys][ds_ld] (bf16, unsharded only): the dK/dV kernel
    // stores its dS tiles there and dQ becomes one batched GEMM dS^T . K_hat (which & 2).
    __nv_bfloat16* ds = nullptr;
    int ds_ld = 0;
    // Query chunk of a materialised-dS backward too long for one dS buffer: the dK/dV kernel runs
    // over queries [q0, q0 + qn) (dS [B*H][L keys][ds_ld] holds that chunk's columns; acc_add: the
    // chunk's partial dK / dV are added to the accumulators -- every chunk after the first), and the
    // dQ GEMM writes those query rows.  qn = 0: all queries.
    int q0 = 0, qn = 0, acc_add = 0;
    int ring[5] = {0, 0, 0, 0, 0};  // forced ring plan (nst1, nst2, nab, kb1, slice rows), 0 = automatic
    // Optional bf16 copies of dK / dV ([B, L, H, acc_ld], unsharded whole-query launches only):
    // every accumulator column also leaves as bf16 (half the drain bytes of the scalar and pair
    // columns, which bwd_unpack reads from here); dk_acc / dv_acc then receive only the 32-column
    // chunks that hold point / translation columns (cancellation-sensitive, kept fp32).
    __nv_bfloat16* dk16 = nullptr;
    __nv_bfloat16* dv16 = nullptr;
    __nv_bfloat16* dq16 = nullptr;  // same for dQ from the materialised-dS GEMM (its epilogue)
};
bool attn_bwd_supported(const LayerDims& d);
// which: 1 = dK/dV kernel, 2 = dQ kernel, 3 = both
void launch_attn_bwd(const LayerDims& d, const AttnBwdArgs& a, cudaStream_t stream, int which = 3);

struct BwdPrepArgs {
    const __nv_bfloat16* dfeat;   // [BL, feat_ld] dOut . w_out^T (bf16)
    const float* ohat;            // [B, L, H, dv_pad] fp32 (residue-major), saved by the forward
    const float* z1;              // [BL, r*d_z]
    const float* rot;             // [BL, 9]
    const float* trans_c;         // [BL, 3] recentred
    __nv_bfloat16* dohat;         // [B*H, L, dv_pad]
    float* Dvec;                  // [B*H, L]
    float* dz1_epi;               // [BL, r*d_z]
    float* geo_epi;               // [BL, 12]: dR (9) | dt (3) of the epilogue
    int B, L;
};
void launch_bwd_prep(const LayerDims& d, const BwdPrepArgs& a, cudaStream_t stream);

struct BwdUnpackArgs {
    const float* dq_acc;
    const float* dk_acc;
    const float* dv_acc;
    int acc_ld;
    const float* proj;      // [BL, n_proj] forward projections (local points)
    const float* rot;
    const float* trans_c;
    const float* z2;
    const float* head_g;    // [H]
    const float* wl_bias;   // [H, d_z]
    float k_scale;
    const float* dz1_epi;
    const float* geo_epi;   // [BL, 12]
    __nv_bfloat16* dproj;   // [BL, nproj_ld]
    int nproj_ld;
    float* dz1;             // [BL, r*d_z]
    float* dz2;             // [BL, r*d_z]
    float* drot;            // [BL, 9] or null
    float* dt_c;            // [BL, 3] gradient w.r.t. the recentred translations
    float* dg;              // [H]     accumulated (zero first): dL/d(gamma_h w_l w_c)
    float* dwlb;            // [H, d_z] accumulated (zero first): dL/d(w_l w_bias)
    int B, L;
    // bf16 dK / dV (AttnBwdArgs::dk16 / dv16): the scalar and pair columns are read from there
    // (null: from dk_acc / dv_acc); the geometry columns always come from the fp32 accumulators
    const __nv_bfloat16* dk16 = nullptr;
    const __nv_bfloat16* dv16 = nullptr;
    const __nv_bfloat16* dq16 = nullptr;  // (independent of dk16 / dv16: the streaming dQ kernel is fp32)
};
void launch_bwd_unpack(const LayerDims& d, const BwdUnpackArgs& a, cudaStream_t stream);
// Materialised attention backward (FlashIpaLayer::dense_attention_backward), rows of length L with
// stride ld (a multiple of 8): P = bf16(2^(S - lse * log2 e)) (0 for a row whose lse is -inf: no
// valid key); dS = bf16(P (dP - D)).
void launch_dense_softmax(const float* S, int ld, const float* lse, int64_t rows, int L, __nv_bfloat16* P,
                          cudaStream_t stream);
void launch_dense_ds(const __nv_bfloat16* P, const float* dP, int ld, const float* Dvec, int64_t rows, int L,
                     __nv_bfloat16* dS, cudaStream_t stream);

// dOut with masked rows zeroed -> bf16 [BL, ld_out]; db[d_in] += column sums (zero db first).
void launch_bwd_dout(const float* dout, const uint8_t* mask, __nv_bfloat16* out, int ld_out, float* db,
                     int64_t rows, int cols, cudaStream_t stream);
// Column blocks of the fused projection: block i = columns [col0[i], col0[i] + width[i]) of the
// [d_in, n_proj] gradient, written row-major at dst_off[i] (dst_off[6] = d_in * n_proj).
struct ScatterCols {
    int col0[6], width[6];
    int64_t dst_off[7];
};
void launch_scatter_proj_grad(const float* src, int d_in, int n_proj, const ScatterCols& seg, float* dst,
                              cudaStream_t stream);
// scatter + d(w_bias) = red[H..] * scale[H], d(gamma_raw) = red[..H] * scale[..H] in one launch
void launch_finish_weight_grads(const float* src, int d_in, int n_proj, const ScatterCols& seg, float* dst,
                                const float* red, const float* scale, int H, int dz, float* dw_bias, float* dgamma,
                                cudaStream_t stream);
// Translation gradient through the per-sample recentring: dt = mask*(dt_c - mean_valid(dt_c)).
void launch_bwd_recenter(const float* dt_c, const uint8_t* mask, float* dt, int B, int L, cudaStream_t stream);
// acc[i] += x[i]
void launch_add_inplace(float* acc, const float* x, int64_t n, cudaStream_t stream);
// out[i] = in[i] * scale[i % period]
void launch_scale_vec(const float* in, const float* scale, int period, float* out, int n, cudaStream_t stream);

// ------------------------------------------------- pair-factor producer (pair_features.cu)
struct KnnSpec {
    int k, n_bins, pe_dim;
    double d_min, d_max;
};
size_t knn_smem_bytes(const KnnSpec& spec);
// trans [B, L, 3] -> out [B, L, k, n_bins + pe_dim]; d_freq [pe_dim/2] = 10000^(-2p/pe_dim)
void launch_knn_distogram(const float* trans, int B, int L, const KnnSpec& spec, const double* d_freq, float* out,
                          cudaStream_t stream);
// float64 translations and features end to end (the reference's f64 API: no rounding before the distance)
void launch_knn_distogram(const double* trans, int B, int L, const KnnSpec& spec, const double* d_freq, double* out,
                          cudaStream_t stream);
// w [K, N] fp32 row-major -> wt [N, ld] bf16 (K-major B operand), pad columns zeroed
void launch_transpose_to_bf16(const float* w, int K, int N, __nv_bfloat16* wt, int ld, cudaStream_t stream);

// Row-wise fp32 -> bf16 conversion (s input, dOut, ...).
void launch_f32_to_bf16(const float* in, __nv_bfloat16* out, int64_t n, cudaStream_t stream);
// Same for a [rows, cols] matrix written with row stride ld_out (pad columns left untouched).
// s -> bf16 [rows, din_ld] plus the pair-factor blocks bf16(log2(e) z1), bf16(z2) of proj_pack.
bool cast_inputs_supported(int d_in, int din_ld, int rdz);
// (trans != null: the same launch also recentres the B samples' translations into trans_c)
void launch_cast_inputs(const float* s, __nv_bfloat16* s_bf16, int d_in, int din_ld, const float* z1, const float* z2,
                        __nv_bfloat16* z1q, __nv_bfloat16* z2b, int rdz, int64_t rows, cudaStream_t stream,
                        const float* trans = nullptr, const uint8_t* mask = nullptr, float* trans_c = nullptr,
                        int B = 0, int L = 0);
void launch_f32_to_bf16_2d(const float* in, __nv_bfloat16* out, int64_t rows, int cols, int ld_out,
                           cudaStream_t stream);
// Trunk step: s += ipa_out; backbone update of the frames (rot [rows,9], trans [rows,3]) in place.
void launch_trunk_update(float* s, const float* ipa_out, const float* w_bb, const float* b_bb, float* rot,
                         float* trans, const uint8_t* mask, int64_t rows, int d_in, cudaStream_t stream);
// Query-row sharding: per-sample {sum x, sum y, sum z, count} of valid local translations, and
// recentring with (all-reduced) global sums.
void launch_centroid_sums(const float* trans, const uint8_t* mask, float* sums, int B, int L, cudaStream_t stream);
// out = trans - sum/count per sample; rows with zero_masked[row] == 0 are written as 0 when given.
void launch_recenter_with_sums(const float* trans, const float* sums, float* out, int B, int L, cudaStream_t stream,
                               const uint8_t* zero_masked = nullptr);
// flags[b, i] = 1 for every row of a sample without a valid residue (flash_ipa.cpp:156-158)
void launch_fully_masked(const uint8_t* mask, uint8_t* flags, int B, int L, cudaStream_t stream);
// Subtract each sample's translation centroid (exact: the layer is invariant to it).
void launch_recenter(const float* trans, const uint8_t* mask, float* out, int B, int L,
                     cudaStream_t stream);

// ------------------------------------------------------ SIMT fp32 path
void launch_gemm_f32(const float* A, int lda, const float* B, float* C, int M, int N, int K,
                     const float* bias, const uint8_t* row_mask, cudaStream_t stream);
struct AttnF32Args {
    const float* qhat;
    const float* khat;
    const float* vhat;
    const float* colbias;
    const float* z1;
    const float* rot;
    const float* trans;
    float* feat;  // [BL, feat] fp32
    float* lse;
    int B, L;
};
void launch_attn_fwd_f32(const LayerDims& d, const AttnF32Args& a, cudaStream_t stream);
// fp32-accuracy attention on the tensor cores (attn_fwd_f32tc.cu, "3xTF32"): q/k_hat split into
// tf32 hi and lo planes ([B*H, L, dqk_pad] each, launch_split3 planar), v_hat transposed into
// [B*H, dv_pad, Lp] hi / lo planes (launch_split_t; Lp = L rounded up to 4).
struct AttnF32TcArgs {
    const float *q_hi, *q_lo, *k_hi, *k_lo, *v_hi, *v_lo;
    const float* z1;
    const float* rot;
    const float* trans;
    float* feat;  // [BL, feat_ld] fp32
    float* lse;
    int B, L;
};
bool attn_fwd_f32tc_supported(const LayerDims& d);
void launch_attn_fwd_f32tc(const LayerDims& d, const AttnF32TcArgs& a, cudaStream_t stream);

// ------------------------------------------------ quadratic-memory arms (dense.cu)
// Dense IPA forward (reference_forward, proj/src/ipa.cpp:244-310), fp32: materialises the pair
// tensor z [B, L, L, d_z] and the logits / attention [B, H, L, L].
struct DenseArgs {
    int B, L;
    const float* s;
    const float* z1;
    const float* z2;
    const float* rot;
    const float* trans;     // not recentred: differences are formed directly
    const uint8_t* mask;    // [BL] or null
    const float* wproj;     // f32 [d_in, n_proj]
    const float* wout;      // f32 [feat, d_in]
    const float* bout;
    const float* head_g;
    const float* wl_bias;
    float k_scale;
    float* proj;            // [BL, n_proj]
    float* gq;              // [BL, H*Nq*3] global query points
    float* gk;              // [BL, H*Nq*3]
    float* vcat;            // [B, H, L, c + 3Nv]  v | T_j v_p
    float* z;               // [B, L, L, d_z]
    float* logits;          // [B, H, L, L] (softmax in place)
    float* ov;              // [B, H, L, c + 3Nv]
    float* oz;              // [BL, H, d_z]
    float* feat;            // [BL, feat]
    float* out;             // [BL, d_in]
};
void launch_dense_ipa(const LayerDims& d, const DenseArgs& a, cudaStream_t stream);
// Generic attention (attention_kernel.hpp): q, k [H, L, d_qk], v [H, L, d_v], key mask [L].
void launch_naive_attention_f32(int H, int L, int dqk, int dv, const float* q, const float* k, const float* v,
                                const uint8_t* mask, float* logits, float* out, cudaStream_t stream);
bool flash_attention_f32_supported(int dv);
void launch_flash_attention_f32(int H, int L, int dqk, int dv, const float* q, const float* k, const float* v,
                                const uint8_t* mask, float* out, cudaStream_t stream);

}  // namespace fipa_b200
