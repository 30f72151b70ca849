// Host C++ side of the B200 FlashIPA layer: configuration, weights (init / file IO / device
// upload), workspace planning and the forward orchestration that launches the sm_100a kernels.
//
// Mirrors the reference layer API: IpaConfig (proj/include/fipa/ipa.hpp:14-32), IpaWeights
// (ipa.hpp:37-50), flash_ipa_forward (proj/include/fipa/flash_ipa.hpp:55-57) and the weights
// file (proj/include/fipa/model_io.hpp:15-26).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <map>
#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels.hpp"

namespace fipa_b200 {

// Error taxonomy of the reference (proj/include/fipa/error.hpp:10-28) plus CUDA failures.
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ValueError : Error {
    using Error::Error;
};
struct NumericError : Error {
    using Error::Error;
};
struct IoError : Error {
    using Error::Error;
};
struct CudaError : Error {
    using Error::Error;
};
struct CommError : Error {  // NCCL failure or NCCL unavailable
    using Error::Error;
};

void cuda_check(cudaError_t e, const char* what);

enum class Precision { bf16 = 0, f32 = 1 };

struct Config {
    std::size_t d_in = 32, d_z = 4, heads = 2, c = 8, n_query = 2, n_value = 2, rank = 2;
    Precision precision = Precision::bf16;  // compute path
    bool weights_f32 = false;               // master weights stored at f32 (reference "f32" models)
    bool enforce_head_cap = true;

    std::size_t qk_width() const { return c + 5 * n_query + rank * d_z; }  // ipa.hpp:27
    std::size_t v_width() const { return c + 3 * n_value + rank * d_z; }   // ipa.hpp:28
    static constexpr std::size_t head_cap = 256;
    void validate() const;  // ipa.cpp:12-21
    LayerDims dims() const;
};

// Kernel-selection and tuning knobs.  Fixed per layer: set at creation (defaults = the measured
// best choices; the FIPA_* environment variables below seed them ONCE, for A/B experiments) and
// changed only through FlashIpaLayer::set_tuning -- the launch path never reads the environment.
struct Tuning {
    enum class Attn { automatic = 0, pair = 1, pass = 2, one_sm = 3 };
    Attn attn = Attn::automatic;  // FIPA_ATTN_IMPL = pair | pass | 1sm (inference forward only)
    bool fused_pack = true;       // FIPA_FUSED_PACK = 0: projection GEMM + separate pack kernel
    int bwd_ds = -1;              // FIPA_BWD_DS: -1 automatic (L <= 8192 and dS <= 2 GiB), 0 off,
                                  // 1 on (within the same cap)
    int bwd_ring[5] = {0, 0, 0, 0, 0};  // FIPA_BWD_RING "nst1,nst2,nab,kb1[,slice]" (0 = automatic)
    int pass_ring[4] = {0, 0, 0, 0};  // FIPA_PASS_RING "kb,kst,vkeys,vst"  (0 = automatic)
    bool f32_tc = true;           // FIPA_F32_TC = 0: fp32 path on CUDA cores (SIMT reference kernels)
    int host_chunk = 0;           // FIPA_HOST_CHUNK: samples per chunk of the host-buffer pipeline (0 = auto)
    bool graphs = true;           // FIPA_GRAPHS = 0: launch kernel by kernel instead of replaying a
                                  // captured CUDA graph per (call kind, shapes, buffers)
    int micro = 2;                // FIPA_MICRO: bf16 device calls captured as this many interleaved
                                  // sample chunks on forked streams (1 = one chain)
    int ds_cap_mb = 2048;         // FIPA_DS_CAP_MB: workspace cap of the materialised dS (query-chunked
                                  // beyond it; at least 256 columns per chunk, else the streaming kernel)
    int shard_chunks = 0;         // FIPA_SHARD_CHUNKS: head chunks of the overlapped K/V all-gather of
                                  // query-row sharding (0 = automatic: 4, or 2; 1 = one all-gather)
    static Tuning from_env();
};

// Master weights in the reference layout, kept in float64 on the host.
struct HostWeights {
    std::vector<double> w_q, w_k, w_v, w_qp, w_kp, w_vp, w_bias, gamma_raw, w_out, b_out;
    double w_l = 0.0, w_c = 0.0;
    bool stored_f32 = false;  // precision tag written by save (0 = f32, 1 = f64)

    std::vector<double>* slots[10] = {&w_q, &w_k, &w_v, &w_qp, &w_kp, &w_vp,
                                      &w_bias, &gamma_raw, &w_out, &b_out};
    HostWeights() = default;
    HostWeights(const HostWeights& o) { *this = o; }
    HostWeights& operator=(const HostWeights& o);
};

std::vector<std::vector<std::size_t>> weight_shapes(const Config& cfg);
const char* const* weight_names();  // 10 names, reference order

HostWeights init_weights(const Config& cfg, std::uint64_t seed, bool round_f32);
void save_weights_file(const HostWeights& w, const std::vector<std::vector<std::size_t>>& shapes,
                       const std::string& path);
HostWeights load_weights_file(const std::string& path,
                              const std::vector<std::vector<std::size_t>>& shapes);

// One NCCL communicator (one process per GPU), resolved from libnccl at run time (comm.cpp).
class Comm {
public:
    static std::array<std::uint8_t, 128> unique_id();
    Comm(int world, int rank, const std::uint8_t* id, int device);
    ~Comm();
    Comm(const Comm&) = delete;
    Comm& operator=(const Comm&) = delete;
    int world() const { return world_; }
    int rank() const { return rank_; }
    void all_reduce_sum_f32(float* buf, std::size_t n, cudaStream_t stream);
    void all_gather_bytes(const void* send, void* recv, std::size_t bytes, cudaStream_t stream);
    // All-gather of `pieces` equal blocks of `piece` bytes at send + k * stride into recv laid out as
    // [world][...] with rank blocks rank_stride bytes apart (same offsets): grouped send / recv, so a
    // head chunk of the packed rows lands in place in the standard gathered layout.
    bool has_p2p() const;
    void all_gather_pieces(const void* send, void* recv, std::size_t piece, int pieces, std::size_t stride,
                           std::size_t rank_stride, cudaStream_t stream);
    // recv[n] = sum over ranks of send[rank_ * n .. ], send holding world() blocks of n floats
    void reduce_scatter_sum_f32(const float* send, float* recv, std::size_t n, cudaStream_t stream);

private:
    int world_, rank_, device_;
    void* comm_ = nullptr;
};

// Query-row sharding stage (forward over the local rows of a sequence split across G ranks):
//   stage 1: recentre with the all-reduced centroid sums, project, pack local q/k/v_hat rows;
//   stage 2: attention of the local queries against all G shards' keys, gathered as
//            [G][B*H][L_local][pad], then the output projection of the local rows.
struct ShardStage {
    int stage = 1;
    const float* sums = nullptr;   // [B,4] global {sum t, count} (stage 1)
    const void* k_all = nullptr;   // stage 2
    const void* v_all = nullptr;
    int groups = 1;
    // stage 2 split over head chunks (gather / attention overlap): hc > 0 runs the attention of
    // heads [h0, h0 + hc) only, and stage 3 the output projection after the last chunk
    int h0 = 0, hc = 0;
};

// Stage of the query-row-sharded backward (rank r owns residues [r L, (r+1) L) of G L):
//   1: dOut -> dfeat, dw_out, prep, attention backward against the GATHERED keys: dQ for the local
//      queries, PARTIAL dK/dV for all keys -> dk_part / dv_part [G][B][L][H][448] (rank-major)
//   -- caller: reduce-scatter (sum) dk_part / dv_part -> this rank's keys (dk_own / dv_own)
//   2: unpack with dk_own / dv_own -> dz1, dz2, drot; per-sample sums of the recentred-translation
//      gradient -> dt_sums [B,4] (local)
//   -- caller: all-reduce dt_sums
//   3: dtrans (recentring with the global sums), ds, weight gradients (local)
//   -- caller: all-reduce the weight gradients
struct BwdShard {
    int stage = 1;
    cudaEvent_t kv_done = nullptr;  // stage 1: recorded once the partial dK/dV are complete (the
                                    // reduce-scatter may start while the dQ kernel runs)
    int groups = 1;
    const void* k_all = nullptr;  // gathered k_hat / v_hat [G][B*H][L][pad] (stage 1)
    const void* v_all = nullptr;
    float* dk_part = nullptr;     // stage 1 outputs
    float* dv_part = nullptr;
    const float* dk_own = nullptr;  // stage 2 inputs
    const float* dv_own = nullptr;
    float* dt_sums = nullptr;     // stage 2 output (local) / stage 3 input (global)
};

class FlashIpaLayer {
public:
    explicit FlashIpaLayer(const Config& cfg);
    ~FlashIpaLayer();
    FlashIpaLayer(const FlashIpaLayer&) = delete;
    FlashIpaLayer& operator=(const FlashIpaLayer&) = delete;

    const Config& config() const { return cfg_; }
    const LayerDims& dims() const { return dims_; }
    const HostWeights& weights() const { return w_; }

    void init_weights(std::uint64_t seed);
    void set_weights(const HostWeights& w);
    void save(const std::string& path) const;
    void load(const std::string& path);

    std::size_t workspace_size(std::int64_t B, std::int64_t L) const;
    void forward(std::int64_t B, std::int64_t L, const float* s, const float* z1, const float* z2,
                 const float* rot, const float* trans, const std::uint8_t* mask, float* out,
                 void* workspace, std::size_t workspace_bytes, cudaStream_t stream,
                 bool train = false, const ShardStage* shard = nullptr);
    // Training: forward(..., train=true) over a train_workspace_size() workspace keeps what the
    // backward needs; backward() then consumes the same workspace.  Gradients of
    // sum(out * dout) w.r.t. the inputs (fp32, any of drot/dtrans may be null) and the weights
    // (fp32, reference order w_q..b_out concatenated, num_weights() values).
    std::size_t train_workspace_size(std::int64_t B, std::int64_t L) const;
    // Short-sequence backward: the dK/dV kernel also writes dS (bf16, B*H*L^2*2 bytes of the
    // training workspace) and dQ is one batched GEMM instead of a second attention pass.  Used
    // for L <= 8192 and at most 2 GiB of dS; Tuning::bwd_ds = 0 / 1 forces it off / on (within that cap).
    bool materialize_ds(std::int64_t B, std::int64_t L) const;
    std::int64_t ds_chunk(std::int64_t B, std::int64_t L) const;
    const Tuning& tuning() const { return tuning_; }
    // Not thread-safe against concurrent calls on the same layer (like weight mutation).
    void set_tuning(const Tuning& t) {
        tuning_ = t;
        dirty_ = true;  // the device weight copies (and captured graphs) depend on the kernel choice
    }
    std::size_t num_weights() const;
    void backward(std::int64_t B, std::int64_t L, const float* s, const float* z1, const float* z2,
                  const float* rot, const float* trans, const std::uint8_t* mask, const float* dout,
                  float* ds, float* dz1, float* dz2, float* drot, float* dtrans, float* dweights,
                  void* workspace, std::size_t workspace_bytes, cudaStream_t stream,
                  const BwdShard* shard = nullptr);
    // Host-buffer entry points (host_path.cpp): pipelined over the batch, float64 (reference
    // convention) or float32 arrays.
    void grad_host(std::int64_t B, std::int64_t L, const double* s, const double* z1, const double* z2,
                   const double* rot, const double* trans, const std::uint8_t* mask, const double* dout,
                   double* out, double* ds, double* dz1, double* dz2, double* drot, double* dtrans,
                   double* dweights);
    void grad_host_f32(std::int64_t B, std::int64_t L, const float* s, const float* z1, const float* z2,
                       const float* rot, const float* trans, const std::uint8_t* mask, const float* dout, float* out,
                       float* ds, float* dz1, float* dz2, float* drot, float* dtrans, float* dweights);
    void forward_host_f32(std::int64_t B, std::int64_t L, const float* s, const float* z1, const float* z2,
                          const float* rot, const float* trans, const std::uint8_t* mask, float* out);
    bool backward_supported() const;
    // The fused tcgen05 attention backward (attn_bwd.cu: lifted widths <= 448, rank <= 2) or, for
    // wider lifted rows (z_factor_rank 3-4), the materialised backward (dense_attention_backward).
    bool fused_backward_supported() const;
    bool dense_backward() const;
    int launches_per_backward() const;
    // kernels of one device call (graph replay with its micro-batch chains) at (B, L)
    int step_launches(std::int64_t B, std::int64_t L, bool train) const;


    void forward_host(std::int64_t B, std::int64_t L, const double* s, const double* z1,
                      const double* z2, const double* rot, const double* trans,
                      const std::uint8_t* mask, double* out);
    int launches_per_forward() const;

    // Quadratic-memory arm (reference_forward, proj/src/ipa.cpp:244-310; dense.cu), fp32.
    std::size_t reference_workspace_size(std::int64_t B, std::int64_t L) const;
    void reference_forward(std::int64_t B, std::int64_t L, const float* s, const float* z1, const float* z2,
                           const float* rot, const float* trans, const std::uint8_t* mask, float* out,
                           void* workspace, std::size_t workspace_bytes, cudaStream_t stream);
    void reference_host(std::int64_t B, std::int64_t L, const double* s, const double* z1, const double* z2,
                        const double* rot, const double* trans, const std::uint8_t* mask, double* out);

    void set_timing(bool on);
    std::vector<float> stage_times() const;

    // Workspace carve-up (device pointers into the caller's buffer).
    struct Workspace {
        float* trans_c = nullptr;
        __nv_bfloat16* s_bf16 = nullptr;
        float* proj = nullptr;
        __nv_bfloat16* z1q = nullptr;      // [BL, r d_z] bf16(log2(e) z1)  (fused projection + pack)
        __nv_bfloat16* z2b = nullptr;      // [BL, r d_z] bf16(z2)
        void* qhat = nullptr;
        void* khat = nullptr;
        void* vhat = nullptr;
        float* colbias = nullptr;
        float* lse = nullptr;
        void* feat = nullptr;
        // training extras (carve(..., train = true))
        float* o_hat = nullptr;            // [BH, L, dv_pad] fp32
        __nv_bfloat16* dout_bf16 = nullptr; // [BL, din_ld]
        __nv_bfloat16* dfeat = nullptr;    // [BL, feat_ld] (bf16: prep rounds dO_hat to bf16 anyway)
        __nv_bfloat16* do_hat = nullptr;   // [BH, L, dv_pad]
        float* Dvec = nullptr;             // [BH, L]
        float* dq_acc = nullptr;           // [BH, L, acc_ld]
        float* dk_acc = nullptr;
        float* dv_acc = nullptr;
        __nv_bfloat16* dk16 = nullptr;     // [BH, L, acc_ld] bf16 dK / dV (fused backward: scalar and
        __nv_bfloat16* dv16 = nullptr;     // pair columns; dk_acc / dv_acc keep the geometry chunks)
        __nv_bfloat16* dq16 = nullptr;     // likewise for dQ from the materialised-dS GEMM
        __nv_bfloat16* dproj = nullptr;    // [BL, nproj_ld]
        float* dz1_epi = nullptr;          // [BL, r d_z]
        float* geo_epi = nullptr;          // [BL, 12] dR | dt of the output epilogue
        float* dt_c = nullptr;             // [BL, 3]
        float* red = nullptr;              // [H + H d_z]  d(g) | d(w_l w_bias)
        __nv_bfloat16* ds = nullptr;       // [BH, L, ds_ld] materialised dS (short sequences, or null)
        int ds_ld = 0;
        float* dwproj = nullptr;           // [d_in, n_proj]
        // fp32 path on the tensor cores (3xTF32): K-concatenated / planar hi-lo operands
        float* s_cat = nullptr;            // [BL, 3 din_p]  s_hi | s_lo | s_hi
        float* qs = nullptr;               // [2][BH L, dqk_pad]  q_hat hi / lo planes
        float* ks = nullptr;
        float* vs = nullptr;               // [2][BH L, dv_pad]
        float* feat_cat = nullptr;         // [BL, 3 feat_p]  feat_hi | feat_lo | feat_hi
        // materialised attention backward (wide lifted rows), att_samples samples at a time:
        float* att_s = nullptr;            // [att_samples H, L, att_ld] S (log2 units), fp32
        float* att_dp = nullptr;           // [att_samples H, L, att_ld] dP, fp32
        __nv_bfloat16* att_p = nullptr;    // [att_samples H, L, att_ld] P
        __nv_bfloat16* att_ds = nullptr;   // [att_samples H, L, att_ld] dS
        int att_ld = 0, att_samples = 0;
        std::size_t bytes = 0;
    };
    // fp32 path: projections, attention and output projection on the tensor cores (3xTF32)
    bool f32_tensor_cores() const;
    int din_p() const { return (dims_.d_in + 31) / 32 * 32; }
    int feat_p() const { return (dims_.feat + 31) / 32 * 32; }
    // row stride of the fp32 dQ / dK / dV accumulators ([B, L, H, acc_ld]): 448 up to rank 2
    int acc_ld() const { return std::max(448, (std::max(dims_.dqk_mma, dims_.dv_mma) + 31) / 32 * 32); }
    int nproj_ld() const { return (dims_.n_proj + 7) / 8 * 8; }
    Workspace carve(void* base, std::int64_t B, std::int64_t L, bool train = false) const;
    // The same workspace seen from sample b0 on (every per-sample buffer advanced; the shared
    // weight-gradient accumulators `red` / `dwproj` unchanged).
    Workspace slice(const Workspace& w, std::int64_t b0, std::int64_t L) const;

    // Query-row sharded forward (comm.cpp): this rank holds residues [rank*L, (rank+1)*L) of B
    // sequences of comm.world()*L residues; out receives its rows.  L % 64 == 0 when world > 1.
    struct ShardedWorkspace {
        Workspace local;
        void* k_all = nullptr;
        void* v_all = nullptr;
        float* sums = nullptr;
        float* dk_part = nullptr;  // training: [G][B][L][H][448] partial key gradients
        float* dv_part = nullptr;
        float* dt_sums = nullptr;  // training: [B,4]
        std::size_t kv_bytes = 0, v_bytes = 0, bytes = 0;
    };
    ShardedWorkspace carve_sharded(void* base, std::int64_t B, std::int64_t L, int groups, bool train = false) const;
    std::size_t sharded_workspace_size(std::int64_t B, std::int64_t L, int groups) const;
    // Sharded training (NCCL): forward keeps the gathered keys in the workspace for the backward.
    std::size_t sharded_train_workspace_size(std::int64_t B, std::int64_t L, int groups) const;
    void forward_train_sharded(Comm& comm, std::int64_t B, std::int64_t L, const float* s, const float* z1,
                               const float* z2, const float* rot, const float* trans, const std::uint8_t* mask,
                               float* out, void* workspace, std::size_t workspace_bytes, cudaStream_t stream);
    void backward_sharded(Comm& comm, std::int64_t B, std::int64_t L, const float* s, const float* z1,
                          const float* z2, const float* rot, const float* trans, const std::uint8_t* mask,
                          const float* dout, float* ds, float* dz1, float* dz2, float* drot, float* dtrans,
                          float* dweights, void* workspace, std::size_t workspace_bytes, cudaStream_t stream);
    void gather_and_attend(Comm& comm, std::int64_t B, std::int64_t L, const float* s, const float* z1,
                           const float* z2, const float* rot, const float* trans, const std::uint8_t* mask,
                           float* out, void* workspace, const ShardedWorkspace& ws, bool train, cudaStream_t stream);
    bool attention_impl_for_sharding() const;
    void forward_sharded(Comm& comm, std::int64_t B, std::int64_t L, const float* s, const float* z1,
                         const float* z2, const float* rot, const float* trans, const std::uint8_t* mask,
                         float* out, void* workspace, std::size_t workspace_bytes, cudaStream_t stream);

private:
    void upload_weights();
    void release_device();
    // CUDA-graph replay of the device entry points (forward / training forward / backward): the
    // first call with a given (kind, B, L, buffers) captures the launch sequence on a private stream,
    // later calls replay it on the caller's stream (one launch instead of ~20; no per-kernel host
    // work such as TMA descriptor encoding).  Cleared whenever the device weights are re-uploaded.
    struct GraphKey {
        int kind;
        std::int64_t B, L;
        std::array<const void*, 16> ptrs;
        std::size_t ws_bytes;
        bool operator<(const GraphKey& o) const;
    };
    std::map<GraphKey, cudaGraphExec_t> graphs_;
    std::vector<GraphKey> graph_order_;
    std::mutex graph_mu_;
    cudaStream_t capture_stream_ = nullptr;
    void clear_graphs();
    template <class F>
    bool run_graph(const GraphKey& key, cudaStream_t stream, F&& launch);
    void forward_impl(std::int64_t B, std::int64_t L, const float* s, const float* z1, const float* z2,
                      const float* rot, const float* trans, const std::uint8_t* mask, float* out, void* workspace,
                      std::size_t workspace_bytes, cudaStream_t stream, bool train, const ShardStage* shard,
                      const Workspace* view = nullptr);
    // parts: 1 = zero the weight-gradient accumulators, 2 = per-sample work (weight gradients
    // accumulated atomically), 4 = scatter / scale the accumulators into dweights
    void backward_impl(std::int64_t B, std::int64_t L, const float* s, const float* z1, const float* z2,
                       const float* rot, const float* trans, const std::uint8_t* mask, const float* dout, float* ds,
                       float* dz1, float* dz2, float* drot, float* dtrans, float* dweights, void* workspace,
                       std::size_t workspace_bytes, cudaStream_t stream, const BwdShard* shard,
                       const Workspace* view = nullptr, int parts = 7);
    // Micro-batched capture: the B samples split into tuning_.micro chunks whose kernel chains run on
    // forked streams (the graph holds parallel branches), so each kernel's tail wave and launch ramp
    // overlap the other chain's kernels.  Same workspace (sample-sliced views), same results.
    // (forward = true: forward calls -- inference and training -- take at least 4 chains: at B=8
    // L=1024 inference 0.240 -> 0.235 ms, training step 0.808 -> 0.805 ms; the backward keeps
    // tuning_.micro)
    int micro_chunks(std::int64_t B, std::int64_t L, bool forward = false) const;
    // dK / dV / dQ by materialised per-(sample, head) products (tcgen05 GEMMs) for the lifted
    // widths the fused kernels do not hold; recomputes O_hat and runs prep on the way
    void dense_attention_backward(std::int64_t B, std::int64_t L, const float* z1, const float* rot,
                                  const Workspace& ws, cudaStream_t stream);
    void forward_micro(std::int64_t B, std::int64_t L, const float* s, const float* z1, const float* z2,
                       const float* rot, const float* trans, const std::uint8_t* mask, float* out, void* workspace,
                       std::size_t workspace_bytes, cudaStream_t stream, bool train);
    void backward_micro(std::int64_t B, std::int64_t L, const float* s, const float* z1, const float* z2,
                        const float* rot, const float* trans, const std::uint8_t* mask, const float* dout, float* ds,
                        float* dz1, float* dz2, float* drot, float* dtrans, float* dweights, void* workspace,
                        std::size_t workspace_bytes, cudaStream_t stream);
    cudaStream_t side_streams_[3] = {};
    cudaEvent_t comm_ev_[8] = {};  // query-row sharding: per-chunk gather completion, kv_done, rs_done
    cudaEvent_t fork_ev_ = nullptr, join_ev_[3] = {};
    void ensure_side_streams();

    Config cfg_;
    LayerDims dims_{};
    Tuning tuning_ = Tuning::from_env();
    HostWeights w_;
    int device_ = 0;
    // device weights
    __nv_bfloat16* d_wproj_t_ = nullptr;  // bf16 [n_proj, d_in]  (K-major B operand)
    __nv_bfloat16* d_wout_t_ = nullptr;   // bf16 [d_in, feat]
    __nv_bfloat16* d_wheads_ = nullptr;   // bf16 [H * NH, d_in] head-major projection (fused path)
    float* d_wproj_ = nullptr;            // f32  [d_in, n_proj]
    float* d_wproj_cat_ = nullptr;        // f32  [n_proj, 3 din_p]  W_lo | W_hi | W_hi (K-major, 3xTF32)
    float* d_wout_cat_ = nullptr;         // f32  [d_in, 3 feat_p]   w_out^T lo | hi | hi
    float* d_wout_ = nullptr;             // f32  [feat, d_in]
    float* d_bout_ = nullptr;             // [d_in]
    float* d_head_g_ = nullptr;           // [H]
    float* d_wl_bias_ = nullptr;          // [H, d_z]
    float* d_bwd_scale_ = nullptr;        // [H + 1]: w_l w_c sigmoid(gamma_raw_h) | w_l
    float k_scale_ = 0.f;
    bool dirty_ = true;
    std::mutex upload_mu_;
    // host-path pipeline (host_path.cpp: pinned / device slots, copy + compute streams), guarded
    // by host_mu_: the host entry points release the GIL and may be called concurrently on one layer
    std::mutex host_mu_;
    struct HostPipe;
    HostPipe* pipe_ = nullptr;
    HostPipe& host_pipe();
    void release_host_pipe();
    template <class T, class O>
    void host_forward(std::int64_t B, std::int64_t L, const T* s, const T* z1, const T* z2, const T* rot,
                      const T* trans, const std::uint8_t* mask, O* out, bool dense);
    template <class T, class O>
    void host_grad(std::int64_t B, std::int64_t L, const T* s, const T* z1, const T* z2, const T* rot,
                   const T* trans, const std::uint8_t* mask, const T* dout, O* out, O* ds, O* dz1, O* dz2,
                   O* drot, O* dtrans, O* dweights);
    // timing
    bool timing_ = false;
    static constexpr int kStages = 6;
    cudaEvent_t ev_[kStages + 1] = {};
public:
    // backward stages: dout, dfeat, dw_out, prep, attn_kv, attn_q, unpack, recenter, ds, dW, scatter
    static constexpr int kBwdStages = 11;
    std::vector<float> bwd_stage_times() const;
private:
    cudaEvent_t evb_[kBwdStages + 1] = {};
    bool bwd_timed_once_ = false;
    bool timed_once_ = false;
};

}  // namespace fipa_b200
