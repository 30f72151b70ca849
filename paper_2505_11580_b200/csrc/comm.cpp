// Multi-GPU query-row sharding over NCCL (one process per GPU).  SURVEY.md §8(e): a long single
// structure is split into G contiguous residue blocks; every rank projects and packs its own
// rows, the packed key/value rows (k_hat, v_hat: bf16 [B*H][L_local][pad]) are all-gathered over
// NVLink into [G][B*H][L_local][pad] -- exactly the sharded layout the attention kernel's 5-D
// TMA maps read (attn_fwd_2sm.cu) -- and every rank attends its local queries to all keys.  The
// translation centroid used for recentring is all-reduced first (4 floats per sample).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2: the copy torch already loaded, or the
// system one), so the library itself has no link-time NCCL dependency and still loads on hosts
// without it; nccl.h supplies only the types.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "kernels.hpp"
#include "layer.hpp"

namespace fipa_b200 {

namespace {

struct NcclApi {
    void* handle = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                  cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    // point-to-point (optional: the overlapped gather falls back to one all-gather without them)
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            api.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (api.handle) break;
        }
        if (!api.handle) {
            err = "NCCL not found (dlopen libnccl.so.2 failed)";
            return;
        }
        auto sym = [](const char* n) { return dlsym(api.handle, n); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
        api.ReduceScatter = reinterpret_cast<decltype(api.ReduceScatter)>(sym("ncclReduceScatter"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.AllGather || !api.AllReduce ||
            !api.ReduceScatter) {
            err = "NCCL library lacks required symbols";
            api.handle = nullptr;
        }
    });
    if (!api.handle) throw CommError(err);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const auto& api = nccl();
        throw CommError(std::string(what) + ": " + (api.GetErrorString ? api.GetErrorString(r) : "NCCL error"));
    }
}

}  // namespace

std::array<std::uint8_t, 128> Comm::unique_id() {
    static_assert(sizeof(ncclUniqueId) == 128, "unexpected ncclUniqueId size");
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::array<std::uint8_t, 128> out{};
    std::memcpy(out.data(), &id, 128);
    return out;
}

Comm::Comm(int world, int rank, const std::uint8_t* id, int device) : world_(world), rank_(rank), device_(device) {
    if (world < 1 || rank < 0 || rank >= world) throw ValueError("invalid world/rank");
    if (id == nullptr) throw ValueError("null NCCL unique id");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    ncclComm_t c = nullptr;
    nccl_check(nccl().CommInitRank(&c, world, uid, rank), "ncclCommInitRank");
    comm_ = c;
}

Comm::~Comm() {
    if (comm_) nccl().CommDestroy(static_cast<ncclComm_t>(comm_));
}

void Comm::all_reduce_sum_f32(float* buf, std::size_t n, cudaStream_t stream) {
    nccl_check(nccl().AllReduce(buf, buf, n, ncclFloat32, ncclSum, static_cast<ncclComm_t>(comm_), stream),
               "ncclAllReduce");
}

void Comm::all_gather_bytes(const void* send, void* recv, std::size_t bytes, cudaStream_t stream) {
    nccl_check(nccl().AllGather(send, recv, bytes, ncclUint8, static_cast<ncclComm_t>(comm_), stream),
               "ncclAllGather");
}

bool Comm::has_p2p() const {
    const auto& a = nccl();
    return a.Send && a.Recv && a.GroupStart && a.GroupEnd;
}

void Comm::all_gather_pieces(const void* send, void* recv, std::size_t piece, int pieces, std::size_t stride,
                             std::size_t rank_stride, cudaStream_t stream) {
    const auto& a = nccl();
    const char* src = static_cast<const char*>(send);
    char* dst = static_cast<char*>(recv);
    // own blocks: device copies; peers: one grouped send / recv per block and peer
    for (int k = 0; k < pieces; ++k)
        cuda_check(cudaMemcpyAsync(dst + std::size_t(rank_) * rank_stride + k * stride, src + k * stride, piece,
                                   cudaMemcpyDeviceToDevice, stream),
                   "gather copy");
    if (world_ == 1) return;
    if (!has_p2p()) throw CommError("NCCL point-to-point symbols unavailable");
    auto comm = static_cast<ncclComm_t>(comm_);
    nccl_check(a.GroupStart(), "ncclGroupStart");
    for (int g = 0; g < world_; ++g) {
        if (g == rank_) continue;
        for (int k = 0; k < pieces; ++k) {
            nccl_check(a.Send(src + k * stride, piece, ncclUint8, g, comm, stream), "ncclSend");
            nccl_check(a.Recv(dst + std::size_t(g) * rank_stride + k * stride, piece, ncclUint8, g, comm, stream),
                       "ncclRecv");
        }
    }
    nccl_check(a.GroupEnd(), "ncclGroupEnd");
}

void Comm::reduce_scatter_sum_f32(const float* send, float* recv, std::size_t n, cudaStream_t stream) {
    nccl_check(nccl().ReduceScatter(send, recv, n, ncclFloat32, ncclSum, static_cast<ncclComm_t>(comm_), stream),
               "ncclReduceScatter");
}

// ---------------------------------------------------------------- sharded forward
FlashIpaLayer::ShardedWorkspace FlashIpaLayer::carve_sharded(void* base, std::int64_t B, std::int64_t L,
                                                            int groups, bool train) const {
    ShardedWorkspace w;
    w.local = carve(base, B, L, train);
    std::size_t off = (w.local.bytes + 255) / 256 * 256;
    auto take = [&](std::size_t bytes) {
        char* p = reinterpret_cast<char*>(reinterpret_cast<std::uintptr_t>(base) + off);
        off += (bytes + 255) / 256 * 256;
        return p;
    };
    const std::size_t BHL = std::size_t(B) * L * dims_.heads;
    w.kv_bytes = BHL * dims_.dqk_pad * 2;
    w.v_bytes = BHL * dims_.dv_pad * 2;
    w.k_all = take(w.kv_bytes * groups);
    w.v_all = take(w.v_bytes * groups);
    w.sums = reinterpret_cast<float*>(take(std::size_t(B) * 4 * 4));
    if (train) {
        const std::size_t part = std::size_t(groups) * BHL * acc_ld() * 4;
        w.dk_part = reinterpret_cast<float*>(take(part));
        w.dv_part = reinterpret_cast<float*>(take(part));
        w.dt_sums = reinterpret_cast<float*>(take(std::size_t(B) * 4 * 4));
    }
    w.bytes = off;
    return w;
}

std::size_t FlashIpaLayer::sharded_train_workspace_size(std::int64_t B, std::int64_t L, int groups) const {
    return carve_sharded(nullptr, B, L, groups, true).bytes;
}

// Stage 2 of the sharded forward with the K/V all-gather overlapped: the packed rows go out in head
// chunks on a side stream (grouped send / recv straight into the [G][B*H][L][pad] gathered layout)
// and the attention of chunk c starts as soon as its keys have landed, while chunks c+1.. are on
// the wire; the output projection follows the last chunk.  One chunk (or no point-to-point NCCL,
// or a non-pair attention kernel): one all-gather of each tensor, then the attention.
void FlashIpaLayer::gather_and_attend(Comm& comm, std::int64_t B, std::int64_t L, const float* s, const float* z1,
                                      const float* z2, const float* rot, const float* trans,
                                      const std::uint8_t* mask, float* out, void* workspace,
                                      const ShardedWorkspace& ws, bool train, cudaStream_t stream) {
    const int G = comm.world(), H = dims_.heads;
    // automatic: nothing to overlap at world 1; otherwise as many chunks (4 or 2) as keep each
    // chunk's attention launch >= ~6 waves of CTAs (4 chunks of B=8 L=1024 cost 50% in quantisation)
    int chunks = tuning_.shard_chunks;
    if (chunks == 0) {
        chunks = 1;
        const std::int64_t ctas = B * ((L + 127) / 128);  // per head
        for (int c : {4, 2})
            if (G > 1 && H % c == 0 && ctas * (H / c) >= 6 * device_sm_count()) {
                chunks = c;
                break;
            }
    }
    chunks = std::min(chunks, 7);  // comm_ev_[0..6] per chunk
    const bool pair = train || attention_impl_for_sharding();
    if (H % chunks != 0 || !pair || (G > 1 && !comm.has_p2p())) chunks = 1;
    ShardStage st;
    st.k_all = ws.k_all;
    st.v_all = ws.v_all;
    st.groups = G;
    if (chunks == 1) {
        comm.all_gather_bytes(ws.local.khat, ws.k_all, ws.kv_bytes, stream);
        comm.all_gather_bytes(ws.local.vhat, ws.v_all, ws.v_bytes, stream);
        st.stage = 2;
        forward(B, L, s, z1, z2, rot, trans, mask, out, workspace, ws.local.bytes, stream, train, &st);
        return;
    }
    ensure_side_streams();
    for (auto& e : comm_ev_)
        if (!e) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    cudaStream_t cs = side_streams_[0];
    const int hc = H / chunks;
    const std::size_t krow = std::size_t(dims_.dqk_pad) * 2, vrow = std::size_t(dims_.dv_pad) * 2;
    cuda_check(cudaEventRecord(comm_ev_[7], stream), "event record");  // packed rows complete
    cuda_check(cudaStreamWaitEvent(cs, comm_ev_[7], 0), "stream wait");
    for (int c = 0; c < chunks; ++c) {
        const std::size_t ko = std::size_t(c) * hc * L * krow, vo = std::size_t(c) * hc * L * vrow;
        comm.all_gather_pieces(static_cast<const char*>(ws.local.khat) + ko, static_cast<char*>(ws.k_all) + ko,
                               hc * L * krow, int(B), std::size_t(H) * L * krow, ws.kv_bytes, cs);
        comm.all_gather_pieces(static_cast<const char*>(ws.local.vhat) + vo, static_cast<char*>(ws.v_all) + vo,
                               hc * L * vrow, int(B), std::size_t(H) * L * vrow, ws.v_bytes, cs);
        cuda_check(cudaEventRecord(comm_ev_[c], cs), "event record");
    }
    st.stage = 2;
    for (int c = 0; c < chunks; ++c) {
        cuda_check(cudaStreamWaitEvent(stream, comm_ev_[c], 0), "stream wait");
        st.h0 = c * hc;
        st.hc = hc;
        forward(B, L, s, z1, z2, rot, trans, mask, out, workspace, ws.local.bytes, stream, train, &st);
    }
    st.stage = 3;
    st.hc = 0;
    forward(B, L, s, z1, z2, rot, trans, mask, out, workspace, ws.local.bytes, stream, train, &st);
}

// Sharded training step.  Forward as forward_sharded with the training buffers (fp32 O_hat, lse)
// kept; the gathered k_hat / v_hat stay in the workspace for the backward.
void FlashIpaLayer::forward_train_sharded(Comm& comm, std::int64_t B, std::int64_t L, const float* s,
                                          const float* z1, const float* z2, const float* rot,
                                          const float* trans, const std::uint8_t* mask, float* out,
                                          void* workspace, std::size_t workspace_bytes, cudaStream_t stream) {
    const int G = comm.world();
    if (G > 1 && L % 256 != 0) throw ValueError("sharded training needs L_local % 256 == 0");
    const ShardedWorkspace ws = carve_sharded(workspace, B, L, G, true);
    if (workspace == nullptr || workspace_bytes < ws.bytes)
        throw ValueError("sharded train workspace too small: need " + std::to_string(ws.bytes) + " bytes");
    launch_centroid_sums(trans, mask, ws.sums, int(B), int(L), stream);
    comm.all_reduce_sum_f32(ws.sums, std::size_t(B) * 4, stream);
    ShardStage st;
    st.stage = 1;
    st.sums = ws.sums;
    forward(B, L, s, z1, z2, rot, trans, mask, out, workspace, ws.local.bytes, stream, true, &st);
    gather_and_attend(comm, B, L, s, z1, z2, rot, trans, mask, out, workspace, ws, true, stream);
}

// Backward of the sharded step: the three BwdShard stages joined by a reduce-scatter of the partial
// key gradients (fp32, 2 x G x B L H 448 floats per rank), an all-reduce of the translation-gradient
// sums (4 floats per sample) and an all-reduce of the weight gradients.
void FlashIpaLayer::backward_sharded(Comm& comm, std::int64_t B, std::int64_t L, const float* s,
                                     const float* z1, const float* z2, const float* rot, const float* trans,
                                     const std::uint8_t* mask, const float* dout, float* ds, float* dz1,
                                     float* dz2, float* drot, float* dtrans, float* dweights, void* workspace,
                                     std::size_t workspace_bytes, cudaStream_t stream) {
    const int G = comm.world();
    const ShardedWorkspace ws = carve_sharded(workspace, B, L, G, true);
    if (workspace == nullptr || workspace_bytes < ws.bytes)
        throw ValueError("sharded train workspace too small: need " + std::to_string(ws.bytes) + " bytes");
    BwdShard sh;
    sh.groups = G;
    sh.k_all = ws.k_all;
    sh.v_all = ws.v_all;
    sh.dk_part = ws.dk_part;
    sh.dv_part = ws.dv_part;
    sh.stage = 1;
    // the reduce-scatter of the partial key gradients runs on a side stream as soon as the dK/dV
    // kernel is done, overlapping the dQ kernel (which neither reads nor writes them)
    ensure_side_streams();
    for (auto& e : comm_ev_)
        if (!e) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    cudaStream_t cs = side_streams_[0];
    sh.kv_done = comm_ev_[5];
    backward(B, L, s, z1, z2, rot, trans, mask, dout, ds, dz1, dz2, drot, dtrans, dweights, workspace,
             ws.local.bytes, stream, &sh);
    sh.kv_done = nullptr;
    const std::size_t n = std::size_t(B) * L * dims_.heads * acc_ld();
    cuda_check(cudaStreamWaitEvent(cs, comm_ev_[5], 0), "stream wait");
    comm.reduce_scatter_sum_f32(ws.dk_part, ws.local.dk_acc, n, cs);
    comm.reduce_scatter_sum_f32(ws.dv_part, ws.local.dv_acc, n, cs);
    cuda_check(cudaEventRecord(comm_ev_[6], cs), "event record");
    cuda_check(cudaStreamWaitEvent(stream, comm_ev_[6], 0), "stream wait");
    sh.stage = 2;
    sh.dk_own = ws.local.dk_acc;
    sh.dv_own = ws.local.dv_acc;
    sh.dt_sums = ws.dt_sums;
    backward(B, L, s, z1, z2, rot, trans, mask, dout, ds, dz1, dz2, drot, dtrans, dweights, workspace,
             ws.local.bytes, stream, &sh);
    comm.all_reduce_sum_f32(ws.dt_sums, std::size_t(B) * 4, stream);
    sh.stage = 3;
    backward(B, L, s, z1, z2, rot, trans, mask, dout, ds, dz1, dz2, drot, dtrans, dweights, workspace,
             ws.local.bytes, stream, &sh);
    comm.all_reduce_sum_f32(dweights, num_weights(), stream);
}

std::size_t FlashIpaLayer::sharded_workspace_size(std::int64_t B, std::int64_t L, int groups) const {
    return carve_sharded(nullptr, B, L, groups).bytes;
}

void FlashIpaLayer::forward_sharded(Comm& comm, std::int64_t B, std::int64_t L, const float* s, const float* z1,
                                    const float* z2, const float* rot, const float* trans,
                                    const std::uint8_t* mask, float* out, void* workspace,
                                    std::size_t workspace_bytes, cudaStream_t stream) {
    const int G = comm.world();
    if (G > 1 && L % 64 != 0) throw ValueError("query-row sharding needs L_local % 64 == 0");
    const ShardedWorkspace ws = carve_sharded(workspace, B, L, G);
    if (workspace == nullptr || workspace_bytes < ws.bytes)
        throw ValueError("sharded workspace too small: need " + std::to_string(ws.bytes) + " bytes");
    launch_centroid_sums(trans, mask, ws.sums, int(B), int(L), stream);
    comm.all_reduce_sum_f32(ws.sums, std::size_t(B) * 4, stream);
    ShardStage st;
    st.stage = 1;
    st.sums = ws.sums;
    forward(B, L, s, z1, z2, rot, trans, mask, out, workspace, ws.local.bytes, stream, false, &st);
    gather_and_attend(comm, B, L, s, z1, z2, rot, trans, mask, out, workspace, ws, false, stream);
}

}  // namespace fipa_b200
