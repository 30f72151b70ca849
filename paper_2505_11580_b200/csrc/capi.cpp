// extern "C" boundary (include/fipa_b200.h) over the host C++ layer.  Exceptions never cross
// the ABI: they become status codes + a thread-local message (reference error taxonomy,
// proj/include/fipa/error.hpp:10-28).
#include "../../include/fipa_b200.h"

#include <exception>
#include <memory>
#include <vector>
#include <new>
#include <string>

#include "layer.hpp"
#include "producer.hpp"
#include "trunk.hpp"

struct fipa_layer {
    std::unique_ptr<fipa_b200::FlashIpaLayer> owned;  // null for a trunk's borrowed layer view
    fipa_b200::FlashIpaLayer* impl;
    explicit fipa_layer(const fipa_b200::Config& c)
        : owned(std::make_unique<fipa_b200::FlashIpaLayer>(c)), impl(owned.get()) {}
    explicit fipa_layer(fipa_b200::FlashIpaLayer* borrowed) : impl(borrowed) {}
};

struct fipa_trunk {
    fipa_b200::Trunk impl;
    std::vector<std::unique_ptr<fipa_layer>> views;
    fipa_trunk(const fipa_b200::Config& c, int n, uint64_t seed) : impl(c, n, seed) {
        for (int l = 0; l < n; ++l) views.push_back(std::make_unique<fipa_layer>(&impl.layer(l)));
    }
};

struct fipa_comm {
    fipa_b200::Comm impl;
    fipa_comm(int world, int rank, const uint8_t* id, int device) : impl(world, rank, id, device) {}
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return FIPA_OK;
    } catch (const fipa_b200::ValueError& e) {
        g_err = e.what();
        return FIPA_ERR_VALUE;
    } catch (const fipa_b200::NumericError& e) {
        g_err = e.what();
        return FIPA_ERR_NUMERIC;
    } catch (const fipa_b200::IoError& e) {
        g_err = e.what();
        return FIPA_ERR_IO;
    } catch (const fipa_b200::CudaError& e) {
        g_err = e.what();
        return FIPA_ERR_CUDA;
    } catch (const fipa_b200::CommError& e) {
        g_err = e.what();
        return FIPA_ERR_COMM;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return FIPA_ERR_VALUE;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return FIPA_ERR_OTHER;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FIPA_ERR_OTHER;
    }
}

fipa_b200::Config to_cfg(const fipa_config* c) {
    if (c == nullptr) throw fipa_b200::ValueError("null fipa_config");
    fipa_b200::Config cfg;
    cfg.d_in = c->d_in;
    cfg.d_z = c->d_z;
    cfg.heads = c->heads;
    cfg.c = c->c;
    cfg.n_query = c->n_query;
    cfg.n_value = c->n_value;
    cfg.rank = c->rank;
    if (c->precision == FIPA_PREC_BF16) {
        cfg.precision = fipa_b200::Precision::bf16;
    } else if (c->precision == FIPA_PREC_F32) {
        cfg.precision = fipa_b200::Precision::f32;
        cfg.weights_f32 = true;
    } else if (c->precision == FIPA_PREC_F64) {
        cfg.precision = fipa_b200::Precision::f32;  // no GPU f64 path: fp32 compute, f64 masters
    } else {
        throw fipa_b200::ValueError("unknown precision code " + std::to_string(c->precision));
    }
    cfg.enforce_head_cap = c->enforce_head_cap != 0;
    return cfg;
}

fipa_b200::FlashIpaLayer& L(fipa_layer* l) {
    if (l == nullptr) throw fipa_b200::ValueError("null fipa_layer");
    return *l->impl;
}
const fipa_b200::FlashIpaLayer& L(const fipa_layer* l) {
    if (l == nullptr) throw fipa_b200::ValueError("null fipa_layer");
    return *l->impl;
}

}  // namespace

extern "C" {

const char* fipa_last_error(void) { return g_err.c_str(); }

int fipa_config_validate(const fipa_config* cfg) {
    return guarded([&] { to_cfg(cfg).validate(); });
}

uint64_t fipa_config_qk_width(const fipa_config* cfg) {
    return cfg ? cfg->c + 5 * cfg->n_query + cfg->rank * cfg->d_z : 0;
}

uint64_t fipa_config_v_width(const fipa_config* cfg) {
    return cfg ? cfg->c + 3 * cfg->n_value + cfg->rank * cfg->d_z : 0;
}

int fipa_layer_create(const fipa_config* cfg, fipa_layer** out) {
    return guarded([&] {
        if (out == nullptr) throw fipa_b200::ValueError("null output handle");
        *out = nullptr;
        *out = new fipa_layer(to_cfg(cfg));
    });
}

void fipa_layer_destroy(fipa_layer* layer) {
    if (layer != nullptr && layer->owned) delete layer;  // trunk layer views are owned by the trunk
}

int fipa_layer_init_weights(fipa_layer* layer, uint64_t seed) {
    return guarded([&] { L(layer).init_weights(seed); });
}

int fipa_layer_set_weights(fipa_layer* layer, const fipa_host_weights* w) {
    return guarded([&] {
        auto& impl = L(layer);
        if (w == nullptr) throw fipa_b200::ValueError("null weights");
        const auto shapes = fipa_b200::weight_shapes(impl.config());
        const double* src[10] = {w->w_q,  w->w_k,      w->w_v,  w->w_qp, w->w_kp,
                                 w->w_vp, w->w_bias, w->gamma_raw, w->w_out, w->b_out};
        fipa_b200::HostWeights hw;
        for (int i = 0; i < 10; ++i) {
            if (src[i] == nullptr) throw fipa_b200::ValueError("null weights tensor");
            std::size_t n = 1;
            for (auto d : shapes[i]) n *= d;
            hw.slots[i]->assign(src[i], src[i] + n);
        }
        hw.w_l = w->w_l;
        hw.w_c = w->w_c;
        hw.stored_f32 = impl.config().weights_f32;
        impl.set_weights(hw);
    });
}

int fipa_layer_get_weights(const fipa_layer* layer, double* const* w, double* scal) {
    return guarded([&] {
        const auto& impl = L(layer);
        if (w == nullptr || scal == nullptr) throw fipa_b200::ValueError("null output buffers");
        const auto& hw = impl.weights();
        for (int i = 0; i < 10; ++i) {
            if (w[i] == nullptr) throw fipa_b200::ValueError("null weights buffer");
            std::copy(hw.slots[i]->begin(), hw.slots[i]->end(), w[i]);
        }
        scal[0] = hw.w_l;
        scal[1] = hw.w_c;
    });
}

int fipa_layer_save_weights(const fipa_layer* layer, const char* path) {
    return guarded([&] {
        if (path == nullptr) throw fipa_b200::ValueError("null path");
        L(layer).save(path);
    });
}

int fipa_layer_load_weights(fipa_layer* layer, const char* path) {
    return guarded([&] {
        if (path == nullptr) throw fipa_b200::ValueError("null path");
        L(layer).load(path);
    });
}

size_t fipa_layer_workspace_size(const fipa_layer* layer, int64_t B, int64_t L_) {
    if (layer == nullptr || B < 1 || L_ < 1) return 0;
    return layer->impl->workspace_size(B, L_);
}

int fipa_layer_forward(fipa_layer* layer, int64_t B, int64_t L_, const float* s, const float* z1,
                       const float* z2, const float* rot, const float* trans, const uint8_t* mask,
                       float* out, void* workspace, size_t workspace_bytes, void* stream) {
    return guarded([&] {
        L(layer).forward(B, L_, s, z1, z2, rot, trans, mask, out, workspace, workspace_bytes,
                         static_cast<cudaStream_t>(stream));
    });
}

int fipa_fully_masked(int64_t B, int64_t L_, const uint8_t* mask, uint8_t* flags, void* stream) {
    return guarded([&] {
        if (B < 1 || L_ < 1) throw fipa_b200::ValueError("empty frame set");
        if (flags == nullptr) throw fipa_b200::ValueError("null flags buffer");
        fipa_b200::launch_fully_masked(mask, flags, int(B), int(L_), static_cast<cudaStream_t>(stream));
        fipa_b200::cuda_check(cudaGetLastError(), "fully_masked launch");
    });
}

int fipa_fully_masked_host(int64_t B, int64_t L_, const uint8_t* mask, uint8_t* flags) {
    return guarded([&] {
        if (B < 1 || L_ < 1) throw fipa_b200::ValueError("empty frame set");
        if (flags == nullptr) throw fipa_b200::ValueError("null flags buffer");
        const size_t n = size_t(B) * size_t(L_);
        uint8_t* d = nullptr;
        fipa_b200::cuda_check(cudaMalloc(&d, 2 * n), "cudaMalloc");
        struct Free {
            uint8_t* p;
            ~Free() { cudaFree(p); }
        } guard{d};
        if (mask) fipa_b200::cuda_check(cudaMemcpy(d, mask, n, cudaMemcpyHostToDevice), "H2D");
        fipa_b200::launch_fully_masked(mask ? d : nullptr, d + n, int(B), int(L_), nullptr);
        fipa_b200::cuda_check(cudaMemcpy(flags, d + n, n, cudaMemcpyDeviceToHost), "D2H");
    });
}

int fipa_layer_forward_host(fipa_layer* layer, int64_t B, int64_t L_, const double* s,
                            const double* z1, const double* z2, const double* rot,
                            const double* trans, const uint8_t* mask, double* out) {
    return guarded([&] {
        if (!s || !z1 || !z2 || !rot || !trans || !out) throw fipa_b200::ValueError("null buffer");
        L(layer).forward_host(B, L_, s, z1, z2, rot, trans, mask, out);
    });
}

size_t fipa_layer_reference_workspace_size(const fipa_layer* layer, int64_t B, int64_t L_) {
    if (layer == nullptr || B < 1 || L_ < 1) return 0;
    return layer->impl->reference_workspace_size(B, L_);
}

int fipa_layer_reference_forward(fipa_layer* layer, int64_t B, int64_t L_, const float* s, const float* z1,
                                 const float* z2, const float* rot, const float* trans, const uint8_t* mask,
                                 float* out, void* workspace, size_t workspace_bytes, void* stream) {
    return guarded([&] {
        L(layer).reference_forward(B, L_, s, z1, z2, rot, trans, mask, out, workspace, workspace_bytes,
                                   static_cast<cudaStream_t>(stream));
    });
}

int fipa_layer_reference_host(fipa_layer* layer, int64_t B, int64_t L_, const double* s, const double* z1,
                              const double* z2, const double* rot, const double* trans, const uint8_t* mask,
                              double* out) {
    return guarded([&] {
        if (!s || !z1 || !z2 || !rot || !trans || !out) throw fipa_b200::ValueError("null buffer");
        L(layer).reference_host(B, L_, s, z1, z2, rot, trans, mask, out);
    });
}

size_t fipa_naive_attention_workspace_size(int64_t H, int64_t L_) {
    if (H < 1 || L_ < 1) return 0;
    return size_t(H) * size_t(L_) * size_t(L_) * sizeof(float);
}

namespace {
static void check_attention_dims(int64_t H, int64_t L_, int64_t dqk, int64_t dv) {
    if (H < 1 || dqk < 1 || dv < 1) throw fipa_b200::ValueError("attention operands need positive sizes");
    if (L_ < 1) throw fipa_b200::ValueError("attention operands need L >= 1");
    if (H > 65535 || L_ > (int64_t(1) << 31) / 64 || dqk > (1 << 20) || dv > (1 << 20))
        throw fipa_b200::ValueError("attention operands too large");
}
}  // namespace

int fipa_naive_attention(int64_t H, int64_t L_, int64_t dqk, int64_t dv, const float* q, const float* k,
                         const float* v, const uint8_t* mask, float* out, void* workspace, size_t workspace_bytes,
                         void* stream) {
    return guarded([&] {
        check_attention_dims(H, L_, dqk, dv);
        if (!q || !k || !v || !out) throw fipa_b200::ValueError("null buffer");
        if (!workspace || workspace_bytes < fipa_naive_attention_workspace_size(H, L_))
            throw fipa_b200::ValueError("naive attention workspace too small");
        fipa_b200::launch_naive_attention_f32(int(H), int(L_), int(dqk), int(dv), q, k, v, mask,
                                              static_cast<float*>(workspace), out, static_cast<cudaStream_t>(stream));
        fipa_b200::cuda_check(cudaGetLastError(), "kernel launch");
    });
}

int fipa_flash_attention(int64_t H, int64_t L_, int64_t dqk, int64_t dv, const float* q, const float* k,
                         const float* v, const uint8_t* mask, float* out, void* stream) {
    return guarded([&] {
        check_attention_dims(H, L_, dqk, dv);
        if (!q || !k || !v || !out) throw fipa_b200::ValueError("null buffer");
        fipa_b200::launch_flash_attention_f32(int(H), int(L_), int(dqk), int(dv), q, k, v, mask, out,
                                              static_cast<cudaStream_t>(stream));
        fipa_b200::cuda_check(cudaGetLastError(), "kernel launch");
    });
}

int fipa_attention_host(int64_t H, int64_t L_, int64_t dqk, int64_t dv, const double* q, const double* k,
                        const double* v, const uint8_t* mask, double* out, int naive, int device) {
    return guarded([&] {
        check_attention_dims(H, L_, dqk, dv);
        if (!q || !k || !v || !out) throw fipa_b200::ValueError("null buffer");
        using fipa_b200::cuda_check;
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        const size_t nq = size_t(H) * L_ * dqk, nv = size_t(H) * L_ * dv;
        const size_t ws = naive ? fipa_naive_attention_workspace_size(H, L_) : 0;
        std::vector<float> h(2 * nq + 2 * nv);
        for (size_t i = 0; i < nq; ++i) h[i] = float(q[i]);
        for (size_t i = 0; i < nq; ++i) h[nq + i] = float(k[i]);
        for (size_t i = 0; i < nv; ++i) h[2 * nq + i] = float(v[i]);
        char* d = nullptr;
        const size_t bytes = h.size() * 4 + size_t(L_) + ws + 256;
        cuda_check(cudaMalloc(&d, bytes), "cudaMalloc");
        std::unique_ptr<char, void (*)(char*)> guard(d, [](char* p) { cudaFree(p); });
        float* dq = reinterpret_cast<float*>(d);
        float* dk = dq + nq;
        float* dvv = dk + nq;
        float* dout = dvv + nv;
        uint8_t* dm = reinterpret_cast<uint8_t*>(dout + nv);
        void* dws = d + ((h.size() * 4 + size_t(L_) + 255) / 256 * 256);
        cuda_check(cudaMemcpy(d, h.data(), (2 * nq + nv) * 4, cudaMemcpyHostToDevice), "H2D");
        if (mask) cuda_check(cudaMemcpy(dm, mask, size_t(L_), cudaMemcpyHostToDevice), "H2D");
        if (naive) {
            fipa_b200::launch_naive_attention_f32(int(H), int(L_), int(dqk), int(dv), dq, dk, dvv, mask ? dm : nullptr,
                                                  static_cast<float*>(dws), dout, nullptr);
        } else {
            fipa_b200::launch_flash_attention_f32(int(H), int(L_), int(dqk), int(dv), dq, dk, dvv, mask ? dm : nullptr,
                                                  dout, nullptr);
        }
        cuda_check(cudaGetLastError(), "kernel launch");
        cuda_check(cudaMemcpy(h.data(), dout, nv * 4, cudaMemcpyDeviceToHost), "D2H");
        for (size_t i = 0; i < nv; ++i) out[i] = double(h[i]);
    });
}

int fipa_layer_workspace_layout(const fipa_layer* layer, int64_t B, int64_t L_, int64_t* offsets,
                                int64_t* dims) {
    if (layer == nullptr || offsets == nullptr || B < 1 || L_ < 1) return 0;
    const auto w = layer->impl->carve(nullptr, B, L_);
    // carve(nullptr) yields null-based pointers: offsets are the pointer values themselves.
    auto off = [](const void* p, bool present) -> int64_t {
        return present ? static_cast<int64_t>(reinterpret_cast<uintptr_t>(p)) : -1;
    };
    const bool bf16 = layer->impl->config().precision == fipa_b200::Precision::bf16;
    offsets[0] = off(w.trans_c, true);
    offsets[1] = off(w.s_bf16, bf16);
    offsets[2] = off(w.proj, true);
    offsets[3] = off(w.qhat, true);
    offsets[4] = off(w.khat, true);
    offsets[5] = off(w.vhat, true);
    offsets[6] = off(w.colbias, true);
    offsets[7] = off(w.lse, true);
    offsets[8] = off(w.feat, true);
    if (dims != nullptr) {
        const auto& d = layer->impl->dims();
        dims[0] = d.n_proj;
        dims[1] = d.dqk_pad;
        dims[2] = d.dv_pad;
        dims[3] = d.feat;
    }
    return 9;
}

int fipa_layer_forward_launches(const fipa_layer* layer) {
    return layer ? layer->impl->launches_per_forward() : 0;
}

int fipa_layer_step_launches(const fipa_layer* layer, int64_t B, int64_t L_, int train) {
    return layer && B >= 1 && L_ >= 1 ? layer->impl->step_launches(B, L_, train != 0) : 0;
}

int fipa_layer_get_tuning(const fipa_layer* layer, fipa_tuning* out) {
    return guarded([&] {
        if (layer == nullptr || out == nullptr) throw fipa_b200::ValueError("null layer or tuning");
        const auto& t = layer->impl->tuning();
        out->attn_impl = static_cast<int32_t>(t.attn);
        out->fused_pack = t.fused_pack ? 1 : 0;
        out->bwd_ds = t.bwd_ds;
        out->f32_tc = t.f32_tc ? 1 : 0;
        out->bwd_slice = t.bwd_ring[4];
        out->graphs = t.graphs ? 1 : 0;
        out->micro = t.micro;
        out->shard_chunks = t.shard_chunks;
        out->ds_cap_mb = t.ds_cap_mb;
        for (int i = 0; i < 4; ++i) {
            out->bwd_ring[i] = t.bwd_ring[i];
            out->pass_ring[i] = t.pass_ring[i];
        }
    });
}

int fipa_layer_set_tuning(fipa_layer* layer, const fipa_tuning* in) {
    return guarded([&] {
        if (layer == nullptr || in == nullptr) throw fipa_b200::ValueError("null layer or tuning");
        if (in->attn_impl < 0 || in->attn_impl > 3) throw fipa_b200::ValueError("tuning: attn_impl must be 0..3");
        if (in->bwd_ds < -1 || in->bwd_ds > 1) throw fipa_b200::ValueError("tuning: bwd_ds must be -1, 0 or 1");
        if (in->micro < 1 || in->micro > 4) throw fipa_b200::ValueError("tuning: micro must be 1..4");
        fipa_b200::Tuning t = L(layer).tuning();  // fields not in fipa_tuning (host_chunk) kept
        t.micro = in->micro;
        if (in->shard_chunks < 0 || in->shard_chunks > 7) throw fipa_b200::ValueError("tuning: shard_chunks must be 0..7");
        t.shard_chunks = in->shard_chunks;
        if (in->ds_cap_mb < 1) throw fipa_b200::ValueError("tuning: ds_cap_mb must be >= 1");
        t.ds_cap_mb = in->ds_cap_mb;
        t.attn = static_cast<fipa_b200::Tuning::Attn>(in->attn_impl);
        t.fused_pack = in->fused_pack != 0;
        t.bwd_ds = in->bwd_ds;
        t.f32_tc = in->f32_tc != 0;
        t.bwd_ring[4] = in->bwd_slice;
        t.graphs = in->graphs != 0;
        for (int i = 0; i < 4; ++i) {
            t.bwd_ring[i] = in->bwd_ring[i];
            t.pass_ring[i] = in->pass_ring[i];
        }
        L(layer).set_tuning(t);
    });
}

int fipa_layer_set_timing(fipa_layer* layer, int enable) {
    return guarded([&] { L(layer).set_timing(enable != 0); });
}

int fipa_layer_stage_times(const fipa_layer* layer, float* ms, int n) {
    if (layer == nullptr || ms == nullptr) return 0;
    const auto t = layer->impl->stage_times();
    int k = 0;
    for (; k < n && k < int(t.size()); ++k) ms[k] = t[k];
    return k;
}

size_t fipa_layer_train_workspace_size(const fipa_layer* layer, int64_t B, int64_t L_) {
    if (layer == nullptr || B < 1 || L_ < 1) return 0;
    return layer->impl->train_workspace_size(B, L_);
}

int fipa_layer_forward_train(fipa_layer* layer, int64_t B, int64_t L_, const float* s, const float* z1,
                             const float* z2, const float* rot, const float* trans, const uint8_t* mask,
                             float* out, void* workspace, size_t workspace_bytes, void* stream) {
    return guarded([&] {
        L(layer).forward(B, L_, s, z1, z2, rot, trans, mask, out, workspace, workspace_bytes,
                         static_cast<cudaStream_t>(stream), true);
    });
}

uint64_t fipa_layer_num_weights(const fipa_layer* layer) { return layer ? layer->impl->num_weights() : 0; }

int fipa_layer_backward(fipa_layer* layer, int64_t B, int64_t L_, const float* s, const float* z1,
                        const float* z2, const float* rot, const float* trans, const uint8_t* mask,
                        const float* dout, float* ds, float* dz1, float* dz2, float* drot, float* dtrans,
                        float* dweights, void* workspace, size_t workspace_bytes, void* stream) {
    return guarded([&] {
        L(layer).backward(B, L_, s, z1, z2, rot, trans, mask, dout, ds, dz1, dz2, drot, dtrans, dweights,
                          workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
    });
}

int fipa_layer_forward_host_f32(fipa_layer* layer, int64_t B, int64_t L_, const float* s, const float* z1,
                                const float* z2, const float* rot, const float* trans, const uint8_t* mask, float* out) {
    return guarded([&] {
        if (!s || !z1 || !z2 || !rot || !trans || !out) throw fipa_b200::ValueError("null input/output pointer");
        L(layer).forward_host_f32(B, L_, s, z1, z2, rot, trans, mask, out);
    });
}

int fipa_layer_grad_host_f32(fipa_layer* layer, int64_t B, int64_t L_, const float* s, const float* z1,
                             const float* z2, const float* rot, const float* trans, const uint8_t* mask,
                             const float* dout, float* out, float* ds, float* dz1, float* dz2, float* drot,
                             float* dtrans, float* dweights) {
    return guarded([&] {
        if (!s || !z1 || !z2 || !rot || !trans || !dout) throw fipa_b200::ValueError("null input pointer");
        L(layer).grad_host_f32(B, L_, s, z1, z2, rot, trans, mask, dout, out, ds, dz1, dz2, drot, dtrans, dweights);
    });
}

int fipa_layer_grad_host(fipa_layer* layer, int64_t B, int64_t L_, const double* s, const double* z1,
                         const double* z2, const double* rot, const double* trans, const uint8_t* mask,
                         const double* dout, double* out, double* ds, double* dz1, double* dz2,
                         double* drot, double* dtrans, double* dweights) {
    return guarded([&] {
        if (!s || !z1 || !z2 || !rot || !trans || !dout) throw fipa_b200::ValueError("null buffer");
        L(layer).grad_host(B, L_, s, z1, z2, rot, trans, mask, dout, out, ds, dz1, dz2, drot, dtrans, dweights);
    });
}

int fipa_layer_train_workspace_layout(const fipa_layer* layer, int64_t B, int64_t L_, int64_t* offsets,
                                      int64_t* dims) {
    if (layer == nullptr || offsets == nullptr || B < 1 || L_ < 1) return 0;
    const auto w = layer->impl->carve(nullptr, B, L_, true);
    auto off = [](const void* p) { return static_cast<int64_t>(reinterpret_cast<uintptr_t>(p)); };
    offsets[0] = off(w.o_hat);
    offsets[1] = off(w.do_hat);
    offsets[2] = off(w.Dvec);
    offsets[3] = off(w.dq_acc);
    offsets[4] = off(w.dk_acc);
    offsets[5] = off(w.dv_acc);
    offsets[6] = off(w.dproj);
    offsets[7] = off(w.dfeat);
    offsets[8] = w.dk16 ? off(w.dk16) : -1;
    offsets[9] = w.dv16 ? off(w.dv16) : -1;
    offsets[10] = w.dq16 ? off(w.dq16) : -1;
    if (dims != nullptr) {
        dims[0] = layer->impl->acc_ld();
        dims[1] = layer->impl->nproj_ld();
        dims[2] = layer->impl->dims().feat_ld;
    }
    return FIPA_TRAIN_LAYOUT_SLOTS;
}

int fipa_layer_bwd_stage_times(const fipa_layer* layer, float* ms, int n) {
    if (layer == nullptr || ms == nullptr) return 0;
    const auto t = layer->impl->bwd_stage_times();
    int k = 0;
    for (; k < n && k < int(t.size()); ++k) ms[k] = t[k];
    return k;
}

int fipa_layer_backward_launches(const fipa_layer* layer) {
    return layer ? layer->impl->launches_per_backward() : 0;
}

int fipa_comm_unique_id(uint8_t out[128]) {
    return guarded([&] {
        if (out == nullptr) throw fipa_b200::ValueError("null output");
        const auto id = fipa_b200::Comm::unique_id();
        std::copy(id.begin(), id.end(), out);
    });
}

int fipa_comm_create(int world, int rank, const uint8_t id[128], int device, fipa_comm** out) {
    return guarded([&] {
        if (out == nullptr) throw fipa_b200::ValueError("null output handle");
        *out = nullptr;
        *out = new fipa_comm(world, rank, id, device);
    });
}

void fipa_comm_destroy(fipa_comm* comm) { delete comm; }

int fipa_comm_all_reduce_f32(fipa_comm* comm, float* buf, size_t n, void* stream) {
    return guarded([&] {
        if (comm == nullptr) throw fipa_b200::ValueError("null fipa_comm");
        if (buf == nullptr && n > 0) throw fipa_b200::ValueError("null buffer");
        if (n > 0) comm->impl.all_reduce_sum_f32(buf, n, static_cast<cudaStream_t>(stream));
    });
}

size_t fipa_layer_sharded_workspace_size(const fipa_layer* layer, int64_t B, int64_t L_, int world) {
    if (layer == nullptr || B < 1 || L_ < 1 || world < 1) return 0;
    return layer->impl->sharded_workspace_size(B, L_, world);
}

int fipa_layer_forward_sharded(fipa_layer* layer, fipa_comm* comm, int64_t B, int64_t L_, const float* s,
                               const float* z1, const float* z2, const float* rot, const float* trans,
                               const uint8_t* mask, float* out, void* workspace, size_t workspace_bytes,
                               void* stream) {
    return guarded([&] {
        if (comm == nullptr) throw fipa_b200::ValueError("null fipa_comm");
        L(layer).forward_sharded(comm->impl, B, L_, s, z1, z2, rot, trans, mask, out, workspace, workspace_bytes,
                                 static_cast<cudaStream_t>(stream));
    });
}

int fipa_layer_shard_centroid_sums(fipa_layer* layer, int64_t B, int64_t L_, const float* trans,
                                   const uint8_t* mask, float* sums, void* stream) {
    return guarded([&] {
        L(layer);
        if (trans == nullptr || sums == nullptr || B < 1 || L_ < 1) throw fipa_b200::ValueError("bad arguments");
        fipa_b200::launch_centroid_sums(trans, mask, sums, int(B), int(L_), static_cast<cudaStream_t>(stream));
        fipa_b200::cuda_check(cudaGetLastError(), "centroid sums");
    });
}

static int shard_pack_impl(fipa_layer* layer, int64_t B, int64_t L_, const float* s, const float* z1,
                           const float* z2, const float* rot, const float* trans, const uint8_t* mask,
                           const float* sums, void* workspace, size_t workspace_bytes, void* stream,
                           void** khat, size_t* k_bytes, void** vhat, size_t* v_bytes, bool train) {
    return guarded([&] {
        auto& impl = L(layer);
        if (sums == nullptr) throw fipa_b200::ValueError("null centroid sums");
        fipa_b200::ShardStage st;
        st.stage = 1;
        st.sums = sums;
        // out is not written in stage 1; any non-null pointer satisfies the argument check
        impl.forward(B, L_, s, z1, z2, rot, trans, mask, reinterpret_cast<float*>(workspace), workspace,
                     workspace_bytes, static_cast<cudaStream_t>(stream), train, &st);
        const auto w = impl.carve(workspace, B, L_);
        const std::size_t BHL = std::size_t(B) * L_ * impl.dims().heads;
        if (khat) *khat = w.khat;
        if (vhat) *vhat = w.vhat;
        if (k_bytes) *k_bytes = BHL * impl.dims().dqk_pad * 2;
        if (v_bytes) *v_bytes = BHL * impl.dims().dv_pad * 2;
    });
}

static int shard_attend_impl(fipa_layer* layer, int64_t B, int64_t L_, int world, const float* s,
                             const float* z1, const float* z2, const float* rot, const float* trans,
                             const uint8_t* mask, const void* khat_all, const void* vhat_all, float* out,
                             void* workspace, size_t workspace_bytes, void* stream, bool train) {
    return guarded([&] {
        if (khat_all == nullptr || vhat_all == nullptr || world < 1) throw fipa_b200::ValueError("bad key shards");
        if (world > 1 && L_ % 64 != 0) throw fipa_b200::ValueError("query-row sharding needs L_local % 64 == 0");
        fipa_b200::ShardStage st;
        st.stage = 2;
        st.k_all = khat_all;
        st.v_all = vhat_all;
        st.groups = world;
        L(layer).forward(B, L_, s, z1, z2, rot, trans, mask, out, workspace, workspace_bytes,
                         static_cast<cudaStream_t>(stream), train, &st);
    });
}

int fipa_layer_shard_pack(fipa_layer* layer, int64_t B, int64_t L_, const float* s, const float* z1,
                          const float* z2, const float* rot, const float* trans, const uint8_t* mask,
                          const float* sums, void* workspace, size_t workspace_bytes, void* stream,
                          void** khat, size_t* k_bytes, void** vhat, size_t* v_bytes) {
    return shard_pack_impl(layer, B, L_, s, z1, z2, rot, trans, mask, sums, workspace, workspace_bytes, stream, khat,
                           k_bytes, vhat, v_bytes, false);
}

int fipa_layer_shard_attend(fipa_layer* layer, int64_t B, int64_t L_, int world, const float* s, const float* z1,
                            const float* z2, const float* rot, const float* trans, const uint8_t* mask,
                            const void* khat_all, const void* vhat_all, float* out, void* workspace,
                            size_t workspace_bytes, void* stream) {
    return shard_attend_impl(layer, B, L_, world, s, z1, z2, rot, trans, mask, khat_all, vhat_all, out, workspace,
                             workspace_bytes, stream, false);
}

int fipa_layer_shard_pack_train(fipa_layer* layer, int64_t B, int64_t L_, const float* s, const float* z1,
                                const float* z2, const float* rot, const float* trans, const uint8_t* mask,
                                const float* sums, void* workspace, size_t workspace_bytes, void* stream,
                                void** khat, size_t* k_bytes, void** vhat, size_t* v_bytes) {
    return shard_pack_impl(layer, B, L_, s, z1, z2, rot, trans, mask, sums, workspace, workspace_bytes, stream, khat,
                           k_bytes, vhat, v_bytes, true);
}

int fipa_layer_shard_attend_train(fipa_layer* layer, int64_t B, int64_t L_, int world, const float* s,
                                  const float* z1, const float* z2, const float* rot, const float* trans,
                                  const uint8_t* mask, const void* khat_all, const void* vhat_all, float* out,
                                  void* workspace, size_t workspace_bytes, void* stream) {
    return shard_attend_impl(layer, B, L_, world, s, z1, z2, rot, trans, mask, khat_all, vhat_all, out, workspace,
                             workspace_bytes, stream, true);
}

int fipa_layer_shard_backward(fipa_layer* layer, int stage, int world, int64_t B, int64_t L_, const float* s,
                              const float* z1, const float* z2, const float* rot, const float* trans,
                              const uint8_t* mask, const float* dout, const void* khat_all, const void* vhat_all,
                              float* dk_part, float* dv_part, const float* dk_own, const float* dv_own,
                              float* dt_sums, float* ds, float* dz1, float* dz2, float* drot, float* dtrans,
                              float* dweights, void* workspace, size_t workspace_bytes, void* stream) {
    return guarded([&] {
        if (world < 1) throw fipa_b200::ValueError("world must be >= 1");
        fipa_b200::BwdShard sh;
        sh.stage = stage;
        sh.groups = world;
        sh.k_all = khat_all;
        sh.v_all = vhat_all;
        sh.dk_part = dk_part;
        sh.dv_part = dv_part;
        sh.dk_own = dk_own;
        sh.dv_own = dv_own;
        sh.dt_sums = dt_sums;
        L(layer).backward(B, L_, s, z1, z2, rot, trans, mask, dout, ds, dz1, dz2, drot, dtrans, dweights, workspace,
                          workspace_bytes, static_cast<cudaStream_t>(stream), &sh);
    });
}

size_t fipa_layer_sharded_train_workspace_size(const fipa_layer* layer, int64_t B, int64_t L_, int world) {
    if (layer == nullptr || B < 1 || L_ < 1 || world < 1) return 0;
    return layer->impl->sharded_train_workspace_size(B, L_, world);
}

int fipa_layer_forward_train_sharded(fipa_layer* layer, fipa_comm* comm, int64_t B, int64_t L_, const float* s,
                                     const float* z1, const float* z2, const float* rot, const float* trans,
                                     const uint8_t* mask, float* out, void* workspace, size_t workspace_bytes,
                                     void* stream) {
    return guarded([&] {
        if (comm == nullptr) throw fipa_b200::ValueError("null fipa_comm");
        L(layer).forward_train_sharded(comm->impl, B, L_, s, z1, z2, rot, trans, mask, out, workspace,
                                       workspace_bytes, static_cast<cudaStream_t>(stream));
    });
}

int fipa_layer_backward_sharded(fipa_layer* layer, fipa_comm* comm, int64_t B, int64_t L_, const float* s,
                                const float* z1, const float* z2, const float* rot, const float* trans,
                                const uint8_t* mask, const float* dout, float* ds, float* dz1, float* dz2, float* drot,
                                float* dtrans, float* dweights, void* workspace, size_t workspace_bytes,
                                void* stream) {
    return guarded([&] {
        if (comm == nullptr) throw fipa_b200::ValueError("null fipa_comm");
        L(layer).backward_sharded(comm->impl, B, L_, s, z1, z2, rot, trans, mask, dout, ds, dz1, dz2, drot, dtrans,
                                  dweights, workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
    });
}

int fipa_trunk_create(const fipa_config* cfg, int n_layers, uint64_t seed, fipa_trunk** out) {
    return guarded([&] {
        if (out == nullptr) throw fipa_b200::ValueError("null output handle");
        *out = nullptr;
        *out = new fipa_trunk(to_cfg(cfg), n_layers, seed);
    });
}

void fipa_trunk_destroy(fipa_trunk* trunk) { delete trunk; }

int fipa_trunk_num_layers(const fipa_trunk* trunk) { return trunk ? trunk->impl.n_layers() : 0; }

fipa_layer* fipa_trunk_layer(fipa_trunk* trunk, int l) {
    if (trunk == nullptr || l < 0 || l >= trunk->impl.n_layers()) return nullptr;
    return trunk->views[l].get();
}

int fipa_trunk_get_backbone(const fipa_trunk* trunk, int l, double* w, double* b) {
    return guarded([&] {
        if (trunk == nullptr || w == nullptr || b == nullptr) throw fipa_b200::ValueError("null argument");
        if (l < 0 || l >= trunk->impl.n_layers()) throw fipa_b200::ValueError("layer index out of range");
        const auto& bb = trunk->impl.backbone(l);
        std::copy(bb.w.begin(), bb.w.end(), w);
        std::copy(bb.b.begin(), bb.b.end(), b);
    });
}

int fipa_trunk_set_backbone(fipa_trunk* trunk, int l, const double* w, const double* b) {
    return guarded([&] {
        if (trunk == nullptr || w == nullptr || b == nullptr) throw fipa_b200::ValueError("null argument");
        trunk->impl.set_backbone(l, w, b);
    });
}

size_t fipa_trunk_workspace_size(const fipa_trunk* trunk, int64_t B, int64_t L_) {
    if (trunk == nullptr || B < 1 || L_ < 1) return 0;
    return trunk->impl.workspace_size(B, L_);
}

int fipa_trunk_forward(fipa_trunk* trunk, int64_t B, int64_t L_, const float* s, const float* z1, const float* z2,
                       const float* rot, const float* trans, const uint8_t* mask, float* s_out, float* rot_out,
                       float* trans_out, void* workspace, size_t workspace_bytes, void* stream) {
    return guarded([&] {
        if (trunk == nullptr) throw fipa_b200::ValueError("null fipa_trunk");
        trunk->impl.forward(B, L_, s, z1, z2, rot, trans, mask, s_out, rot_out, trans_out, workspace,
                            workspace_bytes, static_cast<cudaStream_t>(stream));
    });
}

int fipa_trunk_forward_launches(const fipa_trunk* trunk) { return trunk ? trunk->impl.launches_per_forward() : 0; }
int fipa_trunk_step_launches(const fipa_trunk* trunk, int64_t B, int64_t L) {
    return trunk && B >= 1 && L >= 1 ? trunk->impl.step_launches(B, L) : 0;
}

}  // extern "C"

namespace {
fipa_b200::KnnSpec knn_spec(uint64_t k, uint64_t n_bins, double d_min, double d_max, uint64_t pe_dim) {
    if (k > (1u << 20) || n_bins > (1u << 20) || pe_dim > (1u << 20)) throw fipa_b200::ValueError("invalid distogram spec");
    fipa_b200::KnnSpec s{};
    s.k = int(k);
    s.n_bins = int(n_bins);
    s.pe_dim = int(pe_dim);
    s.d_min = d_min;
    s.d_max = d_max;
    return s;
}
}  // namespace

extern "C" {

int fipa_knn_distogram(int64_t B, int64_t L_, const float* trans, uint64_t k, uint64_t n_bins, double d_min,
                       double d_max, uint64_t pe_dim, float* out, void* stream) {
    return guarded([&] {
        fipa_b200::knn_distogram(B, L_, trans, knn_spec(k, n_bins, d_min, d_max, pe_dim), out,
                                 static_cast<cudaStream_t>(stream));
    });
}

int fipa_knn_distogram_f64(int64_t B, int64_t L_, const double* trans, uint64_t k, uint64_t n_bins, double d_min,
                           double d_max, uint64_t pe_dim, double* out, void* stream) {
    return guarded([&] {
        fipa_b200::knn_distogram(B, L_, trans, knn_spec(k, n_bins, d_min, d_max, pe_dim), out,
                                 static_cast<cudaStream_t>(stream));
    });
}

int fipa_knn_distogram_host(int64_t B, int64_t L_, const double* trans, uint64_t k, uint64_t n_bins, double d_min,
                            double d_max, uint64_t pe_dim, double* out) {
    return guarded([&] {
        fipa_b200::knn_distogram_host(B, L_, trans, knn_spec(k, n_bins, d_min, d_max, pe_dim), out);
    });
}

size_t fipa_build_factors_workspace_size(int64_t rows, uint64_t f, uint64_t n) {
    return rows < 1 ? 0 : fipa_b200::build_factors_workspace(rows, f, n);
}

int fipa_build_factors(int64_t rows, uint64_t f, const float* features, uint64_t r, uint64_t d_z, const float* w1,
                       const float* w2, float* z1, float* z2, int precision, void* workspace, size_t workspace_bytes,
                       void* stream) {
    return guarded([&] {
        fipa_b200::build_factors(rows, f, features, r, d_z, w1, w2, z1, z2, precision == FIPA_PREC_BF16, workspace,
                                 workspace_bytes, static_cast<cudaStream_t>(stream));
    });
}

int fipa_build_factors_host(int64_t rows, uint64_t f, const double* features, uint64_t r, uint64_t d_z,
                            const double* w1, const double* w2, double* z1, double* z2, int precision) {
    return guarded([&] {
        fipa_b200::build_factors_host(rows, f, features, r, d_z, w1, w2, z1, z2, precision == FIPA_PREC_BF16);
    });
}

}  // extern "C"
