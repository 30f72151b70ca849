// Multi-layer FlashIPA trunk with per-layer backbone frame update (BASELINE cfg3; restated in
// oracle/fipa_oracle.py trunk_forward).  The reference has no trunk; each layer
// is a FlashIpaLayer (the drop-in of flash_ipa_forward, proj/src/flash_ipa.cpp:141-218), frames are
// composed with the reference convention (proj/src/geometry.cpp:78-90).  Per layer, on one stream:
// the 6 layer kernels into a scratch output, then trunk_update (residual + backbone update).
#include "trunk.hpp"

#include <cmath>
#include <cstring>

namespace fipa_b200 {

namespace {
// Reference generator draws for the backbone linear (oracle init_backbone): N(0, (0.1/sqrt(d_in))^2)
// from Rng(seed + 1000 + layer), flat order.
std::vector<double> backbone_draws(std::size_t d_in, std::uint64_t seed) {
    std::vector<double> w(d_in * 6);
    std::uint64_t counter = 0;
    auto next = [&]() {
        counter += 1;
        std::uint64_t z = seed + counter * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    };
    auto uni = [&]() { return static_cast<double>((next() >> 11) + 1) * 0x1.0p-53; };
    const double sd = 0.1 / std::sqrt(static_cast<double>(d_in));
    for (std::size_t k = 0; k < w.size(); k += 2) {  // Box-Muller pairs (cos, sin), reference order
        const double u1 = uni(), u2 = uni();
        const double r = std::sqrt(-2.0 * std::log(u1)), a = 2.0 * M_PI * u2;
        w[k] = sd * (r * std::cos(a));
        if (k + 1 < w.size()) w[k + 1] = sd * (r * std::sin(a));
    }
    return w;
}
}  // namespace

Trunk::Trunk(const Config& cfg, int n_layers, std::uint64_t seed) : cfg_(cfg) {
    if (n_layers < 1) throw ValueError("trunk needs at least one layer");
    for (int l = 0; l < n_layers; ++l) {
        layers_.push_back(std::make_unique<FlashIpaLayer>(cfg));
        layers_.back()->init_weights(seed + l);
        Backbone bb;
        bb.w = backbone_draws(cfg.d_in, seed + 1000 + l);
        bb.b.assign(6, 0.0);
        bb_.push_back(bb);
    }
    dirty_ = true;
}

Trunk::~Trunk() {
    if (d_bb_) cudaFree(d_bb_);
    if (side_) cudaStreamDestroy(side_);
    if (fork_ev_) cudaEventDestroy(fork_ev_);
    if (join_ev_) cudaEventDestroy(join_ev_);
}

int Trunk::chains(std::int64_t B) const { return B >= 2 && layers_[0]->tuning().micro >= 2 ? 2 : 1; }

std::size_t Trunk::chain_bytes(std::int64_t nb, std::int64_t L) const {
    const std::size_t io = (std::size_t(nb) * L * cfg_.d_in * 4 + 255) / 256 * 256;
    return (io + layers_[0]->workspace_size(nb, L) + 255) / 256 * 256;
}

void Trunk::set_backbone(int l, const double* w, const double* b) {
    if (l < 0 || l >= n_layers()) throw ValueError("layer index out of range");
    bb_[l].w.assign(w, w + cfg_.d_in * 6);
    bb_[l].b.assign(b, b + 6);
    dirty_ = true;
}

void Trunk::upload() {
    if (d_bb_) cudaFree(d_bb_);
    d_bb_ = nullptr;
    const std::size_t per = cfg_.d_in * 6 + 6;
    std::vector<float> h(per * bb_.size());
    for (std::size_t l = 0; l < bb_.size(); ++l) {
        for (std::size_t k = 0; k < cfg_.d_in * 6; ++k) h[l * per + k] = static_cast<float>(bb_[l].w[k]);
        for (int k = 0; k < 6; ++k) h[l * per + cfg_.d_in * 6 + k] = static_cast<float>(bb_[l].b[k]);
    }
    cuda_check(cudaMalloc(&d_bb_, h.size() * 4), "cudaMalloc");
    cuda_check(cudaMemcpy(d_bb_, h.data(), h.size() * 4, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
    dirty_ = false;
}

std::size_t Trunk::workspace_size(std::int64_t B, std::int64_t L) const {
    const int n = chains(B);
    std::size_t total = 0;
    for (int c = 0; c < n; ++c) total += chain_bytes(B * (c + 1) / n - B * c / n, L);
    return total;
}

void Trunk::forward(std::int64_t B, std::int64_t L, const float* s, const float* z1, const float* z2,
                    const float* rot, const float* trans, const std::uint8_t* mask, float* s_out, float* rot_out,
                    float* trans_out, void* workspace, std::size_t workspace_bytes, cudaStream_t stream) {
    if (B < 1 || L < 1) throw ValueError("empty batch");
    if (!s || !z1 || !z2 || !rot || !trans || !s_out || !rot_out || !trans_out) throw ValueError("null pointer");
    const std::size_t need = workspace_size(B, L);
    if (workspace == nullptr || workspace_bytes < need) throw ValueError("trunk workspace too small");
    if (dirty_) upload();
    const std::size_t BL = std::size_t(B) * L, din = cfg_.d_in, rdz = std::size_t(cfg_.rank) * cfg_.d_z;
    if (s_out != s) cuda_check(cudaMemcpyAsync(s_out, s, BL * din * 4, cudaMemcpyDeviceToDevice, stream), "copy");
    if (rot_out != rot) cuda_check(cudaMemcpyAsync(rot_out, rot, BL * 9 * 4, cudaMemcpyDeviceToDevice, stream), "copy");
    if (trans_out != trans)
        cuda_check(cudaMemcpyAsync(trans_out, trans, BL * 3 * 4, cudaMemcpyDeviceToDevice, stream), "copy");
    const int n = chains(B);
    if (n > 1) {
        if (!side_) {
            cuda_check(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking), "stream");
            cuda_check(cudaEventCreateWithFlags(&fork_ev_, cudaEventDisableTiming), "event");
            cuda_check(cudaEventCreateWithFlags(&join_ev_, cudaEventDisableTiming), "event");
        }
        cuda_check(cudaEventRecord(fork_ev_, stream), "event record");
        cuda_check(cudaStreamWaitEvent(side_, fork_ev_, 0), "stream wait");
    }
    const std::size_t per = cfg_.d_in * 6 + 6;
    char* base = static_cast<char*>(workspace);
    for (int c = 0; c < n; ++c) {
        const std::int64_t b0 = B * c / n, nb = B * (c + 1) / n - b0;
        const std::size_t r = std::size_t(b0) * L, rows = std::size_t(nb) * L;
        const std::size_t io = (rows * din * 4 + 255) / 256 * 256, bytes = chain_bytes(nb, L);
        cudaStream_t st = c == 0 ? stream : side_;
        float* ipa_out = reinterpret_cast<float*>(base);
        void* lws = base + io;
        for (int l = 0; l < n_layers(); ++l) {
            layers_[l]->forward(nb, L, s_out + r * din, z1 + r * rdz, z2 + r * rdz, rot_out + r * 9, trans_out + r * 3,
                                mask ? mask + r : nullptr, ipa_out, lws, bytes - io, st);
            launch_trunk_update(s_out + r * din, ipa_out, d_bb_ + l * per, d_bb_ + l * per + cfg_.d_in * 6,
                                rot_out + r * 9, trans_out + r * 3, mask ? mask + r : nullptr,
                                static_cast<std::int64_t>(rows), int(cfg_.d_in), st);
        }
        base += bytes;
    }
    if (n > 1) {
        cuda_check(cudaEventRecord(join_ev_, side_), "event record");
        cuda_check(cudaStreamWaitEvent(stream, join_ev_, 0), "stream wait");
    }
    cuda_check(cudaGetLastError(), "trunk launch");
}

int Trunk::launches_per_forward() const { return n_layers() * (layers_[0]->launches_per_forward() + 1); }

int Trunk::step_launches(std::int64_t B, std::int64_t L) const {
    const int n = chains(B);
    int total = 0;
    for (int c = 0; c < n; ++c)
        total += n_layers() * (layers_[0]->step_launches(B * (c + 1) / n - B * c / n, L, false) + 1);
    return total;
}

}  // namespace fipa_b200
