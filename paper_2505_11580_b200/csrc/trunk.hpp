// Multi-layer FlashIPA trunk (BASELINE cfg3).  See trunk.cpp.
#pragma once

#include <memory>
#include <vector>

#include "layer.hpp"

namespace fipa_b200 {

class Trunk {
public:
    struct Backbone {
        std::vector<double> w;  // [d_in, 6] row-major
        std::vector<double> b;  // [6]
    };
    Trunk(const Config& cfg, int n_layers, std::uint64_t seed);
    ~Trunk();
    Trunk(const Trunk&) = delete;
    Trunk& operator=(const Trunk&) = delete;

    int n_layers() const { return static_cast<int>(layers_.size()); }
    FlashIpaLayer& layer(int l) { return *layers_.at(l); }
    const Backbone& backbone(int l) const { return bb_.at(l); }
    void set_backbone(int l, const double* w, const double* b);
    std::size_t workspace_size(std::int64_t B, std::int64_t L) const;
    // s_out / rot_out / trans_out may alias the inputs.
    void forward(std::int64_t B, std::int64_t L, const float* s, const float* z1, const float* z2, const float* rot,
                 const float* trans, const std::uint8_t* mask, float* s_out, float* rot_out, float* trans_out,
                 void* workspace, std::size_t workspace_bytes, cudaStream_t stream);
    int launches_per_forward() const;
    int step_launches(std::int64_t B, std::int64_t L) const;  // chains included

private:
    void upload();
    // Samples are independent through the whole trunk: with the layers' micro-batching on (B >= 2)
    // they run as two sample chains on forked streams with no join between layers, so one chain's
    // layer boundary (GPU drain + frame update) overlaps the other chain's kernels.
    int chains(std::int64_t B) const;
    std::size_t chain_bytes(std::int64_t nb, std::int64_t L) const;
    cudaStream_t side_ = nullptr;
    cudaEvent_t fork_ev_ = nullptr, join_ev_ = nullptr;
    Config cfg_;
    std::vector<std::unique_ptr<FlashIpaLayer>> layers_;
    std::vector<Backbone> bb_;
    float* d_bb_ = nullptr;
    bool dirty_ = true;
};

}  // namespace fipa_b200
