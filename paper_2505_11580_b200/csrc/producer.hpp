// Pair-factor producer.  See producer.cpp / pair_features.cu.
#pragma once

#include <cstdint>

#include "kernels.hpp"
#include "layer.hpp"

namespace fipa_b200 {

void validate_knn(std::int64_t B, std::int64_t L, const KnnSpec& spec);
void knn_distogram(std::int64_t B, std::int64_t L, const float* trans, const KnnSpec& spec, float* out,
                   cudaStream_t stream);
void knn_distogram(std::int64_t B, std::int64_t L, const double* trans, const KnnSpec& spec, double* out,
                   cudaStream_t stream);
std::size_t build_factors_workspace(std::int64_t rows, std::size_t f, std::size_t n);
void build_factors(std::int64_t rows, std::size_t f, const float* features, std::size_t r, std::size_t d_z,
                   const float* w1, const float* w2, float* z1, float* z2, bool bf16, void* workspace,
                   std::size_t workspace_bytes, cudaStream_t stream);

void knn_distogram_host(std::int64_t B, std::int64_t L, const double* trans, const KnnSpec& spec, double* out);
void build_factors_host(std::int64_t rows, std::size_t f, const double* features, std::size_t r, std::size_t d_z,
                        const double* w1, const double* w2, double* z1, double* z2, bool bf16);

}  // namespace fipa_b200
