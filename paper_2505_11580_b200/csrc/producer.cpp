// Host side of the pair-factor producer: validation with the reference's rules
// (proj/src/pair_features.cpp:10-19, 83-93) and the device / host entry points behind the C ABI.
#include "producer.hpp"

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

namespace fipa_b200 {

namespace {
std::size_t round_up8(std::size_t x) { return (x + 7) / 8 * 8; }
}  // namespace

void validate_knn(std::int64_t B, std::int64_t L, const KnnSpec& s) {
    if (B < 1) throw ValueError("batch must be >= 1");
    if (L < 2) throw ValueError("knn_distogram needs at least two residues");
    if (s.k < 1 || s.k > L - 1)
        throw ValueError("neighbor count k=" + std::to_string(s.k) + " must lie in [1, L-1] with L=" + std::to_string(L));
    if (s.n_bins < 2) throw ValueError("distogram needs at least two bins");
    if (!(s.d_min < s.d_max)) throw ValueError("distogram range is empty");
    if (s.pe_dim % 2 != 0 || s.pe_dim < 0) throw ValueError("positional encoding width must be even");
}

namespace {
template <class T, class O>
void knn_distogram_impl(std::int64_t B, std::int64_t L, const T* trans, const KnnSpec& spec, O* out,
                        cudaStream_t stream) {
    validate_knn(B, L, spec);
    if (trans == nullptr || out == nullptr) throw ValueError("null pointer");
    // frequencies as the reference forms them (std::pow on the host, pair_features.cpp:73-75)
    std::vector<double> freq(std::max(1, spec.pe_dim / 2));
    for (int p = 0; p < spec.pe_dim / 2; ++p)
        freq[p] = std::pow(10000.0, -static_cast<double>(2 * p) / static_cast<double>(spec.pe_dim));
    double* d_freq = nullptr;
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&d_freq), freq.size() * sizeof(double), stream), "cudaMallocAsync");
    cuda_check(cudaMemcpyAsync(d_freq, freq.data(), freq.size() * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D");
    launch_knn_distogram(trans, int(B), int(L), spec, d_freq, out, stream);
    cuda_check(cudaGetLastError(), "knn_distogram launch");
    cuda_check(cudaFreeAsync(d_freq, stream), "cudaFreeAsync");
}
}  // namespace

void knn_distogram(std::int64_t B, std::int64_t L, const float* trans, const KnnSpec& spec, float* out,
                   cudaStream_t stream) {
    knn_distogram_impl(B, L, trans, spec, out, stream);
}

void knn_distogram(std::int64_t B, std::int64_t L, const double* trans, const KnnSpec& spec, double* out,
                   cudaStream_t stream) {
    knn_distogram_impl(B, L, trans, spec, out, stream);
}

std::size_t build_factors_workspace(std::int64_t rows, std::size_t f, std::size_t n) {
    const std::size_t ld = round_up8(f);
    return (rows * ld * 2 + 255) / 256 * 256 + 2 * ((n * ld * 2 + 255) / 256 * 256);
}

void build_factors(std::int64_t rows, std::size_t f, const float* features, std::size_t r, std::size_t d_z,
                   const float* w1, const float* w2, float* z1, float* z2, bool bf16, void* workspace,
                   std::size_t workspace_bytes, cudaStream_t stream) {
    if (rows < 1 || f < 1 || r < 1 || d_z < 1) throw ValueError("factor rank and channel width must be positive");
    if (!features || !w1 || !w2 || !z1 || !z2) throw ValueError("null pointer");
    const std::size_t n = r * d_z;
    if (!bf16) {
        launch_gemm_f32(features, int(f), w1, z1, int(rows), int(n), int(f), nullptr, nullptr, stream);
        launch_gemm_f32(features, int(f), w2, z2, int(rows), int(n), int(f), nullptr, nullptr, stream);
        cuda_check(cudaGetLastError(), "build_factors launch");
        return;
    }
    const std::size_t ld = round_up8(f);
    if (workspace == nullptr || workspace_bytes < build_factors_workspace(rows, f, n))
        throw ValueError("build_factors workspace too small");
    char* base = static_cast<char*>(workspace);
    auto* a = reinterpret_cast<__nv_bfloat16*>(base);
    auto* b1 = reinterpret_cast<__nv_bfloat16*>(base + (rows * ld * 2 + 255) / 256 * 256);
    auto* b2 = reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<char*>(b1) + (n * ld * 2 + 255) / 256 * 256);
    launch_f32_to_bf16_2d(features, a, rows, int(f), int(ld), stream);
    launch_transpose_to_bf16(w1, int(f), int(n), b1, int(ld), stream);
    launch_transpose_to_bf16(w2, int(f), int(n), b2, int(ld), stream);
    for (int t = 0; t < 2; ++t) {
        GemmArgs g;
        g.A = a;
        g.lda = ld;
        g.B = t == 0 ? b1 : b2;
        g.ldb = ld;
        g.C = t == 0 ? z1 : z2;
        g.ldc = n;
        g.M = int(rows);
        g.N = int(n);
        g.K = int(f);
        launch_gemm_bf16(g, stream);
    }
    cuda_check(cudaGetLastError(), "build_factors launch");
}

namespace {
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(std::size_t bytes) { cuda_check(cudaMalloc(&p, bytes ? bytes : 16), "cudaMalloc"); }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};
std::vector<float> to_f32(const double* x, std::size_t n) {
    std::vector<float> v(n);
    for (std::size_t i = 0; i < n; ++i) v[i] = static_cast<float>(x[i]);
    return v;
}
}  // namespace

// The reference's f64 API: float64 translations copied as they are and float64 features back --
// neighbour choice and bins bit-exact with proj/src/pair_features.cpp:29-45.
void knn_distogram_host(std::int64_t B, std::int64_t L, const double* trans, const KnnSpec& spec, double* out) {
    validate_knn(B, L, spec);
    if (trans == nullptr || out == nullptr) throw ValueError("null pointer");
    const std::size_t n_in = std::size_t(B) * L * 3, n_out = std::size_t(B) * L * spec.k * (spec.n_bins + spec.pe_dim);
    DevBuf dt(n_in * 8), dout(n_out * 8);
    cuda_check(cudaMemcpy(dt.p, trans, n_in * 8, cudaMemcpyHostToDevice), "H2D");
    knn_distogram(B, L, dt.as<double>(), spec, dout.as<double>(), nullptr);
    cuda_check(cudaMemcpy(out, dout.p, n_out * 8, cudaMemcpyDeviceToHost), "D2H");
}

void build_factors_host(std::int64_t rows, std::size_t f, const double* features, std::size_t r, std::size_t d_z,
                        const double* w1, const double* w2, double* z1, double* z2, bool bf16) {
    if (!features || !w1 || !w2 || !z1 || !z2) throw ValueError("null pointer");
    const std::size_t n = r * d_z;
    const auto fe = to_f32(features, rows * f), a = to_f32(w1, f * n), b = to_f32(w2, f * n);
    DevBuf df(fe.size() * 4), d1(a.size() * 4), d2(b.size() * 4), o1(rows * n * 4), o2(rows * n * 4);
    DevBuf ws(build_factors_workspace(rows, f, n));
    cuda_check(cudaMemcpy(df.p, fe.data(), fe.size() * 4, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(d1.p, a.data(), a.size() * 4, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(d2.p, b.data(), b.size() * 4, cudaMemcpyHostToDevice), "H2D");
    build_factors(rows, f, df.as<float>(), r, d_z, d1.as<float>(), d2.as<float>(), o1.as<float>(), o2.as<float>(), bf16,
                  ws.p, build_factors_workspace(rows, f, n), nullptr);
    std::vector<float> h(rows * n);
    cuda_check(cudaMemcpy(h.data(), o1.p, h.size() * 4, cudaMemcpyDeviceToHost), "D2H");
    for (std::size_t i = 0; i < h.size(); ++i) z1[i] = h[i];
    cuda_check(cudaMemcpy(h.data(), o2.p, h.size() * 4, cudaMemcpyDeviceToHost), "D2H");
    for (std::size_t i = 0; i < h.size(); ++i) z2[i] = h[i];
}

}  // namespace fipa_b200
