// Pair-factor producer on the GPU: the step before the layer that turns
// coordinates into the factorised pair representation z1, z2.
//   knn_distogram        proj/src/pair_features.cpp:10-64
//   positional_encoding  proj/src/pair_features.cpp:66-81
//   build_factors        proj/src/pair_features.cpp:83-97 (two linears; tcgen05 GEMM here)
// Neighbour selection is integer work and must match the reference exactly: translations stay in
// the caller's precision (float64 for the reference's f64 API: no rounding before the distance),
// distances are formed in float64 with the reference's operation order (no FMA contraction: __dmul_rn/__dadd_rn, a
// correctly rounded sqrt), ordered lexicographically by (distance, index) -- the reference's
// partial_sort of (distance, index) pairs gives the lower-index tie-break.  One warp per residue:
// each lane keeps a sorted top-k of its strided candidates in shared memory, then k rounds of a
// warp arg-min merge the 32 lists.  The O(L^2) scan is FP64-bound; memory stays O(L k).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <stdexcept>
#include <vector>

#include "kernels.hpp"

namespace fipa_b200 {

namespace {

constexpr int kWarps = 8;

__device__ __forceinline__ bool lex_less(double da, int ia, double db, int ib) {
    return da < db || (da == db && ia < ib);
}

template <class T, class O>
__global__ void __launch_bounds__(kWarps * 32) knn_distogram_kernel(const T* __restrict__ trans, int B, int L,
                                                                    KnnSpec spec, const double* __restrict__ freq,
                                                                    O* __restrict__ out) {
    extern __shared__ __align__(8) unsigned char smraw[];
    const int k = spec.k;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* s_d = reinterpret_cast<double*>(smraw) + (warp * 32 + lane) * k;
    int* s_i = reinterpret_cast<int*>(reinterpret_cast<double*>(smraw) + kWarps * 32 * k) + (warp * 32 + lane) * k;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
    if (row >= static_cast<int64_t>(B) * L) return;
    const int b = static_cast<int>(row / L), i = static_cast<int>(row % L);
    const T* t = trans + static_cast<int64_t>(b) * L * 3;
    const double xi = t[i * 3], yi = t[i * 3 + 1], zi = t[i * 3 + 2];

    // lane-local sorted top-k of candidates j = lane, lane + 32, ...
    int cnt = 0;
    for (int j = lane; j < L; j += 32) {
        if (j == i) continue;
        const double dx = __dadd_rn(static_cast<double>(t[j * 3]), -xi);
        const double dy = __dadd_rn(static_cast<double>(t[j * 3 + 1]), -yi);
        const double dz = __dadd_rn(static_cast<double>(t[j * 3 + 2]), -zi);
        const double d = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
        if (cnt == k && !lex_less(d, j, s_d[k - 1], s_i[k - 1])) continue;
        int pos = cnt < k ? cnt : k - 1;  // insertion sort from the back
        while (pos > 0 && lex_less(d, j, s_d[pos - 1], s_i[pos - 1])) {
            s_d[pos] = s_d[pos - 1];
            s_i[pos] = s_i[pos - 1];
            --pos;
        }
        s_d[pos] = d;
        s_i[pos] = j;
        if (cnt < k) ++cnt;
    }
    // k rounds of warp arg-min over the lane heads
    const int width = spec.n_bins + spec.pe_dim;
    O* orow = out + row * static_cast<int64_t>(k) * width;
    for (int e = lane; e < k * width; e += 32) orow[e] = O(0);
    __syncwarp();
    const double bin_width = (spec.d_max - spec.d_min) / static_cast<double>(spec.n_bins);
    int head = 0;
    for (int n = 0; n < k; ++n) {
        double bd = head < cnt ? s_d[head] : INFINITY;
        int bi = head < cnt ? s_i[head] : 0x7fffffff;
        int bl = lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, bd, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
            if (lex_less(od, oi, bd, bi)) {
                bd = od;
                bi = oi;
                bl = ol;
            }
        }
        if (lane == bl) ++head;
        // one-hot distance bin (clipped into the end bins) + encoding of the offset j - i
        if (lane == 0) {
            double rel = (bd - spec.d_min) / bin_width;
            rel = rel > 0.0 ? rel : 0.0;
            const double last = static_cast<double>(spec.n_bins - 1);
            const int bin = rel >= last ? spec.n_bins - 1 : static_cast<int>(rel);
            orow[n * width + bin] = O(1);
        }
        const double x = static_cast<double>(bi - i);
        for (int p = lane; p < spec.pe_dim / 2; p += 32) {
            double sv, cv;
            sincos(x * freq[p], &sv, &cv);
            orow[n * width + spec.n_bins + 2 * p] = static_cast<O>(sv);
            orow[n * width + spec.n_bins + 2 * p + 1] = static_cast<O>(cv);
        }
    }
}

__global__ void transpose_to_bf16_kernel(const float* __restrict__ w, int K, int N, __nv_bfloat16* __restrict__ wt,
                                         int ld) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= static_cast<int64_t>(N) * ld) return;
    const int n = static_cast<int>(e / ld), kk = static_cast<int>(e % ld);
    wt[e] = __float2bfloat16_rn(kk < K ? w[static_cast<int64_t>(kk) * N + n] : 0.f);
}

}  // namespace

void launch_transpose_to_bf16(const float* w, int K, int N, __nv_bfloat16* wt, int ld, cudaStream_t stream) {
    const int64_t n = int64_t(N) * ld;
    transpose_to_bf16_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(w, K, N, wt, ld);
}

size_t knn_smem_bytes(const KnnSpec& spec) { return size_t(kWarps) * 32 * spec.k * (sizeof(double) + sizeof(int)); }

template <class T, class O>
void launch_knn_impl(const T* trans, int B, int L, const KnnSpec& spec, const double* d_freq, O* out,
                     cudaStream_t stream) {
    const size_t smem = knn_smem_bytes(spec);
    if (smem > 200 * 1024) throw std::invalid_argument("knn_distogram: k too large for the GPU kernel");
    auto kern = knn_distogram_kernel<T, O>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    const int64_t rows = int64_t(B) * L;
    kern<<<static_cast<unsigned>((rows + kWarps - 1) / kWarps), kWarps * 32, smem, stream>>>(trans, B, L, spec,
                                                                                            d_freq, out);
}

void launch_knn_distogram(const float* trans, int B, int L, const KnnSpec& spec, const double* d_freq, float* out,
                          cudaStream_t stream) {
    launch_knn_impl(trans, B, L, spec, d_freq, out, stream);
}

void launch_knn_distogram(const double* trans, int B, int L, const KnnSpec& spec, const double* d_freq, double* out,
                          cudaStream_t stream) {
    launch_knn_impl(trans, B, L, spec, d_freq, out, stream);
}

}  // namespace fipa_b200
