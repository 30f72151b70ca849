// fp32 SIMT path (precision="f32"): the accuracy path for the 1e-4 gate, and the path for
// shapes the tcgen05 kernels do not cover (lifted widths > 448, e.g. z_factor_rank >= 3).
// Same math and layout as the bf16 path; every product accumulates in fp32 on CUDA cores.
//   gemm_f32        <- linear / matmul_rows   proj/src/tensor.cpp:212-225, 292-317
//   attn_fwd_f32    <- flash_attention        proj/src/attention_kernel.cpp:112-188
//                      + epilogue             proj/src/flash_ipa.cpp:171-210
#include <cuda_runtime.h>

#include <cmath>
#include <stdexcept>

#include "kernels.hpp"

namespace fipa_b200 {

namespace {

constexpr int TM = 64, TN = 64, TK = 16;

// C[M,N] = A[M,K] (row-major) . B[K,N] (row-major) (+bias) with masked rows zeroed.
__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ A,
                                                       const float* __restrict__ B,
                                                       float* __restrict__ C, int M, int N, int K, int lda,
                                                       const float* __restrict__ bias,
                                                       const uint8_t* __restrict__ row_mask) {
    __shared__ float sA[TK][TM + 4];
    __shared__ float sB[TK][TN + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += TK) {
        for (int e = threadIdx.x; e < TM * TK; e += 256) {
            const int r = e / TK, kk = e % TK;
            const int gm = m0 + r, gk = k0 + kk;
            sA[kk][r] = (gm < M && gk < K) ? A[int64_t(gm) * lda + gk] : 0.f;
        }
        for (int e = threadIdx.x; e < TN * TK; e += 256) {
            const int kk = e / TN, cidx = e % TN;
            const int gk = k0 + kk, gn = n0 + cidx;
            sB[kk][cidx] = (gk < K && gn < N) ? B[int64_t(gk) * N + gn] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = sA[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = sB[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gm = m0 + ty * 4 + i;
        if (gm >= M) continue;
        const bool zero = row_mask != nullptr && row_mask[gm] == 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gn = n0 + tx * 4 + j;
            if (gn >= N) continue;
            float v = acc[i][j] + (bias != nullptr ? bias[gn] : 0.f);
            C[int64_t(gm) * N + gn] = zero ? 0.f : v;
        }
    }
}

constexpr int kMaxChunks = 24;  // lifted widths up to 768
constexpr int kWarps = 8;

struct F32Params {
    int L, H, dqk_pad, dv_pad, c, d_z, rank, n_value, seg, feat;
};

// One warp per (sample*head, query row); lanes stride the lifted width.
__global__ void __launch_bounds__(kWarps * 32) attn_fwd_f32_kernel(AttnF32Args a, F32Params p) {
    extern __shared__ float s_o[];  // kWarps x dv_pad
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int bh = blockIdx.y;
    const int qi = blockIdx.x * kWarps + warp;
    if (qi >= p.L) return;
    const int64_t qrow = static_cast<int64_t>(bh) * p.L + qi;
    const float* q = a.qhat + qrow * p.dqk_pad;
    float qr[kMaxChunks], o[kMaxChunks];
#pragma unroll
    for (int e = 0; e < kMaxChunks; ++e) {
        const int col = e * 32 + lane;
        qr[e] = col < p.dqk_pad ? q[col] : 0.f;
        o[e] = 0.f;
    }
    float m = -INFINITY, l = 0.f;
    const float* kb = a.khat + static_cast<int64_t>(bh) * p.L * p.dqk_pad;
    const float* vb = a.vhat + static_cast<int64_t>(bh) * p.L * p.dv_pad;
    // S = q_hat . k_hat is already in log2 units and carries the folded column bias
    // (pack.cu); masked keys hold -1e30 and vanish once any valid key is seen.
    for (int j = 0; j < p.L; ++j) {
        const float* kr = kb + static_cast<int64_t>(j) * p.dqk_pad;
        float dot = 0.f;
#pragma unroll
        for (int e = 0; e < kMaxChunks; ++e) {
            const int col = e * 32 + lane;
            if (col < p.dqk_pad) dot = fmaf(qr[e], kr[col], dot);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
        const float s = dot;
        float w;
        if (s > m) {
            const float scale = exp2f(m - s);  // 0 when m == -inf
            l *= scale;
#pragma unroll
            for (int e = 0; e < kMaxChunks; ++e) o[e] *= scale;
            m = s;
            w = 1.f;
        } else {
            w = exp2f(s - m);
        }
        l += w;
        const float* vr = vb + static_cast<int64_t>(j) * p.dv_pad;
#pragma unroll
        for (int e = 0; e < kMaxChunks; ++e) {
            const int col = e * 32 + lane;
            if (col < p.dv_pad) o[e] = fmaf(w, vr[col], o[e]);
        }
    }
    const float inv_l = l > 0.f ? 1.f / l : 0.f;
    if (lane == 0) a.lse[qrow] = l > 0.f ? (m + log2f(l)) * 0.6931471805599453f : -INFINITY;
    float* so = s_o + warp * p.dv_pad;
#pragma unroll
    for (int e = 0; e < kMaxChunks; ++e) {
        const int col = e * 32 + lane;
        if (col < p.dv_pad) so[col] = o[e] * inv_l;
    }
    __syncwarp();
    const int b = bh / p.H, h = bh % p.H;
    const int64_t grow = static_cast<int64_t>(b) * p.L + qi;
    float* fo = a.feat + grow * p.feat + h * p.seg;
    const float* z1r = a.z1 + grow * (p.rank * p.d_z);
    for (int d = lane; d < p.d_z; d += 32) {
        float acc = 0.f;
        for (int rho = 0; rho < p.rank; ++rho) acc = fmaf(z1r[rho * p.d_z + d], so[p.c + rho * p.d_z + d], acc);
        fo[d] = acc;
    }
    for (int ch = lane; ch < p.c; ch += 32) fo[p.d_z + ch] = so[ch];
    const int base = p.c + p.rank * p.d_z, Nv = p.n_value;
    for (int q2 = lane; q2 < Nv; q2 += 32) {
        const float* R = a.rot + grow * 9;
        const float* t = a.trans + grow * 3;
        const float* pt = so + base;
        // point block = [t hi (3) | t lo (3) | R_j v_p (3Nv)]  (pack.cu)
        const float gx = pt[6 + 3 * q2 + 0] + pt[0] + pt[3] - t[0];
        const float gy = pt[6 + 3 * q2 + 1] + pt[1] + pt[4] - t[1];
        const float gz = pt[6 + 3 * q2 + 2] + pt[2] + pt[5] - t[2];
        const float lx = R[0] * gx + R[3] * gy + R[6] * gz;
        const float ly = R[1] * gx + R[4] * gy + R[7] * gz;
        const float lz = R[2] * gx + R[5] * gy + R[8] * gz;
        float* fp = fo + p.d_z + p.c;
        fp[3 * q2 + 0] = lx;
        fp[3 * q2 + 1] = ly;
        fp[3 * q2 + 2] = lz;
        fp[3 * Nv + q2] = sqrtf(lx * lx + ly * ly + lz * lz);
    }
}

}  // namespace

void launch_gemm_f32(const float* A, int lda, const float* B, float* C, int M, int N, int K,
                     const float* bias, const uint8_t* row_mask, cudaStream_t stream) {
    if (M <= 0 || N <= 0) return;
    dim3 grid((N + TN - 1) / TN, (M + TM - 1) / TM);
    gemm_f32_kernel<<<grid, 256, 0, stream>>>(A, B, C, M, N, K, lda, bias, row_mask);
}

void launch_attn_fwd_f32(const LayerDims& d, const AttnF32Args& a, cudaStream_t stream) {
    if (d.dqk_pad > kMaxChunks * 32 || d.dv_pad > kMaxChunks * 32)
        throw std::invalid_argument("f32 attention: lifted width exceeds 768");
    F32Params p{a.L, d.heads, d.dqk_pad, d.dv_pad, d.c, d.d_z, d.rank, d.n_value, d.seg, d.feat_ld};
    const size_t smem = sizeof(float) * kWarps * d.dv_pad;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(attn_fwd_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    dim3 grid((a.L + kWarps - 1) / kWarps, static_cast<unsigned>(a.B * d.heads));
    attn_fwd_f32_kernel<<<grid, kWarps * 32, smem, stream>>>(a, p);
}

}  // namespace fipa_b200
