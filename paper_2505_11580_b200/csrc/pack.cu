// Frame application + lifted-row packing (K2) and small helpers.
//
// Restates, per residue and head, the reference lifts
//   lift_queries  proj/src/flash_ipa.cpp:23-55
//   lift_keys     proj/src/flash_ipa.cpp:57-94
//   lift_values   proj/src/flash_ipa.cpp:96-126
//   bias_factors  proj/src/pair_features.cpp:141-163 (w_l folded, flash_ipa.cpp:161-167)
//   apply         proj/src/geometry.cpp:63-68
// in the B200 layout.  With A_p = T_i q_p = R_i q_p + t_i and
// B_p = T_j k_p, the reference point term g*sum_p <A_p, B_p> is expanded exactly as
//   g*sum_p <R_i q_p, R_j k_p> + g<Qbar_i, t_j> + g<t_i, W_j>,  Qbar_i = sum_p R_i q_p,
//   W_j = sum_p T_j k_p,
// so the only large (translation-sized) products sit in two 3-vector dot products that are
// carried as bf16 hi/lo splits (a.b ~ a_hi.b_hi + a_hi.b_lo + a_lo.b_hi).  This keeps the
// bf16 logits accurate for protein-scale coordinates (tens of Angstrom), where a plain bf16
// T_i q_p column loses ~1 logit unit.  Per head (L2E = log2 e, queries pre-scaled so that
// S = q_hat . k_hat is in log2 units):
//   q_hat = L2E*[ q | R_i q_p | Qbar hi,hi,lo | t_i hi,lo,hi ] | 1, 1, 0 | 0.. | L2E*z1_i | 0
//   k_hat = [ (w_l/sqrt c) k | g R_j k_p | g t_j hi,lo,hi | g W_j hi,hi,lo ] | cb hi, lo, 1 | 0.. |
//           w_l w_bias[h] (.) z2_j | 0          (the pair block starts at zq = round_up(g0 + 21, 8))
//   cb_j  = L2E * (-g/2 sum_p |T_j k_p|^2)   (-1e30 for masked keys, lo = 0)
// The reference's |T_i q_p|^2 column (paired with -g/2) is constant along a query row and
// cancels in the softmax, so it is dropped; its (ones, -g/2 |k|^2) pair becomes the folded
// column bias cb.  The (0, 1) column does not change the logits; it makes the backward's
// dQ_acc = dS.K_hat carry sum_j dS_ij (as rounded for the MMA), so the translation-sized
// query-side terms can be formed as sum_j dS_ij (t_j - t_i) without cancellation error.  Values:
//   v_hat = [ v | z2_j flat | t_j hi (3) | t_j lo (3) | R_j v_p (3Nv) | 0 ]
// (sum_j p_ij T_j v_p = sum_j p_ij R_j v_p + sum_j p_ij t_j, translation kept to ~2^-17).
// For the fp32 path the same layout is written with hi = value, lo = 0.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "kernels.hpp"
#include "ptx.cuh"

namespace fipa_b200 {

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FIPA_PDL");
        return e == nullptr || std::string(e) != "0";
    }();
    return on;
}

int device_sm_count() {
    static std::atomic<int> cache[64];  // zero-initialised (static storage)
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    int n = cache[dev].load(std::memory_order_relaxed);
    if (n > 0) return n;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
    return n;
}

namespace {

constexpr float kL2E = 1.4426950408889634f;
constexpr float kMaskedBias = -1.0e30f;

template <typename T>
__device__ __forceinline__ void store_pair(T* dst, float a, float b);
template <>
__device__ __forceinline__ void store_pair<__nv_bfloat16>(__nv_bfloat16* dst, float a, float b) {
    *reinterpret_cast<__nv_bfloat162*>(dst) = __floats2bfloat162_rn(a, b);
}
template <>
__device__ __forceinline__ void store_pair<float>(float* dst, float a, float b) {
    *reinterpret_cast<float2*>(dst) = make_float2(a, b);
}

template <typename T>
__device__ __forceinline__ float hi_part(float x) {
    return sizeof(T) == 4 ? x : __bfloat162float(__float2bfloat16_rn(x));
}
template <typename T>
__device__ __forceinline__ float lo_part(float x) {
    return sizeof(T) == 4 ? 0.f : x - __bfloat162float(__float2bfloat16_rn(x));
}

__device__ __forceinline__ void ptx_mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n\tfence.mbarrier_init.release.cluster;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
                 "r"(count)
                 : "memory");
}
__device__ __forceinline__ void ptx_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void ptx_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
                 : "memory");
}
__device__ __forceinline__ void ptx_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))), "r"(parity)
            : "memory");
    }
}

template <typename OutT>
__global__ void __launch_bounds__(256) pack_kernel(LayerDims d, PackArgs a) {
    extern __shared__ float sm[];
    const int H = d.heads, c = d.c, Nq = d.n_query, Nv = d.n_value, rdz = d.rank * d.d_z;
    float* s_proj = sm;                  // n_proj
    float* s_z1 = s_proj + d.n_proj;     // rdz
    float* s_z2 = s_z1 + rdz;            // rdz
    float* s_rq = s_z2 + rdz;            // H*Nq*3   R_i q_p
    float* s_rk = s_rq + H * Nq * 3;     // H*Nq*3   R_j k_p
    float* s_rv = s_rk + H * Nq * 3;     // H*Nv*3   R_j v_p
    float* s_hd = s_rv + H * Nv * 3;     // H*8: Qbar(3), W(3), |Tk|^2, pad

    const int64_t row = blockIdx.x;  // b*L + i
    const int b = static_cast<int>(row / a.L);
    const int i = static_cast<int>(row % a.L);
    const int tid = threadIdx.x;

    const float* prow = a.proj + row * d.n_proj;
    for (int e = tid; e < d.n_proj; e += blockDim.x) s_proj[e] = prow[e];
    for (int e = tid; e < rdz; e += blockDim.x) {
        s_z1[e] = a.z1[row * rdz + e];
        s_z2[e] = a.z2[row * rdz + e];
    }
    float R[9], t[3];
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = a.rot[row * 9 + k];
#pragma unroll
    for (int k = 0; k < 3; ++k) t[k] = a.trans[row * 3 + k];
    __syncthreads();

    // Column offsets of the fused projection (reference order w_q|w_k|w_v|w_qp|w_kp|w_vp).
    const int off_q = 0, off_k = H * c, off_v = 2 * H * c;
    const int off_qp = 3 * H * c, off_kp = off_qp + H * Nq * 3, off_vp = off_kp + H * Nq * 3;
    const int npts = H * Nq * 2 + H * Nv;
    for (int e = tid; e < npts; e += blockDim.x) {
        const float* src;
        float* dst;
        if (e < H * Nq) {
            src = s_proj + off_qp + e * 3;
            dst = s_rq + e * 3;
        } else if (e < 2 * H * Nq) {
            src = s_proj + off_kp + (e - H * Nq) * 3;
            dst = s_rk + (e - H * Nq) * 3;
        } else {
            src = s_proj + off_vp + (e - 2 * H * Nq) * 3;
            dst = s_rv + (e - 2 * H * Nq) * 3;
        }
        const float x = src[0], y = src[1], z = src[2];
        dst[0] = fmaf(R[0], x, fmaf(R[1], y, R[2] * z));
        dst[1] = fmaf(R[3], x, fmaf(R[4], y, R[5] * z));
        dst[2] = fmaf(R[6], x, fmaf(R[7], y, R[8] * z));
    }
    __syncthreads();
    for (int h = tid; h < H; h += blockDim.x) {
        float qb[3] = {0.f, 0.f, 0.f}, w[3] = {0.f, 0.f, 0.f}, kn = 0.f;
        for (int p = 0; p < Nq; ++p) {
#pragma unroll
            for (int x = 0; x < 3; ++x) {
                qb[x] += s_rq[(h * Nq + p) * 3 + x];
                const float tk = s_rk[(h * Nq + p) * 3 + x] + t[x];
                w[x] += tk;
                kn = fmaf(tk, tk, kn);
            }
        }
        float* hd = s_hd + h * 8;
        hd[0] = qb[0];
        hd[1] = qb[1];
        hd[2] = qb[2];
        hd[3] = w[0];
        hd[4] = w[1];
        hd[5] = w[2];
        hd[6] = kn;
    }
    __syncthreads();

    const bool valid = a.mask == nullptr || a.mask[row] != 0;
    OutT* qh = static_cast<OutT*>(a.qhat);
    OutT* kh = static_cast<OutT*>(a.khat);
    OutT* vh = static_cast<OutT*>(a.vhat);
    const int g0 = c + 3 * Nq;        // start of the 21 translation/bias columns
    const int zq = d.zq;              // start of the pair-factor columns (8-aligned)
    const int qk_used = d.dqk_used;
    const int v_pair = c + rdz, v_used = d.dv_used;

    for (int h = 0; h < H; ++h) {
        const int64_t hrow = (static_cast<int64_t>(b) * H + h) * a.L + i;
        const float g = a.head_g[h];
        const float* hd = s_hd + h * 8;
        const float cb = valid ? kL2E * (-0.5f * g * hd[6]) : kMaskedBias;
        OutT* q = qh + hrow * d.dqk_pad;
        OutT* k = kh + hrow * d.dqk_pad;
        OutT* v = vh + hrow * d.dv_pad;
        for (int col = 2 * tid; col < d.dqk_pad; col += 2 * blockDim.x) {
            float qv[2], kv[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int cc = col + u;
                if (cc < c) {
                    qv[u] = kL2E * s_proj[off_q + h * c + cc];
                    kv[u] = a.k_scale * s_proj[off_k + h * c + cc];
                } else if (cc < g0) {
                    qv[u] = kL2E * s_rq[h * Nq * 3 + (cc - c)];
                    kv[u] = g * s_rk[h * Nq * 3 + (cc - c)];
                } else if (cc < zq) {
                    const int e = cc - g0;     // 0..20
                    const int x = e % 3;
                    if (e < 9) {               // <Qbar_i, g t_j>:  [Qh Qh Ql] . [th tl th]
                        const float qq = kL2E * hd[x], tt = g * t[x];
                        qv[u] = e < 6 ? hi_part<OutT>(qq) : lo_part<OutT>(qq);
                        kv[u] = (e >= 3 && e < 6) ? lo_part<OutT>(tt) : hi_part<OutT>(tt);
                    } else if (e < 18) {       // <t_i, g W_j>:     [th tl th] . [Wh Wh Wl]
                        const float tq = kL2E * t[x], ww = g * hd[3 + x];
                        qv[u] = (e >= 12 && e < 15) ? lo_part<OutT>(tq) : hi_part<OutT>(tq);
                        kv[u] = e < 15 ? hi_part<OutT>(ww) : lo_part<OutT>(ww);
                    } else if (e < 20) {       // folded column bias: [1 1] . [cb_hi cb_lo]
                        qv[u] = 1.0f;
                        kv[u] = e == 18 ? hi_part<OutT>(cb) : (valid ? lo_part<OutT>(cb) : 0.f);
                    } else if (e == 20) {      // [0] . [1]: logit-neutral; in the backward
                        qv[u] = 0.f;           // dS.K_hat picks up sum_j dS_ij here
                        kv[u] = 1.0f;
                    } else {                   // alignment padding up to zq
                        qv[u] = 0.f;
                        kv[u] = 0.f;
                    }
                } else if (cc < qk_used) {
                    const int e = cc - zq;
                    qv[u] = kL2E * s_z1[e];
                    kv[u] = a.wl_bias[h * d.d_z + (e % d.d_z)] * s_z2[e];
                } else {
                    qv[u] = 0.f;
                    kv[u] = 0.f;
                }
            }
            store_pair<OutT>(q + col, qv[0], qv[1]);
            store_pair<OutT>(k + col, kv[0], kv[1]);
        }
        for (int col = 2 * tid; col < d.dv_pad; col += 2 * blockDim.x) {
            float vv[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int cc = col + u;
                float x;
                if (cc < c) {
                    x = s_proj[off_v + h * c + cc];
                } else if (cc < v_pair) {
                    x = s_z2[cc - c];
                } else if (cc < v_pair + 3) {
                    x = hi_part<OutT>(t[cc - v_pair]);
                } else if (cc < v_pair + 6) {
                    x = lo_part<OutT>(t[cc - v_pair - 3]);
                } else if (cc < v_used) {
                    x = s_rv[h * Nv * 3 + (cc - v_pair - 6)];
                } else {
                    x = 0.f;
                }
                vv[u] = x;
            }
            store_pair<OutT>(v + col, vv[0], vv[1]);
        }
        if (tid == 0) a.colbias[hrow] = valid ? -0.5f * g * hd[6] : -INFINITY;
    }
}

// bf16 path of K2, restructured for HBM: one block per residue; the projection row and the two
// pair-factor rows arrive by bulk copies (TMA engine, one instruction each), warp w assembles the
// lifted rows of heads w, w+8, .. in shared memory (same column recipe as pack_kernel above), and
// the block writes the 3*H rows with coalesced 16-byte stores.
__device__ __forceinline__ void bulk_g2s_pack(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))), "l"(reinterpret_cast<uint64_t>(src)),
                 "r"(bytes), "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
                 : "memory");
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

__global__ void __launch_bounds__(256, 4) pack_bf16_kernel(LayerDims d, PackArgs a) {
    extern __shared__ __align__(16) float sm[];
    const int H = d.heads, c = d.c, Nq = d.n_query, Nv = d.n_value, rdz = d.rank * d.d_z;
    const int nw = blockDim.x >> 5;
    float* s_proj = sm;                                  // n_proj (bulk)
    float* s_z1 = s_proj + ((d.n_proj + 3) & ~3);        // rdz (bulk)
    float* s_z2 = s_z1 + ((rdz + 3) & ~3);               // rdz (bulk)
    float* s_rq = s_z2 + ((rdz + 3) & ~3);               // H*Nq*3
    float* s_rk = s_rq + H * Nq * 3;                     // H*Nq*3
    float* s_rv = s_rk + H * Nq * 3;                     // H*Nv*3
    float* s_hd = s_rv + H * Nv * 3;                     // H*8: Qbar(3), W(3), |Tk|^2
    __nv_bfloat16* s_out = reinterpret_cast<__nv_bfloat16*>(
        (reinterpret_cast<uintptr_t>(s_hd + H * 8) + 15) & ~uintptr_t(15));  // H x (q | k | v) rows
    uint64_t* bar = reinterpret_cast<uint64_t*>(s_out + H * (2 * d.dqk_pad + d.dv_pad));
    const int64_t row = blockIdx.x;
    const int b = static_cast<int>(row / a.L), i = static_cast<int>(row % a.L);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool bulk = ((d.n_proj * 4) & 15) == 0 && ((rdz * 4) & 15) == 0;
    if (threadIdx.x == 0) {
        ptx_mbar_init(bar, 1);
        if (bulk) {
            ptx_expect_tx(bar, (d.n_proj + 2 * rdz) * 4);
            bulk_g2s_pack(s_proj, a.proj + row * d.n_proj, d.n_proj * 4, bar);
            bulk_g2s_pack(s_z1, a.z1 + row * rdz, rdz * 4, bar);
            bulk_g2s_pack(s_z2, a.z2 + row * rdz, rdz * 4, bar);
        } else {
            ptx_arrive(bar);
        }
    }
    if (!bulk) {
        for (int e = threadIdx.x; e < d.n_proj; e += blockDim.x) s_proj[e] = a.proj[row * d.n_proj + e];
        for (int e = threadIdx.x; e < rdz; e += blockDim.x) {
            s_z1[e] = a.z1[row * rdz + e];
            s_z2[e] = a.z2[row * rdz + e];
        }
    }
    float R[9], t[3];
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = __ldg(a.rot + row * 9 + k);
#pragma unroll
    for (int k = 0; k < 3; ++k) t[k] = __ldg(a.trans + row * 3 + k);
    const bool valid = a.mask == nullptr || a.mask[row] != 0;
    __syncthreads();
    ptx_wait(bar, 0);

    const int off_q = 0, off_k = H * c, off_v = 2 * H * c;
    const int off_qp = 3 * H * c, off_kp = off_qp + H * Nq * 3, off_vp = off_kp + H * Nq * 3;
    for (int e = threadIdx.x; e < H * Nq * 2 + H * Nv; e += blockDim.x) {
        const float* src;
        float* dst;
        if (e < H * Nq) {
            src = s_proj + off_qp + e * 3;
            dst = s_rq + e * 3;
        } else if (e < 2 * H * Nq) {
            src = s_proj + off_kp + (e - H * Nq) * 3;
            dst = s_rk + (e - H * Nq) * 3;
        } else {
            src = s_proj + off_vp + (e - 2 * H * Nq) * 3;
            dst = s_rv + (e - 2 * H * Nq) * 3;
        }
        const float x = src[0], y = src[1], z = src[2];
        dst[0] = fmaf(R[0], x, fmaf(R[1], y, R[2] * z));
        dst[1] = fmaf(R[3], x, fmaf(R[4], y, R[5] * z));
        dst[2] = fmaf(R[6], x, fmaf(R[7], y, R[8] * z));
    }
    __syncthreads();
    for (int h = threadIdx.x; h < H; h += blockDim.x) {
        float qb[3] = {0.f, 0.f, 0.f}, w[3] = {0.f, 0.f, 0.f}, kn = 0.f;
        for (int p = 0; p < Nq; ++p) {
#pragma unroll
            for (int x = 0; x < 3; ++x) {
                qb[x] += s_rq[(h * Nq + p) * 3 + x];
                const float tk = s_rk[(h * Nq + p) * 3 + x] + t[x];
                w[x] += tk;
                kn = fmaf(tk, tk, kn);
            }
        }
        float* hd = s_hd + h * 8;
        hd[0] = qb[0];
        hd[1] = qb[1];
        hd[2] = qb[2];
        hd[3] = w[0];
        hd[4] = w[1];
        hd[5] = w[2];
        hd[6] = kn;
    }
    __syncthreads();

    const int g0 = c + 3 * Nq, zq = d.zq, qk_used = d.dqk_used;
    const int v_pair = c + rdz, v_used = d.dv_used;
    const int rowlen = 2 * d.dqk_pad + d.dv_pad;
    const bool vec = (c % 4) == 0 && (rdz % 4) == 0 && (d.d_z % 4) == 0;
    for (int h = warp; h < H; h += nw) {
        const float g = a.head_g[h];
        const float* hd = s_hd + h * 8;
        const float cb = valid ? kL2E * (-0.5f * g * hd[6]) : kMaskedBias;
        __nv_bfloat16* q = s_out + h * rowlen;
        __nv_bfloat16* k = q + d.dqk_pad;
        __nv_bfloat16* v = k + d.dqk_pad;
        // column recipe of one q_hat / k_hat element (pack.cu header); used for the 21 geometric
        // columns and, for shapes without 4-aligned blocks, for every column
        auto qk_col = [&](int cc, float& qv, float& kv) {
            if (cc < c) {
                qv = kL2E * s_proj[off_q + h * c + cc];
                kv = a.k_scale * s_proj[off_k + h * c + cc];
            } else if (cc < g0) {
                qv = kL2E * s_rq[h * Nq * 3 + (cc - c)];
                kv = g * s_rk[h * Nq * 3 + (cc - c)];
            } else if (cc < zq) {
                const int e = cc - g0;
                const int x = e % 3;
                if (e < 9) {
                    const float qq = kL2E * hd[x], tt = g * t[x];
                    qv = e < 6 ? hi_part<__nv_bfloat16>(qq) : lo_part<__nv_bfloat16>(qq);
                    kv = (e >= 3 && e < 6) ? lo_part<__nv_bfloat16>(tt) : hi_part<__nv_bfloat16>(tt);
                } else if (e < 18) {
                    const float tq = kL2E * t[x], ww = g * hd[3 + x];
                    qv = (e >= 12 && e < 15) ? lo_part<__nv_bfloat16>(tq) : hi_part<__nv_bfloat16>(tq);
                    kv = e < 15 ? hi_part<__nv_bfloat16>(ww) : lo_part<__nv_bfloat16>(ww);
                } else if (e < 20) {
                    qv = 1.0f;
                    kv = e == 18 ? hi_part<__nv_bfloat16>(cb) : (valid ? lo_part<__nv_bfloat16>(cb) : 0.f);
                } else {
                    qv = 0.f;
                    kv = e == 20 ? 1.0f : 0.f;
                }
            } else if (cc < qk_used) {
                const int e = cc - zq;
                qv = kL2E * s_z1[e];
                kv = a.wl_bias[h * d.d_z + (e % d.d_z)] * s_z2[e];
            } else {
                qv = 0.f;
                kv = 0.f;
            }
        };
        auto v_col = [&](int cc) {
            if (cc < c) return s_proj[off_v + h * c + cc];
            if (cc < v_pair) return s_z2[cc - c];
            if (cc < v_pair + 3) return hi_part<__nv_bfloat16>(t[cc - v_pair]);
            if (cc < v_pair + 6) return lo_part<__nv_bfloat16>(t[cc - v_pair - 3]);
            if (cc < v_used) return s_rv[h * Nv * 3 + (cc - v_pair - 6)];
            return 0.f;
        };
        if (vec) {
            // segment-wise: 4 columns per lane step with 8-byte shared stores, no per-element branching
            const float* pq = s_proj + off_q + h * c;
            const float* pk = s_proj + off_k + h * c;
            const float* pv = s_proj + off_v + h * c;
            for (int j = lane; 4 * j < c; j += 32) {
                const float4 x = *reinterpret_cast<const float4*>(pq + 4 * j);
                const float4 y = *reinterpret_cast<const float4*>(pk + 4 * j);
                const float4 z = *reinterpret_cast<const float4*>(pv + 4 * j);
                const float ks = a.k_scale;
                *reinterpret_cast<uint2*>(q + 4 * j) = make_uint2(pack2(kL2E * x.x, kL2E * x.y), pack2(kL2E * x.z, kL2E * x.w));
                *reinterpret_cast<uint2*>(k + 4 * j) = make_uint2(pack2(ks * y.x, ks * y.y), pack2(ks * y.z, ks * y.w));
                *reinterpret_cast<uint2*>(v + 4 * j) = make_uint2(pack2(z.x, z.y), pack2(z.z, z.w));
            }
            for (int cc = c + lane; cc < zq; cc += 32) {  // rotated points + geometric columns
                float qv, kv;
                qk_col(cc, qv, kv);
                q[cc] = __float2bfloat16_rn(qv);
                k[cc] = __float2bfloat16_rn(kv);
            }
            const float* wb = a.wl_bias + h * d.d_z;
            for (int j = lane; 4 * j < rdz; j += 32) {  // pair factors (zq % 8 == 0, c % 4 == 0)
                const float4 z1v = *reinterpret_cast<const float4*>(s_z1 + 4 * j);
                const float4 z2v = *reinterpret_cast<const float4*>(s_z2 + 4 * j);
                const float4 w4 = __ldg(reinterpret_cast<const float4*>(wb + (4 * j) % d.d_z));
                *reinterpret_cast<uint2*>(q + zq + 4 * j) =
                    make_uint2(pack2(kL2E * z1v.x, kL2E * z1v.y), pack2(kL2E * z1v.z, kL2E * z1v.w));
                *reinterpret_cast<uint2*>(k + zq + 4 * j) =
                    make_uint2(pack2(w4.x * z2v.x, w4.y * z2v.y), pack2(w4.z * z2v.z, w4.w * z2v.w));
                *reinterpret_cast<uint2*>(v + c + 4 * j) = make_uint2(pack2(z2v.x, z2v.y), pack2(z2v.z, z2v.w));
            }
            for (int cc = qk_used + lane; cc < d.dqk_pad; cc += 32) {
                q[cc] = __float2bfloat16_rn(0.f);
                k[cc] = __float2bfloat16_rn(0.f);
            }
            for (int cc = v_pair + lane; cc < d.dv_pad; cc += 32) v[cc] = __float2bfloat16_rn(v_col(cc));
        } else {
            for (int col = 2 * lane; col < d.dqk_pad; col += 64) {
                float q0, k0, q1, k1;
                qk_col(col, q0, k0);
                qk_col(col + 1, q1, k1);
                store_pair<__nv_bfloat16>(q + col, q0, q1);
                store_pair<__nv_bfloat16>(k + col, k0, k1);
            }
            for (int col = 2 * lane; col < d.dv_pad; col += 64)
                store_pair<__nv_bfloat16>(v + col, v_col(col), v_col(col + 1));
        }
        if (lane == 0) a.colbias[(static_cast<int64_t>(b) * H + h) * a.L + i] = valid ? -0.5f * g * hd[6] : -INFINITY;
    }
    __syncthreads();
    // 16-byte coalesced copy-out: per head q_hat, k_hat (dqk_pad) and v_hat (dv_pad) rows
    const int nq16 = d.dqk_pad / 8, nv16 = d.dv_pad / 8, per_head = 2 * nq16 + nv16;
    for (int e = threadIdx.x; e < H * per_head; e += blockDim.x) {
        const int h = e / per_head, r = e - h * per_head;
        const int64_t hrow = (static_cast<int64_t>(b) * H + h) * a.L + i;
        const uint4 val = reinterpret_cast<const uint4*>(s_out + h * rowlen)[r];
        if (r < nq16) {
            reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.qhat) + hrow * d.dqk_pad)[r] = val;
        } else if (r < 2 * nq16) {
            reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.khat) + hrow * d.dqk_pad)[r - nq16] = val;
        } else {
            reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.vhat) + hrow * d.dv_pad)[r - 2 * nq16] = val;
        }
    }
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                   int64_t n) {
    const int64_t n4 = n / 4;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n4;
         e += int64_t(gridDim.x) * blockDim.x) {
        const float4 v = reinterpret_cast<const float4*>(in)[e];
        __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&lo);
        w.y = *reinterpret_cast<uint32_t*>(&hi);
        reinterpret_cast<uint2*>(out)[e] = w;
    }
    for (int64_t e = n4 * 4 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
         e += int64_t(gridDim.x) * blockDim.x) {
        out[e] = __float2bfloat16_rn(in[e]);
    }
}

__global__ void f32_to_bf16_2d_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                      int64_t rows, int cols, int ld_out) {
    const int64_t n = rows * cols;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / cols;
        out[r * ld_out + (e - r * cols)] = __float2bfloat16_rn(in[e]);
    }
}

// Block-wide: translations of sample b minus the centroid of its valid residues.
__device__ __forceinline__ void recenter_sample(const float* __restrict__ trans, const uint8_t* __restrict__ mask,
                                                float* __restrict__ out, int L, int b) {
    __shared__ float red[4][32];
    const float* t = trans + int64_t(b) * L * 3;
    float sx = 0.f, sy = 0.f, sz = 0.f, cnt = 0.f;
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        const bool ok = mask == nullptr || mask[int64_t(b) * L + i] != 0;
        if (ok) {
            sx += t[i * 3 + 0];
            sy += t[i * 3 + 1];
            sz += t[i * 3 + 2];
            cnt += 1.f;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        sx += __shfl_xor_sync(0xffffffffu, sx, o);
        sy += __shfl_xor_sync(0xffffffffu, sy, o);
        sz += __shfl_xor_sync(0xffffffffu, sz, o);
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        red[0][w] = sx;
        red[1][w] = sy;
        red[2][w] = sz;
        red[3][w] = cnt;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const int nw = blockDim.x >> 5;
        float v[4];
        for (int k = 0; k < 4; ++k) {
            v[k] = l < nw ? red[k][l] : 0.f;
            for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
        }
        if (l == 0) {
            const float n = v[3] > 0.f ? v[3] : 1.f;
            red[0][0] = v[0] / n;
            red[1][0] = v[1] / n;
            red[2][0] = v[2] / n;
        }
    }
    __syncthreads();
    const float cx = red[0][0], cy = red[1][0], cz = red[2][0];
    float* o = out + int64_t(b) * L * 3;
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        o[i * 3 + 0] = t[i * 3 + 0] - cx;
        o[i * 3 + 1] = t[i * 3 + 1] - cy;
        o[i * 3 + 2] = t[i * 3 + 2] - cz;
    }
}

// Inputs of the fused projection + pack kernel in one pass: s -> bf16 rows of din_ld, and the
// head-independent pair-factor column blocks of the lifted rows, bf16(log2(e) z1) (q_hat) and
// bf16(z2) (v_hat; k_hat scales it per head), so proj_pack copies them instead of converting the
// fp32 rows once per head and tensor.  float4 loads, 8-byte stores; thread = 4 columns.
__global__ void cast_inputs_kernel(const float* __restrict__ s, __nv_bfloat16* __restrict__ s_bf16, int d_in,
                                   int din_ld, const float* __restrict__ z1, const float* __restrict__ z2,
                                   __nv_bfloat16* __restrict__ z1q, __nv_bfloat16* __restrict__ z2b, int rdz,
                                   int64_t rows, const float* __restrict__ trans, const uint8_t* __restrict__ mask,
                                   float* __restrict__ trans_c, int L, int nrec) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    // the first nrec blocks also recentre one sample's translations each (one launch instead of two)
    if (static_cast<int>(blockIdx.x) < nrec) recenter_sample(trans, mask, trans_c, L, blockIdx.x);
    const int q_s = (d_in + 3) / 4, q_z = rdz / 4;
    const bool vec_s = d_in % 4 == 0;
    const int64_t n_s = rows * q_s, n = n_s + 2 * rows * q_z;
    // kUnroll float4 loads of one thread in flight before their stores (a grid-stride loop of one
    // load each kept ~1/3 of the HBM bandwidth busy)
    constexpr int kUnroll = 4;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    auto locate = [&](int64_t e, const float*& src, __nv_bfloat16*& dst, float& sc) {
        sc = 1.f;
        if (e < n_s) {
            const int64_t r = e / q_s;
            const int c4 = int(e - r * q_s);
            src = s + r * d_in + 4 * c4;
            dst = s_bf16 + r * din_ld + 4 * c4;
        } else {
            const int64_t f = e - n_s;
            const bool second = f >= rows * q_z;
            const int64_t g = second ? f - rows * q_z : f;
            src = (second ? z2 : z1) + 4 * g;
            dst = (second ? z2b : z1q) + 4 * g;
            sc = second ? 1.f : 1.4426950408889634f;
        }
    };
    for (int64_t e0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e0 < n; e0 += kUnroll * stride) {
        float4 v[kUnroll];
        __nv_bfloat16* dst[kUnroll];
        float sc[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int64_t e = e0 + u * stride;
            dst[u] = nullptr;
            if (e < n) {
                const float* src;
                locate(e, src, dst[u], sc[u]);
                if (e < n_s && !vec_s) {  // unaligned rows: element-wise
                    const int c4 = int(e - (e / q_s) * q_s);
                    for (int k = 0; k < 4 && 4 * c4 + k < d_in; ++k) dst[u][k] = __float2bfloat16_rn(src[k]);
                    dst[u] = nullptr;
                } else {
                    v[u] = __ldg(reinterpret_cast<const float4*>(src));
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
            if (dst[u] != nullptr)
                *reinterpret_cast<uint2*>(dst[u]) = make_uint2(ptx::pack_bf16x2(sc[u] * v[u].x, sc[u] * v[u].y),
                                                               ptx::pack_bf16x2(sc[u] * v[u].z, sc[u] * v[u].w));
    }
}

// One block per sample: subtract the centroid of the valid residues' translations.
// 3xTF32 operand split (fp32 path): each element x becomes hi = tf32(x) and lo = x - hi (exact),
// written into up to three K-concatenated parts (or planes) per row.
__device__ __forceinline__ float tf32_round(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__global__ void split3_kernel(const float* __restrict__ in, int64_t rows, int cols, int64_t ld_in,
                              float* __restrict__ out, int ld_part, int64_t ld_out, int lo_mask, int nparts,
                              int64_t plane) {
    const int64_t n = rows * ld_part;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = e / ld_part;
        const int c = static_cast<int>(e - r * ld_part);
        const float x = c < cols ? in[r * ld_in + c] : 0.f;
        const float hi = tf32_round(x), lo = x - hi;
        for (int p = 0; p < nparts; ++p) {
            const float v = (lo_mask >> p) & 1 ? lo : hi;
            if (plane) out[p * plane + r * ld_part + c] = v;
            else out[r * ld_out + int64_t(p) * ld_part + c] = v;
        }
    }
}

// Transposing hi/lo split of v_hat: in [BH][L][D] -> out planes [2][BH][D][Lp] (keys contiguous:
// the K-major B operand of the 3xTF32 P.V products).  32 x 32 tiles through shared memory.
__global__ void split_t_kernel(const float* __restrict__ in, int L, int D, float* __restrict__ out, int Lp,
                               int64_t plane) {
    __shared__ float tile[32][33];
    const int bh = blockIdx.z;
    const int l0 = blockIdx.x * 32, d0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
    const float* src = in + static_cast<int64_t>(bh) * L * D;
    for (int r = ty; r < 32; r += 8) {
        const int l = l0 + r, d = d0 + tx;
        tile[r][tx] = (l < L && d < D) ? src[static_cast<int64_t>(l) * D + d] : 0.f;
    }
    __syncthreads();
    float* dst = out + static_cast<int64_t>(bh) * D * Lp;
    for (int r = ty; r < 32; r += 8) {
        const int d = d0 + r, l = l0 + tx;
        if (d < D && l < Lp) {
            const float x = tile[tx][r];
            const float hi = tf32_round(x);
            dst[static_cast<int64_t>(d) * Lp + l] = hi;
            dst[plane + static_cast<int64_t>(d) * Lp + l] = x - hi;
        }
    }
}

__global__ void add_inplace_kernel(float* __restrict__ acc, const float* __restrict__ x, int64_t n) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x)
        acc[e] += x[e];
}

// fully_masked flags (proj/src/flash_ipa.cpp:156-158): every row of a sample without a valid
// residue is flagged (its output is all zeros); one block per sample.
__global__ void fully_masked_kernel(const uint8_t* __restrict__ mask, uint8_t* __restrict__ flags, int L) {
    const int b = blockIdx.x;
    int any = 0;
    for (int i = threadIdx.x; i < L && !any; i += blockDim.x) any = mask == nullptr || mask[int64_t(b) * L + i] != 0;
    any = __syncthreads_or(any);
    for (int i = threadIdx.x; i < L; i += blockDim.x) flags[int64_t(b) * L + i] = any ? 0 : 1;
}


__global__ void recenter_kernel(const float* __restrict__ trans, const uint8_t* __restrict__ mask,
                                float* __restrict__ out, int L) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    recenter_sample(trans, mask, out, L, blockIdx.x);
}

// Query-row sharding: per-sample partial sums {sum x, sum y, sum z, count} of the valid local
// translations (all-reduced across shards by the caller), then recentring with the global sums.
__global__ void centroid_sums_kernel(const float* __restrict__ trans, const uint8_t* __restrict__ mask,
                                     float* __restrict__ sums, int L) {
    __shared__ float red[4][32];
    const int b = blockIdx.x;
    const float* t = trans + int64_t(b) * L * 3;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        if (mask == nullptr || mask[int64_t(b) * L + i] != 0) {
            v[0] += t[i * 3];
            v[1] += t[i * 3 + 1];
            v[2] += t[i * 3 + 2];
            v[3] += 1.f;
        }
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    for (int k = 0; k < 4; ++k) {
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
        if (l == 0) red[k][w] = v[k];
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        float acc = 0.f;
        for (int k = 0; k < int(blockDim.x >> 5); ++k) acc += red[threadIdx.x][k];
        sums[b * 4 + threadIdx.x] = acc;
    }
}

__global__ void recenter_with_sums_kernel(const float* __restrict__ trans, const float* __restrict__ sums,
                                          const uint8_t* __restrict__ zero_masked, float* __restrict__ out, int L) {
    const int b = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= L) return;
    const float n = sums[b * 4 + 3] > 0.f ? sums[b * 4 + 3] : 1.f;
    const int64_t r = (int64_t(b) * L + i) * 3;
    const bool zero = zero_masked != nullptr && zero_masked[int64_t(b) * L + i] == 0;
    for (int x = 0; x < 3; ++x) out[r + x] = zero ? 0.f : trans[r + x] - sums[b * 4 + x] / n;
}

// Trunk step (BASELINE cfg3, oracle/fipa_oracle.py trunk_forward): s <- s + ipa_out, then the
// backbone update u = s.W_bb + b_bb, dR = R(normalised (1, u0, u1, u2)) (proj/src/geometry.cpp:
// 107-132 matrix), T <- compose(T, (dR, u[3:6])) = (R dR, R u[3:6] + t) (geometry.cpp:78-90).
// One warp per residue; masked residues keep their frames (their IPA output is already zero).
__global__ void trunk_update_kernel(float* __restrict__ s, const float* __restrict__ ipa_out,
                                    const float* __restrict__ w_bb, const float* __restrict__ b_bb,
                                    float* __restrict__ rot, float* __restrict__ trans,
                                    const uint8_t* __restrict__ mask, int64_t rows, int d_in) {
    const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    float u[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int k = lane; k < d_in; k += 32) {
        const float v = s[row * d_in + k] + ipa_out[row * d_in + k];
        s[row * d_in + k] = v;
#pragma unroll
        for (int j = 0; j < 6; ++j) u[j] = fmaf(v, w_bb[k * 6 + j], u[j]);
    }
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        for (int o = 16; o > 0; o >>= 1) u[j] += __shfl_xor_sync(0xffffffffu, u[j], o);
        u[j] += b_bb[j];
    }
    if (lane != 0 || (mask != nullptr && mask[row] == 0)) return;
    const float n = sqrtf(1.f + u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
    const float qw = 1.f / n, qx = u[0] / n, qy = u[1] / n, qz = u[2] / n;
    const float d[9] = {1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qw * qz), 2 * (qx * qz + qw * qy),
                        2 * (qx * qy + qw * qz), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qw * qx),
                        2 * (qx * qz - qw * qy), 2 * (qy * qz + qw * qx), 1 - 2 * (qx * qx + qy * qy)};
    float R[9], nr[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = rot[row * 9 + k];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) nr[3 * a + c] = R[3 * a] * d[c] + R[3 * a + 1] * d[3 + c] + R[3 * a + 2] * d[6 + c];
#pragma unroll
    for (int a = 0; a < 3; ++a)
        trans[row * 3 + a] += R[3 * a] * u[3] + R[3 * a + 1] * u[4] + R[3 * a + 2] * u[5];
#pragma unroll
    for (int k = 0; k < 9; ++k) rot[row * 9 + k] = nr[k];
}

}  // namespace

void launch_trunk_update(float* s, const float* ipa_out, const float* w_bb, const float* b_bb, float* rot,
                         float* trans, const uint8_t* mask, int64_t rows, int d_in, cudaStream_t stream) {
    const int64_t threads = rows * 32;
    trunk_update_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, stream>>>(s, ipa_out, w_bb, b_bb, rot,
                                                                                          trans, mask, rows, d_in);
}

void launch_centroid_sums(const float* trans, const uint8_t* mask, float* sums, int B, int L, cudaStream_t stream) {
    centroid_sums_kernel<<<B, 256, 0, stream>>>(trans, mask, sums, L);
}

void launch_recenter_with_sums(const float* trans, const float* sums, float* out, int B, int L, cudaStream_t stream,
                               const uint8_t* zero_masked) {
    dim3 grid((L + 255) / 256, B);
    recenter_with_sums_kernel<<<grid, 256, 0, stream>>>(trans, sums, zero_masked, out, L);
}

void launch_pack(const LayerDims& d, const PackArgs& a, cudaStream_t stream) {
    const int rdz = d.rank * d.d_z;
    const dim3 grid(static_cast<unsigned>(int64_t(a.B) * a.L));
    if (a.out_f32) {
        const size_t smem =
            sizeof(float) * (d.n_proj + 2 * rdz + d.heads * (d.n_query * 6 + d.n_value * 3) + 8 * d.heads);
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(pack_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        pack_kernel<float><<<grid, 256, smem, stream>>>(d, a);
        return;
    }
    if (d.dqk_pad % 8 || d.dv_pad % 8) throw std::invalid_argument("pack: padded widths must be multiples of 8");
    const size_t smem = sizeof(float) * (((d.n_proj + 3) & ~3) + 2 * ((rdz + 3) & ~3) +
                                         d.heads * (d.n_query * 6 + d.n_value * 3) + 8 * d.heads) +
                        16 + 2 * size_t(d.heads) * (2 * d.dqk_pad + d.dv_pad) + 16;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(pack_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    pack_bf16_kernel<<<grid, 256, smem, stream>>>(d, a);
}

void launch_f32_to_bf16(const float* in, __nv_bfloat16* out, int64_t n, cudaStream_t stream) {
    if (n <= 0) return;
    const int64_t blocks = std::min<int64_t>((n / 4 + 255) / 256 + 1, 148 * 16);
    f32_to_bf16_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(in, out, n);
}

void launch_f32_to_bf16_2d(const float* in, __nv_bfloat16* out, int64_t rows, int cols, int ld_out,
                           cudaStream_t stream) {
    if (cols == ld_out) return launch_f32_to_bf16(in, out, rows * cols, stream);
    const int64_t n = rows * cols;
    if (n <= 0) return;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
    f32_to_bf16_2d_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(in, out, rows, cols, ld_out);
}

bool cast_inputs_supported(int, int din_ld, int rdz) { return din_ld % 4 == 0 && rdz % 4 == 0; }

void launch_cast_inputs(const float* s, __nv_bfloat16* s_bf16, int d_in, int din_ld, const float* z1, const float* z2,
                        __nv_bfloat16* z1q, __nv_bfloat16* z2b, int rdz, int64_t rows, cudaStream_t stream,
                        const float* trans, const uint8_t* mask, float* trans_c, int B, int L) {
    if (!cast_inputs_supported(d_in, din_ld, rdz)) throw std::invalid_argument("cast_inputs: widths must be multiples of 4");
    if (din_ld > d_in) cudaMemsetAsync(s_bf16, 0, size_t(rows) * din_ld * 2, stream);  // padding columns
    const int64_t n = rows * ((d_in + 3) / 4 + 2 * (rdz / 4));
    if (n <= 0) return;
    const int nrec = trans != nullptr ? B : 0;
    const int64_t blocks = std::max<int64_t>(nrec, std::min<int64_t>((n + 255) / 256, int64_t(device_sm_count()) * 8));
    launch_pdl(cast_inputs_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, stream, s, s_bf16, d_in, din_ld,
               z1, z2, z1q, z2b, rdz, rows, trans, mask, trans_c, L, nrec);
}

void launch_split3(const float* in, int64_t rows, int cols, int64_t ld_in, float* out, int ld_part, int64_t ld_out,
                   int lo_mask, int nparts, cudaStream_t stream, int64_t plane) {
    const int64_t n = rows * ld_part;
    if (n <= 0) return;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, int64_t(device_sm_count()) * 16);
    split3_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(in, rows, cols, ld_in, out, ld_part, ld_out,
                                                                      lo_mask, nparts, plane);
}

void launch_split_t(const float* in, int BH, int L, int D, float* out, int Lp, int64_t plane, cudaStream_t stream) {
    dim3 grid((Lp + 31) / 32, (D + 31) / 32, BH);
    split_t_kernel<<<grid, 256, 0, stream>>>(in, L, D, out, Lp, plane);
}

void launch_add_inplace(float* acc, const float* x, int64_t n, cudaStream_t stream) {
    if (n <= 0) return;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, int64_t(device_sm_count()) * 8);
    add_inplace_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(acc, x, n);
}

void launch_fully_masked(const uint8_t* mask, uint8_t* flags, int B, int L, cudaStream_t stream) {
    fully_masked_kernel<<<B, 256, 0, stream>>>(mask, flags, L);
}

void launch_recenter(const float* trans, const uint8_t* mask, float* out, int B, int L,
                     cudaStream_t stream) {
    launch_pdl(recenter_kernel, dim3(B), dim3(1024), 0, stream, trans, mask, out, L);  // one block per sample
}

}  // namespace fipa_b200
