// FlashIPA attention forward on tcgen05 tensor cores, with the output epilogue fused.
//
// Replaces the reference's tiled online-softmax kernel
//   flash_attention -> flash_block   proj/src/attention_kernel.cpp:112-188, 213-243
// and the per-row epilogue that follows it
//   split / pair contraction / apply_inverse / norms   proj/src/flash_ipa.cpp:171-210
//
// One CTA = one (sample, head, 128-query tile).  Per KV tile of 64 keys:
//   S  = Q_hat . K_hat^T      tcgen05.mma SS, M=128 N=64, K=dqk_pad   -> TMEM cols [448,512)
//   P  = exp2(S*log2e + colbias*log2e - m)   softmax warps, fp32; P (bf16) -> TMEM cols [448,480)
//   O += P . V_hat            tcgen05.mma TS (A = P from TMEM), N = dv_pad (<=256 + rest)
//                                                                -> TMEM cols [0, dv_pad)
// Key mask -> -inf colbias, rows with no valid key -> zeros (attention_kernel.cpp:140-143,
// 184-186).  The running max is only moved when it grows by more than 2^8 (the P values stay
// <= 256, exact in fp32 and representable in bf16), so the O rescale through TMEM is rare.
//
// Warp roles (192 threads): w0 TMA producer, w1 TMEM alloc + MMA issue, w2..w5 softmax and
// epilogue (warp w owns TMEM lanes 32*(w%4).., thread = query row).
// SMEM: Q resident [n_qkb][128 rows][128 B], K [n_qkb][64][128 B], V [n_vb][64 keys][128 B]
// (all SWIZZLE_128B; K-major for Q/K, MN-major for V).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <stdexcept>

#include "kernels.hpp"
#include "ptx.cuh"
#include "tma_host.hpp"

namespace fipa_b200 {

namespace {

constexpr int BM = 128;
constexpr int BN = 64;
constexpr int kThreads = 192;
constexpr uint32_t kSCol = 448;  // S / P region in TMEM
constexpr int kMaxPts = 48;      // 3*Nv + 6 handled by the fused epilogue
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

struct AttnParams {
    int L, H, dqk_pad, dv_pad, n_qkb, n_vb;
    int c, d_z, rank, n_value, seg, feat;
    const float* colbias;
    const float* z1;
    const float* rot;
    const float* trans;
    __nv_bfloat16* feat_out;
    float* lse;
};

struct Bars {
    uint64_t q_full, k_full, k_empty, v_full, v_empty, s_full, p_full, pv_done, o_full;
    uint32_t tmem_slot;
};

__device__ __forceinline__ void st_bf16(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap mapQ,
                    const __grid_constant__ CUtensorMap mapK,
                    const __grid_constant__ CUtensorMap mapV, AttnParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + p.n_qkb * (BM * 128);
    uint8_t* sV = sK + p.n_qkb * (BN * 128);
    Bars* bars = reinterpret_cast<Bars*>(sV + p.n_vb * (BN * 128));

    const int warp = ptx::warp_id();
    const int lane = ptx::lane_id();
    const int bh = blockIdx.y;
    const int q0 = blockIdx.x * BM;
    const int ntiles = (p.L + BN - 1) / BN;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&mapQ);
        ptx::tma_prefetch(&mapK);
        ptx::tma_prefetch(&mapV);
        ptx::mbar_init(&bars->q_full, 1);
        ptx::mbar_init(&bars->k_full, 1);
        ptx::mbar_init(&bars->k_empty, 1);
        ptx::mbar_init(&bars->v_full, 1);
        ptx::mbar_init(&bars->v_empty, 1);
        ptx::mbar_init(&bars->s_full, 1);
        ptx::mbar_init(&bars->p_full, 128);
        ptx::mbar_init(&bars->pv_done, 1);
        ptx::mbar_init(&bars->o_full, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(&bars->tmem_slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = bars->tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            ptx::mbar_expect_tx(&bars->q_full, p.n_qkb * BM * 128);
            for (int b = 0; b < p.n_qkb; ++b)
                ptx::tma_load_3d(sQ + b * BM * 128, &mapQ, &bars->q_full, b * 64, q0, bh);
            for (int j = 0; j < ntiles; ++j) {
                if (j > 0) ptx::mbar_wait(&bars->k_empty, (j - 1) & 1);
                ptx::mbar_expect_tx(&bars->k_full, p.n_qkb * BN * 128);
                for (int b = 0; b < p.n_qkb; ++b)
                    ptx::tma_load_3d(sK + b * BN * 128, &mapK, &bars->k_full, b * 64, j * BN, bh);
                if (j > 0) ptx::mbar_wait(&bars->v_empty, (j - 1) & 1);
                ptx::mbar_expect_tx(&bars->v_full, p.n_vb * BN * 128);
                for (int b = 0; b < p.n_vb; ++b)
                    ptx::tma_load_3d(sV + b * BN * 128, &mapV, &bars->v_full, b * 64, j * BN, bh);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc_qk = ptx::idesc_bf16(BM, BN, false, false);
            const int n1 = p.dv_pad < 256 ? p.dv_pad : 256;
            const int n2 = p.dv_pad - n1;
            const uint32_t idesc_pv1 = ptx::idesc_bf16(BM, n1, false, true);
            const uint32_t idesc_pv2 = ptx::idesc_bf16(BM, n2 > 0 ? n2 : 16, false, true);
            const uint32_t q_base = ptx::smem_u32(sQ);
            const uint32_t k_base = ptx::smem_u32(sK);
            const uint32_t v_base = ptx::smem_u32(sV);
            const int qk_steps = p.dqk_pad / 16;
            ptx::mbar_wait(&bars->q_full, 0);
            for (int j = 0; j < ntiles; ++j) {
                ptx::mbar_wait(&bars->k_full, j & 1);
                if (j > 0) ptx::mbar_wait(&bars->pv_done, (j - 1) & 1);
                ptx::tc_fence_after();
                for (int kk = 0; kk < qk_steps; ++kk) {
                    const uint32_t blk = kk >> 2, sub = (kk & 3) * 32;
                    const uint64_t da = ptx::sw128_desc(q_base + blk * (BM * 128) + sub, 16, 1024);
                    const uint64_t db = ptx::sw128_desc(k_base + blk * (BN * 128) + sub, 16, 1024);
                    ptx::mma_ss(tmem + kSCol, da, db, idesc_qk, kk > 0);
                }
                ptx::mma_commit(&bars->k_empty);
                ptx::mma_commit(&bars->s_full);
                ptx::mbar_wait(&bars->p_full, j & 1);
                ptx::mbar_wait(&bars->v_full, j & 1);
                ptx::tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < BN / 16; ++kk) {
                    const uint32_t a_tm = tmem + kSCol + kk * 8;
                    const uint64_t db1 = ptx::sw128_desc(v_base + kk * 2048, BN * 128, 1024);
                    ptx::mma_ts(tmem, a_tm, db1, idesc_pv1, (j > 0 || kk > 0));
                    if (n2 > 0) {
                        const uint64_t db2 =
                            ptx::sw128_desc(v_base + 4 * (BN * 128) + kk * 2048, BN * 128, 1024);
                        ptx::mma_ts(tmem + 256, a_tm, db2, idesc_pv2, (j > 0 || kk > 0));
                    }
                }
                ptx::mma_commit(&bars->v_empty);
                ptx::mma_commit(&bars->pv_done);
            }
            ptx::mma_commit(&bars->o_full);
        }
    } else {
        // ------------------------------------------------- softmax + fused epilogue
        const int quad = warp & 3;
        const int row = quad * 32 + lane;
        const int qi = q0 + row;
        const uint32_t tl = tmem + (uint32_t(quad * 32) << 16);
        const float* cbp = p.colbias + static_cast<int64_t>(bh) * p.L;
        float m = -INFINITY;  // running max, log2 domain
        float l = 0.f;
        for (int j = 0; j < ntiles; ++j) {
            ptx::mbar_wait(&bars->s_full, j & 1);
            ptx::tc_fence_after();
            uint32_t sr[64];
            ptx::tmem_ld32(tl + kSCol, sr);
            ptx::tmem_ld32(tl + kSCol + 32, sr + 32);
            ptx::tmem_wait_ld();
            float x[64];
            float mt = -INFINITY;
            const int key0 = j * BN;
#pragma unroll
            for (int cc = 0; cc < 64; ++cc) {
                const int key = key0 + cc;
                const float cb = key < p.L ? __ldg(cbp + key) : -INFINITY;
                x[cc] = fmaf(__uint_as_float(sr[cc]), kLog2e, cb * kLog2e);
                mt = fmaxf(mt, x[cc]);
            }
            const bool need = mt > m + 8.0f;  // true when m == -inf and mt finite
            float scale = 1.0f;
            if (need) {
                scale = exp2f(m - mt);  // 0 when m == -inf
                m = mt;
                l *= scale;
            }
            if (j > 0 && __any_sync(0xffffffffu, need)) {
                for (int c0 = 0; c0 < p.dv_pad; c0 += 16) {
                    uint32_t o[16];
                    ptx::tmem_ld16(tl + c0, o);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * scale);
                    ptx::tmem_st16(tl + c0, o);
                }
                ptx::tmem_wait_st();
            }
            const float mm = m == -INFINITY ? 0.f : m;
            uint32_t pk[32];
            float ls = 0.f;
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) {
                const float p0 = exp2f(x[2 * cc] - mm);
                const float p1 = exp2f(x[2 * cc + 1] - mm);
                ls += p0 + p1;
                pk[cc] = ptx::pack_bf16x2(p0, p1);
            }
            l += ls;
            ptx::tmem_st32(tl + kSCol, pk);
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            ptx::mbar_arrive(&bars->p_full);
        }

        // ------------------------------------------------------------- epilogue
        ptx::mbar_wait(&bars->o_full, 0);
        ptx::tc_fence_after();
        const bool ok = qi < p.L;
        const float inv_l = l > 0.f ? 1.0f / l : 0.f;
        const int H = p.H;
        const int b = bh / H, h = bh % H;
        const int64_t grow = static_cast<int64_t>(b) * p.L + (ok ? qi : 0);
        if (ok) p.lse[static_cast<int64_t>(bh) * p.L + qi] = l > 0.f ? (m + log2f(l)) * kLn2 : -INFINITY;
        __nv_bfloat16* fo = p.feat_out + grow * p.feat + h * p.seg;
        const float* z1r = p.z1 + grow * (p.rank * p.d_z);
        // scalar aggregate -> block [d_z, d_z + c)
        for (int c0 = 0; c0 < p.c; c0 += 32) {
            uint32_t r[32];
            ptx::tmem_ld32(tl + c0, r);
            ptx::tmem_wait_ld();
            if (ok) {
                for (int e = 0; e < 32 && c0 + e < p.c; ++e)
                    st_bf16(fo + p.d_z + c0 + e, __uint_as_float(r[e]) * inv_l);
            }
        }
        // pair contraction: o~[d] = sum_rho z1[i,rho,d] * O[c + rho*d_z + d]  -> block [0, d_z)
        for (int d0 = 0; d0 < p.d_z; d0 += 32) {
            float acc[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) acc[e] = 0.f;
            for (int rho = 0; rho < p.rank; ++rho) {
                uint32_t r[32];
                ptx::tmem_ld32(tl + p.c + rho * p.d_z + d0, r);
                ptx::tmem_wait_ld();
                if (ok) {
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const float zz = (d0 + e < p.d_z) ? z1r[rho * p.d_z + d0 + e] : 0.f;
                        acc[e] = fmaf(zz, __uint_as_float(r[e]), acc[e]);
                    }
                }
            }
            if (ok) {
                for (int e = 0; e < 32 && d0 + e < p.d_z; ++e) st_bf16(fo + d0 + e, acc[e] * inv_l);
            }
        }
        // points: O[c + r d_z + 3p + xyz] (R_j v_p aggregate) + translation aggregate (hi+lo)
        {
            const int base = p.c + p.rank * p.d_z;
            const int npt = 3 * p.n_value + 6;
            float pts[kMaxPts];
#pragma unroll
            for (int c0 = 0; c0 < kMaxPts; c0 += 16) {
                if (c0 < npt) {
                    uint32_t r[16];
                    ptx::tmem_ld16(tl + base + c0, r);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 16; ++e) pts[c0 + e] = __uint_as_float(r[e]);
                }
            }
            if (ok) {
                const int Nv = p.n_value;
                float R[9], t[3], ta[3];
#pragma unroll
                for (int k = 0; k < 9; ++k) R[k] = p.rot[grow * 9 + k];
#pragma unroll
                for (int k = 0; k < 3; ++k) t[k] = p.trans[grow * 3 + k];
                for (int k = 0; k < 3; ++k) ta[k] = (pts[3 * Nv + k] + pts[3 * Nv + 3 + k]) * inv_l;
                __nv_bfloat16* fp = fo + p.d_z + p.c;
                for (int q = 0; q < Nv; ++q) {
                    const float gx = pts[3 * q + 0] * inv_l + ta[0] - t[0];
                    const float gy = pts[3 * q + 1] * inv_l + ta[1] - t[1];
                    const float gz = pts[3 * q + 2] * inv_l + ta[2] - t[2];
                    // apply_inverse: R^T (g - t)   (proj/src/geometry.cpp:70-76)
                    const float lx = fmaf(R[0], gx, fmaf(R[3], gy, R[6] * gz));
                    const float ly = fmaf(R[1], gx, fmaf(R[4], gy, R[7] * gz));
                    const float lz = fmaf(R[2], gx, fmaf(R[5], gy, R[8] * gz));
                    st_bf16(fp + 3 * q + 0, lx);
                    st_bf16(fp + 3 * q + 1, ly);
                    st_bf16(fp + 3 * q + 2, lz);
                    st_bf16(fp + 3 * Nv + q, sqrtf(lx * lx + ly * ly + lz * lz));
                }
            }
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

}  // namespace

void launch_attn_fwd_tc(const LayerDims& d, const AttnArgs& a, cudaStream_t stream) {
    if (d.dqk_pad > 448 || d.dv_pad > 448)
        throw std::invalid_argument("tcgen05 attention: lifted width exceeds 448 (use precision='f32')");
    if (3 * d.n_value + 6 > kMaxPts)
        throw std::invalid_argument("tcgen05 attention: n_value > 14 unsupported (use precision='f32')");
    AttnParams p{};
    p.L = a.L;
    p.H = d.heads;
    p.dqk_pad = d.dqk_pad;
    p.dv_pad = d.dv_pad;
    p.n_qkb = (d.dqk_pad + 63) / 64;
    p.n_vb = (d.dv_pad + 63) / 64;
    p.c = d.c;
    p.d_z = d.d_z;
    p.rank = d.rank;
    p.n_value = d.n_value;
    p.seg = d.seg;
    p.feat = d.feat;
    p.colbias = a.colbias;
    p.z1 = a.z1;
    p.rot = a.rot;
    p.trans = a.trans;
    p.feat_out = a.feat;
    p.lse = a.lse;
    const uint64_t BH = static_cast<uint64_t>(a.B) * d.heads;
    const CUtensorMap mapQ = make_map_3d_bf16(a.qhat, d.dqk_pad, a.L, BH, d.dqk_pad, 64, BM);
    const CUtensorMap mapK = make_map_3d_bf16(a.khat, d.dqk_pad, a.L, BH, d.dqk_pad, 64, BN);
    const CUtensorMap mapV = make_map_3d_bf16(a.vhat, d.dv_pad, a.L, BH, d.dv_pad, 64, BN);
    const int smem = p.n_qkb * (BM * 128 + BN * 128) + p.n_vb * (BN * 128) + 1024 + 256;
    cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    dim3 grid((a.L + BM - 1) / BM, static_cast<unsigned>(BH));
    attn_fwd_kernel<<<grid, kThreads, smem, stream>>>(mapQ, mapK, mapV, p);
}

}  // namespace fipa_b200
