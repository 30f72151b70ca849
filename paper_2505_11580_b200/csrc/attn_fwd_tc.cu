// FlashIPA attention forward on tcgen05 tensor cores, with the output epilogue fused.
//
// Replaces the reference's tiled online-softmax kernel
//   flash_attention -> flash_block   proj/src/attention_kernel.cpp:112-188, 213-243
// and the per-row epilogue that follows it
//   split / pair contraction / apply_inverse / norms   proj/src/flash_ipa.cpp:171-210
//
// One CTA = one (sample, head, 128-query tile).  Per KV tile j of 64 keys:
//   S_j  = Q_hat . K_hat_j^T   tcgen05.mma SS, M=128 N=64 K=dqk_pad   -> TMEM cols [416,480)
//          (log2 units, column bias folded into two K columns, pack.cu)
//   P_j  = exp2(S_j - m)       softmax warps (fp32), bf16 -> TMEM cols [480,512)
//   O   += P_j . V_hat_j       tcgen05.mma TS (A = P from TMEM), N = dv_tc = 256 + 160
//                                                                     -> TMEM cols [0,416)
//   the <= 16 trailing value columns (dv_tc..dv_used) are accumulated by the softmax warps
//   on CUDA cores from the V tile in shared memory (the TMEM budget is 416 + 64 + 32 = 512).
// The tensor pipe runs QK_{j+1} while the softmax warps turn S_j into P_j (S and P have their
// own TMEM columns), then PV_j.  The running max moves only when it grows by more than 2^8, so
// the O rescale through TMEM is rare.  Key mask: masked keys carry a -1e30 column bias and
// vanish as soon as any valid key is seen; keys beyond L are forced to -inf; rows with no valid
// key are zeroed by the output projection (proj/src/flash_ipa.cpp:213-216).
//
// Warp roles (224 threads): w0 Q/K TMA producer, w1 TMEM alloc + MMA issue (elect.sync, so the
// descriptor math stays in uniform registers), w2..w5 softmax + epilogue (warp w owns TMEM lanes
// 32*(w%4).., one thread per query row), w6 V TMA producer.
// SMEM: Q resident [n_qkb][128 rows][128 B], K [n_qkb][64][128 B], V [n_vb][64 keys][128 B]
// (SWIZZLE_128B; K-major for Q/K, MN-major for V); reused as the epilogue staging buffer.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>

#include "kernels.hpp"
#include "ptx.cuh"
#include "tma_host.hpp"

namespace fipa_b200 {

namespace {

constexpr int BM = 128;
constexpr int BN = 64;
constexpr int kThreads = 224;
constexpr uint32_t kSCol = 416;  // S tile (64 fp32 columns)
constexpr uint32_t kPCol = 480;  // P tile (64 bf16 = 32 columns)
constexpr int kMaxSimt = 16;
constexpr float kLn2 = 0.6931471805599453f;

struct AttnParams {
    int L, H, dqk_mma, dv_tc, dv_simt, dv_used, n_qkb, n_vb;
    int c, d_z, rank, n_value, seg, feat_ld;
    const float* z1;
    const float* rot;
    const float* trans;
    __nv_bfloat16* feat_out;
    float* lse;
};

struct Bars {
    uint64_t q_full, k_full, k_empty, v_full, v_empty, s_full, s_free, p_full, pv_done, o_full;
    uint32_t tmem_slot;
};

// Optional per-event timestamps of CTA (0,0) for pipeline analysis (tools/attn_trace.cu).
#ifdef FIPA_ATTN_TRACE
__device__ long long g_attn_trace[16 * 256];
#define FIPA_TRACE(ev, j)                                                        \
    do {                                                                         \
        if (blockIdx.x == 0 && blockIdx.y == 0 && (j) < 256)                     \
            g_attn_trace[(ev) * 256 + (j)] = clock64();                          \
    } while (0)
#else
#define FIPA_TRACE(ev, j) \
    do {                  \
    } while (0)
#endif

__host__ __device__ constexpr int epilogue_smem(int seg) {
    return BM * ((seg + 7) / 8 * 8 + 8) * 2 + BM * 49 * 4;
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// bf16 value at (key, col) of a V tile stored as [col/64][64 keys][128 B] with SWIZZLE_128B.
__device__ __forceinline__ const uint4* v_chunk(const uint8_t* sV, int key, int col) {
    const int atom = col >> 6, chunk = (col & 63) >> 3;
    return reinterpret_cast<const uint4*>(sV + atom * (BN * 128) + key * 128 +
                                          ((chunk ^ (key & 7)) << 4));
}

// Fused output epilogue (proj/src/flash_ipa.cpp:171-210), one thread per query row, reading
// the row's O accumulator straight from TMEM (+ the CUDA-core value columns):
//   feat block = [ sum_rho z1[i,rho,:] * O_pair[rho,:] | O_scalar | R_i^T(g_p - t_i) | |.| ]
// with g_p = agg(R_j v_p) + agg(t_j hi) + agg(t_j lo).  Rows are assembled as bf16 in shared
// memory, then the 128 x seg block is written out with coalesced 16-byte stores.
__device__ __forceinline__ void fused_epilogue(const AttnParams& p, uint32_t tl, const float* acc_s,
                                               float inv_l, int row, int q0, int bh, uint8_t* smem) {
    const int seg = p.seg, sst = (seg + 7) / 8 * 8 + 8;  // staging row stride (bf16)
    __nv_bfloat16* fst = reinterpret_cast<__nv_bfloat16*>(smem);
    __nv_bfloat16* frow = fst + row * sst;
    float* pts = reinterpret_cast<float*>(smem + BM * sst * 2) + row * 49;
    const int H = p.H, b = bh / H, h = bh % H;
    const int q = q0 + row;
    const bool ok = q < p.L;
    const int64_t grow = static_cast<int64_t>(b) * p.L + (ok ? q : 0);
    const int c = p.c, dz = p.d_z, Nv = p.n_value;
    const int base = c + p.rank * dz, npt = 3 * Nv + 6;

    // scalar aggregate -> [d_z, d_z + c)
    for (int c0 = 0; c0 < c; c0 += 16) {
        uint32_t o[16];
        ptx::tmem_ld16(tl + c0, o);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e)
            if (c0 + e < c) frow[dz + c0 + e] = __float2bfloat16_rn(__uint_as_float(o[e]) * inv_l);
    }
    // pair contraction -> [0, d_z)
    const float* z1r = p.z1 + grow * (p.rank * dz);
    for (int d0 = 0; d0 < dz; d0 += 16) {
        float acc[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[e] = 0.f;
        for (int rho = 0; rho < p.rank; ++rho) {
            float z[16];
            const float* zp = z1r + rho * dz + d0;
            if (d0 + 16 <= dz && (reinterpret_cast<uintptr_t>(zp) & 15) == 0) {
#pragma unroll
                for (int v4 = 0; v4 < 4; ++v4) {
                    const float4 f = __ldg(reinterpret_cast<const float4*>(zp) + v4);
                    z[4 * v4] = f.x;
                    z[4 * v4 + 1] = f.y;
                    z[4 * v4 + 2] = f.z;
                    z[4 * v4 + 3] = f.w;
                }
            } else {
#pragma unroll
                for (int e = 0; e < 16; ++e) z[e] = d0 + e < dz ? __ldg(zp + e) : 0.f;
            }
            uint32_t o[16];
            ptx::tmem_ld16(tl + c + rho * dz + d0, o);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[e] = fmaf(z[e], __uint_as_float(o[e]), acc[e]);
        }
#pragma unroll
        for (int e = 0; e < 16; ++e)
            if (d0 + e < dz) frow[d0 + e] = __float2bfloat16_rn(acc[e] * inv_l);
    }
    // point block [base, base + npt) of O_hat -> per-row scratch
    for (int c0 = 0; c0 < npt; c0 += 16) {
        if (base + c0 < p.dv_tc) {
            uint32_t o[16];
            ptx::tmem_ld16(tl + base + c0, o);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e)
                if (c0 + e < npt && base + c0 + e < p.dv_tc) pts[c0 + e] = __uint_as_float(o[e]) * inv_l;
        }
    }
#pragma unroll
    for (int k = 0; k < kMaxSimt; ++k) {
        const int idx = p.dv_tc + k - base;
        if (k < p.dv_simt && idx >= 0 && idx < npt) pts[idx] = acc_s[k] * inv_l;
    }
    if (ok) {
        const float* R = p.rot + grow * 9;
        const float* t = p.trans + grow * 3;
        float Rm[9], tg[3];
#pragma unroll
        for (int k = 0; k < 9; ++k) Rm[k] = __ldg(R + k);
#pragma unroll
        for (int y = 0; y < 3; ++y) tg[y] = pts[y] + pts[3 + y] - __ldg(t + y);
        __nv_bfloat16* fp = frow + dz + c;
        for (int pt = 0; pt < Nv; ++pt) {
            const float* pv = pts + 6 + 3 * pt;  // point block = [t hi | t lo | R_j v_p]
            const float gx = pv[0] + tg[0], gy = pv[1] + tg[1], gz = pv[2] + tg[2];
            // apply_inverse: R^T g   (proj/src/geometry.cpp:70-76)
            const float lx = fmaf(Rm[0], gx, fmaf(Rm[3], gy, Rm[6] * gz));
            const float ly = fmaf(Rm[1], gx, fmaf(Rm[4], gy, Rm[7] * gz));
            const float lz = fmaf(Rm[2], gx, fmaf(Rm[5], gy, Rm[8] * gz));
            fp[3 * pt] = __float2bfloat16_rn(lx);
            fp[3 * pt + 1] = __float2bfloat16_rn(ly);
            fp[3 * pt + 2] = __float2bfloat16_rn(lz);
            fp[3 * Nv + pt] = __float2bfloat16_rn(sqrtf(lx * lx + ly * ly + lz * lz));
        }
    }
    named_bar_sync(1, 128);
    // coalesced copy-out of the 128 x seg bf16 block
    const int tid = threadIdx.x - 64;
    const int rows = min(BM, p.L - q0);
    __nv_bfloat16* gout = p.feat_out + (static_cast<int64_t>(b) * p.L + q0) * p.feat_ld + h * seg;
    if (seg % 8 == 0 && p.feat_ld % 8 == 0 && ((h * seg) % 8) == 0) {
        const int per_row = seg / 8;
        for (int e = tid; e < rows * per_row; e += 128) {
            const int r = e / per_row, k = e - r * per_row;
            *reinterpret_cast<uint4*>(gout + static_cast<int64_t>(r) * p.feat_ld + 8 * k) =
                *reinterpret_cast<const uint4*>(fst + r * sst + 8 * k);
        }
    } else {
        for (int e = tid; e < rows * seg; e += 128) {
            const int r = e / seg, k = e - r * seg;
            gout[static_cast<int64_t>(r) * p.feat_ld + k] = fst[r * sst + k];
        }
    }
}

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
    const int region = p.n_qkb * (BM * 128 + BN * 128) + p.n_vb * (BN * 128);
    const int stage_bytes = epilogue_smem(p.seg);
    Bars* bars = reinterpret_cast<Bars*>(smem + (region > stage_bytes ? region : stage_bytes));

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
        ptx::mbar_init(&bars->v_empty, p.dv_simt > 0 ? 5 : 1);
        ptx::mbar_init(&bars->s_full, 1);
        ptx::mbar_init(&bars->s_free, 4);
        ptx::mbar_init(&bars->p_full, 4);
        ptx::mbar_init(&bars->pv_done, 1);
        ptx::mbar_init(&bars->o_full, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(&bars->tmem_slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, bars->tmem_slot, 0);

    if (warp == 0) {
        // ------------------------------------------------------- Q/K TMA producer
        if (lane == 0) {
            ptx::mbar_expect_tx(&bars->q_full, p.n_qkb * BM * 128);
            for (int b = 0; b < p.n_qkb; ++b)
                ptx::tma_load_3d(sQ + b * BM * 128, &mapQ, &bars->q_full, b * 64, q0, bh);
            for (int j = 0; j < ntiles; ++j) {
                if (j > 0) ptx::mbar_wait(&bars->k_empty, (j - 1) & 1);
                FIPA_TRACE(0, j);
                ptx::mbar_expect_tx(&bars->k_full, p.n_qkb * BN * 128);
                for (int b = 0; b < p.n_qkb; ++b)
                    ptx::tma_load_3d(sK + b * BN * 128, &mapK, &bars->k_full, b * 64, j * BN, bh);
            }
        }
    } else if (warp == 6) {
        // --------------------------------------------------------- V TMA producer
        if (lane == 0) {
            for (int j = 0; j < ntiles; ++j) {
                if (j > 0) ptx::mbar_wait(&bars->v_empty, (j - 1) & 1);
                FIPA_TRACE(1, j);
                ptx::mbar_expect_tx(&bars->v_full, p.n_vb * BN * 128);
                for (int b = 0; b < p.n_vb; ++b)
                    ptx::tma_load_3d(sV + b * BN * 128, &mapV, &bars->v_full, b * 64, j * BN, bh);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        const uint32_t idesc_qk = ptx::idesc_bf16(BM, BN, false, false);
        const int n1 = p.dv_tc < 256 ? p.dv_tc : 256;
        const int n2 = p.dv_tc - n1;
        const uint32_t idesc_pv1 = ptx::idesc_bf16(BM, n1, false, true);
        const uint32_t idesc_pv2 = ptx::idesc_bf16(BM, n2 > 0 ? n2 : 16, false, true);
        const uint32_t q_base = ptx::smem_u32(sQ);
        const uint32_t k_base = ptx::smem_u32(sK);
        const uint32_t v_base = ptx::smem_u32(sV);
        const int qk_steps = p.dqk_mma / 16;
        ptx::mbar_wait(&bars->q_full, 0);
        for (int j = 0; j <= ntiles; ++j) {
            if (j < ntiles) {
                ptx::mbar_wait(&bars->k_full, j & 1);
                if (j > 0) ptx::mbar_wait(&bars->s_free, (j - 1) & 1);
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    FIPA_TRACE(2, j);
                    for (int kk = 0; kk < qk_steps; ++kk) {
                        const uint32_t blk = kk >> 2, sub = (kk & 3) * 32;
                        const uint64_t da = ptx::sw128_desc(q_base + blk * (BM * 128) + sub, 16, 1024);
                        const uint64_t db = ptx::sw128_desc(k_base + blk * (BN * 128) + sub, 16, 1024);
                        ptx::mma_ss(tmem + kSCol, da, db, idesc_qk, kk > 0);
                    }
                    ptx::mma_commit(&bars->k_empty);
                    ptx::mma_commit(&bars->s_full);
                }
                __syncwarp();
            }
            if (j > 0) {
                const int jj = j - 1;
                ptx::mbar_wait(&bars->p_full, jj & 1);
                ptx::mbar_wait(&bars->v_full, jj & 1);
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    FIPA_TRACE(3, jj);
#pragma unroll
                    for (int kk = 0; kk < BN / 16; ++kk) {
                        const uint32_t a_tm = tmem + kPCol + kk * 8;
                        const uint64_t db1 = ptx::sw128_desc(v_base + kk * 2048, BN * 128, 1024);
                        ptx::mma_ts(tmem, a_tm, db1, idesc_pv1, (jj > 0 || kk > 0));
                        if (n2 > 0) {
                            const uint64_t db2 =
                                ptx::sw128_desc(v_base + 4 * (BN * 128) + kk * 2048, BN * 128, 1024);
                            ptx::mma_ts(tmem + 256, a_tm, db2, idesc_pv2, (jj > 0 || kk > 0));
                        }
                    }
                    ptx::mma_commit(&bars->v_empty);
                    ptx::mma_commit(&bars->pv_done);
                    if (j == ntiles) ptx::mma_commit(&bars->o_full);
                }
                __syncwarp();
            }
        }
    } else {
        // ----------------------------------------------- softmax (+ SIMT value columns)
        const int quad = warp & 3;
        const int row = quad * 32 + lane;
        const uint32_t tl = tmem + (uint32_t(quad * 32) << 16);
        float m = -INFINITY;  // running max, log2 units
        float l = 0.f;
        float acc_s[kMaxSimt];
#pragma unroll
        for (int k = 0; k < kMaxSimt; ++k) acc_s[k] = 0.f;
        for (int j = 0; j < ntiles; ++j) {
            ptx::mbar_wait(&bars->s_full, j & 1);
            if (threadIdx.x == 64) FIPA_TRACE(4, j);
            ptx::tc_fence_after();
            uint32_t sr[64];
            ptx::tmem_ld32(tl + kSCol, sr);
            ptx::tmem_ld32(tl + kSCol + 32, sr + 32);
            ptx::tmem_wait_ld();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&bars->s_free);

            float x[64];
            float mt = -INFINITY;
            const int kvalid = p.L - j * BN;  // keys >= L in the last tile are not real
#pragma unroll
            for (int cc = 0; cc < 64; ++cc) {
                x[cc] = cc < kvalid ? __uint_as_float(sr[cc]) : -INFINITY;
                mt = fmaxf(mt, x[cc]);
            }
            const bool need = mt > m + 8.0f;  // also true on the first finite tile
            float scale = 1.0f;
            if (need) {
                scale = exp2f(m - mt);  // 0 when m == -inf
                m = mt;
                l *= scale;
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

            // P_j may only overwrite P_{j-1} (and O may only be rescaled) once PV_{j-1} is done.
            if (j > 0) {
                ptx::mbar_wait(&bars->pv_done, (j - 1) & 1);
                if (threadIdx.x == 64) FIPA_TRACE(5, j);
                ptx::tc_fence_after();
                if (__any_sync(0xffffffffu, need)) {
                    for (int c0 = 0; c0 < p.dv_tc; c0 += 16) {
                        uint32_t o[16];
                        ptx::tmem_ld16(tl + c0, o);
                        ptx::tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * scale);
                        ptx::tmem_st16(tl + c0, o);
                    }
                }
            }
            ptx::tmem_st32(tl + kPCol, pk);
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&bars->p_full);
            if (threadIdx.x == 64) FIPA_TRACE(6, j);

            // Trailing value columns on CUDA cores (same bf16 P as the tensor cores see).
            if (p.dv_simt > 0) {
#pragma unroll
                for (int k = 0; k < kMaxSimt; ++k) acc_s[k] *= scale;
                ptx::mbar_wait(&bars->v_full, j & 1);
#pragma unroll
                for (int cc = 0; cc < BN / 2; ++cc) {
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int key = 2 * cc + u;
                        const float pb = __uint_as_float(u ? (pk[cc] & 0xffff0000u) : (pk[cc] << 16));
                        const uint4 c0 = *v_chunk(sV, key, p.dv_tc);
                        const uint4 c1 = *v_chunk(sV, key, p.dv_tc + 8);
                        const uint32_t w[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
                        for (int k = 0; k < kMaxSimt; k += 2) {
                            acc_s[k] = fmaf(pb, __uint_as_float(w[k >> 1] << 16), acc_s[k]);
                            acc_s[k + 1] = fmaf(pb, __uint_as_float(w[k >> 1] & 0xffff0000u), acc_s[k + 1]);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&bars->v_empty);
                if (threadIdx.x == 64) FIPA_TRACE(7, j);
            }
        }

        // ---------------------------------------------------------------- epilogue
        // Phase 1: normalised O_hat row -> shared staging (fp32, row stride dv_used|1).
        ptx::mbar_wait(&bars->o_full, 0);
        if (threadIdx.x == 64) FIPA_TRACE(8, 0);
        ptx::tc_fence_after();
        const float inv_l = l > 0.f ? 1.0f / l : 0.f;
        const int qi = q0 + row;
        if (qi < p.L)
            p.lse[static_cast<int64_t>(bh) * p.L + qi] = l > 0.f ? (m + log2f(l)) * kLn2 : -INFINITY;
        fused_epilogue(p, tl, acc_s, inv_l, row, q0, bh, smem);
        if (threadIdx.x == 64) FIPA_TRACE(8, 2);
    }

    if (threadIdx.x == 64) FIPA_TRACE(8, 1);
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

}  // namespace

void launch_attn_fwd_tc(const LayerDims& d, const AttnArgs& a, cudaStream_t stream) {
    if (d.dqk_mma > 448)
        throw std::invalid_argument("tcgen05 attention: lifted q/k width exceeds 448 (use precision='f32')");
    if (d.dv_simt > kMaxSimt)
        throw std::invalid_argument("tcgen05 attention: lifted value width exceeds 432 (use precision='f32')");
    if (3 * d.n_value + 6 > 48 || d.c + d.rank * d.d_z > d.dv_tc)
        throw std::invalid_argument("tcgen05 attention: value layout unsupported (use precision='f32')");
    AttnParams p{};
    p.L = a.L;
    p.H = d.heads;
    p.dqk_mma = d.dqk_mma;
    p.dv_tc = d.dv_tc;
    p.dv_simt = d.dv_simt;
    p.dv_used = d.dv_used;
    p.n_qkb = (d.dqk_mma + 63) / 64;
    p.n_vb = (d.dv_pad + 63) / 64;
    p.c = d.c;
    p.d_z = d.d_z;
    p.rank = d.rank;
    p.n_value = d.n_value;
    p.seg = d.seg;
    p.feat_ld = d.feat_ld;
    p.z1 = a.z1;
    p.rot = a.rot;
    p.trans = a.trans;
    p.feat_out = a.feat;
    p.lse = a.lse;
    const uint64_t BH = static_cast<uint64_t>(a.B) * d.heads;
    const CUtensorMap mapQ = make_map_3d_bf16(a.qhat, d.dqk_pad, a.L, BH, d.dqk_pad, 64, BM);
    const CUtensorMap mapK = make_map_3d_bf16(a.khat, d.dqk_pad, a.L, BH, d.dqk_pad, 64, BN);
    const CUtensorMap mapV = make_map_3d_bf16(a.vhat, d.dv_pad, a.L, BH, d.dv_pad, 64, BN);
    const int region = p.n_qkb * (BM * 128 + BN * 128) + p.n_vb * (BN * 128);
    const int stage = epilogue_smem(d.seg);
    const int smem = std::max(region, stage) + 1024 + 256;
    if (smem > 232448) throw std::invalid_argument("tcgen05 attention: shared memory budget exceeded");
    cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    dim3 grid((a.L + BM - 1) / BM, static_cast<unsigned>(BH));
    attn_fwd_kernel<<<grid, kThreads, smem, stream>>>(mapQ, mapK, mapV, p);
}

}  // namespace fipa_b200
