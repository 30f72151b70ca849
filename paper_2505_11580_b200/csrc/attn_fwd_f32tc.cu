// FlashIPA attention forward at fp32 accuracy on the tcgen05 tensor cores ("3xTF32"): the
// precision="f32" / "f64" path of the layer (the reference computes in double,
// proj/src/attention_kernel.cpp:112-188, proj/src/flash_ipa.cpp:171-210; gate 1e-4).
//
// Every fp32 operand x is split as x = hi + lo with hi = tf32(x) (cvt.rna) and lo = x - hi
// (exact), stored as two planes (pack.cu split3).  A product a.b is formed as
//   a_lo b_lo + a_hi b_lo + a_lo b_hi + a_hi b_hi   (small terms first)
// with tcgen05.mma kind::tf32 chains into the same fp32 TMEM accumulator.  The lo.lo term (~2^-22
// relative) costs no time here -- the kernel is bound by the operand stream, not the tensor pipe --
// and keeps the layer inside the 1e-4 gate at protein-scale (30 A) coordinates.
//
// One CTA = one (sample, head, 128-query tile).  Per key tile j of 64 keys:
//   S_j  = Q_hat . K_hat_j^T  (log2 units, column bias folded in, pack.cu)  -> TMEM [448, 512)
//          The lifted width (432 fp32 columns in hi and lo planes, 442 KB for a 128-row tile) does
//          not fit shared memory, so Q is streamed with K in 32-column chunks: per chunk the
//          q_hi | q_lo | k_hi | k_lo sub-tiles land in one 48 KB ring stage (TMA) and 12 MMAs
//          (M=128, N=64, K=8) run over it.
//   P_j  = 2^(S_j - m) in fp32 by the softmax warps (lazy rescale: the running max moves only
//          when it grows by more than 2^8), split into P_hi | P_lo in shared memory
//          (K-major, 128 rows x 64 keys each).
//   O   += P_j . V_hat_j      three chains P_hi V_hi + P_lo V_hi + P_hi V_lo, V^T streamed in
//          128-column chunks (hi and lo planes, K-major: keys contiguous), N = 128, 128, 128, 48
//          -> TMEM [0, 432)
// The tensor pipe runs S_{j+1} while the softmax warps turn S_j into P_j.  Epilogue: the same
// split / pair contraction / inverse frame / norms as the bf16 kernels, fp32 features staged in
// shared memory and written with coalesced stores.
//
// Warp roles (224 threads): w0 Q/K TMA producer, w1 TMEM alloc + MMA issue (elect.sync), w2..w5
// softmax + epilogue (one thread per query row, warp w owns TMEM lanes 32*(w%4)..), w6 V producer.
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
constexpr uint32_t kSCol = 448;    // S tile: 64 fp32 columns
constexpr int kQKStages = 2;
constexpr int kVStages = 2;
constexpr int kQChunk = BM * 128;  // 32 fp32 columns x 128 rows
constexpr int kKChunk = BN * 128;  // 32 fp32 columns x 64 keys
constexpr int kQKStage = 2 * kQChunk + 2 * kKChunk;  // q_hi | q_lo | k_hi | k_lo
constexpr int kVNc = 128;                            // value columns per V chunk
constexpr int kVStage = BN * kVNc * 4;               // 128 value columns x 64 keys: 2 atoms of 32 keys
constexpr int kPBytes = BM * BN * 4;                 // one P plane: 2 atoms of 128 rows x 128 B
constexpr float kLn2 = 0.6931471805599453f;

struct Params {
    int L, H, nkc, dv_mma, c, d_z, rank, n_value, seg, feat_ld;
    const float* z1;
    const float* rot;
    const float* trans;
    float* feat;
    float* lse;
};

struct Bars {
    uint64_t qk_full[kQKStages], qk_empty[kQKStages];
    uint64_t v_full[kVStages], v_empty[kVStages];
    uint64_t s_full, s_free, p_full, pv_done, o_full;
    uint32_t tmem_slot;
};

struct Layout {
    int qk, p, v, bars, total;
};
__host__ __device__ constexpr Layout smem_layout() {
    Layout l{};
    l.qk = 0;
    l.p = kQKStages * kQKStage;
    l.v = l.p + 2 * kPBytes;
    l.bars = l.v + kVStages * kVStage;
    l.total = l.bars + static_cast<int>(sizeof(Bars));
    return l;
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_f32tc_kernel(const __grid_constant__ CUtensorMap mQh, const __grid_constant__ CUtensorMap mQl,
                          const __grid_constant__ CUtensorMap mKh, const __grid_constant__ CUtensorMap mKl,
                          const __grid_constant__ CUtensorMap mVh, const __grid_constant__ CUtensorMap mVl,
                          Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    constexpr Layout lay = smem_layout();
    uint8_t* sQK = smem + lay.qk;
    uint8_t* sP = smem + lay.p;  // P_hi plane, then P_lo plane
    uint8_t* sV = smem + lay.v;
    Bars* bars = reinterpret_cast<Bars*>(smem + lay.bars);

    const int warp = ptx::warp_id();
    const int lane = ptx::lane_id();
    const int bh = blockIdx.y;
    const int q0 = blockIdx.x * BM;
    const int ntiles = (p.L + BN - 1) / BN;
    const int nvc = (p.dv_mma + kVNc - 1) / kVNc;  // V column chunks per key tile

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&mQh);
        ptx::tma_prefetch(&mQl);
        ptx::tma_prefetch(&mKh);
        ptx::tma_prefetch(&mKl);
        ptx::tma_prefetch(&mVh);
        ptx::tma_prefetch(&mVl);
        for (int s = 0; s < kQKStages; ++s) {
            ptx::mbar_init(&bars->qk_full[s], 1);
            ptx::mbar_init(&bars->qk_empty[s], 1);
        }
        for (int s = 0; s < kVStages; ++s) {
            ptx::mbar_init(&bars->v_full[s], 1);
            ptx::mbar_init(&bars->v_empty[s], 1);
        }
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
        // ------------------------------------------- Q / K chunk producer (hi and lo planes)
        if (lane == 0) {
            int it = 0;
            for (int j = 0; j < ntiles; ++j) {
                for (int kc = 0; kc < p.nkc; ++kc, ++it) {
                    const int s = it % kQKStages;
                    if (it >= kQKStages) ptx::mbar_wait(&bars->qk_empty[s], ((it / kQKStages) - 1) & 1);
                    uint8_t* st = sQK + s * kQKStage;
                    ptx::mbar_expect_tx(&bars->qk_full[s], kQKStage);
                    ptx::tma_load_3d(st, &mQh, &bars->qk_full[s], kc * 32, q0, bh);
                    ptx::tma_load_3d(st + kQChunk, &mQl, &bars->qk_full[s], kc * 32, q0, bh);
                    ptx::tma_load_3d(st + 2 * kQChunk, &mKh, &bars->qk_full[s], kc * 32, j * BN, bh);
                    ptx::tma_load_3d(st + 2 * kQChunk + kKChunk, &mKl, &bars->qk_full[s], kc * 32, j * BN, bh);
                }
            }
        }
    } else if (warp == 6) {
        // ------------------------------------------- V chunk producer (hi, lo per column chunk)
        if (lane == 0) {
            int it = 0;
            for (int j = 0; j < ntiles; ++j) {
                for (int nc = 0; nc < nvc; ++nc) {
                    for (int plane = 0; plane < 2; ++plane, ++it) {
                        const int s = it % kVStages;
                        if (it >= kVStages) ptx::mbar_wait(&bars->v_empty[s], ((it / kVStages) - 1) & 1);
                        uint8_t* st = sV + s * kVStage;
                        ptx::mbar_expect_tx(&bars->v_full[s], kVStage);
                        for (int a = 0; a < 2; ++a)  // keys [32a, 32a + 32) x 128 value columns
                            ptx::tma_load_3d(st + a * (kVNc * 128), plane ? &mVl : &mVh, &bars->v_full[s],
                                             j * BN + 32 * a, nc * kVNc, bh);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------- MMA issue
        const uint32_t idesc_s = ptx::idesc_tf32(BM, BN, false, false);
        const uint32_t qk_base = ptx::smem_u32(sQK);
        const uint32_t p_base = ptx::smem_u32(sP);
        const uint32_t v_base = ptx::smem_u32(sV);
        const uint64_t d_qk = ptx::sw128_desc(qk_base, 16, 1024);
        const uint64_t d_p = ptx::sw128_desc(p_base, 16, 1024);
        // K-major V^T chunk: 128 value-column rows of 128 B (32 keys) per atom, atoms 16 KB apart
        const uint64_t d_v = ptx::sw128_desc(v_base, 16, 1024);
        int it = 0, vit = 0;
        for (int j = 0; j <= ntiles; ++j) {
            if (j < ntiles) {
                if (j > 0) ptx::mbar_wait(&bars->s_free, (j - 1) & 1);
                for (int kc = 0; kc < p.nkc; ++kc, ++it) {
                    const int s = it % kQKStages;
                    ptx::mbar_wait(&bars->qk_full[s], (it / kQKStages) & 1);
                    ptx::tc_fence_after();
                    if (ptx::elect_one()) {
                        const uint64_t so = static_cast<uint64_t>((s * kQKStage) >> 4);
                        const uint64_t qh = d_qk + so, ql = qh + (kQChunk >> 4);
                        const uint64_t kh = qh + ((2 * kQChunk) >> 4), kl = kh + (kKChunk >> 4);
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {  // K = 8 per MMA: +32 B
                            const uint64_t o = static_cast<uint64_t>(2 * kk);
                            // small terms first within the step; the lo.lo term is free here (the
                            // kernel is bound by the operand stream, not the tensor pipe)
                            ptx::mma_ss_tf32(tmem + kSCol, ql + o, kl + o, idesc_s, (kc | kk) != 0);
                            ptx::mma_ss_tf32(tmem + kSCol, qh + o, kl + o, idesc_s, 1u);
                            ptx::mma_ss_tf32(tmem + kSCol, ql + o, kh + o, idesc_s, 1u);
                            ptx::mma_ss_tf32(tmem + kSCol, qh + o, kh + o, idesc_s, 1u);
                        }
                        ptx::mma_commit(&bars->qk_empty[s]);
                        if (kc == p.nkc - 1) ptx::mma_commit(&bars->s_full);
                    }
                    __syncwarp();
                }
            }
            if (j > 0) {
                const int jj = j - 1;
                ptx::mbar_wait(&bars->p_full, jj & 1);
                ptx::tc_fence_after();
                for (int nc = 0; nc < nvc; ++nc) {
                    const int ncols = min(kVNc, p.dv_mma - nc * kVNc);
                    const uint32_t idesc_v = ptx::idesc_tf32(BM, ncols, false, false);
                    const int sh = vit % kVStages, sl = (vit + 1) % kVStages;
                    ptx::mbar_wait(&bars->v_full[sh], (vit / kVStages) & 1);
                    ptx::mbar_wait(&bars->v_full[sl], ((vit + 1) / kVStages) & 1);
                    ptx::tc_fence_after();
                    if (ptx::elect_one()) {
                        const uint64_t vh = d_v + static_cast<uint64_t>((sh * kVStage) >> 4);
                        const uint64_t vl = d_v + static_cast<uint64_t>((sl * kVStage) >> 4);
                        const uint32_t acc_col = tmem + nc * kVNc;
#pragma unroll
                        for (int kk = 0; kk < BN / 8; ++kk) {
                            // A (P, K-major): 8 keys = +32 B within a 32-key atom, atoms 16 KB apart
                            const uint64_t pa = d_p + static_cast<uint64_t>(((kk >> 2) * (BM * 128) + (kk & 3) * 32) >> 4);
                            const uint64_t pl = pa + static_cast<uint64_t>(kPBytes >> 4);
                            const uint64_t o = static_cast<uint64_t>(((kk >> 2) * (kVNc * 128) + (kk & 3) * 32) >> 4);
                            const uint32_t first = (jj > 0 || kk > 0) ? 1u : 0u;
                            ptx::mma_ss_tf32(acc_col, pl, vl + o, idesc_v, first);
                            ptx::mma_ss_tf32(acc_col, pl, vh + o, idesc_v, 1u);
                            ptx::mma_ss_tf32(acc_col, pa, vl + o, idesc_v, 1u);
                            ptx::mma_ss_tf32(acc_col, pa, vh + o, idesc_v, 1u);
                        }
                        ptx::mma_commit(&bars->v_empty[sh]);
                        ptx::mma_commit(&bars->v_empty[sl]);
                    }
                    __syncwarp();
                    vit += 2;
                }
                if (ptx::elect_one()) {
                    ptx::mma_commit(&bars->pv_done);
                    if (j == ntiles) ptx::mma_commit(&bars->o_full);
                }
                __syncwarp();
            }
        }
    } else {
        // ------------------------------------------------------------------ softmax
        const int quad = warp & 3;
        const int row = quad * 32 + lane;
        const uint32_t tl = tmem + (uint32_t(quad * 32) << 16);
        float m = -INFINITY;  // running max (log2 units) the probabilities are relative to
        float l = 0.f;
        for (int j = 0; j < ntiles; ++j) {
            ptx::mbar_wait(&bars->s_full, j & 1);
            ptx::tc_fence_after();
            uint32_t sr[64];
            ptx::tmem_ld32(tl + kSCol, sr);
            ptx::tmem_ld32(tl + kSCol + 32, sr + 32);
            ptx::tmem_wait_ld();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&bars->s_free);

            const int kvalid = p.L - j * BN;  // keys >= L in the last tile are not real
            float mt = -INFINITY;
#pragma unroll
            for (int cc = 0; cc < 64; ++cc) {
                if (cc >= kvalid) sr[cc] = __float_as_uint(-INFINITY);
                mt = fmaxf(mt, __uint_as_float(sr[cc]));
            }
            const bool need = mt > m + 8.0f;  // also true on the first finite tile
            float scale = 1.0f;
            if (need) {
                scale = exp2f(m - mt);  // 0 when m == -inf
                m = mt;
                l *= scale;
            }
            const float mm = m == -INFINITY ? 0.f : m;
            float ls = 0.f;
#pragma unroll
            for (int cc = 0; cc < 64; ++cc) {
                const float pv = exp2f(__uint_as_float(sr[cc]) - mm);
                ls += pv;
                sr[cc] = __float_as_uint(pv);
            }
            l += ls;

            // P_j may only overwrite P_{j-1} (and O may only be rescaled) once PV_{j-1} is done.
            if (j > 0) {
                ptx::mbar_wait(&bars->pv_done, (j - 1) & 1);
                ptx::tc_fence_after();
                if (__any_sync(0xffffffffu, need)) {
                    for (int c0 = 0; c0 < p.dv_mma; c0 += 16) {
                        uint32_t o[16];
                        ptx::tmem_ld16(tl + c0, o);
                        ptx::tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * scale);
                        ptx::tmem_st16(tl + c0, o);
                    }
                    ptx::tmem_wait_st();
                }
            }
            // P rows -> shared memory, K-major 128-byte swizzled: keys [32a, 32a+32) in atom a,
            // 16-byte chunk q of a row at ((q ^ (row & 7)) << 4)
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                uint8_t* rh = sP + a * (BM * 128) + row * 128;
                uint8_t* rl = rh + kPBytes;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    float hi[4], lo[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float x = __uint_as_float(sr[32 * a + 4 * q + e]);
                        hi[e] = ptx::tf32_hi(x);
                        lo[e] = x - hi[e];
                    }
                    const int off = (q ^ (row & 7)) << 4;
                    *reinterpret_cast<float4*>(rh + off) = make_float4(hi[0], hi[1], hi[2], hi[3]);
                    *reinterpret_cast<float4*>(rl + off) = make_float4(lo[0], lo[1], lo[2], lo[3]);
                }
            }
            ptx::fence_proxy_async_smem();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&bars->p_full);
        }

        // ------------------------------------------------------------------ epilogue
        ptx::mbar_wait(&bars->o_full, 0);
        ptx::tc_fence_after();
        const float inv_l = l > 0.f ? 1.0f / l : 0.f;
        const int qi = q0 + row;
        const bool ok = qi < p.L;
        if (ok) p.lse[static_cast<int64_t>(bh) * p.L + qi] = l > 0.f ? (m + log2f(l)) * kLn2 : -INFINITY;
        // all MMAs are done: the operand rings are free for the fp32 feature staging [128][seg | 1]
        // (the barrier makes every softmax thread's last P store precede the staging writes without
        // relying on the o_full chain alone)
        named_bar_sync(1, 128);
        const int sst = p.seg | 1;
        float* frow = reinterpret_cast<float*>(smem) + row * sst;
        const int H = p.H, b = bh / H, h = bh - b * H;
        const int64_t grow = static_cast<int64_t>(b) * p.L + (ok ? qi : 0);
        const int c = p.c, dz = p.d_z, Nv = p.n_value;
        const int base = c + p.rank * dz;  // point block = [t hi | t lo | R_j v_p]
        for (int c0 = 0; c0 < c; c0 += 16) {  // scalar aggregate -> [d_z, d_z + c)
            uint32_t o[16];
            ptx::tmem_ld16(tl + c0, o);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e)
                if (c0 + e < c) frow[dz + c0 + e] = __uint_as_float(o[e]) * inv_l;
        }
        const float* z1r = p.z1 + grow * (p.rank * dz);
        for (int d0 = 0; d0 < dz; d0 += 16) {  // pair contraction -> [0, d_z)
            float acc[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[e] = 0.f;
            for (int rho = 0; rho < p.rank; ++rho) {
                uint32_t o[16];
                ptx::tmem_ld16(tl + c + rho * dz + d0, o);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    if (d0 + e < dz) acc[e] = fmaf(__ldg(z1r + rho * dz + d0 + e), __uint_as_float(o[e]), acc[e]);
            }
#pragma unroll
            for (int e = 0; e < 16; ++e)
                if (d0 + e < dz) frow[d0 + e] = acc[e] * inv_l;
        }
        {
            // point block [t hi | t lo | R_j v_p] (<= 48 columns) into registers
            float pts[48];
#pragma unroll
            for (int c0 = 0; c0 < 48; c0 += 16) {
                if (c0 < 6 + 3 * Nv) {
                    uint32_t o[16];
                    ptx::tmem_ld16(tl + base + c0, o);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 16; ++e) pts[c0 + e] = __uint_as_float(o[e]) * inv_l;
                } else {
#pragma unroll
                    for (int e = 0; e < 16; ++e) pts[c0 + e] = 0.f;
                }
            }
            float Rm[9], tg[3];
#pragma unroll
            for (int k = 0; k < 9; ++k) Rm[k] = __ldg(p.rot + grow * 9 + k);
#pragma unroll
            for (int y = 0; y < 3; ++y) tg[y] = pts[y] + pts[3 + y] - __ldg(p.trans + grow * 3 + y);
            float* fp = frow + dz + c;
#pragma unroll
            for (int pt = 0; pt < 14; ++pt) {  // compile-time point index keeps pts[] in registers
                if (pt < Nv) {
                    const float gx = pts[6 + 3 * pt] + tg[0], gy = pts[7 + 3 * pt] + tg[1], gz = pts[8 + 3 * pt] + tg[2];
                    // apply_inverse: R^T g   (proj/src/geometry.cpp:70-76)
                    const float lx = fmaf(Rm[0], gx, fmaf(Rm[3], gy, Rm[6] * gz));
                    const float ly = fmaf(Rm[1], gx, fmaf(Rm[4], gy, Rm[7] * gz));
                    const float lz = fmaf(Rm[2], gx, fmaf(Rm[5], gy, Rm[8] * gz));
                    fp[3 * pt] = lx;
                    fp[3 * pt + 1] = ly;
                    fp[3 * pt + 2] = lz;
                    fp[3 * Nv + pt] = sqrtf(lx * lx + ly * ly + lz * lz);
                }
            }
        }
        named_bar_sync(1, 128);
        // coalesced copy-out of the 128 x seg fp32 block
        const int tid = threadIdx.x - 64;
        const int rows = min(BM, p.L - q0);
        float* gout = p.feat + (static_cast<int64_t>(b) * p.L + q0) * p.feat_ld + h * p.seg;
        const float* fst = reinterpret_cast<const float*>(smem);
        for (int e = tid; e < rows * p.seg; e += 128) {
            const int r = e / p.seg, k = e - r * p.seg;
            gout[static_cast<int64_t>(r) * p.feat_ld + k] = fst[r * sst + k];
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

}  // namespace

bool attn_fwd_f32tc_supported(const LayerDims& d) {
    // TMEM: O (dv_mma) + S (64) <= 512; the point block fits the epilogue's 48 registers; the
    // fp32 feature staging [128][seg | 1] reuses the operand rings
    return d.dv_mma <= 448 && d.dv_pad % 32 == 0 && d.dqk_pad % 32 == 0 && 3 * d.n_value + 6 <= 48 &&
           (d.seg | 1) * BM * 4 <= smem_layout().bars;
}

void launch_attn_fwd_f32tc(const LayerDims& d, const AttnF32TcArgs& a, cudaStream_t stream) {
    if (!attn_fwd_f32tc_supported(d))
        throw std::invalid_argument("3xTF32 attention: lifted value width exceeds 448");
    Params p{};
    p.L = a.L;
    p.H = d.heads;
    p.nkc = (d.dqk_mma + 31) / 32;
    p.dv_mma = d.dv_mma;
    p.c = d.c;
    p.d_z = d.d_z;
    p.rank = d.rank;
    p.n_value = d.n_value;
    p.seg = d.seg;
    p.feat_ld = d.feat_ld;
    p.z1 = a.z1;
    p.rot = a.rot;
    p.trans = a.trans;
    p.feat = a.feat;
    p.lse = a.lse;
    const uint64_t BH = static_cast<uint64_t>(a.B) * d.heads;
    const CUtensorMap mQh = make_map_3d_f32(a.q_hi, d.dqk_pad, a.L, BH, d.dqk_pad, 32, BM);
    const CUtensorMap mQl = make_map_3d_f32(a.q_lo, d.dqk_pad, a.L, BH, d.dqk_pad, 32, BM);
    const CUtensorMap mKh = make_map_3d_f32(a.k_hi, d.dqk_pad, a.L, BH, d.dqk_pad, 32, BN);
    const CUtensorMap mKl = make_map_3d_f32(a.k_lo, d.dqk_pad, a.L, BH, d.dqk_pad, 32, BN);
    const uint64_t Lp = (static_cast<uint64_t>(a.L) + 3) / 4 * 4;
    const CUtensorMap mVh = make_map_3d_f32(a.v_hi, a.L, d.dv_pad, BH, Lp, 32, kVNc);
    const CUtensorMap mVl = make_map_3d_f32(a.v_lo, a.L, d.dv_pad, BH, Lp, 32, kVNc);
    constexpr Layout lay = smem_layout();
    const int smem = lay.total + 1024;
    static_assert(smem_layout().total + 1024 <= 232448, "3xTF32 attention: shared memory budget");
    cudaFuncSetAttribute(attn_fwd_f32tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    dim3 grid((a.L + BM - 1) / BM, static_cast<unsigned>(BH));
    attn_fwd_f32tc_kernel<<<grid, kThreads, smem, stream>>>(mQh, mQl, mKh, mKl, mVh, mVl, p);
}

}  // namespace fipa_b200
