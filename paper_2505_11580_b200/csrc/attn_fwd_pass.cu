// FlashIPA attention forward for wide lifted rows (z_factor_rank 3-4: D_qk 560-688, D_v 554-682)
// on a CTA pair (tcgen05 cta_group::2, M = 256), two passes over the keys.
//
// Same algorithm as attn_fwd_2sm.cu (proj/src/attention_kernel.cpp:112-188 + the epilogue of
// proj/src/flash_ipa.cpp:171-210); what changes is the budget.  The value accumulator of a
// 128-row tile no longer fits TMEM (512 columns) next to S, and a whole K tile no longer fits
// shared memory next to the resident Q tile, so:
//   * the value columns are split in two passes.  Pass 0 accumulates O0 = [v | z2 rho < rho_a]
//     with the online softmax; between the passes the epilogue writes the scalar block straight
//     to the features and parks the partial pair aggregate sum_{rho<rho_a} z1 * O0 in TMEM.
//     Pass 1 recomputes S (bit-identical MMAs), applies the FINAL running max and 1/l of pass 0
//     (no rescales, no denominator), accumulates O1 = [z2 rho >= rho_a | t hi | t lo | R v_p] and
//     finishes the pair contraction and the points.  Extra work: one Q.K^T per pass (x1.5 FLOPs
//     at rank 3-4) in exchange for tensor cores instead of the fp32 SIMT path.
//   * K streams through a ring of 128-byte column-block groups (kb blocks x 32 keys per CTA)
//     instead of whole tiles; V slices are 16 or 32 keys.  Ring depths are chosen on the host
//     from the shared-memory budget.
// TMEM: S [0,64) | P [64,96) (bf16 pairs, the A operand of the P.V MMAs: no shared-memory P tile,
// which leaves that 16 KB to the operand rings) | partial pair aggregate (bf16 pairs) [96, 96+d_z/2)
// | O1 [96+d_z/2, ...) ; O0 [512-N0, 512) (O0 may overlap the aggregate only in its scalar columns,
// which are consumed first).
//
// Warps (352 threads per CTA): w0 Q/K producer, w1 TMEM alloc (+ MMA issue on the even CTA),
// w2..w9 softmax + epilogue (quadrant w%4, key half (w-2)/4), w10 V producer.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "kernels.hpp"
#include "ptx.cuh"
#include "tma_host.hpp"

namespace fipa_b200 {

namespace {

constexpr int BM = 128;  // query rows per CTA (256 per pair)
constexpr int BN = 64;   // keys per tile
constexpr int kThreads = 352;
constexpr int kMaxPoints = 14;
constexpr uint32_t kPc = 64;   // TMEM column of the bf16 P tile (64 keys = 32 columns)
constexpr uint32_t kOz = 96;   // TMEM column of the bf16-packed partial pair aggregate (d_z / 2 columns)
constexpr float kLn2 = 0.6931471805599453f;
constexpr int kSmemLimit = 232448;

struct PassParams {
    int L, H, Lk, kchunk;
    int n_qkb, qk_steps;
    int kb, kst, nkst;  // K ring: blocks per stage, stages, stages per tile
    int vkeys, vst;     // V ring: keys per slice, stages
    int N[2], na[2], nb[2], boxa[2], boxb[2], vcol0[2], ob[2];
    int rho_a;
    int c, d_z, rank, n_value, seg, feat_ld;
    const float* z1;
    const float* rot;
    const float* trans;
    __nv_bfloat16* feat_out;
    float* lse;
};

struct Bars {
    uint64_t q_full;
    uint64_t k_full[4], k_empty[4];
    uint64_t v_full[4], v_empty[4];
    uint64_t s_full, s_free, p_full, pv_done, o_full;
    uint32_t tmem_slot;
};

struct Layout {
    int q, p, k, v, xch, bars, total, kstage, vstage;
};
__host__ __device__ inline Layout smem_layout(int n_qkb, int kb, int kst, int vkeys, int vst, int vboxes) {
    Layout l{};
    l.kstage = kb * 32 * 128;
    l.vstage = vboxes * vkeys * 128;
    l.q = 0;
    l.p = 0;  // (P lives in TMEM)
    l.k = n_qkb * BM * 128;
    l.v = l.k + kst * l.kstage;
    l.xch = l.v + vst * l.vstage;
    l.bars = l.xch + 2 * 2 * BM * 4;
    l.total = l.bars + static_cast<int>(sizeof(Bars));
    return l;
}
__host__ __device__ constexpr int stage_stride(int seg) { return (seg + 7) / 8 * 8 + 8; }

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void load_z16(const float* zp, bool vec, int rem, float* z) {
    if (vec && rem >= 16) {
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
        for (int e = 0; e < 16; ++e) z[e] = e < rem ? __ldg(zp + e) : 0.f;
    }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    attn_fwd_pass_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
                         const __grid_constant__ CUtensorMap mapV, PassParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int vboxes = max(p.boxa[0] + p.boxb[0], p.boxa[1] + p.boxb[1]);
    const Layout lay = smem_layout(p.n_qkb, p.kb, p.kst, p.vkeys, p.vst, vboxes);
    uint8_t* sQ = smem + lay.q;
    uint8_t* sK = smem + lay.k;
    uint8_t* sV = smem + lay.v;
    Bars* bars = reinterpret_cast<Bars*>(smem + lay.bars);

    const int warp = ptx::warp_id();
    const int lane = ptx::lane_id();
    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    const int bh = blockIdx.y;
    const int q0 = blockIdx.x * BM;
    const int ntiles = (p.Lk + BN - 1) / BN;
    const int T = 2 * ntiles;  // tiles over both passes
    const int slices = BN / p.vkeys;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&mapQ);
        ptx::tma_prefetch(&mapK);
        ptx::tma_prefetch(&mapV);
        ptx::mbar_init(&bars->q_full, 1);
        for (int s = 0; s < p.kst; ++s) {
            ptx::mbar_init(&bars->k_full[s], 1);
            ptx::mbar_init(&bars->k_empty[s], 1);
        }
        for (int s = 0; s < p.vst; ++s) {
            ptx::mbar_init(&bars->v_full[s], 1);
            ptx::mbar_init(&bars->v_empty[s], 1);
        }
        ptx::mbar_init(&bars->s_full, 1);
        ptx::mbar_init(&bars->s_free, 16);
        ptx::mbar_init(&bars->p_full, 16);
        ptx::mbar_init(&bars->pv_done, 1);
        ptx::mbar_init(&bars->o_full, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc_2sm(&bars->tmem_slot, 512);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, bars->tmem_slot, 0);

    if (warp == 0) {
        // --------------------------------------------------------- Q / K producer
        if (lane == 0) {
            if (leader) ptx::mbar_expect_tx(&bars->q_full, 2 * p.n_qkb * BM * 128);
            ptx::tma_load_4d_2sm(sQ, &mapQ, &bars->q_full, 0, q0, 0, bh);
            int n = 0;
            for (int t = 0; t < T; ++t) {
                const int j = t % ntiles;
                const int key = j * BN + 32 * static_cast<int>(rank);
                const int g = key / p.kchunk;
                for (int u = 0; u < p.nkst; ++u, ++n) {
                    const int s = n % p.kst;
                    if (n >= p.kst) ptx::mbar_wait(&bars->k_empty[s], ((n / p.kst) - 1) & 1);
                    if (leader) ptx::mbar_expect_tx(&bars->k_full[s], 2 * lay.kstage);
                    ptx::tma_load_5d_2sm(sK + s * lay.kstage, &mapK, &bars->k_full[s], 0, key - g * p.kchunk,
                                         u * p.kb, bh, g);
                }
            }
        }
    } else if (warp == 10) {
        // --------------------------------------------------------------- V producer
        if (lane == 0) {
            int n = 0;
            for (int t = 0; t < T; ++t) {
                const int ps = t / ntiles, j = t % ntiles;
                const int ha = p.na[ps] / 2, hb = p.nb[ps] / 2;
                for (int h2 = 0; h2 < slices; ++h2, ++n) {
                    const int s = n % p.vst;
                    if (n >= p.vst) ptx::mbar_wait(&bars->v_empty[s], ((n / p.vst) - 1) & 1);
                    if (leader) ptx::mbar_expect_tx(&bars->v_full[s], 2 * (p.boxa[ps] + p.boxb[ps]) * p.vkeys * 128);
                    uint8_t* dst = sV + s * lay.vstage;
                    const int key = j * BN + h2 * p.vkeys;
                    const int g = key / p.kchunk, kk = key - g * p.kchunk;
                    const int c0 = p.vcol0[ps];
                    for (int x = 0; x < p.boxa[ps]; ++x)
                        ptx::tma_load_4d_2sm(dst + x * p.vkeys * 128, &mapV, &bars->v_full[s],
                                             c0 + ha * static_cast<int>(rank) + 64 * x, kk, bh, g);
                    for (int x = 0; x < p.boxb[ps]; ++x)
                        ptx::tma_load_4d_2sm(dst + (p.boxa[ps] + x) * p.vkeys * 128, &mapV, &bars->v_full[s],
                                             c0 + p.na[ps] + hb * static_cast<int>(rank) + 64 * x, kk, bh, g);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issue (even CTA only)
        if (leader) {
            const uint32_t idesc_qk = ptx::idesc_bf16(256, BN, false, false);
            const uint32_t q_base = ptx::smem_u32(sQ);
            const uint32_t k_base = ptx::smem_u32(sK);
            const uint32_t v_base = ptx::smem_u32(sV);
            ptx::mbar_wait(&bars->q_full, 0);
            // ring slots / phases and the (pass, tile) position advance by counters: no integer
            // division on the issue path
            int ks = 0, kph = 0, vs = 0, vph = 0;
            const uint64_t dq0 = ptx::sw128_desc(q_base, 16, 1024);
            const uint64_t dk0 = ptx::sw128_desc(k_base, 16, 1024);
            const uint64_t dv0 = ptx::sw128_desc(v_base, p.vkeys * 128, 1024);
            for (int t = 0, ps_prev = 0, jj = -1; t <= T; ++t) {
                if (t < T) {
                    if (t > 0) ptx::mbar_wait_cluster(&bars->s_free, (t - 1) & 1);
                    for (int u = 0; u < p.nkst; ++u) {
                        ptx::mbar_wait(&bars->k_full[ks], kph);
                        ptx::tc_fence_after();
                        if (ptx::elect_one()) {
                            const uint64_t dks = dk0 + static_cast<uint64_t>((ks * lay.kstage) >> 4);
                            const int k_lo = u * p.kb * 4;
                            const int k_n = min(p.qk_steps - k_lo, p.kb * 4);
#pragma unroll 8
                            for (int e = 0; e < k_n; ++e) {
                                const int kk = k_lo + e;
                                const uint64_t da = dq0 + static_cast<uint64_t>(((kk >> 2) * (BM * 128) + (kk & 3) * 32) >> 4);
                                const uint64_t db = dks + static_cast<uint64_t>(((e >> 2) * (32 * 128) + (e & 3) * 32) >> 4);
                                ptx::mma2_ss(tmem, da, db, idesc_qk, kk != 0);
                            }
                            ptx::mma_commit_2sm(&bars->k_empty[ks], 0x3);
                            if (u == p.nkst - 1) ptx::mma_commit_2sm(&bars->s_full, 0x3);
                        }
                        __syncwarp();
                        if (++ks == p.kst) {
                            ks = 0;
                            kph ^= 1;
                        }
                    }
                }
                if (t > 0) {
                    const int tt = t - 1;
                    if (++jj == ntiles) {
                        jj = 0;
                        ps_prev = 1;
                    }
                    const int ps = ps_prev;
                    const uint32_t idesc_a = ptx::idesc_bf16(256, p.na[ps], false, true);
                    const uint32_t idesc_b = ptx::idesc_bf16(256, p.nb[ps] > 0 ? p.nb[ps] : 16, false, true);
                    const uint32_t boxb = p.vkeys * 128;
                    const uint32_t oa = tmem + p.ob[ps], obb = oa + p.na[ps];
                    const bool two = p.nb[ps] > 0;
                    ptx::mbar_wait_cluster(&bars->p_full, tt & 1);
                    for (int h2 = 0; h2 < slices; ++h2) {
                        ptx::mbar_wait(&bars->v_full[vs], vph);
                        ptx::tc_fence_after();
                        if (ptx::elect_one()) {
                            const uint64_t db0 = dv0 + static_cast<uint64_t>((vs * lay.vstage) >> 4);
                            for (int kk = 0; kk < p.vkeys / 16; ++kk) {
                                // A = P from TMEM: 16 keys = 8 columns of bf16 pairs
                                const uint32_t a_tm = tmem + kPc + (h2 * (p.vkeys / 16) + kk) * 8;
                                const uint64_t db = db0 + static_cast<uint64_t>((kk * 2048) >> 4);
                                const uint32_t acc = (jj > 0 || h2 > 0 || kk > 0) ? 1u : 0u;
                                ptx::mma2_ts(oa, a_tm, db, idesc_a, acc);
                                if (two)
                                    ptx::mma2_ts(obb, a_tm, db + static_cast<uint64_t>((p.boxa[ps] * boxb) >> 4),
                                                 idesc_b, acc);
                            }
                            ptx::mma_commit_2sm(&bars->v_empty[vs], 0x3);
                        }
                        __syncwarp();
                        if (++vs == p.vst) {
                            vs = 0;
                            vph ^= 1;
                        }
                    }
                    if (ptx::elect_one()) {
                        ptx::mma_commit_2sm(&bars->pv_done, 0x3);
                        if (tt == T - 1) ptx::mma_commit_2sm(&bars->o_full, 0x3);
                    }
                    __syncwarp();
                }
            }
        }
    } else {
        // ------------------------------------------------------- softmax + epilogue
        const int sw = warp - 2;
        const int quad = warp & 3;
        const int half = sw >> 2;
        const int row = quad * 32 + lane;
        const uint32_t tl = tmem + (uint32_t(quad * 32) << 16);
        const uint32_t s_free_remote = ptx::mapa(&bars->s_free, 0);
        const uint32_t p_full_remote = ptx::mapa(&bars->p_full, 0);
        float* xch = reinterpret_cast<float*>(smem + lay.xch);  // [2 parity][2 half][128 rows]
        const int H = p.H, b = bh / H, h = bh % H;
        const int qi = q0 + row;
        const bool ok = qi < p.L;
        const int64_t grow = static_cast<int64_t>(b) * p.L + (ok ? qi : 0);
        const int c = p.c, dz = p.d_z, Nv = p.n_value;
        const float* z1r = p.z1 + grow * (p.rank * dz);
        const bool zvec = (reinterpret_cast<uintptr_t>(z1r) & 15) == 0;
        float m = -INFINITY, l = 0.f, inv_l = 0.f;

        for (int t = 0; t < T; ++t) {
            const int ps = t / ntiles, j = t % ntiles;
            ptx::mbar_wait(&bars->s_full, t & 1);
            ptx::tc_fence_after();
            uint32_t sr[32];
            ptx::tmem_ld32(tl + 32 * half, sr);
            ptx::tmem_wait_ld();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster_relaxed(s_free_remote);

            float x[32];
            const int kvalid = p.Lk - j * BN - 32 * half;
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) x[cc] = cc < kvalid ? __uint_as_float(sr[cc]) : -INFINITY;
            bool need = false;
            float scale = 1.0f;
            if (ps == 0) {
                float mx[8];
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    mx[k] = fmaxf(fmaxf(x[4 * k], x[4 * k + 1]), fmaxf(x[4 * k + 2], x[4 * k + 3]));
#pragma unroll
                for (int k = 0; k < 4; ++k) mx[k] = fmaxf(mx[k], mx[k + 4]);
                float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
                float* xb = xch + (j & 1) * 256;
                xb[half * 128 + row] = mt;
                named_bar_sync(2 + quad, 64);
                mt = fmaxf(mt, xb[(half ^ 1) * 128 + row]);
                need = mt > m + 8.0f;
                if (need) {
                    scale = ptx::ex2(m - mt);
                    m = mt;
                    l *= scale;
                }
            }
            const float mm = m == -INFINITY ? 0.f : m;
            uint32_t pk[16];
            float ls[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int cc = 0; cc < 16; ++cc) {
                const float p0 = ptx::ex2(x[2 * cc] - mm);
                const float p1 = ptx::ex2(x[2 * cc + 1] - mm);
                ls[cc & 3] += p0 + p1;
                pk[cc] = ptx::pack_bf16x2(p0, p1);
            }
            if (ps == 0) l += (ls[0] + ls[1]) + (ls[2] + ls[3]);

            if (t > 0) {
                ptx::mbar_wait(&bars->pv_done, (t - 1) & 1);
                ptx::tc_fence_after();
                if (ps == 0 && __any_sync(0xffffffffu, need)) {
                    const int n16 = p.N[0] / 16;
                    const int lo = half ? (n16 + 1) / 2 : 0, hi = half ? n16 : (n16 + 1) / 2;
                    for (int ch = lo; ch < hi; ++ch) {
                        uint32_t o[16];
                        ptx::tmem_ld16(tl + p.ob[0] + 16 * ch, o);
                        ptx::tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * scale);
                        ptx::tmem_st16(tl + p.ob[0] + 16 * ch, o);
                    }
                    ptx::tmem_wait_st();
                }
            }
            if (t == ntiles) {
                // ------------------------------------------ between the passes (epilogue 1)
                // O0 is final (pv_done of the last pass-0 tile).  Denominator of the row.
                float* lb = xch + (ntiles & 1) * 256;
                lb[half * 128 + row] = l;
                named_bar_sync(2 + quad, 64);
                l += lb[(half ^ 1) * 128 + row];
                inv_l = l > 0.f ? 1.0f / l : 0.f;
                if (half == 0 && ok)
                    p.lse[static_cast<int64_t>(bh) * p.L + qi] = l > 0.f ? (m + log2f(l)) * kLn2 : -INFINITY;
                // scalar aggregate -> features [d_z, d_z + c), straight to global memory
                __nv_bfloat16* frow = p.feat_out + grow * p.feat_ld + h * p.seg + dz;
                const bool fvec = (reinterpret_cast<uintptr_t>(frow) & 15) == 0;
                const int nsc = c / 16;
                for (int ch = half ? (nsc + 1) / 2 : 0; ch < (half ? nsc : (nsc + 1) / 2); ++ch) {
                    uint32_t o[16];
                    ptx::tmem_ld16(tl + p.ob[0] + 16 * ch, o);
                    ptx::tmem_wait_ld();
                    if (ok) {
                        uint32_t w[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e)
                            w[e] = ptx::pack_bf16x2(__uint_as_float(o[2 * e]) * inv_l, __uint_as_float(o[2 * e + 1]) * inv_l);
                        if (fvec) {
                            uint4* dst = reinterpret_cast<uint4*>(frow + 16 * ch);
                            dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
                            dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
                        } else {
#pragma unroll
                            for (int e = 0; e < 8; ++e) {
                                frow[16 * ch + 2 * e] = __ushort_as_bfloat16(static_cast<unsigned short>(w[e] & 0xFFFF));
                                frow[16 * ch + 2 * e + 1] = __ushort_as_bfloat16(static_cast<unsigned short>(w[e] >> 16));
                            }
                        }
                    }
                }
                // both halves have read the scalar columns, which the aggregate may overwrite
                ptx::tc_fence_before();
                named_bar_sync(2 + quad, 64);
                ptx::tc_fence_after();
                const int npc = (dz + 15) / 16;
                for (int ch = half ? (npc + 1) / 2 : 0; ch < (half ? npc : (npc + 1) / 2); ++ch) {
                    const int d0 = 16 * ch;
                    float acc[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) acc[e] = 0.f;
                    for (int rho = 0; rho < p.rho_a; ++rho) {
                        float z[16];
                        load_z16(z1r + rho * dz + d0, zvec, dz - d0, z);
                        uint32_t o[16];
                        ptx::tmem_ld16(tl + p.ob[0] + c + rho * dz + d0, o);
                        ptx::tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 16; ++e) acc[e] = fmaf(z[e], __uint_as_float(o[e]), acc[e]);
                    }
                    uint32_t o[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) o[e] = ptx::pack_bf16x2(acc[2 * e] * inv_l, acc[2 * e + 1] * inv_l);
                    ptx::tmem_st8(tl + kOz + d0 / 2, o);
                }
                ptx::tmem_wait_st();
            }
            // P row half into TMEM (bf16 pairs): the A operand of this tile's P.V MMAs
            ptx::tmem_st16(tl + kPc + 16 * half, pk);
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_remote(p_full_remote);
        }

        // ---------------------------------------------------------- final epilogue
        ptx::mbar_wait(&bars->o_full, 0);
        ptx::tc_fence_after();
        const int seg = p.seg, sst = stage_stride(seg);
        __nv_bfloat16* fst = reinterpret_cast<__nv_bfloat16*>(smem);  // all MMAs done: smem is free
        __nv_bfloat16* frow = fst + row * sst;
        const uint32_t o1 = tl + p.ob[1];
        const int pbase = (p.rank - p.rho_a) * dz;  // point block inside O1
        if (half == 0) {
            uint32_t o[48];
            ptx::tmem_ld16(o1 + pbase, o);
            ptx::tmem_ld16(o1 + pbase + 16, o + 16);
            ptx::tmem_ld16(o1 + pbase + 32, o + 32);
            ptx::tmem_wait_ld();
            if (ok) {
                const float* R = p.rot + grow * 9;
                const float* tr = p.trans + grow * 3;
                float Rm[9], tg[3];
#pragma unroll
                for (int k = 0; k < 9; ++k) Rm[k] = __ldg(R + k);
#pragma unroll
                for (int y = 0; y < 3; ++y)
                    tg[y] = (__uint_as_float(o[y]) + __uint_as_float(o[3 + y])) * inv_l - __ldg(tr + y);
                __nv_bfloat16* fp = frow + dz + c;
#pragma unroll
                for (int pt = 0; pt < kMaxPoints; ++pt) {
                    if (pt < Nv) {
                        const float gx = __uint_as_float(o[6 + 3 * pt]) * inv_l + tg[0];
                        const float gy = __uint_as_float(o[7 + 3 * pt]) * inv_l + tg[1];
                        const float gz = __uint_as_float(o[8 + 3 * pt]) * inv_l + tg[2];
                        const float lx = fmaf(Rm[0], gx, fmaf(Rm[3], gy, Rm[6] * gz));
                        const float ly = fmaf(Rm[1], gx, fmaf(Rm[4], gy, Rm[7] * gz));
                        const float lz = fmaf(Rm[2], gx, fmaf(Rm[5], gy, Rm[8] * gz));
                        fp[3 * pt] = __float2bfloat16_rn(lx);
                        fp[3 * pt + 1] = __float2bfloat16_rn(ly);
                        fp[3 * pt + 2] = __float2bfloat16_rn(lz);
                        fp[3 * Nv + pt] = __float2bfloat16_rn(sqrtf(lx * lx + ly * ly + lz * lz));
                    }
                }
            }
        }
        const int npc = (dz + 15) / 16;
        for (int ch = half ? (npc + 1) / 2 : 0; ch < (half ? npc : (npc + 1) / 2); ++ch) {
            const int d0 = 16 * ch;
            float acc[16];
            {
                uint32_t o8[8];
                ptx::tmem_ld8(tl + kOz + d0 / 2, o8);
                ptx::tmem_wait_ld();
                uint32_t o[16];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    o[2 * e] = o8[e] << 16;              // low bf16 -> float bits
                    o[2 * e + 1] = o8[e] & 0xFFFF0000u;  // high bf16
                }
#pragma unroll
                for (int e = 0; e < 16; ++e) acc[e] = 0.f;
                for (int rho = p.rho_a; rho < p.rank; ++rho) {
                    float z[16];
                    load_z16(z1r + rho * dz + d0, zvec, dz - d0, z);
                    uint32_t v[16];
                    ptx::tmem_ld16(o1 + (rho - p.rho_a) * dz + d0, v);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 16; ++e) acc[e] = fmaf(z[e], __uint_as_float(v[e]), acc[e]);
                }
#pragma unroll
                for (int e = 0; e < 16; ++e) acc[e] = fmaf(acc[e], inv_l, __uint_as_float(o[e]));
            }
#pragma unroll
            for (int e = 0; e < 16; ++e)
                if (d0 + e < dz) frow[d0 + e] = __float2bfloat16_rn(acc[e]);
        }
        named_bar_sync(1, 256);
        const int tid = threadIdx.x - 64;
        const int rows = min(BM, p.L - q0);
        if (rows > 0) {
            __nv_bfloat16* gout = p.feat_out + (static_cast<int64_t>(b) * p.L + q0) * p.feat_ld + h * seg;
            // the row minus the scalar block (written between the passes): [0, d_z) and [d_z + c, seg)
            const int tail0 = dz + c, tail = seg - tail0;
            if (dz % 8 == 0 && tail0 % 8 == 0 && tail % 8 == 0 && p.feat_ld % 8 == 0 && (h * seg) % 8 == 0) {
                const int pa = dz / 8, per_row = pa + tail / 8;
                for (int e = tid; e < rows * per_row; e += 256) {
                    const int r = e / per_row, k = e - r * per_row;
                    const int col = k < pa ? 8 * k : tail0 + 8 * (k - pa);
                    *reinterpret_cast<uint4*>(gout + static_cast<int64_t>(r) * p.feat_ld + col) =
                        *reinterpret_cast<const uint4*>(fst + r * sst + col);
                }
            } else {
                const int per_row = dz + tail;
                for (int e = tid; e < rows * per_row; e += 256) {
                    const int r = e / per_row, k = e - r * per_row;
                    const int col = k < dz ? k : tail0 + (k - dz);
                    gout[static_cast<int64_t>(r) * p.feat_ld + col] = fst[r * sst + col];
                }
            }
        }
    }

    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 1) ptx::tmem_dealloc_2sm(tmem, 512);
}

// Host-side plan: value split, TMEM columns, ring depths that fit shared memory.
bool make_plan(const LayerDims& d, PassParams& p, Layout& lay, const int* ring = nullptr) {
    p = PassParams{};
    const int c = d.c, dz = d.d_z, r = d.rank;
    if (c % 16 != 0 || dz % 16 != 0 || r < 1 || 3 * d.n_value + 6 > 48 || d.dqk_pad % 64 != 0 ||
        d.dv_pad % 64 != 0 || d.seg > 4096)
        return false;
    // largest rho_a with pass-0 width N0 = c + rho_a*d_z inside TMEM beside S and the aggregate
    int rho_a = -1;
    // TS MMAs (A = P from TMEM) need N % 32 == 0: both passes are padded to 32 columns
    auto up32 = [](int x) { return (x + 31) / 32 * 32; };
    if (dz % 32 != 0) return false;
    for (int ra = r; ra >= 0; --ra) {
        const int N0 = c + ra * dz, N1 = up32(d.dv_mma - N0);
        const int ob0 = 512 - N0, ob1 = static_cast<int>(kOz) + dz / 2;
        if (N0 < 32 || N0 % 32 != 0 || N1 < 32 || N0 > 448) continue;
        if (ob0 < static_cast<int>(kPc) + 32 || ob0 + c < ob1) continue;  // aggregate overlaps scalar cols only
        if (ob1 + N1 > 512 || N0 + N1 > d.dv_pad) continue;
        rho_a = ra;
        break;
    }
    if (rho_a < 0) return false;
    p.rho_a = rho_a;
    p.N[0] = c + rho_a * dz;
    p.N[1] = up32(d.dv_mma - p.N[0]);
    p.vcol0[0] = 0;
    p.vcol0[1] = p.N[0];
    p.ob[0] = 512 - p.N[0];
    p.ob[1] = static_cast<int>(kOz) + dz / 2;
    for (int ps = 0; ps < 2; ++ps) {
        p.na[ps] = std::min(p.N[ps], 256);
        p.nb[ps] = p.N[ps] - p.na[ps];
        if (p.nb[ps] > 256) return false;
        p.boxa[ps] = (p.na[ps] / 2 + 63) / 64;
        p.boxb[ps] = (p.nb[ps] / 2 + 63) / 64;
    }
    p.n_qkb = (d.dqk_mma + 63) / 64;
    p.qk_steps = d.dqk_mma / 16;
    const int vboxes = std::max(p.boxa[0] + p.boxb[0], p.boxa[1] + p.boxb[1]);
    // ring depths, preferred first: bytes in flight and few, large K stages (each stage costs a
    // barrier round trip; 4 KB stages measured 1.3x slower than 12 KB ones at rank 3)
    const int cand[][4] = {{4, 3, 32, 2}, {3, 3, 32, 2}, {4, 2, 32, 2}, {3, 2, 32, 2}, {2, 3, 32, 2}, {3, 2, 16, 3}, {3, 2, 16, 2},
                           {2, 2, 32, 2}, {2, 2, 16, 3}, {2, 2, 16, 2}, {1, 4, 16, 2}, {1, 3, 16, 2}, {1, 2, 16, 2}};
    int forced[4] = {0, 0, 0, 0};  // AttnArgs::pass_ring (Tuning::pass_ring): tuning experiments
    if (ring != nullptr)
        for (int i = 0; i < 4; ++i) forced[i] = ring[i];
    for (const auto& cd0 : cand) {
        const int* cd = forced[0] > 0 ? forced : cd0;
        if (cd[1] > 4 || cd[3] > 4) return false;
        const Layout l = smem_layout(p.n_qkb, cd[0], cd[1], cd[2], cd[3], vboxes);
        if (l.total + 1024 <= kSmemLimit && BM * stage_stride(d.seg) * 2 <= l.xch) {
            p.kb = cd[0];
            p.kst = cd[1];
            p.vkeys = cd[2];
            p.vst = cd[3];
            p.nkst = (p.n_qkb + p.kb - 1) / p.kb;
            lay = l;
            return true;
        }
    }
    return false;
}

}  // namespace

bool attn_fwd_pass_supported(const LayerDims& d) {
    PassParams p;
    Layout l;
    return make_plan(d, p, l);
}

void launch_attn_fwd_pass(const LayerDims& d, const AttnArgs& a, cudaStream_t stream) {
    PassParams p;
    Layout lay;
    if (!make_plan(d, p, lay, a.pass_ring))
        throw std::invalid_argument("tcgen05 two-pass attention: lifted widths unsupported (use precision='f32')");
    if (a.o_save != nullptr) throw std::invalid_argument("two-pass attention: no training forward (O_hat save)");
    p.L = a.L;
    p.H = d.heads;
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
    p.Lk = a.Lk > 0 ? a.Lk : a.L;
    p.kchunk = a.kchunk > 0 ? a.kchunk : p.Lk;
    const int G = (p.Lk + p.kchunk - 1) / p.kchunk;
    if (G * p.kchunk != p.Lk || (G > 1 && p.kchunk % BN != 0))
        throw std::invalid_argument("attention: key shards must be equal and a multiple of 64 rows");
    const uint64_t BH = static_cast<uint64_t>(a.B) * d.heads;
    const CUtensorMap mapQ = make_map_blocks_bf16(a.qhat, a.L, BH, d.dqk_pad, BM, p.n_qkb);
    const CUtensorMap mapK = make_map_blocks_bf16_sharded(a.khat, p.kchunk, BH, G, d.dqk_pad, 32, p.kb);
    const CUtensorMap mapV = make_map_4d_bf16_sharded(a.vhat, d.dv_pad, p.kchunk, BH, G, 64, p.vkeys);
    const int smem = lay.total + 1024;
    cudaFuncSetAttribute(attn_fwd_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int qtiles = (a.L + BM - 1) / BM;
    dim3 grid(static_cast<unsigned>((qtiles + 1) / 2 * 2), static_cast<unsigned>(BH));
    attn_fwd_pass_kernel<<<grid, kThreads, smem, stream>>>(mapQ, mapK, mapV, p);
}

}  // namespace fipa_b200
