// FlashIPA attention forward on a CTA pair (tcgen05 cta_group::2, M = 256), fused epilogue.
//
// Replaces the reference's tiled online-softmax kernel
//   flash_attention -> flash_block   proj/src/attention_kernel.cpp:112-188, 213-243
// and the per-row epilogue that follows it
//   split / pair contraction / apply_inverse / norms   proj/src/flash_ipa.cpp:171-210
//
// A cluster of two CTAs owns 256 consecutive query rows of one (sample, head); each CTA keeps
// its 128 rows of Q_hat resident in shared memory and its 128 rows of O in its own TMEM.  The
// even CTA issues every MMA for the pair:
//   S_j = Q_hat . K_hat_j^T   M=256 N=64  (each CTA stages 32 of the 64 keys)  -> TMEM [448,512)
//   P_j = exp2(S_j - m)       softmax warps of both CTAs, bf16 P -> shared memory (K-major)
//   O  += P_j . V_hat_j       M=256 N=256+176 (each CTA stages half of every N block)
//                                                                              -> TMEM [0,432)
// Lifted rows are in log2 units with the column bias folded in (pack.cu) and stored with a
// 64-element (128-byte) row stride, so Q and each K tile arrive as ONE 4-D TMA box of 128-byte
// column blocks (the TMA engine costs ~100 cycles per box, so box count matters more than
// bytes).  K (whole tiles) and V (32-key slices) stream through two-stage rings fed by 2-SM TMA
// loads whose bytes are counted on the even CTA's barriers; consumption is signalled back to
// both CTAs by multicast tcgen05.commit.
// The tensor pipe runs QK_{j+1} while the softmax warps turn S_j into P_j, then PV_j.  The
// running max moves only when it grows by more than 2^8, so the O rescale is rare.
// Masked keys carry a -1e30 bias and vanish once any valid key is seen; keys >= L are forced
// to -inf; rows with no valid key are zeroed by the output projection (flash_ipa.cpp:213-216).
//
// Warps (352 threads per CTA): w0 Q/K producer, w1 TMEM alloc (+ MMA issue on the even CTA),
// w2..w9 softmax (warp w owns TMEM lanes 32*(w%4).. and key half (w-2)/4, thread = query row;
// all eight also run the epilogue), w10 V producer.
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

constexpr int BM = 128;      // query rows per CTA (256 per pair)
constexpr int BN = 64;       // keys per tile
constexpr int kThreads = 352;
constexpr int kKStages = 2;  // K ring: whole tiles (32 keys per CTA x all 128-byte blocks)
constexpr int kVStages = 2;  // V ring: 32-key slices x half the value width
constexpr int kVKeys = 32;
constexpr int kVBoxBytes = kVKeys * 128;  // one 64-wide MN atom column block of 32 keys
constexpr uint32_t kSCol = 448;
constexpr float kLn2 = 0.6931471805599453f;

struct Attn2Params {
    int L, H, dqk_mma, dv_mma, n_qkb, n1, n2, nb1, nb2;
    int Lk, kchunk;  // keys: Lk total, stored as shards of kchunk rows (kchunk % 64 == 0 or == Lk)
    int c, d_z, rank, n_value, seg, feat_ld;
    int z1_tma;  // z1 staged by TMA into shared memory for the epilogue
    const float* z1;
    const float* rot;
    const float* trans;
    __nv_bfloat16* feat_out;
    float* lse;
    float* o_save;  // [BH, L, dv_pad] normalised O_hat (fp32) for the backward, or null
    int dv_pad;
    int feat_tma;  // feature blocks written by per-warp TMA stores (fast epilogue shapes)
    int h0, hc;    // head sub-range [h0, h0 + hc) of every sample (grid.y = B * hc); hc = H: all
};

struct Bars {
    uint64_t q_full;
    uint64_t k_full[kKStages], k_empty[kKStages];
    uint64_t v_full[kVStages], v_empty[kVStages];
    uint64_t s_full, s_free, p_full, pv_done, o_full, z_full;
    uint32_t tmem_slot;
};

struct Layout {
    int q, p, k, v, xch, bars, total, kstage, vstage;
};
__host__ __device__ inline Layout smem_layout(int n_qkb, int nb1, int nb2) {
    Layout l{};
    l.kstage = n_qkb * 32 * 128;
    l.vstage = (nb1 + nb2) * kVBoxBytes;
    l.q = 0;
    l.p = n_qkb * BM * 128;
    l.k = l.p + BM * 128;
    l.v = l.k + kKStages * l.kstage;
    l.xch = l.v + kVStages * l.vstage;
    l.bars = l.xch + 2 * 2 * BM * 4;
    l.total = l.bars + static_cast<int>(sizeof(Bars));
    return l;
}
__host__ __device__ constexpr int epilogue_smem(int seg) {
    // row-major staging rows of (seg rounded to 8) + 8 bf16, or 64-column swizzled blocks
    return (BM * ((seg + 7) / 8 * 8 + 8) * 2 + 1023) / 1024 * 1024 > (seg + 63) / 64 * BM * 128
               ? (BM * ((seg + 7) / 8 * 8 + 8) * 2 + 1023) / 1024 * 1024
               : (seg + 63) / 64 * BM * 128;
}

// Optional per-event timestamps of clusters (0,0) for pipeline analysis (tools/attn_trace2.cu).
#ifdef FIPA_ATTN_TRACE
__device__ long long g_attn_trace[2 * 16 * 16 * 128];  // [cta][warp][event][index]
#define FIPA_TRACE(ev, j)                                                                          \
    do {                                                                                           \
        if (blockIdx.x < 2 && blockIdx.y == 0 && (j) < 128)                                         \
            g_attn_trace[((blockIdx.x * 16 + ptx::warp_id()) * 16 + (ev)) * 128 + (j)] = clock64(); \
    } while (0)
#else
#define FIPA_TRACE(ev, j) \
    do {                  \
    } while (0)
#endif

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Fused output epilogue (proj/src/flash_ipa.cpp:171-210), one thread per query row reading the
// row's O accumulator straight from TMEM; the two warps of a lane quadrant split the columns:
//   feat block = [ sum_rho z1[i,rho,:] * O_pair[rho,:] | O_scalar | R_i^T(g_p - t_i) | |.| ]
// with g_p = agg(t_j hi) + agg(t_j lo) + agg(R_j v_p) (value point block [t hi|t lo|R v_p]).
// z1 rows arrive by one TMA (swizzled 128-byte blocks, conflict-free 16-byte reads) issued when
// the accumulator is final; shapes the TMA path does not cover read z1 from global instead.
// Rows are assembled as bf16 in shared memory and written out with coalesced 16-byte stores.
constexpr int kMaxPoints = 14;

__device__ __forceinline__ void load_z16_global(const float* zp, bool vec, int rem, float* z) {
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

// 16 consecutive floats (f % 16 == 0) of row `row` from the swizzled z1 staging block.
__device__ __forceinline__ void load_z16_smem(const uint8_t* zs, int row, int f, float* z) {
    const uint8_t* rb = zs + (f >> 5) * (BM * 128) + row * 128;
    const int k0 = (f & 31) >> 2;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float4 v = *reinterpret_cast<const float4*>(rb + (((k0 + k) ^ (row & 7)) << 4));
        z[4 * k] = v.x;
        z[4 * k + 1] = v.y;
        z[4 * k + 2] = v.z;
        z[4 * k + 3] = v.w;
    }
}

// Points block of one row (half 0), branch-free over kMaxPoints so the independent points
// interleave: local = R_i^T (g - t_i) (proj/src/geometry.cpp:70-76) and |local|, as bf16 pairs.
template <bool SW>
__device__ __forceinline__ void epilogue_points(uint32_t tl_pts, float inv_l, int Nv, const float* Rm,
                                                const float* tv, __nv_bfloat16* fp, bool ok,
                                                uint8_t* blk = nullptr, int row = 0) {
    uint32_t o[48];  // warp-collective TMEM loads: every lane, rows past L included
    ptx::tmem_ld16(tl_pts, o);
    ptx::tmem_ld16(tl_pts + 16, o + 16);
    ptx::tmem_ld16(tl_pts + 32, o + 32);
    ptx::tmem_wait_ld();
    if (!ok) return;
    float tg[3];
#pragma unroll
    for (int y = 0; y < 3; ++y) tg[y] = (__uint_as_float(o[y]) + __uint_as_float(o[3 + y])) * inv_l - tv[y];
    float v[3 * kMaxPoints], nrm[kMaxPoints];
#pragma unroll
    for (int pt = 0; pt < kMaxPoints; ++pt) {
        const float gx = fmaf(__uint_as_float(o[6 + 3 * pt]), inv_l, tg[0]);
        const float gy = fmaf(__uint_as_float(o[7 + 3 * pt]), inv_l, tg[1]);
        const float gz = fmaf(__uint_as_float(o[8 + 3 * pt]), inv_l, tg[2]);
        const float lx = fmaf(Rm[0], gx, fmaf(Rm[3], gy, Rm[6] * gz));
        const float ly = fmaf(Rm[1], gx, fmaf(Rm[4], gy, Rm[7] * gz));
        const float lz = fmaf(Rm[2], gx, fmaf(Rm[5], gy, Rm[8] * gz));
        v[3 * pt] = lx;
        v[3 * pt + 1] = ly;
        v[3 * pt + 2] = lz;
        const float n2 = fmaf(lx, lx, fmaf(ly, ly, lz * lz));
        nrm[pt] = n2 > 0.f ? n2 * rsqrtf(n2) : 0.f;
    }
    // [x0 y0 z0 x1 ... | n0 n1 ...]: 3*Nv coordinates then Nv norms
    const int nc = 3 * Nv;
    if (SW) {  // Nv even: bf16 pairs into the swizzled staging block (element e in chunk e / 8)
        auto put2 = [&](int e, float x0, float x1) {
            *reinterpret_cast<uint32_t*>(blk + row * 128 + ((((e >> 3) ^ (row & 7))) << 4) + ((2 * e) & 15)) =
                ptx::pack_bf16x2(x0, x1);
        };
#pragma unroll
        for (int e = 0; e < 3 * kMaxPoints / 2; ++e)
            if (2 * e + 1 < nc) put2(2 * e, v[2 * e], v[2 * e + 1]);
#pragma unroll
        for (int i = 0; i < kMaxPoints / 2; ++i)
            if (2 * i + 1 < Nv) put2(nc + 2 * i, nrm[2 * i], nrm[2 * i + 1]);
        return;
    }
    if ((reinterpret_cast<uintptr_t>(fp) & 3) != 0) {
#pragma unroll
        for (int e = 0; e < 3 * kMaxPoints; ++e)
            if (e < nc) fp[e] = __float2bfloat16_rn(v[e]);
#pragma unroll
        for (int pt = 0; pt < kMaxPoints; ++pt)
            if (pt < Nv) fp[nc + pt] = __float2bfloat16_rn(nrm[pt]);
        return;
    }
    uint32_t* fp2 = reinterpret_cast<uint32_t*>(fp);
#pragma unroll
    for (int e = 0; e < 3 * kMaxPoints / 2; ++e) {
        if (2 * e + 1 < nc) {
            fp2[e] = ptx::pack_bf16x2(v[2 * e], v[2 * e + 1]);
        } else if (2 * e < nc) {
            fp[2 * e] = __float2bfloat16_rn(v[2 * e]);
        }
    }
    if ((nc & 1) == 0) {
#pragma unroll
        for (int i = 0; i < kMaxPoints / 2; ++i) {
            if (2 * i + 1 < Nv) {
                fp2[nc / 2 + i] = ptx::pack_bf16x2(nrm[2 * i], nrm[2 * i + 1]);
            } else if (2 * i < Nv) {
                fp[nc + 2 * i] = __float2bfloat16_rn(nrm[2 * i]);
            }
        }
    } else {
#pragma unroll
        for (int pt = 0; pt < kMaxPoints; ++pt)
            if (pt < Nv) fp[nc + pt] = __float2bfloat16_rn(nrm[pt]);
    }
}

// Scalar and pair blocks of one row for c = d_z = 128 and z1 staged in shared memory: each half
// owns four 16-column chunks of each block, every loop trip count and index compile-time, four
// TMEM loads in flight per wait.
__device__ __forceinline__ void put16_vec(__nv_bfloat16* dst, const float* x) {
    uint4 w0, w1;
    w0.x = ptx::pack_bf16x2(x[0], x[1]);
    w0.y = ptx::pack_bf16x2(x[2], x[3]);
    w0.z = ptx::pack_bf16x2(x[4], x[5]);
    w0.w = ptx::pack_bf16x2(x[6], x[7]);
    w1.x = ptx::pack_bf16x2(x[8], x[9]);
    w1.y = ptx::pack_bf16x2(x[10], x[11]);
    w1.z = ptx::pack_bf16x2(x[12], x[13]);
    w1.w = ptx::pack_bf16x2(x[14], x[15]);
    reinterpret_cast<uint4*>(dst)[0] = w0;
    reinterpret_cast<uint4*>(dst)[1] = w1;
}

// 16 bf16 into a 128-byte-swizzled [128 rows][64 cols] staging block (TMA store layout) at column
// col (col % 16 == 0): 16-byte chunk j of row r sits at r * 128 + ((j ^ (r & 7)) << 4)
__device__ __forceinline__ void put16_sw(uint8_t* blk, int row, int col, const float* x) {
    uint4 w0, w1;
    w0.x = ptx::pack_bf16x2(x[0], x[1]);
    w0.y = ptx::pack_bf16x2(x[2], x[3]);
    w0.z = ptx::pack_bf16x2(x[4], x[5]);
    w0.w = ptx::pack_bf16x2(x[6], x[7]);
    w1.x = ptx::pack_bf16x2(x[8], x[9]);
    w1.y = ptx::pack_bf16x2(x[10], x[11]);
    w1.z = ptx::pack_bf16x2(x[12], x[13]);
    w1.w = ptx::pack_bf16x2(x[14], x[15]);
    const int j = col >> 3;
    *reinterpret_cast<uint4*>(blk + row * 128 + ((j ^ (row & 7)) << 4)) = w0;
    *reinterpret_cast<uint4*>(blk + row * 128 + (((j + 1) ^ (row & 7)) << 4)) = w1;
}

// SW: write into the swizzled staging block `blk` (columns relative to the block) instead of
// the row-major feature row `frow`
template <bool SW>
__device__ __forceinline__ void epilogue_scalar128(uint32_t tl, float inv_l, int half, int row,
                                                   __nv_bfloat16* frow, uint8_t* blk) {
    uint32_t o[4][16];
#pragma unroll
    for (int k = 0; k < 4; ++k) ptx::tmem_ld16(tl + 64 * half + 16 * k, o[k]);
    ptx::tmem_wait_ld();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        float x[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) x[e] = __uint_as_float(o[k][e]) * inv_l;
        if (SW) {
            put16_sw(blk, row, 16 * k, x);
        } else {
            put16_vec(frow + 128 + 64 * half + 16 * k, x);
        }
    }
}

template <int RANK, bool SW>
__device__ __forceinline__ void epilogue_pair128(uint32_t tl, float inv_l, int half, int row, const uint8_t* zs,
                                                 __nv_bfloat16* frow, uint8_t* blk) {
    constexpr int CB = 4 / RANK;  // chunks per TMEM wait
#pragma unroll
    for (int b0 = 0; b0 < 4; b0 += CB) {
        uint32_t o[CB][RANK][16];
#pragma unroll
        for (int k = 0; k < CB; ++k)
#pragma unroll
            for (int r = 0; r < RANK; ++r) ptx::tmem_ld16(tl + 128 + r * 128 + 64 * half + 16 * (b0 + k), o[k][r]);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < CB; ++k) {
            const int d0 = 64 * half + 16 * (b0 + k);
            float acc[16];
#pragma unroll
            for (int r = 0; r < RANK; ++r) {
                float z[16];
                load_z16_smem(zs, row, r * 128 + d0, z);
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    acc[e] = r == 0 ? z[e] * __uint_as_float(o[k][r][e]) : fmaf(z[e], __uint_as_float(o[k][r][e]), acc[e]);
            }
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[e] *= inv_l;
            if (SW) {
                put16_sw(blk, row, 16 * (b0 + k), acc);
            } else {
                put16_vec(frow + d0, acc);
            }
        }
    }
}

__device__ __forceinline__ void fused_epilogue(const Attn2Params& p, uint32_t tl, float inv_l,
                                               int row, int q0, int bh, uint8_t* smem, int half,
                                               const uint8_t* zs, uint64_t* z_full, const float* Rm,
                                               const float* tv, const CUtensorMap* map_f,
                                               const CUtensorMap* map_fp) {
    const int seg = p.seg, sst = (seg + 7) / 8 * 8 + 8;
    __nv_bfloat16* fst = reinterpret_cast<__nv_bfloat16*>(smem);
    __nv_bfloat16* frow = fst + row * sst;
    const int H = p.H, b = bh / H, h = bh % H;
    const int q = q0 + row;
    const bool ok = q < p.L;
    const int64_t grow = static_cast<int64_t>(b) * p.L + (ok ? q : 0);
    const int c = p.c, dz = p.d_z, Nv = p.n_value;
    const int base = c + p.rank * dz;

    // 16 bf16 of a feature row as two 16-byte shared-memory stores where aligned
    const bool vrow = (c % 16) == 0 && (dz % 16) == 0 && (sst % 8) == 0;
    auto put16 = [&](int col, const float* x, int n) {
        if (vrow) {
            uint4 w0, w1;
            w0.x = ptx::pack_bf16x2(x[0], x[1]);
            w0.y = ptx::pack_bf16x2(x[2], x[3]);
            w0.z = ptx::pack_bf16x2(x[4], x[5]);
            w0.w = ptx::pack_bf16x2(x[6], x[7]);
            w1.x = ptx::pack_bf16x2(x[8], x[9]);
            w1.y = ptx::pack_bf16x2(x[10], x[11]);
            w1.z = ptx::pack_bf16x2(x[12], x[13]);
            w1.w = ptx::pack_bf16x2(x[14], x[15]);
            reinterpret_cast<uint4*>(frow + col)[0] = w0;
            reinterpret_cast<uint4*>(frow + col)[1] = w1;
        } else {
#pragma unroll
            for (int e = 0; e < 16; ++e)
                if (e < n) frow[col + e] = __float2bfloat16_rn(x[e]);
        }
    };

    if ((threadIdx.x & 31) == 0) FIPA_TRACE(15, 0);
    const bool fast = c == 128 && dz == 128 && (p.rank == 1 || p.rank == 2) && zs != nullptr;
    if (p.feat_tma) {
        // c = d_z = 128, z1 staged, Nv even: each warp stages its 32 rows of a 64-column block
        // swizzled and writes it with one TMA store as soon as the block is complete, so the
        // feature writes overlap the rest of the epilogue: blocks [pair lo|pair hi|scalar lo|
        // scalar hi|points] of 16 KB each
        const int r0 = row & ~31;
        auto store_box = [&](int cb, const CUtensorMap* map, int col) {
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if ((threadIdx.x & 31) == 0) {
                ptx::tma_store_3d(map, smem + cb * (BM * 128) + r0 * 128, h * seg + col, q0 + r0, b);
                ptx::bulk_commit_group();
            }
        };
        epilogue_scalar128<true>(tl, inv_l, half, row, frow, smem + (2 + half) * (BM * 128));
        store_box(2 + half, map_f, 128 + 64 * half);
        if ((threadIdx.x & 31) == 0) FIPA_TRACE(15, 1);
        if (half == 0) {
            epilogue_points<true>(tl + base, inv_l, Nv, Rm, tv, nullptr, ok, smem + 4 * (BM * 128), row);
            store_box(4, map_fp, 256);
        }
        if ((threadIdx.x & 31) == 0) FIPA_TRACE(15, 2);
        ptx::mbar_wait(z_full, 0);
        if ((threadIdx.x & 31) == 0) FIPA_TRACE(15, 3);
        if (p.rank == 1) {
            epilogue_pair128<1, true>(tl, inv_l, half, row, zs, frow, smem + half * (BM * 128));
        } else {
            epilogue_pair128<2, true>(tl, inv_l, half, row, zs, frow, smem + half * (BM * 128));
        }
        store_box(half, map_f, 64 * half);
        if ((threadIdx.x & 31) == 0) {
            FIPA_TRACE(15, 4);
            FIPA_TRACE(15, 5);
            ptx::bulk_wait_group_read<0>();  // staging read before the CTA exits
        }
        return;
    }
    if (fast) {
        epilogue_scalar128<false>(tl, inv_l, half, row, frow, nullptr);
        if ((threadIdx.x & 31) == 0) FIPA_TRACE(15, 1);
        if (half == 0) epilogue_points<false>(tl + base, inv_l, Nv, Rm, tv, frow + dz + c, ok);
        if ((threadIdx.x & 31) == 0) FIPA_TRACE(15, 2);
        ptx::mbar_wait(z_full, 0);
        if ((threadIdx.x & 31) == 0) FIPA_TRACE(15, 3);
        if (p.rank == 1) {
            epilogue_pair128<1, false>(tl, inv_l, half, row, zs, frow, nullptr);
        } else {
            epilogue_pair128<2, false>(tl, inv_l, half, row, zs, frow, nullptr);
        }
    } else {
    // scalar aggregate -> [d_z, d_z + c): 16-column chunks split between the halves, four TMEM
    // loads in flight per wait (a TMEM load costs ~0.5k cycles of latency)
    const int nsc = (c + 15) / 16;
    const int sc_lo = half ? (nsc + 1) / 2 : 0, sc_hi = half ? nsc : (nsc + 1) / 2;
    for (int ch0 = sc_lo; ch0 < sc_hi; ch0 += 4) {
        uint32_t o[64];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (ch0 + k < sc_hi) ptx::tmem_ld16(tl + 16 * (ch0 + k), o + 16 * k);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (ch0 + k < sc_hi) {
                float x[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) x[e] = __uint_as_float(o[16 * k + e]) * inv_l;
                put16(dz + 16 * (ch0 + k), x, c - 16 * (ch0 + k));
            }
        }
    }
    if ((threadIdx.x & 31) == 0) FIPA_TRACE(15, 1);
    // points (half 0), all in registers: local = R_i^T (g - t_i)   (proj/src/geometry.cpp:70-76)
    if (half == 0) epilogue_points<false>(tl + base, inv_l, Nv, Rm, tv, frow + dz + c, ok);
    // pair contraction -> [0, d_z): 16-column chunks split between the halves
    const float* z1r = p.z1 + grow * (p.rank * dz);
    const bool vec = (reinterpret_cast<uintptr_t>(z1r) & 15) == 0;
    if ((threadIdx.x & 31) == 0) FIPA_TRACE(15, 2);
    if (zs != nullptr) ptx::mbar_wait(z_full, 0);
    if ((threadIdx.x & 31) == 0) FIPA_TRACE(15, 3);
    const int npc = (dz + 15) / 16;
    const int pc_lo = half ? (npc + 1) / 2 : 0, pc_hi = half ? npc : (npc + 1) / 2;
    if (p.rank <= 2) {
        // two chunks x both ranks: four TMEM loads in flight per wait
        for (int ch0 = pc_lo; ch0 < pc_hi; ch0 += 2) {
            uint32_t o[2][2][16];
#pragma unroll
            for (int k = 0; k < 2; ++k)
#pragma unroll
                for (int r = 0; r < 2; ++r)
                    if (ch0 + k < pc_hi && r < p.rank) ptx::tmem_ld16(tl + c + r * dz + 16 * (ch0 + k), o[k][r]);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (ch0 + k < pc_hi) {
                    const int d0 = 16 * (ch0 + k);
                    float acc[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) acc[e] = 0.f;
#pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        if (r < p.rank) {
                            float z[16];
                            if (zs != nullptr) {
                                load_z16_smem(zs, row, r * dz + d0, z);
                            } else {
                                load_z16_global(z1r + r * dz + d0, vec, dz - d0, z);
                            }
#pragma unroll
                            for (int e = 0; e < 16; ++e) acc[e] = fmaf(z[e], __uint_as_float(o[k][r][e]), acc[e]);
                        }
                    }
#pragma unroll
                    for (int e = 0; e < 16; ++e) acc[e] *= inv_l;
                    put16(d0, acc, dz - d0);
                }
            }
        }
    } else {
        constexpr int kMaxRank = 4;
        for (int ch = pc_lo; ch < pc_hi; ++ch) {
            const int d0 = 16 * ch;
            float acc[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[e] = 0.f;
            for (int r0 = 0; r0 < p.rank; r0 += kMaxRank) {
                uint32_t o[kMaxRank][16];  // every rank's TMEM chunk in flight before one wait
#pragma unroll
                for (int k = 0; k < kMaxRank; ++k)
                    if (r0 + k < p.rank) ptx::tmem_ld16(tl + c + (r0 + k) * dz + d0, o[k]);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int k = 0; k < kMaxRank; ++k) {
                    if (r0 + k < p.rank) {
                        float z[16];
                        if (zs != nullptr) {
                            load_z16_smem(zs, row, (r0 + k) * dz + d0, z);
                        } else {
                            load_z16_global(z1r + (r0 + k) * dz + d0, vec, dz - d0, z);
                        }
#pragma unroll
                        for (int e = 0; e < 16; ++e) acc[e] = fmaf(z[e], __uint_as_float(o[k][e]), acc[e]);
                    }
                }
            }
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[e] *= inv_l;
            put16(d0, acc, dz - d0);
        }
    }
    }  // generic shapes
    const int rows = min(BM, p.L - q0);
    __nv_bfloat16* gout = p.feat_out + (static_cast<int64_t>(b) * p.L + q0) * p.feat_ld + h * seg;
    const bool bulk = (seg * 2) % 16 == 0 && (p.feat_ld * 2) % 16 == 0 &&
                      (reinterpret_cast<uintptr_t>(gout) & 15) == 0;
    if (bulk) ptx::fence_proxy_async_smem();  // row visible to the bulk-copy engine
    if ((threadIdx.x & 31) == 0) FIPA_TRACE(15, 4);
    named_bar_sync(1, 256);
    if ((threadIdx.x & 31) == 0) FIPA_TRACE(15, 5);
    if (rows <= 0) return;
    const int tid = threadIdx.x - 64;  // 0..255 over warps 2..9
    if (bulk) {
        // one contiguous seg-wide bf16 row segment per query row, by the bulk-copy engine
        if (tid < rows) {
            ptx::bulk_store_s2g(gout + static_cast<int64_t>(tid) * p.feat_ld, fst + tid * sst, seg * 2);
            ptx::bulk_commit_group();
            ptx::bulk_wait_group_read<0>();  // shared memory stays valid until read
        }
    } else {
        for (int e = tid; e < rows * seg; e += 256) {
            const int r = e / seg, k = e - r * seg;
            gout[static_cast<int64_t>(r) * p.feat_ld + k] = fst[r * sst + k];
        }
    }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    attn_fwd_2sm_kernel(const __grid_constant__ CUtensorMap mapQ,
                        const __grid_constant__ CUtensorMap mapK,
                        const __grid_constant__ CUtensorMap mapV,
                        const __grid_constant__ CUtensorMap mapZ,
                        const __grid_constant__ CUtensorMap mapO,
                        const __grid_constant__ CUtensorMap mapF,   // features [B][L][feat_ld], box {64, 32, 1}
                        const __grid_constant__ CUtensorMap mapFP,  // same, box {4 n_value, 32, 1}
                        Attn2Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const Layout lay = smem_layout(p.n_qkb, p.nb1, p.nb2);
    uint8_t* sQ = smem + lay.q;
    uint8_t* sP = smem + lay.p;
    uint8_t* sK = smem + lay.k;
    uint8_t* sV = smem + lay.v;
    Bars* bars = reinterpret_cast<Bars*>(smem + lay.bars);

    const int warp = ptx::warp_id();
    const int lane = ptx::lane_id();
    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    // (sample, head) of this CTA pair: a head sub-range lets query-row sharding start the heads whose
    // gathered keys have landed while the rest are still on the wire (comm.cpp)
    const int bh = static_cast<int>(blockIdx.y / p.hc) * p.H + p.h0 + static_cast<int>(blockIdx.y % p.hc);
    const int q0 = blockIdx.x * BM;
    const int ntiles = (p.Lk + BN - 1) / BN;
    const int qk_steps = p.dqk_mma / 16;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&mapQ);
        ptx::tma_prefetch(&mapK);
        ptx::tma_prefetch(&mapV);
        if (p.z1_tma) ptx::tma_prefetch(&mapZ);
        if (p.feat_tma) {
            ptx::tma_prefetch(&mapF);
            ptx::tma_prefetch(&mapFP);
        }
        span_mark(0);
        ptx::mbar_init(&bars->q_full, 1);
        for (int s = 0; s < kKStages; ++s) {
            ptx::mbar_init(&bars->k_full[s], 1);
            ptx::mbar_init(&bars->k_empty[s], 1);
        }
        for (int s = 0; s < kVStages; ++s) {
            ptx::mbar_init(&bars->v_full[s], 1);
            ptx::mbar_init(&bars->v_empty[s], 1);
        }
        ptx::mbar_init(&bars->s_full, 1);
        ptx::mbar_init(&bars->s_free, 16);
        ptx::mbar_init(&bars->p_full, 16);
        ptx::mbar_init(&bars->pv_done, 1);
        ptx::mbar_init(&bars->o_full, 1);
        ptx::mbar_init(&bars->z_full, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc_2sm(&bars->tmem_slot, 512);
    ptx::tc_fence_before();
    ptx::cluster_sync();  // barrier inits + TMEM address visible to the pair
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, bars->tmem_slot, 0);
    ptx::pdl_wait();  // q/k/v_hat, colbias of the preceding pack
    ptx::pdl_trigger();

    if (warp == 0) {
        // --------------------------------------------------------- Q / K producer
        if (lane == 0) {
            if (leader) ptx::mbar_expect_tx(&bars->q_full, 2 * p.n_qkb * BM * 128);
            ptx::tma_load_4d_2sm(sQ, &mapQ, &bars->q_full, 0, q0, 0, bh);
            for (int j = 0; j < ntiles; ++j) {
                const int s = j % kKStages;
                if (j >= kKStages) ptx::mbar_wait(&bars->k_empty[s], ((j / kKStages) - 1) & 1);
                FIPA_TRACE(5, j);
                if (leader) ptx::mbar_expect_tx(&bars->k_full[s], 2 * lay.kstage);
                const int key = j * BN + 32 * static_cast<int>(rank);
                const int g = key / p.kchunk;  // keys past Lk land in shard G: TMA zero fill
                ptx::tma_load_5d_2sm(sK + s * lay.kstage, &mapK, &bars->k_full[s], 0, key - g * p.kchunk, 0, bh, g);
            }
        }
    } else if (warp == 10) {
        // --------------------------------------------------------------- V producer
        if (lane == 0) {
            const int half1 = p.n1 / 2, half2 = p.n2 / 2;
            const int nslices = ntiles * (BN / kVKeys);
            for (int n = 0; n < nslices; ++n) {
                const int s = n % kVStages;
                if (n >= kVStages) ptx::mbar_wait(&bars->v_empty[s], ((n / kVStages) - 1) & 1);
                FIPA_TRACE(6, n);
                if (leader) ptx::mbar_expect_tx(&bars->v_full[s], 2 * lay.vstage);
                uint8_t* dst = sV + s * lay.vstage;
                const int key = n * kVKeys;
                const int g = key / p.kchunk, kk = key - g * p.kchunk;
                for (int x = 0; x < p.nb1; ++x)
                    ptx::tma_load_4d_2sm(dst + x * kVBoxBytes, &mapV, &bars->v_full[s],
                                         half1 * static_cast<int>(rank) + 64 * x, kk, bh, g);
                for (int x = 0; x < p.nb2; ++x)
                    ptx::tma_load_4d_2sm(dst + (p.nb1 + x) * kVBoxBytes, &mapV, &bars->v_full[s],
                                         p.n1 + half2 * static_cast<int>(rank) + 64 * x, kk, bh, g);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issue (even CTA only)
        if (leader) {
            const uint32_t idesc_qk = ptx::idesc_bf16(256, BN, false, false);
            const uint32_t idesc_pv1 = ptx::idesc_bf16(256, p.n1, false, true);
            const uint32_t idesc_pv2 = ptx::idesc_bf16(256, p.n2 > 0 ? p.n2 : 16, false, true);
            const uint32_t q_base = ptx::smem_u32(sQ);
            const uint32_t p_base = ptx::smem_u32(sP);
            const uint32_t k_base = ptx::smem_u32(sK);
            const uint32_t v_base = ptx::smem_u32(sV);
            // descriptors advance by 64-bit adds of (byte offset >> 4)
            const uint64_t d_q = ptx::sw128_desc(q_base, 16, 1024);
            const uint64_t d_k = ptx::sw128_desc(k_base, 16, 1024);
            const uint64_t d_p = ptx::sw128_desc(p_base, 16, 1024);
            const uint64_t d_v = ptx::sw128_desc(v_base, kVBoxBytes, 1024);
            ptx::mbar_wait(&bars->q_full, 0);
            for (int j = 0; j <= ntiles; ++j) {
                if (j < ntiles) {
                    if (j > 0) ptx::mbar_wait_cluster(&bars->s_free, (j - 1) & 1);
                    if (lane == 0) FIPA_TRACE(7, j);
                    const int ks = j % kKStages;
                    ptx::mbar_wait(&bars->k_full[ks], (j / kKStages) & 1);
                    if (lane == 0) FIPA_TRACE(0, j);
                    ptx::tc_fence_after();
                    if (ptx::elect_one()) {
                        const uint64_t dk0 = d_k + static_cast<uint64_t>((ks * lay.kstage) >> 4);
                        for (int blk = 0; 4 * blk < qk_steps; ++blk) {
                            const uint64_t da_b = d_q + static_cast<uint64_t>((blk * (BM * 128)) >> 4);
                            const uint64_t db_b = dk0 + static_cast<uint64_t>((blk * (32 * 128)) >> 4);
#pragma unroll
                            for (int sub = 0; sub < 4; ++sub)
                                if (4 * blk + sub < qk_steps)
                                    ptx::mma2_ss(tmem + kSCol, da_b + 2 * sub, db_b + 2 * sub, idesc_qk, (blk | sub) != 0);
                        }
                        ptx::mma_commit_2sm(&bars->k_empty[ks], 0x3);
                        ptx::mma_commit_2sm(&bars->s_full, 0x3);
                    }
                    __syncwarp();
                }
                if (j > 0) {
                    const int jj = j - 1;
                    ptx::mbar_wait_cluster(&bars->p_full, jj & 1);
                    if (lane == 0) FIPA_TRACE(8, jj);
                    for (int h2 = 0; h2 < BN / kVKeys; ++h2) {
                        const int n = jj * (BN / kVKeys) + h2;
                        const int vs = n % kVStages;
                        ptx::mbar_wait(&bars->v_full[vs], (n / kVStages) & 1);
                        if (lane == 0 && h2 == 0) FIPA_TRACE(1, jj);
                        ptx::tc_fence_after();
                        if (ptx::elect_one()) {
#pragma unroll
                            for (int kk = 0; kk < kVKeys / 16; ++kk) {
                                const uint64_t da = d_p + static_cast<uint64_t>(((2 * h2 + kk) * 32) >> 4);
                                const uint64_t db = d_v + static_cast<uint64_t>((vs * lay.vstage + kk * 2048) >> 4);
                                const uint32_t acc = (jj > 0 || h2 > 0 || kk > 0) ? 1u : 0u;
                                ptx::mma2_ss(tmem, da, db, idesc_pv1, acc);
                                if (p.n2 > 0)
                                    ptx::mma2_ss(tmem + p.n1, da, db + static_cast<uint64_t>((p.nb1 * kVBoxBytes) >> 4),
                                                 idesc_pv2, acc);
                            }
                            ptx::mma_commit_2sm(&bars->v_empty[vs], 0x3);
                        }
                        __syncwarp();
                    }
                    if (lane == 0) FIPA_TRACE(11, jj);
                    if (ptx::elect_one()) {
                        ptx::mma_commit_2sm(&bars->pv_done, 0x3);
                        if (j == ntiles) ptx::mma_commit_2sm(&bars->o_full, 0x3);
                    }
                    __syncwarp();
                }
            }
        }
    } else {
        // ------------------------------------------------------------------ softmax
        // Eight warps: warp w handles TMEM lane quadrant w%4 (its 32 rows) and key half
        // (w-2)/4 of every S tile; the two warps of a quadrant exchange their row maxima through
        // shared memory once per tile so both halves of P share one scale.
        const int sw = warp - 2;
        const int quad = warp & 3;
        const int half = sw >> 2;
        const int row = quad * 32 + lane;
        const uint32_t tl = tmem + (uint32_t(quad * 32) << 16);
        const uint32_t s_free_remote = ptx::mapa(&bars->s_free, 0);
        const uint32_t p_full_remote = ptx::mapa(&bars->p_full, 0);
        float* xch = reinterpret_cast<float*>(smem + lay.xch);  // [2 parity][2 half][128 rows]
        uint8_t* prow = sP + row * 128;
        const int n16 = p.dv_mma / 16;                 // O rescale: 16-column chunks split by half
        const int c_lo = half ? (n16 + 1) / 2 : 0, c_hi = half ? n16 : (n16 + 1) / 2;
        float m = -INFINITY;  // running max, log2 units (identical in both halves)
        float l = 0.f;        // this half's partial denominator
        for (int j = 0; j < ntiles; ++j) {
            ptx::mbar_wait(&bars->s_full, j & 1);
            if (lane == 0) FIPA_TRACE(2, j);
            ptx::tc_fence_after();
            uint32_t sr[32];
            ptx::tmem_ld32(tl + kSCol + 32 * half, sr);
            ptx::tmem_wait_ld();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster_relaxed(s_free_remote);
            if (lane == 0) FIPA_TRACE(12, j);

            float x[32];
            const int kvalid = p.Lk - j * BN - 32 * half;  // keys >= Lk are not real
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) x[cc] = cc < kvalid ? __uint_as_float(sr[cc]) : -INFINITY;
            float mx[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) mx[k] = fmaxf(fmaxf(x[4 * k], x[4 * k + 1]), fmaxf(x[4 * k + 2], x[4 * k + 3]));
#pragma unroll
            for (int k = 0; k < 4; ++k) mx[k] = fmaxf(mx[k], mx[k + 4]);
            float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
            float* xb = xch + (j & 1) * 256;
            xb[half * 128 + row] = mt;
            named_bar_sync(2 + quad, 64);
            mt = fmaxf(mt, xb[(half ^ 1) * 128 + row]);
            const bool need = mt > m + 8.0f;  // also true on the first finite tile
            float scale = 1.0f;
            if (need) {
                scale = ptx::ex2(m - mt);  // 0 when m == -inf
                m = mt;
                l *= scale;
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
            l += (ls[0] + ls[1]) + (ls[2] + ls[3]);
            if (lane == 0) FIPA_TRACE(13, j);

            // P_j overwrites P_{j-1} (and O may be rescaled) only once PV_{j-1} is done.
            if (j > 0) {
                ptx::mbar_wait(&bars->pv_done, (j - 1) & 1);
                if (lane == 0) FIPA_TRACE(3, j);
                ptx::tc_fence_after();
                if (__any_sync(0xffffffffu, need)) {
                    for (int ch = c_lo; ch < c_hi; ++ch) {
                        uint32_t o[16];
                        ptx::tmem_ld16(tl + 16 * ch, o);
                        ptx::tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * scale);
                        ptx::tmem_st16(tl + 16 * ch, o);
                    }
                    ptx::tmem_wait_st();
                }
            }
            if (lane == 0) FIPA_TRACE(14, j);
            // P row half (32 keys, 64 B) in the SWIZZLE_128B K-major layout: 16-byte chunk k of
            // row r lives at chunk k ^ (r % 8).
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int chunk = 4 * half + k;
                const uint4 v = make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
                *reinterpret_cast<uint4*>(prow + ((chunk ^ (row & 7)) << 4)) = v;
            }
            ptx::fence_proxy_async_smem();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_remote(p_full_remote);
            if (lane == 0) FIPA_TRACE(4, j);
        }

        // -------------------------------------------------------------- epilogue
        float* lb = xch + (ntiles & 1) * 256;
        lb[half * 128 + row] = l;
        named_bar_sync(2 + quad, 64);
        l += lb[(half ^ 1) * 128 + row];
        // residue frame for the point epilogue, fetched while the last PV MMAs run
        float Rm[9], tv[3];
        {
            const int qi = q0 + row;
            const int64_t g = static_cast<int64_t>(bh / p.H) * p.L + (qi < p.L ? qi : 0);
            if (half == 0) {
#pragma unroll
                for (int k = 0; k < 9; ++k) Rm[k] = __ldg(p.rot + g * 9 + k);
#pragma unroll
                for (int y = 0; y < 3; ++y) tv[y] = __ldg(p.trans + g * 3 + y);
            }
        }
        ptx::mbar_wait(&bars->o_full, 0);
        if (lane == 0) FIPA_TRACE(9, 0);
        if (warp == 2 && lane == 0) span_mark(1);
        ptx::tc_fence_after();
        const float inv_l = l > 0.f ? 1.0f / l : 0.f;
        const int qi = q0 + row;
        if (half == 0 && qi < p.L)
            p.lse[static_cast<int64_t>(bh) * p.L + qi] = l > 0.f ? (m + log2f(l)) * kLn2 : -INFINITY;
        uint8_t* zs = smem + epilogue_smem(p.seg);
        // z1 rows by TMA (all MMAs are complete, so the Q/K/V/P regions are free), issued before the
        // O_hat save when the save's staging chunks [0, 64 KB) stay clear of the z1 region
        const bool z_early = epilogue_smem(p.seg) >= 4 * BM * 128;
        auto issue_z1 = [&]() {
            if (p.z1_tma && warp == 2 && lane == 0) {
                ptx::mbar_expect_tx(&bars->z_full, BM * p.rank * p.d_z * 4);
                ptx::tma_load_3d(zs, &mapZ, &bars->z_full, 0, (bh / p.H) * p.L + q0, 0);
            }
        };
        if (z_early || p.o_save == nullptr) issue_z1();
        if (p.o_save != nullptr) {
            // Training: keep the normalised O_hat row in fp32 for bwd_prep.  D = rowsum(dO*O) is
            // compared against dP = dO.V_j^T of the (often near one-hot) attended keys, where
            // dP - D is a small difference: a bf16 O would put its 2^-9 rounding straight into dS.
            // Residue-major [B, L, H, dv_pad] (bwd_prep stages a residue's H rows with one copy),
            // written as 32-column x 128-row TMA tensor stores from four rotating 16 KB
            // 128-byte-swizzled shared-memory chunks (the feature-staging region, free until the
            // fused epilogue): coalesced full-line writes, rows past L clipped by the map.
            const int ob = bh / p.H, oh = bh - ob * p.H;
            const int nchunks = (p.dv_mma + 31) / 32;
            for (int ch = 0; ch < nchunks; ++ch) {
                uint8_t* cb = smem + (ch & 3) * (BM * 128);
                if (ch >= 4) {
                    if (warp == 2 && lane == 0) ptx::bulk_wait_group_read<3>();  // chunk ch-4's store has read cb
                    named_bar_sync(1, 256);
                }
                const int c0 = 32 * ch + 16 * half;
                uint32_t o[16];
                if (c0 < p.dv_mma) {  // warp-uniform
                    ptx::tmem_ld16(tl + c0, o);
                    ptx::tmem_wait_ld();
                } else {
#pragma unroll
                    for (int e = 0; e < 16; ++e) o[e] = 0u;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    *reinterpret_cast<float4*>(cb + row * 128 + (((4 * half + k) ^ (row & 7)) << 4)) =
                        make_float4(__uint_as_float(o[4 * k]) * inv_l, __uint_as_float(o[4 * k + 1]) * inv_l,
                                    __uint_as_float(o[4 * k + 2]) * inv_l, __uint_as_float(o[4 * k + 3]) * inv_l);
                ptx::fence_proxy_async_smem();
                named_bar_sync(1, 256);
                if (warp == 2 && lane == 0) {
                    ptx::tma_store_4d(&mapO, cb, 32 * ch, oh, q0, ob);
                    ptx::bulk_commit_group();
                }
            }
            if (warp == 2 && lane == 0) ptx::bulk_wait_group_read<0>();  // staging free for the epilogue
            named_bar_sync(1, 256);
            if (!z_early) issue_z1();
        }
        fused_epilogue(p, tl, inv_l, row, q0, bh, smem, half, p.z1_tma ? zs : nullptr, &bars->z_full, Rm, tv, &mapF, &mapFP);
        if (lane == 0) FIPA_TRACE(9, 1);
    }

    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 1) ptx::tmem_dealloc_2sm(tmem, 512);
    if (warp == 0 && lane == 0) span_mark(2);
}

}  // namespace

bool attn_fwd_2sm_supported(const LayerDims& d) {
    const int n1 = std::min(d.dv_mma, 256), n2 = d.dv_mma - n1;
    const int nb1 = (n1 / 2 + 63) / 64, nb2 = (n2 / 2 + 63) / 64;
    const int n_qkb = (d.dqk_mma + 63) / 64;
    const Layout lay = smem_layout(n_qkb, nb1, nb2);
    return d.dv_mma <= 448 && n1 % 16 == 0 && n2 % 16 == 0 && 3 * d.n_value + 6 <= 48 &&
           d.dqk_pad % 64 == 0 && d.dv_pad % 64 == 0 && n_qkb * 64 <= d.dqk_pad &&
           lay.total + 1024 <= 232448 && epilogue_smem(d.seg) <= lay.xch;
}

void launch_attn_fwd_2sm(const LayerDims& d, const AttnArgs& a, cudaStream_t stream) {
    if (!attn_fwd_2sm_supported(d))
        throw std::invalid_argument("tcgen05 attention: lifted widths unsupported (use precision='f32')");
    Attn2Params p{};
    p.L = a.L;
    p.H = d.heads;
    p.dqk_mma = d.dqk_mma;
    p.dv_mma = d.dv_mma;
    p.n_qkb = (d.dqk_mma + 63) / 64;
    p.n1 = std::min(d.dv_mma, 256);
    p.n2 = d.dv_mma - p.n1;
    p.nb1 = (p.n1 / 2 + 63) / 64;
    p.nb2 = (p.n2 / 2 + 63) / 64;
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
    p.o_save = a.o_save;
    p.dv_pad = d.dv_pad;
    p.h0 = a.hc > 0 ? a.h0 : 0;
    p.hc = a.hc > 0 ? a.hc : d.heads;
    if (p.h0 < 0 || p.h0 + p.hc > d.heads) throw std::invalid_argument("attention: head range out of bounds");
    const uint64_t BH = static_cast<uint64_t>(a.B) * d.heads;
    const CUtensorMap mapQ = make_map_blocks_bf16(a.qhat, a.L, BH, d.dqk_pad, BM, p.n_qkb);
    p.Lk = a.Lk > 0 ? a.Lk : a.L;
    p.kchunk = a.kchunk > 0 ? a.kchunk : p.Lk;
    const int G = (p.Lk + p.kchunk - 1) / p.kchunk;
    if (G * p.kchunk != p.Lk || (G > 1 && p.kchunk % BN != 0))
        throw std::invalid_argument("attention: key shards must be equal and a multiple of 64 rows");
    const CUtensorMap mapK = make_map_blocks_bf16_sharded(a.khat, p.kchunk, BH, G, d.dqk_pad, 32, p.n_qkb);
    const CUtensorMap mapV = make_map_4d_bf16_sharded(a.vhat, d.dv_pad, p.kchunk, BH, G, 64, kVKeys);
    const int rdz = d.rank * d.d_z;
    const Layout lay0 = smem_layout(p.n_qkb, p.nb1, p.nb2);
    p.z1_tma = (rdz % 32 == 0 && rdz / 32 <= 256 && (reinterpret_cast<uintptr_t>(a.z1) & 15) == 0 &&
                epilogue_smem(d.seg) + BM * rdz * 4 <= lay0.xch)
                   ? 1
                   : 0;
    const CUtensorMap mapZ = p.z1_tma ? make_map_blocks_f32(a.z1, static_cast<uint64_t>(a.B) * a.L, rdz, BM, rdz / 32)
                                      : mapV;
    const Layout lay = smem_layout(p.n_qkb, p.nb1, p.nb2);
    const int smem = lay.total + 1024;
    if (a.o_save != nullptr && d.dv_pad % 32 != 0)
        throw std::invalid_argument("attention: O_hat rows must be a multiple of 32 floats");
    // O_hat rows keep the dv_pad stride; the map stops at dv_used, so the padding columns of the
    // last 32-column chunk are not written (prep keeps them out of D)
    CUtensorMap mapO = mapV;
    if (a.o_save != nullptr) {
        const uint64_t od[4] = {uint64_t(d.dv_used), uint64_t(d.heads), uint64_t(a.L), uint64_t(a.B)};
        const uint64_t os[3] = {uint64_t(d.dv_pad) * 4, uint64_t(d.dv_pad) * d.heads * 4,
                                uint64_t(d.dv_pad) * d.heads * a.L * 4};
        const uint32_t ob[4] = {32, 1, BM, 1};
        mapO = make_map_4d_f32_strided(a.o_save, od, os, ob);
    }
    cudaFuncSetAttribute(attn_fwd_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int qtiles = (a.L + BM - 1) / BM;
    dim3 grid(static_cast<unsigned>((qtiles + 1) / 2 * 2), static_cast<unsigned>(a.B * p.hc));
    // fast epilogue with per-warp TMA feature stores: c = d_z = 128, rank 1-2, z1 staged,
    // even n_value (points block a whole number of 16-byte chunks), 16-byte aligned rows
    p.feat_tma = (d.c == 128 && d.d_z == 128 && (d.rank == 1 || d.rank == 2) && p.z1_tma && d.n_value % 2 == 0 &&
                  d.n_value <= kMaxPoints && d.seg == 256 + 4 * d.n_value && (d.feat_ld * 2) % 16 == 0 &&
                  (reinterpret_cast<uintptr_t>(a.feat) & 15) == 0)
                     ? 1
                     : 0;
    const CUtensorMap mapF = p.feat_tma ? make_map_3d_bf16(a.feat, d.feat, a.L, a.B, d.feat_ld, 64, 32) : mapV;
    const CUtensorMap mapFP =
        p.feat_tma ? make_map_3d_bf16(a.feat, d.feat, a.L, a.B, d.feat_ld, 4 * d.n_value, 32) : mapV;
    launch_pdl(attn_fwd_2sm_kernel, grid, dim3(kThreads), size_t(smem), stream, mapQ, mapK, mapV, mapZ, mapO, mapF,
               mapFP, p);
}

}  // namespace fipa_b200
