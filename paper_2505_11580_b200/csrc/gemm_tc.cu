// Generic bf16 GEMM on 5th-gen tensor cores (tcgen05.mma kind::f16, fp32 accumulators in
// TMEM), TMA-fed through a STAGES-deep mbarrier ring, warp-specialised:
//   warp 0      : TMA producer (one elected lane)
//   warp 1      : TMEM allocator + MMA issuer (one elected lane)
//   warps 2..5  : epilogue, TMEM -> registers -> global (warp w owns TMEM lanes 32*(w%4)..)
// One 128 x BN output tile per CTA.  TF32 = true: fp32 operands, tcgen05.mma kind::tf32 (the
// fp32 path; 3xTF32 accuracy comes from K-concatenated hi/lo operands, see launch_gemm_tf32x3).  Serves the projection GEMM (reference
// project_inputs, proj/src/ipa.cpp:201-217 -> linear, proj/src/tensor.cpp:292-317), the
// output projection (proj/src/flash_ipa.cpp:212) and the backward GEMMs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

#include "kernels.hpp"
#include "ptx.cuh"
#include "tma_host.hpp"

namespace fipa_b200 {

namespace {

constexpr int BM = 128;
constexpr int kThreads = 192;

template <int BN, bool TF32 = false>
struct GemmCfg {
    static constexpr int BK = TF32 ? 32 : 64;  // K elements per stage: one 128-byte swizzle row
    // Output staging buffers per epilogue warp: 2 keep up once the epilogue math is branch-free
    // (tools/gemm_bench.cu: 4 buffers at the cost of ring stages measured no faster on the
    // short-K shapes and 13% slower on a square 8192^3 product).
    static constexpr int kStages = BN > 128 ? 4 : 6;
    static constexpr int kCBuf = 2;
    static constexpr int kABytes = BM * 128;
    // B rows of whole 64-element (128-byte) blocks: BN = 224 stages four blocks, the MMA reads 3.5
    static constexpr int kBBlocks = (BN + 63) / 64;
    static constexpr int kBBytes = kBBlocks * 64 * 128;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStageC = 4 * kCBuf * 32 * 128;  // fp32 output staging: 4 warps x kCBuf x (32 rows x 128 B)
    static constexpr int kSmem = kStages * kStageBytes + kStageC + 1024 /*align*/ + 256 /*barriers*/;
    static_assert(2 * BN <= 512, "double-buffered accumulator must fit TMEM");
};

// CTA-pair tiles: each CTA stages 128 A rows and BN / 2 B rows per stage.
template <int BN>
struct GemmCfg2 {
    static constexpr int BK = 64;
    static constexpr int kStages = 6;
    static constexpr int kCBuf = 2;
    static constexpr int kABytes = BM * 128;
    static constexpr int kBBytes = (BN / 2) * 128;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStageC = 4 * kCBuf * 32 * 128;
    static constexpr int kSmem = kStages * kStageBytes + kStageC + 1024 + 256;
    static_assert(BN % 128 == 0 && 2 * BN <= 512, "pair tile: BN / 2 whole 64-column blocks, 2 x BN TMEM columns");
};

struct EpiParams {
    void* C;
    int64_t ldc;
    int M, N, K;
    bool out_bf16, accumulate;
    bool tma_c;  // plain fp32 C: 32x32 chunks staged in shared memory and written by TMA stores
    int split_k;
    float alpha;
    const float* bias;
    const uint8_t* row_mask;
    int batch, batch_h;  // batched products (see GemmArgs)
    int a_blk, b_blk;    // MN-major operand loaded as ONE 4-D box of 64-column blocks (ld % 64 == 0)
    bool tma_c16 = false;  // plain bf16 C: two 32-column chunks per 32 x 64 box, TMA stores
    bool c16_split = false;      // batched fp32 C with a bf16 copy (GemmArgs::C16)
    uint32_t c16_f32_chunks = 0;  // chunks also written in fp32
};

#ifdef FIPA_GEMM_TRACE
__device__ long long g_gemm_trace[2][8][24];  // [epilogue warp 2 | MMA warp][unit][event], CTA 0
#define GTRACE(w, u, ev)                                                              \
    do {                                                                              \
        if (blockIdx.x == 0 && (u) < 8 && (ev) < 24) g_gemm_trace[w][u][ev] = clock64(); \
    } while (0)
#else
#define GTRACE(w, u, ev) \
    do {                 \
    } while (0)
#endif

// Persistent: each CTA walks work units u = blockIdx.x, += gridDim.x over (split, m-tile, n-tile).
// The smem ring runs continuously across units; the accumulator is double-buffered in TMEM
// (2 x BN columns) so the epilogue warps drain unit u while the tensor pipe computes unit u+1.
template <int BN, bool A_MN, bool B_MN, bool TF32 = false>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapB,
                     const __grid_constant__ CUtensorMap mapC,
                     const __grid_constant__ CUtensorMap mapC16, EpiParams p) {
    using Cfg = GemmCfg<BN, TF32>;
    constexpr int BK = Cfg::BK;
    static_assert(!TF32 || (!A_MN && !B_MN), "tf32 GEMM: K-major operands only");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint8_t* tiles = smem;
    uint8_t* stage_c = smem + Cfg::kStages * Cfg::kStageBytes;  // [4 warps][2][32 rows][128 B]
    uint64_t* full = reinterpret_cast<uint64_t*>(stage_c + Cfg::kStageC);
    uint64_t* empty = full + Cfg::kStages;
    uint64_t* acc_full = empty + Cfg::kStages;   // [2]
    uint64_t* acc_empty = acc_full + 2;          // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int warp = ptx::warp_id();
    const int lane = ptx::lane_id();
    const int n_tiles_n = (p.N + BN - 1) / BN;
    const int n_tiles_m = (p.M + BM - 1) / BM;
    const int per_batch = n_tiles_n * n_tiles_m * p.split_k;
    const int units = per_batch * p.batch;
    const int nk_all = (p.K + BK - 1) / BK;
    auto unit_coords = [&](int u, int& m0, int& n0, int& kb0, int& nk) {
        u -= (u / per_batch) * per_batch;
        const int z = u / (n_tiles_n * n_tiles_m);
        const int r = u - z * (n_tiles_n * n_tiles_m);
        m0 = (r / n_tiles_n) * BM;
        n0 = (r % n_tiles_n) * BN;
        kb0 = static_cast<int>((int64_t(nk_all) * z) / p.split_k);
        nk = static_cast<int>((int64_t(nk_all) * (z + 1)) / p.split_k) - kb0;
    };
    // power-of-two allocation covering the double-buffered accumulator (2 x 224 -> 512)
    constexpr uint32_t kTmemCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&mapA);
        ptx::tma_prefetch(&mapB);
        for (int s = 0; s < Cfg::kStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&acc_full[b], 1);
            ptx::mbar_init(&acc_empty[b], 4);  // one arrive per epilogue warp
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(tmem_slot, kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    ptx::pdl_wait();  // operands (and split-K's zeroed C) of the preceding kernels
    ptx::pdl_trigger();

    if (warp == 0) {
        if (lane == 0) {
            int it = 0;  // global k-block counter (ring position)
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                int m0, n0, kb0, nk;
                unit_coords(u, m0, n0, kb0, nk);
                const int zb = u / per_batch;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % Cfg::kStages;
                    if (it >= Cfg::kStages) ptx::mbar_wait(&empty[s], ((it / Cfg::kStages) - 1) & 1);
                    uint8_t* sa = tiles + s * Cfg::kStageBytes;
                    uint8_t* sb = sa + Cfg::kABytes;
                    ptx::mbar_expect_tx(&full[s], Cfg::kStageBytes);
                    const int kc = (kb0 + kb) * BK;
                    // (the TMA engine costs ~100 cycles per box: one box per operand and stage)
                    if (A_MN && p.a_blk) {
                        ptx::tma_load_4d(sa, &mapA, &full[s], 0, kc, m0 / 64, zb);
                    } else if (A_MN) {
                        for (int mb = 0; mb < BM / 64; ++mb)
                            ptx::tma_load_3d(sa + mb * 64 * 128, &mapA, &full[s], m0 + mb * 64, kc, zb);
                    } else {
                        ptx::tma_load_3d(sa, &mapA, &full[s], kc, m0, zb);
                    }
                    if (B_MN && p.b_blk) {
                        ptx::tma_load_4d(sb, &mapB, &full[s], 0, kc, n0 / 64, zb);
                    } else if (B_MN) {
                        for (int nb = 0; nb < Cfg::kBBlocks; ++nb)
                            ptx::tma_load_3d(sb + nb * 64 * 128, &mapB, &full[s], n0 + nb * 64, kc, zb);
                    } else {
                        ptx::tma_load_3d(sb, &mapB, &full[s], kc, n0, zb);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // The whole warp runs the loop and one elected lane issues (warp-uniform descriptors in
        // uniform registers; a lane-0-only loop paid ~45 cycles of R2UR per MMA, which left the
        // N=128 MMAs issue-bound); descriptors advance by 64-bit adds of (byte offset >> 4).
        constexpr uint32_t idesc = TF32 ? ptx::idesc_tf32(BM, BN, A_MN, B_MN) : ptx::idesc_bf16(BM, BN, A_MN, B_MN);
        const uint32_t tiles_u32 = ptx::smem_u32(tiles);
        const uint64_t da0 = A_MN ? ptx::sw128_desc(tiles_u32, 64 * 128, 1024) : ptx::sw128_desc(tiles_u32, 16, 1024);
        const uint64_t db0 = B_MN ? ptx::sw128_desc(tiles_u32 + Cfg::kABytes, 64 * 128, 1024)
                                  : ptx::sw128_desc(tiles_u32 + Cfg::kABytes, 16, 1024);
        constexpr uint64_t kStepA = A_MN ? (2048 >> 4) : (32 >> 4);  // one MMA K step (16 bf16 / 8 tf32 = 32 B)
        constexpr uint64_t kStepB = B_MN ? (2048 >> 4) : (32 >> 4);
        int it = 0, lu = 0;  // k-block counter, local unit counter
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++lu) {
            int m0, n0, kb0, nk;
            unit_coords(u, m0, n0, kb0, nk);
            const int buf = lu & 1;
            if (lane == 0) GTRACE(1, lu, 0);
            if (lu >= 2) ptx::mbar_wait(&acc_empty[buf], ((lu >> 1) - 1) & 1);
            if (lane == 0) GTRACE(1, lu, 1);
            ptx::tc_fence_after();
            const uint32_t acc = tmem + buf * BN;
            for (int kb = 0; kb < nk; ++kb, ++it) {
                const int s = it % Cfg::kStages;
                ptx::mbar_wait(&full[s], (it / Cfg::kStages) & 1);
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    const uint64_t so = static_cast<uint64_t>((s * Cfg::kStageBytes) >> 4);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        if constexpr (TF32)
                            ptx::mma_ss_tf32(acc, da0 + so + kk * kStepA, db0 + so + kk * kStepB, idesc, (kb | kk) != 0);
                        else
                            ptx::mma_ss(acc, da0 + so + kk * kStepA, db0 + so + kk * kStepB, idesc, (kb | kk) != 0);
                    }
                    ptx::mma_commit(&empty[s]);
                }
                __syncwarp();
            }
            if (ptx::elect_one()) ptx::mma_commit(&acc_full[buf]);
            __syncwarp();
            if (lane == 0) GTRACE(1, lu, 2);
        }
    } else {
        // Epilogue: warp w reads TMEM lanes [32*(w%4), +32); thread = one output row.
        const int quad = warp & 3;
        uint8_t* my_stage = stage_c + quad * (Cfg::kCBuf * 32 * 128);
        int nstore = 0;  // TMA stores issued by this warp (staging buffer = nstore % kCBuf)
        int lu = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++lu) {
            int m0, n0, kb0, nk;
            unit_coords(u, m0, n0, kb0, nk);
            const int buf = lu & 1;
            const int zb = u / per_batch, zh = zb % p.batch_h, zo = zb / p.batch_h;
            if (warp == 2 && lane == 0) GTRACE(0, lu, 0);
            ptx::mbar_wait(&acc_full[buf], (lu >> 1) & 1);
            if (warp == 2 && lane == 0) GTRACE(0, lu, 1);
            ptx::tc_fence_after();
            const int row = m0 + quad * 32 + lane;
            const bool row_ok = row < p.M;
            const bool zero_row = row_ok && p.row_mask != nullptr && p.row_mask[row] == 0;
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t r[32];
                ptx::tmem_ld32(tmem + buf * BN + (uint32_t(quad * 32) << 16) + c0, r);
                ptx::tmem_wait_ld();
                if (warp == 2 && lane == 0) GTRACE(0, lu, 2 + 2 * (c0 / 32));
                const int col0 = n0 + c0;
                if (p.tma_c || p.tma_c16) {
                    // warp-collective path: rows past M are clipped by the TMA store; nk == 0 (an
                    // empty split) cannot occur without split-K
                    if (col0 >= p.N || m0 + quad * 32 >= p.M) continue;
                } else {
                    if (!row_ok || nk <= 0) continue;
                    if (col0 >= p.N) continue;
                }
                if (p.split_k > 1) {
                    float* out = reinterpret_cast<float*>(p.C) + int64_t(row) * p.ldc + col0;
                    if (col0 + 32 <= p.N && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            atomicAdd(reinterpret_cast<float4*>(out) + q,
                                      make_float4(__uint_as_float(r[4 * q]) * p.alpha, __uint_as_float(r[4 * q + 1]) * p.alpha,
                                                  __uint_as_float(r[4 * q + 2]) * p.alpha, __uint_as_float(r[4 * q + 3]) * p.alpha));
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i)  // compile-time indices keep r[] in registers
                            if (col0 + i < p.N) atomicAdd(out + i, __uint_as_float(r[i]) * p.alpha);
                    }
                    continue;
                }
                // (a per-element `bias != null && col < N` test compiled to 32 dependent branches,
                // ~2k cycles per chunk: tools/gemm_trace.cu; the bias test is uniform, hoist it)
                float v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * p.alpha;
                if (p.bias != nullptr) {
                    if (col0 + 32 <= p.N && (reinterpret_cast<uintptr_t>(p.bias + col0) & 15) == 0) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const float4 bq = __ldg(reinterpret_cast<const float4*>(p.bias + col0) + q);
                            v[4 * q] += bq.x;
                            v[4 * q + 1] += bq.y;
                            v[4 * q + 2] += bq.z;
                            v[4 * q + 3] += bq.w;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (col0 + i < p.N) v[i] += __ldg(p.bias + col0 + i);
                    }
                }
                if (zero_row) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = 0.0f;
                }
                if (p.tma_c16) {
                    // bf16 C: chunk pairs fill one 128-byte line per row of a 32 x 64 box (stores
                    // from registers wrote each 32-byte sector in two 16-byte halves from two
                    // instructions: partial-sector writes)
                    const int hsel = (c0 >> 5) & 1;
                    uint8_t* sb = my_stage + (nstore % Cfg::kCBuf) * (32 * 128);
                    if (hsel == 0) {
                        if (nstore >= Cfg::kCBuf && lane == 0) ptx::bulk_wait_group_read<Cfg::kCBuf - 1>();
                        __syncwarp();
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint4 w;
                        w.x = ptx::pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
                        w.y = ptx::pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
                        w.z = ptx::pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
                        w.w = ptx::pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
                        *reinterpret_cast<uint4*>(sb + lane * 128 + (((4 * hsel + q) ^ (lane & 7)) << 4)) = w;
                    }
                    if (hsel == 1 || col0 + 32 >= p.N) {
                        ptx::fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            ptx::tma_store_4d(&mapC, sb, col0 - 32 * hsel, zh, m0 + quad * 32, zo);
                            ptx::bulk_commit_group();
                        }
                        ++nstore;
                    }
                    continue;
                }
                if (p.c16_split) {
                    // bf16 copy of every chunk pair (buffer 0, stored after the odd chunk) and fp32
                    // boxes of the flagged chunks (buffer 1); explicit waits order the two buffers
                    const int hsel = (c0 >> 5) & 1;
                    uint8_t* b16 = my_stage;
                    uint8_t* b32 = my_stage + 32 * 128;
                    if (hsel == 0) {
                        if (lane == 0) ptx::bulk_wait_group_read<0>();
                        __syncwarp();
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint4 w;
                        w.x = ptx::pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
                        w.y = ptx::pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
                        w.z = ptx::pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
                        w.w = ptx::pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
                        *reinterpret_cast<uint4*>(b16 + lane * 128 + (((4 * hsel + q) ^ (lane & 7)) << 4)) = w;
                    }
                    if (hsel == 1 || col0 + 32 >= p.N) {
                        ptx::fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            ptx::tma_store_4d(&mapC16, b16, col0 - 32 * hsel, zh, m0 + quad * 32, zo);
                            ptx::bulk_commit_group();
                        }
                    }
                    if ((col0 >> 5) < 32 && ((p.c16_f32_chunks >> (col0 >> 5)) & 1u)) {
                        if (hsel == 1) {  // buffer 1's previous fp32 box (chunk c0 - 32) has been read
                            if (lane == 0) ptx::bulk_wait_group_read<1>();
                            __syncwarp();
                        }
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            *reinterpret_cast<float4*>(b32 + lane * 128 + ((q ^ (lane & 7)) << 4)) =
                                make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                        ptx::fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            ptx::tma_store_4d(&mapC, b32, col0, zh, m0 + quad * 32, zo);
                            ptx::bulk_commit_group();
                        }
                    }
                    continue;
                }
                if (p.tma_c) {
                    // this warp's 32 rows x 32 columns -> swizzled staging -> one TMA store
                    uint8_t* sb = my_stage + (nstore % Cfg::kCBuf) * (32 * 128);
                    if (nstore >= Cfg::kCBuf && lane == 0)
                        ptx::bulk_wait_group_read<Cfg::kCBuf - 1>();  // buffer's last store has read it
                    __syncwarp();
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        *reinterpret_cast<float4*>(sb + lane * 128 + ((q ^ (lane & 7)) << 4)) =
                            make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        ptx::tma_store_4d(&mapC, sb, col0, zh, m0 + quad * 32, zo);
                        ptx::bulk_commit_group();
                        if (warp == 2) GTRACE(0, lu, 3 + 2 * (c0 / 32));
                    }
                    ++nstore;
                    continue;
                }
                const size_t esz = p.out_bf16 ? 2 : 4;
                const bool full_chunk = col0 + 32 <= p.N &&
                                        ((reinterpret_cast<uintptr_t>(p.C) + (size_t(row) * p.ldc + col0) * esz) & 15) == 0;
                if (p.out_bf16) {
                    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.C) + int64_t(row) * p.ldc + col0;
                    if (full_chunk) {
                        uint4* o4 = reinterpret_cast<uint4*>(out);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            uint4 w;
                            w.x = ptx::pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
                            w.y = ptx::pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
                            w.z = ptx::pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
                            w.w = ptx::pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
                            o4[q] = w;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (col0 + i < p.N) out[i] = __float2bfloat16_rn(v[i]);
                    }
                } else {
                    float* out = reinterpret_cast<float*>(p.C) + int64_t(row) * p.ldc + col0;
                    if (full_chunk) {
                        float4* o4 = reinterpret_cast<float4*>(out);
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            float4 w = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                            if (p.accumulate) {
                                const float4 o = o4[q];
                                w.x += o.x; w.y += o.y; w.z += o.z; w.w += o.w;
                            }
                            o4[q] = w;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (col0 + i < p.N) out[i] = p.accumulate ? out[i] + v[i] : v[i];
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&acc_empty[buf]);
        }
        if (p.tma_c && lane == 0) ptx::bulk_wait_group_read<0>();
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc(tmem, kTmemCols);
}

// CTA-pair version (tcgen05 cta_group::2): a cluster of two CTAs computes a 256 x BN tile -- each
// CTA stages its own 128 A rows and HALF of the tile's B rows / columns, so every SM reads half the
// B bytes per MMA of the single-CTA kernel (the batched dQ product: 96 -> 64 B/clk of operand
// traffic at the MMA rate).  The pair leader issues the MMAs; ring, accumulator and epilogue
// barriers as in gemm_bf16_kernel, with the full barriers and acc_empty counted at the leader.
template <int BN, bool A_MN, bool B_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm2_bf16_kernel(const __grid_constant__ CUtensorMap mapA,
                      const __grid_constant__ CUtensorMap mapB,
                      const __grid_constant__ CUtensorMap mapC,
                     const __grid_constant__ CUtensorMap mapC16, EpiParams p) {
    using Cfg = GemmCfg2<BN>;
    constexpr int BK = Cfg::BK;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint8_t* tiles = smem;
    uint8_t* stage_c = smem + Cfg::kStages * Cfg::kStageBytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(stage_c + Cfg::kStageC);
    uint64_t* empty = full + Cfg::kStages;
    uint64_t* acc_full = empty + Cfg::kStages;   // [2]
    uint64_t* acc_empty = acc_full + 2;          // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int warp = ptx::warp_id();
    const int lane = ptx::lane_id();
    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    const int cluster = static_cast<int>(blockIdx.x >> 1), nclusters = static_cast<int>(gridDim.x >> 1);
    const int n_tiles_n = (p.N + BN - 1) / BN;
    const int n_tiles_m = (p.M + 2 * BM - 1) / (2 * BM);
    const int per_batch = n_tiles_n * n_tiles_m * p.split_k;
    const int units = per_batch * p.batch;
    const int nk_all = (p.K + BK - 1) / BK;
    // m0: this CTA's first row (pair tile rows + 128 * rank); n0: the tile's first column
    auto unit_coords = [&](int u, int& m0, int& n0, int& kb0, int& nk) {
        u -= (u / per_batch) * per_batch;
        const int z = u / (n_tiles_n * n_tiles_m);
        const int r = u - z * (n_tiles_n * n_tiles_m);
        m0 = (r / n_tiles_n) * 2 * BM + static_cast<int>(rank) * BM;
        n0 = (r % n_tiles_n) * BN;
        kb0 = static_cast<int>((int64_t(nk_all) * z) / p.split_k);
        nk = static_cast<int>((int64_t(nk_all) * (z + 1)) / p.split_k) - kb0;
    };
    constexpr uint32_t kTmemCols = 2 * BN <= 256 ? 256 : 512;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&mapA);
        ptx::tma_prefetch(&mapB);
        for (int s = 0; s < Cfg::kStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&acc_full[b], 1);
            ptx::mbar_init(&acc_empty[b], 8);  // 4 epilogue warps x 2 CTAs (the leader's counts)
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc_2sm(tmem_slot, kTmemCols);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const uint32_t acc_empty_leader = ptx::mapa(acc_empty, 0);

    if (warp == 0) {
        if (lane == 0) {
            int it = 0;
            for (int u = cluster; u < units; u += nclusters) {
                int m0, n0, kb0, nk;
                unit_coords(u, m0, n0, kb0, nk);
                const int zb = u / per_batch;
                const int nh = n0 + static_cast<int>(rank) * (BN / 2);  // this CTA's half of the B columns
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % Cfg::kStages;
                    if (it >= Cfg::kStages) ptx::mbar_wait(&empty[s], ((it / Cfg::kStages) - 1) & 1);
                    uint8_t* sa = tiles + s * Cfg::kStageBytes;
                    uint8_t* sb = sa + Cfg::kABytes;
                    if (leader) ptx::mbar_expect_tx(&full[s], 2 * Cfg::kStageBytes);
                    const int kc = (kb0 + kb) * BK;
                    if (A_MN && p.a_blk) {
                        ptx::tma_load_4d_2sm(sa, &mapA, &full[s], 0, kc, m0 / 64, zb);
                    } else if (A_MN) {
                        for (int mb = 0; mb < BM / 64; ++mb)
                            ptx::tma_load_3d_2sm(sa + mb * 64 * 128, &mapA, &full[s], m0 + mb * 64, kc, zb);
                    } else {
                        ptx::tma_load_3d_2sm(sa, &mapA, &full[s], kc, m0, zb);
                    }
                    if (B_MN && p.b_blk) {
                        ptx::tma_load_4d_2sm(sb, &mapB, &full[s], 0, kc, nh / 64, zb);
                    } else if (B_MN) {
                        for (int nb = 0; nb < BN / 128; ++nb)
                            ptx::tma_load_3d_2sm(sb + nb * 64 * 128, &mapB, &full[s], nh + nb * 64, kc, zb);
                    } else {
                        ptx::tma_load_3d_2sm(sb, &mapB, &full[s], kc, nh, zb);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {
            constexpr uint32_t idesc = ptx::idesc_bf16(2 * BM, BN, A_MN, B_MN);
            const uint32_t tiles_u32 = ptx::smem_u32(tiles);
            const uint64_t da0 = A_MN ? ptx::sw128_desc(tiles_u32, 64 * 128, 1024) : ptx::sw128_desc(tiles_u32, 16, 1024);
            const uint64_t db0 = B_MN ? ptx::sw128_desc(tiles_u32 + Cfg::kABytes, 64 * 128, 1024)
                                      : ptx::sw128_desc(tiles_u32 + Cfg::kABytes, 16, 1024);
            constexpr uint64_t kStepA = A_MN ? (2048 >> 4) : (32 >> 4);
            constexpr uint64_t kStepB = B_MN ? (2048 >> 4) : (32 >> 4);
            int it = 0, lu = 0;
            for (int u = cluster; u < units; u += nclusters, ++lu) {
                int m0, n0, kb0, nk;
                unit_coords(u, m0, n0, kb0, nk);
                const int buf = lu & 1;
                if (lu >= 2) ptx::mbar_wait_cluster(&acc_empty[buf], ((lu >> 1) - 1) & 1);
                ptx::tc_fence_after();
                const uint32_t acc = tmem + buf * BN;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % Cfg::kStages;
                    ptx::mbar_wait(&full[s], (it / Cfg::kStages) & 1);
                    ptx::tc_fence_after();
                    if (ptx::elect_one()) {
                        const uint64_t so = static_cast<uint64_t>((s * Cfg::kStageBytes) >> 4);
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            ptx::mma2_ss(acc, da0 + so + kk * kStepA, db0 + so + kk * kStepB, idesc, (kb | kk) != 0);
                        ptx::mma_commit_2sm(&empty[s], 0x3);
                    }
                    __syncwarp();
                }
                if (ptx::elect_one()) ptx::mma_commit_2sm(&acc_full[buf], 0x3);
                __syncwarp();
            }
        }
    } else {
        // Epilogue: warp w reads TMEM lanes [32*(w%4), +32); thread = one output row.
        const int quad = warp & 3;
        uint8_t* my_stage = stage_c + quad * (Cfg::kCBuf * 32 * 128);
        int nstore = 0;  // TMA stores issued by this warp (staging buffer = nstore % kCBuf)
        int lu = 0;
        for (int u = cluster; u < units; u += nclusters, ++lu) {
            int m0, n0, kb0, nk;
            unit_coords(u, m0, n0, kb0, nk);
            const int buf = lu & 1;
            const int zb = u / per_batch, zh = zb % p.batch_h, zo = zb / p.batch_h;
            if (warp == 2 && lane == 0) GTRACE(0, lu, 0);
            ptx::mbar_wait(&acc_full[buf], (lu >> 1) & 1);
            if (warp == 2 && lane == 0) GTRACE(0, lu, 1);
            ptx::tc_fence_after();
            const int row = m0 + quad * 32 + lane;
            const bool row_ok = row < p.M;
            const bool zero_row = row_ok && p.row_mask != nullptr && p.row_mask[row] == 0;
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t r[32];
                ptx::tmem_ld32(tmem + buf * BN + (uint32_t(quad * 32) << 16) + c0, r);
                ptx::tmem_wait_ld();
                if (warp == 2 && lane == 0) GTRACE(0, lu, 2 + 2 * (c0 / 32));
                const int col0 = n0 + c0;
                if (p.tma_c || p.tma_c16) {
                    // warp-collective path: rows past M are clipped by the TMA store; nk == 0 (an
                    // empty split) cannot occur without split-K
                    if (col0 >= p.N || m0 + quad * 32 >= p.M) continue;
                } else {
                    if (!row_ok || nk <= 0) continue;
                    if (col0 >= p.N) continue;
                }
                if (p.split_k > 1) {
                    float* out = reinterpret_cast<float*>(p.C) + int64_t(row) * p.ldc + col0;
                    if (col0 + 32 <= p.N && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            atomicAdd(reinterpret_cast<float4*>(out) + q,
                                      make_float4(__uint_as_float(r[4 * q]) * p.alpha, __uint_as_float(r[4 * q + 1]) * p.alpha,
                                                  __uint_as_float(r[4 * q + 2]) * p.alpha, __uint_as_float(r[4 * q + 3]) * p.alpha));
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i)  // compile-time indices keep r[] in registers
                            if (col0 + i < p.N) atomicAdd(out + i, __uint_as_float(r[i]) * p.alpha);
                    }
                    continue;
                }
                // (a per-element `bias != null && col < N` test compiled to 32 dependent branches,
                // ~2k cycles per chunk: tools/gemm_trace.cu; the bias test is uniform, hoist it)
                float v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * p.alpha;
                if (p.bias != nullptr) {
                    if (col0 + 32 <= p.N && (reinterpret_cast<uintptr_t>(p.bias + col0) & 15) == 0) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const float4 bq = __ldg(reinterpret_cast<const float4*>(p.bias + col0) + q);
                            v[4 * q] += bq.x;
                            v[4 * q + 1] += bq.y;
                            v[4 * q + 2] += bq.z;
                            v[4 * q + 3] += bq.w;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (col0 + i < p.N) v[i] += __ldg(p.bias + col0 + i);
                    }
                }
                if (zero_row) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = 0.0f;
                }
                if (p.tma_c16) {
                    // bf16 C: chunk pairs fill one 128-byte line per row of a 32 x 64 box (stores
                    // from registers wrote each 32-byte sector in two 16-byte halves from two
                    // instructions: partial-sector writes)
                    const int hsel = (c0 >> 5) & 1;
                    uint8_t* sb = my_stage + (nstore % Cfg::kCBuf) * (32 * 128);
                    if (hsel == 0) {
                        if (nstore >= Cfg::kCBuf && lane == 0) ptx::bulk_wait_group_read<Cfg::kCBuf - 1>();
                        __syncwarp();
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint4 w;
                        w.x = ptx::pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
                        w.y = ptx::pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
                        w.z = ptx::pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
                        w.w = ptx::pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
                        *reinterpret_cast<uint4*>(sb + lane * 128 + (((4 * hsel + q) ^ (lane & 7)) << 4)) = w;
                    }
                    if (hsel == 1 || col0 + 32 >= p.N) {
                        ptx::fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            ptx::tma_store_4d(&mapC, sb, col0 - 32 * hsel, zh, m0 + quad * 32, zo);
                            ptx::bulk_commit_group();
                        }
                        ++nstore;
                    }
                    continue;
                }
                if (p.c16_split) {
                    // bf16 copy of every chunk pair (buffer 0, stored after the odd chunk) and fp32
                    // boxes of the flagged chunks (buffer 1); explicit waits order the two buffers
                    const int hsel = (c0 >> 5) & 1;
                    uint8_t* b16 = my_stage;
                    uint8_t* b32 = my_stage + 32 * 128;
                    if (hsel == 0) {
                        if (lane == 0) ptx::bulk_wait_group_read<0>();
                        __syncwarp();
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint4 w;
                        w.x = ptx::pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
                        w.y = ptx::pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
                        w.z = ptx::pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
                        w.w = ptx::pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
                        *reinterpret_cast<uint4*>(b16 + lane * 128 + (((4 * hsel + q) ^ (lane & 7)) << 4)) = w;
                    }
                    if (hsel == 1 || col0 + 32 >= p.N) {
                        ptx::fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            ptx::tma_store_4d(&mapC16, b16, col0 - 32 * hsel, zh, m0 + quad * 32, zo);
                            ptx::bulk_commit_group();
                        }
                    }
                    if ((col0 >> 5) < 32 && ((p.c16_f32_chunks >> (col0 >> 5)) & 1u)) {
                        if (hsel == 1) {  // buffer 1's previous fp32 box (chunk c0 - 32) has been read
                            if (lane == 0) ptx::bulk_wait_group_read<1>();
                            __syncwarp();
                        }
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            *reinterpret_cast<float4*>(b32 + lane * 128 + ((q ^ (lane & 7)) << 4)) =
                                make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                        ptx::fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            ptx::tma_store_4d(&mapC, b32, col0, zh, m0 + quad * 32, zo);
                            ptx::bulk_commit_group();
                        }
                    }
                    continue;
                }
                if (p.tma_c) {
                    // this warp's 32 rows x 32 columns -> swizzled staging -> one TMA store
                    uint8_t* sb = my_stage + (nstore % Cfg::kCBuf) * (32 * 128);
                    if (nstore >= Cfg::kCBuf && lane == 0)
                        ptx::bulk_wait_group_read<Cfg::kCBuf - 1>();  // buffer's last store has read it
                    __syncwarp();
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        *reinterpret_cast<float4*>(sb + lane * 128 + ((q ^ (lane & 7)) << 4)) =
                            make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        ptx::tma_store_4d(&mapC, sb, col0, zh, m0 + quad * 32, zo);
                        ptx::bulk_commit_group();
                        if (warp == 2) GTRACE(0, lu, 3 + 2 * (c0 / 32));
                    }
                    ++nstore;
                    continue;
                }
                const size_t esz = p.out_bf16 ? 2 : 4;
                const bool full_chunk = col0 + 32 <= p.N &&
                                        ((reinterpret_cast<uintptr_t>(p.C) + (size_t(row) * p.ldc + col0) * esz) & 15) == 0;
                if (p.out_bf16) {
                    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.C) + int64_t(row) * p.ldc + col0;
                    if (full_chunk) {
                        uint4* o4 = reinterpret_cast<uint4*>(out);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            uint4 w;
                            w.x = ptx::pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
                            w.y = ptx::pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
                            w.z = ptx::pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
                            w.w = ptx::pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
                            o4[q] = w;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (col0 + i < p.N) out[i] = __float2bfloat16_rn(v[i]);
                    }
                } else {
                    float* out = reinterpret_cast<float*>(p.C) + int64_t(row) * p.ldc + col0;
                    if (full_chunk) {
                        float4* o4 = reinterpret_cast<float4*>(out);
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            float4 w = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                            if (p.accumulate) {
                                const float4 o = o4[q];
                                w.x += o.x; w.y += o.y; w.z += o.z; w.w += o.w;
                            }
                            o4[q] = w;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (col0 + i < p.N) out[i] = p.accumulate ? out[i] + v[i] : v[i];
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster_relaxed(acc_empty_leader + buf * 8);  // the leader's barrier
        }
        if (p.tma_c && lane == 0) ptx::bulk_wait_group_read<0>();
    }

    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 1) ptx::tmem_dealloc_2sm(tmem, kTmemCols);
}

template <int BN, bool A_MN, bool B_MN, bool TF32 = false>
void launch_impl(const GemmArgs& a, cudaStream_t stream) {
    using Cfg = GemmCfg<BN, TF32>;
    constexpr int BK = Cfg::BK;
    // TMA maps: K-major operands are [rows=M|N, cols=K] with box {64, rows-per-tile};
    // MN-major operands are [rows=K, cols=M|N] with box {64, BK}.
    // TMA maps (dim 2 = batch, dense stacks): K-major operands are [rows=M|N, cols=K] with box
    // {64, rows-per-tile}; MN-major operands are [rows=K, cols=M|N] with box {64, BK}.
    const uint64_t nb = static_cast<uint64_t>(std::max(1, a.batch));
    // MN-major operands whose row stride is a whole number of 64-column blocks (and covers the
    // tile's columns) come in as ONE 4-D box {64, BK, tile/64 blocks} per stage
    const bool a_blk = A_MN && a.lda % 64 == 0 && a.lda >= a.M;
    const bool b_blk = B_MN && BN % 64 == 0 && a.ldb % 64 == 0 && a.ldb >= a.N;
    CUtensorMap mapA, mapB;
    if constexpr (TF32) {
        mapA = make_map_3d_f32(a.A, a.K, a.M, nb, a.lda, 32, BM);
        mapB = make_map_3d_f32(a.B, a.K, a.N, nb, a.ldb, 32, BN);
    } else {
        mapA = a_blk  ? make_map_blocks_bf16(a.A, a.K, nb, a.lda, BK, BM / 64)
               : A_MN ? make_map_3d_bf16(a.A, a.M, a.K, nb, a.lda, 64, BK)
                      : make_map_3d_bf16(a.A, a.K, a.M, nb, a.lda, 64, BM);
        mapB = b_blk  ? make_map_blocks_bf16(a.B, a.K, nb, a.ldb, BK, BN / 64)
               : B_MN ? make_map_3d_bf16(a.B, a.N, a.K, nb, a.ldb, 64, BK)
                      : make_map_3d_bf16(a.B, a.K, a.N, nb, a.ldb, 64, BN);
    }
    const bool tma_c = !a.out_bf16 && !a.accumulate && a.split_k <= 1 && (a.ldc * 4) % 16 == 0 &&
                       (reinterpret_cast<uintptr_t>(a.C) & 15) == 0;
    const int bh = std::max(1, a.batch_h);
    EpiParams p{a.C, a.ldc, a.M, a.N, a.K, a.out_bf16, a.accumulate, tma_c, std::max(1, a.split_k), a.alpha, a.bias,
                a.row_mask, static_cast<int>(nb), bh, a_blk ? 1 : 0, b_blk ? 1 : 0};
    // C as [batch / batch_h][M][batch_h][N]: box {32 cols, 1, 32 rows, 1} (the 2-D 32 x 32 box)
    CUtensorMap mapC = mapA;
    // plain bf16 C (single product): 32 x 64 boxes
    p.tma_c16 = a.out_bf16 && !a.accumulate && a.split_k <= 1 && nb == 1 && (a.ldc * 2) % 16 == 0 &&
                (reinterpret_cast<uintptr_t>(a.C) & 15) == 0;
    if (p.tma_c16) {
        const uint64_t cd[4] = {static_cast<uint64_t>(a.N), 1, static_cast<uint64_t>(a.M), 1};
        const uint64_t cs[3] = {static_cast<uint64_t>(a.ldc) * 2, static_cast<uint64_t>(a.ldc) * 2,
                                static_cast<uint64_t>(a.M) * a.ldc * 2};
        const uint32_t cb[4] = {64, 1, 32, 1};
        mapC = make_map_4d_bf16_strided(a.C, cd, cs, cb);
    }
    if (tma_c) {
        const uint64_t cd[4] = {static_cast<uint64_t>(a.N), static_cast<uint64_t>(bh), static_cast<uint64_t>(a.M),
                                nb / bh};
        const uint64_t cs[3] = {static_cast<uint64_t>(nb > 1 ? a.ldc_h : a.ldc) * 4, static_cast<uint64_t>(a.ldc) * 4,
                                static_cast<uint64_t>(nb > 1 ? a.ldc_b : int64_t(a.M) * a.ldc) * 4};
        const uint32_t cb[4] = {32, 1, 32, 1};
        mapC = make_map_4d_f32_strided(a.C, cd, cs, cb);
    }
    CUtensorMap mapC16 = mapC;
    if (a.C16 != nullptr) {
        if (!tma_c || nb <= 1) throw std::invalid_argument("gemm: the bf16 copy of C is for batched fp32 products");
        p.c16_split = true;
        p.c16_f32_chunks = a.c16_f32_chunks;
        const uint64_t cd[4] = {static_cast<uint64_t>(a.N), static_cast<uint64_t>(bh), static_cast<uint64_t>(a.M),
                                nb / bh};
        const uint64_t cs[3] = {static_cast<uint64_t>(a.ldc_h) * 2, static_cast<uint64_t>(a.ldc) * 2,
                                static_cast<uint64_t>(a.ldc_b) * 2};
        const uint32_t cb[4] = {64, 1, 32, 1};
        mapC16 = make_map_4d_bf16_strided(a.C16, cd, cs, cb);
    }
    auto kern = gemm_bf16_kernel<BN, A_MN, B_MN, TF32>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);  // per device
    const int units = ((a.N + BN - 1) / BN) * ((a.M + BM - 1) / BM) * std::max(1, a.split_k) * static_cast<int>(nb);
    const int sms = device_sm_count();
    dim3 grid(static_cast<unsigned>(std::min(units, sms)));
    launch_pdl(kern, grid, dim3(kThreads), size_t(Cfg::kSmem), stream, mapA, mapB, mapC, mapC16, p);
}

// CTA pairs of a kernel resident at once (persistent grid size), cached per (device, kernel).
int resident_pairs(const void* kern, int smem) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({dev, kern});
    if (it != cache.end()) return it->second;
    int n = 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * 1024, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = static_cast<size_t>(smem);
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
        cudaGetLastError();
        n = std::max(1, device_sm_count() / 2 - 2);
    }
    cache[{dev, kern}] = n;
    return n;
}

template <int BN, bool A_MN, bool B_MN>
void launch_impl2(const GemmArgs& a, cudaStream_t stream) {
    using Cfg = GemmCfg2<BN>;
    constexpr int BK = Cfg::BK;
    const uint64_t nb = static_cast<uint64_t>(std::max(1, a.batch));
    const bool a_blk = A_MN && a.lda % 64 == 0 && a.lda >= a.M;
    const bool b_blk = B_MN && a.ldb % 64 == 0 && a.ldb >= a.N;
    // per CTA: its 128 A rows and HALF of the tile's B rows (K-major) / columns (MN-major)
    const CUtensorMap mapA = a_blk  ? make_map_blocks_bf16(a.A, a.K, nb, a.lda, BK, BM / 64)
                             : A_MN ? make_map_3d_bf16(a.A, a.M, a.K, nb, a.lda, 64, BK)
                                    : make_map_3d_bf16(a.A, a.K, a.M, nb, a.lda, 64, BM);
    const CUtensorMap mapB = b_blk  ? make_map_blocks_bf16(a.B, a.K, nb, a.ldb, BK, BN / 128)
                             : B_MN ? make_map_3d_bf16(a.B, a.N, a.K, nb, a.ldb, 64, BK)
                                    : make_map_3d_bf16(a.B, a.K, a.N, nb, a.ldb, 64, BN / 2);
    const bool tma_c = !a.out_bf16 && !a.accumulate && a.split_k <= 1 && (a.ldc * 4) % 16 == 0 &&
                       (reinterpret_cast<uintptr_t>(a.C) & 15) == 0;
    const int bh = std::max(1, a.batch_h);
    EpiParams p{a.C, a.ldc, a.M, a.N, a.K, a.out_bf16, a.accumulate, tma_c, std::max(1, a.split_k), a.alpha, a.bias,
                a.row_mask, static_cast<int>(nb), bh, a_blk ? 1 : 0, b_blk ? 1 : 0};
    CUtensorMap mapC = mapA;
    // plain bf16 C (single product): 32 x 64 boxes
    p.tma_c16 = a.out_bf16 && !a.accumulate && a.split_k <= 1 && nb == 1 && (a.ldc * 2) % 16 == 0 &&
                (reinterpret_cast<uintptr_t>(a.C) & 15) == 0;
    if (p.tma_c16) {
        const uint64_t cd[4] = {static_cast<uint64_t>(a.N), 1, static_cast<uint64_t>(a.M), 1};
        const uint64_t cs[3] = {static_cast<uint64_t>(a.ldc) * 2, static_cast<uint64_t>(a.ldc) * 2,
                                static_cast<uint64_t>(a.M) * a.ldc * 2};
        const uint32_t cb[4] = {64, 1, 32, 1};
        mapC = make_map_4d_bf16_strided(a.C, cd, cs, cb);
    }
    if (tma_c) {
        const uint64_t cd[4] = {static_cast<uint64_t>(a.N), static_cast<uint64_t>(bh), static_cast<uint64_t>(a.M),
                                nb / bh};
        const uint64_t cs[3] = {static_cast<uint64_t>(nb > 1 ? a.ldc_h : a.ldc) * 4, static_cast<uint64_t>(a.ldc) * 4,
                                static_cast<uint64_t>(nb > 1 ? a.ldc_b : int64_t(a.M) * a.ldc) * 4};
        const uint32_t cb[4] = {32, 1, 32, 1};
        mapC = make_map_4d_f32_strided(a.C, cd, cs, cb);
    }
    CUtensorMap mapC16 = mapC;
    if (a.C16 != nullptr) {
        if (!tma_c || nb <= 1) throw std::invalid_argument("gemm: the bf16 copy of C is for batched fp32 products");
        p.c16_split = true;
        p.c16_f32_chunks = a.c16_f32_chunks;
        const uint64_t cd[4] = {static_cast<uint64_t>(a.N), static_cast<uint64_t>(bh), static_cast<uint64_t>(a.M),
                                nb / bh};
        const uint64_t cs[3] = {static_cast<uint64_t>(a.ldc_h) * 2, static_cast<uint64_t>(a.ldc) * 2,
                                static_cast<uint64_t>(a.ldc_b) * 2};
        const uint32_t cb[4] = {64, 1, 32, 1};
        mapC16 = make_map_4d_bf16_strided(a.C16, cd, cs, cb);
    }
    auto kern = gemm2_bf16_kernel<BN, A_MN, B_MN>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    const int units = ((a.N + BN - 1) / BN) * ((a.M + 2 * BM - 1) / (2 * BM)) * std::max(1, a.split_k) *
                      static_cast<int>(nb);
    const int pairs = std::min(units, resident_pairs(reinterpret_cast<const void*>(kern), Cfg::kSmem));
    launch_pdl(kern, dim3(static_cast<unsigned>(2 * pairs)), dim3(kThreads), size_t(Cfg::kSmem), stream, mapA, mapB,
               mapC, mapC16, p);
}

}  // namespace

// fp32 GEMM on the tensor cores at ~fp32 accuracy ("3xTF32"): the caller passes K-concatenated
// operands, e.g. A' = [A_hi | A_lo | A_hi] and B'^T = [B_lo | B_hi | B_hi] (split3 layout, each part
// `K` columns), so one kind::tf32 product over K' = 3K sums A_hi B_lo + A_lo B_hi + A_hi B_hi
// (small cross terms first; dropped: A_lo B_lo ~ 2^-22 relative).  Operands fp32, K-major, row
// strides multiples of 4.
void launch_gemm_tf32(const GemmF32Args& a, cudaStream_t stream) {
    if (a.M <= 0 || a.N <= 0 || a.K <= 0) return;
    if ((a.lda * 4) % 16 != 0 || (a.ldb * 4) % 16 != 0 || (a.ldc * 4) % 16 != 0)
        throw std::invalid_argument("tf32 gemm: row strides must be multiples of 4 elements");
    GemmArgs g;
    g.A = reinterpret_cast<const __nv_bfloat16*>(a.A);
    g.B = reinterpret_cast<const __nv_bfloat16*>(a.B);
    g.C = a.C;
    g.lda = a.lda;
    g.ldb = a.ldb;
    g.ldc = a.ldc;
    g.M = a.M;
    g.N = a.N;
    g.K = a.K;
    g.bias = a.bias;
    g.row_mask = a.row_mask;
    if (a.N >= 2048 || (a.N % 256 == 0 && a.N >= 512))
        launch_impl<256, false, false, true>(g, stream);
    else
        launch_impl<128, false, false, true>(g, stream);
}

int pair_gemm_mode() {
    static const int mode = [] {
        const char* e = std::getenv("FIPA_PAIR_GEMM");
        return e == nullptr ? 1 : std::atoi(e);
    }();
    return mode;
}
bool pair_gemm_enabled() { return pair_gemm_mode() > 0; }

void launch_gemm_bf16(const GemmArgs& a, cudaStream_t stream) {
    if (a.M <= 0 || a.N <= 0 || a.K <= 0) return;
    // K tails need no special case: TMA zero-fills the out-of-range part of the last K block.
    // TMA does need 16-byte aligned row strides.
    if ((a.lda * 2) % 16 != 0 || (a.ldb * 2) % 16 != 0)
        throw std::invalid_argument("gemm: operand row strides must be multiples of 8 elements");
    if (a.accumulate && a.out_bf16) throw std::invalid_argument("gemm: accumulate needs fp32 C");
    if (a.split_k > 1 && (a.out_bf16 || a.bias || a.row_mask))
        throw std::invalid_argument("gemm: split-K accumulates plain fp32 C");
    if (a.batch > 1 && (a.out_bf16 || a.accumulate || a.split_k > 1 || a.row_mask || (a.ldc * 4) % 16 != 0 ||
                        (a.ldc_h * 4) % 16 != 0 || (a.ldc_b * 4) % 16 != 0 || a.batch % std::max(1, a.batch_h) != 0 ||
                        (reinterpret_cast<uintptr_t>(a.C) & 15) != 0))
        throw std::invalid_argument("gemm: batched products write plain, 16-byte aligned fp32 C");
    // 256-wide tiles halve the shared-memory traffic per MMA (A is re-read per N tile); batched
    // products with N in (256, 512] (dQ: N = 432) cover N with two of them.  (Two 224-wide tiles
    // compute 448 instead of 512 columns but measured slower: dQ 0.073 -> 0.076 ms at B=8 L=1024,
    // their B operand needs four 3-D TMA boxes per stage instead of one 4-D box.)
    const int sel = (a.a_mn_major ? 1 : 0) | (a.b_mn_major ? 2 : 0);
    // (FIPA_PAIR_GEMM=2 also routes wide single products -- dfeat: N = 2432, K = 256 -- to pairs:
    // no gain measured there, the short-K product is epilogue-bound)
    const bool pair_wide = pair_gemm_mode() >= 2 && a.batch <= 1 && a.split_k <= 1 && a.N >= 2048 && a.M >= 4096;
    if (pair_gemm_enabled() && ((a.batch > 1 && a.N > 256 && a.M >= 256) || pair_wide)) {
        // batched dQ (and wide single products): 256 x 256 tiles over CTA pairs (half the B operand
        // bytes per SM)
        switch (sel) {
            case 0: return launch_impl2<256, false, false>(a, stream);
            case 1: return launch_impl2<256, true, false>(a, stream);
            case 2: return launch_impl2<256, false, true>(a, stream);
            default: return launch_impl2<256, true, true>(a, stream);
        }
    }
    const bool wide = a.N >= 2048 || (a.N % 256 == 0 && a.N >= 512) || (a.batch > 1 && a.N > 256);
    if (wide) {
        switch (sel) {
            case 0: return launch_impl<256, false, false>(a, stream);
            case 1: return launch_impl<256, true, false>(a, stream);
            case 2: return launch_impl<256, false, true>(a, stream);
            default: return launch_impl<256, true, true>(a, stream);
        }
    }
    switch (sel) {
        case 0: return launch_impl<128, false, false>(a, stream);
        case 1: return launch_impl<128, true, false>(a, stream);
        case 2: return launch_impl<128, false, true>(a, stream);
        default: return launch_impl<128, true, true>(a, stream);
    }
}

}  // namespace fipa_b200
