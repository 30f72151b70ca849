// FlashIPA attention backward on tcgen05 (the reference has no backward -- proj/SPEC.md:8 --
// so this differentiates its forward, proj/src/attention_kernel.cpp:112-188, against the oracle
// backward in oracle/fipa_oracle.py, itself pinned by finite differences of the reference).
//
// With S = Q_hat K_hat^T in log2 units (pack.cu), P = 2^(S - lse2) (lse saved by the forward),
// dO_hat and D = rowsum(dO_hat * O_hat) from bwd_prep (bwd.cu):
//   dP = dO_hat V_hat^T,  dS = P * (dP - D)            (natural-logit gradient)
//   dV_acc = P^T dO_hat,  dK_acc = dS^T Q_hat,  dQ_acc = dS K_hat
// The lifted head width (432 columns for the north-star shape) is the constraint that shapes the
// design: one accumulator of 128 rows x 432 fp32 fills 432 of a CTA's 512 TMEM columns, so
// dK and dV of the same keys cannot share an SM, and a 128 x 448 bf16 stationary tile fills half
// of the shared memory.  Each kernel therefore runs a CLUSTER OF FOUR: two tcgen05 CTA pairs
// (cta_group::2, M = 256 rows) over the same 256 rows of one (sample, head):
//   "P pair"  (ranks 0,1): X = A_stat . B1_j^T into TMEM, P = 2^(X - lse2) (bf16) into one of
//                          two shared-memory buffers, optional acc += P . B2_j, and the 16 KB P
//                          tile pushed to the peer pair with ONE cp.async.bulk smem->DSMEM copy
//                          (completion counted on the peer's mbarrier);
//   "dS pair" (ranks 2,3): X = A_stat . B1_j^T -> dP, dS = P (dP - D) written over the received P
//                          in place (double-buffered), acc += dS . B2_j; the MMA commit that
//                          retires dS releases that buffer to the P pair (multicast commit).
// Measured (tools/attn_bwd_trace.cu): per-thread st.async stores moved the tile at ~9 B/clk and
// serialised the pairs; the bulk copy runs at ~16 B/clk.  The remaining limiter is the B2 ring
// (3 x 8 KB next to the 112 KB stationary tile): TMA latency exceeds its lead time.
// KV kernel (rows = keys, tile columns = 64 queries):
//   P pair : A_stat = K_hat, B1 = Q_hat tiles, B2 = dO_hat slices -> acc = dV_acc
//   dS pair: A_stat = V_hat, B1 = dO_hat tiles, B2 = Q_hat slices -> acc = dK_acc
// Q kernel (rows = queries, tile columns = 64 keys):
//   P pair : A_stat = Q_hat, B1 = K_hat tiles (no second MMA)
//   dS pair: A_stat = dO_hat, B1 = V_hat tiles, B2 = K_hat slices -> acc = dQ_acc
// Per-query vectors (lse, D) are per tile column in the KV kernel and per row in the Q kernel.
// The ring structure (whole 32-row B1 tiles, 32-row B2 slices split over the pair) is the
// forward's (attn_fwd_2sm.cu); MMA1 writes TMEM columns [448,512), the accumulator [0,n2).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>
#include <tuple>

#include "kernels.hpp"
#include "ptx.cuh"
#include "tma_host.hpp"

namespace fipa_b200 {

namespace {

constexpr int BM = 128;       // rows per CTA (256 per pair)
constexpr int BN = 64;        // tile columns
constexpr int kThreads = 480; // w0 stat/B1 producer, w1 TMEM + MMA, w2..w9 elementwise, w10 B2 producer,
                              // w11..w14 accumulator epilogue (one per TMEM lane quadrant)
constexpr int kMaxStages1 = 6;  // B1 ring: whole 32-row tile halves, or groups of KB1 column blocks
constexpr int kMaxStages2 = 6;  // 16-row B2 slices (see finish_params)
// B2 slices of 16 or 32 rows (template SL): TMA throughput per SM grows with the box size
// (profiles/r1_tma_microbench.txt: 2 KB boxes ~20 B/clk, 4 KB ~40 B/clk), so 32-row slices halve
// the number of boxes per tile at the same ring bytes.
constexpr uint32_t kXCol = 448;
constexpr float kL2E = 1.4426950408889634f;

struct RoleDims {
    int k1;        // MMA1 K extent (multiple of 16)
    int nb1;       // 64-wide blocks of the stationary tile / B1 tiles
    int n2;        // MMA2 N extent (accumulator columns), 0 = no second MMA
    int n2a, n2b;  // split into N <= 256 MMAs
    int nba, nbb;  // per-CTA 64-wide TMA boxes of each half of a B2 slice
};

struct BwdParams {
    int Lrow, Lcol, H, B, BH;   // rows (keys in KV, queries in Q) / tile columns; BH = B * H
    int col0, ncol;             // tile columns [col0, col0 + ncol) of this launch (query chunks, KV kernel)
    int acc_add;                // accumulators reduced into (TMA add) instead of stored: later chunks
    int stat_chunk, col_chunk;  // rows per shard of the stationary / column operands (sharded keys)
    int stat_sharded, col_sharded;  // 1: operand read through the 5-D / 4-D rank-major maps (measured
                                    // ~10% slower per box than the unsharded 4-D / 3-D maps)
    RoleDims role[2];  // 0 = P pair, 1 = dS pair
    int stat_bytes, b1_stage, b2_stage, nst2;
    int kb1;           // column blocks per B1 stage (= nb1: whole tiles)
    int nst1;          // B1 ring depth (1 or 2)
    int nab;           // P / dS exchange buffers (2 or 3)
    int slice;         // B2 slice rows (16 or 32)
    const float* lse;  // [BH, L] natural-log LSE of the forward
    const float* Dvec; // [BH, L] rowsum(dO_hat * O_hat)
    float* acc_out[2]; // [BH, L, acc_ld] fp32 (null = none)
    int acc_ld;
    int acc_col0[2];   // first accumulator column each pair writes (dQ split over the pairs)
    int b2_col0[2];    // first B2 column each pair streams
    int ds_store;      // KV kernel: dS tiles also written to global [BH][Lk][ds_ld] (bf16) for dQ
    int acc16;         // KV kernel: accumulators leave as bf16 (accP16 / accD16), plus fp32 for the
    uint32_t f32_chunks[2];  // 32-column chunks flagged here (per role: point / translation columns)
};

struct Bars {
    uint64_t stat_full;
    uint64_t b1_full[kMaxStages1], b1_empty[kMaxStages1];
    uint64_t b2_full[kMaxStages2], b2_empty[kMaxStages2];
    uint64_t stat_empty;
    uint64_t x_full, x_free, a_full, acc_full, acc_empty, acc_empty_b;
    uint64_t mma2_done[3], pin_full[3], pin_free[3];  // per P / dS exchange buffer (2 or 3)
    uint64_t dsin_full[3];                            // Q kernel: dS returned to the P pair
    uint32_t tmem_slot;
};

struct Layout {
    int stat, abuf, b1, b2, stage, bars, total;
};
__host__ __device__ inline Layout smem_layout(const BwdParams& p) {
    Layout l{};
    l.stat = 0;
    l.abuf = p.stat_bytes;
    l.b1 = l.abuf + p.nab * BM * 128;  // P (P pair) / received-P-then-dS (dS pair) exchange buffers
    l.b2 = l.b1 + p.nst1 * p.b1_stage;
    l.stage = (l.b2 + p.nst2 * p.b2_stage + 1023) & ~1023;  // 4 epilogue warps x one 4 KB TMA-store box
    l.bars = l.stage + 4 * 4096;
    l.total = l.bars + static_cast<int>(sizeof(Bars));
    return l;
}

// Optional per-event timestamps of cluster (0, bh 0) for pipeline analysis (tools/attn_bwd_trace.cu).
#ifdef FIPA_ATTN_BWD_TRACE
__device__ long long g_bwd_trace[4 * 12 * 16 * 64];  // [cta][warp][event][tile]
#define BTRACE(ev, j)                                                                                    \
    do {                                                                                                 \
        if (blockIdx.x < 4 && blockIdx.y == 0 && (j) < 64)                                               \
            g_bwd_trace[((blockIdx.x * 12 + ptx::warp_id()) * 16 + (ev)) * 64 + (j)] = clock64();        \
    } while (0)
// Per-unit events of the first cluster (persistent loop): [cta][unit][event]
__device__ long long g_unit_trace[4 * 16 * 8];
#define UTRACE(ev, itv)                                                                                  \
    do {                                                                                                 \
        if (blockIdx.x < 4 && (itv) < 16) g_unit_trace[(blockIdx.x * 16 + (itv)) * 8 + (ev)] = clock64(); \
    } while (0)
#else
#define BTRACE(ev, j) \
    do {              \
    } while (0)
#define UTRACE(ev, itv) \
    do {                \
    } while (0)
#endif

// Bulk copy (async proxy) of `bytes` from this CTA's shared memory into a peer CTA's shared
// memory; completion is counted on the peer's mbarrier.  One 16 KB copy per tile sustains far more
// than per-thread st.async stores, which each carry their own mbarrier transaction (measured
// ~9 B/clk, tools/attn_bwd_trace.cu).
__device__ __forceinline__ void bulk_copy_s2cluster(uint32_t dst_cluster, const void* src, uint32_t bytes,
                                                    uint32_t bar_cluster) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst_cluster), "r"(ptx::smem_u32(src)), "r"(bytes), "r"(bar_cluster)
                 : "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// 32 consecutive per-query floats starting at q (entries >= L come back as `fill`).
__device__ __forceinline__ void load_vec32(const float* base, int q, int L, float fill, float* out) {
    if (q + 32 <= L && (reinterpret_cast<uintptr_t>(base + q) & 15) == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float4 f = __ldg(reinterpret_cast<const float4*>(base + q) + k);
            out[4 * k] = f.x;
            out[4 * k + 1] = f.y;
            out[4 * k + 2] = f.z;
            out[4 * k + 3] = f.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < 32; ++k) out[k] = q + k < L ? __ldg(base + q + k) : fill;
    }
}

// TMA tensor reduction store (fp32 add into global): later query chunks of the materialised-dS
// backward add their partial dK / dV to the accumulators the first chunk stored
__device__ __forceinline__ void tma_reduce_add_5d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3,
                                                  int c4) {
    asm volatile("cp.reduce.async.bulk.tensor.5d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];"
                 ::"l"(reinterpret_cast<uint64_t>(map)), "r"(ptx::smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
                   "r"(c4)
                 : "memory");
}

// NST2: depth of the B2 ring, a compile-time constant -- the slice refill sits on the critical path
// and a runtime ring index measured ~8% slower (same-box A/B at B=8 L=1024).
//
// Persistent: the grid holds as many 4-CTA clusters as fit at once (33 on B200), and each cluster
// walks the work units (sample-head, 256-row block) u = cluster, cluster + nclusters, ...  Every
// ring, exchange buffer and barrier phase runs on counters global over the cluster's tiles, so the
// next unit's operand loads, first Q.K^T and softmax overlap the previous unit's last tiles, and
// four dedicated epilogue warps (w11..w14, one per TMEM lane quadrant) drain the accumulator while
// the elementwise warps start the next unit:
//   stat_empty (MMA commit after a unit's last MMA1)   -> the producer reloads the stationary tile;
//   acc_empty / acc_empty_b (8 epilogue-warp arrivals) -> columns [0, n2a) / [n2a, n2) are out of
//                                                         TMEM; the next unit's first MMA2 may run.
// The drain leaves through 4 KB TMA-store boxes; an SM stores at most ~32 B/clk
// (tools/store_microbench.cu), so the 221 KB accumulator of a unit still holds the next unit's
// first MMA2 back a few thousand cycles.  Measured (B=8 L=1024, dK/dV): 0.300 -> 0.28 ms; the
// non-persistent kernel idled the tensor pipe through each CTA's prologue and epilogue (6 + 5.7 us
// of a 36 us lifetime) and ran 1024 CTAs in 7.76 waves.  tcgen05.ld 16x256b read TMEM ~3x slower
// than 32x32b here (9.5k vs 3k cycles for 128 x 432 fp32), and stores whose 32-byte sectors were
// completed by two different instructions ran ~10x slower (partial-sector writes).
template <bool KV, int kStages1, int NST2, int NAB, int KB1, int SL>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(kThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap statP, const __grid_constant__ CUtensorMap b1P,
                    const __grid_constant__ CUtensorMap b2P, const __grid_constant__ CUtensorMap statD,
                    const __grid_constant__ CUtensorMap b1D, const __grid_constant__ CUtensorMap b2D,
                    const __grid_constant__ CUtensorMap mapDS, const __grid_constant__ CUtensorMap accP,
                    const __grid_constant__ CUtensorMap accD, const __grid_constant__ CUtensorMap accP16,
                    const __grid_constant__ CUtensorMap accD16, BwdParams p) {
    constexpr int kSlice = SL, kSliceBox = SL * 128;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const Layout lay = smem_layout(p);
    uint8_t* sStat = smem + lay.stat;
    uint8_t* sA = smem + lay.abuf;
    uint8_t* sB1 = smem + lay.b1;
    uint8_t* sB2 = smem + lay.b2;
    Bars* bars = reinterpret_cast<Bars*>(smem + lay.bars);

    const int warp = ptx::warp_id();
    const int lane = ptx::lane_id();
    const uint32_t crank = ptx::cluster_ctarank();  // 0..3
    const int role = static_cast<int>(crank >> 1);  // 0 = P pair, 1 = dS pair
    const uint32_t prank = crank & 1u;              // rank within the pair
    const bool leader = prank == 0;
    const uint16_t pair_mask = static_cast<uint16_t>(0x3u << (crank & 2u));
    const RoleDims rd = p.role[role];
    const int ntiles = (p.ncol + BN - 1) / BN;
    const int nrb = (p.Lrow + 255) / 256;                // 256-row blocks per (sample, head)
    const int nunits = p.BH * nrb;
    const int cluster = static_cast<int>(blockIdx.x >> 2), nclusters = static_cast<int>(gridDim.x >> 2);
    const bool has_mma2 = rd.n2 > 0;
    const CUtensorMap* mStat = role ? &statD : &statP;
    const CUtensorMap* mB1 = role ? &b1D : &b1P;
    const CUtensorMap* mB2 = role ? &b2D : &b2P;
    auto unit_bh = [&](int u) { return u / nrb; };
    auto unit_r0 = [&](int u) { return (u - (u / nrb) * nrb) * 256 + static_cast<int>(prank) * BM; };
    if (warp == 0 && lane == 0) {
        span_mark(0);
        ptx::tma_prefetch(mStat);
        ptx::tma_prefetch(mB1);
        if (has_mma2) ptx::tma_prefetch(mB2);
        ptx::mbar_init(&bars->stat_full, 1);
        ptx::mbar_init(&bars->stat_empty, 1);
        for (int s = 0; s < kStages1; ++s) {
            ptx::mbar_init(&bars->b1_full[s], 1);
            ptx::mbar_init(&bars->b1_empty[s], 1);
        }
        for (int s = 0; s < p.nst2; ++s) {
            ptx::mbar_init(&bars->b2_full[s], 1);
            ptx::mbar_init(&bars->b2_empty[s], 1);
        }
        ptx::mbar_init(&bars->x_full, 1);
        ptx::mbar_init(&bars->x_free, 16);
        // Q kernel, P pair: the MMA operand (dS) arrives by copy; the odd CTA forwards its arrival
        ptx::mbar_init(&bars->a_full, (!KV && role == 0) ? 1 : 16);
        ptx::mbar_init(&bars->acc_full, 1);
        ptx::mbar_init(&bars->acc_empty, 8);    // columns [0, n2a) read out: 4 epilogue warps x 2 CTAs
        ptx::mbar_init(&bars->acc_empty_b, 8);  // columns [n2a, n2) read out
        for (int b = 0; b < 3; ++b) {
            ptx::mbar_init(&bars->mma2_done[b], 1);
            ptx::mbar_init(&bars->pin_full[b], 1);
            // materialised dS: the buffer is also released by the dS CTA once its TMA store has read it
            ptx::mbar_init(&bars->pin_free[b], (KV && p.ds_store) ? 2 : 1);
            ptx::mbar_init(&bars->dsin_full[b], 1);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc_2sm(&bars->tmem_slot, 512);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, bars->tmem_slot, 0);
    ptx::pdl_wait();  // dO_hat, D of the preceding prep (and, per query chunk, the previous dQ GEMM)
    ptx::pdl_trigger();

    if (warp == 0) {
        // ------------------------------------------- stationary tile + B1 tile producer
        if (lane == 0) {
            const int nk1 = KB1 ? (rd.nb1 + KB1 - 1) / KB1 : 1;  // B1 stages per tile
            const int stage = (KB1 ? KB1 : rd.nb1) * 32 * 128;
            int n = 0;  // B1 stages issued (ring slot n % kStages1)
            int it = 0;
            for (int u = cluster; u < nunits; u += nclusters, ++it) {
                const int bh = unit_bh(u), r0 = unit_r0(u);
                // the previous unit's last MMA1 has read the stationary tile
                if (it > 0) ptx::mbar_wait(&bars->stat_empty, (it - 1) & 1);
                UTRACE(6, it);
                if (leader) ptx::mbar_expect_tx(&bars->stat_full, 2 * rd.nb1 * BM * 128);
                if (p.stat_sharded) {
                    const int g = r0 / p.stat_chunk;  // rows past the end land in shard G: TMA zero fill
                    ptx::tma_load_5d_2sm(sStat, mStat, &bars->stat_full, 0, r0 - g * p.stat_chunk, 0, bh, g);
                } else {
                    ptx::tma_load_4d_2sm(sStat, mStat, &bars->stat_full, 0, r0, 0, bh);
                }
                for (int j = 0; j < ntiles; ++j) {
                    if (it == 0) BTRACE(11, j);
                    const int key = p.col0 + j * BN + 32 * static_cast<int>(prank);
                    const int g = p.col_sharded ? key / p.col_chunk : 0;
                    for (int uu = 0; uu < nk1; ++uu, ++n) {
                        const int s = n % kStages1;
                        if (n >= kStages1) ptx::mbar_wait(&bars->b1_empty[s], ((n / kStages1) - 1) & 1);
                        if (leader) ptx::mbar_expect_tx(&bars->b1_full[s], 2 * stage);
                        if (p.col_sharded) {
                            ptx::tma_load_5d_2sm(sB1 + s * p.b1_stage, mB1, &bars->b1_full[s], 0,
                                                 key - g * p.col_chunk, uu * KB1, bh, g);
                        } else {
                            ptx::tma_load_4d_2sm(sB1 + s * p.b1_stage, mB1, &bars->b1_full[s], 0, key, uu * KB1, bh);
                        }
                    }
                }
            }
        }
    } else if (warp == 10) {
        // ------------------------------------------------------------ B2 slice producer
        if (lane == 0 && has_mma2) {
            // the refill of a slice sits on the critical path: no division or branching between the
            // empty-barrier wait and the TMA issues (slot / phase by counters, columns precomputed)
            const int halfa = rd.n2a / 2, halfb = rd.n2b / 2;
            const int stage_bytes = (rd.nba + rd.nbb) * kSliceBox;
            const int nslices = ntiles * (BN / kSlice);
            const int col_a = p.b2_col0[role] + halfa * static_cast<int>(prank);
            const int col_b = p.b2_col0[role] + rd.n2a + halfb * static_cast<int>(prank);
            int s = 0, ph = 0, n = 0;
            for (int u = cluster; u < nunits; u += nclusters) {
                const int bh = unit_bh(u);
                int g = 0, rloc = 0;
                for (int i = 0; i < nslices; ++i, ++n) {
                    if (n >= NST2) ptx::mbar_wait(&bars->b2_empty[s], ph ^ 1);
                    if (n < 64) BTRACE(12, n);
                    if (leader) ptx::mbar_expect_tx(&bars->b2_full[s], 2 * stage_bytes);
                    uint8_t* dst = sB2 + s * p.b2_stage;
                    if (p.col_sharded) {
                        for (int x = 0; x < rd.nba; ++x)
                            ptx::tma_load_4d_2sm(dst + x * kSliceBox, mB2, &bars->b2_full[s], col_a + 64 * x, rloc, bh, g);
                        for (int x = 0; x < rd.nbb; ++x)
                            ptx::tma_load_4d_2sm(dst + (rd.nba + x) * kSliceBox, mB2, &bars->b2_full[s],
                                                 col_b + 64 * x, rloc, bh, g);
                    } else {
                        const int row = p.col0 + i * kSlice;
                        for (int x = 0; x < rd.nba; ++x)
                            ptx::tma_load_3d_2sm(dst + x * kSliceBox, mB2, &bars->b2_full[s], col_a + 64 * x, row, bh);
                        for (int x = 0; x < rd.nbb; ++x)
                            ptx::tma_load_3d_2sm(dst + (rd.nba + x) * kSliceBox, mB2, &bars->b2_full[s], col_b + 64 * x,
                                                 row, bh);
                    }
                    rloc += kSlice;  // shard-local row of the next slice
                    if (rloc >= p.col_chunk) {
                        rloc -= p.col_chunk;
                        ++g;
                    }
                    if (++s == NST2) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // -------------------------------------------------- MMA issue (pair leaders)
        if (!leader && !KV && role == 0 && has_mma2) {
            // Q kernel, odd CTA of the P pair: forward the arrival of each returned dS tile to the
            // leader (a bulk copy can only complete on a barrier of the destination CTA)
            if (lane == 0) {
                const uint32_t a_full_leader = ptx::mapa(&bars->a_full, crank & 2u);
                const int ntot = ((nunits - cluster + nclusters - 1) / nclusters) * ntiles;
                for (int t = 0; t < ntot; ++t) {
                    ptx::mbar_wait(&bars->dsin_full[t % NAB], (t / NAB) & 1);
                    ptx::mbar_arrive_remote(a_full_leader);
                }
            }
        }
        if (leader) {
            const uint32_t idesc1 = ptx::idesc_bf16(256, BN, false, false);
            const uint32_t idesc2a = ptx::idesc_bf16(256, rd.n2a > 0 ? rd.n2a : 16, false, true);
            const uint32_t idesc2b = ptx::idesc_bf16(256, rd.n2b > 0 ? rd.n2b : 16, false, true);
            const uint32_t stat_base = ptx::smem_u32(sStat);
            const uint32_t a_base = ptx::smem_u32(sA);
            const uint32_t b1_base = ptx::smem_u32(sB1);
            const uint32_t b2_base = ptx::smem_u32(sB2);
            const int k1_steps = rd.k1 / 16;
            const int nk1 = KB1 ? (rd.nb1 + KB1 - 1) / KB1 : 1;
            // descriptors advance by 64-bit adds of (byte offset >> 4): the issue thread's work per
            // MMA is a couple of integer ops (it is on the critical path with ~35 MMAs per tile)
            const uint64_t d_stat = ptx::sw128_desc(stat_base, 16, 1024);
            const uint64_t d_b1 = ptx::sw128_desc(b1_base, 16, 1024);
            const uint64_t d_a = ptx::sw128_desc(a_base, 16, 1024);
            const uint64_t d_b2 = ptx::sw128_desc(b2_base, kSliceBox, 1024);
            int it = 0, t = 0;  // t: global tile index of MMA1 (tile j of unit it)
            int n1 = 0, n2 = 0;  // B1 stages / B2 slices consumed
            for (int u = cluster; u < nunits; u += nclusters, ++it) {
                ptx::mbar_wait(&bars->stat_full, it & 1);
                if (lane == 0) UTRACE(0, it);
                for (int j = 0; j <= ntiles; ++j) {
                    if (j < ntiles) {
                        if (t > 0) ptx::mbar_wait_cluster(&bars->x_free, (t - 1) & 1);
                        if (lane == 0 && it == 0) BTRACE(2, j);
                        for (int uu = 0; uu < nk1; ++uu, ++n1) {
                            const int s = n1 % kStages1;
                            ptx::mbar_wait(&bars->b1_full[s], (n1 / kStages1) & 1);
                            if (lane == 0 && uu == 0 && it == 0) BTRACE(0, j);
                            ptx::tc_fence_after();
                            if (ptx::elect_one()) {
                                const uint64_t db0 = d_b1 + static_cast<uint64_t>((s * p.b1_stage) >> 4);
                                const int b_lo = uu * KB1, b_hi = KB1 ? min(rd.nb1, (uu + 1) * KB1) : rd.nb1;
                                for (int blk = b_lo; blk < b_hi; ++blk) {
                                    const uint64_t da_b = d_stat + static_cast<uint64_t>((blk * (BM * 128)) >> 4);
                                    const uint64_t db_b = db0 + static_cast<uint64_t>(((blk - b_lo) * (32 * 128)) >> 4);
#pragma unroll
                                    for (int sub = 0; sub < 4; ++sub) {
                                        if (4 * blk + sub < k1_steps)
                                            ptx::mma2_ss(tmem + kXCol, da_b + 2 * sub, db_b + 2 * sub, idesc1,
                                                         (blk | sub) != 0);
                                    }
                                }
                                ptx::mma_commit_2sm(&bars->b1_empty[s], pair_mask);
                                if (uu == nk1 - 1) {
                                    ptx::mma_commit_2sm(&bars->x_full, pair_mask);
                                    // last MMA1 of the unit: the stationary tile may be reloaded
                                    if (j == ntiles - 1) ptx::mma_commit_2sm(&bars->stat_empty, pair_mask);
                                }
                            }
                            __syncwarp();
                        }
                        ++t;
                    }
                    if (j > 0 && has_mma2) {
                        const int jj = j - 1, tt = t - (j < ntiles ? 2 : 1);  // global index of tile jj
                        if (!KV && role == 0) ptx::mbar_wait(&bars->dsin_full[tt % NAB], (tt / NAB) & 1);
                        ptx::mbar_wait_cluster(&bars->a_full, tt & 1);
                        // the previous unit's epilogue has read the accumulator out of TMEM: columns
                        // [0, n2a) first -- the first tile's n2a-wide MMAs go as soon as those are
                        // out (both of its B2 slices are resident), the n2b-wide ones after the rest
                        if (jj == 0 && it > 0) ptx::mbar_wait_cluster(&bars->acc_empty, (it - 1) & 1);
                        if (lane == 0 && jj == 0) UTRACE(1, it);
                        if (lane == 0 && it == 0) BTRACE(1, jj);
                        const bool split_first = jj == 0 && it > 0 && rd.n2b > 0 && NST2 >= BN / kSlice;
                        if (split_first) {
                            const int n2s = n2;
                            for (int h2 = 0; h2 < BN / kSlice; ++h2) {
                                const int s = (n2s + h2) % NST2;
                                ptx::mbar_wait(&bars->b2_full[s], ((n2s + h2) / NST2) & 1);
                                ptx::tc_fence_after();
                                if (ptx::elect_one()) {
#pragma unroll
                                    for (int kk = 0; kk < kSlice / 16; ++kk) {
                                        const uint64_t da = d_a + static_cast<uint64_t>(
                                            ((tt % NAB) * (BM * 128) + ((kSlice / 16) * h2 + kk) * 32) >> 4);
                                        const uint64_t db = d_b2 + static_cast<uint64_t>((s * p.b2_stage + kk * 2048) >> 4);
                                        ptx::mma2_ss(tmem, da, db, idesc2a, (h2 > 0 || kk > 0) ? 1u : 0u);
                                    }
                                }
                                __syncwarp();
                            }
                            ptx::mbar_wait_cluster(&bars->acc_empty_b, (it - 1) & 1);
                            ptx::tc_fence_after();
                            for (int h2 = 0; h2 < BN / kSlice; ++h2, ++n2) {
                                const int s = n2 % NST2;
                                if (ptx::elect_one()) {
#pragma unroll
                                    for (int kk = 0; kk < kSlice / 16; ++kk) {
                                        const uint64_t da = d_a + static_cast<uint64_t>(
                                            ((tt % NAB) * (BM * 128) + ((kSlice / 16) * h2 + kk) * 32) >> 4);
                                        const uint64_t db = d_b2 + static_cast<uint64_t>((s * p.b2_stage + kk * 2048) >> 4);
                                        ptx::mma2_ss(tmem + rd.n2a, da, db + static_cast<uint64_t>((rd.nba * kSliceBox) >> 4),
                                                     idesc2b, (h2 > 0 || kk > 0) ? 1u : 0u);
                                    }
                                    ptx::mma_commit_2sm(&bars->b2_empty[s], pair_mask);
                                }
                                __syncwarp();
                            }
                        } else {
                        if (jj == 0 && it > 0 && rd.n2b > 0) ptx::mbar_wait_cluster(&bars->acc_empty_b, (it - 1) & 1);
                        for (int h2 = 0; h2 < BN / kSlice; ++h2, ++n2) {
                            const int s = n2 % NST2;
                            ptx::mbar_wait(&bars->b2_full[s], (n2 / NST2) & 1);
                            if (lane == 0 && h2 == BN / kSlice - 1 && it == 0) BTRACE(13, jj);
                            ptx::tc_fence_after();
                            if (ptx::elect_one()) {
#pragma unroll
                                for (int kk = 0; kk < kSlice / 16; ++kk) {
                                    const uint64_t da = d_a + static_cast<uint64_t>(
                                        ((tt % NAB) * (BM * 128) + ((kSlice / 16) * h2 + kk) * 32) >> 4);
                                    const uint64_t db = d_b2 + static_cast<uint64_t>((s * p.b2_stage + kk * 2048) >> 4);
                                    const uint32_t acc = (jj > 0 || h2 > 0 || kk > 0) ? 1u : 0u;
                                    ptx::mma2_ss(tmem, da, db, idesc2a, acc);
                                    if (rd.n2b > 0)
                                        ptx::mma2_ss(tmem + rd.n2a, da,
                                                     db + static_cast<uint64_t>((rd.nba * kSliceBox) >> 4), idesc2b, acc);
                                }
                                ptx::mma_commit_2sm(&bars->b2_empty[s], pair_mask);
                            }
                            __syncwarp();
                        }
                        }  // !split_first
                        if (ptx::elect_one()) {
                            // P pair: its P buffer is free again.  dS pair: the received-P buffer
                            // is free -> the P pair may send the next tile.
                            if (role == 0) ptx::mma_commit_2sm(&bars->mma2_done[tt % NAB], pair_mask);
                            else ptx::mma_commit_2sm(&bars->pin_free[tt % NAB], 0x3);
                            if (j == ntiles) ptx::mma_commit_2sm(&bars->acc_full, pair_mask);
                        }
                        __syncwarp();
                    }
                }
            }
        }
    } else if (warp >= 11) {
        // ---------------------------------------------- accumulator epilogue (own warps)
        // drains unit u's accumulator while the elementwise warps start unit u+1's tiles; the
        // next unit's first MMA2 waits on acc_empty
        const int quad = warp & 3;
        const uint32_t tl = tmem + (uint32_t(quad * 32) << 16);
        const uint32_t acc_empty_remote = ptx::mapa(&bars->acc_empty, crank & 2u);
        const uint32_t acc_empty_b_remote = ptx::mapa(&bars->acc_empty_b, crank & 2u);
        int it = 0;
        for (int u = cluster; u < nunits; u += nclusters, ++it) {
            if (!has_mma2) break;
            const int bh = unit_bh(u), r0 = unit_r0(u);
            float* out = p.acc_out[role];
            if (warp == 11 && lane == 0) UTRACE(3, it);
            ptx::mbar_wait(&bars->acc_full, it & 1);
            ptx::tc_fence_after();
            if (warp == 11 && lane == 0) UTRACE(4, it);
            if (warp == 11 && lane == 0 && it == 0) span_mark(1);
            if (out != nullptr) {
                const int bb = bh / p.H, hh = bh - bb * p.H;
                // thread = row (TMEM lane, tcgen05.ld 32x32b: the 16x256b shape read TMEM ~3x slower,
                // 9.5k vs 3k cycles for a 128 x 432 fp32 tile).  Each 32-column chunk is staged as a
                // 128-byte-swizzled 32 x 32 box (this warp's 4 KB) and leaves by one TMA tensor
                // store of 32 full 128-byte lines; stores straight from registers (32-byte sectors
                // of 32 rows per instruction) ran at ~25 B/clk per SM and held the next unit's
                // first MMA2 back for the whole drain.  The next chunk's TMEM load is in flight
                // while the previous box is read out.
                const int g = (r0 + quad * 32) / p.stat_chunk, gi = r0 + quad * 32 - g * p.stat_chunk;
                const bool rows_ok = r0 + quad * 32 < p.Lrow;
                const CUtensorMap* mAcc = role ? &accD : &accP;
                uint8_t* box = smem + lay.stage + (warp - 11) * 4096;
                const int n32 = (rd.n2 + 31) / 32;
                uint32_t o0[32], o1[32];
                auto stage_box = [&](const uint32_t* w, int cb) {
                    if (lane == 0) ptx::bulk_wait_group_read<0>();  // the previous box has been read
                    __syncwarp();
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        *reinterpret_cast<uint4*>(box + lane * 128 + ((k ^ (lane & 7)) << 4)) =
                            make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0 && rows_ok) {
                        if (p.acc_add)
                            tma_reduce_add_5d(mAcc, box, 32 * cb, hh, gi, bb, g);
                        else
                            ptx::tma_store_5d(mAcc, box, 32 * cb, hh, gi, bb, g);
                        ptx::bulk_commit_group();
                    }
                };
                // columns [0, n2a) out of TMEM -> acc_empty (the next unit's first n2a-wide MMAs)
                const int na32 = rd.n2b > 0 ? rd.n2a / 32 : n32;
                auto read_out_a = [&](int cb) {
                    if (cb + 1 == na32) {
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive_cluster_relaxed(acc_empty_remote);
                    }
                };
                ptx::tmem_ld32(tl, o0);
                if (p.acc16) {
                    // chunk pairs -> one 32 x 64 bf16 box (128-byte lines); the chunks holding point /
                    // translation columns also leave in fp32
                    const CUtensorMap* mAcc16 = role ? &accD16 : &accP16;
                    const uint32_t f32m = p.f32_chunks[role];
                    for (int cb = 0; cb < n32; cb += 2) {
                        const bool has1 = cb + 1 < n32;
                        ptx::tmem_wait_ld();
                        read_out_a(cb);
                        if (has1) {
                            ptx::tmem_ld32(tl + 32 * (cb + 1), o1);
                            ptx::tmem_wait_ld();
                            read_out_a(cb + 1);
                        }
                        if (lane == 0) ptx::bulk_wait_group_read<0>();
                        __syncwarp();
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const uint32_t* w = k < 4 ? o0 + 8 * k : o1 + 8 * (k - 4);
                            uint4 q = make_uint4(0u, 0u, 0u, 0u);
                            if (k < 4 || has1)
                                q = make_uint4(ptx::pack_bf16x2(__uint_as_float(w[0]), __uint_as_float(w[1])),
                                               ptx::pack_bf16x2(__uint_as_float(w[2]), __uint_as_float(w[3])),
                                               ptx::pack_bf16x2(__uint_as_float(w[4]), __uint_as_float(w[5])),
                                               ptx::pack_bf16x2(__uint_as_float(w[6]), __uint_as_float(w[7])));
                            *reinterpret_cast<uint4*>(box + lane * 128 + ((k ^ (lane & 7)) << 4)) = q;
                        }
                        ptx::fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0 && rows_ok) {
                            ptx::tma_store_5d(mAcc16, box, 32 * cb, hh, gi, bb, g);
                            ptx::bulk_commit_group();
                        }
                        if ((f32m >> cb) & 1u) stage_box(o0, cb);
                        if (has1 && ((f32m >> (cb + 1)) & 1u)) stage_box(o1, cb + 1);
                        if (cb + 2 < n32) ptx::tmem_ld32(tl + 32 * (cb + 2), o0);
                    }
                } else
                for (int cb = 0; cb < n32; cb += 2) {
                    ptx::tmem_wait_ld();
                    read_out_a(cb);
                    if (cb + 1 < n32) ptx::tmem_ld32(tl + 32 * (cb + 1), o1);
                    stage_box(o0, cb);
                    if (cb + 1 < n32) {
                        ptx::tmem_wait_ld();
                        read_out_a(cb + 1);
                        if (cb + 2 < n32) ptx::tmem_ld32(tl + 32 * (cb + 2), o0);
                        stage_box(o1, cb + 1);
                    }
                }
            } else {
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive_cluster_relaxed(acc_empty_remote);
            }
            // accumulator read out: the next unit's first MMA2 may overwrite it
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster_relaxed(acc_empty_b_remote);
            if (warp == 11 && lane == 0) UTRACE(5, it);
        }
        if (lane == 0) ptx::bulk_wait_group_read<0>();  // staging read before the CTA exits
    } else {
        // ------------------------------------------------------------- elementwise
        const int sw = warp - 2;
        const int quad = warp & 3;
        const int half = sw >> 2;
        const int row = quad * 32 + lane;
        const uint32_t tl = tmem + (uint32_t(quad * 32) << 16);
        const uint32_t leader_rank = crank & 2u;
        const uint32_t x_free_remote = ptx::mapa(&bars->x_free, leader_rank);
        const uint32_t a_full_remote = ptx::mapa(&bars->a_full, leader_rank);
        const uint32_t peer_rank = crank + 2u;  // P pair -> dS pair partner
        int it = 0, t = 0;  // t: global tile index
        for (int u = cluster; u < nunits; u += nclusters, ++it) {
            const int bh = unit_bh(u), r0 = unit_r0(u);
            const int64_t vec_base = static_cast<int64_t>(bh) * (KV ? p.Lcol : p.Lrow);  // per-query vectors
            const int grow = r0 + row;  // global row (key in KV, query in Q)
            // Per-row vector (Q kernel): lse2 for the P pair, D for the dS pair.  lse2 = lse * log2(e)
            // is rounded on its own (__fmul_rn, never contracted into the ex2 argument) in both
            // kernels, so the two dQ paths see bitwise-equal P and dS (the contraction otherwise
            // follows register allocation: measured 2e-4 drift between the paths).
            float row_v = 0.f;
            if (!KV && grow < p.Lrow) row_v = role == 0 ? __fmul_rn(__ldg(p.lse + vec_base + grow), kL2E)
                                                     : __ldg(p.Dvec + vec_base + grow);
            for (int j = 0; j < ntiles; ++j, ++t) {
                const int c0 = p.col0 + j * BN + 32 * half;  // first tile column of this thread's half
                const int buf = t % NAB;
                uint8_t* abuf = sA + buf * (BM * 128);
                uint8_t* arow = abuf + row * 128;
                if (role == 1 && warp == 2 && lane == 0) ptx::mbar_expect_tx(&bars->pin_full[buf], BM * 128);
                // per-column vector (KV kernel)
                float cv[32];
                if (KV) {
                    if (role == 0) {
                        load_vec32(p.lse + vec_base, c0, p.Lcol, INFINITY, cv);
#pragma unroll
                        for (int k = 0; k < 32; ++k) cv[k] = __fmul_rn(cv[k], kL2E);
                    } else {
                        load_vec32(p.Dvec + vec_base, c0, p.Lcol, 0.f, cv);
                    }
                }
                ptx::mbar_wait(&bars->x_full, t & 1);
                if (lane == 0 && it == 0) BTRACE(3, j);
                if (warp == 2 && lane == 0 && j == 0) UTRACE(2, it);
                ptx::tc_fence_after();
                uint32_t xr[32];
                ptx::tmem_ld32(tl + kXCol + 32 * half, xr);
                ptx::tmem_wait_ld();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive_cluster_relaxed(x_free_remote);

                uint32_t pk[16];
                if (role == 0) {
                    // P = 2^(X - lse2), zero past the sequence end (padding rows of K/Q tiles)
#pragma unroll
                    for (int cc = 0; cc < 16; ++cc) {
                        float pv[2];
#pragma unroll
                        for (int uu = 0; uu < 2; ++uu) {
                            const int k = 2 * cc + uu;
                            const float x = __uint_as_float(xr[k]);
                            if (KV) {
                                pv[uu] = ptx::ex2(x - cv[k]);  // cv = +inf past L -> 0
                            } else {
                                pv[uu] = c0 + k < p.Lcol ? ptx::ex2(x - row_v) : 0.f;
                            }
                        }
                        pk[cc] = ptx::pack_bf16x2(pv[0], pv[1]);
                    }
                    if (lane == 0 && it == 0) BTRACE(4, j);
                    // Buffer `buf` held P_{t-NAB}: free once the local dV MMA of that tile (KV) and the
                    // dS pair's MMA of it (which implies the copy landed) are done; the latter also
                    // frees the dS pair's buffer `buf` for the copy of P_t.
                    if (t >= NAB) {
                        if (has_mma2) ptx::mbar_wait(&bars->mma2_done[buf], ((t / NAB) - 1) & 1);
                        ptx::mbar_wait_cluster(&bars->pin_free[buf], ((t / NAB) - 1) & 1);
                        ptx::tc_fence_after();
                    }
                    // Q kernel: dS_t comes back into this buffer once the dS pair has it (the copy of
                    // P_t out of it has completed by then)
                    if (!KV && has_mma2 && warp == 2 && lane == 0) ptx::mbar_expect_tx(&bars->dsin_full[buf], BM * 128);
                    if (lane == 0 && it == 0) BTRACE(5, j);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int chunk = 4 * half + k;
                        *reinterpret_cast<uint4*>(arow + ((chunk ^ (row & 7)) << 4)) =
                            make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
                    }
                    ptx::fence_proxy_async_smem();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (KV && has_mma2 && lane == 0) ptx::mbar_arrive_remote(a_full_remote);
                    // all 128 rows written -> one bulk copy of the 16 KB tile into the dS pair
                    named_bar_sync(1, 256);
                    if (warp == 2 && lane == 0) {
                        bulk_copy_s2cluster(ptx::mapa(abuf, peer_rank), abuf, BM * 128,
                                            ptx::mapa(&bars->pin_full[buf], peer_rank));
                        if (it == 0) BTRACE(7, j);
                    }
                } else {
                    if (KV && p.ds_store && t > 0 && warp == 2 && lane == 0) {
                        // dS_{t-1}'s store has read its buffer: release it to the P pair
                        ptx::bulk_wait_group_read<0>();
                        ptx::mbar_arrive_remote(ptx::mapa(&bars->pin_free[(t - 1) % NAB], crank - 2u));
                    }
                    ptx::mbar_wait_cluster(&bars->pin_full[buf], (t / NAB) & 1);
                    if (lane == 0 && it == 0) BTRACE(9, j);
                    uint4 pin[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int chunk = 4 * half + k;
                        pin[k] = *reinterpret_cast<const uint4*>(arow + ((chunk ^ (row & 7)) << 4));
                    }
                    const uint32_t* pw = reinterpret_cast<const uint32_t*>(pin);
#pragma unroll
                    for (int cc = 0; cc < 16; ++cc) {
                        const float d0 = KV ? cv[2 * cc] : row_v;
                        const float d1 = KV ? cv[2 * cc + 1] : row_v;
                        const float s0 = bf_lo(pw[cc]) * (__uint_as_float(xr[2 * cc]) - d0);
                        const float s1 = bf_hi(pw[cc]) * (__uint_as_float(xr[2 * cc + 1]) - d1);
                        pk[cc] = ptx::pack_bf16x2(s0, s1);
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int chunk = 4 * half + k;
                        *reinterpret_cast<uint4*>(arow + ((chunk ^ (row & 7)) << 4)) =
                            make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
                    }
                    ptx::fence_proxy_async_smem();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive_remote(a_full_remote);
                    if (lane == 0 && it == 0) BTRACE(10, j);
                    if (KV && p.ds_store) {
                        // the whole 128-key x 64-query dS tile (already in the 128-byte-swizzled
                        // K-major layout of the TMA box) -> dS[bh][key][query] for the dQ GEMM
                        named_bar_sync(1, 256);
                        if (warp == 2 && lane == 0) {
                            ptx::tma_store_3d(&mapDS, abuf, j * BN, r0, bh);
                            ptx::bulk_commit_group();
                        }
                    }
                    if (!KV && p.role[0].n2 > 0) {
                        // Q kernel: the P pair accumulates the other half of dQ from the same dS tile
                        named_bar_sync(1, 256);
                        if (warp == 2 && lane == 0)
                            bulk_copy_s2cluster(ptx::mapa(abuf, crank - 2u), abuf, BM * 128,
                                                ptx::mapa(&bars->dsin_full[buf], crank - 2u));
                    }
                }
            }

        }
        if (KV && p.ds_store && role == 1 && warp == 2 && lane == 0) {
            ptx::bulk_wait_group_read<0>();  // last dS store done reading before the CTA exits
            if (t > 0) ptx::mbar_arrive_remote(ptx::mapa(&bars->pin_free[(t - 1) % NAB], crank - 2u));
        }
    }

    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 1) ptx::tmem_dealloc_2sm(tmem, 512);
    if (warp == 0 && lane == 0) span_mark(2);
}

RoleDims make_role(int k1, int n2) {
    RoleDims r{};
    r.k1 = k1;
    r.nb1 = (k1 + 63) / 64;
    r.n2 = n2;
    r.n2a = std::min(n2, 256);
    r.n2b = n2 - r.n2a;
    r.nba = (r.n2a / 2 + 63) / 64;
    r.nbb = (r.n2b / 2 + 63) / 64;
    return r;
}

// Ring plan: the stationary tile (128 rows x all column blocks) and the two P/dS buffers are
// fixed; whole 32-row B1 tile halves (1 or 2 stages) and B2 slices of 16 or 32 rows
// (compile-time depth) share the rest.  Whole-tile B1 stages measured faster than column-block
// groups (dK/dV 0.406 vs 0.439 ms at B=8 L=1024, same-box A/B).
void finish_params(BwdParams& p, bool kv, const int* ring = nullptr) {
    int nb1 = std::max(p.role[0].nb1, p.role[1].nb1);
    int nb2 = std::max(p.role[0].nba + p.role[0].nbb, p.role[1].nba + p.role[1].nbb);
    p.stat_bytes = nb1 * BM * 128;
    p.kb1 = nb1;
    p.b1_stage = nb1 * 32 * 128;
    int forced[5] = {0, 0, 0, 0, 0};  // AttnBwdArgs::ring (Tuning::bwd_ring): tuning experiments
    if (ring != nullptr)
        for (int i = 0; i < 5; ++i) forced[i] = ring[i];
    // (B1 stages, B2 stages, exchange buffers, kb1, B2 slice rows), preferred first.  Measured
    // (B=8 L=1024, same box, tools/bwd_ab.py): dK/dV kernel (3,2,2,4,32) 0.369 ms vs (2,3,2,4,32)
    // 0.373 vs (4,2,2,3,32) 0.378 vs (1,3,2,0,32) 0.385 vs (1,6,2,0,16) 0.395 vs (6,2,2,2,32) 0.400;
    // dQ kernel (1,2,3,0,32) 0.336 vs (1,4,3,0,16) 0.349 vs (2,6,2,0,16) 0.358.  The trace
    // (tools/attn_bwd_trace.cu) shows the critical loop MMA1(j) -> B1(j+1) TMA (~1.4k cycles under
    // load) -> MMA1(j+1): B1 in 4-block groups over 3 stages lets the next tile's first group land
    // while MMA1(j) runs.  (kb1 = 0: whole-tile B1 stages)
    const int plans_kv[][5] = {{3, 2, 2, 4, 32}, {2, 2, 2, 4, 32}, {1, 3, 2, 0, 32}, {2, 6, 2, 0, 16}, {1, 6, 2, 0, 16}, {2, 3, 2, 0, 16},
                               {2, 2, 2, 0, 16}, {1, 4, 3, 0, 16}, {1, 6, 3, 0, 16}, {3, 4, 2, 4, 16},
                               {1, 2, 3, 0, 32}, {2, 3, 2, 0, 32}, {2, 2, 2, 0, 32}, {3, 2, 2, 4, 32},
                               {2, 3, 2, 4, 32}, {4, 2, 2, 3, 32}, {6, 2, 2, 2, 32}, {4, 4, 2, 3, 16}};
    const int plans_q[][5] = {{1, 2, 3, 0, 32}, {1, 4, 3, 0, 16}, {2, 6, 2, 0, 16}, {1, 6, 2, 0, 16},
                              {2, 3, 2, 0, 16}, {2, 2, 2, 0, 16}, {1, 6, 3, 0, 16}, {3, 4, 2, 4, 16},
                              {1, 3, 2, 0, 32}, {2, 3, 2, 0, 32}, {2, 2, 2, 0, 32}, {3, 2, 2, 4, 32},
                              {2, 3, 2, 4, 32}, {4, 2, 2, 3, 32}, {6, 2, 2, 2, 32}, {4, 4, 2, 3, 16}};
    const int(*plans)[5] = kv ? plans_kv : plans_q;
    const int nplans = kv ? int(sizeof(plans_kv) / sizeof(plans_kv[0])) : int(sizeof(plans_q) / sizeof(plans_q[0]));
    for (int pass = 0; pass < 2; ++pass) {
        for (int pi = 0; pi < nplans; ++pi) {
            const int* pl = plans[pi];
            if (pass == 0 && forced[0] > 0 &&
                (pl[0] != forced[0] || pl[1] != forced[1] || pl[2] != forced[2] || pl[3] != forced[3] ||
                 (forced[4] > 0 && pl[4] != forced[4])))
                continue;
            if (pass == 0 && forced[0] == 0) break;
            p.nst1 = pl[0];
            p.nst2 = pl[1];
            p.nab = pl[2];
            p.kb1 = pl[3] ? pl[3] : nb1;
            p.slice = pl[4];
            p.b1_stage = p.kb1 * 32 * 128;
            p.b2_stage = std::max(nb2, 1) * p.slice * 128;
            if (smem_layout(p).total + 1024 <= 232448) return;
        }
    }
    throw std::invalid_argument("attention backward: no ring plan fits shared memory");
}

// 4-CTA clusters of one kernel that fit on the device at once (the persistent grid size), cached
// per (device, kernel, shared memory).  The occupancy query can report 0 for compile-time cluster
// dims on some drivers: then 7/8 of SMs / 4 (B200: 33 of 37 4-SM groups fit, the GPCs' odd SMs left
// over) -- an over-estimate would leave whole clusters waiting for a second round.
int resident_clusters(const void* kern, int smem) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, int>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(dev, kern, smem);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int n = 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(4 * 1024, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = static_cast<size_t>(smem);
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
        cudaGetLastError();
        n = std::max(1, device_sm_count() * 7 / 32);
    }
    cache[key] = n;
    return n;
}

template <bool KV, int NS1, int NST2, int NAB, int KB1 = 0, int SL = 16>
void launch_depth(const LayerDims& d, const AttnBwdArgs& a, const BwdParams& p, const CUtensorMap* maps,
                  cudaStream_t stream) {
    const Layout lay = smem_layout(p);
    const int smem = lay.total + 1024;
    if (smem > 232448) throw std::invalid_argument("attention backward: shared memory budget exceeded");
    auto kern = attn_bwd_kernel<KV, NS1, NST2, NAB, KB1, SL>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int units = p.BH * ((p.Lrow + 255) / 256);
    const int clusters = std::min(units, resident_clusters(reinterpret_cast<const void*>(kern), smem));
    dim3 grid(static_cast<unsigned>(clusters * 4), 1u);
    launch_pdl(kern, grid, dim3(kThreads), size_t(smem), stream, maps[0], maps[1], maps[2], maps[3], maps[4], maps[5],
               maps[6], maps[7], maps[8], maps[9], maps[10], p);
}

template <bool KV>
void launch(const LayerDims& d, const AttnBwdArgs& a, const BwdParams& p, const CUtensorMap* maps,
            cudaStream_t stream) {
    if (p.slice == 32) {
        if (p.kb1 == 4 && p.nst1 == 3) launch_depth<KV, 3, 2, 2, 4, 32>(d, a, p, maps, stream);
        else if (p.kb1 == 3 && p.nst1 == 4) launch_depth<KV, 4, 2, 2, 3, 32>(d, a, p, maps, stream);
        else if (p.kb1 == 2 && p.nst1 == 6) launch_depth<KV, 6, 2, 2, 2, 32>(d, a, p, maps, stream);
        else if (p.kb1 == 4 && p.nst1 == 2 && p.nst2 == 2) launch_depth<KV, 2, 2, 2, 4, 32>(d, a, p, maps, stream);
        else if (p.kb1 == 4 && p.nst1 == 2) launch_depth<KV, 2, 3, 2, 4, 32>(d, a, p, maps, stream);
        else if (p.nab == 3) launch_depth<KV, 1, 2, 3, 0, 32>(d, a, p, maps, stream);
        else if (p.nst1 == 2 && p.nst2 == 3) launch_depth<KV, 2, 3, 2, 0, 32>(d, a, p, maps, stream);
        else if (p.nst1 == 2) launch_depth<KV, 2, 2, 2, 0, 32>(d, a, p, maps, stream);
        else launch_depth<KV, 1, 3, 2, 0, 32>(d, a, p, maps, stream);
    } else if (p.kb1 == 4 && p.nst1 == 3) {
        launch_depth<KV, 3, 4, 2, 4>(d, a, p, maps, stream);
    } else if (p.kb1 == 3 && p.nst1 == 4) {
        launch_depth<KV, 4, 4, 2, 3>(d, a, p, maps, stream);
    } else if (p.nab == 3) {
        if (p.nst2 == 4) launch_depth<KV, 1, 4, 3>(d, a, p, maps, stream);
        else launch_depth<KV, 1, 6, 3>(d, a, p, maps, stream);
    } else if (p.nst1 == 1) {
        launch_depth<KV, 1, 6, 2>(d, a, p, maps, stream);
    } else if (p.nst2 == 6) {
        launch_depth<KV, 2, 6, 2>(d, a, p, maps, stream);
    } else if (p.nst2 == 3) {
        launch_depth<KV, 2, 3, 2>(d, a, p, maps, stream);
    } else {
        launch_depth<KV, 2, 2, 2>(d, a, p, maps, stream);
    }
}

}  // namespace

bool attn_bwd_supported(const LayerDims& d) {
    if (d.dqk_mma > 448 || d.dv_mma > 448 || d.dqk_pad % 64 || d.dv_pad % 64) return false;
    BwdParams p{};
    p.role[0] = make_role(d.dqk_mma, d.dv_mma);
    p.role[1] = make_role(d.dv_mma, d.dqk_mma);
    try {
        finish_params(p, true);
    } catch (const std::invalid_argument&) {
        return false;
    }
    return smem_layout(p).total + 1024 <= 232448;
}

// Accumulator output map for one role: rank-major [G][B][chunk][H][acc_ld] fp32 from column col0,
// n2 columns wide (clipped), boxes of 32 columns x 32 rows.
CUtensorMap acc_map(float* out, int col0, int n2, int H, int chunk, int B, int G, int acc_ld) {
    const uint64_t row = uint64_t(acc_ld) * 4;
    const uint64_t dims[5] = {uint64_t(n2), uint64_t(H), uint64_t(chunk), uint64_t(B), uint64_t(G)};
    const uint64_t strides[4] = {row, row * H, row * H * chunk, row * H * chunk * B};
    const uint32_t box[5] = {32, 1, 32, 1, 1};
    return make_map_5d_f32_strided(out + col0, dims, strides, box);
}

// bf16 copy of the same accumulator: boxes of 64 columns x 32 rows.
CUtensorMap acc_map16(__nv_bfloat16* out, int n2, int H, int chunk, int B, int G, int acc_ld) {
    const uint64_t row = uint64_t(acc_ld) * 2;
    const uint64_t dims[5] = {uint64_t(n2), uint64_t(H), uint64_t(chunk), uint64_t(B), uint64_t(G)};
    const uint64_t strides[4] = {row, row * H, row * H * chunk, row * H * chunk * B};
    const uint32_t box[5] = {64, 1, 32, 1, 1};
    return make_map_5d_bf16_strided(out, dims, strides, box);
}

// 32-column chunks of [0, n) that intersect columns [lo, hi)
uint32_t chunk_mask(int lo, int hi, int n) {
    uint32_t m = 0;
    for (int k = 0; 32 * k < n && k < 32; ++k)
        if (32 * k < hi && 32 * k + 32 > lo) m |= 1u << k;
    return m;
}

void launch_attn_bwd(const LayerDims& d, const AttnBwdArgs& a, cudaStream_t stream, int which) {
    if (!attn_bwd_supported(d)) throw std::invalid_argument("tcgen05 attention backward: unsupported widths");
    const uint64_t BH = static_cast<uint64_t>(a.B) * d.heads;
    const int nqk = (d.dqk_mma + 63) / 64, nv = (d.dv_mma + 63) / 64;
    auto ld_of = [&](const void* x) { return (x == a.vhat || x == a.dohat) ? d.dv_pad : d.dqk_pad; };
    // every operand through the sharded (rank-major) maps; local operands are one shard of L rows
    const int Lk = a.Lk > 0 ? a.Lk : a.L, kc = a.kchunk > 0 ? a.kchunk : Lk;
    const int G = (Lk + kc - 1) / kc;
    if (G * kc != Lk || (G > 1 && kc % 256 != 0))
        throw std::invalid_argument("attention backward: key shards must be equal and a multiple of 256 rows");
    auto is_key = [&](const void* x) { return x == a.khat || x == a.vhat; };
    auto chunk_of = [&](const void* x) { return is_key(x) ? kc : a.L; };
    auto sharded = [&](const void* x) { return is_key(x) && G > 1; };
    auto stat = [&](const void* x, int nb) {
        return sharded(x) ? make_map_blocks_bf16_sharded(x, kc, BH, G, ld_of(x), BM, nb)
                          : make_map_blocks_bf16(x, chunk_of(x), BH, ld_of(x), BM, nb);
    };
    auto tile = [&](const void* x, int kb) {
        return sharded(x) ? make_map_blocks_bf16_sharded(x, kc, BH, G, ld_of(x), 32, kb)
                          : make_map_blocks_bf16(x, chunk_of(x), BH, ld_of(x), 32, kb);
    };
    auto slice = [&](const void* x, int sl) {
        return sharded(x) ? make_map_4d_bf16_sharded(x, ld_of(x), kc, BH, G, 64, sl)
                          : make_map_3d_bf16(x, ld_of(x), chunk_of(x), BH, ld_of(x), 64, sl);
    };
    if (which & 1) {  // KV kernel: P pair K_hat/Q_hat/dO_hat -> dV ; dS pair V_hat/dO_hat/Q_hat -> dK
        BwdParams p{};
        p.Lrow = Lk;  // rows = keys (all shards)
        p.Lcol = a.L; // tile columns = local queries (this launch: [q0, q0 + qn))
        p.col0 = a.q0;
        p.ncol = a.qn > 0 ? a.qn : a.L - a.q0;
        p.acc_add = a.acc_add;
        if (p.col0 < 0 || p.col0 + p.ncol > a.L || (a.qn > 0 && a.q0 % BN != 0))
            throw std::invalid_argument("attention backward: query chunk out of range or not 64-aligned");
        p.stat_chunk = kc;
        p.col_chunk = a.L;
        p.stat_sharded = G > 1;
        p.col_sharded = 0;
        p.H = d.heads;
        p.B = a.B;
        p.BH = a.B * d.heads;
        p.role[0] = make_role(d.dqk_mma, d.dv_mma);
        p.role[1] = make_role(d.dv_mma, d.dqk_mma);
        finish_params(p, true, a.ring);
        p.lse = a.lse;
        p.Dvec = a.Dvec;
        p.acc_out[0] = a.dv_acc;
        p.acc_out[1] = a.dk_acc;
        p.acc_ld = a.acc_ld;
        p.ds_store = a.ds != nullptr ? 1 : 0;
        // bf16 accumulators (unsharded, whole-query launches): fp32 kept for the chunks holding the
        // point / translation columns -- dV: [c + r d_z, dv_used), dK: [c, zq)
        p.acc16 = a.dk16 != nullptr && a.dv16 != nullptr && !p.acc_add && G == 1 && a.acc_ld % 8 == 0;
        p.f32_chunks[0] = p.acc16 ? chunk_mask(d.c + d.rank * d.d_z, d.dv_used, p.role[0].n2) : 0xFFFFFFFFu;
        p.f32_chunks[1] = p.acc16 ? chunk_mask(d.c, d.zq, p.role[1].n2) : 0xFFFFFFFFu;
        if (p.ds_store && (G > 1 || a.ds_ld % 8 != 0 || a.ds_ld < p.ncol))
            throw std::invalid_argument("attention backward: materialised dS needs unsharded keys, ds_ld >= chunk, % 8");
        if (p.acc_add && G > 1) throw std::invalid_argument("attention backward: chunked accumulation is unsharded only");
        const CUtensorMap m0 = stat(a.khat, nqk);
        const CUtensorMap maps[11] = {
            m0, tile(a.qhat, p.kb1), slice(a.dohat, p.slice), stat(a.vhat, nv), tile(a.dohat, p.kb1),
            slice(a.qhat, p.slice), p.ds_store ? make_map_3d_bf16(a.ds, p.ncol, a.L, BH, a.ds_ld, 64, BM) : m0,
            a.dv_acc ? acc_map(a.dv_acc, 0, p.role[0].n2, d.heads, kc, a.B, G, a.acc_ld) : m0,
            a.dk_acc ? acc_map(a.dk_acc, 0, p.role[1].n2, d.heads, kc, a.B, G, a.acc_ld) : m0,
            p.acc16 ? acc_map16(a.dv16, p.role[0].n2, d.heads, kc, a.B, G, a.acc_ld) : m0,
            p.acc16 ? acc_map16(a.dk16, p.role[1].n2, d.heads, kc, a.B, G, a.acc_ld) : m0};
        launch<true>(d, a, p, maps, stream);
    }
    if ((which & 2) && a.ds != nullptr) {
        // dQ from the materialised dS: per (sample, head) dQ_acc[q, :] = sum_key dS[key, q] K_hat[key, :],
        // one batched tcgen05 GEMM (both operands MN-major) straight into the residue-major
        // [B, L, H, acc_ld] accumulator -- no second pass over S, dP and the softmax
        GemmArgs g{};
        const int qn = a.qn > 0 ? a.qn : a.L - a.q0;
        g.A = a.ds;
        g.lda = a.ds_ld;
        g.a_mn_major = true;
        g.B = a.khat;
        g.ldb = d.dqk_pad;
        g.b_mn_major = true;
        g.C = a.dq_acc + int64_t(a.q0) * d.heads * a.acc_ld;  // this chunk's query rows
        g.ldc = int64_t(d.heads) * a.acc_ld;
        g.ldc_h = a.acc_ld;
        g.ldc_b = int64_t(a.L) * d.heads * a.acc_ld;
        g.M = qn;
        g.N = d.dqk_mma;
        g.K = a.L;
        g.batch = static_cast<int>(BH);
        g.batch_h = d.heads;
        if (a.dq16 != nullptr) {  // bf16 copy for the unpack; fp32 only for the point / translation chunks
            g.C16 = a.dq16 + int64_t(a.q0) * d.heads * a.acc_ld;
            g.c16_f32_chunks = chunk_mask(d.c, d.zq, d.dqk_mma);
        }
        launch_gemm_bf16(g, stream);
        which &= ~2;
    }
    if (which & 2) {  // Q kernel: P pair Q_hat/K_hat ; dS pair dO_hat/V_hat/K_hat -> dQ
        // dQ = dS.K_hat split over both pairs by columns: the P pair receives dS back from the
        // dS pair and accumulates columns [0, nq0), the dS pair [nq0, dqk): one S (or dP) GEMM and
        // half a dQ GEMM per pair and tile, instead of the P pair idling through the dS pair's two.
        const int nq0 = (d.dqk_mma / 2 + 15) / 16 * 16;
        BwdParams p{};
        p.Lrow = a.L;  // rows = local queries
        p.Lcol = Lk;   // tile columns = keys (all shards)
        p.col0 = 0;
        p.ncol = Lk;
        p.stat_chunk = a.L;
        p.col_chunk = kc;
        p.stat_sharded = 0;
        p.col_sharded = G > 1;
        p.H = d.heads;
        p.B = a.B;
        p.BH = a.B * d.heads;
        p.role[0] = make_role(d.dqk_mma, nq0);
        p.role[1] = make_role(d.dv_mma, d.dqk_mma - nq0);
        finish_params(p, false, a.ring);
        p.lse = a.lse;
        p.Dvec = a.Dvec;
        p.acc_out[0] = a.dq_acc;
        p.acc_out[1] = a.dq_acc;
        p.acc_col0[0] = 0;
        p.acc_col0[1] = nq0;
        p.b2_col0[0] = 0;
        p.b2_col0[1] = nq0;
        p.acc_ld = a.acc_ld;
        const CUtensorMap q0map = stat(a.qhat, nqk);
        const CUtensorMap maps[11] = {q0map, tile(a.khat, p.kb1), slice(a.khat, p.slice),
                                      stat(a.dohat, nv), tile(a.vhat, p.kb1),  slice(a.khat, p.slice), q0map,
                                      acc_map(a.dq_acc, 0, nq0, d.heads, a.L, a.B, 1, a.acc_ld),
                                      acc_map(a.dq_acc, nq0, d.dqk_mma - nq0, d.heads, a.L, a.B, 1, a.acc_ld), q0map,
                                      q0map};
        launch<false>(d, a, p, maps, stream);
    }
}

}  // namespace fipa_b200
