// Fused projection + frame application + lifted-row packing (K1 + K2, bf16 path).
//
// Replaces   project_inputs  proj/src/ipa.cpp:201-217 (six bias-free linears)
//            lift_qkv        proj/src/flash_ipa.cpp:23-139 (+ bias_factors, pair_features.cpp:141-163)
// One CTA = 128 residues x one head.  The head's 468 projection columns
// (q | k | v | q_p | k_p | v_p, head-major weight copy padded to NH = 480) are one tcgen05 GEMM
// (M=128, N=256+224, K=d_in) into TMEM, fed by a 2-stage TMA ring.  The epilogue warps (thread =
// residue) apply the residue's frame and build the q_hat / k_hat / v_hat rows of pack.cu's layout
// directly from TMEM, one tensor at a time, into a 128-byte-swizzled shared-memory tile that
// leaves by TMA tensor stores.  The fp32 [B*L, 3744] projection round trip of the unfused path
// (write + read ~250 MB at B=8, L=1024) disappears; only the point columns (needed by the
// backward) are written to the projection buffer.
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
constexpr int BK = 64;
constexpr int kThreads = 320;  // w0 TMA, w1 TMEM + MMA, w2..w9 epilogue (two warps per TMEM quadrant)
constexpr int kStages = 2;
constexpr int kMaxQ = 8;       // points held in registers by the epilogue
constexpr int kMaxV = 12;
constexpr float kL2E = 1.4426950408889634f;
constexpr float kMaskedBias = -1.0e30f;

struct PPParams {
    int M, L, H, c, Nq, Nv, dz, rdz, NH, N1, N2, nk;
    int dqk_used, dqk_pad, dv_used, dv_pad, zq, n_proj, chunk_ok;
    int write_points;  // training: raw point columns into proj for the backward
    const float* z1;
    const float* z2;
    const __nv_bfloat16* z1q;  // bf16(log2(e) z1): q_hat pair block, copied
    const __nv_bfloat16* z2b;  // bf16(z2): v_hat pair block copied, k_hat's scaled per head
    const float* rot;
    const float* trans;  // recentred
    const uint8_t* mask;
    const float* head_g;
    const float* wl_bias;
    float k_scale;
    float* proj;     // [M, n_proj]: point columns written (backward)
    float* colbias;  // [B*H, L]
    __nv_bfloat16* qhat;
    __nv_bfloat16* khat;
    __nv_bfloat16* vhat;
};

// Optional timestamps of CTA (0, 0) for pipeline analysis (tools/proj_pack_trace.cu).
#ifdef FIPA_PP_TRACE
__device__ long long g_pp_trace[10 * 16];  // [warp][event]
#define PPTRACE(ev)                                                                                   \
    do {                                                                                              \
        if (blockIdx.x == 0 && blockIdx.y == 0 && (threadIdx.x & 31) == 0)                           \
            g_pp_trace[(threadIdx.x >> 5) * 16 + (ev)] = clock64();                                   \
    } while (0)
#else
#define PPTRACE(ev) \
    do {            \
    } while (0)
#endif

__device__ __forceinline__ float bf_hi(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
__device__ __forceinline__ float bf_lo(float x) { return x - __bfloat162float(__float2bfloat16_rn(x)); }

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
                 ::"l"(reinterpret_cast<uint64_t>(map)), "r"(ptx::smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
// 16-byte asynchronous global -> shared copy (L2 only) and its completion wait
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ptx::smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// One element of the 128 x W bf16 staging tile: [W/64 blocks][128 rows][128 B], 16-byte chunk
// index XOR (row % 8) -- the TMA SWIZZLE_128B layout.
__device__ __forceinline__ void stage_put(uint8_t* tile, int row, int col, float v) {
    uint8_t* p = tile + (col >> 6) * (BM * 128) + row * 128 + ((((col & 63) >> 3) ^ (row & 7)) << 4) + ((col & 7) << 1);
    *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(v);
}
// 8 consecutive columns (col % 8 == 0) as one 16-byte store
__device__ __forceinline__ void stage_put8(uint8_t* tile, int row, int col, const float* v) {
    uint8_t* p = tile + (col >> 6) * (BM * 128) + row * 128 + ((((col & 63) >> 3) ^ (row & 7)) << 4);
    uint4 w;
    w.x = ptx::pack_bf16x2(v[0], v[1]);
    w.y = ptx::pack_bf16x2(v[2], v[3]);
    w.z = ptx::pack_bf16x2(v[4], v[5]);
    w.w = ptx::pack_bf16x2(v[6], v[7]);
    *reinterpret_cast<uint4*>(p) = w;
}

// Frame-apply up to MAXP points held in TMEM registers u[32] | w[16] (x, y, z interleaved); every
// index is a compile-time constant so the arrays stay in registers.
template <int MAXP>
__device__ __forceinline__ void rotate_points(const uint32_t* u, const uint32_t* w, int n, const float* R, float* out) {
#pragma unroll
    for (int q = 0; q < MAXP; ++q) {
        if (q < n) {
            const float x = __uint_as_float(3 * q < 32 ? u[3 * q] : w[3 * q - 32]);
            const float y = __uint_as_float(3 * q + 1 < 32 ? u[3 * q + 1] : w[3 * q + 1 - 32]);
            const float z = __uint_as_float(3 * q + 2 < 32 ? u[3 * q + 2] : w[3 * q + 2 - 32]);
            out[3 * q] = fmaf(R[0], x, fmaf(R[1], y, R[2] * z));
            out[3 * q + 1] = fmaf(R[3], x, fmaf(R[4], y, R[5] * z));
            out[3 * q + 2] = fmaf(R[6], x, fmaf(R[7], y, R[8] * z));
        }
    }
}
// Raw point columns (training only) into the projection row: float4 stores where aligned.
__device__ __forceinline__ void store_points(float* dst, const uint32_t* u, const uint32_t* w, int n) {
    if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0 && (n & 3) == 0) {
#pragma unroll
        for (int e4 = 0; e4 < 12; ++e4) {
            if (4 * e4 < n) {
                float4 f;
                f.x = __uint_as_float(4 * e4 < 32 ? u[4 * e4] : w[4 * e4 - 32]);
                f.y = __uint_as_float(4 * e4 + 1 < 32 ? u[4 * e4 + 1] : w[4 * e4 + 1 - 32]);
                f.z = __uint_as_float(4 * e4 + 2 < 32 ? u[4 * e4 + 2] : w[4 * e4 + 2 - 32]);
                f.w = __uint_as_float(4 * e4 + 3 < 32 ? u[4 * e4 + 3] : w[4 * e4 + 3 - 32]);
                reinterpret_cast<float4*>(dst)[e4] = f;
            }
        }
    } else {
#pragma unroll
        for (int e = 0; e < 48; ++e)
            if (e < n) dst[e] = __uint_as_float(e < 32 ? u[e] : w[e - 32]);
    }
}

__global__ void __launch_bounds__(kThreads, 1)
    proj_pack_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                     const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
                     const __grid_constant__ CUtensorMap mapV, PPParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int a_bytes = BM * BK * 2, b_bytes = p.NH * BK * 2, stage_bytes = a_bytes + b_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kStages;
    uint64_t* done = empty + kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    uint64_t* tile_ready = done + 2;  // [2] staging tile complete (one arrive per epilogue warp)
    uint64_t* tile_free = done + 4;   // tile 0 read by tensor 0's stores (tensor 2 may overwrite it)
    uint8_t* ring = smem + 1024;
    // two output staging tiles (alternating tensors) reuse the ring once the MMAs are done
    uint8_t* tiles = ring;
    const int tile_bytes = BM * (p.dqk_pad > p.dv_pad ? p.dqk_pad : p.dv_pad) * 2;

    const int warp = ptx::warp_id(), lane = ptx::lane_id();
    const int m0 = blockIdx.x * BM, h = blockIdx.y;
    if (warp == 0 && lane == 0) {
        span_mark(0);
        ptx::tma_prefetch(&mapA);
        ptx::tma_prefetch(&mapB);
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_init(done, 1);
        ptx::mbar_init(&tile_ready[0], 8);
        ptx::mbar_init(&tile_ready[1], 8);
        ptx::mbar_init(tile_free, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(tmem_slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    ptx::pdl_wait();  // inputs (s_bf16, pair blocks, frames) written by the preceding kernels
    ptx::pdl_trigger();

    if (warp == 0) {
        PPTRACE(0);
        if (lane == 0) {
            for (int kb = 0; kb < p.nk; ++kb) {
                const int s = kb % kStages;
                if (kb >= kStages) ptx::mbar_wait(&empty[s], ((kb / kStages) - 1) & 1);
                uint8_t* sa = ring + s * stage_bytes;
                ptx::mbar_expect_tx(&full[s], stage_bytes);
                ptx::tma_load_2d(sa, &mapA, &full[s], kb * BK, m0);
                ptx::tma_load_2d(sa + a_bytes, &mapB, &full[s], kb * BK, h * p.NH);
                ptx::tma_load_2d(sa + a_bytes + (p.NH / 2) * 128, &mapB, &full[s], kb * BK, h * p.NH + p.NH / 2);
            }
            if (p.chunk_ok) {
                // output stores: this otherwise idle thread issues every tile's TMA stores, so the
                // epilogue warps go on building the next tensor while the previous one drains
                // (issuing from the epilogue warps stalled them ~5k cycles per tensor on the
                // store queue)
                // tensor order q (tile 0), v (tile 1), k (tile 0 again: its pair block is v's, scaled)
                for (int tsel = 0; tsel < 3; ++tsel) {
                    const int tb = tsel & 1, T = tsel == 0 ? 0 : tsel == 1 ? 2 : 1;
                    ptx::mbar_wait(&tile_ready[tb], (tsel >> 1) & 1);
                    const uint8_t* tile = tiles + tb * tile_bytes;
                    const int width = T < 2 ? p.dqk_pad : p.dv_pad;
                    const CUtensorMap* map = T == 0 ? &mapQ : T == 1 ? &mapK : &mapV;
                    // 32-row chunks never straddle two samples (L % 32 == 0)
                    for (int ch = 0; ch < BM / 32; ++ch) {
                        const int rr = m0 + ch * 32;
                        if (rr >= p.M) break;
                        const int cb_ = rr / p.L, ci = rr - cb_ * p.L;
                        for (int blk = 0; blk < width / 64; ++blk)
                            tma_store_3d(map, tile + blk * (BM * 128) + ch * 32 * 128, blk * 64, ci, cb_ * p.H + h);
                    }
                    bulk_commit();
                    if (tsel == 0) {
                        bulk_wait_read0();  // tile 0 read by the q stores: free for k
                        ptx::mbar_arrive(tile_free);
                    }
                }
                bulk_wait_read0();  // staging read before the CTA exits
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t id1 = ptx::idesc_bf16(BM, p.N1, false, false);
            const uint32_t id2 = ptx::idesc_bf16(BM, p.N2 > 0 ? p.N2 : 16, false, false);
            for (int kb = 0; kb < p.nk; ++kb) {
                const int s = kb % kStages;
                ptx::mbar_wait(&full[s], (kb / kStages) & 1);
                ptx::tc_fence_after();
                const uint32_t sa = ptx::smem_u32(ring + s * stage_bytes);
                const uint32_t sb = sa + a_bytes;
#pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk) {
                    const uint64_t da = ptx::sw128_desc(sa + kk * 32, 16, 1024);
                    ptx::mma_ss(tmem, da, ptx::sw128_desc(sb + kk * 32, 16, 1024), id1, (kb | kk) != 0);
                    if (p.N2 > 0)
                        ptx::mma_ss(tmem + p.N1, da, ptx::sw128_desc(sb + p.N1 * 128 + kk * 32, 16, 1024), id2,
                                    (kb | kk) != 0);
                }
                ptx::mma_commit(&empty[s]);
            }
            ptx::mma_commit(done);
        }
        PPTRACE(1);
    } else {
        // ---------------------------------------------------------------- epilogue
        const int quad = warp & 3;
        const int half = (warp - 2) >> 2;  // 0: scalar channels, 1: geometry columns (phase A)
        const int r = quad * 32 + lane;  // row of the tile = TMEM lane
        const uint32_t tl = tmem + (uint32_t(quad * 32) << 16);
        const int row = m0 + r;
        const bool ok = row < p.M;
        const int rowc = ok ? row : p.M - 1;
        const int b = rowc / p.L, i = rowc - b * p.L;
        const int c = p.c, Nq = p.Nq, Nv = p.Nv, rdz = p.rdz;
        const int cq = 0, ck = c, cv = 2 * c, cqp = 3 * c, ckp = cqp + 3 * Nq, cvp = ckp + 3 * Nq;  // TMEM columns
        float R[9], t[3];
#pragma unroll
        for (int k = 0; k < 9; ++k) R[k] = __ldg(p.rot + int64_t(rowc) * 9 + k);
#pragma unroll
        for (int k = 0; k < 3; ++k) t[k] = __ldg(p.trans + int64_t(rowc) * 3 + k);
        const bool valid = p.mask == nullptr || p.mask[rowc] != 0;
        const float g = p.head_g[h];
        {  // warm L2 with this row's bf16 pair factors (phase B copies them) while the GEMM runs
            const char* z1r = reinterpret_cast<const char*>(p.z1q + int64_t(rowc) * rdz);
            const char* z2r = reinterpret_cast<const char*>(p.z2b + int64_t(rowc) * rdz);
            for (int o = 128 * half; o < rdz * 2; o += 256) {
                asm volatile("prefetch.global.L2 [%0];" ::"l"(z1r + o));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(z2r + o));
            }
        }
        PPTRACE(0);
        ptx::mbar_wait(done, 0);
        ptx::tc_fence_after();
        PPTRACE(1);
        if (warp == 2 && lane == 0) span_mark(1);

        // points: frame-rotated (geometry half only); the raw copies into proj (training) go out
        // after the three tensors
        float rq[3 * kMaxQ], rk[3 * kMaxQ], rv[3 * kMaxV];
        if (half == 1) {
            uint32_t u[32], w[16];
            ptx::tmem_ld32(tl + cqp, u);
            ptx::tmem_ld16(tl + cqp + 32, w);
            ptx::tmem_wait_ld();
            rotate_points<kMaxQ>(u, w, Nq, R, rq);
            ptx::tmem_ld32(tl + ckp, u);
            ptx::tmem_ld16(tl + ckp + 32, w);
            ptx::tmem_wait_ld();
            rotate_points<kMaxQ>(u, w, Nq, R, rk);
            ptx::tmem_ld32(tl + cvp, u);
            ptx::tmem_ld16(tl + cvp + 32, w);
            ptx::tmem_wait_ld();
            rotate_points<kMaxV>(u, w, Nv, R, rv);
        }
        float qb[3] = {0.f, 0.f, 0.f}, W[3] = {0.f, 0.f, 0.f}, kn = 0.f;
#pragma unroll
        for (int q = 0; q < kMaxQ; ++q) {
            if (half == 1 && q < Nq) {
#pragma unroll
                for (int x = 0; x < 3; ++x) {
                    qb[x] += rq[3 * q + x];
                    const float tk = rk[3 * q + x] + t[x];
                    W[x] += tk;
                    kn = fmaf(tk, tk, kn);
                }
            }
        }
        const float cb = valid ? kL2E * (-0.5f * g * kn) : kMaskedBias;
        if (ok && half == 1) p.colbias[(int64_t(b) * p.H + h) * p.L + i] = valid ? -0.5f * g * kn : -INFINITY;
        const int g0 = c + 3 * Nq, zq = p.zq;
        const int64_t hrow = (int64_t(b) * p.H + h) * p.L + i;

        // Three tensors through two alternating staging tiles.  Phase A (thread = row): columns
        // derived from TMEM and the frame.  Phase B (warp-cooperative, lanes across columns): the
        // pair-factor columns, straight from coalesced z1 / z2 row loads.
        const float* wbh = p.wl_bias + h * p.dz;
        // head-independent pair block (q_hat: bf16(log2 e z1), v_hat: bf16(z2)) -> staging tile
        // columns [col0, col0 + rdz): 16-byte cp.async per (row, 8 columns), a warp per row
        // segment (coalesced 512 B), all 4096 copies of the tile in flight at once
        const int etid = threadIdx.x - 64;
        auto copy_pair = [&](uint8_t* tile, const __nv_bfloat16* src, int col0) {
            const int nch = rdz / 8;
            auto one = [&](int rr, int j) {
                const int grow = m0 + rr < p.M ? m0 + rr : p.M - 1;
                const int col = col0 + 8 * j;
                cp_async16(tile + (col >> 6) * (BM * 128) + rr * 128 + ((((col & 63) >> 3) ^ (rr & 7)) << 4),
                           src + int64_t(grow) * rdz + 8 * j);
            };
            if (nch == 32) {  // rank 2 x d_z 128: lane = 16-byte chunk, warp = row (no division)
                for (int rr = etid >> 5; rr < BM; rr += 8) one(rr, etid & 31);
            } else {
                for (int e = etid; e < BM * nch; e += 256) one(e / nch, e % nch);
            }
        };
        PPTRACE(2);
        for (int tsel = 0; tsel < 3; ++tsel) {
            // T: 0 = q_hat (tile 0), 2 = v_hat (tile 1), 1 = k_hat (tile 0 once the q stores read it)
            const int T = tsel == 0 ? 0 : tsel == 1 ? 2 : 1;
            uint8_t* tile = tiles + (tsel & 1) * tile_bytes;
            PPTRACE(3 + 4 * tsel);
            if (tsel == 2) {
                // tile 0 is reused: tensor 0's stores (or row copies) must have read it
                if (p.chunk_ok) {
                    ptx::mbar_wait(tile_free, 0);
                } else {
                    named_sync(1, 256);
                }
            }
            const int width = T < 2 ? p.dqk_pad : p.dv_pad;
            if (T == 0) copy_pair(tile, p.z1q, zq);
            if (T == 2) copy_pair(tile, p.z2b, c);
            float v8[8];
            // ---- phase A, half 0: [0, c) scalar channels from TMEM, 16 per load
            const float sc = T == 0 ? kL2E : T == 1 ? p.k_scale : 1.f;
            const int tcol = T == 0 ? cq : T == 1 ? ck : cv;
            if (half == 0 && c % 32 == 0) {
                // two TMEM loads in flight per wait (each round trip costs ~0.5k cycles; four
                // spill at this kernel's 168-register cap)
                for (int c0 = 0; c0 < c; c0 += 32) {
                    uint32_t u[2][16];
#pragma unroll
                    for (int k = 0; k < 2; ++k) ptx::tmem_ld16(tl + tcol + c0 + 16 * k, u[k]);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int k = 0; k < 2; ++k) {
#pragma unroll
                        for (int e = 0; e < 8; ++e) v8[e] = sc * __uint_as_float(u[k][e]);
                        stage_put8(tile, r, c0 + 16 * k, v8);
#pragma unroll
                        for (int e = 0; e < 8; ++e) v8[e] = sc * __uint_as_float(u[k][8 + e]);
                        stage_put8(tile, r, c0 + 16 * k + 8, v8);
                    }
                }
            } else {
                for (int c0 = 0; c0 < (half == 0 ? c : 0); c0 += 16) {
                    uint32_t u[16];
                    ptx::tmem_ld16(tl + tcol + c0, u);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 8; ++e) v8[e] = sc * __uint_as_float(u[e]);
                    stage_put8(tile, r, c0, v8);
#pragma unroll
                    for (int e = 0; e < 8; ++e) v8[e] = sc * __uint_as_float(u[8 + e]);
                    stage_put8(tile, r, c0 + 8, v8);
                }
            }
            if (half == 0) {
            } else if (T < 2) {
                // rotated points, the 21 translation / bias columns and the zq padding
                const float gs = T == 0 ? kL2E : g;
                const float* pts = T == 0 ? rq : rk;
                // translation / bias column e of the [g0, zq) block (q_hat if T == 0, else k_hat)
                auto tcolv = [&](int e) -> float {
                    const int x = e % 3;
                    float qv, kv;
                    if (e < 9) {
                        const float qq = kL2E * qb[x], tt = g * t[x];
                        qv = e < 6 ? bf_hi(qq) : bf_lo(qq);
                        kv = (e >= 3 && e < 6) ? bf_lo(tt) : bf_hi(tt);
                    } else if (e < 18) {
                        const float tq = kL2E * t[x], ww = g * W[x];
                        qv = (e >= 12 && e < 15) ? bf_lo(tq) : bf_hi(tq);
                        kv = e < 15 ? bf_hi(ww) : bf_lo(ww);
                    } else if (e < 20) {
                        qv = 1.0f;
                        kv = e == 18 ? bf_hi(cb) : (valid ? bf_lo(cb) : 0.f);
                    } else {
                        qv = 0.f;
                        kv = e == 20 ? 1.0f : 0.f;
                    }
                    return T == 0 ? qv : kv;
                };
                if (3 * Nq == 3 * kMaxQ && c % 8 == 0 && zq - g0 == 24 && p.dqk_used % 8 == 0) {
                    // 16-byte stores: 3 point chunks, 3 translation chunks, the pad chunks
#pragma unroll
                    for (int k8 = 0; k8 < 3; ++k8) {
#pragma unroll
                        for (int e = 0; e < 8; ++e) v8[e] = gs * pts[8 * k8 + e];
                        stage_put8(tile, r, c + 8 * k8, v8);
                    }
#pragma unroll
                    for (int k8 = 0; k8 < 3; ++k8) {
#pragma unroll
                        for (int e = 0; e < 8; ++e) v8[e] = tcolv(8 * k8 + e);
                        stage_put8(tile, r, g0 + 8 * k8, v8);
                    }
#pragma unroll
                    for (int e = 0; e < 8; ++e) v8[e] = 0.f;
                    for (int e = p.dqk_used; e < width; e += 8) stage_put8(tile, r, e, v8);
                } else {
#pragma unroll
                    for (int e = 0; e < 3 * kMaxQ; ++e)
                        if (e < 3 * Nq) stage_put(tile, r, c + e, gs * pts[e]);
                    for (int e = 0; e < zq - g0; ++e) stage_put(tile, r, g0 + e, tcolv(e));
                    for (int e = p.dqk_used; e < width; ++e) stage_put(tile, r, e, 0.f);
                }
            } else {
                const int vp = c + rdz;
                // [t hi (3) | t lo (3) | R v_p (3 Nv) | 0 ...] from column vp to the row end
                auto vcolv = [&](int e) -> float {
                    if (e < 3) return bf_hi(t[e]);
                    if (e < 6) return bf_lo(t[e - 3]);
                    return e - 6 < 3 * Nv ? rv[e - 6] : 0.f;
                };
                if (vp % 8 == 0 && width - vp == 64) {
#pragma unroll
                    for (int k8 = 0; k8 < 8; ++k8) {
#pragma unroll
                        for (int e = 0; e < 8; ++e) v8[e] = (8 * k8 + e < 6 + 3 * kMaxV) ? vcolv(8 * k8 + e) : 0.f;
                        stage_put8(tile, r, vp + 8 * k8, v8);
                    }
                } else {
#pragma unroll
                    for (int x = 0; x < 3; ++x) {
                        stage_put(tile, r, vp + x, bf_hi(t[x]));
                        stage_put(tile, r, vp + 3 + x, bf_lo(t[x]));
                    }
#pragma unroll
                    for (int e = 0; e < 3 * kMaxV; ++e)
                        if (e < 3 * Nv) stage_put(tile, r, vp + 6 + e, rv[e]);
                    for (int e = p.dv_used; e < width; ++e) stage_put(tile, r, e, 0.f);
                }
            }
            PPTRACE(4 + 4 * tsel);
            // ---- phase B: pair factors.  q / v: the copies issued above; k: bf16(w_l w_bias[h] z2),
            // warp covers rows quad*32 + half*16 .. +16, lane = 8-column chunk, 16 rows in flight
            if (T == 1) {
                // k_hat pair block = w_l w_bias[h] (.) bf16(z2): scaled from v_hat's block in tile 1
                // (every thread's copies into it completed before this barrier)
                named_sync(1, 256);
                const uint8_t* vt = tiles + tile_bytes;
                const int nchunk = rdz / 8;
                for (int j = lane; j < nchunk; j += 32) {
                    float wm[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) wm[e] = __ldg(wbh + (8 * j + e) % p.dz);
                    const int col = c + 8 * j;
#pragma unroll 4
                    for (int u = 0; u < 16; ++u) {
                        const int rr = quad * 32 + 16 * half + u;
                        const uint4 za = *reinterpret_cast<const uint4*>(
                            vt + (col >> 6) * (BM * 128) + rr * 128 + ((((col & 63) >> 3) ^ (rr & 7)) << 4));
                        const uint32_t w4[4] = {za.x, za.y, za.z, za.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            v8[2 * e] = wm[2 * e] * __uint_as_float(w4[e] << 16);
                            v8[2 * e + 1] = wm[2 * e + 1] * __uint_as_float(w4[e] & 0xffff0000u);
                        }
                        stage_put8(tile, rr, zq + 8 * j, v8);
                    }
                }
            } else {
                cp_async_wait_all();
            }
            PPTRACE(5 + 4 * tsel);
            if (p.chunk_ok) {
                ptx::fence_proxy_async_smem();  // rows visible to the TMA stores of warp 0
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&tile_ready[tsel & 1]);
                PPTRACE(6 + 4 * tsel);
            } else {
                named_sync(1, 256);
                PPTRACE(6 + 4 * tsel);
            }
            if (!p.chunk_ok && ok && half == 0) {
                // generic shapes: each thread copies its own row (16-byte chunks, un-swizzled)
                __nv_bfloat16* dst = (T == 0 ? p.qhat : T == 1 ? p.khat : p.vhat) + hrow * width;
                for (int ch8 = 0; ch8 < width / 8; ++ch8) {
                    const uint8_t* src = tile + (ch8 >> 3) * (BM * 128) + r * 128 + (((ch8 & 7) ^ (r & 7)) << 4);
                    reinterpret_cast<uint4*>(dst)[ch8] = *reinterpret_cast<const uint4*>(src);
                }
            }
        }
        // raw point columns for the backward, after the three tensors: their scattered global
        // stores no longer compete with the staging-tile writes of tensor 0 (TMEM still holds them)
        if (half == 1 && p.write_points) {
            float* prow = p.proj + int64_t(rowc) * p.n_proj;
            const int oq = 3 * p.H * c + h * 3 * Nq, okp = oq + 3 * p.H * Nq, ov = 3 * p.H * c + 6 * p.H * Nq + h * 3 * Nv;
            const int cols[3] = {cqp, ckp, cvp}, offs[3] = {oq, okp, ov}, ns[3] = {3 * Nq, 3 * Nq, 3 * Nv};
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                uint32_t u[32], w[16];
                ptx::tmem_ld32(tl + cols[k], u);
                ptx::tmem_ld16(tl + cols[k] + 32, w);
                ptx::tmem_wait_ld();
                if (ok) store_points(prow + offs[k], u, w, ns[k]);
            }
        }
        PPTRACE(15);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc(tmem, 512);
    if (warp == 0 && lane == 0) span_mark(2);
}

}  // namespace

bool proj_pack_supported(const LayerDims& d) {
    const int NH = (3 * d.c + 6 * d.n_query + 3 * d.n_value + 15) / 16 * 16;
    const size_t ring = size_t(kStages) * (BM * BK * 2 + NH * BK * 2);
    const size_t tile = size_t(BM) * std::max(d.dqk_pad, d.dv_pad) * 2;
    return d.n_query <= kMaxQ && d.n_value <= kMaxV && d.c % 16 == 0 && (d.rank * d.d_z) % 8 == 0 &&
           d.d_z % 8 == 0 && d.zq % 8 == 0 && NH <= 512 && (NH / 2) % 8 == 0 && NH / 2 <= 256 &&
           d.dqk_pad % 64 == 0 && d.dv_pad % 64 == 0 && d.din_ld % 8 == 0 &&
           std::max(ring, 2 * tile) + 2048 <= 232448;
}

int proj_pack_head_width(const LayerDims& d) { return (3 * d.c + 6 * d.n_query + 3 * d.n_value + 15) / 16 * 16; }

void launch_proj_pack(const LayerDims& d, const ProjPackArgs& a, cudaStream_t stream) {
    if (!proj_pack_supported(d)) throw std::invalid_argument("fused projection+pack: unsupported shape");
    if (a.z1q == nullptr || a.z2b == nullptr) throw std::invalid_argument("fused projection+pack: bf16 pair factors missing");
    PPParams p{};
    p.M = a.B * a.L;
    p.L = a.L;
    p.H = d.heads;
    p.c = d.c;
    p.Nq = d.n_query;
    p.Nv = d.n_value;
    p.dz = d.d_z;
    p.rdz = d.rank * d.d_z;
    p.NH = proj_pack_head_width(d);
    p.N1 = std::min(p.NH, 256);
    p.N2 = p.NH - p.N1;
    p.nk = (d.d_in + BK - 1) / BK;
    p.dqk_used = d.dqk_used;
    p.dqk_pad = d.dqk_pad;
    p.dv_used = d.dv_used;
    p.dv_pad = d.dv_pad;
    p.zq = d.zq;
    p.n_proj = d.n_proj;
    p.chunk_ok = (a.L % 32) == 0 ? 1 : 0;
    p.write_points = a.write_points ? 1 : 0;
    p.z1 = a.z1;
    p.z2 = a.z2;
    p.z1q = a.z1q;
    p.z2b = a.z2b;
    p.rot = a.rot;
    p.trans = a.trans;
    p.mask = a.mask;
    p.head_g = a.head_g;
    p.wl_bias = a.wl_bias;
    p.k_scale = a.k_scale;
    p.proj = a.proj;
    p.colbias = a.colbias;
    p.qhat = a.qhat;
    p.khat = a.khat;
    p.vhat = a.vhat;
    const uint64_t BH = uint64_t(a.B) * d.heads;
    const CUtensorMap mapA = make_map_2d_bf16(a.s_bf16, uint64_t(p.M), d.d_in, d.din_ld, 64, BM);
    const CUtensorMap mapB = make_map_2d_bf16(a.w_heads, uint64_t(d.heads) * p.NH, d.d_in, d.din_ld, 64, p.NH / 2);
    const CUtensorMap mapQ = make_map_3d_bf16(a.qhat, d.dqk_pad, a.L, BH, d.dqk_pad, 64, 32);
    const CUtensorMap mapK = make_map_3d_bf16(a.khat, d.dqk_pad, a.L, BH, d.dqk_pad, 64, 32);
    const CUtensorMap mapV = make_map_3d_bf16(a.vhat, d.dv_pad, a.L, BH, d.dv_pad, 64, 32);
    const size_t ring = size_t(kStages) * (BM * BK * 2 + p.NH * BK * 2);
    const size_t tile = size_t(BM) * std::max(d.dqk_pad, d.dv_pad) * 2;
    const int smem = int(std::max(ring, 2 * tile)) + 1024 + 1024;
    cudaFuncSetAttribute(proj_pack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    dim3 grid(static_cast<unsigned>((p.M + BM - 1) / BM), static_cast<unsigned>(d.heads));
    launch_pdl(proj_pack_kernel, grid, dim3(kThreads), size_t(smem), stream, mapA, mapB, mapQ, mapK, mapV, p);
}

}  // namespace fipa_b200
