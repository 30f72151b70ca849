// Memory-bound kernels of the FlashIPA backward (the reference has no backward, proj/SPEC.md:8;
// these differentiate its forward, pinned by finite differences in tests/test_oracle.py):
//
//   bwd_prep   : the output epilogue (proj/src/flash_ipa.cpp:171-210, apply_inverse
//                proj/src/geometry.cpp:70-76) run backwards.  From dfeat = dOut . w_out^T and the
//                saved O_hat it writes dO_hat in the v_hat column layout of pack.cu
//                ([dv | z1 (.) d(pair) | sum_p dg_p | sum_p dg_p | dg_p]), D = rowsum(dO_hat*O_hat)
//                (bf16-rounded dO_hat as the MMAs see it, fp32 O_hat) and the epilogue's own gradients
//                (z1 through the pair contraction, frames through R^T(g - t)).
//   bwd_unpack : the lifts (proj/src/flash_ipa.cpp:23-126, pack.cu) run backwards.  It maps
//                the attention accumulators dQ_acc = dS.K_hat, dK_acc = dS^T.Q_hat,
//                dV_acc = P^T.dO_hat in the lifted layout back to natural gradients: the
//                projection columns (reference order w_q|w_k|w_v|w_qp|w_kp|w_vp), z1, z2,
//                rotations, translations, d(gamma w_l w_c) and d(w_l w_bias).  The column
//                bookkeeping is the one checked on the CPU by tests/bwd_emulation.py.
// Logits are q_hat.k_hat in log2 units, so dL/d(q_hat) = ln2 dQ_acc, dL/d(k_hat) = ln2 dK_acc;
// q_hat carries a log2(e) factor, which cancels on the query side.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>

#include "kernels.hpp"
#include "ptx.cuh"

namespace fipa_b200 {

namespace {

constexpr float kLn2 = 0.6931471805599453f;
constexpr float kL2E = 1.4426950408889634f;

__device__ __forceinline__ uint32_t ptx_pack(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ float bfr(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// four consecutive bf16 (8-byte aligned) as floats
__device__ __forceinline__ float4 ld4_bf16(const __nv_bfloat16* p) {
    const uint2 w = *reinterpret_cast<const uint2*>(p);
    return make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xffff0000u), __uint_as_float(w.y << 16),
                       __uint_as_float(w.y & 0xffff0000u));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Bulk (TMA-engine) copy of `bytes` contiguous global bytes into shared memory, completion
// counted on a local mbarrier.  The memory-bound backward kernels stage whole rows this way: one
// instruction moves a 1.7-10 KB row, so the LSU queues (the "lg_throttle" stall that dominated
// the per-lane version, profiles/r1_bwd_ncu_summary.json) stay empty and many KB stay in flight.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(ptx::smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(ptx::smem_u32(bar))
                 : "memory");
}

// One block per residue (b, i), warp w handles heads w, w+8, ...  The residue's dfeat row and the
// H saved O_hat rows arrive by bulk copies; dO_hat rows are assembled in shared memory and
// written with 16-byte stores; cross-head sums (dz1, frames) go through per-warp slices.
__global__ void __launch_bounds__(256, 4) bwd_prep_kernel(LayerDims d, BwdPrepArgs a) {
    extern __shared__ __align__(16) float sm[];
    const int H = d.heads, c = d.c, dz = d.d_z, rdz = d.rank * d.d_z, Nv = d.n_value;
    const int nw = blockDim.x >> 5;
    __nv_bfloat16* s_df = reinterpret_cast<__nv_bfloat16*>(sm);  // feat_ld   dfeat row (bf16)
    float* s_o = sm + d.feat_ld / 2;                // H x dv_pad  O_hat rows (feat_ld % 8 == 0)
    float* s_z1 = s_o + H * d.dv_pad;               // rdz
    float* s_pair = s_z1 + ((rdz + 3) & ~3);        // nw x rdz   per-warp dz1 partials
    float* s_geo = s_pair + nw * rdz;               // nw x 12    per-warp dR (9) | dt (3)
    float* s_dopt = s_geo + nw * 12;                // nw x 3*Nv
    __nv_bfloat16* s_out = reinterpret_cast<__nv_bfloat16*>(
        (reinterpret_cast<uintptr_t>(s_dopt + nw * 3 * Nv) + 15) & ~uintptr_t(15));  // H x dv_pad
    uint64_t* bar = reinterpret_cast<uint64_t*>(s_out + H * d.dv_pad);
    const int64_t row = blockIdx.x;
    const int b = static_cast<int>(row / a.L), i = static_cast<int>(row % a.L);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        ptx::mbar_init(bar, 1);
        ptx::fence_mbar_init();
        const uint32_t df_bytes = d.feat_ld * 2, o_bytes = d.dv_pad * 4;
        ptx::mbar_expect_tx(bar, df_bytes + H * o_bytes);
        bulk_g2s(s_df, a.dfeat + row * d.feat_ld, df_bytes, bar);
        bulk_g2s(s_o, a.ohat + row * H * d.dv_pad, H * o_bytes, bar);  // residue-major O_hat rows
    }
    for (int e = threadIdx.x; e < rdz; e += blockDim.x) s_z1[e] = a.z1[row * rdz + e];
    // s_pair needs no clearing when every warp owns exactly one head (its slice is overwritten)
    const bool one_head = H <= nw;
    for (int e = threadIdx.x; e < (one_head ? 0 : nw * rdz) + nw * 12; e += blockDim.x)
        s_pair[(one_head ? nw * rdz : 0) + e] = 0.f;  // s_pair (several heads per warp) + s_geo
    float R[9], t[3];
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = __ldg(a.rot + row * 9 + k);
#pragma unroll
    for (int k = 0; k < 3; ++k) t[k] = __ldg(a.trans_c + row * 3 + k);
    __syncthreads();
    ptx::mbar_wait(bar, 0);

    const int vpair = c + rdz, vpts = vpair + 6, vend = vpts + 3 * Nv;
    float* dopt_s = s_dopt + warp * 3 * Nv;
    float* pair_s = s_pair + warp * rdz;
    const bool vec = (c % 4) == 0 && (rdz % 4) == 0 && (dz % 4) == 0 && (d.seg % 4) == 0;
    float dR[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, dt[3] = {0.f, 0.f, 0.f};
    for (int h = warp; h < H; h += nw) {
        const int64_t hrow = (static_cast<int64_t>(b) * H + h) * a.L + i;
        const float* o = s_o + h * d.dv_pad;
        const __nv_bfloat16* df = s_df + h * d.seg;
        float ds[3] = {0.f, 0.f, 0.f};
        if (lane < Nv) {
            const int p = lane;
            float y[3], loc[3];
#pragma unroll
            for (int x = 0; x < 3; ++x) y[x] = o[vpts + 3 * p + x] + o[vpair + x] + o[vpair + 3 + x] - t[x];
#pragma unroll
            for (int x = 0; x < 3; ++x) loc[x] = R[x] * y[0] + R[3 + x] * y[1] + R[6 + x] * y[2];
            const float nrm = sqrtf(loc[0] * loc[0] + loc[1] * loc[1] + loc[2] * loc[2]);
            const float sc = nrm > 0.f ? __bfloat162float(df[dz + c + 3 * Nv + p]) / nrm : 0.f;
            float dl[3];
#pragma unroll
            for (int x = 0; x < 3; ++x) dl[x] = __bfloat162float(df[dz + c + 3 * p + x]) + sc * loc[x];
#pragma unroll
            for (int x = 0; x < 3; ++x) {
                ds[x] = R[3 * x] * dl[0] + R[3 * x + 1] * dl[1] + R[3 * x + 2] * dl[2];
                dopt_s[3 * p + x] = ds[x];
                dt[x] -= ds[x];
            }
            // local = R^T y  =>  dR[b][a] += y_b dl_a
#pragma unroll
            for (int bb = 0; bb < 3; ++bb)
#pragma unroll
                for (int aa = 0; aa < 3; ++aa) dR[3 * bb + aa] += y[bb] * dl[aa];
        }
#pragma unroll
        for (int x = 0; x < 3; ++x) ds[x] = warp_sum(ds[x]);
        __syncwarp();
        __nv_bfloat16* out = s_out + h * d.dv_pad;
        float Dp = 0.f;
        if (vec) {
            // segment-wise, 4 columns per lane step: [dv | z1 (.) d(pair) | sum dg x2 | dg_p | 0],
            // written straight to the global dO_hat row (8-byte stores, coalesced across the warp)
            __nv_bfloat16* gout = a.dohat + hrow * d.dv_pad;
            for (int j = lane; 4 * j < c; j += 32) {
                const float4 dv = ld4_bf16(df + dz + 4 * j);
                const float4 ov = *reinterpret_cast<const float4*>(o + 4 * j);
                Dp += dv.x * ov.x + dv.y * ov.y + dv.z * ov.z + dv.w * ov.w;
                *reinterpret_cast<uint2*>(gout + 4 * j) = make_uint2(ptx_pack(dv.x, dv.y), ptx_pack(dv.z, dv.w));
            }
            for (int rho = 0; rho < d.rank; ++rho) {  // pair block rho: d(pair) columns repeat per rank
                for (int j = lane; 4 * j < dz; j += 32) {
                    const int e = rho * dz + 4 * j;
                    const float4 zz = *reinterpret_cast<const float4*>(s_z1 + e);
                    const float4 dpc = ld4_bf16(df + 4 * j);
                    const float4 ov = *reinterpret_cast<const float4*>(o + c + e);
                    const float v0 = bfr(zz.x * dpc.x), v1 = bfr(zz.y * dpc.y), v2 = bfr(zz.z * dpc.z), v3 = bfr(zz.w * dpc.w);
                    Dp += v0 * ov.x + v1 * ov.y + v2 * ov.z + v3 * ov.w;
                    float4 ps = one_head ? make_float4(0.f, 0.f, 0.f, 0.f)
                                         : *reinterpret_cast<float4*>(pair_s + e);  // warp-private slice
                    ps.x += ov.x * dpc.x;
                    ps.y += ov.y * dpc.y;
                    ps.z += ov.z * dpc.z;
                    ps.w += ov.w * dpc.w;
                    *reinterpret_cast<float4*>(pair_s + e) = ps;
                    *reinterpret_cast<uint2*>(gout + c + e) = make_uint2(ptx_pack(v0, v1), ptx_pack(v2, v3));
                }
            }
            for (int col = vpair + lane; col < d.dv_pad; col += 32) {
                float v = 0.f;
                if (col < vpts) {
                    const int x = (col - vpair) % 3;  // select, not an indexed load: keeps ds[] in registers
                    v = x == 0 ? ds[0] : (x == 1 ? ds[1] : ds[2]);
                }
                else if (col < vend) v = dopt_s[col - vpts];
                v = bfr(v);
                gout[col] = __float2bfloat16_rn(v);
                if (col < d.dv_used) Dp += v * o[col];
            }
        } else {
            for (int c4 = lane; 4 * c4 < d.dv_pad; c4 += 32) {
            const float4 ov = *reinterpret_cast<const float4*>(o + 4 * c4);
            const float oo[4] = {ov.x, ov.y, ov.z, ov.w};
            float v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int col = 4 * c4 + u;
                if (col < c) {
                    v[u] = __bfloat162float(df[dz + col]);
                } else if (col < vpair) {
                    const int e = col - c;
                    const float dpc = __bfloat162float(df[e % dz]);
                    v[u] = s_z1[e] * dpc;
                    pair_s[e] = (one_head ? 0.f : pair_s[e]) + oo[u] * dpc;  // warp-private slice, one lane per e
                } else if (col < vpts) {
                    const int x = (col - vpair) % 3;
                    v[u] = x == 0 ? ds[0] : (x == 1 ? ds[1] : ds[2]);
                } else if (col < vend) {
                    v[u] = dopt_s[col - vpts];
                } else {
                    v[u] = 0.f;
                }
                v[u] = __bfloat162float(__float2bfloat16_rn(v[u]));
                if (col < d.dv_used) Dp += v[u] * oo[u];
            }
            uint2 w;
            w.x = ptx_pack(v[0], v[1]);
            w.y = ptx_pack(v[2], v[3]);
            *reinterpret_cast<uint2*>(out + 4 * c4) = w;
        }
        }
        Dp = warp_sum(Dp);
        if (lane == 0) a.Dvec[hrow] = Dp;
        __syncwarp();
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) dR[k] = warp_sum(dR[k]);
#pragma unroll
    for (int k = 0; k < 3; ++k) dt[k] = warp_sum(dt[k]);
    if (lane < 12) s_geo[warp * 12 + lane] = lane < 9 ? dR[lane] : dt[lane - 9];
    __syncthreads();
    const int per_row = d.dv_pad / 8;  // 16-byte chunks per dO_hat row (staged rows: generic shapes)
    for (int e = threadIdx.x; !vec && e < H * per_row; e += blockDim.x) {
        const int h = e / per_row, k = e - h * per_row;
        reinterpret_cast<uint4*>(a.dohat + ((static_cast<int64_t>(b) * H + h) * a.L + i) * d.dv_pad)[k] =
            reinterpret_cast<const uint4*>(s_out + h * d.dv_pad)[k];
    }
    for (int e = threadIdx.x; e < rdz; e += blockDim.x) {
        float acc = 0.f;
        const int nslices = one_head ? H : nw;  // (one head per warp: only the first H slices are written)
        for (int w = 0; w < nslices; ++w) acc += s_pair[w * rdz + e];
        a.dz1_epi[row * rdz + e] = acc;
    }
    if (threadIdx.x < 12) {
        float acc = 0.f;
        for (int w = 0; w < nw; ++w) acc += s_geo[w * 12 + threadIdx.x];
        a.geo_epi[row * 12 + threadIdx.x] = acc;
    }
}

// Compile-time-shaped prep (c = d_z = 128, rank 1-2, 12 value points: every BASELINE training
// config): one WARP per residue looping over its heads, lanes across columns.  The generic kernel
// above (block per residue, warp per head, runtime-shaped loops) ran issue bound -- 9.1k warp
// instructions per residue, a third of them index arithmetic, plus per-head cross-warp reductions
// through shared memory (ncu: 74% issue slots busy, DRAM 28%).  Here the pair-factor row z1, the
// dz1 partial sums and the frame gradient stay in registers across the heads, every global access
// is a coalesced 8/16-byte lane access, and the only cross-lane work per head is D (one warp sum)
// and the translation-column sum of the point gradients.
template <int C, int DZ, int RANK, int NV, int DVPAD>
__global__ void __launch_bounds__(256, 3) bwd_prep_warp_kernel(LayerDims d, BwdPrepArgs a) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    constexpr int RDZ = RANK * DZ, VPAIR = C + RDZ, VPTS = VPAIR + 6, VEND = VPTS + 3 * NV, TAIL = DVPAD - VPAIR;
    constexpr int SEG = DZ + C + 4 * NV;
    static_assert(C % 128 == 0 && DZ % 128 == 0 && TAIL % 64 == 0 && VEND <= DVPAD && NV <= 32, "prep shape");
    __shared__ float s_pt[8][3 * NV];  // per-warp point gradients of the current head
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row = int64_t(blockIdx.x) * 8 + warp;
    if (row >= int64_t(a.B) * a.L) return;  // no block-level synchronisation below
    const int b = static_cast<int>(row / a.L), i = static_cast<int>(row - int64_t(b) * a.L);
    const int H = d.heads;
    float R[9], t[3];
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = __ldg(a.rot + row * 9 + k);
#pragma unroll
    for (int k = 0; k < 3; ++k) t[k] = __ldg(a.trans_c + row * 3 + k);
    float4 z1v[RDZ / 128], dz1[RDZ / 128];
#pragma unroll
    for (int k = 0; k < RDZ / 128; ++k) {
        z1v[k] = __ldg(reinterpret_cast<const float4*>(a.z1 + row * RDZ + 128 * k) + lane);
        dz1[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float dR[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, dt[3] = {0.f, 0.f, 0.f};
    float* spt = s_pt[warp];
#pragma unroll 1
    for (int h = 0; h < H; ++h) {
        const float* o = a.ohat + (row * H + h) * DVPAD;
        const __nv_bfloat16* df = a.dfeat + row * d.feat_ld + h * SEG;
        // all of the head's loads first (one memory latency per head)
        float4 os[C / 128], op[RDZ / 128], dv[C / 128], dp[DZ / 128];
        float2 ot[TAIL / 64];
#pragma unroll
        for (int k = 0; k < C / 128; ++k) {
            os[k] = __ldg(reinterpret_cast<const float4*>(o + 128 * k) + lane);
            dv[k] = ld4_bf16(df + DZ + 128 * k + 4 * lane);
        }
#pragma unroll
        for (int k = 0; k < RDZ / 128; ++k) op[k] = __ldg(reinterpret_cast<const float4*>(o + C + 128 * k) + lane);
#pragma unroll
        for (int k = 0; k < DZ / 128; ++k) dp[k] = ld4_bf16(df + 128 * k + 4 * lane);
#pragma unroll
        for (int k = 0; k < TAIL / 64; ++k) ot[k] = __ldg(reinterpret_cast<const float2*>(o + VPAIR + 64 * k) + lane);
        // value points: lane p < NV.  y = global point - t; loc = R^T y; the feature block holds
        // loc (3) and |loc| (1) per point; ds = R dl is the gradient of the global point.
        float ds[3] = {0.f, 0.f, 0.f};
        if (lane < NV) {
            const int p = lane;
            float y[3], loc[3], dl[3];
#pragma unroll
            for (int x = 0; x < 3; ++x) y[x] = __ldg(o + VPTS + 3 * p + x) + __ldg(o + VPAIR + x) + __ldg(o + VPAIR + 3 + x) - t[x];
#pragma unroll
            for (int x = 0; x < 3; ++x) loc[x] = R[x] * y[0] + R[3 + x] * y[1] + R[6 + x] * y[2];
            const float nrm = sqrtf(loc[0] * loc[0] + loc[1] * loc[1] + loc[2] * loc[2]);
            const float sc = nrm > 0.f ? __bfloat162float(df[DZ + C + 3 * NV + p]) / nrm : 0.f;
#pragma unroll
            for (int x = 0; x < 3; ++x) dl[x] = __bfloat162float(df[DZ + C + 3 * p + x]) + sc * loc[x];
#pragma unroll
            for (int x = 0; x < 3; ++x) {
                ds[x] = R[3 * x] * dl[0] + R[3 * x + 1] * dl[1] + R[3 * x + 2] * dl[2];
                spt[3 * p + x] = bfr(ds[x]);
                dt[x] -= ds[x];
            }
#pragma unroll
            for (int bb = 0; bb < 3; ++bb)
#pragma unroll
                for (int aa = 0; aa < 3; ++aa) dR[3 * bb + aa] += y[bb] * dl[aa];
        }
#pragma unroll
        for (int x = 0; x < 3; ++x) ds[x] = bfr(warp_sum(ds[x]));  // translation hi and lo columns
        __syncwarp();
        __nv_bfloat16* gout = a.dohat + ((int64_t(b) * H + h) * a.L + i) * DVPAD;
        float Dp = 0.f;
#pragma unroll
        for (int k = 0; k < C / 128; ++k) {
            Dp += dv[k].x * os[k].x + dv[k].y * os[k].y + dv[k].z * os[k].z + dv[k].w * os[k].w;
            *reinterpret_cast<uint2*>(gout + 128 * k + 4 * lane) =
                make_uint2(ptx_pack(dv[k].x, dv[k].y), ptx_pack(dv[k].z, dv[k].w));
        }
#pragma unroll
        for (int k = 0; k < RDZ / 128; ++k) {  // pair block rho = k / (DZ / 128): d(pair) repeats per rank
            const float4 dpc = dp[k % (DZ / 128)], zz = z1v[k], ov = op[k];
            const float v0 = bfr(zz.x * dpc.x), v1 = bfr(zz.y * dpc.y), v2 = bfr(zz.z * dpc.z), v3 = bfr(zz.w * dpc.w);
            Dp += v0 * ov.x + v1 * ov.y + v2 * ov.z + v3 * ov.w;
            dz1[k].x += ov.x * dpc.x;
            dz1[k].y += ov.y * dpc.y;
            dz1[k].z += ov.z * dpc.z;
            dz1[k].w += ov.w * dpc.w;
            *reinterpret_cast<uint2*>(gout + C + 128 * k + 4 * lane) = make_uint2(ptx_pack(v0, v1), ptx_pack(v2, v3));
        }
#pragma unroll
        for (int k = 0; k < TAIL / 64; ++k) {
            float v[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int col = VPAIR + 64 * k + 2 * lane + u;
                const int x = (col - VPAIR) % 3;
                v[u] = col < VPTS ? (x == 0 ? ds[0] : (x == 1 ? ds[1] : ds[2])) : col < VEND ? spt[col - VPTS] : 0.f;
            }
            // padding columns of O_hat are never written: keep them out of D
            const int col0 = VPAIR + 64 * k + 2 * lane;
            if (col0 < VEND) Dp += v[0] * ot[k].x;
            if (col0 + 1 < VEND) Dp += v[1] * ot[k].y;
            *reinterpret_cast<uint32_t*>(gout + col0) = ptx_pack(v[0], v[1]);
        }
        Dp = warp_sum(Dp);
        if (lane == 0) a.Dvec[(int64_t(b) * H + h) * a.L + i] = Dp;
        __syncwarp();  // spt reused by the next head
    }
#pragma unroll
    for (int k = 0; k < RDZ / 128; ++k) reinterpret_cast<float4*>(a.dz1_epi + row * RDZ + 128 * k)[lane] = dz1[k];
#pragma unroll
    for (int k = 0; k < 9; ++k) dR[k] = warp_sum(dR[k]);
#pragma unroll
    for (int k = 0; k < 3; ++k) dt[k] = warp_sum(dt[k]);
    float gv = 0.f;
#pragma unroll
    for (int k = 0; k < 12; ++k) gv = lane == k ? (k < 9 ? dR[k] : dt[k - 9]) : gv;  // no indexed (local) array
    if (lane < 12) a.geo_epi[row * 12 + lane] = gv;
}

constexpr int kUnpackRows = 8;
constexpr int kUnpackMaxH = 16;

// Lifts^T (pack.cu / proj_pack.cu reversed), in two launches so each half runs at its own
// occupancy:
//  bwd_unpack_geo_kernel   block = 8 residues, one warp per residue with lanes over (head, point)
//                          tasks: frame-applied point gradients -> dproj point columns; dR, dt
//                          summed over the residue's heads by one warp reduction -> drot, dt_c;
//                          dgamma terms summed over the block's residues in shared memory -> dg.
//                          (launch bounds 256 x 4 cap it at 64 registers; ptxas -v: no spills)
//  bwd_unpack_kernel       block streams kUnpackRows residues; every accumulator column of the
//                          scalar and pair blocks is read by exactly one thread with coalesced
//                          loads (no staging, all loads of a residue in flight at once):
//                          scalar q | k (x w_l/sqrt(c) ln2) | v -> bf16 pairs of the dproj row;
//                          pair e: dz1 = dz1_epi + sum_h dq[zq+e],
//                          dz2 = sum_h (w_l w_bias[h, e % d_z] ln2 dk[zq+e] + dv[c+e]),
//                          d(w_l w_bias)[h, e % d_z] += ln2 dk[zq+e] z2[e] (register partials).
// The two write disjoint outputs.  (Forking the geometry kernel onto a side stream beside the
// streaming one: unpack 0.109 -> 0.100 ms in one chain, but the micro-batched step 0.860 -> 0.874.)
// The geometry of one residue (warp-wide; lanes over (head, point) tasks): frame-applied point
// gradients -> dproj point columns, dR / dt summed over the heads -> drot, dt_c, per-head dgamma
// terms -> s_dg (this warp's kUnpackMaxH floats of shared memory).
__device__ __forceinline__ void unpack_geo_row(const LayerDims& d, const BwdUnpackArgs& a, int64_t row, int lane,
                                               float* s_dg) {
    const int H = d.heads, c = d.c, rdz = d.rank * d.d_z, Nq = d.n_query, Nv = d.n_value;
    const int off_qp = 3 * H * c, off_kp = off_qp + H * Nq * 3, off_vp = off_kp + H * Nq * 3;
    const int g0 = c + 3 * Nq, vpair = c + rdz;
    if (lane < kUnpackMaxH) s_dg[lane] = 0.f;
    __syncwarp();
    const int64_t acc_h = a.acc_ld;
    const float* qrow = a.dq_acc + row * H * acc_h;
    const float* krow = a.dk_acc + row * H * acc_h;
    const float* vrow = a.dv_acc + row * H * acc_h;
    __nv_bfloat16* dp = a.dproj + row * a.nproj_ld;
    const float* pr = a.proj + row * d.n_proj;
    float R[9], t[3];
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = __ldg(a.rot + row * 9 + k);
#pragma unroll
    for (int k = 0; k < 3; ++k) t[k] = __ldg(a.trans_c + row * 3 + k);
    float dR[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, dt[3] = {0.f, 0.f, 0.f};
    // ---- query / key points: task = (head, point)
    for (int task = lane; task < H * Nq; task += 32) {
        const int h = task / Nq, p = task - h * Nq;
        const float* qa = qrow + h * acc_h;
        const float* ka = krow + h * acc_h;
        const float g = __ldg(a.head_g + h);
        const float cs = __ldg(ka + g0 + 18);
        const float S1 = __ldg(qa + g0 + 20);  // sum_j dS_ij, as rounded for the MMAs
        float qp[3], gB[3], kp[3], kc[3], dW[3];
#pragma unroll
        for (int x = 0; x < 3; ++x) {
            qp[x] = __ldg(pr + off_qp + (h * Nq + p) * 3 + x);
            gB[x] = __ldg(qa + c + 3 * p + x) + __ldg(qa + g0 + x) + __ldg(qa + g0 + 3 + x);
            kp[x] = __ldg(pr + off_kp + (h * Nq + p) * 3 + x);
            kc[x] = __ldg(ka + c + 3 * p + x);
            dW[x] = g * kLn2 * (__ldg(ka + g0 + 9 + x) + __ldg(ka + g0 + 12 + x));
        }
        // query point: A = R q_p + t,  dA = g sum_j dS_ij (B_jp - A) = [g sum_j dS B] - g A S1
        // (subtracting g A S1 with the same rounded dS cancels the translation-sized common mode)
        float A[3], dA[3], B[3], dB[3];
#pragma unroll
        for (int x = 0; x < 3; ++x) A[x] = R[3 * x] * qp[0] + R[3 * x + 1] * qp[1] + R[3 * x + 2] * qp[2] + t[x];
#pragma unroll
        for (int x = 0; x < 3; ++x) {
            dA[x] = gB[x] - g * A[x] * S1;
            dt[x] += dA[x];
        }
        // d/dg of -g/2 |A - B|^2 summed with dS: A.(sum_j dS B) - |A|^2 S1 / 2 (+ key part)
        // gB carries the factor g; a head whose g rounds to 0 (very negative gamma_raw) has
        // gB == 0 too, and its term is taken as 0 instead of 0/0
        const float inv_g = g != 0.f ? 1.f / g : 0.f;
        float dgh = (A[0] * gB[0] + A[1] * gB[1] + A[2] * gB[2]) * inv_g -
                    0.5f * (A[0] * A[0] + A[1] * A[1] + A[2] * A[2]) * S1;
#pragma unroll
        for (int x = 0; x < 3; ++x) {
            dp[off_qp + (h * Nq + p) * 3 + x] = __float2bfloat16_rn(R[x] * dA[0] + R[3 + x] * dA[1] + R[6 + x] * dA[2]);
#pragma unroll
            for (int y = 0; y < 3; ++y) dR[3 * x + y] += dA[x] * qp[y];
        }
        // key point: B = R k_p + t
#pragma unroll
        for (int x = 0; x < 3; ++x) B[x] = R[3 * x] * kp[0] + R[3 * x + 1] * kp[1] + R[3 * x + 2] * kp[2] + t[x];
#pragma unroll
        for (int x = 0; x < 3; ++x) {
            dB[x] = g * kLn2 * kc[x] + dW[x] - g * B[x] * cs;
            dt[x] -= g * B[x] * cs;
        }
        dgh += -0.5f * (B[0] * B[0] + B[1] * B[1] + B[2] * B[2]) * cs;
#pragma unroll
        for (int x = 0; x < 3; ++x) {
            dp[off_kp + (h * Nq + p) * 3 + x] = __float2bfloat16_rn(R[x] * dB[0] + R[3 + x] * dB[1] + R[6 + x] * dB[2]);
#pragma unroll
            for (int y = 0; y < 3; ++y) dR[3 * x + y] += dB[x] * kp[y];
        }
        atomicAdd(&s_dg[h], dgh);
    }
    // ---- value points
    for (int task = lane; task < H * Nv; task += 32) {
        const int h = task / Nv, p = task - h * Nv;
        const float* va = vrow + h * acc_h;
        float vp[3], dV[3];
#pragma unroll
        for (int x = 0; x < 3; ++x) {
            vp[x] = __ldg(pr + off_vp + (h * Nv + p) * 3 + x);
            dV[x] = __ldg(va + vpair + 6 + 3 * p + x);
        }
#pragma unroll
        for (int x = 0; x < 3; ++x) {
            dp[off_vp + (h * Nv + p) * 3 + x] = __float2bfloat16_rn(R[x] * dV[0] + R[3 + x] * dV[1] + R[6 + x] * dV[2]);
#pragma unroll
            for (int y = 0; y < 3; ++y) dR[3 * x + y] += dV[x] * vp[y];
        }
    }
    // ---- per-head translation terms (key frame columns, value translation columns)
    for (int h = lane; h < H; h += 32) {
        const float* ka = krow + h * acc_h;
        const float* va = vrow + h * acc_h;
        const float g = __ldg(a.head_g + h);
#pragma unroll
        for (int x = 0; x < 3; ++x) {
            const float dW = g * kLn2 * (__ldg(ka + g0 + 9 + x) + __ldg(ka + g0 + 12 + x));
            dt[x] += g * kLn2 * (__ldg(ka + g0 + x) + __ldg(ka + g0 + 6 + x)) + float(Nq) * dW  // key
                     + __ldg(va + vpair + x);                                                   // value
        }
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) dR[k] = warp_sum(dR[k]);
#pragma unroll
    for (int k = 0; k < 3; ++k) dt[k] = warp_sum(dt[k]);
    if (lane < 12) {
        const float v = (lane < 9 ? dR[lane] : dt[lane - 9]) + __ldg(a.geo_epi + row * 12 + lane);
        if (lane < 9) {
            if (a.drot != nullptr) a.drot[row * 9 + lane] = v;
        } else {
            a.dt_c[row * 3 + lane - 9] = v;
        }
    }
}

__global__ void __launch_bounds__(256, 4) bwd_unpack_geo_kernel(LayerDims d, BwdUnpackArgs a) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    // One warp per residue; lanes run over (head, point) tasks so every lane works (the per-head
    // form left 20 of 32 lanes idle and was issue bound).  dR / dt are summed over the residue's
    // heads with one warp reduction; per-head dgamma terms go through shared memory.
    // The block's 8 residues' dgamma terms are summed here (one atomic per head and block), so the
    // streaming kernel does not depend on this one and the two run concurrently.
    __shared__ float s_dg[8][kUnpackMaxH];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + warp;
    if (lane < kUnpackMaxH) s_dg[warp][lane] = 0.f;
    __syncwarp();
    if (row < static_cast<int64_t>(a.B) * a.L) unpack_geo_row(d, a, row, lane, s_dg[warp]);
    __syncthreads();
    if (threadIdx.x < d.heads) {
        float acc = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) acc += s_dg[w][threadIdx.x];
        atomicAdd(&a.dg[threadIdx.x], acc);
    }
}

// Accumulator element i from the bf16 copy (H16: scalar / pair columns of dK, dV) or fp32.
template <bool H16>
__device__ __forceinline__ float acc_at(const float* f, const __nv_bfloat16* b, int64_t i) {
    if constexpr (H16) return __bfloat162float(b[i]);
    else return __ldg(f + i);
}
// Scalar-column pair (even element i) of accumulator tsel (0 dQ, 1 dK, 2 dV), from the bf16
// copies where they exist (Q16: dQ, H16: dK / dV).
template <bool H16, bool Q16>
__device__ __forceinline__ float2 acc2_sel(const BwdUnpackArgs& a, int tsel, int64_t i) {
    if ((tsel == 0 && Q16) || (tsel != 0 && H16)) {
        const __nv_bfloat16* b = tsel == 0 ? a.dq16 : (tsel == 1 ? a.dk16 : a.dv16);
        const uint32_t u = __ldg(reinterpret_cast<const unsigned int*>(b + i));
        return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xFFFF0000u));
    }
    return __ldg(reinterpret_cast<const float2*>((tsel == 0 ? a.dq_acc : (tsel == 1 ? a.dk_acc : a.dv_acc)) + i));
}

// FAST: H <= 8 heads, one pair column per thread, the row's scalar columns in kBatchF float2 per
// thread (every training config); the general form otherwise.  (Two instantiations so the fast
// loop's register budget holds only its 8 head partials: spills there cost ~2x.)
template <bool ACC16, bool Q16, bool FAST>
__global__ void __launch_bounds__(256, 2) bwd_unpack_kernel(LayerDims d, BwdUnpackArgs a) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    extern __shared__ __align__(16) float sm[];
    const int H = d.heads, c = d.c, dz = d.d_z, rdz = d.rank * d.d_z;
    const int tid = threadIdx.x;
    float* s_dwlb = sm;                 // H x dz
    float* s_wlb = s_dwlb + H * dz;     // H x dz
    const int zq = d.zq;
    const int64_t BL = static_cast<int64_t>(a.B) * a.L;
    const int64_t ngroups = (BL + kUnpackRows - 1) / kUnpackRows;
    const int64_t acc_h = a.acc_ld;     // accumulator rows are residue-major [BL, H, acc_ld]
    const float kscale = a.k_scale * kLn2;
    const int half_c = c / 2;
    const bool pairs = (c % 2) == 0 && (a.acc_ld % 2) == 0 && (a.nproj_ld % 2) == 0;
    const bool reg_dwlb = rdz <= static_cast<int>(blockDim.x);  // one pair column per thread
    for (int e = tid; e < H * dz; e += blockDim.x) {
        s_dwlb[e] = 0.f;
        s_wlb[e] = a.wl_bias[e];
    }
    __syncthreads();
    constexpr int kPw = FAST ? 8 : kUnpackMaxH;
    float pw[kPw];  // this thread's d(w_l w_bias) partials over the block's residues
#pragma unroll
    for (int h = 0; h < kPw; ++h) pw[h] = 0.f;

    // Fast path (H <= 8, one pair column per thread, a row's scalar columns in kBatchF float2 per
    // thread): ALL of a row's loads -- 24 pair-column loads and the scalar float2 loads -- are
    // issued before any use, so each row costs one memory latency instead of two.
    constexpr int kBatchF = 6;  // (unpack_fast() on the host selects FAST)
    // persistent: groups of kUnpackRows residues strided over a grid of (SMs x resident blocks)
    for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const int64_t row_begin = grp * kUnpackRows;
    const int nrows = static_cast<int>(BL - row_begin < kUnpackRows ? BL - row_begin : kUnpackRows);
    // raw loaded bits, converted only at use (a conversion right after a load would wait for it
    // and serialise the row's loads: measured 2x on the bf16 copies)
    struct RowLoads {
        uint32_t qq[8], kq[8], vq[8];  // fp32 bits, or a bf16 in the low half (Q16 / ACC16)
        uint2 v[kBatchF];              // fp32 pair, or a bf16 pair in .x
        float z2v, s1;
    };
    auto raw16 = [](const __nv_bfloat16* b, int64_t i) -> uint32_t {
        return __ldg(reinterpret_cast<const unsigned short*>(b + i));
    };
    auto as_f = [](uint32_t r) { return ACC16 ? __uint_as_float(r << 16) : __uint_as_float(r); };
    auto as_fq = [](uint32_t r) { return Q16 ? __uint_as_float(r << 16) : __uint_as_float(r); };
    const int total = 3 * H * half_c;
    auto load_row = [&](int64_t row, RowLoads& L) {
        const int64_t base = row * H * acc_h;
        L.z2v = __ldg(a.z2 + row * rdz + tid);
        L.s1 = __ldg(a.dz1_epi + row * rdz + tid);
        const int64_t ko = base + zq + tid, vo = base + c + tid;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int h = min(u, H - 1);
            if constexpr (Q16) L.qq[u] = raw16(a.dq16, ko + h * acc_h);
            else L.qq[u] = __float_as_uint(__ldg(a.dq_acc + ko + h * acc_h));
            if constexpr (ACC16) {
                L.kq[u] = raw16(a.dk16, ko + h * acc_h);
                L.vq[u] = raw16(a.dv16, vo + h * acc_h);
            } else {
                L.kq[u] = __float_as_uint(__ldg(a.dk_acc + ko + h * acc_h));
                L.vq[u] = __float_as_uint(__ldg(a.dv_acc + vo + h * acc_h));
            }
        }
#pragma unroll
        for (int u = 0; u < kBatchF; ++u) {
            const int idx = min(tid + u * static_cast<int>(blockDim.x), total - 1);
            const int tsel = idx / (H * half_c), rem = idx - tsel * (H * half_c);
            const int h = rem / half_c, cc = 2 * (rem - h * half_c);
            const int64_t i = base + h * acc_h + cc;
            if ((ACC16 && tsel != 0) || (Q16 && tsel == 0)) {
                L.v[u].x = __ldg(reinterpret_cast<const unsigned int*>(
                    (tsel == 0 ? a.dq16 : (tsel == 1 ? a.dk16 : a.dv16)) + i));
                L.v[u].y = 0u;
            } else {
                L.v[u] = __ldg(reinterpret_cast<const uint2*>(
                    (tsel == 0 ? a.dq_acc : (tsel == 1 ? a.dk_acc : a.dv_acc)) + i));
            }
        }
    };
    auto finish_row = [&](int64_t row, const RowLoads& L) {
        const int dd = tid % dz;
        float s1 = L.s1, s2 = 0.f;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (u < H) {
                const float k2 = kLn2 * as_f(L.kq[u]);
                s1 += as_fq(L.qq[u]);
                s2 += s_wlb[u * dz + dd] * k2 + as_f(L.vq[u]);
                pw[u] = fmaf(k2, L.z2v, pw[u]);
            }
        }
        a.dz1[row * rdz + tid] = s1;
        a.dz2[row * rdz + tid] = s2;
        __nv_bfloat16* dp = a.dproj + row * a.nproj_ld;
#pragma unroll
        for (int u = 0; u < kBatchF; ++u) {
            const int idx = tid + u * static_cast<int>(blockDim.x);
            if (idx < total) {
                // dproj column of the same (tensor, head, channel pair): idx * 2 in [q | k | v] order
                const bool kcol = idx >= H * half_c && idx < 2 * H * half_c;
                const float sc = kcol ? kscale : 1.f;
                float vx, vy;
                if (idx >= H * half_c ? ACC16 : Q16) {  // a bf16 pair
                    vx = __uint_as_float(L.v[u].x << 16);
                    vy = __uint_as_float(L.v[u].x & 0xFFFF0000u);
                } else {
                    vx = __uint_as_float(L.v[u].x);
                    vy = __uint_as_float(L.v[u].y);
                }
                *reinterpret_cast<uint32_t*>(dp + 2 * idx) = ptx_pack(vx * sc, vy * sc);
            }
        }
        for (int x = d.n_proj + tid; x < a.nproj_ld; x += blockDim.x) dp[x] = __float2bfloat16_rn(0.f);
    };
    // two residues' loads in flight per thread before either is used
    if constexpr (FAST)
    for (int rr = 0; rr < nrows; rr += 2) {
        RowLoads L0, L1;
        load_row(row_begin + rr, L0);
        if (rr + 1 < nrows) load_row(row_begin + rr + 1, L1);
        finish_row(row_begin + rr, L0);
        if (rr + 1 < nrows) finish_row(row_begin + rr + 1, L1);
    }

    if constexpr (!FAST)
    for (int rr = 0; rr < nrows; ++rr) {
        const int64_t row = row_begin + rr;
        const int64_t rbase = row * H * acc_h;
        __nv_bfloat16* dp = a.dproj + row * a.nproj_ld;
        // ---- pair columns
        for (int e = tid; e < rdz; e += blockDim.x) {
            const int dd = e % dz;
            const float z2v = __ldg(a.z2 + row * rdz + e);
            float s1 = __ldg(a.dz1_epi + row * rdz + e), s2 = 0.f;
            for (int h0 = 0; h0 < H; h0 += 8) {
                // all 24 loads of the chunk issued before any use (the compiler otherwise waits
                // on each head's load in turn)
                float qq[8], kq[8], vq[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int h = min(h0 + u, H - 1);
                    qq[u] = acc_at<Q16>(a.dq_acc, a.dq16, rbase + h * acc_h + zq + e);
                    kq[u] = acc_at<ACC16>(a.dk_acc, a.dk16, rbase + h * acc_h + zq + e);
                    vq[u] = acc_at<ACC16>(a.dv_acc, a.dv16, rbase + h * acc_h + c + e);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int h = h0 + u;
                    if (h < H) {
                        const float k2 = kLn2 * kq[u];
                        s1 += qq[u];
                        s2 += s_wlb[h * dz + dd] * k2 + vq[u];
                        if (reg_dwlb) pw[(u + h0) % kPw] = fmaf(k2, z2v, pw[(u + h0) % kPw]);
                        else atomicAdd(&s_dwlb[h * dz + dd], k2 * z2v);
                    }
                }
            }
            a.dz1[row * rdz + e] = s1;
            a.dz2[row * rdz + e] = s2;
        }
        // ---- scalar columns (bf16 pairs)
        if (pairs) {
            constexpr int kBatch = 6;  // loads of kBatch iterations in flight before the stores
            const int total = 3 * H * half_c;
            for (int base = tid; base < total; base += kBatch * blockDim.x) {
                float2 v[kBatch];
                int dst[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    const int idx = min(base + u * static_cast<int>(blockDim.x), total - 1);
                    const int tsel = idx / (H * half_c), rem = idx - tsel * (H * half_c);
                    const int h = rem / half_c, cc = 2 * (rem - h * half_c);
                    const int64_t i = rbase + h * acc_h + cc;
                    v[u] = acc2_sel<ACC16, Q16>(a, tsel, i);
                    dst[u] = tsel * H * c + h * c + cc;
                    if (tsel == 1) {
                        v[u].x *= kscale;
                        v[u].y *= kscale;
                    }
                }
#pragma unroll
                for (int u = 0; u < kBatch; ++u)
                    if (base + u * static_cast<int>(blockDim.x) < total)
                        *reinterpret_cast<uint32_t*>(dp + dst[u]) = ptx_pack(v[u].x, v[u].y);
            }
        } else {
            for (int idx = tid; idx < 3 * H * c; idx += blockDim.x) {
                const int tsel = idx / (H * c), rem = idx - tsel * (H * c);
                const int h = rem / c, cc = rem - h * c;
                const int64_t i = rbase + h * acc_h + cc;
                const float x = tsel == 0 ? acc_at<Q16>(a.dq_acc, a.dq16, i)
                                          : (tsel == 1 ? acc_at<ACC16>(a.dk_acc, a.dk16, i) : acc_at<ACC16>(a.dv_acc, a.dv16, i));
                dp[tsel * H * c + h * c + cc] = __float2bfloat16_rn(x * (tsel == 1 ? kscale : 1.f));
            }
        }
        for (int e = d.n_proj + tid; e < a.nproj_ld; e += blockDim.x) dp[e] = __float2bfloat16_rn(0.f);
    }
    }  // groups
    if (reg_dwlb && tid < rdz) {
#pragma unroll
        for (int h = 0; h < kUnpackMaxH; ++h)
            if (h < H && h < kPw) atomicAdd(&s_dwlb[h * dz + tid % dz], pw[h]);
    }
    __syncthreads();
    for (int e = tid; e < H * dz; e += blockDim.x) atomicAdd(&a.dwlb[e], s_dwlb[e]);
}

// dOut with masked rows zeroed -> bf16, plus column sums (db_out).  Block = 64 columns x 32 rows:
// 16 threads cover a row's 64 columns with float4 loads (256 B contiguous), 16 row lanes stride the
// rows with all their loads independent; column partials reduced in shared memory, one atomic per
// column and block.
__global__ void __launch_bounds__(256) bwd_dout_kernel(const float* __restrict__ dout, const uint8_t* __restrict__ mask,
                                                       __nv_bfloat16* __restrict__ out, int ld_out, float* __restrict__ db,
                                                       int64_t rows, int cols, int rows_per_block) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    __shared__ float red[16][65];
    const int cq = threadIdx.x & 15, ry = threadIdx.x >> 4;
    const int col = blockIdx.x * 64 + 4 * cq;
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per_block;
    const int64_t r1 = min(rows, r0 + rows_per_block);
    const bool vec = col + 4 <= cols && (cols & 3) == 0 && (ld_out & 3) == 0;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    if (col < cols) {
#pragma unroll
        for (int64_t r = r0 + ry; r < r1; r += 16) {
            const bool ok = mask == nullptr || mask[r] != 0;
            float v[4];
            if (vec) {
                const float4 f = ok ? __ldg(reinterpret_cast<const float4*>(dout + r * cols + col))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                v[0] = f.x;
                v[1] = f.y;
                v[2] = f.z;
                v[3] = f.w;
                uint2 w;
                w.x = ptx_pack(v[0], v[1]);
                w.y = ptx_pack(v[2], v[3]);
                *reinterpret_cast<uint2*>(out + r * ld_out + col) = w;
            } else {
                for (int e = 0; e < 4; ++e) {
                    v[e] = (ok && col + e < cols) ? dout[r * cols + col + e] : 0.f;
                    if (col + e < cols) out[r * ld_out + col + e] = __float2bfloat16_rn(v[e]);
                }
            }
            a0 += v[0];
            a1 += v[1];
            a2 += v[2];
            a3 += v[3];
        }
    }
    red[ry][4 * cq] = a0;
    red[ry][4 * cq + 1] = a1;
    red[ry][4 * cq + 2] = a2;
    red[ry][4 * cq + 3] = a3;
    __syncthreads();
    if (threadIdx.x < 64) {
        const int c = blockIdx.x * 64 + threadIdx.x;
        if (c < cols) {
            float sum = 0.f;
#pragma unroll
            for (int k = 0; k < 16; ++k) sum += red[k][threadIdx.x];
            atomicAdd(&db[c], sum);
        }
    }
}

// Scatter the fused projection-weight gradient [d_in, n_proj] into the reference tensors
// w_q | w_k | w_v | w_qp | w_kp | w_vp (each [d_in, width], concatenated in `dst`).
// Scatter the fused projection-weight gradient [d_in, n_proj] into the reference tensors
// w_q | w_k | w_v | w_qp | w_kp | w_vp (each [d_in, width], concatenated in `dst`).  One block per
// source row: coalesced row read, per-column segment lookup with 32-bit arithmetic.
__global__ void scatter_proj_grad_kernel(const float* __restrict__ src, int d_in, int n_proj, ScatterCols seg,
                                         float* __restrict__ dst) {
    const int r = blockIdx.x;
    const float* srow = src + static_cast<int64_t>(r) * n_proj;
    for (int c = threadIdx.x; c < n_proj; c += blockDim.x) {
        int i = 0;
#pragma unroll
        for (int k = 1; k < 6; ++k) i += c >= seg.col0[k] ? 1 : 0;
        const int cc = c - seg.col0[i];
        dst[seg.dst_off[i] + static_cast<int64_t>(r) * seg.width[i] + cc] = srow[c];
    }
}

// The backward's last launch: the fused projection-weight gradient scattered into w_q .. w_vp
// (one block per source row, float4 when every segment is 4-aligned) plus the two tiny scalings
// d(w_bias) = w_l . d(w_l w_bias) and d(gamma_raw) = w_l w_c sigmoid(gamma_raw) . dg (the last
// block) -- one launch instead of three latency-bound ones.
__global__ void finish_weight_grads_kernel(const float* __restrict__ src, int d_in, int n_proj, ScatterCols seg,
                                           float* __restrict__ dst, int vec4, const float* __restrict__ red,
                                           const float* __restrict__ scale, int H, int dz, float* __restrict__ dw_bias,
                                           float* __restrict__ dgamma) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int r = blockIdx.x;
    if (r == d_in) {  // d(w_bias) [H, dz] and d(gamma_raw) [H]
        for (int e = threadIdx.x; e < H * dz; e += blockDim.x) dw_bias[e] = red[H + e] * scale[H];
        for (int e = threadIdx.x; e < H; e += blockDim.x) dgamma[e] = red[e] * scale[e];
        return;
    }
    const float* srow = src + static_cast<int64_t>(r) * n_proj;
    if (vec4) {
        for (int c = 4 * threadIdx.x; c < n_proj; c += 4 * blockDim.x) {
            int i = 0;
#pragma unroll
            for (int k = 1; k < 6; ++k) i += c >= seg.col0[k] ? 1 : 0;
            const int cc = c - seg.col0[i];
            *reinterpret_cast<float4*>(dst + seg.dst_off[i] + static_cast<int64_t>(r) * seg.width[i] + cc) =
                *reinterpret_cast<const float4*>(srow + c);
        }
        return;
    }
    for (int c = threadIdx.x; c < n_proj; c += blockDim.x) {
        int i = 0;
#pragma unroll
        for (int k = 1; k < 6; ++k) i += c >= seg.col0[k] ? 1 : 0;
        dst[seg.dst_off[i] + static_cast<int64_t>(r) * seg.width[i] + (c - seg.col0[i])] = srow[c];
    }
}

__global__ void bwd_recenter_kernel(const float* __restrict__ dtc, const uint8_t* __restrict__ mask,
                                    float* __restrict__ dt, int L) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    __shared__ float red[4][32];
    const int b = blockIdx.x;
    const float* g = dtc + int64_t(b) * L * 3;
    float sx = 0.f, sy = 0.f, sz = 0.f, cnt = 0.f;
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        if (mask == nullptr || mask[int64_t(b) * L + i] != 0) {
            sx += g[i * 3];
            sy += g[i * 3 + 1];
            sz += g[i * 3 + 2];
            cnt += 1.f;
        }
    }
    sx = warp_sum(sx);
    sy = warp_sum(sy);
    sz = warp_sum(sz);
    cnt = warp_sum(cnt);
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
        for (int k = 0; k < 4; ++k) {
            float v = l < nw ? red[k][l] : 0.f;
            v = warp_sum(v);
            if (l == 0) red[k][0] = v;
        }
    }
    __syncthreads();
    const float n = red[3][0] > 0.f ? red[3][0] : 1.f;
    const float mx = red[0][0] / n, my = red[1][0] / n, mz = red[2][0] / n;
    float* o = dt + int64_t(b) * L * 3;
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        const bool ok = mask == nullptr || mask[int64_t(b) * L + i] != 0;
        o[i * 3] = ok ? g[i * 3] - mx : 0.f;
        o[i * 3 + 1] = ok ? g[i * 3 + 1] - my : 0.f;
        o[i * 3 + 2] = ok ? g[i * 3 + 2] - mz : 0.f;
    }
}

__global__ void scale_vec_kernel(const float* in, const float* scale, int period, float* out, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[i] * scale[i % period];
}

}  // namespace

void launch_bwd_prep(const LayerDims& d, const BwdPrepArgs& a, cudaStream_t stream) {
    const int rdz = d.rank * d.d_z;
    const int64_t BL = int64_t(a.B) * a.L;
    const bool aligned = d.feat_ld % 4 == 0 && d.seg % 4 == 0;
    if (aligned && d.c == 128 && d.d_z == 128 && d.n_value == 12 && d.rank == 2 && d.dv_pad == 448) {
        launch_pdl(bwd_prep_warp_kernel<128, 128, 2, 12, 448>, dim3(static_cast<unsigned>((BL + 7) / 8)), dim3(256), 0,
                   stream, d, a);
        return;
    }
    if (aligned && d.c == 128 && d.d_z == 128 && d.n_value == 12 && d.rank == 1 && d.dv_pad == 320) {
        launch_pdl(bwd_prep_warp_kernel<128, 128, 1, 12, 320>, dim3(static_cast<unsigned>((BL + 7) / 8)), dim3(256), 0,
                   stream, d, a);
        return;
    }
    if (d.feat_ld % 8 || (d.dv_pad * 4) % 16 || d.dv_pad % 8)
        throw std::invalid_argument("bwd_prep: row strides must be multiples of 16 bytes");
    const size_t smem = sizeof(float) * (d.feat_ld + d.heads * d.dv_pad + ((rdz + 3) & ~3) +
                                         8 * (rdz + 12 + 3 * d.n_value)) +
                        16 + 2 * size_t(d.heads) * d.dv_pad + 16;
    if (smem > 48 * 1024) cudaFuncSetAttribute(bwd_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    bwd_prep_kernel<<<static_cast<unsigned>(int64_t(a.B) * a.L), 256, smem, stream>>>(d, a);
}

// The streaming kernel's fast form (see bwd_unpack_kernel): 256 threads, one pair column each.
bool unpack_fast(const LayerDims& d, int acc_ld, int nproj_ld) {
    const int rdz = d.rank * d.d_z;
    const bool pairs = d.c % 2 == 0 && acc_ld % 2 == 0 && nproj_ld % 2 == 0;
    return d.heads <= 8 && pairs && rdz == 256 && 3 * d.heads * (d.c / 2) <= 6 * 256;
}

void launch_bwd_unpack(const LayerDims& d, const BwdUnpackArgs& a, cudaStream_t stream) {
    if (std::max(d.dqk_used, d.dv_used) > a.acc_ld) throw std::invalid_argument("bwd_unpack: accumulator stride");
    if (d.heads > kUnpackMaxH) throw std::invalid_argument("bwd_unpack: at most 16 heads");
    if (d.n_query > 32 || d.n_value > 32) throw std::invalid_argument("bwd_unpack: at most 32 points per head");
    const int64_t BL = int64_t(a.B) * a.L;
    // (running the geometry inside the streaming kernel's group loop measured slower: 0.134 vs
    // 0.114 ms -- it serialises behind the streaming loads and spills at the 128-register cap)
    launch_pdl(bwd_unpack_geo_kernel, dim3(static_cast<unsigned>((BL + 7) / 8)), dim3(256), 0, stream, d, a);
    const size_t smem = sizeof(float) * 2 * size_t(d.heads) * d.d_z;
    if ((a.dk16 == nullptr) != (a.dv16 == nullptr)) throw std::invalid_argument("bwd_unpack: dk16 and dv16 go together");
    const bool fast = unpack_fast(d, a.acc_ld, a.nproj_ld);
    using K = void (*)(LayerDims, BwdUnpackArgs);
    const K kerns[8] = {bwd_unpack_kernel<false, false, false>, bwd_unpack_kernel<false, false, true>,
                        bwd_unpack_kernel<false, true, false>,  bwd_unpack_kernel<false, true, true>,
                        bwd_unpack_kernel<true, false, false>,  bwd_unpack_kernel<true, false, true>,
                        bwd_unpack_kernel<true, true, false>,   bwd_unpack_kernel<true, true, true>};
    const K kern = kerns[(a.dk16 != nullptr ? 4 : 0) + (a.dq16 != nullptr ? 2 : 0) + (fast ? 1 : 0)];
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    const int sms = device_sm_count();
    const int64_t groups = (BL + kUnpackRows - 1) / kUnpackRows;
    const int64_t grid = std::min<int64_t>(groups, int64_t(sms) * 2);  // 2 resident blocks per SM
    launch_pdl(kern, dim3(static_cast<unsigned>(grid)), dim3(256), smem, stream, d, a);
}

// Streaming row kernels of the materialised backward: one block per (sample, head, query) row, 8
// columns per thread and step (two float4 / one uint4 per operand).  Same rounding as the fused
// kernels: lse2 = __fmul_rn(lse, log2 e), P = ex2(S - lse2) rounded to bf16, dS = P (dP - D).
__global__ void __launch_bounds__(256) dense_softmax_kernel(const float* __restrict__ S, int ld,
                                                            const float* __restrict__ lse, int L,
                                                            __nv_bfloat16* __restrict__ P) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int64_t row = blockIdx.x;
    const float l = __ldg(lse + row);
    const bool none = !(l > -INFINITY);
    const float l2 = none ? 0.f : __fmul_rn(l, kL2E);
    const float* s = S + row * ld;
    __nv_bfloat16* p = P + row * ld;
    for (int c = threadIdx.x * 8; c < L; c += blockDim.x * 8) {
        const float4 a = *reinterpret_cast<const float4*>(s + c);
        const float4 b = *reinterpret_cast<const float4*>(s + c + 4);
        const float x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            w[k] = none ? 0u : ptx::pack_bf16x2(ptx::ex2(x[2 * k] - l2), ptx::ex2(x[2 * k + 1] - l2));
        *reinterpret_cast<uint4*>(p + c) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

__global__ void __launch_bounds__(256) dense_ds_kernel(const __nv_bfloat16* __restrict__ P,
                                                       const float* __restrict__ dP, int ld,
                                                       const float* __restrict__ Dvec, int L,
                                                       __nv_bfloat16* __restrict__ dS) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int64_t row = blockIdx.x;
    const float D = __ldg(Dvec + row);
    const __nv_bfloat16* p = P + row * ld;
    const float* g = dP + row * ld;
    __nv_bfloat16* o = dS + row * ld;
    for (int c = threadIdx.x * 8; c < L; c += blockDim.x * 8) {
        const uint4 pw = *reinterpret_cast<const uint4*>(p + c);
        const float4 a = *reinterpret_cast<const float4*>(g + c);
        const float4 b = *reinterpret_cast<const float4*>(g + c + 4);
        const uint32_t pv[4] = {pw.x, pw.y, pw.z, pw.w};
        const float x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            w[k] = ptx::pack_bf16x2(__uint_as_float(pv[k] << 16) * (x[2 * k] - D),
                                    __uint_as_float(pv[k] & 0xFFFF0000u) * (x[2 * k + 1] - D));
        *reinterpret_cast<uint4*>(o + c) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

void launch_dense_softmax(const float* S, int ld, const float* lse, int64_t rows, int L, __nv_bfloat16* P,
                          cudaStream_t stream) {
    if (ld % 8 != 0 || ld < L) throw std::invalid_argument("dense softmax: row stride must be >= L and % 8");
    launch_pdl(dense_softmax_kernel, dim3(static_cast<unsigned>(rows)), dim3(std::min(256, (L + 7) / 8 + 31) / 32 * 32),
               0, stream, S, ld, lse, L, P);
}

void launch_dense_ds(const __nv_bfloat16* P, const float* dP, int ld, const float* Dvec, int64_t rows, int L,
                     __nv_bfloat16* dS, cudaStream_t stream) {
    if (ld % 8 != 0 || ld < L) throw std::invalid_argument("dense dS: row stride must be >= L and % 8");
    launch_pdl(dense_ds_kernel, dim3(static_cast<unsigned>(rows)), dim3(std::min(256, (L + 7) / 8 + 31) / 32 * 32), 0,
               stream, P, dP, ld, Dvec, L, dS);
}

void launch_bwd_dout(const float* dout, const uint8_t* mask, __nv_bfloat16* out, int ld_out, float* db,
                     int64_t rows, int cols, cudaStream_t stream) {
    const int rpb = 32;  // 2 rows per thread: 4x the blocks of 128-row tiles, loads all in flight
    dim3 grid((cols + 63) / 64, static_cast<unsigned>((rows + rpb - 1) / rpb));
    launch_pdl(bwd_dout_kernel, grid, dim3(256), 0, stream, dout, mask, out, ld_out, db, rows, cols, rpb);
}

void launch_scatter_proj_grad(const float* src, int d_in, int n_proj, const ScatterCols& seg, float* dst,
                              cudaStream_t stream) {
    scatter_proj_grad_kernel<<<static_cast<unsigned>(d_in), 256, 0, stream>>>(src, d_in, n_proj, seg, dst);
}

void launch_finish_weight_grads(const float* src, int d_in, int n_proj, const ScatterCols& seg, float* dst,
                                const float* red, const float* scale, int H, int dz, float* dw_bias, float* dgamma,
                                cudaStream_t stream) {
    bool vec4 = n_proj % 4 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
    for (int i = 0; i < 6; ++i) vec4 = vec4 && seg.col0[i] % 4 == 0 && seg.width[i] % 4 == 0 && seg.dst_off[i] % 4 == 0;
    launch_pdl(finish_weight_grads_kernel, dim3(static_cast<unsigned>(d_in + 1)), dim3(256), 0, stream, src, d_in, n_proj,
               seg, dst, vec4 ? 1 : 0, red, scale, H, dz, dw_bias, dgamma);
}

void launch_bwd_recenter(const float* dt_c, const uint8_t* mask, float* dt, int B, int L, cudaStream_t stream) {
    launch_pdl(bwd_recenter_kernel, dim3(B), dim3(1024), 0, stream, dt_c, mask, dt, L);
}

void launch_scale_vec(const float* in, const float* scale, int period, float* out, int n, cudaStream_t stream) {
    if (n > 0) scale_vec_kernel<<<(n + 255) / 256, 256, 0, stream>>>(in, scale, period, out, n);
}

}  // namespace fipa_b200
