// Quadratic-memory arms on the GPU and the reference's generic attention entry
// points.  These are the baselines the linear-memory path is compared against, so they
// deliberately materialise what the reference materialises:
//   naive_attention      proj/src/attention_kernel.cpp:192-211  logits [H, L, L] -> softmax -> P.V
//   flash_attention      proj/src/attention_kernel.cpp:213-243  online softmax, O(L) memory
//   reference_forward    proj/src/ipa.cpp:244-310               dense pair tensor z [L, L, d_z],
//                        logits [H, L, L], softmax, aggregation (attention x z / v / points)
// All fp32 on CUDA cores: generic shapes (any d, +-700 logits in the reference tests) and the
// 1e-4 gate.  The dense IPA arm is the paper's Fig. 2 comparison (memory and time vs L).
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>
#include <stdexcept>

#include "kernels.hpp"

namespace fipa_b200 {

namespace {

// ------------------------------------------------------------------ batched fp32 GEMM
// C[b] = A[b] (M x K, row-major, lda) . op(B[b]) ; op(B) = B (K x N, ldb) or B^T (B is N x K).
constexpr int GM = 64, GN = 64, GK = 16;

__global__ void __launch_bounds__(256) gemm_f32_strided_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                               float* __restrict__ C, int M, int N, int K, int64_t lda,
                                                               int64_t ldb, int64_t ldc, int64_t sA, int64_t sB,
                                                               int64_t sC, bool transB) {
    __shared__ float sAt[GK][GM + 4];
    __shared__ float sBt[GK][GN + 4];
    const int64_t bz = blockIdx.z;
    A += bz * sA;
    B += bz * sB;
    C += bz * sC;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int m0 = blockIdx.y * GM, n0 = blockIdx.x * GN;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += GK) {
        for (int e = threadIdx.x; e < GM * GK; e += 256) {
            const int r = e / GK, kk = e % GK;
            const int gm = m0 + r, gk = k0 + kk;
            sAt[kk][r] = (gm < M && gk < K) ? A[gm * lda + gk] : 0.f;
        }
        if (transB) {
            for (int e = threadIdx.x; e < GN * GK; e += 256) {
                const int n = e / GK, kk = e % GK;
                const int gn = n0 + n, gk = k0 + kk;
                sBt[kk][n] = (gk < K && gn < N) ? B[gn * ldb + gk] : 0.f;
            }
        } else {
            for (int e = threadIdx.x; e < GN * GK; e += 256) {
                const int kk = e / GN, n = e % GN;
                const int gk = k0 + kk, gn = n0 + n;
                sBt[kk][n] = (gk < K && gn < N) ? B[gk * ldb + gn] : 0.f;
            }
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < GK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = sAt[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = sBt[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gm = m0 + ty * 4 + i;
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gn = n0 + tx * 4 + j;
            if (gn < N) C[gm * ldc + gn] = acc[i][j];
        }
    }
}

void gemm_strided(const float* A, const float* B, float* C, int M, int N, int K, int64_t lda, int64_t ldb,
                  int64_t ldc, int64_t sA, int64_t sB, int64_t sC, int batch, bool transB, cudaStream_t st) {
    if (M <= 0 || N <= 0 || batch <= 0) return;
    for (int b0 = 0; b0 < batch; b0 += 65535) {
        const int nb = batch - b0 < 65535 ? batch - b0 : 65535;
        dim3 grid((N + GN - 1) / GN, (M + GM - 1) / GM, nb);
        gemm_f32_strided_kernel<<<grid, 256, 0, st>>>(A + b0 * sA, B + b0 * sB, C + b0 * sC, M, N, K, lda, ldb, ldc,
                                                      sA, sB, sC, transB);
    }
}

// ------------------------------------------------------------------ row softmax (in place)
// rows of length L grouped `rows_per_mask` to a key mask row; masked keys get zero weight,
// rows without a valid key become zeros (attention_kernel.cpp:140-143, 184-186).
__global__ void __launch_bounds__(256) softmax_rows_kernel(float* __restrict__ x, int64_t L, int64_t rows_per_mask,
                                                           const uint8_t* __restrict__ mask) {
    __shared__ float red[32];
    const int64_t row = blockIdx.x;
    float* xr = x + row * L;
    const uint8_t* mr = mask ? mask + (row / rows_per_mask) * L : nullptr;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float m = -INFINITY;
    for (int64_t j = threadIdx.x; j < L; j += blockDim.x)
        if (!mr || mr[j]) m = fmaxf(m, xr[j]);
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) red[warp] = m;
    __syncthreads();
    if (warp == 0) {
        float v = lane < (blockDim.x >> 5) ? red[lane] : -INFINITY;
        for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) red[0] = v;
    }
    __syncthreads();
    m = red[0];
    __syncthreads();
    float s = 0.f;
    for (int64_t j = threadIdx.x; j < L; j += blockDim.x) {
        const float p = (m != -INFINITY && (!mr || mr[j])) ? expf(xr[j] - m) : 0.f;
        xr[j] = p;
        s += p;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (warp == 0) {
        float v = lane < (blockDim.x >> 5) ? red[lane] : 0.f;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[0] = v;
    }
    __syncthreads();
    const float inv = red[0] > 0.f ? 1.f / red[0] : 0.f;
    for (int64_t j = threadIdx.x; j < L; j += blockDim.x) xr[j] *= inv;
}

// ------------------------------------------------------------------ generic flash attention
// One block = 32 query rows of one head; keys stream in tiles of 64; Q/K stream through shared
// memory in 32-wide column chunks (any d_qk); the O accumulator [32][d_v] lives in shared memory.
constexpr int FBM = 32, FBN = 64, FDC = 32;

__global__ void __launch_bounds__(256) flash_f32_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                                        const float* __restrict__ v, const uint8_t* __restrict__ mask,
                                                        float* __restrict__ out, int L, int dqk, int dv, int dv_ld) {
    extern __shared__ float fsm[];
    float* Qc = fsm;                     // [FBM][FDC + 1]
    float* Kc = Qc + FBM * (FDC + 1);    // [FBN][FDC + 1]
    float* Ps = Kc + FBN * (FDC + 1);    // [FBM][FBN + 1]
    float* Vc = Ps + FBM * (FBN + 1);    // [FBN][64 + 4]
    float* rs = Vc + FBN * 68;           // [FBM] rescale
    float* O = rs + FBM;                 // [FBM][dv_ld]
    const int h = blockIdx.y;
    const int q0 = blockIdx.x * FBM;
    const float* qh = q + static_cast<int64_t>(h) * L * dqk;
    const float* kh = k + static_cast<int64_t>(h) * L * dqk;
    const float* vh = v + static_cast<int64_t>(h) * L * dv;
    const int t = threadIdx.x;
    for (int e = t; e < FBM * dv_ld; e += 256) O[e] = 0.f;
    // S micro-tile: rows 2*sy, 2*sy+1; keys 4*sx .. 4*sx+3
    const int sy = t / 16, sx = t % 16;
    // softmax: 8 threads per row
    const int srow = t / 8, spart = t % 8;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j0 = 0; j0 < L; j0 += FBN) {
        float acc[2][4] = {};
        for (int d0 = 0; d0 < dqk; d0 += FDC) {
            __syncthreads();
            for (int e = t; e < FBM * FDC; e += 256) {
                const int r = e / FDC, c = e % FDC;
                Qc[r * (FDC + 1) + c] = (q0 + r < L && d0 + c < dqk) ? qh[static_cast<int64_t>(q0 + r) * dqk + d0 + c] : 0.f;
            }
            for (int e = t; e < FBN * FDC; e += 256) {
                const int r = e / FDC, c = e % FDC;
                Kc[r * (FDC + 1) + c] = (j0 + r < L && d0 + c < dqk) ? kh[static_cast<int64_t>(j0 + r) * dqk + d0 + c] : 0.f;
            }
            __syncthreads();
#pragma unroll 8
            for (int c = 0; c < FDC; ++c) {
                const float a0 = Qc[(2 * sy) * (FDC + 1) + c], a1 = Qc[(2 * sy + 1) * (FDC + 1) + c];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const float b = Kc[(4 * sx + jj) * (FDC + 1) + c];
                    acc[0][jj] = fmaf(a0, b, acc[0][jj]);
                    acc[1][jj] = fmaf(a1, b, acc[1][jj]);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int j = j0 + 4 * sx + jj;
                const bool valid = j < L && (!mask || mask[j]);
                Ps[(2 * sy + i) * (FBN + 1) + 4 * sx + jj] = valid ? acc[i][jj] : -INFINITY;
            }
        __syncthreads();
        // online softmax of row srow (8 keys per thread), rescale factor for O
        {
            float x[8], mx = -INFINITY;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                x[e] = Ps[srow * (FBN + 1) + spart * 8 + e];
                mx = fmaxf(mx, x[e]);
            }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            const float m_new = fmaxf(m_run, mx);
            const float scale = m_new == -INFINITY ? 1.f : expf(m_run - m_new);
            float ps = 0.f;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const float p = m_new == -INFINITY ? 0.f : expf(x[e] - m_new);
                Ps[srow * (FBN + 1) + spart * 8 + e] = p;
                ps += p;
            }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
            l_run = l_run * scale + ps;
            m_run = m_new;
            if (spart == 0) rs[srow] = scale;
        }
        // O = O * scale + P . V_tile, 64 value columns at a time (thread: 2 rows x 4 columns)
        for (int c0 = 0; c0 < dv; c0 += 64) {
            __syncthreads();
            for (int e = t; e < FBN * 64; e += 256) {
                const int r = e / 64, c = e % 64;
                Vc[r * 68 + c] = (j0 + r < L && c0 + c < dv) ? vh[static_cast<int64_t>(j0 + r) * dv + c0 + c] : 0.f;
            }
            __syncthreads();
            float o[2][4];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const int cc = c0 + 4 * sx + jj;
                    o[i][jj] = cc < dv_ld ? O[(2 * sy + i) * dv_ld + cc] * rs[2 * sy + i] : 0.f;
                }
#pragma unroll 8
            for (int kk = 0; kk < FBN; ++kk) {
                const float p0 = Ps[(2 * sy) * (FBN + 1) + kk], p1 = Ps[(2 * sy + 1) * (FBN + 1) + kk];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const float b = Vc[kk * 68 + 4 * sx + jj];
                    o[0][jj] = fmaf(p0, b, o[0][jj]);
                    o[1][jj] = fmaf(p1, b, o[1][jj]);
                }
            }
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const int cc = c0 + 4 * sx + jj;
                    if (cc < dv_ld) O[(2 * sy + i) * dv_ld + cc] = o[i][jj];
                }
        }
    }
    __syncthreads();
    if (spart == 0) rs[srow] = l_run > 0.f ? 1.f / l_run : 0.f;
    __syncthreads();
    float* oh = out + static_cast<int64_t>(h) * L * dv;
    for (int e = t; e < FBM * dv; e += 256) {
        const int r = e / dv, c = e % dv;
        if (q0 + r < L) oh[static_cast<int64_t>(q0 + r) * dv + c] = O[r * dv_ld + c] * rs[r];
    }
}

int flash_dv_ld(int dv) { return (dv + 63) / 64 * 64 + 1; }
size_t flash_smem(int dv) {
    return sizeof(float) *
           (FBM * (FDC + 1) + FBN * (FDC + 1) + FBM * (FBN + 1) + FBN * 68 + FBM + static_cast<size_t>(FBM) * flash_dv_ld(dv));
}

// ------------------------------------------------------------------ dense IPA arm
// Global points (apply, geometry.cpp:63-68) and the per-head value rows [v | T_j v_p].
__global__ void dense_points_kernel(const float* __restrict__ proj, const float* __restrict__ rot,
                                    const float* __restrict__ trans, int64_t BL, int L, int H, int c, int Nq,
                                    int Nv, int n_proj, float* __restrict__ gq, float* __restrict__ gk,
                                    float* __restrict__ vcat) {
    const int64_t r = blockIdx.x;  // residue b*L + i
    if (r >= BL) return;
    const float* pr = proj + r * n_proj;
    const float* R = rot + r * 9;
    const float* tt = trans + r * 3;
    const int vw = c + 3 * Nv;
    const int64_t b = r / L, i = r % L;
    for (int e = threadIdx.x; e < H * (2 * Nq + Nv); e += blockDim.x) {
        const float* src;
        float* dst;
        int h;
        if (e < H * Nq) {
            h = e / Nq;
            src = pr + 3 * H * c + 3 * e;
            dst = gq + r * (H * Nq * 3) + 3 * e;
        } else if (e < 2 * H * Nq) {
            const int ee = e - H * Nq;
            h = ee / Nq;
            src = pr + 3 * H * c + 3 * H * Nq + 3 * ee;
            dst = gk + r * (H * Nq * 3) + 3 * ee;
        } else {
            const int ee = e - 2 * H * Nq;
            h = ee / Nv;
            const int p = ee % Nv;
            src = pr + 3 * H * c + 6 * H * Nq + 3 * ee;
            dst = vcat + ((b * H + h) * L + i) * vw + c + 3 * p;
        }
        (void)h;
        const float x = src[0], y = src[1], z = src[2];
        dst[0] = fmaf(R[0], x, fmaf(R[1], y, R[2] * z)) + tt[0];
        dst[1] = fmaf(R[3], x, fmaf(R[4], y, R[5] * z)) + tt[1];
        dst[2] = fmaf(R[6], x, fmaf(R[7], y, R[8] * z)) + tt[2];
    }
    for (int e = threadIdx.x; e < H * c; e += blockDim.x) {
        const int h = e / c, ch = e % c;
        vcat[((b * H + h) * L + i) * vw + ch] = pr[2 * H * c + e];
    }
}

// z[b,i,j,:] = sum_rho z1[b,i,rho,:] * z2[b,j,rho,:]   (dense_pair_from_factors)
__global__ void dense_pair_kernel(const float* __restrict__ z1, const float* __restrict__ z2, int L, int r, int dz,
                                  float* __restrict__ z) {
    const int64_t b = blockIdx.z, i = blockIdx.y;
    const int64_t j0 = static_cast<int64_t>(blockIdx.x) * 8;
    const float* a = z1 + (b * L + i) * r * dz;
    for (int jj = 0; jj < 8; ++jj) {
        const int64_t j = j0 + jj;
        if (j >= L) break;
        const float* bb = z2 + (b * L + j) * r * dz;
        float* dst = z + ((b * L + i) * L + j) * dz;
        for (int d = threadIdx.x; d < dz; d += blockDim.x) {
            float acc = 0.f;
            for (int rho = 0; rho < r; ++rho) acc = fmaf(a[rho * dz + d], bb[rho * dz + d], acc);
            dst[d] = acc;
        }
    }
}

// logits[b,h,i,j] = w_l q.k/sqrt(c) + sum_d z_ijd w_l w_bias[h,d] - g_h/2 sum_p |T_i q_p - T_j k_p|^2
// (ipa.hpp:62-64, ipa.cpp:95-96).  16 x 16 (i, j) tile per block, all heads.
constexpr int kDenseMaxH = 16;
__global__ void __launch_bounds__(256) dense_logits_kernel(const float* __restrict__ proj, const float* __restrict__ gq,
                                                           const float* __restrict__ gk, const float* __restrict__ z,
                                                           const float* __restrict__ head_g,
                                                           const float* __restrict__ wl_bias, float k_scale, int L,
                                                           int H, int c, int Nq, int dz, int n_proj,
                                                           float* __restrict__ logits) {
    extern __shared__ float dsm[];
    float* qs = dsm;                 // [16][33]
    float* ks = qs + 16 * 33;        // [16][33]
    float* wb = ks + 16 * 33;        // [H][dz]
    float* pq = wb + H * dz;         // [16][H*Nq*3]
    float* pk = pq + 16 * H * Nq * 3;
    const int64_t b = blockIdx.z;
    const int i0 = blockIdx.y * 16, j0 = blockIdx.x * 16;
    const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
    const int i = i0 + ty, j = j0 + tx;
    const int np = H * Nq * 3;
    for (int e = threadIdx.x; e < H * dz; e += 256) wb[e] = wl_bias[e];
    for (int e = threadIdx.x; e < 16 * np; e += 256) {
        const int rr = e / np, cc = e % np;
        pq[e] = (i0 + rr < L) ? gq[(b * L + i0 + rr) * np + cc] : 0.f;
        pk[e] = (j0 + rr < L) ? gk[(b * L + j0 + rr) * np + cc] : 0.f;
    }
    __syncthreads();
    float lg[kDenseMaxH];
#pragma unroll
    for (int h = 0; h < kDenseMaxH; ++h) lg[h] = 0.f;
    // pair bias: one pass over z_ij for every head
    if (i < L && j < L) {
        const float* zr = z + ((b * L + i) * L + j) * dz;
        for (int d = 0; d < dz; ++d) {
            const float zv = zr[d];
#pragma unroll
            for (int h = 0; h < kDenseMaxH; ++h)
                if (h < H) lg[h] = fmaf(zv, wb[h * dz + d], lg[h]);
        }
    }
    // scalar q.k per head, 32-wide chunks through shared memory
    for (int h = 0; h < H; ++h) {
        float qk = 0.f;
        for (int d0 = 0; d0 < c; d0 += 32) {
            __syncthreads();
            for (int e = threadIdx.x; e < 16 * 32; e += 256) {
                const int rr = e / 32, cc = e % 32;
                qs[rr * 33 + cc] = (i0 + rr < L && d0 + cc < c) ? proj[(b * L + i0 + rr) * n_proj + h * c + d0 + cc] : 0.f;
                ks[rr * 33 + cc] =
                    (j0 + rr < L && d0 + cc < c) ? proj[(b * L + j0 + rr) * n_proj + H * c + h * c + d0 + cc] : 0.f;
            }
            __syncthreads();
#pragma unroll 8
            for (int cc = 0; cc < 32; ++cc) qk = fmaf(qs[ty * 33 + cc], ks[tx * 33 + cc], qk);
        }
        float dist = 0.f;
        for (int p = 0; p < Nq; ++p) {
            const float* a = pq + ty * np + (h * Nq + p) * 3;
            const float* bb = pk + tx * np + (h * Nq + p) * 3;
            const float dx = a[0] - bb[0], dy = a[1] - bb[1], dzz = a[2] - bb[2];
            dist = fmaf(dx, dx, fmaf(dy, dy, fmaf(dzz, dzz, dist)));
        }
        float bias = 0.f;
#pragma unroll
        for (int hh = 0; hh < kDenseMaxH; ++hh)
            if (hh == h) bias = lg[hh];
        if (i < L && j < L)
            logits[((b * H + h) * L + i) * L + j] = fmaf(k_scale, qk, bias) - 0.5f * head_g[h] * dist;
    }
}

// oz[b,i,h,:] = sum_j P[b,h,i,j] z[b,i,j,:]  (aggregate_core's pair term): block per (b, i).
__global__ void __launch_bounds__(128) dense_pair_aggregate_kernel(const float* __restrict__ P, const float* __restrict__ z,
                                                                   int L, int H, int dz, float* __restrict__ oz) {
    __shared__ float ps[kDenseMaxH][64];
    const int64_t b = blockIdx.y, i = blockIdx.x;
    float acc[kDenseMaxH][2];
#pragma unroll
    for (int h = 0; h < kDenseMaxH; ++h) acc[h][0] = acc[h][1] = 0.f;
    const float* zi = z + (b * L + i) * static_cast<int64_t>(L) * dz;
    for (int j0 = 0; j0 < L; j0 += 64) {
        __syncthreads();
        for (int e = threadIdx.x; e < H * 64; e += 128) {
            const int h = e / 64, jj = e % 64;
            ps[h][jj] = (j0 + jj < L) ? P[((b * H + h) * L + i) * static_cast<int64_t>(L) + j0 + jj] : 0.f;
        }
        __syncthreads();
        const int jn = min(64, L - j0);
        for (int jj = 0; jj < jn; ++jj) {
            const float* zr = zi + static_cast<int64_t>(j0 + jj) * dz;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int d = threadIdx.x + 128 * u;
                if (d < dz) {
                    const float zv = zr[d];
#pragma unroll
                    for (int h = 0; h < kDenseMaxH; ++h)
                        if (h < H) acc[h][u] = fmaf(ps[h][jj], zv, acc[h][u]);
                }
            }
        }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int d = threadIdx.x + 128 * u;
        if (d < dz)
#pragma unroll
            for (int h = 0; h < kDenseMaxH; ++h)
                if (h < H) oz[((b * L + i) * H + h) * dz + d] = acc[h][u];
    }
}

// feature block per head: [oz | scalar | R_i^T (g - t_i) | |.|]   (aggregate_core + apply_inverse)
__global__ void dense_feat_kernel(const float* __restrict__ oz, const float* __restrict__ ov,
                                  const float* __restrict__ rot, const float* __restrict__ trans, int L, int H,
                                  int c, int Nv, int dz, int feat_ld, float* __restrict__ feat) {
    const int64_t r = blockIdx.x;  // b*L + i
    const int64_t b = r / L, i = r % L;
    const int seg = dz + c + 4 * Nv, vw = c + 3 * Nv;
    const float* R = rot + r * 9;
    const float* tt = trans + r * 3;
    float* fr = feat + r * feat_ld;
    for (int e = threadIdx.x; e < H * seg; e += blockDim.x) {
        const int h = e / seg, k = e % seg;
        const float* ovr = ov + ((b * H + h) * L + i) * vw;
        float val;
        if (k < dz) {
            val = oz[(r * H + h) * dz + k];
        } else if (k < dz + c) {
            val = ovr[k - dz];
        } else {
            const int kk = k - dz - c;
            const int p = kk < 3 * Nv ? kk / 3 : kk - 3 * Nv;
            const float gx = ovr[c + 3 * p] - tt[0], gy = ovr[c + 3 * p + 1] - tt[1], gz = ovr[c + 3 * p + 2] - tt[2];
            const float lx = fmaf(R[0], gx, fmaf(R[3], gy, R[6] * gz));
            const float ly = fmaf(R[1], gx, fmaf(R[4], gy, R[7] * gz));
            const float lz = fmaf(R[2], gx, fmaf(R[5], gy, R[8] * gz));
            if (kk < 3 * Nv) {
                const int a = kk % 3;
                val = a == 0 ? lx : (a == 1 ? ly : lz);
            } else {
                val = sqrtf(lx * lx + ly * ly + lz * lz);
            }
        }
        fr[e] = val;
    }
}

}  // namespace

// ------------------------------------------------------------------ host launchers
void launch_naive_attention_f32(int H, int L, int dqk, int dv, const float* q, const float* k, const float* v,
                                const uint8_t* mask, float* logits, float* out, cudaStream_t st) {
    gemm_strided(q, k, logits, L, L, dqk, dqk, dqk, L, int64_t(L) * dqk, int64_t(L) * dqk, int64_t(L) * L, H, true, st);
    softmax_rows_kernel<<<static_cast<unsigned>(int64_t(H) * L), 256, 0, st>>>(logits, L, int64_t(H) * L, mask);
    gemm_strided(logits, v, out, L, dv, L, L, dv, dv, int64_t(L) * L, int64_t(L) * dv, int64_t(L) * dv, H, false, st);
}

bool flash_attention_f32_supported(int dv) { return flash_smem(dv) <= 200 * 1024; }

void launch_flash_attention_f32(int H, int L, int dqk, int dv, const float* q, const float* k, const float* v,
                                const uint8_t* mask, float* out, cudaStream_t st) {
    if (!flash_attention_f32_supported(dv)) throw std::invalid_argument("flash_attention: value width too large");
    const size_t smem = flash_smem(dv);
    cudaFuncSetAttribute(flash_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    dim3 grid((L + FBM - 1) / FBM, H);
    flash_f32_kernel<<<grid, 256, smem, st>>>(q, k, v, mask, out, L, dqk, dv, flash_dv_ld(dv));
}

void launch_dense_ipa(const LayerDims& d, const DenseArgs& a, cudaStream_t st) {
    const int B = a.B, L = a.L, H = d.heads, c = d.c, Nq = d.n_query, Nv = d.n_value, dz = d.d_z, r = d.rank;
    if (H > kDenseMaxH || dz > 256) throw std::invalid_argument("dense arm: heads <= 16 and d_z <= 256");
    const int64_t BL = int64_t(B) * L;
    const int vw = c + 3 * Nv;
    launch_gemm_f32(a.s, d.d_in, a.wproj, a.proj, int(BL), d.n_proj, d.d_in, nullptr, nullptr, st);
    dense_points_kernel<<<static_cast<unsigned>(BL), 128, 0, st>>>(a.proj, a.rot, a.trans, BL, L, H, c, Nq, Nv,
                                                                   d.n_proj, a.gq, a.gk, a.vcat);
    dense_pair_kernel<<<dim3((L + 7) / 8, L, B), 128, 0, st>>>(a.z1, a.z2, L, r, dz, a.z);
    const size_t lsm = sizeof(float) * (2 * 16 * 33 + H * dz + 2 * 16 * H * Nq * 3);
    cudaFuncSetAttribute(dense_logits_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(lsm));
    dense_logits_kernel<<<dim3((L + 15) / 16, (L + 15) / 16, B), 256, lsm, st>>>(
        a.proj, a.gq, a.gk, a.z, a.head_g, a.wl_bias, a.k_scale, L, H, c, Nq, dz, d.n_proj, a.logits);
    softmax_rows_kernel<<<static_cast<unsigned>(BL * H), 256, 0, st>>>(a.logits, L, int64_t(H) * L, a.mask);
    gemm_strided(a.logits, a.vcat, a.ov, L, vw, L, L, vw, vw, int64_t(L) * L, int64_t(L) * vw, int64_t(L) * vw, B * H,
                 false, st);
    dense_pair_aggregate_kernel<<<dim3(L, B), 128, 0, st>>>(a.logits, a.z, L, H, dz, a.oz);
    dense_feat_kernel<<<static_cast<unsigned>(BL), 256, 0, st>>>(a.oz, a.ov, a.rot, a.trans, L, H, c, Nv, dz, d.feat,
                                                                 a.feat);
    launch_gemm_f32(a.feat, d.feat, a.wout, a.out, int(BL), d.d_in, d.feat, a.bout, a.mask, st);
}

}  // namespace fipa_b200
