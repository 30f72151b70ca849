// Pipeline trace + timing of the attention backward kernels (cluster 0 of (sample, head) 0),
// north-star shape, random lifted rows.  Build: see tools/README (nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2505_11580_b200/csrc).
#define FIPA_ATTN_BWD_TRACE 1
#define FIPA_SPAN_TRACE 1
#include "../paper_2505_11580_b200/csrc/attn_bwd.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "span_summary.hpp"

using namespace fipa_b200;

int main(int argc, char** argv) {
    const int B = argc > 1 ? atoi(argv[1]) : 8;
    const int L = argc > 2 ? atoi(argv[2]) : 1024;
    const int which = argc > 3 ? atoi(argv[3]) : 1;
    LayerDims d{};
    d.d_in = 256; d.d_z = 128; d.heads = 8; d.c = 128; d.n_query = 8; d.n_value = 12; d.rank = 2;
    d.zq = 176; d.dqk_used = 176 + 256; d.dqk_mma = 432; d.dqk_pad = 448;
    d.dv_used = 128 + 256 + 36 + 6; d.dv_mma = 432; d.dv_pad = 448;
    const size_t BH = size_t(B) * d.heads;
    std::vector<__nv_bfloat16> hq(BH * L * 448);
    std::vector<float> hl(BH * L);
    srand(1);
    for (auto& x : hq) x = __float2bfloat16((rand() / float(RAND_MAX) - 0.5f) * 0.2f);
    for (auto& x : hl) x = 3.0f + rand() / float(RAND_MAX);
    __nv_bfloat16 *q, *k, *v, *dO;
    float *lse, *D, *acc;
    const size_t rows = BH * L * 448 * 2;
    cudaMalloc(&q, rows); cudaMalloc(&k, rows); cudaMalloc(&v, rows); cudaMalloc(&dO, rows);
    cudaMalloc(&lse, BH * L * 4); cudaMalloc(&D, BH * L * 4);
    cudaMalloc(&acc, 3 * BH * L * 448 * 4);
    for (auto* p : {q, k, v, dO}) cudaMemcpy(p, hq.data(), rows, cudaMemcpyHostToDevice);
    cudaMemcpy(lse, hl.data(), BH * L * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(D, hl.data(), BH * L * 4, cudaMemcpyHostToDevice);
    AttnBwdArgs a{q, k, v, dO, lse, D, acc, acc + BH * L * 448, acc + 2 * BH * L * 448, 448, B, L};
    if (argc > 4 && atoi(argv[4]) == 1) {  // materialised dS (the default path at L <= 2048)
        a.ds_ld = (L + 63) / 64 * 64;
        cudaMalloc(&a.ds, BH * L * size_t(a.ds_ld) * 2);
    }
    if (argc > 5) sscanf(argv[5], "%d,%d,%d,%d,%d", &a.ring[0], &a.ring[1], &a.ring[2], &a.ring[3], &a.ring[4]);
    if (!(argc > 6 && atoi(argv[6]) == 0)) {  // bf16 dK / dV hand-off (the layer's default)
        cudaMalloc(&a.dk16, BH * L * 448 * 2);
        cudaMalloc(&a.dv16, BH * L * 448 * 2);
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int it = 0; it < 3; ++it) launch_attn_bwd(d, a, 0, which);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int it = 0; it < reps; ++it) launch_attn_bwd(d, a, 0, which);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("status %s  B=%d L=%d which=%d  %.3f ms\n", cudaGetErrorString(err), B, L, which, ms);
    std::vector<long long> t(4 * 12 * 16 * 64);
    cudaMemcpyFromSymbol(t.data(), g_bwd_trace, t.size() * sizeof(long long));
    auto T = [&](int cta, int w, int ev, int j) { return t[((cta * 12 + w) * 16 + ev) * 64 + j]; };
    const long long t0 = T(0, 1, 0, 0);
    const int nt = (L + 63) / 64;
    const int spt = (argc > 5 && a.ring[4] == 16) ? 4 : 2;  // B2 slices per tile
    for (int cta : {0, 2}) {
        printf("leader cta%d: tile xfree_ok mma1_issue a_full_ok(mma2 issue) b2_last_full | b1_issue b2_issue(first slice of tile j)\n", cta);
        for (int j = 0; j < nt && j < 64; ++j)
            printf("  %3d %8lld %8lld %8lld %8lld | %8lld %8lld\n", j, T(cta,1,2,j)-t0, T(cta,1,0,j)-t0, T(cta,1,1,j)-t0,
                   T(cta,1,13,j)-t0, T(cta,0,11,j)-t0, T(cta,10,12,spt*j)-t0);
    }
    printf("P cta0 w2: tile x_full p_done mma2done_ok pin_free_ok\n");
    for (int j = 0; j < nt && j < 64; ++j)
        printf("  %3d %8lld %8lld %8lld %8lld\n", j, T(0,2,3,j)-t0, T(0,2,4,j)-t0, T(0,2,5,j)-t0, T(0,2,7,j)-t0);
    printf("dS cta2 w2: tile x_full pin_full_ok a_full_arrive\n");
    for (int j = 0; j < nt && j < 64; ++j)
        printf("  %3d %8lld %8lld %8lld\n", j, T(2,2,3,j)-t0, T(2,2,9,j)-t0, T(2,2,10,j)-t0);
    {
        std::vector<long long> ut(4 * 16 * 8);
        cudaMemcpyFromSymbol(ut.data(), g_unit_trace, ut.size() * sizeof(long long));
        for (int cta : {0, 2}) {
            const long long u0 = ut[(cta * 16) * 8 + 6];
            printf("cta%d units: stat_issue stat_full x_full(0) mma2(0) epi_enter acc_full epi_done\n", cta);
            for (int u = 0; u < 16; ++u) {
                const long long* e = &ut[(cta * 16 + u) * 8];
                if (!e[0]) break;
                printf("  %2d %8lld %8lld %8lld %8lld %8lld %8lld %8lld\n", u, e[6] - u0, e[0] - u0, e[2] - u0, e[1] - u0,
                       e[3] - u0, e[4] - u0, e[5] - u0);
            }
        }
    }
    span_summary("attn_bwd", 4 * ((L + 255) / 256) * int(BH));
    return 0;
}
