// Pipeline trace of the CTA-pair attention kernel (leader CTA of cluster (0,0)), north-star
// shape.  Events (SM clock): QK first-block ready, PV first-stage ready, softmax S ready,
// softmax PV(j-1) done, softmax P published, K/V load issue, MMA s_free / p_full observed.
#define FIPA_ATTN_TRACE 1
#define FIPA_SPAN_TRACE 1
#include "../paper_2505_11580_b200/csrc/attn_fwd_2sm.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "span_summary.hpp"

using namespace fipa_b200;

int main(int argc, char** argv) {
    const int B = argc > 1 ? atoi(argv[1]) : 8;
    const int L = argc > 2 ? atoi(argv[2]) : 1024;
    LayerDims d{};
    d.d_in = 256; d.d_z = 128; d.heads = 8; d.c = 128; d.n_query = 8; d.n_value = 12; d.rank = 2;
    d.zq = 176; d.dqk_used = 176 + 256; d.dqk_mma = 432; d.dqk_pad = 448;
    d.dv_used = 128 + 256 + 36 + 6; d.dv_mma = 432; d.dv_pad = 448; d.dv_tc = 416; d.dv_simt = 10;
    d.seg = 304; d.feat = 8 * 304; d.feat_ld = d.feat; d.din_ld = 256;
    const size_t BH = size_t(B) * d.heads, BL = size_t(B) * L;
    std::vector<__nv_bfloat16> hq(BH * L * d.dqk_pad), hv(BH * L * d.dv_pad);
    srand(1);
    for (auto& x : hq) x = __float2bfloat16((rand() / float(RAND_MAX) - 0.5f) * 0.2f);
    for (auto& x : hv) x = __float2bfloat16((rand() / float(RAND_MAX) - 0.5f));
    __nv_bfloat16 *q, *k, *v, *feat;
    float *z1, *rot, *trans, *lse;
    cudaMalloc(&q, hq.size() * 2);
    cudaMalloc(&k, hq.size() * 2);
    cudaMalloc(&v, hv.size() * 2);
    cudaMalloc(&feat, BL * d.feat * 2);
    cudaMalloc(&z1, BL * 256 * 4);
    cudaMalloc(&rot, BL * 9 * 4);
    cudaMalloc(&trans, BL * 3 * 4);
    cudaMalloc(&lse, BH * L * 4);
    cudaMemcpy(q, hq.data(), hq.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(k, hq.data(), hq.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(v, hv.data(), hv.size() * 2, cudaMemcpyHostToDevice);
    cudaMemset(z1, 0, BL * 256 * 4);
    cudaMemset(rot, 0, BL * 9 * 4);
    cudaMemset(trans, 0, BL * 3 * 4);
    AttnArgs a{};
    a.qhat = q; a.khat = k; a.vhat = v; a.colbias = nullptr; a.z1 = z1; a.rot = rot; a.trans = trans;
    a.feat = feat; a.lse = lse; a.B = B; a.L = L;
    if (argc > 3 && atoi(argv[3]) != 0) {  // training forward: also save the fp32 O_hat
        float* o;
        cudaMalloc(&o, BL * d.heads * d.dv_pad * 4);
        a.o_save = o;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int it = 0; it < 3; ++it) launch_attn_fwd_2sm(d, a, 0);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int it = 0; it < reps; ++it) launch_attn_fwd_2sm(d, a, 0);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    const double flops = 2.0 * BH * L * double(L) * (424 + 420);
    printf("status %s  B=%d L=%d  %.3f ms  %.1f TFLOP/s\n", cudaGetErrorString(err), B, L, ms,
           flops / ms / 1e9);
    std::vector<long long> t(2 * 16 * 16 * 128);
    cudaMemcpyFromSymbol(t.data(), g_attn_trace, t.size() * sizeof(long long));
    auto T = [&](int cta, int w, int ev, int j) { return t[((cta * 16 + w) * 16 + ev) * 128 + j]; };
    const long long t0 = T(0, 1, 0, 0);
    const int nt = (L + 63) / 64;
    printf("MMA leader: tile sfree kfull pfull(j) pv0(j) pvend(j) | Kissue(j) Vissue(2j) Vissue(2j+1)\n");
    for (int j = 0; j < nt && j < 64; ++j)
        printf("  %3d %8lld %8lld %8lld %8lld %8lld | %8lld %8lld %8lld\n", j, T(0,1,7,j)-t0, T(0,1,0,j)-t0,
               T(0,1,8,j)-t0, T(0,1,1,j)-t0, T(0,1,11,j)-t0, T(0,0,5,j)-t0, T(0,10,6,2*j)-t0, T(0,10,6,2*j+1)-t0);
    for (int cta = 0; cta < 2; ++cta)
        for (int w : {2, 6}) {
            printf("softmax cta%d w%d: tile sfull sfree expd pvdone resc ppub\n", cta, w);
            for (int j = 0; j < nt && j < 64; j += (w == 2 && cta == 0 ? 1 : 4))
                printf("  %3d %8lld %8lld %8lld %8lld %8lld %8lld\n", j, T(cta,w,2,j)-t0, T(cta,w,12,j)-t0,
                       T(cta,w,13,j)-t0, j ? T(cta,w,3,j)-t0 : 0, T(cta,w,14,j)-t0, T(cta,w,4,j)-t0);
        }
    span_summary("attn_fwd_2sm", 2 * ((L + 255) / 256) * int(BH));
    printf("o_full %lld  end %lld\n", T(0,2,9,0)-t0, T(0,2,9,1)-t0);
    for (int cta = 0; cta < 2; ++cta)
        for (int w = 2; w < 10; ++w)
            printf("epi cta%d w%d: pre %6lld scalar %6lld points %6lld zwait %6lld pair %6lld bar %6lld store %6lld\n", cta, w,
                   T(cta,w,15,0)-T(cta,w,9,0), T(cta,w,15,1)-T(cta,w,15,0), T(cta,w,15,2)-T(cta,w,15,1), T(cta,w,15,3)-T(cta,w,15,2),
                   T(cta,w,15,4)-T(cta,w,15,3), T(cta,w,15,5)-T(cta,w,15,4), T(cta,w,9,1)-T(cta,w,15,5));
    return 0;
}
