// Timestamps of one CTA of the fused projection + pack kernel (north-star shape, random data).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2505_11580_b200/csrc
//        -o tools/proj_pack_trace_bin tools/proj_pack_trace.cu
#define FIPA_PP_TRACE 1
#define FIPA_SPAN_TRACE 1
#include "../paper_2505_11580_b200/csrc/proj_pack.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "span_summary.hpp"

using namespace fipa_b200;

int main(int argc, char** argv) {
    const int B = 8, L = 1024, H = 8, din = 256;
    LayerDims d{};
    d.d_in = din; d.d_z = 128; d.heads = H; d.c = 128; d.n_query = 8; d.n_value = 12; d.rank = 2;
    d.n_proj = H * (3 * 128 + 6 * 8 + 3 * 12);
    d.zq = 176; d.dqk_used = 432; d.dqk_mma = 432; d.dqk_pad = 448;
    d.dv_used = 426; d.dv_mma = 432; d.dv_pad = 448; d.din_ld = 256; d.seg = 304; d.feat = H * 304; d.feat_ld = H * 304;
    const int NH = proj_pack_head_width(d);
    const size_t BL = size_t(B) * L;
    auto dalloc = [](size_t bytes) { void* p; cudaMalloc(&p, bytes); cudaMemset(p, 0, bytes); return p; };
    std::vector<__nv_bfloat16> hs(BL * din), hw(size_t(H) * NH * din);
    for (auto& x : hs) x = __float2bfloat16((rand() / float(RAND_MAX) - 0.5f));
    for (auto& x : hw) x = __float2bfloat16((rand() / float(RAND_MAX) - 0.5f) * 0.1f);
    std::vector<float> hz(BL * 256), hr(BL * 9, 0.f), ht(BL * 3);
    for (auto& x : hz) x = rand() / float(RAND_MAX) - 0.5f;
    for (size_t i = 0; i < BL; ++i) { hr[i * 9] = hr[i * 9 + 4] = hr[i * 9 + 8] = 1.f; }
    for (auto& x : ht) x = rand() / float(RAND_MAX) - 0.5f;
    ProjPackArgs a{};
    a.s_bf16 = (__nv_bfloat16*)dalloc(hs.size() * 2);
    a.w_heads = (__nv_bfloat16*)dalloc(hw.size() * 2);
    cudaMemcpy((void*)a.s_bf16, hs.data(), hs.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy((void*)a.w_heads, hw.data(), hw.size() * 2, cudaMemcpyHostToDevice);
    float* z = (float*)dalloc(hz.size() * 4);
    cudaMemcpy(z, hz.data(), hz.size() * 4, cudaMemcpyHostToDevice);
    a.z1 = z; a.z2 = z;
    {
        std::vector<__nv_bfloat16> hzb(hz.size());
        for (size_t i = 0; i < hz.size(); ++i) hzb[i] = __float2bfloat16(hz[i]);
        __nv_bfloat16* zb = (__nv_bfloat16*)dalloc(hzb.size() * 2);
        cudaMemcpy(zb, hzb.data(), hzb.size() * 2, cudaMemcpyHostToDevice);
        a.z1q = zb; a.z2b = zb;
    }
    float* rot = (float*)dalloc(hr.size() * 4);
    cudaMemcpy(rot, hr.data(), hr.size() * 4, cudaMemcpyHostToDevice);
    float* tr = (float*)dalloc(ht.size() * 4);
    cudaMemcpy(tr, ht.data(), ht.size() * 4, cudaMemcpyHostToDevice);
    a.rot = rot; a.trans = tr; a.mask = nullptr;
    std::vector<float> hg(H, 0.1f), hwl(H * 128, 0.05f);
    float* g = (float*)dalloc(H * 4); cudaMemcpy(g, hg.data(), H * 4, cudaMemcpyHostToDevice);
    float* wl = (float*)dalloc(H * 128 * 4); cudaMemcpy(wl, hwl.data(), H * 128 * 4, cudaMemcpyHostToDevice);
    a.head_g = g; a.wl_bias = wl; a.k_scale = 0.05f;
    a.proj = (float*)dalloc(BL * d.n_proj * 4);
    a.colbias = (float*)dalloc(BL * H * 4);
    a.qhat = (__nv_bfloat16*)dalloc(BL * H * 448 * 2);
    a.khat = (__nv_bfloat16*)dalloc(BL * H * 448 * 2);
    a.vhat = (__nv_bfloat16*)dalloc(BL * H * 448 * 2);
    a.B = B; a.L = L;
    a.write_points = argc > 1 && atoi(argv[1]) != 0;  // training forward
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) launch_proj_pack(d, a, 0);
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) launch_proj_pack(d, a, 0);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("status %s  %.4f ms per launch\n", cudaGetErrorString(err), ms / 10);
    std::vector<long long> t(10 * 16);
    cudaMemcpyFromSymbol(t.data(), g_pp_trace, t.size() * sizeof(long long));
    const long long t0 = t[0 * 16 + 0];
    const char* names[16] = {"start/wait0", "done", "epi begin", "t0 A", "t0 B", "t0 B end", "t0 synced",
                             "t1 A", "t1 B", "t1 B end", "t1 synced", "t2 A", "t2 B", "t2 B end", "t2 synced", "end"};
    for (int w = 0; w < 10; ++w) {
        printf("w%d:", w);
        for (int ev = 0; ev < 16; ++ev) if (t[w * 16 + ev]) printf(" %s=%lld", names[ev], t[w * 16 + ev] - t0);
        printf("\n");
    }
    span_summary("proj_pack", (B * L / 128) * H);
    return 0;
}
