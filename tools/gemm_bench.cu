// Standalone timing of the tcgen05 GEMM (gemm_tc.cu) on the layer's shapes and a large square one.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/gemm_bench.cu -o tools/gemm_bench_bin -lcuda
#include "../paper_2505_11580_b200/csrc/gemm_tc.cu"

#include <cstdio>
#include <vector>

using namespace fipa_b200;

static float time_gemm(const GemmArgs& g, int reps = 20) {
    for (int i = 0; i < 3; ++i) launch_gemm_bf16(g, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) launch_gemm_bf16(g, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
}

int main() {
    const size_t big = size_t(8192) * 8192;
    __nv_bfloat16 *A, *B;
    float* C;
    cudaMalloc(&A, big * 2);
    cudaMalloc(&B, big * 2);
    cudaMalloc(&C, big * 4);
    cudaMemset(A, 0, big * 2);
    cudaMemset(B, 0, big * 2);
    struct Case { const char* name; int M, N, K; bool amn, bmn; bool bf16out; };
    const Case cases[] = {{"square 8192^3", 8192, 8192, 8192, false, false, false},
                          {"square 8192^3 bf16 out", 8192, 8192, 8192, false, false, true},
                          {"out GEMM 8192x256x2432", 8192, 256, 2432, false, false, false},
                          {"dfeat 8192x2432x256 (B MN)", 8192, 2432, 256, false, true, true},
                          {"dfeat shape, f32 out", 8192, 2432, 256, false, true, false},
                          {"dfeat shape, B K-major", 8192, 2432, 256, false, false, true},
                          {"dfeat shape, B K-major f32", 8192, 2432, 256, false, false, false},
                          {"8192x2560x256 K-major", 8192, 2560, 256, false, false, false},
                          {"8192x2048x512 K-major", 8192, 2048, 512, false, false, false},
                          {"8192x2048x2048", 8192, 2048, 2048, false, false, false},
                          {"long K 1024x256x65536", 1024, 256, 65536 / 8, false, false, false}};
    for (const auto& c : cases) {
        GemmArgs g;
        g.A = A;
        g.B = B;
        g.C = C;
        g.M = c.M;
        g.N = c.N;
        g.K = c.K;
        g.a_mn_major = c.amn;
        g.b_mn_major = c.bmn;
        g.lda = c.amn ? c.M : c.K;
        g.ldb = c.bmn ? c.N : c.K;
        g.ldc = c.N;
        g.out_bf16 = c.bf16out;
        const float ms = time_gemm(g);
        const double tf = 2.0 * c.M * c.N * double(c.K) / (ms * 1e-3) / 1e12;
        printf("%-32s %8.3f ms  %7.1f TFLOP/s  (%s)\n", c.name, ms, tf, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
