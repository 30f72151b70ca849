// Epilogue / MMA timeline of CTA 0 of the tcgen05 GEMM (gemm_tc.cu), one shape.
#define FIPA_GEMM_TRACE 1
#include "../paper_2505_11580_b200/csrc/gemm_tc.cu"
#include <cstdio>
#include <cstdlib>
using namespace fipa_b200;
int main(int argc, char** argv) {
    const int M = argc > 1 ? atoi(argv[1]) : 8192, N = argc > 2 ? atoi(argv[2]) : 2048, K = argc > 3 ? atoi(argv[3]) : 512;
    const int bf16out = argc > 4 ? atoi(argv[4]) : 0;
    const int b_mn = argc > 5 ? atoi(argv[5]) : 0;  // 1: B stored [K][N] (MN-major)
    __nv_bfloat16 *A, *B;
    float* C;
    cudaMalloc(&A, size_t(M) * K * 2);
    cudaMalloc(&B, size_t(N) * K * 2);
    cudaMalloc(&C, size_t(M) * N * 4);
    cudaMemset(A, 0, size_t(M) * K * 2);
    cudaMemset(B, 0, size_t(N) * K * 2);
    GemmArgs g;
    g.A = A; g.B = B; g.C = C; g.M = M; g.N = N; g.K = K; g.lda = K; g.ldb = b_mn ? N : K; g.ldc = N; g.out_bf16 = bf16out;
    g.b_mn_major = b_mn != 0;
    for (int i = 0; i < 5; ++i) launch_gemm_bf16(g, 0);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) launch_gemm_bf16(g, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("M=%d N=%d K=%d bf16out=%d b_mn=%d: %.4f ms per launch, %.1f TFLOP/s\n", M, N, K, bf16out, b_mn, ms / 20,
           2.0 * M * N * K / (ms / 20 * 1e-3) / 1e12);
    long long t[2][8][24];
    cudaMemcpyFromSymbol(t, g_gemm_trace, sizeof(t));
    const long long t0 = t[1][0][0];
    for (int u = 0; u < 6; ++u) {
        printf("unit %d  MMA: start %7lld acc_free %7lld committed %7lld | EPI: wait %7lld full %7lld |", u, t[1][u][0] - t0,
               t[1][u][1] - t0, t[1][u][2] - t0, t[0][u][0] - t0, t[0][u][1] - t0);
        for (int c = 0; c < 8; ++c) printf(" %lld/%lld", t[0][u][2 + 2 * c] - t0, t[0][u][3 + 2 * c] - t0);
        printf("\n");
    }
    return 0;
}
