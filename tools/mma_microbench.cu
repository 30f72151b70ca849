// Microbenchmark: tcgen05.mma issue throughput vs N and operand source (SS vs TS), to size the
// attention kernel's tiles (shared-memory read bandwidth of the A operand at small N).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2505_11580_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace fipa_b200;

template <int N, bool TS, int CHAINS>
__global__ void __launch_bounds__(128, 1) mma_bench(int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc(&slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    long long t0 = 0, t1 = 0;
    if (warp == 0) {
        const uint32_t a = ptx::smem_u32(smem);
        const uint32_t b = a + 128 * 128;  // A tile 16 KB, then B tile (N rows x 128 B)
        const uint32_t idesc = ptx::idesc_bf16(128, N, false, false);
        // warm
        if (ptx::elect_one()) {
            for (int k = 0; k < 4; ++k)
                ptx::mma_ss(tmem, ptx::sw128_desc(a + k * 32, 16, 1024), ptx::sw128_desc(b + k * 32, 16, 1024), idesc, 1);
            ptx::mma_commit(&bar);
        }
        __syncwarp();
        ptx::mbar_wait(&bar, 0);
        t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t db = ptx::sw128_desc(b + k * 32, 16, 1024);
                const uint32_t d = tmem + (CHAINS > 1 ? (k % CHAINS) * 64 : 0);
                const uint64_t da = ptx::sw128_desc(a + k * 32, 16, 1024);
                if (ptx::elect_one()) {
                    if (TS) {
                        ptx::mma_ts(d, tmem + 256 + k * 8, db, idesc, 1);
                    } else {
                        ptx::mma_ss(d, da, db, idesc, 1);
                    }
                }
                __syncwarp();
            }
        }
        if (ptx::elect_one()) ptx::mma_commit(&bar);
        __syncwarp();
        ptx::mbar_wait(&bar, 1);
        t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

template <int N, bool TS, int CHAINS = 1>
void run(int blocks) {
    const int iters = 4096;
    long long* d;
    cudaMalloc(&d, sizeof(long long) * blocks);
    const int smem = 128 * 128 + 256 * 128 + 1024;
    cudaFuncSetAttribute(mma_bench<N, TS, CHAINS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mma_bench<N, TS, CHAINS><<<blocks, 128, smem>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < blocks; ++i) mean += h[i];
    mean /= blocks;
    const double per = mean / (iters * 4.0);
    const double macs = 128.0 * N * 16;
    printf("chains=%d N=%3d %s blocks=%3d: %.2f cycles/MMA  -> %.0f MAC/cycle/SM  (ideal %.1f cyc)  %s\n",
           CHAINS, N, TS ? "TS" : "SS", blocks, per, macs / per, macs / 4096.0, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    run<64, false, 2>(1);
    run<64, false, 4>(1);
    run<32, false, 4>(1);
    run<64, true, 2>(1);
    run<64, true, 4>(1);
    for (int blocks : {1}) {
        run<32, false>(blocks);
        run<64, false>(blocks);
        run<128, false>(blocks);
        run<256, false>(blocks);
        run<64, true>(blocks);
        run<128, true>(blocks);
        run<256, true>(blocks);
    }
    return 0;
}
