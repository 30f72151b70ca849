// Microbenchmark: TMA (cp.async.bulk.tensor) latency / throughput for the box shapes the
// attention kernel uses (64 bf16 = 128 B inner, 16..128 rows, 864 B row stride).
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "tma_host.hpp"

using namespace fipa_b200;

__global__ void tma_bench(const __grid_constant__ CUtensorMap map, int nbox, int box_bytes, int rows,
                          int three_d, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        ptx::tma_prefetch(&map);
        // warm-up round (fills L2)
        for (int rep = 0; rep < 3; ++rep) {
            const long long t0 = clock64();
            ptx::mbar_expect_tx(&bar, nbox * box_bytes);
            for (int b = 0; b < nbox; ++b) {
                const int row0 = (blockIdx.x * nbox + b) * rows;
                if (three_d)
                    ptx::tma_load_3d(smem + (b % 16) * box_bytes, &map, &bar, 0, row0, 0);
                else
                    ptx::tma_load_2d(smem + (b % 16) * box_bytes, &map, &bar, 0, row0);
            }
            ptx::mbar_wait(&bar, rep & 1);
            const long long t1 = clock64();
            if (rep == 2) out[blockIdx.x] = t1 - t0;
        }
    }
}

int main() {
    const int ld = 432;  // elements per row (864 B), like the lifted rows
    const size_t rows_total = 1 << 20;
    void* buf;
    cudaMalloc(&buf, rows_total * ld * 2);
    cudaMemset(buf, 0, rows_total * ld * 2);
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    for (int three_d = 0; three_d < 2; ++three_d) {
        for (int rows : {16, 32, 64, 128}) {
            for (int nbox : {1, 4, 16}) {
                for (int blocks : {1, 148}) {
                    CUtensorMap m = three_d ? make_map_3d_bf16(buf, ld, rows_total, 1, ld, 64, rows)
                                            : make_map_2d_bf16(buf, rows_total, ld, ld, 64, rows);
                    const int box_bytes = rows * 128;
                    const int smem = 16 * box_bytes;
                    cudaFuncSetAttribute(tma_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                    tma_bench<<<blocks, 32, smem>>>(m, nbox, box_bytes, rows, three_d, d);
                    cudaError_t e = cudaDeviceSynchronize();
                    long long h[148];
                    cudaMemcpy(h, d, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
                    double mean = 0;
                    for (int i = 0; i < blocks; ++i) mean += h[i];
                    mean /= blocks;
                    printf("%s rows=%3d boxes=%2d blocks=%3d: %8.0f cycles  (%.1f B/cycle/SM)  %s\n",
                           three_d ? "3D" : "2D", rows, nbox, blocks, mean, nbox * box_bytes / mean,
                           cudaGetErrorString(e));
                }
            }
        }
    }
    return 0;
}
