// Store-path microbenchmark: one CTA per SM writes a 128-row x 432-column fp32 tile (221 KB, the
// attention-backward accumulator) from registers / shared memory with different instruction
// patterns; prints cycles per CTA (clock64) and aggregate GB/s.  Rows are `stride` floats apart.
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__global__ void k_v4(float* out, int stride, int nwarps, long long* cyc) {
    // thread = row (32 rows per warp, 4 warps = 128 rows), 16-byte stores along the row
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* row = out + (size_t(blockIdx.x) * 128 + warp * 32 + lane) * stride;
    __syncthreads();
    long long t0 = clock64();
    for (int c = 0; c < 432; c += 4) reinterpret_cast<float4*>(row + c)[0] = make_float4(c, c, c, c);
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

__global__ void k_coal(float* out, int stride, int nwarps, long long* cyc) {
    // 8 threads per row, 16 bytes each: one 128-byte line per row per instruction (4 rows / instr)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    long long t0 = clock64();
    const int rpw = 128 / nwarps;
    for (int r = warp * rpw; r < warp * rpw + rpw; r += 4) {
        float* row = out + (size_t(blockIdx.x) * 128 + r + lane / 8) * stride;
        for (int c = 4 * (lane & 7); c < 432; c += 32) reinterpret_cast<float4*>(row + c)[0] = make_float4(c, c, c, c);
    }
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

__global__ void k_contig(float* out, int stride, int nwarps, long long* cyc) {
    // fully contiguous 221 KB per CTA, coalesced float4
    float* base = out + size_t(blockIdx.x) * 128 * stride;
    __syncthreads();
    long long t0 = clock64();
    for (int i = threadIdx.x; i < 128 * 432 / 4; i += blockDim.x) reinterpret_cast<float4*>(base)[i] = make_float4(i, i, i, i);
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    long long* cyc;
    const int strides[2] = {448, 448 * 8};
    cudaMalloc(&out, size_t(sms) * 128 * 448 * 8 * 4);
    cudaMalloc(&cyc, sms * sizeof(long long));
    for (int nt : {128, 256, 512}) {
        for (int kind = 1; kind < 3; ++kind) {
            auto launch = [&]() {
                if (kind == 1) k_coal<<<8, nt>>>(out, 3584, nt / 32, cyc);
                if (kind == 2) k_contig<<<8, nt>>>(out, 448, nt / 32, cyc);
            };
            for (int w = 0; w < 3; ++w) launch();
            cudaDeviceSynchronize();
            std::vector<long long> h(8);
            cudaMemcpy(h.data(), cyc, 8 * sizeof(long long), cudaMemcpyDeviceToHost);
            double mean = 0;
            for (auto x : h) mean += double(x) / 8;
            printf("threads %3d kind %d: %8.0f cycles/CTA (%.1f B/clk/SM)\n", nt, kind, mean, 128.0 * 432 * 4 / mean);
        }
    }
    for (int nblk : {8, sms}) {
        for (int si = 0; si < 2; ++si) {
            const int stride = strides[si];
            const char* names[3] = {"thread-row v4", "8 thr/row v4 ", "contiguous   "};
            for (int kind = 0; kind < 3; ++kind) {
                auto launch = [&]() {
                    if (kind == 0) k_v4<<<nblk, 128>>>(out, stride, 4, cyc);
                    if (kind == 1) k_coal<<<nblk, 128>>>(out, stride, 4, cyc);
                    if (kind == 2) k_contig<<<nblk, 128>>>(out, 448, 4, cyc);
                };
                for (int w = 0; w < 3; ++w) launch();
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                cudaEventRecord(a);
                launch();
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                std::vector<long long> h(nblk);
                cudaMemcpy(h.data(), cyc, nblk * sizeof(long long), cudaMemcpyDeviceToHost);
                double mean = 0;
                for (auto x : h) mean += double(x) / nblk;
                printf("blocks %3d stride %5d %s: %8.0f cycles/CTA (%.1f B/clk/SM), %.0f GB/s\n", nblk, stride,
                       names[kind], mean, 128.0 * 432 * 4 / mean, nblk * 128.0 * 432 * 4 / ms / 1e6);
            }
        }
    }
    return 0;
}
