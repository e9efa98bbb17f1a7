// Write-bandwidth probe (not part of libdgal): which streaming-store shape reaches
// the HBM write roof on this GPU for a 40 GB fill.
#include <cstdio>
#include <cuda_runtime.h>
template <int U, bool CS>
__global__ void zero_k(int4 *p, size_t nvec) {
    size_t i = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x * U;
    for (; i + (U - 1) * blockDim.x < nvec; i += stride) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (CS) __stcs(p + i + u * blockDim.x, make_int4(0, 0, 0, 0));
            else p[i + u * blockDim.x] = make_int4(0, 0, 0, 0);
        }
    }
    for (; i < nvec; i += blockDim.x) p[i] = make_int4(0, 0, 0, 0);
}
// one contiguous chunk of U*blockDim int4 per block, blocks in address order
template <int U>
__global__ void zero_chunk(int4 *p, size_t nvec) {
    const size_t base = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const size_t i = base + (size_t)u * blockDim.x;
        if (i < nvec) __stcs(p + i, make_int4(0, 0, 0, 0));
    }
}
template <int U>
float run_chunk(int4 *p, size_t nvec, int block) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const size_t grid = (nvec + (size_t)block * U - 1) / ((size_t)block * U);
    zero_chunk<U><<<(unsigned)grid, block>>>(p, nvec);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) zero_chunk<U><<<(unsigned)grid, block>>>(p, nvec);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); return ms / 3;
}
template <int U, bool CS>
float run(int4 *p, size_t nvec, int grid, int block) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    zero_k<U, CS><<<grid, block>>>(p, nvec);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) zero_k<U, CS><<<grid, block>>>(p, nvec);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); return ms / 3;
}
int main() {
    size_t bytes = 40000000000ull, nvec = bytes / 16;
    int4 *p; cudaMalloc(&p, bytes);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int g : {sms * 4, sms * 8, sms * 16, sms * 32}) {
        printf("grid %5d  U1 cs %.3f  U1 plain %.3f  U4 cs %.3f  U4 plain %.3f ms\n", g,
               run<1, true>(p, nvec, g, 256), run<1, false>(p, nvec, g, 256),
               run<4, true>(p, nvec, g, 256), run<4, false>(p, nvec, g, 256));
    }
    printf("chunk U1 b256 %.3f  U4 b256 %.3f  U8 b256 %.3f  U4 b512 %.3f  U16 b128 %.3f ms\n",
           run_chunk<1>(p, nvec, 256), run_chunk<4>(p, nvec, 256), run_chunk<8>(p, nvec, 256),
           run_chunk<4>(p, nvec, 512), run_chunk<16>(p, nvec, 128));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaMemsetAsync(p, 0, bytes); cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) cudaMemsetAsync(p, 0, bytes);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("cudaMemsetAsync %.3f ms (%.0f GB/s)\n", ms / 3, bytes / (ms / 3) / 1e6);
    return 0;
}
