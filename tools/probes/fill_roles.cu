// Write-bandwidth probe (not part of libdgal): can a persistent subset of CTAs
// reach the HBM write roof for the 40 GB cfg5 fill?  (The fused fill + candidate
// design in dgal_pwindex.cu gives the fill to a fraction of the CTAs.)
#include <cstdio>
#include <cuda_runtime.h>
// each CTA: its slice of band b (bands in order), U * 256 int4 per step
template <int U>
__global__ void __launch_bounds__(256) zero_bands(int4 *p, size_t nvec, int bands, int fillers) {
    if ((int)blockIdx.x >= fillers) return;
    const size_t per_band = (nvec + bands - 1) / bands;
    for (int b = 0; b < bands; ++b) {
        const size_t b0 = (size_t)b * per_band, b1 = min(nvec, b0 + per_band);
        const size_t per_cta = (b1 - b0 + fillers - 1) / fillers;
        const size_t c0 = b0 + per_cta * blockIdx.x, c1 = min(b1, c0 + per_cta);
        for (size_t i = c0 + threadIdx.x; i < c1; i += 256 * U) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const size_t k = i + (size_t)u * 256;
                if (k < c1) __stcs(p + k, make_int4(0, 0, 0, 0));
            }
        }
    }
}
template <int U>
float run(int4 *p, size_t nvec, int grid, int fillers, int bands) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    zero_bands<U><<<grid, 256>>>(p, nvec, bands, fillers);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) zero_bands<U><<<grid, 256>>>(p, nvec, bands, fillers);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); return ms / 3;
}
int main() {
    size_t bytes = 40000000000ull, nvec = bytes / 16;
    int4 *p; cudaMalloc(&p, bytes);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int bands : {1, 16, 64}) {
        for (int f : {sms / 2, sms, sms * 3 / 2, sms * 2}) {
            printf("bands %3d fillers %4d of %d: U4 %.3f ms  U8 %.3f ms\n", bands, f, 2 * sms,
                   run<4>(p, nvec, 2 * sms, f, bands), run<8>(p, nvec, 2 * sms, f, bands));
        }
    }
    return 0;
}
