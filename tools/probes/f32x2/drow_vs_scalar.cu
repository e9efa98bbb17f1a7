// Decision rows packed (f2mul_nc products) vs scalar cross_rn, bitwise: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../../paper_2011_11134_b200/csrc drow_vs_scalar.cu
// (with f2mul instead of f2mul_nc ptxas fuses the products into FFMA2: 26 % of values 1 ulp off)
#include <cstdio>
#include <cstdint>
#include <cstring>
#include "dgal_core.cuh"
using namespace dgal;
__global__ void k(const float *in, float *out, int n) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    Poly<4> P, Q;
    for (int k = 0; k < 4; ++k) { P.x[k] = in[16*t+k]; P.y[k] = in[16*t+4+k]; Q.x[k] = in[16*t+8+k]; Q.y[k] = in[16*t+12+k]; }
    float fx[4], fy[4];
    for (int i = 0; i < 4; ++i) { fx[i] = Q.x[(i+1)%4] - Q.x[i]; fy[i] = Q.y[(i+1)%4] - Q.y[i]; }
    float *o = out + 32 * t;
    for (int i = 0; i < 4; ++i) {
        const uint64_t px = f2pack(P.x[i], P.x[i]), py = f2pack(P.y[i], P.y[i]);
        const uint64_t tiny2 = f2pack(kTiny, kTiny);
        for (int q = 0; q < 2; ++q) {
            const uint64_t Dx = f2sub(px, f2pack(Q.x[2 * q], Q.x[2 * q + 1]));
            const uint64_t Dy = f2sub(py, f2pack(Q.y[2 * q], Q.y[2 * q + 1]));
            const uint64_t fx2 = f2pack(fx[2 * q], fx[2 * q + 1]), fy2 = f2pack(fy[2 * q], fy[2 * q + 1]);
            f2unpack(f2add(f2sub(f2fma(fx2, Dy, 0ull), f2fma(fy2, Dx, 0ull)), tiny2), o[4*i+2 * q], o[4*i+2 * q + 1]);
        }
        for (int j = 0; j < 4; ++j) {
            const float Dx = __fsub_rn(P.x[i], Q.x[j]), Dy = __fsub_rn(P.y[i], Q.y[j]);
            o[16 + 4*i+j] = __fadd_rn(cross_rn(fx[j], fy[j], Dx, Dy), kTiny);
        }
    }
}
int main() {
    const int n = 1 << 16;
    float *h = new float[16 * n], *ho = new float[32 * n];
    uint32_t s = 777;
    for (int i = 0; i < 16 * n; ++i) { s = s * 1664525u + 1013904223u; h[i] = ((int)(s >> 8) - (1 << 23)) / 1048576.0f; }
    float *d, *dout; cudaMalloc(&d, 64 * n); cudaMalloc(&dout, 128 * n);
    cudaMemcpy(d, h, 64 * n, cudaMemcpyHostToDevice);
    k<<<n / 256, 256>>>(d, dout, n);
    cudaMemcpy(ho, dout, 128 * n, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int t = 0; t < n; ++t) for (int q = 0; q < 16; ++q) {
        uint32_t a, b; memcpy(&a, &ho[32*t+q], 4); memcpy(&b, &ho[32*t+16+q], 4);
        if (a != b) { if (bad < 5) printf("t %d q %d %08x %08x  %.9g %.9g\n", t, q, a, b, ho[32*t+q], ho[32*t+16+q]); bad++; }
    }
    printf("bad %d of %d\n", bad, 16 * n);
}
