// Packed FP32 (FADD2/FMUL2/FFMA2) vs scalar, bitwise, incl. subnormals: nvcc -O3 -gencode arch=compute_100a,code=sm_100a ops_vs_scalar.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
__device__ __forceinline__ uint64_t pk(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void upk(uint64_t v, float &a, float &b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__global__ void k(const float *x, const float *y, float *o, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (2 * i + 1 >= n) return;
    float a0 = x[2*i], a1 = x[2*i+1], b0 = y[2*i], b1 = y[2*i+1];
    uint64_t A = pk(a0, a1), B = pk(b0, b1), S, M, D, F;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(S) : "l"(A), "l"(B));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(M) : "l"(A), "l"(B));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(D) : "l"(A), "l"(B));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(F) : "l"(A), "l"(B), "l"(A));
    float s0, s1, m0, m1, d0, d1, f0, f1;
    upk(S, s0, s1); upk(M, m0, m1); upk(D, d0, d1); upk(F, f0, f1);
    float *p = o + 16 * i;
    p[0] = s0; p[1] = s1; p[2] = m0; p[3] = m1; p[4] = d0; p[5] = d1; p[6] = f0; p[7] = f1;
    p[8] = __fsub_rn(a0, b0); p[9] = __fsub_rn(a1, b1); p[10] = __fmul_rn(a0, b0); p[11] = __fmul_rn(a1, b1);
    p[12] = __fadd_rn(a0, b0); p[13] = __fadd_rn(a1, b1); p[14] = __fmaf_rn(a0, b0, a0); p[15] = __fmaf_rn(a1, b1, a1);
}
int main() {
    const int n = 1 << 20;
    float *hx = new float[n], *hy = new float[n], *ho = new float[8 * n];
    uint32_t s = 12345;
    auto rnd = [&]() { s = s * 1664525u + 1013904223u; return s; };
    for (int i = 0; i < n; ++i) {
        uint32_t u = rnd(), v = rnd();
        int mode = i % 4;
        if (mode == 0) { memcpy(&hx[i], &u, 4); memcpy(&hy[i], &v, 4); }  // any bit pattern
        else if (mode == 1) { hx[i] = (int)(u % 2001) - 1000; hy[i] = hx[i] * ((v & 1) ? 1 : -1); }
        else if (mode == 2) { hx[i] = 1e-30f * (u % 7); hy[i] = 1e-30f * (v % 5); }
        else { hx[i] = (float)u / 4e9f; hy[i] = (float)v / 4e9f * 1e-38f; }
    }
    float *dx, *dy, *dout;
    cudaMalloc(&dx, 4 * n); cudaMalloc(&dy, 4 * n); cudaMalloc(&dout, 32 * n);
    cudaMemcpy(dx, hx, 4 * n, cudaMemcpyHostToDevice); cudaMemcpy(dy, hy, 4 * n, cudaMemcpyHostToDevice);
    k<<<(n / 2 + 255) / 256, 256>>>(dx, dy, dout, n);
    cudaMemcpy(ho, dout, 32 * n, cudaMemcpyDeviceToHost);
    int bad[4] = {0, 0, 0, 0};
    for (int i = 0; i < n / 2; ++i) for (int q = 0; q < 8; ++q) {
        uint32_t a, b; memcpy(&a, &ho[16 * i + q], 4); memcpy(&b, &ho[16 * i + 8 + q], 4);
        bool nan = (a & 0x7fffffff) > 0x7f800000 && (b & 0x7fffffff) > 0x7f800000;
        if (a != b && !nan) { if (bad[q / 2] < 3) printf("op %d pair %d: %08x vs %08x (x=%g y=%g)\n", q / 2, i, a, b, hx[2*i+q%2], hy[2*i+q%2]); bad[q / 2]++; }
    }
    printf("mismatches sub %d mul %d add %d fma %d\n", bad[0], bad[1], bad[2], bad[3]);
}
