// Latency of the scalar FP64 operations on the encoders' serial chains
// (one thread, dependent chains, clock64).  nvcc -arch=sm_100a -O3 -fmad=false
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double x0) {
    double x = x0;
    long long t0, t1;
#define MEASURE(name, expr, it)                                  \
    t0 = clock64();                                              \
    for (int i = 0; i < it; i++) { x = expr; }                   \
    t1 = clock64();                                              \
    out[0] += x;                                                 \
    printf("%-12s %8.1f cycles\n", name, (double)(t1 - t0) / it);
    MEASURE("dadd", x + 1e-300, 1000)
    MEASURE("dmul", x * 1.0000001, 1000)
    MEASURE("dfma", __fma_rn(x, 1.0000001, 1e-300), 1000)
    MEASURE("ddiv_rn", __ddiv_rn(1.0, x) , 200)
    MEASURE("log10", log10(x) + 2.0, 200)
    MEASURE("exp10", exp10(-x * 1e-3), 200)
    MEASURE("sqrt", sqrt(x) + 1.0, 200)
    MEASURE("rint", rint(x * 3.3) + 0.25, 200)
    MEASURE("floor", floor(x * 1.5) + 0.5, 200)
    MEASURE("ldexp", ldexp(x, 3) * 0.125, 200)
    MEASURE("i2d", (double)(int)(x) + 0.5, 200)
}
int main() {
    double* o; long long* c;
    cudaMalloc(&o, 64); cudaMalloc(&c, 64); cudaMemset(o, 0, 64);
    k<<<1, 1>>>(o, c, 1.5);
    cudaDeviceSynchronize();
    return 0;
}
