// Latency of warp-collective and shared-memory operations on one warp
// (dependent chains, clock64).  nvcc -arch=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned* out, double* dout) {
    __shared__ unsigned su[64];
    __shared__ double sd[64];
    const int lane = threadIdx.x;
    su[lane] = lane; su[lane + 32] = lane; sd[lane] = lane; sd[lane + 32] = lane;
    __syncwarp();
    unsigned v = lane;
    double d = lane;
    long long t0, t1;
#define M(name, stmt, it) t0 = clock64(); for (int i = 0; i < it; i++) { stmt; } t1 = clock64(); \
    if (lane == 0) printf("%-22s %8.1f cycles\n", name, (double)(t1 - t0) / it);
    M("reduce_max_sync u32", v = __reduce_max_sync(0xffffffffu, v) + lane, 200)
    M("reduce_add_sync u32", v = __reduce_add_sync(0xffffffffu, v) ^ lane, 200)
    M("shfl_xor u32", v = __shfl_xor_sync(0xffffffffu, v, 1) + 1, 200)
    M("shfl_xor f64", d = __shfl_xor_sync(0xffffffffu, d, 1) + 1.0, 200)
    M("ballot", v = __ballot_sync(0xffffffffu, v & 1) + lane, 200)
    M("lds u32 dep", v = su[(v + lane) & 63], 200)
    M("lds f64 dep", d = sd[((int)d + lane) & 63], 200)
    M("sts+lds u32", { su[lane] = v; __syncwarp(); v = su[lane ^ 1] + 1; }, 200)
    M("syncwarp", __syncwarp(), 200)
    out[lane] = v; dout[lane] = d;
}
__global__ void kb(unsigned* out) {
    long long t0 = clock64();
    for (int i = 0; i < 200; i++) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) printf("%-22s %8.1f cycles (%d threads)\n", "syncthreads", (double)(t1 - t0) / 200, blockDim.x);
}
int main() {
    unsigned* o; double* d;
    cudaMalloc(&o, 4096); cudaMalloc(&d, 4096);
    k<<<1, 32>>>(o, d);
    kb<<<1, 256>>>(o);
    kb<<<1, 1024>>>(o);
    cudaDeviceSynchronize();
    return 0;
}
