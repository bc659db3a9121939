// ubench.cu -- per-SM throughput of the instructions the encoder/decoder
// designs lean on (smem atomics vs stores, f64 conversions, DFMA, FLO, ...).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench tools/ubench.cu
// Output: lane-ops per clock per SM for each op (1 SM fully occupied).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int NT = 1024;

__global__ void k_sts(unsigned long long* cyc, uint32_t* sink) {
    __shared__ uint32_t s[NT * 2];
    uint32_t v = threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < ITERS; i++) {
        s[(threadIdx.x + i) & (2 * NT - 1)] = v;
        v = v * 3 + 1;
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (v == 7) sink[0] = s[threadIdx.x];
}
__global__ void k_atoms(unsigned long long* cyc, uint32_t* sink) {
    __shared__ uint32_t s[NT * 2];
    s[threadIdx.x] = 0; s[threadIdx.x + NT] = 0;
    uint32_t v = threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < ITERS; i++) {
        atomicOr(&s[(threadIdx.x + i) & (2 * NT - 1)], v);
        v = v * 3 + 1;
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (v == 7) sink[0] = s[threadIdx.x];
}
__global__ void k_atoms2(unsigned long long* cyc, uint32_t* sink) {  // 2 lanes per word
    __shared__ uint32_t s[NT * 2];
    s[threadIdx.x] = 0; s[threadIdx.x + NT] = 0;
    uint32_t v = threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < ITERS; i++) {
        atomicOr(&s[((threadIdx.x >> 1) + i) & (2 * NT - 1)], v);
        v = v * 3 + 1;
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (v == 7) sink[0] = s[threadIdx.x];
}

#define CHAINS 8
template <int OP>
__global__ void k_alu(unsigned long long* cyc, double* sinkd, float* sinkf) {
    double d[CHAINS];
    float f[CHAINS];
    int q[CHAINS];
    for (int c = 0; c < CHAINS; c++) { d[c] = threadIdx.x * 0.37 + c; f[c] = (float)d[c]; q[c] = threadIdx.x + c; }
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < ITERS / CHAINS; i++) {
#pragma unroll
        for (int c = 0; c < CHAINS; c++) {
            if (OP == 0) d[c] = __fma_rn(d[c], 1.0000001, 0.5);             // DFMA
            if (OP == 1) d[c] = (double)f[c] + d[c] * 0.0;                   // F2F.F64.F32 (+DFMA)
            if (OP == 2) f[c] = __double2float_rn(d[c] + (double)i);         // F2F.F32.F64 (+DADD)
            if (OP == 3) q[c] = __double2int_rn(d[c] + (double)q[c]);        // F2I.F64 (+I2F +DADD)
            if (OP == 4) q[c] = __clz(q[c] ^ i) + q[c];                      // FLO
            if (OP == 5) q[c] = __reduce_add_sync(0xffffffffu, q[c] + i);   // REDUX
            if (OP == 6) q[c] = __shfl_xor_sync(0xffffffffu, q[c], 1) + i;   // SHFL
            if (OP == 7) d[c] = d[c] * 1.0000001 + 0.5;                      // DMUL+DADD
            if (OP == 8) f[c] = (float)((double)f[c] * 1.0000001);           // F2F both ways + DMUL
            if (OP == 9) q[c] = q[c] * 7 + (q[c] >> 3);                      // IMAD + SHF
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    double acc = 0;
    for (int c = 0; c < CHAINS; c++) acc += d[c] + f[c] + q[c];
    if (acc == 12345.0) sinkd[0] = acc;
}

static const char* names[] = {"DFMA", "F2F.F64.F32(+DFMA)", "F2F.F32.F64(+DADD)", "F2I.F64+I2F+DADD",
                              "FLO+LOP", "REDUX+IADD", "SHFL+IADD", "DMUL+DADD", "F2F x2 + DMUL",
                              "IMAD+SHF+IADD"};

template <int OP>
void run_alu(unsigned long long* d_cyc, double* sd, float* sf, int clk_khz) {
    k_alu<OP><<<148, NT>>>(d_cyc, sd, sf);
    cudaDeviceSynchronize();
    unsigned long long c[148];
    cudaMemcpy(c, d_cyc, sizeof(c), cudaMemcpyDeviceToHost);
    double cycles = 0;
    for (int i = 0; i < 148; i++) cycles += c[i];
    cycles /= 148;
    double lane_ops = (double)NT * ITERS;
    printf("%-24s %8.2f lane-ops/clk/SM  (%.0f cycles)\n", names[OP], lane_ops / cycles, cycles);
}

int main() {
    unsigned long long* d_cyc;
    uint32_t* sink;
    double* sd;
    float* sf;
    cudaMalloc(&d_cyc, 148 * 8);
    cudaMalloc(&sink, 64);
    cudaMalloc(&sd, 64);
    cudaMalloc(&sf, 64);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    auto run = [&](void (*k)(unsigned long long*, uint32_t*), const char* nm) {
        k<<<148, NT>>>(d_cyc, sink);
        cudaDeviceSynchronize();
        unsigned long long c[148];
        cudaMemcpy(c, d_cyc, sizeof(c), cudaMemcpyDeviceToHost);
        double cycles = 0;
        for (int i = 0; i < 148; i++) cycles += c[i];
        cycles /= 148;
        printf("%-24s %8.2f lane-ops/clk/SM  (%.0f cycles)\n", nm, (double)NT * ITERS / cycles, cycles);
    };
    for (int rep = 0; rep < 2; rep++) {
        run(k_sts, "STS.32 spread");
        run(k_atoms, "ATOMS.OR spread");
        run(k_atoms2, "ATOMS.OR 2 lanes/word");
        run_alu<0>(d_cyc, sd, sf, clk);
        run_alu<1>(d_cyc, sd, sf, clk);
        run_alu<2>(d_cyc, sd, sf, clk);
        run_alu<3>(d_cyc, sd, sf, clk);
        run_alu<4>(d_cyc, sd, sf, clk);
        run_alu<5>(d_cyc, sd, sf, clk);
        run_alu<6>(d_cyc, sd, sf, clk);
        run_alu<7>(d_cyc, sd, sf, clk);
        run_alu<8>(d_cyc, sd, sf, clk);
        run_alu<9>(d_cyc, sd, sf, clk);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
