// Exhaustive-ish check: Markstein quotient q*rs + fma correction vs __ddiv_rn
// for every scale code mantissa M (s = M * 2^E) and integer q in a range.
#include <cstdio>
#include <cstdint>
__global__ void k(long long qlo, long long qhi, int E, unsigned long long* bad, unsigned long long* cnt) {
    int M = 1024 + blockIdx.y;               // 1024..2047
    double s = ldexp((double)M, E);
    double rs = __ddiv_rn(1.0, s);
    unsigned long long nb = 0, nc = 0;
    for (long long q = qlo + blockIdx.x * (long long)blockDim.x + threadIdx.x; q < qhi;
         q += (long long)gridDim.x * blockDim.x) {
        double r = (double)q;
        double y0 = r * rs;
        double e = __fma_rn(-s, y0, r);
        double y = __fma_rn(e, rs, y0);
        double ref = __ddiv_rn(r, s);
        nc++;
        if (__double_as_longlong(y) != __double_as_longlong(ref)) nb++;
        float yf = __double2float_rn(y), rf = __double2float_rn(ref);
        if (__float_as_int(yf) != __float_as_int(rf)) nb++;
    }
    atomicAdd(bad, nb);
    atomicAdd(cnt, nc);
}
int main() {
    unsigned long long *bad, *cnt;
    cudaMallocManaged(&bad, 8); cudaMallocManaged(&cnt, 8);
    int Es[] = {-41, -30, -20, -10, 0, 5, 20, -60, -100};
    for (int E : Es) {
        *bad = 0; *cnt = 0;
        k<<<dim3(256, 1024), 256>>>(-(1LL << 22), 1LL << 22, E, bad, cnt);
        cudaDeviceSynchronize();
        printf("E=%d checked=%llu mismatches=%llu\n", E, *cnt, *bad);
        *bad = 0; *cnt = 0;
        k<<<dim3(256, 1024), 256>>>((1LL << 31) - (1LL << 20), (1LL << 31), E, bad, cnt);
        cudaDeviceSynchronize();
        printf("E=%d high q checked=%llu mismatches=%llu\n", E, *cnt, *bad);
    }
    return 0;
}
