// apax_device.cuh -- shared device helpers for the B200 APAX kernels.
//
// Bit-exactness rules: every TU is compiled with
// -fmad=false so no multiply-add on a bit-deciding path is contracted; IEEE
// division/sqrt are used explicitly; numpy's pairwise summation order is
// reproduced exactly (block_pairwise_*).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/apax_status.h"

namespace apax {

constexpr int kNT = 256;           // threads per CTA (encode / decode)
constexpr int kWarps = kNT / 32;
constexpr int kFileHeader = 28;
constexpr int kMaxExponent = 34;
constexpr int kScaleCodeOne = 31 << 10;

// ---------------------------------------------------------------------------
// dtype traits.  Wire codes: i8 0, i16 1, i32 2, f32 3, f64 4
// (reference dtypes.py:24-28).  Q = storage type of quantized samples;
// WIDE = first/second differences need 64-bit arithmetic.
// ---------------------------------------------------------------------------
template <int DT> struct DT_;
template <> struct DT_<0> { using T = int8_t;  using Q = int32_t; static constexpr bool F = false, WIDE = false; static constexpr int W = 1, HDR = 4; static constexpr long long LO = -128LL, HI = 127LL; };
template <> struct DT_<1> { using T = int16_t; using Q = int32_t; static constexpr bool F = false, WIDE = false; static constexpr int W = 2, HDR = 4; static constexpr long long LO = -32768LL, HI = 32767LL; };
template <> struct DT_<2> { using T = int32_t; using Q = int32_t; static constexpr bool F = false, WIDE = true;  static constexpr int W = 4, HDR = 4; static constexpr long long LO = -2147483648LL, HI = 2147483647LL; };
template <> struct DT_<3> { using T = float;   using Q = int32_t; static constexpr bool F = true,  WIDE = true;  static constexpr int W = 4, HDR = 6; static constexpr long long LO = 0, HI = 0; };
template <> struct DT_<4> { using T = double;  using Q = long long; static constexpr bool F = true, WIDE = true; static constexpr int W = 8, HDR = 6; static constexpr long long LO = 0, HI = 0; };
// cast variants of the generic encoder (kKdtI64, kKdtF64F32 below)
template <> struct DT_<5> { using T = long long; using Q = long long; static constexpr bool F = false, WIDE = true; static constexpr int W = 8, HDR = 4; static constexpr long long LO = 0, HI = 0; };
template <> struct DT_<6> { using T = double;  using Q = long long; static constexpr bool F = true, WIDE = true; static constexpr int W = 8, HDR = 6; static constexpr long long LO = 0, HI = 0; };

// kernel sample types beyond the container dtypes: encode_stream's casts
// (reference codec.py:266-272 widens every input to int64 / float64 first)
constexpr int kKdtI64 = 5;      // int64 samples, integer container (clip at decode)
constexpr int kKdtF64F32 = 6;   // float64 samples, f32 container
__host__ __device__ inline bool kdt_float(int dt) { return dt == 3 || dt == 4 || dt == kKdtF64F32; }
__host__ __device__ inline int hdr_size(int dt) { return kdt_float(dt) ? 6 : 4; }
__host__ __device__ inline int dt_width(int dt) {
    return dt == 0 ? 1 : dt == 1 ? 2 : (dt == 2 || dt == 3) ? 4 : 8;
}

// worst-case block bytes for samples of kernel type dt: group exponents are
// bounded by 8w+2 for native integer samples, 34 otherwise
__host__ __device__ inline long long max_block_bytes(int dt, int bs) {
    long long g = bs / 4;
    long long emax = (kdt_float(dt) || dt == kKdtI64) ? 34
                   : (8LL * dt_width(dt) + 2 < 34 ? 8LL * dt_width(dt) + 2 : 34);
    return hdr_size(dt) + (3 * g + 1) / 2 + (4 * emax * g + 7) / 8;
}
// worst case of any valid container block (a decoder must take every block
// the reference's decoder takes, exponents up to 34 whatever the dtype)
__host__ __device__ inline long long max_block_bytes_any(int dt, int bs) {
    long long g = bs / 4;
    return hdr_size(dt) + (3 * g + 1) / 2 + (4 * 34 * g + 7) / 8;
}

// ---------------------------------------------------------------------------
// scale code (reference dtypes.py:109-128) as exact bit manipulation:
// code = ((unbiased exponent + 31) << 10) | top 10 fraction bits; valid for
// a in [2^-31, 2^33) (callers guarantee the range).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int encode_scale_code(double a) {
    unsigned long long b = (unsigned long long)__double_as_longlong(a);
    int e = (int)((b >> 52) & 0x7FF) - 1023;
    int f = (int)((b >> 42) & 0x3FF);
    return ((e + 31) << 10) | f;
}
__host__ __device__ __forceinline__ double decode_scale_code(int code) {
    int e = code >> 10, f = code & 0x3FF;
    // ldexp(1024 + f, e - 41): exact
    return (double)(1024 + f) * ldexp(1.0, e - 41);
}

// ---------------------------------------------------------------------------
// floor(math.log2(s)) as glibc computes it (codec.py:120): log2 rounded to
// nearest, then floored.  Only values just below a power of two can round
// up to the next integer; that is decided exactly here.
// ---------------------------------------------------------------------------
__device__ inline long long floor_log2_rn(double s) {
    int e = ilogb(s);                       // exact floor(log2 s) for normal s
    double m = scalbn(s, -e);               // [1, 2)
    if (m < 2.0 - 0x1p-40) return e;
    // log2(s) = e + 1 - t with t = -log2(m/2) > 0 (tiny)
    double delta = 2.0 - m;                 // exact (Sterbenz)
    double h = 0.5 * delta;                 // 1 - m/2
    double t = (h + 0.5 * h * h) * 1.4426950408889634;  // -log2(1-h) ~ (h + h^2/2)/ln 2
    long long k1 = (long long)e + 1;        // candidate integer
    if (k1 == 0) return e;                  // value = -t != 0 -> floor is -1 = e
    double ak = fabs((double)k1);
    int ek = ilogb(ak);
    double ulp = ldexp(1.0, ek - 52);
    // spacing on the side where e+1-t lies: below k1 for k1 > 0 (toward 0),
    // above |k1| in magnitude for k1 < 0.
    double half;
    if (k1 > 0) half = (ak == ldexp(1.0, ek)) ? 0.25 * ulp : 0.5 * ulp;
    else half = 0.5 * ulp;
    // round-half-even: at an exact tie k1 (integer, low bit of mantissa 0 for
    // |k1| < 2^52) wins; ties are measure-zero for t from a real log anyway.
    return (t <= half) ? k1 : (long long)e;
}

// ---------------------------------------------------------------------------
// warp / CTA reductions (all threads of the CTA must call)
// ---------------------------------------------------------------------------
template <typename T, typename Op>
__device__ __forceinline__ T warp_allreduce(T v, Op op) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

struct MaxOp { template <typename T> __device__ __forceinline__ T operator()(T a, T b) const { return a > b ? a : b; } };
struct SumOp { template <typename T> __device__ __forceinline__ T operator()(T a, T b) const { return a + b; } };
struct MinOp { template <typename T> __device__ __forceinline__ T operator()(T a, T b) const { return a < b ? a : b; } };

// bswap of a 32-bit word (MSB-first bitstream <-> little-endian smem words)
__device__ __forceinline__ uint32_t bswap32(uint32_t v) { return __byte_perm(v, 0, 0x0123); }

// MSB-first bit writer into a zeroed word buffer; every word is merged with
// atomicOr so neighbouring threads may share boundary words.
struct BitWriter {
    uint32_t* w;
    unsigned long long acc;
    int nacc;
    long long wpos;
    __device__ __forceinline__ void init(uint32_t* words, long long bitpos) {
        w = words;
        wpos = bitpos >> 5;
        nacc = (int)(bitpos & 31);
        acc = 0;
    }
    __device__ __forceinline__ void put32(uint32_t v, int nb) {  // nb in [1, 32]
        acc |= ((unsigned long long)v << (64 - nacc - nb));
        nacc += nb;
        if (nacc >= 32) {
            atomicOr(&w[wpos], bswap32((uint32_t)(acc >> 32)));
            acc <<= 32;
            nacc -= 32;
            wpos++;
        }
    }
    __device__ __forceinline__ void put(unsigned long long v, int nb) {  // nb in [0, 64]
        if (nb > 32) {
            put32((uint32_t)(v >> 32) & (0xffffffffu >> (64 - nb)), nb - 32);
            put32((uint32_t)v, 32);
        } else if (nb > 0) {
            put32((uint32_t)v & (0xffffffffu >> (32 - nb)), nb);
        }
    }
    __device__ __forceinline__ void flush() {
        if (nacc > 0) atomicOr(&w[wpos], bswap32((uint32_t)(acc >> 32)));
    }
};

// group width of one sample (reference entropy.py:38-55): 0 for 0, else
// bit_length(v >= 0 ? v : -v-1) + 1.
__device__ __forceinline__ int width64(long long v) {
    unsigned long long u = (unsigned long long)(v ^ (v >> 63));
    return v == 0 ? 0 : 65 - __clzll((long long)u);
}
__device__ __forceinline__ int width32(int v) {
    unsigned u = (unsigned)(v ^ (v >> 31));
    return v == 0 ? 0 : 33 - __clz((int)u);
}

// x86 cvttsd2si semantics of numpy astype(int64) for out-of-range values
__device__ __forceinline__ long long f2i64(double v) {
    if (v >= -9223372036854775808.0 && v < 9223372036854775808.0) return (long long)v;
    return (long long)0x8000000000000000ULL;
}

// acquire / release helpers for the decoupled look-back
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

constexpr unsigned long long kFlagAgg = 1ULL << 62;
constexpr unsigned long long kFlagInc = 2ULL << 62;
constexpr unsigned long long kValMask = (1ULL << 62) - 1;

// ---------------------------------------------------------------------------
// Warp-parallel decoupled look-back over unit byte lengths (call with the
// whole warp).  Publishes AGG(len), sums predecessors 32 at a time until the
// nearest INC, publishes INC(prefix + len) and returns the exclusive prefix.
// ---------------------------------------------------------------------------
__device__ __forceinline__ long long warp_lookback(unsigned long long* lb, long long u, long long len) {
    const int lane = threadIdx.x & 31;
    if (u == 0) {
        if (lane == 0) st_release(&lb[0], kFlagInc | (unsigned long long)len);
        return 0;
    }
    if (lane == 0) st_release(&lb[u], kFlagAgg | (unsigned long long)len);
    long long prefix = 0;
    long long k = u - 1;
    for (;;) {
        const long long idx = k - lane;
        unsigned long long v = (idx >= 0) ? ld_acquire(&lb[idx]) : kFlagInc;
        const unsigned long long fl = v & ~kValMask;
        const unsigned inc = __ballot_sync(0xffffffffu, fl == kFlagInc);
        const unsigned nrd = __ballot_sync(0xffffffffu, fl == 0);
        const int first_inc = inc ? __ffs(inc) - 1 : 32;
        const unsigned need = first_inc >= 31 ? 0xffffffffu : ((2u << first_inc) - 1u);
        if (nrd & need) {       // a predecessor before the nearest INC is not ready
            __nanosleep(32);
            continue;
        }
        unsigned long long part = (lane <= first_inc) ? (v & kValMask) : 0ULL;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        prefix += (long long)part;
        if (inc) break;
        k -= 32;
    }
    if (lane == 0) st_release(&lb[u], kFlagInc | (unsigned long long)(prefix + len));
    return prefix;
}

// status words: [0] min non-finite index, [1] min (block << 8 | code) error
// key, [2] total output bytes / misc, [3] error detail
__device__ __forceinline__ void report_error(unsigned long long* status, long long block, int code) {
    atomicMin(&status[1], ((unsigned long long)block << 8) | (unsigned)code);
}

// ---------------------------------------------------------------------------
// byte copies from a 4-aligned word source (smem or global) to an arbitrary
// global byte range; bytes outside [dst, dst+len) are never written.
// ---------------------------------------------------------------------------
template <bool SRC_SHARED>
__device__ void copy_out(uint8_t* dst, const uint32_t* src, long long len) {
    if (len <= 0) return;
    const int tid = threadIdx.x;
    uintptr_t d0 = (uintptr_t)dst;
    long long head = (long long)((16 - (d0 & 15)) & 15);
    if (head > len) head = len;
    const uint8_t* sb = (const uint8_t*)src;
    for (long long i = tid; i < head; i += blockDim.x) dst[i] = sb[i];
    long long body = (len - head) & ~15LL;
    long long nchunks = body >> 4;
    uint4* d16 = (uint4*)(dst + head);
    const uint32_t sh = (uint32_t)(head & 3) * 8;
    const long long wbase = head >> 2;
    for (long long c = tid; c < nchunks; c += blockDim.x) {
        long long w = wbase + 4 * c;
        uint32_t a0 = src[w], a1 = src[w + 1], a2 = src[w + 2], a3 = src[w + 3], a4 = src[w + 4];
        uint4 v;
        v.x = __funnelshift_r(a0, a1, sh);
        v.y = __funnelshift_r(a1, a2, sh);
        v.z = __funnelshift_r(a2, a3, sh);
        v.w = __funnelshift_r(a3, a4, sh);
        d16[c] = v;
    }
    for (long long i = head + body + tid; i < len; i += blockDim.x) dst[i] = sb[i];
}

namespace tma {
// ---------------------------------------------------------------------------
// TMA bulk copy + mbarrier
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t sa(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(b)) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(sa(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(sa(dst)), "l"(src), "r"(bytes), "r"(sa(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(sa(bar)), "r"(phase) : "memory");
    }
}

}  // namespace tma

}  // namespace apax
