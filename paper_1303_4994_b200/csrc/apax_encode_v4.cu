// apax_encode_v4.cu -- block-parallel packer of the split encoder (bs 4096,
// i16 / i32 / f32 / f64 containers).
//
// The reference encoder (pkg/src/apax/codec.py:192-285) is a serial chain
// only through its gain: block j's scale code depends on block j-1's exact
// byte count (fixed rate, codec.py:228-243) or measured SRR (fixed quality,
// codec.py:244-252).  Everything else a block needs from its predecessors is
// local: the derivative history is the last two quantized samples of block
// j-1 (transform.py:31-49) and the selector is the argmin of block j-1's
// three stream costs (transform.py:107-113).  So the encode splits in two:
//
//   * the chain (apax_encode_v3.cu instantiated with META): per segment (or
//     per whole stream) it runs only what the gain recurrence needs and
//     writes each block's quantizer (multiplier, scale code, block exponent)
//     to a 16-byte record;
//   * this kernel: every block on its own CTA in ticket order, with no
//     serial dependency left: it re-quantizes the block with its record,
//     recomputes the previous block's last two samples for its history,
//     computes the three streams' group widths (entropy.py:38-55) and costs,
//     publishes them, takes the selector from block j-1's published costs,
//     codes the JEE tokens (entropy.py:63-104) and MSB-first mantissas
//     (entropy.py:222-240) into a shared-memory window and writes the block
//     straight to its final byte offset, found by a decoupled look-back over
//     the block lengths (no per-unit slot round trip).
//
// LOSSLESS needs no chain at all (gain 1: q = x), so a whole-stream LOSSLESS
// container is this one kernel.  The output is byte-identical to the
// reference (and to the fused v3 kernel).  Samples come straight from global
// memory into registers (16 contiguous samples per thread, 4 groups), the
// next block's samples are prefetched into L2 when its ticket is taken.
#include <cstdint>
#include <cuda_runtime.h>

#include "apax_device.cuh"
#include "apax_kernels.cuh"

namespace apax {
namespace v4 {

constexpr int NW = 8;              // warps
constexpr int NT = NW * 32;        // threads
constexpr int SPT = 16;            // samples per thread
constexpr int BS = 4096;           // block size of this kernel
constexpr int GB = BS / 4;         // groups of a full block
constexpr double kMagic = 6755399441055744.0;   // 1.5 * 2^52

// window bytes: the largest block of the dtype (exponents up to 8w+2 for
// native integers, 34 for floats) + 32 bytes of slack, 128-aligned
constexpr int win_bytes(int dt) {
    const int w = dt == 1 ? 2 : (dt == 4 ? 8 : 4);
    const int emax = dt >= 3 ? 34 : (8 * w + 2 < 34 ? 8 * w + 2 : 34);
    const int mb = (dt >= 3 ? 6 : 4) + (3 * GB + 1) / 2 + (4 * emax * GB + 7) / 8;
    return (mb + 32 + 127) & ~127;
}

struct __align__(16) St4 {
    long long blk, next;            // this CTA's current / next ticketed block
    unsigned pc[NW][2];             // per warp: s0 | s1 << 16, s2 | flips << 16
    unsigned edge[NW][2];           // widths (D0, D1, D2 bytes) of the warp's first / last group
    unsigned emw[NW];               // per warp: widest group (64-bit warps)
    unsigned jw[NW];                // JEE nibbles of the warp: lo16 carry-in 0, hi16 carry-in 1
    int jc[NW];                     // bit0: a thread breaks the pairing run, bit1: its carry-out
    int mbw[NW];                    // mantissa bits of the warp
    int monc[NW], monf[NW];         // exact monitor partials
    int sel, bad;
    long long prefix;
};

__device__ __forceinline__ void bar() { __syncthreads(); }
__device__ __forceinline__ int bitlen32(unsigned v) {
    int r;
    asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(v));
    return r + 1;
}
__device__ __forceinline__ int bitlen64(unsigned long long v) { return 64 - __clzll((long long)v); }
__device__ __forceinline__ unsigned wb32(int v) { return (unsigned)((v << 1) ^ v); }
__device__ __forceinline__ unsigned long long wb64(long long v) { return (unsigned long long)((v << 1) ^ v); }
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}

// consumed mask of the JEE positions given the carry-in (entropy.py:63-88 as
// a 2-state automaton: a pairable position not consumed by its predecessor
// consumes its successor)
__device__ __forceinline__ uint32_t consumed_word(uint32_t P, uint32_t cin, uint32_t* cout) {
    const uint32_t even = 0x55555555u;
    const uint32_t P2 = P & ~cin;
    const uint32_t follows = (P2 << 1) | cin;
    const uint32_t odd_starts = P2 & ~even & ~follows;
    unsigned long long s = (unsigned long long)odd_starts + P2;
    *cout = (uint32_t)(s >> 32);
    const uint32_t inv = (uint32_t)s << 1;
    return (even ^ inv) & follows;
}

// MSB-first piece writer: `c` (nb <= 32 bits) at bit `pos` of the window
__device__ __forceinline__ void put_bits(uint32_t* win, int pos, uint32_t c, int nb) {
    const uint32_t a = c << (32 - nb);
    const int sh = pos & 31;
    uint32_t* w = win + (pos >> 5);
    atomicOr(w, bswap32(a >> sh));
    if (sh + nb > 32) atomicOr(w + 1, bswap32(a << (32 - sh)));
}
__device__ __forceinline__ void put_bits64(uint32_t* win, int pos, unsigned long long c, int nb) {
    const unsigned long long a = c << (64 - nb);
    const int sh = pos & 31;
    uint32_t* w = win + (pos >> 5);
    atomicOr(w, bswap32((uint32_t)(a >> (32 + sh))));
    if (sh + nb > 32) atomicOr(w + 1, bswap32((uint32_t)(a >> sh)));
    if (sh + nb > 64) atomicOr(w + 2, bswap32((uint32_t)(a << (32 - sh))));
}

// quantize one sample with the block's multiplier (codec.py:94-132): the low
// word of x*sq + 1.5*2^52; x*sq is exact in f64 for <= 32-bit samples, f64
// samples round the product first (np.rint(x * scale))
template <int DT>
__device__ __forceinline__ int quant(typename DT_<DT>::T x, double sq) {
    if (DT == 4) return __double2loint(__dadd_rn(__dmul_rn((double)x, sq), kMagic));
    return __double2loint(__fma_rn((double)x, sq, kMagic));
}

// costs of a block as published for its successor: the three width sums
// (<= 34 * 1024 each) in 20-bit fields + a ready flag
__device__ __forceinline__ unsigned long long pack_costs(int t0, int t1, int t2) {
    return (1ULL << 63) | (unsigned long long)t0 | ((unsigned long long)t1 << 20) |
           ((unsigned long long)t2 << 40);
}

// copy `len` bytes of the window (4-aligned smem words) to global dst, any
// alignment; bytes outside [dst, dst+len) are not written
__device__ __forceinline__ void window_out(uint8_t* dst, const uint32_t* src, int len, int tid) {
    const uintptr_t d0 = (uintptr_t)dst;
    int head = (int)((16 - (d0 & 15)) & 15);
    if (head > len) head = len;
    const uint8_t* sb = (const uint8_t*)src;
    if (tid < head) dst[tid] = sb[tid];
    const int body = (len - head) & ~15;
    const int nchunks = body >> 4;
    uint4* d16 = (uint4*)(dst + head);
    const uint32_t sh = (uint32_t)(head & 3) * 8;
    const int wbase = head >> 2;
    for (int c = tid; c < nchunks; c += NT) {
        const int w = wbase + 4 * c;
        const uint32_t a0 = src[w], a1 = src[w + 1], a2 = src[w + 2], a3 = src[w + 3], a4 = src[w + 4];
        uint4 v;
        v.x = __funnelshift_r(a0, a1, sh);
        v.y = __funnelshift_r(a1, a2, sh);
        v.z = __funnelshift_r(a2, a3, sh);
        v.w = __funnelshift_r(a3, a4, sh);
        d16[c] = v;
    }
    const int t0 = head + body;
    if (tid < len - t0) dst[t0 + tid] = sb[t0 + tid];
}

// decoupled look-back over block lengths (one warp): exclusive prefix of
// block b from its predecessors' aggregate / inclusive records
__device__ __forceinline__ long long block_prefix(unsigned long long* lb, long long b) {
    const int lane = threadIdx.x & 31;
    long long prefix = 0;
    long long kk = b - 1;
    for (;;) {
        const long long idx = kk - lane;
        const unsigned long long v = (idx >= 0) ? ld_acquire(&lb[idx]) : kFlagInc;
        const unsigned long long fl = v & ~kValMask;
        const unsigned inc = __ballot_sync(0xffffffffu, fl == kFlagInc);
        const unsigned nrd = __ballot_sync(0xffffffffu, fl == 0);
        const int first_inc = inc ? __ffs(inc) - 1 : 32;
        const unsigned need = first_inc >= 31 ? 0xffffffffu : ((2u << first_inc) - 1u);
        if (nrd & need) {           // a predecessor is still coding: re-poll
            __nanosleep(32);
            continue;
        }
        unsigned long long part = (lane <= first_inc) ? (v & kValMask) : 0ULL;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        prefix += (long long)part;
        if (inc) break;
        kk -= 32;
    }
    return prefix;
}

template <int DT>
__global__ void __launch_bounds__(NT, 4) pack_kernel(EncParams P, const BlockMeta* __restrict__ meta,
                                                    unsigned long long* __restrict__ costs,
                                                    unsigned long long* __restrict__ lb) {
    using Tr = DT_<DT>;
    using T = typename Tr::T;
    constexpr bool F = Tr::F;
    constexpr int HS = Tr::HDR;
    constexpr int WB = win_bytes(DT);
    extern __shared__ __align__(128) unsigned char smem[];
    St4* S = (St4*)smem;
    uint8_t* wins = smem + ((sizeof(St4) + 127) & ~(size_t)127);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long nblk = P.n_blocks;
    const long long Pseg = P.unit_blocks;     // blocks per segment (n_blocks: whole stream)
    const bool warm = P.policy == 1 && P.mode == 1 && P.unit_blocks < P.n_blocks;

    // windows start zeroed; each block re-zeroes the bytes it copied out
    for (int i = tid; i < 2 * WB / 16; i += NT) ((uint4*)wins)[i] = make_uint4(0u, 0u, 0u, 0u);
    if (tid == 0) {
        S->blk = (long long)atomicAdd((unsigned long long*)P.ticket, 1ULL);
        if (S->blk < nblk) {
            const long long b = S->blk;
            const long long nb = (P.n - b * BS) < BS ? (P.n - b * BS) : BS;
            prefetch_l2((const T*)P.x + b * BS, (uint32_t)((nb * sizeof(T)) & ~15LL));
        }
    }
    bar();
    int kw = 0;         // window of this block
    int prev_len = 0;   // bytes the previous block used in the other window
    for (;;) {
        const long long b = S->blk;
        if (b >= nblk) break;
        uint32_t* win = (uint32_t*)(wins + kw * WB);
        // warm L2 with the samples of the block one grid-round ahead (some
        // CTA takes its ticket about when this one finishes)
        if (tid == 0) {
            const long long nb = b + gridDim.x;
            if (nb < nblk) {
                const long long nn = (P.n - nb * BS) < BS ? (P.n - nb * BS) : BS;
                prefetch_l2((const T*)P.x + nb * BS, (uint32_t)((nn * sizeof(T)) & ~15LL));
            }
        }
        const long long base = b * BS;
        const int n = (int)((P.n - base) < BS ? (P.n - base) : BS);
        const int G = (n + 3) >> 2;
        const int np = 4 * G;
        const bool restart = (b % Pseg) == 0;
        const double sq = meta ? meta[b].sq : 1.0;
        const int code = meta ? meta[b].code : kScaleCodeOne;
        const int fbe = meta ? meta[b].fbe : 0;
        const bool bwide = meta ? (meta[b].wide != 0) : false;
        const int p0 = 4 * tid;                       // first group of this thread
        const bool active = p0 < G;
        const int ng = active ? min(4, G - p0) : 0;   // valid groups of this thread

        // ---- samples -> q (registers), history ----
        int q[SPT];
        {
            const T* xs = (const T*)P.x + base + SPT * tid;
            if (n == BS) {
                if (sizeof(T) == 2) {
                    const uint4* x4 = (const uint4*)xs;
#pragma unroll
                    for (int m = 0; m < 2; m++) {
                        const uint4 v = __ldg(x4 + m);
                        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int k = 0; k < 4; k++) {
                            q[8 * m + 2 * k] = quant<DT>((T)(int16_t)(w[k] & 0xffffu), sq);
                            q[8 * m + 2 * k + 1] = quant<DT>((T)(int16_t)(w[k] >> 16), sq);
                        }
                    }
                } else if (sizeof(T) == 4) {
                    const uint4* x4 = (const uint4*)xs;
#pragma unroll
                    for (int m = 0; m < 4; m++) {
                        const uint4 v = __ldg(x4 + m);
                        q[4 * m] = quant<DT>(*(const T*)&v.x, sq);
                        q[4 * m + 1] = quant<DT>(*(const T*)&v.y, sq);
                        q[4 * m + 2] = quant<DT>(*(const T*)&v.z, sq);
                        q[4 * m + 3] = quant<DT>(*(const T*)&v.w, sq);
                    }
                } else {
                    const double2* x2 = (const double2*)xs;
#pragma unroll
                    for (int m = 0; m < 8; m++) {
                        const double2 v = __ldg(x2 + m);
                        q[2 * m] = quant<DT>((T)v.x, sq);
                        q[2 * m + 1] = quant<DT>((T)v.y, sq);
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < SPT; k++) q[k] = (SPT * tid + k < n) ? quant<DT>(xs[k], sq) : 0;
            }
        }
        // q[t0-1], q[t0-2]: the previous thread's last two samples, or the
        // history entering the block (the previous block's last two samples
        // quantized with its own multiplier; (0, 0) at a restart)
        int hq1 = __shfl_up_sync(0xffffffffu, q[SPT - 1], 1);
        int hq2 = __shfl_up_sync(0xffffffffu, q[SPT - 2], 1);
        if (lane == 0 && active) {
            if (tid > 0) {
                const T* xp = (const T*)P.x + base + SPT * tid;
                hq1 = quant<DT>(xp[-1], sq);
                hq2 = quant<DT>(xp[-2], sq);
            } else if (restart) {
                hq1 = 0; hq2 = 0;
            } else {
                const double sp = meta ? meta[b - 1].sq : 1.0;
                const T* xp = (const T*)P.x + base;
                hq1 = quant<DT>(xp[-1], sp);
                hq2 = quant<DT>(xp[-2], sp);
            }
        }

        // ---- phase C: group widths of D0/D1/D2 (entropy.py:38-55), costs,
        // sign flips (bound of the monitor's centre-frequency gate) ----
        uint32_t epk0 = 0u, epk1 = 0u, epk2 = 0u;   // byte g = width of group g
        int flips = 0;
        unsigned emax = 0;
        bool ww = bwide;
        if (!bwide) {
            if (active) {
                int m1 = hq1, dprev = hq1 - hq2;
                unsigned sgn = (unsigned)hq1 >> 31;
#pragma unroll
                for (int g = 0; g < 4; g++) {
                    unsigned o0 = 0, o1 = 0, o2 = 0;
#pragma unroll
                    for (int kk = 0; kk < 4; kk++) {
                        const int v0 = q[4 * g + kk];
                        const int v1 = v0 - m1;
                        const int v2 = v1 - dprev;
                        o0 |= wb32(v0); o1 |= wb32(v1); o2 |= wb32(v2);
                        sgn = __funnelshift_l((unsigned)v0, sgn, 1);
                        m1 = v0; dprev = v1;
                    }
                    if (g < ng) {
                        epk0 |= (uint32_t)bitlen32(o0) << (8 * g);
                        epk1 |= (uint32_t)bitlen32(o1) << (8 * g);
                        epk2 |= (uint32_t)bitlen32(o2) << (8 * g);
                    }
                }
                flips = __popc((sgn ^ (sgn >> 1)) & 0xffffu);
            }
            // 32-bit arithmetic is exact while every |q| <= 2^30 and every
            // |d1| < 2^30: floats guarantee the first by their headroom
            // (else the record says wide), integers check a D0 width of 32
            // (q outside [-2^30, 2^30)), and a D1 width of 32 flags the
            // second (wrapped differences included)
            bool bad = active && ((epk1 & 0x20202020u) != 0 || (!F && (epk0 & 0x20202020u) != 0));
            if (tid == 0) {
                const long long d = (long long)hq1 - (long long)hq2;
                bad = bad || d < -(1LL << 30) || d >= (1LL << 30) || hq1 < -(1 << 30) || hq1 > (1 << 30) ||
                      hq2 < -(1 << 30) || hq2 > (1 << 30);
            }
            ww = __any_sync(0xffffffffu, bad);
            if (ww) { epk0 = epk1 = epk2 = 0u; flips = 0; }
        }
        if (ww && active) {
            long long m1 = hq1, dprev = (long long)hq1 - (long long)hq2;
#pragma unroll
            for (int g = 0; g < 4; g++) {
                unsigned long long o0 = 0, o1 = 0, o2 = 0;
#pragma unroll
                for (int kk = 0; kk < 4; kk++) {
                    const long long v0 = q[4 * g + kk];
                    const long long v1 = v0 - m1;
                    const long long v2 = v1 - dprev;
                    o0 |= wb64(v0); o1 |= wb64(v1); o2 |= wb64(v2);
                    flips += (int)((unsigned long long)(v0 ^ m1) >> 63);
                    m1 = v0; dprev = v1;
                }
                if (g < ng) {
                    const int w0 = bitlen64(o0), w1 = bitlen64(o1), w2 = bitlen64(o2);
                    const unsigned wm = (unsigned)max(w0, max(w1, w2));
                    emax = wm > emax ? wm : emax;
                    epk0 |= (uint32_t)min(w0, 255) << (8 * g);
                    epk1 |= (uint32_t)min(w1, 255) << (8 * g);
                    epk2 |= (uint32_t)min(w2, 255) << (8 * g);
                }
            }
        }
        if (active && tid == 0) flips -= (int)((unsigned)(q[0] ^ hq1) >> 31);   // no predecessor in the block
        auto bsum = [](uint32_t e) -> int { return (int)__dp4a(e, 0x01010101u, 0u); };
        {
            const unsigned s01 = __reduce_add_sync(0xffffffffu, (unsigned)bsum(epk0) | ((unsigned)bsum(epk1) << 16));
            const unsigned s2f = __reduce_add_sync(0xffffffffu, (unsigned)bsum(epk2) | ((unsigned)flips << 16));
            const unsigned em = __reduce_max_sync(0xffffffffu, emax);
            // widths of the warp's first and last group (lane 0's group 0,
            // lane 31's group 3) for the neighbouring warps' JEE edges
            const unsigned f0 = __shfl_sync(0xffffffffu, (epk0 & 0xffu) | ((epk1 & 0xffu) << 8) | ((epk2 & 0xffu) << 16), 0);
            const unsigned l0 = __shfl_sync(0xffffffffu, (epk0 >> 24) | ((epk1 >> 24) << 8) | ((epk2 >> 24) << 16), 31);
            if (lane == 0) {
                S->pc[warp][0] = s01; S->pc[warp][1] = s2f;
                S->emw[warp] = em;
                S->edge[warp][0] = f0; S->edge[warp][1] = l0;
            }
        }
        bar();   // B1
        // the other window held the previous block, copied out before B1:
        // re-zero the bytes it used (this block's successor packs into it)
        {
            uint4* w4 = (uint4*)(wins + (kw ^ 1) * WB);
            for (int i = tid; i < (prev_len + 16 + 15) >> 4; i += NT) w4[i] = make_uint4(0u, 0u, 0u, 0u);
        }

        // ---- totals, costs for the successor, the exact gate, the selector ----
        int tt0, tt1, tt2, flt;
        {
            const int w = lane & (NW - 1);
            const unsigned a = lane < NW ? S->pc[w][0] : 0u, c = lane < NW ? S->pc[w][1] : 0u;
            const int a0 = (int)(a & 0xffffu), a1 = (int)(a >> 16), a2 = (int)(c & 0xffffu), af = (int)(c >> 16);
            tt0 = __reduce_add_sync(0xffffffffu, a0);
            tt1 = __reduce_add_sync(0xffffffffu, a1);
            tt2 = __reduce_add_sync(0xffffffffu, a2);
            flt = __reduce_add_sync(0xffffffffu, af);
        }
        if (tid == 0) st_release(&costs[b], pack_costs(tt0, tt1, tt2));
        int gate = 0;
        if (3LL * flt > 2LL * (np - 1)) {
            // exact monitor (transform.py:67-83): sign changes of the nonzero
            // subsequence of the padded q, in order across threads
            int ch = 0, fs = 0, lsg = 0;
            if (active) {
#pragma unroll
                for (int k = 0; k < SPT; k++) {
                    const int sg = (q[k] > 0) - (q[k] < 0);
                    if (SPT * tid + k < np && sg) {
                        if (lsg) ch += (sg != lsg);
                        else fs = sg;
                        lsg = sg;
                    }
                }
            }
            for (int o = 1; o < 32; o <<= 1) {
                const int och = __shfl_down_sync(0xffffffffu, ch, o);
                const int ofl = __shfl_down_sync(0xffffffffu, (fs + 1) | ((lsg + 1) << 2), o);
                if (((lane & (2 * o - 1)) == 0) && lane + o < 32) {
                    const int of = (ofl & 3) - 1, ol = ((ofl >> 2) & 3) - 1;
                    ch += och + ((lsg != 0 && of != 0 && lsg != of) ? 1 : 0);
                    if (!fs) fs = of;
                    if (ol) lsg = ol;
                }
            }
            if (lane == 0) { S->monc[warp] = ch; S->monf[warp] = (fs + 1) | ((lsg + 1) << 2); }
            bar();
            int ch2 = 0, f = 0, l = 0;
            for (int w = 0; w < NW; w++) {
                const int of = (S->monf[w] & 3) - 1, ol = ((S->monf[w] >> 2) & 3) - 1;
                ch2 += S->monc[w] + ((l != 0 && of != 0 && l != of) ? 1 : 0);
                if (!f) f = of;
                if (ol) l = ol;
            }
            gate = ((double)ch2 / (2.0 * (double)(np - 1))) > 1.0 / 3.0;
        }
        if (tid == 0) {
            int sel = 0;
            if (!restart) {
                // block b-1's costs (published by the CTA that holds it,
                // which took its ticket before this one)
                unsigned long long pcv;
                do { pcv = ld_acquire(&costs[b - 1]); } while (!(pcv >> 63));
                const int c0 = (int)(pcv & 0xfffffu), c1 = (int)((pcv >> 20) & 0xfffffu),
                          c2 = (int)((pcv >> 40) & 0xfffffu);
                sel = c1 < c0 ? 1 : 0;
                if (c2 < (sel ? c1 : c0)) sel = 2;
            } else if (warm) {
                // warm_self (App. C E8): prev_costs preset to the block's own
                // costs at the jumped gain
                sel = tt1 < tt0 ? 1 : 0;
                if (tt2 < (sel ? tt1 : tt0)) sel = 2;
            }
            if (gate) sel = 0;
            S->sel = sel;
            unsigned em = 0;
            for (int w = 0; w < NW; w++) em = S->emw[w] > em ? S->emw[w] : em;
            S->bad = em > (unsigned)kMaxExponent ? APAX_ERR_INTERNAL : 0;
            if (S->bad) report_error(P.status, b, S->bad);
            if (P.trace) {
                double* tr = P.trace + 10 * b;
                if (!meta) { tr[0] = 0.0; tr[1] = 1.0; tr[2] = kScaleCodeOne; tr[3] = 0.0; }   // LOSSLESS: gain 1
                tr[4] = sel;
                tr[5] = (double)(4LL * tt0 + 4LL * G); tr[6] = (double)(4LL * tt1 + 4LL * G);
                tr[7] = (double)(4LL * tt2 + 4LL * G);
                tr[9] = restart ? 1.0 : 0.0;
            }
        }
        bar();   // B2
        const int sel = S->sel;

        // ---- JEE structure of the selected stream (entropy.py:63-88):
        // pair / escape / valid masks of the thread's 4 positions, the carry
        // transfer, nibble and mantissa-bit counts in one packed warp scan ----
        const uint32_t esel = sel == 0 ? epk0 : (sel == 1 ? epk1 : epk2);
        int eprev = __shfl_up_sync(0xffffffffu, (int)(esel >> 24), 1);
        int enext = __shfl_down_sync(0xffffffffu, (int)(esel & 0xffu), 1);
        if (lane == 0 && warp > 0) eprev = (int)((S->edge[warp - 1][1] >> (8 * sel)) & 0xffu);
        if (lane == 31 && warp < NW - 1) enext = (int)((S->edge[warp + 1][0] >> (8 * sel)) & 0xffu);
        uint32_t Pb, Eb, Vb;
        unsigned jscan, jown, nonA, kbits;
        {
            const int e1 = (int)(esel & 0xffu), e2 = (int)((esel >> 8) & 0xffu);
            const int e3 = (int)((esel >> 16) & 0xffu), e4 = (int)(esel >> 24);
            const int d1 = e1 - eprev, d2 = e2 - e1, d3 = e3 - e2, d4 = e4 - e3, d5 = enext - e4;
            const uint32_t S1 = ((unsigned)(d1 + 1) < 3u ? 1u : 0u) | ((unsigned)(d2 + 1) < 3u ? 2u : 0u) |
                                ((unsigned)(d3 + 1) < 3u ? 4u : 0u) | ((unsigned)(d4 + 1) < 3u ? 8u : 0u) |
                                ((unsigned)(d5 + 1) < 3u ? 16u : 0u);
            const uint32_t S2 = ((unsigned)(d1 + 2) < 5u ? 1u : 0u) | ((unsigned)(d2 + 2) < 5u ? 2u : 0u) |
                                ((unsigned)(d3 + 2) < 5u ? 4u : 0u) | ((unsigned)(d4 + 2) < 5u ? 8u : 0u);
            const int npr = active ? max(0, min(4, G - 1 - p0)) : 0;   // positions with p + 1 < G
            Vb = (1u << ng) - 1u;
            const uint32_t first = (p0 == 0) ? 1u : 0u;                // position 0: always an escape
            Pb = S1 & (S1 >> 1) & ((1u << npr) - 1u) & ~first;
            Eb = Vb & ~Pb & (~S2 | first);
            const int mbo = 4 * bsum(esel);
            uint32_t c0o, c1o;
            const uint32_t C0 = consumed_word(Pb, 0u, &c0o) & 0xFu;
            const uint32_t C1 = consumed_word(Pb, 1u, &c1o) & 0xFu;
            const uint32_t T0 = Vb & ~C0, T1 = Vb & ~C1;
            const int n0 = __popc(T0) + 2 * __popc(T0 & Eb);
            const int n1 = __popc(T1) + 2 * __popc(T1 & Eb);
            const uint32_t co0 = (Pb >> 3) & ~(C0 >> 3) & 1u;
            nonA = __ballot_sync(0xffffffffu, Pb != 0xFu);
            kbits = __ballot_sync(0xffffffffu, co0 != 0);
            const unsigned below = nonA & ((1u << lane) - 1u);
            unsigned v;
            if (below) {
                const int cin = (kbits >> (31 - __clz((int)below))) & 1u;
                v = (unsigned)(cin ? n1 : n0) * 0x201u;
            } else {
                v = (unsigned)n0 | ((unsigned)n1 << 9);
            }
            v |= (unsigned)(mbo >> 2) << 18;
            jown = v;
            unsigned x = v;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned o = __shfl_up_sync(0xffffffffu, x, d);
                if (lane >= d) x += o;
            }
            jscan = x;
            if (lane == 31) {
                S->jw[warp] = (x & 0x1ffu) | (((x >> 9) & 0x1ffu) << 16);
                S->mbw[warp] = 4 * (int)(x >> 18);
                const int top = nonA ? 31 - __clz((int)nonA) : 0;
                S->jc[warp] = (nonA ? 1 : 0) | (nonA ? (int)(((kbits >> top) & 1u) << 1) : 0);
            }
        }
        bar();   // B3

        // ---- warp carry chain and prefixes (lanes 0..NW-1 = warps) ----
        int cin_w, nib_pre, mb_pre, nib_total, mb_total;
        {
            const int w = lane & (NW - 1);
            const unsigned jwv = S->jw[w];
            const int jcv = S->jc[w];
            const int mbv = S->mbw[w];
            int hk = (lane < NW) ? (jcv & 3) : 0;
#pragma unroll
            for (int d = 1; d < NW; d <<= 1) {
                const int o = __shfl_up_sync(0xffffffffu, hk, d);
                if (lane >= d && !(hk & 1)) hk = o;
            }
            const int phk = __shfl_up_sync(0xffffffffu, hk, 1);
            const int cin = (lane == 0) ? 0 : ((phk & 1) ? (phk >> 1) & 1 : 0);
            const int nw_ = (lane < NW) ? (int)(cin ? (jwv >> 16) : (jwv & 0xffffu)) : 0;
            const int mw_ = (lane < NW) ? mbv : 0;
            const unsigned own = (unsigned)nw_ | ((unsigned)(mw_ >> 2) << 14);
            unsigned nm = own;
#pragma unroll
            for (int d = 1; d < NW; d <<= 1) {
                const unsigned o = __shfl_up_sync(0xffffffffu, nm, d);
                if (lane >= d) nm += o;
            }
            const unsigned tot = __shfl_sync(0xffffffffu, nm, NW - 1);
            nib_total = (int)(tot & 0x3fffu);
            mb_total = 4 * (int)(tot >> 14);
            const unsigned pre = __shfl_sync(0xffffffffu, nm - own, warp);
            cin_w = __shfl_sync(0xffffffffu, cin, warp);
            nib_pre = (int)(pre & 0x3fffu);
            mb_pre = 4 * (int)(pre >> 14);
        }
        const int jee_bytes = (nib_total + 1) >> 1;
        const int blen = HS + jee_bytes + (mb_total + 7) / 8;
        // the block's byte offset: publish the aggregate, look back (warp 0)
        if (warp == 0) {
            long long prefix = 0;
            if (b == 0) {
                if (lane == 0) st_release(&lb[0], kFlagInc | (unsigned long long)blen);
            } else {
                if (lane == 0) st_release(&lb[b], kFlagAgg | (unsigned long long)blen);
                prefix = block_prefix(lb, b);
                if (lane == 0) st_release(&lb[b], kFlagInc | (unsigned long long)(prefix + blen));
            }
            if (lane == 0) {
                S->prefix = prefix;
                if (P.block_offsets) P.block_offsets[b] = kFileHeader + prefix;
                if (b == nblk - 1) {
                    P.status[2] = (unsigned long long)(kFileHeader + prefix + blen);
                    if (P.block_offsets) P.block_offsets[nblk] = kFileHeader + prefix + blen;
                }
                if (P.trace) P.trace[10 * b + 8] = (double)blen;
            }
        }
        const int bad = S->bad;

        // ---- phase D: header, JEE tokens, mantissas into the window ----
        const bool pack = !bad && !P.count_only;
        if (active && pack) {
            const unsigned below = nonA & ((1u << lane) - 1u);
            const int cin_t = below ? (int)((kbits >> (31 - __clz((int)below))) & 1u) : cin_w;
            const unsigned jx = jscan - jown;
            const int nib_off = nib_pre + (int)(cin_w ? ((jx >> 9) & 0x1ffu) : (jx & 0x1ffu));
            const int mb_off = mb_pre + 4 * (int)(jx >> 18);
            {
                uint32_t co;
                const uint32_t cons = consumed_word(Pb, (uint32_t)cin_t, &co) & 0xFu;
                const uint32_t Tm = Vb & ~cons;
                const int e[6] = {eprev, (int)(esel & 0xffu), (int)((esel >> 8) & 0xffu),
                                  (int)((esel >> 16) & 0xffu), (int)(esel >> 24), enext};
                unsigned long long acc = 0;
                int nbits = 0;
#pragma unroll
                for (int k2 = 0; k2 < 4; k2++) {
                    const int d = e[k2 + 1] - e[k2];
                    const bool tk = (Tm >> k2) & 1u;
                    const bool pk = (Pb >> k2) & 1u;
                    const bool xk = (Eb >> k2) & 1u;
                    const uint32_t val = pk ? (uint32_t)((d + 1) * 3 + (e[k2 + 2] - e[k2 + 1] + 1))
                                            : (xk ? (0xF00u | (uint32_t)e[k2 + 1]) : (uint32_t)(11 + d));
                    const int nb = tk ? (xk ? 12 : 4) : 0;
                    acc = (acc << nb) | (tk ? val : 0u);
                    nbits += nb;
                }
                const int pos = 8 * HS + 4 * nib_off;
                if (nbits > 32) {
                    put_bits(win, pos, (uint32_t)(acc >> 32) & (0xffffffffu >> (64 - nbits)), nbits - 32);
                    put_bits(win, pos + nbits - 32, (uint32_t)acc, 32);
                } else if (nbits > 0) {
                    put_bits(win, pos, (uint32_t)acc, nbits);
                }
            }
            int pos = 8 * (HS + jee_bytes) + mb_off;
            if (!ww) {
                auto emit_groups = [&](auto SELC) {
                    constexpr int SL = decltype(SELC)::value;
                    int m1 = hq1, dprev = hq1 - hq2;
#pragma unroll
                    for (int g = 0; g < 4; g++) {
                        int vs[4];
#pragma unroll
                        for (int kk = 0; kk < 4; kk++) {
                            const int v0 = q[4 * g + kk];
                            const int v1 = v0 - m1;
                            const int v2 = v1 - dprev;
                            m1 = v0; dprev = v1;
                            vs[kk] = SL == 0 ? v0 : (SL == 1 ? v1 : v2);
                        }
                        const int w = (int)((esel >> (8 * g)) & 0xffu);
                        if (g >= ng || w == 0) continue;
                        const uint32_t m = 0xffffffffu >> (32 - w);
                        if (w <= 16) {
                            const uint32_t pw = 1u << w;
                            const uint32_t hi = ((uint32_t)vs[0] & m) * pw + ((uint32_t)vs[1] & m);
                            const uint32_t lo = ((uint32_t)vs[2] & m) * pw + ((uint32_t)vs[3] & m);
                            put_bits64(win, pos, ((unsigned long long)hi << (2 * w)) | lo, 4 * w);
                        } else {
#pragma unroll
                            for (int kk = 0; kk < 4; kk++) put_bits(win, pos + kk * w, (uint32_t)vs[kk] & m, w);
                        }
                        pos += 4 * w;
                    }
                };
                if (sel == 0) emit_groups(std::integral_constant<int, 0>{});
                else if (sel == 1) emit_groups(std::integral_constant<int, 1>{});
                else emit_groups(std::integral_constant<int, 2>{});
            } else {
                long long m1 = hq1, dprev = (long long)hq1 - (long long)hq2;
#pragma unroll
                for (int g = 0; g < 4; g++) {
                    const int w = (int)((esel >> (8 * g)) & 0xffu);
#pragma unroll
                    for (int kk = 0; kk < 4; kk++) {
                        const long long v0 = q[4 * g + kk];
                        const long long v1 = v0 - m1;
                        const long long v2 = v1 - dprev;
                        m1 = v0; dprev = v1;
                        if (g < ng && w) {
                            const unsigned long long v = (unsigned long long)(sel == 0 ? v0 : (sel == 1 ? v1 : v2));
                            if (w > 32) {
                                put_bits(win, pos, (uint32_t)(v >> 32) & (0xffffffffu >> (64 - w)), w - 32);
                                put_bits(win, pos + w - 32, (uint32_t)v, 32);
                            } else {
                                put_bits(win, pos, (uint32_t)v & (0xffffffffu >> (32 - w)), w);
                            }
                            pos += w;
                        }
                    }
                }
            }
        }
        if (tid == 0 && !P.count_only) {
            // block header (dtypes.py:156-165)
            const uint32_t hb[6] = {(uint32_t)((sel & 3) | (restart ? 4 : 0)), (uint32_t)(code & 0xFF),
                                    (uint32_t)((code >> 8) & 0xFF), 0u, (uint32_t)(uint8_t)(int8_t)fbe, 0u};
            win[0] |= hb[0] | (hb[1] << 8) | (hb[2] << 16) | (hb[3] << 24);
            if (HS == 6) atomicOr(&win[1], hb[4] | (hb[5] << 8));
            if (b == 0) {   // the file header (codec.py:277-279)
                unsigned char h[kFileHeader];
                h[0] = 'A'; h[1] = 'P'; h[2] = 'A'; h[3] = 'X';
                h[4] = 1; h[5] = (unsigned char)DT; h[6] = (unsigned char)P.mode; h[7] = 0;
                for (int k2 = 0; k2 < 4; k2++) h[8 + k2] = (unsigned char)((unsigned)BS >> (8 * k2));
                for (int k2 = 0; k2 < 8; k2++) h[12 + k2] = (unsigned char)((unsigned long long)P.n >> (8 * k2));
                const unsigned long long tb = (unsigned long long)__double_as_longlong(P.target);
                for (int k2 = 0; k2 < 8; k2++) h[20 + k2] = (unsigned char)(tb >> (8 * k2));
                for (int k2 = 0; k2 < kFileHeader; k2++) P.out[k2] = h[k2];
            }
        }
        bar();   // B4: window complete, prefix known
        if (pack) window_out(P.out + kFileHeader + S->prefix, win, blen, tid);
        prev_len = P.count_only ? 0 : blen;
        // the next ticket only now: blocks start in ticket order, so a
        // block's predecessor is always already being coded
        if (tid == 0) S->blk = (long long)atomicAdd((unsigned long long*)P.ticket, 1ULL);
        kw ^= 1;
        bar();   // B5: S->blk of the next block
    }
}

}  // namespace v4

using v4::pack_kernel;

size_t encode_v4_smem_bytes(int dt) {
    return ((sizeof(v4::St4) + 127) & ~(size_t)127) + 2 * (size_t)v4::win_bytes(dt);
}

bool encode_v4_supported(int dt, int bs) { return bs == v4::BS && dt >= 1 && dt <= 4; }

static const void* v4_fn(int dt) {
    switch (dt) {
        case 1: return (const void*)pack_kernel<1>;
        case 2: return (const void*)pack_kernel<2>;
        case 3: return (const void*)pack_kernel<3>;
        default: return (const void*)pack_kernel<4>;
    }
}

int encode_v4_resident_ctas(int dt) {
    int dev = 0, nsm = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = encode_v4_smem_bytes(dt);
    cudaFuncSetAttribute(v4_fn(dt), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, v4_fn(dt), v4::NT, smem) != cudaSuccess || per < 1)
        per = 1;
    return per * (nsm > 0 ? nsm : 148);
}

// pack every block of the stream (P.n_blocks; P.unit_blocks = segment
// length, or n_blocks for a whole stream).  meta: per-block quantizer
// records from the chain (nullptr: LOSSLESS, gain 1).  costs / lb: n_blocks
// words each, zeroed; P.ticket zeroed.
int launch_encode_v4(int dt, const EncParams& P, const BlockMeta* meta, unsigned long long* costs,
                     unsigned long long* lb, cudaStream_t st) {
    const void* fn = v4_fn(dt);
    const size_t smem = encode_v4_smem_bytes(dt);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return APAX_ERR_CUDA;
    const int res = encode_v4_resident_ctas(dt);
    const long long g = P.n_blocks < res ? P.n_blocks : res;
    EncParams p = P;
    void* args[] = {&p, (void*)&meta, &costs, &lb};
    note_launches(1);
    // every CTA resident (a block waits only on lower tickets, held by running CTAs)
    if (cudaLaunchCooperativeKernel(fn, dim3((unsigned)g), dim3(v4::NT), args, smem, st) != cudaSuccess)
        return APAX_ERR_CUDA;
    return APAX_OK;
}

}  // namespace apax
