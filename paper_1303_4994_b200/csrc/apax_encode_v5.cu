// apax_encode_v5.cu -- B200 encoder, v5: segmented fixed-rate / fixed-quality
// containers of full 4096-sample blocks (i16 / i32 / f32), the headline path.
//
// Same contract and byte-exact output as apax_encode_v3.cu (reference
// encode_stream pkg/src/apax/codec.py:258-285, encode_block :192-255).  What
// changes is who does what inside the CTA that codes a segment:
//
//   * 8 pack warps (256 threads, 16 contiguous samples each) do the data
//     work of a block: the fixed-quality sums in numpy's pairwise order
//     (codec.py:248-249), quantization (codec.py:94-132) straight into
//     registers, the three streams' group widths (entropy.py:38-55) and
//     costs (transform.py:52-64), the JEE structure of the selected stream
//     (entropy.py:63-88) and the MSB-first emission (entropy.py:222-240).
//     q never leaves the registers between quantization and emission.
//     They also stage the next block (cp.async into a two-buffer ring, padded
//     leaf layout) and take its peak.
//   * 1 service warp runs everything scalar or asynchronous: the gain
//     recurrence (fixed-quality / fixed-rate update, attenuation ->
//     scale code -> quantizer multiplier, codec.py:94-132,155-189,228-252),
//     the window's bulk store to the segment's slot and its re-zeroing.
//
// The pack warps never wait for the scalar chain: in fixed-quality mode the
// service warp has the next block's quantizer ready while the pack warps
// are still coding the current block (the chain only needs the block's
// sums, which come first); in fixed-rate mode it overlaps the emission.
// Hand-offs are named barriers (bar.arrive on one side, bar.sync on the
// other) over double-buffered records, three blocking barriers per block
// for the pack warps instead of five CTA barriers with thread-0 sections.
#include <cstdint>
#include <cstdlib>
#include <type_traits>
#include <cuda_runtime.h>

#include "apax_device.cuh"
#include "apax_kernels.cuh"

namespace apax {
namespace v5 {

constexpr int NPW = 8;             // pack warps
constexpr int NPT = NPW * 32;      // pack threads
constexpr int NT = NPT + 32;       // + service warp
constexpr int BS = 4096;
constexpr int SPT = 16;            // samples per pack thread
constexpr int GB = BS / 4;
constexpr int ST_BYTES = 1024;
constexpr double kMagic = 6755399441055744.0;        // 1.5 * 2^52
constexpr double kMagicI = 6755401588539392.0;       // 1.5 * 2^52 + 2^31

constexpr int dtw(int dt) { return dt == 1 ? 2 : 4; }
constexpr int leaf_bytes(int dt) { return 128 * dtw(dt) + 32; }     // 128 samples + 8 words of padding
constexpr int x_bytes(int dt) { return 32 * leaf_bytes(dt); }
constexpr int win_bytes(int dt) {
    const int w = dtw(dt);
    const int emax = dt >= 3 ? 34 : (8 * w + 2 < 34 ? 8 * w + 2 : 34);
    const int mb = (dt >= 3 ? 6 : 4) + (3 * GB + 1) / 2 + (4 * emax * GB + 7) / 8;
    return (mb + 48 + 127) & ~127;
}

// the quantizer of one pass (service warp -> pack warps)
struct __align__(16) Blk {
    double sq;          // quantizer multiplier (floats: S, 0 for a zero block; ints: a_q)
    double sd, rs;      // dequantizer: divisor and its reciprocal (floats: S, 1/S; ints: a_q, 1/a_q)
    int code, fbe, wide, bad, idq, pad;
};
// the results of one pass (pack warps -> service warp)
struct __align__(16) Res {
    double pd[NPW], px[NPW];   // fixed quality: per-warp pairwise sums of (x-y)^2, x^2
    long long blen;            // exact block bytes
    int mincost;               // min of the three width sums
    int pad;
};
struct __align__(16) St {
    unsigned long long full[2];
    Blk blk[2];
    Res res[2];
    unsigned pc[NPW][2];       // per warp: s0 | s1 << 16, s2 | flips << 16
    unsigned edge[NPW][2];     // widths (D0, D1, D2 bytes) of the warp's first / last group
    unsigned emw[NPW];
    unsigned jw[NPW];          // JEE nibbles of the warp: lo16 carry-in 0, hi16 carry-in 1
    int jc[NPW];
    int mbw[NPW];
    int monc[NPW], monf[NPW];
    int hq[2][2];              // history entering the next block: q[n-1], q[n-2]
    unsigned pkw[2][NPW], pnw[2][NPW];   // per-warp peak partials of the next pass's block
    long long slot_len, slot_b0, slot_b1, fin_prefix;
    long long unit;
};
static_assert(sizeof(St) <= ST_BYTES, "St too large");

using namespace apax::tma;

#ifdef APAX_V5_PROF
__device__ unsigned long long g_prof[16];
#endif
#ifdef APAX_V5_TIMES
// per-CTA timeline (tools/cta_times.py): globaltimer at start, at the end of
// the last unit's coding, at exit; SM id
__device__ unsigned long long g_times[8192 * 4];
__device__ unsigned long long g_times2[8192 * 2];   // prefix known, copy done
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
template <int ID, int N> __device__ __forceinline__ void bar_sync() { asm volatile("bar.sync %0, %1;" :: "n"(ID), "n"(N) : "memory"); }
template <int ID, int N> __device__ __forceinline__ void bar_arrive() { asm volatile("bar.arrive %0, %1;" :: "n"(ID), "n"(N) : "memory"); }
// barrier ids: 1 quantizer ready (service -> pack), 2 window ready + widths done
// (service -> pack, pack <-> pack), 3 results ready (pack -> service), 4 window
// complete (pack -> service), 5 pack-only, 6 next block's peak ready (pack ->
// service), 7 unit end (everyone)
__device__ __forceinline__ int bitlen32(unsigned v) {
    int r;
    asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(v));
    return r + 1;
}
__device__ __forceinline__ int bitlen64(unsigned long long v) { return 64 - __clzll((long long)v); }
__device__ __forceinline__ unsigned wb32(int v) { return (unsigned)((v << 1) ^ v); }
__device__ __forceinline__ unsigned long long wb64(long long v) { return (unsigned long long)((v << 1) ^ v); }

__device__ __forceinline__ double scale_code_value(int code) {
    const unsigned long long e = (unsigned long long)(code >> 10), f = (unsigned long long)(code & 0x3FF);
    return __longlong_as_double((long long)(((e + 992ull) << 52) | (f << 42)));
}
__device__ __forceinline__ double clamp_att(double att, double lo) {
    double m = (lo > att) ? lo : att;
    return (0.0 < m) ? 0.0 : m;
}
__device__ __forceinline__ double att_to_a(double att) {
    double p = exp10(att / 20.0);  // 10.0 ** (att / 20.0) (dtypes.py:199)
    double m = (4.656612873077393e-10 > p) ? 4.656612873077393e-10 : p;
    return (1.0 < m) ? 1.0 : m;
}
__device__ __forceinline__ double clamp_step(double d) {
    double m = (d < 6.0) ? d : 6.0;
    return (m > -6.0) ? m : -6.0;
}
__device__ __forceinline__ unsigned long long pol_evict_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                 :: "l"(gdst), "r"(sa(ssrc)), "r"(bytes), "l"(pol_evict_last()) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void discard_l2(const void* p) {
    asm volatile("discard.global.L2 [%0], 128;" :: "l"(p) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src) : "memory");
}
// one net arrival per pack thread once its earlier cp.async copies have landed
__device__ __forceinline__ void stage_arrive(unsigned long long* bar) {
    asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" :: "r"(sa(bar)) : "memory");
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" :: "r"(sa(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init_n(unsigned long long* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sa(b)), "r"(n) : "memory");
}
// block b of the stream into a staging buffer, padded leaf layout: 16-byte
// chunk c of the block (c = tid + 256 k) goes to leaf c >> 5, chunk c & 31
// (i16: 16 chunks per leaf), all at immediate offsets from two per-thread bases
template <int DT>
__device__ __forceinline__ void stage_block(unsigned char* xbuf, const void* src, unsigned long long* bar) {
    constexpr int LB = leaf_bytes(DT);
    constexpr int CPL = 128 * dtw(DT) / 16;            // chunks per leaf (32 or 16)
    constexpr int NCH = BS * dtw(DT) / 16;             // chunks per block
    const int tid = threadIdx.x;
    const uint32_t d0 = sa(xbuf) + (uint32_t)((tid / CPL) * LB + (tid % CPL) * 16);
    const unsigned char* s0 = (const unsigned char*)src + tid * 16;
#pragma unroll
    for (int k = 0; k < NCH / NPT; k++)
        cp_async16(d0 + (uint32_t)(k * (NPT / CPL) * LB), s0 + k * NPT * 16);
    stage_arrive(bar);
}
__device__ __forceinline__ double warp_tree8(const double* v) {
    return ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
}

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
// OR a word into the window when it is non-zero: a predicated reduction (no
// branch around the atomic; a zero word is what a piece contributes to a word
// it does not reach)
__device__ __forceinline__ void or_word(uint32_t* w, uint32_t v) {
    asm volatile("{ .reg .pred p; setp.ne.u32 p, %1, 0; @p red.shared.or.b32 [%0], %1; }"
                 :: "r"(sa(w)), "r"(v) : "memory");
}
// MSB-first piece writers: `c` (nb bits) at bit position pos of the window
__device__ __forceinline__ void put_bits(uint32_t* win, int pos, uint32_t c, int nb) {
    const uint32_t a = c << (32 - nb);
    const int sh = pos & 31;
    uint32_t* w = win + (pos >> 5);
    or_word(w, bswap32(a >> sh));
    or_word(w + 1, bswap32(__funnelshift_r(0u, a, sh)));   // a << (32 - sh), 0 when sh == 0
}
__device__ __forceinline__ void put_bits64(uint32_t* win, int pos, unsigned long long c, int nb) {
    const unsigned long long a = c << (64 - nb);
    const int sh = pos & 31;
    const uint32_t hi = (uint32_t)(a >> 32), lo = (uint32_t)a;
    uint32_t* w = win + (pos >> 5);
    or_word(w, bswap32(hi >> sh));
    or_word(w + 1, bswap32(__funnelshift_r(lo, hi, sh)));
    or_word(w + 2, bswap32(__funnelshift_r(0u, lo, sh)));      // lo << (32 - sh), 0 when sh == 0
}

template <int DT>
__device__ __forceinline__ double xd_of(typename DT_<DT>::T xv) {
    if (DT_<DT>::F) return (double)xv;
    return __hiloint2double(0x43380000, (int)xv ^ (int)0x80000000) - kMagicI;
}
// rint(x * sq) as the low word of x*sq + 1.5*2^52 (x*sq is exact in f64 for
// <= 32-bit samples)
template <int DT>
__device__ __forceinline__ int quant(typename DT_<DT>::T x, double sq) {
    return __double2loint(__fma_rn(xd_of<DT>(x), sq, kMagic));
}
// dequantize (codec.py:135-146): Markstein quotient with the block's reciprocal
template <int DT>
__device__ __forceinline__ double deq_of(double qd, double s, double rs) {
    using Tr = DT_<DT>;
    const double y0 = qd * rs;
    const double e = __fma_rn(-s, y0, qd);
    const double y = __fma_rn(e, rs, y0);
    if (Tr::F) return (double)__double2float_rn(y);
    double yi = (y + kMagic) - kMagic;   // rint (|y| < 2^51)
    const double lo = (double)Tr::LO, hi = (double)Tr::HI;
    yi = yi < lo ? lo : (yi > hi ? hi : yi);
    return yi;
}

// the 16 contiguous samples of a pack thread, quantized
template <int DT>
__device__ __forceinline__ void load_q(const typename DT_<DT>::T* xc, double sq, int (&q)[SPT]) {
    using T = typename DT_<DT>::T;
    const uint4* x4 = (const uint4*)xc;
    if (sizeof(T) == 2) {
#pragma unroll
        for (int m = 0; m < 2; m++) {
            const uint4 v = x4[m];
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; k++) {
                q[8 * m + 2 * k] = quant<DT>((T)(int16_t)(w[k] & 0xffffu), sq);
                q[8 * m + 2 * k + 1] = quant<DT>((T)(int16_t)(w[k] >> 16), sq);
            }
        }
    } else {
#pragma unroll
        for (int m = 0; m < 4; m++) {
            const uint4 v = x4[m];
            q[4 * m] = quant<DT>(*(const T*)&v.x, sq);
            q[4 * m + 1] = quant<DT>(*(const T*)&v.y, sq);
            q[4 * m + 2] = quant<DT>(*(const T*)&v.z, sq);
            q[4 * m + 3] = quant<DT>(*(const T*)&v.w, sq);
        }
    }
}

// ---------------------------------------------------------------------------
// cold paths
// ---------------------------------------------------------------------------
// 64-bit widths of a thread's four groups (a block or warp whose differences
// may leave int32): epk0, epk1, epk2, flips | emax << 16
template <int DT>
__device__ __noinline__ uint4 cold_wide_widths(const typename DT_<DT>::T* xc, double sq, int hq1, int hq2) {
    int q[SPT];
    load_q<DT>(xc, sq, q);
    uint32_t epk0 = 0, epk1 = 0, epk2 = 0;
    int flips = 0;
    unsigned emax = 0;
    long long m1 = hq1, dprev = (long long)hq1 - (long long)hq2;
#pragma unroll 1
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
        const int w0 = bitlen64(o0), w1 = bitlen64(o1), w2 = bitlen64(o2);
        const unsigned wm = (unsigned)max(w0, max(w1, w2));
        emax = wm > emax ? wm : emax;
        epk0 |= (uint32_t)min(w0, 255) << (8 * g);
        epk1 |= (uint32_t)min(w1, 255) << (8 * g);
        epk2 |= (uint32_t)min(w2, 255) << (8 * g);
    }
    return make_uint4(epk0, epk1, epk2, (unsigned)flips | (emax << 16));
}
// 64-bit mantissa emission of a thread's four groups
template <int DT>
__device__ __noinline__ void cold_wide_emit(const typename DT_<DT>::T* xc, double sq, int hq1, int hq2, int sel,
                                            uint32_t esel, uint32_t* win, int pos) {
    int q[SPT];
    load_q<DT>(xc, sq, q);
    long long m1 = hq1, dprev = (long long)hq1 - (long long)hq2;
#pragma unroll 1
    for (int g = 0; g < 4; g++) {
        const int w = (int)((esel >> (8 * g)) & 0xffu);
#pragma unroll
        for (int kk = 0; kk < 4; kk++) {
            const long long v0 = q[4 * g + kk];
            const long long v1 = v0 - m1;
            const long long v2 = v1 - dprev;
            m1 = v0; dprev = v1;
            if (w) {
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
// exact monitor (transform.py:67-83) over the pack threads; q from smem
template <int DT>
__device__ __noinline__ int cold_monitor(const typename DT_<DT>::T* xc, double sq, St* S) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int q[SPT];
    load_q<DT>(xc, sq, q);
    int ch = 0, fs = 0, lsg = 0;
#pragma unroll
    for (int k = 0; k < SPT; k++) {
        const int sg = (q[k] > 0) - (q[k] < 0);
        if (sg) {
            if (lsg) ch += (sg != lsg);
            else fs = sg;
            lsg = sg;
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
    bar_sync<5, NPT>();
    int ch2 = 0, f = 0, l = 0;
    for (int w = 0; w < NPW; w++) {
        const int of = (S->monf[w] & 3) - 1, ol = ((S->monf[w] >> 2) & 3) - 1;
        ch2 += S->monc[w] + ((l != 0 && of != 0 && l != of) ? 1 : 0);
        if (!f) f = of;
        if (ol) l = ol;
    }
    bar_sync<5, NPT>();
    return ((double)ch2 / (2.0 * (double)(BS - 1))) > 1.0 / 3.0;
}
// first non-finite sample of a block in the padded leaf layout
template <int DT>
__device__ __noinline__ void cold_nonfinite(const unsigned char* xb, long long base, unsigned long long* status) {
    using T = typename DT_<DT>::T;
    for (int i = 0; i < BS; i++) {
        const T v = *(const T*)(xb + (i >> 7) * leaf_bytes(DT) + (i & 127) * (int)sizeof(T));
        if (!isfinite((double)v)) {
            atomicMin(&status[0], (unsigned long long)(base + i));
            break;
        }
    }
}

// copy len bytes from a 4-aligned global word source to an arbitrary byte offset
__device__ void group_copy_out(uint8_t* dst, const uint32_t* src, long long len, int lane, int nth) {
    if (len <= 0) return;
    const uintptr_t d0 = (uintptr_t)dst;
    long long head = (long long)((16 - (d0 & 15)) & 15);
    if (head > len) head = len;
    const uint8_t* sb = (const uint8_t*)src;
    if (lane < head) dst[lane] = sb[lane];
    const long long body = (len - head) & ~15LL;
    const long long nchunks = body >> 4;
    uint4* d16 = (uint4*)(dst + head);
    const uint32_t sh = (uint32_t)(head & 3) * 8;
    const long long wbase = head >> 2;
    long long c = lane;
    for (; c + 3 * nth < nchunks; c += 4 * nth) {
        uint32_t a[4][5];
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const long long w = wbase + 4 * (c + (long long)nth * r);
#pragma unroll
            for (int k = 0; k < 5; k++) a[r][k] = src[w + k];
        }
#pragma unroll
        for (int r = 0; r < 4; r++) {
            uint4 v;
            v.x = __funnelshift_r(a[r][0], a[r][1], sh);
            v.y = __funnelshift_r(a[r][1], a[r][2], sh);
            v.z = __funnelshift_r(a[r][2], a[r][3], sh);
            v.w = __funnelshift_r(a[r][3], a[r][4], sh);
            d16[c + (long long)nth * r] = v;
        }
    }
    for (; c < nchunks; c += nth) {
        const long long w = wbase + 4 * c;
        const uint32_t a0 = src[w], a1 = src[w + 1], a2 = src[w + 2], a3 = src[w + 3], a4 = src[w + 4];
        uint4 v;
        v.x = __funnelshift_r(a0, a1, sh);
        v.y = __funnelshift_r(a1, a2, sh);
        v.z = __funnelshift_r(a2, a3, sh);
        v.w = __funnelshift_r(a3, a4, sh);
        d16[c] = v;
    }
    for (long long i = head + body + lane; i < len; i += nth) dst[i] = sb[i];
}

// decoupled look-back (one warp): exclusive byte prefix of unit u
__device__ __forceinline__ long long unit_prefix(unsigned long long* lookback, long long u) {
    const int lane = threadIdx.x & 31;
    long long prefix = 0;
    long long kk = u - 1;
    unsigned nap = 256;
    // most of the wait is for the neighbours to finish coding: one lane
    // polls the predecessor's word (cheap) before the 32-wide look-back
    if (lane == 0) {
        while (ld_acquire(&lookback[u - 1]) == 0ULL) __nanosleep(1000);
    }
    __syncwarp();
    for (;;) {
        const long long idx = kk - lane;
        const unsigned long long v = (idx >= 0) ? ld_acquire(&lookback[idx]) : kFlagInc;
        const unsigned long long fl = v & ~kValMask;
        const unsigned inc = __ballot_sync(0xffffffffu, fl == kFlagInc);
        const unsigned nrd = __ballot_sync(0xffffffffu, fl == 0);
        const int first_inc = inc ? __ffs(inc) - 1 : 32;
        const unsigned need = first_inc >= 31 ? 0xffffffffu : ((2u << first_inc) - 1u);
        if (nrd & need) {
            __nanosleep(nap);
            nap = nap < 4096 ? 2 * nap : 4096;
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

// the finished unit, placed by all NT threads: warp 0 resolves the prefix,
// everyone copies from the slot to the final offset
__device__ __noinline__ void final_place(long long u, long long n_units, long long n_blocks,
                                        unsigned long long* lookback, unsigned long long* status,
                                        long long* block_offsets, uint8_t* out, St* S, uint8_t* slot) {
    const int tid = threadIdx.x;
    bar_sync<7, NT>();
    const long long len = S->slot_len;
    const long long b0 = S->slot_b0, b1 = S->slot_b1;
    if (tid < 32) {
        long long prefix = 0;
        if (u > 0) {
            prefix = unit_prefix(lookback, u);
            if (tid == 0) st_release(&lookback[u], kFlagInc | (unsigned long long)(prefix + len));
        }
#ifdef APAX_V5_TIMES
        if (tid == 0 && blockIdx.x < 8192) g_times2[2 * blockIdx.x] = gtimer();
#endif
        if (tid == 0) {
            S->fin_prefix = prefix;
            if (u == n_units - 1) {
                status[2] = (unsigned long long)(kFileHeader + prefix + len);
                if (block_offsets) block_offsets[n_blocks] = kFileHeader + prefix + len;
            }
        }
    }
    bar_sync<7, NT>();
    const long long prefix = S->fin_prefix;
    group_copy_out(out + kFileHeader + prefix, (const uint32_t*)slot, len, tid, NT);
    bar_sync<7, NT>();   // every thread has read its slot words: the lines are dead
#ifdef APAX_V5_TIMES
    if (tid == 0 && blockIdx.x < 8192) g_times2[2 * blockIdx.x + 1] = gtimer();
#endif
    for (long long l = (long long)tid * 128; l < len; l += (long long)NT * 128) discard_l2(slot + l);
    if (block_offsets)
        for (long long bb = b0 + tid; bb < b1; bb += NT) block_offsets[bb] += kFileHeader + prefix;
}

// ---------------------------------------------------------------------------
// the service warp: one unit
// ---------------------------------------------------------------------------
// what the service warp needs of the launch parameters (by value: a reference
// to the kernel's parameter block would force a local copy of it; keep it at
// 80 bytes -- a 96-byte version faulted in the noinline call)
struct SvcArgs {
    const void* x;
    unsigned long long* status;
    unsigned long long* lookback;
    long long* block_offsets;
    double* trace;
    double target, att_lo, pow10_t20, sqrt12;
    int mode;
};

template <int DT, bool FQ>
__device__ __noinline__ void service_unit(const SvcArgs P, St* S, unsigned char* xb0, uint32_t* win, uint8_t* slot,
                                          long long u, long long b0, long long b1, bool warm, uint32_t& phs) {
    using Tr = DT_<DT>;
    using T = typename Tr::T;
    constexpr bool F = Tr::F;
    constexpr int HS = Tr::HDR;
    constexpr int LB = leaf_bytes(DT);
    constexpr int XB = x_bytes(DT);
    constexpr bool NEED_PEAK = F || DT == 2;
    constexpr bool SQX = (DT != 2);
    const int lane = threadIdx.x & 31;
    const long long npass = (warm ? 1 : 0) + (b1 - b0);

    // CodecState (codec.py:66-82), lane 0
    double att = 0.0, a_cur = 1.0;
    int initialized = 0, emitted = 0;
    int tail_len = 0;
    long long wbase = 0;
    uint32_t tail[4] = {0u, 0u, 0u, 0u};
    bool store_pending = false;
    unsigned pk0 = 0, pn0 = 0;          // the first block's peak (warm_self codes it twice)

    // store the finished block of pass pk (block pb) to the slot and clean the window
    auto flush = [&](int pk, long long pb) {
        const long long blen = S->res[pk & 1].blen;
        const long long total = tail_len + blen;
        const long long full = total & ~15LL;
        if (lane == 0) {
            if (full > 0) {
                bulk_store(slot + wbase, win, (uint32_t)full);
                store_pending = true;
            }
            const int w0 = (int)(full >> 2);
            tail[0] = win[w0]; tail[1] = win[w0 + 1]; tail[2] = win[w0 + 2]; tail[3] = win[w0 + 3];
            if (P.block_offsets) P.block_offsets[pb] = wbase + tail_len;   // unit-relative
            if (store_pending) { bulk_wait_read(); }
        }
        __syncwarp();
        {
            uint4* w4 = (uint4*)win;
            int nz = (int)((total + 15 + 32) >> 4);
            nz = nz < win_bytes(DT) / 16 ? nz : win_bytes(DT) / 16;
            for (int i = lane; i < nz; i += 32) w4[i] = make_uint4(0u, 0u, 0u, 0u);
        }
        __syncwarp();
        wbase += full;
        tail_len = (int)(total - full);
        if (lane == 0) *(uint4*)win = make_uint4(tail[0], tail[1], tail[2], tail[3]);
    };

    for (long long kp = 0; kp < npass; kp++) {
        const bool pre = warm && kp == 0;                 // warm_self: cost-only pass at gain 1
        const long long bi = warm ? (kp == 0 ? 0 : kp - 1) : kp;
        const long long b = b0 + bi;
        const int buf = (int)(bi & 1);
        const unsigned char* xb = xb0 + buf * XB;
        const bool emit = !pre;
        // ---- peak of the block: the first pass reads it here, later passes take
        // the pack warps' partials (computed during the previous pass) ----
        unsigned pk = 0, pn = 0;
        if (kp == 0) {
            mbar_wait(&S->full[buf], (phs >> buf) & 1u);
            if (NEED_PEAK) {
                int ms = 0;
                unsigned mu = 0;
                int mx = 0, mn = 0;
#pragma unroll 4
                for (int k = 0; k < 32; k++) {
                    const uint4 v = *(const uint4*)(xb + k * LB + 16 * lane);
                    if (DT == 3) {
                        ms = __vimax3_s32(ms, (int)v.x, (int)v.y);
                        ms = __vimax3_s32(ms, (int)v.z, (int)v.w);
                        mu = __vimax3_u32(mu, v.x, v.y);
                        mu = __vimax3_u32(mu, v.z, v.w);
                    } else {
                        mx = __vimax3_s32(mx, (int)v.x, (int)v.y);
                        mx = __vimax3_s32(mx, (int)v.z, (int)v.w);
                        mn = __vimin3_s32(mn, (int)v.x, (int)v.y);
                        mn = __vimin3_s32(mn, (int)v.z, (int)v.w);
                    }
                }
                if (DT == 3) { pk = (unsigned)ms; pn = mu; }
                else { pk = (unsigned)mx; pn = (unsigned)(-(long long)mn); }
                pk = (unsigned)__reduce_max_sync(0xffffffffu, (int)pk);
                pn = __reduce_max_sync(0xffffffffu, pn);
            }
            pk0 = pk; pn0 = pn;
        }
        double px0 = 0.0;
        if (FQ && emit && !initialized) {
            // lane = leaf: numpy's 8 accumulators over the leaf's 16 rows, then the tree
            const T* xl = (const T*)(xb + lane * LB);
            double r[8];
#pragma unroll
            for (int j = 0; j < 8; j++) { const double xd = xd_of<DT>(xl[j]); r[j] = xd * xd; }
#pragma unroll 1
            for (int i = 1; i < 16; i++) {
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const double xd = xd_of<DT>(xl[8 * i + j]);
                    r[j] = SQX ? __fma_rn(xd, xd, r[j]) : r[j] + xd * xd;
                }
            }
            double t = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            px0 = t;
        }
        if (kp > 0) bar_sync<3, NT>();      // the previous pass's results
        int bad = 0;
        if (lane == 0) {
            // ---- the loops on the previous pass's results ----
            if (kp > 0) {
                const Res* R = &S->res[(kp - 1) & 1];
                const bool ppre = warm && kp == 1;
                if (ppre) {
                    // warm_self (App. C E8): the FR init jump from the gain-1 costs
                    const double bps0 = (double)(4LL * R->mincost + 4LL * GB + 8LL * HS) / (double)BS;
                    att = clamp_att(0.0 - 6.02 * (bps0 - P.target), P.att_lo);
                    a_cur = att_to_a(att);
                } else if (FQ) {
                    // quality loop (codec.py:244-252, 179-189)
                    const double px = warp_tree8(R->px), pd = warp_tree8(R->pd);
                    const double pxm = px / (double)BS, pdm = pd / (double)BS;
                    if (pxm > 0.0 && pdm != 0.0 && pxm / pdm == 0.0) bad = APAX_ERR_MATH_DOMAIN;
                    if (pxm > 0.0) {
                        const double measured = (pdm == 0.0) ? INFINITY : 10.0 * log10(pxm / pdm);
                        if (isfinite(measured))
                            att = clamp_att(att - clamp_step(0.5 * (measured - P.target)), P.att_lo);
                    }
                    a_cur = att_to_a(att);
                    if (bad) report_error(P.status, b - 1, bad);
                    bad = 0;
                    emitted += 1;
                } else {
                    // rate loop (codec.py:228-243) on the block's exact byte count
                    if (emitted == 0) {
                        const double bps0 = (double)(4LL * R->mincost + 4LL * GB + 8LL * HS) / (double)BS;
                        att = clamp_att(att - 6.02 * (bps0 - P.target), P.att_lo);
                    } else {
                        const double err = (double)(R->blen * 8) / (double)BS - P.target;
                        att = clamp_att(att - clamp_step(0.75 * err), P.att_lo);
                    }
                    a_cur = att_to_a(att);
                    emitted += 1;
                }
            }
        }
        if (kp > 0) {
            bar_sync<6, NT>();              // this pass's peak partials
            if (warm && kp == 1) { pk = pk0; pn = pn0; }
            else if (NEED_PEAK) {
                const int w = lane & (NPW - 1);
                pk = (unsigned)__reduce_max_sync(0xffffffffu, DT == 3 ? (int)S->pkw[kp & 1][w] : (int)S->pkw[kp & 1][w]);
                pn = __reduce_max_sync(0xffffffffu, S->pnw[kp & 1][w]);
            }
        }
        if (lane == 0) {
            // ---- S1: gain, scale code, quantizer (codec.py:94-132) ----
            double peak;
            bool nonfin = false;
            if (F) {
                const unsigned pos = ((int)pk >= 0) ? pk : 0u;
                const unsigned neg = (pn >= 0x80000000u) ? (pn & 0x7fffffffu) : 0u;
                const unsigned pkb = pos > neg ? pos : neg;
                nonfin = pkb >= 0x7f800000u;
                peak = (double)__uint_as_float(pkb);
            } else {
                peak = (double)((pk > pn) ? pk : pn);
            }
            if (nonfin) { mbar_wait(&S->full[buf], (phs >> buf) & 1u); cold_nonfinite<DT>(xb, b * (long long)BS, P.status); }
            if (emit && !initialized) {
                if (FQ) {  // _init_attenuation (codec.py:155-168)
                    const double rms = sqrt(px0 / (double)BS);
                    double att0 = 0.0;
                    if (rms != 0.0) {
                        const double rqa = F ? (1073741824.0 * rms) / peak : rms;
                        const double a0 = P.pow10_t20 / (P.sqrt12 * rqa);
                        const double m = (1e-300 > a0) ? 1e-300 : a0;
                        att0 = 20.0 * log10(m);
                    }
                    att = clamp_att(att0, P.att_lo);
                }
                initialized = 1;
                a_cur = att_to_a(att);
            }
            const double a = pre ? 1.0 : a_cur;
            int zero = 0, fbe = 0, code;
            double s = 1.0, aq = 1.0;
            long long qpk;
            if (!F) {
                code = encode_scale_code(a);
                aq = scale_code_value(code);
                qpk = (aq == 1.0) ? (long long)peak : (long long)rint(peak * aq);
                if (!NEED_PEAK) qpk = 32768;
            } else if (nonfin || peak == 0.0) {
                code = kScaleCodeOne; zero = 1; qpk = 0;
            } else {
                const double s_des = (a * 1073741824.0) / peak;
                if (!isfinite(s_des)) {
                    bad = APAX_ERR_OVERFLOW; code = kScaleCodeOne; zero = 1; qpk = 0;
                } else {
                    const unsigned long long sb = (unsigned long long)__double_as_longlong(s_des);
                    const long long l2 = ((sb & 0xFFFFFFFFFFFFFull) < 0xFFFFFFFFFF000ull && (sb >> 52) != 0)
                                             ? (long long)(sb >> 52) - 1023
                                             : floor_log2_rn(s_des);
                    long long fb = (-31 <= l2 && l2 <= 31) ? 0 : l2 - 31;
                    fb = fb < -127 ? -127 : (fb > 127 ? 127 : fb);
                    double rem = fb ? ldexp(s_des, (int)-fb) : s_des;
                    const double nxt = 8589934591.999999;
                    const double mm = (nxt < rem) ? nxt : rem;
                    rem = (mm > 4.656612873077393e-10) ? mm : 4.656612873077393e-10;
                    code = encode_scale_code(rem);
                    for (;;) {  // overflow guard (codec.py:126-131)
                        s = fb ? decode_scale_code(code) * ldexp(1.0, (int)fb) : scale_code_value(code);
                        const double qm = rint(peak * s);
                        if (qm < 2147483648.0 || fb <= -127) {
                            qpk = qm < 9.2e18 ? (long long)qm : (1LL << 62);
                            break;
                        }
                        fb -= 1;
                    }
                    fbe = (int)fb;
                }
            }
            Blk* B = &S->blk[kp & 1];
            B->code = code; B->fbe = fbe;
            B->sq = F ? (zero ? 0.0 : s) : aq;
            B->sd = F ? s : aq;
            B->rs = F ? __ddiv_rn(1.0, s) : ((aq != 1.0) ? __ddiv_rn(1.0, aq) : 1.0);
            B->idq = (!F && aq == 1.0) ? 1 : 0;
            B->wide = (qpk > (1LL << 30)) ? 1 : 0;
            B->bad = bad;
            if (emit && P.trace) {
                double* tr = P.trace + 10 * b;
                tr[0] = att; tr[1] = a; tr[2] = code; tr[3] = fbe;
            }
        }
        if (emit) initialized = 1;           // (every lane: the px0 branch above must stay convergent)
        __syncwarp();
        __threadfence_block();
        bar_arrive<1, NT>();                 // the pass's quantizer is ready
        if (kp > 0) {
            bar_sync<4, NT>();               // the previous pass is finished
            const bool ppre = warm && kp == 1;
            if (!ppre) {
                const long long pbi = warm ? kp - 2 : kp - 1;
                flush((int)(kp - 1), b0 + pbi);
            }
        }
        __threadfence_block();
        bar_arrive<2, NT>();                 // the window is clean
        if (emit) phs ^= 1u << buf;
    }
    // ---- unit end: the last pass's hand-offs (results, peak, window) ----
    bar_sync<3, NT>();
    bar_sync<6, NT>();
    bar_sync<4, NT>();
    {
        const long long pbi = (b1 - b0) - 1;
        if (FQ && lane == 0) {
            // the last block's quality-loop error status (codec.py:251)
            const Res* R = &S->res[(npass - 1) & 1];
            const double px = warp_tree8(R->px), pd = warp_tree8(R->pd);
            const double pxm = px / (double)BS, pdm = pd / (double)BS;
            if (pxm > 0.0 && pdm != 0.0 && pxm / pdm == 0.0) report_error(P.status, b1 - 1, APAX_ERR_MATH_DOMAIN);
        }
        flush((int)(npass - 1), b0 + pbi);
    }
    if (lane == 0) {
        if (store_pending) bulk_wait_all();
        if (tail_len > 0) *(uint4*)(slot + wbase) = make_uint4(tail[0], tail[1], tail[2], tail[3]);
        *(uint4*)win = make_uint4(0u, 0u, 0u, 0u);
        const long long Lu = wbase + tail_len;
        __threadfence();
        st_release(&P.lookback[u], (u == 0 ? kFlagInc : kFlagAgg) | (unsigned long long)Lu);
        S->slot_len = Lu; S->slot_b0 = b0; S->slot_b1 = b1;
        __threadfence_block();
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------
// the pack warps: one unit
// ---------------------------------------------------------------------------
template <int DT, bool FQ>
__device__ __forceinline__ void pack_unit(const EncParams& P, St* S, unsigned char* xb0, uint32_t* win,
                                          long long b0, long long b1, bool warm, uint32_t& phs) {
    using Tr = DT_<DT>;
    using T = typename Tr::T;
    constexpr bool F = Tr::F;
    constexpr int HS = Tr::HDR;
    constexpr int LB = leaf_bytes(DT);
    constexpr int LS = LB / (int)sizeof(T);     // leaf stride in samples
    constexpr int XB = x_bytes(DT);
 constexpr bool SQX = (DT != 2);
    constexpr bool NEED_PEAK = F || DT == 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nblk = (int)(b1 - b0);
    const int npass = (warm ? 1 : 0) + nblk;
#ifdef APAX_V5_PROF
    // phase cycles of thread 0 (tools/prof_v5.py): acc[k] += clock at mark k - clock at the previous mark
    unsigned long long prof_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long prof_last = clock64();
#define PMARK(k) do { if (tid == 0) { const long long c_ = clock64(); prof_acc[k] += (unsigned long long)(c_ - prof_last); prof_last = c_; } } while (0)
#else
#define PMARK(k) do { } while (0)
#endif
    int wb = 0;                 // window bytes carried in from the previous block (< 16)
    int sel_next = 0;           // argmin of the previous block's costs
    bool has_pc = false;
    auto bsum = [](uint32_t e) -> int { return (int)__dp4a(e, 0x01010101u, 0u); };

    // the unit's first two blocks (every buffer is free: the previous unit is placed)
    stage_block<DT>(xb0, (const T*)P.x + b0 * (long long)BS, &S->full[0]);
    if (b0 + 1 < b1) stage_block<DT>(xb0 + XB, (const T*)P.x + (b0 + 1) * (long long)BS, &S->full[1]);
    for (int kp = 0; kp < npass; kp++) {
        const bool pre = warm && kp == 0;
        const bool emit = !pre;
        const int bi = warm ? (kp == 0 ? 0 : kp - 1) : kp;
        const long long b = b0 + bi;
        const int buf = bi & 1;
        const bool restart = (bi == 0);
        PMARK(0);
        bar_sync<1, NT>();
        PMARK(1);
        const Blk* B = &S->blk[kp & 1];
        const double sq = B->sq;
        const bool bwide = B->wide != 0;
        mbar_wait(&S->full[buf], (phs >> buf) & 1u);
        if (emit) phs ^= 1u << buf;
        const T* xl = (const T*)(xb0 + buf * XB) + (tid >> 3) * LS;   // this thread's leaf
        // the other buffer's block is finished (every pack thread is past its
        // emission): stage the next block into it, four leaves per warp
        const bool has_next = bi + 1 < nblk;
        if (emit && bi >= 1 && has_next)
            stage_block<DT>(xb0 + (buf ^ 1) * XB, (const T*)P.x + (b + 1) * (long long)BS, &S->full[buf ^ 1]);

        // ---- fixed-quality sums, numpy's pairwise order (codec.py:248-249) ----
        if (FQ) {
            const double sd = B->sd, rs = B->rs;
            const bool idq = B->idq != 0;
            const T* xp = xl + (tid & 7);
            double rpd = 0.0, rpx = 0.0;
#pragma unroll
            for (int i = 0; i < 16; i++) {
                const double xd = xd_of<DT>(xp[8 * i]);
                const double qd = __fma_rn(xd, sq, kMagic) - kMagic;
                const double y = idq ? qd : deq_of<DT>(qd, sd, rs);
                const double d = xd - y;
                const double d2 = d * d;
                rpd = (i == 0) ? d2 : rpd + d2;
                rpx = (i == 0) ? xd * xd : (SQX ? __fma_rn(xd, xd, rpx) : rpx + xd * xd);
            }
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                rpd += __shfl_xor_sync(0xffffffffu, rpd, o);
                rpx += __shfl_xor_sync(0xffffffffu, rpx, o);
            }
            if (lane == 0) { S->res[kp & 1].pd[warp] = rpd; S->res[kp & 1].px[warp] = rpx; }
            __threadfence_block();
            bar_arrive<3, NT>();
        }

        PMARK(2);
        // ---- samples -> q (registers), history ----
        const T* xc = xl + SPT * (tid & 7);
        int q[SPT];
        load_q<DT>(xc, sq, q);
        int hq1 = __shfl_up_sync(0xffffffffu, q[SPT - 1], 1);
        int hq2 = __shfl_up_sync(0xffffffffu, q[SPT - 2], 1);
        if (lane == 0) {
            if (warp > 0) {
                const T* xh = xl - LS + 126;         // the previous leaf's last two samples
                hq2 = quant<DT>(xh[0], sq);
                hq1 = quant<DT>(xh[1], sq);
            } else if (restart) {
                hq1 = 0; hq2 = 0;
            } else {
                hq1 = S->hq[kp & 1][0]; hq2 = S->hq[kp & 1][1];
            }
        }
        if (tid == NPT - 1 && emit) { S->hq[(kp + 1) & 1][0] = q[SPT - 1]; S->hq[(kp + 1) & 1][1] = q[SPT - 2]; }

        // ---- group widths of D0/D1/D2 (entropy.py:38-55), costs, sign flips ----
        uint32_t epk0 = 0u, epk1 = 0u, epk2 = 0u;
        int flips = 0;
        unsigned emax = 0;
        bool ww = bwide;
        if (!bwide) {
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
                epk0 |= (uint32_t)bitlen32(o0) << (8 * g);
                epk1 |= (uint32_t)bitlen32(o1) << (8 * g);
                epk2 |= (uint32_t)bitlen32(o2) << (8 * g);
            }
            flips = __popc((sgn ^ (sgn >> 1)) & 0xffffu);
            // 32-bit arithmetic is exact while every |q| <= 2^30 and every
            // |d1| < 2^30 (see apax_encode_v4.cu)
            bool badw = (epk1 & 0x20202020u) != 0 || (!F && (epk0 & 0x20202020u) != 0);
            if (tid == 0) {
                const long long d = (long long)hq1 - (long long)hq2;
                badw = badw || d < -(1LL << 30) || d >= (1LL << 30) || hq1 < -(1 << 30) || hq1 > (1 << 30) ||
                       hq2 < -(1 << 30) || hq2 > (1 << 30);
            }
            ww = __any_sync(0xffffffffu, badw);
        }
        if (ww) {
            const uint4 r = cold_wide_widths<DT>(xc, sq, hq1, hq2);
            epk0 = r.x; epk1 = r.y; epk2 = r.z;
            flips = (int)(r.w & 0xffffu);
            emax = r.w >> 16;
        }
        if (tid == 0) flips -= (int)((unsigned)(q[0] ^ hq1) >> 31);   // no predecessor in the block
        {
            const unsigned s01 = __reduce_add_sync(0xffffffffu, (unsigned)bsum(epk0) | ((unsigned)bsum(epk1) << 16));
            const unsigned s2f = __reduce_add_sync(0xffffffffu, (unsigned)bsum(epk2) | ((unsigned)flips << 16));
            const unsigned em = __reduce_max_sync(0xffffffffu, emax);
            const unsigned f0 = __shfl_sync(0xffffffffu, (epk0 & 0xffu) | ((epk1 & 0xffu) << 8) | ((epk2 & 0xffu) << 16), 0);
            const unsigned l0 = __shfl_sync(0xffffffffu, (epk0 >> 24) | ((epk1 >> 24) << 8) | ((epk2 >> 24) << 16), 31);
            if (lane == 0) {
                S->pc[warp][0] = s01; S->pc[warp][1] = s2f;
                S->emw[warp] = em;
                S->edge[warp][0] = f0; S->edge[warp][1] = l0;
            }
        }
        // ---- peak of the next block (staged at the start of this pass, landed by now) for the
        // service warp's next quantizer ----
        if (NEED_PEAK && has_next) {
            const int nbuf = buf ^ 1;
            mbar_wait(&S->full[nbuf], (phs >> nbuf) & 1u);
            const uint4* xn = (const uint4*)((const T*)(xb0 + nbuf * XB) + (tid >> 3) * LS + SPT * (tid & 7));
            unsigned pk, pn;
            if (DT == 3) {
                int ms = 0;
                unsigned mu = 0;
#pragma unroll
                for (int m = 0; m < 4; m++) {
                    const uint4 v = xn[m];
                    ms = __vimax3_s32(ms, (int)v.x, (int)v.y);
                    ms = __vimax3_s32(ms, (int)v.z, (int)v.w);
                    mu = __vimax3_u32(mu, v.x, v.y);
                    mu = __vimax3_u32(mu, v.z, v.w);
                }
                pk = (unsigned)__reduce_max_sync(0xffffffffu, ms);
                pn = __reduce_max_sync(0xffffffffu, mu);
            } else {
                int mx = 0, mi = 0;
#pragma unroll
                for (int m = 0; m < 4; m++) {
                    const uint4 v = xn[m];
                    mx = __vimax3_s32(mx, (int)v.x, (int)v.y);
                    mx = __vimax3_s32(mx, (int)v.z, (int)v.w);
                    mi = __vimin3_s32(mi, (int)v.x, (int)v.y);
                    mi = __vimin3_s32(mi, (int)v.z, (int)v.w);
                }
                pk = (unsigned)__reduce_max_sync(0xffffffffu, mx);
                pn = (unsigned)(-(long long)__reduce_min_sync(0xffffffffu, mi));
            }
            if (lane == 0) { S->pkw[(kp + 1) & 1][warp] = pk; S->pnw[(kp + 1) & 1][warp] = pn; }
        }
        __threadfence_block();
        bar_arrive<6, NT>();

        PMARK(3);
        bar_sync<2, NT>();   // every warp's widths; the window is clean
        PMARK(4);

        // ---- totals, the exact gate, the selector ----
        int tt0, tt1, tt2, flt;
        unsigned emt;
        {
            const int w = lane & (NPW - 1);
            const unsigned a = lane < NPW ? S->pc[w][0] : 0u, c = lane < NPW ? S->pc[w][1] : 0u;
            const unsigned e = lane < NPW ? S->emw[w] : 0u;
            tt0 = __reduce_add_sync(0xffffffffu, (int)(a & 0xffffu));
            tt1 = __reduce_add_sync(0xffffffffu, (int)(a >> 16));
            tt2 = __reduce_add_sync(0xffffffffu, (int)(c & 0xffffu));
            flt = __reduce_add_sync(0xffffffffu, (int)(c >> 16));
            emt = __reduce_max_sync(0xffffffffu, e);
        }
        int mn = tt0 < tt1 ? tt0 : tt1;
        mn = tt2 < mn ? tt2 : mn;
        int own = tt1 < tt0 ? 1 : 0;
        if (tt2 < (own ? tt1 : tt0)) own = 2;
        if (pre) {
            // cost-only pass: the service warp turns the costs into the init jump
            if (tid == 0) {
                S->res[kp & 1].mincost = mn;
                if (emt > (unsigned)kMaxExponent) report_error(P.status, b, APAX_ERR_INTERNAL);
            }
            __threadfence_block();
            bar_arrive<3, NT>();
            bar_arrive<4, NT>();
            continue;
        }
        // exact monitor only when the sign-flip bound cannot rule out the 1/3
        // gate (transform.py:67-83,107-113)
        const int gate = (3LL * flt > 2LL * (BS - 1)) ? cold_monitor<DT>(xc, sq, S) : 0;
        int sel_pre = has_pc ? sel_next : 0;
        if (warm && restart) sel_pre = own;   // warm_self: the block's own costs
        const int sel = gate ? 0 : sel_pre;
        sel_next = own;
        has_pc = true;

        // ---- JEE structure of the selected stream (entropy.py:63-88) ----
        const uint32_t esel = sel == 0 ? epk0 : (sel == 1 ? epk1 : epk2);
        int eprev = __shfl_up_sync(0xffffffffu, (int)(esel >> 24), 1);
        int enext = __shfl_down_sync(0xffffffffu, (int)(esel & 0xffu), 1);
        if (lane == 0 && warp > 0) eprev = (int)((S->edge[warp - 1][1] >> (8 * sel)) & 0xffu);
        if (lane == 31 && warp < NPW - 1) enext = (int)((S->edge[warp + 1][0] >> (8 * sel)) & 0xffu);
        uint32_t Pb, Eb;
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
            const uint32_t npm = (tid == NPT - 1) ? 7u : 15u;        // positions with p + 1 < G
            const uint32_t first = (tid == 0) ? 1u : 0u;             // position 0: always an escape
            Pb = S1 & (S1 >> 1) & npm & ~first;
            Eb = 0xFu & ~Pb & (~S2 | first);
            const int mbo = 4 * bsum(esel);
            uint32_t c0o, c1o;
            const uint32_t C0 = consumed_word(Pb, 0u, &c0o) & 0xFu;
            const uint32_t C1 = consumed_word(Pb, 1u, &c1o) & 0xFu;
            const uint32_t T0 = 0xFu & ~C0, T1 = 0xFu & ~C1;
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
        PMARK(5);
        bar_sync<5, NPT>();
        PMARK(6);

        // ---- warp carry chain and prefixes (lanes 0..NPW-1 = warps) ----
        int cin_w, nib_pre, mb_pre, nib_total, mb_total;
        {
            const int w = lane & (NPW - 1);
            const unsigned jwv = S->jw[w];
            const int jcv = S->jc[w];
            const int mbv = S->mbw[w];
            int hk = (lane < NPW) ? (jcv & 3) : 0;
#pragma unroll
            for (int d = 1; d < NPW; d <<= 1) {
                const int o = __shfl_up_sync(0xffffffffu, hk, d);
                if (lane >= d && !(hk & 1)) hk = o;
            }
            const int phk = __shfl_up_sync(0xffffffffu, hk, 1);
            const int cin = (lane == 0) ? 0 : ((phk & 1) ? (phk >> 1) & 1 : 0);
            const int nw_ = (lane < NPW) ? (int)(cin ? (jwv >> 16) : (jwv & 0xffffu)) : 0;
            const int mw_ = (lane < NPW) ? mbv : 0;
            const unsigned ownw = (unsigned)nw_ | ((unsigned)(mw_ >> 2) << 14);
            unsigned nm = ownw;
#pragma unroll
            for (int d = 1; d < NPW; d <<= 1) {
                const unsigned o = __shfl_up_sync(0xffffffffu, nm, d);
                if (lane >= d) nm += o;
            }
            const unsigned tot = __shfl_sync(0xffffffffu, nm, NPW - 1);
            nib_total = (int)(tot & 0x3fffu);
            mb_total = 4 * (int)(tot >> 14);
            const unsigned prew = __shfl_sync(0xffffffffu, nm - ownw, warp);
            cin_w = __shfl_sync(0xffffffffu, cin, warp);
            nib_pre = (int)(prew & 0x3fffu);
            mb_pre = 4 * (int)(prew >> 14);
        }
        const int jee_bytes = (nib_total + 1) >> 1;
        const int blen = HS + jee_bytes + (mb_total + 7) / 8;
        int bad = B->bad;
        if (emt > (unsigned)kMaxExponent && !bad) bad = APAX_ERR_INTERNAL;
        if (tid == 0) {
            S->res[kp & 1].blen = blen;
            S->res[kp & 1].mincost = mn;
            if (bad) report_error(P.status, b, bad);
            if (P.trace) {
                double* tr = P.trace + 10 * b;
                tr[4] = sel;
                tr[5] = (double)(4LL * tt0 + 4LL * GB); tr[6] = (double)(4LL * tt1 + 4LL * GB);
                tr[7] = (double)(4LL * tt2 + 4LL * GB); tr[8] = (double)blen;
                tr[9] = restart ? 1.0 : 0.0;
            }
        }
        if (!FQ) {
            __threadfence_block();
            bar_arrive<3, NT>();
        }
        PMARK(7);
        // ---- JEE tokens + mantissas into the window ----
        if (!bad) {
            const unsigned below = nonA & ((1u << lane) - 1u);
            const int cin_t = below ? (int)((kbits >> (31 - __clz((int)below))) & 1u) : cin_w;
            const unsigned jx = jscan - jown;
            const int nib_off = nib_pre + (int)(cin_w ? ((jx >> 9) & 0x1ffu) : (jx & 0x1ffu));
            const int mb_off = mb_pre + 4 * (int)(jx >> 18);
            {
                uint32_t co;
                const uint32_t cons = consumed_word(Pb, (uint32_t)cin_t, &co) & 0xFu;
                const uint32_t Tm = 0xFu & ~cons;
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
                const int pos = 8 * (wb + HS) + 4 * nib_off;
                if (nbits > 32) {
                    put_bits(win, pos, (uint32_t)(acc >> 32) & (0xffffffffu >> (64 - nbits)), nbits - 32);
                    put_bits(win, pos + nbits - 32, (uint32_t)acc, 32);
                } else if (nbits > 0) {
                    put_bits(win, pos, (uint32_t)acc, nbits);
                }
            }
            int pos = 8 * (wb + HS + jee_bytes) + mb_off;
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
                        if (w == 0) continue;
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
                cold_wide_emit<DT>(xc, sq, hq1, hq2, sel, esel, win, pos);
            }
        }
        if (tid == 0) {
            // block header (dtypes.py:156-165)
            const int code = B->code;
            const uint32_t hb[6] = {(uint32_t)((sel & 3) | (restart ? 4 : 0)), (uint32_t)(code & 0xFF),
                                    (uint32_t)((code >> 8) & 0xFF), 0u, (uint32_t)(uint8_t)(int8_t)B->fbe, 0u};
#pragma unroll
            for (int k2 = 0; k2 < HS; k2++) {
                const int bp = wb + k2;
                atomicOr(&win[bp >> 2], hb[k2] << (8 * (bp & 3)));
            }
        }
        wb = (wb + blen) & 15;
        fence_proxy_async();     // window writes -> async proxy (the service warp's bulk store)
        __threadfence_block();
        bar_arrive<4, NT>();
    }
#ifdef APAX_V5_PROF
    if (tid == 0) for (int k2 = 0; k2 < 8; k2++) atomicAdd(&g_prof[k2], prof_acc[k2]);
#endif
}

// FQ: fixed quality (else fixed rate): each instantiation carries only its own loop
template <int DT, bool FQ>
__global__ void __launch_bounds__(NT, 4) encode_v5_kernel(EncParams P) {
    extern __shared__ __align__(128) unsigned char smem[];
    St* S = (St*)smem;
    unsigned char* xb0 = smem + ST_BYTES;
    uint32_t* win = (uint32_t*)(smem + ST_BYTES + 2 * x_bytes(DT));
    const int tid = threadIdx.x, warp = tid >> 5;
    uint8_t* slot = P.slots + (long long)blockIdx.x * P.slot_bytes;
#ifdef APAX_V5_TIMES
    if (tid == 0 && blockIdx.x < 8192) {
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        g_times[4 * blockIdx.x] = gtimer();
        g_times[4 * blockIdx.x + 3] = smid;
    }
#endif
    // one-wave launches: register on this SM (see the unit numbering below)
    const bool by_rank = P.nsm > 0 && (P.unit_end - P.unit_begin) == (long long)gridDim.x;
    unsigned* const tab = (unsigned*)P.ticket + 64;   // [8 * smid ..): count + ids; [2048, 2056): rank counts; [2112, ..): claims
    unsigned my_sm = 0;
    if (by_rank && tid == 0) {
        asm volatile("mov.u32 %0, %smid;" : "=r"(my_sm));
        my_sm &= 255u;
        const unsigned slot = atomicAdd(&tab[8 * my_sm], 1u);
        if (slot < 7u) atomicExch(&tab[8 * my_sm + 1 + slot], blockIdx.x + 1u);
    }
    if (tid == 0) {
        mbar_init_n(&S->full[0], NPT);
        mbar_init_n(&S->full[1], NPT);
        fence_mbar_init();
    }
    for (int i = tid; i < win_bytes(DT) / 16; i += NT) ((uint4*)win)[i] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    uint32_t phs = 0u;          // bit k: mbarrier phase parity of buffer k (each role keeps its own copy)
    uint32_t phs_v = 0u;
    const bool warm = !FQ && P.policy == 1;
    // units by ticket: a CTA that finishes a unit takes the next one (several
    // units per CTA balance dynamically; a unit's placement waits only for
    // lower units, all of which are running or done)
    // One-wave launches (one unit per CTA) number the units by the CTAs'
    // rank on their SM: the warp scheduler favours older warps, the CTAs of
    // an SM finish in blockIdx order (tools/cta_times.py: 147 of 148 SMs),
    // the first ~25% before the last, and a unit's placement waits for every
    // lower unit -- with rank-major numbers the early finishers place while
    // the late ones still code, instead of one burst of copies at the end.
    // Claim words keep the numbering a bijection whatever the hardware's
    // distribution (or a late registration) was.
    for (int iter = 0;; iter++) {
        __syncthreads();
        if (tid == 0) {
            if (by_rank) {
                long long unit = P.unit_end;
                if (iter == 0) {
                    // the other CTAs of this SM register within ~0.5 us of the launch
                    // (a grid of at most one CTA per SM has nothing to rank)
                    if (gridDim.x > (unsigned)P.nsm) __nanosleep(1000);
                    const unsigned cnt = *(volatile unsigned*)&tab[8 * my_sm];
                    unsigned rank = 0;
                    for (unsigned k = 0; k < cnt && k < 7u; k++) {
                        const unsigned id = *(volatile unsigned*)&tab[8 * my_sm + 1 + k];
                        if (id != 0u && id - 1u < blockIdx.x) rank++;
                    }
                    const unsigned idx = atomicAdd(&tab[2048 + (rank < 7u ? rank : 7u)], 1u);
                    const long long nu = P.unit_end - P.unit_begin;
                    const long long pref = (long long)rank * P.nsm + idx;
                    unsigned* claim = tab + 2112;
                    if (pref < nu && idx < (unsigned)P.nsm && atomicCAS(&claim[pref], 0u, 1u) == 0u) {
                        unit = P.unit_begin + pref;
                    } else {
                        for (long long c = nu - 1; c >= 0; c--)
                            if (atomicCAS(&claim[c], 0u, 1u) == 0u) { unit = P.unit_begin + c; break; }
                    }
                }
                S->unit = unit;
            } else {
                S->unit = P.unit_begin + (long long)atomicAdd(P.ticket, 1u);
            }
        }
        __syncthreads();
        const long long u = S->unit;
        if (u >= P.unit_end) break;
        const long long b0 = u * P.unit_blocks;
        const long long b1 = (b0 + P.unit_blocks < P.n_blocks) ? b0 + P.unit_blocks : P.n_blocks;
        if (warp == NPW) {
            SvcArgs A;
            A.x = P.x; A.status = P.status; A.lookback = P.lookback; A.block_offsets = P.block_offsets;
            A.trace = P.trace; A.target = P.target; A.att_lo = P.att_lo; A.pow10_t20 = P.pow10_t20;
            A.sqrt12 = P.sqrt12; A.mode = P.mode;
            service_unit<DT, FQ>(A, S, xb0, win, slot, u, b0, b1, warm, phs_v);
        } else {
            pack_unit<DT, FQ>(P, S, xb0, win, b0, b1, warm, phs);
        }
#ifdef APAX_V5_TIMES
        if (tid == 0 && blockIdx.x < 8192) g_times[4 * blockIdx.x + 1] = gtimer();
#endif
        if (u == 0 && tid < kFileHeader) {
            unsigned char h[kFileHeader];
            h[0] = 'A'; h[1] = 'P'; h[2] = 'A'; h[3] = 'X';
            h[4] = 1; h[5] = (unsigned char)DT; h[6] = (unsigned char)P.mode; h[7] = 0;
            for (int k2 = 0; k2 < 4; k2++) h[8 + k2] = (unsigned char)((unsigned)BS >> (8 * k2));
            for (int k2 = 0; k2 < 8; k2++) h[12 + k2] = (unsigned char)((unsigned long long)P.n >> (8 * k2));
            const unsigned long long tb = (unsigned long long)__double_as_longlong(P.target);
            for (int k2 = 0; k2 < 8; k2++) h[20 + k2] = (unsigned char)(tb >> (8 * k2));
            P.out[tid] = h[tid];
        }
        final_place(u, P.n_units, P.n_blocks, P.lookback, P.status, P.block_offsets, P.out, S, slot);
    }
#ifdef APAX_V5_TIMES
    if (tid == 0 && blockIdx.x < 8192) g_times[4 * blockIdx.x + 2] = gtimer();
#endif
}

}  // namespace v5

#ifdef APAX_V5_PROF
extern "C" int apax_debug_prof5(unsigned long long* host, int reset) {
    if (reset) { unsigned long long z[16] = {0}; return (int)cudaMemcpyToSymbol(v5::g_prof, z, sizeof(z)); }
    return (int)cudaMemcpyFromSymbol(host, v5::g_prof, 16 * sizeof(unsigned long long));
}
#endif
#ifdef APAX_V5_TIMES
extern "C" int apax_debug_cta_times5(unsigned long long* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, v5::g_times, (size_t)n * 4 * sizeof(unsigned long long));
}
extern "C" int apax_debug_cta_times5b(unsigned long long* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, v5::g_times2, (size_t)n * 2 * sizeof(unsigned long long));
}
#endif

size_t encode_v5_smem_bytes(int dt) { return (size_t)v5::ST_BYTES + 2 * (size_t)v5::x_bytes(dt) + (size_t)v5::win_bytes(dt); }

bool encode_v5_supported(int dt, int bs, int mode, const EncParams& P) {
    if (getenv("APAX_ENC_V5") && atoi(getenv("APAX_ENC_V5")) == 0) return false;
    return dt >= 1 && dt <= 3 && bs == v5::BS && (mode == 1 || mode == 2) && !P.halo && !P.meta && !P.stats &&
           (((uintptr_t)P.x) & 15) == 0;
}

static const void* v5_fn(int dt, bool fq) {
    switch (dt) {
        case 1: return fq ? (const void*)v5::encode_v5_kernel<1, true> : (const void*)v5::encode_v5_kernel<1, false>;
        case 2: return fq ? (const void*)v5::encode_v5_kernel<2, true> : (const void*)v5::encode_v5_kernel<2, false>;
        default: return fq ? (const void*)v5::encode_v5_kernel<3, true> : (const void*)v5::encode_v5_kernel<3, false>;
    }
}

int encode_v5_resident_ctas(int dt) {
    // (per device and dtype: the occupancy queries cost host time on every launch otherwise)
    static int cached[64][5] = {};
    int dev = 0, nsm = 0, per = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && dt >= 0 && dt < 5 && cached[dev][dt] > 0) return cached[dev][dt];
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = encode_v5_smem_bytes(dt);
    for (int fq = 0; fq < 2; fq++) {   // both instantiations must fit
        int p = 0;
        cudaFuncSetAttribute(v5_fn(dt, fq != 0), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p, v5_fn(dt, fq != 0), v5::NT, smem) != cudaSuccess || p < 1)
            p = 1;
        per = fq == 0 ? p : (p < per ? p : per);
    }
    const int res = per * (nsm > 0 ? nsm : 148);
    if (dev >= 0 && dev < 64 && dt >= 0 && dt < 5) cached[dev][dt] = res;
    return res;
}

// units [u0, u1) of full blocks; one slot per CTA (P.slots holds >= grid slots)
int launch_encode_v5(int dt, const EncParams& P, long long u0, long long u1, cudaStream_t st) {
    const void* fn = v5_fn(dt, P.mode == 2);
    const size_t smem = encode_v5_smem_bytes(dt);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return APAX_ERR_CUDA;
    const long long res = encode_v5_resident_ctas(dt);
    const long long nu = u1 - u0;
    EncParams p = P;
    p.unit_begin = u0;
    p.unit_end = u1;
    {
        int dev = 0, nsm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const char* e = getenv("APAX_V5_RANK");
        p.nsm = (e && atoi(e) == 0) ? 0 : (nsm > 0 && nsm <= 256 ? nsm : 0);
    }
    const int g = (int)(nu < res ? nu : res);
    void* args[] = {&p};
    note_launches(1);
    if (cudaLaunchCooperativeKernel(fn, dim3(g), dim3(v5::NT), args, smem, st) != cudaSuccess) return APAX_ERR_CUDA;
    return APAX_OK;
}

}  // namespace apax
