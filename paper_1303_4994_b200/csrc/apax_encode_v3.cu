// apax_encode_v3.cu -- B200 encoder, v3: the hot path for i8/i16/i32/f32
// containers with power-of-two block sizes 128..4096.
//
// Same contract and byte-exact output as apax_encode.cu / apax_encode_v2.cu
// (reference encode_stream pkg/src/apax/codec.py:258-285, encode_block
// :192-255).  CTA = 8 compute warps (one unit = segment at a time, blocks in
// order) + 1 placement warp.  Per block:
//
//   * staging   cp.async 16-byte chunks put each full block into shared
//               memory in the transposed leaf layout x[i*256 + 8L + j] for
//               sample 128L + 8i + j, so numpy's pairwise order (8
//               accumulators per 128-sample leaf; codec.py:159,248) reads
//               conflict-free; an mbarrier that every compute thread
//               arrives on (cp.async.mbarrier.arrive) tracks completion.
//               The next block is staged while this one is coded.
//   * phase A   peak |x| of the NEXT block (floats, i32), overlapped.
//   * S1        thread 0: gain, scale code, float block exponent
//               (codec.py:94-132 on scalars: max|q| = rint(peak*s)).
//   * phase B   leaf mapping: q = low word of fma(x, s, 1.5*2^52) (x*s is
//               exact in f64, so this is rint); fixed quality adds the
//               Markstein dequantize and the pairwise x^2, (x-y)^2 sums.
//               q goes to a swizzled int32 buffer (conflict-free both ways).
//   * phase C   16 contiguous samples per thread: D0/D1/D2, group widths
//               (entropy.py:38-55), costs, sign-flip bound of the monitor,
//               and the JEE token structure of the stream the previous
//               block's costs select, reduced to per-warp carry transfer
//               functions + nibble/bit counts (ballots + one packed scan).
//   * phase D   after ONE barrier every thread knows its nibble/bit
//               offsets; JEE tokens and MSB-first mantissas are OR-ed into
//               the window, which reuses the block's dead staging buffer.
//   * flush     one TMA bulk store (cp.async.bulk.global.shared) of the
//               window's whole 16-byte chunks into the unit's slot.
//   * placement the placement warp walks the decoupled look-back for each
//               finished unit and copies it from its slot to its final
//               offset, off the compute warps' critical path.
// Blocks whose differences may leave int32 (max|q| >= 2^29) take a 64-bit
// phase C/D.
#include <cstdint>
#include <cstdlib>
#include <type_traits>
#include <cuda_runtime.h>

#include "apax_device.cuh"
#include "apax_kernels.cuh"

#ifndef APAX_V3_MINB_NP
#define APAX_V3_MINB_NP 4   // one-wave launches: no placement warp, 256 threads, 64 registers
#endif
#ifndef APAX_V3_MINB
#define APAX_V3_MINB 3
#endif


namespace apax {
namespace v3 {
#ifdef APAX_V3_PROF2
// S1 anatomy (tools/prof_s1.py): cycles of thread 0's S1 chain, of thread
// 32's wait for the previous window store, and of thread 0's wait at B2
__device__ unsigned long long g_prof2[4];
#endif
#ifdef APAX_V3_TIMES
// per-CTA timeline (tools/cta_times.py): globaltimer at start, at the end of
// the last unit's coding, at exit; SM id
__device__ unsigned long long g_times[8192 * 4];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif

constexpr int NCW = 8;             // compute warps
constexpr int NCT = NCW * 32;      // compute threads
constexpr int NT = NCT + 32;       // + placement warp
constexpr int SPT = 16;            // samples per thread, phase C/D
constexpr int MAXBS = 4096;
constexpr int RS = 256;            // leaf-layout row stride (samples)
constexpr double kMagic = 6755399441055744.0;        // 1.5 * 2^52
constexpr double kMagicI = 6755401588539392.0;       // 1.5 * 2^52 + 2^31

struct __align__(16) St {
    // CodecState (codec.py:66-82)
    double att;
    long long p1, p2;
    long long pc[3];
    long long emitted;
    int has_pc, initialized;
    // per-block scalars (thread 0, S1)
    double a, s, rs, aq, ra, sq;
    long long qpk;
    int code, fbe, wide, bad, sel_spec, gate, zlen;
    // phase A partials (next block)
    unsigned pkw[NCW];
    unsigned pnw[NCW];
    double pxw[NCW];
    // phase B partials
    double pdw[NCW], pxbw[NCW];
    double sxyw[NCW], syyw[NCW];    // META with stats: sum x*y, sum y*y of the warp
    // phase C per-warp results
    int sew[3][NCW];
    int flw[NCW];
    int emw[NCW];
    unsigned jw[NCW];      // JEE nibbles of the warp: lo16 = warp carry-in 0, hi16 = carry-in 1
    int jc[NCW];           // bit0: a thread breaks the pairing run, bit1: its carry-out
    int mbw[NCW];          // mantissa bits of the warp
    int monc[NCW], monf[NCW];
    long long blen;
    int tl_next;
    // window / unit bookkeeping
    long long win_base;
    int tail_len;
    uint32_t tail[4];
    long long unit_len;
    int store_pending;
    // slots handed to the placement warp
    long long slot_len[2], slot_b0[2], slot_b1[2];
    long long fin_prefix;
    unsigned long long mb_stage[2];
};

using namespace apax::tma;

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
// slot hand-off between the compute warps and the placement warp: named
// barriers 2/3 ("slot s full": compute arrives, placement waits) and 4/5
// ("slot s free": placement arrives, compute waits).  Waiting warps do not
// issue, unlike a polling loop.
template <int ID> __device__ __forceinline__ void nb_arrive_() { asm volatile("bar.arrive %0, 288;" :: "n"(ID) : "memory"); }
template <int ID> __device__ __forceinline__ void nb_sync_() { asm volatile("bar.sync %0, 288;" :: "n"(ID) : "memory"); }
__device__ __forceinline__ void nb_full_arrive(int sl) { if (sl) nb_arrive_<3>(); else nb_arrive_<2>(); }
__device__ __forceinline__ void nb_full_sync(int sl) { if (sl) nb_sync_<3>(); else nb_sync_<2>(); }
__device__ __forceinline__ void nb_free_arrive(int sl) { if (sl) nb_arrive_<5>(); else nb_arrive_<4>(); }
__device__ __forceinline__ void nb_free_sync(int sl) { if (sl) nb_sync_<5>(); else nb_sync_<4>(); }
__device__ __forceinline__ int bitlen32(unsigned v) {  // bfind gives -1 for 0
    int r;
    asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(v));
    return r + 1;
}
__device__ __forceinline__ int bitlen64(unsigned long long v) { return 64 - __clzll((long long)v); }
__device__ __forceinline__ unsigned wb32(int v) { return (unsigned)((v << 1) ^ v); }
__device__ __forceinline__ unsigned long long wb64(long long v) {
    return (unsigned long long)((v << 1) ^ v);
}

// swizzled int32 q buffer: 16-byte chunk k lives at chunk k ^ g(k); the
// phase-B leaf stores and the phase-C chunk loads are both conflict-free.
__device__ __forceinline__ int swz(int k) { return k ^ (((k >> 3) & 3) ^ (((k >> 5) & 3) << 1)); }
__device__ __forceinline__ int qw(int s) { return (swz(s >> 2) << 2) | (s & 3); }

// decode_scale_code (dtypes.py:124-128) built from the bits: (1 + f/1024) *
// 2^(e-31) is a normal double for every code
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

// L2 policies: the input streams through once (evict first); the unit slots
// are re-read by the placement copy and then discarded (evict last), so the
// slot round trip stays in L2 instead of DRAM
__device__ __forceinline__ unsigned long long pol_evict_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long pol_evict_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// (no L2::cache_hint on the 16-byte copies: with a policy operand the 64-register
// instantiations faulted with an illegal instruction on the LDGSTS descriptor;
// the input's evict-first policy rides on the bulk L2 prefetch instead)
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src) : "memory");
}
// one net arrival per thread once its earlier cp.async copies have landed
// (the inc form + a release arrive also publishes plain st.shared writes)
__device__ __forceinline__ void stage_arrive(unsigned long long* bar) {
    asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" :: "r"(sa(bar)) : "memory");
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" :: "r"(sa(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" :: "r"(sa(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init_n(unsigned long long* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait_acq(unsigned long long* bar, uint32_t phase) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(sa(bar)), "r"(phase) : "memory");
    }
}
// polling wait for the placement warp (sleeps between probes: it must not
// steal issue slots from the compute warps)
__device__ __forceinline__ void mbar_wait_sleep(unsigned long long* bar, uint32_t phase) {
    for (;;) {
        uint32_t ok;
        asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(sa(bar)), "r"(phase) : "memory");
        if (ok) return;
        __nanosleep(1000);
    }
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                 :: "l"(gdst), "r"(sa(ssrc)), "r"(bytes), "l"(pol_evict_last()) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
// drop a 128-byte L2 line without writing it back (a consumed slot line)
__device__ __forceinline__ void discard_l2(const void* p) {
    asm volatile("discard.global.L2 [%0], 128;" :: "l"(p) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" :: "l"(p), "r"(bytes),
                 "l"(pol_evict_first()) : "memory");
}

// numpy's pairwise combine of nwd (1, 2, 4 or 8) per-warp leaf sums
__device__ __forceinline__ double warp_tree(const double* v, int nwd) {
    if (nwd == 1) return v[0];
    if (nwd == 2) return v[0] + v[1];
    if (nwd == 4) return (v[0] + v[1]) + (v[2] + v[3]);
    return ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
}

// consumed mask of 32 JEE positions given the carry-in (see v2)
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

// MSB-first piece writer: `c` (nb <= 32 bits) at bit position pos of the
// window, OR-ed into at most two words (ATOMS.OR runs at STS rate on B200).
__device__ __forceinline__ void put_bits(uint32_t* win, int pos, uint32_t c, int nb) {
    const uint32_t a = c << (32 - nb);           // left-aligned
    const int sh = pos & 31;
    uint32_t* w = win + (pos >> 5);
    atomicOr(w, bswap32(a >> sh));
    if (sh + nb > 32) atomicOr(w + 1, bswap32(a << (32 - sh)));
}
// the same for a piece of 1..64 bits (at most three words)
__device__ __forceinline__ void put_bits64(uint32_t* win, int pos, unsigned long long c, int nb) {
    const unsigned long long a = c << (64 - nb);  // left-aligned
    const int sh = pos & 31;
    uint32_t* w = win + (pos >> 5);
    atomicOr(w, bswap32((uint32_t)(a >> (32 + sh))));
    if (sh + nb > 32) atomicOr(w + 1, bswap32((uint32_t)(a >> sh)));
    if (sh + nb > 64) atomicOr(w + 2, bswap32((uint32_t)(a << (32 - sh))));
}

// ---------------------------------------------------------------------------
// cold paths (out of line: keeps the hot loop in the instruction cache)
// ---------------------------------------------------------------------------
// numpy pairwise sum (one thread) of term(i) over [0, n)
template <typename F>
__device__ __forceinline__ double pw_leaf(F& term, int s, int n) {
    if (n < 8) {
        double r = -0.0;
        for (int i = 0; i < n; i++) r += term(s + i);
        return r;
    }
    double r[8];
    for (int j = 0; j < 8; j++) r[j] = term(s + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; j++) r[j] += term(s + i + j);
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += term(s + i);
    return res;
}
template <typename F>
__device__ __forceinline__ double pw_seq(F& term, int s0, int n0) {
    int fs[16], fn[16], fst[16];
    double fl[16];
    int sp = 0;
    fs[0] = s0; fn[0] = n0; fst[0] = 0; sp = 1;
    double val = 0.0;
    bool have = false;
    while (sp > 0) {
        const int t = sp - 1;
        if (have) {
            if (fst[t] == 1) {
                fl[t] = val;
                fst[t] = 2;
                int n2 = fn[t] / 2;
                n2 -= n2 % 8;
                fs[sp] = fs[t] + n2; fn[sp] = fn[t] - n2; fst[sp] = 0; sp++;
                have = false;
            } else {
                val = fl[t] + val;
                sp--;
            }
            continue;
        }
        if (fn[t] <= 128) {
            val = pw_leaf(term, fs[t], fn[t]);
            have = true;
            sp--;
            continue;
        }
        fst[t] = 1;
        int n2 = fn[t] / 2;
        n2 -= n2 % 8;
        fs[sp] = fs[t]; fn[sp] = n2; fst[sp] = 0; sp++;
    }
    return val;
}

template <int DT>
__device__ __forceinline__ double xd_of(typename DT_<DT>::T xv) {
    if (DT_<DT>::F) return (double)xv;
    return __hiloint2double(0x43380000, (int)xv ^ (int)0x80000000) - kMagicI;
}

// dequantize to the dtype's value in double (codec.py:135-146); Markstein
// quotient with a per-block reciprocal (profiles/r1_markstein_division_check.txt)
template <int DT>
__device__ __forceinline__ double deq_of(double qd, double s, double rs) {
    using Tr = DT_<DT>;
    const double y0 = qd * rs;
    const double e = __fma_rn(-s, y0, qd);
    const double y = __fma_rn(e, rs, y0);
    if (Tr::F) return (DT == 3) ? (double)__double2float_rn(y) : y;
    double yi = (y + kMagic) - kMagic;   // rint (|y| < 2^51)
    const double lo = (double)Tr::LO, hi = (double)Tr::HI;
    yi = yi < lo ? lo : (yi > hi ? hi : yi);
    return yi;
}

// quantize one sample (codec.py:94-132): rint(x * s) as the low word of
// x*s + 1.5*2^52.  i8/i16/i32/f32 samples have <= 32-bit mantissas, so x*s is
// exact in f64 and one fma suffices; f64 rounds the product first (the
// reference's np.rint(x * scale)), then adds.
template <int DT>
__device__ __forceinline__ double qround(double xd, double sq) {
    if (DT == 4) return __dadd_rn(__dmul_rn(xd, sq), kMagic);
    return __fma_rn(xd, sq, kMagic);
}

// sum of x^2 over a partial (linear-layout) block, numpy order
template <int DT>
__device__ __noinline__ double cold_px(const typename DT_<DT>::T* xs, int n) {
    auto t2 = [&](int i) { const double v = xd_of<DT>(xs[i]); return v * v; };
    return pw_seq(t2, 0, n);
}
// sum of (x - y)^2 over a partial block, numpy order
template <int DT>
__device__ __noinline__ double cold_pd(const typename DT_<DT>::T* xs, const int* qbuf, int n, double s,
                                       double rs, bool int_id) {
    auto td = [&](int i) {
        const double xd = xd_of<DT>(xs[i]);
        const double qd = (double)qbuf[qw(i)];
        const double y = int_id ? qd : deq_of<DT>(qd, s, rs);
        const double d = xd - y;
        return d * d;
    };
    return pw_seq(td, 0, n);
}
// first non-finite sample of a block (floats)
template <int DT>
__device__ __noinline__ void cold_nonfinite(const typename DT_<DT>::T* xs, int n, bool leaf, long long base,
                                            unsigned long long* status) {
    for (int i = 0; i < n; i++) {
        const int li = leaf ? ((i & 127) >> 3) * RS + 8 * (i >> 7) + (i & 7) : i;
        if (!isfinite((double)xs[li])) {
            atomicMin(&status[0], (unsigned long long)(base + i));
            break;
        }
    }
}
// exact monitor (transform.py:67-83) on the q buffer; all compute threads
__device__ __noinline__ int cold_monitor(const int* qbuf, St* S, int np) {
    const int ct = threadIdx.x, lane = ct & 31, warp = ct >> 5;
    const int t0 = SPT * ct;
    int ch = 0, fs = 0, lsg = 0;
    if (t0 < np) {
        // only the padded block's np samples: past np the q buffer holds the
        // previous pass's values (a partial last block of 1..12 groups)
        for (int k2 = 0; k2 < SPT && t0 + k2 < np; k2++) {
            const int v = qbuf[qw(t0 + k2)];
            const int sg = (v > 0) - (v < 0);
            if (sg) {
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
    cbar();
    int ch2 = 0, f = 0, l = 0;
    for (int w = 0; w < NCW; w++) {
        const int of = (S->monf[w] & 3) - 1, ol = ((S->monf[w] >> 2) & 3) - 1;
        ch2 += S->monc[w] + ((l != 0 && of != 0 && l != of) ? 1 : 0);
        if (!f) f = of;
        if (ol) l = ol;
    }
    cbar();
    const double cf = (double)ch2 / (2.0 * (double)(np - 1));
    return cf > 1.0 / 3.0;
}

// width of group gi of stream sl, read from the q buffer (boundary lanes)
__device__ __noinline__ int cold_gw(const int* qbuf, int sl, int gi, int np, long long hp1, long long hp2) {
    const int base = 4 * gi;
    long long a[6];
    for (int m = 0; m < 6; m++) {
        const int i = base - 2 + m;
        a[m] = i < 0 ? (i == -1 ? hp1 : hp2) : (i < np ? (long long)qbuf[qw(i)] : 0LL);
    }
    unsigned long long o = 0;
    for (int m = 2; m < 6; m++) {
        const long long v0 = a[m], v1 = a[m] - a[m - 1], v2 = v1 - (a[m - 1] - a[m - 2]);
        o |= wb64(sl == 0 ? v0 : (sl == 1 ? v1 : v2));
    }
    return bitlen64(o);
}

// copy len bytes from a 4-aligned global word source to an arbitrary byte
// offset with `nth` threads (thread index `lane` in 0..nth-1): one warp in
// the placement loop, the whole CTA for the CTA's last unit
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

// decoupled look-back (one warp): exclusive byte prefix of unit u from the
// predecessors' aggregate / inclusive flags
__device__ __forceinline__ long long unit_prefix(unsigned long long* lookback, long long u) {
    const int lane = threadIdx.x & 31;
    long long prefix = 0;
    long long kk = u - 1;
    unsigned nap = 256;   // exponential back-off: a waiting warp must not steal
                          // issue slots from the CTAs still coding (one-wave tails)
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

// placement warp: resolve every finished unit of this CTA and copy it out
__device__ __noinline__ void placement_loop(long long unit_begin, long long unit_end, long long n_units,
                                            long long n_blocks, unsigned long long* lookback,
                                            unsigned long long* status, long long* block_offsets, uint8_t* out,
                                            St* S, uint8_t* slot0, uint8_t* slot1) {
    const int lane = threadIdx.x & 31;
    int k = 0;
    // every unit of this CTA but the last (the whole CTA places that one,
    // final_place)
    for (long long u = unit_begin + blockIdx.x; u + (long long)gridDim.x < unit_end; u += gridDim.x, k++) {
        const int sl = k & 1;
        nb_full_sync(sl);
        const long long len = S->slot_len[sl];
        const long long b0 = S->slot_b0[sl], b1 = S->slot_b1[sl];
        long long prefix = 0;
        if (u > 0) {
            prefix = unit_prefix(lookback, u);
            if (lane == 0) st_release(&lookback[u], kFlagInc | (unsigned long long)(prefix + len));
        }
        if (u == n_units - 1 && lane == 0) {
            status[2] = (unsigned long long)(kFileHeader + prefix + len);
            if (block_offsets) block_offsets[n_blocks] = kFileHeader + prefix + len;
        }
#ifndef APAX_V3_NOCOPY
        group_copy_out(out + kFileHeader + prefix, (const uint32_t*)(sl ? slot1 : slot0), len, lane, 32);
#endif
        __syncwarp();
        for (long long l = (long long)lane * 128; l < len; l += 32 * 128) discard_l2((sl ? slot1 : slot0) + l);
        if (block_offsets)
            for (long long bb = b0 + lane; bb < b1; bb += 32) block_offsets[bb] += kFileHeader + prefix;
        __syncwarp();
        __threadfence_block();
        if (u + 2 * (long long)gridDim.x < unit_end) nb_free_arrive(sl);   // the slot is reused
    }
}

// the CTA's last unit, placed by all NT threads once the compute warps have
// published it and the placement warp has placed the earlier units: warp 0
// resolves the prefix, everyone copies (a one-warp copy of the whole unit
// was the tail of one-wave launches)
template <int NTT>
__device__ __forceinline__ void fbar() { asm volatile("bar.sync 7, %0;" :: "n"(NTT) : "memory"); }
template <int NTT>
__device__ __noinline__ void final_place(long long u, int sl, long long n_units, long long n_blocks,
                                        unsigned long long* lookback, unsigned long long* status,
                                        long long* block_offsets, uint8_t* out, St* S, uint8_t* slot) {
    const int tid = threadIdx.x;
    fbar<NTT>();
    const long long len = S->slot_len[sl];
    const long long b0 = S->slot_b0[sl], b1 = S->slot_b1[sl];
    if (tid < 32) {
        long long prefix = 0;
        if (u > 0) {
            prefix = unit_prefix(lookback, u);
            if (tid == 0) st_release(&lookback[u], kFlagInc | (unsigned long long)(prefix + len));
        }
        if (tid == 0) {
            S->fin_prefix = prefix;
            if (u == n_units - 1) {
                status[2] = (unsigned long long)(kFileHeader + prefix + len);
                if (block_offsets) block_offsets[n_blocks] = kFileHeader + prefix + len;
            }
        }
    }
    fbar<NTT>();
    const long long prefix = S->fin_prefix;
#ifndef APAX_V3_NOCOPY
    group_copy_out(out + kFileHeader + prefix, (const uint32_t*)slot, len, tid, NTT);
#endif
    fbar<NTT>();   // every thread has read its slot words: the lines are dead
    for (long long l = (long long)tid * 128; l < len; l += (long long)NTT * 128) discard_l2(slot + l);
    if (block_offsets)
        for (long long bb = b0 + tid; bb < b1; bb += NTT) block_offsets[bb] += kFileHeader + prefix;
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
// FIX: every block of this launch is a full 4096-sample block; the block
// geometry is then compile-time (the partial last block of a stream goes
// through a second, generic launch over its unit).
// PW: a placement warp places finished units while the next ones are coded
// (more units than resident CTAs).  Without it (one-wave launches: one unit
// per CTA) the CTA is 256 threads and four fit on an SM.
constexpr int fix_stage_bytes(int dt) {
    // encode_v3_stage_bytes(dt, MAXBS): max(MAXBS * width, max block bytes + 32), 128-aligned
    const int w = dt == 0 ? 1 : (dt == 1 ? 2 : (dt == 4 ? 8 : 4));
    const int g = MAXBS / 4;
    const int emax = dt >= 3 ? 34 : (8 * w + 2 < 34 ? 8 * w + 2 : 34);
    const int mb = (dt >= 3 ? 6 : 4) + (3 * g + 1) / 2 + (4 * emax * g + 7) / 8 + 32;
    const int xb = MAXBS * w;
    return ((xb > mb ? xb : mb) + 127) & ~127;
}

// META: the chain of the split encoder (apax_encode_v4.cu): only what the
// gain recurrence needs runs (fixed quality: quantize + powers; fixed rate:
// + widths, JEE counts, exact byte count), no output; each block's quantizer
// record goes to P.meta
template <int DT, bool FIX, bool PW, bool META = false>
__global__ void __launch_bounds__(PW ? NT : NCT, PW ? APAX_V3_MINB : APAX_V3_MINB_NP) encode_v3_kernel(EncParams P) {
    using Tr = DT_<DT>;
    using T = typename Tr::T;
    constexpr bool F = Tr::F;
    constexpr int HS = Tr::HDR;
    constexpr bool TRL = (DT != 0);             // transposed leaf staging (16-byte rows)
    constexpr int CH = 16 / (int)sizeof(T);     // samples per 16-byte chunk
    constexpr bool NEED_PEAK = F || DT == 2;
    constexpr bool SQX = (DT != 2 && DT != 4);  // x*x exact in f64: the square can be fused

    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bs = FIX ? MAXBS : P.bs;
    const int NL = FIX ? 32 : (bs >> 7);        // leaves of a full block
    const bool FQ = (P.mode == 2);
    // bytes per staging buffer: a compile-time constant for the bs-4096
    // instantiation (encode_v3_stage_bytes), so every shared-memory address
    // folds into an immediate offset instead of being rematerialised
    const int XB = FIX ? fix_stage_bytes(DT) : P.stage_bytes;

    St* S = (St*)smem;
    const int xoff = (int)((sizeof(St) + 127) & ~(size_t)127);
    int* qbuf = (int*)(smem + xoff + 2 * XB);
    uint8_t* slot0 = P.slots + (long long)blockIdx.x * (PW ? 2 : 1) * P.slot_bytes;
    uint8_t* slot1 = slot0 + P.slot_bytes;

#ifdef APAX_V3_TIMES
    if (tid == 0 && blockIdx.x < 8192) {
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        g_times[4 * blockIdx.x] = gtimer();
        g_times[4 * blockIdx.x + 3] = smid;
    }
#endif
    if (tid == 0) {
        mbar_init_n(&S->mb_stage[0], NCT);
        mbar_init_n(&S->mb_stage[1], NCT);
        fence_mbar_init();
        S->store_pending = 0;
        S->tail_len = 0;
    }
    __syncthreads();
    if (PW && warp == NCW) {
        placement_loop(P.unit_begin, P.unit_end, P.n_units, P.n_blocks, P.lookback, P.status, P.block_offsets,
                       P.out, S, slot0, slot1);
        const long long u0 = P.unit_begin + blockIdx.x;
        if (u0 < P.unit_end) {   // this CTA's last unit, with the compute warps
            const long long nu = (P.unit_end - u0 + gridDim.x - 1) / gridDim.x;
            const int sll = (int)((nu - 1) & 1);
            final_place<NT>(u0 + (nu - 1) * gridDim.x, sll, P.n_units, P.n_blocks, P.lookback, P.status,
                            P.block_offsets, P.out, S, sll ? slot1 : slot0);
        }
        return;
    }
    // ---------------- compute warps (named barrier 1, 256 threads) ----------------
#ifdef APAX_V3_PROF
    // phase timing of thread 0 (tools/prof_v3.py): acc[k] += clock(k) - clock(k-1)
    unsigned long long prof_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long prof_wait = 0;
    long long prof_last = clock64();
#define PROF_MARK(k) do { if (tid == 0) { const long long c_ = clock64(); prof_acc[k] += (unsigned long long)(c_ - prof_last); prof_last = c_; } } while (0)
#else
#define PROF_MARK(k) do { } while (0)
#endif
    auto xbuf = [&](int k) -> T* { return (T*)(smem + xoff + (k ? XB : 0)); };
    // staging state of the two buffers, in scalars (no local memory)
    // block held by buffer 0 / 1 (kNone: empty; block -1 is a range encode's halo)
    constexpr long long kNone = -(1LL << 62);
    long long bb0 = kNone, bb1 = kNone;
    uint32_t wst = 3u;                  // bit k: buffer k already waited on
    uint32_t phs = 0u;                  // bit k: mbarrier phase parity of buffer k
    auto bufblk_get = [&](int k) -> long long { return k ? bb1 : bb0; };
    auto bufblk_set = [&](int k, long long v) { if (k) bb1 = v; else bb0 = v; };

    auto block_len = [&](long long b) -> int {   // exact
        long long r = P.n - b * (long long)bs;
        return (int)(r < bs ? r : bs);
    };
    auto block_n = [&](long long b) -> int { return FIX ? MAXBS : block_len(b); };
    // stage block b into buffer k (all compute threads)
    auto stage = [&](long long b, int k) {
        const int n = block_n(b);
        const T* src = (const T*)P.x + b * (long long)bs;
        T* dst = xbuf(k);
        if (n == bs && (((uintptr_t)P.x) & 15) == 0) {
            const uint32_t d0 = sa(dst);
            const int nch = bs / CH;
            for (int c = tid; c < nch; c += NCT) {
                const int s0 = c * CH;
                const int di = TRL ? ((s0 & 127) >> 3) * RS + 8 * (s0 >> 7) + (s0 & 7) : s0;
                cp_async16(d0 + (uint32_t)di * (uint32_t)sizeof(T), src + s0);
            }
        } else if (n == bs) {
            for (int i = tid; i < n; i += NCT)
                dst[TRL ? ((i & 127) >> 3) * RS + 8 * (i >> 7) + (i & 7) : i] = src[i];
        } else {
            for (int i = tid; i < n; i += NCT) dst[i] = src[i];   // partial block: linear
        }
        stage_arrive(&S->mb_stage[k]);
        bufblk_set(k, b);
        wst &= ~(1u << k);
    };
    auto wait_buf = [&](int k) {
        if (!((wst >> k) & 1u)) {
#ifdef APAX_V3_PROF
            const long long w0_ = clock64();
            mbar_wait_acq(&S->mb_stage[k], (phs >> k) & 1u);
            if (tid == 0) prof_wait += (unsigned long long)(clock64() - w0_);
#else
            mbar_wait_acq(&S->mb_stage[k], (phs >> k) & 1u);
#endif
            phs ^= 1u << k;
            wst |= 1u << k;
        }
    };

    // ---- phase A: peak (+ pairwise x^2 for the fixed-quality init) ----
    auto phaseA = [&](int k, int n, bool want_px) {
        const T* xs = xbuf(k);
        unsigned pk = 0, pn = 0;   // f32: max signed / max unsigned bit patterns; ints: max / -min
        double pxs = 0.0;
        if (NEED_PEAK) {
            // full blocks sit in the leaf layout: rows of 8*NL samples, stride RS
            const bool lay = TRL && n == bs;
            const int lgr = FIX ? 8 : 3 + __ffs(NL) - 1;   // log2(8 * NL)
            if (DT == 4) {
                // max |x| bit pattern (sign cleared; NaN/inf sort above every
                // finite value), split into hi / lo words for the warp slots
                const ulonglong2* x2 = (const ulonglong2*)xs;
                unsigned long long m = 0;
                const int n2 = n >> 1;
                for (int i = tid; i < n2; i += NCT) {
                    const int p2 = lay ? (((i >> (lgr - 1)) << 7) | (i & ((1 << (lgr - 1)) - 1))) : i;
                    const ulonglong2 v = x2[p2];
                    const unsigned long long a0 = v.x & 0x7fffffffffffffffull, a1 = v.y & 0x7fffffffffffffffull;
                    m = a0 > m ? a0 : m;
                    m = a1 > m ? a1 : m;
                }
                for (int i = (n2 << 1) + tid; i < n; i += NCT) {
                    const unsigned long long a0 = (unsigned long long)__double_as_longlong((double)xs[i]) &
                                                  0x7fffffffffffffffull;
                    m = a0 > m ? a0 : m;
                }
                pk = (unsigned)(m >> 32);
                pn = (unsigned)m;
            } else if (DT == 3) {
                const uint4* x4 = (const uint4*)xs;
                int ms = 0;
                unsigned mu = 0;
                const int n4 = n >> 2;
                for (int i = tid; i < n4; i += NCT) {
                    const int p4 = lay ? (((i >> (lgr - 2)) << 6) | (i & ((1 << (lgr - 2)) - 1))) : i;
                    const uint4 v = x4[p4];
                    ms = __vimax3_s32(ms, (int)v.x, (int)v.y);
                    ms = __vimax3_s32(ms, (int)v.z, (int)v.w);
                    mu = __vimax3_u32(mu, v.x, v.y);
                    mu = __vimax3_u32(mu, v.z, v.w);
                }
                for (int i = (n4 << 2) + tid; i < n; i += NCT) {
                    const unsigned v = __float_as_uint((float)xs[i]);
                    ms = max(ms, (int)v);
                    mu = max(mu, v);
                }
                pk = (unsigned)ms;
                pn = mu;
            } else {
                int mx = 0, mn = 0;
                for (int i = tid; i < n; i += NCT) {
                    const int v = (int)xs[lay ? (((i >> lgr) << 8) | (i & ((1 << lgr) - 1))) : i];
                    mx = max(mx, v);
                    mn = min(mn, v);
                }
                pk = (unsigned)mx;
                pn = (unsigned)(-(long long)mn);
            }
        }
        if (want_px && n == bs) {
            const int L = tid >> 3, j = tid & 7;
            double r = 0.0;
            if (L < NL) {
                const T* xp = xs + (TRL ? 8 * L + j : 128 * L + j);
#pragma unroll
                for (int i = 0; i < 16; i++) {
                    const double xd = xd_of<DT>(xp[TRL ? i * RS : 8 * i]);
                    r = (i == 0) ? xd * xd : (SQX ? __fma_rn(xd, xd, r) : r + xd * xd);
                }
            }
            r += __shfl_xor_sync(0xffffffffu, r, 1);
            r += __shfl_xor_sync(0xffffffffu, r, 2);
            r += __shfl_xor_sync(0xffffffffu, r, 4);
            if (NL >= 2) r += __shfl_xor_sync(0xffffffffu, r, 8);
            if (NL >= 4) r += __shfl_xor_sync(0xffffffffu, r, 16);
            pxs = r;
        }
        if (NEED_PEAK && DT == 4) {
            // lanes holding the warp's largest hi word compete on the lo word
            const unsigned hmax = __reduce_max_sync(0xffffffffu, pk);
            pn = __reduce_max_sync(0xffffffffu, pk == hmax ? pn : 0u);
            pk = hmax;
        } else if (NEED_PEAK) {
            pk = (unsigned)__reduce_max_sync(0xffffffffu, (int)pk);
            pn = __reduce_max_sync(0xffffffffu, pn);
        }
        if (lane == 0) { S->pkw[warp] = pk; S->pnw[warp] = pn; S->pxw[warp] = pxs; }
    };

    auto first_block = [&](long long uu) -> long long {
        const long long bb = uu * P.unit_blocks;
        return (P.halo && bb + P.gblock0 > 0) ? bb - 1 : bb;
    };
    long long a_done = kNone;
    int kunit = 0;

    for (long long u = P.unit_begin + blockIdx.x; u < P.unit_end; u += gridDim.x, kunit++) {
        const int sl = kunit & 1;
        uint8_t* slot = sl ? slot1 : slot0;
        const long long b0 = u * P.unit_blocks;
        const long long b1 = (b0 + P.unit_blocks < P.n_blocks) ? b0 + P.unit_blocks : P.n_blocks;
        const bool halo = P.halo && b0 + P.gblock0 > 0;
        const bool warm = !P.halo && P.policy == 1 && P.mode == 1;
        // warm_self (App. C E8): one cost-only pass of the segment's first block
        // at gain 1 gives the FR init jump; the first block's selector is then
        // its own cost argmin (the reference preset: prev_costs = the block's
        // own costs at the jumped gain), decided in resolve -- the costs of
        // the gain-1 pass only seed the speculation
        const int npre = halo ? 1 : (warm ? 1 : 0);
        const long long npass = npre + (b1 - b0);
        auto pass_block = [&](long long k) -> long long {
            if (halo) return k == 0 ? b0 - 1 : b0 + k - 1;
            if (warm) return k < 1 ? b0 : b0 + k - 1;
            return b0 + k;
        };
        if (tid == 0) {
            S->att = 0.0; S->p1 = 0; S->p2 = 0; S->has_pc = 0; S->initialized = 0;
            S->emitted = 0; S->win_base = 0; S->tail_len = 0; S->unit_len = 0; S->blen = 0; S->tl_next = 0;
            S->tail[0] = S->tail[1] = S->tail[2] = S->tail[3] = 0u;
            if (P.halo && b0 + P.gblock0 > 1) {  // history entering block b0-1 (App. C E2)
                const T* xh = (const T*)P.x + (b0 - 1) * (long long)bs;
                S->p1 = (long long)xh[-1];
                S->p2 = (long long)xh[-2];
            }
        }
        if (PW && kunit >= 2) nb_free_sync(sl);   // the slot's previous unit has been placed
        {
            const long long bf = pass_block(0);
            if (a_done != bf) {
                int k = (bb0 == bf) ? 0 : ((bb1 == bf) ? 1 : -1);
                cbar();
                if (k < 0) {
                    if (tid == 32 && S->store_pending) { bulk_wait_read(); S->store_pending = 0; }
                    cbar();
                    k = (bb0 == kNone) ? 0 : ((bb1 == kNone) ? 1 : 0);
                    stage(bf, k);
                }
                wait_buf(k);
                phaseA(k, block_n(bf), FQ);
                a_done = bf;
            }
        }
        cbar();

        for (long long kp = 0; kp < npass; kp++) {
            const long long b = pass_block(kp);
            const int kind = halo ? (kp == 0 ? 1 : 0) : (warm ? (kp == 0 ? 2 : 0) : 0);
            const int n = block_n(b);
            const int G = FIX ? MAXBS / 4 : (n + 3) >> 2;
            const int np = FIX ? MAXBS : 4 * G;
            const bool regular = FIX ? true : (n == bs);
            const int cur = (bb0 == b) ? 0 : 1;
            T* xs = xbuf(cur);
            const bool emit = (kind == 0);
            const bool fq_emit = FQ && emit;

            PROF_MARK(0);
            // ============ S1 (thread 0): gain, code, scale ============
            // the previous block's bulk store must have read its window
            // before B2 (this block stages into that buffer after B2)
#ifdef APAX_V3_PROF2
            long long p2_t0 = clock64();
#endif
            if (tid == 32 && S->store_pending) { bulk_wait_read(); S->store_pending = 0; }
#ifdef APAX_V3_PROF2
            if (tid == 32) atomicAdd(&g_prof2[1], (unsigned long long)(clock64() - p2_t0));
            p2_t0 = clock64();
#endif
            if (tid == 0) {
                unsigned pks = 0, pku = 0;
                unsigned long long pk64 = 0;
                for (int w = 0; w < NCW; w++) {
                    pks = max(pks, S->pkw[w]);
                    pku = max(pku, S->pnw[w]);
                    const unsigned long long v = ((unsigned long long)S->pkw[w] << 32) | S->pnw[w];
                    pk64 = v > pk64 ? v : pk64;
                }
                double peak;
                bool nonfin = false;
                if (DT == 4) {
                    nonfin = pk64 >= 0x7ff0000000000000ull;
                    peak = __longlong_as_double((long long)pk64);
                } else if (F) {
                    // max |x| bit pattern from the signed / unsigned maxima
                    const unsigned pos = ((int)pks >= 0) ? pks : 0u;
                    const unsigned neg = (pku >= 0x80000000u) ? (pku & 0x7fffffffu) : 0u;
                    const unsigned pk = pos > neg ? pos : neg;
                    nonfin = pk >= 0x7f800000u;
                    peak = (double)__uint_as_float(pk);
                } else {
                    peak = (double)((pks > pku) ? pks : pku);
                }
                if (nonfin) cold_nonfinite<DT>(xs, n, regular && TRL, b * (long long)bs, P.status);
                if (emit && !S->initialized) {
                    if (FQ) {  // _init_attenuation (codec.py:155-168)
                        double px;
                        if (regular) {
                            px = warp_tree(S->pxw, (NL + 3) / 4);
                        } else {
                            px = cold_px<DT>(xs, n);
                        }
                        double rms = sqrt(px / (double)n);
                        double att0 = 0.0;
                        if (rms != 0.0) {
                            double rqa = F ? (1073741824.0 * rms) / peak : rms;
                            double a0 = P.pow10_t20 / (P.sqrt12 * rqa);
                            double m = (1e-300 > a0) ? 1e-300 : a0;
                            att0 = 20.0 * log10(m);
                        }
                        S->att = clamp_att(att0, P.att_lo);
                    }
                    S->initialized = 1;
                    S->a = (P.mode == 0) ? 1.0 : att_to_a(S->att);
                }
                double a;
                if (kind == 1 || kind == 2) a = 1.0;
                else if (kind == 3) a = S->a;
                else if (P.mode == 0) a = 1.0;
                else a = S->a;
                int bad = 0, zero = 0, fbe = 0, code;
                double s = 1.0, aq = 1.0;
                long long qpk;
                if (!F) {
                    code = encode_scale_code(a);
                    aq = scale_code_value(code);
                    qpk = (aq == 1.0) ? (long long)peak : (long long)rint(peak * aq);
                } else if (nonfin || peak == 0.0) {
                    code = kScaleCodeOne; zero = 1; qpk = 0;
                } else {
                    double s_des = (a * 1073741824.0) / peak;
                    if (!isfinite(s_des)) {
                        bad = APAX_ERR_OVERFLOW; code = kScaleCodeOne; zero = 1; qpk = 0;
                    } else {
                        // floor(log2 s_des) from the bits; only mantissas within
                        // 2^-40 of 2 can round up (floor_log2_rn decides those)
                        const unsigned long long sb = (unsigned long long)__double_as_longlong(s_des);
                        const long long l2 = ((sb & 0xFFFFFFFFFFFFFull) < 0xFFFFFFFFFF000ull && (sb >> 52) != 0)
                                                 ? (long long)(sb >> 52) - 1023
                                                 : floor_log2_rn(s_des);
                        long long fb = (-31 <= l2 && l2 <= 31) ? 0 : l2 - 31;
                        fb = fb < -127 ? -127 : (fb > 127 ? 127 : fb);
                        double rem = fb ? ldexp(s_des, (int)-fb) : s_des;
                        const double nxt = 8589934591.999999;
                        double mm = (nxt < rem) ? nxt : rem;
                        rem = (mm > 4.656612873077393e-10) ? mm : 4.656612873077393e-10;
                        code = encode_scale_code(rem);
                        for (;;) {  // overflow guard (codec.py:126-131)
                            s = fb ? decode_scale_code(code) * ldexp(1.0, (int)fb) : scale_code_value(code);
                            double qm = rint(peak * s);
                            if (qm < 2147483648.0 || fb <= -127) {
                                qpk = qm < 9.2e18 ? (long long)qm : (1LL << 62);
                                break;
                            }
                            fb -= 1;
                        }
                        fbe = (int)fb;
                    }
                }
                S->code = code; S->fbe = fbe; S->s = s; S->aq = aq;
                if (emit && P.trace) {   // the attenuation in force for this block
                    double* tr = P.trace + 10 * b;
                    tr[0] = S->att; tr[1] = a; tr[2] = code; tr[3] = fbe;
                }
                S->rs = F ? __ddiv_rn(1.0, s) : 1.0;
                S->ra = (!F && aq != 1.0) ? __ddiv_rn(1.0, aq) : 1.0;
                S->sq = F ? (zero ? 0.0 : s) : aq;      // quantizer multiplier
                S->qpk = qpk;
                // 32-bit phase C/D is exact while every |q| <= 2^30 (floats:
                // the headroom guarantees it) and every |d1| < 2^30 (checked
                // per warp in phase C)
                S->wide = (qpk > (1LL << 30)) ? 1 : 0;
                // the block exponent stops at -127 (an int8 field): f64 samples
                // beyond 2^189 then quantize past the q buffers' 32 bits.  From
                // 2^33 on the reference raises "sample outside 34-bit range"
                // (entropy.py:53-54) for the block; so does this kernel from 2^31
                // on (between the two the reference raises unless both
                // differences of the block stay inside 34 bits)
                if (F && qpk >= (1LL << 31) && !bad) bad = APAX_ERR_INTERNAL;
                S->bad = bad;
                int sel = 0;
                if (S->has_pc) {
                    if (S->pc[1] < S->pc[sel]) sel = 1;
                    if (S->pc[2] < S->pc[sel]) sel = 2;
                }
                S->sel_spec = sel;
                // window bytes to zero: a guess from the previous block, fixed up after B4
                // (tl_next: the window tail after this block's flush, which
                // thread 32 may be writing to S->tail_len right now)
                const long long pbl = S->blen;
                long long zg = S->tl_next + HS + (pbl + (pbl >> 2)) + 256;
                zg = (zg + 15) & ~15LL;
                if (!pbl || zg > XB) zg = XB;
                S->zlen = (int)zg;
            }
#ifdef APAX_V3_PROF2
            if (tid == 0) atomicAdd(&g_prof2[0], (unsigned long long)(clock64() - p2_t0));
            p2_t0 = clock64();
#endif
            cbar();  // B2
#ifdef APAX_V3_PROF2
            if (tid == 0) { atomicAdd(&g_prof2[2], (unsigned long long)(clock64() - p2_t0)); atomicAdd(&g_prof2[3], 1ull); }
#endif
            PROF_MARK(1);

            // stage the next distinct block into the other buffer
            {
                long long nb = kNone;
                for (long long kk = kp + 1; kk < npass; kk++) {
                    const long long bb = pass_block(kk);
                    if (bb != b) { nb = bb; break; }
                }
                if (nb == kNone && u + gridDim.x < P.unit_end) {
                    const long long bb = first_block(u + gridDim.x);
                    if (bb != b) nb = bb;
                }
                if (nb != kNone && bufblk_get(cur ^ 1) != nb) {
                    stage(nb, cur ^ 1);
                    if (tid == 0) {
                        const long long pb = nb + 1;   // warm L2 one block further ahead
                        if (pb < P.n_blocks) {
                            const long long bytes = (long long)block_len(pb) * (long long)sizeof(T);
                            const T* psrc = (const T*)P.x + pb * (long long)bs;
                            if ((((uintptr_t)psrc) & 15) == 0 && (bytes & 15) == 0 && bytes > 0)
                                prefetch_l2(psrc, (uint32_t)bytes);
                        }
                    }
                }
            }
            const bool wide = S->wide;
            const int hp1 = (int)S->p1, hp2 = (int)S->p2;

            // quality loop (codec.py:244-252, 179-189).  Full blocks run it on
            // thread 0 just before B5 (its inputs are the warp partials, its
            // output feeds the next S1), where warp 0 would otherwise wait
            // for the slowest phase-D warp; partial blocks read xs here,
            // before the window zeroing overwrites it.
            auto fq_update = [&](double px, double pd) {
                const double pxm = px / (double)n, pdm = pd / (double)n;
                // math.log10 of a ratio that underflowed (or of px / inf) raises
                if (pxm > 0.0 && pdm != 0.0 && pxm / pdm == 0.0 && !S->bad) S->bad = APAX_ERR_MATH_DOMAIN;
                if (pxm > 0.0) {
                    const double measured = (pdm == 0.0) ? INFINITY : 10.0 * log10(pxm / pdm);
                    if (isfinite(measured))
                        S->att = clamp_att(S->att - clamp_step(0.5 * (measured - P.target)), P.att_lo);
                }
                S->a = att_to_a(S->att);
            };
            // ============ phase B: quantize (+ fixed-quality powers) ============
            {
                const double sq = S->sq;
                if (regular) {
                    const int L = tid >> 3, j = tid & 7;
                    // q word of sample 128L + 8i + j = qb ^ C_i (see swz)
                    const int qb = (128 * L + (j & 3)) ^ (4 * ((j >> 2) ^ ((L & 3) << 1)));
                    const T* xp = xs + (TRL ? 8 * L + j : 128 * L + j);
                    if (fq_emit) {
                        const double s = S->s, rs = F ? S->rs : S->ra;
                        const double sd = F ? s : S->aq;
                        const bool idq = !F && S->aq == 1.0;
                        double rpd = 0.0, rpx = 0.0;
                        double rxy = 0.0, ryy = 0.0;   // META with stats (the profiler's sweep)
                        const bool wst = META && P.stats;
                        if (L < NL) {
#pragma unroll
                            for (int i = 0; i < 16; i++) {
                                const double xd = xd_of<DT>(xp[TRL ? i * RS : 8 * i]);
                                const double t = qround<DT>(xd, sq);
                                qbuf[qb ^ (4 * ((2 * i) ^ (i >> 2)))] = __double2loint(t);
                                const double qd = t - kMagic;
                                const double y = idq ? qd : deq_of<DT>(qd, sd, rs);
                                const double d = xd - y;
                                const double d2 = d * d;
                                rpd = (i == 0) ? d2 : rpd + d2;
                                rpx = (i == 0) ? xd * xd : (SQX ? __fma_rn(xd, xd, rpx) : rpx + xd * xd);
                                if (META && wst) { rxy += xd * y; ryy += y * y; }
                            }
                        }
                        if (META && wst) {
                            rxy = warp_allreduce(rxy, SumOp());
                            ryy = warp_allreduce(ryy, SumOp());
                            if (lane == 0) { S->sxyw[warp] = rxy; S->syyw[warp] = ryy; }
                        }
                        // leaf combine (all lanes: the shuffles use the full mask)
                        rpd += __shfl_xor_sync(0xffffffffu, rpd, 1);
                        rpx += __shfl_xor_sync(0xffffffffu, rpx, 1);
                        rpd += __shfl_xor_sync(0xffffffffu, rpd, 2);
                        rpx += __shfl_xor_sync(0xffffffffu, rpx, 2);
                        rpd += __shfl_xor_sync(0xffffffffu, rpd, 4);
                        rpx += __shfl_xor_sync(0xffffffffu, rpx, 4);
                        if (NL >= 2) {
                            rpd += __shfl_xor_sync(0xffffffffu, rpd, 8);
                            rpx += __shfl_xor_sync(0xffffffffu, rpx, 8);
                        }
                        if (NL >= 4) {
                            rpd += __shfl_xor_sync(0xffffffffu, rpd, 16);
                            rpx += __shfl_xor_sync(0xffffffffu, rpx, 16);
                        }
                        if (lane == 0) { S->pdw[warp] = rpd; S->pxbw[warp] = rpx; }
                    } else if (L < NL) {
#pragma unroll
                        for (int i = 0; i < 16; i++) {
                            const double xd = xd_of<DT>(xp[TRL ? i * RS : 8 * i]);
                            const double t = qround<DT>(xd, sq);
                            qbuf[qb ^ (4 * ((2 * i) ^ (i >> 2)))] = __double2loint(t);
                        }
                    }
                } else {
                    for (int i = tid; i < np; i += NCT) {
                        int q = 0;
                        if (i < n) q = __double2loint(qround<DT>(xd_of<DT>(xs[i]), sq));
                        qbuf[qw(i)] = q;
                    }
                }
                cbar();  // B3
                PROF_MARK(2);
                if (fq_emit && !regular) {
                    if (tid == 0) {
                        const double pxb = cold_px<DT>(xs, n);
                        if (META && P.stats) {   // the sweep's (x, y) sums of a partial block
                            const bool idq = !F && S->aq == 1.0;
                            double sxy = 0.0, syy = 0.0;
                            for (int i = 0; i < n; i++) {
                                const double xd = xd_of<DT>(xs[i]);
                                const double qd = (double)qbuf[qw(i)];
                                const double y = idq ? qd : deq_of<DT>(qd, F ? S->s : S->aq, F ? S->rs : S->ra);
                                sxy += xd * y; syy += y * y;
                            }
                            P.stats[3 * b] = pxb; P.stats[3 * b + 1] = sxy; P.stats[3 * b + 2] = syy;
                        }
                        fq_update(pxb, cold_pd<DT>(xs, qbuf, n, F ? S->s : S->aq, F ? S->rs : S->ra, !F && S->aq == 1.0));
                    }
                    cbar();  // thread 0 read xs; the window zeroing follows
                }
            }

            long long tt0 = 0, tt1 = 0, tt2 = 0;
            if (META && FQ) {
                // the quality loop needs no stream work: the buffer is free
                if (emit) bufblk_set(cur, kNone);
            } else {
            // ============ phase C: streams, widths, costs, JEE structure ============
            const int sel_spec = S->sel_spec;
            const int t0 = SPT * tid;
            const bool active = FIX ? true : t0 < np;
            const int p0 = 4 * tid;                    // first group of this thread
            const int4* qb4 = (const int4*)qbuf;
            // physical chunk of this thread's chunk m is qpb ^ m (see swz)
            const int qpb = (4 * tid) ^ (((tid >> 1) & 3) ^ (((tid >> 3) & 3) << 1));
            uint32_t epk0 = 0u, epk1 = 0u, epk2 = 0u;  // byte g = width of group g (D0, D1, D2)
            int flips = 0;
            unsigned emax = 0;
            int hq1 = hp1, hq2 = hp2;                  // q[t0-1], q[t0-2]
            bool ww = wide;                            // this warp: 64-bit arithmetic
            {
                int q[SPT];
                const int ng = FIX ? 4 : min(4, G - p0);   // valid groups of this thread (>= 1)
                if (active) {
#pragma unroll
                    for (int m = 0; m < 4; m++) {
                        const int4 v = qb4[qpb ^ m];
                        q[4 * m] = v.x; q[4 * m + 1] = v.y; q[4 * m + 2] = v.z; q[4 * m + 3] = v.w;
                    }
                    if (tid > 0) {
                        const int2 h = *(const int2*)&qbuf[(swz(4 * tid - 1) << 2) + 2];
                        hq2 = h.x; hq1 = h.y;
                    }
                }
                if (!wide) {
                    if (active) {
                        int m1 = hq1, dprev = hq1 - hq2;
                        unsigned sgn = (unsigned)hq1 >> 31;   // sign bits, oldest first
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
                        // sign-bit flips between neighbours (17 bits: q[t0-1] .. q[t0+15])
                        flips = __popc((sgn ^ (sgn >> 1)) & 0xffffu);
                    }
                    // exact only when every |d1| < 2^30 (a D1 width of 32 flags it,
                    // wrapped values included) and, for thread 0, the history
                    // entering the block is inside the same bounds
                    bool bad = active && (epk1 & 0x20202020u) != 0;
                    if (tid == 0) {
                        const long long d = (long long)hq1 - (long long)hq2;
                        bad = bad || d < -(1LL << 30) || d >= (1LL << 30) || hq1 < -(1 << 30) || hq1 > (1 << 30) ||
                              hq2 < -(1 << 30) || hq2 > (1 << 30);
                    }
                    ww = __any_sync(0xffffffffu, bad);
                    if (ww) { epk0 = epk1 = epk2 = 0u; flips = 0; }
                }
                if (active && ww) {
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
                if (active && t0 == 0) flips -= (int)((unsigned)(q[0] ^ hq1) >> 31);  // no predecessor in the block
            }
            // byte sums of the packed widths
            auto bsum = [](uint32_t e) -> int { return (int)__dp4a(e, 0x01010101u, 0u); };
            // width of the group starting at sample i0 of stream sl2 (boundary lanes only)
            auto edge_w = [&](int sl2, int4 a, long long m1, long long m2) -> int {
                const long long v[4] = {a.x, a.y, a.z, a.w};
                long long dp = m1 - m2;
                unsigned long long o = 0;
#pragma unroll
                for (int kk = 0; kk < 4; kk++) {
                    const long long v1 = v[kk] - m1, v2 = v1 - dp;
                    o |= wb64(sl2 == 0 ? v[kk] : (sl2 == 1 ? v1 : v2));
                    m1 = v[kk]; dp = v1;
                }
                return bitlen64(o);
            };
            // JEE structure of stream sl2 (entropy.py:63-88): per-thread
            // pair / escape / valid masks, the carry transfer of the 4
            // positions, and the warp scans of nibble and mantissa-bit counts
            uint32_t Pb = 0, Eb = 0, Vb = 0;
            uint32_t esel = 0;                  // packed widths of the selected stream
            int eprev = 0, enext = 0;
            unsigned jscan = 0, jown = 0;       // packed nibble scan (inclusive) and own value
            int mbo = 0;                        // mantissa bits of this thread
            unsigned nonA = 0, kbits = 0;
            auto jee_prep = [&](int sl2) {
                const uint32_t es = sl2 == 0 ? epk0 : (sl2 == 1 ? epk1 : epk2);
                esel = es;
                eprev = __shfl_up_sync(0xffffffffu, (int)(es >> 24), 1);
                enext = __shfl_down_sync(0xffffffffu, (int)(es & 0xffu), 1);
                // lane 0: the previous warp's last group; lane 31: the next
                // warp's first group -- one divergent pass for both lanes
                const bool ed0 = lane == 0 && active && p0 > 0;
                const bool ed31 = lane == 31 && active && p0 + 4 < G;
                if (ed0 || ed31) {
                    const int4 a = qb4[swz(ed0 ? 4 * tid - 1 : 4 * tid + 4)];
                    // the two samples before that group: chunk 4t-2 (lane 0) or
                    // this thread's own last chunk (lane 31: q14, q15)
                    const int2 h = *(const int2*)&qbuf[(swz(ed0 ? 4 * tid - 2 : 4 * tid + 3) << 2) + 2];
                    const int ew = edge_w(sl2, a, h.y, h.x);   // the neighbour warp may be 64-bit
                    if (ed0) eprev = ew;
                    else enext = ew;
                }
                const int e1 = (int)(es & 0xffu), e2 = (int)((es >> 8) & 0xffu);
                const int e3 = (int)((es >> 16) & 0xffu), e4 = (int)(es >> 24);
                const int d1 = e1 - eprev, d2 = e2 - e1, d3 = e3 - e2, d4 = e4 - e3, d5 = enext - e4;
                const uint32_t S1 = ((unsigned)(d1 + 1) < 3u ? 1u : 0u) | ((unsigned)(d2 + 1) < 3u ? 2u : 0u) |
                                    ((unsigned)(d3 + 1) < 3u ? 4u : 0u) | ((unsigned)(d4 + 1) < 3u ? 8u : 0u) |
                                    ((unsigned)(d5 + 1) < 3u ? 16u : 0u);
                const uint32_t S2 = ((unsigned)(d1 + 2) < 5u ? 1u : 0u) | ((unsigned)(d2 + 2) < 5u ? 2u : 0u) |
                                    ((unsigned)(d3 + 2) < 5u ? 4u : 0u) | ((unsigned)(d4 + 2) < 5u ? 8u : 0u);
                const int nv = FIX ? 4 : (active ? min(4, G - p0) : 0);    // valid positions
                const int npr = FIX ? (tid == NCT - 1 ? 3 : 4)
                                    : (active ? max(0, min(4, G - 1 - p0)) : 0);   // positions with p+1 < G
                Vb = (1u << nv) - 1u;
                const uint32_t first = (p0 == 0) ? 1u : 0u;                // position 0: always an escape
                Pb = S1 & (S1 >> 1) & ((1u << npr) - 1u) & ~first;
                Eb = Vb & ~Pb & (~S2 | first);
                mbo = 4 * bsum(es);
                uint32_t c0o, c1o;
                const uint32_t C0 = consumed_word(Pb, 0u, &c0o) & 0xFu;
                const uint32_t C1 = consumed_word(Pb, 1u, &c1o) & 0xFu;
                const uint32_t T0 = Vb & ~C0, T1 = Vb & ~C1;
                const int n0 = __popc(T0) + 2 * __popc(T0 & Eb);
                const int n1 = __popc(T1) + 2 * __popc(T1 & Eb);
                const uint32_t co0 = (Pb >> 3) & ~(C0 >> 3) & 1u;   // consumed(p0+4), carry-in 0
                nonA = __ballot_sync(0xffffffffu, Pb != 0xFu);
                kbits = __ballot_sync(0xffffffffu, co0 != 0);     // the carry-out when Pb != 0xF
                const unsigned below = nonA & ((1u << lane) - 1u);
                unsigned v;
                // one packed word per lane: nibbles under carry-in 0 (bits 0-8) and 1
                // (bits 9-17), exponent sum = mantissa bits / 4 (bits 18-31); a warp
                // holds <= 32 * 12 nibbles and <= 32 * 4 * 65 exponent units
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
            };
            if (emit) jee_prep(sel_spec);
            {
                const int s0 = __reduce_add_sync(0xffffffffu, bsum(epk0));
                const int s1 = __reduce_add_sync(0xffffffffu, bsum(epk1));
                const int s2 = __reduce_add_sync(0xffffffffu, bsum(epk2));
                const int fl = __reduce_add_sync(0xffffffffu, flips);
                const unsigned em = __reduce_max_sync(0xffffffffu, emax);
                if (lane == 0) {
                    S->sew[0][warp] = s0; S->sew[1][warp] = s1; S->sew[2][warp] = s2;
                    S->flw[warp] = fl;
                    S->emw[warp] = (int)em;
                }
            }
            // zero the window (this block's staging buffer is dead now):
            // chunk 0 carries the previous block's tail
            const int zlen = S->zlen;
            if (META && emit) bufblk_set(cur, kNone);
            if (!META && emit) {
                uint4* w4 = (uint4*)xs;
                const int nz = zlen >> 4;
                for (int i = tid; i < nz; i += NCT) w4[i] = make_uint4(0u, 0u, 0u, 0u);
                if (tid == 0) w4[0] = make_uint4(S->tail[0], S->tail[1], S->tail[2], S->tail[3]);
                bufblk_set(cur, kNone);
            }
            cbar();  // B4
            PROF_MARK(3);

            // ============ resolve: totals, selector, offsets ============
            int flt;
            unsigned emt;
            {
                const int w = lane & (NCW - 1);
                const int a0 = S->sew[0][w], a1 = S->sew[1][w], a2 = S->sew[2][w];
                const int af = S->flw[w];
                const unsigned ae = (unsigned)S->emw[w];
                tt0 = __reduce_add_sync(0xffffffffu, lane < NCW ? a0 : 0);
                tt1 = __reduce_add_sync(0xffffffffu, lane < NCW ? a1 : 0);
                tt2 = __reduce_add_sync(0xffffffffu, lane < NCW ? a2 : 0);
                flt = __reduce_add_sync(0xffffffffu, lane < NCW ? af : 0);
                emt = __reduce_max_sync(0xffffffffu, lane < NCW ? ae : 0u);
            }
            // exact monitor only when the sign-flip bound cannot rule out the
            // 1/3 gate (transform.py:67-83,107-113)
            const int gate = (3LL * flt > 2LL * (np - 1)) ? cold_monitor(qbuf, S, np) : 0;
            int sel_pre = sel_spec;
            if (warm && emit && S->emitted == 0) {   // warm_self: the block's own costs
                sel_pre = tt1 < tt0 ? 1 : 0;
                if (tt2 < (sel_pre ? tt1 : tt0)) sel_pre = 2;
            }
            const int sel = gate ? 0 : sel_pre;
            if (emit && sel != sel_spec) {
                cbar();   // everyone read the per-warp JEE words
                jee_prep(sel);
                cbar();
            }
            if (!emit) {
                // cost-only passes: lossless halo / warm_self (codec.py:216-222)
                if (tid == 0) {
                    const long long g4 = 4LL * G;
                    if (emt > (unsigned)kMaxExponent && !S->bad) S->bad = APAX_ERR_INTERNAL;
                    if (kind == 1) {
                        S->has_pc = 1;
                        S->pc[0] = 4 * tt0 + g4; S->pc[1] = 4 * tt1 + g4; S->pc[2] = 4 * tt2 + g4;
                        S->p1 = qbuf[qw(np - 1)]; S->p2 = qbuf[qw(np - 2)];
                        S->emitted = 1; S->initialized = 1;
                        S->a = 1.0;
                    } else if (kind == 2) {
                        long long mn = tt0;
                        mn = tt1 < mn ? tt1 : mn;
                        mn = tt2 < mn ? tt2 : mn;
                        const double bps0 = (double)(4 * mn + g4 + 8LL * HS) / (double)bs;
                        const double att0 = clamp_att(0.0 - 6.02 * (bps0 - P.target), P.att_lo);
                        S->att = att0;
                        S->a = att_to_a(att0);
                        S->has_pc = 1;   // speculation only (resolve takes the own-cost argmin)
                        S->pc[0] = 4 * tt0 + g4; S->pc[1] = 4 * tt1 + g4; S->pc[2] = 4 * tt2 + g4;
                    } else {
                        S->has_pc = 1;
                        S->pc[0] = 4 * tt0 + g4; S->pc[1] = 4 * tt1 + g4; S->pc[2] = 4 * tt2 + g4;
                    }
                    if (S->bad) report_error(P.status, b, S->bad);
                }
            } else {
                // warp-level carry chain and prefixes (lanes 0..NCW-1 = warps)
                int cin_w, nib_pre, mb_pre, nib_total, mb_total;
                {
                    const int w = lane & (NCW - 1);
                    const unsigned jwv = S->jw[w];
                    const int jcv = S->jc[w];
                    const int mbv = S->mbw[w];
                    // transfer f_w(c) = has ? k : c, composed left to right
                    // (has, k) in bits 0, 1 of one word
                    int hk = (lane < NCW) ? (jcv & 3) : 0;
#pragma unroll
                    for (int d = 1; d < NCW; d <<= 1) {
                        const int o = __shfl_up_sync(0xffffffffu, hk, d);
                        if (lane >= d && !(hk & 1)) hk = o;
                    }
                    const int phk = __shfl_up_sync(0xffffffffu, hk, 1);
                    const int cin = (lane == 0) ? 0 : ((phk & 1) ? (phk >> 1) & 1 : 0);
                    const int nw_ = (lane < NCW) ? (int)(cin ? (jwv >> 16) : (jwv & 0xffffu)) : 0;
                    const int mw_ = (lane < NCW) ? mbv : 0;
                    // nibbles (bits 0-13, <= 8 * 384) and exponent units = mantissa
                    // bits / 4 (bits 14-31, <= 8 * 8320) in one word
                    const unsigned own = (unsigned)nw_ | ((unsigned)(mw_ >> 2) << 14);
                    unsigned nm = own;
#pragma unroll
                    for (int d = 1; d < NCW; d <<= 1) {
                        const unsigned o = __shfl_up_sync(0xffffffffu, nm, d);
                        if (lane >= d) nm += o;
                    }
                    const unsigned tot = __shfl_sync(0xffffffffu, nm, NCW - 1);
                    nib_total = (int)(tot & 0x3fffu);
                    mb_total = 4 * (int)(tot >> 14);
                    const unsigned pre = __shfl_sync(0xffffffffu, nm - own, warp);
                    cin_w = __shfl_sync(0xffffffffu, cin, warp);
                    nib_pre = (int)(pre & 0x3fffu);
                    mb_pre = 4 * (int)(pre >> 14);
                }
                const int jee_bytes = (nib_total + 1) >> 1;
                const long long blen = HS + jee_bytes + ((long long)mb_total + 7) / 8;
                const int wb = S->tail_len;
                // window zero fix-up when the guess was short (rare)
                if (!META && wb + blen + 16 > zlen) {
                    uint4* w4 = (uint4*)xs;
                    const int nz = (int)((wb + blen + 16 + 15) >> 4);
                    for (int i = (zlen >> 4) + tid; i < nz; i += NCT) w4[i] = make_uint4(0u, 0u, 0u, 0u);
                    cbar();
                }
                // this thread's carry-in and offsets
                const unsigned below = nonA & ((1u << lane) - 1u);
                const int cin_t = below ? (int)((kbits >> (31 - __clz((int)below))) & 1u) : cin_w;
                const unsigned jx = jscan - jown;
                const int nib_off = nib_pre + (int)(cin_w ? ((jx >> 9) & 0x1ffu) : (jx & 0x1ffu));
                const int mb_off = mb_pre + 4 * (int)(jx >> 18);
                if (emt > (unsigned)kMaxExponent && tid == 0 && !S->bad) S->bad = APAX_ERR_INTERNAL;
                // FR loop needs this block's exact byte count (codec.py:228-243)
                if (tid == 0) {
                    S->blen = blen;
                    S->tl_next = (int)((wb + blen) & 15);
                    S->gate = gate;
                    S->sel_spec = sel_pre;   // the block's pre-gate selector (trace)
                }
                const int bad = S->bad;
                // ============ phase D: JEE tokens + mantissas into the window ============
                uint32_t* win = (uint32_t*)xs;
                if (!META && active && !bad) {
                    // JEE tokens of this thread's positions, gathered into <= 48 bits
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
                        const int pos = 8 * (wb + HS) + 4 * nib_off;
                        if (nbits > 32) {
                            put_bits(win, pos, (uint32_t)(acc >> 32) & (0xffffffffu >> (64 - nbits)), nbits - 32);
                            put_bits(win, pos + nbits - 32, (uint32_t)acc, 32);
                        } else if (nbits > 0) {
                            put_bits(win, pos, (uint32_t)acc, nbits);
                        }
                    }
                    // mantissas of the selected stream (q reloaded from the q buffer)
                    int q[SPT];
#pragma unroll
                    for (int m = 0; m < 4; m++) {
                        const int4 v = qb4[qpb ^ m];
                        q[4 * m] = v.x; q[4 * m + 1] = v.y; q[4 * m + 2] = v.z; q[4 * m + 3] = v.w;
                    }
                    int pos = 8 * (wb + HS + jee_bytes) + mb_off;
                    const int ng = FIX ? 4 : min(4, G - p0);
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
                                    // one uniform path for every width <= 16: the group's
                                    // 4w bits as one 64-bit piece (no <=8 / <=16 divergence)
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
                if (!META && tid == 0) {
                    // block header (dtypes.py:156-165)
                    const int restart = (S->emitted == 0);
                    const int code = S->code;
                    const uint32_t hb[6] = {(uint32_t)((sel & 3) | (restart ? 4 : 0)), (uint32_t)(code & 0xFF),
                                            (uint32_t)((code >> 8) & 0xFF), 0u,
                                            (uint32_t)(uint8_t)(int8_t)S->fbe, 0u};
#pragma unroll
                    for (int k2 = 0; k2 < HS; k2++) {
                        const int bp = wb + k2;
                        atomicOr(&win[bp >> 2], hb[k2] << (8 * (bp & 3)));
                    }
                }
            }

            }   // stream work (skipped by the fixed-quality chain)
            PROF_MARK(4);
            // ============ phase A of the next pass block (overlaps this block's tail) ============
            {
                long long nb = kNone;
                bool nfirst = false;
                if (kp + 1 < npass) nb = pass_block(kp + 1);
                else if (u + gridDim.x < P.unit_end) { nb = first_block(u + gridDim.x); nfirst = true; }
                a_done = kNone;
                if (nb != kNone) {
                    const int k = (bb0 == nb) ? 0 : ((bb1 == nb) ? 1 : -1);
                    if (k >= 0) {
                        wait_buf(k);
                        phaseA(k, block_n(nb), FQ && nfirst);
                        a_done = nb;
                    }
                }
            }
            if (fq_emit && regular && tid == 0) {
                const double pxb = warp_tree(S->pxbw, (NL + 3) / 4);
                if (META && P.stats) {   // (x, y = the decode) sums of the block for the profiler's sweep
                    double sxy = 0.0, syy = 0.0;
                    for (int w = 0; w < NCW; w++) { sxy += S->sxyw[w]; syy += S->syyw[w]; }
                    P.stats[3 * b] = pxb; P.stats[3 * b + 1] = sxy; P.stats[3 * b + 2] = syy;
                }
                fq_update(pxb, warp_tree(S->pdw, (NL + 3) / 4));
            }
            if (emit && P.mode == 1 && tid == 0) {
                // rate loop (codec.py:228-243) on this block's exact byte count;
                // like the quality loop it only feeds the next S1
                const long long g4 = 4LL * G;
                if (S->emitted == 0) {
                    long long mn = tt0 < tt1 ? tt0 : tt1;
                    mn = tt2 < mn ? tt2 : mn;
                    const double bps0 = (double)(4 * mn + g4 + 8LL * HS) / (double)bs;
                    S->att = clamp_att(S->att - 6.02 * (bps0 - P.target), P.att_lo);
                } else {
                    const double err = (double)(S->blen * 8) / (double)bs - P.target;
                    S->att = clamp_att(S->att - clamp_step(0.75 * err), P.att_lo);
                }
                S->a = att_to_a(S->att);
            }
            if (emit && !META) fence_proxy_async();  // window writes -> async proxy (bulk store)
            cbar();  // B5
            PROF_MARK(5);

            // ============ flush (thread 32) || bookkeeping + next S1 (thread 0) ============
            // Thread 32 owns the window bytes: bulk store, tail, offsets,
            // win_base / tail_len, and the store's read wait before the next
            // barrier; thread 0 goes straight on to the next block's S1.
            if (!META && emit && tid == 32) {
                const int wb = S->tail_len;
                const long long blen = S->blen;
                const uint32_t* win = (const uint32_t*)xs;
                const long long total = wb + blen;
                const long long full = total & ~15LL;
                const long long wbase = S->win_base;
                if (full > 0) {
                    bulk_store(slot + wbase, win, (uint32_t)full);
                    S->store_pending = 1;
                }
                const int w0 = (int)(full >> 2);
                S->tail[0] = win[w0]; S->tail[1] = win[w0 + 1];
                S->tail[2] = win[w0 + 2]; S->tail[3] = win[w0 + 3];
                if (P.block_offsets) P.block_offsets[b] = wbase + wb;  // unit-relative
                S->win_base = wbase + full;
                S->tail_len = (int)(total - full);
            }
            if (emit && tid == 0) {
                const long long blen = S->blen;
                const int sel = S->gate ? 0 : S->sel_spec;
                if (META) {
                    BlockMeta m;
                    // (a block in error: a zero quantizer, the packer codes a silent block)
                    m.sq = S->bad ? 0.0 : S->sq; m.code = S->code; m.fbe = (short)S->fbe;
                    m.wide = S->bad ? (short)0 : (short)S->wide;
                    P.meta[b] = m;   // (trace: S1 wrote the gain, the packer adds the rest)
                } else if (P.trace) {
                    double* tr = P.trace + 10 * b;
                    tr[4] = sel;
                    tr[5] = (double)(4 * tt0 + 4LL * G); tr[6] = (double)(4 * tt1 + 4LL * G);
                    tr[7] = (double)(4 * tt2 + 4LL * G); tr[8] = (double)blen;
                    tr[9] = (S->emitted == 0);
                }
                if (S->bad) report_error(P.status, b, S->bad);
                S->has_pc = 1;
                const long long g4 = 4LL * G;
                S->pc[0] = 4 * tt0 + g4; S->pc[1] = 4 * tt1 + g4; S->pc[2] = 4 * tt2 + g4;
                S->p1 = qbuf[qw(np - 1)];
                S->p2 = qbuf[qw(np - 2)];
                S->emitted += 1;
                S->unit_len += blen;
            }
        }

        PROF_MARK(6);
        // ---------------- unit end: last tail, publish, hand to the placement warp ----------------
        if (META) {
            cbar();
            continue;
        }
        if (tid == 32) {
            if (S->store_pending) { bulk_wait_all(); S->store_pending = 0; }
            if (S->tail_len > 0) {
                const uint4 t4 = make_uint4(S->tail[0], S->tail[1], S->tail[2], S->tail[3]);
                *(uint4*)(slot + S->win_base) = t4;
            }
        }
        cbar();
        if (tid == 0) {
            const long long Lu = S->unit_len;
            st_release(&P.lookback[u], (u == 0 ? kFlagInc : kFlagAgg) | (unsigned long long)Lu);
            S->slot_len[sl] = Lu; S->slot_b0[sl] = b0; S->slot_b1[sl] = b1;
            __threadfence_block();
        }
        const bool last_unit = !PW || u + (long long)gridDim.x >= P.unit_end;
        if (PW && !last_unit) nb_full_arrive(sl);
        if (u == 0 && tid < kFileHeader) {
            unsigned char h[kFileHeader];
            h[0] = 'A'; h[1] = 'P'; h[2] = 'A'; h[3] = 'X';
            h[4] = 1; h[5] = (unsigned char)DT; h[6] = (unsigned char)P.mode; h[7] = 0;
            for (int k2 = 0; k2 < 4; k2++) h[8 + k2] = (unsigned char)((unsigned)bs >> (8 * k2));
            for (int k2 = 0; k2 < 8; k2++) h[12 + k2] = (unsigned char)((unsigned long long)P.n >> (8 * k2));
            const unsigned long long tb = (unsigned long long)__double_as_longlong(P.target);
            for (int k2 = 0; k2 < 8; k2++) h[20 + k2] = (unsigned char)(tb >> (8 * k2));
            P.out[tid] = h[tid];
        }
#ifdef APAX_V3_TIMES
        if (last_unit && tid == 0 && blockIdx.x < 8192) g_times[4 * blockIdx.x + 1] = gtimer();
#endif
        if (last_unit)
            final_place<PW ? NT : NCT>(u, sl, P.n_units, P.n_blocks, P.lookback, P.status, P.block_offsets, P.out,
                                       S, slot);
    }
#ifdef APAX_V3_TIMES
    if (tid == 0 && blockIdx.x < 8192) g_times[4 * blockIdx.x + 2] = gtimer();
#endif
#ifdef APAX_V3_PROF
    if (tid == 0 && P.trace) {
        const long long c_ = clock64();
        prof_acc[7] = prof_wait;   // staging waits (inside the phases above)
        for (int k2 = 0; k2 < 8; k2++) atomicAdd((unsigned long long*)(P.trace + 10 * P.n_blocks) + k2, prof_acc[k2]);
    }
#endif
}

}  // namespace v3

#ifdef APAX_V3_PROF2
extern "C" int apax_debug_prof2(unsigned long long* host) {
    return (int)cudaMemcpyFromSymbol(host, v3::g_prof2, 4 * sizeof(unsigned long long));
}
#endif
#ifdef APAX_V3_TIMES
extern "C" int apax_debug_cta_times(unsigned long long* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, v3::g_times, (size_t)n * 4 * sizeof(unsigned long long));
}
#endif

size_t encode_v3_smem_bytes(int dt, int bs, int stage_bytes) {
    (void)dt; (void)bs;
    auto al = [](size_t v) { return (v + 127) & ~(size_t)127; };
    return al(sizeof(v3::St)) + 2 * (size_t)stage_bytes + (size_t)v3::MAXBS * 4;
}

int encode_v3_stage_bytes(int dt, int bs) {
    // the leaf layout always spans 16 rows of 256 samples
    long long xb = (long long)v3::MAXBS * dt_width(dt);
    long long mb = max_block_bytes(dt, bs) + 32;
    long long v = xb > mb ? xb : mb;
    return (int)((v + 127) & ~127LL);
}

bool encode_v3_supported(int dt, int bs) {
    return dt >= 0 && dt <= 4 && bs >= 128 && bs <= v3::MAXBS && (bs & (bs - 1)) == 0;
}

template <int DT, bool FIX>
static void* v3_fn(bool pw) {
    return pw ? (void*)v3::encode_v3_kernel<DT, FIX, true> : (void*)v3::encode_v3_kernel<DT, FIX, false>;
}

static void* v3_kernel(int dt, bool fix, bool pw) {
    switch (dt) {
        case 0: return v3_fn<0, false>(pw);
        case 1: return fix ? v3_fn<1, true>(pw) : v3_fn<1, false>(pw);
        case 2: return fix ? v3_fn<2, true>(pw) : v3_fn<2, false>(pw);
        case 3: return fix ? v3_fn<3, true>(pw) : v3_fn<3, false>(pw);
        default: return fix ? v3_fn<4, true>(pw) : v3_fn<4, false>(pw);
    }
}

static int v3_resident(int dt, size_t smem, bool pw) {
    int dev = 0, nsm = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int r = nsm > 0 ? nsm : 148;
    for (int f = 0; f < 2; f++) {   // both instantiations must fit (the FIX one may use fewer registers)
        const void* fn = v3_kernel(dt, f == 1 && dt >= 1, pw);
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int p = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p, fn, pw ? v3::NT : v3::NCT, smem) != cudaSuccess || p < 1)
            p = 1;
        per = f == 0 ? p : (p < per ? p : per);
    }
    return per * r;
}

// resident CTAs with the placement warp (persistent multi-unit launches)
int encode_v3_resident_ctas(int dt, size_t smem) { return v3_resident(dt, smem, true); }
// resident CTAs of the one-wave variant (no placement warp)
int encode_v3_resident_ctas_wave(int dt, size_t smem) {
    if (getenv("APAX_V3_PW")) return 0;   // tuning: force the placement-warp kernel
    return v3_resident(dt, smem, false);
}

static int launch_v3_range(int dt, bool fix, const EncParams& P, long long u0, long long u1, int grid,
                           size_t smem, cudaStream_t st) {
    // one unit per CTA fits: the 256-thread kernel; otherwise the persistent
    // kernel with its placement warp
    const long long nu = u1 - u0;
    const bool pw = nu > encode_v3_resident_ctas_wave(dt, smem);
    const void* fn = v3_kernel(dt, fix, pw);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return APAX_ERR_CUDA;
    EncParams p = P;
    p.unit_begin = u0;
    p.unit_end = u1;
    const int g = pw ? (int)(nu < grid ? nu : grid) : (int)nu;
    void* args[] = {&p};
    note_launches(1);
    if (cudaLaunchCooperativeKernel(fn, dim3(g), dim3(pw ? v3::NT : v3::NCT), args, smem, st) != cudaSuccess)
        return APAX_ERR_CUDA;
    return APAX_OK;
}

template <int DT, bool FIX>
static void* v3_chain_fn() { return (void*)v3::encode_v3_kernel<DT, FIX, false, true>; }

static void* v3_chain_kernel(int dt, bool fix) {
    switch (dt) {
        case 1: return fix ? v3_chain_fn<1, true>() : v3_chain_fn<1, false>();
        case 2: return fix ? v3_chain_fn<2, true>() : v3_chain_fn<2, false>();
        case 3: return fix ? v3_chain_fn<3, true>() : v3_chain_fn<3, false>();
        default: return fix ? v3_chain_fn<4, true>() : v3_chain_fn<4, false>();
    }
}

// the split encoder's chain over every unit: quantizer records only
int launch_encode_v3_chain(int dt, const EncParams& P, size_t smem, cudaStream_t st) {
    if (dt < 1 || dt > 4 || P.bs != v3::MAXBS || P.stage_bytes != v3::fix_stage_bytes(dt) || !P.meta)
        return APAX_ERR_INTERNAL;
    long long ufull = P.n_units;
    if ((P.n % v3::MAXBS) != 0) ufull = P.n_units - 1;
    for (int part = 0; part < 2; part++) {
        const long long u0 = part ? ufull : 0, u1 = part ? P.n_units : ufull;
        if (u1 <= u0) continue;
        const void* fn = v3_chain_kernel(dt, part == 0);
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return APAX_ERR_CUDA;
        int dev = 0, nsm = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, v3::NCT, smem) != cudaSuccess || per < 1) per = 1;
        const long long res = (long long)per * (nsm > 0 ? nsm : 148);
        EncParams p = P;
        p.unit_begin = u0;
        p.unit_end = u1;
        const long long g = (u1 - u0) < res ? (u1 - u0) : res;
        note_launches(1);
        void* args[] = {&p};
        if (cudaLaunchKernel(fn, dim3((unsigned)g), dim3(v3::NCT), args, smem, st) != cudaSuccess)
            return APAX_ERR_CUDA;
    }
    return APAX_OK;
}

int launch_encode_v3(int dt, const EncParams& P, int grid, size_t smem, cudaStream_t st) {
    if (P.bs == v3::MAXBS && P.stage_bytes != v3::fix_stage_bytes(dt)) return APAX_ERR_INTERNAL;
    // bs 4096 (i16/i32/f32): units made only of full blocks take the
    // compile-time-geometry kernel; the unit holding a partial last block
    // follows in a generic launch (its look-back reads the first launch's
    // published lengths)
    const bool fixable = P.bs == v3::MAXBS && dt >= 1 && dt <= 4 && getenv("APAX_V3_NOFIX") == nullptr;
    long long ufull = P.n_units;
    if (fixable && (P.n % v3::MAXBS) != 0) ufull = P.n_units - 1;
    if (!fixable) ufull = 0;
    if (ufull > 0) {
        // segments of full blocks: the v5 kernel (pack warps + a service warp)
        // when it takes the container, else the fused v3 kernel
        // (v5 places a unit only after coding it: it takes the one-wave launches,
        // the persistent v3 kernel with its placement warp the longer ones;
        // APAX_ENC_V5=2 forces v5)
        const char* e5 = getenv("APAX_ENC_V5");
        // (and units of one or two blocks stay on v3: v5's unit start -- the
        // service warp's first peak and quantizer before any pack warp moves --
        // costs ~2 us more than v3's, 5-8% of such launches: profiles/r2d_cfg5_sweep.jsonl)
        const bool use5 = fixable && encode_v5_supported(dt, P.bs, P.mode, P) &&
                          ((ufull <= encode_v5_resident_ctas(dt) && P.unit_blocks >= 3) || (e5 && atoi(e5) == 2));
        const int r = use5 ? launch_encode_v5(dt, P, 0, ufull, st) : launch_v3_range(dt, true, P, 0, ufull, grid, smem, st);
        if (r) return r;
    }
    if (ufull < P.n_units) return launch_v3_range(dt, false, P, ufull, P.n_units, grid, smem, st);
    return APAX_OK;
}

}  // namespace apax
