// apax_encode_ws.cu -- the whole-stream chain of the split encoder
// (fast exact whole-stream fixed-rate / fixed-quality).
//
// A whole-stream container (the reference's own encode_stream,
// pkg/src/apax/codec.py:258-285) carries one gain recurrence through every
// block: block j's scale code needs block j-1's exact byte count (fixed
// rate, codec.py:228-243) or its measured SRR (fixed quality, :244-252).
// That recurrence cannot be split, so its latency per block is the whole
// story.  This kernel runs it on one 1024-thread CTA (one group of 4
// samples per thread, 4096-sample blocks) and only what the recurrence
// needs:
//   * fixed rate: quantize, the three streams' group widths
//     (entropy.py:38-55) for the selector costs, the JEE token count of the
//     selected stream (entropy.py:63-88, a 2-state automaton composed per
//     warp by bit tricks and across warps by one shuffle scan) and the
//     mantissa bits -> the block's exact byte count -> the rate loop;
//   * fixed quality: quantize, dequantize, numpy's pairwise sums of x^2 and
//     (x - y)^2 (leaves of 128 samples with 8 sequential accumulators, one
//     warp per leaf, then the leaf butterfly) -> the quality loop.
// Each block's quantizer record goes to P.meta; the block-parallel packer
// (apax_encode_v4.cu) then writes the container.  Samples stream in by TMA
// one block ahead.  Output is byte-identical to the reference.
#include <cstdint>
#include <cuda_runtime.h>

#include "apax_device.cuh"
#include "apax_kernels.cuh"

namespace apax {
namespace ws {

constexpr int NW = 32;
constexpr int NT = NW * 32;
constexpr int BS = 4096;
constexpr double kMagic = 6755399441055744.0;   // 1.5 * 2^52

constexpr int NBUF = 4;              // staging ring: TMA runs 3 blocks ahead

struct __align__(16) Sw {
    unsigned long long mbar[NBUF];
    double pxb;                      // this block's sum of x^2 (quality loop)
    double att, a;                   // AttenuatorState (dtypes.py:183-205)
    double sq, rs, aq;               // block quantizer: multiplier, 1/S (floats), a_q (ints)
    int code, fbe, wide, bad, sel, gate, initialized;
    int pc[3], has_pc;               // previous block's costs (sum of widths per stream)
    int p1, p2;                      // history: previous block's last two quantized samples
    int h1, h2;                      // this block's last two quantized samples
    unsigned pk[NW], pn[NW];         // peak partials
    unsigned cs01[NW], cs2f[NW];     // width sums: w0 | w1 << 16, w2 | flips << 16
    unsigned em[NW];
    unsigned edge[NW][2];            // widths (D0, D1, D2 bytes) of the warp's first / last group
    unsigned jw[NW];                 // JEE nibbles for carry-in 0 / 1 (lo16 / hi16)
    int jc[NW];                      // bit0: constant transfer, bit1: the constant
    int mb[NW];                      // mantissa bits of the warp (selected stream)
    double lx[NW], ld[NW];           // leaf sums of x^2 and (x - y)^2
    int monc[NW], monf[NW];
};

__device__ __forceinline__ void bar() { __syncthreads(); }
__device__ __forceinline__ unsigned wb32(int v) { return (unsigned)((v << 1) ^ v); }
__device__ __forceinline__ unsigned long long wb64(long long v) { return (unsigned long long)((v << 1) ^ v); }
__device__ __forceinline__ int bitlen32(unsigned v) {
    int r;
    asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(v));
    return r + 1;
}
__device__ __forceinline__ int bitlen64(unsigned long long v) { return 64 - __clzll((long long)v); }

__device__ __forceinline__ double scale_code_value(int code) {
    const unsigned long long e = (unsigned long long)(code >> 10), f = (unsigned long long)(code & 0x3FF);
    return __longlong_as_double((long long)(((e + 992ull) << 52) | (f << 42)));
}
__device__ __forceinline__ double clamp_att(double att, double lo) {
    double m = (lo > att) ? lo : att;
    return (0.0 < m) ? 0.0 : m;
}
__device__ __forceinline__ double att_to_a(double att) {
    double p = exp10(att / 20.0);   // 10.0 ** (att / 20.0) (dtypes.py:199)
    double m = (4.656612873077393e-10 > p) ? 4.656612873077393e-10 : p;
    return (1.0 < m) ? 1.0 : m;
}
// scale code of a = clamp(10^(att/20), 2^-31, 1) (dtypes.py:195-205,109-121)
// for an integer block, which needs only a's top 11 bits: 2^(att log2(10)/20)
// in single precision decides them unless a lies within 2^-10 of a code
// boundary (~0.2% of blocks), where the exact double path runs; exact
// points stay exact (att = 0 is a = 1)
__device__ __forceinline__ int code_of_att(double att) {
    if (att == 0.0) return kScaleCodeOne;
    const double y = att * 0.16609640474436813;            // log2(10) / 20
    if (y > -31.0 + 1e-6 && y < -1e-6) {
        const double e = floor(y);
        const float fr = exp2f((float)(y - e));            // [1, 2), rel. error ~2^-22
        const float u = (fr - 1.0f) * 1024.0f;
        const float uf = floorf(u);
        if (u - uf > 1e-3f && u - uf < 1.0f - 1e-3f && fr > 1.0f + 1e-6f && fr < 2.0f - 1e-6f)
            return (((int)e + 31) << 10) | (int)uf;
    }
    return encode_scale_code(att_to_a(att));
}
__device__ __forceinline__ double clamp_step(double d) {
    double m = (d < 6.0) ? d : 6.0;
    return (m > -6.0) ? m : -6.0;
}
template <int DT>
__device__ __forceinline__ int quant(double xd, double sq) {
    if (DT == 4) return __double2loint(__dadd_rn(__dmul_rn(xd, sq), kMagic));
    return __double2loint(__fma_rn(xd, sq, kMagic));
}
// dequantize (codec.py:135-146): Markstein quotient against the block's
// reciprocal (bit-identical to IEEE division, profiles/r1_markstein_division_check.txt)
template <int DT>
__device__ __forceinline__ double deq(double qd, double s, double rs) {
    using Tr = DT_<DT>;
    const double y0 = qd * rs;
    const double e = __fma_rn(-s, y0, qd);
    const double y = __fma_rn(e, rs, y0);
    if (Tr::F) return (DT == 3) ? (double)__double2float_rn(y) : y;
    double yi = (y + kMagic) - kMagic;
    const double lo = (double)Tr::LO, hi = (double)Tr::HI;
    return yi < lo ? lo : (yi > hi ? hi : yi);
}
// consumed mask of 32 JEE positions given the carry-in (see apax_encode_v4.cu)
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
// numpy pairwise sum (one thread) of v[0..n) (partial last block): leaves
// of <= 128 with 8 accumulators, halves rounded down to a multiple of 8;
// iterative (an explicit stack instead of recursion)
__device__ __forceinline__ double pw_leaf(const double* v, int n) {
    if (n < 8) {
        double r = -0.0;
        for (int i = 0; i < n; i++) r += v[i];
        return r;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = v[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] += v[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += v[i];
    return res;
}
__device__ __noinline__ double pairwise(const double* v, int n0) {
    int fs[16], fn[16], fst[16];
    double fl[16];
    int sp = 1;
    fs[0] = 0; fn[0] = n0; fst[0] = 0;
    double val = 0.0;
    bool have = false;
    while (sp > 0) {
        const int t = sp - 1;
        if (have) {
            if (fst[t] == 1) {          // left half done: do the right half
                fl[t] = val;
                fst[t] = 2;
                int n2 = fn[t] / 2;
                n2 -= n2 % 8;
                fs[sp] = fs[t] + n2; fn[sp] = fn[t] - n2; fst[sp] = 0; sp++;
                have = false;
            } else {                    // both halves: combine
                val = fl[t] + val;
                sp--;
            }
            continue;
        }
        if (fn[t] <= 128) {
            val = pw_leaf(v + fs[t], fn[t]);
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

#ifdef APAX_WS_PROF
// per-phase cycles of thread 0 (tools/prof_ws.py): acc[k] += clock at mark k - clock at the previous mark
__device__ unsigned long long g_ws_prof[16];
#define WSP(k) do { if (threadIdx.x == 0) { const long long c_ = clock64(); wsp_acc[k] += (unsigned long long)(c_ - wsp_last); wsp_last = c_; } } while (0)
#else
#define WSP(k) do { } while (0)
#endif

template <int DT, bool FQ>
__global__ void __launch_bounds__(NT, 1) chain_kernel(EncParams P) {
#ifdef APAX_WS_PROF
    unsigned long long wsp_acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long wsp_last = clock64();
#endif
    using Tr = DT_<DT>;
    using T = typename Tr::T;
    constexpr bool F = Tr::F;
    constexpr int HS = Tr::HDR;
    constexpr bool NEED_PEAK = F || DT == 2;
    constexpr int XB = BS * (int)sizeof(T);
    // fixed-rate 16-bit samples need no block peak: the next block's
    // quantizer comes straight out of the rate loop (no S1 round trip)
    constexpr bool FOLD = !FQ && !NEED_PEAK;
    extern __shared__ __align__(128) unsigned char smem[];
    Sw* S = (Sw*)smem;
    uint8_t* xbuf = smem + ((sizeof(Sw) + 127) & ~(size_t)127);   // NBUF staging buffers
    double* scr = (double*)(xbuf + NBUF * XB);                       // FQ: x^2 | (x - y)^2, 4096 each
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long nblk = P.n_blocks;
    auto blk_n = [&](long long bb) -> int { return (int)((P.n - bb * BS) < BS ? (P.n - bb * BS) : BS); };
    // TMA of a full block into its ring slot (the slot's previous block is
    // done: every thread passed that block's last barrier)
    auto stage = [&](long long bb) {
        if (bb < nblk && blk_n(bb) == BS) {
            tma::fence_proxy_async();
            tma::tma_load(xbuf + (int)(bb % NBUF) * XB, (const T*)P.x + bb * BS, (uint32_t)XB,
                          &S->mbar[bb % NBUF]);
        }
    };
    // a block's samples into registers, its peak partials and (fixed
    // quality) its x^2 leaf sums -- done during the previous block's tail
    auto prep = [&](long long bb, double* xv) {
        const int nn = blk_n(bb);
        if (nn == BS) {
            tma::mbar_wait(&S->mbar[bb % NBUF], (uint32_t)((bb / NBUF) & 1));
            const T* xs = (const T*)(xbuf + (int)(bb % NBUF) * XB) + 4 * tid;
#pragma unroll
            for (int k = 0; k < 4; k++) xv[k] = (double)xs[k];
        } else {
            const T* xg = (const T*)P.x + bb * BS + 4 * tid;
#pragma unroll
            for (int k = 0; k < 4; k++) xv[k] = (4 * tid + k < nn) ? (double)xg[k] : 0.0;
        }
        if (NEED_PEAK) {
            unsigned long long m = 0;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const unsigned long long v = (unsigned long long)__double_as_longlong(xv[k]) & 0x7fffffffffffffffull;
                m = v > m ? v : m;   // |x| as a bit pattern (NaN / inf sort above every finite value)
            }
            const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(m >> 32));
            const unsigned lo = __reduce_max_sync(0xffffffffu, (unsigned)(m >> 32) == hi ? (unsigned)m : 0u);
            if (lane == 0) { S->pk[warp] = hi; S->pn[warp] = lo; }
        }
        if (FQ) {
            double* X2 = scr;
#pragma unroll
            for (int k = 0; k < 4; k++) X2[4 * tid + k] = xv[k] * xv[k];
            __syncwarp();
            // leaf `warp` (128 samples): accumulator j = lane (0..7) over samples 8i + j
            double r = 0.0;
            if (lane < 8) {
                const double* v = X2 + 128 * warp + lane;
                r = v[0];
#pragma unroll
                for (int i = 1; i < 16; i++) r += v[8 * i];
            }
            r += __shfl_xor_sync(0xffffffffu, r, 1);
            r += __shfl_xor_sync(0xffffffffu, r, 2);
            r += __shfl_xor_sync(0xffffffffu, r, 4);
            if (lane == 0) S->lx[warp] = r;
        }
    };

    if (tid == 0) {
        for (int k = 0; k < NBUF; k++) tma::mbar_init(&S->mbar[k]);
        tma::fence_mbar_init();
        S->att = 0.0; S->a = 1.0; S->initialized = 0; S->has_pc = 0; S->p1 = 0; S->p2 = 0;
        if (FOLD) {   // block 0 at gain 1
            S->initialized = 1;
            S->code = kScaleCodeOne; S->fbe = 0; S->aq = 1.0; S->sq = 1.0; S->rs = 1.0; S->wide = 0;
            S->bad = 0; S->sel = 0;
            BlockMeta mt;
            mt.sq = 1.0; mt.code = kScaleCodeOne; mt.fbe = 0; mt.wide = 0;
            P.meta[0] = mt;
            if (P.trace) { P.trace[0] = 0.0; P.trace[1] = 1.0; P.trace[2] = kScaleCodeOne; P.trace[3] = 0.0; }
        }
    }
    bar();
    if (tid == 32)
        for (int k = 0; k < NBUF - 1; k++) stage(k);
    double xd[4];
    prep(0, xd);
    bar();
    for (long long b = 0; b < nblk; b++) {
        const long long base = b * BS;
        const int n = blk_n(b);
        const bool full = n == BS;
        const int G = (n + 3) >> 2;
        const bool active = tid < G;
        if (tid == 32 && FOLD) stage(b + NBUF - 1);
        WSP(0);

        // ---- S1 (warp 0: the peak and x^2 leaf trees; thread 0: gain,
        // scale code, float block exponent) ----
        if (!FOLD && warp == 0) {
            double peak = 0.0;
            bool nonfin = false;
            if (NEED_PEAK) {
                const unsigned hi = __reduce_max_sync(0xffffffffu, S->pk[lane]);
                const unsigned lo = __reduce_max_sync(0xffffffffu, S->pk[lane] == hi ? S->pn[lane] : 0u);
                const unsigned long long m = ((unsigned long long)hi << 32) | lo;
                nonfin = m >= 0x7ff0000000000000ull;
                peak = __longlong_as_double((long long)m);
            }
            double px = 0.0;
            if (FQ) {   // numpy's pairwise tree over the 32 leaves: the xor butterfly
                if (full) {
                    px = S->lx[lane];
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) px += __shfl_xor_sync(0xffffffffu, px, o);
                } else if (lane == 0) {
                    px = pairwise(scr, n);
                }
            }
          if (lane == 0) {
            if (nonfin) {
                for (int i = 0; i < n; i++)
                    if (!isfinite((double)((const T*)P.x)[base + i])) {
                        atomicMin(&P.status[0], (unsigned long long)(base + i));
                        break;
                    }
            }
            if (FQ) {
                S->pxb = px;
                if (!S->initialized) {   // _init_attenuation (codec.py:155-168)
                    const double rms = sqrt(px / (double)n);
                    double att0 = 0.0;
                    if (rms != 0.0) {
                        const double rqa = F ? (1073741824.0 * rms) / peak : rms;
                        const double a0 = P.pow10_t20 / (P.sqrt12 * rqa);
                        const double m = (1e-300 > a0) ? 1e-300 : a0;
                        att0 = 20.0 * log10(m);
                    }
                    S->att = clamp_att(att0, P.att_lo);
                    S->a = att_to_a(S->att);
                }
            }
            S->initialized = 1;
            const double a = S->a;
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
                    for (;;) {   // overflow guard (codec.py:126-131)
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
            S->code = code; S->fbe = fbe; S->aq = aq;
            S->sq = F ? (zero ? 0.0 : s) : aq;
            S->rs = FQ ? (F ? __ddiv_rn(1.0, s) : (aq != 1.0 ? __ddiv_rn(1.0, aq) : 1.0)) : 1.0;
            S->wide = qpk > (1LL << 30) ? 1 : 0;
            // f64 samples quantized past 32 bits (the block exponent stops at
            // -127): "sample outside 34-bit range", see apax_encode_v3.cu
            if (F && qpk >= (1LL << 31) && !bad) bad = APAX_ERR_INTERNAL;
            S->bad = bad;
            int sel = 0;
            if (S->has_pc) {
                if (S->pc[1] < S->pc[sel]) sel = 1;
                if (S->pc[2] < S->pc[sel]) sel = 2;
            }
            S->sel = sel;
            BlockMeta mt;
            // (a block in error: a zero quantizer, the packer codes a silent block)
            mt.sq = bad ? 0.0 : S->sq; mt.code = code; mt.fbe = (short)fbe; mt.wide = bad ? (short)0 : (short)S->wide;
            P.meta[b] = mt;
            if (P.trace) {
                double* tr = P.trace + 10 * b;
                tr[0] = S->att; tr[1] = a; tr[2] = code; tr[3] = fbe;
            }
          }
        }
        WSP(1);
        if (!FOLD) bar();   // B2
        if (tid == 32 && !FOLD) stage(b + NBUF - 1);   // (after thread 0's S1: off its critical path)
        WSP(2);
        const double sq = S->sq;
        int q[4];
#pragma unroll
        for (int k = 0; k < 4; k++) q[k] = active ? quant<DT>(xd[k], sq) : 0;
        if (tid == G - 1) { S->h1 = q[3]; S->h2 = q[2]; }   // the padded block's last two samples

        if (FQ) {
            // ---- dequantize and the leaf sums of (x - y)^2 (codec.py:244-252) ----
            double* D2 = scr + BS;
            const double sd = F ? sq : S->aq, rs = S->rs;
            const bool idq = !F && S->aq == 1.0;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const double qd = (double)q[k];
                const double y = idq ? qd : deq<DT>(qd, sd, rs);
                const double d = xd[k] - y;
                D2[4 * tid + k] = (4 * tid + k < n) ? d * d : 0.0;
            }
            if (full) {
                __syncwarp();
                double r = 0.0;
                if (lane < 8) {
                    const double* v = D2 + 128 * warp + lane;
                    r = v[0];
#pragma unroll
                    for (int i = 1; i < 16; i++) r += v[8 * i];
                }
                r += __shfl_xor_sync(0xffffffffu, r, 1);
                r += __shfl_xor_sync(0xffffffffu, r, 2);
                r += __shfl_xor_sync(0xffffffffu, r, 4);
                if (lane == 0) S->ld[warp] = r;
            }
            WSP(3);
            bar();   // B3
            WSP(4);
            if (warp == 0) {
                // numpy's pairwise tree over the 32 leaves: the xor butterfly
                double pd;
                if (full) {
                    pd = S->ld[lane];
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) pd += __shfl_xor_sync(0xffffffffu, pd, o);
                } else {
                    pd = lane == 0 ? pairwise(D2, n) : 0.0;
                }
                if (lane == 0) {
                    const double pxm = S->pxb / (double)n, pdm = pd / (double)n;
                    if (pxm > 0.0 && pdm != 0.0 && pxm / pdm == 0.0 && !S->bad) S->bad = APAX_ERR_MATH_DOMAIN;
                    if (pxm > 0.0) {
                        const double measured = (pdm == 0.0) ? INFINITY : 10.0 * log10(pxm / pdm);
                        if (isfinite(measured))
                            S->att = clamp_att(S->att - clamp_step(0.5 * (measured - P.target)), P.att_lo);
                    }
                    S->a = att_to_a(S->att);
                    if (S->bad) report_error(P.status, b, S->bad);
                }
            }
            WSP(5);
            if (b + 1 < nblk) prep(b + 1, xd);   // the next block's samples, peak, x^2 leaves
            WSP(6);
            bar();   // B4
            WSP(7);
            continue;
        }

        // ---- fixed rate: widths of the thread's group, D0/D1/D2 ----
        int hq1 = __shfl_up_sync(0xffffffffu, q[3], 1);
        int hq2 = __shfl_up_sync(0xffffffffu, q[2], 1);
        if (lane == 0) {
            if (tid == 0) { hq1 = S->p1; hq2 = S->p2; }
            else if (active) {
                const T* xs = full ? (const T*)(xbuf + (int)(b % NBUF) * XB) : (const T*)P.x + base;
                hq1 = quant<DT>((double)xs[4 * tid - 1], sq);
                hq2 = quant<DT>((double)xs[4 * tid - 2], sq);
            }
        }
        const bool bwide = S->wide != 0;
        int w0 = 0, w1 = 0, w2 = 0, flips = 0;
        unsigned emax = 0;
        bool ww = bwide;
        if (!bwide) {
            if (active) {
                unsigned o0 = 0, o1 = 0, o2 = 0;
                int m1 = hq1, dprev = hq1 - hq2;
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const int v1 = q[k] - m1, v2 = v1 - dprev;
                    o0 |= wb32(q[k]); o1 |= wb32(v1); o2 |= wb32(v2);
                    flips += (int)((unsigned)(q[k] ^ m1) >> 31);
                    m1 = q[k]; dprev = v1;
                }
                w0 = bitlen32(o0); w1 = bitlen32(o1); w2 = bitlen32(o2);
            }
            bool bad = active && (w1 >= 32 || (!F && w0 >= 32));
            if (tid == 0) {
                const long long d = (long long)hq1 - (long long)hq2;
                bad = bad || d < -(1LL << 30) || d >= (1LL << 30) || hq1 < -(1 << 30) || hq1 > (1 << 30) ||
                      hq2 < -(1 << 30) || hq2 > (1 << 30);
            }
            ww = __any_sync(0xffffffffu, bad);
        }
        if (ww) {
            w0 = w1 = w2 = 0; flips = 0;
            if (active) {
                unsigned long long o0 = 0, o1 = 0, o2 = 0;
                long long m1 = hq1, dprev = (long long)hq1 - (long long)hq2;
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const long long v0 = q[k], v1 = v0 - m1, v2 = v1 - dprev;
                    o0 |= wb64(v0); o1 |= wb64(v1); o2 |= wb64(v2);
                    flips += (int)((unsigned long long)(v0 ^ m1) >> 63);
                    m1 = v0; dprev = v1;
                }
                w0 = bitlen64(o0); w1 = bitlen64(o1); w2 = bitlen64(o2);
                emax = (unsigned)max(w0, max(w1, w2));
            }
        }
        if (tid == 0) flips -= (int)((unsigned)(q[0] ^ hq1) >> 31);   // no predecessor in the block
        // ---- JEE of the speculated selector (the previous block's cost
        // argmin; a centre-frequency gate forces D0 and re-runs this) ----
        auto jee = [&](int sel) {
            const int e = sel == 0 ? w0 : (sel == 1 ? w1 : w2);
            int ep = __shfl_up_sync(0xffffffffu, e, 1);
            int en = __shfl_down_sync(0xffffffffu, e, 1);
            // the neighbour warps' edge groups (exchanged through shared memory)
            if (lane == 0 && warp > 0) ep = (int)((S->edge[warp - 1][1] >> (8 * sel)) & 0xffu);
            if (lane == 31 && warp < NW - 1) en = (int)((S->edge[warp + 1][0] >> (8 * sel)) & 0xffu);
            const int d = e - ep, dn = en - e;
            const bool pr = active && tid > 0 && tid + 1 < G && (unsigned)(d + 1) < 3u && (unsigned)(dn + 1) < 3u;
            const bool es = active && !pr && (tid == 0 || (unsigned)(d + 2) >= 5u);
            const uint32_t Pm = __ballot_sync(0xffffffffu, pr);
            const uint32_t Em = __ballot_sync(0xffffffffu, es);
            const uint32_t Vm = __ballot_sync(0xffffffffu, active);
            uint32_t c0o, c1o;
            const uint32_t C0 = consumed_word(Pm, 0u, &c0o), C1 = consumed_word(Pm, 1u, &c1o);
            const int n0 = __popc(Vm & ~C0) + 2 * __popc(Vm & ~C0 & Em);
            const int n1 = __popc(Vm & ~C1) + 2 * __popc(Vm & ~C1 & Em);
            const int mbits = __reduce_add_sync(0xffffffffu, active ? 4 * e : 0);
            if (lane == 0) {
                S->jw[warp] = (unsigned)n0 | ((unsigned)n1 << 16);
                // transfer: identity when every position pairs (an even run), else a constant
                S->jc[warp] = (c0o == c1o) ? (1 | (int)(c0o << 1)) : 0;
                S->mb[warp] = mbits;
            }
        };
        {   // widths of the warp's first and last group, for the neighbour warps' JEE
            const unsigned ew = (unsigned)w0 | ((unsigned)w1 << 8) | ((unsigned)w2 << 16);
            if (lane == 0) S->edge[warp][0] = ew;
            if (lane == 31) S->edge[warp][1] = ew;
        }
        bar();   // B2b
        const int sel_spec = S->sel;
        jee(sel_spec);
        {
            const unsigned s01 = __reduce_add_sync(0xffffffffu, (unsigned)w0 | ((unsigned)w1 << 16));
            const unsigned s2f = __reduce_add_sync(0xffffffffu, (unsigned)w2 | ((unsigned)flips << 16));
            const unsigned em = __reduce_max_sync(0xffffffffu, emax);
            if (lane == 0) { S->cs01[warp] = s01; S->cs2f[warp] = s2f; S->em[warp] = em; }
        }
        WSP(3);
        bar();   // B3
        WSP(4);
        // totals (every warp, redundantly: lane w = warp w's partials)
        int t0, t1, t2, flt;
        {
            const unsigned a = S->cs01[lane], c = S->cs2f[lane];
            t0 = __reduce_add_sync(0xffffffffu, (int)(a & 0xffffu));
            t1 = __reduce_add_sync(0xffffffffu, (int)(a >> 16));
            t2 = __reduce_add_sync(0xffffffffu, (int)(c & 0xffffu));
            flt = __reduce_add_sync(0xffffffffu, (int)(c >> 16));
        }
        const int np = 4 * G;
        if (3LL * flt > 2LL * (np - 1)) {
            // exact monitor (transform.py:67-83) over the padded q
            int ch = 0, fs = 0, lsg = 0;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int sg = (q[k] > 0) - (q[k] < 0);
                if (active && sg) {
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
            bar();
            int ch2 = 0, f = 0, l = 0;
            for (int w = 0; w < NW; w++) {
                const int of = (S->monf[w] & 3) - 1, ol = ((S->monf[w] >> 2) & 3) - 1;
                ch2 += S->monc[w] + ((l != 0 && of != 0 && l != of) ? 1 : 0);
                if (!f) f = of;
                if (ol) l = ol;
            }
            const int gate = ((double)ch2 / (2.0 * (double)(np - 1))) > 1.0 / 3.0;
            if (gate && sel_spec != 0) {   // D0 after all: its JEE count
                bar();
                jee(0);
                bar();
            }
        }
        // ---- warp 0: block bytes and the rate loop; the other warps stage
        // the next block meanwhile ----
        if (warp == 0) {
            const unsigned jwv = S->jw[lane];
            const int jcv = S->jc[lane];
            // the carry entering warp w: the constant of the nearest earlier
            // warp whose transfer is constant, else 0 (identity transfers pass
            // the carry through; the block starts with none)
            const unsigned cst = __ballot_sync(0xffffffffu, jcv & 1);
            const unsigned val = __ballot_sync(0xffffffffu, (jcv >> 1) & 1);
            const unsigned before = cst & ((1u << lane) - 1u);
            const int cin = before ? (int)((val >> (31 - __clz((int)before))) & 1u) : 0;
            const int nib = __reduce_add_sync(0xffffffffu, (int)(cin ? (jwv >> 16) : (jwv & 0xffffu)));
            const int mbt = __reduce_add_sync(0xffffffffu, S->mb[lane]);
            const unsigned emt = __reduce_max_sync(0xffffffffu, S->em[lane]);
            if (lane == 0) {
                const long long blen = HS + (nib + 1) / 2 + (mbt + 7) / 8;
                if (emt > (unsigned)kMaxExponent && !S->bad) S->bad = APAX_ERR_INTERNAL;
                if (S->bad) report_error(P.status, b, S->bad);
                // rate loop (codec.py:228-243); bs is the configured block size
                if (b == 0) {
                    const long long g4 = 4LL * G;
                    long long mn = t0 < t1 ? t0 : t1;
                    mn = t2 < mn ? t2 : mn;
                    const double bps0 = (double)(4 * mn + g4 + 8LL * HS) / (double)BS;
                    S->att = clamp_att(S->att - 6.02 * (bps0 - P.target), P.att_lo);
                } else {
                    const double err = (double)(blen * 8) / (double)BS - P.target;
                    S->att = clamp_att(S->att - clamp_step(0.75 * err), P.att_lo);
                }
                if (FOLD) {
                    // the next block's quantizer (integers: a_q only) and selector
                    if (b + 1 < nblk) {
                        const int code = code_of_att(S->att);
                        const double aq = scale_code_value(code);
                        S->code = code; S->aq = aq; S->sq = aq;
                        int sel = 0;
                        if (t1 < t0) sel = 1;
                        if (t2 < (sel ? t1 : t0)) sel = 2;
                        S->sel = sel;
                        BlockMeta mt;
                        mt.sq = aq; mt.code = code; mt.fbe = 0; mt.wide = 0;
                        P.meta[b + 1] = mt;
                        if (P.trace) {
                            double* tr = P.trace + 10 * (b + 1);
                            tr[0] = S->att; tr[1] = att_to_a(S->att); tr[2] = code; tr[3] = 0.0;
                        }
                    }
                } else {
                    S->a = att_to_a(S->att);
                }
                S->has_pc = 1;
                S->pc[0] = t0; S->pc[1] = t1; S->pc[2] = t2;
                S->p1 = S->h1; S->p2 = S->h2;
            }
        }
        WSP(5);
        if (b + 1 < nblk) prep(b + 1, xd);   // the next block's samples and peak
        WSP(6);
        bar();   // B4
        WSP(7);
    }
#ifdef APAX_WS_PROF
    if (threadIdx.x == 0)
        for (int k = 0; k < 10; k++) g_ws_prof[k] = wsp_acc[k];
#endif
}

}  // namespace ws

#ifdef APAX_WS_PROF
extern "C" int apax_debug_ws_prof(unsigned long long* host) {
    return (int)cudaMemcpyFromSymbol(host, ws::g_ws_prof, 15 * sizeof(unsigned long long));
}
#endif

bool encode_ws_supported(int dt, int bs) { return bs == ws::BS && dt >= 1 && dt <= 4; }

size_t encode_ws_smem_bytes(int dt, int mode) {
    const size_t xb = (size_t)ws::BS * dt_width(dt);
    return ((sizeof(ws::Sw) + 127) & ~(size_t)127) + ws::NBUF * xb + (mode == 2 ? 2 * (size_t)ws::BS * 8 : 0);
}

template <int DT, bool FQ>
static int launch_ws_t(const EncParams& P, size_t smem, cudaStream_t st) {
    if (cudaFuncSetAttribute(ws::chain_kernel<DT, FQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return APAX_ERR_CUDA;
    note_launches(1);
    ws::chain_kernel<DT, FQ><<<1, ws::NT, smem, st>>>(P);
    return cudaGetLastError() == cudaSuccess ? APAX_OK : APAX_ERR_CUDA;
}

// the whole-stream chain: P.meta receives every block's quantizer record;
// P.x must be 16-byte aligned
int launch_encode_ws_chain(int dt, const EncParams& P, cudaStream_t st) {
    const size_t smem = encode_ws_smem_bytes(dt, P.mode);
    const bool fq = P.mode == 2;
    switch (dt) {
        case 1: return fq ? launch_ws_t<1, true>(P, smem, st) : launch_ws_t<1, false>(P, smem, st);
        case 2: return fq ? launch_ws_t<2, true>(P, smem, st) : launch_ws_t<2, false>(P, smem, st);
        case 3: return fq ? launch_ws_t<3, true>(P, smem, st) : launch_ws_t<3, false>(P, smem, st);
        case 4: return fq ? launch_ws_t<4, true>(P, smem, st) : launch_ws_t<4, false>(P, smem, st);
    }
    return APAX_ERR_ARG;
}

}  // namespace apax
