// apax_jee.cuh -- exact warp-parallel JEE decoder (reference entropy.py:118-191)
// shared by the decode kernels and the block walk.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "apax_device.cuh"

namespace apax {

// read one nibble k of the payload (first nibble in the high half)
__device__ __forceinline__ int nib_at(const uint8_t* p, long long k) {
    uint8_t b = p[k >> 1];
    return (k & 1) ? (b & 15) : (b >> 4);
}

// ---------------------------------------------------------------------------
// Warp-parallel JEE decode (entropy.py:118-164): all 32 lanes of the calling
// warp participate.  Writes exponents to e[0..G) and returns status (0..5)
// and nibbles consumed via refs (valid in every lane).  `total` = nibbles
// available.  Semantics identical to the serial kernel, including which
// error is reported first.
// ---------------------------------------------------------------------------
static __device__ __noinline__ int warp_jee_decode(const uint8_t* p, long long total, int G, uint8_t* e,
                               long long& used, long long& esum) {
    const int lane = threadIdx.x & 31;
    long long base = 0;     // nibble index of window start
    int skip = 0;           // leading nibbles of the window covered by an escape
    int cnt = 0;            // exponents produced so far
    int last = 0;           // value of the last exponent
    long long sum = 0;
    for (;;) {
        const long long pos = base + lane;
        const bool valid = pos < total;
        const int nib = valid ? nib_at(p, pos) : 0;
        const unsigned F = __ballot_sync(0xffffffffu, valid && nib == 15);
        // token starts: positions >= skip not covered by an earlier escape
        unsigned cover = 0, escs = 0;
        unsigned f = F & (0xffffffffu << skip);
        unsigned long long spill = 0;  // coverage beyond the window
        while (f) {
            int q = __ffs(f) - 1;
            f &= f - 1;
            if ((cover >> q) & 1u) continue;
            escs |= 1u << q;
            unsigned long long cm = 3ULL << (q + 1);
            cover |= (unsigned)cm;
            spill |= cm >> 32;
        }
        const unsigned starts = (0xffffffffu << skip) & ~cover;
        const bool is_start = (starts >> lane) & 1u;
        const bool is_esc = (escs >> lane) & 1u;
        // per-token evaluation (meaningful for start lanes only)
        int kind = 0;     // 0 none, 1 esc, 2 joint, 3 single, 4 reserved
        int nexp = 0, d1 = 0, d2 = 0, absval = 0;
        int terr = 0;     // error detected before needing the running values
        if (is_start) {
            if (!valid) { terr = 1; }
            else if (nib == 14) { kind = 4; terr = 2; }
            else if (is_esc) {
                kind = 1; nexp = 1;
                // serial check `pos + 1 >= total` after consuming the 15
                if (pos + 2 >= total) terr = 1;
                else {
                    absval = (nib_at(p, pos + 1) << 4) | nib_at(p, pos + 2);
                    if (absval > 34) terr = 3;
                }
            } else if (nib >= 9) { kind = 3; nexp = 1; d1 = nib - 11; }
            else { kind = 2; nexp = 2; d1 = nib / 3 - 1; d2 = nib % 3 - 1; }
        }
        // exclusive prefix of exponent counts -> index of the token's first exponent
        int incl = nexp;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int o = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += o;
        }
        const int idx = cnt + incl - nexp;
        // segmented scan of values: escape resets to absval, others add deltas
        int seg_flag = (kind == 1) ? 1 : 0;
        int seg_val = (kind == 1) ? absval : (d1 + d2);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int of = __shfl_up_sync(0xffffffffu, seg_flag, d);
            int ov = __shfl_up_sync(0xffffffffu, seg_val, d);
            if (lane >= d && !seg_flag) { seg_val += ov; seg_flag |= of; }
        }
        const int after = seg_flag ? seg_val : last + seg_val;      // value after token
        int before = __shfl_up_sync(0xffffffffu, after, 1);
        if (lane == 0) before = last;
        // full error evaluation in serial order
        int err = 0;
        int v1 = 0, v2 = 0;
        if (is_start && idx < G) {
            if (terr == 1 && !valid) err = 1;
            else if (terr == 2) err = 2;
            else if (kind == 1) { err = terr; v1 = absval; }
            else if (idx == 0) err = 5;
            else if (kind == 3) {
                v1 = before + d1;
                if (v1 < 0 || v1 > 34) err = 3;
            } else if (kind == 2) {
                v1 = before + d1;
                if (v1 < 0 || v1 > 34) err = 3;
                else if (idx + 1 >= G) err = 4;
                else {
                    v2 = v1 + d2;
                    if (v2 < 0 || v2 > 34) err = 3;
                }
            }
        }
        // the token that completes the stream (no error): idx < G <= idx + nexp
        const bool active = is_start && idx < G;
        const unsigned errm = __ballot_sync(0xffffffffu, active && err);
        const unsigned donem = __ballot_sync(0xffffffffu, active && !err && idx + nexp >= G);
        // tokens before the first error / completion are final: write them
        const int first_err = errm ? __ffs(errm) - 1 : 32;
        const int first_done = donem ? __ffs(donem) - 1 : 32;
        const int stop = first_err < first_done ? first_err : first_done;
        if (active && lane <= stop && !(lane == first_err)) {
            if (kind == 1 || kind == 3) { e[idx] = (uint8_t)v1; sum += v1; }
            else if (kind == 2) { e[idx] = (uint8_t)v1; e[idx + 1] = (uint8_t)v2; sum += v1 + v2; }
        }
        if (errm && first_err <= first_done) {
            int code = __shfl_sync(0xffffffffu, err, first_err);
            // nibbles consumed up to the failing read (for completeness)
            used = base + first_err + 1;
            esum = 0;
            return code;
        }
        if (donem) {
            int kd = __shfl_sync(0xffffffffu, kind, first_done);
            used = base + first_done + (kd == 1 ? 3 : 1);
            // reduce the exponent sum over lanes
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            esum = sum;
            return 0;
        }
        // advance to the next window
        cnt = __shfl_sync(0xffffffffu, idx + nexp, 31);
        last = __shfl_sync(0xffffffffu, after, 31);
        base += 32;
        // 0b01 -> window position 0 covered; 0b11 -> positions 0 and 1
        skip = (spill & 2ULL) ? 2 : (spill & 1ULL ? 1 : 0);
        if (base >= total + 2) {
            // nothing left: the next start position is past the end
            used = total;
            esum = 0;
            return 1;
        }
    }
}

// ---------------------------------------------------------------------------
// JEE decode of one block by one warp (entropy.py:118-164), reading the
// nibble stream straight from global memory (read-only path): 128 nibbles
// per step, 4 per lane.  Two consecutive non-15 nibbles always precede a
// token start, so every lane finds the token starts in its slice from a
// 16-nibble window; one warp scan of (exponent count, escape reset, running
// value) places the exponents.  Returns 0 with e[0..G) and *used (nibbles
// consumed), or -1 on ANY irregularity (reserved nibble, range, truncation,
// missing opening escape, joint token past the last group): the caller then
// runs the exact parser (apax_jee.cuh), which reports the reference's first
// error.  e must hold G + 128 bytes (tokens are written before validation).
// ---------------------------------------------------------------------------
// LDG false: p / pend may point into shared memory (a staged copy whose
// bytes keep their global alignment mod 4, with >= 4 bytes before p)
template <bool LDG = true>
static __device__ __forceinline__ int warp_jee_fast(const uint8_t* p, const uint8_t* pend, int total, int G,
                                             uint8_t* e, int& used) {
    const int lane = threadIdx.x & 31;
    constexpr unsigned long long LUT_C = 0x43210cbaba9a98ull;    // bit 3 joint, bits 0-2 delta sum + 2
    constexpr unsigned long long LUT_D1 = 0x43210333222111ull;   // first exponent's delta + 2
    constexpr unsigned LUT_D2 = 0x24924u;                        // (2-bit) second delta + 1
    int cbase = 0, vbase = 0;
    for (int base = 0; base < total + 4; base += 128) {
        const int p0 = base + 4 * lane;
        // nibbles p0-4 .. p0+11 (zero beyond `total`); bytes before p are the
        // block header (>= 4 bytes), so p0 = 0 reads inside the container
        unsigned long long W = 0ULL;
        if (p0 - 4 < total) {
            const uint8_t* bp = p + (p0 >> 1) - 2;
            const uintptr_t a = (uintptr_t)bp;
            const uint32_t* wp = (const uint32_t*)(a & ~(uintptr_t)3);
            const unsigned sh = (unsigned)(a & 3) * 8u;
            uint32_t w0, w1, w2;
            if ((const uint8_t*)(wp + 3) <= pend) {
                if (LDG) { w0 = bswap32(__ldg(wp)); w1 = bswap32(__ldg(wp + 1)); w2 = bswap32(__ldg(wp + 2)); }
                else { w0 = bswap32(wp[0]); w1 = bswap32(wp[1]); w2 = bswap32(wp[2]); }
            } else {   // the last words of the container: bytewise, zero past the end
                uint32_t w[3];
                for (int k = 0; k < 3; k++) {
                    uint32_t v = 0;
                    for (int c = 0; c < 4; c++) {
                        const uint8_t* q = (const uint8_t*)(wp + k) + c;
                        v = (v << 8) | (q < pend ? (uint32_t)*q : 0u);
                    }
                    w[k] = v;
                }
                w0 = w[0]; w1 = w[1]; w2 = w[2];
            }
            W = ((unsigned long long)__funnelshift_l(w1, w0, sh) << 32) | __funnelshift_l(w2, w1, sh);
            const int rem = total - (p0 - 4);
            if (rem < 16) W = rem <= 0 ? 0ULL : (W & (~0ULL << (4 * (16 - rem))));
        }
        auto nw = [&](int k) -> int { return (int)((W >> (4 * (11 - k))) & 15ULL); };   // k in -4..11
        // leading positions covered by an escape that started before p0
        int skip = 0;
        if (p0 > 0 && p0 < total + 4) {
            const bool f1 = nw(-1) == 15, f2 = nw(-2) == 15, f3 = nw(-3) == 15, f4 = nw(-4) == 15;
            if (!f1 && !f2) skip = 0;
            else if (!f2 && !f3) skip = f1 ? 2 : 0;
            else if (!f3 && !f4) skip = f2 ? 1 : (f1 ? 2 : 0);
            else {
                // long escape run: walk back to a definite start (rare)
                auto nb = [&](int k) -> int {
                    if (k >= total) return 0;
                    const uint8_t b = p[k >> 1];
                    return (k & 1) ? (b & 15) : (b >> 4);
                };
                int q = p0;
                while (q > 0 && !(nb(q - 1) != 15 && (q < 2 || nb(q - 2) != 15))) q--;
                int pos = q;
                while (pos < p0) pos += (nb(pos) == 15) ? 3 : 1;
                skip = pos - p0;
            }
        }
        const bool n0f = nw(0) == 15, n1f = nw(1) == 15, n2f = nw(2) == 15;
        const bool st0 = skip == 0;
        const bool st1 = skip == 1 || (st0 && !n0f);
        const bool st2 = skip == 2 || (st1 && !n1f);
        const bool st3 = (st2 && !n2f) || (st0 && n0f);
        const bool stv[4] = {st0, st1, st2, st3};
        const bool live = p0 < total + 4;
        int cnt = 0, flag = 0, val = 0;
        int kv[4], kab[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int v = nw(k);
            const int ab = (int)((W >> (4 * (9 - k))) & 0xffULL);   // nibbles k+1, k+2
            kv[k] = v;
            kab[k] = ab;
            const int cd = (int)((LUT_C >> (4 * v)) & 15ull);
            const bool esc = v == 15;
            const int c = esc ? 1 : (cd >> 3) + 1;
            const int dv = (cd & 7) - 2;
            const bool t = stv[k] && live;
            cnt += t ? c : 0;
            val = t ? (esc ? ab : val + dv) : val;
            flag |= (t && esc) ? 1 : 0;
        }
        // warp scan of (cnt, flag, val): A then B = (cA+cB, fA|fB, fB ? vB : vA+vB),
        // packed in one word (cnt bits 0-14, flag bit 15, val bits 16-31 signed:
        // |cnt| <= 256, -256 <= val <= 509 over a warp), so a step is one shuffle
        auto pk = [](int c, int f, int v) -> unsigned { return (unsigned)c | ((unsigned)f << 15) | ((unsigned)v << 16); };
        unsigned X = pk(cnt, flag, val);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned O = __shfl_up_sync(0xffffffffu, X, d);
            if (lane >= d) X += (X & 0x8000u) ? (O & 0x7fffu) : O;
        }
        unsigned EX = __shfl_up_sync(0xffffffffu, X, 1);
        if (lane == 0) EX = 0;
        const int ec = (int)(EX & 0x7fffu), ef = (int)((EX >> 15) & 1u), evv = (int)EX >> 16;
        int idx = cbase + ec;
        int curv = ef ? evv : vbase + evv;
        int key = 0x7fffffff;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int pos = p0 + k;
            const int v = kv[k];
            const bool t = stv[k] && live && idx < G;   // tokens after the G-th exponent are not read
            const bool esc = v == 15;
            const int cd = (int)((LUT_C >> (4 * v)) & 15ull);
            const bool joint = !esc && (cd >> 3) != 0;
            const int e1 = esc ? kab[k] : curv + (int)((LUT_D1 >> (4 * v)) & 15ull) - 2;
            const int e2 = e1 + (int)((LUT_D2 >> (2 * v)) & 3u) - 1;
            const bool bad = (pos + (esc ? 2 : 0) >= total) | (v == 14) | (!esc & (idx == 0)) |
                             ((unsigned)e1 > 34u) | (joint & ((idx + 1 >= G) | ((unsigned)e2 > 34u)));
            const int nexp = joint ? 2 : 1;
            const bool done = idx + nexp >= G;
            if (t) {
                e[idx] = (uint8_t)e1;
                if (joint) e[idx + 1] = (uint8_t)e2;
            }
            const int kk2 = bad ? 1 : (done ? ((pos + (esc ? 3 : 1)) << 1) : 0x7fffffff);
            key = t ? min(key, kk2) : key;
            curv = t ? (joint ? e2 : e1) : curv;
            idx += t ? nexp : 0;
        }
        key = __reduce_min_sync(0xffffffffu, key);
        if (key != 0x7fffffff) {
            if (key & 1) return -1;
            used = key >> 1;
            return 0;
        }
        // the next step continues the scan
        const unsigned TX = __shfl_sync(0xffffffffu, X, 31);
        const int tc = (int)(TX & 0x7fffu), tf = (int)((TX >> 15) & 1u), tv = (int)TX >> 16;
        cbase += tc;
        vbase = tf ? tv : vbase + tv;
    }
    return -1;
}


}  // namespace apax
