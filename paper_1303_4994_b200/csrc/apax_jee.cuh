// apax_jee.cuh -- exact warp-parallel JEE decoder (reference entropy.py:118-191)
// shared by the decode kernels and the block walk.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

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


}  // namespace apax
