// apax_encode.cu -- B200 APAX encoder (K1 lossless / K2 adaptive segments /
// K3 look-back placement, SURVEY.md §2 "B200 kernels the build writes").
//
// Reproduces reference `encode_stream` (pkg/src/apax/codec.py:258-285) and
// `encode_block` (codec.py:192-255) byte for byte:
//   * one persistent CTA walks one *unit* of consecutive blocks serially
//     (the adaptive attenuator of codec.py:228-252 is a per-block serial
//     chain); units are handed out by an atomic ticket so lower units are
//     always resident or finished (deadlock-free look-back);
//   * unit = container segment (fresh CodecState, restart flag) for FR/FQ
//     segments or whole stream; for LOSSLESS whole-stream encodes a unit is
//     an arbitrary block range whose CodecState is rebuilt from the halo
//     (history = previous two samples, prev_costs = previous block's costs),
//     which is byte-identical to the serial reference;
//   * per block: quantize (codec.py:94-132) -> monitor (transform.py:67-83)
//     -> derive d0/d1/d2 (transform.py:86-91) -> select (transform.py:107-113)
//     -> group exponents x3 (entropy.py:38-55) -> JEE (entropy.py:63-88) as a
//     2-state automaton scan -> MSB-first mantissa pack (entropy.py:222-240)
//     into a shared-memory staging window -> loop update;
//   * unit byte lengths are placed by a single-pass decoupled look-back, then
//     the staged bytes are copied to their final offset.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "apax_device.cuh"
#include "apax_kernels.cuh"

namespace apax {


// per-CTA state living in shared memory (codec.py:66-82 CodecState)
struct EncState {
    double att;           // AttenuatorState.att_db
    long long p1, p2;     // DerivativeHistory
    long long pc[3];      // prev_costs (Σe per stream; cost = 4Σe + 4g)
    int has_pc;
    int initialized;
    long long emitted;    // blocks_emitted within the unit's CodecState
    // per-block broadcast values
    double a, s, aq, px, pd, peak;
    int code, fbe, sel, bad, nonfinite;
    long long sum_e[3];
    int gate;
    long long nib_total, bits_total, block_bytes;
    // staging window bookkeeping
    long long staged;     // bytes used in the window
    long long win_base;   // unit-relative byte offset of window byte 0
    int direct;           // window flushes go straight to the final output
    long long unit_len;   // bytes emitted so far in this unit
    long long unit;       // current unit id
    long long prefix;     // unit's final byte offset (after header)
    double red_d[kWarps * 4];
    long long red_l[kWarps * 4];
    unsigned red_u[kWarps * 4];
    int leaf_n;
};

// ---------------------------------------------------------------------------
// numpy pairwise summation of term(i), i in [0, n), over the CTA.
// Regular sizes (n = 64 or 128 * 2^k) use an 8-lane-per-leaf butterfly that
// is exactly numpy's association tree; other sizes enumerate the leaves.
// Result valid in thread 0.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool pairwise_regular(int n) {
    if (n == 64) return true;
    if (n < 128 || n > 16384 || (n & 127)) return false;
    int L = n >> 7;
    return (L & (L - 1)) == 0;
}

template <typename F>
__device__ double leaf_sum(F& term, int start, int len) {
    if (len < 8) {
        double r = -0.0;
        for (int i = 0; i < len; i++) r += term(start + i);
        return r;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = term(start + j);
    int i = 8;
    for (; i < len - (len % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] += term(start + i + j);
    }
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < len; i++) res += term(start + i);
    return res;
}

// generic-size tree: leaves enumerated by thread 0 into smem
struct LeafList {
    int start[320];
    int len[320];
    double sum[320];
};

__device__ int enumerate_leaves(int n, LeafList* L) {
    // iterative DFS, left-to-right
    int st_s[32], st_l[32], sp = 0, k = 0;
    st_s[sp] = 0; st_l[sp] = n; sp++;
    while (sp) {
        sp--;
        int s = st_s[sp], l = st_l[sp];
        if (l <= 128) {
            L->start[k] = s; L->len[k] = l; k++;
        } else {
            int n2 = l / 2;
            n2 -= n2 % 8;
            st_s[sp] = s + n2; st_l[sp] = l - n2; sp++;   // right, popped later
            st_s[sp] = s; st_l[sp] = n2; sp++;            // left
        }
    }
    return k;
}

__device__ double combine_leaves(int s, int l, const LeafList* L, int& k) {
    if (l <= 128) return L->sum[k++];
    int n2 = l / 2;
    n2 -= n2 % 8;
    double a = combine_leaves(s, n2, L, k);
    double b = combine_leaves(s + n2, l - n2, L, k);
    return a + b;
}

// `term` may have side effects that must happen exactly once per index
// (quantize-and-store); in the regular path every index is visited once.
template <typename F>
__device__ double block_pairwise(F term, int n, EncState* S, LeafList* LL) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double result = 0.0;
    if (pairwise_regular(n)) {
        const int j = lane & 7;          // accumulator index within the leaf
        const int grp = tid >> 3;        // 8-lane group id, 0..31
        if (n == 64) {
            double r = 0.0;
            if (warp == 0 && grp == 0) {
                r = term(j);
#pragma unroll
                for (int i = 1; i < 8; i++) r += term(8 * i + j);
            }
            if (warp == 0) {
                r += __shfl_xor_sync(0xffffffffu, r, 1);
                r += __shfl_xor_sync(0xffffffffu, r, 2);
                r += __shfl_xor_sync(0xffffffffu, r, 4);
            }
            if (tid == 0) result = r;
            __syncthreads();
            return result;
        }
        const int L = n >> 7;                       // leaves
        const int groups = L < 32 ? L : 32;          // active 8-lane groups
        const int lpg = L / groups;                  // leaves per group (1,2,4)
        double gsum = 0.0;
        // warp-uniform: every lane of a warp holding an active group takes
        // part in the shuffles (inactive groups shuffle zeros among themselves)
        if (warp * 4 < groups) {
            double ls[4];
            for (int q = 0; q < lpg; q++) {
                double r = 0.0;
                if (grp < groups) {
                    int base = (grp * lpg + q) << 7;
                    r = term(base + j);
#pragma unroll 4
                    for (int i = 1; i < 16; i++) r += term(base + 8 * i + j);
                }
                r += __shfl_xor_sync(0xffffffffu, r, 1);
                r += __shfl_xor_sync(0xffffffffu, r, 2);
                r += __shfl_xor_sync(0xffffffffu, r, 4);
                ls[q] = r;
            }
            if (lpg == 1) gsum = ls[0];
            else if (lpg == 2) gsum = ls[0] + ls[1];
            else gsum = (ls[0] + ls[1]) + (ls[2] + ls[3]);
        }
        // butterfly across the 4 groups of a warp (only between active groups)
        const int gw = groups < 4 ? groups : 4;
        if (warp * 4 < groups) {
            if (gw >= 2) gsum += __shfl_xor_sync(0xffffffffu, gsum, 8);
            if (gw >= 4) gsum += __shfl_xor_sync(0xffffffffu, gsum, 16);
        }
        const int nw = (groups + 3) / 4;              // warps holding data
        if (lane == 0 && warp < nw) S->red_d[warp] = gsum;
        __syncthreads();
        if (tid == 0) {
            double v[8];
            for (int w = 0; w < nw; w++) v[w] = S->red_d[w];
            for (int stride = 1; stride < nw; stride <<= 1)
                for (int w = 0; w + stride < nw; w += 2 * stride) v[w] = v[w] + v[w + stride];
            result = v[0];
        }
        __syncthreads();
        return result;
    }
    // generic tree
    if (tid == 0) S->leaf_n = enumerate_leaves(n, LL);
    __syncthreads();
    const int nl = S->leaf_n;
    for (int k = tid; k < nl; k += kNT) LL->sum[k] = leaf_sum(term, LL->start[k], LL->len[k]);
    __syncthreads();
    if (tid == 0) {
        int k = 0;
        result = combine_leaves(0, n, LL, k);
    }
    __syncthreads();
    return result;
}

// ---------------------------------------------------------------------------
// ordered monitor combine (transform.py:67-83): sign changes in the nonzero
// subsequence.  Packed as {first(2b) last(2b) has(1b)} + changes + nnz.
// ---------------------------------------------------------------------------
struct Mon {
    int first, last;   // -1 / +1, 0 = none
    int changes;
    int nnz;
};
__device__ __forceinline__ Mon mon_combine(const Mon& a, const Mon& b) {
    Mon r;
    r.changes = a.changes + b.changes + ((a.nnz && b.nnz && a.last != b.first) ? 1 : 0);
    r.first = a.nnz ? a.first : b.first;
    r.last = b.nnz ? b.last : a.last;
    r.nnz = a.nnz + b.nnz;
    return r;
}

// ---------------------------------------------------------------------------
// JEE 2-state automaton (entropy.py:63-88).  State at a group position:
// S (token starts here) or C (consumed by the previous joint token).
// A thread's local function maps its input state to (output state, nibbles);
// packed: bit0 out(S), bit1 out(C), bits 2..16 nib(S), bits 17..31 nib(C).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t jf_pack(int o0, int o1, int n0, int n1) {
    return (uint32_t)o0 | ((uint32_t)o1 << 1) | ((uint32_t)n0 << 2) | ((uint32_t)n1 << 17);
}
__device__ __forceinline__ uint32_t jf_compose(uint32_t a, uint32_t b) {  // a then b
    int ao0 = a & 1, ao1 = (a >> 1) & 1;
    int an0 = (a >> 2) & 0x7fff, an1 = (a >> 17) & 0x7fff;
    int bo[2] = {(int)(b & 1), (int)((b >> 1) & 1)};
    int bn[2] = {(int)((b >> 2) & 0x7fff), (int)((b >> 17) & 0x7fff)};
    return jf_pack(bo[ao0], bo[ao1], an0 + bn[ao0], an1 + bn[ao1]);
}
constexpr uint32_t kJfIdentity = 0u | (1u << 1);  // out(S)=S, out(C)=C, 0 nibbles

// token kind at position i in state S: 0 joint, 1 single, 2 escape
__device__ __forceinline__ int jee_kind(const uint8_t* e, int i, int G) {
    if (i == 0) return 2;
    int d = (int)e[i] - (int)e[i - 1];
    if (i + 1 < G && d >= -1 && d <= 1) {
        int d2 = (int)e[i + 1] - (int)e[i];
        if (d2 >= -1 && d2 <= 1) return 0;
    }
    return (d >= -2 && d <= 2) ? 1 : 2;
}

__device__ __forceinline__ void jee_local(const uint8_t* e, int lo, int hi, int G, int in_state,
                                          int& out_state, int& nib) {
    int s = in_state, k = 0;
    for (int i = lo; i < hi; i++) {
        if (s) { s = 0; continue; }
        int kind = jee_kind(e, i, G);
        if (kind == 0) { k += 1; s = 1; }
        else if (kind == 1) { k += 1; }
        else { k += 3; }
    }
    out_state = s;
    nib = k;
}

// CTA-wide exclusive scan of (jee function, mantissa bits).  Returns the
// thread's exclusive prefix; totals land in S->nib_total / S->bits_total.
__device__ __forceinline__ void cta_scan_jee(uint32_t f, unsigned bits, uint32_t& f_excl,
                                             unsigned& bits_excl, EncState* S) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t fi = f;
    unsigned bi = bits;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t of = __shfl_up_sync(0xffffffffu, fi, d);
        unsigned ob = __shfl_up_sync(0xffffffffu, bi, d);
        if (lane >= d) { fi = jf_compose(of, fi); bi += ob; }
    }
    uint32_t fx = __shfl_up_sync(0xffffffffu, fi, 1);
    unsigned bx = __shfl_up_sync(0xffffffffu, bi, 1);
    if (lane == 0) { fx = kJfIdentity; bx = 0; }
    if (lane == 31) { S->red_u[warp] = fi; S->red_u[kWarps + warp] = bi; }
    __syncthreads();
    if (tid == 0) {
        uint32_t acc = kJfIdentity;
        unsigned accb = 0;
        for (int w = 0; w < kWarps; w++) {
            uint32_t wf = S->red_u[w];
            unsigned wb = S->red_u[kWarps + w];
            S->red_u[w] = acc;
            S->red_u[kWarps + w] = accb;
            acc = jf_compose(acc, wf);
            accb += wb;
        }
        S->nib_total = (long long)((acc >> 2) & 0x7fff);  // applied to S (state 0)
        S->bits_total = accb;
    }
    __syncthreads();
    f_excl = jf_compose(S->red_u[warp], fx);
    bits_excl = S->red_u[kWarps + warp] + bx;
}

// ---------------------------------------------------------------------------
// the encoder kernel
// ---------------------------------------------------------------------------
template <int DT>
__global__ void __launch_bounds__(kNT) encode_kernel(EncParams P) {
    using Tr = DT_<DT>;
    using T = typename Tr::T;
    using Q = typename Tr::Q;
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x;
    const int bs = P.bs;
    const int Gfull = bs / 4;
    const int gpt = (Gfull + kNT - 1) / kNT;  // groups per thread

    // carve shared memory
    EncState* S = (EncState*)smem;
    size_t off = (sizeof(EncState) + 15) & ~(size_t)15;
    LeafList* LL = (LeafList*)(smem + off);
    off += (sizeof(LeafList) + 15) & ~(size_t)15;
    T* const xs_smem = (T*)(smem + off);
    if (P.x_in_smem) off += ((size_t)bs * sizeof(T) + 15) & ~(size_t)15;
    const T* xb = xs_smem;  // current block's samples (smem copy or global)
    Q* qb = (Q*)(smem + off);
    off += ((size_t)(bs + 4) * sizeof(Q) + 15) & ~(size_t)15;
    uint8_t* es = (uint8_t*)(smem + off);       // 3 x Gfull exponents
    off += ((size_t)3 * Gfull + 16 + 15) & ~(size_t)15;
    uint32_t* stage = (uint32_t*)(smem + off);  // staging window (+16 pad)
    const int stage_words = P.stage_bytes / 4;

    uint8_t* slot = P.slots + (long long)blockIdx.x * P.slot_bytes;
    const int hs = Tr::HDR;

    for (;;) {
        // ---------------- acquire a unit ----------------
        if (tid == 0) S->unit = (long long)atomicAdd(P.ticket, 1u);
        for (int i = tid; i < stage_words + 4; i += kNT) stage[i] = 0u;
        __syncthreads();
        const long long u = S->unit;
        if (u >= P.n_units) break;
        const long long b0 = u * P.unit_blocks;
        const long long b1 = (b0 + P.unit_blocks < P.n_blocks) ? b0 + P.unit_blocks : P.n_blocks;
        if (tid == 0) {
            S->att = 0.0; S->p1 = 0; S->p2 = 0; S->has_pc = 0; S->initialized = 0;
            S->emitted = 0; S->staged = 0; S->win_base = 0; S->unit_len = 0;
            S->direct = (u == 0);
            S->prefix = 0;
            if (P.state) {   // encode_block: the caller's CodecState (codec.py:66-82)
                const apax_block_state* cs = P.state;
                S->att = cs->att_db; S->p1 = cs->prev1; S->p2 = cs->prev2;
                S->has_pc = cs->has_costs;
                S->pc[0] = cs->costs[0]; S->pc[1] = cs->costs[1]; S->pc[2] = cs->costs[2];
                S->initialized = cs->initialized;
                S->emitted = cs->blocks_emitted;
            }
        }
        __syncthreads();

        // ---------------- per-block pass (lambda-like via local function) --
        // mode_pass: 0 = emit, 1 = cost-only with forced a and history (0,0)
        //            or halo history set by the caller
        auto load_block = [&](long long b, int n) {
            const T* src = (const T*)P.x + b * (long long)bs;
            if (!P.x_in_smem) {  // large blocks: read the samples from global / L2
                xb = src;
                return;
            }
            T* dst = xs_smem;
            xb = dst;
            // 16-byte vector loads when aligned
            const int bytes = n * (int)sizeof(T);
            if ((((uintptr_t)src) & 15) == 0) {
                const int nv = bytes >> 4;
                const uint4* s4 = (const uint4*)src;
                uint4* d4 = (uint4*)dst;
                for (int i = tid; i < nv; i += kNT) d4[i] = __ldcs(s4 + i);
                for (int i = (nv << 4) / (int)sizeof(T) + tid; i < n; i += kNT) dst[i] = src[i];
            } else {
                for (int i = tid; i < n; i += kNT) dst[i] = src[i];
            }
        };

        // Quantize + stats + exponents + selection for the block in xb.
        // force_a >= 0 -> use that gain (cost-only passes).  Returns nothing;
        // results in S and smem (qb, es).
        auto analyze = [&](long long b, int n, double force_a, bool fq_update) {
            const int G = (n + 3) >> 2;
            const int np = G * 4;
            // ---- phase A: peak / non-finite / px ----
            if (Tr::F || P.mode == 2) {
                double pk = 0.0;
                int nf = 0;
                for (int i = tid; i < n; i += kNT) {
                    double v = (double)xb[i];
                    if (Tr::F && !isfinite(v)) { nf = 1; continue; }
                    double av = fabs(v);
                    pk = av > pk ? av : pk;
                }
                pk = warp_allreduce(pk, MaxOp());
                nf = __syncthreads_or(nf);
                if ((tid & 31) == 0) S->red_d[kWarps + (tid >> 5)] = pk;
                __syncthreads();
                if (tid == 0) {
                    double m = 0.0;
                    for (int w = 0; w < kWarps; w++) m = S->red_d[kWarps + w] > m ? S->red_d[kWarps + w] : m;
                    S->peak = m;
                    S->nonfinite = nf;
                }
                if (P.mode == 2) {
                    double px = block_pairwise([&](int i) { double v = (double)xb[i]; return v * v; }, n, S, LL);
                    if (tid == 0) S->px = px;
                } else {
                    __syncthreads();
                }
            } else {
                if (tid == 0) S->nonfinite = 0;
            }
            // ---- scalar: gain, code, scale (thread 0) ----
            if (tid == 0) {
                if (Tr::F && S->nonfinite) {
                    // report the first non-finite index of the block
                    for (int i = 0; i < n; i++) {
                        if (!isfinite((double)xb[i])) {
                            atomicMin(&P.status[0], (unsigned long long)(b * (long long)bs + i));
                            break;
                        }
                    }
                }
                if (force_a < 0.0 && !S->initialized) {
                    if (P.mode == 2) {
                        // _init_attenuation (codec.py:155-168)
                        double rms = sqrt(S->px / (double)n);
                        double att0 = 0.0;
                        if (rms != 0.0) {
                            double rqa = Tr::F ? (1073741824.0 * rms) / S->peak : rms;
                            double a0 = P.pow10_t20 / (P.sqrt12 * rqa);
                            double m = (1e-300 > a0) ? 1e-300 : a0;
                            att0 = 20.0 * log10(m);
                        }
                        double mm = (P.att_lo > att0) ? P.att_lo : att0;
                        S->att = (0.0 < mm) ? 0.0 : mm;
                    }
                    S->initialized = 1;
                }
                double a;
                if (force_a >= 0.0) a = force_a;
                else if (P.mode == 0) a = 1.0;
                else {
                    double p = pow(10.0, S->att / 20.0);
                    double m = (4.656612873077393e-10 > p) ? 4.656612873077393e-10 : p;
                    a = (1.0 < m) ? 1.0 : m;
                }
                S->a = a;
                S->bad = 0;
                if (!Tr::F) {
                    int code = encode_scale_code(a);
                    S->code = code;
                    S->aq = decode_scale_code(code);
                    S->fbe = 0;
                } else {
                    double peak = S->peak;
                    if (S->nonfinite || peak == 0.0) {
                        S->code = kScaleCodeOne; S->fbe = 0; S->s = 0.0;  // zeros
                    } else {
                        double s_des = (a * 1073741824.0) / peak;
                        if (!isfinite(s_des)) {
                            S->bad = APAX_ERR_OVERFLOW;
                            S->code = kScaleCodeOne; S->fbe = 0; S->s = 0.0;
                        } else {
                            long long l2 = floor_log2_rn(s_des);
                            long long fb = (-31 <= l2 && l2 <= 31) ? 0 : l2 - 31;
                            fb = fb < -127 ? -127 : (fb > 127 ? 127 : fb);
                            double rem = ldexp(s_des, (int)-fb);
                            const double nxt = 8589934591.999999;  // nextafter(2^33, 0)
                            double mm = (nxt < rem) ? nxt : rem;
                            rem = (mm > 4.656612873077393e-10) ? mm : 4.656612873077393e-10;
                            S->code = encode_scale_code(rem);
                            S->fbe = (int)fb;
                            S->s = decode_scale_code(S->code) * ldexp(1.0, (int)fb);
                        }
                    }
                }
            }
            __syncthreads();
            // ---- phase B: quantize (+ FQ residual power) ----
            // retry loop for the float overflow guard (codec.py:126-131)
            for (;;) {
                const double s = S->s, aq = S->aq;
                const bool zero = Tr::F && (S->s == 0.0);
                double qmax = 0.0;
                auto quant = [&](int i) -> Q {
                    if (Tr::F) {
                        if (zero) return (Q)0;
                        double r = rint((double)xb[i] * s);
                        double ar = fabs(r);
                        if (!(ar <= qmax)) qmax = (ar != ar) ? INFINITY : ar;
                        return (Q)f2i64(r);
                    } else {
                        long long xv = (long long)xb[i];
                        if (aq == 1.0) return (Q)xv;
                        return (Q)f2i64(rint((double)xv * aq));
                    }
                };
                const bool fq_stats = fq_update && P.mode == 2;
                if (fq_stats) {
                    // dequantize_block (codec.py:135-146) fused with d*d
                    const int code = S->code, fbe = S->fbe;
                    const double deq_s = decode_scale_code(code) * ldexp(1.0, fbe);
                    const double deq_a = decode_scale_code(code);
                    double pd = block_pairwise([&](int i) {
                        Q qv = quant(i);
                        qb[i] = qv;
                        double xv = (double)xb[i];
                        double yv;
                        if (Tr::F) {
                            double y = __ddiv_rn((double)(long long)qv, deq_s);
                            yv = (DT == 3 || DT == 6) ? (double)__double2float_rn(y) : y;
                        } else {
                            long long yi = (deq_a == 1.0) ? (long long)qv
                                                          : f2i64(rint(__ddiv_rn((double)(long long)qv, deq_a)));
                            const long long lo = DT == 5 ? P.clip_lo : Tr::LO, hi = DT == 5 ? P.clip_hi : Tr::HI;
                            yi = yi < lo ? lo : (yi > hi ? hi : yi);
                            yv = (double)yi;
                        }
                        double d = xv - yv;
                        return d * d;
                    }, n, S, LL);
                    if (tid == 0) S->pd = pd;
                } else {
                    for (int i = tid; i < n; i += kNT) qb[i] = quant(i);
                }
                for (int i = n + tid; i < np; i += kNT) qb[i] = (Q)0;
                if (!Tr::F) { __syncthreads(); break; }
                // float: max |q| guard
                qmax = warp_allreduce(qmax, MaxOp());
                if ((tid & 31) == 0) S->red_d[2 * kWarps + (tid >> 5)] = qmax;
                __syncthreads();
                int retry = 0;
                if (tid == 0) {
                    double m = 0.0;
                    bool nan = false;
                    for (int w = 0; w < kWarps; w++) {
                        double v = S->red_d[2 * kWarps + w];
                        if (v != v || v == INFINITY) nan = true;
                        m = v > m ? v : m;
                    }
                    bool ok = (!nan && m < 2147483648.0) || S->fbe <= -127 || zero;
                    if (!ok) {
                        S->fbe -= 1;
                        S->s = decode_scale_code(S->code) * ldexp(1.0, S->fbe);
                        retry = 1;
                    }
                    S->red_u[0] = retry;
                }
                __syncthreads();
                retry = S->red_u[0];
                __syncthreads();
                if (!retry) break;
            }
            // ---- phase C: streams, exponents, costs, monitor ----
            {
                const long long hp1 = S->p1, hp2 = S->p2;
                long long se0 = 0, se1 = 0, se2 = 0;
                int emax = 0;
                Mon mon = {0, 0, 0, 0};
                const int g0 = tid * gpt;
                const int g1 = (g0 + gpt < G) ? g0 + gpt : G;
                for (int g = g0; g < g1; g++) {
                    int w0 = 0, w1 = 0, w2 = 0;
                    const int i0 = 4 * g;
                    long long qm1 = i0 >= 1 ? (long long)qb[i0 - 1] : hp1;
                    long long qm2 = i0 >= 2 ? (long long)qb[i0 - 2] : (i0 == 1 ? hp1 : hp2);
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        long long qv = (long long)qb[i0 + k];
                        // monitor
                        int sg = (qv > 0) - (qv < 0);
                        if (sg) {
                            if (mon.nnz == 0) mon.first = sg;
                            else if (sg != mon.last) mon.changes++;
                            mon.last = sg;
                            mon.nnz++;
                        }
                        if (Tr::WIDE) {
                            unsigned long long d1 = (unsigned long long)qv - (unsigned long long)qm1;
                            unsigned long long d1p = (unsigned long long)qm1 - (unsigned long long)qm2;
                            long long d2 = (long long)(d1 - d1p);
                            int a0 = width64(qv), a1 = width64((long long)d1), a2 = width64(d2);
                            w0 = a0 > w0 ? a0 : w0; w1 = a1 > w1 ? a1 : w1; w2 = a2 > w2 ? a2 : w2;
                        } else {
                            int q32 = (int)qv, m1 = (int)qm1, m2 = (int)qm2;
                            int d1 = q32 - m1, d2 = d1 - (m1 - m2);
                            int a0 = width32(q32), a1 = width32(d1), a2 = width32(d2);
                            w0 = a0 > w0 ? a0 : w0; w1 = a1 > w1 ? a1 : w1; w2 = a2 > w2 ? a2 : w2;
                        }
                        qm2 = qm1;
                        qm1 = qv;
                    }
                    int wm = w0 > w1 ? w0 : w1;
                    wm = wm > w2 ? wm : w2;
                    emax = wm > emax ? wm : emax;
                    es[g] = (uint8_t)(w0 > 255 ? 255 : w0);
                    es[Gfull + g] = (uint8_t)(w1 > 255 ? 255 : w1);
                    es[2 * Gfull + g] = (uint8_t)(w2 > 255 ? 255 : w2);
                    se0 += w0; se1 += w1; se2 += w2;
                }
                // CTA reductions: sums, emax, ordered monitor
                se0 = warp_allreduce(se0, SumOp());
                se1 = warp_allreduce(se1, SumOp());
                se2 = warp_allreduce(se2, SumOp());
                emax = warp_allreduce(emax, MaxOp());
                // ordered monitor within warp (lane order)
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    Mon oth;
                    oth.first = __shfl_down_sync(0xffffffffu, mon.first, o);
                    oth.last = __shfl_down_sync(0xffffffffu, mon.last, o);
                    oth.changes = __shfl_down_sync(0xffffffffu, mon.changes, o);
                    oth.nnz = __shfl_down_sync(0xffffffffu, mon.nnz, o);
                    if (((tid & 31) & (2 * o - 1)) == 0 && (tid & 31) + o < 32) mon = mon_combine(mon, oth);
                }
                const int warp = tid >> 5;
                if ((tid & 31) == 0) {
                    S->red_l[warp] = se0;
                    S->red_l[kWarps + warp] = se1;
                    S->red_l[2 * kWarps + warp] = se2;
                    S->red_u[warp] = (unsigned)emax;
                    S->red_l[3 * kWarps + warp] = ((long long)mon.changes << 32) | (unsigned)mon.nnz;
                    S->red_d[warp] = (double)(mon.first + 2) + 4.0 * (double)(mon.last + 2);
                }
                __syncthreads();
                if (tid == 0) {
                    long long t0 = 0, t1 = 0, t2 = 0;
                    int em = 0;
                    Mon m = {0, 0, 0, 0};
                    for (int w = 0; w < kWarps; w++) {
                        t0 += S->red_l[w]; t1 += S->red_l[kWarps + w]; t2 += S->red_l[2 * kWarps + w];
                        em = (int)S->red_u[w] > em ? (int)S->red_u[w] : em;
                        Mon o;
                        long long cn = S->red_l[3 * kWarps + w];
                        o.changes = (int)(cn >> 32);
                        o.nnz = (int)(cn & 0xffffffff);
                        int fl = (int)S->red_d[w];
                        o.first = (fl & 3) - 2;
                        o.last = ((fl >> 2) & 7) - 2;
                        m = mon_combine(m, o);
                    }
                    S->sum_e[0] = t0; S->sum_e[1] = t1; S->sum_e[2] = t2;
                    if (em > kMaxExponent && !S->bad) S->bad = APAX_ERR_INTERNAL;
                    // centre-frequency gate: cf = changes / (2 (np-1)) > 1/3
                    double cf = 0.0;
                    if (np > 1 && m.nnz > 1) cf = (double)m.changes / (2.0 * (double)(np - 1));
                    S->gate = cf > 1.0 / 3.0;
                }
                __syncthreads();
            }
        };

        // select_stream (transform.py:107-113) + state update after a block
        auto select_and_costs = [&]() {
            if (tid == 0) {
                int sel;
                if (!S->has_pc) sel = 0;
                else if (S->gate) sel = 0;
                else {
                    sel = 0;
                    if (S->pc[1] < S->pc[sel]) sel = 1;
                    if (S->pc[2] < S->pc[sel]) sel = 2;
                }
                S->sel = sel;
            }
        };

        // ---------------- unit prologue (halo / warm_self) ----------------
        if (P.halo && b0 > 0) {
            // lossless: rebuild the CodecState entering block b0 (App. C E2)
            const long long pb = b0 - 1;
            if (tid == 0) {
                if (pb >= 1) {
                    const T* xs = (const T*)P.x + pb * (long long)bs;
                    S->p1 = (long long)xs[-1];
                    S->p2 = (long long)xs[-2];
                } else { S->p1 = 0; S->p2 = 0; }
            }
            load_block(pb, bs);
            __syncthreads();
            analyze(pb, bs, 1.0, false);
            if (tid == 0) {
                S->has_pc = 1;
                for (int k = 0; k < 3; k++) S->pc[k] = 4 * S->sum_e[k] + 4 * (long long)Gfull;
                S->p1 = (long long)qb[bs - 1];
                S->p2 = (long long)qb[bs - 2];
                S->emitted = 1;
                S->initialized = 1;
                if (S->bad) report_error(P.status, pb, S->bad);
            }
            __syncthreads();
        } else if (P.policy == 1 && P.mode == 1) {
            // warm_self
            const int n0 = (int)((P.n - b0 * bs) < bs ? (P.n - b0 * bs) : bs);
            const int G0 = (n0 + 3) >> 2;
            load_block(b0, n0);
            __syncthreads();
            analyze(b0, n0, 1.0, false);
            if (tid == 0) {
                // the cost pass at gain 1 can fail on its own (widened samples
                // beyond 34 bits): the preset pass below starts a new status
                if (S->bad) report_error(P.status, b0, S->bad);
                long long c0 = 4 * S->sum_e[0] + 4 * (long long)G0;
                long long c1 = 4 * S->sum_e[1] + 4 * (long long)G0;
                long long c2 = 4 * S->sum_e[2] + 4 * (long long)G0;
                long long mn = c0 < c1 ? c0 : c1;
                mn = c2 < mn ? c2 : mn;
                double bps0 = (double)(mn + 8LL * hs) / (double)bs;
                double att0 = 0.0 - 6.02 * (bps0 - P.target);
                double mm = (P.att_lo > att0) ? P.att_lo : att0;
                S->att = (0.0 < mm) ? 0.0 : mm;
                double p = pow(10.0, S->att / 20.0);
                double m2 = (4.656612873077393e-10 > p) ? 4.656612873077393e-10 : p;
                S->a = (1.0 < m2) ? 1.0 : m2;
                S->p1 = 0; S->p2 = 0;
            }
            __syncthreads();
            analyze(b0, n0, S->a, false);
            if (tid == 0) {
                S->has_pc = 1;
                for (int k = 0; k < 3; k++) S->pc[k] = 4 * S->sum_e[k] + 4 * (long long)G0;
                S->p1 = 0; S->p2 = 0;
                if (S->bad) report_error(P.status, b0, S->bad);
            }
            __syncthreads();
        }

        // ---------------- blocks of the unit ----------------
        for (long long b = b0; b < b1; b++) {
            const int n = (int)((P.n - b * bs) < bs ? (P.n - b * bs) : bs);
            const int G = (n + 3) >> 2;
            const int np = 4 * G;
            load_block(b, n);
            __syncthreads();
            analyze(b, n, -1.0, true);
            select_and_costs();
            __syncthreads();
            const int sel = S->sel;
            const uint8_t* e = es + sel * Gfull;
            // ---- phase D: JEE automaton + mantissa bits scan ----
            const int g0 = tid * gpt;
            const int g1 = (g0 + gpt < G) ? g0 + gpt : G;
            uint32_t f = kJfIdentity;
            unsigned mbits = 0;
            if (g0 < g1) {
                int o0, n0, o1, n1;
                jee_local(e, g0, g1, G, 0, o0, n0);
                jee_local(e, g0, g1, G, 1, o1, n1);
                f = jf_pack(o0, o1, n0, n1);
                for (int g = g0; g < g1; g++) mbits += 4u * e[g];
            }
            uint32_t fx;
            unsigned bx;
            cta_scan_jee(f, mbits, fx, bx, S);
            // block size and staging-window capacity
            if (tid == 0) {
                long long jee_bytes = (S->nib_total + 1) >> 1;
                long long mant_bytes = (S->bits_total + 7) >> 3;
                // a block in error emits its header only: its widths (up to 64
                // bits for samples outside the 34-bit range) say nothing about
                // the window, which is sized for legal blocks
                S->block_bytes = S->bad ? hs : hs + jee_bytes + mant_bytes;
                if (S->staged + S->block_bytes + 4 > (long long)P.stage_bytes) S->red_u[0] = 1;
                else S->red_u[0] = 0;
            }
            __syncthreads();
            if (S->red_u[0]) {
                // flush whole words of the window to the unit's slot (or to
                // the final output when the unit's offset is already known)
                const long long whole = S->staged & ~3LL;
                uint8_t* dst = S->direct ? (P.out + kFileHeader + S->win_base) : (slot + S->win_base);
                copy_out<true>(dst, stage, whole);
                __syncthreads();
                const int rem = (int)(S->staged & 3);
                uint32_t keep = stage[whole >> 2];
                __syncthreads();
                for (int i = tid; i < stage_words + 4; i += kNT) stage[i] = 0u;
                __syncthreads();
                if (tid == 0) {
                    if (rem) stage[0] = keep;
                    S->win_base += whole;
                    S->staged = rem;
                }
                __syncthreads();
            }
            // ---- write header, JEE nibbles, mantissa into the window ----
            const long long bstart = S->staged;  // window byte offset of this block
            const long long jee_bytes = (S->nib_total + 1) >> 1;
            if (g0 < g1 && !S->bad) {
                // JEE nibbles
                int state = (fx >> 0) & 1;         // exclusive prefix applied to S
                int nib0 = (fx >> 2) & 0x7fff;
                BitWriter bw;
                bw.init(stage, 8 * (bstart + hs) + 4LL * nib0);
                for (int i = g0; i < g1; i++) {
                    if (state) { state = 0; continue; }
                    int kind = jee_kind(e, i, G);
                    if (kind == 0) {
                        int d1 = (int)e[i] - (int)e[i - 1];
                        int d2 = (int)e[i + 1] - (int)e[i];
                        bw.put32((uint32_t)((d1 + 1) * 3 + (d2 + 1)), 4);
                        state = 1;
                    } else if (kind == 1) {
                        int d = (int)e[i] - (int)e[i - 1];
                        bw.put32((uint32_t)(11 + d), 4);
                    } else {
                        bw.put32(0xF00u | (uint32_t)e[i], 12);
                    }
                }
                bw.flush();
                // mantissa bits of the selected stream
                BitWriter mw;
                mw.init(stage, 8 * (bstart + hs + jee_bytes) + (long long)bx);
                const long long hp1 = S->p1, hp2 = S->p2;
                for (int g = g0; g < g1; g++) {
                    const int w = e[g];
                    if (!w) continue;
                    const int i0 = 4 * g;
                    long long qm1 = i0 >= 1 ? (long long)qb[i0 - 1] : hp1;
                    long long qm2 = i0 >= 2 ? (long long)qb[i0 - 2] : (i0 == 1 ? hp1 : hp2);
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        long long qv = (long long)qb[i0 + k];
                        unsigned long long v;
                        if (sel == 0) v = (unsigned long long)qv;
                        else if (sel == 1) v = (unsigned long long)qv - (unsigned long long)qm1;
                        else v = ((unsigned long long)qv - (unsigned long long)qm1) -
                                 ((unsigned long long)qm1 - (unsigned long long)qm2);
                        mw.put(v, w);
                        qm2 = qm1;
                        qm1 = qv;
                    }
                }
                mw.flush();
            }
            __syncthreads();
            if (tid == 0) {
                // block header (dtypes.py:156-165)
                const int restart = (S->emitted == 0);
                const int code = S->code;
                uint32_t hb[6];
                hb[0] = (uint32_t)((sel & 3) | (restart ? 4 : 0));
                hb[1] = (uint32_t)(code & 0xFF);
                hb[2] = (uint32_t)((code >> 8) & 0xFF);
                hb[3] = 0;
                hb[4] = (uint32_t)(uint8_t)(int8_t)S->fbe;
                hb[5] = 0;
                for (int k = 0; k < hs; k++) {
                    long long bp = bstart + k;
                    atomicOr(&stage[bp >> 2], hb[k] << (8 * (bp & 3)));
                }
                if (P.block_offsets) P.block_offsets[b] = S->win_base + bstart;  // unit-relative
                if (P.trace) {
                    double* tr = P.trace + 10 * b;
                    tr[0] = S->att; tr[1] = S->a; tr[2] = code; tr[3] = S->fbe; tr[4] = sel;
                    tr[5] = (double)(4 * S->sum_e[0] + 4LL * G); tr[6] = (double)(4 * S->sum_e[1] + 4LL * G);
                    tr[7] = (double)(4 * S->sum_e[2] + 4LL * G); tr[8] = (double)S->block_bytes;
                    tr[9] = restart;
                }
                if (S->bad) report_error(P.status, b, S->bad);
                // state update (codec.py:220-221, 228-254)
                S->has_pc = 1;
                for (int k = 0; k < 3; k++) S->pc[k] = 4 * S->sum_e[k] + 4LL * G;
                S->p2 = (long long)qb[np - 2];
                S->p1 = (long long)qb[np - 1];
                if (P.mode == 1) {
                    long long actual_bits = S->block_bytes * 8;
                    if (S->emitted == 0) {
                        long long mn = S->pc[0] < S->pc[1] ? S->pc[0] : S->pc[1];
                        mn = S->pc[2] < mn ? S->pc[2] : mn;
                        long long est_bits = mn + 8LL * hs;
                        double bps0 = (double)est_bits / (double)bs;
                        double att = S->att - 6.02 * (bps0 - P.target);
                        double mm = (P.att_lo > att) ? P.att_lo : att;
                        S->att = (0.0 < mm) ? 0.0 : mm;
                    } else {
                        double err = (double)actual_bits / (double)bs - P.target;
                        double d = 0.75 * err;
                        double m = (d < 6.0) ? d : 6.0;
                        double step = (m > -6.0) ? m : -6.0;
                        double att = S->att - step;
                        double mm = (P.att_lo > att) ? P.att_lo : att;
                        S->att = (0.0 < mm) ? 0.0 : mm;
                    }
                } else if (P.mode == 2) {
                    double px = S->px / (double)n, pd = S->pd / (double)n;
                    // math.log10 of a ratio that underflowed (or of px / inf) raises
                    if (px > 0.0 && pd != 0.0 && px / pd == 0.0) report_error(P.status, b, APAX_ERR_MATH_DOMAIN);
                    if (px > 0.0) {
                        double measured = (pd == 0.0) ? INFINITY : 10.0 * log10(px / pd);
                        if (isfinite(measured)) {
                            double d = 0.5 * (measured - P.target);
                            double m = (d < 6.0) ? d : 6.0;
                            double delta = (m > -6.0) ? m : -6.0;
                            double att = S->att - delta;
                            double mm = (P.att_lo > att) ? P.att_lo : att;
                            S->att = (0.0 < mm) ? 0.0 : mm;
                        }
                    }
                }
                S->emitted += 1;
                S->staged += S->block_bytes;
                S->unit_len += S->block_bytes;
            }
            __syncthreads();
        }

        if (P.state && tid == 0) {   // the state after the block
            apax_block_state* cs = P.state;
            cs->att_db = S->att; cs->prev1 = S->p1; cs->prev2 = S->p2;
            cs->has_costs = S->has_pc;
            cs->costs[0] = S->pc[0]; cs->costs[1] = S->pc[1]; cs->costs[2] = S->pc[2];
            cs->initialized = S->initialized;
            cs->blocks_emitted = S->emitted;
        }
        // ---------------- placement: decoupled look-back ----------------
        if (tid < 32) {
            const long long L = S->unit_len;
            const long long prefix = warp_lookback(P.lookback, u, L);
            if (tid == 0) {
                S->prefix = prefix;
                if (u == P.n_units - 1) {
                    P.status[2] = (unsigned long long)(kFileHeader + prefix + L);
                    if (P.block_offsets) P.block_offsets[P.n_blocks] = kFileHeader + prefix + L;
                }
            }
        }
        __syncthreads();
        const long long prefix = S->prefix;
        uint8_t* dst = P.out + kFileHeader + prefix;
        const long long total = S->unit_len;
        if (total + kFileHeader + prefix > P.out_cap) {
            if (tid == 0) report_error(P.status, b0, APAX_ERR_CAPACITY);
        } else {
            // earlier window flushes (in the slot unless direct)
            if (!S->direct && S->win_base > 0) {
                copy_out<false>(dst, (const uint32_t*)slot, S->win_base);
            }
            copy_out<true>(dst + S->win_base, stage, S->staged);
            if (u == 0 && tid < kFileHeader) {
                // file header "<4sBBBBIQd" (codec.py:277-279)
                unsigned char h[kFileHeader];
                h[0] = 'A'; h[1] = 'P'; h[2] = 'A'; h[3] = 'X';
                h[4] = 1; h[5] = (unsigned char)(DT >= 5 ? P.wire : DT); h[6] = (unsigned char)P.mode; h[7] = 0;
                unsigned bsz = (unsigned)bs;
                for (int k = 0; k < 4; k++) h[8 + k] = (unsigned char)(bsz >> (8 * k));
                unsigned long long cnt = (unsigned long long)P.n;
                for (int k = 0; k < 8; k++) h[12 + k] = (unsigned char)(cnt >> (8 * k));
                unsigned long long tb = (unsigned long long)__double_as_longlong(P.target);
                for (int k = 0; k < 8; k++) h[20 + k] = (unsigned char)(tb >> (8 * k));
                P.out[tid] = h[tid];
            }
        }
        if (P.block_offsets) {
            for (long long b = b0 + tid; b < b1; b += kNT) P.block_offsets[b] += kFileHeader + prefix;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// host-side launch helper
// ---------------------------------------------------------------------------
size_t encode_smem_bytes(int dt, int bs, int stage_bytes, int x_in_smem) {
    auto al = [](size_t v) { return (v + 15) & ~(size_t)15; };
    size_t w = (size_t)dt_width(dt);
    size_t qw = dt_width(dt) == 8 ? 8 : 4;
    return al(sizeof(EncState)) + al(sizeof(LeafList)) + (x_in_smem ? al((size_t)bs * w) : 0) +
           al((size_t)(bs + 4) * qw) + al((size_t)3 * (bs / 4) + 16) + (size_t)stage_bytes + 16;
}

template <int DT>
static int launch_encode_t(const EncParams& P, int grid, size_t smem, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(encode_kernel<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return APAX_ERR_CUDA;
    note_launches(1);
    encode_kernel<DT><<<grid, kNT, smem, st>>>(P);
    return cudaGetLastError() == cudaSuccess ? APAX_OK : APAX_ERR_CUDA;
}

template <int DT>
static int resident_t(size_t smem) {
    int per = 0;
    cudaFuncSetAttribute(encode_kernel<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, encode_kernel<DT>, kNT, smem) != cudaSuccess) per = 1;
    return per;
}

int encode_resident_ctas(int dt, size_t smem) {
    int dev = 0, nsm = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    switch (dt) {
        case 0: per = resident_t<0>(smem); break;
        case 1: per = resident_t<1>(smem); break;
        case 2: per = resident_t<2>(smem); break;
        case 3: per = resident_t<3>(smem); break;
        case 4: per = resident_t<4>(smem); break;
        case 5: per = resident_t<5>(smem); break;
        default: per = resident_t<6>(smem); break;
    }
    if (per < 1) per = 1;
    return per * (nsm > 0 ? nsm : 148);
}

int launch_encode(int dt, const EncParams& P, int grid, size_t smem, cudaStream_t st) {
    switch (dt) {
        case 0: return launch_encode_t<0>(P, grid, smem, st);
        case 1: return launch_encode_t<1>(P, grid, smem, st);
        case 2: return launch_encode_t<2>(P, grid, smem, st);
        case 3: return launch_encode_t<3>(P, grid, smem, st);
        case 4: return launch_encode_t<4>(P, grid, smem, st);
        case kKdtI64: return launch_encode_t<kKdtI64>(P, grid, smem, st);
        case kKdtF64F32: return launch_encode_t<kKdtF64F32>(P, grid, smem, st);
    }
    return APAX_ERR_ARG;
}

}  // namespace apax
