// apax_encode_v2.cu -- instruction-lean B200 encoder for block sizes
// 128..4096 (powers of two): the hot path of every BASELINE config.
//
// Same contract and byte-exact output as apax_encode.cu (reference
// encode_stream, pkg/src/apax/codec.py:258-285 / encode_block :192-255); the
// v1 kernel remains the general path (any block size 64..16384).
//
// Per CTA (256 threads, persistent, round-robin units of consecutive blocks):
//   * TMA bulk copies (cp.async.bulk + mbarrier) double-buffer the next
//     block's samples into shared memory while the current one is coded;
//   * phase A  block peak (|x| bit-max) and, for fixed quality, numpy's
//              pairwise sum of x^2 (8 lanes per 128-sample leaf, exactly the
//              association tree of np.add.reduce; codec.py:159,248);
//   * scalar   thread 0: gain / scale code / float block exponent.  max|q|
//              equals rint(peak*s) exactly, so the overflow-retry loop of
//              codec.py:126-131 runs on scalars only;
//   * phase B  fixed quality: quantize + dequantize (Markstein quotient with a
//              per-block reciprocal, bit-identical to IEEE division) + the
//              pairwise residual power; other modes quantize in phase C;
//   * phase C  16 contiguous samples per thread in registers: d1/d2
//              (transform.py:86-91), group widths via bit_length((v<<1)^v)
//              OR-accumulated per group (= entropy.py:38-55), the three costs
//              (transform.py:94-97) and the ordered sign-change monitor
//              (transform.py:67-83);
//   * phase D  JEE greedy pairing as a CTA scan of 2-state transfer
//              functions (entropy.py:63-88) fused with the mantissa bit
//              offsets; MSB-first packing into a shared-memory window
//              (entropy.py:194-240); whole 16-byte chunks are flushed after
//              every block, so the window only holds one block plus a tail;
//   * placement  decoupled look-back over unit byte lengths, then the unit's
//              bytes move from its scratch slot to their final offset.
// Blocks whose streams need 64-bit differences (max|q| >= 2^29) take a
// recomputing 64-bit path; f64 blocks whose quantized samples leave int32
// (|x| >= ~2^188) are handled there too.
#include <cstdint>
#include <cuda_runtime.h>

#include "apax_device.cuh"
#include "apax_kernels.cuh"

#ifndef APAX_ENC_MINB
#define APAX_ENC_MINB 4
#endif

namespace apax {
namespace v2 {

constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int SPT = 16;          // samples per thread in the contiguous mapping
constexpr int MAXBS = 4096;
constexpr int LEAF_STRIDE = 136; // padded 128-sample leaf in qbuf (bank spread)

struct St {
    // CodecState (codec.py:66-82)
    double att;
    long long p1, p2;
    long long pc[3];
    long long emitted;
    int has_pc, initialized;
    // per-block broadcast
    double a, s, rs, aq, ra, px, pd, peak_d;
    long long qpk;
    int code, fbe, sel, wide, zero, gate, bad, nonfinite;
    long long sum_e[3];
    long long blen, jee_nib, bits;
    long long last1, last2;     // q[np-1], q[np-2] of the block
    // window / slot
    long long win_base;
    int tail_len;
    uint32_t tail[4];
    long long unit_len, unit, prefix;
    int direct;
    // reductions
    double pxw[NW], pdw[NW];
    unsigned long long pkw[NW];
    int sew[3][NW];
    int monc[NW], monf[NW];
    unsigned emaxw[NW];
    int exact_mon;
    uint32_t edge_first[NW], edge_last[NW];   // per stream first/last group width of each warp
    uint32_t pw[32], ew[32], tw[32], xw[32], jw[32];
    int nibpre[32];
    unsigned mbw[NW], mbpre[NW];
    unsigned long long mbar[2];
    // deferred placement of the previous unit (look-back + copy-out)
    long long pend_u, pend_len, pend_b0, pend_b1, pend_k, pend_acc, pend_prefix;
    int pend_slot, pend_ready;
};

using namespace apax::tma;

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ int bitlen32(unsigned v) { return 32 - __clz((int)v); }
__device__ __forceinline__ int bitlen64(unsigned long long v) { return 64 - __clzll((long long)v); }
__device__ __forceinline__ unsigned wbits32(int v) { return (unsigned)((v << 1) ^ v); }
__device__ __forceinline__ unsigned long long wbits64(long long v) {
    return (unsigned long long)((v << 1) ^ v);
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

// JEE transfer functions (see apax_encode.cu): bit0 out(S), bit1 out(C),
// bits 2..16 nibbles from S, 17..31 nibbles from C
__device__ __forceinline__ uint32_t jf_pack(int o0, int o1, int n0, int n1) {
    return (uint32_t)o0 | ((uint32_t)o1 << 1) | ((uint32_t)n0 << 2) | ((uint32_t)n1 << 17);
}
__device__ __forceinline__ uint32_t jf_compose(uint32_t a, uint32_t b) {  // a then b
    uint32_t ao0 = a & 1u, ao1 = (a >> 1) & 1u;
    uint32_t bo0 = b & 1u, bo1 = (b >> 1) & 1u;
    uint32_t bn0 = (b >> 2) & 0x7fffu, bn1 = (b >> 17) & 0x7fffu;
    uint32_t r_o0 = ao0 ? bo1 : bo0, r_o1 = ao1 ? bo1 : bo0;
    uint32_t r_n0 = ((a >> 2) & 0x7fffu) + (ao0 ? bn1 : bn0);
    uint32_t r_n1 = ((a >> 17) & 0x7fffu) + (ao1 ? bn1 : bn0);
    return r_o0 | (r_o1 << 1) | (r_n0 << 2) | (r_n1 << 17);
}
constexpr uint32_t kJfId = 2u;  // out(S)=S(0), out(C)=C(1), 0 nibbles

// generic pairwise sum (numpy), sequential on one thread, term(i) on the fly.
// Iterative (explicit stack) so no device recursion / stack frames are needed.
template <typename F>
__device__ double pw_leaf(F& term, int s, int n) {
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
__device__ double pw_seq(F& term, int s0, int n0) {
    // frames: (start, len, stage, left partial)
    int fs[16], fn[16], fst[16];
    double fl[16];
    int sp = 0;
    fs[0] = s0; fn[0] = n0; fst[0] = 0; sp = 1;
    double val = 0.0;
    bool have = false;
    while (sp > 0) {
        const int t = sp - 1;
        if (have) {               // deliver val to frame t
            if (fst[t] == 1) {    // left done -> start right
                fl[t] = val;
                fst[t] = 2;
                int n2 = fn[t] / 2;
                n2 -= n2 % 8;
                fs[sp] = fs[t] + n2; fn[sp] = fn[t] - n2; fst[sp] = 0; sp++;
                have = false;
            } else {              // right done
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
        // descend left
        fst[t] = 1;
        int n2 = fn[t] / 2;
        n2 -= n2 % 8;
        fs[sp] = fs[t]; fn[sp] = n2; fst[sp] = 0; sp++;
    }
    return val;
}

__device__ __forceinline__ int qaddr(int i) { return (i >> 7) * LEAF_STRIDE + (i & 127); }

// ---------------------------------------------------------------------------
// 32-position JEE words: C[i+1] = P[i] & ~C[i] (a position following a joint
// token is consumed), solved with the odd-run carry trick (the escape-scanner
// identity popularised by simdjson).  Returns consumed mask, *cout = C[32].
// ---------------------------------------------------------------------------
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

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <int DT>
__global__ void __launch_bounds__(NT, APAX_ENC_MINB) encode_v2_kernel(EncParams P) {
    using Tr = DT_<DT>;
    using T = typename Tr::T;
    constexpr bool F = Tr::F;
    constexpr int HS = Tr::HDR;
    // x^2 is exact in double for 8/16-bit ints and f32
    constexpr bool SQ_EXACT = (DT == 0 || DT == 1 || DT == 3);

    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bs = P.bs;
    const bool FQ = (P.mode == 2);

    St* S = (St*)smem;
    size_t off = (sizeof(St) + 127) & ~(size_t)127;
    T* xbuf[2];
    xbuf[0] = (T*)(smem + off);
    off += ((size_t)MAXBS * sizeof(T) + 127) & ~(size_t)127;
    xbuf[1] = (T*)(smem + off);
    off += ((size_t)MAXBS * sizeof(T) + 127) & ~(size_t)127;
    uint32_t* win = (uint32_t*)(smem + off);
    const int win_words = P.stage_bytes / 4;

    uint8_t* slots2[2];
    slots2[0] = P.slots + (long long)blockIdx.x * 2 * P.slot_bytes;
    slots2[1] = slots2[0] + P.slot_bytes;
    int cur_slot = 0;
    uint8_t* slot = slots2[0];

    if (tid == 0) {
        mbar_init(&S->mbar[0]);
        mbar_init(&S->mbar[1]);
        fence_mbar_init();
        S->pend_u = -1;
        S->pend_ready = 0;
    }
    __syncthreads();
    uint32_t phase[2] = {0u, 0u};

    // ---- deferred placement helpers ----
    // one look-back window (32 predecessors) for the pending unit; warp 0.
    auto lookback_try = [&](bool blocking) {
        if (S->pend_u < 0 || S->pend_ready) return;
        for (;;) {
            const long long kq = S->pend_k;
            const long long idx = kq - lane;
            unsigned long long vq = (idx >= 0) ? ld_acquire(&P.lookback[idx]) : kFlagInc;
            const unsigned long long fl = vq & ~kValMask;
            const unsigned inc = __ballot_sync(0xffffffffu, fl == kFlagInc);
            const unsigned nrd = __ballot_sync(0xffffffffu, fl == 0);
            const int first_inc = inc ? __ffs(inc) - 1 : 32;
            const int first_nrd = nrd ? __ffs(nrd) - 1 : 32;
            // consume the ready prefix of the window (up to the first INC)
            const int upto = first_inc < first_nrd ? first_inc : first_nrd - 1;  // inclusive
            unsigned long long part = (lane <= upto) ? (vq & kValMask) : 0ULL;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            __syncwarp();
            if (lane == 0) {
                S->pend_acc += (long long)part;
                S->pend_k -= (upto + 1);
            }
            __syncwarp();
            if (first_inc < first_nrd) {  // resolved
                if (lane == 0) {
                    const long long prefix = S->pend_acc;
                    st_release(&P.lookback[S->pend_u], kFlagInc | (unsigned long long)(prefix + S->pend_len));
                    S->pend_prefix = prefix;
                    S->pend_ready = 1;
                    if (S->pend_u == P.n_units - 1) {
                        P.status[2] = (unsigned long long)(kFileHeader + prefix + S->pend_len);
                        if (P.block_offsets) P.block_offsets[P.n_blocks] = kFileHeader + prefix + S->pend_len;
                    }
                }
                __syncwarp();
                return;
            }
            if (!blocking) return;
            if (first_nrd < 32) __nanosleep(64);
        }
    };
    // copy the resolved pending unit to its final place (all threads)
    auto place_pending = [&]() {
        const long long prefix = S->pend_prefix;
        copy_out<false>(P.out + kFileHeader + prefix, (const uint32_t*)slots2[S->pend_slot], S->pend_len);
        if (P.block_offsets)
            for (long long bb = S->pend_b0 + tid; bb < S->pend_b1; bb += NT) P.block_offsets[bb] += kFileHeader + prefix;
        __syncthreads();
        if (tid == 0) { S->pend_u = -1; S->pend_ready = 0; }
        __syncthreads();
    };

    auto block_n = [&](long long b) -> int {
        long long r = P.n - b * (long long)bs;
        return (int)(r < bs ? r : bs);
    };
    auto tma_ok = [&](long long b) -> bool {
        const T* src = (const T*)P.x + b * (long long)bs;
        long long bytes = (long long)block_n(b) * (long long)sizeof(T);
        return ((((uintptr_t)src) & 15) == 0) && ((bytes & 15) == 0);
    };
    auto first_block = [&](long long uu) -> long long {
        const long long bb = uu * P.unit_blocks;
        return (P.halo && bb > 0) ? bb - 1 : bb;
    };
    long long loaded_b = -1, inflight_b = -1;
    int cur = 0, inflight_buf = 0;
    // units are assigned round-robin; the launch is cooperative, so every
    // unit's predecessor is on a co-resident CTA (look-back cannot deadlock)
    for (long long u = blockIdx.x; u < P.n_units; u += gridDim.x) {
        const long long b0 = u * P.unit_blocks;
        const long long b1 = (b0 + P.unit_blocks < P.n_blocks) ? b0 + P.unit_blocks : P.n_blocks;
        if (tid == 0) {
            S->att = 0.0; S->p1 = 0; S->p2 = 0; S->has_pc = 0; S->initialized = 0;
            S->emitted = 0; S->win_base = 0; S->tail_len = 0; S->unit_len = 0;
            S->tail[0] = S->tail[1] = S->tail[2] = S->tail[3] = 0u;
            S->direct = (u == 0);
            S->prefix = 0;
            if (P.halo && b0 > 1) {  // history entering block b0-1 (App. C E2)
                const T* xh = (const T*)P.x + (b0 - 1) * (long long)bs;
                S->p1 = (long long)xh[-1];
                S->p2 = (long long)xh[-2];
            }
        }
        // pass list: [halo] | [warm1, warm2] then the unit's blocks
        const bool halo = P.halo && b0 > 0;
        const bool warm = !P.halo && P.policy == 1 && P.mode == 1;
        const int npre = halo ? 1 : (warm ? 2 : 0);
        const long long npass = npre + (b1 - b0);
        auto pass_block = [&](long long k) -> long long {
            if (halo) return k == 0 ? b0 - 1 : b0 + k - 1;
            if (warm) return k < 2 ? b0 : b0 + k - 2;
            return b0 + k;
        };
        __syncthreads();
        {
            const long long bfirst = pass_block(0);
            if (bfirst != loaded_b && bfirst != inflight_b) {
                inflight_b = bfirst;
                inflight_buf = cur ^ 1;
                if (tma_ok(bfirst) && tid == 0) {
                    fence_proxy_async();
                    tma_load(xbuf[inflight_buf], (const T*)P.x + bfirst * (long long)bs,
                             (uint32_t)(block_n(bfirst) * sizeof(T)), &S->mbar[inflight_buf]);
                }
            }
        }

        for (long long k = 0; k < npass; k++) {
            const long long b = pass_block(k);
            // kind: 0 emit, 1 halo costs, 2 warm pass 1 (a = 1), 3 warm pass 2
            const int kind = halo ? (k == 0 ? 1 : 0) : (warm ? (k == 0 ? 2 : (k == 1 ? 3 : 0)) : 0);
            const int n = block_n(b);
            const int G = (n + 3) >> 2;
            const int np = 4 * G;
            // ---------------- block b's samples -> smem ----------------
            if (b != loaded_b) {
                if (inflight_b == b) {
                    cur = inflight_buf;
                    if (tma_ok(b)) {
                        mbar_wait(&S->mbar[cur], phase[cur]);
                        phase[cur] ^= 1u;
                    } else {
                        const T* src = (const T*)P.x + b * (long long)bs;
                        for (int i = tid; i < n; i += NT) xbuf[cur][i] = src[i];
                    }
                } else {
                    cur ^= 1;
                    const T* src = (const T*)P.x + b * (long long)bs;
                    for (int i = tid; i < n; i += NT) xbuf[cur][i] = src[i];
                }
                loaded_b = b;
                inflight_b = -1;
                long long nb = -1;
                for (long long kk = k + 1; kk < npass; kk++) {
                    long long bb = pass_block(kk);
                    if (bb != b) { nb = bb; break; }
                }
                if (nb < 0 && u + gridDim.x < P.n_units) {  // next unit's first block
                    const long long bb = first_block(u + gridDim.x);
                    if (bb != b) nb = bb;
                }
                __syncthreads();  // the other buffer's readers are done
                if (nb >= 0) {
                    inflight_b = nb;
                    inflight_buf = cur ^ 1;
                    if (tma_ok(nb) && tid == 0) {
                        fence_proxy_async();
                        tma_load(xbuf[inflight_buf], (const T*)P.x + nb * (long long)bs,
                                 (uint32_t)(block_n(nb) * sizeof(T)), &S->mbar[inflight_buf]);
                    }
                }
            }
            const T* xs = xbuf[cur];
            if (kind == 0) {  // window: carried tail + zeros
                uint4* w4 = (uint4*)win;
                for (int i = 1 + tid; i < win_words / 4 + 2; i += NT) w4[i] = make_uint4(0u, 0u, 0u, 0u);
                if (tid == 0) w4[0] = make_uint4(S->tail[0], S->tail[1], S->tail[2], S->tail[3]);
            }

            // ================= phase A: peak (+ px, fixed quality) =================
            const int leaf = warp * 4 + (lane >> 3);
            const int jj = lane & 7;
            const int L = n >> 7;                      // full 128-sample leaves
            const bool regular = (n == bs);            // bs is a power of two >= 128
            {
                unsigned long long pk = 0;             // max |x| (bit pattern for floats)
                double pxs = 0.0;
                auto absbits = [&](T v) -> unsigned long long {
                    if (DT == 3) return (unsigned)__float_as_uint((float)v) & 0x7fffffffu;
                    if (DT == 4) return (unsigned long long)__double_as_longlong((double)v) & 0x7fffffffffffffffULL;
                    long long iv = (long long)v;
                    return (unsigned long long)(iv < 0 ? -iv : iv);
                };
                if (FQ && regular) {
                    // pairwise x^2 over 8-lane leaves (numpy order) + peak
                    if (warp * 4 < L) {
                        double r = 0.0;
                        if (leaf < L) {
                            const int base = leaf * 128 + jj;
                            const T x0 = xs[base];
                            const double v = (double)x0;
                            r = v * v;
                            pk = absbits(x0);
#pragma unroll
                            for (int i = 1; i < 16; i++) {
                                const T xi = xs[base + 8 * i];
                                const double w = (double)xi;
                                if (SQ_EXACT) r = __fma_rn(w, w, r);
                                else r = r + w * w;
                                const unsigned long long ab = absbits(xi);
                                pk = ab > pk ? ab : pk;
                            }
                        }
                        r += __shfl_xor_sync(0xffffffffu, r, 1);
                        r += __shfl_xor_sync(0xffffffffu, r, 2);
                        r += __shfl_xor_sync(0xffffffffu, r, 4);
                        if (L >= 2) r += __shfl_xor_sync(0xffffffffu, r, 8);
                        if (L >= 4) r += __shfl_xor_sync(0xffffffffu, r, 16);
                        pxs = r;
                    }
                } else if (F || DT == 2 || FQ) {
                    // floats: scale from the peak; i32: 64-bit stream decision
                    if (DT == 3 && (n & 3) == 0) {
                        const uint4* x4 = (const uint4*)xs;
                        unsigned m = 0;
                        for (int i = tid; i < (n >> 2); i += NT) {
                            uint4 v = x4[i];
                            m = max(m, max(max(v.x & 0x7fffffffu, v.y & 0x7fffffffu),
                                           max(v.z & 0x7fffffffu, v.w & 0x7fffffffu)));
                        }
                        pk = m;
                    } else {
                        for (int i = tid; i < n; i += NT) {
                            const unsigned long long ab = absbits(xs[i]);
                            pk = ab > pk ? ab : pk;
                        }
                    }
                }
                unsigned long long pkr = pk;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    unsigned long long t = __shfl_xor_sync(0xffffffffu, pkr, o);
                    pkr = t > pkr ? t : pkr;
                }
                if (lane == 0) { S->pkw[warp] = pkr; S->pxw[warp] = pxs; }
            }
            __syncthreads();  // B1
            // ================= scalar: gain, code, scale (thread 0) =================
            if (tid == 0) {
                unsigned long long pk = 0;
                for (int w = 0; w < NW; w++) pk = S->pkw[w] > pk ? S->pkw[w] : pk;
                double px = 0.0;
                if (FQ) {
                    if (regular) {
                        const int nwd = (L + 3) / 4;
                        double v[NW];
                        for (int w = 0; w < nwd; w++) v[w] = S->pxw[w];
                        for (int st = 1; st < nwd; st <<= 1)
                            for (int w = 0; w + st < nwd; w += 2 * st) v[w] = v[w] + v[w + st];
                        px = v[0];
                    } else {
                        auto t2 = [&](int i) { double v = (double)xs[i]; return v * v; };
                        px = pw_seq(t2, 0, n);
                    }
                    S->px = px;
                }
                double peak;
                bool nonfin = false;
                if (F) {
                    if (DT == 3) {
                        nonfin = pk >= 0x7f800000ULL;
                        peak = (double)__uint_as_float((unsigned)pk);
                    } else {
                        nonfin = pk >= 0x7ff0000000000000ULL;
                        peak = __longlong_as_double((long long)pk);
                    }
                } else {
                    peak = (double)pk;
                }
                S->nonfinite = nonfin;
                if (nonfin) {
                    for (int i = 0; i < n; i++) {
                        if (!isfinite((double)xs[i])) {
                            atomicMin(&P.status[0], (unsigned long long)(b * (long long)bs + i));
                            break;
                        }
                    }
                }
                if (kind == 0 && !S->initialized) {
                    if (FQ) {  // _init_attenuation (codec.py:155-168)
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
                }
                double a;
                if (kind == 1 || kind == 2) a = 1.0;
                else if (kind == 3) a = S->a;
                else if (P.mode == 0) a = 1.0;
                else a = att_to_a(S->att);
                S->a = a;
                int bad = 0, zero = 0, fbe = 0, code;
                double s = 1.0, aq = 1.0;
                long long qpk;
                if (!F) {
                    code = encode_scale_code(a);
                    aq = decode_scale_code(code);
                    qpk = (aq == 1.0) ? (long long)peak : (long long)rint(peak * aq);
                } else if (nonfin || peak == 0.0) {
                    code = kScaleCodeOne; zero = 1; qpk = 0;
                } else {
                    double s_des = (a * 1073741824.0) / peak;
                    if (!isfinite(s_des)) {
                        bad = APAX_ERR_OVERFLOW; code = kScaleCodeOne; zero = 1; qpk = 0;
                    } else {
                        long long l2 = floor_log2_rn(s_des);
                        long long fb = (-31 <= l2 && l2 <= 31) ? 0 : l2 - 31;
                        fb = fb < -127 ? -127 : (fb > 127 ? 127 : fb);
                        double rem = ldexp(s_des, (int)-fb);
                        const double nxt = 8589934591.999999;
                        double mm = (nxt < rem) ? nxt : rem;
                        rem = (mm > 4.656612873077393e-10) ? mm : 4.656612873077393e-10;
                        code = encode_scale_code(rem);
                        // overflow guard (codec.py:126-131): max|q| = rint(peak*s)
                        for (;;) {
                            s = decode_scale_code(code) * ldexp(1.0, (int)fb);
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
                S->code = code; S->fbe = fbe; S->s = s; S->aq = aq; S->zero = zero;
                S->rs = F ? __ddiv_rn(1.0, s) : (aq == 1.0 ? 1.0 : __ddiv_rn(1.0, aq));
                S->qpk = qpk;
                // 64-bit streams when |d2| could reach 2^31 (or q leaves int32)
                S->wide = (qpk >= (1LL << 29)) ? 1 : 0;
                S->bad = bad;
            }
            __syncthreads();  // B2
            const double s = S->s, rs = S->rs, aq = S->aq;
            const bool zero = F && S->zero;
            const bool wide = S->wide;
            const bool fq_emit = FQ && kind == 0;
            const long long hp1 = S->p1, hp2 = S->p2;

            // quantize one sample (codec.py:94-132); fast form valid when |q| < 2^31
            auto quant32 = [&](T xv) -> int {
                if (F) return zero ? 0 : __double2int_rn((double)xv * s);
                if (DT == 2) return aq == 1.0 ? (int)xv : __double2int_rn((double)xv * aq);
                return aq == 1.0 ? (int)xv : __double2int_rn((double)(int)xv * aq);
            };
            auto quant64 = [&](T xv) -> long long {
                if (F) return zero ? 0 : f2i64(rint((double)xv * s));
                const long long v = (long long)xv;
                return aq == 1.0 ? v : f2i64(rint((double)v * aq));
            };
            // dequantize to the dtype's value in double (codec.py:135-146)
            auto deq = [&](long long q) -> double {
                const double r = (double)q;
                if (F) {
                    double y0 = r * rs;
                    double e = __fma_rn(-s, y0, r);
                    double y = __fma_rn(e, rs, y0);
                    return (DT == 3) ? (double)__double2float_rn(y) : y;
                } else {
                    long long yi;
                    if (aq == 1.0) yi = q;
                    else {
                        double y0 = r * rs;
                        double e = __fma_rn(-aq, y0, r);
                        yi = f2i64(rint(__fma_rn(e, rs, y0)));
                    }
                    yi = yi < Tr::LO ? Tr::LO : (yi > Tr::HI ? Tr::HI : yi);
                    return (double)yi;
                }
            };
            auto qat = [&](int i) -> long long {  // 64-bit q with block context
                if (i < 0) return i == -1 ? hp1 : hp2;
                if (i >= n) return 0;
                return wide ? quant64(xs[i]) : (long long)quant32(xs[i]);
            };

            // ================= phase B: fixed-quality residual power =================
            if (fq_emit) {
                double pds = 0.0;
                if (regular) {
                    if (warp * 4 < L) {
                        double r = 0.0;
                        if (leaf < L) {
                            const int base = leaf * 128 + jj;
#pragma unroll 4
                            for (int i = 0; i < 16; i++) {
                                const T xv = xs[base + 8 * i];
                                const long long q = wide ? quant64(xv) : (long long)quant32(xv);
                                const double d = (double)xv - deq(q);
                                const double d2 = d * d;
                                r = (i == 0) ? d2 : r + d2;
                            }
                        }
                        r += __shfl_xor_sync(0xffffffffu, r, 1);
                        r += __shfl_xor_sync(0xffffffffu, r, 2);
                        r += __shfl_xor_sync(0xffffffffu, r, 4);
                        if (L >= 2) r += __shfl_xor_sync(0xffffffffu, r, 8);
                        if (L >= 4) r += __shfl_xor_sync(0xffffffffu, r, 16);
                        pds = r;
                    }
                }
                if (lane == 0) S->pdw[warp] = pds;
            }

            // ================= phase C: streams, widths, costs, sign flips =================
            const int t0 = SPT * tid;
            const bool active = t0 < np;
            int q[SPT];
            int hq1 = 0, hq2 = 0;
            uint32_t epk[3] = {0u, 0u, 0u};
            int se[3] = {0, 0, 0};
            unsigned emax = 0;
            int flips = 0;
            if (!wide) {
                if (active) {
                    if (DT == 3 && t0 + SPT <= n) {
                        const float4* x4 = (const float4*)(xs + t0);
#pragma unroll
                        for (int c = 0; c < SPT / 4; c++) {
                            const float4 v = x4[c];
                            q[4 * c] = quant32((T)v.x); q[4 * c + 1] = quant32((T)v.y);
                            q[4 * c + 2] = quant32((T)v.z); q[4 * c + 3] = quant32((T)v.w);
                        }
                    } else {
#pragma unroll
                        for (int k2 = 0; k2 < SPT; k2++) {
                            const int i = t0 + k2;
                            q[k2] = (i < n) ? quant32(xs[i]) : 0;
                        }
                    }
                    hq1 = t0 >= 1 ? quant32(xs[t0 - 1]) : (int)hp1;
                    hq2 = t0 >= 2 ? quant32(xs[t0 - 2]) : (int)hp2;
                    int m1 = hq1, dprev = hq1 - hq2;
#pragma unroll
                    for (int g = 0; g < 4; g++) {
                        unsigned o0 = 0, o1 = 0, o2 = 0;
#pragma unroll
                        for (int kk = 0; kk < 4; kk++) {
                            const int v0 = q[4 * g + kk];
                            const int v1 = v0 - m1;
                            const int v2 = v1 - dprev;
                            o0 |= wbits32(v0); o1 |= wbits32(v1); o2 |= wbits32(v2);
                            flips += (int)((unsigned)(v0 ^ m1) >> 31);
                            m1 = v0; dprev = v1;
                        }
                        const bool gv = (t0 + 4 * g) < np;
                        const int w0 = gv ? bitlen32(o0) : 0, w1 = gv ? bitlen32(o1) : 0,
                                  w2 = gv ? bitlen32(o2) : 0;
                        epk[0] |= (uint32_t)w0 << (8 * g);
                        epk[1] |= (uint32_t)w1 << (8 * g);
                        epk[2] |= (uint32_t)w2 << (8 * g);
                        se[0] += w0; se[1] += w1; se[2] += w2;
                    }
                    if (t0 == 0) flips -= (int)((unsigned)(q[0] ^ hq1) >> 31);  // no predecessor in the block
#pragma unroll
                    for (int k2 = 0; k2 < SPT; k2++) {
                        if (t0 + k2 == np - 1) S->last1 = q[k2];
                        if (t0 + k2 == np - 2) S->last2 = q[k2];
                    }
                }
            } else {
                // 64-bit streams, samples recomputed from x (rare path)
                if (active) {
                    long long m1 = qat(t0 - 1), m2 = qat(t0 - 2);
                    long long dprev = (long long)((unsigned long long)m1 - (unsigned long long)m2);
                    for (int g = 0; g < 4; g++) {
                        unsigned long long o0 = 0, o1 = 0, o2 = 0;
                        for (int kk = 0; kk < 4; kk++) {
                            const long long v0 = qat(t0 + 4 * g + kk);
                            const long long v1 = (long long)((unsigned long long)v0 - (unsigned long long)m1);
                            const long long v2 = (long long)((unsigned long long)v1 - (unsigned long long)dprev);
                            o0 |= wbits64(v0); o1 |= wbits64(v1); o2 |= wbits64(v2);
                            if (v0 >= (1LL << 62) || v0 < -(1LL << 62)) o0 |= 1ULL << 63;
                            if (v1 >= (1LL << 62) || v1 < -(1LL << 62)) o1 |= 1ULL << 63;
                            if (v2 >= (1LL << 62) || v2 < -(1LL << 62)) o2 |= 1ULL << 63;
                            if (t0 + 4 * g + kk > 0) flips += ((v0 ^ m1) < 0) ? 1 : 0;
                            m1 = v0; dprev = v1;
                        }
                        const bool gv = (t0 + 4 * g) < np;
                        int w0 = gv ? bitlen64(o0) : 0, w1 = gv ? bitlen64(o1) : 0, w2 = gv ? bitlen64(o2) : 0;
                        const unsigned wm = (unsigned)max(w0, max(w1, w2));
                        emax = wm > emax ? wm : emax;
                        w0 = min(w0, 255); w1 = min(w1, 255); w2 = min(w2, 255);
                        epk[0] |= (uint32_t)w0 << (8 * g);
                        epk[1] |= (uint32_t)w1 << (8 * g);
                        epk[2] |= (uint32_t)w2 << (8 * g);
                        se[0] += w0; se[1] += w1; se[2] += w2;
                    }
                    if (t0 <= np - 1 && np - 1 < t0 + SPT) {
                        S->last1 = qat(np - 1);
                        S->last2 = qat(np - 2);
                    }
                }
            }
            {
                const int s0 = __reduce_add_sync(0xffffffffu, se[0]);
                const int s1 = __reduce_add_sync(0xffffffffu, se[1]);
                const int s2 = __reduce_add_sync(0xffffffffu, se[2]);
                const unsigned em = __reduce_max_sync(0xffffffffu, emax);
                const int fl = __reduce_add_sync(0xffffffffu, flips);
                if (lane == 0) {
                    S->sew[0][warp] = s0; S->sew[1][warp] = s1; S->sew[2][warp] = s2;
                    S->emaxw[warp] = em;
                    S->monc[warp] = fl;
                    S->edge_first[warp] = epk[0] & 0xffu | ((epk[1] & 0xffu) << 8) | ((epk[2] & 0xffu) << 16);
                }
                if (lane == 31) S->edge_last[warp] = (epk[0] >> 24) | ((epk[1] >> 24) << 8) | ((epk[2] >> 24) << 16);
            }
            __syncthreads();  // B4
            if (tid == 0) {
                long long tt[3] = {0, 0, 0};
                unsigned em = 0;
                int fl = 0;
                for (int w = 0; w < NW; w++) {
                    tt[0] += S->sew[0][w]; tt[1] += S->sew[1][w]; tt[2] += S->sew[2][w];
                    em = S->emaxw[w] > em ? S->emaxw[w] : em;
                    fl += S->monc[w];
                }
                S->sum_e[0] = tt[0]; S->sum_e[1] = tt[1]; S->sum_e[2] = tt[2];
                if (em > (unsigned)kMaxExponent && !S->bad) S->bad = APAX_ERR_INTERNAL;
                // every sign change of the nonzero subsequence is witnessed by a
                // distinct sign-bit flip between neighbours, so cf <= flips /
                // (2 (np-1)); the exact monitor is only needed above the gate
                S->exact_mon = (3LL * fl > 2LL * (np - 1)) ? 1 : 0;
                S->gate = 0;
                if (fq_emit) {
                    double pd;
                    if (regular) {
                        const int nwd = (L + 3) / 4;
                        double v[NW];
                        for (int w = 0; w < nwd; w++) v[w] = S->pdw[w];
                        for (int st = 1; st < nwd; st <<= 1)
                            for (int w = 0; w + st < nwd; w += 2 * st) v[w] = v[w] + v[w + st];
                        pd = v[0];
                    } else {
                        auto td = [&](int i) {
                            const double d = (double)xs[i] - deq(qat(i));
                            return d * d;
                        };
                        pd = pw_seq(td, 0, n);
                    }
                    S->pd = pd;
                }
            }
            __syncthreads();  // B5
            if (S->exact_mon) {
                // exact monitor (transform.py:67-83): ordered sign-change count
                int ch = 0, fs = 0, lsg = 0;
                if (active) {
                    for (int k2 = 0; k2 < SPT; k2++) {
                        const long long v = qat(t0 + k2 < np ? t0 + k2 : np + 4);
                        const int sg = (v > 0) - (v < 0);
                        if (sg) {
                            if (lsg) ch += (sg != lsg);
                            else fs = sg;
                            lsg = sg;
                        }
                    }
                }
#pragma unroll
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
                __syncthreads();
                if (tid == 0) {
                    int ch2 = 0, f = 0, l = 0;
                    for (int w = 0; w < NW; w++) {
                        const int of = (S->monf[w] & 3) - 1, ol = ((S->monf[w] >> 2) & 3) - 1;
                        ch2 += S->monc[w] + ((l != 0 && of != 0 && l != of) ? 1 : 0);
                        if (!f) f = of;
                        if (ol) l = ol;
                    }
                    const double cf = (double)ch2 / (2.0 * (double)(np - 1));
                    S->gate = cf > 1.0 / 3.0;
                }
                __syncthreads();
            }
            if (tid == 0) {
                int sel = 0;
                if (S->has_pc && !S->gate) {
                    if (S->pc[1] < S->pc[sel]) sel = 1;
                    if (S->pc[2] < S->pc[sel]) sel = 2;
                }
                S->sel = sel;
                if (kind != 0) {
                    // cost-only passes (lossless halo / warm_self)
                    const long long g4 = 4LL * G;
                    if (kind == 1) {
                        S->has_pc = 1;
                        for (int c = 0; c < 3; c++) S->pc[c] = 4 * S->sum_e[c] + g4;
                        S->p1 = S->last1; S->p2 = S->last2;
                        S->emitted = 1; S->initialized = 1;
                    } else if (kind == 2) {
                        long long mn = S->sum_e[0];
                        mn = S->sum_e[1] < mn ? S->sum_e[1] : mn;
                        mn = S->sum_e[2] < mn ? S->sum_e[2] : mn;
                        const double bps0 = (double)(4 * mn + g4 + 8LL * HS) / (double)bs;
                        const double att0 = clamp_att(0.0 - 6.02 * (bps0 - P.target), P.att_lo);
                        S->att = att0;
                        S->a = att_to_a(att0);
                    } else {
                        S->has_pc = 1;
                        for (int c = 0; c < 3; c++) S->pc[c] = 4 * S->sum_e[c] + g4;
                    }
                    if (S->bad) report_error(P.status, b, S->bad);
                }
            }
            __syncthreads();  // B6
            if (kind != 0) continue;

            // ================= phase D: JEE (bitmask) + mantissa offsets =================
            const int sel = S->sel;
            const uint32_t es = sel == 0 ? epk[0] : (sel == 1 ? epk[1] : epk[2]);
            const int g0 = 4 * tid;                  // first group of this thread
            int ev[5];
            int enext;
            {
                const uint32_t up = __shfl_up_sync(0xffffffffu, es, 1);
                const uint32_t dn = __shfl_down_sync(0xffffffffu, es, 1);
                ev[0] = lane > 0 ? (int)(up >> 24)
                                 : (warp > 0 ? (int)((S->edge_last[warp - 1] >> (8 * sel)) & 0xffu) : 0);
#pragma unroll
                for (int g = 0; g < 4; g++) ev[g + 1] = (int)((es >> (8 * g)) & 0xffu);
                enext = lane < 31 ? (int)(dn & 0xffu)
                                  : (warp < NW - 1 ? (int)((S->edge_first[warp + 1] >> (8 * sel)) & 0xffu) : 0);
                int pb = 0, eb = 0;
#pragma unroll
                for (int k2 = 0; k2 < 4; k2++) {
                    const int p = g0 + k2;
                    const int d = ev[k2 + 1] - ev[k2];
                    const int dn2 = (k2 < 3 ? ev[k2 + 2] : enext) - ev[k2 + 1];
                    const bool s1 = (unsigned)(d + 1) <= 2u, s1n = (unsigned)(dn2 + 1) <= 2u;
                    const bool s2 = (unsigned)(d + 2) <= 4u;
                    const bool pr = p != 0 && p + 1 < G && s1 && s1n;
                    if (pr) pb |= 1 << k2;
                    else if (p == 0 || !s2) eb |= 1 << k2;
                }
                // 32-position words: 8 lanes x 4 positions
                const int sh = 4 * (lane & 7);
                uint32_t pw = (uint32_t)pb << sh, ew = (uint32_t)eb << sh;
                pw |= __shfl_xor_sync(0xffffffffu, pw, 1);
                ew |= __shfl_xor_sync(0xffffffffu, ew, 1);
                pw |= __shfl_xor_sync(0xffffffffu, pw, 2);
                ew |= __shfl_xor_sync(0xffffffffu, ew, 2);
                pw |= __shfl_xor_sync(0xffffffffu, pw, 4);
                ew |= __shfl_xor_sync(0xffffffffu, ew, 4);
                if ((lane & 7) == 0) { S->pw[warp * 4 + (lane >> 3)] = pw; S->ew[warp * 4 + (lane >> 3)] = ew; }
            }
            // mantissa bits of this thread and warp-inclusive prefix
            unsigned mb = 0;
#pragma unroll
            for (int g = 0; g < 4; g++) mb += (g0 + g < G) ? 4u * (unsigned)ev[g + 1] : 0u;
            unsigned mbi = mb;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned o = __shfl_up_sync(0xffffffffu, mbi, d);
                if (lane >= d) mbi += o;
            }
            if (lane == 31) S->mbw[warp] = mbi;
            __syncthreads();  // B7
            if (warp == 0) {
                // word m = positions 32m .. 32m+31
                const int m = lane;
                const uint32_t Pm = S->pw[m], Em = S->ew[m];
                const int lo = 32 * m;
                const uint32_t V = (G >= lo + 32) ? 0xffffffffu : (G > lo ? ((1u << (G - lo)) - 1u) : 0u);
                uint32_t c0, c1;
                const uint32_t C0 = consumed_word(Pm, 0u, &c0);
                const uint32_t C1 = consumed_word(Pm, 1u, &c1);
                // carry scan of 1-bit transfer functions f(c) = c ? c1 : c0
                uint32_t f0 = c0, f1 = c1;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t o0 = __shfl_up_sync(0xffffffffu, f0, d);
                    const uint32_t o1 = __shfl_up_sync(0xffffffffu, f1, d);
                    if (lane >= d) {
                        const uint32_t n0 = o0 ? f1 : f0, n1 = o1 ? f1 : f0;
                        f0 = n0; f1 = n1;
                    }
                }
                uint32_t cin = __shfl_up_sync(0xffffffffu, f0, 1);  // exclusive, applied to 0
                if (lane == 0) cin = 0u;
                const uint32_t Cm = cin ? C1 : C0;
                const uint32_t Tm = V & ~Cm;          // token starts
                const uint32_t Xm = Tm & Em;          // escapes
                const int nibm = __popc(Tm) + 2 * __popc(Xm);
                int ni = nibm;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int o = __shfl_up_sync(0xffffffffu, ni, d);
                    if (lane >= d) ni += o;
                }
                S->tw[m] = Tm; S->xw[m] = Xm; S->jw[m] = Tm & Pm;
                S->nibpre[m] = ni - nibm;
                unsigned mbx = 0, mbt = 0;
                if (lane < NW) mbx = S->mbw[lane];
                unsigned mbs = mbx;
#pragma unroll
                for (int d = 1; d < NW; d <<= 1) {
                    const unsigned o = __shfl_up_sync(0xffffffffu, mbs, d);
                    if (lane >= d) mbs += o;
                }
                mbt = __shfl_sync(0xffffffffu, mbs, NW - 1);
                if (lane < NW) S->mbpre[lane] = mbs - mbx;
                const int nib_total = __shfl_sync(0xffffffffu, ni, 31);
                if (lane == 0) {
                    S->jee_nib = nib_total;
                    S->bits = mbt;
                    S->blen = HS + ((nib_total + 1) >> 1) + ((long long)mbt + 7) / 8;
                }
            }
            __syncthreads();  // B8
            const long long wb = S->tail_len;            // window byte of block start
            const long long jee_bytes = (S->jee_nib + 1) >> 1;
            if (g0 < G && !S->bad) {
                const int w = tid >> 3, sh = 4 * (tid & 7);
                const uint32_t below = (1u << sh) - 1u;
                const uint32_t Tw = S->tw[w], Xw = S->xw[w], Jw = S->jw[w];
                const int nib_off = S->nibpre[w] + __popc(Tw & below) + 2 * __popc(Xw & below);
                const int Tb = (Tw >> sh) & 15, Xb = (Xw >> sh) & 15, Jb = (Jw >> sh) & 15;
                BitWriter bw;
                bw.init(win, 8 * (wb + HS) + 4LL * nib_off);
#pragma unroll
                for (int k2 = 0; k2 < 4; k2++) {
                    if (!((Tb >> k2) & 1)) continue;
                    const int e = ev[k2 + 1];
                    const int d = e - ev[k2];
                    if ((Jb >> k2) & 1) {
                        const int dn2 = (k2 < 3 ? ev[k2 + 2] : enext) - e;
                        bw.put32((uint32_t)((d + 1) * 3 + (dn2 + 1)), 4);
                    } else if ((Xb >> k2) & 1) {
                        bw.put32(0xF00u | (uint32_t)e, 12);
                    } else {
                        bw.put32((uint32_t)(11 + d), 4);
                    }
                }
                bw.flush();
            }
            if (g0 < G && !S->bad) {
                const unsigned mbx = S->mbpre[warp] + (mbi - mb);
                BitWriter mw;
                mw.init(win, 8 * (wb + HS + jee_bytes) + (long long)mbx);
                if (!wide) {
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
                            vs[kk] = sel == 0 ? v0 : (sel == 1 ? v1 : v2);
                        }
                        const int w = ev[g + 1];
                        if (g0 + g >= G || w == 0) continue;
                        if (w <= 8) {
                            const uint32_t m = (1u << w) - 1u;
                            const uint32_t c = ((uint32_t)vs[0] & m) << (3 * w) | ((uint32_t)vs[1] & m) << (2 * w) |
                                               ((uint32_t)vs[2] & m) << w | ((uint32_t)vs[3] & m);
                            mw.put32(c, 4 * w);
                        } else if (w <= 16) {
                            const uint32_t m = (1u << w) - 1u;
                            mw.put32(((uint32_t)vs[0] & m) << w | ((uint32_t)vs[1] & m), 2 * w);
                            mw.put32(((uint32_t)vs[2] & m) << w | ((uint32_t)vs[3] & m), 2 * w);
                        } else {
#pragma unroll
                            for (int kk = 0; kk < 4; kk++) mw.put32((uint32_t)vs[kk] & (0xffffffffu >> (32 - w)), w);
                        }
                    }
                } else {
                    long long m1 = qat(t0 - 1), m2 = qat(t0 - 2);
                    long long dprev = (long long)((unsigned long long)m1 - (unsigned long long)m2);
                    for (int g = 0; g < 4; g++) {
                        const int w = ev[g + 1];
                        for (int kk = 0; kk < 4; kk++) {
                            const long long v0 = qat(t0 + 4 * g + kk);
                            const long long v1 = (long long)((unsigned long long)v0 - (unsigned long long)m1);
                            const long long v2 = (long long)((unsigned long long)v1 - (unsigned long long)dprev);
                            m1 = v0; dprev = v1;
                            if (g0 + g < G && w) mw.put((unsigned long long)(sel == 0 ? v0 : (sel == 1 ? v1 : v2)), w);
                        }
                    }
                }
                mw.flush();
            }
            if (tid == 0) {
                // block header (dtypes.py:156-165)
                const int restart = (S->emitted == 0);
                const int code = S->code;
                const uint32_t hb[6] = {(uint32_t)((sel & 3) | (restart ? 4 : 0)), (uint32_t)(code & 0xFF),
                                        (uint32_t)((code >> 8) & 0xFF), 0u,
                                        (uint32_t)(uint8_t)(int8_t)S->fbe, 0u};
                for (int k2 = 0; k2 < HS; k2++) {
                    const long long bp = wb + k2;
                    atomicOr(&win[bp >> 2], hb[k2] << (8 * (bp & 3)));
                }
            }
            __syncthreads();  // B9
            // ---- flush whole 16-byte chunks; keep the tail ----
            {
                const long long total = wb + S->blen;
                const long long full = total & ~15LL;
                if (S->direct) {
                    copy_out<true>(P.out + kFileHeader + S->win_base, win, full);
                } else {
                    uint4* dst = (uint4*)(slot + S->win_base);
                    const uint4* src = (const uint4*)win;
                    for (long long c = tid; c < (full >> 4); c += NT) dst[c] = src[c];
                }
                if (tid == 0) {
                    const int w0 = (int)(full >> 2);
                    S->tail[0] = win[w0]; S->tail[1] = win[w0 + 1];
                    S->tail[2] = win[w0 + 2]; S->tail[3] = win[w0 + 3];
                    // bookkeeping (codec.py:220-254)
                    if (P.block_offsets) P.block_offsets[b] = S->win_base + wb;  // unit-relative
                    if (P.trace) {
                        double* tr = P.trace + 10 * b;
                        tr[0] = S->att; tr[1] = S->a; tr[2] = S->code; tr[3] = S->fbe; tr[4] = sel;
                        tr[5] = (double)(4 * S->sum_e[0] + 4LL * G); tr[6] = (double)(4 * S->sum_e[1] + 4LL * G);
                        tr[7] = (double)(4 * S->sum_e[2] + 4LL * G); tr[8] = (double)S->blen;
                        tr[9] = (S->emitted == 0);
                    }
                    if (S->bad) report_error(P.status, b, S->bad);
                    S->has_pc = 1;
                    for (int c = 0; c < 3; c++) S->pc[c] = 4 * S->sum_e[c] + 4LL * G;
                    S->p1 = S->last1;
                    S->p2 = S->last2;
                    if (P.mode == 1) {
                        if (S->emitted == 0) {
                            long long mn = S->pc[0] < S->pc[1] ? S->pc[0] : S->pc[1];
                            mn = S->pc[2] < mn ? S->pc[2] : mn;
                            const double bps0 = (double)(mn + 8LL * HS) / (double)bs;
                            S->att = clamp_att(S->att - 6.02 * (bps0 - P.target), P.att_lo);
                        } else {
                            const double err = (double)(S->blen * 8) / (double)bs - P.target;
                            S->att = clamp_att(S->att - clamp_step(0.75 * err), P.att_lo);
                        }
                    } else if (P.mode == 2) {
                        const double px = S->px / (double)n, pd = S->pd / (double)n;
                        if (px > 0.0) {
                            const double measured = (pd == 0.0) ? INFINITY : 10.0 * log10(px / pd);
                            if (isfinite(measured))
                                S->att = clamp_att(S->att - clamp_step(0.5 * (measured - P.target)), P.att_lo);
                        }
                    }
                    S->emitted += 1;
                    S->unit_len += S->blen;
                    S->win_base += full;
                    S->tail_len = (int)(total - full);
                }
            }
            if (warp == NW - 1) lookback_try(false);
            __syncthreads();  // B10
            if (S->pend_ready) place_pending();
        }

        // ---------------- unit end: last tail, publish, defer placement ----------------
        if (S->tail_len > 0) {
            if (S->direct) {
                if (tid < S->tail_len)
                    P.out[kFileHeader + S->win_base + tid] = ((const uint8_t*)S->tail)[tid];
            } else if (tid == 0) {
                const uint4 t4 = make_uint4(S->tail[0], S->tail[1], S->tail[2], S->tail[3]);
                *(uint4*)(slot + S->win_base) = t4;
            }
        }
        // at most one unit pending: finish the previous one first
        if (warp == NW - 1) lookback_try(true);
        __syncthreads();
        if (S->pend_ready) place_pending();
        if (tid == 0) {
            const long long Lu = S->unit_len;
            if (u == 0) {
                st_release(&P.lookback[0], kFlagInc | (unsigned long long)Lu);
                if (P.n_units == 1) {
                    P.status[2] = (unsigned long long)(kFileHeader + Lu);
                    if (P.block_offsets) P.block_offsets[P.n_blocks] = kFileHeader + Lu;
                }
            } else {
                st_release(&P.lookback[u], kFlagAgg | (unsigned long long)Lu);
                S->pend_u = u; S->pend_len = Lu; S->pend_b0 = b0; S->pend_b1 = b1;
                S->pend_k = u - 1; S->pend_acc = 0; S->pend_slot = cur_slot; S->pend_ready = 0;
            }
        }
        if (u == 0) {
            if (tid < kFileHeader) {
                unsigned char h[kFileHeader];
                h[0] = 'A'; h[1] = 'P'; h[2] = 'A'; h[3] = 'X';
                h[4] = 1; h[5] = (unsigned char)DT; h[6] = (unsigned char)P.mode; h[7] = 0;
                for (int k2 = 0; k2 < 4; k2++) h[8 + k2] = (unsigned char)((unsigned)bs >> (8 * k2));
                for (int k2 = 0; k2 < 8; k2++) h[12 + k2] = (unsigned char)((unsigned long long)P.n >> (8 * k2));
                const unsigned long long tb = (unsigned long long)__double_as_longlong(P.target);
                for (int k2 = 0; k2 < 8; k2++) h[20 + k2] = (unsigned char)(tb >> (8 * k2));
                P.out[tid] = h[tid];
            }
            if (P.block_offsets)
                for (long long bb = b0 + tid; bb < b1; bb += NT) P.block_offsets[bb] += kFileHeader;
        }
        cur_slot ^= 1;
        slot = slots2[cur_slot];
        __syncthreads();
    }
    // drain the last pending unit
    if (warp == NW - 1) lookback_try(true);
    __syncthreads();
    if (S->pend_ready) place_pending();
}

}  // namespace v2

size_t encode_v2_smem_bytes(int dt, int mode, int window_bytes) {
    auto al = [](size_t v) { return (v + 127) & ~(size_t)127; };
    (void)mode;
    size_t w = (size_t)dt_width(dt);
    return al(sizeof(v2::St)) + 2 * al((size_t)v2::MAXBS * w) + (size_t)window_bytes + 32;
}

bool encode_v2_supported(int bs) {
    return bs >= 128 && bs <= v2::MAXBS && (bs & (bs - 1)) == 0;
}

template <int DT>
static void* v2_fn() { return (void*)v2::encode_v2_kernel<DT>; }

static void* v2_kernel(int dt) {
    switch (dt) {
        case 0: return v2_fn<0>();
        case 1: return v2_fn<1>();
        case 2: return v2_fn<2>();
        case 3: return v2_fn<3>();
        default: return v2_fn<4>();
    }
}

int encode_v2_resident_ctas(int dt, size_t smem) {
    int dev = 0, nsm = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const void* fn = v2_kernel(dt);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, v2::NT, smem) != cudaSuccess || per < 1)
        per = 1;
    return per * (nsm > 0 ? nsm : 148);
}

int launch_encode_v2(int dt, const EncParams& P, int grid, size_t smem, cudaStream_t st) {
    const void* fn = v2_kernel(dt);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return APAX_ERR_CUDA;
    EncParams p = P;
    void* args[] = {&p};
    // cooperative: co-residency of all CTAs (round-robin units look back at
    // their predecessors' CTAs)
    if (cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(v2::NT), args, smem, st) != cudaSuccess)
        return APAX_ERR_CUDA;
    return APAX_OK;
}

}  // namespace apax
