// apax_decode_v2.cu -- CTA-parallel B200 APAX decoder for block sizes <= 4096.
//
// Same contract and bit-exact output as apax_decode.cu (reference
// decode_stream, pkg/src/apax/codec.py:308-329), which stays the general
// path (block sizes up to 16384) and the exact error reporter.
//
// Per block (one CTA of 256 threads, 4 groups = 16 samples per thread):
//   * the block's payload (from the side-band offset table) is staged in
//     shared memory with 16-byte loads;
//   * JEE (entropy.py:118-164) is parsed by all threads at once, 4 nibbles
//     per thread per pass: a thread finds its first token start locally
//     (two consecutive non-15 nibbles always precede a token start), then a
//     CTA scan of (exponent count, escape-reset value) gives every token its
//     exponent index and running value.  Any irregularity (a status the
//     reference would raise) re-runs the exact serial parser for the status;
//   * mantissas (entropy.py:262-276) are read at scanned bit offsets;
//   * reconstruct (transform.py:116-129) as CTA prefix sums, cross-block
//     history through the affine-map decoupled look-back;
//   * dequantize (codec.py:135-146) with a per-block reciprocal (Markstein
//     quotient == IEEE division) and store the [:n] slice from registers.
#include <cstdint>
#include <cuda_runtime.h>

#include "apax_device.cuh"
#include "apax_kernels.cuh"
#include "apax_jee.cuh"

#ifndef APAX_DEC_MINB
#define APAX_DEC_MINB 3
#endif

namespace apax {


namespace d2 {

constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int MAXBS = 4096;
constexpr int NIB_PER_PASS = 4 * NT;  // 4 nibbles per thread per pass

struct St {
    long long block;
    int sel, restart, code, fbe, err, fallback;
    long long pay_off, avail, staged;
    long long used, jee_bytes, mant_bits;
    long long p1, p2;
    int first_event;          // nibble position of the first event in a pass
    int event_done;           // 1: the first event completes the stream
    int cnt_base, val_base;   // carried into the next pass
    int emax;
    // scan scratch
    int sc_cnt[NW], sc_flag[NW], sc_val[NW];
    int pre_cnt[NW], pre_flag[NW], pre_val[NW];
    int ev_min[NW], ev_done[NW];
    long long red[NW + 1];
    long long l1, l2;
    unsigned long long mbar[2];
    long long ld_a[2], ld_boff[2], ld_bend[2];
    int ld_tma[2];
    unsigned redu[NW + 1];
};


// exclusive CTA scan of a 32-bit unsigned value
__device__ __forceinline__ unsigned cta_scan_u32(unsigned v, unsigned* red, unsigned& total) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned o = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += o;
    }
    if (lane == 31) red[warp] = x;
    __syncthreads();
    if (tid == 0) {
        unsigned acc = 0;
        for (int w = 0; w < NW; w++) { const unsigned t = red[w]; red[w] = acc; acc += t; }
        red[NW] = acc;
    }
    __syncthreads();
    const unsigned ex = red[warp] + x - v;
    total = red[NW];
    __syncthreads();
    return ex;
}

// exclusive CTA scan of a 64-bit value (mod 2^64)
__device__ __forceinline__ unsigned long long cta_scan_u64(unsigned long long v, long long* red) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned long long x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long o = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += o;
    }
    if (lane == 31) red[warp] = (long long)x;
    __syncthreads();
    if (tid == 0) {
        unsigned long long acc = 0;
        for (int w = 0; w < NW; w++) {
            const unsigned long long t = (unsigned long long)red[w];
            red[w] = (long long)acc;
            acc += t;
        }
    }
    __syncthreads();
    const unsigned long long ex = (unsigned long long)red[warp] + x - v;
    __syncthreads();
    return ex;
}

__device__ __forceinline__ unsigned long long read_bits(const uint32_t* w, long long bp, int nb) {
    const long long k = bp >> 5;
    const int sh = (int)(bp & 31);
    const unsigned long long hi = ((unsigned long long)bswap32(w[k]) << 32) | bswap32(w[k + 1]);
    unsigned long long t = hi << sh;
    if (sh) t |= (unsigned long long)bswap32(w[k + 2]) >> (32 - sh);
    return t >> (64 - nb);
}

struct Aff {
    unsigned long long m11, m12, m21, m22, c1, c2;
};
__device__ __forceinline__ Aff aff_compose(const Aff& A, const Aff& B) {  // A after B
    Aff r;
    r.m11 = A.m11 * B.m11 + A.m12 * B.m21;
    r.m12 = A.m11 * B.m12 + A.m12 * B.m22;
    r.m21 = A.m21 * B.m11 + A.m22 * B.m21;
    r.m22 = A.m21 * B.m12 + A.m22 * B.m22;
    r.c1 = A.m11 * B.c1 + A.m12 * B.c2 + A.c1;
    r.c2 = A.m21 * B.c1 + A.m22 * B.c2 + A.c2;
    return r;
}

template <int DT>
__global__ void __launch_bounds__(NT, APAX_DEC_MINB) decode_v2_kernel(DecParams P) {
    using Tr = DT_<DT>;
    using T = typename Tr::T;
    constexpr int HS = Tr::HDR;
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bs = P.bs;

    St* S = (St*)smem;
    size_t off = (sizeof(St) + 127) & ~(size_t)127;
    uint8_t* e = smem + off;                   // group exponents
    off += ((size_t)MAXBS / 4 + 64 + 127) & ~(size_t)127;
    const int bufsz = (P.payload_cap + 64 + 127) & ~127;
    uint8_t* pbuf[2];
    pbuf[0] = smem + off;                      // header + payload (16B-aligned superset)
    pbuf[1] = smem + off + bufsz;
    const long long limit = P.nbytes & ~15LL;   // TMA never reads past the blob

    using namespace apax::tma;
    if (tid == 0) {
        mbar_init(&S->mbar[0]);
        mbar_init(&S->mbar[1]);
        fence_mbar_init();
    }
    __syncthreads();
    uint32_t phase[2] = {0u, 0u};
    const long long stride = gridDim.x;
    // thread 0 keeps the offsets of the block after next (loaded one block ahead)
    long long nx0 = -1, nx1 = -1;
    // issue the load of block bb (offsets o0, o1) into buffer slot (thread 0)
    auto issue = [&](long long bb, long long o0, long long o1, int slot) {
        long long hi = o1 > o0 + HS ? o1 : o0 + HS;
        const long long a0 = (o0 >= 0 ? o0 : 0) & ~15LL;
        const long long e1 = (hi + 15) & ~15LL;
        const long long len = e1 - a0;
        S->ld_a[slot] = a0;
        S->ld_boff[slot] = o0;
        S->ld_bend[slot] = o1;
        // bulk copy only when the 16-byte superset lies inside the blob
        const bool ok = o0 >= 0 && len > 0 && len <= bufsz && e1 <= limit &&
                        ((((uintptr_t)(P.blob + a0)) & 15) == 0);
        S->ld_tma[slot] = ok ? 1 : 0;
        if (ok) {
            fence_proxy_async();
            tma_load(pbuf[slot], P.blob + a0, (uint32_t)len, &S->mbar[slot]);
        }
        (void)bb;
    };
    if (tid == 0 && blockIdx.x < P.n_blocks) {
        const long long bb = blockIdx.x;
        issue(bb, P.offsets[bb], P.offsets[bb + 1], 0);
        if (bb + stride < P.n_blocks) { nx0 = P.offsets[bb + stride]; nx1 = P.offsets[bb + stride + 1]; }
    }
    __syncthreads();  // publish the first load descriptor

    int kk = 0;
    for (long long b = blockIdx.x; b < P.n_blocks; b += stride, kk++) {
        const int cur = kk & 1;
        uint8_t* pay = pbuf[cur];
        const long long start = b * (long long)bs;
        const int n = (int)((P.n - start) < bs ? (P.n - start) : bs);
        const int G = (n + 3) >> 2;
        const int np = 4 * G;
        unsigned long long* cw = P.carry + 16 * b;   // [0] flag, [1..6] map, [8..9] value
        // prefetch the next block of this CTA (its offsets were read one block ago)
        if (tid == 0 && b + stride < P.n_blocks) {
            issue(b + stride, nx0, nx1, cur ^ 1);
            if (b + 2 * stride < P.n_blocks) {
                nx0 = P.offsets[b + 2 * stride];
                nx1 = P.offsets[b + 2 * stride + 1];
            }
        }
        // wait for this block's bytes
        const bool was_tma = S->ld_tma[cur] != 0;
        const long long a0 = S->ld_a[cur];
        const long long boff = S->ld_boff[cur];
        const long long bend = S->ld_bend[cur];
        if (was_tma) {
            mbar_wait(&S->mbar[cur], phase[cur]);
            phase[cur] ^= 1u;
        } else if (boff >= 0) {
            long long hi = bend > boff + HS ? bend : boff + HS;
            long long e1 = hi < P.nbytes ? hi : P.nbytes;
            long long len = e1 - a0;
            if (len > bufsz) len = bufsz;
            for (long long i = tid; i < len; i += NT) pay[i] = P.blob[a0 + i];
        }
        __syncthreads();
        if (tid == 0) {
            S->err = 0;
            S->fallback = 0;
            if (boff < 0) {
                S->err = -1;
            } else if (P.nbytes - boff < HS) {
                S->err = APAX_ERR_BLOCK_HDR_TRUNCATED;
            } else {
                const uint8_t* h = pay + (boff - a0);
                S->sel = h[0] & 3;
                S->restart = (h[0] >> 2) & 1;
                S->code = h[1] | (h[2] << 8);
                S->fbe = Tr::F ? (int)(int8_t)h[4] : 0;
                if (S->sel == 3) S->err = APAX_ERR_SELECTOR;
                const long long ps = boff + HS;
                long long pe = bend > ps ? bend : ps;
                long long e1 = (pe + 15) & ~15LL;
                if (e1 > limit) e1 = limit;
                long long staged_end = a0 + (e1 - a0 < bufsz ? e1 - a0 : bufsz);
                if (!was_tma) staged_end = a0 + min((long long)bufsz, min(pe, P.nbytes) - a0);
                S->pay_off = ps - a0;
                S->avail = P.nbytes - ps;
                S->staged = staged_end - ps;
                S->cnt_base = 0;
                S->val_base = 0;
            }
        }
        __syncthreads();
        // ---- JEE (entropy.py:118-164): one warp parses the block from global
        // memory (apax_jee.cuh); any irregularity re-runs the exact parser
        if (S->err == 0 && warp == 0) {
            const long long maxj = (3LL * G + 2) / 2;
            const long long nbj = S->avail < maxj ? S->avail : maxj;
            int u = 0;
            int st = warp_jee_fast(P.blob + boff + HS, P.blob + P.nbytes, (int)(2 * nbj), G, e, u);
            if (st < 0) {
                long long u2 = 0, esum = 0;
                st = warp_jee_decode(P.blob + boff + HS, 2 * nbj, G, e, u2, esum);
                u = (int)u2;
            }
            if (lane == 0) {
                if (st) S->err = st;
                else S->used = u;
            }
        }
        __syncthreads();
        if (tid == 0 && S->err == 0) {
            S->jee_bytes = (S->used + 1) >> 1;
        }
        __syncthreads();
        // ---- mantissa offsets ----
        const int g0 = 4 * tid;
        int ew[4];
        unsigned lbits = 0;
        if (S->err == 0) {
#pragma unroll
            for (int g = 0; g < 4; g++) {
                ew[g] = (g0 + g < G) ? (int)e[g0 + g] : 0;
                lbits += 4u * (unsigned)ew[g];
            }
        }
        unsigned tbits = 0;
        const unsigned bitpos = cta_scan_u32(lbits, S->redu, tbits);
        if (tid == 0 && S->err == 0) {
            const long long mant_bytes = ((long long)tbits + 7) / 8;
            if (S->avail < S->jee_bytes + mant_bytes) S->err = APAX_ERR_MANTISSA_TRUNCATED;
            else if (S->jee_bytes + mant_bytes > S->staged) S->err = APAX_ERR_ARG;  // offsets inconsistent
        }
        __syncthreads();
        const int err = S->err;
        if (err) {
            if (tid == 0) {
                if (err > 0) report_error(P.status, b, err);
                cw[8] = 0; cw[9] = 0;
                __threadfence();
                st_release(&cw[0], kFlagInc);
            }
            __syncthreads();
            continue;
        }
        // ---- unpack 16 samples per thread ----
        long long v[16];
        {
            const uint32_t* w = (const uint32_t*)pay;
            long long bp = 8 * (S->pay_off + S->jee_bytes) + bitpos;
#pragma unroll
            for (int g = 0; g < 4; g++) {
                const int wd = ew[g];
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    long long x = 0;
                    if (wd) {
                        unsigned long long r = read_bits(w, bp, wd);
                        bp += wd;
                        if (r >> (wd - 1)) r -= (1ULL << wd);
                        x = (long long)r;
                    }
                    v[4 * g + k] = x;
                }
            }
        }
        // ---- reconstruct (transform.py:116-129) ----
        const int sel = S->sel;
        if (sel >= 1) {
            unsigned long long acc = 0;
#pragma unroll
            for (int i = 0; i < 16; i++) { acc += (unsigned long long)v[i]; v[i] = (long long)acc; }
            const unsigned long long ex = cta_scan_u64(acc, S->red);
#pragma unroll
            for (int i = 0; i < 16; i++) v[i] = (long long)((unsigned long long)v[i] + ex);
            if (sel == 2) {
                unsigned long long acc2 = 0;
#pragma unroll
                for (int i = 0; i < 16; i++) { acc2 += (unsigned long long)v[i]; v[i] = (long long)acc2; }
                const unsigned long long ex2 = cta_scan_u64(acc2, S->red);
#pragma unroll
                for (int i = 0; i < 16; i++) v[i] = (long long)((unsigned long long)v[i] + ex2);
            }
        }
        // local carry of the block: last two (local) values
        if (g0 < G && g0 + 4 >= G) {  // thread holding samples np-1, np-2
#pragma unroll
            for (int i = 0; i < 16; i++) {
                if (g0 * 4 + i == np - 1) S->l1 = v[i];
                if (g0 * 4 + i == np - 2) S->l2 = v[i];
            }
        }
        __syncthreads();
        if (warp == 0) {
            const unsigned long long L1 = (unsigned long long)S->l1;
            const unsigned long long L2 = (unsigned long long)S->l2;
            const unsigned long long unp = (unsigned long long)np;
            Aff M;
            if (sel == 0) M = {0, 0, 0, 0, L1, L2};
            else if (sel == 1) M = {1, 0, 1, 0, L1, L2};
            else M = {unp + 1, 0ULL - unp, unp, 0ULL - (unp - 1), L1, L2};
            unsigned long long in1 = P.entry_p1, in2 = P.entry_p2;   // history entering block 0
            // the block's history map (constant for restart / D0 blocks); kept
            // in cw[1..6] for every block: apax_decode_range composes them
            if (sel == 0 || S->restart) M = {0, 0, 0, 0, M.c1, M.c2};
            if (lane == 0) {
                cw[1] = M.m11; cw[2] = M.m12; cw[3] = M.m21; cw[4] = M.m22; cw[5] = M.c1; cw[6] = M.c2;
            }
            if (sel != 0 && !S->restart && b > 0) {
                if (lane == 0) {
                    __threadfence();
                    st_release(&cw[0], kFlagAgg);
                }
                // warp-parallel look-back: lane l examines block b-1-l
                Aff acc = {1, 0, 0, 1, 0, 0};   // composition of the blocks passed so far
                long long base = b - 1;
                for (;;) {
                    const long long k = base - lane;
                    unsigned long long fl = kFlagInc;
                    const unsigned long long* ck = P.carry + 16 * (k >= 0 ? k : 0);
                    if (k >= 0) fl = ld_acquire(&ck[0]);
                    const unsigned inc = __ballot_sync(0xffffffffu, fl == kFlagInc);
                    const unsigned nrd = __ballot_sync(0xffffffffu, fl != kFlagInc && fl != kFlagAgg);
                    const int first_inc = inc ? __ffs(inc) - 1 : 32;
                    const unsigned need = first_inc >= 31 ? 0xffffffffu : ((2u << first_inc) - 1u);
                    if (nrd & need) { __nanosleep(32); continue; }
                    Aff Ml = {1, 0, 0, 1, 0, 0};
                    if (lane < first_inc) {
                        Ml = {__ldcg(&ck[1]), __ldcg(&ck[2]), __ldcg(&ck[3]), __ldcg(&ck[4]),
                              __ldcg(&ck[5]), __ldcg(&ck[6])};
                    } else if (lane == first_inc) {
                        Ml = {0, 0, 0, 0, (k >= 0 ? __ldcg(&ck[8]) : P.entry_p1),
                              (k >= 0 ? __ldcg(&ck[9]) : P.entry_p2)};
                    }
                    // ordered tree: lane 0 ends with M_0 o M_1 o ... o M_31
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        Aff O;
                        O.m11 = __shfl_down_sync(0xffffffffu, Ml.m11, d);
                        O.m12 = __shfl_down_sync(0xffffffffu, Ml.m12, d);
                        O.m21 = __shfl_down_sync(0xffffffffu, Ml.m21, d);
                        O.m22 = __shfl_down_sync(0xffffffffu, Ml.m22, d);
                        O.c1 = __shfl_down_sync(0xffffffffu, Ml.c1, d);
                        O.c2 = __shfl_down_sync(0xffffffffu, Ml.c2, d);
                        if ((lane & (2 * d - 1)) == 0 && lane + d < 32) Ml = aff_compose(Ml, O);
                    }
                    Aff tot;
                    tot.m11 = __shfl_sync(0xffffffffu, Ml.m11, 0);
                    tot.m12 = __shfl_sync(0xffffffffu, Ml.m12, 0);
                    tot.m21 = __shfl_sync(0xffffffffu, Ml.m21, 0);
                    tot.m22 = __shfl_sync(0xffffffffu, Ml.m22, 0);
                    tot.c1 = __shfl_sync(0xffffffffu, Ml.c1, 0);
                    tot.c2 = __shfl_sync(0xffffffffu, Ml.c2, 0);
                    acc = aff_compose(acc, tot);
                    if (inc) {  // acc is constant now (ends in a concrete history)
                        in1 = acc.c1;
                        in2 = acc.c2;
                        break;
                    }
                    base -= 32;
                }
            }
            if (sel == 0 || S->restart) { in1 = 0; in2 = 0; }   // history reset / unused
            if (lane == 0) {
                cw[8] = M.m11 * in1 + M.m12 * in2 + M.c1;
                cw[9] = M.m21 * in1 + M.m22 * in2 + M.c2;
                __threadfence();
                st_release(&cw[0], kFlagInc);
                S->p1 = (long long)in1;
                S->p2 = (long long)in2;
            }
        }
        __syncthreads();
        // ---- finalize, dequantize, store ----
        {
            const unsigned long long p1 = (unsigned long long)S->p1, p2 = (unsigned long long)S->p2;
            const unsigned long long dd = p1 - p2;
            T* y = (T*)P.y + start;
            const int i0 = 4 * g0;
            T out[16];
            if (Tr::F) {
                const double s = decode_scale_code(S->code) * ldexp(1.0, S->fbe);
                const double rs = __ddiv_rn(1.0, s);
#pragma unroll
                for (int i = 0; i < 16; i++) {
                    unsigned long long qv = (unsigned long long)v[i];
                    if (sel == 1) qv += p1;
                    else if (sel == 2) qv += p1 + (unsigned long long)(i0 + i + 1) * dd;
                    const double r = (double)(long long)qv;
                    const double y0 = r * rs;
                    const double ee = __fma_rn(-s, y0, r);
                    out[i] = (T)__fma_rn(ee, rs, y0);
                }
            } else {
                const double a = decode_scale_code(S->code);
                const double ra = __ddiv_rn(1.0, a);
#pragma unroll
                for (int i = 0; i < 16; i++) {
                    unsigned long long qv = (unsigned long long)v[i];
                    if (sel == 1) qv += p1;
                    else if (sel == 2) qv += p1 + (unsigned long long)(i0 + i + 1) * dd;
                    long long yi;
                    if (a == 1.0) yi = (long long)qv;
                    else {
                        const double r = (double)(long long)qv;
                        const double y0 = r * ra;
                        const double ee = __fma_rn(-a, y0, r);
                        yi = f2i64(rint(__fma_rn(ee, ra, y0)));
                    }
                    yi = yi < Tr::LO ? Tr::LO : (yi > Tr::HI ? Tr::HI : yi);
                    out[i] = (T)yi;
                }
            }
            if (i0 + 16 <= n && ((((uintptr_t)(y + i0)) & 15) == 0)) {
                constexpr int PER = 16 / (int)sizeof(T);
#pragma unroll
                for (int c = 0; c < 16 / PER; c++) {
                    uint4 w4;
                    memcpy(&w4, &out[c * PER], 16);
                    __stcs((uint4*)(y + i0) + c, w4);
                }
            } else {
#pragma unroll
                for (int i = 0; i < 16; i++)
                    if (i0 + i < n) y[i0 + i] = out[i];
            }
        }
        __syncthreads();
    }
}

}  // namespace d2

size_t decode_v2_smem_bytes(int dt, int bs, int payload_cap) {
    (void)dt; (void)bs;
    auto al = [](size_t v) { return (v + 127) & ~(size_t)127; };
    return al(sizeof(d2::St)) + al((size_t)d2::MAXBS / 4 + 64) + 2 * al((size_t)payload_cap + 64);
}

bool decode_v2_supported(int bs) { return bs <= d2::MAXBS; }

template <int DT>
static void* d2_fn() { return (void*)d2::decode_v2_kernel<DT>; }
static void* d2_kernel(int dt) {
    switch (dt) {
        case 0: return d2_fn<0>();
        case 1: return d2_fn<1>();
        case 2: return d2_fn<2>();
        case 3: return d2_fn<3>();
        default: return d2_fn<4>();
    }
}

int decode_v2_resident_ctas(int dt, size_t smem) {
    int dev = 0, nsm = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const void* fn = d2_kernel(dt);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, d2::NT, smem) != cudaSuccess || per < 1)
        per = 1;
    return per * (nsm > 0 ? nsm : 148);
}

// aggregate history map of blocks [0, nb): M_{nb-1} o ... o M_0 from the
// per-block maps the decode left in the carry records (cw[1..6])
__global__ void __launch_bounds__(256) compose_maps_kernel(const unsigned long long* carry, long long nb,
                                                           unsigned long long* out) {
    using d2::Aff;
    using d2::aff_compose;
    __shared__ Aff part[256];
    const int t = threadIdx.x;
    const long long per = (nb + 255) / 256;
    const long long k0 = (long long)t * per, k1 = (k0 + per < nb) ? k0 + per : nb;
    Aff acc = {1, 0, 0, 1, 0, 0};
    for (long long k = k0; k < k1; k++) {
        const unsigned long long* c = carry + 16 * k;
        const Aff M = {c[1], c[2], c[3], c[4], c[5], c[6]};
        acc = aff_compose(M, acc);
    }
    part[t] = acc;
    __syncthreads();
    for (int d = 1; d < 256; d <<= 1) {   // ordered: later ranges after earlier ones
        Aff r = part[t];
        if ((t & (2 * d - 1)) == 0 && t + d < 256) r = aff_compose(part[t + d], part[t]);
        __syncthreads();
        part[t] = r;
        __syncthreads();
    }
    if (t == 0) {
        out[0] = part[0].m11; out[1] = part[0].m12; out[2] = part[0].m21;
        out[3] = part[0].m22; out[4] = part[0].c1; out[5] = part[0].c2;
    }
}

int launch_compose_maps(const unsigned long long* carry, long long nb, unsigned long long* out, cudaStream_t st) {
    note_launches(1);
    compose_maps_kernel<<<1, 256, 0, st>>>(carry, nb, out);
    return cudaGetLastError() == cudaSuccess ? APAX_OK : APAX_ERR_CUDA;
}

int launch_decode_v2(int dt, const DecParams& P, int grid, size_t smem, cudaStream_t st) {
    const void* fn = d2_kernel(dt);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return APAX_ERR_CUDA;
    DecParams p = P;
    void* args[] = {&p};
    // cooperative: all CTAs co-resident, so the carry look-back between
    // round-robin neighbours can never wait on an unscheduled CTA
    note_launches(1);
    if (cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(d2::NT), args, smem, st) != cudaSuccess)
        return APAX_ERR_CUDA;
    return APAX_OK;
}

}  // namespace apax
