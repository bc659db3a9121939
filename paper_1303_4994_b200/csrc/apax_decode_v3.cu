// apax_decode_v3.cu -- segment-serial B200 decoder (block sizes 128..4096,
// powers of two) for containers whose segments are known: every
// `segment_blocks`-th block starts a segment (restart flag), as
// written by apax_encode with segment_blocks > 0.
//
// Same bit-exact output as the reference decode_stream
// (pkg/src/apax/codec.py:308-329); the block walk is replaced by the
// side-band offsets.  One CTA decodes a segment's blocks in order, so the
// derivative history (transform.py:31-49) stays in shared memory and no
// cross-block carry protocol is needed; segments are spread over the CTAs.
//
// Blocks go in batches of JB = 8:
//   * JEE (entropy.py:118-164): warp w parses block w of the batch straight
//     from global memory, 4 nibbles per lane and 128 per step (two
//     consecutive non-15 nibbles always precede a token start, so each lane
//     finds its token starts from a 16-nibble window; one warp scan of
//     (count, escape reset, running value) places the exponents); no CTA
//     barrier inside, and any irregularity re-runs the exact parser
//     (apax_jee.cuh) for the reference's status code;
//   * then the CTA decodes the batch's blocks in order (256 threads, 16
//     samples per thread), each block (header + payload) arriving by one TMA
//     bulk copy issued while the previous block was decoded:
//   * mantissa bit offsets: a CTA scan of 4*sum(e) over the thread's 4
//     groups; 32-bit funnel windows + signed bit-field extracts unpack them
//     (entropy.py:249-277);
//   * D1/D2 (transform.py:116-129): one CTA scan of (sum, sum of partial
//     sums) in 64-bit gives each thread its entry values; narrow blocks then
//     run the per-sample sums in 32-bit wrap-around arithmetic (exact: the
//     entry values bound every output inside int32);
//   * dequantize (codec.py:135-146) with the Markstein quotient, y staged in
//     the block's own (now dead) payload buffer (f64: its own buffer), one
//     TMA bulk store per block.
#include <type_traits>
#include <cstdint>
#include <cuda_runtime.h>

#include "apax_device.cuh"
#include "apax_kernels.cuh"
#include "apax_jee.cuh"

#ifndef APAX_D3_MINB
#define APAX_D3_MINB 4
#endif

namespace apax {
namespace d3 {
#ifdef APAX_D3_TIMES
// per-CTA timeline (tools/cta_times_dec.py): globaltimer at start and exit, SM id
__device__ unsigned long long g_times[8192 * 4];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif

constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int SPT = 16;
constexpr int MAXBS = 4096;
constexpr int JB = 8;                                  // blocks per JEE batch (one warp each)
constexpr int EBS = MAXBS / 4 + 128;                   // exponent bytes per batch slot

struct __align__(16) St {
    // block descriptor (thread 0 at issue time) for the two payload buffers
    long long ld_a[2], ld_boff[2], ld_bend[2];
    int ld_tma[2];
    // per-slot header geometry (thread 0 at issue time): pre-header error,
    // header offset in the buffer, payload offset, bytes available / staged
    int ld_err[2], ld_hoff[2], ld_payoff[2], ld_avail[2], ld_staged[2];
    unsigned long long mbar[2];
    // history (q[np-1], q[np-2] of the previous block)
    long long p1, p2;
    // JEE pass state
    int cnt_base, val_base, first_event, used, fallback, err;
    int sc_cnt[NW], sc_flag[NW], sc_val[NW], ev_min[NW];
    unsigned bits_w[NW];
    long long rs_w[NW], rt_w[NW];
    int store_pending;
    int4 jinfo[JB];           // JEE batch per slot: packed header, JEE status (0 ok), nibbles used
    unsigned wbits[JB][8];    // mantissa bits up to the end of each decode warp's 128 groups
    unsigned short tpre[JB][NT];
    double2 dq[JB];           // dequantize scale and its reciprocal per slot   // each thread's mantissa bit offset inside its decode warp
};

using namespace apax::tma;

// a segment's history map x -> A x + c on (p1, p2) over Z / 2^64
struct Aff { unsigned long long a11, a12, a21, a22, c1, c2; };
// (second after first): x -> s(f(x))
__device__ __forceinline__ Aff aff_after(const Aff& s2, const Aff& f) {
    Aff r;
    r.a11 = s2.a11 * f.a11 + s2.a12 * f.a21;
    r.a12 = s2.a11 * f.a12 + s2.a12 * f.a22;
    r.a21 = s2.a21 * f.a11 + s2.a22 * f.a21;
    r.a22 = s2.a21 * f.a12 + s2.a22 * f.a22;
    r.c1 = s2.a11 * f.c1 + s2.a12 * f.c2 + s2.c1;
    r.c2 = s2.a21 * f.c1 + s2.a22 * f.c2 + s2.c2;
    return r;
}

__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(gdst), "r"(sa(ssrc)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ int bfe_s(uint32_t v, int pos, int len) {
    int r;
    asm("bfe.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(v), "r"(pos), "r"(len));
    return r;
}
__device__ __forceinline__ int sar32(int v, uint32_t n) {
    int r;
    asm("shr.s32 %0, %1, %2;" : "=r"(r) : "r"(v), "r"(n));
    return r;
}
__device__ __forceinline__ uint32_t shl32(uint32_t v, uint32_t n) {
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(v), "r"(n));
    return r;
}
// 32 bits of the MSB-first stream starting at bit position bp (word array
// in shared memory, little-endian words holding big-endian bytes)
__device__ __forceinline__ uint32_t r32(const uint32_t* w, int bp) {
    const int k = bp >> 5;
    return __funnelshift_l(bswap32(w[k + 1]), bswap32(w[k]), (unsigned)(bp & 31));
}


// TP: 0 a segmented container; 1 pass 1 of a two-pass decode (segment
// history maps, no samples); 2 pass 2 (segments start from composed entries).
// A template parameter so the segmented hot path carries none of it.
template <int DT, bool FIX, int TP>
__global__ void __launch_bounds__(NT, APAX_D3_MINB) decode_v3_kernel(DecParams P) {
    using Tr = DT_<DT>;
    using T = typename Tr::T;
    constexpr int HS = Tr::HDR;
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bs = FIX ? MAXBS : P.bs;

    St* S = (St*)smem;
    size_t off = (sizeof(St) + 127) & ~(size_t)127;
    uint8_t* ebufs = smem + off;                          // group exponents, JB slots
    off += (size_t)JB * (((size_t)EBS + 127) & ~(size_t)127);
    // decoded block: f64 has its own buffer; narrower types reuse the block's
    // payload buffer, dead once every thread holds its unpacked values
    constexpr bool YOWN = (DT == 4);
    T* ybuf_own = (T*)(smem + off);
    if (YOWN) off += ((size_t)MAXBS * sizeof(T) + 127) & ~(size_t)127;
    const int bufsz = (P.payload_cap + 64 + 127) & ~127;
    uint8_t* pbuf0 = smem + off;
    uint8_t* pbuf1 = smem + off + bufsz;
    const long long limit = P.nbytes & ~15LL;             // TMA never reads past the blob

#ifdef APAX_D3_TIMES
    if (tid == 0 && blockIdx.x < 8192) {
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        g_times[4 * blockIdx.x] = gtimer();
        g_times[4 * blockIdx.x + 3] = smid;
    }
#endif
    if (tid == 0) {
        mbar_init(&S->mbar[0]);
        mbar_init(&S->mbar[1]);
        fence_mbar_init();
        S->store_pending = 0;
    }
    __syncthreads();
    uint32_t phs = 0u;

    long long P_seg = P.segment_blocks;
    long long s_begin = P.seg_begin, s_end = P.seg_end;
    // index-less decode: the speculative segment path (TP 0) or the two-pass
    // decode that replaces it (TP 1, 2) -- exactly one of them runs
    const bool spec = TP == 0 && P.il_gate && !P.il_gate2;
    IlGate* hg = nullptr;   // the gate a segment head without a restart flag clears
    if (P.il_gate) {
        const bool ok1 = il_seg_ok(P.il_gate);
        const bool ok2 = P.il_gate2 && il_seg_ok(P.il_gate2);
        if (TP == 0) {
            if (P.il_gate2 ? (ok1 || !ok2) : !ok1) return;
            hg = P.il_gate2 ? P.il_gate2 : P.il_gate;
            P_seg = (long long)hg->first;
            const long long nseg = (P.n_blocks + P_seg - 1) / P_seg;
            const long long sfull = (P.n % bs) ? nseg - 1 : nseg;
            s_begin = P.seg_part == 2 ? sfull : 0;
            s_end = P.seg_part == 1 ? sfull : nseg;
        } else if (ok1 || ok2) {
            return;
        }
    }

    const bool k5_rec = TP == 1 && P.jee_k5 && P.jee_k5[0] == 0 && P.jee_k5[1] == 0;
    // issue the load of block bb into buffer slot (thread 0)
    auto issue = [&](long long bb, int slot) {
        const long long o0 = P.offsets[bb], o1 = P.offsets[bb + 1];
        const long long hi = o1 > o0 + HS ? o1 : o0 + HS;
        const long long a0 = (o0 >= 0 ? o0 : 0) & ~15LL;
        const long long e1 = (hi + 15) & ~15LL;
        const long long len = e1 - a0;
        S->ld_a[slot] = a0;
        S->ld_boff[slot] = o0;
        S->ld_bend[slot] = o1;
        const bool ok = o0 >= 0 && len > 0 && len <= bufsz && e1 <= limit &&
                        ((((uintptr_t)(P.blob + a0)) & 15) == 0);
        S->ld_tma[slot] = ok ? 1 : 0;
        {
            int derr = 0, hoff = 0, payoff = 0, av = 0, stg = 0;
            if (o0 < 0) derr = APAX_ERR_ARG;
            else if (P.nbytes - o0 < HS) derr = APAX_ERR_BLOCK_HDR_TRUNCATED;
            else {
                const long long ps = o0 + HS;
                const long long pe = o1 > ps ? o1 : ps;
                long long ee = (pe + 15) & ~15LL;
                if (ee > limit) ee = limit;
                long long staged_end = a0 + (ee - a0 < bufsz ? ee - a0 : bufsz);
                if (!ok) staged_end = a0 + min((long long)bufsz, min(pe, P.nbytes) - a0);
                hoff = (int)(o0 - a0);
                payoff = (int)(ps - a0);
                const long long avl = P.nbytes - ps;
                av = (int)(avl < (1LL << 30) ? avl : (1LL << 30));
                stg = (int)(staged_end - ps);
            }
            S->ld_err[slot] = derr; S->ld_hoff[slot] = hoff; S->ld_payoff[slot] = payoff;
            S->ld_avail[slot] = av; S->ld_staged[slot] = stg;
        }
        if (ok) {
            fence_proxy_async();
            tma_load(slot ? pbuf1 : pbuf0, P.blob + a0, (uint32_t)len, &S->mbar[slot]);
        }
    };
    // the first block of this CTA
    if (tid == 0 && s_begin + blockIdx.x < s_end) issue((s_begin + blockIdx.x) * P_seg, 0);
    __syncthreads();

    int kk = 0;   // blocks decoded by this CTA (buffer parity)
    for (long long sg = s_begin + blockIdx.x; sg < s_end; sg += gridDim.x) {
        const long long b0 = sg * P_seg;
        const long long b1 = (b0 + P_seg < P.n_blocks) ? b0 + P_seg : P.n_blocks;
        // history entering the segment: (0, 0) at a restart (a segmented
        // container), or the composed entry of pass 2 of a two-pass decode
        if (TP == 2 && !P.seg_entry) {
            // the entry of segment sg: the maps of segments 0 .. sg-1 (pass 1)
            // applied in order to (0, 0).  Composition is associative: every
            // thread composes a run of maps, the warps and the CTA combine the
            // runs in order (no launch of its own for a few hundred maps)
            Aff acc = {1ULL, 0ULL, 0ULL, 1ULL, 0ULL, 0ULL};
            const long long per = (sg + NT - 1) / NT;
            const long long k1 = ((long long)tid + 1) * per < sg ? ((long long)tid + 1) * per : sg;
            for (long long k = (long long)tid * per; k < k1; k++) {
                const ulonglong2* m = (const ulonglong2*)(P.seg_map + 6 * k);
                const ulonglong2 m0 = m[0], m1 = m[1], m2 = m[2];
                const Aff f = {m0.x, m0.y, m1.x, m1.y, m2.x, m2.y};
                acc = aff_after(f, acc);
            }
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                Aff o;
                o.a11 = __shfl_down_sync(0xffffffffu, acc.a11, d); o.a12 = __shfl_down_sync(0xffffffffu, acc.a12, d);
                o.a21 = __shfl_down_sync(0xffffffffu, acc.a21, d); o.a22 = __shfl_down_sync(0xffffffffu, acc.a22, d);
                o.c1 = __shfl_down_sync(0xffffffffu, acc.c1, d); o.c2 = __shfl_down_sync(0xffffffffu, acc.c2, d);
                if ((lane & (2 * d - 1)) == 0) acc = aff_after(o, acc);   // the later run after the earlier
            }
            Aff* wa = (Aff*)ebufs;
            if (lane == 0) wa[warp] = acc;
            cbar();
            if (tid == 0) {
                Aff tot = wa[0];
#pragma unroll
                for (int w8 = 1; w8 < NW; w8++) tot = aff_after(wa[w8], tot);
                S->p1 = (long long)tot.c1;
                S->p2 = (long long)tot.c2;
            }
            cbar();   // ebufs are the JEE phase's from here on
        } else if (tid == 0) {
            S->p1 = TP == 2 ? (long long)P.seg_entry[2 * sg] : 0;
            S->p2 = TP == 2 ? (long long)P.seg_entry[2 * sg + 1] : 0;
        }
        // pass 1: the segment's history map, A composed block by block (c is
        // the history leaving the segment from a (0, 0) entry)
        unsigned long long A11 = 1, A12 = 0, A21 = 0, A22 = 1;
        for (long long bb = b0; bb < b1; bb += JB) {
        const int nbat = (int)((b1 - bb) < JB ? (b1 - bb) : JB);
        // ---- JEE of the batch (entropy.py:118-164): warp w parses block bb + w
        // from global memory, no CTA barrier inside; the CTA phases below use it
        // pass 2: the parse pass 1 saved; pass 1 of an index-less decode: the
        // parse the block discovery saved (every block but the last, whose
        // group count the discovery did not know)
        const bool rec_load = warp < nbat && P.jee_cache &&
                              (TP == 2 || (TP == 1 && k5_rec && bb + warp + 1 < P.n_blocks));
        if (rec_load) {
            {
                const uint8_t* rec = P.jee_cache + (size_t)(bb + warp) * (size_t)kJeeRecBytes;
                uint8_t* ej = ebufs + (size_t)warp * (((size_t)EBS + 127) & ~(size_t)127);
                if (lane == 0) {
                    S->jinfo[warp] = *(const int4*)rec;
                    S->dq[warp] = *(const double2*)(rec + 16);
                }
                if (lane < 8) S->wbits[warp][lane] = ((const unsigned*)(rec + 32))[lane];
                uint32_t* tp = (uint32_t*)&S->tpre[warp][0];
#pragma unroll
                for (int i = 0; i < 4; i++) tp[lane + 32 * i] = ((const uint32_t*)(rec + 64))[lane + 32 * i];
                ((uint4*)ej)[lane] = ((const uint4*)(rec + 576))[lane];
                ((uint4*)ej)[lane + 32] = ((const uint4*)(rec + 576))[lane + 32];
            }
        } else if (warp < nbat) {
            const long long bj = bb + warp;
            const long long sj = bj * (long long)bs;
            const int nj = FIX ? MAXBS : (int)((P.n - sj) < bs ? (P.n - sj) : bs);
            const int Gj = FIX ? MAXBS / 4 : (nj + 3) >> 2;
            const long long o0 = P.offsets[bj];
            int st = 0, u = 0, hdr = 0;
            unsigned wmax = 64;
            if (o0 >= 0 && P.nbytes - o0 >= HS) {
                // block header (dtypes.py:156-180) packed for the decode phase:
                // selector | restart << 2 | code << 8 | fbe << 24
                if (lane == 0) {
                    const uint8_t* h = P.blob + o0;
                    hdr = (int)(h[0] & 7) | ((int)h[1] << 8) | ((int)h[2] << 16) |
                          (Tr::F ? ((int)h[4] << 24) : 0);
                }
                const long long ps = o0 + HS;
                const long long avl = P.nbytes - ps;
                const int maxj = (3 * Gj + 2) / 2;
                const int nbj = (int)(avl < maxj ? avl : maxj);
                uint8_t* ej = ebufs + (size_t)warp * (((size_t)EBS + 127) & ~(size_t)127);
                st = warp_jee_fast(P.blob + ps, P.blob + P.nbytes, 2 * nbj, Gj, ej, u);
                if (st < 0) {   // exact serial semantics and status code (apax_jee.cuh)
                    long long u2 = 0, esum = 0;
                    st = warp_jee_decode(P.blob + ps, 2LL * nbj, Gj, ej, u2, esum);
                    u = (int)u2;
                }
                if (st == 0) {
                    // mantissa bits (entropy.py:209-219) per decode warp (128 groups
                    // = 4 lanes of 32 here): the decode phase then needs only a warp scan
                    unsigned sb = 0, em = 0, wb[8];
#pragma unroll
                    for (int k = 0; k < 32; k += 4) {
                        const int g = 32 * lane + k;
                        uint32_t ew;
                        if (FIX || g + 4 <= Gj) ew = *(const uint32_t*)(ej + g);
                        else {
                            ew = 0;
                            for (int c = 0; c < 4; c++) ew |= (g + c < Gj ? (uint32_t)ej[g + c] : 0u) << (8 * c);
                        }
                        wb[k >> 2] = 4u * (unsigned)__dp4a(ew, 0x01010101u, 0u);
                        sb += wb[k >> 2];
                        em = __vmaxu4(em, ew);
                    }
                    const unsigned own = sb;
                    // the block's widest group: <= 16 lets the reconstruct scan
                    // carry the value sums in 32 bits (CTA-uniform choice)
                    em = max(max(em & 0xffu, (em >> 8) & 0xffu), max((em >> 16) & 0xffu, em >> 24));
                    wmax = __reduce_max_sync(0xffffffffu, em);
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const unsigned o = __shfl_up_sync(0xffffffffu, sb, d);
                        if (lane >= d) sb += o;
                    }
                    if ((lane & 3) == 3) S->wbits[warp][lane >> 2] = sb;
                    // per decode thread (8 per lane: 4 groups each), relative to its
                    // decode warp (4 lanes here; < 128 * 4 * 34 bits): no scan there
                    const unsigned sx = sb - own;
                    unsigned run = sx - __shfl_sync(0xffffffffu, sx, lane & ~3);
#pragma unroll
                    for (int i = 0; i < 8; i++) { S->tpre[warp][8 * lane + i] = (unsigned short)run; run += wb[i]; }
                }
            }
            if (lane == 0) {
                S->jinfo[warp] = make_int4(hdr, st, u, (int)wmax);
                // codec.py:135-146 scale (floats: times 2^fbe) and the reciprocal
                // the Markstein quotient uses; once per block, not per thread
                const int code = (hdr >> 8) & 0xFFFF;
                const double ds = Tr::F ? decode_scale_code(code) * ldexp(1.0, hdr >> 24) : decode_scale_code(code);
                S->dq[warp] = make_double2(ds, __ddiv_rn(1.0, ds));
            }
            if (TP == 1 && P.jee_cache) {
                // pass 1: save the parse for pass 2 (a block with an error keeps
                // its status in jinfo; the rest of its record is not used)
                __syncwarp();
                uint8_t* rec = P.jee_cache + (size_t)bj * (size_t)kJeeRecBytes;
                const uint8_t* ej = ebufs + (size_t)warp * (((size_t)EBS + 127) & ~(size_t)127);
                if (lane == 0) {
                    *(int4*)rec = S->jinfo[warp];
                    *(double2*)(rec + 16) = S->dq[warp];
                }
                if (lane < 8) ((unsigned*)(rec + 32))[lane] = S->wbits[warp][lane];
                const uint32_t* tp = (const uint32_t*)&S->tpre[warp][0];
#pragma unroll
                for (int i = 0; i < 4; i++) ((uint32_t*)(rec + 64))[lane + 32 * i] = tp[lane + 32 * i];
                ((uint4*)(rec + 576))[lane] = ((const uint4*)ej)[lane];
                ((uint4*)(rec + 576))[lane + 32] = ((const uint4*)ej)[lane + 32];
            }
        }
        cbar();
        for (int kb = 0; kb < nbat; kb++, kk++) {
            const long long b = bb + kb;
            uint8_t* ebuf = ebufs + (size_t)kb * (((size_t)EBS + 127) & ~(size_t)127);
            const int cur = kk & 1;
            uint8_t* pay = cur ? pbuf1 : pbuf0;
            const long long start = b * (long long)bs;
            const int n = FIX ? MAXBS : (int)((P.n - start) < bs ? (P.n - start) : bs);
            const int G = FIX ? MAXBS / 4 : (n + 3) >> 2;
            const int np = FIX ? MAXBS : 4 * G;
            // prefetch the next block of this CTA
            if (tid == 0) {
                long long nb = -1;
                if (b + 1 < b1) nb = b + 1;
                else if (sg + gridDim.x < s_end) nb = (sg + gridDim.x) * P_seg;
                // the other buffer may still be read by the previous block's y store
                if (!YOWN && S->store_pending) { bulk_wait_read(); S->store_pending = 0; }
                if (nb >= 0) issue(nb, cur ^ 1);
            }
            const bool was_tma = S->ld_tma[cur] != 0;
            const long long a0 = S->ld_a[cur];
            const long long boff = S->ld_boff[cur];
            const long long bend = S->ld_bend[cur];
            if (was_tma) {
                mbar_wait(&S->mbar[cur], (phs >> cur) & 1u);
                phs ^= 1u << cur;
            } else if (boff >= 0) {
                long long hi = bend > boff + HS ? bend : boff + HS;
                long long e1 = hi < P.nbytes ? hi : P.nbytes;
                long long len = e1 - a0;
                if (len > bufsz) len = bufsz;
                for (long long i = tid; i < len; i += NT) pay[i] = P.blob[a0 + i];
                cbar();
            }
            // ---- block header (dtypes.py:156-180), read by every thread ----
            // (header and JEE results: from the batch's warp, one 16-byte read)
            int err = S->ld_err[cur];
            const int pay_off = S->ld_payoff[cur], avail = S->ld_avail[cur], staged = S->ld_staged[cur];
            const int4 ji = S->jinfo[kb];
            const int sel = ji.x & 3, restart = (ji.x >> 2) & 1;   // scale code, fbe: S->dq
            // speculative segments: a segment head without a restart flag
            // sends the container to the two-pass decode
            if (hg && b == b0 && b0 > 0 && !restart && tid == 0) atomicExch(&hg->gp, 0u);
            if (!err) err = (sel == 3) ? APAX_ERR_SELECTOR : ji.y;
            const int used = ji.z;
            const bool bnarrow = ji.w <= 16;
            const int jee_bytes = (used + 1) >> 1;
            // ---- mantissa offsets (entropy.py:209-219): CTA scan of 4*sum(e) ----
            const int g0 = 4 * tid;
            const bool active = FIX ? true : (g0 < G);
            uint32_t epk = 0;
            if (!err && active) {
                if (FIX || g0 + 4 <= G) epk = *(const uint32_t*)(ebuf + g0);
                else
                    for (int g = 0; g < 4; g++) epk |= (g0 + g < G ? (uint32_t)ebuf[g0 + g] : 0u) << (8 * g);
            }
            // bit offsets from the JEE warp (S->wbits, S->tpre): no scan here
            const unsigned btot = err ? 0u : S->wbits[kb][NW - 1];
            const unsigned bpre = err ? 0u : (warp == 0 ? 0u : S->wbits[kb][warp - 1]) + (unsigned)S->tpre[kb][tid];
            if (!err) {
                const long long mant_bytes = ((long long)btot + 7) / 8;
                if (avail < jee_bytes + mant_bytes) err = APAX_ERR_MANTISSA_TRUNCATED;
                else if (jee_bytes + mant_bytes > staged) err = APAX_ERR_ARG;   // offsets inconsistent
                else if (spec) {
                    // the walk's recurrence (codec.py:317-323) on the speculative
                    // offsets: block b ends where block b + 1 starts
                    const long long bend_true = boff + HS + jee_bytes + mant_bytes;
                    if (b + 1 < P.n_blocks) {
                        if (bend_true != bend) err = -2;
                    } else if (tid == 0) {
                        ((long long*)P.offsets)[P.n_blocks] = bend_true;
                    }
                }
            }
            if (err) {
                // speculative offsets: any error or inconsistency hands the
                // container to the full discovery, which reports the
                // reference's error
                if (tid == 0) {
                    if (spec) atomicExch(&P.il_gate->gp, 0u);
                    else if (err > 0) report_error(P.status, b, err);
                }
                cbar();
                continue;
            }
            // ---- unpack, reconstruct, dequantize ----
            const unsigned wm = max(max(epk & 0xffu, (epk >> 8) & 0xffu), max((epk >> 16) & 0xffu, epk >> 24));
            // warp-uniform: every group width <= 16, so |v| < 2^15 and the
            // thread sums below are exact in 32 bits
            const bool narrow = !__any_sync(0xffffffffu, wm > 16);
            const long long p1 = S->p1, p2 = S->p2;
            const unsigned long long h1 = restart ? 0ULL : (unsigned long long)p1;
            const unsigned long long h2 = restart ? 0ULL : (unsigned long long)p2;
            const int i0 = SPT * tid;
            const int j1 = (np - 1) % SPT;            // outgoing history: q[np-1], q[np-2] (padded block)
            const bool hist_thread = tid == (np - 1) / SPT;
            // CTA exclusive prefix of the thread aggregates (s = sum v, t = sum of
            // local partial sums); ranges compose as (s, t, m): A then B =
            // (sA+sB, tA+tB+mB*sA, mA+mB) (transform.py:116-129 as a scan)
            // The count m of a range is implied by the lanes it covers (the B side of
            // step d spans d lanes / warps), so only s and t travel.  VS is the
            // type of s: 32 bits when the block's widest group is <= 16 (|CTA sum|
            // < 4096 * 2^15), else 64.
            // WT (compile time): carry t (D2); D1 needs the value prefix only.
            // VT: the type of the warp-level t (32 bits when the block's widest
            // group is <= 14: a warp's weighted sum is < 512 * 513 / 2 * 2^13 < 2^31).
            auto recon_scan = [&](auto s, auto t, unsigned long long& ps, unsigned long long& pt,
                                  auto wt_tag) {
                constexpr bool wt = decltype(wt_tag)::value;
                using VS = decltype(s);
                using VT = decltype(t);
                auto wide = [](VS v) -> unsigned long long { return (unsigned long long)(long long)v; };
                auto widet = [](VT v) -> unsigned long long { return (unsigned long long)(long long)v; };
                VS xs = s;
                VT xt = t;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const VS os = __shfl_up_sync(0xffffffffu, xs, d);
                    if constexpr (wt) {
                        const VT ot = __shfl_up_sync(0xffffffffu, xt, d);
                        if (lane >= d) xt = ot + xt + (VT)(d * SPT) * (VT)os;
                    }
                    if (lane >= d) xs += os;
                }
                if (lane == 31) { S->rs_w[warp] = (long long)xs; S->rt_w[warp] = (long long)xt; }
                cbar();
                VS ws = (lane < NW) ? (VS)S->rs_w[lane & (NW - 1)] : (VS)0;
                unsigned long long wtt = (wt && lane < NW) ? (unsigned long long)S->rt_w[lane & (NW - 1)] : 0ULL;
#pragma unroll
                for (int d = 1; d < NW; d <<= 1) {
                    const VS os = __shfl_up_sync(0xffffffffu, ws, d);
                    if constexpr (wt) {
                        const unsigned long long ot = __shfl_up_sync(0xffffffffu, wtt, d);
                        if (lane >= d) wtt = ot + wtt + (unsigned long long)(d * 32 * SPT) * wide(os);
                    }
                    if (lane >= d) ws += os;
                }
                VS es = __shfl_up_sync(0xffffffffu, ws, 1);
                unsigned long long et = wt ? __shfl_up_sync(0xffffffffu, wtt, 1) : 0ULL;
                if (lane == 0) { es = 0; et = 0; }
                const VS pws = __shfl_sync(0xffffffffu, es, warp);
                const unsigned long long pwt = wt ? __shfl_sync(0xffffffffu, et, warp) : 0ULL;
                VS ls = __shfl_up_sync(0xffffffffu, xs, 1);
                unsigned long long lt = wt ? widet(__shfl_up_sync(0xffffffffu, xt, 1)) : 0ULL;
                if (lane == 0) { ls = 0; lt = 0; }
                ps = wide(pws) + wide(ls);
                pt = pwt + lt + (unsigned long long)(lane * SPT) * wide(pws);
            };
            // dequantize one reconstructed sample (codec.py:135-146): Markstein
            // quotient against a per-block reciprocal, bit-identical to IEEE
            // division (profiles/r1_markstein_division_check.txt)
            const double2 dqv = S->dq[kb];
            const double dq_s = dqv.x, dq_r = dqv.y;
            auto deq = [&](double r) -> T {
                if (Tr::F) {
                    const double y0 = r * dq_r;
                    const double ee = __fma_rn(-dq_s, y0, r);
                    return (T)__fma_rn(ee, dq_r, y0);
                } else {
                    long long yi = (long long)r;
                    if (dq_s != 1.0) {
                        const double y0 = r * dq_r;
                        const double ee = __fma_rn(-dq_s, y0, r);
                        yi = f2i64(rint(__fma_rn(ee, dq_r, y0)));
                    }
                    yi = yi < Tr::LO ? Tr::LO : (yi > Tr::HI ? Tr::HI : yi);
                    return (T)yi;
                }
            };
            // I2F.F64 on the conversion pipe: the magic-number form cost an ALU
            // op per sample on the decoder's busiest pipe
            auto i2d = [](int v) -> double { return (double)v; };
            T out[SPT];
            constexpr bool want_y = TP != 1;   // pass 1 of a two-pass decode needs the history only
            const uint32_t* w = (const uint32_t*)pay;
            int bp = 8 * ((int)pay_off + jee_bytes) + (int)bpre;
            if (narrow) {
                int v[SPT];
#pragma unroll
                for (int g = 0; g < 4; g++) {   // two 32-bit windows per group
                    const int wd = (int)((epk >> (8 * g)) & 0xffu);
                    // sign-extending shifts (PTX: shifts >= 32 saturate); a zero
                    // width zeroes the windows instead of selecting every value
                    const uint32_t c0 = wd ? r32(w, bp) : 0u, c1 = wd ? r32(w, bp + 2 * wd) : 0u;
                    const uint32_t rs = 32u - (uint32_t)wd;
                    v[4 * g + 0] = sar32((int)c0, rs);
                    v[4 * g + 1] = sar32((int)shl32(c0, (uint32_t)wd), rs);
                    v[4 * g + 2] = sar32((int)c1, rs);
                    v[4 * g + 3] = sar32((int)shl32(c1, (uint32_t)wd), rs);
                    bp += 4 * wd;
                }
                unsigned long long q0 = 0, d0 = 0;   // q and d1 entering this thread (exact, 64-bit)
                if (TP == 1 && bnarrow && sel >= 1) {
                    // pass 1 needs only the history leaving the block: the last
                    // sample of D1 is h1 + sum v, of D2 h1 + np (h1 - h2) +
                    // sum (np - i) v_i, the one before it follows from the last
                    // difference -- CTA sums instead of the scan (widths <= 16:
                    // the warp sums fit 32 bits; the totals are exact mod 2^64)
                    int s32 = 0, t32 = 0;
#pragma unroll
                    for (int i = 0; i < SPT; i++) { s32 += v[i]; t32 += s32; }
                    const long long bq = (long long)(np - i0 - SPT) * (long long)s32 + (long long)t32;
                    const int aw = __reduce_add_sync(0xffffffffu, s32);
                    const unsigned blo = __reduce_add_sync(0xffffffffu, (unsigned)(bq & 0xffff));
                    const int bhi = __reduce_add_sync(0xffffffffu, (int)(bq >> 16));
                    if (lane == 0) {
                        S->rs_w[warp] = (long long)aw;
                        S->rt_w[warp] = (long long)bhi * 65536LL + (long long)blo;
                    }
                    cbar();
                    if (hist_thread) {
                        unsigned long long A = 0, B = 0;
#pragma unroll
                        for (int w8 = 0; w8 < NW; w8++) {
                            A += (unsigned long long)S->rs_w[w8];
                            B += (unsigned long long)S->rt_w[w8];
                        }
                        int vlast = 0;
#pragma unroll
                        for (int i = 0; i < SPT; i++)
                            if (i == j1) vlast = v[i];
                        unsigned long long P1, P2;
                        if (sel == 1) {
                            P1 = h1 + A;
                            P2 = P1 - (unsigned long long)(long long)vlast;
                        } else {
                            const unsigned long long dl = (h1 - h2) + A;
                            P1 = h1 + (unsigned long long)np * (h1 - h2) + B;
                            P2 = P1 - dl;
                        }
                        S->p1 = (long long)P1;
                        S->p2 = (long long)P2;
                    }
                } else {
                if (sel >= 1) {
                    int s32 = 0, t32 = 0;
#pragma unroll
                    for (int i = 0; i < SPT; i++) { s32 += v[i]; t32 += s32; }
                    unsigned long long ps, pt;
                    const unsigned long long t64 = (unsigned long long)(long long)t32;
                    if (sel == 1) {
                        if (bnarrow) recon_scan(s32, t32, ps, pt, std::false_type{});
                        else recon_scan((long long)s32, t64, ps, pt, std::false_type{});
                    } else {
                        if (ji.w <= 14) recon_scan(s32, t32, ps, pt, std::true_type{});
                        else if (bnarrow) recon_scan(s32, t64, ps, pt, std::true_type{});
                        else recon_scan((long long)s32, t64, ps, pt, std::true_type{});
                    }
                    if (sel == 1) {
                        q0 = h1 + ps;
                    } else {
                        d0 = (h1 - h2) + ps;
                        q0 = h1 + (unsigned long long)i0 * (h1 - h2) + pt;
                    }
                }
                // the 16 outputs stay inside int32 when |q0| + 16|d0| + 136 * 2^15 < 2^31:
                // then 32-bit wrap-around arithmetic gives the exact values
                const long long aq = (long long)q0 < 0 ? -(long long)q0 : (long long)q0;
                const long long ad = (long long)d0 < 0 ? -(long long)d0 : (long long)d0;
                const bool fits = sel == 0 || (aq < (1LL << 30) && ad < (1LL << 24));
                if (fits) {
                    // selector-specialised loops (a per-sample select costs as much as the sums)
                    if (sel == 1) {
                        int qa = (int)q0;
#pragma unroll
                        for (int i = 0; i < SPT; i++) { qa += v[i]; v[i] = qa; }
                    } else if (sel == 2) {
                        int qa = (int)q0, da = (int)d0;
#pragma unroll
                        for (int i = 0; i < SPT; i++) { da += v[i]; qa += da; v[i] = qa; }
                    }
                    if (hist_thread) {
#pragma unroll
                        for (int i = 0; i < SPT; i++) {
                            if (i == j1) S->p1 = v[i];
                            if (i == j1 - 1) S->p2 = v[i];
                        }
                    }
                    if (want_y) {
#pragma unroll
                        for (int i = 0; i < SPT; i++) out[i] = deq(i2d(v[i]));
                    }
                } else {
                    unsigned long long qa = q0, da = d0;
#pragma unroll
                    for (int i = 0; i < SPT; i++) {
                        long long qv;
                        if (sel == 1) { qa += (unsigned long long)(long long)v[i]; qv = (long long)qa; }
                        else { da += (unsigned long long)(long long)v[i]; qa += da; qv = (long long)qa; }
                        if (hist_thread && i == j1) S->p1 = qv;
                        if (hist_thread && i == j1 - 1) S->p2 = qv;
                        if (want_y) out[i] = deq((double)qv);
                    }
                }
                }   // scan path
            } else {
                long long q[SPT];
#pragma unroll
                for (int g = 0; g < 4; g++) {
                    const int wd = (int)((epk >> (8 * g)) & 0xffu);
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        const int pb = bp + k * wd;
                        if (wd == 0) q[4 * g + k] = 0;
                        else if (wd <= 32) q[4 * g + k] = bfe_s(r32(w, pb), 32 - wd, wd);
                        else {
                            const unsigned long long hi = ((unsigned long long)r32(w, pb) << 32) | r32(w, pb + 32);
                            q[4 * g + k] = (long long)hi >> (64 - wd);
                        }
                    }
                    bp += 4 * wd;
                }
                if (sel >= 1) {
                    unsigned long long s = 0, t = 0;
#pragma unroll
                    for (int i = 0; i < SPT; i++) { s += (unsigned long long)q[i]; t += s; }
                    unsigned long long ps, pt;
                    if (sel == 1) recon_scan((long long)s, t, ps, pt, std::false_type{});
                    else recon_scan((long long)s, t, ps, pt, std::true_type{});
                    if (sel == 1) {
                        unsigned long long acc = h1 + ps;
#pragma unroll
                        for (int i = 0; i < SPT; i++) { acc += (unsigned long long)q[i]; q[i] = (long long)acc; }
                    } else {
                        unsigned long long d1 = (h1 - h2) + ps;
                        unsigned long long acc = h1 + (unsigned long long)i0 * (h1 - h2) + pt;
#pragma unroll
                        for (int i = 0; i < SPT; i++) {
                            d1 += (unsigned long long)q[i];
                            acc += d1;
                            q[i] = (long long)acc;
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < SPT; i++) {
                    if (hist_thread && i == j1) S->p1 = q[i];
                    if (hist_thread && i == j1 - 1) S->p2 = q[i];
                    const long long qv = q[i];
                    if (want_y) out[i] = deq(qv == (long long)(int)qv ? i2d((int)qv) : (double)qv);
                }
            }
            // ---- y staged in shared memory, one TMA bulk store per block ----
            if (TP == 1 && tid == 0) {
                // the block's history map (transform.py:116-129): D0 and
                // restart blocks forget the entry; D1 adds it; D2 adds a line
                unsigned long long b11, b12, b21, b22;
                const unsigned long long unp = (unsigned long long)np;
                if (sel == 0 || restart) { b11 = b12 = b21 = b22 = 0; }
                else if (sel == 1) { b11 = 1; b12 = 0; b21 = 1; b22 = 0; }
                else { b11 = unp + 1; b12 = 0ULL - unp; b21 = unp; b22 = 0ULL - (unp - 1); }
                const unsigned long long n11 = b11 * A11 + b12 * A21, n12 = b11 * A12 + b12 * A22;
                const unsigned long long n21 = b21 * A11 + b22 * A21, n22 = b21 * A12 + b22 * A22;
                A11 = n11; A12 = n12; A21 = n21; A22 = n22;
            }
            T* ybuf = YOWN ? ybuf_own : (T*)pay;
            if (YOWN && tid == 0 && S->store_pending) { bulk_wait_read(); S->store_pending = 0; }
            // the y buffer is free: the previous store has read it (f64); the payload
            // is unpacked by every thread (D1/D2: the reconstruct scan's barrier did it)
            if (YOWN || sel == 0) cbar();
            if (active && want_y) {
                constexpr int PER = 16 / (int)sizeof(T);
                uint4* y4 = (uint4*)(ybuf + SPT * tid);
#pragma unroll
                for (int c = 0; c < SPT / PER; c++) {
                    uint4 w4;
                    memcpy(&w4, &out[c * PER], 16);
                    y4[c] = w4;
                }
            }
            fence_proxy_async();
            cbar();
            if (tid == 0 && want_y) {
                T* y = (T*)P.y + start;
                const int bytes = n * (int)sizeof(T);
                const int full = bytes & ~15;
                if (full > 0 && (((uintptr_t)y) & 15) == 0) {
                    bulk_store(y, ybuf, (uint32_t)full);
                    S->store_pending = 1;
                    for (int i = full; i < bytes; i++) ((uint8_t*)y)[i] = ((const uint8_t*)ybuf)[i];
                } else {
                    for (int i = 0; i < bytes; i++) ((uint8_t*)y)[i] = ((const uint8_t*)ybuf)[i];
                }
            }
        }   // blocks of the batch
        }   // batches
        if (TP == 1 && tid == 0) {   // S->p1/p2 are final: the last block's barriers ordered them
            unsigned long long* m = P.seg_map + 6 * sg;
            m[0] = A11; m[1] = A12; m[2] = A21; m[3] = A22;
            m[4] = (unsigned long long)S->p1; m[5] = (unsigned long long)S->p2;
        }
    }
    if (tid == 0 && S->store_pending) bulk_wait_all();
#ifdef APAX_D3_TIMES
    if (tid == 0 && blockIdx.x < 8192) g_times[4 * blockIdx.x + 2] = gtimer();
#endif
}

}  // namespace d3

#ifdef APAX_D3_TIMES
extern "C" int apax_debug_cta_times_d3(unsigned long long* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, d3::g_times, (size_t)n * 4 * sizeof(unsigned long long));
}
#endif

size_t decode_v3_smem_bytes(int dt, int payload_cap) {
    auto al = [](size_t v) { return (v + 127) & ~(size_t)127; };
    return al(sizeof(d3::St)) + (size_t)d3::JB * al((size_t)d3::EBS) + (dt == 4 ? al((size_t)d3::MAXBS * 8) : 0) +
           2 * (size_t)((payload_cap + 64 + 127) & ~127);
}

bool decode_v3_supported(int dt, int bs) {
    return dt >= 0 && dt <= 4 && bs >= 128 && bs <= d3::MAXBS && (bs & (bs - 1)) == 0;
}

template <int DT, bool FIX>
static void* d3_fn(int tp) {
    return tp == 1 ? (void*)d3::decode_v3_kernel<DT, FIX, 1>
                   : (tp == 2 ? (void*)d3::decode_v3_kernel<DT, FIX, 2> : (void*)d3::decode_v3_kernel<DT, FIX, 0>);
}
static void* d3_kernel(int dt, bool fix, int tp = 0) {
    switch (dt) {
        case 0: return d3_fn<0, false>(tp);
        case 1: return fix ? d3_fn<1, true>(tp) : d3_fn<1, false>(tp);
        case 2: return fix ? d3_fn<2, true>(tp) : d3_fn<2, false>(tp);
        case 3: return fix ? d3_fn<3, true>(tp) : d3_fn<3, false>(tp);
        default: return fix ? d3_fn<4, true>(tp) : d3_fn<4, false>(tp);
    }
}

int decode_v3_resident_ctas(int dt, size_t smem) {
    int dev = 0, nsm = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const void* fn = d3_kernel(dt, false);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, d3::NT, smem) != cudaSuccess || per < 1)
        per = 1;
    return per * (nsm > 0 ? nsm : 148);
}

static int launch_d3_range(int dt, bool fix, const DecParams& P, long long s0, long long s1, int grid,
                           size_t smem, cudaStream_t st, int tp) {
    const void* fn = d3_kernel(dt, fix, tp);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return APAX_ERR_CUDA;
    DecParams p = P;
    p.seg_begin = s0;
    p.seg_end = s1;
    const long long ns = s1 - s0;
    const int g = (int)(ns < grid ? ns : grid);
    void* args[] = {&p};
    note_launches(1);
    if (cudaLaunchKernel(fn, dim3(g), dim3(d3::NT), args, smem, st) != cudaSuccess) return APAX_ERR_CUDA;
    return APAX_OK;
}

// entries of a two-pass decode: e_0 = (0, 0), e_{k+1} = F_k(e_k).  The maps
// are affine on (p1, p2) over Z / 2^64 and composition is associative, so the
// entries are the translation parts of the prefix compositions: a scan in
// shared memory, 512 segments at a time (one thread walking the maps in
// global memory took 172 us for 592 segments: longer than a decode pass).
constexpr int CE_T = 512;
using d3::Aff;
using d3::aff_after;
__global__ void __launch_bounds__(CE_T) compose_entries_kernel(const unsigned long long* maps, long long nseg,
                                                               unsigned long long* entries, const IlGate* gate,
                                                               const IlGate* gate2) {
    if (gate && (il_seg_ok(gate) || (gate2 && il_seg_ok(gate2)))) return;
    __shared__ Aff sm[CE_T];
    __shared__ Aff carry;     // composition of every segment before this chunk
    const int tid = threadIdx.x;
    if (tid == 0) { carry.a11 = 1; carry.a12 = 0; carry.a21 = 0; carry.a22 = 1; carry.c1 = 0; carry.c2 = 0; }
    for (long long base = 0; base < nseg; base += CE_T) {
        const long long k = base + tid;
        Aff me;
        if (k < nseg) {
            const unsigned long long* m = maps + 6 * k;
            me.a11 = m[0]; me.a12 = m[1]; me.a21 = m[2]; me.a22 = m[3]; me.c1 = m[4]; me.c2 = m[5];
        } else {
            me.a11 = 1; me.a12 = 0; me.a21 = 0; me.a22 = 1; me.c1 = 0; me.c2 = 0;
        }
        sm[tid] = me;
        __syncthreads();
        for (int d = 1; d < CE_T; d <<= 1) {      // inclusive scan: me = F_k after ... after F_base
            Aff prev;
            const bool has = tid >= d;
            if (has) prev = sm[tid - d];
            __syncthreads();
            if (has) { me = aff_after(me, prev); sm[tid] = me; }
            __syncthreads();
        }
        const Aff c = carry;
        // the entry of segment k: every earlier segment applied to (0, 0)
        if (k < nseg) {
            unsigned long long e1 = c.c1, e2 = c.c2;
            if (tid > 0) {
                const Aff g = aff_after(sm[tid - 1], c);
                e1 = g.c1; e2 = g.c2;
            }
            entries[2 * k] = e1;
            entries[2 * k + 1] = e2;
        }
        __syncthreads();
        if (tid == CE_T - 1) carry = aff_after(me, c);
        __syncthreads();
    }
}

static int launch_decode_v3_tp(int dt, const DecParams& P, int grid, size_t smem, cudaStream_t st, int tp);

// any container through d3: pseudo-segments of P blocks (one wave), pass 1
// for their history maps, a sequential composition, pass 2 with the entries
int launch_decode_v3_two_pass(int dt, DecParams P, int grid, size_t smem, unsigned long long* scratch,
                              cudaStream_t st) {
    const long long seg = (P.n_blocks + grid - 1) / grid;
    const long long nseg = (P.n_blocks + seg - 1) / seg;
    unsigned long long* maps = scratch;
    unsigned long long* entries = scratch + 6 * nseg;
    P.segment_blocks = seg;
    P.seg_map = maps;
    P.seg_entry = nullptr;
    P.no_store = 1;
    int r = launch_decode_v3_tp(dt, P, grid, smem, st, 1);
    if (r) return r;
    // the entries: composed by pass 2's CTAs themselves, or (APAX_D3_COMPOSE=1)
    // by a scan kernel of its own
    const char* ce = getenv("APAX_D3_COMPOSE");
    if (ce && atoi(ce) == 1) {
        note_launches(1);
        compose_entries_kernel<<<1, CE_T, 0, st>>>(maps, nseg, entries, P.il_gate, P.il_gate2);
        if (cudaGetLastError() != cudaSuccess) return APAX_ERR_CUDA;
        P.seg_map = nullptr;
        P.seg_entry = entries;
    } else {
        P.seg_entry = nullptr;   // maps stay in P.seg_map
    }
    P.no_store = 0;
    return launch_decode_v3_tp(dt, P, grid, smem, st, 2);
}

// index-less segment path: P.il_gate set, the segment length
// and count read on the device (full-block segments on the compile-time-
// geometry kernel, the segment with a partial last block on the generic one)
int launch_decode_v3_seg_dev(int dt, DecParams P, int grid, size_t smem, cudaStream_t st) {
    const bool fixable = P.bs == d3::MAXBS && dt >= 1 && dt <= 4;
    const bool partial = (P.n % P.bs) != 0;
    P.segment_blocks = 1;
    P.seg_begin = 0;
    P.seg_end = 0;
    if (fixable) {
        P.seg_part = partial ? 1 : 0;
        const void* fn = d3_kernel(dt, true, 0);
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return APAX_ERR_CUDA;
        void* args[] = {&P};
        note_launches(1);
        if (cudaLaunchKernel(fn, dim3(grid), dim3(d3::NT), args, smem, st) != cudaSuccess) return APAX_ERR_CUDA;
        if (!partial) return APAX_OK;
    }
    P.seg_part = fixable ? 2 : 0;
    const void* fn = d3_kernel(dt, false, 0);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return APAX_ERR_CUDA;
    void* args[] = {&P};
    note_launches(1);
    if (cudaLaunchKernel(fn, dim3(fixable ? 1 : grid), dim3(d3::NT), args, smem, st) != cudaSuccess)
        return APAX_ERR_CUDA;
    return APAX_OK;
}

int launch_decode_v3(int dt, const DecParams& P, int grid, size_t smem, cudaStream_t st) {
    return launch_decode_v3_tp(dt, P, grid, smem, st, 0);
}

static int launch_decode_v3_tp(int dt, const DecParams& P, int grid, size_t smem, cudaStream_t st, int tp) {
    const long long nseg = (P.n_blocks + P.segment_blocks - 1) / P.segment_blocks;
    // full-block segments take the compile-time-geometry kernel; the segment
    // holding a partial last block follows in a generic launch
    const bool fixable = P.bs == d3::MAXBS && dt >= 1 && dt <= 4;
    long long sfull = fixable ? nseg : 0;
    if (fixable && (P.n % d3::MAXBS) != 0) sfull = nseg - 1;
    if (sfull > 0) {
        const int r = launch_d3_range(dt, true, P, 0, sfull, grid, smem, st, tp);
        if (r) return r;
    }
    if (sfull < nseg) return launch_d3_range(dt, false, P, sfull, nseg, grid, smem, st, tp);
    return APAX_OK;
}

}  // namespace apax
