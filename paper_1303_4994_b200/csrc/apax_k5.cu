// apax_k5.cu -- index-less parallel block discovery (K5, SURVEY.md §7 hard
// part 4): the block offsets of a container without a side-band index.
//
// The reference finds block boundaries with a serial walk (codec.py:317-323):
// parse block b's header + JEE stream + mantissa length, step to block b+1.
// A B200 warp doing that walk reaches ~1 GB/s.  K5 instead parses every
// byte position that *could* start a block, in parallel, and recovers the
// walk's chain from the candidates:
//
//   1. signature scan: a block written by the encoder has header byte 0 in
//      {0,1,2,4,5,6} (selector | restart << 2, dtypes.py:156-165), byte 3 =
//      0, byte 5 = 0 for float dtypes, and its payload opens with the JEE
//      escape nibble 15 followed by the high nibble of an exponent <= 34
//      (entropy.py:60-64) -> first payload byte in {F0,F1,F2}.  One pass:
//      16 positions per thread from 24 loaded bytes with SIMD byte compares,
//      the (rare) matches of a chunk sorted in shared memory and placed in
//      position order after the chunks before it by decoupled look-back;
//   2. one warp per candidate runs the same exact JEE parse as the walk
//      (warp_jee_decode) with a full block's group count and records the
//      position of the following block (next[]), or -1 on any error;
//   3. fast path: when every candidate is a block (count == n_blocks, the
//      usual case) and each points at the next, the candidates are the
//      offsets.  Otherwise candidates nobody points at (other than the head
//      at byte 28) are dropped, twice; the survivors in position order are
//      the chain (these kernels return at once on the fast path);
//   4. verification: survivor b sits at the position survivor b-1 points to,
//      for every b < n_blocks, and survivor 0 is at byte 28.  That is
//      exactly the serial walk's recurrence, so the offsets are the walk's.
//
// The last block (its group count may be smaller) and every anomaly --
// candidate overflow, a break in the chain, a parse error anywhere on the
// path -- are handed to the serial walk kernel (apax_decode.cu), which then
// reproduces the reference's exact error and its block index.  Candidate
// rates on codec output are ~1e-9/byte (float) and ~1e-6/byte (int), so the
// chain is almost always whole.
#include <cstdint>
#include <cuda_runtime.h>

#include "apax_device.cuh"
#include "apax_jee.cuh"
#include "apax_kernels.cuh"

namespace apax {
namespace k5 {

constexpr int NT = 256;
constexpr int NW = NT / 32;

struct Hdr {
    unsigned long long ncand;   // candidates found (may exceed cap -> fail)
    unsigned long long nkept;
    int fail;
    int chain_bad;              // the fast path did not hold: prune
    unsigned int barrier;       // scan_place_kernel's grid barrier
    int pad;
};

constexpr int LBMAX = 4096;    // scan CTAs at most
constexpr int SCB = 16384;     // bytes per scan chunk (one TMA bulk copy)
constexpr int KCAP = 1024;     // candidates of one chunk held in shared memory
constexpr int KSTAGE = 2048;   // staged bytes per parse warp (>= 16 + 1537 + 8 for 4096-sample blocks)
constexpr int KREC = 32 + 512;  // per parse warp: the record's warp bits and thread bit offsets

struct Ws {
    Hdr* hdr;
    long long* cpos;              // cap
    long long* cnext;             // cap
    int* succ;                    // cap
    uint8_t* keep0;               // cap
    uint8_t* keep1;               // cap
    int* nodeidx;                 // n_blocks
    unsigned* ctot;               // LBMAX candidates per scan CTA
    long long cap;
};

static size_t al(size_t v) { return (v + 255) & ~(size_t)255; }

static long long cap_for(long long n_blocks) { return 2 * n_blocks + 4096; }

static size_t layout(long long n_blocks, uint8_t* base, Ws* w) {
    const long long cap = cap_for(n_blocks);
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t at = o; o += al(bytes); return base ? base + at : nullptr; };
    uint8_t* h = take(sizeof(Hdr));
    uint8_t* ccp = take((size_t)LBMAX * 4);
    uint8_t* cp = take((size_t)cap * 8);
    uint8_t* cn = take((size_t)cap * 8);
    uint8_t* su = take((size_t)cap * 4);
    uint8_t* k0 = take((size_t)cap);
    uint8_t* k1 = take((size_t)cap);
    uint8_t* ni = take((size_t)(n_blocks > 0 ? n_blocks : 1) * 4);
    if (w) {
        w->ctot = (unsigned*)ccp;
        w->hdr = (Hdr*)h;
        w->cpos = (long long*)cp; w->cnext = (long long*)cn; w->succ = (int*)su;
        w->keep0 = k0; w->keep1 = k1; w->nodeidx = (int*)ni; w->cap = cap;
    }
    return o;
}

__device__ __forceinline__ bool is_cand(const uint8_t* b, long long p, int hs) {
    const uint8_t b0 = b[p];
    if ((b0 & 0xF8) || (b0 & 3) == 3) return false;
    if (b[p + 3] != 0) return false;
    if (hs == 6 && b[p + 5] != 0) return false;
    const uint8_t f = b[p + hs];
    return f >= 0xF0 && f <= 0xF2;
}

// per-byte flags (0x80 where true) of a 4-byte little-endian word
__device__ __forceinline__ unsigned zero_bytes(unsigned x) {      // byte == 0 (exact per byte: no carries)
    return ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;
}
__device__ __forceinline__ unsigned low2_ok(unsigned z, unsigned hi) {   // (b & hi) == 0 && (b & 3) != 3
    return zero_bytes((z & hi) | (z & (z >> 1) & 0x01010101u));
}

// the candidates among positions p0 .. p0+15 (bytes p0 .. p0+23 in w, also
// readable at base[0..23]) -> sc (any order; *scount counts all, sc keeps
// KCAP).  A position is a candidate when header byte 0 is valid, bytes +3 (and
// +5 for floats) are 0 and the payload byte +hs is F0..F2 (is_cand).  The
// dense part tests only the most selective and cheapest condition, a zero
// byte at +3 (one byte in 256 of codec output): approximate per-byte flags
// (x - 0x01..) & ~x & 0x80.. cost two operations a word and can only
// over-report (a byte 0x01 above a zero byte); the flagged positions, about
// one per 256 bytes, are then checked exactly byte by byte.
__device__ __forceinline__ void test16(const unsigned* w, const uint8_t* base, long long p0, int hs, long long phi,
                                       long long* sc, int* scount) {
    if (p0 >= phi) return;
    unsigned m = 0;   // bit j: byte j + 3 may be zero
#pragma unroll
    for (int k = 0; k < 5; k++) {
        const unsigned f = (w[k] - 0x01010101u) & ~w[k] & 0x80808080u;
        // the four flags of the word as a nibble (bits 7, 15, 23, 31 -> 28..31)
        const unsigned nib = (((f >> 7) & 0x01010101u) * 0x10204080u) >> 28;
        // byte 4k + t is position 4k + t - 3
        if (k == 0) m |= nib >> 3;
        else m |= nib << (4 * k - 3);
    }
    m &= 0xffffu;
    if (p0 < kFileHeader) m &= (kFileHeader - p0 >= 16) ? 0u : ~((1u << (kFileHeader - p0)) - 1u);
    if (p0 + 16 > phi) m &= (1u << (phi - p0)) - 1u;
    while (m) {
        const int i = __ffs(m) - 1;
        m &= m - 1;
        const uint8_t b0 = base[i], b3 = base[i + 3], f = base[i + hs];
        bool ok = !(b0 & 0xF8) && (b0 & 3) != 3 && b3 == 0 && f >= 0xF0 && f <= 0xF2;
        if (hs == 6) ok = ok && base[i + 5] == 0;
        if (ok) {
            const int at = atomicAdd(scount, 1);
            if (at < KCAP) sc[at] = p0 + i;
        }
    }
}

// bytes p0 .. p0+23 of the container (zero past the end) from global memory
__device__ __forceinline__ void load24(const uint8_t* blob, long long nbytes, long long p0, unsigned* w) {
    if (p0 + 24 <= nbytes) {
        const uint4 v = __ldg((const uint4*)(blob + p0));
        const uint2 u = __ldg((const uint2*)(blob + p0 + 16));
        w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w; w[4] = u.x; w[5] = u.y;
    } else {
#pragma unroll
        for (int k = 0; k < 6; k++) {
            unsigned x = 0;
            for (int b = 0; b < 4; b++) {
                const long long q = p0 + 4 * k + b;
                x |= (q < nbytes ? (unsigned)blob[q] : 0u) << (8 * b);
            }
            w[k] = x;
        }
    }
}

// the candidates of chunk c (SCB bytes from the 16-aligned address a0), from
// global memory (the ordered re-scan of a CTA whose list overflowed)
__device__ void scan_chunk_global(const uint8_t* blob, long long nbytes, int hs, uintptr_t a0, long long c,
                                  long long* sc, int* scount) {
    const long long phi = nbytes - hs;
    const long long pc = (long long)(a0 + (uintptr_t)(c * SCB)) - (long long)(uintptr_t)blob;
    for (int o = 16 * threadIdx.x; o < SCB; o += 16 * NT) {
        unsigned w[6];
        if (pc + o >= phi) break;
        load24(blob, nbytes, pc + o, w);
        test16(w, blob + (pc + o), pc + o, hs, phi, sc, scount);
    }
}

// sorted positions of the n (<= KCAP) candidates in sc -> dst[0..n)
__device__ __forceinline__ void put_sorted(const long long* sc, int n, long long* dst) {
    for (int i = threadIdx.x; i < n; i += NT) {
        const long long p = sc[i];
        int r = 0;
        for (int k = 0; k < n; k++) r += sc[k] < p ? 1 : 0;
        dst[r] = p;
    }
}

struct ScanSm {
    unsigned long long mbar[2];
    int ld[2];          // bytes staged per buffer
    int n;              // candidates of this CTA (may exceed KCAP)
    long long base, total;
    long long red[NT / 32], red2[NT / 32];
    long long sc[KCAP];
};

__device__ __forceinline__ void grid_barrier(unsigned int* count, unsigned int G) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(count, 1u);
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
            if (v < G) __nanosleep(64);
        } while (v < G);
    }
    __syncthreads();
}

// Signature scan and in-order compaction in one cooperative launch: CTA g
// scans its contiguous run of SCB-byte chunks (TMA bulk copies, double
// buffered, into shared memory), keeps its candidates there, and after a
// grid barrier writes them sorted at the sum of the candidate counts of the
// CTAs before it.  A CTA with more than KCAP candidates re-scans its chunks
// one by one from global memory.  With a gate (index-less speculation) the
// candidates are also written as the speculative offsets, and gate->spec
// says whether there is exactly one per block, the first at byte 28.
__global__ void __launch_bounds__(NT) scan_place_kernel(const uint8_t* blob, long long nbytes, int hs, uintptr_t a0,
                                                        long long nchunks, Ws W, long long n_blocks,
                                                        long long* offsets, IlGate* gate, IlGate* gate2) {
    extern __shared__ __align__(128) unsigned char smem_sp[];
    ScanSm* S = (ScanSm*)smem_sp;
    uint8_t* buf0 = smem_sp + ((sizeof(ScanSm) + 127) & ~(size_t)127);
    constexpr int BUFB = SCB + 128;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long G = gridDim.x, g = blockIdx.x;
    const long long per = (nchunks + G - 1) / G;
    const long long c0 = g * per < nchunks ? g * per : nchunks;
    const long long c1 = c0 + per < nchunks ? c0 + per : nchunks;
    const long long base_addr = (long long)(uintptr_t)blob;
    const long long phi = nbytes - hs;
    using namespace apax::tma;
    if (tid == 0) {
        mbar_init(&S->mbar[0]);
        mbar_init(&S->mbar[1]);
        fence_mbar_init();
        S->n = 0;
        if (gate && g == 0) {
            gate->first = ~0ULL;
            gate->gp = 0xFFFFFFFFu;
            gate->spec = 1u;   // cleared below (after the grid barrier) when not
            offsets[n_blocks] = nbytes;   // the last block's end: checked by the decode
            if (gate2) { gate2->first = ~0ULL; gate2->gp = 0xFFFFFFFFu; gate2->spec = 0xFFFFFFFFu; }
        }
    }
    __syncthreads();
    // chunk c -> buffer slot: SCB bytes + 16 (the last positions' look-ahead),
    // whole 16-byte units inside the container
    auto issue = [&](long long c, int slot) {
        const uintptr_t addr = a0 + (uintptr_t)(c * SCB);
        const long long avail = base_addr + nbytes - (long long)addr;
        long long bytes = avail < SCB + 16 ? avail : SCB + 16;
        bytes = bytes > 0 ? (bytes & ~15LL) : 0;
        S->ld[slot] = (int)bytes;
        if (bytes > 0) {
            fence_proxy_async();
            tma_load(buf0 + slot * BUFB, (const void*)addr, (uint32_t)bytes, &S->mbar[slot]);
        }
    };
    if (tid == 0 && c0 < c1) issue(c0, 0);
    uint32_t phs = 0;
    for (long long c = c0; c < c1; c++) {
        const int slot = (int)((c - c0) & 1);
        if (tid == 0 && c + 1 < c1) issue(c + 1, slot ^ 1);
        __syncthreads();   // S->ld[slot] visible
        const int ld = S->ld[slot];
        if (ld > 0) {
            mbar_wait(&S->mbar[slot], (phs >> slot) & 1u);
            phs ^= 1u << slot;
        }
        const uint8_t* b = buf0 + slot * BUFB;
        const long long pc = (long long)(a0 + (uintptr_t)(c * SCB)) - base_addr;
#pragma unroll
        for (int q = 0; q < SCB / (16 * NT); q++) {
            const int o = q * 16 * NT + 16 * tid;
            unsigned w[6];
            if (o + 24 <= ld) {
                const uint4 v = *(const uint4*)(b + o);
                const uint2 u = *(const uint2*)(b + o + 16);
                w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w; w[4] = u.x; w[5] = u.y;
                test16(w, b + o, pc + o, hs, phi, S->sc, &S->n);
            } else {
                if (pc + o >= phi) continue;
                load24(blob, nbytes, pc + o, w);
                test16(w, blob + (pc + o), pc + o, hs, phi, S->sc, &S->n);
            }
        }
        __syncthreads();   // the buffer is free for the chunk after next
    }
    const int n = S->n;
    if (tid == 0) W.ctot[g] = (unsigned)n;
    grid_barrier(&W.hdr->barrier, (unsigned)G);
    // base = candidates of the CTAs before g; total = all of them
    long long pre = 0, all = 0;
    for (long long h = tid; h < G; h += NT) {
        const long long v = (long long)W.ctot[h];
        all += v;
        pre += h < g ? v : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        pre += __shfl_xor_sync(0xffffffffu, pre, o);
        all += __shfl_xor_sync(0xffffffffu, all, o);
    }
    if (lane == 0) { S->red[warp] = pre; S->red2[warp] = all; }
    __syncthreads();
    if (tid == 0) {
        long long a = 0, t = 0;
        for (int k = 0; k < NT / 32; k++) { a += S->red[k]; t += S->red2[k]; }
        S->base = a;
        S->total = t;
        if (g == G - 1) {
            W.hdr->ncand = (unsigned long long)t;
            if (t > W.cap) W.hdr->fail = 1;
        }
    }
    __syncthreads();
    const long long base = S->base, total = S->total;
    if (total > W.cap) {
        if (gate && g == 0 && tid == 0) gate->spec = 0u;
        return;
    }
    const bool spec = gate && total == n_blocks;
    if (gate && g == 0 && tid == 0 && total != n_blocks) gate->spec = 0u;
    if (n <= KCAP) {
        for (int i = tid; i < n; i += NT) {
            const long long p = S->sc[i];
            int r = 0;
            for (int k = 0; k < n; k++) r += S->sc[k] < p ? 1 : 0;
            W.cpos[base + r] = p;
            if (spec) offsets[base + r] = p;
            if (spec && base + r == 0 && p != kFileHeader) gate->spec = 0u;
            // the first restarting block > 0 is the segment length (header byte 0, bit 2)
            if (spec && base + r > 0 && ((blob[p] >> 2) & 1)) atomicMin(&gate->first, (unsigned long long)(base + r));
        }
        return;
    }
    // overflow: the chunks again, one at a time, in order
    long long run = base;
    for (long long c = c0; c < c1; c++) {
        __syncthreads();
        if (tid == 0) S->n = 0;
        __syncthreads();
        scan_chunk_global(blob, nbytes, hs, a0, c, S->sc, &S->n);
        __syncthreads();
        const int m = S->n;
        if (m > KCAP) {
            if (tid == 0) {
                atomicExch(&W.hdr->fail, 1);
                if (gate) gate->spec = 0u;
            }
            return;
        }
        for (int i = tid; i < m; i += NT) {
            const long long p = S->sc[i];
            int r = 0;
            for (int k = 0; k < m; k++) r += S->sc[k] < p ? 1 : 0;
            W.cpos[run + r] = p;
            if (spec) offsets[run + r] = p;
            if (spec && run + r == 0 && p != kFileHeader) gate->spec = 0u;
            if (spec && run + r > 0 && ((blob[p] >> 2) & 1)) atomicMin(&gate->first, (unsigned long long)(run + r));
        }
        run += m;
    }
}

// warp per candidate: exact JEE parse (same code and checks as the walk)
// with a full block's group count -> next block position or -1; then the
// index of the candidate at that position (usually the next one)
__global__ void __launch_bounds__(NT) parse_kernel(const uint8_t* blob, long long nbytes, int bs, int dt, Ws W,
                                                   const IlGate* gate, uint8_t* jee_cache, long long n_blocks) {
    if (gate && il_seg_ok(gate)) return;
    extern __shared__ __align__(16) unsigned char smem_k5[];
    if (W.hdr->fail) return;
    const long long nc = (long long)W.hdr->ncand;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int G = bs >> 2;
    const int ebytes = (G + 16 + 15) & ~15;   // the fast parser may write e[G]
    uint8_t* e = smem_k5 + warp * (ebytes + KSTAGE + KREC);
    uint8_t* stg = e + ebytes;                  // the candidate's JEE bytes, staged
    unsigned* rwb = (unsigned*)(stg + KSTAGE);  // record: bits up to the end of each decode warp
    unsigned short* rtp = (unsigned short*)(rwb + 8);   // record: each decode thread's bit offset
    const int hs = hdr_size(dt);
    const long long maxj = (3LL * G + 2) / 2;
    const long long nwarps = (long long)gridDim.x * NW;
    for (long long i = (long long)blockIdx.x * NW + warp; i < nc; i += nwarps) {
        const long long pos = W.cpos[i];
        long long nxt = -1;
        const long long avail = nbytes - pos - hs;
        if (avail >= 0) {
            const long long nbj = avail < maxj ? avail : maxj;
            long long used = 0, esum = 0;
            // fast parse (128 nibbles per step); any irregularity -- which
            // most false candidates hit within a few tokens -- takes the
            // exact parser, which decides the candidate
            int u = 0;
            int st = -1;
            // stage [ps - 16, ps - 16 + KSTAGE) (16-aligned start) in one round of
            // loads, then parse from shared memory: the parse's serial steps no
            // longer wait on global memory
            const long long ps = pos + hs;
            const long long g0 = (ps - 16) & ~15LL;
            if (g0 >= 0 && ps + nbj + 8 <= g0 + KSTAGE) {
#pragma unroll
                for (int k = 0; k < KSTAGE / 512; k++) {
                    const long long o = g0 + 512 * k + 16 * lane;
                    uint4 v;
                    if (o + 16 <= nbytes) v = __ldg((const uint4*)(blob + o));
                    else {
                        uint32_t t[4];
                        for (int q = 0; q < 4; q++) {
                            uint32_t x = 0;
                            for (int b = 0; b < 4; b++) {
                                const long long a = o + 4 * q + b;
                                x |= (a < nbytes ? (uint32_t)blob[a] : 0u) << (8 * b);
                            }
                            t[q] = x;
                        }
                        v = make_uint4(t[0], t[1], t[2], t[3]);
                    }
                    *(uint4*)(stg + 512 * k + 16 * lane) = v;
                }
                __syncwarp();
                const long long lim = nbytes - g0;
                st = warp_jee_fast<false>(stg + (ps - g0), stg + (lim < KSTAGE ? lim : KSTAGE), (int)(2 * nbj), G, e, u);
            } else {
                st = warp_jee_fast(blob + ps, blob + nbytes, (int)(2 * nbj), G, e, u);
            }
            __syncwarp();
            if (st == 0) {
                used = u;
                unsigned sb = 0;
                for (int g = 4 * lane; g < G; g += 128) {
                    uint32_t ew;
                    if (g + 4 <= G) ew = *(const uint32_t*)(e + g);
                    else {
                        ew = 0;
                        for (int c = 0; c < 4; c++) ew |= (g + c < G ? (uint32_t)e[g + c] : 0u) << (8 * c);
                    }
                    sb += (unsigned)__dp4a(ew, 0x01010101u, 0u);
                }
                esum = __reduce_add_sync(0xffffffffu, sb);
            } else {
                st = warp_jee_decode(blob + pos + hs, 2 * nbj, G, e, used, esum);
            }
            const long long sz = (used + 1) / 2 + (4 * esum + 7) / 8;
            if (!st && avail >= sz) nxt = pos + hs + sz;
            if (!st && jee_cache && i + 1 < n_blocks) {
                // candidate i's parse as block i's record of the two-pass decode
                // (the JEE phase of decode_v3_kernel, same layout and values):
                // used by pass 1 when every candidate turns out to be a block
                __syncwarp();
                unsigned sb = 0, em = 0, wb[8];
#pragma unroll
                for (int k = 0; k < 32; k += 4) {
                    const int g = 32 * lane + k;
                    uint32_t ew;
                    if (g + 4 <= G) ew = *(const uint32_t*)(e + g);
                    else {
                        ew = 0;
                        for (int c = 0; c < 4; c++) ew |= (g + c < G ? (uint32_t)e[g + c] : 0u) << (8 * c);
                    }
                    wb[k >> 2] = 4u * (unsigned)__dp4a(ew, 0x01010101u, 0u);
                    sb += wb[k >> 2];
                    em = __vmaxu4(em, ew);
                }
                const unsigned own = sb;
                em = max(max(em & 0xffu, (em >> 8) & 0xffu), max((em >> 16) & 0xffu, em >> 24));
                const unsigned wmax = __reduce_max_sync(0xffffffffu, em);
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const unsigned o = __shfl_up_sync(0xffffffffu, sb, d);
                    if (lane >= d) sb += o;
                }
                if ((lane & 3) == 3) rwb[lane >> 2] = sb;
                const unsigned sx = sb - own;
                unsigned run = sx - __shfl_sync(0xffffffffu, sx, lane & ~3);
#pragma unroll
                for (int q = 0; q < 8; q++) { rtp[8 * lane + q] = (unsigned short)run; run += wb[q]; }
                __syncwarp();
                uint8_t* rec = jee_cache + (size_t)i * (size_t)kJeeRecBytes;
                if (lane == 0) {
                    const uint8_t* h = blob + pos;
                    const bool isf = dt >= 3;
                    const int hdr = (int)(h[0] & 7) | ((int)h[1] << 8) | ((int)h[2] << 16) | (isf ? ((int)h[4] << 24) : 0);
                    const int code = (hdr >> 8) & 0xFFFF;
                    const double ds = isf ? decode_scale_code(code) * ldexp(1.0, hdr >> 24) : decode_scale_code(code);
                    *(int4*)rec = make_int4(hdr, 0, (int)used, (int)wmax);
                    *(double2*)(rec + 16) = make_double2(ds, __ddiv_rn(1.0, ds));
                }
                if (lane < 8) ((unsigned*)(rec + 32))[lane] = rwb[lane];
                const uint32_t* tp = (const uint32_t*)rtp;
#pragma unroll
                for (int q = 0; q < 4; q++) ((uint32_t*)(rec + 64))[lane + 32 * q] = tp[lane + 32 * q];
                ((uint4*)(rec + 576))[lane] = ((const uint4*)e)[lane];
                ((uint4*)(rec + 576))[lane + 32] = ((const uint4*)e)[lane + 32];
            }
        }
        // successor index: the candidate at position nxt (32-ary search)
        int s = -1;
        if (nxt >= 0) {
            if (i + 1 < nc && W.cpos[i + 1] == nxt) s = (int)(i + 1);
            else {
                long long lo = i + 1, hi = nc;   // positions are sorted and nxt > pos
                while (hi - lo > 32) {
                    const long long step = (hi - lo + 31) / 32;
                    const long long k = lo + lane * step;
                    const bool le = k < hi && W.cpos[k] <= nxt;
                    const unsigned m = __ballot_sync(0xffffffffu, le);
                    if (!m) { hi = lo; break; }
                    const int l = 31 - __clz(m);
                    lo = lo + l * step;
                    hi = lo + step < hi ? lo + step : hi;
                }
                const long long k = lo + lane;
                const unsigned m = __ballot_sync(0xffffffffu, k < hi && W.cpos[k] == nxt);
                if (m) s = (int)(lo + __ffs(m) - 1);
            }
        }
        if (lane == 0) {
            W.cnext[i] = nxt;
            W.succ[i] = s;
        }
        __syncwarp();
    }
}

// fast path: every candidate is a block and points at the next one ->
// offsets = candidate positions.  Also clears the prune path's state.
__global__ void __launch_bounds__(NT) chain_kernel(long long n_blocks, long long* offsets, Ws W, const IlGate* gate) {
    if (gate && il_seg_ok(gate)) return;
    const long long nc = (long long)W.hdr->ncand;
    const long long stride = (long long)gridDim.x * NT;
    const long long i0 = (long long)blockIdx.x * NT + threadIdx.x;
    for (long long i = i0; i < W.cap; i += stride) { W.keep0[i] = 0; W.keep1[i] = 0; }
    for (long long b = i0; b < n_blocks; b += stride) W.nodeidx[b] = -1;
    if (W.hdr->fail) return;
    bool bad = nc != n_blocks;
    if (!bad) {
        for (long long b = i0; b < n_blocks; b += stride) {
            const long long p = W.cpos[b];
            offsets[b] = p;
            if (b == 0 && p != kFileHeader) bad = true;
            if (b + 1 < n_blocks && W.cnext[b] != W.cpos[b + 1]) bad = true;
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(&W.hdr->chain_bad, 1);
}

// the prune path in one CTA (runs only when the fast path did not hold):
// keep the candidates some kept candidate points at (twice, the head always),
// list the survivors in position order, check the walk's recurrence
__global__ void __launch_bounds__(1024) prune_kernel(long long n_blocks, long long* offsets, Ws W, const IlGate* gate) {
    __shared__ int wc[32];
    if (gate && il_seg_ok(gate)) return;
    if (W.hdr->fail || !W.hdr->chain_bad) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long nc = (long long)W.hdr->ncand;
    for (int pass = 0; pass < 2; pass++) {
        uint8_t* out = pass ? W.keep1 : W.keep0;
        for (long long i = tid; i < nc; i += 1024) {
            if (i == 0 && W.cpos[0] == kFileHeader) out[0] = 1;
            if (pass && !W.keep0[i]) continue;
            const int sidx = W.succ[i];
            if (sidx >= 0) out[sidx] = 1;
        }
        __syncthreads();
    }
    long long run = 0;
    for (long long t0 = 0; t0 < nc; t0 += 1024) {
        const long long i = t0 + tid;
        const bool f = i < nc && W.keep1[i];
        const unsigned m = __ballot_sync(0xffffffffu, f);
        if (lane == 0) wc[warp] = __popc(m);
        __syncthreads();
        int before = 0, tot = 0;
        for (int k = 0; k < 32; k++) {
            before += k < warp ? wc[k] : 0;
            tot += wc[k];
        }
        const long long b = run + before + __popc(m & ((1u << lane) - 1u));
        if (f && b < n_blocks) {
            offsets[b] = W.cpos[i];
            W.nodeidx[b] = (int)i;
        }
        run += tot;
        __syncthreads();
    }
    bool bad = false;
    for (long long b = tid; b < n_blocks; b += 1024) {
        const int i = W.nodeidx[b];
        if (i < 0) { bad = true; continue; }
        if (b == 0 && offsets[0] != kFileHeader) bad = true;
        if (b + 1 < n_blocks && W.cnext[i] != offsets[b + 1]) bad = true;
    }
    if (__syncthreads_or(bad) && tid == 0) atomicExch(&W.hdr->fail, 1);
}

static size_t scan_smem() { return ((sizeof(ScanSm) + 127) & ~(size_t)127) + 2 * (SCB + 128); }

static int scan_grid(long long nchunks) {
    static int per_sm = -1;
    if (per_sm < 0) {
        cudaFuncSetAttribute(scan_place_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)scan_smem());
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scan_place_kernel, NT, scan_smem()) != cudaSuccess ||
            per_sm < 1)
            per_sm = 1;
    }
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    long long g = (long long)per_sm * (nsm > 0 ? nsm : 148);
    if (g > LBMAX) g = LBMAX;
    if (g > nchunks) g = nchunks;
    return (int)(g < 1 ? 1 : g);
}

// candidates in position order -> cpos, ncand (and, with a gate, the
// speculative offsets): one cooperative launch over SCB-byte chunks from a
// 16-aligned start
static int launch_scan(const uint8_t* blob, long long nbytes, int hs, const Ws& W, long long n_blocks,
                       long long* offsets, IlGate* gate, IlGate* gate2, cudaStream_t st) {
    const uintptr_t a0 = ((uintptr_t)blob + kFileHeader) & ~(uintptr_t)15;
    const long long span = (long long)((uintptr_t)blob + (uintptr_t)nbytes) - (long long)a0;
    const long long nchunks = span > 0 ? (span + SCB - 1) / SCB : 1;
    if (cudaMemsetAsync(W.hdr, 0, sizeof(Hdr), st) != cudaSuccess) return APAX_ERR_CUDA;
    const int grid = scan_grid(nchunks);
    const size_t sm = scan_smem();
    if (cudaFuncSetAttribute(scan_place_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
        return APAX_ERR_CUDA;
    void* args[] = {(void*)&blob, (void*)&nbytes, (void*)&hs, (void*)&a0, (void*)&nchunks, (void*)&W,
                    (void*)&n_blocks, (void*)&offsets, (void*)&gate, (void*)&gate2};
    note_launches(1);
    if (cudaLaunchCooperativeKernel((const void*)scan_place_kernel, dim3(grid), dim3(NT), args, sm, st) != cudaSuccess)
        return APAX_ERR_CUDA;
    return APAX_OK;
}

static int sm_count() {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return nsm > 0 ? nsm : 148;
}

}  // namespace k5

size_t find_blocks_k5_ws_bytes(long long n_blocks) { return k5::layout(n_blocks, nullptr, nullptr); }

int launch_k5_speculate(const uint8_t* blob, long long nbytes, int dt, long long n_blocks, long long* offsets,
                        void* ws, IlGate* gate, IlGate* gate2, cudaStream_t st) {
    using namespace k5;
    Ws W;
    layout(n_blocks, (uint8_t*)ws, &W);
    return launch_scan(blob, nbytes, hdr_size(dt), W, n_blocks, offsets, gate, gate2, st);
}

const int* k5_flags(void* ws, long long n_blocks) {
    k5::Ws W;
    k5::layout(n_blocks, (uint8_t*)ws, &W);
    static_assert(offsetof(k5::Hdr, chain_bad) == offsetof(k5::Hdr, fail) + sizeof(int), "fail, chain_bad adjacent");
    return &W.hdr->fail;
}

int launch_find_blocks_k5(const uint8_t* blob, long long nbytes, long long n, int bs, int dt, long long n_blocks,
                          long long* offsets, unsigned long long* status, void* ws, cudaStream_t st,
                          const IlGate* gate, uint8_t* jee_cache) {
    using namespace k5;
    Ws W;
    layout(n_blocks, (uint8_t*)ws, &W);
    const int hs = hdr_size(dt);
    const int nsm = sm_count();
    if (!gate) {
        const int r = launch_scan(blob, nbytes, hs, W, n_blocks, offsets, nullptr, nullptr, st);
        if (r) return r;
    }
    const size_t psmem = (size_t)NW * ((((bs >> 2) + 16 + 15) & ~15) + KSTAGE + KREC);
    if (bs > 4096) jee_cache = nullptr;   // the records hold up to 1024 groups
    if (cudaFuncSetAttribute(parse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem) != cudaSuccess)
        return APAX_ERR_CUDA;
    long long pgrid = (W.cap + NW - 1) / NW;
    if (pgrid > (long long)nsm * 8) pgrid = (long long)nsm * 8;
    note_launches(1);
    parse_kernel<<<(int)pgrid, NT, psmem, st>>>(blob, nbytes, bs, dt, W, gate, jee_cache, n_blocks);
    long long cgrid = (W.cap + NT - 1) / NT;
    if (cgrid > (long long)nsm * 4) cgrid = (long long)nsm * 4;
    note_launches(1);
    chain_kernel<<<(int)cgrid, NT, 0, st>>>(n_blocks, offsets, W, gate);
    note_launches(1);
    prune_kernel<<<1, 1024, 0, st>>>(n_blocks, offsets, W, gate);
    if (cudaGetLastError() != cudaSuccess) return APAX_ERR_CUDA;
    // last block (true group count) or, on any anomaly, the full serial walk
    return launch_walk_after_k5(blob, nbytes, n, bs, dt, n_blocks, offsets, status, &W.hdr->fail, st, gate);
}

}  // namespace apax
