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
//      (entropy.py:60-64) -> first payload byte in {F0,F1,F2}.  Positions
//      matching are compacted, in order, into cand[] (count/scan/emit);
//   2. one warp per candidate runs the same exact JEE parse as the walk
//      (warp_jee_decode) with a full block's group count and records the
//      position of the following block (next[]), or -1 on any error;
//   3. candidates nobody points at (other than the head at byte 28) are
//      dropped, twice; the survivors in position order are the chain;
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
constexpr int CMAX = 2048;   // chunks of the count/scan/emit passes

struct Hdr {
    unsigned long long ncand;   // candidates found (may exceed cap -> fail)
    unsigned long long nkept;
    int fail;
    int pad[3];
};

struct Ws {
    Hdr* hdr;
    unsigned long long* ccount;   // CMAX
    unsigned long long* cbase;    // CMAX
    long long* cpos;              // cap
    long long* cnext;             // cap
    int* succ;                    // cap
    uint8_t* keep0;               // cap
    uint8_t* keep1;               // cap
    int* nodeidx;                 // n_blocks
    long long cap;
};

static size_t al(size_t v) { return (v + 255) & ~(size_t)255; }

static long long cap_for(long long n_blocks) { return 2 * n_blocks + 4096; }

static size_t layout(long long n_blocks, uint8_t* base, Ws* w) {
    const long long cap = cap_for(n_blocks);
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t at = o; o += al(bytes); return base ? base + at : nullptr; };
    uint8_t* h = take(sizeof(Hdr));
    uint8_t* cc = take(CMAX * 8);
    uint8_t* cb = take(CMAX * 8);
    uint8_t* cp = take((size_t)cap * 8);
    uint8_t* cn = take((size_t)cap * 8);
    uint8_t* su = take((size_t)cap * 4);
    uint8_t* k0 = take((size_t)cap);
    uint8_t* k1 = take((size_t)cap);
    uint8_t* ni = take((size_t)(n_blocks > 0 ? n_blocks : 1) * 4);
    if (w) {
        w->hdr = (Hdr*)h; w->ccount = (unsigned long long*)cc; w->cbase = (unsigned long long*)cb;
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

// chunk c of the candidate positions [kFileHeader, nbytes - hs)
__device__ __forceinline__ void chunk_range(long long lo_all, long long hi_all, int c, int nc, long long& lo,
                                            long long& hi) {
    const long long span = hi_all > lo_all ? hi_all - lo_all : 0;
    const long long per = (span + nc - 1) / nc;
    lo = lo_all + per * c;
    hi = lo + per;
    if (lo > hi_all) lo = hi_all;
    if (hi > hi_all) hi = hi_all;
}

__device__ __forceinline__ unsigned long long block_sum(unsigned long long v) {
    __shared__ unsigned long long red[NW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    unsigned long long t = 0;
#pragma unroll
    for (int k = 0; k < NW; k++) t += red[k];
    return t;
}

// pass 1: candidate count per chunk
__global__ void __launch_bounds__(NT) count_kernel(const uint8_t* blob, long long nbytes, int hs, int nc,
                                                   unsigned long long* ccount) {
    long long lo, hi;
    chunk_range(kFileHeader, nbytes - hs, blockIdx.x, nc, lo, hi);
    unsigned long long c = 0;
    for (long long p = lo + threadIdx.x; p < hi; p += NT) c += is_cand(blob, p, hs) ? 1 : 0;
    c = block_sum(c);
    if (threadIdx.x == 0) ccount[blockIdx.x] = c;
}

// exclusive scan of nc (<= CMAX) chunk counts by one CTA of 1024 threads
__global__ void __launch_bounds__(1024) scan_kernel(const unsigned long long* cnt, int nc, unsigned long long* base,
                                                    unsigned long long* total, long long cap, int* fail) {
    __shared__ unsigned long long wsum[32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const unsigned long long a = (2 * t < nc) ? cnt[2 * t] : 0;
    const unsigned long long b = (2 * t + 1 < nc) ? cnt[2 * t + 1] : 0;
    unsigned long long v = a + b, incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        unsigned long long o = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += o;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        unsigned long long s = wsum[lane], si = s;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            unsigned long long o = __shfl_up_sync(0xffffffffu, si, d);
            if (lane >= d) si += o;
        }
        wsum[lane] = si - s;
        if (lane == 31) {
            *total = si;
            if ((long long)si > cap) *fail = 1;
        }
    }
    __syncthreads();
    const unsigned long long ex = wsum[warp] + incl - v;
    if (2 * t < nc) base[2 * t] = ex;
    if (2 * t + 1 < nc) base[2 * t + 1] = ex + a;
}

// in-order emit of the flagged items of one chunk: tile of NT items per
// iteration, ballot + CTA prefix, written at base + running count
template <typename Flag, typename Put>
__device__ __forceinline__ void emit_chunk(long long lo, long long hi, unsigned long long base, Flag flag, Put put) {
    __shared__ int wc[NW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long run = base;
    for (long long t0 = lo; t0 < hi; t0 += NT) {
        const long long p = t0 + threadIdx.x;
        const bool f = p < hi && flag(p);
        if (!__syncthreads_or(f)) continue;
        const unsigned m = __ballot_sync(0xffffffffu, f);
        if (lane == 0) wc[warp] = __popc(m);
        __syncthreads();
        int before = 0, tot = 0;
#pragma unroll
        for (int k = 0; k < NW; k++) {
            before += (k < warp) ? wc[k] : 0;
            tot += wc[k];
        }
        if (f) put(run + before + __popc(m & ((1u << lane) - 1u)), p);
        run += tot;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(NT) emit_kernel(const uint8_t* blob, long long nbytes, int hs, int nc, Ws W) {
    if (W.hdr->fail) return;
    long long lo, hi;
    chunk_range(kFileHeader, nbytes - hs, blockIdx.x, nc, lo, hi);
    emit_chunk(lo, hi, W.cbase[blockIdx.x], [&](long long p) { return is_cand(blob, p, hs); },
               [&](unsigned long long at, long long p) { W.cpos[at] = p; });
}

// warp per candidate: exact JEE parse (same code and checks as the walk)
// with a full block's group count -> next block position or -1; then the
// index of the candidate at that position (usually the next one)
__global__ void __launch_bounds__(NT) parse_kernel(const uint8_t* blob, long long nbytes, int bs, int dt, Ws W) {
    extern __shared__ __align__(16) unsigned char smem_k5[];
    if (W.hdr->fail) return;
    const long long nc = (long long)W.hdr->ncand;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int G = bs >> 2;
    uint8_t* e = smem_k5 + warp * ((G + 16 + 15) & ~15);   // the fast parser may write e[G]
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
            int st = warp_jee_fast(blob + pos + hs, blob + nbytes, (int)(2 * nbj), G, e, u);
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

// keep_out[succ[i]] = 1 for every kept i (all candidates when keep_in is
// null); the head (candidate 0 at byte 28) is always kept
__global__ void __launch_bounds__(NT) mark_kernel(const uint8_t* keep_in, uint8_t* keep_out, Ws W) {
    if (W.hdr->fail) return;
    const long long nc = (long long)W.hdr->ncand;
    for (long long i = (long long)blockIdx.x * NT + threadIdx.x; i < nc; i += (long long)gridDim.x * NT) {
        if (i == 0 && W.cpos[0] == kFileHeader) keep_out[0] = 1;
        if (keep_in && !keep_in[i]) continue;
        const int s = W.succ[i];
        if (s >= 0) keep_out[s] = 1;
    }
}

__global__ void __launch_bounds__(NT) kcount_kernel(const uint8_t* keep, int nc, Ws W) {
    if (W.hdr->fail) return;
    long long lo, hi;
    chunk_range(0, (long long)W.hdr->ncand, blockIdx.x, nc, lo, hi);
    unsigned long long c = 0;
    for (long long i = lo + threadIdx.x; i < hi; i += NT) c += keep[i] ? 1 : 0;
    c = block_sum(c);
    if (threadIdx.x == 0) W.ccount[blockIdx.x] = c;
}

// survivor b (in position order) -> offsets[b], nodeidx[b]
__global__ void __launch_bounds__(NT) kemit_kernel(const uint8_t* keep, int nc, long long n_blocks, long long* offsets,
                                                   Ws W) {
    if (W.hdr->fail) return;
    long long lo, hi;
    chunk_range(0, (long long)W.hdr->ncand, blockIdx.x, nc, lo, hi);
    emit_chunk(lo, hi, W.cbase[blockIdx.x], [&](long long i) { return keep[i] != 0; },
               [&](unsigned long long b, long long i) {
                   if ((long long)b < n_blocks) {
                       offsets[b] = W.cpos[i];
                       W.nodeidx[b] = (int)i;
                   }
               });
}

// the walk's recurrence on the survivors: offsets[0] = 28 and
// offsets[b+1] = next(offsets[b]) for b < n_blocks - 1
__global__ void __launch_bounds__(NT) verify_kernel(long long n_blocks, const long long* offsets, Ws W) {
    if (W.hdr->fail) return;
    bool bad = false;
    for (long long b = (long long)blockIdx.x * NT + threadIdx.x; b < n_blocks; b += (long long)gridDim.x * NT) {
        const int i = W.nodeidx[b];
        if (i < 0) { bad = true; continue; }
        if (b == 0 && offsets[0] != kFileHeader) bad = true;
        if (b + 1 < n_blocks && W.cnext[i] != offsets[b + 1]) bad = true;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(&W.hdr->fail, 1);
}

}  // namespace k5

size_t find_blocks_k5_ws_bytes(long long n_blocks) { return k5::layout(n_blocks, nullptr, nullptr); }

int launch_find_blocks_k5(const uint8_t* blob, long long nbytes, long long n, int bs, int dt, long long n_blocks,
                          long long* offsets, unsigned long long* status, void* ws, cudaStream_t st) {
    using namespace k5;
    Ws W;
    layout(n_blocks, (uint8_t*)ws, &W);
    const int hs = hdr_size(dt);
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (cudaMemsetAsync(W.hdr, 0, sizeof(Hdr), st) != cudaSuccess) return APAX_ERR_CUDA;
    if (cudaMemsetAsync(W.keep0, 0, (size_t)W.cap, st) != cudaSuccess) return APAX_ERR_CUDA;
    if (cudaMemsetAsync(W.keep1, 0, (size_t)W.cap, st) != cudaSuccess) return APAX_ERR_CUDA;
    if (cudaMemsetAsync(W.nodeidx, 0xFF, (size_t)n_blocks * 4, st) != cudaSuccess) return APAX_ERR_CUDA;
    // byte chunks: ~32 KB each, at most CMAX
    long long span = nbytes - hs - kFileHeader;
    int ncb = (int)((span + 32767) / 32768);
    ncb = ncb < 1 ? 1 : (ncb > CMAX ? CMAX : ncb);
    note_launches(1);
    count_kernel<<<ncb, NT, 0, st>>>(blob, nbytes, hs, ncb, W.ccount);
    note_launches(1);
    scan_kernel<<<1, 1024, 0, st>>>(W.ccount, ncb, W.cbase, &W.hdr->ncand, W.cap, &W.hdr->fail);
    note_launches(1);
    emit_kernel<<<ncb, NT, 0, st>>>(blob, nbytes, hs, ncb, W);
    const size_t psmem = (size_t)NW * (((bs >> 2) + 16 + 15) & ~15);
    if (cudaFuncSetAttribute(parse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem) != cudaSuccess)
        return APAX_ERR_CUDA;
    long long pgrid = (W.cap + NW - 1) / NW;
    if (pgrid > (long long)nsm * 8) pgrid = (long long)nsm * 8;
    note_launches(1);
    parse_kernel<<<(int)pgrid, NT, psmem, st>>>(blob, nbytes, bs, dt, W);
    long long mgrid = (W.cap + NT - 1) / NT;
    if (mgrid > (long long)nsm * 8) mgrid = (long long)nsm * 8;
    note_launches(1);
    mark_kernel<<<(int)mgrid, NT, 0, st>>>(nullptr, W.keep0, W);
    note_launches(1);
    mark_kernel<<<(int)mgrid, NT, 0, st>>>(W.keep0, W.keep1, W);
    // survivors in order: chunks over the candidate index (<= cap)
    int nck = (int)((W.cap + 4095) / 4096);
    nck = nck < 1 ? 1 : (nck > CMAX ? CMAX : nck);
    note_launches(1);
    kcount_kernel<<<nck, NT, 0, st>>>(W.keep1, nck, W);
    note_launches(1);
    scan_kernel<<<1, 1024, 0, st>>>(W.ccount, nck, W.cbase, &W.hdr->nkept, (long long)1 << 62, &W.hdr->fail);
    note_launches(1);
    kemit_kernel<<<nck, NT, 0, st>>>(W.keep1, nck, n_blocks, offsets, W);
    long long vgrid = (n_blocks + NT - 1) / NT;
    if (vgrid > (long long)nsm * 8) vgrid = (long long)nsm * 8;
    note_launches(1);
    verify_kernel<<<(int)vgrid, NT, 0, st>>>(n_blocks, offsets, W);
    if (cudaGetLastError() != cudaSuccess) return APAX_ERR_CUDA;
    // last block (true group count) or, on any anomaly, the full serial walk
    return launch_walk_after_k5(blob, nbytes, n, bs, dt, n_blocks, offsets, status, &W.hdr->fail, st);
}

}  // namespace apax
