// apax_decode.cu -- B200 APAX decoder (K4) and container block walk (K5-lite).
//
// Reproduces reference `decode_stream` (pkg/src/apax/codec.py:308-329):
//   * block header parse (dtypes.py:167-180), JEE decode with the exact
//     status semantics of entropy.py:118-191 as a warp-parallel token parse
//     (32 nibbles per step; escape coverage resolved with ballots),
//     mantissa unpack + sign extension (entropy.py:249-277), reconstruct
//     (transform.py:116-129) as CTA prefix scans, dequantize
//     (codec.py:135-146) and a coalesced store of the [:n] slice;
//   * the cross-block derivative history (transform.py:31-49) is carried by
//     a decoupled look-back over affine maps: a block's
//     output history is M * input + c; restart / D0 blocks publish a
//     concrete value immediately, others publish their map and compose
//     their predecessors' until a concrete value is found.
#include <cstdint>
#include <cuda_runtime.h>

#include "apax_device.cuh"
#include "apax_kernels.cuh"
#include "apax_jee.cuh"

namespace apax {


struct DecState {
    long long block;
    int sel, restart, code, fbe, err;
    long long pay_off;       // smem byte offset of payload start
    long long avail;         // payload bytes available in the blob
    long long used_nibs;
    long long jee_bytes;
    long long mant_bits;
    long long p1, p2;        // input history for this block
    long long red[kWarps * 2];
};

// ---------------------------------------------------------------------------
// CTA inclusive scan of a per-thread int64 total; returns exclusive prefix
// ---------------------------------------------------------------------------
__device__ __forceinline__ long long cta_excl_scan(long long v, long long* red, long long& total) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    long long x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        long long o = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += o;
    }
    if (lane == 31) red[warp] = x;
    __syncthreads();
    if (tid == 0) {
        long long acc = 0;
        for (int w = 0; w < kWarps; w++) { long long t = red[w]; red[w] = acc; acc += t; }
        red[kWarps] = acc;
    }
    __syncthreads();
    long long ex = red[warp] + x - v;
    total = red[kWarps];
    __syncthreads();
    return ex;
}

// read nb (1..64) bits MSB-first at bit position `bp` of a 4-aligned smem
// byte buffer (padded by >= 12 bytes)
__device__ __forceinline__ unsigned long long read_bits(const uint32_t* w, long long bp, int nb) {
    long long k = bp >> 5;
    int sh = (int)(bp & 31);
    unsigned long long hi = ((unsigned long long)bswap32(w[k]) << 32) | bswap32(w[k + 1]);
    unsigned long long t = hi << sh;
    if (sh) t |= (unsigned long long)bswap32(w[k + 2]) >> (32 - sh);
    return t >> (64 - nb);
}

// 2x2 affine map on the history (p1, p2), arithmetic mod 2^64
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
__global__ void __launch_bounds__(kNT) decode_kernel(DecParams P) {
    using Tr = DT_<DT>;
    using T = typename Tr::T;
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x;
    const int bs = P.bs;
    const int Gfull = bs / 4;
    const int gpt = (Gfull + kNT - 1) / kNT;
    const int hs = Tr::HDR;

    DecState* S = (DecState*)smem;
    size_t off = (sizeof(DecState) + 15) & ~(size_t)15;
    long long* qb = (long long*)(smem + off);
    off += ((size_t)(bs + 4) * 8 + 15) & ~(size_t)15;
    uint8_t* e = (uint8_t*)(smem + off);
    off += ((size_t)Gfull + 16 + 15) & ~(size_t)15;
    uint8_t* pay = (uint8_t*)(smem + off);  // payload_cap + 32

    for (;;) {
        if (tid == 0) S->block = (long long)atomicAdd(P.ticket, 1u);
        __syncthreads();
        const long long b = S->block;
        if (b >= P.n_blocks) break;
        const long long start = b * (long long)bs;
        const int n = (int)((P.n - start) < bs ? (P.n - start) : bs);
        const int G = (n + 3) >> 2;
        const int np = 4 * G;
        unsigned long long* cw = P.carry + 16 * b;  // [0] flag, [1..6] map, [8..9] value
        const long long boff = P.offsets[b];
        const long long bend = P.offsets[b + 1];

        if (tid == 0) {
            S->err = 0;
            if (boff < 0) {
                S->err = -1;  // not present (walk stopped earlier)
            } else if (P.nbytes - boff < hs) {
                S->err = APAX_ERR_BLOCK_HDR_TRUNCATED;
            } else {
                uint8_t h0 = P.blob[boff];
                S->sel = h0 & 3;
                S->restart = (h0 >> 2) & 1;
                S->code = P.blob[boff + 1] | (P.blob[boff + 2] << 8);
                S->fbe = Tr::F ? (int)(int8_t)P.blob[boff + 4] : 0;
                if (S->sel == 3) S->err = APAX_ERR_SELECTOR;
            }
        }
        __syncthreads();
        // stage the payload bytes [boff + hs, end) into smem (16B-aligned superset)
        if (S->err == 0) {
            const long long ps = boff + hs;
            long long pe = (bend > ps) ? bend : ps;
            const long long maxj = (3LL * G + 2) / 2;
            if (pe < ps + maxj) pe = ps + maxj;      // JEE may read past the block end
            if (pe > P.nbytes) pe = P.nbytes;
            long long a0 = ps & ~15LL;
            long long len = pe - a0;
            if (len > P.payload_cap) len = P.payload_cap;
            const long long full = (P.nbytes & ~15LL);
            for (long long i = 16 * tid; i < len; i += 16 * kNT) {
                long long src = a0 + i;
                if (src + 16 <= full) {
                    *(uint4*)(pay + i) = __ldcs((const uint4*)(P.blob + src));
                } else {
                    for (int k = 0; k < 16; k++)
                        pay[i + k] = (src + k < P.nbytes) ? P.blob[src + k] : 0;
                }
            }
            if (tid == 0) {
                S->pay_off = ps - a0;
                S->avail = P.nbytes - ps;
            }
        }
        __syncthreads();
        // ---- JEE (warp 0) ----
        if (S->err == 0 && tid < 32) {
            const uint8_t* p = pay + S->pay_off;
            long long maxj = (3LL * G + 2) / 2;
            long long nbj = S->avail < maxj ? S->avail : maxj;
            long long used = 0, esum = 0;
            int st = warp_jee_decode(p, 2 * nbj, G, e, used, esum);
            if (tid == 0) {
                if (st) S->err = st;
                else {
                    S->used_nibs = used;
                    S->jee_bytes = (used + 1) / 2;
                    S->mant_bits = 4 * esum;
                    long long mant_bytes = (4 * esum + 7) / 8;
                    if (S->avail < S->jee_bytes + mant_bytes) S->err = APAX_ERR_MANTISSA_TRUNCATED;
                    else if (S->pay_off + S->jee_bytes + mant_bytes + 16 > P.payload_cap) S->err = APAX_ERR_ARG;
                }
            }
        }
        __syncthreads();
        const int err = S->err;
        if (err) {
            if (tid == 0) {
                if (err > 0) report_error(P.status, b, err);
                // publish a dummy concrete history so successors never stall
                cw[8] = 0; cw[9] = 0;
                __threadfence();
                st_release(&cw[0], kFlagInc);
            }
            __syncthreads();
            continue;
        }
        // ---- mantissa unpack (entropy.py:262-276) ----
        const int g0 = tid * gpt;
        const int g1 = (g0 + gpt < G) ? g0 + gpt : G;
        long long lbits = 0;
        for (int g = g0; g < g1; g++) lbits += 4 * (long long)e[g];
        long long tot;
        long long bitpos = cta_excl_scan(lbits, S->red, tot);
        {
            const uint32_t* w = (const uint32_t*)pay;
            long long bp = 8 * (S->pay_off + S->jee_bytes) + bitpos;
            for (int g = g0; g < g1; g++) {
                const int wd = e[g];
                for (int k = 0; k < 4; k++) {
                    long long v = 0;
                    if (wd) {
                        unsigned long long r = read_bits(w, bp, wd);
                        bp += wd;
                        if (r >> (wd - 1)) r -= (wd >= 64 ? 0ULL : (1ULL << wd));
                        v = (long long)r;
                    }
                    qb[4 * g + k] = v;
                }
            }
        }
        // ---- reconstruct (transform.py:116-129) ----
        const int sel = S->sel;
        // local inclusive scans over the thread's contiguous samples
        const int i0 = 4 * g0, i1 = 4 * g1;
        Aff M;
        if (sel >= 1) {
            unsigned long long acc = 0;
            for (int i = i0; i < i1; i++) { acc += (unsigned long long)qb[i]; qb[i] = (long long)acc; }
            long long t;
            long long ex = cta_excl_scan((long long)acc, S->red, t);
            for (int i = i0; i < i1; i++) qb[i] = (long long)((unsigned long long)qb[i] + (unsigned long long)ex);
            __syncthreads();
            if (sel == 2) {
                unsigned long long acc2 = 0;
                for (int i = i0; i < i1; i++) { acc2 += (unsigned long long)qb[i]; qb[i] = (long long)acc2; }
                long long ex2 = cta_excl_scan((long long)acc2, S->red, t);
                for (int i = i0; i < i1; i++) qb[i] = (long long)((unsigned long long)qb[i] + (unsigned long long)ex2);
                __syncthreads();
            }
        } else {
            __syncthreads();
        }
        // ---- carry look-back (affine maps) ----
        if (tid == 0) {
            const unsigned long long L1 = (unsigned long long)qb[np - 1];
            const unsigned long long L2 = (unsigned long long)qb[np - 2];
            const unsigned long long unp = (unsigned long long)np;
            if (sel == 0) { M = {0, 0, 0, 0, L1, L2}; }
            else if (sel == 1) { M = {1, 0, 1, 0, L1, L2}; }
            else { M = {unp + 1, (unsigned long long)0 - unp, unp, (unsigned long long)0 - (unp - 1), L1, L2}; }
            // history entering block 0 of the launch (apax_decode_range); restart
            // and D0 blocks have a constant map.  Every block keeps its map in
            // cw[1..6] (apax_decode_range composes them).
            unsigned long long in1 = P.entry_p1, in2 = P.entry_p2;
            if (sel == 0 || S->restart) { M = {0, 0, 0, 0, M.c1, M.c2}; in1 = 0; in2 = 0; }
            cw[1] = M.m11; cw[2] = M.m12; cw[3] = M.m21; cw[4] = M.m22; cw[5] = M.c1; cw[6] = M.c2;
            if (sel != 0 && !S->restart && b > 0) {
                // publish my map, then look back
                __threadfence();
                st_release(&cw[0], kFlagAgg);
                Aff acc = {1, 0, 0, 1, 0, 0};
                long long k = b - 1;
                for (;;) {
                    const unsigned long long* ck = P.carry + 16 * k;
                    unsigned long long fl = ld_acquire(&ck[0]);
                    if (fl == kFlagInc) {
                        unsigned long long p1 = ck[8], p2 = ck[9];
                        in1 = acc.m11 * p1 + acc.m12 * p2 + acc.c1;
                        in2 = acc.m21 * p1 + acc.m22 * p2 + acc.c2;
                        break;
                    }
                    if (fl == kFlagAgg) {
                        Aff Mk = {ck[1], ck[2], ck[3], ck[4], ck[5], ck[6]};
                        acc = aff_compose(acc, Mk);
                        k--;
                        continue;
                    }
                    __nanosleep(32);
                }
            }
            // concrete output history of this block
            unsigned long long o1 = M.m11 * in1 + M.m12 * in2 + M.c1;
            unsigned long long o2 = M.m21 * in1 + M.m22 * in2 + M.c2;
            cw[8] = o1; cw[9] = o2;
            __threadfence();
            st_release(&cw[0], kFlagInc);
            S->p1 = (long long)in1;
            S->p2 = (long long)in2;
        }
        __syncthreads();
        // ---- finalize q, dequantize, store (coalesced) ----
        {
            const unsigned long long p1 = (unsigned long long)S->p1, p2 = (unsigned long long)S->p2;
            const unsigned long long dd = p1 - p2;
            T* y = (T*)P.y + start;
            if (Tr::F) {
                const double s = decode_scale_code(S->code) * ldexp(1.0, S->fbe);
                for (int i = tid; i < n; i += kNT) {
                    unsigned long long qv = (unsigned long long)qb[i];
                    if (sel == 1) qv += p1;
                    else if (sel == 2) qv += p1 + (unsigned long long)(i + 1) * dd;
                    double v = __ddiv_rn((double)(long long)qv, s);
                    y[i] = (T)v;
                }
            } else {
                const double a = decode_scale_code(S->code);
                for (int i = tid; i < n; i += kNT) {
                    unsigned long long qv = (unsigned long long)qb[i];
                    if (sel == 1) qv += p1;
                    else if (sel == 2) qv += p1 + (unsigned long long)(i + 1) * dd;
                    long long yi = (a == 1.0) ? (long long)qv : f2i64(rint(__ddiv_rn((double)(long long)qv, a)));
                    yi = yi < Tr::LO ? Tr::LO : (yi > Tr::HI ? Tr::HI : yi);
                    y[i] = (T)yi;
                }
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Block walk (the serial boundary walk of codec.py:317-323): one warp parses
// each block's header + JEE + mantissa length.  offsets[b] = header offset,
// offsets[nb] = end.  Stops at the first error (status key).
// ---------------------------------------------------------------------------
// After K5 (apax_k5.cu, `k5_fail` non-null): on success only the last block
// is parsed (its group count may be short); on failure the offsets K5 wrote
// are reset and the full walk runs, reporting the reference's exact error.
__global__ void walk_kernel(const uint8_t* blob, long long nbytes, long long n, int bs, int dt,
                            long long n_blocks, long long* offsets, unsigned long long* status,
                            const int* k5_fail, const IlGate* gate) {
    if (gate && il_seg_ok(gate)) return;
    extern __shared__ __align__(16) unsigned char smem_w[];
    uint8_t* e = smem_w;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x >= 32) return;
    const int hs = hdr_size(dt);
    long long pos = kFileHeader;
    long long b0 = 0;
    if (k5_fail) {
        if (*k5_fail == 0) {
            b0 = n_blocks - 1;
            pos = offsets[b0];
        } else {
            for (long long b = lane; b <= n_blocks; b += 32) offsets[b] = -1;
            __syncwarp();
        }
    }
    for (long long b = b0; b < n_blocks; b++) {
        const long long start = b * (long long)bs;
        const int nn = (int)((n - start) < bs ? (n - start) : bs);
        const int G = (nn + 3) >> 2;
        if (lane == 0) offsets[b] = pos;
        if (nbytes - pos < hs) { if (lane == 0) report_error(status, b, APAX_ERR_BLOCK_HDR_TRUNCATED); return; }
        if ((blob[pos] & 3) == 3) { if (lane == 0) report_error(status, b, APAX_ERR_SELECTOR); return; }
        const uint8_t* p = blob + pos + hs;
        const long long avail = nbytes - pos - hs;
        const long long maxj = (3LL * G + 2) / 2;
        const long long nbj = avail < maxj ? avail : maxj;
        long long used = 0, esum = 0;
        int st = -1;
        if (b0 > 0) {   // after K5: the last block, fast parser first
            int u = 0;
            st = warp_jee_fast(p, blob + nbytes, (int)(2 * nbj), G, e, u);
            __syncwarp();
            if (st == 0) {
                unsigned sb = 0;
                for (int g = lane; g < G; g += 32) sb += e[g];
                esum = __reduce_add_sync(0xffffffffu, sb);
                used = u;
            }
        }
        if (st != 0) st = warp_jee_decode(p, 2 * nbj, G, e, used, esum);
        if (st) { if (lane == 0) report_error(status, b, st); return; }
        long long sz = (used + 1) / 2 + (4 * esum + 7) / 8;
        if (avail < sz) { if (lane == 0) report_error(status, b, APAX_ERR_MANTISSA_TRUNCATED); return; }
        pos += hs + sz;
        __syncwarp();
    }
    if (lane == 0) offsets[n_blocks] = pos;
}

size_t decode_smem_bytes(int dt, int bs, int payload_cap) {
    auto al = [](size_t v) { return (v + 15) & ~(size_t)15; };
    return al(sizeof(DecState)) + al((size_t)(bs + 4) * 8) + al((size_t)(bs / 4) + 16) +
           (size_t)payload_cap + 32;
}

template <int DT>
static int launch_decode_t(const DecParams& P, int grid, size_t smem, cudaStream_t st) {
    if (cudaFuncSetAttribute(decode_kernel<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return APAX_ERR_CUDA;
    note_launches(1);
    decode_kernel<DT><<<grid, kNT, smem, st>>>(P);
    return cudaGetLastError() == cudaSuccess ? APAX_OK : APAX_ERR_CUDA;
}

int decode_resident_ctas(int dt, size_t smem) {
    int dev = 0, nsm = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t err;
    switch (dt) {
        case 0: cudaFuncSetAttribute(decode_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, decode_kernel<0>, kNT, smem); break;
        case 1: cudaFuncSetAttribute(decode_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, decode_kernel<1>, kNT, smem); break;
        case 2: cudaFuncSetAttribute(decode_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, decode_kernel<2>, kNT, smem); break;
        case 3: cudaFuncSetAttribute(decode_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, decode_kernel<3>, kNT, smem); break;
        default: cudaFuncSetAttribute(decode_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, decode_kernel<4>, kNT, smem); break;
    }
    if (err != cudaSuccess || per < 1) per = 1;
    return per * (nsm > 0 ? nsm : 148);
}

int launch_decode(int dt, const DecParams& P, int grid, size_t smem, cudaStream_t st) {
    switch (dt) {
        case 0: return launch_decode_t<0>(P, grid, smem, st);
        case 1: return launch_decode_t<1>(P, grid, smem, st);
        case 2: return launch_decode_t<2>(P, grid, smem, st);
        case 3: return launch_decode_t<3>(P, grid, smem, st);
        case 4: return launch_decode_t<4>(P, grid, smem, st);
    }
    return APAX_ERR_ARG;
}

int launch_walk(const uint8_t* blob, long long nbytes, long long n, int bs, int dt, long long n_blocks,
                long long* offsets, unsigned long long* status, cudaStream_t st) {
    size_t smem = (size_t)(bs / 4) + 64;
    note_launches(1);
    walk_kernel<<<1, 32, smem, st>>>(blob, nbytes, n, bs, dt, n_blocks, offsets, status, nullptr, nullptr);
    return cudaGetLastError() == cudaSuccess ? APAX_OK : APAX_ERR_CUDA;
}

int launch_walk_after_k5(const uint8_t* blob, long long nbytes, long long n, int bs, int dt, long long n_blocks,
                         long long* offsets, unsigned long long* status, const int* k5_fail, cudaStream_t st,
                         const IlGate* gate) {
    size_t smem = (size_t)(bs / 4) + 64;
    note_launches(1);
    walk_kernel<<<1, 32, smem, st>>>(blob, nbytes, n, bs, dt, n_blocks, offsets, status, k5_fail, gate);
    return cudaGetLastError() == cudaSuccess ? APAX_OK : APAX_ERR_CUDA;
}

}  // namespace apax
