// apax_kernels.cuh -- parameter blocks and launch entry points shared by
// the kernels (apax_encode.cu, apax_decode.cu) and the C ABI (apax_capi.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/apax_b200.h"

namespace apax {

// per-block quantizer record of the split encoder: the chain writes it, the
// packer (apax_encode_v4.cu) re-quantizes the block with it
struct __align__(16) BlockMeta {
    double sq;       // quantizer multiplier (codec.py:94-132: a_q for ints, the float scale S)
    int code;        // 16-bit scale code
    short fbe;       // float block exponent
    short wide;      // max |q| > 2^30: 64-bit differences
};

struct EncParams {
    const void* x;
    long long n;
    int mode;              // 0 lossless, 1 fixed-rate, 2 fixed-quality
    int bs;
    double target;
    long long n_blocks;
    long long unit_blocks;
    long long n_units;
    long long unit_begin, unit_end;  // units processed by this launch (v3)
    int halo;              // 1: lossless whole-stream units (no restart)
    int policy;            // 0 cold, 1 warm_self (FR only)
    uint8_t* out;
    long long out_cap;
    long long* block_offsets;     // nullable, n_blocks + 1
    unsigned long long* status;   // 4 words
    unsigned long long* lookback; // n_units
    unsigned int* ticket;
    uint8_t* slots;               // gridDim.x slots of slot_bytes
    long long slot_bytes;
    int stage_bytes;              // staging window (bytes, multiple of 16)
    int x_in_smem;                // 1: stage each block's samples in smem
    double att_lo;                // 20*log10(2^-31), glibc (dtypes.py:202)
    double pow10_t20;             // 10**(T/20), glibc (codec.py:167)
    double sqrt12;                // math.sqrt(12)
    double* trace;                // nullable, 10 doubles per block
    long long gblock0;            // v3 lossless range encode: global index of block 0
                                  // (x[-bs-2 .. 0) holds the halo when > 0)
    // cast variants (generic kernel, kdt 5 / 6): the container's wire code and,
    // for integer containers, the dequantizer's clip range (codec.py:143-145)
    int wire;
    long long clip_lo, clip_hi;
    BlockMeta* meta;              // v5 (apax_encode_v5.cu): segments of full 4096-sample blocks, pack warps + a service warp
size_t encode_v5_smem_bytes(int dt);
bool encode_v5_supported(int dt, int bs, int mode, const EncParams& P);
int encode_v5_resident_ctas(int dt);
int launch_encode_v5(int dt, const EncParams& P, long long u0, long long u1, cudaStream_t st);
// split encoder: the chain's per-block records (v3 META)
    apax_block_state* state;      // generic kernel, one unit: CodecState in / out (encode_block)
    double* stats;                // fixed-quality chain: per block sum x^2, sum x*y, sum y*y (y = the decode)
    int count_only;               // packer: container length only, no output written
    int nsm;                      // v5 one-wave launches: SM count (units numbered by arrival rank), 0: by ticket
};

// Index-less decode state (apax_decode without offsets, apax_capi.cu):
// spec = 1 when the signature scan found exactly one candidate per block
// starting at byte 28 and wrote them as speculative offsets; first = the
// first restarting block > 0 (~0: none, a whole-stream container); gp =
// 0xFFFFFFFF while nothing contradicts the speculation.  The segment path
// runs while il_seg_ok; otherwise the full discovery (K5 parse, prune,
// walk) and the two-pass decode run.
struct IlGate {
    unsigned long long first;
    unsigned int gp;
    unsigned int spec;
};
__device__ __forceinline__ bool il_seg_ok(const IlGate* g) {
    return g->spec && g->first != ~0ULL && g->first > 0 && g->gp == 0xFFFFFFFFu;
}

struct DecParams {
    const uint8_t* blob;
    long long nbytes;
    const long long* offsets;   // n_blocks + 1 (entries < 0: block not present)
    void* y;
    long long n;
    int bs;
    long long n_blocks;
    unsigned long long* status; // 4 words
    unsigned long long* carry;  // 8 words per block
    unsigned int* ticket;
    int payload_cap;            // smem bytes reserved for one block payload
    long long segment_blocks;   // d3: every segment_blocks-th block starts a segment
    long long seg_begin, seg_end;
    // v2 range decode (apax_decode_range): derivative history entering
    // block 0 of this launch when it is not a restart block (default 0, 0)
    unsigned long long entry_p1, entry_p2;
    // d3 two-pass decode of any container (apax_decode): pass 1 writes each
    // segment's history map (A11, A12, A21, A22, c1, c2) to seg_map and skips
    // the samples (no_store); pass 2 starts segment k from seg_entry[2k..2k+1]
    unsigned long long* seg_map;
    const unsigned long long* seg_entry;
    int no_store;
    // index-less decode (apax_decode without offsets), see IlGate: d3 with
    // il_gate set and TP 0 decodes the speculative segments (seg_part 1: the
    // full-block segments, 2: the last one, 0: all), checking every block's
    // length against the speculative offsets; the two-pass kernels with
    // il_gate set run only when that path was not taken or failed
    IlGate* il_gate;
    // the second chance of an index-less decode: after the full discovery
    // (the speculation failed, e.g. a false candidate in integer data), the
    // segment path on the verified offsets (il_gate2->first, normal error
    // reports); the two-pass kernels then run only when neither path did
    IlGate* il_gate2;
    int seg_part;
    // two-pass decode: pass 1 saves every block's parsed JEE (group widths,
    // mantissa bit offsets, header, scale: kJeeRecBytes per block) and pass 2
    // loads it instead of parsing the tokens again (nullptr: parse again)
    uint8_t* jee_cache;
    // index-less decode: the block discovery's candidate parse filled the
    // records of blocks 0 .. n_blocks-2 when its two flags (fail, chain_bad)
    // are both zero -- every candidate was a block; pass 1 then loads them too
    const int* jee_k5;
};
constexpr long long kJeeRecBytes = 1600;   // 16 jinfo + 16 scale + 32 warp bits + 512 thread bits + 1024 widths

// kernel launches enqueued by the library (apax_launch_count)
void note_launches(int k);

size_t encode_smem_bytes(int dt, int bs, int stage_bytes, int x_in_smem);
int encode_resident_ctas(int dt, size_t smem);
int launch_encode(int dt, const EncParams& P, int grid, size_t smem, cudaStream_t st);
size_t decode_smem_bytes(int dt, int bs, int payload_cap);
int decode_resident_ctas(int dt, size_t smem);
size_t encode_v3_smem_bytes(int dt, int bs, int stage_bytes);
int encode_v3_stage_bytes(int dt, int bs);
bool encode_v3_supported(int dt, int bs);
int encode_v3_resident_ctas(int dt, size_t smem);
int encode_v3_resident_ctas_wave(int dt, size_t smem);
int launch_encode_v3(int dt, const EncParams& P, int grid, size_t smem, cudaStream_t st);
// v5 (apax_encode_v5.cu): segments of full 4096-sample blocks, pack warps + a service warp
size_t encode_v5_smem_bytes(int dt);
bool encode_v5_supported(int dt, int bs, int mode, const EncParams& P);
int encode_v5_resident_ctas(int dt);
int launch_encode_v5(int dt, const EncParams& P, long long u0, long long u1, cudaStream_t st);
// split encoder: the chain (v3 with META: quantizer records, no output) and
// the block-parallel packer (apax_encode_v4.cu)
int launch_encode_v3_chain(int dt, const EncParams& P, size_t smem, cudaStream_t st);
size_t encode_v4_smem_bytes(int dt);
bool encode_v4_supported(int dt, int bs);
int encode_v4_resident_ctas(int dt);
bool encode_ws_supported(int dt, int bs);
size_t encode_ws_smem_bytes(int dt, int mode);
int launch_encode_ws_chain(int dt, const EncParams& P, cudaStream_t st);
int launch_encode_v4(int dt, const EncParams& P, const BlockMeta* meta, unsigned long long* costs,
                     unsigned long long* lb, cudaStream_t st);
int launch_decode(int dt, const DecParams& P, int grid, size_t smem, cudaStream_t st);
size_t decode_v3_smem_bytes(int dt, int payload_cap);
bool decode_v3_supported(int dt, int bs);
int decode_v3_resident_ctas(int dt, size_t smem);
int launch_decode_v3(int dt, const DecParams& P, int grid, size_t smem, cudaStream_t st);
int launch_decode_v3_seg_dev(int dt, DecParams P, int grid, size_t smem, cudaStream_t st);
// index-less speculation (apax_k5.cu): signature scan + speculative offsets;
// the scan also sets gate->first (the first restarting block > 0) from the
// candidates it places and initialises gate2 (all ones) for the second chance
int launch_k5_speculate(const uint8_t* blob, long long nbytes, int dt, long long n_blocks, long long* offsets,
                        void* ws, IlGate* gate, IlGate* gate2, cudaStream_t st);
int launch_decode_v3_two_pass(int dt, DecParams P, int grid, size_t smem, unsigned long long* scratch,
                              cudaStream_t st);
size_t decode_v2_smem_bytes(int dt, int bs, int payload_cap);
bool decode_v2_supported(int bs);
int decode_v2_resident_ctas(int dt, size_t smem);
int launch_decode_v2(int dt, const DecParams& P, int grid, size_t smem, cudaStream_t st);
int launch_compose_maps(const unsigned long long* carry, long long nb, unsigned long long* out, cudaStream_t st);
int profile_sums(const void* x, const void* y, long long n, int dt, int pass, double mx, double my,
                 double md, double* partials, unsigned long long* counts, int grid, cudaStream_t st);
size_t profile_welch_smem(int seg);
int profile_welch(const void* x, const void* y, long long n, int dt, int which, int seg, int lg,
                  long long nframes, const double* tw, double* partials, int grid, cudaStream_t st);
int profile_select(const void* x, const void* y, long long n, int dt, int pass,
                   const unsigned long long* prefixes, int npre, unsigned* hist, int ydiff, int grid,
                   cudaStream_t st);
int launch_walk(const uint8_t* blob, long long nbytes, long long n, int bs, int dt, long long n_blocks,
                long long* offsets, unsigned long long* status, cudaStream_t st);
int launch_walk_after_k5(const uint8_t* blob, long long nbytes, long long n, int bs, int dt, long long n_blocks,
                         long long* offsets, unsigned long long* status, const int* k5_fail, cudaStream_t st,
                         const IlGate* gate = nullptr);
// K5 index-less block discovery (apax_k5.cu); ws of find_blocks_k5_ws_bytes
size_t find_blocks_k5_ws_bytes(long long n_blocks);
// gate non-null: the discovery after launch_k5_speculate (scan reused),
// every kernel returns at once while il_seg_ok(gate)
// jee_cache non-null (block sizes up to 4096): the candidate parse also writes
// candidate i's parse as record i (DecParams::jee_cache); k5_flags(ws) are the
// two ints that say whether candidate i is block i (DecParams::jee_k5)
int launch_find_blocks_k5(const uint8_t* blob, long long nbytes, long long n, int bs, int dt, long long n_blocks,
                          long long* offsets, unsigned long long* status, void* ws, cudaStream_t st,
                          const IlGate* gate = nullptr, uint8_t* jee_cache = nullptr);
const int* k5_flags(void* ws, long long n_blocks);

}  // namespace apax
