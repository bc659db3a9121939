/*
 * apax_b200.h -- C ABI of the B200-native APAX codec (libapax_b200.so).
 *
 * Plain pointers and sizes only (no torch types).  All buffer arguments are
 * DEVICE pointers (cudaMalloc / torch CUDA tensors) unless marked host; every
 * call enqueues on `stream` (a cudaStream_t, NULL = legacy default stream)
 * and returns without synchronising.  Host return values are synchronous
 * argument/launch errors; data-dependent errors (corrupt stream, non-finite
 * input, ...) land in the 4-word device `status` buffer, read after the
 * caller synchronises:
 *     status[0]  first non-finite sample index (UINT64_MAX if none)
 *     status[1]  (block_index << 8) | apax_status of the first failing block
 *                (UINT64_MAX if none; lowest block wins, like the serial walk)
 *     status[2]  encode: total container bytes written
 *     status[3]  reserved
 * Status codes: include/apax_status.h (1:1 with the reference exceptions).
 *
 * Reference interfaces replaced (paths relative to the reference package):
 *   apax_encode           <- encode_stream       pkg/src/apax/codec.py:258-285
 *                            (+ encode_block     pkg/src/apax/codec.py:192-255)
 *   apax_decode           <- decode_stream       pkg/src/apax/codec.py:308-329
 *   apax_find_blocks      <- the block walk in   pkg/src/apax/codec.py:317-323
 *   apax_max_encoded_bytes: output sizing (no reference counterpart; the
 *                            reference returns fresh `bytes`)
 *   apax_parse_file_header <- parse_file_header  pkg/src/apax/codec.py:288-305
 *                            (host pointer, host-side)
 */
#ifndef APAX_B200_H
#define APAX_B200_H

#include <stdint.h>

#include "apax_status.h"

#ifdef __cplusplus
extern "C" {
#endif

/* wire codes (reference dtypes.py:24-28, 55-58) */
enum { APAX_I8 = 0, APAX_I16 = 1, APAX_I32 = 2, APAX_F32 = 3, APAX_F64 = 4 };
enum { APAX_LOSSLESS = 0, APAX_FIXED_RATE = 1, APAX_FIXED_QUALITY = 2 };
enum { APAX_POLICY_COLD = 0, APAX_POLICY_WARM_SELF = 1 };

/* The reference's per-stream encoder state (CodecState, codec.py:66-82):
 * attenuation, derivative history, the previous block's stream costs
 * (StreamCosts: 4*sum(e) + 4*groups per stream), blocks emitted, and
 * whether the fixed-quality gain was initialised.  apax_encode_block reads
 * it and writes the state after the block back. */
typedef struct {
    double att_db;
    int64_t prev1, prev2;
    int64_t costs[3];
    int32_t has_costs;
    int32_t initialized;
    int64_t blocks_emitted;
} apax_block_state;

/* Library version string. */
const char* apax_version(void);

/* Kernel launches this library has enqueued since it was loaded (every
 * entry point counts its own launches; for launch accounting in benchmarks). */
int64_t apax_launch_count(void);

/* Human-readable text for a status code. */
const char* apax_status_string(int code);

/* Worst-case container size for n samples (28-byte file header included). */
int64_t apax_max_encoded_bytes(int64_t n, int dtype, int block_size);

/* Segment length (blocks) that gives every resident encoder CTA of this
 * device exactly one segment of n samples: the one-wave schedule.  A
 * convenience for choosing segment_blocks; the container depends only on
 * the value passed to apax_encode. */
int64_t apax_encode_wave_segment_blocks(int64_t n, int dtype, int mode, int block_size);

/* Name of the kernel that codes the full blocks of a container with these
 * parameters on this device (for profiler look-ups and benchmark labels;
 * the library's dispatch, not a knob). */
const char* apax_encode_kernel_name(int dtype, int mode, int block_size, int64_t segment_blocks);

/* Decode blocks [b0, b1) of a container of n samples (whole-stream or
 * segmented) given the GLOBAL side-band index `block_offsets` and the
 * derivative history (q[-1], q[-2] as two's-complement u64) entering block b0
 * (ignored when b0 is a restart or D0 block; transform.py:31-49).  y receives
 * samples b0*bs .. min(n, b1*bs); status block indices are relative to b0.
 * map_out (nullable, 6 device words) receives the range's history map
 * (m11, m12, m21, m22, c1, c2): the history leaving block b1-1 is
 * M*(entry) + c, mod 2^64.  Multi-GPU decode of a whole-stream container
 * (SURVEY.md §8(e)): every rank decodes its block range with entry (0, 0)
 * and map_out, all-gathers the maps, composes them in rank order and
 * re-decodes with its exact entry (paper_1303_4994_b200/distributed.py).
 * Workspace: apax_decode_workspace_bytes(samples of the range, dtype, bs). */
int apax_decode_range(const uint8_t* blob, int64_t nbytes, int64_t n, int dtype, int block_size,
                      const int64_t* block_offsets, int64_t b0, int64_t b1, uint64_t entry_p1,
                      uint64_t entry_p2, void* y, uint64_t* map_out, uint64_t* status, void* ws,
                      int64_t ws_bytes, void* stream);

/* LOSSLESS whole-stream encode of the blocks from first_block on, as a
 * container of their own whose body (bytes after the 28-byte file header)
 * equals those blocks' bytes in the one-call whole-stream container
 * (apax_encode, segment_blocks <= 0): x[0] is global sample first_block*bs
 * and x[-halo .. 0) must hold the preceding samples, halo >= bs + 2 (bs for
 * first_block == 1, 0 for first_block == 0): the previous block and the two
 * samples before it rebuild the first block's codec state (selector costs
 * and derivative history; reference codec.py:192-255).
 * The multi-GPU LOSSLESS encode of SURVEY.md §8(e): rank r receives that
 * halo from rank r-1.  Power-of-two block sizes 128..4096. */
int apax_encode_lossless_range(const void* x, int64_t halo, int64_t n, int dtype, int block_size,
                               int64_t first_block, uint8_t* out, int64_t out_cap, int64_t* block_offsets,
                               uint64_t* status, void* ws, int64_t ws_bytes, void* stream);

/* Segment length of a container from its block index (device pointers):
 * writes P to *segment_blocks_out when block b carries the restart flag
 * (header byte 0, bit 2) exactly for b % P == 0, else 0 (a
 * whole-stream container, or any other pattern).  Lets an index-less decode
 * of a segmented container (offsets from apax_find_blocks) take
 * apax_decode_segments.  One CTA; enqueued on `stream`. */
int apax_detect_segments(const uint8_t* blob, int64_t nbytes, const int64_t* block_offsets, int64_t n_blocks,
                         uint64_t* segment_blocks_out, void* stream);

/* Copy n_words (1..32) status words from a device status buffer to PAGE-LOCKED
 * HOST memory (cudaHostAlloc / torch pin_memory) with stores issued by one
 * thread block, enqueued on `stream`.  For pipelined host round trips: a
 * 32-byte copy-engine D2H would queue behind the bulk sample copies of other
 * chunks.  No reference counterpart (the reference is synchronous). */
int apax_status_to_host(const uint64_t* status, uint64_t* host_dst, int n_words, void* stream);

/* Device workspace needed by apax_encode for these arguments. */
int64_t apax_encode_workspace_bytes(int64_t n, int dtype, int mode, int block_size,
                                    int64_t segment_blocks);

/* Encode n samples of `dtype` at x (device) into a container at out (device).
 *   segment_blocks <= 0 : whole-stream semantics, byte-identical to the
 *                         reference encode_stream (LOSSLESS is still block
 *                         parallel; FIXED_RATE / FIXED_QUALITY run as one
 *                         serial chain).
 *   segment_blocks  > 0 : container of independent segments of that many
 *                         blocks, each a fresh CodecState with restart flag
 *                         (decodable by the unmodified reference decoder).
 *   policy              : APAX_POLICY_COLD (= reference encode_stream per
 *                         segment) or APAX_POLICY_WARM_SELF (FIXED_RATE:
 *                         attenuator preset from the segment's first block).
 *                         Ignored when segment_blocks <= 0: a whole stream
 *                         is always the reference's encode_stream.
 *   out_cap must be >= apax_max_encoded_bytes(n, dtype, block_size).
 *   block_offsets (nullable, n_blocks + 1 int64): byte offset of every block
 *   header, then the container length (side-band index for apax_decode).
 *   trace (nullable, 10 doubles per block): att_db, a, code, fbe, selector,
 *   cost0..2, block bytes, restart.
 *   status: 4 uint64 (device).  ws/ws_bytes: device workspace. */
int apax_encode(const void* x, int64_t n, int dtype, int mode, double target, int block_size,
                int64_t segment_blocks, int policy, uint8_t* out, int64_t out_cap,
                int64_t* block_offsets, uint64_t* status, double* trace, void* ws,
                int64_t ws_bytes, void* stream);

/* encode_stream's input conversions (reference codec.py:266-272 widens every
 * input to int64 for integer configs and to float64 for float configs, then
 * quantizes those values).  in_kind:
 *   APAX_IN_NATIVE  samples already of `dtype` (= apax_encode);
 *   APAX_IN_INT64   int64 samples, integer dtype: values outside the dtype's
 *                   range are coded as they are (exponents up to 34) and
 *                   clipped by the decoder (codec.py:143-145);
 *   APAX_IN_FLOAT64 float64 samples, F32 (or F64) dtype: quantized from the
 *                   f64 values, the fixed-quality loop measures the f32 y.
 * The cast kinds run the generic encoder (any block size).  out_cap must be
 * >= apax_max_encoded_bytes_cast (exponents up to 34 for every block). */
enum { APAX_IN_NATIVE = 0, APAX_IN_INT64 = 1, APAX_IN_FLOAT64 = 2 };
int64_t apax_max_encoded_bytes_cast(int64_t n, int in_kind, int dtype, int block_size);
int64_t apax_encode_cast_workspace_bytes(int64_t n, int in_kind, int dtype, int mode, int block_size,
                                         int64_t segment_blocks);
int apax_encode_cast(const void* x, int in_kind, int64_t n, int dtype, int mode, double target, int block_size,
                     int64_t segment_blocks, int policy, uint8_t* out, int64_t out_cap, int64_t* block_offsets,
                     uint64_t* status, void* ws, int64_t ws_bytes, void* stream);

/* ---- the reference's lower-level block API (codec.py:94-255) ----
 * quantize_block: x (device) holds n samples widened as the reference does
 * (float64 for float dtypes, int64 for integer ones); q (device, int64[n])
 * receives the quantized block, hdr (device, int32[2]) the scale code and the
 * float block exponent.  Errors (non-finite input, s_des overflow) land in
 * status as block 0.  One CTA. */
int apax_quantize_block(const void* x, int64_t n, int dtype, double a, int64_t* q, int32_t* hdr,
                        uint64_t* status, void* stream);
/* dequantize_block: y (device, n samples of dtype) = the decoder's dual of
 * q under (scale code, float block exponent). */
int apax_dequantize_block(const int64_t* q, int64_t n, int dtype, int code, int fbe, void* y, void* stream);
/* encode_block: one block of n <= block_size samples (widened as above)
 * under the state at *state (device), which receives the state after the
 * block; out (device) receives the 28-byte file header, the block header and
 * payload (status[2] = total bytes).  Workspace:
 * apax_encode_cast_workspace_bytes(block_size, in_kind, dtype, mode,
 * block_size, 0). */
int apax_encode_block(const void* x, int64_t n, int dtype, int mode, double target, int block_size,
                      apax_block_state* state, uint8_t* out, int64_t out_cap, uint64_t* status, void* ws,
                      int64_t ws_bytes, void* stream);

/* The profiler's output-free sweep point (rate_correlation_sweep,
 * profiler.py:176-199): a whole-stream fixed-quality encode of x at
 * `target` that writes no container -- status[2] receives the container's
 * length and stats[3b .. 3b+2] block b's (sum x^2, sum x*y, sum y*y) with y
 * the decode of x (the encoder's own dequantized block, bit-identical to
 * the decoder's).  Block size 4096, dtype
 * i16/i32/f32/f64, x 16-byte aligned; stats holds 3 * n_blocks doubles. */
int64_t apax_sweep_point_workspace_bytes(int64_t n, int dtype);
int apax_sweep_point(const void* x, int64_t n, int dtype, double target, double* stats, uint64_t* status, void* ws,
                     int64_t ws_bytes, void* stream);

/* Device workspace needed by apax_decode (with offsets == NULL it includes
 * room for the block walk's offset table; for block sizes up to 4096 also
 * 1600 bytes per block: the parse pass 1 of a two-pass decode saves for
 * pass 2). */
int64_t apax_decode_workspace_bytes(int64_t n, int dtype, int block_size);

/* Decode a container body.  blob (device) holds the full container of
 * `nbytes` bytes (file header included; the caller parsed the header with
 * apax_parse_file_header for n / dtype / block_size).  block_offsets
 * (device, nullable): n_blocks + 1 offsets from apax_encode or
 * apax_find_blocks; NULL runs block discovery (K5, see apax_find_blocks)
 * first.  y (device) receives n
 * samples of dtype. */
int apax_decode(const uint8_t* blob, int64_t nbytes, int64_t n, int dtype, int block_size,
                const int64_t* block_offsets, void* y, uint64_t* status, void* ws,
                int64_t ws_bytes, void* stream);

/* Decode a container of independent segments (every segment_blocks-th
 * block carries the restart flag, as apax_encode writes with
 * segment_blocks > 0) given its side-band block index: one CTA per segment,
 * history kept on chip.  Same arguments and status contract as apax_decode;
 * falls back to apax_decode when the fast path does not apply (no index,
 * segment_blocks <= 0, f64, or block sizes other than powers of two in
 * 128..4096).  Workspace: apax_decode_segments_workspace_bytes. */
int64_t apax_decode_segments_workspace_bytes(int64_t n, int dtype, int block_size);
int apax_decode_segments(const uint8_t* blob, int64_t nbytes, int64_t n, int dtype, int block_size,
                         const int64_t* block_offsets, int64_t segment_blocks, void* y, uint64_t* status,
                         void* ws, int64_t ws_bytes, void* stream);

/* Block boundaries of a container without a side-band index (replaces the
 * reference's serial walk, codec.py:317-323): offsets (device,
 * n_blocks + 1) receives every block header offset and the end offset;
 * errors go to status[1] with the walk's block index.  Runs K5 (parallel
 * signature candidates + per-candidate JEE parse + exact verification of
 * the walk recurrence, apax_k5.cu) with the serial walk as the exact
 * fallback; APAX_K5=0 in the environment forces the serial walk.  Scratch
 * comes from the stream-ordered allocator (cudaMallocAsync).  apax_decode
 * with block_offsets == NULL runs the same discovery in its workspace. */
int apax_find_blocks(const uint8_t* blob, int64_t nbytes, int64_t n, int dtype, int block_size,
                     int64_t* offsets, uint64_t* status, void* stream);

/* ---- profiler statistics (reference pkg/src/apax/profiler.py) ----
 * x, y: device arrays of n samples of `dtype` (input and decoded output);
 * d = x - y in double precision.  Every call writes per-CTA partials
 * (apax_profile_grid() of them) that the caller sums in CTA order, so
 * results are run-to-run deterministic. */
int apax_profile_grid(void);

/* pass 0: partials[g*8 + k] = sums over CTA g of
 *   k = 0 x, 1 y, 2 d, 3 x^2, 4 y^2, 5 d^2, 6 x*y      (pearson_r :40-48,
 *   window2_metrics :127-159); counts[0] += #(x == 0 and d != 0),
 *   counts[1] += #(d == 0) (caller zeroes counts).
 * pass 1 (centred, for the two-pass std): k = 3 (x-mean_x)^2,
 *   4 (y-mean_y)^2, 5 (d-mean_d)^2. */
int apax_profile_sums(const void* x, const void* y, int64_t n, int dtype, int pass, double mean_x, double mean_y,
                      double mean_d, double* partials, uint64_t* counts, void* stream);

/* Welch power sums (welch_spectrum :61-74): frames of `seg` samples (power
 * of two, 2..4096) at hop seg/2; partials[g*(seg/2+1) + k] = sum over the
 * frames of CTA g of |FFT(hann * frame)_k|^2.  which: 0 x, 1 y, 2 d.
 * tables (device): seg/2 twiddles exp(-2 pi i k/seg) as (re, im) pairs,
 * then the seg window values. */
int apax_profile_welch(const void* x, const void* y, int64_t n, int dtype, int which, int seg,
                       const double* tables, double* partials, void* stream);

/* One pass of the 4-pass radix multi-select over the per-sample ratio keys
 * (s2r_distribution :105-124): key = bits of |x| / |d| (d == 0: +inf,
 * x == 0 != d: 0; the sign bit is 0), d = x - y when y_is_output, else y
 * itself is d.  Digits, most significant first: pass 0 bits 62..48 (15
 * bits, hist[digit], 2^15 uint32, prefixes unused), passes 1..3 bits
 * 47..32, 31..16, 15..0 of the keys whose higher bits equal one of the
 * sorted, unique `prefixes`: hist[j * 65536 + digit].  The caller zeroes
 * hist; n < 2^32. */
int apax_profile_select(const void* x, const void* y, int64_t n, int dtype, int pass, const uint64_t* prefixes,
                        int n_prefixes, uint32_t* hist, int y_is_output, void* stream);

/* Host-side parse of the 28-byte file header (host pointer).  Returns an
 * apax_status code; *detail carries the offending value for messages. */
int apax_parse_file_header(const uint8_t* host_blob, int64_t len, int* dtype, int* mode,
                           int* block_size, int64_t* count, double* target, int64_t* detail);

#ifdef __cplusplus
}
#endif

#endif
