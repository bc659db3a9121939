// apax_capi.cu -- extern "C" boundary of libapax_b200.so (include/apax_b200.h).
//
// Host side: argument validation, workspace carving, glibc-evaluated host
// constants (the clamp bound 20*log10(2^-31) of reference dtypes.py:202 and
// 10**(T/20) of codec.py:167 are computed here with the same libm the
// reference's CPython calls), status-buffer reset, kernel launches.
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <cuda_runtime.h>

#include "../../include/apax_b200.h"
#include "apax_device.cuh"

#include "apax_kernels.cuh"

using namespace apax;

namespace apax {
static std::atomic<long long> g_launches{0};
void note_launches(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
}  // namespace apax

namespace {

constexpr long long kLosslessUnit = 4;  // blocks per CTA unit, lossless whole stream

struct EncPlan {
    long long n_blocks, unit_blocks, n_units;
    int halo;
    int stage_bytes;
    int x_in_smem;
    int v3;
    int split;             // chain (v3 META) + block-parallel packer (v4)
    size_t smem;
    int grid;
    long long slot_bytes;
    long long ws_lookback, ws_ticket, ws_slots, ws_v4, ws_total;
};

bool valid_dtype(int dt) { return dt >= 0 && dt <= 4; }

int env_int(const char* name, int def) {
    const char* v = getenv(name);
    if (!v || !*v) return def;
    return atoi(v);
}

// kdt: the kernel's sample type -- a container dtype 0..4, or a cast variant
// (kKdtI64: int64 samples for an integer container, kKdtF64F32: float64
// samples for an f32 container; generic v1 kernel only)
int plan_encode(long long n, int kdt, int mode, int bs, long long seg, EncPlan* p) {
    if (kdt < 0 || kdt > kKdtF64F32 || mode < 0 || mode > 2) return APAX_ERR_ARG;
    if (bs < 64 || bs > 16384) return APAX_ERR_CFG_BLOCK_RANGE;
    if (bs % 4) return APAX_ERR_CFG_BLOCK_MULT;
    if (n < 1) return APAX_ERR_EMPTY;
    p->n_blocks = (n + bs - 1) / bs;
    if (seg > 0) {
        p->unit_blocks = seg < p->n_blocks ? seg : p->n_blocks;
        p->halo = 0;
    } else if (mode == APAX_LOSSLESS) {
        p->unit_blocks = kLosslessUnit;
        p->halo = 1;
    } else {
        p->unit_blocks = p->n_blocks;
        p->halo = 0;
    }
    p->n_units = (p->n_blocks + p->unit_blocks - 1) / p->unit_blocks;
    const long long mbb = max_block_bytes(kdt, bs);
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess ||
        optin <= 0)
        optin = 227 * 1024;
    p->v3 = kdt <= 4 && encode_v3_supported(kdt, bs) && env_int("APAX_FORCE_V1", 0) == 0;
    long long v3_slots = 0;
    if (p->v3) {
        p->stage_bytes = encode_v3_stage_bytes(kdt, bs);
        p->x_in_smem = 1;
        p->smem = encode_v3_smem_bytes(kdt, bs, p->stage_bytes);
        if (p->smem > (size_t)optin) p->v3 = 0;
    }
    if (p->v3) {
        // one unit per CTA fits: the 256-thread one-wave kernel (one slot per
        // CTA); else the persistent kernel with a placement warp (two slots)
        const int rw = encode_v3_resident_ctas_wave(kdt, p->smem);
        const int resident = encode_v3_resident_ctas(kdt, p->smem);
        if (p->n_units <= rw) {
            p->grid = (int)p->n_units;
            v3_slots = p->n_units;
        } else {
            p->grid = (int)(p->n_units < resident ? p->n_units : resident);
            v3_slots = 2LL * p->grid > rw ? 2LL * p->grid : rw;   // a sub-range may run one-wave
        }
    } else {
        // generic kernel (any block size, the cast variants)
        long long want = env_int("APAX_STAGE_BYTES", 48 * 1024);
        long long st = want > mbb + 64 ? want : mbb + 64;
        st = (st + 15) & ~15LL;
        p->stage_bytes = (int)st;
        p->x_in_smem = 1;
        p->smem = encode_smem_bytes(kdt, bs, p->stage_bytes, 1);
        if (p->smem > (size_t)optin) {
            p->x_in_smem = 0;
            p->smem = encode_smem_bytes(kdt, bs, p->stage_bytes, 0);
        }
        int resident = encode_resident_ctas(kdt, p->smem);
        p->grid = (int)(p->n_units < resident ? p->n_units : resident);
    }
    if (p->grid < 1) p->grid = 1;
    p->slot_bytes = (p->n_units > 1 || p->v3) ? ((p->unit_blocks * mbb + 64 + 255) & ~255LL) : 0;
    p->ws_lookback = 0;
    p->ws_ticket = (p->n_units * 8 + 255) & ~255LL;
    // ticket words, then v5's unit numbering tables (per-SM arrival counts,
    // per-rank counts, one claim word per unit)
    p->ws_slots = p->ws_ticket + 256 + ((8448 + 4 * p->n_units + 255) & ~255LL);
    p->ws_total = p->ws_slots + p->slot_bytes * (p->v3 ? v3_slots : (long long)p->grid);
    // split encoder (bs 4096, i16/i32/f32/f64): per-block quantizer records,
    // published costs, look-back words, one ticket counter
    // (segmented fixed-rate / fixed-quality containers stay on the fused v3
    // kernel: one CTA per segment is faster there, tools/time_encode.py)
    const int sp = env_int("APAX_ENC_SPLIT", -1);
    p->split = p->v3 && encode_v4_supported(kdt, bs) &&
               (sp == 1 || (sp < 0 && (seg <= 0 || mode == APAX_LOSSLESS)));
    p->ws_v4 = (p->ws_total + 255) & ~255LL;
    if (p->split) p->ws_total = p->ws_v4 + p->n_blocks * (16 + 8 + 8) + 256;
    return APAX_OK;
}

struct DecPlan {
    long long n_blocks;
    int payload_cap;
    int v2;
    size_t smem;
    int grid;
    long long ws_carry, ws_ticket, ws_offsets, ws_k5, ws_jee, ws_total;
};

int plan_decode(long long n, int dt, int bs, DecPlan* p) {
    if (!valid_dtype(dt)) return APAX_ERR_ARG;
    if (bs < 64 || bs > 16384) return APAX_ERR_CFG_BLOCK_RANGE;
    if (bs % 4) return APAX_ERR_CFG_BLOCK_MULT;
    if (n < 0) return APAX_ERR_ARG;
    p->n_blocks = (n + bs - 1) / bs;
    long long cap = max_block_bytes_any(dt, bs) + 64;
    p->payload_cap = (int)((cap + 15) & ~15LL);
    p->v2 = decode_v2_supported(bs) && env_int("APAX_FORCE_V1", 0) == 0;
    int resident;
    if (p->v2) {
        p->smem = decode_v2_smem_bytes(dt, bs, p->payload_cap);
        resident = decode_v2_resident_ctas(dt, p->smem);
    } else {
        p->smem = decode_smem_bytes(dt, bs, p->payload_cap);
        resident = decode_resident_ctas(dt, p->smem);
    }
    long long g = p->n_blocks < resident ? p->n_blocks : resident;
    p->grid = (int)(g < 1 ? 1 : g);
    p->ws_carry = 0;
    p->ws_ticket = (p->n_blocks * 128 + 255) & ~255LL;
    p->ws_offsets = p->ws_ticket + 256;
    p->ws_k5 = p->ws_offsets + (((p->n_blocks + 1) * 8 + 255) & ~255LL);
    p->ws_jee = (p->ws_k5 + (long long)find_blocks_k5_ws_bytes(p->n_blocks) + 255) & ~255LL;
    // the two-pass decode's saved JEE parse (apax_decode_v3.cu, DecParams::jee_cache)
    p->ws_total = p->ws_jee + (decode_v3_supported(dt, bs) ? p->n_blocks * kJeeRecBytes : 0);
    return APAX_OK;
}

}  // namespace

namespace {
// segment structure of a container from its block index: the restart flags
// (header byte 0, bit 2) must sit exactly on the multiples of the first
// restart block's index P > 0; out[0] = P, or 0 when the pattern does not
// hold (or no block but the first restarts)
__global__ void detect_segments_kernel(const uint8_t* blob, long long nbytes, const long long* offs,
                                       long long nb, unsigned long long* out) {
    __shared__ unsigned long long first;
    __shared__ int broken;
    if (threadIdx.x == 0) { first = ~0ULL; broken = 0; }
    __syncthreads();
    for (long long b = 1 + threadIdx.x; b < nb; b += blockDim.x) {
        const long long o = offs[b];
        if (o < 0 || o >= nbytes) { broken = 1; continue; }
        if ((blob[o] >> 2) & 1) atomicMin(&first, (unsigned long long)b);
    }
    __syncthreads();
    const unsigned long long P = first;
    if (P != ~0ULL) {
        for (long long b = 1 + threadIdx.x; b < nb; b += blockDim.x) {
            const long long o = offs[b];
            const int r = (o >= 0 && o < nbytes) ? ((blob[o] >> 2) & 1) : 0;
            if (r != ((unsigned long long)b % P == 0 ? 1 : 0)) broken = 1;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[0] = (P == ~0ULL || broken) ? 0ULL : P;
}

// index-less decode: the first restarting block > 0 (the segment length of
// a segmented container) -> target->first.  The speculative pass (skip
// null) runs on the candidate offsets when the scan found one per block;
// the second (after the full discovery, skip = the first gate) only when
// the speculation failed, and clears target->gp on a discovery error.
__global__ void seg_first_kernel(const uint8_t* blob, long long nbytes, const long long* offs, long long nb,
                                 IlGate* target, const IlGate* skip, const unsigned long long* status) {
    if (skip && il_seg_ok(skip)) return;
    if (!target->spec) return;
    const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (status && i0 == 0 && status[1] != ~0ULL) atomicExch(&target->gp, 0u);
    unsigned long long mine = ~0ULL;
    bool bad = false;
    for (long long b = 1 + i0; b < nb; b += (long long)gridDim.x * blockDim.x) {
        const long long o = offs[b];
        if (o < 0 || o >= nbytes) { bad = true; continue; }
        if (((blob[o] >> 2) & 1) && (unsigned long long)b < mine) mine = (unsigned long long)b;
    }
    if (mine != ~0ULL) atomicMin(&target->first, mine);
    if (bad && status) atomicExch(&target->gp, 0u);
}

static int seg_first_grid(long long nb) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    long long g = (nb + 255) / 256;
    if (g > nsm) g = nsm;
    return (int)(g < 1 ? 1 : g);
}

// status words to pinned host memory by plain stores from an SM: a copy-engine
// D2H of 32 bytes would queue behind the bulk copies of a pipelined round trip
__global__ void status_to_host_kernel(const unsigned long long* src, unsigned long long* dst, int n) {
    const int i = threadIdx.x;
    if (i < n) dst[i] = src[i];
    __threadfence_system();
}
}  // namespace

namespace {
// ---------------------------------------------------------------------------
// Index-less decode: the fall-back behind the speculative segment decode
// (full discovery, second-chance segment decode, two-pass decode: nine
// kernels) is needed only when the speculation failed, which only the device
// knows.  Launched unconditionally, the nine kernels return at once but still
// cost a launch each (~27 us for cfg2's 0.19 ms decode).  Instead they are
// captured once into the body of a CUDA-graph IF node whose condition a
// one-thread kernel sets from the gate word; the instantiated graph is kept
// for repeated decodes with the same buffers (built at the second decode of a
// set of buffers: a build costs ~0.4 ms of host time).  Any failure of the
// graph path falls back to the plain launches.
// ---------------------------------------------------------------------------
__global__ void il_gate_setter_kernel(const IlGate* gate, cudaGraphConditionalHandle h) {
    cudaGraphSetConditional(h, il_seg_ok(gate) ? 0u : 1u);
}

struct IlGraphKey {
    const void* blob; long long nbytes, n; int dt, bs, dev; const void* y; const void* status; const void* ws;
    bool operator==(const IlGraphKey& o) const {
        return blob == o.blob && nbytes == o.nbytes && n == o.n && dt == o.dt && bs == o.bs && dev == o.dev &&
               y == o.y && status == o.status && ws == o.ws;
    }
};
struct IlGraphEntry { IlGraphKey key; cudaGraphExec_t exec; unsigned long long stamp; };
constexpr int kIlGraphSlots = 16;
std::mutex g_il_mu;
IlGraphEntry g_il_cache[kIlGraphSlots];
int g_il_count = 0;
unsigned long long g_il_stamp = 0;
cudaStream_t g_il_capture_stream[64] = {};
IlGraphKey g_il_seen[kIlGraphSlots];
bool g_il_seen_valid[kIlGraphSlots] = {};
int g_il_seen_next = 0;

// enqueue(stream) must enqueue the fall-back on the given stream
template <typename F>
int launch_gated_fallback(const IlGraphKey& key, const IlGate* gate, F&& enqueue, cudaStream_t s) {
    std::lock_guard<std::mutex> lock(g_il_mu);
    for (int i = 0; i < g_il_count; i++) {
        if (g_il_cache[i].key == key) {
            g_il_cache[i].stamp = ++g_il_stamp;
            return cudaGraphLaunch(g_il_cache[i].exec, s) == cudaSuccess ? APAX_OK : APAX_ERR_CUDA;
        }
    }
    if (key.dev < 0 || key.dev >= 64) return APAX_ERR_ARG;
    // building a graph costs ~0.4 ms of host time: only for buffers seen before
    // (a one-off decode takes the plain launches)
    {
        bool seen = false;
        for (int i = 0; i < kIlGraphSlots; i++) seen = seen || (g_il_seen_valid[i] && g_il_seen[i] == key);
        if (!seen) {
            g_il_seen[g_il_seen_next] = key;
            g_il_seen_valid[g_il_seen_next] = true;
            g_il_seen_next = (g_il_seen_next + 1) % kIlGraphSlots;
            return APAX_ERR_ARG;
        }
    }
    cudaStream_t& cap = g_il_capture_stream[key.dev];
    if (!cap && cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess) { cap = nullptr; return APAX_ERR_CUDA; }
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ex = nullptr;
    bool ok = cudaGraphCreate(&g, 0) == cudaSuccess;
    cudaGraphConditionalHandle h;
    ok = ok && cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault) == cudaSuccess;
    cudaGraphNode_t n_set = nullptr, n_if = nullptr;
    if (ok) {
        void* kargs[] = {(void*)&gate, (void*)&h};
        cudaKernelNodeParams kp;
        memset(&kp, 0, sizeof(kp));
        kp.func = (void*)il_gate_setter_kernel;
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(1);
        kp.kernelParams = kargs;
        ok = cudaGraphAddKernelNode(&n_set, g, nullptr, 0, &kp) == cudaSuccess;
    }
    cudaGraph_t body = nullptr;
    if (ok) {
        cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeIf;
        cp.conditional.size = 1;
        ok = cudaGraphAddNode(&n_if, g, &n_set, 1, &cp) == cudaSuccess;
        if (ok) body = cp.conditional.phGraph_out[0];
    }
    if (ok) {
        ok = cudaStreamBeginCaptureToGraph(cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) == cudaSuccess;
        if (ok) {
            const int st = enqueue(cap);
            cudaGraph_t got = nullptr;
            ok = cudaStreamEndCapture(cap, &got) == cudaSuccess && st == APAX_OK;
        }
    }
    ok = ok && cudaGraphInstantiate(&ex, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    if (!ok) {
        if (ex) cudaGraphExecDestroy(ex);
        cudaGetLastError();
        return APAX_ERR_CUDA;
    }
    int slot = g_il_count;
    if (g_il_count < kIlGraphSlots) g_il_count++;
    else {
        slot = 0;
        for (int i = 1; i < kIlGraphSlots; i++) if (g_il_cache[i].stamp < g_il_cache[slot].stamp) slot = i;
        cudaGraphExecDestroy(g_il_cache[slot].exec);
    }
    g_il_cache[slot].key = key;
    g_il_cache[slot].exec = ex;
    g_il_cache[slot].stamp = ++g_il_stamp;
    return cudaGraphLaunch(ex, s) == cudaSuccess ? APAX_OK : APAX_ERR_CUDA;
}
}  // namespace

extern "C" {

const char* apax_version(void) { return "apax-b200 0.2.0 (sm_100a)"; }

int64_t apax_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char* apax_status_string(int code) {
    switch (code) {
        case APAX_OK: return "ok";
        case APAX_ERR_JEE_TRUNCATED: return "JEE nibble stream exhausted";
        case APAX_ERR_JEE_RESERVED: return "reserved JEE nibble 14";
        case APAX_ERR_JEE_RANGE: return "decoded exponent outside [0, 34]";
        case APAX_ERR_JEE_TOO_MANY: return "JEE token stream yields too many exponents";
        case APAX_ERR_JEE_NO_ABS: return "JEE stream must start with an absolute exponent";
        case APAX_ERR_SELECTOR: return "reserved selector value 3";
        case APAX_ERR_NOT_APAX: return "bad magic";
        case APAX_ERR_VERSION: return "container version";
        case APAX_ERR_NONFINITE: return "non-finite value at index";
        case APAX_ERR_INTERNAL: return "sample outside 34-bit range";
        case APAX_ERR_MANTISSA_TRUNCATED: return "mantissa section truncated";
        case APAX_ERR_BLOCK_HDR_TRUNCATED: return "block header truncated";
        case APAX_ERR_FILE_HDR_TRUNCATED: return "file header truncated";
        case APAX_ERR_DTYPE_WIRE: return "unknown dtype wire code";
        case APAX_ERR_MODE_WIRE: return "unknown mode code";
        case APAX_ERR_CFG_BLOCK_RANGE: return "block_size outside [64, 16384]";
        case APAX_ERR_CFG_BLOCK_MULT: return "block_size not a multiple of 4";
        case APAX_ERR_CFG_LOSSLESS_FLOAT: return "lossless unsupported for floats";
        case APAX_ERR_CFG_FR_TARGET: return "FixedRate target must be > 0 bits/sample";
        case APAX_ERR_EMPTY: return "element_count must be >= 1";
        case APAX_ERR_OVERFLOW: return "cannot convert float infinity to integer";
        case APAX_ERR_RANGE: return "attenuation outside [2^-31, 2^33)";
        case APAX_ERR_INTERNAL_WIDTH: return "sample exceeds its group exponent width";
        case APAX_ERR_NONFINITE_BLOCK: return "non-finite float input";
        case APAX_ERR_MATH_DOMAIN: return "math domain error";
        case APAX_ERR_CAPACITY: return "output buffer too small";
        case APAX_ERR_ALLOC: return "allocation failure";
        case APAX_ERR_ARG: return "invalid argument";
        case APAX_ERR_CUDA: return "CUDA error";
        case APAX_ERR_WORKSPACE: return "workspace too small";
    }
    return "unknown status";
}

int64_t apax_max_encoded_bytes(int64_t n, int dtype, int block_size) {
    if (!valid_dtype(dtype) || block_size < 64 || block_size % 4 || n < 0) return -1;
    int64_t nb = (n + block_size - 1) / block_size;
    return kFileHeader + nb * max_block_bytes(dtype, block_size);
}

int64_t apax_encode_workspace_bytes(int64_t n, int dtype, int mode, int block_size,
                                    int64_t segment_blocks) {
    EncPlan p;
    if (plan_encode(n, dtype, mode, block_size, segment_blocks, &p)) return -1;
    return p.ws_total;
}

int apax_encode(const void* x, int64_t n, int dtype, int mode, double target, int block_size,
                int64_t segment_blocks, int policy, uint8_t* out, int64_t out_cap,
                int64_t* block_offsets, uint64_t* status, double* trace, void* ws,
                int64_t ws_bytes, void* stream) {
    EncPlan p;
    int st = plan_encode(n, dtype, mode, block_size, segment_blocks, &p);
    if (st) return st;
    // the policy belongs to segments: a whole stream is the reference's encode_stream
    if (segment_blocks <= 0) policy = APAX_POLICY_COLD;
    if (mode == APAX_LOSSLESS && dtype >= APAX_F32) return APAX_ERR_CFG_LOSSLESS_FLOAT;
    if (mode == APAX_FIXED_RATE && !(target > 0)) return APAX_ERR_CFG_FR_TARGET;
    if (!x || !out || !status || (p.ws_total > 0 && !ws)) return APAX_ERR_ARG;
    if (out_cap < apax_max_encoded_bytes(n, dtype, block_size)) return APAX_ERR_CAPACITY;
    if (ws_bytes < p.ws_total) return APAX_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* w = (uint8_t*)ws;
    if (cudaMemsetAsync(status, 0xFF, 4 * sizeof(uint64_t), s) != cudaSuccess) return APAX_ERR_CUDA;
    if (cudaMemsetAsync(w, 0, (size_t)p.ws_slots, s) != cudaSuccess) return APAX_ERR_CUDA;
    EncParams P;
    memset(&P, 0, sizeof(P));
    P.x = x;
    P.n = n;
    P.mode = mode;
    P.bs = block_size;
    P.target = target;
    P.n_blocks = p.n_blocks;
    P.unit_blocks = p.unit_blocks;
    P.n_units = p.n_units;
    P.halo = p.halo;
    P.policy = policy;
    P.out = out;
    P.out_cap = out_cap;
    P.block_offsets = (long long*)block_offsets;
    P.status = (unsigned long long*)status;
    P.lookback = (unsigned long long*)(w + p.ws_lookback);
    P.ticket = (unsigned int*)(w + p.ws_ticket);
    P.slots = w + p.ws_slots;
    P.slot_bytes = p.slot_bytes;
    P.stage_bytes = p.stage_bytes;
    P.x_in_smem = p.x_in_smem;
    // glibc-evaluated constants (same libm as the reference's CPython)
    P.att_lo = 20.0 * log10(ldexp(1.0, -31));
    P.pow10_t20 = pow(10.0, target / 20.0);
    P.sqrt12 = sqrt(12.0);
    P.trace = trace;
    if (p.split && (((uintptr_t)x) & 15) == 0) {
        // the chain writes each block's quantizer record; the packer codes
        // every block on its own at its final offset (apax_encode_v4.cu)
        uint8_t* v4 = w + p.ws_v4;
        BlockMeta* meta = (BlockMeta*)v4;
        unsigned long long* costs = (unsigned long long*)(v4 + p.n_blocks * 16);
        unsigned long long* lb = costs + p.n_blocks;
        unsigned long long* ticket = lb + p.n_blocks;
        if (cudaMemsetAsync(costs, 0, (size_t)p.n_blocks * 16 + 8, s) != cudaSuccess) return APAX_ERR_CUDA;
        if (mode != APAX_LOSSLESS) {
            P.meta = meta;
            // whole stream: the latency-optimised one-CTA chain (apax_encode_ws.cu);
            // segments: the v3 kernel as a chain, one CTA per segment
            // (fixed quality: the v3 chain measured faster, tools/time_encode.py)
            const int wse = env_int("APAX_WS_CHAIN", -1);
            const bool wsc = segment_blocks <= 0 && encode_ws_supported(dtype, block_size) &&
                             (wse == 1 || (wse < 0 && mode == APAX_FIXED_RATE));
            int r = wsc ? launch_encode_ws_chain(dtype, P, s) : launch_encode_v3_chain(dtype, P, p.smem, s);
            if (r) return r;
        }
        EncParams Q = P;
        Q.unit_blocks = segment_blocks > 0 ? p.unit_blocks : p.n_blocks;   // restart every unit_blocks
        Q.ticket = (unsigned int*)ticket;
        return launch_encode_v4(dtype, Q, mode != APAX_LOSSLESS ? meta : nullptr, costs, lb, s);
    }
    if (p.v3) return launch_encode_v3(dtype, P, p.grid, p.smem, s);
    return launch_encode(dtype, P, p.grid, p.smem, s);
}

static int kdt_of_cast(int in_kind, int dtype) {
    if (!valid_dtype(dtype)) return -1;
    if (in_kind == 0) return dtype;
    if (in_kind == APAX_IN_INT64 && dtype <= APAX_I32) return kKdtI64;
    if (in_kind == APAX_IN_FLOAT64 && dtype == APAX_F32) return kKdtF64F32;
    if (in_kind == APAX_IN_FLOAT64 && dtype == APAX_F64) return APAX_F64;
    return -1;
}

int64_t apax_max_encoded_bytes_cast(int64_t n, int in_kind, int dtype, int block_size) {
    const int kdt = kdt_of_cast(in_kind, dtype);
    if (kdt < 0 || block_size < 64 || block_size % 4 || n < 0) return -1;
    int64_t nb = (n + block_size - 1) / block_size;
    return kFileHeader + nb * max_block_bytes(kdt, block_size);
}

int64_t apax_encode_cast_workspace_bytes(int64_t n, int in_kind, int dtype, int mode, int block_size,
                                         int64_t segment_blocks) {
    const int kdt = kdt_of_cast(in_kind, dtype);
    if (kdt < 0) return -1;
    EncPlan p;
    if (plan_encode(n, kdt, mode, block_size, segment_blocks, &p)) return -1;
    return p.ws_total;
}

int apax_encode_cast(const void* x, int in_kind, int64_t n, int dtype, int mode, double target, int block_size,
                     int64_t segment_blocks, int policy, uint8_t* out, int64_t out_cap, int64_t* block_offsets,
                     uint64_t* status, void* ws, int64_t ws_bytes, void* stream) {
    // encode_stream's input conversions (codec.py:266-272): int64 samples
    // into an integer container (values outside its range are coded as they
    // are and clipped by the decoder), float64 samples into an f32 container
    // (quantized from the f64 values; the FQ loop sees the f32 dequantized y)
    const int kdt = kdt_of_cast(in_kind, dtype);
    if (kdt < 0) return APAX_ERR_ARG;
    if (kdt == dtype)
        return apax_encode(x, n, dtype, mode, target, block_size, segment_blocks, policy, out, out_cap,
                           block_offsets, status, nullptr, ws, ws_bytes, stream);
    EncPlan p;
    int st = plan_encode(n, kdt, mode, block_size, segment_blocks, &p);
    if (st) return st;
    if (segment_blocks <= 0) policy = APAX_POLICY_COLD;
    if (mode == APAX_LOSSLESS && dtype >= APAX_F32) return APAX_ERR_CFG_LOSSLESS_FLOAT;
    if (mode == APAX_FIXED_RATE && !(target > 0)) return APAX_ERR_CFG_FR_TARGET;
    if (!x || !out || !status || (p.ws_total > 0 && !ws)) return APAX_ERR_ARG;
    if (out_cap < apax_max_encoded_bytes_cast(n, in_kind, dtype, block_size)) return APAX_ERR_CAPACITY;
    if (ws_bytes < p.ws_total) return APAX_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* w = (uint8_t*)ws;
    if (cudaMemsetAsync(status, 0xFF, 4 * sizeof(uint64_t), s) != cudaSuccess) return APAX_ERR_CUDA;
    if (cudaMemsetAsync(w, 0, (size_t)p.ws_slots, s) != cudaSuccess) return APAX_ERR_CUDA;
    EncParams P;
    memset(&P, 0, sizeof(P));
    P.x = x;
    P.n = n;
    P.mode = mode;
    P.bs = block_size;
    P.target = target;
    P.n_blocks = p.n_blocks;
    P.unit_blocks = p.unit_blocks;
    P.n_units = p.n_units;
    P.halo = p.halo;
    P.policy = policy;
    P.out = out;
    P.out_cap = out_cap;
    P.block_offsets = (long long*)block_offsets;
    P.status = (unsigned long long*)status;
    P.lookback = (unsigned long long*)(w + p.ws_lookback);
    P.ticket = (unsigned int*)(w + p.ws_ticket);
    P.slots = w + p.ws_slots;
    P.slot_bytes = p.slot_bytes;
    P.stage_bytes = p.stage_bytes;
    P.x_in_smem = p.x_in_smem;
    P.att_lo = 20.0 * log10(ldexp(1.0, -31));
    P.pow10_t20 = pow(10.0, target / 20.0);
    P.sqrt12 = sqrt(12.0);
    P.wire = dtype;
    P.clip_lo = dtype == APAX_I8 ? -128LL : (dtype == APAX_I16 ? -32768LL : -2147483648LL);
    P.clip_hi = dtype == APAX_I8 ? 127LL : (dtype == APAX_I16 ? 32767LL : 2147483647LL);
    return launch_encode(kdt, P, p.grid, p.smem, s);
}

int apax_encode_block(const void* x, int64_t n, int dtype, int mode, double target, int block_size,
                      apax_block_state* state, uint8_t* out, int64_t out_cap, uint64_t* status, void* ws,
                      int64_t ws_bytes, void* stream) {
    // the reference's encode_block (codec.py:192-255): one block under the
    // caller's CodecState, on the generic kernel (x widened: f64 / i64)
    if (!state || n < 1 || n > block_size) return APAX_ERR_ARG;
    const int in_kind = dtype >= APAX_F32 ? APAX_IN_FLOAT64 : APAX_IN_INT64;
    const int kdt = dtype == APAX_F64 ? APAX_F64 : kdt_of_cast(in_kind, dtype);
    if (kdt < 0) return APAX_ERR_ARG;
    EncPlan p;
    int st = plan_encode(n, kdt, mode, block_size, 0, &p);
    if (st) return st;
    if (mode == APAX_LOSSLESS && dtype >= APAX_F32) return APAX_ERR_CFG_LOSSLESS_FLOAT;
    if (mode == APAX_FIXED_RATE && !(target > 0)) return APAX_ERR_CFG_FR_TARGET;
    if (!x || !out || !status || (p.ws_total > 0 && !ws)) return APAX_ERR_ARG;
    if (out_cap < kFileHeader + max_block_bytes(kdt, block_size)) return APAX_ERR_CAPACITY;
    if (ws_bytes < p.ws_total) return APAX_ERR_WORKSPACE;
    // the generic kernel: force it (v3 has no state input)
    p.v3 = 0;
    {
        long long want = 48 * 1024;
        long long mbb = max_block_bytes(kdt, block_size);
        long long stb = want > mbb + 64 ? want : mbb + 64;
        p.stage_bytes = (int)((stb + 15) & ~15LL);
        p.x_in_smem = 1;
        p.smem = encode_smem_bytes(kdt, block_size, p.stage_bytes, 1);
        p.grid = 1;
    }
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* w = (uint8_t*)ws;
    if (cudaMemsetAsync(status, 0xFF, 4 * sizeof(uint64_t), s) != cudaSuccess) return APAX_ERR_CUDA;
    if (cudaMemsetAsync(w, 0, (size_t)p.ws_slots, s) != cudaSuccess) return APAX_ERR_CUDA;
    EncParams P;
    memset(&P, 0, sizeof(P));
    P.x = x;
    P.n = n;
    P.mode = mode;
    P.bs = block_size;
    P.target = target;
    P.n_blocks = 1;
    P.unit_blocks = 1;
    P.n_units = 1;
    P.out = out;
    P.out_cap = out_cap;
    P.status = (unsigned long long*)status;
    P.lookback = (unsigned long long*)(w + p.ws_lookback);
    P.ticket = (unsigned int*)(w + p.ws_ticket);
    P.slots = w + p.ws_slots;
    P.slot_bytes = p.slot_bytes;
    P.stage_bytes = p.stage_bytes;
    P.x_in_smem = p.x_in_smem;
    P.att_lo = 20.0 * log10(ldexp(1.0, -31));
    P.pow10_t20 = pow(10.0, target / 20.0);
    P.sqrt12 = sqrt(12.0);
    P.wire = dtype;
    P.clip_lo = dtype == APAX_I8 ? -128LL : (dtype == APAX_I16 ? -32768LL : -2147483648LL);
    P.clip_hi = dtype == APAX_I8 ? 127LL : (dtype == APAX_I16 ? 32767LL : 2147483647LL);
    P.state = state;
    return launch_encode(kdt, P, 1, p.smem, s);
}

int64_t apax_sweep_point_workspace_bytes(int64_t n, int dtype) {
    if (n < 1 || !encode_v4_supported(dtype, 4096)) return -1;
    const int64_t nb = (n + 4095) / 4096;
    return nb * (16 + 8 + 8 + 24) + 512;
}

int apax_sweep_point(const void* x, int64_t n, int dtype, double target, double* stats, uint64_t* status, void* ws,
                     int64_t ws_bytes, void* stream) {
    // rate_correlation_sweep's point (profiler.py:176-199) without the
    // container: the chain with per-block (x, y) sums, then the packer
    // counting bytes only (whole-stream fixed quality, bs 4096)
    const int64_t need = apax_sweep_point_workspace_bytes(n, dtype);
    if (need < 0 || !x || !stats || !status || !ws || ws_bytes < need || (((uintptr_t)x) & 15)) return APAX_ERR_ARG;
    EncPlan p;
    int st = plan_encode(n, dtype, APAX_FIXED_QUALITY, 4096, 0, &p);
    if (st) return st;
    if (!p.v3) return APAX_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nb = p.n_blocks;
    uint8_t* w = (uint8_t*)ws;
    BlockMeta* meta = (BlockMeta*)w;
    unsigned long long* costs = (unsigned long long*)(w + nb * 16);
    unsigned long long* lb = costs + nb;
    unsigned long long* ticket = lb + nb;
    if (cudaMemsetAsync(status, 0xFF, 4 * sizeof(uint64_t), s) != cudaSuccess) return APAX_ERR_CUDA;
    if (cudaMemsetAsync(costs, 0, (size_t)nb * 16 + 8, s) != cudaSuccess) return APAX_ERR_CUDA;
    EncParams P;
    memset(&P, 0, sizeof(P));
    P.x = x;
    P.n = n;
    P.mode = APAX_FIXED_QUALITY;
    P.bs = 4096;
    P.target = target;
    P.n_blocks = nb;
    P.unit_blocks = nb;
    P.n_units = 1;
    P.status = (unsigned long long*)status;
    P.stage_bytes = p.stage_bytes;
    P.x_in_smem = 1;
    P.att_lo = 20.0 * log10(ldexp(1.0, -31));
    P.pow10_t20 = pow(10.0, target / 20.0);
    P.sqrt12 = sqrt(12.0);
    P.meta = meta;
    P.stats = stats;
    st = launch_encode_v3_chain(dtype, P, p.smem, s);
    if (st) return st;
    EncParams Q = P;
    Q.stats = nullptr;
    Q.count_only = 1;
    Q.ticket = (unsigned int*)ticket;
    return launch_encode_v4(dtype, Q, meta, costs, lb, s);
}

int apax_encode_lossless_range(const void* x, int64_t halo, int64_t n, int dtype, int block_size,
                               int64_t first_block, uint8_t* out, int64_t out_cap, int64_t* block_offsets,
                               uint64_t* status, void* ws, int64_t ws_bytes, void* stream) {
    // blocks first_block .. of a whole-stream LOSSLESS container, as their own
    // container (its body concatenates with the neighbouring ranges' bodies
    // into the one-GPU container): x[0] is sample first_block * bs, and the
    // (bs + 2)-sample halo x[-bs-2 .. 0) rebuilds the first block's state
    // (App. C E2)
    if (first_block < 0) return APAX_ERR_ARG;
    const long long need = first_block == 0 ? 0 : (first_block == 1 ? block_size : block_size + 2);
    if (halo < need) return APAX_ERR_ARG;
    EncPlan p;
    int st = plan_encode(n, dtype, APAX_LOSSLESS, block_size, 0, &p);
    if (st) return st;
    if (dtype >= APAX_F32) return APAX_ERR_CFG_LOSSLESS_FLOAT;
    if (!p.v3) return APAX_ERR_ARG;        // power-of-two block sizes 128..4096
    if (!x || !out || !status || (p.ws_total > 0 && !ws)) return APAX_ERR_ARG;
    if (out_cap < apax_max_encoded_bytes(n, dtype, block_size)) return APAX_ERR_CAPACITY;
    if (ws_bytes < p.ws_total) return APAX_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* w = (uint8_t*)ws;
    if (cudaMemsetAsync(status, 0xFF, 4 * sizeof(uint64_t), s) != cudaSuccess) return APAX_ERR_CUDA;
    if (cudaMemsetAsync(w, 0, (size_t)p.ws_slots, s) != cudaSuccess) return APAX_ERR_CUDA;
    EncParams P;
    memset(&P, 0, sizeof(P));
    P.x = x;
    P.n = n;
    P.mode = APAX_LOSSLESS;
    P.bs = block_size;
    P.n_blocks = p.n_blocks;
    P.unit_blocks = p.unit_blocks;
    P.n_units = p.n_units;
    P.halo = 1;
    P.gblock0 = first_block;
    P.out = out;
    P.out_cap = out_cap;
    P.block_offsets = (long long*)block_offsets;
    P.status = (unsigned long long*)status;
    P.lookback = (unsigned long long*)(w + p.ws_lookback);
    P.ticket = (unsigned int*)(w + p.ws_ticket);
    P.slots = w + p.ws_slots;
    P.slot_bytes = p.slot_bytes;
    P.stage_bytes = p.stage_bytes;
    P.x_in_smem = p.x_in_smem;
    P.att_lo = 20.0 * log10(ldexp(1.0, -31));
    P.pow10_t20 = 1.0;
    P.sqrt12 = sqrt(12.0);
    return launch_encode_v3(dtype, P, p.grid, p.smem, s);
}

int64_t apax_decode_workspace_bytes(int64_t n, int dtype, int block_size) {
    DecPlan p;
    if (plan_decode(n, dtype, block_size, &p)) return -1;
    return p.ws_total;
}

int apax_find_blocks(const uint8_t* blob, int64_t nbytes, int64_t n, int dtype, int block_size,
                     int64_t* offsets, uint64_t* status, void* stream) {
    if (!valid_dtype(dtype) || block_size < 64 || block_size > 16384 || block_size % 4 || n < 0)
        return APAX_ERR_ARG;
    if (!blob || !offsets || !status) return APAX_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    long long nb = (n + block_size - 1) / block_size;
    if (cudaMemsetAsync(status, 0xFF, 4 * sizeof(uint64_t), s) != cudaSuccess) return APAX_ERR_CUDA;
    if (cudaMemsetAsync(offsets, 0xFF, (size_t)(nb + 1) * 8, s) != cudaSuccess) return APAX_ERR_CUDA;
    if (nb == 0) return APAX_OK;
    if (nb < 2 || !env_int("APAX_K5", 1))
        return launch_walk(blob, nbytes, n, block_size, dtype, nb, (long long*)offsets,
                           (unsigned long long*)status, s);
    // K5 scratch from the stream-ordered pool (this entry point takes no
    // workspace); the pool keeps its memory across calls instead of
    // returning it at every synchronisation (re-mapping cost ms per call)
    static std::once_flag pool_once;
    std::call_once(pool_once, [] {
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            unsigned long long keep = ~0ULL;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
    });
    void* ws = nullptr;
    if (cudaMallocAsync(&ws, find_blocks_k5_ws_bytes(nb), s) != cudaSuccess) return APAX_ERR_CUDA;
    int st = launch_find_blocks_k5(blob, nbytes, n, block_size, dtype, nb, (long long*)offsets,
                                   (unsigned long long*)status, ws, s);
    if (cudaFreeAsync(ws, s) != cudaSuccess && st == APAX_OK) st = APAX_ERR_CUDA;
    return st;
}

int apax_decode(const uint8_t* blob, int64_t nbytes, int64_t n, int dtype, int block_size,
                const int64_t* block_offsets, void* y, uint64_t* status, void* ws,
                int64_t ws_bytes, void* stream) {
    DecPlan p;
    int st = plan_decode(n, dtype, block_size, &p);
    if (st) return st;
    if (!blob || !status || (n > 0 && !y)) return APAX_ERR_ARG;
    if (ws_bytes < p.ws_total || !ws) return APAX_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* w = (uint8_t*)ws;
    if (cudaMemsetAsync(status, 0xFF, 4 * sizeof(uint64_t), s) != cudaSuccess) return APAX_ERR_CUDA;
    if (p.n_blocks == 0) return APAX_OK;
    if (cudaMemsetAsync(w, 0, (size_t)p.ws_offsets, s) != cudaSuccess) return APAX_ERR_CUDA;
    const long long* offs = (const long long*)block_offsets;
    IlGate* gate = nullptr;
    // index-less: the discovery's candidate parse fills the two-pass decode's
    // per-block records (DecParams::jee_cache, jee_k5)
    uint8_t* k5_cache = (decode_v3_supported(dtype, block_size) && env_int("APAX_DEC_VER", 0) != 2 &&
                         env_int("APAX_JEE_CACHE", 1) && env_int("APAX_JEE_K5", 1))
                            ? w + p.ws_jee : nullptr;
    const int* k5_flag = nullptr;
    if (!offs) {
        long long* wo = (long long*)(w + p.ws_offsets);
        if (cudaMemsetAsync(wo, 0xFF, (size_t)(p.n_blocks + 1) * 8, s) != cudaSuccess) return APAX_ERR_CUDA;
        const bool k5 = p.n_blocks >= 2 && env_int("APAX_K5", 1);
        if (k5 && decode_v3_supported(dtype, block_size) && env_int("APAX_DEC_VER", 0) != 2 &&
            env_int("APAX_IL_SPEC", 1)) {
            // index-less, speculative: the signature scan's candidates as the
            // offsets (checked block by block by the segment decode below);
            // the full discovery runs only when that path is not taken
            // (the scan also finds the first restarting block > 0, the segment
            // length, and initialises the second gate)
            gate = (IlGate*)(w + p.ws_ticket + 64);
            st = launch_k5_speculate(blob, nbytes, dtype, p.n_blocks, wo, w + p.ws_k5, gate,
                                     (IlGate*)(w + p.ws_ticket + 96), s);
            if (st) return st;
        } else if (k5) {
            st = launch_find_blocks_k5(blob, nbytes, n, block_size, dtype, p.n_blocks, wo,
                                       (unsigned long long*)status, w + p.ws_k5, s, nullptr, k5_cache);
            k5_flag = k5_cache ? k5_flags(w + p.ws_k5, p.n_blocks) : nullptr;
        } else {
            st = launch_walk(blob, nbytes, n, block_size, dtype, p.n_blocks, wo, (unsigned long long*)status, s);
        }
        if (st) return st;
        offs = wo;
    }
    DecParams P;
    memset(&P, 0, sizeof(P));
    P.blob = blob;
    P.nbytes = nbytes;
    P.offsets = offs;
    P.y = y;
    P.n = n;
    P.bs = block_size;
    P.n_blocks = p.n_blocks;
    P.status = (unsigned long long*)status;
    P.carry = (unsigned long long*)(w + p.ws_carry);
    P.ticket = (unsigned int*)(w + p.ws_ticket);
    P.payload_cap = p.payload_cap;
    if (decode_v3_supported(dtype, block_size) && env_int("APAX_DEC_VER", 0) != 2) {
        if (env_int("APAX_JEE_CACHE", 1)) P.jee_cache = w + p.ws_jee;
        const size_t sm3 = decode_v3_smem_bytes(dtype, p.payload_cap);
        const int g3 = decode_v3_resident_ctas(dtype, sm3);
        if (gate) {
            // the speculative segment decode; then (gated on the device) the
            // full discovery for everything it did not take (whole-stream
            // containers, other candidate sets, any inconsistency or error),
            // the segment decode on the verified offsets when they show
            // segments, else the two-pass decode
            IlGate* gate2 = (IlGate*)(w + p.ws_ticket + 96);
            P.il_gate = gate;
            st = launch_decode_v3_seg_dev(dtype, P, g3, sm3, s);
            if (st) return st;
            auto fallback = [&](cudaStream_t fs) -> int {
                int r = launch_find_blocks_k5(blob, nbytes, n, block_size, dtype, p.n_blocks, (long long*)offs,
                                              (unsigned long long*)status, w + p.ws_k5, fs, gate, k5_cache);
                if (r) return r;
                note_launches(1);
                seg_first_kernel<<<seg_first_grid(p.n_blocks), 256, 0, fs>>>(blob, nbytes, offs, p.n_blocks, gate2,
                                                                            gate, (const unsigned long long*)status);
                if (cudaGetLastError() != cudaSuccess) return APAX_ERR_CUDA;
                DecParams Q = P;
                Q.il_gate2 = gate2;
                if (k5_cache && Q.jee_cache) Q.jee_k5 = k5_flags(w + p.ws_k5, p.n_blocks);
                r = launch_decode_v3_seg_dev(dtype, Q, g3, sm3, fs);
                if (r) return r;
                return launch_decode_v3_two_pass(dtype, Q, g3, sm3, Q.carry, fs);
            };
            if (env_int("APAX_IL_GRAPH", 1)) {
                int dev = 0;
                cudaGetDevice(&dev);
                const IlGraphKey key{blob, nbytes, n, dtype, block_size, dev, y, status, ws};
                if (launch_gated_fallback(key, gate, fallback, s) == APAX_OK) return APAX_OK;
            }
            return fallback(s);
        }
        // any container through the segment-serial decoder: one-wave pseudo-
        // segments, pass 1 for their history maps, pass 2 with the composed
        // entries (the carry region holds maps + entries)
        if (k5_flag && P.jee_cache) P.jee_k5 = k5_flag;
        return launch_decode_v3_two_pass(dtype, P, g3, sm3, P.carry, s);
    }
    if (p.v2) return launch_decode_v2(dtype, P, p.grid, p.smem, s);
    return launch_decode(dtype, P, p.grid, p.smem, s);
}

int apax_decode_range(const uint8_t* blob, int64_t nbytes, int64_t n, int dtype, int block_size,
                      const int64_t* block_offsets, int64_t b0, int64_t b1, uint64_t entry_p1,
                      uint64_t entry_p2, void* y, uint64_t* map_out, uint64_t* status, void* ws,
                      int64_t ws_bytes, void* stream) {
    // blocks [b0, b1) of a container of n samples, as a container of their own
    // whose history enters at (entry_p1, entry_p2): the global side-band index
    // is read from entry b0 on, y receives samples b0*bs .. min(n, b1*bs)
    if (!block_offsets || b0 < 0 || b1 <= b0 || block_size <= 0) return APAX_ERR_ARG;
    const long long nb_all = (n + block_size - 1) / block_size;
    if (b1 > nb_all) return APAX_ERR_ARG;
    const long long s0 = b0 * (long long)block_size;
    const long long s1 = (b1 * (long long)block_size < n) ? b1 * (long long)block_size : n;
    const long long nr = s1 - s0;
    DecPlan p;
    int st = plan_decode(nr, dtype, block_size, &p);
    if (st) return st;
    if (!blob || !status || !y) return APAX_ERR_ARG;
    if (ws_bytes < p.ws_total || !ws) return APAX_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* w = (uint8_t*)ws;
    if (cudaMemsetAsync(status, 0xFF, 4 * sizeof(uint64_t), s) != cudaSuccess) return APAX_ERR_CUDA;
    if (cudaMemsetAsync(w, 0, (size_t)p.ws_offsets, s) != cudaSuccess) return APAX_ERR_CUDA;
    DecParams P;
    memset(&P, 0, sizeof(P));
    P.blob = blob;
    P.nbytes = nbytes;
    P.offsets = (const long long*)block_offsets + b0;
    P.y = y;
    P.n = nr;
    P.bs = block_size;
    P.n_blocks = p.n_blocks;
    P.status = (unsigned long long*)status;
    P.carry = (unsigned long long*)(w + p.ws_carry);
    P.ticket = (unsigned int*)(w + p.ws_ticket);
    P.payload_cap = p.payload_cap;
    P.entry_p1 = entry_p1;
    P.entry_p2 = entry_p2;
    st = p.v2 ? launch_decode_v2(dtype, P, p.grid, p.smem, s) : launch_decode(dtype, P, p.grid, p.smem, s);
    if (st) return st;
    if (map_out) return launch_compose_maps(P.carry, p.n_blocks, (unsigned long long*)map_out, s);
    return APAX_OK;
}

int64_t apax_encode_wave_segment_blocks(int64_t n, int dtype, int mode, int block_size) {
    // segment length that gives every resident encoder CTA one segment
    // (a one-wave schedule); the container then depends on this value only
    EncPlan p;
    if (plan_encode(n, dtype, mode, block_size, 1, &p)) return -1;
    int resident = p.grid;
    if (p.v3) {
        resident = encode_v3_resident_ctas_wave(dtype, p.smem);
        if (resident < 1) resident = encode_v3_resident_ctas(dtype, p.smem);
        EncParams P;
        memset(&P, 0, sizeof(P));
        if (encode_v5_supported(dtype, block_size, mode, P)) resident = encode_v5_resident_ctas(dtype);
    }
    if (resident < 1) resident = 1;
    return (p.n_blocks + resident - 1) / resident;
}

const char* apax_encode_kernel_name(int dtype, int mode, int block_size, int64_t segment_blocks) {
    // the kernel that codes the full blocks of such a container (mirrors the
    // dispatch of apax_encode / launch_encode_v3)
    EncPlan p;
    if (plan_encode(1 << 20, dtype, mode, block_size, segment_blocks, &p)) return "";
    if (p.split) return mode == APAX_LOSSLESS ? "pack_kernel" : "chain + pack_kernel";
    if (p.v3) {
        EncParams P;
        memset(&P, 0, sizeof(P));
        P.halo = p.halo;
        // (one-wave launches; longer ones take the persistent v3 kernel)
        return (encode_v5_supported(dtype, block_size, mode, P) && p.unit_blocks >= 3) ? "encode_v5_kernel"
                                                                                      : "encode_v3_kernel";
    }
    return "encode_kernel";
}

int64_t apax_decode_segments_workspace_bytes(int64_t n, int dtype, int block_size) {
    return apax_decode_workspace_bytes(n, dtype, block_size);
}

int apax_decode_segments(const uint8_t* blob, int64_t nbytes, int64_t n, int dtype, int block_size,
                         const int64_t* block_offsets, int64_t segment_blocks, void* y, uint64_t* status,
                         void* ws, int64_t ws_bytes, void* stream) {
    // segment-serial decoder (apax_decode_v3.cu): needs the side-band index
    // and the container's segment length; anything else takes apax_decode
    if (segment_blocks <= 0 || !block_offsets || !decode_v3_supported(dtype, block_size) ||
        env_int("APAX_DEC_VER", 0) == 2)
        return apax_decode(blob, nbytes, n, dtype, block_size, block_offsets, y, status, ws, ws_bytes, stream);
    DecPlan p;
    int st = plan_decode(n, dtype, block_size, &p);
    if (st) return st;
    if (!blob || !status || (n > 0 && !y)) return APAX_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(status, 0xFF, 4 * sizeof(uint64_t), s) != cudaSuccess) return APAX_ERR_CUDA;
    if (p.n_blocks == 0) return APAX_OK;
    DecParams P;
    memset(&P, 0, sizeof(P));
    P.blob = blob;
    P.nbytes = nbytes;
    P.offsets = (const long long*)block_offsets;
    P.y = y;
    P.n = n;
    P.bs = block_size;
    P.n_blocks = p.n_blocks;
    P.status = (unsigned long long*)status;
    P.payload_cap = p.payload_cap;
    P.segment_blocks = segment_blocks;
    const size_t smem = decode_v3_smem_bytes(dtype, p.payload_cap);
    const int grid = decode_v3_resident_ctas(dtype, smem);
    return launch_decode_v3(dtype, P, grid, smem, s);
}

// ---------------------------------------------------------------------------
// profiler statistics (reference profiler.py): per-CTA partials, summed by
// the caller in CTA order
// ---------------------------------------------------------------------------
int apax_profile_grid(void) {
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || nsm <= 0) nsm = 148;
    return 2 * nsm;
}

int apax_profile_sums(const void* x, const void* y, int64_t n, int dtype, int pass, double mean_x, double mean_y,
                      double mean_d, double* partials, uint64_t* counts, void* stream) {
    if (!valid_dtype(dtype) || n < 0 || !x || !y || !partials || !counts || pass < 0 || pass > 1)
        return APAX_ERR_ARG;
    return profile_sums(x, y, n, dtype, pass, mean_x, mean_y, mean_d, partials,
                        (unsigned long long*)counts, apax_profile_grid(), (cudaStream_t)stream);
}

int apax_profile_welch(const void* x, const void* y, int64_t n, int dtype, int which, int seg,
                       const double* tables, double* partials, void* stream) {
    if (!valid_dtype(dtype) || !x || !tables || !partials || which < 0 || which > 2 || (which && !y))
        return APAX_ERR_ARG;
    if (seg < 2 || seg > 4096 || (seg & (seg - 1)) || n < seg) return APAX_ERR_ARG;
    int lg = 0;
    while ((1 << lg) < seg) lg++;
    const long long nframes = (n - seg) / (seg / 2) + 1;
    return profile_welch(x, y ? y : x, n, dtype, which, seg, lg, nframes, tables, partials, apax_profile_grid(),
                         (cudaStream_t)stream);
}

int apax_profile_select(const void* x, const void* y, int64_t n, int dtype, int pass, const uint64_t* prefixes,
                        int n_prefixes, uint32_t* hist, int y_is_output, void* stream) {
    if (!valid_dtype(dtype) || !x || !y || !hist || pass < 0 || pass > 3 || n < 0 || n >= (1LL << 32))
        return APAX_ERR_ARG;
    if (pass > 0 && (!prefixes || n_prefixes < 1 || n_prefixes > 1024)) return APAX_ERR_ARG;
    return profile_select(x, y, n, dtype, pass, (const unsigned long long*)prefixes, n_prefixes, (unsigned*)hist,
                          y_is_output ? 1 : 0, apax_profile_grid(), (cudaStream_t)stream);
}

int apax_parse_file_header(const uint8_t* d, int64_t len, int* dt, int* mode, int* bs,
                           int64_t* count, double* target, int64_t* detail) {
    // reference parse_file_header (codec.py:288-305) + StreamConfig.validate
    *detail = -1;
    if (len < kFileHeader) return APAX_ERR_FILE_HDR_TRUNCATED;
    if (memcmp(d, "APAX", 4) != 0) return APAX_ERR_NOT_APAX;
    if (d[4] != 1) { *detail = d[4]; return APAX_ERR_VERSION; }
    if (d[5] > 4) { *detail = d[5]; return APAX_ERR_DTYPE_WIRE; }
    if (d[6] > 2) { *detail = d[6]; return APAX_ERR_MODE_WIRE; }
    uint32_t b32;
    uint64_t c64;
    memcpy(&b32, d + 8, 4);
    memcpy(&c64, d + 12, 8);
    memcpy(target, d + 20, 8);
    *dt = d[5];
    *mode = d[6];
    *bs = (int)b32;
    *count = (int64_t)c64;
    *detail = (int64_t)b32;
    if (!(64 <= b32 && b32 <= 16384)) return APAX_ERR_CFG_BLOCK_RANGE;
    if (b32 % 4) return APAX_ERR_CFG_BLOCK_MULT;
    if (*mode == APAX_LOSSLESS && *dt >= APAX_F32) return APAX_ERR_CFG_LOSSLESS_FLOAT;
    if (*mode == APAX_FIXED_RATE && !(*target > 0)) return APAX_ERR_CFG_FR_TARGET;
    *detail = -1;
    return APAX_OK;
}

int apax_detect_segments(const uint8_t* blob, int64_t nbytes, const int64_t* block_offsets, int64_t n_blocks,
                         uint64_t* segment_blocks_out, void* stream) {
    if (!blob || !block_offsets || !segment_blocks_out || n_blocks < 1) return APAX_ERR_ARG;
    note_launches(1);
    detect_segments_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(blob, nbytes, (const long long*)block_offsets,
                                                                 n_blocks, (unsigned long long*)segment_blocks_out);
    return cudaGetLastError() == cudaSuccess ? APAX_OK : APAX_ERR_CUDA;
}

int apax_status_to_host(const uint64_t* status, uint64_t* host_dst, int n_words, void* stream) {
    if (!status || !host_dst || n_words < 1 || n_words > 32) return APAX_ERR_ARG;
    void* dptr = nullptr;
    if (cudaHostGetDevicePointer(&dptr, host_dst, 0) != cudaSuccess || !dptr) {
        cudaGetLastError();
        return APAX_ERR_ARG;   // not page-locked host memory
    }
    note_launches(1);
    status_to_host_kernel<<<1, 32, 0, (cudaStream_t)stream>>>((const unsigned long long*)status,
                                                             (unsigned long long*)dptr, n_words);
    return cudaGetLastError() == cudaSuccess ? APAX_OK : APAX_ERR_CUDA;
}

}  // extern "C"
