// apax_block_api.cu -- the reference's lower-level block API on the device
// (pkg/src/apax/codec.py:94-146 quantize_block / dequantize_block; the
// stateful encode_block :192-255 runs the generic encoder with a CodecState
// in / out, apax_capi.cu).  Used by the drop-in Python layer
// (paper_1303_4994_b200/block.py) so the reference's block-level KATs and
// demos run against the same kernels' arithmetic.
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

#include "apax_device.cuh"
#include "apax_kernels.cuh"

namespace apax {
namespace blk {

constexpr int NT = 256;

// quantize_block (codec.py:94-132) on one CTA: x widened as the reference
// does (f64 for floats, i64 for integers)
template <bool F>
__global__ void __launch_bounds__(NT) quantize_kernel(const void* xv, long long n, double a, long long* q,
                                                      int* hdr, unsigned long long* status) {
    __shared__ double sp[NT / 32];
    __shared__ int snf[NT / 32];
    __shared__ double s_scale;
    __shared__ int s_zero;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (!F) {
        // integers: code = encode(a), q = x when a_q == 1, else rint(x * a_q)
        const long long* x = (const long long*)xv;
        const int code = encode_scale_code(a);
        const double aq = decode_scale_code(code);
        for (long long i = tid; i < n; i += NT) q[i] = aq == 1.0 ? x[i] : f2i64(rint((double)x[i] * aq));
        if (tid == 0) { hdr[0] = code; hdr[1] = 0; }
        return;
    }
    const double* x = (const double*)xv;
    double pk = 0.0;
    int nf = 0;
    for (long long i = tid; i < n; i += NT) {
        const double v = fabs(x[i]);
        if (!(v <= 1.79769313486231570815e308)) nf = 1;   // NaN or inf
        else pk = v > pk ? v : pk;
    }
    pk = warp_allreduce(pk, MaxOp());
    nf = __any_sync(0xffffffffu, nf);
    if (lane == 0) { sp[warp] = pk; snf[warp] = nf; }
    __syncthreads();
    if (tid == 0) {
        double peak = 0.0;
        int nonfin = 0;
        for (int w = 0; w < NT / 32; w++) { peak = sp[w] > peak ? sp[w] : peak; nonfin |= snf[w]; }
        int code = kScaleCodeOne, fbe = 0, zero = 0, bad = 0;
        double s = 0.0;
        if (nonfin) {
            bad = APAX_ERR_NONFINITE_BLOCK;
            zero = 1;
        } else if (peak == 0.0) {
            zero = 1;
        } else {
            const double s_des = (a * 1073741824.0) / peak;
            if (!isfinite(s_des)) {
                bad = APAX_ERR_OVERFLOW;
                zero = 1;
            } else {
                long long l2 = floor_log2_rn(s_des);
                long long fb = (-31 <= l2 && l2 <= 31) ? 0 : l2 - 31;
                fb = fb < -127 ? -127 : (fb > 127 ? 127 : fb);
                double rem = ldexp(s_des, (int)-fb);
                const double nxt = 8589934591.999999;   // nextafter(2^33, 0)
                const double mm = (nxt < rem) ? nxt : rem;
                rem = (mm > 4.656612873077393e-10) ? mm : 4.656612873077393e-10;
                code = encode_scale_code(rem);
                for (;;) {   // overflow guard: max|q| = rint(peak * S) (rounding is monotone)
                    s = decode_scale_code(code) * ldexp(1.0, (int)fb);
                    const double qm = rint(peak * s);
                    if (qm < 2147483648.0 || fb <= -127) break;
                    fb -= 1;
                }
                fbe = (int)fb;
            }
        }
        if (bad) report_error(status, 0, bad);
        hdr[0] = code;
        hdr[1] = fbe;
        s_scale = s;
        s_zero = zero;
    }
    __syncthreads();
    const double s = s_scale;
    const bool zero = s_zero;
    for (long long i = tid; i < n; i += NT) q[i] = zero ? 0LL : f2i64(rint(x[i] * s));
}

// dequantize_block (codec.py:135-146): floats (q / S) in the dtype; integers
// q when a == 1, else rint(q / a), clipped to the dtype's range
template <int DT>
__global__ void dequantize_kernel(const long long* q, long long n, int code, int fbe, void* yv) {
    using Tr = DT_<DT>;
    using T = typename Tr::T;
    T* y = (T*)yv;
    const double a = decode_scale_code(code);
    const double s = Tr::F ? a * ldexp(1.0, fbe) : a;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        if (Tr::F) {
            y[i] = (T)__ddiv_rn((double)q[i], s);
        } else {
            long long v = (a == 1.0) ? q[i] : f2i64(rint(__ddiv_rn((double)q[i], a)));
            v = v < Tr::LO ? Tr::LO : (v > Tr::HI ? Tr::HI : v);
            y[i] = (T)v;
        }
    }
}

}  // namespace blk
}  // namespace apax

using namespace apax;

extern "C" int apax_quantize_block(const void* x, int64_t n, int dtype, double a, int64_t* q, int32_t* hdr,
                                   uint64_t* status, void* stream) {
    if (dtype < 0 || dtype > 4 || n < 0 || (n > 0 && (!x || !q)) || !hdr || !status) return APAX_ERR_ARG;
    if (dtype < 3 && !(a >= 4.656612873077393e-10 && a < 8589934592.0)) return APAX_ERR_RANGE;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(status, 0xFF, 4 * sizeof(uint64_t), s) != cudaSuccess) return APAX_ERR_CUDA;
    note_launches(1);
    if (dtype >= 3)
        blk::quantize_kernel<true><<<1, blk::NT, 0, s>>>(x, n, a, (long long*)q, (int*)hdr, (unsigned long long*)status);
    else
        blk::quantize_kernel<false><<<1, blk::NT, 0, s>>>(x, n, a, (long long*)q, (int*)hdr, (unsigned long long*)status);
    return cudaGetLastError() == cudaSuccess ? APAX_OK : APAX_ERR_CUDA;
}

extern "C" int apax_dequantize_block(const int64_t* q, int64_t n, int dtype, int code, int fbe, void* y,
                                     void* stream) {
    if (dtype < 0 || dtype > 4 || n < 0 || (n > 0 && (!q || !y)) || code < 0 || code > 0xFFFF) return APAX_ERR_ARG;
    if (n == 0) return APAX_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = (int)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
    const long long* qq = (const long long*)q;
    note_launches(1);
    switch (dtype) {
        case 0: blk::dequantize_kernel<0><<<grid, 256, 0, s>>>(qq, n, code, fbe, y); break;
        case 1: blk::dequantize_kernel<1><<<grid, 256, 0, s>>>(qq, n, code, fbe, y); break;
        case 2: blk::dequantize_kernel<2><<<grid, 256, 0, s>>>(qq, n, code, fbe, y); break;
        case 3: blk::dequantize_kernel<3><<<grid, 256, 0, s>>>(qq, n, code, fbe, y); break;
        default: blk::dequantize_kernel<4><<<grid, 256, 0, s>>>(qq, n, code, fbe, y); break;
    }
    return cudaGetLastError() == cudaSuccess ? APAX_OK : APAX_ERR_CUDA;
}
