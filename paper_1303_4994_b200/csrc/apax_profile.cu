// apax_profile.cu -- profiler statistics on B200 (reference
// pkg/src/apax/profiler.py, statistics half): fused single-pass sums for
// pearson_r / window2_metrics (:40-48, :127-159), the Welch PSD of x, y and
// d = x - y (:61-74, scipy.signal.welch: periodic Hann, 50% overlap, no
// detrend, "spectrum" scaling), and an exact radix multi-select over the
// per-sample ratio |x| / |d| that gives the S2R 2-sigma margin and CDF
// order statistics (:88-124) -- log10 is monotone, so the host applies
// numpy's log10 to the selected ratios only.
//
// Determinism: every reduction writes per-CTA partials in a fixed order; the
// host sums them in CTA order.  Counts use integer atomics (exact).
#include <cstdint>
#include <cuda_runtime.h>

#include "apax_device.cuh"
#include "apax_kernels.cuh"

namespace apax {
namespace prof {

constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int NSUM = 8;   // sums per CTA partial

template <int DT>
__device__ __forceinline__ double ld_as_double(const void* p, long long i) {
    using T = typename DT_<DT>::T;
    return (double)((const T*)p)[i];
}

// pass 0: [sx, sy, sd, sxx, syy, sdd, sxy, 0]; pass 1 (centred): [0,0,0,
// s(x-mx)^2, s(y-my)^2, s(d-md)^2, 0, 0]; counts: [#(x==0 & d!=0), #(d==0)]
template <int DT>
__global__ void __launch_bounds__(NT) sums_kernel(const void* x, const void* y, long long n, int pass, double mx,
                                                  double my, double md, double* partials,
                                                  unsigned long long* counts) {
    __shared__ double red[NSUM][NW];
    double a[NSUM];
#pragma unroll
    for (int k = 0; k < NSUM; k++) a[k] = 0.0;
    unsigned long long z0 = 0, zd = 0;
    for (long long i = (long long)blockIdx.x * NT + threadIdx.x; i < n; i += (long long)gridDim.x * NT) {
        const double xv = ld_as_double<DT>(x, i);
        const double yv = ld_as_double<DT>(y, i);
        const double dv = xv - yv;
        if (pass == 0) {
            a[0] += xv; a[1] += yv; a[2] += dv;
            a[3] += xv * xv; a[4] += yv * yv; a[5] += dv * dv; a[6] += xv * yv;
            z0 += (xv == 0.0 && dv != 0.0) ? 1ULL : 0ULL;
            zd += (dv == 0.0) ? 1ULL : 0ULL;
        } else {
            const double cx = xv - mx, cy = yv - my, cd = dv - md;
            a[3] += cx * cx; a[4] += cy * cy; a[5] += cd * cd;
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NSUM; k++) {
        double v = a[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[k][warp] = v;
    }
    if (pass == 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            z0 += __shfl_xor_sync(0xffffffffu, z0, o);
            zd += __shfl_xor_sync(0xffffffffu, zd, o);
        }
        if (lane == 0) {
            if (z0) atomicAdd(&counts[0], z0);
            if (zd) atomicAdd(&counts[1], zd);
        }
    }
    __syncthreads();
    if (threadIdx.x < NSUM) {
        double v = 0.0;
        for (int w = 0; w < NW; w++) v += red[threadIdx.x][w];
        partials[(long long)blockIdx.x * NSUM + threadIdx.x] = v;
    }
}

// ---------------------------------------------------------------------------
// Welch: one frame per CTA iteration, radix-2 DIT complex FFT of the
// windowed frame in shared memory, |X_k|^2 accumulated per CTA.
// which: 0 = x, 1 = y, 2 = d = x - y.
// ---------------------------------------------------------------------------
template <int DT>
__global__ void __launch_bounds__(NT) welch_kernel(const void* x, const void* y, long long n, int which, int seg,
                                                   int lg, long long nframes, const double* tw,
                                                   double* partials) {
    extern __shared__ __align__(16) unsigned char smem[];
    double2* a = (double2*)smem;                    // seg complex
    double2* w = a + seg;                           // seg/2 twiddles
    double* acc = (double*)(w + seg / 2);           // seg/2 + 1 bins
    const int tid = threadIdx.x;
    const int nb = seg / 2 + 1;
    for (int k = tid; k < seg / 2; k += NT) w[k] = ((const double2*)tw)[k];
    for (int k = tid; k < nb; k += NT) acc[k] = 0.0;
    const double* hann = tw + seg;                  // seg window values after the twiddles
    __syncthreads();
    const long long hop = seg / 2;
    for (long long f = blockIdx.x; f < nframes; f += gridDim.x) {
        const long long base = f * hop;
        for (int k = tid; k < seg; k += NT) {
            const long long i = base + k;
            const double xv = ld_as_double<DT>(x, i);
            double v;
            if (which == 0) v = xv;
            else {
                const double yv = ld_as_double<DT>(y, i);
                v = which == 1 ? yv : xv - yv;
            }
            const int r = (int)(__brev((unsigned)k) >> (32 - lg));
            a[r] = make_double2(hann[k] * v, 0.0);
        }
        __syncthreads();
        for (int s = 1; s <= lg; s++) {
            const int half = 1 << (s - 1);
            const int tstride = seg >> s;           // twiddle index stride
            for (int j = tid; j < seg / 2; j += NT) {
                const int grp = j >> (s - 1), pos = j & (half - 1);
                const int i0 = (grp << s) + pos, i1 = i0 + half;
                const double2 t = w[pos * tstride];
                const double2 b = a[i1];
                const double tr = t.x * b.x - t.y * b.y;
                const double ti = t.x * b.y + t.y * b.x;
                const double2 c = a[i0];
                a[i1] = make_double2(c.x - tr, c.y - ti);
                a[i0] = make_double2(c.x + tr, c.y + ti);
            }
            __syncthreads();
        }
        for (int k = tid; k < nb; k += NT) {
            const double2 c = a[k];
            acc[k] += c.x * c.x + c.y * c.y;
        }
        __syncthreads();
    }
    for (int k = tid; k < nb; k += NT) partials[(long long)blockIdx.x * nb + k] = acc[k];
}

// ---------------------------------------------------------------------------
// radix multi-select over the ratio keys (bit patterns of |x| / |d| as
// non-negative doubles; d == 0 -> +inf, x == 0 != d -> 0): pass p counts
// digit p (4 bits, most significant first) of every key whose higher bits
// equal one of the (sorted, unique) active prefixes.
// ---------------------------------------------------------------------------
template <int DT>
__device__ __forceinline__ unsigned long long ratio_key(const void* x, const void* y, long long i, int ydiff) {
    const double xv = ld_as_double<DT>(x, i);
    const double yv = ld_as_double<DT>(y, i);
    const double ad = fabs(ydiff ? xv - yv : yv), ax = fabs(xv);
    double r;
    if (ad == 0.0) r = INFINITY;
    else if (ax == 0.0) r = 0.0;
    else r = __ddiv_rn(ax, ad);
    return (unsigned long long)__double_as_longlong(r);
}

// digit plan of the 4-pass select: the key's sign bit is 0, so bits 62..0
// split into 15 + 16 + 16 + 16 (most significant first)
__host__ __device__ __forceinline__ int sel_shift(int pass) { return pass == 0 ? 48 : 48 - 16 * pass; }
__host__ __device__ __forceinline__ int sel_width(int pass) { return pass == 0 ? 15 : 16; }

// pass 0: one (empty) prefix, a 2^15-bin histogram per CTA in shared memory
template <int DT>
__global__ void __launch_bounds__(NT) select0_kernel(const void* x, const void* y, long long n,
                                                     unsigned* hist, int ydiff) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned* h = (unsigned*)smem;   // 2^15 bins
    for (int k = threadIdx.x; k < (1 << 15); k += NT) h[k] = 0u;
    __syncthreads();
    for (long long i = (long long)blockIdx.x * NT + threadIdx.x; i < n; i += (long long)gridDim.x * NT)
        atomicAdd(&h[(int)((ratio_key<DT>(x, y, i, ydiff) >> 48) & 0x7fffULL)], 1u);
    __syncthreads();
    for (int k = threadIdx.x; k < (1 << 15); k += NT)
        if (h[k]) atomicAdd(&hist[k], h[k]);
}

// passes 1..3: 16-bit digits of the keys whose higher bits equal one of the
// sorted, unique prefixes, counted straight into hist[prefix][digit] (only
// the keys in the target buckets get that far)
template <int DT>
__global__ void __launch_bounds__(NT) select_kernel(const void* x, const void* y, long long n, int pass,
                                                    const unsigned long long* prefixes, int npre,
                                                    unsigned* hist, int ydiff) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long* pre = (unsigned long long*)smem;   // npre
    for (int k = threadIdx.x; k < npre; k += NT) pre[k] = prefixes[k];
    __syncthreads();
    const int sh = sel_shift(pass);
    for (long long i = (long long)blockIdx.x * NT + threadIdx.x; i < n; i += (long long)gridDim.x * NT) {
        const unsigned long long key = ratio_key<DT>(x, y, i, ydiff);
        const unsigned long long hi = key >> (sh + 16);
        int lo = 0, up = npre;
        while (lo < up) {
            const int mid = (lo + up) >> 1;
            if (pre[mid] < hi) lo = mid + 1;
            else up = mid;
        }
        if (lo < npre && pre[lo] == hi) atomicAdd(&hist[(long long)lo * 65536 + (int)((key >> sh) & 0xffffULL)], 1u);
    }
}

}  // namespace prof

int profile_sums(const void* x, const void* y, long long n, int dt, int pass, double mx, double my,
                 double md, double* partials, unsigned long long* counts, int grid, cudaStream_t st) {
    switch (dt) {
        case 0: note_launches(1); prof::sums_kernel<0><<<grid, prof::NT, 0, st>>>(x, y, n, pass, mx, my, md, partials, counts); break;
        case 1: note_launches(1); prof::sums_kernel<1><<<grid, prof::NT, 0, st>>>(x, y, n, pass, mx, my, md, partials, counts); break;
        case 2: note_launches(1); prof::sums_kernel<2><<<grid, prof::NT, 0, st>>>(x, y, n, pass, mx, my, md, partials, counts); break;
        case 3: note_launches(1); prof::sums_kernel<3><<<grid, prof::NT, 0, st>>>(x, y, n, pass, mx, my, md, partials, counts); break;
        default: note_launches(1); prof::sums_kernel<4><<<grid, prof::NT, 0, st>>>(x, y, n, pass, mx, my, md, partials, counts); break;
    }
    return cudaGetLastError() == cudaSuccess ? APAX_OK : APAX_ERR_CUDA;
}

size_t profile_welch_smem(int seg) {
    return (size_t)seg * 16 + (size_t)(seg / 2) * 16 + (size_t)(seg / 2 + 1) * 8;
}

int profile_welch(const void* x, const void* y, long long n, int dt, int which, int seg, int lg,
                  long long nframes, const double* tw, double* partials, int grid, cudaStream_t st) {
    const size_t smem = profile_welch_smem(seg);
    auto go = [&](auto kfn) -> int {
        if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return APAX_ERR_CUDA;
        note_launches(1);
        kfn<<<grid, prof::NT, smem, st>>>(x, y, n, which, seg, lg, nframes, tw, partials);
        return cudaGetLastError() == cudaSuccess ? APAX_OK : APAX_ERR_CUDA;
    };
    switch (dt) {
        case 0: return go(prof::welch_kernel<0>);
        case 1: return go(prof::welch_kernel<1>);
        case 2: return go(prof::welch_kernel<2>);
        case 3: return go(prof::welch_kernel<3>);
        default: return go(prof::welch_kernel<4>);
    }
}

int profile_select(const void* x, const void* y, long long n, int dt, int pass,
                   const unsigned long long* prefixes, int npre, unsigned* hist, int ydiff, int grid,
                   cudaStream_t st) {
    auto go0 = [&](auto kfn) -> int {
        const size_t smem = (size_t)4 << 15;
        if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return APAX_ERR_CUDA;
        int dev = 0, nsm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        note_launches(1);
        kfn<<<nsm > 0 ? nsm : 148, prof::NT, smem, st>>>(x, y, n, hist, ydiff);
        return cudaGetLastError() == cudaSuccess ? APAX_OK : APAX_ERR_CUDA;
    };
    auto go = [&](auto kfn) -> int {
        const size_t smem = (size_t)npre * 8;
        note_launches(1);
        kfn<<<grid, prof::NT, smem, st>>>(x, y, n, pass, prefixes, npre, hist, ydiff);
        return cudaGetLastError() == cudaSuccess ? APAX_OK : APAX_ERR_CUDA;
    };
    if (pass == 0) {
        switch (dt) {
            case 0: return go0(prof::select0_kernel<0>);
            case 1: return go0(prof::select0_kernel<1>);
            case 2: return go0(prof::select0_kernel<2>);
            case 3: return go0(prof::select0_kernel<3>);
            default: return go0(prof::select0_kernel<4>);
        }
    }
    switch (dt) {
        case 0: return go(prof::select_kernel<0>);
        case 1: return go(prof::select_kernel<1>);
        case 2: return go(prof::select_kernel<2>);
        case 3: return go(prof::select_kernel<3>);
        default: return go(prof::select_kernel<4>);
    }
}

}  // namespace apax
