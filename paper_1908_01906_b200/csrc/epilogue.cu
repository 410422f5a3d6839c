// epilogue.cu -- device post-processing of a rendered frame.
//
// Every viewer frame and CLI image post-processes the framebuffer on the host
// (imgio.py, metrics.py): round-half-up quantisation of the RGB channels
// (imgio.py:36-39, 76-78), the sample-count heatmap normalised by the frame
// maximum through a 256-entry LUT (imgio.py:81-87), and the sweep harness's
// mean SSIM against the reference render (metrics.py:36-80).  Here they run
// on the frame while it is still in HBM, so a viewer frame leaves the GPU as
// 3 + 3 bytes per pixel instead of 32 + 8:
//   quantize_kernel   floor(clip(c, 0, 1) * 255 + 0.5), bit-identical to numpy;
//   heatmap_kernel    max-reduction of the counts (one atomicMax per CTA),
//                     then t = c / peak, floor(t * 255 + 0.5) -> LUT (exact);
//   ssim_kernel       Rec.709 luminance of both u8 images, the 11x11 Gaussian
//                     window (host-built weights, scipy.ndimage.correlate with
//                     mode='constant' and the valid-region crop) and the SSIM
//                     map, reduced to its mean -- floating-point reductions in
//                     a different order than scipy's, so the parity test holds
//                     it to a relative 1e-12.
// Compiled with -fmad=false like the render kernels.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>

#include "tetray_b200.h"
#include "tr_internal.h"

namespace {

constexpr int MAX_WIN = 31;

__device__ __forceinline__ uint8_t quant(double v) {   // imgio.py:36-39
    const double c = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    return (uint8_t)floor(c * 255.0 + 0.5);
}

__global__ void quantize_kernel(const double *__restrict__ rgba, int64_t n, uint8_t *rgb) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double2 a = __ldg(reinterpret_cast<const double2 *>(rgba) + 2 * i);
        const double2 b = __ldg(reinterpret_cast<const double2 *>(rgba) + 2 * i + 1);
        rgb[3 * i] = quant(a.x);
        rgb[3 * i + 1] = quant(a.y);
        rgb[3 * i + 2] = quant(b.x);
    }
}

__global__ void count_max_kernel(const int64_t *__restrict__ counts, int64_t n,
                                 unsigned long long *peak) {
    long long m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, (long long)counts[i]);
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ long long s[32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = max(m, s[w]);
        if (m > 0) atomicMax(peak, (unsigned long long)m);
    }
}

__global__ void heatmap_kernel(const int64_t *__restrict__ counts, int64_t n,
                               const unsigned long long *peak, const uint8_t *__restrict__ lut,
                               uint8_t *rgb) {
    __shared__ uint8_t s_lut[768];
    for (int i = threadIdx.x; i < 768; i += blockDim.x) s_lut[i] = lut[i];
    __syncthreads();
    const double pk = (double)(long long)*peak;   // counts.max() as float64
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double t = pk > 0.0 ? (double)counts[i] / pk : 0.0;   // imgio.py:84-85
        const int64_t idx = (int64_t)floor(t * 255.0 + 0.5);
        rgb[3 * i] = s_lut[3 * idx];
        rgb[3 * i + 1] = s_lut[3 * idx + 1];
        rgb[3 * i + 2] = s_lut[3 * idx + 2];
    }
}

__device__ __forceinline__ double luma(const uint8_t *p, const double *w) {  // metrics.py:40-41
    return ((double)p[0] * w[0] + (double)p[1] * w[1]) + (double)p[2] * w[2];
}

// One thread per valid-region pixel: the five windowed moments (zero
// outside the image, scipy's mode='constant'), then the SSIM term; CTA sums
// go to a double atomic (the mean is divided on the host side of the call).
__global__ void ssim_kernel(const uint8_t *__restrict__ a, const uint8_t *__restrict__ b, int64_t h,
                            int64_t w, int win, const double *__restrict__ weights,
                            const double *__restrict__ rec709, double c1, double c2,
                            double *sum) {
    const int half = win / 2;
    const int64_t vh = h - 2 * half, vw = w - 2 * half, n = vh * vw;
    double local = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t y = i / vw + half, x = i % vw + half;
        double ma = 0.0, mb = 0.0, saa = 0.0, sbb = 0.0, sab = 0.0;
        for (int dy = 0; dy < win; ++dy) {
            const int64_t yy = y + dy - half;
            for (int dx = 0; dx < win; ++dx) {
                const int64_t xx = x + dx - half;
                const double wt = weights[dy * win + dx];
                const double la = luma(a + 3 * (yy * w + xx), rec709);
                const double lb = luma(b + 3 * (yy * w + xx), rec709);
                ma += wt * la;
                mb += wt * lb;
                saa += wt * (la * la);
                sbb += wt * (lb * lb);
                sab += wt * (la * lb);
            }
        }
        const double s_aa = saa - ma * ma, s_bb = sbb - mb * mb, s_ab = sab - ma * mb;
        const double num = (2.0 * ma * mb + c1) * (2.0 * s_ab + c2);
        const double den = (ma * ma + mb * mb + c1) * (s_aa + s_bb + c2);
        local += num / den;
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(sum, local);
}

int cuda_fail(cudaError_t e, const char *where) {
    std::string m = std::string(where) + ": " + cudaGetErrorString(e);
    return tr_fail(TR_ECUDA, m.c_str());
}

unsigned blocks_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace

extern "C" {

int tr_quantize_rgb(const double *rgba, int64_t n_pixels, uint8_t *rgb, void *stream) {
    if (n_pixels < 0 || (n_pixels > 0 && (!rgba || !rgb)))
        return tr_fail(TR_EINVAL, "tr_quantize_rgb: invalid arguments");
    if (n_pixels == 0) return TR_OK;
    quantize_kernel<<<blocks_for(n_pixels), 256, 0, (cudaStream_t)stream>>>(rgba, n_pixels, rgb);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TR_OK : cuda_fail(e, "quantize_kernel");
}

int tr_heatmap_rgb(const int64_t *counts, int64_t n_pixels, const uint8_t *lut, uint8_t *rgb,
                   uint64_t *peak, void *stream) {
    if (n_pixels < 0 || (n_pixels > 0 && (!counts || !lut || !rgb || !peak)))
        return tr_fail(TR_EINVAL, "tr_heatmap_rgb: invalid arguments");
    if (n_pixels == 0) return TR_OK;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(peak, 0, sizeof(uint64_t), st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(peak)");
    count_max_kernel<<<blocks_for(n_pixels), 256, 0, st>>>(counts, n_pixels,
                                                           (unsigned long long *)peak);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "count_max_kernel");
    heatmap_kernel<<<blocks_for(n_pixels), 256, 0, st>>>(counts, n_pixels,
                                                         (const unsigned long long *)peak, lut, rgb);
    e = cudaGetLastError();
    return e == cudaSuccess ? TR_OK : cuda_fail(e, "heatmap_kernel");
}

int tr_ssim_rgb(const uint8_t *a, const uint8_t *b, int64_t height, int64_t width, int32_t window,
                const double *weights, const double *rec709, double c1, double c2, double *sum,
                void *stream) {
    if (!a || !b || !weights || !rec709 || !sum || window < 1 || window > MAX_WIN ||
        (window % 2) == 0 || height < window || width < window)
        return tr_fail(TR_EINVAL, "tr_ssim_rgb: invalid arguments");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(sum, 0, sizeof(double), st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(sum)");
    const int64_t n = (height - window + 1) * (width - window + 1);
    ssim_kernel<<<blocks_for(n), 256, 0, st>>>(a, b, height, width, window, weights, rec709, c1,
                                                c2, sum);
    e = cudaGetLastError();
    return e == cudaSuccess ? TR_OK : cuda_fail(e, "ssim_kernel");
}

}  // extern "C"
