// meta.cu -- transfer-function partition metadata on the device.
//
// Replaces update_transfer_function's per-partition loop (transfer.py:95-167,
// the paper's "parallelized across the partitions" step): for every partition
// the TF rows overlapping its value range (the interpolated ends plus the
// table rows strictly inside, transfer.py:96-110), their maximum opacity and
// the variance of the opacity-weighted colours (transfer.py:113-124), then the
// min-max normalisation to sigma and the active flags (transfer.py:127-141).
// One thread per partition; the rows are regenerated on the fly instead of
// stored, and every reduction keeps numpy's order -- the axis-0 mean summed
// sequentially, the final mean with numpy's pairwise summation -- so the
// results equal the host restatement (tr_tf_meta) and the reference bit for
// bit (tests/test_tf_meta_device.py).  Compiled with -fmad=false like the
// render kernels.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>

#include "glibc_pow.cuh"
#include "tetray_b200.h"
#include "tr_internal.h"

namespace {

#if TR_HAVE_GLIBC_POW
__constant__ unsigned long long c_lhead[] = TR_POW_LOG_HEAD_INIT;
__constant__ unsigned long long c_ehead[] = TR_POW_EXP_HEAD_INIT;
__device__ const __align__(32) unsigned long long d_ltab[] = TR_POW_LOG_TAB_INIT;
__device__ const __align__(32) unsigned long long d_etab[] = TR_POW_EXP_TAB_INIT;
#endif

// step_size (K:20-22) per partition: max(s1 + (s2 - s1) * |min(sigma, 1) - 1|^p, s1),
// with glibc's pow restated (glibc_pow.cuh) -- bit-identical to the host's
// tr_step_sizes wherever the restated path applies; elsewhere the entry is
// NaN and *inexact is set (render() checks it and raises: the host precheck
// admitted a sigma it should not have).  Also the K:27 exponent step / s1.
__device__ __forceinline__ void epoch_steps_body(int64_t t0, int64_t stride, int64_t n,
                                                 const double *__restrict__ sigma, double s1,
                                                 double s2, double p, double *step, double *ratio,
                                                 int *inexact) {
    for (int64_t i = t0; i < n; i += stride) {
        const double sg = sigma[i];
        const double m = (1.0 < sg) ? 1.0 : sg;   // Python min(sigma, 1.0)
        const double x = fabs(m - 1.0);
        double pw = 0.0;
        bool ok = true;
        if (x == 1.0) pw = 1.0;                    // glibc: pow(1, y) == 1
        else if (x == 0.0 && p > 0.0) pw = 0.0;    // glibc: pow(+0, y > 0) == +0
#if TR_HAVE_GLIBC_POW
        else if (tr_pow_glibc_supported(x, p)) {
            bool exact;
            pw = tr_pow_glibc(x, p, (const uint64_t *)c_lhead, (const uint64_t *)d_ltab,
                              (const uint64_t *)c_ehead, (const uint64_t *)d_etab, &exact);
            ok = exact;
        }
#endif
        else ok = false;
        if (!ok) {
            atomicExch(inexact, 1);
            step[i] = ratio[2 * i] = ratio[2 * i + 1] = __longlong_as_double(0x7ff8000000000000ll);
            continue;
        }
        const double v = s1 + (s2 - s1) * pw;
        const double st = (s1 > v) ? s1 : v;       // Python max(v, s1)
        step[i] = st;
        ratio[2 * i] = st;
        ratio[2 * i + 1] = st / s1;
    }
}

__global__ void epoch_steps_kernel(int64_t n, const double *__restrict__ sigma, double s1,
                                   double s2, double p, double *step, double *ratio, int *inexact) {
    epoch_steps_body(blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
                     (int64_t)gridDim.x * blockDim.x, n, sigma, s1, s2, p, step, ratio, inexact);
}

struct Rows {  // the overlapping rows of one partition (transfer.py:96-110)
    const double *T;
    int64_t n, j0, k;
    double lo, hi, rmin, rmax;
};

// K:74-90
__device__ void tf_lookup(const double *T, int64_t n, double lo, double hi, double v, double c[4]) {
    const double u = (v - lo) / (hi - lo) * (double)(n - 1);
    if (u <= 0.0) { for (int q = 0; q < 4; ++q) c[q] = T[q]; return; }
    if (u >= (double)(n - 1)) { for (int q = 0; q < 4; ++q) c[q] = T[4 * (n - 1) + q]; return; }
    const int64_t j = (int64_t)floor(u);
    const double f = u - (double)j;
    for (int q = 0; q < 4; ++q) c[q] = T[4 * j + q] + f * (T[4 * (j + 1) + q] - T[4 * j + q]);
}

__device__ void row(const Rows &R, int64_t i, double c[4]) {
    if (i == 0) { tf_lookup(R.T, R.n, R.lo, R.hi, R.rmin, c); return; }
    if (i == R.k - 1) { tf_lookup(R.T, R.n, R.lo, R.hi, R.rmax, c); return; }
    const double *t = R.T + 4 * (R.j0 + i - 1);
    for (int q = 0; q < 4; ++q) c[q] = t[q];
}

// squared distance of row i's opacity-weighted colour to the mean
__device__ double sqdist(const Rows &R, int64_t i, const double mean[3]) {
    double c[4];
    row(R, i, c);
    const double d0 = c[0] * c[3] - mean[0], d1 = c[1] * c[3] - mean[1], d2 = c[2] * c[3] - mean[2];
    return ((d0 * d0) + (d1 * d1)) + (d2 * d2);
}

// numpy's pairwise summation (add.reduce over a contiguous float64 vector):
// blocks of <= 128 summed with 8 accumulators, larger ranges split at
// n/2 rounded down to a multiple of 8 and the halves added.  Walked with an
// explicit stack -- recursion would need a dynamically sized device stack.
__device__ double pairwise_block(const Rows &R, const double mean[3], int64_t a, int64_t n) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; ++i) r += sqdist(R, a + i, mean);
        return r;
    }
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = sqdist(R, a + j, mean);
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; ++j) r[j] += sqdist(R, a + i + j, mean);
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += sqdist(R, a + i, mean);
    return res;
}

__device__ double pairwise(const Rows &R, const double mean[3], int64_t a0, int64_t n0) {
    constexpr int DEPTH = 64;  // halving from 2^63 rows
    int64_t sa[DEPTH], sn[DEPTH];
    double sl[DEPTH];
    int sp = 0;
    bool right[DEPTH];
    sa[0] = a0; sn[0] = n0; right[0] = false;
    for (;;) {
        if (sn[sp] > 128) {  // descend into the left half
            int64_t n2 = sn[sp] / 2;
            n2 -= n2 % 8;
            sa[sp + 1] = sa[sp]; sn[sp + 1] = n2; right[sp + 1] = false;
            ++sp;
            continue;
        }
        double ret = pairwise_block(R, mean, sa[sp], sn[sp]);
        for (;;) {  // hand the sum up: a left half starts its sibling, a right half adds
            if (sp == 0) return ret;
            if (!right[sp]) {
                const int64_t n2 = sn[sp];
                sl[sp - 1] = ret;
                sa[sp] = sa[sp - 1] + n2; sn[sp] = sn[sp - 1] - n2; right[sp] = true;
                break;
            }
            --sp;
            ret = sl[sp] + ret;
        }
    }
}

__global__ void tf_meta_kernel(int64_t P, const double *__restrict__ vrange, const double *T,
                               int64_t n, double lo, double hi, double *mop, double *raw,
                               int *err) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= P) return;
    Rows R;
    R.T = T; R.n = n; R.lo = lo; R.hi = hi;
    R.rmin = vrange[2 * p];
    R.rmax = vrange[2 * p + 1];
    if (R.rmin > R.rmax) { atomicExch(err, 1); return; }
    const double u_min = (R.rmin - lo) / (hi - lo) * (double)(n - 1);
    const double u_max = (R.rmax - lo) / (hi - lo) * (double)(n - 1);
    // Python int(floor(.)) semantics, clamped so the cast cannot overflow
    const double fl = fmin(fmax(floor(u_min), -2.0), (double)n + 2.0);
    const double cl = fmin(fmax(ceil(u_max), -2.0), (double)n + 2.0);
    const int64_t j0 = max((int64_t)fl + 1, (int64_t)0);
    const int64_t j1 = min((int64_t)cl - 1, n - 1);
    R.j0 = j0;
    R.k = 2 + ((j1 >= j0) ? j1 - j0 + 1 : 0);
    // alpha.max() and the axis-0 mean of the weighted colours (sequential)
    double amax = -INFINITY, s[3] = {0.0, 0.0, 0.0};
    for (int64_t i = 0; i < R.k; ++i) {
        double c[4];
        row(R, i, c);
        amax = (c[3] > amax) ? c[3] : amax;
        for (int q = 0; q < 3; ++q) {
            const double w = c[q] * c[3];
            s[q] = (i == 0) ? w : s[q] + w;
        }
    }
    const double mean[3] = {s[0] / (double)R.k, s[1] / (double)R.k, s[2] / (double)R.k};
    raw[p] = pairwise(R, mean, 0, R.k) / (double)R.k;
    mop[p] = amax;
}

// normalize_variances (transfer.py:127-141): one CTA reduces min / max
__global__ void tf_normalize_kernel(int64_t P, const double *mop, const double *raw, double *sigma,
                                    uint8_t *active) {
    __shared__ double s_min[1024], s_max[1024];
    double vmin = INFINITY, vmax = -INFINITY;
    for (int64_t p = threadIdx.x; p < P; p += blockDim.x) {
        vmin = fmin(vmin, raw[p]);
        vmax = fmax(vmax, raw[p]);
    }
    s_min[threadIdx.x] = vmin;
    s_max[threadIdx.x] = vmax;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            s_min[threadIdx.x] = fmin(s_min[threadIdx.x], s_min[threadIdx.x + o]);
            s_max[threadIdx.x] = fmax(s_max[threadIdx.x], s_max[threadIdx.x + o]);
        }
        __syncthreads();
    }
    vmin = s_min[0];
    vmax = s_max[0];
    for (int64_t p = threadIdx.x; p < P; p += blockDim.x) {
        if (sigma) sigma[p] = (vmax == vmin) ? 1.0 : (raw[p] - vmin) / (vmax - vmin);
        if (active) active[p] = mop[p] > 0.0 ? 1 : 0;
    }
}

int cuda_fail(cudaError_t e, const char *where) {
    std::string m = std::string(where) + ": " + cudaGetErrorString(e);
    return tr_fail(TR_ECUDA, m.c_str());
}

}  // namespace

extern "C" int tr_epoch_steps_device(int64_t n, const double *sigma, double s1, double s2,
                                     double p, double *step, double *step_ratio, int32_t *inexact,
                                     void *stream) {
    if (n < 0 || (n > 0 && (!sigma || !step || !step_ratio || !inexact)))
        return tr_fail(TR_EINVAL, "tr_epoch_steps_device: invalid arguments");
    if (n == 0) return TR_OK;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    epoch_steps_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(n, sigma, s1, s2, p, step,
                                                                         step_ratio, inexact);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TR_OK : cuda_fail(e, "epoch_steps_kernel");
}

extern "C" int tr_tf_meta_device(int64_t n_parts, const double *vrange, const double *tf_table,
                                 int64_t n_tf, double tf_lo, double tf_hi, double *max_opacity,
                                 double *raw_variance, double *sigma, uint8_t *active,
                                 void *stream) {
    if (n_parts <= 0 || !vrange || !tf_table || n_tf < 2 || !(tf_lo < tf_hi) || !max_opacity ||
        !raw_variance)
        return tr_fail(TR_EINVAL, "tr_tf_meta_device: invalid arguments");
    cudaStream_t st = (cudaStream_t)stream;
    int *d_err = nullptr;
    cudaError_t e = cudaMallocAsync(&d_err, sizeof(int), st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
    cudaMemsetAsync(d_err, 0, sizeof(int), st);
    const int64_t blocks = (n_parts + 127) / 128;
    tf_meta_kernel<<<(unsigned)blocks, 128, 0, st>>>(n_parts, vrange, tf_table, n_tf, tf_lo, tf_hi,
                                                     max_opacity, raw_variance, d_err);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "tf_meta_kernel");
    tf_normalize_kernel<<<1, 1024, 0, st>>>(n_parts, max_opacity, raw_variance, sigma, active);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "tf_normalize_kernel");
    int h_err = 0;
    e = cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFreeAsync(d_err, st);
    if (e != cudaSuccess) return cuda_fail(e, "tr_tf_meta_device");
    if (h_err) return tr_fail(TR_EINVAL, "tr_tf_meta_device: invalid value range (min > max)");
    return TR_OK;
}

namespace {
inline int64_t a64(int64_t x) { return (x + 63) / 64 * 64; }
}

// The epoch's device buffer, 64-B aligned sections:
//   step f64[P] | (step, step / s1) f64[P,2] | sigma f64[P] | tf f64[n_tf,4] |
//   active u8[P] | bnode activity u8[n_b] | knode activity u8[n_k] | inexact i32
// (the inexact word is zero in the staging buffer, so every upload resets it)
extern "C" int64_t tr_epoch_bytes(int64_t n_parts, int64_t n_tf, int64_t n_bnodes,
                                  int64_t n_knodes) {
    const int64_t o_ratio = a64(8 * n_parts), o_sigma = a64(o_ratio + 16 * n_parts);
    const int64_t o_tf = a64(o_sigma + 8 * n_parts), o_act = a64(o_tf + 32 * n_tf);
    const int64_t o_bact = a64(o_act + n_parts), o_kact = a64(o_bact + n_bnodes);
    return a64(o_kact + n_knodes) + 64;
}

extern "C" int tr_epoch_upload(int64_t n_parts, const double *sigma, const uint8_t *active,
                               const uint8_t *bnode_active, int64_t n_bnodes,
                               const uint8_t *knode_active, int64_t n_knodes,
                               const double *tf_table, int64_t n_tf, double tf_lo, double tf_hi,
                               double s1, double s2, double p, int32_t steps_on_device,
                               void *host_buf, void *dev_buf, int64_t buf_bytes, TrEpoch *out,
                               int64_t *h2d_bytes, void *stream) {
    if (n_parts < 1 || !sigma || !active || !tf_table || n_tf < 2 || !host_buf || !dev_buf || !out ||
        n_bnodes < 0 || n_knodes < 0 || (n_bnodes && !bnode_active) || (n_knodes && !knode_active))
        return tr_fail(TR_EINVAL, "tr_epoch_upload: invalid arguments");
    if (buf_bytes < tr_epoch_bytes(n_parts, n_tf, n_bnodes, n_knodes))
        return tr_fail(TR_EINVAL, "tr_epoch_upload: buffer too small");
    const int64_t o_ratio = a64(8 * n_parts), o_sigma = a64(o_ratio + 16 * n_parts);
    const int64_t o_tf = a64(o_sigma + 8 * n_parts), o_act = a64(o_tf + 32 * n_tf);
    const int64_t o_bact = a64(o_act + n_parts), o_kact = a64(o_bact + n_bnodes);
    const int64_t o_flag = a64(o_kact + n_knodes), nbytes = o_flag + 64;
    char *h = static_cast<char *>(host_buf), *d = static_cast<char *>(dev_buf);
    std::memset(h + o_flag, 0, 64);
    int32_t *inexact = reinterpret_cast<int32_t *>(d + o_flag);
    std::memcpy(h + o_sigma, sigma, 8 * n_parts);
    std::memcpy(h + o_tf, tf_table, 32 * n_tf);
    std::memcpy(h + o_act, active, n_parts);
    if (n_bnodes) std::memcpy(h + o_bact, bnode_active, n_bnodes);
    if (n_knodes) std::memcpy(h + o_kact, knode_active, n_knodes);
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e;
    if (steps_on_device) {
        // only sigma, the TF and the activity bits cross PCIe
        e = cudaMemcpyAsync(d + o_sigma, h + o_sigma, nbytes - o_sigma, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return cuda_fail(e, "tr_epoch_upload H2D");
        if (int rc = tr_epoch_steps_device(n_parts, reinterpret_cast<const double *>(d + o_sigma), s1,
                                           s2, p, reinterpret_cast<double *>(d),
                                           reinterpret_cast<double *>(d + o_ratio), inexact, stream))
            return rc;
        if (h2d_bytes) *h2d_bytes = nbytes - o_sigma;
    } else {
        if (int rc = tr_epoch_steps(n_parts, sigma, s1, s2, p, reinterpret_cast<double *>(h),
                                    reinterpret_cast<double *>(h + o_ratio)))
            return rc;
        e = cudaMemcpyAsync(d, h, nbytes, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return cuda_fail(e, "tr_epoch_upload H2D");
        if (h2d_bytes) *h2d_bytes = nbytes;
    }
    out->active = reinterpret_cast<const uint8_t *>(d + o_act);
    out->bnode_active = reinterpret_cast<const uint8_t *>(d + o_bact);
    out->step = reinterpret_cast<const double *>(d);
    out->tf_table = reinterpret_cast<const double *>(d + o_tf);
    out->n_tf = n_tf;
    out->tf_lo = tf_lo;
    out->tf_hi = tf_hi;
    out->knode_active = reinterpret_cast<const uint8_t *>(d + o_kact);
    out->step_ratio = reinterpret_cast<const double *>(d + o_ratio);
    out->inexact = steps_on_device ? inexact : nullptr;
    return TR_OK;
}

// A packed epoch's re-upload in one launch: the sections after the steps
// (sigma, TF, activity bits) are read from the page-locked block over PCIe
// (mapped host memory) and stored in HBM, and the steps are recomputed from
// the sigma read (epoch_steps_kernel's arithmetic).  The inexact word is not
// touched: the block is the one whose first upload zeroed and then checked it,
// and the same sigma gives the same steps.
__global__ void __launch_bounds__(256) epoch_refresh_kernel(const int4 *__restrict__ src, int4 *dst,
                                                            int64_t n16, int64_t n,
                                                            const double *sigma_h, double s1,
                                                            double s2, double p, double *step,
                                                            double *ratio, int *inexact) {
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = t0; i < n16; i += stride) dst[i] = src[i];
    epoch_steps_body(t0, stride, n, sigma_h, s1, s2, p, step, ratio, inexact);
}

extern "C" int tr_epoch_upload_s(const TrEpochUpload *u, TrEpoch *out, int64_t *h2d_bytes,
                                 void *stream) {
    if (!u) return tr_fail(TR_EINVAL, "tr_epoch_upload_s: invalid arguments");
    if (u->packed && u->steps_on_device) {
        const int64_t n = u->n_parts;
        if (n < 1 || !u->host_buf || !u->dev_buf || !out ||
            u->buf_bytes < tr_epoch_bytes(n, u->n_tf, u->n_bnodes, u->n_knodes))
            return tr_fail(TR_EINVAL, "tr_epoch_upload_s: packed re-upload of an epoch never uploaded");
        const int64_t o_ratio = a64(8 * n), o_sigma = a64(o_ratio + 16 * n);
        const int64_t o_tf = a64(o_sigma + 8 * n), o_act = a64(o_tf + 32 * u->n_tf);
        const int64_t o_bact = a64(o_act + n), o_kact = a64(o_bact + u->n_bnodes);
        const int64_t o_flag = a64(o_kact + u->n_knodes);
        void *hd = nullptr;
        cudaError_t e = cudaHostGetDevicePointer(&hd, u->host_buf, 0);
        if (e != cudaSuccess) return cuda_fail(e, "tr_epoch_upload_s: host block not mapped");
        const char *h = static_cast<const char *>(hd);
        char *d = static_cast<char *>(u->dev_buf);
        const int64_t n16 = (o_flag - o_sigma) / 16;   // offsets are 64-B aligned
        int64_t blocks = (n16 + 255) / 256;
        if (blocks > 148) blocks = 148;
        epoch_refresh_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
            reinterpret_cast<const int4 *>(h + o_sigma), reinterpret_cast<int4 *>(d + o_sigma), n16, n,
            reinterpret_cast<const double *>(h + o_sigma), u->s1, u->s2, u->p,
            reinterpret_cast<double *>(d), reinterpret_cast<double *>(d + o_ratio),
            reinterpret_cast<int *>(d + o_flag));
        if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "epoch_refresh_kernel");
        if (h2d_bytes) *h2d_bytes = o_flag - o_sigma;
        out->active = reinterpret_cast<const uint8_t *>(d + o_act);
        out->bnode_active = reinterpret_cast<const uint8_t *>(d + o_bact);
        out->step = reinterpret_cast<const double *>(d);
        out->tf_table = reinterpret_cast<const double *>(d + o_tf);
        out->n_tf = u->n_tf;
        out->tf_lo = u->tf_lo;
        out->tf_hi = u->tf_hi;
        out->knode_active = reinterpret_cast<const uint8_t *>(d + o_kact);
        out->step_ratio = reinterpret_cast<const double *>(d + o_ratio);
        out->inexact = reinterpret_cast<int32_t *>(d + o_flag);
        return TR_OK;
    }
    return tr_epoch_upload(u->n_parts, u->sigma, u->active, u->bnode_active, u->n_bnodes,
                           u->knode_active, u->n_knodes, u->tf_table, u->n_tf, u->tf_lo, u->tf_hi,
                           u->s1, u->s2, u->p, u->steps_on_device, u->host_buf, u->dev_buf,
                           u->buf_bytes, out, h2d_bytes, stream);
}
