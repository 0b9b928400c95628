// Noise calibration on the GPU (the reference's
// noise_calib.cpp:102-182): the disparity-error histograms behind the Kalman
// filter's q (process noise: ground truth warped by the ego-motion vs the next
// frame's ground truth) and r (measurement noise: full-range SGM vs ground
// truth), and the per-pixel accumulated warp error map.
//
// The heavy stages reuse the step's kernels (the forward warp A6 and the
// full-range cost / aggregation / WTA chain). This file adds:
//   gt_state_kernel     state_from_gt (noise_calib.cpp:71-78): d = gt, p = 0,
//                       valid iff gt > 0
//   error_hist_kernel   ErrorHistogram::add (noise_calib.cpp:16-33) over a
//                       batch of maps: integer tallies (exact, any order) and
//                       the gated FP64 sums in a FIXED reduction order (thread
//                       strides, block tree, serial over blocks), so results
//                       are deterministic run to run and independent of the
//                       device; they differ from the reference's raster-order
//                       sums only by FP64 reassociation (tests: variance 1e-9 relative; on
//                       12 M samples the difference measured 1.7e-12)
//   error_map_kernel    accumulate_error_map (noise_calib.cpp:149-182): one
//                       thread per pixel adds |warped - gt| over the pairs in
//                       frame order, i.e. the reference's own order: bit-exact
#include "common.cuh"

namespace tsgm {

constexpr int kHistBlocks = 1184;  // fixed (not per-device): the sums' order is fixed
constexpr int kHistThreads = 256;
constexpr int kHistSmemBins = 8192;

__global__ void gt_state_kernel(const double* gt, size_t P, int n, const int* slots, double* sd,
                                double* sp, uint8_t* sv) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    const int a = blockIdx.y;
    if (i >= P) return;
    const double g = gt[static_cast<size_t>(a) * P + i];
    const size_t t = static_cast<size_t>(slots[a]) * P + i;
    const bool v = g > 0.0;
    sd[t] = v ? g : 0.0;
    sp[t] = 0.0;
    sv[t] = v ? 1 : 0;
}

void launch_gt_state(const Bufs& b, const double* gt, int n, Launch L) {
    gt_state_kernel<<<dim3((b.P + 255) / 256, n), 256, 0, L.st>>>(gt, b.P, n, b.slots, b.sd, b.sp,
                                                                 b.sv);
    ++*L.counter;
}

// est: per-slot maps (slot stride P) of T = double (warped d) or int32 (WTA),
// est_v their validity; gt: n maps, batch-major.
template <typename T>
__global__ void __launch_bounds__(kHistThreads)
    error_hist_kernel(const T* est, const uint8_t* est_v, const int* slots, const double* gt,
                      size_t P, int n, HistSpec hs, HistAcc acc) {
    extern __shared__ unsigned int hsm[];
    __shared__ double red[2][kHistThreads];
    __shared__ unsigned long long tal[4];
    const bool smem_bins = hs.nbins <= kHistSmemBins;
    if (smem_bins)
        for (int k = threadIdx.x; k < hs.nbins; k += blockDim.x) hsm[k] = 0u;
    if (threadIdx.x < 4) tal[threadIdx.x] = 0ull;
    __syncthreads();
    double sum = 0.0, sq = 0.0;
    unsigned int under = 0, over = 0, within = 0, gated = 0;
    const size_t total = P * static_cast<size_t>(n);
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total; i += stride) {
        const size_t a = i / P, p = i - a * P;
        const size_t t = static_cast<size_t>(slots[a]) * P + p;
        const double g = gt[i];
        if (!est_v[t] || !(g > 0.0)) continue;
        const double e = static_cast<double>(est[t]) - g;
        if (fabs(e) <= 1.0) ++within;
        if (e < hs.lo) {
            ++under;
            continue;
        }
        if (e >= hs.hi) {
            ++over;
            continue;
        }
        size_t bin = static_cast<size_t>(__ddiv_rn(__dsub_rn(e, hs.lo), hs.bw));
        if (bin >= static_cast<size_t>(hs.nbins)) bin = static_cast<size_t>(hs.nbins) - 1;
        if (smem_bins) atomicAdd(hsm + bin, 1u);
        else atomicAdd(acc.counts + bin, 1ull);
        ++gated;
        sum = __dadd_rn(sum, e);
        sq = __dadd_rn(sq, __dmul_rn(e, e));
    }
    // tallies: exact in any order
    atomicAdd(&tal[0], static_cast<unsigned long long>(under));
    atomicAdd(&tal[1], static_cast<unsigned long long>(over));
    atomicAdd(&tal[2], static_cast<unsigned long long>(within));
    atomicAdd(&tal[3], static_cast<unsigned long long>(gated));
    // sums: fixed block tree
    red[0][threadIdx.x] = sum;
    red[1][threadIdx.x] = sq;
    __syncthreads();
    for (int o = kHistThreads / 2; o > 0; o >>= 1) {
        if (static_cast<int>(threadIdx.x) < o) {
            red[0][threadIdx.x] = __dadd_rn(red[0][threadIdx.x], red[0][threadIdx.x + o]);
            red[1][threadIdx.x] = __dadd_rn(red[1][threadIdx.x], red[1][threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        acc.partial[2 * blockIdx.x] = red[0][0];
        acc.partial[2 * blockIdx.x + 1] = red[1][0];
    }
    if (threadIdx.x < 4) atomicAdd(acc.tallies + threadIdx.x, tal[threadIdx.x]);
    if (smem_bins)
        for (int k = threadIdx.x; k < hs.nbins; k += blockDim.x)
            if (hsm[k]) atomicAdd(acc.counts + k, static_cast<unsigned long long>(hsm[k]));
}

// Serial over the blocks in block order, added to the running sums of earlier
// batches (sums[0], sums[1]).
__global__ void hist_sums_kernel(const double* partial, int blocks, double* sums) {
    double s = sums[0], q = sums[1];
    for (int k = 0; k < blocks; ++k) {
        s = __dadd_rn(s, partial[2 * k]);
        q = __dadd_rn(q, partial[2 * k + 1]);
    }
    sums[0] = s;
    sums[1] = q;
}

size_t hist_partial_doubles() { return 2 * static_cast<size_t>(kHistBlocks); }

template <typename T>
static void launch_hist(const T* est, const uint8_t* est_v, const Bufs& b, const double* gt,
                        int n, const HistSpec& hs, const HistAcc& acc, Launch L) {
    const size_t smem = hs.nbins <= kHistSmemBins ? sizeof(unsigned int) * hs.nbins : 0;
    error_hist_kernel<T><<<kHistBlocks, kHistThreads, smem, L.st>>>(est, est_v, b.slots, gt, b.P, n,
                                                                     hs, acc);
    hist_sums_kernel<<<1, 1, 0, L.st>>>(acc.partial, kHistBlocks, acc.sums);
    *L.counter += 2;
}

void launch_error_hist_warped(const Bufs& b, const double* gt, int n, const HistSpec& hs,
                              const HistAcc& acc, Launch L) {
    launch_hist(b.wd, b.wv, b, gt, n, hs, acc, L);
}

void launch_error_hist_wta(const Bufs& b, const double* gt, int n, const HistSpec& hs,
                           const HistAcc& acc, Launch L) {
    launch_hist(b.md, b.mv, b, gt, n, hs, acc, L);
}

// acc[p] += |wd - gt| over the batch's pairs in order (pair a: slot slots[a]
// against gt map a); overlap counts the contributing samples.
__global__ void error_map_kernel(const Bufs b, const double* gt, int n, double* acc,
                                 unsigned long long* overlap) {
    const size_t p = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    unsigned int cnt = 0;
    if (p < b.P) {
        double s = acc[p];
        for (int a = 0; a < n; ++a) {
            const size_t t = static_cast<size_t>(b.slots[a]) * b.P + p;
            const double g = gt[static_cast<size_t>(a) * b.P + p];
            if (b.wv[t] && g > 0.0) {
                s = __dadd_rn(s, fabs(__dsub_rn(b.wd[t], g)));
                ++cnt;
            }
        }
        acc[p] = s;
    }
    const unsigned int w = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0 && w) atomicAdd(overlap, static_cast<unsigned long long>(w));
}

void launch_error_map(const Bufs& b, const double* gt, int n, double* acc,
                      unsigned long long* overlap, Launch L) {
    error_map_kernel<<<static_cast<unsigned>((b.P + 255) / 256), 256, 0, L.st>>>(b, gt, n, acc,
                                                                                 overlap);
    ++*L.counter;
}

}  // namespace tsgm
