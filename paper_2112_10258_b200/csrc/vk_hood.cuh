// vk_hood.cuh -- accumulation of a keypoint neighbourhood's (bin, vote)
// stream into a per-CTA histogram.
//
// The fast paths of orientation (orient.py:89-125) and SIFT-Rank
// (descriptor.py:227-263) turn every ball voxel into one (bin, fp32 vote)
// pair.  Votes are added with fire-and-forget fp64 reductions (RED.ADD.F64)
// into a small per-CTA histogram in global memory, which stays in L2: no
// warp-level conflict resolution, no shared-memory CAS loops (sm_100 has no
// native shared-memory float atomics), and the fp64 sum of fp32 votes differs
// from any other fp64 summation order by at most gamma_n -- the callers'
// certification bounds only need the vote error (kVoteRel) and that term.
#pragma once

#include "vk_common.cuh"

namespace vk {

// Each CTA accumulates into kVoteCopies copies of its histogram, lane l
// voting into copy l % kVoteCopies; the copies are summed when the histogram
// is read (fp64, any order: the bounds hold for every summation order).
// Measured on B200 after the walks were pipelined: 2 copies make the
// SIFT-Rank walk 13% faster than 1 (4: same as 2, 8 / 16: slower; spreading
// the entries of one copy over more sectors, VK_BIN_STRIDE, slower).
#ifndef VK_VOTE_COPIES
#define VK_VOTE_COPIES 2
#endif
constexpr int kVoteCopies = VK_VOTE_COPIES;
// Histogram entry i lives at hist[i * kBinStride] (entries spread over more
// L2 sectors / slices).
#ifndef VK_BIN_STRIDE
#define VK_BIN_STRIDE 1
#endif
constexpr int kBinStride = VK_BIN_STRIDE;
// Doubles per copy (>= VK_MAX_FRAMES x 64 SIFT-Rank bins and >= VK_MAX_DIRS
// orientation bins, times the entry stride).
constexpr int kCopyStride = VK_MAX_FRAMES * 64 * kBinStride;
// Offset of SIFT-Rank frame f's 64 bins: hist + f * kHistFrame.
constexpr int kHistFrame = 64 * kBinStride;
// Histogram slots per CTA in the accumulation workspace.
constexpr int kAccumSlot = kCopyStride * kVoteCopies;
// Persistent grids launch at most this many CTAs per SM.
#ifndef VK_ACCUM_CTAS_PER_SM
#define VK_ACCUM_CTAS_PER_SM 4
#endif
constexpr int kAccumCtasPerSm = VK_ACCUM_CTAS_PER_SM;

// Grid of a persistent accumulation kernel: every CTA resident at once (the
// occupancy the kernel's registers allow, at most kAccumCtasPerSm per SM), so
// no CTA waits for a second wave with its share of the items.
template <class Kernel>
inline int accum_grid(Kernel kernel, int threads, int n_items, size_t dyn_smem = 0) {
    int dev = 0, sms = 148, occ = kAccumCtasPerSm;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, dyn_smem) != cudaSuccess || occ < 1) occ = 1;
    const int g = sms * (occ < kAccumCtasPerSm ? occ : kAccumCtasPerSm);
    return n_items < g ? n_items : g;
}

// First item of persistent CTA b: within each round of gridDim.x items, the
// CTAs b, b + nsm, b + 2 nsm, ... -- co-resident on one SM under the in-order
// block dispatch of a grid of nsm x occupancy CTAs -- take consecutive items
// (neighbouring keypoints: their balls overlap in the SM's L1).  A bijection
// on [0, gridDim.x) whatever the actual placement (identity when the grid is
// not a multiple of the SM count); round r adds r x gridDim.x.
#ifndef VK_SM_LOCAL_ITEMS
#define VK_SM_LOCAL_ITEMS 0  // measured: orientation -6% / SIFT-Rank +8% on one batch, whole step -3%: off
#endif
VK_D int first_item() {
    const int b = blockIdx.x, g = gridDim.x;
    if (!VK_SM_LOCAL_ITEMS) return b;
    unsigned nsm;
    asm("mov.u32 %0, %%nsmid;" : "=r"(nsm));
    const int c = (int)nsm;
    if (c <= 0 || g % c != 0) return b;
    return (b % c) * (g / c) + b / c;
}

// This thread's copy of the CTA histogram.
VK_D double* vote_copy(double* hist) { return hist + (threadIdx.x & (kVoteCopies - 1)) * kCopyStride; }

VK_D void red_vote(double* hist, int bin, float v) {
    if (bin >= 0) atomicAdd(hist + bin * kBinStride, (double)v);  // result unused -> RED.E.ADD.F64.RN
}

// Zero the first n entries of every copy (the caller synchronises).
VK_D void zero_hist(double* hist, int n) {
    for (int i = threadIdx.x; i < n * kVoteCopies; i += blockDim.x) hist[(i / n) * kCopyStride + (i % n) * kBinStride] = 0.0;
}

// Entry i summed over the copies, after a __syncthreads (L2, bypassing L1).
VK_D double read_hist(const double* hist, int i) {
    double s = __ldcg(hist + i * kBinStride);
#pragma unroll
    for (int c = 1; c < kVoteCopies; ++c) s += __ldcg(hist + c * kCopyStride + i * kBinStride);
    return s;
}

}  // namespace vk
