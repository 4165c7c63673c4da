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

// Histogram slots per CTA in the accumulation workspace (>= VK_MAX_FRAMES x 64
// SIFT-Rank bins and >= VK_MAX_DIRS orientation bins).
constexpr int kAccumSlot = VK_MAX_FRAMES * 64;
// Persistent grids launch at most this many CTAs per SM.
constexpr int kAccumCtasPerSm = 4;

VK_D void red_vote(double* hist, int bin, float v) {
    if (bin >= 0) atomicAdd(hist + bin, (double)v);  // result unused -> RED.E.ADD.F64.RN
}

// Zero this CTA's first n histogram entries (the caller synchronises).
VK_D void zero_hist(double* hist, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) hist[i] = 0.0;
}

// Read a reduced entry back after a __syncthreads (L2, bypassing L1).
VK_D double read_hist(const double* hist, int i) { return __ldcg(hist + i); }

}  // namespace vk
