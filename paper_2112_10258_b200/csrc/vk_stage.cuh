// vk_stage.cuh -- plane-staged walk of an interior keypoint ball.
//
// The orientation (orient.py:89-125) and SIFT-Rank (descriptor.py:227-263)
// fast paths visit every voxel of the keypoint's integer ball and need its
// six axis neighbours (central differences, volume.py:244-264).  Gathering
// those from L1/L2 per visit leaves the walks latency-bound (~12% issue
// utilisation measured on B200).  Here the ball's bounding box (+1 halo) is
// staged plane by plane into a 4-slot shared-memory ring with cp.async
// (coalesced row segments, three planes ahead of the visits), and each ball
// plane oz is visited from the staged planes oz-1, oz, oz+1: six shared loads
// per visit, bit-identical values.  One barrier per plane.
//
// Only for balls whose box lies inside the volume (ball_interior) and whose
// radius is <= kStageMaxR; the caller keeps its global-memory walk otherwise.
#pragma once

#include "vk_common.cuh"

namespace vk {

constexpr int kStageMaxR = 17;
constexpr int kStageMaxW = 2 * kStageMaxR + 3;
constexpr int kStageSlots = 4;
constexpr int kStageFloats = kStageSlots * kStageMaxW * kStageMaxW;

// visit(valid, ox, oy, oz, nb): every ball voxel once (z-major order inside a
// plane, consecutive threads take consecutive entries); called by every
// thread of the CTA the same number of times per plane (valid = false past
// the plane's entries), so visit may use warp collectives.
// plane_starts[k] .. [k+1] are the z-major entries of ball plane oz = k - r.
template <class Visit>
VK_D void staged_ball_walk(const float* __restrict__ data, int nx, int ny, const vk_kp& kp, const vk_ball& ball,
                           const int* __restrict__ zoffs, const int* __restrict__ plane_starts, float* ring,
                           Visit&& visit) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int r = ball.r, W = 2 * r + 3, WW = W * W, NP = 2 * r + 3;
    const unsigned plane = (unsigned)nx * (unsigned)ny;
    // staged plane p <-> z = iz - r - 1 + p, rows iy - r - 1 .., columns ix - r - 1 ..
    const float* box = data + ((size_t)(kp.iz - r - 1) * plane + (size_t)(kp.iy - r - 1) * nx + (kp.ix - r - 1));
    auto stage = [&](int p) {
        if (p < NP) {
            float* d = ring + (p & 3) * WW;
            const float* s = box + (size_t)p * plane;
            for (int e = tid; e < WW; e += nt) {
                const int row = e / W;
                cp_async4(d + e, s + row * nx + (e - row * W));
            }
        }
        cp_async_commit();  // (an empty group keeps the wait_group count uniform)
    };
    stage(0);
    stage(1);
    stage(2);
    for (int k = 0; k <= 2 * r; ++k) {
        stage(k + 3);        // slot (k + 3) & 3 was last read in iteration k - 1 (barrier at its end)
        cp_async_wait<1>();  // planes <= k + 2 have landed (this thread's copies)
        __syncthreads();     // ... and everyone's
        const float* s0 = ring + (k & 3) * WW;
        const float* s1 = ring + ((k + 1) & 3) * WW;
        const float* s2 = ring + ((k + 2) & 3) * WW;
        const int oz = k - r;
        const int e0 = __ldg(plane_starts + k), e1 = __ldg(plane_starts + k + 1);
        for (int base = e0; base < e1; base += nt) {
            const int e = base + tid;
            const bool valid = e < e1;
            const int pk = valid ? __ldg(zoffs + e) : 0;
            const int ox = unpack_off(pk, 0), oy = unpack_off(pk, 1);
            Nb6 nb{};
            if (valid) {
                const int c = (oy + r + 1) * W + (ox + r + 1);
                nb.xh = s1[c + 1];
                nb.xl = s1[c - 1];
                nb.yh = s1[c + W];
                nb.yl = s1[c - W];
                nb.zh = s2[c];
                nb.zl = s0[c];
            }
            nb.sx = nb.sy = nb.sz = 0.5f;
            visit(valid, ox, oy, oz, nb);
        }
        __syncthreads();
    }
    cp_async_wait<0>();
}

}  // namespace vk
