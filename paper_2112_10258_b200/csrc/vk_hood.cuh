// vk_hood.cuh -- keypoint neighbourhoods staged in shared memory, and
// warp-level accumulation of (bin, vote) streams.
//
// A keypoint's integer ball (orient.py:244-255) is walked plane by plane
// (z-major point table, tables.BallTable).  Its bounding box is streamed into
// shared memory as z-slabs of T ball planes plus one halo plane on each side,
// each plane a W x W tile (W = 2r + 3), loaded with coalesced cp.async rows.
// Out-of-volume tile entries hold the clamped (replicated) voxel, so the
// central / one-sided gradient of volume.py:244-264 reads its neighbours
// straight from the tile and only the divisor depends on the volume bounds.
#pragma once

#include "vk_common.cuh"

namespace vk {

struct Box {
    int x0, y0;  // tile origin (cx - r - 1, cy - r - 1)
    int W;       // tile side, 2r + 3
    int nx, ny, nz;
};

// Stage planes z_first .. z_first + nplanes - 1 (clamped) of the box.
VK_D void stage_slab(float* buf, const float* __restrict__ data, const Box& b, int z_first, int nplanes) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int rows = nplanes * b.W;
    for (int row = warp; row < rows; row += nw) {
        const int p = row / b.W, yy = row - p * b.W;
        const int z = clampi(z_first + p, 0, b.nz - 1), y = clampi(b.y0 + yy, 0, b.ny - 1);
        const float* src = data + ((long long)z * b.ny + y) * b.nx;
        float* dst = buf + row * b.W;
        for (int xx = lane; xx < b.W; xx += 32) cp_async4(dst + xx, src + clampi(b.x0 + xx, 0, b.nx - 1));
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
}

// The six neighbours of lattice point (x, y, z) from a staged slab whose
// first plane is volume plane zb.
VK_D Nb6 slab_nb6(const float* buf, const Box& b, int zb, int x, int y, int z) {
    const int W = b.W;
    const int c = ((z - zb) * W + (y - b.y0)) * W + (x - b.x0);
    Nb6 n;
    n.xh = buf[c + 1];
    n.xl = buf[c - 1];
    n.yh = buf[c + W];
    n.yl = buf[c - W];
    n.zh = buf[c + W * W];
    n.zl = buf[c - W * W];
    n.sx = (min(x + 1, b.nx - 1) - max(x - 1, 0)) == 2 ? 0.5f : 1.0f;
    n.sy = (min(y + 1, b.ny - 1) - max(y - 1, 0)) == 2 ? 0.5f : 1.0f;
    n.sz = (min(z + 1, b.nz - 1) - max(z - 1, 0)) == 2 ? 0.5f : 1.0f;
    return n;
}

// Add every lane's (bin, v) into this warp's private histogram (fp64).  If
// all voting lanes share one bin (the common case: a warp walks 32
// neighbouring voxels) the votes are butterfly-summed in fp32 and added by one
// lane.  Otherwise runs of equal bins in lane order are reduced with a
// segmented fp32 shuffle scan and added by their last lane; runs of the same
// bin that are not contiguous are added in successive rounds, so no two lanes
// ever update one bin at once.  All 32 lanes must call this (bin < 0 = no
// vote).  Each vote passes a depth <= 5 fp32 addition tree (kRunRel) before
// the fp64 accumulation; callers bound the difference to reference order.
VK_D void warp_accum(double* hist, int bin, float v) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned act = __ballot_sync(FULL, bin >= 0);
    if (act == 0) return;
    const int b0 = __shfl_sync(FULL, bin, __ffs(act) - 1);
    if (__all_sync(FULL, bin < 0 || bin == b0)) {
        float s = bin >= 0 ? v : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s = fadd(s, __shfl_xor_sync(FULL, s, o));
        if (lane == 0) hist[b0] = dadd(hist[b0], (double)s);
        __syncwarp();
        return;
    }
    const int prev = __shfl_up_sync(FULL, bin, 1);
    const bool head = lane == 0 || prev != bin;
    const unsigned heads = __ballot_sync(FULL, head);
    const int start = 31 - __clz(heads & (FULL >> (31 - lane)));
    float s = bin >= 0 ? v : 0.f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float t = __shfl_up_sync(FULL, s, o);
        if (lane - o >= start) s = fadd(s, t);
    }
    const bool tail = lane == 31 || ((heads >> (lane + 1)) & 1u);
    const bool on = tail && bin >= 0;
    const unsigned peers = __match_any_sync(FULL, on ? bin : -1 - lane);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    const int rounds = __reduce_max_sync(FULL, on ? (unsigned)__popc(peers) : 0u);
    for (int r = 0; r < rounds; ++r) {
        if (on && rank == r) hist[bin] = dadd(hist[bin], (double)s);
        __syncwarp();
    }
}

// Register-resident variant: this warp's histogram lives in registers, lane L
// owning bins L (acc0) and L + 32 (acc1).  Uniform warps butterfly-sum and the
// owner adds; otherwise runs of equal bins are scan-reduced and each run's
// (bin, sum) is broadcast from its last lane to the owner.  Same error model
// as warp_accum (depth-5 fp32 tree per vote, then fp64).
VK_D void warp_accum_reg(double& acc0, double& acc1, int bin, float v) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned act = __ballot_sync(FULL, bin >= 0);
    if (act == 0) return;
    const int b0 = __shfl_sync(FULL, bin, __ffs(act) - 1);
    if (__all_sync(FULL, bin < 0 || bin == b0)) {
        float s = bin >= 0 ? v : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s = fadd(s, __shfl_xor_sync(FULL, s, o));
        if ((b0 & 31) == lane) {
            if (b0 < 32) acc0 = dadd(acc0, (double)s);
            else acc1 = dadd(acc1, (double)s);
        }
        return;
    }
    const int prev = __shfl_up_sync(FULL, bin, 1);
    const unsigned heads = __ballot_sync(FULL, lane == 0 || prev != bin);
    const int start = 31 - __clz(heads & (FULL >> (31 - lane)));
    float s = bin >= 0 ? v : 0.f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float t = __shfl_up_sync(FULL, s, o);
        if (lane - o >= start) s = fadd(s, t);
    }
    // tails: last lane of every run that votes
    unsigned tails = __ballot_sync(FULL, bin >= 0 && (lane == 31 || ((heads >> (lane + 1)) & 1u)));
    while (tails) {
        const int t = __ffs(tails) - 1;
        tails &= tails - 1;
        const int bt = __shfl_sync(FULL, bin, t);
        const float st = __shfl_sync(FULL, s, t);
        if ((bt & 31) == lane) {
            if (bt < 32) acc0 = dadd(acc0, (double)st);
            else acc1 = dadd(acc1, (double)st);
        }
    }
}

// Ball plane range [oz0, oz0 + nT) -> z-major point index range.
VK_D void plane_range(const int* __restrict__ plane_starts, const vk_ball& ball, int oz0, int nT, int& ps, int& pe) {
    ps = __ldg(plane_starts + ball.pstart + oz0 + ball.r);
    pe = __ldg(plane_starts + ball.pstart + oz0 + nT + ball.r);
}

}  // namespace vk
