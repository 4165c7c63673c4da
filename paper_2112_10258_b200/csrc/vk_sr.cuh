// vk_sr.cuh -- device building blocks of the SIFT-Rank walk (descriptor.py:227-263):
// certified fp32 octant bins, deferred uncertain octants, the fast / pipelined ball
// walks, stable ranks and the exact repair of uncertain bins.  Shared by
// siftrank_kernel (vk_describe.cu) and the fused kernel (vk_orsr.cu).
#pragma once

#include "vk_hood.cuh"

namespace vk {

#ifndef VK_SR_THREADS
#define VK_SR_THREADS 256
#endif
constexpr int kSrThreads = VK_SR_THREADS;
constexpr int kPrefetchPlanes = 3;  // z-plane lead of the L1 prefetch in the ball walk
constexpr int kSrBins = 64;

VK_D int sr_vote(const float* data, int nx, int ny, int nz, int cx, int cy, int cz, int packed, const double* R,
                 double& mag, bool& inside) {
    const int ox = unpack_off(packed, 0), oy = unpack_off(packed, 1), oz = unpack_off(packed, 2);
    const int x = cx + ox, y = cy + oy, z = cz + oz;
    inside = x >= 0 && y >= 0 && z >= 0 && x < nx && y < ny && z < nz;
    if (!inside) return -1;
    double gx, gy, gz;
    gradient_at(data, nx, ny, nz, x, y, z, gx, gy, gz);
    const double o0 = (double)ox, o1 = (double)oy, o2 = (double)oz;
    // offs @ R and grads @ R: out[j] = sum_k v[k] R[k][j] (FMA chain over k)
    const double r0 = dot3_blas(o0, o1, o2, R[0], R[3], R[6]);
    const double r1 = dot3_blas(o0, o1, o2, R[1], R[4], R[7]);
    const double r2 = dot3_blas(o0, o1, o2, R[2], R[5], R[8]);
    const double g0 = dot3_blas(gx, gy, gz, R[0], R[3], R[6]);
    const double g1 = dot3_blas(gx, gy, gz, R[1], R[4], R[7]);
    const double g2 = dot3_blas(gx, gy, gz, R[2], R[5], R[8]);
    const int sp = (r0 > 0.0) + 2 * (r1 > 0.0) + 4 * (r2 > 0.0);
    const int orr = (g0 > 0.0) + 2 * (g1 > 0.0) + 4 * (g2 > 0.0);
    mag = norm3_numpy(g0, g1, g2);
    return sp * 8 + orr;
}

// Rare path, out of line: the reference's fp64 FMA-chain octant bits.
static __device__ __noinline__ int sr_bin_exact(int ox, int oy, int oz, double x64, double y64, double z64,
                                         const double* R) {
    const double o0 = (double)ox, o1 = (double)oy, o2 = (double)oz;
    const double r0 = dot3_blas(o0, o1, o2, R[0], R[3], R[6]);
    const double r1 = dot3_blas(o0, o1, o2, R[1], R[4], R[7]);
    const double r2 = dot3_blas(o0, o1, o2, R[2], R[5], R[8]);
    const double g0 = dot3_blas(x64, y64, z64, R[0], R[3], R[6]);
    const double g1 = dot3_blas(x64, y64, z64, R[1], R[4], R[7]);
    const double g2 = dot3_blas(x64, y64, z64, R[2], R[5], R[8]);
    return 8 * ((r0 > 0.0) + 2 * (r1 > 0.0) + 4 * (r2 > 0.0)) + (g0 > 0.0) + 2 * (g1 > 0.0) + 4 * (g2 > 0.0);
}

// Rare path: reference fp64 octant bits of the rotated gradient (reloads the
// neighbours: only the fp32 gradient is at hand).
#ifndef VK_SR_GBITS_INLINE
#define VK_SR_GBITS_INLINE 0
#endif
#if VK_SR_GBITS_INLINE
static __device__ __forceinline__
#else
static __device__ __noinline__
#endif
int sr_gbits_exact(const float* data, int nx, int ny, int nz, int x, int y, int z,
                                           const double* R) {
    const Nb6 n = load_nb6(data, nx, ny, nz, x, y, z);
    double x64, y64, z64;
    grad64(n, x64, y64, z64);
    const double g0 = dot3_blas(x64, y64, z64, R[0], R[3], R[6]);
    const double g1 = dot3_blas(x64, y64, z64, R[1], R[4], R[7]);
    const double g2 = dot3_blas(x64, y64, z64, R[2], R[5], R[8]);
    return (g0 > 0.0) + 2 * (g1 > 0.0) + 4 * (g2 > 0.0);
}

// Rare path: reference fp64 octant bits of the rotated integer offset.
#ifndef VK_SR_OBITS_INLINE
#define VK_SR_OBITS_INLINE 1  // measured: inline 1.3% faster than a call
#endif
#if VK_SR_OBITS_INLINE
static __device__ __forceinline__
#else
static __device__ __noinline__
#endif
int sr_obits_exact(int ox, int oy, int oz, const double* R) {
    const double o0 = (double)ox, o1 = (double)oy, o2 = (double)oz;
    return (dot3_blas(o0, o1, o2, R[0], R[3], R[6]) > 0.0) + 2 * (dot3_blas(o0, o1, o2, R[1], R[4], R[7]) > 0.0) +
           4 * (dot3_blas(o0, o1, o2, R[2], R[5], R[8]) > 0.0);
}

// Fast SIFT-Rank bin of one voxel for one frame.  Each octant bit is taken
// from the fp32 rotated component when it clears its error bound (<= ~5 u32 of
// the L1 norm; bound 1e-6), otherwise from the reference's fp64 FMA chain
// (out of line, so the common path issues no fp64 at all): offset components
// need only the integer offset and R (offsets on lines / planes through the
// centre give exact zeros for axes with zero coordinates), gradient
// components need the exact fp64 gradient (rare).
//
// Rc holds each frame column j = (R[0][j], R[1][j], R[2][j]) as fp32 pairs
// (cx, cx, cy, cy), (cz, cz, -, -) in shared memory, read with volatile vector
// loads per use: the compiler would otherwise hoist 9 x F rotation floats into
// registers for the whole walk and halve the resident warps of this
// latency-bound loop.  The offset and gradient components of one column are
// evaluated together with packed fp32x2 multiply / FMA (same per-lane
// rounding as the scalar chain fmaf(z, cz, fmaf(y, cy, x * cx))).
constexpr int kRcPerFrame = 6;  // float4 slots per frame
#ifndef VK_SR_PACKED
#define VK_SR_PACKED 1
#endif
#ifndef VK_SR_SIGNBITS
#define VK_SR_SIGNBITS 1
#endif
#ifndef VK_SR_ZERO_RULE
#define VK_SR_ZERO_RULE 0  // measured slower (extra per-frame work outweighs the avoided fallbacks)
#endif

VK_D void lds_col(const float4* p, float2& xx, float2& yy, float2& zz, int& zmask) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(xx.x), "=f"(xx.y), "=f"(yy.x), "=f"(yy.y)
                 : "r"(a));
#if VK_SR_ZERO_RULE
    float zm, pad;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(zz.x), "=f"(zz.y), "=f"(zm), "=f"(pad)
                 : "r"(a + 16u));
    zmask = __float_as_int(zm);
#else
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(zz.x), "=f"(zz.y) : "r"(a + 16u));
    zmask = 0;
#endif
}

// Bits k of the components that are exactly nonzero.
VK_D int nonzero_bits(float a, float b, float c) { return (a != 0.f) | ((b != 0.f) << 1) | ((c != 0.f) << 2); }

VK_D int sr_bin_fast(int ox, int oy, int oz, float gx, float gy, float gz, const double* R, const float4* Rc,
                     const float* data, int nx, int ny, int nz, int x, int y, int z) {
    const float fx = (float)ox, fy = (float)oy, fz = (float)oz;
    const float eo = 1.0e-6f * (fabsf(fx) + fabsf(fy) + fabsf(fz));
    const float eg = 1.0e-6f * (fabsf(gx) + fabsf(gy) + fabsf(gz)) + 1.0e-40f;
    const float2 vx = make_float2(fx, gx), vy = make_float2(fy, gy), vz = make_float2(fz, gz);
    int sp = 0, og = 0;
    unsigned sneg = 0u, gneg = 0u;
    bool osure = true, gsure = true;
#if VK_SR_ZERO_RULE
    // exact-zero rule: when every nonzero component of the offset (gradient)
    // meets an exactly-zero fp64 entry of column j, both our chain and the
    // reference's give +-0, i.e. bit 0, whatever the bound test says
    const int nzo = nonzero_bits(fx, fy, fz), nzg = nonzero_bits(gx, gy, gz);
#endif
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        float2 cxx, cyy, czz;
        int zmask;
        lds_col(Rc + 2 * j, cxx, cyy, czz, zmask);
#if VK_SR_PACKED
        const float2 t = __ffma2_rn(vz, czz, __ffma2_rn(vy, cyy, __fmul2_rn(vx, cxx)));  // (r_j, g_j)
#else
        const float2 t = make_float2(fmaf(fz, czz.x, fmaf(fy, cyy.x, fx * cxx.x)),
                                     fmaf(gz, czz.x, fmaf(gy, cyy.x, gx * cxx.x)));
#endif
#if VK_SR_SIGNBITS
        // bit j = (t > 0): wherever the bound test passes t != 0, so it is the inverted sign bit
        sneg |= (__float_as_uint(t.x) >> 31) << j;
        gneg |= (__float_as_uint(t.y) >> 31) << j;
#else
        sp |= (int)(t.x > 0.f) << j;
        og |= (int)(t.y > 0.f) << j;
#endif
#if VK_SR_ZERO_RULE
        osure = osure && (fabsf(t.x) > eo || (nzo & ~zmask) == 0);
        gsure = gsure && (fabsf(t.y) > eg || (nzg & ~zmask) == 0);
#else
        osure = osure && fabsf(t.x) > eo;
        gsure = gsure && fabsf(t.y) > eg;
#endif
    }
#if VK_SR_SIGNBITS
    sp = (int)(~sneg & 7u);
    og = (int)(~gneg & 7u);
#endif
    if (!osure) sp = sr_obits_exact(ox, oy, oz, R);
    if (!gsure) og = sr_gbits_exact(data, nx, ny, nz, x, y, z, R);
    return 8 * sp + og;
}

// sr_bin_fast without the fallbacks: the fp32 bin and which halves are
// certain (bit 0: offset octant, bit 1: gradient octant).
VK_D int sr_bin_try(int ox, int oy, int oz, float gx, float gy, float gz, const float4* Rc, int& sure) {
    const float fx = (float)ox, fy = (float)oy, fz = (float)oz;
    const float eo = 1.0e-6f * (fabsf(fx) + fabsf(fy) + fabsf(fz));
    const float eg = 1.0e-6f * (fabsf(gx) + fabsf(gy) + fabsf(gz)) + 1.0e-40f;
    const float2 vx = make_float2(fx, gx), vy = make_float2(fy, gy), vz = make_float2(fz, gz);
    unsigned sneg = 0u, gneg = 0u;
    bool osure = true, gsure = true;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        float2 cxx, cyy, czz;
        int zm;
        lds_col(Rc + 2 * j, cxx, cyy, czz, zm);
        const float2 t = __ffma2_rn(vz, czz, __ffma2_rn(vy, cyy, __fmul2_rn(vx, cxx)));  // (r_j, g_j)
        sneg |= (__float_as_uint(t.x) >> 31) << j;
        gneg |= (__float_as_uint(t.y) >> 31) << j;
        osure = osure && fabsf(t.x) > eo;
        gsure = gsure && fabsf(t.y) > eg;
    }
    sure = (int)osure | ((int)gsure << 1);
    return 8 * (int)(~sneg & 7u) + (int)(~gneg & 7u);
}

// Fast walk of one keypoint's ball for NF frames; returns the number of
// in-volume ball voxels seen by this thread.  INTERIOR: the whole ball and its
// gradient stencil lie inside the volume (no bounds tests, no one-sided
// differences).  With a precomputed gradient volume (g4 != null) each visit is
// one float4 load.
template <int NF, bool INTERIOR>
VK_D int sr_walk(const vk_kp& kp, const vk_level& L, const float* data, const float4* g4, const vk_ball& ball,
                 const int* __restrict__ ball_offsets, const double* Rs, const float4* Rc, double* hist, int F) {
    const int tid = threadIdx.x;
    const int step = blockDim.x;
    const unsigned plane = (unsigned)L.nx * (unsigned)L.ny;
    int cnt = 0;
    hist = vote_copy(hist);
    int pn = tid < ball.count ? __ldg(ball_offsets + ball.zstart + tid) : 0;
    for (int base = 0; base < ball.count; base += step) {
        const int j = base + tid;
        const int p = pn;
        if (j + step < ball.count) pn = __ldg(ball_offsets + ball.zstart + j + step);
        bool has = false;
        int ox = 0, oy = 0, oz = 0, x = 0, y = 0, z = 0;
        float gx = 0.f, gy = 0.f, gz = 0.f, mag = 0.f;
        if (j < ball.count) {
            ox = unpack_off(p, 0);
            oy = unpack_off(p, 1);
            oz = unpack_off(p, 2);
            x = kp.ix + ox;
            y = kp.iy + oy;
            z = kp.iz + oz;
            if (INTERIOR || (x >= 0 && y >= 0 && z >= 0 && x < L.nx && y < L.ny && z < L.nz)) {
                ++cnt;
                const unsigned c = ((unsigned)z * (unsigned)L.ny + (unsigned)y) * (unsigned)L.nx + (unsigned)x;
                if (g4) {
                    const float4 q = __ldg(g4 + c);
                    gx = q.x;
                    gy = q.y;
                    gz = q.z;
                    mag = q.w;
                    has = mag > 0.f;  // gradient_volume_kernel: |g| >= 2^-149 exactly when the fp64 g != 0
                } else {
                    prefetch_plane_ahead(data, L.nx, L.ny, L.nz, x, y, z, kPrefetchPlanes);
                    const Nb6 nb = INTERIOR ? load_nb6_interior(data, (unsigned)L.nx, plane, c)
                                            : load_nb6(data, L.nx, L.ny, L.nz, x, y, z);
                    grad32(nb, gx, gy, gz);
                    has = grad_nonzero(nb);  // zero vote: no bin changes
                    if (has) mag = nz_vote(norm3_f32(gx, gy, gz));
                }
            }
        }
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            if (f >= F) break;
            const int bin = has ? sr_bin_fast(ox, oy, oz, gx, gy, gz, Rs + 9 * f, Rc + kRcPerFrame * f, data, L.nx, L.ny, L.nz, x,
                                              y, z)
                                : -1;
            red_vote(hist + f * kHistFrame, bin, mag);
        }
    }
    return cnt;
}

// Interior walk with the six neighbour loads of the thread's next voxel issued
// before the current voxel's bins are computed (two voxels in flight per
// thread): the walk is bound by L1 hit latency, not by issue.
#ifndef VK_SR_DEFER
#define VK_SR_DEFER 1
#endif
// A deferred (voxel, frame) vote: exact octant bits where the fp32 ones were
// uncertain, then the vote.  e = (packed offset, f | fast bin << 2 | sure << 8, mag bits).
VK_D void sr_resolve(int4 e, const vk_kp& kp, const vk_level& L, const float* data, const double* Rs,
                     double* hist) {
    const int ox = unpack_off(e.x, 0), oy = unpack_off(e.x, 1), oz = unpack_off(e.x, 2);
    const int f = e.y & 3, bin = (e.y >> 2) & 63, sure = (e.y >> 8) & 3;
    const int sp = (sure & 1) ? (bin >> 3) : sr_obits_exact(ox, oy, oz, Rs + 9 * f);
    const int og = (sure & 2) ? (bin & 7) : sr_gbits_exact(data, L.nx, L.ny, L.nz, kp.ix + ox, kp.iy + oy, kp.iz + oz,
                                                           Rs + 9 * f);
    red_vote(hist + f * kHistFrame, 8 * sp + og, __int_as_float(e.z));
}
#ifndef VK_SR_PIPE_PREFETCH
#define VK_SR_PIPE_PREFETCH 1  // L1 prefetch kPrefetchPlanes planes ahead in the pipelined interior walk
#endif
#ifndef VK_SR_X_LATE
#define VK_SR_X_LATE 0  // 1: next voxel's x loads issued after the frames (no spill of them; measured 1.5% slower: exposed latency)
#endif
#ifndef VK_SR_DEPTH
#define VK_SR_DEPTH 2  // voxels in flight per thread (sr_walk_pipe)
#endif
constexpr int kSrQueue = 32 + 4 * 32;  // per-warp deferred (voxel, frame) entries: flush at >= 32, one step adds <= 128

template <int NF, bool INTERIOR>
VK_D int sr_walk_pipe(const vk_kp& kp, const vk_level& L, const float* data, const vk_ball& ball,
                      const int* __restrict__ ball_offsets, const double* Rs, const float4* Rc, double* hist, int F,
                      int4* queue, int* qcount) {
    const int tid = threadIdx.x;
    const int step = blockDim.x;
    const int nx = L.nx, plane = L.nx * L.ny;
    const int kc = (kp.iz * L.ny + kp.iy) * nx + kp.ix;
    const int zpf = L.nz - kPrefetchPlanes - kp.iz;  // prefetch plane exists while oz < zpf
    const int* offs = ball_offsets + ball.zstart;
    hist = vote_copy(hist);
    auto issue = [&](int pk, Nb6& n, bool with_x) {
        const int ox = unpack_off(pk, 0), oy = unpack_off(pk, 1), oz = unpack_off(pk, 2);
        if (INTERIOR) {
            const int c = kc + oz * plane + oy * nx + ox;
#if VK_SR_PIPE_PREFETCH
            if (oz < zpf) asm volatile("prefetch.global.L1 [%0];" ::"l"(data + c + kPrefetchPlanes * plane));
#endif
            if (with_x) {
                n = load_nb6_interior(data, (unsigned)nx, (unsigned)plane, (unsigned)c);
            } else {  // x neighbours issued after the current voxel's frames (VK_SR_X_LATE)
                n.yh = __ldg(data + ((unsigned)c + (unsigned)nx));
                n.yl = __ldg(data + ((unsigned)c - (unsigned)nx));
                n.zh = __ldg(data + ((unsigned)c + (unsigned)plane));
                n.zl = __ldg(data + ((unsigned)c - (unsigned)plane));
            }
        } else {
            // branch-free clamped loads (the centre clamped into the volume too: values of
            // outside voxels are never used); the scales are recomputed at use, so a ring slot
            // carries only the six values
            const int x = clampi(kp.ix + ox, 0, L.nx - 1), y = clampi(kp.iy + oy, 0, L.ny - 1),
                      z = clampi(kp.iz + oz, 0, L.nz - 1);
            const unsigned c = ((unsigned)z * (unsigned)L.ny + (unsigned)y) * (unsigned)L.nx + (unsigned)x;
            const unsigned pl = (unsigned)L.nx * (unsigned)L.ny;
            n.xh = __ldg(data + (c + (x < L.nx - 1)));
            n.xl = __ldg(data + (c - (x > 0)));
            n.yh = __ldg(data + (c + (y < L.ny - 1 ? (unsigned)L.nx : 0u)));
            n.yl = __ldg(data + (c - (y > 0 ? (unsigned)L.nx : 0u)));
            n.zh = __ldg(data + (c + (z < L.nz - 1 ? pl : 0u)));
            n.zl = __ldg(data + (c - (z > 0 ? pl : 0u)));
        }
    };
    // ring: voxel j + d * step has its neighbours issued (d < D - 1) and its
    // packed offset loaded D - 1 steps ahead of use
    constexpr int D = VK_SR_DEPTH;
    // x neighbours of the next voxel issued late (after this voxel's frames) in the interior walk: at the
    // 80-register cap the compiler otherwise spilled those two in-flight loads, waiting on them at the store
    constexpr bool kXLate = VK_SR_X_LATE && INTERIOR && D == 2;
    int pk[D];
    Nb6 nb[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const int jj = tid + d * step;
        pk[d] = jj < ball.count ? __ldg(offs + jj) : 0;
        if (d < D - 1 && jj < ball.count) issue(pk[d], nb[d], true);
    }
    int cnt = 0;
    for (int base = 0; base < ball.count; base += step) {
        const int j = base + tid;
        const int pc = pk[0];
        Nb6 cur0 = nb[0];
        cur0.sx = cur0.sy = cur0.sz = 0.5f;
#pragma unroll
        for (int d = 0; d + 1 < D; ++d) {
            pk[d] = pk[d + 1];
            nb[d] = nb[d + 1];
        }
        if (j + (D - 1) * step < ball.count) {
            issue(pk[D - 2], nb[D - 2], !kXLate);
            if (j + D * step < ball.count) pk[D - 1] = __ldg(offs + j + D * step);
        }
        bool in = j < ball.count;
        Nb6 cur = cur0;
        if (!INTERIOR && in) {
            const int x = kp.ix + unpack_off(pc, 0), y = kp.iy + unpack_off(pc, 1), z = kp.iz + unpack_off(pc, 2);
            in = x >= 0 && y >= 0 && z >= 0 && x < L.nx && y < L.ny && z < L.nz;
            cur.sx = (x > 0 && x < L.nx - 1) ? 0.5f : 1.0f;
            cur.sy = (y > 0 && y < L.ny - 1) ? 0.5f : 1.0f;
            cur.sz = (z > 0 && z < L.nz - 1) ? 0.5f : 1.0f;
        }
        if (in) {
            ++cnt;
            float gx, gy, gz;
            grad32(cur, gx, gy, gz);
            if (grad_nonzero(cur)) {  // zero vote: no bin changes
                const float mag = nz_vote(norm3_f32(gx, gy, gz));
                const int ox = unpack_off(pc, 0), oy = unpack_off(pc, 1), oz = unpack_off(pc, 2);
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    if (f >= F) break;
#if VK_SR_DEFER
                    // uncertain octants (~1.5% of visit-frames) are deferred: resolved in place they
                    // would stall the whole warp in ~40% of its steps
                    int sure;
                    const int bin = sr_bin_try(ox, oy, oz, gx, gy, gz, Rc + kRcPerFrame * f, sure);
                    if (sure == 3) {
                        red_vote(hist + f * kHistFrame, bin, mag);
                    } else {
                        const int pos = atomicAdd(qcount, 1);
                        queue[pos] = make_int4(pc, f | (bin << 2) | (sure << 8), __float_as_int(mag), 0);
                    }
#else
                    const int bin = sr_bin_fast(ox, oy, oz, gx, gy, gz, Rs + 9 * f, Rc + kRcPerFrame * f, data, L.nx,
                                                L.ny, L.nz, kp.ix + ox, kp.iy + oy, kp.iz + oz);
                    red_vote(hist + f * kHistFrame, bin, mag);
#endif
                }
            }
        }
        if (kXLate && j + step < ball.count) {
            const int p2 = pk[0];  // the next voxel (D == 2: shifted into slot 0 above)
            const unsigned c = (unsigned)(kc + unpack_off(p2, 2) * plane + unpack_off(p2, 1) * nx + unpack_off(p2, 0));
            nb[0].xh = __ldg(data + (c + 1u));
            nb[0].xl = __ldg(data + (c - 1u));
        }
#if VK_SR_DEFER
        __syncwarp();
        int qn = *reinterpret_cast<volatile int*>(qcount);
        if (qn >= 32) {
            do {
                sr_resolve(queue[qn - 32 + (tid & 31)], kp, L, data, Rs, hist);
                qn -= 32;
            } while (qn >= 32);
            __syncwarp();
            if ((tid & 31) == 0) *qcount = qn;
            __syncwarp();
        }
#endif
    }
#if VK_SR_DEFER
    __syncwarp();
    const int qn = *reinterpret_cast<volatile int*>(qcount);
    if ((tid & 31) < qn) sr_resolve(queue[tid & 31], kp, L, data, Rs, hist);
    __syncwarp();
    if ((tid & 31) == 0) *qcount = 0;
    __syncwarp();
#endif
    return cnt;
}

// Interior walk with the neighbour gathers in flight in SHARED memory instead
// of registers (VK_SR_ASYNC): each voxel's six neighbours are copied by
// cp.async (LDGSTS, L1-allocating) into the thread's slot of a per-CTA ring,
// VK_SR_ADEPTH voxels ahead, and read back with conflict-free LDS once their
// group has landed.  In-flight loads then cost no registers (the register
// pipeline above spills two of its six at the 80-register cap and so waits on
// them), and the depth is free.
#ifndef VK_SR_ASYNC
#define VK_SR_ASYNC 0
#endif
#ifndef VK_SR_ADEPTH
#define VK_SR_ADEPTH 3
#endif
constexpr int kSrRingFloats = VK_SR_ASYNC ? VK_SR_ADEPTH * 6 * kSrThreads : 1;

template <int NF>
VK_D int sr_walk_async(const vk_kp& kp, const vk_level& L, const float* data, const vk_ball& ball,
                       const int* __restrict__ ball_offsets, const double* Rs, const float4* Rc, double* hist,
                       int F, int4* queue, int* qcount, float* ring) {
    static_assert(VK_SR_DEFER, "the shared-memory pipelined walk defers uncertain octants");
    const int tid = threadIdx.x;
    const int step = blockDim.x;
    const int nx = L.nx, plane = L.nx * L.ny;
    const int kc = (kp.iz * L.ny + kp.iy) * nx + kp.ix;
    const int zpf = L.nz - kPrefetchPlanes - kp.iz;
    const int* offs = ball_offsets + ball.zstart;
    hist = vote_copy(hist);
    constexpr int D = VK_SR_ADEPTH;
    float* mine = ring + tid;  // slot s, value k at mine[(6 s + k) * kSrThreads]
    auto issue = [&](int pk, int slot) {
        const int ox = unpack_off(pk, 0), oy = unpack_off(pk, 1), oz = unpack_off(pk, 2);
        const unsigned c = (unsigned)(kc + oz * plane + oy * nx + ox);
#if VK_SR_PIPE_PREFETCH
        if (oz < zpf) asm volatile("prefetch.global.L1 [%0];" ::"l"(data + c + kPrefetchPlanes * plane));
#endif
        float* d = mine + 6 * slot * kSrThreads;
        cp_async4(d, data + (c + 1u));
        cp_async4(d + kSrThreads, data + (c - 1u));
        cp_async4(d + 2 * kSrThreads, data + (c + (unsigned)nx));
        cp_async4(d + 3 * kSrThreads, data + (c - (unsigned)nx));
        cp_async4(d + 4 * kSrThreads, data + (c + (unsigned)plane));
        cp_async4(d + 5 * kSrThreads, data + (c - (unsigned)plane));
    };
    // packed offsets of voxels j .. j + (D - 1) step: pk[d]; groups in flight for j .. j + (D - 2) step
    int pk[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const int jj = tid + d * step;
        pk[d] = jj < ball.count ? __ldg(offs + jj) : 0;
        if (d < D - 1) {
            if (jj < ball.count) issue(pk[d], d);
            cp_async_commit();
        }
    }
    int cnt = 0, slot = 0;
    for (int base = 0; base < ball.count; base += step) {
        const int j = base + tid;
        const int pc = pk[0];
#pragma unroll
        for (int d = 0; d + 1 < D; ++d) pk[d] = pk[d + 1];
        {
            int ns = slot + (D - 1);
            if (ns >= D) ns -= D;
            if (j + (D - 1) * step < ball.count) {
                issue(pk[D - 2], ns);
                if (j + D * step < ball.count) pk[D - 1] = __ldg(offs + j + D * step);
            }
            cp_async_commit();
        }
        cp_async_wait<D - 1>();  // this voxel's group has landed
        if (j < ball.count) {
            ++cnt;
            const float* d = mine + 6 * slot * kSrThreads;
            Nb6 cur;
            cur.xh = d[0];
            cur.xl = d[kSrThreads];
            cur.yh = d[2 * kSrThreads];
            cur.yl = d[3 * kSrThreads];
            cur.zh = d[4 * kSrThreads];
            cur.zl = d[5 * kSrThreads];
            cur.sx = cur.sy = cur.sz = 0.5f;
            float gx, gy, gz;
            grad32(cur, gx, gy, gz);
            if (grad_nonzero(cur)) {
                const float mag = nz_vote(norm3_f32(gx, gy, gz));
                const int ox = unpack_off(pc, 0), oy = unpack_off(pc, 1), oz = unpack_off(pc, 2);
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    if (f >= F) break;
                    int sure;
                    const int bin = sr_bin_try(ox, oy, oz, gx, gy, gz, Rc + kRcPerFrame * f, sure);
                    if (sure == 3) {
                        red_vote(hist + f * kHistFrame, bin, mag);
                    } else {
                        const int pos = atomicAdd(qcount, 1);
                        queue[pos] = make_int4(pc, f | (bin << 2) | (sure << 8), __float_as_int(mag), 0);
                    }
                }
            }
        }
        if (++slot == D) slot = 0;
        __syncwarp();
        int qn = *reinterpret_cast<volatile int*>(qcount);
        if (qn >= 32) {
            do {
                sr_resolve(queue[qn - 32 + (tid & 31)], kp, L, data, Rs, hist);
                qn -= 32;
            } while (qn >= 32);
            __syncwarp();
            if ((tid & 31) == 0) *qcount = qn;
            __syncwarp();
        }
    }
    cp_async_wait<0>();
    __syncwarp();
    const int qn = *reinterpret_cast<volatile int*>(qcount);
    if ((tid & 31) < qn) sr_resolve(queue[tid & 31], kp, L, data, Rs, hist);
    __syncwarp();
    if ((tid & 31) == 0) *qcount = 0;
    __syncwarp();
    return cnt;
}

#ifndef VK_SR_PIPE
#define VK_SR_PIPE 1
#endif
#ifndef VK_SR_PIPE_BORDER
#define VK_SR_PIPE_BORDER 0  // border-crossing balls pipelined too in the all-keypoints kernel (register pressure)
#endif
// PIPE_BORDER: also pipeline border-crossing balls (the border-only launch).
template <bool INTERIOR, bool PIPE_BORDER = (VK_SR_PIPE_BORDER != 0)>
VK_D int sr_walk_frames(const vk_kp& kp, const vk_level& L, const float* data, const float4* g4, const vk_ball& ball,
                        const int* __restrict__ ball_offsets, const double* Rs, const float4* Rc, double* hist,
                        int F, int4* queue, int* qcount, float* ring = nullptr) {
    if (VK_SR_ASYNC && INTERIOR && ring != nullptr && !g4 && F <= 4) {
        switch (F) {
            case 1: return sr_walk_async<1>(kp, L, data, ball, ball_offsets, Rs, Rc, hist, F, queue, qcount, ring);
            case 2: return sr_walk_async<2>(kp, L, data, ball, ball_offsets, Rs, Rc, hist, F, queue, qcount, ring);
            case 3: return sr_walk_async<3>(kp, L, data, ball, ball_offsets, Rs, Rc, hist, F, queue, qcount, ring);
            default: return sr_walk_async<4>(kp, L, data, ball, ball_offsets, Rs, Rc, hist, F, queue, qcount, ring);
        }
    }
    if (VK_SR_PIPE && (INTERIOR || PIPE_BORDER) && !g4 && F <= 4) {
        switch (F) {
            case 1: return sr_walk_pipe<1, INTERIOR>(kp, L, data, ball, ball_offsets, Rs, Rc, hist, F, queue, qcount);
            case 2: return sr_walk_pipe<2, INTERIOR>(kp, L, data, ball, ball_offsets, Rs, Rc, hist, F, queue, qcount);
            case 3: return sr_walk_pipe<3, INTERIOR>(kp, L, data, ball, ball_offsets, Rs, Rc, hist, F, queue, qcount);
            default: return sr_walk_pipe<4, INTERIOR>(kp, L, data, ball, ball_offsets, Rs, Rc, hist, F, queue, qcount);
        }
    }
    switch (F) {
        case 1: return sr_walk<1, INTERIOR>(kp, L, data, g4, ball, ball_offsets, Rs, Rc, hist, F);
        case 2: return sr_walk<2, INTERIOR>(kp, L, data, g4, ball, ball_offsets, Rs, Rc, hist, F);
        case 3: return sr_walk<3, INTERIOR>(kp, L, data, g4, ball, ball_offsets, Rs, Rc, hist, F);
        case 4: return sr_walk<4, INTERIOR>(kp, L, data, g4, ball, ball_offsets, Rs, Rc, hist, F);
        default: {  // > 4 frames: two passes of up to 4 frames
            const int cnt = sr_walk<4, INTERIOR>(kp, L, data, g4, ball, ball_offsets, Rs, Rc, hist, 4);
            sr_walk<4, INTERIOR>(kp, L, data, g4, ball, ball_offsets, Rs + 36, Rc + 4 * kRcPerFrame, hist + 4 * kHistFrame, F - 4);
            return cnt;
        }
    }
}

// Stable ascending ranks of 64 values: rank_b = #{j : w_j < w_b or (w_j == w_b and j < b)}.
VK_D int stable_rank(const double* w, int n, int b) {
    const double wb = w[b];
    int r = 0;
    for (int j = 0; j < n; ++j) r += (w[j] < wb) || (w[j] == wb && j < b);
    return r;
}

// Exact reference order for one frame (out of line: keeps its fp64 register
// footprint out of the fast loop): chunked exact votes by all threads, then
// warp 0 adds them bin by bin in ball order (np.add.at).  Writes w[64].
static __device__ __noinline__ void sr_exact_frame(const float* data, const vk_level& L, const vk_kp& kp, const vk_ball& ball,
                                            const int* __restrict__ ball_offsets, const double* Rsm, double* w,
                                            int* xb, double* xv) {
    const int tid = threadIdx.x;
    double R[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) R[e] = Rsm[e];
    double acc0 = 0.0, acc1 = 0.0;
    for (int base = 0; base < ball.count; base += blockDim.x) {
        const int j = base + tid;
        double mg = 0.0;
        bool inside;
        int bin = -1;
        if (j < ball.count)
            bin = sr_vote(data, L.nx, L.ny, L.nz, kp.ix, kp.iy, kp.iz, __ldg(ball_offsets + ball.start + j), R, mg,
                          inside);
        xb[tid] = bin;
        xv[tid] = mg;
        __syncthreads();
        if (tid < 32) {
            const int m = min((int)blockDim.x, ball.count - base);
#pragma unroll 8
            for (int q = 0; q < m; ++q) {
                const int bs = xb[q];
                const double vs = xv[q];
                if (bs == tid) acc0 = dadd(acc0, vs);
                else if (bs == tid + 32) acc1 = dadd(acc1, vs);
            }
        }
        __syncthreads();
    }
    if (tid < 32) {
        w[tid] = acc0;
        w[tid + 32] = acc1;
    }
    __syncthreads();
}

// Cheap exact repair of an uncertain rank vector: only the bins in unc[]
// (members of an adjacent sorted pair whose separation was not certified) are
// re-accumulated, in the reference's ball order (x-major, np.add.at), with the
// reference's fp64 votes; every other bin keeps its fast sum.  The ranks of
// the repaired vector equal the reference's: a certified gap separates the
// true values as well, and inside an uncertain run the comparisons are now
// between exact values.  Bins come from the exact fast binning; a vote is
// computed in fp64 only for voxels in an uncertain bin, and the ordered sums
// take one thread a few additions per 256-voxel chunk (warp ballots of the
// contributing entries).
static __device__ __noinline__ void sr_exact_subset(const float* data, const vk_level& L, const vk_kp& kp,
                                             const vk_ball& ball, const int* __restrict__ ball_offsets,
                                             const double* Rsm, const float4* Rc, const int* unc, double* w, int* xb,
                                             double* xv, unsigned* wmask) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid < kSrBins && unc[tid]) w[tid] = 0.0;
    for (int base = 0; base < ball.count; base += blockDim.x) {
        const int j = base + tid;
        int bin = -1;
        double v = 0.0;
        if (j < ball.count) {
            const int p = __ldg(ball_offsets + ball.start + j);
            const int ox = unpack_off(p, 0), oy = unpack_off(p, 1), oz = unpack_off(p, 2);
            const int x = kp.ix + ox, y = kp.iy + oy, z = kp.iz + oz;
            if (x >= 0 && y >= 0 && z >= 0 && x < L.nx && y < L.ny && z < L.nz) {
                const Nb6 nb = load_nb6(data, L.nx, L.ny, L.nz, x, y, z);
                float gx, gy, gz;
                grad32(nb, gx, gy, gz);
                if (grad_nonzero(nb)) {
                    const int b = sr_bin_fast(ox, oy, oz, gx, gy, gz, Rsm, Rc, data, L.nx, L.ny, L.nz, x, y, z);
                    if (unc[b]) {
                        double x64, y64, z64;
                        grad64(nb, x64, y64, z64);
                        const double g0 = dot3_blas(x64, y64, z64, Rsm[0], Rsm[3], Rsm[6]);
                        const double g1 = dot3_blas(x64, y64, z64, Rsm[1], Rsm[4], Rsm[7]);
                        const double g2 = dot3_blas(x64, y64, z64, Rsm[2], Rsm[5], Rsm[8]);
                        v = norm3_numpy(g0, g1, g2);
                        bin = b;
                    }
                }
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, bin >= 0);
        if (lane == 0) wmask[wid] = m;
        xb[tid] = bin;
        xv[tid] = v;
        __syncthreads();
        if (tid == 0) {
            for (int g = 0; g < (int)(blockDim.x >> 5); ++g)
                for (unsigned t = wmask[g]; t; t &= t - 1) {
                    const int q = 32 * g + __ffs(t) - 1;
                    w[xb[q]] = dadd(w[xb[q]], xv[q]);
                }
        }
        __syncthreads();
    }
    __syncthreads();
}

}  // namespace vk
