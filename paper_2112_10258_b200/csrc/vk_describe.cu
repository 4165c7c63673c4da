// vk_describe.cu -- SIFT-Rank, BRIEF and RRIEF descriptors.
//
// Reference: descriptor.py:227-263 (sift_rank_descriptor), descriptor.py:77-83
// (rank_vector), descriptor.py:86-111 (extract_patch), descriptor.py:196-224
// (preblur_patch, _pair_samples, brief/rrief), descriptor.py:309-321 (packing).
//
// SIFT-Rank: one 256-thread CTA per keypoint (all of its frames at once),
// persistent.  The ball is walked in z-major order; each voxel's fp32
// gradient is computed once and voted (fp32 |g|, within kVoteRel + kVoteAbs of
// the reference's fp64 |R^T g|) into the spatial-octant x gradient-octant bin
// of every frame.  Octant bits come from fp32 rotated components where they
// clear their error bound; uncertain (voxel, frame) pairs are deferred to a
// per-warp queue and resolved with the reference's fp64 FMA chains.  Votes go
// into a per-CTA fp64 histogram in L2 by fire-and-forget reductions (any
// order).  The output is only the stable rank vector: if every adjacent pair
// of the sorted bins is separated by more than the bound between that sum and
// the reference's sequential np.add.at, the ranks are exact; otherwise only
// the bins of the unseparated pairs are re-accumulated in reference order
// with fp64 votes (sr_exact_subset).
//
// BRIEF / RRIEF: one CTA per frame.  The side^3 reoriented patch is sampled
// from the source volume (fp64 trilinear, cast to fp32) straight into shared
// memory, pre-blurred there with the same non-FMA separable blur as the
// pyramid, then the point pairs are sampled (fp64 trilinear on the fp32 patch)
// and turned into packed bits or stable ranks.
#include "vk_hood.cuh"

namespace vk {

#ifndef VK_SR_THREADS
#define VK_SR_THREADS 256
#endif
constexpr int kSrThreads = VK_SR_THREADS;
constexpr int kPrefetchPlanes = 3;  // z-plane lead of the L1 prefetch in the ball walk
constexpr int kSrBins = 64;
constexpr int kPatchThreads = 256;
constexpr int kMaxSide = 31;

struct PatchParams {
    double grid[kMaxSide];
    float taps[VK_MAX_TAPS];
};

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
__device__ __noinline__ int sr_bin_exact(int ox, int oy, int oz, double x64, double y64, double z64,
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
__device__ __forceinline__
#else
__device__ __noinline__
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
__device__ __forceinline__
#else
__device__ __noinline__
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
            red_vote(hist + f * kSrBins, bin, mag);
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
    red_vote(hist + f * kSrBins, 8 * sp + og, __int_as_float(e.z));
}
constexpr int kSrQueue = 32 + 4 * 32;  // per-warp deferred (voxel, frame) entries: flush at >= 32, one step adds <= 128

template <int NF>
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
    auto issue = [&](int pk, Nb6& n) {
        const int ox = unpack_off(pk, 0), oy = unpack_off(pk, 1), oz = unpack_off(pk, 2);
        const int c = kc + oz * plane + oy * nx + ox;
        if (oz < zpf) asm volatile("prefetch.global.L1 [%0];" ::"l"(data + c + kPrefetchPlanes * plane));
        n = load_nb6_interior(data, (unsigned)nx, (unsigned)plane, (unsigned)c);
    };
    int p = tid < ball.count ? __ldg(offs + tid) : 0;
    Nb6 nb{};
    if (tid < ball.count) issue(p, nb);
    int pn = tid + step < ball.count ? __ldg(offs + tid + step) : 0;
    int cnt = 0;
    for (int base = 0; base < ball.count; base += step) {
        const int j = base + tid;
        const int pc = p;
        const Nb6 cur = nb;
        p = pn;
        if (j + step < ball.count) {
            issue(p, nb);
            if (j + 2 * step < ball.count) pn = __ldg(offs + j + 2 * step);
        }
        if (j < ball.count) {
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
                        red_vote(hist + f * kSrBins, bin, mag);
                    } else {
                        const int pos = atomicAdd(qcount, 1);
                        queue[pos] = make_int4(pc, f | (bin << 2) | (sure << 8), __float_as_int(mag), 0);
                    }
#else
                    const int bin = sr_bin_fast(ox, oy, oz, gx, gy, gz, Rs + 9 * f, Rc + kRcPerFrame * f, data, L.nx,
                                                L.ny, L.nz, kp.ix + ox, kp.iy + oy, kp.iz + oz);
                    red_vote(hist + f * kSrBins, bin, mag);
#endif
                }
            }
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

template <bool INTERIOR>
VK_D int sr_walk_frames(const vk_kp& kp, const vk_level& L, const float* data, const float4* g4, const vk_ball& ball,
                        const int* __restrict__ ball_offsets, const double* Rs, const float4* Rc, double* hist,
                        int F, int4* queue, int* qcount) {
#ifndef VK_SR_PIPE
#define VK_SR_PIPE 1
#endif
    if (VK_SR_PIPE && INTERIOR && !g4 && F <= 4) {
        switch (F) {
            case 1: return sr_walk_pipe<1>(kp, L, data, ball, ball_offsets, Rs, Rc, hist, F, queue, qcount);
            case 2: return sr_walk_pipe<2>(kp, L, data, ball, ball_offsets, Rs, Rc, hist, F, queue, qcount);
            case 3: return sr_walk_pipe<3>(kp, L, data, ball, ball_offsets, Rs, Rc, hist, F, queue, qcount);
            default: return sr_walk_pipe<4>(kp, L, data, ball, ball_offsets, Rs, Rc, hist, F, queue, qcount);
        }
    }
    switch (F) {
        case 1: return sr_walk<1, INTERIOR>(kp, L, data, g4, ball, ball_offsets, Rs, Rc, hist, F);
        case 2: return sr_walk<2, INTERIOR>(kp, L, data, g4, ball, ball_offsets, Rs, Rc, hist, F);
        case 3: return sr_walk<3, INTERIOR>(kp, L, data, g4, ball, ball_offsets, Rs, Rc, hist, F);
        case 4: return sr_walk<4, INTERIOR>(kp, L, data, g4, ball, ball_offsets, Rs, Rc, hist, F);
        default: {  // > 4 frames: two passes of up to 4 frames
            const int cnt = sr_walk<4, INTERIOR>(kp, L, data, g4, ball, ball_offsets, Rs, Rc, hist, 4);
            sr_walk<4, INTERIOR>(kp, L, data, g4, ball, ball_offsets, Rs + 36, Rc + 4 * kRcPerFrame, hist + 4 * kSrBins, F - 4);
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
__device__ __noinline__ void sr_exact_frame(const float* data, const vk_level& L, const vk_kp& kp, const vk_ball& ball,
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
__device__ __noinline__ void sr_exact_subset(const float* data, const vk_level& L, const vk_kp& kp,
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

// One CTA per work item = one keypoint and its F frames (contiguous in the
// frame list).  The ball is walked in z-major order (coalesced gathers);
// each voxel's gradient is computed once and voted into all F frames.
#ifndef VK_SR_MIN_BLOCKS
#define VK_SR_MIN_BLOCKS 3
#endif
__global__ void __launch_bounds__(kSrThreads, VK_SR_MIN_BLOCKS)
siftrank_kernel(const vk_frame* __restrict__ frames, const double* __restrict__ rot,
                const int* __restrict__ item_first, const int* __restrict__ item_count,
                const int* __restrict__ n_items_dev, int n_items_max, const vk_kp* __restrict__ kps,
                const vk_level* __restrict__ levels, const vk_ball* __restrict__ balls,
                const int* __restrict__ ball_offsets, int max_f,
                uint8_t* __restrict__ out, int exact_only, int* __restrict__ stats,
                const vk_gradlevel* __restrict__ grads, double* __restrict__ work) {
    double* hist = work + (long long)blockIdx.x * kAccumSlot;  // [F][64] fp64, L2-resident
    __shared__ double w[kSrBins];
    __shared__ double Rs[VK_MAX_FRAMES * 9];
    __shared__ float4 Rc[VK_MAX_FRAMES * kRcPerFrame];
    __shared__ int xb[kSrThreads];
    __shared__ double xv[kSrThreads];
    __shared__ int n_inside;
    __shared__ int unc[kSrBins];
    __shared__ double w4[kSrThreads / kSrBins][kSrBins];
    __shared__ int order4[kSrThreads / kSrBins][kSrBins];
    __shared__ int badf[kSrThreads / kSrBins];
    __shared__ int4 sq[kSrThreads / 32][kSrQueue];  // deferred uncertain votes, per warp
    __shared__ int sqn[kSrThreads / 32];
    __shared__ unsigned wmask[kSrThreads / 32];
    const int tid = threadIdx.x;
    const int n = n_items_dev ? min(*n_items_dev, n_items_max) : n_items_max;
    if (tid < kSrThreads / 32) sqn[tid] = 0;  // (first use is after the item's __syncthreads)
    for (int item = blockIdx.x; item < n; item += gridDim.x) {
        const int F = min(item_count[item], max_f);
        if (F <= 0) continue;
        const int first = item_first[item];
        const vk_kp kp = kps[frames[first].kp];
        const vk_level L = levels[kp.lvl];
        const float* data = L.base + (long long)kp.vol * L.vol_stride;
        const vk_ball ball = balls[kp.ball];
        __syncthreads();  // previous item done with the shared buffers
        for (int i = tid; i < F * 9; i += kSrThreads) {
            Rs[i] = rot[(long long)first * 9 + i];
        }
        __syncthreads();
        for (int i = tid; i < F * 3; i += kSrThreads) {
            const double* R = Rs + 9 * (i / 3);
            const int j = i % 3;
            const float cx = (float)R[j], cy = (float)R[3 + j], cz = (float)R[6 + j];
            const int zmask = (R[j] == 0.0) | ((R[3 + j] == 0.0) << 1) | ((R[6 + j] == 0.0) << 2);  // exact fp64 zeros
            Rc[(i / 3) * kRcPerFrame + 2 * j] = make_float4(cx, cx, cy, cy);
            Rc[(i / 3) * kRcPerFrame + 2 * j + 1] = make_float4(cz, cz, __int_as_float(zmask), 0.f);
        }
        zero_hist(hist, F * kSrBins);
        if (tid == 0) n_inside = 0;
        __syncthreads();
        int cnt = 0;
        const bool fast = !exact_only;
        if (fast) {
            // z-major ball walk: consecutive lanes take consecutive x -> coalesced gathers
            const float4* g4 = nullptr;
            if (grads) {
                const vk_gradlevel GL = grads[kp.lvl];
                if (GL.g4 && GL.kind == 0) g4 = reinterpret_cast<const float4*>(GL.g4) + (long long)kp.vol * GL.vol_stride;
            }
            if (ball_interior(kp.ix, kp.iy, kp.iz, ball.r, L.nx, L.ny, L.nz))
                cnt = sr_walk_frames<true>(kp, L, data, g4, ball, ball_offsets, Rs, Rc, hist, F, sq[tid >> 5],
                                           sqn + (tid >> 5));
            else
                cnt = sr_walk_frames<false>(kp, L, data, g4, ball, ball_offsets, Rs, Rc, hist, F, sq[tid >> 5],
                                            sqn + (tid >> 5));
        } else {
            for (int j = tid; j < ball.count; j += kSrThreads) {
                const int p = __ldg(ball_offsets + ball.start + j);
                const int x = kp.ix + unpack_off(p, 0), y = kp.iy + unpack_off(p, 1), z = kp.iz + unpack_off(p, 2);
                cnt += x >= 0 && y >= 0 && z >= 0 && x < L.nx && y < L.ny && z < L.nz;
            }
        }
        if (cnt) atomicAdd(&n_inside, cnt);
        __syncthreads();
        if (fast) {
            // all frames of the item at once, up to 4 per pass: thread (f, b) = (tid / 64, tid % 64)
            const double epsrel = 2.0 * (kVoteRel + gamma_k((double)n_inside + 64.0));
            const double epsabs = kVoteAbs * n_inside;
            const int fl = tid >> 6, b = tid & (kSrBins - 1);
            for (int f0 = 0; f0 < F; f0 += kSrThreads / kSrBins) {
                const int f = f0 + fl;
                const bool mine = f < F;
                if (mine) w4[fl][b] = read_hist(hist, f * kSrBins + b);
                if (tid < kSrThreads / kSrBins) badf[tid] = 0;
                __syncthreads();
                int myrank = 0;
                if (mine) {
                    myrank = stable_rank(w4[fl], kSrBins, b);
                    order4[fl][myrank] = b;
                }
                __syncthreads();
                // every adjacent pair of the sorted bins must be separated by more than
                // the bound between our summation and the reference's sequential one
                int bad = 0;
                if (mine && b + 1 < kSrBins) {
                    const double x = w4[fl][order4[fl][b]], y = w4[fl][order4[fl][b + 1]];
                    // exact empty-bin ties are order-independent: a fast bin is 0 exactly when
                    // no voxel with a nonzero fp64 gradient voted into it (grad_nonzero, nz_vote),
                    // i.e. exactly when the reference's bin is 0
                    if (!(x == 0.0 && y == 0.0)) {
                        const double xhi = x == 0.0 ? 0.0 : dadd(x, x * epsrel + epsabs);
                        const double ylo = dsub(y, y * epsrel + epsabs);
                        bad = !(xhi < ylo);
                    }
                }
                if (bad) badf[fl] = 1;
                if (__syncthreads_or(bad)) {
                    // rare: repair the uncertain frames one at a time (whole CTA)
                    for (int g = 0; g < kSrThreads / kSrBins && f0 + g < F; ++g) {
                        if (!badf[g]) continue;
                        if (tid == 0 && stats) atomicAdd(stats, 1);  // fallback counter (diagnostics)
                        if (tid < kSrBins) {
                            unc[tid] = 0;
                            w[tid] = w4[g][tid];
                        }
                        __syncthreads();
                        if (fl == g && bad) unc[order4[g][b]] = unc[order4[g][b + 1]] = 1;
                        __syncthreads();
                        sr_exact_subset(data, L, kp, ball, ball_offsets, Rs + 9 * (f0 + g), Rc + kRcPerFrame * (f0 + g),
                                        unc, w, xb, xv, wmask);
                        if (fl == g) myrank = stable_rank(w, kSrBins, b);
                        __syncthreads();
                    }
                }
                if (mine) out[(long long)(first + f) * kSrBins + b] = (uint8_t)myrank;
                __syncthreads();
            }
        } else {
            for (int f = 0; f < F; ++f) {
                sr_exact_frame(data, L, kp, ball, ball_offsets, Rs + 9 * f, w, xb, xv);
                if (tid < kSrBins) out[(long long)(first + f) * kSrBins + tid] = (uint8_t)stable_rank(w, kSrBins, tid);
                __syncthreads();
            }
        }
    }
}

__global__ void __launch_bounds__(kPatchThreads)
patch_kernel(int kind, const vk_frame* __restrict__ frames, const double* __restrict__ rot, const int* __restrict__ n_dev,
             int n_max, const vk_kp* __restrict__ kps, const double* __restrict__ pos, const double* __restrict__ sigma,
             const vk_level* __restrict__ source, int side, PatchParams pp, int radius,
             const double* __restrict__ pts, int npairs, uint8_t* __restrict__ bits_out, uint16_t* __restrict__ ranks_out,
             float* __restrict__ patch_out) {
    extern __shared__ float pbuf[];  // 2 x side^3 floats, then npairs doubles
    const int n3 = side * side * side;
    float* p0 = pbuf;
    float* p1 = pbuf + n3;
    double* diff = reinterpret_cast<double*>(pbuf + 2 * ((n3 + 1) & ~1));
    const int tid = threadIdx.x;
    const int n = n_dev ? min(*n_dev, n_max) : n_max;
    const vk_level S = source[0];
    const int s2 = side * side;
    for (int item = blockIdx.x; item < n; item += gridDim.x) {
        const vk_frame fr = frames[item];
        const vk_kp kp = kps[fr.kp];
        const float* data = S.base + (long long)kp.vol * S.vol_stride;
        const double c0 = pos[3 * fr.kp], c1 = pos[3 * fr.kp + 1], c2 = pos[3 * fr.kp + 2];
        const double sc = dmul(2.0, sigma[fr.kp]);  // PAIR_SUPPORT_RADIUS * kp.sigma
        double R[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) R[e] = __ldg(rot + (long long)item * 9 + e);
        // 1. reoriented patch from the source volume (descriptor.py:107-111)
        for (int i = tid; i < n3; i += kPatchThreads) {
            const int a = i / s2, bb = (i / side) % side, c = i % side;
            const double o0 = dmul(pp.grid[a], sc), o1 = dmul(pp.grid[bb], sc), o2 = dmul(pp.grid[c], sc);
            // offsets @ R.T: out[j] = sum_k o[k] R[j][k]
            const double px = dadd(c0, dot3_blas(o0, o1, o2, R[0], R[1], R[2]));
            const double py = dadd(c1, dot3_blas(o0, o1, o2, R[3], R[4], R[5]));
            const double pz = dadd(c2, dot3_blas(o0, o1, o2, R[6], R[7], R[8]));
            auto at = [&](int x, int y, int z) {
                return (double)__ldg(data + ((long long)z * S.ny + y) * S.nx + x);
            };
            p0[i] = (float)trilinear(at, S.nx, S.ny, S.nz, px, py, pz);
        }
        __syncthreads();
        // 2. pre-blur: axis 0 (slowest), axis 1, axis 2 with replicate borders
        float* cur = p0;
        if (radius > 0) {
            float* nxt = p1;
            for (int axis = 0; axis < 3; ++axis) {
                const int stride = axis == 0 ? s2 : (axis == 1 ? side : 1);
                for (int i = tid; i < n3; i += kPatchThreads) {
                    const int cidx = axis == 0 ? i / s2 : (axis == 1 ? (i / side) % side : i % side);
                    const float* base = cur + (i - cidx * stride);
                    float acc = fmul(pp.taps[0], base[clampi(cidx - radius, 0, side - 1) * stride]);
                    for (int t = 1; t <= 2 * radius; ++t)
                        acc = fadd(acc, fmul(pp.taps[t], base[clampi(cidx - radius + t, 0, side - 1) * stride]));
                    nxt[i] = acc;
                }
                __syncthreads();
                float* t = cur;
                cur = nxt;
                nxt = t;
            }
        }
        if (kind == 0) {  // the (pre-blurred) patch itself, [x][y][z] like Patch.data
            for (int i = tid; i < n3; i += kPatchThreads) patch_out[(long long)item * n3 + i] = cur[i];
            __syncthreads();
            continue;
        }
        // 3. pair samples (descriptor.py:205-212) and their differences
        for (int k = tid; k < npairs; k += kPatchThreads) {
            auto at = [&](int x, int y, int z) { return (double)cur[(x * side + y) * side + z]; };
            const double* q1 = pts + 3 * k;
            const double* q2 = pts + 3 * (npairs + k);
            const double sa = trilinear(at, side, side, side, q1[0], q1[1], q1[2]);
            const double sb = trilinear(at, side, side, side, q2[0], q2[1], q2[2]);
            diff[k] = dsub(sa, sb);
        }
        __syncthreads();
        if (kind == 1) {
            const int nbytes = (npairs + 7) / 8;
            for (int by = tid; by < nbytes; by += kPatchThreads) {
                unsigned v = 0;
                for (int t = 0; t < 8; ++t) {
                    const int k = by * 8 + t;
                    if (k < npairs && diff[k] > 0.0) v |= 0x80u >> t;
                }
                bits_out[(long long)item * nbytes + by] = (uint8_t)v;
            }
        } else {
            for (int k = tid; k < npairs; k += kPatchThreads) {
                const double dk = diff[k];
                int r = 0;
                for (int j = 0; j < npairs; ++j) r += (diff[j] < dk) || (diff[j] == dk && j < k);
                ranks_out[(long long)item * npairs + k] = (uint16_t)r;
            }
        }
        __syncthreads();
    }
}

}  // namespace vk

using namespace vk;

static int grid_for(int n, int per_sm) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return n < sms * per_sm ? n : sms * per_sm;
}

extern "C" int vk_describe_siftrank(const vk_frame* frames, const double* rot, const int* item_first,
                                    const int* item_count, const int* n_items_dev, int n_items_max, int max_f,
                                    const vk_kp* kps, const vk_level* levels, const vk_ball* balls,
                                    const int* ball_offsets, uint8_t* ranks_out,
                                    int exact_only, int* stats, const vk_gradlevel* grads, double* work,
                                    void* stream) {
    if (!frames || !rot || !item_first || !item_count || n_items_max < 0 || max_f < 1 || max_f > VK_MAX_FRAMES ||
        !kps || !levels || !balls || !ball_offsets || !ranks_out || !work) {
        set_error("vk_describe_siftrank: bad arguments");
        return VK_ERR_PARAMETER;
    }
    if (n_items_max == 0) return VK_OK;
    siftrank_kernel<<<accum_grid(siftrank_kernel, kSrThreads, n_items_max), kSrThreads, 0, as_stream(stream)>>>(
        frames, rot, item_first, item_count, n_items_dev, n_items_max, kps, levels, balls, ball_offsets, max_f,
        ranks_out, exact_only, stats, grads, work);
    count_launch();
    return cuda_status(cudaGetLastError(), "siftrank launch");
}

extern "C" int vk_describe_patch(int kind, const vk_frame* frames, const double* rot, const int* n_frames_dev,
                                 int n_frames_max, const vk_kp* kps, const double* pos, const double* sigma,
                                 const vk_level* source, int side, const double* grid_host, const float* taps_host,
                                 int radius, const double* pts, int npairs, uint8_t* bits_out, uint16_t* ranks_out,
                                 void* stream) {
    if ((kind != 1 && kind != 2) || !frames || !rot || n_frames_max < 0 || !kps || !pos || !sigma || !source ||
        side < 1 || side > kMaxSide || (side % 2) == 0 || !grid_host || radius < 0 || 2 * radius + 1 > VK_MAX_TAPS ||
        (radius > 0 && !taps_host) || !pts || npairs < 1 || npairs > VK_MAX_PAIRS || (kind == 1 && !bits_out) ||
        (kind == 2 && !ranks_out)) {
        set_error("vk_describe_patch: bad arguments (kind=%d side=%d npairs=%d)", kind, side, npairs);
        return VK_ERR_PARAMETER;
    }
    if (n_frames_max == 0) return VK_OK;
    PatchParams pp{};
    for (int i = 0; i < side; ++i) pp.grid[i] = grid_host[i];
    for (int i = 0; i < 2 * radius + 1 && radius > 0; ++i) pp.taps[i] = taps_host[i];
    const int n3 = side * side * side;
    const int smem = 2 * ((n3 + 1) & ~1) * 4 + npairs * 8;
    static int configured = 0;
    if (smem > 48 * 1024 && configured < smem) {
        cudaError_t e = cudaFuncSetAttribute(patch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return cuda_status(e, "patch attribute");
        configured = smem;
    }
    patch_kernel<<<grid_for(n_frames_max, 4), kPatchThreads, smem, as_stream(stream)>>>(
        kind, frames, rot, n_frames_dev, n_frames_max, kps, pos, sigma, source, side, pp, radius, pts, npairs, bits_out,
        ranks_out, nullptr);
    count_launch();
    return cuda_status(cudaGetLastError(), "patch launch");
}

extern "C" int vk_extract_patches(const vk_frame* frames, const double* rot, const int* n_frames_dev, int n_frames_max,
                                  const vk_kp* kps, const double* pos, const double* sigma, const vk_level* source,
                                  int side, const double* grid_host, const float* taps_host, int radius,
                                  float* patch_out, void* stream) {
    if (!frames || !rot || n_frames_max < 0 || !kps || !pos || !sigma || !source || side < 1 || side > kMaxSide ||
        (side % 2) == 0 || !grid_host || radius < 0 || 2 * radius + 1 > VK_MAX_TAPS || (radius > 0 && !taps_host) ||
        !patch_out) {
        set_error("vk_extract_patches: bad arguments (side=%d radius=%d)", side, radius);
        return VK_ERR_PARAMETER;
    }
    if (n_frames_max == 0) return VK_OK;
    PatchParams pp{};
    for (int i = 0; i < side; ++i) pp.grid[i] = grid_host[i];
    for (int i = 0; i < 2 * radius + 1 && radius > 0; ++i) pp.taps[i] = taps_host[i];
    const int n3 = side * side * side;
    const int smem = 2 * ((n3 + 1) & ~1) * 4;
    static int configured = 0;
    if (smem > 48 * 1024 && configured < smem) {
        cudaError_t e = cudaFuncSetAttribute(patch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return cuda_status(e, "patch attribute");
        configured = smem;
    }
    patch_kernel<<<grid_for(n_frames_max, 4), kPatchThreads, smem, as_stream(stream)>>>(
        0, frames, rot, n_frames_dev, n_frames_max, kps, pos, sigma, source, side, pp, radius, nullptr, 0, nullptr,
        nullptr, patch_out);
    count_launch();
    return cuda_status(cudaGetLastError(), "patch launch");
}
