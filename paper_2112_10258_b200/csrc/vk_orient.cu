// vk_orient.cu -- spherical gradient histograms and orientation frames.
//
// Reference: orient.py:89-125 (gradient_histogram), orient.py:128-168
// (dominant_orientations), pipeline.py:41-67 (assign_orientations).
//
// orient_kernel: one 256-thread CTA per keypoint, persistent over the keypoint
// list (the count lives in device memory so the whole pipeline can be
// graph-captured).  Fast path: the ball is walked in z-major order (coalesced
// gathers); each voxel's vote is the fp32 |g| x window (within kVoteRel +
// kVoteAbs of the reference's fp64 vote) and its bin the exact nearest
// icosphere direction (lookup table, boundary cells deferred to a per-warp
// queue and resolved by a screened fp32 argmax with an fp64 fallback).  Votes
// are added with fire-and-forget fp64 reductions into a per-CTA histogram in
// L2 (any order).  Every decision the frames depend on (the top of the weight
// order, the secondary_ratio threshold) is checked against a rigorous bound on
// the difference between that sum and the reference's sequential np.add.at;
// only the bins of an uncertain decision are re-accumulated in the reference's
// order with fp64 votes (ori_exact_subset).  Either way the frames are the
// reference's.
#include "vk_hood.cuh"
#include "vk_stage.cuh"

namespace vk {

#ifndef VK_ORI_THREADS
#define VK_ORI_THREADS 256
#endif
constexpr int kOriThreads = VK_ORI_THREADS;
#ifndef VK_ORI_PREFETCH
#define VK_ORI_PREFETCH 0  // z-plane lead of an L1 prefetch in the ball walk (0: none)
#endif

#ifndef VK_ORI_STAGED
#define VK_ORI_STAGED 0  // 1: interior balls walked from plane-staged shared memory (vk_stage.cuh); measured
                         // slower on B200 (2.20 vs 2.13 ms / 8 volumes: +23% instructions, barrier stalls)
#endif

constexpr int kOriQueue = 64;  // per-warp deferred entries of the fast walk (flush at >= 32)

struct OriShared {
    double xv[kOriThreads];
    int xb[kOriThreads];
    double dirs[VK_MAX_DIRS * 3];
    double w[VK_MAX_DIRS];
    int order[VK_MAX_DIRS];
    uint8_t ok[VK_MAX_DIRS * VK_MAX_DIRS];
    int unc[VK_MAX_DIRS];
    unsigned wmask[kOriThreads / 32];
    int2 queue[kOriThreads / 32][kOriQueue];  // deferred boundary-cell voxels of the fast walk (ori_walk)
    int n_inside;
    int exact;
    int repair;
};

// Nearest direction: first index of the maximum fp64 dot (np.argmax).
VK_D int nearest_dir(const double* dirs, int K, double gx, double gy, double gz) {
    int best = 0;
    double bv = dot3_blas(gx, gy, gz, dirs[0], dirs[1], dirs[2]);
    for (int k = 1; k < K; ++k) {
        double v = dot3_blas(gx, gy, gz, dirs[3 * k], dirs[3 * k + 1], dirs[3 * k + 2]);
        if (v > bv) { bv = v; best = k; }
    }
    return best;
}

// Exact vote of ball entry j (reference arithmetic, brute-force argmax), or
// bin -1 (outside / zero gradient).  Used by the reference-order path.
VK_D int ori_vote(const float* data, int nx, int ny, int nz, int cx, int cy, int cz, int packed,
                  const double* __restrict__ win, const double* dirs, int K, double& vote, bool& inside) {
    const int ox = unpack_off(packed, 0), oy = unpack_off(packed, 1), oz = unpack_off(packed, 2);
    const int x = cx + ox, y = cy + oy, z = cz + oz;
    inside = x >= 0 && y >= 0 && z >= 0 && x < nx && y < ny && z < nz;
    if (!inside) return -1;
    double gx, gy, gz;
    gradient_at(data, nx, ny, nz, x, y, z, gx, gy, gz);
    const double mag = norm3_numpy(gx, gy, gz);
    if (!(mag > 0.0)) return -1;
    vote = dmul(mag, __ldg(win + (ox * ox + oy * oy + oz * oz)));
    return nearest_dir(dirs, K, gx, gy, gz);
}

// Icosphere structure for the screened argmax.  The 12 icosahedron vertices
// are (0, +-1, +-phi), (+-1, +-phi, 0), (+-phi, 0, +-1) (normalised); for a
// gradient g the best vertex of each of the three groups follows from the
// signs of g and its dot is |gy| + phi|gz|, |gx| + phi|gy|, phi|gx| + |gz| (up
// to the common norm).  The nearest of all 42 directions is always the
// nearest vertex or one of its 5 edge midpoints (a midpoint's Voronoi cell lies
// in the union of its two endpoints' vertex cells; tests/test_host_logic.py),
// so: screen vertices analytically with a generous margin, score the
// surviving vertices + their midpoints with fp32 dots, and fall back to the
// reference's fp64 FMA-chain dots only when the fp32 winner is not separated
// by more than its error bound.  Ties keep the lowest index (np.argmax).
struct IcoT {
    int valid;
    int vert[12];  // vertex of construction order 6*a + 3*b + group (tables.icosphere_structure)
    int adj[12][5];
    int kind[12][5];  // the same midpoints by neighbour kind (fast argmax)
};

struct IcoSh {
    float4 cd[12 * 6];  // per vertex slot: the vertex and its 5 midpoints (fp32 xyz)
    int ci[12 * 6];     // their direction indices
    int fk[12 * 6];     // per vertex slot: the vertex, then its midpoints by kind
};

// Rare path (kept out of line so its fp64 work is never hoisted): exact
// reference dots over the candidates whose fp32 score is within the window.
__device__ __noinline__ int nearest_dir_ico_exact(const double* dirs, const IcoSh& ic, unsigned slots, float gx,
                                                  float gy, float gz, float floor32, double x64, double y64,
                                                  double z64) {
    double bv = -INFINITY;
    int bi = 1 << 30;
    for (unsigned t = slots; t; t &= t - 1) {
        const int v = __ffs(t) - 1;
        for (int c = 0; c < 6; ++c) {
            const float4 dd = ic.cd[6 * v + c];
            const int k = ic.ci[6 * v + c];
            if (fmaf(gz, dd.z, fmaf(gy, dd.y, gx * dd.x)) < floor32) continue;
            const double val = dot3_blas(x64, y64, z64, dirs[3 * k], dirs[3 * k + 1], dirs[3 * k + 2]);
            if (val > bv || (val == bv && k < bi)) {
                bv = val;
                bi = k;
            }
        }
    }
    return bi;
}

// Fast exact argmax for the common case: one icosahedron vertex clearly
// nearest (its group value leads the others by more than the screen margin and
// both of its signs are clear).  The nearest of the 42 directions is then the
// vertex or one of its 5 edge midpoints, and all of those scores follow from
// |g| components: in the winning group's axes (p, q, r) the vertex scores
// (|p| + phi|q|) / |V| and the midpoint with neighbour W scores
// (V.g + W.g) / (2 phi) with W.g in {phi|p| +- |r|, |q| +- phi|r|, phi|q| - |p|}.
// Each score is within ~3e-7 |g|_1 of the exact dot, so a winner clear of the
// runner-up by 2e-6 |g|_1 is the exact np.argmax; otherwise the caller falls
// back.  Returns -1 when the fast case does not apply or is not certain.
VK_D int nearest_dir_fast(const IcoSh& ic, float gx, float gy, float gz, float ax, float ay, float az, float l1,
                          float vA, float vB, float vC, float m) {
    constexpr float PHI = 1.6180339887498949f;
    constexpr float CV = 0.52573111211913359f;  // 1 / sqrt(2 + phi)
    constexpr float CM = 0.30901699437494742f;  // 1 / (2 phi)
    // winning group and its (p, q, r) = (+-1 axis, +-phi axis, zero axis)
    float best, second, p, q, r, gp, gq, gr;
    int grp;
    if (vA >= vB && vA >= vC) {
        best = vA; second = fmaxf(vB, vC); grp = 0; p = ay; q = az; r = ax; gp = gy; gq = gz; gr = gx;
    } else if (vB >= vC) {
        best = vB; second = fmaxf(vA, vC); grp = 1; p = ax; q = ay; r = az; gp = gx; gq = gy; gr = gz;
    } else {
        best = vC; second = fmaxf(vA, vB); grp = 2; p = az; q = ax; r = ay; gp = gz; gq = gx; gr = gy;
    }
    if (!(best - second > m) || 2.f * p <= m || 2.f * PHI * q <= m) return -1;
    const int slot = 6 * (gp > 0.f) + 3 * (gq > 0.f) + grp;
    const float c0 = CV * best;
    const float c1 = CM * (best + fmaf(PHI, p, r)), c2 = CM * (best + fmaf(PHI, p, -r));
    const float c3 = CM * (best + fmaf(PHI, r, q)), c4 = CM * (best + fmaf(-PHI, r, q));
    const float c5 = CM * (best + fmaf(PHI, q, -p));
    // top two of six (pairwise, then across the pair winners)
    const bool s01 = c0 >= c1, s23 = c2 >= c3, s45 = c4 >= c5;
    const float m01 = s01 ? c0 : c1, n01 = s01 ? c1 : c0;
    const float m23 = s23 ? c2 : c3, n23 = s23 ? c3 : c2;
    const float m45 = s45 ? c4 : c5, n45 = s45 ? c5 : c4;
    float b1, b2;
    int w;
    if (m01 >= m23 && m01 >= m45) {
        b1 = m01; b2 = fmaxf(n01, fmaxf(m23, m45)); w = s01 ? 0 : 1;
    } else if (m23 >= m45) {
        b1 = m23; b2 = fmaxf(n23, fmaxf(m01, m45)); w = s23 ? 2 : 3;
    } else {
        b1 = m45; b2 = fmaxf(n45, fmaxf(m01, m23)); w = s45 ? 4 : 5;
    }
    if (!(b1 - b2 > 2.0e-6f * l1)) return -1;
    // candidate -> neighbour kind: c1/c2 = (p-phi, r sign == / != sign(g_r)), c3/c4 likewise, c5
    const bool rp = gr > 0.f;
    int kind = w;  // 0: the vertex itself
    if (w == 1) kind = rp ? 1 : 2;
    else if (w == 2) kind = rp ? 2 : 1;
    else if (w == 3) kind = rp ? 3 : 4;
    else if (w == 4) kind = rp ? 4 : 3;
    return ic.fk[6 * slot + kind];
}

// Table lookup of the exact argmax (tables.icosphere_lut): canonical face
// point (p / r, q / r) of |g| -> cell -> canonical direction -> actual
// direction by (permutation, sign bits).  -1 when the cell is crossed by a
// Voronoi boundary (2.7% of cells) or |g| is too small for the division.
constexpr int kLutN = 128;
constexpr int kLutBytes = kLutN * kLutN + 42 * 24;

VK_D int nearest_dir_lut(const uint8_t* lut, float gx, float gy, float gz, float ax, float ay, float az) {
    float p, q, r;
    int perm;
    if (az >= ax && az >= ay) { p = ax; q = ay; r = az; perm = 0; }
    else if (ax >= ay) { p = ay; q = az; r = ax; perm = 1; }
    else { p = az; q = ax; r = ay; perm = 2; }
    if (!(r > 1.0e-30f)) return -1;
    const int iu = min(__float2int_rz(__fdividef(p, r) * (float)kLutN), kLutN - 1);
    const int iv = min(__float2int_rz(__fdividef(q, r) * (float)kLutN), kLutN - 1);
    const int c = lut[iv * kLutN + iu];
    if (c == 255) return -1;
    const int sb = (gx < 0.f) | ((gy < 0.f) << 1) | ((gz < 0.f) << 2);
    return lut[kLutN * kLutN + c * 24 + perm * 8 + sb];
}

// Rare path: tiny gradients (|g|_1 < 1e-30, down to fp32 subnormals or an
// fp32 gradient that rounded to 0), where the fp32 scores and margins below
// lose their relative accuracy: the reference's 42 fp64 dots directly.
__device__ __noinline__ int nearest_dir_tiny(const double* dirs, const Nb6& nb) {
    double x64, y64, z64;
    grad64(nb, x64, y64, z64);
    return nearest_dir(dirs, 42, x64, y64, z64);
}

VK_D int nearest_dir_ico(const double* dirs, const IcoSh& ic, const uint8_t* lut, float gx, float gy, float gz,
                         const Nb6& nb) {
    constexpr float PHI = 1.6180339887498949f;
    const float ax = fabsf(gx), ay = fabsf(gy), az = fabsf(gz);
    if (lut) {
        const int k = nearest_dir_lut(lut, gx, gy, gz, ax, ay, az);
        if (k >= 0) return k;
    }
    const float l1 = ax + ay + az;
    if (!(l1 >= 1.0e-30f)) return nearest_dir_tiny(dirs, nb);
    const float vA = fmaf(PHI, az, ay), vB = fmaf(PHI, ay, ax), vC = fmaf(PHI, ax, az);
    const float m = 1.0e-5f * 2.7f * l1;
    const int fast = nearest_dir_fast(ic, gx, gy, gz, ax, ay, az, l1, vA, vB, vC, m);
    if (fast >= 0) return fast;
    const float best = fmaxf(vA, fmaxf(vB, vC));
    // candidate vertex slots: construction index 6*a + 3*b + group, a/b = 1 for the + sign
    unsigned slots = 0;
    auto add_group = [&](float v, int grp, float ca, float cb, float wa, float wb) {
        // ca / cb: the g components paired with the +-1 and +-phi coordinates, wa / wb their weights
        if (v < best - m) return;
        const int sa = ca > 0.f, sb = cb > 0.f;
        const bool fa = 2.f * wa * fabsf(ca) <= m, fb = 2.f * wb * fabsf(cb) <= m;
        slots |= 1u << (6 * sa + 3 * sb + grp);
        if (fa) slots |= 1u << (6 * (1 - sa) + 3 * sb + grp);
        if (fb) slots |= 1u << (6 * sa + 3 * (1 - sb) + grp);
        if (fa && fb) slots |= 1u << (6 * (1 - sa) + 3 * (1 - sb) + grp);
    };
    add_group(vA, 0, gy, gz, 1.f, PHI);  // (0, a, b)
    add_group(vB, 1, gx, gy, 1.f, PHI);  // (a, b, 0)
    add_group(vC, 2, gz, gx, 1.f, PHI);  // (b, 0, a)
    float b1 = -INFINITY, b2 = -INFINITY;
    int i1 = 1 << 30;
    for (unsigned t = slots; t; t &= t - 1) {
        const int v = __ffs(t) - 1;
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            const float4 dd = ic.cd[6 * v + c];
            const int k = ic.ci[6 * v + c];
            const float d = fmaf(gz, dd.z, fmaf(gy, dd.y, gx * dd.x));
            if (k != i1) {
                if (d > b1 || (d == b1 && k < i1)) {
                    b2 = fmaxf(b2, b1);
                    b1 = d;
                    i1 = k;
                } else {
                    b2 = fmaxf(b2, d);
                }
            }
        }
    }
    const float sep = 2.0e-6f * l1;
    if (b1 - b2 > sep) return i1;
    // near tie: exact fp64 dots over every candidate within the separation window
    double x64, y64, z64;
    grad64(nb, x64, y64, z64);
    return nearest_dir_ico_exact(dirs, ic, slots, gx, gy, gz, b1 - sep, x64, y64, z64);
}

// Fast vote of one ball voxel: fp32 magnitude x fp32 window (relative error
// <= kVoteRel against the reference vote) into the exactly determined nearest
// direction.  Returns -1 for zero gradients (mag == 0 exactly in the reference).
VK_D int ori_vote_fast(const Nb6& n, const float* __restrict__ win32, int d2, const double* dirs, const IcoSh* ic,
                       const uint8_t* lut, int K, float& vote) {
    float gx, gy, gz;
    grad32(n, gx, gy, gz);
    if (!grad_nonzero(n)) return -1;
    vote = nz_vote(fmul(norm3_f32(gx, gy, gz), __ldg(win32 + d2)));
    if (ic) return nearest_dir_ico(dirs, *ic, lut, gx, gy, gz, n);
    double x64, y64, z64;
    grad64(n, x64, y64, z64);
    return nearest_dir(dirs, K, x64, y64, z64);
}

// Fast z-major ball walk (consecutive lanes take consecutive x: coalesced
// gathers); INTERIOR: ball and gradient stencil inside the volume.  Returns
// this thread's count of in-volume voxels.
//
// With the lookup table, the ~3% of voxels whose canonical cell is crossed by
// a Voronoi boundary are not resolved in place (their screened argmax would
// run in more than half of all warp steps with a lane or two active): they go
// to a per-warp queue of (voxel, vote) and are resolved 32 at a time with the
// whole warp (neighbours reloaded, screened + exact argmax), then voted.
template <bool INTERIOR>
VK_D int ori_walk(const vk_kp& kp, const vk_level& L, const float* data, const vk_ball& ball,
                  const int* __restrict__ ball_offsets, const float* __restrict__ win32, const double* dirs,
                  const IcoSh* icp, const uint8_t* lut, int K, double* hist, int2* queue) {
    const int tid = threadIdx.x, lane = tid & 31;
    const unsigned plane = (unsigned)L.nx * (unsigned)L.ny;
    hist = vote_copy(hist);
    const bool defer = icp != nullptr && lut != nullptr;  // CTA-uniform
    auto resolve = [&](int2 e) {
        const unsigned c = (unsigned)e.x;
        const int z = (int)(c / plane), rem = (int)(c - (unsigned)z * plane);
        const int y = rem / L.nx, x = rem - y * L.nx;
        const Nb6 nb = load_nb6(data, L.nx, L.ny, L.nz, x, y, z);
        float gx, gy, gz;
        grad32(nb, gx, gy, gz);
        red_vote(hist, nearest_dir_ico(dirs, *icp, nullptr, gx, gy, gz, nb), __int_as_float(e.y));
    };
    int qn = 0;  // warp-uniform queue fill
    int inside_cnt = 0;
    int pn = tid < ball.count ? __ldg(ball_offsets + ball.zstart + tid) : 0;
    for (int base = 0; base < ball.count; base += kOriThreads) {
        const int j = base + tid;
        const int p = pn;
        if (j + kOriThreads < ball.count) pn = __ldg(ball_offsets + ball.zstart + j + kOriThreads);
        int bin = -1;
        float vote = 0.f;
        bool miss = false;
        unsigned c = 0;
        if (j < ball.count) {
            const int ox = unpack_off(p, 0), oy = unpack_off(p, 1), oz = unpack_off(p, 2);
            const int x = kp.ix + ox, y = kp.iy + oy, z = kp.iz + oz;
            if (INTERIOR || (x >= 0 && y >= 0 && z >= 0 && x < L.nx && y < L.ny && z < L.nz)) {
                ++inside_cnt;
#if VK_ORI_PREFETCH
                prefetch_plane_ahead(data, L.nx, L.ny, L.nz, x, y, z, VK_ORI_PREFETCH);
#endif
                c = ((unsigned)z * (unsigned)L.ny + (unsigned)y) * (unsigned)L.nx + (unsigned)x;
                const Nb6 nb = INTERIOR ? load_nb6_interior(data, (unsigned)L.nx, plane, c)
                                        : load_nb6(data, L.nx, L.ny, L.nz, x, y, z);
                if (defer) {
                    float gx, gy, gz;
                    grad32(nb, gx, gy, gz);
                    if (grad_nonzero(nb)) {
                        vote = nz_vote(fmul(norm3_f32(gx, gy, gz), __ldg(win32 + (ox * ox + oy * oy + oz * oz))));
                        bin = nearest_dir_lut(lut, gx, gy, gz, fabsf(gx), fabsf(gy), fabsf(gz));
                        miss = bin < 0;
                    }
                } else {
                    bin = ori_vote_fast(nb, win32, ox * ox + oy * oy + oz * oz, dirs, icp, lut, K, vote);
                }
            }
        }
        red_vote(hist, bin, vote);
        if (defer) {
            const unsigned mm = __ballot_sync(0xffffffffu, miss);
            if (mm) {
                if (miss) queue[qn + __popc(mm & ((1u << lane) - 1u))] = make_int2((int)c, __float_as_int(vote));
                qn += __popc(mm);
                if (qn >= 32) {
                    __syncwarp();
                    resolve(queue[qn - 32 + lane]);
                    qn -= 32;
                    __syncwarp();
                }
            }
        }
    }
    if (defer && qn > 0) {
        __syncwarp();
        if (lane < qn) resolve(queue[lane]);
        __syncwarp();
    }
    return inside_cnt;
}

// ori_walk<true> over the plane-staged ball (vk_stage.cuh): the same votes,
// bins and deferred queue, neighbours from shared memory.  Returns the ball
// size on thread 0 (every voxel of an interior ball is inside).
VK_D int ori_walk_staged(const vk_kp& kp, const vk_level& L, const float* data, const vk_ball& ball,
                         const int* __restrict__ ball_offsets, const float* __restrict__ win32, const double* dirs,
                         const IcoSh* icp, const uint8_t* lut, double* hist, int2* queue, float* ring) {
    const int lane = threadIdx.x & 31;
    hist = vote_copy(hist);
    const unsigned plane = (unsigned)L.nx * (unsigned)L.ny;
    auto resolve = [&](int2 e) {
        const unsigned c = (unsigned)e.x;
        const int z = (int)(c / plane), rem = (int)(c - (unsigned)z * plane);
        const int y = rem / L.nx, x = rem - y * L.nx;
        const Nb6 nb = load_nb6(data, L.nx, L.ny, L.nz, x, y, z);
        float gx, gy, gz;
        grad32(nb, gx, gy, gz);
        red_vote(hist, nearest_dir_ico(dirs, *icp, nullptr, gx, gy, gz, nb), __int_as_float(e.y));
    };
    int qn = 0;  // warp-uniform queue fill
    const unsigned cc = ((unsigned)kp.iz * (unsigned)L.ny + (unsigned)kp.iy) * (unsigned)L.nx + (unsigned)kp.ix;
    staged_ball_walk(data, L.nx, L.ny, kp, ball, ball_offsets + ball.zstart, ball_offsets + ball.pstart, ring,
                     [&](bool valid, int ox, int oy, int oz, const Nb6& nb) {
        int bin = -1;
        float vote = 0.f;
        bool miss = false;
        if (valid && grad_nonzero(nb)) {
            float gx, gy, gz;
            grad32(nb, gx, gy, gz);
            vote = nz_vote(fmul(norm3_f32(gx, gy, gz), __ldg(win32 + (ox * ox + oy * oy + oz * oz))));
            bin = nearest_dir_lut(lut, gx, gy, gz, fabsf(gx), fabsf(gy), fabsf(gz));
            miss = bin < 0;
        }
        red_vote(hist, bin, vote);
        const unsigned mm = __ballot_sync(0xffffffffu, miss);
        if (mm) {
            if (miss) {
                const unsigned c = cc + (unsigned)(oz * (int)plane + oy * L.nx + ox);
                queue[qn + __popc(mm & ((1u << lane) - 1u))] = make_int2((int)c, __float_as_int(vote));
            }
            qn += __popc(mm);
            if (qn >= 32) {
                __syncwarp();
                resolve(queue[qn - 32 + lane]);
                qn -= 32;
                __syncwarp();
            }
        }
    });
    if (qn > 0) {
        __syncwarp();
        if (lane < qn) resolve(queue[lane]);
        __syncwarp();
    }
    return threadIdx.x == 0 ? ball.count : 0;
}

// Dense per-voxel gradient data for a batched level: (gx, gy, gz, |g|) with
// |g| evaluated in fp64 (no fp32 underflow for tiny nonzero gradients) and
// rounded once, plus the exact nearest icosphere direction (255 for g == 0).
__global__ void __launch_bounds__(256)
gradient_volume_kernel(const float* __restrict__ level, float4* __restrict__ g4, uint8_t* __restrict__ bins, int nx,
                       int ny, int nz, long long total, const double* __restrict__ dirs_g, IcoT ico) {
    __shared__ double dirs[42 * 3];
    __shared__ IcoSh ic;
    const int tid = threadIdx.x;
    for (int i = tid; i < 42 * 3; i += blockDim.x) dirs[i] = dirs_g[i];
    if (tid < 72) {
        const int v = tid / 6, c = tid % 6;
        const int k = c == 0 ? ico.vert[v] : ico.adj[v][c - 1];
        ic.ci[tid] = k;
        ic.cd[tid] = make_float4((float)dirs_g[3 * k], (float)dirs_g[3 * k + 1], (float)dirs_g[3 * k + 2], 0.f);
        ic.fk[tid] = c == 0 ? ico.vert[v] : ico.kind[v][c - 1];
    }
    __syncthreads();
    const long long vol = (long long)nx * ny * nz;
    for (long long i = (long long)blockIdx.x * blockDim.x + tid; i < total; i += (long long)gridDim.x * blockDim.x) {
        const long long b = i / vol;
        const unsigned r = (unsigned)(i - b * vol);
        const unsigned plane = (unsigned)nx * (unsigned)ny;
        const int z = (int)(r / plane);
        const unsigned rem = r - (unsigned)z * plane;
        const int y = (int)(rem / (unsigned)nx);
        const int x = (int)(rem - (unsigned)y * (unsigned)nx);
        const Nb6 n = load_nb6(level + b * vol, nx, ny, nz, x, y, z);
        float gx, gy, gz;
        grad32(n, gx, gy, gz);
        float4 o = make_float4(gx, gy, gz, 0.f);
        int bin = 255;
        if (grad_nonzero(n)) {
            double x64, y64, z64;
            grad64(n, x64, y64, z64);
            o.w = nz_vote((float)norm3_numpy(x64, y64, z64));
            bin = nearest_dir_ico(dirs, ic, nullptr, gx, gy, gz, n);
        }
        g4[i] = o;
        bins[i] = (uint8_t)bin;
    }
}

// Orientation field of a batched level: per voxel the fp32 magnitude of the
// fp32 gradient (norm3_f32: the fast path's vote before the window) and the
// exact nearest icosphere direction (255 for g == 0).  Keypoint-independent,
// so the ball walks of all keypoints on this level gather 5 bytes per visit
// instead of recomputing a 6-neighbour gradient and an argmax.
constexpr int kFieldPlanes = 16;  // z planes per CTA of orient_field_kernel

__global__ void __launch_bounds__(256)
orient_field_kernel(const float* __restrict__ level, float* __restrict__ mag, uint8_t* __restrict__ bins, int nx,
                    int ny, int nz, int nzc, const double* __restrict__ dirs_g, IcoT ico,
                    const uint8_t* __restrict__ ico_lut) {
    __shared__ double dirs[42 * 3];
    __shared__ IcoSh ic;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    for (int i = tid; i < 42 * 3; i += 256) dirs[i] = dirs_g[i];
    if (tid < 72) {
        const int v = tid / 6, c = tid % 6;
        const int k = c == 0 ? ico.vert[v] : ico.adj[v][c - 1];
        ic.ci[tid] = k;
        ic.cd[tid] = make_float4((float)dirs_g[3 * k], (float)dirs_g[3 * k + 1], (float)dirs_g[3 * k + 2], 0.f);
        ic.fk[tid] = c == 0 ? ico.vert[v] : ico.kind[v][c - 1];
    }
    __syncthreads();
    // block = 32 x-columns x 8 rows x kFieldPlanes planes (blockIdx.z = volume * nzc + z chunk);
    // the lookup table is read through L1 (16 KB, hot)
    const int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y;
    if (x >= nx || y >= ny) return;
    const int b = blockIdx.z / nzc, z0 = (blockIdx.z - b * nzc) * kFieldPlanes;
    const long long vol = (long long)nx * ny * nz;
    const float* lv = level + b * vol;
    const int z1 = min(nz, z0 + kFieldPlanes);
    for (int z = z0; z < z1; ++z) {
        const long long i = b * vol + ((long long)z * ny + y) * nx + x;
        const Nb6 n = load_nb6(lv, nx, ny, nz, x, y, z);
        float gx, gy, gz;
        grad32(n, gx, gy, gz);
        float m = 0.f;
        int bin = 255;
        if (grad_nonzero(n)) {
            m = nz_vote(norm3_f32(gx, gy, gz));
            bin = nearest_dir_ico(dirs, ic, ico_lut, gx, gy, gz, n);
        }
        mag[i] = m;
        bins[i] = (uint8_t)bin;
    }
}

// Ball walk over an orientation field: U voxels per thread per step with all
// their gathers in flight, packed offsets of the next step prefetched.
// INTERIOR: ball inside the volume (no bounds tests).  Votes are the fast
// path's fp32 |g| x window, bit for bit.
template <bool INTERIOR>
VK_D int field_walk(const vk_kp& kp, const vk_level& L, const float* __restrict__ mag,
                    const uint8_t* __restrict__ bins, const vk_ball& ball, const int* __restrict__ ball_offsets,
                    const float* __restrict__ win32, double* hist) {
    constexpr int U = 4;
    const int tid = threadIdx.x;
    const int* offs = ball_offsets + ball.zstart;
    const int nx = L.nx, plane = L.nx * L.ny;
    const int kc = (kp.iz * L.ny + kp.iy) * nx + kp.ix;
    hist = vote_copy(hist);
    int cnt = 0;
    int pn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int j = u * kOriThreads + tid;
        pn[u] = j < ball.count ? __ldg(offs + j) : 0;
    }
    for (int base = 0; base < ball.count; base += U * kOriThreads) {
        int idx[U], d2[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = base + u * kOriThreads + tid;
            const int p = pn[u];
            const int jn = j + U * kOriThreads;
            pn[u] = jn < ball.count ? __ldg(offs + jn) : 0;
            const int ox = unpack_off(p, 0), oy = unpack_off(p, 1), oz = unpack_off(p, 2);
            ok[u] = j < ball.count;
            if (!INTERIOR) {
                const int x = kp.ix + ox, y = kp.iy + oy, z = kp.iz + oz;
                ok[u] = ok[u] && x >= 0 && y >= 0 && z >= 0 && x < L.nx && y < L.ny && z < L.nz;
            }
            idx[u] = ok[u] ? kc + oz * plane + oy * nx + ox : kc;
            d2[u] = ok[u] ? ox * ox + oy * oy + oz * oz : 0;
        }
        int b[U];
        float m[U], w[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            b[u] = ok[u] ? (int)__ldg(bins + idx[u]) : 255;
            m[u] = __ldg(mag + idx[u]);
            w[u] = __ldg(win32 + d2[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            cnt += ok[u];
            red_vote(hist, b[u] == 255 ? -1 : b[u], nz_vote(fmul(m[u], w[u])));
        }
    }
    return cnt;
}

// Frames from a weight vector whose comparisons are exact (dominant_orientations).
// order[] must hold the bins sorted by (-w, index).
VK_D int frames_from(const double* w, const int* order, int K, const uint8_t* ok, double ratio, int max_frames,
                     int* prim, int* sec) {
    const double top = w[order[0]];
    if (!(top > 0.0)) return 0;
    const double thr = dmul(ratio, top);
    int nf = 0, taken = 0;
    for (int r = 0; r < K && taken < max_frames; ++r) {
        const int p = order[r];
        if (!(w[p] >= thr)) continue;
        ++taken;
        for (int q2 = 0; q2 < K; ++q2) {
            const int q = order[q2];
            if (q == p) continue;
            if (ok[p * K + q]) {
                prim[nf] = p;
                sec[nf] = q;
                ++nf;
                break;
            }
        }
    }
    return nf;
}

// order[] by (-w, index): parallel rank computation over the CTA.
VK_D void sort_desc(const double* w, int K, int* order) {
    for (int b = threadIdx.x; b < K; b += blockDim.x) {
        int r = 0;
        const double wb = w[b];
        for (int j = 0; j < K; ++j) r += (w[j] > wb) || (w[j] == wb && j < b);
        order[r] = b;
    }
}

// Are all decisions of frames_from() the same for every weight vector within
// +-eps of w?  Only the top of the order matters: primaries are the first
// max_frames bins above the threshold and each secondary is the first usable
// bin of the order, so positions 0..m (m = max_frames + 2) and the gap below
// them decide every frame.  Marks the bins whose exact value could change a
// decision: both members of every unseparated adjacent pair among those
// positions, and a bin with an undecided threshold test together with the top
// bin (the threshold is ratio x top).  Returns whether any bin was marked.
// With one warp: lane r tests the adjacent pair (r, r + 1) and the threshold
// decision at position r (m <= VK_MAX_FRAMES + 2 < 32); returns the warp-wide
// any.
VK_D bool warp_mark_uncertain(const double* w, const int* order, int K, double epsrel, double epsabs, double ratio,
                              int max_frames, int* unc) {
    const int lane = threadIdx.x & 31;
    auto lo = [&](double v) { return v == 0.0 ? 0.0 : dsub(v, v * epsrel + epsabs); };
    auto hi = [&](double v) { return v == 0.0 ? 0.0 : dadd(v, v * epsrel + epsabs); };
    bool any = false;
    const int m = min(K - 1, max_frames + 2);
    if (lane < m) {
        const double a = w[order[lane]], b = w[order[lane + 1]];
        if (b != 0.0 && !(lo(a) > hi(b))) {
            unc[order[lane]] = unc[order[lane + 1]] = 1;
            any = true;
        }
    }
    const double top = w[order[0]];
    if (top > 0.0 && lane <= m) {
        const double thr_lo = dmul(ratio, lo(top));
        const double thr_hi = dmul(ratio, hi(top));
        const double v = w[order[lane]];
        if (!(lo(v) >= thr_hi) && !(hi(v) < thr_lo)) {
            unc[order[lane]] = unc[order[0]] = 1;
            any = true;
        }
    }
    return __any_sync(0xffffffffu, any);
}

// frames_from with one warp (orient.py:310-350 semantics): primaries are the
// positions of the (-w, index) order whose weight reaches ratio x top, at most
// max_frames of them counted whether or not a secondary exists; each
// secondary is the first bin of the order != primary with pair_ok, found with
// a ballot over the order.  Writes nframes[0], prim[0..], sec[0..].
VK_D void warp_frames_from(const double* w, const int* order, int K, const uint8_t* ok, double ratio, int max_frames,
                           int* nframes, int* prim, int* sec) {
    const int lane = threadIdx.x & 31;
    int nf = 0;
    const double top = w[order[0]];
    if (top > 0.0) {
        const double thr = dmul(ratio, top);
        const unsigned q0 = __ballot_sync(0xffffffffu, lane < K && w[order[lane]] >= thr);
        const unsigned q1 = __ballot_sync(0xffffffffu, lane + 32 < K && w[order[lane + 32]] >= thr);
        int taken = 0;
        for (int h = 0; h < 2; ++h) {
            for (unsigned qm = h ? q1 : q0; qm && taken < max_frames; qm &= qm - 1) {
                const int p = order[32 * h + __ffs(qm) - 1];
                ++taken;
                const int oa = order[lane], ob = lane + 32 < K ? order[lane + 32] : p;
                const unsigned m0 = __ballot_sync(0xffffffffu, lane < K && oa != p && ok[p * K + oa]);
                const unsigned m1 = __ballot_sync(0xffffffffu, ob != p && ok[p * K + ob]);
                const int q2 = m0 ? __ffs(m0) - 1 : (m1 ? 32 + __ffs(m1) - 1 : -1);
                if (q2 >= 0) {
                    if (lane == 0) {
                        prim[nf] = p;
                        sec[nf] = order[q2];
                    }
                    ++nf;
                }
            }
        }
    }
    if (lane == 0) *nframes = nf;
}

// Reference-order re-accumulation of the uncertain bins only (see
// sr_exact_subset in vk_describe.cu): exact fast binning, the reference's
// fp64 vote |g| x window for voxels of an uncertain bin, ordered sums by one
// thread over ballot-compacted entries.  Certified bins keep their fast sums.
__device__ __noinline__ void ori_exact_subset(const float* data, const vk_level& L, const vk_kp& kp,
                                              const vk_ball& ball, const int* __restrict__ ball_offsets,
                                              const double* __restrict__ win, const double* dirs, const IcoSh* icp,
                                              const uint8_t* lut, int K, OriShared& sh) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid < K && sh.unc[tid]) sh.w[tid] = 0.0;
    for (int base = 0; base < ball.count; base += kOriThreads) {
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
                    double x64, y64, z64;
                    grad64(nb, x64, y64, z64);
                    const int b = icp ? nearest_dir_ico(dirs, *icp, lut, gx, gy, gz, nb) : nearest_dir(dirs, K, x64, y64, z64);
                    if (sh.unc[b]) {
                        v = dmul(norm3_numpy(x64, y64, z64), __ldg(win + (ox * ox + oy * oy + oz * oz)));
                        bin = b;
                    }
                }
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, bin >= 0);
        if (lane == 0) sh.wmask[wid] = m;
        sh.xb[tid] = bin;
        sh.xv[tid] = v;
        __syncthreads();
        if (tid == 0) {
            for (int g = 0; g < kOriThreads / 32; ++g)
                for (unsigned t = sh.wmask[g]; t; t &= t - 1) {
                    const int q = 32 * g + __ffs(t) - 1;
                    sh.w[sh.xb[q]] = dadd(sh.w[sh.xb[q]], sh.xv[q]);
                }
        }
        __syncthreads();
    }
    __syncthreads();
}

#ifndef VK_ORI_MIN_BLOCKS
#define VK_ORI_MIN_BLOCKS 4
#endif
__global__ void __launch_bounds__(kOriThreads, VK_ORI_MIN_BLOCKS)
orient_kernel(const vk_kp* __restrict__ kps, const int* __restrict__ n_kp_dev, int n_kp_max,
              const vk_level* __restrict__ levels, const vk_ball* __restrict__ balls,
              const int* __restrict__ ball_offsets, const double* __restrict__ windows,
              const float* __restrict__ windows32, const double* __restrict__ dirs_g, int K,
              const uint8_t* __restrict__ pair_ok, double ratio, int max_frames, double* __restrict__ weights,
              int* __restrict__ nframes, int* __restrict__ prim, int* __restrict__ sec, int* __restrict__ status,
              int exact_only, IcoT ico, const uint8_t* __restrict__ ico_lut, const vk_gradlevel* __restrict__ grads,
              double* __restrict__ work) {
    __shared__ OriShared sh;
    __shared__ IcoSh ic;
    __shared__ __align__(16) uint8_t lut[kLutBytes];
#if VK_ORI_STAGED
    extern __shared__ __align__(16) float ring[];  // kStageFloats (dynamic: the static part is ~34 KB)
#endif
    double* hist = work + (long long)blockIdx.x * kAccumSlot;  // [K] fp64, L2-resident
    const int tid = threadIdx.x;
    for (int i = tid; i < 3 * K; i += kOriThreads) sh.dirs[i] = dirs_g[i];
    if (ico.valid && tid < 72) {
        const int v = tid / 6, c = tid % 6;
        const int k = c == 0 ? ico.vert[v] : ico.adj[v][c - 1];
        ic.ci[tid] = k;
        ic.cd[tid] = make_float4((float)dirs_g[3 * k], (float)dirs_g[3 * k + 1], (float)dirs_g[3 * k + 2], 0.f);
        ic.fk[tid] = c == 0 ? ico.vert[v] : ico.kind[v][c - 1];
    }
    for (int i = tid; i < K * K; i += kOriThreads) sh.ok[i] = pair_ok[i];
    const int n_kp = n_kp_dev ? min(*n_kp_dev, n_kp_max) : n_kp_max;
    const IcoSh* icp = ico.valid ? &ic : nullptr;
    const uint8_t* lutp = ico.valid && ico_lut ? lut : nullptr;
    if (lutp)
        for (int i = tid; i < kLutBytes / 4; i += kOriThreads)
            reinterpret_cast<uint32_t*>(lut)[i] = __ldg(reinterpret_cast<const uint32_t*>(ico_lut) + i);
    __syncthreads();

    for (int item = blockIdx.x; item < n_kp; item += gridDim.x) {
        const vk_kp kp = kps[item];
        const vk_level L = levels[kp.lvl];
        const float* data = L.base + (long long)kp.vol * L.vol_stride;
        const vk_ball ball = balls[kp.ball];
        const double* win = windows + ball.window_start;
        const float* win32 = windows32 + ball.window_start;
        zero_hist(hist, K);
        if (tid == 0) { sh.n_inside = 0; sh.exact = exact_only; sh.repair = 0; }
        __syncthreads();
        int inside_cnt = 0;
        const vk_gradlevel GL = grads ? grads[kp.lvl] : vk_gradlevel{};
        if (!exact_only && GL.bin != nullptr && GL.kind == 1) {
            const float* fm = reinterpret_cast<const float*>(GL.g4) + (long long)kp.vol * GL.vol_stride;
            const uint8_t* fb = GL.bin + (long long)kp.vol * GL.vol_stride;
            inside_cnt = ball_interior(kp.ix, kp.iy, kp.iz, ball.r, L.nx, L.ny, L.nz)
                             ? field_walk<true>(kp, L, fm, fb, ball, ball_offsets, win32, hist)
                             : field_walk<false>(kp, L, fm, fb, ball, ball_offsets, win32, hist);
        } else if (!exact_only && GL.bin != nullptr) {
            // precomputed gradient volume: one coalesced (bin, |g|) pair per visit
            const uint8_t* bl = GL.bin + (long long)kp.vol * GL.vol_stride;
            const float4* gl = reinterpret_cast<const float4*>(GL.g4) + (long long)kp.vol * GL.vol_stride;
            int pn = tid < ball.count ? __ldg(ball_offsets + ball.zstart + tid) : 0;
            for (int base = 0; base < ball.count; base += kOriThreads) {
                const int j = base + tid;
                const int p = pn;
                if (j + kOriThreads < ball.count) pn = __ldg(ball_offsets + ball.zstart + j + kOriThreads);
                int bin = -1;
                float vote = 0.f;
                if (j < ball.count) {
                    const int ox = unpack_off(p, 0), oy = unpack_off(p, 1), oz = unpack_off(p, 2);
                    const int x = kp.ix + ox, y = kp.iy + oy, z = kp.iz + oz;
                    if (x >= 0 && y >= 0 && z >= 0 && x < L.nx && y < L.ny && z < L.nz) {
                        ++inside_cnt;
                        const unsigned idx = ((unsigned)z * (unsigned)L.ny + (unsigned)y) * (unsigned)L.nx + (unsigned)x;
                        const int b = __ldg(bl + idx);
                        if (b != 255) {
                            bin = b;
                            vote = nz_vote(fmul(__ldg(&gl[idx].w), __ldg(win32 + (ox * ox + oy * oy + oz * oz))));
                        }
                    }
                }
                red_vote(vote_copy(hist), bin, vote);
            }
        } else if (!exact_only && VK_ORI_STAGED && lutp && ball.r <= kStageMaxR &&
                   ball_interior(kp.ix, kp.iy, kp.iz, ball.r, L.nx, L.ny, L.nz)) {
#if VK_ORI_STAGED
            inside_cnt = ori_walk_staged(kp, L, data, ball, ball_offsets, win32, sh.dirs, icp, lutp, hist,
                                         sh.queue[tid >> 5], ring);
#endif
        } else if (!exact_only) {
            inside_cnt = ball_interior(kp.ix, kp.iy, kp.iz, ball.r, L.nx, L.ny, L.nz)
                             ? ori_walk<true>(kp, L, data, ball, ball_offsets, win32, sh.dirs, icp, lutp, K, hist,
                                              sh.queue[tid >> 5])
                             : ori_walk<false>(kp, L, data, ball, ball_offsets, win32, sh.dirs, icp, lutp, K, hist,
                                               sh.queue[tid >> 5]);
        } else {
            for (int j = tid; j < ball.count; j += kOriThreads) {
                const int p = __ldg(ball_offsets + ball.start + j);
                const int x = kp.ix + unpack_off(p, 0), y = kp.iy + unpack_off(p, 1), z = kp.iz + unpack_off(p, 2);
                inside_cnt += x >= 0 && y >= 0 && z >= 0 && x < L.nx && y < L.ny && z < L.nz;
            }
        }
        if (inside_cnt) atomicAdd(&sh.n_inside, inside_cnt);
        __syncthreads();
        if (sh.n_inside == 0) {
            // DataError: orientation neighbourhood entirely outside (orient.py:291-292)
            if (tid == 0) {
                atomicOr(status, 1);
                nframes[item] = 0;
            }
            __syncthreads();
            continue;
        }
        if (!sh.exact) {
            for (int b = tid; b < K; b += kOriThreads) sh.w[b] = read_hist(hist, b);
            __syncthreads();
            sort_desc(sh.w, K, sh.order);
            for (int b = tid; b < K; b += kOriThreads) sh.unc[b] = 0;
            __syncthreads();
            if (tid < 32) {
                // fp32 votes (kVoteRel) summed in fp64 in some order vs the reference's
                const double epsrel = 2.0 * (kVoteRel + gamma_k((double)sh.n_inside + 64.0));
                const double epsabs = kVoteAbs * sh.n_inside;
                if (warp_mark_uncertain(sh.w, sh.order, K, epsrel, epsabs, ratio, max_frames, sh.unc) && tid == 0) {
                    sh.repair = 1;
                    atomicAdd(status + 1, 1);  // fallback counter (diagnostics)
                }
            }
            __syncthreads();
            if (sh.repair) {
                ori_exact_subset(data, L, kp, ball, ball_offsets, win, sh.dirs, icp, lutp, K, sh);
                sort_desc(sh.w, K, sh.order);
                __syncthreads();
            }
        }
        if (sh.exact) {
            // Exact reference order: all threads compute a chunk of exact votes,
            // then warp 0 adds them bin by bin in ball order (np.add.at).
            double acc0 = 0.0, acc1 = 0.0;
            for (int base = 0; base < ball.count; base += kOriThreads) {
                const int j = base + tid;
                double vote = 0.0;
                bool inside;
                int bin = -1;
                if (j < ball.count)
                    bin = ori_vote(data, L.nx, L.ny, L.nz, kp.ix, kp.iy, kp.iz, __ldg(ball_offsets + ball.start + j), win,
                                   sh.dirs, K, vote, inside);
                sh.xb[tid] = bin;
                sh.xv[tid] = vote;
                __syncthreads();
                if (tid < 32) {
                    const int m = min(kOriThreads, ball.count - base);
#pragma unroll 8
                    for (int q = 0; q < m; ++q) {
                        const int bs = sh.xb[q];
                        const double vs = sh.xv[q];
                        if (bs == tid) acc0 = dadd(acc0, vs);
                        else if (bs == tid + 32) acc1 = dadd(acc1, vs);
                    }
                }
                __syncthreads();
            }
            if (tid < 32) {
                if (tid < K) sh.w[tid] = acc0;
                if (tid + 32 < K) sh.w[tid + 32] = acc1;
            }
            __syncthreads();
            sort_desc(sh.w, K, sh.order);
            __syncthreads();
        }
        if (weights)
            for (int b = tid; b < K; b += kOriThreads) weights[(long long)item * K + b] = sh.w[b];
        if (tid < 32) warp_frames_from(sh.w, sh.order, K, sh.ok, ratio, max_frames, nframes + item,
                                       prim + (long long)item * max_frames, sec + (long long)item * max_frames);
        __syncthreads();
    }
}

// Frames from host-supplied weights (dominant_orientations on a histogram).
__global__ void frames_from_weights_kernel(const double* __restrict__ weights, int n, int K,
                                           const uint8_t* __restrict__ pair_ok, double ratio, int max_frames,
                                           int* __restrict__ nframes, int* __restrict__ prim, int* __restrict__ sec) {
    __shared__ double w[VK_MAX_DIRS];
    __shared__ int order[VK_MAX_DIRS];
    __shared__ uint8_t ok[VK_MAX_DIRS * VK_MAX_DIRS];
    for (int i = threadIdx.x; i < K * K; i += blockDim.x) ok[i] = pair_ok[i];
    for (int item = blockIdx.x; item < n; item += gridDim.x) {
        __syncthreads();
        for (int b = threadIdx.x; b < K; b += blockDim.x) w[b] = weights[(long long)item * K + b];
        __syncthreads();
        sort_desc(w, K, order);
        __syncthreads();
        if (threadIdx.x == 0) {
            int pr[VK_MAX_FRAMES], se[VK_MAX_FRAMES];
            const int nf = frames_from(w, order, K, ok, ratio, max_frames, pr, se);
            nframes[item] = nf;
            for (int f = 0; f < nf; ++f) {
                prim[item * max_frames + f] = pr[f];
                sec[item * max_frames + f] = se[f];
            }
        }
    }
}

// Ordered expansion of per-keypoint frames: a single-CTA scan writes each
// keypoint's first frame slot, then a wide kernel scatters the frames.
__global__ void __launch_bounds__(1024)
frame_offsets_kernel(const int* __restrict__ nframes, const int* __restrict__ n_kp_dev, int n_kp_max,
                     int* __restrict__ first, int* __restrict__ n_frames_dev, int* __restrict__ dropped_dev) {
    __shared__ int warp_sums[32];
    __shared__ int carry_s, dropped_s;
    const int n = n_kp_dev ? min(*n_kp_dev, n_kp_max) : n_kp_max;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) { carry_s = 0; dropped_s = 0; }
    __syncthreads();
    for (int base = 0; base < n; base += 1024) {
        const int i = base + tid;
        const int nf = i < n ? nframes[i] : 0;
        const unsigned zero_mask = __ballot_sync(0xffffffffu, i < n && nf == 0);
        if (lane == 0 && zero_mask) atomicAdd(&dropped_s, __popc(zero_mask));
        int v = nf;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
        }
        if (lane == 31) warp_sums[wid] = v;
        __syncthreads();
        if (wid == 0) {
            int sacc = warp_sums[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, sacc, o);
                if (lane >= o) sacc += t;
            }
            warp_sums[lane] = sacc;
        }
        __syncthreads();
        const int excl = carry_s + v - nf + (wid > 0 ? warp_sums[wid - 1] : 0);
        if (i < n) first[i] = excl;
        __syncthreads();
        if (tid == 1023) carry_s = excl + nf;
        __syncthreads();
    }
    if (tid == 0) {
        n_frames_dev[0] = carry_s;
        dropped_dev[0] = dropped_s;
    }
}

__global__ void frame_write_kernel(const int* __restrict__ nframes, const int* __restrict__ prim,
                                   const int* __restrict__ sec, const int* __restrict__ first,
                                   const int* __restrict__ n_kp_dev, int n_kp_max, int max_frames,
                                   const double* __restrict__ rot_table, int K, vk_frame* __restrict__ frames,
                                   double* __restrict__ rot, int frame_cap) {
    const int n = n_kp_dev ? min(*n_kp_dev, n_kp_max) : n_kp_max;
    // one thread per (keypoint, frame slot, rotation entry)
    const long long total = (long long)n * max_frames * 9;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int e = (int)(t % 9);
        const long long kf = t / 9;
        const int i = (int)(kf / max_frames), f = (int)(kf % max_frames);
        if (f >= nframes[i]) continue;
        const int o = first[i] + f;
        if (o >= frame_cap) continue;
        const int p = prim[i * max_frames + f], q = sec[i * max_frames + f];
        rot[(long long)o * 9 + e] = rot_table[((long long)p * K + q) * 9 + e];
        if (e == 0) {
            vk_frame fr;
            fr.kp = i;
            fr.prim = p;
            fr.sec = q;
            fr.pad_ = 0;
            frames[o] = fr;
        }
    }
}

}  // namespace vk

using namespace vk;

extern "C" int vk_orient(const vk_kp* kps, const int* n_kp_dev, int n_kp_max, const vk_level* levels,
                         const vk_ball* balls, const int* ball_offsets, const double* windows, const float* windows32,
                         const double* dirs, int K, const uint8_t* pair_ok, double secondary_ratio, int max_frames,
                         double* weights, int* nframes, int* prim, int* sec, int* status, int exact_only,
                         const int* ico_host, const uint8_t* ico_lut, const vk_gradlevel* grads, double* work,
                         void* stream) {
    if (!kps || n_kp_max < 0 || !levels || !balls || !ball_offsets || !windows || !windows32 || !dirs || K < 1 || !work ||
        K > VK_MAX_DIRS || !pair_ok || !nframes || !prim || !sec || !status || max_frames < 1 ||
        max_frames > VK_MAX_FRAMES || !(secondary_ratio > 0.0 && secondary_ratio <= 1.0)) {
        set_error("vk_orient: bad arguments (K=%d max_frames=%d)", K, max_frames);
        return VK_ERR_PARAMETER;
    }
    if (n_kp_max == 0) return VK_OK;
    const size_t dyn = VK_ORI_STAGED ? kStageFloats * sizeof(float) : 0;
    static bool configured = false;
    if (dyn && !configured) {
        cudaError_t e = cudaFuncSetAttribute(orient_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        if (e != cudaSuccess) return cuda_status(e, "orient smem attribute");
        configured = true;
    }
    const int grid = accum_grid(orient_kernel, kOriThreads, n_kp_max, dyn);
    IcoT ico{};
    if (ico_host && K == 42) {
        ico.valid = 1;
        for (int v = 0; v < 12; ++v) {
            ico.vert[v] = ico_host[v];
            for (int m = 0; m < 5; ++m) ico.adj[v][m] = ico_host[12 + 5 * v + m];
            for (int m = 0; m < 5; ++m) ico.kind[v][m] = ico_host[72 + 5 * v + m];
        }
    }
    orient_kernel<<<grid, kOriThreads, dyn, as_stream(stream)>>>(kps, n_kp_dev, n_kp_max, levels, balls, ball_offsets,
                                                               windows, windows32, dirs, K, pair_ok, secondary_ratio,
                                                               max_frames, weights, nframes, prim, sec, status,
                                                               exact_only, ico, ico_lut, grads, work);
    count_launch();
    return cuda_status(cudaGetLastError(), "orient launch");
}

extern "C" int vk_frames_from_weights(const double* weights, int n, int K, const uint8_t* pair_ok,
                                      double secondary_ratio, int max_frames, int* nframes, int* prim, int* sec,
                                      void* stream) {
    if (!weights || n < 0 || K < 1 || K > VK_MAX_DIRS || !pair_ok || !nframes || !prim || !sec || max_frames < 1 ||
        max_frames > VK_MAX_FRAMES || !(secondary_ratio > 0.0 && secondary_ratio <= 1.0)) {
        set_error("vk_frames_from_weights: bad arguments");
        return VK_ERR_PARAMETER;
    }
    if (n == 0) return VK_OK;
    frames_from_weights_kernel<<<n < 1024 ? n : 1024, 64, 0, as_stream(stream)>>>(weights, n, K, pair_ok, secondary_ratio,
                                                                                   max_frames, nframes, prim, sec);
    count_launch();
    return cuda_status(cudaGetLastError(), "frames launch");
}

extern "C" int vk_expand_frames(const int* nframes, const int* prim, const int* sec, const int* n_kp_dev, int n_kp_max,
                                int max_frames, const double* rot_table, int K, vk_frame* frames, double* rot,
                                int* n_frames_dev, int* dropped_dev, int frame_cap, int* scratch, void* stream) {
    if (!nframes || !prim || !sec || n_kp_max < 0 || max_frames < 1 || !rot_table || K < 1 || !frames || !rot ||
        !n_frames_dev || !dropped_dev || frame_cap < 0 || (n_kp_max > 0 && !scratch)) {
        set_error("vk_expand_frames: bad arguments");
        return VK_ERR_PARAMETER;
    }
    cudaStream_t st = as_stream(stream);
    frame_offsets_kernel<<<1, 1024, 0, st>>>(nframes, n_kp_dev, n_kp_max, scratch, n_frames_dev, dropped_dev);
    count_launch();
    if (n_kp_max > 0) {
        const long long work = (long long)n_kp_max * max_frames * 9;
        long long blocks = (work + 255) / 256;
        if (blocks > 148 * 8) blocks = 148 * 8;
        frame_write_kernel<<<(unsigned)blocks, 256, 0, st>>>(nframes, prim, sec, scratch, n_kp_dev, n_kp_max, max_frames,
                                                           rot_table, K, frames, rot, frame_cap);
        count_launch();
    }
    return cuda_status(cudaGetLastError(), "expand launch");
}

extern "C" int vk_orient_field(const float* level, float* mag, uint8_t* bin, int nb, int nx, int ny, int nz,
                               const double* dirs, const int* ico_host, const uint8_t* ico_lut, void* stream) {
    if (!level || !mag || !bin || nb < 0 || nx < 1 || ny < 1 || nz < 1 || !dirs || !ico_host) {
        set_error("vk_orient_field: bad arguments");
        return VK_ERR_PARAMETER;
    }
    const long long total = (long long)nb * nx * ny * nz;
    if (total == 0) return VK_OK;
    IcoT ico{};
    ico.valid = 1;
    for (int v = 0; v < 12; ++v) {
        ico.vert[v] = ico_host[v];
        for (int m = 0; m < 5; ++m) ico.adj[v][m] = ico_host[12 + 5 * v + m];
        for (int m = 0; m < 5; ++m) ico.kind[v][m] = ico_host[72 + 5 * v + m];
    }
    const int nzc = (nz + kFieldPlanes - 1) / kFieldPlanes;
    const dim3 grid((nx + 31) / 32, (ny + 7) / 8, (unsigned)(nb * nzc));
    orient_field_kernel<<<grid, dim3(32, 8), 0, as_stream(stream)>>>(level, mag, bin, nx, ny, nz, nzc, dirs, ico,
                                                                      ico_lut);
    count_launch();
    return cuda_status(cudaGetLastError(), "orient field launch");
}

extern "C" int vk_gradient_volume(const float* level, void* g4, uint8_t* bin, int nb, int nx, int ny, int nz,
                                  const double* dirs, const int* ico_host, void* stream) {
    if (!level || !g4 || !bin || nb < 0 || nx < 1 || ny < 1 || nz < 1 || !dirs || !ico_host) {
        set_error("vk_gradient_volume: bad arguments");
        return VK_ERR_PARAMETER;
    }
    const long long total = (long long)nb * nx * ny * nz;
    if (total == 0) return VK_OK;
    IcoT ico{};
    ico.valid = 1;
    for (int v = 0; v < 12; ++v) {
        ico.vert[v] = ico_host[v];
        for (int m = 0; m < 5; ++m) ico.adj[v][m] = ico_host[12 + 5 * v + m];
        for (int m = 0; m < 5; ++m) ico.kind[v][m] = ico_host[72 + 5 * v + m];
    }
    long long blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    gradient_volume_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(level, static_cast<float4*>(g4), bin, nx, ny,
                                                                            nz, total, dirs, ico);
    count_launch();
    return cuda_status(cudaGetLastError(), "gradient volume launch");
}
