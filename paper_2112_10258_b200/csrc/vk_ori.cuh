// vk_ori.cuh -- device building blocks of the orientation walk (orient.py:89-168):
// icosphere argmax tiers, fast / staged / field ball walks, certified frame
// selection and the exact repair of uncertain bins.  Shared by orient_kernel
// (vk_orient.cu) and the fused orientation + SIFT-Rank kernel (vk_orsr.cu).
#pragma once

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

// pair_ok (orient.py:128-168's usable secondary pairs) as a bitset in shared memory: 512 B instead of 4 KB,
// which keeps orient_kernel's static shared memory under 1/3 of a 100 KB carveout (3 CTAs/SM with the larger
// L1 share)
constexpr int kOkWords = VK_MAX_DIRS * VK_MAX_DIRS / 32;
VK_D bool ok_bit(const unsigned* okb, int i) { return (okb[i >> 5] >> (i & 31)) & 1u; }
VK_D void load_ok_bits(unsigned* okb, const uint8_t* __restrict__ pair_ok, int K) {
    const int n = K * K;
    for (int w = threadIdx.x; w < (n + 31) / 32; w += blockDim.x) {
        unsigned v = 0u;
        for (int b = 0; b < 32; ++b) {
            const int i = 32 * w + b;
            if (i < n && pair_ok[i]) v |= 1u << b;
        }
        okb[w] = v;
    }
}

struct OriShared {
    double xv[kOriThreads];
    int xb[kOriThreads];
    double dirs[VK_MAX_DIRS * 3];
    double w[VK_MAX_DIRS];
    int order[VK_MAX_DIRS];
    unsigned okb[kOkWords];  // pair_ok as bits (bytes would cost 3.5 KB more: see load_ok_bits)
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
static __device__ __noinline__ int nearest_dir_ico_exact(const double* dirs, const IcoSh& ic, unsigned slots, float gx,
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
// (fp64 gradient formed by the caller: a noinline callee taking the Nb6 by
// reference would force every walk iteration to store it to the stack)
static __device__ __noinline__ int nearest_dir_tiny(const double* dirs, double x64, double y64, double z64) {
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
    if (!(l1 >= 1.0e-30f)) {
        double x64, y64, z64;
        grad64(nb, x64, y64, z64);
        return nearest_dir_tiny(dirs, x64, y64, z64);
    }
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

// ori_walk<true> (lookup-table path) with the six neighbour loads of the
// thread's next voxel issued before the current voxel is binned: two voxels
// in flight per thread, so the L1 / L2 latency of one gather overlaps the
// arithmetic of the previous one (the walk is latency-bound, not issue-bound:
// long-scoreboard stalls dominate orient_kernel).  Same votes, bins, deferred
// queue.
#ifndef VK_ORI_PIPE
#define VK_ORI_PIPE 1
#endif
#ifndef VK_ORI_DEPTH
#define VK_ORI_DEPTH 2  // voxels in flight per thread (3 was 2% faster than 2 with one vote copy; 2 is 1% faster with two)
#endif
template <bool INTERIOR>
VK_D int ori_walk_pipe(const vk_kp& kp, const vk_level& L, const float* data, const vk_ball& ball,
                       const int* __restrict__ ball_offsets, const float* __restrict__ win32, const double* dirs,
                       const IcoSh* icp, const uint8_t* lut, double* hist, int2* queue) {
    const int tid = threadIdx.x, lane = tid & 31, step = kOriThreads;
    const int nx = L.nx, plane = L.nx * L.ny;
    const int kc = (kp.iz * L.ny + kp.iy) * nx + kp.ix;
    const int* offs = ball_offsets + ball.zstart;
    const int count = ball.count;
    hist = vote_copy(hist);
    auto resolve = [&](int2 e) {
        const unsigned c = (unsigned)e.x;
        const int z = (int)(c / (unsigned)plane), rem = (int)(c - (unsigned)z * (unsigned)plane);
        const int y = rem / nx, x = rem - y * nx;
        const Nb6 nb = load_nb6(data, L.nx, L.ny, L.nz, x, y, z);
        float gx, gy, gz;
        grad32(nb, gx, gy, gz);
        red_vote(hist, nearest_dir_ico(dirs, *icp, nullptr, gx, gy, gz, nb), __int_as_float(e.y));
    };
    auto issue = [&](int pk, Nb6& n) {
        const int ox = unpack_off(pk, 0), oy = unpack_off(pk, 1), oz = unpack_off(pk, 2);
        if (INTERIOR) {
            n = load_nb6_interior(data, (unsigned)nx, (unsigned)plane, (unsigned)(kc + oz * plane + oy * nx + ox));
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
    int qn = 0, cnt = 0;
    // ring: voxel j + d * step has its neighbours loaded (d < D - 1) and its
    // packed offset loaded D - 1 steps ahead of use
    constexpr int D = VK_ORI_DEPTH;
    int pk[D];
    Nb6 nb[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const int jj = tid + d * step;
        pk[d] = jj < count ? __ldg(offs + jj) : 0;
        if (d < D - 1 && jj < count) issue(pk[d], nb[d]);
    }
    for (int base = 0; base < count; base += step) {
        const int j = base + tid;
        const int pc = pk[0];
        Nb6 cur0 = nb[0];
        cur0.sx = cur0.sy = cur0.sz = 0.5f;
#pragma unroll
        for (int d = 0; d + 1 < D; ++d) {
            pk[d] = pk[d + 1];
            nb[d] = nb[d + 1];
        }
        if (j + (D - 1) * step < count) {
            issue(pk[D - 2], nb[D - 2]);
            if (j + D * step < count) pk[D - 1] = __ldg(offs + j + D * step);
        }        int bin = -1;
        float vote = 0.f;
        bool miss = false;
        int c = 0;
        bool in = j < count;
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
            if (grad_nonzero(cur)) {
                const int ox = unpack_off(pc, 0), oy = unpack_off(pc, 1), oz = unpack_off(pc, 2);
                vote = nz_vote(fmul(norm3_f32(gx, gy, gz), __ldg(win32 + (ox * ox + oy * oy + oz * oz))));
                bin = nearest_dir_lut(lut, gx, gy, gz, fabsf(gx), fabsf(gy), fabsf(gz));
                miss = bin < 0;
                c = kc + oz * plane + oy * nx + ox;
            }
        }
        red_vote(hist, bin, vote);
        const unsigned mm = __ballot_sync(0xffffffffu, miss);
        if (mm) {
            if (miss) queue[qn + __popc(mm & ((1u << lane) - 1u))] = make_int2(c, __float_as_int(vote));
            qn += __popc(mm);
            if (qn >= 32) {
                __syncwarp();
                resolve(queue[qn - 32 + lane]);
                qn -= 32;
                __syncwarp();
            }
        }
    }
    if (qn > 0) {
        __syncwarp();
        if (lane < qn) resolve(queue[lane]);
        __syncwarp();
    }
    return cnt;
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
VK_D int frames_from(const double* w, const int* order, int K, const unsigned* okb, double ratio, int max_frames,
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
            if (ok_bit(okb, p * K + q)) {
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

// frames_from with one warp (orient.py:128-168 semantics): primaries are the
// positions of the (-w, index) order whose weight reaches ratio x top, at most
// max_frames of them counted whether or not a secondary exists; each
// secondary is the first bin of the order != primary with pair_ok, found with
// a ballot over the order.  Writes nframes[0], prim[0..], sec[0..].
VK_D void warp_frames_from(const double* w, const int* order, int K, const unsigned* okb, double ratio, int max_frames,
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
                const unsigned m0 = __ballot_sync(0xffffffffu, lane < K && oa != p && ok_bit(okb, p * K + oa));
                const unsigned m1 = __ballot_sync(0xffffffffu, ob != p && ok_bit(okb, p * K + ob));
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
static __device__ __noinline__ void ori_exact_subset(const float* data, const vk_level& L, const vk_kp& kp,
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

}  // namespace vk
