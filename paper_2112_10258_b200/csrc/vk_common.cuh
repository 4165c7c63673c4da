// vk_common.cuh -- shared helpers for the sm_100a volkey kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/volkey_b200.h"

#define VK_HD __host__ __device__ __forceinline__
#define VK_D __device__ __forceinline__

namespace vk {

// Thread-local last-error text (vk_api.cu) and the helpers that set it.
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);
// Number of kernels this library has launched (vk_launch_count()).
void count_launch(int n = 1);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

template <typename T>
VK_HD T clampi(T v, T lo, T hi) { return v < lo ? lo : (v > hi ? hi : v); }

// ---- cp.async (LDGSTS) helpers -------------------------------------------
VK_D void cp_async4(void* smem, const void* gmem) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
// (memory clobbers: shared-memory reads of the landed data must not move above the wait)
VK_D void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
VK_D void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// ---- exact-rounding arithmetic (no contraction) ---------------------------
// The reference evaluates every product and sum as a separately rounded numpy
// ufunc; these wrappers make that explicit (the build also uses -fmad=false).
VK_D float fmul(float a, float b) { return __fmul_rn(a, b); }
VK_D float fadd(float a, float b) { return __fadd_rn(a, b); }
VK_D double dmul(double a, double b) { return __dmul_rn(a, b); }
VK_D double dadd(double a, double b) { return __dadd_rn(a, b); }
VK_D double dsub(double a, double b) { return __dsub_rn(a, b); }
VK_D double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }

// OpenBLAS dgemm order for a K=3 inner product:
// fma(x2, y2, fma(x1, y1, x0*y0)).
VK_D double dot3_blas(double x0, double x1, double x2, double y0, double y1, double y2) {
    return dfma(x2, y2, dfma(x1, y1, dmul(x0, y0)));
}

// np.linalg.norm(axis=1) on an (N, 3) float64 array: sqrt((x*x + y*y) + z*z).
VK_D double norm3_numpy(double x, double y, double z) {
    return __dsqrt_rn(dadd(dadd(dmul(x, x), dmul(y, y)), dmul(z, z)));
}

// Packed ball offset: 10 bits per axis, biased by 512 (|offset| <= 511).
VK_HD int unpack_off(int p, int axis) { return ((p >> (20 - 10 * axis)) & 1023) - 512; }

// Trilinear interpolation with clamping, fp64 arithmetic on fp32 samples --
// sample_trilinear_array (volume.py:203-236) step for step.  `at(x, y, z)`
// fetches one voxel.
template <typename F>
VK_D double trilinear(F at, int nx, int ny, int nz, double px, double py, double pz) {
    const int n[3] = {nx, ny, nz};
    double p[3] = {px, py, pz};
    int i0[3], i1[3];
    double f[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double hi = (double)n[a] - 1.0;
        double q = fmin(fmax(p[a], 0.0), hi);  // np.clip(pts, 0.0, hi)
        long long fl = (long long)floor(q);
        long long cap = n[a] - 2 > 0 ? n[a] - 2 : 0;
        if (fl > cap) fl = cap;
        i0[a] = (int)fl;
        f[a] = dsub(q, (double)fl);
        i1[a] = i0[a] + 1 < n[a] - 1 ? i0[a] + 1 : n[a] - 1;
    }
    auto lerp = [](double a, double b, double t) { return dadd(dmul(a, dsub(1.0, t)), dmul(b, t)); };
    double c000 = at(i0[0], i0[1], i0[2]), c100 = at(i1[0], i0[1], i0[2]);
    double c010 = at(i0[0], i1[1], i0[2]), c110 = at(i1[0], i1[1], i0[2]);
    double c001 = at(i0[0], i0[1], i1[2]), c101 = at(i1[0], i0[1], i1[2]);
    double c011 = at(i0[0], i1[1], i1[2]), c111 = at(i1[0], i1[1], i1[2]);
    double c00 = lerp(c000, c100, f[0]);
    double c10 = lerp(c010, c110, f[0]);
    double c01 = lerp(c001, c101, f[0]);
    double c11 = lerp(c011, c111, f[0]);
    double c0 = lerp(c00, c10, f[1]);
    double c1 = lerp(c01, c11, f[1]);
    return lerp(c0, c1, f[2]);
}

// Central / one-sided gradient in fp64 (volume.py:244-264) at lattice point
// (x, y, z) of an x-fastest fp32 volume.
VK_D void gradient_at(const float* __restrict__ d, int nx, int ny, int nz, int x, int y, int z,
                      double& gx, double& gy, double& gz) {
    const long long sy = nx, sz = (long long)nx * ny;
    const long long c = (long long)z * sz + (long long)y * sy + x;
    int xh = min(x + 1, nx - 1), xl = max(x - 1, 0);
    int yh = min(y + 1, ny - 1), yl = max(y - 1, 0);
    int zh = min(z + 1, nz - 1), zl = max(z - 1, 0);
    double vxh = (double)__ldg(d + c + (xh - x)), vxl = (double)__ldg(d + c + (xl - x));
    double vyh = (double)__ldg(d + c + (long long)(yh - y) * sy), vyl = (double)__ldg(d + c + (long long)(yl - y) * sy);
    double vzh = (double)__ldg(d + c + (long long)(zh - z) * sz), vzl = (double)__ldg(d + c + (long long)(zl - z) * sz);
    // (up - dn) / max(hi - lo, 1): the divisor is 1.0 or 2.0, both exact.
    // x / 2.0 == x * 0.5 exactly, so multiply instead of dividing.
    gx = dmul(dsub(vxh, vxl), (xh - xl) == 2 ? 0.5 : 1.0);
    gy = dmul(dsub(vyh, vyl), (yh - yl) == 2 ? 0.5 : 1.0);
    gz = dmul(dsub(vzh, vzl), (zh - zl) == 2 ? 0.5 : 1.0);
}

// Prefetch the voxel `ahead` planes above (x, y, z) into L1: the z-major ball
// walks touch each plane first as the z+1 neighbour of the plane below, so a
// few planes of lead time hide the L2 / HBM latency of that first touch.
VK_D void prefetch_plane_ahead(const float* __restrict__ d, int nx, int ny, int nz, int x, int y, int z, int ahead) {
    if (z + ahead < nz) {
        const float* p = d + (((unsigned)(z + ahead) * (unsigned)ny + (unsigned)y) * (unsigned)nx + (unsigned)x);
        asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
    }
}

// L2 prefetch of the rows of a keypoint's ball plus its stencil halo (rows
// with dy^2 + dz^2 <= (r + 1)^2, the whole x span of each, clamped to the
// volume), issued by the whole CTA for the NEXT keypoint of a persistent walk:
// the keypoint levels are HBM-resident when the walks start (a batch's levels
// exceed L2), and the ball gathers then wait on HBM latency.
#ifndef VK_PREFETCH_NEXT
#define VK_PREFETCH_NEXT 0  // measured 2.5% slower on B200 (the walks are L1 / issue bound, not HBM-latency bound)
#endif
VK_D void prefetch_ball_l2(const float* __restrict__ d, int nx, int ny, int nz, int cx, int cy, int cz, int r) {
    const int h = r + 1, w = 2 * h + 1;
    const int x0 = max(cx - h, 0), x1 = min(cx + h, nx - 1);
    for (int t = threadIdx.x; t < w * w; t += blockDim.x) {
        const int dy = t % w - h, dz = t / w - h;
        const int y = cy + dy, z = cz + dz;
        if (dy * dy + dz * dz > h * h || y < 0 || y >= ny || z < 0 || z >= nz) continue;
        const float* row = d + ((size_t)z * ny + y) * nx;
        for (int x = x0; x < x1; x += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + x));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(row + x1));
    }
}

// The six axis neighbours of (x, y, z) as loaded fp32 values plus the
// central/one-sided divisor scale per axis (volume.py:244-264).
struct Nb6 {
    float xh, xl, yh, yl, zh, zl;
    float sx, sy, sz;  // 0.5 (central) or 1.0 (one-sided)
};

VK_D Nb6 load_nb6(const float* __restrict__ d, int nx, int ny, int nz, int x, int y, int z) {
    // Unsigned 32-bit element indices (a volume holds < 2^31 voxels) so each
    // address is one wide multiply-add; clamped neighbours collapse onto the
    // voxel itself (one-sided differences, volume.py:259-263).
    const unsigned plane = (unsigned)nx * (unsigned)ny;
    const unsigned c = ((unsigned)z * (unsigned)ny + (unsigned)y) * (unsigned)nx + (unsigned)x;
    const unsigned hx = x < nx - 1, lx = x > 0;
    const unsigned hy = y < ny - 1 ? (unsigned)nx : 0u, ly = y > 0 ? (unsigned)nx : 0u;
    const unsigned hz = z < nz - 1 ? plane : 0u, lz = z > 0 ? plane : 0u;
    Nb6 n;
    n.xh = __ldg(d + (c + hx));
    n.xl = __ldg(d + (c - lx));
    n.yh = __ldg(d + (c + hy));
    n.yl = __ldg(d + (c - ly));
    n.zh = __ldg(d + (c + hz));
    n.zl = __ldg(d + (c - lz));
    n.sx = (hx & lx) ? 0.5f : 1.0f;
    n.sy = (hy && ly) ? 0.5f : 1.0f;
    n.sz = (hz && lz) ? 0.5f : 1.0f;
    return n;
}

// load_nb6 for a voxel with all six neighbours inside the volume (central
// differences on every axis); c is its linear index, plane = nx * ny.
VK_D Nb6 load_nb6_interior(const float* __restrict__ d, unsigned nx, unsigned plane, unsigned c) {
    Nb6 n;
    n.xh = __ldg(d + (c + 1u));
    n.xl = __ldg(d + (c - 1u));
    n.yh = __ldg(d + (c + nx));
    n.yl = __ldg(d + (c - nx));
    n.zh = __ldg(d + (c + plane));
    n.zl = __ldg(d + (c - plane));
    n.sx = n.sy = n.sz = 0.5f;
    return n;
}

// Every voxel of a keypoint's ball (offsets within +-r per axis) has all six
// neighbours inside the volume.
VK_HD bool ball_interior(int cx, int cy, int cz, int r, int nx, int ny, int nz) {
    return cx > r && cy > r && cz > r && cx + r + 1 < nx && cy + r + 1 < ny && cz + r + 1 < nz;
}

// Exact fp64 gradient from the loaded neighbours: the fp64 difference of two
// fp32 values is exact and the scale is a power of two.
VK_D void grad64(const Nb6& n, double& gx, double& gy, double& gz) {
    gx = dmul(dsub((double)n.xh, (double)n.xl), (double)n.sx);
    gy = dmul(dsub((double)n.yh, (double)n.yl), (double)n.sy);
    gz = dmul(dsub((double)n.zh, (double)n.zl), (double)n.sz);
}

// fp32 gradient: each component within u32 relative of the exact value.
VK_D void grad32(const Nb6& n, float& gx, float& gy, float& gz) {
    gx = fmul(__fsub_rn(n.xh, n.xl), n.sx);
    gy = fmul(__fsub_rn(n.yh, n.yl), n.sy);
    gz = fmul(__fsub_rn(n.zh, n.zl), n.sz);
}

// Does the reference vote for this voxel?  Its fp64 gradient is nonzero
// exactly when some neighbour pair differs (volume.py:244-264) -- also when the
// fp32 gradient rounds to zero (a one-subnormal-ulp difference halved).
VK_D bool grad_nonzero(const Nb6& n) { return n.xh != n.xl || n.yh != n.yl || n.zh != n.zl; }

constexpr float kMinSub = 1.40129846e-45f;  // 2^-149, the smallest positive fp32 subnormal
constexpr float kFltMin = 1.17549435e-38f;  // 2^-126, the smallest normal fp32

// Rare path of norm3_f32 (|v| < ~1.1e-19, where the fp32 squares underflow):
// the components are scaled by 2^64 first (exact: they are < 2^-63 here, so
// the scaled values are normal and small), the norm is taken with a correctly
// rounded sqrt and scaled back (exact unless the result is subnormal, then
// within 2^-150 absolute).
static __device__ __noinline__ float norm3_f32_tiny(float x, float y, float z) {
    const float k = 18446744073709551616.0f, ik = 5.42101086242752217e-20f;  // 2^64, 2^-64
    const float a = fmul(x, k), b = fmul(y, k), c = fmul(z, k);
    return fmul(__fsqrt_rn(fadd(fadd(fmul(a, a), fmul(b, b)), fmul(c, c))), ik);
}

// |v| in fp32: within 4 u32 relative of the exact Euclidean norm when the
// fp32 sum of squares is normal (it carries <= 3.5 u32, halved by the square
// root, plus the hardware sqrt.approx.f32 (MUFU.SQRT) error, <= 1.678 x 2^-24
// relative over all 2^31 - 2^23 - 1 positive finite fp32 inputs (exhaustive
// sweep on B200, scripts/micro/sqrt_approx_err.cu -> profiles/r02/
// sqrt_approx_sweep.txt: max 1.0001e-7 at x = 3.1166e-36): 1.75 + 1.678 < 4 u32);
// below that the squares would underflow (|v| ~ 1e-19 can
// give s == 0), so the rescaled rare path above takes over: everywhere the
// error is <= 4 u32 relative + 2^-150 absolute.
#ifndef VK_APPROX_SQRT
#define VK_APPROX_SQRT 1
#endif
VK_D float norm3_f32(float x, float y, float z) {
    const float s = fadd(fadd(fmul(x, x), fmul(y, y)), fmul(z, z));
    if (s < kFltMin) return norm3_f32_tiny(x, y, z);
#if VK_APPROX_SQRT
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(s));
    return r;
#else
    return __fsqrt_rn(s);
#endif
}

// The fast path's vote of a voxel the reference votes for (grad_nonzero):
// never 0, because the reference's fp64 vote of a nonzero gradient is
// positive and the certifications treat bins that are 0 in the fast sums as
// exactly empty in the reference too.  The clamp to 2^-149 (e.g. a tiny |g|
// times the window underflowing) moves a vote by less than kVoteAbs.
VK_D float nz_vote(float v) { return fmaxf(v, kMinSub); }

// Error bound of a fast fp32 vote against the reference's fp64 vote:
// relative 4 u32 for the norm (norm3_f32, valid for every |g| incl. tiny and
// subnormal ones), 1 u32 for the window cast, 1 u32 for the product, rounded
// up generously; absolute: subnormal rounding of the components, the norm, the
// product and the nz_vote clamp (each <= 2^-149 ~ 1.4e-45).
constexpr double kVoteRel = 1.0e-6;
constexpr double kVoteAbs = 1.0e-43;

// Unit roundoff of fp64 and a rigorous bound factor for recursive summation:
// |fl(sum) - sum| <= gamma_k * sum|x| with gamma_k = k u / (1 - k u).
constexpr double kU64 = 1.1102230246251565e-16;
VK_HD double gamma_k(double k) { return (k * kU64) / (1.0 - k * kU64); }

}  // namespace vk
