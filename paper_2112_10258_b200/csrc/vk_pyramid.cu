// vk_pyramid.cu -- separable 3-D Gaussian blur with fused DoG and 2x
// subsample epilogues, standalone subsample / difference, layout transposes.
//
// Reference: scalespace.py:45-109 (convolve_array, subsample_half) and
// scalespace.py:209-223 (build_dog_pyramid).
//
// Blur design (x-fastest volumes, one CTA = 32x32 (x,y) columns x a z-range):
//  * 2.5-D z streaming: every input plane z' (clamped = replicate padding) is
//    staged in shared memory with cp.async (double-buffered), x-pass'd into a
//    (32+2R) x 32 tile, y-pass'd into registers and pushed into a per-column
//    register ring of 2R+1 y-blurred planes; the z-pass of plane z'-R is then
//    a dot product over the ring.  Each level is read once from HBM (halo
//    re-reads hit L1/L2) and written once.
//  * Bit parity with numpy: products are rounded to fp32 and added in tap
//    order -R..+R (__fmul_rn/__fadd_rn, -fmad=false), pass order x, y, z.
//  * Epilogues on the freshly produced plane: DoG = src - dst (the finer level
//    minus the coarser one), and the ordered 2x2x2 mean of the handoff level
//    for the next octave (needs even tile origins and an even z start).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>

#include "vk_common.cuh"

namespace vk {

struct Taps {
    float w[VK_MAX_TAPS];
    float mz;  // -0.0f, a launch-time value (see prod2)
};

constexpr int kTX = 32;       // output tile width in x
constexpr int kTY = 32;       // output tile height in y
constexpr int kThreads = 256;
constexpr int kMaxRingR = 10; // streaming kernel covers radius 1..10

// Shared-memory geometry of the streaming blur for radius R.
//  * in_s: the clamped input plane, (kTY+2R) rows x (kTX+2R) columns, stored
//    as float2 row PAIRS ((row 2i, row 2i+1) at each column) so the x-pass
//    multiplies two rows with one packed FMUL2 from one aligned register pair.
//    Pitch COLSP (in float2) is 1 mod 16: the 4 row pairs x 4 segments of a
//    half-warp hit 16 distinct 8-byte bank pairs.  Two buffers.
//  * x_s: x-blurred rows, row-major, read by the y-pass as (x, x+1) pairs.
//    Two buffers.
template <int R>
struct BlurGeom {
    static constexpr int P = 2 * R + 1;
    static constexpr int ROWS = kTY + 2 * R;       // even
    static constexpr int RP = ROWS / 2;
    static constexpr int COLS = kTX + 2 * R;
    static constexpr int COLSP = ((COLS + 15) / 16) * 16 + 1;  // == 1 mod 16
    static constexpr int IN_F2 = RP * COLSP;         // float2 per staging buffer
    static constexpr int XS = kTX + 4;               // x_s pitch (floats)
    static constexpr int LROWS = (ROWS + 7) / 8;     // staging rows per warp
    static constexpr int SMEM = (2 * IN_F2 * 2 + 2 * ROWS * XS + ROWS) * 4;
};

// Two taps' products with one packed op and two running sums with one packed
// FADD2, each lane rounded exactly like the scalar fmul / fadd sequence.
// ptxas contracts a packed multiply feeding a packed add into FFMA2 even with
// --fmad=false and explicit .rn (scripts/micro: PTX mul.rn.f32x2 +
// add.rn.f32x2 -> SASS FFMA2), which would drop the product's rounding.  The
// product is therefore formed as FFMA2(w, v, mz) with mz = -0.0 passed at
// launch: w*v + (-0) rounds to exactly round(w*v) (also for +-0 products), and
// an FMA result feeding an add cannot be contracted further.
#ifndef VK_PACKED_SUMS
#define VK_PACKED_SUMS 0  // measured: no gain on B200 (the blur is FP-pipe bound, not issue bound)
#endif
VK_D float2 prod2(const Taps& taps, float w, float2 v) {
#if VK_PACKED_SUMS
    return __ffma2_rn(make_float2(w, w), v, make_float2(taps.mz, taps.mz));
#else
    return __fmul2_rn(make_float2(w, w), v);
#endif
}
VK_D void acc2(float2& a, float2 p) {
#if VK_PACKED_SUMS
    a = __fadd2_rn(a, p);
#else
    a.x = fadd(a.x, p.x);
    a.y = fadd(a.y, p.y);
#endif
}

// One arriving y-blurred plane (z') in the z-pass.  The accumulator ring holds
// the 2R+1 outputs z'-R .. z'+R in slots (phase + k) mod P; the arriving value
// is multiplied once per distinct tap distance d (the kernel is symmetric, so
// w[R-d] == w[R+d] and one product serves outputs z'-d and z'+d: the reference
// rounds the same product twice, bit for bit the same number).  Output z'+R
// starts (first tap: assignment), output z'-R receives its last tap and is
// returned.  Every output still receives its taps in order -R..+R.
template <int R, int C>
VK_D void z_arrive(float2 (&r0)[2 * R + 1], float2 (&r1)[2 * R + 1], float2 v0, float2 v1, const Taps& taps,
                   float2& o0, float2& o1) {
    constexpr int P = 2 * R + 1;
#pragma unroll
    for (int d = 0; d <= R; ++d) {
        const float w = taps.w[R + d];
        const float2 p0 = prod2(taps, w, v0), p1 = prod2(taps, w, v1);
        if (d == 0) {
            acc2(r0[C], p0);
            acc2(r1[C], p1);
        } else {
            const int up = (C + d) % P, dn = (C - d + P) % P;
            if (d == R) {
                r0[up] = p0;
                r1[up] = p1;
            } else {
                acc2(r0[up], p0);
                acc2(r1[up], p1);
            }
            acc2(r0[dn], p0);
            acc2(r1[dn], p1);
        }
    }
    o0 = r0[(C - R + P) % P];
    o1 = r1[(C - R + P) % P];
}

// Binary dispatch on the (CTA-uniform) ring phase so every ring index is a
// compile-time constant: the ring stays in registers and never moves.
template <int R, int LO, int HI>
VK_D void z_dispatch(int c, float2 (&r0)[2 * R + 1], float2 (&r1)[2 * R + 1], float2 v0, float2 v1,
                     const Taps& taps, float2& o0, float2& o1) {
    if constexpr (HI - LO == 1) {
        z_arrive<R, LO>(r0, r1, v0, v1, taps, o0, o1);
    } else {
        constexpr int MID = (LO + HI) / 2;
        if (c < MID) z_dispatch<R, LO, MID>(c, r0, r1, v0, v1, taps, o0, o1);
        else z_dispatch<R, MID, HI>(c, r0, r1, v0, v1, taps, o0, o1);
    }
}

// Single-ring variant (one float2 column pair per thread) for blur_z_kernel.
template <int R, int C>
VK_D float2 z_arrive1(float2 (&r0)[2 * R + 1], float2 v0, const Taps& taps) {
    constexpr int P = 2 * R + 1;
#pragma unroll
    for (int d = 0; d <= R; ++d) {
        const float w = taps.w[R + d];
        const float2 p0 = prod2(taps, w, v0);
        if (d == 0) {
            acc2(r0[C], p0);
        } else {
            const int up = (C + d) % P, dn = (C - d + P) % P;
            if (d == R) r0[up] = p0;
            else acc2(r0[up], p0);
            acc2(r0[dn], p0);
        }
    }
    return r0[(C - R + P) % P];
}

template <int R, int LO, int HI>
VK_D float2 z_dispatch1(int c, float2 (&r0)[2 * R + 1], float2 v0, const Taps& taps) {
    if constexpr (HI - LO == 1) {
        return z_arrive1<R, LO>(r0, v0, taps);
    } else {
        constexpr int MID = (LO + HI) / 2;
        if (c < MID) return z_dispatch1<R, LO, MID>(c, r0, v0, taps);
        return z_dispatch1<R, MID, HI>(c, r0, v0, taps);
    }
}

// Two consecutive arrivals per dispatch (phases C, C+1): halves the dispatch
// cost per plane in blur_z_kernel.
template <int R, int LO, int HI>
VK_D void z_dispatch2(int c, float2 (&r0)[2 * R + 1], float2 v0, float2 v1, const Taps& taps, float2& o0, float2& o1) {
    if constexpr (HI - LO == 1) {
        o0 = z_arrive1<R, LO>(r0, v0, taps);
        o1 = z_arrive1<R, (LO + 1) % (2 * R + 1)>(r0, v1, taps);
    } else {
        constexpr int MID = (LO + HI) / 2;
        if (c < MID) z_dispatch2<R, LO, MID>(c, r0, v0, v1, taps, o0, o1);
        else z_dispatch2<R, MID, HI>(c, r0, v0, v1, taps, o0, o1);
    }
}

// Radii >= 8 need more than 128 registers for the ring: one CTA per SM.
template <int R>
constexpr int blur_min_blocks() { return R >= 8 ? 1 : 2; }

// Streaming separable blur (x-fastest volumes): one CTA = a 32x32 (x, y)
// output tile x a z-range.  Per distinct input plane: cp.async staging
// (clamped = replicate padding), x-pass of (32+2R) rows, y-pass to 2x2
// outputs per thread, then the plane "arrives" in the z ring.  Planes outside
// [0, nz) are the clamped border plane: their x/y-passes are not recomputed,
// the same value just arrives again.  Epilogues on each finished output
// plane: level store, DoG = src - dst (finer minus coarser; the src values
// are prefetched a plane ahead), and the ordered 2x2x2 mean of the handoff
// level from the thread's own 2x2 (x, y) block and the previous plane (tile
// origins and z_start are even).
//
// One barrier per plane: the x-pass of plane q reads in_s[q&1] and writes
// x_s[q&1]; after the barrier the staging of plane q+2 into in_s[q&1] is
// issued and the y-pass reads x_s[q&1] while other threads may already run
// the x-pass of q+1 (other buffers).  Element offsets are 32-bit (the host
// checks nb * volume < 2^32).
template <int R>
__global__ void __launch_bounds__(kThreads, blur_min_blocks<R>())
blur3d_stream_kernel(const float* __restrict__ src, float* __restrict__ dst, float* __restrict__ dog,
                     float* __restrict__ half, int nx, int ny, int nz, int tz, int nzc, Taps taps) {
    using G = BlurGeom<R>;
    constexpr int P = G::P;
    extern __shared__ float4 smem4[];
    float2* in2 = reinterpret_cast<float2*>(smem4);
    float* x_s = reinterpret_cast<float*>(in2 + 2 * G::IN_F2);           // 2 buffers
    unsigned* roff_s = reinterpret_cast<unsigned*>(x_s + 2 * G::ROWS * G::XS);

    const int b = blockIdx.z / nzc;
    const int zc = blockIdx.z - b * nzc;
    const int z_start = zc * tz;
    const int z_end = min(nz, z_start + tz);
    const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
    const unsigned plane = (unsigned)nx * (unsigned)ny;
    const unsigned vbase = (unsigned)b * plane * (unsigned)nz;  // element offset of volume b
    const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;

    // Staging: warp wy loads rows wy + 8k, lane loads columns lane and
    // lane + 32; smem float index of (row r, column c) is
    // ((r>>1)*COLSP + c)*2 + (r&1).  Clamped row offsets live in shared
    // memory (kept out of registers: the z ring needs them).
    const unsigned cx0 = (unsigned)clampi(x0 - R + lane, 0, nx - 1);
    const unsigned cx1 = (unsigned)clampi(x0 - R + lane + 32, 0, nx - 1);
    const int sbase = ((wy >> 1) * G::COLSP + lane) * 2 + (wy & 1);
    for (int r = tid; r < G::ROWS; r += kThreads) roff_s[r] = vbase + (unsigned)clampi(y0 - R + r, 0, ny - 1) * (unsigned)nx;
    __syncthreads();

    auto load_plane = [&](int q, int buf) {
        const unsigned qoff = (unsigned)q * plane;
        float* d = reinterpret_cast<float*>(in2 + buf * G::IN_F2) + sbase;
#pragma unroll
        for (int k = 0; k < G::LROWS; ++k) {
            if (wy + 8 * k < G::ROWS) {
                const unsigned ro = roff_s[wy + 8 * k] + qoff;
                cp_async4(d + k * 8 * G::COLSP, src + (ro + cx0));
                if (lane + 32 < G::COLS) cp_async4(d + k * 8 * G::COLSP + 64, src + (ro + cx1));
            }
        }
        cp_async_commit();
    };

    float2 r0[P], r1[P];
#pragma unroll
    for (int t = 0; t < P; ++t) r0[t] = r1[t] = make_float2(0.f, 0.f);
    float2 pv0 = make_float2(0.f, 0.f), pv1 = make_float2(0.f, 0.f);

    // x-pass role: lane -> (segment xsg = lane / 4 of 8, row pair xrp = warp * 4 + lane % 4)
    const int xsg = lane >> 2, xrp = wy * 4 + (lane & 3);
    // y-pass / z / epilogue role: column pair cp, row pair yp (2x2 outputs)
    const int cp = tid & 15, yp = tid >> 4;
    const int gx = x0 + 2 * cp, gy = y0 + 2 * yp;
    const bool okx0 = gx < nx, okx1 = gx + 1 < nx, oky0 = gy < ny, oky1 = gy + 1 < ny;
    const unsigned e00 = vbase + (unsigned)min(gy, ny - 1) * (unsigned)nx + (unsigned)min(gx, nx - 1);
    const unsigned rowst = oky1 ? (unsigned)nx : 0u;  // clamped: in-bounds dummy reads only
    const unsigned colst = okx1 ? 1u : 0u;

    const int za = z_start - R, zb = z_end - 1 + R;  // arriving planes (unclamped)
    const int qlo = max(0, za), qhi = min(nz - 1, zb);
    int a = 0, c = 0;
    load_plane(qlo, 0);
    cp_async_wait<0>();
    __syncthreads();
    if (qlo < qhi) load_plane(qlo + 1, 1);
    for (int q = qlo; q <= qhi; ++q) {
        const int it = q - qlo;
        const int reps = 1 + (q == qlo ? qlo - za : 0) + (q == qhi ? zb - qhi : 0);
        // Prefetch the DoG sources of the first output this plane completes.
        float s00 = 0.f, s01 = 0.f, s10 = 0.f, s11 = 0.f;
        const int zo_first = z_start + a - 2 * R;
        if (dog != nullptr && a >= 2 * R) {
            const float* sv = src + (e00 + (unsigned)zo_first * plane);
            s00 = __ldg(sv);
            s01 = __ldg(sv + colst);
            s10 = __ldg(sv + rowst);
            s11 = __ldg(sv + rowst + colst);
        }
        // ---- x-pass: 2 rows x 4 outputs per thread, inputs streamed ----
        float* xs = x_s + (it & 1) * G::ROWS * G::XS;
        if (xrp < G::RP) {
            const float2* row = in2 + (it & 1) * G::IN_F2 + xrp * G::COLSP + 4 * xsg;
            float2 acc[4];
#pragma unroll
            for (int i = 0; i < 4 + 2 * R; ++i) {
                const float2 v = row[i];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int t = i - k;
                    if (t < 0 || t > 2 * R) continue;
                    const int dd = t < R ? R - t : t - R;
                    const float w = taps.w[R + dd];
                    const float2 p = prod2(taps, w, v);
                    if (t == 0) acc[k] = p;
                    else acc2(acc[k], p);
                }
            }
            *reinterpret_cast<float4*>(xs + (2 * xrp) * G::XS + 4 * xsg) = make_float4(acc[0].x, acc[1].x, acc[2].x, acc[3].x);
            *reinterpret_cast<float4*>(xs + (2 * xrp + 1) * G::XS + 4 * xsg) = make_float4(acc[0].y, acc[1].y, acc[2].y, acc[3].y);
        }
        cp_async_wait<0>();  // plane q+1 staged (this thread's part)
        __syncthreads();
        if (q + 2 <= qhi) load_plane(q + 2, it & 1);
        // ---- y-pass: rows 2yp, 2yp+1 x columns (2cp, 2cp+1) ----
        float2 v0, v1;
        {
            const float* col = xs + (2 * yp) * G::XS + 2 * cp;
#pragma unroll
            for (int i = 0; i < 2 + 2 * R; ++i) {
                const float2 v = *reinterpret_cast<const float2*>(col + i * G::XS);
                if (i <= 2 * R) {
                    const int dd = i < R ? R - i : i - R;
                    const float w = taps.w[R + dd];
                    const float2 p = prod2(taps, w, v);
                    if (i == 0) v0 = p;
                    else acc2(v0, p);
                }
                if (i >= 1) {
                    const int t = i - 1;
                    const int dd = t < R ? R - t : t - R;
                    const float w = taps.w[R + dd];
                    const float2 p = prod2(taps, w, v);
                    if (t == 0) v1 = p;
                    else acc2(v1, p);
                }
            }
        }
        // ---- z-pass: the plane arrives once, or repeatedly at clamped borders ----
        for (int rep = 0; rep < reps; ++rep) {
            float2 o0, o1;
            z_dispatch<R, 0, P>(c, r0, r1, v0, v1, taps, o0, o1);
            if (a >= 2 * R) {
                const int zo = z_start + a - 2 * R;
                const unsigned eo = e00 + (unsigned)zo * plane;
                if (dog != nullptr && rep > 0) {  // later outputs of a border plane
                    const float* sv = src + eo;
                    s00 = __ldg(sv);
                    s01 = __ldg(sv + colst);
                    s10 = __ldg(sv + rowst);
                    s11 = __ldg(sv + rowst + colst);
                }
                float* dv = dst + eo;
                if (oky0) {
                    if (okx0) dv[0] = o0.x;
                    if (okx1) dv[1] = o0.y;
                }
                if (oky1) {
                    if (okx0) dv[nx] = o1.x;
                    if (okx1) dv[nx + 1] = o1.y;
                }
                if (dog != nullptr) {
                    float* gv = dog + eo;
                    if (oky0) {
                        if (okx0) gv[0] = __fsub_rn(s00, o0.x);
                        if (okx1) gv[1] = __fsub_rn(s01, o0.y);
                    }
                    if (oky1) {
                        if (okx0) gv[nx] = __fsub_rn(s10, o1.x);
                        if (okx1) gv[nx + 1] = __fsub_rn(s11, o1.y);
                    }
                }
                if (half != nullptr && (zo & 1)) {
                    const int hnx = nx >> 1, hny = ny >> 1, hnz = nz >> 1;
                    const int hx = gx >> 1, hy = gy >> 1, hz = zo >> 1;
                    if (hx < hnx && hy < hny && hz < hnz) {
                        // (dx, dy, dz) order of scalespace.py:101-107, then /8.
                        float sm = pv0.x;
                        sm = fadd(sm, o0.x);
                        sm = fadd(sm, pv1.x);
                        sm = fadd(sm, o1.x);
                        sm = fadd(sm, pv0.y);
                        sm = fadd(sm, o0.y);
                        sm = fadd(sm, pv1.y);
                        sm = fadd(sm, o1.y);
                        half[(((long long)b * hnz + hz) * hny + hy) * hnx + hx] = fmul(sm, 0.125f);
                    }
                }
                pv0 = o0;
                pv1 = o1;
            }
            ++a;
            c = (c + 1 == P) ? 0 : c + 1;
        }
    }
}

// ---------------------------------------------------------------------------
// Split blur: an (x, y) pass kernel writing an intermediate level, then a z
// pass kernel with the fused epilogues.  Same arithmetic as above (x, then y,
// then z; every product rounded, sums in tap order; the z pass in accumulator
// form with one product per tap distance), but two simple kernels: no z ring
// in the (x, y) kernel (short-lived CTAs, one plane each, high occupancy) and
// no shared memory or barriers in the z kernel (one column pair per thread,
// coalesced loads).  The intermediate costs 8 more HBM bytes per voxel; both
// kernels then run near their own roofline.
constexpr int kXyTX = 32;  // (x, y) tile of the xy kernel: 32 x TY (TY = 64, 96 or 176)

template <int R, int TY>
struct XyGeom {
    static constexpr int YR = TY / 16;                // y-pass rows per thread (16 row groups)
    static constexpr int ROWS = TY + 2 * R;           // even
    static constexpr int RP = ROWS / 2;
    static constexpr int COLS = kXyTX + 2 * R;
    static constexpr int COLSP = ((COLS + 15) / 16) * 16 + 1;
    static constexpr int IN_F2 = (RP * COLSP + 1) & ~1;  // even: x_s stays 16-byte aligned
    static constexpr int XS = kXyTX + 4;
    static constexpr int SMEM = (IN_F2 * 2 + ROWS * XS + ROWS) * 4;
    static constexpr int ITEMS = RP * 4;               // x-pass items: row pair x 8-output segment
};

template <int R, int TY>
__global__ void __launch_bounds__(kThreads, 4)
blur_xy_kernel(const float* __restrict__ src, float* __restrict__ tmp, int tp, int nx, int ny, int nz, Taps taps,
               const float* __restrict__ prev, float* __restrict__ pdog) {
    using G = XyGeom<R, TY>;
    extern __shared__ float4 smem4[];
    float2* in2 = reinterpret_cast<float2*>(smem4);
    float* x_s = reinterpret_cast<float*>(in2 + G::IN_F2);
    unsigned* roff_s = reinterpret_cast<unsigned*>(x_s + G::ROWS * G::XS);
    const int bz = blockIdx.z;  // b * nz + z
    const int x0 = blockIdx.x * kXyTX, y0 = blockIdx.y * TY;
    const unsigned plane = (unsigned)nx * (unsigned)ny;
    const unsigned pbase = (unsigned)bz * plane;
    const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;
    for (int r = tid; r < G::ROWS; r += kThreads) roff_s[r] = pbase + (unsigned)clampi(y0 - R + r, 0, ny - 1) * (unsigned)nx;
    __syncthreads();
    // Stage the clamped plane tile into the row-pair interleaved layout: one
    // warp instruction copies 16 columns x a row pair, lane l taking column
    // l/2 of row 2*rp + (l&1), so the 32 lanes write 32 consecutive floats
    // (conflict-free); clamped column offsets are per-thread constants.
    {
        constexpr int NCH = (G::COLS + 15) / 16;
        const int sdr = lane & 1, sdc = lane >> 1;
        unsigned cx[NCH];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) cx[ch] = (unsigned)clampi(x0 - R + 16 * ch + sdc, 0, nx - 1);
        float* d = reinterpret_cast<float*>(in2) + lane;
#pragma unroll 2
        for (int rp = wy; rp < G::RP; rp += 8) {
            const unsigned ro = roff_s[2 * rp + sdr];
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch)
                if (16 * ch + sdc < G::COLS) cp_async4(d + (rp * G::COLSP + 16 * ch) * 2, src + (ro + cx[ch]));
        }
        cp_async_commit();
        cp_async_wait<0>();
    }
    __syncthreads();
    if (prev != nullptr) {  // DoG of the previous pair on the tile core: prev - src (staged, intact)
        const float* inf = reinterpret_cast<const float*>(in2);
        for (int e = tid; e < kXyTX * TY; e += kThreads) {
            const int cx = e & (kXyTX - 1), cy = e / kXyTX;
            const int x = x0 + cx, y = y0 + cy;
            if (x < nx && y < ny) {
                const int r = cy + R, col = cx + R;
                const unsigned gi = pbase + (unsigned)y * (unsigned)nx + (unsigned)x;
                pdog[gi] = __fsub_rn(__ldg(prev + gi), inf[((r >> 1) * G::COLSP + col) * 2 + (r & 1)]);
            }
        }
    }
    // x-pass: items (row pair, 8-output segment), 2 rows x 8 outputs each
    for (int it = tid; it < G::ITEMS; it += kThreads) {
        const int rp = it >> 2, sg = it & 3;
        const float2* row = in2 + rp * G::COLSP + 8 * sg;
        float2 acc[8];
#pragma unroll
        for (int i = 0; i < 8 + 2 * R; ++i) {
            const float2 v = row[i];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int t = i - k;
                if (t < 0 || t > 2 * R) continue;
                const int dd = t < R ? R - t : t - R;
                const float w = taps.w[R + dd];
                const float2 pr = prod2(taps, w, v);
                if (t == 0) acc[k] = pr;
                else acc2(acc[k], pr);
            }
        }
        float4* xa = reinterpret_cast<float4*>(x_s + (2 * rp) * G::XS + 8 * sg);
        float4* xb = reinterpret_cast<float4*>(x_s + (2 * rp + 1) * G::XS + 8 * sg);
        xa[0] = make_float4(acc[0].x, acc[1].x, acc[2].x, acc[3].x);
        xa[1] = make_float4(acc[4].x, acc[5].x, acc[6].x, acc[7].x);
        xb[0] = make_float4(acc[0].y, acc[1].y, acc[2].y, acc[3].y);
        xb[1] = make_float4(acc[4].y, acc[5].y, acc[6].y, acc[7].y);
    }
    __syncthreads();
    // y-pass: column pair cp (16), row group yq (16): 2 x YR outputs per thread
    constexpr int YR = G::YR;
    const int cp = tid & 15, yq = tid >> 4;
    const float* col = x_s + (YR * yq) * G::XS + 2 * cp;
    float2 o[YR];
#pragma unroll
    for (int i = 0; i < YR + 2 * R; ++i) {
        const float2 v = *reinterpret_cast<const float2*>(col + i * G::XS);
#pragma unroll
        for (int k = 0; k < YR; ++k) {
            const int t = i - k;
            if (t < 0 || t > 2 * R) continue;
            const int dd = t < R ? R - t : t - R;
            const float w = taps.w[R + dd];
            const float2 pr = prod2(taps, w, v);
            if (t == 0) o[k] = pr;
            else acc2(o[k], pr);
        }
    }
    const int gx = x0 + 2 * cp;
#pragma unroll
    for (int k = 0; k < YR; ++k) {
        const int gy = y0 + YR * yq + k;
        if (gy < ny) {
            float* t = tmp + ((unsigned)bz * (unsigned)tp * (unsigned)ny + (unsigned)gy * (unsigned)tp + (unsigned)gx);
            if (gx < tp) t[0] = gx < nx ? o[k].x : 0.f;  // pad columns [nx, tp) hold zeros
            if (gx + 1 < tp) t[1] = gx + 1 < nx ? o[k].y : 0.f;
        }
    }
}

// ---------------------------------------------------------------------------
// Whole-plane (x, y) pass with register rings (default split path).
//
// One CTA = one (volume, z) plane.  The plane is staged into shared memory
// with ONE bulk asynchronous copy (cp.async.bulk, TMA engine, completion on an
// mbarrier) of its 16-byte-aligned byte superset: rows keep the global pitch
// nx, no pitched level layout needed.  Then
//  * x-pass: thread t walks row t along x with a ring of 2R+1 accumulators in
//    registers (outputs x-R .. x+R in flight): each arriving value is
//    multiplied once per tap distance (R+1 products, shared by the symmetric
//    taps) and added into the 2R outputs that use it, in tap order -- the
//    minimum fp32 work for bit parity (R+1 products + 2R adds per output, vs
//    ~19.5 + 20 at R = 10 for the register-blocked tile kernel).  Results are
//    written back in place (an output is complete R arrivals after its input
//    position was read, and no later arrival reads it).
//  * y-pass: thread t walks column t along y with the same ring and writes the
//    (x, y)-blurred values straight to the intermediate (lanes = consecutive
//    x: coalesced stores, conflict-free shared reads).
// Ring indices are compile-time constants: arrivals run in chunks of 2R+1
// with the phase unrolled, the tail by a uniform compile-time chain.
template <int R, int C>
VK_D float ring_arrive(float (&r)[2 * R + 1], float v, const Taps& taps) {
    constexpr int P = 2 * R + 1;
#pragma unroll
    for (int d = 0; d <= R; ++d) {
        const float p = fmul(taps.w[R + d], v);
        if (d == 0) {
            r[C] = fadd(r[C], p);
        } else {
            const int up = (C + d) % P, dn = (C - d + P) % P;
            if (d == R) r[up] = p;
            else r[up] = fadd(r[up], p);
            r[dn] = fadd(r[dn], p);
        }
    }
    return r[(C - R + P) % P];
}

// Arrivals k0 + C, ... up to the chunk end (FULL) or `left` arrivals.  SAFE:
// every arrival of the chunk has an unclamped prefetch position and a valid
// output (no clamps, no store predicate).  The line accessor provides
// at(k0, j) = value at position k0 + j - R (clamped unless SAFE) and
// put(k0, j, v) = store of output k0 + j - 2R; with a per-chunk base and a
// compile-time j both become one shared-memory / global access.
template <int R, int C, bool FULL, bool SAFE, class Line>
VK_D void ring_steps(float (&r)[2 * R + 1], int k0, int left, Line& ln, const Taps& taps, float (&pf)[2]) {
    constexpr int P = 2 * R + 1;
    if constexpr (C < P) {
        if (FULL || C < left) {
            const float v = pf[0];  // two arrivals of load lead (a shifting pair: P is odd)
            pf[0] = pf[1];
            pf[1] = ln.template at<SAFE>(k0, C + 2);
            const float o = ring_arrive<R, C>(r, v, taps);
            if (SAFE || k0 + C >= 2 * R) ln.put(k0, C, o);
            ring_steps<R, C + 1, FULL, SAFE>(r, k0, left, ln, taps, pf);
        }
    }
}

// One line of n values: arrival k (k = 0 .. n+2R-1) brings the value at
// position clamp(k - R, 0, n - 1) (replicate padding, scalespace.py:45-92);
// output o = k - 2R is complete after arrival k.
template <int R, class Line>
VK_D void ring_line(int n, Line& ln, const Taps& taps) {
    constexpr int P = 2 * R + 1;
    float r[P];
#pragma unroll
    for (int t = 0; t < P; ++t) r[t] = 0.f;
    const int A = n + 2 * R;
    float pf[2] = {ln.template at<false>(0, 0), ln.template at<false>(0, 1)};
    int k0 = 0;
    // a chunk is SAFE when k0 >= 2R and its last prefetch position k0 + P + 1 - R <= n - 1
    for (; k0 + P <= A; k0 += P) {
        if (k0 >= 2 * R && k0 + P + 1 - R <= n - 1) ring_steps<R, 0, true, true>(r, k0, P, ln, taps, pf);
        else ring_steps<R, 0, true, false>(r, k0, P, ln, taps, pf);
    }
    if (k0 < A) ring_steps<R, 0, false, false>(r, k0, A - k0, ln, taps, pf);
}

// x-pass line: a row in shared memory, blurred in place.
struct RowLine {
    float* row;
    int n, R;
    template <bool SAFE>
    VK_D float at(int k0, int j) const {
        return SAFE ? row[k0 - R + j] : row[clampi(k0 + j - R, 0, n - 1)];
    }
    VK_D void put(int k0, int j, float v) const { row[k0 + j - 2 * R] = v; }
};

// y-pass line: a column of the shared plane (stride nx) -> the intermediate.
#ifndef VK_COL_RUNNING
#define VK_COL_RUNNING 1  // running load / store offsets (y pass: 5-6 address instructions per arrival -> 2)
#endif
struct ColLine {
    const float* col;
    float* out;
    int n, R;
    unsigned nx, tp;
#if VK_COL_RUNNING
    // at() is called for consecutive positions -R, -R+1, ... and put() for consecutive outputs 0, 1, ...:
    // the next load position's element offset and the next store's pointer advance by one stride per call
    const float* ip = col - R * (int)nx;
    template <bool SAFE>
    VK_D float at(int k0, int j) {
        const float v = SAFE ? *ip : col[(unsigned)clampi(k0 + j - R, 0, n - 1) * nx];
        ip += nx;
        return v;
    }
    VK_D void put(int, int, float v) {
        *out = v;
        out += tp;
    }
#else
    template <bool SAFE>
    VK_D float at(int k0, int j) const {
        return SAFE ? col[(unsigned)(k0 - R + j) * nx] : col[(unsigned)clampi(k0 + j - R, 0, n - 1) * nx];
    }
    VK_D void put(int k0, int j, float v) const { out[(unsigned)(k0 + j - 2 * R) * tp] = v; }
#endif
};

constexpr int kPlaneThreads = 192;
#ifndef VK_DOG_WARPS
#define VK_DOG_WARPS 4  // warps of blur_xy_plane_kernel computing the previous pair's DoG (2 -> 4: pyramid -5.5%: the DoG warps were the CTA's critical path)
#endif
constexpr int kDogThreads = 32 * VK_DOG_WARPS;

VK_D void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
VK_D void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
VK_D void mbar_wait(uint64_t* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
VK_D void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
VK_D void bulk_g2s(void* smem, const void* gmem, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            (unsigned)__cvta_generic_to_shared(smem)),
        "l"(gmem), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
        : "memory");
}

template <int R>
__global__ void __launch_bounds__(kPlaneThreads + kDogThreads, 2)
blur_xy_plane_kernel(const float* __restrict__ src, float* __restrict__ tmp, int tp, int nx, int ny, Taps taps,
                     const float* __restrict__ prev, float* __restrict__ pdog) {
    extern __shared__ float4 smem4[];
    __shared__ uint64_t bar;
    const int tid = threadIdx.x;
    const unsigned plane = (unsigned)nx * (unsigned)ny;
    const float* g = src + (size_t)blockIdx.x * plane;  // plane (b * nz + z)
    const uintptr_t ga = reinterpret_cast<uintptr_t>(g);
    const uintptr_t a0 = ga & ~(uintptr_t)15;
    const unsigned bytes = (unsigned)(((ga + 4ull * plane) - a0 + 15) & ~(uintptr_t)15);
    float* s = reinterpret_cast<float*>(smem4) + (ga - a0) / 4;  // element (0, 0) of the staged plane
    if (tid == 0) {
        mbar_init(&bar, 1);
        mbar_expect_tx(&bar, bytes);
        bulk_g2s(smem4, reinterpret_cast<const void*>(a0), bytes, &bar);
    }
    __syncthreads();  // barrier initialised before anyone waits on it
    if (tid >= kPlaneThreads) {
        // VK_DOG_WARPS DoG warps (launched only with prev): the previous pair's difference prev - src over the
        // contiguous plane, read from global (src is L2-hot: the bulk copy just streamed it), concurrent
        // with the x / y passes of the other six warps
        const size_t pb = (size_t)blockIdx.x * plane;
        const int w = tid - kPlaneThreads;
        constexpr int NW = kDogThreads, U = 8;
        if (((plane & 1) | ((reinterpret_cast<uintptr_t>(prev + pb) | reinterpret_cast<uintptr_t>(pdog + pb) |
                             reinterpret_cast<uintptr_t>(g)) & 7)) == 0) {
            const float2* pv2 = reinterpret_cast<const float2*>(prev + pb);
            const float2* sv2 = reinterpret_cast<const float2*>(g);
            float2* pd2 = reinterpret_cast<float2*>(pdog + pb);
            const unsigned n2 = plane / 2;
            for (unsigned i0 = w; i0 < n2; i0 += NW * U) {
                float2 a[U], c[U];
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const unsigned i = i0 + j * NW;
                    if (i < n2) {
                        a[j] = __ldg(pv2 + i);
                        c[j] = __ldg(sv2 + i);
                    }
                }
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const unsigned i = i0 + j * NW;
                    if (i < n2) pd2[i] = make_float2(__fsub_rn(a[j].x, c[j].x), __fsub_rn(a[j].y, c[j].y));
                }
            }
        } else {
            for (unsigned i = w; i < plane; i += NW) pdog[pb + i] = __fsub_rn(__ldg(prev + pb + i), __ldg(g + i));
        }
        return;
    }
    mbar_wait(&bar, 0);
    if (tid < ny) {
        RowLine ln{s + tid * nx, nx, R};
        ring_line<R>(nx, ln, taps);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kPlaneThreads) : "memory");  // the pass warps only
    float* out = tmp + (size_t)blockIdx.x * (unsigned)tp * (unsigned)ny + tid;
    if (tid < nx) {
        ColLine ln{s + tid, out, ny, R, (unsigned)nx, (unsigned)tp};
        ring_line<R>(ny, ln, taps);
    } else if (tid < tp) {  // pad columns [nx, tp) of the pitched intermediate hold zeros
        for (int y = 0; y < ny; ++y) out[(unsigned)y * (unsigned)tp] = 0.f;
    }
}

// Persistent variant of blur_xy_plane_kernel (VK_XY_STREAM): one CTA per SM
// holds two independent plane groups (6 pass warps + one staged plane each)
// that take planes from a work counter.  Group 1 starts its first load only
// once group 0's first plane has landed, so the two run out of phase: one
// group's bulk copy streams while the other computes (two plane CTAs per SM
// start, load and compute in lockstep).  The DoG warps take planes from a
// second counter and run independently.  counters[0..1] are zero at launch
// (the launcher memsets them).
constexpr int kStreamDogThreads = 2 * kDogThreads;
template <int R>
__global__ void __launch_bounds__(2 * kPlaneThreads + kStreamDogThreads, 1)
blur_xy_stream_kernel(const float* __restrict__ src, float* __restrict__ tmp, int tp, int nx, int ny, int nplanes,
                      unsigned buf_floats, Taps taps, const float* __restrict__ prev, float* __restrict__ pdog,
                      unsigned* __restrict__ counters) {
    extern __shared__ float4 smem4[];
    __shared__ uint64_t bar[2];
    __shared__ int cur_plane[2];
    const unsigned plane = (unsigned)nx * (unsigned)ny;
    if (threadIdx.x >= 2 * kPlaneThreads) {
        // DoG warps: one plane per warp at a time, prev - src, read from global
        const int lane = threadIdx.x & 31;
        for (;;) {
            unsigned p = 0;
            if (lane == 0) p = atomicAdd(&counters[1], 1u);
            p = __shfl_sync(0xffffffffu, p, 0);
            if (p >= (unsigned)nplanes) break;
            const size_t pb = (size_t)p * plane;
            const float* g = src + pb;
            constexpr int U = 8;
            if (((plane & 1) | ((reinterpret_cast<uintptr_t>(prev + pb) | reinterpret_cast<uintptr_t>(pdog + pb) |
                                 reinterpret_cast<uintptr_t>(g)) & 7)) == 0) {
                const float2* pv2 = reinterpret_cast<const float2*>(prev + pb);
                const float2* sv2 = reinterpret_cast<const float2*>(g);
                float2* pd2 = reinterpret_cast<float2*>(pdog + pb);
                const unsigned n2 = plane / 2;
                for (unsigned i0 = lane; i0 < n2; i0 += 32 * U) {
                    float2 a[U], c[U];
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const unsigned i = i0 + j * 32;
                        if (i < n2) {
                            a[j] = __ldg(pv2 + i);
                            c[j] = __ldg(sv2 + i);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const unsigned i = i0 + j * 32;
                        if (i < n2) pd2[i] = make_float2(__fsub_rn(a[j].x, c[j].x), __fsub_rn(a[j].y, c[j].y));
                    }
                }
            } else {
                for (unsigned i = lane; i < plane; i += 32) pdog[pb + i] = __fsub_rn(__ldg(prev + pb + i), __ldg(g + i));
            }
        }
        return;
    }
    const int grp = threadIdx.x >= kPlaneThreads;
    const int tid = threadIdx.x - grp * kPlaneThreads;
    float* buf = reinterpret_cast<float*>(smem4) + (size_t)grp * buf_floats;
    __shared__ uint64_t started;  // one phase: group 0's first plane has landed (or it had none)
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_init(&started, 1);
    }
    asm volatile("bar.sync 3, %0;" ::"n"(2 * kPlaneThreads) : "memory");  // the pass warps of both groups
    // named barriers 1 / 2: the two groups
    for (int it = 0;; ++it) {
        if (tid == 0) {
            if (grp == 1 && it == 0) mbar_wait(&started, 0);  // start out of phase with group 0
            const int p = (int)atomicAdd(&counters[0], 1u);
            cur_plane[grp] = p;
            if (p < nplanes) {
                const uintptr_t ga = reinterpret_cast<uintptr_t>(src + (size_t)p * plane);
                const uintptr_t a0 = ga & ~(uintptr_t)15;
                const unsigned bytes = (unsigned)(((ga + 4ull * plane) - a0 + 15) & ~(uintptr_t)15);
                // the previous plane's generic-proxy accesses of the buffer precede the async-proxy write
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&bar[grp], bytes);
                bulk_g2s(buf, reinterpret_cast<const void*>(a0), bytes, &bar[grp]);
            }
        }
        if (grp == 0) asm volatile("bar.sync 1, %0;" ::"n"(kPlaneThreads) : "memory");
        else asm volatile("bar.sync 2, %0;" ::"n"(kPlaneThreads) : "memory");
        const int p = cur_plane[grp];
        if (p >= nplanes) {
            if (grp == 0 && tid == 0 && it == 0) mbar_arrive(&started);
            break;
        }
        const uintptr_t ga = reinterpret_cast<uintptr_t>(src + (size_t)p * plane);
        float* s = buf + (ga & 15) / 4;
        mbar_wait(&bar[grp], (unsigned)it & 1u);
        if (grp == 0 && tid == 0 && it == 0) mbar_arrive(&started);
        if (tid < ny) {
            RowLine ln{s + tid * nx, nx, R};
            ring_line<R>(nx, ln, taps);
        }
        if (grp == 0) asm volatile("bar.sync 1, %0;" ::"n"(kPlaneThreads) : "memory");
        else asm volatile("bar.sync 2, %0;" ::"n"(kPlaneThreads) : "memory");
        float* out = tmp + (size_t)p * (unsigned)tp * (unsigned)ny + tid;
        if (tid < nx) {
            ColLine ln{s + tid, out, ny, R, (unsigned)nx, (unsigned)tp};
            ring_line<R>(ny, ln, taps);
        } else if (tid < tp) {
            for (int y = 0; y < ny; ++y) out[(unsigned)y * (unsigned)tp] = 0.f;
        }
        if (grp == 0) asm volatile("bar.sync 1, %0;" ::"n"(kPlaneThreads) : "memory");
        else asm volatile("bar.sync 2, %0;" ::"n"(kPlaneThreads) : "memory");
    }
}

// z pass over the (x, y)-blurred intermediate: thread = column pair
// (gx, gx+1) of row gy; warp = 16 column pairs x rows (y, y+1) so the 2x2x2
// subsample block of a thread is completed by lane ^ 16.  Planes outside
// [0, nz) are the clamped border plane (re-read, L1-resident).
template <int R>
__global__ void __launch_bounds__(kThreads, 3)
blur_z_kernel(const float* __restrict__ tmp, int tp, const float* __restrict__ src, float* __restrict__ dst,
              float* __restrict__ dog, float* __restrict__ half, int nx, int ny, int nz, int tz, int nzc, Taps taps) {
    constexpr int P = 2 * R + 1;
    const int b = blockIdx.z / nzc;
    const int zc = blockIdx.z - b * nzc;
    const int z_start = zc * tz;
    const int z_end = min(nz, z_start + tz);
    const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;
    const int gx = blockIdx.x * 32 + 2 * (lane & 15);
    const int gy = blockIdx.y * 16 + 2 * wy + (lane >> 4);
    const bool okx0 = gx < nx, okx1 = gx + 1 < nx, oky = gy < ny;
    const unsigned plane = (unsigned)nx * (unsigned)ny;
    const unsigned vbase = (unsigned)b * plane * (unsigned)nz;
    const unsigned e0 = vbase + (unsigned)min(gy, ny - 1) * (unsigned)nx + (unsigned)min(gx, nx - 1);
    const unsigned cst = okx1 ? 1u : 0u;
    const unsigned tplane = (unsigned)tp * (unsigned)ny;
    const unsigned t0 = (unsigned)b * tplane * (unsigned)nz + (unsigned)min(gy, ny - 1) * (unsigned)tp +
                        (unsigned)min(gx, nx - 1);
    float2 r0[P];
#pragma unroll
    for (int t = 0; t < P; ++t) r0[t] = make_float2(0.f, 0.f);
    float2 pv = make_float2(0.f, 0.f);
    const int za = z_start - R, zb = z_end - 1 + R;
    auto ld = [&](const float* base, int zp) {
        const float* t = base + (e0 + (unsigned)clampi(zp, 0, nz - 1) * plane);
        return make_float2(__ldg(t), __ldg(t + cst));
    };
    auto ldt = [&](int zp) {
        const float* t = tmp + (t0 + (unsigned)clampi(zp, 0, nz - 1) * tplane);
        return make_float2(__ldg(t), __ldg(t + cst));
    };
    // Two arrivals per step (the arrival count tz + 2R is even); loads run two
    // steps ahead for the intermediate and one step ahead for the DoG source.
    float2 q0 = ldt(za), q1 = ldt(za + 1), q2 = ldt(za + 2), q3 = ldt(za + 3);
    const bool want_src = dog != nullptr;
    float2 s0 = want_src ? ld(src, z_start) : make_float2(0.f, 0.f);
    float2 s1 = want_src ? ld(src, z_start + 1) : make_float2(0.f, 0.f);
    int c = 0;
    auto epilogue = [&](int zo, float2 o, float2 sv) {
        float* dv = dst + (e0 + (unsigned)zo * plane);
        if (oky) {
            if (okx0) dv[0] = o.x;
            if (okx1) dv[1] = o.y;
        }
        if (want_src && oky) {
            float* gv = dog + (e0 + (unsigned)zo * plane);
            if (okx0) gv[0] = __fsub_rn(sv.x, o.x);
            if (okx1) gv[1] = __fsub_rn(sv.y, o.y);
        }
        if (half != nullptr) {
            // (dx, dy, dz) order of scalespace.py:101-107: this thread holds
            // rows y (lanes 0-15) or y+1 (lanes 16-31) of planes zo-1 (pv), zo (o)
            const float2 qv = make_float2(__shfl_xor_sync(0xffffffffu, pv.x, 16), __shfl_xor_sync(0xffffffffu, pv.y, 16));
            const float2 qo = make_float2(__shfl_xor_sync(0xffffffffu, o.x, 16), __shfl_xor_sync(0xffffffffu, o.y, 16));
            const int hnx = nx >> 1, hny = ny >> 1, hnz = nz >> 1;
            const int hx = gx >> 1, hy = gy >> 1, hz = zo >> 1;
            if ((zo & 1) && lane < 16 && hx < hnx && hy < hny && hz < hnz) {
                float sm = pv.x;
                sm = fadd(sm, o.x);
                sm = fadd(sm, qv.x);
                sm = fadd(sm, qo.x);
                sm = fadd(sm, pv.y);
                sm = fadd(sm, o.y);
                sm = fadd(sm, qv.y);
                sm = fadd(sm, qo.y);
                half[(((long long)b * hnz + hz) * hny + hy) * hnx + hx] = fmul(sm, 0.125f);
            }
        }
        pv = o;
    };
    for (int zp = za; zp <= zb; zp += 2) {
        const float2 v0 = q0, v1 = q1;
        q0 = q2;
        q1 = q3;
        if (zp + 4 <= zb) q2 = ldt(zp + 4);
        if (zp + 5 <= zb) q3 = ldt(zp + 5);
        const int zo = zp - R;  // outputs zo, zo + 1 (zo and z_start are even)
        const bool out = zo >= z_start;
        const float2 sv0 = s0, sv1 = s1;
        if (out && want_src) {
            if (zo + 2 < z_end) s0 = ld(src, zo + 2);
            if (zo + 3 < z_end) s1 = ld(src, zo + 3);
        }
        float2 o0, o1;
        z_dispatch2<R, 0, P>(c, r0, v0, v1, taps, o0, o1);
        c += 2;
        if (c >= P) c -= P;
        if (!out) continue;
        epilogue(zo, o0, sv0);
        if (zo + 1 < z_end) epilogue(zo + 1, o1, sv1);
    }
}

// ---------------------------------------------------------------------------
// z pass, four columns per thread (default).  The (x, y)-blurred intermediate
// is PITCHED (row pitch tp = nx rounded up to 4 floats, pad columns zero), so
// a thread's columns x0..x0+3 (x0 = 4 k) are one aligned 16-byte load per
// plane.  A warp is 8 such float4 columns x 4 rows: one plane of a warp is
// 4 x 128 contiguous bytes, and the y partner of the handoff subsample is
// lane ^ 8.  Same arithmetic as blur_z_kernel (accumulator ring, one rounded
// product per tap distance, adds in tap order); with PK the products are
// FFMA2(w, v, -0) and the sums FADD2 -- bit-identical per lane to the scalar
// fmul / fadd sequence, half the issue slots (the z pass is issue-bound, not
// FP-pipe bound: loads, addresses and epilogue stores are amortised over four
// columns as well).
constexpr int kZ4Threads = 128;

template <bool PK>
VK_D float2 prodk(const Taps& taps, float w, float2 v) {
    if constexpr (PK) return __ffma2_rn(make_float2(w, w), v, make_float2(taps.mz, taps.mz));
    else return __fmul2_rn(make_float2(w, w), v);
}
template <bool PK>
VK_D void acck(float2& a, float2 p) {
    if constexpr (PK) {
        a = __fadd2_rn(a, p);
    } else {
        a.x = fadd(a.x, p.x);
        a.y = fadd(a.y, p.y);
    }
}

template <int R, int C, bool PK>
VK_D void z4_arrive(float2 (&r0)[2 * R + 1], float2 (&r1)[2 * R + 1], float4 v, const Taps& taps, float4& o) {
    constexpr int P = 2 * R + 1;
    const float2 va = make_float2(v.x, v.y), vb = make_float2(v.z, v.w);
#pragma unroll
    for (int d = 0; d <= R; ++d) {
        const float w = taps.w[R + d];
        const float2 pa = prodk<PK>(taps, w, va), pb = prodk<PK>(taps, w, vb);
        if (d == 0) {
            acck<PK>(r0[C], pa);
            acck<PK>(r1[C], pb);
        } else {
            const int up = (C + d) % P, dn = (C - d + P) % P;
            if (d == R) {
                r0[up] = pa;
                r1[up] = pb;
            } else {
                acck<PK>(r0[up], pa);
                acck<PK>(r1[up], pb);
            }
            acck<PK>(r0[dn], pa);
            acck<PK>(r1[dn], pb);
        }
    }
    constexpr int OUT = (C - R + P) % P;
    o = make_float4(r0[OUT].x, r0[OUT].y, r1[OUT].x, r1[OUT].y);
}

template <int R, int LO, int HI, bool PK>
VK_D void z4_dispatch2(int c, float2 (&r0)[2 * R + 1], float2 (&r1)[2 * R + 1], float4 v0, float4 v1,
                       const Taps& taps, float4& o0, float4& o1) {
    if constexpr (HI - LO == 1) {
        z4_arrive<R, LO, PK>(r0, r1, v0, taps, o0);
        z4_arrive<R, (LO + 1) % (2 * R + 1), PK>(r0, r1, v1, taps, o1);
    } else {
        constexpr int MID = (LO + HI) / 2;
        if (c < MID) z4_dispatch2<R, LO, MID, PK>(c, r0, r1, v0, v1, taps, o0, o1);
        else z4_dispatch2<R, MID, HI, PK>(c, r0, r1, v0, v1, taps, o0, o1);
    }
}

template <int R>
constexpr int z4_min_blocks() { return R >= 8 ? 3 : 4; }

template <int R, bool HALF, bool PK>
__global__ void __launch_bounds__(kZ4Threads, z4_min_blocks<R>())
blur_z4_kernel(const float* __restrict__ tmp, int tp, const float* __restrict__ src, float* __restrict__ dst,
               float* __restrict__ dog, float* __restrict__ half, int nx, int ny, int nz, int tz, int nzc, Taps taps) {
    constexpr int P = 2 * R + 1;
    const int b = blockIdx.z / nzc;
    const int zc = blockIdx.z - b * nzc;
    const int z_start = zc * tz;
    const int z_end = min(nz, z_start + tz);
    const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;
    const int x0 = 4 * (blockIdx.x * 8 + (lane & 7));
    const int ry = lane >> 3;  // row within the warp's 4
    const int gy = blockIdx.y * 16 + 4 * wy + ry;
    const bool oky = gy < ny;
    const int nvalid = oky ? max(0, min(4, nx - x0)) : 0;  // stored columns of this thread
    const unsigned plane = (unsigned)nx * (unsigned)ny;
    const unsigned tplane = (unsigned)tp * (unsigned)ny;
    const int yc = min(gy, ny - 1);
    const unsigned t0 = (unsigned)b * tplane * (unsigned)nz + (unsigned)yc * (unsigned)tp + (unsigned)min(x0, tp - 4);
    const unsigned e0 = (unsigned)b * plane * (unsigned)nz + (unsigned)yc * (unsigned)nx + (unsigned)min(x0, nx - 1);
    float2 r0[P], r1[P];
#pragma unroll
    for (int t = 0; t < P; ++t) r0[t] = r1[t] = make_float2(0.f, 0.f);
    const int za = z_start - R, zb = z_end - 1 + R;
    auto ldt = [&](int zp) {
        return __ldg(reinterpret_cast<const float4*>(tmp + (t0 + (unsigned)clampi(zp, 0, nz - 1) * tplane)));
    };
    const bool want_src = dog != nullptr;
    auto lds = [&](int zp) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (want_src) {
            const float* t = src + (e0 + (unsigned)zp * plane);
            if (nvalid > 0) v.x = __ldg(t);
            if (nvalid > 1) v.y = __ldg(t + 1);
            if (nvalid > 2) v.z = __ldg(t + 2);
            if (nvalid > 3) v.w = __ldg(t + 3);
        }
        return v;
    };
    float4 q0 = ldt(za), q1 = ldt(za + 1), q2 = ldt(za + 2), q3 = ldt(za + 3);
    float4 s0 = lds(z_start), s1 = z_start + 1 < z_end ? lds(z_start + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 pv = make_float4(0.f, 0.f, 0.f, 0.f);
    int c = 0;
    auto epilogue = [&](int zo, float4 o, float4 sv) {
        float* dv = dst + (e0 + (unsigned)zo * plane);
        if (nvalid > 0) dv[0] = o.x;
        if (nvalid > 1) dv[1] = o.y;
        if (nvalid > 2) dv[2] = o.z;
        if (nvalid > 3) dv[3] = o.w;
        if (want_src) {
            float* gv = dog + (e0 + (unsigned)zo * plane);
            if (nvalid > 0) gv[0] = __fsub_rn(sv.x, o.x);
            if (nvalid > 1) gv[1] = __fsub_rn(sv.y, o.y);
            if (nvalid > 2) gv[2] = __fsub_rn(sv.z, o.z);
            if (nvalid > 3) gv[3] = __fsub_rn(sv.w, o.w);
        }
        if constexpr (HALF) {
            // (dx, dy, dz) order of scalespace.py:101-107 for the column pairs
            // (x0, x0+1) and (x0+2, x0+3); rows y (even ry) and y+1 (lane ^ 8),
            // planes zo-1 (pv) and zo (o)
            float4 qv, qo;
            qv.x = __shfl_xor_sync(0xffffffffu, pv.x, 8);
            qv.y = __shfl_xor_sync(0xffffffffu, pv.y, 8);
            qv.z = __shfl_xor_sync(0xffffffffu, pv.z, 8);
            qv.w = __shfl_xor_sync(0xffffffffu, pv.w, 8);
            qo.x = __shfl_xor_sync(0xffffffffu, o.x, 8);
            qo.y = __shfl_xor_sync(0xffffffffu, o.y, 8);
            qo.z = __shfl_xor_sync(0xffffffffu, o.z, 8);
            qo.w = __shfl_xor_sync(0xffffffffu, o.w, 8);
            const int hnx = nx >> 1, hny = ny >> 1, hnz = nz >> 1;
            const int hy = gy >> 1, hz = zo >> 1;
            if ((zo & 1) && !(ry & 1) && hy < hny && hz < hnz) {
                float* hp = half + (((long long)b * hnz + hz) * hny + hy) * hnx;
                const int hx = x0 >> 1;
                if (hx < hnx) {
                    float sm = pv.x;
                    sm = fadd(sm, o.x);
                    sm = fadd(sm, qv.x);
                    sm = fadd(sm, qo.x);
                    sm = fadd(sm, pv.y);
                    sm = fadd(sm, o.y);
                    sm = fadd(sm, qv.y);
                    sm = fadd(sm, qo.y);
                    hp[hx] = fmul(sm, 0.125f);
                }
                if (hx + 1 < hnx) {
                    float sm = pv.z;
                    sm = fadd(sm, o.z);
                    sm = fadd(sm, qv.z);
                    sm = fadd(sm, qo.z);
                    sm = fadd(sm, pv.w);
                    sm = fadd(sm, o.w);
                    sm = fadd(sm, qv.w);
                    sm = fadd(sm, qo.w);
                    hp[hx + 1] = fmul(sm, 0.125f);
                }
            }
            pv = o;
        }
    };
    for (int zp = za; zp <= zb; zp += 2) {
        const float4 v0 = q0, v1 = q1;
        q0 = q2;
        q1 = q3;
        if (zp + 4 <= zb) q2 = ldt(zp + 4);
        if (zp + 5 <= zb) q3 = ldt(zp + 5);
        const int zo = zp - R;  // outputs zo, zo + 1 (zo and z_start are even)
        const bool out = zo >= z_start;
        const float4 sv0 = s0, sv1 = s1;
        if (out) {
            if (zo + 2 < z_end) s0 = lds(zo + 2);
            if (zo + 3 < z_end) s1 = lds(zo + 3);
        }
        float4 o0, o1;
        z4_dispatch2<R, 0, P, PK>(c, r0, r1, v0, v1, taps, o0, o1);
        c += 2;
        if (c >= P) c -= P;
        if (!out) continue;
        epilogue(zo, o0, sv0);
        if (zo + 1 < z_end) epilogue(zo + 1, o1, sv1);
    }
}

// ---------------------------------------------------------------------------
// z pass fed by the TMA engine (default).  Same thread layout and arithmetic
// as blur_z4_kernel (4 columns x 1 row per thread, warp = 8 float4 columns x
// 4 rows, CTA = 32 x 16 columns x a z-range), but no loads are issued by the
// math threads: a ring of kZtSlots shared-memory slots, each holding
//  * the 32 x 16 intermediate tile of one arriving plane, loaded by ONE
//    cp.async.bulk.tensor.3d (tensor map over the pitched intermediate:
//    dims (tp, ny, nb * nz); rows >= ny / columns >= tp are zero-filled, z
//    clamping = the plane coordinate we ask for), and
//  * the 16 source rows (the DoG minuend) of the output plane that arrival
//    completes (R planes behind), each a 1-D cp.async.bulk of the 16-byte
//    aligned superset of the row segment (levels keep the unpitched x-fastest
//    layout of the API),
// completing on the slot's mbarrier.  Warp 0 refills the two slots of a step
// right after every thread has copied them to registers, so kZtSlots - 2
// planes of loads are always in flight per CTA without holding registers.
#ifndef VK_ZT_SLOTS
#define VK_ZT_SLOTS 12  // 8 -> 12 (late round 2): pyramid -0.8%, step +0.2% (scripts/gpu_step_ab.sh)
#endif
#ifndef VK_ZT_SRC_TMA
#define VK_ZT_SRC_TMA 0  // 1: DoG source rows staged by 1-D bulk copies (measured slower: ~16 small copies per plane)
#endif
constexpr int kZtSlots = VK_ZT_SLOTS;
constexpr int kZtTmpFloats = 32 * 16;   // tmp tile floats per slot (2 KB)
constexpr int kZtSrcPitch = 40;         // floats per staged source row (<= 36 used)
constexpr int kZtSrcFloats = VK_ZT_SRC_TMA ? 16 * kZtSrcPitch : 0;  // (no staging slots unless used)
#ifndef VK_ZT_TSTORE
#define VK_ZT_TSTORE 0  // 1: warp-transposed row stores (measured slower: 214 vs 126 us at R = 10)
#endif
constexpr int kZtSmem = kZtSlots * (kZtTmpFloats + kZtSrcFloats) * 4 + 2 * kZtSlots * 8 + 4 * 128 * 4;

constexpr int kZtThreads = kZ4Threads + 32;  // 4 consumer (math) warps + 1 producer warp

template <int R>
constexpr int zt_min_blocks() { return 3; }


template <int R, bool HALF>
__global__ void __launch_bounds__(kZtThreads, zt_min_blocks<R>())
blur_zt_kernel(const __grid_constant__ CUtensorMap tmap, const float* __restrict__ src, float* __restrict__ dst,
               float* __restrict__ dog, float* __restrict__ half, int nx, int ny, int nz, int tz, int nzc, Taps taps) {
    constexpr int P = 2 * R + 1;
    extern __shared__ __align__(128) float4 zsm4[];
    float* tmp_s = reinterpret_cast<float*>(zsm4);
    float* src_s = tmp_s + kZtSlots * kZtTmpFloats;
    uint64_t* full = reinterpret_cast<uint64_t*>(src_s + kZtSlots * kZtSrcFloats);
    uint64_t* empty = full + kZtSlots;
    const int b = blockIdx.z / nzc;
    const int zc = blockIdx.z - b * nzc;
    const int z_start = zc * tz;
    const int z_end = min(nz, z_start + tz);
    const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;
    const int X0 = blockIdx.x * 32, Y0 = blockIdx.y * 16;
    const unsigned plane = (unsigned)nx * (unsigned)ny;
    const bool want_src = dog != nullptr;
    const int A = (z_end - z_start) + 2 * R;  // arrivals
    const int za = z_start - R;
    if (tid == 0) {
        for (int k = 0; k < kZtSlots; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], 4);
        }
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    }
    __syncthreads();
    if (wy == 4) {
        // producer warp: arrival a = tmp plane za + a and the source rows of output plane za + a - R
        for (int a = 0; a < A; ++a) {
            const int k = a % kZtSlots;
            if (a >= kZtSlots) mbar_wait(&empty[k], (unsigned)(a / kZtSlots - 1) & 1u);
            const int zp = za + a, zs = zp - R;
            const bool has_src = VK_ZT_SRC_TMA && want_src && zs >= z_start && zs < z_end;
            const int y = Y0 + lane;
            uintptr_t a0 = 0;
            unsigned sz = 0;
            if (has_src && lane < 16 && y < ny) {
                const uintptr_t st =
                    reinterpret_cast<uintptr_t>(src + ((size_t)(b * nz + zs) * plane + (size_t)y * nx + X0));
                const uintptr_t en = st + 4u * (unsigned)min(32, nx - X0);
                a0 = st & ~(uintptr_t)15;
                sz = (unsigned)(((en + 15) & ~(uintptr_t)15) - a0);
            }
            unsigned tot = sz;
#pragma unroll
            for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
            if (lane == 0) {
                mbar_expect_tx(&full[k], tot + kZtTmpFloats * 4);
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                    "%4}], [%5];" ::"r"((unsigned)__cvta_generic_to_shared(tmp_s + k * kZtTmpFloats)),
                    "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(X0), "r"(Y0), "r"(b * nz + clampi(zp, 0, nz - 1)),
                    "r"((unsigned)__cvta_generic_to_shared(&full[k]))
                    : "memory");
            }
            __syncwarp();
            if (sz)
                bulk_g2s(src_s + k * kZtSrcFloats + lane * kZtSrcPitch, reinterpret_cast<const void*>(a0), sz,
                         &full[k]);
        }
        return;
    }
    const int xl = 4 * (lane & 7), ry = lane >> 3, yl = 4 * wy + ry;
    const int x0 = X0 + xl, gy = Y0 + yl;
    const bool oky = gy < ny;
    const int nvalid = oky ? max(0, min(4, nx - x0)) : 0;
    const int yc = min(gy, ny - 1);
    const unsigned e0 = (unsigned)b * plane * (unsigned)nz + (unsigned)yc * (unsigned)nx + (unsigned)min(x0, nx - 1);
    // this thread's float4 of a tmp tile, and its 4 source values of a staged row
    auto rd_tmp = [&](int k) { return *reinterpret_cast<const float4*>(tmp_s + k * kZtTmpFloats + yl * 32 + xl); };
    auto rd_src = [&](int k, int zs) {
        if (!VK_ZT_SRC_TMA) {
            const float* t = src + (e0 + (unsigned)zs * plane);
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (nvalid > 0) v.x = __ldg(t);
            if (nvalid > 1) v.y = __ldg(t + 1);
            if (nvalid > 2) v.z = __ldg(t + 2);
            if (nvalid > 3) v.w = __ldg(t + 3);
            return v;
        }
        const uintptr_t st =
            reinterpret_cast<uintptr_t>(src + ((size_t)(b * nz + zs) * plane + (size_t)yc * nx + X0));
        const float* r = src_s + k * kZtSrcFloats + yl * kZtSrcPitch + (int)((st & 15) >> 2) + xl;
        return make_float4(r[0], r[1], r[2], r[3]);  // columns >= nvalid are never used
    };
    float2 r0[P], r1[P];
#pragma unroll
    for (int t = 0; t < P; ++t) r0[t] = r1[t] = make_float2(0.f, 0.f);
    float4 pv = make_float4(0.f, 0.f, 0.f, 0.f);
    int c = 0;
    // Stores: the warp's 4 rows x 32 columns go through a warp-private shared
    // transpose so that each store instruction writes 32 consecutive floats of
    // one row (the per-thread float4 columns of the unpitched level would
    // touch every sector of 4 rows with 4-byte pieces, 4 instructions each).
    float* wst = reinterpret_cast<float*>(empty + kZtSlots) + wy * 128;
    const unsigned rb = (unsigned)b * plane * (unsigned)nz + (unsigned)(Y0 + 4 * wy) * (unsigned)nx + (unsigned)(X0 + lane);
    const int nrows = min(4, ny - (Y0 + 4 * wy));
    const bool okc = X0 + lane < nx;
    auto store_rows = [&](float* base, float4 v) {
        if (VK_ZT_TSTORE) {
            *reinterpret_cast<float4*>(wst + ry * 32 + xl) = v;
            __syncwarp();
            if (okc)
                for (int r = 0; r < nrows; ++r) base[rb + (unsigned)r * (unsigned)nx] = wst[r * 32 + lane];
            __syncwarp();
        } else {
            float* t = base + e0;
            if (nvalid > 0) t[0] = v.x;
            if (nvalid > 1) t[1] = v.y;
            if (nvalid > 2) t[2] = v.z;
            if (nvalid > 3) t[3] = v.w;
        }
    };
    auto epilogue = [&](int zo, float4 o, float4 sv) {
        store_rows(dst + (size_t)zo * plane, o);
        if (want_src)
            store_rows(dog + (size_t)zo * plane,
                       make_float4(__fsub_rn(sv.x, o.x), __fsub_rn(sv.y, o.y), __fsub_rn(sv.z, o.z), __fsub_rn(sv.w, o.w)));
        if constexpr (HALF) {
            float4 qv, qo;
            qv.x = __shfl_xor_sync(0xffffffffu, pv.x, 8);
            qv.y = __shfl_xor_sync(0xffffffffu, pv.y, 8);
            qv.z = __shfl_xor_sync(0xffffffffu, pv.z, 8);
            qv.w = __shfl_xor_sync(0xffffffffu, pv.w, 8);
            qo.x = __shfl_xor_sync(0xffffffffu, o.x, 8);
            qo.y = __shfl_xor_sync(0xffffffffu, o.y, 8);
            qo.z = __shfl_xor_sync(0xffffffffu, o.z, 8);
            qo.w = __shfl_xor_sync(0xffffffffu, o.w, 8);
            const int hnx = nx >> 1, hny = ny >> 1, hnz = nz >> 1;
            const int hy = gy >> 1, hz = zo >> 1;
            if ((zo & 1) && !(ry & 1) && hy < hny && hz < hnz) {
                float* hp = half + (((long long)b * hnz + hz) * hny + hy) * hnx;
                const int hx = x0 >> 1;
                if (hx < hnx) {
                    float sm = pv.x;
                    sm = fadd(sm, o.x);
                    sm = fadd(sm, qv.x);
                    sm = fadd(sm, qo.x);
                    sm = fadd(sm, pv.y);
                    sm = fadd(sm, o.y);
                    sm = fadd(sm, qv.y);
                    sm = fadd(sm, qo.y);
                    hp[hx] = fmul(sm, 0.125f);
                }
                if (hx + 1 < hnx) {
                    float sm = pv.z;
                    sm = fadd(sm, o.z);
                    sm = fadd(sm, qv.z);
                    sm = fadd(sm, qo.z);
                    sm = fadd(sm, pv.w);
                    sm = fadd(sm, o.w);
                    sm = fadd(sm, qv.w);
                    sm = fadd(sm, qo.w);
                    hp[hx + 1] = fmul(sm, 0.125f);
                }
            }
            pv = o;
        }
    };
    for (int a = 0; a < A; a += 2) {
        const int k0 = a % kZtSlots, k1 = (a + 1) % kZtSlots;
        const unsigned ph = (unsigned)(a / kZtSlots) & 1u;  // a even, kZtSlots even: a and a+1 share the use count
        const int zo = za + a - R;                          // outputs zo, zo + 1 complete in this step
        const bool out = zo >= z_start;
        mbar_wait(&full[k0], ph);
        const float4 v0 = rd_tmp(k0);
        const float4 sv0 = (out && want_src) ? rd_src(k0, zo) : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 v1 = make_float4(0.f, 0.f, 0.f, 0.f), sv1 = v1;
        const bool two = a + 1 < A;
        if (two) {
            mbar_wait(&full[k1], ph);
            v1 = rd_tmp(k1);
            if (out && want_src && zo + 1 < z_end) sv1 = rd_src(k1, zo + 1);
        }
        __syncwarp();
        if (lane == 0) {  // this warp is done with both slots
            mbar_arrive(&empty[k0]);
            if (two) mbar_arrive(&empty[k1]);
        }
        float4 o0, o1;
        z4_dispatch2<R, 0, P, true>(c, r0, r1, v0, v1, taps, o0, o1);
        c += 2;
        if (c >= P) c -= P;
        if (!out) continue;
        epilogue(zo, o0, sv0);
        if (zo + 1 < z_end) epilogue(zo + 1, o1, sv1);
    }
}

// ---------------------------------------------------------------------------
// Small octaves in one launch.  Once a level fits in shared memory three times
// over, one CTA per volume runs every remaining octave there: each blur is
// three out-of-place 1-D passes (same arithmetic as above: fp32 products
// added in tap order, replicate borders, x then y then z), the DoG and the
// handoff subsample are written as the levels are produced, and the next
// octave starts from the subsampled level.  Removes ~5 latency-bound launches
// per small octave.
constexpr int kSmallMaxVox = 16384;  // 3 buffers x 64 KB
constexpr int kSmallMaxOct = 8;
constexpr int kSmallMaxLev = 12;

struct SmallOctaves {
    int n_oct, levels, handoff;
    int dims[kSmallMaxOct][3];
    float* lv[kSmallMaxOct][kSmallMaxLev];    // batched level tensors
    float* dog[kSmallMaxOct][kSmallMaxLev];   // batched DoG tensors
    int radius[kSmallMaxLev];                 // blur radius of level i (i >= 1)
    float taps[kSmallMaxLev][VK_MAX_TAPS];
};

VK_D void small_pass(const float* __restrict__ in, float* __restrict__ out, int nx, int ny, int nz, int axis, int R,
                     const float* w) {
    const int n = nx * ny * nz;
    const int st = axis == 0 ? 1 : (axis == 1 ? nx : nx * ny);
    const int len = axis == 0 ? nx : (axis == 1 ? ny : nz);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int c = axis == 0 ? i % nx : (axis == 1 ? (i / nx) % ny : i / (nx * ny));
        const float* base = in + (i - c * st);
        float acc = fmul(w[0], base[clampi(c - R, 0, len - 1) * st]);
        for (int t = 1; t <= 2 * R; ++t) acc = fadd(acc, fmul(w[t], base[clampi(c - R + t, 0, len - 1) * st]));
        out[i] = acc;
    }
}

// Radius-specialised pass: taps unrolled from registers, the line coordinate by
// multiply-high division (exact for < 2^16 voxels), unclamped taps away from
// the borders.  Same products and tap-order sums as small_pass.
template <int R, int AXIS>
VK_D void small_pass_r(const float* __restrict__ in, float* __restrict__ out, int nx, int ny, int nz, unsigned mx,
                       unsigned my, const float* w) {
    constexpr int P = 2 * R + 1;
    float wr[P];
#pragma unroll
    for (int t = 0; t < P; ++t) wr[t] = w[t];
    const int n = nx * ny * nz;
    const int st = AXIS == 0 ? 1 : (AXIS == 1 ? nx : nx * ny);
    const int len = AXIS == 0 ? nx : (AXIS == 1 ? ny : nz);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const unsigned q1 = mx ? __umulhi((unsigned)i, mx) : (unsigned)i;  // i / nx
        int c;
        if (AXIS == 0) {
            c = i - (int)q1 * nx;
        } else {
            const unsigned q2 = my ? __umulhi(q1, my) : q1;  // i / (nx ny)
            c = AXIS == 1 ? (int)q1 - (int)q2 * ny : (int)q2;
        }
        const float* base = in + (i - c * st);
        float acc;
        if (c >= R && c + R < len) {
            const float* q = base + (c - R) * st;
            acc = fmul(wr[0], q[0]);
#pragma unroll
            for (int t = 1; t < P; ++t) acc = fadd(acc, fmul(wr[t], q[t * st]));
        } else {
            acc = fmul(wr[0], base[clampi(c - R, 0, len - 1) * st]);
#pragma unroll
            for (int t = 1; t < P; ++t) acc = fadd(acc, fmul(wr[t], base[clampi(c - R + t, 0, len - 1) * st]));
        }
        out[i] = acc;
    }
}

template <int AXIS>
VK_D void small_pass_any(const float* in, float* out, int nx, int ny, int nz, unsigned mx, unsigned my, int R,
                         const float* w) {
    switch (R) {
        case 1: small_pass_r<1, AXIS>(in, out, nx, ny, nz, mx, my, w); break;
        case 2: small_pass_r<2, AXIS>(in, out, nx, ny, nz, mx, my, w); break;
        case 3: small_pass_r<3, AXIS>(in, out, nx, ny, nz, mx, my, w); break;
        case 4: small_pass_r<4, AXIS>(in, out, nx, ny, nz, mx, my, w); break;
        case 5: small_pass_r<5, AXIS>(in, out, nx, ny, nz, mx, my, w); break;
        case 6: small_pass_r<6, AXIS>(in, out, nx, ny, nz, mx, my, w); break;
        case 7: small_pass_r<7, AXIS>(in, out, nx, ny, nz, mx, my, w); break;
        case 8: small_pass_r<8, AXIS>(in, out, nx, ny, nz, mx, my, w); break;
        case 9: small_pass_r<9, AXIS>(in, out, nx, ny, nz, mx, my, w); break;
        case 10: small_pass_r<10, AXIS>(in, out, nx, ny, nz, mx, my, w); break;
        default: small_pass(in, out, nx, ny, nz, AXIS, R, w); break;
    }
}

#ifndef VK_SMALL_THREADS
#define VK_SMALL_THREADS 1024
#endif
#ifndef VK_SMALL_FAST
#define VK_SMALL_FAST 1  // radius-specialised passes (0: the generic runtime-radius pass)
#endif
constexpr int kSmallThreads = VK_SMALL_THREADS;

__global__ void __launch_bounds__(kSmallThreads)
small_octaves_kernel(SmallOctaves so) {
    extern __shared__ float4 sm4[];
    float* A = reinterpret_cast<float*>(sm4);
    float* Bf = A + kSmallMaxVox;
    float* C = Bf + kSmallMaxVox;
    const int b = blockIdx.x;
    for (int o = 0; o < so.n_oct; ++o) {
        const int nx = so.dims[o][0], ny = so.dims[o][1], nz = so.dims[o][2];
        const int n = nx * ny * nz;
        const long long vb = (long long)b * n;
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) A[i] = so.lv[o][0][vb + i];
        __syncthreads();
        float* src = A;
        float* xb = Bf;
        float* yb = C;
        // multiply-high reciprocals of nx and nx * ny (0: divisor 1)
        const unsigned mx = nx > 1 ? 0xFFFFFFFFu / (unsigned)nx + 1u : 0u;
        const unsigned my = ny > 1 ? 0xFFFFFFFFu / (unsigned)ny + 1u : 0u;
        for (int lvi = 1; lvi < so.levels; ++lvi) {
            const int R = so.radius[lvi];
            const float* w = so.taps[lvi];
            if (VK_SMALL_FAST) {
                small_pass_any<0>(src, xb, nx, ny, nz, mx, my, R, w);
                __syncthreads();
                small_pass_any<1>(xb, yb, nx, ny, nz, mx, my, R, w);
                __syncthreads();
                small_pass_any<2>(yb, xb, nx, ny, nz, mx, my, R, w);  // xb now holds level lvi
            } else {
                small_pass(src, xb, nx, ny, nz, 0, R, w);
                __syncthreads();
                small_pass(xb, yb, nx, ny, nz, 1, R, w);
                __syncthreads();
                small_pass(yb, xb, nx, ny, nz, 2, R, w);
            }
            __syncthreads();
            float* lo = so.lv[o][lvi] + vb;
            float* dg = so.dog[o][lvi - 1] + vb;
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                lo[i] = xb[i];
                dg[i] = __fsub_rn(src[i], xb[i]);
            }
            if (lvi == so.handoff && o + 1 < so.n_oct) {
                const int hx = nx >> 1, hy = ny >> 1, hz = nz >> 1, hn = hx * hy * hz;
                float* hdst = so.lv[o + 1][0] + (long long)b * hn;
                for (int i = threadIdx.x; i < hn; i += blockDim.x) {
                    const int x = i % hx, y = (i / hx) % hy, z = i / (hx * hy);
                    auto at = [&](int dx, int dy, int dz) {
                        return xb[((2 * z + dz) * ny + (2 * y + dy)) * nx + (2 * x + dx)];
                    };
                    float sm = at(0, 0, 0);
                    sm = fadd(sm, at(0, 0, 1));
                    sm = fadd(sm, at(0, 1, 0));
                    sm = fadd(sm, at(0, 1, 1));
                    sm = fadd(sm, at(1, 0, 0));
                    sm = fadd(sm, at(1, 0, 1));
                    sm = fadd(sm, at(1, 1, 0));
                    sm = fadd(sm, at(1, 1, 1));
                    hdst[i] = fmul(sm, 0.125f);
                }
            }
            __syncthreads();
            float* t = src;  // the new level becomes the source of the next blur
            src = xb;
            xb = t;
        }
    }
}

// ---------------------------------------------------------------------------
// Generic fallback for radius > 10: three 1-D passes through global scratch.
__global__ void blur_axis_kernel(const float* __restrict__ src, float* __restrict__ dst, int nx, int ny, int nz,
                                 long long total, int axis, int R, Taps taps) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    long long plane = (long long)nx * ny;
    long long vol = plane * nz;
    long long b = i / vol, rem = i - b * vol;
    int z = (int)(rem / plane);
    int y = (int)((rem - (long long)z * plane) / nx);
    int x = (int)(rem - (long long)z * plane - (long long)y * nx);
    int n = axis == 0 ? nx : (axis == 1 ? ny : nz);
    int c = axis == 0 ? x : (axis == 1 ? y : z);
    long long stride = axis == 0 ? 1 : (axis == 1 ? nx : plane);
    const float* base = src + i - (long long)c * stride;
    float acc = fmul(taps.w[0], __ldg(base + (long long)clampi(c - R, 0, n - 1) * stride));
    for (int t = 1; t <= 2 * R; ++t)
        acc = fadd(acc, fmul(taps.w[t], __ldg(base + (long long)clampi(c - R + t, 0, n - 1) * stride)));
    dst[i] = acc;
}

__global__ void dog_half_epilogue_kernel(const float* __restrict__ src, const float* __restrict__ dst,
                                         float* __restrict__ dog, long long total) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < total) dog[i] = __fsub_rn(src[i], dst[i]);
}

__global__ void subsample_kernel(const float* __restrict__ src, float* __restrict__ dst, int nx, int ny, int nz,
                                 long long total) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int hx = nx >> 1, hy = ny >> 1, hz = nz >> 1;
    long long hplane = (long long)hx * hy, hvol = hplane * hz;
    long long b = i / hvol, rem = i - b * hvol;
    int z = (int)(rem / hplane);
    int y = (int)((rem - (long long)z * hplane) / hx);
    int x = (int)(rem - (long long)z * hplane - (long long)y * hx);
    const long long plane = (long long)nx * ny;
    const float* s = src + b * plane * nz;
    auto at = [&](int dx, int dy, int dz) {
        return __ldg(s + (long long)(2 * z + dz) * plane + (long long)(2 * y + dy) * nx + (2 * x + dx));
    };
    float sm = at(0, 0, 0);
    sm = fadd(sm, at(0, 0, 1));
    sm = fadd(sm, at(0, 1, 0));
    sm = fadd(sm, at(0, 1, 1));
    sm = fadd(sm, at(1, 0, 0));
    sm = fadd(sm, at(1, 0, 1));
    sm = fadd(sm, at(1, 1, 0));
    sm = fadd(sm, at(1, 1, 1));
    dst[i] = fmul(sm, 0.125f);
}

__global__ void difference_kernel(const float4* __restrict__ a, const float4* __restrict__ b, float4* __restrict__ o,
                                  long long n4) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n4; i += (long long)gridDim.x * blockDim.x) {
        float4 x = __ldg(a + i), y = __ldg(b + i);
        o[i] = make_float4(__fsub_rn(x.x, y.x), __fsub_rn(x.y, y.y), __fsub_rn(x.z, y.z), __fsub_rn(x.w, y.w));
    }
}

__global__ void difference_tail_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ o,
                                       long long start, long long n) {
    long long i = start + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) o[i] = __fsub_rn(a[i], b[i]);
}

// [b][x][y][z] (z fastest) <-> [b][z][y][x] (x fastest): a 2-D transpose of
// the (x, z) axes for every (b, y).  in_dims = (n0 slowest-major axis, n2).
__global__ void transpose_xz_kernel(const float* __restrict__ src, float* __restrict__ dst, int n0, int ny, int n2) {
    __shared__ float tile[32][33];
    const int by = blockIdx.z;  // b * ny + y
    const int b = by / ny, y = by - b * ny;
    const long long vol = (long long)n0 * ny * n2;
    const int i2 = blockIdx.x * 32 + threadIdx.x;   // fast axis of src
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        int i0 = blockIdx.y * 32 + k;
        if (i0 < n0 && i2 < n2) tile[k][threadIdx.x] = src[b * vol + ((long long)i0 * ny + y) * n2 + i2];
    }
    __syncthreads();
    const int o0 = blockIdx.y * 32 + threadIdx.x;  // becomes the fast axis of dst
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        int o2 = blockIdx.x * 32 + k;
        if (o0 < n0 && o2 < n2) dst[b * vol + ((long long)o2 * ny + y) * n0 + o0] = tile[threadIdx.x][k];
    }
}

template <int R>
static int launch_ring(const float* src, float* dst, float* dog, float* half, int nb, int nx, int ny, int nz,
                       const Taps& taps, cudaStream_t st) {
    using G = BlurGeom<R>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(blur3d_stream_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        if (e != cudaSuccess) return cuda_status(e, "blur3d attribute");
        configured = true;
    }
    const int tiles = ((nx + kTX - 1) / kTX) * ((ny + kTY - 1) / kTY);
    // z-chunking: every chunk re-stages and re-blurs (x, y) 2R halo planes, so
    // pick the chunk count that minimises waves x planes per CTA (chunks of at
    // least 16 planes, even starts for the subsample epilogue).
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long slots = (long long)sms * blur_min_blocks<R>();
    int nzc = 1, tz = nz + (nz & 1);
    double best = -1.0;
    for (int n = 1; n <= 16; ++n) {
        int t = (nz + n - 1) / n;
        t += t & 1;
        const int nc = (nz + t - 1) / t;
        if (n > 1 && t < 16) break;
        const long long ctas = (long long)tiles * nb * nc;
        const double waves = (double)((ctas + slots - 1) / slots);
        const double cost = waves * (t + (nc > 1 ? 2 * R : R));
        if (best < 0 || cost < best * 0.97) {
            best = cost;
            nzc = nc;
            tz = t;
        }
    }
    dim3 grid((nx + kTX - 1) / kTX, (ny + kTY - 1) / kTY, nb * nzc);
    blur3d_stream_kernel<R><<<grid, kThreads, G::SMEM, st>>>(src, dst, dog, half, nx, ny, nz, tz, nzc, taps);
    count_launch();
    return cuda_status(cudaGetLastError(), "blur3d launch");
}

// Split path: (x, y) kernel into `work` (nb * volume floats), then the z kernel.
static int kZWaves = 1, kZMinChunkR = 12;  // z chunking: long chunks measured best in the multi-stream bench -- the 2R warm-up
                                          // arrivals per chunk cost more than the lost parallelism (env-overridable)
template <int R, int TY>
static int launch_xy(const float* src, float* work, int tp, int nb, int nx, int ny, int nz, const Taps& taps,
                     cudaStream_t st, const float* prev, float* pdog) {
    using G = XyGeom<R, TY>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(blur_xy_kernel<R, TY>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        if (e != cudaSuccess) return cuda_status(e, "blur xy attribute");
        configured = true;
    }
    dim3 g1((nx + kXyTX - 1) / kXyTX, (ny + TY - 1) / TY, nb * nz);
    blur_xy_kernel<R, TY><<<g1, kThreads, G::SMEM, st>>>(src, work, tp, nx, ny, nz, taps, prev, pdog);
    count_launch();
    return cuda_status(cudaGetLastError(), "blur xy launch");
}

// Whole-plane (x, y) kernel: planes up to kPlaneThreads rows and columns and
// small enough for two CTAs per SM.
static bool plane_kernel_fits(int nx, int ny) {
    return nx <= kPlaneThreads && ny <= kPlaneThreads && (long long)nx * ny * 4 + 32 <= 110 * 1024;
}

template <int R>
static int launch_xy_plane(const float* src, float* work, int tp, int nb, int nx, int ny, int nz, const Taps& taps,
                           cudaStream_t st, const float* prev, float* pdog) {
    const int smem = nx * ny * 4 + 32;
    static int configured = 0;
    if (configured < smem) {
        cudaError_t e = cudaFuncSetAttribute(blur_xy_plane_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             110 * 1024);
        if (e != cudaSuccess) return cuda_status(e, "blur xy plane attribute");
        configured = 110 * 1024;
    }
    blur_xy_plane_kernel<R><<<nb * nz, kPlaneThreads + (prev ? kDogThreads : 0), smem, st>>>(src, work, tp, nx, ny, taps, prev,
                                                                                  pdog);
    count_launch();
    return cuda_status(cudaGetLastError(), "blur xy plane launch");
}

// Persistent double-buffered plane kernel: two staged planes per CTA, one CTA per SM.
static bool plane_stream_fits(int nx, int ny) {
    return nx <= kPlaneThreads && ny <= kPlaneThreads && 2 * ((long long)nx * ny * 4 + 32) <= 220 * 1024;
}

template <int R>
static int launch_xy_stream(const float* src, float* work, int tp, int nb, int nx, int ny, int nz, const Taps& taps,
                            cudaStream_t st, const float* prev, float* pdog, unsigned* counters, int sms) {
    const unsigned buf_floats = (unsigned)(((long long)nx * ny + 8 + 3) & ~3LL);  // + 16-byte alignment slack
    const int smem = (int)(2 * buf_floats * 4);
    static int configured = 0;
    if (configured < smem) {
        cudaError_t e = cudaFuncSetAttribute(blur_xy_stream_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             220 * 1024);
        if (e != cudaSuccess) return cuda_status(e, "blur xy stream attribute");
        configured = 220 * 1024;
    }
    cudaError_t e = cudaMemsetAsync(counters, 0, 2 * sizeof(unsigned), st);
    if (e != cudaSuccess) return cuda_status(e, "blur xy stream counters");
    const int nplanes = nb * nz;
    const int grid = nplanes < sms ? nplanes : sms;
    blur_xy_stream_kernel<R><<<grid, 2 * kPlaneThreads + (prev ? kStreamDogThreads : 0), smem, st>>>(
        src, work, tp, nx, ny, nplanes, buf_floats, taps, prev, pdog, counters);
    count_launch();
    return cuda_status(cudaGetLastError(), "blur xy stream launch");
}

#ifndef VK_XY_STREAM
#define VK_XY_STREAM 0
#endif
static int g_xy_kernel = VK_XY_STREAM ? 2 : 0;  // 0: whole-plane ring kernel where it fits, 1: tile kernel (A/B),
                                               // 2: persistent double-buffered plane kernel
static int g_z_kernel = 0;  // 0: TMA-fed four-column kernel, 1: register-fed four-column kernel (packed sums),
                            // 2: four-column scalar sums, 3: column-pair kernel
static int kZ4Waves = 2, kZ4MinChunkR = 6;

template <int R, bool HALF, bool PK>
static void launch_z4(const float* work, int tp, const float* src, float* dst, float* dog, float* half, int nb,
                      int nx, int ny, int nz, const Taps& taps, cudaStream_t st, int zchunk, int sms) {
    const long long ctas = (long long)((tp + 31) / 32) * ((ny + 15) / 16) * nb;
    const long long slots = (long long)sms * z4_min_blocks<R>();
    int nzc = 1;
    while (ctas * nzc < (long long)kZ4Waves * slots && (nz + nzc) / (nzc + 1) >= kZ4MinChunkR * R && nzc < 64) ++nzc;
    if (zchunk > 0) nzc = (nz + zchunk - 1) / zchunk;  // caller-chosen granularity (convolve_separable's chunk)
    int tz = (nz + nzc - 1) / nzc;
    tz += tz & 1;
    nzc = (nz + tz - 1) / tz;
    dim3 g((tp + 31) / 32, (ny + 15) / 16, nb * nzc);
    blur_z4_kernel<R, HALF, PK><<<g, kZ4Threads, 0, st>>>(work, tp, src, dst, dog, half, nx, ny, nz, tz, nzc, taps);
    count_launch();
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static int g_encode_state = 0;  // 0 unknown, 1 available, -1 unavailable

static bool get_encode() {
    if (g_encode_state == 0) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess && fn) {
            g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
            g_encode_state = 1;
        } else {
            g_encode_state = -1;
        }
    }
    return g_encode_state == 1;
}

// Tensor map over the pitched intermediate (tp, ny, nb * nz), box 32 x 16 x 1.
static bool encode_tmp_map(CUtensorMap* m, const float* work, int tp, int ny, long long planes) {
    if (!get_encode() || (tp & 3) || (reinterpret_cast<uintptr_t>(work) & 15)) return false;
    cuuint64_t dims[3] = {(cuuint64_t)tp, (cuuint64_t)ny, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)tp * 4, (cuuint64_t)tp * ny * 4};
    cuuint32_t box[3] = {32, 16, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(work), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int kZtWaves = 2, kZtMinChunkR = 6;

template <int R, bool HALF>
static bool launch_zt(const float* work, int tp, const float* src, float* dst, float* dog, float* half, int nb,
                      int nx, int ny, int nz, const Taps& taps, cudaStream_t st, int zchunk, int sms) {
    CUtensorMap m;
    if (!encode_tmp_map(&m, work, tp, ny, (long long)nb * nz)) return false;
    static bool configured = false;
    if (!configured) {
        if (cudaFuncSetAttribute(blur_zt_kernel<R, HALF>, cudaFuncAttributeMaxDynamicSharedMemorySize, kZtSmem) !=
            cudaSuccess)
            return false;
        configured = true;
    }
    const long long ctas = (long long)((tp + 31) / 32) * ((ny + 15) / 16) * nb;
    const long long slots = (long long)sms * zt_min_blocks<R>();
    int nzc = 1;
    while (ctas * nzc < (long long)kZtWaves * slots && (nz + nzc) / (nzc + 1) >= kZtMinChunkR * R && nzc < 64) ++nzc;
    if (zchunk > 0) nzc = (nz + zchunk - 1) / zchunk;
    int tz = (nz + nzc - 1) / nzc;
    tz += tz & 1;
    nzc = (nz + tz - 1) / tz;
    dim3 g((tp + 31) / 32, (ny + 15) / 16, nb * nzc);
    blur_zt_kernel<R, HALF><<<g, kZtThreads, kZtSmem, st>>>(m, src, dst, dog, half, nx, ny, nz, tz, nzc, taps);
    count_launch();
    return true;
}

template <int R>
static int launch_split(const float* src, float* dst, float* dog, float* half, int nb, int nx, int ny, int nz,
                        const Taps& taps, float* work, int tp, cudaStream_t st, int zchunk, const float* prev,
                        float* pdog, unsigned* counters) {
    static bool env_read = false;
    if (!env_read) {
        if (const char* e = getenv("VK_Z_WAVES")) kZWaves = atoi(e) > 0 ? atoi(e) : kZWaves;
        if (const char* e = getenv("VK_Z_MINCHUNK")) kZMinChunkR = atoi(e) > 0 ? atoi(e) : kZMinChunkR;
        if (const char* e = getenv("VK_Z4_WAVES")) kZ4Waves = atoi(e) > 0 ? atoi(e) : kZ4Waves;
        if (const char* e = getenv("VK_Z4_MINCHUNK")) kZ4MinChunkR = atoi(e) > 0 ? atoi(e) : kZ4MinChunkR;
        if (const char* e = getenv("VK_Z_KERNEL")) g_z_kernel = atoi(e);
        if (const char* e = getenv("VK_XY_KERNEL")) g_xy_kernel = atoi(e);
        if (const char* e = getenv("VK_ZT_WAVES")) kZtWaves = atoi(e) > 0 ? atoi(e) : kZtWaves;
        if (const char* e = getenv("VK_ZT_MINCHUNK")) kZtMinChunkR = atoi(e) > 0 ? atoi(e) : kZtMinChunkR;
        env_read = true;
    }
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // taller tiles (less x-pass halo, fewer y-pass loads) unless they waste rows
    const bool tall = ((ny + 95) / 96) * 96 <= ((ny + 63) / 64) * 64;
    // 97..176 rows: one tile spans the whole y extent (no recomputed x-pass halo rows between y tiles;
    // measured 3.6% faster pyramid on 145x174x145 despite 2 CTAs/SM instead of 4)
    const int rc1 = g_xy_kernel == 2 && counters && plane_stream_fits(nx, ny)
                        ? launch_xy_stream<R>(src, work, tp, nb, nx, ny, nz, taps, st, prev, pdog, counters, sms)
                    : g_xy_kernel != 1 && plane_kernel_fits(nx, ny)
                        ? launch_xy_plane<R>(src, work, tp, nb, nx, ny, nz, taps, st, prev, pdog)
                    : ny <= 176 && ny > 96 ? launch_xy<R, 176>(src, work, tp, nb, nx, ny, nz, taps, st, prev, pdog)
                    : tall               ? launch_xy<R, 96>(src, work, tp, nb, nx, ny, nz, taps, st, prev, pdog)
                                         : launch_xy<R, 64>(src, work, tp, nb, nx, ny, nz, taps, st, prev, pdog);
    if (rc1 != VK_OK) return rc1;
    if (g_z_kernel == 0) {
        const bool ok = half ? launch_zt<R, true>(work, tp, src, dst, dog, half, nb, nx, ny, nz, taps, st, zchunk, sms)
                             : launch_zt<R, false>(work, tp, src, dst, dog, half, nb, nx, ny, nz, taps, st, zchunk, sms);
        if (ok) return cuda_status(cudaGetLastError(), "blur zt launch");
        // no tensor-map support: the register-fed four-column kernel
    }
    if (g_z_kernel != 3) {
        const bool pk = g_z_kernel != 2;
        if (half) {
            if (pk) launch_z4<R, true, true>(work, tp, src, dst, dog, half, nb, nx, ny, nz, taps, st, zchunk, sms);
            else launch_z4<R, true, false>(work, tp, src, dst, dog, half, nb, nx, ny, nz, taps, st, zchunk, sms);
        } else {
            if (pk) launch_z4<R, false, true>(work, tp, src, dst, dog, half, nb, nx, ny, nz, taps, st, zchunk, sms);
            else launch_z4<R, false, false>(work, tp, src, dst, dog, half, nb, nx, ny, nz, taps, st, zchunk, sms);
        }
        return cuda_status(cudaGetLastError(), "blur z4 launch");
    }
    // z chunks: enough CTAs for ~4 waves, each chunk >= 4R planes (the 2R
    // warm-up arrivals are overhead), even starts for the subsample epilogue
    const long long cols = (long long)((nx + 31) / 32) * ((ny + 15) / 16) * nb;
    int nzc = 1;
    while (cols * nzc < (long long)kZWaves * 8 * sms && (nz + nzc) / (nzc + 1) >= kZMinChunkR * R && nzc < 64) ++nzc;
    if (zchunk > 0) nzc = (nz + zchunk - 1) / zchunk;  // caller-chosen granularity (convolve_separable's chunk)
    int tz = (nz + nzc - 1) / nzc;
    tz += tz & 1;
    nzc = (nz + tz - 1) / tz;
    dim3 g2((nx + 31) / 32, (ny + 15) / 16, nb * nzc);
    blur_z_kernel<R><<<g2, kThreads, 0, st>>>(work, tp, src, dst, dog, half, nx, ny, nz, tz, nzc, taps);
    count_launch();
    return cuda_status(cudaGetLastError(), "blur split launch");
}

static int launch_generic(const float* src, float* dst, float* dog, float* half, int nb, int nx, int ny, int nz,
                          int R, const Taps& taps, cudaStream_t st) {
    const long long total = (long long)nb * nx * ny * nz;
    float *t1 = nullptr, *t2 = nullptr;
    cudaError_t e = cudaMallocAsync(&t1, total * 4, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&t2, total * 4, st);
    if (e != cudaSuccess) return cuda_status(e, "blur scratch");
    const int th = 256;
    const unsigned blocks = (unsigned)((total + th - 1) / th);
    blur_axis_kernel<<<blocks, th, 0, st>>>(src, t1, nx, ny, nz, total, 0, R, taps);
    count_launch();
    blur_axis_kernel<<<blocks, th, 0, st>>>(t1, t2, nx, ny, nz, total, 1, R, taps);
    count_launch();
    blur_axis_kernel<<<blocks, th, 0, st>>>(t2, dst, nx, ny, nz, total, 2, R, taps);
    count_launch();
    if (dog) {
        dog_half_epilogue_kernel<<<blocks, th, 0, st>>>(src, dst, dog, total);
        count_launch();
    }
    if (half && nx >= 2 && ny >= 2 && nz >= 2) {
        long long ht = (long long)nb * (nx / 2) * (ny / 2) * (nz / 2);
        subsample_kernel<<<(unsigned)((ht + th - 1) / th), th, 0, st>>>(dst, half, nx, ny, nz, ht);
        count_launch();
    }
    cudaFreeAsync(t1, st);
    cudaFreeAsync(t2, st);
    return cuda_status(cudaGetLastError(), "blur generic launch");
}

}  // namespace vk

using namespace vk;

// 0: split (x, y) + z kernels (default), 1: fused streaming kernel.
static int g_blur_path = 0;

extern "C" int vk_set_blur_path(int path) {
    if (path < 0 || path > 1) {
        set_error("vk_set_blur_path: path must be 0 (split xy + z) or 1 (fused streaming)");
        return VK_ERR_PARAMETER;
    }
    g_blur_path = path;
    return VK_OK;
}

extern "C" int vk_set_xy_kernel(int k) {
    if (k < 0 || k > 2) {
        set_error("vk_set_xy_kernel: 0 (whole-plane ring kernel), 1 (tile kernel) or 2 (persistent double-buffered "
                  "plane kernel)");
        return VK_ERR_PARAMETER;
    }
    g_xy_kernel = k;
    return VK_OK;
}

extern "C" int vk_set_z_kernel(int k) {
    if (k < 0 || k > 3) {
        set_error("vk_set_z_kernel: 0 (TMA-fed), 1 (four-column, packed sums), 2 (four-column, scalar sums) or "
                  "3 (column pair)");
        return VK_ERR_PARAMETER;
    }
    g_z_kernel = k;
    return VK_OK;
}

static int blur3d_impl(const float* src, float* dst, float* dog_out, float* half_out, int nb, int nx, int ny, int nz,
                       const float* taps_host, int radius, float* work, long long work_floats, int zchunk,
                       void* stream, const float* prev = nullptr, float* prev_dog = nullptr);
extern "C" int vk_difference(const float* a, const float* b, float* out, long long n, void* stream);

extern "C" int vk_blur3d_ws(const float* src, float* dst, float* dog_out, float* half_out, int nb, int nx, int ny,
                            int nz, const float* taps_host, int radius, float* work, long long work_floats,
                            void* stream) {
    return blur3d_impl(src, dst, dog_out, half_out, nb, nx, ny, nz, taps_host, radius, work, work_floats, 0, stream);
}

extern "C" int vk_blur3d_ws2(const float* src, float* dst, float* dog_out, float* half_out, const float* prev,
                             float* prev_dog, int nb, int nx, int ny, int nz, const float* taps_host, int radius,
                             float* work, long long work_floats, void* stream) {
    if ((prev == nullptr) != (prev_dog == nullptr)) {
        set_error("vk_blur3d_ws2: prev and prev_dog must both be given or both be NULL");
        return VK_ERR_PARAMETER;
    }
    return blur3d_impl(src, dst, dog_out, half_out, nb, nx, ny, nz, taps_host, radius, work, work_floats, 0, stream,
                       prev, prev_dog);
}

extern "C" int vk_blur3d_chunked(const float* src, float* dst, int nb, int nx, int ny, int nz, const float* taps_host,
                                 int radius, int zchunk, void* stream) {
    if (zchunk < 1) {
        set_error("vk_blur3d_chunked: chunk must be >= 1, got %d", zchunk);
        return VK_ERR_PARAMETER;
    }
    return blur3d_impl(src, dst, nullptr, nullptr, nb, nx, ny, nz, taps_host, radius, nullptr, 0, zchunk, stream);
}

static int blur3d_impl(const float* src, float* dst, float* dog_out, float* half_out, int nb, int nx, int ny, int nz,
                       const float* taps_host, int radius, float* work, long long work_floats, int zchunk,
                       void* stream, const float* prev, float* prev_dog) {
    if (!src || !dst || !taps_host || nb < 0 || nx < 1 || ny < 1 || nz < 1 || radius < 1 ||
        2 * radius + 1 > VK_MAX_TAPS || work_floats < 0) {
        set_error("vk_blur3d: bad arguments (nb=%d dims=%d,%d,%d radius=%d)", nb, nx, ny, nz, radius);
        return VK_ERR_PARAMETER;
    }
    if (nb == 0) return VK_OK;
    Taps taps{};
    for (int i = 0; i < 2 * radius + 1; ++i) taps.w[i] = taps_host[i];
    taps.mz = -0.0f;
    cudaStream_t st = as_stream(stream);
    if (half_out && (nx < 2 || ny < 2 || nz < 2)) half_out = nullptr;
    // Both kernels share each product between the two taps at the same
    // distance; Gaussian taps (scalespace.py:35-42) are exactly symmetric.
    bool symmetric = true;
    for (int i = 0; i < radius; ++i) symmetric = symmetric && taps.w[i] == taps.w[2 * radius - i];
    // ... and address the batch with 32-bit element offsets.
    const long long total = (long long)nb * nx * ny * nz;
    const bool small = (unsigned long long)total < (1ull << 32);
    // the (x, y) intermediate of the split path is pitched: rows of tp = nx rounded up to 4 floats
    const int tp = (nx + 3) & ~3;
    const long long wtotal = (long long)nb * tp * ny * nz;
    const bool split = g_blur_path == 0 && symmetric && small && radius <= kMaxRingR &&
                       (unsigned long long)wtotal < (1ull << 32);
    if (prev && !split) {  // only the split path's (x, y) kernels fuse the previous pair's DoG
        const int rc = vk_difference(prev, src, prev_dog, total, stream);
        if (rc != VK_OK) return rc;
        prev = nullptr;
        prev_dog = nullptr;
    }
    if (!symmetric || !small || radius > kMaxRingR)
        return launch_generic(src, dst, dog_out, half_out, nb, nx, ny, nz, radius, taps, st);
    if (g_blur_path == 0) {
        if (!split) return launch_generic(src, dst, dog_out, half_out, nb, nx, ny, nz, radius, taps, st);
        float* w = work;
        const bool own = w == nullptr || work_floats < wtotal || (reinterpret_cast<uintptr_t>(w) & 15) != 0;
        if (own) {
            cudaError_t e = cudaMallocAsync(&w, (wtotal + 4) * 4, st);
            if (e != cudaSuccess) return cuda_status(e, "blur scratch");
        }
        // work counters of the persistent (x, y) kernel: 4 floats past the intermediate, when the caller's
        // work buffer has them (else that kernel is not used)
        unsigned* counters = (own || work_floats >= wtotal + 4) ? reinterpret_cast<unsigned*>(w + wtotal) : nullptr;
        int rc;
        switch (radius) {
            case 1: rc = launch_split<1>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, w, tp, st, zchunk, prev, prev_dog, counters); break;
            case 2: rc = launch_split<2>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, w, tp, st, zchunk, prev, prev_dog, counters); break;
            case 3: rc = launch_split<3>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, w, tp, st, zchunk, prev, prev_dog, counters); break;
            case 4: rc = launch_split<4>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, w, tp, st, zchunk, prev, prev_dog, counters); break;
            case 5: rc = launch_split<5>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, w, tp, st, zchunk, prev, prev_dog, counters); break;
            case 6: rc = launch_split<6>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, w, tp, st, zchunk, prev, prev_dog, counters); break;
            case 7: rc = launch_split<7>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, w, tp, st, zchunk, prev, prev_dog, counters); break;
            case 8: rc = launch_split<8>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, w, tp, st, zchunk, prev, prev_dog, counters); break;
            case 9: rc = launch_split<9>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, w, tp, st, zchunk, prev, prev_dog, counters); break;
            default: rc = launch_split<10>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, w, tp, st, zchunk, prev, prev_dog, counters); break;
        }
        if (own) cudaFreeAsync(w, st);
        return rc;
    }
    switch (radius) {
        case 1: return launch_ring<1>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, st);
        case 2: return launch_ring<2>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, st);
        case 3: return launch_ring<3>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, st);
        case 4: return launch_ring<4>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, st);
        case 5: return launch_ring<5>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, st);
        case 6: return launch_ring<6>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, st);
        case 7: return launch_ring<7>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, st);
        case 8: return launch_ring<8>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, st);
        case 9: return launch_ring<9>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, st);
        default: return launch_ring<10>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, st);
    }
}

extern "C" int vk_blur3d(const float* src, float* dst, float* dog_out, float* half_out, int nb, int nx, int ny,
                         int nz, const float* taps_host, int radius, void* stream) {
    return vk_blur3d_ws(src, dst, dog_out, half_out, nb, nx, ny, nz, taps_host, radius, nullptr, 0, stream);
}

extern "C" int vk_subsample_half(const float* src, float* dst, int nb, int nx, int ny, int nz, void* stream) {
    if (!src || !dst || nb < 0 || nx < 2 || ny < 2 || nz < 2) {
        set_error("vk_subsample_half: cannot subsample dims (%d, %d, %d): every dim must be >= 2", nx, ny, nz);
        return VK_ERR_PARAMETER;
    }
    long long total = (long long)nb * (nx / 2) * (ny / 2) * (nz / 2);
    if (total == 0) return VK_OK;
    subsample_kernel<<<(unsigned)((total + 255) / 256), 256, 0, as_stream(stream)>>>(src, dst, nx, ny, nz, total);
    count_launch();
    return cuda_status(cudaGetLastError(), "subsample launch");
}

extern "C" int vk_difference(const float* a, const float* b, float* out, long long n, void* stream) {
    if (!a || !b || !out || n < 0) {
        set_error("vk_difference: bad arguments");
        return VK_ERR_PARAMETER;
    }
    if (n == 0) return VK_OK;
    cudaStream_t st = as_stream(stream);
    bool aligned = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    long long n4 = aligned ? n / 4 : 0;
    if (n4 > 0) {
        long long blocks = (n4 + 255) / 256;
        if (blocks > 148 * 16) blocks = 148 * 16;
        difference_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const float4*>(a),
                                                            reinterpret_cast<const float4*>(b),
                                                            reinterpret_cast<float4*>(out), n4);
        count_launch();
    }
    long long start = n4 * 4;
    if (start < n) {
        difference_tail_kernel<<<(unsigned)((n - start + 255) / 256), 256, 0, st>>>(a, b, out, start, n);
        count_launch();
    }
    return cuda_status(cudaGetLastError(), "difference launch");
}

extern "C" int vk_transpose_zfast_to_xfast(const float* src, float* dst, int nb, int nx, int ny, int nz, void* stream) {
    if (!src || !dst || nb < 0 || nx < 1 || ny < 1 || nz < 1) {
        set_error("vk_transpose: bad arguments");
        return VK_ERR_PARAMETER;
    }
    if (nb == 0) return VK_OK;
    // src [b][x][y][z]: slow axis x (n0 = nx), fast axis z (n2 = nz).
    dim3 grid((nz + 31) / 32, (nx + 31) / 32, nb * ny);
    transpose_xz_kernel<<<grid, dim3(32, 8), 0, as_stream(stream)>>>(src, dst, nx, ny, nz);
    count_launch();
    return cuda_status(cudaGetLastError(), "transpose launch");
}

extern "C" int vk_transpose_xfast_to_zfast(const float* src, float* dst, int nb, int nx, int ny, int nz, void* stream) {
    if (!src || !dst || nb < 0 || nx < 1 || ny < 1 || nz < 1) {
        set_error("vk_transpose: bad arguments");
        return VK_ERR_PARAMETER;
    }
    if (nb == 0) return VK_OK;
    // src [b][z][y][x]: slow axis z (n0 = nz), fast axis x (n2 = nx).
    dim3 grid((nx + 31) / 32, (nz + 31) / 32, nb * ny);
    transpose_xz_kernel<<<grid, dim3(32, 8), 0, as_stream(stream)>>>(src, dst, nz, ny, nx);
    count_launch();
    return cuda_status(cudaGetLastError(), "transpose launch");
}

extern "C" int vk_small_octaves(int n_oct, int levels, int handoff, const int* dims_host, float* const* level_ptrs_host,
                                float* const* dog_ptrs_host, const int* radius_host, const float* taps_host, int nb,
                                void* stream) {
    if (n_oct < 1 || n_oct > kSmallMaxOct || levels < 2 || levels > kSmallMaxLev || !dims_host || !level_ptrs_host ||
        !dog_ptrs_host || !radius_host || !taps_host || nb < 0) {
        set_error("vk_small_octaves: bad arguments (n_oct=%d levels=%d)", n_oct, levels);
        return VK_ERR_PARAMETER;
    }
    SmallOctaves so{};
    so.n_oct = n_oct;
    so.levels = levels;
    so.handoff = handoff;
    for (int o = 0; o < n_oct; ++o) {
        for (int a = 0; a < 3; ++a) so.dims[o][a] = dims_host[3 * o + a];
        if ((long long)so.dims[o][0] * so.dims[o][1] * so.dims[o][2] > kSmallMaxVox) {
            set_error("vk_small_octaves: octave %d has more than %d voxels", o, kSmallMaxVox);
            return VK_ERR_PARAMETER;
        }
        for (int i = 0; i < levels; ++i) so.lv[o][i] = level_ptrs_host[o * levels + i];
        for (int i = 0; i + 1 < levels; ++i) so.dog[o][i] = dog_ptrs_host[o * levels + i];
    }
    for (int i = 1; i < levels; ++i) {
        so.radius[i] = radius_host[i];
        if (so.radius[i] < 1 || 2 * so.radius[i] + 1 > VK_MAX_TAPS) {
            set_error("vk_small_octaves: bad radius %d", so.radius[i]);
            return VK_ERR_PARAMETER;
        }
        for (int t = 0; t < 2 * so.radius[i] + 1; ++t) so.taps[i][t] = taps_host[i * VK_MAX_TAPS + t];
    }
    if (nb == 0) return VK_OK;
    const int smem = 3 * kSmallMaxVox * 4;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(small_octaves_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return cuda_status(e, "small octaves attribute");
        configured = true;
    }
    small_octaves_kernel<<<nb, kSmallThreads, smem, as_stream(stream)>>>(so);
    count_launch();
    return cuda_status(cudaGetLastError(), "small octaves launch");
}
