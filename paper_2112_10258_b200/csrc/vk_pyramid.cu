// vk_pyramid.cu -- separable 3-D Gaussian blur with fused DoG and 2x
// subsample epilogues, standalone subsample / difference, layout transposes.
//
// Reference: scalespace.py:73-137 (convolve_array, subsample_half) and
// scalespace.py:237-251 (build_dog_pyramid).
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
#include <stdio.h>

#include "vk_common.cuh"

namespace vk {

struct Taps {
    float w[VK_MAX_TAPS];
};

constexpr int kTX = 32;       // tile width in x (one warp lane per column)
constexpr int kTY = 32;       // tile height in y (8 warps x 4 rows)
constexpr int kThreads = 256;
constexpr int kMaxRingR = 10; // register-ring kernel covers radius 1..10

template <int R>
struct BlurGeom {
    static constexpr int P = 2 * R + 1;
    static constexpr int ROWS = kTY + 2 * R;               // rows of the x-pass tile
    static constexpr int COLS = kTX + 2 * R;               // input columns per row
    static constexpr int V4 = (8 + 2 * R + 3) / 4;         // float4 per x-pass segment
    static constexpr int XPW = 24 + 4 * V4;                // input row pitch (>= COLS)
    static constexpr int XS = kTX + 4;                     // x-pass tile pitch
    static constexpr int SMEM = (2 * ROWS * XPW + ROWS * XS) * 4;
};

// Products of two taps at once: packed FMUL2 (two IEEE-rounded products); the
// sums stay scalar FADDs in tap order.  ptxas never contracts FMUL2 + FADD
// (it does contract FMUL2 + FADD2 into FFMA2, which would break parity).
VK_D float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

template <int R>
__global__ void __launch_bounds__(kThreads, 2)
blur3d_ring_kernel(const float* __restrict__ src, float* __restrict__ dst, float* __restrict__ dog,
                   float* __restrict__ half, int nx, int ny, int nz, int tz, int nzc, Taps taps) {
    using G = BlurGeom<R>;
    constexpr int P = G::P;
    extern __shared__ float4 smem4[];
    float* in_s = reinterpret_cast<float*>(smem4);
    float* x_s = in_s + 2 * G::ROWS * G::XPW;

    const int b = blockIdx.z / nzc;
    const int zc = blockIdx.z - b * nzc;
    const int z_start = zc * tz;
    const int z_end = min(nz, z_start + tz);
    const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
    const long long plane = (long long)nx * ny;
    const long long vol = plane * nz;
    const float* s = src + b * vol;
    const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;

    // Loop-invariant clamped x offsets of this lane's (up to 2) tile columns.
    constexpr int NCOL = (G::COLS + 31) / 32;
    int gxo[NCOL];
#pragma unroll
    for (int k = 0; k < NCOL; ++k) gxo[k] = clampi(x0 - R + lane + 32 * k, 0, nx - 1);

    auto load_plane = [&](int zp, int buf) {
        const float* sp = s + (long long)clampi(zp, 0, nz - 1) * plane;
        float* d = in_s + buf * G::ROWS * G::XPW;
#pragma unroll
        for (int r = wy; r < G::ROWS; r += kThreads / 32) {
            const unsigned roff = (unsigned)clampi(y0 - R + r, 0, ny - 1) * (unsigned)nx;
            float* drow = d + r * G::XPW + lane;
#pragma unroll
            for (int k = 0; k < NCOL; ++k)
                if (lane + 32 * k < G::COLS) cp_async4(drow + 32 * k, sp + (roff + (unsigned)gxo[k]));
        }
        cp_async_commit();
    };

    float ring[4][P];
    float prev[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        prev[j] = 0.f;
#pragma unroll
        for (int t = 0; t < P; ++t) ring[j][t] = 0.f;
    }

    const int zp0 = z_start - R;
    const int nplanes = (z_end - z_start) + 2 * R;
    load_plane(zp0, 0);
    for (int p = 0; p < nplanes; ++p) {
        if (p + 1 < nplanes) load_plane(zp0 + p + 1, (p + 1) & 1);
        else cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        // ---- x-pass: 4 threads per tile row, 8 outputs each (pairs of outputs share FMUL2) ----
        {
            const int r = tid >> 2, sg = tid & 3;
            if (r < G::ROWS) {
                const float4* row = reinterpret_cast<const float4*>(in_s + (p & 1) * G::ROWS * G::XPW + r * G::XPW + sg * 8);
                float v[4 * G::V4];
#pragma unroll
                for (int q = 0; q < G::V4; ++q) {
                    float4 t4 = row[q];
                    v[4 * q] = t4.x; v[4 * q + 1] = t4.y; v[4 * q + 2] = t4.z; v[4 * q + 3] = t4.w;
                }
                float o[8];
#pragma unroll
                for (int k = 0; k < 8; k += 2) {
                    float2 pr = fmul2(make_float2(taps.w[0], taps.w[0]), make_float2(v[k], v[k + 1]));
                    float a0 = pr.x, a1 = pr.y;
#pragma unroll
                    for (int t = 1; t < P; ++t) {
                        pr = fmul2(make_float2(taps.w[t], taps.w[t]), make_float2(v[k + t], v[k + 1 + t]));
                        a0 = fadd(a0, pr.x);
                        a1 = fadd(a1, pr.y);
                    }
                    o[k] = a0;
                    o[k + 1] = a1;
                }
                float4* xo = reinterpret_cast<float4*>(x_s + r * G::XS + sg * 8);
                xo[0] = make_float4(o[0], o[1], o[2], o[3]);
                xo[1] = make_float4(o[4], o[5], o[6], o[7]);
            }
        }
        __syncthreads();
        // ---- y-pass into the per-column z ring ----
        {
            float col[4 + 2 * R];
#pragma unroll
            for (int i = 0; i < 4 + 2 * R; ++i) col[i] = x_s[(4 * wy + i) * G::XS + lane];
#pragma unroll
            for (int j = 0; j < 4; j += 2) {
                float2 pr = fmul2(make_float2(taps.w[0], taps.w[0]), make_float2(col[j], col[j + 1]));
                float a0 = pr.x, a1 = pr.y;
#pragma unroll
                for (int t = 1; t < P; ++t) {
                    pr = fmul2(make_float2(taps.w[t], taps.w[t]), make_float2(col[j + t], col[j + 1 + t]));
                    a0 = fadd(a0, pr.x);
                    a1 = fadd(a1, pr.y);
                }
#pragma unroll
                for (int t = 0; t < P - 1; ++t) {
                    ring[j][t] = ring[j][t + 1];
                    ring[j + 1][t] = ring[j + 1][t + 1];
                }
                ring[j][P - 1] = a0;
                ring[j + 1][P - 1] = a1;
            }
        }
        if (p < 2 * R) continue;
        // ---- z-pass + epilogues for output plane zo ----
        const int zo = zp0 + p - R;
        const int gx = x0 + lane;
        float out[4];
#pragma unroll
        for (int j = 0; j < 4; j += 2) {
            float2 pr = fmul2(make_float2(taps.w[0], taps.w[0]), make_float2(ring[j][0], ring[j + 1][0]));
            float a0 = pr.x, a1 = pr.y;
#pragma unroll
            for (int t = 1; t < P; ++t) {
                pr = fmul2(make_float2(taps.w[t], taps.w[t]), make_float2(ring[j][t], ring[j + 1][t]));
                a0 = fadd(a0, pr.x);
                a1 = fadd(a1, pr.y);
            }
            out[j] = a0;
            out[j + 1] = a1;
        }
        {
            // 32-bit offsets within the volume (a volume holds < 2^31 voxels)
            float* dv = dst + b * vol + (long long)zo * plane;
            float* gv = dog ? dog + b * vol + (long long)zo * plane : nullptr;
            const float* sv = src + b * vol + (long long)zo * plane;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int gy = y0 + 4 * wy + j;
                if (gx < nx && gy < ny) {
                    const unsigned o = (unsigned)gy * (unsigned)nx + (unsigned)gx;
                    dv[o] = out[j];
                    if (gv) gv[o] = __fsub_rn(__ldg(sv + o), out[j]);
                }
            }
        }
        if (half != nullptr && (zo & 1)) {
            float np_[4], no_[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                np_[j] = __shfl_down_sync(0xffffffffu, prev[j], 1);
                no_[j] = __shfl_down_sync(0xffffffffu, out[j], 1);
            }
            const int hx = gx >> 1, hz = zo >> 1;
            const int hnx = nx >> 1, hny = ny >> 1, hnz = nz >> 1;
            if ((lane & 1) == 0 && hx < hnx && hz < hnz) {
#pragma unroll
                for (int j = 0; j < 4; j += 2) {
                    const int hy = (y0 + 4 * wy + j) >> 1;
                    if (hy < hny) {
                        // (dx, dy, dz) order of scalespace.py:129-135, then /8.
                        float sm = prev[j];
                        sm = fadd(sm, out[j]);
                        sm = fadd(sm, prev[j + 1]);
                        sm = fadd(sm, out[j + 1]);
                        sm = fadd(sm, np_[j]);
                        sm = fadd(sm, no_[j]);
                        sm = fadd(sm, np_[j + 1]);
                        sm = fadd(sm, no_[j + 1]);
                        half[(((long long)b * hnz + hz) * hny + hy) * hnx + hx] = fmul(sm, 0.125f);
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) prev[j] = out[j];
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

__global__ void __launch_bounds__(512)
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
        for (int lvi = 1; lvi < so.levels; ++lvi) {
            const int R = so.radius[lvi];
            const float* w = so.taps[lvi];
            small_pass(src, xb, nx, ny, nz, 0, R, w);
            __syncthreads();
            small_pass(xb, yb, nx, ny, nz, 1, R, w);
            __syncthreads();
            small_pass(yb, xb, nx, ny, nz, 2, R, w);  // xb now holds level lvi
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
        cudaError_t e = cudaFuncSetAttribute(blur3d_ring_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        if (e != cudaSuccess) return cuda_status(e, "blur3d attribute");
        configured = true;
    }
    const int tiles = ((nx + kTX - 1) / kTX) * ((ny + kTY - 1) / kTY);
    // z-chunking only when the batch does not fill ~1.5 waves (2 CTAs / SM):
    // every chunk re-reads and re-blurs 2R halo planes.
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int nzc = 1;
    while ((long long)tiles * nb * nzc < 3 * sms && (nz + nzc) / (nzc + 1) >= 16) ++nzc;
    int tz = (nz + nzc - 1) / nzc;
    tz += tz & 1;
    nzc = (nz + tz - 1) / tz;
    dim3 grid((nx + kTX - 1) / kTX, (ny + kTY - 1) / kTY, nb * nzc);
    blur3d_ring_kernel<R><<<grid, kThreads, G::SMEM, st>>>(src, dst, dog, half, nx, ny, nz, tz, nzc, taps);
    count_launch();
    return cuda_status(cudaGetLastError(), "blur3d launch");
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

extern "C" int vk_blur3d(const float* src, float* dst, float* dog_out, float* half_out, int nb, int nx, int ny,
                         int nz, const float* taps_host, int radius, void* stream) {
    if (!src || !dst || !taps_host || nb < 0 || nx < 1 || ny < 1 || nz < 1 || radius < 1 ||
        2 * radius + 1 > VK_MAX_TAPS) {
        set_error("vk_blur3d: bad arguments (nb=%d dims=%d,%d,%d radius=%d)", nb, nx, ny, nz, radius);
        return VK_ERR_PARAMETER;
    }
    if (nb == 0) return VK_OK;
    Taps taps{};
    for (int i = 0; i < 2 * radius + 1; ++i) taps.w[i] = taps_host[i];
    cudaStream_t st = as_stream(stream);
    if (half_out && (nx < 2 || ny < 2 || nz < 2)) half_out = nullptr;
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
        case 10: return launch_ring<10>(src, dst, dog_out, half_out, nb, nx, ny, nz, taps, st);
        default: return launch_generic(src, dst, dog_out, half_out, nb, nx, ny, nz, radius, taps, st);
    }
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
    small_octaves_kernel<<<nb, 512, smem, as_stream(stream)>>>(so);
    count_launch();
    return cuda_status(cudaGetLastError(), "small octaves launch");
}
