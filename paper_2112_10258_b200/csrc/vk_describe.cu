// vk_describe.cu -- SIFT-Rank, BRIEF and RRIEF descriptors.
//
// Reference: descriptor.py:227-263 (sift_rank_descriptor), descriptor.py:77-83
// (rank_vector), descriptor.py:96-111 (extract_patch), descriptor.py:196-224
// (preblur_patch, _pair_samples, brief/rrief), descriptor.py:309-316 (packing).
//
// SIFT-Rank: one CTA per (keypoint, frame), persistent.  Votes (|R^T g| into
// spatial-octant x gradient-octant bins) are bit-exact; the 64 bins are
// summed in a parallel order with a rigorous bound against the reference's
// sequential np.add.at order.  The output is only the stable rank vector, so
// if every adjacent pair of the sorted bins is separated by more than the
// bound the ranks are exact; otherwise the CTA re-accumulates in reference
// order (one warp, lane-by-lane broadcast).
//
// BRIEF / RRIEF: one CTA per frame.  The side^3 reoriented patch is sampled
// from the source volume (fp64 trilinear, cast to fp32) straight into shared
// memory, pre-blurred there with the same non-FMA separable blur as the
// pyramid, then the point pairs are sampled (fp64 trilinear on the fp32 patch)
// and turned into packed bits or stable ranks.
#include "vk_common.cuh"

namespace vk {

constexpr int kSrThreads = 128;
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

// Fast vote: fp32 magnitude (|R^T g| = |g|, relative error <= kVoteRel against
// the reference's fp64 |R^T g|) and octant bits decided in fp32 whenever the
// rotated component clears its error bound; otherwise that voxel's bits are
// recomputed with the reference's fp64 FMA chain.  Returns -1 for zero
// gradients (their reference vote is exactly 0.0 and changes no bin).
VK_D int sr_vote_fast(const float* data, int nx, int ny, int nz, int cx, int cy, int cz, int packed, const double* R,
                      const float* Rf, float& mag, bool& inside) {
    const int ox = unpack_off(packed, 0), oy = unpack_off(packed, 1), oz = unpack_off(packed, 2);
    const int x = cx + ox, y = cy + oy, z = cz + oz;
    inside = x >= 0 && y >= 0 && z >= 0 && x < nx && y < ny && z < nz;
    if (!inside) return -1;
    const Nb6 n = load_nb6(data, nx, ny, nz, x, y, z);
    float gx, gy, gz;
    grad32(n, gx, gy, gz);
    if (gx == 0.f && gy == 0.f && gz == 0.f) return -1;
    mag = norm3_f32(gx, gy, gz);
    const float fx = (float)ox, fy = (float)oy, fz = (float)oz;
    // rotated offset / gradient (error <= ~5 u32 of the L1 norms; bound 1e-6)
    const float eo = 1.0e-6f * (fabsf(fx) + fabsf(fy) + fabsf(fz));
    const float eg = 1.0e-6f * (fabsf(gx) + fabsf(gy) + fabsf(gz)) + 1.0e-40f;
    float r[3], g[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        r[j] = fmaf(fz, Rf[6 + j], fmaf(fy, Rf[3 + j], fx * Rf[j]));
        g[j] = fmaf(gz, Rf[6 + j], fmaf(gy, Rf[3 + j], gx * Rf[j]));
    }
    const bool zero_off = (ox | oy | oz) == 0;
    const bool sure = (zero_off || (fabsf(r[0]) > eo && fabsf(r[1]) > eo && fabsf(r[2]) > eo)) &&
                      fabsf(g[0]) > eg && fabsf(g[1]) > eg && fabsf(g[2]) > eg;
    if (sure)
        return 8 * ((r[0] > 0.f) + 2 * (r[1] > 0.f) + 4 * (r[2] > 0.f)) + (g[0] > 0.f) + 2 * (g[1] > 0.f) +
               4 * (g[2] > 0.f);
    double x64, y64, z64;
    grad64(n, x64, y64, z64);
    const double o0 = (double)ox, o1 = (double)oy, o2 = (double)oz;
    const double r0 = dot3_blas(o0, o1, o2, R[0], R[3], R[6]);
    const double r1 = dot3_blas(o0, o1, o2, R[1], R[4], R[7]);
    const double r2 = dot3_blas(o0, o1, o2, R[2], R[5], R[8]);
    const double g0 = dot3_blas(x64, y64, z64, R[0], R[3], R[6]);
    const double g1 = dot3_blas(x64, y64, z64, R[1], R[4], R[7]);
    const double g2 = dot3_blas(x64, y64, z64, R[2], R[5], R[8]);
    return 8 * ((r0 > 0.0) + 2 * (r1 > 0.0) + 4 * (r2 > 0.0)) + (g0 > 0.0) + 2 * (g1 > 0.0) + 4 * (g2 > 0.0);
}

// Stable ascending ranks of 64 values: rank_b = #{j : w_j < w_b or (w_j == w_b and j < b)}.
VK_D int stable_rank(const double* w, int n, int b) {
    const double wb = w[b];
    int r = 0;
    for (int j = 0; j < n; ++j) r += (w[j] < wb) || (w[j] == wb && j < b);
    return r;
}

__global__ void __launch_bounds__(kSrThreads)
siftrank_kernel(const vk_frame* __restrict__ frames, const double* __restrict__ rot, const int* __restrict__ n_dev,
                int n_max, const vk_kp* __restrict__ kps, const vk_level* __restrict__ levels,
                const vk_ball* __restrict__ balls, const int* __restrict__ ball_offsets, uint8_t* __restrict__ out,
                int exact_only) {
    extern __shared__ double part[];  // [64][kSrThreads]
    __shared__ double w[kSrBins];
    __shared__ int order[kSrBins];
    __shared__ double Rs[9];
    __shared__ float Rfs[9];
    __shared__ int n_inside, exact;
    const int tid = threadIdx.x;
    const int n = n_dev ? min(*n_dev, n_max) : n_max;
    for (int item = blockIdx.x; item < n; item += gridDim.x) {
        const vk_frame fr = frames[item];
        const vk_kp kp = kps[fr.kp];
        const vk_level L = levels[kp.lvl];
        const float* data = L.base + (long long)kp.vol * L.vol_stride;
        const vk_ball ball = balls[kp.ball];
        if (tid < 9) {
            Rs[tid] = rot[(long long)item * 9 + tid];
            Rfs[tid] = (float)Rs[tid];
        }
        if (tid == 0) { n_inside = 0; exact = exact_only; }
        for (int b = 0; b < kSrBins; ++b) part[b * kSrThreads + tid] = 0.0;
        __syncthreads();
        double R[9];
        float Rf[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) {
            R[e] = Rs[e];
            Rf[e] = Rfs[e];
        }
        int cnt = 0;
        if (!exact_only) {
            for (int j = tid; j < ball.count; j += kSrThreads) {
                float mag;
                bool inside;
                const int bin = sr_vote_fast(data, L.nx, L.ny, L.nz, kp.ix, kp.iy, kp.iz,
                                             __ldg(ball_offsets + ball.start + j), R, Rf, mag, inside);
                cnt += inside;
                if (bin >= 0) part[bin * kSrThreads + tid] = dadd(part[bin * kSrThreads + tid], (double)mag);
            }
            if (cnt) atomicAdd(&n_inside, cnt);
            __syncthreads();
            if (tid < kSrBins) {
                double s = 0.0;
                for (int t = 0; t < kSrThreads; ++t) s = dadd(s, part[tid * kSrThreads + t]);
                w[tid] = s;
            }
            __syncthreads();
            if (tid < kSrBins) order[stable_rank(w, kSrBins, tid)] = tid;
            __syncthreads();
            if (tid == 0) {
                const double per = (double)((ball.count + kSrThreads - 1) / kSrThreads) + kSrThreads;
                const double epsrel = 2.0 * (kVoteRel + gamma_k((double)n_inside) + gamma_k(per));
                const double epsabs = kVoteAbs * n_inside;
                for (int r = 0; r + 1 < kSrBins; ++r) {
                    const double a = w[order[r]], b = w[order[r + 1]];
                    if (a == 0.0 && b == 0.0) continue;  // exact empty-bin ties
                    const double ahi = a == 0.0 ? 0.0 : dadd(a, a * epsrel + epsabs);
                    const double blo = dsub(b, b * epsrel + epsabs);
                    if (!(ahi < blo)) { exact = 1; break; }
                }
            }
            __syncthreads();
        }
        if (exact) {
            if (tid < 32) {
                double acc0 = 0.0, acc1 = 0.0;
                for (int base = 0; base < ball.count; base += 32) {
                    const int j = base + tid;
                    double mag = 0.0;
                    bool inside;
                    int bin = -1;
                    if (j < ball.count)
                        bin = sr_vote(data, L.nx, L.ny, L.nz, kp.ix, kp.iy, kp.iz, __ldg(ball_offsets + ball.start + j), R,
                                      mag, inside);
                    for (int s = 0; s < 32; ++s) {
                        const int bs = __shfl_sync(0xffffffffu, bin, s);
                        const double vs = __shfl_sync(0xffffffffu, mag, s);
                        if (bs == tid) acc0 = dadd(acc0, vs);
                        else if (bs == tid + 32) acc1 = dadd(acc1, vs);
                    }
                }
                w[tid] = acc0;
                w[tid + 32] = acc1;
            }
            __syncthreads();
        }
        if (tid < kSrBins) out[(long long)item * kSrBins + tid] = (uint8_t)stable_rank(w, kSrBins, tid);
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kPatchThreads)
patch_kernel(int kind, const vk_frame* __restrict__ frames, const double* __restrict__ rot, const int* __restrict__ n_dev,
             int n_max, const vk_kp* __restrict__ kps, const double* __restrict__ pos, const double* __restrict__ sigma,
             const vk_level* __restrict__ source, int side, PatchParams pp, int radius,
             const double* __restrict__ pts, int npairs, uint8_t* __restrict__ bits_out, uint16_t* __restrict__ ranks_out) {
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

extern "C" int vk_describe_siftrank(const vk_frame* frames, const double* rot, const int* n_frames_dev, int n_frames_max,
                                    const vk_kp* kps, const vk_level* levels, const vk_ball* balls,
                                    const int* ball_offsets, uint8_t* ranks_out, int exact_only, void* stream) {
    if (!frames || !rot || n_frames_max < 0 || !kps || !levels || !balls || !ball_offsets || !ranks_out) {
        set_error("vk_describe_siftrank: bad arguments");
        return VK_ERR_PARAMETER;
    }
    if (n_frames_max == 0) return VK_OK;
    const int smem = kSrBins * kSrThreads * 8;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(siftrank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return cuda_status(e, "siftrank attribute");
        configured = true;
    }
    siftrank_kernel<<<grid_for(n_frames_max, 3), kSrThreads, smem, as_stream(stream)>>>(
        frames, rot, n_frames_dev, n_frames_max, kps, levels, balls, ball_offsets, ranks_out, exact_only);
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
        ranks_out);
    count_launch();
    return cuda_status(cudaGetLastError(), "patch launch");
}
