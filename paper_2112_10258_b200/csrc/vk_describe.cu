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
#include "vk_sr.cuh"

namespace vk {

constexpr int kPatchThreads = 256;
constexpr int kMaxSide = 31;

struct PatchParams {
    double grid[kMaxSide];
    float taps[VK_MAX_TAPS];
};


// One CTA per work item = one keypoint and its F frames (contiguous in the
// frame list).  The ball is walked in z-major order (coalesced gathers);
// each voxel's gradient is computed once and voted into all F frames.
#ifndef VK_SR_MIN_BLOCKS
#define VK_SR_MIN_BLOCKS 3
#endif
// MODE 0: every keypoint; MODE 1 / 2: the fast path (no gradient volumes) for
// interior (1) or border-crossing (2) balls only, each launch compiled with its
// own pipelined walk (see orient_kernel).
template <int MODE>
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
    __shared__ float sring[kSrRingFloats];  // VK_SR_ASYNC: in-flight neighbour gathers of the interior walk
    const int tid = threadIdx.x;
    const int n = n_items_dev ? min(*n_items_dev, n_items_max) : n_items_max;
    if (tid < kSrThreads / 32) sqn[tid] = 0;  // (first use is after the item's __syncthreads)
    for (int item = first_item(); item < n; item += gridDim.x) {
        const int F = min(item_count[item], max_f);
        if (F <= 0) continue;
        const int first = item_first[item];
        const vk_kp kp = kps[frames[first].kp];
        const vk_level L = levels[kp.lvl];
        const float* data = L.base + (long long)kp.vol * L.vol_stride;
        const vk_ball ball = balls[kp.ball];
        if (MODE != 0 && (MODE == 1) != ball_interior(kp.ix, kp.iy, kp.iz, ball.r, L.nx, L.ny, L.nz)) continue;
        if (VK_PREFETCH_NEXT && item + (int)gridDim.x < n && item_count[item + gridDim.x] > 0) {
            const vk_kp nk = kps[item + gridDim.x];  // items are keypoints (their frames are contiguous)
            const vk_level NL = levels[nk.lvl];
            prefetch_ball_l2(NL.base + (long long)nk.vol * NL.vol_stride, NL.nx, NL.ny, NL.nz, nk.ix, nk.iy, nk.iz,
                             balls[nk.ball].r);
        }
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
            if constexpr (MODE == 1)
                cnt = sr_walk_frames<true>(kp, L, data, nullptr, ball, ball_offsets, Rs, Rc, hist, F, sq[tid >> 5],
                                           sqn + (tid >> 5), sring);
            else if constexpr (MODE == 2)
                cnt = sr_walk_frames<false, true>(kp, L, data, nullptr, ball, ball_offsets, Rs, Rc, hist, F,
                                                  sq[tid >> 5], sqn + (tid >> 5));
            else if (ball_interior(kp.ix, kp.iy, kp.iz, ball.r, L.nx, L.ny, L.nz))
                cnt = sr_walk_frames<true>(kp, L, data, g4, ball, ball_offsets, Rs, Rc, hist, F, sq[tid >> 5],
                                           sqn + (tid >> 5), sring);
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
#ifndef VK_SR_SPLIT
#define VK_SR_SPLIT 0  // 1: interior / border keypoints in two launches (measured slower: 2.55 vs 2.08 ms)
#endif
    if (VK_SR_SPLIT && !exact_only && !grads) {
        for (int m = 1; m <= 2; ++m) {
            auto* kern = m == 1 ? siftrank_kernel<1> : siftrank_kernel<2>;
            kern<<<accum_grid(kern, kSrThreads, n_items_max), kSrThreads, 0, as_stream(stream)>>>(
                frames, rot, item_first, item_count, n_items_dev, n_items_max, kps, levels, balls, ball_offsets, max_f,
                ranks_out, exact_only, stats, grads, work);
            count_launch();
        }
        return cuda_status(cudaGetLastError(), "siftrank launch");
    }
    siftrank_kernel<0><<<accum_grid(siftrank_kernel<0>, kSrThreads, n_items_max), kSrThreads, 0, as_stream(stream)>>>(
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
