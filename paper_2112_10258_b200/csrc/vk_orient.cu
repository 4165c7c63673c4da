// vk_orient.cu -- spherical gradient histograms and orientation frames.
//
// Reference: orient.py:89-125 (gradient_histogram), orient.py:128-168
// (dominant_orientations), pipeline.py:41-67 (assign_orientations).
//
// orient_kernel: one 256-thread CTA per keypoint, persistent over the keypoint
// list (the count lives in device memory so the whole pipeline can be
// graph-captured), 3 CTAs/SM.  Fast path: the ball is walked in z-major order
// (coalesced gathers; interior balls software-pipelined, the neighbour loads of
// the next voxel in flight while the current one is binned, ori_walk_pipe);
// each voxel's vote is the fp32 |g| x window (within kVoteRel +
// kVoteAbs of the reference's fp64 vote) and its bin the exact nearest
// icosphere direction (lookup table, boundary cells deferred to a per-warp
// queue and resolved by a screened fp32 argmax with an fp64 fallback).  Votes
// are added with fire-and-forget fp64 reductions into a per-CTA histogram in
// L2 (two copies, by lane parity; any order).  Every decision the frames depend on (the top of the weight
// order, the secondary_ratio threshold) is checked against a rigorous bound on
// the difference between that sum and the reference's sequential np.add.at;
// only the bins of an uncertain decision are re-accumulated in the reference's
// order with fp64 votes (ori_exact_subset).  Either way the frames are the
// reference's.
#include "vk_ori.cuh"

namespace vk {


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



#ifndef VK_ORI_PIPE_BORDER
#define VK_ORI_PIPE_BORDER 0  // pipelined walk also for balls crossing the boundary: spills at 80 regs, measured slower
#endif
#ifndef VK_ORI_MIN_BLOCKS
#define VK_ORI_MIN_BLOCKS 3  // with the pipelined walk: 3 CTAs/SM without spills beat 4 with (B200)
#endif
// MODE 0: every keypoint, every path (exact, gradient / field volumes, staged,
// pipelined, plain).  MODE 1 / 2: the default fast path only (lookup table, no
// precomputed volumes), for the keypoints whose ball lies inside the volume
// (1) or crosses its boundary (2) -- two launches, each compiled with only its
// own pipelined walk, so neither pays the other's registers.
template <int MODE>
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
    load_ok_bits(sh.okb, pair_ok, K);
    const int n_kp = n_kp_dev ? min(*n_kp_dev, n_kp_max) : n_kp_max;
    const IcoSh* icp = ico.valid ? &ic : nullptr;
    const uint8_t* lutp = ico.valid && ico_lut ? lut : nullptr;
    if (lutp)
        for (int i = tid; i < kLutBytes / 4; i += kOriThreads)
            reinterpret_cast<uint32_t*>(lut)[i] = __ldg(reinterpret_cast<const uint32_t*>(ico_lut) + i);
    __syncthreads();

    for (int item = first_item(); item < n_kp; item += gridDim.x) {
        const vk_kp kp = kps[item];
        const vk_level L = levels[kp.lvl];
        const float* data = L.base + (long long)kp.vol * L.vol_stride;
        const vk_ball ball = balls[kp.ball];
        const double* win = windows + ball.window_start;
        const float* win32 = windows32 + ball.window_start;
        if (MODE != 0) {
            const bool interior = ball_interior(kp.ix, kp.iy, kp.iz, ball.r, L.nx, L.ny, L.nz);
            if ((MODE == 1) != interior) continue;  // CTA-uniform: the other launch takes this keypoint
        }
        if (VK_PREFETCH_NEXT && item + (int)gridDim.x < n_kp) {
            const vk_kp nk = kps[item + gridDim.x];
            const vk_level NL = levels[nk.lvl];
            prefetch_ball_l2(NL.base + (long long)nk.vol * NL.vol_stride, NL.nx, NL.ny, NL.nz, nk.ix, nk.iy, nk.iz,
                             balls[nk.ball].r);
        }
        zero_hist(hist, K);
        if (tid == 0) { sh.n_inside = 0; sh.exact = exact_only; sh.repair = 0; }
        __syncthreads();
        int inside_cnt = 0;
        const vk_gradlevel GL = grads ? grads[kp.lvl] : vk_gradlevel{};
        if constexpr (MODE != 0) {
            inside_cnt = MODE == 1 ? ori_walk_pipe<true>(kp, L, data, ball, ball_offsets, win32, sh.dirs, icp, lutp,
                                                         hist, sh.queue[tid >> 5])
                                   : ori_walk_pipe<false>(kp, L, data, ball, ball_offsets, win32, sh.dirs, icp, lutp,
                                                          hist, sh.queue[tid >> 5]);
        } else if (!exact_only && GL.bin != nullptr && GL.kind == 1) {
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
        } else if (!exact_only && VK_ORI_PIPE && lutp && icp &&
                   (VK_ORI_PIPE_BORDER || ball_interior(kp.ix, kp.iy, kp.iz, ball.r, L.nx, L.ny, L.nz))) {
#if VK_ORI_PIPE_BORDER
            inside_cnt = ball_interior(kp.ix, kp.iy, kp.iz, ball.r, L.nx, L.ny, L.nz)
                             ? ori_walk_pipe<true>(kp, L, data, ball, ball_offsets, win32, sh.dirs, icp, lutp, hist,
                                                   sh.queue[tid >> 5])
                             : ori_walk_pipe<false>(kp, L, data, ball, ball_offsets, win32, sh.dirs, icp, lutp, hist,
                                                    sh.queue[tid >> 5]);
#else
            inside_cnt = ori_walk_pipe<true>(kp, L, data, ball, ball_offsets, win32, sh.dirs, icp, lutp, hist,
                                             sh.queue[tid >> 5]);
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
            // DataError: orientation neighbourhood entirely outside (orient.py:109-110)
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
        if (tid < 32) warp_frames_from(sh.w, sh.order, K, sh.okb, ratio, max_frames, nframes + item,
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
    __shared__ unsigned okb[kOkWords];
    load_ok_bits(okb, pair_ok, K);
    for (int item = blockIdx.x; item < n; item += gridDim.x) {
        __syncthreads();
        for (int b = threadIdx.x; b < K; b += blockDim.x) w[b] = weights[(long long)item * K + b];
        __syncthreads();
        sort_desc(w, K, order);
        __syncthreads();
        if (threadIdx.x == 0) {
            int pr[VK_MAX_FRAMES], se[VK_MAX_FRAMES];
            const int nf = frames_from(w, order, K, okb, ratio, max_frames, pr, se);
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
        cudaError_t e = cudaFuncSetAttribute(orient_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        if (e != cudaSuccess) return cuda_status(e, "orient smem attribute");
        configured = true;
    }
    IcoT ico{};
    if (ico_host && K == 42) {
        ico.valid = 1;
        for (int v = 0; v < 12; ++v) {
            ico.vert[v] = ico_host[v];
            for (int m = 0; m < 5; ++m) ico.adj[v][m] = ico_host[12 + 5 * v + m];
            for (int m = 0; m < 5; ++m) ico.kind[v][m] = ico_host[72 + 5 * v + m];
        }
    }
#ifndef VK_ORI_SPLIT
#define VK_ORI_SPLIT 0  // 1: interior / border keypoints in two launches (measured slower: 2.11 vs 1.87 ms)
#endif
    const bool split = VK_ORI_SPLIT && !exact_only && !grads && ico.valid && ico_lut && !VK_ORI_STAGED;
    if (split) {
        for (int m = 1; m <= 2; ++m) {
            auto* kern = m == 1 ? orient_kernel<1> : orient_kernel<2>;
            const int grid = accum_grid(kern, kOriThreads, n_kp_max, 0);
            kern<<<grid, kOriThreads, 0, as_stream(stream)>>>(kps, n_kp_dev, n_kp_max, levels, balls, ball_offsets,
                                                              windows, windows32, dirs, K, pair_ok, secondary_ratio,
                                                              max_frames, weights, nframes, prim, sec, status,
                                                              exact_only, ico, ico_lut, grads, work);
            count_launch();
        }
        return cuda_status(cudaGetLastError(), "orient launch");
    }
    const int grid = accum_grid(orient_kernel<0>, kOriThreads, n_kp_max, dyn);
    orient_kernel<0><<<grid, kOriThreads, dyn, as_stream(stream)>>>(kps, n_kp_dev, n_kp_max, levels, balls, ball_offsets,
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
