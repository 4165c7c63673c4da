// vk_orsr.cu -- orientation frames and SIFT-Rank descriptors of a keypoint in
// one CTA (fused orient_kernel + siftrank_kernel).
//
// Reference: orient.py:89-125 (gradient_histogram), orient.py:128-168
// (dominant_orientations), pipeline.py:41-67 (assign_orientations),
// descriptor.py:227-263 (sift_rank_descriptor).  Both stages visit the same
// integer ball around the same lattice centre (orient.py:63-74 offsets,
// keypoint_local) and need the same central-difference gradients
// (volume.py:244-264).
//
// The separate kernels each gather the ball's six-neighbour stencils from
// L1 / L2 / HBM: latency-bound walks (long-scoreboard stalls), and the
// SIFT-Rank kernel re-reads the keypoint levels from HBM after the
// orientation kernel evicted them.  Here one persistent CTA per keypoint
// stages the stencil set of its ball ONCE into shared memory -- a compact
// row-by-row layout of the ball plus its axis neighbours (tables.ball_sphere:
// 11.5 / 21.7 / 41.2 KB for the three keypoint levels of the default config),
// one cp.async row per warp instruction, the next keypoint's rows prefetched
// into L2 meanwhile -- and both walks read their neighbours with shared loads
// through a per-voxel index table.  In between, the frames are decided in the
// CTA (certified fast sums + exact repair, vk_ori.cuh), so the SIFT-Rank walk
// runs right after the orientation walk on the same staged data.
//
// Votes, certification bounds, deferred uncertain decisions and exact repairs
// are those of the separate kernels (the same device functions), so the
// frames and rank vectors are the reference's bit for bit.  Spheres that
// cross the volume boundary are staged with clamped (replicated) coordinates:
// the staged neighbour pairs are then those of the reference's one-sided
// differences.  Every ball of the plan must fit the staging buffer (the host
// falls back to the separate kernels otherwise).
//
// Output: frame counts / (primary, secondary) pairs per keypoint like
// vk_orient, and each frame's 64 ranks in a per-keypoint slot
// (desc_kp[(kp * max_frames + f) * 64]); vk_scatter_frame_rows moves them into
// the frame order vk_expand_frames assigns.
#include "vk_ori.cuh"
#include "vk_sr.cuh"

namespace vk {

constexpr int kOsThreads = kOriThreads;  // OriShared / ori_exact_subset are sized for this
static_assert(kOsThreads % kSrBins == 0, "ranking maps threads to (frame, bin)");

struct OsShared {
    OriShared o;  // orientation walk / certification / repair (xb, xv, wmask reused by SIFT-Rank)
    IcoSh ic;
    __align__(16) uint8_t lut[kLutBytes];
    double Rs[VK_MAX_FRAMES * 9];
    float4 Rc[VK_MAX_FRAMES * kRcPerFrame];
    double w[kSrBins];
    int unc[kSrBins];
    double w4[kOsThreads / kSrBins][kSrBins];
    int order4[kOsThreads / kSrBins][kSrBins];
    int badf[kOsThreads / kSrBins];
    int4 sq[kOsThreads / 32][kSrQueue];  // deferred uncertain SIFT-Rank octants, per warp
    int sqn[kOsThreads / 32];
    int prim[VK_MAX_FRAMES], sec[VK_MAX_FRAMES];
    int nf;
};
constexpr size_t kOsStateBytes = (sizeof(OsShared) + 15) & ~size_t(15);

// Copy the keypoint's stencil sphere rows into box: each warp loads 32 row
// records at once and issues one 4-byte cp.async per lane and element of each
// row (rows are <= 31 floats for balls up to radius ~14).  CLAMP: the sphere
// crosses the volume boundary -- coordinates are clamped (replicate), so the
// staged x / y / z neighbour pairs of a border voxel are exactly the pairs of
// the reference's one-sided differences (volume.py:259-263); voxels outside
// the volume are staged but never visited.  The caller waits and synchronises.
template <bool CLAMP>
VK_D void stage_sphere(const float* __restrict__ data, int nx, int ny, int nz, const vk_kp& kp,
                       const int4* __restrict__ rows, int n_rows, float* box) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const unsigned plane = (unsigned)nx * (unsigned)ny;
    for (int r0 = 32 * wid; r0 < n_rows; r0 += 32 * nw) {
        const int4 mine = r0 + lane < n_rows ? __ldg(rows + r0 + lane) : make_int4(0, 0, 0, 0);
        const int nr = min(32, n_rows - r0);
        for (int k = 0; k < nr; ++k) {
            const int dy = __shfl_sync(0xffffffffu, mine.x, k), dz = __shfl_sync(0xffffffffu, mine.y, k);
            const int m = __shfl_sync(0xffffffffu, mine.z, k), st = __shfl_sync(0xffffffffu, mine.w, k);
            for (int l = lane; l <= 2 * m; l += 32) {
                int x = kp.ix - m + l, y = kp.iy + dy, z = kp.iz + dz;
                if (CLAMP) {
                    x = clampi(x, 0, nx - 1);
                    y = clampi(y, 0, ny - 1);
                    z = clampi(z, 0, nz - 1);
                }
                cp_async4(box + st + l, data + ((unsigned)z * plane + (unsigned)y * (unsigned)nx + (unsigned)x));
            }
        }
    }
    cp_async_commit();
}

// L2 prefetch of a keypoint's stencil rows (both ends of each row).
VK_D void prefetch_sphere(const float* __restrict__ data, unsigned nx, unsigned plane, const vk_kp& kp,
                          const int4* __restrict__ rows, int n_rows) {
    for (int r = threadIdx.x; r < n_rows; r += blockDim.x) {
        const int4 rw = __ldg(rows + r);
        const float* src = data + ((unsigned)(kp.iz + rw.y) * plane + (unsigned)(kp.iy + rw.x) * nx +
                                   (unsigned)(kp.ix - rw.z));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(src));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(src + 2 * rw.z));
    }
}

// The six neighbours of a staged ball voxel (entry e of tables.ball_sphere).
VK_D Nb6 sphere_nb6(const float* box, const int4& e) {
    const int c = e.y & 0xffff;
    Nb6 n;
    n.xh = box[c + 1];
    n.xl = box[c - 1];
    n.yh = box[(unsigned)e.y >> 16];
    n.yl = box[e.z & 0xffff];
    n.zh = box[(unsigned)e.z >> 16];
    n.zl = box[e.w];
    n.sx = n.sy = n.sz = 0.5f;
    return n;
}

// ori_walk over the staged sphere: the same votes, bins and deferred
// lookup-table misses (resolved from global memory, where the values are the
// same).  !INTERIOR: voxels outside the volume are skipped and border axes
// take one-sided differences.  Returns this thread's count of in-volume voxels.
template <bool INTERIOR>
VK_D int ori_walk_sphere(const vk_kp& kp, const vk_level& L, const float* data, const float* box,
                         const int4* __restrict__ ent, int count, const float* __restrict__ win32, const double* dirs,
                         const IcoSh* icp, const uint8_t* lut, double* hist, int2* queue) {
    const int tid = threadIdx.x, lane = tid & 31, step = blockDim.x;
    const int nx = L.nx, plane = L.nx * L.ny;
    const int kc = (kp.iz * L.ny + kp.iy) * nx + kp.ix;
    hist = vote_copy(hist);
    auto resolve = [&](int2 e) {
        const unsigned c = (unsigned)e.x;
        const unsigned z = c / (unsigned)plane, rem = c - z * (unsigned)plane;
        const unsigned y = rem / (unsigned)nx, x = rem - y * (unsigned)nx;
        const Nb6 nb = load_nb6(data, L.nx, L.ny, L.nz, (int)x, (int)y, (int)z);
        float gx, gy, gz;
        grad32(nb, gx, gy, gz);
        red_vote(hist, nearest_dir_ico(dirs, *icp, nullptr, gx, gy, gz, nb), __int_as_float(e.y));
    };
    int qn = 0, cnt = 0;
    int4 en = tid < count ? __ldg(ent + tid) : make_int4(0, 0, 0, 0);
    int4 en2 = tid + step < count ? __ldg(ent + tid + step) : make_int4(0, 0, 0, 0);
    for (int base = 0; base < count; base += step) {
        const int j = base + tid;
        const int4 e = en;
        en = en2;
        if (j + 2 * step < count) en2 = __ldg(ent + j + 2 * step);
        int bin = -1;
        float vote = 0.f;
        bool miss = false;
        int c = 0;
        if (j < count) {
            const int ox = unpack_off(e.x, 0), oy = unpack_off(e.x, 1), oz = unpack_off(e.x, 2);
            const int x = kp.ix + ox, y = kp.iy + oy, z = kp.iz + oz;
            if (INTERIOR || (x >= 0 && y >= 0 && z >= 0 && x < L.nx && y < L.ny && z < L.nz)) {
                ++cnt;
                Nb6 nb = sphere_nb6(box, e);
                if (!INTERIOR) {
                    nb.sx = (x > 0 && x < L.nx - 1) ? 0.5f : 1.0f;
                    nb.sy = (y > 0 && y < L.ny - 1) ? 0.5f : 1.0f;
                    nb.sz = (z > 0 && z < L.nz - 1) ? 0.5f : 1.0f;
                }
                float gx, gy, gz;
                grad32(nb, gx, gy, gz);
                if (grad_nonzero(nb)) {
                    vote = nz_vote(fmul(norm3_f32(gx, gy, gz), __ldg(win32 + (ox * ox + oy * oy + oz * oz))));
                    bin = nearest_dir_lut(lut, gx, gy, gz, fabsf(gx), fabsf(gy), fabsf(gz));
                    miss = bin < 0;
                    c = kc + oz * plane + oy * nx + ox;
                }
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

// sr_walk_pipe over the staged sphere for NF frames: each voxel's fp32
// gradient once, voted into every frame; uncertain octants deferred per warp
// and resolved with the reference's fp64 chains (sr_resolve, global reload).
template <int NF, bool INTERIOR>
VK_D void sr_walk_sphere(const vk_kp& kp, const vk_level& L, const float* data, const float* box,
                         const int4* __restrict__ ent, int count, const double* Rs, const float4* Rc, double* hist,
                         int F, int4* queue, int* qcount) {
    const int tid = threadIdx.x, step = blockDim.x;
    hist = vote_copy(hist);
    int4 en = tid < count ? __ldg(ent + tid) : make_int4(0, 0, 0, 0);
    int4 en2 = tid + step < count ? __ldg(ent + tid + step) : make_int4(0, 0, 0, 0);
    for (int base = 0; base < count; base += step) {
        const int j = base + tid;
        const int4 e = en;
        en = en2;
        if (j + 2 * step < count) en2 = __ldg(ent + j + 2 * step);
        const int ox = unpack_off(e.x, 0), oy = unpack_off(e.x, 1), oz = unpack_off(e.x, 2);
        const int x = kp.ix + ox, y = kp.iy + oy, z = kp.iz + oz;
        if (j < count && (INTERIOR || (x >= 0 && y >= 0 && z >= 0 && x < L.nx && y < L.ny && z < L.nz))) {
            Nb6 cur = sphere_nb6(box, e);
            if (!INTERIOR) {
                cur.sx = (x > 0 && x < L.nx - 1) ? 0.5f : 1.0f;
                cur.sy = (y > 0 && y < L.ny - 1) ? 0.5f : 1.0f;
                cur.sz = (z > 0 && z < L.nz - 1) ? 0.5f : 1.0f;
            }
            float gx, gy, gz;
            grad32(cur, gx, gy, gz);
            if (grad_nonzero(cur)) {  // zero vote: no bin changes
                const float mag = nz_vote(norm3_f32(gx, gy, gz));
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    if (f >= F) break;
                    int sure;
                    const int bin = sr_bin_try(ox, oy, oz, gx, gy, gz, Rc + kRcPerFrame * f, sure);
                    if (sure == 3) {
                        red_vote(hist + f * kHistFrame, bin, mag);
                    } else {
                        const int pos = atomicAdd(qcount, 1);
                        queue[pos] = make_int4(e.x, f | (bin << 2) | (sure << 8), __float_as_int(mag), 0);
                    }
                }
            }
        }
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
    __syncwarp();
    const int qn = *reinterpret_cast<volatile int*>(qcount);
    if ((tid & 31) < qn) sr_resolve(queue[tid & 31], kp, L, data, Rs, hist);
    __syncwarp();
    if ((tid & 31) == 0) *qcount = 0;
    __syncwarp();
}

template <bool INTERIOR>
VK_D void sr_walk_sphere_frames(const vk_kp& kp, const vk_level& L, const float* data, const float* box,
                                const int4* ent, int count, const double* Rs, const float4* Rc, double* hist, int F,
                                int4* queue, int* qcount) {
    for (int f0 = 0; f0 < F; f0 += 4) {  // up to 4 frames per pass
        const int n = min(4, F - f0);
        const double* R = Rs + 9 * f0;
        const float4* C = Rc + kRcPerFrame * f0;
        double* h = hist + kHistFrame * f0;
        switch (n) {
            case 1: sr_walk_sphere<1, INTERIOR>(kp, L, data, box, ent, count, R, C, h, n, queue, qcount); break;
            case 2: sr_walk_sphere<2, INTERIOR>(kp, L, data, box, ent, count, R, C, h, n, queue, qcount); break;
            case 3: sr_walk_sphere<3, INTERIOR>(kp, L, data, box, ent, count, R, C, h, n, queue, qcount); break;
            default: sr_walk_sphere<4, INTERIOR>(kp, L, data, box, ent, count, R, C, h, n, queue, qcount); break;
        }
    }
}

// STAGE = false: the same fused per-keypoint pipeline without the shared
// sphere -- both walks gather from global memory (the separate kernels' walks),
// the SIFT-Rank walk right after the orientation walk on L1 / L2-warm data,
// at 3 CTAs/SM (the 58 KB CTA state only).
template <bool STAGE>
__global__ void __launch_bounds__(kOsThreads, STAGE ? 2 : 3)
orsr_kernel(const vk_kp* __restrict__ kps, const int* __restrict__ n_kp_dev, int n_kp_max,
            const vk_level* __restrict__ levels, const vk_ball* __restrict__ balls,
            const int* __restrict__ ball_offsets, const double* __restrict__ windows,
            const float* __restrict__ windows32, const double* __restrict__ dirs_g, int K,
            const uint8_t* __restrict__ pair_ok, double ratio, int max_frames, const double* __restrict__ rot_table,
            int* __restrict__ nframes, int* __restrict__ prim, int* __restrict__ sec, uint8_t* __restrict__ desc_kp,
            int* __restrict__ status, IcoT ico, const uint8_t* __restrict__ ico_lut, const int4* __restrict__ sph_ball,
            const int4* __restrict__ sph_rows, const int4* __restrict__ sph_ent, int box_cap,
            double* __restrict__ work) {
    // dynamic shared memory: the CTA state (58 KB, over the static limit), then
    // box_cap floats for the staged stencil sphere
    extern __shared__ __align__(16) unsigned char dsm[];
    OsShared& sh = *reinterpret_cast<OsShared*>(dsm);
    float* box = reinterpret_cast<float*>(dsm + kOsStateBytes);
    double* hist = work + (long long)blockIdx.x * kAccumSlot;  // [K] then [F][64] fp64, L2-resident
    const int tid = threadIdx.x, wid = tid >> 5;
    for (int i = tid; i < 3 * K; i += kOsThreads) sh.o.dirs[i] = dirs_g[i];
    if (tid < 72) {
        const int v = tid / 6, c = tid % 6;
        const int k = c == 0 ? ico.vert[v] : ico.adj[v][c - 1];
        sh.ic.ci[tid] = k;
        sh.ic.cd[tid] = make_float4((float)dirs_g[3 * k], (float)dirs_g[3 * k + 1], (float)dirs_g[3 * k + 2], 0.f);
        sh.ic.fk[tid] = c == 0 ? ico.vert[v] : ico.kind[v][c - 1];
    }
    load_ok_bits(sh.o.okb, pair_ok, K);
    for (int i = tid; i < kLutBytes / 4; i += kOsThreads)
        reinterpret_cast<uint32_t*>(sh.lut)[i] = __ldg(reinterpret_cast<const uint32_t*>(ico_lut) + i);
    if (tid < kOsThreads / 32) sh.sqn[tid] = 0;
    const int n_kp = n_kp_dev ? min(*n_kp_dev, n_kp_max) : n_kp_max;

    for (int item = blockIdx.x; item < n_kp; item += gridDim.x) {
        const vk_kp kp = kps[item];
        const vk_level L = levels[kp.lvl];
        const float* data = L.base + (long long)kp.vol * L.vol_stride;
        const vk_ball ball = balls[kp.ball];
        const int4 sb = sph_ball[kp.ball];  // rows start, n_rows, compact size, entries start
        const bool interior = ball_interior(kp.ix, kp.iy, kp.iz, ball.r, L.nx, L.ny, L.nz);
        __syncthreads();  // the previous item is done with box and the shared state
        if (STAGE) {
            if (interior)
                stage_sphere<false>(data, L.nx, L.ny, L.nz, kp, sph_rows + sb.x, sb.y, box);
            else
                stage_sphere<true>(data, L.nx, L.ny, L.nz, kp, sph_rows + sb.x, sb.y, box);
        }
        if (STAGE) {
            const int next = item + gridDim.x;
            if (next < n_kp) {
                const vk_kp nk = kps[next];
                const vk_level NL = levels[nk.lvl];
                const vk_ball nb = balls[nk.ball];
                const int4 ns = sph_ball[nk.ball];
                if (ball_interior(nk.ix, nk.iy, nk.iz, nb.r, NL.nx, NL.ny, NL.nz))
                    prefetch_sphere(NL.base + (long long)nk.vol * NL.vol_stride, (unsigned)NL.nx,
                                    (unsigned)NL.nx * (unsigned)NL.ny, nk, sph_rows + ns.x, ns.y);
            }
        }
        zero_hist(hist, K);
        if (tid == 0) {
            sh.o.n_inside = 0;
            sh.o.repair = 0;
        }
        if (STAGE) cp_async_wait<0>();
        __syncthreads();
        // ---- orientation walk (orient.py:89-125)
        const int4* ent = sph_ent + sb.w;
        int inside_cnt;
        if (STAGE)
            inside_cnt =
                interior ? ori_walk_sphere<true>(kp, L, data, box, ent, ball.count, windows32 + ball.window_start,
                                                 sh.o.dirs, &sh.ic, sh.lut, hist, sh.o.queue[wid])
                         : ori_walk_sphere<false>(kp, L, data, box, ent, ball.count, windows32 + ball.window_start,
                                                  sh.o.dirs, &sh.ic, sh.lut, hist, sh.o.queue[wid]);
        else
            inside_cnt = interior ? ori_walk_pipe<true>(kp, L, data, ball, ball_offsets, windows32 + ball.window_start,
                                                        sh.o.dirs, &sh.ic, sh.lut, hist, sh.o.queue[wid])
                                  : ori_walk<false>(kp, L, data, ball, ball_offsets, windows32 + ball.window_start,
                                                    sh.o.dirs, &sh.ic, sh.lut, K, hist, sh.o.queue[wid]);
        if (inside_cnt) atomicAdd(&sh.o.n_inside, inside_cnt);
        __syncthreads();
        const int n_inside = sh.o.n_inside;
        if (n_inside == 0) {
            // DataError: orientation neighbourhood entirely outside (orient.py:109-110)
            if (tid == 0) {
                atomicOr(status, 1);
                nframes[item] = 0;
            }
            continue;  // (the loop head synchronises)
        }
        // ---- certified frames (orient.py:128-168)
        for (int b = tid; b < K; b += kOsThreads) sh.o.w[b] = read_hist(hist, b);
        __syncthreads();
        sort_desc(sh.o.w, K, sh.o.order);
        for (int b = tid; b < K; b += kOsThreads) sh.o.unc[b] = 0;
        __syncthreads();
        if (tid < 32) {
            const double epsrel = 2.0 * (kVoteRel + gamma_k((double)n_inside + 64.0));
            const double epsabs = kVoteAbs * n_inside;
            if (warp_mark_uncertain(sh.o.w, sh.o.order, K, epsrel, epsabs, ratio, max_frames, sh.o.unc) && tid == 0) {
                sh.o.repair = 1;
                atomicAdd(status + 1, 1);  // orientation fallback counter (diagnostics)
            }
        }
        __syncthreads();
        if (sh.o.repair) {
            ori_exact_subset(data, L, kp, ball, ball_offsets, windows + ball.window_start, sh.o.dirs, &sh.ic, sh.lut, K,
                             sh.o);
            sort_desc(sh.o.w, K, sh.o.order);
            __syncthreads();
        }
        if (tid < 32)
            warp_frames_from(sh.o.w, sh.o.order, K, sh.o.okb, ratio, max_frames, &sh.nf, sh.prim, sh.sec);
        __syncthreads();
        const int F = sh.nf;
        if (tid < max_frames) {
            prim[(long long)item * max_frames + tid] = tid < F ? sh.prim[tid] : 0;
            sec[(long long)item * max_frames + tid] = tid < F ? sh.sec[tid] : 0;
        }
        if (tid == 0) nframes[item] = F;
        if (F == 0) continue;
        // ---- the frames' rotations (orient.py:160-167 via the host frame table)
        for (int i = tid; i < F * 9; i += kOsThreads) {
            const int f = i / 9, e = i - 9 * f;
            sh.Rs[i] = __ldg(rot_table + ((long long)sh.prim[f] * K + sh.sec[f]) * 9 + e);
        }
        __syncthreads();
        for (int i = tid; i < F * 3; i += kOsThreads) {
            const double* R = sh.Rs + 9 * (i / 3);
            const int j = i % 3;
            const float cx = (float)R[j], cy = (float)R[3 + j], cz = (float)R[6 + j];
            const int zmask = (R[j] == 0.0) | ((R[3 + j] == 0.0) << 1) | ((R[6 + j] == 0.0) << 2);
            sh.Rc[(i / 3) * kRcPerFrame + 2 * j] = make_float4(cx, cx, cy, cy);
            sh.Rc[(i / 3) * kRcPerFrame + 2 * j + 1] = make_float4(cz, cz, __int_as_float(zmask), 0.f);
        }
        zero_hist(hist, F * kSrBins);
        __syncthreads();
        // ---- SIFT-Rank walk (descriptor.py:227-263) on the same stencils
        if (!STAGE) {
            if (interior)
                sr_walk_frames<true>(kp, L, data, nullptr, ball, ball_offsets, sh.Rs, sh.Rc, hist, F, sh.sq[wid],
                                     sh.sqn + wid);
            else
                sr_walk_frames<false>(kp, L, data, nullptr, ball, ball_offsets, sh.Rs, sh.Rc, hist, F, sh.sq[wid],
                                      sh.sqn + wid);
        } else if (interior) {
            sr_walk_sphere_frames<true>(kp, L, data, box, ent, ball.count, sh.Rs, sh.Rc, hist, F, sh.sq[wid],
                                        sh.sqn + wid);
        } else {
            sr_walk_sphere_frames<false>(kp, L, data, box, ent, ball.count, sh.Rs, sh.Rc, hist, F, sh.sq[wid],
                                         sh.sqn + wid);
        }
        __syncthreads();
        // ---- certified stable ranks, all frames of the keypoint (siftrank_kernel)
        const double epsrel = 2.0 * (kVoteRel + gamma_k((double)n_inside + 64.0));
        const double epsabs = kVoteAbs * n_inside;
        const int fl = tid >> 6, b = tid & (kSrBins - 1);
        for (int f0 = 0; f0 < F; f0 += kOsThreads / kSrBins) {
            const int f = f0 + fl;
            const bool mine = f < F;
            if (mine) sh.w4[fl][b] = read_hist(hist, f * kSrBins + b);
            if (tid < kOsThreads / kSrBins) sh.badf[tid] = 0;
            __syncthreads();
            int myrank = 0;
            if (mine) {
                myrank = stable_rank(sh.w4[fl], kSrBins, b);
                sh.order4[fl][myrank] = b;
            }
            __syncthreads();
            int bad = 0;
            if (mine && b + 1 < kSrBins) {
                const double x = sh.w4[fl][sh.order4[fl][b]], y = sh.w4[fl][sh.order4[fl][b + 1]];
                if (!(x == 0.0 && y == 0.0)) {  // exact empty-bin ties are order-independent
                    const double xhi = x == 0.0 ? 0.0 : dadd(x, x * epsrel + epsabs);
                    const double ylo = dsub(y, y * epsrel + epsabs);
                    bad = !(xhi < ylo);
                }
            }
            if (bad) sh.badf[fl] = 1;
            if (__syncthreads_or(bad)) {
                for (int g = 0; g < kOsThreads / kSrBins && f0 + g < F; ++g) {
                    if (!sh.badf[g]) continue;
                    if (tid == 0) atomicAdd(status + 2, 1);  // SIFT-Rank fallback counter (diagnostics)
                    if (tid < kSrBins) {
                        sh.unc[tid] = 0;
                        sh.w[tid] = sh.w4[g][tid];
                    }
                    __syncthreads();
                    if (fl == g && bad) sh.unc[sh.order4[g][b]] = sh.unc[sh.order4[g][b + 1]] = 1;
                    __syncthreads();
                    sr_exact_subset(data, L, kp, ball, ball_offsets, sh.Rs + 9 * (f0 + g),
                                    sh.Rc + kRcPerFrame * (f0 + g), sh.unc, sh.w, sh.o.xb, sh.o.xv, sh.o.wmask);
                    if (fl == g) myrank = stable_rank(sh.w, kSrBins, b);
                    __syncthreads();
                }
            }
            if (mine) desc_kp[((long long)item * max_frames + f) * kSrBins + b] = (uint8_t)myrank;
            __syncthreads();
        }
    }
}

// desc[o] = desc_kp[kp(o) * max_frames + (o - first[kp(o)])] for every frame o
// vk_expand_frames wrote (frame order = keypoint order, frames in weight order).
__global__ void scatter_rows_kernel(const vk_frame* __restrict__ frames, const int* __restrict__ first,
                                    const int* __restrict__ n_frames_dev, int frame_cap, int max_frames,
                                    const uint4* __restrict__ src, uint4* __restrict__ dst) {
    const int n = min(*n_frames_dev, frame_cap);
    const long long total = (long long)n * 4;  // 64 bytes = 4 x uint4 per row
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int o = (int)(t >> 2), q = (int)(t & 3);
        const int kp = frames[o].kp;
        const long long s = (long long)kp * max_frames + (o - first[kp]);
        dst[(long long)o * 4 + q] = src[s * 4 + q];
    }
}

}  // namespace vk

using namespace vk;

extern "C" int vk_orient_siftrank(const vk_kp* kps, const int* n_kp_dev, int n_kp_max, const vk_level* levels,
                                  const vk_ball* balls, const int* ball_offsets, const double* windows,
                                  const float* windows32, const double* dirs, int K, const uint8_t* pair_ok,
                                  double secondary_ratio, int max_frames, const double* rot_table, int* nframes,
                                  int* prim, int* sec, uint8_t* desc_kp, int* status, const int* ico_host,
                                  const uint8_t* ico_lut, const int* sph_ball, const int* sph_rows,
                                  const int* sph_ent, int box_cap, double* work, void* stream) {
    if (!kps || n_kp_max < 0 || !levels || !balls || !ball_offsets || !windows || !windows32 || !dirs || K != 42 ||
        !pair_ok || !rot_table || !nframes || !prim || !sec || !desc_kp || !status || !ico_host || !ico_lut ||
        !sph_ball || !sph_rows || !sph_ent || box_cap < 0 || box_cap > 40000 || !work || max_frames < 1 ||
        max_frames > VK_MAX_FRAMES || !(secondary_ratio > 0.0 && secondary_ratio <= 1.0)) {
        set_error("vk_orient_siftrank: bad arguments (K=%d max_frames=%d box_cap=%d)", K, max_frames, box_cap);
        return VK_ERR_PARAMETER;
    }
    if (n_kp_max == 0) return VK_OK;
    const size_t dyn = kOsStateBytes + (size_t)box_cap * sizeof(float);
    static size_t configured[2] = {0, 0};
    const int stage = box_cap > 0;
    if (dyn > configured[stage]) {
        cudaError_t e = cudaFuncSetAttribute(stage ? orsr_kernel<true> : orsr_kernel<false>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        if (e != cudaSuccess) return cuda_status(e, "orsr smem attribute");
        configured[stage] = dyn;
    }
    IcoT ico{};
    ico.valid = 1;
    for (int v = 0; v < 12; ++v) {
        ico.vert[v] = ico_host[v];
        for (int m = 0; m < 5; ++m) ico.adj[v][m] = ico_host[12 + 5 * v + m];
        for (int m = 0; m < 5; ++m) ico.kind[v][m] = ico_host[72 + 5 * v + m];
    }
    auto* kern = stage ? orsr_kernel<true> : orsr_kernel<false>;
    const int grid = accum_grid(kern, kOsThreads, n_kp_max, dyn);
    kern<<<grid, kOsThreads, dyn, as_stream(stream)>>>(
        kps, n_kp_dev, n_kp_max, levels, balls, ball_offsets, windows, windows32, dirs, K, pair_ok, secondary_ratio,
        max_frames, rot_table, nframes, prim, sec, desc_kp, status, ico, ico_lut,
        reinterpret_cast<const int4*>(sph_ball), reinterpret_cast<const int4*>(sph_rows),
        reinterpret_cast<const int4*>(sph_ent), box_cap, work);
    count_launch();
    return cuda_status(cudaGetLastError(), "orsr launch");
}

extern "C" int vk_scatter_frame_rows(const vk_frame* frames, const int* frame_first, const int* n_frames_dev,
                                     int frame_cap, int max_frames, const uint8_t* rows_kp, uint8_t* rows,
                                     void* stream) {
    if (!frames || !frame_first || !n_frames_dev || frame_cap < 0 || max_frames < 1 || !rows_kp || !rows) {
        set_error("vk_scatter_frame_rows: bad arguments");
        return VK_ERR_PARAMETER;
    }
    if (frame_cap == 0) return VK_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    scatter_rows_kernel<<<2 * sms, 256, 0, as_stream(stream)>>>(frames, frame_first, n_frames_dev, frame_cap,
                                                                 max_frames, reinterpret_cast<const uint4*>(rows_kp),
                                                                 reinterpret_cast<uint4*>(rows));
    count_launch();
    return cuda_status(cudaGetLastError(), "scatter launch");
}
