// vk_detect.cu -- 80-neighbour scale-space extrema and ordered keypoint output.
//
// Reference: detect.py:48-79 (sum_of_signs_map), detect.py:82-140
// (extract_extrema), detect.py:149-182 (detect_keypoints ordering).
//
// Detection never materialises the int16 map on the pipeline path: a voxel is
// a peak iff its "peak deficit" dp = 80 - m is <= band (and m > 0), a valley
// iff dv = 80 + m <= band (and m < 0).  Both deficits only grow, so a thread
// stops at the first neighbour that pushes both past the band -- for band 0
// that is after ~3 of the 80 comparisons on average.  Survivors are appended
// as 64-bit keys (segment, z, y, x, valley) whose numeric order is exactly the
// reference order (octave, level, z, y, x, peak-before-valley); a rank-by-count
// kernel then scatters them into the final keypoint records.
#include "vk_common.cuh"

namespace vk {

constexpr int kMaxDog = 32;
constexpr int kMaxSeg = 128;

struct DogPtrs {
    const float* p[kMaxDog];
};

struct SegInfo {
    int octave[kMaxSeg];
    int level[kMaxSeg];
    int lvl[kMaxSeg];
    int ball[kMaxSeg];
    double sigma[kMaxSeg];
};

VK_D unsigned long long make_key(int seg, int x, int y, int z, int valley) {
    return ((unsigned long long)seg << 52) | ((unsigned long long)z << 35) | ((unsigned long long)y << 18) |
           ((unsigned long long)x << 1) | (unsigned long long)valley;
}

__global__ void __launch_bounds__(128)
detect_kernel(DogPtrs dogs, int nlev, int nx, int ny, int nz, int seg_base, int band, float cmin,
              unsigned long long* __restrict__ keys, int* __restrict__ counts, int cap) {
    const int x = 1 + blockIdx.x * 32 + threadIdx.x;
    const int y = 1 + blockIdx.y * 4 + threadIdx.y;
    const int iz = nz - 2;
    const int z = 1 + blockIdx.z % iz;
    const int rest = blockIdx.z / iz;
    const int lev = 1 + rest % nlev;
    const int b = rest / nlev;
    const long long plane = (long long)nx * ny;
    const long long vol = plane * nz;
    const long long idx = (long long)b * vol + (long long)z * plane + (long long)y * nx + x;

    bool peak = false, valley = false;
    if (x < nx - 1 && y < ny - 1) {
        const float c = __ldg(dogs.p[lev] + idx);
        if (fabsf(c) >= cmin) {
            int dp = 0, dv = 0;
            bool dead = false;
#pragma unroll 1
            for (int dl = 0; dl < 3 && !dead; ++dl) {
                // centre level first: most voxels die on an in-plane neighbour
                const int L = dl == 0 ? lev : (dl == 1 ? lev - 1 : lev + 1);
                const float* v = dogs.p[L] + idx;
#pragma unroll
                for (int o = 0; o < 27; ++o) {
                    const int dz = o / 9 - 1, dy = (o / 3) % 3 - 1, dx = o % 3 - 1;
                    if (dl == 0 && o == 13) continue;
                    const float n = __ldg(v + (long long)dz * plane + (long long)dy * nx + dx);
                    dp += (c > n) ? 0 : (c == n ? 1 : 2);
                    dv += (c < n) ? 0 : (c == n ? 1 : 2);
                    if (dp > band && dv > band) { dead = true; break; }
                }
            }
            if (!dead) {
                peak = dp <= band && dp < 80;
                valley = dv <= band && dv < 80;
            }
        }
    }
    const bool hit = peak || valley;
    // warp-aggregated append
    const unsigned mask = __ballot_sync(0xffffffffu, hit);
    if (mask == 0) return;
    const int lane = (threadIdx.y * 32 + threadIdx.x) & 31;
    const int leader = __ffs(mask) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(counts + b, __popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (hit) {
        const int slot = base + __popc(mask & ((1u << lane) - 1));
        if (slot < cap) keys[(long long)b * cap + slot] = make_key(seg_base + lev, x, y, z, valley ? 1 : 0);
    }
}

// Band 0 (the default): a strict extremum must first beat its 26 same-level
// neighbours (prefilter on in-plane 3x3 max / min of the previous, current and
// next plane, streamed in registers); survivors (a few per cent) are confirmed
// against the 54 neighbours in the adjacent DoG levels with exactly the
// reference comparisons (detect.py:65-76); NaN neighbours never let a
// non-extremum through the confirmation because it uses > / < like numpy.
// Band 0, register-blocked: a warp covers 30 output columns (lanes 1..30;
// lanes 0 and 31 only load the x halo) and each thread 4 consecutive output
// rows, streaming z.  Per plane a thread loads 6 rows of its column (coalesced,
// one plane ahead), the x neighbours come from the adjacent lanes (shuffles),
// so the 3x3 in-plane max / min costs ~1.6 loads per voxel instead of 9.
// Same prefilter + exact 54-neighbour confirmation as detect_band0_kernel.
// Three-input float max / min (FMNMX3 on sm_100a): exact, NaN operands ignored
// like fmaxf / fminf chains.
VK_D float max3f(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
VK_D float min3f(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

#ifndef VK_DET_ROWS
#define VK_DET_ROWS 4  // output rows per thread (2 -> 4: detection -6% on B200)
#endif
constexpr int kDetRows = VK_DET_ROWS;  // output rows per thread
__global__ void __launch_bounds__(128)
detect_band0_rb_kernel(DogPtrs dogs, int nlev, int nx, int ny, int nz, int seg_base, float cmin,
                       unsigned long long* __restrict__ keys, int* __restrict__ counts, int cap, int tz, int nzc) {
    const int lane = threadIdx.x, wy = threadIdx.y;
    const int x = blockIdx.x * 30 + lane;                       // this lane's column (output if lane 1..30)
    const int y0 = 1 + blockIdx.y * (4 * kDetRows) + kDetRows * wy;  // first output row
    const int zc = blockIdx.z % nzc;
    const int lev = 1 + (blockIdx.z / nzc) % nlev;
    const int b = blockIdx.z / (nzc * nlev);
    const int z_lo = 1 + zc * tz, z_hi = min(nz - 2, z_lo + tz - 1);  // output planes of this chunk
    const long long plane = (long long)nx * ny;
    const long long vol = plane * nz;
    const int xc = min(x, nx - 1);
    const float* base = dogs.p[lev] + (long long)b * vol + xc;
    unsigned roff[kDetRows + 2];
#pragma unroll
    for (int i = 0; i < kDetRows + 2; ++i) roff[i] = (unsigned)min(y0 - 1 + i, ny - 1) * (unsigned)nx;
    const bool xout = lane >= 1 && lane <= 30 && x <= nx - 2;
    int* cnt = counts + b;
    unsigned long long* kb = keys + (long long)b * cap;
    // this lane's two adjacent-level neighbours (o = lane, lane + 32 of the 54,
    // level-major then z, y, x like detect.py:65-76) as pointer offsets
    auto nb_ptr = [&](int o) {
        const int r = o % 27;
        return dogs.p[o < 27 ? lev - 1 : lev + 1] + (long long)b * vol + (long long)(r / 9 - 1) * plane +
               (long long)((r / 3) % 3 - 1) * nx + (r % 3 - 1);
    };
    const float* nb1 = nb_ptr(lane);
    const bool has2 = lane + 32 < 54;
    const float* nb2 = nb_ptr(has2 ? lane + 32 : lane);

    // per-plane stats for the kDetRows outputs: M9/m9 (3x3 incl. centre), M8/m8 (8-neighbourhood), c
    auto stats = [&](const float (&r)[kDetRows + 2], float (&M9)[kDetRows], float (&m9)[kDetRows],
                     float (&M8)[kDetRows], float (&m8)[kDetRows], float (&c)[kDetRows]) {
        float hM[kDetRows + 2], hm[kDetRows + 2], L[kDetRows + 2], Rr[kDetRows + 2];
#pragma unroll
        for (int i = 0; i < kDetRows + 2; ++i) {
            L[i] = __shfl_up_sync(0xffffffffu, r[i], 1);
            Rr[i] = __shfl_down_sync(0xffffffffu, r[i], 1);
            hM[i] = max3f(L[i], r[i], Rr[i]);
            hm[i] = min3f(L[i], r[i], Rr[i]);
        }
#pragma unroll
        for (int k = 0; k < kDetRows; ++k) {
            const float a = fmaxf(hM[k], hM[k + 2]), am = fminf(hm[k], hm[k + 2]);
            M8[k] = max3f(a, L[k + 1], Rr[k + 1]);
            m8[k] = min3f(am, L[k + 1], Rr[k + 1]);
            M9[k] = fmaxf(a, hM[k + 1]);
            m9[k] = fminf(am, hm[k + 1]);
            c[k] = r[k + 1];
        }
    };
    auto load = [&](float (&r)[kDetRows + 2], int z) {
        const float* p = base + (long long)z * plane;
#pragma unroll
        for (int i = 0; i < kDetRows + 2; ++i) r[i] = __ldg(p + roff[i]);
    };

    float rp[kDetRows + 2], rc[kDetRows + 2], rn[kDetRows + 2];
    float Mp[kDetRows], mp[kDetRows], Mc[kDetRows], mc[kDetRows], cc[kDetRows];
    if (z_lo > z_hi) return;
    {
        float t8[kDetRows], u8[kDetRows], tc[kDetRows];
        load(rp, z_lo - 1);
        stats(rp, Mp, mp, t8, u8, tc);
        load(rc, z_lo);
        float d9[kDetRows], e9[kDetRows];
        stats(rc, d9, e9, Mc, mc, cc);
        load(rn, z_lo + 1);
    }
    for (int z = z_lo; z <= z_hi; ++z) {
        float Mn9[kDetRows], mn9[kDetRows], Mn8[kDetRows], mn8[kDetRows], cn[kDetRows];
        stats(rn, Mn9, mn9, Mn8, mn8, cn);
        if (z + 2 <= z_hi + 1) load(rn, z + 2);
#pragma unroll
        for (int k = 0; k < kDetRows; ++k) {
            const int y = y0 + k;  // warp-uniform
            bool pk = false, vl = false;
            if (xout && y <= ny - 2 && fabsf(cc[k]) >= cmin) {
                pk = cc[k] > max3f(Mp[k], Mc[k], Mn9[k]);
                vl = cc[k] < min3f(mp[k], mc[k], mn9[k]);
            }
            // Confirm every surviving candidate against its 54 neighbours in the
            // adjacent DoG levels with the whole warp (lane l checks neighbours l
            // and l + 32): no divergent per-lane loops.
            bool hit = false;
            const long long cpos = (long long)z * plane + (long long)y * nx;
            for (unsigned cm = __ballot_sync(0xffffffffu, pk || vl); cm; cm &= cm - 1) {
                const int src = __ffs(cm) - 1;
                const float cv = __shfl_sync(0xffffffffu, cc[k], src);
                const bool cpk = __shfl_sync(0xffffffffu, pk, src);
                const long long at = cpos + (blockIdx.x * 30 + src);
                const float n1 = __ldg(nb1 + at);
                bool ok = cpk ? (cv > n1) : (cv < n1);
                if (has2) {
                    const float n2 = __ldg(nb2 + at);
                    ok = ok && (cpk ? (cv > n2) : (cv < n2));
                }
                const bool all = __all_sync(0xffffffffu, ok);
                if (lane == src) hit = all;
            }
            const bool valley = vl;
            const unsigned mask = __ballot_sync(0xffffffffu, hit);
            if (mask) {
                const int leader = __ffs(mask) - 1;
                int bs = 0;
                if (lane == leader) bs = atomicAdd(cnt, __popc(mask));
                bs = __shfl_sync(0xffffffffu, bs, leader);
                if (hit) {
                    const int slot = bs + __popc(mask & ((1u << lane) - 1));
                    if (slot < cap) kb[slot] = make_key(seg_base + lev, x, y, z, valley ? 1 : 0);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < kDetRows; ++k) {
            Mp[k] = fmaxf(Mc[k], cc[k]);
            mp[k] = fminf(mc[k], cc[k]);
            Mc[k] = Mn8[k];
            mc[k] = mn8[k];
            cc[k] = cn[k];
        }
    }
}

__global__ void sum_of_signs_kernel(const float* __restrict__ prev, const float* __restrict__ cur,
                                    const float* __restrict__ next, int16_t* __restrict__ out, int nx, int ny, int nz,
                                    long long total) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const long long plane = (long long)nx * ny, vol = plane * nz;
    long long rem = i % vol;
    int z = (int)(rem / plane);
    int y = (int)((rem - (long long)z * plane) / nx);
    int x = (int)(rem - (long long)z * plane - (long long)y * nx);
    if (x < 1 || y < 1 || z < 1 || x >= nx - 1 || y >= ny - 1 || z >= nz - 1) {
        out[i] = 0;
        return;
    }
    const float c = cur[i];
    int m = 0;
    const float* vols[3] = {prev, cur, next};
#pragma unroll
    for (int l = 0; l < 3; ++l) {
#pragma unroll
        for (int o = 0; o < 27; ++o) {
            if (l == 1 && o == 13) continue;
            const float n = __ldg(vols[l] + i + (long long)(o / 9 - 1) * plane + (long long)((o / 3) % 3 - 1) * nx + (o % 3 - 1));
            m += (c > n) - (c < n);
        }
    }
    out[i] = (int16_t)m;
}

// Candidates from a precomputed sum-of-signs map (extract_extrema, detect.py:82-140).
__global__ void extrema_from_map_kernel(const int16_t* __restrict__ map, const float* __restrict__ dogc, int nx, int ny,
                                        int nz, int seg, int band, float cmin, unsigned long long* __restrict__ keys,
                                        int* __restrict__ counts, int cap) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long plane = (long long)nx * ny, vol = plane * nz;
    bool hit = false, valley = false;
    int x = 0, y = 0, z = 0;
    if (i < vol) {
        z = (int)(i / plane);
        y = (int)((i - (long long)z * plane) / nx);
        x = (int)(i - (long long)z * plane - (long long)y * nx);
        if (x >= 1 && y >= 1 && z >= 1 && x < nx - 1 && y < ny - 1 && z < nz - 1 && fabsf(dogc[i]) >= cmin) {
            const int m = map[i];
            const bool pk = m >= 80 - band && m > 0;
            valley = m <= -80 + band && m < 0;
            hit = pk || valley;
        }
    }
    const unsigned mask = __ballot_sync(0xffffffffu, hit);
    if (mask == 0) return;
    const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(counts, __popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (hit) {
        const int slot = base + __popc(mask & ((1u << lane) - 1));
        if (slot < cap) keys[slot] = make_key(seg, x, y, z, valley ? 1 : 0);
    }
}

// Exclusive prefix of min(count, cap) over the batch; total[0] = keypoints,
// total[1] = 1 if any volume overflowed its candidate capacity.  One warp,
// 32 volumes per shuffle scan.
__global__ void batch_offsets_kernel(const int* __restrict__ counts, int nb, int cap, int* __restrict__ vol_offset,
                                     int* __restrict__ total) {
    const int lane = threadIdx.x;
    if (lane >= 32) return;
    int carry = 0;
    bool over = false;
    for (int b0 = 0; b0 < nb; b0 += 32) {
        const int b = b0 + lane;
        int c = b < nb ? counts[b] : 0;
        over = over || c > cap;
        c = min(c, cap);
        int v = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
        }
        if (b < nb) vol_offset[b] = carry + v - c;
        carry += __shfl_sync(0xffffffffu, v, 31);
    }
    const bool any_over = __any_sync(0xffffffffu, over);
    if (lane == 0) {
        total[0] = carry;
        total[1] = any_over ? 1 : 0;
    }
}

// Keypoint order (detect.py:149-182: octave, level, z, y, x, peak before
// valley) = numeric order of the 64-bit candidate keys.  Each run of
// kSortChunk keys of a volume is bitonic-sorted in shared memory (in place),
// then every key finds its global rank by binary searches over the runs:
// O(n log n) per volume in total work, with n / kSortChunk searches per key.
constexpr int kSortChunk = 2048;

__global__ void __launch_bounds__(1024) chunk_sort_kernel(unsigned long long* __restrict__ keys,
                                                          const int* __restrict__ counts, int cap) {
    __shared__ unsigned long long s[kSortChunk];
    const int b = blockIdx.y, c0 = blockIdx.x * kSortChunk;
    const int n = min(counts[b], cap);
    if (c0 >= n) return;
    unsigned long long* kb = keys + (long long)b * cap + c0;
    const int m = min(kSortChunk, n - c0);
    for (int i = threadIdx.x; i < kSortChunk; i += blockDim.x) s[i] = i < m ? kb[i] : ~0ull;
    __syncthreads();
    for (int k = 2; k <= kSortChunk; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < kSortChunk; i += blockDim.x) {
                const int p = i ^ j;
                if (p > i) {
                    const unsigned long long a = s[i], c = s[p];
                    if ((a > c) == ((i & k) == 0)) {
                        s[i] = c;
                        s[p] = a;
                    }
                }
            }
            __syncthreads();
        }
    for (int i = threadIdx.x; i < m; i += blockDim.x) kb[i] = s[i];
}

__global__ void __launch_bounds__(256)
order_kernel(const unsigned long long* __restrict__ keys, const int* __restrict__ counts, int cap,
             const int* __restrict__ vol_offset, SegInfo seg, const vk_level* __restrict__ dog_levels,
             vk_kp* __restrict__ kps, double* __restrict__ pos, double* __restrict__ sigma, float* __restrict__ dogv,
             int8_t* __restrict__ sign, int kp_cap) {
    const int b = blockIdx.y;
    const int n = min(counts[b], cap);
    const int i = blockIdx.x * 256 + threadIdx.x;
    const unsigned long long* kb = keys + (long long)b * cap;
    if (i >= n) return;
    const unsigned long long key = kb[i];
    // keys are unique; each kSortChunk-run of kb is sorted (chunk_sort_kernel):
    // the rank is the sum of the lower bounds of the key in every run
    int rank = 0;
    for (int c0 = 0; c0 < n; c0 += kSortChunk) {
        int lo = 0, hi = min(kSortChunk, n - c0);
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (kb[c0 + mid] < key) lo = mid + 1;
            else hi = mid;
        }
        rank += lo;
    }
    const int out = vol_offset[b] + rank;
    if (out >= kp_cap) return;
    const int s = (int)(key >> 52);
    const int z = (int)((key >> 35) & 0x1FFFF), y = (int)((key >> 18) & 0x1FFFF), x = (int)((key >> 1) & 0x1FFFF);
    const int octave = seg.octave[s];
    vk_kp k;
    k.vol = b;
    k.lvl = seg.lvl[s];
    k.ix = x;
    k.iy = y;
    k.iz = z;
    k.ball = seg.ball[s];
    k.octave = octave;
    k.level = seg.level[s];
    kps[out] = k;
    // position = i * 2^o + (2^o - 1) / 2 in fp64 (detect.py:105-131)
    const double scale = ldexp(1.0, octave);
    const double off = (scale - 1.0) / 2.0;
    pos[3 * out + 0] = dadd(dmul((double)x, scale), off);
    pos[3 * out + 1] = dadd(dmul((double)y, scale), off);
    pos[3 * out + 2] = dadd(dmul((double)z, scale), off);
    sigma[out] = seg.sigma[s];
    const vk_level L = dog_levels[s];
    dogv[out] = L.base[b * L.vol_stride + ((long long)z * L.ny + y) * L.nx + x];
    sign[out] = (key & 1ull) ? -1 : 1;
}

// Optional sub-voxel / sub-level refinement of the keypoints (not a reference
// stage: volkey reports lattice positions; north_star asks for
// the refinement as an extra output).  One Newton step of the quadratic
// (Taylor) model of the DoG around the extremum, in (x, y, z, level) of its
// octave: gradient and Hessian by central differences over the 3x3x3x3
// neighbourhood (DoG levels l-1, l, l+1), H d = -g solved by Gaussian
// elimination with partial pivoting in fp64, every operation separately
// rounded in a fixed order (the oracle restates it operation for operation).
// Output per keypoint (6 doubles): refined position in input-volume
// coordinates, refined sigma (kp sigma x kappa^d_level), refined DoG value
// D + g.d / 2, and a status: 0 = converged (|d_i| <= 0.5 on every axis),
// 1 = offset above 0.5 (the extremum lies nearer another sample), 2 =
// singular Hessian (offset 0).  The parity fields (kps, pos, sigma, dog) are
// untouched.
__global__ void refine_kernel(const vk_kp* __restrict__ kps, const int* __restrict__ n_dev, int n_max,
                              const vk_level* __restrict__ dog_levels, int levels_per_octave, double kappa,
                              const double* __restrict__ sigma, double* __restrict__ out) {
    const int n = min(*n_dev, n_max);
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const vk_kp kp = kps[k];
        const int D0 = kp.octave * (levels_per_octave) + kp.level;  // DoG level table index of (octave, level)
        const vk_level Lm = dog_levels[D0 - 1], Lc = dog_levels[D0], Lp = dog_levels[D0 + 1];
        const int nx = Lc.nx, ny = Lc.ny, nz = Lc.nz;
        auto at = [&](const vk_level& L, int dx, int dy, int dz) -> double {
            const int x = clampi(kp.ix + dx, 0, nx - 1), y = clampi(kp.iy + dy, 0, ny - 1),
                      z = clampi(kp.iz + dz, 0, nz - 1);
            return (double)L.base[(long long)kp.vol * L.vol_stride + ((long long)z * ny + y) * nx + x];
        };
        // samples along axis a (0..3 = x, y, z, level) at offsets -1, 0, +1 (others 0)
        auto s1 = [&](int a, int o) -> double {
            if (a == 3) return at(o < 0 ? Lm : (o > 0 ? Lp : Lc), 0, 0, 0);
            return at(Lc, a == 0 ? o : 0, a == 1 ? o : 0, a == 2 ? o : 0);
        };
        auto s2 = [&](int a, int oa, int b, int ob) -> double {  // a < b
            const vk_level& L = b == 3 ? (ob < 0 ? Lm : Lp) : Lc;
            int d[3] = {0, 0, 0};
            d[a] = oa;
            if (b < 3) d[b] = ob;
            return at(L, d[0], d[1], d[2]);
        };
        const double c = s1(0, 0);
        double g[4], H[4][4];
        for (int a = 0; a < 4; ++a) {
            const double p = s1(a, 1), m = s1(a, -1);
            g[a] = dmul(dsub(p, m), 0.5);
            H[a][a] = dsub(dadd(p, m), dmul(2.0, c));
        }
        for (int a = 0; a < 4; ++a)
            for (int b = a + 1; b < 4; ++b) {
                const double v = dsub(dsub(s2(a, 1, b, 1), s2(a, 1, b, -1)), dsub(s2(a, -1, b, 1), s2(a, -1, b, -1)));
                H[a][b] = H[b][a] = dmul(v, 0.25);
            }
        // Gaussian elimination with partial pivoting on [H | -g]
        double A[4][5];
        for (int i = 0; i < 4; ++i) {
            for (int j = 0; j < 4; ++j) A[i][j] = H[i][j];
            A[i][4] = -g[i];
        }
        int status = 0;
        for (int col = 0; col < 4 && status == 0; ++col) {
            int piv = col;
            for (int r = col + 1; r < 4; ++r)
                if (fabs(A[r][col]) > fabs(A[piv][col])) piv = r;
            if (!(fabs(A[piv][col]) > 0.0)) {
                status = 2;
                break;
            }
            if (piv != col)
                for (int j = 0; j < 5; ++j) {
                    const double t = A[col][j];
                    A[col][j] = A[piv][j];
                    A[piv][j] = t;
                }
            for (int r = col + 1; r < 4; ++r) {
                const double f = __ddiv_rn(A[r][col], A[col][col]);
                for (int j = col; j < 5; ++j) A[r][j] = dsub(A[r][j], dmul(f, A[col][j]));
            }
        }
        double d[4] = {0.0, 0.0, 0.0, 0.0};
        if (status == 0) {
            for (int i = 3; i >= 0; --i) {
                double acc = A[i][4];
                for (int j = i + 1; j < 4; ++j) acc = dsub(acc, dmul(A[i][j], d[j]));
                d[i] = __ddiv_rn(acc, A[i][i]);
            }
            for (int i = 0; i < 4; ++i)
                if (fabs(d[i]) > 0.5) status = 1;
        }
        const double scale = ldexp(1.0, kp.octave);
        const double off = (scale - 1.0) / 2.0;
        double* o = out + 6LL * k;
        o[0] = dadd(dmul(dadd((double)kp.ix, d[0]), scale), off);
        o[1] = dadd(dmul(dadd((double)kp.iy, d[1]), scale), off);
        o[2] = dadd(dmul(dadd((double)kp.iz, d[2]), scale), off);
        o[3] = dmul(sigma[k], pow(kappa, d[3]));
        double gd = 0.0;
        for (int i = 0; i < 4; ++i) gd = dadd(gd, dmul(g[i], d[i]));
        o[4] = dadd(c, dmul(0.5, gd));
        o[5] = (double)status;
    }
}

}  // namespace vk

using namespace vk;

extern "C" int vk_sum_of_signs(const float* prev, const float* cur, const float* next, int16_t* out, int nb, int nx,
                               int ny, int nz, void* stream) {
    if (!prev || !cur || !next || !out || nb < 0 || nx < 1 || ny < 1 || nz < 1) {
        set_error("vk_sum_of_signs: bad arguments");
        return VK_ERR_PARAMETER;
    }
    long long total = (long long)nb * nx * ny * nz;
    if (total == 0) return VK_OK;
    sum_of_signs_kernel<<<(unsigned)((total + 255) / 256), 256, 0, as_stream(stream)>>>(prev, cur, next, out, nx, ny,
                                                                                        nz, total);
    count_launch();
    return cuda_status(cudaGetLastError(), "sum_of_signs launch");
}

extern "C" int vk_detect_octave(const float* const* dogs_host, int ndog, int nb, int nx, int ny, int nz, int seg_base,
                                int band, float contrast_min, unsigned long long* cand_keys, int* cand_count, int cap,
                                void* stream) {
    if (!dogs_host || ndog < 3 || ndog > kMaxDog || nb < 0 || !cand_keys || !cand_count || cap < 0 || band < 0 ||
        band > 80 || seg_base < 0 || seg_base + ndog > 4095 || nx > 131071 || ny > 131071 || nz > 131071) {
        set_error("vk_detect_octave: bad arguments (ndog=%d band=%d)", ndog, band);
        return VK_ERR_PARAMETER;
    }
    if (nb == 0 || nx < 3 || ny < 3 || nz < 3) return VK_OK;
    const int nlev = ndog - 2;
    const long long vol = (long long)nx * ny * nz;
    // grid.z <= 65535: split the batch into chunks
    const long long zdiv = band == 0 ? 32LL * nlev : (long long)(nz - 2) * nlev;  // band 0: up to 32 z chunks
    const int per = (int)(65535 / zdiv) > 0 ? (int)(65535 / zdiv) : 1;
    for (int b0 = 0; b0 < nb; b0 += per) {
        const int nbc = nb - b0 < per ? nb - b0 : per;
        DogPtrs d{};
        for (int i = 0; i < ndog; ++i) d.p[i] = dogs_host[i] + (long long)b0 * vol;
        if (band == 0) {
            // z chunks (>= 8 planes) so the serial plane stream is not the latency bound
            const long long cols = (long long)((nx - 2 + 29) / 30) * ((ny - 2 + 4 * kDetRows - 1) / (4 * kDetRows)) *
                                   nlev * nbc;
            int nzc = 1;
            while (cols * nzc < 16LL * 148 && (nz - 2) / (nzc + 1) >= 8 && nzc < 32) ++nzc;
            const int tz = (nz - 2 + nzc - 1) / nzc;
            nzc = (nz - 2 + tz - 1) / tz;
            dim3 grid((nx - 2 + 29) / 30, (ny - 2 + 4 * kDetRows - 1) / (4 * kDetRows), (unsigned)(nlev * nbc * nzc));
            detect_band0_rb_kernel<<<grid, dim3(32, 4), 0, as_stream(stream)>>>(
                d, nlev, nx, ny, nz, seg_base, contrast_min, cand_keys + (long long)b0 * cap, cand_count + b0, cap, tz,
                nzc);
        } else {
            dim3 grid((nx - 2 + 31) / 32, (ny - 2 + 3) / 4, (unsigned)((long long)(nz - 2) * nlev * nbc));
            detect_kernel<<<grid, dim3(32, 4), 0, as_stream(stream)>>>(d, nlev, nx, ny, nz, seg_base, band, contrast_min,
                                                                       cand_keys + (long long)b0 * cap, cand_count + b0,
                                                                       cap);
        }
        count_launch();
    }
    return cuda_status(cudaGetLastError(), "detect launch");
}

extern "C" int vk_order_keypoints(unsigned long long* cand_keys, const int* cand_count, int nb, int cap,
                                  const int* seg_info_host, const double* seg_sigma_host, int nseg,
                                  const vk_level* dog_levels, vk_kp* kps, double* pos, double* sigma, float* dog,
                                  int8_t* sign, int* vol_offset, int* total, int kp_cap, void* stream) {
    if (!cand_keys || !cand_count || nb < 0 || cap < 0 || !seg_info_host || !seg_sigma_host || nseg < 1 ||
        nseg > kMaxSeg || !dog_levels || !kps || !pos || !sigma || !dog || !sign || !vol_offset || !total) {
        set_error("vk_order_keypoints: bad arguments (nseg=%d)", nseg);
        return VK_ERR_PARAMETER;
    }
    cudaStream_t st = as_stream(stream);
    if (nb == 0) return VK_OK;
    SegInfo s{};
    for (int i = 0; i < nseg; ++i) {
        s.octave[i] = seg_info_host[4 * i + 0];
        s.level[i] = seg_info_host[4 * i + 1];
        s.lvl[i] = seg_info_host[4 * i + 2];
        s.ball[i] = seg_info_host[4 * i + 3];
        s.sigma[i] = seg_sigma_host[i];
    }
    batch_offsets_kernel<<<1, 32, 0, st>>>(cand_count, nb, cap, vol_offset, total);
    count_launch();
    if (cap > 0) {
        chunk_sort_kernel<<<dim3((cap + kSortChunk - 1) / kSortChunk, nb), 1024, 0, st>>>(
            cand_keys, cand_count, cap);
        count_launch();
        dim3 grid((cap + 255) / 256, nb);
        order_kernel<<<grid, 256, 0, st>>>(cand_keys, cand_count, cap, vol_offset, s, dog_levels, kps, pos, sigma, dog,
                                           sign, kp_cap);
        count_launch();
    }
    return cuda_status(cudaGetLastError(), "order launch");
}

extern "C" int vk_extrema_from_map(const int16_t* map, const float* dog_cur, int nx, int ny, int nz, int seg, int band,
                                   float contrast_min, unsigned long long* cand_keys, int* cand_count, int cap,
                                   void* stream) {
    if (!map || !dog_cur || !cand_keys || !cand_count || nx < 1 || ny < 1 || nz < 1 || band < 0 || band > 80 ||
        seg < 0 || seg > 4095 || cap < 0) {
        set_error("vk_extrema_from_map: bad arguments");
        return VK_ERR_PARAMETER;
    }
    const long long vol = (long long)nx * ny * nz;
    extrema_from_map_kernel<<<(unsigned)((vol + 255) / 256), 256, 0, as_stream(stream)>>>(
        map, dog_cur, nx, ny, nz, seg, band, contrast_min, cand_keys, cand_count, cap);
    count_launch();
    return cuda_status(cudaGetLastError(), "extrema launch");
}

extern "C" int vk_refine_keypoints(const vk_kp* kps, const int* n_kp_dev, int n_kp_max, const vk_level* dog_levels,
                                   int levels_per_octave, double kappa, const double* sigma, double* out,
                                   void* stream) {
    if (!kps || !n_kp_dev || n_kp_max < 0 || !dog_levels || levels_per_octave < 4 || !(kappa > 1.0) || !sigma ||
        !out) {
        set_error("vk_refine_keypoints: bad arguments");
        return VK_ERR_PARAMETER;
    }
    if (n_kp_max == 0) return VK_OK;
    const int grid = n_kp_max < 256 * 148 ? (n_kp_max + 255) / 256 : 148;
    refine_kernel<<<grid, 256, 0, as_stream(stream)>>>(kps, n_kp_dev, n_kp_max, dog_levels, levels_per_octave, kappa,
                                                       sigma, out);
    count_launch();
    return cuda_status(cudaGetLastError(), "refine launch");
}
