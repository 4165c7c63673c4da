// vk_match_tc.cu -- nearest / second-nearest neighbour search for int8 rank
// descriptors (SIFT-Rank, RRIEF) on the 5th-generation tensor cores.
//
// Reference: match.py:70-121 (euclidean_distances + nearest_neighbor_matches):
// d2 = |a|^2 + |b|^2 - 2 a.b in float64, np.argmin (first minimum), second
// order statistic, ratio test.  For int8 rows the dot products are exact in
// int32 (tcgen05.mma kind::i8, s32 accumulators) and so is d2, so the integer
// minimum / tie order is identical to the reference's float64 one.
//
// One CTA = 128 query rows (M = 128) x a slice of reference rows, swept in
// tiles of 128 rows (N = 128; two CTAs per SM, 256 TMEM columns each):
//   * the query tile sits in shared memory for the whole sweep; reference
//     tiles are staged with cp.async (16-byte chunks) into the canonical
//     no-swizzle K-major core-matrix layout (8 rows x 16 bytes per core
//     matrix), double-buffered;
//   * one elected thread issues K/32 tcgen05.mma per tile into one of two
//     128-column TMEM accumulators and commits to an mbarrier, so the MMA of
//     tile t+1 runs while all 8 warps reduce tile t;
//   * epilogue: warp w reads TMEM lanes 32*(w%4).. (its query rows), columns
//     128*(w/4).. of the tile (tcgen05.ld 32x32b.x32), forms d' = |b|^2 - 2 a.b
//     and keeps the running (first) minimum + second minimum, testing four
//     columns at a time against the current second minimum;
//   * per (slice, row) partial results are merged in slice order by
//     match_merge_kernel (vk_match.cu), which adds |a|^2 and applies the
//     sqrt + ratio test in float64.
// Rows [ex_lo, ex_hi) of the reference set are skipped (database matching:
// the query subject's own rows) and later indices are reported compacted; the
// range is either one for all queries or per query row (row_ex), so a whole
// database of subjects is matched in one launch.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <climits>

#include "vk_common.cuh"

namespace vk {

constexpr int kTcM = 128;        // query rows per CTA
constexpr int kTcN = 128;        // reference rows per tile (2 CTAs / SM share TMEM)
constexpr int kTcThreads = 256;  // 8 warps

// Canonical K-major no-swizzle layout: core matrix (8 rows x 16 B) at
// (row / 8) * SBO + (kbyte / 16) * LBO, rows 16 B apart inside it.
template <int KB>
struct TcGeom {
    static constexpr int KBYTES = 32 * KB;        // bytes per row (K)
    static constexpr int LBO = 128;               // next 16-byte K chunk
    static constexpr int SBO = (KBYTES / 16) * 128;  // next 8-row group
    static constexpr int A_BYTES = kTcM * KBYTES;
    static constexpr int B_BYTES = kTcN * KBYTES;
    // smem: A | B[2] | norms[3][kTcN] | partial exchange | mbarriers | tmem addr
    // (norms of tile t live in slot t % 3: tile t+2 is staged while the
    // epilogue of tile t still reads them)
    static constexpr int OFF_B = A_BYTES;
    static constexpr int OFF_N = OFF_B + 2 * B_BYTES;
    static constexpr int OFF_X = OFF_N + 3 * kTcN * 4;
    static constexpr int OFF_BAR = OFF_X + kTcM * 16;
    static constexpr int SMEM = OFF_BAR + 32;
};

VK_D unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

VK_D unsigned long long umma_desc(unsigned saddr, int lbo, int sbo) {
    unsigned long long d = 0;
    d |= (unsigned long long)((saddr & 0x3FFFF) >> 4);
    d |= (unsigned long long)((lbo >> 4) & 0x3FFF) << 16;
    d |= (unsigned long long)((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;  // descriptor version (sm_100)
    return d;         // base offset 0, no swizzle
}

// kind::i8 instruction descriptor: D s32, A/B signed 8-bit, both K-major.
constexpr unsigned tc_idesc(int m, int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((unsigned)(n >> 3) << 17) | ((unsigned)(m >> 4) << 24);
}

VK_D void cp16(unsigned dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0));
}

VK_D void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
VK_D void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

VK_D void mbar_wait_parity(unsigned bar, unsigned parity) {
    unsigned ok = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    } while (!ok);
}

VK_D void tmem_ld32(unsigned taddr, int (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct Top2 {
    int m1, m2, i1;
};

VK_D void top2_push(Top2& t, int d, int j) {
    if (d < t.m1) {
        t.m2 = t.m1;
        t.m1 = d;
        t.i1 = j;
    } else if (d < t.m2) {
        t.m2 = d;
    }
}

// Stage reference tile rows [j0, j0 + kTcN) (zero rows past nb) + their norms.
template <int KB>
VK_D void stage_b(const uint8_t* __restrict__ b, const int* __restrict__ bnorm, int nb, int j0, unsigned sb,
                  unsigned sn) {
    using G = TcGeom<KB>;
    constexpr int CH = G::KBYTES / 16;  // 16-byte chunks per row
    for (int e = threadIdx.x; e < kTcN * CH; e += kTcThreads) {
        const int r = e / CH, c = e - r * CH;
        const int j = j0 + r;
        const bool ok = j < nb;
        cp16(sb + (unsigned)((r >> 3) * G::SBO + c * G::LBO + (r & 7) * 16),
             b + (long long)(ok ? j : 0) * G::KBYTES + 16 * c, ok);
    }
    // the norms array is padded (zeros) to whole tiles
    for (int e = threadIdx.x; e < kTcN / 4; e += kTcThreads) cp16(sn + 16u * e, bnorm + j0 + 4 * e, true);
    asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int KB>
__global__ void __launch_bounds__(kTcThreads, 2)
match_i8_tc_kernel(const uint8_t* __restrict__ a, int na, const uint8_t* __restrict__ b, const int* __restrict__ bnorm,
                   const int* __restrict__ neq_flag, int nb, int tiles_per_slice, int ex_lo_all, int ex_hi_all,
                   const int2* __restrict__ row_ex,
                   long long* __restrict__ pm1, long long* __restrict__ pm2, int* __restrict__ pi1) {
    using G = TcGeom<KB>;
    constexpr int CH = G::KBYTES / 16;
    extern __shared__ __align__(1024) uint8_t smem[];
    const unsigned s0 = su32(smem);
    const unsigned sA = s0, sB = s0 + G::OFF_B, sN = s0 + G::OFF_N;
    const int* nrm_s = reinterpret_cast<const int*>(smem + G::OFF_N);
    int4* xch = reinterpret_cast<int4*>(smem + G::OFF_X);
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + G::OFF_BAR);
    unsigned* tmem_slot = reinterpret_cast<unsigned*>(smem + G::OFF_BAR + 16);
    const unsigned bar0 = su32(bars), bar1 = bar0 + 8;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int q0 = blockIdx.x * kTcM;
    const int t_first = blockIdx.y * tiles_per_slice;
    const int n_tiles = (nb + kTcN - 1) / kTcN;
    const int t_last = min(n_tiles, t_first + tiles_per_slice);  // exclusive

    // ---- setup: TMEM (2 x 256 columns), mbarriers, query tile, first tile ----
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int e = tid; e < kTcM * CH; e += kTcThreads) {
        const int r = e / CH, c = e - r * CH;
        const int q = q0 + r;
        cp16(sA + (unsigned)((r >> 3) * G::SBO + c * G::LBO + (r & 7) * 16),
             a + (long long)(q < na ? q : 0) * G::KBYTES + 16 * c, q < na);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (t_first < t_last) stage_b<KB>(b, bnorm, nb, t_first * kTcN, sB, sN);
    if (t_first + 1 < t_last)
        stage_b<KB>(b, bnorm, nb, (t_first + 1) * kTcN, sB + (unsigned)G::B_BYTES, sN + (unsigned)(kTcN * 4));
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const unsigned tmem = *tmem_slot;
    const bool eq = neq_flag[0] == 0;  // every reference row has the same norm
    const int cnorm = bnorm[0];
    constexpr unsigned IDESC = tc_idesc(kTcM, kTcN);

    auto issue_mma = [&](int buf) {
        if (tid == 0) {
#pragma unroll
            for (int k = 0; k < KB; ++k) {
                const unsigned long long da = umma_desc(sA + 256u * k, G::LBO, G::SBO);
                const unsigned long long db = umma_desc(sB + (unsigned)(buf * G::B_BYTES) + 256u * k, G::LBO, G::SBO);
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                    " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}"
                    ::"r"(tmem + (unsigned)(buf * kTcN)), "l"(da), "l"(db), "r"(IDESC), "r"(k));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                         ::"r"(buf ? bar1 : bar0) : "memory");
        }
    };

    if (t_first < t_last) issue_mma(0);

    // Epilogue role: query row lr = 32 * (warp % 4) + lane, columns kTcN/2 * (warp / 4) ...
    const int lr = 32 * (warp & 3) + lane;
    const int ch = warp >> 2;
    const unsigned trow = tmem + ((unsigned)(32 * (warp & 3)) << 16);
    Top2 best{INT_MAX, INT_MAX, -1};
    int ex_lo = ex_lo_all, ex_hi = ex_hi_all;
    if (row_ex != nullptr) {
        const int2 e = row_ex[min(q0 + lr, na - 1)];
        ex_lo = e.x;
        ex_hi = e.y;
    }

    for (int t = t_first; t < t_last; ++t) {
        const int it = t - t_first, buf = it & 1;
        mbar_wait_parity(buf ? bar1 : bar0, (unsigned)(it >> 1) & 1u);
        tc_fence_after();
        // tile t+1 is staged (issued during the previous tile): start its MMA now.
        if (t + 1 < t_last) {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tc_fence_before();
            __syncthreads();
            tc_fence_after();
            issue_mma(buf ^ 1);
            // MMA t has finished reading its B buffer: stage tile t+2 into it.
            if (t + 2 < t_last) stage_b<KB>(b, bnorm, nb, (t + 2) * kTcN, sB + (unsigned)(buf * G::B_BYTES),
                                             sN + (unsigned)(((it + 2) % 3) * kTcN * 4));
        }
        // ---- epilogue of tile t ----
        const int j0 = t * kTcN + (kTcN / 2) * ch;
        const int* nt = nrm_s + (it % 3) * kTcN + (kTcN / 2) * ch;
        const unsigned tcol = trow + (unsigned)(buf * kTcN + (kTcN / 2) * ch);
        int v[kTcN / 2];
        tmem_ld32(tcol, *reinterpret_cast<int(*)[32]>(v));
        tmem_ld32(tcol + 32, *reinterpret_cast<int(*)[32]>(v + 32));
        const int4* n4 = reinterpret_cast<const int4*>(nt);
        if (!((j0 + kTcN / 2 > nb) || (j0 < ex_hi && j0 + kTcN / 2 > ex_lo))) {
            if (eq) {
                // All reference norms equal C (rank permutations): d' = C - 2 a.b,
                // so only dots above T = floor((C - m2) / 2) can enter the top 2.
                int T = (int)(((long long)cnorm - best.m2) >> 1);
#pragma unroll
                for (int g = 0; g < kTcN / 16; ++g) {
                    const int* w = v + 8 * g;
                    const int mx = max(__vimax3_s32(w[0], w[1], w[2]), __vimax3_s32(w[3], w[4], w[5]));
                    if (__builtin_expect(max(mx, max(w[6], w[7])) > T, 0)) {
                        const int jb = j0 + 8 * g;
#pragma unroll
                        for (int k = 0; k < 8; ++k) top2_push(best, cnorm - 2 * w[k], jb + k);
                        T = (int)(((long long)cnorm - best.m2) >> 1);
                    }
                }
            } else {
#pragma unroll
                for (int g = 0; g < kTcN / 16; ++g) {
                    const int4 na_ = n4[2 * g], nb_ = n4[2 * g + 1];
                    const int* w = v + 8 * g;
                    const int d0 = na_.x - 2 * w[0], d1 = na_.y - 2 * w[1], d2 = na_.z - 2 * w[2], d3 = na_.w - 2 * w[3];
                    const int d4 = nb_.x - 2 * w[4], d5 = nb_.y - 2 * w[5], d6 = nb_.z - 2 * w[6], d7 = nb_.w - 2 * w[7];
                    const int mn = min(__vimin3_s32(d0, d1, d2), __vimin3_s32(d3, d4, min(d5, min(d6, d7))));
                    if (__builtin_expect(mn < best.m2, 0)) {
                        const int jb = j0 + 8 * g;
                        top2_push(best, d0, jb);
                        top2_push(best, d1, jb + 1);
                        top2_push(best, d2, jb + 2);
                        top2_push(best, d3, jb + 3);
                        top2_push(best, d4, jb + 4);
                        top2_push(best, d5, jb + 5);
                        top2_push(best, d6, jb + 6);
                        top2_push(best, d7, jb + 7);
                    }
                }
            }
        } else {  // ragged last tile or excluded rows inside this half tile
#pragma unroll
            for (int k = 0; k < kTcN / 2; ++k) {
                const int j = j0 + k;
                if (j < nb && (j < ex_lo || j >= ex_hi)) top2_push(best, nt[k] - 2 * v[k], j);
            }
        }
        tc_fence_before();
    }

    // ---- merge the two column halves of each row ----
    __syncthreads();
    if (ch == 1) xch[lr] = make_int4(best.m1, best.m2, best.i1, 0);
    __syncthreads();
    if (ch == 0) {
        const int4 o = xch[lr];
        Top2 m = best;
        // the halves interleave by tile: ties go to the lower column index
        if (o.x < m.m1 || (o.x == m.m1 && (unsigned)o.z < (unsigned)m.i1)) {
            m.m2 = min(m.m1, o.y);
            m.m1 = o.x;
            m.i1 = o.z;
        } else {
            m.m2 = min(m.m2, o.x);
        }
        const int q = q0 + lr;
        if (q < na) {
            // |a|^2 from the staged query row (dp4a over its 16-byte chunks).
            int na2 = 0;
            for (int c = 0; c < CH; ++c) {
                const uint4 w = *reinterpret_cast<const uint4*>(smem + (lr >> 3) * G::SBO + c * G::LBO + (lr & 7) * 16);
                na2 = __dp4a((int)w.x, (int)w.x, na2);
                na2 = __dp4a((int)w.y, (int)w.y, na2);
                na2 = __dp4a((int)w.z, (int)w.z, na2);
                na2 = __dp4a((int)w.w, (int)w.w, na2);
            }
            const long long o1 = (long long)blockIdx.y * na + q;
            pm1[o1] = m.m1 == INT_MAX ? LLONG_MAX : (long long)na2 + m.m1;
            pm2[o1] = m.m2 == INT_MAX ? LLONG_MAX : (long long)na2 + m.m2;
            pi1[o1] = m.i1 < 0 ? -1 : (m.i1 < ex_lo ? m.i1 : (m.i1 >= ex_hi ? m.i1 - (ex_hi - ex_lo) : m.i1));
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}


// ---------------------------------------------------------------------------
// Warp-specialised persistent variant (default): one CTA per SM, 256 query
// rows (two M = 128 halves) x a slice of reference tiles of N = 128 rows.
//   * warp 0 (producer): TMA (cp.async.bulk.tensor.2d) loads -- the query
//     block once, then each reference tile, one box of 16 bytes x rows per
//     16-byte K chunk, straight into the canonical no-swizzle K-major layout
//     (a chunk's rows are 16 bytes apart: SBO = 128 B between 8-row core
//     matrices, LBO = rows x 16 B between K chunks); rows past the end are
//     zero-filled by the TMA unit; an 8-stage ring with full / empty
//     mbarriers;
//   * warp 1 (MMA): one elected thread issues 2 x K/32 tcgen05.mma.kind::i8
//     (M = 128 per query half, N = 128, s32) per tile into one of two TMEM
//     accumulator pairs (the whole 512 columns) and commits to the stage's
//     empty barrier and the accumulator's full barrier;
//   * warps 2..9 (epilogue): each thread owns one query row (lane quadrant =
//     warp % 4, query half = (warp - 2) / 4) and all 128 columns of a tile:
//     it copies its dot products out of TMEM, releases the accumulator (the
//     MMA of tile t + 2 may start) and screens them against the running second
//     minimum, 32 columns per vimax3 / vimin3 reduction.
// Two query halves per reference tile halve the L2 -> SM traffic per pair
// against an M = 128 CTA, and no CTA-wide barrier sits inside the sweep: TMA,
// MMA and epilogue overlap tile by tile.  Same integer arithmetic, tie order
// and merge as match_i8_tc_kernel.
constexpr int kWsM = 256, kWsN = 128, kWsStages = 8;
#ifndef VK_WS_EPI_WARPS
#define VK_WS_EPI_WARPS 8  // epilogue warps: 8 (one query row x 128 columns each) or 16 (x 64 columns; measured
                           // 8.96 vs 12.5 Tpairs/s: 113-register budget at 576 threads)
#endif
constexpr int kWsEpi = VK_WS_EPI_WARPS;
static_assert(kWsEpi == 8 || kWsEpi == 16, "8 or 16 epilogue warps");
constexpr int kWsCols = kWsN * 8 / kWsEpi;  // columns of a tile per epilogue thread
constexpr int kWsThreads = 64 + 32 * kWsEpi;  // producer warp, MMA warp, epilogue warps

template <int KB>
struct WsGeom {
    static constexpr int KBYTES = 32 * KB;
    static constexpr int CH = KBYTES / 16;        // 16-byte K chunks per row
    static constexpr int A_LBO = kWsM * 16;       // 4 KB between A K-chunks
    static constexpr int B_LBO = kWsN * 16;       // 2 KB between B K-chunks
    static constexpr int SBO = 128;               // next 8-row core matrix
    static constexpr int A_BYTES = kWsM * KBYTES;
    static constexpr int B_BYTES = kWsN * KBYTES;
    static constexpr int OFF_B = A_BYTES;
    static constexpr int OFF_X = OFF_B + kWsStages * B_BYTES;  // column-part exchange (16 epilogue warps)
    static constexpr int OFF_BAR = OFF_X + kWsM * 16;
    static constexpr int SMEM = OFF_BAR + 256;
};

VK_D void ws_wait(unsigned bar, unsigned parity) { mbar_wait_parity(bar, parity); }
VK_D void ws_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

template <int KB>
__global__ void __launch_bounds__(kWsThreads, 1)
match_i8_ws_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap, int na,
                   const uint8_t* __restrict__ a, const int* __restrict__ bnorm, const int* __restrict__ neq_flag,
                   int nb, int tiles_per_slice, int ex_lo_all, int ex_hi_all, const int2* __restrict__ row_ex,
                   long long* __restrict__ pm1, long long* __restrict__ pm2, int* __restrict__ pi1) {
    using G = WsGeom<KB>;
    extern __shared__ __align__(1024) uint8_t smem[];
    const unsigned s0 = su32(smem);
    const unsigned sA = s0, sB = s0 + G::OFF_B;
    const unsigned bars = s0 + G::OFF_BAR;  // full[8] empty[8] accf[2] acce[2] afull, tmem slot
    auto full = [&](int s) { return bars + 8u * s; };
    auto empty = [&](int s) { return bars + 64u + 8u * s; };
    auto accf = [&](int x) { return bars + 128u + 8u * x; };
    auto acce = [&](int x) { return bars + 144u + 8u * x; };
    const unsigned afull = bars + 160u;
    unsigned* tmem_slot = reinterpret_cast<unsigned*>(smem + G::OFF_BAR + 168);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int q0 = blockIdx.x * kWsM;
    const int t_first = blockIdx.y * tiles_per_slice;
    const int n_tiles = (nb + kWsN - 1) / kWsN;
    const int t_last = min(n_tiles, t_first + tiles_per_slice);
    const int nt = max(0, t_last - t_first);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 32) {
        for (int s = 0; s < kWsStages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full(s)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(empty(s)));
        }
        for (int x = 0; x < 2; ++x) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(accf(x)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(acce(x)), "n"(kWsEpi));
        }
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(afull));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const unsigned tmem = *tmem_slot;

    if (warp == 0) {
        // ---- producer: the query block once, then the reference tiles through the ring
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&bmap)) : "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(afull), "r"(G::A_BYTES)
                         : "memory");
            for (int c = 0; c < G::CH; ++c)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                    "[%4];" ::"r"(sA + (unsigned)(c * G::A_LBO)),
                    "l"(reinterpret_cast<uint64_t>(&amap)), "r"(16 * c), "r"(q0), "r"(afull)
                    : "memory");
            for (int it = 0; it < nt; ++it) {
                const int s = it % kWsStages;
                ws_wait(empty(s), ((unsigned)(it / kWsStages) & 1u) ^ 1u);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full(s)), "r"(G::B_BYTES)
                             : "memory");
                const int j0 = (t_first + it) * kWsN;
                for (int c = 0; c < G::CH; ++c)
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                        "%3}], [%4];" ::"r"(sB + (unsigned)(s * G::B_BYTES + c * G::B_LBO)),
                        "l"(reinterpret_cast<uint64_t>(&bmap)), "r"(16 * c), "r"(j0), "r"(full(s))
                        : "memory");
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ---- MMA issuer: accumulator x, query half m -> TMEM columns (2x + m) * 128
        constexpr unsigned IDESC = tc_idesc(128, kWsN);
        if (lane == 0) {
            ws_wait(afull, 0);
            for (int it = 0; it < nt; ++it) {
                const int s = it % kWsStages, x = it & 1;
                ws_wait(full(s), (unsigned)(it / kWsStages) & 1u);
                ws_wait(acce(x), ((unsigned)(it >> 1) & 1u) ^ 1u);
                tc_fence_after();
#pragma unroll
                for (int m = 0; m < 2; ++m)
#pragma unroll
                    for (int k = 0; k < KB; ++k) {
                        const unsigned long long da =
                            umma_desc(sA + (unsigned)(m * 128 * 16 + 2 * k * G::A_LBO), G::A_LBO, G::SBO);
                        const unsigned long long db =
                            umma_desc(sB + (unsigned)(s * G::B_BYTES + 2 * k * G::B_LBO), G::B_LBO, G::SBO);
                        asm volatile(
                            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                            " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}"
                            ::"r"(tmem + (unsigned)((2 * x + m) * kWsN)), "l"(da), "l"(db), "r"(IDESC), "r"(k));
                    }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                             ::"r"(empty(s)) : "memory");
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                             ::"r"(accf(x)) : "memory");
            }
        }
        __syncwarp();
    } else {
        // ---- epilogue: query row q, kWsCols columns (column part h) of each tile
        const int e = warp - 2;
        const int m = (e >> 2) & 1, h = e >> 3;  // query half, column part
        const int lr = 32 * (warp & 3) + lane;
        const int q = q0 + 128 * m + lr;
        const unsigned trow = tmem + ((unsigned)(32 * (warp & 3)) << 16);
        const bool eq = neq_flag[0] == 0;  // every reference row has the same norm
        const int cnorm = bnorm[0];
        Top2 best{INT_MAX, INT_MAX, -1};
        int ex_lo = ex_lo_all, ex_hi = ex_hi_all;
        if (row_ex != nullptr) {
            const int2 e2 = row_ex[min(q, na - 1)];
            ex_lo = e2.x;
            ex_hi = e2.y;
        }
        for (int it = 0; it < nt; ++it) {
            const int x = it & 1;
            ws_wait(accf(x), (unsigned)(it >> 1) & 1u);
            tc_fence_after();
            int v[kWsCols];
            const unsigned tcol = trow + (unsigned)((2 * x + m) * kWsN + kWsCols * h);
#pragma unroll
            for (int c4 = 0; c4 < kWsCols / 32; ++c4)
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                    "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
                    "[%32];"
                    : "=r"(v[32 * c4 + 0]), "=r"(v[32 * c4 + 1]), "=r"(v[32 * c4 + 2]), "=r"(v[32 * c4 + 3]),
                      "=r"(v[32 * c4 + 4]), "=r"(v[32 * c4 + 5]), "=r"(v[32 * c4 + 6]), "=r"(v[32 * c4 + 7]),
                      "=r"(v[32 * c4 + 8]), "=r"(v[32 * c4 + 9]), "=r"(v[32 * c4 + 10]), "=r"(v[32 * c4 + 11]),
                      "=r"(v[32 * c4 + 12]), "=r"(v[32 * c4 + 13]), "=r"(v[32 * c4 + 14]), "=r"(v[32 * c4 + 15]),
                      "=r"(v[32 * c4 + 16]), "=r"(v[32 * c4 + 17]), "=r"(v[32 * c4 + 18]), "=r"(v[32 * c4 + 19]),
                      "=r"(v[32 * c4 + 20]), "=r"(v[32 * c4 + 21]), "=r"(v[32 * c4 + 22]), "=r"(v[32 * c4 + 23]),
                      "=r"(v[32 * c4 + 24]), "=r"(v[32 * c4 + 25]), "=r"(v[32 * c4 + 26]), "=r"(v[32 * c4 + 27]),
                      "=r"(v[32 * c4 + 28]), "=r"(v[32 * c4 + 29]), "=r"(v[32 * c4 + 30]), "=r"(v[32 * c4 + 31])
                    : "r"(tcol + 32u * c4));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) ws_arrive(acce(x));  // the accumulator may be overwritten (tile it + 2)
            const int j0 = (t_first + it) * kWsN + kWsCols * h;
            if (!((j0 + kWsCols > nb) || (j0 < ex_hi && j0 + kWsCols > ex_lo))) {
                if (eq) {
                    // d' = C - 2 a.b: only dots above T = floor((C - m2) / 2) can enter the top 2
                    int T = (int)(((long long)cnorm - best.m2) >> 1);
#pragma unroll
                    for (int g = 0; g < kWsCols / 32; ++g) {
                        const int* w = v + 32 * g;
                        int mx = __vimax3_s32(w[0], w[1], w[2]);
#pragma unroll
                        for (int k = 3; k < 31; k += 2) mx = __vimax3_s32(mx, w[k], w[k + 1]);
                        mx = max(mx, w[31]);
                        if (__builtin_expect(mx > T, 0)) {
#pragma unroll
                            for (int k = 0; k < 32; ++k) top2_push(best, cnorm - 2 * w[k], j0 + 32 * g + k);
                            T = (int)(((long long)cnorm - best.m2) >> 1);
                        }
                    }
                } else {
                    const int* nt_ = bnorm + j0;
#pragma unroll
                    for (int g = 0; g < kWsCols / 8; ++g) {
                        const int4 na_ = __ldg(reinterpret_cast<const int4*>(nt_ + 8 * g));
                        const int4 nb_ = __ldg(reinterpret_cast<const int4*>(nt_ + 8 * g + 4));
                        const int* w = v + 8 * g;
                        const int d0 = na_.x - 2 * w[0], d1 = na_.y - 2 * w[1], d2 = na_.z - 2 * w[2],
                                  d3 = na_.w - 2 * w[3];
                        const int d4 = nb_.x - 2 * w[4], d5 = nb_.y - 2 * w[5], d6 = nb_.z - 2 * w[6],
                                  d7 = nb_.w - 2 * w[7];
                        const int mn = min(__vimin3_s32(d0, d1, d2), __vimin3_s32(d3, d4, min(d5, min(d6, d7))));
                        if (__builtin_expect(mn < best.m2, 0)) {
                            const int jb = j0 + 8 * g;
                            top2_push(best, d0, jb);
                            top2_push(best, d1, jb + 1);
                            top2_push(best, d2, jb + 2);
                            top2_push(best, d3, jb + 3);
                            top2_push(best, d4, jb + 4);
                            top2_push(best, d5, jb + 5);
                            top2_push(best, d6, jb + 6);
                            top2_push(best, d7, jb + 7);
                        }
                    }
                }
            } else {  // ragged last tile or excluded rows inside this column part
#pragma unroll
                for (int k = 0; k < kWsCols; ++k) {
                    const int j = j0 + k;
                    if (j < nb && (j < ex_lo || j >= ex_hi)) top2_push(best, __ldg(bnorm + j) - 2 * v[k], j);
                }
            }
        }
        if (kWsEpi == 16) {
            // merge the two column parts of each row (epilogue warps only: named barrier 1); the parts
            // interleave by tile, so ties go to the lower column index
            int4* xch = reinterpret_cast<int4*>(smem + G::OFF_X);
            if (h == 1) xch[128 * m + lr] = make_int4(best.m1, best.m2, best.i1, 0);
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kWsEpi) : "memory");
            if (h == 0) {
                const int4 o = xch[128 * m + lr];
                if (o.x < best.m1 || (o.x == best.m1 && (unsigned)o.z < (unsigned)best.i1)) {
                    best.m2 = min(best.m1, o.y);
                    best.m1 = o.x;
                    best.i1 = o.z;
                } else {
                    best.m2 = min(best.m2, o.x);
                }
            }
        }
        if (q < na && (kWsEpi == 8 || h == 0)) {
            int na2 = 0;
            const uint4* row = reinterpret_cast<const uint4*>(a + (long long)q * G::KBYTES);
            for (int c = 0; c < G::CH; ++c) {
                const uint4 w = __ldg(row + c);
                na2 = __dp4a((int)w.x, (int)w.x, na2);
                na2 = __dp4a((int)w.y, (int)w.y, na2);
                na2 = __dp4a((int)w.z, (int)w.z, na2);
                na2 = __dp4a((int)w.w, (int)w.w, na2);
            }
            const long long o1 = (long long)blockIdx.y * na + q;
            pm1[o1] = best.m1 == INT_MAX ? LLONG_MAX : (long long)na2 + best.m1;
            pm2[o1] = best.m2 == INT_MAX ? LLONG_MAX : (long long)na2 + best.m2;
            pi1[o1] = best.i1 < 0 ? -1
                                  : (best.i1 < ex_lo ? best.i1 : (best.i1 >= ex_hi ? best.i1 - (ex_hi - ex_lo) : best.i1));
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Squared norms of int8 rows (KBYTES bytes each); rows past n are 0.  neq[0]
// (preset to 0) is set if any row's norm differs from row 0's.
__global__ void row_norms_i8_kernel(const uint8_t* __restrict__ b, int n, int kbytes, int* __restrict__ out, int n_pad,
                                    int* __restrict__ neq) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_pad) return;
    int s = 0, s0 = 0;
    if (j < n) {
        const uint32_t* r = reinterpret_cast<const uint32_t*>(b + (long long)j * kbytes);
        const uint32_t* r0 = reinterpret_cast<const uint32_t*>(b);
        for (int w = 0; w < kbytes / 4; ++w) {
            const int v = (int)__ldg(r + w), v0 = (int)__ldg(r0 + w);
            s = __dp4a(v, v, s);
            s0 = __dp4a(v0, v0, s0);
        }
        if (s != s0) neq[0] = 1;
    }
    out[j] = s;
}

// vk_match.cu: merge (slice, row) partials in slice order + sqrt + ratio test.
void launch_merge_ll(const long long* pm1, const long long* pm2, const int* pi1, int na, int slices, int metric,
                     double ratio, int* best, double* d1, double* d2, uint8_t* keep, cudaStream_t st);

template <int KB>
static int launch_tc(const uint8_t* a, int na, const uint8_t* b, int nb, double ratio, int ex_lo, int ex_hi,
                     const int2* row_ex, int* best, double* d1, double* d2, uint8_t* keep, cudaStream_t st) {
    using G = TcGeom<KB>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(match_i8_tc_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        if (e != cudaSuccess) return cuda_status(e, "match tc attribute");
        configured = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int qtiles = (na + kTcM - 1) / kTcM;
    const int n_tiles = (nb + kTcN - 1) / kTcN;
    // (query tile, slice) CTAs: about four waves of two CTAs per SM, so long
    // reference sets are split even when there are few query tiles
    int slices = (8 * sms + qtiles - 1) / qtiles;
    if (slices > n_tiles / 8) slices = n_tiles / 8;  // >= 8 tiles per CTA: amortise setup and the merge
    if (slices < 1) slices = 1;
    const int per = (n_tiles + slices - 1) / slices;
    slices = (n_tiles + per - 1) / per;
    const int n_pad = n_tiles * kTcN;
    const size_t part = (size_t)slices * na;
    void* scratch = nullptr;
    const size_t bytes = part * 16 + part * 4 + (size_t)n_pad * 4 + 32;
    cudaError_t e = cudaMallocAsync(&scratch, bytes, st);
    if (e != cudaSuccess) return cuda_status(e, "match tc scratch");
    long long* pm1 = static_cast<long long*>(scratch);
    long long* pm2 = pm1 + part;
    int* pi1 = reinterpret_cast<int*>(pm2 + part);
    int* norms = pi1 + part + ((4 - (part & 3)) & 3);  // 16-byte aligned (part*20 bytes precede)
    int* neq = norms + n_pad;
    e = cudaMemsetAsync(neq, 0, 4, st);
    if (e != cudaSuccess) return cuda_status(e, "match tc flag");
    row_norms_i8_kernel<<<(n_pad + 255) / 256, 256, 0, st>>>(b, nb, G::KBYTES, norms, n_pad, neq);
    count_launch();
    match_i8_tc_kernel<KB><<<dim3(qtiles, slices), kTcThreads, G::SMEM, st>>>(a, na, b, norms, neq, nb, per, ex_lo,
                                                                             ex_hi, row_ex, pm1, pm2, pi1);
    count_launch();
    launch_merge_ll(pm1, pm2, pi1, na, slices, 1, ratio, best, d1, d2, keep, st);
    cudaFreeAsync(scratch, st);
    return cuda_status(cudaGetLastError(), "match tc launch");
}

static PFN_cuTensorMapEncodeTiled_v12000 g_enc = nullptr;

static bool ws_encode(CUtensorMap* m, const uint8_t* base, int rows, int kbytes, int box_rows) {
    if (!g_enc) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        g_enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    // 2-D view (kbytes, rows) of the int8 rows; a box is one 16-byte K chunk of box_rows rows
    cuuint64_t dims[2] = {(cuuint64_t)kbytes, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)kbytes};
    cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    return g_enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 0: warp-specialised TMA kernel (match_i8_ws_kernel, default), 1: match_i8_tc_kernel (A/B)
static int g_tc_kernel = 0;

template <int KB>
static int launch_ws(const uint8_t* a, int na, const uint8_t* b, int nb, double ratio, int ex_lo, int ex_hi,
                     const int2* row_ex, int* best, double* d1, double* d2, uint8_t* keep, cudaStream_t st) {
    using G = WsGeom<KB>;
    CUtensorMap amap, bmap;
    if (!ws_encode(&amap, a, na, G::KBYTES, kWsM) || !ws_encode(&bmap, b, nb, G::KBYTES, kWsN)) return -1;
    static bool configured = false;
    if (!configured) {
        cudaError_t e =
            cudaFuncSetAttribute(match_i8_ws_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        if (e != cudaSuccess) return cuda_status(e, "match ws attribute");
        configured = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int qtiles = (na + kWsM - 1) / kWsM;
    const int n_tiles = (nb + kWsN - 1) / kWsN;
    // (query tile, slice) CTAs, one per SM at a time, >= 8 reference tiles per CTA: the slice
    // count whose CTA total fills its last wave best (>= 95% wave efficiency: the smallest such
    // count, fewer partials to merge), at least one full wave when the shape allows
    const int s_max = max(1, min(n_tiles / 8, 256));
    int slices = 1;
    double best_eff = -1.0;
    for (int sc = 1; sc <= s_max; ++sc) {
        const int per_ = (n_tiles + sc - 1) / sc, real = (n_tiles + per_ - 1) / per_;
        const long long ctas = (long long)qtiles * real;
        const double eff = (double)ctas / (double)(((ctas + sms - 1) / sms) * sms);
        const bool full = ctas >= sms;
        const double score = eff + (full ? 1.0 : 0.0);
        if (score > best_eff + 1e-9) {
            best_eff = score;
            slices = real;
        }
        if (full && eff >= 0.95) break;
    }
    const int per = (n_tiles + slices - 1) / slices;
    slices = (n_tiles + per - 1) / per;
    const int n_pad = n_tiles * kWsN;
    const size_t part = (size_t)slices * na;
    void* scratch = nullptr;
    const size_t bytes = part * 16 + part * 4 + (size_t)n_pad * 4 + 32;
    cudaError_t e = cudaMallocAsync(&scratch, bytes, st);
    if (e != cudaSuccess) return cuda_status(e, "match ws scratch");
    long long* pm1 = static_cast<long long*>(scratch);
    long long* pm2 = pm1 + part;
    int* pi1 = reinterpret_cast<int*>(pm2 + part);
    int* norms = pi1 + part + ((4 - (part & 3)) & 3);  // 16-byte aligned
    int* neq = norms + n_pad;
    e = cudaMemsetAsync(neq, 0, 4, st);
    if (e != cudaSuccess) return cuda_status(e, "match ws flag");
    row_norms_i8_kernel<<<(n_pad + 255) / 256, 256, 0, st>>>(b, nb, G::KBYTES, norms, n_pad, neq);
    count_launch();
    match_i8_ws_kernel<KB><<<dim3(qtiles, slices), kWsThreads, G::SMEM, st>>>(
        amap, bmap, na, a, norms, neq, nb, per, ex_lo, ex_hi, row_ex, pm1, pm2, pi1);
    count_launch();
    launch_merge_ll(pm1, pm2, pi1, na, slices, 1, ratio, best, d1, d2, keep, st);
    cudaFreeAsync(scratch, st);
    return cuda_status(cudaGetLastError(), "match ws launch");
}

// Entry from vk_match_excluding for metric 1 rows whose byte width is a
// multiple of 32 (<= 128) and 16-byte aligned pointers; returns -1 when the
// shape is not covered (caller falls back to the dp4a kernel).
int match_i8_tensor(const uint8_t* a, int na, const uint8_t* b, int nb, int dim, double ratio, int ex_lo, int ex_hi,
                    const int2* row_ex, int* best, double* d1, double* d2, uint8_t* keep, cudaStream_t st) {
    if (dim % 32 != 0 || dim > 128 || ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15))
        return -1;
    if (g_tc_kernel == 0) {
        int rc = -1;
        switch (dim / 32) {
            case 1: rc = launch_ws<1>(a, na, b, nb, ratio, ex_lo, ex_hi, row_ex, best, d1, d2, keep, st); break;
            case 2: rc = launch_ws<2>(a, na, b, nb, ratio, ex_lo, ex_hi, row_ex, best, d1, d2, keep, st); break;
            case 3: rc = launch_ws<3>(a, na, b, nb, ratio, ex_lo, ex_hi, row_ex, best, d1, d2, keep, st); break;
            default: rc = launch_ws<4>(a, na, b, nb, ratio, ex_lo, ex_hi, row_ex, best, d1, d2, keep, st); break;
        }
        if (rc >= 0) return rc;  // (no tensor-map support: the barrier-synchronised kernel)
    }
    switch (dim / 32) {
        case 1: return launch_tc<1>(a, na, b, nb, ratio, ex_lo, ex_hi, row_ex, best, d1, d2, keep, st);
        case 2: return launch_tc<2>(a, na, b, nb, ratio, ex_lo, ex_hi, row_ex, best, d1, d2, keep, st);
        case 3: return launch_tc<3>(a, na, b, nb, ratio, ex_lo, ex_hi, row_ex, best, d1, d2, keep, st);
        default: return launch_tc<4>(a, na, b, nb, ratio, ex_lo, ex_hi, row_ex, best, d1, d2, keep, st);
    }
}

}  // namespace vk

extern "C" int vk_set_match_tc_kernel(int k) {
    if (k < 0 || k > 1) {
        vk::set_error("vk_set_match_tc_kernel: 0 (warp-specialised TMA kernel) or 1 (barrier-synchronised kernel)");
        return VK_ERR_PARAMETER;
    }
    vk::g_tc_kernel = k;
    return VK_OK;
}
