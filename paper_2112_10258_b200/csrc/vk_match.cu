// vk_match.cu -- nearest / second-nearest neighbour matching with ratio test.
//
// Reference: match.py:64-121 (hamming_distances, euclidean_distances,
// nearest_neighbor_matches).
//
// Integer descriptors (SIFT-Rank / RRIEF ranks, packed BRIEF bits) are matched
// in exact integer arithmetic: squared Euclidean distance as
// |a|^2 + |b|^2 - 2 a.b in int64 (the reference's float64 evaluation of the same
// expression is exact for these magnitudes), Hamming as popcount of XOR.
// The best index is the first minimum (np.argmin), the second distance is the
// second order statistic of the row (np.partition(d, 1), match.py:110-113);
// distances are converted to float64 (sqrt for Euclidean) only at the end and
// the ratio test d1 <= ratio_max * d2 is evaluated in float64.
//
// Work split: each thread owns one query row; the reference rows are split
// into slices (grid.y) so that small query sets still fill the GPU; slices are
// merged in index order so ties keep the lowest index.
#include <climits>

#include "vk_common.cuh"

namespace vk {

constexpr int kMatchThreads = 128;

// 0: tensor-core path for int8 rows when the shape allows (default);
// 1: the dp4a kernel (vk_set_match_path, used by the tests to cross-check).
static int g_match_path = 0;
static int match_path() { return g_match_path; }
constexpr int kTileRows = 64;

struct Best {
    long long m1, m2;
    int i1;
};

VK_D void consider(Best& b, long long d, int j) {
    if (d < b.m1) {
        b.m2 = b.m1;
        b.m1 = d;
        b.i1 = j;
    } else if (d < b.m2) {
        b.m2 = d;
    }
}

// a: na rows, b: nbr rows.  metric 0: dim = bytes per row (multiple of 8);
// metric 1: dim = int8 values per row (multiple of 4).
template <int METRIC>
__global__ void __launch_bounds__(kMatchThreads)
match_int_kernel(const uint8_t* __restrict__ a, int na, const uint8_t* __restrict__ b, int nbr, int dim, int slice,
                 long long* __restrict__ pm1, long long* __restrict__ pm2, int* __restrict__ pi1, int ex_lo, int ex_hi) {
    extern __shared__ uint4 tile4[];
    uint8_t* tile = reinterpret_cast<uint8_t*>(tile4);
    __shared__ long long nrm[kTileRows];
    const int q = blockIdx.x * kMatchThreads + threadIdx.x;
    const int j0 = blockIdx.y * slice, j1 = min(nbr, j0 + slice);
    const int words = dim / 4;  // 32-bit words per row
    Best best{LLONG_MAX, LLONG_MAX, -1};
    long long na2 = 0;
    const uint32_t* arow = reinterpret_cast<const uint32_t*>(a + (long long)min(q, na - 1) * dim);
    if (METRIC == 1) {
        for (int w = 0; w < words; ++w) {
            const int v = (int)__ldg(arow + w);
            na2 += __dp4a(v, v, 0);
        }
    }
    for (int t = j0; t < j1; t += kTileRows) {
        const int rows = min(kTileRows, j1 - t);
        __syncthreads();
        const uint32_t* src = reinterpret_cast<const uint32_t*>(b + (long long)t * dim);
        uint32_t* dst = reinterpret_cast<uint32_t*>(tile);
        for (int i = threadIdx.x; i < rows * words; i += kMatchThreads) dst[i] = __ldg(src + i);
        __syncthreads();
        if (METRIC == 1 && threadIdx.x < rows) {
            long long s = 0;
            for (int w = 0; w < words; ++w) {
                const int v = (int)dst[threadIdx.x * words + w];
                s += __dp4a(v, v, 0);
            }
            nrm[threadIdx.x] = s;
        }
        __syncthreads();
        if (q < na) {
            for (int r = 0; r < rows; ++r) {
                const uint32_t* brow = dst + r * words;
                long long d;
                if (METRIC == 0) {
                    int pc = 0;
                    for (int w = 0; w < words; ++w) pc += __popc(__ldg(arow + w) ^ brow[w]);
                    d = pc;
                } else {
                    int dot = 0;
                    for (int w = 0; w < words; ++w) dot = __dp4a((int)__ldg(arow + w), (int)brow[w], dot);
                    d = na2 + nrm[r] - 2ll * dot;
                }
                const int jj = t + r;
                if (jj < ex_lo) consider(best, d, jj);
                else if (jj >= ex_hi) consider(best, d, jj - (ex_hi - ex_lo));
            }
        }
    }
    if (q < na) {
        const long long o = (long long)blockIdx.y * na + q;
        pm1[o] = best.m1;
        pm2[o] = best.m2;
        pi1[o] = best.i1;
    }
}

// fp64 descriptors: d2 = |a|^2 + |b|^2 - 2 a.b evaluated in fp64.
__global__ void __launch_bounds__(kMatchThreads)
match_f64_kernel(const double* __restrict__ a, int na, const double* __restrict__ b, int nbr, int dim, int slice,
                 double* __restrict__ pm1, double* __restrict__ pm2, int* __restrict__ pi1, int ex_lo, int ex_hi) {
    const int q = blockIdx.x * kMatchThreads + threadIdx.x;
    if (q >= na) return;
    const int j0 = blockIdx.y * slice, j1 = min(nbr, j0 + slice);
    const double* ar = a + (long long)q * dim;
    double na2 = 0.0;
    for (int k = 0; k < dim; ++k) na2 = dadd(na2, dmul(ar[k], ar[k]));
    double m1 = INFINITY, m2 = INFINITY;
    int i1 = -1;
    for (int j = j0; j < j1; ++j) {
        if (j >= ex_lo && j < ex_hi) continue;
        const double* br = b + (long long)j * dim;
        double nb2 = 0.0, dot = 0.0;
        for (int k = 0; k < dim; ++k) {
            nb2 = dadd(nb2, dmul(br[k], br[k]));
            dot = dadd(dot, dmul(ar[k], br[k]));
        }
        const double d2 = fmax(dsub(dadd(na2, nb2), dmul(2.0, dot)), 0.0);
        const int jo = j < ex_lo ? j : j - (ex_hi - ex_lo);
        if (d2 < m1) { m2 = m1; m1 = d2; i1 = jo; }
        else if (d2 < m2) m2 = d2;
    }
    const long long o = (long long)blockIdx.y * na + q;
    pm1[o] = m1;
    pm2[o] = m2;
    pi1[o] = i1;
}

template <typename T>
__global__ void match_merge_kernel(const T* __restrict__ pm1, const T* __restrict__ pm2, const int* __restrict__ pi1,
                                   int na, int slices, int metric, double ratio, int* __restrict__ best,
                                   double* __restrict__ d1, double* __restrict__ d2, uint8_t* __restrict__ keep) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= na) return;
    T m1 = pm1[q], m2 = pm2[q];
    int i1 = pi1[q];
    for (int s = 1; s < slices; ++s) {
        const long long o = (long long)s * na + q;
        const T b1 = pm1[o], b2 = pm2[o];
        if (b1 < m1) {
            m2 = m1 < b2 ? m1 : b2;
            m1 = b1;
            i1 = pi1[o];
        } else {
            m2 = m2 < b1 ? m2 : b1;
        }
    }
    double e1, e2;
    if (metric == 0) {
        e1 = (double)m1;
        e2 = (double)m2;
    } else {
        e1 = __dsqrt_rn((double)m1 > 0.0 ? (double)m1 : 0.0);
        e2 = __dsqrt_rn((double)m2 > 0.0 ? (double)m2 : 0.0);
    }
    if (e2 < e1) e2 = e1;  // np.maximum(d2, d1)
    best[q] = i1;
    d1[q] = e1;
    d2[q] = e2;
    keep[q] = e1 <= dmul(ratio, e2) ? 1 : 0;
}

void launch_merge_ll(const long long* pm1, const long long* pm2, const int* pi1, int na, int slices, int metric,
                     double ratio, int* best, double* d1, double* d2, uint8_t* keep, cudaStream_t st) {
    match_merge_kernel<long long><<<(na + 255) / 256, 256, 0, st>>>(pm1, pm2, pi1, na, slices, metric, ratio, best, d1,
                                                                    d2, keep);
    count_launch();
}

// vk_match_tc.cu: tcgen05 kind::i8 path for rank descriptors (-1: shape not covered).
int match_i8_tensor(const uint8_t* a, int na, const uint8_t* b, int nb, int dim, double ratio, int ex_lo, int ex_hi,
                    const int2* row_ex, int* best, double* d1, double* d2, uint8_t* keep, cudaStream_t st);

}  // namespace vk

using namespace vk;

extern "C" int vk_match_excluding(int metric, const void* a, int na, const void* b, int nb_rows, int dim,
                                  double ratio_max, int ex_lo, int ex_hi, int* best, double* d1, double* d2,
                                  uint8_t* keep, void* stream) {
    if (ex_lo < 0 || ex_hi < ex_lo || ex_hi > nb_rows) ex_lo = ex_hi = 0;
    if (metric < 0 || metric > 2 || !a || !b || na < 0 || nb_rows - (ex_hi - ex_lo) < 2 || dim < 1 || !best || !d1 ||
        !d2 || !keep || !(ratio_max > 0.0 && ratio_max <= 1.0) || (metric == 0 && dim % 8) ||
        (metric == 1 && dim % 4)) {
        set_error("vk_match: bad arguments (metric=%d na=%d nb=%d dim=%d)", metric, na, nb_rows, dim);
        return VK_ERR_PARAMETER;
    }
    if (na == 0) return VK_OK;
    cudaStream_t st = as_stream(stream);
    if (metric == 1 && match_path() == 0) {
        const int rc = match_i8_tensor(static_cast<const uint8_t*>(a), na, static_cast<const uint8_t*>(b), nb_rows, dim,
                                       ratio_max, ex_lo, ex_hi, nullptr, best, d1, d2, keep, st);
        if (rc >= 0) return rc;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int qblocks = (na + kMatchThreads - 1) / kMatchThreads;
    int slices = (2 * sms + qblocks - 1) / qblocks;
    int max_slices = (nb_rows + kTileRows - 1) / kTileRows;
    if (slices > max_slices) slices = max_slices;
    if (slices < 1) slices = 1;
    int slice = (nb_rows + slices - 1) / slices;
    slice = ((slice + kTileRows - 1) / kTileRows) * kTileRows;
    slices = (nb_rows + slice - 1) / slice;
    const size_t part = (size_t)slices * na;
    void* scratch = nullptr;
    const size_t bytes = part * 16 + part * 4;
    cudaError_t e = cudaMallocAsync(&scratch, bytes, st);
    if (e != cudaSuccess) return cuda_status(e, "match scratch");
    char* p = static_cast<char*>(scratch);
    dim3 grid(qblocks, slices);
    if (metric == 2) {
        double* pm1 = reinterpret_cast<double*>(p);
        double* pm2 = pm1 + part;
        int* pi1 = reinterpret_cast<int*>(pm2 + part);
        match_f64_kernel<<<grid, kMatchThreads, 0, st>>>(static_cast<const double*>(a), na, static_cast<const double*>(b),
                                                         nb_rows, dim, slice, pm1, pm2, pi1, ex_lo, ex_hi);
        count_launch();
        match_merge_kernel<double><<<(na + 255) / 256, 256, 0, st>>>(pm1, pm2, pi1, na, slices, metric, ratio_max, best,
                                                                     d1, d2, keep);
        count_launch();
    } else {
        long long* pm1 = reinterpret_cast<long long*>(p);
        long long* pm2 = pm1 + part;
        int* pi1 = reinterpret_cast<int*>(pm2 + part);
        const int smem = kTileRows * dim;
        if (metric == 0)
            match_int_kernel<0><<<grid, kMatchThreads, smem, st>>>(static_cast<const uint8_t*>(a), na,
                                                                   static_cast<const uint8_t*>(b), nb_rows, dim, slice,
                                                                   pm1, pm2, pi1, ex_lo, ex_hi);
        else
            match_int_kernel<1><<<grid, kMatchThreads, smem, st>>>(static_cast<const uint8_t*>(a), na,
                                                                   static_cast<const uint8_t*>(b), nb_rows, dim, slice,
                                                                   pm1, pm2, pi1, ex_lo, ex_hi);
        count_launch();
        match_merge_kernel<long long><<<(na + 255) / 256, 256, 0, st>>>(pm1, pm2, pi1, na, slices, metric, ratio_max,
                                                                        best, d1, d2, keep);
        count_launch();
    }
    cudaFreeAsync(scratch, st);
    return cuda_status(cudaGetLastError(), "match launch");
}

extern "C" int vk_match_rows_excluding(const void* a, int na, const void* b, int nb_rows, int dim, double ratio_max,
                                       const int* row_ex, int* best, double* d1, double* d2, uint8_t* keep,
                                       void* stream) {
    if (!a || !b || na < 0 || nb_rows < 3 || dim < 1 || !row_ex || !best || !d1 || !d2 || !keep ||
        !(ratio_max > 0.0 && ratio_max <= 1.0)) {
        set_error("vk_match_rows_excluding: bad arguments (na=%d nb=%d dim=%d)", na, nb_rows, dim);
        return VK_ERR_PARAMETER;
    }
    if (na == 0) return VK_OK;
    const int rc = match_i8_tensor(static_cast<const uint8_t*>(a), na, static_cast<const uint8_t*>(b), nb_rows, dim,
                                   ratio_max, 0, 0, reinterpret_cast<const int2*>(row_ex), best, d1, d2, keep,
                                   as_stream(stream));
    if (rc < 0) {
        set_error("vk_match_rows_excluding: rows must be 32/64/96/128 bytes at 16-byte aligned addresses");
        return VK_ERR_PARAMETER;
    }
    return rc;
}

extern "C" int vk_set_match_path(int path) {
    if (path < 0 || path > 1) {
        set_error("vk_set_match_path: path must be 0 (tensor cores) or 1 (dp4a)");
        return VK_ERR_PARAMETER;
    }
    g_match_path = path;
    return VK_OK;
}

extern "C" int vk_match(int metric, const void* a, int na, const void* b, int nb_rows, int dim, double ratio_max,
                        int* best, double* d1, double* d2, uint8_t* keep, void* stream) {
    return vk_match_excluding(metric, a, na, b, nb_rows, dim, ratio_max, 0, 0, best, d1, d2, keep, stream);
}
