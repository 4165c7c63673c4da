// vk_consensus.cpp -- 7-DOF Hough consensus (match.py:124-359) as native host code.
//
// The reference's consensus is scalar Python over ~10^3 matches: per match a
// vote transform (match.py:124-133), coarse rotation bins (match.py:184-207),
// a smeared cell accumulator (match.py:246-268), then for at most 16 distinct
// clusters a least-squares refinement (Umeyama, match.py:136-162) and inlier
// sets (_agrees, match.py:210-224).  Everything the reference computes with a
// numpy / LAPACK call is computed here with the SAME call: the OpenBLAS that
// numpy itself links (dlopen'ed by path, vk_hough_init), with the arguments
// numpy's matmul / dot / linalg wrappers pass (cblas_dgemm for 3x3 @ 3x3 and
// (3,n) @ (n,3), cblas_dgemv for matrix @ vector and vector @ matrix,
// cblas_ddot for 1-D dot / norm, dgesdd 'A' with numpy's workspace query for
// np.linalg.svd, dgetrf for the sign of np.linalg.det).  Host-side float
// arithmetic follows CPython / numpy step for step: libm log / atan2 / acos,
// Python float %, pairwise summation for ndarray.sum(), sequential row sums
// for mean(axis=0).  tests/test_consensus.py checks the result against
// golden vectors made by the unmodified reference.
//
// One step stays numpy: the two nearest directions of _rotation_bins are
// np.argsort(-dots)[:2], and votes of frames built from the same icosphere
// often have EXACTLY equal dots, whose order is whatever numpy's (unstable,
// possibly SIMD) sort does on the host.  vk_hough_dots returns the dots, the
// host takes np.argsort of them, and vk_hough_consensus consumes the result.
#include <dlfcn.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <set>
#include <vector>

#include "volkey_b200.h"

namespace vk {
void set_error(const char* fmt, ...);
}

namespace {

typedef int64_t blasint;  // scipy-openblas64 ILP64 interface
enum { RowMajor = 101, NoTrans = 111, Trans = 112 };
typedef void (*dgemm_t)(blasint, blasint, blasint, blasint, blasint, blasint, double, const double*, blasint,
                        const double*, blasint, double, double*, blasint);
typedef void (*dgemv_t)(blasint, blasint, blasint, blasint, double, const double*, blasint, const double*, blasint,
                        double, double*, blasint);
typedef double (*ddot_t)(blasint, const double*, blasint, const double*, blasint);
typedef void (*dgesdd_t)(const char*, const blasint*, const blasint*, double*, const blasint*, double*, double*,
                         const blasint*, double*, const blasint*, double*, const blasint*, blasint*, blasint*, size_t);
typedef void (*dgetrf_t)(const blasint*, const blasint*, double*, const blasint*, blasint*, blasint*);

struct Blas {
    dgemm_t gemm = nullptr;
    dgemv_t gemv = nullptr;
    ddot_t dot = nullptr;
    dgesdd_t gesdd = nullptr;
    dgetrf_t getrf = nullptr;
    bool ok() const { return gemm && gemv && dot && gesdd && getrf; }
};
Blas g_blas;

constexpr int kOk = 0, kParam = 5, kNoConsensus = 6, kNotInit = 9, kRange = 10;
const double kRadToDeg = 180.0 / M_PI;  // CPython math.degrees
const double kTwoPi = 2.0 * M_PI;

struct M3 {
    double a[9];
};
struct V3 {
    double v[3];
};
struct Xform {
    double scale;
    M3 R;
    V3 t;
};

// 3-element kernels of this host's OpenBLAS.  The BLAS calls cost ~150 ns
// each (interface + dispatch), the hot loops make ~10^5 of them, so
// vk_hough_init pins inline restatements of the three kernels against the
// library on random operands and uses them only where they agree on every
// sample (kernels differ between DYNAMIC_ARCH core types: e.g. ddot is a
// plain sequential sum on Haswell / Zen and an FMA chain on SkylakeX);
// otherwise every product goes through the library call.
int g_dot_mode = -1, g_mv_mode = -1, g_mm_mode = -1;  // -1: call OpenBLAS
bool g_dirs_inline = false;  // the (K, 3) @ 3 direction dots through gemv_row_k too

inline double dot3_k(int mode, const double* a, const double* b) {
    if (mode == 0) return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
    return fma(a[2], b[2], fma(a[1], b[1], a[0] * b[0]));
}
// row r of a RowMajor NoTrans dgemv (a transposed-kernel dot)
inline double gemv_row_k(int mode, const double* r, const double* x) {
    if (mode == 0) return fma(r[2], x[2], fma(r[0], x[0], r[1] * x[1]));
    return fma(r[2], x[2], fma(r[1], x[1], r[0] * x[0]));
}
// C[i][j] of a 3x3x3 dgemm (row i of A, column j of B given as a strided vector)
inline double gemm_k(int mode, const double* r, const double* c, int cs) {
    if (mode == 0) return fma(r[2], c[2 * cs], fma(r[1], c[cs], r[0] * c[0]));
    return (r[0] * c[0] + r[1] * c[cs]) + r[2] * c[2 * cs];
}

// A @ B (numpy matmul of two C-contiguous 3x3)
inline M3 mm_nn(const M3& A, const M3& B) {
    M3 C;
    if (g_mm_mode < 0) {
        g_blas.gemm(RowMajor, NoTrans, NoTrans, 3, 3, 3, 1.0, A.a, 3, B.a, 3, 0.0, C.a, 3);
    } else {
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) C.a[3 * i + j] = gemm_k(g_mm_mode, A.a + 3 * i, B.a + j, 3);
    }
    return C;
}
// A @ B.T
inline M3 mm_nt(const M3& A, const M3& B) {
    M3 C;
    if (g_mm_mode < 0) {
        g_blas.gemm(RowMajor, NoTrans, Trans, 3, 3, 3, 1.0, A.a, 3, B.a, 3, 0.0, C.a, 3);
    } else {
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) C.a[3 * i + j] = gemm_k(g_mm_mode, A.a + 3 * i, B.a + 3 * j, 1);
    }
    return C;
}
// A @ x (matrix @ vector) == x' @ A.T (vector @ matrix): one dgemv
inline V3 mv(const M3& A, const double* x) {
    V3 y;
    if (g_mv_mode < 0) {
        g_blas.gemv(RowMajor, NoTrans, 3, 3, 1.0, A.a, 3, x, 1, 0.0, y.v, 1);
    } else {
        for (int j = 0; j < 3; ++j) y.v[j] = gemv_row_k(g_mv_mode, A.a + 3 * j, x);
    }
    return y;
}
inline double dot3(const double* a, const double* b) {
    return g_dot_mode < 0 ? g_blas.dot(3, a, 1, b, 1) : dot3_k(g_dot_mode, a, b);
}
inline double norm3(const double* a) { return sqrt(dot3(a, a)); }

// Pin the inline kernels against the library (vk_hough_init).
void pin_kernels() {
    uint64_t st = 0x9E3779B97F4A7C15ull;
    auto rnd = [&]() {  // splitmix64 -> normal-ish doubles over many binades
        st += 0x9E3779B97F4A7C15ull;
        uint64_t z = st;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const double u = (double)(z >> 11) * (1.0 / 9007199254740992.0) - 0.5;
        return ldexp(u, (int)(z % 24) - 8);
    };
    const int kTrials = 20000;
    bool dot_ok[2] = {true, true}, mv_ok[2] = {true, true}, mm_ok[2] = {true, true};
    for (int t = 0; t < kTrials; ++t) {
        M3 A, B, C;
        double x[3], y[3];
        for (int e = 0; e < 9; ++e) {
            A.a[e] = rnd();
            B.a[e] = rnd();
        }
        for (int c = 0; c < 3; ++c) x[c] = rnd();
        const double d = g_blas.dot(3, A.a, 1, x, 1);
        for (int m = 0; m < 2; ++m) dot_ok[m] = dot_ok[m] && dot3_k(m, A.a, x) == d;
        g_blas.gemv(RowMajor, NoTrans, 3, 3, 1.0, A.a, 3, x, 1, 0.0, y, 1);
        for (int m = 0; m < 2; ++m)
            for (int j = 0; j < 3; ++j) mv_ok[m] = mv_ok[m] && gemv_row_k(m, A.a + 3 * j, x) == y[j];
        g_blas.gemm(RowMajor, NoTrans, Trans, 3, 3, 3, 1.0, A.a, 3, B.a, 3, 0.0, C.a, 3);
        for (int m = 0; m < 2; ++m)
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) mm_ok[m] = mm_ok[m] && gemm_k(m, A.a + 3 * i, B.a + 3 * j, 1) == C.a[3 * i + j];
        g_blas.gemm(RowMajor, NoTrans, NoTrans, 3, 3, 3, 1.0, A.a, 3, B.a, 3, 0.0, C.a, 3);
        for (int m = 0; m < 2; ++m)
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) mm_ok[m] = mm_ok[m] && gemm_k(m, A.a + 3 * i, B.a + j, 3) == C.a[3 * i + j];
    }
    // the K-row gemv of the direction dots may take another code path of the kernel
    bool dirs_ok[2] = {true, true};
    for (int t = 0; t < kTrials / 8; ++t) {
        double D[3 * 48], x[3], y[48];
        for (int e = 0; e < 3 * 48; ++e) D[e] = rnd();
        for (int c = 0; c < 3; ++c) x[c] = rnd();
        const int K = 42 + t % 7;
        g_blas.gemv(RowMajor, NoTrans, K, 3, 1.0, D, 3, x, 1, 0.0, y, 1);
        for (int m = 0; m < 2; ++m)
            for (int k = 0; k < K; ++k) dirs_ok[m] = dirs_ok[m] && gemv_row_k(m, D + 3 * k, x) == y[k];
    }
    g_dot_mode = dot_ok[0] ? 0 : dot_ok[1] ? 1 : -1;
    g_mv_mode = mv_ok[0] ? 0 : mv_ok[1] ? 1 : -1;
    g_mm_mode = mm_ok[0] ? 0 : mm_ok[1] ? 1 : -1;
    g_dirs_inline = g_mv_mode >= 0 && dirs_ok[g_mv_mode];
}

// numpy pairwise summation (ndarray.sum over a contiguous run)
double pairwise(const double* a, long n) {
    if (n < 8) {
        double r = 0.0;
        for (long i = 0; i < n; ++i) r += a[i];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        long i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    long n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise(a, n2) + pairwise(a + n2, n - n2);
}

// Python float %: result has the sign of the divisor
inline double py_mod(double x, double w) {
    double m = fmod(x, w);
    if (m != 0.0) {
        if ((w < 0) != (m < 0)) m += w;
    } else {
        m = copysign(0.0, w);
    }
    return m;
}
inline long long py_imod(long long a, long long b) {
    long long m = a % b;
    return (m != 0 && ((m < 0) != (b < 0))) ? m + b : m;
}
inline long long py_floor(double x) { return (long long)floor(x); }

// sign of np.linalg.det (LU with partial pivoting, numpy's slogdet sign)
double det_sign(const M3& A) {
    double f[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) f[i + 3 * j] = A.a[3 * i + j];  // Fortran copy
    blasint n = 3, piv[3], info = 0;
    g_blas.getrf(&n, &n, f, &n, piv, &info);
    if (info > 0) return 0.0;
    double s = 1.0;
    for (int i = 0; i < 3; ++i) {
        if (piv[i] != i + 1) s = -s;
        if (f[i + 3 * i] < 0) s = -s;
    }
    return s;
}

// np.linalg.svd(A) (full_matrices): dgesdd 'A' on a Fortran copy, workspace from a query
bool svd3(const M3& A, M3& U, double* S, M3& VT) {
    double f[9], u[9], vt[9], q = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) f[i + 3 * j] = A.a[3 * i + j];
    blasint n = 3, lw = -1, info = 0, iw[24];
    g_blas.gesdd("A", &n, &n, f, &n, S, u, &n, vt, &n, &q, &lw, iw, &info, 1);
    if (info != 0) return false;
    lw = (blasint)q;
    if (lw < 1) lw = 1;
    std::vector<double> work((size_t)lw);
    g_blas.gesdd("A", &n, &n, f, &n, S, u, &n, vt, &n, work.data(), &lw, iw, &info, 1);
    if (info != 0) return false;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            U.a[3 * i + j] = u[i + 3 * j];
            VT.a[3 * i + j] = vt[i + 3 * j];
        }
    return true;
}

// similarity_from_correspondences (match.py:136-162) on rows idx of src / dst;
// false where the reference raises ParameterError (degenerate input)
bool umeyama(const double* src, const double* dst, const std::vector<int>& idx, Xform& out) {
    const long n = (long)idx.size();
    double mu_s[3], mu_d[3];
    for (int c = 0; c < 3; ++c) {
        mu_s[c] = src[3 * idx[0] + c];
        mu_d[c] = dst[3 * idx[0] + c];
    }
    for (long k = 1; k < n; ++k)
        for (int c = 0; c < 3; ++c) {
            mu_s[c] += src[3 * idx[k] + c];
            mu_d[c] += dst[3 * idx[k] + c];
        }
    for (int c = 0; c < 3; ++c) {
        mu_s[c] /= (double)n;
        mu_d[c] /= (double)n;
    }
    std::vector<double> ds(3 * n), dd(3 * n), sq(3 * n);
    for (long k = 0; k < n; ++k)
        for (int c = 0; c < 3; ++c) {
            ds[3 * k + c] = src[3 * idx[k] + c] - mu_s[c];
            dd[3 * k + c] = dst[3 * idx[k] + c] - mu_d[c];
            sq[3 * k + c] = ds[3 * k + c] * ds[3 * k + c];
        }
    M3 cov;
    g_blas.gemm(RowMajor, Trans, NoTrans, 3, 3, n, 1.0, dd.data(), 3, ds.data(), 3, 0.0, cov.a, 3);  // dd.T @ ds
    for (int e = 0; e < 9; ++e) cov.a[e] /= (double)n;
    M3 U, VT;
    double S[3];
    if (!svd3(cov, U, S, VT)) return false;  // (numpy raises LinAlgError; not reached for finite input)
    M3 sign = {{1, 0, 0, 0, 1, 0, 0, 0, 1}};
    if (det_sign(U) * det_sign(VT) < 0) sign.a[8] = -1.0;
    const M3 R = mm_nn(mm_nn(U, sign), VT);
    const double var_s = pairwise(sq.data(), 3 * n) / (double)n;
    if (var_s <= 0) return false;
    const double sd[3] = {S[0] * sign.a[0], S[1] * sign.a[4], S[2] * sign.a[8]};
    const double scale = pairwise(sd, 3) / var_s;
    if (scale <= 0) return false;
    M3 sR;
    for (int e = 0; e < 9; ++e) sR.a[e] = scale * R.a[e];
    const V3 m = mv(sR, mu_s);
    out.scale = scale;
    out.R = R;
    for (int c = 0; c < 3; ++c) out.t.v[c] = mu_d[c] - m.v[c];
    return true;
}

struct Ctx {
    int n;
    const int64_t* ia;
    const int64_t* ib;
    const double* src;  // (n, 3) keypoint a positions
    const double* dst;  // (n, 3) keypoint b positions
    std::vector<Xform> votes;
    std::vector<double> log_scale;
    double log_tol, rot_tol, trans_tol;

    // refine (match.py:275-290)
    Xform refine(const std::vector<int>& indices) const {
        if (indices.size() < 3) return votes[indices[0]];
        // {(index_a, index_b): i}: the last i of each pair, then sorted
        std::vector<std::pair<std::pair<int64_t, int64_t>, int>> last;
        last.reserve(indices.size());
        for (int i : indices) last.push_back({{ia[i], ib[i]}, i});
        std::stable_sort(last.begin(), last.end(),
                         [](const auto& x, const auto& y) { return x.first < y.first; });
        std::vector<int> idx;
        for (size_t k = 0; k < last.size(); ++k)
            if (k + 1 == last.size() || last[k + 1].first != last[k].first) idx.push_back(last[k].second);
        std::sort(idx.begin(), idx.end());
        if (idx.size() < 3) idx = indices;
        Xform t;
        if (!umeyama(src, dst, idx, t)) return votes[indices[0]];
        return t;
    }
    // np.linalg.norm(x_b - c.apply(x_a))
    double residual(const Xform& c, int i) const {
        const V3 y = mv(c.R, src + 3 * i);  // atleast_2d(x_a) @ R.T
        double d[3];
        for (int k = 0; k < 3; ++k) d[k] = dst[3 * i + k] - (c.scale * y.v[k] + c.t.v[k]);
        return norm3(d);
    }
    // [i for i, t in enumerate(votes) if _agrees(t, src[i], dst[i], c, s)] (match.py:210-224, 292-295)
    std::vector<int> agreeing(const Xform& c) const {
        std::vector<int> out;
        const double lc = log(c.scale);
        for (int i = 0; i < n; ++i) {
            if (fabs(log_scale[i] - lc) > log_tol) continue;
            // the three tests are pure: the cheap residual runs before the rotation angle
            if (!(residual(c, i) <= trans_tol)) continue;
            const M3 r = mm_nt(votes[i].R, c.R);
            const double cc = ((r.a[0] + r.a[4]) + r.a[8] - 1.0) / 2.0;
            const double ang = acos(std::min(1.0, std::max(-1.0, cc))) * kRadToDeg;
            if (ang > rot_tol) continue;
            out.push_back(i);
        }
        return out;
    }
    // evaluate (match.py:297-325)
    Xform evaluate(const std::vector<int>& cell, std::vector<int>& inl) const {
        Xform c = refine(cell);
        inl = agreeing(c);
        for (int it = 0; it < 3; ++it) {
            if (inl.size() < 3) break;
            c = refine(inl);
            std::vector<int> upd = agreeing(c);
            if (upd == inl) break;
            inl.swap(upd);
        }
        if (inl.size() >= 3) {
            for (double tol : {trans_tol / 2, trans_tol / 4}) {
                std::vector<int> tight;
                for (int i : inl)
                    if (residual(c, i) <= tol) tight.push_back(i);
                std::vector<std::pair<int64_t, int64_t>> distinct;
                for (int i : tight) distinct.push_back({ia[i], ib[i]});
                std::sort(distinct.begin(), distinct.end());
                distinct.erase(std::unique(distinct.begin(), distinct.end()), distinct.end());
                if (distinct.size() < 4) break;
                c = refine(tight);
            }
        }
        return c;
    }
};

// vote_transform (match.py:124-133) of match i
Xform vote_of(int i, const double* sig_a, const double* sig_b, const double* rot_a, const double* rot_b,
              const double* pos_a, const double* pos_b) {
    Xform t;
    t.scale = sig_b[i] / sig_a[i];
    M3 Ra, Rb;
    memcpy(Ra.a, rot_a + 9 * i, sizeof(Ra.a));
    memcpy(Rb.a, rot_b + 9 * i, sizeof(Rb.a));
    t.R = mm_nt(Rb, Ra);
    M3 sR;
    for (int e = 0; e < 9; ++e) sR.a[e] = t.scale * t.R.a[e];
    const V3 m = mv(sR, pos_a + 3 * i);
    for (int c = 0; c < 3; ++c) t.t.v[c] = pos_b[3 * i + c] - m.v[c];
    return t;
}

const double kEx[3] = {1.0, 0.0, 0.0}, kEy[3] = {0.0, 1.0, 0.0};

struct CellKey {
    long long k[6];
    bool operator<(const CellKey& o) const {
        for (int c = 0; c < 6; ++c)
            if (k[c] != o.k[c]) return k[c] < o.k[c];
        return false;
    }
    bool operator==(const CellKey& o) const { return memcmp(k, o.k, sizeof(k)) == 0; }
};

}  // namespace

// Bind numpy's OpenBLAS (path of numpy.libs/libscipy_openblas64_*.so, or any
// ILP64 OpenBLAS exporting the scipy_-prefixed, 64_-suffixed names).
extern "C" int vk_hough_init(const char* blas_path) {
    if (!blas_path) {
        vk::set_error("vk_hough_init: no BLAS path");
        return kParam;
    }
    void* h = dlopen(blas_path, RTLD_NOW | RTLD_LOCAL);
    if (!h) {
        vk::set_error("vk_hough_init: dlopen(%s) failed: %s", blas_path, dlerror());
        return kNotInit;
    }
    Blas b;
    b.gemm = (dgemm_t)dlsym(h, "scipy_cblas_dgemm64_");
    b.gemv = (dgemv_t)dlsym(h, "scipy_cblas_dgemv64_");
    b.dot = (ddot_t)dlsym(h, "scipy_cblas_ddot64_");
    b.gesdd = (dgesdd_t)dlsym(h, "scipy_dgesdd_64_");
    b.getrf = (dgetrf_t)dlsym(h, "scipy_dgetrf_64_");
    if (!b.ok()) {
        vk::set_error("vk_hough_init: %s lacks the scipy-openblas64 symbols", blas_path);
        return kNotInit;
    }
    g_blas = b;
    g_dot_mode = g_mv_mode = g_mm_mode = -1;
    pin_kernels();
    return kOk;
}

// Which inline kernels vk_hough_init pinned (-1 = the library call): for tests.
extern "C" int vk_hough_kernel_modes(int* modes) {
    if (!modes) return kParam;
    modes[0] = g_dot_mode;
    modes[1] = g_mv_mode;
    modes[2] = g_mm_mode;
    modes[3] = g_dirs_inline ? g_mv_mode : -1;
    return kOk;
}

// directions @ (R @ ex) for the vote transform R of every match
// (match.py:191-192): dots (n, K), row i = match i.
extern "C" int vk_hough_dots(int n, const double* rot_a, const double* rot_b, const double* dirs, int K,
                             double* dots) {
    if (!g_blas.ok()) {
        vk::set_error("vk_hough_dots: vk_hough_init was not called");
        return kNotInit;
    }
    if (n < 0 || K < 3 || (n > 0 && (!rot_a || !rot_b || !dirs || !dots))) {
        vk::set_error("vk_hough_dots: bad arguments");
        return kParam;
    }
    for (int i = 0; i < n; ++i) {
        M3 Ra, Rb;
        memcpy(Ra.a, rot_a + 9 * i, sizeof(Ra.a));
        memcpy(Rb.a, rot_b + 9 * i, sizeof(Rb.a));
        const M3 R = mm_nt(Rb, Ra);
        const V3 u = mv(R, kEx);
        if (!g_dirs_inline)
            g_blas.gemv(RowMajor, NoTrans, K, 3, 1.0, dirs, 3, u.v, 1, 0.0, dots + (size_t)i * K, 1);
        else
            for (int k = 0; k < K; ++k) dots[(size_t)i * K + k] = gemv_row_k(g_mv_mode, dirs + 3 * k, u.v);
    }
    return kOk;
}

// hough_consensus (match.py:227-348) for n matches.
//   ia, ib        : match.index_a / index_b (pair identity for deduplication)
//   sig_a, sig_b  : keypoint sigmas of the matched pairs
//   rot_a, rot_b  : (n, 9) frame rotations, C order
//   pos_a, pos_b  : (n, 3) keypoint positions
//   near          : (n, 2) np.argsort(-dots)[:, :2] of vk_hough_dots' output
//   b1, b2        : (K, 3) per-direction in-plane bases of _rotation_bins
//                   (match.py:195-199)
//   set           : log_scale_bin, trans_bin, log_scale_tol, rot_tol_deg, trans_tol
// Outputs: inliers (cap n) + count, the winning cell's vote count, the
// consensus transform.  Returns 0, 6 (NoConsensusError: *cell_votes = the
// densest cell's count), 5 (bad arguments) or 9 (vk_hough_init not called).
extern "C" int vk_hough_consensus(int n, const int64_t* ia, const int64_t* ib, const double* sig_a,
                                  const double* sig_b, const double* rot_a, const double* rot_b, const double* pos_a,
                                  const double* pos_b, const int64_t* near, const double* b1, const double* b2, int K,
                                  const double* set, int min_votes, int64_t* inliers, int* n_inliers, int* cell_votes,
                                  double* scale_out, double* rot_out, double* trans_out) {
    if (!g_blas.ok()) {
        vk::set_error("vk_hough_consensus: vk_hough_init was not called");
        return kNotInit;
    }
    if (n < 1 || K < 3 || !ia || !ib || !sig_a || !sig_b || !rot_a || !rot_b || !pos_a || !pos_b || !near || !b1 ||
        !b2 || !set || !inliers || !n_inliers || !cell_votes || !scale_out || !rot_out || !trans_out) {
        vk::set_error("vk_hough_consensus: bad arguments");
        return kParam;
    }
    const double log_bin = set[0], trans_bin = set[1];
    Ctx cx;
    cx.n = n;
    cx.ia = ia;
    cx.ib = ib;
    cx.src = pos_a;
    cx.dst = pos_b;
    cx.log_tol = set[2];
    cx.rot_tol = set[3];
    cx.trans_tol = set[4];
    cx.votes.resize(n);
    cx.log_scale.resize(n);
    std::vector<CellKey> keys((size_t)n * 64);  // 64 smeared cells per vote (duplicates included)
    for (int i = 0; i < n; ++i) {
        Xform& t = cx.votes[i];
        t = vote_of(i, sig_a, sig_b, rot_a, rot_b, pos_a, pos_b);
        // _rotation_bins (match.py:184-207); near = np.argsort(-dots)[:2] from the host
        const int n0 = (int)near[2 * i], n1 = (int)near[2 * i + 1];
        if (n0 < 0 || n0 >= K || n1 < 0 || n1 >= K) {
            vk::set_error("vk_hough_consensus: direction index out of range");
            return kParam;
        }
        const V3 v = mv(t.R, kEy);
        int rb[4][2];
        const int nd[2] = {n0, n1};
        for (int q = 0; q < 2; ++q) {
            const int d = nd[q];
            const double y = dot3(v.v, b2 + 3 * d), x = dot3(v.v, b1 + 3 * d);
            const double angle = py_mod(atan2(y, x), kTwoPi);
            const double frac = angle / kTwoPi * 8;
            const long long tr = (long long)frac;
            const long long sector = py_imod(tr, 8);
            const long long nb = py_imod(sector + ((frac - (double)tr) >= 0.5 ? 1 : -1), 8);
            rb[2 * q][0] = d;
            rb[2 * q][1] = (int)sector;
            rb[2 * q + 1][0] = d;
            rb[2 * q + 1][1] = (int)nb;
        }
        // smeared cells (match.py:246-268): a vote counts once per cell
        const double ls = log(t.scale);
        cx.log_scale[i] = ls;
        const long long sb[2] = {py_floor((ls - log_bin / 2) / log_bin), py_floor((ls + log_bin / 2) / log_bin)};
        long long tb[3][2];
        for (int a = 0; a < 3; ++a) {
            tb[a][0] = py_floor((t.t.v[a] - trans_bin / 2) / trans_bin);
            tb[a][1] = py_floor((t.t.v[a] + trans_bin / 2) / trans_bin);
        }
        CellKey* kv = &keys[(size_t)i * 64];
        for (int s0 = 0; s0 < 2; ++s0)
            for (int r = 0; r < 4; ++r)
                for (int x0 = 0; x0 < 2; ++x0)
                    for (int y0 = 0; y0 < 2; ++y0)
                        for (int z0 = 0; z0 < 2; ++z0)
                            *kv++ = {{sb[s0], rb[r][0], rb[r][1], tb[0][x0], tb[1][y0], tb[2][z0]}};
    }
    auto T = [] {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    };
    const double t1 = T();
    // The accumulator: cell -> member votes in append order, a vote counted
    // once per cell (match.py:261-268).  Keys are packed into one mixed-radix
    // integer per cell (numeric order == lexicographic tuple order), paired
    // with the vote index, and radix-sorted: cells come out in key order with
    // their members in vote order.
    long long lo[6], hi[6];
    for (int c = 0; c < 6; ++c) lo[c] = hi[c] = keys[0].k[c];
    for (const CellKey& k : keys)
        for (int c = 0; c < 6; ++c) {
            lo[c] = std::min(lo[c], k.k[c]);
            hi[c] = std::max(hi[c], k.k[c]);
        }
    int vbits = 1;
    while ((1ll << vbits) < n) ++vbits;
    unsigned __int128 span_all = (unsigned __int128)1 << vbits;
    unsigned long long span[6];
    bool fits = true;
    for (int c = 0; c < 6; ++c) {
        const unsigned __int128 sp = (unsigned __int128)((__int128)hi[c] - (__int128)lo[c]) + 1;
        span[c] = (unsigned long long)sp;
        span_all *= sp;
        if ((sp >> 62) || (span_all >> 63)) fits = false;
    }
    if (!fits) {
        vk::set_error("vk_hough_consensus: cell keys span more than 63 bits");
        return kRange;
    }
    std::vector<unsigned long long> code((size_t)n * 64), tmp((size_t)n * 64);
    for (size_t e = 0; e < code.size(); ++e) {
        unsigned long long v = 0;
        for (int c = 0; c < 6; ++c) v = v * span[c] + (unsigned long long)(keys[e].k[c] - lo[c]);
        code[e] = (v << vbits) | (unsigned long long)(e / 64);
    }
    unsigned long long maxv = 0;
    for (unsigned long long v : code) maxv = std::max(maxv, v);
    std::vector<size_t> cnt(2049);
    for (int shift = 0; shift < 64 && (maxv >> shift); shift += 11) {  // LSD radix sort, 11-bit digits
        std::fill(cnt.begin(), cnt.end(), 0);
        for (unsigned long long v : code) ++cnt[((v >> shift) & 2047) + 1];
        for (int d = 0; d < 2048; ++d) cnt[d + 1] += cnt[d];
        for (unsigned long long v : code) tmp[cnt[(v >> shift) & 2047]++] = v;
        code.swap(tmp);
    }
    code.erase(std::unique(code.begin(), code.end()), code.end());  // a vote once per cell
    struct Cell {
        size_t begin, count;
    };
    std::vector<Cell> groups;
    std::vector<int> member(code.size());
    const unsigned long long vmask = (1ull << vbits) - 1;
    size_t max_count = 0;
    for (size_t k = 0; k < code.size();) {
        const unsigned long long cell = code[k] >> vbits;
        size_t e = k;
        while (e < code.size() && (code[e] >> vbits) == cell) {
            member[e] = (int)(code[e] & vmask);
            ++e;
        }
        groups.push_back({k, e - k});
        max_count = std::max(max_count, e - k);
        k = e;
    }
    // sorted(cells, key=lambda k: (-len(cells[k]), k)): a stable counting sort
    // by count of the key-ordered groups
    {
        std::vector<size_t> start(max_count + 2, 0);
        for (const Cell& g : groups) ++start[max_count - g.count + 1];
        for (size_t c = 0; c <= max_count; ++c) start[c + 1] += start[c];
        std::vector<Cell> by(groups.size());
        for (const Cell& g : groups) by[start[max_count - g.count]++] = g;
        groups.swap(by);
    }
    if ((int)groups[0].count < min_votes) {
        *cell_votes = (int)groups[0].count;
        vk::set_error("densest cell has %d votes; %d required", (int)groups[0].count, min_votes);
        return kNoConsensus;
    }
    const double t2 = T();
    bool have = false;
    Xform best{};
    std::vector<int> best_inl;
    int best_cell = 0;
    std::set<std::vector<int>> seen;
    for (const Cell& g : groups) {
        if ((int)g.count < min_votes || seen.size() >= 16) break;
        std::vector<int> members(g.count);
        for (size_t k = 0; k < g.count; ++k) members[k] = member[g.begin + k];
        if (!seen.insert(members).second) continue;
        std::vector<int> inl;
        const Xform c = cx.evaluate(members, inl);
        if (!have || inl.size() > best_inl.size()) {
            have = true;
            best = c;
            best_inl = inl;
            best_cell = (int)g.count;
        }
    }
    if (getenv("VK_HOUGH_PROFILE")) fprintf(stderr, "hough: sort %.2f ms, evaluate %.2f ms, %zu cells\n", t2 - t1, T() - t2, groups.size());
    *n_inliers = (int)best_inl.size();
    for (size_t k = 0; k < best_inl.size(); ++k) inliers[k] = best_inl[k];
    *cell_votes = best_cell;
    *scale_out = best.scale;
    memcpy(rot_out, best.R.a, sizeof(best.R.a));
    memcpy(trans_out, best.t.v, sizeof(best.t.v));
    return kOk;
}
