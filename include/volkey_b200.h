/*
 * volkey_b200.h -- C ABI of the B200-native volkey hot path.
 *
 * The reference (/root/reference/pkg/src/volkey) is pure Python and has no
 * FFI; the drop-in boundary is therefore this C ABI, bound from Python with
 * ctypes (INTEGRATION.md shows the binding).  Every entry point names the
 * reference function it replaces (file:line, paths relative to
 * /root/reference/pkg/src/volkey).
 *
 * Conventions
 *  - Plain pointers and sizes only.  All array pointers are DEVICE pointers
 *    unless the parameter name ends in _host.  Work is enqueued on `stream`
 *    (a cudaStream_t passed as void*, NULL = legacy default stream) and is
 *    stream-ordered; nothing synchronises unless the function says so.
 *  - Volumes are float32, x-fastest ("on-disk" order, volume.py:4-5):
 *    element (x, y, z) of volume b lives at ((b*nz + z)*ny + y)*nx + x.
 *    The reference's in-memory numpy layout data[x, y, z] (z fastest) is
 *    converted with vk_transpose_* at the boundary.
 *  - Return value: VK_OK or an error code mirroring errors.py exit codes
 *    (5 parameter, 7 data); CUDA failures are VK_ERR_CUDA.  The message of
 *    the last failure on the calling thread is vk_last_error().  No C++
 *    exception crosses the ABI.
 *  - Caller owns every buffer.  Scratch space, when needed, is passed in.
 */
#ifndef VOLKEY_B200_H
#define VOLKEY_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VK_ABI_VERSION 2

#define VK_OK 0
#define VK_ERR_PARAMETER 5 /* errors.py:32-36 ParameterError */
#define VK_ERR_DATA 7      /* errors.py:46-50 DataError */
#define VK_ERR_CUDA 20
#define VK_ERR_CAPACITY 21 /* a caller-sized output buffer was too small */

#define VK_MAX_TAPS 65        /* blur radius <= 32 */
#define VK_MAX_DIRS 64        /* orientation direction-set size */
#define VK_MAX_FRAMES 8       /* frames per keypoint */
#define VK_MAX_PAIRS 256      /* BRIEF/RRIEF point pairs */

/* One pyramid level of a batch: volume b starts at base + b*vol_stride. */
typedef struct vk_level {
    const float* base;
    long long vol_stride;
    int nx, ny, nz;
    int pad_;
} vk_level;

/* Precomputed per-voxel gradient data of one pyramid level (batch strided):
 * g4[v] = (gx, gy, gz, |g|) in fp32 (|g| from fp64), bin[v] = nearest of the
 * 42 icosphere directions (exact np.argmax semantics) or 255 for g == 0. */
typedef struct vk_gradlevel {
    const void* g4;       /* kind 0: float4 (gx, gy, gz, |g|); kind 1: float |g| (vk_orient_field) */
    const uint8_t* bin;
    long long vol_stride;
    int nx, ny, nz;
    int kind;             /* 0: gradient volume (orientation + SIFT-Rank), 1: orientation field */
} vk_gradlevel;

/* One keypoint (device record). */
typedef struct vk_kp {
    int vol;      /* volume index within the batch */
    int lvl;      /* index into the level table (orientation / SIFT-Rank level) */
    int ix, iy, iz; /* lattice centre in that level's grid (orient.py:76-86) */
    int ball;     /* index into the ball table */
    int octave;
    int level;
} vk_kp;

/* Integer ball of offsets (orient.py:63-74): `count` packed offsets
 * starting at `start` in the offset table (reference x-major order);
 * windows[window_start + d2] is the orientation window for squared offset
 * length d2 (orient.py:116-117); windows32 (where taken) is its fp32 cast.
 * The same points in z-major order (ox fastest: coalesced gathers) start at
 * `zstart`; plane starts (pstart, r) are kept for tools. */
typedef struct vk_ball {
    int start;
    int count;
    int window_start;
    int max_d2;
    int zstart;
    int pstart;
    int r;
    int pad_;
} vk_ball;

/* One oriented frame: keypoint index plus the (primary, secondary) direction
 * pair that spawned it (-1 when the rotation was supplied directly). */
typedef struct vk_frame {
    int kp;
    int prim;
    int sec;
    int pad_;
} vk_frame;

const char* vk_last_error(void);
int vk_abi_version(void);
int vk_device_sm_count(int device);
/* Stream-ordered zero fill (graph-capturable); used for per-step counters. */
int vk_memset_async(void* ptr, long long bytes, void* stream);
/* Kernels launched by this library since load (instrumentation for bench.py). */
long long vk_launch_count(void);

/* ---------------------------------------------------------------- layout */
/* volume.py:64-70 conversions: data[x,y,z] (z fastest) <-> x-fastest. */
int vk_transpose_zfast_to_xfast(const float* src, float* dst, int nb, int nx, int ny, int nz, void* stream);
int vk_transpose_xfast_to_zfast(const float* src, float* dst, int nb, int nx, int ny, int nz, void* stream);

/* ----------------------------------------------------------- scale space */
/* convolve_array / convolve_separable (scalespace.py:45-92): replicate-
 * padded separable blur, x then y then z pass, fp32 products added in tap
 * order (no FMA).  taps_host: 2*radius+1 float32 weights (gaussian_kernel,
 * scalespace.py:35-42).  Optional fused epilogues:
 *   dog_out  != NULL: dog_out = src - dst        (build_dog_pyramid, scalespace.py:209-223)
 *   half_out != NULL: half_out = subsample_half(dst) (scalespace.py:95-109)  */
int vk_blur3d(const float* src, float* dst, float* dog_out, float* half_out,
              int nb, int nx, int ny, int nz, const float* taps_host, int radius, void* stream);

/* vk_blur3d with caller-owned scratch for the split (x, y) + z path: work
 * holds work_floats floats (>= nb*nz*ny*tp with tp = nx rounded up to a
 * multiple of 4: the intermediate's rows are pitched; 16-byte aligned; else
 * the call allocates its own, stream-ordered). */
int vk_blur3d_ws(const float* src, float* dst, float* dog_out, float* half_out, int nb, int nx, int ny, int nz,
                 const float* taps_host, int radius, float* work, long long work_floats, void* stream);

/* vk_blur3d_ws that also writes the PREVIOUS pair's difference
 * prev_dog = prev - src (the DoG level one below dog_out) from the (x, y)
 * pass's staged copy of src, so each pyramid level is read from HBM by one
 * kernel only.  prev and prev_dog: both NULL or both volumes of src's shape.
 * Results are bit-identical to separate vk_difference calls. */
int vk_blur3d_ws2(const float* src, float* dst, float* dog_out, float* half_out, const float* prev, float* prev_dog,
                  int nb, int nx, int ny, int nz, const float* taps_host, int radius, float* work,
                  long long work_floats, void* stream);

/* vk_blur3d with a caller-chosen work granularity: the z pass runs in chunks
 * of `zchunk` output planes per CTA (each chunk re-reads 2R warm-up planes),
 * the analogue of the reference's chunk (scalespace.py convolve_separable,
 * parallel.py task size).  Output is independent of zchunk. */
int vk_blur3d_chunked(const float* src, float* dst, int nb, int nx, int ny, int nz, const float* taps_host,
                      int radius, int zchunk, void* stream);

/* Blur kernel selection: 0 = split (x, y) kernel + z kernel through an
 * intermediate level (default), 1 = fused single-pass streaming kernel.
 * Results are bit-identical. */
int vk_set_blur_path(int path);

/* (x, y) kernel of the split path: 0 = whole-plane register-ring kernel
 * (bulk-copy staged plane, thread per row / column; default wherever the
 * plane fits two CTAs per SM), 1 = tiled kernel, 2 = persistent plane kernel
 * (one CTA per SM, two out-of-phase plane groups fed from a work counter).
 * Results are bit-identical. */
int vk_set_xy_kernel(int k);

/* z-pass kernel selection (A/B; results are bit-identical): 0 = TMA-fed
 * four-column kernel (default), 1 = register-fed four columns per thread with
 * packed FFMA2/FADD2 arithmetic, 2 = four columns with scalar sums,
 * 3 = column-pair kernel. */
int vk_set_z_kernel(int k);

/* The tail of the pyramid in one launch (scalespace.py:158-223 for octaves
 * whose levels hold <= 16384 voxels): one CTA per volume runs every level of
 * octaves 0..n_oct-1 of this call in shared memory.  dims_host: 3 per octave;
 * level_ptrs_host / dog_ptrs_host: n_oct*levels batched device pointers
 * (level 0 of the first octave must already be filled; level 0 of the next
 * octaves is written by the handoff subsample); radius_host[i] / taps_host
 * [i*VK_MAX_TAPS ...]: blur of level i (i >= 1). */
int vk_small_octaves(int n_oct, int levels, int handoff, const int* dims_host, float* const* level_ptrs_host,
                     float* const* dog_ptrs_host, const int* radius_host, const float* taps_host, int nb,
                     void* stream);

/* subsample_half (scalespace.py:95-109): floor dims, ordered 8-sum, /8. */
int vk_subsample_half(const float* src, float* dst, int nb, int nx, int ny, int nz, void* stream);

/* DoG difference a - b over n elements (scalespace.py:219-220). */
int vk_difference(const float* a, const float* b, float* out, long long n, void* stream);

/* ------------------------------------------------------------- detection */
/* sum_of_signs_map (detect.py:48-79): int16 80-neighbour map, border 0. */
int vk_sum_of_signs(const float* prev, const float* cur, const float* next, int16_t* out,
                    int nb, int nx, int ny, int nz, void* stream);

/* extract_extrema over every interior DoG level of one octave
 * (detect.py:82-140, 149-178).  dogs: ndog device pointers (host array) to
 * batched DoG levels of one octave.  Appends candidate keys
 *   key = seg << 52 | z << 35 | y << 18 | x << 1 | valley,  seg = seg_base + level
 * to cand_keys[b*cap ...] and bumps cand_count[b].  contrast_min is compared
 * in float32 (numpy NEP 50 semantics of detect.py:104). */
int vk_detect_octave(const float* const* dogs_host, int ndog, int nb, int nx, int ny, int nz,
                     int seg_base, int band, float contrast_min,
                     unsigned long long* cand_keys, int* cand_count, int cap, void* stream);

/* Candidates from a precomputed int16 sum-of-signs map of one DoG level
 * (extract_extrema with a caller-supplied map, detect.py:82-140). */
int vk_extrema_from_map(const int16_t* map, const float* dog_cur, int nx, int ny, int nz, int seg, int band,
                        float contrast_min, unsigned long long* cand_keys, int* cand_count, int cap, void* stream);

/* Order candidates (detect.py:179-181: octave, level, z, y, x) and emit the
 * keypoint records of the whole batch, volume-major (total[0] = count,
 * total[1] = 1 if a volume overflowed `cap`).  seg_info_host: per
 * segment {octave, level, level_table_index, ball_index}; dog_levels: device
 * vk_level table indexed like seg (for dog_value).  Writes kps[0..total),
 * pos[3*i], sigma[i], dog[i], sign[i] (+1 peak, -1 valley), vol_offset[b]
 * and total[0].  seg_sigma_host: keypoint sigma per segment (detect.py:110,143-146).
 * The candidate keys are reordered in place (sorted runs of 2048). */
int vk_order_keypoints(unsigned long long* cand_keys, const int* cand_count, int nb, int cap,
                       const int* seg_info_host, const double* seg_sigma_host, int nseg,
                       const vk_level* dog_levels, vk_kp* kps, double* pos, double* sigma, float* dog,
                       int8_t* sign, int* vol_offset, int* total, int kp_cap, void* stream);

/* Bytes of device scratch vk_orient / vk_describe_siftrank need on `device`:
 * one fp64 histogram slot per CTA of their persistent grids, which the fast
 * paths reduce votes into (fp64 RED, L2-resident).  -1 if no such device. */
long long vk_accum_work_bytes(int device);

/* ----------------------------------------------------------- orientation */
/* gradient_histogram + dominant_orientations (orient.py:89-168) for n_kp
 * keypoints (n_kp_dev: device count, read by the kernel; n_kp_max bounds it).
 * dirs: K x 3 fp64 directions; pair_ok: K x K uint8 (norm of projection > 1e-6,
 * orient.py:157-161).  Outputs: weights (n x K fp64, nullable), nframes[n],
 * prim/sec[n*max_frames].  status[1] counts exact-order fallbacks.  status[0] |= 1 when a keypoint's neighbourhood lies
 * outside its volume (DataError, orient.py:109-110).  ico_host (nullable, K==42
 * only): int[132] = 12 icosahedron-vertex indices into dirs, 12x5 indices of
 * the edge midpoints around each vertex, and the same 12x5 midpoints ordered
 * by neighbour kind (tables.icosphere_structure), enabling the screened and
 * the fast argmax.  ico_lut (nullable, device, with ico_host): uint8[128*128 +
 * 42*24] exact-argmax lookup table (tables.icosphere_lut), tried first.
 * exact_only != 0 forces the reference accumulation order and the brute-force
 * argmax for every keypoint (weights then bit-identical to the reference).
 * grads (nullable, indexed like levels): precomputed gradient volumes
 * (vk_gradient_volume); levels without one use direct gathers.
 * work: vk_accum_work_bytes() of device scratch owned by this call while it
 * runs (one per concurrently running stream). */
int vk_orient(const vk_kp* kps, const int* n_kp_dev, int n_kp_max, const vk_level* levels,
              const vk_ball* balls, const int* ball_offsets, const double* windows,
              const float* windows32, const double* dirs, int K, const uint8_t* pair_ok,
              double secondary_ratio, int max_frames,
              double* weights, int* nframes, int* prim, int* sec, int* status,
              int exact_only, const int* ico_host, const uint8_t* ico_lut, const vk_gradlevel* grads,
              double* work, void* stream);

/* dominant_orientations (orient.py:128-168) on n caller-supplied K-bin
 * weight vectors (exact comparisons). */
int vk_frames_from_weights(const double* weights, int n, int K, const uint8_t* pair_ok, double secondary_ratio,
                           int max_frames, int* nframes, int* prim, int* sec, void* stream);

/* Dense gradient volume of a batched level for the orientation / SIFT-Rank
 * fast paths (volume.py:244-264 gradients, orient.py:123 nearest direction
 * with the default icosphere; ico_host as in vk_orient). */
/* Orientation field of a batched level (nb x nz x ny x nx, x fastest): mag[v]
 * = fp32 |g| of the fp32 central-difference gradient (the orientation fast
 * path's vote before the window), bin[v] = exact nearest of the 42 icosphere
 * directions (np.argmax semantics) or 255 for g == 0.  ico_lut nullable.
 * vk_orient walks it when the level's vk_gradlevel has kind 1. */
int vk_orient_field(const float* level, float* mag, uint8_t* bin, int nb, int nx, int ny, int nz, const double* dirs,
                    const int* ico_host, const uint8_t* ico_lut, void* stream);
int vk_gradient_volume(const float* level, void* g4, uint8_t* bin, int nb, int nx, int ny, int nz,
                       const double* dirs, const int* ico_host, void* stream);

/* Expand per-keypoint frames into the ordered frame list (pipeline.py:55-67:
 * keypoints with zero frames are dropped).  rot_table: K*K*9 fp64 rotations
 * (column-stacked axes, orient.py:164-165).  Writes frames[], rot[9*j],
 * n_frames_dev[0], dropped_dev[0].  scratch: n_kp_max ints (device). */
int vk_expand_frames(const int* nframes, const int* prim, const int* sec, const int* n_kp_dev,
                     int n_kp_max, int max_frames, const double* rot_table, int K,
                     vk_frame* frames, double* rot, int* n_frames_dev, int* dropped_dev,
                     int frame_cap, int* scratch, void* stream);

/* ------------------------------------------------------------ descriptors */
/* sift_rank_descriptor (descriptor.py:227-263): 64 stable ranks (uint8) per
 * frame.  Work item i = one keypoint and its item_count[i] frames starting at
 * frame item_first[i] (frames of an item share a keypoint; the pipeline uses
 * one item per keypoint so gradients are computed once for all its frames,
 * the stage API one item per frame).  rot: 9 fp64 per frame (row-major 3x3).
 * max_f bounds item_count.  stats (nullable): stats[0] counts frames that fell
 * back to the exact accumulation order.  exact_only forces that order.
 * work: as for vk_orient. */
int vk_describe_siftrank(const vk_frame* frames, const double* rot, const int* item_first,
                         const int* item_count, const int* n_items_dev, int n_items_max, int max_f,
                         const vk_kp* kps, const vk_level* levels, const vk_ball* balls,
                         const int* ball_offsets, uint8_t* ranks_out,
                         int exact_only, int* stats, const vk_gradlevel* grads, double* work, void* stream);

/* extract_patch + preblur_patch + brief/rrief (descriptor.py:96-111,
 * 196-224).  kind 1 = BRIEF (packed big-endian bits, ceil(n/8) bytes per
 * frame, descriptor.py:309-316), kind 2 = RRIEF (n stable ranks, uint16).
 * sources: level table of the unblurred source volumes (one entry, batch
 * strided); pos/sigma: keypoint position (base coords) and sigma.
 * grid_host: side linspace values; taps_host: pre-blur taps (radius 0 = off);
 * pts: device, 2*n*3 fp64 pair sample points already mapped to patch
 * index space (descriptor.py:205-212). */
int vk_describe_patch(int kind, const vk_frame* frames, const double* rot, const int* n_frames_dev,
                      int n_frames_max, const vk_kp* kps, const double* pos, const double* sigma,
                      const vk_level* source, int side, const double* grid_host,
                      const float* taps_host, int radius, const double* pts, int npairs,
                      uint8_t* bits_out, uint16_t* ranks_out, void* stream);
/* extract_patch (descriptor.py:96-111), optionally followed by preblur_patch
 * (descriptor.py:196-202) when radius > 0: the side^3 reoriented fp32 patch of
 * each frame, [x][y][z] (z fastest) like Patch.data, into patch_out
 * (n_frames x side^3, device).  Same arguments as vk_describe_patch. */
int vk_extract_patches(const vk_frame* frames, const double* rot, const int* n_frames_dev, int n_frames_max,
                       const vk_kp* kps, const double* pos, const double* sigma, const vk_level* source, int side,
                       const double* grid_host, const float* taps_host, int radius, float* patch_out, void* stream);

/* --------------------------------------------------------------- matching */
/* nearest_neighbor_matches (match.py:81-121).  metric 0 = hamming on packed
 * bytes (nbytes per row), 1 = euclidean on int8 rows (dim bytes per row;
 * rows of 32/64/96/128 bytes at 16-byte aligned addresses run on the tensor
 * cores, tcgen05.mma kind::i8 with s32 accumulators; other widths on a dp4a
 * kernel), 2 = euclidean on fp64 rows.  Outputs per query: best index, d1, d2
 * (fp64), keep (d1 <= ratio_max * d2). */
int vk_match(int metric, const void* a, int na, const void* b, int nb_rows, int dim,
             double ratio_max, int* best, double* d1, double* d2, uint8_t* keep, void* stream);

/* Database matching (SURVEY.md §8(d) configs[4]): as vk_match against the
 * reference rows with [ex_lo, ex_hi) removed (the query subject's own rows);
 * reported indices are into the remaining rows (concat of the other subjects). */
int vk_match_excluding(int metric, const void* a, int na, const void* b, int nb_rows, int dim,
                       double ratio_max, int ex_lo, int ex_hi, int* best, double* d1, double* d2,
                       uint8_t* keep, void* stream);

/* Database matching in one launch (tensor cores): int8 rank rows of
 * dim = 32/64/96/128 bytes; query row i excludes the reference rows
 * [row_ex[2i], row_ex[2i+1]) (device array) and reports compacted indices.
 * Each query's remaining reference set must hold >= 2 rows. */
int vk_match_rows_excluding(const void* a, int na, const void* b, int nb_rows, int dim, double ratio_max,
                            const int* row_ex, int* best, double* d1, double* d2, uint8_t* keep, void* stream);

/* ------------------------------------------------------ point evaluations */
/* gradients_at (volume.py:244-264): fp64 central / one-sided differences at
 * n integer voxels idx[3i..3i+2] = (x, y, z) of an x-fastest fp32 volume
 * (device pointers); out[3i..3i+2]. */
int vk_gradients_at(const float* data, int nx, int ny, int nz, const long long* idx, long long n, double* out,
                    void* stream);
/* sample_trilinear_array (volume.py:203-236): clamped trilinear interpolation
 * in fp64 at n points pts[3i..3i+2] (index units); out[i]. */
int vk_sample_trilinear(const float* data, int nx, int ny, int nz, const double* pts, long long n, double* out,
                        void* stream);

/* ------------------------------------------------------------- key files */
/* Host-side formatter of keyfiles.py:35-122 text lines (no device work):
 * "x y z sigma octave level dog_value sign" (+ 9 row-major rotation reals when
 * rot != NULL) (+ payload: kind 1 = payload_len decimal ranks per record,
 * kind 2 = payload_len packed bytes as lowercase hex), reals as "%.9g".
 * Writes at most cap bytes into out and returns the bytes the n records need
 * (call again with a larger buffer if that exceeds cap); -1 on bad arguments. */
long long vk_format_records(long long n, const double* pos, const double* sigma, const int* octave,
                            const int* level, const double* dog, const signed char* sign, const double* rot,
                            const unsigned char* payload, int payload_kind, int payload_len, char* out,
                            long long cap);

/* Select the int8 euclidean kernel: 0 = tensor cores where the shape allows
 * (default), 1 = dp4a everywhere (cross-checks and benchmarks). */
int vk_set_match_path(int path);

/* Select the tensor-core kernel of the int8 euclidean path: 0 = warp-
 * specialised persistent kernel (TMA reference tiles, N = 256, two TMEM
 * accumulators; default), 1 = the barrier-synchronised N = 128 kernel (A/B). */
int vk_set_match_tc_kernel(int kernel);

/* Optional sub-voxel / sub-level refinement (an extension: volkey reports
 * lattice positions): one Newton step of the DoG's quadratic
 * model in (x, y, z, level) from central differences over the 3x3x3x3
 * neighbourhood of each keypoint, fp64, fixed operation order.  out[6 * k]:
 * refined x, y, z (input-volume coordinates), sigma * kappa^d_level,
 * D + g.d / 2, status (0 converged, 1 |d_i| > 0.5, 2 singular Hessian).
 * dog_levels: the DoG level table (index octave * levels_per_octave + level). */
int vk_refine_keypoints(const vk_kp* kps, const int* n_kp_dev, int n_kp_max, const vk_level* dog_levels,
                        int levels_per_octave, double kappa, const double* sigma, double* out, void* stream);

/* ------------------------------------- fused orientation + SIFT-Rank */
/* assign_orientations + sift_rank_descriptor (pipeline.py:41-67,
 * orient.py:89-168, descriptor.py:227-263) in one kernel: per keypoint, the
 * ball's stencil set is staged once in shared memory (sph_* tables from
 * tables.sphere_tables: per ball (rows start, n_rows, compact floats, entries
 * start), rows (dy, dz, m, start), entries (packed offset, c | yh << 16,
 * yl | zh << 16, zl)), both walks read it, the frames are decided in between.
 * Writes nframes / prim / sec per keypoint like vk_orient (status[0] bit 1 =
 * DataError, status[1] / status[2] = orientation / SIFT-Rank repair counts)
 * and each frame's 64 ranks at desc_kp[(kp * max_frames + f) * 64].  K must be
 * 42 (icosphere lookup table).  box_cap: staging buffer floats (balls with a
 * larger stencil, or one leaving the volume, are walked from global memory). */
int vk_orient_siftrank(const vk_kp* kps, const int* n_kp_dev, int n_kp_max, const vk_level* levels,
                       const vk_ball* balls, const int* ball_offsets, const double* windows, const float* windows32,
                       const double* dirs, int K, const uint8_t* pair_ok, double secondary_ratio, int max_frames,
                       const double* rot_table, int* nframes, int* prim, int* sec, uint8_t* desc_kp, int* status,
                       const int* ico_host, const uint8_t* ico_lut, const int* sph_ball, const int* sph_rows,
                       const int* sph_ent, int box_cap, double* work, void* stream);
/* rows[o] = rows_kp[frames[o].kp * max_frames + (o - frame_first[frames[o].kp])]
 * (64-byte rows) for the n_frames (<= frame_cap) frames of vk_expand_frames. */
int vk_scatter_frame_rows(const vk_frame* frames, const int* frame_first, const int* n_frames_dev, int frame_cap,
                          int max_frames, const uint8_t* rows_kp, uint8_t* rows, void* stream);

/* ------------------------------------------------------ Hough consensus */
/* Host-side (CPU, native C++) 7-DOF Hough consensus; replaces the scalar
 * Python of hough_consensus (match.py:227-348) with vote_transform
 * (match.py:124-133), _rotation_bins (match.py:184-207), _agrees
 * (match.py:210-224) and similarity_from_correspondences (match.py:136-162).
 * vk_hough_init binds the ILP64 OpenBLAS numpy links (scipy-openblas64
 * symbol names), so every BLAS / LAPACK step is the call numpy makes.
 * vk_hough_dots: directions @ (R @ ex) per match (match.py:191-192); the
 * host takes np.argsort(-dots)[:, :2] (the reference's own unstable sort
 * decides exact ties) and passes it as `near` to vk_hough_consensus.
 * Returns 0, 5 (bad arguments), 6 (no cell reaches min_votes; *cell_votes =
 * the densest count) or 9 (not initialised). */
int vk_hough_init(const char* blas_path);
int vk_hough_dots(int n, const double* rot_a, const double* rot_b, const double* dirs, int K, double* dots);
int vk_hough_consensus(int n, const int64_t* index_a, const int64_t* index_b, const double* sigma_a,
                       const double* sigma_b, const double* rot_a, const double* rot_b, const double* pos_a,
                       const double* pos_b, const int64_t* near, const double* b1, const double* b2, int K,
                       const double* settings /* log_scale_bin, trans_bin, log_scale_tol, rot_tol_deg, trans_tol */,
                       int min_votes, int64_t* inliers, int* n_inliers, int* cell_votes, double* scale,
                       double* rotation, double* translation);

#ifdef __cplusplus
}
#endif
#endif /* VOLKEY_B200_H */
