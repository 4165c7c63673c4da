// vk_sample.cu -- point evaluations on a volume: finite-difference gradients
// at integer voxels (volume.py:244-264, gradients_at) and clamped trilinear
// interpolation at continuous points (volume.py:203-236,
// sample_trilinear_array), one thread per point, with the same fp64
// arithmetic the orientation / descriptor kernels use (vk_common.cuh).
#include "vk_common.cuh"

namespace vk {

__global__ void gradients_at_kernel(const float* __restrict__ data, int nx, int ny, int nz,
                                    const long long* __restrict__ idx, long long n, double* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double gx, gy, gz;
    gradient_at(data, nx, ny, nz, (int)idx[3 * i], (int)idx[3 * i + 1], (int)idx[3 * i + 2], gx, gy, gz);
    out[3 * i] = gx;
    out[3 * i + 1] = gy;
    out[3 * i + 2] = gz;
}

__global__ void trilinear_kernel(const float* __restrict__ data, int nx, int ny, int nz, const double* __restrict__ pts,
                                 long long n, double* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    auto at = [&](int x, int y, int z) {
        return (double)__ldg(data + (((long long)z * ny + y) * nx + x));
    };
    out[i] = trilinear(at, nx, ny, nz, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
}

}  // namespace vk

using namespace vk;

extern "C" int vk_gradients_at(const float* data, int nx, int ny, int nz, const long long* idx, long long n,
                               double* out, void* stream) {
    if (!data || nx < 1 || ny < 1 || nz < 1 || n < 0 || (n && (!idx || !out))) {
        set_error("vk_gradients_at: bad arguments");
        return VK_ERR_PARAMETER;
    }
    if (n == 0) return VK_OK;
    gradients_at_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(data, nx, ny, nz, idx, n, out);
    count_launch();
    return cuda_status(cudaGetLastError(), "gradients_at launch");
}

extern "C" int vk_sample_trilinear(const float* data, int nx, int ny, int nz, const double* pts, long long n,
                                   double* out, void* stream) {
    if (!data || nx < 1 || ny < 1 || nz < 1 || n < 0 || (n && (!pts || !out))) {
        set_error("vk_sample_trilinear: bad arguments");
        return VK_ERR_PARAMETER;
    }
    if (n == 0) return VK_OK;
    trilinear_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(data, nx, ny, nz, pts, n, out);
    count_launch();
    return cuda_status(cudaGetLastError(), "trilinear launch");
}
