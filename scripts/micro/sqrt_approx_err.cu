// Exhaustive error of the hardware sqrt.approx.f32 (MUFU.SQRT) on sm_100a:
// every positive finite fp32 bit pattern 0x00000001 .. 0x7F7FFFFF (all
// binades incl. subnormals), against the correctly rounded fp64 sqrt.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 sqrt_approx_err.cu -o /tmp/sq && /tmp/sq
// Result recorded next to norm3_f32 (paper_2112_10258_b200/csrc/vk_common.cuh).
#include <cstdio>
#include <cmath>
#include <cstdint>

__global__ void k(double* maxrel, unsigned* argmax, unsigned long long* nonzero_out, unsigned lo, unsigned hi) {
    double m = 0.0;
    unsigned am = 0;
    unsigned long long bad0 = 0;
    for (unsigned long long i = (unsigned long long)lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const float x = __uint_as_float((unsigned)i);
        float r;
        asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
        const double e = sqrt((double)x);
        if (!(r > 0.f)) ++bad0;  // a positive input must give a positive root
        const double rel = fabs((double)r - e) / e;
        if (rel > m) { m = rel; am = (unsigned)i; }
    }
    // per-thread max -> global (bit patterns of positive doubles order like the values)
    unsigned long long mb = __double_as_longlong(m);
    unsigned long long old = atomicMax((unsigned long long*)maxrel, mb);
    if (mb > old) atomicExch(argmax, am);
    if (bad0) atomicAdd(nonzero_out, bad0);
}

int main() {
    double* d;
    unsigned* a;
    unsigned long long* z;
    cudaMalloc(&d, 8);
    cudaMalloc(&a, 4);
    cudaMalloc(&z, 8);
    cudaMemset(d, 0, 8);
    cudaMemset(a, 0, 4);
    cudaMemset(z, 0, 8);
    const unsigned last = 0x7F7FFFFFu;  // largest finite
    for (unsigned long long lo = 1; lo <= last; lo += (1ull << 28)) {
        unsigned long long hi = lo + (1ull << 28);
        if (hi > (unsigned long long)last + 1) hi = (unsigned long long)last + 1;
        k<<<148 * 16, 256>>>(d, a, z, (unsigned)lo, (unsigned)hi);
    }
    double h;
    unsigned am;
    unsigned long long nz;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&am, a, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&nz, z, 8, cudaMemcpyDeviceToHost);
    printf("sqrt.approx.f32 exhaustive over %u positive finite inputs: max rel err = %.4e (= %.3f x 2^-24) at "
           "bits 0x%08x (x = %.9g); non-positive results: %llu\n",
           last, h, h / 5.9604644775390625e-8, am, (double)__builtin_bit_cast(float, am), nz);
    return 0;
}
