// Microbenchmark: issue throughput of the fp32 instruction forms the blur uses
// (FADD, FMUL, FMUL2 reg x uniform, FADD2, FFMA, mixed FADD+FMUL2) on one B200.
#include <cstdio>
#include <cuda_runtime.h>
#define N 8
#define ITERS 4096
__global__ void k_fadd(float* out, float w) {
  float a[N]; for (int i = 0; i < N; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < N; ++i) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(w));
  float s = 0; for (int i = 0; i < N; ++i) s += a[i]; if (s == 1.2345f) out[0] = s;
}
__global__ void k_fmul(float* out, float w) {
  float a[N]; for (int i = 0; i < N; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < N; ++i) asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(w));
  float s = 0; for (int i = 0; i < N; ++i) s += a[i]; if (s == 1.2345f) out[0] = s;
}
__global__ void k_ffma(float* out, float w) {
  float a[N]; float b = threadIdx.x; for (int i = 0; i < N; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < N; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(w), "f"(b));
  float s = 0; for (int i = 0; i < N; ++i) s += a[i]; if (s == 1.2345f) out[0] = s;
}
__global__ void k_fmul2(float* out, float w) {
  unsigned long long a[N]; for (int i = 0; i < N; ++i) { float2 f = make_float2(threadIdx.x, i); a[i] = *(unsigned long long*)&f; }
  float2 ww = make_float2(w, w); unsigned long long wb = *(unsigned long long*)&ww;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < N; ++i) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(wb));
  unsigned long long s = 0; for (int i = 0; i < N; ++i) s ^= a[i]; if (s == 12345) out[0] = 1;
}
__global__ void k_fadd2(float* out, float w) {
  unsigned long long a[N]; for (int i = 0; i < N; ++i) { float2 f = make_float2(threadIdx.x, i); a[i] = *(unsigned long long*)&f; }
  float2 ww = make_float2(w, w); unsigned long long wb = *(unsigned long long*)&ww;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < N; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(wb));
  unsigned long long s = 0; for (int i = 0; i < N; ++i) s ^= a[i]; if (s == 12345) out[0] = 1;
}
__global__ void k_ffma2(float* out, float w) {
  unsigned long long a[N]; for (int i = 0; i < N; ++i) { float2 f = make_float2(threadIdx.x, i); a[i] = *(unsigned long long*)&f; }
  float2 ww = make_float2(w, w); unsigned long long wb = *(unsigned long long*)&ww;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < N; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(a[i]) : "l"(wb));
  unsigned long long s = 0; for (int i = 0; i < N; ++i) s ^= a[i]; if (s == 12345) out[0] = 1;
}
// mixed: per element one mul.f32x2 (tap product pair) + two scalar adds (the blur's inner step)
__global__ void k_mix(float* out, float w) {
  unsigned long long p[N/2]; float a[N];
  for (int i = 0; i < N; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int i = 0; i < N/2; ++i) { float2 f = make_float2(threadIdx.x, i); p[i] = *(unsigned long long*)&f; }
  float2 ww = make_float2(w, w); unsigned long long wb = *(unsigned long long*)&ww;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < N/2; ++i) {
      unsigned long long q;
      asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(q) : "l"(p[i]), "l"(wb));
      float2 f = *(float2*)&q;
      asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[2*i]) : "f"(f.x));
      asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[2*i+1]) : "f"(f.y));
    }
  float s = 0; for (int i = 0; i < N; ++i) s += a[i]; if (s == 1.2345f) out[0] = s;
}
// mixed 2: mul.f32x2 + add.f32x2 (packed adds) -- can ptxas fuse with explicit .rn?
__global__ void k_mix2(float* out, float w) {
  unsigned long long p[N/2], a[N/2];
  for (int i = 0; i < N/2; ++i) { float2 f = make_float2(threadIdx.x, i); p[i] = *(unsigned long long*)&f; a[i] = p[i]; }
  float2 ww = make_float2(w, w); unsigned long long wb = *(unsigned long long*)&ww;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < N/2; ++i) {
      unsigned long long q;
      asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(q) : "l"(p[i]), "l"(wb));
      asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(q));
    }
  unsigned long long s = 0; for (int i = 0; i < N/2; ++i) s ^= a[i]; if (s == 12345) out[0] = 1;
}

// mixed 3: product via fma(p, w, -0) (== round(p*w)), then packed add
__global__ void k_mix3(float* out, float w) {
  unsigned long long p[N/2], a[N/2];
  for (int i = 0; i < N/2; ++i) { float2 f = make_float2(threadIdx.x, i); p[i] = *(unsigned long long*)&f; a[i] = p[i]; }
  float2 ww = make_float2(w, w); unsigned long long wb = *(unsigned long long*)&ww;
  float2 nz = make_float2(-0.0f, -0.0f); unsigned long long z = *(unsigned long long*)&nz;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < N/2; ++i) {
      unsigned long long q;
      asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(q) : "l"(p[i]), "l"(wb), "l"(z));
      asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(q));
    }
  unsigned long long s = 0; for (int i = 0; i < N/2; ++i) s ^= a[i]; if (s == 12345) out[0] = 1;
}
// mixed 4: product via mul, add via fma(q, 1, acc)
__global__ void k_mix4(float* out, float w) {
  unsigned long long p[N/2], a[N/2];
  for (int i = 0; i < N/2; ++i) { float2 f = make_float2(threadIdx.x, i); p[i] = *(unsigned long long*)&f; a[i] = p[i]; }
  float2 ww = make_float2(w, w); unsigned long long wb = *(unsigned long long*)&ww;
  float2 one = make_float2(1.0f, 1.0f); unsigned long long o = *(unsigned long long*)&one;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < N/2; ++i) {
      unsigned long long q;
      asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(q) : "l"(p[i]), "l"(wb));
      asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a[i]) : "l"(q), "l"(o));
    }
  unsigned long long s = 0; for (int i = 0; i < N/2; ++i) s ^= a[i]; if (s == 12345) out[0] = 1;
}
typedef void (*K)(float*, float);
int main() {
  float* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  struct { const char* name; K k; int instr_per_iter; int lanes_ops; } ks[] = {
    {"FADD", k_fadd, N, 1}, {"FMUL", k_fmul, N, 1}, {"FFMA", k_ffma, N, 1}, {"FMUL2", k_fmul2, N, 2},
    {"FADD2", k_fadd2, N, 2}, {"FFMA2", k_ffma2, N, 2}, {"MUL2+2FADD", k_mix, 3 * N / 2, 0}, {"MUL2+ADD2", k_mix2, N, 0}, {"FMA2z+ADD2", k_mix3, N, 0}, {"MUL2+FMA2one", k_mix4, N, 0}};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (auto& k : ks) {
    for (int threads : {256, 512, 1024}) {
      int blocks = sms * (2048 / threads);
      k.k<<<blocks, threads>>>(d, 1.0001f);
      cudaEventRecord(e0);
      k.k<<<blocks, threads>>>(d, 1.0001f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double warp_instr = (double)blocks * threads / 32 * ITERS * k.instr_per_iter;
      double per_smsp_clk = warp_instr / (sms * 4) / (ms * 1e-3 * clk * 1e3);
      printf("%-12s threads=%4d  %.3f ms  warp-instr/clk/SMSP=%.3f\n", k.name, threads, ms, per_smsp_clk);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
