// Issue-rate microbenchmark on B200: SM-clock-timed (clock64) throughput of
// instruction mixes, 16 warps/SM resident, all chains independent.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 2048
#define CH 8
template <int MODE>
__global__ void kern(float* out, long long* cyc, float w) {
  float a[CH]; unsigned u[CH]; unsigned long long p[CH / 2];
  for (int i = 0; i < CH; ++i) { a[i] = threadIdx.x * 1e-3f + i; u[i] = threadIdx.x + i; }
  for (int i = 0; i < CH / 2; ++i) { float2 f = make_float2(threadIdx.x, i); p[i] = *(unsigned long long*)&f; }
  float2 ww = make_float2(w, w); unsigned long long wb = *(unsigned long long*)&ww;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (MODE == 0) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(w));                     // FADD
      if (MODE == 1) { asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(w));                     // FADD + FMUL
                       asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(a[(i + 4) % CH]) : "f"(w)); }
      if (MODE == 2) { asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(w));                     // FADD + IADD
                       asm volatile("add.u32 %0, %0, %1;" : "+r"(u[i]) : "r"(7)); }
      if (MODE == 3) { asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(w));                     // FADD + MOV-ish (prmt)
                       asm volatile("prmt.b32 %0, %0, %1, 0x3210;" : "+r"(u[i]) : "r"(u[(i+1)%CH])); }
      if (MODE == 4 && (i & 1) == 0) {                                                                   // FMUL2 + 2 FADD
        unsigned long long q;
        asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(q) : "l"(p[i / 2]), "l"(wb));
        float2 f = *(float2*)&q;
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(f.x));
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i + 1]) : "f"(f.y)); }
      if (MODE == 5) asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(w));                     // FMUL
      if (MODE == 6 && (i & 1) == 0) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(p[i / 2]) : "l"(wb)); // FMUL2
      if (MODE == 7) { asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(w));                     // FADD + FMUL2 (1:1)
                       asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(p[i / 2]) : "l"(wb)); }
      if (MODE == 8) { asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(w));                     // FMUL + IADD
                       asm volatile("add.u32 %0, %0, %1;" : "+r"(u[i]) : "r"(7)); }
      if (MODE == 9) asm volatile("add.u32 %0, %0, %1;" : "+r"(u[i]) : "r"(7));                         // IADD
    }
  }
  long long t1 = clock64();
  float s = 0; unsigned us = 0; unsigned long long ps = 0;
  for (int i = 0; i < CH; ++i) { s += a[i]; us ^= u[i]; }
  for (int i = 0; i < CH / 2; ++i) ps ^= p[i];
  if (s == 1.2345f || us == 12345 || ps == 12345) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE> void run(const char* name, int ninstr_per_i, float* d, long long* c, int sms) {
  kern<MODE><<<sms * 2, 256>>>(d, c, 1.0001f);  // 16 warps/SM, 4 per SMSP
  cudaDeviceSynchronize();
  long long h[1024]; cudaMemcpy(h, c, sizeof(long long) * sms * 2, cudaMemcpyDeviceToHost);
  double mx = 0; for (int i = 0; i < sms * 2; ++i) mx = h[i] > mx ? h[i] : mx;
  // warp-instructions issued per SMSP per clock: 4 warps per SMSP
  double wi = 4.0 * ITERS * CH * ninstr_per_i / 2.0;
  printf("%-16s %.3f warp-instr/clk/SMSP  (cycles %.0f)\n", name, wi / mx, mx);
}
int main() {
  float* d; long long* c; cudaMalloc(&d, 4); cudaMalloc(&c, 8 * 1024);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("FADD", 2, d, c, sms);
  run<5>("FMUL", 2, d, c, sms);
  run<9>("IADD", 2, d, c, sms);
  run<6>("FMUL2", 1, d, c, sms);
  run<1>("FADD+FMUL", 4, d, c, sms);
  run<2>("FADD+IADD", 4, d, c, sms);
  run<3>("FADD+PRMT", 4, d, c, sms);
  run<8>("FMUL+IADD", 4, d, c, sms);
  run<4>("FMUL2+2FADD", 3, d, c, sms);
  run<7>("FADD+FMUL2", 4, d, c, sms);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
