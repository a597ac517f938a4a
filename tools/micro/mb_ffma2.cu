// Microbenchmark: issue rate of FFMA / FADD vs the packed FFMA2 / FADD2 (fma.rn.f32x2,
// add.rn.f32x2, sm_100a) per SMSP.  16 independent accumulator chains per thread.
#include <cstdio>
#include <cstdint>
#define N_IT 4096
__global__ void k_ffma(float* out, float a, float b) {
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x + i;
  long long t0 = clock64();
  for (int it = 0; it < N_IT; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(acc[i]) : "f"(a), "f"(b));
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}
__global__ void k_ffma2(float* out, float a, float b) {
  unsigned long long acc[8];
  unsigned long long A, B;
  { float2 fa = make_float2(a, a), fb = make_float2(b, b);
    A = *reinterpret_cast<unsigned long long*>(&fa); B = *reinterpret_cast<unsigned long long*>(&fb); }
#pragma unroll
  for (int i = 0; i < 8; ++i) { float2 v = make_float2(threadIdx.x + i, i); acc[i] = *reinterpret_cast<unsigned long long*>(&v); }
  long long t0 = clock64();
  for (int it = 0; it < N_IT; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[i]) : "l"(A), "l"(B));
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) { float2 v = *reinterpret_cast<float2*>(&acc[i]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}
__global__ void k_fadd(float* out, float a, float b) {
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x + i;
  long long t0 = clock64();
  for (int it = 0; it < N_IT; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(acc[i]) : "f"(a));
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}
__global__ void k_fadd2(float* out, float a, float b) {
  unsigned long long acc[8];
  unsigned long long A;
  { float2 fa = make_float2(a, a); A = *reinterpret_cast<unsigned long long*>(&fa); }
#pragma unroll
  for (int i = 0; i < 8; ++i) { float2 v = make_float2(threadIdx.x + i, i); acc[i] = *reinterpret_cast<unsigned long long*>(&v); }
  long long t0 = clock64();
  for (int it = 0; it < N_IT; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(acc[i]) : "l"(A));
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) { float2 v = *reinterpret_cast<float2*>(&acc[i]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}
// mixed: FFMA2 interleaved with LDS-free IMAD-free FADD (scalar) to see co-issue
__global__ void k_mix(float* out, float a, float b) {
  unsigned long long acc[8]; float sc[8];
  unsigned long long A, B;
  { float2 fa = make_float2(a, a), fb = make_float2(b, b);
    A = *reinterpret_cast<unsigned long long*>(&fa); B = *reinterpret_cast<unsigned long long*>(&fb); }
#pragma unroll
  for (int i = 0; i < 8; ++i) { float2 v = make_float2(threadIdx.x + i, i); acc[i] = *reinterpret_cast<unsigned long long*>(&v); sc[i] = i; }
  long long t0 = clock64();
  for (int it = 0; it < N_IT; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[i]) : "l"(A), "l"(B));
      asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(sc[i]) : "f"(a));
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) { float2 v = *reinterpret_cast<float2*>(&acc[i]); s += v.x + v.y + sc[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}
int main() {
  float* d; cudaMalloc(&d, 148 * 1024 * 4 * 4);
  float h;
  const char* names[5] = {"ffma", "ffma2", "fadd", "fadd2", "ffma2+fadd"};
  void (*ks[5])(float*, float, float) = {k_ffma, k_ffma2, k_fadd, k_fadd2, k_mix};
  const int per_thread[5] = {16, 8, 16, 8, 16};
  for (int w : {4, 8, 16, 32}) {
    for (int i = 0; i < 5; ++i) {
      ks[i]<<<148, 32 * w>>>(d, 1.0001f, 0.5f);
      ks[i]<<<148, 32 * w>>>(d, 1.0001f, 0.5f);
      cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
      // warp-instructions issued per SMSP per cycle
      const double wi = (double)per_thread[i] * N_IT * (w / 4.0);
      printf("warps/SM %2d %-11s cycles %9.0f  warp-instr/clk/SMSP %.3f\n", w, names[i], h, wi / h);
    }
  }
  return 0;
}
