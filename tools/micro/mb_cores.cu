// Co-residency probe (sm_100a): how many worker CTAs of a given cluster size fit on the
// SMs that the 64^3 resident kernel's 16-CTA clusters (512 threads, 180 KB smem, one CTA
// per SM) leave free.  Kernel A holds its SMs (spins on a host-mapped stop flag); kernel B
// (cluster size C, 512 threads, S KB smem) is launched on a second stream, each CTA counts
// itself in and spins; after 200 ms the host reads how many B CTAs started, then stops both.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mb_cores mb_cores.cu && ./mb_cores
#include <cstdio>
#include <cstdint>
#include <unistd.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ int smid() { int s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); return s; }

__global__ void k_hold(volatile int* stop, int* cnt, int* sms) {
  extern __shared__ float sm[];
  if (threadIdx.x == 0) {
    sms[blockIdx.x] = smid();
    atomicAdd(cnt, 1);
    while (*stop == 0) __nanosleep(1000);
  }
  __syncthreads();
  if (threadIdx.x == 0 && sm[0] == 12345.f) cnt[1] = 1;
}

__global__ void k_work(volatile int* stop, int* cnt, int* sms) {
  extern __shared__ float sm[];
  if (threadIdx.x == 0) {
    sms[blockIdx.x] = smid();
    atomicAdd(cnt, 1);
    while (*stop == 0) __nanosleep(1000);
  }
  __syncthreads();
  if (threadIdx.x == 0 && sm[0] == 12345.f) cnt[1] = 1;
}

static cudaError_t launch(void (*k)(volatile int*, int*, int*), int grid, int cl, int smem,
                          cudaStream_t s, volatile int* stop, int* cnt, int* sms) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, stop, cnt, sms);
}

int main() {
  CK(cudaFuncSetAttribute(k_hold, cudaFuncAttributeMaxDynamicSharedMemorySize, 180 * 1024));
  CK(cudaFuncSetAttribute(k_hold, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(k_work, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(k_work, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  int *stop_h, *stop_d, *cnt, *sms;
  CK(cudaHostAlloc(&stop_h, 4, cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer(&stop_d, stop_h, 0));
  int* cnt_h;
  CK(cudaHostAlloc(&cnt_h, 16, cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer(&cnt, cnt_h, 0));
  CK(cudaMalloc(&sms, 4096 * 4));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  const int cls[] = {2, 4, 6, 8, 10, 12};
  for (int hold = 0; hold < 2; ++hold) {
    for (int ci = 0; ci < 6; ++ci) {
      const int C = cls[ci];
      *stop_h = 0;
      for (int i = 0; i < 4; ++i) cnt_h[i] = 0;
      CK(cudaDeviceSynchronize());
      int h = 0;
      if (hold) {
        CK(launch(k_hold, 7 * 16, 16, 180 * 1024, s1, stop_d, cnt, sms));
        usleep(100000);
        h = ((volatile int*)cnt_h)[0];
      }
      int* cnt2 = cnt + 2;
      const int grid = (148 / C) * C;
      CK(launch(k_work, grid, C, 100 * 1024, s2, stop_d, cnt2, sms + 1024));
      usleep(200000);
      const int w = ((volatile int*)cnt_h)[2];
      *stop_h = 1;
      CK(cudaDeviceSynchronize());
      printf("{\"hold_16cta_clusters\": %d, \"held_ctas\": %d, \"worker_cluster\": %d, \"worker_ctas_coresident\": %d, \"worker_grid\": %d}\n",
             hold ? 7 : 0, h, C, w, grid);
    }
  }
  return 0;
}
