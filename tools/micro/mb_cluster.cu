// Microbenchmarks for the cluster-resident brick solver design (sm_100a):
//  1) max active clusters for cluster sizes 8/16 at ~208 KB smem, 512 threads
//  2) TMEM tcgen05.ld / tcgen05.st throughput (32x32b.x32) with 16 warps
//  3) cluster barrier round trip
//  4) DSMEM bulk copy smem->remote smem throughput (cp.async.bulk.shared::cluster)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_tmem(int iters, float* out, long long* cyc) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr_s;
  const uint32_t ta = base + ((uint32_t)(32 * (warp & 3)) << 16) + 128 * (warp >> 2);
  uint32_t v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(1.0f + threadIdx.x + i);
  // store 128 cols
  for (int c = 0; c < 128; c += 32)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      :: "r"(ta + c), "r"(v[0]),"r"(v[1]),"r"(v[2]),"r"(v[3]),"r"(v[4]),"r"(v[5]),"r"(v[6]),"r"(v[7]),"r"(v[8]),"r"(v[9]),"r"(v[10]),"r"(v[11]),"r"(v[12]),"r"(v[13]),"r"(v[14]),"r"(v[15]),"r"(v[16]),"r"(v[17]),"r"(v[18]),"r"(v[19]),"r"(v[20]),"r"(v[21]),"r"(v[22]),"r"(v[23]),"r"(v[24]),"r"(v[25]),"r"(v[26]),"r"(v[27]),"r"(v[28]),"r"(v[29]),"r"(v[30]),"r"(v[31]));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  __syncthreads();
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int c = 0; c < 128; c += 32) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])
        : "r"(ta + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += __uint_as_float(v[i]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  long long t2 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int c = 0; c < 128; c += 32)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
        :: "r"(ta + c), "r"(v[0]),"r"(v[1]),"r"(v[2]),"r"(v[3]),"r"(v[4]),"r"(v[5]),"r"(v[6]),"r"(v[7]),"r"(v[8]),"r"(v[9]),"r"(v[10]),"r"(v[11]),"r"(v[12]),"r"(v[13]),"r"(v[14]),"r"(v[15]),"r"(v[16]),"r"(v[17]),"r"(v[18]),"r"(v[19]),"r"(v[20]),"r"(v[21]),"r"(v[22]),"r"(v[23]),"r"(v[24]),"r"(v[25]),"r"(v[26]),"r"(v[27]),"r"(v[28]),"r"(v[29]),"r"(v[30]),"r"(v[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  __syncthreads();
  long long t3 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) { cyc[2 * blockIdx.x] = t1 - t0; cyc[2 * blockIdx.x + 1] = t3 - t2; }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(base));
}

// smem LDS.128 throughput for comparison (512 threads, 64 KB)
__global__ void k_lds(int iters, float* out, long long* cyc) {
  extern __shared__ float4 sm4[];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm4[i] = make_float4(i, 1, 2, 3);
  __syncthreads();
  float4 a = make_float4(0, 0, 0, 0);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int j = 0; j < 8; ++j) {
      float4 v = sm4[(threadIdx.x + j * 512 + it) & 4095];
      a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a.x + a.y + a.z + a.w;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_cbar(int iters, long long* cyc) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;");
    asm volatile("barrier.cluster.wait.acquire.aligned;");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// each CTA bulk-copies 2 x 16 KB of its smem into its +1 / -1 cluster neighbours per round
__global__ void k_dsmem(int iters, long long* cyc) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank(), cs = cl.num_blocks();
  unsigned char* src = sm;            // 32 KB source
  unsigned char* dst = sm + 32768;    // 2 x 16 KB halo
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) src[i] = (unsigned char)i;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  cl.sync();
  const int nin = (rank > 0) + (rank + 1 < cs);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar)), "r"(nin * 16384));
      for (int s = 0; s < 2; ++s) {
        const int peer = s ? rank + 1 : (int)rank - 1;
        if (peer < 0 || peer >= (int)cs) continue;
        uint32_t rdst, rbar;
        const uint32_t ldst = smem_u32(dst + (s ? 0 : 16384));   // my +1 neighbour stores into its slot 0
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(ldst), "r"(peer));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(&bar)), "r"(peer));
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(rdst), "r"(smem_u32(src + s * 16384)), "r"(16384), "r"(rbar) : "memory");
      }
    }
    // wait own barrier phase it&1
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(smem_u32(&bar)), "r"(it & 1));
    }
    asm volatile("barrier.cluster.arrive.release.aligned;");
    asm volatile("barrier.cluster.wait.acquire.aligned;");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  printf("device %s SMs %d smemOptin %zu\n", pr.name, pr.multiProcessorCount, pr.sharedMemPerBlockOptin);
  long long* dcyc; float* dout;
  CK(cudaMalloc(&dcyc, 4096 * sizeof(long long))); CK(cudaMalloc(&dout, 148 * 1024 * sizeof(float)));
  long long hc[4096];
  // 1) occupancy
  CK(cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  for (int smem_kb : {100, 160, 208, 220}) {
    CK(cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024));
    for (int cs : {2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * 8); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = smem_kb * 1024;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int nc = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, k_dsmem, &cfg);
      printf("occupancy smem %d KB cluster %2d: max active clusters %d (%s) -> %d CTAs\n", smem_kb, cs, nc, cudaGetErrorString(e), nc * cs);
    }
  }
  // 2) TMEM throughput: one CTA per SM
  const int it = 2000;
  k_tmem<<<148, 512>>>(it, dout, dcyc); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(hc, dcyc, 2 * 148 * sizeof(long long), cudaMemcpyDeviceToHost));
  double bytes = (double)it * 128 * 4 * 512;
  printf("TMEM ld: %.1f cyc per 256KB sweep -> %.1f B/cyc/SM; st: %.1f B/cyc/SM\n", (double)hc[0] / it, bytes / hc[0], bytes / hc[1]);
  CK(cudaFuncSetAttribute(k_lds, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  k_lds<<<148, 512, 65536>>>(it, dout, dcyc); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(hc, dcyc, 148 * sizeof(long long), cudaMemcpyDeviceToHost));
  printf("LDS.128: %.1f B/cyc/SM\n", (double)it * 8 * 16 * 512 / hc[0]);
  // 3) cluster barrier
  CK(cudaFuncSetAttribute(k_cbar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  for (int cs : {4, 8, 16}) {
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(cs * (cs == 16 ? 8 : 16)); cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_cbar, 1000, dcyc)); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hc, dcyc, sizeof(long long), cudaMemcpyDeviceToHost));
    printf("cluster %d barrier: %.1f cyc\n", cs, hc[0] / 1000.0);
  }
  // 4) DSMEM bulk halo exchange 2 x 16 KB + barrier
  for (int cs : {8, 16}) {
    CK(cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(cs * (cs == 16 ? 8 : 16)); cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = 65536;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_dsmem, 1000, dcyc)); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hc, dcyc, 2 * sizeof(long long), cudaMemcpyDeviceToHost));
    printf("cluster %d DSMEM 2x16KB exchange + barrier: %.1f cyc/round (rank1: %.1f)\n", cs, hc[0] / 1000.0, hc[1] / 1000.0);
  }
  printf("done\n");
  return 0;
}
