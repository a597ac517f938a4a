// Microbenchmark: cluster-wide reduction round trip patterns on a 16-CTA cluster, 512 thr.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ uint32_t sptr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ int cl_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" :: "r"(sptr(bar)), "r"(ph) : "memory");
}
__device__ __forceinline__ void expect(uint64_t* bar, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sptr(bar)), "r"(b) : "memory"); }
__device__ __forceinline__ void sta64(uint32_t a, double v, uint32_t bar) { asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" :: "r"(a), "l"(__double_as_longlong(v)), "r"(bar) : "memory"); }
__device__ __forceinline__ void sta32(uint32_t a, float v, uint32_t bar) { asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" :: "r"(a), "r"(__float_as_uint(v)), "r"(bar) : "memory"); }
__device__ __forceinline__ void sta4(uint32_t a, float4 v, uint32_t bar) { asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1,%2,%3,%4}, [%5];" :: "r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(bar) : "memory"); }

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(int iters, long long* cyc, double* out) {
  extern __shared__ __align__(16) float sm[];
  __shared__ __align__(8) uint64_t bar[3];
  __shared__ double slots[2][16];
  __shared__ float wslots[2][256];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, rank = cl_rank();
  if (t == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sptr(&bar[0]))); asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sptr(&bar[1]))); asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sptr(&bar[2]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  for (int i = t; i < 16384; i += 512) sm[i] = 1.f;
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  uint32_t ph = 0, phs[2] = {0, 0};
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int b = it & 1;
    if (MODE == 0) {          // thread 0 sends 16 x f64, all threads wait, all sum 16
      if (t == 0) { expect(&bar[b], 16 * 8); for (int c = 0; c < 16; ++c) sta64(mapa(sptr(&slots[b][rank]), c), 1.0 + it, mapa(sptr(&bar[b]), c)); }
      mbar_wait(&bar[b], phs[b]); phs[b] ^= 1;
      double s = 0; for (int c = 0; c < 16; ++c) s += slots[b][c]; acc += s;
    } else if (MODE == 1) {   // lanes 0..15 of warp 0 send, warp 0 waits, bar.sync
      if (warp == 0) {
        if (lane == 0) expect(&bar[b], 16 * 8);
        if (lane < 16) sta64(mapa(sptr(&slots[b][rank]), lane), 1.0 + it, mapa(sptr(&bar[b]), lane));
        mbar_wait(&bar[b], phs[b]);
        double s = 0; for (int c = 0; c < 16; ++c) s += slots[b][c]; acc += s;
      }
      phs[b] ^= 1;
      __syncthreads();
    } else if (MODE == 2) {   // warp-direct 256 x f32, all wait, each lane sums 8
      if (t == 0) expect(&bar[b], 256 * 4);
      if (lane < 16) sta32(mapa(sptr(&wslots[b][rank * 16 + warp]), lane), 1.f, mapa(sptr(&bar[b]), lane));
      mbar_wait(&bar[b], phs[b]); phs[b] ^= 1;
      double s = 0; for (int i = 0; i < 8; ++i) s += wslots[b][lane * 8 + i]; acc += s;
    } else if (MODE == 3) {   // halo: every thread 4 x 16 B to +-1 neighbours, all wait
      const int nn = (rank > 0) + (rank < 15);
      if (t == 0) expect(&bar[2], nn * 16384);
      float4 v = make_float4(1, 2, 3, 4);
      for (int i = 0; i < 2; ++i) {
        if (rank > 0) sta4(mapa(sptr(sm + 4096 * 2 + (i * 512 + t) * 4), rank - 1), v, mapa(sptr(&bar[2]), rank - 1));
        if (rank < 15) sta4(mapa(sptr(sm + 4096 * 3 + (i * 512 + t) * 4), rank + 1), v, mapa(sptr(&bar[2]), rank + 1));
      }
      mbar_wait(&bar[2], ph); ph ^= 1;
      acc += sm[4096 * 2 + t];
      // a reduction round between halo rounds (as in the solver) keeps CTAs within one phase
      if (t == 0) { expect(&bar[b], 16 * 8); for (int c = 0; c < 16; ++c) sta64(mapa(sptr(&slots[b][rank]), c), 1.0, mapa(sptr(&bar[b]), c)); }
      mbar_wait(&bar[b], phs[b]); phs[b] ^= 1;
    }
  }
  long long t1 = clock64();
  if (t == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * 512 + t] = acc;
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int MODE> int run(long long* dcyc, double* dout) {
  CK(cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(16 * 7); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 65536;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  const int iters = 2000;
  CK(cudaLaunchKernelEx(&cfg, k<MODE>, iters, dcyc, dout)); CK(cudaDeviceSynchronize());
  long long h[112]; CK(cudaMemcpy(h, dcyc, sizeof h, cudaMemcpyDeviceToHost));
  printf("mode %d: %.1f cycles per round (cta0), %.1f (cta5)\n", MODE, h[0] / (double)iters, h[5] / (double)iters);
  return 0;
}
int main() {
  long long* dcyc; double* dout; CK(cudaMalloc(&dcyc, 4096 * 8)); CK(cudaMalloc(&dout, 112 * 512 * 8));
  run<0>(dcyc, dout); run<1>(dcyc, dout); run<2>(dcyc, dout); run<3>(dcyc, dout);
  return 0;
}
