// pyramid.cu -- SURVEY §8(a) row a8: LOD pyramid by 2^3 mean, fused multi-level.
//
// Reading c12: level l+1 voxel (X,Y,Z) = mean of the present children (2X..2X+1, ...)
// of level l; dims ceil(d/2); integers: round-half-up floor((s + floor(cnt/2)) / cnt),
// bit-exact; f32: fixed pairwise order ((c000+c100)+(c010+c110))+((c001+c101)+(c011+c111))
// over present children, then one IEEE division by cnt.
//
// One CTA reads a 32^3 box of the input level once and produces up to 5 levels
// (16^3, 8^3, 4^3, 2^3, 1) from shared memory, so HBM traffic is one read of the input
// plus the (1/8 + 1/64 + ...) outputs: ~2.29 B per u16 input voxel.
#include <type_traits>

#include "rw_common.cuh"
#include "tma.cuh"

namespace rw {

__device__ __forceinline__ int floor_div(int a, int b) {  // b > 0
  int q = a / b;
  if ((a % b) != 0 && a < 0) --q;
  return q;
}

template <typename A> struct Term { A v; int n; };

template <typename A>
__device__ __forceinline__ Term<A> tadd(Term<A> a, Term<A> b) {
  if (a.n == 0) return b;
  if (b.n == 0) return a;
  return Term<A>{a.v + b.v, a.n + b.n};
}

template <typename T, typename A>
__device__ __forceinline__ T finish(Term<A> s);
template <> __device__ __forceinline__ float finish<float, float>(Term<float> s) {
  return s.v / (float)s.n;
}
template <typename T, typename A>
__device__ __forceinline__ T finish(Term<A> s) {
  return (T)floor_div(s.v + s.n / 2, s.n);
}

// mean of the present children; get(dx,dy,dz, &val) returns presence
template <typename T, typename A, typename G>
__device__ __forceinline__ T mean8(G get) {
  Term<A> t[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int dx = k & 1, dy = (k >> 1) & 1, dz = k >> 2;
    A v = 0;
    const bool ok = get(dx, dy, dz, v);
    t[k] = Term<A>{ok ? v : (A)0, ok ? 1 : 0};
  }
  const Term<A> s01 = tadd(tadd(t[0], t[1]), tadd(t[2], t[3]));
  const Term<A> s23 = tadd(tadd(t[4], t[5]), tadd(t[6], t[7]));
  return finish<T, A>(tadd(s01, s23));
}

__device__ __forceinline__ int pe3(int l) { const int e = 16 >> l; return (2 * e) * (2 * e) * (2 * e); }

// in: input level, plane zb (global) at in[0]; level dims nx,ny,nz; process planes
// [zb, zb+zc) (zb multiple of 2^L, zc multiple of 2^L unless zb+zc == nz).
// USE_TMA: the CTA's 32^3 input box is staged in shared memory by one TMA load
// (cp.async.bulk.tensor, zero-filled outside the volume) instead of scattered 1-4 byte
// global loads; requires nx * sizeof(T) % 16 == 0 (tensor-map row pitch).
template <typename T, bool USE_TMA>
__global__ void __launch_bounds__(256)
k_pyramid(const T* __restrict__ in, int nx, int ny, int nz, int zb, int zc, int L, PyrOut o,
          const __grid_constant__ CUtensorMap map) {
  using A = typename std::conditional<std::is_same<T, float>::value, float, int>::type;
  extern __shared__ __align__(128) unsigned char dsm[];
  const T* box = reinterpret_cast<const T*>(dsm);
  uint64_t* bar = reinterpret_cast<uint64_t*>(dsm + 32 * 32 * 32 * sizeof(T));
  if (USE_TMA) {
    // two 32x32x16 loads on two mbarriers: level 1's lower half (output planes 0..7)
    // starts as soon as the lower half of the box has landed
    if (threadIdx.x == 0) {
      mbar_init(&bar[0], 1);
      mbar_init(&bar[1], 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      constexpr uint32_t half = 32 * 32 * 16 * sizeof(T);
      mbar_arrive_expect_tx(&bar[0], half);
      tma_load_3d(dsm, &map, &bar[0], blockIdx.x * 32, blockIdx.y * 32, blockIdx.z * 32);
      mbar_arrive_expect_tx(&bar[1], half);
      tma_load_3d(dsm + half, &map, &bar[1], blockIdx.x * 32, blockIdx.y * 32, blockIdx.z * 32 + 16);
    }
  }
  // level buffers 1..4 (16^3, 8^3, 4^3, 2^3) in one array of the input type (every level
  // mean fits it), so three CTAs of a 2-byte type fit one SM; offsets computed, not indexed
  // through a pointer table (which would live in local memory)
  __shared__ T lv[4096 + 512 + 64 + 8];
  T* s1 = lv;
  const long long pin = (long long)nx * ny;
  // level 1 from global
  {
    const int X0 = blockIdx.x * 16, Y0 = blockIdx.y * 16, Z0 = (zb >> 1) + blockIdx.z * 16;
    T* out = (T*)o.p[0];
    const long long po = (long long)o.nx[0] * o.ny[0];
    for (int idx = threadIdx.x; idx < 4096; idx += 256) {
      if (USE_TMA && (idx & 2047) < 256) mbar_wait(&bar[idx >> 11], 0);   // half 0, then 1
      const int lx = idx & 15, ly = (idx >> 4) & 15, lz = idx >> 8;
      const int X = X0 + lx, Y = Y0 + ly, Z = Z0 + lz;
      A v = 0;
      if (USE_TMA && 2 * X + 1 < nx && 2 * Y + 1 < ny && 2 * Z + 1 < nz && 2 * Z + 1 < zb + zc) {
        // interior fast path: all 8 children present -> same rule, no count bookkeeping
        const T* c = box + ((2 * lz) * 32 + 2 * ly) * 32 + 2 * lx;
        T r;
        if (std::is_same<T, float>::value) {
          const float s01 = ((float)c[0] + (float)c[1]) + ((float)c[32] + (float)c[33]);
          const float s23 = ((float)c[1024] + (float)c[1025]) + ((float)c[1056] + (float)c[1057]);
          r = (T)((s01 + s23) / 8.0f);
        } else {
          const int s = ((int)c[0] + (int)c[1]) + ((int)c[32] + (int)c[33]) +
                        ((int)c[1024] + (int)c[1025]) + ((int)c[1056] + (int)c[1057]);
          r = (T)((s + 4) >> 3);                // floor((s + 4) / 8), arithmetic shift
        }
        out[(long long)Z * po + (long long)Y * o.nx[0] + X] = r;
        v = (A)r;
      } else if (X < o.nx[0] && Y < o.ny[0] && Z < o.nz[0] && 2 * Z < zb + zc) {
        const T r = mean8<T, A>([&](int dx, int dy, int dz, A& val) {
          const int x = 2 * X + dx, y = 2 * Y + dy, z = 2 * Z + dz;
          if (x >= nx || y >= ny || z >= nz) return false;
          val = USE_TMA ? (A)box[((2 * lz + dz) * 32 + (2 * ly + dy)) * 32 + (2 * lx + dx)]
                        : (A)in[(long long)(z - zb) * pin + (long long)y * nx + x];
          return true;
        });
        out[(long long)Z * po + (long long)Y * o.nx[0] + X] = r;
        v = (A)r;
      }
      s1[idx] = (T)v;
    }
  }
  // levels 2..L from shared memory
#pragma unroll
  for (int l = 1; l < 5; ++l) {
    if (l >= L) break;
    __syncthreads();
    const int e = 16 >> l;                // box extent at this level
    const int X0 = blockIdx.x * e, Y0 = blockIdx.y * e, Z0 = (zb >> (l + 1)) + blockIdx.z * e;
    const int off_src = l == 1 ? 0 : (l == 2 ? 4096 : (l == 3 ? 4608 : 4672));
    const T* src = lv + off_src;
    T* dst = (l < 4) ? lv + off_src + pe3(l) : nullptr;
    T* out = (T*)o.p[l];
    const long long po = (long long)o.nx[l] * o.ny[l];
    const int pe = 2 * e;                 // child box extent
    for (int idx = threadIdx.x; idx < e * e * e; idx += 256) {
      const int lx = idx % e, ly = (idx / e) % e, lz = idx / (e * e);
      const int X = X0 + lx, Y = Y0 + ly, Z = Z0 + lz;
      A v = 0;
      const int zend = (zb + zc + (1 << l) - 1) >> l;   // slab end at the child level
      if (2 * X + 1 < o.nx[l - 1] && 2 * Y + 1 < o.ny[l - 1] && 2 * Z + 1 < o.nz[l - 1] &&
          2 * Z + 1 < zend) {                           // interior: 8 children present
        const T* c = src + ((2 * lz) * pe + 2 * ly) * pe + 2 * lx;
        const int pp = pe * pe;
        T r;
        if (std::is_same<T, float>::value) {
          const float s01 = ((float)c[0] + (float)c[1]) + ((float)c[pe] + (float)c[pe + 1]);
          const float s23 = ((float)c[pp] + (float)c[pp + 1]) + ((float)c[pp + pe] + (float)c[pp + pe + 1]);
          r = (T)((s01 + s23) / 8.0f);
        } else {
          const int s = ((int)c[0] + (int)c[1]) + ((int)c[pe] + (int)c[pe + 1]) +
                        ((int)c[pp] + (int)c[pp + 1]) + ((int)c[pp + pe] + (int)c[pp + pe + 1]);
          r = (T)((s + 4) >> 3);
        }
        out[(long long)Z * po + (long long)Y * o.nx[l] + X] = r;
        v = (A)r;
      } else if (X < o.nx[l] && Y < o.ny[l] && Z < o.nz[l] && 2 * Z < zend) {
        const T r = mean8<T, A>([&](int dx, int dy, int dz, A& val) {
          const int x = 2 * X + dx, y = 2 * Y + dy, z = 2 * Z + dz;
          if (x >= o.nx[l - 1] || y >= o.ny[l - 1] || z >= o.nz[l - 1]) return false;
          val = (A)src[((2 * lz + dz) * pe + (2 * ly + dy)) * pe + (2 * lx + dx)];
          return true;
        });
        out[(long long)Z * po + (long long)Y * o.nx[l] + X] = r;
        v = (A)r;
      }
      if (dst) dst[idx] = (T)v;
    }
  }
}

template <typename T>
static cudaError_t launch_t(const void* in, int nx, int ny, int nz, int zb, int zc, int L,
                           const PyrOut& o, const CUtensorMap* map, cudaStream_t s) {
  const dim3 g((nx + 31) / 32, (ny + 31) / 32, (zc + 31) / 32);
  if (map) {
    const int smem = 32 * 32 * 32 * sizeof(T) + 16;
    static int attr = 0;
    if (attr < smem) {
      const cudaError_t e = cudaFuncSetAttribute(k_pyramid<T, true>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      attr = smem;
    }
    k_pyramid<T, true><<<g, 256, smem, s>>>((const T*)in, nx, ny, nz, zb, zc, L, o, *map);
  } else {
    CUtensorMap dummy{};
    k_pyramid<T, false><<<g, 256, 0, s>>>((const T*)in, nx, ny, nz, zb, zc, L, o, dummy);
  }
  return cudaGetLastError();
}

cudaError_t launch_pyramid_group(const void* in, int dtype, int nx, int ny, int nz, int zb,
                                 int zc, int L, const PyrOut& o, const CUtensorMap* map,
                                 cudaStream_t s) {
  switch (dtype) {
    case 0: return launch_t<uint8_t>(in, nx, ny, nz, zb, zc, L, o, map, s);
    case 1: return launch_t<uint16_t>(in, nx, ny, nz, zb, zc, L, o, map, s);
    case 2: return launch_t<int16_t>(in, nx, ny, nz, zb, zc, L, o, map, s);
    default: return launch_t<float>(in, nx, ny, nz, zb, zc, L, o, map, s);
  }
}

}  // namespace rw
