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

// in: input level, plane zb (global) at in[0]; level dims nx,ny,nz; process planes
// [zb, zb+zc) (zb multiple of 2^L, zc multiple of 2^L unless zb+zc == nz).
template <typename T>
__global__ void __launch_bounds__(256)
k_pyramid(const T* __restrict__ in, int nx, int ny, int nz, int zb, int zc, int L, PyrOut o) {
  using A = typename std::conditional<std::is_same<T, float>::value, float, int>::type;
  __shared__ A s1[16 * 16 * 16];
  __shared__ A s2[8 * 8 * 8];
  __shared__ A s3[4 * 4 * 4];
  __shared__ A s4[2 * 2 * 2];
  A* sl[4] = {s1, s2, s3, s4};
  const long long pin = (long long)nx * ny;
  // level 1 from global
  {
    const int X0 = blockIdx.x * 16, Y0 = blockIdx.y * 16, Z0 = (zb >> 1) + blockIdx.z * 16;
    T* out = (T*)o.p[0];
    const long long po = (long long)o.nx[0] * o.ny[0];
    for (int idx = threadIdx.x; idx < 4096; idx += 256) {
      const int lx = idx & 15, ly = (idx >> 4) & 15, lz = idx >> 8;
      const int X = X0 + lx, Y = Y0 + ly, Z = Z0 + lz;
      A v = 0;
      if (X < o.nx[0] && Y < o.ny[0] && Z < o.nz[0] && 2 * Z < zb + zc) {
        const T r = mean8<T, A>([&](int dx, int dy, int dz, A& val) {
          const int x = 2 * X + dx, y = 2 * Y + dy, z = 2 * Z + dz;
          if (x >= nx || y >= ny || z >= nz) return false;
          val = (A)in[(long long)(z - zb) * pin + (long long)y * nx + x];
          return true;
        });
        out[(long long)Z * po + (long long)Y * o.nx[0] + X] = r;
        v = (A)r;
      }
      s1[idx] = v;
    }
  }
  // levels 2..L from shared memory
  for (int l = 1; l < L; ++l) {
    __syncthreads();
    const int e = 16 >> l;                // box extent at this level
    const int X0 = blockIdx.x * e, Y0 = blockIdx.y * e, Z0 = (zb >> (l + 1)) + blockIdx.z * e;
    const A* src = sl[l - 1];
    A* dst = (l < 4) ? sl[l] : nullptr;
    T* out = (T*)o.p[l];
    const long long po = (long long)o.nx[l] * o.ny[l];
    const int pe = 2 * e;                 // child box extent
    for (int idx = threadIdx.x; idx < e * e * e; idx += 256) {
      const int lx = idx % e, ly = (idx / e) % e, lz = idx / (e * e);
      const int X = X0 + lx, Y = Y0 + ly, Z = Z0 + lz;
      A v = 0;
      if (X < o.nx[l] && Y < o.ny[l] && Z < o.nz[l] && 2 * Z < ((zb + zc + (1 << l) - 1) >> l)) {
        const T r = mean8<T, A>([&](int dx, int dy, int dz, A& val) {
          const int x = 2 * X + dx, y = 2 * Y + dy, z = 2 * Z + dz;
          if (x >= o.nx[l - 1] || y >= o.ny[l - 1] || z >= o.nz[l - 1]) return false;
          val = src[((2 * lz + dz) * pe + (2 * ly + dy)) * pe + (2 * lx + dx)];
          return true;
        });
        out[(long long)Z * po + (long long)Y * o.nx[l] + X] = r;
        v = (A)r;
      }
      if (dst) dst[idx] = v;
    }
  }
}

cudaError_t launch_pyramid_group(const void* in, int dtype, int nx, int ny, int nz, int zb,
                                 int zc, int L, const PyrOut& o, cudaStream_t s) {
  const dim3 g((nx + 31) / 32, (ny + 31) / 32, (zc + 31) / 32);
  switch (dtype) {
    case 0: k_pyramid<uint8_t><<<g, 256, 0, s>>>((const uint8_t*)in, nx, ny, nz, zb, zc, L, o); break;
    case 1: k_pyramid<uint16_t><<<g, 256, 0, s>>>((const uint16_t*)in, nx, ny, nz, zb, zc, L, o); break;
    case 2: k_pyramid<int16_t><<<g, 256, 0, s>>>((const int16_t*)in, nx, ny, nz, zb, zc, L, o); break;
    default: k_pyramid<float><<<g, 256, 0, s>>>((const float*)in, nx, ny, nz, zb, zc, L, o); break;
  }
  return cudaGetLastError();
}

}  // namespace rw
