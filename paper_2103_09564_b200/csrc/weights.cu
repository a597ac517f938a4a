// weights.cu -- SURVEY §8(a) rows a1/a2: normalisation + Grady edge weights + Jacobi dinv.
//
// w_pq = exp(-beta (n[p]-n[q])^2); + eps (reading c1).  One thread owns 4
// consecutive x voxels (one float4 of each output plane) and reads the 7-point
// neighbourhood of intensities (x-1, x+4, y+-1, z+-1).  The three "forward" weights of a
// voxel are stored (unless W == nullptr: the solver's on-the-fly modes only need dinv);
// the three "backward" weights needed for dinv are recomputed with the identical operand
// order (d = g[v] - g[v - e_a]) so they are bit-identical to the forward weight stored at
// v - e_a.  HBM-bound: 1-4 B in, 4-16 B out per voxel.
#include "rw_common.cuh"

namespace rw {

template <typename T> struct Vec4;
template <> struct Vec4<float> { using type = float4; };
template <> struct Vec4<uint16_t> { using type = ushort4; };
template <> struct Vec4<int16_t> { using type = short4; };
template <> struct Vec4<uint8_t> { using type = uchar4; };

template <typename T>
__device__ __forceinline__ void load4(const T* p, float s, float o, float g[4]) {
  typename Vec4<T>::type v = *reinterpret_cast<const typename Vec4<T>::type*>(p);
  g[0] = normv((float)v.x, s, o);
  g[1] = normv((float)v.y, s, o);
  g[2] = normv((float)v.z, s, o);
  g[3] = normv((float)v.w, s, o);
}

template <typename T>
__global__ void __launch_bounds__(256)
k_weights(const T* __restrict__ vol, float sc, float of, int B, int nx, int ny, int nz,
          float nbl2, float eps, float* __restrict__ W, float* __restrict__ dinv,
          const uint8_t* __restrict__ fixed) {
  const long long n = (long long)nx * ny * nz;
  const long long groups = (long long)B * n / 4;
  const long long plane = (long long)nx * ny;
  const long long BN = (long long)B * n;
  for (long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x; gi < groups;
       gi += (long long)gridDim.x * blockDim.x) {
    const long long i = gi * 4;               // first voxel (global index incl. brick)
    const long long li = i % n;               // brick-local
    const int x = (int)(li % nx);
    const int y = (int)((li / nx) % ny);
    const int z = (int)(li / plane);
    float g[4], gyp[4] = {0.f, 0.f, 0.f, 0.f}, gym[4] = {0.f, 0.f, 0.f, 0.f};
    float gzp[4] = {0.f, 0.f, 0.f, 0.f}, gzm[4] = {0.f, 0.f, 0.f, 0.f};
    load4<T>(vol + i, sc, of, g);
    const float gxm = (x > 0) ? normv((float)vol[i - 1], sc, of) : 0.f;
    const float gxp = (x + 4 < nx) ? normv((float)vol[i + 4], sc, of) : 0.f;
    if (y + 1 < ny) load4<T>(vol + i + nx, sc, of, gyp);
    if (y > 0) load4<T>(vol + i - nx, sc, of, gym);
    if (z + 1 < nz) load4<T>(vol + i + plane, sc, of, gzp);
    if (z > 0) load4<T>(vol + i - plane, sc, of, gzm);
    float wx[4], wy[4], wz[4], dv[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float gn = (c < 3) ? g[c + 1] : gxp;
      const float gp = (c > 0) ? g[c - 1] : gxm;
      wx[c] = (x + c + 1 < nx) ? grady(__fsub_rn(gn, g[c]), nbl2, eps) : 0.f;
      const float wxm = (x + c > 0) ? grady(__fsub_rn(g[c], gp), nbl2, eps) : 0.f;
      wy[c] = (y + 1 < ny) ? grady(__fsub_rn(gyp[c], g[c]), nbl2, eps) : 0.f;
      const float wym = (y > 0) ? grady(__fsub_rn(g[c], gym[c]), nbl2, eps) : 0.f;
      wz[c] = (z + 1 < nz) ? grady(__fsub_rn(gzp[c], g[c]), nbl2, eps) : 0.f;
      const float wzm = (z > 0) ? grady(__fsub_rn(g[c], gzm[c]), nbl2, eps) : 0.f;
      // fixed summation order (the same as k_dinv)
      const float s = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(wx[c], wxm), wy[c]), wym), wz[c]), wzm);
      dv[c] = (s > 0.f) ? __frcp_rn(s) : 0.f;
    }
    if (W) {
      *reinterpret_cast<float4*>(W + i) = make_float4(wx[0], wx[1], wx[2], wx[3]);
      *reinterpret_cast<float4*>(W + BN + i) = make_float4(wy[0], wy[1], wy[2], wy[3]);
      *reinterpret_cast<float4*>(W + 2 * BN + i) = make_float4(wz[0], wz[1], wz[2], wz[3]);
    }
    if (dinv) {
      if (fixed) {
        const uchar4 f = *reinterpret_cast<const uchar4*>(fixed + i);
        if (f.x) dv[0] = 0.f;
        if (f.y) dv[1] = 0.f;
        if (f.z) dv[2] = 0.f;
        if (f.w) dv[3] = 0.f;
      }
      *reinterpret_cast<float4*>(dinv + i) = make_float4(dv[0], dv[1], dv[2], dv[3]);
    }
  }
}

// dinv from caller-provided weight planes (same summation order as k_weights).
__global__ void __launch_bounds__(256)
k_dinv(const float* __restrict__ W, int B, int nx, int ny, int nz,
       const uint8_t* __restrict__ fixed, float* __restrict__ dinv) {
  const long long n = (long long)nx * ny * nz;
  const long long groups = (long long)B * n / 4;
  const long long plane = (long long)nx * ny;
  const long long BN = (long long)B * n;
  for (long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x; gi < groups;
       gi += (long long)gridDim.x * blockDim.x) {
    const long long i = gi * 4;
    const long long li = i % n;
    const int x = (int)(li % nx);
    const int y = (int)((li / nx) % ny);
    const int z = (int)(li / plane);
    const float4 wx = *reinterpret_cast<const float4*>(W + i);
    const float4 wy = *reinterpret_cast<const float4*>(W + BN + i);
    const float4 wz = *reinterpret_cast<const float4*>(W + 2 * BN + i);
    const float wxm0 = (x > 0) ? W[i - 1] : 0.f;
    float4 wym = make_float4(0.f, 0.f, 0.f, 0.f), wzm = wym;
    if (y > 0) wym = *reinterpret_cast<const float4*>(W + BN + i - nx);
    if (z > 0) wzm = *reinterpret_cast<const float4*>(W + 2 * BN + i - plane);
    const float a[4] = {wx.x, wx.y, wx.z, wx.w};
    const float bm[4] = {wxm0, wx.x, wx.y, wx.z};
    const float c[4] = {wy.x, wy.y, wy.z, wy.w};
    const float cm[4] = {wym.x, wym.y, wym.z, wym.w};
    const float e[4] = {wz.x, wz.y, wz.z, wz.w};
    const float em[4] = {wzm.x, wzm.y, wzm.z, wzm.w};
    float dv[4];
    uchar4 f = make_uchar4(0, 0, 0, 0);
    if (fixed) f = *reinterpret_cast<const uchar4*>(fixed + i);
    const unsigned char fv[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float s = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(a[k], bm[k]), c[k]), cm[k]), e[k]), em[k]);
      dv[k] = (fv[k] || !(s > 0.f)) ? 0.f : __frcp_rn(s);
    }
    *reinterpret_cast<float4*>(dinv + i) = make_float4(dv[0], dv[1], dv[2], dv[3]);
  }
}

static int grid_for(long long groups, int dev_sms) {
  long long g = (groups + 255) / 256;
  const long long cap = (long long)dev_sms * 8;
  return (int)(g < cap ? (g < 1 ? 1 : g) : cap);
}

cudaError_t launch_weights(const void* vol, int dtype, float sc, float of, int B, int nx,
                           int ny, int nz, float beta, float eps, float* W, float* dinv,
                           const uint8_t* fixed, int sms, cudaStream_t s) {
  const long long groups = (long long)B * nx * ny * nz / 4;
  const int grid = grid_for(groups, sms);
  const float nbl2 = nbl2_of(beta);
  switch (dtype) {
    case 0: k_weights<uint8_t><<<grid, 256, 0, s>>>((const uint8_t*)vol, sc, of, B, nx, ny, nz, nbl2, eps, W, dinv, fixed); break;
    case 1: k_weights<uint16_t><<<grid, 256, 0, s>>>((const uint16_t*)vol, sc, of, B, nx, ny, nz, nbl2, eps, W, dinv, fixed); break;
    case 2: k_weights<int16_t><<<grid, 256, 0, s>>>((const int16_t*)vol, sc, of, B, nx, ny, nz, nbl2, eps, W, dinv, fixed); break;
    default: k_weights<float><<<grid, 256, 0, s>>>((const float*)vol, sc, of, B, nx, ny, nz, nbl2, eps, W, dinv, fixed); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_dinv(const float* W, int B, int nx, int ny, int nz, const uint8_t* fixed,
                        float* dinv, int sms, cudaStream_t s) {
  const long long groups = (long long)B * nx * ny * nz / 4;
  k_dinv<<<grid_for(groups, sms), 256, 0, s>>>(W, B, nx, ny, nz, fixed, dinv);
  return cudaGetLastError();
}

}  // namespace rw
