// weights_ex.cu -- SURVEY §8(f) row f3: the paper's alternative edge-weight functions.
//
//   Poisson: w = exp(-1/2 (sqrt(n_p) - sqrt(n_q))^2) + eps, n = raw * count_scale
//                     clipped at 0 (reading R19)
//   Gaussian ([28]): sigma^2 = mean squared 6-neighbour difference of g over the
//                     brick (fp64, floored 1e-8); w = exp(-(g_p - g_q)^2 / (2 sigma^2)) + eps
//                     (reading R20)
//   t-test   ([29]): Welch's t of the (2R+1)^3 neighbourhoods of p and q (clipped
//                     at the brick border, unbiased variances floored 1e-8), two-tailed
//                     normal p-value erfc(|t|/sqrt 2) + eps (reading R21)
// Output layout as rw_brick_weights: W[a][b][z][y][x] = w(v, v + e_a), 0 across the + faces.
// Computed once per solve (not on the CG path): one thread per voxel, fp32 arithmetic with
// fp64 only for the per-brick variance sum (fixed order, one CTA per brick).
#include "rw_common.cuh"

namespace rw {

namespace wex {

struct Geo {
  int B, nx, ny, nz;
  long long n, BN, plane;
};

__device__ __forceinline__ void coords(const Geo& G, long long i, int& x, int& y, int& z) {
  const long long li = i % G.n;
  x = (int)(li % G.nx);
  y = (int)((li / G.nx) % G.ny);
  z = (int)(li / G.plane);
}

template <typename T>
__device__ __forceinline__ float counts(const T* v, long long i, float cs) {
  return fmaxf((float)v[i] * cs, 0.f);
}

}  // namespace wex

using wex::Geo;

// ---------------------------------------------------------------------------- Poisson
template <typename T>
__global__ void __launch_bounds__(256)
k_wpoisson(const T* __restrict__ vol, Geo G, float cs, float eps, float* __restrict__ W) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < G.BN;
       i += (long long)gridDim.x * blockDim.x) {
    int x, y, z;
    wex::coords(G, i, x, y, z);
    const float sp = sqrtf(wex::counts(vol, i, cs));
    const long long off[3] = {1, G.nx, G.plane};
    const bool in[3] = {x + 1 < G.nx, y + 1 < G.ny, z + 1 < G.nz};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      float w = 0.f;
      if (in[a]) {
        const float d = __fsub_rn(sqrtf(wex::counts(vol, i + off[a], cs)), sp);
        w = __fadd_rn(expf(-0.5f * __fmul_rn(d, d)), eps);
      }
      W[a * G.BN + i] = w;
    }
  }
}

// ---------------------------------------------------------------------------- Gaussian
// sigma^2 of brick b: one CTA, fp64 sums of fp32 differences in a fixed order
template <typename T>
__global__ void __launch_bounds__(256)
k_sigma2(const T* __restrict__ vol, Geo G, float sc, float of, double* __restrict__ sig2) {
  __shared__ double red[256 / 32];
  const int b = blockIdx.x;
  const long long base = (long long)b * G.n;
  double acc = 0.0;
  for (long long li = threadIdx.x; li < G.n; li += blockDim.x) {
    int x, y, z;
    wex::coords(G, base + li, x, y, z);
    const float g = normv((float)vol[base + li], sc, of);
    if (x + 1 < G.nx) {
      const float d = __fsub_rn(normv((float)vol[base + li + 1], sc, of), g);
      acc = __fma_rn((double)d, (double)d, acc);
    }
    if (y + 1 < G.ny) {
      const float d = __fsub_rn(normv((float)vol[base + li + G.nx], sc, of), g);
      acc = __fma_rn((double)d, (double)d, acc);
    }
    if (z + 1 < G.nz) {
      const float d = __fsub_rn(normv((float)vol[base + li + G.plane], sc, of), g);
      acc = __fma_rn((double)d, (double)d, acc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    const double edges = (double)(G.nx - 1) * G.ny * G.nz + (double)G.nx * (G.ny - 1) * G.nz +
                         (double)G.nx * G.ny * (G.nz - 1);
    const double v = edges > 0 ? s / edges : 0.0;
    sig2[b] = v > 1e-8 ? v : 1e-8;
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
k_wgauss(const T* __restrict__ vol, Geo G, float sc, float of, const double* __restrict__ sig2,
         float eps, float* __restrict__ W) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < G.BN;
       i += (long long)gridDim.x * blockDim.x) {
    int x, y, z;
    wex::coords(G, i, x, y, z);
    const float k = (float)(-0.5 / sig2[i / G.n]);   // -1 / (2 sigma^2)
    const float g = normv((float)vol[i], sc, of);
    const long long off[3] = {1, G.nx, G.plane};
    const bool in[3] = {x + 1 < G.nx, y + 1 < G.ny, z + 1 < G.nz};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      float w = 0.f;
      if (in[a]) {
        const float d = __fsub_rn(normv((float)vol[i + off[a]], sc, of), g);
        w = __fadd_rn(expf(__fmul_rn(__fmul_rn(d, d), k)), eps);
      }
      W[a * G.BN + i] = w;
    }
  }
}

// ---------------------------------------------------------------------------- t-test
// per voxel: mean and var/n of the clipped (2R+1)^3 neighbourhood (two-pass, fp32)
template <typename T>
__global__ void __launch_bounds__(256)
k_tstats(const T* __restrict__ vol, Geo G, float sc, float of, int R, float* __restrict__ mean,
         float* __restrict__ vn) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < G.BN;
       i += (long long)gridDim.x * blockDim.x) {
    int x, y, z;
    wex::coords(G, i, x, y, z);
    const long long base = i - ((long long)z * G.plane + (long long)y * G.nx + x);
    const int z0 = max(z - R, 0), z1 = min(z + R, G.nz - 1);
    const int y0 = max(y - R, 0), y1 = min(y + R, G.ny - 1);
    const int x0 = max(x - R, 0), x1 = min(x + R, G.nx - 1);
    float s = 0.f;
    for (int zz = z0; zz <= z1; ++zz)
      for (int yy = y0; yy <= y1; ++yy)
        for (int xx = x0; xx <= x1; ++xx)
          s = __fadd_rn(s, normv((float)vol[base + (long long)zz * G.plane + (long long)yy * G.nx + xx], sc, of));
    const int cnt = (z1 - z0 + 1) * (y1 - y0 + 1) * (x1 - x0 + 1);
    const float m = __fdiv_rn(s, (float)cnt);
    float ss = 0.f;
    for (int zz = z0; zz <= z1; ++zz)
      for (int yy = y0; yy <= y1; ++yy)
        for (int xx = x0; xx <= x1; ++xx) {
          const float d = __fsub_rn(normv((float)vol[base + (long long)zz * G.plane + (long long)yy * G.nx + xx], sc, of), m);
          ss = __fmaf_rn(d, d, ss);
        }
    float var = cnt > 1 ? __fdiv_rn(ss, (float)(cnt - 1)) : 0.f;
    var = fmaxf(var, 1e-8f);
    mean[i] = m;
    vn[i] = __fdiv_rn(var, (float)cnt);
  }
}

__global__ void __launch_bounds__(256)
k_wttest(const float* __restrict__ mean, const float* __restrict__ vn, Geo G, float eps,
         float* __restrict__ W) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < G.BN;
       i += (long long)gridDim.x * blockDim.x) {
    int x, y, z;
    wex::coords(G, i, x, y, z);
    const long long off[3] = {1, G.nx, G.plane};
    const bool in[3] = {x + 1 < G.nx, y + 1 < G.ny, z + 1 < G.nz};
    const float mp = mean[i], vp = vn[i];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      float w = 0.f;
      if (in[a]) {
        const long long j = i + off[a];
        // |t| / sqrt 2 = |m_p - m_q| / sqrt(2 (v_p/n_p + v_q/n_q))
        const float u = __fdiv_rn(fabsf(__fsub_rn(mp, mean[j])),
                                  sqrtf(__fmul_rn(2.f, __fadd_rn(vp, vn[j]))));
        w = __fadd_rn(erfcf(u), eps);
      }
      W[a * G.BN + i] = w;
    }
  }
}

// ---------------------------------------------------------------------------- launchers
static int grid_for(long long items, int sms) {
  long long g = (items + 255) / 256;
  const long long cap = (long long)sms * 8;
  return (int)(g < cap ? (g < 1 ? 1 : g) : cap);
}

template <typename T>
static cudaError_t launch_kind(const T* vol, const Geo& G, int kind, float sc, float of,
                               float eps, float cs, int R, float* W, void* ws, int sms,
                               cudaStream_t s) {
  const int grid = grid_for(G.BN, sms);
  if (kind == 1) {
    k_wpoisson<T><<<grid, 256, 0, s>>>(vol, G, cs, eps, W);
  } else if (kind == 2) {
    double* sig2 = reinterpret_cast<double*>(ws);
    k_sigma2<T><<<G.B, 256, 0, s>>>(vol, G, sc, of, sig2);
    k_wgauss<T><<<grid, 256, 0, s>>>(vol, G, sc, of, sig2, eps, W);
  } else {
    float* mean = reinterpret_cast<float*>(ws);
    float* vn = mean + G.BN;
    k_tstats<T><<<grid, 256, 0, s>>>(vol, G, sc, of, R, mean, vn);
    k_wttest<<<grid, 256, 0, s>>>(mean, vn, G, eps, W);
  }
  return cudaGetLastError();
}

size_t weights_ex_workspace(int kind, int B, long long n) {
  if (kind == 2) return (size_t)B * sizeof(double);
  if (kind == 3) return (size_t)2 * B * n * sizeof(float);
  return 0;
}

cudaError_t launch_weights_ex(const void* vol, int dtype, float sc, float of, int B, int nx,
                              int ny, int nz, int kind, float eps, float cs, int R, float* W,
                              void* ws, int sms, cudaStream_t s) {
  Geo G;
  G.B = B; G.nx = nx; G.ny = ny; G.nz = nz;
  G.plane = (long long)nx * ny;
  G.n = G.plane * nz;
  G.BN = (long long)B * G.n;
  switch (dtype) {
    case 0: return launch_kind((const uint8_t*)vol, G, kind, sc, of, eps, cs, R, W, ws, sms, s);
    case 1: return launch_kind((const uint16_t*)vol, G, kind, sc, of, eps, cs, R, W, ws, sms, s);
    case 2: return launch_kind((const int16_t*)vol, G, kind, sc, of, eps, cs, R, W, ws, sms, s);
    default: return launch_kind((const float*)vol, G, kind, sc, of, eps, cs, R, W, ws, sms, s);
  }
}

}  // namespace rw
