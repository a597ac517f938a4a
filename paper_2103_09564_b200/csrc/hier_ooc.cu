// hier_ooc.cu -- device kernels of the out-of-core hierarchical driver rw_hier_segment_ooc
// (SURVEY §8(f) f1 at constant device memory; "applicable to arbitrarily large
// out-of-core datasets", P:109-111 volumes of any size, P:151 nearest computed ancestor).
// The orchestration is in api.cu.
//
// The level fields are never stored densely.  Level l keeps a page table PT_l over its
// bricks (int32 slot or -1) into one brick pool of s^3 fp32 values:
//   * a solved brick's s^3 (the contracted window solution, Eq. 3) gets a slot;
//   * an unsolved brick is, by the dense driver's definition (reading R26: every level's field
//     starts as the trilinear upsample of the parent field and solved bricks overwrite their
//     s^3), the upsample of level l+1 -- materialised into a slot only where a window or a
//     finer materialisation samples it (k_ooc_materialize, planned on the host from the
//     coarsest missing ancestor down);
//   * the full-resolution output is produced slab by slab (k_ooc_out): per level, a dense
//     buffer over the planes the slab needs = pool values where materialised, else the upsample
//     of the coarser slab buffer -- the same values the dense driver computes.
// All trilinear samples use the arithmetic of hier.cu (hier::pcoord / sample, k_upsample), so
// the field is bit-identical to rw_hier_segment's on cubic s 2^k volumes.
// Volumes of any dims (reading R31): level dims ceil(d/2), smaller border bricks, windows of
// side min(s_e, d_l) per axis; windows whose x side is not a multiple of 4 (the solver's
// float4 rows) are padded in x with fixed voxels whose edges to the window get weight 0
// (k_ooc_wfix), which leaves the system on the real voxels unchanged.
#include "rw_common.cuh"

namespace rw {

namespace ooc {

__device__ __forceinline__ void pcoord(int i, int np, int& i0, int& i1, float& f) {
  float u = fminf(fmaxf(0.5f * (float)i - 0.25f, 0.f), (float)(np - 1));
  i0 = (int)floorf(u);
  i1 = min(i0 + 1, np - 1);
  f = u - (float)i0;
}

// value of level m at voxel (z, y, x): its brick must be materialised
__device__ __forceinline__ float at(const OocGeo& G, const int* __restrict__ PT,
                                    const float* __restrict__ pool, int m, int z, int y, int x) {
  const int s = G.s;
  const int bz = z / s, by = y / s, bx = x / s;
  const int slot = PT[G.pt[m] + ((long long)bz * G.by[m] + by) * G.bx[m] + bx];
  const long long s3 = (long long)s * s * s;
  return pool[slot * s3 + ((long long)(z - bz * s) * s + (y - by * s)) * s + (x - bx * s)];
}

// trilinear sample of level m+1 at the centre of level-m voxel (z, y, x) (hier::sample order)
__device__ __forceinline__ float sample_up(const OocGeo& G, const int* __restrict__ PT,
                                           const float* __restrict__ pool, int m, int z, int y,
                                           int x) {
  const int p = m + 1;
  int z0, z1, y0, y1, x0, x1;
  float fz, fy, fx;
  pcoord(z, G.nz[p], z0, z1, fz);
  pcoord(y, G.ny[p], y0, y1, fy);
  pcoord(x, G.nx[p], x0, x1, fx);
  auto P = [&](int a, int b, int c) { return at(G, PT, pool, p, a, b, c); };
  const float c00 = __fmaf_rn(fx, P(z0, y0, x1), (1.f - fx) * P(z0, y0, x0));
  const float c01 = __fmaf_rn(fx, P(z0, y1, x1), (1.f - fx) * P(z0, y1, x0));
  const float c10 = __fmaf_rn(fx, P(z1, y0, x1), (1.f - fx) * P(z1, y0, x0));
  const float c11 = __fmaf_rn(fx, P(z1, y1, x1), (1.f - fx) * P(z1, y1, x0));
  const float c0 = __fmaf_rn(fy, c01, (1.f - fy) * c00);
  const float c1 = __fmaf_rn(fy, c11, (1.f - fy) * c10);
  return __fmaf_rn(fz, c1, (1.f - fz) * c0);
}

}  // namespace ooc

// level-0 labels (0 / 1 fg / 2 bg) of a z-slab -> level-1 bits: OR of the present children's
// bits (reading R22, R31).  Output planes [z0/2, ceil((z0 + nzs)/2)); z0 even.
__global__ void k_ooc_seedor0(const uint8_t* __restrict__ seeds, int z0, int nzs, OocGeo G,
                              uint8_t* __restrict__ out) {
  const int nx = G.nx[0], ny = G.ny[0], nz = G.nz[0];
  const int ox = G.nx[1], oy = G.ny[1];
  const int Z0 = z0 / 2, Z1 = (z0 + nzs + 1) / 2;
  const long long n = (long long)(Z1 - Z0) * oy * ox;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int X = (int)(i % ox), Y = (int)((i / ox) % oy), Z = Z0 + (int)(i / ((long long)ox * oy));
    uint32_t acc = 0;
    for (int dz = 0; dz < 2; ++dz) {
      const int z = 2 * Z + dz;
      if (z >= nz || z >= z0 + nzs) continue;
      for (int dy = 0; dy < 2; ++dy) {
        const int y = 2 * Y + dy;
        if (y >= ny) continue;
        for (int dx = 0; dx < 2; ++dx) {
          const int x = 2 * X + dx;
          if (x >= nx) continue;
          const uint8_t v = seeds[((long long)(z - z0) * ny + y) * nx + x];
          acc |= (v == 1 ? 1u : 0u) | (v == 2 ? 2u : 0u);
        }
      }
    }
    out[((long long)Z * oy + Y) * ox + X] = (uint8_t)acc;
  }
}

// one-vs-rest seeds of class `cls` ("only seeds for the current class are considered
// foreground and all other seeds as background"), in place on a freshly copied slot:
// class label (0 unseeded, 1..K) -> 0 / 1 (fg: label == cls) / 2 (bg: any other class)
__global__ void k_ooc_remap(uint8_t* __restrict__ seeds, long long n, int cls) {
  // words when the slot's seed part is 4-byte aligned, bytes otherwise (odd u8 volumes)
  const long long n4 = (reinterpret_cast<uintptr_t>(seeds) & 3u) == 0 ? n / 4 : 0;
  uint32_t* s4 = reinterpret_cast<uint32_t*>(seeds);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const uint32_t v = s4[i];
    uint32_t o = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t c = (v >> (8 * b)) & 0xffu;
      o |= (c == 0u ? 0u : (c == (uint32_t)cls ? 1u : 2u)) << (8 * b);
    }
    s4[i] = o;
  }
  for (long long i = 4 * n4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const uint8_t c = seeds[i];
    seeds[i] = c == 0 ? 0 : (c == cls ? 1 : 2);
  }
}

// bits of level m -> level m+1 (any dims)
__global__ void k_ooc_seedor(const uint8_t* __restrict__ in, int m, OocGeo G,
                             uint8_t* __restrict__ out) {
  const int nx = G.nx[m], ny = G.ny[m], nz = G.nz[m];
  const int ox = G.nx[m + 1], oy = G.ny[m + 1], oz = G.nz[m + 1];
  const long long n = (long long)oz * oy * ox;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int X = (int)(i % ox), Y = (int)((i / ox) % oy), Z = (int)(i / ((long long)ox * oy));
    uint32_t acc = 0;
    for (int dz = 0; dz < 2; ++dz)
      for (int dy = 0; dy < 2; ++dy)
        for (int dx = 0; dx < 2; ++dx) {
          const int z = 2 * Z + dz, y = 2 * Y + dy, x = 2 * X + dx;
          if (z < nz && y < ny && x < nx) acc |= in[((long long)z * ny + y) * nx + x];
        }
    out[i] = (uint8_t)acc;
  }
}

// Materialise unsolved bricks of level m as the upsample of level m+1 (reading R26).
// job = (bx, by, bz, slot); one CTA per job; the page-table entry is written last.
__global__ void k_ooc_materialize(const int4* __restrict__ jobs, int m, OocGeo G,
                                  int* __restrict__ PT, float* __restrict__ pool) {
  const int4 jb = jobs[blockIdx.x];
  const int s = G.s;
  const int cx = min(s, G.nx[m] - jb.x * s), cy = min(s, G.ny[m] - jb.y * s),
            cz = min(s, G.nz[m] - jb.z * s);
  const long long s3 = (long long)s * s * s;
  float* dst = pool + jb.w * s3;
  const int nc = cx * cy * cz;
  for (int t = threadIdx.x; t < nc; t += blockDim.x) {
    const int lx = t % cx, ly = (t / cx) % cy, lz = t / (cx * cy);
    dst[((long long)lz * s + ly) * s + lx] =
        ooc::sample_up(G, PT, pool, m, jb.z * s + lz, jb.y * s + ly, jb.x * s + lx);
  }
  if (threadIdx.x == 0)
    PT[G.pt[m] + ((long long)jb.z * G.by[m] + jb.y) * G.bx[m] + jb.x] = jb.w;
}

// One expanded window per active brick at level l (Eq. 3, readings R23-R25, R31): window
// dims (wx, wy, wz) at origin org[j], stored with x padded to wxp.  Intensities: level l >= 1
// from the device pyramid into wvol; level 0 arrive already gathered in wvol (host side).
// Seeds: level >= 1 from the bits pyramid, level 0 from the gathered labels wseed.  Parent
// field (root: none -> 0.5) through the page tables.  Padded columns: fixed, value 0.
template <typename T>
__global__ void k_ooc_gather(const T* __restrict__ vol_l, const uint8_t* __restrict__ bits_l,
                             const uint8_t* __restrict__ wseed, int l, bool root, OocGeo G,
                             const int* __restrict__ PT, const float* __restrict__ pool, int wx,
                             int wy, int wz, int wxp, const int4* __restrict__ org, int nb,
                             T* __restrict__ wvol, uint8_t* __restrict__ fixed,
                             float* __restrict__ values, float* __restrict__ x0) {
  const long long nw = (long long)wxp * wy * wz;
  const int nx = G.nx[l], ny = G.ny[l], nz = G.nz[l];
  const int pl = wxp * wy;
  for (long long jp = blockIdx.x; jp < (long long)nb * wz; jp += gridDim.x) {
    const int j = (int)(jp / wz), lz = (int)(jp % wz);
    const int4 o = org[j];
    for (int t = threadIdx.x; t < pl; t += blockDim.x) {
      const int lx = t % wxp, ly = t / wxp;
      const long long i = (long long)j * nw + (long long)lz * pl + t;
      if (lx >= wx) {                       // x padding (k_ooc_wfix cuts its edges)
        if (vol_l) wvol[i] = T(0);
        fixed[i] = 1;
        values[i] = 0.f;
        x0[i] = 0.f;
        continue;
      }
      const int x = o.x + lx, y = o.y + ly, z = o.z + lz;
      const long long g = ((long long)z * ny + y) * nx + x;
      uint8_t b;
      if (vol_l) {
        wvol[i] = vol_l[g];
        b = bits_l[g];
      } else {
        const uint8_t sv = wseed[i];
        b = (sv == 1 ? 1 : 0) | (sv == 2 ? 2 : 0);
      }
      bool fx = (b == 1 || b == 2);                       // exactly one of fg / bg (R22)
      float v = b == 1 ? 1.f : 0.f;
      const float ps = root ? 0.5f : ooc::sample_up(G, PT, pool, l, z, y, x);
      if (!fx) {
        const bool shell = (lx == 0 && o.x > 0) || (lx == wx - 1 && o.x + wx < nx) ||
                           (ly == 0 && o.y > 0) || (ly == wy - 1 && o.y + wy < ny) ||
                           (lz == 0 && o.z > 0) || (lz == wz - 1 && o.z + wz < nz);
        if (shell) {
          fx = true;
          v = ps;
        }
      }
      fixed[i] = fx ? 1 : 0;
      values[i] = fx ? v : 0.f;
      x0[i] = ps;
    }
  }
}

// padded windows: the +x edge of the last real column (to the padding) gets weight 0
__global__ void k_ooc_wfix(float* __restrict__ W, int nb, int wx, int wy, int wz, int wxp) {
  const long long rows = (long long)nb * wz * wy;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows;
       r += (long long)gridDim.x * blockDim.x)
    W[r * wxp + wx - 1] = 0.f;          // W_x plane: [B][wz][wy][wxp]
}

// N^-1 (Eq. 3): the brick core of window j into its pool slot + min / max / conflict ->
// state 0 keep refining, 1 hom, 2 dt, 3 seed conflict.  brick[j] =
// (bx, by, bz, slot).
__global__ void __launch_bounds__(256)
k_ooc_contract(const float* __restrict__ wprob, int wx, int wy, int wz, int wxp,
               const int4* __restrict__ org, const int4* __restrict__ brick, int l, OocGeo G,
               const uint8_t* __restrict__ bits_l, int* __restrict__ PT,
               float* __restrict__ pool, float t_hom, float t_bin, int prune,
               int* __restrict__ state) {
  __shared__ float smn[8], smx[8];
  __shared__ int scf[8];
  const int j = blockIdx.x;
  const int4 o = org[j], b = brick[j];
  const int s = G.s;
  const long long nw = (long long)wxp * wy * wz;
  const float* wp = wprob + (long long)j * nw;
  const int cx = min(s, G.nx[l] - b.x * s), cy = min(s, G.ny[l] - b.y * s),
            cz = min(s, G.nz[l] - b.z * s);
  const long long s3 = (long long)s * s * s;
  float* dst = pool + (long long)b.w * s3;
  float mn = 1e30f, mx = -1e30f;
  int cf = 0;
  const int nc = cx * cy * cz;
  for (int t = threadIdx.x; t < nc; t += blockDim.x) {
    const int lx = t % cx, ly = (t / cx) % cy, lz = t / (cx * cy);
    const int x = b.x * s + lx, y = b.y * s + ly, z = b.z * s + lz;
    const float v = wp[((long long)(z - o.z) * wy + (y - o.y)) * wxp + (x - o.x)];
    dst[((long long)lz * s + ly) * s + lx] = v;
    mn = fminf(mn, v);
    mx = fmaxf(mx, v);
    if (bits_l) cf |= bits_l[((long long)z * G.ny[l] + y) * G.nx[l] + x] == 3;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, off));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    cf |= __shfl_xor_sync(0xffffffffu, cf, off);
  }
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { smn[warp] = mn; smx[warp] = mx; scf[warp] = cf; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      mn = fminf(mn, smn[w]);
      mx = fmaxf(mx, smx[w]);
      cf |= scf[w];
    }
    int st = 0;
    if (cf) st = 3;
    else if (prune && t_hom >= 0.f && mx - mn < t_hom) st = 1;
    else if (prune && t_bin >= 0.f && (mn - 0.5f > t_bin || 0.5f - mx > t_bin)) st = 2;
    state[j] = st;
    PT[G.pt[l] + ((long long)b.z * G.by[l] + b.y) * G.bx[l] + b.x] = b.w;
  }
}

// Output slab of level m over planes [z0, z0 + zc): pool values where the brick is
// materialised, else the upsample of the level-(m+1) slab buffer `par` (planes from pz0).
// Level 0 also writes u8 labels (p > 0.5, reading R10) when `lab` is set.
__global__ void k_ooc_out(int m, OocGeo G, const int* __restrict__ PT,
                          const float* __restrict__ pool, const float* __restrict__ par,
                          int pz0, int z0, int zc, float* __restrict__ out,
                          uint8_t* __restrict__ lab) {
  const int nx = G.nx[m], ny = G.ny[m], s = G.s;
  const long long n = (long long)zc * ny * nx;
  const long long s3 = (long long)s * s * s;
  const int p = m + 1;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % nx), y = (int)((i / nx) % ny), z = z0 + (int)(i / ((long long)nx * ny));
    const int bz = z / s, by = y / s, bx = x / s;
    const int slot = PT[G.pt[m] + ((long long)bz * G.by[m] + by) * G.bx[m] + bx];
    float v;
    if (slot >= 0) {
      v = pool[slot * s3 + ((long long)(z - bz * s) * s + (y - by * s)) * s + (x - bx * s)];
    } else {
      int z0_, z1_, y0, y1, x0, x1;
      float fz, fy, fx;
      ooc::pcoord(z, G.nz[p], z0_, z1_, fz);
      ooc::pcoord(y, G.ny[p], y0, y1, fy);
      ooc::pcoord(x, G.nx[p], x0, x1, fx);
      const int pnx = G.nx[p], pny = G.ny[p];
      auto P = [&](int a, int b, int c) {
        return par[((long long)(a - pz0) * pny + b) * pnx + c];
      };
      const float c00 = __fmaf_rn(fx, P(z0_, y0, x1), (1.f - fx) * P(z0_, y0, x0));
      const float c01 = __fmaf_rn(fx, P(z0_, y1, x1), (1.f - fx) * P(z0_, y1, x0));
      const float c10 = __fmaf_rn(fx, P(z1_, y0, x1), (1.f - fx) * P(z1_, y0, x0));
      const float c11 = __fmaf_rn(fx, P(z1_, y1, x1), (1.f - fx) * P(z1_, y1, x0));
      const float c0 = __fmaf_rn(fy, c01, (1.f - fy) * c00);
      const float c1 = __fmaf_rn(fy, c11, (1.f - fy) * c10);
      v = __fmaf_rn(fz, c1, (1.f - fz) * c0);
    }
    if (out) out[i] = v;
    if (lab) lab[i] = v > 0.5f ? 1 : 0;
  }
}

static int grid_n(long long n, int sms) {
  long long g = (n + 255) / 256;
  const long long cap = (long long)sms * 16;
  return (int)(g < cap ? (g < 1 ? 1 : g) : cap);
}

cudaError_t launch_ooc_seedor0(const uint8_t* seeds, int z0, int nzs, const OocGeo& G,
                               uint8_t* out, int sms, cudaStream_t s) {
  const long long n = (long long)((z0 + nzs + 1) / 2 - z0 / 2) * G.ny[1] * G.nx[1];
  k_ooc_seedor0<<<grid_n(n, sms), 256, 0, s>>>(seeds, z0, nzs, G, out);
  return cudaGetLastError();
}

cudaError_t launch_ooc_remap(uint8_t* seeds, long long n, int cls, int sms, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_ooc_remap<<<grid_n((n + 3) / 4, sms), 256, 0, s>>>(seeds, n, cls);
  return cudaGetLastError();
}

cudaError_t launch_ooc_seedor(const uint8_t* in, int m, const OocGeo& G, uint8_t* out, int sms,
                              cudaStream_t s) {
  const long long n = (long long)G.nz[m + 1] * G.ny[m + 1] * G.nx[m + 1];
  k_ooc_seedor<<<grid_n(n, sms), 256, 0, s>>>(in, m, G, out);
  return cudaGetLastError();
}

cudaError_t launch_ooc_materialize(const int4* jobs, int nj, int m, const OocGeo& G, int* PT,
                                   float* pool, cudaStream_t s) {
  if (nj <= 0) return cudaSuccess;
  k_ooc_materialize<<<nj, 256, 0, s>>>(jobs, m, G, PT, pool);
  return cudaGetLastError();
}

cudaError_t launch_ooc_gather(const void* vol_l, int dtype, const uint8_t* bits_l,
                              const uint8_t* wseed, int l, bool root, const OocGeo& G,
                              const int* PT, const float* pool, int wx, int wy, int wz, int wxp,
                              const int4* org, int nb, void* wvol, uint8_t* fixed, float* values,
                              float* x0, int sms, cudaStream_t s) {
  long long rows = (long long)nb * wz;
  const long long cap = (long long)sms * 8;
  const int grid = (int)(rows < cap ? (rows < 1 ? 1 : rows) : cap);
  switch (dtype) {
    case 0: k_ooc_gather<uint8_t><<<grid, 256, 0, s>>>((const uint8_t*)vol_l, bits_l, wseed, l, root, G, PT, pool, wx, wy, wz, wxp, org, nb, (uint8_t*)wvol, fixed, values, x0); break;
    case 1: k_ooc_gather<uint16_t><<<grid, 256, 0, s>>>((const uint16_t*)vol_l, bits_l, wseed, l, root, G, PT, pool, wx, wy, wz, wxp, org, nb, (uint16_t*)wvol, fixed, values, x0); break;
    case 2: k_ooc_gather<int16_t><<<grid, 256, 0, s>>>((const int16_t*)vol_l, bits_l, wseed, l, root, G, PT, pool, wx, wy, wz, wxp, org, nb, (int16_t*)wvol, fixed, values, x0); break;
    default: k_ooc_gather<float><<<grid, 256, 0, s>>>((const float*)vol_l, bits_l, wseed, l, root, G, PT, pool, wx, wy, wz, wxp, org, nb, (float*)wvol, fixed, values, x0); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_ooc_wfix(float* W, int nb, int wx, int wy, int wz, int wxp, int sms,
                            cudaStream_t s) {
  k_ooc_wfix<<<grid_n((long long)nb * wz * wy, sms), 256, 0, s>>>(W, nb, wx, wy, wz, wxp);
  return cudaGetLastError();
}

cudaError_t launch_ooc_contract(const float* wprob, int wx, int wy, int wz, int wxp,
                                const int4* org, const int4* brick, int nb, int l,
                                const OocGeo& G, const uint8_t* bits_l, int* PT, float* pool,
                                float t_hom, float t_bin, int prune, int* state, cudaStream_t s) {
  k_ooc_contract<<<nb, 256, 0, s>>>(wprob, wx, wy, wz, wxp, org, brick, l, G, bits_l, PT, pool,
                                    t_hom, t_bin, prune, state);
  return cudaGetLastError();
}

cudaError_t launch_ooc_out(int m, const OocGeo& G, const int* PT, const float* pool,
                           const float* par, int pz0, int z0, int zc, float* out, uint8_t* lab,
                           int sms, cudaStream_t s) {
  const long long n = (long long)zc * G.ny[m] * G.nx[m];
  k_ooc_out<<<grid_n(n, sms), 256, 0, s>>>(m, G, PT, pool, par, pz0, z0, zc, out, lab);
  return cudaGetLastError();
}

}  // namespace rw
