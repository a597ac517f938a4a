// hier.cu -- SURVEY §8(f) row f1: device kernels of the hierarchical driver.
// The orchestration (levels, brick lists, batched solves) is rw_hier_segment in api.cu.
//
//   k_seed_bits / k_seed_or   rasterised labels -> per-level fg/bg bits (OR over the 2^3
//                             children; fg+bg = conflict; reading R22)
//   k_upsample                dense trilinear upsample of the parent level's probability
//                             field (reading R25): the starting field of every level, so
//                             pruned regions inherit their nearest solved ancestor (R26)
//   k_gather                  one expanded window N(n) per active brick (Eq. 3, reading R23):
//                             intensities, user seeds, continuous border seeds sampled from the
//                             parent field on window faces interior to the volume (R24),
//                             initial guess = parent field
//   k_contract                N^-1: the brick's s^3 of the window solution into the level
//                             field + min / max / conflict -> prunable
#include <cstdlib>

#include "rw_common.cuh"

namespace rw {

namespace hier {

// parent-voxel coordinate of child voxel centre i, clamped: u = (i + 0.5)/2 - 0.5
__device__ __forceinline__ void pcoord(int i, int np, int& i0, int& i1, float& f) {
  float u = fminf(fmaxf(0.5f * (float)i - 0.25f, 0.f), (float)(np - 1));
  i0 = (int)floorf(u);
  i1 = min(i0 + 1, np - 1);
  f = u - (float)i0;
}

// trilinear sample of the parent field P (np^3) at child voxel (z, y, x)
__device__ __forceinline__ float sample(const float* __restrict__ P, int np, int z, int y, int x) {
  int z0, z1, y0, y1, x0, x1;
  float fz, fy, fx;
  pcoord(z, np, z0, z1, fz);
  pcoord(y, np, y0, y1, fy);
  pcoord(x, np, x0, x1, fx);
  const long long pl = (long long)np * np;
  auto at = [&](int a, int b, int c) { return P[(long long)a * pl + (long long)b * np + c]; };
  const float c00 = __fmaf_rn(fx, at(z0, y0, x1), (1.f - fx) * at(z0, y0, x0));
  const float c01 = __fmaf_rn(fx, at(z0, y1, x1), (1.f - fx) * at(z0, y1, x0));
  const float c10 = __fmaf_rn(fx, at(z1, y0, x1), (1.f - fx) * at(z1, y0, x0));
  const float c11 = __fmaf_rn(fx, at(z1, y1, x1), (1.f - fx) * at(z1, y1, x0));
  const float c0 = __fmaf_rn(fy, c01, (1.f - fy) * c00);
  const float c1 = __fmaf_rn(fy, c11, (1.f - fy) * c10);
  return __fmaf_rn(fz, c1, (1.f - fz) * c0);
}

}  // namespace hier

// cls == 0: labels are 0 / 1 fg / 2 bg.  cls > 0 (multi-class): class cls is the
// foreground, every other nonzero label background.  16 voxels per thread (n % 16 == 0,
// 16-byte aligned buffers: D = s 2^k with s % 4 == 0).
__device__ __forceinline__ uint32_t seed_bits4(uint32_t w, int cls) {
  uint32_t o = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int s = (w >> (8 * e)) & 0xff;
    const uint32_t b = cls == 0 ? ((s == 1 ? 1u : 0u) | (s == 2 ? 2u : 0u))
                                : (s == cls ? 1u : (s != 0 ? 2u : 0u));
    o |= b << (8 * e);
  }
  return o;
}
__global__ void k_seed_bits(const uint8_t* __restrict__ seeds, long long n, int cls,
                            uint8_t* __restrict__ bits) {
  const long long n16 = n / 16;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n16;
       i += (long long)gridDim.x * blockDim.x) {
    const uint4 v = reinterpret_cast<const uint4*>(seeds)[i];
    reinterpret_cast<uint4*>(bits)[i] =
        make_uint4(seed_bits4(v.x, cls), seed_bits4(v.y, cls), seed_bits4(v.z, cls), seed_bits4(v.w, cls));
  }
}

// running argmax over the class fields ("the class of a voxel is the one that
// maximizes the foreground probability"): strict > keeps the lowest class id on ties
__global__ void k_label_max(const float* __restrict__ P, long long n, int cls,
                            float* __restrict__ best, uint8_t* __restrict__ lab) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float p = P[i];
    if (cls == 1 || p > best[i]) {
      best[i] = p;
      lab[i] = (uint8_t)cls;
    }
  }
}

// level l (D^3) -> level l+1 ((D/2)^3): OR of the 2^3 children.  One block-stride loop over
// output rows (z, y); a thread ORs 4 outputs from 8-byte loads of the 4 child rows
// (D % 8 == 0 whenever a coarser level exists).
__global__ void k_seed_or(const uint8_t* __restrict__ in, int D, uint8_t* __restrict__ out) {
  const int h = D / 2, hq = h / 4;
  for (long long row = blockIdx.x; row < (long long)h * h; row += gridDim.x) {
    const int z = (int)(row / h), y = (int)(row % h);
    for (int g = threadIdx.x; g < hq; g += blockDim.x) {
      uint32_t acc = 0;
#pragma unroll
      for (int dz = 0; dz < 2; ++dz)
#pragma unroll
        for (int dy = 0; dy < 2; ++dy) {
          const uint2 v = *reinterpret_cast<const uint2*>(
              in + ((long long)(2 * z + dz) * D + (2 * y + dy)) * D + 8 * g);
          // output byte e = OR of input bytes 2e, 2e+1
          const uint32_t a = v.x | (v.x >> 8), b = v.y | (v.y >> 8);
          acc |= (a & 0xffu) | ((a >> 8) & 0xff00u) | ((b & 0xffu) << 16) | ((b & 0xff0000u) << 8);
        }
      reinterpret_cast<uint32_t*>(out + row * h)[g] = acc;
    }
  }
}

// Dense trilinear upsample (reading R25), one block-stride loop over output rows: the parent
// coordinates of the row (z, y) are computed once, a thread writes 4 consecutive outputs
// with one 16-byte store.  Same arithmetic as hier::sample (bit-identical values).
__global__ void k_upsample(const float* __restrict__ P, int np, float* __restrict__ out, int D) {
  const long long pl = (long long)np * np;
  const int h = D / 2;
  // quads of output rows (2Z..2Z+1) x (2Y..2Y+1): their 16 parent-row reads touch 9
  // distinct rows, so a block reuses them from L1 (row-by-row order re-read each parent row
  // from DRAM ~5 times at 2048^3: 23 GB for a 4.3 GB parent level, 30 % L2 hit rate)
  for (long long quad = blockIdx.x; quad < (long long)h * h; quad += gridDim.x)
  for (int sub = 0; sub < 4; ++sub) {
    const int z = 2 * (int)(quad / h) + (sub >> 1), y = 2 * (int)(quad % h) + (sub & 1);
    const long long row = (long long)z * D + y;
    int z0, z1, y0, y1;
    float fz, fy;
    hier::pcoord(z, np, z0, z1, fz);
    hier::pcoord(y, np, y0, y1, fy);
    const float* r00 = P + (long long)z0 * pl + (long long)y0 * np;
    const float* r01 = P + (long long)z0 * pl + (long long)y1 * np;
    const float* r10 = P + (long long)z1 * pl + (long long)y0 * np;
    const float* r11 = P + (long long)z1 * pl + (long long)y1 * np;
    const float* rr[4] = {r00, r01, r10, r11};
    for (int g = threadIdx.x; g < D / 4; g += blockDim.x) {
      float o[4];
      if (g > 0 && 2 * g + 2 <= np - 1) {
        // interior: outputs 4g..4g+3 use parents 2g-1..2g+2 with (x0, x1, fx) =
        // (2g-1, 2g, .75), (2g, 2g+1, .25), (2g, 2g+1, .75), (2g+1, 2g+2, .25) -- exactly
        // what pcoord gives; three 8-byte loads per parent row instead of eight scalars
        float c[4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 a = *reinterpret_cast<const float2*>(rr[q] + 2 * g - 2);
          const float2 b = *reinterpret_cast<const float2*>(rr[q] + 2 * g);
          const float2 d = *reinterpret_cast<const float2*>(rr[q] + 2 * g + 2);
          c[q][0] = __fmaf_rn(0.75f, b.x, (1.f - 0.75f) * a.y);
          c[q][1] = __fmaf_rn(0.25f, b.y, (1.f - 0.25f) * b.x);
          c[q][2] = __fmaf_rn(0.75f, b.y, (1.f - 0.75f) * b.x);
          c[q][3] = __fmaf_rn(0.25f, d.x, (1.f - 0.25f) * b.y);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float c0 = __fmaf_rn(fy, c[1][e], (1.f - fy) * c[0][e]);
          const float c1 = __fmaf_rn(fy, c[3][e], (1.f - fy) * c[2][e]);
          o[e] = __fmaf_rn(fz, c1, (1.f - fz) * c0);
        }
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          int x0, x1;
          float fx;
          hier::pcoord(4 * g + e, np, x0, x1, fx);
          const float c00 = __fmaf_rn(fx, r00[x1], (1.f - fx) * r00[x0]);
          const float c01 = __fmaf_rn(fx, r01[x1], (1.f - fx) * r01[x0]);
          const float c10 = __fmaf_rn(fx, r10[x1], (1.f - fx) * r10[x0]);
          const float c11 = __fmaf_rn(fx, r11[x1], (1.f - fx) * r11[x0]);
          const float c0 = __fmaf_rn(fy, c01, (1.f - fy) * c00);
          const float c1 = __fmaf_rn(fy, c11, (1.f - fy) * c10);
          o[e] = __fmaf_rn(fz, c1, (1.f - fz) * c0);
        }
      }
      // streaming (evict-first) store: the 34 GB output of a 2048^3 level would otherwise push
      // the parent rows out of L2 (ncu: 23 GB of parent re-reads, 30 % L2 hit rate)
      __stcs(reinterpret_cast<float4*>(out + row * D) + g, make_float4(o[0], o[1], o[2], o[3]));
    }
  }
}

// Dense trilinear upsample of a large level as a z walk (same values as k_upsample /
// hier::sample, bit for bit: per output the same three fma in the order x, y, z).
// A work item is (z chunk, quad column Y, x segment): its threads own 4 consecutive output x
// each and walk the parent planes p of the chunk.  A plane costs 3 parent-row reads (4 in the
// clamped first / last column), one x-interpolation per row and one y-interpolation per output
// row pair; with the previous plane's result carried in registers every step then emits the
// output rows z = 2p-1 (f = .25) and z = 2p (f = .75), which both blend planes p-1 and p.
// Against k_upsample (every output row re-reads and re-interpolates its 4 parent rows:
// 44 instructions per output, 21 GB of DRAM reads for a 4.3 GB parent level, 18.1 ms for a
// 2048^3 level, profiles/r02/r02_j_upsample.md) this is 15 instructions per output, 5.5 GB of
// DRAM reads and 7.8 ms (5.1 TB/s) with the next plane's loads in flight during a step.
// the 4 parent values a thread's 4 outputs can touch in one parent row: x = 2g-1 .. 2g+2,
// clamped into the row (x = a, y, z, w = d)
__device__ __forceinline__ float4 up_raw(const float* __restrict__ r, int g, int np) {
  const float2 bc = *reinterpret_cast<const float2*>(r + 2 * g);
  return make_float4(r[max(2 * g - 1, 0)], bc.x, bc.y, r[min(2 * g + 2, np - 1)]);
}
__device__ __forceinline__ void up_xrow(const float4 v, int g, int np, bool xin, float (&c)[4]) {
  if (xin) {
    c[0] = __fmaf_rn(0.75f, v.y, (1.f - 0.75f) * v.x);
    c[1] = __fmaf_rn(0.25f, v.z, (1.f - 0.25f) * v.y);
    c[2] = __fmaf_rn(0.75f, v.z, (1.f - 0.75f) * v.y);
    c[3] = __fmaf_rn(0.25f, v.w, (1.f - 0.25f) * v.z);
  } else {   // first / last group of the row: clamped parent coordinates, as hier::sample
    auto pick = [&](int x) {
      const int k = x - (2 * g - 1);
      return k <= 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
    };
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int x0, x1;
      float fx;
      hier::pcoord(4 * g + e, np, x0, x1, fx);
      // g = 0: x0 = 0 is v.y (k = 1); v.x holds the clamped duplicate of the same value
      c[e] = __fmaf_rn(fx, pick(x1), (1.f - fx) * pick(x0));
    }
  }
}

__global__ void __launch_bounds__(256, 3)
k_upsample_walk(const float* __restrict__ P, int np, float* __restrict__ out, int D, int zsplit) {
  const long long pl = (long long)np * np;
  const int h = D / 2, G = D / 4;
  const int nxs = (G + (int)blockDim.x - 1) / (int)blockDim.x;
  const int pzc = (np + zsplit - 1) / zsplit;          // parent planes per z chunk
  const long long items = (long long)zsplit * h * nxs;
  for (long long it = blockIdx.x; it < items; it += gridDim.x) {
    const int xs = (int)(it % nxs), Yq = (int)((it / nxs) % h), zc = (int)(it / ((long long)nxs * h));
    const int g = xs * (int)blockDim.x + (int)threadIdx.x;
    const int pa = zc * pzc, pb = min(np, pa + pzc);
    if (g >= G || pa >= pb) continue;
    int y0[2], y1[2];
    float fy[2];
    hier::pcoord(2 * Yq, np, y0[0], y1[0], fy[0]);
    hier::pcoord(2 * Yq + 1, np, y0[1], y1[1], fy[1]);
    const bool ydup = y1[0] == y0[1];                  // interior column: 3 distinct parent rows
    const bool xin = g > 0 && 2 * g + 2 <= np - 1;
    const float* r0 = P + (long long)y0[0] * np;
    const float* r1 = P + (long long)y1[0] * np;
    const float* r2 = P + (long long)y0[1] * np;
    const float* r3 = P + (long long)y1[1] * np;
    // raw parent values of plane p (the loads of plane p+1 are issued before plane p is
    // interpolated, so a thread always has one plane in flight)
    auto load = [&](int p, float4 (&R)[4]) {
      const long long o = (long long)p * pl;
      R[0] = up_raw(r0 + o, g, np);
      R[1] = up_raw(r1 + o, g, np);
      if (!ydup) R[2] = up_raw(r2 + o, g, np);
      R[3] = up_raw(r3 + o, g, np);
    };
    // y-interpolated x-interpolations of a parent plane for the two output rows 2Yq, 2Yq+1
    auto plane = [&](const float4 (&R)[4], float (&cy)[2][4]) {
      float c0[4], c1[4], c2[4], c3[4];
      up_xrow(R[0], g, np, xin, c0);
      up_xrow(R[1], g, np, xin, c1);
      if (ydup) {
#pragma unroll
        for (int e = 0; e < 4; ++e) c2[e] = c1[e];
      } else {
        up_xrow(R[2], g, np, xin, c2);
      }
      up_xrow(R[3], g, np, xin, c3);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        cy[0][e] = __fmaf_rn(fy[0], c1[e], (1.f - fy[0]) * c0[e]);
        cy[1][e] = __fmaf_rn(fy[1], c3[e], (1.f - fy[1]) * c2[e]);
      }
    };
    // output plane z from the planes lo = pcoord(z).i0 and hi = pcoord(z).i1
    auto emit = [&](int z, const float (&lo)[2][4], const float (&hi)[2][4]) {
      int z0, z1;
      float fz;
      hier::pcoord(z, np, z0, z1, fz);
#pragma unroll
      for (int ys = 0; ys < 2; ++ys) {
        float o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) o[e] = __fmaf_rn(fz, hi[ys][e], (1.f - fz) * lo[ys][e]);
        const long long row = (long long)z * D + (2 * Yq + ys);
        __stcs(reinterpret_cast<float4*>(out + row * D) + g, make_float4(o[0], o[1], o[2], o[3]));
      }
    };
    float prev[2][4], cur[2][4];
    float4 Rc[4], Rn[4];
    const int p0 = max(pa, 1) - 1;
    load(p0, Rc);
    if (p0 + 1 < pb) load(p0 + 1, Rn);
    plane(Rc, prev);
    for (int p = p0 + 1; p < pb; ++p) {
#pragma unroll
      for (int i = 0; i < 4; ++i) Rc[i] = Rn[i];
      if (p + 1 < pb) load(p + 1, Rn);
      plane(Rc, cur);
      if (p == 1) emit(0, prev, cur);                  // z = 0: planes (0, 1), f = 0
      emit(2 * p - 1, prev, cur);                      // planes (p-1, p), f = .25
      emit(2 * p, prev, cur);                          // planes (p-1, p), f = .75
#pragma unroll
      for (int ys = 0; ys < 2; ++ys)
#pragma unroll
        for (int e = 0; e < 4; ++e) prev[ys][e] = cur[ys][e];
    }
    if (pb == np) emit(D - 1, prev, prev);             // z = D-1: plane np-1 twice, f = 0
  }
}

// Window w of active brick list entry j: origin org[j] (level voxels), side se.
template <typename T>
__global__ void k_gather(const T* __restrict__ vol, const uint8_t* __restrict__ bits,
                         const float* __restrict__ Ppar, const float* __restrict__ Pold, int D,
                         int se, const int4* __restrict__ org, int nb, T* __restrict__ wvol,
                         uint8_t* __restrict__ fixed, float* __restrict__ values,
                         float* __restrict__ x0) {
  const long long nw = (long long)se * se * se;
  const int np = D / 2, pl = se * se;
  // one block-stride loop over (window, plane) pairs; threads over the plane (32-bit math)
  for (long long jp = blockIdx.x; jp < (long long)nb * se; jp += gridDim.x) {
   const int j = (int)(jp / se), lz = (int)(jp % se);
   const int4 o = org[j];
   for (int t = threadIdx.x; t < pl; t += blockDim.x) {
    const int lx = t % se, ly = t / se;
    const long long i = (long long)j * nw + (long long)lz * pl + t;
    const int x = o.x + lx, y = o.y + ly, z = o.z + lz;
    const long long g = ((long long)z * D + y) * D + x;
    wvol[i] = vol[g];
    const uint8_t b = bits[g];
    bool fx = (b == 1 || b == 2);                       // exactly one of fg / bg (R22)
    float v = b == 1 ? 1.f : 0.f;
    const float ps = Ppar ? hier::sample(Ppar, np, z, y, x) : 0.5f;   // root: x0 = 0.5
    if (!fx) {
      // continuous border seed on window faces interior to the volume (R24)
      const bool shell = (lx == 0 && o.x > 0) || (lx == se - 1 && o.x + se < D) ||
                         (ly == 0 && o.y > 0) || (ly == se - 1 && o.y + se < D) ||
                         (lz == 0 && o.z > 0) || (lz == se - 1 && o.z + se < D);
      if (shell) {
        fx = true;
        v = ps;
      }
    }
    fixed[i] = fx ? 1 : 0;
    values[i] = fx ? v : 0.f;
    x0[i] = Pold ? Pold[g] : ps;   // incremental: the previous solution
   }
  }
}

// One CTA per brick: decide the brick's fate and write its s^3 into the level field.
// state: 0 keep refining, 1 hom, 2 dt, 3 seed conflict (vetoes pruning),
// 4 reused (incremental H_it: the previous node was computed, max |new - old| < t_inc over
// the s^3 and no conflict involving a changed label; the old values stay).
__global__ void __launch_bounds__(256)
k_contract(const float* __restrict__ wprob, int se, const int4* __restrict__ org,
           const int4* __restrict__ brick, int s, int D, const uint8_t* __restrict__ bits,
           const uint8_t* __restrict__ obits, float* __restrict__ P, float t_hom, float t_bin,
           int prune, float t_inc, uint8_t* __restrict__ computed, int* __restrict__ state,
           float2* __restrict__ range) {
  __shared__ float smn[8], smx[8], sdf[8];
  __shared__ int scf[8], sdc[8];
  __shared__ int s_reuse;
  const int j = blockIdx.x;
  const int4 o = org[j], b = brick[j];
  const long long nw = (long long)se * se * se;
  const float* wp = wprob + (long long)j * nw;
  const int nbs = D / s;
  const long long bi = ((long long)b.z * nbs + b.y) * nbs + b.x;
  const bool inc = obits != nullptr;
  float mn = 1e30f, mx = -1e30f, df = 0.f;
  int cf = 0, dc = 0;
  const long long ns = (long long)s * s * s;
  auto gidx = [&](long long t, long long& wi) {
    const int bx = (int)(t % s), by = (int)((t / s) % s), bz = (int)(t / ((long long)s * s));
    const int x = b.x * s + bx, y = b.y * s + by, z = b.z * s + bz;
    wi = ((long long)(z - o.z) * se + (y - o.y)) * se + (x - o.x);
    return ((long long)z * D + y) * D + x;
  };
  for (long long t = threadIdx.x; t < ns; t += blockDim.x) {
    long long wi;
    const long long g = gidx(t, wi);
    const float v = wp[wi];
    mn = fminf(mn, v);
    mx = fmaxf(mx, v);
    const uint8_t nb = bits[g];
    cf |= nb == 3;
    if (inc) {
      df = fmaxf(df, fabsf(v - P[g]));
      dc |= (nb == 3) && (nb != obits[g]);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, off));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    df = fmaxf(df, __shfl_xor_sync(0xffffffffu, df, off));
    cf |= __shfl_xor_sync(0xffffffffu, cf, off);
    dc |= __shfl_xor_sync(0xffffffffu, dc, off);
  }
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { smn[warp] = mn; smx[warp] = mx; sdf[warp] = df; scf[warp] = cf; sdc[warp] = dc; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      mn = fminf(mn, smn[w]);
      mx = fmaxf(mx, smx[w]);
      df = fmaxf(df, sdf[w]);
      cf |= scf[w];
      dc |= sdc[w];
    }
    int st = 0;
    if (inc && computed[bi] && !dc && df < t_inc) st = 4;
    else if (cf) st = 3;
    else if (prune && t_hom >= 0.f && mx - mn < t_hom) st = 1;
    else if (prune && t_bin >= 0.f && (mn - 0.5f > t_bin || 0.5f - mx > t_bin)) st = 2;
    state[j] = st;
    range[j] = make_float2(mn, mx);
    computed[bi] = 1;
    s_reuse = st == 4;
  }
  __syncthreads();
  if (s_reuse) return;                       // the previous node and its values stay
  for (long long t = threadIdx.x; t < ns; t += blockDim.x) {
    long long wi;
    const long long g = gidx(t, wi);
    P[g] = wp[wi];
  }
}

// pruned region (H_p) in incremental mode: the brick's s^3 of the level field becomes the
// upsampled parent field and the brick no longer holds a computed node
__global__ void k_fill(const float* __restrict__ Ppar, int np, float* __restrict__ P, int D,
                       int s, const int4* __restrict__ brick, uint8_t* __restrict__ computed) {
  const int j = blockIdx.x;
  const int4 b = brick[j];
  const long long ns = (long long)s * s * s;
  for (long long t = threadIdx.x; t < ns; t += blockDim.x) {
    const int x = b.x * s + (int)(t % s), y = b.y * s + (int)((t / s) % s);
    const int z = b.z * s + (int)(t / ((long long)s * s));
    P[((long long)z * D + y) * D + x] = hier::sample(Ppar, np, z, y, x);
  }
  if (threadIdx.x == 0) {
    const int nbs = D / s;
    computed[((long long)b.z * nbs + b.y) * nbs + b.x] = 0;
  }
}

static int grid_n(long long n, int sms) {
  long long g = (n + 255) / 256;
  const long long cap = (long long)sms * 16;
  return (int)(g < cap ? (g < 1 ? 1 : g) : cap);
}

cudaError_t launch_seed_bits(const uint8_t* seeds, long long n, int cls, uint8_t* bits, int sms,
                             cudaStream_t s) {
  k_seed_bits<<<grid_n(n / 16, sms), 256, 0, s>>>(seeds, n, cls, bits);
  return cudaGetLastError();
}

static int grid_rows(long long rows, int sms) {
  const long long cap = (long long)sms * 8;
  return (int)(rows < cap ? (rows < 1 ? 1 : rows) : cap);
}

cudaError_t launch_label_max(const float* P, long long n, int cls, float* best, uint8_t* lab,
                             int sms, cudaStream_t s) {
  k_label_max<<<grid_n(n, sms), 256, 0, s>>>(P, n, cls, best, lab);
  return cudaGetLastError();
}

cudaError_t launch_seed_or(const uint8_t* in, int D, uint8_t* out, int sms, cudaStream_t s) {
  const long long h = D / 2;
  k_seed_or<<<grid_rows(h * h, sms), h / 4 < 256 ? (int)((h / 4 + 31) / 32 * 32) : 256, 0, s>>>(in, D, out);
  return cudaGetLastError();
}

cudaError_t launch_upsample(const float* P, int np, float* out, int D, int sms, cudaStream_t s) {
  const int th = D / 4 < 256 ? (D / 4 + 31) / 32 * 32 : 256;
  // levels of side >= 512: the z walk (RW_UPSAMPLE_V=0 forces the row-quad kernel, for A/B runs)
  static const int v = [] { const char* e = getenv("RW_UPSAMPLE_V"); return e ? atoi(e) : 1; }();
  const int h = D / 2;
  if (v != 0 && h >= 256) {
    // ~8 waves of work items over the 3 blocks per SM that 80 registers allow
    const int mb = 3;
    const long long cols = (long long)h * ((D / 4 + 255) / 256);
    int zsplit = (int)((8LL * sms * mb + cols - 1) / cols);
    zsplit = zsplit < 1 ? 1 : (zsplit > np / 16 ? (np / 16 < 1 ? 1 : np / 16) : zsplit);
    const long long items = cols * zsplit;
    k_upsample_walk<<<(int)(items < sms * mb ? items : sms * mb), 256, 0, s>>>(P, np, out, D, zsplit);
  } else {
    k_upsample<<<grid_rows((long long)D * D / 4, sms), th, 0, s>>>(P, np, out, D);
  }
  return cudaGetLastError();
}

cudaError_t launch_gather(const void* vol, int dtype, const uint8_t* bits, const float* Ppar,
                          const float* Pold, int D, int se, const int4* org, int nb, void* wvol,
                          uint8_t* fixed, float* values, float* x0, int sms, cudaStream_t s) {
  const int grid = grid_rows((long long)nb * se, sms);
  switch (dtype) {
    case 0: k_gather<uint8_t><<<grid, 256, 0, s>>>((const uint8_t*)vol, bits, Ppar, Pold, D, se, org, nb, (uint8_t*)wvol, fixed, values, x0); break;
    case 1: k_gather<uint16_t><<<grid, 256, 0, s>>>((const uint16_t*)vol, bits, Ppar, Pold, D, se, org, nb, (uint16_t*)wvol, fixed, values, x0); break;
    case 2: k_gather<int16_t><<<grid, 256, 0, s>>>((const int16_t*)vol, bits, Ppar, Pold, D, se, org, nb, (int16_t*)wvol, fixed, values, x0); break;
    default: k_gather<float><<<grid, 256, 0, s>>>((const float*)vol, bits, Ppar, Pold, D, se, org, nb, (float*)wvol, fixed, values, x0); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_contract(const float* wprob, int se, const int4* org, const int4* brick,
                            int nb, int s, int D, const uint8_t* bits, const uint8_t* obits,
                            float* P, float t_hom, float t_bin, int prune, float t_inc,
                            uint8_t* computed, int* state, float2* range, cudaStream_t st) {
  k_contract<<<nb, 256, 0, st>>>(wprob, se, org, brick, s, D, bits, obits, P, t_hom, t_bin,
                                 prune, t_inc, computed, state, range);
  return cudaGetLastError();
}

cudaError_t launch_fill(const float* Ppar, int np, float* P, int D, int s, const int4* brick,
                        int nb, uint8_t* computed, cudaStream_t st) {
  k_fill<<<nb, 256, 0, st>>>(Ppar, np, P, D, s, brick, computed);
  return cudaGetLastError();
}

}  // namespace rw
