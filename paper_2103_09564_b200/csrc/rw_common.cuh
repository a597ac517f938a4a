// rw_common.cuh -- shared host/device definitions of librw (sm_100a).
//
// Layout (include/rw.h): idx = ((r*B + b)*nz + z)*ny*nx + y*nx + x, nx % 4 == 0.
// Tiling: every per-brick kernel of the CG path works on "units": a box of
// TX x TY columns x ZC planes of one brick.  A CTA of 256 threads covers the TX x TY
// columns (tpx threads along x, each owning 4 consecutive voxels = one float4) and
// marches over the ZC planes.  Per-brick dot products are reduced to one fp64 partial
// per (unit, quantity); consumers sum the U partials of a brick in a fixed order, so
// results are deterministic and independent of the batch (a brick solved alone or in
// a batch of 512 gives identical bits).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define RW_THREADS 256

namespace rw {

struct Plan {
  int nx, ny, nz;
  long long n;          // voxels per brick
  int B, R;             // bricks, right-hand sides
  int tpx, TX, TY, ZC;  // threads along x, tile extents
  int tiles_x, tiles_y, tiles_z, U;
  int TXP;              // smem row pitch (floats) = TX + 8 (col -1 .. TX, aligned)
};

// Per-(rhs,brick) status (0 = active); values match include/rw.h RW_ST_*.
enum { ST_ACTIVE = 0, ST_CONVERGED = 1, ST_MAXITER = 2, ST_TRIVIAL = 3, ST_ZERO_B = 4,
       ST_BREAKDOWN = 5 };

struct Bufs {
  const float* W;     // [3][B][n]
  const float* dinv;  // [B][n]  (0 on fixed voxels)
  const uint8_t* fixed;  // [B][n]
  const float* values;   // [R][B][n]
  const float* x0;       // [R][B][n] or null
  float* x;           // [R][B][n]   iterate (aliases the prob output)
  float* r;           // [R][B][n]
  float* p0;          // [R][B][n]   p buffers: P[k&1] holds p_{k-1} at the start of it. k
  float* p1;
  float* q;           // [R][B][n]
  double* PA;         // [2][R*B][U]       p.q partials (slot k&1 written by pass A(k))
  double2* PB;        // [2][R*B][U]       (r.z, r.r) partials (slot k&1 = state k)
  double4* PS;        // [R*B][U]          (b.b, n_fixed, n_unknown, 0) from setup
  int* status;        // [R*B]
  int* iters;         // [R*B]
  int* ctr;           // [2] active (rhs,brick) count per iteration parity
};

struct Ctl {
  float tol;
  int tol_mode;
  int max_iter;
};

// Outputs of one fused pyramid group (<= 5 levels).
struct PyrOut {
  void* p[5];
  int nx[5], ny[5], nz[5];
};

__host__ __device__ inline long long vidx(const Plan& P, int rb, int z, int y, int x) {
  return ((long long)rb * P.nz + z) * (long long)P.ny * P.nx + (long long)y * P.nx + x;
}

}  // namespace rw
