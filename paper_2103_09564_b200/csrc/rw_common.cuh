// rw_common.cuh -- shared host/device definitions of librw (sm_100a).
//
// Layout (include/rw.h): idx = ((r*B + b)*nz + z)*ny*nx + y*nx + x, nx % 4 == 0.
// Tiling: every per-brick kernel of the CG path works on "units": a box of
// TX x TY columns x ZC planes of one brick.  A CTA covers the TX x TY columns (tpx
// threads along x, each owning 4 consecutive voxels = one float4, TY rows) and marches
// over the ZC planes.  Per-brick dot products are reduced to one fp64 partial per
// (unit, quantity); consumers sum the U partials of a brick in a fixed order, so results
// are deterministic and independent of the batch (a brick solved alone or in a batch of
// 512 gives identical bits).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define RW_MAX_THREADS 256

namespace rw {

// Weight source of the CG operator: stored fp32 planes (W given by the caller, or a
// dtype/shape the TMA boxes cannot carry) or recomputed from the intensities each pass.
enum { VM_STORED = 0, VM_U8 = 1, VM_U16 = 2, VM_I16 = 3, VM_F32 = 4 };

struct Plan {
  int nx, ny, nz;
  long long n;          // voxels per brick
  int B, R;             // bricks, right-hand sides
  int threads;          // CTA size of the CG kernels
  int tpx, TX, TY, ZC;  // threads along x, tile extents
  int hx, TXh;          // x halo offset of fp32 TMA boxes (0 when TX == nx, else 4), TX + 2 hx
  int hxv, TXhv;        // same for the intensity box: 16 B / element size (TMA box starts
                        // must be 16-byte aligned in x), TX + 2 hxv
  int tiles_x, tiles_y, tiles_z, U;
  int TXP;              // smem row pitch (floats) of p_new planes = TX + 8 (cols -1..TX)
  int vm;               // VM_* weight mode
  int one;              // 1: one-pass CG (pass A only, see passA.cu), 0: passes A + B
  int rc;               // right-hand sides per pass-A CTA (0: automatic, passA_rc)
  int ns;               // pass-A TMA ring depth (0: kStages; passA_stages)
  int pf;               // pass-A L2 prefetch distance in planes beyond the ring (0: off)
  int lastdec;          // one-pass mode, large bricks (U >= kLastDecMinU): the last CTA of a
                        // (rhs, brick) to finish pass k sums the U partials once and stores the
                        // decision of pass k+1 (Bufs.SD) instead of every CTA of pass k+1
                        // re-summing them (same sums, same order: bit-identical)
};

// U from which the last-CTA decision is used (api.cu; env RW_LASTDEC_MIN_U overrides)
constexpr int kLastDecMinU = 16;

// Per-(rhs,brick) status (0 = active); values match include/rw.h RW_ST_*.
enum { ST_ACTIVE = 0, ST_CONVERGED = 1, ST_MAXITER = 2, ST_TRIVIAL = 3, ST_ZERO_B = 4,
       ST_BREAKDOWN = 5 };

struct Bufs {
  const float* W;     // [3][B][n] (VM_STORED) or null
  const void* vol;    // [B][n] intensities (VM_U8..VM_F32) or null
  const float* dinv;  // [B][n]  (0 on fixed voxels)
  const uint8_t* fixed;  // [B][n]
  const float* values;   // [R][B][n]
  const float* x0;       // [R][B][n] or null
  float* x;           // [R][B][n]   iterate (aliases the prob output)
  float* r;           // [2][R][B][n] (two-pass mode uses slot 0 only; one-pass: R[k&1]
                      //               holds r_{k-1} at the start of iteration k)
  float* p;           // [2][R][B][n]  P[k&1] holds p_{k-1} at the start of iteration k
  float* q;           // [2][R][B][n]  (as r)
  double* PA;         // [2][R*B][U][5] p.q partials (slot k&1 written by pass A(k)); one-pass
                      //               mode: (r.z, r.r, p.q, q.D r, q.D q) of iteration k
  double2* PB;        // [2][R*B][U]       (r.z, r.r) partials (slot k&1 = state k)
  double4* PS;        // [R*B][U]          (b.b, n_fixed, n_unknown, 0) from setup
  int* status;        // [R*B]
  int* iters;         // [R*B]
  int* ctr;           // [4]: [0..1] active (rhs,brick) count per iteration parity,
                      //      [2] resident brick counter, [3] iteration index (device loop)
  const int* kdev;    // device-driven loop: pass A reads its iteration index here (ctr + 3);
                      // null: the index is the kernel argument (host-driven loop)
  float4* SD;         // [2][R*B] (Plan.lastdec) decision of pass k in slot k&1: (alpha, beta)
  int* cnt;           // [R*B]    (Plan.lastdec) CTAs of pass k done with their partials
};

struct Ctl {
  float tol;
  int tol_mode;
  int max_iter;
  float scale, offset, nbl2, eps;  // normalisation + weights (nbl2 = -beta log2 e)
  int noxlag;       // pass A: the lagged x update was already applied (residual replacement)
  int rr;           // residual replacement interval (0: off): after pass B(k) with
                    // (k+1) % rr == 0 and k < max_iter-1, alpha_k p_k is already in x
};

// Geometry of the out-of-core hierarchical driver (hier_ooc.cu, reading R31): per level the
// dims, the bricks per axis and the offset of the level's page table.
struct OocGeo {
  int nx[17], ny[17], nz[17];      // level dims
  int bx[17], by[17], bz[17];      // bricks per axis
  long long pt[17];                // page-table offset of each level
  int s, k;                        // brick side, root level
};

// Outputs of one fused pyramid group (<= 5 levels).
struct PyrOut {
  void* p[5];
  int nx[5], ny[5], nz[5];
};

__host__ __device__ inline long long vidx(const Plan& P, int rb, int z, int y, int x) {
  return ((long long)rb * P.nz + z) * (long long)P.ny * P.nx + (long long)y * P.nx + x;
}

// a1: g = clamp(v*scale + offset, 0, 1) in fp32 (reading c2)
__device__ __forceinline__ float normv(float v, float s, float o) {
  return fminf(fmaxf(__fmaf_rn(v, s, o), 0.f), 1.f);
}

// a2 (P:77 + reading c1): w = exp(-beta d^2) + eps with d = g[v + e_a] - g[v], evaluated
// as 2^(d^2 * nbl2) + eps with nbl2 = -beta * log2(e) rounded once on the host, on the
// MUFU ex2 unit (ex2.approx.ftz: ~2 ulp; results below 2^-126 flush to 0, i.e. w = eps,
// which differs from the exact weight by < 1e-38).  Every kernel that needs a weight
// evaluates exactly this expression on the same operands, so a weight recomputed on the
// fly is bit-identical to the stored one.
__device__ __forceinline__ float ex2_approx(float a) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}
__device__ __forceinline__ float grady(float d, float nbl2, float eps) {
  return __fadd_rn(ex2_approx(__fmul_rn(__fmul_rn(d, d), nbl2)), eps);
}
inline float nbl2_of(float beta) { return (float)(-(double)beta * 1.4426950408889634); }

template <int VM> struct VolT;
template <> struct VolT<VM_U8> { using T = uint8_t; };
template <> struct VolT<VM_U16> { using T = uint16_t; };
template <> struct VolT<VM_I16> { using T = int16_t; };
template <> struct VolT<VM_F32> { using T = float; };
template <> struct VolT<VM_STORED> { using T = float; };

}  // namespace rw
