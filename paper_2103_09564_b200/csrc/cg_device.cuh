// cg_device.cuh -- device helpers shared by the CG kernels (cg.cu, passA.cu).
#pragma once
#include "rw_common.cuh"

namespace rw {

// --------------------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;  // identical in every lane (a+b == b+a in IEEE)
}

// Sum of a[0..U) (stride `stride`) in a fixed order by one warp; result in all lanes.
__device__ __forceinline__ double warp_sum_array(const double* a, int U, int stride, int lane) {
  double s = 0.0;
  for (int u = lane; u < U; u += 32) s += a[(long long)u * stride];
  return warp_sum(s);
}

// As warp_sum_array, reading through L2 (partials written by other CTAs of the same launch).
__device__ __forceinline__ double warp_sum_array_cg(const double* a, int U, int stride, int lane) {
  double s = 0.0;
  for (int u = lane; u < U; u += 32) s += __ldcg(a + (long long)u * stride);
  return warp_sum(s);
}

// Block-wide fixed-order reduction of NV values per thread; result written by thread 0.
// Callers separate consecutive calls with __syncthreads().
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* out) {
  __shared__ double red[RW_MAX_THREADS / 32][NV];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = warp_sum(v[j]);
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) red[warp][j] = v[j];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += red[w][j];
      out[j] = s;
    }
  }
}

// --------------------------------------------------------------------------- tiles
struct Tile {
  int x0, y0, z0, z1, lx, ly, x, y;
  bool in;  // this thread's 4 columns exist and are inside the brick
};

__device__ __forceinline__ Tile make_tile(const Plan& P, int u) {
  Tile t;
  const int tx = u % P.tiles_x;
  const int rest = u / P.tiles_x;
  const int ty = rest % P.tiles_y;
  const int tz = rest / P.tiles_y;
  t.x0 = tx * P.TX;
  t.y0 = ty * P.TY;
  t.z0 = tz * P.ZC;
  t.z1 = min(t.z0 + P.ZC, P.nz);
  t.lx = threadIdx.x % P.tpx;
  t.ly = threadIdx.x / P.tpx;
  t.x = t.x0 + 4 * t.lx;
  t.y = t.y0 + t.ly;
  // P.threads % tpx may be != 0: threads past the TY rows own nothing
  t.in = (t.x < P.nx) && (t.y < P.ny) && (t.ly < P.TY);
  return t;
}

// --------------------------------------------------------------------------- float4 math
// explicit _rn intrinsics everywhere: no contraction freedom for the compiler, so every
// template instantiation produces the same bits
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float4 f4(float a) { return make_float4(a, a, a, a); }
__device__ __forceinline__ float4 fma4(float a, float4 x, float4 y) {
  return make_float4(__fmaf_rn(a, x.x, y.x), __fmaf_rn(a, x.y, y.y), __fmaf_rn(a, x.z, y.z),
                     __fmaf_rn(a, x.w, y.w));
}
__device__ __forceinline__ float4 mul4(float4 a, float4 b) {
  return make_float4(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y), __fmul_rn(a.z, b.z),
                     __fmul_rn(a.w, b.w));
}
// p_new = beta * p_old + dinv * r   (z = dinv r never stored)
__device__ __forceinline__ float4 pnew4(float be, float4 po, float4 d, float4 r) {
  return fma4(be, po, mul4(d, r));
}
__device__ __forceinline__ float pnew1(float be, float po, float d, float r) {
  return __fmaf_rn(be, po, __fmul_rn(d, r));
}
// fp64 accumulation of a float4 dot product in a fixed order
__device__ __forceinline__ double dot4_acc(float4 a, float4 b, double acc) {
  acc = __fma_rn((double)a.x, (double)b.x, acc);
  acc = __fma_rn((double)a.y, (double)b.y, acc);
  acc = __fma_rn((double)a.z, (double)b.z, acc);
  return __fma_rn((double)a.w, (double)b.w, acc);
}
// fp32 dot of a float4 pair in a fixed order (explicit fma chain)
__device__ __forceinline__ float dot4f(float4 a, float4 b) {
  float s = __fmul_rn(a.x, b.x);
  s = __fmaf_rn(a.y, b.y, s);
  s = __fmaf_rn(a.z, b.z, s);
  return __fmaf_rn(a.w, b.w, s);
}
__device__ __forceinline__ float comp(const float4& v, int c) {
  return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}

// edge-difference stencil of one voxel (reading c8): q = sum_a w_a (p - p_a), fixed -> 0
__device__ __forceinline__ float stencil1(float p, float xp, float xm, float yp, float ym,
                                          float zp, float zm, float wx, float wxm, float wy,
                                          float wym, float wz, float wzm, float dv) {
  float q = __fmul_rn(wx, __fsub_rn(p, xp));
  q = __fmaf_rn(wxm, __fsub_rn(p, xm), q);
  q = __fmaf_rn(wy, __fsub_rn(p, yp), q);
  q = __fmaf_rn(wym, __fsub_rn(p, ym), q);
  q = __fmaf_rn(wz, __fsub_rn(p, zp), q);
  q = __fmaf_rn(wzm, __fsub_rn(p, zm), q);
  return dv == 0.f ? 0.f : q;
}

// ---- packed fp32 pairs for pass A (sm_100a FFMA2 / FADD2 / FMUL2): every lane computes
// exactly the IEEE round-to-nearest result of the scalar op it replaces (negation is exact,
// so a - b == a + (-b)), so the packed forms are bit-identical to pnew4 / fma4 / mul4 /
// stencil1 / grady and only take fewer issue slots.  A float4 quad is the register pairs
// (x, y) and (z, w).
__device__ __forceinline__ float2 pa_lo(float4 v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 pa_hi(float4 v) { return make_float2(v.z, v.w); }
__device__ __forceinline__ float4 pa_cat(float2 a, float2 b) { return make_float4(a.x, a.y, b.x, b.y); }
__device__ __forceinline__ float2 pa_sub(float2 a, float2 b) {
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
__device__ __forceinline__ float4 pa_fma4(float a, float4 x, float4 y) {     // = fma4
  const float2 aa = make_float2(a, a);
  return pa_cat(__ffma2_rn(aa, pa_lo(x), pa_lo(y)), __ffma2_rn(aa, pa_hi(x), pa_hi(y)));
}
__device__ __forceinline__ float4 pa_mul4(float4 a, float4 b) {             // = mul4
  return pa_cat(__fmul2_rn(pa_lo(a), pa_lo(b)), __fmul2_rn(pa_hi(a), pa_hi(b)));
}
__device__ __forceinline__ float4 pa_pnew4(float be, float4 po, float4 d, float4 r) {   // = pnew4
  return pa_fma4(be, po, pa_mul4(d, r));
}
// grady(a_e - b_e) of 4 lanes (= four grady(__fsub_rn(a, b)) calls)
__device__ __forceinline__ float4 pa_grady4(float4 a, float4 b, float nbl2, float eps) {
  const float2 n2 = make_float2(nbl2, nbl2), e2 = make_float2(eps, eps);
  const float2 d0 = pa_sub(pa_lo(a), pa_lo(b)), d1 = pa_sub(pa_hi(a), pa_hi(b));
  float2 t0 = __fmul2_rn(__fmul2_rn(d0, d0), n2), t1 = __fmul2_rn(__fmul2_rn(d1, d1), n2);
  t0 = make_float2(ex2_approx(t0.x), ex2_approx(t0.y));
  t1 = make_float2(ex2_approx(t1.x), ex2_approx(t1.y));
  return pa_cat(__fadd2_rn(t0, e2), __fadd2_rn(t1, e2));
}
// q += wp (p - pp) then q += wm (p - pm), per lane (the +a / -a term pair of stencil1)
__device__ __forceinline__ float4 pa_terms2(float4 q, float4 p, float4 pp, float4 pm, float4 wp,
                                            float4 wm) {
  float2 a = __ffma2_rn(pa_lo(wp), pa_sub(pa_lo(p), pa_lo(pp)), pa_lo(q));
  float2 b = __ffma2_rn(pa_hi(wp), pa_sub(pa_hi(p), pa_hi(pp)), pa_hi(q));
  a = __ffma2_rn(pa_lo(wm), pa_sub(pa_lo(p), pa_lo(pm)), a);
  b = __ffma2_rn(pa_hi(wm), pa_sub(pa_hi(p), pa_hi(pm)), b);
  return pa_cat(a, b);
}
// stencil1 of the quad p (x-neighbours xl / xr across it), same term order:
// q = wx (p - p[+x]); q += wxm (p - p[-x]); +y, -y, +z, -z; q = 0 where dv == 0.
// The x differences: p_i - p_{i+1} = d_i, and p_i - p_{i-1} = -d_{i-1} exactly.
__device__ __forceinline__ float4 pa_stencil4(float4 p, float xl, float xr, float4 yp, float4 ym,
                                              float4 zp, float4 zm, float4 wx, float4 wxm,
                                              float4 wy, float4 wym, float4 wz, float4 wzm,
                                              float4 dv) {
  const float d0 = __fsub_rn(p.x, p.y), d1 = __fsub_rn(p.y, p.z), d2 = __fsub_rn(p.z, p.w);
  const float d3 = __fsub_rn(p.w, xr), dm = __fsub_rn(p.x, xl);
  float2 a = __fmul2_rn(pa_lo(wx), make_float2(d0, d1));
  float2 b = __fmul2_rn(pa_hi(wx), make_float2(d2, d3));
  a = __ffma2_rn(pa_lo(wxm), make_float2(dm, -d0), a);
  b = __ffma2_rn(pa_hi(wxm), make_float2(-d1, -d2), b);
  float4 q = pa_terms2(pa_cat(a, b), p, yp, ym, wy, wym);
  q = pa_terms2(q, p, zp, zm, wz, wzm);
  return make_float4(dv.x == 0.f ? 0.f : q.x, dv.y == 0.f ? 0.f : q.y,
                     dv.z == 0.f ? 0.f : q.z, dv.w == 0.f ? 0.f : q.w);
}

// --------------------------------------------------------------------------- scalars
// Decision of pass A(k) for one (rhs, brick), computed redundantly by every CTA of the
// brick from the same partials in the same order (so every CTA agrees).
struct Scal {
  int active;
  float beta, alpha;
};

__device__ inline Scal passA_scalars(const Plan& P, const Bufs& Bf, const Ctl& C, int rb, int k,
                                     int u, int lane) {
  Scal s = {0, 0.f, 0.f};
  const int st = Bf.status[rb];
  if (st != ST_ACTIVE) return s;
  const long long RBU = (long long)P.R * P.B * P.U;
  const double* pb = reinterpret_cast<const double*>(Bf.PB);
  const double rz_k = warp_sum_array(pb + 2 * ((k & 1) * RBU + (long long)rb * P.U), P.U, 2, lane);
  const double rr_k = warp_sum_array(pb + 2 * ((k & 1) * RBU + (long long)rb * P.U) + 1, P.U, 2, lane);
  const double* ps = reinterpret_cast<const double*>(Bf.PS) + 4LL * rb * P.U;
  const double bb = warp_sum_array(ps + 0, P.U, 4, lane);
  int nst = ST_ACTIVE;
  double rz_km1 = 0.0, pq_km1 = 0.0;
  if (k == 0) {
    const double nf = warp_sum_array(ps + 1, P.U, 4, lane);
    const double nu = warp_sum_array(ps + 2, P.U, 4, lane);
    if (nf == 0.0 || nu == 0.0) nst = ST_TRIVIAL;
    else if (bb == 0.0) nst = ST_ZERO_B;
  } else {
    rz_km1 = warp_sum_array(pb + 2 * (((k - 1) & 1) * RBU + (long long)rb * P.U), P.U, 2, lane);
    pq_km1 = warp_sum_array(Bf.PA + ((k - 1) & 1) * RBU + (long long)rb * P.U, P.U, 1, lane);
    if (!(pq_km1 > 0.0) || !isfinite(rz_k) || !isfinite(pq_km1)) nst = ST_BREAKDOWN;
  }
  if (nst == ST_ACTIVE) {
    const double t2 = (double)C.tol * (double)C.tol;
    const bool conv = (C.tol_mode == 0) ? (rr_k <= t2 * bb) : (rr_k <= t2);
    if (conv) nst = ST_CONVERGED;
    else if (k >= C.max_iter) nst = ST_MAXITER;
  }
  if (nst != ST_ACTIVE) {
    if (u == 0 && lane == 0) {
      Bf.status[rb] = nst;
      Bf.iters[rb] = (nst == ST_TRIVIAL || nst == ST_ZERO_B) ? 0 : k;
    }
    return s;
  }
  if (u == 0 && lane == 0) atomicAdd(Bf.ctr + (k & 1), 1);
  s.active = 1;
  if (k > 0) {
    s.alpha = (float)(rz_km1 / pq_km1);
    s.beta = (float)(rz_k / rz_km1);
  }
  return s;
}

// Decision of pass k for (rhs, brick) rb from pass k-1's partials (the math of
// passA_scalars1).  CG = true: the partials come from other CTAs of the running launch (read
// through L2).  Out: status (ST_ACTIVE or the stop reason), iters at a stop, alpha / beta.
template <bool CG>
__device__ inline int passA_decide1(const Plan& P, const Bufs& Bf, const Ctl& C, int rb, int k,
                                    int lane, Scal& s, int& it) {
  auto wsum = [&](const double* a, int stride) {
    return CG ? warp_sum_array_cg(a, P.U, stride, lane) : warp_sum_array(a, P.U, stride, lane);
  };
  const long long RBU = (long long)P.R * P.B * P.U;
  const double* ps = reinterpret_cast<const double*>(Bf.PS) + 4LL * rb * P.U;
  const double bb = wsum(ps + 0, 4);
  const double t2 = (double)C.tol * (double)C.tol;
  auto conv = [&](double rr) { return (C.tol_mode == 0) ? (rr <= t2 * bb) : (rr <= t2); };
  int nst = ST_ACTIVE;
  it = 0;
  double rz = 0.0, pq = 0.0, qdr = 0.0, qdq = 0.0;
  if (k == 0) {
    const double* pb = reinterpret_cast<const double*>(Bf.PB);     // setup: (r0.z0, r0.r0)
    const double rr0 = wsum(pb + 2 * ((long long)rb * P.U) + 1, 2);
    const double nf = wsum(ps + 1, 4);
    const double nu = wsum(ps + 2, 4);
    if (nf == 0.0 || nu == 0.0) nst = ST_TRIVIAL;
    else if (bb == 0.0) nst = ST_ZERO_B;
    else if (conv(rr0)) nst = ST_CONVERGED;
  } else {
    const double* pa = Bf.PA + 5 * (((k - 1) & 1) * RBU + (long long)rb * P.U);
    rz = wsum(pa + 0, 5);
    const double rr = wsum(pa + 1, 5);
    pq = wsum(pa + 2, 5);
    qdr = wsum(pa + 3, 5);
    qdq = wsum(pa + 4, 5);
    it = k - 1;
    if (k > 1 && conv(rr)) nst = ST_CONVERGED;
    else if (it >= C.max_iter) nst = ST_MAXITER;
    else if (!(pq > 0.0) || !isfinite(pq) || !isfinite(rz) || !(rz > 0.0)) nst = ST_BREAKDOWN;
  }
  s = {0, 0.f, 0.f};
  if (nst != ST_ACTIVE) return nst;
  s.active = 1;
  if (k > 0) {
    s.alpha = (float)(rz / pq);
    const double a = (double)s.alpha;
    double rz1 = rz - 2.0 * a * qdr + a * a * qdq;
    if (!(rz1 > 0.0)) rz1 = 0.0;        // below the rounding level: restart the direction
    s.beta = (float)(rz1 / rz);
  }
  return nst;
}

// One-pass mode (passA.cu): at the start of pass k the partials of pass k-1 give the TRUE
// r_{k-1}.z_{k-1}, ||r_{k-1}||^2 and p.q, q.D r, q.D q of iteration k-1.  Decisions run on the
// true residual of r_{k-1} (x_{k-1} was written by pass k-1, so it is the result), alpha_{k-1}
// = r.z / p.q, beta_{k-1} from the one-step expansion of r_k.z_k.  iters = k-1 at a stop.
// With P.lastdec the decision of pass k >= 1 was taken by the last CTA of pass k-1
// (passA_last_decide) and is read from Bufs.SD; a stop was already written to status.
__device__ inline Scal passA_scalars1(const Plan& P, const Bufs& Bf, const Ctl& C, int rb, int k,
                                      int u, int lane) {
  Scal s = {0, 0.f, 0.f};
  const int st = Bf.status[rb];
  if (st != ST_ACTIVE) return s;
  if (P.lastdec && k > 0) {
    const float4 d = Bf.SD[(long long)(k & 1) * P.R * P.B + rb];
    s.active = 1;
    s.alpha = d.x;
    s.beta = d.y;
  } else {
    int it = 0;
    const int nst = passA_decide1<false>(P, Bf, C, rb, k, lane, s, it);
    if (nst != ST_ACTIVE) {
      if (u == 0 && lane == 0) {
        Bf.status[rb] = nst;
        Bf.iters[rb] = it;
      }
      return s;
    }
  }
  if (u == 0 && lane == 0) atomicAdd(Bf.ctr + (k & 1), 1);
  return s;
}

// P.lastdec, end of pass k, one warp of the CTA that finished (rhs, brick) rb last: the
// decision of pass k+1 -- a stop goes to status / iters, else (alpha, beta) to SD[(k+1)&1].
__device__ inline void passA_last_decide(const Plan& P, const Bufs& Bf, const Ctl& C, int rb,
                                         int k, int lane) {
  Scal s;
  int it = 0;
  const int nst = passA_decide1<true>(P, Bf, C, rb, k + 1, lane, s, it);
  if (lane == 0) {
    if (nst != ST_ACTIVE) {
      Bf.status[rb] = nst;
      Bf.iters[rb] = it;
    } else {
      Bf.SD[(long long)((k + 1) & 1) * P.R * P.B + rb] = make_float4(s.alpha, s.beta, 0.f, 0.f);
    }
    Bf.cnt[rb] = 0;
  }
}

}  // namespace rw
