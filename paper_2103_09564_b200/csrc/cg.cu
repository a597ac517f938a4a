// cg.cu -- SURVEY §8(a) rows a3-a7: implicit assembly, fused Jacobi-PCG passes, finalise.
//
// The method: x_U solves L_UU x_U = -B^T x_S; solver: Jacobi-preconditioned CG
// (P:197, P:33 fn 2).  Matrix-free: the SpMV is the edge-difference stencil
//     q_i = sum_{j ~ i} w_ij (p_i - p_j)       (reading c8; p = 0 on fixed voxels)
// which equals (L_UU p)_i with an exactly zero row sum in fp32.
//
// One CG iteration k = two kernels (the two global reductions of CG):
//   pass A(k):  beta_{k-1} = rho_k / rho_{k-1};  p_k = z_k + beta p_{k-1}, z = dinv r
//               (recomputed for the tile and its x/y halo, so z is never stored);
//               x_k = x_{k-1} + alpha_{k-1} p_{k-1} (lagged);  q = A p_k;  partial p.q
//   pass B(k):  alpha_k = rho_k / (p.q);  r -= alpha q;  partial rho_{k+1} = r.(dinv r), r.r
// Per-(rhs,brick) scalars are never stored: every CTA of a brick re-sums the brick's
// fp64 partials (fixed order) of the previous passes, so all CTAs take identical
// decisions.  Convergence (reading c5) is tested in pass A on ||r_k||; a stopped
// (rhs,brick) skips all later passes ("converged bricks drop out of the batch").
// All right-hand sides of a chunk share the operator loads (W, dinv) per plane.
#include "rw_common.cuh"

namespace rw {

// --------------------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;  // identical in every lane (a+b == b+a in IEEE)
}

// Sum of a[0..U) in a fixed order by one warp; result in all lanes.
__device__ __forceinline__ double warp_sum_array(const double* a, int U, int stride, int lane) {
  double s = 0.0;
  for (int u = lane; u < U; u += 32) s += a[(long long)u * stride];
  return warp_sum(s);
}

// Block-wide fixed-order reduction of NV values per thread; result written by thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* out, int out_stride) {
  __shared__ double red[RW_THREADS / 32][NV > 0 ? NV : 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = warp_sum(v[j]);
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) red[warp][j] = v[j];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double s = 0.0;
      for (int w = 0; w < RW_THREADS / 32; ++w) s += red[w][j];
      out[j * out_stride] = s;
    }
  }
}

struct Tile {
  int x0, y0, z0, z1, lx, ly, x, y;
  bool in;  // this thread's 4 columns are inside the brick
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
  // 256 % tpx may be != 0: threads past the TY rows own nothing
  t.in = (t.x < P.nx) && (t.y < P.ny) && (t.ly < P.TY);
  return t;
}

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
// fp64 accumulation of a float4 dot product in a fixed order (explicit fma, no contraction
// freedom, so all instantiations agree bit for bit)
__device__ __forceinline__ double dot4_acc(float4 a, float4 b, double acc) {
  acc = __fma_rn((double)a.x, (double)b.x, acc);
  acc = __fma_rn((double)a.y, (double)b.y, acc);
  acc = __fma_rn((double)a.z, (double)b.z, acc);
  return __fma_rn((double)a.w, (double)b.w, acc);
}
__device__ __forceinline__ float get(const float4& v, int c) {
  return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}

// --------------------------------------------------------------------------- setup (a3)
// x = values on S, x0 (or 0.5) on U;  r0_i = sum_j w_ij (x_j - x_i) on U (= b - L_UU x0),
// 0 on S;  p_{-1} = 0;  partials rho_0 = r.(dinv r), ||r0||^2, ||b||^2, counts.
__global__ void __launch_bounds__(RW_THREADS)
k_setup(Plan P, Bufs Bf) {
  const int u = blockIdx.x, b = blockIdx.y, r = blockIdx.z;
  const int rb = r * P.B + b;
  const Tile t = make_tile(P, u);
  const long long BN = (long long)P.B * P.n;
  const long long plane = (long long)P.nx * P.ny;
  double acc[5] = {0, 0, 0, 0, 0};  // rz, rr, bb, nfixed, nunknown
  if (t.in) {
    for (int z = t.z0; z < t.z1; ++z) {
      const long long ib = vidx(P, b, z, t.y, t.x);   // operator index (brick b)
      const long long iv = vidx(P, rb, z, t.y, t.x);  // per-rhs index
      auto X = [&](long long ob, long long ov) -> float {  // x of a voxel (brick/rhs idx)
        if (Bf.fixed[ob]) return Bf.values[ov];
        return Bf.x0 ? Bf.x0[ov] : 0.5f;
      };
      float xs[4], rr[4];
      const float4 dv = ld4(Bf.dinv + ib);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const long long ob = ib + c, ov = iv + c;
        const int xc = t.x + c;
        const bool fx = Bf.fixed[ob] != 0;
        const float xi = X(ob, ov);
        xs[c] = xi;
        float res = 0.f, bi = 0.f;
        if (!fx) {
          // six neighbours: +x, -x, +y, -y, +z, -z
          const long long dob[6] = {1, -1, P.nx, -(long long)P.nx, plane, -plane};
          const bool ok[6] = {xc + 1 < P.nx, xc > 0, t.y + 1 < P.ny, t.y > 0, z + 1 < P.nz, z > 0};
#pragma unroll
          for (int e = 0; e < 6; ++e) {
            if (!ok[e]) continue;
            const long long jb = ob + dob[e], jv = ov + dob[e];
            const int a = e >> 1;
            const float w = (e & 1) ? Bf.W[a * BN + jb] : Bf.W[a * BN + ob];
            const float xj = X(jb, jv);
            res = fmaf(w, xj - xi, res);
            if (Bf.fixed[jb]) bi = fmaf(w, xj, bi);
          }
        }
        rr[c] = res;
        const float d = get(dv, c);
        acc[0] = __fma_rn((double)res, (double)__fmul_rn(d, res), acc[0]);
        acc[1] = __fma_rn((double)res, (double)res, acc[1]);
        acc[2] = __fma_rn((double)bi, (double)bi, acc[2]);
        acc[3] += fx ? 1.0 : 0.0;
        acc[4] += fx ? 0.0 : 1.0;
      }
      st4(Bf.x + iv, make_float4(xs[0], xs[1], xs[2], xs[3]));
      st4(Bf.r + iv, make_float4(rr[0], rr[1], rr[2], rr[3]));
      st4(Bf.p0 + iv, f4(0.f));
    }
  }
  double v2[2] = {acc[0], acc[1]};
  block_sum<2>(v2, reinterpret_cast<double*>(Bf.PB + (long long)rb * P.U + u), 1);
  double v3[3] = {acc[2], acc[3], acc[4]};
  __syncthreads();
  block_sum<3>(v3, reinterpret_cast<double*>(Bf.PS + (long long)rb * P.U + u), 1);
}

// --------------------------------------------------------------------------- scalars
// Decision of pass A(k) for one (rhs, brick), computed redundantly by every CTA of the
// brick from the same partials in the same order (so every CTA agrees).
struct Scal {
  int active;
  float beta, alpha;
};

__device__ Scal passA_scalars(const Plan& P, const Bufs& Bf, const Ctl& C, int rb, int k,
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

// --------------------------------------------------------------------------- pass A (a4)
template <int RC>
__global__ void __launch_bounds__(RW_THREADS)
k_passA(Plan P, Bufs Bf, Ctl C, int k, int r_first) {
  extern __shared__ float4 smem_dyn[];
  float* sp = reinterpret_cast<float*>(smem_dyn);   // [2][RC][TY+2][TXP]
  __shared__ float s_beta[RC], s_alpha[RC];
  __shared__ int s_act[RC];
  const int u = blockIdx.x, b = blockIdx.y;
  const int rbase = r_first + blockIdx.z * RC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < RC) {
    Scal s = {0, 0.f, 0.f};
    if (rbase + warp < P.R) s = passA_scalars(P, Bf, C, (rbase + warp) * P.B + b, k, u, lane);
    if (lane == 0) { s_act[warp] = s.active; s_beta[warp] = s.beta; s_alpha[warp] = s.alpha; }
  }
  __syncthreads();
  bool any = false;
#pragma unroll
  for (int c = 0; c < RC; ++c) any |= (s_act[c] != 0);
  if (!any) return;

  const Tile t = make_tile(P, u);
  const long long BN = (long long)P.B * P.n;
  const long long plane = (long long)P.nx * P.ny;
  const float* Pold = (k & 1) ? Bf.p1 : Bf.p0;
  float* Pnew = (k & 1) ? Bf.p0 : Bf.p1;
  const int rowsz = (P.TY + 2) * P.TXP;
  float be[RC], al[RC];
  bool act[RC];
  long long rofs[RC];
#pragma unroll
  for (int c = 0; c < RC; ++c) {
    act[c] = s_act[c] != 0;
    be[c] = s_beta[c];
    al[c] = s_alpha[c];
    rofs[c] = (long long)(rbase + c) * BN;   // per-rhs offset of index b*n + v
  }
  const long long ob0 = (long long)b * P.n;  // operator offset of brick b

  // p_new at an arbitrary voxel (brick-local linear index lv) for rhs c
  auto pnew1 = [&](int c, long long lv) -> float {
    const long long o = ob0 + lv;
    return __fmaf_rn(be[c], Pold[rofs[c] + o], __fmul_rn(Bf.dinv[o], Bf.r[rofs[c] + o]));
  };

  float4 pm[RC], pc[RC], pn[RC], poc[RC], pon[RC];
  float4 dvc = f4(0.f), dvn = f4(0.f), wzm = f4(0.f);
  const long long lcol = (long long)t.y * P.nx + t.x;  // brick-local column offset
  if (t.in) {
    const long long o = ob0 + (long long)t.z0 * plane + lcol;
    dvc = ld4(Bf.dinv + o);
    if (t.z0 > 0) wzm = ld4(Bf.W + 2 * BN + o - plane);
#pragma unroll
    for (int c = 0; c < RC; ++c) {
      pm[c] = pc[c] = poc[c] = f4(0.f);
      if (!act[c]) continue;
      poc[c] = ld4(Pold + rofs[c] + o);
      pc[c] = fma4(be[c], poc[c], mul4(dvc, ld4(Bf.r + rofs[c] + o)));
      if (t.z0 > 0) {
        const float4 dm = ld4(Bf.dinv + o - plane);
        pm[c] = fma4(be[c], ld4(Pold + rofs[c] + o - plane), mul4(dm, ld4(Bf.r + rofs[c] + o - plane)));
      }
    }
  }
  double acc[RC];
#pragma unroll
  for (int c = 0; c < RC; ++c) acc[c] = 0.0;

  const int nhx = 2 * P.tpx;                 // row-halo float4 items
  const int nhalo = nhx + 2 * P.TY;          // + column-halo scalar items
  for (int z = t.z0; z < t.z1; ++z) {
    const int buf = (z - t.z0) & 1;
    const long long oz = ob0 + (long long)z * plane;
    // next plane
    if (t.in && z + 1 < P.nz) {
      const long long o = oz + plane + lcol;
      dvn = ld4(Bf.dinv + o);
#pragma unroll
      for (int c = 0; c < RC; ++c) {
        if (!act[c]) continue;
        pon[c] = ld4(Pold + rofs[c] + o);
        pn[c] = fma4(be[c], pon[c], mul4(dvn, ld4(Bf.r + rofs[c] + o)));
      }
    } else {
#pragma unroll
      for (int c = 0; c < RC; ++c) pn[c] = pon[c] = f4(0.f);
      dvn = f4(0.f);
    }
    // centre + halo of plane z into shared memory
#pragma unroll
    for (int c = 0; c < RC; ++c) {
      float* s = sp + (buf * RC + c) * rowsz;
      st4(s + (t.ly + 1) * P.TXP + 4 + 4 * t.lx, t.in ? pc[c] : f4(0.f));
    }
    for (int h = threadIdx.x; h < nhalo; h += RW_THREADS) {
      if (h < nhx) {                               // rows y0-1 / y0+TY, 4 voxels
        const int side = h / P.tpx, gx = h % P.tpx;
        const int hy = side ? t.y0 + P.TY : t.y0 - 1;
        const int hx = t.x0 + 4 * gx;
        const int srow = side ? P.TY + 1 : 0;
        const bool ok = hy >= 0 && hy < P.ny && hx < P.nx;
#pragma unroll
        for (int c = 0; c < RC; ++c) {
          float4 v = f4(0.f);
          if (ok && act[c]) {
            const long long lv = (long long)z * plane + (long long)hy * P.nx + hx;
            const long long o = ob0 + lv;
            v = fma4(be[c], ld4(Pold + rofs[c] + o), mul4(ld4(Bf.dinv + o), ld4(Bf.r + rofs[c] + o)));
          }
          st4(sp + (buf * RC + c) * rowsz + srow * P.TXP + 4 + 4 * gx, v);
        }
      } else {                                     // columns x0-1 / x0+TX, 1 voxel
        const int hh = h - nhx;
        const int side = hh / P.TY, ry = hh % P.TY;
        const int hx = side ? t.x0 + P.TX : t.x0 - 1;
        const int hy = t.y0 + ry;
        const int scol = side ? 4 + P.TX : 3;
        const bool ok = hx >= 0 && hx < P.nx && hy < P.ny;
#pragma unroll
        for (int c = 0; c < RC; ++c) {
          float v = 0.f;
          if (ok && act[c]) v = pnew1(c, (long long)z * plane + (long long)hy * P.nx + hx);
          sp[(buf * RC + c) * rowsz + (ry + 1) * P.TXP + scol] = v;
        }
      }
    }
    __syncthreads();
    if (t.in) {
      const long long o = oz + lcol;
      const float4 wx = ld4(Bf.W + o);
      const float wxm0 = (t.x > 0) ? Bf.W[o - 1] : 0.f;
      const float4 wxm = make_float4(wxm0, wx.x, wx.y, wx.z);
      const float4 wy = ld4(Bf.W + BN + o);
      const float4 wym = (t.y > 0) ? ld4(Bf.W + BN + o - P.nx) : f4(0.f);
      const float4 wz = ld4(Bf.W + 2 * BN + o);
#pragma unroll
      for (int c = 0; c < RC; ++c) {
        if (!act[c]) continue;
        const float* s = sp + (buf * RC + c) * rowsz;
        const int cc = 4 + 4 * t.lx;
        const float4 up = ld4(s + (t.ly + 2) * P.TXP + cc);   // y+1
        const float4 dn = ld4(s + (t.ly) * P.TXP + cc);       // y-1
        const float xl = s[(t.ly + 1) * P.TXP + cc - 1];
        const float xr = s[(t.ly + 1) * P.TXP + cc + 4];
        const float4 p = pc[c];
        const float4 pxp = make_float4(p.y, p.z, p.w, xr);
        const float4 pxm = make_float4(xl, p.x, p.y, p.z);
        float4 q;
        // explicit rn intrinsics: no contraction choices left to the compiler, so every
        // template instantiation (RC = 1..4) produces the same bits
#define RW_Q(comp)                                                                        \
  q.comp = __fmul_rn(wx.comp, __fsub_rn(p.comp, pxp.comp));                               \
  q.comp = __fmaf_rn(wxm.comp, __fsub_rn(p.comp, pxm.comp), q.comp);                      \
  q.comp = __fmaf_rn(wy.comp, __fsub_rn(p.comp, up.comp), q.comp);                        \
  q.comp = __fmaf_rn(wym.comp, __fsub_rn(p.comp, dn.comp), q.comp);                       \
  q.comp = __fmaf_rn(wz.comp, __fsub_rn(p.comp, pn[c].comp), q.comp);                     \
  q.comp = __fmaf_rn(wzm.comp, __fsub_rn(p.comp, pm[c].comp), q.comp);                    \
  if (dvc.comp == 0.f) q.comp = 0.f;
        RW_Q(x) RW_Q(y) RW_Q(z) RW_Q(w)
#undef RW_Q
        const long long ov = rofs[c] + o;
        if (k > 0) st4(Bf.x + ov, fma4(al[c], poc[c], ld4(Bf.x + ov)));
        st4(Pnew + ov, p);
        st4(Bf.q + ov, q);
        acc[c] = dot4_acc(p, q, acc[c]);
      }
      wzm = wz;
    }
#pragma unroll
    for (int c = 0; c < RC; ++c) { pm[c] = pc[c]; pc[c] = pn[c]; poc[c] = pon[c]; }
    dvc = dvn;
  }
  // per-rhs CTA partial of p.q
  const long long RBU = (long long)P.R * P.B * P.U;
#pragma unroll
  for (int c = 0; c < RC; ++c) {
    double v[1] = {acc[c]};
    __syncthreads();
    if (act[c]) block_sum<1>(v, Bf.PA + (k & 1) * RBU + (long long)((rbase + c) * P.B + b) * P.U + u, 1);
  }
}

// --------------------------------------------------------------------------- pass B (a5)
template <int RC>
__global__ void __launch_bounds__(RW_THREADS)
k_passB(Plan P, Bufs Bf, int k, int r_first) {
  __shared__ float s_alpha[RC];
  __shared__ int s_act[RC];
  const int u = blockIdx.x, b = blockIdx.y;
  const int rbase = r_first + blockIdx.z * RC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long RBU = (long long)P.R * P.B * P.U;
  if (warp < RC) {
    int act = 0;
    float al = 0.f;
    const int r = rbase + warp;
    if (r < P.R) {
      const int rb = r * P.B + b;
      if (Bf.status[rb] == ST_ACTIVE) {
        act = 1;
        const double* pb = reinterpret_cast<const double*>(Bf.PB);
        const double rz = warp_sum_array(pb + 2 * ((k & 1) * RBU + (long long)rb * P.U), P.U, 2, lane);
        const double pq = warp_sum_array(Bf.PA + (k & 1) * RBU + (long long)rb * P.U, P.U, 1, lane);
        al = (pq > 0.0 && isfinite(pq)) ? (float)(rz / pq) : 0.f;
      }
    }
    if (lane == 0) { s_act[warp] = act; s_alpha[warp] = al; }
  }
  __syncthreads();
  bool any = false;
#pragma unroll
  for (int c = 0; c < RC; ++c) any |= (s_act[c] != 0);
  if (!any) return;
  const Tile t = make_tile(P, u);
  const long long BN = (long long)P.B * P.n;
  const long long plane = (long long)P.nx * P.ny;
  const long long ob0 = (long long)b * P.n;
  double a0[RC], a1[RC];
#pragma unroll
  for (int c = 0; c < RC; ++c) a0[c] = a1[c] = 0.0;
  if (t.in) {
    const long long lcol = (long long)t.y * P.nx + t.x;
    for (int z = t.z0; z < t.z1; ++z) {
      const long long o = ob0 + (long long)z * plane + lcol;
      const float4 dv = ld4(Bf.dinv + o);
#pragma unroll
      for (int c = 0; c < RC; ++c) {
        if (!s_act[c]) continue;
        const long long ov = (long long)(rbase + c) * BN + o;
        const float al = -s_alpha[c];
        const float4 r = fma4(al, ld4(Bf.q + ov), ld4(Bf.r + ov));
        st4(Bf.r + ov, r);
        const float4 zz = mul4(dv, r);
        a0[c] = dot4_acc(r, zz, a0[c]);
        a1[c] = dot4_acc(r, r, a1[c]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < RC; ++c) {
    double v[2] = {a0[c], a1[c]};
    __syncthreads();
    if (s_act[c])
      block_sum<2>(v, reinterpret_cast<double*>(Bf.PB + ((k + 1) & 1) * RBU +
                                                (long long)((rbase + c) * P.B + b) * P.U + u), 1);
  }
}

// --------------------------------------------------------------------------- finalise (a6)
__global__ void __launch_bounds__(RW_THREADS)
k_finalize(Plan P, Bufs Bf, Ctl C, float* resid, int* status_out, uint8_t* labels) {
  const int u = blockIdx.x, b = blockIdx.y, r = blockIdx.z;
  const int rb = r * P.B + b;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long RBU = (long long)P.R * P.B * P.U;
  __shared__ float s_alpha;
  const int st = Bf.status[rb];
  const int k = Bf.iters[rb];
  if (warp == 0) {
    const double* pb = reinterpret_cast<const double*>(Bf.PB);
    float al = 0.f;
    if ((st == ST_CONVERGED || st == ST_MAXITER) && k >= 1) {
      const double rz = warp_sum_array(pb + 2 * (((k - 1) & 1) * RBU + (long long)rb * P.U), P.U, 2, lane);
      const double pq = warp_sum_array(Bf.PA + ((k - 1) & 1) * RBU + (long long)rb * P.U, P.U, 1, lane);
      al = (float)(rz / pq);
    }
    if (u == 0) {
      double res = 0.0;
      if (st == ST_CONVERGED || st == ST_MAXITER || st == ST_BREAKDOWN) {
        const double rr = warp_sum_array(pb + 2 * ((k & 1) * RBU + (long long)rb * P.U) + 1, P.U, 2, lane);
        const double* ps = reinterpret_cast<const double*>(Bf.PS) + 4LL * rb * P.U;
        const double bb = warp_sum_array(ps, P.U, 4, lane);
        res = sqrt(rr);
        if (C.tol_mode == 0) res = bb > 0.0 ? res / sqrt(bb) : 0.0;
      }
      if (lane == 0) {
        if (resid) resid[rb] = (float)res;
        if (status_out) status_out[rb] = st;
      }
    }
    if (lane == 0) s_alpha = al;
  }
  __syncthreads();
  const float al = s_alpha;
  const Tile t = make_tile(P, u);
  if (!t.in) return;
  const long long BN = (long long)P.B * P.n;
  const long long plane = (long long)P.nx * P.ny;
  const float* Plast = (k & 1) ? Bf.p1 : Bf.p0;   // p_{k-1}
  for (int z = t.z0; z < t.z1; ++z) {
    const long long lv = (long long)z * plane + (long long)t.y * P.nx + t.x;
    const long long ob = (long long)b * P.n + lv;
    const long long ov = (long long)r * BN + ob;
    float4 xv = ld4(Bf.x + ov);
    if (al != 0.f) xv = fma4(al, ld4(Plast + ov), xv);
    const uchar4 f = *reinterpret_cast<const uchar4*>(Bf.fixed + ob);
    const float4 val = ld4(Bf.values + ov);
    float o[4] = {xv.x, xv.y, xv.z, xv.w};
    const unsigned char fx[4] = {f.x, f.y, f.z, f.w};
    const float vv[4] = {val.x, val.y, val.z, val.w};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (fx[c]) o[c] = vv[c];
      else if (st == ST_ZERO_B) o[c] = 0.f;
      else o[c] = fminf(fmaxf(o[c], 0.f), 1.f);
    }
    st4(Bf.x + ov, make_float4(o[0], o[1], o[2], o[3]));
    if (labels && r == 0)
      *reinterpret_cast<uchar4*>(labels + ob) =
          make_uchar4(o[0] > 0.5f, o[1] > 0.5f, o[2] > 0.5f, o[3] > 0.5f);
  }
}

// --------------------------------------------------------------------------- labels (a7)
// seeds (0 = unseeded, 1..K) -> fixed mask and K-1 one-vs-rest value planes.
__global__ void k_labels_prep(const uint8_t* __restrict__ seeds, long long BN, int K,
                              uint8_t* __restrict__ fixed, float* __restrict__ values) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < BN;
       i += (long long)gridDim.x * blockDim.x) {
    const int s = seeds[i];
    fixed[i] = s != 0;
    for (int r = 0; r < K - 1; ++r) values[r * BN + i] = (s == r + 1) ? 1.f : 0.f;
  }
}

// argmax over classes 1..K with p_K = clamp(1 - sum_{k<K} p_k); ties -> lowest id.
__global__ void k_argmax(const float* __restrict__ prob, long long BN, int K,
                         uint8_t* __restrict__ labels) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < BN;
       i += (long long)gridDim.x * blockDim.x) {
    float best = -1.f, sum = 0.f;
    int arg = 0;
    for (int r = 0; r < K - 1; ++r) {
      const float p = prob[r * BN + i];
      sum += p;
      if (p > best) { best = p; arg = r + 1; }
    }
    const float pk = fminf(fmaxf(1.f - sum, 0.f), 1.f);
    if (pk > best) arg = K;
    labels[i] = (uint8_t)arg;
  }
}

// --------------------------------------------------------------------------- launchers
size_t passA_smem(const Plan& P, int RC) { return (size_t)2 * RC * (P.TY + 2) * P.TXP * sizeof(float); }

static void set_smem_attr() {
  static bool done = false;
  if (done) return;
  done = true;
  cudaFuncSetAttribute(k_passA<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_passA<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_passA<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_passA<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

cudaError_t launch_setup(const Plan& P, const Bufs& Bf, cudaStream_t s) {
  set_smem_attr();
  k_setup<<<dim3(P.U, P.B, P.R), RW_THREADS, 0, s>>>(P, Bf);
  return cudaGetLastError();
}

// RC = rhs per CTA (operator shared across them); chunks of up to 4.
cudaError_t launch_iteration_A(const Plan& P, const Bufs& Bf, const Ctl& C, int k, cudaStream_t s) {
  for (int r0 = 0; r0 < P.R; r0 += 4) {
    const int rc = P.R - r0 < 4 ? P.R - r0 : 4;
    const dim3 g(P.U, P.B, 1);
    const size_t sm = passA_smem(P, rc);
    switch (rc) {
      case 1: k_passA<1><<<g, RW_THREADS, sm, s>>>(P, Bf, C, k, r0); break;
      case 2: k_passA<2><<<g, RW_THREADS, sm, s>>>(P, Bf, C, k, r0); break;
      case 3: k_passA<3><<<g, RW_THREADS, sm, s>>>(P, Bf, C, k, r0); break;
      default: k_passA<4><<<g, RW_THREADS, sm, s>>>(P, Bf, C, k, r0); break;
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_iteration_B(const Plan& P, const Bufs& Bf, int k, cudaStream_t s) {
  for (int r0 = 0; r0 < P.R; r0 += 4) {
    const int rc = P.R - r0 < 4 ? P.R - r0 : 4;
    const dim3 g(P.U, P.B, 1);
    switch (rc) {
      case 1: k_passB<1><<<g, RW_THREADS, 0, s>>>(P, Bf, k, r0); break;
      case 2: k_passB<2><<<g, RW_THREADS, 0, s>>>(P, Bf, k, r0); break;
      case 3: k_passB<3><<<g, RW_THREADS, 0, s>>>(P, Bf, k, r0); break;
      default: k_passB<4><<<g, RW_THREADS, 0, s>>>(P, Bf, k, r0); break;
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_finalize(const Plan& P, const Bufs& Bf, const Ctl& C, float* resid,
                            int* status_out, uint8_t* labels, cudaStream_t s) {
  k_finalize<<<dim3(P.U, P.B, P.R), RW_THREADS, 0, s>>>(P, Bf, C, resid, status_out, labels);
  return cudaGetLastError();
}

cudaError_t launch_labels_prep(const uint8_t* seeds, long long BN, int K, uint8_t* fixed,
                               float* values, int sms, cudaStream_t s) {
  long long g = (BN + RW_THREADS - 1) / RW_THREADS;
  if (g > sms * 8LL) g = sms * 8LL;
  k_labels_prep<<<(int)g, RW_THREADS, 0, s>>>(seeds, BN, K, fixed, values);
  return cudaGetLastError();
}

cudaError_t launch_argmax(const float* prob, long long BN, int K, uint8_t* labels, int sms,
                          cudaStream_t s) {
  long long g = (BN + RW_THREADS - 1) / RW_THREADS;
  if (g > sms * 8LL) g = sms * 8LL;
  k_argmax<<<(int)g, RW_THREADS, 0, s>>>(prob, BN, K, labels);
  return cudaGetLastError();
}

}  // namespace rw
