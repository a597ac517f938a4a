// passA.cu -- SURVEY §8(a) row a4: CG pass A, the SpMV pass (dominant kernel).
//
// For iteration k and every active (rhs, brick):   (readings c5, c8)
//   p_k = dinv*r_k + beta_{k-1} p_{k-1}            (z = dinv r never stored)
//   x_k = x_{k-1} + alpha_{k-1} p_{k-1}            (lagged x update)
//   q   = L_UU p_k   as  q_i = sum_j w_ij (p_i - p_j),  q = 0 on fixed voxels
//   partial p_k . q  (fp64, fixed order)
//
// One-pass mode (ONE, the default streaming loop): pass B is folded in.  Pass k first forms
//   r_k = r_{k-1} - alpha_{k-1} q_{k-1}   (centre and x/y halo, from double-buffered r, q)
// then p_k, x_k, q_k as above, and writes r_k, p_k, x_k, q_k with the partials of r_k.z_k,
// r_k.r_k, p_k.q_k, q_k.D r_k, q_k.D q_k.  alpha_k = r.z / p.q as in plain CG; beta_k uses
// r_{k+1}.z_{k+1} = r.z - 2 alpha q.D r + alpha^2 q.D q, a one-step expansion anchored on
// the true dot of the same pass (passA_scalars1).  One HBM pass per iteration: 38 B per
// voxel-iteration (r, q, p, x, dinv, u16 in; r, p, x, q out) instead of 30 + 16.
//
// B200 design.  A CTA owns a TX x TY column tile of one brick and marches over ZC planes.
// One elected thread streams each plane's boxes (r, p_{k-1}, x, dinv and either the three
// weight planes or the raw intensities) into a 4-stage (default; 3 for the multi-rhs
// variants) shared-memory ring with TMA
// (cp.async.bulk.tensor, mbarrier completion), so HBM reads run two planes ahead of the
// math with no register cost.  The y/x halo of r, p, dinv (needed to form p_k at the
// tile's neighbours) comes in the same boxes; out-of-brick cells are zero-filled by TMA.
// p_k of plane z is shared through a padded smem plane for the x/y neighbours; the z
// neighbours stay in registers (sliding window).  Edge weights are either read (VM_STORED)
// or recomputed from the intensities (VM_U8..F32: 1-4 B/voxel instead of 12 B), with the
// same grady() expression every other kernel uses, so the operator is bit-identical.
#include "cg_device.cuh"
#include "passA.cuh"
#include "tma.cuh"

namespace rw {

template <int RC, int VM, bool ONE, int NS>
__global__ void __launch_bounds__(RW_MAX_THREADS, 2)
k_passA(Plan P, Bufs Bf, Ctl C, int k, int r_first, const __grid_constant__ Maps M) {
  using T = typename VolT<VM>::T;
  // NS = a_stages(P): ring depth, a compile-time constant (a runtime modulo in the ring
  // indexing measured 7 % slower)
  extern __shared__ __align__(128) unsigned char smem[];
  if (Bf.kdev) k = *reinterpret_cast<const volatile int*>(Bf.kdev);   // device-driven loop
  __shared__ float s_beta[RC], s_alpha[RC];
  __shared__ int s_act[RC];
  // grid.x = U units x nl rhs layers, the layer fastest: the CTAs of the nl layers of one unit
  // are launched together and stream the same tile's operator boxes (intensities, dinv) at
  // about the same planes, so all but the first read them from L2
  const int nl = gridDim.x / P.U;
  const int u = blockIdx.x / nl, b = blockIdx.y;
  const int rbase = r_first + (blockIdx.x % nl) * RC;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const ALayout L = a_layout(P, RC, VM);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bars);
  if (warp < RC) {
    Scal s = {0, 0.f, 0.f};
    if (rbase + warp < P.R)
      s = ONE ? passA_scalars1(P, Bf, C, (rbase + warp) * P.B + b, k, u, lane)
              : passA_scalars(P, Bf, C, (rbase + warp) * P.B + b, k, u, lane);
    if (lane == 0) { s_act[warp] = s.active; s_beta[warp] = s.beta; s_alpha[warp] = s.alpha; }
  }
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) mbar_init(bar + s, 1);
    fence_mbar_init();
  }
  __syncthreads();
  bool act[RC];
  float be[RC], al[RC];
  bool any = false;
#pragma unroll
  for (int c = 0; c < RC; ++c) {
    act[c] = s_act[c] != 0;
    be[c] = s_beta[c];
    al[c] = s_alpha[c];
    any |= act[c];
  }
  if (!any) return;
#pragma unroll
  for (int c = 0; c < RC; ++c) act[c] = act[c] || RC == 1;   // RC == 1: active if we got here

  // ---------------------------------------------------------------- hoisted geometry
  const Tile t = make_tile(P, u);
  const int nz = P.nz, TX = P.TX, TY = P.TY, TXh = P.TXh, TXP = P.TXP, tpx = P.tpx;
  const int hx = P.hx, TXhv = P.TXhv;
  const int zs = max(t.z0 - 1, 0), ze = min(t.z1, nz - 1);  // planes streamed
  const int np = ze - zs + 1;
  const float nbl2 = C.nbl2, eps = C.eps, gsc = C.scale, gof = C.offset;
  const long long BN = (long long)P.B * P.n;
  const long long plane = (long long)P.nx * P.ny;
  const long long RBN = (long long)P.R * BN;
  const bool in = t.in;
  // boundary predicates of this thread's 4 voxels (nx % 4 == 0: only the outer ones vary)
  const bool hasl = t.x > 0, hasr = t.x + 4 < P.nx, hasu = t.y + 1 < P.ny, hasd = t.y > 0;
  const int crow = (t.ly + 1) * TXh + hx + 4 * t.lx;   // centre in (TY+2) x TXh boxes
  const int xrow = t.ly * TX + 4 * t.lx;               // centre in TY x TX boxes
  const int vrow = (t.ly + 1) * TXhv + P.hxv + 4 * t.lx;  // centre in the intensity box
  const int spo = (t.ly + 1) * TXP + 4 + 4 * t.lx;     // centre in a p_new plane
  const int spc = (TY + 2) * TXP;                      // floats per p_new plane (one rhs)
  float* const sp = reinterpret_cast<float*>(smem + L.sp);
  float* const Wys = reinterpret_cast<float*>(smem + L.wys);   // [2][TY][TX] +y weights
  const long long ocol = (long long)b * P.n + (long long)t.y * P.nx + t.x;
  float* const Pnew = Bf.p + (long long)((k + 1) & 1) * RBN;
  const int par = k & 1;
  const bool xup = k > 0 && !C.noxlag;   // lagged x update of this pass
  const bool qin = ONE && k > 0;         // one-pass: r_k = r_{k-1} - alpha q_{k-1}
  float* const Rout = Bf.r + (long long)((k + 1) & 1) * RBN;
  float* const Qout = ONE ? Bf.q + (long long)((k + 1) & 1) * RBN : Bf.q;

  // ---------------------------------------------------------------- producer (tid 0)
  // plane j (z = zs + j) -> ring slot j % NS; its n-th use completes phase n & 1
  auto issue = [&](int j) {
    if (j >= np) return;
    const int zz = zs + j;
    unsigned char* st = smem + (j % NS) * L.stage;
    uint64_t* bj = bar + (j % NS);
    uint32_t bytes = L.eRP + (VM == VM_STORED ? L.eWx + L.eWy + L.eWz : L.eV);
#pragma unroll
    for (int c = 0; c < RC; ++c)
      if (act[c]) bytes += (qin ? 3 : 2) * L.eRP + ((xup && !ONE) ? L.eX : 0);
    mbar_arrive_expect_tx(bj, bytes);
    const int xb = t.x0 - hx, yb = t.y0 - 1;
#pragma unroll
    for (int c = 0; c < RC; ++c) {
      if (!act[c]) continue;
      const int pr = ((rbase + c) * P.B + b) * nz + zz;
      const int pp = ((par * P.R + rbase + c) * P.B + b) * nz + zz;
      tma_load_3d(st + L.oR + c * L.bRP, &M.r, bj, xb, yb, ONE ? pp : pr);
      tma_load_3d(st + L.oP + c * L.bRP, &M.p, bj, xb, yb, pp);
      if (qin) tma_load_3d(st + L.oQ + c * L.bRP, &M.q, bj, xb, yb, pp);
      if (xup && !ONE) tma_load_3d(st + L.oX + c * L.bX, &M.x, bj, t.x0, t.y0, pr);
    }
    const int pd = b * nz + zz;
    tma_load_3d(st + L.oD, &M.d, bj, xb, yb, pd);
    if (VM == VM_STORED) {
      tma_load_3d(st + L.oW, &M.wx, bj, xb, t.y0, pd);
      tma_load_3d(st + L.oW + L.bWx, &M.wy, bj, t.x0, yb, (P.B + b) * nz + zz);
      tma_load_3d(st + L.oW + L.bWx + L.bWy, &M.wz, bj, t.x0, t.y0, (2 * P.B + b) * nz + zz);
    } else {
      tma_load_3d(st + L.oW, &M.v, bj, t.x0 - P.hxv, yb, pd);
    }
  };
  // the same boxes of plane j pulled into L2 ahead of the ring (Plan.pf planes beyond it)
  auto pref = [&](int j) {
    if (j >= np) return;
    const int zz = zs + j;
    const int xb = t.x0 - hx, yb = t.y0 - 1;
#pragma unroll
    for (int c = 0; c < RC; ++c) {
      if (!act[c]) continue;
      const int pr = ((rbase + c) * P.B + b) * nz + zz;
      const int pp = ((par * P.R + rbase + c) * P.B + b) * nz + zz;
      tma_prefetch_3d(&M.r, xb, yb, ONE ? pp : pr);
      tma_prefetch_3d(&M.p, xb, yb, pp);
      if (qin) tma_prefetch_3d(&M.q, xb, yb, pp);
    }
    const int pd = b * nz + zz;
    tma_prefetch_3d(&M.d, xb, yb, pd);
    if (VM == VM_STORED) {
      tma_prefetch_3d(&M.wx, xb, t.y0, pd);
      tma_prefetch_3d(&M.wy, t.x0, yb, (P.B + b) * nz + zz);
      tma_prefetch_3d(&M.wz, t.x0, t.y0, (2 * P.B + b) * nz + zz);
    } else {
      tma_prefetch_3d(&M.v, t.x0 - P.hxv, yb, pd);
    }
  };
  auto wait = [&](int j) { mbar_wait(bar + (j % NS), (uint32_t)((j / NS) & 1)); };
  auto stg = [&](int j) -> const unsigned char* { return smem + (j % NS) * L.stage; };
  auto F = [](const unsigned char* st, int off) { return reinterpret_cast<const float*>(st + off); };
  // r of this iteration at box offset `off` (one-pass: r_{k-1} - alpha_{k-1} q_{k-1})
  auto rk4 = [&](const unsigned char* st, int c, int off) -> float4 {
    const float4 r = ld4(F(st, L.oR + c * L.bRP) + off);
    return qin ? pa_fma4(-al[c], ld4(F(st, L.oQ + c * L.bRP) + off), r) : r;
  };
  auto rk1 = [&](const unsigned char* st, int c, int off) -> float {
    const float r = F(st, L.oR + c * L.bRP)[off];
    return qin ? __fmaf_rn(-al[c], F(st, L.oQ + c * L.bRP)[off], r) : r;
  };
  auto centre_pnew = [&](const unsigned char* st, int c) -> float4 {
    return pa_pnew4(be[c], ld4(F(st, L.oP + c * L.bRP) + crow), ld4(F(st, L.oD) + crow),
                 rk4(st, c, crow));
  };
  // normalised intensities of 4 consecutive intensity-box elements (one vector smem load)
  auto gvol4 = [&](const unsigned char* st, int off, float g[4]) {
    const T* v = reinterpret_cast<const T*>(st + L.oW) + off;
    if (sizeof(T) == 4) {
      const float4 a = *reinterpret_cast<const float4*>(v);
      g[0] = a.x; g[1] = a.y; g[2] = a.z; g[3] = a.w;
    } else if (sizeof(T) == 2) {
      const uint2 a = *reinterpret_cast<const uint2*>(v);
      const T* e = reinterpret_cast<const T*>(&a);
      g[0] = (float)e[0]; g[1] = (float)e[1]; g[2] = (float)e[2]; g[3] = (float)e[3];
    } else {
      const uint32_t a = *reinterpret_cast<const uint32_t*>(v);
      const T* e = reinterpret_cast<const T*>(&a);
      g[0] = (float)e[0]; g[1] = (float)e[1]; g[2] = (float)e[2]; g[3] = (float)e[3];
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) g[e] = normv(g[e], gsc, gof);
  };
  auto g4 = [](const float g[4]) { return make_float4(g[0], g[1], g[2], g[3]); };
  auto gvol1 = [&](const unsigned char* st, int off) -> float {
    return normv((float)reinterpret_cast<const T*>(st + L.oW)[off], gsc, gof);
  };

  if (tid == 0) {
    prefetch_tmap(&M.r);
    prefetch_tmap(&M.p);
    prefetch_tmap(&M.d);
    prefetch_tmap(VM == VM_STORED ? &M.wx : &M.v);
    // planes 0 .. jz0 + NS - 2 now; step z issues plane (z - zs) + NS - 1
    for (int j = 0; j <= (t.z0 - zs) + NS - 2; ++j) issue(j);
    if (P.pf > 0)
      for (int j = (t.z0 - zs) + NS - 1; j <= (t.z0 - zs) + NS - 2 + P.pf; ++j) pref(j);
  }
  // out-of-tile halo columns of the p_new planes stay zero when the tile spans the brick
  if (hx == 0) {
    for (int h = tid; h < 2 * 2 * RC * TY; h += blockDim.x) {
      const int side = h & 1, ry = (h >> 1) % TY, pc_ = (h >> 1) / TY;   // pc_ = buf*RC + c
      sp[pc_ * spc + (ry + 1) * TXP + (side ? TX + 4 : 3)] = 0.f;
    }
  }

  float4 pm[RC], pc[RC], pn[RC];
  float4 wzm = f4(0.f);
  float gcur[4] = {0.f, 0.f, 0.f, 0.f};     // VM modes: normalised intensities of plane z
#pragma unroll
  for (int c = 0; c < RC; ++c) pm[c] = pc[c] = pn[c] = f4(0.f);
  const int jz0 = t.z0 - zs;
  if (t.z0 > 0) {                            // plane z0-1 = stage 0: z-neighbour + Wz(z0-1)
    wait(0);
    if (in) {
#pragma unroll
      for (int c = 0; c < RC; ++c)
        if (act[c]) pm[c] = centre_pnew(stg(0), c);
      if (VM == VM_STORED) wzm = ld4(F(stg(0), L.oW + L.bWx + L.bWy) + xrow);
    }
  }
  wait(jz0);
  if (in) {
#pragma unroll
    for (int c = 0; c < RC; ++c)
      if (act[c]) pc[c] = centre_pnew(stg(jz0), c);
    if (VM != VM_STORED) {
      gvol4(stg(jz0), vrow, gcur);
      if (t.z0 > 0) {
        float gm[4];
        gvol4(stg(0), vrow, gm);
        wzm = pa_grady4(g4(gcur), g4(gm), nbl2, eps);
      }
    }
  }

  double acc[RC];
  double acc1[RC][4];   // one-pass: r.z, r.r, q.D r, q.D q
#pragma unroll
  for (int c = 0; c < RC; ++c) {
    acc[c] = 0.0;
#pragma unroll
    for (int e = 0; e < 4; ++e) acc1[c][e] = 0.0;
  }
  const int nrow = 2 * tpx;                   // row-halo float4 items per rhs
  const int nhalo = nrow + (hx ? 2 * TY : 0); // + column-halo scalar items

  for (int z = t.z0; z < t.z1; ++z) {
    const int jz = z - zs;
    const bool hasn = z + 1 <= ze;
    float4 xz[RC];                            // one-pass: x_{k-1} of plane z, loaded early
    if (ONE && xup && in) {
#pragma unroll
      for (int c = 0; c < RC; ++c)
        xz[c] = act[c] ? ld4(Bf.x + (long long)(rbase + c) * BN + ocol + (long long)z * plane)
                       : f4(0.f);
    }
    const unsigned char* s0 = stg(jz);
    const unsigned char* s1 = stg(jz + 1);
    const int buf = z & 1;
    if (hasn) wait(jz + 1);
    if (in) {
#pragma unroll
      for (int c = 0; c < RC; ++c) pn[c] = (hasn && act[c]) ? centre_pnew(s1, c) : f4(0.f);
    }
    // p_k of plane z (centre + x/y halo) into shared plane `buf`
    float* spz = sp + buf * RC * spc;
    if (t.ly < TY) {
#pragma unroll
      for (int c = 0; c < RC; ++c) st4(spz + c * spc + spo, (in && act[c]) ? pc[c] : f4(0.f));
    }
    for (int h = tid; h < nhalo; h += blockDim.x) {
      if (h < nrow) {                        // rows y0-1 / y0+TY (zero-filled if outside)
        const int side = h >= tpx, g = side ? h - tpx : h;
        const int brow = side ? TY + 1 : 0;
        const int off = brow * TXh + hx + 4 * g;
#pragma unroll
        for (int c = 0; c < RC; ++c) {
          float4 v = f4(0.f);
          if (act[c])
            v = pa_pnew4(be[c], ld4(F(s0, L.oP + c * L.bRP) + off), ld4(F(s0, L.oD) + off),
                      rk4(s0, c, off));
          st4(spz + c * spc + brow * TXP + 4 + 4 * g, v);
        }
      } else {                               // columns x0-1 / x0+TX (tile narrower than brick)
        const int hh = h - nrow;
        const int side = hh >= TY, ry = side ? hh - TY : hh;
        const int off = (ry + 1) * TXh + (side ? hx + TX : hx - 1);
#pragma unroll
        for (int c = 0; c < RC; ++c) {
          float v = 0.f;
          if (act[c])
            v = pnew1(be[c], F(s0, L.oP + c * L.bRP)[off], F(s0, L.oD)[off], rk1(s0, c, off));
          spz[c * spc + (ry + 1) * TXP + (side ? TX + 4 : 3)] = v;
        }
      }
    }
    // ---- edge weights of this thread's 4 voxels
    float4 wx, wxm, wy, wym, wz;
    float gz[4] = {0.f, 0.f, 0.f, 0.f};
    if (VM != VM_STORED && in) {
      // forward weights of the own voxels; -x of voxels 1..3 is +x of voxels 0..2, -y comes
      // from the row above through shared memory, -z from the previous plane (registers)
      float gu[4];
      if (hasn) gvol4(s1, vrow, gz);
      gvol4(s0, vrow + TXhv, gu);
      const float gl = hasl ? gvol1(s0, vrow - 1) : 0.f;
      const float gr = hasr ? gvol1(s0, vrow + 4) : 0.f;
      const bool hz = z + 1 < nz;
      const float4 gc4 = g4(gcur);
      wx = pa_grady4(make_float4(gcur[1], gcur[2], gcur[3], gr), gc4, nbl2, eps);
      if (!hasr) wx.w = 0.f;
      const float am0 = hasl ? grady(__fsub_rn(gcur[0], gl), nbl2, eps) : 0.f;
      wxm = make_float4(am0, wx.x, wx.y, wx.z);
      wy = hasu ? pa_grady4(g4(gu), gc4, nbl2, eps) : f4(0.f);
      wz = hz ? pa_grady4(g4(gz), gc4, nbl2, eps) : f4(0.f);
      st4(Wys + buf * TY * TX + xrow, wy);
      wym = f4(0.f);
      if (t.ly == 0 && hasd) {               // first tile row: -y weights from the halo row
        float gd[4];
        gvol4(s0, vrow - TXhv, gd);
        wym = pa_grady4(g4(gcur), g4(gd), nbl2, eps);
      }
    }
    __syncthreads();                          // p_new plane + Wys of plane z complete
    if (tid == 0) {
      issue(jz + NS - 1);                // refill the slot of plane z-1 (all done with it)
      if (P.pf > 0) pref(jz + NS - 1 + P.pf);
    }
    if (in) {
      if (VM == VM_STORED) {
        const float* Wxb = F(s0, L.oW);
        wx = ld4(Wxb + t.ly * TXh + hx + 4 * t.lx);
        const float wl = hasl ? Wxb[t.ly * TXh + hx + 4 * t.lx - 1] : 0.f;
        wxm = make_float4(wl, wx.x, wx.y, wx.z);
        wy = ld4(F(s0, L.oW + L.bWx) + xrow + TX);
        wym = ld4(F(s0, L.oW + L.bWx) + xrow);
        wz = ld4(F(s0, L.oW + L.bWx + L.bWy) + xrow);
      } else if (t.ly > 0) {
        wym = ld4(Wys + buf * TY * TX + xrow - TX);
      }
      const float4 dvc = ld4(F(s0, L.oD) + crow);
      const long long o = ocol + (long long)z * plane;
#pragma unroll
      for (int c = 0; c < RC; ++c) {
        if (!act[c]) continue;
        const float* s = spz + c * spc;
        const float4 yp = ld4(s + spo + TXP);
        const float4 ym = ld4(s + spo - TXP);
        const float xl = s[spo - 1];
        const float xr = s[spo + 4];
        const float4 p = pc[c];
        const float4 q = pa_stencil4(p, xl, xr, yp, ym, pn[c], pm[c], wx, wxm, wy, wym, wz, wzm, dvc);
        const long long ov = (long long)(rbase + c) * BN + o;
        if (xup) {
          const float4 po = ld4(F(s0, L.oP + c * L.bRP) + crow);
          const float4 xo = ONE ? xz[c] : ld4(F(s0, L.oX + c * L.bX) + xrow);
          st4(Bf.x + ov, pa_fma4(al[c], po, xo));
        }
        st4(Pnew + ov, p);
        st4(Qout + ov, q);
        acc[c] += (double)dot4f(p, q);
        if (ONE) {
          const float4 rk = rk4(s0, c, crow);
          st4(Rout + ov, rk);
          const float4 dr = pa_mul4(dvc, rk), dq = pa_mul4(dvc, q);
          acc1[c][0] += (double)dot4f(rk, dr);
          acc1[c][1] += (double)dot4f(rk, rk);
          acc1[c][2] += (double)dot4f(q, dr);
          acc1[c][3] += (double)dot4f(q, dq);
        }
      }
      wzm = wz;
#pragma unroll
      for (int e = 0; e < 4; ++e) gcur[e] = gz[e];
    }
#pragma unroll
    for (int c = 0; c < RC; ++c) { pm[c] = pc[c]; pc[c] = pn[c]; }
  }
  // per-rhs CTA partial of p.q
  const long long RBU = (long long)P.R * P.B * P.U;
#pragma unroll
  for (int c = 0; c < RC; ++c) {
    __syncthreads();
    if (ONE) {
      double v[5] = {acc1[c][0], acc1[c][1], acc[c], acc1[c][2], acc1[c][3]};
      if (act[c])
        block_sum<5>(v, Bf.PA + 5 * ((k & 1) * RBU + (long long)((rbase + c) * P.B + b) * P.U + u));
    } else {
      double v[1] = {acc[c]};
      if (act[c]) block_sum<1>(v, Bf.PA + (k & 1) * RBU + (long long)((rbase + c) * P.B + b) * P.U + u);
    }
  }
  if (ONE && P.lastdec) {
    // the CTA that completes a (rhs, brick)'s U partials takes the decision of pass k+1 once
    // (threadfence reduction: partial stores -> fence -> arrival count)
    __shared__ int s_last[RC];
    if (tid == 0) {
      __threadfence();
#pragma unroll
      for (int c = 0; c < RC; ++c)
        s_last[c] = act[c] ? (atomicAdd(Bf.cnt + (rbase + c) * P.B + b, 1) == P.U - 1) : 0;
    }
    __syncthreads();
    if (warp < RC && s_last[warp]) {
      __threadfence();
      passA_last_decide(P, Bf, C, (rbase + warp) * P.B + b, k, lane);
    }
  }
}

// ------------------------------------------------------------------------- launcher
template <int RC, int VM, bool ONE, int NS>
static cudaError_t launch_one(const Plan& P, const Bufs& Bf, const Ctl& C, int k, int r0, int nz,
                              const Maps& M, cudaStream_t s) {
  static int attr = 48 * 1024;   // largest dynamic smem opted in so far for this instance
  const ALayout L = a_layout(P, RC, VM);
  if (L.total > attr) {
    const cudaError_t e = cudaFuncSetAttribute(k_passA<RC, VM, ONE, NS>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
    if (e != cudaSuccess) return e;
    attr = L.total;
  }
  k_passA<RC, VM, ONE, NS><<<dim3(P.U * nz, P.B, 1), P.threads, L.total, s>>>(P, Bf, C, k, r0, M);
  return cudaGetLastError();
}

template <int RC, int VM>
static cudaError_t launch_rc(const Plan& P, const Bufs& Bf, const Ctl& C, int k, int r0, int nz,
                             const Maps& M, cudaStream_t s) {
  if (P.one && a_stages(P) == kStages - 1)
    return launch_one<RC, VM, true, kStages - 1>(P, Bf, C, k, r0, nz, M, s);
  return P.one ? launch_one<RC, VM, true, kStages>(P, Bf, C, k, r0, nz, M, s)
               : launch_one<RC, VM, false, kStages>(P, Bf, C, k, r0, nz, M, s);
}

template <int VM>
static cudaError_t launch_vm(const Plan& P, const Bufs& Bf, const Ctl& C, int k, int r0, int rc,
                             int nz, const Maps& M, cudaStream_t s) {
  switch (rc) {
    case 1: return launch_rc<1, VM>(P, Bf, C, k, r0, nz, M, s);
    case 2: return launch_rc<2, VM>(P, Bf, C, k, r0, nz, M, s);
    case 3: return launch_rc<3, VM>(P, Bf, C, k, r0, nz, M, s);
    default: return launch_rc<4, VM>(P, Bf, C, k, r0, nz, M, s);
  }
}

// right-hand sides per CTA: up to 4 sharing one operator load, as long as two CTAs still fit
// one SM (measured on cfg4, 256^3 with 3 rhs: one launch of 3 single-rhs CTA layers 884 ms
// vs 2 + 1 rhs per CTA at one CTA per SM 1060 ms, bit-identical); P.rc > 0: fixed by the
// caller (RW_PASSA_RC)
int passA_rc(const Plan& P) {
  if (P.rc > 0) return P.rc < P.R ? P.rc : P.R;
  int rc = P.R < 4 ? P.R : 4;
  while (rc > 1 && a_layout(P, rc, P.vm).total > 112 * 1024) --rc;
  return rc;
}

// One-pass mode: a ring of kStages - 1 planes where kStages would leave one CTA per SM
// (e.g. f32 intensities with x halos: 123 KB at 4 stages, 97 KB at 3; cfg4 256^3 f32 runs
// at 12 % warp occupancy with 4 stages, ncu gpurun_out/c4)
void passA_stages(Plan& P) {
  P.ns = kStages;
  if (P.one && a_layout(P, passA_rc(P), P.vm).total > 112 * 1024) P.ns = kStages - 1;
  // L2 prefetch of the boxes 2 planes beyond the ring where the ring is one stage short
  // (measured, tools/gpu_pf.sh: cfg4 822 -> 757 ms at 3 stages; with 4 stages it costs --
  // cfg3 1577 -> 1707 ms, cfg2 streaming 148 -> 144 G); RW_PASSA_PF overrides
  if (P.pf < 0) P.pf = P.ns < kStages ? 2 : 0;
}

size_t passA_smem(const Plan& P, int rc) { return (size_t)a_layout(P, rc, P.vm).total; }

// One launch per group of right-hand sides: R / rc CTA layers (grid z) when rc divides R,
// else ceil(R / rc) launches (the last one narrower).
cudaError_t launch_iteration_A(const Plan& P, const Bufs& Bf, const Ctl& C, int k,
                               const Maps& M, cudaStream_t s) {
  const int rcmax = passA_rc(P);
  const int layers = P.R % rcmax == 0 ? P.R / rcmax : 1;
  for (int r0 = 0; r0 < P.R; r0 += rcmax * layers) {
    const int rc = P.R - r0 < rcmax ? P.R - r0 : rcmax;
    cudaError_t e;
    switch (P.vm) {
      case VM_U8: e = launch_vm<VM_U8>(P, Bf, C, k, r0, rc, layers, M, s); break;
      case VM_U16: e = launch_vm<VM_U16>(P, Bf, C, k, r0, rc, layers, M, s); break;
      case VM_I16: e = launch_vm<VM_I16>(P, Bf, C, k, r0, rc, layers, M, s); break;
      case VM_F32: e = launch_vm<VM_F32>(P, Bf, C, k, r0, rc, layers, M, s); break;
      default: e = launch_vm<VM_STORED>(P, Bf, C, k, r0, rc, layers, M, s); break;
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace rw
