// resident.cu -- SURVEY §8(f) f2/f4: the brick-resident CG solver.
//
// Same method as the streaming passes (cg.cu / passA.cu): Jacobi-preconditioned CG
// (P:197, P:33 fn 2) on L_UU x_U = -B^T x_S, edge-difference SpMV (reading c8),
// fp64 fixed-order reductions, the same stopping rule and status codes (reading c5).
// What changes is where the state lives.  The streaming path re-reads the whole CG state
// from HBM every iteration (two passes, ~46 B per voxel-iteration).  Here one
// thread-block cluster owns one brick for its whole solve (bricks are independent,
// P:167): the brick is split into CL z-slabs of ZS = 4 planes, one CTA (one SM) per slab,
// and every iteration runs on chip:
//
//   shared memory : p (own planes + one halo plane on each side), x, the -y / -z weights
//                   this thread does not own                          (208 KB at 64^3)
//   tensor memory : dinv and the three forward edge weights of the thread's 32 voxels
//                   (tcgen05.st once per brick, tcgen05.ld every iteration; 128 columns)
//   registers     : r and q of the thread's 32 voxels
//
// Halo planes of p travel to the neighbouring CTAs through distributed shared memory
// (st.async.shared::cluster, completing in bytes on the receiver's mbarrier); the two dot
// products per iteration are reduced over the cluster by st.async'ing each CTA's fp64
// partial into every CTA's slot array and summing the CL slots in rank order once that
// CTA's mbarrier phase completes, so every CTA takes the same alpha/beta/stop decision
// and no cluster barrier is needed inside the iteration loop.  The cluster grabs the next brick from a global counter when it is done
// (persistent, load-balanced over bricks with different iteration counts).  HBM traffic
// per brick is one read of W/dinv/x/r and one write of the result; per iteration none.
//
// Thread map (N = brick x/y extent, QX = N/4 quads per row, T = QX * N/2 threads):
// thread t owns the x-quad qx = t % QX of rows y = 2j, 2j+1 (j = t / QX) in all ZS planes
// of its slab: 2*ZS "items" of 4 voxels.  The x-neighbours of a quad come by warp shuffle,
// the y-neighbours and z-neighbours from the shared p planes.
#include "cg_device.cuh"
#include "resident.cuh"
#include "tma.cuh"

namespace rw {

namespace res {

template <int N, int CL>
struct Cfg {
  // CTA grid over the brick: GY slabs along y x GZ along z (2-D split: half the halo of a
  // z-only split for the same voxels per CTA)
  static constexpr int GY = CL >= 16 ? 4 : 2;
  static constexpr int GZ = CL / GY;
  static constexpr int NZ = N;              // cubic bricks
  static constexpr int BY = N / GY;         // rows per CTA
  static constexpr int BZ = NZ / GZ;        // planes per CTA
  static constexpr int QX = N / 4;          // quads per row
  static constexpr int NJ = BY / 2;         // row pairs per CTA
  static constexpr int NG = BZ / 4;         // groups of 4 planes per CTA
  static constexpr int T = QX * NJ * NG;    // threads per CTA: one per (quad, row pair, group)
  static constexpr int NI = 8;              // items (quads) per thread: 2 rows x 4 planes
  static constexpr int PR = BY + 2;         // rows of a padded p plane (halo rows -1, BY)
  static constexpr int PP = PR * N;         // floats per padded p plane
  static constexpr int FZ = BY * N;         // floats of a z face
  static constexpr int FY = BZ * N;         // floats of a y face
  static constexpr int oP = 0;                          // p   [BZ+2][BY+2][N] (halo faces)
  static constexpr int oWX = oP + (BZ + 2) * PP;        // +x weights [BZ][BY][N]
  static constexpr int oWYM = oWX + BZ * BY * N;        // -y weight of rows 2j [BZ][NJ][N]
  static constexpr int oWZM = oWYM + BZ * NJ * N;       // -z weight of plane 4g [NG][BY][N]
  static constexpr int oZH = oWZM + NG * BY * N;        // z = dinv r of the cells across the
                                                        // 4 faces: -z, +z [BY][N], -y, +y [BZ][N]
  static constexpr int nF = oZH + 2 * FZ + 2 * FY;
  static constexpr int SMEM = nF * 4;
  static constexpr int NW = T / 32;
  static constexpr int TCOLS = T >= 512 ? 512 : 128;    // 128 columns per thread
  static_assert(T % 128 == 0, "thread count must be a multiple of 4 warps");
  static_assert(BZ % 4 == 0 && BY % 2 == 0, "block must hold whole groups / row pairs");
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

__device__ __forceinline__ uint32_t sptr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cl4(uint32_t a, float4 v) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};"
               :: "r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ void st_cl_f64(uint32_t a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" :: "r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void st_cl_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" :: "r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void cl_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cl_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ int cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return (int)r;
}

// TMEM: one x4 load (32-bit lanes x 4 columns) completed before the registers are used:
// the wait sits in the same asm statement, so no use of the outputs can be hoisted above it.
__device__ __forceinline__ float4 tm_ld4(uint32_t ta) {
  uint32_t a, b, c, d;
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(ta));
  return make_float4(__uint_as_float(a), __uint_as_float(b), __uint_as_float(c), __uint_as_float(d));
}
// three x4 loads, one wait
__device__ __forceinline__ void tm_ld4x3(uint32_t t0, uint32_t t1, uint32_t t2, float4& u,
                                         float4& v, float4& w) {
  uint32_t a[12];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%12];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4, %5, %6, %7}, [%13];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%8, %9, %10, %11}, [%14];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]),
        "=r"(a[7]), "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11])
      : "r"(t0), "r"(t1), "r"(t2));
  u = make_float4(__uint_as_float(a[0]), __uint_as_float(a[1]), __uint_as_float(a[2]), __uint_as_float(a[3]));
  v = make_float4(__uint_as_float(a[4]), __uint_as_float(a[5]), __uint_as_float(a[6]), __uint_as_float(a[7]));
  w = make_float4(__uint_as_float(a[8]), __uint_as_float(a[9]), __uint_as_float(a[10]), __uint_as_float(a[11]));
}
__device__ __forceinline__ void tm_st4(uint32_t ta, float4 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};"
               :: "r"(ta), "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)),
                  "r"(__float_as_uint(v.z)), "r"(__float_as_uint(v.w)) : "memory");
}
__device__ __forceinline__ void tm_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// 32 consecutive columns (8 float4) in one load
__device__ __forceinline__ void tm_ld32(uint32_t ta, float4 (&v)[8]) {
  uint32_t a[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]),
        "=r"(a[7]), "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]),
        "=r"(a[14]), "=r"(a[15]), "=r"(a[16]), "=r"(a[17]), "=r"(a[18]), "=r"(a[19]),
        "=r"(a[20]), "=r"(a[21]), "=r"(a[22]), "=r"(a[23]), "=r"(a[24]), "=r"(a[25]),
        "=r"(a[26]), "=r"(a[27]), "=r"(a[28]), "=r"(a[29]), "=r"(a[30]), "=r"(a[31])
      : "r"(ta));
#pragma unroll
  for (int i = 0; i < 8; ++i)
    v[i] = make_float4(__uint_as_float(a[4 * i]), __uint_as_float(a[4 * i + 1]),
                       __uint_as_float(a[4 * i + 2]), __uint_as_float(a[4 * i + 3]));
}
// 8 columns (2 float4)
__device__ __forceinline__ void tm_ld8(uint32_t ta, float4& u, float4& v) {
  uint32_t a[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]),
        "=r"(a[7])
      : "r"(ta));
  u = make_float4(__uint_as_float(a[0]), __uint_as_float(a[1]), __uint_as_float(a[2]), __uint_as_float(a[3]));
  v = make_float4(__uint_as_float(a[4]), __uint_as_float(a[5]), __uint_as_float(a[6]), __uint_as_float(a[7]));
}
// three 8-column loads, one wait
__device__ __forceinline__ void tm_ld8x3(uint32_t t0, uint32_t t1, uint32_t t2, float4& a0,
                                         float4& a1, float4& b0, float4& b1, float4& c0,
                                         float4& c1) {
  uint32_t a[24];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%24];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%8, %9, %10, %11, %12, %13, %14, %15}, [%25];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%16, %17, %18, %19, %20, %21, %22, %23}, [%26];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]),
        "=r"(a[7]), "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]),
        "=r"(a[14]), "=r"(a[15]), "=r"(a[16]), "=r"(a[17]), "=r"(a[18]), "=r"(a[19]),
        "=r"(a[20]), "=r"(a[21]), "=r"(a[22]), "=r"(a[23])
      : "r"(t0), "r"(t1), "r"(t2));
  auto F = [&](int i) {
    return make_float4(__uint_as_float(a[i]), __uint_as_float(a[i + 1]), __uint_as_float(a[i + 2]),
                       __uint_as_float(a[i + 3]));
  };
  a0 = F(0); a1 = F(4); b0 = F(8); b1 = F(12); c0 = F(16); c1 = F(20);
}
// DSMEM stores that complete (in bytes) on the receiving CTA's mbarrier
__device__ __forceinline__ void st_async4(uint32_t a, float4 v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
               :: "r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(bar) : "memory");
}
__device__ __forceinline__ void st_async_f64(uint32_t a, double v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
               :: "r"(a), "l"(__double_as_longlong(v)), "r"(bar) : "memory");
}
__device__ __forceinline__ void st_async_f64x2(uint32_t a, double u, double v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];"
               :: "r"(a), "l"(__double_as_longlong(u)), "l"(__double_as_longlong(v)), "r"(bar)
               : "memory");
}
// edge-difference stencil (reading c8) of one quad: voxel e has x-neighbours (e-1, e+1)
// inside the quad or xl / xr across it; same term order as stencil1
__device__ __forceinline__ float4 stencil4(float4 p, float xl, float xr, float4 yp, float4 ym,
                                           float4 zp, float4 zm, float4 wx, float4 wxm,
                                           float4 wy, float4 wym, float4 wz, float4 wzm) {
  float4 q;
  q.x = stencil1(p.x, p.y, xl, yp.x, ym.x, zp.x, zm.x, wx.x, wxm.x, wy.x, wym.x, wz.x, wzm.x, 1.f);
  q.y = stencil1(p.y, p.z, p.x, yp.y, ym.y, zp.y, zm.y, wx.y, wxm.y, wy.y, wym.y, wz.y, wzm.y, 1.f);
  q.z = stencil1(p.z, p.w, p.y, yp.z, ym.z, zp.z, zm.z, wx.z, wxm.z, wy.z, wym.z, wz.z, wzm.z, 1.f);
  q.w = stencil1(p.w, xr, p.z, yp.w, ym.w, zp.w, zm.w, wx.w, wxm.w, wy.w, wym.w, wz.w, wzm.w, 1.f);
  return q;
}
// edge-difference stencil (reading c8) split by axis, same term order as stencil1:
// q = wx (p - p[+x]);  q += wxm (p - p[-x]);  then +y, -y, +z, -z the same way
__device__ __forceinline__ float4 xterms(float4 p, float xl, float xr, float4 wx, float wl) {
  float4 q;
  q.x = __fmaf_rn(wl, __fsub_rn(p.x, xl), __fmul_rn(wx.x, __fsub_rn(p.x, p.y)));
  q.y = __fmaf_rn(wx.x, __fsub_rn(p.y, p.x), __fmul_rn(wx.y, __fsub_rn(p.y, p.z)));
  q.z = __fmaf_rn(wx.y, __fsub_rn(p.z, p.y), __fmul_rn(wx.z, __fsub_rn(p.z, p.w)));
  q.w = __fmaf_rn(wx.z, __fsub_rn(p.w, p.z), __fmul_rn(wx.w, __fsub_rn(p.w, xr)));
  return q;
}
__device__ __forceinline__ float4 terms2(float4 q, float4 p, float4 pp, float4 pm, float4 wp,
                                         float4 wm) {
  q.x = __fmaf_rn(wm.x, __fsub_rn(p.x, pm.x), __fmaf_rn(wp.x, __fsub_rn(p.x, pp.x), q.x));
  q.y = __fmaf_rn(wm.y, __fsub_rn(p.y, pm.y), __fmaf_rn(wp.y, __fsub_rn(p.y, pp.y), q.y));
  q.z = __fmaf_rn(wm.z, __fsub_rn(p.z, pm.z), __fmaf_rn(wp.z, __fsub_rn(p.z, pp.z), q.z));
  q.w = __fmaf_rn(wm.w, __fsub_rn(p.w, pm.w), __fmaf_rn(wp.w, __fsub_rn(p.w, pp.w), q.w));
  return q;
}
__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;   // identical in every lane
}
// q = 0 on fixed voxels (bit e of fm)
__device__ __forceinline__ float4 mask4(float4 q, uint32_t fm) {
  if (fm & 1u) q.x = 0.f;
  if (fm & 2u) q.y = 0.f;
  if (fm & 4u) q.z = 0.f;
  if (fm & 8u) q.w = 0.f;
  return q;
}

}  // namespace res


template <int N, int CL>
__global__ void __launch_bounds__(res::Cfg<N, CL>::T, 1) k_resident(ResArgs A) {
  using G = res::Cfg<N, CL>;
  using namespace res;
  constexpr int QX = G::QX, NI = G::NI, NW = G::NW, BY = G::BY, BZ = G::BZ, PP = G::PP;
  constexpr int GY = G::GY, GZ = G::GZ, FZ = G::FZ, FY = G::FY;
  extern __shared__ __align__(16) float sm[];
  // mbarriers: [0] halo z values in, [1] p.q partials in, [2] (r.z, r.r) partials in
  __shared__ __align__(8) uint64_t s_bar[3];
  __shared__ __align__(16) double s_pq_slots[CL];  // p.q partial of every CTA (rank order)
  __shared__ __align__(16) double2 s_rz_slots[CL];  // (r.z, r.r) partial of every CTA
  __shared__ float2 s_bredf[NW];
  __shared__ int s_brick;
  // CG scalars, updated by thread 0 only (fp64 state kept out of the per-thread registers)
  __shared__ double s_rz, s_rrn, s_bb, s_pq, s_thr;
  __shared__ int s_st, s_k;
  __shared__ float s_be, s_al;
  __shared__ uint32_t s_taddr;
  const int t = threadIdx.x, warp = t >> 5;
  const int rank = cl_rank();
  const int gy = rank % GY, gz = rank / GY;
  const int qx = t % QX, j = (t / QX) % G::NJ, g = t / (QX * G::NJ);
  float* const P = sm + G::oP;
  float* const WX = sm + G::oWX;
  float* const WYM = sm + G::oWYM;
  float* const WZM = sm + G::oWZM;
  float* const ZH = sm + G::oZH;
  // padded p index of (local plane zl in -1..BZ, local row y in -1..BY), x = 0
  auto pidx = [&](int zl, int y) { return ((zl + 1) * G::PR + (y + 1)) * N; };

  // ---- tensor memory: 128 columns per thread (lane = 32*(warp%4) + lane id)
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(sptr(&s_taddr)), "n"(G::TCOLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (t == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(&s_bar[i], 1);
    fence_mbar_init();
  }
  // p starts at 0 everywhere, halo faces included (faces on the brick boundary stay 0)
  for (int i = t; i < G::oWX; i += G::T) P[i] = 0.f;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = s_taddr + ((uint32_t)(32 * (warp & 3)) << 16) + 128u * (uint32_t)(warp >> 2);
  // column map: dinv(it) = 4it, x(it) = 32+4it, wy(it) = 64+4it, wz(it) = 96+4it with
  // it = 2i + rr (i = plane within the thread's group of 4, rr = row of the pair); the +x
  // weights live in shared memory (tensor memory is full)
  const uint32_t cD = tb, cX = tb + 32u, cY = tb + 64u, cZ = tb + 96u;

  const int y0 = gy * BY, z0 = gz * BZ;
  const long long n = (long long)N * N * G::NZ;
  const long long PL = (long long)N * N;
  const long long BN = (long long)A.B * n;
  // neighbours across the 4 faces f = -z, +z, -y, +y (bit f of hmask) and where my boundary
  // z values go: my plane 0 feeds the -z neighbour's +z face, my last plane the +z
  // neighbour's -z face, my row 0 the -y neighbour's +y face, my last row the +y
  // neighbour's -y face.  (Scalars and constant-index arrays only: no local memory.)
  const uint32_t hmask = (gz > 0 ? 1u : 0u) | (gz < GZ - 1 ? 2u : 0u) | (gy > 0 ? 4u : 0u) |
                         (gy < GY - 1 ? 8u : 0u);
  auto foff = [](int f) { return f < 2 ? f * FZ : 2 * FZ + (f - 2) * FY; };
  auto face_of = [](int e) { return e < FZ ? 0 : e < 2 * FZ ? 1 : e < 2 * FZ + FY ? 2 : 3; };
  const uint32_t halo_bytes = ((hmask & 1u) ? FZ * 4u : 0u) + ((hmask & 2u) ? FZ * 4u : 0u) +
                              ((hmask & 4u) ? FY * 4u : 0u) + ((hmask & 8u) ? FY * 4u : 0u);
  uint32_t rface[4], rbar[4];
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int nb = f == 0 ? rank - GY : f == 1 ? rank + GY : f == 2 ? rank - 1 : rank + 1;
    const bool h = (hmask >> f) & 1u;
    rface[f] = h ? mapa(sptr(ZH + foff(f ^ 1)), nb) : 0u;
    rbar[f] = h ? mapa(sptr(&s_bar[0]), nb) : 0u;
  }
  const uint32_t brk = sptr(&s_brick);
  uint32_t ph0 = 0, ph1 = 0, ph2 = 0;   // mbarrier phase parities

  // Cluster-wide fp64 sum of nv (1 or 2) per-thread fp32 partials, identical in every
  // thread of every CTA: warp xor-shuffle tree -> per-warp partials -> thread 0 adds them
  // in warp order (fp64) and st.async's the CTA partial into slot `rank` of every CTA (one
  // 8/16-byte message per CTA pair, completing on that CTA's mbarrier `bi`; many small
  // messages cost far more, tools/micro/mb_red.cu); warp 0 waits for the CL partials,
  // thread 0 adds them in rank order, and a CTA barrier hands the result to every thread.
  auto cluster_sum = [&](float f0, float f1, int nv, int bi, auto* slots, uint32_t& ph,
                         auto&& shadow, auto&& epilogue) {
    f0 = warp_sum_f(f0);
    if (nv > 1) f1 = warp_sum_f(f1);
    if ((t & 31) == 0) s_bredf[warp] = make_float2(f0, f1);
    __syncthreads();
    if (t == 0) {
      double a0 = 0.0, a1 = 0.0;
      for (int w = 0; w < NW; ++w) {
        const float2 e = s_bredf[w];
        a0 += (double)e.x;
        a1 += (double)e.y;
      }
      mbar_arrive_expect_tx(&s_bar[bi], CL * 8u * nv);
      const uint32_t slot = sptr(&slots[rank]), bar = sptr(&s_bar[bi]);
      for (int c = 0; c < CL; ++c) {
        if (nv == 1) st_async_f64(mapa(slot, c), a0, mapa(bar, c));
        else st_async_f64x2(mapa(slot, c), a0, a1, mapa(bar, c));
      }
    }
    shadow();   // independent work while the partials travel
    if (warp == 0) {
      mbar_wait(&s_bar[bi], ph);
      if (t == 0) {
        double a0 = 0.0, a1 = 0.0;
        for (int c = 0; c < CL; ++c) {
          if (nv == 1) {
            a0 += reinterpret_cast<const double*>(slots)[c];
          } else {
            const double2 e = reinterpret_cast<const double2*>(slots)[c];
            a0 += e.x;
            a1 += e.y;
          }
        }
        epilogue(make_double2(a0, a1));   // thread 0 updates the CG scalars
      }
    }
    ph ^= 1u;
    __syncthreads();
  };

  float4 r[NI], q[NI];
  while (true) {
    // ---- next brick (rank 0 draws it, DSMEM broadcast, cluster barrier)
    if (rank == 0 && t == 0) {
      const int nb = atomicAdd(A.next, 1);
      for (int c = 0; c < CL; ++c) st_cl_u32(mapa(brk, c), (uint32_t)nb);
    }
    cl_arrive();
    cl_wait();
    const int b = s_brick;
    if (b >= A.B) break;
    const long long gb = (long long)b * n;

    // ---- load the block: W, dinv -> TMEM; r -> registers; x, -y/-z weights -> smem
    uint32_t fixm = 0;   // bit 4*it+e: voxel is fixed (dinv == 0)
#pragma unroll
    for (int it = 0; it < NI; ++it) {
      const int i = it >> 1, rr = it & 1, zl = 4 * g + i, y = 2 * j + rr;
      const long long gi = gb + (long long)(z0 + zl) * PL + (y0 + y) * N + 4 * qx;
      const float4 dv = ld4(A.dinv + gi);
      tm_st4(cD + 4u * it, dv);
      tm_st4(cX + 4u * it, ld4(A.x + gi));
      tm_st4(cY + 4u * it, ld4(A.W + BN + gi));
      tm_st4(cZ + 4u * it, ld4(A.W + 2 * BN + gi));
      fixm |= (dv.x == 0.f ? 1u : 0u) << (4 * it);
      fixm |= (dv.y == 0.f ? 2u : 0u) << (4 * it);
      fixm |= (dv.z == 0.f ? 4u : 0u) << (4 * it);
      fixm |= (dv.w == 0.f ? 8u : 0u) << (4 * it);
      r[it] = ld4(A.r0 + gi);
      st4(WX + (zl * BY + y) * N + 4 * qx, ld4(A.W + gi));
      st4(P + pidx(zl, y) + 4 * qx, f4(0.f));
      if (rr == 0)
        st4(WYM + (zl * G::NJ + j) * N + 4 * qx, y0 + y > 0 ? ld4(A.W + BN + gi - N) : f4(0.f));
      if (i == 0)
        st4(WZM + (g * BY + y) * N + 4 * qx, z0 + zl > 0 ? ld4(A.W + 2 * BN + gi - PL) : f4(0.f));
    }
    // z0 = dinv r0 of the cells across my faces (the neighbours send the later ones)
    for (int u = t; u < (2 * FZ + 2 * FY) / 4; u += G::T) {
      const int e = 4 * u;
      const int f = face_of(e);
      const int c = e - foff(f), a = c / N, x = c % N;   // a = row (z faces) / plane (y faces)
      float4 zv = f4(0.f);
      if ((hmask >> f) & 1u) {
        const int gz_ = f == 0 ? z0 - 1 : f == 1 ? z0 + BZ : z0 + a;
        const int gy_ = f == 2 ? y0 - 1 : f == 3 ? y0 + BY : y0 + a;
        const long long gi = gb + (long long)gz_ * PL + gy_ * N + x;
        zv = mul4(ld4(A.dinv + gi), ld4(A.r0 + gi));
      }
      st4(ZH + e, zv);
    }
    res::tm_wait_st();
    // ---- initial scalars from the setup partials (fixed order), decision of iteration 0
    // (as passA_scalars): thread 0 owns the CG scalars from here on
    if (t == 0) {
      double rz = 0.0, rrn = 0.0, bb = 0.0, nf = 0.0, nu = 0.0;
      for (int u = 0; u < A.U; ++u) {
        const double2 pb = A.PB[(long long)b * A.U + u];
        const double4 ps = A.PS[(long long)b * A.U + u];
        rz += pb.x; rrn += pb.y; bb += ps.x; nf += ps.y; nu += ps.z;
      }
      const double t2 = (double)A.C.tol * (double)A.C.tol;
      s_thr = A.C.tol_mode == 0 ? t2 * bb : t2;
      int st = ST_ACTIVE;
      if (nf == 0.0 || nu == 0.0) st = ST_TRIVIAL;
      else if (bb == 0.0) st = ST_ZERO_B;
      else if (rrn <= s_thr) st = ST_CONVERGED;
      else if (A.C.max_iter <= 0) st = ST_MAXITER;
      s_st = st;
      s_k = 0;
      s_rz = rz;
      s_rrn = rrn;
      s_bb = bb;
      s_be = 0.f;
    }
    __syncthreads();

    int k = 0;
    float al = 0.f;   // alpha_k
    while (true) {
      if (s_st != ST_ACTIVE) {
        if (k > 0) {   // consume the halo phase iteration k-1 sent (keeps phases in step)
          mbar_wait(&s_bar[0], ph0);
          ph0 ^= 1u;
        }
        break;
      }
      const float be = s_be;
#ifdef RW_RES_TIMING
      long long tp0 = A.dbg ? clock64() : 0;
      auto TP = [&](int i) {   // debug phase timer: cluster 0, per rank
        if (A.dbg && t == 0 && blockIdx.x < CL) {
          const long long now = clock64();
          A.dbg[rank * 8 + i] += now - tp0;
          tp0 = now;
        }
      };
#else
      auto TP = [](int) {};
#endif

      // ---- step 1: p_k = z_k + beta p_{k-1} on the own cells (z = dinv r) and on the halo
      // faces (z of the cells across the faces arrived during the previous reduction)
      {
        float4 dv[NI];
        tm_ld32(cD, dv);
#pragma unroll
        for (int it = 0; it < NI; ++it) {
          const int i = it >> 1, rr = it & 1, zl = 4 * g + i, y = 2 * j + rr;
          const int so = pidx(zl, y) + 4 * qx;
          st4(P + so, pnew4(be, ld4(P + so), dv[it], r[it]));
        }
      }
      TP(0);
      if (k > 0) {
        mbar_wait(&s_bar[0], ph0);
        ph0 ^= 1u;
      }
      TP(1);
      for (int u = t; u < (2 * FZ + 2 * FY) / 4; u += G::T) {
        const int e = 4 * u;
        const int f = face_of(e);
        if (!((hmask >> f) & 1u)) continue;
        const int c = e - foff(f), a = c / N, x = c % N;
        const int po = (f == 0 ? pidx(-1, a) : f == 1 ? pidx(BZ, a)
                        : f == 2 ? pidx(a, -1) : pidx(a, BY)) + x;
        st4(P + po, fma4(be, ld4(P + po), ld4(ZH + e)));
      }
      __syncthreads();
      TP(2);

      // ---- step 2: q = L_UU p (edge-difference stencil), partial p.q; one row pair
      // (items 2i, 2i+1) at a time.  Halo faces are part of the padded p planes.
      float apq = 0.f;   // this thread's p.q (fp32 over its 32 voxels; fp64 beyond)
      {
        // sliding window over the thread's 4 planes: rows 2j, 2j+1 of planes zl-1, zl, zl+1
        const int sb = pidx(4 * g, 2 * j) + 4 * qx;
        float4 pm0 = ld4(P + sb - PP), pm1 = ld4(P + sb - PP + N);
        float4 p0 = ld4(P + sb), p1 = ld4(P + sb + N);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int zl = 4 * g + i;
          const int so = sb + i * PP;
          const float4 pn0 = ld4(P + so + PP), pn1 = ld4(P + so + PP + N);
          float4 q0, q1;
          {  // x terms (same term order as stencil1: +x, -x, +y, -y, +z, -z)
            const float* wxp = WX + (zl * BY + 2 * j) * N + 4 * qx;
            const float4 wx0 = ld4(wxp), wx1 = ld4(wxp + N);
            const float xl0 = __shfl_up_sync(0xffffffffu, p0.w, 1, QX);
            const float xr0 = __shfl_down_sync(0xffffffffu, p0.x, 1, QX);
            const float xl1 = __shfl_up_sync(0xffffffffu, p1.w, 1, QX);
            const float xr1 = __shfl_down_sync(0xffffffffu, p1.x, 1, QX);
            const float wl0 = __shfl_up_sync(0xffffffffu, wx0.w, 1, QX);
            const float wl1 = __shfl_up_sync(0xffffffffu, wx1.w, 1, QX);
            q0 = xterms(p0, xl0, xr0, wx0, qx > 0 ? wl0 : 0.f);
            q1 = xterms(p1, xl1, xr1, wx1, qx > 0 ? wl1 : 0.f);
          }
          {  // y terms: row 2j+1 is +y of row 2j (and row 2j is -y of row 2j+1)
            float4 wy0, wy1;
            tm_ld8(cY + 8u * i, wy0, wy1);
            const float4 wym0 = ld4(WYM + (zl * G::NJ + j) * N + 4 * qx);
            q0 = terms2(q0, p0, p1, ld4(P + so - N), wy0, wym0);
            q1 = terms2(q1, p1, ld4(P + so + 2 * N), p0, wy1, wy0);
          }
          {  // z terms
            float4 wz0, wz1, wzm0, wzm1;
            tm_ld8(cZ + 8u * i, wz0, wz1);
            if (i == 0) {
              wzm0 = ld4(WZM + (g * BY + 2 * j) * N + 4 * qx);
              wzm1 = ld4(WZM + (g * BY + 2 * j + 1) * N + 4 * qx);
            } else {
              tm_ld8(cZ + 8u * (i - 1), wzm0, wzm1);
            }
            q0 = terms2(q0, p0, pn0, pm0, wz0, wzm0);
            q1 = terms2(q1, p1, pn1, pm1, wz1, wzm1);
          }
          const uint32_t fm = fixm >> (8 * i);
          q0 = mask4(q0, fm);
          q1 = mask4(q1, fm >> 4);
          q[2 * i] = q0;
          q[2 * i + 1] = q1;
          apq = __fadd_rn(apq, __fadd_rn(dot4f(p0, q0), dot4f(p1, q1)));
          pm0 = p0; pm1 = p1; p0 = pn0; p1 = pn1;
        }
      }
      TP(3);
      cluster_sum(apq, 0.f, 1, 1, s_pq_slots, ph1, [] {}, [&](double2 v) {
        const double pq = v.x;
        s_pq = pq;
        s_al = (pq > 0.0 && isfinite(pq)) ? (float)(s_rz / pq) : 0.f;
      });
      al = s_al;
      TP(4);

      // ---- step 3: r -= alpha q;  z = dinv r;  boundary z to the neighbours' face buffers
      // (st.async, landing while the reduction below runs);  partials r.z, r.r
      if (t == 0 && halo_bytes) mbar_arrive_expect_tx(&s_bar[0], halo_bytes);
      float arz = 0.f, arr = 0.f;
      {
        float4 dv[NI];
        tm_ld32(cD, dv);
#pragma unroll
        for (int it = 0; it < NI; ++it) {
          const int i = it >> 1, rr = it & 1, zl = 4 * g + i, y = 2 * j + rr;
          const float4 rn = fma4(-al, q[it], r[it]);
          r[it] = rn;
          const float4 zn = mul4(dv[it], rn);
          if (zl == 0 && (hmask & 1u)) st_async4(rface[0] + (uint32_t)(y * N + 4 * qx) * 4u, zn, rbar[0]);
          if (zl == BZ - 1 && (hmask & 2u)) st_async4(rface[1] + (uint32_t)(y * N + 4 * qx) * 4u, zn, rbar[1]);
          if (y == 0 && (hmask & 4u)) st_async4(rface[2] + (uint32_t)(zl * N + 4 * qx) * 4u, zn, rbar[2]);
          if (y == BY - 1 && (hmask & 8u)) st_async4(rface[3] + (uint32_t)(zl * N + 4 * qx) * 4u, zn, rbar[3]);
          arz = __fadd_rn(arz, dot4f(rn, zn));
          arr = __fadd_rn(arr, dot4f(rn, rn));
        }
      }
      TP(5);
      // x_{k+1} = x_k + alpha_k p_k (own cells, x in tensor memory) in the reduction's shadow
      cluster_sum(arz, arr, 2, 2, s_rz_slots, ph2, [&] {
        float4 xv[NI];
        tm_ld32(cX, xv);
#pragma unroll
        for (int it = 0; it < NI; ++it) {
          const int zl = 4 * g + (it >> 1), y = 2 * j + (it & 1);
          tm_st4(cX + 4u * it, fma4(al, ld4(P + pidx(zl, y) + 4 * qx), xv[it]));
        }
        res::tm_wait_st();
      }, [&](double2 v) {   // thread 0: decision of iteration k+1 (as passA_scalars), beta_k
        const double rz_new = v.x, pq = s_pq;
        int st = ST_ACTIVE;
        if (!(pq > 0.0) || !isfinite(rz_new) || !isfinite(pq)) st = ST_BREAKDOWN;
        else if (v.y <= s_thr) st = ST_CONVERGED;
        else if (s_k + 1 >= A.C.max_iter) st = ST_MAXITER;
        s_st = st;
        s_be = (float)(rz_new / s_rz);
        s_rz = rz_new;
        s_rrn = v.y;
        s_k = s_k + 1;
      });
      TP(6);
      ++k;
    }

    // ---- finalise (row a6): clamp, fixed values kept, labels.  x already holds x_k (the
    // update of iteration k-1 ran in the shadow of its last reduction).
    const int st = s_st;
    float4 xfin[NI];
    tm_ld32(cX, xfin);
#pragma unroll
    for (int it = 0; it < NI; ++it) {
      const int i = it >> 1, rr = it & 1, zl = 4 * g + i, y = 2 * j + rr;
      const float4 xv = xfin[it];
      const uint32_t fm = fixm >> (4 * it);
      float o[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (fm & (1u << e)) continue;            // fixed: x holds the Dirichlet value
        o[e] = st == ST_ZERO_B ? 0.f : fminf(fmaxf(o[e], 0.f), 1.f);
      }
      const long long gi = gb + (long long)(z0 + zl) * PL + (y0 + y) * N + 4 * qx;
      st4(A.x + gi, make_float4(o[0], o[1], o[2], o[3]));
      if (A.labels)
        *reinterpret_cast<uchar4*>(A.labels + gi) =
            make_uchar4(o[0] > 0.5f, o[1] > 0.5f, o[2] > 0.5f, o[3] > 0.5f);
    }
    if (rank == 0 && t == 0) {
      A.status[b] = st;
      A.iters[b] = (st == ST_TRIVIAL || st == ST_ZERO_B) ? 0 : k;
      if (A.resid) {
        double res = 0.0;
        if (st == ST_CONVERGED || st == ST_MAXITER || st == ST_BREAKDOWN) {
          res = sqrt(s_rrn);
          if (A.C.tol_mode == 0) res = s_bb > 0.0 ? res / sqrt(s_bb) : 0.0;
        }
        A.resid[b] = (float)res;
      }
    }
  }
  // ---- release tensor memory
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;"
                 :: "r"(s_taddr), "n"(G::TCOLS) : "memory");
}

// ------------------------------------------------------------------------- launcher
// Supported shapes: N x N x 4*CL bricks with (N, CL) in {(64, 16), (32, 8)}.
template <int N, int CL>
static int resident_clusters() {
  static int cached = -1;
  if (cached >= 0) return cached;
  using G = res::Cfg<N, CL>;
  int nc = 0;
  if (cudaFuncSetAttribute(k_resident<N, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           G::SMEM) != cudaSuccess ||
      (CL > 8 && cudaFuncSetAttribute(k_resident<N, CL>,
                                      cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)) {
    cudaGetLastError();
    cached = 0;
    return 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL);
  cfg.blockDim = dim3(G::T);
  cfg.dynamicSmemBytes = G::SMEM;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (cudaOccupancyMaxActiveClusters(&nc, k_resident<N, CL>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    nc = 0;
  }
  cached = nc;
  return nc;
}

template <int N, int CL>
static cudaError_t launch_res(const ResArgs& A, cudaStream_t s) {
  using G = res::Cfg<N, CL>;
  const int nc = resident_clusters<N, CL>();
  if (nc < 1) return cudaErrorNotSupported;
  const int ncl = nc < A.B ? nc : A.B;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncl * CL);
  cfg.blockDim = dim3(G::T);
  cfg.dynamicSmemBytes = G::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_resident<N, CL>, A);
}

// Is the resident solver available for this brick shape (and device)?
bool resident_supported(int nx, int ny, int nz, int R) {
  if (R != 1) return false;
  if (nx == 64 && ny == 64 && nz == 64) return resident_clusters<64, 16>() > 0;
  if (nx == 32 && ny == 32 && nz == 32) return resident_clusters<32, 8>() > 0;
  return false;
}

cudaError_t launch_resident(int nx, const ResArgs& A, cudaStream_t s) {
  if (nx == 64) return launch_res<64, 16>(A, s);
  return launch_res<32, 8>(A, s);
}

}  // namespace rw
