// passA.cuh -- TMA descriptors and shared-memory layout of the CG pass-A kernel.
#pragma once
#include <cuda.h>

#include "rw_common.cuh"

namespace rw {

// 3-D tiled tensor maps (x, y, plane) over the arrays pass A streams.  Arrays indexed
// [q][b][z] collapse (q, b, z) into one plane coordinate (q*B + b)*nz + z.
struct Maps {
  CUtensorMap r;    // r      [2][R][B] planes, box {TXh, TY+2, 1}
  CUtensorMap q;    // q      [2][R][B],    box {TXh, TY+2, 1}   (one-pass mode)
  CUtensorMap p;    // P      [2][R][B],    box {TXh, TY+2, 1}
  CUtensorMap x;    // x      [R][B],       box {TX, TY, 1}
  CUtensorMap d;    // dinv   [B],          box {TXh, TY+2, 1}
  CUtensorMap wx;   // W      [3][B],       box {TXh, TY, 1}     (VM_STORED)
  CUtensorMap wy;   //                      box {TX, TY+1, 1}    (VM_STORED)
  CUtensorMap wz;   //                      box {TX, TY, 1}      (VM_STORED)
  CUtensorMap v;    // vol    [B],          box {TXhv, TY+2, 1}  (VM_U8..VM_F32)
};

constexpr int kStages = 4;  // TMA ring depth (planes issued ~2 steps before use)
// one-pass mode streams the q box instead of the x box (x is read straight from global
// memory, it has no halo), so 4 stages still fit two CTAs per SM
// (kStages - 1 when the one-pass layout would otherwise drop to one CTA per SM, passA_stages)
__host__ __device__ inline int a_stages(const Plan& P) { return P.ns > 0 ? P.ns : kStages; }

__host__ __device__ inline int rup128(int b) { return (b + 127) & ~127; }
__host__ __device__ inline int vm_esize(int vm) {
  return vm == VM_U8 ? 1 : ((vm == VM_U16 || vm == VM_I16) ? 2 : 4);
}

struct ALayout {
  int eRP, eX, eWx, eWy, eWz, eV;   // exact box bytes (mbarrier transaction counts)
  int bRP, bX, bWx, bWy, bWz, bV;   // 128-byte rounded smem footprints
  int oR, oP, oQ, oX, oD, oW;       // offsets inside a stage (rhs c adds c * b..)
  int stage, sp, wys, bars, total;  // stage size; p_new planes; +y weights; mbarriers; total
};

__host__ __device__ inline ALayout a_layout(const Plan& P, int RC, int vm) {
  ALayout L;
  L.eRP = P.TXh * (P.TY + 2) * 4;
  L.eX = P.TX * P.TY * 4;
  L.eWx = P.TXh * P.TY * 4;
  L.eWy = P.TX * (P.TY + 1) * 4;
  L.eWz = L.eX;
  L.eV = P.TXhv * (P.TY + 2) * vm_esize(vm);
  L.bRP = rup128(L.eRP);
  L.bX = P.one ? 0 : rup128(L.eX);   // one-pass mode reads x straight from global memory
  L.bWx = rup128(L.eWx);
  L.bWy = rup128(L.eWy);
  L.bWz = rup128(L.eWz);
  L.bV = rup128(L.eV);
  L.oR = 0;
  L.oP = RC * L.bRP;
  L.oQ = 2 * RC * L.bRP;                      // one-pass mode: q_{k-1} boxes
  L.oX = (P.one ? 3 : 2) * RC * L.bRP;
  L.oD = L.oX + RC * L.bX;
  L.oW = L.oD + L.bRP;
  L.stage = L.oW + (vm == VM_STORED ? L.bWx + L.bWy + L.bWz : L.bV);
  L.sp = a_stages(P) * L.stage;
  L.wys = L.sp + rup128(2 * RC * (P.TY + 2) * P.TXP * 4);
  L.bars = L.wys + (vm == VM_STORED ? 0 : rup128(2 * P.TY * P.TX * 4));
  L.total = L.bars + a_stages(P) * 8;
  return L;
}

}  // namespace rw
