// resident.cuh -- arguments of the brick-resident CG kernel (resident.cu).
#pragma once
#include "rw_common.cuh"

namespace rw {

struct ResArgs {
  const float* W;      // [3][B][n]
  const float* dinv;   // [B][n]   0 on fixed voxels
  const float* r0;     // [B][n]   initial residual (k_setup)
  float* x;            // [B][n]   in: x0 with fixed values (k_setup); out: prob
  const double2* PB;   // [2][B][U] setup partials (r.z, r.r) in slot 0
  const double4* PS;   // [B][U]    (b.b, n_fixed, n_unknown, 0)
  int B, U;            // B: batch of the arrays (plane stride of W); U: setup partials per brick
  int nsolve;          // bricks 0 .. nsolve-1 are solved (<= B; the rest run elsewhere)
  int* next;           // brick counter (zeroed before the launch)
  int* iters;          // [B]
  int* status;         // [B]
  float* resid;        // [B] or null
  uint8_t* labels;     // [B][n] or null
  Ctl C;
  long long* dbg;      // debug: per-(rank, phase) clock64 sums, or null (RW_DEBUG_RES_TIMING)
};

bool resident_supported(int nx, int ny, int nz, int R);
cudaError_t launch_resident(int nx, const ResArgs& A, cudaStream_t s);

}  // namespace rw
