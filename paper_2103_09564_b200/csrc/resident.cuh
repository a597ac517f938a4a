// resident.cuh -- arguments of the brick-resident CG kernel (resident.cu).
#pragma once
#include "rw_common.cuh"

namespace rw {

struct ResArgs {
  const float* W;      // [3][B][n]
  const float* dinv;   // [B][n]   0 on fixed voxels
  const float* r0;     // [R][B][n] initial residual (k_setup)
  float* x;            // [R][B][n] in: x0 with fixed values (k_setup); out: prob
  const double2* PB;   // [2][R][B][U] setup partials (r.z, r.r) in slot 0
  const double4* PS;   // [R][B][U]    (b.b, n_fixed, n_unknown, 0)
  int B, U;            // B: batch of the arrays (plane stride of W); U: setup partials per brick
  int nb;              // bricks 0 .. nb-1 of every rhs are solved here (<= B; the rest run
                       // elsewhere)
  int nsolve;          // (rhs, brick) pairs solved = R * nb; pair i = (i / nb, i % nb)
  int* next;           // pair counter (zeroed before the launch)
  int* iters;          // [R][B]
  int* status;         // [R][B]
  float* resid;        // [R][B] or null
  uint8_t* labels;     // [B][n] or null (R == 1 only)
  Ctl C;
  // fused assembly (vol != null): weights, dinv, x0 and r0 are formed in the brick load
  // phase from the intensities, the Dirichlet mask / values and x0 (no k_weights / k_setup)
  const void* vol;       // [B][n] of dtype vdt, or null (then W / dinv / r0 / x / PB / PS)
  int vdt;               // VM_U8 .. VM_F32
  const uint8_t* fixed;  // [B][n]
  const float* values;   // [R][B][n]
  const float* x0;       // [R][B][n] or null (0.5)
  long long* dbg;      // debug builds only (-DRW_RES_TIMING): per-(rank, phase) clock64 sums
                       // in a caller-provided buffer; null in the library
  // host-streamed solve (rw_solve_bricks_host, ring > 0): brick b's vol / fixed / values /
  // x / labels live in device slot b % ring (its iters / status / resid at [b]); a brick of
  // chunk c = b / chunk is started only once in_ready[c] != 0 (written by the H2D copy
  // stream after the chunk's inputs); the last finished brick of chunk c sets host_done[c]
  // (host-mapped) so the host can start the chunk's D2H copy while the launch goes on
  int ring;
  int chunk;
  const int* in_ready;   // [nchunks] device
  int* done;             // [nchunks] device, zeroed before the launch
  int* host_done;        // [nchunks] host-mapped, zeroed before the launch
  int* abort;            // device, zeroed: set when a chunk's inputs did not arrive within 2 s
                         // (e.g. a profiler serialising the launch): every cluster then exits
                         // and the host falls back to the chunked pipeline
};

// L2 workers (resident.cu k_l2res): storage of the worker clusters' CG state in global memory
struct L2Args {
  float* buf;          // nw * stride floats
  long long stride;    // floats per worker cluster (7 arrays of the brick)
  int rmin;            // a worker takes a brick only while more than rmin remain undrawn
  int* nsolved;        // debug (RW_DEBUG_L2W): bricks solved by the workers, or null
  int* done;           // experiment (RW_L2_HOLD): worker CTAs count themselves out here, or null
};
// experiment (RW_L2_HOLD): idle 16-CTA clusters holding the resident kernel's SMs until
// `target` worker CTAs have exited (or ~5 s)
cudaError_t launch_hold16(int ncl, int* done, int target, cudaStream_t s);
int l2res_workers(int ncl_res);
size_t l2res_bytes_per_worker();
int resident_clusters64(int vdt);
cudaError_t launch_l2res(const ResArgs& A, const L2Args& W, int nw, cudaStream_t s);

// vdt: the VM_* mode the launch will use (VM_U16 / VM_F32 fused from intensities, else
// VM_STORED); wide: RW_OPT_RESIDENT_WIDE
bool resident_supported(int nx, int ny, int nz, int R, int vdt, int wide);
bool resident_fused(int vdt);
cudaError_t launch_resident(int nx, const ResArgs& A, int wide, cudaStream_t s);

}  // namespace rw
