// queue.cu -- SURVEY §8(a) row a9: pinned, double-buffered host->device brick queue.
//
// North star item 5 / P:105 ("constant memory", brick-wise loading): inputs larger than
// HBM stream through a ring of `depth` slots.  Each slot = one pinned host buffer + one
// device buffer + two events: `ready` (H2D copy done, recorded on the copy stream) and
// `freed` (its consumers done, recorded on the compute stream).  With depth >= 2 the H2D
// copy of slot k+1 overlaps the kernels consuming slot k; the host-side staging copy of
// slot k+2 overlaps both.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/rw.h"

struct rw_queue {
  size_t slot_bytes = 0;
  int depth = 0;
  int next = 0;
  std::vector<void*> host, dev;
  std::vector<cudaEvent_t> ready, freed;
  std::vector<bool> used;
  std::vector<bool> released;   // released since its last push (or never pushed)
};

namespace rw { void set_last_error(const char* msg); }

namespace {
rw_status qfail(rw_status s, const char* m) { rw::set_last_error(m); return s; }

void parallel_copy(void* dst, const void* src, size_t bytes) {
  // pageable -> pinned staging copy split over host threads (>= 2 MB each): one thread's
  // memcpy (~10-20 GB/s) is slower than the PCIe H2D copy it feeds
  const size_t min_per = 2u << 20;
  unsigned nt = std::thread::hardware_concurrency();
  if (nt > 16) nt = 16;
  if ((size_t)nt * min_per > bytes) nt = (unsigned)(bytes / min_per);
  if (nt < 2) { std::memcpy(dst, src, bytes); return; }
  size_t per = (bytes + nt - 1) / nt;
  per = (per + 4095) & ~(size_t)4095;
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t) {
    const size_t o = (size_t)t * per;
    if (o >= bytes) break;
    const size_t n = (o + per > bytes) ? bytes - o : per;
    th.emplace_back([=] { std::memcpy((char*)dst + o, (const char*)src + o, n); });
  }
  for (auto& x : th) x.join();
}
}  // namespace

extern "C" rw_status rw_queue_create(size_t slot_bytes, int32_t depth, rw_queue** q) {
  if (!q || depth < 2 || depth > 64 || slot_bytes == 0)
    return qfail(RW_EINVAL, "rw_queue_create: need q != NULL, 2 <= depth <= 64, slot_bytes > 0");
  rw_queue* Q = new rw_queue;
  Q->slot_bytes = slot_bytes;
  Q->depth = depth;
  for (int i = 0; i < depth; ++i) {
    void *h = nullptr, *d = nullptr;
    cudaEvent_t a, b;
    if (cudaHostAlloc(&h, slot_bytes, cudaHostAllocDefault) != cudaSuccess ||
        cudaMalloc(&d, slot_bytes) != cudaSuccess ||
        cudaEventCreateWithFlags(&a, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&b, cudaEventDisableTiming) != cudaSuccess) {
      if (h) cudaFreeHost(h);
      if (d) cudaFree(d);
      rw_queue_destroy(Q);
      return qfail(RW_ENOMEM, "rw_queue_create: pinned/device allocation failed");
    }
    Q->host.push_back(h);
    Q->dev.push_back(d);
    Q->ready.push_back(a);
    Q->freed.push_back(b);
    Q->used.push_back(false);
    Q->released.push_back(true);
  }
  *q = Q;
  return RW_OK;
}

extern "C" rw_status rw_queue_push(rw_queue* q, const void* host_src, size_t bytes,
                                   void* copy_stream, void** dev_slot, int32_t* slot_id) {
  if (!q || !host_src || !dev_slot || bytes > q->slot_bytes)
    return qfail(RW_EINVAL, "rw_queue_push: bad arguments or bytes > slot_bytes");
  const int s = q->next;
  // pushing more than `depth` slots ahead of rw_queue_release would overwrite a slot whose
  // consumers were never enqueued: refuse instead of racing
  if (!q->released[s])
    return qfail(RW_EINVAL, "rw_queue_push: the next slot has not been released (more than "
                            "depth pushes ahead of rw_queue_release)");
  q->next = (q->next + 1) % q->depth;
  // the slot's previous H2D copy must be done (host buffer reuse) and its consumers must
  // have released it (device buffer reuse)
  if (q->used[s] && (cudaEventSynchronize(q->ready[s]) != cudaSuccess ||
                     cudaEventSynchronize(q->freed[s]) != cudaSuccess))
    return qfail(RW_ECUDA, "rw_queue_push: waiting for slot release failed");
  // a pinned (page-locked / registered) source is copied to the device directly, without
  // the staging copy; a pageable one goes through the slot's pinned buffer
  cudaPointerAttributes pa{};
  const bool pinned = cudaPointerGetAttributes(&pa, host_src) == cudaSuccess &&
                      pa.type == cudaMemoryTypeHost;
  cudaGetLastError();   // pageable pointers may report an error on some drivers
  const void* src = host_src;
  if (!pinned) {
    parallel_copy(q->host[s], host_src, bytes);
    src = q->host[s];
  }
  cudaStream_t cs = (cudaStream_t)copy_stream;
  if (cudaMemcpyAsync(q->dev[s], src, bytes, cudaMemcpyHostToDevice, cs) != cudaSuccess ||
      cudaEventRecord(q->ready[s], cs) != cudaSuccess)
    return qfail(RW_ECUDA, "rw_queue_push: H2D copy enqueue failed");
  q->used[s] = true;
  q->released[s] = false;
  *dev_slot = q->dev[s];
  if (slot_id) *slot_id = s;
  return RW_OK;
}

// Library-internal (rw_hier_segment_ooc): push a slot whose pinned buffer is filled by
// `fill` (e.g. a host-side gather of many small pieces) instead of one contiguous source.
namespace rw {
size_t queue_slot_bytes(const rw_queue* q) { return q ? q->slot_bytes : 0; }
int queue_depth(const rw_queue* q) { return q ? q->depth : 0; }
// the pinned host buffer of slot i (rw_hier_segment_ooc stages its D2H output there once
// every push has completed)
void* queue_host_slot(rw_queue* q, int i) { return q->host[i]; }
void host_parallel_copy(void* dst, const void* src, size_t bytes) { parallel_copy(dst, src, bytes); }
// true when p is page-locked host memory (cudaMallocHost / cudaHostAlloc / cudaHostRegister)
bool host_is_pinned(const void* p) {
  if (!p) return false;
  cudaPointerAttributes pa{};
  const bool pinned = cudaPointerGetAttributes(&pa, p) == cudaSuccess && pa.type == cudaMemoryTypeHost;
  cudaGetLastError();   // pageable pointers may report an error on some drivers
  return pinned;
}
// Two pinned host pieces copied straight into the next slot's device buffer, back to back
// (no staging copy through the slot's host buffer); otherwise as rw_queue_push.
rw_status queue_push_pinned2(rw_queue* q, const void* src0, size_t bytes0, const void* src1,
                             size_t bytes1, cudaStream_t copy_s, void** dev_slot, int32_t* slot_id) {
  if (!q || !dev_slot || bytes0 + bytes1 > q->slot_bytes)
    return qfail(RW_EINVAL, "rw_queue: bad pinned push (bytes > slot_bytes?)");
  const int s = q->next;
  if (!q->released[s])
    return qfail(RW_EINVAL, "rw_queue: the next slot has not been released");
  q->next = (q->next + 1) % q->depth;
  if (q->used[s] && (cudaEventSynchronize(q->ready[s]) != cudaSuccess ||
                     cudaEventSynchronize(q->freed[s]) != cudaSuccess))
    return qfail(RW_ECUDA, "rw_queue: waiting for slot release failed");
  if ((bytes0 > 0 && cudaMemcpyAsync(q->dev[s], src0, bytes0, cudaMemcpyHostToDevice, copy_s) != cudaSuccess) ||
      (bytes1 > 0 && cudaMemcpyAsync((char*)q->dev[s] + bytes0, src1, bytes1, cudaMemcpyHostToDevice,
                                     copy_s) != cudaSuccess))
    return qfail(RW_ECUDA, "rw_queue: H2D copy enqueue failed");
  if (cudaEventRecord(q->ready[s], copy_s) != cudaSuccess)
    return qfail(RW_ECUDA, "rw_queue: event record failed");
  q->used[s] = true;
  q->released[s] = false;
  *dev_slot = q->dev[s];
  if (slot_id) *slot_id = s;
  return RW_OK;
}
// The non-zero `seg`-byte segments of p[0, n), found on host threads; adjacent segments are
// merged.  Returns false (segs unspecified) when more than max_segs segments are non-zero.
bool host_nonzero_segments(const uint8_t* p, size_t n, size_t seg, size_t max_segs,
                           std::vector<std::pair<size_t, size_t>>& segs) {
  segs.clear();
  const size_t nseg = (n + seg - 1) / seg;
  unsigned nt = std::thread::hardware_concurrency();
  if (nt > 16) nt = 16;
  if (nt < 1) nt = 1;
  if (nseg < (size_t)nt * 64) nt = 1;
  std::vector<std::vector<size_t>> hit(nt);
  auto scan = [&](unsigned t) {
    const size_t a = nseg * t / nt, b = nseg * (t + 1) / nt;
    for (size_t i = a; i < b && hit[t].size() <= max_segs; ++i) {
      const uint8_t* q = p + i * seg;
      const size_t len = std::min(seg, n - i * seg);
      uint64_t acc = 0;
      size_t j = 0;
      for (; j + 64 <= len; j += 64) {
        uint64_t v[8];
        std::memcpy(v, q + j, 64);
        acc |= v[0] | v[1] | v[2] | v[3] | v[4] | v[5] | v[6] | v[7];
      }
      for (; j < len; ++j) acc |= q[j];
      if (acc) hit[t].push_back(i);
    }
  };
  if (nt == 1) scan(0);
  else {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) th.emplace_back(scan, t);
    for (auto& x : th) x.join();
  }
  size_t total = 0;
  for (auto& h : hit) total += h.size();
  if (total > max_segs) return false;
  for (auto& h : hit)
    for (size_t i : h) {
      const size_t off = i * seg, len = std::min(seg, n - off);
      if (!segs.empty() && segs.back().first + segs.back().second == off) segs.back().second += len;
      else segs.emplace_back(off, len);
    }
  return true;
}
// One slot = [piece 0 | sparse piece 1]: piece 0 (bytes0, may be 0) is copied whole (directly
// when page-locked, else staged through the slot's host buffer); piece 1 (bytes1) is zeroed on
// the device and only its listed non-zero segments are copied.  Otherwise as rw_queue_push.
rw_status queue_push_sparse(rw_queue* q, const void* src0, size_t bytes0, bool pinned0,
                            const uint8_t* src1, size_t bytes1, bool pinned1,
                            const std::vector<std::pair<size_t, size_t>>& segs,
                            cudaStream_t copy_s, void** dev_slot, int32_t* slot_id) {
  if (!q || !dev_slot || bytes0 + bytes1 > q->slot_bytes)
    return qfail(RW_EINVAL, "rw_queue: bad sparse push (bytes > slot_bytes?)");
  const int s = q->next;
  if (!q->released[s])
    return qfail(RW_EINVAL, "rw_queue: the next slot has not been released");
  q->next = (q->next + 1) % q->depth;
  if (q->used[s] && (cudaEventSynchronize(q->ready[s]) != cudaSuccess ||
                     cudaEventSynchronize(q->freed[s]) != cudaSuccess))
    return qfail(RW_ECUDA, "rw_queue: waiting for slot release failed");
  char* hs = (char*)q->host[s];
  char* ds = (char*)q->dev[s];
  bool ok = true;
  if (bytes0 > 0) {
    const void* src = src0;
    if (!pinned0) { parallel_copy(hs, src0, bytes0); src = hs; }
    ok = cudaMemcpyAsync(ds, src, bytes0, cudaMemcpyHostToDevice, copy_s) == cudaSuccess;
  }
  if (ok && bytes1 > 0) ok = cudaMemsetAsync(ds + bytes0, 0, bytes1, copy_s) == cudaSuccess;
  for (size_t i = 0; ok && i < segs.size(); ++i) {
    const size_t off = segs[i].first, len = segs[i].second;
    const void* src = src1 + off;
    if (!pinned1) { std::memcpy(hs + bytes0 + off, src1 + off, len); src = hs + bytes0 + off; }
    ok = cudaMemcpyAsync(ds + bytes0 + off, src, len, cudaMemcpyHostToDevice, copy_s) == cudaSuccess;
  }
  if (!ok) return qfail(RW_ECUDA, "rw_queue: H2D copy enqueue failed");
  if (cudaEventRecord(q->ready[s], copy_s) != cudaSuccess)
    return qfail(RW_ECUDA, "rw_queue: event record failed");
  q->used[s] = true;
  q->released[s] = false;
  *dev_slot = q->dev[s];
  if (slot_id) *slot_id = s;
  return RW_OK;
}
rw_status queue_push_fill(rw_queue* q, size_t bytes, void (*fill)(void* dst, void* ctx),
                          void* ctx, cudaStream_t copy_s, void** dev_slot, int32_t* slot_id) {
  if (!q || !fill || !dev_slot || bytes > q->slot_bytes)
    return qfail(RW_EINVAL, "rw_queue: bad fill push (bytes > slot_bytes?)");
  const int s = q->next;
  if (!q->released[s])
    return qfail(RW_EINVAL, "rw_queue: the next slot has not been released");
  q->next = (q->next + 1) % q->depth;
  if (q->used[s] && (cudaEventSynchronize(q->ready[s]) != cudaSuccess ||
                     cudaEventSynchronize(q->freed[s]) != cudaSuccess))
    return qfail(RW_ECUDA, "rw_queue: waiting for slot release failed");
  fill(q->host[s], ctx);
  if (bytes > 0 && (cudaMemcpyAsync(q->dev[s], q->host[s], bytes, cudaMemcpyHostToDevice,
                                    copy_s) != cudaSuccess))
    return qfail(RW_ECUDA, "rw_queue: H2D copy enqueue failed");
  if (cudaEventRecord(q->ready[s], copy_s) != cudaSuccess)
    return qfail(RW_ECUDA, "rw_queue: event record failed");
  q->used[s] = true;
  q->released[s] = false;
  *dev_slot = q->dev[s];
  if (slot_id) *slot_id = s;
  return RW_OK;
}
}  // namespace rw

extern "C" rw_status rw_queue_wait(rw_queue* q, int32_t slot_id, void* compute_stream) {
  if (!q || slot_id < 0 || slot_id >= q->depth) return qfail(RW_EINVAL, "rw_queue_wait: bad slot");
  if (cudaStreamWaitEvent((cudaStream_t)compute_stream, q->ready[slot_id], 0) != cudaSuccess)
    return qfail(RW_ECUDA, "rw_queue_wait: cudaStreamWaitEvent failed");
  return RW_OK;
}

extern "C" rw_status rw_queue_release(rw_queue* q, int32_t slot_id, void* compute_stream) {
  if (!q || slot_id < 0 || slot_id >= q->depth) return qfail(RW_EINVAL, "rw_queue_release: bad slot");
  if (cudaEventRecord(q->freed[slot_id], (cudaStream_t)compute_stream) != cudaSuccess)
    return qfail(RW_ECUDA, "rw_queue_release: cudaEventRecord failed");
  q->released[slot_id] = true;
  return RW_OK;
}

extern "C" void rw_queue_destroy(rw_queue* q) {
  if (!q) return;
  for (size_t i = 0; i < q->host.size(); ++i) {
    cudaEventSynchronize(q->freed[i]);
    cudaFreeHost(q->host[i]);
    cudaFree(q->dev[i]);
    cudaEventDestroy(q->ready[i]);
    cudaEventDestroy(q->freed[i]);
  }
  delete q;
}
