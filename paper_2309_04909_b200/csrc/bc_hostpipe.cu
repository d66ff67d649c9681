// bc_hostpipe.cu -- host-buffer entry points (bc_drelu_host, bc_relu_host):
// shares in host memory, H2D copy / fused kernel / D2H copy pipelined in
// chunks over a small ring of CUDA streams, so that both PCIe directions and
// the kernels overlap.  This is the end-to-end path of a caller whose shares
// live on the host (bench.py "e2e").
//
// Chunk c runs on stream c % NS, all of its steps in order; chunk c + NS on the
// same stream therefore starts only after chunk c's D2H finished, which is
// what makes a workspace of NS chunk slots sufficient.  Device memory is the
// caller's workspace; the streams and events are created once per device and
// cached (the only library-owned CUDA objects).
#include <atomic>
#include <mutex>

#include "bc_common.cuh"

using namespace bc;
using namespace bc::host;

namespace {

#ifndef BC_HOST_NS
#define BC_HOST_NS 3
#endif
constexpr int NS = BC_HOST_NS;  // streams (and workspace chunk slots) in the ring
constexpr int MAX_DEV = 64;

struct Ring {
  bool init = false;
  cudaStream_t s[NS];
  cudaEvent_t ev[NS];
  cudaEvent_t start;
  std::mutex start_mu;  // one caller at a time between recording `start` and the ring's waits on it
  std::atomic<uint64_t> next{0};  // chunk rotation continues across calls (async calls pipeline evenly)
};

std::mutex g_ring_mu;
Ring g_ring[MAX_DEV];

int ring_for(int dev, Ring** out) {
  if (dev < 0 || dev >= MAX_DEV) return BC_EINVAL;
  std::lock_guard<std::mutex> lk(g_ring_mu);
  Ring& r = g_ring[dev];
  if (!r.init) {
    for (int i = 0; i < NS; ++i) {
      if (cudaStreamCreateWithFlags(&r.s[i], cudaStreamNonBlocking) != cudaSuccess) return check_launch();
      if (cudaEventCreateWithFlags(&r.ev[i], cudaEventDisableTiming) != cudaSuccess) return check_launch();
    }
    if (cudaEventCreateWithFlags(&r.start, cudaEventDisableTiming) != cudaSuccess) return check_launch();
    r.init = true;
  }
  *out = &r;
  return BC_OK;
}

size_t slot_bytes(size_t chunk) { return 4 * chunk * sizeof(uint64_t); }

// SYNC: order after the caller's stream and return with the host outputs
// complete.  Otherwise (the _async entries) only enqueue: consecutive calls
// share the ring streams, so call k+1's copies overlap call k's tail (chunk c
// always runs on stream c % NS, and stream order keeps each workspace slot's
// uses apart); the caller's stream is made to wait for every chunk.
template <bool RELU, bool SYNC>
int host_run(const uint64_t* x0, const uint64_t* x1, uint64_t* y0, uint64_t* y1, size_t n, uint64_t base,
             const bc_params* prm, const bc_seeds* seeds, void* ws, size_t ws_bytes, size_t chunk, void* stream) {
  const int rc = check_params(prm);
  if (rc) return rc;
  if (n == 0) return BC_OK;
  if (!x0 || !x1 || !y0 || !y1 || !seeds || !ws || chunk == 0 || (chunk & 7)) return BC_EINVAL;
  if (!aligned16(ws) || (base & 7)) return BC_EALIGN;
  if (!index_range_ok(base, n)) return BC_ERANGE;  // global indices j < BC_MAX_INDEX
  if (ws_bytes < NS * slot_bytes(chunk)) return BC_EINVAL;
  const size_t nb = n * 8;
  if (overlap(y0, nb, x0, nb) || overlap(y0, nb, x1, nb) || overlap(y1, nb, x0, nb) || overlap(y1, nb, x1, nb) ||
      overlap(y0, nb, y1, nb))
    return BC_EALIAS;
  int dev = 0;
  cudaGetDevice(&dev);
  Ring* ring = nullptr;
  const int rr = ring_for(dev, &ring);
  if (rr) return rr;
  cudaStream_t caller = static_cast<cudaStream_t>(stream);
  if (SYNC) {  // order after the caller's prior work on `stream`
    // held across record and waits: a concurrent caller's record in between would make this
    // call's chunks wait on THAT caller's stream instead of its own (cudaStreamWaitEvent takes
    // the event's most recent record at the time of the call)
    std::lock_guard<std::mutex> lk(ring->start_mu);
    cudaEventRecord(ring->start, caller);
    for (int i = 0; i < NS; ++i) cudaStreamWaitEvent(ring->s[i], ring->start, 0);
  }
  uint8_t* wsb = static_cast<uint8_t*>(ws);
  // chunk -> stream (and workspace slot) by a rotation that continues across calls, so
  // back-to-back async calls spread evenly over the ring; stream order keeps each slot's uses apart
  const uint64_t nchunks = (n + chunk - 1) / chunk;
  const uint64_t c0 = ring->next.fetch_add(nchunks);
  size_t c = 0;
  for (size_t a = 0; a < n; a += chunk, ++c) {
    const size_t m = (n - a < chunk) ? n - a : chunk;
    const int k = (int)((c0 + c) % NS);
    cudaStream_t s = ring->s[k];
    uint64_t* bx0 = reinterpret_cast<uint64_t*>(wsb + k * slot_bytes(chunk));
    uint64_t* bx1 = bx0 + chunk;
    uint64_t* by0 = bx1 + chunk;
    uint64_t* by1 = by0 + chunk;
    cudaMemcpyAsync(bx0, x0 + a, m * 8, cudaMemcpyDefault, s);
    cudaMemcpyAsync(bx1, x1 + a, m * 8, cudaMemcpyDefault, s);
    const int kr = RELU ? bc_relu(bx0, bx1, by0, by1, m, base + a, prm, seeds, nullptr, s)
                        : bc_drelu(bx0, bx1, by0, by1, m, base + a, prm, seeds, nullptr, s);
    if (kr) return kr;
    cudaMemcpyAsync(y0 + a, by0, m * 8, cudaMemcpyDefault, s);
    cudaMemcpyAsync(y1 + a, by1, m * 8, cudaMemcpyDefault, s);
  }
  // the caller's stream resumes after every chunk; the host outputs are complete on return
  for (int i = 0; i < NS; ++i) {
    cudaEventRecord(ring->ev[i], ring->s[i]);
    cudaStreamWaitEvent(caller, ring->ev[i], 0);
  }
  if (SYNC)
    for (int i = 0; i < NS; ++i)
      if (cudaStreamSynchronize(ring->s[i]) != cudaSuccess) return check_launch();
  return check_launch();
}

}  // namespace

extern "C" {

size_t bc_host_workspace_bytes(size_t chunk) { return NS * slot_bytes((chunk + 7) & ~(size_t)7); }

int bc_drelu_host(const uint64_t* x0, const uint64_t* x1, uint64_t* y0, uint64_t* y1, size_t n, uint64_t elem_base,
                  const bc_params* prm, const bc_seeds* seeds, void* ws, size_t ws_bytes, size_t chunk,
                  void* stream) {
  return host_run<false, true>(x0, x1, y0, y1, n, elem_base, prm, seeds, ws, ws_bytes, chunk, stream);
}

int bc_drelu_host_async(const uint64_t* x0, const uint64_t* x1, uint64_t* y0, uint64_t* y1, size_t n,
                        uint64_t elem_base, const bc_params* prm, const bc_seeds* seeds, void* ws, size_t ws_bytes,
                        size_t chunk, void* stream) {
  return host_run<false, false>(x0, x1, y0, y1, n, elem_base, prm, seeds, ws, ws_bytes, chunk, stream);
}

int bc_relu_host(const uint64_t* x0, const uint64_t* x1, uint64_t* y0, uint64_t* y1, size_t n, uint64_t elem_base,
                 const bc_params* prm, const bc_seeds* seeds, void* ws, size_t ws_bytes, size_t chunk,
                 void* stream) {
  return host_run<true, true>(x0, x1, y0, y1, n, elem_base, prm, seeds, ws, ws_bytes, chunk, stream);
}

int bc_relu_host_async(const uint64_t* x0, const uint64_t* x1, uint64_t* y0, uint64_t* y1, size_t n,
                       uint64_t elem_base, const bc_params* prm, const bc_seeds* seeds, void* ws, size_t ws_bytes,
                       size_t chunk, void* stream) {
  return host_run<true, false>(x0, x1, y0, y1, n, elem_base, prm, seeds, ws, ws_bytes, chunk, stream);
}

}  // extern "C"
