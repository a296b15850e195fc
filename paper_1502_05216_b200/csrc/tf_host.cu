// tf_host.cu -- host-buffer entry point of libtwofold_b200.so (tf_eval_host).
//
// The reference evaluates host (numpy) arrays (explog.py:333-349 api(width)
// methods); this entry point takes HOST arrays and streams them through a
// three-stage chunk pipeline on the device:
//
//   copy-in streams  H2D of chunk k into ring slot k % RING (x0 and x1 on two
//                    streams: 95 vs 93 GB/s both directions, tools/pcie_streams_probe.py)
//   compute stream   tf_eval of chunk k           (waits for both H2D)
//   copy-out streams D2H of chunk k's results z0 / z1 (wait for its kernel)
//
// A slot is refilled only after its previous copy-out completed.  The copy
// engines therefore run both PCIe directions at once (measured 55 GB/s H2D,
// 57 GB/s D2H, 99 GB/s together on the B200 box, tools/pcie_probe.py), while the
// kernel time per chunk is ~2% of the copy time.
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstring>
#include <mutex>

#include "tf_abi.h"

using tfabi::cuda_check;
using tfabi::fail;

namespace {

constexpr int RING = 4;
constexpr int MAX_DEV = 64;
// elements per chunk: 8 MiB per binary64 array.  tools/pcie_pattern_probe.py
// (one call = 2 x 2^24 binary64 in, 2 x 2^24 out, host-synchronised): 2^19
// pays a per-copy overhead (6.7 ms for copies alone), 2^22 a longer pipeline fill and drain; 2^20 and
// 2^21 both give 6.4 ms against 5.4 ms for the same bytes as two independent
// bulk copies.  A geometric ramp of chunk sizes at both ends did not help: the
// D2H stream trails by one chunk whatever the sizes (both directions run at
// ~49.5 GB/s together), so the tail is set by the largest chunk.
constexpr int64_t DEFAULT_CHUNK = 1 << 20;

struct HostPipe {
  bool ready = false;
  int64_t cap_bytes = 0;  // bytes per ring buffer
  // two copy streams per direction: x0 / z0 on in / out, x1 / z1 on in2 / out2
  cudaStream_t in = nullptr, in2 = nullptr, comp = nullptr, out = nullptr, out2 = nullptr;
  cudaEvent_t loaded[RING], loaded2[RING], done[RING], freed[RING], freed2[RING], entry;
  bool used[RING] = {};
  void* buf[RING][4] = {};
};

// A small pool of pipelines per device: concurrent calls from different host
// threads (e.g. two independent functions of one step) each take a free
// pipeline, so one call's fill and drain overlap the other's copies.
constexpr int POOL = 2;
HostPipe g_pipe[MAX_DEV][POOL];
std::mutex g_pipe_mu[MAX_DEV][POOL];

bool dotted_fn(int fn) {
  return fn == TF_FN_PEXP0 || fn == TF_FN_TEXP0 || fn == TF_FN_PEXPM10 || fn == TF_FN_TEXPM10 ||
         fn == TF_FN_PLOG0 || fn == TF_FN_TLOG0 || fn == TF_FN_PLOG1P0 || fn == TF_FN_TLOG1P0;
}

int setup(HostPipe& p, int64_t bytes) {
  if (!p.ready) {
    if (cudaStreamCreateWithFlags(&p.in, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&p.in2, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&p.out2, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&p.comp, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&p.out, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&p.entry, cudaEventDisableTiming) != cudaSuccess)
      return cuda_check("tf_eval_host: stream/event creation");
    for (int s = 0; s < RING; ++s)
      if (cudaEventCreateWithFlags(&p.loaded[s], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&p.loaded2[s], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&p.freed2[s], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&p.done[s], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&p.freed[s], cudaEventDisableTiming) != cudaSuccess)
        return cuda_check("tf_eval_host: event creation");
    p.ready = true;
  }
  if (bytes > p.cap_bytes) {
    // the previous call returned only after its copy-out stream drained, so
    // no ring buffer is in flight here
    for (int s = 0; s < RING; ++s)
      for (int a = 0; a < 4; ++a) {
        if (p.buf[s][a]) cudaFree(p.buf[s][a]);
        p.buf[s][a] = nullptr;
      }
    p.cap_bytes = 0;
    for (int s = 0; s < RING; ++s)
      for (int a = 0; a < 4; ++a)
        if (cudaMalloc(&p.buf[s][a], (size_t)bytes) != cudaSuccess)
          return cuda_check("tf_eval_host: ring buffer allocation");
    p.cap_bytes = bytes;
  }
  return TF_OK;
}

// Small calls (the reference's own scalar convention, audit.py:343-349: one
// element per call) skip the chunk pipeline: the operands go into a mapped
// pinned buffer the kernel reads and writes directly over PCIe (zero-copy).
// Up to 32 elements take the tiny kernel: operands by value with the launch,
// results into the mapped buffer, then a sequence number into a mapped flag.
// The caller spins on that flag instead of synchronising the stream (a kernel
// that never stores it -- a launch or device fault -- is caught by the bounded
// spin, then by the stream status).  Consecutive calls may use different
// streams: a kernel's last access to the buffer is its flag store, which the
// previous call waited for.
constexpr int64_t SMALL_N = 1024;
constexpr int64_t TINY_N = 32;
struct SmallBuf {
  bool ready = false;
  void* host = nullptr;  // 4 x SMALL_N doubles + the completion flag, cudaHostAllocMapped
  void* dev = nullptr;   // its device alias
  cudaStream_t own = nullptr;  // used when the caller passes no stream
  unsigned seq = 0;
  std::mutex mu;
};
SmallBuf g_small[MAX_DEV];

int eval_small(int dev, int fn, int width, const void* x0, const void* x1, void* z0, void* z1,
               int64_t n, bool dotted, void* stream, int flags) {
  SmallBuf& b = g_small[dev];
  std::lock_guard<std::mutex> lk(b.mu);
  const size_t slot = SMALL_N * sizeof(double);
  if (!b.ready) {
    if (cudaHostAlloc(&b.host, 4 * slot + 64, cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(&b.dev, b.host, 0) != cudaSuccess ||
        cudaStreamCreateWithFlags(&b.own, cudaStreamNonBlocking) != cudaSuccess)
      return cuda_check("tf_eval_host: mapped staging buffer");
    *static_cast<volatile unsigned*>(static_cast<void*>(static_cast<char*>(b.host) + 4 * slot)) = 0;
    b.ready = true;
  }
  // no caller stream: a library stream that does not serialise with the
  // device's other work (the operands are host values, nothing to wait for)
  if (!stream) stream = b.own;
  const size_t sz = width / 8, bytes = (size_t)n * sz;
  char* h = static_cast<char*>(b.host);
  char* d = static_cast<char*>(b.dev);
  if (n <= TINY_N && flags == 0) {
    volatile unsigned* flag = reinterpret_cast<volatile unsigned*>(h + 4 * slot);
    const unsigned seq = ++b.seq ? b.seq : ++b.seq;   // never 0 (the initial value)
    int rc = tfabi::tiny_eval(fn, width, x0, dotted ? x0 : x1, d + 2 * slot, d + 3 * slot, n,
                              stream, reinterpret_cast<unsigned*>(d + 4 * slot), seq);
    if (rc) return rc;
    const auto t0 = std::chrono::steady_clock::now();
    for (unsigned k = 0; *flag != seq; ++k) {
      if ((k & 1023) == 1023 &&
          std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(50)) {
        // slow (a busy device) or failed: the stream decides
        if (cudaStreamSynchronize(static_cast<cudaStream_t>(stream)) != cudaSuccess)
          return cuda_check("tf_eval_host: small-call synchronisation");
        if (*flag != seq) return fail(TF_ERR_CUDA, "tf_eval_host: tiny kernel did not complete%s");
        break;
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
  } else {
    memcpy(h, x0, bytes);
    if (!dotted) memcpy(h + slot, x1, bytes);
    int rc = tf_eval(fn, width, d, dotted ? d : d + slot, d + 2 * slot, d + 3 * slot, n, stream,
                     flags);
    if (rc) return rc;
    if (cudaStreamSynchronize(static_cast<cudaStream_t>(stream)) != cudaSuccess)
      return cuda_check("tf_eval_host: small-call synchronisation");
  }
  memcpy(z0, h + 2 * slot, bytes);
  memcpy(z1, h + 3 * slot, bytes);
  return TF_OK;
}

}  // namespace

extern "C" TF_API int tf_eval_host(int fn, int width, const void* x0, const void* x1, void* z0,
                                   void* z1, int64_t n, int64_t chunk, void* stream, int flags) {
  if (n < 0) return fail(TF_ERR_ARG, "negative element count%s");
  if (width != 32 && width != 64) return fail(TF_ERR_ARG, "unsupported width (expected 32 or 64)%s");
  if (fn < 0 || fn >= TF_FN_COUNT) return fail(TF_ERR_ARG, "unknown function code%s");
  if (chunk < 0) return fail(TF_ERR_ARG, "negative chunk%s");
  if (n == 0) return TF_OK;
  const bool dotted = dotted_fn(fn);
  if (!x0 || (!x1 && !dotted) || !z0 || !z1) return fail(TF_ERR_ARG, "null pointer%s");
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cuda_check("tf_eval_host: cudaGetDevice");
  if (dev < 0 || dev >= MAX_DEV) return fail(TF_ERR_ARG, "device index out of range%s");
  if (n <= SMALL_N && chunk == 0)
    return eval_small(dev, fn, width, x0, x1, z0, z1, n, dotted && (!x1 || x1 == x0), stream, flags);
  const int64_t sz = width / 8;
  const int64_t c = chunk > 0 ? (chunk < n ? chunk : n) : (DEFAULT_CHUNK < n ? DEFAULT_CHUNK : n);
  const bool copy_x1 = !dotted || (x1 && x1 != x0);

  std::unique_lock<std::mutex> lk;
  int slot = -1;
  for (int i = 0; i < POOL && slot < 0; ++i) {
    std::unique_lock<std::mutex> t(g_pipe_mu[dev][i], std::try_to_lock);
    if (t.owns_lock()) {
      lk = std::move(t);
      slot = i;
    }
  }
  if (slot < 0) {                                 // all busy: queue on the first
    slot = 0;
    lk = std::unique_lock<std::mutex>(g_pipe_mu[dev][0]);
  }
  HostPipe& p = g_pipe[dev][slot];
  int rc = setup(p, c * sz);
  if (rc) return rc;
  // On an error after the first enqueue, copies that touch the caller's host
  // buffers may still be in flight: drain all three streams before returning
  // (their own status is ignored; the first error is what gets reported), and
  // forget the ring state so the next call starts clean.
  struct Drain {
    HostPipe& p;
    bool armed = true;
    ~Drain() {
      if (!armed) return;
      cudaStreamSynchronize(p.in);
      cudaStreamSynchronize(p.in2);
      cudaStreamSynchronize(p.out2);
      cudaStreamSynchronize(p.comp);
      cudaStreamSynchronize(p.out);
      for (int s = 0; s < RING; ++s) p.used[s] = false;
    }
  } drain{p};
  // start after the work already queued on the caller's stream
  if (cudaEventRecord(p.entry, static_cast<cudaStream_t>(stream)) != cudaSuccess ||
      cudaStreamWaitEvent(p.in, p.entry, 0) != cudaSuccess ||
      cudaStreamWaitEvent(p.in2, p.entry, 0) != cudaSuccess)
    return cuda_check("tf_eval_host: stream ordering");
  const char* hx0 = static_cast<const char*>(x0);
  const char* hx1 = static_cast<const char*>(x1);
  char* hz0 = static_cast<char*>(z0);
  char* hz1 = static_cast<char*>(z1);
  int64_t k = 0;
  for (int64_t off = 0; off < n; off += c, ++k) {
    const int64_t m = c < n - off ? c : n - off;
    const size_t bytes = (size_t)(m * sz), at = (size_t)(off * sz);
    const int s = (int)(k % RING);
    void *d0 = p.buf[s][0], *d1 = copy_x1 ? p.buf[s][1] : p.buf[s][0];
    void *e0 = p.buf[s][2], *e1 = p.buf[s][3];
    // a slot is refilled after BOTH of its copy-outs (z0 and z1) are done
    if (p.used[s] && (cudaStreamWaitEvent(p.in, p.freed[s], 0) != cudaSuccess ||
                      cudaStreamWaitEvent(p.in, p.freed2[s], 0) != cudaSuccess ||
                      cudaStreamWaitEvent(p.in2, p.freed[s], 0) != cudaSuccess ||
                      cudaStreamWaitEvent(p.in2, p.freed2[s], 0) != cudaSuccess))
      return cuda_check("tf_eval_host: ring wait");
    if (cudaMemcpyAsync(d0, hx0 + at, bytes, cudaMemcpyHostToDevice, p.in) != cudaSuccess ||
        cudaEventRecord(p.loaded[s], p.in) != cudaSuccess ||
        cudaStreamWaitEvent(p.comp, p.loaded[s], 0) != cudaSuccess ||
        (copy_x1 && (cudaMemcpyAsync(d1, hx1 + at, bytes, cudaMemcpyHostToDevice, p.in2) != cudaSuccess ||
                     cudaEventRecord(p.loaded2[s], p.in2) != cudaSuccess ||
                     cudaStreamWaitEvent(p.comp, p.loaded2[s], 0) != cudaSuccess)))
      return cuda_check("tf_eval_host: copy-in");
    rc = tf_eval(fn, width, d0, d1, e0, e1, m, p.comp, flags);
    if (rc) return rc;
    if (cudaEventRecord(p.done[s], p.comp) != cudaSuccess ||
        cudaStreamWaitEvent(p.out, p.done[s], 0) != cudaSuccess ||
        cudaStreamWaitEvent(p.out2, p.done[s], 0) != cudaSuccess ||
        cudaMemcpyAsync(hz0 + at, e0, bytes, cudaMemcpyDeviceToHost, p.out) != cudaSuccess ||
        cudaMemcpyAsync(hz1 + at, e1, bytes, cudaMemcpyDeviceToHost, p.out2) != cudaSuccess ||
        cudaEventRecord(p.freed[s], p.out) != cudaSuccess ||
        cudaEventRecord(p.freed2[s], p.out2) != cudaSuccess)
      return cuda_check("tf_eval_host: copy-out");
    p.used[s] = true;
  }
  // the results are on the host when the call returns
  if (cudaStreamSynchronize(p.out) != cudaSuccess || cudaStreamSynchronize(p.out2) != cudaSuccess)
    return cuda_check("tf_eval_host: drain");
  drain.armed = false;
  return TF_OK;
}
