// Error plumbing and small C-ABI utilities.
#include <stdarg.h>
#include <stdio.h>

#include <mutex>
#include <vector>

#include "common.cuh"

namespace {
thread_local char g_err[1024] = "";
}

namespace dicm {

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_cuda(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return DICM_OK;
  return fail(DICM_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

int last_launch(const char* where) { return check_cuda(cudaGetLastError(), where); }

// Library-owned side streams: one per (host thread, device, purpose), created
// outside any capture (relaxed capture mode), with a fork and a join event.
// DICM_FORK=0 turns every fork off (the work stays on the caller's stream).
Fork* side_fork(int purpose) {
  static const bool off = [] {
    const char* e = getenv("DICM_FORK");
    return e && e[0] == '0';
  }();
  if (off || purpose < 0 || purpose >= kForkPurposes) return nullptr;
  constexpr int kMaxDev = 64;
  thread_local Fork forks[kMaxDev][kForkPurposes];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
  Fork& f = forks[dev][purpose];
  if (!f.side) {
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&mode);
    const bool ok = cudaStreamCreateWithFlags(&f.side, cudaStreamNonBlocking) == cudaSuccess &&
                    cudaEventCreateWithFlags(&f.fork, cudaEventDisableTiming) == cudaSuccess &&
                    cudaEventCreateWithFlags(&f.join, cudaEventDisableTiming) == cudaSuccess;
    cudaThreadExchangeStreamCaptureMode(&mode);
    if (!ok) {
      cudaGetLastError();
      f.side = nullptr;
      return nullptr;
    }
  }
  return &f;
}

cudaStream_t fork_begin(Fork* f, cudaStream_t main) {
  if (!f) return main;
  cudaEventRecord(f->fork, main);
  cudaStreamWaitEvent(f->side, f->fork, 0);
  return f->side;
}

void fork_end(Fork* f, cudaStream_t main) {
  if (!f) return;
  cudaEventRecord(f->join, f->side);
  cudaStreamWaitEvent(main, f->join, 0);
}

// Kernel timing probe: CUDA events recorded on the launching stream around
// the dominant kernels, read back by bench.py for the roofline.
namespace {
struct ProbeRec {
  int kernel;
  cudaEvent_t a, b;
};
std::mutex g_probe_mu;
bool g_probe_on = false;
std::vector<ProbeRec> g_probe;
std::vector<cudaEvent_t> g_probe_free;

cudaEvent_t probe_event() {
  if (!g_probe_free.empty()) {
    cudaEvent_t e = g_probe_free.back();
    g_probe_free.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

void probe_recycle() {
  for (auto& r : g_probe) {
    g_probe_free.push_back(r.a);
    g_probe_free.push_back(r.b);
  }
  g_probe.clear();
}
}  // namespace

int probe_begin(int kernel, cudaStream_t st) {
  if (!g_probe_on) return -1;
  std::lock_guard<std::mutex> lk(g_probe_mu);
  ProbeRec r{kernel, probe_event(), probe_event()};
  cudaEventRecord(r.a, st);
  g_probe.push_back(r);
  return (int)g_probe.size() - 1;
}

void probe_end(int slot, cudaStream_t st) {
  if (slot < 0) return;
  std::lock_guard<std::mutex> lk(g_probe_mu);
  if (slot < (int)g_probe.size()) cudaEventRecord(g_probe[slot].b, st);
}

}  // namespace dicm

extern "C" {

const char* dicm_last_error(void) { return g_err; }

int dicm_version(void) { return 1; }

int dicm_device_arch(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return -1;
  return p.major * 10 + p.minor;
}

int dicm_probe_enable(int on) {
  std::lock_guard<std::mutex> lk(dicm::g_probe_mu);
  dicm::probe_recycle();
  dicm::g_probe_on = on != 0;
  return DICM_OK;
}

int dicm_probe_read(int kernel, float* ms, int max, int* n) {
  std::lock_guard<std::mutex> lk(dicm::g_probe_mu);
  int k = 0;
  for (auto& r : dicm::g_probe) {
    if (r.kernel != kernel) continue;
    if (k < max) {
      int rc = dicm::check_cuda(cudaEventSynchronize(r.b), "dicm_probe_read");
      if (rc) return rc;
      rc = dicm::check_cuda(cudaEventElapsedTime(&ms[k], r.a, r.b), "dicm_probe_read");
      if (rc) return rc;
    }
    ++k;
  }
  *n = k < max ? k : max;
  return DICM_OK;
}

int dicm_zero_async(void* ptr, size_t bytes, dicm_stream_t stream) {
  if (!bytes) return DICM_OK;
  return dicm::check_cuda(cudaMemsetAsync(ptr, 0, bytes, (cudaStream_t)stream), "dicm_zero_async");
}

}  // extern "C"
