// mf_setup.cu -- per-device, thread-safe kernel launch setup.
//
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies to the CURRENT device only, and
// the SM count / resident-CTA figures are properties of a device.  Launchers therefore look
// them up here, keyed by (device, kernel), under one mutex: a process that drives several
// GPUs (one context per device, or a multi-device context) sets every opt-in on every
// device it launches on, and concurrent first calls from several host threads never see a
// half-initialised entry.
#include <map>
#include <mutex>
#include <tuple>

#include <nvtx3/nvToolsExt.h>

#include "mf_launch.h"

namespace mf {

namespace {
struct Entry {
  size_t smem_set = 0;   // largest dynamic-smem opt-in applied on this device
  int sms = 0;
  std::map<std::pair<int, size_t>, int> resident;  // (threads, smem) -> CTAs per SM
};
std::mutex g_mu;
std::map<std::pair<int, const void*>, Entry> g_entries;
}  // namespace

cudaError_t kernel_setup(const void* func, size_t smem, int threads, LaunchInfo* out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(g_mu);
  Entry& en = g_entries[{dev, func}];
  if (!en.sms) {
    e = cudaDeviceGetAttribute(&en.sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
  }
  if (smem > en.smem_set) {
    if (smem > 48 * 1024) {
      e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    en.smem_set = smem;
  }
  int res = 0;
  if (threads > 0) {
    auto it = en.resident.find({threads, smem});
    if (it == en.resident.end()) {
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res, func, threads, smem);
      if (e != cudaSuccess) return e;
      if (res < 1) res = 1;
      en.resident[{threads, smem}] = res;
    } else {
      res = it->second;
    }
  }
  if (out) *out = LaunchInfo{en.sms, res};
  return cudaSuccess;
}

namespace {
thread_local PhaseTrace* t_trace = nullptr;
}

void phase_begin(PhaseTrace* t) {
  t_trace = t;
  if (!t) return;
  t->n = 0;
  t->open = true;
}

void phase_mark(cudaStream_t s, const char* name) {
  nvtxMarkA(name);
  PhaseTrace* t = t_trace;
  if (!t || !t->open || t->n >= PhaseTrace::kMax) return;
  if (!t->ev[t->n] && cudaEventCreate(&t->ev[t->n]) != cudaSuccess) return;
  if (cudaEventRecord(t->ev[t->n], s) != cudaSuccess) return;
  t->name[t->n++] = name;
}

void phase_end(cudaStream_t s) {
  PhaseTrace* t = t_trace;
  t_trace = nullptr;
  if (!t || !t->open) return;
  t->open = false;
  if (!t->ev[t->n] && cudaEventCreate(&t->ev[t->n]) != cudaSuccess) { t->n = 0; return; }
  if (cudaEventRecord(t->ev[t->n], s) != cudaSuccess) t->n = 0;
}

}  // namespace mf
