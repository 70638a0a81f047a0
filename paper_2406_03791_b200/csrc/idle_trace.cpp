// idle_trace.cpp — GPU idle fraction of a decode from CUPTI kernel activity
// records (the real-hardware counterpart of the reference's simulated
// TimingReport.idle_fraction = 1 - device_busy / span, engine.cpp:329-366,
// analysis.cpp:25-28).  Kernel nodes launched by CUDA graphs (including the
// bodies of conditional WHILE nodes) are reported individually.
#include <cuda_runtime.h>
#include <cupti.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <utility>
#include <vector>

#include "../../include/rnntg.h"

namespace {

std::mutex g_mu;
std::vector<std::pair<uint64_t, uint64_t>> g_iv;
bool g_on = false;

void CUPTIAPI buffer_requested(uint8_t** buf, size_t* size, size_t* max_records) {
  *size = 16u << 20;
  *buf = static_cast<uint8_t*>(std::aligned_alloc(64, *size));
  *max_records = 0;
}

void CUPTIAPI buffer_completed(CUcontext, uint32_t, uint8_t* buf, size_t, size_t valid) {
  CUpti_Activity* rec = nullptr;
  std::lock_guard<std::mutex> lk(g_mu);
  while (cuptiActivityGetNextRecord(buf, valid, &rec) == CUPTI_SUCCESS) {
    if (rec->kind == CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL || rec->kind == CUPTI_ACTIVITY_KIND_KERNEL) {
      const auto* k = reinterpret_cast<const CUpti_ActivityKernel9*>(rec);
      g_iv.emplace_back(k->start, k->end);
    }
  }
  std::free(buf);
}

}  // namespace

extern "C" {

rnntg_status rnntg_trace_begin(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_iv.clear();
  if (!g_on) {
    if (cuptiActivityRegisterCallbacks(buffer_requested, buffer_completed) != CUPTI_SUCCESS)
      return RNNTG_E_CUDA;
    g_on = true;
  }
  if (cuptiActivityEnable(CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL) != CUPTI_SUCCESS) return RNNTG_E_CUDA;
  return RNNTG_OK;
}

rnntg_status rnntg_trace_end(double* busy_ms, double* span_ms, int64_t* kernels) {
  cudaDeviceSynchronize();
  cuptiActivityFlushAll(1);
  cuptiActivityDisable(CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL);
  std::vector<std::pair<uint64_t, uint64_t>> iv;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    iv.swap(g_iv);
  }
  if (kernels) *kernels = (int64_t)iv.size();
  if (iv.empty()) {
    if (busy_ms) *busy_ms = 0.0;
    if (span_ms) *span_ms = 0.0;
    return RNNTG_OK;
  }
  std::sort(iv.begin(), iv.end());
  uint64_t busy = 0, cs = iv[0].first, ce = iv[0].second, hi = iv[0].second;
  for (size_t i = 1; i < iv.size(); ++i) {
    hi = std::max(hi, iv[i].second);
    if (iv[i].first > ce) {
      busy += ce - cs;
      cs = iv[i].first;
      ce = iv[i].second;
    } else {
      ce = std::max(ce, iv[i].second);
    }
  }
  busy += ce - cs;
  if (busy_ms) *busy_ms = busy * 1e-6;
  if (span_ms) *span_ms = (hi - iv[0].first) * 1e-6;
  return RNNTG_OK;
}

}  // extern "C"
