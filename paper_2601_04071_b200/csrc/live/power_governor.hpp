// Power governor shared by the live runtimes (live.cpp, session.cpp).
#pragma once

#include <cuda_runtime_api.h>
#include <dlfcn.h>
#include <nvml.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>

#include "microslice/json.hpp"

namespace microslice {

// Power governor (B200-specific; no reference counterpart).  A full-GPU tcgen05 GEMM
// drives a B200 into its 1 kW cap (sw_power_cap, SM clock ~1.5 GHz instead of 1.965); the
// clock recovers only on a ~10 ms scale, so HP work issued right after an LP burst runs
// 10-25% slower and misses its SLO.  This thread samples the SM clock through NVML every
// 5 ms and moves the LP SM budget: -6 SMs whenever the clock sits more than `slack` MHz
// below max (default 40), +3 after 50 ms within it.  LP launches read the budget (LiveRun::lp_sms).  NVML is loaded with dlopen
// (driver library), so hosts without it simply run ungoverned.
class PowerGovernor {
 public:
  PowerGovernor(int ordinal, int n_sm, int min_sms, int start, unsigned slack_mhz)
      : n_sm_(n_sm), min_sms_(min_sms), slack_(slack_mhz), target_(start) {
    lib_ = dlopen("libnvidia-ml.so.1", RTLD_NOW | RTLD_LOCAL);
    if (!lib_) return;
    auto sym = [&](const char* n) { return dlsym(lib_, n); };
    init_ = reinterpret_cast<nvmlReturn_t (*)()>(sym("nvmlInit_v2"));
    shutdown_ = reinterpret_cast<nvmlReturn_t (*)()>(sym("nvmlShutdown"));
    by_pci_ = reinterpret_cast<nvmlReturn_t (*)(const char*, nvmlDevice_t*)>(sym("nvmlDeviceGetHandleByPciBusId_v2"));
    clock_ = reinterpret_cast<nvmlReturn_t (*)(nvmlDevice_t, nvmlClockType_t, unsigned int*)>(sym("nvmlDeviceGetClockInfo"));
    max_clock_ = reinterpret_cast<nvmlReturn_t (*)(nvmlDevice_t, nvmlClockType_t, unsigned int*)>(sym("nvmlDeviceGetMaxClockInfo"));
    char bus[64] = {0};
    if (!init_ || !by_pci_ || !clock_ || !max_clock_ || init_() != NVML_SUCCESS) return;
    if (cudaDeviceGetPCIBusId(bus, sizeof(bus), ordinal) != cudaSuccess || by_pci_(bus, &dev_) != NVML_SUCCESS ||
        max_clock_(dev_, NVML_CLOCK_SM, &max_mhz_) != NVML_SUCCESS)
      return;
    ok_ = true;
    th_ = std::thread([this] { loop(); });
  }
  ~PowerGovernor() {
    stop_.store(true);
    if (th_.joinable()) th_.join();
    if (ok_ && shutdown_) shutdown_();
    if (lib_) dlclose(lib_);
  }
  bool ok() const { return ok_; }
  int target() const { return target_.load(std::memory_order_relaxed); }
  json summary() const {
    json j = json::object();
    j["enabled"] = json(ok_);
    j["samples"] = json(static_cast<long long>(samples_));
    j["max_mhz"] = json(static_cast<long long>(max_mhz_));
    j["mean_lp_sms"] = json(samples_ ? sum_target_ / static_cast<double>(samples_) : 0.0);
    j["mean_sm_mhz"] = json(samples_ ? sum_mhz_ / static_cast<double>(samples_) : 0.0);
    j["at_max_fraction"] = json(samples_ ? static_cast<double>(at_max_) / static_cast<double>(samples_) : 0.0);
    return j;
  }

 private:
  void loop() {
    int hold = 0;
    while (!stop_.load(std::memory_order_relaxed)) {
      unsigned int mhz = 0;
      if (clock_(dev_, NVML_CLOCK_SM, &mhz) == NVML_SUCCESS) {
        int t = target();
        if (mhz + slack_ < max_mhz_) {
          t = std::max(min_sms_, t - 6);
          hold = 0;
        } else if (++hold >= 10) {
          t = std::min(n_sm_ - 1, t + 3);
          hold = 0;
        }
        target_.store(t, std::memory_order_relaxed);
        ++samples_;
        sum_target_ += t;
        sum_mhz_ += mhz;
        at_max_ += mhz + slack_ >= max_mhz_ ? 1 : 0;
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(5));
    }
  }
  void* lib_ = nullptr;
  nvmlReturn_t (*init_)() = nullptr;
  nvmlReturn_t (*shutdown_)() = nullptr;
  nvmlReturn_t (*by_pci_)(const char*, nvmlDevice_t*) = nullptr;
  nvmlReturn_t (*clock_)(nvmlDevice_t, nvmlClockType_t, unsigned int*) = nullptr;
  nvmlReturn_t (*max_clock_)(nvmlDevice_t, nvmlClockType_t, unsigned int*) = nullptr;
  nvmlDevice_t dev_{};
  unsigned int max_mhz_ = 0;
  bool ok_ = false;
  int n_sm_, min_sms_;
  unsigned slack_;
  std::atomic<int> target_;
  std::atomic<bool> stop_{false};
  std::thread th_;
  long long samples_ = 0, at_max_ = 0;
  double sum_target_ = 0, sum_mhz_ = 0;
};


}  // namespace microslice
