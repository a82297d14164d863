// Latency probe for the preemption path's host<->device signalling primitives on B200.
// Measures: host-mapped flag propagation (ld.acquire.sys vs ld.relaxed.sys), the
// host<->%globaltimer clock offset, stream-memop doorbell release latency, plain launch
// latency, and flag->exit latency of a 148-CTA persistent spinner.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o latency_probe latency_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <time.h>
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
#define CKD(x) do { CUresult e = (x); if (e != CUDA_SUCCESS) { const char* s; cuGetErrorString(e, &s); printf("CU %s @%d: %s\n", #x, __LINE__, s); exit(1);} } while (0)

static inline int64_t host_ns() { timespec ts; clock_gettime(CLOCK_REALTIME, &ts); return ts.tv_sec * 1000000000ll + ts.tv_nsec; }
__device__ __forceinline__ uint64_t gtimer() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint32_t ld_acq_sys(const uint32_t* p) { uint32_t v; asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ uint32_t ld_rlx_sys(const uint32_t* p) { uint32_t v; asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_rel_sys(uint32_t* p, uint32_t v) { asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }

// ping-pong echo: device waits for ping==k, stamps globaltimer, writes pong=k.
__global__ void echo_kernel(const uint32_t* ping, uint32_t* pong, uint64_t* stamps, int n, int mode) {
  for (int k = 1; k <= n; ++k) {
    while ((mode ? ld_rlx_sys(ping) : ld_acq_sys(ping)) < (uint32_t)k) {}
    stamps[k - 1] = gtimer();
    st_rel_sys(pong, k);
  }
}

__global__ void stamp_kernel(uint64_t* out) { out[0] = gtimer(); }

// persistent spinner: each CTA "works" in chunks of `work_ns`, polls the flag between chunks.
__global__ void spinner(const uint32_t* flag, uint32_t* dflag, uint64_t* exit_ts, uint64_t* seen_ts, uint64_t work_ns, int mode) {
  __shared__ int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  while (true) {
    uint64_t t0 = gtimer();
    while (gtimer() - t0 < work_ns) {}
    if (threadIdx.x == 0) {
      uint32_t f;
      if (mode == 0) f = ld_acq_sys(flag);
      else {  // mode 1: CTA 0 mirrors host flag into device memory, others poll device mirror
        if (blockIdx.x == 0) { f = ld_acq_sys(flag); if (f) { asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(dflag), "r"(f) : "memory"); } }
        else { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(dflag) : "memory"); }
      }
      if (f) { stop = 1; seen_ts[blockIdx.x] = gtimer(); }
    }
    __syncthreads();
    if (stop) break;
    __syncthreads();
  }
  if (threadIdx.x == 0) exit_ts[blockIdx.x] = gtimer();
}

static void stats(const char* name, std::vector<double> v) {
  std::sort(v.begin(), v.end());
  auto pct = [&](double q) { size_t r = (size_t)(q * v.size()); if (r >= v.size()) r = v.size() - 1; return v[r]; };
  printf("%-44s n=%zu min=%.2f p50=%.2f p90=%.2f p99=%.2f max=%.2f us\n", name, v.size(), v[0] / 1e3, pct(0.5) / 1e3, pct(0.9) / 1e3, pct(0.99) / 1e3, v.back() / 1e3);
}

int main() {
  CK(cudaSetDevice(0));
  CKD(cuInit(0));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s sms=%d cc=%d.%d\n", prop.name, prop.multiProcessorCount, prop.major, prop.minor);
  CUdevice cud; CKD(cuDeviceGet(&cud, 0));
  int memops = 0; cuDeviceGetAttribute(&memops, CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_MEM_OPS_V1, cud);
  int lo, hi; CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  printf("stream_mem_ops=%d prio_range=[%d,%d]\n", memops, lo, hi);

  uint32_t* h; CK(cudaHostAlloc(&h, 4096, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(h, 0, 4096);
  uint32_t* d; CK(cudaHostGetDevicePointer(&d, h, 0));
  volatile uint32_t* hping = h; volatile uint32_t* hpong = h + 32;
  uint64_t* dstamps; CK(cudaMalloc(&dstamps, 1 << 20));
  uint32_t* dflag; CK(cudaMalloc(&dflag, 64)); CK(cudaMemset(dflag, 0, 64));
  cudaStream_t s_lo, s_hi, s_mid;
  CK(cudaStreamCreateWithPriority(&s_lo, cudaStreamNonBlocking, lo));
  CK(cudaStreamCreateWithPriority(&s_hi, cudaStreamNonBlocking, hi));
  CK(cudaStreamCreateWithPriority(&s_mid, cudaStreamNonBlocking, lo));

  // ---- 1. ping-pong clock calibration / flag RTT
  double best_off = 0;
  for (int mode = 0; mode < 2; ++mode) {
    const int N = 2000;
    *hping = 0; *hpong = 0;
    echo_kernel<<<1, 1, 0, s_mid>>>(d, d + 32, dstamps, N, mode);
    std::vector<int64_t> t0(N), t1(N);
    for (int k = 1; k <= N; ++k) {
      int64_t a = host_ns();
      while (host_ns() - a < 5000) {}
      t0[k - 1] = host_ns();
      __atomic_store_n((uint32_t*)hping, (uint32_t)k, __ATOMIC_RELEASE);
      while (__atomic_load_n((uint32_t*)hpong, __ATOMIC_ACQUIRE) < (uint32_t)k) {}
      t1[k - 1] = host_ns();
    }
    CK(cudaStreamSynchronize(s_mid));
    std::vector<uint64_t> g(N); CK(cudaMemcpy(g.data(), dstamps, N * 8, cudaMemcpyDeviceToHost));
    std::vector<double> rtt(N);
    int bi = 0;
    for (int i = 0; i < N; ++i) { rtt[i] = (double)(t1[i] - t0[i]); if (rtt[i] < rtt[bi]) bi = i; }
    double off = (double)g[bi] - 0.5 * (double)(t0[bi] + t1[bi]);
    if (mode == 0) best_off = off;
    std::vector<double> oneway(N);
    for (int i = 0; i < N; ++i) oneway[i] = (double)g[i] - off - (double)t0[i];
    stats(mode ? "flag RTT (relaxed.sys)" : "flag RTT (acquire.sys)", rtt);
    stats(mode ? "host->dev one-way (relaxed)" : "host->dev one-way (acquire)", oneway);
    printf("globaltimer - host offset = %.0f ns (min rtt %.0f)\n", off, rtt[bi]);
  }
  // ---- 2. plain launch latency on hi stream (host call -> kernel start)
  {
    std::vector<double> v;
    for (int i = 0; i < 500; ++i) {
      int64_t a = host_ns();
      stamp_kernel<<<1, 1, 0, s_hi>>>(dstamps + i);
      CK(cudaStreamSynchronize(s_hi));
      (void)a;
    }
    std::vector<uint64_t> g(500);
    // redo with host stamps captured
    std::vector<int64_t> hs(500);
    for (int i = 0; i < 500; ++i) { hs[i] = host_ns(); stamp_kernel<<<1, 1, 0, s_hi>>>(dstamps + i); CK(cudaStreamSynchronize(s_hi)); }
    CK(cudaMemcpy(g.data(), dstamps, 500 * 8, cudaMemcpyDeviceToHost));
    for (int i = 0; i < 500; ++i) v.push_back((double)g[i] - best_off - (double)hs[i]);
    stats("launch: host call -> kernel start", v);
  }
  // ---- 3. stream-memop doorbell: wait(doorbell>=k) then stamp kernel
  if (memops) {
    std::vector<double> v;
    volatile uint32_t* door = h + 64; *door = 0;
    CUdeviceptr ddoor = (CUdeviceptr)(d + 64);
    for (int k = 1; k <= 300; ++k) {
      CKD(cuStreamWaitValue32((CUstream)s_hi, ddoor, k, CU_STREAM_WAIT_VALUE_GEQ));
      stamp_kernel<<<1, 1, 0, s_hi>>>(dstamps + k);
      int64_t a = host_ns(); while (host_ns() - a < 200000) {}  // let it arm
      int64_t t = host_ns();
      __atomic_store_n((uint32_t*)door, (uint32_t)k, __ATOMIC_RELEASE);
      CK(cudaStreamSynchronize(s_hi));
      uint64_t g; CK(cudaMemcpy(&g, dstamps + k, 8, cudaMemcpyDeviceToHost));
      v.push_back((double)g - best_off - (double)t);
    }
    stats("doorbell (cuStreamWaitValue32) -> kernel start", v);
  }
  // ---- 4. persistent spinner preemption: host flag -> last CTA exit
  for (int mode = 0; mode < 2; ++mode)
  for (uint64_t work : {1000ull, 4000ull}) {
    std::vector<double> seen, last;
    uint64_t *exit_ts, *seen_ts; CK(cudaMalloc(&exit_ts, 148 * 8 * 4)); CK(cudaMalloc(&seen_ts, 148 * 8 * 4));
    volatile uint32_t* flag = h + 96;
    for (int it = 0; it < 100; ++it) {
      *flag = 0; CK(cudaMemset(dflag, 0, 4));
      spinner<<<148, 128, 0, s_lo>>>(d + 96, dflag, exit_ts, seen_ts, work, mode);
      int64_t a = host_ns(); while (host_ns() - a < 300000) {}
      int64_t t = host_ns();
      __atomic_store_n((uint32_t*)flag, 1u, __ATOMIC_RELEASE);
      CK(cudaStreamSynchronize(s_lo));
      std::vector<uint64_t> ev(148), sv(148);
      CK(cudaMemcpy(ev.data(), exit_ts, 148 * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(sv.data(), seen_ts, 148 * 8, cudaMemcpyDeviceToHost));
      uint64_t mx = *std::max_element(ev.begin(), ev.end());
      uint64_t mn = *std::min_element(sv.begin(), sv.end());
      last.push_back((double)mx - best_off - (double)t);
      seen.push_back((double)mn - best_off - (double)t);
    }
    char nm[128];
    snprintf(nm, sizeof nm, "spinner mode%d work=%lluns: flag->first seen", mode, (unsigned long long)work); stats(nm, seen);
    snprintf(nm, sizeof nm, "spinner mode%d work=%lluns: flag->last exit", mode, (unsigned long long)work); stats(nm, last);
  }
  printf("done\n");
  return 0;
}
