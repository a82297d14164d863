// Gate -> successor latency on B200: stream order vs programmatic dependent launch (PDL)
// vs CUDA graph, for a tiny successor and a 144 KB-smem successor; plus a poll-loop probe.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o gate_probe gate_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <time.h>
#include <algorithm>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
static inline long long hns() { timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec * 1000000000ll + t.tv_nsec; }
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ unsigned ldacq(const unsigned* p) { unsigned v; asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }

__global__ void gate(const unsigned* door, unsigned seq, unsigned long long* t_gate, int pdl) {
  if (threadIdx.x) return;
  while ((int)(ldacq(door) - seq) < 0) __nanosleep(20);
  *t_gate = gt();
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__global__ void tiny(unsigned long long* t) { if (threadIdx.x == 0) atomicMin(t, gt()); }
__global__ void big(unsigned long long* t) {
  extern __shared__ char sm[];
  if (threadIdx.x == 0) { sm[0] = 1; atomicMin(t, gt()); }
}
__global__ void big_wait(unsigned long long* t) {
  extern __shared__ char sm[];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) { sm[0] = 1; atomicMin(t, gt()); }
}
__global__ void big_nowait(unsigned long long* t) {
  extern __shared__ char sm[];
  if (threadIdx.x == 0) { sm[0] = 1; atomicMin(t, gt()); }
}

int main() {
  CK(cudaSetDevice(0));
  int lo, hi; CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  cudaStream_t s; CK(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi));
  unsigned* h; CK(cudaHostAlloc(&h, 4096, cudaHostAllocMapped)); memset(h, 0, 4096);
  unsigned* d; CK(cudaHostGetDevicePointer(&d, h, 0));
  unsigned long long* t; CK(cudaMalloc(&t, 64));
  const int SM = 144 * 1024;
  CK(cudaFuncSetAttribute(big, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
  CK(cudaFuncSetAttribute(big_wait, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
  CK(cudaFuncSetAttribute(big_nowait, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
  unsigned seq = 0;
  auto run = [&](const char* name, int mode) {
    std::vector<double> v;
    for (int it = 0; it < 200; ++it) {
      ++seq;
      CK(cudaMemsetAsync(t, 0xFF, 16, s));
      gate<<<1, 32, 0, s>>>(d, seq, t + 1, mode >= 2);
      if (mode == 0) tiny<<<64, 256, 0, s>>>(t);
      else if (mode == 1) big<<<64, 256, SM, s>>>(t);
      else {
        cudaLaunchConfig_t cfg{}; cfg.gridDim = 64; cfg.blockDim = 256; cfg.dynamicSmemBytes = SM; cfg.stream = s;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
        if (mode == 2) CK(cudaLaunchKernelEx(&cfg, big_wait, t));
        else CK(cudaLaunchKernelEx(&cfg, big_nowait, t));
      }
      long long a = hns(); while (hns() - a < 300000) {}
      __atomic_store_n(h, seq, __ATOMIC_RELEASE);
      CK(cudaStreamSynchronize(s));
      unsigned long long r[2]; CK(cudaMemcpy(r, t, 16, cudaMemcpyDeviceToHost));
      v.push_back((double)((long long)r[0] - (long long)r[1]));
    }
    std::sort(v.begin(), v.end());
    printf("%-40s gate->first CTA p50 %.2f p90 %.2f p99 %.2f min %.2f us\n", name, v[100] / 1e3, v[180] / 1e3, v[198] / 1e3, v[0] / 1e3);
  };
  run("stream order, tiny successor", 0);
  run("stream order, 144KB successor", 1);
  run("PDL (launch_dependents + wait), 144KB", 2);
  run("PDL (launch_dependents, no wait), 144KB", 3);
  // graph: gate + big captured
  {
    std::vector<double> v;
    for (int it = 0; it < 200; ++it) {
      ++seq;
      cudaGraph_t g; cudaGraphExec_t ge;
      CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
      gate<<<1, 32, 0, s>>>(d, seq, t + 1, 0);
      big<<<64, 256, SM, s>>>(t);
      CK(cudaStreamEndCapture(s, &g));
      CK(cudaGraphInstantiate(&ge, g, 0));
      CK(cudaMemsetAsync(t, 0xFF, 16, s));
      CK(cudaGraphLaunch(ge, s));
      long long a = hns(); while (hns() - a < 300000) {}
      __atomic_store_n(h, seq, __ATOMIC_RELEASE);
      CK(cudaStreamSynchronize(s));
      unsigned long long r[2]; CK(cudaMemcpy(r, t, 16, cudaMemcpyDeviceToHost));
      v.push_back((double)((long long)r[0] - (long long)r[1]));
      cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    }
    std::sort(v.begin(), v.end());
    printf("%-40s gate->first CTA p50 %.2f p90 %.2f p99 %.2f min %.2f us\n", "graph (gate + 144KB)", v[100] / 1e3, v[180] / 1e3, v[198] / 1e3, v[0] / 1e3);
  }
  // cuStreamWaitValue32 despite the attribute
  {
    CUstream cs = (CUstream)s;
    CUresult r = cuStreamWaitValue32(cs, (CUdeviceptr)(d + 64), 1, CU_STREAM_WAIT_VALUE_GEQ);
    printf("cuStreamWaitValue32 -> %d\n", (int)r);
    if (r == CUDA_SUCCESS) {
      std::vector<double> v;
      CK(cudaMemsetAsync(t, 0xFF, 16, s));
      big<<<64, 256, SM, s>>>(t);
      long long a = hns(); while (hns() - a < 300000) {}
      long long tr = hns();
      __atomic_store_n(h + 64, 1u, __ATOMIC_RELEASE);
      CK(cudaStreamSynchronize(s));
      printf("waitvalue path completed (host %lld ns)\n", hns() - tr);
    }
  }
  printf("done\n");
  return 0;
}
