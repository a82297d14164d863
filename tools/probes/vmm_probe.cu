// Probe: can one VMM virtual range mix local-HBM and host-DRAM (HOST_NUMA) 2 MB chunks,
// and what read bandwidth does a kernel see from each tier?  (memory tier design check)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); \
  printf("FAIL %s -> %d %s\n", #x, (int)r_, s); return 1; } } while (0)

__global__ void fill(uint4* p, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(i ^ seed, i + seed, (unsigned)(i >> 3), seed);
}
__global__ void rsum(const uint4* p, size_t n, unsigned long long* out) {
  unsigned long long s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = p[i]; s += v.x + v.y + v.z + v.w;
  }
  atomicAdd(out, s);
}

static int map_range(CUdeviceptr* va, size_t chunk, int n, const std::vector<int>& where, int dev, int numa) {
  CK(cuMemAddressReserve(va, chunk * n, 0, 0, 0));
  for (int i = 0; i < n; ++i) {
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    if (where[i] < 0) { prop.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA; prop.location.id = numa; }
    else { prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE; prop.location.id = where[i]; }
    CUmemGenericAllocationHandle h;
    CK(cuMemCreate(&h, chunk, &prop, 0));
    CK(cuMemMap(*va + chunk * i, chunk, 0, h, 0));
    CK(cuMemRelease(h));
  }
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = dev; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(*va, chunk * n, &ad, 1));
  return 0;
}

int main() {
  CK(cuInit(0));
  int ndev = 0; CK(cuDeviceGetCount(&ndev));
  printf("devices %d\n", ndev);
  for (int a = 0; a < ndev; ++a) for (int b = 0; b < ndev; ++b) if (a != b) {
    int ok = 0; cudaDeviceCanAccessPeer(&ok, a, b); printf("p2p %d->%d %d\n", a, b, ok); }
  CUdevice d; CK(cuDeviceGet(&d, 0));
  int numa = -1; cuDeviceGetAttribute(&numa, CU_DEVICE_ATTRIBUTE_HOST_NUMA_ID, d);
  int vmm = 0; cuDeviceGetAttribute(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, d);
  printf("host_numa_id %d vmm %d\n", numa, vmm);
  cudaSetDevice(0); cudaFree(0);
  CUmemAllocationProp gp = {}; gp.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  gp.location.type = CU_MEM_LOCATION_TYPE_DEVICE; gp.location.id = 0;
  size_t g = 0; CK(cuMemGetAllocationGranularity(&g, &gp, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  CUmemAllocationProp hp = gp; hp.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA; hp.location.id = numa < 0 ? 0 : numa;
  size_t gh = 0; CUresult rh = cuMemGetAllocationGranularity(&gh, &hp, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
  printf("granularity dev %zu host %zu (rc %d)\n", g, gh, (int)rh);
  const size_t chunk = 2 << 20; const int n = 256;  // 512 MB per range
  for (int mode = 0; mode < 3; ++mode) {
    std::vector<int> where(n);
    for (int i = 0; i < n; ++i) where[i] = mode == 0 ? 0 : mode == 1 ? -1 : (i % 8 == 7 ? -1 : 0);
    CUdeviceptr va;
    if (map_range(&va, chunk, n, where, 0, numa < 0 ? 0 : numa)) { printf("mode %d map failed\n", mode); continue; }
    uint4* p = (uint4*)va; size_t cnt = chunk * n / 16;
    unsigned long long* out; cudaMalloc(&out, 8);
    fill<<<148 * 4, 512>>>(p, cnt, 7); 
    cudaError_t e = cudaDeviceSynchronize(); if (e) { printf("fill err %s\n", cudaGetErrorString(e)); return 1; }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaMemset(out, 0, 8);
      cudaEventRecord(e0); rsum<<<148 * 4, 512>>>(p, cnt, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    unsigned long long h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    // host-side check of the sum
    unsigned long long want = 0;
    for (size_t i = 0; i < cnt; ++i) want += (unsigned)(i ^ 7) + (unsigned)(i + 7) + (unsigned)(i >> 3) + 7u;
    printf("mode %s: read %.1f MB in %.3f ms = %.1f GB/s  sum %s\n", mode == 0 ? "local" : mode == 1 ? "host" : "mixed 1/8 host",
           chunk * n / 1e6, best, chunk * n / (best * 1e6), h == want ? "ok" : "MISMATCH");
    // ping probe: 4 MB local -> range copy
    void* src; cudaMalloc(&src, 4 << 20);
    float pb = 1e9;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(e0); cudaMemcpyAsync(p + (mode == 2 ? (7 * chunk / 16) : 0), src, 2 << 20, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < pb) pb = ms; }
    printf("  probe 2MB copy into chunk: %.2f us\n", pb * 1e3);
    cuMemUnmap(va, chunk * n); cuMemAddressFree(va, chunk * n); cudaFree(src); cudaFree(out);
  }
  return 0;
}
