// B200 device layer: implementation of include/ms_b200.h.
//
// Owns per device: a low-priority LP stream, a highest-priority HP stream, the pinned
// host-mapped control page (MsHostPage), the device mirror of the preempt epoch, the
// per-kernel control blocks, and the registered LP kernels / HP chains with their TMA
// descriptors.  No CPU fallback: every entry point fails with MS_E_CUDA / MS_E_NODEV when
// the device or the sm_100a images are unavailable.
#include <cudaTypedefs.h>
#include <emmintrin.h>
#include <time.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "ms_b200.h"
#include "stream_kernels.cuh"
#include "tc_gemm.cuh"
#include "hp_fused.cuh"
#include "hp_gemv.cuh"
#include "tc_gemm2.cuh"
#include "hp_ops.cuh"
#include "lp_optim.cuh"

using namespace msdev;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& what) {
  g_err = what;
  return code;
}

#define MS_CUDA(expr)                                                                              \
  do {                                                                                             \
    cudaError_t e__ = (expr);                                                                      \
    if (e__ != cudaSuccess)                                                                        \
      return fail(MS_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e__));                 \
  } while (0)

int64_t now_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return static_cast<int64_t>(ts.tv_sec) * 1000000000ll + ts.tv_nsec;
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

int encode_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
              uint64_t row_stride = 0) {
  // bf16 [rows, cols] row-major (row stride `row_stride` elements, 0 = cols), box = 64 cols
  // (128 B, swizzle 128B) x box_rows.
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return fail(MS_E_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {(row_stride ? row_stride : cols) * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MS_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return 0;
}

// C (bf16 [rows][cols]) for the TMA-store epilogue: 32 x 32 boxes, 64B swizzle.
int encode_c(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols) {
  if (!g_encode) {
    CUtensorMap dummy;
    if (int rc = encode_2d(&dummy, base, 128, 64, 64)) return rc;
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MS_E_CUDA, "cuTensorMapEncodeTiled(C) failed: " + std::to_string(r));
  return 0;
}

int encode_kblock_major(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  // bf16 [cols/64][rows][64]; box = 64 x box_rows x 1 = box_rows x 128 B contiguous.
  if (!g_encode) {
    CUtensorMap dummy;
    if (int rc = encode_2d(&dummy, base, 128, 64, 64)) return rc;
  }
  cuuint64_t dims[3] = {64, rows, cols / 64};
  cuuint64_t strides[2] = {128, rows * 128};
  cuuint32_t box[3] = {64, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MS_E_CUDA, "cuTensorMapEncodeTiled(3d) failed: " + std::to_string(r));
  return 0;
}

constexpr int kRedoCap = 8192;
constexpr int kMaxChainOps = 512;
constexpr int kGemvHeadKbDefault = 0;  // head prefetch (hp_gemv.cuh), A/B: tools/gemv_head_ab.py
constexpr bool kGemvDynamicDefault = false;  // decided by tools/gemv_dynamic_ab.py  // per-op chains (config-2 ResNet-50: ~160 ops); fused / GEMV plans are shorter

// FFI callers may pass any id: every entry point that indexes a slot checks it first.
#define MS_CHECK_LP(d, id) \
  if (!(d) || (id) < 0 || (id) >= MS_MAX_LP || !(d)->lp_slots[id].used) return fail(MS_E_ARG, "bad LP id")
#define MS_CHECK_CHAIN(d, cid) \
  if (!(d) || (cid) < 0 || (cid) >= MS_MAX_HP_CHAINS || !(d)->chains[cid].used) return fail(MS_E_ARG, "bad chain")
constexpr int kAxpyMaxPad = 200 * 1024;  // residency-capping dynamic smem of the HBM streamer
constexpr int kGateSmem = 40 * 1024;

struct LpSlot {
  bool used = false;
  bool pair = false;  // GEMM on CTA pairs (tc_gemm2.cuh): 256 x pair_tn tiles
  int pair_tn = 256;
  long long half_base = 0;  // pair_tn 512: units >= half_base are column parts of the last wave's tiles
  int half_units = 0;       // part units (tail_parts per tile)
  int tail_parts = 2;       // 2: 256-column halves, 4: 128-column quarters
  ms_lp_desc desc{};
  uint64_t total_tiles = 0;
  int tiles_m = 0, tiles_n = 0;
  CUtensorMap tma_a{}, tma_b{}, tma_c{};
  CUtensorMap tma_bq{};  // pair GEMMs: B with 64-row boxes (quarter units)
  unsigned long long* redo[2] = {nullptr, nullptr};
  uint64_t run_id = 0;
  uint64_t redo_carry = 0;  // redo entries waiting in redo[run_id % 2] for the next run
  uint64_t last_begin = 0, last_end = 0, last_redo_in = 0;
  int64_t t_launch_host = 0;
  bool launched = false;
  int split = 1;                    // GEMM k-slices per tile (units = tiles x split)
  float* ws = nullptr;              // split-K fp32 partials [tiles][split][128 x BN]
  unsigned int* tile_cnt = nullptr; // split-K: slices finished per tile (self-resetting)
  uint8_t* slow = nullptr;          // streamer off-device tile groups (ms_lp_set_slow_tiles)
  unsigned int* slow_sem = nullptr;
  int slow_group = 0, slow_max = 0;
};

struct HpOpRt {
  ms_hp_op op{};
  CUtensorMap tma_a{}, tma_b{}, tma_c{};
  int tiles_m = 0, tiles_n = 0;
  int ctl_index = 0;
  int split = 1;
  float* ws = nullptr;
  unsigned int* tile_cnt = nullptr;
  __nv_bfloat16* b_tiled = nullptr;  // k-block-major copy of the weights (captured at registration)
  int reduce_ctl_index = 0;          // control block of the split-K reduce kernel
  __nv_bfloat16* tmp = nullptr;      // GEMM_SWIGLU per-op path: [m x 2n] gate|up before the SwiGLU
  int act_ctl_index = 0;             // GEMM_SWIGLU per-op path: control block of the SwiGLU kernel
  bool gemv = false;                 // m == 1 GEMM / GEMM_SWIGLU: runs in the HBM-streaming GEMV chain
};

struct HpChain {
  bool used = false;
  std::vector<HpOpRt> ops;
  // Fused plan (hp_fused.cuh): the chain's kernel ops [fused_first, fused_last] as one launch.
  bool fusable = false;
  int fused_first = -1, fused_last = -1;
  int fused_grid = 0;
  int fused_ctl = 0;
  int fused_cs = 1;  // cluster size (k-slices reduced through DSMEM) or 1
  int fused_bn = 128;  // output tile width of the fused plan (32: narrow plan)
  int n_phases = 0;
  FusedProgram* prog_d = nullptr;
  uint32_t* phase_d = nullptr;
  std::vector<FusedOpDesc> descs;  // copied into the launch parameters
  int l2_prefetch = 1;
  std::vector<float*> fused_ws;
  // Batch-1 chain (every kernel op has m == 1): one hp_gemv_kernel launch (hp_gemv.cuh).
  bool gemv = false;
  std::vector<GemvOpDesc> gemv_descs;
  GemvOpDesc* gemv_descs_d = nullptr;  // device copy (bulk-loaded by every CTA)
  uint32_t* wire_d = nullptr;       // tagged op->op handoff words
  mutable uint32_t launches = 0;    // wire tag source (one tag per launch, stream-ordered)
  // Leading H2D ops (e2e request input) run on the hpcopy stream when armed; the chain
  // kernels wait for this event.
  int lead_copies = 0;
  cudaEvent_t in_ev = nullptr;
  // SM pull of the leading H2D (default e2e mode): device views of the host sources
  std::vector<uint64_t> pull_src;
  unsigned int* pull_done = nullptr;
};

}  // namespace

struct ms_dev {
  int ordinal = 0;
  cudaDeviceProp prop{};
  int prio_low = 0, prio_high = 0;
  cudaStream_t lp = nullptr, hp = nullptr, aux = nullptr;
  // e2e request input: an armed chain whose first op is an H2D copy gets a second gate on
  // this stream, so the copy engine starts at the ring, concurrent with the LP drain; the
  // chain on `hp` waits for the copy's event instead of queueing the copy itself.
  cudaStream_t hpcopy = nullptr;
  MsHostPage* page = nullptr;    // host view
  MsHostPage* page_d = nullptr;  // device view of the same page
  MsDevMirror* mirror = nullptr;
  MsLpCtl* ctl = nullptr;        // [MS_N_CTL]
  MsHpCtl* hp_ctl = nullptr;     // [MS_MAX_HP_CHAINS]
  unsigned long long* dummy_redo = nullptr;
  LpSlot lp_slots[MS_MAX_LP];
  HpChain chains[MS_MAX_HP_CHAINS];
  int next_hp_ctl = MS_MAX_LP;
  int stream_memops = 0;
  // device-side event trace (ms_trace_enable / ms_trace_drain)
  bool trace_on = false;
  MsTrace* trace_dev = nullptr;          // device copy of the descriptor
  MsTraceEvent* trace_ev = nullptr;      // pinned host ring
  unsigned long long* trace_head = nullptr;
  uint64_t trace_cap = 0, trace_read = 0, trace_lost = 0;
  uint32_t hp_seq = 0;  // monotonic doorbell sequence of this device
  unsigned long long* dbg = nullptr;  // per-CTA phase stamps of the next LP run (diagnostics)
  unsigned long long* dbg_buf = nullptr;
  // SMs an LP grid leaves free: the parked HP gate's home.  A gate parked on an SM keeps an
  // LP CTA (and, measured, a whole CTA pair) of a grid that needs every SM off that SM
  // until the next ring (tools/pair_gate_probe.py: a 74-pair grid never completes while a
  // gate is armed).  CTA-pair grids round the reserve up to a whole TPC (2 SMs): 73 pairs.
  int lp_sm_reserve = 1;
  int lp_align_clusters[5] = {0, 0, 0, 0, 0};  // max active C-CTA clusters of the LP GEMM (MS_LP_CLUSTER_ALIGN)
  int hp_fused = 1;       // 0: per-op kernels; 1: fused launch (cluster split-K when it fits); 2: fused, no clusters
};

namespace {

int set_smem_attrs() {
  static bool done = false;
  if (done) return 0;
  MS_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               GemmCfg<256>::kSmemBytes));
  MS_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               GemmCfg<128>::kSmemBytes));
  MS_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               GemmCfg<64>::kSmemBytes));
  MS_CUDA(cudaFuncSetAttribute(hp_fused_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               FusedCfg<1>::kSmemBytes));
  MS_CUDA(cudaFuncSetAttribute(hp_fused_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               FusedCfg<2>::kSmemBytes));
  MS_CUDA(cudaFuncSetAttribute(hp_fused_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               FusedCfg<4>::kSmemBytes));
  MS_CUDA(cudaFuncSetAttribute(hp_fused_kernel<1, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               FusedCfg<1, 32>::kSmemBytes));
  MS_CUDA(cudaFuncSetAttribute(hp_gemv_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemvSmemBytes));
  MS_CUDA(cudaFuncSetAttribute(hp_gemv_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemvSmemBytes));
  MS_CUDA(cudaFuncSetAttribute(attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnSmemBytes));
  MS_CUDA(cudaFuncSetAttribute(tc_gemm2_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               Gemm2Cfg<256>::kSmemBytes));
  MS_CUDA(cudaFuncSetAttribute(tc_gemm2_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               Gemm2Cfg<512>::kSmemBytes));
  MS_CUDA(cudaFuncSetAttribute(axpy_kernel<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kAxpyMaxPad));
  MS_CUDA(cudaFuncSetAttribute(axpy_kernel<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kAxpyMaxPad));
  MS_CUDA(cudaFuncSetAttribute(axpy_kernel<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kAxpyMaxPad));
  MS_CUDA(cudaFuncSetAttribute(axpy_kernel<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kAxpyMaxPad));
  // Every kernel asks for the maximum shared-memory carveout.  An SM takes the carveout of
  // the first kernel that lands on it while it is idle; a small kernel (the HP gate, the
  // input pull, a streamer CTA) that configured an SM for little shared memory would keep
  // a later 210 KB LP GEMM CTA off that SM until it exits — with the gate parked there
  // until the next ring, a persistent LP grid that needs every SM never becomes fully
  // resident (observed: a CTA pair starting only after the HP chain, and a drain deadlock
  // when the scheduler waits for LP before ringing the armed gate).
  const int mx = cudaSharedmemCarveoutMaxShared;
#define MS_CARVE(...) MS_CUDA(cudaFuncSetAttribute(__VA_ARGS__, cudaFuncAttributePreferredSharedMemoryCarveout, mx))
  MS_CARVE(gate_kernel);
  MS_CARVE(hp_pull_kernel);
  MS_CARVE(hp_notify_kernel);
  MS_CARVE(echo_kernel);
  MS_CARVE(init_ctl_kernel);
  MS_CARVE(kblock_major_kernel);
  MS_CARVE(kblock_major_swiglu_kernel);
  MS_CARVE(synth_fill_kernel);
  MS_CARVE(synth_fill_f32_kernel);
  MS_CARVE(add_ln_kernel);
  MS_CARVE(attn_kernel);
  MS_CARVE(avgpool_kernel);
  MS_CARVE(maxpool_kernel);
  MS_CARVE(bias_act_kernel);
  MS_CARVE(bias_gelu_kernel);
  MS_CARVE(im2col_kernel);
  MS_CARVE(silu_mul_kernel);
  MS_CARVE(splitk_reduce_kernel);
  MS_CARVE(axpy_kernel<1, 1>);
  MS_CARVE(axpy_kernel<2, 1>);
  MS_CARVE(axpy_kernel<4, 1>);
  MS_CARVE(axpy_kernel<8, 1>);
  MS_CARVE(axpy_kernel<1, kAxpyGroups>);
  MS_CARVE(axpy_kernel<2, kAxpyGroups>);
  MS_CARVE(axpy_kernel<4, kAxpyGroups>);
  MS_CARVE(axpy_kernel<8, kAxpyGroups>);
  MS_CARVE(optim_kernel<1>);
  MS_CARVE(optim_kernel<2>);
  MS_CARVE(optim_kernel<4>);
  MS_CARVE(optim_kernel<8>);
  MS_CARVE(tc_gemm_kernel<64>);
  MS_CARVE(tc_gemm_kernel<128>);
  MS_CARVE(tc_gemm_kernel<256>);
  MS_CARVE(tc_gemm2_kernel<256>);
  MS_CARVE(tc_gemm2_kernel<512>);
  MS_CARVE(hp_fused_kernel<1>);
  MS_CARVE(hp_fused_kernel<2>);
  MS_CARVE(hp_fused_kernel<4>);
  MS_CARVE(hp_fused_kernel<1, 32>);
  MS_CARVE(hp_gemv_kernel<false>);
  MS_CARVE(hp_gemv_kernel<true>);
#undef MS_CARVE
  done = true;
  return 0;
}

TileRun base_run(ms_dev* d, int ctl_index) {
  TileRun r{};
  r.ctl = d->ctl + ctl_index;
  r.redo_in = d->dummy_redo;
  r.redo_out = d->dummy_redo + 16;
  r.host_line = reinterpret_cast<const uint64_t*>(&d->page_d->lp_line[0]);
  r.mirror = d->mirror;
  r.trace = d->trace_on ? d->trace_dev : nullptr;
  return r;
}

// `pdl`: launch with programmatic stream serialisation, so the kernel is scheduled as soon
// as its predecessor triggers griddepcontrol.launch_dependents (HP chains only).
template <typename K, typename... Args>
cudaError_t launch_kc(K kernel, int grid, int block, int smem, cudaStream_t st, bool pdl, int cluster, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}
template <typename K, typename... Args>
cudaError_t launch_k(K kernel, int grid, int block, int smem, cudaStream_t st, bool pdl, Args... args) {
  return launch_kc(kernel, grid, block, smem, st, pdl, 1, args...);
}

int launch_gemm(ms_dev* d, int block_n, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                const GemmParams& p, int grid, cudaStream_t st, bool pdl = false) {
  switch (block_n) {
    case 256:
      MS_CUDA(launch_k(tc_gemm_kernel<256>, grid, 256, GemmCfg<256>::kSmemBytes, st, pdl, ta, tb, tc, p));
      break;
    case 128:
      MS_CUDA(launch_k(tc_gemm_kernel<128>, grid, 256, GemmCfg<128>::kSmemBytes, st, pdl, ta, tb, tc, p));
      break;
    case 64:
      MS_CUDA(launch_k(tc_gemm_kernel<64>, grid, 256, GemmCfg<64>::kSmemBytes, st, pdl, ta, tb, tc, p));
      break;
    default:
      return fail(MS_E_ARG, "block_n must be 64, 128 or 256");
  }
  (void)d;
  return 0;
}

bool is_copy(const ms_hp_op& op) { return op.kind == MS_HP_H2D || op.kind == MS_HP_D2H; }
// Config-2/3 glue ops (hp_ops.cuh): per-op kernels only (never fused / GEMV-planned).
bool is_glue(int kind) {
  return kind == MS_HP_IM2COL || kind == MS_HP_BIAS_ACT || kind == MS_HP_MAXPOOL || kind == MS_HP_AVGPOOL ||
         kind == MS_HP_ATTN || kind == MS_HP_ADD_LN;
}

int launch_glue(ms_dev* d, const HpOpRt& o, const TileRun& r, bool pdl) {
  HpOpParams q{};
  q.run = r;
  q.a = reinterpret_cast<const __nv_bfloat16*>(o.op.a);
  q.b = reinterpret_cast<const __nv_bfloat16*>(o.op.b);
  q.bias = reinterpret_cast<const __nv_bfloat16*>(o.op.bias);
  q.c = reinterpret_cast<__nv_bfloat16*>(o.op.c);
  q.m = static_cast<int>(o.op.m);
  q.n = static_cast<int>(o.op.n);
  const ms_hp_geo& g = o.op.geo;
  q.h = g.h;
  q.w = g.w;
  q.cin = g.cin;
  q.kh = g.kh;
  q.kw = g.kw;
  q.stride = g.stride;
  q.pad = g.pad;
  q.flags = g.flags;
  if (g.stride > 0) {
    q.ho = (g.h + 2 * g.pad - g.kh) / g.stride + 1;
    q.wo = (g.w + 2 * g.pad - g.kw) / g.stride + 1;
  }
  const int sms = d->prop.multiProcessorCount;
  auto grid_for = [&](long long vecs) {
    return static_cast<int>(std::max<long long>(1, std::min<long long>((vecs + kHpOpThreads - 1) / kHpOpThreads, 4ll * sms)));
  };
  switch (o.op.kind) {
    case MS_HP_IM2COL:
      MS_CUDA(launch_k(im2col_kernel, grid_for(o.op.m * (o.op.n / 8)), kHpOpThreads, 0, d->hp, pdl, q));
      break;
    case MS_HP_BIAS_ACT:
      MS_CUDA(launch_k(bias_act_kernel, grid_for(o.op.m * (o.op.n / 8)), kHpOpThreads, 0, d->hp, pdl, q));
      break;
    case MS_HP_MAXPOOL:
      MS_CUDA(launch_k(maxpool_kernel, grid_for(o.op.m * (g.cin / 8)), kHpOpThreads, 0, d->hp, pdl, q));
      break;
    case MS_HP_AVGPOOL:
      MS_CUDA(launch_k(avgpool_kernel, grid_for(o.op.m * (o.op.n / 8)), kHpOpThreads, 0, d->hp, pdl, q));
      break;
    case MS_HP_ATTN:
      MS_CUDA(launch_k(attn_kernel, static_cast<int>((o.op.n / 64) * (o.op.m / 16)), 128, kAttnSmemBytes, d->hp, pdl, q));
      break;
    case MS_HP_ADD_LN:
      MS_CUDA(launch_k(add_ln_kernel, static_cast<int>(std::min<int64_t>(o.op.m, sms)), kHpOpThreads, 0, d->hp, pdl, q));
      break;
    default:
      return fail(MS_E_ARG, "not a glue op");
  }
  return 0;
}

// Registration checks of a glue op (shapes the kernels above assume).
int check_glue(const ms_hp_op& op) {
  const ms_hp_geo& g = op.geo;
  if (op.m <= 0 || op.n <= 0 || op.n % 8 || !op.a || !op.c) return fail(MS_E_ARG, "glue op: m, n > 0, n % 8 == 0, a, c");
  if ((op.a | op.b | op.c | op.bias) % 16) return fail(MS_E_ARG, "glue op operands must be 16-byte aligned");
  switch (op.kind) {
    case MS_HP_IM2COL:
    case MS_HP_MAXPOOL: {
      if (g.h <= 0 || g.w <= 0 || g.cin <= 0 || g.kh <= 0 || g.kw <= 0 || g.stride <= 0 || g.pad < 0)
        return fail(MS_E_ARG, "im2col / maxpool geometry");
      const int64_t ho = (g.h + 2 * g.pad - g.kh) / g.stride + 1, wo = (g.w + 2 * g.pad - g.kw) / g.stride + 1;
      if (op.m < ho * wo) return fail(MS_E_ARG, "im2col / maxpool: m < output pixels");
      if (op.kind == MS_HP_IM2COL && op.n < static_cast<int64_t>(g.kh) * g.kw * g.cin)
        return fail(MS_E_ARG, "im2col: n < kh * kw * cin");
      if (op.kind == MS_HP_MAXPOOL && (g.cin % 8 || op.n != g.cin)) return fail(MS_E_ARG, "maxpool: n == cin, cin % 8 == 0");
      return 0;
    }
    case MS_HP_BIAS_ACT:
      if (!op.bias) return fail(MS_E_ARG, "bias_act needs a bias");
      return 0;
    case MS_HP_AVGPOOL:
      if (g.h <= 0 || g.w <= 0) return fail(MS_E_ARG, "avgpool: h, w");
      return 0;
    case MS_HP_ATTN:
      if (op.n % 64 || op.m % 16 || op.m > kAttnMaxS) return fail(MS_E_ARG, "attn: n % 64 == 0, m % 16 == 0, m <= 256");
      return 0;
    case MS_HP_ADD_LN:
      if (!op.b || !op.bias || op.n > 8 * kHpOpThreads) return fail(MS_E_ARG, "add_ln: b, bias, n <= 2048");
      return 0;
  }
  return fail(MS_E_ARG, "not a glue op");
}

int launch_hp_op(ms_dev* d, int chain_id, const HpChain& ch, size_t i, uint32_t seq, bool after_gate,
                 bool after_pull = false) {
  const HpOpRt& o = ch.ops[i];
  if (o.op.kind == MS_HP_H2D || o.op.kind == MS_HP_D2H) {
    MS_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(o.op.c), reinterpret_cast<const void*>(o.op.a),
                            static_cast<size_t>(o.op.m), cudaMemcpyDefault, d->hp));
    if (i + 1 == ch.ops.size()) {
      hp_notify_kernel<<<1, 1, 0, d->hp>>>(d->hp_ctl + chain_id, &d->page_d->hp[chain_id], seq,
                                           d->trace_on ? d->trace_dev : nullptr, chain_id);
      MS_CUDA(cudaGetLastError());
    }
    return 0;
  }
  // first / last *kernel* of the chain carry the chain's start stamp / completion record
  size_t first_k = 0, last_k = ch.ops.size() - 1;
  while (first_k < ch.ops.size() && is_copy(ch.ops[first_k].op)) ++first_k;
  while (last_k > 0 && is_copy(ch.ops[last_k].op)) --last_k;
  TileRun r = base_run(d, o.ctl_index);
  r.hp_ctl = d->hp_ctl + chain_id;
  r.slot = chain_id;  // (HP runs are not preemptible: slot only names the chain in the trace)
  r.hp_rec = &d->page_d->hp[chain_id];
  r.hp_first = i == first_k;
  r.dbg = d->dbg;
  r.hp_last = i == last_k && !is_copy(ch.ops.back().op);
  r.hp_seq = seq;
  // PDL when the stream predecessor is a kernel (the gate, or the previous chain kernel);
  // the chain's first kernel does not depend on the gate's output, later ones wait.
  const bool prev_is_kernel = after_pull || (i > 0 ? !is_copy(ch.ops[i - 1].op) : after_gate);
  r.pdl_wait = (i > 0 && prev_is_kernel) || after_pull;
  if (after_pull) r.hp_first = 0;  // the pull kernel stamps t_first_cta when the input is resident
  if (is_glue(o.op.kind)) return launch_glue(d, o, r, prev_is_kernel);
  if (o.op.kind == MS_HP_GEMM_SWIGLU) {
    // GEMM into tmp ([gate | up] halves), then the SwiGLU kernel (PDL) writes c.
    const bool last = r.hp_last;
    GemmParams p{};
    p.run = r;
    p.run.hp_last = 0;
    p.run.begin = 0;
    p.run.end = p.run.budget0 = static_cast<unsigned long long>(o.tiles_m) * o.tiles_n;
    p.split_k = 1;
    p.m = static_cast<int>(o.op.m);
    p.n = static_cast<int>(2 * o.op.n);
    p.k = static_cast<int>(o.op.k);
    p.tiles_m = o.tiles_m;
    p.tiles_n = o.tiles_n;
    p.group_m = 16;
    p.c = o.tmp;
    const int grid = static_cast<int>(std::min<uint64_t>(p.run.end, d->prop.multiProcessorCount));
    if (int rc = launch_gemm(d, 128, o.tma_a, o.tma_b, o.tma_c, p, grid, d->hp, prev_is_kernel)) return rc;
    BiasGeluParams q{};
    q.run = base_run(d, o.act_ctl_index);
    q.run.hp_ctl = r.hp_ctl;
    q.run.hp_rec = r.hp_rec;
    q.run.hp_last = last;
    q.run.hp_seq = seq;
    q.run.pdl_wait = 1;
    q.run.dbg = d->dbg;
    q.run.begin = 0;
    q.run.end = q.run.budget0 = static_cast<unsigned long long>(o.op.m);
    q.x = o.tmp;
    q.out = reinterpret_cast<__nv_bfloat16*>(o.op.c);
    q.rows = static_cast<int>(o.op.m);
    q.cols = static_cast<int>(o.op.n);
    const int qgrid = static_cast<int>(std::min<int64_t>(o.op.m, d->prop.multiProcessorCount));
    MS_CUDA(launch_k(silu_mul_kernel, qgrid, 256, 0, d->hp, true, q));
    return 0;
  }
  if (o.op.kind == MS_HP_GEMM) {
    GemmParams p{};
    p.run = r;
    p.run.begin = 0;
    p.run.end = p.run.budget0 = static_cast<unsigned long long>(o.tiles_m) * o.tiles_n * o.split;
    p.split_k = o.split;
    p.ws = o.ws;
    p.tile_cnt = nullptr;  // split-K partials are reduced by the next (PDL) kernel
    p.b_kblock_major = o.b_tiled != nullptr || o.op.b_layout == 2;
    p.m = static_cast<int>(o.op.m);
    p.n = static_cast<int>(o.op.n);
    p.k = static_cast<int>(o.op.k);
    p.tiles_m = o.tiles_m;
    p.tiles_n = o.tiles_n;
    p.group_m = 16;
    p.c = reinterpret_cast<__nv_bfloat16*>(o.op.c);
    const __nv_bfloat16* e_bias = reinterpret_cast<const __nv_bfloat16*>(o.op.bias);
    const __nv_bfloat16* e_resid = reinterpret_cast<const __nv_bfloat16*>(o.op.resid);
    const int e_act = (o.op.geo.flags & 1) ? 1 : (o.op.geo.flags & 2) ? 2 : 0;
    const int grid = static_cast<int>(std::min<uint64_t>(p.run.end, d->prop.multiProcessorCount));
    if (o.split == 1) {
      p.bias = e_bias;
      p.resid = e_resid;
      p.act = e_act;
      return launch_gemm(d, o.op.block_n, o.tma_a, o.tma_b, o.tma_c, p, grid, d->hp, prev_is_kernel);
    }
    // split-K: the GEMM streams partials; the reduce kernel carries the chain's last-op role
    const bool last = p.run.hp_last;
    p.run.hp_last = 0;
    if (int rc = launch_gemm(d, o.op.block_n, o.tma_a, o.tma_b, o.tma_c, p, grid, d->hp, prev_is_kernel)) return rc;
    SplitReduceParams rp{};
    rp.run = base_run(d, o.reduce_ctl_index);
    rp.run.hp_ctl = r.hp_ctl;
    rp.run.hp_rec = r.hp_rec;
    rp.run.hp_first = 0;
    rp.run.hp_last = last;
    rp.run.hp_seq = seq;
    rp.run.pdl_wait = 1;
    rp.run.dbg = d->dbg;
    rp.ws = reinterpret_cast<const float4*>(o.ws);
    rp.c = reinterpret_cast<__nv_bfloat16*>(o.op.c);
    rp.n = static_cast<int>(o.op.n);
    rp.tiles_m = o.tiles_m;
    rp.tiles_n = o.tiles_n;
    rp.group_m = 16;
    rp.bn = o.op.block_n;
    rp.split = o.split;
    rp.total = static_cast<long long>(o.tiles_m) * o.tiles_n * (o.op.block_n / 4) * kBM;
    rp.bias = e_bias;
    rp.resid = e_resid;
    rp.act = e_act;
    const int rgrid = static_cast<int>(std::min<long long>((rp.total + 255) / 256, 2ll * d->prop.multiProcessorCount));
    MS_CUDA(launch_k(splitk_reduce_kernel, rgrid, 256, 0, d->hp, true, rp));
    return 0;
  }
  BiasGeluParams p{};
  p.run = r;
  p.run.begin = 0;
  p.run.end = p.run.budget0 = static_cast<unsigned long long>(o.op.m);
  p.x = reinterpret_cast<const __nv_bfloat16*>(o.op.a);
  p.bias = reinterpret_cast<const __nv_bfloat16*>(o.op.bias);
  p.out = reinterpret_cast<__nv_bfloat16*>(o.op.c);
  p.rows = static_cast<int>(o.op.m);
  p.cols = static_cast<int>(o.op.n);
  const int grid = static_cast<int>(std::min<int64_t>(o.op.m, d->prop.multiProcessorCount));
  if (o.op.kind == MS_HP_SILU_MUL)
    MS_CUDA(launch_k(silu_mul_kernel, grid, 256, 0, d->hp, prev_is_kernel, p));
  else
    MS_CUDA(launch_k(bias_gelu_kernel, grid, 256, 0, d->hp, prev_is_kernel, p));
  return 0;
}

// Build the fused plan of a registered chain (no-op when the chain does not qualify).
int plan_fused(ms_dev* d, HpChain& ch) {
  int first = -1, last = -1;
  for (int i = 0; i < static_cast<int>(ch.ops.size()); ++i)
    if (!is_copy(ch.ops[i].op)) {
      if (first < 0) first = i;
      last = i;
    }
  if (first < 0) return 0;
  for (int i = first; i <= last; ++i) {
    const ms_hp_op& op = ch.ops[i].op;
    if (is_copy(op)) return 0;  // copies between kernels: keep per-op launches
    if (is_glue(op.kind)) return 0;
    if (op.kind == MS_HP_GEMM && (op.bias || op.resid || op.geo.flags)) return 0;  // epilogue: per-op path
    if (last - first + 1 > kFusedMaxOps) return 0;
    if (op.kind == MS_HP_GEMM && (op.m % kBM || op.n % 32 || op.k % kBK)) return 0;
    if (op.kind == MS_HP_GEMM && op.n % kFusedBN && !(op.m == kBM && d->hp_fused == 1)) return 0;
    if (op.kind == MS_HP_GEMM_SWIGLU && (op.m % kBM || op.n % 64 || op.k % kBK)) return 0;
    if ((op.kind == MS_HP_BIAS_GELU || op.kind == MS_HP_SILU_MUL) && op.n % 8) return 0;
  }
  const int sms = d->prop.multiProcessorCount;
  FusedProgram prog{};
  prog.n_ops = last - first + 1;
  // Grid <= SMs - 1: a preemptible LP kernel's CTA 0 (its host poller) may hold one SM
  // until its not-yet-resident CTAs have run; a fused chain that needed every SM could then
  // wait at its first grid phase for an SM that only frees after the LP stragglers run.
  const int max_grid = sms - 1;
  // Narrow plan (opt-in, MS_FUSED_NARROW=1; BN = 32, whole K per unit, no clusters): chains
  // of m = 128 GEMMs without SwiGLU run one 128 x 32 output tile per CTA — no split-K
  // exchange and no cluster placement.  Measured slower on the config-1 chain (90 vs 57 us):
  // 128 CTAs re-reading the same 1 MB activation from L2 per op cost more than the DSMEM
  // exchange + cluster reduction they replace.
  int bn = kFusedBN;
  {
    const char* env = getenv("MS_FUSED_NARROW");
    bool narrow = d->hp_fused == 1 && env && atoi(env) == 1;
    int widest = 0;
    for (int i = first; i <= last && narrow; ++i) {
      const ms_hp_op& op = ch.ops[i].op;
      if (op.kind == MS_HP_GEMM_SWIGLU) narrow = false;
      if (op.kind == MS_HP_GEMM) {
        if (op.m != kBM || op.n % 32 || op.n / 32 > max_grid || op.split_k > 1) narrow = false;
        widest = std::max(widest, static_cast<int>(op.n / 32));
      }
    }
    if (narrow && widest > 0) bn = 32;
  }
  for (int i = first; i <= last; ++i)
    if (ch.ops[i].op.kind == MS_HP_GEMM && ch.ops[i].op.n % bn) return 0;  // per-op launches
  struct GemmShape {
    int idx, tiles, kbs, req;
  };
  std::vector<GemmShape> gemms;
  for (int i = first; i <= last; ++i) {
    const ms_hp_op& op = ch.ops[i].op;
    if (op.kind == MS_HP_GEMM_SWIGLU)  // SwiGLU epilogue needs whole k: split 1
      gemms.push_back({i - first, static_cast<int>(op.m / kBM) * static_cast<int>(2 * op.n / kFusedBN),
                       static_cast<int>(op.k / kBK), 1});
    if (op.kind != MS_HP_GEMM) continue;
    gemms.push_back({i - first, static_cast<int>(op.m / kBM) * static_cast<int>(op.n / bn),
                     static_cast<int>(op.k / kBK), bn == kFusedBN ? op.split_k : 1});
  }
  std::vector<int> splits(prog.n_ops, 1);
  int cs = 1, max_units = 0;
  // (1) Cluster split-K (k-slices reduced through DSMEM): each GEMM op gets split CS when its
  // tiles x CS fit one unit per CTA (else split 1, tiles spread over the grid); all CTAs
  // must be co-resident as clusters (the grid phases need co-residency).
  for (int c : {4, 2}) {
    if (d->hp_fused == 2 || gemms.empty() || bn != kFusedBN) break;
    std::vector<int> sp(prog.n_ops, 1);
    int mu = 0, n_split = 0;
    bool ok = true;
    for (const GemmShape& g : gemms) {
      int split = 1;
      if (g.req > 0) {
        if (g.req != 1 && g.req != c) ok = false;
        split = g.req;
      } else if (g.tiles * c <= max_grid && g.kbs % c == 0 && g.kbs / c >= 2) {
        split = c;
      }
      if (split > 1 && g.kbs % split) ok = false;
      sp[g.idx] = split;
      n_split += split > 1;
      mu = std::max(mu, g.tiles * split);
    }
    if (!ok || n_split == 0) continue;
    const int grid_c = std::min(mu, max_grid) / c * c;
    for (const GemmShape& g : gemms)
      if (sp[g.idx] > 1 && g.tiles * sp[g.idx] > grid_c) ok = false;
    if (!ok || grid_c < c) continue;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid_c);
    cfg.blockDim = dim3(256);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int max_clusters = 0;
    cudaError_t e;
    if (c == 2) {
      cfg.dynamicSmemBytes = FusedCfg<2>::kSmemBytes;
      e = cudaOccupancyMaxActiveClusters(&max_clusters, hp_fused_kernel<2>, &cfg);
    } else {
      cfg.dynamicSmemBytes = FusedCfg<4>::kSmemBytes;
      e = cudaOccupancyMaxActiveClusters(&max_clusters, hp_fused_kernel<4>, &cfg);
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (max_clusters * c < grid_c) continue;
    // Only worth it when no GEMM op loses parallelism against the no-cluster plan (k-slices
    // doubled while the units fit the SMs): e.g. a [128 x 2048] x [2048 x 8192]^T op keeps
    // 128 units with 8 global k-slices but only 32 with cluster pairs.
    bool keeps = true;
    for (const GemmShape& g : gemms) {
      int gs = g.req > 0 ? g.req : 1;
      if (g.req <= 0)
        while (g.tiles * gs * 2 <= sms && g.kbs % (gs * 2) == 0 && g.kbs / (gs * 2) >= 4) gs *= 2;
      const int u_global = std::min(g.tiles * gs, max_grid), u_cluster = std::min(g.tiles * sp[g.idx], grid_c);
      if (10 * u_cluster < 9 * u_global) keeps = false;
    }
    if (!keeps) continue;
    cs = c;
    splits = sp;
    max_units = grid_c;  // grid of the cluster launch
    break;
  }
  // (2) No clusters: k-slices reduced through global partials + a grid phase; split doubles
  // while the units still fit the SMs.
  if (cs == 1)
    for (const GemmShape& g : gemms) {
      int split = g.req > 0 ? g.req : 1;
      if (g.req <= 0)
        while (g.tiles * split * 2 <= sms && g.kbs % (split * 2) == 0 && g.kbs / (split * 2) >= 4) split *= 2;
      splits[g.idx] = split;
      max_units = std::max(max_units, g.tiles * split);
    }
  const bool any_gemm = !gemms.empty();
  const bool absorb_gelu = !getenv("MS_FUSED_NO_EPI_GELU");
  int np = 0, grid = std::min(std::max(max_units, 1), max_grid);
  for (int i = first; i <= last; ++i) {
    const HpOpRt& o = ch.ops[i];
    FusedOp& f = prog.ops[i - first];
    f.d.m = static_cast<int>(o.op.m);
    f.d.n = static_cast<int>(o.op.n);
    f.d.k = static_cast<int>(o.op.k);
    f.d.c = reinterpret_cast<__nv_bfloat16*>(o.op.c);
    f.d.in_phase = i > first ? prog.ops[i - first - 1].d.ready_phase : -1;
    if (o.op.kind == MS_HP_GEMM || o.op.kind == MS_HP_GEMM_SWIGLU) {
      f.d.kind = kFusedGemm;
      f.d.swiglu = o.op.kind == MS_HP_GEMM_SWIGLU;
      f.d.tiles_m = f.d.m / kBM;
      f.d.tiles_n = (f.d.swiglu ? 2 * f.d.n : f.d.n) / bn;
      const int split = splits[i - first];
      f.d.split = split;
      f.d.kb_per_unit = f.d.k / kBK / split;
      f.d.units = f.d.tiles_m * f.d.tiles_n * split;
      if (int rc = encode_2d(&f.tma_a, reinterpret_cast<void*>(o.op.a), o.op.m, o.op.k, kBM, o.op.lda)) return rc;
      if (o.b_tiled || o.op.b_layout == 2) {
        f.d.b_kmajor = 1;
        const void* wb = o.b_tiled ? static_cast<const void*>(o.b_tiled) : reinterpret_cast<const void*>(o.op.b);
        const uint64_t bn_rows = f.d.swiglu ? 2 * o.op.n : o.op.n;
        if (int rc = encode_kblock_major(&f.tma_b, wb, bn_rows, o.op.k, bn)) return rc;
      } else {
        if (int rc = encode_2d(&f.tma_b, reinterpret_cast<void*>(o.op.b), o.op.n, o.op.k, bn)) return rc;
      }
      if (cs > 1 && split > 1) {  // slices reduced inside the cluster: one phase (output ready)
        f.d.mma_phase = -1;
        f.d.ready_phase = np++;
      } else {
        if (split > 1) {
          MS_CUDA(cudaMalloc(&f.d.ws, sizeof(float) * static_cast<size_t>(split) * f.d.m * f.d.n));
          ch.fused_ws.push_back(f.d.ws);
        }
        f.d.mma_phase = np++;
        f.d.ready_phase = split > 1 ? np++ : f.d.mma_phase;
      }
    } else if (i > first && o.op.kind == MS_HP_BIAS_GELU && absorb_gelu && cs > 1 &&
               prog.ops[i - first - 1].d.kind == kFusedGemm && prog.ops[i - first - 1].d.mma_phase < 0 &&
               !prog.ops[i - first - 1].d.swiglu && bn == kFusedBN &&
               reinterpret_cast<uint64_t>(prog.ops[i - first - 1].d.c) == o.op.a &&
               prog.ops[i - first - 1].d.m == f.d.m && prog.ops[i - first - 1].d.n == f.d.n) {
      // gelu(C + bias) straight after a cluster-reduced GEMM on its own output: computed in
      // that GEMM's epilogue from the same bf16-rounded C (bit-identical to the phase), so
      // the chain saves a grid phase and a 2-pass sweep over C.
      FusedOpDesc& g = prog.ops[i - first - 1].d;
      g.gelu_c = f.d.c;
      g.gelu_bias = reinterpret_cast<const __nv_bfloat16*>(o.op.bias);
      f.d.kind = kFusedAbsorbed;
      f.d.mma_phase = -1;
      f.d.ready_phase = g.ready_phase;
    } else {
      f.d.kind = o.op.kind == MS_HP_SILU_MUL ? kFusedSiluMul : kFusedBiasGelu;
      f.d.x = reinterpret_cast<const __nv_bfloat16*>(o.op.a);
      f.d.bias = reinterpret_cast<const __nv_bfloat16*>(o.op.bias);
      f.d.mma_phase = -1;
      f.d.ready_phase = np++;
      if (!any_gemm) {
        const long long chunks = o.op.m * o.op.n / 8;
        grid = std::max<int>(grid, static_cast<int>(std::min<long long>((chunks + 127) / 128, max_grid)));
      }
    }
  }
  if (cs > 1) grid = max_units;  // a multiple of the cluster size
  ch.fused_cs = cs;
  ch.fused_bn = bn;
  prog.n_phases = np;
  // L2 prefetch of the next op's weights: measured +2% on cluster launches (config-1 chain
  // 59.7 vs 60.9 us) but -11% on long non-cluster chains (config-4 step 1.03 vs 0.92 ms: the
  // prefetch backlog delays the grid phases' own loads and fences).
  prog.l2_prefetch = cs > 1 && !getenv("MS_FUSED_NO_PREFETCH");
  MS_CUDA(cudaMalloc(&ch.prog_d, sizeof(FusedProgram)));
  MS_CUDA(cudaMemcpy(ch.prog_d, &prog, sizeof(FusedProgram), cudaMemcpyHostToDevice));
  MS_CUDA(cudaMalloc(&ch.phase_d, sizeof(uint32_t) * std::max(np, 1)));
  MS_CUDA(cudaMemset(ch.phase_d, 0, sizeof(uint32_t) * std::max(np, 1)));
  ch.fused_ctl = d->next_hp_ctl++;
  if (ch.fused_ctl >= MS_N_CTL) return fail(MS_E_ARG, "out of HP control blocks");
  ch.descs.clear();
  for (int i = 0; i < prog.n_ops; ++i) ch.descs.push_back(prog.ops[i].d);
  ch.l2_prefetch = prog.l2_prefetch;
  ch.fused_first = first;
  ch.fused_last = last;
  ch.fused_grid = grid;
  ch.n_phases = np;
  ch.fusable = true;
  return 0;
}

// Plan of a batch-1 chain (hp_gemv.cuh): per op, the unit size (whole rows, <= one 16 KB
// stage) and the chain-wide unit counter at its first unit, so units are dealt to CTAs
// round-robin across op boundaries.  Grid = SMs - 1 (same co-residency rule as plan_fused).
int plan_gemv(ms_dev* d, HpChain& ch) {
  int first = -1, last = -1;
  for (int i = 0; i < static_cast<int>(ch.ops.size()); ++i)
    if (!is_copy(ch.ops[i].op)) {
      if (first < 0) first = i;
      last = i;
    }
  for (int i = first; i <= last; ++i)
    if (is_copy(ch.ops[i].op)) return fail(MS_E_ARG, "batch-1 chains: copies only before/after the kernel ops");
  if (last - first + 1 > kGemvMaxOps) return fail(MS_E_ARG, "batch-1 chain too long");
  ch.gemv_descs.clear();
  // Grid: SMs - 1 (one SM stays free for the doorbell gate), or MS_GEMV_GRID (A/B: a smaller
  // chain starts once that many SMs are free instead of waiting for the last LP CTA to drain)
  const int grid = [&] {
    const char* e = getenv("MS_GEMV_GRID");
    const int g = e ? atoi(e) : 0;
    return g > 0 && g < d->prop.multiProcessorCount ? g : d->prop.multiProcessorCount - 1;
  }();
  int64_t unit_ctr = 0;
  for (int i = first; i <= last; ++i) {
    const ms_hp_op& op = ch.ops[i].op;
    GemvOpDesc g{};
    g.n = static_cast<int>(op.n);
    g.k = static_cast<int>(op.k);
    g.x = reinterpret_cast<const __nv_bfloat16*>(op.a);
    g.w = reinterpret_cast<const __nv_bfloat16*>(op.b);
    g.bias = reinterpret_cast<const __nv_bfloat16*>(op.bias);
    g.y = reinterpret_cast<__nv_bfloat16*>(op.c);
    if (op.kind == MS_HP_GEMM || op.kind == MS_HP_GEMM_SWIGLU) {
      const bool sw = op.kind == MS_HP_GEMM_SWIGLU;
      g.kind = sw ? kGemvSwiglu : kGemvMatvec;
      g.rows = std::min(32, kGemvStageBytes / (static_cast<int>(op.k) * 2 * (sw ? 2 : 1)));  // <= one output per lane
      g.units = (g.n + g.rows - 1) / g.rows;
      g.unit_base = static_cast<int>(unit_ctr % grid);
      unit_ctr += g.units;
    } else {
      g.kind = op.kind == MS_HP_SILU_MUL ? kGemvSiluMul : kGemvBiasGelu;
      g.k = 0;
    }
    ch.gemv_descs.push_back(g);
  }
  // Wires: op j whose input lies inside the output of the latest earlier op i reads it
  // from op i's tagged wire (no grid phase); any other input orders op j behind op j-1's
  // phase counter.  Wire offsets are 4-word aligned (16-byte vector polls).
  const int n = static_cast<int>(ch.gemv_descs.size());
  std::vector<int64_t> wire_off(n, -1);
  std::vector<std::pair<int, int64_t>> src(n, {-1, 0});  // (producer op, word offset in its output)
  int64_t words = 0;
  for (int j = 1; j < n; ++j) {
    GemvOpDesc& g = ch.gemv_descs[j];
    const uint64_t a = reinterpret_cast<uint64_t>(g.x);
    const uint64_t in_bytes = 2ull * (g.kind == kGemvMatvec || g.kind == kGemvSwiglu ? g.k
                                      : g.kind == kGemvSiluMul ? 2 * g.n : g.n);
    for (int i = j - 1; i >= 0; --i) {
      const uint64_t c = reinterpret_cast<uint64_t>(ch.gemv_descs[i].y);
      const uint64_t c_bytes = 2ull * ch.gemv_descs[i].n;
      if (a + in_bytes <= c || a >= c + c_bytes) continue;  // no overlap: look further back
      if (a >= c && a + in_bytes <= c + c_bytes && (a - c) % 8 == 0) src[j] = {i, static_cast<int64_t>((a - c) / 2)};
      break;  // latest producer overlapping the input decides
    }
    if (src[j].first >= 0 && wire_off[src[j].first] < 0) {
      wire_off[src[j].first] = words;
      words += (ch.gemv_descs[src[j].first].n + 3) / 4 * 4;
    }
  }
  if (words > 0) {
    MS_CUDA(cudaMalloc(&ch.wire_d, sizeof(uint32_t) * words));
    MS_CUDA(cudaMemset(ch.wire_d, 0, sizeof(uint32_t) * words));
  }
  for (int i = 0; i < n; ++i)
    if (wire_off[i] >= 0) ch.gemv_descs[i].y_wire = ch.wire_d + wire_off[i];
  for (int j = 1; j < n; ++j) {
    GemvOpDesc& g = ch.gemv_descs[j];
    if (src[j].first >= 0) {
      g.x_wire = ch.gemv_descs[src[j].first].y_wire + src[j].second;
    } else {
      g.wait_phase = 1;
      ch.gemv_descs[j - 1].arrive = 1;
    }
  }
  MS_CUDA(cudaMalloc(&ch.gemv_descs_d, sizeof(GemvOpDesc) * n));
  MS_CUDA(cudaMemcpy(ch.gemv_descs_d, ch.gemv_descs.data(), sizeof(GemvOpDesc) * n, cudaMemcpyHostToDevice));
  const int np = n;
  // [0, n): grid phase counters; [n, 2n): dynamic unit-claim counters (both reset by the
  // last CTA of each launch)
  // [2n]: CTAs started (head prefetch)
  MS_CUDA(cudaMalloc(&ch.phase_d, sizeof(uint32_t) * (2 * np + 1)));
  MS_CUDA(cudaMemset(ch.phase_d, 0, sizeof(uint32_t) * (2 * np + 1)));
  ch.fused_ctl = d->next_hp_ctl++;
  if (ch.fused_ctl >= MS_N_CTL) return fail(MS_E_ARG, "out of HP control blocks");
  ch.fused_first = first;
  ch.fused_last = last;
  ch.fused_grid = grid;
  ch.fused_cs = 1;
  ch.n_phases = 2 * np + 1;
  ch.gemv = true;
  ch.fusable = true;
  return 0;
}

int launch_gemv(ms_dev* d, int chain_id, const HpChain& ch, uint32_t seq, bool pdl, bool after_pull = false) {
  GemvParams p{};
  p.run = base_run(d, ch.fused_ctl);
  p.run.hp_ctl = d->hp_ctl + chain_id;
  p.run.slot = chain_id;
  p.run.hp_rec = &d->page_d->hp[chain_id];
  p.run.hp_first = after_pull ? 0 : 1;
  p.run.pdl_wait = after_pull ? 1 : 0;
  p.run.hp_last = !is_copy(ch.ops.back().op);
  p.run.hp_seq = seq;
  p.run.dbg = d->dbg;
  p.run.reset_words = ch.phase_d;
  p.run.n_reset = ch.n_phases;
  p.phase_cnt = ch.phase_d;
  p.claim = ch.phase_d + ch.gemv_descs.size();
  const bool dynamic = [] {
    const char* e = getenv("MS_GEMV_DYNAMIC");  // 1: units claimed per op (hp_gemv_kernel<true>)
    return e ? atoi(e) != 0 : kGemvDynamicDefault;
  }();
  p.claim_batch = [] {
    const char* e = getenv("MS_GEMV_CLAIM_BATCH");
    return e ? std::max(1, atoi(e)) : 4;
  }();
  p.n_ops = static_cast<int>(ch.gemv_descs.size());
  p.ops = ch.gemv_descs_d;
  p.tag = (++ch.launches) & 0xFFFFu;
  static const int inflight = [] {
    const char* e = getenv("MS_GEMV_INFLIGHT");
    const int v = e ? atoi(e) : kGemvStages;
    return v < 1 ? 1 : v > kGemvStages ? kGemvStages : v;
  }();
  p.inflight = inflight;
  static const int prefetch = [] {
    const char* e = getenv("MS_GEMV_PREFETCH");
    return e ? std::max(0, atoi(e)) : 16;
  }();
  p.prefetch = prefetch;
  static const int head_kb = [] {
    const char* e = getenv("MS_GEMV_HEAD_KB");  // 0: no head prefetch
    return e ? std::max(0, atoi(e)) : kGemvHeadKbDefault;
  }();
  p.head_kb = head_kb;
  p.start_cnt = ch.phase_d + 2 * ch.gemv_descs.size();
  if (dynamic)
    MS_CUDA(launch_kc(hp_gemv_kernel<true>, ch.fused_grid, kGemvThreads, kGemvSmemBytes, d->hp, pdl, 1, p));
  else
    MS_CUDA(launch_kc(hp_gemv_kernel<false>, ch.fused_grid, kGemvThreads, kGemvSmemBytes, d->hp, pdl, 1, p));
  return 0;
}

int launch_fused(ms_dev* d, int chain_id, const HpChain& ch, uint32_t seq, bool pdl, bool after_pull = false) {
  FusedParams p{};
  p.run = base_run(d, ch.fused_ctl);
  p.run.hp_ctl = d->hp_ctl + chain_id;
  p.run.slot = chain_id;
  p.run.hp_rec = &d->page_d->hp[chain_id];
  p.run.hp_first = after_pull ? 0 : 1;
  p.run.pdl_wait = after_pull ? 1 : 0;
  p.run.hp_last = !is_copy(ch.ops.back().op);
  p.run.hp_seq = seq;
  p.run.dbg = d->dbg;
  p.run.reset_words = ch.phase_d;
  p.run.n_reset = ch.n_phases;
  p.prog = ch.prog_d;
  p.phase_cnt = ch.phase_d;
  p.n_ops = static_cast<int>(ch.descs.size());
  p.l2_prefetch = ch.l2_prefetch;
  static const int full_fence = [] {
    const char* e = getenv("MS_FUSED_FULL_FENCE");
    return e ? atoi(e) : 0;  // the release reduction suffices: 58 vs 60 us per config-1 chain
  }();
  p.full_fence = full_fence;
  for (size_t i = 0; i < ch.descs.size(); ++i) p.ops[i] = ch.descs[i];
  if (ch.fused_bn == 32) {
    MS_CUDA(launch_kc(hp_fused_kernel<1, 32>, ch.fused_grid, 256, FusedCfg<1, 32>::kSmemBytes, d->hp, pdl, 1, p));
    return 0;
  }
  switch (ch.fused_cs) {
    case 4:
      MS_CUDA(launch_kc(hp_fused_kernel<4>, ch.fused_grid, 256, FusedCfg<4>::kSmemBytes, d->hp, pdl, 4, p));
      break;
    case 2:
      MS_CUDA(launch_kc(hp_fused_kernel<2>, ch.fused_grid, 256, FusedCfg<2>::kSmemBytes, d->hp, pdl, 2, p));
      break;
    default:
      MS_CUDA(launch_kc(hp_fused_kernel<1>, ch.fused_grid, 256, FusedCfg<1>::kSmemBytes, d->hp, pdl, 1, p));
  }
  return 0;
}

// Enqueue a chain's work on the HP stream (after its gate when `after_gate`).
// `after_pull`: the kernel before op first_op is the e2e input pull (hp_pull_kernel).
int launch_chain(ms_dev* d, int cid, const HpChain& ch, uint32_t seq, bool after_gate, size_t first_op = 0,
                 bool after_pull = false) {
  // batch-1 chains have no per-op kernels: the GEMV chain is their only implementation
  const bool fused = (d->hp_fused && ch.fusable) || ch.gemv;
  for (size_t i = first_op; i < ch.ops.size(); ++i) {
    const bool pulled = after_pull && i == first_op;
    if (fused && static_cast<int>(i) >= ch.fused_first && static_cast<int>(i) <= ch.fused_last) {
      if (static_cast<int>(i) == ch.fused_first) {
        const bool pdl = (after_gate && i == 0) || pulled;
        if (int rc = ch.gemv ? launch_gemv(d, cid, ch, seq, pdl, pulled) : launch_fused(d, cid, ch, seq, pdl, pulled))
          return rc;
      }
      continue;
    }
    if (int rc = launch_hp_op(d, cid, ch, i, seq, after_gate, pulled)) return rc;
  }
  return 0;
}

}  // namespace

extern "C" {

const char* ms_last_error(void) { return g_err.c_str(); }
int ms_internal_fail(int code, const char* what) { return fail(code, what ? what : ""); }
// Memory tier: wait for LP work only (an armed HP gate keeps the HP stream busy until rung).
int ms_internal_lp_sync(ms_dev* d) {
  MS_CUDA(cudaStreamSynchronize(d->lp));
  return 0;
}
int64_t ms_host_now_ns(void) { return now_ns(); }

int ms_dev_open(int ordinal, ms_dev** out) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= ordinal) return fail(MS_E_NODEV, "no CUDA device");
  auto* d = new ms_dev();
  d->ordinal = ordinal;
  if (const char* e = getenv("MS_LP_SM_RESERVE")) d->lp_sm_reserve = std::max(0, atoi(e));  // A/B knob
  MS_CUDA(cudaSetDevice(ordinal));
  MS_CUDA(cudaGetDeviceProperties(&d->prop, ordinal));
  if (d->prop.major != 10) {
    delete d;
    return fail(MS_E_NODEV, "ms_b200 requires an sm_100 (B200) device");
  }
  MS_CUDA(cudaDeviceGetStreamPriorityRange(&d->prio_low, &d->prio_high));
  MS_CUDA(cudaStreamCreateWithPriority(&d->lp, cudaStreamNonBlocking, d->prio_low));
  MS_CUDA(cudaStreamCreateWithPriority(&d->hp, cudaStreamNonBlocking, d->prio_high));
  MS_CUDA(cudaStreamCreateWithPriority(&d->aux, cudaStreamNonBlocking, d->prio_low));
  MS_CUDA(cudaStreamCreateWithPriority(&d->hpcopy, cudaStreamNonBlocking, d->prio_high));
  MS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&d->page), sizeof(MsHostPage),
                        cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(d->page, 0, sizeof(MsHostPage));
  MS_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d->page_d), d->page, 0));
  MS_CUDA(cudaMalloc(&d->mirror, sizeof(MsDevMirror)));
  MS_CUDA(cudaMemset(d->mirror, 0, sizeof(MsDevMirror)));
  const int n_ctl = MS_N_CTL;
  MS_CUDA(cudaMalloc(&d->ctl, sizeof(MsLpCtl) * n_ctl));
  MS_CUDA(cudaMalloc(&d->hp_ctl, sizeof(MsHpCtl) * MS_MAX_HP_CHAINS));
  MS_CUDA(cudaMemset(d->hp_ctl, 0, sizeof(MsHpCtl) * MS_MAX_HP_CHAINS));
  MS_CUDA(cudaMalloc(&d->dummy_redo, 64 * sizeof(unsigned long long)));
  init_ctl_kernel<<<(n_ctl + 127) / 128, 128>>>(d->ctl, n_ctl, d->hp_ctl, MS_MAX_HP_CHAINS);
  MS_CUDA(cudaGetLastError());
  MS_CUDA(cudaDeviceSynchronize());
  if (int rc = set_smem_attrs()) return rc;
  int attr = 0;
  cudaDeviceGetAttribute(&attr, static_cast<cudaDeviceAttr>(CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_MEM_OPS_V1), ordinal);
  d->stream_memops = attr;
  *out = d;
  return 0;
}

int ms_dev_close(ms_dev* d) {
  if (!d) return 0;
  cudaSetDevice(d->ordinal);
  cudaDeviceSynchronize();
  for (auto& s : d->lp_slots)
    for (auto* r : s.redo)
      if (r) cudaFree(r);
  cudaFree(d->mirror);
  cudaFree(d->ctl);
  cudaFree(d->hp_ctl);
  cudaFree(d->dummy_redo);
  cudaFreeHost(d->page);
  if (d->trace_ev) cudaFreeHost(d->trace_ev);
  if (d->trace_head) cudaFree(d->trace_head);
  if (d->trace_dev) cudaFree(d->trace_dev);
  cudaStreamDestroy(d->lp);
  cudaStreamDestroy(d->hp);
  cudaStreamDestroy(d->aux);
  cudaStreamDestroy(d->hpcopy);
  delete d;
  return 0;
}

int ms_dev_get_info(ms_dev* d, ms_dev_info* info) {
  std::memset(info, 0, sizeof(*info));
  info->ordinal = d->ordinal;
  info->sm_count = d->prop.multiProcessorCount;
  info->cc_major = d->prop.major;
  info->cc_minor = d->prop.minor;
  info->stream_memops = d->stream_memops;
  info->prio_low = d->prio_low;
  info->prio_high = d->prio_high;
  info->hbm_bytes = static_cast<int64_t>(d->prop.totalGlobalMem);
  std::snprintf(info->name, sizeof info->name, "%s", d->prop.name);
  return 0;
}

int ms_dev_sync(ms_dev* d) {
  MS_CUDA(cudaSetDevice(d->ordinal));
  MS_CUDA(cudaDeviceSynchronize());
  return 0;
}

int ms_host_alloc(ms_dev* d, size_t bytes, uint64_t* p) {
  MS_CUDA(cudaSetDevice(d->ordinal));
  void* ptr = nullptr;
  MS_CUDA(cudaHostAlloc(&ptr, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  *p = reinterpret_cast<uint64_t>(ptr);
  return 0;
}
int ms_host_free(ms_dev*, uint64_t p) {
  MS_CUDA(cudaFreeHost(reinterpret_cast<void*>(p)));
  return 0;
}

int ms_mem_alloc(ms_dev* d, size_t bytes, uint64_t* p) {
  MS_CUDA(cudaSetDevice(d->ordinal));
  void* ptr = nullptr;
  MS_CUDA(cudaMalloc(&ptr, bytes));
  *p = reinterpret_cast<uint64_t>(ptr);
  return 0;
}
int ms_mem_free(ms_dev*, uint64_t p) {
  MS_CUDA(cudaFree(reinterpret_cast<void*>(p)));
  return 0;
}
int ms_memcpy_h2d(ms_dev* d, uint64_t dst, const void* src, size_t bytes) {
  MS_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(dst), src, bytes, cudaMemcpyHostToDevice, d->aux));
  MS_CUDA(cudaStreamSynchronize(d->aux));
  return 0;
}
int ms_memcpy_d2h(ms_dev* d, void* dst, uint64_t src, size_t bytes) {
  MS_CUDA(cudaMemcpyAsync(dst, reinterpret_cast<const void*>(src), bytes, cudaMemcpyDeviceToHost, d->aux));
  MS_CUDA(cudaStreamSynchronize(d->aux));
  return 0;
}
int ms_memset(ms_dev* d, uint64_t dst, int value, size_t bytes) {
  MS_CUDA(cudaMemsetAsync(reinterpret_cast<void*>(dst), value, bytes, d->aux));
  MS_CUDA(cudaStreamSynchronize(d->aux));
  return 0;
}
int ms_fill_synth_f32(ms_dev* d, uint64_t dst, uint64_t n, uint64_t seed, uint64_t tensor, float scale) {
  synth_fill_f32_kernel<<<d->prop.multiProcessorCount * 8, 256, 0, d->aux>>>(reinterpret_cast<float*>(dst), n, seed,
                                                                             tensor, scale);
  MS_CUDA(cudaGetLastError());
  MS_CUDA(cudaStreamSynchronize(d->aux));
  return 0;
}
int ms_fill_synth_bf16(ms_dev* d, uint64_t dst, uint64_t n, uint64_t seed, uint64_t tensor, float scale) {
  synth_fill_kernel<<<d->prop.multiProcessorCount * 8, 256, 0, d->aux>>>(reinterpret_cast<__nv_bfloat16*>(dst), n,
                                                                         seed, tensor, scale);
  MS_CUDA(cudaGetLastError());
  MS_CUDA(cudaStreamSynchronize(d->aux));
  return 0;
}

// ------------------------------------------------------------------ LP kernels
int ms_lp_register(ms_dev* d, const ms_lp_desc* desc, int* id, uint64_t* total_tiles) {
  int slot = -1;
  for (int i = 0; i < MS_MAX_LP; ++i)
    if (!d->lp_slots[i].used) {
      slot = i;
      break;
    }
  if (slot < 0) return fail(MS_E_ARG, "too many LP kernels");
  LpSlot& s = d->lp_slots[slot];
  const uint64_t keep_run_id = s.run_id;
  s = LpSlot{};
  s.run_id = keep_run_id;
  s.desc = *desc;
  if (desc->kind == MS_LP_GEMM) {
    const int bn = desc->block_n ? desc->block_n : 256;
    s.desc.block_n = bn;
    if (bn != 64 && bn != 128 && bn != 256) return fail(MS_E_ARG, "block_n must be 64/128/256");
    if (desc->m % kBM || desc->n % bn || desc->k % kBK || desc->k < kBK)
      return fail(MS_E_ARG, "GEMM shape must be a multiple of (128, block_n, 64)");
    if (desc->m > (1ll << 31) || desc->n > (1ll << 31) || desc->k > (1ll << 31)) return fail(MS_E_ARG, "shape too large");
    // Large GEMMs run on CTA pairs (cta_group::2, tc_gemm2.cuh) with 256 x 512 tiles: 8192^3
    // at 1463-1477 TFLOP/s burst on the 73 pairs left beside the gate's TPC (1574-1585 on 74
    // pairs) vs 1331-1346 for the single-CTA 128 x 256 kernel and 1610-1612 for cuBLAS on the
    // same box (tools/gemm_ab2.py, profiles/r02_gemm_ab.json).
    // Chosen when the shape has >= 4 waves of pair tiles (fewer tiles lose more to the last
    // wave than the pair saves) and no k-split.  MS_LP_GEMM_PAIR=0 forces the single-CTA
    // kernel, =1 pairs with 256 x 256 tiles, =2 pairs with 256 x 512 tiles.
    const char* pe = getenv("MS_LP_GEMM_PAIR");
    int pair_mode = pe ? atoi(pe) : -1;
    if (pair_mode < 0) {
      const int64_t pair_tiles = desc->n % 512 == 0 ? (desc->m / 256) * (desc->n / 512) : 0;
      pair_mode = (desc->split_k <= 1 && pair_tiles >= 4 * (d->prop.multiProcessorCount / 2)) ? 2 : 0;
    }
    s.pair_tn = pair_mode == 2 && desc->n % 512 == 0 ? 512 : 256;
    s.pair = bn == 256 && desc->m % 256 == 0 && desc->n % s.pair_tn == 0 && pair_mode != 0 && desc->split_k <= 1;
    const int tm = s.pair ? 256 : kBM;
    s.tiles_m = static_cast<int>(desc->m / tm);
    s.tiles_n = static_cast<int>(desc->n / (s.pair ? s.pair_tn : bn));
    s.split = desc->split_k > 1 ? desc->split_k : 1;
    if (s.split > 1) {
      if (s.pair) return fail(MS_E_ARG, "split_k is not supported on CTA pairs");
      if ((desc->k / kBK) % s.split) return fail(MS_E_ARG, "split_k must divide K / 64");
      const size_t tiles = static_cast<size_t>(s.tiles_m) * s.tiles_n;
      MS_CUDA(cudaMalloc(&s.ws, sizeof(float) * tiles * s.split * kBM * bn));
      // reduction-tree group counters: <= split per tile (tc_gemm.cuh split_tree_reduce)
      MS_CUDA(cudaMalloc(&s.tile_cnt, sizeof(unsigned int) * tiles * s.split));
      MS_CUDA(cudaMemset(s.tile_cnt, 0, sizeof(unsigned int) * tiles * s.split));
    }
    s.total_tiles = static_cast<uint64_t>(s.tiles_m) * s.tiles_n * s.split;
    // Wave tail (pairs, 256 x 512 tiles): 512 tiles of 8192^3 on the 73 pairs left beside the
    // gate's TPC are 7 waves + 1 tile, and that tile alone takes ~0.7 of a wave (71 of 802 us,
    // profiles/r02s3_gemm_wave_probe.json) while every other pair idles.  When the last wave
    // is at most half (a quarter) full, its tiles run as 256-column halves (128-column
    // quarters) on twice (four times) the pairs: units half_base.., tc_gemm2.cuh pair_unit.
    // Measured (profiles/r02s3_gemm_wave_probe_quarters.json, one box): 7 waves 705 us, whole
    // tail tile +44 us, halves +23 us, quarters +23 us — a lone part unit is bound by its ring's
    // load latency (4 stages in flight: ~0.18 us per k-block whatever the unit's width), so
    // quarters only spend twice the pairs; halves are the default, MS_LP_PAIR_TAIL_PARTS=4
    // selects quarters (parity-tested), MS_LP_PAIR_HALF_TAIL=0 disables the split.
    s.half_base = 0;
    s.half_units = 0;
    s.tail_parts = 2;
    if (s.pair && s.pair_tn == 512) {
      const char* e = getenv("MS_LP_PAIR_HALF_TAIL");
      const char* ep = getenv("MS_LP_PAIR_TAIL_PARTS");
      const uint64_t max_parts = ep ? static_cast<uint64_t>(std::max(2, std::min(4, atoi(ep)))) : 2;
      const int pairs = (d->prop.multiProcessorCount - ((d->lp_sm_reserve + 1) & ~1)) / 2;
      const uint64_t tiles = s.total_tiles;
      const uint64_t tail = pairs > 0 ? tiles % static_cast<uint64_t>(pairs) : 0;
      if (!(e && atoi(e) == 0) && pairs > 0 && tiles >= static_cast<uint64_t>(pairs) && tail > 0 &&
          2 * tail <= static_cast<uint64_t>(pairs)) {
        const uint64_t parts = (max_parts >= 4 && 4 * tail <= static_cast<uint64_t>(pairs)) ? 4 : 2;
        s.tail_parts = static_cast<int>(parts);
        s.half_base = static_cast<long long>(tiles - tail);
        s.half_units = static_cast<int>(parts * tail);
        s.total_tiles = tiles - tail + parts * tail;
      }
    }
    if (int rc = encode_2d(&s.tma_a, reinterpret_cast<void*>(desc->a), desc->m, desc->k, kBM)) return rc;
    if (int rc = encode_2d(&s.tma_b, reinterpret_cast<void*>(desc->b), desc->n, desc->k, s.pair ? 128 : bn)) return rc;
    if (s.pair)
      if (int rc = encode_2d(&s.tma_bq, reinterpret_cast<void*>(desc->b), desc->n, desc->k, 64)) return rc;
    if (int rc = encode_c(&s.tma_c, reinterpret_cast<void*>(desc->c), desc->m, desc->n)) return rc;
  } else if (desc->kind == MS_LP_AXPY) {
    s.desc.tile_elems = desc->tile_elems ? desc->tile_elems : 8192;
    s.desc.ctas_per_sm = desc->ctas_per_sm ? desc->ctas_per_sm : 1;  // default: grouped, one CTA per SM
    if (s.desc.tile_elems % (kStreamThreads * 8) || s.desc.tile_elems > kStreamThreads * 8 * 8)
      return fail(MS_E_ARG, "tile_elems must be a multiple of 2048 and <= 16384");
    if (desc->n_elems % 8) return fail(MS_E_ARG, "n_elems must be a multiple of 8");
    s.total_tiles = (static_cast<uint64_t>(desc->n_elems) + s.desc.tile_elems - 1) / s.desc.tile_elems;
  } else if (desc->kind == MS_LP_OPTIM) {
    s.desc.tile_elems = desc->tile_elems ? desc->tile_elems : 4096;
    if (s.desc.tile_elems % (kStreamThreads * 4) || s.desc.tile_elems > kStreamThreads * 4 * 8)
      return fail(MS_E_ARG, "optimizer tile_elems must be a multiple of 1024 and <= 8192");
    if (desc->n_elems % 4 || desc->n_elems <= 0) return fail(MS_E_ARG, "n_elems must be a positive multiple of 4");
    if (desc->opt_mode != 0 && desc->opt_mode != 1) return fail(MS_E_ARG, "opt_mode must be 0 (AdamW) or 1 (SGD)");
    if (!desc->a || !desc->b || !desc->x || (desc->opt_mode == 0 && !desc->c)) return fail(MS_E_ARG, "optimizer buffers");
    if ((desc->a | desc->b | desc->c) % 16 || desc->x % 8) return fail(MS_E_ARG, "optimizer buffers must be aligned");
    s.total_tiles = (static_cast<uint64_t>(desc->n_elems) + s.desc.tile_elems - 1) / s.desc.tile_elems;
  } else {
    return fail(MS_E_ARG, "unknown LP kernel kind");
  }
  for (auto*& r : s.redo) MS_CUDA(cudaMalloc(&r, kRedoCap * sizeof(unsigned long long)));
  s.used = true;
  *id = slot;
  *total_tiles = s.total_tiles;
  return 0;
}

int ms_lp_unregister(ms_dev* d, int id) {
  if (id < 0 || id >= MS_MAX_LP || !d->lp_slots[id].used) return fail(MS_E_ARG, "bad LP id");
  MS_CUDA(cudaStreamSynchronize(d->lp));
  LpSlot& s = d->lp_slots[id];
  for (auto*& r : s.redo) {
    if (r) cudaFree(r);
    r = nullptr;
  }
  if (s.slow) cudaFree(s.slow);
  if (s.slow_sem) cudaFree(s.slow_sem);
  if (s.ws) cudaFree(s.ws);
  if (s.tile_cnt) cudaFree(s.tile_cnt);
  const uint64_t keep_run_id = s.run_id;  // run ids stay monotonic per slot (exit records)
  s = LpSlot{};
  s.run_id = keep_run_id;
  return 0;
}

int ms_lp_set_slow_tiles(ms_dev* d, int id, const uint8_t* slow_groups, uint64_t n_groups, int tiles_per_group,
                         int max_inflight) {
  if (id < 0 || id >= MS_MAX_LP || !d->lp_slots[id].used) return fail(MS_E_ARG, "bad LP id");
  LpSlot& s = d->lp_slots[id];
  if (s.desc.kind != MS_LP_AXPY && s.desc.kind != MS_LP_GEMM)
    return fail(MS_E_ARG, "slow-tile admission: streamer (MS_LP_AXPY) or GEMM kernels");
  MS_CUDA(cudaStreamSynchronize(d->lp));
  if (s.slow) cudaFree(s.slow);
  s.slow = nullptr;
  if (!slow_groups || n_groups == 0) return 0;  // disable
  if (tiles_per_group <= 0 || max_inflight <= 0) return fail(MS_E_ARG, "tiles_per_group and max_inflight must be > 0");
  // (CTA-pair GEMMs: one entry per tile; the half-tile units of the last wave use their tile's)
  const uint64_t map_len = s.half_units ? static_cast<uint64_t>(s.half_base) + s.half_units / s.tail_parts : s.total_tiles;
  if (n_groups * static_cast<uint64_t>(tiles_per_group) < map_len)
    return fail(MS_E_ARG, "slow-tile map does not cover the kernel's tiles");
  MS_CUDA(cudaMalloc(&s.slow, n_groups));
  MS_CUDA(cudaMemcpy(s.slow, slow_groups, n_groups, cudaMemcpyHostToDevice));
  if (!s.slow_sem) {
    MS_CUDA(cudaMalloc(&s.slow_sem, sizeof(unsigned int)));
    MS_CUDA(cudaMemset(s.slow_sem, 0, sizeof(unsigned int)));
  }
  s.slow_group = tiles_per_group;
  s.slow_max = max_inflight;
  return 0;
}

int ms_lp_run(ms_dev* d, int id, uint64_t begin, uint64_t end, uint64_t budget) {
  return ms_lp_run_ex(d, id, begin, end, budget, 0);
}

int ms_lp_run_ex(ms_dev* d, int id, uint64_t begin, uint64_t end, uint64_t budget, int flags) {
  MS_CHECK_LP(d, id);
  LpSlot& s = d->lp_slots[id];
  if (end > s.total_tiles || begin > end) return fail(MS_E_ARG, "tile range out of bounds");
  if (budget > end) budget = end;
  const uint64_t run_id = ++s.run_id;
  const uint64_t nr_in = s.redo_carry;
  TileRun r = base_run(d, id);
  r.begin = begin;
  r.end = end;
  r.budget0 = budget;
  r.nr_in = static_cast<unsigned int>(nr_in);
  r.redo_in = s.redo[(run_id - 1) & 1];
  r.redo_out = s.redo[run_id & 1];
  r.preemptible = (flags & MS_RUN_NONPREEMPTIBLE) ? 0 : 1;
  r.host_progress = reinterpret_cast<unsigned long long*>(&d->page_d->progress[id]);
  r.dbg = d->dbg;
  r.run_epoch = __atomic_load_n(&d->page->epoch, __ATOMIC_ACQUIRE);
  r.host_line = reinterpret_cast<const uint64_t*>(&d->page_d->lp_line[id]);
  r.slot = id;
  r.exit_rec = &d->page_d->lp_exit[id];
  r.run_id = run_id;
  __atomic_store_n(&d->page->lp_line[id].budget, ((run_id & 0xFFFFFFull) << 40) | budget, __ATOMIC_RELEASE);
  __atomic_store_n(&d->page->progress[id], 0ull, __ATOMIC_RELEASE);
  s.last_begin = begin;
  s.last_end = end;
  s.last_redo_in = nr_in;
  s.t_launch_host = now_ns();
  s.launched = true;
  const uint64_t work = (end - begin) + nr_in;
  if (s.desc.kind == MS_LP_GEMM) {
    GemmParams p{};
    p.run = r;
    p.m = static_cast<int>(s.desc.m);
    p.n = static_cast<int>(s.desc.n);
    p.k = static_cast<int>(s.desc.k);
    p.tiles_m = s.tiles_m;
    p.tiles_n = s.tiles_n;
    p.group_m = s.desc.group_m ? s.desc.group_m : 16;
    p.c = reinterpret_cast<__nv_bfloat16*>(s.desc.c);
    p.split_k = s.split;
    p.ws = s.ws;
    p.tile_cnt = s.tile_cnt;  // the tile's last unit reduces the slices in-kernel
    const int mma_lag = [] {  // read per launch (A/B probes flip it in-process)
      const char* e = getenv("MS_LP_MMA_LAG");
      // default 2: unbounded is +2.5% TFLOP/s alone (profiles/r01_mma_lag_ab.json) but under the
      // 1 kW cap it lowers the HP clock (bench A/B: SLO -2 points, p99 +0.25 us;
      // profiles/r01_lag_bench_ab/)
      const int v = e ? atoi(e) : 2;
      return v < 0 ? 0 : v > 4 ? 4 : v;
    }();
    p.mma_lag = mma_lag;
    // k-split units stream their operands from HBM (no reuse across CTAs): bound the loads in
    // flight to ~96 KB per SM, which still covers the SM's share of HBM bandwidth at the
    // loaded latency (tools/drain23_stamps.py: producer stop 8-9 us after the flag with the
    // whole ring in flight).  MS_LP_TMA_INFLIGHT overrides (0 = unbounded).
    {
      const char* e = getenv("MS_LP_TMA_INFLIGHT");
      const int stage_bytes = (kBM + s.desc.block_n) * kBK * 2;
      p.tma_inflight = e ? std::max(0, atoi(e)) : (s.split > 1 ? std::max(2, (96 * 1024) / stage_bytes) : 0);
    }
    p.slow = s.slow;  // memory tier: bounded off-device admission (ms_lp_set_slow_tiles)
    p.slow_sem = s.slow_sem;
    p.slow_group = s.slow_group;
    p.slow_max = s.slow_max;
    p.half_base = s.half_base;
    p.half_units = s.half_units;
    p.tail_parts = s.tail_parts;
    if (s.pair) {
      // one CTA pair per tile; pairs of SMs left after the reserve
      const int reserve = (d->lp_sm_reserve + 1) & ~1;  // whole TPCs
      const int pairs = static_cast<int>(std::max<uint64_t>(
          1, std::min<uint64_t>(work, static_cast<uint64_t>(std::max(2, d->prop.multiProcessorCount - reserve) / 2))));
      p.group_m = s.desc.group_m ? s.desc.group_m : 8;
      if (s.pair_tn == 512)
        MS_CUDA(launch_kc(tc_gemm2_kernel<512>, 2 * pairs, 256, Gemm2Cfg<512>::kSmemBytes, d->lp, false, 2, s.tma_a,
                          s.tma_b, s.tma_bq, s.tma_c, p));
      else
        MS_CUDA(launch_kc(tc_gemm2_kernel<256>, 2 * pairs, 256, Gemm2Cfg<256>::kSmemBytes, d->lp, false, 2, s.tma_a,
                          s.tma_b, s.tma_bq, s.tma_c, p));
      return 0;
    }
    const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(work, d->prop.multiProcessorCount - d->lp_sm_reserve)));
    // Experimental (MS_LP_CLUSTER_ALIGN=C): launch the LP GEMM as C-CTA clusters and keep
    // one cluster slot of the machine free, so the HP chain's first C-CTA cluster finds C
    // empty SMs of one GPC without waiting for LP CTAs to exit.
    const char* ca = std::getenv("MS_LP_CLUSTER_ALIGN");
    const int align = ca ? atoi(ca) : 0;
    if ((align == 2 || align == 4) && s.desc.block_n == 256) {
      if (d->lp_align_clusters[align] == 0) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(align * 64);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = GemmCfg<256>::kSmemBytes;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim = {static_cast<unsigned>(align), 1, 1};
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int mc = 0;
        MS_CUDA(cudaOccupancyMaxActiveClusters(&mc, tc_gemm_kernel<256>, &cfg));
        d->lp_align_clusters[align] = mc;
      }
      const int slots = std::min(d->lp_align_clusters[align] - 1, grid / align);
      const int gc = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((work + align - 1) / align, std::max(1, slots))));
      MS_CUDA(launch_kc(tc_gemm_kernel<256>, gc * align, 256, GemmCfg<256>::kSmemBytes, d->lp, false, align, s.tma_a,
                        s.tma_b, s.tma_c, p));
      return 0;
    }
    return launch_gemm(d, s.desc.block_n, s.tma_a, s.tma_b, s.tma_c, p, grid, d->lp);
  }
  if (s.desc.kind == MS_LP_OPTIM) {
    OptimParams q{};
    q.run = r;
    q.p = reinterpret_cast<float*>(s.desc.a);
    q.m = reinterpret_cast<float*>(s.desc.b);
    q.v = reinterpret_cast<float*>(s.desc.c);
    q.g = reinterpret_cast<const __nv_bfloat16*>(s.desc.x);
    q.n = static_cast<unsigned long long>(s.desc.n_elems);
    q.tile_elems = s.desc.tile_elems;
    q.mode = s.desc.opt_mode;
    q.lr = s.desc.opt[0];
    q.b1 = s.desc.opt[1];
    q.b2 = s.desc.opt[2];
    q.eps = s.desc.opt[3];
    q.wd = s.desc.opt[4];
    q.c1 = s.desc.opt[5];
    q.c2 = s.desc.opt[6];
    const uint64_t cap = static_cast<uint64_t>(std::max(1, d->prop.multiProcessorCount - d->lp_sm_reserve));
    const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((work + kAxpyGroups - 1) / kAxpyGroups, cap)));
    const int threads = kAxpyGroups * kStreamThreads + 64;
    switch (s.desc.tile_elems / (kStreamThreads * 4)) {
      case 1: optim_kernel<1><<<grid, threads, 0, d->lp>>>(q); break;
      case 2: optim_kernel<2><<<grid, threads, 0, d->lp>>>(q); break;
      case 4: optim_kernel<4><<<grid, threads, 0, d->lp>>>(q); break;
      case 8: optim_kernel<8><<<grid, threads, 0, d->lp>>>(q); break;
      default: return fail(MS_E_ARG, "optimizer tile_elems must be 1024 * {1,2,4,8}");
    }
    MS_CUDA(cudaGetLastError());
    return 0;
  }
  StreamParams p{};
  p.run = r;
  p.x = reinterpret_cast<const __nv_bfloat16*>(s.desc.x);
  p.y = reinterpret_cast<__nv_bfloat16*>(s.desc.y);
  p.alpha = s.desc.alpha;
  p.n = static_cast<unsigned long long>(s.desc.n_elems);
  p.tile_elems = s.desc.tile_elems;
  p.slow = s.slow;
  p.slow_sem = s.slow_sem;
  p.slow_group = s.slow_group;
  p.slow_max = s.slow_max;
  // ctas_per_sm == 1: the grouped one-CTA-per-SM streamer (3 x 256 streaming threads)
  const bool grouped = s.desc.ctas_per_sm == 1;
  const uint64_t per_cta = grouped ? kAxpyGroups : 1;
  const uint64_t cap = static_cast<uint64_t>(std::max(1, d->prop.multiProcessorCount - d->lp_sm_reserve)) *
                       (grouped ? 1 : s.desc.ctas_per_sm);
  const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((work + per_cta - 1) / per_cta, cap)));
  const int vpt = s.desc.tile_elems / (kStreamThreads * 8);
  // Residency is capped at 4 CTAs per SM by registers (__launch_bounds__(320, 4): 48
  // registers, a 5th CTA does not fit), so the grid ((SMs - reserve) x 4) really leaves the
  // reserved SM empty for the first HP CTA.  (Capping it with unused dynamic shared memory
  // instead shrank the L1 carve-out and cost 20% of the streaming bandwidth; an uncapped
  // 53-register build fitted only 3 CTAs per SM and left 144 CTAs pending, which tripled the
  // preemption drain.)
  const int pad = 0;
  if (grouped) {
    const int threads = kAxpyGroups * kStreamThreads + 64;
    switch (vpt) {
      case 1: axpy_kernel<1, kAxpyGroups><<<grid, threads, 0, d->lp>>>(p); break;
      case 2: axpy_kernel<2, kAxpyGroups><<<grid, threads, 0, d->lp>>>(p); break;
      case 4: axpy_kernel<4, kAxpyGroups><<<grid, threads, 0, d->lp>>>(p); break;
      case 8: axpy_kernel<8, kAxpyGroups><<<grid, threads, 0, d->lp>>>(p); break;
      default: return fail(MS_E_ARG, "tile_elems must be 2048 * {1,2,4,8}");
    }
  } else {
    switch (vpt) {
      case 1: axpy_kernel<1, 1><<<grid, kStreamThreads + 64, pad, d->lp>>>(p); break;
      case 2: axpy_kernel<2, 1><<<grid, kStreamThreads + 64, pad, d->lp>>>(p); break;
      case 4: axpy_kernel<4, 1><<<grid, kStreamThreads + 64, pad, d->lp>>>(p); break;
      case 8: axpy_kernel<8, 1><<<grid, kStreamThreads + 64, pad, d->lp>>>(p); break;
      default: return fail(MS_E_ARG, "tile_elems must be 2048 * {1,2,4,8}");
    }
  }
  MS_CUDA(cudaGetLastError());
  return 0;
}

int ms_set_lp_sm_reserve(ms_dev* d, int n) {
  if (n < 0 || n >= d->prop.multiProcessorCount) return fail(MS_E_ARG, "bad SM reserve");
  d->lp_sm_reserve = n;
  return 0;
}

int ms_debug_stamps(ms_dev* d, int enable, unsigned long long* out, size_t n) {
  // Stream-local operations only: a device-wide sync (cudaFree / legacy-stream memset)
  // would deadlock against a resident doorbell gate.
  constexpr size_t kWords = 4096 * 8;
  if (!d->dbg_buf) MS_CUDA(cudaMalloc(&d->dbg_buf, kWords * sizeof(unsigned long long)));
  if (enable) {
    MS_CUDA(cudaMemsetAsync(d->dbg_buf, 0, kWords * sizeof(unsigned long long), d->aux));
    MS_CUDA(cudaStreamSynchronize(d->aux));
    d->dbg = d->dbg_buf;
    return 0;
  }
  if (out) {
    MS_CUDA(cudaMemcpyAsync(out, d->dbg_buf, std::min(n, kWords) * 8, cudaMemcpyDeviceToHost, d->aux));
    MS_CUDA(cudaStreamSynchronize(d->aux));
  }
  d->dbg = nullptr;
  return 0;
}

uint64_t ms_lp_total_tiles(ms_dev* d, int id) {
  return (d && id >= 0 && id < MS_MAX_LP && d->lp_slots[id].used) ? d->lp_slots[id].total_tiles : 0;
}

int ms_lp_tile_ctas(ms_dev* d, int id) {
  if (!d || id < 0 || id >= MS_MAX_LP || !d->lp_slots[id].used) return fail(MS_E_ARG, "bad LP kernel id");
  return d->lp_slots[id].pair ? 2 : 1;
}

uint64_t ms_lp_progress(ms_dev* d, int id) {
  if (!d || id < 0 || id >= MS_MAX_LP || !d->lp_slots[id].used) return 0;
  return __atomic_load_n(&d->page->progress[id], __ATOMIC_ACQUIRE);
}

int ms_lp_set_budget(ms_dev* d, int id, uint64_t budget) {
  MS_CHECK_LP(d, id);
  LpSlot& s = d->lp_slots[id];
  if (budget > s.last_end) budget = s.last_end;
  __atomic_store_n(&d->page->lp_line[id].budget, ((s.run_id & 0xFFFFFFull) << 40) | budget, __ATOMIC_RELEASE);
  return 0;
}

int ms_lp_poll(ms_dev* d, int id, ms_lp_status* st) {
  MS_CHECK_LP(d, id);
  if (!st) return fail(MS_E_ARG, "null status");
  LpSlot& s = d->lp_slots[id];
  const MsLpExit& e = d->page->lp_exit[id];
  const uint64_t rid = __atomic_load_n(&e.run_id, __ATOMIC_ACQUIRE);
  std::memset(st, 0, sizeof(*st));
  st->run_id = s.run_id;
  st->begin = s.last_begin;
  st->end = s.last_end;
  st->redo_in = s.last_redo_in;
  st->t_launch_host = s.t_launch_host;
  if (!s.launched || rid != s.run_id) return 0;
  st->cursor = e.cursor;
  st->redo_count = e.redo_count;
  st->tiles_done = e.tiles_done;
  st->preempted = static_cast<int32_t>(e.preempted);
  st->t_start = e.t_start;
  st->t_seen = e.t_seen;
  st->t_exit = e.t_exit;
  st->t_free = e.t_free;
  st->done = 1;
  s.redo_carry = e.redo_count;
  return 1;
}

int ms_lp_wait(ms_dev* d, int id, int64_t timeout_ns, ms_lp_status* st) {
  MS_CHECK_LP(d, id);
  if (!d->lp_slots[id].launched) return fail(MS_E_ARG, "LP kernel has no run to wait for");
  const int64_t t0 = now_ns();
  for (;;) {
    const int r = ms_lp_poll(d, id, st);
    if (r < 0) return r;
    if (r) return 0;
    if (timeout_ns >= 0 && now_ns() - t0 > timeout_ns) {
      const cudaError_t e = cudaStreamQuery(d->lp);
      if (e != cudaSuccess && e != cudaErrorNotReady)
        return fail(MS_E_CUDA, std::string("LP stream error: ") + cudaGetErrorString(e));
      return fail(MS_E_TIMEOUT, "LP run did not exit in time");
    }
  }
}

int ms_lp_reset(ms_dev* d, int id) {
  MS_CHECK_LP(d, id);
  LpSlot& s = d->lp_slots[id];
  // A run still in flight would publish a carry after the reset: refuse.
  if (s.launched && __atomic_load_n(&d->page->lp_exit[id].run_id, __ATOMIC_ACQUIRE) != s.run_id)
    return fail(MS_E_ARG, "ms_lp_reset: an LP run is still in flight");
  s.redo_carry = 0;
  // The last exit record is consumed: a later ms_lp_poll must not restore its carry.
  s.launched = false;
  // A fresh pass: slices of half-finished split-K tiles from an abandoned pass must not
  // count towards the new pass's reductions.
  if (s.tile_cnt)
    MS_CUDA(cudaMemsetAsync(s.tile_cnt, 0, sizeof(unsigned int) * s.tiles_m * s.tiles_n * s.split, d->lp));
  return 0;
}

int ms_preempt_raise(ms_dev* d, uint32_t* epoch, int64_t* t_host) {
  const uint32_t e = __atomic_add_fetch(&d->page->epoch, 1u, __ATOMIC_RELEASE);
  for (int i = 0; i < MS_MAX_LP; ++i) __atomic_store_n(&d->page->lp_line[i].epoch, static_cast<uint64_t>(e), __ATOMIC_RELEASE);
  if (t_host) *t_host = now_ns();
  if (epoch) *epoch = e;
  return 0;
}

uint32_t ms_preempt_epoch(ms_dev* d) { return __atomic_load_n(&d->page->epoch, __ATOMIC_ACQUIRE); }

// ------------------------------------------------------------------ HP chains
int ms_hp_register_chain(ms_dev* d, const ms_hp_op* ops, int n_ops, int* chain_id) {
  int cid = -1;
  for (int i = 0; i < MS_MAX_HP_CHAINS; ++i)
    if (!d->chains[i].used) {
      cid = i;
      break;
    }
  if (cid < 0 || n_ops < 1 || n_ops > kMaxChainOps) return fail(MS_E_ARG, "bad HP chain");
  // Batch-1 (m == 1) GEMM ops run as one HBM-streaming GEMV chain; they cannot share a
  // chain with tcgen05 (m >= 128) GEMMs.  Checked before anything is allocated.
  bool any_gemv = false, any_mat = false;
  for (int i = 0; i < n_ops; ++i) {
    const bool mm = ops[i].kind == MS_HP_GEMM || ops[i].kind == MS_HP_GEMM_SWIGLU;
    any_gemv |= mm && ops[i].m == 1;
    any_mat |= mm && ops[i].m != 1;
  }
  if (any_gemv && any_mat) return fail(MS_E_ARG, "an HP chain cannot mix m == 1 and m >= 128 GEMM ops");
  for (int i = 0; i < n_ops && any_gemv; ++i) {
    if ((ops[i].kind == MS_HP_BIAS_GELU || ops[i].kind == MS_HP_SILU_MUL) && ops[i].m != 1)
      return fail(MS_E_ARG, "batch-1 chain: elementwise ops must have m == 1");
    if (is_glue(ops[i].kind)) return fail(MS_E_ARG, "batch-1 chain: conv / attention glue ops need m >= 16 rows");
    if (ops[i].kind == MS_HP_GEMM && ops[i].m == 1 && (ops[i].bias || ops[i].resid || ops[i].geo.flags))
      return fail(MS_E_ARG, "batch-1 chain: GEMM epilogues are not supported (use BIAS_GELU / SILU_MUL ops)");
  }
  if (any_gemv && n_ops > kGemvMaxOps) return fail(MS_E_ARG, "batch-1 chain too long");
  HpChain ch;
  for (int i = 0; i < n_ops; ++i) {
    HpOpRt o;
    o.op = ops[i];
    o.ctl_index = d->next_hp_ctl++;
    if (o.ctl_index >= MS_N_CTL) return fail(MS_E_ARG, "out of HP control blocks");
    if ((o.op.kind == MS_HP_GEMM || o.op.kind == MS_HP_GEMM_SWIGLU) && o.op.m == 1) {
      // Batch-1 op: HBM-streaming matrix-vector product over the row-major weights in place
      // (hp_gemv.cuh).  A whole row (gate + up row for SWIGLU) must fit one 16 KB stage.
      const int64_t row_cap = kGemvStageBytes / 2 / (o.op.kind == MS_HP_GEMM_SWIGLU ? 2 : 1);
      if (o.op.n < 1 || o.op.k < 8 || o.op.k % 8 || o.op.k > row_cap) return fail(MS_E_ARG, "HP batch-1 GEMM shape");
      if ((o.op.a | o.op.b) % 16) return fail(MS_E_ARG, "HP batch-1 GEMM operands must be 16-byte aligned");
      o.gemv = true;
      o.split = 1;
    } else if (o.op.kind == MS_HP_GEMM) {
      if ((o.op.bias % 16) || (o.op.resid % 16) || ((o.op.geo.flags & 3) == 3) || (o.op.resid && o.op.n % 8))
        return fail(MS_E_ARG, "HP GEMM epilogue: 16-byte aligned bias / resid, one activation");
      const int bn = o.op.block_n ? o.op.block_n : 128;
      o.op.block_n = bn;
      if (o.op.m % kBM || o.op.n % bn || o.op.k % kBK) return fail(MS_E_ARG, "HP GEMM shape");
      o.tiles_m = static_cast<int>(o.op.m / kBM);
      o.tiles_n = static_cast<int>(o.op.n / bn);
      // Skinny HP GEMMs (M = 128) have too few tiles to pull HBM bandwidth from every SM:
      // split K so (tiles x slices) covers the SMs; slices must divide the k-blocks.
      const int tiles = o.tiles_m * o.tiles_n;
      const int kbs = static_cast<int>(o.op.k / kBK);
      int split = o.op.split_k;
      if (split <= 0) {
        split = 1;
        while (tiles * split * 2 <= d->prop.multiProcessorCount && kbs % (split * 2) == 0 && kbs / (split * 2) >= 4)
          split *= 2;
      }
      if (kbs % split) return fail(MS_E_ARG, "split_k must divide K / 64");
      o.split = split;
      if (split > 1) {
        MS_CUDA(cudaMalloc(&o.ws, sizeof(float) * static_cast<size_t>(split) * o.op.m * o.op.n));
        o.reduce_ctl_index = d->next_hp_ctl++;
        if (o.reduce_ctl_index >= MS_N_CTL) return fail(MS_E_ARG, "out of HP control blocks");
      }
      if (o.op.lda && (o.op.lda < o.op.k || o.op.lda % 8)) return fail(MS_E_ARG, "lda must be >= k and a multiple of 8");
      if (int rc = encode_2d(&o.tma_a, reinterpret_cast<void*>(o.op.a), o.op.m, o.op.k, kBM, o.op.lda)) return rc;
      if (int rc = encode_c(&o.tma_c, reinterpret_cast<void*>(o.op.c), o.op.m, o.op.n)) return rc;
      if (o.op.b_layout == 1) {
        if (int rc = encode_2d(&o.tma_b, reinterpret_cast<void*>(o.op.b), o.op.n, o.op.k, bn)) return rc;
      } else {
        const void* wb = reinterpret_cast<const void*>(o.op.b);
        if (o.op.b_layout == 0) {  // capture a k-block-major copy of the weights now
          MS_CUDA(cudaMalloc(&o.b_tiled, static_cast<size_t>(o.op.n) * o.op.k * 2));
          kblock_major_kernel<<<d->prop.multiProcessorCount * 4, 256, 0, d->aux>>>(
              reinterpret_cast<const __nv_bfloat16*>(o.op.b), o.b_tiled, o.op.n, o.op.k);
          MS_CUDA(cudaGetLastError());
          MS_CUDA(cudaStreamSynchronize(d->aux));
          wb = o.b_tiled;
        }
        if (int rc = encode_kblock_major(&o.tma_b, wb, o.op.n, o.op.k, bn)) return rc;
      }
    } else if (o.op.kind == MS_HP_GEMM_SWIGLU) {
      // per-op path: GEMM over the row-major [gate; up] weights into tmp, then SwiGLU kernel;
      // fused path: interleaved k-block-major copy, SwiGLU in the GEMM epilogue.
      if (o.op.m % kBM || o.op.n % 64 || o.op.k % kBK) return fail(MS_E_ARG, "HP GEMM_SWIGLU shape");
      if (o.op.lda && (o.op.lda < o.op.k || o.op.lda % 8)) return fail(MS_E_ARG, "lda must be >= k and a multiple of 8");
      o.op.block_n = 128;
      o.tiles_m = static_cast<int>(o.op.m / kBM);
      o.tiles_n = static_cast<int>(2 * o.op.n / 128);
      o.split = 1;
      o.act_ctl_index = d->next_hp_ctl++;
      if (o.act_ctl_index >= MS_N_CTL) return fail(MS_E_ARG, "out of HP control blocks");
      MS_CUDA(cudaMalloc(&o.tmp, static_cast<size_t>(o.op.m) * 2 * o.op.n * 2));
      if (int rc = encode_2d(&o.tma_a, reinterpret_cast<void*>(o.op.a), o.op.m, o.op.k, kBM, o.op.lda)) return rc;
      if (int rc = encode_c(&o.tma_c, o.tmp, o.op.m, 2 * o.op.n)) return rc;
      if (int rc = encode_2d(&o.tma_b, reinterpret_cast<void*>(o.op.b), 2 * o.op.n, o.op.k, 128)) return rc;
      MS_CUDA(cudaMalloc(&o.b_tiled, static_cast<size_t>(2 * o.op.n) * o.op.k * 2));
      kblock_major_swiglu_kernel<<<d->prop.multiProcessorCount * 4, 256, 0, d->aux>>>(
          reinterpret_cast<const __nv_bfloat16*>(o.op.b), o.b_tiled, o.op.n, o.op.k);
      MS_CUDA(cudaGetLastError());
      MS_CUDA(cudaStreamSynchronize(d->aux));
    } else if (o.op.kind == MS_HP_BIAS_GELU || o.op.kind == MS_HP_SILU_MUL) {
      if (o.op.n % 8) return fail(MS_E_ARG, "elementwise cols must be a multiple of 8");
    } else if (o.op.kind == MS_HP_H2D || o.op.kind == MS_HP_D2H) {
      if (o.op.m <= 0) return fail(MS_E_ARG, "copy size must be > 0");
    } else if (is_glue(o.op.kind)) {
      if (int rc = check_glue(o.op)) return rc;
    } else {
      return fail(MS_E_ARG, "unknown HP op");
    }
    ch.ops.push_back(o);
  }
  if (any_gemv) {
    if (int rc = plan_gemv(d, ch)) return rc;
  } else if (int rc = plan_fused(d, ch)) {
    return rc;
  }
  while (ch.lead_copies < static_cast<int>(ch.ops.size()) && ch.ops[ch.lead_copies].op.kind == MS_HP_H2D)
    ++ch.lead_copies;
  if (ch.lead_copies == static_cast<int>(ch.ops.size())) ch.lead_copies = 0;  // copy-only chain: plain path
  if (ch.lead_copies) {
    MS_CUDA(cudaEventCreateWithFlags(&ch.in_ev, cudaEventDisableTiming));
    // SM pull needs a device-mapped view of each pinned source and 16-byte granules
    bool ok = true;
    for (int i = 0; i < ch.lead_copies && ok; ++i) {
      const ms_hp_op& op = ch.ops[i].op;
      void* dp = nullptr;
      ok = op.m % 16 == 0 && op.a % 16 == 0 && op.c % 16 == 0 &&
           cudaHostGetDevicePointer(&dp, reinterpret_cast<void*>(op.a), 0) == cudaSuccess;
      if (ok) ch.pull_src.push_back(reinterpret_cast<uint64_t>(dp));
    }
    cudaGetLastError();  // (a non-mapped source is not an error: the copy-engine path runs)
    if (!ok) ch.pull_src.clear();
    MS_CUDA(cudaMalloc(&ch.pull_done, sizeof(unsigned int) * ch.lead_copies));
    MS_CUDA(cudaMemset(ch.pull_done, 0, sizeof(unsigned int) * ch.lead_copies));
  }
  ch.used = true;
  d->chains[cid] = ch;
  *chain_id = cid;
  return 0;
}

int ms_hp_unregister_chain(ms_dev* d, int cid) {
  if (cid < 0 || cid >= MS_MAX_HP_CHAINS || !d->chains[cid].used) return fail(MS_E_ARG, "bad chain");
  MS_CUDA(cudaStreamSynchronize(d->hp));
  MS_CUDA(cudaStreamSynchronize(d->hpcopy));
  HpChain& ch = d->chains[cid];
  if (ch.in_ev) cudaEventDestroy(ch.in_ev);
  if (ch.pull_done) cudaFree(ch.pull_done);
  for (HpOpRt& o : ch.ops) {
    if (o.ws) cudaFree(o.ws);
    if (o.tile_cnt) cudaFree(o.tile_cnt);
    if (o.b_tiled) cudaFree(o.b_tiled);
    if (o.tmp) cudaFree(o.tmp);
  }
  for (float* w : ch.fused_ws) cudaFree(w);
  if (ch.prog_d) cudaFree(ch.prog_d);
  if (ch.phase_d) cudaFree(ch.phase_d);
  if (ch.wire_d) cudaFree(ch.wire_d);
  if (ch.gemv_descs_d) cudaFree(ch.gemv_descs_d);
  ch = HpChain{};
  return 0;
}

int ms_hp_set_fused(ms_dev* d, int mode) {
  if (mode < 0 || mode > 2) return fail(MS_E_ARG, "fused mode must be 0, 1 or 2");
  d->hp_fused = mode;
  return 0;
}

int ms_hp_chain_info(ms_dev* d, int cid, int* fused_grid, int* cluster) {
  if (cid < 0 || cid >= MS_MAX_HP_CHAINS || !d->chains[cid].used) return fail(MS_E_ARG, "bad chain");
  const HpChain& ch = d->chains[cid];
  if (fused_grid) *fused_grid = ch.fusable ? ch.fused_grid : 0;
  if (cluster) *cluster = ch.fusable ? ch.fused_cs : 0;
  return 0;
}

int ms_hp_arm(ms_dev* d, int cid, uint32_t seq) {
  MS_CHECK_CHAIN(d, cid);
  const HpChain& ch = d->chains[cid];
  // 40 KB of (unused) shared memory keeps a 193 KB LP GEMM CTA off the gate's SM: an LP
  // CTA co-resident with the spinning gate observed preemptions ~5 us late.
  static const int gate_smem = [] {
    const char* e = std::getenv("MS_GATE_SMEM");
    return e ? std::max(0, std::min(atoi(e), kGateSmem)) : kGateSmem;
  }();
  // e2e input modes (MS_E2E_MODE): 2 = SM pull on the HP stream (default), 1 = copy engine on
  // its own gated stream + event, 0 = copy queued behind the HP gate
  const int e2e_mode = ch.lead_copies == 0 ? -1 : [] {
    const char* e = std::getenv("MS_E2E_MODE");
    return e ? atoi(e) : 2;
  }();
  const bool pull = e2e_mode == 2 && static_cast<int>(ch.pull_src.size()) == ch.lead_copies;
  const bool overlap = e2e_mode == 1;
  if (overlap) {
    // e2e input: its own gate on the copy stream, so the H2D starts at the ring (no SM
    // work needed, it overlaps the LP drain); the chain waits for the copy's event.
    gate_kernel<<<1, 32, gate_smem, d->hpcopy>>>(&d->page_d->doorbell, seq, nullptr, nullptr, nullptr);  // (smem: stays off LP SMs)
    MS_CUDA(cudaGetLastError());
    for (int i = 0; i < ch.lead_copies; ++i) {
      const ms_hp_op& op = ch.ops[i].op;
      MS_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(op.c), reinterpret_cast<const void*>(op.a),
                              static_cast<size_t>(op.m), cudaMemcpyDefault, d->hpcopy));
    }
    MS_CUDA(cudaEventRecord(ch.in_ev, d->hpcopy));
  }
  static const int gate_warps = [] {  // A/B knob (tools/gate_pollers_ab.py)
    const char* e = std::getenv("MS_GATE_WARPS");
    return e ? std::max(1, std::min(atoi(e), 32)) : kGateWarps;
  }();
  gate_kernel<<<1, 32 * gate_warps, gate_smem, d->hp>>>(&d->page_d->doorbell, seq, &d->page_d->hp[cid], d->mirror,
                                                        d->trace_on ? d->trace_dev : nullptr);
  MS_CUDA(cudaGetLastError());
  if (pull) {
    for (int i = 0; i < ch.lead_copies; ++i) {
      const ms_hp_op& op = ch.ops[i].op;
      PullParams q{};
      q.src = reinterpret_cast<const uint4*>(ch.pull_src[i]);
      q.dst = reinterpret_cast<uint4*>(op.c);
      q.n16 = static_cast<unsigned long long>(op.m) / 16;
      q.hp_ctl = d->hp_ctl + cid;
      q.done = ch.pull_done + i;
      static const int pull_ctas = [] {  // A/B knob (tools/e2e_tail_probe.py)
        const char* e = std::getenv("MS_PULL_CTAS");
        return e ? std::max(1, std::min(atoi(e), 64)) : kPullCtas;
      }();
      MS_CUDA(launch_k(hp_pull_kernel, pull_ctas, kPullThreads, 0, d->hp, true, q));
    }
    return launch_chain(d, cid, ch, seq, false, static_cast<size_t>(ch.lead_copies), true);
  }
  if (overlap) {
    MS_CUDA(cudaStreamWaitEvent(d->hp, ch.in_ev, 0));
    return launch_chain(d, cid, ch, seq, false, static_cast<size_t>(ch.lead_copies));
  }
  return launch_chain(d, cid, ch, seq, true);
}

uint32_t ms_hp_next_seq(ms_dev* d) { return ++d->hp_seq; }

int ms_hp_ring(ms_dev* d, uint32_t seq, int64_t* t_host) {
  if (!d) return fail(MS_E_ARG, "null device");
  const uint64_t e = __atomic_load_n(&d->page->epoch, __ATOMIC_ACQUIRE);
  // The doorbell only moves forward (serial-number order on the seq): ringing an older seq
  // must not re-close a gate a newer ring already opened.
  uint64_t cur = __atomic_load_n(&d->page->doorbell, __ATOMIC_ACQUIRE);
  for (;;) {
    const uint32_t s_cur = static_cast<uint32_t>(cur);
    const uint32_t s_new = static_cast<int32_t>(seq - s_cur) >= 0 ? seq : s_cur;
    if (__atomic_compare_exchange_n(&d->page->doorbell, &cur, (e << 32) | s_new, false, __ATOMIC_RELEASE,
                                    __ATOMIC_ACQUIRE))
      break;
  }
  if (t_host) *t_host = now_ns();
  return 0;
}

int ms_hp_launch_direct(ms_dev* d, int cid, uint32_t seq) {
  MS_CHECK_CHAIN(d, cid);
  const HpChain& ch = d->chains[cid];
  return launch_chain(d, cid, ch, seq, false);
}

int ms_hp_poll(ms_dev* d, int cid, uint32_t seq, ms_hp_times* t) {
  MS_CHECK_CHAIN(d, cid);
  if (!t) return fail(MS_E_ARG, "null times");
  const MsHpRecord& r = d->page->hp[cid];
  // 16-byte atomic read of the completion pair (aligned SSE load; written by one PCIe write).
  const __m128i v = _mm_load_si128(reinterpret_cast<const __m128i*>(&r.done_first));
  const uint64_t first = static_cast<uint64_t>(_mm_cvtsi128_si64(v));
  const uint64_t seq_dur = static_cast<uint64_t>(_mm_cvtsi128_si64(_mm_unpackhi_epi64(v, v)));
  std::memset(t, 0, sizeof(*t));
  t->seq = seq;
  if (static_cast<int32_t>(static_cast<uint32_t>(seq_dur >> 32) - seq) < 0) return 0;
  t->done = 1;
  t->t_gate = __atomic_load_n(&r.seq_gate, __ATOMIC_ACQUIRE) == seq ? r.t_gate : 0;
  t->t_first_cta = first;
  t->t_done = first + (seq_dur & 0xFFFFFFFFull);
  return 1;
}

int ms_hp_wait(ms_dev* d, int cid, uint32_t seq, int64_t timeout_ns, ms_hp_times* t) {
  MS_CHECK_CHAIN(d, cid);
  const int64_t t0 = now_ns();
  for (;;) {
    const int r = ms_hp_poll(d, cid, seq, t);
    if (r < 0) return r;
    if (r) return 0;
    if (timeout_ns >= 0 && now_ns() - t0 > timeout_ns) {
      const cudaError_t e = cudaStreamQuery(d->hp);
      if (e != cudaSuccess && e != cudaErrorNotReady)
        return fail(MS_E_CUDA, std::string("HP stream error: ") + cudaGetErrorString(e));
      return fail(MS_E_TIMEOUT, "HP chain did not complete in time");
    }
  }
}

// ------------------------------------------------------------------ clocks / timing
int ms_trace_enable(ms_dev* d, size_t capacity) {
  if (!d) return fail(MS_E_ARG, "null device");
  if (capacity == 0) {
    d->trace_on = false;
    return 0;
  }
  if (capacity & (capacity - 1)) return fail(MS_E_ARG, "trace capacity must be a power of two");
  if (capacity > (1u << 26)) return fail(MS_E_ARG, "trace capacity too large");
  if (d->trace_ev && d->trace_cap != capacity)
    return fail(MS_E_ARG, "trace already allocated with capacity " + std::to_string(d->trace_cap));
  if (!d->trace_ev) {
    // Stream-local operations only (a device-wide sync would wait for a parked HP gate).
    MS_CUDA(cudaHostAlloc(&d->trace_ev, capacity * sizeof(MsTraceEvent), cudaHostAllocMapped));
    std::memset(d->trace_ev, 0, capacity * sizeof(MsTraceEvent));
    MS_CUDA(cudaMalloc(&d->trace_head, sizeof(unsigned long long)));
    MS_CUDA(cudaMalloc(&d->trace_dev, sizeof(MsTrace)));
    MsTrace t{};
    MS_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&t.ev), d->trace_ev, 0));
    t.head = d->trace_head;
    t.cap_mask = static_cast<uint32_t>(capacity - 1);
    MS_CUDA(cudaMemsetAsync(d->trace_head, 0, sizeof(unsigned long long), d->aux));
    MS_CUDA(cudaMemcpyAsync(d->trace_dev, &t, sizeof(t), cudaMemcpyHostToDevice, d->aux));
    MS_CUDA(cudaStreamSynchronize(d->aux));
    d->trace_cap = capacity;
    d->trace_read = 0;
    d->trace_lost = 0;
  }
  d->trace_on = true;  // kernels launched from now on carry the trace
  return 0;
}

int ms_trace_drain(ms_dev* d, ms_event* out, size_t max, uint64_t* lost) {
  if (!d) return fail(MS_E_ARG, "null device");
  static_assert(sizeof(ms_event) == sizeof(MsTraceEvent), "ms_event layout");
  size_t n = 0;
  if (d->trace_ev && out) {
    const uint64_t mask = d->trace_cap - 1;
    while (n < max) {
      const uint64_t i = d->trace_read;
      MsTraceEvent* e = d->trace_ev + (i & mask);
      const uint64_t seq = __atomic_load_n(&e->seq, __ATOMIC_ACQUIRE);
      if (seq == i + 1) {
        ms_event ev;
        std::memcpy(&ev, e, sizeof(ev));
        if (__atomic_load_n(&e->seq, __ATOMIC_ACQUIRE) != seq) continue;  // overwritten while copied
        ev.seq = seq;
        out[n++] = ev;
        d->trace_read = i + 1;
      } else if (seq > i + 1) {  // the writer lapped the reader: skip to the oldest slot still held
        const uint64_t next = seq - d->trace_cap;
        d->trace_lost += next - i;
        d->trace_read = next;
      } else {
        break;  // not written yet
      }
    }
  }
  if (lost) *lost = d->trace_lost;
  return static_cast<int>(n);
}

int ms_clock_calibrate(ms_dev* d, int rounds, int64_t* offset_ns, int64_t* rtt_min) {
  if (rounds < 1) rounds = 1;
  unsigned long long* stamps = nullptr;
  MS_CUDA(cudaMalloc(&stamps, sizeof(unsigned long long) * rounds));
  __atomic_store_n(&d->page->ping, 0u, __ATOMIC_RELEASE);
  __atomic_store_n(&d->page->pong, 0u, __ATOMIC_RELEASE);
  echo_kernel<<<1, 1, 0, d->aux>>>(&d->page_d->ping, &d->page_d->pong, stamps, rounds);
  MS_CUDA(cudaGetLastError());
  std::vector<int64_t> t0(rounds), t1(rounds);
  for (int k = 1; k <= rounds; ++k) {
    t0[k - 1] = now_ns();
    __atomic_store_n(&d->page->ping, static_cast<uint32_t>(k), __ATOMIC_RELEASE);
    const int64_t deadline = t0[k - 1] + 1000000000ll;
    while (__atomic_load_n(&d->page->pong, __ATOMIC_ACQUIRE) < static_cast<uint32_t>(k)) {
      if (now_ns() > deadline) {
        cudaFree(stamps);
        return fail(MS_E_TIMEOUT, "clock echo timed out");
      }
    }
    t1[k - 1] = now_ns();
  }
  MS_CUDA(cudaStreamSynchronize(d->aux));
  std::vector<unsigned long long> g(rounds);
  MS_CUDA(cudaMemcpy(g.data(), stamps, sizeof(unsigned long long) * rounds, cudaMemcpyDeviceToHost));
  cudaFree(stamps);
  int best = 0;
  for (int i = 1; i < rounds; ++i)
    if (t1[i] - t0[i] < t1[best] - t0[best]) best = i;
  *rtt_min = t1[best] - t0[best];
  *offset_ns = static_cast<int64_t>(g[best]) - (t0[best] + t1[best]) / 2;
  return 0;
}

int ms_lp_time_full(ms_dev* d, int id, int reps, float* ms_per_run) {
  MS_CHECK_LP(d, id);
  if (reps < 1) return fail(MS_E_ARG, "reps must be >= 1");
  LpSlot& s = d->lp_slots[id];
  cudaEvent_t a, b;
  MS_CUDA(cudaEventCreate(&a));
  MS_CUDA(cudaEventCreate(&b));
  ms_lp_reset(d, id);
  ms_lp_status st;
  if (int rc = ms_lp_run(d, id, 0, s.total_tiles, s.total_tiles)) return rc;  // warm-up
  if (int rc = ms_lp_wait(d, id, 20000000000ll, &st)) return rc;
  MS_CUDA(cudaEventRecord(a, d->lp));
  for (int i = 0; i < reps; ++i)
    if (int rc = ms_lp_run(d, id, 0, s.total_tiles, s.total_tiles)) return rc;
  MS_CUDA(cudaEventRecord(b, d->lp));
  MS_CUDA(cudaEventSynchronize(b));
  float ms = 0;
  MS_CUDA(cudaEventElapsedTime(&ms, a, b));
  *ms_per_run = ms / reps;
  ms_lp_poll(d, id, &st);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return 0;
}

int ms_lp_time_range(ms_dev* d, int id, uint64_t begin, uint64_t end, int reps, float* ms_per_run) {
  MS_CHECK_LP(d, id);
  LpSlot& s = d->lp_slots[id];
  if (begin >= end || end > s.total_tiles || reps < 1) return fail(MS_E_ARG, "bad tile range");
  cudaEvent_t a, b;
  MS_CUDA(cudaEventCreate(&a));
  MS_CUDA(cudaEventCreate(&b));
  ms_lp_status st;
  ms_lp_reset(d, id);
  if (int rc = ms_lp_run(d, id, begin, end, end)) return rc;  // warm-up
  if (int rc = ms_lp_wait(d, id, 20000000000ll, &st)) return rc;
  MS_CUDA(cudaEventRecord(a, d->lp));
  for (int i = 0; i < reps; ++i)  // unpreempted runs leave no redo carry
    if (int rc = ms_lp_run(d, id, begin, end, end)) return rc;
  MS_CUDA(cudaEventRecord(b, d->lp));
  MS_CUDA(cudaEventSynchronize(b));
  float ms = 0;
  MS_CUDA(cudaEventElapsedTime(&ms, a, b));
  *ms_per_run = ms / reps;
  ms_lp_poll(d, id, &st);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return 0;
}

int ms_hp_time_chain(ms_dev* d, int cid, int reps, float* ms_per_chain) {
  MS_CHECK_CHAIN(d, cid);
  if (reps < 1) return fail(MS_E_ARG, "reps must be >= 1");
  cudaEvent_t a, b;
  MS_CUDA(cudaEventCreate(&a));
  MS_CUDA(cudaEventCreate(&b));
  if (int rc = ms_hp_launch_direct(d, cid, 0)) return rc;
  MS_CUDA(cudaStreamSynchronize(d->hp));
  MS_CUDA(cudaEventRecord(a, d->hp));
  for (int i = 0; i < reps; ++i)
    if (int rc = ms_hp_launch_direct(d, cid, 0)) return rc;
  MS_CUDA(cudaEventRecord(b, d->hp));
  MS_CUDA(cudaEventSynchronize(b));
  float ms = 0;
  MS_CUDA(cudaEventElapsedTime(&ms, a, b));
  *ms_per_chain = ms / reps;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return 0;
}

}  // extern "C"
