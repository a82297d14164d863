// Layout of the control words shared by the host runtime and the sm_100a kernels.
//
// HBM / host-memory placement:
//   * HostPage   — one 4 KB pinned, host-mapped page per device (cudaHostAllocMapped).
//                  Host -> device: preempt epoch, HP doorbell, LP budgets (release
//                  stores by the host, one elected device poller reads them with
//                  ld.acquire.sys).  Device -> host: LP exit records and HP completion
//                  records (st.release.sys), polled by the scheduler thread instead of
//                  cudaStreamSynchronize.
//   * DevMirror  — device-memory copies of the epoch / budgets, 8 copies on separate
//                  128 B lines so 148 CTAs' polls spread over L2 slices.  Written only by
//                  the elected poller (CTA 0 of the running LP kernel).
//   * LpCtl      — per registered LP kernel: the tile-claim counter (the cursor), the
//                  exit counter, and timestamps; self-resetting at the end of each run.
#pragma once
#include <stdint.h>

#define MS_MAX_LP 96  /* config-2 LP: the ~63 distinct GEMM shapes of a ResNet-50 training step */
#define MS_MAX_HP_CHAINS 64
#define MS_N_CTL (MS_MAX_LP + 8192)  // control blocks: LP slots, then HP chain kernels
#define MS_MIRROR_COPIES 8
#define MS_MIRROR_STRIDE 32  // uint32 elements = 128 B

struct MsLpExit {                 // device -> host, one per LP slot (72 B)
  uint64_t run_id;                // written last (release); host waits for its run id
  uint64_t cursor;                // next never-claimed tile of [begin, end)
  uint64_t redo_count;            // claimed-but-unfinished tiles carried to the next run
  uint64_t tiles_done;            // tiles completed in this run
  uint64_t t_start;               // first CTA start (globaltimer ns)
  uint64_t t_seen;                // first CTA to observe the preempt epoch (0 = none)
  uint64_t t_exit;                // last CTA exit
  uint64_t preempted;             // 1 if the run ended because of the epoch
  uint64_t t_free;                // LP grids: every CTA but CTA 0 gone and CTA 0's work done
};

struct MsHpRecord {               // device -> host, one per HP chain slot (64 B)
  // Completion: ONE 16-byte store {t_first_cta, (seq << 32) | (t_done - t_first_cta)} —
  // a single PCIe write, so no system-scope fence (MEMBAR.SYS costs ~8 us) is needed.
  uint64_t done_first;            // t_first_cta of the completed seq
  uint64_t done_seq_dur;          // (seq << 32) | duration
  uint64_t t_gate;                // gate kernel observed the doorbell
  uint32_t seq_gate;              // gate released for this seq
  uint32_t pad0;
  uint64_t pad[4];
};

// One 64 B line per LP slot: the LP run's elected poller fetches {epoch, budget} with a
// single 16-byte ld.acquire.sys (one PCIe round trip per poll iteration).
struct MsLpLine {
  uint64_t epoch;                 // copy of the preempt epoch (host writes every line on raise)
  uint64_t budget;                // (run tag << 40) | soft end tile id
  uint64_t pad[6];
};

struct MsHostPage {
  uint32_t epoch;                 // preempt epoch (monotonic, canonical host copy)
  uint32_t pad0[31];
  uint64_t doorbell;              // HP doorbell: (epoch << 32) | seq, one release store
  uint64_t pad1[15];
  MsLpLine lp_line[MS_MAX_LP];
  uint64_t progress[MS_MAX_LP];   // device -> host: claim counter of the running LP run
  MsLpExit lp_exit[MS_MAX_LP];
  MsHpRecord hp[MS_MAX_HP_CHAINS];
  uint32_t ping, pad3[31];        // clock calibration echo
  uint32_t pong, pad4[31];
};

// Device-side event trace (ms_trace_enable / ms_trace_drain): events in pinned host memory,
// positions handed out by a device-memory counter; `seq` is stored last (release) so the
// host can tell a complete slot from one still being written or already overwritten.
struct MsTraceEvent {  // == ms_event
  uint64_t seq;
  uint64_t t_ns;
  uint32_t kind;
  uint32_t id;
  uint64_t a, b;
};
struct MsTrace {
  MsTraceEvent* ev;          // host-mapped ring (device pointer)
  unsigned long long* head;  // device memory: events written so far
  uint32_t cap_mask;         // capacity - 1 (power of two)
};

struct MsDevMirror {
  uint32_t epoch[MS_MIRROR_COPIES * MS_MIRROR_STRIDE];
  uint64_t budget[MS_MAX_LP][16];
};

struct alignas(128) MsLpCtl {
  unsigned long long claim;       // virtual claim index: redo_in entries first, then fresh tiles
  unsigned long long t_free;      // LP grids: max over CTAs != 0 of their exit (0 = none yet)
  unsigned long long t_start;     // min over CTAs
  unsigned long long t_seen;      // min over CTAs that saw the epoch
  unsigned int exited;            // CTAs finished (relaxed; read by CTA 0's host poller)
  unsigned int redo_out_n;
  unsigned int preempted;
  unsigned int pad[17];
  unsigned long long top;  // exit counter: (tiles done << 32) | CTAs exited, own 128 B line
  unsigned long long pad2[15];
};

struct MsHpCtl {                  // per HP chain slot, device memory
  unsigned long long t_first_cta;
  unsigned int exited[16];        // per chain kernel exit counters
};
