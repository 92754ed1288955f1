// Device-side data layout shared by the host driver (pool.cu) and the kernels
// (explore.cuh). B200-native IVM store: one contiguous block per explorer, bulk-copied
// into shared memory by the persistent explore kernel and written back when it exits.
#pragma once

#include <cstdint>

namespace pbbgpu {

enum : int { kEmpty = 0, kActive = 1, kInit = 2 };  // Ivm::State (ivm.hpp:23) + replay
enum : int { kFwd = 0, kBwd = 1 };                   // BranchDir (bound.hpp:14)
enum : int { kLB1 = 1, kLB2 = 2 };

constexpr int kMaxN = 64;        // smem-resident IVM store: cells as int8, free sets as u64
constexpr int kImpCap = 4096;    // improvement records per round
constexpr int kHistMax = 512;

// Persistent per-explorer block header (8 bytes).
struct IvmHdr {
  int16_t level;    // I, -1 when exhausted
  uint8_t state;    // kEmpty / kActive / kInit
  uint8_t has_end;  // end vector set (end < n!)
  uint8_t d1, d2;   // forward / backward fixed jobs of the node at `level`
  uint8_t rlev;     // kInit: next replay level
  uint8_t nrep;     // kInit: replay decompositions so far (L)
};

// Byte offsets inside one explorer block (same in global memory and shared memory
// for the persistent part; the scratch part exists only in shared memory).
struct IvmLayout {
  int n, m, mp;        // jobs, machines, machines rounded up to 4
  int o_cells;         // int8 [n(n+1)/2] triangular rows, row l holds n-l cells
  int o_v, o_dir, o_end, o_tgt;  // int8 [n] each
  int o_ft;            // uint16 [(n+1)*m]: FS[d] at slot d, TS[d] at slot n-d
  int o_r;             // uint16 [m]: per-machine sum of the jobs of row `level`
  int ftb;             // bytes per FT / R entry: 2, or 4 for wide times ((n+m)*max p >= 2^16, LB1)
  int gstride;         // persistent bytes per explorer (multiple of 16)
  // shared-memory scratch (per explorer)
  int o_fr, o_tl, o_rm, o_rt, o_frm;  // int32 [m]: front, tail, remain, remain+tail, front+remain (rt, frm: LB1)
  int o_lbf;           // int32 [n] lbf then int32 [n] lbb
  int o_free;          // uint8 [kMaxN]: free jobs of the node in decode order
  int o_heads, o_tails;  // uint16 [kMaxN*m] LB2 child heads / tails
  int o_lst;           // int4 [kMaxN] LB2 per-pair compacted Johnson sequence
  int o_pos;           // uint8 [kMaxN] LB2 job -> position in the compacted sequence
  int o_msk;           // uint32 [rounds][32] LB2 row masks (warp explorers, n <= 32; 0 = none)
  int sstride;         // shared bytes per explorer (== 16 mod 128: conflict-free LDS.128)
};

// Counters accumulated on the device (totals over all explorers).
struct DevCounters {
  unsigned long long decomposed;   // raw (PoolStats.decomposed semantics, explorer.hpp:46)
  unsigned long long dups;         // replay duplicates: sum of min(L, lnz(a))
  unsigned long long leaves;
  unsigned long long improvements;
  unsigned long long steals;
  unsigned long long steal_phases;
  unsigned long long inits;        // intervals_initialized
  unsigned long long steps;        // explore steps executed (select + process)
  int active;                      // explorers not Empty after the last steal phase
  int imp_count;                   // improvement records written this round
  int best;                        // device incumbent (makespan units)
  int round_live;                  // explorers not Empty when the last explore launch started
  unsigned int census_count;       // leaf positions recorded (record_census)
  int pad;
};

struct ImpRecord {
  int mk;
  int pad;
  int8_t perm[kMaxN];
};

struct ExploreParams {
  IvmLayout L;
  unsigned char* state;       // K * gstride
  int K;
  int steps;                  // max explore steps per explorer in this launch
  int prune_mode;             // 0 = prune against incumbent, 1 = pinned ub, 2 = disabled
  int pinned_ub;
  const int* p32;             // [n*mp] job-major, int32, rows padded to mp
  const int* ptot;            // [m] sum over all jobs
  int npairs;
  const uint8_t* pk;          // [npairs]
  const uint8_t* pl;          // [npairs]
  const uint8_t* order;       // [npairs*n]
  const uint16_t* lag;        // [npairs*n] indexed by job
  const uint32_t* packed;     // [n*npairs] transposed packed order (warp-per-explorer LB2)
  const uint8_t* invord;      // [n*npairs] position of job j in pair q's order
  DevCounters* ctr;
  unsigned long long* hist;   // [n+1] decomposed nodes by free-job count (raw)
  unsigned long long* dhist;  // [n+1] replay duplicates by free-job count
  ImpRecord* imp;             // [kImpCap]
  int smem_inst_bytes;        // bytes of the per-CTA instance region
  unsigned long long budget_ns;  // round length in device time (0 = steps only)
  int free_replay;            // init_at replay levels do not consume steps (reference policy)
  int census_cap;             // record_census: capacity of `census` (0 = off)
  unsigned long long* census; // leaf positions as decimals (position_u64, explorer.cpp:47)
  float* lens;                // [K] steal-phase remaining work written at the write-back (kLensInKernel
                              // variants; null = lens_kernel after the launch)
  const float* lgfact;        // [n+1] log2(k!)
  int lens_mode;              // split mode of the steal phase (explorer_lens)
};

}  // namespace pbbgpu
