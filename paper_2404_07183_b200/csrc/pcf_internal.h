// Internal launch interfaces shared by the kernel translation units and the C-ABI layer.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/pcf_b200.h"

namespace pcfb {
// dynamic shared memory the pairwise planner may give one tile CTA: the sm_100 opt-in
// maximum (227 KB) less the tile kernels' static shared memory (A/B at App-A 30k: 220 KB
// -> 227 KB, fast 437 -> 434 ms, exact 581 -> 579 ms)
constexpr int64_t kPlanSmemBudget = 227 * 1024 - 64;

constexpr int kTileThreads = 512;  // CTA size of the persistent tile kernels
// K1s column prefetch ring: slots per lane (pcf_tiles.cuh kRingSlots); the ring takes
// kRingSlots * kTileThreads records at the top of the dynamic shared memory
constexpr int kK1sRingSlots = 8;
constexpr int kK1sThreads = 640;  // K1s CTA size (pcf_tiles.cuh kRingThreads)

typedef pcf_work_item PcfWorkItem;

struct FillArgs {
  const void* recs;
  const void* recs8;
  const int64_t* soff;
  const int64_t* goff8;
  const int32_t* perm;
  int64_t M;
  const PcfWorkItem* items;
  int n_items;
  int* counter;
  int op;
  double p, a, b;
  int apply_root;
  void* out;
  int out_f32;
  int64_t ld;
  unsigned long long* err;
  int smem_mode;
  int smem_bytes;
  int rec_bytes;  // 16: float64 records, 8: float32 records (recs/recs8 point to Rec32)
  int num_sms;
  // optional per-item completion counters (pcf_matrix_host): item i adds 1 to
  // tag_done[item_tag[i]] after its stores; null = no signalling
  const int32_t* item_tag = nullptr;
  int32_t* tag_done = nullptr;
};

struct RowsArgs {
  const void* recs;
  const int64_t* soff;
  const int32_t* inv;
  int64_t M, r0, r1;
  int op;
  double p, a, b;
  int apply_root, diag;
  void* slab;
  int out_f32;
  unsigned long long* err;
};

int hkind_of(int op, double p);
inline bool pcf_op_ok(int op) {
  const int base = op & ~PCF_OP_FAST_POW;
  return base == PCF_OP_LP || base == PCF_OP_INNER;
}
cudaError_t launch_fill_tiles(const FillArgs& A, cudaStream_t st);
cudaError_t launch_diag(const void* recs, const int64_t* soff, const int32_t* perm, int64_t M,
                        int gram, double a, double b, void* out, int out_f32, int64_t ld,
                        unsigned long long* err, cudaStream_t st);
cudaError_t launch_fill_rows(const RowsArgs& A, cudaStream_t st);
cudaError_t launch_pair_list(const void* recs, const int64_t* soff, const int64_t* pairs,
                             int64_t npairs, int op, double p, double a, double b, double* res,
                             cudaStream_t st);
cudaError_t launch_pack(const void* tcat, const void* vcat, int f32, const int64_t* off,
                        const int32_t* perm, const int64_t* soff, int64_t M, void* recs,
                        const int64_t* goff8, void* recs8, cudaStream_t st);

cudaError_t launch_pack32(const float* tcat, const float* vcat, const int64_t* off,
                          const int32_t* perm, const int64_t* soff, int64_t M, void* recs32,
                          const int64_t* goff16, void* recs32g, cudaStream_t st);

cudaError_t launch_sweep_cells(const void* recs, const int64_t* soff, int64_t s, int64_t q,
                               double a, double b, double* cells, int64_t cap, int64_t* count,
                               cudaStream_t st);

constexpr int kRedBytes = 4 * kTileThreads * 8;  // K1 segment partials + tails, 2 buffers

void set_error(const char* fmt, ...);

}  // namespace pcfb
