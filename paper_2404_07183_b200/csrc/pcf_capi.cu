// C-ABI layer: argument checking, error text, the tile planner and the host-buffer
// mirrors of the reference kernel module.  No exceptions cross this boundary.
#include <stdarg.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>
#include <algorithm>
#include <vector>
#include "pcf_internal.h"
#include "pcf_pow.cuh"

namespace pcfb {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static int cuda_fail(cudaError_t e, const char* where) {
  set_error("%s: %s", where, cudaGetErrorString(e));
  return PCF_ERR_CUDA;
}

static int num_sms_current() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  return n > 0 ? n : 148;
}

}  // namespace pcfb

using namespace pcfb;

extern "C" {

const char* pcf_version(void) { return "pcfb200 0.1.0 (sm_100a)"; }
const char* pcf_last_error(void) { return g_err; }
int pcf_tile_threads(void) { return kTileThreads; }

int pcf_pack_sorted(const void* tcat_dev, const void* vcat_dev, int is_f32,
                    const int64_t* off_dev, const int32_t* perm_dev, const int64_t* soff_dev,
                    int64_t M, void* recs_dev, const int64_t* goff8_dev, void* recs8_dev,
                    void* stream) {
  if (M < 0 || (M > 0 && (!tcat_dev || !vcat_dev || !off_dev || !perm_dev || !soff_dev || !recs_dev))) {
    set_error("pcf_pack_sorted: bad arguments");
    return PCF_ERR_ARG;
  }
  if (M == 0) return PCF_OK;
  cudaError_t e = launch_pack(tcat_dev, vcat_dev, is_f32, off_dev, perm_dev, soff_dev, M, recs_dev,
                              goff8_dev, recs8_dev, (cudaStream_t)stream);
  return e == cudaSuccess ? PCF_OK : cuda_fail(e, "pcf_pack_sorted");
}

// ------------------------------------------------------------------------------ planner
// Offsets of the slot-interleaved 8-row groups (record k of sorted PCF s at
// goff8[s/8] + 8k + s%8): group g spans 8 * sizes[8g] records (sizes sorted descending).
int pcf_group_offsets(const int64_t* sizes, int64_t M, int32_t group, int64_t* goff) {
  if (M < 0 || (M > 0 && (!sizes || !goff)) || (group != 8 && group != 16)) {
    set_error("pcf_group_offsets: bad arguments");
    return PCF_ERR_ARG;
  }
  const int64_t ng = (M + group - 1) / group;
  goff[0] = 0;
  for (int64_t g = 0; g < ng; ++g) goff[g + 1] = goff[g] + group * sizes[group * g];
  return PCF_OK;
}

int pcf_pack_sorted32(const float* tcat_dev, const float* vcat_dev, const int64_t* off_dev,
                      const int32_t* perm_dev, const int64_t* soff_dev, int64_t M,
                      void* recs32_dev, const int64_t* goff16_dev, void* recs32g_dev,
                      void* stream) {
  if (M <= 0) return PCF_OK;
  if (!tcat_dev || !vcat_dev || !off_dev || !perm_dev || !soff_dev || !recs32_dev ||
      !goff16_dev || !recs32g_dev) {
    set_error("pcf_pack_sorted32: bad arguments");
    return PCF_ERR_ARG;
  }
  cudaError_t e = launch_pack32(tcat_dev, vcat_dev, off_dev, perm_dev, soff_dev, M, recs32_dev,
                                goff16_dev, recs32g_dev, (cudaStream_t)stream);
  return e == cudaSuccess ? PCF_OK : cuda_fail(e, "pcf_pack_sorted32");
}

// Row blocks of the size-sorted collection are one or two 8-row groups.  Each gets the
// smallest merge-path split G (quarter-warps per pair, 64 quarters = RG x C x G) whose
// shared-memory tile -- interleaved rows + two streamed chunks of C columns + the
// segment-partial buffer -- fits the budget; blocks whose rows do not fit at any G go to
// the global-memory kernel.  Column ranges are cut into items of at most max_cols
// columns; items are returned cost-descending (LPT order for the persistent kernels'
// atomic queues), shared-memory items first.
int pcf_plan_pairwise(const int64_t* sizes, int64_t M, int64_t smem_budget, int64_t max_cols,
                      int32_t max_log2G, int32_t rec_bytes, pcf_work_item* items, int64_t cap,
                      int64_t* n_items, int32_t* smem_bytes) {
  if (M < 0 || (M > 0 && !sizes) || !n_items || smem_budget <= 0 ||
      (rec_bytes != 8 && rec_bytes != 16)) {
    set_error("pcf_plan_pairwise: bad arguments");
    return PCF_ERR_ARG;
  }
  std::vector<int64_t> S(M + 1, 0);
  for (int64_t i = 0; i < M; ++i) {
    if (sizes[i] < 1 || (i > 0 && sizes[i] > sizes[i - 1])) {
      set_error("pcf_plan_pairwise: sizes must be >= 1 and sorted descending");
      return PCF_ERR_ARG;
    }
    S[i + 1] = S[i] + sizes[i];
  }
  const int GW = 128 / rec_bytes;        // rows per interleaved group / lanes per smem phase
  const int LOGU = GW == 16 ? 5 : 6;     // log2 of phase units per CTA (512 / GW)
  const int64_t RB = rec_bytes;
  if (max_log2G < 0) max_log2G = 0;
  if (max_log2G > LOGU) max_log2G = LOGU;
  auto al = [](int64_t x) { return (x + 127) & ~(int64_t)127; };
  auto group_recs = [&](int64_t r) { return (int64_t)GW * sizes[r]; };  // r: first row of a group
  const int T = kTileThreads;
  constexpr int64_t kK1rMinRecs = 1024;
  static const int kSingleMinLogG =
      getenv("PCF_SINGLE_MIN_LOG2G") ? atoi(getenv("PCF_SINGLE_MIN_LOG2G")) : 1;
  // largest G accepted for single-buffered K1 on rows whose group misses double buffering
  static const bool kK1cEnabled = getenv("PCF_NO_K1C") == nullptr;
  static const bool kExactPartial = getenv("PCF_NO_EXACT_PARTIAL") == nullptr;
  static const bool kK1sEnabled = getenv("PCF_NO_K1S") == nullptr;
  // at equal G, one 8-row group with twice the columns instead of two groups (A/B knob)
  static const bool kPreferRG1 = getenv("PCF_PREFER_RG1") != nullptr;
  // per-item K1 configs (A/B: PCF_NO_ITEM_CONFIG=1 keeps the row block's config everywhere)
  static const bool kPerItem = getenv("PCF_NO_ITEM_CONFIG") == nullptr;
  static const bool kExactSingle = getenv("PCF_NO_EXACT_SINGLE") == nullptr;
  // K1s with one 8-row group (80 columns per pass) even where two fit (A/B knob)
  static const bool kK1sRG1 = getenv("PCF_K1S_RG1") != nullptr;
  // a single column buffer exposes one chunk copy per chunk; PCF_SINGLE_MIN_STEPS=n keeps
  // double buffering unless each lane walks >= n cells per chunk (A/B: 256 made App-A 30k
  // 437 -> 469 ms and c1/c2 no faster, so the default is 0 -- always halve G)
  static const int kSingleMinSteps =
      getenv("PCF_SINGLE_MIN_STEPS") ? atoi(getenv("PCF_SINGLE_MIN_STEPS")) : 0;
  auto long_walk = [&](int64_t n_row, int64_t n_col, int lg_new) {
    return ((n_row + n_col) >> std::max(lg_new, 0)) >= kSingleMinSteps;
  };
  static const bool kRedOnlyG = getenv("PCF_RED_ALWAYS") == nullptr;
  // K1 segment partials: [2][512] doubles plus [2][512 / G] tails, only when G > 1
  auto red_bytes = [&](int lg) -> int64_t {
    if (!kRedOnlyG) return kRedBytes;
    return lg > 0 ? (int64_t)(2 * kTileThreads + 2 * (kTileThreads >> lg)) * 8 : 0;
  };
  // per-item single-buffer configs may take up to 2^kSingleMaxUp times the columns
  static const int kSingleMaxUp =
      getenv("PCF_SINGLE_MAX_UP") ? atoi(getenv("PCF_SINGLE_MAX_UP")) : 1;
  static const int kFastRingMinLogG =
      getenv("PCF_FAST_RING_MINLOG2G") ? atoi(getenv("PCF_FAST_RING_MINLOG2G")) : -1;
  // K1r merge-path split: with the column rings one lane per pair is fastest (c4 K1r
  // 71.8 ms at G = 1 vs 87.8 ms at G <= 32: each segment pays a co-rank search and a ring
  // fill from L2), and it is the bitwise sum
  static const int kK1rMaxLogG = getenv("PCF_K1R_MAXLOG2G") ? atoi(getenv("PCF_K1R_MAXLOG2G")) : 0;
  static const int kSingleFallbackLogG =
      getenv("PCF_SINGLE_FALLBACK_LOG2G") ? atoi(getenv("PCF_SINGLE_FALLBACK_LOG2G")) : -1;
  std::vector<pcf_work_item> runs[5];  // by kernel: K1 (mode 1), K1c (3), K1s (4), K1r (2), K1g (0)
  int64_t need_max = 0, k1r_need = 0, k1c_need = 0, k1s_need = 0;
  // K1s prefetch rings at the top of shared memory, 1 KB aligned
  const int64_t k1s_ring = (int64_t)kK1sRingSlots * kK1sThreads * RB + 1024;
  // K1r: rings of the 512 lanes, 8 or 4 slots
  const int64_t k1r_ring8 = (int64_t)kK1sRingSlots * kTileThreads * RB + 1024;
  const int64_t k1r_ring4 = (int64_t)4 * kTileThreads * RB + 1024;
  const int64_t n_groups = (M + GW - 1) / GW;
  // K1c (one long row resident, interleaved column groups streamed): the best config for a
  // column range starting at group ks -- largest CG (fewest segments) that fits, double
  // buffered if possible.  Returns false if not even one group fits.
  // K1c segment partials as K1's: [2][512] + tails [2][512 / G], nothing without a split
  static const bool kK1cRedFull = getenv("PCF_RED_ALWAYS") != nullptr;
  auto k1c_red = [&](int g) -> int64_t {
    if (kK1cRedFull) return kRedBytes;
    return g > 0 ? (int64_t)(2 * kTileThreads + 2 * (kTileThreads >> g)) * 8 : 0;
  };
  auto k1c_config = [&](int64_t r, int64_t ks, int* lcg, int* lg, bool* one, int64_t* need) {
    const int64_t row_need = al((sizes[r] + 4) * RB + 16);
    for (int l = LOGU; l >= 0; --l) {
      const int g = LOGU - l;
      if (g > max_log2G) break;
      const int64_t ke = std::min<int64_t>(ks + ((int64_t)1 << l), n_groups);
      int64_t chunk = 0;
      for (int64_t k = ks; k < ke; ++k) chunk += group_recs(GW * k) * RB;
      for (int nb = 2; nb >= 1; --nb) {
        const int64_t nd = row_need + nb * al(chunk + 16) + k1c_red(g);
        if (nd <= smem_budget) {
          *lcg = l;
          *lg = g;
          *one = nb == 1;
          *need = nd;
          return true;
        }
      }
    }
    return false;
  };
  if (max_cols < 1) max_cols = 1 << 30;
  {
    // small collections: cut the column ranges finer so the persistent kernels see
    // ~8 items per SM (c1's 1000 PCFs are 63 row blocks: one item each would leave
    // 85 of 148 SMs idle)
    const double target = 8.0 * 148.0;
    const double want = (double)(M / 8 + 1) * (double)M / (2.0 * target);
    int64_t mc = 64;
    while (mc < want && mc < max_cols) mc <<= 1;
    max_cols = std::min<int64_t>(max_cols, mc);
  }
  int64_t r0 = 0;
  while (r0 < M - 1) {
    int best_logRG = -1, best_logC = 0, best_logG = 99;
    int64_t best_need = 0;
    for (int logRG = 1; logRG >= 0; --logRG) {
      if (logRG == 1 && r0 + GW >= M - 1) continue;  // second group would have no pairs
      int64_t rows_b = group_recs(r0) * RB;
      if (logRG == 1) rows_b += group_recs(r0 + GW) * RB;
      for (int logC = LOGU - logRG; logC >= 0; --logC) {
        const int logG = LOGU - logRG - logC;
        if (logG > max_log2G) break;
        const int64_t C = 1 << logC;
        const int64_t c0 = r0 + 1, ce = std::min<int64_t>(c0 + C, M);
        const int64_t need =
            al(rows_b) + 2 * al((S[ce] - S[c0]) * RB + 32) + kRedBytes;
        if (need > smem_budget) continue;
        if (logG < best_logG ||
            (logG == best_logG && (kPreferRG1 ? logRG < best_logRG : logRG > best_logRG))) {
          best_logRG = logRG;
          best_logC = logC;
          best_logG = logG;
          best_need = need;
        }
        break;  // larger logC with this RG already failed or this one fits; keep smallest G
      }
    }
    bool single = false;
    if (best_logRG < 0 && max_log2G == 0 && kExactPartial && (r0 % GW) == 0) {
      // exact mode (G = 1): 64 columns per chunk do not fit next to this row block, so
      // run K1 with idle quarters -- the most lanes (rows x columns) that fit, at least
      // half the CTA, double-buffered when that keeps as many lanes -- instead of K1g
      // (c2 exact, 200-record rows at 256 lanes: 30.8 -> 18.3 ms; App-A rows of 500+
      // records reach only 64-128 lanes, which measured 1.8x slower than K1g)
      constexpr int kExactMinLanes = kTileThreads / 2;
      int best_lanes = 0;
      for (int logRG = 1; logRG >= 0; --logRG) {
        if (logRG == 1 && r0 + GW >= M - 1) continue;
        int64_t rows_b = group_recs(r0) * RB;
        if (logRG == 1) rows_b += group_recs(r0 + GW) * RB;
        for (int nb = 2; nb >= 1; --nb)
          for (int logC = LOGU - logRG; logC >= 2; --logC) {
            const int64_t c0 = r0 + 1, ce = std::min<int64_t>(c0 + ((int64_t)1 << logC), M);
            const int64_t need = al(rows_b) + nb * al((S[ce] - S[c0]) * RB + 32) + kRedBytes;
            if (need > smem_budget) continue;
            const int lanes = (GW << logRG) << logC;
            if (lanes >= kExactMinLanes && lanes > best_lanes) {
              best_lanes = lanes;
              best_logRG = logRG;
              best_logC = logC;
              best_logG = 0;
              best_need = need;
              single = nb == 1;
            }
            break;
          }
      }
    }
    if (best_logRG < 0 && kSingleFallbackLogG >= 0 && (r0 % GW) == 0) {
      // the 8-row group fits only with ONE column buffer: K1 single-buffered at the
      // largest column count that fits (instead of K1r / K1g)
      const int64_t rows_b = group_recs(r0) * RB;
      for (int lc = LOGU; lc >= 0; --lc) {
        const int lg = LOGU - lc;
        if (lg > max_log2G || lg > kSingleFallbackLogG) break;
        const int64_t c0 = r0 + 1, ce = std::min<int64_t>(c0 + ((int64_t)1 << lc), M);
        const int64_t need1 = al(rows_b) + al((S[ce] - S[c0]) * RB + 32) + kRedBytes;
        if (need1 <= smem_budget) {
          best_logRG = 0;
          best_logC = lc;
          best_logG = lg;
          best_need = need1;
          single = true;
          break;
        }
      }
    }
    bool smem = best_logRG >= 0 && (r0 % GW) == 0;
    // fast plan, long rows: K1 would split each pair into >= 2^kFastRingMinLogG merge-path
    // segments; K1s (one lane per pair, columns through prefetch rings) instead
    const bool use_ring = smem && kFastRingMinLogG >= 0 && best_logG >= kFastRingMinLogG &&
                          kK1sEnabled && al(group_recs(r0) * RB) + k1s_ring <= smem_budget;
    if (use_ring) smem = false;
    int rows, logC, logG, s_mode = -1;
    bool ring4 = false;  // K1r: 4-slot column rings (flag bit 9 of logC)
    if (smem && !single && best_logG >= kSingleMinLogG &&
        long_walk(sizes[r0], sizes[std::min<int64_t>(r0 + 1, M - 1)], best_logG - 1)) {
      // long rows: G >= 16 merge-path segments of a few dozen steps each.  A single
      // column buffer of twice the columns halves G (half the co-rank searches and
      // partial sums per cell) at the price of one exposed chunk load per chunk.
      const int64_t rows_b = group_recs(r0) * RB + (best_logRG ? group_recs(r0 + GW) * RB : 0);
      const int64_t C2 = (int64_t)1 << (best_logC + 1);
      const int64_t c0 = r0 + 1, ce = std::min<int64_t>(c0 + C2, M);
      const int64_t need1 = al(rows_b) + al((S[ce] - S[c0]) * RB + 32) + kRedBytes;
      if (need1 <= smem_budget) {
        single = true;
        best_logC += 1;
        best_logG -= 1;
        best_need = need1;
      }
    }
    if (smem) {
      rows = GW << best_logRG;
      logC = best_logC;
      logG = best_logG;
    } else if (sizes[r0] >= kK1rMinRecs &&
               al(sizes[r0] * RB) + k1r_ring4 <= smem_budget) {
      // K1r: this long row alone resident in shared memory, C columns x G segments per
      // pass; G keeps >= ~128 walk steps per lane (row length dominates long-row pairs).
      // Short rows that miss K1 (exact mode: G = 1 needs 64 staged columns) stay on K1g,
      // whose 32-row passes re-use each column from L1.
      rows = 1;
      logG = 0;
      while (logG < std::min(std::min(max_log2G, 5), kK1rMaxLogG) &&
             (sizes[r0] >> (logG + 1)) >= 128)
        ++logG;
      logC = 9 - logG;
      // the lanes' column rings (8 slots; 4 when the row leaves no room for 8: flag bit 9)
      if (al(sizes[r0] * RB) + k1r_ring8 <= smem_budget) {
        k1r_need = std::max(k1r_need, al(sizes[r0] * RB) + k1r_ring8);
      } else {
        k1r_need = std::max(k1r_need, al(sizes[r0] * RB) + k1r_ring4);
        ring4 = true;
      }
    } else if ((max_log2G == 0 || use_ring) && kK1sEnabled && (r0 % GW) == 0 &&
               al(group_recs(r0) * RB) + k1s_ring <= smem_budget) {
      // K1s (exact mode): the row block staged as in K1, columns through each lane's
      // prefetch ring, 64 quarters = RG x C columns per pass
      int64_t rows_b = group_recs(r0) * RB;
      int lrg = 0;
      if (!kK1sRG1 && r0 + GW < M - 1 &&
          al(rows_b + group_recs(r0 + GW) * RB) + k1s_ring <= smem_budget) {
        rows_b += group_recs(r0 + GW) * RB;
        lrg = 1;
      }
      rows = GW << lrg;
      logG = 0;
      logC = LOGU - lrg;
      s_mode = 4;
      k1s_need = std::max(k1s_need, al(rows_b) + k1s_ring);
    } else {  // rows too long for shared memory: operands from L1/L2 (K1g)
      logG = std::min(max_log2G, 5);
      const int P = T >> logG;
      rows = P <= 64 ? GW : 32;
      logC = 0;
      while ((rows << (logC + 1)) <= P) ++logC;
    }
    int mode = smem ? 1 : (s_mode == 4 ? 4 : (rows == 1 ? 2 : 0));
    int64_t Rr = std::min<int64_t>(rows, M - r0);
    int64_t c_split = M;  // columns >= c_split of this row go to K1c
    if (mode == 2 && kK1cEnabled) {
      // the first column group small enough for K1c (group sizes fall along the sort)
      int64_t lo = (r0 + 1) / GW, hi = n_groups;
      int lcg, lg;
      bool one;
      int64_t nd;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (k1c_config(r0, mid, &lcg, &lg, &one, &nd)) hi = mid;
        else lo = mid + 1;
      }
      if (lo < n_groups) {
        c_split = std::max<int64_t>(r0 + 1, lo * GW);
        // items of about max_cols columns, each with the config of its own first group
        // (columns shorten along the sort, so later items stage more groups per chunk)
        const int64_t span_c = std::max<int64_t>(GW, (max_cols / GW) * GW);
        for (int64_t c0 = c_split; c0 < M; c0 = ((c0 / GW) * GW) + span_c) {
          const int64_t c1 = std::min<int64_t>(((c0 / GW) * GW) + span_c, M);
          k1c_config(r0, c0 / GW, &lcg, &lg, &one, &nd);
          k1c_need = std::max(k1c_need, nd);
          pcf_work_item w;
          w.row0 = (int32_t)r0;
          w.nrows = 1;
          w.col0 = (int32_t)c0;
          w.col1 = (int32_t)c1;
          w.logC = lcg | (one ? 0x100 : 0);
          w.log2G = lg;
          w.smem_mode = 3;
          const double cells = (double)(S[c1] - S[c0]) + (double)(c1 - c0) * sizes[r0];
          w.cost_hi = (int32_t)std::min(2.0e9, cells / 1048576.0);
          runs[1].push_back(w);
        }
      }
    }
    const int64_t c_end = mode == 2 ? c_split : M;
    // rows outside K1 stop at the next group boundary so that K1 can resume on an
    // aligned interleaved group
    if (!smem && (r0 % GW) != 0) Rr = std::min<int64_t>(Rr, GW - r0 % GW);
    const int C = 1 << logC;
    const int64_t span = std::max<int64_t>(C, (max_cols / C) * C);
    const int64_t rows_pts = S[r0 + Rr] - S[r0];
    for (int64_t c0 = r0 + 1; c0 < c_end; c0 += span) {
      const int64_t c1 = std::min<int64_t>(c0 + span, c_end);
      int i_logC = logC, i_logG = logG, i_mode = mode;
      bool i_single = single;
      if (kPerItem && (mode == 1 || mode == 4) && (r0 % GW) == 0) {
        // per-item K1 config: the row block's config was sized on its FIRST columns (the
        // longest: the sort is descending), but later items' columns are shorter, so more
        // of them fit per chunk -- a smaller merge-path split G (fewer co-rank searches and
        // partial sums per cell), or K1 instead of K1s for exact-mode items
        const int lrg = Rr > GW ? 1 : 0;
        const int64_t rows_b = group_recs(r0) * RB + (lrg ? group_recs(r0 + GW) * RB : 0);
        for (int lc = LOGU - lrg; lc >= 0; --lc) {
          const int lg = LOGU - lrg - lc;
          if (lg > max_log2G) break;
          const int64_t ce = std::min<int64_t>(c0 + ((int64_t)1 << lc), c1);
          // (the segment partials area is only touched when G > 1)
          const int64_t need2 = al(rows_b) + 2 * al((S[ce] - S[c0]) * RB + 32) + red_bytes(lg);
          if (need2 > smem_budget) continue;
          int nlc = lc, nlg = lg;
          bool nsingle = false;
          int64_t nneed = need2;
          if (lg >= kSingleMinLogG && long_walk(sizes[r0], sizes[c0], lg - 1)) {
            // one column buffer instead of two: the most columns that fit (2C, 4C, ...)
            // divide G accordingly, at the price of one exposed chunk copy per chunk
            for (int up = kSingleMaxUp; up >= 1; --up) {
              if (lg - up < 0) continue;
              const int64_t ce2 = std::min<int64_t>(c0 + ((int64_t)1 << (lc + up)), c1);
              const int64_t need1 = al(rows_b) + al((S[ce2] - S[c0]) * RB + 32) + red_bytes(lg - up);
              if (need1 <= smem_budget) {
                nlc = lc + up;
                nlg = lg - up;
                nsingle = true;
                nneed = need1;
                break;
              }
            }
          }
          // take it if it splits pairs less than the row block's config, keeps more lanes
          // busy, or double-buffers at the same split (for a K1s row block: whenever a full
          // 512-lane K1 config fits)
          const bool better =
              mode == 4 ? nlg == 0
                        : (nlg < logG || (nlg == logG && nlc > logC) ||  // fewer splits / more lanes
                           (nlg == logG && nlc == logC && single && !nsingle));  // 2 buffers
          if (better) {
            i_logC = nlc;
            i_logG = nlg;
            i_single = nsingle;
            i_mode = 1;
            need_max = std::max(need_max, nneed);
          }
          break;
        }
        if (max_log2G == 0 && kExactSingle && !(i_mode == 1 && i_logC == LOGU - lrg)) {
          // exact mode: a full 512-lane K1 chunk (64 / RG columns) in ONE buffer, where two
          // do not fit -- K1 instead of K1s, or all lanes instead of K1's idle quarters
          const int lc = LOGU - lrg;
          const int64_t ce = std::min<int64_t>(c0 + ((int64_t)1 << lc), c1);
          const int64_t need1 = al(rows_b) + al((S[ce] - S[c0]) * RB + 32) + red_bytes(0);
          if (need1 <= smem_budget) {
            i_logC = lc;
            i_logG = 0;
            i_single = true;
            i_mode = 1;
            need_max = std::max(need_max, need1);
          }
        }
      }
      pcf_work_item w;
      w.row0 = (int32_t)r0;
      w.nrows = (int32_t)Rr;
      w.col0 = (int32_t)c0;
      w.col1 = (int32_t)c1;
      w.logC = i_logC | (i_single ? 0x100 : 0) | (ring4 ? 0x200 : 0);
      w.log2G = i_logG;
      w.smem_mode = i_mode;
      const double cells = (double)Rr * (double)(S[c1] - S[c0]) + (double)(c1 - c0) * rows_pts;
      w.cost_hi = (int32_t)std::min(2.0e9, cells / 1048576.0);
      runs[i_mode == 1 ? 0 : (i_mode == 4 ? 2 : (i_mode == 2 ? 3 : 4))].push_back(w);
    }
    if (smem) need_max = std::max(need_max, best_need);
    r0 += Rr;
  }
  auto by_cost = [](const pcf_work_item& x, const pcf_work_item& y) {
    return x.cost_hi > y.cost_hi;
  };
  for (auto& r : runs) std::stable_sort(r.begin(), r.end(), by_cost);
  int64_t total = 0;
  for (auto& r : runs) total += (int64_t)r.size();
  *n_items = total;
  if (smem_bytes)
    *smem_bytes = (int32_t)std::max(std::max(need_max, k1r_need), std::max(k1c_need, k1s_need));
  if (items) {
    if (cap < total) {
      set_error("pcf_plan_pairwise: capacity %lld < %lld items", (long long)cap, (long long)total);
      return PCF_ERR_ARG;
    }
    pcf_work_item* dst = items;
    for (auto& r : runs) dst = std::copy(r.begin(), r.end(), dst);
  }
  return PCF_OK;
}

int pcf_fill_matrix(const void* recs_dev, const void* recs8_dev, const int64_t* soff_dev,
                    const int64_t* goff8_dev, const int32_t* perm_dev,
                    int64_t M, const pcf_work_item* items_dev, int64_t n_items,
                    int32_t smem_bytes, int32_t smem_mode, int32_t rec_bytes,
                    int32_t* counter_dev, int op,
                    double p, int apply_root, double a, double b, void* out_dev,
                    int out_is_f32, int64_t ld, unsigned long long* err_dev, void* stream) {
  if (n_items <= 0) return PCF_OK;
  if (!recs_dev || !soff_dev || !perm_dev || !items_dev || !counter_dev || !out_dev || !err_dev ||
      (smem_mode && (!recs8_dev || !goff8_dev)) ||
      ld < M || !pcf_op_ok(op) || !(a >= 0.0) || !(a < b) ||
      n_items > 0x7fffffff) {
    set_error("pcf_fill_matrix: bad arguments");
    return PCF_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(counter_dev, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return cuda_fail(e, "pcf_fill_matrix memset");
  FillArgs A;
  A.recs = recs_dev;
  A.recs8 = recs8_dev;
  A.soff = soff_dev;
  A.goff8 = goff8_dev;
  A.perm = perm_dev;
  A.M = M;
  A.items = items_dev;
  A.n_items = (int)n_items;
  A.counter = counter_dev;
  A.op = op;
  A.p = p;
  A.a = a;
  A.b = b;
  A.apply_root = apply_root;
  A.out = out_dev;
  A.out_f32 = out_is_f32;
  A.ld = ld;
  A.err = err_dev;
  A.smem_mode = smem_mode;
  A.smem_bytes = smem_bytes;
  A.rec_bytes = rec_bytes == 8 ? 8 : 16;
  A.num_sms = num_sms_current();
  e = launch_fill_tiles(A, st);
  return e == cudaSuccess ? PCF_OK : cuda_fail(e, "pcf_fill_matrix");
}

int pcf_fill_diagonal(const void* recs_dev, const int64_t* soff_dev, const int32_t* perm_dev,
                      int64_t M, int gram, double a, double b, void* out_dev, int out_is_f32,
                      int64_t ld, unsigned long long* err_dev, void* stream) {
  if (M <= 0) return PCF_OK;
  if (!recs_dev || !soff_dev || !perm_dev || !out_dev || !err_dev || ld < M) {
    set_error("pcf_fill_diagonal: bad arguments");
    return PCF_ERR_ARG;
  }
  cudaError_t e = launch_diag(recs_dev, soff_dev, perm_dev, M, gram, a, b, out_dev, out_is_f32,
                              ld, err_dev, (cudaStream_t)stream);
  return e == cudaSuccess ? PCF_OK : cuda_fail(e, "pcf_fill_diagonal");
}

int pcf_fill_rows(const void* recs_dev, const int64_t* soff_dev, const int32_t* inv_dev,
                  int64_t M, int64_t r0, int64_t r1, int op, double p, int apply_root,
                  int diag, double a, double b, void* slab_dev, int out_is_f32,
                  unsigned long long* err_dev, void* stream) {
  if (r1 <= r0) return PCF_OK;
  if (!recs_dev || !soff_dev || !inv_dev || !slab_dev || !err_dev || r0 < 0 || r1 > M ||
      !pcf_op_ok(op)) {
    set_error("pcf_fill_rows: bad arguments");
    return PCF_ERR_ARG;
  }
  RowsArgs A;
  A.recs = recs_dev;
  A.soff = soff_dev;
  A.inv = inv_dev;
  A.M = M;
  A.r0 = r0;
  A.r1 = r1;
  A.op = op;
  A.p = p;
  A.a = a;
  A.b = b;
  A.apply_root = apply_root;
  A.diag = diag;
  A.slab = slab_dev;
  A.out_f32 = out_is_f32;
  A.err = err_dev;
  cudaError_t e = launch_fill_rows(A, (cudaStream_t)stream);
  return e == cudaSuccess ? PCF_OK : cuda_fail(e, "pcf_fill_rows");
}

int pcf_pair_list(const void* recs_dev, const int64_t* soff_dev, const int64_t* pairs_dev,
                  int64_t npairs, int op, double p, double a, double b, double* res_dev,
                  void* stream) {
  if (npairs <= 0) return PCF_OK;
  if (!recs_dev || !soff_dev || !pairs_dev || !res_dev || !pcf_op_ok(op)) {
    set_error("pcf_pair_list: bad arguments");
    return PCF_ERR_ARG;
  }
  cudaError_t e = launch_pair_list(recs_dev, soff_dev, pairs_dev, npairs, op, p, a, b, res_dev,
                                   (cudaStream_t)stream);
  return e == cudaSuccess ? PCF_OK : cuda_fail(e, "pcf_pair_list");
}

// ------------------------------------------------------------------ host-buffer mirrors
namespace {
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t n) { return cudaMalloc(&p, n ? n : 16); }
};
}  // namespace

int pcf_integrate_pair_host(const double* ft, const double* fv, int64_t nf, const double* gt,
                            const double* gv, int64_t ng, double a, double b, int op, double p,
                            double* result) {
  if (!ft || !fv || !gt || !gv || !result || nf < 1 || ng < 1 || !pcf_op_ok(op)) {
    set_error("pcf_integrate_pair_host: bad arguments");
    return PCF_ERR_ARG;
  }
  // One pinned staging block and one device block per host thread, reused across calls:
  // [t: N][v: N][off: 3][perm: 2 x int32 + pad][pairs: 2] goes up in ONE copy, the pack
  // and the pair kernel run on the thread's stream, 8 bytes come back.
  struct PairWs {
    char* host = nullptr;
    char* dev = nullptr;
    size_t cap = 0;
    cudaStream_t st = nullptr;
    int device = -1;
    ~PairWs() {
      if (host) cudaFreeHost(host);
      if (dev) cudaFree(dev);
      if (st) cudaStreamDestroy(st);
    }
  };
  thread_local PairWs ws;
  const int64_t N = nf + ng;
  const size_t up = (size_t)N * 16 + 24 + 16 + 16;  // t, v, off, perm (padded), pairs
  const size_t rec_at = (up + 15) & ~(size_t)15;       // 16-byte records
  const size_t need = rec_at + (size_t)N * 16 + 8;     // + records + result
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return cuda_fail(e, "pcf_integrate_pair_host device");
  if (ws.device != dev) {
    if (ws.dev) cudaFree(ws.dev);
    if (ws.st) cudaStreamDestroy(ws.st);
    ws.dev = nullptr;
    ws.st = nullptr;
    ws.cap = 0;
    ws.device = dev;
  }
  if (!ws.st && (e = cudaStreamCreateWithFlags(&ws.st, cudaStreamNonBlocking)))
    return cuda_fail(e, "pcf_integrate_pair_host stream");
  if (ws.cap < need) {
    if (ws.host) cudaFreeHost(ws.host);
    if (ws.dev) cudaFree(ws.dev);
    ws.host = ws.dev = nullptr;
    ws.cap = 0;
    const size_t cap = std::max<size_t>(need, 1 << 16);
    if ((e = cudaHostAlloc((void**)&ws.host, cap, cudaHostAllocDefault)) ||
        (e = cudaMalloc((void**)&ws.dev, cap)))
      return cuda_fail(e, "pcf_integrate_pair_host alloc");
    ws.cap = cap;
  }
  double* ht = (double*)ws.host;
  double* hv = ht + N;
  int64_t* hoff = (int64_t*)(hv + N);
  int32_t* hperm = (int32_t*)(hoff + 3);
  int64_t* hpairs = (int64_t*)((char*)hperm + 16);
  memcpy(ht, ft, nf * 8);
  memcpy(ht + nf, gt, ng * 8);
  memcpy(hv, fv, nf * 8);
  memcpy(hv + nf, gv, ng * 8);
  hoff[0] = 0;
  hoff[1] = nf;
  hoff[2] = N;
  hperm[0] = 0;
  hperm[1] = 1;
  hpairs[0] = 0;
  hpairs[1] = 1;
  char* d = ws.dev;
  const double* dt = (const double*)d;
  const double* dv = dt + N;
  const int64_t* doff = (const int64_t*)(dv + N);
  const int32_t* dperm = (const int32_t*)(doff + 3);
  const int64_t* dpairs = (const int64_t*)((const char*)dperm + 16);
  void* drec = d + rec_at;
  double* dres = (double*)(d + rec_at + (size_t)N * 16);
  if ((e = cudaMemcpyAsync(d, ws.host, up, cudaMemcpyHostToDevice, ws.st)) ||
      (e = launch_pack(dt, dv, 0, doff, dperm, doff, 2, drec, nullptr, nullptr, ws.st)) ||
      (e = launch_pair_list(drec, doff, dpairs, 1, op, p, a, b, dres, ws.st)) ||
      (e = cudaMemcpyAsync(ws.host, dres, 8, cudaMemcpyDeviceToHost, ws.st)) ||
      (e = cudaStreamSynchronize(ws.st)))
    return cuda_fail(e, "pcf_integrate_pair_host");
  memcpy(result, ws.host, 8);
  return PCF_OK;
}

int pcf_sweep_cells(const void* recs_dev, const int64_t* soff_dev, int64_t s, int64_t q,
                    double a, double b, double* cells_dev, int64_t cap, int64_t* count_dev,
                    void* stream) {
  if (!recs_dev || !soff_dev || !cells_dev || !count_dev || s < 0 || cap < 0 || !(a >= 0.0) ||
      !(a < b)) {
    set_error("pcf_sweep_cells: bad arguments");
    return PCF_ERR_ARG;
  }
  cudaError_t e = launch_sweep_cells(recs_dev, soff_dev, s, q, a, b, cells_dev, cap, count_dev,
                                     (cudaStream_t)stream);
  return e == cudaSuccess ? PCF_OK : cuda_fail(e, "pcf_sweep_cells");
}

int pcf_fill_block_host(const double* tcat, const double* vcat, const int64_t* off, int64_t M,
                        int64_t r0, int64_t r1, int op, double p, int apply_root, int diag,
                        double a, double b, double* out, int64_t ld, int64_t* err_i,
                        int64_t* err_j) {
  if (err_i) *err_i = -1;
  if (err_j) *err_j = -1;
  if (!tcat || !vcat || !off || !out || M < 1 || r0 < 0 || r1 > M || ld < M) {
    set_error("pcf_fill_block_host: bad arguments");
    return PCF_ERR_ARG;
  }
  if (r1 <= r0) return PCF_OK;
  const int64_t N = off[M];
  std::vector<int32_t> ident(M);
  for (int64_t i = 0; i < M; ++i) ident[i] = (int32_t)i;
  const int64_t rows = r1 - r0;
  DevBuf dt, dv, doff, dperm, drec, dslab, derr;
  cudaError_t e;
  if ((e = dt.alloc(N * 8)) || (e = dv.alloc(N * 8)) || (e = doff.alloc((M + 1) * 8)) ||
      (e = dperm.alloc(M * 4)) || (e = drec.alloc(N * 16)) || (e = dslab.alloc(rows * M * 8)) ||
      (e = derr.alloc(8)))
    return cuda_fail(e, "pcf_fill_block_host alloc");
  cudaMemcpy(dt.p, tcat, N * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dv.p, vcat, N * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(doff.p, off, (M + 1) * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dperm.p, ident.data(), M * 4, cudaMemcpyHostToDevice);
  cudaMemset(derr.p, 0xff, 8);
  if ((e = launch_pack(dt.p, dv.p, 0, (int64_t*)doff.p, (int32_t*)dperm.p, (int64_t*)doff.p, M,
                       drec.p, nullptr, nullptr, 0)))
    return cuda_fail(e, "pcf_fill_block_host pack");
  RowsArgs A;
  A.recs = drec.p;
  A.soff = (int64_t*)doff.p;
  A.inv = (int32_t*)dperm.p;
  A.M = M;
  A.r0 = r0;
  A.r1 = r1;
  A.op = op;
  A.p = p;
  A.a = a;
  A.b = b;
  A.apply_root = apply_root;
  A.diag = diag;
  A.slab = dslab.p;
  A.out_f32 = 0;
  A.err = (unsigned long long*)derr.p;
  if ((e = launch_fill_rows(A, 0))) return cuda_fail(e, "pcf_fill_block_host kernel");
  std::vector<double> slab(rows * M);
  unsigned long long ekey = ~0ull;
  if ((e = cudaMemcpy(slab.data(), dslab.p, rows * M * 8, cudaMemcpyDeviceToHost)) ||
      (e = cudaMemcpy(&ekey, derr.p, 8, cudaMemcpyDeviceToHost)))
    return cuda_fail(e, "pcf_fill_block_host copy");
  // The reference stops at the first non-finite entry of the block (row-major) and
  // leaves the entries after it untouched; mirror that.
  const int64_t stop_i = ekey == ~0ull ? r1 : (int64_t)(ekey / M);
  const int64_t stop_j = ekey == ~0ull ? M : (int64_t)(ekey % M);
  for (int64_t i = r0; i < r1; ++i) {
    for (int64_t j = i + (diag ? 0 : 1); j < M; ++j) {
      if (i == stop_i && j == stop_j) goto done;
      const double x = slab[(i - r0) * M + j];
      out[i * ld + j] = x;
      out[j * ld + i] = x;
    }
  }
done:
  if (ekey != ~0ull) {
    if (err_i) *err_i = stop_i;
    if (err_j) *err_j = stop_j;
  }
  return PCF_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ FP64 peak probe
// Measures the dense FP64 FMA rate of this GPU (DFMA, 8 independent chains per thread,
// full occupancy).  bench.py uses it as the roofline denominator for the pairwise
// kernels, whose work is FP64-pipe / issue bound (no FP64 figure in MEASURED_PEAKS.json).
namespace pcfb {
__global__ void k_probe_dfma(double* out, int iters, double seed) {
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4,
         a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
    a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
  }
  const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;  // keep the work alive
}
}  // namespace pcfb

namespace pcfb {
__global__ void k_pow_batch(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                            double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = pcfpow::pow(x[i], y[i]);
}
}  // namespace pcfb

extern "C" int pcf_pow_batch(const double* x_dev, const double* y_dev, int64_t n,
                             double* out_dev, void* stream) {
  if (n < 0 || (n > 0 && (!x_dev || !y_dev || !out_dev))) {
    set_error("pcf_pow_batch: bad arguments");
    return PCF_ERR_ARG;
  }
  if (n == 0) return PCF_OK;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  pcfb::k_pow_batch<<<grid, 256, 0, (cudaStream_t)stream>>>(x_dev, y_dev, n, out_dev);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PCF_OK : cuda_fail(e, "pcf_pow_batch");
}

extern "C" int pcf_probe_fp64(double* out_dev, int iters, int blocks_per_sm, void* stream) {
  const int nsm = num_sms_current();
  pcfb::k_probe_dfma<<<nsm * blocks_per_sm, 256, 0, (cudaStream_t)stream>>>(out_dev, iters, 1.0);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PCF_OK : cuda_fail(e, "pcf_probe_fp64");
}
