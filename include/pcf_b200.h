/* pcf_b200.h -- C ABI of the B200 rectangle-iteration engine (libpcfb200.so).
 *
 * This is the drop-in boundary for the reference's kernel plugin.  The reference
 * selects a kernel module through pcflib._backend._Backend
 * (pkg/src/pcflib/_backend.py:25-49), whose three calls map onto this ABI as follows:
 *
 *   _Backend.integrate_pair(f, g, a, b, op, p)  _backend.py:31-38 -> pcf_integrate_pair_host
 *       (= _sweepkern.integrate_pair, _sweepkern.pyx:62-69)
 *   _Backend.pack(collection)                   _backend.py:40-41 -> pcf_collection_create
 *       (= _sweepkern.pack, _sweepkern.pyx:72-85; device-resident, size-sorted handle;
 *        pcf_pack_sorted is the device-pointer form)
 *   _Backend.fill_block(packed, r0, r1, ...)    _backend.py:43-46 -> pcf_collection_fill_block
 *       (= _sweepkern.fill_block, pyx:88-121; pcf_fill_rows / pcf_fill_block_host are the
 *        device-pointer and stateless host forms)
 *
 * plus the whole-matrix path the GPU needs (MatrixJob.run's block loop,
 * pkg/src/pcflib/matrix.py:156-234, moved on-device): pcf_plan_pairwise + pcf_fill_matrix,
 * and the reduction path that has no boundary in the reference (reduce.py:31-63,189-238):
 * pcf_tree_level / pcf_tree_merge_level(s) per level, pcf_finalize to finalise (the older
 * flag + compact pair pcf_scale_flag / pcf_std_flag + pcf_compact remains available).
 *
 * Conventions
 *  - All functions return PCF_OK (0) or an error code; pcf_last_error() gives the text.
 *    Nothing throws across the ABI.
 *  - "_dev" pointers are CUDA device pointers; `stream` is a cudaStream_t (NULL = legacy
 *    default).  Device-pointer entry points never allocate and never synchronise.
 *  - "_host" entry points take host arrays, allocate/free device memory internally and
 *    synchronise before returning (the reference's calling convention).
 *  - op: PCF_OP_LP (h = |x-y|^p) or PCF_OP_INNER (h = x*y): same codes as
 *    _sweepkern.OP_LP / OP_INNER (pyx:14-15).
 *  - Records: one PCF with rows (t_k, v_k), k < n, is n 16-byte records
 *    {double t_next, double v}; t_next = t_{k+1}, +inf for the last.  Collections are
 *    concatenated in size-sorted (descending) order with int64 offsets `soff`.
 *  - err_dev: one unsigned 64-bit word initialised by the caller to UINT64_MAX; receives
 *    atomicMin(i*M + j) of the first (row-major, original indices, i <= j) non-finite
 *    entry, i.e. the pair the reference's serial fill_block would report (pyx:109-112).
 */
#ifndef PCF_B200_H
#define PCF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCF_OK 0
#define PCF_ERR_ARG 1
#define PCF_ERR_CUDA 2
#define PCF_ERR_NOMEM 3
#define PCF_ERR_NONFINITE 4

#define PCF_OP_LP 0
#define PCF_OP_INNER 1
/* Flag or'ed into op: L_p cells with p != 1 may use d*d, d*d*|d| or CUDA's pow instead of
 * the default, the C library's pow restated bit for bit (csrc/pcf_pow.cuh), which makes
 * every p bitwise equal to the reference in the exact plan.  Roots always use the latter. */
#define PCF_OP_FAST_POW 0x10

/* One work item of the pairwise tile scheduler (32 bytes, device-resident array). */
typedef struct pcf_work_item {
  int32_t row0;      /* first size-sorted row of the row block */
  int32_t nrows;     /* rows in the block (K1: 8 or 16 = one or two interleaved groups) */
  int32_t col0;      /* first size-sorted column of this item */
  int32_t col1;      /* one past the last column */
  int32_t logC;      /* columns per streamed chunk = 1 << (logC & 0xff); bit 8: K1 streams
                        the columns through ONE buffer (twice the columns, half the G) */
  int32_t log2G;     /* merge-path segments per pair = 1 << log2G */
  int32_t smem_mode; /* 1: K1 shared-memory tiles, 3: K1c one resident long row against
                        streamed interleaved column groups, 2: K1r one resident long row,
                        4: K1s (exact mode) staged row groups, columns through L1,
                        0: K1g one lane per pair from L1/L2 (exact mode, long rows) */
  int32_t cost_hi;   /* estimated cells / 2^20 (scheduling order only) */
} pcf_work_item;

const char* pcf_version(void);
const char* pcf_last_error(void);
/* Threads per CTA the tile kernels are compiled for. */
int pcf_tile_threads(void);

/* ---- K3 sort-pack: reference pack() output (original order) -> sorted records ---- */
/* tcat/vcat: float32 (is_f32=1) or float64 SoA concatenations, off: int64[M+1] original
 * offsets, perm: int32[M] sorted->original, soff: int64[M+1] sorted offsets,
 * recs: 16*soff[M] bytes. */
int pcf_pack_sorted(const void* tcat_dev, const void* vcat_dev, int is_f32,
                    const int64_t* off_dev, const int32_t* perm_dev, const int64_t* soff_dev,
                    int64_t M, void* recs_dev, const int64_t* goff8_dev, void* recs8_dev,
                    void* stream);
/* Slot-interleaved copy used by K1's row blocks (recs8, optional: pass NULLs to skip):
 * record k of sorted PCF s lives at goff8[s/8] + 8k + s%8, so a quarter-warp reading the
 * 8 rows of one group always hits 8 distinct shared-memory bank groups.
 * goff8: int64[(M+7)/8 + 1], from pcf_group_offsets (host). */
int pcf_group_offsets(const int64_t* sizes_sorted, int64_t M, int32_t group, int64_t* goff);
/* float32 collections: 8-byte records {float t_next, float v} (the kernels widen them to
 * float64 after the shared-memory load, as the reference widens every operand):
 * recs32 = contiguous sorted records (allocate soff[M] + 2 records), recs32g = the
 * 16-row slot-interleaved copy (goff16 from pcf_group_offsets(..., 16, ...)). */
int pcf_pack_sorted32(const float* tcat_dev, const float* vcat_dev, const int64_t* off_dev,
                      const int32_t* perm_dev, const int64_t* soff_dev, int64_t M,
                      void* recs32_dev, const int64_t* goff16_dev, void* recs32g_dev,
                      void* stream);

/* ---- planner (host): sizes in sorted order -> work items, cost-descending ---- */
/* Returns the dynamic shared memory the items need in *smem_bytes.  `items` may be NULL
 * to query the count.  max_cols bounds the columns per item (load-balance granularity).
 * rec_bytes: 16 (float64 records, 8-row groups) or 8 (float32 records, 16-row groups).
 * max_log2G caps the merge-path split: 0 = one lane per pair everywhere, which sums every
 * entry strictly left to right exactly like the reference (bitwise for p=1 and INNER);
 * 6 = up to 64 segments per pair (fastest; same cell products, summed in G runs).
 * Items come in one contiguous, cost-descending run per kernel, in the order
 * K1 (smem_mode 1: 8/16-row groups + streamed columns resident in shared memory),
 * K1r (smem_mode 2: one row resident, columns from L1/L2),
 * K1g (smem_mode 0: rows too long for shared memory, operands from L1/L2);
 * launch pcf_fill_matrix once per run with that run's smem_mode. */
int pcf_plan_pairwise(const int64_t* sizes_sorted, int64_t M, int64_t smem_budget,
                      int64_t max_cols, int32_t max_log2G, int32_t rec_bytes,
                      pcf_work_item* items, int64_t cap, int64_t* n_items,
                      int32_t* smem_bytes);

/* ---- K1: whole upper triangle (diagonal excluded) of the pairwise matrix ---- */
/* out_dev: M x M row-major (leading dim ld) float64 (out_is_f32=0) or float32; entries
 * (perm[p], perm[q]) and mirror are written for every pair covered by items
 * [0, n_items).  counter_dev: int32 initialised to 0.  p: Lp exponent (ignored for
 * INNER).  apply_root: r = x^(1/p) as in pdist.  b may be +inf.  smem_mode: the run's
 * kernel (see pcf_plan_pairwise); smem_bytes: the planner's *smem_bytes. */
int pcf_fill_matrix(const void* recs_dev, const void* recs8_dev, const int64_t* soff_dev,
                    const int64_t* goff8_dev, const int32_t* perm_dev,
                    int64_t M, const pcf_work_item* items_dev, int64_t n_items,
                    int32_t smem_bytes, int32_t smem_mode, int32_t rec_bytes,
                    int32_t* counter_dev, int op,
                    double p, int apply_root, double a, double b, void* out_dev,
                    int out_is_f32, int64_t ld, unsigned long long* err_dev, void* stream);

/* Diagonal: Gram <f,f> (gram=1) or exact zeros for distances (gram=0). */
int pcf_fill_diagonal(const void* recs_dev, const int64_t* soff_dev, const int32_t* perm_dev,
                      int64_t M, int gram, double a, double b, void* out_dev, int out_is_f32,
                      int64_t ld, unsigned long long* err_dev, void* stream);

/* ---- fill_block mirror on device: rows [r0, r1) (original order), j > i (j >= i with
 * diag), written to a compact (r1-r0) x M slab.  inv_dev: original->sorted. ---- */
int pcf_fill_rows(const void* recs_dev, const int64_t* soff_dev, const int32_t* inv_dev,
                  int64_t M, int64_t r0, int64_t r1, int op, double p, int apply_root,
                  int diag, double a, double b, void* slab_dev, int out_is_f32,
                  unsigned long long* err_dev, void* stream);

/* Raw integrals (no root) of explicit sorted-index pairs; +-inf on divergence. */
int pcf_pair_list(const void* recs_dev, const int64_t* soff_dev, const int64_t* pairs_dev,
                  int64_t npairs, int op, double p, double a, double b, double* res_dev,
                  void* stream);

/* ---- host-buffer mirrors of the reference kernel module (synchronous) ---- */
/* _sweepkern.integrate_pair (pyx:62-69): raw integral, +-inf on divergence. */
int pcf_integrate_pair_host(const double* ft, const double* fv, int64_t nf, const double* gt,
                            const double* gv, int64_t ng, double a, double b, int op, double p,
                            double* result);
/* sweep.iterate_rectangles / iterate_segments (pkg/src/pcflib/sweep.py:67-116): the cells
 * of sorted PCFs s and q (q < 0: the segments of s alone) on [a, b), in order, as
 * cells_dev[4k..4k+3] = (l, r, v_f, v_g); *count_dev = number of cells (only the first
 * cap are written; cap = n_s + n_q suffices).  One device thread. */
int pcf_sweep_cells(const void* recs_dev, const int64_t* soff_dev, int64_t s, int64_t q,
                    double a, double b, double* cells_dev, int64_t cap, int64_t* count_dev,
                    void* stream);

/* _sweepkern.fill_block (pyx:88-121) on host arrays: tcat/vcat/off = pack() output
 * (float64), out = host M x M (ld) float64, rows [r0,r1).  *err_i/*err_j = -1 or the
 * first non-finite pair. */
int pcf_fill_block_host(const double* tcat, const double* vcat, const int64_t* off, int64_t M,
                        int64_t r0, int64_t r1, int op, double p, int apply_root, int diag,
                        double a, double b, double* out, int64_t ld, int64_t* err_i,
                        int64_t* err_j);

/* ---- kernel-plugin handle: _Backend.pack / fill_block (pkg/src/pcflib/_backend.py:40-46,
 * _sweepkern.pack / fill_block pyx:72-121) for a plugin inside the reference's MatrixJob
 * (matrix.py:169-227: pack once, fill_block on disjoint row blocks from many threads).
 * pcf_collection_create uploads the pack() layout (tcat/vcat float64, or float32 when
 * is_f32; off int64[M+1]) once and packs it size-sorted on the current device.
 * pcf_collection_fill_block writes rows [r0, r1) (j >= i with diag, else j > i) and their
 * mirrors into the host matrix `out` (float64, or float32 when out_is_f32; leading
 * dimension ld) exactly as _sweepkern.fill_block does: returns with *err_i/*err_j = the
 * block's first non-finite entry in row-major order (-1 if none), entries after it
 * untouched.  The first call for a given (op, p, apply_root, diag, a, b, max_log2G)
 * computes the whole matrix on the device with the tile kernels and caches it on the
 * handle (float64); every call copies its rows from that cache.  max_log2G 0 = exact plan
 * (bitwise equal to pcf_integrate_pair_host and to the reference for every p), > 0 = fast
 * plan.  Thread-safe: concurrent fill_block calls on one handle are allowed. */
int pcf_collection_create(const void* tcat, const void* vcat, int is_f32, const int64_t* off,
                          int64_t M, void** handle);
void pcf_collection_free(void* handle);
int pcf_collection_fill_block(void* handle, int64_t r0, int64_t r1, int op, double p,
                              int apply_root, int diag, double a, double b, int32_t max_log2G,
                              void* out, int out_is_f32, int64_t ld, int64_t* err_i,
                              int64_t* err_j);

/* Whole matrix from host buffers (serialised per process): MatrixJob.run over the compiled module
 * (pkg/src/pcflib/matrix.py:156-234 -> pack, fill_block per row block; pyx:72-121) in one
 * call.  tcat/vcat/off: the reference pack() layout in host memory (float64, or float32
 * when is_f32); out: host M x M (leading dimension ld) of the same kind, written in
 * original order (diagonal: exact 0 for LP, <f,f> for INNER when diag).  The work queue
 * sweeps the column ranges right to left in max(n_chunks, 512) cost-balanced chunks; the
 * rows each chunk finishes are copied to `out` on internal copy streams while later chunks
 * compute (pin `out` with cudaHostRegister / cudaMallocHost for the copies to overlap).
 * max_log2G as in
 * pcf_plan_pairwise.  *err_i/*err_j = -1, or the first (row-major, i < j) non-finite
 * pair.  Compute runs on `stream` (NULL: an internal stream), copies on internal
 * streams joined back into it; synchronises before returning.  Device buffers are cached
 * between calls (pcf_release_workspace frees them). */
int pcf_matrix_host(const void* tcat, const void* vcat, int is_f32, const int64_t* off,
                    int64_t M, int op, double p, int apply_root, int diag, double a, double b,
                    int32_t max_log2G, int32_t n_chunks, void* out, int64_t ld, int64_t* err_i,
                    int64_t* err_j, void* stream);
void pcf_release_workspace(void);

/* ---- user combination integrals (CombinationIntegral, combine_integrate(_timedep),
 * integrate_single, pairwise: pkg/src/pcflib/integrate.py:51-203, matrix.py:273-283).
 * `defs` = C definitions generated from the Python integrand (jit.py): PCF_MODE (0: h(x,y),
 * 1: antiderivative H(x,y,t)), PCF_HAS_R, PCF_HAS_U and the __device__ functions pcf_h /
 * pcf_H / pcf_r / pcf_u.  NVRTC compiles them with the kernel template
 * (csrc/pcf_jit_kernels.cuh) for sm_100a with --fmad=false.
 * pcf_jit_cubin: compile only (no GPU needed); pcf_jit_load: compile + load a module.
 * Each entry is walked by one thread in the reference's cell order (sweep.py:67-116).
 * Status per entry: 0 ok, 1 divergent tail, 2 non-finite.  errs_dev[2] (init UINT64_MAX):
 * atomicMin of the row-major original-index key of the first divergent / non-finite entry. */
int pcf_jit_cubin(const char* defs, void* cubin_out, int64_t cap, int64_t* size, char* log,
                  int64_t logcap);
int pcf_jit_load(const char* defs, void** module, char* log, int64_t logcap);
void pcf_jit_release(void* module);
/* sorted rows [r0, r1) x columns (sym: q >= s, mirrored; else all q) -> out (original order) */
int pcf_jit_matrix(void* module, const void* recs_dev, const int64_t* soff_dev,
                   const int32_t* perm_dev, int64_t M, int sym, double a, double b,
                   void* out_dev, int out_f32, int64_t ld, int64_t r0, int64_t r1,
                   unsigned long long* errs_dev, void* stream);
/* explicit (sorted-index) pairs -> value after rounding to the kind and r, status */
int pcf_jit_pairs(void* module, const void* recs_dev, const int64_t* soff_dev,
                  const int64_t* pairs_dev, int64_t npairs, double a, double b, int out_f32,
                  double* res_dev, int32_t* status_dev, void* stream);
/* The tile kernels K1 / K1c / K1r / K1g / K1s (pcf_fill_matrix) instantiated for a user
 * integrand h (PCF_MODE 0, declared symmetric): NVRTC compiles csrc/pcf_tiles.cuh with
 * h in place of |x - y|^p and r in place of the p-th root, for one record kind
 * (is_f32: 8-byte float32 records, float output).  Replaces the per-rectangle Python
 * callback of the reference's custom-integral matrix (pkg/src/pcflib/matrix.py:184-196).
 * Fills the strict upper triangle of the plan's pairs, mirrored (the diagonal is the
 * caller's: pcf_jit_pairs on (s, s)); err_dev (init UINT64_MAX): atomicMin of the
 * (min, max) original-index key of the first non-finite / divergent entry. */
int pcf_jit_tiles_cubin(const char* defs, int is_f32, int64_t* size, char* log, int64_t logcap);
int pcf_jit_tiles_load(const char* defs, int is_f32, void** module, char* log, int64_t logcap);
void pcf_jit_tiles_release(void* module);
int pcf_jit_fill_tiles(void* module, int smem_mode, const void* recs_dev, const void* recsg_dev,
                       const int64_t* soff_dev, const int64_t* goff_dev, const int32_t* perm_dev,
                       int64_t M, const void* items_dev, int64_t n_items, int32_t smem_bytes,
                       int32_t* counter_dev, int has_r, double a, double b, void* out_dev,
                       int64_t ld, unsigned long long* err_dev, void* stream);
/* integrate_single of every (sorted) PCF with pcf_u */
int pcf_jit_single(void* module, const void* recs_dev, const int64_t* soff_dev, int64_t M,
                   double a, double b, int out_f32, double* res_dev, int32_t* status_dev,
                   void* stream);

/* out[i] = pow(x[i], y[i]) with the device restatement of the C library's pow that every
 * L_p kernel uses (csrc/pcf_pow.cuh; bit-identical to glibc 2.39 libm pow, the reference's
 * pow at _sweepkern.pyx:43-46,98,114).  For verification and for host callers that want
 * the same rounding on the device. */
int pcf_pow_batch(const double* x_dev, const double* y_dev, int64_t n, double* out_dev,
                  void* stream);

/* Dense FP64 FMA throughput probe: nsm*blocks_per_sm CTAs x 256 threads x 8 chains x iters
 * DFMA (2 flops each); time it with events on `stream` for the FP64 roofline. */
int pcf_probe_fp64(double* out_dev, int iters, int blocks_per_sm, void* stream);

/* ---- reduction path (mean / std / tree_reduce; pcf_level.cu, pcf_reduce.cu) ----
 * The reference has no kernel boundary here (reduce.py:31-63,189-238 call the Python
 * sweep directly); these entry points are the device replacement.  A tree level maps
 * nodes (SoA times/values, int64 offsets) to output nodes: output k merges input nodes
 * src[k], src[k]+1 (cnt[k]=2) or passes src[k] through (cnt[k]=1).
 * pcf_compact: exclusive scan of keep flags (ntot candidates, tiled; no library scan) +
 * scatter of the kept points + output node offsets (after pcf_scale_flag / pcf_std_flag;
 * pcf_finalize does flag + compact in one call without the flag arrays). */
int pcf_scan_workspace(int64_t ntot, int64_t* bytes);
/* value_bytes: element size of sv/sv2 (4 or 8); sv2 may be NULL. */
int pcf_compact(int is_f32, const void* st_dev, const void* sv_dev, const void* sv2_dev,
                int value_bytes, const int32_t* flag_dev, int64_t ntot, const int64_t* off_in_dev,
                const int64_t* src_dev, int64_t nout, int64_t* pos_dev, void* temp_dev,
                int64_t temp_bytes, void* t_out_dev, void* v_out_dev, void* v2_out_dev,
                int64_t* off_out_dev, void* stream);
/* Whole tree level, tiled single pass (stage windows -> merge walk with reduce_pair's keep
 * flags -> block scan -> decoupled look-back -> coalesced writes).  kind 0..3 = add/max/min/mul on v (the PCFs' kind); 4 = moments
 * (v = mean, v2 = M2, both float64; leaves_dev = leaf counts per input node).  Writes
 * t_out/v_out(/v2_out) and off_out[nout+1]; workspace from pcf_tree_level_workspace. */
int pcf_tree_level_workspace(int64_t ntot, int64_t* bytes);
int pcf_tree_level(int kind, int is_f32, const void* t_dev, const void* v_dev,
                   const double* v2_dev, const int64_t* off_dev, const int64_t* src_dev,
                   const int32_t* cnt_dev, const int64_t* leaves_dev, int64_t nout,
                   int64_t ntot, void* t_out_dev, void* v_out_dev, double* v2_out_dev,
                   int64_t* off_out_dev, void* ws_dev, int64_t ws_bytes, int32_t* status_dev,
                   void* stream);
/* Non-compacting level for (nearly) distinct breakpoint times: the same merge, every
 * candidate kept at its own input position (node offsets unchanged).  A time present in
 * both children yields a zero-width piece followed by the exact point; the finalisation
 * drops zero-width pieces when given the times (t_dev below).  Same workspace. */
int pcf_tree_merge_level(int kind, int is_f32, const void* t_dev, const void* v_dev,
                         const double* v2_dev, const int64_t* off_dev, const int64_t* src_dev,
                         const int32_t* cnt_dev, const int64_t* leaves_dev, int64_t nout,
                         int64_t ntot, void* t_out_dev, void* v_out_dev, double* v2_out_dev,
                         int64_t* off_out_dev, void* ws_dev, int64_t ws_bytes, void* stream);
/* Several non-compacting merge levels in one pass (K5w, csrc/pcf_wmerge.cu): output node q
 * of the last level combines the nlev-level subtree over input nodes
 * [nfirst[q], nfirst[q] + ncnt[q]) (ncnt <= 2^nlev, nlev <= 4) in the reference tree shape
 * (reduce.py:189-208), bit-identical to nlev successive pcf_tree_merge_level calls.
 * leaves_dev: leaf count per INPUT node (kind 4 only).  Workspace from
 * pcf_tree_merge_levels_workspace. */
int pcf_tree_merge_levels_workspace(int64_t ntot, int64_t nout, int64_t* bytes);
int pcf_tree_merge_levels(int kind, int is_f32, const void* t_dev, const void* v_dev,
                          const double* v2_dev, const int64_t* off_dev,
                          const int64_t* nfirst_dev, const int32_t* ncnt_dev,
                          const int64_t* leaves_dev, int64_t nout, int32_t nlev, int64_t ntot,
                          void* t_out_dev, void* v_out_dev, double* v2_out_dev,
                          int64_t* off_out_dev, void* ws_dev, int64_t ws_bytes, void* stream);
/* Equal-time coincidences between neighbouring nodes (2p, 2p+1) of a level, over nsample
 * pairs spread across it: counts[0] = coincidences, counts[1] = points examined.  Lets the
 * host run a tree non-compacting from level 0 when breakpoints are nearly distinct. */
int pcf_tree_dup_sample(int is_f32, const void* t_dev, const int64_t* off_dev, int64_t nnodes,
                        int32_t nsample, unsigned long long* counts_dev, void* stream);
/* Whole finalisation of a reduction tree's root level(s) in two tiled passes (no flag or
 * scaled-value arrays in HBM): kind 0 = mean, v * T(scale[seg]) (core.scale + the final
 * minimize_discretization, reduce.py:211-217); kind 1 = variance T(M2 * scale[seg]);
 * kind 2 = std, T(sqrt(variance)) (reduce.py:220-238).  Zero-width pieces of non-compacting
 * levels (equal times within a node) are dropped first.  src_dev: v (kind 0) or M2
 * (float64, kinds 1-2); t_dev/off_dev: the level; nseg nodes.  Writes the kept points to
 * t_out/v_out (record kind) and off_out[nseg+1]; status |= 1 on a non-finite value.
 * Workspace from pcf_finalize_workspace. */
int pcf_finalize_workspace(int64_t ntot, int64_t* bytes);
int pcf_finalize(int kind, int is_f32, const void* src_dev, const void* t_dev,
                 const int64_t* off_dev, int64_t nseg, const double* scale_dev, int64_t ntot,
                 void* t_out_dev, void* v_out_dev, int64_t* off_out_dev, int32_t* status_dev,
                 void* ws_dev, int64_t ws_bytes, void* stream);
/* mean finalisation: v * T(scale[seg]) (core.scale) + keep-where-changed flags.
 * t_dev (optional): the node times; zero-width pieces (next point of the node at the same
 * time) get flag 0 and survivors compare with the previous survivor. */
int pcf_scale_flag(int is_f32, const void* v_dev, const void* t_dev, const int64_t* off_dev,
                   int64_t nseg, const double* scale_dev, int64_t ntot, void* sv_dev,
                   int32_t* flag_dev, int32_t* status_dev, void* stream);
/* variance / std finalisation from M2: T(M2 * scale[seg]) [then T(sqrt(.))] + flags;
 * t_dev as for pcf_scale_flag. */
int pcf_std_flag(int is_f32, int take_sqrt, const double* m2_dev, const void* t_dev,
                 const int64_t* off_dev, int64_t nseg, const double* scale_dev, int64_t ntot,
                 void* sv_dev, int32_t* flag_dev, int32_t* status_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PCF_B200_H */
