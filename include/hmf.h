/*
 * libhmf — C ABI of the B200-native SGD matrix-factorization hot path.
 *
 * Every entry point takes plain pointers and sizes (no torch types).  Device
 * pointers must be CUDA device memory on the current device; `stream` is a
 * cudaStream_t (NULL = legacy default stream).  All kernels are asynchronous
 * and stream-ordered; nothing here frees caller memory.
 *
 * Reference interface replaced by each entry point (paths relative to
 * /root/reference/pkg/src/hetmf/):
 *
 *   hmf_sgd_range_{f32,f16,f64}   kernels.sgd_range            kernels.py:61-133
 *   hmf_sgd_block_qband_{f32,f16} BatchEngine.compute on a staged item band
 *   hmf_sgd_block_qband_u16_*     (the same, uint16 tile-relative row ids)
 *   hmf_sgd_block_qband_u16_tiles_*  (the same over several row tiles)
 *   hmf_sgd_block_runs_{,u16_,u8_}*
 *                                 (the same, P tile in shared memory)
 *                                                              workers.py:186-255
 *   hmf_lease_*                   GridScheduler.acquire / release / abort for
 *                                 column units across GPU processes
 *                                                              scheduler.py:333-423
 *   hmf_qband_resolve_*, _slots_per_sm, _chain_lanes, _max_items
 *                                 (layout queries; no reference counterpart)
 *   hmf_visit_order               sgd_range's visit order      kernels.py:77-119
 *   hmf_mix64                     kernels.mix64                kernels.py:32-48
 *   hmf_residual_sums_{f32,f16,f64}
 *                                 sgd.rmse / sgd.regularized_loss
 *                                                              sgd.py:134-188
 *   hmf_memcpy_peer_async, hmf_ipc_*
 *                                 BatchEngine.stage_in/stage_out item-band copies
 *                                                              workers.py:186-218
 *   hmf_bucket_triples            data.build_grid bucketing    data.py:238-280
 *   hmf_synthetic_{count,cells,fill}
 *                                 data.synthetic_ratings law   data.py:311-336
 *
 * Return convention: int64 entry points return a count >= 0 on success and a
 * negative HMF_ERR_* code on failure; int entry points return HMF_OK (0) or a
 * negative code.  hmf_last_error() gives the message of the calling thread's
 * last failure.  The reference's sgd_range raises nothing and returns 0 for an
 * empty range (kernels.py:74-76); so does hmf_sgd_range_*.
 */
#ifndef HMF_H_
#define HMF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ABI 4: launch options per call (hmf_qband_opts).  ABI 5: implementation 7
 * (hmf_sgd_block_ptile_*, hmf_ptile_bins_per_tile) removed;
 * hmf_runs_chains_per_warp takes the element size; hmf_lease_claim added;
 * hmf_qband_opts.runs_wide. */
#define HMF_ABI_VERSION 5

#define HMF_OK 0
#define HMF_ERR_ARG (-1)
#define HMF_ERR_CUDA (-2)
#define HMF_ERR_UNSUPPORTED (-3)
#define HMF_ERR_ABORTED (-4) /* the multi-GPU run was aborted (hmf_lease_abort) */

/* Visit-order modes of hmf_sgd_range_*. */
#define HMF_MODE_HOGWILD 0     /* throughput: many warps, lock-free delta reductions */
#define HMF_MODE_ORDERED 1     /* reference visit order, one warp, fp32 arithmetic   */
#define HMF_MODE_EXACT 2       /* reference visit order, f64 reference arithmetic   */
#define HMF_MODE_HOGWILD_LWW 3 /* HOGWILD with plain stores (last writer wins)      */

/* Reference visit-order window (kernels.py:24). */
#define HMF_SHUFFLE_WINDOW 4096

int hmf_abi_version(void);
const char* hmf_last_error(void);

/* Tuning knobs (benchmark sweeps).  HMF_TUNE_VARIANT selects the HOGWILD
 * kernel's ILP / block-shape variant (0..7, -1 = per-shape default) for f32 and
 * f16 storage. */
#define HMF_TUNE_VARIANT 1
int hmf_set_tuning(int32_t key, int32_t value);

/*
 * One SGD pass over triples [start, stop) — kernels.sgd_range (kernels.py:61-133).
 *
 * user_f: (rows of the band) x k row-major factors, indexed rows[i] - row_base.
 * item_f: (cols of the band) x k row-major factors, indexed cols[i] - col_base.
 * rows/cols/vals: triple arrays (device); only [start, stop) is touched.
 * Updates user_f/item_f in place; returns stop - start (0 if empty) or < 0.
 * seed: the per-block order seed (workers.block_order_seed, workers.py:77-83).
 * In HOGWILD mode the seed permutes the chunk visit order; in ORDERED/EXACT
 * modes it drives the reference windowed Fisher-Yates order exactly.
 */
int64_t hmf_sgd_range_f32(float* user_f, float* item_f, int64_t k, const int32_t* rows,
                          const int32_t* cols, const float* vals, int64_t start, int64_t stop,
                          double lr, double reg_user, double reg_item, uint64_t seed,
                          int64_t row_base, int64_t col_base, int32_t mode, void* stream);

/* fp16 storage (IEEE binary16 bits), fp32 arithmetic, f32 ratings. */
int64_t hmf_sgd_range_f16(uint16_t* user_f, uint16_t* item_f, int64_t k, const int32_t* rows,
                          const int32_t* cols, const float* vals, int64_t start, int64_t stop,
                          double lr, double reg_user, double reg_item, uint64_t seed,
                          int64_t row_base, int64_t col_base, int32_t mode, void* stream);

/* f64 storage and f64 ratings (the reference's own storage type). */
int64_t hmf_sgd_range_f64(double* user_f, double* item_f, int64_t k, const int32_t* rows,
                          const int32_t* cols, const double* vals, int64_t start, int64_t stop,
                          double lr, double reg_user, double reg_item, uint64_t seed,
                          int64_t row_base, int64_t col_base, int32_t mode, void* stream);

/*
 * Q-band-stationary update of one block (the engine's fast path,
 * BatchEngine.compute on a staged item band, workers.py:186-266): the block's
 * triples are bucketed into n_sub column sub-bands (stable), sub-band s being
 * triples [sub_ptr[s], sub_ptr[s+1]) whose items lie in [sub_cuts[s],
 * sub_cuts[s+1]) (absolute item ids; device arrays).  A warp (implementation
 * 0) or a lane-group chain (4-6) owns a sub-band: the current item's Q row
 * stays on chip (exact sequential SGD on Q), P changes go back by vector
 * reductions or plain stores.  k in {32, 64, 128, 256}; ratings are f32.
 * Same update rule and indexing (row_base / col_base) as hmf_sgd_range_*.
 * Returns 0 or < 0.
 *
 * Row tiles: with n_tiles > 1 the block's triples are bucketed tile-major
 * (n_tiles row tiles x n_sub sub-bands, sub_ptr holding n_tiles*n_sub + 1
 * offsets); tile t's sub-band s is [sub_ptr[t*n_sub+s], sub_ptr[t*n_sub+s+1]).
 * The launch walks the tiles in a seeded rotation so that one tile's P rows
 * stay resident in L2.
 *
 * Every launch-shaping choice is an argument (ABI version 4): `opts` (NULL =
 * all defaults) is read during the call only.  Nothing is process-global, so
 * threads launching different layouts concurrently do not interfere.
 */
typedef struct hmf_qband_opts {
  /* Implementation: -1 = default (5); 0 = one warp per rating on its
   * sub-band's Q rows in shared memory (each sub-band at most
   * hmf_qband_max_items(k, f16, 0) items); 4 = chained item runs (several
   * lane-group chains per warp, the item's Q row in registers; whole runs
   * per sub-band); 5 = 4 with Q deltas: runs of one item may be split over
   * chains, each adds its change back with vector reductions and re-reads the
   * row every `qsync` ratings (bounded staleness); 6 = 5 publishing only at
   * item and bin changes; 8 = run groups over a tile-resident P
   * (hmf_sgd_block_runs_* only; 7, item bins over that tile, was removed in
   * ABI 5: run groups beat it at every k). */
  int32_t impl;
  /* Chained-kernel configuration 2, 4, 5 or 6 (lanes per chain, prefetch
   * distance, occupancy); -1 = by k and storage
   * (hmf_qband_resolve_chain_cfg). */
  int32_t chain_cfg;
  /* P write-back of the chained kernel: -1/0 vector reductions of the change
   * (no update lost), 1 plain stores of the updated row (fp32 rows with
   * configuration 5 or 6; reductions elsewhere) — the reference's racing-lane
   * semantics (workers.py:222-266): a concurrent update of the same user by
   * another chain may be lost. */
  int32_t pstore;
  /* Implementation 5: ratings between Q-delta publications; -1 = 32, 0 =
   * only at item and bin changes. */
  int32_t qsync;
  /* -1/1: the launch may fill the GPU; d in 2..64: its grid is capped at 1/d
   * of the resident CTA slots, so d launches on separate streams (several
   * column blocks of one row band) run side by side. */
  int32_t grid_share;
  /* Chains of a warp change bins together: bit 0 static, bit 1 dynamic
   * scheduler; -1 = 3. */
  int32_t lockstep;
  /* Implementation 8 at k = 32: 1 = more run-group chains per SM (fp32: 20
   * warps; fp16: 2-lane chains), 8-12 % faster but each item's Q changes
   * land staler — data.bucket_qbands sets it only under the staleness
   * bound; -1 / 0 = the default 128 chains per SM.  Ignored elsewhere. */
  int32_t runs_wide;
} hmf_qband_opts;

/* Default implementation / chain configuration for k and storage. */
int32_t hmf_qband_resolve_impl(int64_t k, int32_t f16);
int32_t hmf_qband_resolve_chain_cfg(int64_t k, int32_t f16);
/* Sub-band slots per SM of the launch `opts` describes (warps for
 * implementation 0, chains for 4-6); needs a current CUDA device (per-device
 * occupancy).  f16 != 0 for fp16 storage. */
int32_t hmf_qband_slots_per_sm(int64_t k, int32_t f16, const hmf_qband_opts* opts);
/* Lanes per chain of configuration cfg (-1: the default) at k. */
int32_t hmf_qband_chain_lanes(int64_t k, int32_t f16, int32_t cfg);
/* Items one sub-band may span under implementation impl (1<<30: unbounded;
 * 0: k unsupported). */
int32_t hmf_qband_max_items(int64_t k, int32_t f16, int32_t impl);

/* cols may be NULL with implementations 4-6 when every sub-band is a single
 * item (sub_cuts[s+1] = sub_cuts[s] + 1): the item of sub-band s is then
 * sub_cuts[s] (8 instead of 12 bytes per rating on a host stream). */
int64_t hmf_sgd_block_qband_f32(float* user_f, float* item_f, int64_t k, const int32_t* rows,
                                const int32_t* cols, const float* vals, const int64_t* sub_ptr,
                                const int32_t* sub_cuts, int64_t n_sub, int64_t n_tiles,
                                const hmf_qband_opts* opts, double lr, double reg_user,
                                double reg_item, uint64_t seed, int64_t row_base, int64_t col_base,
                                void* stream);
int64_t hmf_sgd_block_qband_f16(uint16_t* user_f, uint16_t* item_f, int64_t k,
                                const int32_t* rows, const int32_t* cols, const float* vals,
                                const int64_t* sub_ptr, const int32_t* sub_cuts, int64_t n_sub,
                                int64_t n_tiles, const hmf_qband_opts* opts, double lr,
                                double reg_user, double reg_item, uint64_t seed, int64_t row_base,
                                int64_t col_base, void* stream);

/* The chained kernel (implementations 4-6) with uint16 row ids: row =
 * rows[i] - row_base, so a row tile of at most 65536 rows streams 2-byte ids
 * with row_base = -(the tile's first row).  Same contract as
 * hmf_sgd_block_qband_*. */
int64_t hmf_sgd_block_qband_u16_f32(float* user_f, float* item_f, int64_t k,
                                    const uint16_t* rows, const int32_t* cols, const float* vals,
                                    const int64_t* sub_ptr, const int32_t* sub_cuts, int64_t n_sub,
                                    int64_t n_tiles, const hmf_qband_opts* opts, double lr,
                                    double reg_user, double reg_item, uint64_t seed,
                                    int64_t row_base, int64_t col_base, void* stream);
int64_t hmf_sgd_block_qband_u16_f16(uint16_t* user_f, uint16_t* item_f, int64_t k,
                                    const uint16_t* rows, const int32_t* cols, const float* vals,
                                    const int64_t* sub_ptr, const int32_t* sub_cuts, int64_t n_sub,
                                    int64_t n_tiles, const hmf_qband_opts* opts, double lr,
                                    double reg_user, double reg_item, uint64_t seed,
                                    int64_t row_base, int64_t col_base, void* stream);

/* uint16 row ids over n_tiles row tiles in one launch: a rating of tile t
 * updates row tile_row0[t] + rows[i] (tile_row0: device int32[n_tiles], the
 * tiles' first rows in user_f).  Lets a host stream stage several tiles of a
 * block as one chunk at 2 bytes per user id.  Same contract as
 * hmf_sgd_block_qband_u16_* otherwise (there is no row_base). */
int64_t hmf_sgd_block_qband_u16_tiles_f32(float* user_f, float* item_f, int64_t k,
                                          const uint16_t* rows, const int32_t* cols,
                                          const float* vals, const int64_t* sub_ptr,
                                          const int32_t* sub_cuts, int64_t n_sub, int64_t n_tiles,
                                          const int32_t* tile_row0, const hmf_qband_opts* opts,
                                          double lr, double reg_user, double reg_item,
                                          uint64_t seed, int64_t col_base, void* stream);
int64_t hmf_sgd_block_qband_u16_tiles_f16(uint16_t* user_f, uint16_t* item_f, int64_t k,
                                          const uint16_t* rows, const int32_t* cols,
                                          const float* vals, const int64_t* sub_ptr,
                                          const int32_t* sub_cuts, int64_t n_sub, int64_t n_tiles,
                                          const int32_t* tile_row0, const hmf_qband_opts* opts,
                                          double lr, double reg_user, double reg_item,
                                          uint64_t seed, int64_t col_base, void* stream);

/* Rows of one P tile in shared memory for the run-group kernel (208 KB of
 * P rows: 416 users at fp32 k = 128). */
int32_t hmf_ptile_max_rows(int64_t k, int32_t f16);

/*
 * Run groups over a tile-resident P (implementation 8): the block's users cut
 * into n_tiles row tiles (tile t = rows [tile_cut[t], tile_cut[t+1]) of
 * user_f, absolute indices, i.e. rows[i] - row_base; device int32[n_tiles +
 * 1]; at most max_tile_rows rows <= hmf_ptile_max_rows(k, f16)); inside a
 * tile the ratings are grouped into runs (all ratings of one item, in the
 * block's order), runs sorted by
 * length, longest first.  runs: int32[n_runs][4] descriptors, 16-byte
 * aligned; run r = {first, len, item, r} holds ratings [first, first + len)
 * of rows / vals (offsets relative to those pointers), all of item `item`
 * (absolute, minus col_base); tile t's runs are [tile_run[t],
 * tile_run[t+1]).  Device arrays; data.bucket_qbands with impl 8 builds
 * them.  A persistent CTA per SM holds one tile's P rows in shared memory; each warp takes groups of hmf_runs_chains_per_warp(k, f16)
 * consecutive runs, one per lane-group chain, the item's Q row in registers,
 * Q changes added back by vector reductions at the run's end.  rows: int32
 * user ids (minus row_base), or with the _u16 entry points uint16 ids
 * relative to the tile (tiles of at most 65536 rows; the streamed form:
 * 6 bytes per rating, items implicit in the runs).  opts.impl must be -1 or
 * 8; grid_share applies.  Same update rule and return convention as
 * hmf_sgd_block_qband_*.
 */
int32_t hmf_runs_chains_per_warp(int64_t k, int32_t f16);
int64_t hmf_sgd_block_runs_f32(float* user_f, float* item_f, int64_t k, const int32_t* rows,
                               const float* vals, const int32_t* runs, const int32_t* tile_run,
                               const int32_t* tile_cut, int64_t n_tiles, int32_t max_tile_rows,
                               const hmf_qband_opts* opts, double lr, double reg_user,
                               double reg_item, uint64_t seed, int64_t row_base, int64_t col_base,
                               void* stream);
int64_t hmf_sgd_block_runs_f16(uint16_t* user_f, uint16_t* item_f, int64_t k,
                               const int32_t* rows, const float* vals, const int32_t* runs,
                               const int32_t* tile_run, const int32_t* tile_cut, int64_t n_tiles,
                               int32_t max_tile_rows, const hmf_qband_opts* opts, double lr,
                               double reg_user, double reg_item, uint64_t seed, int64_t row_base,
                               int64_t col_base, void* stream);
int64_t hmf_sgd_block_runs_u16_f32(float* user_f, float* item_f, int64_t k, const uint16_t* rows,
                                   const float* vals, const int32_t* runs,
                                   const int32_t* tile_run, const int32_t* tile_cut,
                                   int64_t n_tiles, int32_t max_tile_rows,
                                   const hmf_qband_opts* opts, double lr, double reg_user,
                                   double reg_item, uint64_t seed, int64_t row_base,
                                   int64_t col_base, void* stream);
int64_t hmf_sgd_block_runs_u16_f16(uint16_t* user_f, uint16_t* item_f, int64_t k,
                                   const uint16_t* rows, const float* vals, const int32_t* runs,
                                   const int32_t* tile_run, const int32_t* tile_cut,
                                   int64_t n_tiles, int32_t max_tile_rows,
                                   const hmf_qband_opts* opts, double lr, double reg_user,
                                   double reg_item, uint64_t seed, int64_t row_base,
                                   int64_t col_base, void* stream);
/* uint8 ids relative to tiles of at most 256 rows: 5 bytes per streamed
 * rating (the user's byte + the fp32 rating). */
int64_t hmf_sgd_block_runs_u8_f32(float* user_f, float* item_f, int64_t k, const uint8_t* rows,
                                  const float* vals, const int32_t* runs, const int32_t* tile_run,
                                  const int32_t* tile_cut, int64_t n_tiles, int32_t max_tile_rows,
                                  const hmf_qband_opts* opts, double lr, double reg_user,
                                  double reg_item, uint64_t seed, int64_t row_base,
                                  int64_t col_base, void* stream);
int64_t hmf_sgd_block_runs_u8_f16(uint16_t* user_f, uint16_t* item_f, int64_t k,
                                  const uint8_t* rows, const float* vals, const int32_t* runs,
                                  const int32_t* tile_run, const int32_t* tile_cut,
                                  int64_t n_tiles, int32_t max_tile_rows,
                                  const hmf_qband_opts* opts, double lr, double reg_user,
                                  double reg_item, uint64_t seed, int64_t row_base,
                                  int64_t col_base, void* stream);

/*
 * The reference visit order of a range of n triples under `seed`
 * (kernels.py:77-119): perm[t] = offset (relative to start) of the t-th
 * triple updated.  perm: device int32[n], n < 2^31.
 */
int hmf_visit_order(int64_t n, uint64_t seed, int32_t* perm, void* stream);

/* kernels.mix64 (kernels.py:32-48): splitmix64 fold, clipped to 63 bits. */
uint64_t hmf_mix64(const uint64_t* parts, int32_t n_parts);

/*
 * Residual sums over n triples (sgd.py:134-188), accumulated in f64:
 *   out[0] = sum (vals[i] - P[u]·Q[v])^2
 *   out[1] = sum |P[u]|^2          (only when with_reg != 0, else 0)
 *   out[2] = sum |Q[v]|^2          (only when with_reg != 0, else 0)
 * u = rows[i] - row_base, v = cols[i] - col_base.  out: device double[3].
 * rmse = sqrt(out[0] / n); regularized_loss = out[0] + reg_u*out[1] + reg_i*out[2].
 * Deterministic: the reduction order depends only on n and the device.
 */
int hmf_residual_sums_f32(const float* user_f, const float* item_f, int64_t k,
                          const int32_t* rows, const int32_t* cols, const float* vals, int64_t n,
                          int64_t row_base, int64_t col_base, int32_t with_reg, double* out,
                          void* stream);
int hmf_residual_sums_f16(const uint16_t* user_f, const uint16_t* item_f, int64_t k,
                          const int32_t* rows, const int32_t* cols, const float* vals, int64_t n,
                          int64_t row_base, int64_t col_base, int32_t with_reg, double* out,
                          void* stream);
int hmf_residual_sums_f64(const double* user_f, const double* item_f, int64_t k,
                          const int32_t* rows, const int32_t* cols, const double* vals, int64_t n,
                          int64_t row_base, int64_t col_base, int32_t with_reg, double* out,
                          void* stream);

/*
 * Block bucketing — data.build_grid (data.py:238-280).
 * Block id of triple i = row_band(rows[i]) * n_col_bands + col_band(cols[i]),
 * bands found by binary search in row_cuts / col_cuts (device int64 arrays of
 * n_row_bands+1 / n_col_bands+1 ascending cuts).  Writes the triples
 * block-major into out_* — a stable partition: input order is preserved inside
 * each block, as the reference's argsort(kind="stable") does — and the CSR
 * offsets into block_ptr (device int64[n_blocks + 1]).  Ratings are f32.
 */
int hmf_bucket_triples(const int32_t* rows, const int32_t* cols, const float* vals, int64_t n,
                       const int64_t* row_cuts, int32_t n_row_bands, const int64_t* col_cuts,
                       int32_t n_col_bands, int32_t* out_rows, int32_t* out_cols,
                       float* out_vals, int64_t* block_ptr, void* stream);

/*
 * Synthetic instance generator with the synthetic_ratings law
 * (data.py:311-336), for shapes the reference generator cannot reach.
 * Cells: each cell of rows [row_base, row_base + n_rows) x [0, n_cols) is
 * selected independently with probability p (geometric skipping along each
 * row, counter-based RNG keyed by seed and the GLOBAL row id), so the
 * selected set is uniform given its size, and a row band generated alone is
 * exactly that band of the whole matrix (one matrix across ranks).
 *   hmf_synthetic_count: row_ptr (device int64[n_rows + 1]) <- CSR offsets of
 *     the selected cells of the band; returns the total count (synchronises
 *     `stream`).
 *   hmf_synthetic_cells: writes the selected (global row, col) pairs, row-major.
 * Values: vals[i] = sum_{r<rank} A[rows[i], r] * B[cols[i], r] + N(0, noise),
 * A, B entries U[0, factor_scale/sqrt(rank)] from a hash of (seed, row/col, r),
 * the noise from a hash of (seed, row, col): a function of the cell only.
 */
int64_t hmf_synthetic_count(int64_t n_rows, int64_t n_cols, double p, uint64_t seed,
                            int64_t row_base, int64_t* row_ptr, void* stream);
int hmf_synthetic_cells(int64_t n_rows, int64_t n_cols, double p, uint64_t seed,
                        int64_t row_base, const int64_t* row_ptr, int32_t* out_rows,
                        int32_t* out_cols, void* stream);
/* out[i] = in[pi(i)] for i < n_out, pi a keyed pseudo-random permutation of
 * [0, n_in) (Feistel network with cycle walking): the reference's
 * permutation(chosen)[:target] without a sort or an index array. */
int hmf_permute_cells(const int32_t* in_rows, const int32_t* in_cols, int64_t n_in,
                      int32_t* out_rows, int32_t* out_cols, int64_t n_out, uint64_t seed,
                      void* stream);
int hmf_synthetic_fill(const int32_t* rows, const int32_t* cols, int64_t n, int32_t rank,
                       double noise, double factor_scale, uint64_t seed, float* vals,
                       void* stream);
/* Held-out split keyed by the cell: mask[i] = 1 iff a hash of (seed, rows[i],
 * cols[i]) falls below `fraction` (device uint8[n]), so every row band agrees
 * with the whole matrix on its test cells. */
int hmf_cell_mask(const int32_t* rows, const int32_t* cols, int64_t n, double fraction,
                  uint64_t seed, uint8_t* mask, void* stream);

/* Device / peer utilities for the multi-GPU item-band hand-off. */
int hmf_device_count(int32_t* n);
int hmf_set_device(int32_t dev);
int hmf_enable_peer_access(int32_t dev, int32_t peer);
int hmf_memcpy_peer_async(void* dst, int32_t dst_dev, const void* src, int32_t src_dev,
                          int64_t bytes, void* stream);
int hmf_stream_synchronize(void* stream);
/* CUDA IPC: 64-byte handle of the allocation holding dptr (and dptr's byte
 * offset inside it), to be opened in another process of the same node. */
int hmf_ipc_get_handle(const void* dptr, uint8_t* handle64, int64_t* offset);
int hmf_ipc_open_handle(const uint8_t* handle64, void** dptr);
int hmf_ipc_close_handle(void* dptr);

/*
 * Node-local column-lease table of the multi-GPU engine (replaces the
 * reference's in-process GridScheduler.acquire/release for column units,
 * scheduler.py:333-409; the torch.distributed TCPStore compare-and-set in
 * distributed.LeaseTable is the portable alternative).  A POSIX shared-memory
 * segment `name` ("/..."): per column band its holder (-1 free) and last
 * owner (-1 none), and a ticket counter; every operation is one lock-free
 * atomic (host code, no GPU needed).
 *   hmf_lease_open: create != 0 (one process, before the others open it)
 *     makes a fresh segment with every column free; otherwise maps the
 *     existing one (n_cols must match).  *table is an opaque handle.
 *   hmf_lease_try_acquire: 1 granted, 0 held by someone, < 0 error.
 *   hmf_lease_acquire_first: tries cands[0..n) in order; *got = the first
 *     granted column, or -1 if every candidate is held.
 *   hmf_lease_release: records rank as the column's owner, then frees it;
 *     error if rank does not hold it.
 *   hmf_lease_ticket: a global sequence number (1, 2, ...).
 *   hmf_lease_ops: atomic operations served so far (all processes).
 *   hmf_lease_abort: marks the run aborted by `rank` (the first abort wins);
 *     every later acquire returns HMF_ERR_ABORTED (scheduler.abort,
 *     scheduler.py:415-423; workers.py:300-302).  hmf_lease_aborted: the
 *     aborting rank, or -1.
 */
int hmf_lease_open(const char* name, int32_t n_cols, int32_t create, void** table);
int hmf_lease_close(void* table, int32_t unlink_segment);
int32_t hmf_lease_try_acquire(void* table, int32_t c, int32_t rank);
int hmf_lease_acquire_first(void* table, const int32_t* cands, int32_t n, int32_t rank,
                            int32_t* got);
int32_t hmf_lease_release(void* table, int32_t c, int32_t rank);
int hmf_lease_owner(void* table, int32_t c, int32_t* owner);
int hmf_lease_holder(void* table, int32_t c, int32_t* holder);
int64_t hmf_lease_ticket(void* table);
int64_t hmf_lease_ops(void* table);
/* The free policy's job-wide work counter (scheduler.py:411-429, POLICY_FREE:
 * an epoch is n_blocks block updates, taken by whoever is free): claims the
 * next block update if fewer than `target` were claimed — returns its ordinal
 * (1, 2, ...) — else 0; HMF_ERR_ABORTED once the run is aborted. */
int64_t hmf_lease_claim(void* table, int64_t target);
int hmf_lease_abort(void* table, int32_t rank);
int32_t hmf_lease_aborted(void* table);

#ifdef __cplusplus
}
#endif

#endif /* HMF_H_ */
