/*
 * pm2l.h — C ABI of the B200-native (sm_100a) PM2Lat latency-prediction path.
 *
 * Library: paper_2603_00549_b200/libpm2l_b200.so (nvcc, -gencode
 * arch=compute_100a,code=sm_100a, static cudart).  Plain C types only: no torch,
 * no CUDA headers needed by a caller (streams are passed as void*).
 *
 * Every entry point returns PM2L_OK (0) or a negative status; the message of the
 * last failure on the calling thread is pm2l_last_error().  Unresolved grid
 * points are NOT errors: like the reference they come out as NaN latency
 * (pm2lat/_kernels.pyx:115-118) with curve id -1, blocks 0 and waves 0.
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/pm2lat):
 *   pm2l_predict_grid_slice    <- _kernels.pyx:76-133  predict_grid_slice(...)
 *                                 (the only native FFI of the reference; same 25
 *                                 arguments in the same order, array lengths added)
 *   pm2l_tables_create         <- nascache.py:174-241  PreparedGrid.tables()
 *                                 (stages those arrays in HBM once per grid triple)
 *   pm2l_grid_predict          <- backend.py:49-88     predict_grid/_predict_grid_compiled
 *   pm2l_grid_predict_host     <- backend.py:49-88     the same with the result in a host
 *                                 buffer (backend.predict_grid returns a numpy array)
 *   pm2l_grid_dplan_*          <- nascache.py:140-245 + backend.py:58-76: the per-grid
 *                                 planning (PreparedGrid / tables() / axis logs) on the GPU
 *   pm2l_points_predict(_ext)  <- compute.py:251-268 + 150-193
 *                                 ConfigResolver.resolve + predict_generic, batched
 *                                 (_ext: coordinates >= 2^22 via a libm-log2 extension)
 *   pm2l_points_predict_curve  <- compute.py:150-193   predict_generic with an explicit
 *                                 kernel (no resolution; "mode X")
 *   pm2l_membound_predict      <- membound.py:117-127  predict_membound, batched
 *   pm2l_store_encode          <- nascache.py:308-333  precompute's record writer
 *                                 (big-endian records of resolved points)
 *   pm2l_store_lookup          <- nascache.py:408-424  CacheStore.lookup, batched
 *   pm2l_segment_fsum          <- aggregate.py:193     math.fsum of per-layer latencies,
 *                                 per model segment (correctly rounded)
 *   pm2l_grid_error_report     <- curvefit.py:192-219  grid_error_report
 *   pm2l_partition_scan        <- partition.py:53-100  partition_two_device's cut scan
 */
#ifndef PM2L_H_
#define PM2L_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PM2L_ABI_VERSION 1

enum {
  PM2L_OK = 0,
  PM2L_ERR_INVALID = -1,  /* bad argument / inconsistent tables            */
  PM2L_ERR_CUDA = -2,     /* a CUDA runtime call or kernel launch failed    */
  PM2L_ERR_NOMEM = -3,    /* host or device allocation failed               */
  PM2L_ERR_NODEVICE = -4  /* no CUDA device visible (no CPU fallback exists) */
};

/* ------------------------------------------------------------------ misc */
int pm2l_abi_version(void);
/* Hash of the sources the library was built from (build-staleness check). */
const char* pm2l_source_hash(void);
const char* pm2l_last_error(void);
/* Number of visible CUDA devices (0 on a CPU-only host; never an error). */
int pm2l_device_count(void);

/* ------------------------------------------------------ staged tables ---
 * Host view of PreparedGrid.tables() (nascache.py:174-241) for ONE
 * (family, dtype, transpose) triple.  R candidate records in the resolver's
 * scan order (sorted by (m, n, k, batch), nascache.py:149), C curves.
 *
 * exact_keys/exact_curve: the reference's packed u64 keys
 *   (b<<48 | m<<32 | n<<16 | k, each field < 2^16) sorted ascending, with the
 *   curve index per key (nascache.py:188-194).  Alternatively pass
 *   exact_coords (R x 4 u64, row-major batch,m,n,k; any width) and leave
 *   exact_keys NULL — the B200 build then serves coordinates >= 2^16, which
 *   the reference only handles on its Python path (nascache.py:163-168).
 * log_m/log_n/log_k: log2 of the candidate coordinates (R each).
 * cand_curve: curve index of each candidate, -1 = recorded kernel has no curve.
 * sample_offsets (C+1), sample_dims / sample_thrs (sample_offsets[C] each).
 * ref_dim/ref_dur/ref_thr/ref_waves (C): reference point of each curve.
 * tile_m/tile_n/split_k/blocks_per_wave (C), family_rowblock (C, 0/1).
 */
typedef struct pm2l_tables_view {
  int64_t n_records;
  const uint64_t* exact_keys;    /* R, or NULL when exact_coords is given */
  const uint64_t* exact_coords;  /* R*4, or NULL */
  const int64_t* exact_curve;    /* R */
  const double* log_m;
  const double* log_n;
  const double* log_k;
  const int64_t* cand_curve;
  int64_t n_curves;
  const int64_t* sample_offsets;
  const double* sample_dims;
  const double* sample_thrs;
  const double* ref_dim;
  const double* ref_dur;
  const double* ref_thr;
  const double* ref_waves;
  const uint64_t* tile_m;
  const uint64_t* tile_n;
  const uint64_t* split_k;
  const uint64_t* blocks_per_wave;
  const uint8_t* family_rowblock;
} pm2l_tables_view;

typedef struct pm2l_tables pm2l_tables; /* opaque, HBM-resident */

/* Validate + reorganise the tables (candidate groups by distinct log_k) and
 * upload them to `device`.  The view is not retained. */
int pm2l_tables_create(const pm2l_tables_view* view, int device, pm2l_tables** out);
int pm2l_tables_destroy(pm2l_tables* t);
/* Number of candidate groups (distinct log_k values) — diagnostics. */
int64_t pm2l_tables_groups(const pm2l_tables* t);

/* ------------------------------------------------------------ grid mode ---
 * Canonical (batch, m, n, k) product grid, k innermost (nascache.py:98-99).
 * Fills batch indices [b_lo, b_hi): output element
 *   ((ib - b_lo)*|m| + im)*|n|*|k| + jn*|k| + ik.
 * axis_* are HOST arrays (a few KB; copied per call).  out_* are DEVICE
 * pointers; out_curve / out_blocks / out_waves may be NULL (verification
 * outputs; excluded from the throughput byte count).  stream = cudaStream_t
 * or NULL for the legacy default stream.  Asynchronous w.r.t. the host. */
int pm2l_grid_predict(pm2l_tables* t,
                      const uint64_t* batch_vals, int64_t n_batch,
                      const uint64_t* m_vals, int64_t n_m,
                      const uint64_t* n_vals, int64_t n_n,
                      const uint64_t* k_vals, int64_t n_k,
                      int64_t b_lo, int64_t b_hi,
                      double* out_lat, int32_t* out_curve,
                      uint64_t* out_blocks, uint64_t* out_waves,
                      void* stream);

/* Reusable launch plan of one grid slice: the axis values, their host-libm
 * log2, the exact-hit fix-up list and the per-(curve, k) base workspace are
 * staged in HBM once; pm2l_grid_plan_launch then only launches kernels (no
 * host work, no copies — CUDA-graph capturable).  The tables must outlive the
 * plan.  nan_stats (DEVICE, 3 x u64, nullable; a launch that includes the
 * base-table stage resets it to {~0, 0, 0} itself, otherwise initialise it):
 * [0] first NaN slice index (UnresolvedPoint semantics, nascache.py:298-306),
 * [1] NaN count, [2] set when [0] must be re-derived with pm2l_nan_scan.
 * stages: bitmask 1 = base table, 2 = grid kernel, 4 = exact fix-ups
 * (0 or 7 = all; separate stages let a caller time each kernel). */
typedef struct pm2l_grid_plan pm2l_grid_plan;
int pm2l_grid_plan_create(pm2l_tables* t,
                          const uint64_t* batch_vals, int64_t n_batch,
                          const uint64_t* m_vals, int64_t n_m,
                          const uint64_t* n_vals, int64_t n_n,
                          const uint64_t* k_vals, int64_t n_k,
                          int64_t b_lo, int64_t b_hi, pm2l_grid_plan** out);
int pm2l_grid_plan_launch(pm2l_grid_plan* p, double* out_lat, int32_t* out_curve,
                          uint64_t* out_blocks, uint64_t* out_waves, uint64_t* nan_stats,
                          int stages, void* stream);
/* info[0] slice cardinality, [1] exact fix-ups, [2] workspace bytes,
 * [3] bytes staged host->device at creation. */
int pm2l_grid_plan_info(const pm2l_grid_plan* p, int64_t* info);
/* Which grid kernel a launch with these outputs would run (diagnostics and
 * tests): 0 general k-group sweep, 1 sweep + tie mask, 2 one-class closed
 * form, 3 one-class lookup path; negative on error. */
int pm2l_grid_plan_kernel(const pm2l_grid_plan* p, const double* out_lat, int verify);
int pm2l_grid_plan_destroy(pm2l_grid_plan* p);
/* Device-planned grid slices.  The per-slice planning of pm2l_grid_plan_create
 * (host libm log2 of the axes, the k-only half of the nearest-config argmin,
 * the exact-record join of _kernels.pyx:107-110, the per-(curve, k) base
 * table) runs as one GPU kernel in the launch's stream, so a sweep over many
 * grids never returns to the host between slices (and a launch is CUDA-graph
 * capturable).  Axes are DEVICE arrays in canonical GridSpec order (strictly
 * ascending, every m/n/k value in [1, 2^22)); a violation sets a sticky bit
 * read by pm2l_grid_dplan_status (1: value out of range, 2: not ascending) and
 * the slice's outputs are then undefined.  Capacities bound the axis lengths
 * of every launch.  Outputs, nan_stats and stages as pm2l_grid_plan_launch
 * (stage 1 = the planner kernel, which also builds the base table).
 * pm2l_grid_predict plans on the device by itself whenever the host axes are
 * canonical. */
typedef struct pm2l_grid_dplan pm2l_grid_dplan;
int pm2l_grid_dplan_create(pm2l_tables* t, int64_t max_batch, int64_t max_m, int64_t max_n,
                           int64_t max_k, pm2l_grid_dplan** out);
int pm2l_grid_dplan_launch(pm2l_grid_dplan* p,
                           const uint64_t* batch_vals, int64_t n_batch,
                           const uint64_t* m_vals, int64_t n_m,
                           const uint64_t* n_vals, int64_t n_n,
                           const uint64_t* k_vals, int64_t n_k,
                           int64_t b_lo, int64_t b_hi,
                           double* out_lat, int32_t* out_curve, uint64_t* out_blocks,
                           uint64_t* out_waves, uint64_t* nan_stats, int stages, void* stream);
/* Synchronises the device; returns and clears the sticky status bits. */
int pm2l_grid_dplan_status(pm2l_grid_dplan* p, uint32_t* status);
/* Grid kernel of the last launch (codes as pm2l_grid_plan_kernel). */
int pm2l_grid_dplan_kernel(const pm2l_grid_dplan* p);
/* Exact-record fix-ups planned for the last launch (synchronises). */
int pm2l_grid_dplan_fixups(pm2l_grid_dplan* p, int64_t* count);
int pm2l_grid_dplan_destroy(pm2l_grid_dplan* p);

/* first NaN index of lat[0..n) -> atomicMin into *first (DEVICE u64). */
int pm2l_nan_scan(const double* lat, int64_t n, uint64_t* first, void* stream);

/* Same, but every curve for every point ("mode X": shape x all candidate
 * kernels, predict_generic per (shape, kernel), compute.py:150-193).
 * out_lat is [C][cardinality of the slice], curve-major. */
int pm2l_grid_predict_all_curves(pm2l_tables* t,
                                 const uint64_t* batch_vals, int64_t n_batch,
                                 const uint64_t* m_vals, int64_t n_m,
                                 const uint64_t* n_vals, int64_t n_n,
                                 const uint64_t* k_vals, int64_t n_k,
                                 int64_t b_lo, int64_t b_hi,
                                 double* out_lat, void* stream);

/* -------------------------------------------- explicit-descriptor mode ---
 * n ops, DEVICE array `shapes` of n x uint4-like records {b, m, n, k} (u32
 * each, 16 B per op), resolved against the staged triple `t`
 * (ConfigResolver.resolve semantics, pm2lat/compute.py:251-268: exact match
 * first, else nearest by Chebyshev distance in log2 space, first index on
 * ties) and predicted (compute.py:163-193).
 * Query log2 values are host-libm log2 (math.log2, as the reference's
 * resolver takes them): a per-device table covers coordinates below
 * pm2l_points_log2_table_size() (2^22); larger coordinates need an entry in
 * the caller's extension -- DEVICE arrays ext_coords (ascending, unique u32)
 * and ext_log2 (libm log2 of each), n_ext entries (pm2l_points_predict has
 * none).  Nullable outputs: out_curve (curve id, -1 unresolved), out_waves
 * (saturated at 2^32-1), out_match (0 exact, 1 nearest, -1 no candidates,
 * -2 invalid coordinate (0, or no log2 for it), -3 block count >= 2^64,
 * which the reference's unbounded-integer Python path would still answer),
 * out_record (matched record: scan index for nearest; position in the exact
 * arrays given at pm2l_tables_create for exact hits -- the first record of
 * that shape), out_dist (ResolvedConfig.distance: 0 exact, Chebyshev log2
 * distance otherwise), out_detail (_ext only; 4 doubles per op, the
 * Prediction.components of compute.py:177-193: base_us,
 * new_throughput_gflops, wave_scale, waves; NaN when unresolved). */
int pm2l_points_predict_ext(pm2l_tables* t, const uint32_t* shapes, int64_t n,
                            const uint32_t* ext_coords, const double* ext_log2, int64_t n_ext,
                            double* out_lat, int32_t* out_curve, uint32_t* out_waves,
                            int8_t* out_match, int32_t* out_record, double* out_dist,
                            double* out_detail, void* stream);
int pm2l_points_predict(pm2l_tables* t, const uint32_t* shapes, int64_t n,
                        double* out_lat, int32_t* out_curve, uint32_t* out_waves,
                        int8_t* out_match, int32_t* out_record, double* out_dist,
                        void* stream);
int64_t pm2l_points_log2_table_size(void);

/* n ops with an explicit curve each (DEVICE int32 curve ids; no resolution;
 * predict_generic, compute.py:150-193).  out_detail (nullable) receives 4
 * doubles per op: base_us, new_throughput_gflops, wave_scale, waves.  A block
 * count >= 2^64 gives NaN everywhere (see pm2l_points_predict_ext). */
int pm2l_points_predict_curve(pm2l_tables* t, const uint32_t* shapes,
                              const int32_t* curve_ids, int64_t n,
                              double* out_lat, uint32_t* out_waves, double* out_detail,
                              void* stream);

/* ------------------------------------------------------- memory-bound ---
 * predict_membound (membound.py:117-127) for n ops.  DEVICE arrays:
 * features n x 5 (flops, int_ops, bytes_loaded, bytes_stored,
 * total_bytes_accessed), model_ids n (int32 into weights/intercepts),
 * weights n_models x 5, intercepts n_models, floors n_models.
 * raw = fma-chain dot(w, f) + intercept;  lat = raw < floor ? floor : raw.
 * out_floored (nullable) = 1 where the floor applied. */
int pm2l_membound_predict(const double* features, const int32_t* model_ids, int64_t n,
                          const double* weights, const double* intercepts,
                          const double* floors, int64_t n_models,
                          double* out_lat, uint8_t* out_floored, void* stream);
/* The same, plus (nullable) out_raw: the pre-floor value (the reference's
 * Prediction component "raw_us", membound.py:117-127). */
int pm2l_membound_predict_raw(const double* features, const int32_t* model_ids, int64_t n,
                              const double* weights, const double* intercepts,
                              const double* floors, int64_t n_models, double* out_lat,
                              uint8_t* out_floored, double* out_raw, void* stream);

/* ------------------------------------------------ audits (§8f row 4) ---
 * curvefit.grid_error_report (pm2lat/curvefit.py:192-219) for one curve:
 * DEVICE arrays dims (int64, ascending sample dims) and thrs (throughputs),
 * n_samples in [2, 1024]; per sample interval [lo, hi) the scan is
 * range(lo, hi, stride) plus hi, the error |interp - truth| / truth, and
 * out_err / out_argmax (n_samples - 1 each) the first maximum of the
 * interval (initial (-1.0, lo)).  truth: the oracle's value per scan point,
 * intervals concatenated, interval i starting at scan_off[i] -- or null
 * with rational (a HOST array {a, b, c, d}): truth = (a*x + b) / (c*x + d). */
int pm2l_grid_error_report(const int64_t* dims, const double* thrs, int64_t n_samples,
                           int64_t stride, const double* truth, const int64_t* scan_off,
                           const double* rational, double* out_err, int64_t* out_argmax,
                           void* stream);

/* partition.partition_two_device's cut scan (pm2lat/partition.py:53-100):
 * DEVICE per-layer latencies of the two devices (n_layers each) and an
 * optional per-cut transfer term (n_layers + 1); for every cut in
 * [0, n_layers]: stage_a = left-to-right sum of lat_a[:cut], stage_b =
 * left-to-right sum of lat_b[cut:] + transfer[cut], bottleneck = Python
 * max(stage_a, stage_b); out_best_cut = the first cut of minimum
 * bottleneck (the reference's strict-< scan). */
int pm2l_partition_scan(const double* lat_a, const double* lat_b, int64_t n_layers,
                        const double* transfer, double* out_stage_a, double* out_stage_b,
                        double* out_bottleneck, int64_t* out_best_cut, void* stream);

/* --------------------------------------------------- per-model totals ---
 * Correctly rounded sum (== math.fsum) of values[offsets[s] .. offsets[s+1])
 * for each of n_segments segments (DEVICE arrays; offsets has n_segments+1
 * entries).  Values of either sign (a raw membound layer under a
 * non-positive floor is negative); NaN, or both infinities, in a segment give
 * a NaN total (math.fsum raises there), one infinity gives that infinity.
 * Exact warp-segmented two's-complement fixed-point reduction. */
int pm2l_segment_fsum(const double* values, const int64_t* offsets, int64_t n_segments,
                      double* out_totals, void* stream);

/* Store encoder (nascache.py:308-333 record section): for the
 * grid slice whose canonical latencies are lat[0..n) (DEVICE) and whose axis
 * values are B/M/N/K (DEVICE u64; batch = the slice's batch values), write
 * the 40-byte big-endian records (b, m, n, k, latency) of every resolved
 * (non-NaN) point in canonical order into `records` (DEVICE, >= 40*n bytes)
 * and their number into *count (DEVICE i64).  workspace: DEVICE, at least
 * pm2l_store_encode_workspace(n) bytes.  Stream-ordered, no host sync. */
int64_t pm2l_store_encode_workspace(int64_t n);
int pm2l_store_encode(const double* lat, int64_t n, const uint64_t* batch_vals,
                      const uint64_t* m_vals, int64_t n_m, const uint64_t* n_vals, int64_t n_n,
                      const uint64_t* k_vals, int64_t n_k, void* workspace, uint8_t* records,
                      int64_t* count, void* stream);

/* Batched CacheStore.lookup (nascache.py:408-424):
 * records = the store's record section (DEVICE, n_records x 40 bytes,
 * sorted), queries = n x 4 u64 (batch, m, n, k) (DEVICE).  out[i] = the
 * stored latency or NaN when absent; *first_missing (DEVICE u64, initialise
 * to ~0) = the smallest absent query index.  axes/axis_lens (DEVICE axes of
 * the store's grid, may be NULL): when given and the store is dense (every
 * grid point present, n_records == product of the lengths) a query is
 * direct-indexed instead of binary-searched. */
int pm2l_store_lookup(const uint8_t* records, int64_t n_records, const uint64_t* const* axes,
                      const int64_t* axis_lens, const uint64_t* queries, int64_t n, double* out,
                      uint64_t* first_missing, void* stream);

/* backend.predict_grid's host-output form (pm2lat/backend.py:49-88 returns a
 * numpy array): the slice [b_lo, b_hi) of the staged triple's grid (HOST
 * axis arrays) into the HOST buffer `out` -- one D2H copy when `out` is
 * page-locked, else chunked D2H through a pinned ring drained by a host
 * copy pool (the same path as pm2l_predict_grid_slice).  Synchronous. */
int pm2l_grid_predict_host(pm2l_tables* t, const uint64_t* batch_vals, int64_t n_batch,
                           const uint64_t* m_vals, int64_t n_m, const uint64_t* n_vals,
                           int64_t n_n, const uint64_t* k_vals, int64_t n_k, int64_t b_lo,
                           int64_t b_hi, double* out);

/* ------------------------------------------------ reference FFI drop-in ---
 * Exactly pm2lat._kernels.predict_grid_slice (_kernels.pyx:76-133): HOST
 * arrays in, HOST `out` (length (b_hi-b_lo)*n_m*n_n*n_k) written in place,
 * synchronous, thread-safe (concurrent calls on disjoint slices, as
 * backend.py:78-87 issues them).  Runs on the current CUDA device; tables
 * are staged per call (cached by content).  Array lengths are the extra
 * n_* arguments the memoryviews carried implicitly.  A page-locked `out`
 * (cudaHostAlloc / cudaHostRegister) is written by one direct device-to-host
 * copy; a pageable one through a pinned staging ring. */
int pm2l_predict_grid_slice(
    const uint64_t* batch_vals, int64_t n_batch,
    const uint64_t* m_vals, int64_t n_m,
    const uint64_t* n_vals, int64_t n_n,
    const uint64_t* k_vals, int64_t n_k,
    int64_t b_lo, int64_t b_hi,
    const uint64_t* exact_keys, const int64_t* exact_curve, int64_t n_records,
    const double* log_m, const double* log_n, const double* log_k,
    const int64_t* cand_curve,
    const int64_t* sample_offsets, const double* sample_dims, const double* sample_thrs,
    int64_t n_curves,
    const double* ref_dim, const double* ref_dur, const double* ref_thr,
    const double* ref_waves,
    const uint64_t* tile_m, const uint64_t* tile_n, const uint64_t* split_k,
    const uint64_t* blocks_per_wave, const uint8_t* family_rowblock,
    double* out);

#ifdef __cplusplus
}
#endif
#endif /* PM2L_H_ */
