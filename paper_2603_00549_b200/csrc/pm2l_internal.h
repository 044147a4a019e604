// Internal layout shared by the host planner (tables.cpp, abi.cpp) and the
// sm_100a kernels (kernels.cu).  Not part of the public ABI (include/pm2l.h).
#pragma once

#include <cstdint>

#include <vector_types.h>

#include "../../include/pm2l.h"
#include <string>
#include <vector>

namespace pm2l {

// ---------------------------------------------------------------------------
// HBM-resident staged tables of one (family, dtype, transpose) triple.
//
// Candidates are regrouped by their distinct log2(k) value ("k-groups"):
// the nearest-config distance of candidate i is  max(D_i(m,n), |lk_i - qk|)
// with D_i = max(|lm_i - qm|, |ln_i - qn|), so inside one group the k term is
// shared and the argmin over the group reduces to a prefix-minimum staircase
// of D_i over the candidates in scan order (built per (m, n) row in shared
// memory).  Original scan indices are kept so ties break exactly as the
// reference's strict '<' scan (_kernels.pyx:29-47).
// Wave-class parameters (grid_row_kernel's W table inputs), one per class.
struct alignas(16) WcParam {
  uint64_t tm, tn, sk, bpw;
  double rw;        // ref_waves
  uint32_t dm[3];   // u32 division magic for tm, tn, bpw (common.cuh ceil_div_c)
  uint32_t ds[3];
};

struct TablesDev {
  int32_t R = 0;        // candidate records
  int32_t C = 0;        // curves
  int32_t G = 0;        // k-groups
  int32_t n_exact = 0;  // exact records (== R)
  int32_t all_gemm = 1; // no row-block curve referenced
  int32_t all_rowblock = 0;  // >= 1 curve referenced, all of them row-block
  int32_t lowest_wins = 0;  // equal logs imply equal coordinates (all < 2^44)
  int32_t single_mn = 0;    // one member class whose members all share one (log m, log n)
  int32_t n_samples = 0;
  // per curve [C]
  const double* ref_dim = nullptr;
  const double* ref_dur = nullptr;
  const double* ref_thr = nullptr;
  const double* ref_waves = nullptr;
  const uint64_t* tile_m = nullptr;
  const uint64_t* tile_n = nullptr;
  const uint64_t* split_k = nullptr;
  const uint64_t* bpw = nullptr;     // blocks per wave (sm_count * blocks_per_sm)
  // u32 division magic for (tile_m, tile_n, bpw) of each curve [3*C]:
  // dv_m = multiplier, dv_s = sh1 | sh2 << 8 | valid << 16 (Granlund-Montgomery)
  const uint32_t* dv_m = nullptr;
  const uint32_t* dv_s = nullptr;
  // wave classes: curves with identical (rowblock, tile_m, tile_n, split_k,
  // blocks_per_wave, ref_waves) share every blocks / waves / wave-scale value
  int32_t NW = 0;
  const int32_t* wc_of = nullptr;   // [C] class of each curve (-1: no samples)
  const int32_t* wc_rep = nullptr;  // [NW] representative curve of each class
  const uint8_t* rowblock = nullptr;
  const int32_t* s_off = nullptr;    // [C+1] sample offsets
  const double* s_dims = nullptr;
  const double* s_thrs = nullptr;
  // candidates in group order [R]
  const double* g_lm = nullptr;
  const double* g_ln = nullptr;
  const int32_t* g_idx = nullptr;    // original scan index
  const int32_t* cand_curve = nullptr; // by ORIGINAL index [R]
  const int32_t* g_curve = nullptr;    // curve of each candidate in GROUP order [R]
  const int32_t* g_cw = nullptr;       // [2R] (curve, wave class) in GROUP order
  const WcParam* wcp = nullptr;        // [NW]
  const WcParam* wcp_c = nullptr;      // [C] wcp[wc_of[c]] per curve (zero: no samples)
  // groups [G]
  const double* grp_lk = nullptr;
  const int32_t* grp_start = nullptr;
  const int32_t* grp_size = nullptr;
  const int32_t* grp_class = nullptr;
  const int32_t* grp_curve0 = nullptr;  // [G] curve of each group's first member (scan order)
  int32_t n_rec_k = 0;                  // distinct exact-record k values
  const uint64_t* rec_k = nullptr;      // [n_rec_k] ascending
  // member classes: groups whose member (log m, log n) sequences are equal
  // share one D sequence and one staircase per (m, n) row (the shipped
  // presets collect every kernel at every sample k, so all k-groups of a
  // triple fall into ONE class).  NC classes, CM members in total.
  int32_t NC = 0;
  int32_t CM = 0;
  const int32_t* cls_start = nullptr;  // [NC] into cls_lm / cls_ln
  const int32_t* cls_size = nullptr;   // [NC]
  const double* cls_lm = nullptr;      // [CM]
  const double* cls_ln = nullptr;      // [CM]
  // exact records [n_exact], unpacked, sorted by (b,m,n,k)
  const uint64_t* ex_coord = nullptr; // 4 per record
  const int32_t* ex_curve = nullptr;
  const int32_t* ex_rec = nullptr;    // position in the caller's exact arrays
  // the same records, unique, sorted by (m, n, b, k) (device planner)
  int32_t n_mn = 0;
  const uint64_t* ex_mn_coord = nullptr;  // 4 per record
  const int32_t* ex_mn_curve = nullptr;
  // explicit-descriptor mode (points.cu) -----------------------------------
  // exact records with u32 coordinates as an open-addressing hash (linear
  // probing, xh_hash below), staged in shared memory: capacity xh_mask + 1
  // (a power of two >= 2x the records); key b == 0 marks an empty slot; the
  // value is (curve, position in the caller's exact arrays) of the FIRST
  // record of that shape.  xh_mask < 0: no table (bsearch over ex_coord).
  int32_t xh_mask = -1;
  const uint4* xh_key = nullptr;
  const int2* xh_val = nullptr;
  // per slot a nonzero 32-bit tag of the key (xh_tag below), 0 when empty:
  // the kernel probes the tags in shared memory and reads the full key only
  // on a tag match
  const uint32_t* xh_tags = nullptr;
  // one-class row decomposition of class 0's members: the distinct member
  // (log m) values are rows and the distinct (log n) values columns, both
  // ascending; member (i, j) is present iff bit j of rw_mask[i] (bit i of
  // cl_mask[j]).  Valid (rw_n > 0) when every row and column count is <= 64
  // and the deduplicated members in scan order are in (row, column)
  // lexicographic order, so the first member in scan order satisfying a
  // row and a column condition is the lowest row, then the lowest column.
  // rw_pos[rw_off[i] + rank of j in row i] = the member's first position in
  // the class member list.
  int32_t rw_n = 0, cl_n = 0;
  const double* rw_lm = nullptr;
  const double* cl_ln = nullptr;
  const uint64_t* rw_mask = nullptr;
  const uint64_t* cl_mask = nullptr;
  const int32_t* rw_off = nullptr;
  const int32_t* rw_pos = nullptr;
  // rw_lr[2 * (i * (cl_n + 1) + pc) + {0, 1}]: log n of row i's highest
  // present column below column insertion point pc / lowest at or above it
  // (-inf / +inf where none): the row minimum without mask scans
  const double* rw_lr = nullptr;
};

#ifdef __CUDACC__
#define PM2L_HD __host__ __device__ __forceinline__
#else
#define PM2L_HD inline
#endif
// Slot hash of an explicit descriptor (b, m, n, k) for TablesDev::xh_*.
PM2L_HD uint32_t xh_hash(uint32_t b, uint32_t m, uint32_t n, uint32_t k) {
  uint32_t h = (b * 0x9E3779B1u) ^ (m * 0x85EBCA77u) ^ (n * 0xC2B2AE3Du) ^ (k * 0x27D4EB2Fu);
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  return h;
}

// second, independent mix of the same key: the slot tag (never 0)
PM2L_HD uint32_t xh_tag(uint32_t b, uint32_t m, uint32_t n, uint32_t k) {
  uint32_t h = (b * 0xCC9E2D51u) + (m * 0x1B873593u) + (n * 0xE6546B64u) + (k * 0x85EBCA6Bu);
  h ^= h >> 16;
  h *= 0x7FEB352Du;
  h ^= h >> 13;
  return h | 1u;
}

// k chunk of the one-class lookup kernel: ranks of the per-k distance are
// taken inside chunks of this many k values (one warp's byte maps)
constexpr int kKChunk = 2048;
// byte-map bytes per lane for a k axis of nK values (16, 32 or 64)
inline int64_t kmap_lane_bytes(int64_t nK) {
  const int64_t kc = nK < kKChunk ? nK : kKChunk;
  return ((kc + 511) / 512) * 16;
}

// Per-k sweep info, 16 B (one 128-bit load in the grid kernel).
struct alignas(16) KInfo {
  double qk;      // libm log2(k)
  int32_t start;  // #k-groups with grp_lk < qk (outward sweep start)
  int32_t pad;
};

// Exact-hit fix-up of one grid point, bucketed by (m, n) row.
struct alignas(16) FixEntry {
  int32_t ik;     // k index
  int32_t ib;     // batch index, slice-relative
  int32_t curve;  // recorded kernel's curve (-1: no curve -> NaN)
  int32_t wc;     // wave class of the curve (-1 without a curve): the lookup
                  // kernel rescales the tile's base by its W table entry
};

// Per-launch grid description (device pointers into one per-call upload).
struct GridDev {
  int64_t nB = 0, nM = 0, nN = 0, nK = 0;  // full axis lengths
  int64_t b_lo = 0, b_hi = 0;              // slice of the batch axis
  const uint64_t* B = nullptr;
  const uint64_t* M = nullptr;
  const uint64_t* N = nullptr;
  const uint64_t* K = nullptr;
  const double* logM = nullptr;   // libm log2 of each axis value (host computed)
  const double* logN = nullptr;
  const double* logK = nullptr;
  // per k: {log2 k, sweep start = #groups with grp_lk < log2 k}, 16 B each
  const KInfo* kinfo = nullptr;
  // one-class lookup path (null unless 1 <= G <= 255 and nK <= 65535):
  // kfast[ik] = rank(ik) | gB(ik) << 16 | start(ik) << 24, where mn(ik) =
  // distance from log2 k to the nearest k-group, gB = leftmost group
  // attaining it, rank = position in the stable descending order of mn
  // within ik's chunk of kKChunk k values; mn_sorted[chunk start + rank] =
  // mn as ordered |double| bits
  const uint32_t* kfast = nullptr;
  const uint64_t* mn_sorted = nullptr;
  // [chunks x G]: first chunk-local k index with start(ik) > g
  const int32_t* kright = nullptr;
  // exact-hit fix-ups: slice-relative flat index + coordinates + curve
  int64_t n_fix = 0;
  const int64_t* fix_pos = nullptr;
  const uint64_t* fix_coord = nullptr;  // 4 per fix-up
  const int32_t* fix_curve = nullptr;
  // the same fix-ups bucketed by (m, n) row for the in-kernel path:
  // entries {ik, ib (slice-relative), curve, 0}, rows+1 offsets
  const int32_t* fixr_off = nullptr;
  const FixEntry* fixr = nullptr;
  int32_t max_fix_row = 0;
  int32_t k_sorted = 0;  // k axis strictly ascending (lookup kernel precondition)
  // device-planned slices (plan.cu): every array above is written on the GPU
  // by plan_kernel, in the same stream as the grid kernel.  n_fix is then the
  // triple's unique exact records, one fix-up entry each (fix_pos == -1 and
  // ib == -1 for records off the slice); status collects axis violations
  // (kPlanBad*), 0 for a valid plan.
  int32_t dev_planned = 0;
  // device plan already complete when the grid kernel launches (the planner
  // ran in an earlier launch, not as this launch's PDL primary): the per-k
  // tables are fetched at kernel entry instead of after griddepcontrol.wait
  int32_t plan_ready = 0;
  // device plans: per (m, n) row the [lo, hi) range of its records in the
  // fix-up list (entries of records off the slice have ib == -1 and
  // fix_pos == -1); null for host plans (fixr_off)
  const int2* fixr_rng = nullptr;
  uint32_t* status = nullptr;
  const double* lut = nullptr;  // per-device libm log2 table of [0, lut_n)
  int64_t lut_n = 0;
};

// Device planner (plan.cu): the per-slice work of build_grid on the GPU for
// canonical axes (strictly ascending, every value in [1, lut_n)).
enum : uint32_t { kPlanBadValue = 1, kPlanUnsorted = 2 };
struct DPlanCaps {
  int64_t nB = 0, nM = 0, nN = 0, nK = 0;  // axis capacities (batch: the whole axis)
};
// Whether a slice of these sizes can be device-planned with these tables.
bool dplan_supported(const struct TablesDev& t, const DPlanCaps& c);
// Bytes of the device buffer holding a plan of capacity c (incl. axes).
int64_t dplan_bytes(const struct TablesDev& t, const DPlanCaps& c);
// GridDev over a plan buffer for axes of the given lengths (axes: DEVICE
// arrays; nullptr -> the buffer's own axis copies, filled by the caller).
struct GridDev dplan_grid(const struct TablesDev& t, const DPlanCaps& c, void* buf,
                          const uint64_t* const axes[4], const int64_t lens[4], int64_t b_lo,
                          int64_t b_hi);
// Device axis copies inside a plan buffer (for host-side axes uploads).
uint64_t* dplan_axis_slot(const struct TablesDev& t, const DPlanCaps& c, void* buf, int axis);
// plan_kernel: logs, per-k tables, exact-hit join, base table, stats reset.
int launch_dplan(const struct TablesDev& t, const struct GridDev& g, double* base,
                 unsigned long long* nan_stats, bool ranks, void* stream);

// Host-side image of the staged tables (one contiguous byte blob whose
// internal pointers are rebased onto the device copy).
struct TablesHost {
  std::vector<uint8_t> blob;
  TablesDev dev_offsets;  // pointers hold byte OFFSETS into blob
  int64_t max_group = 0;
};

std::string build_tables(const pm2l_tables_view* v, TablesHost* out);
TablesDev rebase(const TablesDev& offsets, const void* base);

struct GridHost {
  std::vector<uint8_t> blob;
  GridDev dev_offsets;
};
std::string build_grid(const TablesHost& th, const uint64_t* const axes[4],
                       const int64_t lens[4], int64_t b_lo, int64_t b_hi, GridHost* out);
GridDev rebase(const GridDev& offsets, const void* base);

// Streaming multiprocessors of the current device (queried once per device).
int sm_count();

// Kernel launchers (kernels.cu).  Return a CUDA error code (0 = success).
struct LaunchOut {
  double* lat = nullptr;
  int32_t* curve = nullptr;
  uint64_t* blocks = nullptr;
  uint64_t* waves = nullptr;
  // unresolved-point statistics: [0] = min slice-relative flat index of a NaN
  // (UINT64_MAX if none), [1] = NaN count, [2] = dirty flag (an exact-hit
  // fix-up removed a NaN; [0] must be re-derived by launch_nan_scan).
  // Caller initialises to {UINT64_MAX, 0, 0}.
  unsigned long long* nan_stats = nullptr;
};
enum : int { kStageBase = 1, kStageGrid = 2, kStageFixup = 4, kStageAll = 7 };
int launch_grid(const TablesDev& t, const GridDev& g, int64_t max_group,
                double* workspace, int64_t workspace_elems, const LaunchOut& out,
                void* stream, int stages = kStageAll);
int64_t grid_workspace_elems(const TablesDev& t, const GridDev& g);
int grid_kernel_path(const TablesDev& t, const GridDev& g, const LaunchOut& out);
#ifdef PM2L_TIMING
int row_timing_copy(unsigned long long* host, int n);  // diagnostic build only
unsigned long long*& plan_timing_buffer();              // plan.cu: per-CTA entry/exit
#endif
int launch_grid_all_curves(const TablesDev& t, const GridDev& g, double* workspace,
                           double* out, void* stream);
// Query log2 sources of the explicit-descriptor mode: the per-device libm
// table for coordinates < lut_n, else a caller-given sorted (coordinate,
// libm log2) extension (host-computed; n_ext may be 0).
struct LogSource {
  const double* lut = nullptr;
  int64_t lut_n = 0;
  const uint32_t* ext_coord = nullptr;
  const double* ext_log = nullptr;
  int64_t n_ext = 0;
};
int launch_points(const TablesDev& t, const uint32_t* shapes, int64_t n, const LogSource& logs,
                  double* out_lat, int32_t* out_curve, uint32_t* out_waves, int8_t* out_match,
                  int32_t* out_record, double* out_dist, double* out_detail, void* stream);
int launch_points_curve(const TablesDev& t, const uint32_t* shapes, const int32_t* curves,
                        int64_t n, double* out_lat, uint32_t* out_waves, double* out_detail,
                        void* stream);
int launch_membound(const double* f, const int32_t* mid, int64_t n, const double* w,
                    const double* b, const double* floors, int64_t n_models, double* out,
                    uint8_t* floored, double* out_raw, void* stream);
int launch_nan_scan(const double* v, int64_t n, unsigned long long* first, void* stream);
int64_t store_encode_workspace(int64_t n);
int launch_store_encode(const double* lat, int64_t n, const uint64_t* B, const uint64_t* M,
                        int64_t nM, const uint64_t* N, int64_t nN, const uint64_t* K, int64_t nK,
                        void* workspace, uint8_t* records, int64_t* count, void* stream);
int launch_store_lookup(const uint8_t* records, int64_t n_rec, const uint64_t* const axes[4],
                        const int64_t lens[4], const uint64_t* queries, int64_t nq, double* out,
                        unsigned long long* first_missing, void* stream);
int launch_grid_error(const int64_t* dims, const double* thrs, int ns, int64_t stride,
                      const double* truth, const int64_t* scan_off, const double* rational,
                      double* out_err, int64_t* out_arg, void* stream);
int launch_partition(const double* la, const double* lb, int64_t n, const double* transfer,
                     double* sa, double* sb, double* bn, int64_t* best, void* stream);
int launch_segment_fsum(const double* v, const int64_t* off, int64_t nseg, double* out,
                        void* stream);

}  // namespace pm2l
